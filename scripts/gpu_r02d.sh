# U-Net PDL A/B, MUFU microbenchmark, full capture of the 18 convs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/rc_d.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mufu_bench scripts/mufu_bench.cu && ./scripts/mufu_bench > gpurun_out/mufu.txt 2>&1; echo "mufu rc=$?" >> gpurun_out/rc_d.txt
timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_parity_configs_gpu.py::test_unet_c4_frame_vs_f32_oracle -x -q --timeout 300 > gpurun_out/t_unet.log 2>&1; echo "unet tests rc=$?" >> gpurun_out/rc_d.txt
for pdl in 0 1 0 1; do echo "PDL=$pdl" >> gpurun_out/unet_pdl.txt; NAR_TC_PDL=$pdl timeout 120 python scripts/prof_unet.py --frames 20 2>&1 | tail -4 >> gpurun_out/unet_pdl.txt; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/unet_layers.csv python scripts/prof_unet.py --frames 1 > /dev/null 2>&1; echo "ncu list rc=$?" >> gpurun_out/rc_d.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc --launch-skip 36 --launch-count 18 -o gpurun_out/r02_unet_full -f python scripts/prof_unet.py --frames 1 > gpurun_out/ncu_unet_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/rc_d.txt
cat gpurun_out/rc_d.txt gpurun_out/mufu.txt gpurun_out/unet_pdl.txt; tail -3 gpurun_out/t_unet.log
