# quick U-Net iteration: parity tests, event timing, per-layer launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_parity_configs_gpu.py::test_unet_c4_frame_vs_f32_oracle tests/test_bounds_gpu.py -x -q --timeout 300 2>&1 | tail -4
timeout 120 python scripts/prof_unet.py --frames 10 2>&1 | tail -3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for d in ${DEBUG_MODES:-0}; do
  NAR_TC_DEBUG=$d timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/unet_it_d$d.csv python scripts/prof_unet.py --frames 1 > /dev/null 2>&1; echo "ncu d$d rc=$?"
done
