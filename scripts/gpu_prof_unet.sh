cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_unet_gpu.py -x -q --timeout 120 > gpurun_out/t_unet.log 2>&1; echo "unet rc=$?"
CMD="python scripts/prof_unet.py --frames 1"
timeout 120 python scripts/prof_unet.py --frames 5 > gpurun_out/u_t.log 2>&1
timeout 120 $CMD > gpurun_out/u_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/u_launch.csv $CMD > /dev/null 2>&1
echo done
