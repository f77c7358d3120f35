cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_unet_gpu.py -x -q --timeout 200 2>&1 | tail -2
timeout 120 python scripts/prof_unet.py --frames 5 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/unet_launches.csv python scripts/prof_unet.py --frames 1 > /dev/null 2>&1; echo "ncu rc=$?"
