cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 400 python -m pytest tests/test_raster_gpu.py -x -q --timeout 200 > gpurun_out/t_raster.log 2>&1; echo "raster rc=$?" >> gpurun_out/rc.txt
timeout 400 python -m pytest tests/test_unet_gpu.py -x -q --timeout 200 > gpurun_out/t_unet.log 2>&1; echo "unet rc=$?" >> gpurun_out/rc.txt
timeout 500 python bench.py --workload c2 --steps 20 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
