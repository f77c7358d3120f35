cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./scripts/rcp_precision > gpurun_out/rcp.log 2>&1
timeout 600 python -m pytest tests/test_raster_gpu.py -x -q --timeout 300 > gpurun_out/t_raster.log 2>&1; echo "raster rc=$?"
for a in "" "--no-hiz" "--sorted"; do echo "== $a"; python scripts/prof_render.py --frames 3 $a 2>&1 | tail -1; done > gpurun_out/p_render.log 2>&1
