cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_raster_gpu.py -x -q --timeout 200 > gpurun_out/t_raster.log 2>&1; echo "raster rc=$?"
python scripts/prof_render.py --frames 5 > gpurun_out/p_render.log 2>&1; echo "prof rc=$?"
python scripts/prof_render.py --frames 3 --sorted > gpurun_out/p_sorted.log 2>&1
python - > gpurun_out/h2d.log 2>&1 <<'PY'
import torch, time
for n in [1<<28, 1<<30]:
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device='cuda')
    d.copy_(h); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
    print('H2D', n, n/a.elapsed_time(b)/1e6, 'GB/s')
    a.record(); h.copy_(d, non_blocking=True); b.record(); torch.cuda.synchronize()
    print('D2H', n, n/a.elapsed_time(b)/1e6, 'GB/s')
PY
