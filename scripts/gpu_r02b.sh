cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/rc2.txt
timeout 900 python -m pytest tests/test_bounds_gpu.py tests/test_parity_configs_gpu.py -x -q --timeout 600 > gpurun_out/t_new2.log 2>&1; echo "new rc=$?" >> gpurun_out/rc2.txt
bash scripts/gpu_unet_probe.sh > gpurun_out/unet_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/rc2.txt
for w in c4 c3 nar1b c5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-gsplat > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?" >> gpurun_out/rc2.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --workload nar1b --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_nar1b_trun.log 2>&1; echo "trun rc=$?" >> gpurun_out/rc2.txt
cat gpurun_out/rc2.txt; tail -3 gpurun_out/t_new2.log; cat gpurun_out/unet_probe.log | tail -8
