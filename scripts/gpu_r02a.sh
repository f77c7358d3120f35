# round 2, first GPU pass: new parity tests, sanitizer, the full suite, bench (ours + reference)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out; rm -f gpurun_out/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 900 python -m pytest tests/test_parity_configs_gpu.py tests/test_integration_patch_gpu.py tests/test_unet_gpu.py -x -q --timeout 600 -rs > gpurun_out/t_new.log 2>&1; echo "new rc=$?" >> gpurun_out/rc.txt
timeout 1200 python -m pytest tests/test_sanitizer_gpu.py -q --timeout 1500 > gpurun_out/t_san.log 2>&1; echo "san rc=$?" >> gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 600 --deselect tests/test_sanitizer_gpu.py > gpurun_out/t_all.log 2>&1; echo "all rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt; tail -3 gpurun_out/t_new.log; tail -3 gpurun_out/t_san.log; tail -3 gpurun_out/t_all.log; tail -c 1500 gpurun_out/bench_c2.log; tail -c 600 gpurun_out/bench_ref.log
