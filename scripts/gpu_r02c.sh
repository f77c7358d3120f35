# round 2 re-entry: full GPU suite, smoke, default bench + reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rs > gpurun_out/t_all.log 2>&1; echo "all rc=$?" >> gpurun_out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt; tail -5 gpurun_out/t_all.log; tail -c 2500 gpurun_out/bench_c2.log; tail -c 800 gpurun_out/bench_ref.log
