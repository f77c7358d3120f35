# full GPU test suite + a default bench line (one gpurun call)
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/rc.txt
timeout 300 python -m pytest tests/test_preprocess_gpu.py -x -q --timeout 200 > gpurun_out/t_pre.log 2>&1; echo "pre rc=$?" >> gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_all.log 2>&1; echo "all rc=$?" >> gpurun_out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt; tail -3 gpurun_out/t_pre.log; tail -3 gpurun_out/t_all.log; tail -1 gpurun_out/bench.log
