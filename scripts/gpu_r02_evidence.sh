# round-2 evidence pass: full GPU suite, smoke, bench lines (default + c4/c3/c5/nar1b + reference
# arm), launch list of the default command, render L2 counters, U-Net per-layer probe
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/rc_ev.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_ev.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/ev_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/rc_ev.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc_ev.txt
timeout 900 python bench.py > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err; echo "bench rc=$?" >> gpurun_out/rc_ev.txt
for w in c4 c3 c5 nar1b; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-gsplat > gpurun_out/ev_bench_$w.json 2> gpurun_out/ev_bench_$w.err; echo "bench $w rc=$?" >> gpurun_out/rc_ev.txt
done
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err; echo "ref rc=$?" >> gpurun_out/rc_ev.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-gsplat --no-parity > gpurun_out/ev_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/rc_ev.txt
bash scripts/gpu_render_prof.sh > gpurun_out/ev_rprof.log 2>&1; echo "rprof rc=$?" >> gpurun_out/rc_ev.txt
DEBUG_MODES="0 3 5 6" bash scripts/gpu_unet_iter.sh > gpurun_out/ev_unet.log 2>&1; echo "unet rc=$?" >> gpurun_out/rc_ev.txt
cat gpurun_out/rc_ev.txt; tail -3 gpurun_out/ev_tests.log; tail -1 gpurun_out/ev_smoke.log; cat gpurun_out/ev_unet.log | tail -6
