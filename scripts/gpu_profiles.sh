# Evidence for profiles/: launch list (+DRAM bytes) of the bench command and
# one --set full capture of the render and of an L0 conv kernel.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 600 $B > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv $B > /dev/null 2> gpurun_out/ncu1.err
echo "launches rc=$?"
C="python scripts/prof_render.py --frames 2"
timeout 300 $C > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:render_pre -s 9 -c 1 -o gpurun_out/r01_render_full -f $C > /dev/null 2>&1
echo "render full rc=$?"
U="python scripts/prof_unet.py --frames 1"
timeout 300 $U > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc -s 1 -c 1 -o gpurun_out/r01_conv_full -f $U > /dev/null 2>&1
echo "conv full rc=$?"
