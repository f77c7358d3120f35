cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
CMD="python scripts/prof_render.py --frames 1"
$CMD > gpurun_out/p_plain.log 2>&1 && ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_hiz.csv $CMD > /dev/null 2>&1
CMD2="python scripts/prof_render.py --frames 1 --no-hiz"
$CMD2 > gpurun_out/p_plain2.log 2>&1 && ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_nohiz.csv $CMD2 > /dev/null 2>&1
for a in "" "--no-hiz" "--sorted"; do python scripts/prof_render.py --frames 3 $a 2>&1 | tail -1; done > gpurun_out/p_t.log
