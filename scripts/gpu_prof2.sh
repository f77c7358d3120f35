cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
CMD="python scripts/prof_render.py --frames 1"
timeout 300 $CMD > gpurun_out/p_plain.log 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_hiz.csv $CMD > /dev/null 2>&1
