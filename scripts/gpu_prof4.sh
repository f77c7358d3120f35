cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python scripts/prof_render.py --frames 1"
timeout 300 $CMD > gpurun_out/p_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:render_tma -s 3 -c 1 -o gpurun_out/prof_render6 -f $CMD > /dev/null 2>&1
