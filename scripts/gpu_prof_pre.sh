cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
C="python scripts/prof_render.py --frames 2"
timeout 300 $C > gpurun_out/pr.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/pre_launches.csv $C > /dev/null 2>&1; echo "list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:render_pre -s 5 -c 1 -o gpurun_out/pre_full -f $C > /dev/null 2>&1; echo "full rc=$?"
