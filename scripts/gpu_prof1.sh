cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_render.py --frames 5 --unet > gpurun_out/p_unet.log 2>&1
python scripts/prof_render.py --frames 3 --sorted > gpurun_out/p_sorted.log 2>&1
CMD="python scripts/prof_render.py --frames 2 --unet"
$CMD > gpurun_out/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_tma -s 1 -c 1 -o gpurun_out/prof_render -f $CMD > gpurun_out/ncu_render.log 2>&1 ; \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
