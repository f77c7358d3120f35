# U-Net per-layer probe: event timing, launch lists under NAR_TC_DEBUG
# (0 = normal, 1 = no epilogue math/stores, 2 = no MMAs, 3 = neither), and one
# --set full capture of every conv of a 1920x1088 forward.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python scripts/prof_unet.py --frames 10 2>&1 | tail -3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for d in 0 1 2 3; do
  NAR_TC_DEBUG=$d timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/unet_d$d.csv python scripts/prof_unet.py --frames 1 > /dev/null 2>&1; echo "ncu d$d rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc --launch-skip 36 --launch-count 18 -o gpurun_out/r02_unet_full -f python scripts/prof_unet.py --frames 1 > gpurun_out/ncu_unet_full.log 2>&1; echo "ncu full rc=$?"
