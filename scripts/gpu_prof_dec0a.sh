cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
U="python scripts/prof_unet.py --frames 1"
timeout 120 $U > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc -s ${SKIP:-16} -c 1 -o gpurun_out/${NAME:-dec0a}_full -f $U > gpurun_out/ncu_dec0a.log 2>&1; echo "rc=$?"
