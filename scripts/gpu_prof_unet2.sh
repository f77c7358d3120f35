cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python scripts/prof_unet.py --frames 1"
timeout 120 $CMD > gpurun_out/u_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc -s 1 -c 1 -o gpurun_out/prof_conv -f $CMD > gpurun_out/ncu_conv.log 2>&1
echo done
