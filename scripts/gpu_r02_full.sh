# round-2 `ncu --set full` captures of the dominant kernels (one launch each):
# C2's last pre-test pass, C4's last dense (exact) pass, and the dec0a / enc1b convs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-gsplat --no-pipeline --no-parity --no-morton"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:render_pre_kernel --launch-skip 19 --launch-count 1 -o gpurun_out/full_c2_pre -f $B > gpurun_out/full_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:render_tma_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/full_c4_tma -f $B --workload c4 > gpurun_out/full_c4.log 2>&1; echo "c4 rc=$?"
U="python scripts/prof_unet.py --frames 1"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc -s 16 -c 1 -o gpurun_out/full_dec0a -f $U > gpurun_out/full_dec0a.log 2>&1; echo "dec0a rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc -s 17 -c 1 -o gpurun_out/full_dec0b -f $U > gpurun_out/full_dec0b.log 2>&1; echo "dec0b rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gated_conv_tc -s 3 -c 1 -o gpurun_out/full_enc1b -f $U > gpurun_out/full_enc1b.log 2>&1; echo "enc1b rc=$?"
