# full ncu capture (with source) of the largest pre-test pass of the C2 frame
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:render_pre_kernel --launch-skip 13 --launch-count 1 -o gpurun_out/c2_pre -f python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu --no-gsplat --no-pipeline --no-parity --no-morton > gpurun_out/c2_pre.log 2>&1; echo "ncu rc=$?"
