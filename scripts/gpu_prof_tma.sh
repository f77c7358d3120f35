# full ncu capture (with source) of one dense exact-kernel pass of the C4 frame
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NAR_RENDER_EZ=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:render_tma_kernel --launch-skip 6 --launch-count 1 -o gpurun_out/c4_tma -f python bench.py --workload c4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-gsplat --no-pipeline --no-parity > gpurun_out/c4_tma.log 2>&1; echo "ncu rc=$?"
