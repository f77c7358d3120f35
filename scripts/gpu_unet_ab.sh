# U-Net A/B over env knobs: tests once, then event timing + a launch list per setting
# usage: AB="NAR_TC_SLIDE_BLOCKS=1 NAR_TC_SLIDE_BLOCKS=2+NAR_TC_PDL=0" bash scripts/gpu_unet_ab.sh  (+ joins settings)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_unet_gpu.py tests/test_parity_configs_gpu.py::test_unet_c4_frame_vs_f32_oracle -x -q --timeout 300 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
i=0
for kv in $AB; do
  echo "== $kv"; env $(echo $kv | tr "+" " ") timeout 120 python scripts/prof_unet.py --frames 6 2>&1 | tail -3
  env $(echo $kv | tr "+" " ") timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ab_$i.csv python scripts/prof_unet.py --frames 1 > /dev/null 2>&1
  i=$((i+1))
done
