# raster parity tests, then render timing A/B over an env knob on the given workloads
# usage: KNOB=NAR_RENDER_MIXED VALS="0 1" WLS="c4 c2" bash scripts/gpu_render_env_ab.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_raster_gpu.py tests/test_parity_configs_gpu.py tests/test_preprocess_gpu.py -x -q --timeout 900 > gpurun_out/t_rab.log 2>&1; echo "raster tests rc=$?"; tail -2 gpurun_out/t_rab.log
for w in ${WLS:-c4 c2}; do for v in ${VALS:-0 1}; do
  env $KNOB=$v timeout 600 python bench.py --workload $w --steps 10 --warmup 5 --no-e2e --no-cpu --no-gsplat --no-pipeline --no-parity > gpurun_out/eab_${w}_$v.json 2> gpurun_out/eab_${w}_$v.err
  python - "$w" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/eab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "render_ms", round(d.get("render_ms", 0), 3), "frac", round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e)
PY
done; done
