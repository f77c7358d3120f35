# render timing A/B over library variants (NAR_B200_LIB) on the given workloads
# usage: LIBS="base:paper_2407_19097_b200/libnar_b200.so w16:scripts/exp/w16.so" WLS="c4 c2" bash scripts/gpu_raster_ab.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for w in ${WLS:-c4 c2}; do for lv in $LIBS; do name=${lv%%:*}; lib=${lv#*:}
  NAR_B200_LIB=$PWD/$lib timeout 600 python bench.py --workload $w --steps 10 --warmup 5 --no-e2e --no-cpu --no-gsplat --no-pipeline --no-parity > gpurun_out/rab_${w}_$name.json 2> gpurun_out/rab_${w}_$name.err
  python - "$w" "$name" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/rab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "render_ms", round(d.get("render_ms", 0), 3), "frac", round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "failed", e)
PY
done; done
