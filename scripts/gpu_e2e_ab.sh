# rasterize() end-to-end A/B over an env knob (C2, e2e leg only)
# usage: KNOB=NAR_ZERO_COPY_OUT VALS="0 1 0 1" bash scripts/gpu_e2e_ab.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
i=0
for v in ${VALS:-0 1}; do
  env $KNOB=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-gsplat --no-pipeline --no-parity --no-morton > gpurun_out/e2e_$i.json 2> gpurun_out/e2e_$i.err
  python - "$i" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/e2e_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(sys.argv[2], "value", round(d["value"], 1), "e2e", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in e.items() if not isinstance(v, (dict, list))})
except Exception as ex:
    print(sys.argv[2], "failed", ex)
PY
  i=$((i+1))
done
