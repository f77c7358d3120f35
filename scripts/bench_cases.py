"""Render-only bench over (env, args) cases on one GPU, one summary line per case.

usage: python scripts/bench_cases.py 'label|K=V,K2=V2|--workload c5 --points 250000000' ...
Each case runs `bench.py --steps 10 --warmup 5` without the e2e / cpu / gsplat /
pipeline / parity legs; raw lines land in gpurun_out/case_<label>.{json,err}.
"""

import json
import os
import subprocess
import sys

os.makedirs("gpurun_out", exist_ok=True)
for case in sys.argv[1:]:
    label, envs, args = (case.split("|") + ["", ""])[:3]
    env = dict(os.environ)
    for kv in filter(None, envs.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    cmd = [sys.executable, "bench.py", "--steps", "10", "--warmup", "5", "--no-e2e", "--no-cpu",
           "--no-gsplat", "--no-pipeline", "--no-parity"] + args.split()
    with open(f"gpurun_out/case_{label}.json", "w") as fo, open(f"gpurun_out/case_{label}.err", "w") as fe:
        rc = subprocess.run(cmd, env=env, stdout=fo, stderr=fe, timeout=900).returncode
    try:
        d = json.loads(open(f"gpurun_out/case_{label}.json").read().strip().splitlines()[-1])
        print(f"{label:28s} value {d['value']:7.1f} ms {d['ms_per_step']:.3f} "
              f"render_ms {d.get('render_ms', 0):.3f} frac {d['roofline']['frac']:.3f}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{label:28s} failed rc={rc} {e}", flush=True)
    stats = [l.strip() for l in open(f"gpurun_out/case_{label}.err") if l.startswith("nar pass")]
    if stats:
        print("   ", " | ".join(stats[-4:]), flush=True)
