"""Per-tile timeline of CTA 0 of one tensor-core gated conv (NAR_TC_DEBUG bit 3):
python scripts/tc_trace.py [--cin 16 --cout 16 --h 1088 --w 1920].  Prints, per
tile, cycles relative to the first stamp: MMA wait for TMEM-empty, per-chunk
full-wait and issue end, epilogue (warp 1) start/end, producer empty wait."""
import argparse
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cin", type=int, default=16)
    ap.add_argument("--cout", type=int, default=16)
    ap.add_argument("--h", type=int, default=1088)
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--debug", type=int, default=8)
    a = ap.parse_args()
    os.environ["NAR_TC_DEBUG"] = str(a.debug)
    import numpy as np
    import torch

    from paper_2407_19097_b200 import _lib
    from paper_2407_19097_b200.neural import gated_conv

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    x = torch.rand((a.h, a.w, a.cin), device=dev)
    fw = rng.normal(0, 0.1, (3, 3, a.cin, a.cout)).astype(np.float32)
    gw = rng.normal(0, 0.1, (3, 3, a.cin, a.cout)).astype(np.float32)
    b = np.zeros(a.cout, np.float32)
    for _ in range(3):
        gated_conv(x, fw, b, gw, b)
    torch.cuda.synchronize()
    n = 16 * 16
    buf = (ctypes.c_ulonglong * n)()
    lib = _lib.load()
    assert lib.nar_debug_tc_trace(buf, n) == 0
    t = np.array(buf, dtype=np.int64).reshape(16, 16)
    t0 = t[0][t[0] > 0].min()
    names = {0: "mma>tempty", 1: "tempty ok", 2: "full0", 3: "issued0", 4: "full1", 5: "issued1",
             6: "full2", 7: "issued2", 10: "epi start", 11: "epi end", 12: "prod>empty", 13: "prod ok"}
    cols = [c for c in names if (t[:, c] > 0).any()]
    print("tile " + " ".join(f"{names[c]:>10s}" for c in cols))
    for i in range(16):
        if not (t[i] > 0).any():
            break
        print(f"{i:4d} " + " ".join(f"{(t[i, c] - t0) if t[i, c] else -1:10d}" for c in cols))


if __name__ == "__main__":
    main()
