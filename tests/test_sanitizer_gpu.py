"""compute-sanitizer over small calls of every device entry point
(scripts/sanitize_small.py): memcheck over all of them, racecheck over the
render + resolve kernels (the shared-memory rings).  The reference has no
bounds checks at all (_native.pyx:1 boundscheck=False); here out-of-bounds or
misaligned accesses and shared-memory hazards must be absent."""

import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SCRIPT = ROOT / "scripts" / "sanitize_small.py"


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool,what", [("memcheck", "all"), ("racecheck", "render")])
def test_sanitizer_clean(cuda, tool, what):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20",
           sys.executable, str(SCRIPT), what]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=ROOT)
    out = res.stdout + res.stderr
    log = ROOT / "gpurun_out" / f"sanitizer_{tool}.log"
    try:
        log.parent.mkdir(exist_ok=True)
        log.write_text(out)
    except OSError:
        pass
    assert "sanitize_small done" in out, out[-3000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", out)
    assert m is not None, out[-3000:]
    assert int(m.group(1)) == 0 and res.returncode == 0, out[-6000:]
