"""compute-sanitizer over the path's kernels (the reference
argues race-freedom by construction, include/graphann/graph.hpp:12-15; here
the warp-synchronous merges and the block-level prune phases are checked).

racecheck (shared-memory hazards) and synccheck (barrier / warp-sync misuse)
run over a small build + search that launches every kernel family; memcheck
runs over the config-0 build (100k x 128 u8, R64 L128, 2% cap)."""
import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and Path(p).exists():
            return p
    pytest.fail("compute-sanitizer not found")


@pytest.mark.parametrize("tool,case", [("racecheck", "small"), ("synccheck", "small"), ("memcheck", "small"),
                                       ("memcheck", "c0")])
def test_sanitizer_clean(tool, case):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, str(ROOT / "tools" / "sanitize_case.py"), case]
    env = dict(os.environ, PYTHONUNBUFFERED="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"sanitizer_{tool}_{case}.log").write_text(out)
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case done" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
