"""Memory-safety evidence without compute-sanitizer (closed on the GPU pool):
the same workloads through the checked library (-DGANN_CHECKED: the kernels
test the bounds of their shared-memory and output writes on the device,
common.cuh GANN_CHECK) report no failed check and return the release
library's results bit for bit. Every kernel family runs: the start vertex,
the build's binned / tensor-core / chunked / warp re-prune kernels, the
back-edge group-by and merge, the three visited modes, ground truth, explicit
alpha_prune and group_by_key, and the config-0 build (R64 L128, 2% cap) with
searches up to L=832."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _run(case, lib):
    env = dict(os.environ)
    env.pop("GANN_LIB", None)
    if lib:
        env["GANN_LIB"] = lib
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "checked_case.py"), case], capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case", ["small", "c0"])
def test_checked_build_clean_and_identical(case):
    assert (ROOT / "paper_2305_04359_b200" / "libgann_checked.so").exists(), "build() makes the checked library"
    chk = _run(case, "libgann_checked.so")
    rel = _run(case, None)
    assert chk["checked_build"] == 1 and rel["checked_build"] == 0
    assert chk["failed_line"] == 0, f"bounds check failed at line {chk['failed_line']}"
    assert chk["out"] == rel["out"]
