"""compute-sanitizer over every kernel family (memcheck, racecheck,
synccheck, initcheck).

The fused kernel has an 8-slot TMA / mbarrier ring, two-barrier shared-memory exchanges
and CTAs that leave early (HGS skipped / identity tiles); the multi-strip step overlaps
edge launches, peer-copy halos on a second stream and the interior launch.  Each case of
tools/sanitize_case.py runs a few steps on a small grid and checks its own parity, so a
clean sanitizer run is also a correct one.  racecheck covers shared-memory hazards
(the ring, the exchange rows), synccheck the barrier use, memcheck out-of-bounds and
misaligned accesses (TMA row copies near the padded row end), initcheck reads of
uninitialised global memory.

Opt-in (CSPH_RUN_SANITIZERS=1): the GPU pool this repo is tested on has closed
compute-sanitizer (its wrapper refuses to run: runs under it left GPUs needing a reset), so the
default `-m gpu` run skips these.  The last clean run of every case is committed in
profiles/r02_sanitizers.txt."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

CASES = {
    "memcheck": ["fused", "general", "staged", "strips", "fp32", "tiles"],
    "racecheck": ["fused", "general", "strips", "fp32"],
    "synccheck": ["fused", "general", "strips", "fp32"],
    "initcheck": ["fused", "staged", "strips"],
}


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2103_15196_b200 import build
    build.build()
    import synth
    synth.build()


@pytest.mark.parametrize("tool,case", [(t, c) for t, cs in CASES.items() for c in cs])
def test_compute_sanitizer(tool, case):
    if os.environ.get("CSPH_RUN_SANITIZERS") != "1":
        pytest.skip("opt-in (CSPH_RUN_SANITIZERS=1): compute-sanitizer is closed on this GPU "
                    "pool; last clean run in profiles/r02_sanitizers.txt")
    if not os.path.exists(CS):
        pytest.fail("compute-sanitizer not found")
    cmd = [CS, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "hazard"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), "--case", case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "case ok: " + case in out, out[-4000:]
    summary = "RACECHECK SUMMARY: 0 hazards" if tool == "racecheck" else "ERROR SUMMARY: 0 errors"
    assert summary in out, out[-4000:]
