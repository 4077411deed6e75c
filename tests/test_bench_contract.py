"""bench.py's JSON line: the reference arm (the oracle, timed on the host) on CPU, and the
GPU arm on a small grid (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", "--config", "C2", "--n", "256",
                        "--cpu-crop", "96"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["unit"] == "Gcell-updates/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["host"]["nproc"] >= 1 and "cpu_model" in d["cpu_baseline"]["host"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the same workload as our arm's line (the crop is the per-step sample)
    assert d["config"]["workload"] == "C2" and d["config"]["grid"] == [256, 256]
    assert "96x96" in d["config"]["sample"]


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """bench.py's own arm on a small grid: the keys the driver reads, a roofline object for
    the fused kernel, the clock sample, e2e through the C-ABI with host buffers, the oracle's
    CPU baseline and a kernel-launch count."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C2", "--n",
                        "1024", "--steps", "5", "--warmup", "3", "--cpu-crop", "96",
                        "--cpu-steps", "2", "--e2e-steps", "5"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["scaling"] == "strong" and d["higher_is_better"] is True
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s" and 0 < ro["frac"] < 1
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    assert d["gpu_launches"] >= 5 * 2  # fused + ctrl per step
    assert len(d["timed_runs_ms"]) == 3 and d["ms_per_step"] * 5 in d["timed_runs_ms"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("halo", ["push", "nccl"])
def test_gpu_arm_dist_path_under_torchrun(halo):
    """The multi-GPU code path of bench.py end to end with one rank under torchrun
    (DESIGN.md 9): torch.distributed NCCL group, the all-gathered balanced bounds, the
    NCCL-id broadcast, csph_create_dist_rows, the steps of either halo transport (push: the
    strip launched whole; nccl: the split launches + send/recv on the comm stream) with the
    max allreduce, and the e2e leg through csph_set_state_rows/get_state_rows."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--dist", "--config", "C5", "--grid-n", "1024",
           "--steps", "4", "--warmup", "3", "--repeats", "1", "--no-cpu-baseline",
           "--e2e-steps", "4", "--tile-rows", "64", "--halo", halo]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip().startswith("{")][-1])
    assert d["value"] > 0 and d["n_gpus"] == 1
    assert d["config"]["partition"]["bounds"] == [0, 1024]
    assert d["config"]["parallelism"].startswith("row strips")
    # per step: the tile-order sort, ctrl and the step kernel -- one rank has no neighbour,
    # so a pushing rank launches its strip whole; the send/recv path launches the edge tile
    # rows and the interior (16 tile rows of 64)
    assert d["gpu_launches"] == 4 * (3 if halo == "push" else 5)
    assert d["e2e"]["value"] > 0
