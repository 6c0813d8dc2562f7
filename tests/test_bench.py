"""bench.py contract: both arms print one JSON line on the SAME workload
(config identical, so the driver's ratio is same-config), the reference arm
runs the unmodified reference on the CPU, our arm carries roofline,
cpu_baseline and e2e (test_bench.cpp:141-177 checks the reference's own
report the same way)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, requires_ref


def _run(args, timeout=900, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@requires_ref
def test_reference_arm_same_workload_cpu():
    ref = _run(["--impl", "reference", "--points", "3e4", "--steps", "5", "--warmup", "3",
                "--check-targets", "200"])
    assert ref["impl"] == "reference" and ref["value"] > 0 and ref["unit"] == "Mpoints/s"
    assert ref["steps"] == 3 and ref["warmup"] == 1        # capped (--ref-steps), reported
    assert ref["config"]["n_points"] == 30000 and ref["config"]["workload"].startswith("laplace3d cube")
    assert ref["cpu_baseline"]["kind"] == "reference" and ref["cpu_baseline"]["cores"] >= 1
    assert ref["e2e"]["h2d_bytes_per_step"] == 0
    assert ref["relerr_vs_direct"] <= 1e-5
    sys.path.insert(0, ROOT)
    import bench
    # our arm's config for the same flags is the identical dict
    old = sys.argv
    try:
        sys.argv = ["bench.py", "--points", "3e4"]
        ours = bench.workload_config(bench.parse())
    finally:
        sys.argv = old
    assert ours == ref["config"]


@pytest.mark.gpu
@requires_ref
def test_bench_line_single_gpu_small():
    out = _run(["--points", "2e5", "--steps", "3", "--warmup", "3", "--cpu-reps", "1",
                "--check-targets", "200"])
    assert out["value"] > 0 and out["n_gpus"] == 1 and out["gpu_launches"] > 0
    assert out["roofline"]["bound"] == "fp64" and out["roofline"]["peak"] > 0
    assert out["e2e"]["h2d_bytes_per_step"] == 2e5 * 8 and out["e2e"]["matches_device_result"]
    assert out["relerr_vs_cpu_ref"] <= 1e-12
    cb = out["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] > 0 and len(cb["times_s"]) == 1
    assert "Model name" in cb["host"] or "CPU(s)" in cb["host"]
    assert out["clocks"]["sm_mhz"] is None or out["clocks"]["sm_mhz"] > 0


@pytest.mark.gpu
def test_bench_line_multi_device_one_process():
    out = _run(["--points", "2e5", "--steps", "3", "--warmup", "3", "--devices", "0,0,0,0",
                "--cpu", "off", "--check-targets", "200"])
    assert out["value"] > 0 and "sharded over devices [0, 0, 0, 0]" in out["parallelism"]
    assert out["relerr_vs_direct"] <= 1e-4 and out["e2e"]["matches_device_result"]
