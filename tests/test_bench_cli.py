"""bench.py's reference arm (the CPU oracle port timed on the host)
as the driver launches it: one JSON line with the contract's keys, and -- run
with a library override that does not exist -- proof that the arm never maps
the product's CUDA library (`vs_reference` was void because it did)."""

import json
import os
import subprocess
import sys

from conftest import REPO


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, capture_output=True, text=True,
                         env=env, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line_and_no_product_library():
    line = _run(["--impl", "reference", "--workload", "C0", "--steps", "1", "--warmup", "0"],
                {"CGL_LIB_OVERRIDE": "/nonexistent/libcglb200.so", "CUDA_VISIBLE_DEVICES": ""})
    assert line["impl"] == "reference" and line["metric"] == "grid-point-steps/s" and line["unit"] == "gp-steps/s"
    assert line["higher_is_better"] is True and line["value"] > 0 and line["steps"] == 1
    assert line["config"]["workload"].startswith("C0") and line["config"]["scheme"] == "strang"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_under_torchrun_env_only_rank0_prints():
    """Ranks other than 0 of a torchrun launch exit 0 without work or output."""
    env = {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1", "CGL_LIB_OVERRIDE": "/nonexistent/libcglb200.so"}
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--workload", "C0",
                          "--steps", "1", "--warmup", "0", "--gpus", "2"], capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
