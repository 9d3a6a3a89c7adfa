"""bench.py's own multi-GPU launcher on CPU (gloo): `--gpus N` without a torchrun environment
re-launches bench.py as N ranks; the host logic (contiguous env slices of SURVEY §8(e), the
max-over-ranks timing reduction, the gather of per-env hashes and their comparison with a
single-process computation on rank 0) runs end to end with --launcher-selftest, which hashes the
synthetic per-env inputs in place of rendered frames (no GPU here)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--launcher-selftest", *args],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [2, 3])
def test_self_launch_weak_scaling(gpus):
    r = _run("--gpus", str(gpus), "--config", "T2", "--steps", "2", "--warmup", "1")
    assert r["n_gpus"] == gpus
    B = 2   # T2 envs per rank
    assert r["slices"] == [[k * B, (k + 1) * B - 1] for k in range(gpus)]
    assert r["config"]["frames_per_step"] == gpus * B
    assert r["max_over_ranks"] == pytest.approx(0.001 * gpus)
    assert r["env_hash_check"] == {"envs_checked": gpus * B, "mismatches": 0}


def test_self_launch_strong_scaling_contiguous_slices():
    r = _run("--gpus", "3", "--config", "C2", "--scaling", "strong", "--steps", "1", "--warmup", "0")
    assert r["n_gpus"] == 3
    sl = r["slices"]
    assert sl[0][0] == 0 and sl[-1][1] == 63
    assert all(sl[k][1] + 1 == sl[k + 1][0] for k in range(2))
    assert r["config"]["frames_per_step"] == 64
    assert r["env_hash_check"]["mismatches"] == 0 and r["env_hash_check"]["envs_checked"] == 12


def test_single_process_is_one_rank():
    r = _run("--config", "T2", "--steps", "1", "--warmup", "0")
    assert r["n_gpus"] == 1 and r["slices"] == [[0, 1]]
