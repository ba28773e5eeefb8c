"""bench.py --gpus N self-launch on CPU: without a torchrun environment it re-runs itself under
torch.distributed.run with N ranks; the --selftest workload exercises the same launcher, barriers
and max-over-ranks timing with gloo (no GPU), so the N-rank plumbing is covered here."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("gpus", [1, 2])
def test_bench_self_launches_n_ranks(gpus):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                              "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--selftest", "--gpus", str(gpus),
                          "--steps", "3"], capture_output=True, text=True, env=env, timeout=280, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["selftest"] and rec["n_gpus"] == gpus
    assert len(rec["per_rank_ms"]) == gpus
    assert rec["ms_per_step"] == pytest.approx(max(rec["per_rank_ms"]))
