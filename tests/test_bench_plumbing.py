"""bench.py --gpus N without a launcher spawns N ranks itself (torchrun),
every rank joins the process group, the row shards (M not a multiple of N:
the last shard padded) are all-gathered, and rank 0 prints ONE JSON line
with n_gpus = the ranks that joined.  CPU / gloo: the per-shard compute is
the oracle, injected from tests/bench_plumbing.py (plumbing, not a bench)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_ranks_and_gathers(n):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env["OMP_NUM_THREADS"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                        "--steps", "2", "--warmup", "1", "--plumbing",
                        os.path.join(ROOT, "tests", "bench_plumbing.py")],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == n
    assert line["comm"]["nranks"] == n and line["comm"]["all_reduce_ok"]
    assert line["gathered_equals_reference"] is True
    shards = line["shard_rows"]
    assert shards[0][0] == 0 and shards[-1][1] == 1001
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    # one communicator line per rank on stderr
    assert r.stderr.count("communicator: nranks=%d" % n) == n
