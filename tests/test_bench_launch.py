"""bench.py's multi-GPU launch path on CPU (VERDICT r1 missing #1): without a
launcher, `bench.py --gpus N` re-runs itself under torchrun with N ranks,
every rank sees WORLD_SIZE == N, and the ranks own contiguous, disjoint,
covering layer blocks (the engine's partition, dist.owned_layers). --dry-run
swaps the GPU for a gloo rendezvous; the real run asserts WORLD_SIZE == --gpus."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*argv, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], cwd=ROOT,
                       env=e, capture_output=True, text=True, timeout=600)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return p.returncode, (json.loads(lines[-1]) if lines else None), p.stderr


@pytest.mark.parametrize("n", [2, 4])
def test_gpus_flag_spawns_n_ranks(n):
    rc, line, err = run_bench("--gpus", str(n), "--dry-run")
    assert rc == 0, err[-2000:]
    assert line["n_gpus"] == n == line["gpus_arg"]
    assert len(line["ranks"]) == n
    import bench
    for name, c in bench.CONFIGS.items():
        blocks = [r[name] for r in line["ranks"]]
        if any(isinstance(b, str) for b in blocks):  # partition refused (e.g. tiny at P > 4)
            assert all(isinstance(b, str) for b in blocks)
            continue
        total = c["n_enc"] + c["n_dec"]
        assert blocks[0][0] == 0 and blocks[-1][1] == total
        for a, b in zip(blocks, blocks[1:]):
            assert a[1] == b[0]


def test_world_size_mismatch_is_refused():
    rc, line, _ = run_bench("--gpus", "2", env={"WORLD_SIZE": "1", "RANK": "0"})
    assert rc == 1 and "WORLD_SIZE=1" in line["error"]


def test_single_rank_dry_run():
    rc, line, err = run_bench("--dry-run")
    assert rc == 0, err[-2000:]
    assert line["n_gpus"] == 1 and len(line["ranks"]) == 1
