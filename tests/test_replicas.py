"""N > 1 path of bench.py on CPU (gloo, world_size 2).

The factorization does not shard ("replicas only"): every rank
factors and solves its own copy; the only collectives are the barrier and
the max-over-ranks reduction of the step time.  These tests run that logic
with two gloo processes, and check that the reference arm does no work on
ranks other than 0.
"""

import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import torch.distributed as dist
import bench
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dist.barrier()
ms = bench.reduce_max(10.0 + 5.0 * rank, dist, "cpu")
rate = bench.whole_job_rate(1.0e9, world, ms)
print(json.dumps({{"rank": rank, "ms": ms, "rate": rate}}), flush=True)
dist.destroy_process_group()
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(code, world=2, extra_env=None):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.update(extra_env or {})
        procs.append(subprocess.Popen([sys.executable, "-c", code], env=env, cwd=ROOT,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=120)
        except subprocess.TimeoutExpired:
            p.kill()
            raise
        assert p.returncode == 0, e
        outs.append(o)
    return outs


def test_max_over_ranks_gloo():
    import json
    outs = _launch(WORKER.format(root=ROOT))
    recs = [json.loads(o.strip().splitlines()[-1]) for o in outs]
    assert all(r["ms"] == 15.0 for r in recs)
    # 2 ranks x 1e9 units over the slowest rank's 15 ms
    assert all(abs(r["rate"] - 2e9 / 0.015) < 1e-3 * r["rate"] for r in recs)


def test_reference_arm_idle_on_nonzero_rank():
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import bench;"
            "sys.argv=['bench.py','--impl','reference','--gpus','2'];"
            "bench.main()")
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == ""


@pytest.mark.parametrize("world", [2])
def test_whole_job_rate_is_weak_scaling(world):
    import bench
    assert bench.whole_job_rate(3.0, world, 1000.0) == 3.0 * world
