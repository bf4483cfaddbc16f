"""N>1 plumbing of bench.py on CPU (gloo, world_size 2): process-group init from
torchrun-style env, barrier, max-over-ranks timing, and rank-0-only reporting of
the reference arm, and the split of the C5 microbenchmark batch across ranks.  The C2
factorization is "replicas only"."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["ROOT"])
import bench
ws, rank, local = bench.dist_init()
assert ws == 2 and rank == int(os.environ["RANK"])
bench.barrier(ws)
v = bench.allmax(ws, 1.5 + rank)          # per-rank step time
assert v == 2.5, v
import torch, torch.distributed as dist
# the C5 microbenchmark batch is split across ranks with no overlap and nothing dropped
for nb in (4096, 1024, 64, 3):
    t = torch.tensor([bench.microbench_shard(nb, ws, rank)], dtype=torch.int64)
    dist.all_reduce(t)
    assert int(t.item()) == nb, (nb, int(t.item()))
# rank != 0 must not run the CPU reference arm
class A: steps = 1; warmup = 0
if rank != 0:
    bench.run_reference(A(), ws, rank)     # returns immediately, no output
dist.barrier()
print(json.dumps({"rank": rank, "max": v}))
dist.destroy_process_group()
'''


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(180)
def test_two_rank_gloo_max_over_ranks(tmp_path):
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, ROOT=ROOT, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=170) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    got = sorted(o.strip().splitlines()[-1] for o, _ in outs)
    assert '"max": 2.5' in got[0] and '"max": 2.5' in got[1]
