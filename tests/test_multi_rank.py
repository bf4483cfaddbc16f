"""N>1 plumbing of bench.py on CPU (gloo, world_size 2): process-group init from
torchrun-style env, barrier, max-over-ranks timing, and rank-0-only reporting of
the reference arm, the split of the C5 microbenchmark batch across ranks, and the subtree
ownership plan of the distributed factorization (the factorization itself needs
GPUs: tests/test_gpu_dist.py)."""
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


PLAN_WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2102_09878_b200 as P
from paper_2102_09878_b200.problems import tall_grid, knn_geometric
dist.init_process_group("gloo", init_method="env://")
ws, rank = dist.get_world_size(), dist.get_rank()
g = ws.bit_length() - 1
for prob in (tall_grid(64), knn_geometric(4096, seed=3, levels=8)):
    plan = P.rank_plan(prob.A, ws, levels=prob.levels, coords=prob.coords)   # host only, every rank
    own = torch.from_numpy(plan["owner"].astype(np.int64))
    allo = [torch.zeros_like(own) for _ in range(ws)]
    dist.all_gather(allo, own)
    assert all(torch.equal(a, own) for a in allo), "ranks disagree on the ownership map"
    o = plan["owner"]
    assert o.min() >= 0 and o.max() < ws
    par, lev = plan["tree_parent"], plan["tree_level"]
    def subtree(v):  # left-to-right index of v's level-(g+1) ancestor (preorder ids: left child = parent + 1)
        if lev[v] <= g:
            return -1
        path = []
        while lev[v] > 1:
            path.append(0 if v == par[v] + 1 else 1)
            v = par[v]
        bits = path[::-1][:g]
        return int("".join(map(str, bits)) or "0", 2)
    node_sub = np.array([subtree(v) for v in range(len(par))])
    cn, cl = plan["cluster_node"], plan["cluster_level"]
    inside = node_sub[cn] >= 0
    # clusters inside a subtree belong to that subtree's rank, at every granularity
    assert np.array_equal(o[inside], node_sub[cn][inside])
    # the top g levels (pieces at granularity <= g) are gathered onto rank 0
    assert np.all(o[(~inside) & (cl <= g)] == 0)
    # every rank owns one whole subtree and the boundary pieces it borders first
    assert set(np.unique(o[inside]).tolist()) == set(range(ws))
    mine = int(np.sum(o == rank))
    tot = torch.tensor([mine], dtype=torch.int64)
    dist.all_reduce(tot)
    assert int(tot.item()) == len(o)
dist.barrier()
print(json.dumps({"rank": rank, "ok": True}))
dist.destroy_process_group()
'''


@pytest.mark.timeout(300)
@pytest.mark.parametrize("ws", [2, 4])
def test_subtree_ownership_plan_gloo(ws):
    """the subtree ownership map (include/spaqr_b200.h spqr_rank_plan, host only)
    computed independently on every rank of a gloo group agrees across ranks, gives each rank
    one whole level-(g+1) subtree, keeps every subtree's clusters on its rank and gathers the
    top g levels onto rank 0."""
    port = free_port()
    procs = []
    for r in range(ws):
        env = dict(os.environ, ROOT=ROOT, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(ws), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", PLAN_WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=280) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
