"""Benchmark of the spaQR hot path on B200 (BASELINE.json metric: spaQR factor+solve
time, s; plus the batched front-QR roofline).

Workload (BASELINE.json configs[1], "C2"): 2D tall sparse least squares on a
512 x 512 grid (N = 262,144 unknowns, M = 2N rows), seeded synthetic data,
geometric nested dissection with 14 levels, sparsification tol 1e-2,
preconditioned CGLS to 1e-12.  One step = one spaqr factorization + one
preconditioned CGLS solve of that problem.

value    : factorize + solve time measured with CUDA events on the pipeline
           stream (A already scaled/permuted/partitioned on the host and
           uploaded — the reference times t_factorize and t_solve the same way,
           pipeline.cpp:55-61, solve.cpp:26,74).
e2e      : the same step through the C ABI from HOST buffers
           (spqr_pipeline_create + spqr_pipeline_solve): partition, upload of A
           and b, factorize, solve, download of x.
--impl reference : the reference's own sources (proj/src, unmodified) compiled
           against the in-repo Eigen API shim into oracle/_ref/libspaqr_ref.so
           (single-threaded, like the reference), timed on this box's host on the
           same problem; the CPU oracle restatement stands in if that .so is absent.
Multi-GPU (--gpus N under torchrun): independent replicas, one per GPU
("replicas only" in round 1), timed as the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

def config(ws):
    """The `config` object of both arms' JSON lines (identical keys and values)."""
    return {"workload": WORKLOAD, "N": 262144, "M": 524288, "levels": 14, "eps": 1e-2, "skip_levels": 3,
            "cgls_tol": 1e-12, "seed": 0,
            "parallelism": (f"subtree split over {ws} GPUs: the stages before the first scale_all run per rank on "
                            "its own subtree (top-separator fronts re-merged after every stage), then gathered "
                            "on rank 0 (spqr_pipeline_create_dist)") if ws > 1 else "1 GPU",
            "l2_flush": "256 MB write between steps (ours); the CPU arm has no device state"}


WORKLOAD = ("C2: 2D tall sparse LS, 512x512 grid, N=262144, M=524288, 5-point rows + 3-nnz random rows, "
            "geometric ND L=14, eps=1e-2, skip_levels=3, CGLS tol 1e-12 (seed 0)")
METRIC = "spaQR factor+solve time (s)"


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # N > 1 runs ONE factorization across the ranks (spqr_pipeline_create_dist): the ranks
    # share the host's cores during the split stages, then rank 0 works alone with all of them
    # (torchrun's OMP_NUM_THREADS=1 would serialise the host bookkeeping)
    if ws > 1:
        ncpu = len(os.sched_getaffinity(0))
        lws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
        os.environ.setdefault("SPQR_HOST_THREADS", str(max(1, (ncpu - 1) // lws)))
        os.environ.setdefault("SPQR_HOST_THREADS_ROOT", str(max(1, ncpu - 1)))
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if os.environ.get("BENCH_SAME_GPU"):  # functional check of the N > 1 path with one GPU: every
            local, backend = 0, "gloo"        # rank on cuda:0, collectives on the host (not a measurement)
        if backend == "nccl":
            torch.cuda.set_device(local)
            # the ranks read each other's values over CUDA IPC peer mappings; a node whose GPUs
            # cannot map one another's memory sends the values through the host transport instead
            # (every rank sees the same devices, so every rank decides the same way)
            n = min(lws, torch.cuda.device_count())
            if not all(torch.cuda.can_device_access_peer(i, j) for i in range(n) for j in range(n) if i != j):
                os.environ.setdefault("SPQR_DIST_HOST", "1")
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, v):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, in-process through
    NVML (a cheap query every 0.25 s; spawning nvidia-smi would steal host cores from the
    host-bound engine); falls back to nvidia-smi when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self._stop = threading.Event()
        self._t = None

    def _nvml_reader(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.device)
        bits = {"hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap}

        def read():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            return float(sm), float(mx), {k for k, v in bits.items() if r & v}
        return read

    def _smi_reader(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

        def read():
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            s = [x.strip() for x in out.split(",")]
            return float(s[0]), float(s[1]), {self.NAMES[i] for i in range(4)
                                              if len(s) > 2 + i and "Active" in s[2 + i] and "Not" not in s[2 + i]}
        return read

    def start(self):
        try:
            read = self._nvml_reader()
            read()
            self.source = "nvml"
        except Exception:
            read = self._smi_reader()
            self.source = "nvidia-smi"

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(read())
                except Exception:
                    pass
                self._stop.wait(0.25)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples])) if self.samples else []
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "source": getattr(self, "source", None)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(family):
    """Mean DRAM bytes (read + write) per launch of a kernel family over one C2 step, from the
    committed ncu launch list summary (profiles/ncu_traffic.json, tools/ncu_traffic.py)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            v = json.load(f).get(family)
        return v if isinstance(v, dict) else None
    except Exception:
        return None


def make_problem():
    from paper_2102_09878_b200.problems import tall_grid
    return tall_grid(512, seed=0)


def cpu_module():
    """The CPU implementation timed as the baseline: the reference's own sources built by
    oracle/Makefile.ref (kind "reference"), else the oracle restatement (kind "port")."""
    from oracle import ref
    if os.path.exists(ref.PATH):
        return ref, "reference"
    import oracle as O
    return O, "port"


def cpu_oracle_step(p, M=None):
    if M is None:
        M = cpu_module()[0]
    t0 = time.perf_counter()
    P = M.Pipeline(p.A, eps=p.eps, levels=p.levels, coords=p.coords)
    x, rep = P.solve(p.b)
    wall = time.perf_counter() - t0
    t = P.times()
    return t["t_factorize"] + rep["t_solve"], wall, rep["iterations"], t["t_partition"]


FP64_PEAK_TFLOPS = 37.1  # DMMA m8n8k4 on this pool's B200, tools/fp64_peak.cu -> profiles/r01_fp64_peak.txt


def microbench_shard(nb, ws, rank):
    """Rows of a batch owned by `rank`: contiguous, sizes differ by at most one (no exchange)."""
    base, rem = divmod(nb, ws)
    return base + (1 if rank < rem else 0)


def front_qr_microbench(local, ws=1, rank=0):
    """BASELINE config 5: batched front QR + Q^T on a 256-column neighbour block,
    through spqr_qr_apply_batched_dev (device buffers, CUDA events inside the call),
    best of 3 after one warm-up; FP64 TFLOP/s against the measured DMMA peak.
    With N ranks the batch is split across GPUs (independent fronts, no exchange;
    SURVEY 8(e)) and the time is the max over ranks."""
    import ctypes as C
    import torch
    import paper_2102_09878_b200 as P
    L = P.lib()
    rows = []
    for (m, n, nb) in ((128, 32, 4096), (512, 128, 1024), (4096, 1024, 64)):
        k = 256
        ntot = n + k
        mine = microbench_shard(nb, ws, rank)
        g = torch.Generator(device=f"cuda:{local}").manual_seed(1000 * rank)
        A0 = torch.randn(max(mine, 1), ntot, m, dtype=torch.float64, device=f"cuda:{local}", generator=g)
        tau = torch.empty(max(mine, 1), n, dtype=torch.float64, device=A0.device)
        sg = torch.empty(max(mine, 1), n, dtype=torch.float64, device=A0.device)
        info = torch.empty(max(mine, 1), dtype=torch.int32, device=A0.device)
        best = 1e30
        for r in range(4):
            A = A0.clone()
            torch.cuda.synchronize()
            barrier(ws)
            ms = C.c_float()
            if mine > 0:
                rc = L.spqr_qr_apply_batched_dev(mine, m, n, ntot, C.c_void_p(A.data_ptr()), C.c_void_p(tau.data_ptr()),
                                                 C.c_void_p(sg.data_ptr()), C.c_void_p(info.data_ptr()), C.byref(ms))
                if rc != 0:
                    raise RuntimeError("spqr_qr_apply_batched_dev failed")
            if r > 0:
                best = min(best, allmax(ws, ms.value))
        fl = (2 * m * n * n - 2 / 3 * n ** 3 + 4 * m * n * k - 2 * n * n * k) * nb
        by = 16.0 * m * ntot * nb
        rows.append({"shape": f"{m}x{n}+{k}", "batch": nb, "n_gpus": ws, "ms": round(best, 3),
                     "TFLOP/s": round(fl / best / 1e9, 2),
                     "frac_fp64": round(fl / best / 1e9 / (FP64_PEAK_TFLOPS * ws), 3),
                     "GB/s": round(by / best / 1e6, 1)})
        del A0, A
    # truncated CPQR (eps 1e-2) of one 256 x 256 interface per block, sigma_i = 0.8^i
    # (spqr_cpqr_batched_dev); bytes = single-pass ideal (read the block, write R)
    import numpy as np
    from paper_2102_09878_b200.problems import decaying_interface
    B = decaying_interface(256, 0.8, seed=0)
    cm = cn = 256
    Bt = torch.from_numpy(np.ascontiguousarray(B.T)).to(f"cuda:{local}")
    for nb in (4096, 1024, 64):
        mine = microbench_shard(nb, ws, rank)
        A0 = Bt.reshape(1, cn, cm).repeat(max(mine, 1), 1, 1).contiguous()
        rk = torch.zeros(max(mine, 1), dtype=torch.int32, device=A0.device)
        best = 1e30
        for r in range(4):
            A = A0.clone()
            torch.cuda.synchronize()
            barrier(ws)
            ms = C.c_float()
            if mine > 0:
                rc = L.spqr_cpqr_batched_dev(mine, cm, cn, C.c_void_p(A.data_ptr()), 1e-2, C.c_void_p(rk.data_ptr()),
                                             C.byref(ms))
                if rc != 0:
                    raise RuntimeError("spqr_cpqr_batched_dev failed")
            if r > 0:
                best = min(best, allmax(ws, ms.value))
        rr = int(rk[0].item())
        fl = (sum(4.0 * (cm - j) * (cn - j - 1) for j in range(rr)) + 2.0 * cm * cn) * nb
        by = (8.0 * cm * cn + 8.0 * rr * cn) * nb
        rows.append({"shape": "cpqr 256x256 eps 1e-2", "batch": nb, "n_gpus": ws, "rank": rr, "ms": round(best, 3),
                     "GFLOP/s": round(fl / best / 1e6, 1), "GB/s": round(by / best / 1e6, 1),
                     "frac_hbm": round(by / best / 1e6 / (load_peaks()[0] * ws), 4)})
        del A0, A
    return {"peak_tflops_per_gpu": FP64_PEAK_TFLOPS, "peak_source": "measured DMMA (tools/fp64_peak.cu)",
            "sharding": "batch split across ranks, no exchange; time = max over ranks", "shapes": rows}


def l2_flush(buf):
    if buf is not None:
        buf.add_(1.0)


def run_ours(args, ws, rank, local):
    import paper_2102_09878_b200 as P
    P.require_gpu()
    p = make_problem()
    flush = None
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
    except Exception:
        flush = None
    A = p.A
    h2d = A.indptr.nbytes + A.indices.nbytes + A.data.nbytes + p.b.nbytes + p.coords.nbytes
    d2h = 8 * A.shape[1]

    group = None
    if ws > 1:  # one factorization across the ranks; its transport is a gloo group on the host
        import torch.distributed as dist
        group = dist.new_group(backend="gloo")

    def step():
        t0 = time.perf_counter()
        g = P.Pipeline(A, eps=p.eps, levels=p.levels, coords=p.coords, device=local, dist_group=group)
        rep = None
        if g.is_root:
            x, rep = g.solve(p.b)
        wall = time.perf_counter() - t0
        t = g.times()
        return g, rep, (t["factorize_event_ms"] + t["solve_event_ms"]) / 1e3, wall

    for _ in range(args.warmup):
        l2_flush(flush)
        step()
    clocks = ClockSampler(local)
    barrier(ws)
    clocks.start()
    dev_t, e2e_t, last = [], [], None
    for _ in range(args.steps):
        l2_flush(flush)
        if flush is not None:
            import torch
            torch.cuda.synchronize()
        g, rep, dt, wall = step()
        dev_t.append(dt)
        e2e_t.append(wall)
        last = (g, rep)
    barrier(ws)
    ck = clocks.stop()
    step_values = [round(v, 4) for v in dev_t]
    value = allmax(ws, sum(dev_t) / len(dev_t))
    e2e = allmax(ws, sum(e2e_t) / len(e2e_t))
    g, rep = last
    if not g.is_root:  # this rank's subtree went to rank 0, which reports the step
        if not args.no_microbench:
            front_qr_microbench(local, ws, rank)
        return
    t = g.times()
    ks = g.kernel_stats()
    # W-sweep family (solve): device time from CUDA events around every sweep, also inside
    # the CGLS graphs; algorithmic bytes per sweep = 8 nnz(W) + 16 gathered entries
    ks["w_sweep"] = {"ms": t["sweep_ms"], "bytes": t["sweep_bytes"] * t["sweeps"],
                     "launches": int(t["sweeps"] * g.sweep_launches / 2)}
    dom = max(ks, key=lambda k: ks[k]["ms"])
    peak, peak_src = load_peaks()
    d = ks[dom]
    achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
    trf = ncu_traffic(dom)
    # front-QR roofline on its own (the kernel BASELINE.json names)
    q = ks["front_qr"]
    qr_gbs = q["bytes"] / (q["ms"] / 1e3) / 1e9 if q["ms"] > 0 else 0.0
    qr_tflops = t["qr_flops"] / (q["ms"] / 1e3) / 1e12 if q["ms"] > 0 else 0.0
    launches = int(g.launches + t["solve_launches"])
    fams = {k: {"device_ms": round(v["ms"], 3), "algorithmic_bytes": v["bytes"], "launches": v["launches"],
                "GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 2) if v["ms"] > 0 else None,
                "frac_hbm": round(v["bytes"] / (v["ms"] / 1e3) / 1e9 / peak, 5) if v["ms"] > 0 else None}
            for k, v in ks.items()}
    out = {
        "metric": METRIC, "value": round(value, 6), "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(value * 1e3, 3), "higher_is_better": False,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config(ws),
        "e2e": {"value": round(e2e, 6), "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "note": "spqr_pipeline_create+solve from host CSC/b to host x, incl. host partition "
                        f"({t['t_partition']:.3f}s)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 5),
                     "traffic": None if trf is None else trf.get("dram_bytes"),
                     "traffic_note": "mean DRAM bytes (read+write) per launch of the family over one C2 step "
                                     "(profiles/ncu_traffic.json, tools/ncu_traffic.py); compare with "
                                     "algorithmic_bytes_per_launch",
                     "algorithmic_bytes_per_launch": round(d["bytes"] / max(d["launches"], 1), 1),
                     "peak_source": peak_src,
                     "algorithmic_bytes": d["bytes"], "device_ms": round(d["ms"], 3), "launches": d["launches"],
                     "bytes_formula": "SURVEY 8(d): cpqr 8mn+8rn (discarded speculative rounds apart), "
                                      "front_qr 16m(n+k), w_sweep 8 nnz(W)+16 gathered, assemble 16/elem",
                     "cpqr_redundant_bytes": t["cpqr_redundant_bytes"],
                     "front_qr": {"GB/s": round(qr_gbs, 2), "frac_hbm": round(qr_gbs / peak, 4),
                                  "TFLOP/s": round(qr_tflops, 4), "launches": q["launches"],
                                  "device_ms": round(q["ms"], 3)},
                     "families": fams,
                     "kernel_ms": {k: round(v["ms"], 3) for k, v in ks.items()}},
        "step_values": step_values,
        "gpu_launches": launches,
        "clocks": ck,
        "solve": {"iterations": rep["iterations"], "converged": rep["converged"],
                  "residual": float(rep["residual_history"][-1]), "nW": g.nW, "nnz_w": g.nnz_w,
                  "factorize_event_s": round(t["factorize_event_ms"] / 1e3, 4),
                  "solve_event_s": round(t["solve_event_ms"] / 1e3, 4), "engine_syncs": g.syncs,
                  "elim_waves": t["elim_waves"], "w_solve_levels": t["w_solve_levels"],
                  "solve_plan_s": round(t["solve_plan_s"], 4), "solve_launches": t["solve_launches"]},
    }
    if ws > 1:
        out["distributed"] = {"exchange_s_rank0": round(g.dist_exchange_s, 4), "exchange_bytes_rank0": g.dist_bytes,
                              "host_threads": [os.environ.get("SPQR_HOST_THREADS"), os.environ.get("SPQR_HOST_THREADS_ROOT")],
                              "note": "each rank eliminates its subtree's clusters through the split stages; the "
                                      "top-separator fronts are re-merged after every stage; ranks > 0 then send "
                                      "their subtree to rank 0, which finishes; exchange bytes = host metadata + "
                                      "values read over peer memory (CUDA IPC); value = max over ranks"}
    if not args.no_microbench:
        try:
            mb = front_qr_microbench(local, ws, rank)
        except Exception as e:  # reported, never fatal for the headline line
            mb = {"error": str(e)[:200]}
        if rank == 0:
            out["front_qr_microbench"] = mb
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        M, kind = cpu_module()
        v, wall, iters, tpart = cpu_oracle_step(p, M)
        what = ("the reference's own proj/src compiled unmodified against the in-repo Eigen API shim "
                "(oracle/_ref)" if kind == "reference" else "the CPU oracle restatement (oracle/)")
        out["cpu_baseline"] = {"value": round(v, 4), "unit": "s", "cores": 1, "kind": kind,
                               "sample": f"full C2 problem, one factorize+solve (t_factorize + t_solve) of {what}, "
                                         f"single-threaded like the reference; {iters} CGLS iterations; "
                                         f"host partition {tpart:.2f}s excluded as in the value"}
    if rank == 0:
        print(json.dumps(out))


def run_reference(args, ws, rank):
    """The reference arm: the reference's CPU implementation (oracle/_ref, else the port) on the
    same C2 problem.  One step = one full factorize + solve (25-60 s on these hosts); the number
    of steps is capped so the run ends within ~4 minutes (a bounded sample of --steps)."""
    if rank != 0:
        return
    M, kind = cpu_module()
    p = make_problem()
    vals, walls, its = [], [], []
    budget = 240.0
    t_start = time.perf_counter()
    for _ in range(max(1, args.steps)):
        v, wall, iters, tpart = cpu_oracle_step(p, M)
        vals.append(v)
        walls.append(wall)
        its.append(iters)
        if time.perf_counter() - t_start + wall > budget:
            break
    v = sum(vals) / len(vals)
    what = ("reference proj/src (unmodified) built against the in-repo Eigen API shim, oracle/_ref"
            if kind == "reference" else "CPU oracle restatement (oracle/); oracle/_ref absent")
    out = {"metric": METRIC, "value": round(v, 4), "unit": "s", "n_gpus": ws, "steps": len(vals),
           "steps_requested": args.steps, "warmup": 0, "ms_per_step": round(v * 1e3, 1),
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference", "config": config(ws),
           "cpu_baseline": {"value": round(v, 4), "unit": "s", "cores": 1, "kind": kind,
                            "sample": f"full C2 problem per step, t_factorize + t_solve, {what}; "
                                      f"{len(vals)} of {args.steps} steps within a {budget:.0f} s budget; "
                                      "no warm-up (no device state)"},
           "e2e": {"value": round(v, 4), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "step_values": [round(x, 3) for x in vals], "iterations": its[-1]}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-microbench", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
