#!/usr/bin/env python
"""bench.py — the CUDASOM hot path on B200, one JSON line on rank 0.

A "step" is one pass of the whole hot path over
one synthetic c2 workload (BASELINE.json configs[1]): 20x20 hex map,
5,000 x 3,000 L2-normalised TF-IDF corpus, 100 epochs of online training
(T = 500,000 samples) from a seeded row init, then batch mapping of all
documents, QE + TE, and the U-matrix.  value = training samples/s over the
whole step, summed over ranks (each rank runs its own independent problem:
weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
  python bench.py --impl reference ...   # the oracle (CPU) on a bounded sample
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, bank_corpus  # noqa: E402

METRIC = "SOM training samples/sec and batch BMU-mapping docs/sec at 1/2/4/8 B200"
ALPHA0 = 0.1


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3"])
    p.add_argument("--epochs", type=int, default=None, help="override epochs (diagnostics only)")
    p.add_argument("--no-baseline", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--map-docs", type=int, default=200000, help="documents in the c5-shaped mapping leg (0 = skip)")
    p.add_argument("--c3-steps", type=int, default=20000, help="steps of the c3 training leg (0 = skip)")
    p.add_argument("--table3-steps", type=int, default=20000, help="steps per map of the Table 3 leg (0 = skip)")
    p.add_argument("--batch-epochs", type=int, default=10, help="epochs of the batch-SOM leg (0 = skip)")
    p.add_argument("--c4-steps", type=int, default=2000, help="steps of the c4 (neuron-sharded at N > 1) leg (0 = skip)")
    p.add_argument("--c4-docs", type=int, default=20000, help="documents of the c4 leg (replicated on every rank)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BENCH_ONE_DEVICE") == "1":   # test hook: every rank on cuda:0 (multi-rank plumbing check)
        local = 0
    return rank, world, local


class Clocks:
    """Sample nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def workload(cfg_name, seed, epochs_override):
    cfg = dict(CONFIGS[cfg_name])
    if epochs_override is not None:
        cfg["epochs"] = epochs_override
    C = bank_corpus(cfg["n"], cfg["d"], seed=seed)
    return cfg, C


def train_peak_tflops():
    """Peak of the training kernel's exact distance element (1 F2F.F64.F32 +
    DADD + DFMA = 3 flop): bound by the measured fp32->fp64 conversion rate
    (profiles/probe_fp64.json) x 148 SMs x max SM clock."""
    path = os.path.join(ROOT, "profiles", "probe_fp64.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return 3.0 * j["train_element_peak_per_s"] / 1e12, ("measured F2F.F64.F32 rate "
                                                            f"{j['f2f_per_clk_per_sm']}/clk/SM x 148 SMs x 1965 MHz "
                                                            "x 3 flop/element (profiles/probe_fp64.json)")
    return 3.0 * 16 * 148 * 1965e6 / 1e12, "nominal 16 F2F/clk/SM x 148 x 1965 MHz x 3 flop (no measurement file)"


def tf32_peak_tflops():
    """Dense TF32 peak: the measured bf16 cuBLAS peak (MEASURED_PEAKS.json,
    burst) x the nominal tf32/bf16 ratio 1.1/2.25 (B200_PROFILING.md)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        return bf16 * 1.1 / 2.25, f"measured bf16 {bf16} TFLOP/s x 1.1/2.25 (MEASURED_PEAKS.json)"
    return 1590.0 * 1.1 / 2.25, "fallback bf16 1590 TFLOP/s x 1.1/2.25 (B200_PROFILING.md)"


def conv_peak_per_s():
    """fp32 -> fp64 conversions per second (F2F.F64.F32, the bound of the
    fp32-stored sparse mapping kernel and of the training distance): the
    measured per-SM rate (profiles/probe_fp64.json) x 148 SMs x max clock."""
    path = os.path.join(ROOT, "profiles", "probe_fp64.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return j["train_element_peak_per_s"], (f"measured F2F.F64.F32 rate {j['f2f_per_clk_per_sm']}/clk/SM x 148 "
                                               "SMs x 1965 MHz (profiles/probe_fp64.json)")
    return 16 * 148 * 1965e6, "nominal 16 F2F/clk/SM x 148 x 1965 MHz (no measurement file)"


def mapping_leg(som, torch, args, local, seed, world=1, rank=0):
    """Batch BMU mapping docs/s on a c5-shaped sample (BASELINE.json configs[4]:
    100x100 map, 20k terms, CSR documents; the full 10M-document job is the
    doc-sharded multi-GPU case) through som_map_csr.  Main: the default (AUTO)
    path, the exact fp64 sparse identity (map_sparse.cu, R25); beside it the
    dense tcgen05 3xTF32 contraction (map_tc.cu) on the same documents, and
    the oracle's sparse-identity mapping on the host cores for a sample."""
    cfg = CONFIGS["c5"]
    n, d, N = args.map_docs, cfg["d"], cfg["rows"] * cfg["cols"]
    C = bank_corpus(n, d, seed=seed + 500)
    Wsrc = bank_corpus(N, d, seed=args.seed + 501).dense()     # the map is replicated on every rank
    W = (0.5 * Wsrc + 0.5 / np.sqrt(d)).astype(np.float32)
    del Wsrc
    mm = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"], device=local)
    som.som_set_stream(mm.h, torch.cuda.current_stream())
    mm.set_weights(torch.from_numpy(W).cuda())
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
    b1 = torch.empty(n, dtype=torch.int32, device="cuda")
    b2 = torch.empty(n, dtype=torch.int32, device="cuda")
    d1 = torch.empty(n, dtype=torch.float32, device="cuda")

    def timed(precision):
        som.som_set_map_precision(mm.h, precision)
        som.som_map_csr(mm.h, rp, ci, va, n, b1, b2, d1)          # warm-up (W^T / W split, scratch)
        times, kern = [], []
        for _ in range(max(3, args.steps)):
            torch.cuda.synchronize()
            som.som_map_csr(mm.h, rp, ci, va, n, b1, b2, d1)
            ms, _, launches = som.som_last_stats(mm.h)
            times.append(ms)
            kern.append(launches)
        return statistics.mean(times), kern[-1]

    ms, launches = timed(som.SOM_MAP_AUTO)
    sp_b1 = b1.cpu().numpy()
    # end to end through the C ABI with pinned HOST buffers: the CSR arrays
    # go host -> device and bmu1, bmu2, D1 come back inside the timed call
    hrp, hci, hva = (torch.from_numpy(a).pin_memory() for a in (C.indptr, C.indices, C.data))
    hb1 = torch.empty(n, dtype=torch.int32).pin_memory()
    hb2 = torch.empty(n, dtype=torch.int32).pin_memory()
    hd1 = torch.empty(n, dtype=torch.float32).pin_memory()
    som.som_map_csr(mm.h, hrp, hci, hva, n, hb1, hb2, hd1)     # warm-up (staging buffers)
    e2e = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        som.som_map_csr(mm.h, hrp, hci, hva, n, hb1, hb2, hd1)
        e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e)
    h2d_map = hrp.numel() * 8 + hci.numel() * 4 + hva.numel() * 4
    d2h_map = n * 12
    # document sharding: every rank maps its own n documents;
    # the job time is the slowest rank's, the error sums are all-reduced
    qe_l, te_l = som.som_errors_csr(mm.h, rp, ci, va, n)
    err_ms, _, _ = som.som_last_stats(mm.h)
    ms_max, qe, te = ms, qe_l, te_l
    if world > 1:
        import torch.distributed as dist
        from paper_1905_09598_b200 import dist as sdist
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        qe, te = sdist.reduce_errors(qe_l, te_l, n, device=torch.device("cuda", local))
    ms_tc, launches_tc = timed(som.SOM_MAP_3XTF32)
    agree = float(np.mean(b1.cpu().numpy() == sp_b1))
    mm.close()
    fma = float(C.nnz) * N
    cpk, cpk_src = conv_peak_per_s()
    icv_peak = 2.0 * min(cpk / (148 * 1965e6), 12.8) * 148 * 1965e6
    flop = 2.0 * n * N * d
    peak, src = tf32_peak_tflops()
    executed = 3.0 * flop / (ms_tc / 1000.0) / 1e12

    cpu = None
    if not args.no_baseline and rank == 0:
        import oracle
        ns = min(n, 40000)                                   # ~10 s on 16 host cores
        t0 = time.perf_counter()
        oracle.map_docs_csr(W, C.indptr[:ns + 1], C.indices[:C.indptr[ns]], C.data[:C.indptr[ns]])
        dt = time.perf_counter() - t0
        cpu = {"value": ns / dt, "unit": "docs/s", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": f"first {ns} documents, fp64 sparse-identity oracle (or_map_csr, OpenMP over docs), "
                         f"{dt:.1f} s"}
    return {"workload": f"c5-shaped sample: {n} CSR docs ({C.nnz / n:.1f} nnz/doc) x {N} units x {d} terms "
                        f"per GPU, document-sharded over {world} GPU(s)",
            "docs_per_s": world * n / (ms_max / 1000.0), "ms": ms_max, "launches": launches, "n_gpus": world,
            "e2e": {"docs_per_s_rank0": n / e2e_s, "h2d_bytes": h2d_map, "d2h_bytes": d2h_map,
                    "what": "som_map_csr with pinned host CSR arrays and host outputs, wall clock per call"},
            "scaling": "weak", "qe": qe, "te": te, "errors_ms_rank0": err_ms,
            "path": "exact fp64 sparse identity (SOM_MAP_SPARSE_F64, AUTO)",
            "roofline": {"bound": "alu", "kernel": "map_sparse_kernel<8, fp32 W^T, integer widening> (rank 0)",
                         "achieved": fma / (ms / 1000.0) / 1e12, "peak": icv_peak / 1e12, "unit": "T conv+FMA/s",
                         "frac": fma / (ms / 1000.0) / icv_peak,
                         "peak_source": "fp32->fp64 widening split 50/50 between the F2F pipe (" + cpk_src + ") and "
                                        "the integer pipe (5 ALU ops per value on 64 lanes/clk/SM = 12.8/clk/SM, "
                                        "B300_MICROARCH pipe rates): 2 x min(15.43, 12.8)/clk/SM x 148 x 1965 MHz; "
                                        "the map is non-negative, so the kernel widens half the values on the "
                                        "integer pipe",
                         "work": "nnz*N fp32->fp64 conversions + fp64 FMAs per call (one per non-zero per unit), "
                                 "incl. the top-2 merge kernel"},
            "cpu_baseline": cpu,
            "tc_3xtf32": {"docs_per_s": n / (ms_tc / 1000.0), "ms": ms_tc, "launches": launches_tc,
                          "bmu1_agreement_with_exact": agree,
                          "roofline": {"bound": "tensor", "kernel": "map_tc_kernel (tcgen05 kind::tf32, 3xTF32)",
                                       "achieved": executed, "peak": peak, "unit": "TFLOP/s",
                                       "frac": executed / peak, "peak_source": src,
                                       "work": "3 x 2*n*N*d executed TF32 flop per call (3xTF32 split), incl. "
                                               "CSR split + merge",
                                       "algorithmic_fp32_tflops": flop / (ms_tc / 1000.0) / 1e12}}}


def updated_units(rows, cols, topo, bmu_log, t0, T, sigma0, eps=1e-4, k=math.log(100.0), sigma_min=1.0):
    """H_t: units inside the cutoff radius of each step's winner (R5), from the
    BMU log and the schedule (host-side bookkeeping for the byte count)."""
    ii, jj = np.divmod(np.arange(rows * cols), cols)
    out = np.empty(len(bmu_log), np.int64)
    for s, c in enumerate(bmu_log):
        tau = (t0 + s) / T
        sig = max(sigma_min, sigma0 * math.exp(-k * tau * tau))
        r2 = 2.0 * sig * sig * math.log(1.0 / eps)
        ic, jc = divmod(int(c), cols)
        di = (ii - ic).astype(np.float64)
        if topo == 0:
            g2 = di * di + (jj - jc) ** 2
        else:
            dx2 = (2 * (jj - jc) + ((ii & 1) - (ic & 1))).astype(np.float64)
            g2 = 0.25 * dx2 * dx2 + 0.75 * di * di
        out[s] = int(np.count_nonzero(g2 <= r2))
    return out


def batch_leg(som, torch, args, local, seed):
    """Batch SOM (R27, som_train_batch_csr) on the c3 shape: 50x50 hex map,
    50,000 CSR documents x 10,000 terms, `--batch-epochs` epochs; every epoch
    maps all documents (exact sparse path), buckets them by BMU, sums them
    per unit in fp64 and applies the lattice kernel (N x N x (d+1) fp64
    contraction)."""
    cfg = CONFIGS["c3"]
    C = bank_corpus(cfg["n"], cfg["d"], seed=seed + 300)
    N = cfg["rows"] * cfg["cols"]
    from synth import init_rows
    W0 = torch.from_numpy(init_rows(C.dense()[:5000], N, seed + 301)).cuda(local)
    rp, ci, va = (torch.from_numpy(a).cuda(local) for a in (C.indptr, C.indices, C.data))
    E = args.batch_epochs
    with som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"], device=local) as m:
        som.som_set_stream(m.h, torch.cuda.current_stream())
        m.set_weights(W0)
        som.som_train_batch_csr(m.h, rp, ci, va, C.n, 1, cfg["sigma0"], None, None)     # warm-up
        m.set_weights(W0)
        som.som_train_batch_csr(m.h, rp, ci, va, C.n, E, cfg["sigma0"], None, None)
        ms, units, launches = som.som_last_stats(m.h)
    gemm_fma = float(N) * N * (cfg["d"] + 1) * E
    return {"workload": f"c3 shape: {cfg['rows']}x{cfg['cols']} hex, {C.n} CSR docs x {cfg['d']} terms, {E} epochs",
            "docs_per_s": units / (ms / 1e3), "ms_per_epoch": ms / E, "launches": launches,
            "upper_bound_gemm_tflops": 2.0 * gemm_fma / (ms / 1e3) / 1e12,
            "note": "upper_bound_gemm_tflops counts the full N x N x (d+1) fp64 contraction per epoch over the "
                    "whole epoch time (mapping, bucketing, sums included); tiles outside the cutoff are skipped"}


def exchange_probe(som, torch, args, local, rank, world):
    """Per-step cost of the winner exchange alone: a map of 16 units per GPU
    with d = 64 (negligible work per step), 20,000 steps; at N > 1 neuron-
    sharded (in-GPU all-gather + cross-GPU mailbox exchange over NVLink),
    at N = 1 the in-GPU all-gather only.  The difference is the cross-GPU
    latency the sharded training pays every step."""
    import torch.distributed as dist
    from synth import uniform_matrix
    side_c = 16
    steps, n = 20000, 2000
    X = torch.from_numpy(uniform_matrix(n, 64, args.seed + 700)).cuda(local)
    W0 = torch.from_numpy(uniform_matrix(world * side_c, 64, args.seed + 701)).cuda(local)
    ok = torch.zeros(1, dtype=torch.float64, device="cuda")
    ms = 0.0
    sm = None
    try:
        if world > 1:
            from paper_1905_09598_b200.dist import ShardedSOM
            sm = ShardedSOM(world, side_c, 64, 1, rank, world, device=local)
            sm.set_weights(W0)
    except Exception:
        ok[0] = 1.0
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MAX)
        if ok.item() > 0:
            return {"error": "set-up failed"}
    try:
        if world > 1:
            dist.barrier()
            som.som_train_online(sm.h, X, n, 10, ALPHA0, 8.0, None, args.seed, 0, steps, None)
            ms, _, _ = som.som_last_stats(sm.h)
            sm.close()
        else:
            with som.SOM(1, side_c, 64, 1, device=local) as m1:
                m1.set_weights(W0)
                som.som_train_online(m1.h, X, n, 10, ALPHA0, 8.0, None, args.seed, 0, steps, None)
                ms, _, _ = som.som_last_stats(m1.h)
    except Exception:
        ok[0] = 1.0
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MAX)
    if ok.item() > 0:
        return {"error": "exchange probe failed"}
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"us_per_step": 1000.0 * float(t[0]) / steps, "units_per_gpu": side_c, "d": 64, "steps": steps,
            "what": ("in-GPU all-gather + cross-GPU mailbox exchange" if world > 1 else "in-GPU all-gather only")}


def c4_leg(som, torch, args, local, rank, world):
    """c4 (BASELINE.json configs[3]: 100x100 hex map, 20,000 terms) online
    training, the first --c4-steps steps.  At N > 1 the map is neuron-sharded
    over the ranks (dist.ShardedSOM: units u = r + P l, X replicated, the
    per-step winner exchanged inside the training kernel through peer-memory
    mailboxes over NVLink); at N = 1 the same steps on one GPU.  Failures are
    contained: every rank reports its status through an all-reduce and the
    leg returns an error entry instead of stopping the bench."""
    import torch.distributed as dist
    rows = cols = 100
    d, n, steps = 20000, args.c4_docs, args.c4_steps
    C = bank_corpus(n, d, seed=args.seed + 400)                  # identical on every rank
    X = torch.from_numpy(C.dense()).cuda(local)
    from synth import init_rows
    W0 = torch.from_numpy(init_rows(C.dense(), rows * cols, args.seed + 401) if n >= rows * cols else
                          (0.5 * bank_corpus(rows * cols, d, seed=args.seed + 402).dense()
                           + 0.5 * C.dense().mean(0)).astype(np.float32)).cuda(local)
    ok = torch.zeros(1, dtype=torch.float64, device="cuda")
    ms, err, chk = 0.0, "", 0.0
    sm = None
    if world > 1:
        # set-up (IPC mailboxes) and training each end in an all-reduced
        # status, so a rank that fails never leaves the others in a collective
        try:
            from paper_1905_09598_b200.dist import ShardedSOM
            sm = ShardedSOM(rows, cols, d, 1, rank, world, device=local)
            sm.set_weights(W0)
        except Exception as e:
            ok[0] = 1.0
            err = "setup: " + str(e)[:200]
        dist.all_reduce(ok, op=dist.ReduceOp.MAX)
        if ok.item() > 0:
            return {"workload": "c4 neuron-sharded training", "error": err or "set-up failed on another rank"}
    try:
        log = torch.empty(steps, dtype=torch.int32, device="cuda")
        if world > 1:
            dist.barrier()
            som.som_train_online(sm.h, X, n, 2, ALPHA0, 50.0, None, args.seed, 0, steps, log)
            ms, _, _ = som.som_last_stats(sm.h)
            g, k = som.som_last_train_config(sm.h)
            sm.close()
        else:
            with som.SOM(rows, cols, d, 1, device=local) as m1:
                m1.set_weights(W0)
                som.som_train_online(m1.h, X, n, 2, ALPHA0, 50.0, None, args.seed, 0, steps, log)
                ms, _, _ = som.som_last_stats(m1.h)
                g, k = som.som_last_train_config(m1.h)
        lg = log.cpu().numpy().astype(np.float64)
        chk = float((lg * (1 + np.arange(steps) % 977)).sum())
    except Exception as e:      # contained: reported below, never left hanging in a collective
        ok[0] = 1.0
        err = str(e)[:200]
        g, k = 0, -1
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MAX)
    if ok.item() > 0:
        return {"workload": "c4 neuron-sharded training", "error": err or "failed on another rank"}
    t = torch.tensor([ms, chk, -chk], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, consistent = float(t[0]), bool(float(t[1]) == -float(t[2]))
    probe = exchange_probe(som, torch, args, local, rank, world)
    return {"exchange_probe": probe,
            "workload": f"c4: 100x100 hex, 20,000 terms, {n} docs replicated, steps [0, {steps}) of 2 epochs, "
                        f"{'neuron-sharded over ' + str(world) + ' GPUs (in-kernel NVLink winner exchange)' if world > 1 else 'one GPU'}",
            "samples_per_s": steps / (ms_max / 1000.0), "us_per_step": 1000.0 * ms_max / steps,
            "units_per_gpu": (rows * cols + world - 1) // world, "grid": g, "kernel": k,
            "scaling": "strong (one map, units split over the ranks)",
            "bmu_log_identical_on_all_ranks": consistent}


TABLE3_PAPER_S = {16: 34.25, 32: 32.81, 64: 33.37, 128: 38.40, 256: 111.03, 512: 431.38}


def table3_leg(som, torch, args, local, seed):
    """The paper's map-size study (Table 3): online training with
    weight length 64 on square hex maps 16x16 ... 512x512, same data (10,000
    uniform rows) and the same number of steps for every map; kernel time
    per map and the ratio per doubling beside the paper's ratios."""
    from synth import uniform_matrix
    n, d, steps = 10000, 64, args.table3_steps
    X = torch.from_numpy(uniform_matrix(n, d, seed + 64)).cuda(local)
    rows, prev = [], None
    for side in (16, 32, 64, 128, 256, 512):
        W0 = torch.from_numpy(uniform_matrix(side * side, d, seed + side)).cuda(local)
        with som.SOM(side, side, d, 1, device=local) as m:
            som.som_set_stream(m.h, torch.cuda.current_stream())
            epochs = (steps + n - 1) // n
            m.set_weights(W0)
            som.som_train_online(m.h, X, n, epochs, ALPHA0, side / 2.0, None, seed, 0, min(steps, 500), None)
            m.set_weights(W0)
            som.som_train_online(m.h, X, n, epochs, ALPHA0, side / 2.0, None, seed, 0, steps, None)
            ms, units, _ = som.som_last_stats(m.h)
            g, k = som.som_last_train_config(m.h)
        rows.append({"map": f"{side}x{side}", "us_per_step": 1000.0 * ms / units, "samples_per_s": units / (ms / 1e3),
                     "ratio": None if prev is None else ms / prev,
                     "paper_ratio": None if side == 16 else TABLE3_PAPER_S[side] / TABLE3_PAPER_S[side // 2],
                     "grid": g})
        prev = ms
    return {"workload": f"Table 3 study: d = 64, hex maps 16^2..512^2, {n} uniform rows, {steps} steps each "
                        "(short-row kernel train_small.cu)", "maps": rows,
            "paper": "CUDASOM on a Quadro P5000, seconds: " + ", ".join(f"{k}^2 {v}" for k, v in TABLE3_PAPER_S.items())}


def train_c3_leg(som, torch, args, local, seed):
    """Online training in the bandwidth-bound regime: c3 (50x50 hex, 50k x 10k,
    W = 100 MB streamed through L2/HBM every step), first `--c3-steps` steps."""
    cfg = CONFIGS["c3"]
    n, d, N = cfg["n"], cfg["d"], cfg["rows"] * cfg["cols"]
    T = cfg["epochs"] * n
    steps = args.c3_steps
    C = bank_corpus(n, d, seed=seed + 300)
    X = torch.from_numpy(C.dense()).cuda()
    mm = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"], device=local)
    som.som_set_stream(mm.h, torch.cuda.current_stream())
    som.som_init_random(mm.h, X, n, seed + 1300)
    log = torch.empty(steps, dtype=torch.int32, device="cuda")
    som.som_train_online(mm.h, X, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, 0, 2000, None)   # warm-up
    som.som_init_random(mm.h, X, n, seed + 1300)
    som.som_train_online(mm.h, X, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, 0, steps, log)
    ms, _, _ = som.som_last_stats(mm.h)
    g, kern = som.som_last_train_config(mm.h)
    H = updated_units(cfg["rows"], cfg["cols"], cfg["topo"], log.cpu().numpy(), 0, T, cfg["sigma0"])
    algo = float(4.0 * N * d * steps + 4.0 * d * H.sum() + 4.0 * d * steps)   # read W, write updated rows, read x
    gbps = algo / (ms / 1000.0) / 1e9
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm = float(json.load(f)["hbm_gbs"])
    l2, l2_src = 12144.0, "measured L2 read+write bandwidth at a 96 MB footprint (profiles/probes_r01.json l2_rw_GBps)"
    try:
        with open(os.path.join(ROOT, "profiles", "probes_r01.json")) as f:
            l2 = float(json.load(f)["l2_rw_GBps"]["96"])
    except Exception:
        l2_src += " (file missing: fallback value)"
    # late window (radius near sigma_min: few units updated): the dense kernel
    # still reads all of W per step; the CSR kernel's sparse distance reads
    # only the non-zero columns
    late = {}
    t0 = T - steps
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
    for name, csr in (("dense", False), ("csr", True)):
        som.som_init_random(mm.h, X, n, seed + 1300)
        if csr:
            som.som_train_online_csr(mm.h, rp, ci, va, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, t0, T, None)
        else:
            som.som_train_online(mm.h, X, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, t0, T, None)
        lms, _, _ = som.som_last_stats(mm.h)
        late[name] = {"us_per_step": 1000.0 * lms / steps, "kernel": som.som_last_train_config(mm.h)[1]}
    mm.close()
    return {"workload": f"c3: {cfg['rows']}x{cfg['cols']} hex, {n} x {d}, steps [0, {steps}) of T = {T}",
            "samples_per_s": steps / (ms / 1000.0), "us_per_step": 1000.0 * ms / steps,
            "mean_updated_units": float(H.mean()),
            "late_window": {"steps": f"[{t0}, {T})", **late},
            "roofline": {"bound": "l2", "kernel": f"som_train_tma_kernel / som_train_glb_kernel (kernel id {kern}), G={g}",
                         "achieved": gbps, "peak": l2, "unit": "GB/s", "frac": gbps / l2,
                         "peak_source": l2_src,
                         "hbm_frac": gbps / hbm,
                         "work": "4*N*d read + 4*H_t*d written + 4*d per sample (H_t from the BMU log); W (100 MB) "
                                 "is kept in L2 by a persisting window, so L2 read+write bandwidth is the bound "
                                 "(hbm_frac: the same bytes against the HBM copy bandwidth)"}}


# ------------------------------------------------------------- oracle legs
def oracle_train_rate(cfg, X, W0, seed, steps):
    import oracle
    T = cfg["epochs"] * cfg["n"]
    t0 = time.perf_counter()
    oracle.train_online(W0, cfg["rows"], cfg["cols"], cfg["topo"], X, cfg["epochs"], ALPHA0, cfg["sigma0"],
                        seed, t_begin=0, t_end=min(steps, T))
    dt = time.perf_counter() - t0
    return min(steps, T) / dt, dt, oracle.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    cfg, C = workload(args.config, args.seed, args.epochs)
    X = C.dense()
    from synth import init_rows
    W0 = init_rows(X, cfg["rows"] * cfg["cols"], args.seed + 1000)
    steps_per = {"c1": 2000, "c2": 400, "c3": 10}[args.config]
    for _ in range(args.warmup):
        oracle_train_rate(cfg, X, W0, args.seed, max(1, steps_per // 4))
    rates, secs = [], 0.0
    for _ in range(args.steps):
        r, dt, nt = oracle_train_rate(cfg, X, W0, args.seed, steps_per)
        rates.append(r)
        secs += dt
    v = args.steps * steps_per / secs
    sample = (f"first {steps_per} of {cfg['epochs'] * cfg['n']} training steps of {args.config} per step "
              f"(fp64 oracle, OpenMP over units)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, **cfg},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": nt, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- B200 leg
def run_b200(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_1905_09598_b200 import som

    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")   # gloo: plumbing check with ranks on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    seed = args.seed + rank                     # independent problem per rank
    cfg, C = workload(args.config, seed, args.epochs)
    n, d, N = cfg["n"], cfg["d"], cfg["rows"] * cfg["cols"]
    T = cfg["epochs"] * n
    X_host = torch.from_numpy(C.dense()).pin_memory()
    X = X_host.cuda()
    stream = torch.cuda.current_stream()
    m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"], device=local)
    som.som_set_stream(m.h, stream)
    # mapping / QE / TE of the step through the exact sparse identity (R25):
    # the TF-IDF rows are put in CSR form on the device
    som.som_set_map_precision(m.h, som.SOM_MAP_SPARSE_F64)
    b1 = torch.empty(n, dtype=torch.int32, device="cuda")
    b2 = torch.empty(n, dtype=torch.int32, device="cuda")
    d1 = torch.empty(n, dtype=torch.float32, device="cuda")
    U = torch.empty(N, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > 126 MB L2
    sched = som.som_schedule_default()

    def one_step(Xs, b1s, b2s, d1s, Us):
        """The whole hot path once; returns per-phase kernel ms and launches."""
        ph, launches = {}, 0
        som.som_init_random(m.h, Xs, n, seed + 1000)
        ms, _, l = som.som_last_stats(m.h)
        launches += 1 if Xs.is_cuda else 0
        som.som_train_online(m.h, Xs, n, cfg["epochs"], ALPHA0, cfg["sigma0"], sched, seed, 0, -1, None)
        ph["train_ms"], _, l = som.som_last_stats(m.h)
        launches += l
        som.som_map(m.h, Xs, n, b1s, b2s, d1s)
        ph["map_ms"], _, l = som.som_last_stats(m.h)
        launches += l
        qe, te = som.som_errors(m.h, Xs, n)
        ph["errors_ms"], _, l = som.som_last_stats(m.h)
        launches += l
        som.som_umatrix(m.h, Us)
        ph["umatrix_ms"], _, l = som.som_last_stats(m.h)
        launches += l
        return ph, launches, qe, te

    for _ in range(args.warmup):
        one_step(X, b1, b2, d1, U)
    torch.cuda.synchronize()

    # ---- timed region: device resident inputs
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phases, launches = [], 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        w0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()                      # L2 flush between timed steps (not timed)
            ev[i][0].record(stream)
            ph, l, qe, te = one_step(X, b1, b2, d1, U)
            ev[i][1].record(stream)
            phases.append(ph)
            launches += l
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t_max = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max.item())
    value = world * args.steps * T / (total_ms / 1000.0)

    # ---- e2e: same step through the C ABI with pinned HOST buffers
    b1h = torch.empty(n, dtype=torch.int32).pin_memory()
    b2h = torch.empty(n, dtype=torch.int32).pin_memory()
    d1h = torch.empty(n, dtype=torch.float32).pin_memory()
    Uh = torch.empty(N, dtype=torch.float32).pin_memory()
    Wh = torch.empty(N, d, dtype=torch.float32).pin_memory()
    e2e_ms = []
    for i in range(max(1, min(args.steps, 3))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        one_step(X_host, b1h, b2h, d1h, Uh)
        som.som_get_weights(m.h, Wh)
        torch.cuda.synchronize()
        e2e_ms.append(1000 * (time.perf_counter() - t0))
    e2e_t = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    xb = n * d * 4
    h2d = 3 * xb                               # X staged by train, map and errors
    d2h = n * 4 * 2 + n * 4 + N * 4 + N * d * 4 + 16

    # ---- roofline of the dominant kernel (the persistent training kernel)
    train_ms = statistics.mean(p["train_ms"] for p in phases)
    flop_per_sample = 3.0 * N * d               # fp64 distance: sub + fma per element (R10)
    achieved = flop_per_sample * T / (train_ms / 1000.0) / 1e12
    peak, peak_src = train_peak_tflops()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("bytes_per_launch")

    g_used, k_used = som.som_last_train_config(m.h)
    kname = {0: "som_train_kernel (W global)", 1: "som_train_kernel (W smem)",
             2: "som_train_reg_kernel (W registers)", 6: "som_train_spec_kernel (W registers, overlapped exchange)",
             7: "som_train_spec_kernel then som_train_reg_kernel (W registers; one call, two launches)"}.get(k_used, "?")
    mapping = mapping_leg(som, torch, args, local, seed, world, rank) if args.map_docs > 0 else None
    train_c3 = train_c3_leg(som, torch, args, local, seed) if args.c3_steps > 0 else None
    table3 = table3_leg(som, torch, args, local, seed) if args.table3_steps > 0 else None
    batch = batch_leg(som, torch, args, local, seed) if args.batch_epochs > 0 else None
    c4 = c4_leg(som, torch, args, local, rank, world) if args.c4_steps > 0 else None

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return

    cpu = None
    if not args.no_baseline:
        import oracle
        from synth import init_rows
        Xn = X_host.numpy()
        W0 = init_rows(Xn, N, seed + 1000)
        steps_s = {"c1": 20000, "c2": 50000, "c3": 200}[args.config]   # ~10 s of host work (c2)
        r, dt, nt = oracle_train_rate(cfg, Xn, W0, seed, steps_s)
        cpu = {"value": r, "unit": "samples/s", "cores": nt, "kind": "oracle",
               "sample": f"first {steps_s} of {T} training steps of {args.config} ({dt:.1f} s, fp64 oracle, "
                         f"OpenMP over units)"}
        # the oracle on one core as well (a shorter prefix)
        steps_1 = max(1, steps_s // 25)
        oracle.set_num_threads(1)
        try:
            r1, dt1, _ = oracle_train_rate(cfg, Xn, W0, seed, steps_1)
        finally:
            oracle.set_num_threads(nt)
        cpu["single_core"] = {"value": r1, "unit": "samples/s", "cores": 1,
                              "sample": f"first {steps_1} training steps ({dt1:.1f} s)"}

    ph_mean = {k: statistics.mean(p[k] for p in phases) for k in phases[0]}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64-acc/f32",
        "data": "synthetic (seeded bank-shaped TF-IDF, synth/corpus.py)",
        "config": {"workload": args.config, "map": f"{cfg['rows']}x{cfg['cols']} {'hex' if cfg['topo'] else 'rect'}",
                   "docs": n, "terms": d, "epochs": cfg["epochs"], "samples_per_step": T,
                   "alpha0": ALPHA0, "sigma0": cfg["sigma0"], "cutoff": 1e-4, "parallelism": f"replicas{world}",
                   "l2": "flushed between timed steps (256 MB write)",
                   "mapping": "exact sparse identity (SOM_MAP_SPARSE_F64, R25)"},
        "secondary": {"map_docs_per_s": n / (ph_mean["map_ms"] / 1000.0),
                      "train_samples_per_s_kernel": T / (train_ms / 1000.0),
                      "us_per_training_step": 1000.0 * train_ms / T, "phase_ms": ph_mean,
                      "qe": qe, "te": te, "wall_s": wall},
        "e2e": {"value": world * T / (float(e2e_t.item()) / 1000.0), "unit": "samples/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "mapping": mapping,
        "train_c3": train_c3,
        "table3": table3,
        "batch_som": batch,
        "train_c4": c4,
        "roofline": {"bound": "alu", "kernel": f"{kname}, G={g_used}", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     "work": "3*N*d fp64 flop per sample (difference + fused square-accumulate)"},
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
