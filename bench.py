#!/usr/bin/env python
"""bench.py — the CUDASOM hot path on B200, one JSON line on rank 0.

Headline (BASELINE.json configs[2], the largest config one GPU holds; c4 and
c5 are the sharded configs, configs[0]/[1] are parity cases): a "step" is one
pass of the whole hot path over the c3 workload:
50x50 hex map, 50,000 x 10,000 L2-normalised TF-IDF corpus (CSR, the DTM of
P:148-154), seeded row init + 10 epochs of online training (T = 500,000
samples) + batch mapping of all 50,000 documents + QE/TE + U-matrix, all in
one libsom call (som_fit_csr).  value = training samples/s of the whole step.

At N > 1 the same job is split: training neuron-sharded (units u = r + N l,
in-kernel NVLink winner exchange), the trained map gathered once, mapping
and errors document-sharded (errors reduced over libsom's NCCL
communicator) — strong scaling of one job.

Secondary keys: the full c5 mapping job (10M CSR documents onto 100x100,
document-sharded), c4 training (neuron-sharded at N > 1; mailbox vs NCCL
exchange latency), the c2 step of round 1, the paper's Table 3 study, batch
SOM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
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
PAPER_44X = ("CUDASOM's average speed-up of 44x over its CPU SOM (PAPER.md:35; 41-47x per run, Table 2 PAPER.md:286-296) "
             "on an NVIDIA Quadro P5000 (Pascal, CUDA 8.0, PyCUDA) vs an Intel Xeon E5-2640 v4 @ 2.4 GHz (PAPER.md:223-225)"
             ": context only, other hardware and a different CPU baseline")
C5_DOCS, C5_BLOCK = 10_000_000, 200_000


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c3", choices=["c1", "c2", "c3"])
    p.add_argument("--epochs", type=int, default=None, help="override epochs (diagnostics only)")
    p.add_argument("--no-baseline", action="store_true", help="skip the cpu_baseline legs")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--c5-docs", type=int, default=C5_DOCS, help="documents of the c5 mapping job (0 = skip)")
    p.add_argument("--c4-steps", type=int, default=2000, help="steps of the c4 training leg (0 = skip)")
    p.add_argument("--c2-steps", type=int, default=1, help="timed c2 steps of the round-1 leg (0 = skip)")
    p.add_argument("--table3-steps", type=int, default=20000, help="steps per map of the Table 3 leg (0 = skip)")
    p.add_argument("--batch-epochs", type=int, default=10, help="epochs of the batch-SOM leg (0 = skip)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BENCH_ONE_DEVICE") == "1":   # test hook: every rank on cuda:0 (multi-rank plumbing check)
        local = 0
        # no persisting-L2 window: its device-wide set-aside can wait behind
        # a peer rank's spinning grid on the shared device
        os.environ.setdefault("SOM_NO_L2_WINDOW", "1")
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


# ------------------------------------------------------------------ peaks
def _json(path):
    with open(os.path.join(ROOT, path)) as f:
        return json.load(f)


def hbm_peak_gbs():
    try:
        return float(_json("MEASURED_PEAKS.json")["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except Exception:
        return 6550.0, "fallback 6.55 TB/s (B200_PROFILING.md)"


def l2_peak_gbs(footprint_mb=96):
    """Measured L2 read+write bandwidth at a footprint just below the L2
    (profiles/probes_r01.json, tools/probes.cu)."""
    try:
        j = _json("profiles/probes_r01.json")["l2_rw_GBps"]
        return float(j[str(footprint_mb)]), f"measured L2 read+write bandwidth at a {footprint_mb} MB footprint " \
                                            "(profiles/probes_r01.json l2_rw_GBps)"
    except Exception:
        return 12144.0, "fallback 12.1 TB/s L2 read+write (profiles/probes_r01.json missing)"


def train_peak_tflops():
    """Peak of the exact distance element (1 F2F.F64.F32 + DADD + DFMA = 3
    flop): the measured fp32->fp64 conversion rate x 148 SMs x max clock."""
    try:
        j = _json("profiles/probe_fp64.json")
        return 3.0 * j["train_element_peak_per_s"] / 1e12, ("measured F2F.F64.F32 rate "
                                                            f"{j['f2f_per_clk_per_sm']}/clk/SM x 148 SMs x 1965 MHz "
                                                            "x 3 flop/element (profiles/probe_fp64.json)")
    except Exception:
        return 3.0 * 16 * 148 * 1965e6 / 1e12, "nominal 16 F2F/clk/SM x 148 x 1965 MHz x 3 flop (no measurement file)"


def tf32_peak_tflops():
    """Dense TF32 peak: the measured bf16 cuBLAS peak (MEASURED_PEAKS.json,
    burst) x the nominal tf32/bf16 ratio 1.1/2.25 (B200_PROFILING.md)."""
    try:
        bf16 = float(_json("MEASURED_PEAKS.json")["bf16_tflops"])
        return bf16 * 1.1 / 2.25, f"measured bf16 {bf16} TFLOP/s x 1.1/2.25 (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0 * 1.1 / 2.25, "fallback bf16 1590 TFLOP/s x 1.1/2.25 (B200_PROFILING.md)"


def conv_peak_per_s():
    """fp32 -> fp64 conversions per second (F2F.F64.F32): the measured per-SM
    rate (profiles/probe_fp64.json) x 148 SMs x max clock."""
    try:
        j = _json("profiles/probe_fp64.json")
        return j["train_element_peak_per_s"], (f"measured F2F.F64.F32 rate {j['f2f_per_clk_per_sm']}/clk/SM x 148 "
                                               "SMs x 1965 MHz (profiles/probe_fp64.json)")
    except Exception:
        return 16 * 148 * 1965e6, "nominal 16 F2F/clk/SM x 148 x 1965 MHz (no measurement file)"


def icv_peak_per_s():
    """Split-widening peak of the sparse mapping kernel: half the values on
    the F2F pipe, half widened exactly on the integer pipe (5 ALU ops); the
    integer rate is the measured one when profiles/probe_icv.json exists."""
    cpk, src = conv_peak_per_s()
    f2f_clk = cpk / (148 * 1965e6)
    try:
        j = _json("profiles/probe_icv.json")
        icv_clk, isrc = float(j["icv_per_clk_per_sm"]), "measured integer widening rate (profiles/probe_icv.json)"
    except Exception:
        icv_clk, isrc = 12.8, "nominal 64 INT lanes/clk/SM / 5 ops (B300_MICROARCH pipe rates)"
    return 2.0 * min(f2f_clk, icv_clk) * 148 * 1965e6, f"2 x min(F2F {f2f_clk:.2f}, ICV {icv_clk:.2f})/clk/SM x 148 " \
                                                         f"x 1965 MHz; F2F: {src}; ICV: {isrc}"


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


def train_bytes(N, d, nnz_x, H, sparse):
    """Algorithmic bytes of one training step:
    dense rows: read W (4 N d) + write the H_t updated rows (4 H_t d) + x_t;
    sparse rows (R25, the kernel family that runs on TF-IDF rows): read and
    write the H_t updated rows (8 H_t d) + one fp32 gathered per non-zero of
    x_t for every other unit (4 nnz (N - H_t)) + x_t's CSR entries."""
    H = np.asarray(H, np.float64)
    if sparse:
        return float(np.sum(8.0 * H * d + 4.0 * nnz_x * (N - H) + 8.0 * nnz_x))
    return float(np.sum(4.0 * N * d + 4.0 * H * d + 4.0 * d))


def nccl_usable():
    """NCCL refuses two ranks on one GPU: the one-device plumbing hook
    (BENCH_ONE_DEVICE=1) reduces the document-sharded error sums over
    torch.distributed instead and skips the NCCL exchange baseline."""
    return os.environ.get("BENCH_ONE_DEVICE") != "1"


def sharded_errors(som, h, rp, ci, va, n, world):
    """QE/TE of a document-sharded corpus: inside libsom over its NCCL
    communicator, or (one-device hook) this rank's values reduced here."""
    if world == 1 or nccl_usable():
        return som.som_errors_csr(h, rp, ci, va, n)
    from paper_1905_09598_b200 import dist as sdist
    qe, te = som.som_errors_csr(h, rp, ci, va, n) if n > 0 else (0.0, 0.0)
    return sdist.reduce_errors(qe, te, n, device="cuda")


def config_dict(name, cfg, world):
    """The config both arms report (identical keys and values)."""
    return {"workload": name, "map": f"{cfg['rows']}x{cfg['cols']} {'hex' if cfg['topo'] else 'rect'}",
            "docs": cfg["n"], "terms": cfg["d"], "epochs": cfg["epochs"], "samples_per_step": cfg["epochs"] * cfg["n"],
            "alpha0": ALPHA0, "sigma0": cfg["sigma0"], "cutoff": 1e-4, "input": "CSR (TF-IDF DTM)",
            "step": "init + full online training + mapping of all docs + QE/TE + U-matrix (som_fit_csr)",
            "parallelism": "1 GPU" if world == 1 else f"neuron-sharded training + document-sharded mapping over "
                                                      f"{world} GPUs",
            "l2": "flushed between timed steps (256 MB write)"}


# ------------------------------------------------------------- c5 corpus
def _c5_block(k):
    C = bank_corpus(C5_BLOCK, CONFIGS["c5"]["d"], seed=9000 + k)
    return C.indptr, C.indices, C.data


def c5_corpus(n_docs, rank, world):
    """This rank's contiguous share of the c5 corpus (BASELINE configs[4]):
    blocks of 200,000 documents generated by seed (the same corpus as
    tests/test_gpu_full_size.py), built in parallel host processes."""
    import multiprocessing as mp
    nb = max(1, n_docs // C5_BLOCK)
    from paper_1905_09598_b200.dist import shard_range
    lo, hi = shard_range(nb, rank, world)
    ks = list(range(lo, hi))
    if not ks:
        return np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32), 0
    with mp.get_context("fork").Pool(min(16, max(1, (os.cpu_count() or 2) // max(1, world)))) as pool:
        parts = pool.map(_c5_block, ks)
    nnz = sum(p[1].size for p in parts)
    n = sum(p[0].size - 1 for p in parts)
    rowptr = np.empty(n + 1, np.int64)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    rowptr[0] = 0
    r = o = 0
    for ip, ci, va in parts:
        m = ip.size - 1
        rowptr[r + 1:r + m + 1] = ip[1:] + o
        col[o:o + ci.size] = ci
        val[o:o + va.size] = va
        r += m
        o += ci.size
    return rowptr, col, val, n


def c5_codebook():
    d = CONFIGS["c5"]["d"]
    return (0.5 * bank_corpus(10000, d, seed=8999).dense() + 0.5 / np.sqrt(d)).astype(np.float32)


# ------------------------------------------------------------- B200 legs
def c5_leg(som, torch, args, local, rank, world, corpus):
    """BASELINE.json configs[4]: batch BMU mapping of 10,000,000 CSR
    documents x 20,000 terms onto a 100x100 hex map, document-sharded over
    the ranks (each maps its contiguous share; QE/TE reduced over libsom's
    NCCL communicator).  docs/s = all documents / slowest rank's device time.
    Default path: the exact fp64 sparse identity (R25, map_sparse.cu)."""
    import torch.distributed as dist
    rowptr, col, val, n = corpus
    cfg = CONFIGS["c5"]
    N, d = cfg["rows"] * cfg["cols"], cfg["d"]
    W = torch.from_numpy(c5_codebook()).cuda(local)
    mm = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"], device=local)
    som.som_set_stream(mm.h, torch.cuda.current_stream())
    if world > 1 and nccl_usable():
        from paper_1905_09598_b200 import dist as sdist
        sdist.init_nccl(mm.h, rank, world, som.SOM_SHARD_DOCS)
    mm.set_weights(W)
    rp, ci, va = (torch.from_numpy(a).cuda(local) for a in (rowptr, col, val))
    b1 = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    b2 = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    d1 = torch.empty(max(n, 1), dtype=torch.float32, device="cuda")
    som.som_map_csr(mm.h, rp, ci, va, n, b1, b2, d1)            # warm-up (W^T, scratch)
    times, launches = [], 0
    for _ in range(max(3, min(args.steps, 5))):
        torch.cuda.synchronize()
        som.som_map_csr(mm.h, rp, ci, va, n, b1, b2, d1)
        ms, _, launches = som.som_last_stats(mm.h)
        times.append(ms)
    ms = statistics.mean(times)
    qe, te = sharded_errors(som, mm.h, rp, ci, va, n, world)    # collective at N > 1
    err_ms = som.som_last_stats(mm.h)[0]
    t = torch.tensor([ms, err_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, err_max = float(t[0]), float(t[1])
    # end to end: pinned host CSR arrays in, host outputs back, wall clock
    hrp, hci, hva = (torch.from_numpy(a).pin_memory() for a in (rowptr, col, val))
    hb1, hb2 = (torch.empty(max(n, 1), dtype=torch.int32).pin_memory() for _ in range(2))
    hd1 = torch.empty(max(n, 1), dtype=torch.float32).pin_memory()
    som.som_map_csr(mm.h, hrp, hci, hva, n, hb1, hb2, hd1)       # warm-up (staging buffers)
    e2e = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        som.som_map_csr(mm.h, hrp, hci, hva, n, hb1, hb2, hd1)
        e2e.append(time.perf_counter() - t0)
    te2e = torch.tensor([statistics.mean(e2e)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te2e, op=dist.ReduceOp.MAX)
    # beside it: the tcgen05 3xTF32 contraction on a 200k-document sample
    ns = min(n, 200_000)
    som.som_set_map_precision(mm.h, som.SOM_MAP_3XTF32)
    som.som_map_csr(mm.h, rp, ci, va, ns, b1, b2, d1)
    tc_ms = []
    for _ in range(2):
        som.som_map_csr(mm.h, rp, ci, va, ns, b1, b2, d1)
        tc_ms.append(som.som_last_stats(mm.h)[0])
    tcm = statistics.mean(tc_ms)
    tc_fallbacks = som.som_last_map_fallbacks(mm.h)
    mm.close()
    nnz = float(val.size)
    work = nnz * N                                               # conversions + FMAs (one per non-zero per unit)
    peak, psrc = icv_peak_per_s()
    tpeak, tsrc = tf32_peak_tflops()
    executed = 3.0 * 2.0 * ns * N * d / (tcm / 1e3) / 1e12
    cpu = None
    if rank == 0 and not args.no_baseline:
        import oracle
        nsb = min(n, 40000)                                        # ~10 s on 16 host cores
        t0 = time.perf_counter()
        oracle.map_docs_csr(c5_codebook(), rowptr[:nsb + 1], col[:rowptr[nsb]], val[:rowptr[nsb]])
        dt = time.perf_counter() - t0
        cpu = {"value": nsb / dt, "unit": "docs/s", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": f"first {nsb} documents of the c5 corpus, fp64 sparse-identity oracle (or_map_csr, "
                         f"OpenMP over documents), {dt:.1f} s"}
    n_all = n * world if world > 1 else n
    total = args.c5_docs if world > 1 else n
    return {"workload": f"c5: {total} CSR docs ({nnz / max(n, 1):.1f} nnz/doc) x 100x100 hex x {d} terms, "
                        f"{'document-sharded over ' + str(world) + ' GPUs' if world > 1 else '1 GPU'}",
            "docs_per_s": total / (ms_max / 1e3), "ms": ms_max, "launches_rank0": launches,
            "scaling": "strong (fixed 10M-document job)" if world > 1 else None, "n_gpus": world,
            "qe": qe, "te": te, "errors_ms": err_max, "docs_rank0": n, "docs_all": n_all,
            "e2e": {"docs_per_s": total / float(te2e[0]), "h2d_bytes_rank0": int(rowptr.nbytes + col.nbytes + val.nbytes),
                    "d2h_bytes_rank0": 12 * n, "what": "som_map_csr with pinned host CSR arrays and host outputs "
                                                        "(max over ranks, wall clock)"},
            "path": "exact fp64 sparse identity (R25; AUTO)",
            "roofline": {"bound": "alu", "kernel": "map_sparse_kernel<8, fp32 W^T, integer widening> (rank 0)",
                         "achieved": work / (ms / 1e3) / 1e12, "peak": peak / 1e12, "unit": "T conv+FMA/s",
                         "frac": work / (ms / 1e3) / peak, "peak_source": psrc,
                         "work": "nnz x N fp32->fp64 conversions + fp64 FMAs per call (incl. the top-2 merge)"},
            "cpu_baseline": cpu,
            "tc_3xtf32": {"docs": ns, "docs_per_s": ns / (tcm / 1e3), "ms": tcm,
                          "exact_fallback_docs": tc_fallbacks,
                          "what": "3xTF32 candidates (4 per document) rescored by the exact fp64 definition and "
                                  "certified (R20b): bmu1/bmu2/D1 exact for every document",
                          "roofline": {"bound": "tensor", "kernel": "map_tc_kernel (tcgen05 kind::tf32, 3xTF32)",
                                       "achieved": executed, "peak": tpeak, "unit": "TFLOP/s",
                                       "frac": executed / tpeak, "peak_source": tsrc,
                                       "work": "3 x 2 n N d executed TF32 flop per call over the whole call "
                                               "(split, GEMM, certified rescoring)"}}}


def c4_leg(som, torch, args, local, rank, world):
    """c4 (BASELINE.json configs[3]: 100x100 hex, 200,000 x 20,000, 2 epochs)
    online training, the first --c4-steps steps.  At N > 1 the map is
    neuron-sharded over the ranks (units u = r + N l; X replicated; the
    per-step winner exchanged inside the training kernel through peer-memory
    mailboxes over NVLink).  Beside it the exchange latency alone (a 16-unit
    map per GPU): in-kernel mailbox vs the NCCL baseline (one step kernel +
    ncclAllReduce(u64, min) per step, CUDA-graph replayed)."""
    import torch.distributed as dist
    cfg = CONFIGS["c4"]
    rows, cols, d = cfg["rows"], cfg["cols"], cfg["d"]
    C = bank_corpus(cfg["n"], d, seed=args.seed + 400)          # identical on every rank
    rp, ci, va = (torch.from_numpy(a).cuda(local) for a in (C.indptr, C.indices, C.data))
    steps = args.c4_steps
    ok = torch.zeros(1, dtype=torch.float64, device="cuda")
    ms, err = 0.0, ""
    g = k = -1
    sm = None
    try:
        if world > 1:
            from paper_1905_09598_b200.dist import ShardedSOM
            sm = ShardedSOM(rows, cols, d, cfg["topo"], rank, world, device=local)
            h = sm.h
        else:
            h = som.som_create(rows, cols, d, cfg["topo"], local)
        som.som_init_random_csr(h, rp, ci, va, C.n, args.seed + 1401)
    except Exception as e:
        ok[0] = 1.0
        err = "setup: " + str(e)[:200]
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MAX)
    if ok.item() > 0:
        return {"workload": "c4 training", "error": err or "set-up failed on another rank"}
    log = torch.empty(steps, dtype=torch.int32, device="cuda")
    try:
        if world > 1:
            dist.barrier()
        som.som_train_online_csr(h, rp, ci, va, C.n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, args.seed, 0, steps,
                                 log)
        ms = som.som_last_stats(h)[0]
        g, k = som.som_last_train_config(h)
    except Exception as e:
        ok[0] = 1.0
        err = str(e)[:200]
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MAX)
    if sm is not None:
        sm.close()
    else:
        som.som_destroy(h)
    if ok.item() > 0:
        return {"workload": "c4 training", "error": err or "failed on another rank"}
    lg = log.cpu().numpy().astype(np.float64)
    chk = float((lg * (1 + np.arange(steps) % 977)).sum())
    t = torch.tensor([ms, chk, -chk], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"workload": f"c4: 100x100 hex, {C.n} CSR docs x {d} terms (replicated), steps [0, {steps}) of "
                        f"{cfg['epochs']} epochs, {'neuron-sharded over ' + str(world) + ' GPUs' if world > 1 else '1 GPU'}",
            "samples_per_s": steps / (float(t[0]) / 1e3), "us_per_step": 1e3 * float(t[0]) / steps,
            "units_per_gpu": (rows * cols + world - 1) // world, "grid": g, "kernel": k,
            "scaling": "strong (one map, units split over the ranks)",
            "bmu_log_identical_on_all_ranks": bool(float(t[1]) == -float(t[2])),
            "exchange_probe": exchange_probe(som, torch, args, local, rank, world)}


def exchange_probe(som, torch, args, local, rank, world):
    """Per-step cost of the winner exchange alone: 16 units per GPU, d = 64
    (negligible work), 20,000 steps.  mailbox: the in-kernel exchange (at
    N = 1 the in-GPU all-gather only); nccl: one step kernel + one
    ncclAllReduce(u64, min) per step (libsom's communicator)."""
    import torch.distributed as dist
    from synth import uniform_matrix
    side_c, steps, n = 16, 20000, 2000
    X = torch.from_numpy(uniform_matrix(n, 64, args.seed + 700)).cuda(local)
    W0 = torch.from_numpy(uniform_matrix(world * side_c, 64, args.seed + 701)).cuda(local)
    out = {"units_per_gpu": side_c, "d": 64, "steps": steps}
    for mode in ("mailbox", "nccl") if nccl_usable() else ("mailbox",):
        ok = torch.zeros(1, dtype=torch.float64, device="cuda")
        ms = 0.0
        h = None
        try:
            h = som.som_create(world, side_c, 64, 1, local)
            if mode == "nccl":
                from paper_1905_09598_b200 import dist as sdist
                sdist.init_nccl(h, rank, world, som.SOM_SHARD_NEURONS)
                som.som_set_exchange(h, som.SOM_XCHG_NCCL)
            elif world > 1:
                from paper_1905_09598_b200.dist import exchange_handles
                som.som_comm_init(h, rank, world)
                som.som_comm_set_peers_ipc(h, exchange_handles(som.som_comm_mailbox_ipc(h)))
            som.som_set_weights(h, W0)
            if world > 1:
                dist.barrier()
            st = steps if mode == "mailbox" else steps // 4
            som.som_train_online(h, X, n, 10, ALPHA0, 8.0, None, args.seed, 0, st, None)
            ms = som.som_last_stats(h)[0] / st
        except Exception as e:
            ok[0] = 1.0
            out[mode + "_error"] = str(e)[:200]
        if h is not None:
            som.som_destroy(h)
        if world > 1:
            dist.all_reduce(ok, op=dist.ReduceOp.MAX)
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[mode + "_us_per_step"] = None if ok.item() > 0 else 1e3 * float(t[0])
    out["what"] = ("in-GPU all-gather + cross-GPU mailbox exchange (mailbox); step kernel + NCCL all-reduce (nccl)"
                   if world > 1 else "one GPU: in-GPU all-gather (mailbox); step kernel + world-1 NCCL all-reduce (nccl)")
    return out


def c2_leg(som, torch, args, local, seed):
    """The round-1 headline for continuity: c2 (20x20 hex, 5,000 x 3,000,
    100 epochs = 500,000 samples) in one som_fit_csr call."""
    cfg = CONFIGS["c2"]
    C = bank_corpus(cfg["n"], cfg["d"], seed=seed)
    rp, ci, va = (torch.from_numpy(a).cuda(local) for a in (C.indptr, C.indices, C.data))
    with som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"], device=local) as m:
        som.som_set_stream(m.h, torch.cuda.current_stream())
        som.som_fit_csr(m.h, rp, ci, va, C.n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, seed + 1000)
        ms = []
        for _ in range(args.c2_steps):
            som.som_fit_csr(m.h, rp, ci, va, C.n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, seed + 1000)
            ms.append(som.som_last_stats(m.h)[0])
        ph, tr = som.som_last_phases(m.h)
        g, k = som.som_last_train_config(m.h)
    T = cfg["epochs"] * cfg["n"]
    return {"workload": "c2 (BASELINE configs[1]): 20x20 hex, 5,000 x 3,000, 100 epochs, som_fit_csr",
            "samples_per_s": T / (statistics.mean(ms) / 1e3), "us_per_training_step": 1e3 * tr / T,
            "train_kernel": k, "grid": g}


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


def batch_leg(som, torch, args, local, seed, C3):
    """Batch SOM (R27, som_train_batch_csr) on the c3 corpus, --batch-epochs
    epochs: exact BMUs, documents bucketed by BMU, per-unit fp64 sums, lattice
    kernel contraction."""
    cfg = CONFIGS["c3"]
    rp, ci, va = C3
    n = rp.numel() - 1
    with som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"], device=local) as m:
        som.som_set_stream(m.h, torch.cuda.current_stream())
        som.som_init_random_csr(m.h, rp, ci, va, n, seed + 301)
        som.som_train_batch_csr(m.h, rp, ci, va, n, 1, cfg["sigma0"], None, None)     # warm-up
        som.som_init_random_csr(m.h, rp, ci, va, n, seed + 301)
        som.som_train_batch_csr(m.h, rp, ci, va, n, args.batch_epochs, cfg["sigma0"], None, None)
        ms, units, launches = som.som_last_stats(m.h)
    return {"workload": f"c3 corpus: 50x50 hex, {n} CSR docs x {cfg['d']} terms, {args.batch_epochs} batch epochs",
            "docs_per_s": units / (ms / 1e3), "ms_per_epoch": ms / args.batch_epochs, "launches": launches}


# ------------------------------------------------------------- oracle legs
def oracle_train_rate(cfg, X, W0, seed, steps, threads=None):
    import oracle
    T = cfg["epochs"] * cfg["n"]
    nt = oracle.num_threads()
    if threads:
        oracle.set_num_threads(threads)
    try:
        t0 = time.perf_counter()
        oracle.train_online(W0, cfg["rows"], cfg["cols"], cfg["topo"], X, cfg["epochs"], ALPHA0, cfg["sigma0"],
                            seed, t_begin=0, t_end=min(steps, T))
        dt = time.perf_counter() - t0
        used = oracle.num_threads()
    finally:
        oracle.set_num_threads(nt)
    return min(steps, T) / dt, dt, used


def corpus_seed(name, seed):
    return seed + 300 if name == "c3" else seed


def oracle_inputs(name, seed):
    """The oracle's dense copy of the same corpus (seeded) and a seeded row init."""
    from synth import init_rows
    cfg = CONFIGS[name]
    X = bank_corpus(cfg["n"], cfg["d"], seed=corpus_seed(name, seed)).dense()
    return X, init_rows(X, cfg["rows"] * cfg["cols"], seed + 1300)


REF_STEPS = {"c1": 2000, "c2": 400, "c3": 300}   # oracle steps per reference-arm step (~3-6 s each on 16 cores)


def run_reference(args, rank, world):
    """The reference arm of this tier: the oracle (plain fp64 CPU SOM), as it
    stands, on the host cores, on bounded samples of the same workload."""
    if rank != 0:
        return
    import oracle
    cfg = dict(CONFIGS[args.config])
    if args.epochs is not None:
        cfg["epochs"] = args.epochs
    X, W0 = oracle_inputs(args.config, args.seed)
    steps_per = REF_STEPS[args.config]
    for _ in range(args.warmup):
        oracle_train_rate(cfg, X, W0, args.seed, max(1, steps_per // 10))
    secs = 0.0
    for _ in range(args.steps):
        _, dt, nt = oracle_train_rate(cfg, X, W0, args.seed, steps_per)
        secs += dt
    v = args.steps * steps_per / secs
    sample = (f"first {steps_per} of {cfg['epochs'] * cfg['n']} training steps of {args.config} per step "
              f"(fp64 oracle, OpenMP over units, {nt} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded bank-shaped TF-IDF, synth/corpus.py)",
            "config": config_dict(args.config, cfg, world),
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": nt, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- B200 arm
def run_b200(args, rank, world, local):
    c5 = c5_corpus(args.c5_docs, rank, world) if args.c5_docs > 0 else None    # host processes before CUDA
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
    seed = args.seed
    cfg = dict(CONFIGS[args.config])
    if args.epochs is not None:
        cfg["epochs"] = args.epochs
    n, d, N = cfg["n"], cfg["d"], cfg["rows"] * cfg["cols"]
    T = cfg["epochs"] * n
    C = bank_corpus(n, d, seed=corpus_seed(args.config, seed))    # identical on every rank
    rp, ci, va = (torch.from_numpy(a).cuda(local) for a in (C.indptr, C.indices, C.data))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > 126 MB L2
    init_seed = seed + 1000

    if world == 1:
        m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"], device=local)
        som.som_set_stream(m.h, stream)
        b1 = torch.empty(n, dtype=torch.int32, device="cuda")
        b2 = torch.empty(n, dtype=torch.int32, device="cuda")
        d1 = torch.empty(n, dtype=torch.float32, device="cuda")
        U = torch.empty(N, dtype=torch.float32, device="cuda")

        def one_step(ins, outs):
            qe, te = som.som_fit_csr(m.h, *ins, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, init_seed, *outs)
            ph, train_ms = som.som_last_phases(m.h)
            return {"phase_ms": dict(zip(["init", "train", "map", "errors", "umatrix"], ph)),
                    "train_kernel_ms": train_ms, "launches": som.som_last_stats(m.h)[2], "qe": qe, "te": te}
        dev_in, dev_out = (rp, ci, va), (b1, b2, d1, U)
    else:
        from paper_1905_09598_b200 import dist as sdist
        sm = sdist.ShardedSOM(cfg["rows"], cfg["cols"], d, cfg["topo"], rank, world, device=local)
        som.som_set_stream(sm.h, stream)
        md = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"], device=local)
        som.som_set_stream(md.h, stream)
        if nccl_usable():
            sdist.init_nccl(md.h, rank, world, som.SOM_SHARD_DOCS)
        lo, hi = sdist.shard_range(n, rank, world)
        ns = hi - lo
        h_srp = (C.indptr[lo:hi + 1] - C.indptr[lo]).astype(np.int64)
        h_sci, h_sva = C.indices[C.indptr[lo]:C.indptr[hi]], C.data[C.indptr[lo]:C.indptr[hi]]
        srp, sci, sva = (torch.from_numpy(np.ascontiguousarray(x)).cuda(local) for x in (h_srp, h_sci, h_sva))
        b1 = torch.empty(max(ns, 1), dtype=torch.int32, device="cuda")
        b2 = torch.empty(max(ns, 1), dtype=torch.int32, device="cuda")
        d1 = torch.empty(max(ns, 1), dtype=torch.float32, device="cuda")
        U = torch.empty(N, dtype=torch.float32, device="cuda")
        Wfull = torch.zeros(N, d, dtype=torch.float32, device="cuda")
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]

        def one_step(ins, outs):
            # ins: the full CSR corpus (every rank trains on all of it) and this
            # rank's document shard; outs: its bmu1, bmu2, D1 and the U-matrix
            # (device tensors, or pinned host buffers for e2e)
            irp, ici, iva, jrp, jci, jva = ins
            ob1, ob2, od1, oU = outs
            launches = 0
            evs[0].record(stream)
            som.som_init_random_csr(sm.h, irp, ici, iva, n, init_seed)
            launches += som.som_last_stats(sm.h)[2]
            evs[1].record(stream)
            dist.barrier()
            som.som_train_online_csr(sm.h, irp, ici, iva, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, 0, -1,
                                     None)
            train_ms, _, tl = som.som_last_stats(sm.h)
            launches += tl
            dist.barrier()
            evs[2].record(stream)
            Wfull.zero_()
            som.som_get_weights(sm.h, Wfull)                 # own rows; all-reduce assembles the map
            dist.all_reduce(Wfull)
            md.set_weights(Wfull)
            som.som_map_csr(md.h, jrp, jci, jva, ns, ob1, ob2, od1)
            launches += som.som_last_stats(md.h)[2]
            evs[3].record(stream)
            qe, te = sharded_errors(som, md.h, jrp, jci, jva, ns, world)   # NCCL-reduced inside libsom
            launches += som.som_last_stats(md.h)[2]
            evs[4].record(stream)
            som.som_umatrix(md.h, oU)
            launches += som.som_last_stats(md.h)[2]
            evs[5].record(stream)
            torch.cuda.synchronize()
            ph = [evs[i].elapsed_time(evs[i + 1]) for i in range(5)]
            return {"phase_ms": dict(zip(["init", "train", "map (gather W + shard)", "errors", "umatrix"], ph)),
                    "train_kernel_ms": train_ms, "launches": launches, "qe": qe, "te": te}
        dev_in, dev_out = (rp, ci, va, srp, sci, sva), (b1, b2, d1, U)

    for _ in range(max(3, args.warmup)):
        one_step(dev_in, dev_out)
    torch.cuda.synchronize()

    # ---- timed region: inputs resident in HBM
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    infos = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()                                # L2 flush between timed steps (not timed)
            ev[i][0].record(stream)
            infos.append(one_step(dev_in, dev_out))
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t_max = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max.item())
    value = args.steps * T / (total_ms / 1e3)

    # ---- e2e: the same calls with pinned HOST inputs and host outputs
    hfull = tuple(torch.from_numpy(a).pin_memory() for a in (C.indptr, C.indices, C.data))
    if world == 1:
        hin, nd = hfull, n
    else:
        hin = hfull + tuple(torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (h_srp, h_sci, h_sva))
        nd = ns
    hout = (torch.empty(max(nd, 1), dtype=torch.int32).pin_memory(),
            torch.empty(max(nd, 1), dtype=torch.int32).pin_memory(),
            torch.empty(max(nd, 1), dtype=torch.float32).pin_memory(), torch.empty(N, dtype=torch.float32).pin_memory())
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 3))):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        one_step(hin, hout)
        torch.cuda.synchronize()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_mean = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_mean, op=dist.ReduceOp.MAX)
    h2d = sum(int(x.numel() * x.element_size()) for x in hin)
    d2h = sum(int(x.numel() * x.element_size()) for x in hout) + 16
    e2e = {"value": T / (float(e2e_mean.item()) / 1e3), "unit": "samples/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h,
           "what": ("som_fit_csr" if world == 1 else "the sharded step's libsom calls") +
                   " with pinned host CSR arrays (staged once per call) and host outputs (bmu1, bmu2, D1, U, QE, "
                   "TE), wall clock per step" + ("" if world == 1 else ", max over ranks; bytes of rank 0")}

    # ---- roofline of the dominant kernel (the training kernel of the step)
    train_ms = statistics.mean(i["train_kernel_ms"] for i in infos)
    roof = None
    g_used = k_used = -1
    if world == 1:
        g_used, k_used = som.som_last_train_config(m.h)
        # the BMU log of the same (deterministic) training, untimed, for H_t
        log = torch.empty(T, dtype=torch.int32, device="cuda")
        som.som_init_random_csr(m.h, rp, ci, va, n, init_seed)
        som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], ALPHA0, cfg["sigma0"], None, seed, 0, -1, log)
        H = updated_units(cfg["rows"], cfg["cols"], cfg["topo"], log.cpu().numpy(), 0, T, cfg["sigma0"])
        nnz_x = C.nnz / n
        sparse = k_used in (4, 10, 11)
        algo = train_bytes(N, d, nnz_x, H, sparse)
        gbps = algo / (train_ms / 1e3) / 1e9
        l2, l2src = l2_peak_gbs(96)
        hbm, hsrc = hbm_peak_gbs()
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj.get("bytes_per_launch") if tj.get("kernel_id", k_used) == k_used else None
        kname = {3: "som_train_tma_kernel (dense rows, W streamed)", 4: "som_train_csr_tma_kernel (sparse distances, "
                 "W streamed through L2)", 2: "som_train_reg_kernel (W in registers)",
                 10: "som_train_tier_kernel (W in TMEM + smem + a streamed remainder, sparse distances)",
                 11: "som_train_tier_kernel while the neighbourhood covers the map, then som_train_csr_tma_kernel "
                     "(sparse distances)"}.get(k_used, f"kernel {k_used}")
        roof = {"bound": "l2", "kernel": f"{kname}, G={g_used}", "achieved": gbps, "peak": l2, "unit": "GB/s",
                "frac": gbps / l2, "traffic": traffic, "peak_source": l2src, "hbm_frac": gbps / hbm,
                "hbm_peak_source": hsrc,
                "work": ("per step: 8 H_t d (read + write the updated rows) + 4 nnz(x_t) (N - H_t) (the sparse "
                         "distance's gathered weights) + 8 nnz(x_t) bytes" if sparse else
                         "per step: 4 N d (read W) + 4 H_t d (write updated rows) + 4 d bytes") +
                        f"; H_t from the BMU log (mean {H.mean():.0f} of {N} units), {algo / T / 1e6:.1f} MB/step",
                "kernel_ms": train_ms, "kernel_share_of_step": train_ms / (total_ms / args.steps)}

    # ---- secondary legs
    legs = {}
    if c5 is not None:
        legs["c5_mapping"] = c5_leg(som, torch, args, local, rank, world, c5)
    if args.c4_steps > 0:
        legs["c4_training"] = c4_leg(som, torch, args, local, rank, world)
    if world == 1:
        if args.c2_steps > 0:
            legs["c2"] = c2_leg(som, torch, args, local, seed)
        if args.table3_steps > 0:
            legs["table3"] = table3_leg(som, torch, args, local, seed)
        if args.batch_epochs > 0 and args.config == "c3":
            legs["batch_som"] = batch_leg(som, torch, args, local, seed, (rp, ci, va))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_baseline:
        X, W0 = oracle_inputs(args.config, seed)
        steps_s = {"c1": 2000, "c2": 20000, "c3": 1500}[args.config]        # ~10 s of host work
        r, dt, nt = oracle_train_rate(cfg, X, W0, seed, steps_s)
        cpu = {"value": r, "unit": "samples/s", "cores": nt, "kind": "oracle",
               "sample": f"first {steps_s} of {T} training steps of {args.config} ({dt:.1f} s, fp64 oracle, OpenMP "
                         f"over units); the mapping/QE/U-matrix share of the step is < 1 % on both sides"}
        steps_1 = {"c1": 400, "c2": 1000, "c3": 60}[args.config]
        r1, dt1, _ = oracle_train_rate(cfg, X, W0, seed, steps_1, threads=1)
        cpu["single_core"] = {"value": r1, "unit": "samples/s", "cores": 1,
                              "sample": f"first {steps_1} training steps ({dt1:.1f} s)"}
        cpu["gpu_over_oracle"] = {"all_cores": value / r, "single_core": value / r1}

    ph_mean = {k: statistics.mean(i["phase_ms"][k] for i in infos) for k in infos[0]["phase_ms"]}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64-acc/f32",
        "data": "synthetic (seeded bank-shaped TF-IDF, synth/corpus.py)",
        "config": config_dict(args.config, cfg, world),
        "secondary": {"map_docs_per_s": n / (ph_mean[list(ph_mean)[2]] / 1e3),
                      "train_samples_per_s_kernel": T / (train_ms / 1e3),
                      "us_per_training_step": 1e3 * train_ms / T, "phase_ms": ph_mean,
                      "qe": infos[-1]["qe"], "te": infos[-1]["te"], "train_kernel": k_used, "grid": g_used},
        "e2e": e2e,
        "gpu_launches": infos[-1]["launches"] * args.steps,
        "roofline": roof,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "paper_context": PAPER_44X,
        **legs,
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
