#!/usr/bin/env python
"""Benchmark driver for the B200 Nested Neumann hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]

Headline (`metric`/`value`): BASELINE config 3 — dense NN inversion, N=32768,
depth p=2, FP64 TFLOP/s.  A *step* is one nest: R = I − A·X (eps fused in)
plus p Horner products, i.e. p+1 = 3 dense 32768³ products
(algorithmic 3·2N³ = 2.11e14 flop).  Inputs are 8.6 GB per matrix (≫ the
126 MB L2), so no L2 flush is needed between steps.  The same line carries
the batched massive-MIMO leg (config 1, inversions/s) and the sparse
factorized leg (config 4, GB/s of algorithmic traffic) under "legs".

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, built from /root/reference/proj/src) on this host's cores on a
bounded sample of the same workload and prints the same metric.
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
from pathlib import Path

_JSON_OUT = sys.stdout  # main() points this at a private duplicate of the original stdout

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = {}
try:
    PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
except Exception:
    pass
HBM_PEAK = PEAKS.get("hbm_gbs", 6650.0)
# Peaks MEASURED_PEAKS.json does not carry, measured on this pool and committed:
# profiles/r02_int8_peak.json (tools/microbench/int8_peak.py: cuBLAS int8 GEMM burst and
# sustained under the power cap; its fp64 entry is the DMMA.8x8x4 microbenchmark of
# tools/microbench/fp64_peak.cu, profiles/r01_fp64_peak.txt).
try:
    EXTRA_PEAKS = json.loads((ROOT / "profiles" / "r02_int8_peak.json").read_text())
except Exception:
    EXTRA_PEAKS = {}
FP64_PEAK_TFLOPS = EXTRA_PEAKS.get("fp64_dmma_tflops", 37.2)
FP64_PEAK_SOURCE = "measured DMMA.8x8x4 microbenchmark, profiles/r01_fp64_peak.txt"
INT8_PEAK_TOPS = EXTRA_PEAKS.get("int8_tops_sustained", 2.0 * PEAKS.get("bf16_tflops_sustained", 1388.0))
INT8_PEAK_SOURCE = ("measured cuBLAS int8 GEMM (torch._int_mm 8192^3) sustained under the power cap, "
                    "profiles/r02_int8_peak.json" if "int8_tops_sustained" in EXTRA_PEAKS else
                    "fallback: 2 x MEASURED_PEAKS bf16_tflops_sustained")
# DRAM traffic per launch of each dominant kernel from the committed ncu --set full captures
try:
    NCU_TRAFFIC = json.loads((ROOT / "profiles" / "r02_ncu_traffic.json").read_text())
except Exception:
    NCU_TRAFFIC = {}


def ncu_traffic(key):
    v = NCU_TRAFFIC.get(key)
    return v["traffic_bytes_per_launch"] if isinstance(v, dict) else None


# ------------------------------------------------------------------ helpers
def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[3 + i]
                          and "Not" not in s[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(force: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or force:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "RANK" not in os.environ:  # --sharded without torchrun: a one-rank group
            import socket

            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, value: float) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, value: float) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


# ------------------------------------------------------------------ dense leg (config 3)
def dense_inputs(n: int, seed: int):
    """A = B·B^T/N + I, B ~ N(0,1) (torch Philox on device); B·B^T runs on libnnb's own GEMM."""
    import torch

    import paper_2212_02406_b200 as nnb

    g = torch.Generator(device="cuda").manual_seed(seed)
    b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    a = nnb.matmul_nt(b, b)  # B·Bᵀ on the K-major GEMM, no transposed copy
    del b
    a = nnb._axpby(1.0 / n, a, 0.0, None, 1.0)  # A/N + I on device
    torch.cuda.synchronize()
    return a


def dense_rows(n: int, seed: int, row0: int, rows: int):
    """Rows [row0, row0+rows) of A = B·B^T/N + I (B regenerated identically on every rank)."""
    import torch

    import paper_2212_02406_b200 as nnb

    g = torch.Generator(device="cuda").manual_seed(seed)
    b = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
    bg = b[row0:row0 + rows].contiguous()
    a = nnb.matmul_nt(bg, b)  # B_g·Bᵀ
    del b, bg
    a = nnb.scale(a, 1.0 / n)
    idx = torch.arange(rows, device="cuda")
    a[idx, idx + row0] += 1.0
    torch.cuda.synchronize()
    return a


def run_dense(args, world, rank):
    import torch

    import paper_2212_02406_b200 as nnb

    n, p = args.n, args.p
    flops_step = (p + 1) * 2.0 * n ** 3  # whole-job work of one nest (strong scaling)
    sharded = world > 1 or args.sharded
    if sharded:
        comm = nnb.Comm.from_torch_distributed()
        row0, rows = nnb.partition_rows(n, world, rank)
        a = dense_rows(n, 2212, row0, rows)
        # X0 = A^T/(|A|_1|A|_inf) (A symmetric), built by the sharded driver's first call
        x, _ = nnb.nn_chain_sharded(comm, a, n, None, p=p, max_iters=0, x0_kind=nnb.X0_TRANSPOSE_NORM)
        chain = lambda xx, k: nnb.nn_chain_sharded(comm, a, n, xx, p=p, max_iters=k, final_residual=False)
    else:
        a = dense_inputs(n, seed=2212)
        x = nnb.x0(a)  # A^T/(|A|_1 |A|_inf) on device
        chain = lambda xx, k: nnb.nn_chain(a, xx, p=p, max_iters=k, final_residual=False)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        x, rep = chain(x, 1)
    torch.cuda.synchronize()
    barrier(world)
    l0 = nnb.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nnb.ozaki_stats(reset=True)
    nnb.ozaki_profile(True)  # CUDA events around each emulation kernel (the live roofline)
    # the timed region is one nn_invert-style call running K nests (a step = one nest), the
    # shape of the C4 workload (12 nests on one A): A's int8 split is formed once per call,
    # as the reference forms nothing per nest for A either (proj/src/solver.cpp:138-159)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        torch.cuda.synchronize()
        e0.record()
        x, rep = chain(x, args.steps)
        e1.record()
        torch.cuda.synchronize()
    nnb.ozaki_profile(False)
    oz = nnb.ozaki_stats(reset=True)
    launches = nnb.kernel_launches() - l0
    eps = [e for _, e in rep.history]
    ms = max_over_ranks(world, e0.elapsed_time(e1))
    barrier(world)
    ms_step = ms / args.steps
    value = flops_step * args.steps / (ms * 1e-3) / 1e12  # whole job: one N^3 nest per step
    dev_ms = rep.device_ms / args.steps
    # the same nests as K one-nest calls (each call re-forms A's split and its buffers),
    # reported beside the headline
    torch.cuda.synchronize()
    barrier(world)
    e0.record()
    for _ in range(args.steps):
        x, _ = chain(x, 1)
    e1.record()
    torch.cuda.synchronize()
    ms_calls = max_over_ranks(world, e0.elapsed_time(e1)) / args.steps
    rows_here = nnb.partition_rows(n, world, rank)[1] if world > 1 else n
    g = oz["gemm"]
    if g["launches"]:
        # dominant kernel: the int8 GEMM of the FP64 emulation (csrc/ozaki.cu), timed live with
        # CUDA events on its stream; work = s moduli x 2*M*N*K int8 ops per launch
        achieved = g["work"] / (g["ms"] * 1e-3) / 1e12
        per_launch = g["work"] / g["launches"]
        moduli = round(per_launch / (2.0 * rows_here * n * n))  # moduli the products actually used
        roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": INT8_PEAK_TOPS, "unit": "TFLOP/s",
                "frac": round(achieved / INT8_PEAK_TOPS, 4),
                "traffic": ncu_traffic("oz_gemm_n32768") if n == 32768 and world == 1 else None,
                "kernel": "oz_gemm_kernel (tcgen05.mma kind::i8 M128 N256 K32, TMEM accumulators x2, 4-stage TMA "
                          "ring, persistent, grouped raster)",
                "unit_note": "int8 tensor ops/s (TOP/s); the FP64-equivalent rate is `value`",
                "per_launch": f"{moduli} moduli x 2*rows*N^2 = {per_launch:.4g} int8 ops (rows={rows_here}, N={n}); "
                              f"{g['launches']} launches, {g['ms'] / g['launches']:.2f} ms mean",
                "share_of_step": round(g["ms"] / (ms / world if world == 1 else dev_ms * args.steps), 4),
                "peak_source": INT8_PEAK_SOURCE,
                "other_kernels": {k: {"ms_per_launch": round(v["ms"] / v["launches"], 3),
                                      "gbs": round(v["work"] / (v["ms"] * 1e-3) / 1e9, 1),
                                      "frac_hbm": round(v["work"] / (v["ms"] * 1e-3) / 1e9 / HBM_PEAK, 3)}
                                  for k, v in oz.items() if k != "gemm" and v["launches"]},
                "fp64_equivalent": {"achieved": round(flops_step / world / (dev_ms * 1e-3) / 1e12, 3),
                                    "dmma_peak": FP64_PEAK_TFLOPS,
                                    "ratio_to_dmma_peak": round(flops_step / world / (dev_ms * 1e-3) / 1e12
                                                                / FP64_PEAK_TFLOPS, 3)}}
    else:
        # DMMA path: the fused FP64 GEMM — the library's device time of a nest is its
        # (p+1) GEMM launches (per rank: its row share of each product)
        achieved = flops_step / world / (dev_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": ncu_traffic("dense_gemm_n32768") if n == 32768 and world == 1 else None,
                "kernel": "gemm_f64_kernel<128x128x16, 2x4 warps, 4 stages> (DMMA.8x8x4 + TMA)",
                "per_launch": f"2*rows*N^2 = {2.0 * rows_here * n * n:.4g} flop (rows={rows_here}, N={n}), "
                              f"{p + 1} launches per nest" + (f" x {world} K-split partials" if world > 1 else ""),
                "peak_source": FP64_PEAK_SOURCE}
    out = dict(value=value, ms_per_step=ms_step, launches=launches, clocks=clk.summary(),
               eps_first=eps[0], eps_last=eps[-1], roofline=roof,
               per_call={"ms_per_nest": round(ms_calls, 2),
                         "tflops": round(flops_step / (ms_calls * 1e-3) / 1e12, 3),
                         "note": "the same nests as one-nest nn_chain calls (A split, buffers and X0 staging "
                                 "per call)"})
    # the same nest with every product on the FP64 tensor pipe (DMMA), for comparison
    if not sharded and args.dmma:
        with nnb.dmma_arithmetic():
            nnb.nn_chain(a, x, p=p, max_iters=1, final_residual=False)  # warm
            torch.cuda.synchronize()
            xd, rd = nnb.nn_chain(a, x, p=p, max_iters=1, final_residual=False)
            torch.cuda.synchronize()
        out["dmma"] = {"arithmetic": "NNB_ARITH_DMMA (every product on DMMA.8x8x4)",
                       "ms_per_nest": round(rd.device_ms, 2),
                       "tflops": round(flops_step / (rd.device_ms * 1e-3) / 1e12, 3),
                       "frac_of_dmma_peak": round(flops_step / (rd.device_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                       "eps_before_nest": rd.history[0][1],
                       "x_rel_frob_vs_headline_nest": float(torch.linalg.norm(xd - chain(x, 1)[0]) / torch.linalg.norm(xd))}
        del xd
    # the 8-rank sharded schedule emulated on this GPU (virtual ranks run one after another):
    # its device time against the single-GPU nest is the per-rank compute efficiency the
    # schedule allows at G=8 (residue splits of the own block, G K-block int8 GEMMs per
    # product, reconstructions of the own rows) before any communication
    if not sharded and args.emulated and n >= 8192:
        out["sharded_emulated"] = run_dense_emulated(nnb, torch, a, x, n, p, 8, ms_step, args.steps)
    # NNB_ORDER_SYMMETRIC on the same nest (A == A^T, X a polynomial in A): upper
    # tile triangles, mirrored — time per nest, reported beside the headline
    if not sharded and args.symmetric:
        out["symmetric"] = run_dense_symmetric(nnb, torch, a, n, p, args)
    # e2e through the C-ABI with HOST buffers (pinned): H2D of A and X, one nest, D2H of X
    if args.e2e:
        shape = tuple(a.shape)
        a_h = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        x_h = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        xo_h = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        a_h.copy_(a)
        x_h.copy_(x)
        del a, x
        torch.cuda.empty_cache()
        nnb.release_cached_memory()  # the legs above left the library's pool holding ≈100 GB
        a_np, x_np, xo_np = a_h.numpy(), x_h.numpy(), xo_h.numpy()
        if sharded:
            call = lambda: nnb.nn_chain_sharded(comm, a_np, n, x_np, p=p, max_iters=1, final_residual=False, out=xo_np)
        else:
            call = lambda: nnb.nn_chain(a_np, x_np, p=p, max_iters=1, final_residual=False, out=xo_np)
        call()  # warm the staging path
        barrier(world)
        t0 = time.perf_counter()
        k_e2e = max(1, min(args.steps, 3))
        for _ in range(k_e2e):
            call()
        t = max_over_ranks(world, time.perf_counter() - t0)
        out["e2e"] = {"value": round(flops_step * k_e2e / t / 1e12, 3), "unit": "TFLOP/s",
                      "h2d_bytes_per_step": 2 * 8 * shape[0] * n * world, "d2h_bytes_per_step": 8 * shape[0] * n * world,
                      "path": ("nnb_nn_chain_sharded_d" if sharded else "nnb_nn_chain_d")
                              + " with pinned host A, X0 and X_out"}
    if sharded:
        comm.close()
    return out


def run_dense_emulated(nnb, torch, a, x, n, p, world, ms_single, k):
    """The `world`-rank sharded schedule as virtual ranks on this GPU, K nests in one call
    (as the headline's K-nest call), against the headline's per-nest time."""
    # warm: the schedule's residue buffers (≈35 GB at N=32768) come from the stream-ordered
    # pool, which grows on the first call (after the other legs' buffers went back)
    torch.cuda.empty_cache()
    nnb.release_cached_memory()
    nnb.nn_chain_sharded_emulated(a, world, x, p=p, max_iters=1, final_residual=False)
    torch.cuda.synchronize()
    nnb.ozaki_stats(reset=True)
    nnb.ozaki_profile(True)
    xe, re_ = nnb.nn_chain_sharded_emulated(a, world, x, p=p, max_iters=k, final_residual=False)
    torch.cuda.synchronize()
    nnb.ozaki_profile(False)
    oz = nnb.ozaki_stats(reset=True)
    # the single-GPU reference timed right after (same clocks: the power-capped int8 GEMM
    # slows as the GPU warms over the legs, so the headline's own time is not the reference)
    xs, rs_ = nnb.nn_chain(a, x, p=p, max_iters=k, final_residual=False)
    torch.cuda.synchronize()
    same = bool(torch.equal(torch.as_tensor(xe, device="cuda"), xs))
    del xe, xs
    torch.cuda.empty_cache()
    ms = re_.device_ms / k
    ms_adj = rs_.device_ms / k
    return {"world": world, "nests": k, "ms_per_nest_all_ranks": round(ms, 2),
            "ms_per_rank_mean": round(ms / world, 2),
            "single_gpu_ms_per_nest": round(ms_adj, 2), "headline_ms_per_nest": round(ms_single, 2),
            "compute_efficiency": round(ms_adj / ms, 4),
            "x_bit_identical_to_single_gpu": same,
            "kernels_ms_per_nest": {c: round(v["ms"] / k, 1) for c, v in oz.items()},
            "note": f"the {world}-rank row-sharded nest (int8-emulated products, residue-block ring) run as {world} "
                    "virtual ranks one after another on this GPU, K nests in one call as the headline; "
                    "communication not included (one GPU)"}


def run_dense_symmetric(nnb, torch, a, n, p, args):
    """The same nests in NNB_ORDER_SYMMETRIC (the order requires the chain to
    build X0 = A^T/(|A|_1|A|_inf) itself, so the K nests run as one call)."""
    k = max(1, min(args.steps, 3))
    nnb.nn_chain(a, None, p=p, max_iters=1, final_residual=False, order=nnb.ORDER_SYMMETRIC)  # warm
    torch.cuda.synchronize()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        xs, rs = nnb.nn_chain(a, None, p=p, max_iters=k, final_residual=False, order=nnb.ORDER_SYMMETRIC)
        torch.cuda.synchronize()
    ms_nest = rs.device_ms / k
    full = (p + 1) * 2.0 * n ** 3
    return {"order": "NNB_ORDER_SYMMETRIC (R = I - A·X full; the p Horner products X·S(R)·R upper tile "
                     "triangle, mirrored)",
            "nests": k, "ms_per_nest": round(ms_nest, 2),
            "tflops_executed": round((1 + p * sym_fraction(n)) * 2.0 * n ** 3 / (ms_nest * 1e-3) / 1e12, 3),
            "full_product_equivalent_tflops": round(full / (ms_nest * 1e-3) / 1e12, 3),
            "eps_first_last": [rs.history[0][1], rs.history[-1][1]], "clocks": clk.summary(),
            "note": "not the headline: the headline times full products, valid for any X0"}


def cpu_dense_sample(n_sample: int, p: int):
    """One reference product (nn::matmul, the routine every NN nest is made of:
    proj/src/kernels.cpp:137-162) on an N=n_sample slice of the config's matrices,
    all host threads (NN_WORKERS=nproc).  The rate is the reference's per-product
    FP64 rate; the N=32768 nest (p+1 products of 2N^3 flop) is extrapolated from it."""
    from oracle import Reference

    from paper_2212_02406_b200 import workloads as W

    cores, _ = cpu_info()
    os.environ["NN_WORKERS"] = str(cores)
    ref = Reference()
    a = W.gram_shifted(n_sample, seed=1, shift=1.0)
    x0 = W.x0_transpose_norm(a)
    ref.matmul(a[:64], a[:, :64])  # warm the worker pool
    t0 = time.perf_counter()
    ref.matmul(a, x0)
    secs = time.perf_counter() - t0
    flops = 2.0 * n_sample ** 3
    return {"value": round(flops / secs / 1e12, 6), "unit": "TFLOP/s", "cores": cores, "kind": "reference",
            "n_sample": n_sample, "extrapolated": True,
            "sample": f"one reference nn::matmul (complex<double>, real data) at N={n_sample}: {secs:.2f} s; "
                      f"the N=32768 nest (p={p}: {p + 1} products) is extrapolated at this per-product rate"}


# ------------------------------------------------------------------ configs 0 and 2 (small / mid dense)
def run_c1(args, rank):
    """BASELINE config 0: N=256 Gram + 0.5 I, X0 = A^T/(|A|_1|A|_inf), Newton (p=1), 30 nests,
    eps per nest.  GPU (device-resident, CUDA events) next to the reference's own loop on the
    same input in the same run (oracle/_ref, all host threads), with the live parity check."""
    import torch

    import paper_2212_02406_b200 as nnb
    from paper_2212_02406_b200 import workloads as W

    a_h = W.gram_shifted(256, seed=2212, shift=0.5)
    a = torch.from_numpy(a_h).cuda()
    for _ in range(3):
        x, rep = nnb.nn_chain(a, None, p=1, max_iters=30)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        x, rep = nnb.nn_chain(a, None, p=1, max_iters=30)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 10 * 1e3
    out = {"metric": "config 0 wall time per 30-nest Newton run (N=256), eps history included", "value": round(ms, 3),
           "unit": "ms", "device_ms": round(rep.device_ms, 3), "products": rep.products,
           "eps_first_last": [rep.history[0][1], rep.history[-1][1]]}
    if rank == 0 and args.cpu:
        from oracle import Reference

        cores, _ = cpu_info()
        os.environ["NN_WORKERS"] = str(cores)
        ref = Reference()
        xr, hr, ir, secs = ref.chain(a_h, W.x0_transpose_norm(a_h), 1, 30)
        xg = x.cpu().numpy()
        out["cpu_reference"] = {"value": round(secs * 1e3, 1), "unit": "ms", "cores": cores, "kind": "reference",
                                "speedup": round(secs * 1e3 / ms, 1)}
        eg = np.array([e for _, e in rep.history])
        above = hr > 1e-12  # floor-region entries compare only as "both below 1e-12"
        out["parity"] = {"x_rel_frob": float(np.linalg.norm(xg - xr.real) / np.linalg.norm(xr.real)),
                         "eps_max_rel_above_floor": float(np.max(np.abs(eg[above] - hr[above]) / hr[above])),
                         "floor_entries_both_below_1e-12": bool(np.all(eg[~above] < 1e-12)),
                         "iterations_equal": rep.iters == ir}
    return out


def sym_fraction(n: int, tile: int = 128) -> float:
    """Share of an n×n product's tiles the symmetric order computes: DMMA's 128×128 tiles
    with tm <= tn below the int8 emulation's crossover (N < 3072), else the int8 GEMM's
    128×256 tiles that meet the upper triangle (128·tm <= 256·tn + 255)."""
    if n >= 3072:
        tm, tn = (n + 127) // 128, (n + 255) // 256
        return sum(1 for m in range(tm) for c in range(tn) if 128 * m <= 256 * c + 255) / (tm * tn)
    t = (n + tile - 1) // tile
    return (t * (t + 1) / 2) / (t * t)


def run_c3(args):
    """BASELINE config 2: N=4096, A = Q diag(lambda) Q^T (kappa 1e3), X0 = A^T/(|A|_1|A|_inf),
    p in {1,2,3}, iterate to eps < 1e-12 — nests needed and TFLOP/s per depth."""
    import torch

    import paper_2212_02406_b200 as nnb

    t0 = time.perf_counter()
    # the reference's own generator, bit for bit (GaussianStream + Householder QR on the device)
    a = torch.from_numpy(nnb.random_spd(4096, 1e3, 3)).cuda()
    gen_s = time.perf_counter() - t0
    res = {}
    for p in (1, 2, 3):
        x, rep = nnb.nn_chain(a, None, p=p, max_iters=80, tol=1e-12)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = nnb.nn_chain(a, None, p=p, max_iters=80, tol=1e-12)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        flops = rep.products * 2.0 * 4096 ** 3
        res[f"p{p}"] = {"nests": rep.iters, "products": rep.products, "stopped": rep.stopped_reason,
                        "eps_last": rep.history[-1][1], "wall_ms": round(wall * 1e3, 2),
                        "device_ms": round(rep.device_ms, 2),
                        "tflops_device": round(flops / (rep.device_ms * 1e-3) / 1e12, 3)}
        # NNB_ORDER_SYMMETRIC: the same chain computing each product's upper tile triangle
        xs, rs = nnb.nn_chain(a, None, p=p, max_iters=80, tol=1e-12, order=nnb.ORDER_SYMMETRIC)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xs, rs = nnb.nn_chain(a, None, p=p, max_iters=80, tol=1e-12, order=nnb.ORDER_SYMMETRIC)
        torch.cuda.synchronize()
        wall_s = time.perf_counter() - t0
        # R = I - A·X products are full, the k·p Horner products upper-triangular
        executed = (rs.products - rs.iters * p + rs.iters * p * sym_fraction(4096)) * 2.0 * 4096 ** 3
        res[f"p{p}"]["symmetric"] = {
            "nests": rs.iters, "stopped": rs.stopped_reason, "eps_last": rs.history[-1][1],
            "wall_ms": round(wall_s * 1e3, 2), "device_ms": round(rs.device_ms, 2),
            "tflops_executed": round(executed / (rs.device_ms * 1e-3) / 1e12, 3),
            "x_rel_frob_vs_full": float(torch.linalg.norm(xs - x) / torch.linalg.norm(x)),
            "speedup_time_to_solution": round(rep.device_ms / rs.device_ms, 3)}
    return {"metric": "config 2: nests to eps < 1e-12 and FP64 TFLOP/s at N=4096 (kappa 1e3)", "depths": res,
            "input": f"nn::random_spd(4096, 1e3, seed=3) on the device, bit-identical to the reference's "
                     f"({gen_s:.2f} s incl. the host GaussianStream)"}


# ------------------------------------------------------------------ MIMO leg (config 1)
def run_mimo(args, world, rank):
    import torch

    import paper_2212_02406_b200 as nnb
    from paper_2212_02406_b200 import workloads as W

    batch = args.mimo_batch
    a = W.mimo_gram_device(batch, seed=1 + rank)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        x, eps = nnb.nn_batched(a, p=2, iters=4)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(args.steps, 5)
    barrier(world)
    e0.record()
    for _ in range(steps):
        x, eps = nnb.nn_batched(a, p=2, iters=4)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(world, e0.elapsed_time(e1)) / steps
    inv_s = sum_over_ranks(world, batch) / (ms * 1e-3)
    # complex 16³ products executed per system: nest 0 from the diagonal Jacobi X0 costs p − 1
    # (its X0·A and P·X0 are scalings), nests 1.. cost p + 1, plus the final residual:
    # 1 + 3·3 + 1 = 11 at p = 2, 4 nests (the generic count would be 13)
    products = (2 - 1) + 3 * (4 - 1) + 1
    # A is exactly Hermitian, so the 7 Horner products (X·poly(P), Hermitian by push-through)
    # compute three of their four 8x8 tiles: 4 + 7·3/4 = 9.25 products' DMMA work executed
    horner = (2 - 1) + 3 * 2
    executed = (products - horner) + 0.75 * horner
    flops = batch * executed * 8.0 * 16 ** 3
    hbm = batch * 2 * 4096.0  # A in + X out (complex128 16x16)
    achieved_tf = flops / (ms * 1e-3) / 1e12
    # a Gram formed by a plain GEMM rounds (i, j) and (j, i) independently, so it is not
    # bit-Hermitian and takes the full products: the rate such a caller sees
    a_gemm = a.clone()
    a_gemm[:, 0, 1] += 1e-17  # one ulp-level asymmetry per system, same conditioning
    for _ in range(2):
        nnb.nn_batched(a_gemm, p=2, iters=4)
    e0.record()
    for _ in range(steps):
        nnb.nn_batched(a_gemm, p=2, iters=4)
    e1.record()
    torch.cuda.synchronize()
    ms_full = max_over_ranks(world, e0.elapsed_time(e1)) / steps
    del a_gemm
    # other user counts (n = 8, 24, 32: batched_generic.cu), the same 262144 systems of NN p=2 ×4
    other_users = {}
    if world == 1:
        for users in (8, 24, 32):
            au = W.mimo_gram_device(batch, seed=5, users=users)
            for _ in range(2):
                nnb.nn_batched(au, p=2, iters=4)
            e0.record()
            for _ in range(3):
                nnb.nn_batched(au, p=2, iters=4)
            e1.record()
            torch.cuda.synchronize()
            ms_u = e0.elapsed_time(e1) / 3
            other_users[f"users_{users}"] = {"ms_per_step": round(ms_u, 3),
                                             "inversions_per_s": round(batch / (ms_u * 1e-3), 1)}
            del au
        torch.cuda.empty_cache()
    # NS baseline of the analytically equivalent term count for 4 nests of p=2: 3^4 - 1 = 80
    for _ in range(2):
        xs = nnb.ns_batched(a, 80)
    e0.record()
    for _ in range(steps):
        xs = nnb.ns_batched(a, 80)
    e1.record()
    torch.cuda.synchronize()
    ms_ns = e0.elapsed_time(e1) / steps
    # accuracy: NN vs NS-80 against torch's inverse on 64 sampled systems
    idx = torch.arange(0, batch, max(1, batch // 64), device="cuda")
    inv = torch.linalg.inv(a[idx])
    rel = lambda y: (torch.linalg.norm(y[idx] - inv, dim=(1, 2)) / torch.linalg.norm(inv, dim=(1, 2))).max().item()
    out = {"metric": "batched inversions/sec (262144 x 16x16 complex128, NN p=2 x4 + eps)",
           "value": round(inv_s, 1), "unit": "inversions/s", "ms_per_step": round(ms, 4),
           "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": FP64_PEAK_TFLOPS,
                        "unit": "TFLOP/s", "frac": round(achieved_tf / FP64_PEAK_TFLOPS, 4),
                        "traffic": ncu_traffic("mimo_batched") if batch == 262144 else None,
                        "hbm_gbs": round(hbm / (ms * 1e-3) / 1e9, 1),
                        "per_launch": f"{batch} systems x {executed} complex 16^3 products executed ({products} "
                                      f"products: nest 0 from the diagonal X0 needs p-1; the {horner} Hermitian "
                                      "Horner products run 3 of 4 8x8 tiles) x 8*16^3 flop (4M-equivalent)",
                        "algorithmic_tflops_13_products": round(batch * 13 * 8.0 * 16 ** 3 / (ms * 1e-3) / 1e12, 3)},
           "other_user_counts": other_users or None,
           "non_hermitian_input": {"ms_per_step": round(ms_full, 4),
                                   "inversions_per_s": round(sum_over_ranks(world, batch) / (ms_full * 1e-3), 1),
                                   "note": "A not bit-Hermitian (a GEMM-formed Gram): all 11 products full"},
           "ns80_baseline": {"ms_per_step": round(ms_ns, 4), "inversions_per_s": round(batch / (ms_ns * 1e-3), 1),
                             "speedup_nn_over_ns": round(ms_ns / ms, 3)},
           "accuracy": {"nn_max_rel_err": rel(x), "ns80_max_rel_err": rel(xs), "eps_max": eps.max().item()}}
    # fused detection: H, y in HBM -> Gram, NN inverse, x̂ = X·Hᴴy
    del x, xs
    h, y, sym = W.mimo_uplink_device(batch, seed=3 + rank)
    for _ in range(2):
        xh, _, _ = nnb.mimo_detect(h, y)
    e0.record()
    for _ in range(steps):
        xh, _, _ = nnb.mimo_detect(h, y)
    e1.record()
    torch.cuda.synchronize()
    ms_det = max_over_ranks(world, e0.elapsed_time(e1)) / steps
    # executed: the Hermitian Gram's three upper 8×8 tiles (¾ of 8·16·16·128), the NN products, z = Hᴴy, x̂ = X·z
    det_flops = batch * (0.75 * 8.0 * 16 * 16 * 128 + executed * 8.0 * 16 ** 3 + 8.0 * 16 * 128 + 8.0 * 256)
    det_bytes = batch * (128 * 16 * 16 + 128 * 16 + 16 * 16)
    sym_ok = ((torch.sign(xh.real) == torch.sign(sym.real)) & (torch.sign(xh.imag) == torch.sign(sym.imag)))
    out["detect"] = {"metric": "fused MIMO detections/sec (Gram + NN p=2 x4 + x̂ = X·Hᴴy, 128x16 uplinks)",
                     "value": round(sum_over_ranks(world, batch) / (ms_det * 1e-3), 1), "unit": "detections/s",
                     "ms_per_step": round(ms_det, 4),
                     "achieved_tflops": round(det_flops / (ms_det * 1e-3) / 1e12, 3),
                     "hbm_gbs": round(det_bytes / (ms_det * 1e-3) / 1e9, 1),
                     "qpsk_symbol_accuracy": round(sym_ok.double().mean().item(), 6)}
    del h, y, sym, xh
    torch.cuda.empty_cache()
    if args.e2e:
        a_h = torch.empty(tuple(a.shape), dtype=torch.complex128, pin_memory=True)
        x_h = torch.empty(tuple(a.shape), dtype=torch.complex128, pin_memory=True)
        a_h.copy_(a)
        a_np, x_np = a_h.numpy(), x_h.numpy()
        nnb.nn_batched(a_np, p=2, iters=4, want_eps=False, out=x_np)
        t0 = time.perf_counter()
        for _ in range(3):
            nnb.nn_batched(a_np, p=2, iters=4, want_eps=False, out=x_np)
        t = (time.perf_counter() - t0) / 3
        out["e2e"] = {"value": round(batch / t, 1), "unit": "inversions/s", "h2d_bytes_per_step": batch * 4096,
                      "d2h_bytes_per_step": batch * 4096, "path": "nnb_nn_batched_z with pinned host A and X"}
    return out


def cpu_mimo_sample(sample: int):
    from oracle import Reference

    from paper_2212_02406_b200 import workloads as W

    cores, _ = cpu_info()
    ref = Reference()
    a = W.mimo_gram_host(sample, seed=1)
    _, _, secs = ref.batched("nn", a, 2, 4, threads=cores)
    return {"value": round(sample / secs, 1), "unit": "inversions/s", "cores": cores, "kind": "reference",
            "sample": f"{sample} systems, reference nn_step x4 (p=2) + residual_epsilon per system, "
                      f"{cores} std::threads ({secs:.2f} s)"}


# ------------------------------------------------------------------ sparse leg (config 4)
def sparse_bytes(n, nnz, nnz_bytes=12):
    """Bytes of one application: nnz_bytes per nonzero, int32 row offsets, t read + t written per row.
    nnz_bytes = 12 (f64 value + int32 column) is SURVEY.md §8(d)'s algorithmic figure and the work unit
    of the metric; the format the kernel actually consumes (1: pair dictionary, 10: f64 + int16 column
    delta, 12) gives the roofline's bytes."""
    return nnz * nnz_bytes + (n + 1) * 4 + 2 * n * 8


def run_sparse(args, world, rank):
    import torch

    import paper_2212_02406_b200 as nnb
    from paper_2212_02406_b200 import workloads as W

    grid = args.grid
    n = grid * grid
    rp, col, val = W.laplacian_5pt(grid)
    dev = lambda v: torch.from_numpy(v).cuda()
    b_full = W.rhs(n, seed=7)
    norm = nnb.Normalization(theta=0.2, valid=True)
    sharded = world > 1 or args.sharded
    if sharded:
        # row slabs with halo exchange (strong scaling: the 4096^2 problem is fixed)
        comm = nnb.Comm.from_torch_distributed()
        r0, rows = nnb.partition_rows(n, world, rank)
        csr = nnb.Csr(dev(rp[r0:r0 + rows + 1].copy()), dev(col), dev(val), n=rows, nnz=col.size)
        b = dev(b_full[r0:r0 + rows].copy())
        # one-shot sharded solve: the slab's format pass runs inside every step, as the
        # single-GPU solve's does, so every N times the same per-solve work
        solve = lambda: nnb.solve_sparse_factorized_sharded(comm, csr, n, b, 63, norm)
        plan = nnb.SparseShardedPlan(comm, csr, n, k=1, stream_like=b)  # planned solve, reported beside it
        plan_solve = lambda: plan.solve(b, 63, norm)
    else:
        csr = nnb.Csr(dev(rp), dev(col), dev(val), n=n, nnz=col.size)
        b = dev(b_full)
        solve = lambda: nnb.solve_sparse_factorized(csr, b, 63, norm)
    for _ in range(args.warmup):
        x, _ = solve()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(args.steps, 100)  # ≈0.35 s of solves: long enough for the clock samples
    barrier(world)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        e0.record()
        for _ in range(steps):
            x, _ = solve()
        e1.record()
        torch.cuda.synchronize()
    ms = max_over_ranks(world, e0.elapsed_time(e1)) / steps
    planned_ms = None
    if sharded:
        for _ in range(2):
            plan_solve()
        barrier(world)
        e0.record()
        for _ in range(steps):
            plan_solve()
        e1.record()
        torch.cuda.synchronize()
        planned_ms = max_over_ranks(world, e0.elapsed_time(e1)) / steps
        plan.close()
        comm.close()
    # the format the device consumed (csrc/sparse.cu): 1 = pair dictionary, 10 = f64 + int16 delta, 12
    fb = nnb.sparse_last_bytes_per_nnz()
    fname = nnb.sparse_last_format()
    fmt = {"row-dictionary": "1-byte row-pattern codes (<= 256 distinct (column - row, value) rows), no row offsets",
           "pair-dictionary-ell": "1-byte (column - row, value) pair-dictionary codes, slot-major ELL (no row offsets)",
           "pair-dictionary-csr": "1-byte pair-dictionary codes, int32 row offsets",
           "csr-int16-delta": "f64 values + int16 column deltas, int32 row offsets",
           "csr-int32": "f64 values + int32 columns, row offsets"}.get(fname, fname)
    mat = sum_over_ranks(world, float(nnb.sparse_last_matrix_bytes())) if sharded else nnb.sparse_last_matrix_bytes()
    general = None
    if not sharded:
        # the same operator shape with per-entry random weights (no value dictionary applies):
        # the general-CSR rate (int16 column deltas + f64 values), beside the stencil formats
        rng = np.random.default_rng(11)
        val_g = val.copy()
        off = val_g != 5.0
        val_g[off] = -rng.uniform(0.5, 1.0, int(off.sum()))
        csr_g = nnb.Csr(dev(rp), dev(col), dev(val_g), n=n, nnz=col.size)
        for _ in range(2):
            nnb.solve_sparse_factorized(csr_g, b, 63, norm)
        e0.record()
        for _ in range(3):
            nnb.solve_sparse_factorized(csr_g, b, 63, norm)
        e1.record()
        torch.cuda.synchronize()
        ms_g = e0.elapsed_time(e1) / 3
        fb_g = nnb.sparse_last_bytes_per_nnz()
        mat_g = nnb.sparse_last_matrix_bytes()
        general = {"ms_per_step": round(ms_g, 3), "format": nnb.sparse_last_format(),
                   "gbs_algorithmic": round(63 * sparse_bytes(n, col.size, 12) / (ms_g * 1e-3) / 1e9, 1),
                   "frac_hbm_consumed_format": round(63 * (mat_g + 2 * n * 8) / (ms_g * 1e-3) / 1e9 / HBM_PEAK, 4),
                   "bytes_per_nnz": fb_g,
                   "note": "same 4096^2 5-point pattern, off-diagonal values random in [-1, -0.5]: no dictionary"}
        del csr_g
    emulated = None
    if not sharded and args.emulated:
        # the 8-slab schedule as 8 virtual ranks one after another on this GPU (halo copies on
        # the device; no NVLink): its time against the single-GPU solve
        for _ in range(2):
            xe, _ = nnb.solve_sparse_factorized_sharded_emulated(csr, b, 63, norm, 8)
        e0.record()
        for _ in range(5):
            xe, _ = nnb.solve_sparse_factorized_sharded_emulated(csr, b, 63, norm, 8)
        e1.record()
        torch.cuda.synchronize()
        ms_e = e0.elapsed_time(e1) / 5
        ms_sched = nnb.sparse_last_solve_ms()  # the last solve without its 8 slab setups
        emulated = {"world": 8, "ms_per_solve_all_ranks": round(ms_e, 3), "single_gpu_ms": round(ms, 3),
                    "compute_efficiency": round(ms / ms_e, 4),
                    "schedule_ms_all_ranks": round(ms_sched, 3),
                    "schedule_efficiency": round(ms / ms_sched, 4) if ms_sched > 0 else None,
                    "format": nnb.sparse_last_format(),
                    "x_bit_identical_to_single_gpu": bool(torch.equal(xe, x)),
                    "note": "row slabs of 512 grid rows, temporal-blocked passes with an 8-row halo exchanged once "
                            "per pass (device copies here); compute_efficiency: one-shot solves incl. the 8 slab "
                            "setups (run in parallel on 8 GPUs, one after another here); schedule_efficiency: the "
                            "factor schedule alone (the single-GPU time includes its format pass)"}
    alg = 63 * sparse_bytes(n, col.size, 12)  # SURVEY §8(d) algorithmic bytes per solve: the work unit
    moved = 63 * (mat + 2 * n * 8)  # bytes of the consumed format (operator + t in + t out): the roofline
    gbs, moved_gbs = alg / (ms * 1e-3) / 1e9, moved / (ms * 1e-3) / 1e9
    if fname == "row-dictionary-stencil-tb":
        # temporal blocking: t crosses HBM once per pass of up to 4 applications (plus halos),
        # so the bytes moved per application are below one read + one write of t
        per_launch = (f"{moved / 63:.0f} bytes moved per application, averaged over the solve's 17 passes "
                      "(t in + t out once per pass of up to 4 applications, 1-byte row codes; whole solve timed "
                      "incl. the per-solve format pass); the pass is issue-bound "
                      "(profiles/r02_ncu_stencil_tb.txt), so this fraction is not its limit")
    else:
        per_launch = (f"{mat:.0f} operator bytes + 2N*8 per application (x63, whole solve timed "
                      f"incl. the per-solve format pass): {fmt}; t in + t out")
    return {"metric": "sparse factorized solve, 4096^2 5-pt Laplacian+I, gamma=63 (GB/s of SURVEY 8(d) algorithmic "
                      "bytes: 12 B per nonzero)", "value": round(gbs, 1),
            "unit": "GB/s", "ms_per_step": round(ms, 3), "format": fname, "format_bytes_per_nnz": fb,
            "planned_ms_per_step": None if planned_ms is None else round(planned_ms, 3),
            "general_csr": general, "sharded_emulated": emulated,
            "parallelism": f"row slabs x{world}, NCCL halo exchange" if sharded else "single GPU",
            "roofline": {"bound": "hbm", "achieved": round(moved_gbs, 1), "peak": HBM_PEAK * world, "unit": "GB/s",
                         "frac": round(moved_gbs / (HBM_PEAK * world), 4),
                         "traffic": ncu_traffic("sparse_application") if grid == 4096 and not sharded else None,
                         "traffic_unit": "bytes per application (63 per solve)",
                         "per_launch": per_launch},
            "clocks": clk.summary()}


def cpu_sparse_sample(grid: int):
    from oracle import Reference

    from paper_2212_02406_b200 import workloads as W

    cores, _ = cpu_info()
    os.environ["NN_WORKERS"] = str(cores)
    ref = Reference()
    rp, col, val = W.laplacian_5pt(grid)
    b = W.rhs(grid * grid, seed=7)
    _, _, secs = ref.sparse_factorized(rp, col, val, b, 63, 0.2)
    gbs = 63 * sparse_bytes(grid * grid, col.size, 12) / secs / 1e9  # same unit as the GPU leg
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"reference solve_sparse_factorized gamma=63 on a {grid}^2 grid ({secs:.2f} s)"}


# ------------------------------------------------------------------ launcher
def relaunch_under_torchrun(argv, gpus: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: start N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1 and return its exit status.  Refuses
    loudly when the node has fewer than N GPUs instead of running fewer ranks."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < gpus:
        print(f"bench.py: --gpus {gpus} requested but this node has {have} CUDA device(s); "
              "refusing to run fewer ranks than requested", file=sys.stderr, flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]
    return subprocess.run(cmd).returncode


# ------------------------------------------------------------------ main
def main():
    # stdout carries exactly the one JSON line: native libraries (NCCL prints its version
    # line at communicator init) write to fd 1, so fd 1 becomes stderr for the run and
    # the JSON goes to a private duplicate of the original stdout
    global _JSON_OUT
    pre = argparse.ArgumentParser(add_help=False)
    pre.add_argument("--gpus", type=int, default=1)
    pre.add_argument("--impl", default="ours")
    pre.add_argument("--sharded", action="store_true")
    known, _ = pre.parse_known_args()
    if "WORLD_SIZE" not in os.environ and known.impl == "ours" and (known.gpus > 1 or known.sharded):
        sys.exit(relaunch_under_torchrun(sys.argv[1:], known.gpus))
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--matrix-n", dest="n", type=int, default=32768)
    ap.add_argument("--depth", dest="p", type=int, default=2)
    ap.add_argument("--mimo-batch", type=int, default=262144)
    ap.add_argument("--grid", type=int, default=4096)
    ap.add_argument("--legs", default="dense,mimo,sparse,c1,c3")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-symmetric", dest="symmetric", action="store_false",
                    help="skip the NNB_ORDER_SYMMETRIC timing beside the headline nest")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-emulated", dest="emulated", action="store_false",
                    help="skip the 8-rank sharded schedule emulated on one GPU")
    ap.add_argument("--no-dmma", dest="dmma", action="store_false",
                    help="skip the DMMA-only timing of the headline nest")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded) dense/sparse paths even at one rank (code-path check)")
    args = ap.parse_args()
    legs = set(args.legs.split(","))
    world, rank, local = dist_setup(args.sharded) if args.impl == "ours" else (int(os.environ.get("WORLD_SIZE", "1")),
                                                                   int(os.environ.get("RANK", "0")), 0)
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch with --nproc-per-node {args.gpus}",
              file=sys.stderr, flush=True)
        sys.exit(2)
    cores, model = cpu_info()
    config = {"workload": f"BASELINE config 3: dense NN inversion N={args.n}, p={args.p}, one nest per step "
                          f"(A=B·B^T/N+I, X0=A^T/(|A|_1|A|_inf)); the K timed steps run as one K-nest "
                          f"nn_chain call (legs.dense_one_nest_calls: K one-nest calls)",
              "n": args.n, "depth_p": args.p, "products_per_step": args.p + 1,
              "l2": "inputs (8*N^2 bytes per matrix) exceed the 126 MB L2; no flush",
              "parallelism": f"row-sharded x{world} (int8-emulated products: column statistics all-gathered, "
                             "residue blocks moved by an NCCL ring overlapped with the K-block int8 GEMMs)"
                             if world > 1 or args.sharded else "single GPU",
              "host_cpu": f"{cores} x {model}"}
    base = {"metric": "NN inversion FP64 TFLOP/s", "unit": "TFLOP/s", "n_gpus": world if args.impl == "ours" else args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded)", "config": config,
            "arithmetic": "NNB_ARITH_FAST: each real N^3 product (N >= 3072) runs as an FP64-accurate emulation on "
                          "the int8 tensor cores (Ozaki scheme II: 53-bit row/column-scaled integers, 16 moduli, "
                          "exact int32 accumulation, CRT-sum reconstruction; csrc/ozaki.cu) - same parity gate as "
                          "DMMA (X within 1e-10, identical nest counts); smaller/complex products on DMMA"}
    if world > 1:
        base["scaling"] = "strong"  # the N=32768 matrix is fixed; ranks split its rows

    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's own CPU path (oracle/_ref), all host threads, bounded sample per step
        t0 = time.perf_counter()
        vals = []
        for _ in range(args.warmup + args.steps):
            vals.append(cpu_dense_sample(1024, args.p))
        v = statistics.median(x["value"] for x in vals[args.warmup:]) if args.steps else vals[-1]["value"]
        cb = dict(vals[-1])
        cb["value"] = v
        # the trend the extrapolation rests on: the same product once at N=2048
        cb["n2048_once"] = cpu_dense_sample(2048, args.p)["value"]
        line = dict(base, impl="reference", value=v, ms_per_step=round((time.perf_counter() - t0) * 1e3 /
                                                                       max(1, len(vals)), 1),
                    cpu_baseline=cb, e2e={"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0})
        print(json.dumps(line), file=_JSON_OUT, flush=True)
        return

    import torch

    import paper_2212_02406_b200 as nnb

    nnb.lib()
    torch.cuda.set_device(local)
    line = dict(base)
    line["legs"] = {}
    if "dense" in legs:
        d = run_dense(args, world, rank)
        line.update(value=round(d["value"], 3), ms_per_step=round(d["ms_per_step"], 2),
                    roofline=d["roofline"], clocks=d["clocks"], gpu_launches=d["launches"])
        line["legs"]["dense_one_nest_calls"] = d["per_call"]
        if "e2e" in d:
            line["e2e"] = d["e2e"]
        if "symmetric" in d:
            line["legs"]["dense_symmetric"] = d["symmetric"]
        if "dmma" in d:
            line["legs"]["dense_dmma"] = d["dmma"]
        if "sharded_emulated" in d:
            line["legs"]["dense_sharded_emulated"] = d["sharded_emulated"]
        config["eps_first_last"] = [d["eps_first"], d["eps_last"]]
    if "mimo" in legs:
        line["legs"]["mimo"] = run_mimo(args, world, rank)
    if "sparse" in legs:
        line["legs"]["sparse"] = run_sparse(args, world, rank)
    if "c1" in legs and world == 1:
        line["legs"]["c1"] = run_c1(args, rank)
    if "c3" in legs and world == 1:
        line["legs"]["c3"] = run_c3(args)
    if rank == 0 and args.cpu:
        line["cpu_baseline"] = cpu_dense_sample(1024, args.p)
        if "mimo" in legs:
            line["legs"]["mimo"]["cpu_baseline"] = cpu_mimo_sample(16384)
        if "sparse" in legs:
            line["legs"]["sparse"]["cpu_baseline"] = cpu_sparse_sample(512)
    if rank == 0:
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    if world > 1 or args.sharded:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
