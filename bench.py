"""bench.py — Galerkin panel-pair entries/s (fp64) and end-to-end C-matrix extraction time.

One step = one full single-dielectric C-matrix extraction of the BASELINE.json
configs[1] workload (3-over-3 crossing bus, graded panels, 6 nets): GPU assembly
of all n(n+1)/2 unique entries, DMMA blocked Cholesky, 6 right-hand sides,
charge reduction.  `value` = unique entries / device step time with the panel
list already in HBM; `e2e` = the same through the host-buffer C-ABI call
(gbem_extract_cmatrix: panel H2D + C-matrix D2H inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

N > 1 (launched under torch.distributed.run): every rank extracts its own
instance of the workload (independent scenes, no data-path collective):
weak scaling, max-over-ranks device time.
`--impl reference` runs the reference's own CPU implementation (the reference
headers compiled in oracle/_ref: u_pair_integral on all host threads, plus the
reference Cholesky loop) on a bounded sample per step, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Galerkin panel-pair entries/s (fp64) and end-to-end C-matrix extraction time"
UNIT = "entries/s"


def _peaks() -> dict:
    p = {}
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        p.update(json.loads(f.read_text()))
    fp = ROOT / "profiles" / "fp64_peaks.json"
    if fp.exists():
        p.update(json.loads(fp.read_text()))
    return p


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML (in-process, a few
    microseconds per query) every 250 ms from a background thread started
    BEFORE the warm-up; summary() keeps the samples inside [mark_start,
    mark_end].  (A polling nvidia-smi child process measurably stalled the
    GPU at its start-up and during sampling, so it is not used.)"""

    def __init__(self, device: int):
        self.device = device
        self.rows: list[tuple[float, dict]] = []
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.h = None

    def start(self):
        if os.environ.get("GBEM_NO_CLOCKS"):
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.h = None
            return self
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        return {"sm": sm, "reasons": r}

    def _run(self):
        while not self._stop.wait(0.25):
            try:
                self.rows.append((time.perf_counter(), self._sample()))
            except Exception:
                return

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()
        if self.h is not None:  # at least one sample at the end of the timed region
            try:
                self.rows.append((self.t1, self._sample()))
            except Exception:
                pass

    def stop(self):
        self._stop.set()

    def summary(self) -> dict:
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        nv = self.nv
        inside = [r for t, r in self.rows if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        rows = inside or [r for _, r in self.rows[-3:]]
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({name for r in rows for name, b in bits.items() if r["reasons"] & b})
        sm = [r["sm"] for r in rows]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(rows), "samples_in_timed_region": len(inside), "source": "NVML"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(config: int, seed: int):
    import paper_2203_11733_b200 as g
    m = g.config_model(config, seed=seed)
    ps = m.partition(1)
    ids = m.net_ids
    col = {nid: k for k, nid in enumerate(ids)}
    net = np.array([col.get(int(v), -1) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
    return m, ps, net, len(ids), m.info()["eps_r"]


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2203_11733_b200 import _native as N

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    m, ps, net, K, eps = workload(args.config, args.seed + rank)
    n = len(ps)
    entries = n * (n + 1) // 2
    ctx = N.Context(local)
    # one dedicated stream for torch and the library: the CUDA events below time
    # exactly the work enqueued on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    # device-resident inputs (panel SoA + net index), outputs
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
         dict(axis=ps.axis.astype(np.uint8), level=ps.level, a0=ps.a0, a1=ps.a1, b0=ps.b0, b1=ps.b1).items()}
    d_net = torch.from_numpy(net).to(dev)
    d_C = torch.zeros(K * K, dtype=torch.float64, device=dev)
    d_res = torch.zeros(K, dtype=torch.float64, device=dev)
    dp = C.POINTER(C.c_double)
    panels = N.GbemPanels(C.cast(C.c_void_p(t["axis"].data_ptr()), C.POINTER(C.c_uint8)),
                          *[C.cast(C.c_void_p(t[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
    cfg = ctx.quad()
    lib = ctx.lib

    def step(astats=None, sstats=None):
        rc = lib.gbem_extract_cmatrix_dev(ctx.h, C.byref(panels), n, C.c_void_p(d_net.data_ptr()), K, eps,
                                          C.byref(cfg), C.c_void_p(d_C.data_ptr()), C.c_void_p(d_res.data_ptr()),
                                          astats, sstats)
        ctx.check(rc)

    clk = ClockSampler(local).start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # one instrumented step outside the timed region: per-phase device times, flop counts
    ast, sst = N.GbemAssemblyStats(), N.GbemSolveStats()
    step(C.byref(ast), C.byref(sst))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # stream-ordered mode for the timed steps: no host synchronisation inside a
    # step (the SPD / non-finite checks are read back once by gbem_ctx_sync)
    ctx.check(lib.gbem_ctx_set_async(ctx.h, 1))
    clk.mark_start()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev0.record(stream)
    step_ev[0].record(stream)
    for k in range(args.steps):
        step()
        step_ev[k + 1].record(stream)
    ev1.record(stream)
    ctx.check(lib.gbem_ctx_sync(ctx.h))
    torch.cuda.synchronize()
    clk.mark_end()
    ctx.check(lib.gbem_ctx_set_async(ctx.h, 0))
    step_ms = [step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(args.steps)]
    clk.stop()
    launches = ctx.launches - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    value = world * entries / (ms * 1e-3)
    Cdev = d_C.cpu().numpy().reshape(K, K)

    # e2e: host buffers through the C-ABI (panel H2D + C D2H inside every step)
    P = ps.arrays()
    for _ in range(max(1, args.warmup // 2)):
        ctx.extract_cmatrix(P, net, K, eps, stats=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Ch, res, _, _ = ctx.extract_cmatrix(P, net, K, eps, stats=False)
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    h2d = n * (1 + 5 * 8) + n * 4
    d2h = K * K * 8 + K * 8

    peaks = _peaks()
    # dominant kernels: the Cholesky DMMA trailing update and the far-field Gauss kernel
    chol_flops = n ** 3 / 3.0
    phases = {"assembly_ms": ast.ms_total, "far_ms": ast.ms_far, "near_ms": ast.ms_near,
              "classify_ms": ast.ms_classify, "factor_ms": sst.ms_factor, "solve_ms": sst.ms_solve,
              "residual_ms": sst.ms_residual}
    dmma_peak = peaks.get("fp64_dmma_tflops", 37.09)
    dfma_peak = peaks.get("fp64_dfma_tflops", 36.75)
    traffic = _ncu_traffic()
    roof_chol = {"bound": "tensor", "kernel": "Cholesky factor (k_potrf_diag + k_trsm_rows + k_syrk_gen DMMA update, bordered: forward substitution fused)",
                 "achieved": chol_flops / (sst.ms_factor * 1e-3) / 1e12, "peak": dmma_peak, "unit": "TFLOP/s",
                 "traffic": traffic.get("k_syrk_gen"),
                 "algorithmic": f"n^3/3 = {chol_flops:.3e} flop per factorisation (n = {n}) / device time of the factor",
                 "peak_source": "tools/fp64_peaks.cu DMMA m8n8k4 loop (no FP64 in MEASURED_PEAKS.json)"}
    roof_chol["frac"] = roof_chol["achieved"] / roof_chol["peak"]
    roof_far = {"bound": "fp64_pipe", "kernel": "k_far", "achieved": ast.far_flops / (ast.ms_far * 1e-3) / 1e12,
                "peak": dfma_peak, "unit": "TFLOP/s", "traffic": traffic.get("k_far"),
                "algorithmic": "counted FP64 flops of the Gauss evaluations (dadd, dmul = 1, dfma = 2) / device time",
                "peak_source": "tools/fp64_peaks.cu DFMA loop (no FP64 in MEASURED_PEAKS.json)"}
    roof_far["frac"] = roof_far["achieved"] / roof_far["peak"]
    # each Gauss evaluation issues one MUFU.RSQ64H; its measured rate bounds k_far before the FP64 pipe does
    rsq_rate = peaks.get("rsqrt_f64_custom_per_s", 2.2e12)
    roof_far["mufu_rsq64_bound_frac"] = (ast.far_evals / rsq_rate) / (ast.ms_far * 1e-3)
    # DFMA and DMMA share one FP64 datapath on B200 (tools/pipe_overlap.cu), so the
    # step as a whole is bounded by its total FP64 work at the FP64 peak
    step_flops = chol_flops + ast.far_flops + 2.0 * n * n * K
    fp64_step = {"flops_per_step": step_flops, "achieved_tflops": step_flops / (ms * 1e-3) / 1e12,
                 "peak_tflops": dmma_peak, "frac": step_flops / (ms * 1e-3) / 1e12 / dmma_peak,
                 "note": "Cholesky n^3/3 + far-field Gauss flops + 2 n^2 K triangular solves per step"}
    dominant, secondary = (roof_chol, roof_far) if sst.ms_factor >= ast.ms_far else (roof_far, roof_chol)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config geometry)",
        "config": {"workload": f"config{args.config}: {m_name(args.config)}", "panels": n, "unique_entries": entries,
                   "nets": K, "eps_r": eps, "seed": args.seed,
                   "l2": f"working set {n * n * 8 / 1e9:.2f} GB matrix > 126 MB L2 (no flush needed)",
                   "parallelism": f"replicas{world}" if world > 1 else "single"},
        "e2e": {"value": world * entries / e2e_s, "unit": UNIT, "seconds_per_extraction": e2e_s,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": dominant, "roofline_secondary": secondary, "fp64_step": fp64_step, "phases_ms": phases,
        "assembly": {"pairs_far": ast.pairs_far, "pairs_coplanar": ast.pairs_coplanar,
                     "pairs_parallel": ast.pairs_parallel, "pairs_orthogonal": ast.pairs_orthogonal,
                     "far_evals": ast.far_evals, "near_evals": ast.near_evals, "not_converged": ast.not_converged,
                     "far_flops": ast.far_flops},
        "step_ms": step_ms, "max_residual": sst.max_residual, "gpu_launches": launches, "clocks": clk.summary(),
        "c_matrix_diag_F": [float(Cdev[k, k]) for k in range(K)],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ps, n, budget_s=args.cpu_seconds)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def _ncu_traffic() -> dict:
    """Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
    dominant kernels from the committed ncu --set full captures (profiles/)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return {k: v for k, v in json.load(open(p)).get("bytes_per_launch", {}).items()}
    except (OSError, ValueError):
        return {}


def m_name(cfg: int) -> str:
    return {1: "two parallel boxes, uniform 0.025 um panels", 2: "3-over-3 crossing bus, graded panels",
            3: "8-over-8 bus + ground plane, graded", 4: "64 random Manhattan boxes", 5: "200k random panels"}[cfg]


def _ref_libs():
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O  # test-side loader of oracle/ (CPU checker), used here only for the CPU arm
    if O.ref_available():
        return O, "ref", "reference"
    return O, "orc", "port"


def cpu_sample_rate(ps, n: int, seconds: float, seed: int = 0):
    """Reference u_pair_integral on all host threads over a seeded uniform sample
    of the n(n+1)/2 unique pairs, plus the reference Cholesky loop timed at a
    small size and extrapolated as n^3/3.  Returns (entries/s, details)."""
    O, which, kind = _ref_libs()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    M = ps.matrix()
    # calibrate with a small batch, then size the sample to ~`seconds` of work
    def timed(k):
        i = rng.integers(0, n, size=k)
        j = rng.integers(0, n, size=k)
        lo, hi = np.minimum(i, j), np.maximum(i, j)
        t0 = time.perf_counter()
        O.u_pairs(which, M[lo], M[hi], nthreads=threads)
        return time.perf_counter() - t0
    t = timed(2000)
    k = int(min(5e6, max(2000, 2000 * 0.6 * seconds / max(t, 1e-6))))
    t = timed(k)
    pair_rate = k / t
    # reference Cholesky loop (solver.hpp:28-44 order), single thread, at m = 800
    mch = 800
    A = rng.normal(size=(mch, mch)); A = A @ A.T + mch * np.eye(mch)
    b = np.ones((1, mch))
    X = np.zeros_like(b); res = np.zeros(1); piv = C.c_int64(-1)
    t0 = time.perf_counter()
    O.orc().orc_cholesky_solve(mch, np.ascontiguousarray(A).ctypes.data, 1, b.ctypes.data, X.ctypes.data,
                               res.ctypes.data, C.byref(piv))
    tc = time.perf_counter() - t0
    chol_rate = (mch ** 3 / 3) / tc
    entries = n * (n + 1) / 2
    step_s = entries / pair_rate + (n ** 3 / 3) / chol_rate
    return entries / step_s, {"kind": kind, "cores": threads, "pairs_sampled": k, "pair_rate_per_s": pair_rate,
                              "cholesky_gflops_1thread": chol_rate / 1e9, "extrapolated_step_s": step_s}


def cpu_baseline(ps, n, budget_s=20.0):
    v, d = cpu_sample_rate(ps, n, budget_s)
    return {"value": v, "unit": UNIT, "cores": d["cores"], "kind": d["kind"],
            "sample": (f"{d['pairs_sampled']} seeded uniform unique pairs of the same panel list through the "
                       f"reference u_pair_integral on {d['cores']} threads ({d['pair_rate_per_s']:.3g} pairs/s) + "
                       f"the reference Cholesky loop timed at n=800 ({d['cholesky_gflops_1thread']:.3g} GFLOP/s, "
                       f"1 thread) extrapolated to n^3/3; full CPU step = {d['extrapolated_step_s']:.1f} s"),
            "extrapolated_step_s": d["extrapolated_step_s"]}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    m, ps, net, K, eps = workload(args.config, args.seed)
    n = len(ps)
    per = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    for s in range(args.warmup + args.steps):
        v, d = cpu_sample_rate(ps, n, per, seed=s)
        if s >= args.warmup:
            vals.append((v, d))
    value = float(np.mean([v for v, _ in vals]))
    d = vals[-1][1]
    step_s = n * (n + 1) / 2 / value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config geometry)",
            "config": {"workload": f"config{args.config}: {m_name(args.config)}", "panels": n,
                       "unique_entries": n * (n + 1) // 2, "nets": K},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": d["cores"], "kind": d["kind"],
                             "sample": f"per step {d['pairs_sampled']} sampled pairs on {d['cores']} threads + "
                                       f"reference Cholesky loop at n=800, extrapolated to the full step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
