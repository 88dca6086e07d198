"""bench.py — Galerkin panel-pair entries/s (fp64) and end-to-end C-matrix extraction time.

N = 1 (default): one step = one full single-dielectric C-matrix extraction of
BASELINE config 3 (8-over-8 crossing bus + ground plane, graded panels, 33,776
panels, 17 nets; the largest single-GPU config): GPU assembly of all n(n+1)/2
unique entries, bordered DMMA Cholesky (forward substitution and C = Y^T Y
fused), backward substitution, residual.  `value` = unique entries / device step
time with the panels already in HBM; `e2e` = the same through the host-buffer
C-ABI call (gbem_extract_cmatrix: panel H2D + C-matrix D2H inside the timed
region).  The line also carries the sharded workloads measured at N = 1
(`sharded_n1`) so the N > 1 lines have their own single-GPU reference.

N > 1 (launched under torch.distributed.run, one rank per GPU, NCCL): one step =
the config-4 C-matrix (96,200 panels, 64 nets) on row-block shards —
full-row assembly with no communication, block-Jacobi PCG with the NCCL
all-gather / all-reduce owned by the library's context (gbem_pcg_extract_cmatrix_dev)
— strong scaling (fixed problem), max-over-ranks device time; plus the config-5
assembly-only stress test (200k panels) on work-balanced row blocks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload extract|sharded] [--config C]

`--impl reference` runs the reference's own CPU implementation (the reference
headers compiled in oracle/_ref: u_pair_integral on all host threads, plus the
reference Cholesky loop in its column-major order) on a bounded sample per
step, rank 0 only, on the same panel list read from workloads/*.npz (no
library of this repository is loaded in that process).
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


def m_name(cfg: int) -> str:
    return {1: "two parallel boxes, uniform 0.025 um panels", 2: "3-over-3 crossing bus, graded panels",
            3: "8-over-8 bus + ground plane, graded", 4: "64 random Manhattan boxes", 5: "200k random panels"}[cfg]


def serialized_workload(config: int):
    """The panel list, net index, K and eps_r of a config from workloads/*.npz
    (pure numpy: the reference arm loads none of this repository's libraries)."""
    d = np.load(ROOT / "workloads" / f"config{config}_panels.npz")
    return d["panels"], d["net"], int(d["nets"]), float(d["eps_r"]), int(d["seed"])


def extract_config(config: int, n: int, K: int, eps: float, seed: int) -> dict:
    """The `config` object of the N = 1 extraction line (identical in both arms)."""
    return {"workload": f"config{config}: {m_name(config)}", "panels": n, "unique_entries": n * (n + 1) // 2,
            "nets": K, "eps_r": eps, "seed": seed,
            "l2": (f"working set {n * n * 8 / 1e9:.2f} GB matrix > 126 MB L2 (no flush needed)" if n * n * 8 > 126e6
                   else f"working set {n * n * 8 / 1e6:.1f} MB matrix fits the 126 MB L2 and is not flushed "
                        "(a secondary config, not the headline)"),
            "parallelism": "single"}


def sharded_config(world: int, n4: int, K4: int, n5: int) -> dict:
    """The `config` object of the N > 1 line (identical in both arms)."""
    return {"workload": "config4 sharded C-matrix (row blocks + block-Jacobi PCG over NCCL); "
                        "config5 assembly-only (work-balanced row blocks)",
            "panels": n4, "unique_entries": n4 * (n4 + 1) // 2, "nets": K4, "seed": 1,
            "config5_panels": n5, "config5_unique_entries": n5 * (n5 + 1) // 2,
            "l2": "row blocks of several GB per rank > 126 MB L2 (no flush needed)",
            "parallelism": f"rowblock{world}"}


def _panels_struct(N, t):
    dp = C.POINTER(C.c_double)
    return N.GbemPanels(C.cast(C.c_void_p(t["axis"].data_ptr()), C.POINTER(C.c_uint8)),
                        *[C.cast(C.c_void_p(t[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])


def _to_dev(P: np.ndarray, dev):
    import torch
    cols = dict(axis=P[:, 0].astype(np.uint8), level=P[:, 1], a0=P[:, 2], a1=P[:, 3], b0=P[:, 4], b1=P[:, 5])
    return {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}


# ----------------------------------------------------------------------------- N = 1: config-3 extraction

def run_extract(args):
    import torch
    from paper_2203_11733_b200 import _native as N
    import paper_2203_11733_b200 as g

    local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    m = g.config_model(args.config, seed=args.seed)
    ps = m.partition(1)
    ids = m.net_ids
    col = {nid: k for k, nid in enumerate(ids)}
    net = np.array([col.get(int(v), -1) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
    K, eps = len(ids), m.info()["eps_r"]
    n = len(ps)
    entries = n * (n + 1) // 2
    ctx = N.Context(local)
    # one dedicated stream for torch and the library: the CUDA events below time
    # exactly the work enqueued on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    t = _to_dev(ps.matrix(), dev)
    panels = _panels_struct(N, t)
    d_net = torch.from_numpy(net).to(dev)
    d_C = torch.zeros(K * K, dtype=torch.float64, device=dev)
    d_res = torch.zeros(K, dtype=torch.float64, device=dev)
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
    launches = ctx.launches - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    value = entries / (ms * 1e-3)
    Cdev = d_C.cpu().numpy().reshape(K, K)

    # e2e: host buffers through the C-ABI (panel H2D + C D2H inside every step)
    P = ps.arrays()
    for _ in range(max(1, args.warmup // 2)):
        ctx.extract_cmatrix(P, net, K, eps, stats=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Ch, res, _, _ = ctx.extract_cmatrix(P, net, K, eps, stats=False)
    e2e_s = (time.perf_counter() - t0) / args.steps
    clk.stop()
    h2d = n * (1 + 5 * 8) + n * 4
    d2h = K * K * 8 + K * 8

    peaks = _peaks()
    chol_flops = n ** 3 / 3.0
    phases = {"assembly_ms": ast.ms_total, "far_ms": ast.ms_far, "near_ms": ast.ms_near,
              "classify_ms": ast.ms_classify, "factor_ms": sst.ms_factor, "solve_ms": sst.ms_solve,
              "residual_ms": sst.ms_residual}
    dmma_peak = peaks.get("fp64_dmma_tflops", 37.09)
    dfma_peak = peaks.get("fp64_dfma_tflops", 36.75)
    traffic = _ncu_traffic()
    roof_chol = {"bound": "tensor", "kernel": "Cholesky factor (k_potrf_diag + k_trsm_rows + k_syrk_bulk DMMA update, "
                                              "bordered: forward substitution fused)",
                 "achieved": chol_flops / (sst.ms_factor * 1e-3) / 1e12, "peak": dmma_peak, "unit": "TFLOP/s",
                 "traffic": traffic.get("k_syrk_bulk", traffic.get("k_syrk_gen")),
                 "algorithmic": f"n^3/3 = {chol_flops:.3e} flop per factorisation (n = {n}) / device time of the factor",
                 "peak_source": "tools/fp64_peaks.cu DMMA m8n8k4 loop (no FP64 in MEASURED_PEAKS.json)"}
    roof_chol["frac"] = roof_chol["achieved"] / roof_chol["peak"]
    upd = _ncu_traffic_file().get("update_kernel", {})
    if upd:
        roof_chol["update_kernel_ncu"] = upd
    roof_far = {"bound": "fp64_pipe", "kernel": "k_far", "achieved": ast.far_flops / (ast.ms_far * 1e-3) / 1e12,
                "peak": dfma_peak, "unit": "TFLOP/s", "traffic": traffic.get("k_far"),
                "algorithmic": "counted FP64 flops of the Gauss evaluations (dadd, dmul = 1, dfma = 2) / device time",
                "peak_source": "tools/fp64_peaks.cu DFMA loop (no FP64 in MEASURED_PEAKS.json)"}
    roof_far["frac"] = roof_far["achieved"] / roof_far["peak"]
    # one MUFU.RSQ64H per node against its measured issue rate, and the node's whole instruction
    # mix (3 DFMA + DMUL + MUFU + the seed's low-word move) against its measured rate
    roof_far["mufu_rsq64h_frac"] = (ast.far_evals / peaks.get("mufu_rsq64h_per_s", 4.62e12)) / (ast.ms_far * 1e-3)
    roof_far["node_mix_frac"] = (ast.far_evals / peaks.get("far_node_mix_per_s", 3.22e12)) / (ast.ms_far * 1e-3)
    pipe = _ncu_traffic_file().get("fp64_pipe_active", {})
    if pipe:
        roof_far["fp64_pipe_active_ncu"] = pipe.get("k_far")
        roof_far["fp64_pipe_active_ncu_source"] = pipe.get("source")
    step_flops = chol_flops + ast.far_flops + 2.0 * n * n * K
    fp64_step = {"flops_per_step": step_flops, "achieved_tflops": step_flops / (ms * 1e-3) / 1e12,
                 "peak_tflops": dmma_peak, "frac": step_flops / (ms * 1e-3) / 1e12 / dmma_peak,
                 "note": "Cholesky n^3/3 + far-field Gauss flops + 2 n^2 K triangular solves per step "
                         "(DFMA and DMMA share one FP64 datapath, tools/pipe_overlap.cu)"}
    dominant, secondary = (roof_chol, roof_far) if sst.ms_factor >= ast.ms_far else (roof_far, roof_chol)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config geometry)",
        "config": extract_config(args.config, n, K, eps, args.seed),
        "e2e": {"value": entries / e2e_s, "unit": UNIT, "seconds_per_extraction": e2e_s,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": dominant, "roofline_secondary": secondary, "fp64_step": fp64_step, "phases_ms": phases,
        "assembly": {"pairs_far": ast.pairs_far, "pairs_coplanar": ast.pairs_coplanar,
                     "pairs_parallel": ast.pairs_parallel, "pairs_orthogonal": ast.pairs_orthogonal,
                     "pairs_near_romberg": ast.pairs_near_romberg, "pairs_near_band": list(ast.pairs_near_band),
                     "far_evals": ast.far_evals, "near_evals": ast.near_evals, "not_converged": ast.not_converged,
                     "far_flops": ast.far_flops},
        "step_ms": step_ms, "max_residual": sst.max_residual, "gpu_launches": launches, "clocks": clk.summary(),
        "c_matrix_diag_F": [float(Cdev[k, k]) for k in range(K)],
    }
    ctx.close()
    del t, d_net, d_C, d_res
    torch.cuda.empty_cache()
    if not args.no_sharded:
        line["sharded_n1"] = sharded_n1(args)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ps.matrix(), n, K, budget_s=args.cpu_seconds)
    print(json.dumps(line), flush=True)


def sharded_n1(args) -> dict:
    """The N > 1 workloads at N = 1 (1 warm-up + 2 timed steps each): the
    single-GPU reference of the strong-scaling lines."""
    import torch
    from paper_2203_11733_b200 import _native as N
    P4, net4, K4, eps4, _ = serialized_workload(4)
    out = {}
    ctx = N.Context(0)
    r = sharded_extract_steps(ctx, P4, net4, K4, eps4, 1, 2, world=1, jacobi_rows=args.jacobi_rows)
    out["config4_pcg"] = r
    ctx.close()
    torch.cuda.empty_cache()
    ctx = N.Context(0)
    out["config5_assembly"] = config5_assembly_steps(ctx, 1, 2, world=1, rank=0)
    ctx.close()
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- sharded workloads

def sharded_extract_steps(ctx, P, net, K, eps, warmup, steps, world, jacobi_rows=12032, group=None):
    """Config-4 C-matrix on row-block shards through gbem_pcg_extract_cmatrix_dev:
    device-timed steps (panels resident) and host-buffer e2e steps
    (paper_2203_11733_b200.pcg.sharded_cmatrix: panel H2D + C D2H inside)."""
    import torch
    import torch.distributed as dist
    from paper_2203_11733_b200 import _native as N
    from paper_2203_11733_b200.pcg import attach, sharded_cmatrix, equal_row_split
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    attach(ctx, group)
    ctx.set_stream(stream.cuda_stream)
    n = len(P)
    t = _to_dev(P, dev)
    panels = _panels_struct(N, t)
    d_net = torch.from_numpy(np.ascontiguousarray(net, dtype=np.int32)).to(dev)
    d_C = torch.zeros(K * K, dtype=torch.float64, device=dev)
    d_res = torch.zeros(K, dtype=torch.float64, device=dev)
    rb, re = equal_row_split(n, world)[dist.get_rank(group) if world > 1 else 0]
    jb = max(1, -(-(re - rb) // jacobi_rows))
    opt = N.GbemPcgOptions(1e-10, 2000, jb)
    cfg = ctx.quad()
    pst, ast = N.GbemPcgStats(), N.GbemAssemblyStats()

    def step():
        ctx.check(ctx.lib.gbem_pcg_extract_cmatrix_dev(ctx.h, C.byref(panels), n, C.c_void_p(d_net.data_ptr()), K,
                                                       eps, C.byref(cfg), C.byref(opt), C.c_void_p(d_C.data_ptr()),
                                                       C.c_void_p(d_res.data_ptr()), None, None, C.byref(pst)))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group)
    torch.cuda.synchronize()
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters = []
    for _ in range(steps):
        step()
        iters.append(pst.iterations)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launches = ctx.launches - l0
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
        ms = float(tt.item())
    # e2e through the public host-buffer API
    Pa = N.PanelArrays.from_matrix(P)
    if world > 1:
        dist.barrier(group)
    t0 = time.perf_counter()
    for _ in range(max(1, steps // 2)):
        Cm, res, _, st2, _ = sharded_cmatrix(ctx, Pa, net, K, eps, tol=1e-10, max_iter=2000, jacobi_blocks=jb,
                                             attach_ranks=False)
    e2e_s = (time.perf_counter() - t0) / max(1, steps // 2)
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
        e2e_s = float(tt.item())
    entries = n * (n + 1) // 2
    peaks = _peaks()
    mv_tf = pst.matvec_flops / (pst.ms_matvec * 1e-3) / 1e12 if pst.ms_matvec > 0 else None
    return {"ms_per_step": ms, "entries_per_s": entries / (ms * 1e-3), "steps": steps, "warmup": warmup,
            "iterations": iters, "jacobi_blocks_per_rank": jb, "rows_local": pst.rows_local,
            "max_rel_resid": float(res.max()), "tol": 1e-10, "gpu_launches": launches,
            "phases_ms": {"assembly": pst.ms_assembly, "precond_setup": pst.ms_precond,
                          "iterations": pst.ms_iterations, "total": pst.ms_total},
            "matvec": {"ms": pst.ms_matvec, "tflops": mv_tf,
                       "frac_dmma": mv_tf / peaks.get("fp64_dmma_tflops", 37.09) if mv_tf else None,
                       "flops": pst.matvec_flops, "shape": f"({pst.rows_local} x {n}) x ({n} x {K})"},
            "e2e": {"value": entries / e2e_s, "unit": UNIT, "seconds": e2e_s,
                    "h2d_bytes_per_step": n * (1 + 5 * 8) + n * 4, "d2h_bytes_per_step": K * K * 8 + K * 8},
            "c_matrix_diag_F_first": float(Cm[0, 0])}


def config5_assembly_steps(ctx, warmup, steps, world, rank, group=None, chunk_gb=40.0):
    """Config-5 assembly-only stress test: this rank's work-balanced upper-
    triangle rows (paper_2203_11733_b200.shard.balanced_row_split), streamed
    through a row buffer of at most chunk_gb; returns device-timed entries/s
    (max over ranks)."""
    import torch
    import torch.distributed as dist
    import paper_2203_11733_b200 as g
    from paper_2203_11733_b200 import _native as N
    from paper_2203_11733_b200.shard import balanced_row_split, row_work
    dev = torch.device("cuda", torch.cuda.current_device())
    ps = g.config_model(5, seed=1).partition(1)
    n = len(ps)
    a, b = balanced_row_split(n, world)[rank]
    ld = (n + 7) // 8 * 8
    rows_chunk = max(1, int(chunk_gb * 1e9 / (8 * ld)))
    nch = max(1, -(-(b - a) // rows_chunk))
    cuts = [a + (b - a) * k // nch for k in range(nch + 1)]
    buf = torch.empty((max(1, cuts[1] - cuts[0] + 1), ld), dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    t = _to_dev(ps.matrix(), dev)
    panels = _panels_struct(N, t)
    cfg = ctx.quad()

    def step(stats=None):
        for c0, c1 in zip(cuts[:-1], cuts[1:]):
            if c1 > c0:
                ctx.check(ctx.lib.gbem_assemble_rows_dev(ctx.h, C.byref(panels), n, c0, c1, C.byref(cfg),
                                                         C.c_void_p(buf.data_ptr()), ld,
                                                         C.byref(stats) if stats is not None else None))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
        ms = float(tt.item())
    entries = n * (n + 1) // 2
    del buf, t
    return {"ms_per_step": ms, "entries_per_s": entries / (ms * 1e-3), "rank_entries": row_work(n, a, b),
            "row_chunks": nch, "steps": steps, "warmup": warmup}


def run_sharded(args):
    """N > 1 (or --workload sharded): config-4 sharded C-matrix + config-5 assembly."""
    import torch
    import torch.distributed as dist
    from paper_2203_11733_b200 import _native as N
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    P4, net4, K4, eps4, _ = serialized_workload(4)
    n4 = len(P4)
    clk = ClockSampler(local).start()
    ctx = N.Context(local)
    clk.mark_start()
    r4 = sharded_extract_steps(ctx, P4, net4, K4, eps4, args.warmup, args.steps, world, args.jacobi_rows)
    clk.mark_end()
    ctx.close()
    torch.cuda.empty_cache()
    ctx = N.Context(local)
    r5 = config5_assembly_steps(ctx, min(args.warmup, 1), max(1, args.steps // 4), world, rank)
    ctx.close()
    clk.stop()
    n5 = 200000
    line = {"metric": METRIC, "value": r4["entries_per_s"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r4["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE config geometry)",
            "config": sharded_config(world, n4, K4, n5),
            "e2e": r4["e2e"], "gpu_launches": r4["gpu_launches"], "clocks": clk.summary(),
            "config4_pcg": r4, "config5_assembly": r5,
            "roofline": {"bound": "tensor", "kernel": "k_gemm_nt_sk_bulk (row-block product A_r P, split-K DMMA, bulk-copy staged)",
                         "achieved": r4["matvec"]["tflops"], "peak": _peaks().get("fp64_dmma_tflops", 37.09),
                         "unit": "TFLOP/s", "frac": r4["matvec"]["frac_dmma"], "traffic": None,
                         "algorithmic": "2 rows n K flop per product / device time of one product"}}
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def _ncu_traffic_file() -> dict:
    """profiles/ncu_traffic.json (committed ncu evidence: per-launch DRAM bytes, pipe utilisation)."""
    try:
        return json.load(open(ROOT / "profiles" / "ncu_traffic.json"))
    except (OSError, ValueError):
        return {}


def _ncu_traffic() -> dict:
    """Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
    dominant kernels from the committed ncu --set full captures (profiles/)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return {k: v for k, v in json.load(open(p)).get("bytes_per_launch", {}).items()}
    except (OSError, ValueError):
        return {}


# ----------------------------------------------------------------------------- CPU reference arm

def _ref_libs():
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O  # test-side loader of oracle/ (CPU checker), used here only for the CPU arm
    if O.ref_available():
        return O, "ref", "reference"
    return O, "orc", "port"


_CHOL_CACHE: dict = {}


def cpu_cholesky_rate(budget_s: float = 8.0):
    """The reference's Cholesky loop (solver.hpp:28-37) in its own storage order
    (Eigen column-major L: the row dot products walk with stride n), one
    thread, timed at the largest n whose factorisation fits ~budget_s
    (calibrated at n = 400, cubic, capped at 3000).  Returns (flop/s, n)."""
    if "rate" in _CHOL_CACHE:
        return _CHOL_CACHE["rate"], _CHOL_CACHE["n"]
    O, _, _ = _ref_libs()
    lib = O.orc()
    f = lib.orc_cholesky_factor_colmajor
    f.restype = C.c_int
    f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    rng = np.random.default_rng(0)

    def run(m):
        A = rng.normal(size=(m, m)) / np.sqrt(m)
        A = np.asfortranarray(A @ A.T + np.eye(m))
        L = np.empty((m, m))
        piv = C.c_int64(-1)
        t0 = time.perf_counter()
        assert f(m, A.ctypes.data, L.ctypes.data, C.byref(piv)) == 0
        return time.perf_counter() - t0

    t = run(400)
    m = int(min(3000, max(400, 400 * (budget_s / max(t, 1e-6)) ** (1 / 3))))
    t = run(m)
    _CHOL_CACHE.update(rate=(m ** 3 / 3) / t, n=m)
    return _CHOL_CACHE["rate"], m


def cpu_sample_rate(P: np.ndarray, n: int, seconds: float, seed: int = 0, chol_budget: float = 8.0):
    """Reference u_pair_integral on all host threads over a seeded uniform
    sample of the n(n+1)/2 unique pairs, plus the reference Cholesky loop
    extrapolated as n^3/3.  Returns (entries/s of the full step, details)."""
    O, which, kind = _ref_libs()
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)

    def timed(k):
        i = rng.integers(0, n, size=k)
        j = rng.integers(0, n, size=k)
        lo, hi = np.minimum(i, j), np.maximum(i, j)
        t0 = time.perf_counter()
        O.u_pairs(which, P[lo], P[hi], nthreads=threads)
        return time.perf_counter() - t0

    t = timed(2000)
    k = int(min(5e6, max(2000, 2000 * 0.9 * seconds / max(t, 1e-6))))
    t = timed(k)
    pair_rate = k / t
    chol_rate, mch = cpu_cholesky_rate(chol_budget)
    entries = n * (n + 1) / 2
    step_s = entries / pair_rate + (n ** 3 / 3) / chol_rate
    return entries / step_s, {"kind": kind, "cores": threads, "pairs_sampled": k, "pair_rate_per_s": pair_rate,
                              "cholesky_gflops_1thread": chol_rate / 1e9, "cholesky_n": mch,
                              "extrapolated_step_s": step_s}


def cpu_baseline(P, n, K, budget_s=20.0):
    v, d = cpu_sample_rate(P, n, budget_s)
    return {"value": v, "unit": UNIT, "cores": d["cores"], "kind": d["kind"],
            "sample": (f"{d['pairs_sampled']} seeded uniform unique pairs of the same panel list through the "
                       f"reference u_pair_integral on {d['cores']} threads ({d['pair_rate_per_s']:.3g} pairs/s) + "
                       f"the reference Cholesky loop (column-major, as Eigen stores L) timed at "
                       f"n={d['cholesky_n']} ({d['cholesky_gflops_1thread']:.3g} GFLOP/s, 1 thread) "
                       f"extrapolated to n^3/3 for n={n}; full CPU step = {d['extrapolated_step_s']:.1f} s "
                       f"(one assembly + one factorisation: the reference's capacitance_matrix repeats both "
                       f"for each of the {K} nets, so this understates its time)"),
            "extrapolated_step_s": d["extrapolated_step_s"]}


def run_reference_full(args, P, n, K, cfgd):
    """A config small enough for the CPU (config 1, the reference's own runnable case): every step is
    the COMPLETE reference step, nothing sampled or extrapolated -- all n(n+1)/2 entries through the
    reference u_pair_integral on all host threads (assemble_single, assembly.hpp:82-104), then the
    reference Cholesky loop (solver.hpp:28-37, column-major) on that matrix, one thread as in the
    reference.  The step count is capped so the run stays within a few minutes."""
    O, which, kind = _ref_libs()
    threads = os.cpu_count() or 1
    lib = O.orc()
    f = lib.orc_cholesky_factor_colmajor
    f.restype = C.c_int
    f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
    times = []
    steps = max(1, min(args.steps, 12))
    warm = min(args.warmup, 1)
    for s in range(warm + steps):
        t0 = time.perf_counter()
        A, _, st = O.assemble(which, P, nthreads=threads)
        t1 = time.perf_counter()
        Af = np.asfortranarray(A)
        L = np.empty((n, n))
        piv = C.c_int64(-1)
        t2 = time.perf_counter()
        rc = f(n, Af.ctypes.data, L.ctypes.data, C.byref(piv))
        t3 = time.perf_counter()
        assert st == 0 and rc == 0, (st, rc, piv.value)
        if s >= warm:
            times.append(((t1 - t0) + (t3 - t2), t1 - t0, t3 - t2))
    step_s = float(np.mean([t[0] for t in times]))
    value = n * (n + 1) / 2 / step_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
            "steps": steps, "warmup": warm, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config geometry)", "config": cfgd,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"the complete step, measured: all {n * (n + 1) // 2} entries through the "
                                       f"reference u_pair_integral on {threads} threads "
                                       f"({np.mean([t[1] for t in times]):.2f} s) + the reference Cholesky loop at "
                                       f"n={n} on one thread ({np.mean([t[2] for t in times]):.2f} s); nothing "
                                       "sampled or extrapolated"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    if world > 1 or args.workload == "sharded":
        P, net, K, eps, seed = serialized_workload(4)
        n = len(P)
        cfgd = sharded_config(world, n, K, 200000)
    else:
        P, net, K, eps, seed = serialized_workload(args.config)
        n = len(P)
        cfgd = extract_config(args.config, n, K, eps, seed)
    if world == 1 and args.workload != "sharded" and n <= 2000:
        return run_reference_full(args, P, n, K, cfgd)
    per = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    for s in range(args.warmup + args.steps):
        v, d = cpu_sample_rate(P, n, per, seed=s)
        if s >= args.warmup:
            vals.append((v, d))
    value = float(np.mean([v for v, _ in vals]))
    d = vals[-1][1]
    step_s = n * (n + 1) / 2 / value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config geometry)", "config": cfgd,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": d["cores"], "kind": d["kind"],
                             "sample": f"per step {d['pairs_sampled']} sampled unique pairs through the reference "
                                       f"u_pair_integral on {d['cores']} threads + the reference Cholesky loop "
                                       f"(column-major) timed at n={d['cholesky_n']}, extrapolated to the full step "
                                       f"({step_s:.0f} s)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["extract", "sharded"],
                    help="default: extract at N = 1, sharded at N > 1")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--jacobi-rows", type=int, default=12032, help="rows per block-Jacobi block")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded", action="store_true", help="N = 1: skip the sharded_n1 measurements")
    args = ap.parse_args()
    world, _, _ = dist_env()
    if args.workload is None:
        args.workload = "sharded" if world > 1 else "extract"
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "sharded":
        run_sharded(args)
    else:
        run_extract(args)


if __name__ == "__main__":
    main()
