#!/usr/bin/env python
"""Throughput of the FP64 matrix-free elasticity apply y = A x on B200 (GDoF/s per apply).

Default workload: BASELINE.json config 5 (64x64x256 Q6, q=8, perturbed trilinear geometry,
per-element LogNormal(0,0.5) material, 683,465,475 DoF) -- the largest configuration that
fits one GPU and the one the multi-GPU (z-slab) runs use.  With N=1 the line also carries
the config-4 p-sweep (p = 1..8 at ~50M DoF, the metric's "vs p=1..8").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

A step = one elas_apply over the whole (rank-local) mesh: init kernel + fused apply kernel
(+ interface exchange for N > 1).  Timing: CUDA events on the op's stream over exactly K
steps, bracketed by barrier + synchronize, max over ranks.  Inputs (49.6 GB at config 5)
are far larger than L2 (126 MB), so no L2 flush is needed between steps.
"""

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FP64_DERIVED = 148 * 64 * 2 * 1.965e9      # DFMA/clk/SM x 2 flop x SMs x max clock


def alg_flops(p, q, ne):
    """plain 3-stage sum factorisation fwd+transpose, 3 comps, + 120 flop/qp."""
    n = p + 1
    return ne * (12 * (2 * q * n ** 3 + 3 * q * q * n * n + 3 * q ** 3 * n) + 120 * q ** 3)


def alg_bytes(ndof, ne, q, per_elem):
    """x read + y write + 9 qdata doubles per point (+ r_e per element)."""
    return 16 * ndof + 72 * q ** 3 * ne + (8 * ne if per_elem else 0)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------------------ clocks

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device_index, period=0.05):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self._stop = period, threading.Event()
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _reasons(self):
        nv = self.nv
        for fn in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            if hasattr(nv, fn):
                return getattr(nv, fn)(self.h)
        return 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self._reasons()
                for bit, name in REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.h is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.h is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------ CPU oracle

def oracle_sample_problem(P, bx, by, bz):
    """A bx x by x bz brick of elements (corner at the origin) carved out of workload P."""
    import synth
    p = P.p
    V = P.vertex_array()[:bz + 1, :by + 1, :bx + 1]
    lam, mu = P.material_arrays()
    lam, mu = lam[:bz, :by, :bx], mu[:bz, :by, :bx]
    Nx, Ny, Nz = P.node_dims
    x = P.x_slab(0, bz * p) if P.x is None else P.x
    x = x.reshape(3, -1, Ny, Nx)[:, :bz * p + 1, :by * p + 1, :bx * p + 1]
    Q = synth.Problem(P.name + "_brick", bx, by, bz, p, P.q, 1.0, 1.0, 1.0, V, lam, mu,
                      np.ascontiguousarray(x).reshape(-1), 0, P.seed)
    return Q


def oracle_time(P, nelem):
    """Run the oracle (as it stands) on a brick of ~nelem elements; return (seconds, elements)."""
    import oracle
    bx = min(P.nx, max(1, int(round(nelem ** (1 / 3)))))
    by = min(P.ny, max(1, int(round((nelem / bx) ** 0.5))))
    bz = min(P.nz, max(1, nelem // (bx * by)))
    Q = oracle_sample_problem(P, bx, by, bz)
    lam, mu = Q.material_arrays()
    m = oracle.Mesh(Q.vertices, Q.p, Q.q, lam, mu, 0)
    elems = [(ex, ey, ez) for ez in range(bz) for ey in range(by) for ex in range(bx)]
    t = time.perf_counter()
    oracle.apply_elements(m, Q.x, elems)
    return time.perf_counter() - t, len(elems), f"{bx}x{by}x{bz} element brick of {P.name}"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count()


def cpu_info():
    """CPU model, physical cores and logical CPUs of this host (lscpu; /proc/cpuinfo fallback)."""
    info = {"cpu_model": None, "physical_cores": None, "logical_cpus": os.cpu_count()}
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for ln in out.splitlines():
            if ":" in ln:
                k, v = ln.split(":", 1)
                kv[k.strip()] = v.strip()
        info["cpu_model"] = kv.get("Model name")
        if kv.get("Core(s) per socket") and kv.get("Socket(s)"):
            info["physical_cores"] = int(kv["Core(s) per socket"]) * int(kv["Socket(s)"])
    except Exception:
        pass
    if info["cpu_model"] is None:
        try:
            with open("/proc/cpuinfo") as f:
                for ln in f:
                    if ln.startswith("model name"):
                        info["cpu_model"] = ln.split(":", 1)[1].strip()
                        break
        except Exception:
            pass
    return info


def cpu_baseline(P, budget_s=12.0):
    nel = 4
    t, ne, desc = oracle_time(P, nel)
    while t < budget_s / 4 and ne < P.num_elements:
        nel = int(ne * max(2.0, min(8.0, budget_s / max(t, 1e-3) / 2)))
        t, ne, desc = oracle_time(P, nel)
    value = P.num_dofs * (ne / P.num_elements) / t / 1e9
    return {"value": value, "unit": "GDoF/s", "cores": blas_threads(), "kind": "oracle", **cpu_info(),
            "sample": f"{desc} ({ne} elements, {t:.1f} s; extrapolated to {P.num_elements} elements)"}


# ------------------------------------------------------------------------------ helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def make_workload(cfg, p):
    import synth
    return synth.make_config(cfg, p, draw_x=False)


def workload_desc(P):
    geo = "perturbed" if P.vertices is not None else "affine"
    mat = "LogNormal(0,0.5) per element" if P.per_element_material else f"lam={float(P.lam)}, mu={float(P.mu)}"
    return (f"{P.name}: {P.nx}x{P.ny}x{P.nz} hexes, Q{P.p} q={P.q}, {geo} trilinear, {mat}, "
            f"faces={P.dirichlet_faces}, {P.num_dofs} DoF")


def reduce_max(val, ws):
    if ws == 1:
        return val
    import torch
    import torch.distributed as dist
    t = torch.tensor([val], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------------ sweep

PEAK_FP32_DERIVED = 148 * 128 * 2 * 1.965e9    # FFMA/clk/SM x 2 flop x SMs x max clock


def sweep_config4(reps=10, warmup=3, variant=0, ps=range(1, 9)):
    """variant 0: AUTO (FP64).  variant 5: the mixed-precision folded kernel (FP32 qdata and
    arithmetic, FP64 vectors): roofline against the FP32 pipe and 36 B of qdata per point."""
    import torch
    import synth
    from paper_2601_08374_b200.elas import Operator, elas_profile, elas_profile_read
    f32 = variant == 5
    peak = PEAK_FP32_DERIVED if f32 else PEAK_FP64_DERIVED
    out = {}
    for p in ps:
        P = synth.make_config(4, p)
        op = Operator.from_problem(P, variant=variant)
        x = torch.from_numpy(P.x).cuda()
        y = torch.empty_like(x)
        for _ in range(warmup):
            op.apply(x, y)
        torch.cuda.synchronize()
        elas_profile(op.h, True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            op.apply(x, y)
        b.record()
        torch.cuda.synchronize()
        kms, nl = elas_profile_read(op.h)
        elas_profile(op.h, False)
        t = a.elapsed_time(b) / reps / 1e3
        tk = kms / nl / 1e3
        F = alg_flops(p, P.q, P.num_elements)
        B = alg_bytes(P.num_dofs, P.num_elements, P.q, False)
        if f32:
            B = 16 * P.num_dofs + 36 * P.q ** 3 * P.num_elements
        roof_t = max(F / peak, B / 8e12)
        out[str(p)] = {"q": P.q, "dofs": P.num_dofs, "elements": P.num_elements,
                       "gdofs": round(P.num_dofs / t / 1e9, 3), "ms_per_apply": round(t * 1e3, 4),
                       "kernel_ms": round(tk * 1e3, 4),
                       ("fp32" if f32 else "fp64") + "_tflops_alg": round(F / tk / 1e12, 2),
                       "roofline_frac": round(roof_t / t, 4),
                       "bound": ("fp32" if f32 else "fp64") if F / peak > B / 8e12 else "hbm"}
        op.close()
        del x, y
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------ ablation (Table 4)

def ablation_bench(p=8, reps=3, warmup=2):
    """The paper's ablation (Table 4: p = 8, 51.17M DoF) on B200 at config 4,
    p = 8 (50.9M DoF): per-apply time of each optimization stage and the marginal speedups.
    Stages 0-2 are the unfused pipelines (ELAS_VARIANT_ABL_*), 3 the fused SIMT kernel, 4 the
    folded kernel (AUTO)."""
    import torch
    import synth
    from paper_2601_08374_b200.elas import (Operator, VARIANT_ABL_PA, VARIANT_ABL_SF, VARIANT_ABL_VOIGT,
                                            VARIANT_SIMT, VARIANT_FOLDED)
    P = synth.make_config(4, p)
    x = torch.from_numpy(P.x).cuda()
    y = torch.empty_like(x)
    stages = [("PA (baseline, Alg. 1: unfused, dense O(p^6) contractions)", VARIANT_ABL_PA),
              ("+ Sum Factorization (C1)", VARIANT_ABL_SF), ("+ Voigt Notation (C2)", VARIANT_ABL_VOIGT),
              ("+ Kernel Fusion (C3)", VARIANT_SIMT), ("+ Loop Structure (B200: folded kernel)", VARIANT_FOLDED)]
    paper = [None, 12.74, 1.01, 2.15, 1.96]
    rows, prev = [], None
    for (name, v), pm in zip(stages, paper):
        op = Operator.from_problem(P, variant=v)
        for _ in range(warmup):
            op.apply(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            op.apply(x, y)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        rows.append({"stage": name, "variant": v, "ms_per_apply": round(ms, 4),
                     "gdofs": round(P.num_dofs / (ms / 1e3) / 1e9, 3),
                     "marginal_speedup": None if prev is None else round(prev / ms, 2),
                     "paper_kernel_marginal_speedup": pm})
        prev = ms
        op.close()
        torch.cuda.empty_cache()
    del x, y
    torch.cuda.empty_cache()
    return {"workload": f"config 4, p = {p} (q = {P.q}, {P.num_dofs} DoF); paper: Kunpeng 920, p = 8, 51.17M DoF "
                        "(kernel column of Table 4, context only)",
            "stages": rows, "overall_speedup": round(rows[0]["ms_per_apply"] / rows[-1]["ms_per_apply"], 2),
            "paper_overall_kernel_speedup": 54.19}


# ------------------------------------------------------------------------------ config 2 hot / cold

def small_configs(reps=20):
    """Config 1 (375 DoF: launch/latency-bound, time only) and config 3 (9.1M DoF,
    Dirichlet face) per-apply numbers on the AUTO kernel."""
    import torch
    import synth
    from paper_2601_08374_b200.elas import Operator
    out = {}
    for cfg in (1, 3):
        P = synth.make_config(cfg)
        op = Operator.from_problem(P)
        x = torch.from_numpy(P.x).cuda()
        y = torch.empty_like(x)
        for _ in range(5):
            op.apply(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            op.apply(x, y)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        out[f"cfg{cfg}"] = {"dofs": P.num_dofs, "ms_per_apply": round(ms, 5),
                            "gdofs": round(P.num_dofs / ms / 1e6, 3) if cfg != 1 else None}
        op.close()
        del x, y
        torch.cuda.empty_cache()
    return out


def anisotropic_sweep(ps=(2, 4, 6, 8), reps=10):
    """General anisotropic material (Eq. 2): config 4 with a seeded SPD Voigt matrix per element."""
    import numpy as np
    import torch
    import synth
    from paper_2601_08374_b200.elas import Operator
    out = {}
    for p in ps:
        P = synth.make_config(4, p)
        x = torch.from_numpy(P.x).cuda()
        y = torch.empty_like(x)
        op = Operator.anisotropic(P, synth.random_C6(np.random.default_rng(p), (P.nz, P.ny, P.nx)))
        for _ in range(3):
            op.apply(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            op.apply(x, y)
        b.record()
        torch.cuda.synchronize()
        out[str(p)] = round(P.num_dofs / (a.elapsed_time(b) / reps / 1e3) / 1e9, 3)
        op.close()
        del x, y
        torch.cuda.empty_cache()
    return {"workload": "config 4, C_e = L L^T + 0.5 I per element (seeded), folded FP64 kernel", "gdofs": out}


def config2_hot_cold(reps=20):
    """Config 2 (823,875 DoF; 77 MB working set < 126 MB L2): back-to-back applies (hot) and
    applies each preceded by a 2 x L2 memset (cold), per SURVEY 8(d)."""
    import torch
    import synth
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_config(2)
    op = Operator.from_problem(P)
    x = torch.from_numpy(P.x).cuda()
    y = torch.empty_like(x)
    flush = torch.empty(2 * 126 * 2 ** 20 // 4, dtype=torch.int32, device="cuda")
    for _ in range(5):
        op.apply(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        op.apply(x, y)
    b.record()
    torch.cuda.synchronize()
    hot = a.elapsed_time(b) / reps
    cold = []
    for _ in range(reps):
        flush.zero_()
        a.record()
        op.apply(x, y)
        b.record()
        torch.cuda.synchronize()
        cold.append(a.elapsed_time(b))
    cold.sort()
    op.close()
    return {"workload": "cfg2: 16^3 hexes, Q4 q=6, perturbed, 823875 DoF", "hot_ms": round(hot, 4),
            "hot_gdofs": round(P.num_dofs / hot / 1e6, 3), "cold_median_ms": round(cold[len(cold) // 2], 4),
            "cold_gdofs": round(P.num_dofs / cold[len(cold) // 2] / 1e6, 3),
            "note": "cold = 2 x L2 memset before each individually timed apply"}


# ------------------------------------------------------------------------------ solver row

def solver_bench(cfg=3, passes=10, rtol=1e-8, maxit=4000):
    """SURVEY 8(f) NEXT rank 1-2 on the GPU: diagonal + power-iteration setup, Chebyshev
    smoothing passes (order 3: 3 applies + 3 fused vector kernels each) and PCG to rtol with
    Chebyshev and Jacobi preconditioning.  Solver throughput as PAPER.md:386 defines it:
    "total degrees of freedom processed per second" = N_dof x iterations / solve time."""
    import torch
    import synth
    from paper_2601_08374_b200.elas import Operator, PC_JACOBI, PC_CHEBYSHEV
    P = synth.make_config(cfg, draw_x=False)
    op = Operator.from_problem(P)
    n = P.num_dofs
    b = torch.from_numpy(synth.splitmix_uniform(n, 11)).cuda()
    x = torch.zeros_like(b)
    torch.cuda.synchronize()
    t = time.perf_counter()
    ch = op.chebyshev(order=3, alpha=0.1, beta=1.1, power_iters=10, seed=1)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t
    ch.apply(b, x)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(passes):
        ch.apply(b, x)
    e.record()
    torch.cuda.synchronize()
    pass_ms = a.elapsed_time(e) / passes
    out = {"workload": workload_desc(P), "chebyshev": {"order": 3, "interval": "[0.1, 1.1] x lambda_max",
           "lambda_max": round(ch.lambda_max, 6), "setup_s_diag_plus_10_power_its": round(setup, 4),
           "ms_per_pass": round(pass_ms, 4), "applies_per_pass": 3,
           "gdofs_per_apply_equiv": round(3 * n / (pass_ms / 1e3) / 1e9, 3)}}
    from paper_2601_08374_b200.elas import VARIANT_FOLDED_F32
    op32 = Operator.from_problem(P, variant=VARIANT_FOLDED_F32)
    ch32 = op32.chebyshev(order=3, alpha=0.1, beta=1.1, power_iters=10, seed=1)
    for name, pc, c in (("pcg_chebyshev", PC_CHEBYSHEV, ch), ("pcg_chebyshev_fp32_smoother", PC_CHEBYSHEV, ch32),
                        ("pcg_jacobi", PC_JACOBI, None)):
        op.pcg(b, x, precond=pc, cheb=c, rtol=rtol, maxit=3)   # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        it, conv, rel, _ = op.pcg(b, x, precond=pc, cheb=c, rtol=rtol, maxit=maxit)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        out[name] = {"rtol": rtol, "iterations": it, "converged": conv, "rel_residual": rel,
                     "solve_s": round(dt, 4), "ms_per_iteration": round(dt / max(it, 1) * 1e3, 4),
                     "solver_mdofs": round(n * it / dt / 1e6, 1)}
    # GMG-preconditioned CG (the paper's solver): 24^3 -> 12^3 -> 6^3 -> 3^3
    from paper_2601_08374_b200.elas import GMG
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = GMG.from_problem(P, levels=4, coarse_maxit=20)
    torch.cuda.synchronize()
    g_setup = time.perf_counter() - t
    g.pcg(b, x, rtol=rtol, maxit=2)   # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    it, conv, rel, _ = g.pcg(b, x, rtol=rtol, maxit=500)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    out["pcg_gmg"] = {"levels": 4, "hierarchy": "24^3 -> 12^3 -> 6^3 -> 3^3 hexes, Q6 on every level; Chebyshev(3) "
                      "pre/post smoothing; coarse: 20 Chebyshev-PCG iterations (no host sync; 10/20/30 measured: 20 best)",
                      "setup_s": round(g_setup, 4), "rtol": rtol, "iterations": it, "converged": conv,
                      "rel_residual": rel, "solve_s": round(dt, 4), "ms_per_iteration": round(dt / max(it, 1) * 1e3, 4),
                      "solver_mdofs": round(n * it / dt / 1e6, 1)}
    g.close()
    # mixed precision: the whole V-cycle on FP32 operators, FP64 CG on the FP64 operator
    from paper_2601_08374_b200.elas import VARIANT_FOLDED_F32, elas_pcg_gmg
    g32 = GMG.from_problem(P, levels=4, coarse_maxit=20, variant=VARIANT_FOLDED_F32)
    elas_pcg_gmg(op.h, g32.h, b, x, rtol, 2)   # warm (captures the graph)
    torch.cuda.synchronize()
    t = time.perf_counter()
    it, conv, rel, _ = elas_pcg_gmg(op.h, g32.h, b, x, rtol, 500)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    out["pcg_gmg_fp32_vcycle"] = {"levels": 4, "rtol": rtol, "iterations": it, "converged": conv,
                                  "rel_residual": rel, "solve_s": round(dt, 4),
                                  "ms_per_iteration": round(dt / max(it, 1) * 1e3, 4),
                                  "solver_mdofs": round(n * it / dt / 1e6, 1),
                                  "note": "FP64 CG and operator; V-cycle (smoothers, transfers, coarse solve) on the "
                                          "mixed-precision operators"}
    g32.close()
    out["pcg_chebyshev_fp32_smoother"]["note"] = ("FP64 CG and operator; the Chebyshev preconditioner runs the "
                                                  "mixed-precision (FP32) operator of the same mesh")
    ch32.close()
    op32.close()
    ch.close()
    op.close()
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------ arms

def run_ours(args):
    import torch
    ws, rank, lrank = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(lrank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    else:
        torch.cuda.set_device(0)
    from paper_2601_08374_b200 import elas
    from paper_2601_08374_b200.elas import Operator

    P = make_workload(args.config, args.p)
    b, e = elas.elas_slab_range(P.nz, rank, ws)
    K0, K1 = b * P.p, e * P.p
    t_gen = time.perf_counter()
    x_np = P.x_slab(K0, K1)
    t_gen = time.perf_counter() - t_gen
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist
        obj = [elas.elas_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream()
    t0 = time.perf_counter()
    op = Operator.from_problem(P, rank=rank, nranks=ws, nccl_id=nccl_id, stream=stream)
    setup_s = time.perf_counter() - t0
    assert op.local_dofs == x_np.size
    x_pin = torch.from_numpy(x_np).pin_memory()
    del x_np
    x = x_pin.cuda()
    y = torch.empty_like(x)

    for _ in range(args.warmup):
        op.apply(x, y)
    torch.cuda.synchronize()
    barrier(ws)
    elas.elas_profile(op.h, True)
    elas.elas_profile_read(op.h)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            op.apply(x, y)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
    elas.elas_profile(op.h, False)
    kern_ms, nlaunch = elas.elas_profile_read(op.h)
    t_ms = reduce_max(ev0.elapsed_time(ev1), ws)
    kern_ms_per_apply = reduce_max(kern_ms / args.steps, ws)
    ms_per_step = t_ms / args.steps
    value = P.num_dofs / (ms_per_step / 1e3) / 1e9

    # per-apply distribution (SURVEY 8(d) timing protocol): one event pair per apply, separate
    # from the timed region above
    per = []
    pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(min(args.steps, 10))]
    for a_, b_ in pe:
        a_.record(stream)
        op.apply(x, y)
        b_.record(stream)
    torch.cuda.synchronize()
    per = sorted(a_.elapsed_time(b_) for a_, b_ in pe)
    per_apply = {"median_ms": round(per[len(per) // 2], 4), "min_ms": round(per[0], 4), "max_ms": round(per[-1], 4),
                 "n": len(per)}

    # the bitwise-reproducible colored scatter (elas_set_deterministic): same op, same inputs
    det = None
    if op.variant in (4, 5):
        op.set_deterministic(True)
        for _ in range(2):
            op.apply(x, y)
        barrier(ws)
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        nd = max(3, args.steps // 2)
        for _ in range(nd):
            op.apply(x, y)
        d1.record(stream)
        torch.cuda.synchronize()
        det_ms = reduce_max(d0.elapsed_time(d1), ws) / nd
        det = {"value": round(P.num_dofs / (det_ms / 1e3) / 1e9, 4), "unit": "GDoF/s", "ms_per_step": round(det_ms, 4),
               "steps": nd, "note": "8 color launches (one contribution per node per launch), y bitwise reproducible"}
        op.set_deterministic(False)

    # geometry on the fly (no stored quadrature data): same workload, separate op
    otf = None
    if ws == 1 and args.config in (3, 5):
        from paper_2601_08374_b200.elas import VARIANT_FOLDED_OTF
        free0 = torch.cuda.mem_get_info()[0]
        op6 = Operator.from_problem(P, variant=VARIANT_FOLDED_OTF, stream=stream)
        used = free0 - torch.cuda.mem_get_info()[0]
        for _ in range(2):
            op6.apply(x, y)
        torch.cuda.synchronize()
        o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        no = max(3, args.steps // 2)
        o0.record(stream)
        for _ in range(no):
            op6.apply(x, y)
        o1.record(stream)
        torch.cuda.synchronize()
        otf_ms = o0.elapsed_time(o1) / no
        otf = {"value": round(P.num_dofs / (otf_ms / 1e3) / 1e9, 4), "unit": "GDoF/s", "ms_per_step": round(otf_ms, 4),
               "steps": no, "operator_bytes": int(used),
               "stored_qdata_bytes": int(72 * P.q ** 3 * P.num_elements),
               "note": "ELAS_VARIANT_FOLDED_OTF: A~ rebuilt per point from the trilinear map (40 doubles per element)"}
        op6.close()
        torch.cuda.empty_cache()

    # end to end through the C ABI with pinned HOST buffers (H2D + apply + D2H each step)
    y_pin = torch.empty_like(x_pin).pin_memory()
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    op.apply_host(x_pin, y_pin)
    barrier(ws)
    t = time.perf_counter()
    for _ in range(e2e_steps):
        op.apply_host(x_pin, y_pin)
    t_e2e = reduce_max(time.perf_counter() - t, ws)
    e2e_value = P.num_dofs / (t_e2e / e2e_steps) / 1e9
    launches = op.launches_per_apply * args.steps

    # roofline of the dominant kernel (the fused apply): algorithmic flops of this rank per apply
    ne_local = P.nx * P.ny * (e - b)
    F = alg_flops(P.p, P.q, ne_local)
    B = alg_bytes(op.local_dofs, ne_local, P.q, P.per_element_material)
    tk = kern_ms_per_apply / 1e3
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    roof = {"bound": "alu", "achieved": round(F / tk / 1e12, 3), "peak": round(PEAK_FP64_DERIVED / 1e12, 2),
            "unit": "TFLOP/s", "frac": round(F / tk / PEAK_FP64_DERIVED, 4), "traffic": None,
            "peak_kind": ("derived FP64 pipe: 148 SM x 64 FMA/clk x 2 flop x 1.965 GHz = 37.2 TF/s (MEASURED_PEAKS.json "
                          "has no FP64 entry); measured on this pool's B200: DMMA 37.1 TF/s, all-register DFMA "
                          "34.1 TF/s (tools/microbench/dmma_rates.cu, fp64_probe.cu; DESIGN.md 6)"),
            "alg_flops_per_apply": F, "alg_bytes_per_apply": B,
            "hbm_achieved_gbs": round(B / tk / 1e9, 1),
            "hbm_frac_of_measured": round(B / tk / 1e9 / hbm_peak, 4) if hbm_peak else None,
            "kernel_share_of_step": round(kern_ms_per_apply / ms_per_step, 4),
            "roofline_frac_step_8tbs": round(max(F / PEAK_FP64_DERIVED, B / 8e12) * ws / (ms_per_step / 1e3), 4)}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(f"cfg{args.config}" + (f"_p{args.p}" if args.config == 4 else ""))
            if tr and ws == 1:
                roof["traffic"] = tr.get("dram_bytes_per_launch")
    except Exception:
        pass

    line = {"metric": "elasticity operator apply GDoF/s (FP64); % of FP64/HBM roofline",
            "value": round(value, 4), "unit": "GDoF/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(P), "dofs": P.num_dofs, "elements": P.num_elements,
                       "p": P.p, "q": P.q, "parallelism": f"z-slabs x{ws}" + (" (NCCL interface sum)" if ws > 1 else ""),
                       "l2": "inputs larger than L2 (no flush needed)"},
            "clocks": clk.summary(),
            "e2e": {"value": round(e2e_value, 4), "unit": "GDoF/s", "steps": e2e_steps,
                    "h2d_bytes_per_step": 8 * op.local_dofs * ws, "d2h_bytes_per_step": 8 * op.local_dofs * ws,
                    "note": "elas_apply_host: pinned host x -> device, apply, device -> pinned host y"},
            "gpu_launches": launches,
            "roofline": roof,
            "per_apply": per_apply,
            "deterministic": det,
            "geometry_on_the_fly": otf,
            "setup_s": round(setup_s, 3), "x_generation_s": round(t_gen, 2)}
    op.close()
    del x, y
    torch.cuda.empty_cache()
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(P)
    if ws == 1 and not args.no_sweep:
        line["config2_hot_cold"] = config2_hot_cold()
        line["configs_1_3"] = small_configs()
        line["anisotropic"] = anisotropic_sweep()
    if ws == 1 and not args.no_sweep:
        line["ablation"] = ablation_bench()
    if ws == 1 and not args.no_solver:
        line["solver"] = solver_bench()
    if ws == 1 and not args.no_sweep:
        line["sweep"] = {"workload": "config 4: m^3 unit cube, m = round(255.44/p), q=p+2, affine, lam=1, mu=0.5, seed 3",
                         "per_p": sweep_config4()}
        line["sweep_mixed_precision"] = {
            "workload": "config 4 as above, ELAS_VARIANT_FOLDED_F32 (FP32 qdata/tables/arithmetic, FP64 x, y, scatter; "
                        "rel. L2 vs oracle <= 1e-5, not the FP64 contract); roofline: FP32 pipe 74.4 TF derived, "
                        "16 B/DoF + 36 B/point",
            "per_p": sweep_config4(variant=5, ps=range(2, 9))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    """The CPU oracle as it stands, on bounded samples of the same workload (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    P = make_workload(args.config, args.p)
    per_step = max(1, args.ref_elems if args.ref_elems else (16 if P.p >= 6 else 64))
    for _ in range(args.warmup):
        oracle_time(P, per_step)
    ts, ne, desc = 0.0, 0, ""
    for _ in range(args.steps):
        t, n, desc = oracle_time(P, per_step)
        ts += t
        ne += n
    sec_per_step = ts / args.steps
    value = P.num_dofs * (ne / args.steps / P.num_elements) / sec_per_step / 1e9
    line = {"metric": "elasticity operator apply GDoF/s (FP64); % of FP64/HBM roofline",
            "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec_per_step * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_desc(P), "dofs": P.num_dofs, "elements": P.num_elements,
                       "p": P.p, "q": P.q},
            "cpu_baseline": {"value": value, "unit": "GDoF/s", "cores": blas_threads(), "kind": "oracle",
                             **cpu_info(),
                             "sample": f"each step: {desc}, extrapolated to {P.num_elements} elements"},
            "e2e": {"value": value, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, choices=[2, 3, 4, 5])
    ap.add_argument("--p", type=int, default=6, help="degree for --config 4")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solver", action="store_true")
    ap.add_argument("--ref-elems", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    ws, _, _ = dist_env()
    if ws != args.gpus:
        if not (ws == 1 and args.gpus == 1):
            print(f"warning: --gpus {args.gpus} but WORLD_SIZE={ws}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
