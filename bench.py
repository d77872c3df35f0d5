#!/usr/bin/env python
"""Benchmark of the S-fraction ROM hot path on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Workload (BASELINE.json configs[1]): config 2 = 8 x 8 x 8 subdomains
of 17^3 nodes, seeded 5-layer medium + 24^3 inclusion, m=4, k=6 (K = 168 ROM
DOF per subdomain), 15 Hz Ricker source, fp64.  A bench "step" is one coupled
leapfrog step of every subdomain; the K timed steps run as ONE persistent
kernel launch.  Models are built on the GPU first (reported as ``rom_build``).

``--impl reference`` times the reference algorithm on the host cores instead:
the CPU oracle port (oracle/sfw_oracle.py, restating reference rom.py and
stepper.py; pinned bitwise to reference golden vectors), which is the
reference's own CPU implementation of the path.  Under torchrun only rank 0
runs it.

Multi-GPU: the north star scopes the path to one GPU, so --gpus N
runs N independent replicas (weak scaling), timed on the device, max over ranks.
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

METRIC = "ROM subdomain-steps/s (fp64 coupled S-fraction leapfrog)"
UNIT = "subdomain-steps/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic(key, steps):
    """ncu DRAM bytes per step of the stepping launch (profiles/traffic.json) x the launch's steps."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            ent = json.load(fh).get(key)
        return ent["dram_bytes_per_step"] * steps if ent else None
    except Exception:
        return None


def _fp64_peak():
    """Measured FP64 DMMA peak (TFLOP/s) of this pool's B200 (profiles/r01_fp64_peak.json, tools/fp64_peak.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as fh:
            return float(json.load(fh)["dmma_f64_tflops"]), "measured (tools/fp64_peak.cu)"
    except Exception:
        return 37.0, "fallback"


def _workload(cfg):
    from paper_1406_6923_b200 import grid as pg
    from paper_1406_6923_b200.configs import locate, make_workload
    wl = make_workload(cfg)
    ext = tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing))
    part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
    alphas = sorted(s.alpha for s in part.subdomains)
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in alphas]
    src_alpha, src_row = locate(wl.sources[0], wl.counts, wl.p)
    node_rx = [locate(ijk, wl.counts, wl.p) for ijk in wl.node_receivers]
    return wl, ops, alphas, (src_alpha, src_row), node_rx


def _describe(wl):
    return (f"{wl.name}: "
            f"{'x'.join(map(str, wl.counts))} subdomains of 17^3 nodes (h=10 m), m={wl.modes_per_face}, "
            f"k={wl.n}, K={wl.layers * wl.width} ROM DOF/subdomain, f0={wl.f0:g} Hz Ricker")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def reduce_max(x: float, device="cuda") -> float:
    """Max over ranks (device-timed seconds); identity on one process."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(n_sub: int, steps: int, world: int, t_max: float) -> float:
    """Whole-job subdomain-steps/s of ``world`` independent replicas."""
    return world * n_sub * steps / t_max


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def cpu_oracle_models(ops, cfg, workers):
    """Models built by the CPU oracle (reference algorithm) with a process pool."""
    from concurrent.futures import ProcessPoolExecutor
    with ProcessPoolExecutor(max_workers=workers) as ex:
        res = list(ex.map(_oracle_build_one, [(cfg, op.alpha) for op in ops], chunksize=4))
    return dict(res)


def _oracle_build_one(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import sfw_oracle as so
    from paper_1406_6923_b200.configs import make_workload
    cfg, alpha = args
    wl = _WL_CACHE.get(cfg)
    if wl is None:
        wl = _WL_CACHE[cfg] = make_workload(int(cfg))
    op = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field, alphas=[alpha])[alpha]
    md = so.build_model(op, wl.modes_per_face, wl.n, wl.shift)
    md.basis = None
    return alpha, md


_WL_CACHE: dict = {}


def oracle_step_rate(models, dt, src, budget_s=15.0, max_steps=400, warmup=1):
    """Time the oracle's coupled leapfrog (reference stepper.py:362-389 loop shape)."""
    from oracle import sfw_oracle as so
    st = so.Coupled(models, dt, sources=[src])
    st.initialize()
    for _ in range(warmup):
        st.advance()
    t0 = time.perf_counter()
    n = 0
    while n < max_steps and (time.perf_counter() - t0) < budget_s:
        st.advance()
        n += 1
    el = time.perf_counter() - t0
    return len(models) * n / el, n, el


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import sfw_oracle as so
    wl, ops, alphas, (src_alpha, src_row), _ = _workload(args.config)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    models = cpu_oracle_models(ops, args.config, cores)
    build_s = time.perf_counter() - t0
    # dt: short power iteration (timing does not depend on dt; 0.5 x the estimate keeps the sample stable)
    lam, _ = so.cfl_power(models, max_iter=40)
    dt = 0.5 * 2.0 / math.sqrt(lam)
    # source needs the basis row: rebuild the source subdomain with its basis
    sop = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field, alphas=[src_alpha])[src_alpha]
    smd = so.build_model(sop, wl.modes_per_face, wl.n, wl.shift)
    vec = so.source_vector(smd, src_row)
    steps = max(1, min(args.steps, 60))
    rate, n, el = oracle_step_rate(models, dt, (src_alpha, vec, so.ricker(wl.f0, wl.delay)),
                                   budget_s=60.0, max_steps=steps, warmup=max(1, min(args.warmup, 3)))
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws, "steps": n,
        "warmup": max(1, min(args.warmup, 3)), "ms_per_step": 1e3 * el / n, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8d)",
        "config": {"workload": _describe(wl), "subdomains": len(models)},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{n} coupled leapfrog steps of all {len(models)} subdomains "
                                   f"(oracle restatement of reference stepper.py, single thread)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "rom_build": {"subdomains_per_s": len(models) / build_s, "seconds": build_s, "cores": cores,
                      "kind": "port (scipy SuperLU + LAPACK, one process per core)"},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import ctypes as C

    import torch

    ws, rank, lrank = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(lrank)
    from paper_1406_6923_b200 import (CoupledStepper, Probe, SourceTerm, _lib, build_models,
                                      cfl_estimate_coupled, make_probe, project_source)
    from paper_1406_6923_b200.rom import LAST_BUILD_STATS
    from paper_1406_6923_b200.pulses import ricker

    wl, ops, alphas, (src_alpha, src_row), node_rx = _workload(args.config)
    n_sub = len(ops)
    w, L = wl.width, wl.layers
    rows = {src_alpha: [src_row]}
    for a, r in node_rx:
        rows.setdefault(a, []).append(r)
    from paper_1406_6923_b200.configs import locate
    for ijk in wl.sources[1:]:
        a, r = locate(ijk, wl.counts, wl.p)
        rows.setdefault(a, []).append(r)
    dev = [torch.empty(n_sub * L * w * w, dtype=torch.float64, device="cuda") for _ in range(3)]
    ptrs = tuple(t.data_ptr() for t in dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows, device_out=ptrs)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    build_stats = dict(LAST_BUILD_STATS)
    scl = dev[2].view(n_sub, L, w, w)
    idx = {a: i for i, a in enumerate(alphas)}
    for a in rows:
        models[a].scales = scl[idx[a]].cpu().numpy()
    t0 = time.perf_counter()
    lam, conv = cfl_estimate_coupled(models, device_coefficients=ptrs)
    cfl_s = time.perf_counter() - t0
    from paper_1406_6923_b200.stepper import LAST_CFL
    cfl_iters = LAST_CFL.get("iterations")
    dt = 0.9 * 2.0 / math.sqrt(lam)
    vec = project_source(models[src_alpha], src_row)
    probes = []
    for alpha, face in wl.face_receivers:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[alpha].state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append(Probe(alpha, wts))
    for a, r in node_rx:
        probes.append(make_probe(models[a], r))
    src = SourceTerm(src_alpha, vec, ricker(wl.f0, wl.delay))
    if len(wl.sources) > 1:
        return _run_shots(args, wl, models, ptrs, dt, lam, conv, probes, ws, rank, build_s, build_stats, cfl_s,
                          cfl_iters)
    if args.precision == "fp32":
        return _run_fp32(args, wl, models, ptrs, dt, lam, conv, src, probes, ws, rank, build_s, build_stats, cfl_s,
                         cfl_iters)
    st = CoupledStepper(models, dt, sources=(src,), device_coefficients=ptrs)
    st.initialize(_probes=probes)
    lib = st._lib
    K = args.steps
    prof_w = np.ascontiguousarray(np.array([[src.profile(k * dt) for k in range(max(args.warmup, 1))]]))
    prof_k = np.ascontiguousarray(np.array([[src.profile(k * dt) for k in range(K)]]))
    ms = C.c_float(0.0)
    eb = _lib.errbuf()
    _lib.check(lib.sfw_step_run_resident(st._h, max(args.warmup, 1), 1, _lib.dptr(prof_w), C.byref(ms), eb, 1024), eb)
    # flush L2 (126 MB) before the timed launch
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    flush.fill_(1.0)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(lrank) as clk:
        t0 = time.perf_counter()
        _lib.check(lib.sfw_step_run_resident(st._h, K, 1, _lib.dptr(prof_k), C.byref(ms), eb, 1024), eb)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if ws > 1:
        dist.barrier()
    kernel_s = ms.value * 1e-3
    t_max = reduce_max(kernel_s)
    value = replica_value(n_sub, K, ws, t_max)
    alg_bytes, alg_flops, streamed = st.traffic()
    # e2e through the public API: host profile/limit tables in, probe rows + norms out, every step
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    times, trace = st.run(K, probes=probes)
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - t0
    e2e_t = reduce_max(e2e_wall)
    e2e_value = replica_value(n_sub, K, ws, e2e_t)
    h2d = 8 * (1 + len(st.sources))  # growth limit + profile value per source
    d2h = 8 * (len(probes) + 1)      # probe row + |U|
    if rank != 0:
        st.close()
        if ws > 1:
            dist.destroy_process_group()
        return
    peak, peak_kind = _peaks()
    achieved = alg_bytes * K / kernel_s / 1e9
    traffic = _traffic(f"config{args.config}", K)  # per launch, like achieved
    # CPU baseline: the oracle (reference algorithm) stepping the same models, bounded sample
    cpu = None
    if not args.no_cpu:
        from oracle import sfw_oracle as so
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        G = dev[0].view(n_sub, L, w, w).cpu().numpy()
        H = dev[1].view(n_sub, L, w, w).cpu().numpy()
        S = scl.cpu().numpy()
        omodels = {a: so.Model(alpha=a, lo=None, shape=None, spacing=None, modes_per_face=wl.modes_per_face,
                               layers=L, shift=wl.shift, neighbors=dict(ops[i].neighbors), face_indices=(),
                               gammas=G[i], gamma_hats=H[i], scales=S[i], basis=None, c=None, mu=None)
                   for i, a in enumerate(alphas)}
        rate, n, el = oracle_step_rate(omodels, dt, (src_alpha, vec, so.ricker(wl.f0, wl.delay)),
                                       budget_s=args.cpu_seconds, max_steps=2000)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{n} coupled leapfrog steps of all {n_sub} subdomains on GPU-built models, "
                         f"{el:.1f} s (oracle restatement of reference stepper.py, single thread)"}
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded medium, SURVEY 8d); models built on the GPU from it",
        "config": {"workload": _describe(wl), "subdomains": n_sub, "rom_dof_per_subdomain": L * w,
                   "sources": 1, "probes": len(probes), "dt": dt, "lambda_hat": lam, "cfl_converged": conv,
                   "l2": ("flushed (512 MB write) before the timed launch; the K steps run in one persistent "
                          "launch that loads the 16 MB of chain coefficients into SMEM once and keeps them there "
                          "(ncu DRAM traffic ~9.5 KB/step)") if args.config == 2 else
                         ("flushed (512 MB write) before the timed launch; the K steps run in one persistent "
                          "launch, so chain coefficients stream HBM->SMEM per step (L2-resident when they fit)"),
                   "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
        "dof_updates_per_s": value * L * w,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "CoupledStepper.run(K, probes) incl. init, profile/limit upload, trace/norm download"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes * K,
                     "alg_bytes_per_step": alg_bytes, "streamed_bytes_per_step": streamed,
                     "alg_flops_per_step": alg_flops,
                     "formula": "8[(2L-1)w(w+1)/2 + 3Lw] bytes per subdomain-step (SURVEY 8d)"},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": 1,
        "kernel_ms": ms.value, "wall_ms": wall * 1e3,
        "rom_build": {"seconds": build_s, "subdomains_per_s": n_sub / build_s, "stages_s": build_stats,
                      "cfl_seconds": cfl_s, "cfl_iterations": cfl_iters,
                      "k_step2_launches_before_timed": (cfl_iters or 0) + 2},
    }
    st.close()
    if args.extra and args.config == 2:
        try:
            line["extra"] = _extra_configs(args)
        except Exception as exc:  # the headline line must still print
            line["extra"] = {"error": str(exc)[:300]}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _extra_configs(args):
    """Kernel-only stepping of the other BASELINE configs (device-timed, L2 flushed), so the default
    bench line carries every config: 3 (fp64 U-form and fp32 W-form), 4 (32 shots, DMMA) and 5
    (fp64 and fp32).  Each entry: ms/step, subdomain-steps/s, roofline fraction, ROM build time."""
    import ctypes as C

    import torch
    from paper_1406_6923_b200 import CoupledStepper, SourceTerm, _lib, build_models, cfl_estimate_coupled
    from paper_1406_6923_b200 import project_source
    from paper_1406_6923_b200.configs import locate, make_workload
    from paper_1406_6923_b200.pulses import ricker
    peak, _ = _peaks()
    fpk, _ = _fp64_peak()
    out = {}

    def flush():
        buf = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
        buf.fill_(1.0)
        torch.cuda.synchronize()

    for cfg in (3, 5):
        wl, ops, alphas, (sa, sr), _ = _workload(cfg)
        n_sub, w, L = len(ops), wl.width, wl.layers
        rows = {sa: [sr]}
        if cfg == 3:  # config 4 = config 3 models + 32 shot sources
            for ijk in make_workload(4).sources:
                a, r = locate(ijk, wl.counts, wl.p)
                rows.setdefault(a, []).append(r)
        dev = [torch.empty(n_sub * L * w * w, dtype=torch.float64, device="cuda") for _ in range(3)]
        ptrs = tuple(t.data_ptr() for t in dev)
        t0 = time.perf_counter()
        models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows, device_out=ptrs)
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
        scl = dev[2].view(n_sub, L, w, w)
        idx = {a: i for i, a in enumerate(alphas)}
        for a in rows:
            models[a].scales = scl[idx[a]].cpu().numpy()
        lam, conv = cfl_estimate_coupled(models, device_coefficients=ptrs)
        dt = 0.9 * 2.0 / math.sqrt(lam)
        src = SourceTerm(sa, project_source(models[sa], sr), ricker(wl.f0, wl.delay))
        K = 300 if cfg == 3 else 150
        # fp64 U-form, one persistent launch
        st = CoupledStepper(models, dt, sources=(src,), device_coefficients=ptrs)
        st.initialize()
        ms = C.c_float(0.0)
        eb = _lib.errbuf()
        _lib.check(st._lib.sfw_step_run_resident(st._h, 5, 1, None, C.byref(ms), eb, 1024), eb)
        flush()
        _lib.check(st._lib.sfw_step_run_resident(st._h, K, 1, None, C.byref(ms), eb, 1024), eb)
        b, _f, _s = st.traffic()
        st.close()
        sec = ms.value * 1e-3
        out[f"config{cfg}"] = {"workload": _describe(wl), "subdomains": n_sub, "steps": K, "ms_per_step": ms.value / K,
                               "value": n_sub * K / sec, "unit": UNIT, "dtype": "f64",
                               "roofline": {"bound": "hbm", "frac": b * K / sec / 1e9 / peak,
                                            "achieved": b * K / sec / 1e9, "peak": peak, "unit": "GB/s"},
                               "rom_build_seconds": build_s, "cfl_converged": conv}
        # fp32 W-form
        st = CoupledStepper(models, dt, sources=(src,), device_coefficients=ptrs, precision="fp32")
        st.run(5)
        flush()
        st.run(K)
        bb, sb = C.c_double(), C.c_double()
        st._lib.sfw_wform_traffic(st._h, C.byref(bb), C.byref(sb))
        sec = st.last_kernel_ms * 1e-3
        st.close()
        out[f"config{cfg}_fp32"] = {"workload": _describe(wl) + ", fp32 W-form", "steps": K,
                                    "ms_per_step": 1e3 * sec / K, "value": n_sub * K / sec, "unit": UNIT,
                                    "dtype": "f32", "roofline": {"bound": "hbm", "frac": bb.value * K / sec / 1e9 / peak,
                                                                 "achieved": bb.value * K / sec / 1e9, "peak": peak,
                                                                 "unit": "GB/s"}}
        if cfg == 3:  # config 4: 32 independent shots on the DMMA path
            wl4 = make_workload(4)
            shots = []
            for ijk in wl4.sources:
                a, r = locate(ijk, wl4.counts, wl4.p)
                shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl4.f0, wl4.delay)))
            K4 = 20
            st = CoupledStepper(models, dt, device_coefficients=ptrs)
            st.run_shots(3, shots)
            flush()
            st.run_shots(K4, shots)
            ab, af, _ = st.shots_traffic()
            sec = st.last_kernel_ms * 1e-3
            st.close()
            t_hbm, t_fp = ab / (peak * 1e9), af / (fpk * 1e12)
            out["config4"] = {"workload": _describe(wl4) + ", S=32 shots", "steps": K4, "ms_per_step": 1e3 * sec / K4,
                              "value": n_sub * K4 / sec, "unit": UNIT, "shot_steps_per_s": 32 * n_sub * K4 / sec,
                              "dtype": "f64", "achieved_tflops": af * K4 / sec / 1e12,
                              "roofline": {"bound": "hbm" if t_hbm >= t_fp else "fp64",
                                           "frac": max(t_hbm, t_fp) * K4 / sec,
                                           "roofline_us_per_step": {"hbm": 1e6 * t_hbm, "fp64": 1e6 * t_fp}}}
        del models, dev
        torch.cuda.empty_cache()
    return out


def _run_fp32(args, wl, models, ptrs, dt, lam, conv, src, probes, ws, rank, build_s, build_stats, cfl_s, cfl_iters):
    """Config 5 fp32 variant: W-form stepping (U_j = G_j W_j), fp32 blocks."""
    import ctypes as C

    import torch
    from paper_1406_6923_b200 import CoupledStepper, _lib
    n_sub = len(models)
    w, L = wl.width, wl.layers
    st = CoupledStepper(models, dt, sources=(src,), device_coefficients=ptrs, precision="fp32")
    st.run(max(args.warmup, 1), probes=probes)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    flush.fill_(1.0)
    torch.cuda.synchronize()
    K = args.steps
    # kernel-only: one launch (rows downloaded after it), CUDA-event time of the launch
    os.environ["SFW_NO_CHUNK"] = "1"
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        st.run(K, probes=probes)
        torch.cuda.synchronize()
    del os.environ["SFW_NO_CHUNK"]
    kernel_s = st.last_kernel_ms * 1e-3
    # e2e: the public call as a user makes it (row downloads overlap later chunks)
    flush.fill_(2.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    times, rows = st.run(K, probes=probes)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    t_max = reduce_max(kernel_s)
    value = replica_value(n_sub, K, ws, t_max)
    e2e_value = replica_value(n_sub, K, ws, reduce_max(wall))
    b, st_b = C.c_double(), C.c_double()
    st._lib.sfw_wform_traffic(st._h, C.byref(b), C.byref(st_b))
    st.close()
    if rank != 0:
        return
    peak, peak_kind = _peaks()
    achieved = b.value * K / kernel_s / 1e9
    line = {
        "metric": METRIC.replace("fp64", "fp32 W-form"), "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded medium, SURVEY 8d); models built on the GPU",
        "config": {"workload": _describe(wl) + ", fp32 W-form variant", "subdomains": n_sub,
                   "rom_dof_per_subdomain": L * w, "dt": dt, "lambda_hat": lam, "cfl_converged": conv,
                   "probes": len(probes), "l2": "flushed before the timed launch", "parallelism": "1 GPU"},
        "dof_updates_per_s": value * L * w,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16, "d2h_bytes_per_step": 8 * (len(probes) + 1),
                "api": "CoupledStepper(precision='fp32').run(K, probes)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _traffic(f"config{args.config}_fp32", K), "peak_kind": peak_kind,
                     "alg_bytes_per_step": b.value,
                     "streamed_bytes_per_step": st_b.value,
                     "formula": "4[(2L-1)w(w+1)/2 + 3Lw] bytes per subdomain-step (SURVEY 8d fp32)"},
        "cpu_baseline": None, "clocks": clk.summary(), "gpu_launches": 2, "kernel_ms": kernel_s * 1e3,
        "rom_build": {"seconds": build_s, "subdomains_per_s": n_sub / build_s, "stages_s": build_stats,
                      "cfl_seconds": cfl_s, "cfl_iterations": cfl_iters},
    }
    print(json.dumps(line), flush=True)


def _run_shots(args, wl, models, ptrs, dt, lam, conv, probes, ws, rank, build_s, build_stats, cfl_s, cfl_iters):
    """Config 4: 32 independent sources stepped together (DMMA path)."""
    import torch
    from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source
    from paper_1406_6923_b200.configs import locate
    from paper_1406_6923_b200.pulses import ricker
    shots = []
    for ijk in wl.sources:
        a, r = locate(ijk, wl.counts, wl.p)
        shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay)))
    n_sub = len(models)
    w, L = wl.width, wl.layers
    st = CoupledStepper(models, dt, device_coefficients=ptrs)
    st.run_shots(max(args.warmup, 1), shots, probes=probes)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    flush.fill_(1.0)
    torch.cuda.synchronize()
    K = args.steps
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        t0 = time.perf_counter()
        times, rows = st.run_shots(K, shots, probes=probes)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    kernel_s = st.last_kernel_ms * 1e-3
    t_max = reduce_max(kernel_s)
    value = replica_value(n_sub, K, ws, t_max)
    e2e_t = reduce_max(wall)
    e2e_value = replica_value(n_sub, K, ws, e2e_t)
    alg_bytes, alg_flops, streamed = st.shots_traffic()
    st.close()
    if rank != 0:
        return
    peak, peak_kind = _peaks()
    achieved = alg_bytes * K / kernel_s / 1e9
    fpk, fpk_kind = _fp64_peak()
    t_hbm = alg_bytes / (peak * 1e9)
    t_fp = alg_flops / (fpk * 1e12)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded medium, SURVEY 8d); models built on the GPU from it",
        "config": {"workload": _describe(wl) + ", S=32 independent shots (one SourceTerm each)",
                   "subdomains": n_sub, "shots": len(shots), "rom_dof_per_subdomain": L * w, "dt": dt,
                   "lambda_hat": lam, "cfl_converged": conv, "probes": len(probes),
                   "l2": "flushed before the timed launch", "parallelism": "1 GPU"},
        "shot_steps_per_s": value * len(shots),
        "dof_updates_per_s": value * L * w * len(shots),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * len(shots),
                "d2h_bytes_per_step": 8 * len(shots) * (len(probes) + 1),
                "api": "CoupledStepper.run_shots(K, 32 shots, probes): profile upload, init, kernel, "
                       "per-shot traces + norms download"},
        "roofline": {"bound": "hbm" if t_hbm >= t_fp else "fp64", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": max(t_hbm, t_fp) * K / kernel_s,
                     "traffic": _traffic("config4", K), "peak_kind": peak_kind, "alg_bytes_per_step": alg_bytes,
                     "streamed_bytes_per_step": streamed, "alg_flops_per_step": alg_flops,
                     "achieved_tflops": alg_flops * K / kernel_s / 1e12, "fp64_peak_tflops": fpk,
                     "fp64_peak_kind": fpk_kind, "roofline_us_per_step": {"hbm": 1e6 * t_hbm, "fp64": 1e6 * t_fp},
                     "frac_note": "slower of HBM bytes and FP64 flops at their measured peaks (north_star)",
                     "formula": "8[(2L-1)w(w+1)/2 + 3LwS] bytes, S(2(2L-1)w^2+5Lw) flops per subdomain-step"},
        "cpu_baseline": None,
        "clocks": clk.summary(),
        "gpu_launches": 2,
        "kernel_ms": st.last_kernel_ms,
        "rom_build": {"seconds": build_s, "subdomains_per_s": n_sub / build_s, "stages_s": build_stats,
                      "cfl_seconds": cfl_s, "cfl_iterations": cfl_iters},
    }
    print(json.dumps(line), flush=True)


def _run_fdtd(args):
    """Fine-grid leapfrog reference solver on the config's full grid: node-steps/s."""
    import torch
    from paper_1406_6923_b200 import assemble_global_operator, run_leapfrog, stability_limit
    from paper_1406_6923_b200 import grid as pg
    from paper_1406_6923_b200.configs import make_workload
    from paper_1406_6923_b200.pulses import ricker
    wl = make_workload(args.config)
    ext = tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing))
    part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
    a = assemble_global_operator(part, wl.c_field)
    t0 = time.perf_counter()
    dt = 0.9 * stability_limit(a)
    cfl_s = time.perf_counter() - t0
    src = int(np.ravel_multi_index(tuple(wl.sources[0]), part.global_shape))
    vec = np.zeros(a.n)
    vec[src] = 1.0 / wl.c_field.ravel()[src]
    kw = dict(source_vec=vec, source_fn=ricker(wl.f0, wl.delay), record_idx=[src], chunk=max(args.steps, 1))
    run_leapfrog(a, dt, max(args.warmup, 1), **kw)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    flush.fill_(1.0)
    torch.cuda.synchronize()
    K = args.steps
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        t0 = time.perf_counter()
        run = run_leapfrog(a, dt, K, **kw)
        wall = time.perf_counter() - t0
    sec = run.kernel_ms * 1e-3
    peak, peak_kind = _peaks()
    alg = 32.0 * a.n  # u, c, u_prev read + u_next written once per node-step (fp64)
    cpu = None
    if not args.no_cpu:  # the reference algorithm (scipy CSR product + numpy leapfrog), bounded sample
        from oracle import sfw_oracle as so
        am = so.global_matrix(part.global_shape, part.spacing, wl.c_field)
        n_cpu = 3
        t0 = time.perf_counter()
        so.leapfrog(am, dt, n_cpu, source_vec=vec, source_fn=so.ricker(wl.f0, wl.delay))
        el = time.perf_counter() - t0
        cpu = {"value": a.n * n_cpu / el, "unit": "node-steps/s", "cores": 1, "kind": "port",
               "sample": f"{n_cpu} fine-grid leapfrog steps of {a.n} nodes incl. the start, {el:.1f} s "
                         "(oracle restatement of reference.py run_leapfrog, scipy CSR)"}
    line = {"metric": "fine-grid leapfrog node-steps/s (reference solver, fp64)", "value": a.n * K / sec,
            "unit": "node-steps/s", "n_gpus": 1, "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * sec / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded medium, SURVEY 8d)",
            "config": {"workload": f"fine grid of {_describe(wl)}", "nodes": a.n, "grid": list(part.global_shape),
                       "dt": dt, "cfl_seconds": cfl_s, "l2": "flushed before the timed run; 2 x 136 MB state > L2"},
            "e2e": {"value": a.n * K / wall, "unit": "node-steps/s", "h2d_bytes_per_step": 8,
                    "d2h_bytes_per_step": 16, "api": "run_leapfrog(a, dt, K, source, receiver)"},
            "roofline": {"bound": "hbm", "achieved": alg * K / sec / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg * K / sec / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                         "formula": "32 B per node-step (u, c, u_prev read once, u_next written once)"},
            "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": 2 * K}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extra", type=int, default=1,
                    help="also measure configs 3, 4, 5 (fp64 and fp32) kernel-only stepping (default on)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--fdtd", action="store_true", help="fine-grid reference solver on the config's full grid")
    args = ap.parse_args()
    if args.fdtd:
        return _run_fdtd(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
