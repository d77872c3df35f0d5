#!/usr/bin/env python
"""Benchmark of the S-fraction ROM hot path on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
                    [--precision fp64|fp32] [--no-cpu] [--extra 0|1] [--fdtd]

Headline workload (BASELINE.json metric, quoted on the largest config): config 5 =
32 x 32 x 16 = 16384 subdomains of 17^3 nodes, seeded 4^3-cell blocky medium + 10
inclusions of 5500 m/s, m=9, k=8 (K = 486 ROM DOF per subdomain), 10 Hz Ricker
source, fp64 U-form, 9224 receivers (z-midplane face coefficients + 8 node
receivers) recorded every step.  A bench "step" is one coupled leapfrog step of
every subdomain; the K timed steps run as ONE persistent kernel launch.  Models
are built on the GPU first (``rom_build``), dt = 0.9 * 2 / sqrt(lambda) from the GPU
CFL power iteration.  ``e2e`` is the same K steps through ``CoupledStepper.run``.
``extra`` carries configs 5 fp32, 3 (fp64/fp32), 4 (32 shots, DMMA) and 2 with the
same work (source, receivers, host profile table).

``--impl reference`` times the reference algorithm on the host cores instead: the
CPU oracle port (oracle/sfw_oracle.py, restating reference rom.py and stepper.py;
pinned bitwise to reference golden vectors) on a stated 4x4x4-subdomain window of
the same medium (a full config-5 CPU build takes about an hour): oracle build,
oracle CFL, then W + K coupled steps with the window's receivers.  Under torchrun
only rank 0 runs it.  ``cpu_baseline`` in the GPU arm's line is the same sample.

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


# ---------------------------------------------------------------------------
# CPU leg: the reference algorithm (oracle port) on a stated subset of the workload

SUBSET = 4  # subdomains per axis of the CPU sample window


def subset_window(wl, n=SUBSET):
    """Low corner (subdomain index) of the n^3-subdomain window centred on the source subdomain."""
    from paper_1406_6923_b200.configs import locate
    sa, _ = locate(wl.sources[0], wl.counts, wl.p)
    return tuple(max(0, min(a - n // 2 + 1, c - n)) for a, c in zip(sa, wl.counts))


_SUB_CTX: dict = {}


def _subset_build_one(alpha):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import sfw_oracle as so
    ctx = _SUB_CTX
    op = so.make_subops(ctx["counts"], ctx["p"], ctx["spacing"], ctx["c"], alphas=[alpha])[alpha]
    md = so.build_model(op, ctx["m"], ctx["n"], ctx["shift"])
    if alpha not in ctx["need_basis"]:
        md.basis = None
    return alpha, md


def cpu_subset_run(cfg, steps, warmup, cores=None, n=SUBSET):
    """The reference's CPU path on an n^3-subdomain window of config ``cfg``'s medium.

    The window (centred on the source subdomain) is a domain of its own: the oracle port of
    reference rom.py builds its n^3 models (one process per core, one BLAS thread each), the
    oracle port of cfl_estimate_coupled (stepper.py:452-487, tol 1e-8) gives dt = 0.9 * 2 / sqrt(lam)
    as for the GPU arm, and the oracle port of CoupledStepper (stepper.py:325-415, one thread:
    the reference's workers > 1 is slower) steps it from rest with the 15/10 Hz
    Ricker source and the configuration's receivers that fall inside the window (z-midplane
    face coefficients + node receivers), recording every step.  ``warmup`` untimed steps, then
    ``steps`` timed ones.  Returns a dict (rate in subdomain-steps/s of the window)."""
    import multiprocessing as mp

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import sfw_oracle as so
    from paper_1406_6923_b200.configs import locate, make_workload
    wl = make_workload(3 if cfg == 4 else cfg)
    lo = subset_window(wl, n)
    counts = (n, n, n)
    sl = tuple(slice(16 * a, 16 * (a + n) + 1) for a in lo)
    c_sub = np.ascontiguousarray(wl.c_field[sl])
    inside = lambda ijk: all(16 * a < x < 16 * (a + n) for x, a in zip(ijk, lo))  # noqa: E731
    local = lambda ijk: tuple(x - 16 * a for x, a in zip(ijk, lo))  # noqa: E731
    src_alpha, src_row = locate(local(wl.sources[0]), counts, wl.p)
    node_rx = [locate(local(ijk), counts, wl.p) for ijk in wl.node_receivers if inside(ijk)]
    kz = wl.counts[2] // 2 - 1 - lo[2]
    face_rx = [((i, j, kz), 5) for i in range(n) for j in range(n)] if 0 <= kz < n else []
    need = {src_alpha} | {a for a, _ in node_rx}
    alphas = [(i, j, k) for i in range(n) for j in range(n) for k in range(n)]
    cores = cores or os.cpu_count() or 1
    _SUB_CTX.update(counts=counts, p=wl.p, spacing=wl.spacing, c=c_sub, m=wl.modes_per_face, n=wl.n,
                    shift=wl.shift, need_basis=need)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(cores, len(alphas))) as pool:
        models = dict(pool.map(_subset_build_one, alphas, chunksize=1))
    build_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    lam, conv = so.cfl_power(models)
    cfl_s = time.perf_counter() - t0
    dt = 0.9 * 2.0 / math.sqrt(lam)
    vec = so.source_vector(models[src_alpha], src_row)
    probes = []
    for a, f in face_rx:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[a].state_size)
            wts[f * wl.modes_per_face + q] = 1.0
            probes.append((a, wts))
    probes += [(a, so.probe_weights(models[a], r)) for a, r in node_rx]
    st = so.Coupled(models, dt, sources=[(src_alpha, vec, so.ricker(wl.f0, wl.delay))])
    st.initialize()
    rows = [st._row(probes)]
    for _ in range(warmup):
        st.advance()
        rows.append(st._row(probes))
    t0 = time.perf_counter()
    for _ in range(steps):
        st.advance()
        rows.append(st._row(probes))
    el = time.perf_counter() - t0
    nsub = len(models)
    return {"rate": nsub * steps / el, "seconds": el, "steps": steps, "warmup": warmup, "subdomains": nsub,
            "window": {"counts": list(counts), "low_subdomain": list(lo)}, "probes": len(probes),
            "dt": dt, "lambda_hat": lam, "cfl_converged": bool(conv), "cfl_seconds": cfl_s,
            "build_seconds": build_s, "build_cores": min(cores, len(alphas)),
            "build_subdomains_per_s": nsub / build_s,
            "sample": (f"{n}x{n}x{n}-subdomain window (low corner {lo}) of the {wl.name} medium, m={wl.modes_per_face} "
                       f"k={wl.n}: oracle-port build ({min(cores, len(alphas))} processes, {build_s:.1f} s) + "
                       f"CPU CFL ({cfl_s:.1f} s) + {steps} timed coupled leapfrog steps ({warmup} warm-up) with the "
                       f"Ricker source and {len(probes)} receivers in the window recorded every step, "
                       f"{el:.2f} s on 1 thread (oracle restatement of reference stepper.py)")}


# ---------------------------------------------------------------------------
# GPU arm

def config_key(wl, n_probes, shots=1):
    """The ``config`` object of both arms (identical for the same workload)."""
    return {"workload": _describe(wl) + (f", S={shots} independent shots" if shots > 1 else ""),
            "subdomains": wl.n_sub, "rom_dof_per_subdomain": wl.layers * wl.width, "sources": shots,
            "probes": n_probes, "record_every": 1,
            "l2": "flushed before the timed launch (512 MB write, then a 256 MB read of another buffer: our "
                  "data evicted, L2 left clean); the K steps run in one persistent launch"}


_CLEAN = []


def flush_l2():
    """Evict the workload from L2 (126 MB): write 512 MB, then read 256 MB of another buffer, so L2
    ends full of clean foreign lines and the write-back of the flush's own dirty lines is not paid
    inside the next timed launch."""
    import torch
    buf = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    buf.fill_(1.0)
    if not _CLEAN:
        _CLEAN.append(torch.ones(32 * 1024 * 1024, dtype=torch.float64, device="cuda"))
    float(_CLEAN[0].sum())
    torch.cuda.synchronize()
    del buf


def prepare(cfg, extra_rows=()):
    """GPU ROM build of a config's workload (chain stacks left in HBM), GPU CFL, source and probes."""
    import torch
    from paper_1406_6923_b200 import Probe, SourceTerm, build_models, cfl_estimate_coupled, make_probe
    from paper_1406_6923_b200 import project_source
    from paper_1406_6923_b200.configs import locate
    from paper_1406_6923_b200.pulses import ricker
    from paper_1406_6923_b200.rom import LAST_BUILD_STATS
    from paper_1406_6923_b200.stepper import LAST_CFL
    wl, ops, alphas, (sa, sr), node_rx = _workload(cfg)
    n_sub, w, L = len(ops), wl.width, wl.layers
    rows = {sa: [sr]}
    for a, r in list(node_rx) + [locate(ijk, wl.counts, wl.p) for ijk in list(wl.sources[1:]) + list(extra_rows)]:
        rows.setdefault(a, []).append(r)
    dev = [torch.empty(n_sub * L * w * w, dtype=torch.float64, device="cuda") for _ in range(3)]
    ptrs = tuple(t.data_ptr() for t in dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows, device_out=ptrs)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stats = dict(LAST_BUILD_STATS)
    scl = dev[2].view(n_sub, L, w, w)
    idx = {a: i for i, a in enumerate(alphas)}
    for a in rows:
        models[a].scales = scl[idx[a]].cpu().numpy()
    t0 = time.perf_counter()
    lam, conv = cfl_estimate_coupled(models, device_coefficients=ptrs)
    cfl_s = time.perf_counter() - t0
    dt = 0.9 * 2.0 / math.sqrt(lam)
    src = SourceTerm(sa, project_source(models[sa], sr), ricker(wl.f0, wl.delay))
    probes = []
    for alpha, face in wl.face_receivers:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[alpha].state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append(Probe(alpha, wts))
    probes += [make_probe(models[a], r) for a, r in node_rx]
    return {"wl": wl, "ops": ops, "alphas": alphas, "models": models, "dev": dev, "ptrs": ptrs, "dt": dt,
            "lam": lam, "conv": conv, "src": src, "probes": probes,
            "build": {"seconds": build_s, "subdomains_per_s": n_sub / build_s, "stages_s": stats,
                      "cfl_seconds": cfl_s, "cfl_iterations": LAST_CFL.get("iterations")}}


def measure_fp64(pp, K, W, lrank=0):
    """Kernel-only (one persistent launch of K steps, CUDA events on the library's stream, probes
    recorded on the device) and e2e (CoupledStepper.run(K, probes): host profile table in, rows +
    norms out) of the fp64 U-form stepper."""
    import ctypes as C

    import torch
    from paper_1406_6923_b200 import CoupledStepper, _lib
    wl, models, dt, src, probes = pp["wl"], pp["models"], pp["dt"], pp["src"], pp["probes"]
    n_sub = len(models)
    st = CoupledStepper(models, dt, sources=(src,), device_coefficients=pp["ptrs"])
    try:
        st.initialize(_probes=probes)
        lib = st._lib
        ms = C.c_float(0.0)
        eb = _lib.errbuf()
        prof_w = st._profile_steps(0, max(W, 1))
        _lib.check(lib.sfw_step_run_resident(st._h, max(W, 1), 1, _lib.dptr(prof_w), C.byref(ms), eb, 1024), eb)
        prof_k = st._profile_steps(max(W, 1), K)
        flush_l2()
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(lrank) as clk:
            t0 = time.perf_counter()
            _lib.check(lib.sfw_step_run_resident(st._h, K, 1, _lib.dptr(prof_k), C.byref(ms), eb, 1024), eb)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        if dist.is_available() and dist.is_initialized():
            dist.barrier()
        kernel_s = ms.value * 1e-3
        alg_bytes, alg_flops, streamed = st.traffic()
        # e2e through the public API, from rest, as a user calls it (after one warm-up call of W steps)
        t0 = time.perf_counter()
        st.run(max(W, 1), probes=probes)
        cold_s = time.perf_counter() - t0
        flush_l2()
        t0 = time.perf_counter()
        times, rows = st.run(K, probes=probes)
        e2e_s = time.perf_counter() - t0
        assert np.all(np.isfinite(rows))
    finally:
        st.close()
    return {"kernel_s": kernel_s, "wall_s": wall, "e2e_s": e2e_s, "e2e_warmup_call_s": cold_s, "alg_bytes": alg_bytes,
            "alg_flops": alg_flops,
            "streamed": streamed, "clocks": clk.summary(), "n_sub": n_sub,
            "h2d": 8 * (1 + len(st.sources)), "d2h": 8 * (len(probes) + 1)}


def measure_fp32(pp, K, W):
    """fp32 W-form: kernel-only single launch (rows downloaded after it) and the chunked e2e call."""
    import ctypes as C

    from paper_1406_6923_b200 import CoupledStepper
    models, dt, src, probes = pp["models"], pp["dt"], pp["src"], pp["probes"]
    st = CoupledStepper(models, dt, sources=(src,), device_coefficients=pp["ptrs"], precision="fp32")
    try:
        st.run(max(W, 1), probes=probes)
        flush_l2()
        os.environ["SFW_NO_CHUNK"] = "1"
        try:
            st.run(K, probes=probes)
        finally:
            del os.environ["SFW_NO_CHUNK"]
        kernel_s = st.last_kernel_ms * 1e-3
        st.run(max(W, 1), probes=probes)  # warm the chunked download path
        flush_l2()
        t0 = time.perf_counter()
        _, rows = st.run(K, probes=probes)
        e2e_s = time.perf_counter() - t0
        assert np.all(np.isfinite(rows))
        b, sb = C.c_double(), C.c_double()
        st._lib.sfw_wform_traffic(st._h, C.byref(b), C.byref(sb))
    finally:
        st.close()
    return {"kernel_s": kernel_s, "e2e_s": e2e_s, "alg_bytes": b.value, "streamed": sb.value, "n_sub": len(models),
            "h2d": 16, "d2h": 8 * (len(probes) + 1)}


def measure_shots(pp, K, W):
    """Config 4: 32 independent single-source wavefields in one DMMA launch (run_shots)."""
    from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source
    from paper_1406_6923_b200.configs import locate, make_workload
    from paper_1406_6923_b200.pulses import ricker
    wl4 = make_workload(4)
    models, dt, probes = pp["models"], pp["dt"], pp["probes"]
    shots = []
    for ijk in wl4.sources:
        a, r = locate(ijk, wl4.counts, wl4.p)
        shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl4.f0, wl4.delay)))
    st = CoupledStepper(models, dt, device_coefficients=pp["ptrs"])
    try:
        st.run_shots(max(W, 1), shots, probes=probes)
        flush_l2()
        t0 = time.perf_counter()
        _, rows = st.run_shots(K, shots, probes=probes)
        e2e_s = time.perf_counter() - t0
        assert np.all(np.isfinite(rows))
        kernel_s = st.last_kernel_ms * 1e-3  # the same call's CUDA-event launch time
        ab, af, sb = st.shots_traffic()
    finally:
        st.close()
    return {"kernel_s": kernel_s, "e2e_s": e2e_s, "alg_bytes": ab, "alg_flops": af, "streamed": sb,
            "n_sub": len(models), "shots": len(shots), "h2d": 8 * len(shots), "d2h": 8 * len(shots) * (len(probes) + 1)}


def roofline(alg_bytes, alg_flops, K, kernel_s, traffic_key=None, fp64=True):
    """HBM roofline of one launch; when flops matter (config 4) the slower of bytes at the measured
    HBM peak and flops at the measured DMMA peak (north_star)."""
    peak, peak_kind = _peaks()
    achieved = alg_bytes * K / kernel_s / 1e9
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": _traffic(traffic_key, K) if traffic_key else None, "peak_kind": peak_kind,
           "alg_bytes_per_launch": alg_bytes * K, "alg_bytes_per_step": alg_bytes}
    if alg_flops:
        fpk, fpk_kind = _fp64_peak()
        t_hbm, t_fp = alg_bytes / (peak * 1e9), alg_flops / (fpk * 1e12)
        out.update({"alg_flops_per_step": alg_flops, "achieved_tflops": alg_flops * K / kernel_s / 1e12,
                    "fp64_peak_tflops": fpk, "fp64_peak_kind": fpk_kind,
                    "roofline_us_per_step": {"hbm": 1e6 * t_hbm, "fp64": 1e6 * t_fp}})
        if t_fp > t_hbm:
            out.update({"bound": "fp64", "frac": t_fp * K / kernel_s})
    return out


def _line(metric, value, K, W, ws, t_max, dtype, cfg_obj):
    return {"metric": metric, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * t_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic (seeded medium, SURVEY 8d); models built on the GPU from it",
            "config": cfg_obj}


def run_ours(args):
    import torch

    ws, rank, lrank = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(lrank)
    K, W = args.steps, args.warmup
    cfg = args.config
    if cfg == 4:  # config 4 = the config-3 models + 32 independent shot sources
        from paper_1406_6923_b200.configs import make_workload
        wl4 = make_workload(4)
        pp = prepare(3, extra_rows=wl4.sources)
        pp["wl"] = wl4
    else:
        pp = prepare(cfg)
    wl = pp["wl"]
    n_sub = len(pp["models"])
    if cfg == 4:
        r = measure_shots(pp, K, W)
        kernel_s = reduce_max(r["kernel_s"])
        value = replica_value(n_sub, K, ws, kernel_s)
        line = _line(METRIC, value, K, W, ws, kernel_s, "f64", config_key(wl, len(pp["probes"]), shots=r["shots"]))
        line["shot_steps_per_s"] = value * r["shots"]
        line["dof_updates_per_s"] = value * wl.layers * wl.width * r["shots"]
        line["roofline"] = roofline(r["alg_bytes"], r["alg_flops"], K, r["kernel_s"], "config4")
        clocks = None
    elif args.precision == "fp32":
        r = measure_fp32(pp, K, W)
        kernel_s = reduce_max(r["kernel_s"])
        value = replica_value(n_sub, K, ws, kernel_s)
        line = _line(METRIC.replace("fp64", "fp32 W-form"), value, K, W, ws, kernel_s, "f32",
                     config_key(wl, len(pp["probes"])))
        line["dof_updates_per_s"] = value * wl.layers * wl.width
        line["roofline"] = roofline(r["alg_bytes"], None, K, r["kernel_s"], f"config{cfg}_fp32")
        clocks = None
    else:
        r = measure_fp64(pp, K, W, lrank)
        kernel_s = reduce_max(r["kernel_s"])
        value = replica_value(n_sub, K, ws, kernel_s)
        line = _line(METRIC, value, K, W, ws, kernel_s, "f64", config_key(wl, len(pp["probes"])))
        line["dof_updates_per_s"] = value * wl.layers * wl.width
        line["roofline"] = roofline(r["alg_bytes"], None, K, r["kernel_s"], f"config{cfg}")
        clocks = r["clocks"]
    e2e_t = reduce_max(r["e2e_s"])
    line["e2e"] = {"value": replica_value(n_sub, K, ws, e2e_t), "unit": UNIT, "h2d_bytes_per_step": r["h2d"],
                   "d2h_bytes_per_step": r["d2h"],
                   "api": ("CoupledStepper.run_shots(K, 32 shots, probes)" if cfg == 4 else
                           "CoupledStepper(precision='fp32').run(K, probes)" if args.precision == "fp32" else
                           "CoupledStepper.run(K, probes)") +
                          ": initialize from rest, host Ricker table in, probe rows + |U| norms out (pinned staging); "
                          "timed after one warm-up call of W steps", "warmup_call_s": r.get("e2e_warmup_call_s")}
    line["roofline"]["streamed_bytes_per_step"] = r["streamed"]
    line["roofline"]["formula"] = ("8[(2L-1)w(w+1)/2 + 3LwS] bytes, S(2(2L-1)w^2+5Lw) flops per subdomain-step"
                                   if cfg == 4 else
                                   f"{4 if args.precision == 'fp32' else 8}[(2L-1)w(w+1)/2 + 3Lw] bytes per "
                                   "subdomain-step (SURVEY 8d)")
    line["run"] = {"dt": pp["dt"], "lambda_hat": pp["lam"], "cfl_converged": pp["conv"],
                   "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU", "kernel_ms": r["kernel_s"] * 1e3}
    line["rom_build"] = pp["build"]
    line["gpu_launches"] = 1
    line["clocks"] = clocks
    if rank != 0:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if clocks is None:
        line["clocks"] = {"note": "see the headline fp64 run"}
    cpu = None
    if not args.no_cpu and ws == 1:
        try:
            c = cpu_subset_run(cfg, min(K, args.cpu_steps), min(W, 3))
            val = c["rate"] / (32 if cfg == 4 else 1)
            cpu = {"value": val, "unit": UNIT, "cores": 1, "kind": "port", "sample": c["sample"] +
                   ("; config 4 = 32 separate single-source runs (SURVEY 8d), so 1/32 of the single-source rate"
                    if cfg == 4 else ""), "detail": c}
        except Exception as exc:  # the GPU line must still print
            cpu = {"value": None, "error": str(exc)[:300]}
    line["cpu_baseline"] = cpu
    # extras on one GPU only: under torchrun the other ranks have left (their measure_* barriers
    # would never be matched), and the scaling line is the headline
    head_pp = pp if (args.extra and cfg == 5 and args.precision == "fp64" and ws == 1) else None
    del pp
    torch.cuda.empty_cache()
    if head_pp is not None:
        try:
            line["extra"] = _extra_configs(args, line, head_pp)
        except Exception as exc:
            line["extra"] = {"error": str(exc)[:300]}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _entry(wl, r, K, metric_dtype, traffic_key, flops=False, shots=1):
    n_sub = r["n_sub"]
    ent = {"workload": _describe(wl) + (f", S={shots} shots" if shots > 1 else ""), "subdomains": n_sub,
           "steps": K, "ms_per_step": 1e3 * r["kernel_s"] / K, "value": n_sub * K / r["kernel_s"], "unit": UNIT,
           "dtype": metric_dtype,
           "roofline": roofline(r["alg_bytes"], r.get("alg_flops") if flops else None, K, r["kernel_s"], traffic_key),
           "e2e": {"value": n_sub * K / r["e2e_s"], "unit": UNIT, "h2d_bytes_per_step": r["h2d"],
                   "d2h_bytes_per_step": r["d2h"]}}
    if shots > 1:
        ent["shot_steps_per_s"] = shots * ent["value"]
    return ent


def _extra_configs(args, head, head_pp=None):
    """The other BASELINE configs with the same work as the headline (source, probes recorded every
    step, host profile table) -- kernel-only launch + e2e through the public API, + CPU sample."""
    import torch
    K, W = args.steps, args.warmup
    out = {}
    # config 5 fp32 W-form on the headline's models (chain stacks still in HBM), then configs 3, 4, 2
    for cfg in (5, 3, 2):
        from paper_1406_6923_b200.configs import make_workload
        extra = make_workload(4).sources if cfg == 3 else ()
        pp = head_pp if (cfg == 5 and head_pp is not None) else prepare(cfg, extra_rows=extra)
        if cfg == 5:
            head_pp = None  # released after its fp32 measurement
        wl = pp["wl"]
        if cfg != 5:
            r = measure_fp64(pp, K, W)
            e = _entry(wl, r, K, "f64", f"config{cfg}")
            e["probes"] = len(pp["probes"])
            e["rom_build"] = pp["build"]
            if not args.no_cpu and cfg == 3:
                try:
                    c = cpu_subset_run(3, min(K, args.cpu_steps), min(W, 3))
                    e["cpu_baseline"] = {"value": c["rate"], "unit": UNIT, "cores": 1, "kind": "port",
                                         "sample": c["sample"]}
                    out["_cpu3"] = c["rate"]
                except Exception as exc:
                    e["cpu_baseline"] = {"error": str(exc)[:200]}
            out[f"config{cfg}"] = e
        if cfg in (5, 3):
            r = measure_fp32(pp, K, W)
            e = _entry(wl, r, K, "f32", f"config{cfg}_fp32")
            e["workload"] += ", fp32 W-form"
            e["probes"] = len(pp["probes"])
            out[f"config{cfg}_fp32"] = e
        if cfg == 3:
            r = measure_shots(pp, K, W)
            wl4 = make_workload(4)
            e = _entry(wl4, r, K, "f64", "config4", flops=True, shots=r["shots"])
            e["probes"] = len(pp["probes"])
            if "_cpu3" in out:
                e["cpu_baseline"] = {"value": out["_cpu3"] / 32, "unit": UNIT, "cores": 1, "kind": "port",
                                     "sample": "config-3 CPU sample rate / 32 (config 4 = 32 separate single-source "
                                               "runs, SURVEY 8d)"}
            out["config4"] = e
        del pp
        torch.cuda.empty_cache()
    out.pop("_cpu3", None)
    return out


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from paper_1406_6923_b200.configs import make_workload
    cfg = args.config
    wl = make_workload(cfg)
    c = cpu_subset_run(cfg, args.steps, args.warmup)
    n_probes = len(wl.face_receivers) * wl.modes_per_face + len(wl.node_receivers)
    val = c["rate"] / (32 if cfg == 4 else 1)
    line = _line(METRIC if args.precision == "fp64" else METRIC.replace("fp64", "fp32 W-form"), val, args.steps,
                 args.warmup, ws, c["seconds"], "f64",
                 config_key(wl, n_probes, shots=32 if cfg == 4 else 1))
    line["ms_per_step"] = 1e3 * c["seconds"] / args.steps
    line["data"] = "synthetic (seeded medium, SURVEY 8d); models built on the host by the oracle port of rom.py"
    line["impl"] = "reference"
    line["cpu_baseline"] = {"value": val, "unit": UNIT, "cores": 1, "kind": "port", "sample": c["sample"]}
    line["e2e"] = {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    line["run"] = {k: c[k] for k in ("dt", "lambda_hat", "cfl_converged", "cfl_seconds", "window", "subdomains",
                                     "probes")}
    line["rom_build"] = {"seconds": c["build_seconds"], "subdomains_per_s": c["build_subdomains_per_s"],
                         "cores": c["build_cores"], "kind": "port (scipy SuperLU + LAPACK, one process per core)"}
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
    run_leapfrog(a, dt, args.steps, **kw)  # warm-up call of the timed shape (per-run buffers sized once)
    flush_l2()
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
            "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": K + 1}  # K x k_fdtd<0> + k_fd_norms
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extra", type=int, default=1,
                    help="with config 5 fp64: also measure configs 5 fp32, 3 (fp64/fp32), 4 and 2 (default on)")
    ap.add_argument("--cpu-steps", type=int, default=200, help="cap on the CPU sample's timed steps")
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
