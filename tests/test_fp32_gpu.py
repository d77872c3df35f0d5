"""fp32 W-form stepping variant (<= 1e-4 vs the fp64 reference).

The W-form (U_j = G_j W_j; Lanczos block-tridiagonal operator; interface mass
1/2) is the reference ROM to rounding; in fp32 it stays ~1e-6 from the fp64
U-form reference where U-form fp32 diverges.
"""

import math

import numpy as np
import pytest

from helpers import face_probes, load_golden, models_from_arrays, partition_for, rel
from oracle import sfw_oracle as so
from paper_1406_6923_b200 import (ConfigError, CoupledStepper, Probe, SourceTerm, build_models,
                                  cfl_estimate_coupled, project_source)
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker

pytestmark = pytest.mark.gpu


def test_fp32_config1_vs_reference_golden():
    g = load_golden("golden_c1.npz")
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src_alpha = tuple(int(x) for x in g["src_alpha"])
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    src = SourceTerm(src_alpha, g["src_vec"], so.ricker(wl.f0, wl.delay))
    with CoupledStepper(models, float(g["dt"]), sources=(src,), precision="fp32") as st:
        times, rows = st.run(wl.n_steps, probes=probes)
        uc = st.u_curr
        with pytest.raises(ConfigError):
            st.energy()
    assert np.array_equal(times, g["times"])
    e = rel(rows, g["rows"])
    print("fp32 config1 traces vs reference", e)
    assert e < 1e-4
    with CoupledStepper(models, float(g["dt"]), sources=(src,)) as st64:
        st64.run(wl.n_steps, probes=probes)
        u64 = st64.u_curr
    num = np.sqrt(sum(np.sum((uc[a] - u64[a]) ** 2) for a in u64))
    den = np.sqrt(sum(np.sum(u64[a] ** 2) for a in u64))
    assert num / den < 1e-4


def test_fp32_m9k8_vs_fp64():
    wl = make_workload(3, counts=(2, 2, 2), n_steps=300)
    ext = tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing))
    part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in sorted(s.alpha for s in part.subdomains)]
    sa, sr = locate(wl.sources[0], wl.counts, wl.p)
    rows_req = {sa: [sr]}
    node = [locate(ijk, wl.counts, wl.p) for ijk in wl.node_receivers]
    for a, r in node:
        rows_req.setdefault(a, []).append(r)
    models = build_models(ops, 9, 8, wl.shift, rows=rows_req)
    lam, _ = cfl_estimate_coupled(models)
    dt = 0.9 * 2.0 / math.sqrt(lam)
    src = SourceTerm(sa, project_source(models[sa], sr), ricker(wl.f0, wl.delay))
    from paper_1406_6923_b200 import make_probe
    probes = [Probe(a, w) for a, w in face_probes(models, wl)] + [make_probe(models[a], r) for a, r in node]
    with CoupledStepper(models, dt, sources=(src,)) as st64:
        _, r64 = st64.run(wl.n_steps, probes=probes)
    with CoupledStepper(models, dt, sources=(src,), precision="fp32") as st32:
        _, r32 = st32.run(wl.n_steps, probes=probes)
    e = rel(r32, r64)
    print("fp32 m9k8 traces vs fp64", e)
    assert e < 1e-4


@pytest.mark.parametrize("record_every", [1, 4])
def test_fp32_chunked_run_equals_single_launch(record_every, monkeypatch):
    """Chunked W-form runs (rows downloaded while later chunks compute) equal one launch bit for bit."""
    g = load_golden("golden_c1.npz")
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src = SourceTerm(tuple(int(x) for x in g["src_alpha"]), g["src_vec"], so.ricker(wl.f0, wl.delay))
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    n = 161
    out = {}
    for mode in ("single", "chunked"):
        if mode == "single":
            monkeypatch.setenv("SFW_NO_CHUNK", "1")
        else:
            monkeypatch.delenv("SFW_NO_CHUNK")
            monkeypatch.setenv("SFW_CHUNK_BYTES", "1")
        with CoupledStepper(models, float(g["dt"]), sources=(src,), precision="fp32") as st:
            t, r = st.run(n, probes=probes, record_every=record_every)
            out[mode] = (t, r, st.u_curr)
    (ts, rs, us), (tc, rc, uc) = out["single"], out["chunked"]
    assert rs.shape == (1 + n // record_every, len(probes))
    assert np.array_equal(ts, tc) and np.array_equal(rs, rc)
    for a in us:
        assert np.array_equal(us[a], uc[a])


def test_no_reads_of_unwritten_device_memory(monkeypatch):
    """With SFW_POISON=a every fresh library allocation is filled with NaN (debug hook in dalloc):
    a kernel that read memory nothing wrote first (e.g. an upload whose DMA had not landed, the
    race fixed by sfw_h2d) would turn the traces into NaN.  fp64 and fp32 config-1 runs stay
    finite and equal to the unpoisoned runs."""
    g = load_golden("golden_c1.npz")
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src = SourceTerm(tuple(int(x) for x in g["src_alpha"]), g["src_vec"], so.ricker(wl.f0, wl.delay))
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    out = {}
    for poison in ("", "a"):
        if poison:
            monkeypatch.setenv("SFW_POISON", poison)
        for prec in ("fp64", "fp32"):
            with CoupledStepper(models, float(g["dt"]), sources=(src,), precision=prec) as st:
                out[(poison, prec)] = st.run(120, probes=probes)[1]
    for prec in ("fp64", "fp32"):
        assert np.isfinite(out[("a", prec)]).all()
        assert np.array_equal(out[("a", prec)], out[("", prec)])


def test_fp32_growth_detector_stops_early():
    """An unstable dt (3x the CFL limit): the library checks |W| chunk by chunk and stops launching
    at the first failing step; run() then replays to that step, so steps_done / u_curr are the
    state at the raise, as the reference's detector leaves them (stepper.py:379-389)."""
    from paper_1406_6923_b200 import InstabilityError
    g = load_golden("golden_c1.npz")
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src_alpha = tuple(int(x) for x in g["src_alpha"])
    src = SourceTerm(src_alpha, g["src_vec"], so.ricker(wl.f0, wl.delay))
    dt = 3.0 * 2.0 / math.sqrt(float(g["lam"]))
    with CoupledStepper(models, dt, sources=(src,), precision="fp32") as st:
        with pytest.raises(InstabilityError):
            st.run(20000)
        k = st.steps_done
        assert 0 < k < 20000
        uk = st.u_curr
        st.run(k - 1)  # one step before the failing one: no raise
        assert st.steps_done == k - 1
    assert all(np.all(np.isfinite(v)) for v in uk.values())
