"""Full-size parity against the REAL reference (golden_c2 / golden_c5) and the CPU oracle.

* Config 2 end to end at full size: GPU build of all 512 m4k6 subdomains + GPU CFL + 1000 GPU
  leapfrog steps vs the reference's own build + CFL + 1000 steps (tests/golden/make_golden.py
  golden_c2), traces on the 264 bench receivers <= 1e-9; the inclusion-cut subdomains' A_j, B_j,
  Gamma_j <= 1e-9 (reference rom.py:359-434, stepper.py:391-415).
* Config 5 recipe: the reference's m9k8 chains of corner / edge / face / interior / source /
  inclusion-cut subdomains of the full 513x513x257 config-5 field vs the GPU build <= 1e-9;
  a full-size (16384-subdomain) fp64 window of 60 steps vs the batched CPU oracle on the same
  GPU-built coefficients (tolerance max(1e-9, 10 x the oracle's own summation floor)),
  and the fp32 W-form variant vs fp64 over 400 steps (<= 1e-4).
"""

import math

import numpy as np
import pytest

from helpers import batched_oracle, load_golden, rel
from paper_1406_6923_b200 import (CoupledStepper, Probe, SourceTerm, build_models, cfl_estimate_coupled,
                                  make_probe, project_source)
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker

pytestmark = pytest.mark.gpu


def _partition(wl):
    ext = tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing))
    return pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))


def _bench_probes(models, wl):
    probes = []
    for alpha, face in wl.face_receivers:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[alpha].state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append(Probe(alpha, wts))
    return probes


def _chain_errors(md, g, i, pre=""):
    """Worst per-block relative error of A_j, B_j, Gamma_j and of Gamma-hat_j, scales (j < L)."""
    e = {}
    L = md.layers
    for key, got, want in (("tdiag", md.tdiag, g[pre + "tdiag"][i]), ("toff", md.toff, g[pre + "toff"][i]),
                           ("gammas", md.gammas, g[pre + "gammas"][i])):
        e[key] = max(rel(got[j], want[j]) for j in range(len(want)))
    for key, got, want in (("hats", md.gamma_hats, g[pre + "hats"][i]), ("scales", md.scales, g[pre + "scales"][i])):
        e[key] = max(rel(got[j], want[j]) for j in range(L - 1))
        e[key + "_L"] = rel(got[L - 1], want[L - 1])
    return e


def test_config2_full_size_end_to_end_vs_reference():
    g = load_golden("golden_c2.npz")
    wl = make_workload(2)
    part = _partition(wl)
    alphas = sorted(s.alpha for s in part.subdomains)
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in alphas]
    sa, sr = locate(wl.sources[0], wl.counts, wl.p)
    node = [locate(ijk, wl.counts, wl.p) for ijk in wl.node_receivers]
    rows = {sa: [sr]}
    for a, r in node:
        rows.setdefault(a, []).append(r)
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows)
    assert len(models) == 512 and all(md.layers == 7 for md in models.values())
    worst = {}
    for i, a in enumerate(tuple(int(x) for x in al) for al in g["sub_alphas"]):
        for k, v in _chain_errors(models[a], g, i, pre="sub_").items():
            worst[k] = max(worst.get(k, 0.0), v)
    print("config-2 inclusion-cut/source/receiver subdomains vs reference:", worst)
    for k in ("tdiag", "toff", "gammas", "hats", "scales"):
        assert worst[k] < 1e-9, (k, worst[k])
    assert worst["hats_L"] < 1e-8 and worst["scales_L"] < 1e-8
    lam, conv = cfl_estimate_coupled(models)
    print("lambda GPU", lam, "reference", float(g["lam"]))
    assert conv and abs(lam - float(g["lam"])) <= 1e-10 * lam
    dt = 0.9 * 2.0 / math.sqrt(lam)
    vec = project_source(models[sa], sr)
    assert rel(vec, g["src_vec"]) < 1e-9
    node_w = np.stack([make_probe(models[a], r).weights for a, r in node])
    assert rel(node_w, g["node_probe_w"]) < 1e-9
    probes = _bench_probes(models, wl) + [Probe(a, w) for (a, _), w in zip(node, node_w)]
    with CoupledStepper(models, dt, sources=(SourceTerm(sa, vec, ricker(wl.f0, wl.delay)),)) as st:
        times, tr = st.run(int(g["n_steps"]), probes=probes)
        assert st.message_count == int(g["message_count"])
        en = st.energy()
    e = rel(tr, g["rows"])
    print(f"config-2 end to end (GPU build+CFL+1000 steps vs reference): traces {e:.2e}, "
          f"energy {abs(en - float(g['energy'])) / abs(float(g['energy'])):.2e}")
    assert np.allclose(times, g["times"], rtol=1e-12, atol=0)
    assert e < 1e-9
    assert abs(en - float(g["energy"])) <= 1e-8 * abs(float(g["energy"]))


@pytest.fixture(scope="module")
def c5():
    wl = make_workload(5)
    part = _partition(wl)
    alphas = sorted(s.alpha for s in part.subdomains)
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in alphas]
    sa, sr = locate(wl.sources[0], wl.counts, wl.p)
    node = [locate(ijk, wl.counts, wl.p) for ijk in wl.node_receivers]
    rows = {sa: [sr]}
    for a, r in node:
        rows.setdefault(a, []).append(r)
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, rows=rows)
    lam, conv = cfl_estimate_coupled(models)
    assert conv
    dt = 0.9 * 2.0 / math.sqrt(lam)
    src = SourceTerm(sa, project_source(models[sa], sr), ricker(wl.f0, wl.delay))
    probes = _bench_probes(models, wl) + [make_probe(models[a], r) for a, r in node]
    return wl, models, dt, src, probes


def test_config5_subdomains_vs_reference(c5):
    wl, models, _, _, _ = c5
    g = load_golden("golden_c5.npz")
    worst = {}
    for i, a in enumerate(tuple(int(x) for x in al) for al in g["alphas"]):
        md = models[a]
        c = wl.c_field[16 * a[0]:16 * a[0] + 17, 16 * a[1]:16 * a[1] + 17, 16 * a[2]:16 * a[2] + 17]
        assert np.array_equal(c, g["c_slices"][i])
        assert md.layers == int(g["layers"][i]) == 9
        e = _chain_errors(md, g, i)
        print("config-5", a, {k: f"{v:.1e}" for k, v in e.items()})
        for k in ("tdiag", "toff", "gammas", "hats", "scales"):
            worst[k] = max(worst.get(k, 0.0), e[k])
            assert e[k] < 1e-9, (a, k, e[k])
        # last layer: cond(Gamma_9) ~ 1e17 -> compared at 10 x the oracle's algorithm floor
        # (measured <= 2.4e-9 on these seven subdomains; the assert is ~10x that)
        assert e["hats_L"] < 3e-8 and e["scales_L"] < 3e-8, (a, e)
    print("config-5 worst", worst)


def test_config5_full_size_fp64_window_vs_oracle(c5):
    wl, models, dt, src, probes = c5
    assert len(models) == 16384
    n = 60
    with CoupledStepper(models, dt, sources=(src,)) as st:
        _, tr = st.run(n, probes=probes)
        uc = st.u_curr
    bo, idx = batched_oracle(models, dt, sources=(src,))
    oprobes = [(idx[p.alpha], p.weights) for p in probes]
    _, ref = bo.run(n, probes=oprobes)
    err = rel(tr, ref)
    order = sorted(models)
    es = rel(np.stack([uc[a] for a in order]), bo.u_curr.reshape(len(order), -1))
    tol = tol_s = 1e-9
    if err > tol or es > tol_s:  # m9k8 floor = the oracle against itself in another summation order
        alt, _ = batched_oracle(models, dt, sources=(src,), alt=True)
        tr_alt = alt.run(n, probes=oprobes)[1]
        tol = max(tol, 10 * rel(tr_alt, ref))
        tol_s = max(tol_s, 10 * rel(alt.u_curr, bo.u_curr))
    print(f"config-5 full size, {n} steps: traces vs oracle {err:.2e} (tol {tol:.1e}), "
          f"state {es:.2e} (tol {tol_s:.1e}: the deep layers carry Gamma-hat_9, cond ~1e17)")
    assert err <= tol and es <= tol_s


def test_config5_fp32_vs_fp64(c5):
    wl, models, dt, src, probes = c5
    n = 400
    with CoupledStepper(models, dt, sources=(src,)) as st:
        _, r64 = st.run(n, probes=probes)
    with CoupledStepper(models, dt, sources=(src,), precision="fp32") as st32:
        _, r32 = st32.run(n, probes=probes)
    e = rel(r32, r64)
    print(f"config-5 fp32 W-form vs fp64 over {n} steps: {e:.2e}")
    assert e <= 1e-4
