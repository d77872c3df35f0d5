"""GPU parity of the off-line stage (batched sm_100a ROM build) through the C ABI.

Contract: Lanczos blocks (A_j, B_j) and Gamma_j within 1e-9
relative per block; Gamma-hat_j and G_j within 1e-9 for j < L; the last layer's
Gamma-hat_L / G_L are intrinsically ill-conditioned at m=9, k=8 (cond(Gamma_9)
~ 1e17), so they are compared at 10 x the oracle's own algorithm floor
(SuperLU vs dense Cholesky: 6.4e-7 / 3.2e-7, SURVEY appendix probe2); the GPU build
measures 5.6e-10 / 2.8e-10 there, so the assert is 1e-8 (a regression of 20x fails).
"""

import numpy as np
import pytest

from helpers import face_probes, load_golden, partition_for, rel
from oracle import sfw_oracle as so
from paper_1406_6923_b200 import (ConfigError, CoupledStepper, NumericalError, Probe, SourceTerm,
                                  build_models, build_subdomain_model, cfl_estimate_coupled, project_source)
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.configs import locate, make_workload

pytestmark = pytest.mark.gpu


def _ops(part, c_field, alphas=None):
    subs = [s.alpha for s in part.subdomains if alphas is None or s.alpha in alphas]
    return [pg.assemble_subdomain_operator(part, a, c_field) for a in sorted(subs)]


def _check_blocks(models, g, order, last_tol=1e-9, pre=""):
    worst = {}
    for i, a in enumerate(order):
        md = models[a]
        L = md.layers
        for key, got, want in [("tdiag", md.tdiag, g[pre + "tdiag"][i]), ("toff", md.toff, g[pre + "toff"][i]),
                               ("gammas", md.gammas, g[pre + "gammas"][i])]:
            for j in range(len(want)):
                e = rel(got[j], want[j])
                worst[key] = max(worst.get(key, 0.0), e)
                assert e < 1e-9, (a, key, j, e)
        for key, got, want in [("hats", md.gamma_hats, g[pre + "hats"][i]), ("scales", md.scales, g[pre + "scales"][i])]:
            for j in range(L):
                e = rel(got[j], want[j])
                worst[key + ("_L" if j == L - 1 else "")] = max(worst.get(key + ("_L" if j == L - 1 else ""), 0.0), e)
                assert e < (last_tol if j == L - 1 else 1e-9), (a, key, j, e)
    return worst


@pytest.mark.parametrize("tag", ["pair", "quad"])
def test_toy_build_matches_reference_golden(tag):
    g = load_golden("golden_toy.npz")
    pre = tag + "_"
    counts = tuple(int(x) for x in g[pre + "counts"])
    part = partition_for(counts, (5, 5, 5), tuple(float(c) for c in counts))
    ops = _ops(part, g[pre + "c_field"])
    order = [op.alpha for op in ops]
    models = build_models(ops, int(g[pre + "m"]), int(g[pre + "n"]), 4.0, basis="all")
    print(_check_blocks(models, g, order, pre=pre))
    for i, a in enumerate(order):
        # V Q is unique up to rounding (positive-diagonal gauges)
        assert rel(models[a].basis, g[pre + "basis"][i]) < 1e-9


def test_config1_build_matches_reference_golden():
    g = load_golden("golden_c1.npz")
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    ops = _ops(part, wl.c_field)
    order = [op.alpha for op in ops]
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift)
    print(_check_blocks(models, g, order))


def test_m9k8_build_matches_reference_golden():
    g = load_golden("golden_m9k8.npz")
    wl = make_workload(3, counts=(3, 3, 3))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    alphas = [tuple(int(x) for x in a) for a in g["alphas"]]
    ops = _ops(part, wl.c_field, set(alphas))
    order = [op.alpha for op in ops]
    assert order == alphas
    models = build_models(ops, 9, 8, wl.shift)
    print(_check_blocks(models, g, order, last_tol=1e-8))  # measured 5.6e-10


def test_config1_end_to_end_traces():
    """GPU build + GPU CFL + GPU stepping vs the reference's build + step (golden traces)."""
    g = load_golden("golden_c1.npz")
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    ops = _ops(part, wl.c_field)
    src_alpha, row = locate(wl.sources[0], wl.counts, wl.p)
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, basis={src_alpha})
    lam, conv = cfl_estimate_coupled(models)
    assert conv and abs(lam - float(g["lam"])) <= 1e-8 * lam
    vec = project_source(models[src_alpha], row)
    assert rel(vec, g["src_vec"]) < 1e-9
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    with CoupledStepper(models, float(g["dt"]), sources=(SourceTerm(src_alpha, vec, so.ricker(wl.f0, wl.delay)),)) as st:
        times, rows = st.run(wl.n_steps, probes=probes)
    e = rel(rows, g["rows"])
    print("end-to-end trace rel err", e)
    assert e < 1e-9


def test_single_subdomain_api_and_errors():
    g = load_golden("golden_toy.npz")
    part = partition_for((2, 1, 1), (5, 5, 5), (2.0, 1.0, 1.0))
    op = pg.assemble_subdomain_operator(part, (0, 0, 0), g["pair_c_field"])
    md = build_subdomain_model(op, 1, 2, 4.0)
    # the depth-2 block deflates (reference sizes [6, 6, 5]): truncated to 2 complete layers
    assert md.layers == 2 and md.truncated and md.deflated
    assert md.gammas.shape == (2, 6, 6) and md.basis.shape == (125, 12)
    assert rel(md.gammas, g["pair_gammas"][0]) < 1e-9
    assert np.linalg.norm(md.gamma_hats[0] - np.eye(6)) < 1e-9
    md1 = build_subdomain_model(op, 1, 1, 4.0)
    assert md1.layers == 2 and not md1.truncated
    with pytest.raises(NumericalError):
        build_subdomain_model(op, 1, 2, 0.0)
    with pytest.raises(ConfigError):
        build_subdomain_model(op, 5, 2, 4.0)
    with pytest.raises(NumericalError):
        build_subdomain_model(op, 1, 0, 4.0)


def test_build_is_bitwise_repeatable():
    """The batched build (DMMA GEMMs, DMMA line passes of the PCG, CholQR2) gives the same bits on every
    run: three builds of a 2 x 2 x 2 m9k8 tiling of the config-3 medium (tools/rom_stress.py is the long
    version: 20 of 20 builds of 512 subdomains equal)."""
    wl = make_workload(3, counts=(2, 2, 2))
    ext = tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing))
    part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in sorted(s.alpha for s in part.subdomains)]
    ref = None
    for _ in range(3):
        models = build_models(ops, wl.modes_per_face, wl.n, wl.shift)
        got = [np.ascontiguousarray(x).tobytes() for a in sorted(models)
               for x in (models[a].gammas, models[a].gamma_hats, models[a].scales, models[a].tdiag, models[a].toff)]
        if ref is None:
            ref = got
        assert got == ref
