"""Generate golden vectors from the REAL reference implementation.

Run in the build container only (the reference is not on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src:/root/repo OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

It imports ``sfwave`` from /root/reference/pkg/src (read-only), feeds it the
seeded inputs of ``paper_1406_6923_b200.configs`` and stores the outputs as
small ``.npz`` fixtures next to this script.  ``tests/test_oracle_golden.py``
pins ``oracle/sfw_oracle.py`` against them; the GPU parity tests then compare
the CUDA path against the pinned oracle and against these fixtures.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from sfwave.grid import (  # noqa: E402  (reference package)
    DomainSpec, MediumModel, assemble_subdomain_operator, build_partition, sample_medium)
from sfwave.rom import (  # noqa: E402
    block_lanczos, build_krylov_basis, build_subdomain_model, project_reduced, subdomain_inputs)
from sfwave.sim import make_pulse  # noqa: E402
from sfwave.stepper import (  # noqa: E402
    CoupledStepper, Probe, SourceTerm, cfl_estimate_coupled, make_probe, project_source)

from paper_1406_6923_b200.configs import locate, make_workload  # noqa: E402


def chain_blocks(op, m, n, shift, layers):
    f = subdomain_inputs(op, m)
    basis, sizes = build_krylov_basis(op.matrix, f, n, shift)
    w = 6 * m
    basis = basis[:, :layers * w]
    at, ft = project_reduced(basis, op.matrix, f)
    ch = block_lanczos(at, ft)
    return np.stack(ch.diag_blocks), np.stack(ch.off_blocks), ch.entry_block


def workload_models(wl, alphas=None):
    spec = DomainSpec(tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing)),
                      wl.counts, wl.p)
    part = build_partition(spec)
    ops, models = {}, {}
    for sub in part.subdomains:
        if alphas is not None and sub.alpha not in alphas:
            continue
        op = assemble_subdomain_operator(part, sub.alpha, wl.c_field)
        ops[sub.alpha] = op
        models[sub.alpha] = build_subdomain_model(op, wl.modes_per_face, wl.n, wl.shift)
    return part, ops, models


def pack_models(out, prefix, ops, models, m, n, shift):
    order = sorted(models)
    out[prefix + "alphas"] = np.array(order)
    out[prefix + "gammas"] = np.stack([models[a].gammas for a in order])
    out[prefix + "hats"] = np.stack([models[a].gamma_hats for a in order])
    out[prefix + "scales"] = np.stack([models[a].scales for a in order])
    tds, tos, ents = [], [], []
    for a in order:
        td, to, en = chain_blocks(ops[a], m, n, shift, models[a].layers)
        tds.append(td)
        tos.append(to)
        ents.append(en)
    out[prefix + "tdiag"] = np.stack(tds)
    out[prefix + "toff"] = np.stack(tos)
    out[prefix + "entry"] = np.stack(ents)


def golden_config(cfg, counts, n_steps, name, record_models=True, basis_rows=True):
    wl = make_workload(cfg, counts=counts, n_steps=n_steps)
    part, ops, models = workload_models(wl)
    out = {"c_field": wl.c_field, "counts": np.array(wl.counts), "m": wl.modes_per_face,
           "n": wl.n, "shift": wl.shift, "n_steps": wl.n_steps, "f0": wl.f0}
    if record_models:
        pack_models(out, "", ops, models, wl.modes_per_face, wl.n, wl.shift)
    lam, conv = cfl_estimate_coupled(models)
    dt = 0.9 * 2.0 / math.sqrt(lam)
    out["lam"] = lam
    out["dt"] = dt
    src_alpha, src_row = locate(wl.sources[0], wl.counts, wl.p)
    pulse = make_pulse("ricker", wl.f0, 1.2 / wl.f0)
    vec = project_source(models[src_alpha], src_row, 1.0)
    out["src_alpha"] = np.array(src_alpha)
    out["src_row"] = src_row
    out["src_vec"] = vec
    if basis_rows:
        out["src_basis_row"] = models[src_alpha].basis[src_row].copy()
    probes = []
    for alpha, face in wl.face_receivers:
        md = models[alpha]
        for q in range(wl.modes_per_face):
            wts = np.zeros(md.state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append(Probe(alpha, wts))
    node_w, node_basis = [], []
    for ijk in wl.node_receivers:
        alpha, row = locate(ijk, wl.counts, wl.p)
        pr = make_probe(models[alpha], row)
        probes.append(pr)
        node_w.append(pr.weights)
        node_basis.append(models[alpha].basis[row].copy())
    if node_w:
        out["node_probe_w"] = np.stack(node_w)
        out["node_basis_rows"] = np.stack(node_basis)
    with CoupledStepper(models, dt, sources=(SourceTerm(src_alpha, vec, pulse),)) as st:
        times, rows = st.run(wl.n_steps, probes=probes)
        out["times"] = times
        out["rows"] = rows
        out["message_count"] = st.message_count
        out["energy"] = st.energy()
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, {k: np.shape(v) for k, v in out.items()})


def golden_toy():
    """Reference-test-sized cases (p=5, unit cube, dimensionless shift 4)."""
    out = {}
    rng = np.random.default_rng(77)
    for tag, counts, m, n, med in [
        ("pair", (2, 1, 1), 1, 2, None),
        ("quad", (2, 2, 1), 4, 2, "layer"),
    ]:
        spec = DomainSpec(tuple(float(c) for c in counts), counts, (5, 5, 5))
        part = build_partition(spec)
        if med == "layer":
            from sfwave.grid import Box
            medium = MediumModel(1.0, ((Box((0.0, 0.0, 0.5), (2.0, 2.0, 1.0)), 1.7),))
        else:
            medium = MediumModel(1.0)
        c = sample_medium(medium, part)
        ops, models = {}, {}
        for sub in part.subdomains:
            ops[sub.alpha] = assemble_subdomain_operator(part, sub.alpha, c)
            models[sub.alpha] = build_subdomain_model(ops[sub.alpha], m, n, 4.0)
        pre = tag + "_"
        out[pre + "c_field"] = c
        out[pre + "counts"] = np.array(counts)
        out[pre + "m"] = m
        out[pre + "n"] = n
        pack_models(out, pre, ops, models, m, n, 4.0)
        order = sorted(models)
        out[pre + "basis"] = np.stack([models[a].basis for a in order])
        out[pre + "matrix0"] = ops[order[0]].matrix.toarray()
        lam, conv = cfl_estimate_coupled(models)
        out[pre + "lam"] = lam
        dt = 0.5 * 2.0 / math.sqrt(lam)
        out[pre + "dt"] = dt
        u0 = {a: rng.standard_normal(models[a].state_size) for a in order}
        # shared-face replicas must agree
        for a in order:
            for f, b in sorted(models[a].neighbors.items()):
                if b > a:
                    u0[b][models[b].face_slice(f ^ 1)] = u0[a][models[a].face_slice(f)]
        v0 = {a: np.zeros(models[a].state_size) for a in order}
        out[pre + "u0"] = np.stack([u0[a] for a in order])
        row = 31  # strictly interior node of a p=5 subdomain
        vec = project_source(models[order[0]], row, 1.0)
        out[pre + "src_vec"] = vec
        pr = make_probe(models[order[-1]], row)
        out[pre + "probe_w"] = pr.weights
        pulse = make_pulse("ricker", 1.0, 1.2)
        with CoupledStepper(models, dt, sources=(SourceTerm(order[0], vec, pulse),)) as st:
            times, rows = st.run(40, probes=[pr], u0=u0, v0=v0)
            out[pre + "times"] = times
            out[pre + "rows"] = rows
            out[pre + "u_curr"] = np.stack([st.u_curr[a] for a in order])
            out[pre + "u_prev"] = np.stack([st.u_prev[a] for a in order])
            out[pre + "energy"] = st.energy()
            out[pre + "messages"] = st.message_count
    np.savez_compressed(os.path.join(HERE, "golden_toy.npz"), **out)
    print("golden_toy.npz", len(out))


def golden_m9k8():
    """One interior m=9, k=8 subdomain of the config-3 medium recipe (3x3x3 tiling)."""
    wl = make_workload(3, counts=(3, 3, 3))
    part, ops, models = workload_models(wl, alphas={(1, 1, 1), (0, 0, 0)})
    out = {"c_field": wl.c_field, "counts": np.array(wl.counts), "m": 9, "n": 8, "shift": wl.shift}
    pack_models(out, "", ops, models, 9, 8, wl.shift)
    np.savez_compressed(os.path.join(HERE, "golden_m9k8.npz"), **out)
    print("golden_m9k8.npz")


def golden_io():
    """Files written by the reference io.py (.rom, coefficient arrays, .trc, .meta.txt) + cache keys."""
    from sfwave.io import TraceRecord, save_model, write_meta, write_traces
    from sfwave.sim import _model_cache_key
    spec = DomainSpec((2.0, 1.0, 1.0), (2, 1, 1), (5, 5, 5))
    part = build_partition(spec)
    c = sample_medium(MediumModel(1.0), part)
    keys = {}
    for sub in part.subdomains:
        op = assemble_subdomain_operator(part, sub.alpha, c)
        md = build_subdomain_model(op, 1, 2, 4.0)
        tag = "".join(map(str, sub.alpha))
        save_model(os.path.join(HERE, f"io_pair{tag}.rom"), md)
        keys["key_" + tag] = _model_cache_key(op, 1, md.layers, 4.0)
    rng = np.random.default_rng(5)
    rec = TraceRecord(coords=rng.standard_normal((3, 3)), dt=0.00125, samples=rng.standard_normal((7, 3)))
    write_traces(os.path.join(HERE, "io.trc"), rec)
    write_meta(os.path.join(HERE, "io.meta.txt"), {"run": "golden", "dt": 0.1 + 0.2, "steps": 7,
                                                    "lambda_hat": np.float64(1.0) / 3.0, "tag": "a: b"})
    np.savez_compressed(os.path.join(HERE, "golden_io.npz"), c_field=c, **{k: np.array(v) for k, v in keys.items()})
    print("golden_io.npz", keys)


def golden_fdtd():
    """Fine-grid leapfrog (reference.py:86-157) on the config-1 grid, driven as sim.run_reference does."""
    from sfwave.grid import assemble_global_operator
    from sfwave.reference import estimate_lambda_max, run_leapfrog
    wl = make_workload(1)
    spec = DomainSpec(tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing)), wl.counts, wl.p)
    part = build_partition(spec)
    a = assemble_global_operator(part, wl.c_field)
    lam = estimate_lambda_max(a)
    dt = 0.9 * 2.0 / math.sqrt(lam)
    shape = part.global_shape
    src = int(np.ravel_multi_index(tuple(wl.sources[0]), shape))
    vec = np.zeros(a.shape[0])
    c_flat = wl.c_field.ravel()
    vec[src] = 1.0 / c_flat[src]
    sx, sy, sz = (int(v) for v in wl.sources[0])
    rec = [int(np.ravel_multi_index((x, sy, sz), shape)) for x in range(0, shape[0], 4)] + [src]
    pulse = make_pulse("ricker", wl.f0, 1.2 / wl.f0)
    run = run_leapfrog(a, dt, 200, source_vec=vec, source_fn=pulse, record_idx=rec, record_every=1)
    av = a @ np.random.default_rng(3).standard_normal(a.shape[0])
    np.savez_compressed(os.path.join(HERE, "golden_fdtd.npz"), c_field=wl.c_field, lam=lam, dt=dt, src=src,
                        rec=np.array(rec), samples=run.samples, times=run.times, u_curr=run.u_curr,
                        u_prev=run.u_prev, av=av)
    print("golden_fdtd.npz", lam, dt, run.samples.shape)


def golden_ntd():
    """Reference ntd_tridiag / ntd_chain of the config-1 and m9k8 golden models over a frequency band."""
    from sfwave.ntd import ntd_chain, ntd_tridiag
    out = {}
    for tag, name in (("c1", "golden_c1.npz"), ("m9", "golden_m9k8.npz")):
        g = np.load(os.path.join(HERE, name))
        omegas = np.geomspace(20.0, 400.0, 5)
        tri = np.stack([[ntd_tridiag(list(g["tdiag"][i]), list(g["toff"][i]), g["entry"][i], w) for w in omegas]
                        for i in range(len(g["tdiag"]))])
        chn = np.stack([[ntd_chain(g["gammas"][i], g["hats"][i], w) for w in omegas] for i in range(len(g["gammas"]))])
        out[tag + "_omegas"] = omegas
        out[tag + "_tridiag"] = tri
        out[tag + "_chain"] = chn
        print(tag, "tridiag vs chain", float(np.max(np.abs(tri - chn)) / np.max(np.abs(tri))))
    np.savez_compressed(os.path.join(HERE, "golden_ntd.npz"), **out)


def golden_ntd_full():
    """Reference ntd_full / ntd_reduced / band_error (ntd.py:62-115, 188-202) on one config-1
    subdomain (N = 4913, w = 24): the face inputs F, the projected pair, and the maps."""
    from sfwave.ntd import band_error, ntd_full, ntd_reduced
    from sfwave.rom import build_krylov_basis, project_reduced, subdomain_inputs
    wl = make_workload(1)
    spec = DomainSpec(tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing)), wl.counts, wl.p)
    part = build_partition(spec)
    alpha = (0, 0, 0)
    op = assemble_subdomain_operator(part, alpha, wl.c_field)
    f_in = subdomain_inputs(op, wl.modes_per_face)
    basis, _ = build_krylov_basis(op.matrix, f_in, wl.n, wl.shift)
    a_t, f_t = project_reduced(basis, op.matrix, f_in)
    omegas = np.geomspace(20.0, 400.0, 5)
    full = np.stack([ntd_full(op.matrix, f_in, w) for w in omegas])
    red = np.stack([ntd_reduced(a_t, f_t, w) for w in omegas])
    out = {"alpha": np.array(alpha), "f": f_in, "omegas": omegas, "full": full, "a_tilde": a_t, "f_tilde": f_t,
           "reduced": red, "band_error": band_error(op.matrix, f_in, a_t, f_t, omegas)}
    print("ntd_full golden: band_error", out["band_error"])
    # the verification sweep of sim.verify_subdomain (sim.py:703-768) on the same subdomain,
    # band = source_band (SOURCE_BAND x 2 pi f0, 12 frequencies), depths 1..3
    from sfwave.ntd import frequency_band, ntd_chain, ntd_tridiag
    from sfwave.rom import block_lanczos
    w_peak = 2.0 * math.pi * wl.f0
    band = frequency_band(0.4 * w_peak, 1.6 * w_peak, 12)
    rows = []
    for n in range(1, 4):
        bas, sizes = build_krylov_basis(op.matrix, f_in, n, wl.shift)
        keep = 0
        for size in sizes:
            if size != f_in.shape[1]:
                break
            keep += 1
        at, ft = project_reduced(bas[:, :keep * f_in.shape[1]], op.matrix, f_in)
        rows.append(band_error(op.matrix, f_in, at, ft, band))
    model = build_subdomain_model(op, wl.modes_per_face, 3, wl.shift)
    chain = block_lanczos(at, ft)
    poles = np.sqrt(np.maximum(-np.linalg.eigvalsh(at), 0.0))
    probe = sorted(band, key=lambda w: -float(np.min(np.abs(poles - w)) / w))
    agreement = 0.0
    for w in probe[:max(1, len(band) // 4)]:
        base = ntd_reduced(at, ft, w)
        scale = max(float(np.linalg.norm(base)), 1e-300)
        tri = ntd_tridiag(chain.diag_blocks, chain.off_blocks, chain.entry_block, w)
        chn = ntd_chain(model.gammas, model.gamma_hats, w)
        agreement = max(agreement, float(np.linalg.norm(tri - base)) / scale, float(np.linalg.norm(chn - base)) / scale)
    out.update({"verify_band": band, "verify_rows": np.array(rows), "verify_agreement": agreement})
    print("verify rows", rows, "agreement", agreement)
    np.savez_compressed(os.path.join(HERE, "golden_ntd_full.npz"), **out)


_POOL_CTX: dict = {}


def _pool_build(alpha):
    """Worker: reference build of one subdomain of the partition in _POOL_CTX (fork start)."""
    part, c_field, m, n, shift = (_POOL_CTX[k] for k in ("part", "c", "m", "n", "shift"))
    op = assemble_subdomain_operator(part, alpha, c_field)
    md = build_subdomain_model(op, m, n, shift)
    td, to, en = chain_blocks(op, m, n, shift, md.layers)
    return alpha, md, td, to


def _reference_models(wl, alphas, workers):
    """Reference build_subdomain_model of ``alphas`` with a fork process pool (one BLAS thread each)."""
    import multiprocessing as mp
    spec = DomainSpec(tuple((g - 1) * h for g, h in zip(wl.global_shape, wl.spacing)), wl.counts, wl.p)
    part = build_partition(spec)
    _POOL_CTX.update(part=part, c=wl.c_field, m=wl.modes_per_face, n=wl.n, shift=wl.shift)
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_pool_build, sorted(alphas), chunksize=2)
    models = {a: md for a, md, _, _ in res}
    blocks = {a: (td, to) for a, _, td, to in res}
    return part, models, blocks


def golden_c2(workers=8):
    """Config 2 at FULL size through the real reference: every one of the 512 m4k6 models
    (shift 8883, the 5000 m/s inclusion cutting interfaces), the reference CFL estimate and
    1000 leapfrog steps recorded on the bench probes (64 z-midplane faces x 4 modes + 8 node
    receivers).  Stored: lambda, dt, source/probe vectors, the full trace table, and the
    coefficients (A_j, B_j, Gamma_j, Gamma-hat_j, scales) of every subdomain the inclusion
    touches plus the source and receiver subdomains (the full stacks would be 80 MB)."""
    import time as _t
    wl = make_workload(2)
    t0 = _t.perf_counter()
    alphas = [(i, j, k) for i in range(8) for j in range(8) for k in range(8)]
    part, models, blocks = _reference_models(wl, alphas, workers)
    print("c2 build", _t.perf_counter() - t0)
    lam, conv = cfl_estimate_coupled(models)
    dt = 0.9 * 2.0 / math.sqrt(lam)
    print("c2 cfl", lam, conv, _t.perf_counter() - t0)
    src_alpha, src_row = locate(wl.sources[0], wl.counts, wl.p)
    pulse = make_pulse("ricker", wl.f0, 1.2 / wl.f0)
    vec = project_source(models[src_alpha], src_row, 1.0)
    probes = []
    for alpha, face in wl.face_receivers:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[alpha].state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append(Probe(alpha, wts))
    node = [locate(ijk, wl.counts, wl.p) for ijk in wl.node_receivers]
    node_w = [make_probe(models[a], r).weights for a, r in node]
    probes += [Probe(a, wv) for (a, _), wv in zip(node, node_w)]
    with CoupledStepper(models, dt, sources=(SourceTerm(src_alpha, vec, pulse),)) as st:
        times, rows = st.run(wl.n_steps, probes=probes)
        msg = st.message_count
        energy = st.energy()
    print("c2 run", _t.perf_counter() - t0)
    cut = np.argwhere(wl.c_field == 5000.0)
    lo, hi = cut.min(0), cut.max(0)
    keep = set()
    for a in alphas:  # subdomains whose node box meets the inclusion box
        if all(16 * a[d] <= hi[d] and 16 * (a[d] + 1) >= lo[d] for d in range(3)):
            keep.add(a)
    keep |= {src_alpha} | {a for a, _ in node}
    keep = sorted(keep)
    out = {"counts": np.array(wl.counts), "m": wl.modes_per_face, "n": wl.n, "shift": wl.shift,
           "n_steps": wl.n_steps, "f0": wl.f0, "lam": lam, "conv": conv, "dt": dt,
           "src_alpha": np.array(src_alpha), "src_row": src_row, "src_vec": vec,
           "node_probe_w": np.stack(node_w), "times": times, "rows": rows, "message_count": msg,
           "energy": energy, "sub_alphas": np.array(keep),
           "sub_tdiag": np.stack([blocks[a][0] for a in keep]),
           "sub_toff": np.stack([blocks[a][1] for a in keep]),
           "sub_gammas": np.stack([models[a].gammas for a in keep]),
           "sub_hats": np.stack([models[a].gamma_hats for a in keep]),
           "sub_scales": np.stack([models[a].scales for a in keep])}
    np.savez_compressed(os.path.join(HERE, "golden_c2.npz"), **out)
    print("golden_c2.npz", len(keep), "subdomains stored; lam", lam, "rows", rows.shape)


def c5_golden_alphas(wl):
    """Config-5 subdomains pinned to the reference: corner, edge, face, interior, the source
    subdomain, and the two subdomains with the most 5500 m/s inclusion nodes that are cut
    (inclusion and background both present)."""
    cz = wl.c_field
    src_alpha, _ = locate(wl.sources[0], wl.counts, wl.p)
    C = wl.counts
    fixed = [(0, 0, 0), (C[0] - 1, 0, C[2] - 1), (0, 5, 7), (17, 9, 6), src_alpha]
    score = []
    for i in range(C[0]):
        for j in range(C[1]):
            for k in range(C[2]):
                blk = cz[16 * i:16 * i + 17, 16 * j:16 * j + 17, 16 * k:16 * k + 17]
                nin = int(np.count_nonzero(blk == 5500.0))
                if 0 < nin < blk.size:
                    score.append((min(nin, blk.size - nin), (i, j, k)))
    score.sort(reverse=True)
    cut = [a for _, a in score if a not in fixed][:2]
    return fixed + cut


def golden_c5(workers=8):
    """Config-5 recipe subdomains (m=9, k=8, shift (2 pi 10)^2, 4^3-cell blocky medium with
    5500 m/s inclusions) built by the real reference on the FULL 513x513x257 config-5 field.
    Stored per subdomain: the 17^3 c slice (the full field is 540 MB; tests regenerate it from
    the seed and check these slices), the neighbour mask, A_j, B_j, Gamma_j, Gamma-hat_j, scales."""
    wl = make_workload(5)
    alphas = c5_golden_alphas(wl)
    part, models, blocks = _reference_models(wl, alphas, workers)
    out = {"counts": np.array(wl.counts), "m": 9, "n": 8, "shift": wl.shift, "alphas": np.array(alphas),
           "c_slices": np.stack([wl.c_field[16 * a[0]:16 * a[0] + 17, 16 * a[1]:16 * a[1] + 17,
                                            16 * a[2]:16 * a[2] + 17] for a in alphas]),
           "tdiag": np.stack([blocks[a][0] for a in alphas]),
           "toff": np.stack([blocks[a][1] for a in alphas]),
           "gammas": np.stack([models[a].gammas for a in alphas]),
           "hats": np.stack([models[a].gamma_hats for a in alphas]),
           "scales": np.stack([models[a].scales for a in alphas]),
           "layers": np.array([models[a].layers for a in alphas])}
    np.savez_compressed(os.path.join(HERE, "golden_c5.npz"), **out)
    print("golden_c5.npz", alphas)


def golden_states():
    """Reference project_state / state_to_nodes (rom.py:437-459) on one config-1 subdomain model,
    and the reference's interface masses (stepper.py:204-210) of the config-1 tiling."""
    from sfwave.rom import project_state, state_to_nodes
    wl = make_workload(1)
    part, ops, models = workload_models(wl)
    a = (1, 0, 1)
    md = models[a]
    rng = np.random.default_rng(21)
    x = rng.standard_normal(md.basis.shape[0])
    u = rng.standard_normal(md.state_size)
    with CoupledStepper(models, 1e-4) as st:
        masses = np.stack([i.mass for i in st.interfaces])
        pairs = np.array([[*i.low, i.low_face, *i.high, i.high_face] for i in st.interfaces])
    np.savez_compressed(os.path.join(HERE, "golden_states.npz"), alpha=np.array(a), x=x, u=u,
                        projected=project_state(md, x), nodes=state_to_nodes(md, u), masses=masses, pairs=pairs)
    print("golden_states.npz", masses.shape)


if __name__ == "__main__":
    which = sys.argv[1:] or ["toy", "c1", "m9k8", "io", "fdtd", "ntd"]
    if "states" in which:
        golden_states()
    if "c2" in which:
        golden_c2()
    if "c5" in which:
        golden_c5()
    if "toy" in which:
        golden_toy()
    if "c1" in which:
        golden_config(1, None, 200, "golden_c1.npz")
    if "m9k8" in which:
        golden_m9k8()
    if "io" in which:
        golden_io()
    if "fdtd" in which:
        golden_fdtd()
    if "ntd" in which:
        golden_ntd()
    if "ntd_full" in which:
        golden_ntd_full()
