"""CPU-side checks: the C-ABI library loads and exports its header, host bookkeeping
mirrors the reference/oracle, and the product path fails loudly without a GPU."""

import os
import re

import numpy as np
import pytest

from helpers import load_golden, models_from_arrays, partition_for
from oracle import sfw_oracle as so
from paper_1406_6923_b200 import (ConfigError, CoupledStepper, DeviceError, ProtocolError, _lib, grid,
                                  project_source)
from paper_1406_6923_b200.configs import locate, make_workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = _lib.load(require_device=False)
    hdr = open(os.path.join(ROOT, "include", "sfw_b200.h")).read()
    names = set(re.findall(r"^\s*(?:int|const char\*)\s+(sfw_\w+)\s*\(", hdr, flags=re.M))
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert set(_lib.SIGNATURES) == names  # nothing bound that the header does not declare


@pytest.mark.parametrize("cname,pytype", [("sfw_step_desc", "StepDesc"), ("sfw_rom_desc", "RomDesc"),
                                          ("sfw_rom_out", "RomOut")])
def test_ctypes_structs_match_header(cname, pytype):
    """The ctypes mirrors declare the header's struct fields, in order."""
    hdr = open(os.path.join(ROOT, "include", "sfw_b200.h")).read()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), hdr, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.split(","):
            fields.append(re.sub(r"\[.*\]", "", part).replace("*", " ").split()[-1])
    assert fields == [f[0] for f in getattr(_lib, pytype)._fields_]


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


@pytest.mark.parametrize("mask", range(64))
def test_face_windows_match_oracle(mask):
    nbr = {f: None for f in range(6) if (mask >> f) & 1}
    for shape in [(17, 17, 17), (5, 6, 7)]:
        for f in range(6):
            mine = grid.face_window(shape, f, nbr)
            idx, ps = so.face_window(shape, f, nbr)
            assert np.array_equal(mine.indices, idx)
            assert tuple(mine.plane_shape) == tuple(ps)


def test_operator_matches_oracle_and_golden():
    g = load_golden("golden_toy.npz")
    part = partition_for((2, 1, 1), (5, 5, 5), (2.0, 1.0, 1.0))
    op = grid.assemble_subdomain_operator(part, (0, 0, 0), g["pair_c_field"], with_matrix=True)
    assert np.allclose(op.matrix.toarray(), g["pair_matrix0"], rtol=0, atol=1e-13)
    oop = so.make_subops((2, 1, 1), (5, 5, 5), (0.25, 0.25, 0.25), g["pair_c_field"])[(0, 0, 0)]
    assert np.array_equal(op.mu, oop.mu) and np.array_equal(op.c, oop.c)


def test_kronecker_factorisation_of_the_operator():
    """A = -C (X_x (+) X_y (+) X_z) C: the identity the GPU solver relies on (csrc/sfw_rom.cu)."""
    wl = make_workload(3, counts=(3, 3, 3))
    ext = tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing))
    part = grid.build_partition(grid.DomainSpec(ext, wl.counts, wl.p))
    op = grid.assemble_subdomain_operator(part, (1, 0, 2), wl.c_field, with_matrix=True)
    P, h = 17, 10.0

    def X1(lo, hi):
        L1 = np.diag(np.r_[1.0, 2.0 * np.ones(P - 2), 1.0]) - np.eye(P, k=1) - np.eye(P, k=-1)
        s = np.ones(P)
        s[0] = np.sqrt(2) if lo else 1
        s[-1] = np.sqrt(2) if hi else 1
        return (s[:, None] * L1 * s[None, :]) / h ** 2
    Xs = [X1((2 * a) in op.neighbors, (2 * a + 1) in op.neighbors) for a in range(3)]
    I = np.eye(P)
    S = np.kron(np.kron(Xs[0], I), I) + np.kron(np.kron(I, Xs[1]), I) + np.kron(np.kron(I, I), Xs[2])
    A = -(op.c[:, None] * S * op.c[None, :])
    Ad = op.matrix.toarray()
    assert np.abs(A - Ad).max() <= 1e-14 * np.abs(Ad).max()


def test_configs_are_seeded_and_sources_interior():
    for cfg in (1, 2, 3, 5):
        a = make_workload(cfg, counts=(2, 2, 2))
        b = make_workload(cfg, counts=(2, 2, 2))
        assert np.array_equal(a.c_field, b.c_field)
        assert a.c_field.min() >= 1500 and a.c_field.max() <= 5500
    wl = make_workload(4, counts=(2, 2, 2))
    assert len(wl.sources) == 32
    for ijk in wl.sources:
        assert all(x % 16 != 0 for x in ijk)
    wl = make_workload(2)
    alpha, row = locate(wl.sources[0], wl.counts, wl.p)
    assert alpha == (3, 3, 3)
    assert np.unravel_index(row, wl.p) == (15, 15, 15)


def test_protocol_and_config_errors_before_any_device_work():
    g = load_golden("golden_toy.npz")
    part = partition_for((2, 1, 1), (5, 5, 5), (2.0, 1.0, 1.0))
    models = models_from_arrays(part, g["pair_c_field"], 1, g["pair_gammas"], g["pair_hats"], g["pair_scales"])
    order = sorted(models)
    with pytest.raises(ConfigError):
        CoupledStepper(models, -1.0)
    with pytest.raises(ProtocolError):
        CoupledStepper({order[0]: models[order[0]]}, 0.01)


def test_product_path_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    g = load_golden("golden_toy.npz")
    part = partition_for((2, 1, 1), (5, 5, 5), (2.0, 1.0, 1.0))
    models = models_from_arrays(part, g["pair_c_field"], 1, g["pair_gammas"], g["pair_hats"], g["pair_scales"],
                                basis=g["pair_basis"])
    with pytest.raises(DeviceError):
        CoupledStepper(models, 0.01)
    with pytest.raises(DeviceError):
        project_source(models[sorted(models)[0]], 31)


def test_growth_limits_match_the_scalar_loop():
    """CoupledStepper._limits (vectorised) == the reference's per-step baseline loop (stepper.py:379-389)."""
    import types

    from paper_1406_6923_b200.stepper import GROWTH_LIMIT, CoupledStepper
    rng = np.random.default_rng(4)
    for n_src, n in ((1, 500), (3, 77), (0, 5)):
        fake = types.SimpleNamespace(dt=0.0013, sources=[object()] * n_src, _baseline=float(rng.random()))
        prof = rng.standard_normal((n_src, n)) if n_src else None
        norms = rng.random(n_src) * 3
        lim, base = CoupledStepper._limits(fake, prof, norms, n)
        b = fake._baseline
        ref = []
        for k in range(n):
            for i in range(n_src):
                b += fake.dt * fake.dt * abs(float(prof[i, k])) * norms[i]
            ref.append(GROWTH_LIMIT * max(b, 1e-300))
        assert np.array_equal(lim, np.array(ref)) and base == b


@pytest.mark.parametrize("name", ["ricker", "gauss_deriv"])
def test_library_pulse_table_is_bit_identical_to_the_callable(name):
    """sfw_pulse_table (host code in the library) equals per-step Python evaluation of
    pulses.py bit for bit, so long runs may tabulate f(t_k) in the library."""
    from paper_1406_6923_b200.pulses import PULSES
    from paper_1406_6923_b200.stepper import profile_table
    rng = np.random.default_rng(5)
    for _ in range(6):
        f0 = float(rng.uniform(2.0, 40.0))
        delay = 1.2 / f0
        dt = float(rng.uniform(1e-4, 3e-3))
        k0 = int(rng.integers(0, 5000))
        n = 20000
        p = PULSES[name](f0, delay)
        tab = profile_table([p], k0, n, dt, _lib.load(require_device=False))[0]
        ref = np.array([p((k0 + k) * dt) for k in range(n)])
        assert np.array_equal(tab, ref)
    # any other callable goes through the per-step path
    g = lambda t: 2.0 * t  # noqa: E731
    assert np.array_equal(profile_table([g], 3, 5, 0.5)[0], [2.0 * (3 + k) * 0.5 for k in range(5)])


def test_resolve_dt_policy():
    """sim.py:444-463 _resolve_dt semantics."""
    from paper_1406_6923_b200 import resolve_dt
    from paper_1406_6923_b200.stepper import _resolve_dt
    assert resolve_dt("auto", 2.0, True, 1.0) == 0.9 * 2.0
    assert resolve_dt("auto", 2.0, False, 1.0) == 0.9 * 1.0
    assert resolve_dt("fine", 2.0, True, 1.0) == 0.9 * 1.0
    assert resolve_dt(1.8, 2.0, True, 1.0) == 1.8
    assert resolve_dt(1.8 * (1 + 5e-13), 2.0, True, 1.0) == 1.8 * (1 + 5e-13)
    with pytest.raises(ConfigError) as ei:
        resolve_dt(1.81, 2.0, True, 1.0)
    assert ei.value.path == "time.dt"

    class Cfg:
        dt = "auto"
    assert _resolve_dt(Cfg, 2.0, True, 1.0) == 0.9 * 2.0


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree absent (GPU box)")
def test_public_signatures_match_reference():
    """Every name we re-export that the reference also exports keeps the reference's parameters
    (names, kinds, defaults, in order); ours may only append optional ones."""
    import importlib
    import inspect
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        ref = importlib.import_module("sfwave")
        ref_mods = {m: importlib.import_module("sfwave." + m) for m in ("rom", "stepper", "grid", "io", "reference")}
    finally:
        sys.path.remove(REF_SRC)
    import paper_1406_6923_b200 as ours
    from paper_1406_6923_b200 import rom, stepper
    pairs = [(n, getattr(ours, n), getattr(ref, n)) for n in ours.__all__ if hasattr(ref, n)]
    pairs += [(n, getattr(rom, n), getattr(ref_mods["rom"], n)) for n in ("project_state", "state_to_nodes")]
    pairs += [(n, getattr(stepper, n), getattr(ref_mods["stepper"], n))
              for n in ("project_source", "make_probe", "cfl_estimate_coupled", "stable_step_coupled",
                        "chain_operator")]
    checked = 0
    for name, mine, theirs in pairs:
        if not callable(theirs):
            continue
        try:
            ps = list(inspect.signature(theirs).parameters.values())
        except (TypeError, ValueError):
            continue
        mp = list(inspect.signature(mine).parameters.values())
        assert len(mp) >= len(ps), name
        for a, b in zip(ps, mp):
            assert (a.name, a.kind) == (b.name, b.kind), (name, a, b)
            assert a.default is inspect.Parameter.empty or a.default == b.default, (name, a, b)
        for extra in mp[len(ps):]:
            assert extra.default is not inspect.Parameter.empty or extra.kind == extra.VAR_KEYWORD, (name, extra)
        checked += 1
    methods = ["initialize", "advance", "run", "energy", "close"]
    for meth in methods:
        ps = list(inspect.signature(getattr(ref.CoupledStepper, meth)).parameters.values())
        mp = list(inspect.signature(getattr(ours.CoupledStepper, meth)).parameters.values())
        for a, b in zip(ps, mp):
            assert (a.name, a.kind, a.default) == (b.name, b.kind, b.default), (meth, a, b)
    assert checked >= 10, checked
