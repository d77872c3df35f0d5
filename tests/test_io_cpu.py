"""Reference-compatible persistence: .rom, .trc, .meta.txt, cache keys.

The fixtures under tests/golden/ were written by the reference's own io.py
(tests/golden/make_golden.py::golden_io); these tests need no GPU.
"""

import os

import numpy as np
import pytest

from helpers import GOLD, load_golden, partition_for
from paper_1406_6923_b200 import DataError
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200 import io as pio


def _read(path):
    with open(path, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("tag", ["000", "100"])
def test_rom_roundtrip_is_byte_identical_to_reference(tag, tmp_path):
    src = os.path.join(GOLD, f"io_pair{tag}.rom")
    md = pio.load_model(src)
    assert md.layers == 2 and md.modes_per_face == 1 and md.basis.shape == (125, 12)
    out = tmp_path / "m.rom"
    pio.save_model(str(out), md)
    assert _read(out) == _read(src)


def test_coefficient_only_model(tmp_path):
    md = pio.load_model(os.path.join(GOLD, "io_pair000.rom"))
    out = str(tmp_path / "c.rom")
    pio.save_model(out, md, basis="none")
    full = _read(os.path.join(GOLD, "io_pair000.rom"))
    part = _read(out)
    assert full[:len(part)] == part and len(full) - len(part) == 125 * 12 * 8
    back = pio.load_model(out, with_basis=False)
    assert back.basis is None
    for name in ("gammas", "gamma_hats", "scales", "c", "mu"):
        assert np.array_equal(getattr(back, name), getattr(md, name))
    assert back.neighbors == md.neighbors and back.alpha == md.alpha
    with pytest.raises(DataError):
        pio.load_model(out, with_basis=True)


def test_model_errors(tmp_path):
    md = pio.load_model(os.path.join(GOLD, "io_pair000.rom"), with_basis=False)
    with pytest.raises(DataError):
        pio.save_model(str(tmp_path / "x.rom"), md)  # no basis
    bad = tmp_path / "bad.rom"
    bad.write_bytes(b"XXXX" + _read(os.path.join(GOLD, "io_pair000.rom"))[4:])
    with pytest.raises(DataError):
        pio.load_model(str(bad))
    trunc = tmp_path / "t.rom"
    trunc.write_bytes(_read(os.path.join(GOLD, "io_pair000.rom"))[:100])
    with pytest.raises(DataError):
        pio.load_model(str(trunc))


def test_cache_key_matches_reference():
    g = load_golden("golden_io.npz")
    part = partition_for((2, 1, 1), (5, 5, 5), (2.0, 1.0, 1.0))
    for alpha, key in (((0, 0, 0), "key_000"), ((1, 0, 0), "key_100")):
        op = pg.assemble_subdomain_operator(part, alpha, g["c_field"], with_matrix=True)
        assert pio.model_cache_key(op, 1, 2, 4.0) == str(g[key])
    op = pg.assemble_subdomain_operator(part, (0, 0, 0), g["c_field"])
    with pytest.raises(DataError):
        pio.model_cache_key(op, 1, 2, 4.0)


def test_traces_and_meta(tmp_path):
    rec = pio.read_traces(os.path.join(GOLD, "io.trc"))
    assert rec.samples.shape == (7, 3) and rec.dt == 0.00125
    out = tmp_path / "t.trc"
    pio.write_traces(str(out), rec)
    assert _read(out) == _read(os.path.join(GOLD, "io.trc"))
    assert np.allclose(rec.times, np.arange(7) * 0.00125)
    meta = pio.read_meta(os.path.join(GOLD, "io.meta.txt"))
    assert meta["steps"] == "7" and meta["tag"] == "a: b"
    out2 = tmp_path / "m.txt"
    pio.write_meta(str(out2), {"run": "golden", "dt": 0.1 + 0.2, "steps": 7, "lambda_hat": np.float64(1.0) / 3.0,
                               "tag": "a: b"})
    assert _read(out2) == _read(os.path.join(GOLD, "io.meta.txt"))
    with pytest.raises(DataError):
        pio.TraceRecord(coords=np.zeros((2, 3)), dt=0.0, samples=np.zeros((1, 2)))
