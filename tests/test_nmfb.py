"""NMFB file IO (matrix.py:180-214) and sketch save/load (compression.py:191-210):
the reference's format tests (test_matrix.py:147-190) restated against this
package, plus a byte-level check against the reference's own writer."""
import importlib
import struct

import numpy as np
import pytest

import paper_1812_04315_b200 as nm
from paper_1812_04315_b200.matrix import _NMFB_HEADER


def _M(rows, cols, seed):
    return np.random.default_rng(seed).standard_normal((rows, cols))


def test_round_trip_bit_exact(tmp_path):
    M = _M(13, 7, 5)
    path = tmp_path / "m.nmfb"
    nm.write_nmfb(path, M)
    back = nm.read_nmfb(path)
    assert back.shape == M.shape and back.dtype == np.float64
    assert M.tobytes() == back.tobytes()


def test_layout_is_header_then_le_f64_row_major(tmp_path):
    M = _M(3, 4, 1)
    path = tmp_path / "m.nmfb"
    nm.write_nmfb(path, M)
    raw = path.read_bytes()
    assert raw[:24] == struct.pack("<4sIQQ", b"NMFB", 1, 3, 4)
    assert raw[24:] == M.astype("<f8").tobytes()


def test_rewrite_is_byte_identical(tmp_path):
    M = _M(6, 6, 8)
    a, b = tmp_path / "a.nmfb", tmp_path / "b.nmfb"
    nm.write_nmfb(a, M)
    nm.write_nmfb(b, M)
    assert a.read_bytes() == b.read_bytes()


def _corrupt(tmp_path, edit):
    path = tmp_path / "bad.nmfb"
    nm.write_nmfb(path, np.ones((2, 2)))
    raw = bytearray(path.read_bytes())
    path.write_bytes(bytes(edit(raw)))
    return path


def test_bad_magic(tmp_path):
    def edit(raw):
        raw[:4] = b"XXXX"
        return raw
    with pytest.raises(ValueError, match="magic"):
        nm.read_nmfb(_corrupt(tmp_path, edit))


def test_bad_version(tmp_path):
    def edit(raw):
        raw[4:8] = struct.pack("<I", 2)
        return raw
    with pytest.raises(ValueError, match="version"):
        nm.read_nmfb(_corrupt(tmp_path, edit))


def test_truncated_payload_and_header(tmp_path):
    with pytest.raises(ValueError, match="expected"):
        nm.read_nmfb(_corrupt(tmp_path, lambda raw: raw[:-8]))
    with pytest.raises(ValueError, match="truncated"):
        nm.read_nmfb(_corrupt(tmp_path, lambda raw: raw[:10]))


def test_degenerate_dimensions(tmp_path):
    path = tmp_path / "z.nmfb"
    path.write_bytes(_NMFB_HEADER.pack(b"NMFB", 1, 0, 3))
    with pytest.raises(nm.DimensionError):
        nm.read_nmfb(path)


def test_non_finite_rejected(tmp_path):
    M = np.ones((2, 3))
    M[1, 2] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        nm.write_nmfb(tmp_path / "n.nmfb", M)
    path = tmp_path / "inf.nmfb"
    path.write_bytes(_NMFB_HEADER.pack(b"NMFB", 1, 1, 2) + np.array([1.0, np.inf]).astype("<f8").tobytes())
    with pytest.raises(ValueError, match="non-finite"):
        nm.read_nmfb(path)


def test_sketch_save_load(tmp_path):
    L, R = _M(4, 30, 2), _M(25, 4, 3)
    sk = nm.SketchPair(L=L, R=R, nu=4, scheme="subspace_iteration", q=3, seed=11)
    nm.save_sketch(sk, tmp_path / "sk")
    back = nm.load_sketch(tmp_path / "sk")
    assert back.L.tobytes() == L.tobytes() and back.R.tobytes() == R.tobytes()
    assert (back.nu, back.scheme, back.q, back.seed) == (4, "subspace_iteration", 3, 11)


def test_same_bytes_as_reference_writer(tmp_path):
    """The reference's own write_nmfb (importable in this container) writes the
    same bytes; skipped where /root/reference is absent (the GPU box)."""
    import sys
    from pathlib import Path
    src = Path("/root/reference/pkg/src")
    if not src.is_dir():
        pytest.skip("reference not present")
    sys.path.insert(0, str(src))
    try:
        spec = importlib.util.find_spec("nenmf.matrix")
        if spec is None:
            pytest.skip("reference not importable")
        ref = importlib.import_module("nenmf.matrix")
    finally:
        sys.path.remove(str(src))
    M = _M(9, 5, 4)
    a, b = tmp_path / "a.nmfb", tmp_path / "b.nmfb"
    nm.write_nmfb(a, M)
    ref.write_nmfb(b, M)
    assert a.read_bytes() == b.read_bytes()
    assert ref.read_nmfb(a).tobytes() == M.tobytes()



def test_trace_csv_round_trip_and_header(tmp_path):
    """tracing.py:85-119: 17 significant digits round-trip every double."""
    recs = [nm.TraceRecord(outer_iter=i, solver_elapsed_s=0.1 * i + 1e-17, wall_elapsed_s=np.pi * i,
                           rre=1.0 / (i + 3), objective=2.0 ** -40 * i) for i in range(5)]
    path = tmp_path / "t.csv"
    nm.write_trace_csv(recs, path)
    assert nm.read_trace_csv(path) == recs
    assert path.read_text().splitlines()[0] == ",".join(nm.TRACE_CSV_HEADER)
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(ValueError, match="header"):
        nm.read_trace_csv(bad)
