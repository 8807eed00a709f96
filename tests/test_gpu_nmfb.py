"""read_nmfb_device: NMFB rows streamed through pinned chunks and converted on
the device (nenmf_convert_f64) against the host reader."""
import numpy as np
import pytest

import paper_1812_04315_b200 as nm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("chunk_bytes", [64, 8 * 1000 + 8, 64 << 20])
def test_device_load_matches_host(tmp_path, dtype, chunk_bytes):
    M = np.random.default_rng(7).standard_normal((301, 77))
    path = tmp_path / "x.nmfb"
    nm.write_nmfb(path, M)
    X = nm.read_nmfb_device(path, dtype=dtype, chunk_bytes=chunk_bytes)
    want = M if dtype == "fp64" else M.astype(np.float32)
    got = X.cpu().numpy()
    assert got.dtype == want.dtype and got.shape == want.shape
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("row0,rows", [(0, 1), (100, 57), (300, 1), (17, 284)])
def test_device_row_block(tmp_path, row0, rows):
    M = np.random.default_rng(3).random((301, 33))  # odd element counts per block
    path = tmp_path / "x.nmfb"
    nm.write_nmfb(path, M)
    X = nm.read_nmfb_device(path, dtype="fp32", row0=row0, rows=rows, chunk_bytes=1000)
    assert X.cpu().numpy().tobytes() == M[row0:row0 + rows].astype(np.float32).tobytes()


def test_device_load_rejects_non_finite_and_bad_rows(tmp_path):
    from paper_1812_04315_b200.matrix import _NMFB_HEADER
    vals = np.ones(40)
    vals[29] = np.inf
    path = tmp_path / "inf.nmfb"
    path.write_bytes(_NMFB_HEADER.pack(b"NMFB", 1, 4, 10) + vals.astype("<f8").tobytes())
    with pytest.raises(ValueError, match="non-finite"):
        nm.read_nmfb_device(path, chunk_bytes=64)
    ok = nm.read_nmfb_device(path, rows=2)  # the bad value is in row 2
    assert ok.shape == (2, 10)
    with pytest.raises(nm.DimensionError):
        nm.read_nmfb_device(path, row0=3, rows=2)


def test_factorize_from_file(tmp_path):
    """A file-fed X gives the same sketch as the in-memory X."""
    rng = np.random.default_rng(5)
    X = rng.random((400, 8)) @ rng.random((8, 300)) + 0.01 * rng.random((400, 300))
    path = tmp_path / "x.nmfb"
    nm.write_nmfb(path, X)
    Xd = nm.read_nmfb_device(path, dtype="fp64")
    a = nm.subspace_iteration_pair(Xd, 12, 2, 9)
    b = nm.subspace_iteration_pair(X, 12, 2, 9)
    # a device X gives a device-resident sketch (no host copy inside the sketch)
    from paper_1812_04315_b200 import _lib

    assert a.L.is_cuda and a.R.is_cuda
    assert np.abs(_lib.to_host(a.L) - b.L).max() == 0.0 and np.abs(_lib.to_host(a.R) - b.R).max() == 0.0


def test_load_row_shard_covers_file(tmp_path):
    from paper_1812_04315_b200 import sharded
    M = np.random.default_rng(1).random((103, 20))
    path = tmp_path / "x.nmfb"
    nm.write_nmfb(path, M)
    parts = []
    for rank in range(3):
        X, n, row0 = sharded.load_row_shard(path, 3, rank, dtype="fp64")
        assert n == 103 and row0 == sharded.row_block(103, 3, rank)[0]
        parts.append(X.cpu().numpy())
    assert np.concatenate(parts).tobytes() == M.tobytes()
