"""On-disk formats on the device: the GPU crc32 is zlib's, MPPF frames load
straight into device memory with GPU checksums and CSR checks (same frame and same solve as the
host path), HFTC checkpoints load straight into the factor tensor."""
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(H):
    return H.Device(0)


@pytest.mark.parametrize("size", [0, 1, 15, 16, 255, 256, 257, 4096, 65536 + 3, 256 * 256 * 3 + 77,
                                  (10 << 20) + 5])
@pytest.mark.parametrize("offset", [0, 1, 7, 13])
def test_crc32_matches_zlib(dev, size, offset):
    rng = np.random.default_rng(size * 31 + offset)
    host = rng.integers(0, 256, size + offset, dtype=np.uint8)
    d = torch.from_numpy(host).cuda()
    got = dev.crc32((d.data_ptr() + offset, size))
    want = zlib.crc32(host[offset:].tobytes())
    assert got == want, (size, offset, hex(got), hex(want))
    assert dev.crc32(host[offset:]) == want  # host path (zlib)


def test_load_mppf_equals_reference(H, ref, dev, tmp_path):
    path = str(tmp_path / "f.mppf")
    ref.write_mppf(65536, 2024, 2, path)
    g = dev.load_mppf(path)
    r = ref.read_mppf(path)
    f = g.to_host()
    np.testing.assert_array_equal(f.cell_order, r["cell_order"])
    np.testing.assert_array_equal(np.asarray(f.A.row_offsets, np.uint64), r["row_offsets"])
    np.testing.assert_array_equal(np.asarray(f.A.col_indices, np.uint32), r["col_indices"])
    assert np.array_equal(np.asarray(f.A.values).view(np.uint64), r["values"].view(np.uint64))
    assert np.array_equal(np.asarray(f.b).view(np.uint64), r["b"].view(np.uint64))
    # the loaded system solves exactly like the same CSR loaded through the host path
    cfg = H.SolveConfig()
    dev.set_precond(1)
    x1 = np.empty(f.n)
    rep1 = dev.solve_ptr(f.b.ctypes.data, x1.ctypes.data, cfg, None, 0)
    d2 = H.Device(0)
    d2.load_csr(f.A)
    d2.set_precond(1)
    x2 = np.empty(f.n)
    rep2 = d2.solve_ptr(f.b.ctypes.data, x2.ctypes.data, cfg, None, 0)
    assert rep1.iterations == rep2.iterations and rep1.converged
    assert np.array_equal(x1, x2)


def test_load_mppf_errors(H, dev, tmp_path):
    fr = H.make_frame(4096, 2024, 1)
    path = str(tmp_path / "f.mppf")
    H.write_mppf(fr, path)
    raw = bytearray(open(path, "rb").read())
    bad = bytearray(raw)
    bad[-100] ^= 1
    open(path, "wb").write(bad)
    with pytest.raises(RuntimeError, match="checksum mismatch"):
        dev.load_mppf(path)
    A = fr.A
    v = np.array(A.values, copy=True)
    ro = np.asarray(A.row_offsets)
    p = int(ro[7])
    while A.col_indices[p] == 7:
        p += 1
    v[p] += 1.0
    fr2 = H.Frame(fr.n, fr.width, fr.height, fr.depth, fr.cell_order, fr.rho,
                  H.CsrMatrix(fr.n, fr.n, A.row_offsets, A.col_indices, v), fr.b, fr.rho_heavy,
                  fr.master_seed, fr.frame_index, fr.barriers)
    H.write_mppf(fr2, path)
    with pytest.raises(ValueError, match="not symmetric"):
        dev.load_mppf(path)
    H.write_mppf(fr, path)  # and a good file loads after the failures
    g = dev.load_mppf(path)
    assert g.n == 4096


def test_load_checkpoint(H, tmp_path):
    fr = H.make_frame(65536, 2024, 0)
    f = H.init_factors(H.build_partition(fr.n, 128), 32, H.FactorInit.jacobi_seed, 1e-2,
                       H.RngStream(2024, 0, H.RngPurpose.factor_init))
    path = str(tmp_path / "m.hftc")
    H.write_checkpoint(f, path)
    d1 = H.Device(0)
    d1.load_csr(fr.A)
    d1.load_checkpoint(path)
    d2 = H.Device(0)
    d2.load_csr(fr.A)
    d2.load_factors(H.read_checkpoint(path).factors)
    assert np.array_equal(d1.apply(fr.b), d2.apply(fr.b))
    raw = bytearray(open(path, "rb").read())
    raw[-5] ^= 2
    open(path, "wb").write(raw)
    with pytest.raises(RuntimeError, match="checksum mismatch"):
        d1.load_checkpoint(path)
