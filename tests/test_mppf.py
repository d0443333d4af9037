"""MPPF v1 frames (mppf.cpp): files written by the reference read back identically here, files
written here read back identically by the reference, and every error path of read_mppf
(checksums, CSR invariants, format) behaves like the reference's. CPU only."""
import os

import numpy as np
import pytest


def same_frame(f, r):
    assert f.n == r["n"] and f.width == r["width"] and f.height == r["height"]
    assert f.rho_heavy == r["rho_heavy"]
    np.testing.assert_array_equal(f.cell_order, r["cell_order"])
    np.testing.assert_array_equal(np.asarray(f.A.row_offsets, np.uint64), r["row_offsets"])
    np.testing.assert_array_equal(np.asarray(f.A.col_indices, np.uint32), r["col_indices"])
    assert np.array_equal(np.asarray(f.A.values).view(np.uint64), r["values"].view(np.uint64))
    assert np.array_equal(np.asarray(f.rho).view(np.uint64), r["rho"].view(np.uint64))
    assert np.array_equal(np.asarray(f.b).view(np.uint64), r["b"].view(np.uint64))


@pytest.mark.parametrize("n", [1024, 2048 + 7, 8192])
def test_reference_file_reads_here(H, ref, tmp_path, n):
    path = str(tmp_path / "ref.mppf")
    ref.write_mppf(n, 2024, 3, path)
    f = H.read_mppf(path)
    r = ref.read_mppf(path)
    same_frame(f, r)
    assert (f.master_seed, f.frame_index) == (2024, 3) == (r["master_seed"], r["frame_index"])
    assert f.barriers == r["barriers"] and len(f.barriers) >= 1


@pytest.mark.parametrize("n", [1024, 4096 + 3])
def test_file_written_here_reads_in_reference(H, ref, tmp_path, n):
    fr = H.make_frame(n, 2024, 5)
    path = str(tmp_path / "ours.mppf")
    H.write_mppf(fr, path)
    r = ref.read_mppf(path)
    same_frame(fr, r)
    assert fr.barriers == r["barriers"]
    back = H.read_mppf(path)
    same_frame(back, r)


def test_errors(H, ref, tmp_path):
    fr = H.make_frame(1024, 2024, 1)
    path = str(tmp_path / "f.mppf")
    H.write_mppf(fr, path)
    raw = bytearray(open(path, "rb").read())
    # a flipped payload byte: checksum mismatch (runtime_error)
    bad = bytearray(raw)
    bad[-9] ^= 0x40
    open(path, "wb").write(bad)
    with pytest.raises(RuntimeError, match="checksum mismatch"):
        H.read_mppf(path)
    with pytest.raises(Exception, match="checksum mismatch"):
        ref.read_mppf(path)
    # bad magic
    bad = bytearray(raw)
    bad[0] = ord("X")
    open(path, "wb").write(bad)
    with pytest.raises(RuntimeError, match="bad magic"):
        H.read_mppf(path)
    # an asymmetric matrix with valid checksums: csr validate -> invalid_argument
    A = fr.A
    v = np.array(A.values, copy=True)
    ro = np.asarray(A.row_offsets)
    i = 5
    p = int(ro[i])
    while A.col_indices[p] == i:
        p += 1
    v[p] *= 1.5
    fr2 = H.Frame(fr.n, fr.width, fr.height, fr.depth, fr.cell_order, fr.rho,
                  H.CsrMatrix(fr.n, fr.n, A.row_offsets, A.col_indices, v), fr.b, fr.rho_heavy,
                  fr.master_seed, fr.frame_index, fr.barriers)
    H.write_mppf(fr2, path)
    with pytest.raises(ValueError, match="not symmetric"):
        H.read_mppf(path)
    with pytest.raises(Exception, match="not symmetric"):
        ref.read_mppf(path)
    # 3D frames have no MPPF v1 form
    with pytest.raises(ValueError):
        H.write_mppf(H.make_frame_3d(4, 4, 4, 1, 0), path)
    os.remove(path)


def test_payload_crc_covers_length_mod_2_32():
    """checkpoint.cpp:28-30 / mppf.cpp:21-24 pass the byte length to zlib as uInt: a payload of
    2^32 + k bytes is checksummed over its first k bytes only. An anonymous mapping keeps the
    4 GiB region virtual (untouched zero pages)."""
    import ctypes
    import mmap
    import zlib

    from paper_2605_13343_b200 import _native as N
    size = (1 << 32) + 4096
    m = mmap.mmap(-1, size)
    try:
        m[:4096] = bytes(range(256)) * 16
        m[size - 8:] = b"tailtail"  # beyond 2^32: not covered, like the reference
        base = ctypes.addressof(ctypes.c_char.from_buffer(m))
        out = ctypes.c_uint32()
        N.check(N.lib.hfpg_payload_crc32(base, size, ctypes.byref(out)))
        assert out.value == zlib.crc32(m[:4096])
        N.check(N.lib.hfpg_payload_crc32(base, 4096, ctypes.byref(out)))
        assert out.value == zlib.crc32(m[:4096])
        del base
    finally:
        try:
            m.close()
        except BufferError:
            pass
