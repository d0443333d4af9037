"""IC(0) factorization (ic0.cpp:10-69) restated in libhfpg's host C++: bit-identical to the
reference's factor on 2D / 3D pressure-Poisson frames, both shift policies, and the reference's
error behaviour. CPU only (the factor is set-up work; the sweeps run on the GPU)."""
import numpy as np
import pytest

from conftest import ROOT  # noqa: F401


def csr_of(A):
    return (np.ascontiguousarray(A.row_offsets, np.uint64), np.ascontiguousarray(A.col_indices, np.uint32),
            np.ascontiguousarray(A.values, np.float64))


@pytest.mark.parametrize("frame", ["2d_8192", "3d_12x10x8"])
@pytest.mark.parametrize("policy", [0, 1])
def test_factor_bit_exact(H, ref, frame, policy):
    fr = H.make_frame(8192, 2024, 0) if frame == "2d_8192" else H.make_frame_3d(12, 10, 8, 2024, 3)
    f = H.ic0_factorize(fr.A, H.Ic0Shift(policy))
    lro, lci, lv, shift = ref.ic0_factorize(csr_of(fr.A), policy)
    assert f.shift == shift
    np.testing.assert_array_equal(np.asarray(f.lower.row_offsets, np.uint64), lro)
    np.testing.assert_array_equal(np.asarray(f.lower.col_indices, np.uint32), lci)
    assert np.array_equal(np.asarray(f.lower.values).view(np.uint64), lv.view(np.uint64))
    # pattern: lower triangle of A, diagonal last (ic0.cpp:21-37)
    ro = np.asarray(f.lower.row_offsets)
    assert all(f.lower.col_indices[ro[i + 1] - 1] == i for i in range(fr.n))


def test_missing_diagonal_and_errors(H, ref):
    # a structurally missing diagonal is a zero entry -> nonpositive pivot (runtime_error)
    A = H.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    with pytest.raises(RuntimeError):
        H.ic0_factorize(A, H.Ic0Shift.none)
    with pytest.raises(Exception, match="nonpositive pivot"):  # the shim reports runtime_error as code 2
        ref.ic0_factorize(csr_of(A), 0)
    # indefinite: [[1, 2], [2, 1]]
    B = H.CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 2.0, 2.0, 1.0]))
    with pytest.raises(RuntimeError):
        H.ic0_factorize(B)
    with pytest.raises(ValueError):
        H.ic0_factorize(H.CsrMatrix(2, 3, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0])))
    # SPD 1x1 with the scaled shift: sqrt(a + 1e-8 a)
    C = H.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([4.0]))
    f = H.ic0_factorize(C)
    assert f.shift == 4e-8 and f.lower.values[0] == np.sqrt(4.0 + 4e-8)
