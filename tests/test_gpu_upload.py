"""Symmetric operator upload (csrc/upload.cu, ops.upload_symmetric): only the declared
triangle of the host array is read; the device operator is the symmetric matrix, bit for
bit, for every storage format, ragged sizes and block sizes; the solve through
DenseMatrix(..., uplo=) equals the one from the full array."""
import numpy as np
import pytest
import torch

import paper_2505_00281_b200 as p
from paper_2505_00281_b200 import ops

pytestmark = pytest.mark.gpu


def _host(n, fmt, uplo, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    a = (a + a.T) / 2
    a = p.round_to(a, fmt) if fmt != p.FpFormat.FP8_E4M3 else p.round_to(np.clip(a, -400, 400), fmt)
    full = torch.from_numpy(a).to(fmt.torch_dtype)
    # poison the triangle that must not be read
    g = a.copy()
    g[np.tril(np.ones((n, n), bool), -1) if uplo == "U" else np.triu(np.ones((n, n), bool), 1)] = 7.0
    garbage = torch.from_numpy(g).to(fmt.torch_dtype)
    return full, (garbage.pin_memory() if torch.cuda.is_available() else garbage)


@pytest.mark.parametrize("fmt", [p.FpFormat.BF16, p.FpFormat.F16, p.FpFormat.F32, p.FpFormat.F64,
                                 p.FpFormat.FP8_E4M3])
@pytest.mark.parametrize("uplo", ["U", "L"])
@pytest.mark.parametrize("n,block", [(1, 0), (33, 32), (517, 64), (1000, 0), (2100, 256)])
def test_upload_symmetric_bitwise(fmt, uplo, n, block):
    full, host = _host(n, fmt, uplo, seed=n + block)
    op = ops.new_operator(n, n, fmt, torch.device("cuda"))
    op.t.fill_(0)
    nbytes = ops.upload_symmetric(op, host, uplo, block_rows=block)
    torch.cuda.synchronize()
    dev = op.t[:, :n].cpu()
    assert torch.equal(dev.view(torch.uint8) if fmt == p.FpFormat.FP8_E4M3 else dev,
                       full.view(torch.uint8) if fmt == p.FpFormat.FP8_E4M3 else full)
    br = block if block > 0 else 2048
    br = max(32, (br + 31) // 32 * 32)
    expect = sum((min(n, r0 + br) - r0) * ((n - r0) if uplo == "U" else min(n, r0 + br))
                 for r0 in range(0, n, br)) * fmt.itemsize
    assert nbytes == expect
    assert nbytes <= (n * n + n * br) // 2 * fmt.itemsize + n * fmt.itemsize


def test_upload_symmetric_rejects_bad_input():
    op = ops.new_operator(64, 64, p.FpFormat.BF16, torch.device("cuda"))
    with pytest.raises(ValueError):
        ops.upload_symmetric(op, torch.zeros(64, 64, dtype=torch.float32), "U")   # wrong dtype
    with pytest.raises(ValueError):
        ops.upload_symmetric(op, torch.zeros(64, 64, dtype=torch.bfloat16), "X")
    with pytest.raises(ValueError):
        ops.upload_symmetric(op, torch.zeros(32, 64, dtype=torch.bfloat16), "U")


def test_dense_matrix_uplo_solve_matches_full():
    n, k, top = 1024, 24, 8
    lam = p.geometric_spectrum(n, top, k)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=7)
    full = A.device_operator(p.FpFormat.BF16).t[:, :n].cpu()
    poisoned = full.clone()
    poisoned[torch.from_numpy(np.tril(np.ones((n, n), bool), -1))] = 3.0
    cfg = p.IterConfig(k=k, m=4, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.TC_BF16, seed=11)
    ref = p.subspace_iter_eig(p.DenseMatrix(full, p.FpFormat.BF16), cfg)
    got = p.subspace_iter_eig(p.DenseMatrix(poisoned.pin_memory(), p.FpFormat.BF16, uplo="U"), cfg)
    np.testing.assert_array_equal(np.asarray(got.values), np.asarray(ref.values))
    np.testing.assert_array_equal(np.asarray(got.residuals), np.asarray(ref.residuals))
