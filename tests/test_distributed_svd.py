"""Row-partitioned partial SVD (SURVEY.md 8(e), C4 shape scaled down) with the real CUDA
kernels: 2 ranks on one GPU over gloo (host-staged collectives; the ranks' kernels never wait
on each other), and 1 forced-partitioned rank over NCCL (the collectives captured as real NCCL
calls), against the single-process solve.  Each rank owns half the rows of the tall A: A_p V
is local, A^T U = sum_p A_p^T U_p is all-reduced, the U basis is built from the all-gathered
U, the Grams are all-reduced partials, the left singular vectors stay row-partitioned."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N1, N2, R, K, TOP, SEED = 3000, 512, 40, 24, 8, 20240901

pytestmark = pytest.mark.gpu


def _matrix():
    rng = np.random.default_rng(SEED)
    g1, _ = np.linalg.qr(rng.standard_normal((N1, R)))
    g2, _ = np.linalg.qr(rng.standard_normal((N2, R)))
    sig = 0.8 ** np.arange(R)
    return (g1 * sig) @ g2.T + 1e-4 * rng.standard_normal((N1, N2)) / np.sqrt(N2)


def _solve(pname, tol, comm=None, r0=0, r1=N1):
    sys.path.insert(0, ROOT)
    import paper_2505_00281_b200 as p
    pol = p.POLICY_PRESETS[pname]
    a = p.round_to(_matrix(), pol.storage)
    A = p.DenseMatrix(np.asfortranarray(a[r0:r1]), p.FpFormat.F64)
    cfg = p.IterConfig(k=K, m=8 if tol is None else 30, iter=1, basis_method=p.BasisMethod.HESS_LEFT,
                       projection="ofrr", policy=pol, seed=SEED, tol=tol, top=TOP if tol else None)
    st = p.RunStats()
    rs = p.subspace_iter_svd(A, cfg, stats=st, comm=comm, n_global=N1)
    return (np.asarray(rs.values), np.asarray(rs.residuals), rs.vectors.data[:, :TOP].copy(),
            rs.right_vectors.data[:, :TOP].copy(), st.iterations)


def _worker(rank, world, port, q, backend, pname, tol):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        from paper_2505_00281_b200.comm import Comm
        comm = Comm.world(forced=backend == "nccl")
        r0, r1 = comm.row_range(N1)
        q.put((rank, _solve(pname, tol, comm=comm, r0=r0, r1=r1)))
    except Exception as e:
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("nccl", 1)])
@pytest.mark.parametrize("pname,tol", [("full-f32", None), ("tc-f16", 2e-3), ("full-f64", 1e-9)])
def test_row_partitioned_svd_matches_single(ofrr_gpu, backend, world, pname, tol):
    single = _solve(pname, tol)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, backend, pname, tol)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
    sv = np.linalg.svd(_matrix(), compute_uv=False)
    rows = []
    for rank in range(world):
        res = out[rank]
        assert not isinstance(res, str), res
        vals, resid, U, V, its = res
        if tol is not None:
            assert its == single[4] and np.all(resid[:TOP] < tol)
        ref_err = np.abs(single[0][:TOP] - sv[:TOP]) / sv[:TOP]
        err = np.abs(vals[:TOP] - sv[:TOP]) / sv[:TOP]
        assert np.max(err) <= max(10 * np.max(ref_err), 1e-6), (err, ref_err)
        assert np.max(resid[:TOP]) <= 2 * np.max(single[1][:TOP]) + 1e-12, (resid[:TOP], single[1][:TOP])
        # right vectors replicated: equal to the single run's to the sums' rounding
        np.testing.assert_allclose(np.abs(np.sum(V * single[3], axis=0)), 1.0, atol=1e-5)
        rows.append(U)
    U = np.vstack(rows)                                  # the ranks' rows of the left vectors
    np.testing.assert_allclose(np.abs(np.sum(U * single[2], axis=0)), 1.0, atol=1e-5)
