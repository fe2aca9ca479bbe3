"""Row-partitioned multi-process OFRR on CPU: world_size 2, gloo.

Each rank owns half the rows of A; the driver's collectives (all-gather of the n x k
block, all-reduce(max) of the column inf-norms, all-reduce(sum) of the partial Grams and
residual sums of squares, all-reduce(max) of the status words) run over torch.distributed
(gloo here, NCCL on the GPU box).  The per-op arithmetic is the test-only oracle backend
(tests/cpu_ops.py), so the single-process and the 2-rank runs must agree to the rounding
of the Gram all-reduce.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, TOP, K, M, SEED = 160, 6, 12, 4, 20240901


def _problem():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as o
    a, _ = o.geometric_symmetric(N, TOP, K, seed=SEED, fmt=o.F32)
    return a


CASES = ((None, False), (1e-4, False), (None, True), (1e-4, True))   # (tol, reuse_av)


def _run(a_rows, n, comm, tol=None, reuse=False):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cpu_ops
    import paper_2505_00281_b200 as p
    from paper_2505_00281_b200.driver import EigEngine
    cfg = p.IterConfig(k=K, m=M, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.FULL_F32, seed=SEED, tol=tol, top=TOP if tol else None, reuse_av=reuse)
    eng = EigEngine(cpu_ops.RowBlock(a_rows, p.FpFormat.F32), cfg, comm=comm, n_global=n, ops=cpu_ops)
    rs = eng.run()
    return rs.values, rs.vectors.data if hasattr(rs.vectors, "data") else None, rs.residuals, eng.stats


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        from paper_2505_00281_b200.comm import Comm
        comm = Comm.world()
        a = _problem()
        r0, r1 = comm.row_range(N)
        for tol, reuse in CASES:
            vals, _, res, st = _run(a[r0:r1], N, comm, tol=tol, reuse=reuse)
            q.put((rank, (tol, reuse), vals, res, st.iterations, st.a_passes))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_row_partitioned_matches_single_process():
    sys.path.insert(0, ROOT)
    from paper_2505_00281_b200.comm import Comm
    a = _problem()
    single = {(tol, reuse): _run(a, N, Comm(), tol=tol, reuse=reuse) for tol, reuse in CASES}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=180) for _ in range(2 * len(CASES))]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, tol, vals, res, iters, passes in out:
        v1, _, r1, st1 = single[tol]
        assert iters == st1.iterations
        assert passes == st1.a_passes
        np.testing.assert_allclose(vals, v1, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(res, r1, rtol=1e-6, atol=1e-12)
    # both ranks hold identical results (redundant pencil solve is deterministic)
    by_tol = {}
    for rank, tol, vals, res, _, _ in out:
        by_tol.setdefault(tol, []).append(vals)
    for tol, vs in by_tol.items():
        np.testing.assert_array_equal(vs[0], vs[1])


def test_reuse_av_single_process():
    """A-pass reuse (IterConfig.reuse_av): the next MatVec comes from the projection's
    W = A U (A U Y = W Y), one A pass per outer iteration after the first instead of
    iter + 1; same Ritz values as the reference's schedule to its precision."""
    sys.path.insert(0, ROOT)
    from paper_2505_00281_b200.comm import Comm
    a = _problem()
    v0, _, r0, st0 = _run(a, N, Comm(), tol=None, reuse=False)
    v1, _, r1, st1 = _run(a, N, Comm(), tol=None, reuse=True)
    assert st0.a_passes == 2 * M and st1.a_passes == M + 1
    np.testing.assert_allclose(v1[:TOP], v0[:TOP], rtol=1e-5)
    assert np.all(r1[:TOP] <= 2 * r0[:TOP] + 1e-6)


def test_comm_row_ranges():
    sys.path.insert(0, ROOT)
    from paper_2505_00281_b200.comm import Comm
    for n in (1, 7, 160, 16384):
        for P in (1, 2, 3, 8):
            rows = [Comm(r, P).row_range(n) for r in range(P)]
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(rows[i][1] == rows[i + 1][0] for i in range(P - 1))


# ---- row-partitioned partial SVD (C4's layout): 2 gloo ranks vs 1 process ----------------
N1, N2, KS, TS = 240, 60, 10, 4


def _tall():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as o
    rng = np.random.default_rng(SEED)
    g1, _ = np.linalg.qr(rng.standard_normal((N1, 20)))
    g2, _ = np.linalg.qr(rng.standard_normal((N2, 20)))
    a = (g1 * 0.8 ** np.arange(20)) @ g2.T + 1e-4 * rng.standard_normal((N1, N2))
    return o.round_to(a, o.F32)


def _svd(a_rows, comm, tol=None):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import cpu_ops
    import paper_2505_00281_b200 as p
    from paper_2505_00281_b200.driver import _subspace_iter_svd
    cfg = p.IterConfig(k=KS, m=5, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                       policy=p.FULL_F32, seed=SEED, tol=tol, top=TS if tol else None)
    st = p.RunStats()
    rs = _subspace_iter_svd(cpu_ops.RowBlock(a_rows, p.FpFormat.F32), cfg, st, comm=comm, n_global=N1, ops=cpu_ops)
    return rs.values, rs.residuals, rs.vectors.data, rs.right_vectors.data, st.iterations


def _svd_worker(rank, world, port, q, tol):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        from paper_2505_00281_b200.comm import Comm
        comm = Comm.world()
        r0, r1 = comm.row_range(N1)
        q.put((rank, _svd(_tall()[r0:r1], comm, tol)))
    except Exception as e:
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tol", [None, 1e-4])
def test_row_partitioned_svd_two_ranks_equals_one(tol):
    sys.path.insert(0, ROOT)
    from paper_2505_00281_b200.comm import Comm
    single = _svd(_tall(), Comm(), tol)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_svd_worker, args=(r, 2, port, q, tol)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    for rank in range(2):
        assert not isinstance(out[rank], str), out[rank]
        vals, res, U, V, its = out[rank]
        # A^T U is summed from the ranks' fp32 partial products (rounded once more than the
        # single run's product): agreement to fp32 rounding
        assert its == single[4]
        np.testing.assert_allclose(vals, single[0], rtol=1e-6)
        assert np.all(res <= 2 * single[1] + 1e-7) and np.all(single[1] <= 2 * res + 1e-7)
        np.testing.assert_allclose(V, single[3], atol=1e-5)
        np.testing.assert_array_equal(out[0][3], out[1][3])        # V replicated bit for bit
    U = np.vstack([out[0][2], out[1][2]])                # row-partitioned left vectors
    np.testing.assert_allclose(U, single[2], atol=1e-5)
