"""The row-partitioned driver path with the real CUDA kernels: 2 ranks on one GPU, gloo
collectives (host-staged; the ranks' kernels never wait on each other), against the
single-process solve.  Exercises the distributed branches of EigEngine end to end: local
block products on each rank's rows of A, all-reduce of column maxima, all-gather of the
block, redundant Hessenberg + pencil, all-reduced Grams, estimates and FP64 residuals.
(NCCL over NVLink replaces gloo on a multi-GPU box; the driver code is the same.)"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, TOP, K, SEED = 2048, 8, 32, 20240901

pytestmark = pytest.mark.gpu


def _solve(pname, comm=None, row0=0, rows=None, tol=None):
    sys.path.insert(0, ROOT)
    import paper_2505_00281_b200 as p
    lam = p.geometric_spectrum(N, TOP, K)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED, device=torch.device("cuda", 0),
                                 row0=row0, rows=rows)
    cfg = p.IterConfig(k=K, m=6 if tol is None else 40, iter=1, basis_method=p.BasisMethod.HESS_LEFT,
                       projection="ofrr", policy=p.POLICY_PRESETS[pname], seed=SEED, tol=tol,
                       top=TOP if tol is not None else None)
    st = p.RunStats()
    rs = p.subspace_iter_eig(A, cfg, stats=st, comm=comm, n_global=N)
    return np.asarray(rs.values), np.asarray(rs.residuals), st.iterations, st.a_passes


def _worker(rank, world, port, q, pname, tol):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, ROOT)
        from paper_2505_00281_b200.comm import Comm
        comm = Comm.world()
        r0, r1 = comm.row_range(N)
        q.put((rank, _solve(pname, comm=comm, row0=r0, rows=r1 - r0, tol=tol)))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("pname,tol", [("full-f32", None), ("tc-bf16", None), ("full-f32", 1e-4),
                                       ("full-f64", 1e-9)])
def test_row_partitioned_gpu_matches_single(ofrr_gpu, pname, tol):
    single = _solve(pname, tol=tol)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, pname, tol)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=120)
    for rank, res in out:
        assert not isinstance(res, str), res
        vals, resid, its, passes = res
        assert its == single[2] and passes == single[3]
        # each rank's block product splits K differently (stream-K over fewer rows), so fp32
        # tensor-core sums differ in order from the single-GPU run: agreement to that rounding
        # (fp32 accumulation) or to fp64 rounding (the int8 Ozaki products are exact integers)
        if pname == "full-f64":
            np.testing.assert_allclose(vals, single[0], rtol=1e-11, atol=1e-14)
        else:
            # 16-bit / fp32-accumulated: the north-star reading, same accuracy as the single run
            import paper_2505_00281_b200 as p
            lam = p.geometric_spectrum(N, TOP, K)
            err = np.max(np.abs(vals[:TOP] - lam[:TOP]) / lam[:TOP])
            ref = np.max(np.abs(single[0][:TOP] - lam[:TOP]) / lam[:TOP])
            assert err <= max(10 * ref, 1e-6), (err, ref)
        # residuals at the basis' rounding floor are noise: the north-star 2x criterion, both ways
        assert np.all(resid[:TOP] <= 2 * single[1][:TOP] + 1e-13)
        assert np.all(single[1][:TOP] <= 2 * resid[:TOP] + 1e-13)
    np.testing.assert_array_equal(out[0][1][0], out[1][1][0])
