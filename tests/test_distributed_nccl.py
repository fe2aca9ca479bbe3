"""The row-partitioned driver path over NCCL, captured into CUDA graphs and the device-side
loop.  The GPU box has one GPU, so this runs ONE NCCL rank with the row-partitioned code
path forced on (Comm(forced=True)): every collective of the path (all-gather of the block,
all-reduce of the column maxima, the partial Grams, the estimates, the FP64 residual sums,
the status word) is a real NCCL call, captured into the iteration / report graphs and
replayed inside the conditional WHILE node of the device loop -- exactly what the 8-GPU run
executes, with the data exchange degenerate.  Results must equal the single-GPU solve."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, TOP, K, SEED = 4096, 16, 32, 20240901

pytestmark = pytest.mark.gpu


def _cfg(p, pname, tol, ladder=None, reuse=False):
    return p.IterConfig(k=K, m=40, iter=1, basis_method=p.BasisMethod.HESS_LEFT, projection="ofrr",
                        policy=p.POLICY_PRESETS[pname], seed=SEED, tol=tol, top=TOP,
                        ladder=p.POLICY_PRESETS[ladder] if ladder else None, reuse_av=reuse)


def _solves(pname, tol, ladder, reuse, comm=None, times=4):
    sys.path.insert(0, ROOT)
    import paper_2505_00281_b200 as p
    lam = p.geometric_spectrum(N, TOP, K)
    A, _ = p.synthetic_symmetric(lam, p.FpFormat.BF16, seed=SEED, device=torch.device("cuda", 0))
    out = []
    for _ in range(times):
        st = p.RunStats()
        rs = p.subspace_iter_eig(A, _cfg(p, pname, tol, ladder, reuse), stats=st, comm=comm, n_global=N)
        out.append((np.asarray(rs.values), np.asarray(rs.residuals), st.iterations, st.a_passes, st.device_loop))
    return out


def _worker(port, q, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sys.path.insert(0, ROOT)
        from paper_2505_00281_b200.comm import Comm
        comm = Comm.world(forced=True)
        assert comm.distributed and comm.graphable
        q.put(_solves(*args, comm=comm))
    except Exception as e:  # surface the failure to the parent
        import traceback
        q.put(repr(e) + traceback.format_exc())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("pname,tol,ladder,reuse", [("full-f32", 1e-4, None, False),
                                                    ("full-f64", 1e-9, "full-f32", True)])
def test_nccl_row_partitioned_graphs_and_device_loop(ofrr_gpu, pname, tol, ladder, reuse):
    single = _solves(pname, tol, ladder, reuse)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_worker, args=(_free_port(), q, (pname, tol, ladder, reuse)))
    pr.start()
    res = q.get(timeout=600)
    pr.join(timeout=120)
    assert not isinstance(res, str), res
    for (v, r, its, passes, loop), (v1, r1, its1, passes1, _) in zip(res, single):
        assert its == its1 and passes == passes1
        np.testing.assert_allclose(v, v1, rtol=1e-12, atol=1e-15)
        assert np.all(r[:TOP] < tol)
    # the later solves ran as one graph launch each, NCCL calls inside the conditional nodes
    assert res[-1][4], "the row-partitioned solve did not run in the device-side loop"
