"""Row-partitioned communication for the multi-GPU path.

A (n x n) is row-partitioned: rank p owns rows [p*rp, min(n, (p+1)*rp)) with
rp = ceil(n / P).  Per power step the ranks all-gather their n/P x k slices of the
block; per projection they all-reduce the k x k partial Grams (fp64) and the k column
maxima.  One process per GPU; torch.distributed (NCCL over NVLink/NVSwitch on the GPU
box, gloo in the CPU tests) is the plumbing.  NCCL collectives are captured into the
driver's CUDA graphs (and replayed inside its device-side loop); gloo runs eagerly.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class Comm:
    rank: int = 0
    size: int = 1
    group: object = None
    forced: bool = False      # the row-partitioned code path even with one rank (tests)

    @classmethod
    def world(cls, forced: bool = False) -> "Comm":
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(), dist.get_world_size(), None, forced)
        return cls()

    @property
    def distributed(self) -> bool:
        return self.size > 1 or self.forced

    @property
    def graphable(self) -> bool:
        """Collectives can be captured into CUDA graphs (NCCL; not gloo)."""
        if not self.distributed:
            return True
        import torch.distributed as dist
        try:
            return dist.get_backend(self.group) == "nccl"
        except Exception:
            return False

    def rows_per(self, n: int) -> int:
        return (int(n) + self.size - 1) // self.size

    def row_range(self, n: int, rank: int = None):
        rank = self.rank if rank is None else rank
        rp = self.rows_per(n)
        r0 = min(n, rank * rp)
        return r0, min(n, r0 + rp)

    # ---- collectives ----------------------------------------------------------------
    def all_reduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.distributed:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max_(self, t: torch.Tensor) -> torch.Tensor:
        if self.distributed:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def all_gather_rows(self, local: torch.Tensor, full: torch.Tensor, n: int, k: int) -> torch.Tensor:
        """Gather column-major row slices.

        ``local``: tensor (k_alloc, ld_local) holding this rank's rows of k columns
        (row j = column j).  ``full``: tensor (k_alloc, ld) receiving all n rows.
        The collective moves every rank's k x rp slice (rp = ceil(n/P), the last rank's
        padded); when this rank's slice already is a contiguous k x rp block (ld_local == rp,
        e.g. n = 65536 on 8 GPUs) it is sent in place.  One strided copy then puts the
        rank-major result into the column-major block."""
        if not self.distributed:
            if full.data_ptr() != local.data_ptr():
                full[:k, :n].copy_(local[:k, :n])
            return full
        import torch.distributed as dist
        rp = self.rows_per(n)
        r0, r1 = self.row_range(n)
        if local.stride(0) == rp and r1 - r0 == rp and local.is_contiguous():
            send = local[:k]
        else:
            send = torch.zeros((k, rp), dtype=local.dtype, device=local.device)
            send[:, : r1 - r0].copy_(local[:k, : r1 - r0])
        recv = torch.empty((self.size * k, rp), dtype=local.dtype, device=local.device)
        # gathered as bytes (every storage format on every backend), rank-major along dim 0
        dist.all_gather_into_tensor(recv.view(torch.uint8), send.view(torch.uint8), group=self.group)
        recv = recv.view(self.size, k, rp)                 # recv[p, j, i] = X[p*rp + i, j]
        if self.size * rp == n:
            full[:k, :n].view(k, self.size, rp).copy_(recv.permute(1, 0, 2))
        else:
            full[:k, :n].copy_(recv.permute(1, 0, 2).reshape(k, self.size * rp)[:, :n])
        return full
