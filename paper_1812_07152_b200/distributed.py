"""Multi-GPU plumbing of the column-sharded evaluation.

One process per GPU (torchrun), the CDS replicated on every rank, the Q columns of W
split into contiguous shards. Y[:, c] depends only on W[:, c] (executor.cpp:119-129,
SURVEY F8), so the data path needs no collective. ``torch.distributed`` is used for the
barrier, the max-over-ranks of timings, the replication check and, only when a caller
wants the full Y on every rank, an all-gather of the column shards.
"""
from __future__ import annotations

import hashlib

import numpy as np

from . import _native as N
from .cds import CDS


def column_shard(q: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [c0, c1) of the q columns for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("column_shard: bad rank/world")
    return q * rank // world, q * (rank + 1) // world


def cds_fingerprint(cds: CDS) -> str:
    """Content hash of a CDS; equal on every rank iff the replicated CDS is identical."""
    h = hashlib.sha256()
    for name in ("perm", "start", "end", "lchild", "rchild", "sranks", "participating", "near_pairs", "far_pairs",
                 "v_order", "dptr", "bptr", "vptr", "dgen", "bgen", "vgen"):
        h.update(np.ascontiguousarray(getattr(cds, name)).tobytes())
    return h.hexdigest()


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def check_replicated(cds: CDS) -> None:
    """Raise if the CDS differs between ranks (all ranks must build/load the same one)."""
    import torch.distributed as dist

    if not dist.is_initialized():
        return
    mine = cds_fingerprint(cds)
    every = [None] * dist.get_world_size()
    dist.all_gather_object(every, mine)
    if any(f != mine for f in every):
        raise RuntimeError("CDS differs between ranks: the column-sharded evaluation needs a replicated CDS")


def gather_columns(y_local: np.ndarray, q_total: int) -> np.ndarray:
    """All-gather the ranks' column shards (n x q_r, Fortran) into the full n x q Y."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    n = y_local.shape[0]
    widths = [column_shard(q_total, world, r) for r in range(world)]
    qmax = max(c1 - c0 for c0, c1 in widths)
    buf = torch.zeros((qmax, n), dtype=torch.float64)
    c0, c1 = widths[rank]
    buf[: c1 - c0] = torch.from_numpy(np.ascontiguousarray(y_local.T))
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    y = np.empty((n, q_total), dtype=np.float64, order="F")
    for r, (a, b) in enumerate(widths):
        y[:, a:b] = parts[r][: b - a].numpy().T
    return y


class SplitPart:
    """One part of the subtree-split fallback (include/hmxg.h hmxg_upload_split).

    For a CDS that does not fit one GPU: part ``part`` of ``nparts`` holds only the
    generators of its own subtrees (plus the replicated top levels). An evaluation is
    stage 0 (upward over its subtrees), a sum-exchange of the skeleton weights T between
    the parts, stage 1 (top levels, far+downward, near/leaf for its targets), and a sum
    of the parts' Y (each part's Y is zero outside its rows).
    """

    def __init__(self, cds: CDS, nparts: int, part: int, device: int = 0):
        import ctypes as C

        from .executor import Context, _check

        self._C, self._check = C, _check
        self.cds, self.nparts, self.part = cds, nparts, part
        self.ctx = Context((device,))
        h = C.c_void_p()
        v = cds.view()
        _check(N.hmxg().hmxg_upload_split(self.ctx.handle, C.byref(v), nparts, part, C.byref(h)))
        self._h = h

    def stage(self, stage: int, w_ptr: int, y_ptr: int, q: int, stream: int = 0) -> None:
        C = self._C
        n = self.cds.n
        self._check(N.hmxg().hmxg_split_stage(self._h, stage, C.c_void_p(w_ptr), n, q, n, C.c_void_p(y_ptr), n,
                                              C.c_void_p(stream) if stream else None))

    def exchange_count(self) -> int:
        C = self._C
        p, c = C.c_void_p(), C.c_size_t()
        self._check(N.hmxg().hmxg_split_exchange_buffer(self._h, C.byref(p), C.byref(c)))
        return int(c.value)

    def exchange(self, buf_ptr: int, count: int, to_matrix: bool, stream: int = 0) -> None:
        C = self._C
        self._check(N.hmxg().hmxg_split_exchange(self._h, C.c_void_p(buf_ptr), count, 1 if to_matrix else 0,
                                                 C.c_void_p(stream) if stream else None))

    def info(self) -> N.Info:
        C = self._C
        inf = N.Info()
        self._check(N.hmxg().hmxg_info_get(self._h, C.byref(inf)))
        return inf

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.hmxg().hmxg_free(self._h)
            self._h = None
        if getattr(self, "ctx", None) is not None:
            self.ctx.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def split_evaluate(cds: CDS, w, parts: list["SplitPart"] | None = None, nparts: int = 2, group=None):
    """Y = K~ W with the subtree-split fallback, W a CUDA tensor of shape (q, n) (= n x q
    column major). In one process all parts run on W's device and the exchange is a
    local sum; under torch.distributed (one part per rank, ``parts=[this rank's part]``)
    the exchanges are all-reduce sums over NCCL."""
    import torch
    import torch.distributed as dist

    q = w.shape[0]
    distributed = dist.is_initialized() and dist.get_world_size() > 1

    def allreduce(x):
        if not distributed:
            return x
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(x, group=group)
            return x
        h = x.cpu()
        dist.all_reduce(h, group=group)
        return h.to(x.device)

    own_parts = parts is None  # parts uploaded here are released here (each holds device memory)
    if own_parts:
        parts = [SplitPart(cds, nparts, k, w.device.index or 0) for k in range(nparts)]
    # every native call runs on torch's current stream, ordered with the tensor ops around it
    from .executor import torch_stream

    try:
        st = torch_stream(w.device)
        ys = [torch.zeros_like(w) for _ in parts]
        for part, y in zip(parts, ys):
            part.stage(0, w.data_ptr(), y.data_ptr(), q, stream=st)
        count = parts[0].exchange_count()
        ts = [torch.empty(count, dtype=torch.float64, device=w.device) for _ in parts]
        for part, t in zip(parts, ts):
            part.exchange(t.data_ptr(), count, to_matrix=False, stream=st)
        total = allreduce(torch.stack(ts).sum(0) if len(ts) > 1 else ts[0])
        for part in parts:
            part.exchange(total.data_ptr(), count, to_matrix=True, stream=st)
        for part, y in zip(parts, ys):
            part.stage(1, w.data_ptr(), y.data_ptr(), q, stream=st)  # (returns when the stage is done)
        return allreduce(torch.stack(ys).sum(0) if len(ys) > 1 else ys[0])
    finally:
        if own_parts:
            for part in parts:
                part.close()


class _DeviceBytes:
    """A device byte range as a torch tensor (``__cuda_array_interface__``, no copy)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


class TorchComm:
    """``hmxg_comm`` over a ``torch.distributed`` process group (one process per GPU).

    The C-ABI calls ``allgatherv`` in place on contiguous blocks in rank order. With NCCL the
    blocks stay on the device and every rank's block is broadcast from its owner on the
    library's stream; with any other backend (gloo) the library stages through pinned host
    memory (``host_buffers``) and the blocks travel as padded byte tensors. A failure returns
    non-zero, which the library reports as HMXG_ECOMM.
    ``hbm_budget``: bytes the resident CDS may use per device before ``hmxg_upload`` falls back
    to the subtree split (0: 3/4 of the device's memory).
    """

    def __init__(self, group=None, hbm_budget: int = 0, host_buffers: bool | None = None):
        import ctypes as C

        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.host_buffers = (backend != "nccl") if host_buffers is None else bool(host_buffers)
        self.errors: list[str] = []
        self._fn = N.ALLGATHERV_FN(self._allgatherv)  # kept alive with the struct
        self.struct = N.Comm(rank=self.rank, size=self.size, allgatherv=self._fn, user=None,
                             host_buffers=1 if self.host_buffers else 0, reserved=0, hbm_budget=int(hbm_budget))
        self._C = C

    def _allgatherv(self, user, send, sendbytes, recv, recvbytes, displs, stream):
        import torch
        import torch.distributed as dist

        C = self._C
        try:
            counts = [int(recvbytes[r]) for r in range(self.size)]
            disp = [int(displs[r]) for r in range(self.size)]
            if self.host_buffers:
                m = max(counts) or 1
                mine = torch.zeros(m, dtype=torch.uint8)
                if sendbytes:
                    C.memmove(mine.data_ptr(), send, sendbytes)
                outs = [torch.empty(m, dtype=torch.uint8) for _ in range(self.size)]
                dist.all_gather(outs, mine, group=self.group)
                for r in range(self.size):
                    if counts[r]:
                        C.memmove(recv + disp[r], outs[r].data_ptr(), counts[r])
            else:
                with torch.cuda.stream(torch.cuda.ExternalStream(stream or 0)):
                    for r in range(self.size):
                        if counts[r]:
                            t = torch.as_tensor(_DeviceBytes(recv + disp[r], counts[r]), device="cuda")
                            dist.broadcast(t, src=dist.get_global_rank(self.group, r) if self.group else r,
                                           group=self.group)
            return 0
        except Exception as e:  # reported by the library as HMXG_ECOMM
            self.errors.append(repr(e))
            return 1
