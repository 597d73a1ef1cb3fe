"""Python mirror of the reference executor API over the B200 C-ABI.

Reference: /root/reference/proj/include/hmx/executor.hpp:18-81 and
proj/src/executor.cpp:259-302.

* ``EvalPlan`` / ``PlanDefaults`` / ``generate_plan`` keep the reference's lowering
  switches. The switches only pick a CPU schedule, and every schedule gives the same
  result. The B200 evaluator accepts a plan and runs its own level-batched schedule
  (``plan_pseudocode`` prints it).
* ``evaluate(cds, plan, w, stats=None)`` has the same semantics as ``hmx::evaluate``.
  A W row count that does not match raises ``ValueError`` (std::invalid_argument,
  executor.cpp:277-278). Q == 0 returns an n x 0 result (:279-282). ``stats`` gets
  ``locked_pairs == 0`` and the wall ``seconds``.
* ``Evaluator`` is the explicit handle: a context over one or more devices plus the
  uploaded matrix. Columns are sharded over the devices.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .cds import CDS


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream as an explicit handle


def torch_stream(device=None) -> int:
    """torch's current CUDA stream as a handle for the C-ABI. torch's default stream has the
    handle 0, which the C-ABI reads as "the evaluator's internal stream", so it is passed as
    cudaStreamLegacy instead (the calls are then ordered with torch's work)."""
    import torch

    h = torch.cuda.current_stream(device).cuda_stream
    return h if h else CUDA_STREAM_LEGACY


class HmxgError(RuntimeError):
    """A non-argument failure of the native evaluator (CUDA, memory, collective)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[hmxg status {code}] {msg}")
        self.code = code


def _check(rc: int) -> None:
    if rc == N.HMXG_OK:
        return
    msg = N.last_error(N.hmxg(), "hmxg")
    if rc == N.HMXG_EINVAL:
        raise ValueError(msg)
    raise HmxgError(rc, msg)


@dataclass
class EvalPlan:
    """Lowering switches (executor.hpp:20-28); results-invariant by construction."""

    block_lowering_near: bool = False
    block_lowering_far: bool = False
    coarsen_lowering: bool = False
    peel_top: bool = False
    p: int = 1
    block_threshold: int = 0
    coarsen_threshold: int = 4


@dataclass
class PlanDefaults:
    block_threshold: int = 0
    coarsen_threshold: int = 4
    p: int = 0


@dataclass
class EvalStats:
    """executor.hpp:43-46 plus the device-side accounting of the B200 run."""

    locked_pairs: int = 0
    seconds: float = 0.0
    device_ms: float = 0.0
    launches: int = 0


def generate_plan(cds: CDS, defaults: PlanDefaults | None = None, top_subtrees: int | None = None) -> EvalPlan:
    """Deterministic plan selection following executor.cpp:259-272."""
    d = defaults or PlanDefaults()
    import os

    num_leaves = int(cds.leaves().shape[0])
    plan = EvalPlan()
    plan.block_threshold = d.block_threshold or num_leaves
    plan.coarsen_threshold = d.coarsen_threshold
    plan.p = d.p or (os.cpu_count() or 1)
    plan.block_lowering_near = cds.num_near > plan.block_threshold
    plan.block_lowering_far = cds.num_far > plan.block_threshold
    plan.coarsen_lowering = cds.height + 1 > plan.coarsen_threshold
    plan.peel_top = plan.coarsen_lowering and top_subtrees is not None and top_subtrees < plan.p
    return plan


def plan_pseudocode(plan: EvalPlan | None = None) -> str:
    """The loop structure the B200 evaluator runs (cf. executor.cpp:485-514)."""
    return (
        "plan(b200: level-batched grouped FP64 GEMM, one CTA per 64x64 output tile)\n"
        "launch gather: Wp = W[perm, :]\n"
        "pass upward:\n"
        "  for height = 0 .. H: one launch over active nodes: T[i] = V[i]^T * (leaf ? Wp[i] : [T[lc]; T[rc]])\n"
        "pass far + downward:\n"
        "  for depth = 0 .. H: one launch over active nodes: S[c] = sum_j B[c,j] * T[j] + V[p][c rows] * S[p]\n"
        "pass near + leaf downward:\n"
        "  one launch over leaves: Y[i] = U[i] * S[i] + sum_j D[i,j] * W[j]\n"
        "launch scatter: Y[perm, :] = Y'\n"
    )


class Context:
    """``hmxg_ctx`` over device ids (repeats allowed: one column shard per entry)."""

    def __init__(self, devices=(0,), comm=None):
        """``comm`` (a distributed.TorchComm): one process per GPU (hmxg_create_comm) on
        ``devices[0]``; uploads then replicate the CDS while it fits the comm's HBM budget and
        hold this rank's subtree part otherwise (evaluation is then collective)."""
        lib = N.hmxg()
        h = C.c_void_p()
        if comm is not None:
            _check(lib.hmxg_create_comm(int(devices[0]), C.byref(comm.struct), C.byref(h)))
        else:
            devs = (C.c_int * len(devices))(*devices)
            _check(lib.hmxg_create(devs, len(devices), C.byref(h)))
        self._h = h
        self.comm = comm  # the collective's callback must outlive the context
        self.devices = tuple(devices)

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h:
            N.hmxg().hmxg_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class Evaluator:
    """A CDS resident on the devices of a context (``hmxg_upload``)."""

    def __init__(self, cds: CDS, devices=(0,), context: Context | None = None, points: np.ndarray | None = None,
                 kernel=None, skeletons: tuple[np.ndarray, np.ndarray] | None = None, near_on_the_fly: bool = False):
        """``points``/``kernel`` (an accuracy.Kernel): generate the near field on the device
        from the points (hmxg_upload_generated); the CDS's dgen is then not read. With
        ``skeletons`` = (skel_ptr, skel_idx) (CSR over nodes) the far blocks are generated too.
        ``near_on_the_fly``: the near blocks are never resident; every evaluation generates
        them wave by wave into a bounded scratch (HMXG_UPLOAD_NEAR_ON_THE_FLY)."""
        self.cds = cds
        self.ctx = context or Context(devices)
        self._own_ctx = context is None
        h = C.c_void_p()
        v = cds.view()
        if points is None:
            _check(N.hmxg().hmxg_upload(self.ctx.handle, C.byref(v), C.byref(h)))
        else:
            pts = np.ascontiguousarray(points, dtype=np.float64)
            if pts.ndim != 2 or pts.shape[0] != cds.n:
                raise ValueError("Evaluator: points must be an n x d array")
            sp = si = None
            if skeletons is not None:
                sp = np.ascontiguousarray(skeletons[0], dtype=np.uint64)
                si = np.ascontiguousarray(skeletons[1], dtype=np.uint32)
            _check(N.hmxg().hmxg_upload_generated_ex(
                self.ctx.handle, C.byref(v), pts.ctypes.data_as(C.c_void_p), pts.shape[1], kernel.code, kernel.h,
                sp.ctypes.data_as(C.POINTER(C.c_uint64)) if sp is not None else None,
                si.ctypes.data_as(N._u32p) if si is not None and si.size else None,
                N.HMXG_UPLOAD_NEAR_ON_THE_FLY if near_on_the_fly else 0, C.byref(h)))
        self._h = h
        self._lock = threading.Lock()

    def info(self) -> N.Info:
        inf = N.Info()
        _check(N.hmxg().hmxg_info_get(self._h, C.byref(inf)))
        return inf

    def phases(self) -> list[dict]:
        """The launch sequence with algorithmic flops/bytes and, after an evaluation run
        with ``time_phases=True``, the device time of every launch (device 0)."""
        lib = N.hmxg()
        out = []
        for i in range(lib.hmxg_phase_count(self._h)):
            ph = N.Phase()
            _check(lib.hmxg_phase_get(self._h, i, C.byref(ph)))
            out.append({"kind": N.PHASE_KINDS[ph.kind], "level": ph.level, "tiles": ph.tiles,
                        "flops_per_col": ph.flops_per_col, "gen_bytes": ph.gen_bytes,
                        "io_bytes_per_col": ph.io_bytes_per_col, "ms": ph.last_ms})
        return out

    def evaluate_host_ptr(self, w_ptr: int, y_ptr: int, q: int, ldw: int | None = None, ldy: int | None = None,
                          time_phases: bool = False, stats: EvalStats | None = None, levels: bool = False) -> None:
        """Host-pointer evaluation (pinned buffers give overlapped PCIe transfers)."""
        n = self.cds.n
        st = N.Stats()
        flags = (N.HMXG_F_TIME_PHASES if time_phases else 0) | (N.HMXG_F_LEVEL_LAUNCHES if levels else 0)
        _check(N.hmxg().hmxg_evaluate(self._h, C.c_void_p(w_ptr), n, q, ldw or n, C.c_void_p(y_ptr), ldy or n,
                                      flags, None, C.byref(st)))
        if stats is not None:
            stats.seconds = float(st.seconds)
            stats.device_ms = float(st.device_ms)
            stats.launches = int(st.launches)

    def evaluate(self, w: np.ndarray, stats: EvalStats | None = None, out: np.ndarray | None = None,
                 levels: bool = False) -> np.ndarray:
        """Y = K~ W with host arrays (column major, float64). ``levels`` runs the
        level-by-level launch sequence instead of the whole-evaluation DAG launch."""
        if w.ndim != 2:
            raise ValueError("evaluate: W must be a 2-D matrix")
        n, q = w.shape
        if n != self.cds.n:
            raise ValueError("evaluate: W row count does not match the point count")
        wf = np.asfortranarray(w, dtype=np.float64)
        y = out if out is not None else np.empty((n, q), dtype=np.float64, order="F")
        if y.shape != (n, q) or y.dtype != np.float64 or not y.flags.f_contiguous:
            raise ValueError("evaluate: out must be an n x q Fortran-ordered float64 array")
        st = N.Stats()
        if q:
            _check(N.hmxg().hmxg_evaluate(self._h, wf.ctypes.data_as(C.c_void_p), n, q, n,
                                          y.ctypes.data_as(C.c_void_p), n,
                                          N.HMXG_F_LEVEL_LAUNCHES if levels else 0, None, C.byref(st)))
        if stats is not None:
            stats.locked_pairs = int(st.locked_pairs)
            stats.seconds = float(st.seconds)
            stats.device_ms = float(st.device_ms)
            stats.launches = int(st.launches)
        return y

    def evaluate_device(self, w_ptr: int, y_ptr: int, q: int, ldw: int | None = None, ldy: int | None = None,
                        stream: int = 0, sync: bool = False, stats: EvalStats | None = None,
                        time_phases: bool = False, graph: bool = True, levels: bool = False) -> None:
        """Device-pointer evaluation (single-device context): W/Y already in HBM,
        enqueued on ``stream`` (a cudaStream_t as int, 0 = internal stream)."""
        n = self.cds.n
        flags = (N.HMXG_F_DEVICE_PTRS | (0 if sync else N.HMXG_F_NO_SYNC) | (N.HMXG_F_TIME_PHASES if time_phases else 0)
                 | (0 if graph else N.HMXG_F_NO_GRAPH) | (N.HMXG_F_LEVEL_LAUNCHES if levels else 0))
        st = N.Stats()
        _check(N.hmxg().hmxg_evaluate(self._h, C.c_void_p(w_ptr), n, q, ldw or n, C.c_void_p(y_ptr), ldy or n,
                                      flags, C.c_void_p(stream) if stream else None, C.byref(st)))
        if stats is not None:
            stats.device_ms = float(st.device_ms)
            stats.launches = int(st.launches)

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.hmxg().hmxg_free(self._h)
            self._h = None
        if self._own_ctx and self.ctx is not None:
            self.ctx.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _evaluator_for(cds: CDS, devices=(0,)) -> Evaluator:
    """The resident upload of ``cds`` for the drop-in ``evaluate``, keyed on the CDS's content
    fingerprint: an in-place edit of any array (or a different CDS at the same address)
    uploads again instead of evaluating a stale copy. The reference's evaluate has no cache
    (executor.cpp:274-302); the fingerprint pass costs one read of the CDS on the host."""
    key = ("evaluator", tuple(devices))
    fp = cds.fingerprint()
    hit = cds._cache.get(key)
    if hit is not None and hit[0] == fp:
        return hit[1]
    if hit is not None:
        hit[1].close()
    ev = Evaluator(cds, devices)
    cds._cache[key] = (fp, ev)
    return ev


def evaluate(cds: CDS, plan: EvalPlan | None, w: np.ndarray, stats: EvalStats | None = None,
             devices=(0,)) -> np.ndarray:
    """``hmx::evaluate(cds, plan, w, &stats)`` on the B200 (executor.cpp:274-302).

    The CDS is uploaded on first use and stays resident (cached on the CDS object, keyed on
    its content fingerprint, so edits are seen). ``Evaluator`` is the explicit handle.
    """
    if w.ndim != 2 or w.shape[0] != cds.n:
        raise ValueError("evaluate: W row count does not match the point count")
    if w.shape[1] == 0:
        if stats is not None:
            stats.locked_pairs, stats.seconds = 0, 0.0
        return np.zeros((cds.n, 0), dtype=np.float64, order="F")
    return _evaluator_for(cds, devices).evaluate(w, stats)
