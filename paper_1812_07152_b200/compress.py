"""GPU compression: the interpolative decomposition of every participating node.

Mirrors ``hmx::compress``'s basis construction (/root/reference/proj/src/compress.cpp:17-148)
on the B200 through ``hmxg_compress`` (include/hmxg.h): bottom-up by level, one CTA per
node, the reference's column-pivoted Householder QR with the same per-column arithmetic.
The far and near blocks that follow (compress.cpp:139-147) are kernel evaluations on the
skeletons / points; the near ones are generated on the device by ``Evaluator(points=...)``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .accuracy import Kernel, _check
from .cds import CDS


@dataclass
class NodeBasis:
    """hmx::NodeBasis (compress.hpp:29-33): srank, skeleton point indices, V (rows x srank)."""

    srank: int
    skeleton: np.ndarray
    v: np.ndarray


_CONTEXTS: dict = {}


def _context(device: int):
    """One evaluator context per device for the process (creating one per call costs more
    than a small compression)."""
    from .executor import Context

    if device not in _CONTEXTS:
        _CONTEXTS[device] = Context((device,))
    return _CONTEXTS[device]


def gpu_compress(points: np.ndarray, kernel: Kernel, cds: CDS, sample_ptr: np.ndarray, sample_idx: np.ndarray,
                 bacc: float, max_rank: int, device: int = 0) -> list[NodeBasis]:
    """Bases of every node of ``cds``'s tree (participation from ``cds.participating``);
    ``sample_ptr``/``sample_idx`` are hmx::SampleInfo::rows in CSR form."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    sp = np.ascontiguousarray(sample_ptr, dtype=np.uint64)
    si = np.ascontiguousarray(sample_idx, dtype=np.uint32)
    if sp.size != cds.num_nodes + 1:
        raise ValueError("compress: sampling info does not match tree")
    ctx = _context(device)
    lib = N.hmxg()
    h = C.c_void_p()

    def u32(a):
        return np.ascontiguousarray(a, dtype=np.uint32).ctypes.data_as(N._u32p)

    arrays = [np.ascontiguousarray(getattr(cds, k), dtype=np.uint32)
              for k in ("lchild", "rchild", "start", "end", "level", "perm")]
    part = np.ascontiguousarray(cds.participating, dtype=np.uint8)
    try:
        _check(lib.hmxg_compress(ctx.handle, pts.ctypes.data_as(C.c_void_p), pts.shape[0], pts.shape[1], kernel.code,
                                 kernel.h, cds.num_nodes, *[a.ctypes.data_as(N._u32p) for a in arrays],
                                 part.ctypes.data_as(C.POINTER(C.c_uint8)), sp.ctypes.data_as(C.POINTER(C.c_uint64)),
                                 si.ctypes.data_as(N._u32p) if si.size else None, bacc, max_rank, C.byref(h)))
        sr, skp, sk, vp, vr, v = (N._u32p(), C.POINTER(C.c_uint64)(), N._u32p(), C.POINTER(C.c_uint64)(),
                                  C.POINTER(C.c_uint64)(), N._f64p())
        lib.hmxg_compressed_get(h, C.byref(sr), C.byref(skp), C.byref(sk), C.byref(vp), C.byref(vr), C.byref(v))
        nn = cds.num_nodes
        sranks = np.ctypeslib.as_array(sr, shape=(nn,)).copy()
        skel_ptr = np.ctypeslib.as_array(skp, shape=(nn + 1,)).copy()
        v_ptr = np.ctypeslib.as_array(vp, shape=(nn + 1,)).copy()
        v_rows = np.ctypeslib.as_array(vr, shape=(nn,)).copy()
        skel = np.ctypeslib.as_array(sk, shape=(int(skel_ptr[-1]),)).copy() if skel_ptr[-1] else np.zeros(0, np.uint32)
        vals = np.ctypeslib.as_array(v, shape=(int(v_ptr[-1]),)).copy() if v_ptr[-1] else np.zeros(0)
        out = []
        for i in range(nn):
            k, rows = int(sranks[i]), int(v_rows[i])
            out.append(NodeBasis(k, skel[skel_ptr[i]:skel_ptr[i + 1]],
                                 vals[v_ptr[i]:v_ptr[i + 1]].reshape((k, rows)).T if k else np.zeros((rows, 0))))
        return out
    finally:
        if h:
            lib.hmxg_compressed_free(h)


def skeleton_csr(bases: list[NodeBasis]) -> tuple[np.ndarray, np.ndarray]:
    """(skel_ptr, skel_idx) over nodes, for Evaluator(skeletons=...)."""
    ptr = np.zeros(len(bases) + 1, dtype=np.uint64)
    for i, b in enumerate(bases):
        ptr[i + 1] = ptr[i] + b.skeleton.size
    idx = np.concatenate([b.skeleton for b in bases]).astype(np.uint32) if ptr[-1] else np.zeros(0, np.uint32)
    return ptr, idx


def cds_from_bases(structure: CDS, bases: list[NodeBasis]) -> CDS:
    """A CDS with ``structure``'s tree, pair lists and storage orders and the V generators
    of ``bases`` (vgen in v_order, each V column major: structure.hpp:104-128); dgen and
    bgen are left empty for the device to generate (Evaluator(points=, skeletons=))."""
    for i, b in enumerate(bases):
        if b.srank != int(structure.sranks[i]):
            raise ValueError(f"cds_from_bases: node {i} has srank {b.srank}, the structure {int(structure.sranks[i])}")
    vptr = np.zeros(structure.v_order.size + 1, dtype=np.uint64)
    parts = []
    for s, node in enumerate(structure.v_order):
        v = bases[int(node)].v
        parts.append(np.asfortranarray(v).ravel(order="F"))
        vptr[s + 1] = vptr[s] + v.size
    if not np.array_equal(vptr, structure.vptr):
        raise ValueError("cds_from_bases: V sizes differ from the structure's vptr")
    kw = {k: getattr(structure, k) for k in structure.__dataclass_fields__ if k not in ("owner", "_cache")}
    kw["vgen"] = np.concatenate(parts) if parts else np.zeros(0)
    kw["dgen"] = np.zeros(0)
    kw["bgen"] = np.zeros(0)
    return CDS(**kw)
