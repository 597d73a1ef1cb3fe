"""On-disk formats of the reference, so its artifacts feed the B200 evaluator directly.

Reference: /root/reference/proj/include/hmx/serial.hpp:49-55, proj/src/serial.cpp:160-308,
proj/src/pipeline.cpp:215-255 (plan.json), proj/tools/hmx.cpp:117-122 (random W).

* ``load_cds(path)`` reads ``hmat.cds`` (tag ``CDS1``, version 1) through the native
  memory-mapped reader (include/hmxg.h ``hmxg_cds_file_open``): the generator arrays stay
  in the mapping and are uploaded from there, with no host copy.
* ``save_cds(path, cds)`` writes a CDS in the same format (one row group / one block per
  blockset and one coarsen level, which keeps the storage order; BlockSet::flat_pairs,
  structure.cpp:21-27, CDS::rebuild_order, structure.cpp:188-203).
* ``load_matrix`` / ``save_matrix``: u64 rows, u64 cols, column-major f64.
* ``load_plan``: the reference's plan.json (EvalPlan fields).

I/O and format failures raise ``IoError`` (the reference's ``io_error``; the CLI maps
it to exit code 3 like proj/tools/hmx.cpp:283-285).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct

import numpy as np

from . import _native as N
from .cds import CDS

CDS_TAG = b"CDS1"
CDS_VERSION = 1


class IoError(OSError):
    """hmx::io_error (proj/include/hmx/io.hpp)."""


class CdsFile:
    """An opened ``hmat.cds``: ``cds`` is a zero-copy CDS over the mapping (kept alive by
    this object), plus the header fields the evaluator does not need."""

    def __init__(self, path: str):
        lib = N.hmxg()
        h = C.c_void_p()
        rc = lib.hmxg_cds_file_open(os.fsencode(path), C.byref(h))
        if rc != N.HMXG_OK:
            msg = lib.hmxg_cds_file_error().decode()
            if rc == N.HMXG_EINVAL:
                raise ValueError(msg)
            raise IoError(msg)
        self._h = h
        self.path = path
        v = N.CdsView()
        lib.hmxg_cds_file_view(h, C.byref(v))
        dim, bacc, max_rank = C.c_uint32(), C.c_double(), C.c_uint32()
        lib.hmxg_cds_file_header(h, C.byref(dim), C.byref(bacc), C.byref(max_rank))
        self.dim, self.bacc, self.max_rank = int(dim.value), float(bacc.value), int(max_rank.value)
        self.cds = CDS.from_view(v, owner=self)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.cds._cache.clear()
            N.hmxg().hmxg_cds_file_close(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def load_cds(path: str) -> CDS:
    """hmx::load_cds (serial.cpp:299-308); the returned CDS keeps the mapping alive."""
    return CdsFile(path).cds


def _u32s(a) -> bytes:
    a = np.ascontiguousarray(a, dtype="<u4")
    return struct.pack("<Q", a.size) + a.tobytes()


def _u64s(a) -> bytes:
    a = np.ascontiguousarray(a, dtype="<u8")
    return struct.pack("<Q", a.size) + a.tobytes()


def _f64s(a) -> bytes:
    a = np.ascontiguousarray(a, dtype="<f8")
    return struct.pack("<Q", a.size) + a.tobytes()


def _blockset(pairs: np.ndarray, far: bool) -> bytes:
    out = [struct.pack("<BI", 1 if far else 0, 1)]
    npairs = int(pairs.shape[0])
    if npairs == 0:
        out.append(struct.pack("<Q", 0))
    else:
        out.append(struct.pack("<QIQQ", 1, 0, 1, npairs))
        out.append(np.ascontiguousarray(pairs, dtype="<u4").tobytes())
    return b"".join(out)


def save_cds(path: str, cds: CDS, dim: int = 0, bacc: float = 0.0, max_rank: int = 0,
             leaf_size: int | None = None) -> None:
    """Write ``cds`` as ``hmat.cds`` (write_cds, serial.cpp:160-178). ``leaf_size`` is the
    tree's leaf parameter (ClusterTree::validate: leaf iff size <= leaf_size); by default
    the largest leaf."""
    sizes = cds.end.astype(np.int64) - cds.start.astype(np.int64)
    if leaf_size is None:
        leaves = cds.lchild == N.HMXG_NO_NODE
        leaf_size = int(sizes[leaves].max()) if leaves.any() else 0
    parts = [
        CDS_TAG, struct.pack("<I", CDS_VERSION),
        struct.pack("<QIIdI", cds.n, dim, cds.num_nodes, bacc, max_rank),
        struct.pack("<I", cds.num_nodes),
        _u32s(cds.parent), _u32s(cds.lchild), _u32s(cds.rchild), _u32s(cds.start), _u32s(cds.end),
        _u32s(cds.level), _u32s(cds.perm), struct.pack("<II", cds.height, leaf_size),
        _u32s(cds.sranks),
        struct.pack("<Q", cds.num_nodes), np.ascontiguousarray(cds.participating, dtype=np.uint8).tobytes(),
        _blockset(cds.near_pairs, far=False), _blockset(cds.far_pairs, far=True),
        # coarsenset: agg, p, one level holding one subtree with the whole V order
        struct.pack("<IIQQd", 1, 1, 1, 1, 0.0), _u32s(cds.v_order),
        _u64s(cds.dptr), _f64s(cds.dgen), _u64s(cds.bptr), _f64s(cds.bgen), _u64s(cds.vptr), _f64s(cds.vgen),
    ]
    try:
        with open(path, "wb") as f:
            for p in parts:
                f.write(p)
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from e


def load_matrix(path: str) -> np.ndarray:
    """hmx::load_matrix (serial.cpp:287-297): n x q column major, as a Fortran array."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open {path}: {e}") from e
    if len(data) < 16:
        raise IoError(f"truncated matrix file {path}")
    rows, cols = struct.unpack_from("<QQ", data, 0)
    if cols != 0 and rows > (1 << 40) // cols:
        raise IoError(f"implausible matrix dimensions in {path}")
    need = 16 + rows * cols * 8
    if len(data) < need:
        raise IoError(f"truncated matrix file {path}")
    if len(data) > need:
        raise IoError(f"trailing bytes in matrix file {path}")
    m = np.frombuffer(data, dtype="<f8", count=rows * cols, offset=16)
    return np.asfortranarray(m.reshape((cols, rows)).T)


def save_matrix(path: str, m: np.ndarray) -> None:
    """hmx::save_matrix (serial.cpp:279-285)."""
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2:
        raise ValueError("save_matrix: expected a 2-D matrix")
    try:
        with open(path, "wb") as f:
            f.write(struct.pack("<QQ", m.shape[0], m.shape[1]))
            f.write(np.asfortranarray(m).tobytes(order="F"))
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from e


def load_plan(path: str):
    """hmx::load_plan (pipeline.cpp:249-255): the EvalPlan fields of plan.json."""
    from .executor import EvalPlan

    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise IoError(f"cannot open plan: {path}") from e
    except json.JSONDecodeError as e:
        raise IoError(f"malformed plan {path}: {e}") from e
    try:
        return EvalPlan(block_lowering_near=bool(j["block_lowering_near"]),
                        block_lowering_far=bool(j["block_lowering_far"]),
                        coarsen_lowering=bool(j["coarsen_lowering"]), peel_top=bool(j["peel_top"]),
                        p=int(j["p"]), block_threshold=int(j["block_threshold"]),
                        coarsen_threshold=int(j["coarsen_threshold"]))
    except (KeyError, TypeError, ValueError) as e:
        raise IoError(f"malformed plan {path}: {e}") from e


def random_w(n: int, q: int, seed: int) -> np.ndarray:
    """The CLI's random right-hand side (hmx.cpp:117-122), bit-identical to the reference."""
    w = np.empty((n, q), dtype=np.float64, order="F")
    if n * q:
        N.hmxb().hmxb_random_w(seed, n, q, w.ctypes.data_as(C.c_void_p))
    return w
