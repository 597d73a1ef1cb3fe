"""Host-side CDS: the reference's computation-ordered generator store as numpy arrays.

Mirrors ``hmx::CDS`` (/root/reference/proj/include/hmx/structure.hpp:83-130): tree
arrays, sranks, participation, near/far pair lists in storage order (``near_order`` /
``far_order``), the V storage order (``v_order``) and the flat ``dptr/bptr/vptr`` +
``dgen/bgen/vgen`` arrays. ``view()`` exposes it as the C-ABI ``hmxg_cds_view``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _native as N


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a.size else C.POINTER(ctype)()


@dataclass
class CDS:
    n: int
    num_nodes: int
    height: int
    parent: np.ndarray
    lchild: np.ndarray
    rchild: np.ndarray
    start: np.ndarray
    end: np.ndarray
    level: np.ndarray
    perm: np.ndarray
    sranks: np.ndarray
    participating: np.ndarray
    near_pairs: np.ndarray  # (num_near, 2) uint32, storage order
    far_pairs: np.ndarray   # (num_far, 2) uint32, storage order
    v_order: np.ndarray
    dptr: np.ndarray
    bptr: np.ndarray
    vptr: np.ndarray
    dgen: np.ndarray
    bgen: np.ndarray
    vgen: np.ndarray
    owner: Any = None  # keeps a native producer alive when arrays are zero-copy views
    _cache: dict = field(default_factory=dict, repr=False)

    def fingerprint(self) -> int:
        """Content hash of every array (``hmxg_cds_fingerprint``): equal only for equal CDSs,
        up to 64-bit hash collisions. One multi-threaded pass over the generators."""
        out = C.c_uint64()
        v = self.view()
        rc = N.hmxg().hmxg_cds_fingerprint(C.byref(v), C.byref(out))
        if rc:
            raise ValueError(N.last_error(N.hmxg(), "hmxg"))
        return int(out.value)

    # ---- reference accessors (structure.hpp:104-128)
    def is_leaf(self, i: int) -> bool:
        return int(self.lchild[i]) == N.HMXG_NO_NODE

    def node_size(self, i: int) -> int:
        return int(self.end[i]) - int(self.start[i])

    def v_width(self, i: int) -> int:
        if self.is_leaf(i):
            return self.node_size(i)
        return int(self.sranks[self.lchild[i]]) + int(self.sranks[self.rchild[i]])

    def leaves(self) -> np.ndarray:
        return np.nonzero(self.lchild == N.HMXG_NO_NODE)[0].astype(np.uint32)

    @property
    def num_near(self) -> int:
        return int(self.near_pairs.shape[0])

    @property
    def num_far(self) -> int:
        return int(self.far_pairs.shape[0])

    def extract_d(self, slot: int) -> np.ndarray:
        i, j = (int(x) for x in self.near_pairs[slot])
        a, b = int(self.dptr[slot]), int(self.dptr[slot + 1])
        return self.dgen[a:b].reshape(self.node_size(j), self.node_size(i)).T

    def extract_b(self, slot: int) -> np.ndarray:
        i, j = (int(x) for x in self.far_pairs[slot])
        a, b = int(self.bptr[slot]), int(self.bptr[slot + 1])
        return self.bgen[a:b].reshape(int(self.sranks[j]), int(self.sranks[i])).T

    def extract_v(self, node: int) -> np.ndarray:
        slot = int(np.nonzero(self.v_order == node)[0][0])
        a, b = int(self.vptr[slot]), int(self.vptr[slot + 1])
        return self.vgen[a:b].reshape(int(self.sranks[node]), self.v_width(node)).T

    # ---- accounting
    @property
    def d_elems(self) -> int:
        return int(self.dptr[-1])

    @property
    def b_elems(self) -> int:
        return int(self.bptr[-1])

    @property
    def v_elems(self) -> int:
        return int(self.vptr[-1])

    def flops(self, q: int) -> float:
        """Algorithmic FP64 flops of one evaluation: 2 Q (2|V| + |B| + |D|)."""
        return 2.0 * q * (2.0 * self.v_elems + self.b_elems + self.d_elems)

    def bytes(self, q: int) -> float:
        """Algorithmic HBM bytes: generators read once, W read once, Y written once."""
        return 8.0 * (self.d_elems + self.b_elems + self.v_elems) + 16.0 * self.n * q

    # ---- C-ABI view
    def view(self) -> N.CdsView:
        v = N.CdsView()
        v.n = self.n
        v.num_nodes = self.num_nodes
        v.height = self.height
        for name in ("parent", "lchild", "rchild", "start", "end", "level", "perm", "sranks", "v_order"):
            setattr(v, name, _ptr(getattr(self, name), C.c_uint32))
        v.participating = _ptr(self.participating, C.c_uint8)
        v.num_near = self.num_near
        v.near_pairs = _ptr(self.near_pairs, C.c_uint32)
        v.num_far = self.num_far
        v.far_pairs = _ptr(self.far_pairs, C.c_uint32)
        v.num_v = int(self.v_order.shape[0])
        v.dptr = _ptr(self.dptr, C.c_uint64)
        v.bptr = _ptr(self.bptr, C.c_uint64)
        v.vptr = _ptr(self.vptr, C.c_uint64)
        v.dgen = _ptr(self.dgen, C.c_double)
        v.bgen = _ptr(self.bgen, C.c_double)
        v.vgen = _ptr(self.vgen, C.c_double)
        return v

    @classmethod
    def from_view(cls, v: N.CdsView, owner: Any = None, copy: bool = False) -> "CDS":
        """Wrap a native view (zero-copy while ``owner`` lives, or copied)."""

        def arr(ptr, count, dtype):
            if count == 0 or not ptr:
                return np.zeros(0, dtype=dtype)
            a = np.ctypeslib.as_array(ptr, shape=(int(count),))
            return a.copy() if copy else a

        nn, n = int(v.num_nodes), int(v.n)
        nnear, nfar, nv = int(v.num_near), int(v.num_far), int(v.num_v)
        dptr = arr(v.dptr, nnear + 1, np.uint64)
        bptr = arr(v.bptr, nfar + 1, np.uint64)
        vptr = arr(v.vptr, nv + 1, np.uint64)
        return cls(
            n=n, num_nodes=nn, height=int(v.height),
            parent=arr(v.parent, nn, np.uint32), lchild=arr(v.lchild, nn, np.uint32),
            rchild=arr(v.rchild, nn, np.uint32), start=arr(v.start, nn, np.uint32),
            end=arr(v.end, nn, np.uint32), level=arr(v.level, nn, np.uint32),
            perm=arr(v.perm, n, np.uint32), sranks=arr(v.sranks, nn, np.uint32),
            participating=arr(v.participating, nn, np.uint8),
            near_pairs=arr(v.near_pairs, 2 * nnear, np.uint32).reshape(nnear, 2),
            far_pairs=arr(v.far_pairs, 2 * nfar, np.uint32).reshape(nfar, 2),
            v_order=arr(v.v_order, nv, np.uint32), dptr=dptr, bptr=bptr, vptr=vptr,
            dgen=arr(v.dgen, int(dptr[-1]) if nnear + 1 else 0, np.float64),
            bgen=arr(v.bgen, int(bptr[-1]), np.float64),
            vgen=arr(v.vgen, int(vptr[-1]), np.float64),
            owner=None if copy else owner,
        )

    def copy(self) -> "CDS":
        kw = {k: (getattr(self, k).copy() if isinstance(getattr(self, k), np.ndarray) else getattr(self, k))
              for k in self.__dataclass_fields__ if k not in ("owner", "_cache")}
        return CDS(**kw)

    def save_npz(self, path: str) -> None:
        np.savez_compressed(path, **{k: getattr(self, k) for k in self.__dataclass_fields__
                                     if k not in ("owner", "_cache")})

    @classmethod
    def load_npz(cls, path: str) -> "CDS":
        z = np.load(path)
        kw = {k: z[k] for k in z.files}
        for k in ("n", "num_nodes", "height"):
            kw[k] = int(kw[k])
        return cls(**kw)
