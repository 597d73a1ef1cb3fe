"""Seeded synthetic instances: the host builder (libhmxb.so) and the BASELINE configs.

``build_instance(spec)`` runs the native builder and returns an ``Instance`` whose
``cds`` is a zero-copy ``CDS`` over the builder's arrays. ``CONFIGS`` holds the five
BASELINE.json configurations, with seeded synthetic points standing in
for the paper's datasets.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _native as N
from .cds import CDS

POINTS = {"uniform": 0, "grid2d": 1, "mixture": 2, "normal": 3, "quantized": 4}
KERNELS = {"gaussian": 0, "exponential": 1, "invdist": 2}
MODES = {"hss": 0, "tau": 1, "budget": 2}
SPLITS = {"auto": 0, "kd": 1, "twomeans": 2}
EXACT_SAMPLING = 0xFFFFFFFF


@dataclass
class InstanceSpec:
    n: int = 4096
    d: int = 3
    points: str = "uniform"
    components: int = 8
    levels: int = 16
    seed: int = 42
    kernel: str = "gaussian"
    h: float = 0.5
    leaf: int = 128
    split: str = "auto"
    mode: str = "hss"
    tau: float = 0.65
    budget: float = 0.03
    max_rank: int = 64
    tol: float = 1e-5
    sample_rows: int = 0  # 0 -> 2 * max_rank, EXACT_SAMPLING -> every non-member row
    knn_k: int = 32
    near_blocksize: int = 2
    far_blocksize: int = 4
    coarsen_p: int = 8
    coarsen_agg: int = 2
    threads: int = 0
    skip_near: bool = False  # leave dgen empty: Evaluator.generated() builds D on the device

    def to_native(self) -> N.BuildSpec:
        s = N.BuildSpec()
        N.hmxb().hmxb_spec_default(C.byref(s))
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "points":
                v = POINTS[v]
            elif f.name == "kernel":
                v = KERNELS[v]
            elif f.name == "mode":
                v = MODES[v]
            elif f.name == "split":
                v = SPLITS[v]
            setattr(s, f.name, v)
        return s


@dataclass
class Instance:
    spec: InstanceSpec
    cds: CDS
    stats: dict = field(default_factory=dict)
    _handle: object = None

    def points(self) -> np.ndarray:
        ptr = C.POINTER(C.c_double)()
        n, d = C.c_uint64(), C.c_uint32()
        N.hmxb().hmxb_points(self._handle, C.byref(ptr), C.byref(n), C.byref(d))
        return np.ctypeslib.as_array(ptr, shape=(n.value, d.value)).copy()

    def dense_rows(self, rows: np.ndarray, w: np.ndarray) -> np.ndarray:
        """Exact (K W)[rows, :] — the dense error oracle of executor.cpp:405-476."""
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        wf = np.asfortranarray(w, dtype=np.float64)
        out = np.zeros((rows.shape[0], wf.shape[1]), dtype=np.float64, order="F")
        rc = N.hmxb().hmxb_dense_rows(self._handle, rows.ctypes.data_as(C.POINTER(C.c_uint32)), rows.shape[0],
                                      wf.ctypes.data_as(C.c_void_p), wf.shape[1], wf.shape[0],
                                      out.ctypes.data_as(C.c_void_p), max(1, rows.shape[0]))
        if rc:
            raise ValueError(N.last_error(N.hmxb(), "hmxb"))
        return out

    def close(self) -> None:
        if self._handle:
            self.cds._cache.clear()
            N.hmxb().hmxb_free(self._handle)
            self._handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def build_instance(spec: InstanceSpec) -> Instance:
    lib = N.hmxb()
    h = C.c_void_p()
    ns = spec.to_native()
    rc = lib.hmxb_build(C.byref(ns), C.byref(h))
    if rc:
        raise ValueError(N.last_error(lib, "hmxb"))
    v = N.CdsView()
    lib.hmxb_view(h, C.byref(v))
    st = N.BuildStats()
    lib.hmxb_stats(h, C.byref(st))
    stats = {name: getattr(st, name) for name, _ in N.BuildStats._fields_}
    inst = Instance(spec=spec, cds=None, stats=stats, _handle=h)  # type: ignore[arg-type]
    inst.cds = CDS.from_view(v, owner=inst)
    return inst


# BASELINE.json configs (index 1..5); "q" is the W column count the metric is quoted on.
CONFIGS: dict[str, tuple[InstanceSpec, int]] = {
    "cfg1-hss": (InstanceSpec(n=4096, d=3, points="uniform", seed=42, kernel="gaussian", h=0.5, leaf=128,
                              mode="hss", max_rank=64, tol=1e-5), 64),
    "cfg2-h2b": (InstanceSpec(n=32768, d=8, points="mixture", seed=42, kernel="gaussian", h=1.0, leaf=128,
                              mode="budget", budget=0.03, max_rank=128, tol=1e-5), 256),
    "cfg3-h2b": (InstanceSpec(n=65536, d=28, points="normal", seed=42, kernel="gaussian", h=3.0, leaf=256,
                              mode="budget", budget=0.03, max_rank=256, tol=1e-7), 1024),
    "cfg4-h2b": (InstanceSpec(n=131072, d=64, points="quantized", levels=16, seed=42, kernel="exponential",
                              h=2.0, leaf=256, mode="budget", budget=0.05, max_rank=256, tol=1e-5), 512),
    "cfg5-hss": (InstanceSpec(n=262144, d=3, points="uniform", seed=42, kernel="gaussian", h=0.1, leaf=256,
                              mode="hss", max_rank=128, tol=1e-6), 2048),
    "cfg5-h2b": (InstanceSpec(n=262144, d=3, points="uniform", seed=42, kernel="gaussian", h=0.1, leaf=256,
                              mode="budget", budget=0.03, max_rank=128, tol=1e-6), 2048),
}


def config(name: str, **overrides) -> tuple[InstanceSpec, int]:
    spec, q = CONFIGS[name]
    spec = InstanceSpec(**{f.name: getattr(spec, f.name) for f in fields(spec)})
    q = overrides.pop("q", q)
    for k, v in overrides.items():
        setattr(spec, k, v)
    return spec, q
