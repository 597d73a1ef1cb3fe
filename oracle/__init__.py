"""Parity oracle for the B200 evaluator — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs import this package, and only to check or time against it; the product package
(paper_1812_07152_b200/) never imports, links or loads anything from here.

Two checkers:
* ``build/libhmxo.so`` — hmx_oracle.c, a C restatement of the reference evaluation
  (/root/reference/proj/src/executor.cpp:23-302, dense.cpp:13-66) that reproduces the
  reference's bits (pinned in tests/test_oracle.py).
* ``_ref/libhmx_ref.so`` — the unmodified reference library compiled from
  /root/reference/proj/src by oracle/Makefile, driven through ref_capi.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields

import numpy as np

from paper_1812_07152_b200 import _native as N
from paper_1812_07152_b200.cds import CDS

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libhmxo.so")
REF_SO = os.path.join(HERE, "_ref", "libhmx_ref.so")

_libs: dict = {}


def _oracle_lib():
    if "o" not in _libs:
        lib = C.CDLL(ORACLE_SO)
        lib.hmxo_evaluate.restype = C.c_int
        lib.hmxo_evaluate.argtypes = [C.POINTER(N.CdsView), C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                      C.c_void_p, C.c_size_t]
        lib.hmxo_flops_per_col.restype = C.c_double
        lib.hmxo_flops_per_col.argtypes = [C.POINTER(N.CdsView)]
        _libs["o"] = lib
    return _libs["o"]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def _ref_lib():
    if "r" not in _libs:
        lib = C.CDLL(REF_SO)
        vp, u64, f64p = C.c_void_p, C.c_uint64, C.POINTER(C.c_double)
        sig = {
            "hmxr_spec_default": (None, [C.POINTER(RefSpec)]),
            "hmxr_instance_new": (C.c_int, [C.POINTER(RefSpec), C.POINTER(vp)]),
            "hmxr_instance_free": (None, [vp]),
            "hmxr_instance_view": (C.c_int, [vp, C.POINTER(N.CdsView)]),
            "hmxr_points": (C.c_int, [vp, C.POINTER(f64p), C.POINTER(u64), C.POINTER(u64)]),
            "hmxr_random_matrix": (C.c_int, [u64, u64, u64, vp]),
            "hmxr_evaluate": (C.c_int, [vp, vp, u64, u64, vp, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]),
            "hmxr_evaluate_ref": (C.c_int, [vp, vp, u64, u64, vp]),
            "hmxr_dense_apply": (C.c_int, [vp, vp, u64, u64, vp]),
            "hmxr_relative_error_dense": (C.c_int, [vp, vp, u64, u64, C.POINTER(C.c_double)]),
            "hmxr_cds_from_view": (C.c_int, [C.POINTER(N.CdsView), C.POINTER(vp)]),
            "hmxr_cds_free": (None, [vp]),
            "hmxr_cds_evaluate": (C.c_int, [vp, vp, u64, u64, vp, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]),
            "hmxr_save_cds": (C.c_int, [vp, C.c_char_p]),
            "hmxr_cds_save": (C.c_int, [vp, C.c_char_p]),
            "hmxr_load_cds": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
            "hmxr_cds_view": (C.c_int, [vp, C.POINTER(N.CdsView)]),
            "hmxr_save_matrix": (C.c_int, [C.c_char_p, vp, u64, u64]),
            "hmxr_load_matrix": (C.c_int, [C.c_char_p, vp, C.POINTER(u64), C.POINTER(u64)]),
            "hmxr_relative_error_vs": (C.c_int, [vp, vp, vp, u64, u64, C.c_int32, u64, C.POINTER(C.c_double)]),
            "hmxr_dense_apply_points": (C.c_int, [vp, u64, u64, C.c_int32, C.c_double, vp, u64, vp]),
            "hmxr_sample_rows": (u64, [u64, u64, vp]),
            "hmxr_samples": (C.c_int, [vp, vp, vp]),
            "hmxr_basis": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(u64), vp, vp]),
            "hmxr_compress_seconds": (C.c_double, [vp]),
            "hmxr_bases_seconds": (C.c_double, [vp, C.POINTER(C.c_uint64)]),
            "hmxr_generate_plan": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_uint32)]),
            "hmxr_mix64": (u64, [u64]),
            "hmxr_rng_fill_pm1": (None, [u64, u64, vp]),
            "hmxr_last_error": (C.c_char_p, []),
            "hmxr_hardware_workers": (C.c_uint, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _libs["r"] = lib
    return _libs["r"]


class RefNumericGuardError(RuntimeError):
    """hmx::numeric_guard_error raised inside the reference."""


def _ref_check(rc: int) -> None:
    if rc:
        msg = _ref_lib().hmxr_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 6:
            raise RefNumericGuardError(msg)
        raise RuntimeError(f"reference status {rc}: {msg}")


def oracle_evaluate(cds: CDS, w: np.ndarray) -> np.ndarray:
    """Y = K~ W by the C restatement (p = 1 semantics of hmx::evaluate)."""
    wf = np.asfortranarray(w, dtype=np.float64)
    n, q = wf.shape
    y = np.zeros((n, q), dtype=np.float64, order="F")
    v = cds.view()
    rc = _oracle_lib().hmxo_evaluate(C.byref(v), wf.ctypes.data_as(C.c_void_p), n, q, n,
                                     y.ctypes.data_as(C.c_void_p), n)
    if rc == 1:
        raise ValueError("evaluate: W row count does not match the point count")
    if rc:
        raise RuntimeError(f"oracle status {rc}")
    return y


class RefSpec(C.Structure):
    """``hmxr_spec`` — tst::InstanceSpec (proj/tests/helpers.hpp:81-99)."""

    _fields_ = [
        ("n", C.c_uint64), ("d", C.c_uint64), ("shape", C.c_int32), ("mode", C.c_int32), ("tau", C.c_double),
        ("leaf", C.c_uint32), ("kernel", C.c_int32), ("h", C.c_double), ("bacc", C.c_double),
        ("max_rank", C.c_uint32), ("sample_exact", C.c_int32), ("budget", C.c_uint32), ("knn_k", C.c_uint32),
        ("p", C.c_uint32), ("agg", C.c_uint32), ("near_bs", C.c_uint32), ("far_bs", C.c_uint32),
        ("seed", C.c_uint64),
    ]


@dataclass
class RefInstanceSpec:
    """Python face of tst::InstanceSpec; shape 0 grid2d / 1 uniform / 2 sphere, mode 0 tau / 1 hss."""

    n: int = 512
    d: int = 2
    shape: int = 1
    mode: int = 1
    tau: float = 0.0
    leaf: int = 64
    kernel: int = 0
    h: float = 1.0
    bacc: float = 1e-5
    max_rank: int = 64
    sample_exact: int = 0
    budget: int = 128
    knn_k: int = 16
    p: int = 4
    agg: int = 2
    near_bs: int = 2
    far_bs: int = 4
    seed: int = 1


class RefInstance:
    """``tst::make_instance`` run by the reference library; ``cds`` is its own CDS."""

    def __init__(self, spec: RefInstanceSpec):
        lib = _ref_lib()
        s = RefSpec()
        for f in fields(spec):
            setattr(s, f.name, getattr(spec, f.name))
        h = C.c_void_p()
        _ref_check(lib.hmxr_instance_new(C.byref(s), C.byref(h)))
        self._h = h
        self.spec = spec
        v = N.CdsView()
        lib.hmxr_instance_view(h, C.byref(v))
        self.cds = CDS.from_view(v, owner=self)

    def evaluate(self, w: np.ndarray, plan_bits: int = 0, p: int = 1) -> np.ndarray:
        return self.evaluate_timed(w, plan_bits, p)[0]

    def evaluate_timed(self, w: np.ndarray, plan_bits: int = 0, p: int = 1) -> tuple[np.ndarray, float]:
        """hmx::evaluate and its EvalStats.seconds (executor.cpp:276,289-294)."""
        wf = np.asfortranarray(w, dtype=np.float64)
        y = np.zeros(wf.shape, dtype=np.float64, order="F")
        sec = C.c_double()
        _ref_check(_ref_lib().hmxr_evaluate(self._h, wf.ctypes.data_as(C.c_void_p), wf.shape[0], wf.shape[1],
                                            y.ctypes.data_as(C.c_void_p), plan_bits, p, C.byref(sec)))
        return y, sec.value

    def generate_plan(self, p: int) -> int:
        """hmx::generate_plan on the instance's tree, blocks and coarsening (lowering bits)."""
        bits = C.c_uint32()
        _ref_check(_ref_lib().hmxr_generate_plan(self._h, p, C.byref(bits)))
        return int(bits.value)

    def evaluate_reference(self, w: np.ndarray) -> np.ndarray:
        wf = np.asfortranarray(w, dtype=np.float64)
        y = np.zeros(wf.shape, dtype=np.float64, order="F")
        _ref_check(_ref_lib().hmxr_evaluate_ref(self._h, wf.ctypes.data_as(C.c_void_p), wf.shape[0], wf.shape[1],
                                                y.ctypes.data_as(C.c_void_p)))
        return y

    def dense_apply(self, w: np.ndarray) -> np.ndarray:
        wf = np.asfortranarray(w, dtype=np.float64)
        y = np.zeros(wf.shape, dtype=np.float64, order="F")
        _ref_check(_ref_lib().hmxr_dense_apply(self._h, wf.ctypes.data_as(C.c_void_p), wf.shape[0], wf.shape[1],
                                               y.ctypes.data_as(C.c_void_p)))
        return y

    def relative_error_dense(self, w: np.ndarray) -> float:
        wf = np.asfortranarray(w, dtype=np.float64)
        eps = C.c_double()
        _ref_check(_ref_lib().hmxr_relative_error_dense(self._h, wf.ctypes.data_as(C.c_void_p), wf.shape[0],
                                                        wf.shape[1], C.byref(eps)))
        return eps.value

    def relative_error_vs(self, y_approx: np.ndarray, w: np.ndarray, mode: int, seed: int = 0) -> float:
        """hmx::relative_error_vs with this instance's kernel and points (mode 0 dense, 1 sampled)."""
        ya = np.asfortranarray(y_approx, dtype=np.float64)
        wf = np.asfortranarray(w, dtype=np.float64)
        eps = C.c_double()
        _ref_check(_ref_lib().hmxr_relative_error_vs(self._h, ya.ctypes.data_as(C.c_void_p),
                                                     wf.ctypes.data_as(C.c_void_p), wf.shape[0], wf.shape[1], mode,
                                                     seed, C.byref(eps)))
        return eps.value

    def samples(self) -> tuple[np.ndarray, np.ndarray]:
        """SampleInfo rows per node as CSR (sample_ptr[num_nodes + 1], sample_idx)."""
        nn = self.cds.num_nodes
        ptr = np.zeros(nn + 1, dtype=np.uint64)
        _ref_lib().hmxr_samples(self._h, ptr.ctypes.data_as(C.c_void_p), None)
        idx = np.zeros(int(ptr[-1]), dtype=np.uint32)
        _ref_lib().hmxr_samples(self._h, None, idx.ctypes.data_as(C.c_void_p))
        return ptr, idx

    def basis(self, node: int) -> tuple[int, np.ndarray, np.ndarray]:
        """(srank, skeleton point indices, V as rows x srank) of the reference's compress."""
        sr, rows = C.c_uint32(), C.c_uint64()
        _ref_check(_ref_lib().hmxr_basis(self._h, node, C.byref(sr), C.byref(rows), None, None))
        skel = np.zeros(sr.value, dtype=np.uint32)
        v = np.zeros((rows.value, sr.value), dtype=np.float64, order="F")
        _ref_check(_ref_lib().hmxr_basis(self._h, node, C.byref(sr), C.byref(rows), skel.ctypes.data_as(C.c_void_p),
                                         v.ctypes.data_as(C.c_void_p)))
        return sr.value, skel, v

    def points(self) -> np.ndarray:
        p, n, d = C.POINTER(C.c_double)(), C.c_uint64(), C.c_uint64()
        _ref_lib().hmxr_points(self._h, C.byref(p), C.byref(n), C.byref(d))
        return np.ctypeslib.as_array(p, shape=(n.value, d.value)).copy()

    def save_cds(self, path: str) -> None:
        """hmx::save_cds of the reference's own CDS (serial.cpp:271-277)."""
        _ref_check(_ref_lib().hmxr_save_cds(self._h, os.fsencode(path)))

    def close(self):
        if self._h:
            self.cds._cache.clear()
            _ref_lib().hmxr_instance_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class RefCds:
    """The reference ``evaluate`` over any CDS (rebuilt as an hmx::CDS from the view), or
    over a CDS the reference read from disk (``RefCds.load``, hmx::load_cds)."""

    def __init__(self, cds: CDS | None):
        self._h = C.c_void_p()
        if cds is None:
            return
        v = cds.view()
        _ref_check(_ref_lib().hmxr_cds_from_view(C.byref(v), C.byref(self._h)))
        self.n = cds.n

    @classmethod
    def load(cls, path: str) -> "RefCds":
        rc = cls(None)
        _ref_check(_ref_lib().hmxr_load_cds(os.fsencode(path), C.byref(rc._h)))
        v = N.CdsView()
        _ref_lib().hmxr_cds_view(rc._h, C.byref(v))
        rc.cds = CDS.from_view(v, owner=rc)
        rc.n = rc.cds.n
        return rc

    def save(self, path: str) -> None:
        _ref_check(_ref_lib().hmxr_cds_save(self._h, os.fsencode(path)))

    def evaluate(self, w: np.ndarray, p: int = 1, plan_bits: int = 0) -> tuple[np.ndarray, float]:
        wf = np.asfortranarray(w, dtype=np.float64)
        y = np.zeros(wf.shape, dtype=np.float64, order="F")
        sec = C.c_double()
        _ref_check(_ref_lib().hmxr_cds_evaluate(self._h, wf.ctypes.data_as(C.c_void_p), wf.shape[0], wf.shape[1],
                                                y.ctypes.data_as(C.c_void_p), plan_bits, p, C.byref(sec)))
        return y, sec.value

    def close(self):
        if self._h:
            _ref_lib().hmxr_cds_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def ref_dense_apply(points: np.ndarray, kernel: int, h: float, w: np.ndarray) -> np.ndarray:
    """hmx::dense_apply (executor.cpp:405-429) over any points; kernel 0 gaussian, 1 invdist."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    wf = np.asfortranarray(w, dtype=np.float64)
    y = np.zeros(wf.shape, dtype=np.float64, order="F")
    _ref_check(_ref_lib().hmxr_dense_apply_points(pts.ctypes.data_as(C.c_void_p), pts.shape[0], pts.shape[1], kernel,
                                                  h, wf.ctypes.data_as(C.c_void_p), wf.shape[1],
                                                  y.ctypes.data_as(C.c_void_p)))
    return y


def ref_sample_rows(n: int, seed: int) -> np.ndarray:
    out = np.zeros(min(n, 256), dtype=np.uint32)
    _ref_lib().hmxr_sample_rows(n, seed, out.ctypes.data_as(C.c_void_p))
    return out


def ref_save_matrix(path: str, m: np.ndarray) -> None:
    """hmx::save_matrix (serial.cpp:279-285)."""
    mf = np.asfortranarray(m, dtype=np.float64)
    _ref_check(_ref_lib().hmxr_save_matrix(os.fsencode(path), mf.ctypes.data_as(C.c_void_p), mf.shape[0],
                                           mf.shape[1]))


def ref_load_matrix(path: str) -> np.ndarray:
    """hmx::load_matrix (serial.cpp:287-297)."""
    r, c = C.c_uint64(), C.c_uint64()
    _ref_check(_ref_lib().hmxr_load_matrix(os.fsencode(path), None, C.byref(r), C.byref(c)))
    out = np.zeros((r.value, c.value), dtype=np.float64, order="F")
    _ref_check(_ref_lib().hmxr_load_matrix(os.fsencode(path), out.ctypes.data_as(C.c_void_p), C.byref(r),
                                           C.byref(c)))
    return out


def ref_cli_random_w(n: int, q: int, seed: int) -> np.ndarray:
    """random_w of the reference CLI (proj/tools/hmx.cpp:117-122) composed from the
    reference's own mix64 and Rng (the tool itself needs the absent vendor libraries)."""
    lib = _ref_lib()
    out = np.zeros((n, q), dtype=np.float64, order="F")
    lib.hmxr_rng_fill_pm1(lib.hmxr_mix64(seed ^ lib.hmxr_mix64(0x77A7)), n * q, out.ctypes.data_as(C.c_void_p))
    return out


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """tst::random_matrix (helpers.hpp:53-58): uniform[-1, 1) via the reference Rng."""
    out = np.zeros((rows, cols), dtype=np.float64, order="F")
    _ref_lib().hmxr_random_matrix(rows, cols, seed, out.ctypes.data_as(C.c_void_p))
    return out


def rel_frob(a: np.ndarray, b: np.ndarray) -> float:
    """helpers.hpp:60-68."""
    num = float(np.sum((np.asarray(a) - np.asarray(b)) ** 2))
    den = float(np.sum(np.asarray(b) ** 2))
    return float(np.sqrt(num)) if den == 0.0 else float(np.sqrt(num / den))
