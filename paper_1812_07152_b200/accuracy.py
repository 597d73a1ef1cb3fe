"""The GPU error oracle: exact kernel products and the relative error of an evaluation.

Mirrors /root/reference/proj/include/hmx/executor.hpp:60-76 and kernel.hpp:
* ``dense_apply(kernel, points, w)`` = K W (executor.cpp:405-429);
* ``relative_error_vs(y_approx, kernel, points, w, mode, seed)`` (:431-476): every entry
  (``ErrorMode.DENSE``, n <= 16384, else ``NumericGuardError``) or 256 sampled rows;
* ``relative_error(cds, kernel, points, w, mode, seed)`` (:478-483): evaluate on the B200,
  then the error.
K is never formed on the host: ``hmxg_kernel_rows`` (include/hmxg.h) generates kernel tiles
from the points on the device and multiplies them with the evaluator's FP64 GEMM.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .cds import CDS


class NumericGuardError(RuntimeError):
    """hmx::numeric_guard_error (executor.hpp:13-16)."""


class ErrorMode(enum.IntEnum):
    DENSE = N.HMXG_ERR_DENSE
    SAMPLED = N.HMXG_ERR_SAMPLED


@dataclass(frozen=True)
class Kernel:
    """hmx::Kernel (kernel.hpp): ``gaussian`` exp(-r^2/(2h^2)), ``invdist`` 1/r (1 at r = 0),
    and the builder's ``exponential`` exp(-r/h)."""

    kind: str = "gaussian"
    h: float = 1.0

    @staticmethod
    def gaussian(h: float) -> "Kernel":
        return Kernel("gaussian", h)

    @staticmethod
    def inverse_distance() -> "Kernel":
        return Kernel("invdist", 1.0)

    @staticmethod
    def exponential(h: float) -> "Kernel":
        return Kernel("exponential", h)

    @property
    def code(self) -> int:
        return {"gaussian": N.HMXG_KERNEL_GAUSSIAN, "exponential": N.HMXG_KERNEL_EXPONENTIAL,
                "invdist": N.HMXG_KERNEL_INVDIST}[self.kind]

    def describe(self) -> str:
        return "invdist" if self.kind == "invdist" else f"{self.kind}:{self.h:f}"


def parse_kernel(spec: str) -> Kernel:
    """hmx::parse_kernel (kernel.cpp:66-78), plus ``exponential:H``."""
    if spec == "invdist":
        return Kernel.inverse_distance()
    for kind in ("gaussian", "exponential"):
        if spec.startswith(kind + ":"):
            h = float(spec[len(kind) + 1:])
            if not h > 0.0:
                raise ValueError("Gaussian kernel: bandwidth must be > 0")
            return Kernel(kind, h)
    raise ValueError(f"unknown kernel spec: {spec} (expected gaussian:H or invdist)")


def _check(rc: int) -> None:
    if rc == N.HMXG_OK:
        return
    from .executor import HmxgError

    msg = N.last_error(N.hmxg(), "hmxg")
    if rc == N.HMXG_EINVAL:
        raise ValueError(msg)
    if rc == N.HMXG_EGUARD:
        raise NumericGuardError(msg)
    raise HmxgError(rc, msg)


def sample_rows(n: int, seed: int) -> np.ndarray:
    """The rows relative_error_vs samples (executor.cpp:446-451)."""
    out = np.zeros(min(n, 256), dtype=np.uint32)
    if out.size:
        N.hmxg().hmxg_sample_rows(n, seed, out.ctypes.data_as(C.c_void_p))
    return out


class DevicePoints:
    """A point set resident on one device with its kernel (``hmxg_points``)."""

    def __init__(self, points: np.ndarray, kernel: Kernel, device: int = 0):
        from .executor import Context

        pts = np.ascontiguousarray(points, dtype=np.float64)
        if pts.ndim != 2:
            raise ValueError("points must be an n x d array")
        self.n, self.d = pts.shape
        self.kernel = kernel
        self.ctx = Context((device,))
        h = C.c_void_p()
        _check(N.hmxg().hmxg_points_upload(self.ctx.handle, pts.ctypes.data_as(C.c_void_p), self.n, self.d,
                                           kernel.code, kernel.h, C.byref(h)))
        self._h = h

    def kernel_rows(self, rows: np.ndarray | None, w: np.ndarray, stats=None) -> np.ndarray:
        """K(x_rows, :) W for host W (n x q); ``rows=None``: every row (dense_apply)."""
        if w.ndim != 2 or w.shape[0] != self.n:
            raise ValueError("dense_apply: W row count mismatch")
        wf = np.asfortranarray(w, dtype=np.float64)
        q = wf.shape[1]
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.uint32)
        nr = self.n if r is None else r.size
        y = np.zeros((nr, q), dtype=np.float64, order="F")
        st = N.Stats()
        _check(N.hmxg().hmxg_kernel_rows(self._h, None if r is None else r.ctypes.data_as(C.c_void_p), nr,
                                         wf.ctypes.data_as(C.c_void_p), self.n, q, self.n,
                                         y.ctypes.data_as(C.c_void_p), max(nr, 1), 0, None, C.byref(st)))
        if stats is not None:
            stats.seconds, stats.device_ms, stats.launches = st.seconds, st.device_ms, st.launches
        return y

    def kernel_rows_device(self, rows: np.ndarray | None, w_ptr: int, y_ptr: int, q: int, ldw: int | None = None,
                           ldy: int | None = None, stream: int = 0, stats=None) -> None:
        """Device-pointer form: W (n x q, ldw) and Y (nrows x q, ldy) live on the device."""
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.uint32)
        nr = self.n if r is None else r.size
        st = N.Stats()
        _check(N.hmxg().hmxg_kernel_rows(self._h, None if r is None else r.ctypes.data_as(C.c_void_p), nr,
                                         C.c_void_p(w_ptr), self.n, q, ldw or self.n, C.c_void_p(y_ptr),
                                         ldy or max(nr, 1), N.HMXG_F_DEVICE_PTRS,
                                         C.c_void_p(stream) if stream else None, C.byref(st)))
        if stats is not None:
            stats.seconds, stats.device_ms, stats.launches = st.seconds, st.device_ms, st.launches

    def dense_apply(self, w: np.ndarray) -> np.ndarray:
        return self.kernel_rows(None, w)

    def relative_error_vs(self, y_approx: np.ndarray, w: np.ndarray, mode: ErrorMode = ErrorMode.SAMPLED,
                          seed: int = 0) -> float:
        if y_approx.shape[0] != self.n or w.shape[0] != self.n or y_approx.shape[1] != w.shape[1]:
            raise ValueError("relative_error: shape mismatch")
        ya = np.asfortranarray(y_approx, dtype=np.float64)
        wf = np.asfortranarray(w, dtype=np.float64)
        eps = C.c_double()
        _check(N.hmxg().hmxg_relative_error(self._h, ya.ctypes.data_as(C.c_void_p), self.n,
                                            wf.ctypes.data_as(C.c_void_p), self.n, wf.shape[1], self.n, int(mode),
                                            seed, 0, C.byref(eps)))
        return eps.value

    def relative_error_vs_device(self, y_ptr: int, w_ptr: int, q: int, mode: ErrorMode = ErrorMode.SAMPLED,
                                 seed: int = 0, ldy: int | None = None, ldw: int | None = None) -> float:
        eps = C.c_double()
        _check(N.hmxg().hmxg_relative_error(self._h, C.c_void_p(y_ptr), ldy or self.n, C.c_void_p(w_ptr), self.n, q,
                                            ldw or self.n, int(mode), seed, N.HMXG_F_DEVICE_PTRS, C.byref(eps)))
        return eps.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.hmxg().hmxg_points_free(self._h)
            self._h = None
        self.ctx.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def dense_apply(kernel: Kernel, points: np.ndarray, w: np.ndarray, device: int = 0) -> np.ndarray:
    """hmx::dense_apply on the B200."""
    with DevicePoints(points, kernel, device) as dp:
        return dp.dense_apply(w)


def relative_error_vs(y_approx: np.ndarray, kernel: Kernel, points: np.ndarray, w: np.ndarray,
                      mode: ErrorMode = ErrorMode.SAMPLED, seed: int = 0, device: int = 0) -> float:
    """hmx::relative_error_vs on the B200 (q == 0 gives 0 by convention)."""
    if mode == ErrorMode.DENSE and points.shape[0] > 16384:
        raise NumericGuardError("dense error oracle limited to n <= 16384; use sampled mode")
    with DevicePoints(points, kernel, device) as dp:
        return dp.relative_error_vs(y_approx, w, mode, seed)


def relative_error(cds: CDS, kernel: Kernel, points: np.ndarray, w: np.ndarray,
                   mode: ErrorMode = ErrorMode.SAMPLED, seed: int = 0, device: int = 0) -> float:
    """hmx::relative_error: evaluate the CDS on the B200, then compare with exact K W."""
    from .executor import evaluate

    y = evaluate(cds, None, w, devices=(device,))
    return relative_error_vs(y, kernel, points, w, mode, seed, device)
