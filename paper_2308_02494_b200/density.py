"""Flat-top feature density, error-warped target and the density KL loss.

Mirror of the reference ``apmg.density`` API (density.py:1-180).  All density
math is float64 and runs in the library's density kernels; per-grid exponents
above ``EXP_CLAMP`` contribute exactly zero.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib as L

__all__ = [
    "EPSILON", "EXP_CLAMP", "TARGET_FLOOR", "DensityBatch", "DensityError", "flat_top", "feature_density",
    "feature_density_terms", "scale_density", "target_density", "density_loss", "cofactor_matrices",
]

EPSILON = 1e-8
EXP_CLAMP = 700.0
TARGET_FLOOR = 1e-300


class DensityError(Exception):
    pass


@dataclass(frozen=True)
class FlatTopParams:
    p: int

    def __post_init__(self):
        if self.p < 1:
            raise DensityError("flat-top strength p must be >= 1")


def flat_top(t, p: int):
    """Unit flat-top gaussian exp(-t^(2p)/2) (density.py:57-69).  A 1-D plotting/documentation
    helper of the reference; the density model itself uses the bump without the 1/2."""
    if p < 1:
        raise DensityError("flat-top strength p must be >= 1")
    t = np.asarray(t, dtype=np.float64)
    with np.errstate(over="ignore"):
        q = 0.5 * (t * t) ** p
    return np.where(q > EXP_CLAMP, 0.0, np.exp(-np.minimum(q, EXP_CLAMP)))


def cofactor_matrices(a: np.ndarray) -> np.ndarray:
    """Cofactors of stacked 3x3 matrices: row i = cross of the other two rows (density.py:72-80)."""
    return np.stack([np.cross(a[:, 1], a[:, 2]), np.cross(a[:, 2], a[:, 0]), np.cross(a[:, 0], a[:, 1])], axis=1)


def _dev_f64(x):
    if hasattr(x, "is_cuda"):
        return None, x.to(dtype=L.require_cuda().float64).contiguous()
    arr = np.asarray(x, dtype=np.float64)
    return arr, L.to_device(arr)


def _transforms_dev(transforms):
    tf = np.asarray(transforms)
    dt = np.float32 if tf.dtype == np.float32 else np.float64
    return dt, L.to_device(tf, dt)


def feature_density_terms(transforms, pts, p: int):
    """(local (M,N,3), dets (M,), bumps (M,N), rho (N,)) in float64 (density.py:83-103)."""
    dt, tf = _transforms_dev(transforms)
    m = tf.shape[0]
    host, x = _dev_f64(np.atleast_2d(np.asarray(pts, dtype=np.float64)) if not hasattr(pts, "is_cuda") else pts)
    n = int(x.shape[0])
    local = L.empty((m, n, 3), np.float64)
    dets = L.empty((m,), np.float64)
    bumps = L.empty((m, n), np.float64)
    rho = L.empty((n,), np.float64)
    L.check(L.lib().apmg_density_terms(L.dtype_code(dt), L.ptr(tf), m, int(p), L.ptr(x), n, L.ptr(local), L.ptr(dets),
                                       L.ptr(bumps), L.ptr(rho), L.stream_handle()), "density_terms")
    return tuple(L.to_host(t) for t in (local, dets, bumps, rho))


def feature_density_dev(transforms, x_dev, p: int):
    dt, tf = _transforms_dev(transforms)
    n = int(x_dev.shape[0])
    rho = L.empty((n,), np.float64)
    L.check(L.lib().apmg_feature_density(L.dtype_code(dt), L.ptr(tf), tf.shape[0], int(p), L.ptr(x_dev), n,
                                         L.ptr(rho), L.stream_handle()), "feature_density")
    return rho


def feature_density(transforms, pts, p: int) -> np.ndarray:
    """rho(x) = sum_i |det A_i| exp(-sum_d local_d^(2p)) on the GPU (density.py:106-108)."""
    if p < 1:
        raise DensityError("flat-top strength p must be >= 1")
    _, x = _dev_f64(np.atleast_2d(np.asarray(pts, dtype=np.float64)))
    return L.to_host(feature_density_dev(transforms, x, p))


def _sum_dev(x_dev):
    n = int(x_dev.shape[0])
    out = L.empty((1,), np.float64)
    ws = L.workspace(L.lib().apmg_sum_workspace_bytes(n))
    L.check(L.lib().apmg_sum_f64(L.ptr(x_dev), n, L.ptr(out), L.ptr(ws), ws.numel(), L.stream_handle()), "sum")
    return out


def scale_density(rho) -> np.ndarray:
    """rho / sum(rho) (density.py:111-117)."""
    _, r = _dev_f64(rho)
    total = _sum_dev(r)
    if not float(total.item()) > 0.0:
        raise DensityError("degenerate batch: feature density sums to zero")
    out = L.empty(tuple(r.shape), np.float64)
    L.check(L.lib().apmg_scale_f64(L.ptr(r), int(r.numel()), L.ptr(total), L.ptr(out), L.stream_handle()), "scale")
    return L.to_host(out)


def target_density(rho_scaled, errors, mean_error: float, epsilon: float = EPSILON) -> np.ndarray:
    """exp(((h_bar+eps)/(h+eps)) log(rho_s+eps)), exact at unit exponent, floored (density.py:120-137)."""
    _, rs = _dev_f64(rho_scaled)
    _, e = _dev_f64(np.broadcast_to(np.asarray(errors, dtype=np.float64), tuple(rs.shape)))
    out = L.empty(tuple(rs.shape), np.float64)
    L.check(L.lib().apmg_target_density(L.ptr(rs), L.ptr(e), int(rs.numel()), float(mean_error), float(epsilon),
                                        L.ptr(out), L.stream_handle()), "target_density")
    return L.to_host(out)


def density_loss(rho_scaled, rho_star, epsilon: float = EPSILON) -> float:
    """(1/N) sum rho_s (log(rho_s+eps) - log rho*) (density.py:140-148)."""
    rs_h = np.asarray(rho_scaled, dtype=np.float64)
    st_h = np.asarray(rho_star, dtype=np.float64)
    if rs_h.shape != st_h.shape or rs_h.size < 1:
        raise DensityError("rho_scaled and rho_star must be equal-length, non-empty")
    rs, st = L.to_device(rs_h.ravel()), L.to_device(st_h.ravel())
    terms = L.empty((rs.numel(),), np.float64)
    L.check(L.lib().apmg_density_loss_terms(L.ptr(rs), L.ptr(st), int(rs.numel()), float(epsilon), L.ptr(terms),
                                            L.stream_handle()), "density_loss")
    return float(_sum_dev(terms).item()) / rs_h.size


@dataclass(frozen=True)
class DensityBatch:
    """One training batch's density state with its invariants (density.py:151-179)."""
    coords: np.ndarray
    rho: np.ndarray
    rho_scaled: np.ndarray
    errors: np.ndarray
    mean_error: float
    epsilon: float = EPSILON

    def __post_init__(self):
        if (self.rho_scaled < 0).any():
            raise DensityError("rho_scaled has negative entries")
        if abs(self.rho_scaled.sum() - 1.0) > 1e-6:
            raise DensityError("rho_scaled does not sum to 1")
        if abs(float(self.errors.mean()) - self.mean_error) > 1e-9:
            raise DensityError("mean_error is not the mean of errors")

    @classmethod
    def from_model_state(cls, transforms, coords, errors, p: int) -> "DensityBatch":
        rho = feature_density(transforms, coords, p)
        errs = np.asarray(errors, dtype=np.float64)
        return cls(coords=np.asarray(coords), rho=rho, rho_scaled=scale_density(rho), errors=errs,
                   mean_error=float(errs.mean()))
