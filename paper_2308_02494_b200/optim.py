"""Loss gradients, masked Adam and the finite-difference harness.

Mirror of the reference ``apmg.optim`` API (optim.py:1-233).  The reconstruction
loss reaches the grids and decoder only; the density loss reaches the top three
transform rows only.  Both run as fused sm_100a kernels:

* ``recon_loss_and_grads`` -> one persistent kernel per batch: encode 64-point
  tiles into shared memory, decoder forward/backward on the tile, per-CTA dW
  accumulation, atomic scatter of feature gradients into channel-last grids,
  then a deterministic dW/loss reduction (optim.py:102-155).
* ``density_loss_and_grads`` -> the four-pass fp64 density pipeline
  (optim.py:158-200).
* ``adam_step`` -> masked elementwise Adam (optim.py:47-73).

Grid gradients are accumulated with float atomics, so their summation order
(and last bits) vary run to run; parity is per-tensor within 1e-3 relative.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .density import DensityError
from .model import ApmgModel

__all__ = ["AdamState", "adam_step", "recon_loss_and_grads", "density_loss_and_grads", "finite_diff_check"]

BETA1 = 0.9
BETA2 = 0.99
ADAM_GUARD = 1e-8


class AdamState:
    """First/second moments and the step counter of a named parameter set (optim.py:38-44)."""

    def __init__(self, params: dict):
        self.m = {k: np.zeros_like(v) for k, v in params.items()}
        self.v = {k: np.zeros_like(v) for k, v in params.items()}
        self.t = 0


def adam_step(params: dict, grads: dict, state: AdamState, lr: float) -> None:
    """One bias-corrected, masked Adam update in place (optim.py:47-73).

    Entries whose gradient is exactly zero keep p, m and v untouched."""
    state.t += 1
    bc1 = 1.0 - BETA1 ** state.t
    bc2 = 1.0 - BETA2 ** state.t
    for key, p in params.items():
        g = grads[key]
        if g.shape != p.shape:
            raise ValueError(f"gradient shape {g.shape} != parameter shape {p.shape} for {key!r}")
        dt = p.dtype
        if dt not in (np.float32, np.float64):
            raise TypeError(f"unsupported parameter dtype {dt}")
        pd = L.to_device(p, dt)
        gd = L.to_device(np.asarray(g), dt)
        md = L.to_device(state.m[key], dt)
        vd = L.to_device(state.v[key], dt)
        L.check(L.lib().apmg_adam_step(L.dtype_code(dt), L.ptr(pd), L.ptr(gd), L.ptr(md), L.ptr(vd), int(p.size),
                                       float(lr), float(bc1), float(bc2), L.stream_handle()), "adam_step")
        p[...] = L.to_host(pd).reshape(p.shape)
        state.m[key][...] = L.to_host(md).reshape(p.shape)
        state.v[key][...] = L.to_host(vd).reshape(p.shape)


def recon_loss_dev(dm, coords_dev, targets_dev):
    """Device-level recon step: returns (loss f64 tensor, sq tensor, d_grids_cl, dw1, dw2, dw3)."""
    n = int(targets_dev.shape[0])
    cfg = dm.config
    dt = dm.np_dtype
    d, h, w = cfg.resolution
    sq = L.empty((n,), dt)
    loss = L.empty((1,), np.float64)
    dgrid = L.zeros((cfg.grids, d, h, w, cfg.channels), dt)
    dw1 = L.empty((64, cfg.feature_len), dt)
    dw2 = L.empty((64, 64), dt)
    dw3 = L.empty((1, 64), dt)
    ws = L.workspace(L.lib().apmg_recon_workspace_bytes(C.byref(dm.desc), n))
    grads = (C.c_void_p * 4)(dgrid.data_ptr(), dw1.data_ptr(), dw2.data_ptr(), dw3.data_ptr())
    L.check(L.lib().apmg_recon_loss_grads(C.byref(dm.desc), L.ptr(coords_dev), L.ptr(targets_dev), n, L.ptr(sq),
                                          L.ptr(loss), grads, L.ptr(ws), ws.numel(), L.stream_handle()),
            "recon_loss_and_grads")
    return loss, sq, dgrid, dw1, dw2, dw3


def recon_loss_and_grads(model: ApmgModel, coords, targets):
    """Mean-squared reconstruction loss, per-point squared errors and grads for
    grids/w1/w2/w3 (no 'transforms' key) (optim.py:102-155)."""
    targets = np.asarray(targets, dtype=model.dtype).ravel()
    if targets.size < 1:
        raise ValueError("empty batch")
    coords = np.atleast_2d(np.asarray(coords, dtype=model.dtype))
    if len(coords) != targets.size:
        raise ValueError(f"{len(coords)} coordinates but {targets.size} targets")
    dm = model.device()
    loss, sq, dgrid, dw1, dw2, dw3 = recon_loss_dev(dm, L.to_device(coords), L.to_device(targets))
    d_grids = np.ascontiguousarray(np.moveaxis(L.to_host(dgrid), -1, 1))
    grads = {"grids": d_grids, "w1": L.to_host(dw1), "w2": L.to_host(dw2), "w3": L.to_host(dw3)}
    return float(loss.item()), L.to_host(sq), grads


def density_loss_and_grads(model: ApmgModel, coords, errors):
    """Density KL loss and its gradient for the top three transform rows (optim.py:158-200)."""
    c64 = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    errors = np.asarray(errors, dtype=np.float64).ravel()
    if len(c64) < 2 or errors.size != len(c64):
        raise ValueError("density batch needs >= 2 coordinates with matching errors")
    dm = model.device()
    coords_m = L.to_device(np.asarray(coords, dtype=model.dtype).reshape(-1, 3))
    n = len(c64)
    loss = L.empty((1,), np.float64)
    total = L.empty((1,), np.float64)
    dtf = L.zeros((model.config.grids, 4, 4), model.dtype)
    ws = L.workspace(L.lib().apmg_density_workspace_bytes(model.config.grids, n))
    errors_d = L.to_device(errors)
    L.check(L.lib().apmg_density_loss_grads(C.byref(dm.desc), L.ptr(coords_m), L.ptr(errors_d), n,
                                            L.ptr(loss), L.ptr(dtf), L.ptr(total), L.ptr(ws), ws.numel(),
                                            L.stream_handle()), "density_loss_and_grads")
    if not float(total.item()) > 0.0:
        raise DensityError("degenerate batch: feature density sums to zero")
    return float(loss.item()), {"transforms": L.to_host(dtf)}


def finite_diff_check(loss_and_grads_fn, params: dict, step: float, samples_per_tensor: int = 50,
                      rng: np.random.Generator | None = None) -> float:
    """Max relative |analytic - central FD| over sampled coordinates (optim.py:203-233).
    Host orchestration around a user loss function; the losses themselves run on the GPU."""
    if step <= 0:
        raise ValueError("finite-difference step must be positive")
    if rng is None:
        rng = np.random.Generator(np.random.Philox(0))
    _, grads = loss_and_grads_fn(params)
    worst = 0.0
    for key, base in params.items():
        count = min(base.size, samples_per_tensor)
        picks = rng.choice(base.size, size=count, replace=False)
        analytic_flat = np.asarray(grads[key], dtype=np.float64).ravel()
        for idx in picks:
            shifted = {k: v.copy() for k, v in params.items()}
            shifted[key].ravel()[idx] = base.ravel()[idx] + step
            plus, _ = loss_and_grads_fn(shifted)
            shifted[key].ravel()[idx] = base.ravel()[idx] - step
            minus, _ = loss_and_grads_fn(shifted)
            numeric = (plus - minus) / (2.0 * step)
            analytic = analytic_flat[idx]
            worst = max(worst, abs(analytic - numeric) / max(abs(analytic), abs(numeric), 1e-8))
    return worst
