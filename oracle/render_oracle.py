"""CPU oracle for the renderer field-query path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference renderer (/root/reference/pkg/src/apmg/render.py) for
the GPU path in ``paper_2308_02494_b200.render``: ray/box hits, transfer-function baking and
lookup, front-to-back compositing and the per-ray sample points.  Pinned against the
reference's own outputs in tests/golden/render.npz (tests/golden/make_golden.py, gen_render)
by tests/test_oracle.py.  Only ``tests/`` may import it.
"""
from __future__ import annotations

import numpy as np

LUT_SIZE = 256


def rays(eye, look_at, up, fov_deg, width, height):
    """Pixel ray directions (render.py:202-220): row-major, pixel centres, unit length."""
    eye = np.asarray(eye, dtype=np.float64)
    f = np.asarray(look_at, dtype=np.float64) - eye
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, dtype=np.float64))
    r = r / np.linalg.norm(r)
    u_axis = np.cross(r, f)
    th = np.tan(np.radians(fov_deg) * 0.5)
    sx = (np.arange(width) + 0.5) / width * 2.0 - 1.0
    sy = 1.0 - (np.arange(height) + 0.5) / height * 2.0
    gu, gv = np.meshgrid(sx * th * (width / height), sy * th)
    d = f + gu[..., None] * r + gv[..., None] * u_axis
    return eye, (d / np.linalg.norm(d, axis=-1, keepdims=True)).reshape(-1, 3)


def box_hits(origin, dirs):
    """Slab test against [-1, 1]^3 (render.py:223-246); parallel rays hit only from inside
    their slab; rays starting inside enter at t = 0."""
    origin = np.asarray(origin, dtype=np.float64)
    dirs = np.asarray(dirs, dtype=np.float64)
    lo = np.full(len(dirs), -np.inf)
    hi = np.full(len(dirs), np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        for k in range(3):
            dk, ok = dirs[:, k], origin[k]
            a, b = (-1.0 - ok) / dk, (1.0 - ok) / dk
            par = dk == 0.0
            inside = abs(ok) <= 1.0
            lo = np.where(par, lo if inside else np.inf, np.maximum(lo, np.minimum(a, b)))
            hi = np.where(par, hi if inside else -np.inf, np.minimum(hi, np.maximum(a, b)))
    enter = np.maximum(lo, 0.0)
    return enter, hi, (hi > enter) & (hi > 0.0) & np.isfinite(enter)


def bake_lut(color_points, opacity_points):
    """256 x RGBA f32 table of the piecewise-linear maps (render.py:115-124)."""
    cps = sorted((float(p), tuple(float(c) for c in rgb)) for p, rgb in color_points)
    ops = sorted((float(p), float(a)) for p, a in opacity_points)
    x = np.linspace(0.0, 1.0, LUT_SIZE)
    lut = np.empty((LUT_SIZE, 4), dtype=np.float32)
    for k in range(3):
        lut[:, k] = np.interp(x, [p for p, _ in cps], [c[k] for _, c in cps])
    lut[:, 3] = np.interp(x, [p for p, _ in ops], [a for _, a in ops])
    return lut


def tf_lookup(lut, window, values, vmin, vmax):
    """Normalise, window-remap, clamp and lerp the LUT in float32 (render.py:126-138)."""
    v = np.asarray(values, dtype=np.float32)
    nrm = (v - np.float32(vmin)) / np.float32(vmax - vmin) if vmax > vmin else np.zeros_like(v)
    lo, hi = window
    w = np.clip((nrm - np.float32(lo)) / np.float32(hi - lo), 0.0, 1.0)
    pos = w * (LUT_SIZE - 1)
    i = np.minimum(pos.astype(np.intp), LUT_SIZE - 2)
    t = (pos - i).astype(np.float32)[..., None]
    return lut[i] * (1.0 - t) + lut[i + 1] * t


def composite(rgba, steps, reference_step, background, early_exit):
    """Front-to-back emission-absorption with step-corrected opacity and early exit
    (render.py:229-264); rgba [n][S][4] f32, steps [n] f32."""
    n, S, _ = rgba.shape
    col = np.zeros((n, 3), dtype=np.float32)
    acc = np.zeros(n, dtype=np.float32)
    expo = np.asarray(steps, dtype=np.float32)[:, None] / np.float32(reference_step)
    corr = 1.0 - np.power(1.0 - rgba[:, :, 3], expo)
    for s in range(S):
        live = np.ones(n, dtype=bool) if early_exit is None else acc < early_exit
        c = (1.0 - acc) * corr[:, s]
        col = np.where(live[:, None], col + c[:, None] * rgba[:, s, :3], col)
        acc = np.where(live, acc + c, acc)
    bg = np.asarray(background, dtype=np.float32)
    rest = (1.0 - acc) * bg[3]
    return np.concatenate([col + rest[:, None] * bg[:3], (acc + rest)[:, None]], axis=1).astype(np.float32)


def ray_samples(origin, dirs, enter, exit_t, samples):
    """Sample points of hit rays (render.py:286-290): t = (s + 0.5) dt + enter, clipped, f32."""
    dt = (exit_t - enter) / samples
    t = (np.arange(samples) + 0.5)[None, :] * dt[:, None] + enter[:, None]
    p = np.asarray(origin, dtype=np.float64)[None, None, :] + t[:, :, None] * dirs[:, None, :]
    return np.clip(p, -1.0, 1.0).reshape(-1, 3).astype(np.float32), dt


def render(field_forward, vmin, vmax, origin, dirs, lut, window, samples, reference_step,
           background=(0.0, 0.0, 0.0, 1.0), early_exit=0.99):
    """_render_rays + render_frame (render.py:277-305) for a host field callable."""
    enter, exit_t, hit = box_hits(origin, dirs)
    out = np.empty((len(dirs), 4), dtype=np.float32)
    out[~hit] = np.asarray(background, dtype=np.float32)
    idx = np.nonzero(hit)[0]
    if len(idx):
        pts, dt = ray_samples(origin, dirs[idx], enter[idx], exit_t[idx], samples)
        vals = np.asarray(field_forward(pts), dtype=np.float32)
        rgba = tf_lookup(lut, window, vals, vmin, vmax).reshape(len(idx), samples, 4)
        out[idx] = composite(rgba, dt.astype(np.float32), reference_step, background, early_exit)
    return out
