"""CPU oracle for the APMGSRN train-and-query hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(/root/reference/pkg/src/apmg, pure numpy).  It exists so the CUDA path can
be checked on seeded inputs of any size, and so ``bench.py --impl reference``
can time the reference algorithm on the GPU box (where /root/reference does not
exist).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
reference / cpu_baseline legs may import it; the product package never does.

Pinning: every function here is checked against fixtures produced by running
the reference itself (tests/golden/make_golden.py -> tests/golden/*.npz) in
tests/test_oracle.py.  Where the reference is elementwise numpy (volume
sampling, interpolation terms, density terms, Adam, hashing, partitioning,
Philox draws) the restatement reproduces it bit for bit; where the reference
uses SIMD einsum/BLAS reductions the restatement uses the same numpy calls.

Third-party arithmetic the reference relies on: numpy (>=1.24 unpinned; 2.3.5
here): Philox4x64-10 + SeedSequence, einsum, bincount, OpenBLAS sgemm, libm
exp/log.  ``philox_block`` restates the Philox4x64-10 bijection with Python
integers so the device generator's counter/key convention is pinned
independently of numpy's C code.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------- constants
HIDDEN = 64                      # model.py:37
ADAM_B1, ADAM_B2, ADAM_EPS = 0.9, 0.99, 1e-8   # optim.py:33-35
DENS_EPS = 1e-8                  # density.py:34
DENS_CLAMP = 700.0               # density.py:35
DENS_FLOOR = 1e-300              # density.py:39
PSNR_CAP = 200.0                 # trainer.py:34


# ---------------------------------------------------------------- Philox
_PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
_PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)
_U64 = (1 << 64) - 1


def philox_key(seed: int) -> tuple[int, int]:
    """Key numpy derives for ``np.random.Philox(seed)`` (SeedSequence, 2 words).

    Follows trainer.py:175 / model.py:260, which construct Philox(seed)."""
    key = np.random.Philox(seed).state["state"]["key"]
    return int(key[0]), int(key[1])


def philox_block(counter: int, key: tuple[int, int]) -> tuple[int, int, int, int]:
    """Philox4x64-10 applied to a 256-bit counter (Random123 convention used by numpy)."""
    c = [(counter >> (64 * i)) & _U64 for i in range(4)]
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0 = (k0 + _PHILOX_W[0]) & _U64
            k1 = (k1 + _PHILOX_W[1]) & _U64
        p0 = _PHILOX_M[0] * c[0]
        p1 = _PHILOX_M[1] * c[2]
        c = [((p1 >> 64) ^ c[1] ^ k0) & _U64, p1 & _U64,
             ((p0 >> 64) ^ c[3] ^ k1) & _U64, p0 & _U64]
    return tuple(c)


def philox_raw(seed: int, start: int, count: int) -> np.ndarray:
    """Raw 64-bit words ``start .. start+count`` of Philox(seed); word j is lane j%4 of
    counter j//4 + 1 (numpy pre-increments its counter before every block)."""
    key = philox_key(seed)
    out = np.empty(count, dtype=np.uint64)
    cache = {}
    for i in range(count):
        j = start + i
        blk = j // 4 + 1
        if blk not in cache:
            cache[blk] = philox_block(blk, key)
        out[i] = cache[blk][j % 4]
    return out


def batch_coords(seed: int, iteration: int, batch: int) -> np.ndarray:
    """Iteration ``iteration``'s (batch, 3) float64 draw of rng.uniform(-1, 1) (trainer.py:189)."""
    rng = np.random.Generator(np.random.Philox(seed))
    if iteration:
        rng.random(3 * batch * iteration)  # one 64-bit word per double, same as uniform()
    return rng.uniform(-1.0, 1.0, size=(batch, 3))


# ---------------------------------------------------------------- volumes
def lattice_axis(n: int) -> np.ndarray:
    """Corner-aligned vertex coordinates of one axis (volume.py:161-165)."""
    if n == 1:
        return np.zeros(1)
    return 2.0 * np.arange(n) / (n - 1) - 1.0


def sample_volume(data: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """fp64 trilinear sampling of a (D, H, W) float32 volume (volume.py:147-199).

    Raises ValueError outside [-1, 1]^3 like Volume.sample_many raises VolumeError."""
    pts = np.asarray(pts, dtype=np.float64)
    if pts.size and (np.abs(pts) > 1.0).any():
        raise ValueError("coordinate outside [-1, 1]^3")
    d, h, w = data.shape
    base, fr, step = [], [], []
    for axis, n in enumerate((w, h, d)):
        if n == 1:
            base.append(np.zeros(len(pts), dtype=np.intp))
            fr.append(np.zeros(len(pts)))
            step.append(0)
            continue
        u = (pts[:, axis] + 1.0) * 0.5 * (n - 1)
        i0 = np.clip(np.floor(u).astype(np.intp), 0, n - 2)
        base.append(i0)
        fr.append(u - i0)
        step.append(1)
    ix, iy, iz = base
    fx, fy, fz = fr
    sx, sy, sz = step

    def at(dz, dy, dx):
        return data[iz + dz * sz, iy + dy * sy, ix + dx * sx].astype(np.float64)

    def mix(a, b, t):
        return a + t * (b - a)

    x00 = mix(at(0, 0, 0), at(0, 0, 1), fx)
    x10 = mix(at(0, 1, 0), at(0, 1, 1), fx)
    x01 = mix(at(1, 0, 0), at(1, 0, 1), fx)
    x11 = mix(at(1, 1, 0), at(1, 1, 1), fx)
    return mix(mix(x00, x10, fy), mix(x01, x11, fy), fz)


def synth_volume(dims, blobs, seed=0, background=0.0, noise=0.0) -> np.ndarray:
    """Gaussian-blob field, f64 accumulation then f32 (volume.py:275-296).

    ``blobs`` is a list of (center(3), sigma(3), amplitude).  Returns (D, H, W) f32."""
    w, h, d = (int(v) for v in dims)
    axes = [lattice_axis(w), lattice_axis(h), lattice_axis(d)]
    acc = np.full((d, h, w), float(background), dtype=np.float64)
    for center, sigma, amp in blobs:
        g = [np.exp(-((axes[a] - center[a]) ** 2) / (2.0 * sigma[a] ** 2)) for a in range(3)]
        acc += amp * g[2][:, None, None] * g[1][None, :, None] * g[0][None, None, :]
    if noise > 0.0:
        acc += np.random.Generator(np.random.Philox(seed)).uniform(-noise, noise, size=acc.shape)
    return acc.astype(np.float32)


# ---------------------------------------------------------------- model
@dataclass
class Params:
    """Model tensors in the reference layout (model.py:90): transforms (M,4,4),
    grids (M,C,D,H,W), w1 (64,M*C), w2 (64,64), w3 (1,64), plus the value range."""
    transforms: np.ndarray
    grids: np.ndarray
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray
    vmin: float = 0.0
    vmax: float = 1.0
    p: int = 10

    @property
    def dtype(self):
        return self.grids.dtype

    def copy(self) -> "Params":
        return Params(self.transforms.copy(), self.grids.copy(), self.w1.copy(), self.w2.copy(),
                      self.w3.copy(), self.vmin, self.vmax, self.p)


def grid_local(tf: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """local = pts . A^T + t (model.py:172-182).

    numpy's einsum("nk,ok->no") accumulates the 3-term k-sum as
    (p0 a0 + p1 a1) + p2 a2 for float32 but (p0 a0 + p2 a2) + p1 a1 for float64
    (its SIMD pairing differs by dtype); both are reproduced bit for bit."""
    a, t = tf[:3, :3], tf[:3, 3]
    cols = []
    for o in range(3):
        t0, t1, t2 = pts[:, 0] * a[o, 0], pts[:, 1] * a[o, 1], pts[:, 2] * a[o, 2]
        s = (t0 + t2) + t1 if pts.dtype == np.float64 else (t0 + t1) + t2
        cols.append(s + t[o])
    return np.stack(cols, axis=1)


def cell_terms(res, local):
    """Inside mask, base vertex and clipped f64 fractions per axis (model.py:198-213)."""
    d, h, w = res
    inside = np.all(np.abs(local) <= 1.0, axis=1)
    base, frac = [], []
    for axis, n in enumerate((w, h, d)):
        u = (local[:, axis] + 1.0) * 0.5 * (n - 1)
        with np.errstate(invalid="ignore"):
            i0 = np.clip(np.floor(u).astype(np.intp), 0, n - 2)
        base.append(i0)
        frac.append(np.clip(u - i0, 0.0, 1.0))
    return inside, base, frac


def interp(grid: np.ndarray, base, frac) -> np.ndarray:
    """Nested lerp, x then y then z, over all channels -> (N, C) (model.py:216-226)."""
    ix, iy, iz = base
    fx, fy, fz = frac

    def mix(a, b, t):
        return a + t * (b - a)

    lo_lo = mix(grid[:, iz, iy, ix], grid[:, iz, iy, ix + 1], fx)
    hi_lo = mix(grid[:, iz, iy + 1, ix], grid[:, iz, iy + 1, ix + 1], fx)
    lo_hi = mix(grid[:, iz + 1, iy, ix], grid[:, iz + 1, iy, ix + 1], fx)
    hi_hi = mix(grid[:, iz + 1, iy + 1, ix], grid[:, iz + 1, iy + 1, ix + 1], fx)
    return mix(mix(lo_lo, hi_lo, fy), mix(lo_hi, hi_hi, fy), fz).T


def encode(prm: Params, pts: np.ndarray, keep_terms: bool = False):
    """Grid-major concatenated features (N, M*C) (model.py:141-150, optim.py:76-89)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=prm.dtype))
    m, c = prm.grids.shape[:2]
    res = prm.grids.shape[2:]
    feats = np.zeros((len(pts), m * c), dtype=prm.dtype)
    terms = []
    for g in range(m):
        inside, base, frac = cell_terms(res, grid_local(prm.transforms[g], pts))
        vals = interp(prm.grids[g], base, frac)
        vals[~inside] = 0
        feats[:, g * c:(g + 1) * c] = vals
        if keep_terms:
            terms.append((inside, base, frac))
    return (feats, terms) if keep_terms else feats


def _rowdot(a, rows):
    return np.einsum("nk,ok->no", a, rows)


def decode_chain(prm: Params, feats: np.ndarray):
    """No-bias MLP with ReLU and value-range scaling (model.py:152-162)."""
    z1 = _rowdot(feats, prm.w1)
    h1 = np.maximum(z1, 0)
    z2 = _rowdot(h1, prm.w2)
    h2 = np.maximum(z2, 0)
    raw = _rowdot(h2, prm.w3)
    span = np.asarray(prm.vmax - prm.vmin, dtype=prm.dtype)
    out = raw[:, 0] * span + np.asarray(prm.vmin, dtype=prm.dtype)
    return z1, h1, z2, h2, out


def forward(prm: Params, pts: np.ndarray) -> np.ndarray:
    """f(x) = d(e(x)) (model.py:164-166)."""
    return decode_chain(prm, encode(prm, pts))[-1]


# ---------------------------------------------------------------- reconstruction loss
def recon_loss_and_grads(prm: Params, coords: np.ndarray, targets: np.ndarray):
    """MSE loss, per-point squared errors and grads for grids/w1/w2/w3 (optim.py:102-155)."""
    targets = np.asarray(targets, dtype=prm.dtype).ravel()
    if targets.size < 1:
        raise ValueError("empty batch")
    coords = np.atleast_2d(np.asarray(coords, dtype=prm.dtype))
    if len(coords) != targets.size:
        raise ValueError("coordinate/target count mismatch")
    feats, terms = encode(prm, coords, keep_terms=True)
    z1, h1, z2, h2, out = decode_chain(prm, feats)
    n = targets.size
    resid = out - targets
    sq = resid * resid
    loss = float(np.mean(sq, dtype=np.float64))

    span = np.asarray(prm.vmax - prm.vmin, dtype=prm.dtype)
    g_out = (resid * (np.asarray(2.0 / n, dtype=prm.dtype) * span))[:, None]
    g_w3 = g_out.T @ h2
    g_z2 = (g_out @ prm.w3) * (z2 > 0)
    g_w2 = g_z2.T @ h1
    g_z1 = (g_z2 @ prm.w2) * (z1 > 0)
    g_w1 = g_z1.T @ feats
    g_feat = g_z1 @ prm.w1

    m, c = prm.grids.shape[:2]
    d, h, w = prm.grids.shape[2:]
    g_grids = np.zeros_like(prm.grids)
    for g in range(m):
        inside, (ix, iy, iz), (fx, fy, fz) = terms[g]
        if not inside.any():
            continue
        sel = np.nonzero(inside)[0]
        ix, iy, iz, fx, fy, fz = ix[sel], iy[sel], iz[sel], fx[sel], fy[sel], fz[sel]
        idx, wts = [], []
        for dz in (0, 1):
            wz = fz if dz else 1.0 - fz
            for dy in (0, 1):
                wy = fy if dy else 1.0 - fy
                for dx in (0, 1):
                    wx = fx if dx else 1.0 - fx
                    idx.append((iz + dz) * (h * w) + (iy + dy) * w + (ix + dx))
                    wts.append(wx * wy * wz)
        idx = np.concatenate(idx)
        wts = np.concatenate(wts)
        for ch in range(c):
            contrib = np.tile(g_feat[sel, g * c + ch], 8) * wts
            acc = np.bincount(idx, weights=contrib, minlength=d * h * w)
            g_grids[g, ch] += acc.reshape(d, h, w).astype(prm.dtype)
    return loss, sq, {"grids": g_grids, "w1": g_w1, "w2": g_w2, "w3": g_w3}


# ---------------------------------------------------------------- feature density
def density_terms(transforms: np.ndarray, pts: np.ndarray, p: int):
    """(local (M,N,3), det (M,), bump (M,N), rho (N,)) all f64 (density.py:83-103)."""
    tf = np.asarray(transforms, dtype=np.float64)
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    a, t = tf[:, :3, :3], tf[:, :3, 3]
    local = np.einsum("mij,nj->mni", a, pts) + t[:, None, :]
    det = np.einsum("mi,mi->m", a[:, 0], np.cross(a[:, 1], a[:, 2]))
    with np.errstate(over="ignore"):
        q = ((local * local) ** p).sum(axis=2)
    bump = np.where(q > DENS_CLAMP, 0.0, np.exp(-np.minimum(q, DENS_CLAMP)))
    rho = (np.abs(det)[:, None] * bump).sum(axis=0)
    return local, det, bump, rho


def normalize_density(rho: np.ndarray) -> np.ndarray:
    """rho / sum(rho); ValueError('degenerate') when the sum is not positive (density.py:111-117)."""
    total = np.asarray(rho, dtype=np.float64).sum()
    if total <= 0.0:
        raise ValueError("degenerate batch: feature density sums to zero")
    return np.asarray(rho, dtype=np.float64) / total


def warped_target(rho_s, errors, mean_error, eps=DENS_EPS):
    """exp(((hbar+eps)/(h+eps)) log(rho_s+eps)), exact when the exponent is 1, floored (density.py:120-137)."""
    rho_s = np.asarray(rho_s, dtype=np.float64)
    expo = (mean_error + eps) / (np.asarray(errors, dtype=np.float64) + eps)
    val = np.where(expo == 1.0, rho_s + eps, np.exp(expo * np.log(rho_s + eps)))
    return np.maximum(val, DENS_FLOOR)


def kl_loss(rho_s, rho_star, eps=DENS_EPS) -> float:
    """(1/N) sum rho_s (log(rho_s+eps) - log rho*) (density.py:140-148)."""
    rho_s = np.asarray(rho_s, dtype=np.float64)
    return float((rho_s * (np.log(rho_s + eps) - np.log(np.asarray(rho_star, np.float64)))).sum()
                 / rho_s.size)


def density_loss_and_grads(prm: Params, coords: np.ndarray, errors: np.ndarray):
    """Density KL loss and the gradient w.r.t. the top three transform rows (optim.py:158-200)."""
    x = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    errors = np.asarray(errors, dtype=np.float64).ravel()
    if len(x) < 2 or errors.size != len(x):
        raise ValueError("density batch needs >= 2 coordinates with matching errors")
    p = prm.p
    local, det, bump, rho = density_terms(prm.transforms, x, p)
    total = rho.sum()
    rho_s = normalize_density(rho)
    star = warped_target(rho_s, errors, float(errors.mean()))
    loss = kl_loss(rho_s, star)
    n = rho.size
    d_s = (np.log(rho_s + DENS_EPS) - np.log(star) + rho_s / (rho_s + DENS_EPS)) / n
    d_rho = (d_s - (d_s * rho_s).sum()) / total

    a = np.asarray(prm.transforms, dtype=np.float64)[:, :3, :3]
    cof = np.stack([np.cross(a[:, 1], a[:, 2]), np.cross(a[:, 2], a[:, 0]),
                    np.cross(a[:, 0], a[:, 1])], axis=1)
    with np.errstate(over="ignore", invalid="ignore"):
        lpow = local * (local * local) ** (p - 1)
    lpow = np.where(bump[:, :, None] > 0, lpow, 0.0)
    wgt = d_rho[None, :] * bump
    s = np.abs(det)[:, None] * wgt
    g_a = (np.sign(det) * wgt.sum(axis=1))[:, None, None] * cof
    g_a -= 2.0 * p * np.einsum("mn,mnr,nc->mrc", s, lpow, x)
    g_t = -2.0 * p * np.einsum("mn,mnr->mr", s, lpow)
    g = np.zeros_like(prm.transforms)
    g[:, :3, :3] = g_a.astype(prm.dtype)
    g[:, :3, 3] = g_t.astype(prm.dtype)
    return loss, {"transforms": g}


# ---------------------------------------------------------------- optimizer
class AdamMoments:
    """Moment buffers + step counter (optim.py:38-44)."""

    def __init__(self, params: dict):
        self.m = {k: np.zeros_like(v) for k, v in params.items()}
        self.v = {k: np.zeros_like(v) for k, v in params.items()}
        self.t = 0


def adam_update(params: dict, grads: dict, st: AdamMoments, lr: float) -> None:
    """Masked, bias-corrected Adam in place; exact-zero grads leave p/m/v alone (optim.py:47-73)."""
    st.t += 1
    c1 = 1.0 - ADAM_B1 ** st.t
    c2 = 1.0 - ADAM_B2 ** st.t
    for name, p in params.items():
        g = grads[name]
        if g.shape != p.shape:
            raise ValueError(f"gradient shape {g.shape} != parameter shape {p.shape}")
        live = g != 0
        if not live.any():
            continue
        gl = g[live]
        m_new = ADAM_B1 * st.m[name][live] + (1.0 - ADAM_B1) * gl
        v_new = ADAM_B2 * st.v[name][live] + (1.0 - ADAM_B2) * (gl * gl)
        st.m[name][live] = m_new
        st.v[name][live] = v_new
        p[live] = p[live] - lr * (m_new / c1) / (np.sqrt(v_new / c2) + ADAM_EPS)


# ---------------------------------------------------------------- training loop
@dataclass
class LoopConfig:
    """Mirror of TrainConfig defaults (trainer.py:37-67)."""
    iterations: int = 50_000
    batch_size: int = 100_000
    lr_main: float = 0.01
    lr_transform: float = 0.001
    delay_start: int = 500
    transform_ma_window: int = 1000
    transform_improve_threshold: float = 1e-4
    transform_hard_stop_fraction: float = 0.8
    plateau_window: int = 500
    plateau_threshold: float = 1e-4
    plateau_factor: float = 10.0
    plateau_max_triggers: int = 3
    seed: int = 0
    train_transforms: bool = True
    plateau_enabled: bool = True

    @property
    def hard_stop_iteration(self) -> int:
        return int(math.ceil(self.transform_hard_stop_fraction * self.iterations))


@dataclass
class LoopLog:
    l_rec: list = field(default_factory=list)
    l_density: list = field(default_factory=list)
    lr: list = field(default_factory=list)
    transform_stop_iteration: int | None = None
    plateau_trigger_iterations: list = field(default_factory=list)
    iterations_run: int = 0


@dataclass
class Plateau:
    window: int
    threshold: float
    factor: float
    max_triggers: int
    lr: float = 1.0
    history: list = field(default_factory=list)
    triggers: int = 0


def plateau_advance(pl: Plateau, ma: float) -> str:
    """Window-to-window MA comparison -> 'none' | 'reduce_lr' | 'stop' (trainer.py:118-138)."""
    pl.history.append(ma)
    if len(pl.history) <= pl.window:
        return "none"
    ref = pl.history[-pl.window - 1]
    gain = (ref - ma) / max(abs(ref), 1e-12)
    if gain >= pl.threshold:
        return "none"
    pl.history.clear()
    pl.triggers += 1
    pl.lr /= pl.factor
    return "stop" if pl.triggers >= pl.max_triggers else "reduce_lr"


def transform_should_stop(hist, cfg: LoopConfig, it: int) -> bool:
    """Hard stop at ceil(frac*iters) or MA-improvement rule (trainer.py:141-157)."""
    if it >= cfg.hard_stop_iteration:
        return True
    w = cfg.transform_ma_window
    if len(hist) < 2 * w:
        return False
    recent = float(np.mean(hist[-w:]))
    prev = float(np.mean(hist[-2 * w:-w]))
    return (prev - recent) / max(abs(prev), 1e-12) < cfg.transform_improve_threshold


def train_single(prm: Params, volume: np.ndarray, cfg: LoopConfig, on_iteration=None):
    """Reference training loop, restated (trainer.py:160-223). Mutates ``prm``; returns the log."""
    log = LoopLog()
    if cfg.iterations == 0:
        return log
    rng = np.random.Generator(np.random.Philox(cfg.seed))
    main = {"grids": prm.grids, "w1": prm.w1, "w2": prm.w2, "w3": prm.w3}
    tfp = {"transforms": prm.transforms}
    st_main, st_tf = AdamMoments(main), AdamMoments(tfp)
    pl = Plateau(cfg.plateau_window, cfg.plateau_threshold, cfg.plateau_factor,
                 cfg.plateau_max_triggers, lr=cfg.lr_main)
    dhist: list = []
    active = cfg.train_transforms
    scale = 1.0
    for it in range(cfg.iterations):
        c64 = rng.uniform(-1.0, 1.0, size=(cfg.batch_size, 3))
        tgt = sample_volume(volume, c64).astype(np.float32)
        c32 = c64.astype(np.float32)
        lr_loss, sq, grads = recon_loss_and_grads(prm, c32, tgt)
        adam_update(main, grads, st_main, cfg.lr_main * scale)
        ld = None
        if active and it >= cfg.delay_start:
            if transform_should_stop(dhist, cfg, it):
                active = False
                log.transform_stop_iteration = it
            else:
                ld, dg = density_loss_and_grads(prm, c32, np.asarray(sq, dtype=np.float64))
                adam_update(tfp, dg, st_tf, cfg.lr_transform * scale)
                dhist.append(ld)
        log.l_rec.append(lr_loss)
        log.l_density.append(ld)
        log.lr.append(cfg.lr_main * scale)
        log.iterations_run = it + 1
        if on_iteration is not None:
            on_iteration(it, prm)
        if cfg.plateau_enabled and len(log.l_rec) >= cfg.plateau_window:
            act = plateau_advance(pl, float(np.mean(log.l_rec[-cfg.plateau_window:])))
            if act != "none":
                log.plateau_trigger_iterations.append(it)
                scale /= cfg.plateau_factor
                if act == "stop":
                    break
    return log


def lattice_points(dims) -> np.ndarray:
    """Every voxel's normalized coordinate, x fastest (volume.py:137-141)."""
    ax = [lattice_axis(n) for n in dims]
    zz, yy, xx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)


def psnr(predict, volume: np.ndarray, chunk: int = 65536) -> float:
    """10 log10(range^2 / MSE) over every voxel, capped at 200 dB (trainer.py:226-247)."""
    lo, hi = float(volume.min()), float(volume.max())
    span = hi - lo
    if span == 0.0:
        return PSNR_CAP
    d, h, w = volume.shape
    pts = lattice_points((w, h, d))
    truth = volume.ravel()
    sse = 0.0
    for s in range(0, len(pts), chunk):
        pred = np.asarray(predict(pts[s:s + chunk].astype(np.float32)), dtype=np.float64)
        diff = pred - truth[s:s + chunk]
        sse += float((diff * diff).sum())
    mse = sse / len(pts)
    if mse == 0.0:
        return PSNR_CAP
    return float(min(10.0 * np.log10(span * span / mse), PSNR_CAP))


# ---------------------------------------------------------------- decomposition
def axis_runs(n: int, parts: int):
    """Even split with the longer runs first; inclusive (lo, hi) (decomposition.py:68-78)."""
    q, r = divmod(n, parts)
    runs, lo = [], 0
    for i in range(parts):
        ln = q + (1 if i < r else 0)
        runs.append((lo, lo + ln - 1))
        lo += ln
    return runs


def brick_extents(dims, counts, ghost):
    """Per flat brick (i fastest): (core_lo, core_hi, ghost_lo, ghost_hi) (decomposition.py:81-109)."""
    runs = [axis_runs(n, c) for n, c in zip(dims, counts)]
    out = []
    for k in range(counts[2]):
        for j in range(counts[1]):
            for i in range(counts[0]):
                lo = (runs[0][i][0], runs[1][j][0], runs[2][k][0])
                hi = (runs[0][i][1], runs[1][j][1], runs[2][k][1])
                glo = tuple(max(0, v - ghost) for v in lo)
                ghi = tuple(min(n - 1, v + ghost) for v, n in zip(hi, dims))
                out.append((lo, hi, glo, ghi))
    return out


def brick_of(pts: np.ndarray, counts) -> np.ndarray:
    """Flat owner i + I*j + I*J*k via floor(count*(p+1)/2) in f64, clamped (decomposition.py:112-123)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    if pts.size and (np.abs(pts) > 1.0).any():
        raise ValueError("coordinate outside [-1, 1]^3")
    cnt = np.array(counts)
    cell = np.minimum(np.floor(cnt * (pts + 1.0) * 0.5).astype(np.int64), cnt - 1)
    return cell[:, 0] + counts[0] * cell[:, 1] + counts[0] * counts[1] * cell[:, 2]


def brick_affines(dims, counts, ghost):
    """Per-brick (scale, offset) mapping the ghost extent onto [-1, 1] (decomposition.py:267-277)."""
    def bound(i, n):
        return 0.0 if n == 1 else 2.0 * i / (n - 1) - 1.0
    ext = brick_extents(dims, counts, ghost)
    scale = np.zeros((len(ext), 3))
    offset = np.zeros((len(ext), 3))
    for b, (_, _, glo, ghi) in enumerate(ext):
        for a in range(3):
            lo, hi = bound(glo[a], dims[a]), bound(ghi[a], dims[a])
            if hi > lo:
                s = 2.0 / (hi - lo)
                scale[b, a] = s
                offset[b, a] = -s * lo - 1.0
    return scale, offset


def decomposed_forward(models, counts, scale, offset, pts) -> np.ndarray:
    """Hash each point to its brick, map to brick-local coords in f64, evaluate (decomposition.py:294-304)."""
    pts = np.atleast_2d(np.asarray(pts))
    owner = brick_of(pts, counts)
    out = np.zeros(len(pts), dtype=np.float32)
    for b in np.unique(owner):
        sel = owner == b
        loc = pts[sel].astype(np.float64) * scale[b] + offset[b]
        out[sel] = forward(models[b], loc.astype(np.float32))
    return out


def brick_seed(seed: int, flat: int) -> int:
    """(seed ^ flat) & 0x7FFFFFFF (decomposition.py:159-160)."""
    return (seed ^ flat) & 0x7FFFFFFF


# ---------------------------------------------------------------- init (host-side in the product too)
def init_params(grids, channels, res, seed, vmin=0.0, vmax=1.0, p=10) -> Params:
    """Seeded initialization (model.py:247-291): Philox normal transforms, U(-1e-4,1e-4) grids,
    Glorot-uniform decoder, all drawn from one stream in the reference's order."""
    rng = np.random.Generator(np.random.Philox(seed))
    d, h, w = res
    tf = np.zeros((grids, 4, 4))
    for g in range(grids):
        while True:
            a = np.zeros((3, 3))
            a[np.diag_indices(3)] = rng.normal(1.0, 0.05, size=3)
            off = rng.normal(0.0, 0.05, size=6)
            a[0, 1], a[0, 2], a[1, 0], a[1, 2], a[2, 0], a[2, 1] = off
            if np.linalg.det(a) > 0:
                break
        tf[g, :3, :3] = a
        tf[g, :3, 3] = rng.normal(0.0, 0.05, size=3)
        tf[g, 3, 3] = 1.0
    gr = rng.uniform(-1e-4, 1e-4, size=(grids, channels, d, h, w))

    def glorot(fi, fo, shape):
        lim = np.sqrt(6.0 / (fi + fo))
        return rng.uniform(-lim, lim, size=shape)

    w1 = glorot(grids * channels, HIDDEN, (HIDDEN, grids * channels))
    w2 = glorot(HIDDEN, HIDDEN, (HIDDEN, HIDDEN))
    w3 = glorot(HIDDEN, 1, (1, HIDDEN))
    f32 = np.float32
    return Params(tf.astype(f32), gr.astype(f32), w1.astype(f32), w2.astype(f32), w3.astype(f32),
                  float(vmin), float(vmax), p)


# ---------------------------------------------------------------- threaded CPU baseline
def _chunks(n: int, parts: int):
    step = -(-n // parts)
    return [(s, min(n, s + step)) for s in range(0, n, step)]


def _recon_partial(prm: Params, coords, targets, n_total):
    """recon_loss_and_grads (optim.py:102-155) on one slice of the batch, with the global batch
    size in the 2/N factor: partial weight gradients, partial f64 grid-gradient sums, sq."""
    feats, terms = encode(prm, coords, keep_terms=True)
    z1, h1, z2, h2, out = decode_chain(prm, feats)
    resid = out - targets
    sq = resid * resid
    span = np.asarray(prm.vmax - prm.vmin, dtype=prm.dtype)
    g_out = (resid * (np.asarray(2.0 / n_total, dtype=prm.dtype) * span))[:, None]
    g_w3 = g_out.T @ h2
    g_z2 = (g_out @ prm.w3) * (z2 > 0)
    g_w2 = g_z2.T @ h1
    g_z1 = (g_z2 @ prm.w2) * (z1 > 0)
    g_w1 = g_z1.T @ feats
    g_feat = g_z1 @ prm.w1
    m, c = prm.grids.shape[:2]
    d, h, w = prm.grids.shape[2:]
    g_grids = np.zeros(prm.grids.shape, dtype=np.float64)
    for g in range(m):
        inside, (ix, iy, iz), (fx, fy, fz) = terms[g]
        sel = np.nonzero(inside)[0]
        if not len(sel):
            continue
        ix, iy, iz, fx, fy, fz = ix[sel], iy[sel], iz[sel], fx[sel], fy[sel], fz[sel]
        idx, wts = [], []
        for dz in (0, 1):
            wz = fz if dz else 1.0 - fz
            for dy in (0, 1):
                wy = fy if dy else 1.0 - fy
                for dx in (0, 1):
                    wx = fx if dx else 1.0 - fx
                    idx.append((iz + dz) * (h * w) + (iy + dy) * w + (ix + dx))
                    wts.append(wx * wy * wz)
        idx = np.concatenate(idx)
        wts = np.concatenate(wts)
        for ch in range(c):
            contrib = np.tile(g_feat[sel, g * c + ch], 8) * wts
            g_grids[g, ch] += np.bincount(idx, weights=contrib, minlength=d * h * w).reshape(d, h, w)
    return sq, g_grids, g_w1, g_w2, g_w3


def recon_loss_and_grads_threaded(prm: Params, coords, targets, pool, parts: int):
    """recon_loss_and_grads over `parts` batch slices on a thread pool (numpy releases the GIL
    in its kernels); partial sums added in slice order.  Same arithmetic per element; the batch
    sums associate differently (CPU-baseline timing only -- parity uses the serial oracle)."""
    targets = np.asarray(targets, dtype=prm.dtype).ravel()
    coords = np.atleast_2d(np.asarray(coords, dtype=prm.dtype))
    n = targets.size
    futs = [pool.submit(_recon_partial, prm, coords[a:b], targets[a:b], n) for a, b in _chunks(n, parts)]
    res = [f.result() for f in futs]
    sq = np.concatenate([r[0] for r in res])
    g_grids = res[0][1]
    for r in res[1:]:
        g_grids += r[1]
    grads = {"grids": g_grids.astype(prm.dtype), "w1": sum(r[2] for r in res), "w2": sum(r[3] for r in res),
             "w3": sum(r[4] for r in res)}
    return float(np.mean(sq, dtype=np.float64)), sq, grads


def density_loss_and_grads_threaded(prm: Params, coords, errors, pool, parts: int):
    """density_loss_and_grads (optim.py:158-200) in three phases over batch slices: per-slice
    rho, the global statistics (serial, O(N)), per-slice transform-gradient sums."""
    x = np.atleast_2d(np.asarray(coords, dtype=np.float64))
    errors = np.asarray(errors, dtype=np.float64).ravel()
    p = prm.p
    sl = _chunks(len(x), parts)
    terms = [f.result() for f in [pool.submit(density_terms, prm.transforms, x[a:b], p) for a, b in sl]]
    rho = np.concatenate([t[3] for t in terms])
    det = terms[0][1]
    total = rho.sum()
    rho_s = normalize_density(rho)
    star = warped_target(rho_s, errors, float(errors.mean()))
    loss = kl_loss(rho_s, star)
    n = rho.size
    d_s = (np.log(rho_s + DENS_EPS) - np.log(star) + rho_s / (rho_s + DENS_EPS)) / n
    d_rho = (d_s - (d_s * rho_s).sum()) / total
    a = np.asarray(prm.transforms, dtype=np.float64)[:, :3, :3]
    cof = np.stack([np.cross(a[:, 1], a[:, 2]), np.cross(a[:, 2], a[:, 0]), np.cross(a[:, 0], a[:, 1])], axis=1)

    def part(k):
        (lo, hi), (local, _, bump, _) = sl[k], terms[k]
        with np.errstate(over="ignore", invalid="ignore"):
            lpow = local * (local * local) ** (p - 1)
        lpow = np.where(bump[:, :, None] > 0, lpow, 0.0)
        wgt = d_rho[None, lo:hi] * bump
        s = np.abs(det)[:, None] * wgt
        return (wgt.sum(axis=1), np.einsum("mn,mnr,nc->mrc", s, lpow, x[lo:hi]),
                np.einsum("mn,mnr->mr", s, lpow))

    res = [f.result() for f in [pool.submit(part, k) for k in range(len(sl))]]
    wsum = sum(r[0] for r in res)
    g_a = (np.sign(det) * wsum)[:, None, None] * cof - 2.0 * p * sum(r[1] for r in res)
    g_t = -2.0 * p * sum(r[2] for r in res)
    g = np.zeros_like(prm.transforms)
    g[:, :3, :3] = g_a.astype(prm.dtype)
    g[:, :3, 3] = g_t.astype(prm.dtype)
    return loss, {"transforms": g}


def train_single_threaded(prm: Params, volume: np.ndarray, cfg: LoopConfig, threads: int, on_iteration=None):
    """train_single (trainer.py:160-223) with each iteration's batch split over `threads` host
    threads (the CPU baseline of bench.py --impl reference: the reference algorithm with all the
    host threads it can use).  Plateau logic as the serial loop; returns the log."""
    import concurrent.futures as cf
    log = LoopLog()
    rng = np.random.Generator(np.random.Philox(cfg.seed))
    main = {"grids": prm.grids, "w1": prm.w1, "w2": prm.w2, "w3": prm.w3}
    tfp = {"transforms": prm.transforms}
    st_main, st_tf = AdamMoments(main), AdamMoments(tfp)
    dhist: list = []
    active = cfg.train_transforms
    parts = max(1, threads)
    with cf.ThreadPoolExecutor(max_workers=parts) as pool:
        for it in range(cfg.iterations):
            c64 = rng.uniform(-1.0, 1.0, size=(cfg.batch_size, 3))
            tgt = np.concatenate([f.result() for f in [pool.submit(sample_volume, volume, c64[a:b])
                                                       for a, b in _chunks(len(c64), parts)]]).astype(np.float32)
            c32 = c64.astype(np.float32)
            lr_loss, sq, grads = recon_loss_and_grads_threaded(prm, c32, tgt, pool, parts)
            adam_update(main, grads, st_main, cfg.lr_main)
            ld = None
            if active and it >= cfg.delay_start:
                if transform_should_stop(dhist, cfg, it):
                    active = False
                    log.transform_stop_iteration = it
                else:
                    ld, dg = density_loss_and_grads_threaded(prm, c32, np.asarray(sq, dtype=np.float64), pool,
                                                             parts)
                    adam_update(tfp, dg, st_tf, cfg.lr_transform)
                    dhist.append(ld)
            log.l_rec.append(lr_loss)
            log.l_density.append(ld)
            log.lr.append(cfg.lr_main)
            log.iterations_run = it + 1
            if on_iteration is not None:
                on_iteration(it, prm)
    return log
