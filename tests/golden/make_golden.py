"""Generate golden fixtures by running the REFERENCE implementation.

Run once in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``apmg`` from /root/reference/pkg/src (the
product package here is ``paper_2308_02494_b200``, so there is no name clash),
runs the reference's own public functions on small seeded inputs, and writes
compressed ``.npz`` fixtures next to this script. The fixtures are committed;
nothing on the GPU box reads /root/reference.

Each fixture records the reference function it came from (file:line in
/root/reference/pkg/src/apmg).
"""
from __future__ import annotations

import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF_SRC))

import apmg  # noqa: E402  (the reference)
from apmg import decomposition as rdec  # noqa: E402
from apmg import density as rden  # noqa: E402
from apmg import model as rmodel  # noqa: E402
from apmg import optim as ropt  # noqa: E402
from apmg import trainer as rtrain  # noqa: E402
from apmg import volume as rvol  # noqa: E402

assert Path(apmg.__file__).resolve().is_relative_to(REF_SRC), apmg.__file__


def model_arrays(prefix: str, m) -> dict:
    return {
        f"{prefix}transforms": m.transforms.copy(), f"{prefix}grids": m.grids.copy(),
        f"{prefix}w1": m.w1.copy(), f"{prefix}w2": m.w2.copy(), f"{prefix}w3": m.w3.copy(),
        f"{prefix}meta": np.array([m.config.grids, m.config.channels, *m.config.resolution,
                                   m.config.flat_top_p], dtype=np.int64),
        f"{prefix}range": np.array([m.vmin, m.vmax], dtype=np.float64),
    }


def perturbed_model(seed, grids, channels, res, dtype, vmin=-0.5, vmax=1.5, tscale=0.15):
    cfg = rmodel.ModelConfig(grids=grids, channels=channels, resolution=res)
    m = rmodel.init_model(cfg, seed=seed, vmin=vmin, vmax=vmax).astype(dtype)
    rng = np.random.default_rng(seed + 4242)
    m.grids[:] = rng.normal(scale=0.5, size=m.grids.shape)
    m.w1[:] = rng.normal(scale=0.25, size=m.w1.shape)
    m.w2[:] = rng.normal(scale=0.25, size=m.w2.shape)
    m.w3[:] = rng.normal(scale=0.25, size=m.w3.shape)
    # move the grids off the identity so inside/outside and multi-grid overlap are exercised
    m.transforms[:, :3, :3] += rng.normal(scale=tscale, size=(grids, 3, 3))
    m.transforms[:, :3, 3] += rng.normal(scale=tscale, size=(grids, 3))
    return m


def gen_encode_forward():
    """model.py:141-166 encode/decode/forward on f32 and f64 models."""
    out = {}
    cases = [("a32_", 3, 4, 2, (5, 4, 6), np.float32), ("a64_", 3, 4, 2, (5, 4, 6), np.float64),
             ("b32_", 11, 16, 2, (12, 10, 8), np.float32), ("c32_", 5, 3, 1, (2, 3, 2), np.float32),
             ("d32_", 8, 8, 3, (6, 7, 5), np.float32)]
    for prefix, seed, g, c, res, dt in cases:
        m = perturbed_model(seed, g, c, res, dt)
        rng = np.random.default_rng(seed + 1)
        pts = rng.uniform(-1.15, 1.15, (3000, 3)).astype(dt)
        pts[:8] = [[1, 1, 1], [-1, -1, -1], [0, 0, 0], [1, -1, 0.5], [-1, 1, -0.25],
                   [0.999, -0.999, 0.0], [1e-7, -1e-7, 1.0], [0.5, 0.5, 0.5]]
        out.update(model_arrays(prefix, m))
        out[prefix + "pts"] = pts
        out[prefix + "feats"] = m.encode(pts)
        out[prefix + "out"] = m.forward(pts)
    np.savez_compressed(OUT / "encode_forward.npz", **out)


def gen_recon():
    """optim.py:102-155 recon_loss_and_grads."""
    out = {}
    for prefix, seed, g, c, res, dt, n in [("a32_", 21, 4, 2, (5, 4, 6), np.float32, 777),
                                            ("a64_", 21, 4, 2, (5, 4, 6), np.float64, 777),
                                            ("b32_", 23, 16, 2, (8, 8, 8), np.float32, 4096),
                                            ("c64_", 25, 3, 1, (4, 4, 4), np.float64, 48)]:
        m = perturbed_model(seed, g, c, res, dt)
        rng = np.random.default_rng(seed + 7)
        coords = rng.uniform(-1, 1, (n, 3)).astype(dt)
        targets = rng.normal(size=n).astype(dt)
        loss, sq, grads = ropt.recon_loss_and_grads(m, coords, targets)
        out.update(model_arrays(prefix, m))
        out[prefix + "coords"] = coords
        out[prefix + "targets"] = targets
        out[prefix + "loss"] = np.array(loss)
        out[prefix + "sq"] = sq
        for k, v in grads.items():
            out[prefix + "g_" + k] = v
    np.savez_compressed(OUT / "recon.npz", **out)


def gen_density():
    """density.py:83-148 and optim.py:158-200."""
    out = {}
    for prefix, seed, g, dt, n, uniform in [("a32_", 31, 4, np.float32, 500, False),
                                             ("a64_", 31, 4, np.float64, 500, False),
                                             ("b32_", 33, 64, np.float32, 4096, False),
                                             ("u64_", 35, 3, np.float64, 64, True)]:
        m = perturbed_model(seed, g, 1, (4, 4, 4), dt, tscale=0.3)
        rng = np.random.default_rng(seed + 3)
        coords = rng.uniform(-1, 1, (n, 3)).astype(dt)
        coords[0] = [5.0, 0.0, 0.0]  # far point: every bump clamps to exactly zero
        errors = np.full(n, 0.2) if uniform else rng.uniform(0.0, 1.0, n) ** 3
        loss, dg = ropt.density_loss_and_grads(m, coords, errors)
        local, dets, bumps, rho = rden.feature_density_terms(m.transforms, coords, m.config.flat_top_p)
        rs = rden.scale_density(rho)
        star = rden.target_density(rs, errors, float(errors.mean()))
        out.update(model_arrays(prefix, m))
        out[prefix + "coords"] = coords
        out[prefix + "errors"] = errors
        out[prefix + "loss"] = np.array(loss)
        out[prefix + "g_transforms"] = dg["transforms"]
        out[prefix + "rho"] = rho
        out[prefix + "rho_scaled"] = rs
        out[prefix + "rho_star"] = star
        out[prefix + "dloss"] = np.array(rden.density_loss(rs, star))
    np.savez_compressed(OUT / "density.npz", **out)


def gen_adam():
    """optim.py:47-73 adam_step, with exact-zero gradient entries."""
    rng = np.random.default_rng(41)
    out = {}
    for prefix, dt in (("f32_", np.float32), ("f64_", np.float64)):
        p = rng.normal(size=257).astype(dt)
        params = {"w": p.copy()}
        state = ropt.AdamState(params)
        grads_seq, traj, ms, vs = [], [], [], []
        for step in range(12):
            g = rng.normal(size=257).astype(dt)
            g[rng.uniform(size=257) < 0.3] = 0
            if step == 5:
                g[:] = 0
            ropt.adam_step(params, {"w": g}, state, lr=0.01 * (0.5 ** (step // 4)))
            grads_seq.append(g)
            traj.append(params["w"].copy())
            ms.append(state.m["w"].copy())
            vs.append(state.v["w"].copy())
        out[prefix + "p0"] = p
        out[prefix + "grads"] = np.stack(grads_seq)
        out[prefix + "traj"] = np.stack(traj)
        out[prefix + "m"] = np.stack(ms)
        out[prefix + "v"] = np.stack(vs)
        out[prefix + "lrs"] = np.array([0.01 * (0.5 ** (s // 4)) for s in range(12)])
    np.savez_compressed(OUT / "adam.npz", **out)


def gen_philox():
    """trainer.py:175,189: Generator(Philox(seed)).uniform(-1, 1, (B, 3)) per iteration."""
    out = {}
    for seed, b, iters in ((0, 5, 3), (9, 7, 2), (123456789, 4, 3), (2**31 - 1, 1, 5), (7, 1000, 2)):
        bitgen = np.random.Philox(seed)
        key = np.array(bitgen.state["state"]["key"], dtype=np.uint64)
        rng = np.random.Generator(np.random.Philox(seed))
        draws = np.stack([rng.uniform(-1.0, 1.0, size=(b, 3)) for _ in range(iters)])
        out[f"s{seed}_b{b}_key"] = key
        out[f"s{seed}_b{b}_draws"] = draws
        raw = np.random.Philox(seed).random_raw(16)
        out[f"s{seed}_b{b}_raw"] = raw
    np.savez_compressed(OUT / "philox.npz", **out)


def gen_volume():
    """volume.py:147-199 sample_many and :275-296 synth_volume."""
    blobs = [rvol.BlobSpec(center=(0.2, -0.1, 0.3), sigma=(0.35, 0.3, 0.4)),
             rvol.BlobSpec(center=(-0.5, 0.4, -0.2), sigma=(0.1, 0.2, 0.15), amplitude=0.7)]
    out = {}
    v1 = rvol.synth_volume((7, 6, 5), blobs, background=0.25)
    v2 = rvol.synth_volume((9, 8, 10), blobs, seed=3, noise=0.05)
    v3 = rvol.synth_volume((5, 1, 4), blobs)  # a 1-voxel axis
    rng = np.random.default_rng(51)
    pts = rng.uniform(-1, 1, (2000, 3))
    pts[:6] = [[1, 1, 1], [-1, -1, -1], [0, 0, 0], [1, -1, 0.5], [-1, 1, -1.0], [0.999999, 0, -0.999999]]
    for tag, v in (("v1", v1), ("v2", v2), ("v3", v3)):
        out[tag + "_data"] = v.data
        out[tag + "_dims"] = np.array(v.dims)
        out[tag + "_samples"] = v.sample_many(pts)
    out["pts"] = pts
    big = rvol.synth_volume((64, 48, 40), blobs, background=0.1)
    out["big_data"] = big.data
    np.savez_compressed(OUT / "volume.npz", **out)


def adaptivity_blobs():
    """test_acceptance.py:156-164 blob list (SURVEY 8d synthetic inputs)."""
    return [
        rvol.BlobSpec(center=(0.45, -0.3, 0.2), sigma=(0.035, 0.035, 0.035)),
        rvol.BlobSpec(center=(-0.2, 0.2, -0.1), sigma=(0.6, 0.5, 0.7), amplitude=0.35),
        rvol.BlobSpec(center=(0.3, 0.4, 0.5), sigma=(0.45, 0.55, 0.4), amplitude=0.25),
        rvol.BlobSpec(center=(-0.5, -0.5, 0.4), sigma=(0.5, 0.4, 0.5), amplitude=0.3),
    ]


def log_arrays(prefix, log):
    return {
        prefix + "l_rec": np.array(log.l_rec),
        prefix + "l_density": np.array([np.nan if v is None else v for v in log.l_density]),
        prefix + "lr": np.array(log.lr),
        prefix + "stop": np.array(-1 if log.transform_stop_iteration is None else log.transform_stop_iteration),
        prefix + "triggers": np.array(log.plateau_trigger_iterations, dtype=np.int64),
        prefix + "iters": np.array(log.iterations_run),
    }


def gen_train_small():
    """trainer.py:160-223 train_single on tiny configs (init + log + final params)."""
    out = {}
    vol = rvol.synth_volume((16, 16, 16), [rvol.BlobSpec(center=(0.2, -0.1, 0.3), sigma=(0.35, 0.3, 0.4))])
    out["blob_data"] = vol.data
    cfg_m = rmodel.ModelConfig(grids=4, channels=1, resolution=(4, 4, 4), seed=9)
    m = rmodel.init_model(cfg_m, seed=9, vmin=vol.vmin, vmax=vol.vmax)
    out.update(model_arrays("init_", m))
    cfg = rtrain.TrainConfig(iterations=40, batch_size=64, delay_start=5, seed=9, plateau_enabled=False)
    m, log = rtrain.train_single(m, vol, cfg)
    out.update(model_arrays("final_", m))
    out.update(log_arrays("log_", log))
    out["psnr"] = np.array(rtrain.psnr(m, vol))
    # hard stop at ceil(0.5*100) and frozen transforms afterwards
    m2 = rmodel.init_model(cfg_m, seed=9, vmin=vol.vmin, vmax=vol.vmax)
    cfg2 = rtrain.TrainConfig(iterations=100, batch_size=32, delay_start=10,
                              transform_hard_stop_fraction=0.5, plateau_enabled=False, seed=3)
    m2, log2 = rtrain.train_single(m2, vol, cfg2)
    out.update(model_arrays("hs_", m2))
    out.update(log_arrays("hslog_", log2))
    # constant volume: 3 plateau triggers, early end (test_trainer.py:98-114)
    const = rvol.Volume(dims=(8, 8, 8), data=np.full((8, 8, 8), 3.25, dtype=np.float32))
    m3 = rmodel.init_model(cfg_m, seed=0, vmin=const.vmin, vmax=const.vmax)
    cfg3 = rtrain.TrainConfig(iterations=4000, batch_size=64, seed=1)
    m3, log3 = rtrain.train_single(m3, const, cfg3)
    out.update(log_arrays("const_", log3))
    np.savez_compressed(OUT / "train_small.npz", **out)


def gen_train_c1(iters=200, batch=2**14, delay=50):
    """C1-shaped parity run: 64 grids 32^3 x2, MLP 2x64, 128^3 blob field, fixed iterations,
    plateau off. Stores the reference's loss log and final PSNR."""
    vol = rvol.synth_volume((128, 128, 128), adaptivity_blobs())
    cfg_m = rmodel.ModelConfig(grids=64, channels=2, resolution=(32, 32, 32))
    m = rmodel.init_model(cfg_m, seed=0, vmin=vol.vmin, vmax=vol.vmax)
    cfg = rtrain.TrainConfig(iterations=iters, batch_size=batch, delay_start=delay, seed=0,
                             plateau_enabled=False)
    t0 = time.perf_counter()
    m, log = rtrain.train_single(m, vol, cfg)
    wall = time.perf_counter() - t0
    p = rtrain.psnr(m, vol)
    out = log_arrays("log_", log)
    out["psnr"] = np.array(p)
    out["wall_seconds"] = np.array(wall)
    out["config"] = np.array([iters, batch, delay])
    out["final_transforms"] = m.transforms
    out["final_w3"] = m.w3
    np.savez_compressed(OUT / "train_c1.npz", **out)
    print(f"C1 parity run: {iters} its x {batch} in {wall:.1f}s, psnr {p:.4f} dB")


def gen_hash_decomp():
    """decomposition.py:81-123 plan_partition/spatial_hash and :258-306 DecomposedField."""
    out = {}
    rng = np.random.default_rng(61)
    for counts in ((1, 1, 1), (2, 2, 2), (3, 1, 2), (4, 3, 2), (4, 4, 4)):
        pts = rng.uniform(-1, 1, (3000, 3))
        edges = []
        for n in counts:
            edges.extend([-1.0 + 2.0 * i / n for i in range(n + 1)])
        e = np.array(edges)
        pts[:len(e), 0] = e
        pts[:len(e), 1] = e[::-1]
        pts[:len(e), 2] = 1.0
        tag = "x".join(map(str, counts))
        out["hash_" + tag + "_pts"] = pts
        out["hash_" + tag + "_owner"] = rdec.spatial_hash(pts, *counts)
    with tempfile.TemporaryDirectory() as tmp:
        tmp = Path(tmp)
        vol = rvol.synth_volume((16, 16, 16), [rvol.BlobSpec(center=(0.3, 0.0, -0.2), sigma=(0.4, 0.5, 0.35))])
        header = rvol.save_volume(vol, tmp / "v.raw")
        plan = rdec.plan_partition(header.dims, 3, 2, 2, ghost=1)
        mcfg = rmodel.ModelConfig(grids=2, channels=1, resolution=(4, 4, 4), seed=7)
        tcfg = rtrain.TrainConfig(iterations=15, batch_size=32, delay_start=10,
                                  transform_hard_stop_fraction=1.0, plateau_enabled=False, seed=7)
        rdec.train_decomposed(tmp / "v.raw", header, plan, mcfg, tcfg, tmp / "dec", workers=1)
        field = rdec.DecomposedField.load(tmp / "dec" / "manifest.json")
        pts = rng.uniform(-1, 1, (2000, 3)).astype(np.float32)
        out["dec_manifest"] = np.frombuffer((tmp / "dec" / "manifest.json").read_bytes(), dtype=np.uint8)
        for i, mdl in enumerate(field.models):
            out.update(model_arrays(f"dec_m{i}_", mdl))
        out["dec_count"] = np.array(len(field.models))
        out["dec_scale"] = field._scale
        out["dec_offset"] = field._offset
        out["dec_pts"] = pts
        out["dec_out"] = field.forward(pts)
        out["dec_vol"] = vol.data
        out["dec_psnr"] = np.array(rtrain.psnr(field, vol))
        out["dec_vmin_vmax_diag"] = np.array([field.vmin, field.vmax, field.voxel_diagonal])
    np.savez_compressed(OUT / "hash_decomp.npz", **out)


def gen_psnr():
    """trainer.py:226-247 psnr of a perturbed model over a small lattice."""
    vol = rvol.synth_volume((9, 11, 10), [rvol.BlobSpec(center=(0.2, -0.1, 0.3), sigma=(0.35, 0.3, 0.4))])
    m = perturbed_model(71, 4, 2, (5, 5, 5), np.float32, vmin=vol.vmin, vmax=vol.vmax)
    m.w1 *= 0.2
    out = model_arrays("m_", m)
    out["vol"] = vol.data
    out["psnr"] = np.array(rtrain.psnr(m, vol))
    out["psnr_b7"] = np.array(rtrain.psnr(m, vol, batch_size=7))
    np.savez_compressed(OUT / "psnr.npz", **out)


def gen_render():
    """Renderer field-query path (render.py): ray/box hits incl. parallel and inside rays,
    transfer-function lookups, single-ray composites, and full frames of a volume field, a
    small model field and a flagship-shaped model field (non-trivial TF, window, early exit)."""
    from apmg import render as rr
    out = {}
    # ray / box
    origin = np.array([0.3, -0.2, 2.5])
    dirs = np.array([[0.0, 0.0, -1.0], [0.0, 1.0, 0.0], [0.6, 0.0, -0.8], [0.0, 0.0, 1.0],
                     [1e-300, 0.0, -1.0], [-0.1, 0.05, -0.99]])
    dirs[-1] /= np.linalg.norm(dirs[-1])
    e, x, h = rr.ray_box_hits(origin, dirs)
    out.update(rb_origin=origin, rb_dirs=dirs, rb_enter=e, rb_exit=x, rb_hit=h)
    e, x, h = rr.ray_box_hits(np.zeros(3), np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -1.0]]))
    out.update(rb0_enter=e, rb0_exit=x, rb0_hit=h)
    e, x, h = rr.ray_box_hits(np.array([0.0, 2.0, 5.0]), np.array([[0.0, 0.0, -1.0]]))
    out.update(rb1_hit=h)
    # transfer function
    tf = rr.TransferFunction(
        color_points=[(0.0, (0.0, 0.0, 0.1)), (0.4, (1.0, 0.2, 0.0)), (1.0, (1.0, 1.0, 1.0))],
        opacity_points=[(0.0, 0.0), (0.3, 0.05), (0.7, 0.9), (1.0, 0.2)], window=(0.1, 0.8))
    vals = np.random.default_rng(5).uniform(-0.7, 1.8, 4096).astype(np.float32)
    vals[:4] = [-0.5, 1.5, 0.5, np.float32(-0.5 + 0.1 * 2.0)]
    out.update(tf_values=vals, tf_lut=tf.lut, tf_rgba=tf.apply(vals, -0.5, 1.5))
    # composites
    rng = np.random.default_rng(6)
    samples = rng.uniform(0, 1, (64, 4)).astype(np.float32)
    out.update(comp_samples=samples,
               comp_a=rr.composite_ray(samples, step=0.01, reference_step=0.02),
               comp_b=rr.composite_ray(samples, step=0.013, reference_step=0.02, background=(0.2, 0.3, 0.4, 0.5),
                                       early_exit_alpha=None),
               comp_c=rr.composite_ray(samples[:7], step=0.05, early_exit_alpha=0.5))
    # frames
    vol = rvol.synth_volume((17, 13, 11), [rvol.BlobSpec(center=(0.2, 0.0, -0.1), sigma=(0.4, 0.5, 0.3))])
    cam = rr.Camera(eye=(1.5, 1.0, 2.5), look_at=(0.0, 0.0, 0.0), width=12, height=10)
    cfg = rr.RenderConfig(samples_per_ray=16)
    out.update(vol_data=vol.data, vol_dims=np.array(vol.dims),
               img_volume=rr.render_frame(rr.VolumeField(vol), cam, rr.TransferFunction(), cfg))
    small = rmodel.init_model(rmodel.ModelConfig(grids=2, channels=1, resolution=(4, 4, 4)), seed=2, vmin=0.0,
                              vmax=1.0)
    small.grids[:] = np.random.default_rng(0).normal(size=small.grids.shape).astype(np.float32)
    out.update(model_arrays("small_", small))
    cam2 = rr.Camera(eye=(0.0, 0.5, 2.9), look_at=(0.0, 0.0, 0.0), width=9, height=9)
    out["img_small"] = rr.render_frame(rr.ModelField(small), cam2, rr.TransferFunction(),
                                       rr.RenderConfig(samples_per_ray=8))
    big = perturbed_model(11, 64, 2, (8, 8, 8), np.float32)
    out.update(model_arrays("big_", big))
    cam3 = rr.Camera(eye=(-1.2, 0.9, 2.2), look_at=(0.1, 0.0, 0.0), fov_deg=50, width=16, height=12)
    cfg3 = rr.RenderConfig(samples_per_ray=24, background=(0.05, 0.05, 0.1, 1.0), early_exit_alpha=0.95)
    out["img_big"] = rr.render_frame(rr.ModelField(big), cam3, tf, cfg3)
    np.savez_compressed(OUT / "render.npz", **out)


def _c1_run(iters, delay, pert, batch=2 ** 14):
    """C1-shaped reference run; pert > 0 nudges a random half of the initial grid values by one
    ulp (the size of a different summation order) to measure the reference's own sensitivity."""
    vol = rvol.synth_volume((128, 128, 128), adaptivity_blobs())
    m = rmodel.init_model(rmodel.ModelConfig(grids=64, channels=2, resolution=(32, 32, 32)), seed=0,
                          vmin=vol.vmin, vmax=vol.vmax)
    if pert:
        rng = np.random.default_rng(pert)
        mask = rng.uniform(size=m.grids.shape) < 0.5
        m.grids[mask] = np.nextafter(m.grids[mask], np.float32(np.inf if pert % 2 else -np.inf))
    cfg = rtrain.TrainConfig(iterations=iters, batch_size=batch, delay_start=delay, seed=0, plateau_enabled=False)
    m, log = rtrain.train_single(m, vol, cfg)
    return rtrain.psnr(m, vol), log


def gen_train_c1_short():
    """60 iterations (density active for the last 20): short enough that trajectories which
    differ by rounding have not decorrelated, so a 0.1 dB PSNR gate is meaningful."""
    p, log = _c1_run(60, 40, 0)
    np.savez_compressed(OUT / "train_c1_60.npz", psnr=np.array(p), config=np.array([60, 2 ** 14, 40]),
                        log_l_rec=np.array(log.l_rec),
                        log_stop=np.array(-1 if log.transform_stop_iteration is None else log.transform_stop_iteration),
                        log_l_density=np.array([np.nan if v is None else v for v in log.l_density]))


def gen_train_c1_ensemble():
    """Reference-vs-reference spread after 60/200/600 iterations under one-ulp perturbations
    (written to train_c1_ensemble.json; ~5 min per 200-iteration run on 8 cores)."""
    import json
    out = {"psnr_unperturbed": _c1_run(200, 50, 0)[0],
           "psnr_perturbed": [_c1_run(200, 50, p)[0] for p in (1, 2, 3, 4)],
           "c60": {"iterations": 60, "delay_start": 40, "psnr": [_c1_run(60, 40, p)[0] for p in (0, 1, 2, 3)]}}
    (OUT / "train_c1_ensemble.json").write_text(json.dumps(out, indent=1))


def gen_crit5_ensemble():
    """Acceptance criterion 5's configuration (8 grids 8^3 x1, 5000 iterations, batch 2048) run by
    the reference: the adaptive PSNR unperturbed and under four one-ulp perturbations of the initial
    grids, plus the frozen-transform PSNR of seeds 0-2 (~90 s per run on 2 cores).  Written to
    crit5_ensemble.json (the committed numbers came from this function)."""
    import json
    vol = rvol.synth_volume((64, 64, 64), adaptivity_blobs())

    def run(seed, adaptive, pert=0):
        m = rmodel.init_model(rmodel.ModelConfig(grids=8, channels=1, resolution=(8, 8, 8)), seed=seed,
                              vmin=vol.vmin, vmax=vol.vmax)
        if pert:
            rng = np.random.default_rng(pert)
            mask = rng.uniform(size=m.grids.shape) < 0.5
            m.grids[mask] = np.nextafter(m.grids[mask], np.float32(np.inf if pert % 2 else -np.inf))
        m, _ = rtrain.train_single(m, vol, rtrain.TrainConfig(iterations=5000, batch_size=2048, seed=seed,
                                                              train_transforms=adaptive, plateau_enabled=False))
        return rtrain.psnr(m, vol)
    out = {"adaptive_psnr_unperturbed": run(0, True), "adaptive_psnr_perturbed": [run(0, True, p) for p in (1, 2, 3, 4)],
           "frozen_psnr_unperturbed": run(0, False),
           "criterion_5_reference_gaps_seeds_0_1_2": [run(s, True) - run(s, False) for s in (0, 1, 2)]}
    (OUT / "crit5_ensemble.json").write_text(json.dumps(out, indent=1))



def gen_to_local():
    """model.py:179-182 to_local on sheared/translated transforms, f32 and f64, incl. points that
    map outside [-1, 1]^3 (the exported apmg_to_local)."""
    out = {}
    rng = np.random.default_rng(77)
    for tag, dt in (("f32", np.float32), ("f64", np.float64)):
        for k in range(3):
            tf = np.eye(4, dtype=dt)
            tf[:3, :3] += rng.normal(scale=0.3, size=(3, 3)).astype(dt)
            tf[:3, 3] = rng.normal(scale=0.4, size=3).astype(dt)
            pts = rng.uniform(-1.3, 1.3, (1000 + 7 * k, 3)).astype(dt)
            out[f"{tag}_{k}_tf"] = tf
            out[f"{tag}_{k}_pts"] = pts
            out[f"{tag}_{k}_local"] = rmodel.to_local(tf, pts)
    np.savez_compressed(OUT / "to_local.npz", **out)

C1_300_MEMBERS = (0, 1, 2, 3, 4, 5, 6, 7)


def gen_train_c1_300_member(pert):
    """BASELINE.md section 3's C1 parity configuration run by the reference (trainer.py:160-223):
    300 iterations, delay_start 100 (hard stop at 240), batch 2^16, plateau off, seed 0.
    ``pert`` 0 is the unperturbed run; 1..5 nudge a random half of the initial grid values by one
    ulp (the reference's own sensitivity to rounding).  ~30 min per member on 2 cores; members
    run as separate processes and are merged by gen_train_c1_300."""
    import json
    t0 = time.perf_counter()
    p, log = _c1_run(300, 100, int(pert), batch=2 ** 16)
    rec = {"pert": int(pert), "psnr": p, "wall_seconds": time.perf_counter() - t0,
           "l_rec": [float(v) for v in log.l_rec],
           "l_density": [None if v is None else float(v) for v in log.l_density],
           "transform_stop_iteration": log.transform_stop_iteration}
    (OUT / f"_c1_300_m{int(pert)}.json").write_text(json.dumps(rec))


def gen_train_c1_300():
    """Merge the per-member runs into train_c1_300.json (the committed fixture)."""
    import json
    mem = [json.loads((OUT / f"_c1_300_m{p}.json").read_text()) for p in C1_300_MEMBERS]
    out = {"config": {"iterations": 300, "batch_size": 2 ** 16, "delay_start": 100, "seed": 0,
                      "plateau_enabled": False, "volume": "128^3 adaptivity blobs",
                      "model": "64 grids 32^3 x2, init_model(seed=0)",
                      "perturbation": "one-ulp nudge of a random half of the initial grid values"},
           "psnr_unperturbed": mem[0]["psnr"],
           "psnr_perturbed": [m["psnr"] for m in mem[1:]],
           "unperturbed_log": {k: mem[0][k] for k in ("l_rec", "l_density", "transform_stop_iteration")},
           "wall_seconds": [m["wall_seconds"] for m in mem],
           "generated_by": "tests/golden/make_golden.py train_c1_300_member <p> + train_c1_300 (reference, CPU)"}
    (OUT / "train_c1_300.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["encode_forward", "recon", "density", "adam", "philox", "volume",
                             "train_small", "hash_decomp", "psnr", "train_c1"]
    if which[0] == "train_c1_300_member":
        gen_train_c1_300_member(which[1])
        sys.exit(0)
    for name in which:
        t0 = time.perf_counter()
        globals()["gen_" + name]()
        print(f"{name}: {time.perf_counter() - t0:.1f}s", flush=True)
