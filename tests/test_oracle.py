"""Pin the CPU oracle against fixtures produced by running the reference itself.

tests/golden/*.npz come from tests/golden/make_golden.py (reference imported
from /root/reference in the build container).  These run on CPU."""
import json

import numpy as np
import pytest

from oracle import apmg_oracle as O


def params_from(g, prefix):
    meta = g[prefix + "meta"]
    rng = g[prefix + "range"]
    return O.Params(g[prefix + "transforms"].copy(), g[prefix + "grids"].copy(), g[prefix + "w1"].copy(),
                    g[prefix + "w2"].copy(), g[prefix + "w3"].copy(), float(rng[0]), float(rng[1]),
                    int(meta[5]))


@pytest.mark.parametrize("prefix", ["a32_", "a64_", "b32_", "c32_", "d32_"])
def test_encode_forward_bit_exact(golden, prefix):
    g = golden("encode_forward")
    prm = params_from(g, prefix)
    feats = O.encode(prm, g[prefix + "pts"])
    assert feats.dtype == g[prefix + "feats"].dtype
    assert np.array_equal(feats, g[prefix + "feats"])
    assert np.array_equal(O.forward(prm, g[prefix + "pts"]), g[prefix + "out"])


@pytest.mark.parametrize("prefix", ["a32_", "a64_", "b32_", "c64_"])
def test_recon_matches_reference(golden, prefix):
    g = golden("recon")
    prm = params_from(g, prefix)
    loss, sq, grads = O.recon_loss_and_grads(prm, g[prefix + "coords"], g[prefix + "targets"])
    assert loss == float(g[prefix + "loss"])
    assert np.array_equal(sq, g[prefix + "sq"])
    for k in ("grids", "w1", "w2", "w3"):
        ref = g[prefix + "g_" + k]
        assert grads[k].dtype == ref.dtype
        np.testing.assert_allclose(grads[k], ref, rtol=0, atol=1e-6 * max(np.abs(ref).max(), 1e-30))


@pytest.mark.parametrize("prefix", ["a32_", "a64_", "b32_", "u64_"])
def test_density_matches_reference(golden, prefix):
    g = golden("density")
    prm = params_from(g, prefix)
    loss, dg = O.density_loss_and_grads(prm, g[prefix + "coords"], g[prefix + "errors"])
    assert loss == pytest.approx(float(g[prefix + "loss"]), rel=1e-12, abs=1e-300)
    np.testing.assert_array_equal(dg["transforms"], g[prefix + "g_transforms"])
    _, _, _, rho = O.density_terms(prm.transforms, g[prefix + "coords"], prm.p)
    np.testing.assert_array_equal(rho, g[prefix + "rho"])
    rs = O.normalize_density(rho)
    np.testing.assert_array_equal(rs, g[prefix + "rho_scaled"])
    star = O.warped_target(rs, g[prefix + "errors"], float(g[prefix + "errors"].mean()))
    np.testing.assert_array_equal(star, g[prefix + "rho_star"])
    e = g[prefix + "errors"]
    if np.all(e == e.mean()):
        assert np.array_equal(star, rs + O.DENS_EPS)  # exact unit-exponent branch


@pytest.mark.parametrize("prefix", ["f32_", "f64_"])
def test_adam_matches_reference(golden, prefix):
    g = golden("adam")
    params = {"w": g[prefix + "p0"].copy()}
    st = O.AdamMoments(params)
    for step in range(len(g[prefix + "grads"])):
        O.adam_update(params, {"w": g[prefix + "grads"][step]}, st, float(g[prefix + "lrs"][step]))
        assert np.array_equal(params["w"], g[prefix + "traj"][step])
        assert np.array_equal(st.m["w"], g[prefix + "m"][step])
        assert np.array_equal(st.v["w"], g[prefix + "v"][step])


def test_philox_restatement_matches_numpy(golden):
    g = golden("philox")
    for key in [k for k in g if k.endswith("_key")]:
        tag = key[:-4]
        seed = int(tag.split("_")[0][1:])
        b = int(tag.split("_")[1][1:])
        assert tuple(int(v) for v in g[key]) == O.philox_key(seed)
        assert np.array_equal(O.philox_raw(seed, 0, 16), g[tag + "_raw"])
        draws = g[tag + "_draws"]
        for it in range(len(draws)):
            assert np.array_equal(O.batch_coords(seed, it, b), draws[it])
            # the device convention: coordinate (n, a) of iteration k is word 3(kB+n)+a
            words = O.philox_raw(seed, 3 * b * it, 3 * b)
            u = -1.0 + 2.0 * ((words >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
            assert np.array_equal(u.reshape(b, 3), draws[it])


def test_volume_sampling_and_synth(golden):
    g = golden("volume")
    blobs = [((0.2, -0.1, 0.3), (0.35, 0.3, 0.4), 1.0), ((-0.5, 0.4, -0.2), (0.1, 0.2, 0.15), 0.7)]
    assert np.array_equal(O.synth_volume((7, 6, 5), blobs, background=0.25), g["v1_data"])
    assert np.array_equal(O.synth_volume((9, 8, 10), blobs, seed=3, noise=0.05), g["v2_data"])
    assert np.array_equal(O.synth_volume((5, 1, 4), blobs), g["v3_data"])
    assert np.array_equal(O.synth_volume((64, 48, 40), blobs, background=0.1), g["big_data"])
    for tag in ("v1", "v2", "v3"):
        assert np.array_equal(O.sample_volume(g[tag + "_data"], g["pts"]), g[tag + "_samples"])
    with pytest.raises(ValueError, match="outside"):
        O.sample_volume(g["v1_data"], np.array([[1.0001, 0.0, 0.0]]))


def _check_log(log, g, prefix):
    assert log.iterations_run == int(g[prefix + "iters"])
    np.testing.assert_array_equal(np.array(log.l_rec), g[prefix + "l_rec"])
    ld = np.array([np.nan if v is None else v for v in log.l_density])
    np.testing.assert_array_equal(ld, g[prefix + "l_density"])
    np.testing.assert_array_equal(np.array(log.lr), g[prefix + "lr"])
    stop = -1 if log.transform_stop_iteration is None else log.transform_stop_iteration
    assert stop == int(g[prefix + "stop"])
    assert log.plateau_trigger_iterations == list(g[prefix + "triggers"])


def test_train_single_bit_exact_small(golden):
    g = golden("train_small")
    prm = params_from(g, "init_")
    log = O.train_single(prm, g["blob_data"], O.LoopConfig(iterations=40, batch_size=64, delay_start=5,
                                                           seed=9, plateau_enabled=False))
    _check_log(log, g, "log_")
    fin = params_from(g, "final_")
    for k in ("transforms", "grids", "w1", "w2", "w3"):
        np.testing.assert_array_equal(getattr(prm, k), getattr(fin, k))
    assert O.psnr(lambda p: O.forward(prm, p), g["blob_data"]) == pytest.approx(float(g["psnr"]), abs=1e-9)


def test_train_hard_stop_and_plateau(golden):
    g = golden("train_small")
    init = params_from(g, "init_")
    log = O.train_single(init, g["blob_data"], O.LoopConfig(iterations=100, batch_size=32, delay_start=10,
                                                            transform_hard_stop_fraction=0.5,
                                                            plateau_enabled=False, seed=3))
    _check_log(log, g, "hslog_")
    const = np.full((8, 8, 8), 3.25, dtype=np.float32)
    prm = O.init_params(4, 1, (4, 4, 4), seed=0, vmin=3.25, vmax=3.25)
    log = O.train_single(prm, const, O.LoopConfig(iterations=4000, batch_size=64, seed=1))
    _check_log(log, g, "const_")


def test_init_matches_reference(golden):
    g = golden("train_small")
    prm = O.init_params(4, 1, (4, 4, 4), seed=9, vmin=float(g["init_range"][0]), vmax=float(g["init_range"][1]))
    ref = params_from(g, "init_")
    for k in ("transforms", "grids", "w1", "w2", "w3"):
        assert np.array_equal(getattr(prm, k), getattr(ref, k))


def test_psnr_matches_reference(golden):
    g = golden("psnr")
    prm = params_from(g, "m_")
    assert O.psnr(lambda p: O.forward(prm, p), g["vol"]) == pytest.approx(float(g["psnr"]), abs=1e-9)
    assert O.psnr(lambda p: O.forward(prm, p), g["vol"], chunk=7) == pytest.approx(float(g["psnr_b7"]), abs=1e-9)


def test_hash_and_decomposed_forward(golden):
    g = golden("hash_decomp")
    for key in [k for k in g if k.startswith("hash_") and k.endswith("_pts")]:
        tag = key[5:-4]
        counts = tuple(int(v) for v in tag.split("x"))
        assert np.array_equal(O.brick_of(g[key], counts), g["hash_" + tag + "_owner"])
    man = json.loads(bytes(g["dec_manifest"]).decode())
    counts = (man["I"], man["J"], man["K"])
    dims = tuple(man["volume_header"]["dims"])
    scale, offset = O.brick_affines(dims, counts, man["ghost"])
    assert np.array_equal(scale, g["dec_scale"]) and np.array_equal(offset, g["dec_offset"])
    ext = O.brick_extents(dims, counts, man["ghost"])
    for b, entry in enumerate(man["bricks"]):
        assert tuple(entry["core_lo"]) == ext[b][0] and tuple(entry["ghost_hi"]) == ext[b][3]
        assert entry["seed"] == O.brick_seed(7, b)
    models = [params_from(g, f"dec_m{i}_") for i in range(int(g["dec_count"]))]
    out = O.decomposed_forward(models, counts, scale, offset, g["dec_pts"])
    assert np.array_equal(out, g["dec_out"])
    p = O.psnr(lambda q: O.decomposed_forward(models, counts, scale, offset, q), g["dec_vol"])
    assert p == pytest.approx(float(g["dec_psnr"]), abs=1e-9)


@pytest.mark.parametrize("tag", ["f32_0", "f32_1", "f32_2", "f64_0", "f64_1", "f64_2"])
def test_to_local_bit_exact(golden, tag):
    """oracle.grid_local vs the reference's to_local (model.py:179-182), incl. einsum's
    dtype-dependent summation order."""
    g = golden("to_local")
    assert np.array_equal(O.grid_local(g[tag + "_tf"], g[tag + "_pts"]), g[tag + "_local"])


def test_threaded_cpu_baseline_matches_serial_oracle():
    """The bench's reference arm (oracle.train_single_threaded: batch slices on host threads)
    takes the same training steps as the serial restatement, up to the association of the
    batch sums."""
    prm = O.init_params(8, 2, (8, 8, 8), seed=1, vmin=0.0, vmax=1.0)
    prm.transforms[:, :3, :3] += np.random.default_rng(2).normal(scale=0.1, size=(8, 3, 3)).astype(np.float32)
    vol = O.synth_volume((20, 18, 16), [((0.1, -0.2, 0.3), (0.4, 0.3, 0.5), 1.0)])
    cfg = O.LoopConfig(iterations=3, batch_size=3000, delay_start=1, transform_hard_stop_fraction=1.0,
                       plateau_enabled=False, seed=4)
    a, b = prm.copy(), prm.copy()
    la = O.train_single(a, vol, cfg)
    lb = O.train_single_threaded(b, vol, cfg, threads=3)
    np.testing.assert_allclose(lb.l_rec, la.l_rec, rtol=1e-6)
    np.testing.assert_allclose([v or 0.0 for v in lb.l_density], [v or 0.0 for v in la.l_density], rtol=1e-6)
    for k in ("grids", "w1", "w2", "w3", "transforms"):
        np.testing.assert_allclose(getattr(b, k), getattr(a, k), rtol=0, atol=2e-5)
