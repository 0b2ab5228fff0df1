"""Renderer oracle (oracle/render_oracle.py) pinned to the reference renderer's own outputs
(tests/golden/render.npz, tests/golden/make_golden.py gen_render), plus the renderer's host
logic (camera / transfer-function validation, LUT baking, progressive schedule).  CPU only."""
import numpy as np
import pytest

from oracle import apmg_oracle as O
from oracle import render_oracle as R
from paper_2308_02494_b200 import render as PR

TF_COLORS = [(0.0, (0.0, 0.0, 0.1)), (0.4, (1.0, 0.2, 0.0)), (1.0, (1.0, 1.0, 1.0))]
TF_ALPHA = [(0.0, 0.0), (0.3, 0.05), (0.7, 0.9), (1.0, 0.2)]


def params(g, prefix):
    meta, rng = g[prefix + "meta"], g[prefix + "range"]
    return O.Params(g[prefix + "transforms"].copy(), g[prefix + "grids"].copy(), g[prefix + "w1"].copy(),
                    g[prefix + "w2"].copy(), g[prefix + "w3"].copy(), float(rng[0]), float(rng[1]), int(meta[5]))


def test_box_hits_bit_exact(golden):
    g = golden("render")
    e, x, h = R.box_hits(g["rb_origin"], g["rb_dirs"])
    assert np.array_equal(e, g["rb_enter"]) and np.array_equal(x, g["rb_exit"]) and np.array_equal(h, g["rb_hit"])
    e, x, h = R.box_hits(np.zeros(3), np.array([[1.0, 0.0, 0.0], [0.0, 0.0, -1.0]]))
    assert np.array_equal(e, g["rb0_enter"]) and np.array_equal(x, g["rb0_exit"]) and np.array_equal(h, g["rb0_hit"])
    assert np.array_equal(R.box_hits(np.array([0.0, 2.0, 5.0]), np.array([[0.0, 0.0, -1.0]]))[2], g["rb1_hit"])


def test_lut_and_lookup_bit_exact(golden):
    g = golden("render")
    lut = R.bake_lut(TF_COLORS, TF_ALPHA)
    assert np.array_equal(lut, g["tf_lut"])
    assert np.array_equal(PR.TransferFunction(TF_COLORS, TF_ALPHA, (0.1, 0.8)).lut, g["tf_lut"])
    assert np.array_equal(R.tf_lookup(lut, (0.1, 0.8), g["tf_values"], -0.5, 1.5), g["tf_rgba"])


def test_composite_bit_exact(golden):
    g = golden("render")
    s = g["comp_samples"]
    one = lambda smp, step, ref, bg, early: R.composite(smp[None], np.array([step], np.float32), ref, bg, early)[0]  # noqa
    assert np.array_equal(one(s, 0.01, 0.02, (0, 0, 0, 1), 0.99), g["comp_a"])
    assert np.array_equal(one(s, 0.013, 0.02, (0.2, 0.3, 0.4, 0.5), None), g["comp_b"])
    assert np.array_equal(one(s[:7], 0.05, PR.DEFAULT_REFERENCE_STEP, (0, 0, 0, 1), 0.5), g["comp_c"])


def test_frames_bit_exact(golden):
    g = golden("render")
    vol = g["vol_data"]
    w, h, d = (int(v) for v in g["vol_dims"])
    diag = float(np.linalg.norm([2.0 / (n - 1) for n in (w, h, d)]))
    origin, dirs = R.rays((1.5, 1.0, 2.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 45.0, 12, 10)
    img = R.render(lambda p: O.sample_volume(vol, p.astype(np.float64)).astype(np.float32), float(vol.min()),
                   float(vol.max()), origin, dirs, R.bake_lut([(0.0, (0, 0, 0)), (1.0, (1, 1, 1))],
                                                              [(0.0, 0.0), (1.0, 1.0)]),
                   (0.0, 1.0), 16, diag)
    assert np.array_equal(img.reshape(10, 12, 4), g["img_volume"])
    small = params(g, "small_")
    origin, dirs = R.rays((0.0, 0.5, 2.9), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 45.0, 9, 9)
    img = R.render(lambda p: O.forward(small, p), small.vmin, small.vmax, origin, dirs,
                   R.bake_lut([(0.0, (0, 0, 0)), (1.0, (1, 1, 1))], [(0.0, 0.0), (1.0, 1.0)]), (0.0, 1.0), 8,
                   PR.DEFAULT_REFERENCE_STEP)
    assert np.array_equal(img.reshape(9, 9, 4), g["img_small"])
    big = params(g, "big_")
    origin, dirs = R.rays((-1.2, 0.9, 2.2), (0.1, 0.0, 0.0), (0.0, 1.0, 0.0), 50.0, 16, 12)
    img = R.render(lambda p: O.forward(big, p), big.vmin, big.vmax, origin, dirs, R.bake_lut(TF_COLORS, TF_ALPHA),
                   (0.1, 0.8), 24, PR.DEFAULT_REFERENCE_STEP, background=(0.05, 0.05, 0.1, 1.0), early_exit=0.95)
    assert np.array_equal(img.reshape(12, 16, 4), g["img_big"])


def test_package_rays_match_oracle():
    cam = PR.Camera(eye=(-1.2, 0.9, 2.2), look_at=(0.1, 0.0, 0.0), fov_deg=50, width=16, height=12)
    o1, d1 = PR.generate_rays(cam)
    o2, d2 = R.rays(cam.eye, cam.look_at, cam.up, cam.fov_deg, cam.width, cam.height)
    assert np.array_equal(o1, o2) and np.array_equal(d1, d2)


def test_camera_and_tf_validation():
    with pytest.raises(PR.RenderError, match="coincide"):
        PR.Camera(eye=(0, 0, 1), look_at=(0, 0, 1))
    with pytest.raises(PR.RenderError, match="parallel"):
        PR.Camera(eye=(0, 0, 2), look_at=(0, 0, 0), up=(0, 0, 1))
    with pytest.raises(PR.RenderError, match="field of view"):
        PR.Camera(eye=(0, 0, 2), look_at=(0, 0, 0), fov_deg=180.0)
    with pytest.raises(PR.RenderError, match="window"):
        PR.TransferFunction(window=(0.8, 0.2))
    with pytest.raises(PR.RenderError, match="outside"):
        PR.TransferFunction(opacity_points=[(1.5, 0.3)])
    with pytest.raises(PR.RenderError, match=">= 1"):
        PR.RenderConfig(samples_per_ray=0)
    cam = PR.Camera(eye=(1, 2, 3), look_at=(0, 0.5, 0), up=(0, 1, 0), fov_deg=30, width=64, height=48)
    assert PR.Camera.from_json(cam.to_json()) == cam
    tf = PR.TransferFunction(TF_COLORS, TF_ALPHA, (0.1, 0.8))
    back = PR.TransferFunction.from_json(tf.to_json())
    assert np.array_equal(back.lut, tf.lut) and back.window == tf.window


def test_progressive_schedule():
    assert [len(px) for _, _, px in PR.progressive_schedule(4, 4)] == [1, 3, 12]
    assert [s for _, s, _ in PR.progressive_schedule(16, 16)] == [16, 8, 4, 2, 1]
    assert PR.progressive_schedule(1, 1)[0][2].tolist() == [[0, 0]]
    for w, h in [(5, 3), (16, 16), (7, 1), (1, 9), (13, 10)]:
        seen = np.zeros((h, w), dtype=int)
        for _, _, px in PR.progressive_schedule(w, h):
            seen[px[:, 1], px[:, 0]] += 1
        assert np.array_equal(seen, np.ones_like(seen))


def test_png_encoding():
    img = np.random.default_rng(0).uniform(-0.2, 1.2, (5, 7, 4)).astype(np.float32)
    a, b = PR.image_to_png_bytes(img), PR.image_to_png_bytes(img)
    assert a == b and a[:8] == b"\x89PNG\r\n\x1a\n"
