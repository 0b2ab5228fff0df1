"""Single-model training loop and evaluation.

Mirror of the reference ``apmg.trainer`` API (trainer.py:1-247).  ``train_single``
runs the whole loop on the GPU (libapmg_cuda ``apmg_train_*``): Philox batch
generation, fp64 target sampling, the fused reconstruction step, masked Adam,
the delayed/gated density step and the plateau scheduler all execute as
device kernels enqueued back to back; the host only polls for an early stop
every few dozen iterations and copies the log once at the end.

``plateau_step`` and ``transform_stop_check`` call the library's host hooks,
which compile the SAME rule code the device controller runs.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .model import ApmgModel, DeviceModel
from .volume import Volume

__all__ = ["TrainConfig", "TrainLog", "PlateauState", "plateau_step", "transform_stop_check", "train_single",
           "psnr", "PSNR_CAP_DB", "TrainSession"]

PSNR_CAP_DB = 200.0


@dataclass
class TrainConfig:
    """trainer.py:37-67."""
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
    # not in the reference (always deterministic on the CPU): True makes GPU training
    # bit-reproducible run to run (stable batch order, fixed-point grid gradients) at some
    # speed cost; APMG_DETERMINISTIC=1 forces it for every session
    deterministic: bool = False

    def __post_init__(self):
        if self.iterations < 0 or self.batch_size < 1:
            raise ValueError("iterations must be >= 0 and batch_size >= 1")
        if self.iterations > 0 and self.delay_start >= self.iterations:
            raise ValueError("delay_start must be < iterations")
        for name in ("lr_main", "lr_transform", "transform_ma_window", "plateau_window",
                     "transform_improve_threshold", "plateau_threshold", "plateau_factor"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    @property
    def hard_stop_iteration(self) -> int:
        return int(np.ceil(self.transform_hard_stop_fraction * self.iterations))


@dataclass
class TrainLog:
    """Per-iteration history (trainer.py:70-102)."""
    l_rec: list = field(default_factory=list)
    l_density: list = field(default_factory=list)
    lr: list = field(default_factory=list)
    transform_stop_iteration: int | None = None
    plateau_trigger_iterations: list = field(default_factory=list)
    iterations_run: int = 0
    wall_seconds: float = 0.0
    setup_seconds: float = 0.0  # volume / parameter upload and session creation (train_single)
    setup_ms: dict = field(default_factory=dict)  # its split (TrainSession.setup_ms)
    loop_ms: float = 0.0  # device time of the iterations (CUDA events on the session's stream)

    def records(self):
        stop = self.transform_stop_iteration
        for i in range(self.iterations_run):
            yield {
                "iter": i, "l_rec": self.l_rec[i], "l_density": self.l_density[i], "lr": self.lr[i],
                "flags": {"transform_frozen": stop is not None and i >= stop,
                          "plateau_triggers": sum(1 for t in self.plateau_trigger_iterations if t <= i)},
            }

    def write_jsonl(self, path) -> None:
        with open(path, "w") as f:
            for rec in self.records():
                f.write(json.dumps(rec) + "\n")


@dataclass
class PlateauState:
    """trainer.py:105-115."""
    lr: float
    window: int
    threshold: float
    factor: float
    max_triggers: int
    history: list = field(default_factory=list)
    triggers: int = 0


def plateau_step(state: PlateauState, current_ma: float) -> str:
    """Advance the plateau scheduler (trainer.py:118-138) through the device rule's host build."""
    cap = state.window + 1
    count = len(state.history)
    ring = np.zeros(cap)
    for i in range(max(0, count - cap), count):
        ring[i % cap] = state.history[i]
    cnt = C.c_int64(count)
    trig = C.c_int64(state.triggers)
    act = L.lib().apmg_host_plateau_step(ring.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cnt), C.byref(trig),
                                         state.window, float(state.threshold), state.max_triggers, float(current_ma))
    if act == 0:
        state.history.append(current_ma)
        return "none"
    state.history.clear()
    state.triggers = int(trig.value)
    state.lr /= state.factor
    return "stop" if act == 2 else "reduce_lr"


def transform_stop_check(history, cfg: TrainConfig, iteration: int) -> bool:
    """trainer.py:141-157 through the device rule's host build."""
    h = np.ascontiguousarray(history, dtype=np.float64)
    if h.size == 0:
        h = np.zeros(1)
        count = 0
    else:
        count = len(history)
    return bool(L.lib().apmg_host_transform_stop(h.ctypes.data_as(C.POINTER(C.c_double)), count,
                                                 cfg.transform_ma_window, float(cfg.transform_improve_threshold),
                                                 cfg.hard_stop_iteration, iteration))


def _bias_table(n: int) -> np.ndarray:
    """(1 - 0.9^t, 1 - 0.99^t) for t = 1..n as Python floats (optim.py:57-58)."""
    tab = np.empty((max(n, 1), 2))
    for t in range(1, n + 1):
        tab[t - 1, 0] = 1.0 - 0.9 ** t
        tab[t - 1, 1] = 1.0 - 0.99 ** t
    return tab


# per-thread flag: sessions run from concurrent worker threads (train_decomposed workers > 1)
# use plain launches -- a CUDA-graph capture must not overlap other threads' CUDA calls
_concurrency = __import__("threading").local()

# The library caches its large per-session blocks (the corner-replicated training volume, up to
# a quarter of free device memory) so back-to-back sessions skip cudaMalloc / cudaFree.  A
# standalone train_single hands them back to the device when it returns; train_decomposed holds
# the cache across its bricks (hold_block_cache) and releases it at the end.
_cache_holders = [0]


class hold_block_cache:
    def __enter__(self):
        _cache_holders[0] += 1
        return self

    def __exit__(self, *exc):
        _cache_holders[0] -= 1
        if _cache_holders[0] == 0:
            release_parked_workspace()
            if L._lib is not None:  # nothing cached before the library loads
                L.lib().apmg_release_cached()


# One parked session workspace (the largest buffer of a session: ~4 GiB at C2 with the sampler's
# corner-replicated volume copy): inside hold_block_cache a closing session parks it and the next
# one takes it when it is large enough, so back-to-back sessions (repeated train_single calls, the
# bricks of train_decomposed) skip the allocation whatever the caching allocator's state; outside
# it the workspace goes back to torch at close.  Concurrent sessions allocate their own.
_ws_park = {"t": None}
_ws_lock = __import__("threading").Lock()


def _take_workspace(nbytes: int):
    with _ws_lock:
        t = _ws_park["t"]
        if t is not None and t.numel() >= nbytes:
            _ws_park["t"] = None
            return t[:nbytes]
    return L.workspace(nbytes)


def _park_workspace(t) -> None:
    if t is None or _cache_holders[0] == 0:  # parked only inside hold_block_cache
        return
    base = t._base if t._base is not None else t
    with _ws_lock:
        cur = _ws_park["t"]
        if cur is None or cur.numel() < base.numel():
            _ws_park["t"] = base


def release_parked_workspace() -> None:
    with _ws_lock:
        _ws_park["t"] = None


class TrainSession:
    """Owns the device copy of one model during training (main group in one flat
    buffer laid out by ``apmg_main_layout``) and the native loop state."""

    def __init__(self, model: ApmgModel, volume: Volume, cfg: TrainConfig):
        t = L.require_cuda()
        t0 = time.perf_counter()
        self.model, self.volume, self.cfg = model, volume, cfg
        dt = model.dtype
        if dt not in (np.float32, np.float64):
            raise TypeError(f"unsupported model dtype {dt}")
        self.dt = dt
        # the session plan first (workspace size; the sampler-copy budget queries free device memory,
        # which took 0.3-70 ms while a DMA was in flight), then the volume's DMA from the page-locked
        # host array is issued and left in flight; the parameters (17 MiB at the flagship shape)
        # are staged through the pinned ring while it runs (their copies queue behind it), then the
        # workspace; apmg_train_create (stream-ordered after both) returns synchronised
        tv = t0
        key = np.random.Philox(cfg.seed).state["state"]["key"]
        self.ccfg = L.ApmgTrainConfigC(
            cfg.iterations, cfg.batch_size, cfg.lr_main, cfg.lr_transform, cfg.delay_start,
            cfg.transform_ma_window, cfg.transform_improve_threshold, cfg.hard_stop_iteration,
            cfg.plateau_window, cfg.plateau_threshold, cfg.plateau_factor, cfg.plateau_max_triggers,
            int(key[0]), int(key[1]), int(bool(cfg.train_transforms)), int(bool(cfg.plateau_enabled)),
            int(bool(cfg.deterministic) or os.environ.get("APMG_DETERMINISTIC", "0") == "1"),
            1 if getattr(_concurrency, "no_graph", False) else 0)
        w, h, d = volume.dims
        shape = DeviceModel.shape_of(model)
        # session workspace + the sampler's private copy of the volume, both from torch's caching
        # allocator (reused by back-to-back sessions, released by torch under memory pressure)
        need = L.lib().apmg_train_workspace_bytes(C.byref(shape), C.byref(self.ccfg))
        need = (need + 255) // 256 * 256 + L.lib().apmg_train_volume_bytes(w, h, d)
        tp = time.perf_counter()
        self.vol = volume.device_data(sync=False)
        t1 = time.perf_counter()
        self.dm = DeviceModel.upload(model)
        off = (C.c_int64 * 5)()
        L.check(L.lib().apmg_main_layout(C.byref(self.dm.desc), off), "main_layout")
        self.off = [int(v) for v in off]
        self.main = L.zeros((self.off[4],), dt)
        o = self.off
        self.main[o[0]:o[0] + self.dm.grids_cl.numel()].copy_(self.dm.grids_cl.reshape(-1))
        self.main[o[1]:o[1] + self.dm.w1.numel()].copy_(self.dm.w1.reshape(-1))
        self.main[o[2]:o[2] + self.dm.w2.numel()].copy_(self.dm.w2.reshape(-1))
        self.main[o[3]:o[3] + self.dm.w3.numel()].copy_(self.dm.w3.reshape(-1))
        self.tf = self.dm.transforms
        t2 = time.perf_counter()
        self.ws = _take_workspace(need)
        t3 = time.perf_counter()
        bias = _bias_table(cfg.iterations)
        st = C.c_void_p()
        L.check(L.lib().apmg_train_create(C.byref(st), C.byref(self.dm.desc), L.ptr(self.main), L.ptr(self.tf),
                                          L.ptr(self.vol), w, h, d, C.byref(self.ccfg),
                                          bias.ctypes.data_as(C.POINTER(C.c_double)), L.ptr(self.ws), self.ws.numel(),
                                          L.stream_handle()), "train_create")
        self.state = st
        self._torch = t
        # host-side setup split (ms): plan, volume DMA issue, parameter upload (behind the DMA),
        # workspace, create (waits for the copies, builds the sampler's volume copy; synchronised)
        self.setup_ms = {"plan": 1e3 * (tp - tv), "volume": 1e3 * (t1 - tp), "params": 1e3 * (t2 - t1),
                         "workspace": 1e3 * (t3 - t2),
                         "create": 1e3 * (time.perf_counter() - t3)}

    def run(self, n: int) -> None:
        L.check(L.lib().apmg_train_run(self.state, int(n), L.stream_handle()), "train_run")

    def status(self) -> tuple[int, bool]:
        it = C.c_int64()
        fin = C.c_int32()
        L.check(L.lib().apmg_train_status(self.state, C.byref(it), C.byref(fin), L.stream_handle()), "train_status")
        return int(it.value), bool(fin.value)

    def pull_params(self) -> None:
        """Copy the device parameters back into the model's host arrays, in place."""
        m, o = self.model, self.off
        c = m.config
        gdev = self.main[o[0]:o[0] + m.grids.size].view(c.grids, *c.resolution, c.channels)
        gdev = gdev.permute(0, 4, 1, 2, 3).contiguous()  # channel-last device -> (G, C, ...) host layout
        if m.grids.flags.c_contiguous and m.grids.dtype == L.torch_to_np(gdev.dtype):
            L.download_into(gdev, m.grids)
        else:
            m.grids[...] = L.to_host(gdev)
        main = L.to_host(self.main[o[1]:])
        o = [x - o[1] for x in o]
        m.w1[...] = main[o[1]:o[1] + m.w1.size].reshape(m.w1.shape)
        m.w2[...] = main[o[2]:o[2] + m.w2.size].reshape(m.w2.shape)
        m.w3[...] = main[o[3]:o[3] + m.w3.size].reshape(m.w3.shape)
        m.transforms[...] = L.to_host(self.tf).reshape(m.transforms.shape)

    def push_params(self) -> None:
        """Re-upload host arrays (an on_iteration callback may have mutated them)."""
        m, o = self.model, self.off
        t = self._torch
        self.main[o[0]:o[0] + m.grids.size].copy_(
            t.from_numpy(np.ascontiguousarray(np.moveaxis(m.grids, 1, -1)).reshape(-1)))
        self.main[o[1]:o[1] + m.w1.size].copy_(t.from_numpy(np.ascontiguousarray(m.w1).reshape(-1)))
        self.main[o[2]:o[2] + m.w2.size].copy_(t.from_numpy(np.ascontiguousarray(m.w2).reshape(-1)))
        self.main[o[3]:o[3] + m.w3.size].copy_(t.from_numpy(np.ascontiguousarray(m.w3).reshape(-1)))
        self.tf.copy_(t.from_numpy(np.ascontiguousarray(m.transforms)))

    def log(self) -> TrainLog:
        n = self.cfg.iterations
        l_rec, l_den, lr = np.zeros(n), np.zeros(n), np.zeros(n)
        stop = C.c_int64()
        trig = np.zeros(max(self.cfg.plateau_max_triggers, 1), dtype=np.int64)
        ntrig = C.c_int64()
        dp = C.POINTER(C.c_double)
        L.check(L.lib().apmg_train_log(self.state, l_rec.ctypes.data_as(dp), l_den.ctypes.data_as(dp),
                                       lr.ctypes.data_as(dp), C.byref(stop),
                                       trig.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(ntrig),
                                       L.stream_handle()), "train_log")
        it, _ = self.status()
        log = TrainLog()
        log.iterations_run = it
        log.l_rec = [float(v) for v in l_rec[:it]]
        log.l_density = [None if math.isnan(v) else float(v) for v in l_den[:it]]
        log.lr = [float(v) for v in lr[:it]]
        log.transform_stop_iteration = None if stop.value < 0 else int(stop.value)
        log.plateau_trigger_iterations = [int(v) for v in trig[:ntrig.value]]
        return log

    def moments(self) -> dict:
        """Adam state after the iterations run so far (optim.py:38-44): host arrays in the
        reference's shapes -- {"grids" | "w1" | "w2" | "w3" | "transforms": (m, v)}."""
        t = self._torch
        mm, mv = L.zeros((self.off[4],), self.dt), L.zeros((self.off[4],), self.dt)
        tm, tv = L.zeros(tuple(self.tf.shape), self.dt), L.zeros(tuple(self.tf.shape), self.dt)
        L.check(L.lib().apmg_train_moments(self.state, L.ptr(mm), L.ptr(mv), L.ptr(tm), L.ptr(tv),
                                           L.stream_handle()), "train_moments")
        c, o = self.model.config, self.off
        out = {}
        for name, (a, b) in (("m", (mm, tm)), ("v", (mv, tv))):
            g = a[o[0]:o[0] + self.model.grids.size].view(c.grids, *c.resolution, c.channels)
            out.setdefault("grids", {})[name] = L.to_host(g.permute(0, 4, 1, 2, 3).contiguous())
            for k, i in (("w1", 1), ("w2", 2), ("w3", 3)):
                shp = getattr(self.model, k).shape
                out.setdefault(k, {})[name] = L.to_host(a[o[i]:o[i] + int(np.prod(shp))]).reshape(shp)
            out.setdefault("transforms", {})[name] = L.to_host(b).reshape(self.model.transforms.shape)
        t.cuda.current_stream().synchronize()
        return {k: (v["m"], v["v"]) for k, v in out.items()}

    def close(self) -> None:
        if self.state:
            L.lib().apmg_train_destroy(self.state)
            self.state = None
        # the workspace (incl. the sampler's 8x volume copy) is parked for the next session now, not
        # released when the garbage collector gets to this one
        _park_workspace(getattr(self, "ws", None))
        self.ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def train_single(model: ApmgModel, volume: Volume, cfg: TrainConfig, on_iteration=None,
                 chunk: int = 64) -> tuple[ApmgModel, TrainLog]:
    """Fit ``model`` to ``volume`` in place on the GPU (trainer.py:160-223).

    ``on_iteration(it, model)`` runs after each iteration's updates with the host
    arrays refreshed (and re-uploaded afterwards); without it the loop never
    synchronises except to poll for a plateau stop every ``chunk`` iterations."""
    log = TrainLog()
    if cfg.iterations == 0:
        return model, log
    t0 = time.perf_counter()
    sess = TrainSession(model, volume, cfg)
    setup = time.perf_counter() - t0  # apmg_train_create returns synchronised
    tcuda = L.torch().cuda
    ev0, ev1 = tcuda.Event(enable_timing=True), tcuda.Event(enable_timing=True)
    ev0.record()
    try:
        if on_iteration is None:
            done = 0
            while done < cfg.iterations:
                step = min(chunk, cfg.iterations - done)
                sess.run(step)
                done += step
                if done < cfg.iterations and sess.status()[1]:
                    break
        else:
            for it in range(cfg.iterations):
                sess.run(1)
                ran, finished = sess.status()
                if ran <= it:
                    break
                sess.pull_params()
                on_iteration(it, model)
                sess.push_params()
                if finished:
                    break
        ev1.record()
        sess.pull_params()
        log = sess.log()
    finally:
        sess.close()
        if _cache_holders[0] == 0:
            L.lib().apmg_release_cached()
    log.wall_seconds = time.perf_counter() - t0
    log.setup_seconds = setup
    log.setup_ms = {k: round(v, 2) for k, v in sess.setup_ms.items()}
    log.loop_ms = float(ev0.elapsed_time(ev1))
    return model, log


def _psnr_from_mse(mse: float, value_range: float) -> float:
    if mse == 0.0:
        return PSNR_CAP_DB
    return float(min(10.0 * np.log10(value_range * value_range / mse), PSNR_CAP_DB))


def lattice_sse_model(dm: DeviceModel, truth_dev, dims, box=None, scale=None, offset=None, sse=None, recon=None,
                      box_local: bool = False):
    """Add the SSE of ``dm`` over a voxel box of the (W,H,D) lattice to the device scalar ``sse``
    (and/or write its predictions to ``recon``).  ``box_local``: truth / recon are dense
    arrays of the box only, as a rank holding one brick of a larger volume has them."""
    w, h, d = dims
    if box is None:
        box = (0, w - 1, 0, h - 1, 0, d - 1)
    b = (C.c_int32 * 6)(*box)
    sc = (C.c_double * 3)(*scale) if scale is not None else None
    of = (C.c_double * 3)(*offset) if offset is not None else None
    fn = L.lib().apmg_brick_sweep if box_local else L.lib().apmg_lattice_sweep
    L.check(fn(C.byref(dm.desc), w, h, d, b, sc, of, L.ptr(truth_dev), L.ptr(sse), L.ptr(recon), L.stream_handle()),
            "lattice_sweep")


def psnr(field, volume: Volume, batch_size: int = 65536) -> float:
    """Data-space PSNR 10 log10(range^2 / MSE) over every voxel, capped at 200 dB (trainer.py:226-247).

    Models and decomposed fields are swept on the GPU (coordinates generated from
    the voxel index, fp64 SSE); any other callable is evaluated chunk by chunk."""
    value_range = volume.vmax - volume.vmin
    if value_range == 0.0:
        return PSNR_CAP_DB
    w, h, d = volume.dims
    count = w * h * d
    if isinstance(field, ApmgModel):
        sse = L.zeros((1,), np.float64)
        lattice_sse_model(field.device(), volume.device_data(), volume.dims, sse=sse)
        return _psnr_from_mse(float(sse.item()) / count, value_range)
    if hasattr(field, "lattice_sse"):
        return _psnr_from_mse(field.lattice_sse(volume) / count, value_range)
    predict = field.forward if isinstance(field, ApmgModel) else field
    pts = volume.lattice_coords()
    truth = volume.host_data().ravel()
    sq_sum = 0.0
    for lo in range(0, len(pts), batch_size):
        pred = np.asarray(predict(pts[lo:lo + batch_size].astype(np.float32)), dtype=np.float64)
        diff = pred - truth[lo:lo + batch_size]
        sq_sum += float((diff * diff).sum())
    return _psnr_from_mse(sq_sum / len(pts), value_range)
