"""ctypes binding of libapmg_cuda.so (the C ABI declared in include/apmg_cuda.h).

PyTorch is used only as plumbing: it owns device memory (tensors) and the
current CUDA stream; every computation runs in the library's sm_100a kernels.
There is no CPU fallback: if the library or a CUDA device is missing, calls
raise immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libapmg_cuda.so"
if os.environ.get("APMG_LIB"):  # A/B builds of the same sources (tools/ab_build.sh); never a fallback
    LIB_PATH = Path(os.environ["APMG_LIB"]).resolve()

APMG_F32, APMG_F64 = 0, 1
APMG_OK, APMG_E_ARG, APMG_E_CUDA, APMG_E_WORKSPACE, APMG_E_UNSUPPORTED = 0, -1, -2, -3, -4


class ApmgModelC(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("grids", C.c_int32), ("channels", C.c_int32), ("depth", C.c_int32),
        ("height", C.c_int32), ("width", C.c_int32), ("hidden", C.c_int32), ("flat_top_p", C.c_int32),
        ("transforms", C.c_void_p), ("grids_cl", C.c_void_p), ("w1", C.c_void_p), ("w2", C.c_void_p),
        ("w3", C.c_void_p), ("vmin", C.c_double), ("vmax", C.c_double),
    ]


class ApmgTrainConfigC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("batch_size", C.c_int64), ("lr_main", C.c_double),
        ("lr_transform", C.c_double), ("delay_start", C.c_int64), ("transform_ma_window", C.c_int64),
        ("transform_improve_threshold", C.c_double), ("hard_stop_iteration", C.c_int64),
        ("plateau_window", C.c_int64), ("plateau_threshold", C.c_double), ("plateau_factor", C.c_double),
        ("plateau_max_triggers", C.c_int64), ("key0", C.c_uint64), ("key1", C.c_uint64),
        ("train_transforms", C.c_int32), ("plateau_enabled", C.c_int32),
        ("deterministic", C.c_int32), ("reserved", C.c_int32),
    ]


_P = C.c_void_p
_I32, _I64, _U64, _D, _SZ = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
_MP = C.POINTER(ApmgModelC)

# name -> (restype, argtypes); mirrors include/apmg_cuda.h
SIGNATURES = {
    "apmg_last_error": (C.c_char_p, []),
    "apmg_version": (C.c_char_p, []),
    "apmg_device_sm_count": (C.c_int, []),
    "apmg_launch_count": (C.c_uint64, []),
    "apmg_release_cached": (C.c_int, []),
    "apmg_host_register": (C.c_int, [_P, C.c_size_t]),
    "apmg_host_unregister": (C.c_int, [_P]),
    "apmg_copy_h2d": (C.c_int, [_P, _P, C.c_size_t, _P]),
    "apmg_forward_tc": (C.c_int, [_MP, _P, _I64, _P, _P]),
    "apmg_generate_rays": (C.c_int, [C.POINTER(C.c_double), C.c_int32, C.c_int32, _P, _P]),
    "apmg_ray_box_hits": (C.c_int, [C.POINTER(C.c_double), _P, _I64, _P, _P, _P, _P]),
    "apmg_ray_points": (C.c_int, [C.POINTER(C.c_double), _P, _P, _I64, C.c_int32, C.c_int32, C.c_int32, _P, _P,
                                  _P, _P]),
    "apmg_tf_apply": (C.c_int, [_P, _I64, _P, C.POINTER(C.c_float), _P, _P]),
    "apmg_composite_chunk": (C.c_int, [_P, _P, _I64, C.c_int32, C.c_int32, _P, _P, _P, C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), _P, _P]),
    "apmg_composite_finish": (C.c_int, [_P, _I64, _P, C.POINTER(C.c_float), _P, _P]),
    "apmg_composite_rgba": (C.c_int, [_P, _P, _I64, C.c_int32, C.POINTER(C.c_float), _P, _P]),
    "apmg_kernel_timing_enable": (C.c_int, [C.c_int]),
    "apmg_kernel_timing_read": (C.c_int, [C.c_char_p, C.POINTER(_D), C.POINTER(_I64), C.c_int]),
    "apmg_to_local": (C.c_int, [_I32, _P, _P, _I64, _P, _P]),
    "apmg_encode": (C.c_int, [_MP, _P, _I64, _P, _P]),
    "apmg_decode": (C.c_int, [_MP, _P, _I64, _P, _P]),
    "apmg_forward": (C.c_int, [_MP, _P, _I64, _P, _P]),
    "apmg_recon_workspace_bytes": (_SZ, [_MP, _I64]),
    "apmg_recon_loss_grads": (C.c_int, [_MP, _P, _P, _I64, _P, _P, C.POINTER(_P), _P, _SZ, _P]),
    "apmg_density_workspace_bytes": (_SZ, [_I32, _I64]),
    "apmg_density_loss_grads": (C.c_int, [_MP, _P, _P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "apmg_feature_density": (C.c_int, [_I32, _P, _I32, _I32, _P, _I64, _P, _P]),
    "apmg_density_terms": (C.c_int, [_I32, _P, _I32, _I32, _P, _I64, _P, _P, _P, _P, _P]),
    "apmg_target_density": (C.c_int, [_P, _P, _I64, _D, _D, _P, _P]),
    "apmg_sum_workspace_bytes": (_SZ, [_I64]),
    "apmg_sum_f64": (C.c_int, [_P, _I64, _P, _P, _SZ, _P]),
    "apmg_density_loss_terms": (C.c_int, [_P, _P, _I64, _D, _P, _P]),
    "apmg_scale_f64": (C.c_int, [_P, _I64, _P, _P, _P]),
    "apmg_adam_step": (C.c_int, [_I32, _P, _P, _P, _P, _I64, _D, _D, _D, _P]),
    "apmg_philox_uniform": (C.c_int, [_U64, _U64, _U64, _I64, _D, _D, _P, _P]),
    "apmg_sample_volume": (C.c_int, [_P, _I32, _I32, _I32, _P, _I64, _P, _P, _P]),
    "apmg_synth_volume": (C.c_int, [_I32, _I32, _I32, _I32, _P, _P, _P, _P, _D, _U64, _U64, _D, _P, _P]),
    "apmg_spatial_hash": (C.c_int, [_I32, _P, _I64, _I32, _I32, _I32, _P, _P, _P]),
    "apmg_decomposed_workspace_bytes": (_SZ, [_I32, _I64]),
    "apmg_owner_bucket_workspace_bytes": (_SZ, [_I32]),
    "apmg_owner_bucket": (C.c_int, [_P, _I64, _I32, _P, C.POINTER(_I64), _P, _SZ, _P]),
    "apmg_permute_rows": (C.c_int, [_P, _P, _I64, _I32, _I32, _P, _P]),
    "apmg_decomposed_forward": (C.c_int, [_MP, _I32, _I32, _I32, _I32, C.POINTER(_D), C.POINTER(_D), _P, _I64,
                                          _P, _P, _SZ, _P]),
    "apmg_decomposed_forward_tc": (C.c_int, [_MP, _I32, _I32, _I32, _I32, C.POINTER(_D), C.POINTER(_D), _P, _I64,
                                          _P, _P, _SZ, _P]),
    "apmg_lattice_sweep": (C.c_int, [_MP, _I32, _I32, _I32, C.POINTER(_I32), C.POINTER(_D), C.POINTER(_D), _P,
                                     _P, _P, _P]),
    "apmg_brick_sweep": (C.c_int, [_MP, _I32, _I32, _I32, C.POINTER(_I32), C.POINTER(_D), C.POINTER(_D), _P,
                                   _P, _P, _P]),
    "apmg_main_layout": (C.c_int, [_MP, C.POINTER(_I64)]),
    "apmg_train_workspace_bytes": (_SZ, [_MP, C.POINTER(ApmgTrainConfigC)]),
    "apmg_train_volume_bytes": (_SZ, [_I32, _I32, _I32]),
    "apmg_train_create": (C.c_int, [C.POINTER(_P), _MP, _P, _P, _P, _I32, _I32, _I32,
                                    C.POINTER(ApmgTrainConfigC), C.POINTER(_D), _P, _SZ, _P]),
    "apmg_train_run": (C.c_int, [_P, _I64, _P]),
    "apmg_train_status": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I32), _P]),
    "apmg_train_log": (C.c_int, [_P, C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), C.POINTER(_I64),
                                 C.POINTER(_I64), C.POINTER(_I64), _P]),
    "apmg_train_destroy": (C.c_int, [_P]),
    "apmg_train_moments": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "apmg_host_plateau_step": (C.c_int, [C.POINTER(_D), C.POINTER(_I64), C.POINTER(_I64), _I64, _D, _I64, _D]),
    "apmg_host_transform_stop": (C.c_int, [C.POINTER(_D), _I64, _I64, _D, _I64, _I64]),
    "apmg_host_pairwise_sum": (_D, [C.POINTER(_D), _I64]),
    "apmg_debug_infer_phases": (C.c_int, [_P]),
    "apmg_debug_tc16_phases": (C.c_int, [_P]),
    "apmg_debug_tc16_warp_phases": (C.c_int, [_P]),
}

_lib = None


class ApmgLibraryError(RuntimeError):
    """The CUDA extension is missing, failed to load, or a CUDA call failed."""


class ApmgArgumentError(ValueError):
    """The library rejected an argument (maps to the reference's ValueError)."""


def lib():
    """Load libapmg_cuda.so once; raise loudly if it is absent (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ApmgLibraryError(
                f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build()) -- there is no CPU fallback")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().apmg_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == APMG_OK:
        return
    msg = last_error()
    if rc == APMG_E_ARG:
        raise ApmgArgumentError(msg)
    raise ApmgLibraryError(f"{what}: {msg} (code {rc})")


# ------------------------------------------------------------------ torch plumbing
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise ApmgLibraryError("a CUDA device is required (B200 / sm_100a); there is no CPU fallback")
    lib()
    return t


def device():
    return require_cuda().device("cuda", torch().cuda.current_device())


def stream_handle():
    return C.c_void_p(require_cuda().cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


_STAGE_BYTES = int(os.environ.get("APMG_STAGE_MB", "32")) << 20
_STAGE_SLOTS = int(os.environ.get("APMG_STAGE_SLOTS", "8"))
_stage = None
_stage_lock = __import__("threading").Lock()  # one transfer through the ring at a time (worker threads)


def _staging():
    """Process-level ring of pinned staging buffers (allocated once) for large uploads."""
    global _stage
    if _stage is None:
        import concurrent.futures as cf
        t = torch()
        bufs = [t.empty(_STAGE_BYTES, dtype=t.uint8, pin_memory=True) for _ in range(_STAGE_SLOTS)]
        _stage = (bufs, [None] * _STAGE_SLOTS, cf.ThreadPoolExecutor(max_workers=_STAGE_SLOTS))
    return _stage


def _ramped_chunks(n: int):
    """(offset, size) pieces of an n-byte transfer: sizes doubling from 2 MiB up to the slot size,
    so the first DMA starts after a short host copy instead of a full-slot one (the pipeline's
    start-up latency was a quarter of a 512 MiB upload)."""
    out, o, m = [], 0, min(2 << 20, _STAGE_BYTES)
    while o < n:
        k = min(m, n - o)
        out.append((o, k))
        o += k
        m = min(2 * m, _STAGE_BYTES)
    return out


def __upload_staged_locked(a: np.ndarray, out) -> None:
    """Pageable host array -> device tensor through the pinned ring: host threads fill the
    slots (numpy copies release the GIL) while the copy engine drains the filled ones, so
    the host memcpy and the PCIe / C2C transfer overlap instead of running back to back
    as the driver's own pageable path does."""
    t = torch()
    bufs, events, pool = _staging()
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(t.uint8)
    n = src.size
    chunks = _ramped_chunks(n)
    st = t.cuda.current_stream()

    def fill(slot, o, m):
        ev = events[slot]
        if ev is not None:
            ev.synchronize()
        np.copyto(bufs[slot][:m].numpy(), src[o:o + m])

    futs = [None] * _STAGE_SLOTS
    for i, (o, m) in enumerate(chunks[:_STAGE_SLOTS]):
        futs[i] = pool.submit(fill, i, o, m)
    for i, (o, m) in enumerate(chunks):
        slot = i % _STAGE_SLOTS
        futs[slot].result()
        dst[o:o + m].copy_(bufs[slot][:m], non_blocking=True)
        ev = t.cuda.Event()
        ev.record(st)
        events[slot] = ev
        j = i + _STAGE_SLOTS
        if j < len(chunks):
            futs[slot] = pool.submit(fill, slot, *chunks[j])
    st.synchronize()


def _leading_chunks(shape, itemsize, cap):
    """C-order pieces of an array of `shape` as tuples of slices, each at most `cap` bytes:
    runs of whole leading-axis slabs, or (when one slab is larger) pieces of one slab."""
    if len(shape) == 0:
        return [()]
    inner = int(np.prod(shape[1:], dtype=np.int64)) * itemsize
    if inner <= cap:
        k = max(1, cap // max(inner, 1))
        return [(slice(i, min(i + k, shape[0])),) for i in range(0, shape[0], k)]
    return [(i,) + rest for i in range(shape[0]) for rest in _leading_chunks(shape[1:], itemsize, cap)]


def _upload_view_locked(view: np.ndarray, out) -> None:
    """Any (strided, memory-mapped) float32 array view -> contiguous device tensor `out`, piece by
    piece through the pinned ring: host threads gather each C-order piece of the view (page-cache /
    disk reads of a memmap included) into a staging slot while the copy engine drains the
    previous ones -- an ingest pipeline with no intermediate full host copy."""
    t = torch()
    bufs, events, pool = _staging()
    flat = out.view(-1)
    pieces = _leading_chunks(view.shape, view.itemsize, _STAGE_BYTES)
    st = t.cuda.current_stream()
    offs, o = [], 0
    for sl in pieces:
        n = int(view[sl].size)  # a view of the view: no data is touched
        offs.append((o, n))
        o += n
    if o != flat.numel():
        raise ValueError(f"upload_view: {o} elements into a {flat.numel()}-element tensor")

    def fill(slot, i):
        ev = events[slot]
        if ev is not None:
            ev.synchronize()
        piece = view[pieces[i]]
        dst = bufs[slot][:offs[i][1] * 4].view(t.float32).numpy()
        np.copyto(dst.reshape(piece.shape), piece, casting="same_kind")

    futs = [None] * _STAGE_SLOTS
    for i in range(min(_STAGE_SLOTS, len(pieces))):
        futs[i] = pool.submit(fill, i, i)
    for i, (o, n) in enumerate(offs):
        slot = i % _STAGE_SLOTS
        futs[slot].result()
        flat[o:o + n].copy_(bufs[slot][:n * 4].view(t.float32), non_blocking=True)
        ev = t.cuda.Event()
        ev.record(st)
        events[slot] = ev
        j = i + _STAGE_SLOTS
        if j < len(pieces):
            futs[slot] = pool.submit(fill, slot, j)
    st.synchronize()


# Host arrays of PIN_MIN bytes and more (a volume) are page-locked in place on their first upload
# (cudaHostRegister) and unregistered when numpy frees them: later uploads of the same array are
# one DMA at the link rate instead of the staging ring's host copy + DMA pipeline.  APMG_PIN_HOST=0
# keeps every upload on the ring.
_PIN_MIN = 64 << 20
_pinned = {}  # data pointer -> nbytes of the ranges registered by pin_host
_pin_lock = __import__("threading").Lock()


def _owner(a: np.ndarray):
    while isinstance(a, np.ndarray) and a.base is not None:
        a = a.base
    return a


def _unpin(ptr: int) -> None:
    with _pin_lock:
        if _pinned.pop(ptr, None) is not None and _lib is not None:
            _lib.apmg_host_unregister(ptr)


def pin_host(a: np.ndarray) -> bool:
    """Page-lock the memory of a C-contiguous array that owns (a whole range of) its buffer;
    False when it cannot be (a memory map, a foreign owner, the driver refused)."""
    if not env_flag_default("APMG_PIN_HOST", True) or not a.flags.c_contiguous or a.nbytes < _PIN_MIN:
        return False
    ptr = a.ctypes.data
    with _pin_lock:
        if ptr in _pinned:
            return _pinned[ptr] >= a.nbytes
    own = _owner(a)
    if not isinstance(own, np.ndarray) or isinstance(own, np.memmap) or own.ctypes.data != ptr or own.nbytes != a.nbytes:
        return False
    if lib().apmg_host_register(ptr, a.nbytes) != 0:
        return False
    with _pin_lock:
        _pinned[ptr] = a.nbytes
    weakref.finalize(own, _unpin, ptr)
    return True


def to_device(arr: np.ndarray, dtype=None, sync: bool = True):
    """Host numpy -> contiguous CUDA tensor (plumbing only); arrays of 4 MiB and more go
    through the pinned staging ring, or -- page-locked in place (pin_host) -- as one DMA.
    sync=False returns while that DMA may still run (stream-ordered for device consumers; the
    caller keeps the host array unchanged until the stream passes the copy)."""
    t = require_cuda()
    a = np.ascontiguousarray(arr if dtype is None else np.asarray(arr, dtype=dtype))
    if a.nbytes >= (4 << 20):
        out = t.empty(a.shape, dtype=t.from_numpy(a[:0].reshape(-1)).dtype, device=device())
        if pin_host(a):
            check(lib().apmg_copy_h2d(ptr(out), a.ctypes.data, a.nbytes, stream_handle()), "copy_h2d")
            if sync or a is not arr:  # a temporary (converted) copy must outlive the DMA
                t.cuda.current_stream().synchronize()
        else:
            _upload_staged(a, out)
        return out
    return t.from_numpy(a).to(device(), non_blocking=False)


def empty(shape, np_dtype):
    t = require_cuda()
    tdt = {np.dtype(np.float32): t.float32, np.dtype(np.float64): t.float64, np.dtype(np.int64): t.int64,
           np.dtype(np.int32): t.int32, np.dtype(np.uint8): t.uint8}[np.dtype(np_dtype)]
    return t.empty(shape, dtype=tdt, device=device())


def zeros(shape, np_dtype):
    return empty(shape, np_dtype).zero_()


def workspace(nbytes: int):
    return empty((max(int(nbytes), 1),), np.uint8)


def _download_into_locked(dev, out: np.ndarray) -> None:
    """Contiguous device tensor -> existing contiguous host array of the same byte size,
    through the pinned ring: the copy engine fills slot i+1 while host threads drain slot i."""
    t = torch()
    src = dev.detach().contiguous().view(-1).view(t.uint8)
    dst = out.reshape(-1).view(np.uint8)
    n = dst.size
    if src.numel() != n:
        raise ValueError(f"download_into: {src.numel()} device bytes into a {n}-byte host array")
    bufs, events, pool = _staging()
    st = t.cuda.current_stream()
    # sizes ramping DOWN to 2 MiB at the end: the last host drain (not overlapped) stays short
    sizes = [k for _, k in _ramped_chunks(n)][::-1]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64) if sizes else []
    chunks = [(int(o), int(k)) for o, k in zip(offs, sizes)]
    futs = [None] * _STAGE_SLOTS

    def drain(slot, ev, o, m):
        ev.synchronize()
        np.copyto(dst[o:o + m], bufs[slot][:m].numpy())

    for i, (o, m) in enumerate(chunks):
        slot = i % _STAGE_SLOTS
        if futs[slot] is not None:
            futs[slot].result()
        bufs[slot][:m].copy_(src[o:o + m], non_blocking=True)
        ev = t.cuda.Event()
        ev.record(st)
        events[slot] = ev
        futs[slot] = pool.submit(drain, slot, ev, o, m)
    for f in futs:
        if f is not None:
            f.result()


def to_host(t) -> np.ndarray:
    if t.numel() * t.element_size() >= (4 << 20):
        out = np.empty(tuple(t.shape), dtype=torch_to_np(t.dtype))
        download_into(t, out)
        return out
    return t.detach().cpu().numpy()


def torch_to_np(dt):
    t = torch()
    return {t.float32: np.float32, t.float64: np.float64, t.int64: np.int64, t.int32: np.int32,
            t.uint8: np.uint8}[dt]


def dtype_code(np_dtype) -> int:
    dt = np.dtype(np_dtype)
    if dt == np.float32:
        return APMG_F32
    if dt == np.float64:
        return APMG_F64
    raise TypeError(f"unsupported model dtype {dt} (float32 or float64)")


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0", "false", "False")


def env_flag_default(name: str, default: bool) -> bool:
    v = os.environ.get(name)
    return default if v is None or v == "" else v not in ("0", "false", "False")


def _upload_staged(*args, **kw):
    with _stage_lock:
        return __upload_staged_locked(*args, **kw)


def download_into(*args, **kw):
    with _stage_lock:
        return _download_into_locked(*args, **kw)


def upload_view(*args, **kw):
    with _stage_lock:
        return _upload_view_locked(*args, **kw)


DEBUG_LIB_PATH = Path(__file__).resolve().parents[1] / "tools" / "libapmg_debug.so"
DEBUG_SIGNATURES = {
    "apmg_debug_umma_gemm": (C.c_int, [_I32, _I32, _I32, _I32, _P, _P, _P, _P]),
    "apmg_debug_umma_bf16": (C.c_int, [_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P]),
    "apmg_peak_probe": (C.c_int, [_I32, _P, _I64, _I32, _P, _P]),
    "apmg_last_error": (C.c_char_p, []),
}
_debug = None


def debug_lib():
    """tools/libapmg_debug.so: tcgen05 self-tests and roofline probes (tests / tools only)."""
    global _debug
    if _debug is None:
        if not DEBUG_LIB_PATH.exists():
            raise ApmgLibraryError(f"{DEBUG_LIB_PATH} is not built; run `make`")
        handle = C.CDLL(str(DEBUG_LIB_PATH))
        for name, (res, args) in DEBUG_SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _debug = handle
    return _debug
