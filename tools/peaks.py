"""Measure the roofline peaks SURVEY 8(d) lists as missing (L2 float2 gather, L2 float2 RED,
FP32, FP64, tcgen05 kind::tf32, warp shuffles) with csrc/peaks.cu and write
profiles/peaks_b200.json.  Each probe: 2 warm-up launches, then best of 5 timed with CUDA
events on the launching stream."""
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch

from paper_2308_02494_b200 import _lib as L


def probe(kind, table, nbytes, iters):
    work = C.c_double()
    st = L.stream_handle()
    for _ in range(2):
        L.check(L.debug_lib().apmg_peak_probe(kind, L.ptr(table), nbytes, iters, C.byref(work), st), "probe")
    best = float("inf")
    s = torch.cuda.current_stream()
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        L.check(L.debug_lib().apmg_peak_probe(kind, L.ptr(table), nbytes, iters, C.byref(work), st), "probe")
        e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return work.value / best, best


def main():
    out = {"gpu": torch.cuda.get_device_name(), "sms": torch.cuda.get_device_properties(0).multi_processor_count}
    for mib in (16, 64):
        t = torch.zeros((mib << 20) // 4, dtype=torch.float32, device="cuda")
        g, dt = probe(0, t, mib << 20, 256)
        out[f"l2_gather_float2_GBps_{mib}MiB"] = g / 1e9
        g4, dt = probe(7, t, mib << 20, 256)
        out[f"l2_gather_float4_GBps_{mib}MiB"] = g4 / 1e9
        g8, dt = probe(10, t, mib << 20, 256)
        out[f"l2_gather_32B_GBps_{mib}MiB"] = g8 / 1e9
        r, dt = probe(1, t, mib << 20, 64)
        out[f"l2_red_float2_Gops_{mib}MiB"] = r / 1e9
        r4, dt = probe(8, t, mib << 20, 64)
        out[f"l2_red_float4_Gops_{mib}MiB"] = r4 / 1e9
    big = torch.zeros((1 << 30) // 4, dtype=torch.float32, device="cuda")
    g, _ = probe(0, big, 1 << 30, 64)
    out["hbm_gather_float2_GBps_1GiB"] = g / 1e9
    del big
    sink = torch.zeros(16, dtype=torch.float32, device="cuda")
    out["fp32_tflops"] = probe(2, sink, 64, 4096)[0] / 1e12
    out["fp64_tflops"] = probe(3, sink, 64, 1024)[0] / 1e12
    out["tf32_tcgen05_tflops"] = probe(4, sink, 64, 4096)[0] / 1e12
    # per-instruction cost of tcgen05.mma kind::f16 K=16 by shape (the MLP kernels issue small N)
    for nb in (64, 128, 192, 256, 1064, 1128, 1256, 1):
        f, dt = probe(9, sink, nb, 4096)
        name = "bf16_m128n64k16_4acc" if nb == 1 else f"bf16_m{64 if nb >= 1000 else 128}n{nb % 1000}k16"
        out[f"{name}_tflops"] = f / 1e12
        out[f"{name}_cycles_per_mma"] = dt * 1.965e9 / 4096
    out["shfl_Ginstr_per_s"] = probe(5, sink, 64, 4096)[0] / 1e9
    out["shfl_per_clk_per_sm"] = out["shfl_Ginstr_per_s"] * 1e9 / (out["sms"] * 1.965e9)
    out["atoms_f32_Ginstr_per_s"] = probe(6, sink, 64, 1024)[0] / 1e9
    out["atoms_per_clk_per_sm"] = out["atoms_f32_Ginstr_per_s"] * 1e9 / (out["sms"] * 1.965e9)
    out["how"] = ("csrc/peaks.cu via tools/peaks.py: best of 5 launches, CUDA events; gather/RED = random float2 / float4 / "
                  "32-byte (ld.global.nc.v8.f32) elements over a power-of-two table (16/64 MiB stay in the 126 MB L2), 8 independent accesses in flight "
                  "per thread, 148x8 CTAs of 256; FP32/FP64 = 8 independent FMA chains per thread; tf32 = "
                  "back-to-back tcgen05.mma M=128 N=256 K=8 from one thread per SM; shfl = 4 independent "
                  "__shfl_sync chains per thread (warp instructions/s)")
    print(json.dumps(out, indent=1))
    (ROOT / "profiles" / "peaks_b200.json").write_text(json.dumps(out, indent=1))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)  # the copy gpurun merges back
    (ROOT / "gpurun_out" / "peaks_b200.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
