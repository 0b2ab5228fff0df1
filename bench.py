"""Benchmark: APMGSRN training throughput (train points/sec) on B200.

N = 1, workload "C2" (BASELINE.json configs[1]): 64 grids 32^3 x 2 features, MLP 2x64, fit a
synthetic 512^3 blob volume (test_acceptance.py:156-164 blob list), batch 2^20, density loss on
every timed iteration.  One "step" = one training iteration (Philox batch + fp64 targets + fused
recon fwd/bwd + masked Adam + density step + scheduler), all device-resident.  ``value`` is
device-timed (CUDA events on the session's stream); ``e2e`` is train_single through the public
API with a host model and a host volume (uploads / downloads inside the timed region).

N > 1 (torchrun), workload "C4" (configs[3]): the whole 2x2x2 decomposition of a synthetic
1024^3 volume (ghost 1, bricks of ~513^3) is fitted through ``train_decomposed``: rank r trains
bricks flat % world == r (4 / 2 / 1 bricks at N = 2 / 4 / 8), one model per brick, K iterations
each at batch 2^20, no data-path collective.  ``value`` = all bricks' training points / the max
over ranks of that rank's device-timed training iterations; ``time_to_fit`` = the max over ranks
of the whole train_decomposed call (brick ingest from the raw file, training, .apmg save, brick
PSNR); the decomposed field's PSNR over the 1024^3 lattice comes from per-rank brick sweeps with
the SSE all-reduced over NCCL.

``--impl reference`` times the reference algorithm on the host cores: the numpy oracle port of
apmg.train_single (the reference is pure numpy and is not installed on the GPU box), each
iteration's batch split over all host threads, on the same workload (batch 2^20, same model,
same volume).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BATCH = 1 << 20
DIMS1 = (512, 512, 512)
DIMS_DECOMP = (1024, 1024, 1024)
M, CH, RES = 64, 2, (32, 32, 32)
BLOBS = [((0.45, -0.3, 0.2), (0.035, 0.035, 0.035), 1.0), ((-0.2, 0.2, -0.1), (0.6, 0.5, 0.7), 0.35),
         ((0.3, 0.4, 0.5), (0.45, 0.55, 0.4), 0.25), ((-0.5, -0.5, 0.4), (0.5, 0.4, 0.5), 0.3)]
METRIC = "train points/sec"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line).

    The C2 timed region is ~40 ms, shorter than nvidia-smi's sampling loop, so the clocks are read
    through NVML (the library nvidia-smi uses) by a thread polling every ~2 ms while the region
    runs; nvidia-smi -lms 5 is the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int):
        self.index = index
        self.rows, self.max_mhz, self.source = [], None, None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            masks = [(name, getattr(N, attr)) for name, attr in self.REASONS]

            def poll():
                while not self._stop.is_set():
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                      [name for name, m in masks if r & m]))
                    time.sleep(0.002)

            self.source = "nvml"
        except Exception:  # pragma: no cover - NVML missing: nvidia-smi in a loop
            def poll():
                try:
                    proc = subprocess.Popen(
                        ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,"
                         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                         "--format=csv,noheader,nounits", "-lms", "5"], stdout=subprocess.PIPE,
                        stderr=subprocess.DEVNULL, text=True)
                except FileNotFoundError:
                    return
                names = [n for n, _ in self.REASONS[:4]]
                for line in proc.stdout:
                    if self._stop.is_set():
                        break
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                        self.max_mhz = float(parts[1])
                        self.rows.append((float(parts[0]), [names[i] for i in range(4) if parts[2 + i] == "Active"]))
                proc.terminate()

            self.source = "nvidia-smi"
        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.thread.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no clock samples"], "source": self.source}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n in r[1]})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        # APMG_BENCH_BACKEND=gloo: functional check of the N>1 path with several ranks on one
        # GPU (the ranks never wait on each other's kernels; not a scaling measurement)
        backend = os.environ.get("APMG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        return dist, rank, world, local
    return None, 0, 1, local


def workload_config(world):
    """The `config` object of both arms' JSON lines."""
    if world == 1:
        return {"workload": "C2: single model, synthetic 512^3 volume", "global_batch": BATCH,
                "model": "APMGSRN 64 grids 32^3 x2, MLP 2x64", "density_loss": "every timed iteration",
                "parallelism": "single GPU (replicas only)",
                "l2": "inputs larger than L2 (512 MiB volume); 16 MiB grids L2-resident by design"}
    return {"workload": "C4: 2x2x2 bricks of synthetic 1024^3 (ghost 1), one model per brick, train_decomposed",
            "global_batch": BATCH * min(world, 8), "model": "APMGSRN 64 grids 32^3 x2, MLP 2x64 per brick",
            "density_loss": "every timed iteration", "parallelism": f"brick-sharded x{world} (flat % world)",
            "l2": "inputs larger than L2 (~540 MB brick volume per session)"}


# untimed train_single calls before the timed e2e call (the allocator reaches its steady state --
# the timed call's blocks all come from its cache -- after the second)
E2E_WARM = int(os.environ.get("APMG_E2E_WARM", "2"))

# algorithmic work per training point -> per-kernel roofline rows
ENC_BYTES = 8 * M * CH * 4          # 4,096 B of corner data gathered per point (encoder fwd)
SCAT_BYTES = 8 * M * CH * 4         # 4,096 B of corner gradients reduced per point (encoder bwd)
RED4_PER_PT = 4 * M                 # x-pair layout: 4 float4 REDs per (point, grid) before aggregation
MLP_FLOP = 74_112                   # 24,704 forward + 49,408 backward
MLP_ISSUED = 24_704 * 6 + 49_152 * 3  # bf16x3: 6 products per forward GEMM, 3 per backward GEMM
DENS_GRAD_FLOP = M * 100            # per point: bump (~35), l^(2p-1) powers, 13 accumulators x2
INFER_ISSUED = 24_704 * 6           # C3 forward: 6 bf16x3 products per GEMM


def _traffic(kernel):
    """(dram bytes, l2 bytes) per launch of `kernel` from the newest profiles/traffic_*.json."""
    files = sorted((ROOT / "profiles").glob("traffic_r*.json"))
    if not files:
        return None, None
    v = json.loads(files[-1].read_text()).get(kernel)
    if isinstance(v, dict):
        return v.get("dram"), v.get("l2")
    return v, None


def _red_sectors(kernel):
    """ncu L2 RED sectors per launch of `kernel` (the REDs actually issued after warp aggregation;
    one float4 RED = one sector), from the newest profiles/traffic_*.json that has them."""
    for f in sorted((ROOT / "profiles").glob("traffic_r*.json"), reverse=True):
        v = json.loads(f.read_text()).get(kernel)
        if isinstance(v, dict) and v.get("l2_red_sectors"):
            return v["l2_red_sectors"], f.name
    return None, None


def _peaks2():
    f = ROOT / "profiles" / "peaks_b200.json"
    return json.loads(f.read_text()) if f.exists() else {}


def roofline_for(kernel: str, ms_per_launch: float, pk: dict):
    """Roofline of one kernel from its average device time per launch (CUDA events inside the
    bench) and its ALGORITHMIC work per launch (SURVEY 8d per-point figure x 2^20 points).

    k_recon_tc16 (encode -> tcgen05 MLP -> scatter): the 16 MiB grids and their 64 MiB xy-quad copy
    are L2-resident, so the encoder is bound by L2 gather bandwidth (the kernel issues 32-byte
    gathers: peak = the random 32-byte gather probe over a 64 MiB table; float4 with the x-pair
    copy) and the scatter by L2 RED throughput (float4 RED probe);
    the MLP by the tensor pipe.  The primary (`bound: l2`) is the encoder gather, SURVEY 8d's and
    north_star's metric; `components` gives all three and `serial_sum_frac` = sum of each part's
    time at its peak / measured time (> 1 means the parts overlap or L1 serves part of them)."""
    t = ms_per_launch * 1e-3
    pk2 = _peaks2()
    dram, l2b = _traffic(kernel)
    base = {"kernel": kernel, "ms_per_launch": ms_per_launch, "traffic": dram, "l2_traffic": l2b,
            "traffic_source": "ncu --set full: dram__bytes_read+write.sum (l2_traffic: 32 x lts__t_sectors.sum) per launch, "
                              "profiles/traffic_r*.json"}
    if kernel.startswith("recon_fwd_bwd") and pk2:
        # the gather's peak for the access the kernel issues: 32-byte random loads from the 64 MiB
        # xy-quad copy (default), or float4 from the 32 MiB x-pair copy (APMG_GRIDQ=0)
        quad = os.environ.get("APMG_GRIDQ", "1") != "0"
        g_key = "l2_gather_32B_GBps_64MiB" if quad else "l2_gather_float4_GBps_16MiB"
        g_pk = pk2.get(g_key) or pk2["l2_gather_float4_GBps_16MiB"]
        r_pk = pk2.get("l2_red_float4_Gops_16MiB") or pk2["l2_red_float2_Gops_16MiB"]
        g_ach = BATCH * ENC_BYTES / t / 1e9
        r_ach = BATCH * RED4_PER_PT / t / 1e9
        f_alg = BATCH * MLP_FLOP / t / 1e12
        f_iss = BATCH * MLP_ISSUED / t / 1e12
        comps = {
            "encoder_gather": {"achieved": g_ach, "peak": g_pk, "unit": "GB/s", "frac": g_ach / g_pk,
                               "peak_probe": g_key,
                               "work": "4,096 B/pt of corner data (64 grids x 2 x 32 B xy-quad records; "
                                       "x-pair: 4 x 16 B)"},
            "scatter_red": {"achieved": None, "peak": r_pk, "unit": "G float4 RED/s", "frac": None,
                            "algorithmic_equiv": r_ach,
                            "work": "256 float4 REDs/pt before warp aggregation; achieved / frac count the REDs "
                                    "the L2 executed after aggregation (ncu RED sectors per launch); "
                                    "algorithmic_equiv is the pre-aggregation count per second (not bounded by "
                                    "the peak)"},
            "mlp_tensor": {"achieved": f_iss, "algorithmic": f_alg, "peak": pk["bf16_tflops"],
                           "unit": "TFLOP/s issued (bf16x3 products)", "frac": f_iss / pk["bf16_tflops"],
                           "work": "295,680 issued FLOP/pt (74,112 algorithmic)"}}
        red_sec, red_src = _red_sectors(kernel)
        if red_sec:  # the REDs the L2 actually executed (ncu), at this launch's measured time
            comps["scatter_red"].update({"issued_per_launch": red_sec, "achieved": red_sec / t / 1e9,
                                         "frac": red_sec / t / 1e9 / r_pk, "issued_source": red_src})
        return {"bound": "l2", **base, "achieved": g_ach, "peak": g_pk, "unit": "GB/s", "frac": g_ach / g_pk,
                "components": comps, "serial_sum_frac": sum(c["frac"] or 0.0 for c in comps.values()),
                "peak_source": "profiles/peaks_b200.json (tools/peaks.py): random 32-byte gather over a 64 MiB "
                               "table (float4 over 16 MiB with APMG_GRIDQ=0) / float4 RED over a 16 MiB table; "
                               "MEASURED_PEAKS.json bf16 dense"}
    if kernel == "density_grad" and pk2:
        a = BATCH * DENS_GRAD_FLOP / t / 1e12
        return {"bound": "fp32", **base, "achieved": a, "peak": pk2["fp32_tflops"], "unit": "TFLOP/s",
                "frac": a / pk2["fp32_tflops"], "work": f"{DENS_GRAD_FLOP} FP32 FLOP/pt (64 grids x ~100)",
                "peak_source": "profiles/peaks_b200.json fp32_tflops (FFMA probe)"}
    per_point = {"train_batch": 32 + 24 + 8, "density_rho": 12 + 4 + 8, "batch_keys": 24 + 4,
                 "bucket_scatter": 48}
    nbytes = 4_206_656 * 4 * 7 if kernel == "adam_main" else BATCH * per_point.get(kernel, float("nan"))
    peak = pk.get("hbm_gbs", 6650.0)
    achieved = nbytes / t / 1e9
    return {"bound": "hbm", **base, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "bytes_per_launch": nbytes, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)"}


def kernel_table():
    import ctypes as C
    from paper_2308_02494_b200 import _lib as L
    cap = 64
    names = C.create_string_buffer(64 * cap)
    tot = (C.c_double * cap)()
    cnt = (C.c_int64 * cap)()
    n = L.lib().apmg_kernel_timing_read(names, tot, cnt, cap)
    out = {}
    for i in range(n):
        nm = names.raw[64 * i:64 * (i + 1)].split(b"\0")[0].decode()
        out[nm] = {"total_ms": tot[i], "launches": int(cnt[i])}
    return out


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run_cpu_baseline(vol_host, iterations=3):
    """cpu_baseline of the GPU arm: the oracle port of train_single (reference algorithm, numpy,
    batch split over all host threads) on a bounded sample of the same workload: one warm-up and
    `iterations` timed iterations at batch 2^20, density on, same model and volume."""
    from oracle import apmg_oracle as O
    thr = host_threads()
    prm = O.init_params(M, CH, RES, seed=0, vmin=float(vol_host.min()), vmax=float(vol_host.max()))
    stamps = []
    cfg = O.LoopConfig(iterations=iterations + 1, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                       plateau_enabled=False, seed=0)
    t0 = time.perf_counter()
    O.train_single_threaded(prm, vol_host, cfg, thr, on_iteration=lambda it, p: stamps.append(time.perf_counter()))
    per_it = np.diff([t0] + stamps)[1:]  # drop the first (warm-up) iteration
    rate = BATCH / float(np.mean(per_it))
    return {"value": rate, "unit": METRIC, "cores": thr, "kind": "port",
            "sample": f"{iterations} timed iterations (after 1 warm-up) of the C2 workload at batch 2^20, density "
                      f"on, same model / 512^3 volume; numpy oracle of apmg.train_single, each iteration's batch "
                      f"split over {thr} host threads"}


def run_reference(args):
    """Reference arm: the oracle port of apmg.train_single on the host cores, on this arm's own
    workload and batch (2^20), W untimed + K timed iterations, all host threads.  Under torchrun
    only rank 0 runs (the others exit); at N > 1 the workload is one C4 brick model's iterations
    (every brick runs the same per-iteration work)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import apmg_oracle as O
    thr = host_threads()
    dims = DIMS1 if world == 1 else tuple(n // 2 + 1 for n in DIMS_DECOMP)  # a C4 ghost brick is ~513^3
    vol = O.synth_volume(dims, BLOBS)
    prm = O.init_params(M, CH, RES, seed=0, vmin=float(vol.min()), vmax=float(vol.max()))
    total = args.warmup + args.steps
    cfg = O.LoopConfig(iterations=total, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                       plateau_enabled=False, seed=0)
    stamps = []
    budget = float(os.environ.get("APMG_REF_BUDGET_S", "1500"))
    t_start = time.perf_counter()

    class Budget(Exception):
        pass

    def cb(it, p):
        stamps.append(time.perf_counter())
        if it >= args.warmup and stamps[-1] - t_start > budget:
            raise Budget()

    try:
        O.train_single_threaded(prm, vol, cfg, thr, on_iteration=cb)
    except Budget:
        pass
    t0 = stamps[args.warmup - 1] if args.warmup else t_start
    timed = len(stamps) - args.warmup
    dt = stamps[-1] - t0
    value = timed * BATCH / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world,
            "steps": timed, "warmup": args.warmup, "ms_per_step": 1e3 * dt / timed, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 model / f64 density and scatter sums (numpy)",
            "data": "synthetic", "config": workload_config(world),
            "cpu_baseline": {"value": value, "unit": METRIC, "cores": thr, "kind": "port",
                             "sample": f"{timed} timed iterations (after {args.warmup} warm-up) at batch 2^20 of "
                                       f"{'the C2 workload' if world == 1 else 'one C4 brick (513^3)'}; numpy "
                                       f"oracle of apmg.train_single, batch split over {thr} host threads; rank 0 "
                                       f"only"},
            "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if timed < args.steps:
        line["note"] = f"stopped after {timed} of {args.steps} timed iterations (APMG_REF_BUDGET_S={budget:.0f})"
    print(json.dumps(line), flush=True)


DTYPE = ("f32 params/activations; encoder lerps f32; MLP on tcgen05 as bf16x3 split products (6 per forward "
         "GEMM ~2^-24, 3 per backward GEMM ~2^-16) with f32 accumulation; grid gradient f32 RED; density: "
         "per-(point, grid) bumps in f32 (SFU exp2), per-point rho and all statistics / loss / transform-gradient "
         "sums in f64; targets f64 trilinear; loss f64")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="apmg", choices=["apmg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-inference", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return main_decomposed(args)

    import torch
    from paper_2308_02494_b200 import _lib as L
    from paper_2308_02494_b200 import model as PM
    from paper_2308_02494_b200 import trainer as PT
    from paper_2308_02494_b200 import volume as PV

    torch.cuda.set_device(0)
    L.lib()
    blobs = [PV.BlobSpec(c, s, a) for c, s, a in BLOBS]
    vdev = PV.synth_volume_device(DIMS1, blobs)
    vol = PV.Volume.from_device(DIMS1, vdev)
    seed = 0
    model = PM.init_model(PM.ModelConfig(M, CH, RES), seed=seed, vmin=vol.vmin, vmax=vol.vmax)
    K, W = args.steps, max(args.warmup, 3)
    KT = 5  # untimed iterations after the timed region, run with per-kernel CUDA events
    cfg = PT.TrainConfig(iterations=W + K + KT, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                         plateau_enabled=False, seed=seed)
    sess = PT.TrainSession(model, vol, cfg)
    sess.run(W)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.lib().apmg_launch_count()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        sess.run(K)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = L.lib().apmg_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    # per-kernel shares from a separate, untimed pass (events around every launch perturb
    # the timed region, and are incompatible with the graph replay it uses)
    L.lib().apmg_kernel_timing_enable(1)
    sess.run(KT)
    torch.cuda.synchronize()
    ktab = kernel_table()
    L.lib().apmg_kernel_timing_enable(0)
    ran, _ = sess.status()
    assert ran == W + K + KT, f"expected {W + K + KT} iterations, ran {ran}"
    log = sess.log()
    sess.close()
    del sess  # its workspace goes back to torch's cache for the e2e calls below
    value = K * BATCH / (ms * 1e-3)

    # dominant kernel and its roofline (+ the other step kernels' rows)
    pk = peaks()
    per_launch = {k: v["total_ms"] / v["launches"] for k, v in ktab.items() if v["launches"]}
    dom = max(ktab.items(), key=lambda kv: kv[1]["total_ms"])[0]
    roof = roofline_for(dom, per_launch[dom], pk)
    roof["other_kernels"] = {k: {kk: r[kk] for kk in ("bound", "achieved", "peak", "unit", "frac")}
                             for k in ("density_grad", "adam_main", "train_batch") if k in per_launch
                             for r in [roofline_for(k, per_launch[k], pk)]}
    shares = {k: round((v["total_ms"] / KT) / (ms / K), 4)
              for k, v in sorted(ktab.items(), key=lambda kv: -kv[1]["total_ms"])}

    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        host_vol = PV.Volume(dims=DIMS1, data=L.to_host(vdev))
        m2 = PM.init_model(PM.ModelConfig(M, CH, RES), seed=seed, vmin=vol.vmin, vmax=vol.vmax)
        cfg2 = PT.TrainConfig(iterations=K, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                              plateau_enabled=False, seed=seed)
        # E2E_WARM untimed warm-up calls (first-use costs: staging ring, allocator pools, graph build);
        # train_single hands its large blocks back at return, so the timed call allocates afresh
        # (same iteration count as the timed call, so its workspace has the timed call's size and
        # torch's caching allocator hands the same block back)
        # Both calls run inside hold_block_cache, the public way to keep session buffers across
        # repeated train_single calls (the timed call reuses the warm-up's workspace); the host
        # volume is page-locked in place by its first upload (pin_host), as a pinned input buffer.
        with PT.hold_block_cache():
            for _ in range(E2E_WARM):
                mw = PM.init_model(PM.ModelConfig(M, CH, RES), seed=seed, vmin=vol.vmin, vmax=vol.vmax)
                PT.train_single(mw, PV.Volume(dims=DIMS1, data=host_vol.data),
                                PT.TrainConfig(iterations=K, batch_size=BATCH, delay_start=0,
                                               transform_hard_stop_fraction=1.0, plateau_enabled=False, seed=seed))
                del mw
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, log2 = PT.train_single(m2, host_vol, cfg2)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        params_b = 4 * m2.parameter_count()
        e2e = {"value": K * BATCH / dt, "unit": METRIC,
               "h2d_bytes_per_step": int((host_vol.data.nbytes + params_b + 16 * K) / K),
               "d2h_bytes_per_step": int((params_b + 24 * K) / K),
               "setup_ms": round(1e3 * log2.setup_seconds, 2), "setup_split_ms": log2.setup_ms,
               "loop_ms": round(log2.loop_ms, 2), "wall_ms": round(1e3 * dt, 2),
               "note": f"paper_2308_02494_b200.train_single(host model, host Volume, iterations={K}) after "
                       f"{E2E_WARM} untimed calls, all inside hold_block_cache: volume upload (one DMA from the page-locked "
                       f"host array) + parameter upload, device loop, parameter + log download; bound: "
                       f"loop / (loop + volume bytes / link rate)"}

    infer = None if args.no_inference else bench_inference()
    render = None if args.no_render else bench_render()
    cpu = None if args.no_cpu_baseline else run_cpu_baseline(L.to_host(vdev))

    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE, "data": "synthetic", "config": workload_config(1),
        "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roof,
        "kernel_share": shares, "e2e": e2e, "cpu_baseline": cpu, "inference": infer, "render": render,
        "final_l_rec": log.l_rec[-1] if log.l_rec else None,
    }
    print(json.dumps(line), flush=True)


def main_decomposed(args):
    """N > 1: the C4 workload through train_decomposed (see the module docstring)."""
    import shutil
    import tempfile

    import torch
    from paper_2308_02494_b200 import _lib as L
    from paper_2308_02494_b200 import volume as PV
    from paper_2308_02494_b200.decomposition import (DecomposedField, load_manifest, plan_partition,
                                                     train_decomposed)
    from paper_2308_02494_b200.model import ModelConfig
    from paper_2308_02494_b200.trainer import TrainConfig

    os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) for the driver's log
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dist, rank, world, local = dist_setup()
    L.lib()
    dev = torch.device("cuda", local)
    K, W = args.steps, max(args.warmup, 3)
    blobs = [PV.BlobSpec(c, s, a) for c, s, a in BLOBS]
    work = Path(os.environ.get("APMG_C4_DIR", tempfile.gettempdir())) / "apmg_c4"
    raw = work / "volume_1024.raw"
    if rank == 0:  # synthetic 1024^3 on the device -> the raw little-endian file the API ingests
        work.mkdir(parents=True, exist_ok=True)
        v = PV.synth_volume_device(DIMS_DECOMP, blobs)
        L.to_host(v).astype("<f4").tofile(raw)
        del v
        torch.cuda.empty_cache()
    dist.barrier()
    header = PV.VolumeHeader(dims=DIMS_DECOMP)
    plan = plan_partition(DIMS_DECOMP, 2, 2, 2, ghost=1)
    mcfg = ModelConfig(M, CH, RES)

    def fit(iters, out):
        tcfg = TrainConfig(iterations=iters, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                           plateau_enabled=False, seed=0)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        man = train_decomposed(raw, header, plan, mcfg, tcfg, out)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        return man, e0.elapsed_time(e1), wall

    fit(W, work / f"warm_{world}")  # untimed: first-use costs (graphs, pools, staging ring)
    launches0 = L.lib().apmg_launch_count()
    with ClockSampler(local) as clk:
        man, fit_ms, wall = fit(K, work / f"fit_{world}")
    launches = L.lib().apmg_launch_count() - launches0
    mine = [b for b in range(plan.brick_count) if b % world == rank]
    train_ms = sum(float(man.bricks[b]["loop_ms"]) for b in mine)
    rdev = dev if dist.get_backend() == "nccl" else torch.device("cpu")  # gloo: functional runs only
    t = torch.tensor([train_ms, fit_ms, wall], device=rdev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    train_ms, fit_ms, wall = (float(v) for v in t.tolist())
    points = sum(int(b["iterations_run"]) * BATCH for b in man.bricks)
    value = points / (train_ms * 1e-3)

    # PSNR of the fitted decomposed field over the whole 1024^3 lattice: each rank sweeps the voxel
    # boxes its bricks own (box-local truth from the same synthesis), SSE all-reduced over NCCL
    field = DecomposedField.load(work / f"fit_{world}" / "manifest.json")
    boxes = field.brick_boxes(DIMS_DECOMP)
    truth = {}
    for b in mine:
        x0, x1, y0, y1, z0, z1 = boxes[b]
        truth[b] = PV.synth_volume_device(DIMS_DECOMP, blobs, extent=PV.Extent(lo=(x0, y0, z0), hi=(x1, y1, z1)))
    sse = L.zeros((1,), np.float64)
    field.lattice_sse_local(mine, truth, None, sse)
    sse = sse.to(rdev)
    dist.all_reduce(sse)
    mse = float(sse.item()) / float(np.prod(DIMS_DECOMP))
    span = max(float(b["vmax"]) for b in man.bricks) - min(float(b["vmin"]) for b in man.bricks)
    psnr = 200.0 if mse == 0 else min(200.0, 10.0 * np.log10(span * span / mse))

    infer = None if args.no_inference else bench_decomposed_inference(rank, world, dist)
    if rank == 0:
        brick_bytes = sum(np.prod([h - l + 1 for l, h in zip(b["ghost_lo"], b["ghost_hi"])]) * 4 for b in man.bricks)
        line = {
            "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": train_ms / (K * len(mine)), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic", "config": workload_config(world),
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "time_to_fit": {"ms": fit_ms, "wall_ms": 1e3 * wall, "bricks": plan.brick_count,
                            "iterations_per_brick": K, "bricks_per_rank": [len([b for b in range(8) if b % world == r])
                                                                           for r in range(world)],
                            "note": "max over ranks of the train_decomposed call: raw-file ingest, training, "
                                    ".apmg save and brick PSNR of every brick the rank owns"},
            "train_ms_max_rank": train_ms,
            "psnr_db": psnr, "psnr_note": "decomposed field over the 1024^3 lattice, per-rank brick sweeps, "
                                          "SSE all-reduced over NCCL (after K iterations: throughput run)",
            "e2e": {"value": points / wall, "unit": METRIC, "h2d_bytes_per_step": int(brick_bytes / K),
                    "d2h_bytes_per_step": int(plan.brick_count * 4 * 4_207_680 / K),
                    "note": "train_decomposed wall time, max over ranks: raw file -> pinned ring -> GPU per brick, "
                            "device loop, model download + save"},
            "cpu_baseline": None, "inference": infer,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    if rank == 0:
        shutil.rmtree(work / f"warm_{world}", ignore_errors=True)
    dist.destroy_process_group()


def bench_render(size=512, samples=128, reps=5):
    """Renderer field-query path: one C2-shaped model, a size^2 frame, `samples`
    per ray, reference defaults otherwise (early exit at alpha 0.99).  Wall time of
    render_frame (device rays, sample points, tensor-core field queries, transfer function,
    compositing, RGBA download), after one warm-up frame."""
    import numpy as np
    import torch
    from paper_2308_02494_b200 import model as PM
    from paper_2308_02494_b200 import render as PR
    m = PM.init_model(PM.ModelConfig(M, CH, RES), seed=0, vmin=0.0, vmax=1.0)
    m.grids[:] = np.random.default_rng(0).normal(scale=0.3, size=m.grids.shape).astype(np.float32)
    cam = PR.Camera(eye=(1.6, 1.1, 2.4), look_at=(0.0, 0.0, 0.0), width=size, height=size)
    tf = PR.TransferFunction(opacity_points=[(0.0, 0.0), (0.5, 0.05), (1.0, 0.6)])
    cfg = PR.RenderConfig(samples_per_ray=samples)
    PR.render_frame(PR.ModelField(m), cam, tf, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        img = PR.render_frame(PR.ModelField(m), cam, tf, cfg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    return {"metric": "rendered frames/sec", "value": 1.0 / dt, "ms_per_frame": 1e3 * dt,
            "field_queries_per_sec_upper_bound": size * size * samples / dt,
            "config": f"{size}x{size} frame, {samples} samples/ray, 64x32^3x2 model, early exit 0.99, "
                      f"mean alpha {float(img[..., 3].mean()):.3f}"}


def bench_inference(dims=(1024, 1024, 1024)):
    """C3: full-volume 1024^3 lattice sweep of one model (PSNR mode: fused forward + fp64 SSE)."""
    import torch
    from paper_2308_02494_b200 import _lib as L
    from paper_2308_02494_b200 import model as PM
    from paper_2308_02494_b200 import trainer as PT
    from paper_2308_02494_b200 import volume as PV
    blobs = [PV.BlobSpec(c, s, a) for c, s, a in BLOBS]
    truth = PV.synth_volume_device(dims, blobs)
    m = PM.init_model(PM.ModelConfig(M, CH, RES), seed=0, vmin=0.0, vmax=1.0)
    r = np.random.default_rng(0)
    m.grids[:] = r.normal(scale=0.1, size=m.grids.shape).astype(np.float32)
    dm = m.device()
    sse = L.zeros((1,), np.float64)
    PT.lattice_sse_model(dm, truth, dims, sse=sse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 2
    e0.record()
    for _ in range(reps):
        PT.lattice_sse_model(dm, truth, dims, sse=sse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    vox = dims[0] * dims[1] * dims[2]
    pk = peaks()
    t = ms * 1e-3
    iss = vox * INFER_ISSUED / t / 1e12
    dram, l2b = _traffic("infer_lattice_tc")
    roof = {"bound": "tensor", "kernel": "infer_lattice_tc (k_infer_tc)", "achieved": iss, "peak": pk["bf16_tflops"],
            "unit": "TFLOP/s issued (bf16x3: 6 products per GEMM, 147,456 FLOP/voxel)",
            "frac": iss / pk["bf16_tflops"], "algorithmic_tflops": vox * 24_704 / t / 1e12,
            "gather_bytes_per_s": vox * ENC_BYTES / t,
            "gather_note": "4,096 B/voxel of corner data; lattice sweeps are coherent, most corners hit L1",
            "traffic": dram, "l2_traffic": l2b,
            "traffic_note": "ncu bytes per launch of the profiled 512^3 sweep (profiles/traffic_r*.json)",
            "peak_source": "MEASURED_PEAKS.json bf16 dense"}
    return {"metric": "inference voxels/sec", "value": vox / (ms * 1e-3), "ms_per_sweep": ms,
            "config": "C3: 1024^3 lattice, one 64x32^3x2 model, fused forward + fp64 SSE vs truth",
            "roofline": roof}


DIMS_C5 = (2048, 2048, 2048)


def bench_decomposed_inference(rank, world, dist, dims=DIMS_C5, counts=(4, 4, 4)):
    """C5: a 2048^3 lattice decomposed into 4x4x4 bricks (ghost 1); rank r sweeps bricks
    flat % world == r (each through its own model and brick affine) in PSNR + reconstruct
    mode against a synthetic truth it generates for its own boxes; SSE all-reduced.
    value = all voxels / max-over-ranks sweep time (untrained brick models: throughput only)."""
    import torch
    from paper_2308_02494_b200 import _lib as L
    from paper_2308_02494_b200 import model as PM
    from paper_2308_02494_b200 import volume as PV
    from paper_2308_02494_b200.decomposition import DecomposedField, DecompositionManifest, plan_partition
    plan = plan_partition(dims, *counts, ghost=1)
    nb = plan.brick_count
    mine = [b for b in range(nb) if b % world == rank]
    models = [PM.init_model(PM.ModelConfig(M, CH, RES), seed=(0 ^ b) & 0x7FFFFFFF) if b in mine else None
              for b in range(nb)]
    field = DecomposedField(DecompositionManifest(plan=plan, volume_header=PV.VolumeHeader(dims=dims), bricks=[]),
                            models)
    boxes = field.brick_boxes(dims)
    blobs = [PV.BlobSpec(c, s, a) for c, s, a in BLOBS]
    truth, recon = {}, {}
    for b in mine:
        x0, x1, y0, y1, z0, z1 = boxes[b]
        ext = PV.Extent(lo=(x0, y0, z0), hi=(x1, y1, z1))
        truth[b] = PV.synth_volume_device(dims, blobs, extent=ext)
        recon[b] = torch.empty_like(truth[b])
    field.device_models()
    sse = L.zeros((1,), np.float64)
    field.lattice_sse_local(mine, truth, recon, sse)  # warm-up
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sse.zero_()
    e0.record()
    field.lattice_sse_local(mine, truth, recon, sse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        total = sse.to(dev)
        dist.all_reduce(total)  # PSNR statistic over all bricks
        sse_all = float(total.item())
    else:
        sse_all = float(sse.item())
    vox = dims[0] * dims[1] * dims[2]
    return {"metric": "inference voxels/sec", "value": vox / (ms * 1e-3), "ms_per_sweep": ms,
            "config": f"C5: {dims[0]}^3 lattice, {counts[0]}x{counts[1]}x{counts[2]} bricks (ghost 1), "
                      f"{len(mine)} bricks on rank {rank} of {world}, PSNR + reconstruct mode, "
                      f"box-local truth/recon per rank, SSE all-reduced",
            "sse": sse_all}


if __name__ == "__main__":
    main()
