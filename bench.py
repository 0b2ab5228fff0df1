"""Benchmark: APMGSRN training throughput (train points/sec) on B200.

Workload (BASELINE.json configs[1], "C2"): 64 grids 32^3 x 2 features, MLP 2x64,
fit a synthetic 512^3 blob volume (test_acceptance.py:156-164 blob list),
batch 2^20, density loss on every timed iteration.  One "step" = one training
iteration (Philox batch + fp64 targets + fused recon fwd/bwd + masked Adam +
fp64 density step + scheduler), all device-resident.

N > 1 (torchrun): weak scaling -- rank r trains brick r of the 2x2x2
decomposition of a synthetic 1024^3 volume (configs[3]); each brick is an
independent model (ghost extent ~513^3), no data-path collective; the timing
is the max over ranks.

``--impl reference`` times the reference algorithm (the numpy oracle port; the
reference itself is pure numpy and not installed on the GPU box) on the host
cores on a bounded sample of the same workload.
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
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows, self.proc = [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:  # nvidia-smi needs a moment to start
                time.sleep(0.02)
            self.rows.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows)}


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


def brick_workload(rank, world):
    """(volume dims, extent or None, description) of this rank's training unit."""
    from paper_2308_02494_b200.decomposition import plan_partition
    if world == 1:
        return DIMS1, None, "C2: single model, synthetic 512^3 volume"
    plan = plan_partition(DIMS_DECOMP, 2, 2, 2, ghost=1)
    brick = plan.bricks[rank % plan.brick_count]
    return DIMS_DECOMP, brick.ghost, f"C4: brick {rank % 8} of 2x2x2 over synthetic 1024^3 (ghost 1)"


# algorithmic work per training point -> per-kernel roofline rows
ENC_BYTES = 8 * M * CH * 4          # 4,096 B of corner data gathered per point (encoder fwd)
SCAT_BYTES = 8 * M * CH * 4         # 4,096 B of corner gradients reduced per point (encoder bwd)
STREAM_BYTES = 12 + 4 + 4           # coords in, target in, squared error out


def roofline_for(kernel: str, ms_per_launch: float, pk: dict):
    """Dominant-kernel roofline.  Bytes are ALGORITHMIC bytes per launch (SURVEY 8d per-point
    figure x the 2^20 points one launch processes); the grid gather/scatter traffic is served
    by L2 (16 MiB grids stay resident), so the HBM copy peak is a conservative denominator."""
    t = ms_per_launch * 1e-3
    per_point = {
        "recon_fwd_bwd_tc": ENC_BYTES + SCAT_BYTES + STREAM_BYTES,
        "recon_fwd_bwd": ENC_BYTES + SCAT_BYTES + STREAM_BYTES,
        "density_grad": 12 + 4,
        "density_rho": 12 + 4 + 8,
        "train_batch": 8 * 4 + 16,
    }
    if kernel == "adam_main":
        nbytes = 4_206_656 * 4 * 7
    else:
        nbytes = BATCH * per_point.get(kernel, float("nan"))
    peak = pk.get("hbm_gbs", 6650.0)
    achieved = nbytes / t / 1e9
    traffic = None
    tf = ROOT / "profiles" / "traffic_r01.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(kernel)
    out = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak, "traffic": traffic, "ms_per_launch": ms_per_launch,
           "bytes_per_launch": nbytes, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)",
           "note": "algorithmic encoder gather + scatter bytes (4096+4096+20 B/pt); served from L2"}
    pf = ROOT / "profiles" / "peaks_b200.json"
    if kernel.startswith("recon_fwd_bwd") and pf.exists():
        # encoder fwd is bound by L2 gather bandwidth, encoder bwd by L2 RED
        # throughput -- algorithmic units of one launch against the probes of tools/peaks.py
        pk2 = json.loads(pf.read_text())
        g_ach = BATCH * ENC_BYTES / t / 1e9
        r_ach = BATCH * (SCAT_BYTES // 8) / t / 1e9
        fl_ach = BATCH * 74112 / t / 1e12
        fl_iss = BATCH * (24704 * 6 + 49152 * 3) / t / 1e12
        out["l2"] = {
            "gather": {"achieved": g_ach, "peak": pk2["l2_gather_float2_GBps_16MiB"], "unit": "GB/s",
                       "frac": g_ach / pk2["l2_gather_float2_GBps_16MiB"]},
            "red": {"achieved": r_ach, "peak": pk2["l2_red_float2_Gops_16MiB"], "unit": "G float2 RED/s",
                    "frac": r_ach / pk2["l2_red_float2_Gops_16MiB"]},
            "mlp_tensor": {"achieved": fl_ach, "issued": fl_iss, "peak": pk["bf16_tflops"],
                           "unit": "TFLOP/s (bf16 tensor pipe)", "frac": fl_iss / pk["bf16_tflops"],
                           "note": "achieved = algorithmic MLP FLOP (74,112/pt); issued = bf16x3 products "
                                   "(6 per forward, 3 per backward product: 295,680 FLOP/pt)"},
            "peak_source": "profiles/peaks_b200.json (tools/peaks.py: random float2 over a 16 MiB table)",
            "note": "gather and RED are the un-aggregated algorithmic counts (512 corner loads and 512 "
                    "float2 REDs per point); warp coherence and aggregation let the kernel exceed the "
                    "random-access RED probe"}
    return out


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


def run_cpu_baseline(vol_host, seconds_budget=25.0):
    """Oracle port (reference algorithm, numpy) on a bounded sample: batch 2^16, density on."""
    from oracle import apmg_oracle as O
    batch = 1 << 16
    prm = O.init_params(M, CH, RES, seed=0, vmin=float(vol_host.min()), vmax=float(vol_host.max()))
    stamps = []
    cfg = O.LoopConfig(iterations=4, batch_size=batch, delay_start=0, transform_hard_stop_fraction=1.0,
                       plateau_enabled=False, seed=0)
    t0 = time.perf_counter()
    O.train_single(prm, vol_host, cfg, on_iteration=lambda it, p: stamps.append(time.perf_counter()))
    per_it = np.diff([t0] + stamps)[1:]  # drop the first (warm-up) iteration
    rate = batch / float(np.mean(per_it))
    return {"value": rate, "unit": METRIC, "cores": os.cpu_count(), "kind": "port",
            "sample": f"3 timed iterations (after 1 warm-up) of batch 2^16, density on, same model/512^3 volume; "
                      f"numpy oracle restating apmg.train_single, {os.cpu_count()} host threads available"}


def run_reference(args):
    dist, rank, world, _ = dist_setup() if int(os.environ.get("WORLD_SIZE", "1")) > 1 else (None, 0, 1, 0)
    if rank != 0:
        return
    from oracle import apmg_oracle as O
    vol = O.synth_volume(DIMS1, BLOBS)
    batch = 1 << 16
    prm = O.init_params(M, CH, RES, seed=0, vmin=float(vol.min()), vmax=float(vol.max()))
    total = args.warmup + args.steps
    cfg = O.LoopConfig(iterations=total, batch_size=batch, delay_start=0, transform_hard_stop_fraction=1.0,
                       plateau_enabled=False, seed=0)
    stamps = []
    budget = float(os.environ.get("APMG_REF_BUDGET_S", "150"))
    t_start = time.perf_counter()

    class Budget(Exception):
        pass

    def cb(it, p):
        stamps.append(time.perf_counter())
        if it >= args.warmup and stamps[-1] - stamps[args.warmup - 1 if args.warmup else 0] > budget:
            raise Budget()

    try:
        O.train_single(prm, vol, cfg, on_iteration=cb)
    except Budget:
        pass
    t0 = stamps[args.warmup - 1] if args.warmup else t_start
    timed = len(stamps) - args.warmup
    dt = stamps[-1] - t0
    value = timed * batch / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world,
            "steps": timed, "warmup": args.warmup, "ms_per_step": 1e3 * dt / timed, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
            "config": {"workload": "C2 sample: 64 grids 32^3x2, MLP 2x64, synthetic 512^3, density on",
                       "global_batch": batch, "note": "reference step = one iteration at batch 2^16 (bounded)"},
            "cpu_baseline": {"value": value, "unit": METRIC, "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{timed} iterations of batch 2^16 (numpy oracle of apmg.train_single)"},
            "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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

    import torch
    from paper_2308_02494_b200 import _lib as L
    from paper_2308_02494_b200 import model as PM
    from paper_2308_02494_b200 import trainer as PT
    from paper_2308_02494_b200 import volume as PV

    dist, rank, world, local = dist_setup()
    torch.cuda.set_device(local)
    L.lib()
    dims, extent, desc = brick_workload(rank, world)
    blobs = [PV.BlobSpec(c, s, a) for c, s, a in BLOBS]
    vdev = PV.synth_volume_device(dims, blobs, extent=extent)
    vshape = extent.shape() if extent is not None else dims
    vol = PV.Volume.from_device(vshape, vdev)
    seed = (0 ^ rank) & 0x7FFFFFFF
    model = PM.init_model(PM.ModelConfig(M, CH, RES), seed=seed, vmin=vol.vmin, vmax=vol.vmax)
    K, W = args.steps, max(args.warmup, 3)
    KT = 5  # untimed iterations after the timed region, run with per-kernel CUDA events
    cfg = PT.TrainConfig(iterations=W + K + KT, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                         plateau_enabled=False, seed=seed)
    sess = PT.TrainSession(model, vol, cfg)
    sess.run(W)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.lib().apmg_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0.record(stream)
        sess.run(K)
        e1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
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
    if dist:
        t = torch.tensor([ms], device="cuda" if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    log = sess.log()
    sess.close()
    value = world * K * BATCH / (ms * 1e-3)

    # dominant kernel and its roofline
    dom = max(ktab.items(), key=lambda kv: kv[1]["total_ms"])
    pk = peaks()
    roof = roofline_for(dom[0], dom[1]["total_ms"] / dom[1]["launches"], pk)
    shares = {k: round((v["total_ms"] / KT) / (ms / K), 4)
              for k, v in sorted(ktab.items(), key=lambda kv: -kv[1]["total_ms"])}

    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        host_vol = PV.Volume(dims=vshape, data=L.to_host(vdev))
        m2 = PM.init_model(PM.ModelConfig(M, CH, RES), seed=seed, vmin=vol.vmin, vmax=vol.vmax)
        cfg2 = PT.TrainConfig(iterations=K, batch_size=BATCH, delay_start=0, transform_hard_stop_fraction=1.0,
                              plateau_enabled=False, seed=seed)
        # one untimed warm-up call (first-use costs: staging ring, allocator pools, graph build)
        mw = PM.init_model(PM.ModelConfig(M, CH, RES), seed=seed, vmin=vol.vmin, vmax=vol.vmax)
        # (its own Volume object: a Volume caches its device copy, and the timed call must upload)
        PT.train_single(mw, PV.Volume(dims=vshape, data=host_vol.data), PT.TrainConfig(iterations=max(W, 1), batch_size=BATCH, delay_start=0,
                                                     transform_hard_stop_fraction=1.0, plateau_enabled=False,
                                                     seed=seed))
        del mw
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        _, log2 = PT.train_single(m2, host_vol, cfg2)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            tt = torch.tensor([dt], device="cuda" if dist.get_backend() == "nccl" else "cpu",
                              dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        params_b = 4 * m2.parameter_count()
        e2e = {"value": world * K * BATCH / dt, "unit": METRIC,
               "h2d_bytes_per_step": int((host_vol.data.nbytes + params_b + 16 * K) / K),
               "d2h_bytes_per_step": int((params_b + 24 * K) / K),
               "setup_ms": round(1e3 * log2.setup_seconds, 2), "setup_split_ms": log2.setup_ms,
               "wall_ms": round(1e3 * dt, 2),
               "note": f"paper_2308_02494_b200.train_single(host model, host Volume, iterations={K}): "
                       f"volume + parameter upload, device loop, parameter + log download"}

    infer = None
    if not args.no_inference:
        infer = bench_inference(model_from_session=None) if world == 1 else \
            bench_decomposed_inference(rank, world, dist)

    render = None
    if rank == 0 and world == 1 and not args.no_render:
        render = bench_render()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(L.to_host(vdev))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (bf16x3 tensor-core MLP: 6-product forward, 3-product backward; f64 density statistics and loss)", "data": "synthetic",
            "config": {"workload": desc, "global_batch": BATCH * world, "model": "APMGSRN 64 grids 32^3 x2, MLP 2x64",
                       "density_loss": "every timed iteration", "parallelism": f"brick-sharded x{world}",
                       "l2": "inputs larger than L2 (512 MiB+ volume per rank); 16 MiB grids L2-resident by design"},
            "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roof,
            "kernel_share": shares, "e2e": e2e, "cpu_baseline": cpu, "inference": infer, "render": render,
            "final_l_rec": log.l_rec[-1] if log.l_rec else None,
        }
        print(json.dumps(line), flush=True)
    if dist:
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


def bench_inference(model_from_session=None, dims=(1024, 1024, 1024)):
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
    return {"metric": "inference voxels/sec", "value": vox / (ms * 1e-3), "ms_per_sweep": ms,
            "config": "C3: 1024^3 lattice, one 64x32^3x2 model, fused forward + fp64 SSE vs truth"}


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
