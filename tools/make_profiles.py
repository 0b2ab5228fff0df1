"""Summarise ncu artefacts into profiles/ (tracked): the per-launch list of one bench-shaped
run (gpu__time_duration, cold-cache and serialised -- compare SHARES) and the `--set full`
capture of the top kernels (duration, DRAM bytes, throughput %, registers)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def launch_list(csv_path):
    rows = list(csv.reader(open(csv_path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(lambda: [0.0, 0])
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name][0] += float(r[vi].replace(",", "")) / 1e3  # ns -> us
        tot[name][1] += 1
    s = sum(v[0] for v in tot.values())
    return [{"kernel": k, "total_us": round(v[0], 1), "launches": v[1], "share": round(v[0] / s, 4)}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0])]


def full_capture(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr, units = rr[0], rr[1]
    want = {"Kernel Name": None, "gpu__time_duration.sum": "dur", "dram__bytes_read.sum": "dram_read",
            "dram__bytes_write.sum": "dram_write", "lts__t_sectors.sum": "l2_sectors",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
            "launch__registers_per_thread": "regs", "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
            "smsp__inst_executed.sum": "warp_instructions",
            "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_lsu_wavefront_pct",
            "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
            "lts__t_sectors_srcunit_tex_op_red.sum": "l2_red_sectors",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum": "l1_ld_hit_sectors",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "l1_ld_sectors",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "l1_shared_wavefronts",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_wavefront_pct",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait"}
    idx = {k: hdr.index(k) for k in want if k in hdr}
    scale = {"sector": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1}
    out = []
    for r in rr[2:]:
        d = {}
        for k, i in idx.items():
            v = r[i]
            if k == "Kernel Name":
                d["kernel"] = v.split("(")[0].replace("void ", "")
                continue
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            d[want[k]] = f * scale.get(units[i], 1)
        if d.get("dur") and d.get("l2_sectors"):  # achieved L2 throughput (all lts__t sectors x 32 B)
            d["l2_GBps"] = 32.0 * d["l2_sectors"] / (d["dur"] * 1e-3) / 1e9  # dur in ms (ncu unit)
        if d.get("dur") and d.get("dram_read") is not None:
            d["dram_GBps"] = (d["dram_read"] + d.get("dram_write", 0.0)) / (d["dur"] * 1e-3) / 1e9
        out.append(d)
    return out


if __name__ == "__main__":
    tag = sys.argv[1]
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    res = {}
    if len(sys.argv) > 2 and sys.argv[2] and Path(sys.argv[2]).exists():
        res["launches"] = launch_list(sys.argv[2])
    if len(sys.argv) > 3 and Path(sys.argv[3]).exists():
        res["full"] = full_capture(sys.argv[3])
    (prof / f"{tag}.json").write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1)[:3000])
