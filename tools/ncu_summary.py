"""Summarise an .ncu-rep (details page) into the metrics we track."""
import csv
import subprocess
import sys

SECTIONS = ('GPU Speed Of Light Throughput', 'Memory Workload Analysis', 'Compute Workload Analysis', 'Occupancy',
            'Launch Statistics', 'Warp State Statistics', 'Scheduler Statistics')


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    hdr = next(r)
    for row in r:
        d = dict(zip(hdr, row))
        if d.get('Section Name', '') in SECTIONS and d.get('Metric Name'):
            print(f"{d['Kernel Name'][:30]:30s} | {d['Section Name'][:20]:20s} | {d['Metric Name'][:50]:50s} | "
                  f"{d['Metric Value']} {d.get('Metric Unit', '')}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr = rr[0]
    want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__pipe_tensor",
            "smsp__average_warp_latency_issue_stalled", "smsp__pcsamp_warps_issue_stalled",
            "l1tex__t_bytes.sum", "sm__inst_executed_pipe_fp64", "lts__t_sectors_op_red.sum",
            "lts__t_sectors_op_atom.sum", "sm__sass_thread_inst_executed_op_dfma", "launch__registers")
    for i, name in enumerate(hdr):
        if any(name.startswith(w) for w in want):
            vals = [row[i] for row in rr[2:]]
            print(f"RAW {name}: {rr[1][i]} {vals[:3]}")


if __name__ == "__main__":
    main(sys.argv[1])
