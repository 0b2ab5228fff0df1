"""profiles/traffic_<tag>.json: DRAM bytes (read + write) and L2 bytes (32 x lts__t_sectors) per launch of each kernel bench.py
names in its roofline, taken from the `--set full` summaries make_profiles.py wrote."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NAMES = {  # ncu kernel name (prefix) -> the launch name bench.py's timer reports
    "k_batch_keys": "batch_keys", "k_bucket_scatter": "bucket_scatter", "k_sample_sorted": "train_batch",
    "tc16::k_recon_tc16": "recon_fwd_bwd_tc", "k_adam_train": "adam_main", "k_dens_rho32": "density_rho",
    "k_dens_grad32c": "density_grad", "k_infer_tc": "infer_lattice_tc"}


def main(tag, *summaries):
    out = {}
    for s in summaries:
        for k in json.loads((ROOT / "profiles" / f"{s}.json").read_text()).get("full", []):
            for pre, name in NAMES.items():
                if k["kernel"].startswith(pre) and name not in out:
                    out[name] = {"dram": float(k["dram_read"]) + float(k["dram_write"]),
                                 "l2": 32.0 * float(k.get("l2_sectors", 0.0)) or None,
                                 "l2_red_sectors": float(k["l2_red_sectors"]) if float(k.get("l2_red_sectors") or 0) > 0 else None}
    (ROOT / "profiles" / f"traffic_{tag}.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], *sys.argv[2:])
