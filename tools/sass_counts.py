"""Per-kernel SASS opcode counts of the built libraries (cuobjdump -sass): the evidence that the
hot kernels run on tcgen05 (UTCHMMA / UTCBAR), TMEM (LDTM / STTM), vector gathers (LDG.E.128) and
float4 REDs (REDG.E.ADD.F32x4...).  Writes profiles/sass_<tag>.json.

    python tools/sass_counts.py r02 [kernel-substring ...]"""
import json
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2308_02494_b200" / "libapmg_cuda.so"
KEEP = ("UTCHMMA", "UTCBAR", "UTCMMA", "LDTM", "STTM", "LDG", "REDG", "REDUX", "SHFL", "MATCH", "LDS", "STS",
        "FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD", "MUFU", "DFMA", "DMUL", "DADD", "SYNCS", "BAR", "BRA",
        "UBLKCP", "UTMALDG")


def counts(lib=LIB):
    out = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
        if m and cur:
            op = m.group(2)
            funcs[cur][op] += 1
    return funcs


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else list(names)


def main(tag, *subs):
    subs = subs or ("k_recon_tc16", "k_infer_tc", "k_dens_grad32cx2", "k_dens_rho32x2", "k_adam_train",
                    "k_sample_sorted_cells", "k_batch_keys")
    funcs = counts()
    names = list(funcs)
    pretty = dict(zip(names, demangle(names)))
    res = {}
    for n, c in funcs.items():
        p = pretty[n]
        if not any(s in p for s in subs):
            continue
        ops = Counter()
        for op, k in c.items():
            base = op if op.startswith(("REDG", "LDG")) else op.split(".")[0]
            if base.startswith(KEEP) or op.startswith(KEEP):
                ops[base] += k
        res[p.split("(")[0] + ("<1>" if "(bool)1" in p or "<true>" in p else "")] = {
            "total_instructions": sum(c.values()), **dict(sorted(ops.items()))}
    (ROOT / "profiles" / f"sass_{tag}.json").write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if len(sys.argv) < 2:
        sys.exit(__doc__)  # a tag is required: a run without one must not overwrite a committed summary
    main(*sys.argv[1:])
