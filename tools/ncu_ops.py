"""Build profiles/ncu_ops.json (read by bench.py's compute roofline) from
`ncu --set full` captures of the fused kernel: per preset, the floating-point
lane operations per point per launch of the residual compute type (from the
SASS source page: DADD/DMUL/DFMA; FADD/FMUL/FFMA + the packed *2 forms x2;
HADD2/HMUL2/HFMA2 x2), the pipe and issue utilisation and the top stall
reasons (raw page).

  python tools/ncu_ops.py <points> DP=<raw.csv>,<src.csv.gz> SPDP=... HPSP=...
"""
import csv
import gzip
import json
import os
import re
import sys

OPS = {
    "DP": {"DADD": 1, "DMUL": 1, "DFMA": 1},
    "SPDP": {"FADD": 1, "FMUL": 1, "FFMA": 1, "FADD2": 2, "FMUL2": 2, "FFMA2": 2},
    "HPSP": {"HADD2": 2, "HMUL2": 2, "HFMA2": 2, "HADD": 1, "HMUL": 1, "HFMA": 1},
}
PIPE = {"DP": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "SPDP": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "HPSP": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"}


def sass_ops(path, preset):
    fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    tot = 0
    n_all = 0
    seen = set()  # an inlined instruction is listed under every source line it maps to
    for r in csv.reader(fh):
        if len(r) < 9 or r[0] != "":
            continue
        try:
            n = int(r[8] or 0)
            addr = int(r[2], 16)
        except ValueError:
            continue
        if addr in seen:
            continue
        seen.add(addr)
        src = r[3].strip()
        if not src:
            continue
        opc = src.split()[0]
        if opc.startswith("@"):
            opc = src.split()[1]
        base = opc.split(".")[0]
        n_all += n
        tot += n * OPS[preset].get(base, 0)
    return tot, n_all


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    h, vals = rows[0], rows[2]
    d = dict(zip(h, vals))
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    st = sorted(((float(d[k]), k[len(pre):-len(suf)]) for k in h
                 if k.startswith(pre) and k.endswith(suf)), reverse=True)
    return d, st


def main():
    pts = float(sys.argv[1])
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "ncu_ops.json")
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for arg in sys.argv[2:]:
        preset, files = arg.split("=", 1)
        raw, src = files.split(",")
        ops, inst = sass_ops(src, preset)
        d, st = raw_metrics(raw)
        out[f"{preset}/fused/ops_per_pt"] = round(ops / pts, 1)
        out[f"{preset}/fused/thread_inst_per_pt"] = round(inst / pts, 1)
        out[f"{preset}/fused/pipe_active_pct"] = round(float(d[PIPE[preset]]), 1)
        out[f"{preset}/fused/issue_active_pct"] = round(
            float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]), 1)
        out[f"{preset}/fused/warps_active_pct"] = round(
            float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]), 1)
        out[f"{preset}/fused/top_stalls"] = [[name, round(v, 2)] for v, name in st[:5]]
        out[f"{preset}/fused/kernel"] = d.get("Kernel Name", "")[:120]
    out["source"] = "tools/ncu_ops.py over ncu --set full captures (256^3, one launch each); see profiles/README.md"
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
