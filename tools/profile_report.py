"""Summarise a gpurun_out/<tag>/ directory (bench.json, raw_<P>.csv from
`ncu --set full`, src_<P>.csv.gz, launches.csv) into markdown for profiles/,
and write profiles/ncu_traffic.json (DRAM bytes per point per fused launch,
used by bench.py for roofline.traffic)."""
import csv, gzip, json, os, re, sys, collections

d = sys.argv[1]; out = sys.argv[2]; npts = int(sys.argv[3]) if len(sys.argv) > 3 else 256 ** 3
BYTES = {"DP": (8, 8, 8, 8), "SPDP": (8, 8, 4, 4), "HPSP": (4, 4, 2, 2), "SP": (4, 4, 4, 4)}
lines = []
b = json.load(open(os.path.join(d, "bench.json"))) if os.path.exists(os.path.join(d, "bench.json")) else None
if b:
    lines.append(f"## bench ({b['config']['workload']}; {b['steps']} steps after {b['warmup']} warm-up)\n")
    lines.append(f"clocks during the timed region: {b.get('clocks')}\n")
    lines.append("| preset | ms / RK step | Gpt/s | B_alg frac of measured HBM |\n|---|---|---|---|")
    for p, v in b["per_precision"].items():
        if "ms_per_step" in v:
            lines.append(f"| {p} | {v['ms_per_step']:.2f} | {v['value']/1e9:.3f} | {100*v['b_alg_frac']:.1f}% |")
    lines.append("")
traffic = {}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for P in ("DP", "SPDP", "HPSP", "SP"):
    f = os.path.join(d, f"raw_{P}.csv")
    if not os.path.exists(f):
        continue
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    vals = rows[2:]
    lines.append(f"## ncu --set full: {P} fused kernel, 256^3, {len(vals)} launch(es)\n")
    lines.append(f"kernel: `{dict(zip(h, vals[0]))['Kernel Name'][:160]}`\n")
    lines.append("| metric | " + " | ".join(f"launch {i}" for i in range(len(vals))) + " | unit |")
    lines.append("|---|" + "---|" * len(vals) + "---|")
    for k in keys:
        if k in h:
            i = h.index(k)
            lines.append(f"| {k} | " + " | ".join(v[i] for v in vals) + f" | {u[i]} |")
    tot = 0.0
    for v in vals:
        dv = dict(zip(h, v)); du = dict(zip(h, u))
        def tobytes(k):
            x = float(dv[k].replace(",", "")); unit = du[k]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        tot += tobytes("dram__bytes_read.sum") + tobytes("dram__bytes_write.sum")
    per_pt = tot / len(vals) / npts
    traffic[P] = per_pt
    bq, bt, br, bw = BYTES[P]
    comp = ((10 * bq + 5 * bt) + 2 * (10 * bq + 10 * bt)) / 3 if len(vals) == 3 else 10 * bq + 5 * bt
    what = ("mean over the 3 substeps: read Q, write Q and Qt, read Qt on substeps 1-2" if len(vals) == 3
            else "substep 0: read Q, write Q and Qt")
    lines.append(f"\nDRAM bytes per point per launch (mean of the captured launches): {per_pt:.1f}; "
                 f"compulsory ({what}): {comp:.1f}\n")
    st = [(float(dict(zip(h, vals[0]))[k]), k[34:-23]) for k in h
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    lines.append("top stall reasons (warps per issue, launch 0): " +
                 ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]) + "\n")
lf = os.path.join(d, "launches.csv")
if os.path.exists(lf):
    txt = open(lf).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.reader(txt[start:]))
    hh = rows[0]
    agg = collections.OrderedDict()
    for r in rows[1:]:
        dd = dict(zip(hh, r))
        if dd.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = dd["Kernel Name"][:70]
        t = float(dd["Metric Value"].replace(",", ""))
        unit = dd.get("Metric Unit", "")
        t *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
        a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += t
    tot = sum(v[1] for v in agg.values())
    lines.append("## launch list (ncu gpu__time_duration, 256^3 DP, warm-up + 1 step; cold, serialised)\n")
    lines.append("| share | launches | avg us | kernel |\n|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {100*t/tot:.1f}% | {c} | {t/c:.1f} | `{k}` |")
    lines.append("")
open(out, "w").write("\n".join(lines) + "\n")
tj = os.path.join(os.path.dirname(out), "ncu_traffic.json")
old = json.load(open(tj)) if os.path.exists(tj) else {}
for P, v in traffic.items():
    old[f"{P}/fused/bytes_per_pt"] = round(v, 2)
old["source"] = f"ncu --set full captures in {d} (256^3), dram__bytes_read.sum + dram__bytes_write.sum"
json.dump(old, open(tj, "w"), indent=1)
print(open(out).read())
