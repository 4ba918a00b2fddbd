"""Summarise an ncu --set full report (raw page) into a markdown table row set."""
import csv, subprocess, sys, re
rep = sys.argv[1]; pts = int(sys.argv[2]) if len(sys.argv) > 2 else 256**3
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines())); hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
print(f"kernel: `{d['Kernel Name'][:150]}`\n")
print("| metric | value | unit | per point |\n|---|---|---|---|")
for k in keys:
    if k not in d: continue
    v = d[k]
    try: per = f"{float(v.replace(',', '')) / pts:.3g}"
    except ValueError: per = ""
    if k.endswith(".sum") and "inst" in k: per = f"{float(v.replace(',', '')) * 32 / pts:.0f} thread-inst"
    print(f"| {k} | {v} | {u.get(k, '')} | {per} |")
stalls = [(float(d[h]), h) for h in hdr if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", h)]
print("\ntop stall reasons (warps per issue): " + ", ".join(f"{h[34:-23]} {v:.2f}" for v, h in sorted(stalls, reverse=True)[:6]))
