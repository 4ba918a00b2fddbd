"""Opcode mix and stall hot spots from an `ncu --page source --csv --print-source sass` export."""
import csv, gzip, sys, collections
f = sys.argv[1]
op = gzip.open(f, "rt") if f.endswith(".gz") else open(f)
rows = list(csv.reader(op))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
mix = collections.Counter(); stall = collections.Counter(); tot = 0; tots = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[ix["Source"]].strip()
    opc = src.split()[0] if src else "?"
    if opc.startswith("@"):
        opc = src.split()[1]
    base = opc.split(".")[0]
    n = int(r[ix["Thread Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    mix[base] += n; tot += n; stall[base] += s; tots += s
pts = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"total thread-inst {tot:.4g}  per point {tot/pts:.1f}")
for k, v in mix.most_common(40):
    print(f"  {k:10s} {v/pts:8.1f}/pt  {100*v/tot:5.1f}%   stall-samples {100*stall[k]/max(tots,1):5.1f}%")
