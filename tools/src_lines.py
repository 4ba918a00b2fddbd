"""Per-CUDA-line instruction counts and stall samples from an
`ncu --page source --csv --print-source cuda,sass` export (gzipped ok)."""
import csv, gzip, sys, collections, os
f = sys.argv[1]; pts = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fh = gzip.open(f, "rt") if f.endswith(".gz") else open(f)
cur = None; hdr = None; agg = collections.Counter(); st = collections.Counter(); txt = {}
tot_i = tot_s = 0
for r in csv.reader(fh):
    if not r: continue
    if r[0] == "File Path": cur = os.path.basename(r[1]); continue
    if r[0] == "Line No": hdr = {k: i for i, k in enumerate(r) if k not in ("Source",)}; continue
    if hdr is None or r[0] == "" or r[0] == "Function Name": continue
    try:
        n = int(r[8] or 0); s = int(r[4] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur, int(r[0])); agg[key] += n; st[key] += s; txt[key] = r[1].strip()[:80]
    tot_i += n; tot_s += s
print(f"thread-inst per point {tot_i/pts:.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -st[kv[0]])[:top]:
    print(f"{k[0]:22s}:{k[1]:<4d} inst/pt {v/pts:7.1f} ({100*v/tot_i:4.1f}%)  stall {100*st[k]/tot_s:4.1f}%  {txt[k]}")
