"""Instructions and stall samples of a fused kernel per barrier-delimited
region (the compiler cannot move code across BAR.SYNC), from an
`ncu --page source --print-source cuda,sass` (or sass) CSV export."""
import csv, gzip, sys, collections
f = sys.argv[1]; pts = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
seen = {}
for r in csv.reader(gzip.open(f, "rt") if f.endswith(".gz") else open(f)):
    if len(r) < 9 or not r[2].startswith("0x"):
        continue
    try:
        a = int(r[2], 16); s = int(r[4] or 0); n = int(r[8] or 0)
    except ValueError:
        continue
    seen[a] = (s, n, r[3].strip())
rows = sorted(seen.items())
bars = [a for a, (s, n, src) in rows if "BAR.SYNC" in src]
regions = collections.OrderedDict()
ops = collections.defaultdict(collections.Counter)
stl = collections.defaultdict(collections.Counter)
for a, (s, n, src) in rows:
    k = sum(1 for b in bars if a > b)
    regions.setdefault(k, [0, 0]); regions[k][0] += n; regions[k][1] += s
    op = src.split()[0]
    if op.startswith("@"): op = src.split()[1]
    ops[k][op.split(".")[0]] += n; stl[k][op.split(".")[0]] += s
ti = sum(v[0] for v in regions.values()); ts = sum(v[1] for v in regions.values())
print(f"barriers at {[hex(b) for b in bars]}; thread-inst/pt {ti/pts:.1f}")
for k, (n, s) in regions.items():
    top = ", ".join(f"{o} {c/pts:.0f}" for o, c in ops[k].most_common(7))
    tops = ", ".join(f"{o} {100*c/ts:.1f}%" for o, c in stl[k].most_common(4))
    print(f"region {k}: inst/pt {n/pts:7.1f} ({100*n/ti:4.1f}%)  stall {100*s/ts:4.1f}%  [{top}]  stalls[{tops}]")
