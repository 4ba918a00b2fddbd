"""Split a fused kernel's SASS (from an `ncu --page source --print-source
cuda,sass` export) into phases by the kernel-file line each instruction
run maps to; prints instructions and stall samples per phase."""
import csv, gzip, sys, os, collections
f, kfile = sys.argv[1], sys.argv[2]
bounds = [int(x) for x in sys.argv[3].split(",")]  # line starts: pre, A, B, D, C, end
names = ["pre", "A", "B", "D", "C", "tail"]
pts = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
fh = gzip.open(f, "rt") if f.endswith(".gz") else open(f)
cur = None; line = None; rows = []
for r in csv.reader(fh):
    if not r: continue
    if r[0] == "File Path": cur = os.path.basename(r[1]); continue
    if r[0] in ("Line No", "Function Name"): continue
    if r[0] != "":
        try: line = int(r[0])
        except ValueError: line = None
        continue
    # sass row: "", "", address, source, stallAll, stallNot, samples, inst, threadinst
    try:
        addr = int(r[2], 16); n = int(r[8] or 0); s = int(r[4] or 0)
    except (ValueError, IndexError):
        continue
    rows.append((addr, cur, line, n, s, r[3].strip()))
rows.sort()
def phase(l):
    for i in range(len(bounds) - 1, -1, -1):
        if l >= bounds[i]: return names[min(i + 1, len(names) - 1)] if i + 1 < len(names) else names[-1]
    return "pre"
ph = "pre"; ins = collections.Counter(); st = collections.Counter(); ops = collections.defaultdict(collections.Counter)
for addr, fi, l, n, s, src in rows:
    if fi == kfile and l is not None:
        ph = phase(l)
    ins[ph] += n; st[ph] += s
    opc = src.split()[0] if src else "?"
    if opc.startswith("@"): opc = src.split()[1]
    ops[ph][opc.split(".")[0]] += n
ti = sum(ins.values()); ts = sum(st.values())
for p in names:
    if ins[p] == 0: continue
    top = ", ".join(f"{k} {v/pts:.0f}" for k, v in ops[p].most_common(8))
    print(f"{p:5s} inst/pt {ins[p]/pts:7.1f} ({100*ins[p]/ti:4.1f}%)  stall {100*st[p]/ts:4.1f}%   {top}")
