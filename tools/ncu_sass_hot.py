"""Summarise an ncu --page source --print-source sass CSV: stall totals and hottest instructions (dev tool)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0] != "Address"]
ci = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for r in data:
    for s in stalls:
        try: tot[s] += int(r[ci[s]])
        except ValueError: pass
allS = sum(tot.values())
print("total samples", allS)
for s, v in tot.most_common(12):
    print(f"  {s:28s} {v:8d} {100*v/max(allS,1):5.1f}%")
ops = collections.Counter(); ops_exec = collections.Counter()
for r in data:
    op = r[ci["Source"]].strip().split()[0] if r[ci["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ci["Source"]].strip().split()[1]
    ops[op.split(".")[0]] += int(r[ci["# Samples"]] or 0)
    ops_exec[op.split(".")[0]] += int(r[ci["Instructions Executed"]] or 0)
te = sum(ops_exec.values())
print("instructions executed by opcode (warp-level):", te)
for o, v in ops_exec.most_common(25):
    print(f"  {o:10s} {v:12d} {100*v/te:5.1f}%   samples {ops[o]}")
data.sort(key=lambda r: -int(r[ci["# Samples"]] or 0))
print("hottest instructions:")
for r in data[:top]:
    s = {k: int(r[ci[k]]) for k in stalls if r[ci[k]] not in ("", "0")}
    best = sorted(s.items(), key=lambda kv: -kv[1])[:3]
    print(f"  {r[ci['# Samples']]:>6s} {r[ci['Source']].strip()[:70]:70s} {best}")
