"""Instructions executed per CUDA source line from `ncu -i R --page source --print-source cuda,sass --csv` (dev tool)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
path = None
agg = collections.Counter(); samp = collections.Counter(); text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and r[0] != "" and len(r) > 8 and r[2] == "-":
        key = (path, int(r[0]))
        try:
            agg[key] += int(r[7]); samp[key] += int(r[6])
        except ValueError:
            pass
        text[key] = r[1].strip()[:100]
tot = sum(agg.values())
print("total warp instructions", tot, "samples", sum(samp.values()))
for k, v in agg.most_common(top):
    print(f"{v:8d} {100*v/tot:5.1f}%  s={samp[k]:3d}  {k[0]}:{k[1]}  {text[k]}")
