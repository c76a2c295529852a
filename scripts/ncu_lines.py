"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
data = []
fname = "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Function Name":
        continue
    if r[0] != "" and len(r) > 7:
        try:
            data.append((float(r[7] or 0), float(r[4] or 0), f"{fname}:{r[0]}", r[1][:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"total warp-inst {tot:.0f}  stall samples {ts:.0f}")
for d in sorted(data, key=lambda x: -(x[0] / tot + x[1] / ts))[:n]:
    print(f"{d[0] / tot * 100:5.1f}% inst {d[1] / ts * 100:5.1f}% samp  {d[2]}: {d[3]}")
