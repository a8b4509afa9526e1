"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv`
export (one kernel block, selected by index): address, samples, executed
count and the instruction, so hot loops can be mapped back to code."""
import csv
import sys

path, which = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
blocks, cur = [], None
for row in csv.reader(open(path)):
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
    elif row and row[0] == "Address":
        cur["hdr"] = row
    elif cur is not None and row:
        cur["rows"].append(row)
b = blocks[which]
h = b["hdr"]
iA, iS, iN, iE = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                        "Instructions Executed"))
rows = [(int(r[iN] or 0), r[iA], int(float(r[iE] or 0)), r[iS]) for r in b["rows"]]
tot = sum(r[0] for r in rows)
print(b["name"], "samples", tot)
for k, (n, a, e, src) in enumerate(rows):
    pass
for n, a, e, src in sorted(rows, reverse=True)[:top]:
    print(f"{a:>6} {n:7d} {100 * n / tot:5.1f}% exec {e:10d}  {src[:90]}")
