"""Top stalled SASS instructions of an ncu source export (--page source --csv
--print-source sass), with their stall breakdown and a window of context."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[iS]) for r in data)
print("total samples", tot)
agg = {h[i]: sum(int(r[i] or 0) for r in data) for i in st}
print({k: round(v / tot, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
order = sorted(range(len(data)), key=lambda j: -int(data[j][iS]))[:n]
for j in sorted(order):
    r = data[j]
    top = sorted(((int(r[i] or 0), h[i][6:]) for i in st), reverse=True)[:3]
    print(f"{j:5d} {int(r[iS]) / tot * 100:5.2f}% ex={r[iE]:>11} {r[1].strip()[:60]:60s} "
          + " ".join(f"{k}={v}" for v, k in top if v))
