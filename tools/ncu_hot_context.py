"""SASS context around the hottest stall sites of an ncu source-page CSV (--print-source sass):
for each of the top-N addresses by warp-stall samples, the instructions before and after it with
their own sample share — to tell which barrier / load a stall belongs to."""
import csv
import io
import sys


def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0


rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read())))
hdr_i = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hdr_i]
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
data, seen = [], set()
for r in rows[hdr_i + 1:]:
    if len(r) == len(h) and r[0] != "Address" and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
tot = sum(f(r[ix[S]]) for r in data) or 1.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6
order = sorted(range(len(data)), key=lambda i: -f(data[i][ix[S]]))[:n]
for i in order:
    print(f"==== {100 * f(data[i][ix[S]]) / tot:5.1f}% at {data[i][ix['Address']]}")
    for j in range(max(0, i - ctx), min(len(data), i + ctx + 1)):
        mark = ">>" if j == i else "  "
        print(f"{mark} {100 * f(data[j][ix[S]]) / tot:5.1f}%  {data[j][ix['Source']][:90]}")
