"""Top SASS lines by warp-stall samples from an ncu source-page CSV (ncu -i rep --page source --csv
--print-source sass), with the dominant stall reasons of each line."""
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
    if len(r) == len(h) and r[0] != "Address" and r[0] not in seen:  # the page repeats each address
        seen.add(r[0])
        data.append(r)
tot = sum(f(r[ix[S]]) for r in data) or 1.0
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
top = sorted(data, key=lambda r: -f(r[ix[S]]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    rs = sorted(((f(r[ix[k]]), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{100 * f(r[ix[S]]) / tot:5.1f}%  {r[ix['Address']]:>6s}  {r[ix['Source']][:60]:60s}  "
          + ", ".join(f"{k}={v:.0f}" for v, k in rs if v > 0))
