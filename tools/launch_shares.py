"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file) into per-kernel shares."""
import csv
import sys
from collections import defaultdict


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    tot, cnt = defaultdict(float), defaultdict(int)
    seq = []
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")[:70]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1e-6)
        tot[short] += ms
        cnt[short] += 1
        seq.append((short, r[idx["Grid Size"]], ms))
    T = sum(tot.values()) or 1.0
    print(f"{'kernel':72s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:72s} {cnt[k]:8d} {v:10.2f} {100 * v / T:6.1f}%")
    print("\nlaunch sequence (grouped GEMMs, first evaluation):")
    n = 0
    for short, grid, ms in seq:
        if "grouped_gemm" in short:
            print(f"  {short[:60]:60s} grid={grid:>16s} {ms:10.3f} ms")
            n += 1
            if n >= 24:
                break


if __name__ == "__main__":
    main(sys.argv[1])
