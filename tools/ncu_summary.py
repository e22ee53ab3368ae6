"""Summarise an ncu report (one launch): throughput, pipes, stalls, opcode mix, smem conflicts."""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def f(x):
    try:
        return float(x)
    except Exception:
        return 0.0


def main(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__registers_per_thread"]
    for r in data:
        d = dict(zip(hdr, r))
        print("kernel:", d.get("Kernel Name", "")[:100])
        for w in want:
            if w in d:
                print(f"  {w:75s} {d[w]:>16s} {units[hdr.index(w)]}")
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    h = src[1]
    idx = {k: i for i, k in enumerate(h)}
    rows = [r for r in src[2:] if len(r) == len(h) and r[0] != "Address"]
    S = "Warp Stall Sampling (All Samples)"
    tot = sum(f(r[idx[S]]) for r in rows) or 1.0
    c, n = Counter(), Counter()
    for r in rows:
        toks = r[idx["Source"]].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        c[op] += f(r[idx[S]])
        n[op] += f(r[idx["Instructions Executed"]])
    print("  stall samples by opcode (% of samples, instructions executed M):")
    for op, v in c.most_common(12):
        print(f"    {op:10s} {100 * v / tot:5.1f}%  {n[op] / 1e6:10.1f}")
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    agg = defaultdict(float)
    for r in rows:
        for k in reasons:
            agg[k] += f(r[idx[k]])
    t2 = sum(agg.values()) or 1.0
    print("  stall reasons:", {k[6:]: round(100 * v / t2, 1) for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v > 0.01 * t2})


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
