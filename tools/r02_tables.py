"""Markdown table of every profiles/r02_bench_<config>_<precision>.json line."""
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"c1": "c1 N=8192 d=6 r=64 b=.03", "c2": "c2 N=65536 d=3 r=256 b=.05", "c3": "c3 N=2²⁰ d=8 r=512 b=.03",
         "c4": "c4 Exponential N=262144 d=3 r=512 b=.15", "c5": "c5 N=2²² d=3 r=1024 b=0"}


def load(c, p):
    f = os.path.join(HERE, "profiles", f"r02_bench_{c}_{p}.json")
    try:
        return json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        return None


def main():
    print("| config (product-compress tree) | FP64 TFLOP/s (% of 37.07) | FP64 e2e | FP32 TFLOP/s (% of 3xTF32) | "
          "FP32 e2e | ms / evaluation (FP64 / FP32) | rel. error vs ref (FP64 / FP32) | CPU reference GF/s | "
          "same-tree GPU / CPU (device, e2e) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for c in ("c1", "c2", "c3", "c4", "c5"):
        a, b = load(c, "fp64"), load(c, "fp32")
        if a is None:
            continue
        e2e = lambda d: f"{d['e2e']['value'] / 1e3:.2f}" if d and d.get("e2e") else "—"  # noqa: E731
        f32 = f"{b['value'] / 1e3:.1f} ({b.get('pct_3xtf32_peak')} %)" if b else "—"
        ms = f"{a['ms_per_step']:.3g} / {b['ms_per_step']:.3g}" if b else f"{a['ms_per_step']:.3g}"
        rel = f"{a.get('rel_error') or 0:.1e} / " + (f"{b.get('rel_error'):.1e}" if b and b.get("rel_error") else "—")
        cpu = (a.get("cpu_baseline") or {}).get("value")
        sc = a.get("same_config") or {}
        ratio = f"{sc.get('ratio_device')}×, {sc.get('ratio_e2e')}×" if sc else "—"
        print(f"| {NAMES[c]} | {a['value'] / 1e3:.2f} ({a.get('pct_fp64_peak')} %) | {e2e(a)} | {f32} | {e2e(b)} | {ms} | "
              f"{rel} | {cpu if cpu else '—'} | {ratio} |")


if __name__ == "__main__":
    sys.exit(main())
