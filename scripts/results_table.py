"""Markdown results table from a directory of bench.py JSON lines.

    python scripts/results_table.py profiles/r02/final
"""
import json
import os
import sys

NAMES = {"A": "A: SBM 1e4, k=8, GPA", "B": "B: SBM 1e6, k=16, FISTA+BT", "C": "C: citation 1e7 / nnz 4.1e8, k=32",
         "Cloc": "Cloc: C with locality on", "D": "D: citation 7e7 / nnz 2.1e9, k=32", "E8": "E8: citation 4e6, k=8",
         "E32": "E32", "E64": "E64", "E128": "E128"}
PEAK = 6452.8


def main():
    d = sys.argv[1]
    print("| Config | iter/s (device) | ms / iter | e2e iter/s | CPU ref iter/s (16 thr) | device / CPU | "
          "tolerance ms / iter | sweep roofline frac | iteration HBM frac | SM MHz |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for c in ["A", "B", "C", "Cloc", "D", "E8", "E32", "E64", "E128"]:
        p = os.path.join(d, f"{c}.jsonl")
        if not os.path.exists(p):
            continue
        r = json.loads(open(p).readline())
        t = r.get("tolerance_mode") or {}
        e = r.get("e2e") or {}
        cpu = (r.get("cpu_baseline") or {}).get("value")
        tol = f"{t['ms_per_step']:.2f} ({t['value']:.1f} iter/s)" if t.get("ms_per_step") else "—"
        sw = f"{r['roofline']['frac']:.2f}" if c != "A" else "launch-bound"
        ratio = f"{r['value'] / cpu:,.0f}×" if cpu else "—"
        cpus = f"{cpu:.4g}" if cpu else "—"
        print(f"| {NAMES[c]} | {r['value']:,.1f} | {r['ms_per_step']:.2f} | {e.get('value', 0):,.1f} | {cpus} | "
              f"{ratio} | {tol} | {sw} | {r['achieved_gbs'] / PEAK:.2f} | {r['clocks']['sm_mhz']:.0f} |")


if __name__ == "__main__":
    main()
