"""Markdown report of a same-box SOTA comparison (scripts/sota.py output).

    python scripts/sota_report.py SOTA.json SOTAGRID.json TITLE > profiles/r02/<name>_vs_sota.md

SOTA.json: the BASELINE configs (list of {config, impl, ms, TFLOP/s | GB/s, ours_over_theirs_time}).
SOTAGRID.json: the C5 grid rows plus a trailing {"relative_cdf_vs_best_library": {...}} summary —
best-library time / our time per shape, as ktune's relative_cdf reports it (ref/pkg/src/ktune/report.py:196-230).
"""

from __future__ import annotations

import json
import sys
from collections import defaultdict


def main(sota_path: str, grid_path: str, title: str) -> None:
    sota = json.load(open(sota_path))
    grid = json.load(open(grid_path))
    print(f"# {title}\n")
    print("Method: `scripts/sota.py` times every implementation on the same device tensors, graph-amortised with CUDA")
    print("events after warm-up; ours go through the shipped dispatch table. `ours/theirs` is a time ratio (below 1 =")
    print("we are faster). Grid ratios are best-library time / our time (above 1 = we are faster).\n")
    print("## BASELINE configs\n")
    print("| config | impl | ms | throughput | ours/theirs (time) |")
    print("|---|---|---|---|---|")
    for r in sota:
        if "config" not in r:
            continue
        tp = f"{r['TFLOP/s']:.0f} TFLOP/s" if "TFLOP/s" in r else f"{r.get('GB/s', 0):.0f} GB/s"
        rat = r.get("ours_over_theirs_time")
        print(f"| {r['config']} | {r['impl']} | {r['ms']:.4f} | {tp} | {'—' if rat is None else f'{rat:.3f}'} |")
    summary = next((r["relative_cdf_vs_best_library"] for r in grid if "relative_cdf_vs_best_library" in r), None)
    rows = defaultdict(dict)
    for r in grid:
        if "config" in r:
            rows[r["config"]][r["impl"]] = r["ms"] * 1e3
    print("\n## C5 grid (µs per call)\n")
    impls = sorted({i for v in rows.values() for i in v}, key=lambda i: (not i.startswith("b200attn"), i))
    print("| shape | " + " | ".join(impls) + " |")
    print("|---|" + "---|" * len(impls))
    for shape, v in rows.items():
        print(f"| {shape} | " + " | ".join(f"{v[i]:.1f}" if i in v else "—" for i in impls) + " |")
    if summary:
        print("\n## relative_cdf vs the best library per shape\n")
        print("| op | shapes | mean | min | max | fraction ≥ 1 |")
        print("|---|---|---|---|---|---|")
        for op, s in summary.items():
            if isinstance(s, dict) and "mean" in s:
                print(f"| {op} | {s['shapes']} | {s['mean']:.3f} | {s['min']:.3f} | {s['max']:.3f} | {s['frac_ge_1']:.2f} |")


if __name__ == "__main__":
    main(*sys.argv[1:4])
