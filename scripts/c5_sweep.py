"""C5 offline sweep: the UNMODIFIED reference autotuner drives our runner.

    python scripts/c5_sweep.py run  --out gpurun_out/c5 [--ops prefill,decode] [--quick]
    python scripts/c5_sweep.py post --out gpurun_out/c5          # no GPU needed

``run`` writes one shapes file per op (batch {1..256} x seq {128..32k}, Llama-3-8B heads) and
calls ``python -m ktune tune --strategy exhaustive`` (ref/pkg/src/ktune/cli.py:255-283) with
``python -m paper_2505_03780_b200.runner`` as the runner (protocol v1), filling a ktune cache
directory (ref/pkg/src/ktune/cache.py).  ktune is imported from ``baseline/_ref`` (pip-installed
from /root/reference, git-ignored, travels with gpurun).

``post`` folds the per-shape results into
  * paper_2505_03780_b200/dispatch_table.json — compact rows {shape, best, median_ms} that
    ``dispatch.load_table`` reads (the per-shape dispatch table the north star asks for);
  * <out>/{op}_{tuned,fixed,heuristic}.csv — ktune report tables (impl, dims..., median_ms);
  * ``ktune report cdf`` of tuned vs the fixed default and vs our untuned heuristic
    (relative_cdf, ref/pkg/src/ktune/report.py:196-230);
  * profiles/r01_c5_summary.json + .md.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = ROOT / "baseline" / "_ref"
SPACES = ROOT / "paper_2505_03780_b200" / "spaces"

BATCHES = [1, 2, 4, 8, 16, 32, 64, 128, 256]
SEQS = [128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768]
HEADS = {"num_q_heads": 32, "num_kv_heads": 8, "head_dim": 128}
SPACE = {"prefill": "flash_attention.space.json", "decode": "paged_decode.space.json"}
BINDING = {"prefill": "prefill.binding.json", "decode": "decode.binding.json"}


# BASELINE.json shapes off the batch x seq grid: C3 (varlen, geometric 128..8192) and one GPU's
# shard of C4 (64 q heads, 32 x 32k) — the configs the bench reports get their own tuned rows
EXTRA = {
    "prefill": [{"op": "prefill", "batch_size": 16, "seq_len_min": 128, "seq_len_max": 8192, "len_dist": "geometric",
                 **HEADS, "causal": True, "dtype": "bfloat16", "seed": 0}],
    "decode": [{"op": "decode", "batch_size": 32, "seq_len": 32768, "num_q_heads": 64, "num_kv_heads": 8,
                "head_dim": 128, "block_size": 16, "dtype": "bfloat16", "seed": 0}],
}


def shapes_for(op: str, quick: bool) -> list[dict]:
    bs = [1, 4, 16, 64] if quick else BATCHES
    ss = [512, 2048, 8192] if quick else SEQS
    out = []
    for b in bs:
        for s in ss:
            d = {"op": op, "batch_size": b, "seq_len": s, **HEADS, "dtype": "bfloat16", "seed": 0}
            if op == "prefill":
                d["causal"] = True
            else:
                d["block_size"] = 16
            out.append(d)
    return out


def ktune(*args, check=True, batch=1, cooldown_ms=0.0):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF), str(ROOT)]), B200ATTN_RUNNER_BATCH=str(batch),
               B200ATTN_RUNNER_COOLDOWN_MS=str(cooldown_ms))
    r = subprocess.run([sys.executable, "-m", "ktune", *args], env=env, capture_output=True, text=True)
    if check and r.returncode != 0:
        sys.stderr.write(r.stdout[-4000:] + r.stderr[-4000:])
        raise SystemExit(f"ktune {args[0]} failed ({r.returncode})")
    return r


def cmd_run(a):
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    for op in a.ops.split(","):
        shapes = EXTRA[op] if a.extra_only else shapes_for(op, a.quick) + EXTRA[op]
        if a.shapes:  # an explicit subset (e.g. the shapes a timed-out run did not reach)
            shapes = [d for d in json.loads(Path(a.shapes).read_text()) if d["op"] == op]
        sf = out / f"{op}_shapes.json"
        sf.write_text(json.dumps(shapes, indent=1))
        runner = f"{sys.executable} -m paper_2505_03780_b200.runner --binding {SPACES / BINDING[op]} --protocol 1 --backend {a.backend}"
        r = ktune("tune", "--space", str(SPACES / SPACE[op]), "--runner", runner, "--shapes", str(sf),
                  "--strategy", "exhaustive", "--cache-dir", str(out / "cache"), "--out", str(out / f"{op}_results"),
                  "--timeout-ms", str(a.timeout_ms), "--json", check=False, batch=a.batch,
                  cooldown_ms=a.cooldown_ms)
        (out / f"{op}_tune.json").write_text(r.stdout)
        (out / f"{op}_tune.err").write_text(r.stderr[-20000:])
        print(f"{op}: ktune tune rc={r.returncode}", flush=True)


# ----------------------------------------------------------------------------- post-processing
def _median(lat):
    return statistics.median(lat)


def _entries(out: Path, op: str):
    for f in sorted((out / f"{op}_results").glob("*.json")):
        doc = json.loads(f.read_text())
        yield doc


def cmd_post(a):
    from paper_2505_03780_b200 import configspace as cs
    from paper_2505_03780_b200 import dispatch

    out = Path(a.out)
    rows_table = []
    summary = {}
    md = ["# C5 sweep: per-shape best config vs fixed default (ktune tune, exhaustive)", ""]
    for op in ("prefill", "decode"):
        if not (out / f"{op}_results").is_dir():
            continue
        space = cs.parse_space((SPACES / SPACE[op]).read_text())
        fixed_cfg = dispatch.PREFILL_FIXED_BASELINE if op == "prefill" else dispatch.DECODE_SPLIT_DEFAULT
        fixed_digest = cs.KernelConfig.from_assignments(fixed_cfg).digest
        tuned, fixed, heur = [], [], []
        per_shape = []
        for doc in _entries(out, op):
            res = doc.get("result", doc)
            shape = doc.get("shape") or res.get("shape")
            best, best_ms = res.get("best"), res.get("best_median_ms")
            if not best or not best_ms:
                per_shape.append({"shape": shape, "best": None, "reason": "no viable config"})
                continue
            if isinstance(best, dict) and "assignments" in best:
                best = best["assignments"]
            meds = {}
            n_ok = n_invalid = 0
            for t in res.get("trace", []):
                o = t["outcome"]
                if o["status"] == "ok":
                    n_ok += 1
                    meds[t["config"]] = min(meds.get(t["config"], 1e30), _median(o["latencies_ms"]))
                elif o["status"] == "invalid":
                    n_invalid += 1
            dims = {k: v for k, v in shape.items()}
            if op == "prefill":
                hcfg = dispatch.PREFILL_DEFAULT
                items_paired = dims["batch_size"] * ((dims.get("seq_len", dims.get("seq_len_max", 0)) + 127) // 128) * \
                    dims["num_q_heads"] // 2
                if items_paired < 148:
                    hcfg = dict(hcfg, BLOCK_M=128)
            else:
                hcfg = dispatch.DECODE_DEFAULT if dispatch.flat_decode_ok(**dims) else dispatch.DECODE_SPLIT_DEFAULT
            h_digest = cs.KernelConfig.from_assignments(hcfg).digest
            row = {"shape": shape, "best": best, "median_ms": best_ms, "configs_ok": n_ok,
                   "configs_invalid": n_invalid}
            if fixed_digest in meds:
                row["fixed_ms"] = meds[fixed_digest]
                fixed.append((dims, meds[fixed_digest]))
                tuned.append((dims, best_ms))
            if h_digest in meds:
                row["heuristic_ms"] = meds[h_digest]
                heur.append((dims, meds[h_digest]))
            per_shape.append(row)
            rows_table.append({"shape": shape, "best": best, "median_ms": best_ms})

        def write_csv(name, impl, rows):
            p = out / f"{op}_{name}.csv"
            if not rows:
                return None
            cols = sorted({c for d, _ in rows for c in d.keys()})
            with open(p, "w", newline="") as fh:
                w = csv.writer(fh)
                w.writerow(["impl", *cols, "median_ms"])
                for dims, ms in rows:
                    w.writerow([impl, *[json.dumps(dims[c]) if isinstance(dims.get(c), bool) else dims.get(c, "")
                                        for c in cols], repr(ms)])
            return p

        t_csv = write_csv("tuned", "tuned", [(d, m) for d, m in ((r["shape"], r["median_ms"]) for r in per_shape
                                                                   if r.get("best"))])
        f_csv = write_csv("fixed", "fixed_default", fixed)
        h_csv = write_csv("heuristic", "heuristic_default", heur)
        # cdf needs exact shape alignment: tuned restricted to shapes the baseline has
        op_sum = {"shapes": len(per_shape), "viable": sum(1 for r in per_shape if r.get("best"))}
        for label, base_csv, base_rows in (("vs_fixed", f_csv, fixed), ("vs_heuristic", h_csv, heur)):
            if base_csv is None:
                continue
            keys = {json.dumps(d, sort_keys=True) for d, _ in base_rows}
            cand = [(r["shape"], r["median_ms"]) for r in per_shape
                    if r.get("best") and json.dumps(r["shape"], sort_keys=True) in keys]
            c_csv = write_csv(f"tuned_{label}", "tuned", cand)
            prefix = out / f"{op}_cdf_{label}"
            r = ktune("report", "cdf", str(c_csv), "--baseline", str(base_csv), "-o", str(prefix), "--no-plot",
                      check=False)
            if r.returncode == 0:
                op_sum[label] = json.loads(Path(str(prefix) + ".json").read_text())
                op_sum[label]["ktune"] = r.stdout.strip()
            else:
                op_sum[label] = {"error": r.stderr.strip()[-500:]}
        summary[op] = {"summary": op_sum, "rows": per_shape}
        md += [f"## {op}", "", "| batch | seq | best | tuned ms | fixed ms | speed-up vs fixed | heuristic ms |",
               "|---|---|---|---|---|---|---|"]
        for r in sorted((r for r in per_shape if r.get("best")),
                        key=lambda r: (r["shape"]["batch_size"], r["shape"].get("seq_len", 0),
                                       r["shape"]["num_q_heads"])):
            s = dict(r["shape"])
            if "seq_len" not in s:
                s["seq_len"] = f"{s['seq_len_min']}..{s['seq_len_max']}"
            if s["num_q_heads"] != 32:
                s["seq_len"] = f"{s['seq_len']} ({s['num_q_heads']}q)"
            bst = ",".join(f"{k}={v}" for k, v in sorted(r["best"].items()))
            fx = r.get("fixed_ms")
            md.append(f"| {s['batch_size']} | {s['seq_len']} | {bst} | {r['median_ms']:.4f} | "
                      f"{fx and f'{fx:.4f}'} | {fx and f'{fx / r['median_ms']:.3f}'} | "
                      f"{r.get('heuristic_ms') and round(r['heuristic_ms'], 4)} |")
        for label in ("vs_fixed", "vs_heuristic"):
            c = op_sum.get(label, {})
            if "mean" in c:
                md.append("")
                md.append(f"relative_cdf {label}: {len(c['ratios'])} shapes, mean {c['mean']:.3f}, "
                          f"min {c['min']:.3f}, max {c['max']:.3f}, frac>=1 {c['frac_ge_1']:.2f}")
        md.append("")
    table_path = ROOT / "paper_2505_03780_b200" / "dispatch_table.json"
    if rows_table and table_path.exists():
        # shapes that were not re-swept (another op, or a sweep cut short) keep their shipped rows
        done = {json.dumps(r["shape"], sort_keys=True) for r in rows_table}
        kept = [r for r in json.loads(table_path.read_text())["rows"] if json.dumps(r["shape"], sort_keys=True) not in done]
        rows_table = kept + rows_table
    if rows_table:
        table_path.write_text(json.dumps({"source": "ktune tune --strategy exhaustive (scripts/c5_sweep.py)",
                                          "rows": rows_table}, indent=0))
    (ROOT / "profiles" / f"{a.tag}_c5_summary.json").write_text(json.dumps(summary, indent=1))
    (ROOT / "profiles" / f"{a.tag}_c5_summary.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["run", "post"])
    ap.add_argument("--out", default="gpurun_out/c5")
    ap.add_argument("--ops", default="prefill,decode")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--batch", type=int, default=1,
                    help="launches per timed graph replay, reported per launch (1 = the reference's semantics)")
    ap.add_argument("--extra-only", action="store_true", help="only the BASELINE shapes off the grid (C3, C4 shard)")
    ap.add_argument("--shapes", help="JSON list of shape dicts to sweep instead of the grid")
    ap.add_argument("--cooldown-ms", type=float, default=0.0, help="idle before timing each config (thermal state)")
    ap.add_argument("--timeout-ms", type=float, default=300000.0)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--backend", default="b200", help="stub: protocol/post-processing dry run without a GPU")
    a = ap.parse_args()
    {"run": cmd_run, "post": cmd_post}[a.cmd](a)


if __name__ == "__main__":
    main()
