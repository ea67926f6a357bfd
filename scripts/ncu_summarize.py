"""Summarise ncu captures into profiles/ (run here, no GPU needed).

usage: ncu_summarize.py full <rep.ncu-rep> <kernel-key> <algorithmic-bytes-or-flops> <bytes|flops>
       ncu_summarize.py launches <launches.csv>
Writes/updates profiles/ncu_summary.json and prints a markdown block.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles" / "ncu_summary.json"
WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    # tensor pipe busy cycles as a share of the SM's active cycles (the one tensor-pipe figure quoted)
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "mufu_pipe_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "smsp__cycles_active.avg": "smsp_cycles_active",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "%": 1, "": 1,
         "register/thread": 1, "cycle": 1, "warp": 1}


def raw_rows(rep):
    """rows of `ncu -i REP --page raw --csv`, or of that export itself when REP is a .csv"""
    if str(rep).endswith(".csv"):
        txt = Path(rep).read_text()
    else:
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def full(rep, key, work, kind):
    head, units, data = raw_rows(rep)
    ik = head.index("Kernel Name")
    out = []
    for r in data:
        m = {"kernel_name": r[ik]}
        for i, n in enumerate(head):
            if n in WANT:
                try:
                    m[WANT[n]] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
        out.append(m)
    m = out[0]
    dram = m.get("dram_read", 0) + m.get("dram_write", 0)
    rec = {"source": str(rep), "kernel_name": m["kernel_name"][:160], "duration_s": m.get("duration"),
           "dram_bytes_per_launch": dram, "dram_read": m.get("dram_read"), "dram_write": m.get("dram_write"),
           "dram_pct_of_peak": m.get("dram_pct_of_peak"), "tensor_pipe_pct": m.get("tensor_pipe_pct"),
           "sm_throughput_pct": m.get("sm_throughput_pct"), "mufu_pipe_pct": m.get("mufu_pipe_pct"),
           "l2_hit_pct": m.get("l2_hit_pct"), "registers": m.get("registers"), "grid": m.get("grid"),
           "block": m.get("block"), "l2_bytes": m.get("l2_bytes"), "sm_clock_hz": m.get("sm_hz"),
           "note": "ncu --set full --clock-control none (serialised, cold-cache replay)"}
    work = float(work)
    if kind == "bytes":
        rec["algorithmic_bytes"] = work
        rec["traffic_over_algorithmic"] = dram / work if work else None
        rec["achieved_GBps_under_ncu"] = work / m["duration"] / 1e9 if m.get("duration") else None
    else:
        rec["algorithmic_flops"] = work
        rec["achieved_TFLOPs_under_ncu"] = work / m["duration"] / 1e12 if m.get("duration") else None
    doc = json.loads(OUT.read_text()) if OUT.exists() else {}
    doc[key] = rec
    OUT.parent.mkdir(exist_ok=True)
    OUT.write_text(json.dumps(doc, indent=1))
    print(json.dumps(rec, indent=1))


def launches(path):
    lines = Path(path).read_text().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1)
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    print("| kernel | launches | total ms | mean us | share |\n|---|---|---|---|---|")
    res = {}
    for n, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{n[:70]}` | {cnt[n]} | {t * 1e3:.3f} | {t / cnt[n] * 1e6:.1f} | {t / allt * 100:.1f}% |")
        res[n] = {"launches": cnt[n], "total_s": t, "share": t / allt}
    return res


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:6])
    else:
        launches(sys.argv[2])
