#!/usr/bin/env python
"""Device-time probes of the kernels (one tool instead of round 1's per-experiment scripts).

  perf.py time    --op prefill|decode --shapes C1,C3,1x16k --cfg '{json}' | --all-variants [--reps N]
      graph-replayed per-launch time (N launches per replay) and TFLOP/s or GB/s
  perf.py single  --op prefill --shapes C3  -- one launch per event pair after an idle gap (cold clocks)
  perf.py prof    --op prefill|decode|c1 [--cfg json] [--n 3]   -- small driver for ncu / sanitizers
  perf.py trace   [BLOCK_M num_stages num_warps]                 -- clock64 trace (needs a -DB200_TRACE build)
  perf.py umma-rate                                              -- tcgen05 MMA issue-rate probe
  perf.py e2e                                                    -- e2e decode step breakdown (C2)
  perf.py dtrace --shapes d64x512                                -- K2' per-CTA timeline (trace build)
"""

from __future__ import annotations

import argparse
import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2505_03780_b200 import _native  # noqa: E402
from paper_2505_03780_b200 import attention as A  # noqa: E402
from paper_2505_03780_b200 import workload as W  # noqa: E402

SHAPES = {
    "C1": ("prefill", W.C1), "C3": ("prefill", W.C3), "1x16k": ("prefill", dict(W.C1, seq_len=16384)),
    "4x8k": ("prefill", dict(W.C1, batch_size=4, seq_len=8192)),
    "16x8k": ("prefill", dict(W.C1, batch_size=16, seq_len=8192)), "1x32k": ("prefill", dict(W.C1, seq_len=32768)),
    "16x2k": ("prefill", dict(W.C1, batch_size=16, seq_len=2048)),
    "4x128": ("prefill", dict(W.C1, batch_size=4, seq_len=128)), "16x128": ("prefill", dict(W.C1, batch_size=16, seq_len=128)),
    "4x512": ("prefill", dict(W.C1, batch_size=4, seq_len=512)), "64x512": ("prefill", dict(W.C1, batch_size=64, seq_len=512)),
    "C2": ("decode", W.C2), "C4shard": ("decode", dict(W.C4, batch_size=32)),
    "C2fp8": ("decode", dict(W.C2, kv_dtype="fp8_e4m3")), "b1x32k": ("decode", dict(W.C2, batch_size=1, seq_len=32768)),
    # kv-head shards (one GPU's share when the kv heads are split): C2 over 4 / 8 GPUs, C4 over 8
    "C2kv2": ("decode", dict(W.C2, num_q_heads=8, num_kv_heads=2)),
    "C2kv1": ("decode", dict(W.C2, num_q_heads=4, num_kv_heads=1)),
    "C4kv1": ("decode", dict(W.C4, num_q_heads=8, num_kv_heads=1)),
    "C4kv4": ("decode", dict(W.C4, batch_size=64, num_q_heads=32, num_kv_heads=4)),
    "b4096": ("decode", dict(W.C2, batch_size=4096, seq_len=256)),
    # small, latency-bound decode shapes of the C5 grid
    "d1x8k": ("decode", dict(W.C2, batch_size=1, seq_len=8192)), "d16x512": ("decode", dict(W.C2, batch_size=16, seq_len=512)),
    "d4x2k": ("decode", dict(W.C2, batch_size=4, seq_len=2048)), "d1x512": ("decode", dict(W.C2, batch_size=1, seq_len=512)),
    "d64x512": ("decode", dict(W.C2, batch_size=64, seq_len=512)),
    "d1x2k": ("decode", dict(W.C2, batch_size=1, seq_len=2048)), "d4x512": ("decode", dict(W.C2, batch_size=4, seq_len=512)),
    "d16x2k": ("decode", dict(W.C2, batch_size=16, seq_len=2048)), "d1x128": ("decode", dict(W.C2, batch_size=1, seq_len=128)),
    "d16x128": ("decode", dict(W.C2, batch_size=16, seq_len=128)),
}


def make_plan(op, shape, cfg):
    if op == "prefill":
        x = W.make_prefill(shape, device="cuda")
        return A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg), x.flops, 1e12, "TFLOP/s"
    d = W.make_decode(shape, device="cuda")
    p = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len, config=cfg,
                     k_scale=d.k_scale, v_scale=d.v_scale)
    return p, d.total_bytes, 1e9, "GB/s"


def graph_ms(fn, reps):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) / reps)
    return statistics.median(out)


def all_prefill_variants():
    for bm in (256, 128):
        for bn in (128, 64):
            for ns in (1, 2, 3, 4):
                yield dict(BLOCK_M=bm, BLOCK_N=bn, num_warps=4, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
        for ns in (1, 2):
            yield dict(BLOCK_M=bm, BLOCK_N=128, num_warps=8, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)


def cmd_time(a):
    for name in a.shapes.split(","):
        op, shape = SHAPES[name]
        cfgs = [json.loads(a.cfg) if a.cfg else None]
        if a.all_variants and op == "prefill":
            cfgs = list(all_prefill_variants())
        for cfg in cfgs:
            try:
                p, work, sc, unit = make_plan(op, shape, cfg)
                reps = a.reps or (200 if name == "C1" else 10)
                ms = graph_ms(p.run_partial if a.partial else p.run, reps)
                print(json.dumps({"tag": a.tag, "shape": name, "cfg": p.config, "us": ms * 1e3,
                                  unit: work / (ms / 1e3) / sc}), flush=True)
                del p
            except Exception as ex:
                print(json.dumps({"tag": a.tag, "shape": name, "cfg": cfg, "error": str(ex)[:200]}), flush=True)
            torch.cuda.empty_cache()


def cmd_single(a):
    """single launches separated by idle gaps (what a protocol-median evaluation sees) vs back-to-back."""
    for name in a.shapes.split(","):
        op, shape = SHAPES[name]
        p, work, sc, unit = make_plan(op, shape, json.loads(a.cfg) if a.cfg else None)
        p.run()
        torch.cuda.synchronize()
        res = {}
        for gap in (0.0, 0.002, 0.05):
            ts = []
            for _ in range(10):
                if gap:
                    time.sleep(gap)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                p.run()
                e.record()
                torch.cuda.synchronize()
                ts.append(s.elapsed_time(e))
            res[f"gap_{gap}s_us"] = statistics.median(ts) * 1e3
        res["graph_amortised_us"] = graph_ms(p.run, 10) * 1e3
        print(json.dumps({"tag": a.tag, "shape": name, **res}), flush=True)


def cmd_prof(a):
    cfg = json.loads(a.cfg) if a.cfg else None
    op, shape = {"decode": SHAPES["C2"], "prefill": SHAPES["C3"], "c1": SHAPES["C1"]}.get(a.op, SHAPES.get(a.op))
    p, *_ = make_plan(op, shape, cfg)
    for _ in range(a.n):
        p.run()
    torch.cuda.synchronize()
    print("done")


def cmd_trace(a):
    lib = _native.load()
    cfg = None
    if len(a.args) >= 3:
        bm, ns, nw = map(int, a.args[:3])
        cfg = dict(BLOCK_M=bm, BLOCK_N=128, num_warps=nw, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
    import numpy as np

    x = W.make_prefill(dict(W.C1, batch_size=4, seq_len=8192), device="cuda")
    p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
    for _ in range(3):
        p.run()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (16 * 512))()
    lib.b200attn_debug_trace(buf, 16 * 512)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(16, 512).astype(np.int64)
    rows = [np.concatenate([t[:, j] - t[0, j], [t[0, j] - t[0, j - 1]]]) for j in range(1, 40)]
    print("config", cfg)
    print("median cycles rel. to S0 of each step:", " ".join(f"{v:.0f}" for v in np.median(np.array(rows[5:]), 0)))


def cmd_c1trace(a):
    """CTA 0's first-item timeline on C1 (trace library): clock64 cycles from CTA entry to barriers
    ready, past griddepcontrol.wait, Q seen by the MMA warp, first S, each step's S, epilogue, exit;
    plus the host-side per-call time of a single launch."""
    import numpy as np

    lib = _native.load()
    cfg = json.loads(a.cfg) if a.cfg else None
    x = W.make_prefill(W.C1, device="cuda")
    p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
    for _ in range(5):
        p.run()
        torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (17 * 512))()
    lib.b200attn_debug_trace(buf, 17 * 512)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(17, 512).astype(np.int64)
    e = t[16, :8] - t[16, 0]
    names = ["entry", "ready", "griddep", "q_seen", "first_S", "epi_start", "epi_done", "exit"]
    steps = [int(t[0, j] - t[16, 0]) for j in range(8) if t[0, j] > 0]
    print(json.dumps({"tag": a.tag, "cfg": p.config, **{n: int(v) for n, v in zip(names, e)}, "S_steps": steps}), flush=True)


def cmd_ptrace(a):
    """K1 per-CTA %globaltimer stamps (trace library) of the last two of N graph-replayed launches:
    kernel span, the gap between consecutive launches, and the spread of CTA entry / finish."""
    import numpy as np

    lib = _native.load()
    lib.b200attn_debug_ptrace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    cfg = json.loads(a.cfg) if a.cfg else None
    for name in a.shapes.split(","):
        x = W.make_prefill(SHAPES[name][1], device="cuda")
        p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
        p.run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(4):
                p.run()
        g.replay()
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (2 * 1024 * 8))()
        cnt = ctypes.c_uint(0)
        assert lib.b200attn_debug_ptrace(buf, 2 * 1024 * 8, ctypes.byref(cnt)) == 0
        t6 = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 8).astype(np.int64)
        t = t6[:, :, :4]
        last, prev = (cnt.value - 1) & 1, (cnt.value - 2) & 1
        res = {"tag": a.tag, "shape": name, "cfg": p.config}
        base = None
        for lbl, par in (("prev", prev), ("last", last)):
            tt = t[par]
            tt = tt[tt[:, 0] > 0]
            if base is None:
                base = tt[:, 0].min()
            r = (tt - base) / 1e3
            res[lbl] = {"ctas": int(len(tt)), "entry": [round(float(r[:, 0].min()), 2), round(float(r[:, 0].max()), 2)],
                        "griddep_max": round(float(r[:, 1].max()), 2), "done": [round(float(r[:, 2].min()), 2),
                        round(float(np.median(r[:, 2])), 2), round(float(r[:, 2].max()), 2)],
                        "exit_max": round(float(r[:, 3].max()), 2)}
        cl = t6[prev][t6[prev][:, 0] > 0]
        if a.per_cta:  # prev launch: per CTA [first item, entry, first-item epilogue done, done] (us)
            b0 = cl[:, 0].min()
            res["per_cta"] = sorted([[int(r[6]), round((r[0] - b0) / 1e3, 2), round((r[7] - b0) / 1e3, 2) if r[7] > r[0] else None,
                                      round((r[2] - b0) / 1e3, 2)] for r in cl], key=lambda v: v[3])
        res["sm_mhz_median"] = round(float(np.median((cl[:, 5] - cl[:, 4]) / np.maximum(cl[:, 3] - cl[:, 0], 1) * 1e3)), 1)
        res["gap_us"] = round(res["last"]["entry"][0] - res["prev"]["exit_max"], 2)
        res["span_us"] = round(res["last"]["exit_max"] - res["last"]["entry"][0], 2)
        print(json.dumps(res), flush=True)


def cmd_umma_rate(a):
    lib = _native.load()
    out = torch.zeros(148, dtype=torch.int64, device="cuda")
    modes = [(0, "SS N128 B-K (QK)", 128), (1, "TS N128 B-MN (PV, P in TMEM)", 128), (2, "SS N128 B-MN", 128),
             (3, "SS N256 B-K", 256), (4, "TS N128 B-K", 128), (5, "SS N64 B-K", 64), (6, "SS N256 B-MN", 256),
             (7, "TS N64 B-MN", 64), (8, "SS N128 B-K + 4 LDTM/STTM warps", 128),
             (9, "TS N128 B-MN + 4 LDTM/STTM warps", 128), (10, "SS N128 B-K + 8 LDTM/STTM warps", 128)]
    for mode, name, N in modes:
        rc = lib.b200attn_debug_umma_rate(mode, 4000, 148, ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert rc == 0, lib.b200attn_last_error()
        cyc = out.float().mean().item()
        ideal = N * 128 / 256 * 8
        print(f"{name:34s}: {cyc:7.1f} cycles / 8 MMAs (floor {ideal:.0f}) -> {ideal / cyc * 100:.0f}% of floor")


def cmd_dtrace(a):
    """K2' per-CTA timeline (needs the -DB200_TRACE library: B200ATTN_LIB=.../libb200attn_trace.so):
    %globaltimer stamps per CTA -> per event the min / median / max offset from the earliest entry."""
    import numpy as np

    lib = _native.load()
    lib.b200attn_debug_dtrace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    names = ["entry", "scan", "first_S", "last_P", "out_written", "merged", "exit", "arrived"]
    for name in a.shapes.split(","):
        op, shape = SHAPES[name]
        p, *_ = make_plan(op, shape, json.loads(a.cfg) if a.cfg else None)
        for _ in range(5):
            p.run()
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (1024 * 8))()
        rc = lib.b200attn_debug_dtrace(buf, 1024 * 8)  # [1024 CTAs][8 events]
        assert rc == 0, f"b200attn_debug_dtrace: cuda error {rc} (is B200ATTN_LIB the trace build?)"
        t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
        n = int(p.num_splits) if p.config.get("TILE_N") == 16 else 0
        t = t[:n] if n else t[:148]
        smid = np.full(len(t), -1)
        t0 = t[:, 0][t[:, 0] > 0].min()
        rel = (t - t0) / 1e3  # us
        out = {"tag": a.tag, "shape": name, "cfg": p.config, "ctas": int(len(t))}
        for k, nm in enumerate(names):
            col = rel[:, k]
            col = col[(t[:, k] > 0)]
            if len(col):
                out[nm] = [round(float(col.min()), 2), round(float(np.median(col)), 2), round(float(col.max()), 2)]
        if a.per_cta:  # per CTA: sm id, first S and last P (us from the earliest entry)
            out["per_cta"] = [[int(smid[i]), round(float(rel[i, 2]), 2), round(float(rel[i, 3]), 2)] for i in range(len(t))]
        print(json.dumps(out), flush=True)


def cmd_e2e(a):
    """Where the e2e decode step's time goes (C2): device-only plan, the copies alone, append alone,
    and attention.DecodeStep (one graph: H2D -> append -> decode -> D2H) at several chunk counts."""
    d = W.make_decode(W.C2, device="cuda")
    B, Hq, D = d.q.shape
    Hkv, bs = d.k_cache.shape[2], d.k_cache.shape[1]
    st = torch.cuda.current_stream()

    def ev_time(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record(st)
        for _ in range(n):
            fn()
        e.record(st)
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e3 / n, (time.perf_counter() - t0) * 1e6 / n

    res = {}
    plan = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len)
    res["decode_graph_us"] = graph_ms(plan.run, 20) * 1e3
    nk = torch.randn(B, Hkv, D, device="cuda").bfloat16()
    slots = torch.full((B,), -1, dtype=torch.int64, device="cuda")
    res["append_graph_us"] = graph_ms(lambda: A.cache_append(nk, nk, d.k_cache, d.v_cache, slots), 20) * 1e3
    for nbytes, name in ((787200, "h2d_787KB"), (524288, "d2h_512KB")):
        h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        dd = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        f = (lambda: dd.copy_(h, non_blocking=True)) if name.startswith("h2d") else (lambda: h.copy_(dd, non_blocking=True))
        res[name + "_us"] = ev_time(f)[0]
    slots_h = torch.full((B,), -1, dtype=torch.int64)
    for chunks, zc in ((1, True), (1, False), (2, False), (4, False)):
        step = A.DecodeStep(d.k_cache, d.v_cache, d.block_table, batch=B, num_q_heads=Hq, max_seq_len=d.max_seq_len,
                            chunks=chunks, zero_copy=zc)
        step.set_inputs(d.q.cpu(), nk.cpu(), nk.cpu(), slots_h, d.seq_lens.cpu())
        dev_us, wall_us = ev_time(step)
        tag = f"step_chunks{chunks}" + ("_zerocopy" if zc else "")
        res[f"{tag}_us"] = dev_us
        res[f"{tag}_wall_us"] = wall_us
        del step
    print(json.dumps({"tag": a.tag, **{k: round(v, 2) for k, v in res.items()}}), flush=True)


def cmd_pfe2e(a):
    """Where the prefill e2e step's time goes (C3): the PCIe copies alone (H2D of q/k/v, D2H of the
    output, and both directions at once) against attention.PrefillStep at several group counts."""
    x = W.make_prefill(W.C3, device="cpu")
    st = torch.cuda.current_stream()

    def ev_time(fn, n=5):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(n):
            fn()
        e.record(st)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n

    res = {}
    nin = (x.q.numel() + x.k.numel() + x.v.numel()) * 2
    nout = x.q.numel() * 2
    hi = torch.empty(nin, dtype=torch.uint8).pin_memory()
    di = torch.empty(nin, dtype=torch.uint8, device="cuda")
    ho = torch.empty(nout, dtype=torch.uint8).pin_memory()
    do = torch.empty(nout, dtype=torch.uint8, device="cuda")
    res["h2d_ms"] = ev_time(lambda: di.copy_(hi, non_blocking=True))
    res["d2h_ms"] = ev_time(lambda: ho.copy_(do, non_blocking=True))
    s2 = torch.cuda.Stream()

    def both():
        s2.wait_stream(st)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
        di.copy_(hi, non_blocking=True)
        st.wait_stream(s2)
    res["both_ms"] = ev_time(both)
    res["h2d_GBps"] = nin / res["h2d_ms"] / 1e6
    res["d2h_GBps"] = nout / res["d2h_ms"] / 1e6
    del hi, di, ho, do
    for chunks in (2, 4, 8, 16):
        step = A.PrefillStep(x.lens, x.q.shape[1], x.k.shape[1], x.q.shape[2], chunks=chunks)
        step.set_inputs(x.q, x.k, x.v)
        res[f"step_chunks{chunks}_ms"] = ev_time(step)
        del step
        torch.cuda.empty_cache()
    print(json.dumps({"tag": a.tag, **{k: round(v, 3) for k, v in res.items()}}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["time", "single", "prof", "trace", "umma-rate", "e2e", "dtrace", "c1trace", "ptrace",
                                    "pfe2e"])
    ap.add_argument("args", nargs="*")
    ap.add_argument("--op", default="prefill")
    ap.add_argument("--shapes", default="C3")
    ap.add_argument("--cfg", default=None)
    ap.add_argument("--all-variants", action="store_true")
    ap.add_argument("--reps", type=int, default=0)
    ap.add_argument("--partial", action="store_true", help="decode: time K2 / K2' alone (no combine)")
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--tag", default="")
    ap.add_argument("--per-cta", action="store_true", help="dtrace: per-CTA sm id / first S / last P")
    a = ap.parse_args()
    {"time": cmd_time, "single": cmd_single, "prof": cmd_prof, "trace": cmd_trace, "umma-rate": cmd_umma_rate, "e2e": cmd_e2e, "pfe2e": cmd_pfe2e, "dtrace": cmd_dtrace,
     "c1trace": cmd_c1trace, "ptrace": cmd_ptrace}[a.cmd](a)


if __name__ == "__main__":
    main()
