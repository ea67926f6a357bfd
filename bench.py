#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json: "attn TFLOP/s (prefill) & KV GB/s (decode) per B200,
% roofline, 1/2/4/8 GPUs").

Headline (``--workload decode``, default): config C2 = Llama-3-8B paged-KV decode, batch 64,
context 4096, 32q/8kv heads, head_dim 128, block_size 16 (BASELINE.json configs[1]).  One step =
one decode pass over the batch; metric = KV bytes read / s (whole job, summed over ranks; weak
scaling: every rank decodes its own 64 sequences).  Inputs (1.07 GB of K+V) exceed the 126-MB L2,
so no flush is needed between steps.
``--workload prefill``: C3 (16-sequence varlen causal prefill) in TFLOP/s, weak.
``--workload c4``: C4 = Llama-3-70B-shaped decode (64q/8kv), batch 256, ctx 32k, STRONG scaling:
the 256 sequences are split over the ranks (parallel.shard_range), each rank holding only its
sequences' pages (34.4 GB of K+V in total; 4.3 GB per GPU at N = 8).

Multi-GPU: one process per GPU.  ``--gpus N`` without a torchrun environment
re-executes itself under ``torch.distributed.run`` with N ranks.  The path shards with no exchange
step, so the timed region has no collective: barrier + synchronize, K graph replays, synchronize +
barrier, time = MAX over ranks of the CUDA-event time.  After it, outputs are gathered to rank 0
over NCCL and a seeded subset is checked against the CPU oracle (the checker, never the measured
path) — for C4 (batch shards) and for C3 split by kv-head group (``extra.c3_heads_strong``), at
every N.

``--impl reference`` times the reference CPU path of the same workload on the host cores: the
reference (ref/pkg) contains no attention arithmetic (ref/SPEC.md:16), so the CPU path is the
oracle port — the PyTorch-native fp32 SDPA (oracle/torch_cpu.py, the paper's normalisation,
ref/PAPER.md:20-21) and the fp64 restatement (oracle/attn_oracle.c, OpenMP), all host cores; the
line reports the faster one.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))  # before ROOT: `oracle/` itself would import as a namespace package

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
PARITY_TOL = 1e-2  # max-abs error vs the fp64 oracle


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return FALLBACK_PEAKS, "fallback"


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- clocks (NVML)
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler(threading.Thread):
    def __init__(self, index: int, period_s: float = 0.005):
        super().__init__(daemon=True)
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], 0
        self.stop_evt = threading.Event()
        self.max_mhz = None
        self.ok = True
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.ok = False

    def run(self):
        if not self.ok:
            return
        nv = self.nv
        while not self.stop_evt.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        names = [n for bit, n in REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- ranks
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_respawn(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N ranks."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gpu = local
    if args.impl != "reference" and torch.cuda.is_available():
        n = torch.cuda.device_count()
        if local >= n:
            # testing the N>1 host path on a 1-GPU box (all ranks on one device, gloo for the plumbing)
            if not os.environ.get("B200_BENCH_ALLOW_SHARED_GPU"):
                raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {n} GPU(s) visible")
            gpu = local % n
        torch.cuda.set_device(gpu)
    if world > 1:
        import torch.distributed as dist

        backend = args.dist_backend
        if args.impl == "reference" or not torch.cuda.is_available():
            backend = "gloo"
        kw = {"device_id": torch.device("cuda", gpu)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    return world, rank, local, gpu


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float) -> float:
    from paper_2505_03780_b200.parallel import max_over_ranks as _max

    return _max(x)


# ----------------------------------------------------------------------------- timing helpers
def cuda_time(fn, reps: int, stream) -> float:
    import torch

    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(stream)
    for _ in range(reps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def capture(fn, n: int = 1):
    import torch

    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm (attributes, descriptor prefetch)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    return g


def timed_replays(g, steps, world, stream):
    """The contract's timed region: barrier + sync, `steps` replays, sync + barrier; max over ranks."""
    import torch

    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        g.replay()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = ev0.elapsed_time(ev1)
    return ms, max_over_ranks(ms)


def ncu_traffic(kernel: str):
    """dram bytes (read+write) per launch of `kernel` from the committed ncu summary, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def errs(out, ref):
    import numpy as np

    o = out.float().cpu().numpy() if hasattr(out, "cpu") else out
    d = np.abs(o - ref)
    return float(d.max()), float((d / np.maximum(np.abs(ref), 1.0)).max())


# ----------------------------------------------------------------------------- CPU reference paths
CPU_VARIANTS = {"torch_bf16_sdpa": "torch_bf16", "torch_fp32_sdpa": "torch", "fp64_oracle": "fp64"}


def cpu_fn(op: str, variant: str):
    """The CPU implementations timed as the reference path: the fp64 oracle (attn_oracle.c, OpenMP)
    and the PyTorch-native SDPA (oracle/torch_cpu.py) in fp32 or bf16, all host cores."""
    import torch

    import oracle
    import torch_cpu

    if variant == "fp64":
        return getattr(oracle, op)
    dt = torch.bfloat16 if variant == "torch_bf16" else torch.float32
    f = getattr(torch_cpu, op)
    return lambda *a: f(*a, dtype=dt)


def cpu_decode(d, target_s: float, variant: str):
    """CPU throughput on a bounded sample of the decode workload: the first n sequences of the same
    batch (their pages gathered into a compact pool), n calibrated to ~target_s, repeated to fill it."""
    import torch

    import oracle
    import torch_cpu

    threads = torch_cpu.set_threads()
    fn = cpu_fn("decode", variant)

    def sample(n):
        bt = d.block_table[:n]
        pages = bt.reshape(-1).long()
        kc = d.k_cache[pages.to(d.k_cache.device)].cpu()
        vc = d.v_cache[pages.to(d.v_cache.device)].cpu()
        nbt = torch.arange(pages.numel(), dtype=torch.int32).reshape(bt.shape)
        return d.q[:n].cpu(), kc, vc, nbt, d.seq_lens[:n].cpu()

    args = sample(1)
    fn(*args)  # warm (build + page in)
    t0 = time.perf_counter()
    fn(*args)
    t1 = time.perf_counter() - t0
    n = max(1, min(d.q.shape[0], int(target_s / max(t1, 1e-6))))
    args = sample(n)
    reps, t0 = 0, time.perf_counter()
    while True:
        fn(*args)
        reps += 1
        if time.perf_counter() - t0 >= min(target_s, 30.0) or reps >= 1000:
            break
    dt = (time.perf_counter() - t0) / reps
    Hkv, D = d.k_cache.shape[2], d.k_cache.shape[3]
    kv = 2 * sum(d.lens[:n]) * Hkv * D * 2
    cores = oracle.num_threads() if variant == "fp64" else threads
    return {"value": kv / dt / 1e9, "cores": cores, "n_seqs": n, "seconds": dt * reps, "kv_bytes": kv,
            "args": args}


def cpu_prefill_c1(variant: str, reps: int = 3):
    """C1 (b=1, s=512, 32q/8kv) IN FULL on the host cores (BASELINE.json configs[0]: "CPU reference
    runs this"): median of `reps` runs after one warm-up."""
    import oracle
    import torch_cpu
    from paper_2505_03780_b200 import workload as W

    threads = torch_cpu.set_threads()
    x = W.make_prefill(W.C1, device="cpu")
    f = cpu_fn("prefill", variant)
    fn = lambda: f(x.q, x.k, x.v, x.cu_seqlens)  # noqa: E731
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ms = statistics.median(ts) * 1e3
    return {"ms": ms, "TFLOP/s": x.flops / (ms / 1e3) / 1e12,
            "cores": oracle.num_threads() if variant == "fp64" else threads}


def cpu_prefill_sample(x, target_s: float, variant: str):
    """C3: the shortest sequences (all heads) until ~target_s of CPU work."""
    import itertools

    import torch

    import oracle
    import torch_cpu

    threads = torch_cpu.set_threads()
    fn = cpu_fn("prefill", variant)
    q, k, v = x.q.cpu(), x.k.cpu(), x.v.cpu()
    lens = x.lens
    order = sorted(range(len(lens)), key=lambda i: lens[i])
    cu = x.cu_seqlens.tolist()
    i0 = order[0]
    qq, kk, vv = (t[cu[i0]:cu[i0 + 1]].contiguous() for t in (q, k, v))
    c = torch.tensor([0, lens[i0]], dtype=torch.int32)
    fn(qq, kk, vv, c)
    t0 = time.perf_counter()
    fn(qq, kk, vv, c)
    per_pair = (time.perf_counter() - t0) / (lens[i0] * (lens[i0] + 1) / 2)
    chosen, cost = [], 0.0
    for i in order:
        pc = per_pair * lens[i] * (lens[i] + 1) / 2
        if chosen and cost + pc > target_s:
            break
        chosen.append(i)
        cost += pc
    qs = torch.cat([q[cu[i]:cu[i + 1]] for i in chosen])
    ks = torch.cat([k[cu[i]:cu[i + 1]] for i in chosen])
    vs = torch.cat([v[cu[i]:cu[i + 1]] for i in chosen])
    cus = torch.tensor([0] + list(itertools.accumulate(lens[i] for i in chosen)), dtype=torch.int32)
    t0 = time.perf_counter()
    fn(qs, ks, vs, cus)
    dt = time.perf_counter() - t0
    Hq, D = q.shape[1], q.shape[2]
    flops = 4 * D * Hq * sum(lens[i] * (lens[i] + 1) // 2 for i in chosen)
    return {"value": flops / dt / 1e12, "cores": oracle.num_threads() if variant == "fp64" else threads,
            "lens": [lens[i] for i in chosen], "seconds": dt}


def cpu_baseline_block(kind_workload, data, seconds):
    """Both CPU variants on the same bounded sample; the faster one is the baseline value."""
    variants = {}
    for var, code in CPU_VARIANTS.items():
        if kind_workload == "prefill":
            r = cpu_prefill_sample(data, seconds / 3, code)
            variants[var] = {"value": r["value"], "unit": "TFLOP/s", "cores": r["cores"],
                             "sample": f"C3 sequences of lengths {r['lens']} (all heads), {r['seconds']:.1f} s"}
        else:
            r = cpu_decode(data, seconds / 3, code)
            variants[var] = {"value": r["value"], "unit": "GB/s", "cores": r["cores"],
                             "sample": f"{r['n_seqs']} of {data.q.shape[0]} sequences (ctx {data.lens[0]}, all "
                                       f"heads; {r['kv_bytes'] / 1e6:.0f} MB K+V per pass), {r['seconds']:.1f} s"}
    best = max(variants, key=lambda k: variants[k]["value"])
    b = variants[best]
    out = {"value": b["value"], "unit": b["unit"], "cores": b["cores"], "kind": "port", "variant": best,
           "sample": b["sample"], "cpu_model": cpu_model(), "host_cores": os.cpu_count(), "variants": variants}
    try:
        out["c1_full"] = {v: cpu_prefill_c1(code) for v, code in CPU_VARIANTS.items()}
    except Exception as ex:  # pragma: no cover
        out["c1_full"] = {"error": str(ex)[:200]}
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    """CPU port on the host cores, same metric/config, bounded sample per step (rank 0 only)."""
    if rank != 0:
        return
    from paper_2505_03780_b200 import workload as W

    import oracle
    import torch_cpu

    torch_cpu.set_threads()
    if args.workload == "prefill":
        x = W.make_prefill(W.C3, device="cpu")
        probe = {v: cpu_prefill_sample(x, args.cpu_step_seconds, v)["value"] for v in CPU_VARIANTS.values()}
        var = max(probe, key=probe.get)
        vals, r = [], None
        for i in range(args.warmup + args.steps):
            r = cpu_prefill_sample(x, args.cpu_step_seconds, var)
            if i >= args.warmup:
                vals.append(r["value"])
        value, unit = statistics.median(vals), "TFLOP/s"
        sample = f"C3 sequences of lengths {r['lens']} (all heads) per step"
        config = {"workload": "C3 varlen causal prefill, 16 seqs 128..8192, 32q/8kv, d128", "global_batch": 16}
        cores = r["cores"]
    else:
        shape = W.C2 if args.workload == "decode" else dict(W.C4, batch_size=8)
        d = W.make_decode(shape, device="cpu")
        probe = {}
        for v in CPU_VARIANTS.values():
            probe[v] = cpu_decode(d, args.cpu_step_seconds, v)
        var = max(probe, key=lambda v: probe[v]["value"])
        sargs, kv = probe[var]["args"], probe[var]["kv_bytes"]
        fn = cpu_fn("decode", var)
        vals = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            fn(*sargs)
            t = time.perf_counter() - t0
            if i >= args.warmup:
                vals.append(kv / t / 1e9)
        value, unit = statistics.median(vals), "GB/s"
        n = probe[var]["n_seqs"]
        sample = f"{n} of {shape['batch_size']} sequences x {shape['seq_len']} ctx x 8 kv heads ({kv / 1e6:.1f} MB K+V) per step"
        config = ({"workload": "C2 paged-KV decode, batch 64, ctx 4096, 32q/8kv, d128, page 16", "global_batch": 64}
                  if args.workload == "decode" else
                  {"workload": "C4 paged-KV decode, 64q/8kv, ctx 32k, d128, page 16 (sequence sample)",
                   "global_batch": 256})
        cores = probe[var]["cores"]
        probe = {k: v["value"] for k, v in probe.items()}
    variant = {c: n for n, c in CPU_VARIANTS.items()}[var]
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "strong" if args.workload == "c4" else "weak", "vs_baseline": None,
            "dtype": {"torch_bf16": "bf16 SDPA (fp32 accumulate)", "torch": "bf16 in, fp32 SDPA",
                      "fp64": "bf16 in, fp64 accumulate"}[var],
            "data": "synthetic (seeded randn -> bf16)",
            "config": dict(config, parallelism="cpu",
                           note="reference has no CPU attention; CPU port timed: the fastest of torch SDPA "
                                "bf16 / fp32 (PyTorch-native, ref/PAPER.md:20-21) and the fp64 oracle"),
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "variant": variant,
                             "sample": sample, "cpu_model": cpu_model(), "probe_values": probe},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- validation (rank 0)
def validate_c4(shape, out_full, check_seqs, gen_device="cpu"):
    """rank 0: rebuild the checked sequences from their seeds (on the device type that generated
    the shards: CUDA and CPU generators differ) and compare with the fp64 oracle."""
    import torch

    import oracle
    from paper_2505_03780_b200 import workload as W

    worst_abs, worst_rel = 0.0, 0.0
    for b in check_seqs:
        q, k, v = (t.cpu() for t in W.decode_sequence(shape, b, device=gen_device))
        n, Hkv, D = k.shape
        bs = int(shape.get("block_size", 16))
        nb = (n + bs - 1) // bs
        pad = torch.zeros((nb * bs - n, Hkv, D), dtype=k.dtype)
        kc = torch.cat([k, pad]).view(nb, bs, Hkv, D)
        vc = torch.cat([v, pad]).view(nb, bs, Hkv, D)
        bt = torch.arange(nb, dtype=torch.int32)[None]
        ref = oracle.decode(q[None], kc, vc, bt, torch.tensor([n], dtype=torch.int32))
        a, r = errs(out_full[b:b + 1], ref)
        worst_abs, worst_rel = max(worst_abs, a), max(worst_rel, r)
    return {"checked_sequences": list(check_seqs), "max_abs": worst_abs, "max_rel": worst_rel,
            "tolerance_max_abs": PARITY_TOL, "pass": worst_abs <= PARITY_TOL}


def validate_c3_heads(shape, out_full_hTd, checks, gen_device="cpu"):
    """rank 0: out_full [Hq, T, D] gathered over head shards; checks = [(seq, kv_head)]."""
    import torch

    import oracle
    from paper_2505_03780_b200 import workload as W

    lens = W.varlen_lengths(shape)
    cu = [0]
    for L in lens:
        cu.append(cu[-1] + L)
    G = int(shape["num_q_heads"]) // int(shape["num_kv_heads"])
    worst_abs, worst_rel = 0.0, 0.0
    for s, kvh in checks:
        q, k, v = (t.cpu() for t in W.prefill_kv_head(shape, kvh, device=gen_device))
        a, b = cu[s], cu[s + 1]
        ref = oracle.prefill_blas(q[a:b], k[a:b], v[a:b], torch.tensor([0, b - a], dtype=torch.int32))
        got = out_full_hTd[kvh * G:(kvh + 1) * G, a:b].transpose(0, 1)
        ea, er = errs(got, ref)
        worst_abs, worst_rel = max(worst_abs, ea), max(worst_rel, er)
    return {"checked": [{"seq": s, "len": lens[s], "kv_head": h} for s, h in checks], "max_abs": worst_abs,
            "max_rel": worst_rel, "tolerance_max_abs": PARITY_TOL, "pass": worst_abs <= PARITY_TOL}


# ----------------------------------------------------------------------------- strong-scaled extras
def c4_strong(args, world, rank, dev, stream, steps, pk):
    """C4 split by batch over the ranks (each rank only its sequences' pages), timed, gathered,
    validated.  Returns (line-dict, plan, data) on every rank."""
    import torch

    from paper_2505_03780_b200 import attention as A
    from paper_2505_03780_b200 import parallel
    from paper_2505_03780_b200 import workload as W

    shape = dict(W.C4)
    total = int(shape["batch_size"])
    sh = parallel.shard_range(total, world, rank)
    d = W.make_decode_shard(shape, sh.start, sh.count, device=dev)
    plan = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len)
    g = capture(plan.run)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ms, ms_max = timed_replays(g, steps, world, stream)
    kv_total = 2 * total * int(shape["seq_len"]) * 8 * 128 * 2
    res = {"workload": "C4: 256 seqs x ctx 32768, 64q/8kv, d128, page 16; batch split over ranks "
                       "(each rank holds only its sequences' pages)",
           "scaling": "strong", "GB/s": kv_total / (ms_max / steps / 1e3) / 1e9, "ms_per_step": ms_max / steps,
           "per_rank_GB/s": d.kv_bytes / (ms / steps / 1e3) / 1e9, "seqs_per_rank": sh.count,
           "kv_bytes_per_rank": d.kv_bytes, "variant": plan.config}
    res["frac_of_measured_hbm_per_gpu"] = res["GB/s"] / world / pk["hbm_gbs"]
    counts = [parallel.shard_range(total, world, r).count for r in range(world)]
    out = plan.run()
    torch.cuda.synchronize()
    full = parallel.gather_to_rank0(out, counts)  # NCCL gather: validation only, outside the timed region
    if rank == 0 and not args.no_validate:
        res["validation"] = validate_c4(shape, full, (0, total // 2 + 1, total - 1), gen_device=dev)
    return res, plan, d


def c3_heads_strong(args, world, rank, dev, stream, steps, pk):
    """C3 prefill split by kv-head group (parallel.kv_head_groups): every group has identical
    causal cost, so balance is exact for any length mix."""
    import torch

    from paper_2505_03780_b200 import attention as A
    from paper_2505_03780_b200 import parallel
    from paper_2505_03780_b200 import workload as W

    shape = dict(W.C3)
    Hkv = int(shape["num_kv_heads"])
    heads = parallel.kv_head_groups(Hkv, world, rank)
    x = W.make_prefill_heads(shape, heads, device=dev)
    plan = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen)
    g = capture(plan.run, n=2)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    n = max(2, steps // 2)
    ms, ms_max = timed_replays(g, n, world, stream)
    per_launch = ms_max / (2 * n)
    Hq, D = int(shape["num_q_heads"]), 128
    flops_total = 4 * D * Hq * sum(L * (L + 1) // 2 for L in x.lens)
    res = {"workload": "C3 varlen causal prefill, 16 seqs 128..8192, 32q/8kv; kv-head groups split over ranks",
           "scaling": "strong", "TFLOP/s": flops_total / (per_launch / 1e3) / 1e12, "ms_per_step": per_launch,
           "per_rank_TFLOP/s": x.flops / (ms / (2 * n) / 1e3) / 1e12, "kv_heads": [heads.start, heads.stop],
           "variant": plan.config}
    res["frac_of_measured_peak_per_gpu"] = res["TFLOP/s"] / world / pk["bf16_tflops"]
    out = plan.run()
    torch.cuda.synchronize()
    counts = [len(parallel.kv_head_groups(Hkv, world, r)) * (Hq // Hkv) for r in range(world)]
    full = parallel.gather_to_rank0(out.transpose(0, 1).contiguous(), counts)  # [Hq, T, D] on rank 0
    if rank == 0 and not args.no_validate:
        res["validation"] = validate_c3_heads(shape, full, [(0, 0), (8, Hkv - 1), (15, 0)], gen_device=dev)
    del plan, x, g
    return res


# ----------------------------------------------------------------------------- e2e (public API, host buffers)
def e2e_decode(d, dev, world, stream, n_steps, chunks=0):
    """One serving step through the public API with HOST buffers, captured as ONE CUDA graph
    (attention.DecodeStep): H2D of q / new K,V / slots / seq_lens from a pinned buffer, cache_append,
    paged_decode, D2H of the output.  The block table stays resident (a serving loop updates one
    entry per sequence every block_size steps)."""
    import torch

    from paper_2505_03780_b200 import attention as A

    B, Hq, D = d.q.shape
    Hkv, bs = d.k_cache.shape[2], d.k_cache.shape[1]
    g = torch.Generator().manual_seed(7)
    new_k = torch.randn(B, Hkv, D, generator=g).bfloat16()
    new_v = torch.randn(B, Hkv, D, generator=g).bfloat16()
    bt_host = d.block_table.cpu()
    slots = torch.tensor([int(bt_host[b, (n - 1) // bs]) * bs + (n - 1) % bs for b, n in enumerate(d.lens)],
                         dtype=torch.int64)
    step = A.DecodeStep(d.k_cache, d.v_cache, d.block_table, batch=B, num_q_heads=Hq, max_seq_len=d.max_seq_len,
                        k_scale=d.k_scale, v_scale=d.v_scale, chunks=chunks)
    # the host-side inputs of a step live in the step's pinned staging buffer
    step.set_inputs(d.q.cpu(), new_k, new_v, slots, d.seq_lens.cpu())
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    e_ms = cuda_time(step, n_steps, stream)
    wall_ms = (time.perf_counter() - t0) * 1e3 / n_steps
    e_ms = max(e_ms, wall_ms)  # host-side API overhead counts too
    e_ms = max_over_ranks(e_ms)
    out = step.out_host.clone()
    return {"value": world * d.kv_bytes / (e_ms / 1e3) / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": step.h2d_bytes, "d2h_bytes_per_step": step.d2h_bytes, "ms_per_step": e_ms,
            "chunks": step.chunks,
            "zero_copy": step.zero_copy,
            "path": ("paper_2505_03780_b200.DecodeStep (public API, one CUDA graph): an ingest kernel reads the "
                     "step's q / seq_lens / new K,V / slots from pinned host memory over PCIe (q, seq_lens -> HBM; "
                     "K,V appended into their pages) -> paged_decode (K2' + K3') writing the output rows straight "
                     "into pinned host memory; paged KV pool and block table resident in HBM"
                     if step.zero_copy else
                     "paper_2505_03780_b200.DecodeStep (public API: one CUDA graph of H2D copy from pinned host "
                     "memory -> cache_append -> paged_decode -> D2H copy of the output, the batch in chunks whose "
                     "copies overlap the other chunks' kernels); paged KV pool and block table resident in HBM")}, out


# ----------------------------------------------------------------------------- the B200 arm
def run_b200(args, world, rank, local, gpu):
    import torch

    from paper_2505_03780_b200 import attention as A
    from paper_2505_03780_b200 import workload as W
    from paper_2505_03780_b200.parallel import weak_scaling_value

    dev = torch.device("cuda", gpu)
    pk, pk_kind = peaks()
    stream = torch.cuda.current_stream()
    extra = {}
    d = x = None

    # ------------------------------------------------------------------ headline workload
    if args.workload == "decode":
        d = W.make_decode(dict(W.C2, seed=rank), device=dev)
        plan = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len)
        units, alg_bytes, unit, scale, scaling = d.kv_bytes, d.total_bytes, "GB/s", 1e9, "weak"
        kernels_per_step = plan.kernels_per_run()
        config = {"workload": "C2 paged-KV decode (Llama-3-8B): batch 64/GPU, ctx 4096, 32q/8kv heads, d128, "
                              "page 16, permuted block table",
                  "global_batch": 64 * world, "seq_len": 4096, "parallelism": f"dp{world} (batch shards)",
                  "variant": plan.config, "num_splits": plan.num_splits,
                  "l2": "inputs > L2 (1.07 GB K+V per GPU); no flush"}
        g = capture(plan.run)
    elif args.workload == "c4":
        from paper_2505_03780_b200 import parallel

        sh = parallel.shard_range(256, world, rank)
        d = W.make_decode_shard(dict(W.C4), sh.start, sh.count, device=dev)
        plan = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len)
        units, alg_bytes, unit, scale, scaling = d.kv_bytes, d.total_bytes, "GB/s", 1e9, "strong"
        kernels_per_step = plan.kernels_per_run()
        config = {"workload": "C4 paged-KV decode (Llama-3-70B-shaped): 256 seqs x ctx 32768, 64q/8kv, d128, "
                              "page 16; batch split over ranks, each rank holding only its sequences' pages",
                  "global_batch": 256, "seq_len": 32768, "parallelism": f"dp{world} (batch shards, strong)",
                  "variant": plan.config, "l2": f"inputs > L2 ({d.kv_bytes / 1e9:.1f} GB K+V per GPU); no flush"}
        g = capture(plan.run)
    else:
        x = W.make_prefill(dict(W.C3, seed=rank), device=dev)
        plan = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen)
        units, unit, scale, scaling = x.flops, "TFLOP/s", 1e12, "weak"
        kernels_per_step = 1 if len(x.lens) == 1 else 2  # + the longest-first schedule kernel
        config = {"workload": "C3 varlen causal prefill (Llama-3-8B): 16 seqs 128..8192 (33430 tok), 32q/8kv, d128",
                  "global_batch": 16 * world, "seq_len": "128..8192", "parallelism": f"dp{world}",
                  "variant": plan.config, "l2": "q/k/v/o 410 MB > L2; no flush"}
        g = capture(plan.run)

    for _ in range(max(args.warmup, 3)):
        g.replay()
    torch.cuda.synchronize()
    barrier(world)

    # ------------------------------------------------------------------ timed region
    sampler = ClockSampler(gpu)
    sampler.start()
    time.sleep(0.02)
    ms, ms_max = timed_replays(g, args.steps, world, stream)
    sampler.stop_evt.set()
    sampler.join()
    if scaling == "weak":
        value = weak_scaling_value(units, args.steps, ms_max, world, scale)
    else:  # strong: the whole job's bytes over the slowest rank's time
        value = 2 * 256 * 32768 * 8 * 128 * 2 * args.steps / (ms_max / 1e3) / scale

    # ------------------------------------------------------------------ dominant kernel roofline
    if args.workload in ("decode", "c4"):
        gp = capture(plan.run_partial, n=20 if args.workload == "decode" else 4)
        gp.replay()
        nrep = 20 if args.workload == "decode" else 4
        k_ms = cuda_time(gp.replay, 10, stream) / nrep
        achieved = alg_bytes / (k_ms / 1e3) / 1e9
        peak = pk["hbm_gbs"]
        kname = "decode_flat_kernel" if int(plan.config["TILE_N"]) == 16 else "decode_split_kernel"
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": ncu_traffic(kname) if args.workload == "decode" else None,
                    "kernel": f"{kname} (K2')", "kernel_ms": k_ms,
                    "algorithmic_bytes_per_launch": alg_bytes, "peak_kind": pk_kind,
                    "frac_of_spec_8000": achieved / 8000.0,
                    "peak_note": "measured peak = torch copy (read+write) bandwidth; this kernel's stream is "
                                 "~99.9% reads, which run closer to the pins, hence frac can exceed 1"}
    else:
        k_ms = ms / args.steps
        achieved = units / (k_ms / 1e3) / 1e12
        peak = pk["bf16_tflops"]
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": ncu_traffic("prefill_fwd_kernel"),
                    "kernel": "prefill_fwd_kernel (K1)", "kernel_ms": k_ms, "algorithmic_flops_per_launch": units,
                    "peak_kind": pk_kind, "frac_of_sustained_peak": achieved / pk.get("bf16_tflops_sustained", peak),
                    "frac_of_spec_2250": achieved / 2250.0}

    # ------------------------------------------------------------------ e2e through the public API
    if d is not None:
        e2e, _ = e2e_decode(d, dev, world, stream, max(10, args.steps // 5) if args.workload == "decode" else 5,
                            chunks=args.e2e_chunks)
        if scaling == "strong":
            e2e["value"] = 2 * 256 * 32768 * 8 * 128 * 2 / (e2e["ms_per_step"] / 1e3) / 1e9
    else:
        step = A.PrefillStep(x.lens, x.q.shape[1], x.k.shape[1], x.q.shape[2], device=dev)
        step.set_inputs(x.q.cpu(), x.k.cpu(), x.v.cpu())
        step()
        torch.cuda.synchronize()
        n_e2e = max(5, args.steps // 10)
        e_ms = max_over_ranks(cuda_time(step, n_e2e, stream))
        e2e = {"value": world * units / (e_ms / 1e3) / 1e12, "unit": unit, "h2d_bytes_per_step": step.h2d_bytes,
               "d2h_bytes_per_step": step.d2h_bytes, "ms_per_step": e_ms, "chunks": step.chunks,
               "path": "paper_2505_03780_b200.PrefillStep (public API: one CUDA graph; the varlen batch in groups of "
                       "sequences, heaviest group first, whose H2D of q/k/v/cu_seqlens from pinned memory, prefill and "
                       "D2H of the output overlap across groups on two copy streams)"}
    del g

    # ------------------------------------------------------------------ strong-scaled, validated extras (any N)
    if not args.no_extra:
        del plan
        if args.workload != "c4":
            d = None
        torch.cuda.empty_cache()
        try:
            if args.workload != "c4":
                extra["c4_strong"], p4, d4 = c4_strong(args, world, rank, dev, stream, 5, pk)
                del p4, d4
                torch.cuda.empty_cache()
            extra["c3_heads_strong"] = c3_heads_strong(args, world, rank, dev, stream, 10, pk)
            torch.cuda.empty_cache()
        except torch.cuda.OutOfMemoryError as ex:  # pragma: no cover
            extra["strong_error"] = str(ex)[:200]

    # ------------------------------------------------------------------ single-GPU secondary configs
    if not args.no_extra and world == 1:
        for name, shp in (("prefill_C3", W.C3), ("prefill_C1", W.C1)):
            xx = W.make_prefill(dict(shp, seed=rank), device=dev)
            pp = A.PrefillPlan(xx.q, xx.k, xx.v, xx.cu_seqlens, xx.max_seqlen)
            n = 20 if name == "prefill_C1" else 10
            gg = capture(pp.run, n=n)
            gg.replay()
            t = cuda_time(gg.replay, 5, stream) / n
            g1 = capture(pp.run)
            single = [cuda_time(g1.replay, 1, stream) for _ in range(10)]
            tf = xx.flops / (t / 1e3) / 1e12
            extra[name] = {"TFLOP/s": tf, "ms": t, "frac_of_measured_peak": tf / pk["bf16_tflops"],
                           "frac_of_spec_2250": tf / 2250.0, "single_launch_median_ms": statistics.median(single),
                           "variant": pp.config}
            del xx, pp, gg, g1
        if args.workload == "decode":
            extra["decode_C2"] = {"frac_of_spec_8000": (units / (ms / args.steps / 1e3) / 1e9) / 8000.0}
        try:  # C4 geometry, one GPU's shard of the 8-GPU config (32 of 256 sequences)
            d4 = W.make_decode(dict(W.C4, batch_size=32, seed=rank), device=dev)
            p4 = A.DecodePlan(d4.q, d4.k_cache, d4.v_cache, d4.block_table, d4.seq_lens, max_seq_len=d4.max_seq_len)
            g4 = capture(p4.run)
            g4.replay()
            t4 = cuda_time(g4.replay, 10, stream)
            extra["decode_C4_shard_of_8"] = {"GB/s": d4.kv_bytes / (t4 / 1e3) / 1e9, "ms": t4,
                                             "frac_of_measured_hbm": d4.kv_bytes / (t4 / 1e3) / 1e9 / pk["hbm_gbs"],
                                             "variant": p4.config, "num_splits": p4.num_splits}
            del d4, p4, g4
        except Exception as ex:  # pragma: no cover
            extra["decode_C4_shard_of_8"] = {"error": str(ex)[:200]}
        try:  # C2 with an fp8 (e4m3) KV cache: same tokens, half the bytes
            d8 = W.make_decode(dict(W.C2, seed=rank, kv_dtype="fp8_e4m3"), device=dev)
            p8 = A.DecodePlan(d8.q, d8.k_cache, d8.v_cache, d8.block_table, d8.seq_lens, max_seq_len=d8.max_seq_len,
                              k_scale=d8.k_scale, v_scale=d8.v_scale)
            g8 = capture(p8.run, n=10)
            g8.replay()
            t8 = cuda_time(g8.replay, 10, stream) / 10
            extra["decode_C2_fp8_kv"] = {"GB/s": d8.total_bytes / (t8 / 1e3) / 1e9, "ms": t8,
                                         "frac_of_measured_hbm": d8.total_bytes / (t8 / 1e3) / 1e9 / pk["hbm_gbs"],
                                         "kv_bytes": d8.kv_bytes,
                                         # against this run's bf16 C2 step (only the decode workload has one)
                                         "speedup_vs_bf16_kv": ((ms / args.steps) / t8
                                                                if args.workload == "decode" else None),
                                         "variant": p8.config}
            del d8, p8, g8
        except Exception as ex:  # pragma: no cover
            extra["decode_C2_fp8_kv"] = {"error": str(ex)[:200]}

    # ------------------------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.workload == "prefill":
            cpu = cpu_baseline_block("prefill", x, args.cpu_seconds)
        else:
            dd = d if d is not None else W.make_decode(dict(W.C2, seed=rank), device=dev)
            cpu = cpu_baseline_block("decode", dd, args.cpu_seconds)

    if rank == 0:
        n_launch = args.steps * kernels_per_step
        line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded randn -> bf16)",
                "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": n_launch, "clocks": sampler.summary(), "impl": "b200",
                "dist": {"world": world, "backend": args.dist_backend if world > 1 else None,
                         "ms_per_rank_max": ms_max / args.steps}}
        if extra:
            line["extra"] = extra
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=["decode", "prefill", "c4"], default="decode")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-validate", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0, help="DecodeStep chunks (0 = auto)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample size (seconds)")
    ap.add_argument("--cpu-step-seconds", type=float, default=0.2, help="reference arm: seconds per step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    maybe_respawn(args)
    world, rank, local, gpu = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_b200(args, world, rank, local, gpu)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
