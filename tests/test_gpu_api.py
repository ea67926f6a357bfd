"""GPU tests of the public API's host-side contract: cross-shape validation, per-stream workspaces
(reentrancy), the one-graph serving step, and the multi-rank bench path (2 ranks: NCCL on two GPUs,
or gloo with both ranks on one GPU when only one is visible)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2505_03780_b200 import attention as A
from paper_2505_03780_b200 import workload as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
DEV = "cuda"


def test_decode_rejects_mismatched_shapes():
    d = W.make_decode(dict(W.C2, batch_size=4, seq_len=64), device=DEV)
    with pytest.raises(ValueError, match="batch mismatch"):
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table[:3], d.seq_lens)
    with pytest.raises(ValueError, match="batch mismatch"):
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens[:2])
    with pytest.raises(ValueError, match="out"):
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, out=torch.empty_like(d.q[:2]))
    with pytest.raises(ValueError, match="head_dim"):
        A.paged_decode(d.q[..., :64].contiguous(), d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    with pytest.raises(ValueError, match="multiple"):
        A.paged_decode(d.q[:, :12].contiguous(), d.k_cache, d.v_cache, d.block_table, d.seq_lens)


def test_prefill_and_append_reject_mismatched_shapes():
    x = W.make_prefill(dict(W.C1, seq_len=64), device=DEV)
    with pytest.raises(ValueError):
        A.prefill_varlen(x.q, x.k[:10], x.v[:10], x.cu_seqlens, 64)
    with pytest.raises(ValueError, match="out"):
        A.prefill_varlen(x.q, x.k, x.v, x.cu_seqlens, 64, out=torch.empty_like(x.q[:5]))
    kc = torch.zeros(4, 16, 8, 128, dtype=torch.bfloat16, device=DEV)
    nk = torch.zeros(3, 8, 128, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(ValueError, match="slot_mapping"):
        A.cache_append(nk, nk, kc, kc.clone(), torch.zeros(2, dtype=torch.int64, device=DEV))
    with pytest.raises(ValueError, match="new_k"):
        A.cache_append(nk[:, :4].contiguous(), nk[:, :4].contiguous(), kc, kc.clone(),
                       torch.zeros(3, dtype=torch.int64, device=DEV))


def test_two_streams_in_flight_do_not_share_workspace():
    """Prefill and decode launched concurrently on two streams (the header's reentrancy promise):
    each stream gets its own workspace, so the self-resetting prefill counter and the decode
    partials never collide — outputs equal the single-stream results exactly."""
    xs = [W.make_prefill(dict(W.C3, batch_size=6, seq_len_min=100, seq_len_max=3000, seed=s), device=DEV)
          for s in (1, 2)]
    ds = [W.make_decode(dict(W.C2, batch_size=48, seq_len=2000, seed=s), device=DEV) for s in (3, 4)]
    ref_p = [A.prefill_varlen(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen).clone() for x in xs]
    ref_d = [A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens).clone() for d in ds]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(5):
        outs_p, outs_d = [None, None], [None, None]
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                outs_p[i] = A.prefill_varlen(xs[i].q, xs[i].k, xs[i].v, xs[i].cu_seqlens, xs[i].max_seqlen)
                outs_d[i] = A.paged_decode(ds[i].q, ds[i].k_cache, ds[i].v_cache, ds[i].block_table, ds[i].seq_lens)
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(outs_p[i], ref_p[i])
            assert torch.equal(outs_d[i], ref_d[i])


@pytest.mark.parametrize("chunks,zero_copy", [(1, True), (1, False), (2, False), (3, False)])
def test_decode_step_graph_matches_eager_api(chunks, zero_copy):
    """DecodeStep (H2D -> cache_append -> paged_decode -> D2H in one CUDA graph, the batch in
    chunks overlapping copies and kernels): the cache pages it writes equal the eager cache_append's
    bit for bit, its output matches the oracle, and with one chunk it equals the eager paged_decode
    bit for bit (chunks change the flat partition's split points, hence fp32 summation order)."""
    lens = [700, 33, 4096, 1, 250, 3000]
    B = len(lens)
    d = W.make_decode(dict(W.C2, batch_size=B, seq_len=4096), device=DEV, lens=lens, extra_blocks=2)
    k2, v2 = d.k_cache.clone(), d.v_cache.clone()
    step = A.DecodeStep(d.k_cache, d.v_cache, d.block_table, batch=B, num_q_heads=32, chunks=chunks,
                        zero_copy=zero_copy)
    assert step.chunks == chunks and step.zero_copy == zero_copy
    g = torch.Generator().manual_seed(1)
    bs = 16
    bt = d.block_table.cpu()
    for it in range(3):
        q = torch.randn(B, 32, 128, generator=g).bfloat16()
        nk, nv = (torch.randn(B, 8, 128, generator=g).bfloat16() for _ in range(2))
        slots = torch.tensor([int(bt[b, (n - 1) // bs]) * bs + (n - 1) % bs for b, n in enumerate(lens)])
        step.set_inputs(q, nk, nv, slots, torch.tensor(lens, dtype=torch.int32))
        out = step(sync=True).clone()
        A.cache_append(nk.to(DEV), nv.to(DEV), k2, v2, slots.to(DEV))
        torch.cuda.synchronize()
        assert torch.equal(d.k_cache, k2) and torch.equal(d.v_cache, v2)
        o = oracle.decode(q, k2.cpu(), v2.cpu(), bt, torch.tensor(lens, dtype=torch.int32))
        assert np.abs(out.float().numpy() - o).max() < 1e-2
        if chunks == 1:  # same sequences per launch as the eager call: bit-identical
            ref = A.paged_decode(q.to(DEV), k2, v2, d.block_table, d.seq_lens)
            assert torch.equal(out, ref.cpu())


def test_decode_step_zero_copy_fp8_cache():
    """The zero-copy DecodeStep over an e4m3 cache: its ingest kernel quantises the new K/V into the
    pages bit for bit like the eager cache_append_fp8, and the output (written by K2'/K3' straight
    into pinned host memory) equals the eager paged_decode's bit for bit and the fp8 oracle."""
    lens = [300, 5, 64, 2000, 17]
    B = len(lens)
    d = W.make_decode(dict(W.C2, batch_size=B, seq_len=2048, kv_dtype="fp8_e4m3"), device=DEV, lens=lens,
                      extra_blocks=2)
    k2, v2 = d.k_cache.clone(), d.v_cache.clone()
    step = A.DecodeStep(d.k_cache, d.v_cache, d.block_table, batch=B, num_q_heads=32, k_scale=d.k_scale,
                        v_scale=d.v_scale)
    assert step.zero_copy
    g = torch.Generator().manual_seed(3)
    bs = 16
    bt = d.block_table.cpu()
    for it in range(2):
        q = torch.randn(B, 32, 128, generator=g).bfloat16()
        nk, nv = (torch.randn(B, 8, 128, generator=g).bfloat16() for _ in range(2))
        slots = torch.tensor([int(bt[b, (n - 1) // bs]) * bs + (n - 1) % bs for b, n in enumerate(lens)])
        step.set_inputs(q, nk, nv, slots, torch.tensor(lens, dtype=torch.int32))
        out = step(sync=True).clone()
        A.cache_append(nk.to(DEV), nv.to(DEV), k2, v2, slots.to(DEV), k_scale=d.k_scale, v_scale=d.v_scale)
        torch.cuda.synchronize()
        assert torch.equal(d.k_cache.view(torch.uint8), k2.view(torch.uint8))
        assert torch.equal(d.v_cache.view(torch.uint8), v2.view(torch.uint8))
        ref = A.paged_decode(q.to(DEV), k2, v2, d.block_table, d.seq_lens, k_scale=d.k_scale, v_scale=d.v_scale)
        assert torch.equal(out, ref.cpu())
        o = oracle.decode_fp8_np(q, k2.cpu(), v2.cpu(), bt, torch.tensor(lens, dtype=torch.int32), d.k_scale,
                                 d.v_scale)
        assert np.abs(out.float().numpy() - o).max() < 1e-2


def test_mapped_ptr_rejects_device_and_pageable_memory():
    """b200attn_mapped_ptr (the zero-copy output / ingest addresses) accepts pinned host memory only."""
    import ctypes

    from paper_2505_03780_b200 import _native

    lib = _native.load()
    out = ctypes.c_void_p()
    pinned = torch.empty(1024, dtype=torch.uint8).pin_memory()
    assert lib.b200attn_mapped_ptr(pinned.data_ptr(), ctypes.byref(out)) == 0 and out.value
    for t in (torch.empty(1024, dtype=torch.uint8, device=DEV), torch.empty(1024, dtype=torch.uint8)):
        assert lib.b200attn_mapped_ptr(t.data_ptr(), ctypes.byref(out)) == _native.BAD_ARGS


@pytest.mark.parametrize("chunks", [1, 3])
def test_prefill_step_graph_matches_eager_api(chunks):
    """PrefillStep (groups of sequences: H2D -> prefill -> D2H overlapped on two copy streams, one
    CUDA graph): with a fixed config each group's launch computes its sequences exactly like the
    eager call on the whole batch (sequences are independent), so the output is bit-identical; and
    it matches the oracle.  Several steps with new inputs through the same graph."""
    lens = [300, 1, 1000, 129, 77, 640]
    cfg = dict(BLOCK_M=256, BLOCK_N=128, num_warps=4, num_stages=3, waves_per_eu=1, PRE_LOAD_V=False)
    step = A.PrefillStep(lens, 16, 4, config=cfg, chunks=chunks, device=DEV)
    assert step.chunks == chunks
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    g = torch.Generator().manual_seed(5)
    for it in range(2):
        q, k, v = (torch.randn(sum(lens), h, 128, generator=g).bfloat16() for h in (16, 4, 4))
        step.set_inputs(q, k, v)
        out = step(sync=True).clone()
        ref = A.prefill_varlen(q.to(DEV), k.to(DEV), v.to(DEV), cu.to(DEV), max(lens), config=cfg)
        assert torch.equal(out, ref.cpu())
        o = oracle.prefill(q, k, v, cu)
        assert np.abs(out.float().numpy() - o).max() < 2e-2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench_2rank(backend, extra_env=None):
    env = dict(os.environ, PYTHONPATH=str(ROOT), **(extra_env or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4",
           "--warmup", "3", "--no-cpu-baseline", "--dist-backend", backend]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return lines[0]


def _check_2rank_line(line):
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    c4, c3 = line["extra"]["c4_strong"], line["extra"]["c3_heads_strong"]
    assert c4["seqs_per_rank"] == 128 and c4["validation"]["pass"], c4
    assert c3["kv_heads"] == [0, 4] and c3["validation"]["pass"], c3


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NCCL ranks)")
def test_bench_two_ranks_nccl():
    _check_2rank_line(_bench_2rank("nccl"))


def test_bench_two_ranks_one_gpu_gloo():
    """The N>1 host path (torchrun ranks, barriers, max-over-ranks timing, C4 batch shards and C3
    kv-head shards, gather to rank 0, oracle validation) with both ranks on one GPU (gloo)."""
    _check_2rank_line(_bench_2rank("gloo", {"B200_BENCH_ALLOW_SHARED_GPU": "1"}))


def test_plans_keep_their_tensors_alive():
    """Plans hold raw pointers in their params struct; they must own references to the tensors
    (a plan built from temporaries used to read freed memory)."""
    import gc

    def make():
        d = W.make_decode(dict(W.C2, batch_size=64, seq_len=1000), device=DEV)
        ref = A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens).clone()
        x = W.make_prefill(dict(W.C1, seq_len=300), device=DEV)
        pref = A.prefill_varlen(x.q, x.k, x.v, x.cu_seqlens, 300).clone()
        return (A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens), ref,
                A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, 300), pref)

    dp, ref, pp, pref = make()
    gc.collect()
    torch.cuda.empty_cache()
    junk = torch.full((1 << 28,), 7, dtype=torch.uint8, device=DEV)  # reuse any freed blocks
    assert torch.equal(dp.run(), ref)
    assert torch.equal(pp.run(), pref)
    del junk
