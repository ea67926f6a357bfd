"""bench.py host helpers (no GPU): the packed staging buffer behind the e2e measurement, the
torchrun re-exec for --gpus N, and the rank-0 validation of strong-sharded outputs."""
import importlib.util
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def _bench(monkeypatch):
    # pinned memory needs a CUDA driver; the packing logic does not
    monkeypatch.setattr(torch.Tensor, "pin_memory", lambda self: self)
    spec = importlib.util.spec_from_file_location("bench_under_test", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_pack_pinned_round_trip(monkeypatch):
    _bench(monkeypatch)
    from paper_2505_03780_b200 import attention as A

    g = torch.Generator().manual_seed(0)
    ts = (torch.randn(64, 32, 128, generator=g).bfloat16(), torch.randn(64, 8, 128, generator=g).bfloat16(),
          torch.randint(0, 1 << 20, (64, 256), generator=g, dtype=torch.int32),
          torch.full((64,), 4096, dtype=torch.int32), torch.arange(64, dtype=torch.int64) * 16 + 15)
    buf, views = A.pack_pinned(ts)
    assert buf.dtype == torch.uint8
    assert buf.numel() >= sum(t.numel() * t.element_size() for t in ts)
    dev = buf.clone()  # stands in for the device twin the single H2D copy fills
    for t, v in zip(ts, views):
        assert v[0] % 256 == 0  # every view starts 256-B aligned
        u = A.unpack_view(dev, v)
        assert u.dtype == t.dtype and u.shape == t.shape and torch.equal(u, t)


def test_gpus_n_reexecs_under_torchrun(monkeypatch):
    b = _bench(monkeypatch)
    seen = {}
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(b.os, "execv", lambda exe, cmd: seen.setdefault("cmd", cmd))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    args = type("A", (), {"gpus": 4})()
    b.maybe_respawn(args)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]
    seen.clear()
    monkeypatch.setenv("WORLD_SIZE", "4")  # already under torchrun: no re-exec
    b.maybe_respawn(args)
    assert not seen


def test_c4_shard_validation_on_cpu(monkeypatch):
    """Two 'ranks' build their own C4-geometry shards (only their pages), 'decode' them (oracle as the
    stand-in kernel), the shards are concatenated as the NCCL gather would, and rank 0's validator
    rebuilds the checked sequences from their seeds: error 0, and a corrupted output is caught."""
    b = _bench(monkeypatch)
    import oracle
    from paper_2505_03780_b200 import parallel
    from paper_2505_03780_b200 import workload as W

    shape = dict(W.C4, batch_size=5, seq_len=70, num_q_heads=16, num_kv_heads=8)
    outs = []
    for r in range(2):
        sh = parallel.shard_range(5, 2, r)
        d = W.make_decode_shard(shape, sh.start, sh.count, device="cpu")
        assert d.k_cache.shape[0] == sh.count * 5  # only this shard's pages
        outs.append(torch.from_numpy(oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)))
    full = torch.cat(outs).to(torch.bfloat16)
    v = b.validate_c4(shape, full, (0, 2, 4))
    assert v["pass"] and v["max_abs"] < 1e-2
    full[2] += 1.0
    assert not b.validate_c4(shape, full, (0, 2, 4))["pass"]


def test_c3_head_shard_validation_on_cpu(monkeypatch):
    b = _bench(monkeypatch)
    import oracle
    from paper_2505_03780_b200 import parallel
    from paper_2505_03780_b200 import workload as W

    shape = dict(W.C3, batch_size=3, seq_len_min=20, seq_len_max=90, num_q_heads=8, num_kv_heads=4)
    parts = []
    for r in range(2):
        x = W.make_prefill_heads(shape, parallel.kv_head_groups(4, 2, r), device="cpu")
        o = torch.from_numpy(oracle.prefill(x.q, x.k, x.v, x.cu_seqlens)).to(torch.bfloat16)
        parts.append(o.transpose(0, 1))
    full = torch.cat(parts)  # [Hq, T, D] as gathered on rank 0
    v = b.validate_c3_heads(shape, full, [(0, 0), (2, 3)])
    assert v["pass"], v
    full[7, -1] += 0.5
    assert not b.validate_c3_heads(shape, full, [(2, 3)])["pass"]
