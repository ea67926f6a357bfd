"""bench.py host helpers (no GPU): the packed staging buffer behind the e2e measurement."""
import importlib.util
from pathlib import Path

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
    b = _bench(monkeypatch)
    g = torch.Generator().manual_seed(0)
    ts = (torch.randn(64, 32, 128, generator=g).bfloat16(), torch.randn(64, 8, 128, generator=g).bfloat16(),
          torch.randint(0, 1 << 20, (64, 256), generator=g, dtype=torch.int32),
          torch.full((64,), 4096, dtype=torch.int32), torch.arange(64, dtype=torch.int64) * 16 + 15)
    buf, views = b.pack_pinned(ts)
    assert buf.dtype == torch.uint8
    assert buf.numel() >= sum(t.numel() * t.element_size() for t in ts)
    dev = buf.clone()  # stands in for the device twin the single H2D copy fills
    for t, v in zip(ts, views):
        assert v[0] % 256 == 0  # every view starts 256-B aligned
        u = b.unpack_view(dev, v)
        assert u.dtype == t.dtype and u.shape == t.shape and torch.equal(u, t)
