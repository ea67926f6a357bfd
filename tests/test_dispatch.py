"""Per-shape dispatch table: lookups against the shipped table and synthetic ones."""
import json

import pytest

from paper_2505_03780_b200 import dispatch as D

HEADS = dict(num_q_heads=32, num_kv_heads=8, head_dim=128)


@pytest.fixture()
def table(tmp_path, monkeypatch):
    rows = [
        {"shape": dict(op="prefill", batch_size=16, seq_len=8192, causal=True, **HEADS),
         "best": dict(BLOCK_M=256, BLOCK_N=128, num_warps=4, num_stages=4, waves_per_eu=1, PRE_LOAD_V=False)},
        {"shape": dict(op="prefill", batch_size=16, seq_len_min=128, seq_len_max=8192, len_dist="geometric",
                       causal=True, **HEADS),
         "best": dict(BLOCK_M=128, BLOCK_N=128, num_warps=4, num_stages=3, waves_per_eu=1, PRE_LOAD_V=False)},
        {"shape": dict(op="decode", batch_size=64, seq_len=4096, block_size=16, **HEADS),
         "best": dict(num_splits=0, num_stages=5, TILE_N=16)},
    ]
    p = tmp_path / "t.json"
    p.write_text(json.dumps({"rows": rows}))
    monkeypatch.setenv("B200ATTN_DISPATCH", str(p))
    D.reset()
    yield
    D.reset()


def test_varlen_row_wins_on_token_count(table):
    c3 = D.default_prefill_config(num_seqs=16, total_tokens=33430, max_seqlen=8192, causal=True, **HEADS)
    assert c3["BLOCK_M"] == 128 and c3["num_stages"] == 3
    uniform = D.default_prefill_config(num_seqs=16, total_tokens=16 * 8192, max_seqlen=8192, causal=True, **HEADS)
    assert uniform["BLOCK_M"] == 256 and uniform["num_stages"] == 4


def test_kv_dtype_is_part_of_the_geometry(table):
    bf16 = D.default_decode_config(batch_size=64, seq_len=4096, block_size=16, **HEADS)
    assert bf16 == {"num_splits": 0, "num_stages": 5, "TILE_N": 16}
    fp8 = D.default_decode_config(batch_size=64, seq_len=4096, block_size=16, kv_dtype="fp8_e4m3", **HEADS)
    assert fp8["TILE_N"] == 16 and fp8["num_stages"] == D.FP8_DECODE_STAGES[(8, 4)]


def test_lookup_is_memoised_and_returns_copies(table):
    a = D.default_decode_config(batch_size=64, seq_len=4096, block_size=16, **HEADS)
    a["num_stages"] = 99
    b = D.default_decode_config(batch_size=64, seq_len=4096, block_size=16, **HEADS)
    assert b["num_stages"] == 5
    assert len(D._lookup_cache) >= 1


def test_odd_gqa_group_never_pairs_heads(table):
    c = D.default_prefill_config(num_seqs=16, total_tokens=131072, max_seqlen=8192, causal=True, num_q_heads=24,
                                 num_kv_heads=8, head_dim=128)
    assert c["BLOCK_M"] == 128


def test_shipped_table_covers_the_baseline_configs():
    D.reset()
    rows = D.table()
    assert len(rows["prefill"]) >= 78 and len(rows["decode"]) >= 81
    c2 = D.default_decode_config(batch_size=64, seq_len=4096, block_size=16, **HEADS)
    assert c2["TILE_N"] == 16


def test_lookup_memo_is_bucketed_and_bounded(table, monkeypatch):
    """A serving loop's drifting token counts must neither grow the memo per step nor miss it."""
    D._lookup_cache.clear()
    for t in range(20000, 20400):  # 400 distinct total_tokens within one quarter-octave bucket
        D.default_prefill_config(num_seqs=16, total_tokens=t, max_seqlen=2048, causal=True, **HEADS)
    assert len(D._lookup_cache) <= 2
    monkeypatch.setattr(D, "_LOOKUP_MAX", 8)
    for b in range(1, 200):
        D.default_decode_config(batch_size=b * 7, seq_len=4096, block_size=16, **HEADS)
    assert len(D._lookup_cache) <= 8


def test_flat_kernel_covers_kv_head_shards_and_large_batches(table):
    """K2' is compiled for 1/2/4/8 kv heads and any batch up to FLAT_MAX_BATCH; Hkv < 8 gets the ring
    depth compiled for every GQA group; odd geometries still fall to the split kernel."""
    assert D.flat_decode_ok(num_q_heads=8, num_kv_heads=1, block_size=16, batch_size=256)
    assert D.flat_decode_ok(num_q_heads=8, num_kv_heads=2, block_size=32, batch_size=4096)
    assert not D.flat_decode_ok(num_q_heads=12, num_kv_heads=3, block_size=16)
    assert not D.flat_decode_ok(num_q_heads=8, num_kv_heads=8, block_size=48)
    assert not D.flat_decode_ok(batch_size=D.FLAT_MAX_BATCH + 1)
    c = D.default_decode_config(batch_size=256, seq_len=32768, num_q_heads=8, num_kv_heads=1, head_dim=128,
                                block_size=16)
    assert c == {"num_splits": 0, "num_stages": D.FLAT_STAGES_NARROW, "TILE_N": 16}
    f = D.default_decode_config(batch_size=256, seq_len=32768, num_q_heads=8, num_kv_heads=1, head_dim=128,
                                block_size=16, kv_dtype="fp8_e4m3")
    assert f["TILE_N"] == 16 and f["num_stages"] == D.FP8_DECODE_STAGES[(1, 8)]
