"""Per-shape dispatch table: the offline sweep's answer to "which compiled variant for this shape".

The paper's in-process Triton autotuning is replaced by an offline sweep (ktune ``tune`` driving
``python -m paper_2505_03780_b200.runner``) whose best configs are exported as a ktune cache bundle
(ref/pkg/src/ktune/cache.py:291-322; entry format ref/pkg/README.md "Result / cache entry").
``load_table`` folds such a bundle (or a directory of ``*.result.json`` entries) into
{op: [(dims, best_config), ...]}; lookups pick the exact shape or else the nearest tuned shape
of the same op and head geometry (log-distance over batch_size and seq_len).
"""

from __future__ import annotations

import json
import math
import os
from collections import OrderedDict
from pathlib import Path
from typing import Optional

PKG_DIR = Path(__file__).resolve().parent
DEFAULT_TABLE = PKG_DIR / "dispatch_table.json"

# fixed defaults: what a user gets without a sweep (and the C5 "fixed default" for prefill
# is SURVEY §8(d)'s BLOCK_M=128, BLOCK_N=128, num_warps=4, num_stages=2, waves_per_eu=1).
PREFILL_DEFAULT = {"BLOCK_M": 256, "BLOCK_N": 128, "num_warps": 4, "num_stages": 3, "waves_per_eu": 1,
                   "PRE_LOAD_V": False}
PREFILL_FIXED_BASELINE = {"BLOCK_M": 128, "BLOCK_N": 128, "num_warps": 4, "num_stages": 2, "waves_per_eu": 1,
                          "PRE_LOAD_V": False}
DECODE_DEFAULT = {"num_splits": 0, "num_stages": 5, "TILE_N": 16}  # flat partition, all kv heads per tile
DECODE_SPLIT_DEFAULT = {"num_splits": 0, "num_stages": 4, "TILE_N": 128}  # any geometry

_GEOM = ("num_q_heads", "num_kv_heads", "head_dim", "block_size", "causal", "kv_dtype")
# fp8 KV (TILE_N=16 only): num_stages = depth of the ring of 16-KB tiles; deepest compiled variant per
# (kv heads, GQA group) — capi.cu kFlat
FP8_DECODE_STAGES = {(8, 1): 8, (8, 2): 8, (8, 4): 8, (8, 8): 6, (4, 2): 8, (4, 4): 8, (4, 8): 6, (2, 4): 8,
                     (2, 8): 6, (1, 8): 8}
# bf16 flat kernels at Hkv < 8 (kv-head shards): ring depth compiled for every GQA group
FLAT_STAGES_NARROW = 4

_table = None


def _entries_from(path: Path):
    doc = json.loads(path.read_text())
    if isinstance(doc, dict) and "entries" in doc:  # ktune bundle
        yield from doc["entries"]
    elif isinstance(doc, dict) and "fingerprint" in doc:  # single cache entry
        yield doc
    elif isinstance(doc, dict) and "rows" in doc:  # our compact table
        for row in doc["rows"]:
            yield {"shape": row["shape"], "result": {"best": row["best"], "best_median_ms": row.get("median_ms")}}


def load_table(path=None) -> dict:
    path = Path(path or os.environ.get("B200ATTN_DISPATCH", DEFAULT_TABLE))
    table: dict = {}
    files = []
    if path.is_dir():
        files = sorted(path.glob("*.result.json"))
    elif path.exists():
        files = [path]
    for f in files:
        for e in _entries_from(f):
            shape = e.get("shape", {})
            best = (e.get("result") or {}).get("best")
            if best and "op" in shape:
                table.setdefault(shape["op"], []).append((dict(shape), dict(best)))
    return table


def table() -> dict:
    global _table
    if _table is None:
        _table = load_table()
    return _table


def reset():
    global _table
    _table = None
    _lookup_cache.clear()


_lookup_cache: "OrderedDict" = OrderedDict()
_LOOKUP_MAX = 4096  # LRU bound (a serving loop's token counts change every step)
_BUCKETED = ("batch_size", "seq_len", "total_tokens", "max_seqlen")


def _memo_key(op: str, dims: dict):
    """Geometry exact, sizes bucketed to quarter-octaves (the lookup's own distance is a log2 sum),
    so a serving loop whose total_tokens / max_seqlen drift every step still hits the memo."""
    items = []
    for k, v in sorted(dims.items()):
        if k in _BUCKETED and isinstance(v, (int, float)) and v > 0:
            v = ("b", round(4 * math.log2(v)))
        items.append((k, v))
    return op, tuple(items)


def lookup(op: str, dims: dict) -> Optional[dict]:
    """Nearest tuned config, memoised per bucketed shape (LRU-bounded)."""
    key = _memo_key(op, dims)
    cfg = _lookup_cache.get(key, _MISS)
    if cfg is not _MISS:
        _lookup_cache.move_to_end(key)
        return cfg
    cfg = _lookup(op, dims)
    _lookup_cache[key] = cfg
    if len(_lookup_cache) > _LOOKUP_MAX:
        _lookup_cache.popitem(last=False)
    return cfg


_MISS = object()


def _lookup(op: str, dims: dict) -> Optional[dict]:
    rows = table().get(op, [])
    best, best_d = None, math.inf
    for shape, cfg in rows:
        if any(k in shape and k in dims and shape[k] != dims[k] for k in _GEOM):
            continue
        if shape.get("kv_dtype", "bfloat16") != dims.get("kv_dtype", "bfloat16"):
            continue
        d = 0.0
        for k in ("batch_size", "seq_len"):
            if k in shape and k in dims and shape[k] and dims[k]:
                d += abs(math.log2(float(shape[k])) - math.log2(float(dims[k])))
        # prefill: varlen batches differ from uniform ones of the same (batch, max length) in their
        # token count; tuned varlen rows (e.g. C3) carry it, uniform rows imply batch * seq_len
        if op == "prefill" and dims.get("total_tokens"):
            tok = _row_tokens(shape)
            if tok:
                d += abs(math.log2(float(tok)) - math.log2(float(dims["total_tokens"])))
        if d < best_d:
            best, best_d = cfg, d
    return best


def _row_tokens(shape: dict) -> int:
    if "seq_len" in shape and "batch_size" in shape:
        return int(shape["batch_size"]) * int(shape["seq_len"])
    if "seq_len_min" in shape:
        from .workload import varlen_lengths

        return sum(varlen_lengths(shape))
    return 0


def default_prefill_config(**dims) -> dict:
    dims = dict(dims)
    num_seqs = dims.pop("num_seqs", 1)
    dims["batch_size"] = num_seqs
    dims["seq_len"] = dims.get("max_seqlen", 0) or dims.get("seq_len_max", 0)
    cfg = lookup("prefill", dims)
    if cfg is None:
        cfg = PREFILL_DEFAULT
        # head pairing halves the work items; when even the unpaired grid cannot fill the SMs,
        # parallelism beats K/V reuse (C1: 4 q blocks x 32 heads -> BLOCK_M=128 is 15% faster)
        items_paired = num_seqs * ((dims.get("max_seqlen", 0) + 127) // 128) * dims.get("num_q_heads", 32) // 2
        if items_paired < 148:
            cfg = dict(cfg, BLOCK_M=128)
    if cfg["BLOCK_M"] == 256 and (dims.get("num_q_heads", 2) // max(dims.get("num_kv_heads", 1), 1)) % 2:
        cfg = dict(cfg, BLOCK_M=128)  # head pairing needs an even GQA group
    return dict(cfg)


FLAT_MAX_BATCH = 8192  # the flat kernel keeps the per-sequence tile prefix in smem (4 B per sequence)


def flat_decode_ok(num_q_heads=32, num_kv_heads=8, block_size=16, batch_size=1, **_) -> bool:
    """Shapes the TILE_N=16 flat-partition kernel is compiled for (else the per-head split kernel):
    1/2/4/8 kv heads x GQA 1/2/4/8, power-of-two pages of >= 16 tokens."""
    return (num_kv_heads in (1, 2, 4, 8) and num_q_heads % num_kv_heads == 0
            and num_q_heads // num_kv_heads in (1, 2, 4, 8)
            and block_size >= 16 and block_size & (block_size - 1) == 0 and batch_size <= FLAT_MAX_BATCH)


def default_decode_config(**dims) -> dict:
    Hkv = max(dims.get("num_kv_heads", 8), 1)
    G = dims.get("num_q_heads", 32) // Hkv
    if str(dims.get("kv_dtype", "bfloat16")).startswith(("fp8", "float8")):
        cfg = lookup("decode", dims)
        if cfg is None or cfg.get("TILE_N") != 16:
            cfg = {"num_splits": 0, "num_stages": FP8_DECODE_STAGES.get((Hkv, G), 4), "TILE_N": 16}
        return dict(cfg)
    cfg = lookup("decode", dims)
    if cfg is None:
        cfg = DECODE_DEFAULT if flat_decode_ok(**dims) else DECODE_SPLIT_DEFAULT
    if cfg.get("TILE_N") == 16 and not flat_decode_ok(**dims):
        cfg = DECODE_SPLIT_DEFAULT
    if cfg.get("TILE_N") == 16 and Hkv < 8:
        cfg = dict(cfg, num_stages=FLAT_STAGES_NARROW)
    if cfg.get("TILE_N") == 16 and Hkv * G == 64 and cfg.get("num_stages", 4) > 4:
        cfg = dict(cfg, num_stages=4)  # 64 q heads: Q/P buffers leave room for 4 ring slots
    return dict(cfg)
