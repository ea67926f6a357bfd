"""libb200attn.so loads and exports every symbol include/b200attn.h declares; validity queries
(no GPU needed) map configs onto compiled variants / rejection reasons."""
import re
from pathlib import Path

import pytest

from paper_2505_03780_b200 import _native
from paper_2505_03780_b200 import attention as A
from paper_2505_03780_b200 import configspace as CS

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "b200attn.h").read_text()
    return set(re.findall(r"\b(b200attn_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    syms = header_symbols()
    assert syms == set(_native.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.b200attn_abi_version() == _native.ABI_VERSION == 2
    assert lib.b200attn_status_string(2) == b"smem_overflow"


def test_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in r.stdout and "sm_90" not in r.stdout


C1 = dict(q_shape=(512, 32, 128), kv_heads=8, num_seqs=1, max_seqlen=512)


def cfg(**kw):
    base = dict(BLOCK_M=256, BLOCK_N=128, num_warps=4, num_stages=3, waves_per_eu=1, PRE_LOAD_V=False)
    base.update(kw)
    return base


def test_prefill_supported_accepts_compiled_variants():
    for bm in (128, 256):
        for bn in (64, 128):
            for ns in (1, 2, 3, 4):
                rc, why = A.prefill_supported(config=cfg(BLOCK_M=bm, BLOCK_N=bn, num_stages=ns), **C1)
                assert rc == _native.OK, why
        for ns in (1, 2):  # two softmax threads per S row
            rc, why = A.prefill_supported(config=cfg(BLOCK_M=bm, num_warps=8, num_stages=ns), **C1)
            assert rc == _native.OK, why


@pytest.mark.parametrize("kw,code", [
    (dict(BLOCK_M=64), _native.UNSUPPORTED_CONFIG),
    (dict(BLOCK_N=32, BLOCK_M=128), _native.UNSUPPORTED_CONFIG),
    (dict(num_warps=2), _native.UNSUPPORTED_CONFIG),
    (dict(num_warps=8, num_stages=3), _native.UNSUPPORTED_CONFIG),
    (dict(num_warps=8, num_stages=2, BLOCK_N=64), _native.UNSUPPORTED_CONFIG),
    (dict(waves_per_eu=2, num_stages=4), _native.UNSUPPORTED_CONFIG),
    (dict(waves_per_eu=2, BLOCK_N=64), _native.UNSUPPORTED_CONFIG),
    (dict(waves_per_eu=2, num_warps=8, num_stages=2), _native.UNSUPPORTED_CONFIG),
    (dict(num_stages=5), _native.UNSUPPORTED_CONFIG),
])
def test_prefill_rejections(kw, code):
    rc, why = A.prefill_supported(config=cfg(**kw), **C1)
    assert rc == code and why


def test_prefill_cta_pair_variants():
    """waves_per_eu = 2: the work item on a CTA pair; BLOCK_M = 256 needs 4 q heads per kv head."""
    for bm in (128, 256):
        for ns in (1, 2, 3):
            rc, why = A.prefill_supported(config=cfg(BLOCK_M=bm, num_stages=ns, waves_per_eu=2), **C1)
            assert rc == _native.OK, why
    rc, why = A.prefill_supported((100, 8, 128), 4, 1, 100, cfg(BLOCK_M=256, waves_per_eu=2))
    assert rc == _native.UNSUPPORTED_CONFIG and "multiple" in why  # group 2
    rc, _ = A.prefill_supported((100, 8, 128), 4, 1, 100, cfg(BLOCK_M=128, waves_per_eu=2))
    assert rc == _native.OK


def test_prefill_head_pair_needs_even_group():
    rc, why = A.prefill_supported((100, 8, 128), 8, 1, 100, cfg(BLOCK_M=256))
    assert rc == _native.UNSUPPORTED_CONFIG and "odd" in why
    rc, _ = A.prefill_supported((100, 8, 128), 8, 1, 100, cfg(BLOCK_M=128))
    assert rc == _native.OK


def test_flash_attention_space_variant_map():
    """Every point of the shipped space is either a compiled variant or has a reason."""
    s = CS.parse_space_file(Path(A.__file__).parent / "spaces" / "flash_attention.space.json")
    ok = 0
    for c in CS.enumerate_configs(s):
        rc, why = A.prefill_supported(config=c.assignments, **C1)
        assert rc in (_native.OK, _native.UNSUPPORTED_CONFIG, _native.SMEM_OVERFLOW), why
        ok += rc == _native.OK
        if rc != _native.OK:
            assert why
    # num_warps 4: BLOCK_M {128,256} x BLOCK_N {64,128} x num_stages 1..4 (x PRE_LOAD_V, which needs
    # stages <= 2) = 24; num_warps 8: BLOCK_M {128,256} x BLOCK_N 128 x num_stages {1,2} x PRE_LOAD_V = 8;
    # CTA pairs (waves_per_eu 2): BLOCK_M {128,256} x BLOCK_N 128 x num_stages 1..3 x PRE_LOAD_V = 10
    assert ok == 42


def test_decode_supported_and_splits():
    dc = dict(num_splits=0, num_stages=4, TILE_N=128)
    rc, why = A.decode_supported((64, 32, 128), (16384, 16, 8, 128), 256, 4096, dc)
    assert rc == _native.OK, why
    s = A.decode_num_splits((64, 32, 128), (16384, 16, 8, 128), 256, 4096, dc)
    assert 1 <= s <= 32
    assert A.decode_num_splits((64, 32, 128), (16384, 16, 8, 128), 256, 4096, dict(dc, num_splits=4)) == 4
    rc, why = A.decode_supported((4, 32, 128), (16384, 16, 8, 128), 256, 4096, dict(dc, TILE_N=64))
    assert rc == _native.UNSUPPORTED_CONFIG
    rc, why = A.decode_supported((4, 40, 128), (16384, 16, 2, 128), 256, 4096, dc)
    assert rc == _native.UNSUPPORTED_CONFIG and "group" in why  # G = 20 > 16
    rc, why = A.decode_supported((4, 32, 128), (16384, 24, 8, 128), 256, 4096, dc)
    assert rc == _native.UNSUPPORTED_CONFIG  # block_size 24
    rc, why = A.decode_supported((4, 32, 128), (16384, 16, 8, 128), 256, 8192, dc)
    assert rc == _native.BAD_ARGS  # exceeds block-table capacity


def test_product_path_refuses_cpu_tensors():
    import torch
    q = torch.zeros(4, 2, 128, dtype=torch.bfloat16)
    cu = torch.tensor([0, 4], dtype=torch.int32)
    with pytest.raises(ValueError, match="CUDA"):
        A.prefill_varlen(q, q[:, :1].contiguous(), q[:, :1].contiguous(), cu, 4)


# ------------------------------------------------------------------ fp8 (e4m3) KV-cache decode
C2_Q, C2_CACHE = (64, 32, 128), (16384, 16, 8, 128)


@pytest.mark.parametrize("hq,ns", [(8, 4), (8, 6), (8, 8), (16, 4), (16, 6), (16, 8), (32, 4), (32, 6), (32, 8), (64, 4), (64, 6)])
def test_fp8_decode_compiled_variants(hq, ns):
    rc, why = A.decode_supported((64, hq, 128), C2_CACHE, 256, 4096, dict(num_splits=0, num_stages=ns, TILE_N=16),
                                 kv_dtype="fp8_e4m3")
    assert rc == _native.OK, why


def test_fp8_decode_rejections():
    rc, why = A.decode_supported(C2_Q, C2_CACHE, 256, 4096, dict(num_splits=0, num_stages=4, TILE_N=128),
                                 kv_dtype="fp8_e4m3")
    assert rc == _native.UNSUPPORTED_CONFIG and "fp8" in why
    rc, why = A.decode_supported(C2_Q, C2_CACHE, 256, 4096, dict(num_splits=0, num_stages=5, TILE_N=16),
                                 kv_dtype="fp8_e4m3")
    assert rc in (_native.UNSUPPORTED_CONFIG, _native.SMEM_OVERFLOW) and why


def test_fp8_default_config_is_compiled():
    from paper_2505_03780_b200 import dispatch
    for hq in (8, 16, 32, 64):
        c = dispatch.default_decode_config(batch_size=64, seq_len=4096, num_q_heads=hq, num_kv_heads=8,
                                           head_dim=128, block_size=16, kv_dtype="fp8_e4m3")
        rc, why = A.decode_supported((64, hq, 128), C2_CACHE, 256, 4096, c, kv_dtype="fp8_e4m3")
        assert rc == _native.OK, (hq, c, why)
