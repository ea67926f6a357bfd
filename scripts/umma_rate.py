import ctypes, torch
from paper_2505_03780_b200 import _native
lib = _native.load()
out = torch.zeros(148, dtype=torch.int64, device="cuda")
modes = [(0, "SS N128 B-K (QK)", 128), (1, "TS N128 B-MN (PV, P in TMEM)", 128), (2, "SS N128 B-MN", 128),
         (3, "SS N256 B-K", 256), (4, "TS N128 B-K (QK, Q in TMEM)", 128), (5, "SS N64 B-K", 64),
         (6, "SS N256 B-MN", 256), (7, "TS N64 B-MN", 64), (8, "SS N128 B-K + 4 LDTM/STTM warps", 128),
         (9, "TS N128 B-MN + 4 LDTM/STTM warps", 128), (10, "SS N128 B-K + 8 LDTM/STTM warps", 128)]
for mode, name, N in modes:
    rc = lib.b200attn_debug_umma_rate(mode, 4000, 148, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0, lib.b200attn_last_error()
    cyc = out.float().mean().item()
    ideal = N * 128 / 256 * 8
    print(f"{name:32s}: {cyc:7.1f} cycles / 8 MMAs (floor {ideal:.0f}) -> {ideal / cyc * 100:.0f}% of floor")
