"""Does cuTensorMapEncodeTiled accept non-monotonic strides (dim1 stride > dim2 stride)?"""
import ctypes
import torch
torch.cuda.init()
x = torch.zeros(1024, 16, 8, 128, dtype=torch.bfloat16, device="cuda")  # [NB, bs, Hkv, D]
cuda = ctypes.CDLL("libcuda.so.1")
raw = (ctypes.c_uint8 * 256)()
addr = (ctypes.addressof(raw) + 63) & ~63
tm = ctypes.c_void_p(addr)
U64 = ctypes.c_uint64 * 3
U64b = ctypes.c_uint64 * 2
U32 = ctypes.c_uint32 * 3
for name, dims, strides, box in [
    ("monotonic {d, head, token}", U64(128, 8, 1024 * 16), U64b(256, 2048), U32(64, 8, 16)),
    ("transposed {d, token, head}", U64(128, 1024 * 16, 8), U64b(2048, 256), U32(64, 16, 8)),
]:
    r = cuda.cuTensorMapEncodeTiled(tm, 9, 3, ctypes.c_void_p(x.data_ptr()), dims, strides, box, U32(1, 1, 1), 0, 3, 2, 0)
    print(name, "->", r)
