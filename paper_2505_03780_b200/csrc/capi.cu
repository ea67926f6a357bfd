// capi.cu — extern "C" entry points of libb200attn.so (declared in include/b200attn.h).
//
// Host responsibilities only: validate, pick the compiled template variant for a config,
// encode TMA tensor maps (cuTensorMapEncodeTiled via the runtime's driver entry point, so the
// library does not link libcuda), size the split-KV grid, and launch on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <set>
#include <utility>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges are free unless a profiler attaches

#include "../../include/b200attn.h"
#include "decode_flat_sm100.cuh"
#include "decode_sm100.cuh"
#include "prefill_sm100.cuh"
#include "selftest_sm100.cuh"

namespace {

// NVTX range around each host entry point (SURVEY §5 tracing): nsys / ncu --nvtx see which API call
// enqueued which kernels
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kMaxSmem = 232448;  // 227 KB opt-in per CTA on sm_100a
constexpr int kNumSMs = 148;
// Every decode workspace starts with kFlatCounters int32 arrival counters (K2' in-kernel merge) at a
// FIXED offset, so launches of different shapes / kernels sharing one workspace never read each
// other's partials as counters (zero before first use; every launch leaves them zero).
constexpr size_t kFlatCounters = 1024;  // batches above this use the K3' combine (no fused merge)

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(B200ATTN_CUDA_ERROR, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

void copy_reason(char* dst, size_t n) {
  if (dst && n) {
    strncpy(dst, g_err, n - 1);
    dst[n - 1] = 0;
  }
}

// ------------------------------------------------------------------ launches
// Programmatic dependent launch (sm_90+): the kernel's prologue overlaps the previous kernel's tail
// in the stream (the kernels call griddep_wait() before touching global memory).  On by default;
// B200ATTN_PDL=0 launches plainly (A/B).
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("B200ATTN_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Same with CTA pairs: clusters of 2 along x (the pair lands on one TPC; cta_group::2 kernels)
template <typename... KArgs, typename... Args>
cudaError_t launch_k_pair(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ tensor maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D bf16 map over [d2][d1][d0] (d0 contiguous) with a {64, box1, box2} SWIZZLE_128B box.
int make_map_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                uint64_t stride2_bytes, uint32_t box1, uint32_t box2) {
  auto fn = encode_fn();
  if (!fn) return fail(B200ATTN_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {64, box1, box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(B200ATTN_BAD_ARGS, "cuTensorMapEncodeTiled failed (%d): dims {%llu,%llu,%llu} box {64,%u,%u}",
                static_cast<int>(r), (unsigned long long)d0, (unsigned long long)d1, (unsigned long long)d2, box1,
                box2);
  return B200ATTN_OK;
}

// 3-D byte map (fp8 pages) over [d2][d1][d0] with a {box0 = 128, box1, box2} SWIZZLE_128B box.
int make_map_u8_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                   uint64_t stride2_bytes, uint32_t box0, uint32_t box1, uint32_t box2) {
  auto fn = encode_fn();
  if (!fn) return fail(B200ATTN_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {box0, box1, box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(B200ATTN_BAD_ARGS, "cuTensorMapEncodeTiled(u8) failed (%d)", static_cast<int>(r));
  return B200ATTN_OK;
}

// Function attributes (the >48-KB dynamic smem opt-in) live in each device's context: track them
// per (kernel, device) so a process that launches on several GPUs sets them on every one.
// Thread-safe; the lock is held only for the set lookup (the attribute call happens once).
constexpr int kMaxDevices = 64;

int ensure_smem_attr(const void* kern, int bytes, const char* what) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  {
    std::lock_guard<std::mutex> g(mu);
    if (done.count({kern, dev})) return B200ATTN_OK;
  }
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return cuda_fail(e, what);
  // the opt-in limit covers static + dynamic shared memory
  if (bytes + (int)fa.sharedSizeBytes > kMaxSmem) bytes = kMaxSmem - (int)fa.sharedSizeBytes;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();  // not sticky: keep it from surfacing in the next launch's error check
    return cuda_fail(e, what);
  }
  std::lock_guard<std::mutex> g(mu);
  done.insert({kern, dev});
  return B200ATTN_OK;
}

int num_sms();

// ------------------------------------------------------------------ prefill variants
using PrefillLauncher = int (*)(const b200attn_prefill_params*, cudaStream_t);
#ifndef B200_PREFILL_EMU
#define B200_PREFILL_EMU 4
#endif
constexpr int kPrefillEmu = B200_PREFILL_EMU;  // 1 pair in 4 on the FMA pipe (session 3, setmaxnreg kernel, C3 TFLOP/s x2: EMU 0 1129/1112, 2 1044/1043, 3 1160/1128, 4 1170/1164, 6 1168/1165)

size_t prefill_ws_ints(const b200attn_prefill_params* p, int* nkeys_out) {
  const int nkeys = (p->max_seqlen + 127) / 128;
  const size_t pairs = (size_t)p->total_tokens / 128 + (size_t)p->num_seqs + 1;
  if (nkeys_out) *nkeys_out = nkeys;
  // items: one int per (seq, q block) pair, or two per (seq, q block, kv head) entry when banded
  return 3 + (size_t)nkeys + 2 * pairs * (size_t)std::max(1, p->num_kv_heads);
}

// L2-aware banded item order (PrefillKernelArgs::band): on when the K/V the CTAs stream exceeds
// ~half of the 126-MB L2, off below (pure longest-first balances small problems best).
// B200ATTN_PREFILL_BAND=<n> forces a band of n q blocks (0 = off) for A/B.
int prefill_band(const b200attn_prefill_params* p) {
  static int forced = -2;
  if (forced == -2) {
    const char* e = getenv("B200ATTN_PREFILL_BAND");
    forced = e ? atoi(e) : -1;
  }
  if (forced >= 0) return forced;
  const double kv_bytes = (double)p->total_tokens * p->num_kv_heads * p->head_dim * 2.0 * 2.0;
  return kv_bytes > 64.0 * 1024 * 1024 ? 32 : 0;
}

// Single-pass speculative softmax on interior tiles (default); B200ATTN_PREFILL_SPECULATE=0 -> two-pass
bool prefill_speculate() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("B200ATTN_PREFILL_SPECULATE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int NQ, int BN, int NS, int SPLIT, bool PAIR = false>
int launch_prefill(const b200attn_prefill_params* p, cudaStream_t stream) {
  using C = b200::PrefillCfg<NQ, BN, NS, SPLIT, PAIR>;
  auto kern = b200::prefill_fwd_kernel<NQ, BN, NS, kPrefillEmu, SPLIT, PAIR>;
  if (int rc0 = ensure_smem_attr(reinterpret_cast<const void*>(kern), C::SMEM_BYTES,
                               "cudaFuncSetAttribute(prefill)"))
    return rc0;
  const int D = 128;
  CUtensorMap mq, mk, mv, mo;
  int rc;
  if ((rc = make_map_3d(&mq, p->q, D, p->num_q_heads, p->total_tokens, D * 2ull, (uint64_t)p->num_q_heads * D * 2,
                        1, C::BM)))
    return rc;
  // O (TMA-store epilogue, C::STAGE_O): the same {64 d, 1 head, 128 tokens} box as Q
  if ((rc = make_map_3d(&mo, p->o, D, p->num_q_heads, p->total_tokens, D * 2ull, (uint64_t)p->num_q_heads * D * 2,
                        1, C::BM)))
    return rc;
  // PAIR: each CTA of the pair loads BN/2 keys of a K tile (and 64 d columns of all BN keys of V)
  if ((rc = make_map_3d(&mk, p->k, D, p->num_kv_heads, p->total_tokens, D * 2ull,
                        (uint64_t)p->num_kv_heads * D * 2, 1, PAIR ? BN / 2 : BN)))
    return rc;
  if ((rc = make_map_3d(&mv, p->v, D, p->num_kv_heads, p->total_tokens, D * 2ull,
                        (uint64_t)p->num_kv_heads * D * 2, 1, BN)))
    return rc;
  int nkeys = 0;
  prefill_ws_ints(p, &nkeys);
  int32_t* ws = reinterpret_cast<int32_t*>(p->workspace);
  // one sequence, or sequences of equal length (total = num_seqs x max_seqlen forces every length to
  // max_seqlen): the kernel decodes items analytically, q blocks longest first across the sequences,
  // so no schedule kernel (a launch and a dependent round trip saved on small batches); the kernel's
  // last CTA re-zeroes the work counter (the workspace starts zeroed, see header)
  const bool single = p->num_seqs == 1 ||
                      (p->max_seqlen > 0 && (long long)p->num_seqs * p->max_seqlen == (long long)p->total_tokens);
  const int band = prefill_band(p);
  cudaError_t e;
  if (!single && band > 0) {
    const int nbands = (nkeys + band - 1) / band;
    e = launch_k(b200::prefill_schedule_banded_kernel, dim3(1), dim3(1024), 0, stream, p->cu_seqlens, p->num_seqs,
                 p->causal, p->num_kv_heads, band, nbands, 3 + nkeys, ws);
    if (e != cudaSuccess) return cuda_fail(e, "prefill schedule launch");
  } else if (!single) {
    const size_t hist_bytes = (size_t)nkeys * sizeof(int32_t);
    if (hist_bytes <= 40 * 1024)
      e = launch_k(b200::prefill_schedule_kernel<true>, dim3(1), dim3(1024), hist_bytes, stream, p->cu_seqlens,
                   p->num_seqs, p->causal, nkeys, ws);
    else
      e = launch_k(b200::prefill_schedule_kernel<false>, dim3(1), dim3(1024), 0, stream, p->cu_seqlens, p->num_seqs,
                   p->causal, nkeys, ws);
    if (e != cudaSuccess) return cuda_fail(e, "prefill schedule launch");
  }
  b200::PrefillKernelArgs a;
  a.cu_seqlens = p->cu_seqlens;
  a.items = ws + 3 + nkeys;
  a.sched = ws;
  a.o = reinterpret_cast<__nv_bfloat16*>(p->o);
  a.lse = p->lse;
  a.total_tokens = p->total_tokens;
  a.num_q_heads = p->num_q_heads;
  a.group = p->num_q_heads / p->num_kv_heads;
  a.causal = p->causal;
  a.num_hg = p->num_q_heads / (NQ * (PAIR ? 2 : 1));
  a.single_nqb = single ? (p->max_seqlen + C::BM - 1) / C::BM : 0;
  a.useqs = single ? p->num_seqs : 0;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : 1.0f / sqrtf((float)p->head_dim);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.speculate = prefill_speculate() ? 1 : 0;
  a.band = band;
  a.hpk = a.num_hg / p->num_kv_heads;
  // persistent: never more CTAs than work items (upper bound without a device read)
  const long long items_ub = ((long long)p->total_tokens / 128 + p->num_seqs) * a.num_hg;
  if constexpr (PAIR) {
    const int pairs = (int)std::min<long long>(num_sms() / 2, std::max<long long>(1, items_ub));
    e = launch_k_pair(kern, dim3(2 * pairs), dim3(C::NTHREADS), C::SMEM_BYTES, stream, mq, mk, mv, mo, a);
  } else {
    const int ctas = (int)std::min<long long>(num_sms(), std::max<long long>(1, items_ub));
    e = launch_k(kern, dim3(ctas), dim3(C::NTHREADS), C::SMEM_BYTES, stream, mq, mk, mv, mo, a);
  }
  if (e != cudaSuccess) return cuda_fail(e, "prefill launch");
  return B200ATTN_OK;
}

struct PrefillEntry {
  int nq, bn, ns, nw;
  PrefillLauncher fn;
  int smem;
  int pair;  // waves_per_eu = 2: the item runs on a CTA pair (cta_group::2)
};

// num_warps = softmax warps per 128-row Q tile: 4 (one thread per S row) or 8 (two threads per
// row, 64 columns each; BLOCK_N = 128 only, and the space's num_warps * num_stages <= 16 caps
// num_stages at 2)
#define PF(NQ, BN, NS, NW)                                                 \
  {NQ, BN, NS, NW, &launch_prefill<NQ, BN, NS, NW / 4>,                    \
   b200::PrefillCfg<NQ, BN, NS, NW / 4>::SMEM_BYTES, 0}
#define PF2(NQ, NS)                                                        \
  {NQ, 128, NS, 4, &launch_prefill<NQ, 128, NS, 1, true>,                  \
   b200::PrefillCfg<NQ, 128, NS, 1, true>::SMEM_BYTES, 1}
const PrefillEntry kPrefill[] = {
    PF(2, 128, 1, 4), PF(2, 128, 2, 4), PF(2, 128, 3, 4), PF(2, 128, 4, 4), PF(2, 64, 1, 4),  PF(2, 64, 2, 4),
    PF(2, 64, 3, 4),  PF(2, 64, 4, 4),  PF(1, 128, 1, 4), PF(1, 128, 2, 4), PF(1, 128, 3, 4), PF(1, 128, 4, 4),
    PF(1, 64, 1, 4),  PF(1, 64, 2, 4),  PF(1, 64, 3, 4),  PF(1, 64, 4, 4),  PF(2, 128, 1, 8), PF(2, 128, 2, 8),
    PF(1, 128, 1, 8), PF(1, 128, 2, 8),
    // CTA pairs (waves_per_eu = 2): BLOCK_M = 256 -> 4 q heads per pair, 128 -> 2
    PF2(2, 1), PF2(2, 2), PF2(2, 3), PF2(1, 1), PF2(1, 2), PF2(1, 3),
};
#undef PF
#undef PF2

int check_prefill(const b200attn_prefill_params* p, const b200attn_prefill_variant* v, const PrefillEntry** out) {
  if (!p || !v) return fail(B200ATTN_BAD_ARGS, "null params/variant");
  if (v->block_m != 128 && v->block_m != 256)
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "BLOCK_M=%d: a tcgen05 cta_group::1 Q tile is 128 rows; BLOCK_M must be 128 (1 tile) or 256 "
                "(2 q heads x 128 rows)",
                v->block_m);
  if (v->block_n != 64 && v->block_n != 128)
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "BLOCK_N=%d: compiled K/V tiles are 64 or 128 rows", v->block_n);
  if (v->num_warps != 4 && v->num_warps != 8)
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "num_warps=%d: a 128-row Q tile has 4 softmax warps (one thread per TMEM lane) or 8 (two "
                "threads per lane, 64 columns each)",
                v->num_warps);
  if (v->num_warps == 8 && v->block_n != 128)
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "num_warps=8 splits 128-column S rows in halves; BLOCK_N must be 128");
  if (v->waves_per_eu != 1 && v->waves_per_eu != 2)
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "waves_per_eu=%d: 1 = one CTA per work item, 2 = a CTA pair (cta_group::2) per work item",
                v->waves_per_eu);
  const int nq = v->block_m / 128;
  const int pair = v->waves_per_eu == 2 ? 1 : 0;
  const PrefillEntry* e = nullptr;
  for (const auto& x : kPrefill)
    if (x.nq == nq && x.bn == v->block_n && x.ns == v->num_stages && x.nw == v->num_warps && x.pair == pair) e = &x;
  if (!e)
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "no compiled variant for BLOCK_M=%d BLOCK_N=%d num_warps=%d num_stages=%d", v->block_m,
                v->block_n, v->num_warps, v->num_stages);
  if (e->smem > kMaxSmem)
    return fail(B200ATTN_SMEM_OVERFLOW, "shared memory %d B > %d B (BLOCK_M=%d BLOCK_N=%d num_stages=%d)",
                e->smem, kMaxSmem, v->block_m, v->block_n, v->num_stages);
  if (p->head_dim != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "head_dim=%d (compiled for 128)", p->head_dim);
  if (p->num_kv_heads <= 0 || p->num_q_heads <= 0 || p->num_q_heads % p->num_kv_heads)
    return fail(B200ATTN_BAD_ARGS, "num_q_heads=%d not a multiple of num_kv_heads=%d", p->num_q_heads,
                p->num_kv_heads);
  const int group = p->num_q_heads / p->num_kv_heads;
  if (nq == 2 && group % 2)
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "BLOCK_M=256 pairs two q heads of one kv head; GQA group %d is odd", group);
  if (pair && group % (2 * nq))
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "waves_per_eu=2 runs %d q heads of one kv head on a CTA pair; GQA group %d is not a multiple",
                2 * nq, group);
  if (p->num_seqs <= 0 || p->num_seqs > 65535 || p->total_tokens < 0 || p->max_seqlen < 0)
    return fail(B200ATTN_BAD_ARGS, "num_seqs=%d total_tokens=%d max_seqlen=%d", p->num_seqs, p->total_tokens,
                p->max_seqlen);
  if ((p->max_seqlen + 127) / 128 > 65535) return fail(B200ATTN_BAD_ARGS, "max_seqlen too large");
  if (reinterpret_cast<uintptr_t>(p->o) % 32)
    return fail(B200ATTN_BAD_ARGS, "o must be 32-byte aligned (the epilogue writes 32-byte row segments)");
  *out = e;
  return B200ATTN_OK;
}

// ------------------------------------------------------------------ decode variants
using DecodeLauncher = int (*)(const b200attn_decode_params*, int splits, int tps, bool combine, cudaStream_t);

template <int NS>
int launch_decode(const b200attn_decode_params* p, int splits, int tps, bool combine, cudaStream_t stream) {
  using C = b200::DecodeCfg<NS>;
  auto kern = b200::decode_split_kernel<NS>;
  if (int rc0 = ensure_smem_attr(reinterpret_cast<const void*>(kern), C::SMEM_BYTES,
                               "cudaFuncSetAttribute(decode)"))
    return rc0;
  const int D = 128, G = p->num_q_heads / p->num_kv_heads;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_map_3d(&mq, p->q, D, p->num_q_heads, p->batch, D * 2ull, (uint64_t)p->num_q_heads * D * 2, G, 1)))
    return rc;
  const uint64_t tokens = (uint64_t)p->num_blocks * p->block_size;
  if ((rc = make_map_3d(&mk, p->k_cache, D, p->num_kv_heads, tokens, D * 2ull, (uint64_t)p->num_kv_heads * D * 2, 1,
                        p->block_size)))
    return rc;
  if ((rc = make_map_3d(&mv, p->v_cache, D, p->num_kv_heads, tokens, D * 2ull, (uint64_t)p->num_kv_heads * D * 2, 1,
                        p->block_size)))
    return rc;
  b200::DecodeKernelArgs a;
  a.block_table = p->block_table;
  a.seq_lens = p->seq_lens;
  a.o = reinterpret_cast<__nv_bfloat16*>(p->o);
  const size_t rows = (size_t)p->batch * p->num_q_heads;
  // partials after the counter header every decode workspace starts with (see flat_workspace_bytes)
  a.part_o = p->workspace ? reinterpret_cast<float*>(reinterpret_cast<int32_t*>(p->workspace) + kFlatCounters)
                          : nullptr;
  a.part_ml = a.part_o ? a.part_o + rows * splits * D : nullptr;
  a.num_q_heads = p->num_q_heads;
  a.group = G;
  a.block_size = p->block_size;
  a.max_blocks = p->max_blocks_per_seq;
  a.num_blocks = p->num_blocks;
  a.num_splits = splits;
  a.tiles_per_split = tps;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : 1.0f / sqrtf((float)p->head_dim);
  a.scale_log2 = scale * 1.4426950408889634f;
  dim3 grid(splits, p->num_kv_heads, p->batch);
  kern<<<grid, C::NTHREADS, C::SMEM_BYTES, stream>>>(mq, mk, mv, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "decode launch");
  if (splits > 1 && combine) {
    b200::decode_combine_kernel<<<(unsigned)rows, 128, 0, stream>>>(a.part_o, a.part_ml,
                                                                    reinterpret_cast<__nv_bfloat16*>(p->o), splits);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "combine launch");
  }
  return B200ATTN_OK;
}

struct DecodeEntry {
  int ns;
  DecodeLauncher fn;
  int smem;
};
#define DF(NS) {NS, &launch_decode<NS>, b200::DecodeCfg<NS>::SMEM_BYTES}
const DecodeEntry kDecode[] = {DF(2), DF(3), DF(4), DF(5), DF(6)};
#undef DF


// ---- K2' flat partition (TILE_N = 16: 16-token page chunks of all kv heads, 128 (chunk, head,
// token) rows per MMA tile)
int num_sms() {  // per device (cached; a process may drive several GPUs)
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kNumSMs;
  std::atomic<int>& c = cache[dev & (kMaxDevices - 1)];
  int n = c.load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
    c.store(n, std::memory_order_relaxed);
  }
  return n;
}

// Persistent CTAs, but at least flat_min_tiles() tiles each when the (host-known upper bound of the)
// tile count is small: fewer partial segments to merge, same memory parallelism.
// B200ATTN_FLAT_MIN_TILES overrides the default 4 (A/B).
int flat_min_tiles() {
  static int v = 0;
  if (v == 0) {
    const char* e = getenv("B200ATTN_FLAT_MIN_TILES");
    v = (e && atoi(e) > 0) ? atoi(e) : 4;  // 4: 1 x 8k 13.9 vs 16.0 us, 16 x 512 12.6 vs 13.0 (r2f/r2g)
  }
  return v;
}

// CTAs of a flat launch (launch_flat and b200attn_decode_launches agree on it)
int flat_ctas(const b200attn_decode_params* p) {
  const int tt = 128 / p->num_kv_heads;  // tokens per tile
  const long long tiles_ub = (long long)p->batch * ((p->max_seq_len + tt - 1) / tt);
  const int mt = flat_min_tiles();
  return (int)std::max<long long>(1, std::min<long long>(num_sms(), (tiles_ub + mt - 1) / mt));
}

// Flat workspace: per-sequence arrival counters at a FIXED offset (see kFlatCounters), then
// partials, then cu_tiles.

size_t flat_workspace_bytes(const b200attn_decode_params* p) {
  const size_t slots = (size_t)num_sms() + p->batch;
  return kFlatCounters * sizeof(int32_t) + slots * p->num_q_heads * (128 + 2) * sizeof(float) +
         ((size_t)p->batch + 1) * sizeof(int32_t);
}

// Merge split sequences inside K2' (the CTA finishing a sequence's last piece merges it, no K3'
// launch) only when asked (B200ATTN_FLAT_MERGE=1, with sequences spanning few CTAs).  Measured
// against the parallel K3' on the same build (r2g mergeab, us): C2 162.8 vs 159.0, C4 shard 653 vs
// 632, 64 x 512 36.7 vs 32.4, C2 at Hkv = 2 52.8 vs 50.5 — the merging CTAs' fence + atomic + L2
// reads sit in the kernel's tail (trace: up to 8 us after the last P) while K3' reduces every
// (sequence, q head) in parallel once streaming is done.
bool flat_fused_merge(int batch, int ctas) {
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("B200ATTN_FLAT_MERGE");
    force = (e && (e[0] == '0' || e[0] == '1')) ? e[0] - '0' : -1;
  }
  if (batch > (int)kFlatCounters) return false;  // the arrival counters cover the first 1024 sequences
  return force == 1 && ctas <= 8 * batch;
}

// K3' launched with PDL behind a late-triggering K2' (B200ATTN_PDL_COMBINE=1; A/B)
bool flat_pdl_combine() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("B200ATTN_PDL_COMBINE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

using FlatLauncher = int (*)(const b200attn_decode_params*, bool combine, cudaStream_t);

template <int HKV, int G, int NS, bool FP8>
int launch_flat(const b200attn_decode_params* p, bool combine, cudaStream_t stream) {
  using C = b200::FlatCfg<HKV, G, NS, FP8>;
  auto kern = b200::decode_flat_kernel<HKV, G, NS, FP8>;
  // the per-sequence tile prefix lives in smem: the launch's dynamic size grows with the batch
  const int smem = C::smem_bytes(p->batch);
  if (smem + 64 > kMaxSmem)  // + the kernel's static shared memory (the scan's warp totals)
    return fail(B200ATTN_SMEM_OVERFLOW, "decode_flat: batch %d needs %d B smem > %d", p->batch, smem, kMaxSmem);
  if (int rc0 = ensure_smem_attr(reinterpret_cast<const void*>(kern), kMaxSmem, "cudaFuncSetAttribute(decode_flat)"))
    return rc0;
  const int D = 128;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_map_3d(&mq, p->q, D, p->num_q_heads, p->batch, D * 2ull, (uint64_t)p->num_q_heads * D * 2,
                        C::NQ, 1)))
    return rc;
  // head-major view of the page pool: dims {d, token, head}, strides {Hkv*D*2, D*2} (transposed)
  const uint64_t tokens = (uint64_t)p->num_blocks * p->block_size;
  if (FP8) {  // one {128 d, 16 tokens, Hkv heads} byte box = a whole 16-token chunk (16 KB at Hkv = 8)
    if ((rc = make_map_u8_3d(&mk, p->k_cache, D, tokens, HKV, (uint64_t)HKV * D, D, D, 16, HKV))) return rc;
    if ((rc = make_map_u8_3d(&mv, p->v_cache, D, tokens, HKV, (uint64_t)HKV * D, D, D, 16, HKV))) return rc;
  } else {
    if ((rc = make_map_3d(&mk, p->k_cache, D, tokens, HKV, (uint64_t)HKV * D * 2, D * 2ull, 16, HKV))) return rc;
    if ((rc = make_map_3d(&mv, p->v_cache, D, tokens, HKV, (uint64_t)HKV * D * 2, D * 2ull, 16, HKV))) return rc;
  }
  const int ctas = flat_ctas(p);
  if (ctas > b200::kFlatMaxCtas)  // K3' keeps one ownership flag per piece in a kFlatMaxCtas smem array
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "decode_flat: %d CTAs > %d", ctas, b200::kFlatMaxCtas);
  const size_t slots = (size_t)num_sms() + p->batch;
  b200::FlatDecodeArgs a;
  a.block_table = p->block_table;
  a.seq_lens = p->seq_lens;
  a.o = reinterpret_cast<__nv_bfloat16*>(p->o);
  int32_t* counters = reinterpret_cast<int32_t*>(p->workspace);
  a.part_o = reinterpret_cast<float*>(counters + kFlatCounters);
  a.part_ml = a.part_o + slots * p->num_q_heads * 128;
  a.cu_tiles_out = reinterpret_cast<int32_t*>(a.part_ml + slots * p->num_q_heads * 2);
  const bool fused = flat_fused_merge(p->batch, ctas);
  const bool pdl_combine = combine && !fused && pdl_enabled() && flat_pdl_combine();
  a.late_trigger = pdl_combine ? 1 : 0;
  a.seq_cnt = fused ? counters : nullptr;
  a.batch = p->batch;
  a.block_size = p->block_size;
  a.max_blocks = p->max_blocks_per_seq;
  const float scale = p->softmax_scale > 0.f ? p->softmax_scale : 1.0f / sqrtf((float)p->head_dim);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.out_scale = 1.f;
  if (FP8) {  // K = e4m3 * k_scale, V = e4m3 * v_scale
    a.scale_log2 *= (p->k_scale > 0.f ? p->k_scale : 1.f);
    a.out_scale = (p->v_scale > 0.f ? p->v_scale : 1.f);
  }
  cudaError_t e = launch_k(kern, dim3(ctas), dim3(C::NTHREADS), smem, stream, mq, mk, mv, a);
  if (e != cudaSuccess) return cuda_fail(e, "decode_flat launch");
  if (combine && !fused) {
    // (warps, pieces in flight per warp) sized so the grid stays one wave (see flat_combine_kernel)
    const long long cg = (long long)p->batch * C::NQ;
    auto ck = cg <= num_sms()       ? b200::flat_combine_kernel<C::NQ, 8, 8, 1>
              : cg <= 4LL * num_sms() ? b200::flat_combine_kernel<C::NQ, 8, 4, 4>
                                      : b200::flat_combine_kernel<C::NQ, 4, 1, 16>;
    const dim3 cgrid(p->batch, C::NQ), cblock(cg <= 4LL * num_sms() ? 256 : 128);
    if (pdl_combine) {  // K2' triggers late, so K3' becomes resident only in K2's tail
      e = launch_k(ck, cgrid, cblock, 0, stream, (const float*)a.part_o, (const float*)a.part_ml,
                   (const int32_t*)a.cu_tiles_out, (int)p->batch, ctas, reinterpret_cast<__nv_bfloat16*>(p->o));
    } else {
      // a plain launch: PDL-launched while K2' triggered at its start, its CTAs sat resident beside
      // K2' and the 1-sequence x 8k decode lost 6 us (22.1 vs 15.9 us, r2d pdlab)
      ck<<<cgrid, cblock, 0, stream>>>(a.part_o, a.part_ml, a.cu_tiles_out, p->batch, ctas,
                                       reinterpret_cast<__nv_bfloat16*>(p->o));
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return cuda_fail(e, "flat combine launch");
  }
  return B200ATTN_OK;
}

struct FlatEntry {
  int hkv, g, ns;
  bool fp8;
  FlatLauncher fn;
  int smem;  // at batch 1024
};
#define FF(H, G, NS) {H, G, NS, false, &launch_flat<H, G, NS, false>, b200::FlatCfg<H, G, NS, false>::SMEM_BYTES}
#define F8(H, G, NS) {H, G, NS, true, &launch_flat<H, G, NS, true>, b200::FlatCfg<H, G, NS, true>::SMEM_BYTES}
const FlatEntry kFlat[] = {FF(8, 1, 3), FF(8, 1, 4), FF(8, 1, 5), FF(8, 1, 6), FF(8, 2, 3), FF(8, 2, 4),
                           FF(8, 2, 5), FF(8, 2, 6), FF(8, 4, 3), FF(8, 4, 4), FF(8, 4, 5), FF(8, 8, 3),
                           FF(8, 8, 4),
                           // Hkv = 1 / 2 / 4 (kv-head shards of GQA models, or such models outright):
                           // PPT = 8 / Hkv page chunks per 128-row tile
                           FF(4, 1, 4), FF(4, 2, 4), FF(4, 4, 4), FF(4, 8, 4), FF(4, 2, 5), FF(4, 4, 5),
                           FF(2, 1, 4), FF(2, 2, 4), FF(2, 4, 4), FF(2, 8, 4), FF(2, 4, 5), FF(2, 8, 5),
                           FF(1, 1, 4), FF(1, 2, 4), FF(1, 4, 4), FF(1, 8, 4), FF(1, 8, 5),
                           // fp8 e4m3 KV: num_stages = depth of the ring of 16-KB tiles
                           F8(8, 1, 4), F8(8, 1, 6), F8(8, 1, 8), F8(8, 2, 4), F8(8, 2, 6), F8(8, 2, 8),
                           F8(8, 4, 4), F8(8, 4, 6), F8(8, 4, 8), F8(8, 8, 4), F8(8, 8, 6), F8(4, 2, 8),
                           F8(4, 4, 8), F8(4, 8, 6), F8(2, 4, 8), F8(2, 8, 6), F8(1, 8, 8)};
#undef FF
#undef F8

int check_flat(const b200attn_decode_params* p, const b200attn_decode_variant* v, const FlatEntry** out) {
  if (v->num_splits != 0)
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "num_splits=%d: TILE_N=16 uses the flat stream partition (one CTA per SM); num_splits must be 0",
                v->num_splits);
  const int H = p->num_kv_heads;
  if (H != 1 && H != 2 && H != 4 && H != 8)
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "TILE_N=16 packs 1/2/4/8 kv heads per 16-token chunk; num_kv_heads=%d",
                H);
  const int G = p->num_q_heads / p->num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "TILE_N=16 compiled for GQA groups 1/2/4/8, got %d", G);
  if (p->block_size < 16 || (p->block_size & (p->block_size - 1)))
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "TILE_N=16 needs a power-of-two block_size >= 16, got %d",
                p->block_size);
  const bool fp8 = p->kv_dtype == B200ATTN_KV_FP8_E4M3;
  const FlatEntry* e = nullptr;
  for (const auto& x : kFlat)
    if (x.hkv == H && x.g == G && x.ns == v->num_stages && x.fp8 == fp8) e = &x;
  if (!e) {
    const int np = 8 * G < 16 ? 16 : 8 * G;
    const int est = v->num_stages * 32768 + 4 * np * 256 + 4096 + 1024;
    if (est > kMaxSmem)
      return fail(B200ATTN_SMEM_OVERFLOW, "TILE_N=16 num_stages=%d with %d q heads needs ~%d B smem > %d",
                  v->num_stages, p->num_q_heads, est, kMaxSmem);
    return fail(B200ATTN_UNSUPPORTED_CONFIG,
                "TILE_N=16: no compiled %s variant for num_stages=%d with %d kv heads x GQA %d", fp8 ? "fp8" : "bf16",
                v->num_stages, H, G);
  }
  const int smem = e->smem + (p->batch - 1024) * 4;  // the cu array is sized per batch
  if (smem + 64 > kMaxSmem)
    return fail(B200ATTN_SMEM_OVERFLOW, "decode_flat: batch %d needs %d B smem > %d", p->batch, smem, kMaxSmem);
  *out = e;
  return B200ATTN_OK;
}

int decode_ctas_per_sm(int smem) {
  const int per_sm = 233472;  // 228 KB per SM
  int n = per_sm / (smem + 1024);
  return n < 1 ? 1 : n;
}

// Resolve the split factor: explicit, or enough CTAs for ~4 waves of the SMs.
void resolve_splits(const b200attn_decode_params* p, const b200attn_decode_variant* v, int smem, int* splits,
                    int* tps) {
  const int tiles = (p->max_seq_len + 127) / 128;
  int s = v->num_splits;
  if (s <= 0) {
    const int units = p->batch * p->num_kv_heads;
    const int slots = kNumSMs * decode_ctas_per_sm(smem);
    s = 1;
    while (s < tiles && units * s < 2 * slots) s *= 2;
  }
  if (s > tiles) s = tiles > 0 ? tiles : 1;
  int t = (tiles + s - 1) / s;
  if (t < 1) t = 1;
  s = (tiles + t - 1) / t;  // drop empty trailing splits
  if (s < 1) s = 1;
  *splits = s;
  *tps = t;
}

int check_decode_common(const b200attn_decode_params* p) {
  if (p->head_dim != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "head_dim=%d (compiled for 128)", p->head_dim);
  if (p->num_kv_heads <= 0 || p->num_q_heads % p->num_kv_heads)
    return fail(B200ATTN_BAD_ARGS, "num_q_heads=%d not a multiple of num_kv_heads=%d", p->num_q_heads,
                p->num_kv_heads);
  const int bs = p->block_size;
  if (bs < 8 || bs > 128 || (bs & (bs - 1)))
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "block_size=%d: pages must be a power of two in [8,128]", bs);
  if (p->batch <= 0 || p->batch > 65535 || p->num_blocks <= 0 || p->max_blocks_per_seq <= 0)
    return fail(B200ATTN_BAD_ARGS, "batch=%d num_blocks=%d max_blocks_per_seq=%d", p->batch, p->num_blocks,
                p->max_blocks_per_seq);
  if (p->max_seq_len > p->max_blocks_per_seq * bs)
    return fail(B200ATTN_BAD_ARGS, "max_seq_len=%d exceeds block_table capacity %d", p->max_seq_len,
                p->max_blocks_per_seq * bs);
  return B200ATTN_OK;
}

int check_decode(const b200attn_decode_params* p, const b200attn_decode_variant* v, const DecodeEntry** out) {
  if (!p || !v) return fail(B200ATTN_BAD_ARGS, "null params/variant");
  if (v->tile_n != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "tile_n=%d (compiled: 16, 128)", v->tile_n);
  const DecodeEntry* e = nullptr;
  for (const auto& x : kDecode)
    if (x.ns == v->num_stages) e = &x;
  if (!e) return fail(B200ATTN_UNSUPPORTED_CONFIG, "num_stages=%d has no compiled decode variant", v->num_stages);
  if (e->smem > kMaxSmem) return fail(B200ATTN_SMEM_OVERFLOW, "decode smem %d B", e->smem);
  if (v->num_splits < 0 || v->num_splits > 1024) return fail(B200ATTN_BAD_ARGS, "num_splits=%d", v->num_splits);
  if (p->head_dim != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "head_dim=%d (compiled for 128)", p->head_dim);
  if (p->num_kv_heads <= 0 || p->num_q_heads % p->num_kv_heads)
    return fail(B200ATTN_BAD_ARGS, "num_q_heads=%d not a multiple of num_kv_heads=%d", p->num_q_heads,
                p->num_kv_heads);
  const int G = p->num_q_heads / p->num_kv_heads;
  if (G > 16) return fail(B200ATTN_UNSUPPORTED_CONFIG, "GQA group %d > 16 (MMA N padded to 16)", G);
  const int bs = p->block_size;
  if (bs < 8 || bs > 128 || (bs & (bs - 1)))
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "block_size=%d: pages must be a power of two in [8,128]", bs);
  if (p->batch <= 0 || p->batch > 65535 || p->num_blocks <= 0 || p->max_blocks_per_seq <= 0)
    return fail(B200ATTN_BAD_ARGS, "batch=%d num_blocks=%d max_blocks_per_seq=%d", p->batch, p->num_blocks,
                p->max_blocks_per_seq);
  if (p->max_seq_len > p->max_blocks_per_seq * bs)
    return fail(B200ATTN_BAD_ARGS, "max_seq_len=%d exceeds block_table capacity %d", p->max_seq_len,
                p->max_blocks_per_seq * bs);
  *out = e;
  return B200ATTN_OK;
}

struct DecodeChoice {
  const DecodeEntry* split = nullptr;
  const FlatEntry* flat = nullptr;
};

int resolve_decode(const b200attn_decode_params* p, const b200attn_decode_variant* v, DecodeChoice* c) {
  if (!p || !v) return fail(B200ATTN_BAD_ARGS, "null params/variant");
  int rc = check_decode_common(p);
  if (rc) return rc;
  if (p->kv_dtype != B200ATTN_KV_BF16 && p->kv_dtype != B200ATTN_KV_FP8_E4M3)
    return fail(B200ATTN_BAD_ARGS, "kv_dtype=%d", p->kv_dtype);
  if (v->tile_n == 16) return check_flat(p, v, &c->flat);
  if (p->kv_dtype == B200ATTN_KV_FP8_E4M3)
    return fail(B200ATTN_UNSUPPORTED_CONFIG, "fp8 KV cache: compiled for TILE_N=16 (flat partition) only");
  return check_decode(p, v, &c->split);
}

}  // namespace

extern "C" {

int b200attn_abi_version(void) { return B200ATTN_ABI_VERSION; }

const char* b200attn_build_info(void) {
  return "b200attn sm_100a (tcgen05/TMEM/TMA)";
}

const char* b200attn_status_string(int s) {
  switch (s) {
    case B200ATTN_OK: return "ok";
    case B200ATTN_UNSUPPORTED_CONFIG: return "unsupported_config";
    case B200ATTN_SMEM_OVERFLOW: return "smem_overflow";
    case B200ATTN_TMEM_OVERFLOW: return "tmem_overflow";
    case B200ATTN_BAD_ARGS: return "bad_args";
    case B200ATTN_CUDA_ERROR: return "cuda_error";
  }
  return "unknown";
}

const char* b200attn_last_error(void) { return g_err; }

int b200attn_prefill_supported(const b200attn_prefill_params* p, const b200attn_prefill_variant* v, char* reason,
                               size_t n) {
  const PrefillEntry* e;
  g_err[0] = 0;
  int rc = check_prefill(p, v, &e);
  copy_reason(reason, n);
  return rc;
}

size_t b200attn_prefill_workspace_size(const b200attn_prefill_params* p) {
  if (!p) return 0;
  return prefill_ws_ints(p, nullptr) * sizeof(int32_t);
}

int b200attn_prefill(const b200attn_prefill_params* p, const b200attn_prefill_variant* v, void* stream) {
  NvtxRange nvtx("b200attn_prefill");
  const PrefillEntry* e;
  g_err[0] = 0;
  int rc = check_prefill(p, v, &e);
  if (rc) return rc;
  if (!p->q || !p->k || !p->v || !p->o || !p->cu_seqlens) return fail(B200ATTN_BAD_ARGS, "null tensor pointer");
  if (p->total_tokens == 0 || p->max_seqlen == 0) return B200ATTN_OK;
  const size_t need = prefill_ws_ints(p, nullptr) * sizeof(int32_t);
  if (!p->workspace || p->workspace_bytes < need)
    return fail(B200ATTN_BAD_ARGS, "prefill workspace %zu B < %zu B", p->workspace_bytes, need);
  return e->fn(p, reinterpret_cast<cudaStream_t>(stream));
}

int b200attn_decode_supported(const b200attn_decode_params* p, const b200attn_decode_variant* v, char* reason,
                              size_t n) {
  DecodeChoice c;
  g_err[0] = 0;
  int rc = resolve_decode(p, v, &c);
  copy_reason(reason, n);
  return rc;
}

int b200attn_decode_num_splits(const b200attn_decode_params* p, const b200attn_decode_variant* v) {
  DecodeChoice c;
  if (resolve_decode(p, v, &c)) return -1;
  if (c.flat) return num_sms();  // stream partition: one range per CTA
  int s, t;
  resolve_splits(p, v, c.split->smem, &s, &t);
  return s;
}

int b200attn_decode_launches(const b200attn_decode_params* p, const b200attn_decode_variant* v) {
  DecodeChoice c;
  if (resolve_decode(p, v, &c)) return -1;
  if (c.flat) {  // K3' only when split sequences are not merged inside K2' (same rule as launch_flat)
    return flat_fused_merge(p->batch, flat_ctas(p)) ? 1 : 2;
  }
  int s, t;
  resolve_splits(p, v, c.split->smem, &s, &t);
  return s > 1 ? 2 : 1;
}

size_t b200attn_decode_workspace_size(const b200attn_decode_params* p, const b200attn_decode_variant* v) {
  DecodeChoice c;
  if (resolve_decode(p, v, &c)) return 0;
  if (c.flat) return flat_workspace_bytes(p);
  int s, t;
  resolve_splits(p, v, c.split->smem, &s, &t);
  if (s <= 1) return 0;
  const size_t rows = (size_t)p->batch * p->num_q_heads;
  return kFlatCounters * sizeof(int32_t) + rows * s * (128 + 2) * sizeof(float);
}

static int decode_impl(const b200attn_decode_params* p, const b200attn_decode_variant* v, void* stream,
                       bool combine) {
  NvtxRange nvtx("b200attn_decode");
  DecodeChoice c;
  g_err[0] = 0;
  int rc = resolve_decode(p, v, &c);
  if (rc) return rc;
  if (!p->q || !p->k_cache || !p->v_cache || !p->block_table || !p->seq_lens || !p->o)
    return fail(B200ATTN_BAD_ARGS, "null tensor pointer");
  if (c.flat) {
    const size_t need = flat_workspace_bytes(p);
    if (!p->workspace || p->workspace_bytes < need)
      return fail(B200ATTN_BAD_ARGS, "workspace %zu B < %zu B needed (flat partition)", p->workspace_bytes, need);
    return c.flat->fn(p, combine, reinterpret_cast<cudaStream_t>(stream));
  }
  int s, t;
  resolve_splits(p, v, c.split->smem, &s, &t);
  if (s > 1) {
    const size_t need =
        kFlatCounters * sizeof(int32_t) + (size_t)p->batch * p->num_q_heads * s * (128 + 2) * sizeof(float);
    if (!p->workspace || p->workspace_bytes < need)
      return fail(B200ATTN_BAD_ARGS, "workspace %zu B < %zu B needed for %d splits", p->workspace_bytes, need, s);
  }
  return c.split->fn(p, s, t, combine, reinterpret_cast<cudaStream_t>(stream));
}

int b200attn_decode(const b200attn_decode_params* p, const b200attn_decode_variant* v, void* stream) {
  return decode_impl(p, v, stream, true);
}

int b200attn_decode_partial(const b200attn_decode_params* p, const b200attn_decode_variant* v, void* stream) {
  return decode_impl(p, v, stream, false);
}

int b200attn_combine(const float* part_o, const float* part_ml, void* o, int32_t rows, int32_t num_splits,
                     void* stream) {
  g_err[0] = 0;
  if (!part_o || !part_ml || !o || rows <= 0 || num_splits <= 0) return fail(B200ATTN_BAD_ARGS, "combine args");
  b200::decode_combine_kernel<<<rows, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      part_o, part_ml, reinterpret_cast<__nv_bfloat16*>(o), num_splits);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "combine launch");
}

int b200attn_cache_append(const void* new_k, const void* new_v, void* k_cache, void* v_cache,
                          const int64_t* slot_mapping, int32_t num_tokens, int32_t num_kv_heads, int32_t head_dim,
                          int32_t block_size, int32_t num_blocks, void* stream) {
  NvtxRange nvtx("b200attn_cache_append");
  g_err[0] = 0;
  if (head_dim != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "head_dim=%d (compiled for 128)", head_dim);
  if (!new_k || !new_v || !k_cache || !v_cache || !slot_mapping || num_tokens < 0 || num_kv_heads <= 0)
    return fail(B200ATTN_BAD_ARGS, "cache_append args");
  if (num_tokens == 0) return B200ATTN_OK;
  const long long warps = (long long)num_tokens * num_kv_heads;
  const int threads = 256;
  const long long blocks = (warps * 32 + threads - 1) / threads;
  b200::cache_append_kernel<<<(unsigned)blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4*>(new_k), reinterpret_cast<const uint4*>(new_v), reinterpret_cast<uint4*>(k_cache),
      reinterpret_cast<uint4*>(v_cache), slot_mapping, num_tokens, num_kv_heads,
      (int64_t)num_blocks * block_size);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "cache_append launch");
}

int b200attn_cache_append_fp8(const void* new_k, const void* new_v, void* k_cache, void* v_cache,
                              const int64_t* slot_mapping, int32_t num_tokens, int32_t num_kv_heads, int32_t head_dim,
                              int32_t block_size, int32_t num_blocks, float k_scale, float v_scale, void* stream) {
  NvtxRange nvtx("b200attn_cache_append_fp8");
  g_err[0] = 0;
  if (head_dim != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "head_dim=%d (compiled for 128)", head_dim);
  if (!new_k || !new_v || !k_cache || !v_cache || !slot_mapping || num_tokens < 0 || num_kv_heads <= 0)
    return fail(B200ATTN_BAD_ARGS, "cache_append_fp8 args");
  if (!(k_scale > 0.f) || !(v_scale > 0.f)) return fail(B200ATTN_BAD_ARGS, "k_scale / v_scale must be > 0");
  if (num_tokens == 0) return B200ATTN_OK;
  const long long rows = (long long)num_tokens * num_kv_heads;  // one 16-lane group per (token, head) row
  const int threads = 256;
  const long long blocks = (rows * 16 + threads - 1) / threads;
  b200::cache_append_fp8_kernel<<<(unsigned)blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4*>(new_k), reinterpret_cast<const uint4*>(new_v),
      reinterpret_cast<uint2*>(k_cache), reinterpret_cast<uint2*>(v_cache), slot_mapping, num_tokens, num_kv_heads,
      (int64_t)num_blocks * block_size, 1.f / k_scale, 1.f / v_scale);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "cache_append_fp8 launch");
}

int b200attn_mapped_ptr(const void* host, void** dev) {
  g_err[0] = 0;
  if (!host || !dev) return fail(B200ATTN_BAD_ARGS, "mapped_ptr args");
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, host);
  if (e != cudaSuccess) return cuda_fail(e, "cudaPointerGetAttributes");
  if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr)
    return fail(B200ATTN_BAD_ARGS, "pointer %p is not pinned, device-mapped host memory", host);
  *dev = at.devicePointer;
  return B200ATTN_OK;
}

int b200attn_decode_ingest(const void* src, void* dst, int64_t copy_bytes, const void* new_k, const void* new_v,
                           const int64_t* slot_mapping, void* k_cache, void* v_cache, int32_t num_tokens,
                           int32_t num_kv_heads, int32_t head_dim, int32_t block_size, int32_t num_blocks,
                           int32_t kv_dtype, float k_scale, float v_scale, void* stream) {
  NvtxRange nvtx("b200attn_decode_ingest");
  g_err[0] = 0;
  if (head_dim != 128) return fail(B200ATTN_UNSUPPORTED_CONFIG, "head_dim=%d (compiled for 128)", head_dim);
  if (copy_bytes < 0 || (copy_bytes & 15) || (copy_bytes && (!src || !dst)) ||
      (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(B200ATTN_BAD_ARGS, "decode_ingest: copy range must be 16-byte aligned (%lld B)", (long long)copy_bytes);
  if (num_tokens < 0 || num_kv_heads <= 0 || (num_tokens && (!new_k || !new_v || !k_cache || !v_cache || !slot_mapping)))
    return fail(B200ATTN_BAD_ARGS, "decode_ingest append args");
  if (kv_dtype != B200ATTN_KV_BF16 && kv_dtype != B200ATTN_KV_FP8_E4M3)
    return fail(B200ATTN_BAD_ARGS, "decode_ingest: kv_dtype %d", kv_dtype);
  const bool fp8 = kv_dtype == B200ATTN_KV_FP8_E4M3;
  if (fp8 && (!(k_scale > 0.f) || !(v_scale > 0.f))) return fail(B200ATTN_BAD_ARGS, "k_scale / v_scale must be > 0");
  const int threads = 256;
  const long long n16 = copy_bytes / 16;
  // enough copy threads for every 16-B load of a C2-sized step (512 KB) to be in flight at once
  const int copy_blocks = (int)std::min<long long>((n16 + threads - 1) / threads, 2LL * num_sms());
  const long long rows = (long long)num_tokens * num_kv_heads;
  const long long append_blocks = (rows * (fp8 ? 16 : 32) + threads - 1) / threads;
  const long long blocks = copy_blocks + append_blocks;
  if (blocks == 0) return B200ATTN_OK;
  b200::decode_ingest_kernel<<<(unsigned)blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), n16, copy_blocks,
      reinterpret_cast<const uint4*>(new_k), reinterpret_cast<const uint4*>(new_v), k_cache, v_cache, slot_mapping,
      num_tokens, num_kv_heads, (int64_t)num_blocks * block_size, fp8 ? 1 : 0, fp8 ? 1.f / k_scale : 1.f,
      fp8 ? 1.f / v_scale : 1.f);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "decode_ingest launch");
}

#ifdef B200_TRACE
int b200attn_debug_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, b200::g_trace, sizeof(unsigned long long) * (size_t)n);
}
int b200attn_debug_ptrace(unsigned long long* host, int n, unsigned* launches) {  // K1 [2][1024][8]
  int rc = (int)cudaMemcpyFromSymbol(host, b200::g_ptrace, sizeof(unsigned long long) * (size_t)n);
  if (!rc && launches) rc = (int)cudaMemcpyFromSymbol(launches, b200::g_plaunch, sizeof(unsigned));
  return rc;
}
int b200attn_debug_dtrace(unsigned long long* host, int n) {  // K2' per-CTA timeline [1024][8]
  return (int)cudaMemcpyFromSymbol(host, b200::g_dtrace, sizeof(unsigned long long) * (size_t)n);
}
#endif

int b200attn_debug_umma_rate(int mode, int iters, int ctas, long long* out_dev, void* stream) {
  const int smem = 32768 + 65536 + 16 + 1024;
  void (*k)(int, long long*) = nullptr;
  switch (mode) {
    case 0: k = b200::umma_rate_kernel<128, false, false>; break;
    case 1: k = b200::umma_rate_kernel<128, true, true>; break;
    case 2: k = b200::umma_rate_kernel<128, false, true>; break;
    case 3: k = b200::umma_rate_kernel<256, false, false>; break;
    case 4: k = b200::umma_rate_kernel<128, true, false>; break;
    case 5: k = b200::umma_rate_kernel<64, false, false>; break;
    case 6: k = b200::umma_rate_kernel<256, false, true>; break;
    case 7: k = b200::umma_rate_kernel<64, true, true>; break;
    case 8: k = b200::umma_rate_kernel<128, false, false, 4>; break;
    case 9: k = b200::umma_rate_kernel<128, true, true, 4>; break;
    case 10: k = b200::umma_rate_kernel<128, false, false, 8>; break;
    default: return fail(B200ATTN_BAD_ARGS, "mode");
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_fail(e, "attr");
  const int threads = mode == 10 ? 384 : (mode >= 8 ? 256 : 128);
  k<<<ctas, threads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(iters, out_dev);
  e = cudaGetLastError();
  return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "umma_rate launch");
}

int b200attn_selftest_umma(int mode, const void* a, const void* b, float* d, void* stream) {
  g_err[0] = 0;
  if (mode < 0 || mode > 5 || !a || !b || !d) return fail(B200ATTN_BAD_ARGS, "selftest args");
  if (mode >= 4) {
    const int smem = 2 * 128 * 128 + 16 + 1024;
    cudaError_t ea = cudaFuncSetAttribute(b200::umma_selftest_fp8_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (ea != cudaSuccess) return cuda_fail(ea, "cudaFuncSetAttribute(selftest fp8)");
    b200::umma_selftest_fp8_kernel<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint8_t*>(a), reinterpret_cast<const uint8_t*>(b), d, mode);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "selftest fp8 launch");
  }
  cudaError_t ea = cudaFuncSetAttribute(b200::umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        b200::kSelftestSmem);
  if (ea != cudaSuccess) return cuda_fail(ea, "cudaFuncSetAttribute(selftest)");
  b200::umma_selftest_kernel<<<1, 128, b200::kSelftestSmem, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(a), reinterpret_cast<const __nv_bfloat16*>(b), d, mode);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? B200ATTN_OK : cuda_fail(e, "selftest launch");
}

}  // extern "C"
