/*
 * b200attn.h — C ABI of the B200-native flash-attention forward (prefill + paged decode).
 *
 * This is the drop-in boundary for the single line of the reference runner that launches a
 * kernel for one (config, shape):
 *     ref/pkg/runner/src/ktune_triton_runner/backends.py:164-165   self.kernel[grid](*args, **kwargs)
 * where `kwargs` are the space parameters mapped by KernelBinding.kernel_kwargs
 * (ref/pkg/runner/src/ktune_triton_runner/binding.py:146-147) and the space is
 * ref/pkg/src/ktune/fixtures/flash_attention.space.json:3-16.  The variant structs below carry
 * exactly those knobs; the params structs carry borrowed device pointers and sizes.
 *
 * Conventions
 *   - All pointers are DEVICE pointers owned by the caller (borrowed for the call). No
 *     allocation happens inside any entry point; split-KV scratch is caller-provided
 *     (size it with b200attn_decode_workspace_size).
 *   - `stream` is a cudaStream_t passed as void*. Launches are stream-ordered and reentrant.
 *   - Return codes map onto the ktune protocol statuses (ref/pkg/runner/src/ktune_triton_runner/
 *     backends.py:200-205, server.py:85-99): UNSUPPORTED_CONFIG / SMEM / TMEM -> "invalid",
 *     BAD_ARGS / CUDA_ERROR -> "error".  b200attn_last_error() holds the message.
 *   - Tensors are bf16 and contiguous: q/k/v/o [tokens, heads, 128]; paged caches
 *     [num_blocks, block_size, kv_heads, 128] (the vLLM paged layout the paper's kernel
 *     family uses).
 */
#ifndef B200ATTN_H_
#define B200ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200ATTN_ABI_VERSION 2 /* 2: kv_dtype / k_scale / v_scale appended to b200attn_decode_params,
                                   b200attn_cache_append_fp8 added */

/* KV-cache element type of b200attn_decode_params.kv_dtype */
#define B200ATTN_KV_BF16 0
#define B200ATTN_KV_FP8_E4M3 1 /* OCP e4m3 bytes, dequantised as x * k_scale (K) / x * v_scale (V):
                                  vLLM's FP8_PER_TENSOR mode, the paper kernel family's upstream home
                                  (vllm/v1/attention/ops/triton_unified_attention.py _cast_kv_tile) */

typedef enum {
  B200ATTN_OK = 0,
  B200ATTN_UNSUPPORTED_CONFIG = 1, /* config has no compiled sm_100a variant      -> invalid */
  B200ATTN_SMEM_OVERFLOW = 2,      /* variant needs > 227 KB shared memory         -> invalid */
  B200ATTN_TMEM_OVERFLOW = 3,      /* variant needs > 512 TMEM columns             -> invalid */
  B200ATTN_BAD_ARGS = 4,           /* shapes / pointers inconsistent               -> error   */
  B200ATTN_CUDA_ERROR = 5          /* launch or device error (see last_error)      -> error   */
} b200attn_status;

/* One point of flash_attention.space.json (ref/pkg/src/ktune/fixtures/flash_attention.space.json:3-16). */
typedef struct {
  int32_t block_m;      /* BLOCK_M: query rows per CTA summed over its q heads: 128 (1 tile) | 256 (head pair) */
  int32_t block_n;      /* BLOCK_N: KV rows per pipeline step: 64 | 128                                         */
  int32_t num_warps;    /* softmax warps per 128-row Q tile: 4 (one thread per TMEM lane) or 8 (two, BLOCK_N 128) */
  int32_t num_stages;   /* K/V ring = (num_stages + 1) x 32 KB of TMA slots (BLOCK_N rows of K or V each)         */
  int32_t waves_per_eu; /* AMD occupancy hint; only 1 is meaningful on sm_100a                                   */
  int32_t pre_load_v;   /* V_j is always issued right behind K_j on the shared ring; accepted for parity         */
} b200attn_prefill_variant;

typedef struct {
  const void* q;              /* [total_tokens, num_q_heads, head_dim] bf16  */
  const void* k;              /* [total_tokens, num_kv_heads, head_dim] bf16 */
  const void* v;              /* [total_tokens, num_kv_heads, head_dim] bf16 */
  void* o;                    /* [total_tokens, num_q_heads, head_dim] bf16, 32-byte aligned */
  const int32_t* cu_seqlens;  /* [num_seqs + 1], device                      */
  float* lse;                 /* optional [num_q_heads, total_tokens] fp32 natural-log LSE, may be NULL */
  int32_t num_seqs;
  int32_t total_tokens;
  int32_t max_seqlen;
  int32_t num_q_heads;
  int32_t num_kv_heads;
  int32_t head_dim;           /* 128 */
  int32_t causal;             /* 1: key j attends iff j <= query position (q_len == k_len) */
  float softmax_scale;        /* <= 0 -> 1/sqrt(head_dim) */
  void* workspace;            /* longest-first work list; b200attn_prefill_workspace_size bytes,
                                 ZERO-FILLED once at allocation (the kernels keep its counter at 0) */
  size_t workspace_bytes;
} b200attn_prefill_params;

/* One point of spaces/paged_decode.space.json. */
typedef struct {
  int32_t num_splits; /* split-KV factor; 0 = heuristic (fill 148 SMs)                        */
  int32_t num_stages; /* depth of the K/V page-gather ring (32-KB slots)                      */
  int32_t tile_n;     /* tokens per MMA tile: 128 (per kv head) | 16 (page of all 8 kv heads)  */
} b200attn_decode_variant;

typedef struct {
  const void* q;              /* [batch, num_q_heads, head_dim] bf16                 */
  const void* k_cache;        /* [num_blocks, block_size, num_kv_heads, head_dim] bf16 (or e4m3, kv_dtype) */
  const void* v_cache;        /* same                                                */
  const int32_t* block_table; /* [batch, max_blocks_per_seq]                         */
  const int32_t* seq_lens;    /* [batch] cached tokens incl. the current one         */
  void* o;                    /* [batch, num_q_heads, head_dim] bf16                 */
  void* workspace;            /* split partials (+ per-sequence arrival counters of the flat kernel);
                                 b200attn_decode_workspace_size bytes, ZERO-FILLED once at allocation
                                 (the counters reset themselves; one workspace per stream in flight) */
  size_t workspace_bytes;
  int32_t batch;
  int32_t num_q_heads;
  int32_t num_kv_heads;
  int32_t head_dim;           /* 128 */
  int32_t block_size;         /* tokens per page: 8..128, power of two */
  int32_t num_blocks;
  int32_t max_blocks_per_seq;
  int32_t max_seq_len;        /* upper bound of seq_lens (sizes the split grid) */
  float softmax_scale;
  int32_t kv_dtype;           /* B200ATTN_KV_BF16 | B200ATTN_KV_FP8_E4M3 (fp8: tile_n 16 variants only) */
  float k_scale;              /* fp8 dequant scales (ignored for bf16); <= 0 -> 1 */
  float v_scale;
} b200attn_decode_params;

int b200attn_abi_version(void);
const char* b200attn_build_info(void);
const char* b200attn_status_string(int status);
const char* b200attn_last_error(void);

/* Validity of a config for a shape without launching; fills `reason` for non-OK codes. */
int b200attn_prefill_supported(const b200attn_prefill_params* p, const b200attn_prefill_variant* v,
                               char* reason, size_t reason_len);
int b200attn_decode_supported(const b200attn_decode_params* p, const b200attn_decode_variant* v,
                              char* reason, size_t reason_len);

/* K1: causal (or full) varlen prefill (schedule kernel + persistent attention kernel). */
size_t b200attn_prefill_workspace_size(const b200attn_prefill_params* p);
int b200attn_prefill(const b200attn_prefill_params* p, const b200attn_prefill_variant* v, void* stream);

/* K2 (+K3): paged split-KV decode; the combine runs iff the resolved num_splits > 1.  tile_n 16 (K2'):
 * sequences split between CTAs are merged by the K3' combine launch (an in-kernel merge by the CTA
 * finishing a sequence's last piece is kept behind B200ATTN_FLAT_MERGE=1).  Kernels are launched with
 * programmatic dependent launch (B200ATTN_PDL=0 disables it): a kernel's prologue may overlap the
 * previous kernel in the stream, and no kernel touches global memory before that one completed. */
size_t b200attn_decode_workspace_size(const b200attn_decode_params* p, const b200attn_decode_variant* v);
int b200attn_decode_num_splits(const b200attn_decode_params* p, const b200attn_decode_variant* v);
/* Number of kernels b200attn_decode enqueues for this shape and config (1 or 2), or -1 if invalid. */
int b200attn_decode_launches(const b200attn_decode_params* p, const b200attn_decode_variant* v);
int b200attn_decode(const b200attn_decode_params* p, const b200attn_decode_variant* v, void* stream);
/* K2 alone: with num_splits > 1 it leaves the unnormalised partials in the workspace (layout: a
 * 4096-byte counter header, then part_o [batch*Hq, splits, 128] fp32, then part_ml [batch*Hq, splits, 2])
 * for b200attn_combine;
 * with one split it writes O directly. */
int b200attn_decode_partial(const b200attn_decode_params* p, const b200attn_decode_variant* v, void* stream);

/* K3 alone: O[rows,128] = combine of part_o [rows, splits, 128] fp32 and part_ml [rows, splits, 2]
 * (running max in log2 units, running sum). */
int b200attn_combine(const float* part_o, const float* part_ml, void* o, int32_t rows, int32_t num_splits,
                     void* stream);

/* Paged KV-cache append: write new_k/new_v [num_tokens, kv_heads, 128] into the
 * pages named by slot_mapping[num_tokens] (slot = page * block_size + offset; < 0 skips the token). */
int b200attn_cache_append(const void* new_k, const void* new_v, void* k_cache, void* v_cache,
                          const int64_t* slot_mapping, int32_t num_tokens, int32_t num_kv_heads,
                          int32_t head_dim, int32_t block_size, int32_t num_blocks, void* stream);

/* Same for an fp8 e4m3 cache: new_k/new_v bf16 are quantised as satfinite_rn(x / k_scale) (resp. v_scale). */
int b200attn_cache_append_fp8(const void* new_k, const void* new_v, void* k_cache, void* v_cache,
                              const int64_t* slot_mapping, int32_t num_tokens, int32_t num_kv_heads,
                              int32_t head_dim, int32_t block_size, int32_t num_blocks, float k_scale, float v_scale,
                              void* stream);

/* One serving decode step's host inputs in ONE kernel (attention.DecodeStep; replaces an H2D copy node
 * + b200attn_cache_append[_fp8]): the SMs read pinned, device-mapped host memory over PCIe and
 *   - copy copy_bytes (16-byte aligned, multiple of 16) from src to dst (the step's q and seq_lens);
 *   - append new_k/new_v [num_tokens, kv_heads, 128] bf16 at slot_mapping[num_tokens] into the paged
 *     cache (bf16, or e4m3 quantised as satfinite_rn(x / k_scale) when kv_dtype = B200ATTN_KV_FP8_E4M3).
 * Host pointers must be the device-side addresses of pinned memory (b200attn_mapped_ptr). The reference
 * has no counterpart: its runner feeds device tensors (ref/pkg/runner/src/ktune_triton_runner/backends.py:164). */
int b200attn_decode_ingest(const void* src, void* dst, int64_t copy_bytes, const void* new_k, const void* new_v,
                           const int64_t* slot_mapping, void* k_cache, void* v_cache, int32_t num_tokens,
                           int32_t num_kv_heads, int32_t head_dim, int32_t block_size, int32_t num_blocks,
                           int32_t kv_dtype, float k_scale, float v_scale, void* stream);

/* Device-side address of pinned (cudaHostAlloc'd / registered) host memory; BAD_ARGS for any other pointer.
 * Lets the decode kernels write their output straight into a pinned host buffer (zero-copy D2H). */
int b200attn_mapped_ptr(const void* host, void** dev);

/* Descriptor self-test of the tcgen05 path (one CTA, no TMA):
 *   mode 0: D[128x128]  = A[128x128] . B[128x128]^T   A, B K-major
 *   mode 1: D[128x128]  = A[128x128] . B[128x128]     B MN-major ([K][N] row-major)
 *   mode 2: D[128x16]   = A^T . B^T   with A [128(K)][128(M)] MN-major, B [16][128] K-major
 *   mode 3: D[128x128]  = A . B^T     with A staged in TMEM (bf16x2 per column), B K-major (TS MMA)
 *   mode 4: D[128x128]  = A . B^T     e4m3 bytes (kind::f8f6f4), A [M][K] and B [N][K] K-major
 *   mode 5: D[128x128]  = A . B^T     e4m3 bytes, A given as [K][M] (MN-major), B K-major
 * A, B bf16 (modes 0-3) or e4m3 byte (modes 4-5) device pointers; D fp32 device pointer. */
int b200attn_selftest_umma(int mode, const void* a, const void* b, float* d, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200ATTN_H_ */
