// decode_flat_sm100.cuh — K2': paged-KV decode, flat (stream-K style) partition, all KV heads
// per CTA, sm_100a.   Selected by TILE_N = 16 (tokens per page chunk).
//
// Why: 16 tokens of a page of the vLLM cache [num_blocks, bs, Hkv, 128] hold 16 x Hkv x 256 B
// contiguous (32 KB at Hkv = 8).  K2 (decode_sm100.cuh) gathers it per kv head as 2-KB strided
// boxes; here one TMA box {64 d, 16 tokens, Hkv heads} per 64-column half moves the whole chunk,
// and the MMA M dimension is 128 (chunk, head, token) rows: one chunk at Hkv = 8, PPT = 8 / Hkv
// chunks (TT = 128 / Hkv tokens) at Hkv = 1, 2, 4.  The tensor map is head-major (strides
// {Hkv*256 B token, 256 B head} — transposed) so smem row r = (chunk*Hkv + head)*16 + token: every
// 16-row group is one (chunk, head), every warp owns two groups; the per-head max over a tile is a
// 16-lane shuffle (plus, at Hkv < 8, a max over the PPT groups of the head through smem).
//
//   S^T[(h,t), qh] = K_page[(h,t), :] . Q[qh, :]^T            M=128 rows, N = Hq (pad 16)
//   O^T[d, qh]    += V_page^T[d, (h,t)] . P^T[(h,t), qh]       P^T block-diagonal: entries with
//                                                              qh / G != h are never written
//                                                              (zeroed once per CTA)
// Work: the tiles of all sequences are laid end to end (cu_tiles) and cut into gridDim.x equal
// contiguous ranges — one persistent CTA per SM, perfectly balanced for any length mix.  A
// range may cover several sequences and parts of sequences; each (CTA, sequence) piece is a
// segment: complete sequences are normalised and written by the CTA, pieces go to partial slot
// (cta + seq) and K3' (flat_combine_kernel) merges them.
//
// FP8 = true (e4m3 KV cache, per-tensor k_scale / v_scale — vLLM's FP8_PER_TENSOR semantics):
// the pages feed tcgen05 kind::f8f6f4 MMAs straight from their TMA tiles (one 16-KB SW128 box
// per page; V as the MN-major A operand of PV) — no conversion pass.  The bf16-precision side
// of each product is split into two e4m3 terms, hi = e4m3(x) and lo = e4m3(16 (x - hi)), stacked
// along N: Q (scaled per q head by a power of two into e4m3 range) for QK^T, and P (scaled by
// 2^4, with the lazy-max threshold at 4 so P*16 <= 256) for PV.  S = S_hi + S_lo / 16 and
// O = O_hi + O_lo / 16 recover ~2^-8 relative precision, i.e. bf16-level operands.
#pragma once
#include "sm100_common.cuh"

namespace b200 {

struct FlatDecodeArgs {
  const int32_t* block_table;  // [B, max_blocks]
  const int32_t* seq_lens;     // [B]
  __nv_bfloat16* o;            // [B, Hq, 128]
  float* part_o;               // [(ctas + B), Hq, 128]
  float* part_ml;              // [(ctas + B), Hq, 2]  (max in log2 units, sum)
  int32_t* cu_tiles_out;       // [B + 1] (written by CTA 0 for the combine)
  int32_t* seq_cnt;            // [B] arrival counters (zeroed workspace, self-resetting), or null:
                               // non-null = the last CTA to finish a piece of a split sequence merges
                               // it in place (no K3' launch)
  int32_t batch;
  int32_t block_size;
  int32_t max_blocks;
  float scale_log2;  // softmax_scale * log2(e)  (fp8: * k_scale)
  float out_scale;   // 1                        (fp8: v_scale)
  int32_t late_trigger;  // PDL: 0 = let the next kernel launch at once; 1 = once this CTA's tile loops end
                         // (a PDL-launched K3' then becomes resident only in K2's tail)
};

template <int HKV_, int G, int NSTAGE, bool FP8 = false>
struct FlatCfg {
  static constexpr int D = 128, HKV = HKV_, ROWS = 128;
  static constexpr int TT = ROWS / HKV;  // tokens per MMA tile
  static constexpr int PPT = TT / 16;    // 16-token page chunks per tile (one TMA box pair each)
  static constexpr int NQ = HKV * G;
  static_assert(HKV == 1 || HKV == 2 || HKV == 4 || HKV == 8, "Hkv in {1,2,4,8}");
  static_assert(!FP8 || NQ >= 8, "fp8 Q split: at least 8 q heads (16 threads per q head)");
  static constexpr int NP = NQ < 16 ? 16 : NQ;  // MMA N per operand term
  static constexpr int NT = FP8 ? 2 : 1;        // terms stacked along N (hi, lo)
  static constexpr int NTHREADS = 192, TMA_WARP = 4, MMA_WARP = 5;
  static constexpr int SLOT = ROWS * D * (FP8 ? 1 : 2), HALF = ROWS * 128;  // one K or V page tile
  static constexpr int QB = NP * 256, QHALF = NP * 128;  // bf16 Q tile (as TMA loads it)
  static constexpr int Q8B = 2 * NP * 128;               // fp8 [Q_hi; Q_lo] tile (FP8)
  static constexpr int PB = FP8 ? 2 * NP * 128 : NP * 256, PHALF = NP * 128;
  static constexpr int OFF_KV = 0;
  static constexpr int OFF_Q = OFF_KV + NSTAGE * SLOT;
  static constexpr int OFF_Q8 = OFF_Q + 2 * QB;
  static constexpr int OFF_P = OFF_Q8 + (FP8 ? 2 * Q8B : 0);
  static constexpr int OFF_ALPHA = OFF_P + 2 * PB;       // [NP] f32 rescale factors + int32 flags[2][4]
  static constexpr int OFF_QS = OFF_ALPHA + 2 * NP * 4;  // [2][NP] f32 per-q-head Q scales (FP8)
  static constexpr int OFF_ML = OFF_QS + 2 * NP * 4;     // [2][NP] f32
  static constexpr int OFF_GRP = OFF_ML + 2 * NP * 4;    // [8][G] f32 per-(chunk, head) max / sum (HKV < 8)
  static constexpr int OFF_BAR = (OFF_GRP + 8 * G * 4 + 7) & ~7;
  static constexpr int NUM_BARS = 4 + 2 * NSTAGE + 8 + 2;
  static constexpr int OFF_CU = OFF_BAR + NUM_BARS * 8 + 16;  // [batch + 1] i32 (sized per launch)
  // dynamic smem of a launch: the cu array grows with the batch (+1024 for the base alignment)
  __host__ __device__ static constexpr int smem_bytes(int batch) { return OFF_CU + (batch + 1) * 4 + 1024; }
  static constexpr int SMEM_BYTES = smem_bytes(1024);  // nominal (the dispatcher's size check)
  static constexpr int TCOLS = 4 * NT * NP;  // S[2] + O[2], NT terms each
  static constexpr uint32_t TMEM_COLS = TCOLS <= 64 ? 64 : (TCOLS <= 128 ? 128 : (TCOLS <= 256 ? 256 : 512));
  __host__ __device__ static constexpr uint32_t S_COL(int i) { return (i & 1) * NT * NP; }                // per tile
  __host__ __device__ static constexpr uint32_t O_COL(int k) { return 2 * NT * NP + (k & 1) * NT * NP; }  // per segment
  static constexpr float LAZY = FP8 ? 4.0f : 8.0f;  // log2 headroom before the running max moves
  // a warp's two 16-row groups hold heads (2w) % HKV and (2w + 1) % HKV: adjacent S column ranges
  // (2 G columns) at HKV >= 2, the same range (G columns) at HKV = 1
  static constexpr int WCOLS = HKV >= 2 ? 2 * G : G;
};

#ifdef B200_TRACE
// debug-only per-CTA timeline (%globaltimer ns): 0 entry, 1 after the tile scan, 2 first S seen by the
// softmax, 3 last P of the range, 4 last segment's output / partial written, 7 arrival counted (fused
// merge), 5 merge done, 6 exit
__device__ unsigned long long g_dtrace[1024][8];
__device__ __forceinline__ void dtrace(int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 1024) g_dtrace[blockIdx.x][ev] = t;
}
#define DTRACE(ev, cond) \
  do {                   \
    if (cond) dtrace(ev); \
  } while (0)
#else
#define DTRACE(ev, cond) \
  do {                   \
  } while (0)
#endif

__device__ __forceinline__ int flat_cta_of(int t, int ctas, int ntiles) {
  return static_cast<int>(((static_cast<long long>(t) + 1) * ctas - 1) / ntiles);
}

// byte offset of element (row, col) of a [rows][128 B] SW128 tile (16-byte chunk ^ row % 8)
__device__ __forceinline__ uint32_t sw128_b(int row, int col) {
  return row * 128 + ((((col >> 4) ^ (row & 7))) << 4) + (col & 15);
}

// (x0, x1) -> e4m3 hi bytes and lo bytes of the split x ~ hi + lo / 16 (satfinite, RN)
__device__ __forceinline__ void e4m3_split2(float x0, float x1, uint16_t& hi, uint16_t& lo) {
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(x1), "f"(x0));
  uint32_t h16;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h16) : "h"(hi));
  const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h16));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"((x1 - hf.y) * 16.f), "f"((x0 - hf.x) * 16.f));
}

__device__ __forceinline__ bool flat_owns(int c, int ctas, int ntiles) {
  return static_cast<long long>(c) * ntiles / ctas != (static_cast<long long>(c) + 1) * ntiles / ctas;
}

// Fused K3' (the 128 softmax/epilogue threads of a CTA that just wrote a partial piece of sequence
// b): arrive on b's counter; the CTA whose arrival completes b merges every piece in place — its
// own from registers (r, ml_s), the others' from L2 — and writes b's output.  In the flat partition
// a sequence split between CTAs c and c+1 is finished last by c (its head piece ends c's range,
// its tail piece starts c+1's), so merges land in the kernel's tail, one per CTA at most.
// Loads are batched (QC q heads x 2 pieces, three loads each, all issued before any use): a
// dependent load chain per piece is what made an earlier in-kernel merge L2-latency-bound.
// Protocol: barrier (the partial stores of all 128 threads happen-before it), then one thread's
// gpu-scope fence + atomicAdd (the fence is cumulative, so only one warp waits for the stores to
// drain); the merging threads fence again and read other CTAs' partials with ld.global.cg (L2,
// never a stale L1 line).
template <int NQ, int NP>
__device__ __forceinline__ void flat_merge_if_last(const FlatDecodeArgs& args, const uint32_t (&r)[NQ],
                                                   const float* ml_s, volatile int* flags, const int32_t* cu,
                                                   int b, int ntiles, int row) {
  constexpr int D = 128;
  const int ctas = static_cast<int>(gridDim.x);
  named_bar_sync(1, 128);  // every thread's partial stores happen-before thread 0's fence (cumulative)
  if (row == 0) {
    __threadfence();
    const int c0 = flat_cta_of(cu[b], ctas, ntiles), c1 = flat_cta_of(cu[b + 1] - 1, ctas, ntiles);
    int pieces = 0;
    for (int c = c0; c <= c1; ++c) pieces += flat_owns(c, ctas, ntiles);
    const int last = atomicAdd(args.seq_cnt + b, 1) == pieces - 1;
    if (last) args.seq_cnt[b] = 0;  // every arrival of this launch is in: reset for the next one
    flags[8] = last;
    flags[9] = c0;
    flags[10] = c1;
  }
  named_bar_sync(1, 128);
  DTRACE(7, row == 0);
  if (!flags[8]) return;
  __threadfence();
  const int c0 = flags[9], c1 = flags[10], self = static_cast<int>(blockIdx.x);
  constexpr int QC = NQ < 16 ? NQ : 16;
#pragma unroll
  for (int q0 = 0; q0 < NQ; q0 += QC) {
    // pieces are folded in CTA order whoever merges (this CTA's own piece from registers at its
    // position), so the fp32 result is bit-identical from launch to launch
    float M[QC], L[QC], acc[QC];
#pragma unroll
    for (int j = 0; j < QC; ++j) {
      M[j] = -INFINITY;
      L[j] = 0.f;
      acc[j] = 0.f;
    }
    auto fold = [&](float mp, float lp, float op, int j) {
      const float mn = fmaxf(M[j], mp);
      if (mn == -INFINITY) return;
      const float wa = fast_exp2(M[j] - mn), wb = fast_exp2(mp - mn);
      L[j] = fmaf(L[j], wa, lp * wb);
      acc[j] = fmaf(acc[j], wa, op * wb);
      M[j] = mn;
    };
    auto fold_self = [&]() {
#pragma unroll
      for (int j = 0; j < QC; ++j) fold(ml_s[q0 + j], ml_s[NP + q0 + j], __uint_as_float(r[q0 + j]) * args.out_scale, j);
    };
    int c = c0;
    while (c <= c1) {
      // the next two owned pieces in CTA order; this CTA's own piece is folded in between
      int ca = -1, cb = -1;
      for (; c <= c1 && ca < 0; ++c)
        if (flat_owns(c, ctas, ntiles)) ca = c;
      if (ca == self) {
        fold_self();
        continue;
      }
      for (; c <= c1 && cb < 0; ++c)
        if (flat_owns(c, ctas, ntiles)) cb = c;
      if (ca < 0) break;
      const bool b_self = (cb == self);
      const size_t sa = static_cast<size_t>(ca) + b, sb = static_cast<size_t>(cb < 0 || b_self ? ca : cb) + b;
      float ma[QC], la[QC], oa[QC], mb[QC], lb[QC], ob[QC];
#pragma unroll
      for (int j = 0; j < QC; ++j) {
        ma[j] = __ldcg(args.part_ml + (sa * NQ + q0 + j) * 2);
        la[j] = __ldcg(args.part_ml + (sa * NQ + q0 + j) * 2 + 1);
        oa[j] = __ldcg(args.part_o + (sa * NQ + q0 + j) * D + row);
        mb[j] = __ldcg(args.part_ml + (sb * NQ + q0 + j) * 2);
        lb[j] = __ldcg(args.part_ml + (sb * NQ + q0 + j) * 2 + 1);
        ob[j] = __ldcg(args.part_o + (sb * NQ + q0 + j) * D + row);
      }
#pragma unroll
      for (int j = 0; j < QC; ++j) fold(ma[j], la[j], oa[j], j);
      if (b_self) {
        fold_self();
      } else if (cb >= 0) {
#pragma unroll
        for (int j = 0; j < QC; ++j) fold(mb[j], lb[j], ob[j], j);
      }
    }
#pragma unroll
    for (int j = 0; j < QC; ++j)
      args.o[(static_cast<size_t>(b) * NQ + q0 + j) * D + row] = __float2bfloat16_rn(L[j] > 0.f ? acc[j] / L[j] : 0.f);
  }
}

template <int HKV, int G, int NSTAGE, bool FP8 = false>
__global__ void __launch_bounds__(FlatCfg<HKV, G, NSTAGE, FP8>::NTHREADS, 1)
    decode_flat_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_k,
                       const __grid_constant__ CUtensorMap tmap_v, const FlatDecodeArgs args) {
  using C = FlatCfg<HKV, G, NSTAGE, FP8>;
  constexpr int NQ = C::NQ, NP = C::NP, D = C::D, NT = C::NT, PPT = C::PPT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sKV = smem + C::OFF_KV;
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sQ8 = smem + C::OFF_Q8;
  uint8_t* sP = smem + C::OFF_P;
  float* alpha_s = reinterpret_cast<float*>(smem + C::OFF_ALPHA);
  float* qs_s = reinterpret_cast<float*>(smem + C::OFF_QS);
  float* ml_s = reinterpret_cast<float*>(smem + C::OFF_ML);
  float* grp_s = reinterpret_cast<float*>(smem + C::OFF_GRP);
  int32_t* cu = reinterpret_cast<int32_t*>(smem + C::OFF_CU);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;       // [2] bf16 Q landed (TMA)
  uint64_t* q_empty = bars + 2;  // [2]
  uint64_t* kv_full = bars + 4;  // [NSTAGE]
  uint64_t* kv_empty = kv_full + NSTAGE;
  uint64_t* s_full = kv_empty + NSTAGE;  // [2]
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 2;
  uint64_t* o_empty = o_full + 2;
  uint64_t* q_conv = o_empty + 2;  // [2] fp8 Q split ready (FP8)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);
  const int warp = warp_id(), lane = lane_id();
  const int B = args.batch;
  DTRACE(0, threadIdx.x == 0);

  // zero Q (padded rows), the fp8 Q split and P^T (block-diagonal zeros) once
  for (int i = threadIdx.x; i < (C::OFF_ALPHA - C::OFF_Q) / 16; i += C::NTHREADS)
    reinterpret_cast<uint4*>(sQ)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&q_conv[i], 128);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 128);
    }
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == C::TMA_WARP && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_k);
    tma_prefetch_desc(&tmap_v);
  }
  griddep_wait();  // PDL: the prologue above overlapped the previous kernel; data access starts here
  if (!args.late_trigger) griddep_launch();
  // ---- tiles per sequence -> cu (exclusive prefix), block-wide: each thread scans a contiguous
  // chunk of sequences (any batch size, no serial chain of loads)
  {
    __shared__ int warp_tot[C::NTHREADS / 32];
    const int per = (B + C::NTHREADS - 1) / C::NTHREADS;
    const int b0 = min(B, static_cast<int>(threadIdx.x) * per), b1 = min(B, b0 + per);
    int local = 0;
    for (int b = b0; b < b1; ++b) local += (args.seq_lens[b] + C::TT - 1) / C::TT;
    int incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += n;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int run = incl - local;
    for (int w = 0; w < warp; ++w) run += warp_tot[w];
    if (threadIdx.x == 0) cu[0] = 0;
    for (int b = b0; b < b1; ++b) {
      run += (args.seq_lens[b] + C::TT - 1) / C::TT;
      cu[b + 1] = run;
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  DTRACE(1, threadIdx.x == 0);
  const int ntiles = cu[B];
  const int T0 = static_cast<int>(static_cast<long long>(blockIdx.x) * ntiles / gridDim.x);
  const int T1 = static_cast<int>((static_cast<long long>(blockIdx.x) + 1) * ntiles / gridDim.x);
  if (blockIdx.x == 0)
    for (int b = threadIdx.x; b <= B; b += C::NTHREADS) args.cu_tiles_out[b] = cu[b];
  if (args.seq_cnt != nullptr) {  // fused merge (no K3'): empty sequences get their zero output here
    for (int b = blockIdx.x; b < B; b += gridDim.x)
      if (cu[b + 1] == cu[b])
        for (int i = threadIdx.x; i < NQ * D / 8; i += C::NTHREADS)
          reinterpret_cast<uint4*>(args.o + static_cast<size_t>(b) * NQ * D)[i] = make_uint4(0, 0, 0, 0);
  }
  if (T0 >= T1) return;  // more CTAs than tiles (uniform per CTA)
  // first sequence with tiles beyond T0
  int b_first;
  {
    int lo = 0, hi = B - 1;  // smallest b with cu[b+1] > T0
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cu[mid + 1] > T0) hi = mid;
      else lo = mid + 1;
    }
    b_first = lo;
  }

  if (warp == C::MMA_WARP) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == C::TMA_WARP) {
    // ------------------------------------------------------------ TMA producer
    const uint64_t stream_once = policy_evict_first();
    const int bs = args.block_size;
    int it = 0, k = 0, b = b_first;
    for (int t = T0; t < T1; ++k) {
      while (cu[b + 1] <= t) ++b;
      const int seg_end = min(T1, cu[b + 1]);
      const int tile0 = cu[b];
      const int len = args.seq_lens[b];
      if (lane == 0) {
        mbar_wait(&q_empty[k & 1], ((k >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[k & 1], 2 * NQ * 128);
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d(sQ + (k & 1) * C::QB + hf * C::QHALF, &tmap_q, &q_full[k & 1], hf * 64, 0, b);
      }
      const int32_t* bt = args.block_table + static_cast<size_t>(b) * args.max_blocks;
      // 16-token page chunks, 32 per warp load of the block table (PPT per tile); chunks past the
      // sequence end (last tile at Hkv < 8) reload its first chunk — masked by the softmax
      auto chunk_tok = [&](int ci) { return ci * 16 < len ? ci * 16 : 0; };
      constexpr int TPB = 32 / PPT;  // tiles per block-table load
      for (int base = t; base < seg_end; base += TPB) {
        const int n = min(TPB, seg_end - base);
        int page = 0;
        if (lane < n * PPT) page = __ldg(bt + chunk_tok((base - tile0) * PPT + lane) / bs);
        // lane l holds the page of chunk l of this batch and issues its boxes itself: PPT lanes
        // issue a tile's PPT chunks at once (at Hkv = 1 a tile is 8 pages x 2 boxes per operand —
        // one issuing thread was the bottleneck)
        const int my_tok = chunk_tok((base - tile0) * PPT + lane);
        const int my_row = page * bs + (my_tok & (bs - 1));
        for (int j = 0; j < n; ++j) {
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++it) {
            const int slot = it % NSTAGE;
            uint8_t* dst = sKV + slot * C::SLOT;
            const CUtensorMap* map = kv ? &tmap_v : &tmap_k;
            if (lane == 0) {
              mbar_wait(&kv_empty[slot], ((it / NSTAGE) & 1) ^ 1);
              mbar_arrive_expect_tx(&kv_full[slot], C::SLOT);
            }
            __syncwarp();  // the slot is free before any lane's TMA writes into it
            const int pc = lane - j * PPT;
            if (pc >= 0 && pc < PPT) {
              uint8_t* d = dst + pc * 16 * HKV * 128;  // rows (chunk, head, token) of 128 B per half
              tma_load_3d_hint(d, map, &kv_full[slot], 0, my_row, 0, stream_once);
              if (!FP8) tma_load_3d_hint(d + C::HALF, map, &kv_full[slot], 64, my_row, 0, stream_once);
            }
          }
        }
      }
      t = seg_end;
    }
  } else if (warp == C::MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer (whole warp, one elected lane issues)
    {
      constexpr uint32_t IDESC_QK =
          FP8 ? idesc_e4m3_f32(C::ROWS, NT * NP, false, false) : idesc_bf16_f32(C::ROWS, NP, false, false);
      constexpr uint32_t IDESC_PV =
          FP8 ? idesc_e4m3_f32(D, NT * NP, true, false) : idesc_bf16_f32(D, NP, true, false);
      const uint64_t k_desc = sdesc_sw128(smem_u32(sKV), 16, 1024);
      const uint64_t v_desc = sdesc_sw128(smem_u32(sKV), FP8 ? 16 : C::HALF, 1024);
      const uint64_t q_desc = sdesc_sw128(smem_u32(FP8 ? sQ8 : sQ), 16, 1024);
      const uint64_t p_desc = sdesc_sw128(smem_u32(sP), 16, 1024);
      auto qk = [&](int i, int qb) {
        const int idx = 2 * i, slot = idx % NSTAGE;
        mbar_wait(&kv_full[slot], (idx / NSTAGE) & 1);
        tc_fence_after();
        const uint64_t kb = k_desc + ((slot * C::SLOT) >> 4);
        if constexpr (FP8) {
          // K = 32 bytes per step along the 128-byte rows of K and of [Q_hi; Q_lo]
          umma_f8_ss_k128<2, 2>(tmem + C::S_COL(i), kb, q_desc + ((qb * C::Q8B) >> 4), IDESC_QK, 0u);
        } else {
          umma_ss_k128<2, C::HALF / 16, 2, C::QHALF / 16>(tmem + C::S_COL(i), kb, q_desc + ((qb * C::QB) >> 4),
                                                          IDESC_QK, 0u);
        }
        umma_commit_w(&s_full[i & 1]);
        umma_commit_w(&kv_empty[slot]);
      };
      // PV of tile i accumulates into segment seg's O buffer (fresh on the segment's first tile,
      // which first waits for the epilogue of segment seg-2 to release the buffer)
      auto pv = [&](int i, int seg, bool first) {
        const int idx = 2 * i + 1, slot = idx % NSTAGE;
        mbar_wait(&kv_full[slot], (idx / NSTAGE) & 1);
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        if (first && seg >= 2) mbar_wait(&o_empty[seg & 1], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint64_t vb = v_desc + ((slot * C::SLOT) >> 4), pb = p_desc + (((i & 1) * C::PB) >> 4);
        if constexpr (FP8) {
          // V^T is the MN-major A operand: 32 (head, token) rows = 4096 B per K step
          umma_f8_ss_k128<((32 * 128) >> 4), 2>(tmem + C::O_COL(seg), vb, pb, IDESC_PV, first ? 0u : 1u);
        } else {
          umma_ss_k128<128, 512, 2, C::PHALF / 16>(tmem + C::O_COL(seg), vb, pb, IDESC_PV, first ? 0u : 1u);
        }
        umma_commit_w(&o_full[i & 1]);  // PV(i) lands: o_full[i & 1], phase (i >> 1) & 1
        umma_commit_w(&kv_empty[slot]);
      };
      // Order: QK(i) then PV(i-1) inside a segment (the softmax of tile i overlaps PV(i-1)); at a
      // segment boundary the previous segment's last PV goes first, so its epilogue never waits on
      // the next segment's Q (which, for fp8, the softmax warps themselves prepare).
      int i = 0, k = 0, b = b_first, pk = 0;
      bool pfirst = false;
      for (int t = T0; t < T1; ++k) {
        while (cu[b + 1] <= t) ++b;
        const int seg_end = min(T1, cu[b + 1]), seg_t0 = t;
        if (i >= 1) pv(i - 1, pk, pfirst);
        mbar_wait(FP8 ? &q_conv[k & 1] : &q_full[k & 1], (k >> 1) & 1);
        for (; t < seg_end; ++t, ++i) {
          qk(i, k & 1);
          if (t == seg_end - 1) umma_commit_w(&q_empty[k & 1]);
          if (t != seg_t0) pv(i - 1, pk, pfirst);
          pk = k;
          pfirst = (t == seg_t0);
        }
      }
      pv(i - 1, pk, pfirst);
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    // O^T accumulates in TMEM across a segment's tiles (PV with acc = 1).  Exponentials use the
    // running max m_run, which only moves when a score exceeds it by more than LAZY (log2 units,
    // FA4's lazy rescale): then, and on a segment's first tile, the CTA takes the slow path —
    // exact per-head max (16-lane shuffles), alpha to smem, and once PV(i-1) has landed every
    // thread rescales its O^T row in TMEM.  The common tile is a vote, G exp2 and G P stores.
    const int row = threadIdx.x;  // S^T row ((chunk*Hkv + head)*16 + token) and O^T row (d)
    const int grp = row >> 4, t16 = row & 15;
    const int h = grp % HKV, pch = grp / HKV;  // kv head, page chunk within the tile
    const bool upper = (lane >> 4) != 0;
    const uint32_t lane_base = static_cast<uint32_t>(warp << 5) << 16;
    const uint32_t col_base = static_cast<uint32_t>(((2 * warp) % HKV) * G);
    const float sl2 = args.scale_log2;
    const uint32_t p_base = smem_u32(sP) + (row >> 6) * C::PHALF + (row & 7) * 2;  // bf16 P^T
    const int rchunk = (row & 63) >> 3;
    volatile int* flags = reinterpret_cast<volatile int*>(alpha_s + NP);  // [2][4] per-warp votes
    constexpr float LAZY = C::LAZY;

    float m_run[G], l_part[G], fac[G];
    int i = 0, b = b_first;
    for (int t = T0, k = 0; t < T1; ++k) {
      while (cu[b + 1] <= t) ++b;
      const int seg_end = min(T1, cu[b + 1]);
      const int tile0 = cu[b];
      const int len = args.seq_lens[b];
      const bool complete = (t == tile0) && (seg_end == cu[b + 1]);
      if constexpr (FP8) {
        // ---- Q (bf16, SW128 halves) -> [Q_hi; Q_lo] e4m3 rows, scaled per q head by 2^e so the
        // largest |q| lands in [128, 256); TPR threads per q head, 8-element chunks
        constexpr int TPR = 128 / NQ, CPT = 16 / TPR;  // threads per row, 8-wide chunks per thread
        mbar_wait(&q_full[k & 1], (k >> 1) & 1);
        const int qh = row / TPR, part = row % TPR;
        const uint8_t* qsrc = sQ + (k & 1) * C::QB;
        uint8_t* qdst = sQ8 + (k & 1) * C::Q8B;
        uint4 v[CPT];
        float amax = 0.f;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int ch = part * CPT + c;  // 8-element chunk of the 128-wide row: half ch/8, chunk ch%8
          v[c] = *reinterpret_cast<const uint4*>(qsrc + (ch >> 3) * C::QHALF + qh * 128 +
                                                  (((ch & 7) ^ (qh & 7)) << 4));
          const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            amax = fmaxf(amax, fmaxf(fabsf(__uint_as_float(w[e] << 16)), fabsf(__uint_as_float(w[e] & 0xFFFF0000u))));
        }
#pragma unroll
        for (int off = 1; off < TPR; off <<= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
        // power-of-two scale: exact, max |q| * qs in [128, 256)
        const float qscale = amax > 0.f ? exp2f(7.f - floorf(__log2f(amax))) : 1.f;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int ch = part * CPT + c, col = ch * 8;
          const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
          uint16_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            e4m3_split2(__uint_as_float(w[e] << 16) * qscale, __uint_as_float(w[e] & 0xFFFF0000u) * qscale, hi[e],
                        lo[e]);
          const uint2 hv = make_uint2(hi[0] | (uint32_t(hi[1]) << 16), hi[2] | (uint32_t(hi[3]) << 16));
          const uint2 lv = make_uint2(lo[0] | (uint32_t(lo[1]) << 16), lo[2] | (uint32_t(lo[3]) << 16));
          *reinterpret_cast<uint2*>(qdst + sw128_b(qh, col)) = hv;
          *reinterpret_cast<uint2*>(qdst + sw128_b(NP + qh, col)) = lv;
        }
        if (part == 0) qs_s[(k & 1) * NP + qh] = 1.f / qscale;
        fence_proxy_async_smem();
        mbar_arrive(&q_conv[k & 1]);
        named_bar_sync(1, 128);  // qs_s visible
#pragma unroll
        for (int g = 0; g < G; ++g) fac[g] = sl2 * qs_s[(k & 1) * NP + h * G + g];
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g) fac[g] = sl2;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        m_run[g] = -INFINITY;
        l_part[g] = 0.f;
      }
      const int seg_i0 = i;
      for (; t < seg_end; ++t, ++i) {
        const int sb = i & 1;
        mbar_wait(&s_full[sb], (i >> 1) & 1);
        // every phase of o_full is observed (compute-sanitizer synccheck): PV(i-2) was issued before
        // QK(i) and tcgen05 ops complete in order, so the phase is complete; probed here, waited on
        // (never in practice) before P(i) is handed over, while PV(i) cannot have been issued
        const bool of_seen = i < 2 || mbar_test(&o_full[(i - 2) & 1], ((i - 2) >> 1) & 1);
        tc_fence_after();
        DTRACE(2, row == 0 && i == 0);
        const int tok = (t - tile0) * C::TT + pch * 16 + t16;
        const bool valid = tok < len;
        float x[G];
        bool need = false;
        {
          constexpr int WC = C::WCOLS, UO = WC - G;  // upper half-warp's column offset (0 at Hkv = 1)
          uint32_t sv[WC];
          tmem_ld_cols<WC>(tmem + lane_base + C::S_COL(i) + col_base, sv);
          if constexpr (FP8) {
            uint32_t sl[WC];
            tmem_ld_cols<WC>(tmem + lane_base + C::S_COL(i) + NP + col_base, sl);
#pragma unroll
            for (int g = 0; g < G; ++g)
              x[g] = valid ? fmaf(__uint_as_float(upper ? sl[UO + g] : sl[g]), 0.0625f,
                                  __uint_as_float(upper ? sv[UO + g] : sv[g])) * fac[g]
                           : -INFINITY;
          } else {
#pragma unroll
            for (int g = 0; g < G; ++g) x[g] = valid ? __uint_as_float(upper ? sv[UO + g] : sv[g]) * fac[g] : -INFINITY;
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) need |= x[g] > m_run[g] + LAZY;
        const bool warp_need = __any_sync(0xffffffffu, need);
        if (lane == 0) flags[sb * 4 + warp] = warp_need;
        named_bar_sync(1, 128);
        if (flags[sb * 4 + 0] | flags[sb * 4 + 1] | flags[sb * 4 + 2] | flags[sb * 4 + 3]) {
          // slow path (CTA-uniform): exact head maxima, rescale factors, O rescale
          float mts[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            float mt = x[g];
#pragma unroll
            for (int off = 1; off < 16; off <<= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
            mts[g] = mt;
          }
          if constexpr (PPT > 1) {  // a head spans PPT 16-row groups (one per page chunk)
            if (t16 == 0)
#pragma unroll
              for (int g = 0; g < G; ++g) grp_s[grp * G + g] = mts[g];
            named_bar_sync(1, 128);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              float m = grp_s[h * G + g];
#pragma unroll
              for (int pc = 1; pc < PPT; ++pc) m = fmaxf(m, grp_s[(pc * HKV + h) * G + g]);
              mts[g] = m;
            }
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float mt = mts[g];
            float alpha = 1.f;
            if (mt > m_run[g] + LAZY) {
              alpha = (m_run[g] == -INFINITY) ? 0.f : fast_exp2(m_run[g] - mt);
              m_run[g] = mt;
              l_part[g] *= alpha;
            }
            if (t16 == 0) alpha_s[h * G + g] = alpha;
          }
          named_bar_sync(1, 128);
          if (i > seg_i0) {  // O holds tiles seg_i0 .. i-1: rescale once PV(i-1) has landed
            mbar_wait(&o_full[(i - 1) & 1], ((i - 1) >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int term = 0; term < NT; ++term) {
              uint32_t r[NQ];
              tmem_ld_cols<NQ>(tmem + lane_base + C::O_COL(k) + term * NP, r);
#pragma unroll
              for (int q = 0; q < NQ; ++q) r[q] = __float_as_uint(__uint_as_float(r[q]) * alpha_s[q]);
              tmem_st_cols<NQ>(tmem + lane_base + C::O_COL(k) + term * NP, r);
            }
            tmem_wait_st();
          }
        }
        uint8_t* pt = sP + sb * C::PB;
        if constexpr (FP8) {
          // P^T as [P_hi; P_lo] e4m3 rows (row = q head, column = this thread's (head, token))
#pragma unroll
          for (int g = 0; g < G; g += 2) {
            float p2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const float mu = (m_run[g + u] == -INFINITY) ? 0.f : m_run[g + u];
              p2[u] = (g + u < G) ? fast_exp2(x[g + u] - mu) : 0.f;
              if (g + u < G) l_part[g + u] += p2[u];
            }
            uint16_t hi, lo;
            e4m3_split2(p2[0] * 16.f, p2[1] * 16.f, hi, lo);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (g + u >= G) break;
              const int qh = h * G + g + u;
              pt[sw128_b(qh, row)] = static_cast<uint8_t>(u ? hi >> 8 : hi & 0xFF);
              pt[sw128_b(NP + qh, row)] = static_cast<uint8_t>(u ? lo >> 8 : lo & 0xFF);
            }
          }
        } else {
          const uint32_t pb = p_base + sb * C::PB;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float mu = (m_run[g] == -INFINITY) ? 0.f : m_run[g];
            const float p = fast_exp2(x[g] - mu);  // x = -inf (invalid / masked) -> 0
            l_part[g] += p;
            const int qh = h * G + g;
            const __nv_bfloat16 p16 = __float2bfloat16_rn(p);
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(pb + qh * 128 + ((rchunk ^ (qh & 7)) << 4)),
                         "h"(*reinterpret_cast<const uint16_t*>(&p16))
                         : "memory");
          }
        }
        if (!valid) {
          // the page's tail slots past the sequence end hold arbitrary bytes (NaN included): P = 0
          // there, but 0 * NaN would poison O, so zero this row of the V tile before PV reads it
          const int vidx = 2 * i + 1, vslot = vidx % NSTAGE;
          mbar_wait(&kv_full[vslot], (vidx / NSTAGE) & 1);
          uint4* vr = reinterpret_cast<uint4*>(sKV + vslot * C::SLOT + row * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            vr[c] = make_uint4(0, 0, 0, 0);
            if (!FP8) vr[C::HALF / 16 + c] = make_uint4(0, 0, 0, 0);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        if (!of_seen) mbar_wait(&o_full[(i - 2) & 1], ((i - 2) >> 1) & 1);
        mbar_arrive(&p_full[sb]);
        DTRACE(3, row == 0 && t == T1 - 1);
      }

      // ---- segment epilogue: O^T (TMEM) / l, or the unnormalised partial for K3'
      float lg[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float l = l_part[g];
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
        lg[g] = l;
      }
      if constexpr (PPT > 1) {  // sum the head's PPT groups
        if (t16 == 0)
#pragma unroll
          for (int g = 0; g < G; ++g) grp_s[grp * G + g] = lg[g];
        named_bar_sync(1, 128);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float l = grp_s[h * G + g];
#pragma unroll
          for (int pc = 1; pc < PPT; ++pc) l += grp_s[(pc * HKV + h) * G + g];
          lg[g] = l;
        }
      }
      if (t16 == 0 && pch == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          ml_s[h * G + g] = m_run[g];
          ml_s[NP + h * G + g] = lg[g];
        }
      }
      // last PV of this segment (in-order completion: every earlier PV has landed too).  Per-parity
      // barriers keep the phase unambiguous: PV(i-3) is complete and PV(i+1) cannot be issued yet.
      mbar_wait(&o_full[(i - 1) & 1], ((i - 1) >> 1) & 1);
      tc_fence_after();
      uint32_t r[NQ];
      tmem_ld_cols<NQ>(tmem + lane_base + C::O_COL(k), r);
      if constexpr (FP8) {
        uint32_t rl[NQ];
        tmem_ld_cols<NQ>(tmem + lane_base + C::O_COL(k) + NP, rl);
        // O = (O_hi + O_lo / 16) / 16 (P was scaled by 16)
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          r[q] = __float_as_uint(fmaf(__uint_as_float(rl[q]), 0.0625f, __uint_as_float(r[q])) * 0.0625f);
      }
      tc_fence_before();
      mbar_arrive(&o_empty[k & 1]);
      named_bar_sync(1, 128);  // ml_s visible
      if (complete) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float l = ml_s[NP + q];
          args.o[(static_cast<size_t>(b) * NQ + q) * D + row] =
              __float2bfloat16_rn(l > 0.f ? __uint_as_float(r[q]) * args.out_scale / l : 0.f);
        }
      } else {
        const size_t slot = static_cast<size_t>(blockIdx.x) + b;
#pragma unroll
        for (int q = 0; q < NQ; ++q) args.part_o[(slot * NQ + q) * D + row] = __uint_as_float(r[q]) * args.out_scale;
        if (row < NQ) {
          args.part_ml[(slot * NQ + row) * 2 + 0] = ml_s[row];
          args.part_ml[(slot * NQ + row) * 2 + 1] = ml_s[NP + row];
        }
        DTRACE(4, row == 0 && seg_end == T1);
        if (args.seq_cnt != nullptr) flat_merge_if_last<NQ, NP>(args, r, ml_s, flags, cu, b, ntiles, row);
      }
      DTRACE(5, row == 0 && seg_end == T1);
      named_bar_sync(1, 128);  // ml_s reads done before the next segment's epilogue rewrites it
    }
  }

  if (args.late_trigger) griddep_launch();
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
  DTRACE(6, threadIdx.x == 0);
}

// K3': merge the partial segments of every split sequence (sequences finished inside one CTA
// were already written by it).
// One CTA per (sequence, q head).  Single pass: every warp folds its share of the pieces (piece i
// to warp i mod NW, U pieces' (max, sum) pairs and 512-byte O rows loaded back to back before any
// is folded) into a running (m, l, acc) with the online-softmax rescale, then warp 0 folds the NW
// warp states in warp order — deterministic, so launches are bit-identical.  One dependent L2 round
// trip per U * NW pieces (the earlier max pass -> weights -> rows chain took 3 + nc / 16).  The
// launcher keeps the grid in one wave: (NW, U) = (8, 8) up to one CTA per SM (a 1-sequence x 8k
// decode: 128 pieces per head in 2 rounds), (8, 4) at 4 CTAs per SM, else (4, 1) at 16 CTAs per SM
// (C2's 2048 CTAs; 76 registers at U = 8 had made that two waves, +1.3 us on the step).
constexpr int kFlatMaxCtas = 1024;
template <int NQ, int NW, int U, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) flat_combine_kernel(const float* __restrict__ part_o,
                                                                     const float* __restrict__ part_ml,
                                                                     const int32_t* __restrict__ cu, int batch,
                                                                     int ctas, __nv_bfloat16* __restrict__ o) {
  __shared__ float ml_w[NW][2];
  __shared__ float4 acc_w[NW][32];
  __shared__ uint8_t own_s[kFlatMaxCtas];
  const int b = blockIdx.x, q = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  griddep_wait();  // PDL: K2' (the predecessor) has completed and its partials are visible
  griddep_launch();
  const int ts = cu[b], te = cu[b + 1], n = cu[batch];
  __nv_bfloat16* out = o + (static_cast<size_t>(b) * NQ + q) * 128;
  if (ts == te) {
    if (tid < 64) reinterpret_cast<uint32_t*>(out)[tid] = 0u;
    return;
  }
  const int c0 = flat_cta_of(ts, ctas, n), c1 = flat_cta_of(te - 1, ctas, n);
  if (c0 == c1) return;  // K2' wrote this sequence's output itself
  const int nc = c1 - c0 + 1;
  // CTAs whose range is empty (fewer tiles than CTAs) wrote nothing: their slots are skipped
  // (flags computed once, one piece per thread, off the load chain)
  for (int i = tid; i < nc; i += NW * 32) {
    const long long c = c0 + i;
    own_s[i] = (c * n / ctas != (c + 1) * n / ctas) ? 1 : 0;
  }
  __syncthreads();
  float m = -INFINITY, l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = warp; i0 < nc; i0 += NW * U) {
    float mp[U], lp[U];
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * NW;
      mp[u] = -INFINITY;
      lp[u] = 0.f;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < nc && own_s[i]) {
        const size_t slot = (static_cast<size_t>(c0 + i) + b) * NQ + q;
        mp[u] = __ldcg(part_ml + slot * 2);
        lp[u] = __ldcg(part_ml + slot * 2 + 1);
        v[u] = __ldcg(reinterpret_cast<const float4*>(part_o + slot * 128) + lane);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float mn = fmaxf(m, mp[u]);
      if (mn == -INFINITY) continue;
      const float wa = fast_exp2(m - mn), wb = fast_exp2(mp[u] - mn);
      l = fmaf(l, wa, lp[u] * wb);
      acc.x = fmaf(acc.x, wa, v[u].x * wb);
      acc.y = fmaf(acc.y, wa, v[u].y * wb);
      acc.z = fmaf(acc.z, wa, v[u].z * wb);
      acc.w = fmaf(acc.w, wa, v[u].w * wb);
      m = mn;
    }
  }
  if (lane == 0) {
    ml_w[warp][0] = m;
    ml_w[warp][1] = l;
  }
  acc_w[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) M = fmaxf(M, ml_w[w][0]);
    float L = 0.f;
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if (ml_w[w][0] == -INFINITY) continue;
      const float s = fast_exp2(ml_w[w][0] - M);
      const float4 a = acc_w[w][lane];
      L = fmaf(ml_w[w][1], s, L);
      r.x = fmaf(a.x, s, r.x);
      r.y = fmaf(a.y, s, r.y);
      r.z = fmaf(a.z, s, r.z);
      r.w = fmaf(a.w, s, r.w);
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(r.x * inv, r.y * inv), hi = __floats2bfloat162_rn(r.z * inv, r.w * inv);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(out + 4 * lane) = pk;
  }
}

}  // namespace b200
