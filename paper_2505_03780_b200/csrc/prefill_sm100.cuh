// prefill_sm100.cuh — K1: causal varlen flash-attention forward (prefill), sm_100a.
//
// Semantics (restated in oracle/attn_oracle.c, the checker):
//   for every sequence s (tokens cu_seqlens[s] .. cu_seqlens[s+1]) and q head h,
//   O[t,h,:] = softmax_j( scale * Q[t,h,:].K[j,h/G,:] , j <= t if causal ) . V[j,h/G,:]
// i.e. FlashAttention-2 forward with GQA (G = Hq/Hkv), the kernel family the paper tunes
// (ref/PAPER.md:108-113; knob names from ref/pkg/src/ktune/fixtures/flash_attention.space.json:3-16).
//
// Work item = one 128-row query block of one sequence for NQ (1 or 2) q heads of the SAME kv
// head, so every K/V tile loaded by TMA feeds NQ x (QK^T + PV) tcgen05 MMAs.  Items are laid
// out by prefill_schedule_kernel in longest-first order (causal cost = q block index + 1) and
// pulled by persistent CTAs (one per SM) from an atomic counter.
//
//   warps 0..W-1    : softmax warps (W = 4*NQ*SPLIT), SPLIT per TMEM lane quadrant of each Q
//                     tile; a thread owns a query row (TMEM lane), or half of it when SPLIT = 2;
//                     they also run the epilogue (O -> bf16 -> global) of their tile
//   warp  W         : scheduler + TMA producer (Q once per item, then K_j / V_j into a ring)
//   warp  W+1       : TMEM allocator + single-thread tcgen05.mma issuer
//   warps W+2, W+3  : idle padding of the producer warpgroup when it hands registers to the
//                     softmax warps (setmaxnreg, REG_SPLIT)
//
// TMEM (512 cols): S_t at [128 t], O_t at [256 + 128 t].  P_t (bf16 pairs) is written back into
// the first BN/2 columns of S_t (each thread overwrites only S values it has already read) and PV
// is a TS MMA (A = P from TMEM, B = V as MN-major SW128 straight from its TMA tile), so P never
// touches shared memory and the freed 64 KB deepen the K/V ring.  tcgen05.mma ops of the issuing
// thread execute in order, so QK_t(j+1) cannot overwrite P_t(j) before PV_t(j) has read it.
// Softmax: a thread owns a whole S row; pass 1 takes the row max straight from TMEM, pass 2
// recomputes exp2(s*scale*log2e - m) — one element in EMU through a degree-3 polynomial on the
// FMA pipe, the rest on MUFU — and stores P.  O is rescaled lazily (only when the running max
// grows by more than 8 in log2 units), which keeps the result exact.
#pragma once
#include "sm100_common.cuh"

namespace b200 {

struct PrefillKernelArgs {
  const int32_t* cu_seqlens;
  const int32_t* items;  // [n_pairs] (seq << 16) | q block, longest first
  int32_t* sched;        // [0] = work counter (atomic), [1] = n_pairs, [2] = CTAs done
  __nv_bfloat16* o;
  float* lse;  // optional [Hq, T]
  int32_t total_tokens;
  int32_t num_q_heads;
  int32_t group;  // Hq / Hkv
  int32_t causal;
  int32_t num_hg;    // Hq / NQ head groups per (seq, q block)
  int32_t single_nqb;  // > 0: uniform batch — `useqs` sequences of this many q blocks each (one
                       // sequence, or equal lengths): no schedule kernel, items are decoded
                       // analytically, q blocks longest first across the sequences
  int32_t useqs;
  float scale_log2;  // softmax_scale * log2(e)
  int32_t speculate;  // 1: interior tiles take the single-pass path against the running max
  // L2-aware order (band > 0; problems whose K/V exceeds ~half of L2): q blocks are taken in bands
  // of `band` blocks, longest band first; inside a band by (sequence, kv head), q block descending,
  // so the CTAs in flight share a few (sequence, kv head) K/V streams instead of all of them.
  // items then holds 2 ints per entry: (seq << 16) | q block, kv head; an entry expands to `hpk`
  // work items (the head groups of that kv head).
  int32_t band;
  int32_t hpk;  // head groups per kv head (num_hg / Hkv)
};

// SPLIT = softmax warps per TMEM lane quadrant (num_warps / 4): with SPLIT = 2 two threads share
// an S row, each owning BN / 2 columns — two warps per SMSP per tile.  In isolation that is the
// faster layout (a 128-column slice: 1053 cycles on two warps vs 1139 on one,
// scripts/probes/softmax_probe.cu); inside the kernel the tile softmax did not get shorter, and the
// sweep picks SPLIT = 2 only for some small shapes (DESIGN.md §4 K1).
// PAIR (waves_per_eu = 2): the work item runs on a CTA pair (2-CTA cluster, cta_group::2).  Each
// CTA keeps its own NQ Q tiles (heads rank*NQ + t of the item's 2*NQ) and loads HALF of every K
// tile (keys rank*BN/2 ..) and HALF of every V tile (d columns rank*64 ..); one M = 256 MMA of the
// leader reads B once for both CTAs' Q tiles, so per CTA a K=16 QK^T step reads 4 KB of Q + 2 KB of
// K in 64 cycles (96 B/clk) instead of 8 KB (128 B/clk, the shared-memory ceiling).
template <int NQ, int BN, int NSTAGE_CFG, int SPLIT = 1, bool PAIR = false>
struct PrefillCfg {
  static constexpr int D = 128;
  static constexpr int BM = 128;
  static constexpr int NCOL = BN / SPLIT;                    // S columns per softmax thread
  static constexpr int KV_BYTES = PAIR ? BN * D : BN * D * 2;  // one K or V tile (per CTA)
  static constexpr int NSLOT = (NSTAGE_CFG + 1) * 32768 / KV_BYTES;  // ring = (num_stages + 1) x 32 KB
  static constexpr int NUM_SOFTMAX_WARPS = 4 * NQ * SPLIT;
  static constexpr int TILE_THREADS = 128 * SPLIT;           // softmax threads per Q tile
  static constexpr int TMA_WARP = NUM_SOFTMAX_WARPS;
  static constexpr int MMA_WARP = NUM_SOFTMAX_WARPS + 1;
  static constexpr int Q_BYTES = BM * D * 2;   // 32 KB per Q tile (2 SW128 halves)
  static constexpr int HALF_Q = BM * 128;
  static constexpr int HALF_KV = BN * 128;     // V: offset of the second 64-column d block (unpaired)
  static constexpr int HALF_K = PAIR ? (BN / 2) * 128 : BN * 128;  // K: offset of the second d half
  // consumer arrivals on the leader's barriers: its own threads arrive locally, the peer's warps
  // arrive remotely, one per warp
  static constexpr int ARRIVE_P = PAIR ? TILE_THREADS + 4 : TILE_THREADS;  // p_full / o_free per tile
  static constexpr int ARRIVE_ITEM_BASE = PAIR ? 2 + TILE_THREADS * NQ + 4 * NQ : 1 + TILE_THREADS * NQ;
  static_assert(!PAIR || (SPLIT == 1 && BN == 128), "CTA pair: 4 softmax warps per tile, BLOCK_N = 128");
  // Q is double-buffered when the ring leaves room: the next item's Q lands during this item
  // SPLIT = 2: per-row exchange of half-row maxima (by step parity) and half-row sums
  static constexpr int XCH_FLOATS = (SPLIT > 1) ? 3 * NQ * SPLIT * 128 : 0;
  static constexpr int QBUF = (2 * NQ * Q_BYTES + (NSTAGE_CFG + 1) * 32768 + XCH_FLOATS * 4 <= 229376) ? 2 : 1;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + QBUF * NQ * Q_BYTES;
  static constexpr int OFF_ITEM = OFF_KV + NSLOT * KV_BYTES;  // int32[2] work-item mailbox, +16: O-store mailbox
  static constexpr int OFF_XCH = OFF_ITEM + 32;
  static constexpr int OFF_BAR = OFF_XCH + XCH_FLOATS * 4;
  // S_t is double-buffered when TMEM has room (NQ = 2 with BLOCK_N = 64, or NQ = 1): QK_t then runs
  // two KV steps ahead of PV_t, so the softmax of step j+1 never waits for PV_t(j) + QK_t(j+1)
  static constexpr int SB = (NQ * 2 * BN + NQ * 128 <= 512) ? 2 : 1;  // S buffers per tile
  static constexpr int LA = SB;                                       // QK lookahead (KV steps)
  // q_full[2], q_empty[2], kv_full/empty[NSLOT], s_full[NQ][SB], p_full[NQ][2], o_done[NQ][2],
  // o_free[NQ], item_full/empty[2], drain, stage_full, stage_free
  static constexpr int NUM_BARS = 4 + 2 * NSLOT + NQ * SB + 2 * NQ + 2 * NQ + NQ + 4 + 1 + 2;
  // O epilogue through TMA stores (when 32 KB of shared memory are left): a tile's softmax threads
  // write their rows of O (bf16, SW128 layout of two {64 d, 1 head, 128 tokens} boxes) into one
  // staging buffer and a store warp issues the two TMA stores; the tiles take turns on the buffer.
  // Blocks that end past their sequence (the last q block) are written row by row instead.
  static constexpr int OFF_STAGE = (OFF_BAR + NUM_BARS * 8 + 16 + 1023) & ~1023;
  // Enabled for the two-threads-per-row variants (num_warps = 8) only: A/B on one box (r2r), 16x2k
  // 563 -> 535 us with BLOCK_M = 256, num_warps = 8; with one thread per row the staged epilogue
  // cost C3 3.5% and C1 4% (the tiles queue on the one staging buffer, the store warp's hand-off
  // lengthens C1's latency chain, and the extra code spills in the NQ = 2 kernel).
  static constexpr bool STAGE_O = !PAIR && SPLIT == 2 && OFF_STAGE + BM * D * 2 + 1024 <= 232448;
  static constexpr int SMEM_BYTES = STAGE_O ? OFF_STAGE + BM * D * 2 + 1024 : OFF_BAR + NUM_BARS * 8 + 16 + 1024;
  static constexpr int ARRIVE_ITEM = ARRIVE_ITEM_BASE + (STAGE_O ? 1 : 0);  // + the store warp
  // Registers: the register file is split per SMSP (16K each) and warp w runs on SMSP w % 4, so
  // each SMSP holds NQ * SPLIT softmax warps + one producer-side warp.  When that leaves the softmax
  // warps short of registers, the producer side is padded to a full warpgroup (TMA, MMA, 2 idle
  // warps) that gives its registers to the softmax warpgroups with setmaxnreg.
  static constexpr int SM_PER_SMSP = NQ * SPLIT;
  static constexpr bool REG_SPLIT = SM_PER_SMSP == 2;  // at 4 per SMSP ptxas cannot fit the softmax in 120
  // + a store warp (STAGE_O): the producer warpgroup's first idle warp, or one more warp
  static constexpr int STORE_WARP = NUM_SOFTMAX_WARPS + 2;
  static constexpr int NTHREADS = 32 * (NUM_SOFTMAX_WARPS + (REG_SPLIT ? 4 : (STAGE_O ? 3 : 2)));
  // setmaxnreg moves registers within the CTA's launch allocation (NTHREADS x the launch-bound
  // count, 65536 / NTHREADS rounded down to 8); an .inc beyond what the .dec warps released blocks
  // forever, so the softmax count is derived from that pool
  static constexpr int REG_LAUNCH = ((65536 / NTHREADS) & ~7) > 255 ? 248 : ((65536 / NTHREADS) & ~7);
#ifndef B200_PREFILL_REG_OTHER
#define B200_PREFILL_REG_OTHER 64
#endif
  static constexpr int REG_OTHER = B200_PREFILL_REG_OTHER;  // producer-warpgroup registers
  static constexpr int REG_SOFTMAX_RAW = ((NTHREADS * REG_LAUNCH - 128 * REG_OTHER) / (32 * NUM_SOFTMAX_WARPS)) & ~7;
  static constexpr int REG_SOFTMAX = REG_SOFTMAX_RAW > 248 ? 248 : REG_SOFTMAX_RAW;
  static_assert(!REG_SPLIT || (REG_SOFTMAX >= REG_LAUNCH &&
                               32 * NUM_SOFTMAX_WARPS * REG_SOFTMAX + 128 * REG_OTHER <= NTHREADS * REG_LAUNCH),
                "setmaxnreg split exceeds the launch allocation");

  static constexpr uint32_t TMEM_COLS = 512;
  __host__ __device__ static constexpr uint32_t S_COL(int t, int b) { return (t * SB + b) * BN; }
  __host__ __device__ static constexpr uint32_t O_COL(int t) { return NQ * SB * BN + t * 128; }
  static_assert(BN == 64 || BN == 128, "BLOCK_N in {64,128}");
  static_assert(SPLIT == 1 || (SPLIT == 2 && BN == 128), "two threads per row need 64-column halves");
};

// 2^x on the FMA pipe (x <= 0): round-to-nearest split x = n + f, f in [-0.5, 0.5], degree-3
// minimax for 2^f (max rel err 7.5e-5, far below bf16's 3.9e-3), n added to the exponent field.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -126.0f);
  const float shifter = 12582912.0f;  // 1.5 * 2^23: x + shifter rounds x to an integer in the mantissa
  const float t = x + shifter;
  const float n = t - shifter;
  const float f = x - n;
  float p = fmaf(0.05517027899622917f, f, 0.2426076978445053f);
  p = fmaf(p, f, 0.693260908126831f);
  p = fmaf(p, f, 0.9999282956123352f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Pair version on FFMA2/FADD2: ~5 issue slots per element instead of one MUFU.EX2 (8 MUFU-pipe
// cycles per warp instruction), so a fraction of the exponentials can move off the MUFU pipe.
// HI_CLAMP (speculative pass, x may be > 0): clamp at 126 so a huge x gives a huge finite value
// (like MUFU's inf, it trips the row-sum check) instead of wrapping the exponent field.
template <bool HI_CLAMP = false>
__device__ __forceinline__ void exp2_poly2(float x0, float x1, float& y0, float& y1) {
  x0 = fmaxf(x0, -126.0f);
  x1 = fmaxf(x1, -126.0f);
  if constexpr (HI_CLAMP) {
    x0 = fminf(x0, 126.0f);
    x1 = fminf(x1, 126.0f);
  }
  const float shifter = 12582912.0f;
  float t0, t1, n0, n1;
  ffma2(t0, t1, x0, x1, 1.0f, shifter);
  ffma2(n0, n1, t0, t1, 1.0f, -shifter);
  float f0, f1;
  ffma2(f0, f1, n0, n1, -1.0f, 0.0f);
  fadd2(f0, f1, x0, x1);  // f = x - n
  float p0 = 0.05517027899622917f, p1 = 0.05517027899622917f;
  float q0, q1;
  ffma2_v(q0, q1, p0, p1, f0, f1, 0.2426076978445053f);
  ffma2_v(p0, p1, q0, q1, f0, f1, 0.693260908126831f);
  ffma2_v(q0, q1, p0, p1, f0, f1, 0.9999282956123352f);
  y0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ void prefill_decode_item(int w, const PrefillKernelArgs& a, int& seq, int& qblk,
                                                    int& hg) {
  if (a.band > 0) {
    if (a.single_nqb > 0) {  // bands from the top q block down (all but the last are full); inside a
                             // band by sequence, kv head, q block descending
      const int per_band = a.band * a.useqs * a.num_hg;
      const int i = w / per_band;
      const int r = w - i * per_band;
      const int nq = min(a.band, a.single_nqb - i * a.band);
      const int per_seq = nq * a.num_hg;
      seq = r / per_seq;
      const int r1 = r - seq * per_seq;
      const int per_kvh = nq * a.hpk;
      const int kvh = r1 / per_kvh;
      const int r2 = r1 - kvh * per_kvh;
      const int e = r2 / a.hpk;
      qblk = a.single_nqb - 1 - i * a.band - e;
      hg = kvh * a.hpk + (r2 - e * a.hpk);
    } else {
      const int e = w / a.hpk;
      const uint32_t it = static_cast<uint32_t>(a.items[2 * e]);
      seq = static_cast<int>(it >> 16);
      qblk = static_cast<int>(it & 0xFFFFu);
      hg = a.items[2 * e + 1] * a.hpk + (w - e * a.hpk);
    }
    return;
  }
  const int pair = w / a.num_hg;
  hg = w - pair * a.num_hg;
  if (a.single_nqb > 0) {  // uniform batch: q block index descending, sequences minor
    if (a.useqs == 1) {      // one sequence (no integer division on the latency-bound path)
      seq = 0;
      qblk = a.single_nqb - 1 - pair;
      return;
    }
    const int r = pair / a.useqs;
    seq = pair - r * a.useqs;
    qblk = a.single_nqb - 1 - r;
    return;
  }
  const uint32_t it = static_cast<uint32_t>(a.items[pair]);  // (seq << 16) | q block, seq < 65536
  seq = static_cast<int>(it >> 16);
  qblk = static_cast<int>(it & 0xFFFFu);
}

// Pass 2 over one S row: P = exp2(S*sl2 - m) -> bf16 pairs written back over the S columns;
// returns the row sum.  MASKED is a compile-time split so the common (interior) tile carries no
// per-element compare/select at all — predicated-off instructions still cost issue slots.
template <int BN, bool MASKED, int EMU>
__device__ __forceinline__ float softmax_pass2(uint32_t s_addr, float sl2, float nmu, int kv0, int lim) {
  // four independent FADD2 accumulators: a single running sum is a 64-deep dependent chain;
  // 32-column chunks with the next chunk's tcgen05.ld in flight (P of chunk c lands on S
  // columns [16c, 16c + 16), all of which were loaded before)
  float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t r[2][32];
  tmem_ld32_nowait(s_addr, r[0]);
  tmem_wait_ld_regs(r[0]);
#pragma unroll
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t(&cur)[32] = r[c & 1];
    if (c + 1 < BN / 32) tmem_ld32_nowait(s_addr + (c + 1) * 32, r[(c + 1) & 1]);
    uint32_t pk[16];
    const int col0 = kv0 + c * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      float x0, x1;
      ffma2(x0, x1, __uint_as_float(cur[i]), __uint_as_float(cur[i + 1]), sl2, nmu);
      float e0, e1;
      if constexpr (!MASKED && EMU > 0) {
        if ((i >> 1) % EMU == EMU - 1) {
          exp2_poly2(x0, x1, e0, e1);
        } else {
          e0 = fast_exp2(x0);
          e1 = fast_exp2(x1);
        }
      } else {
        e0 = fast_exp2(x0);
        e1 = fast_exp2(x1);
      }
      if constexpr (MASKED) {
        if (col0 + i > lim) e0 = 0.f;
        if (col0 + i + 1 > lim) e1 = 0.f;
      }
      const int acc = ((i >> 1) & 3) * 2;
      fadd2(ls[acc], ls[acc + 1], e0, e1);
      pk[i >> 1] = pack_bf16x2(e0, e1);
    }
    if (c + 1 < BN / 32) tmem_wait_ld_regs(r[(c + 1) & 1]);
    tmem_st16(s_addr + c * 16, pk);  // P overwrites S columns this thread has already read
  }
  fadd2(ls[0], ls[1], ls[2], ls[3]);
  fadd2(ls[4], ls[5], ls[6], ls[7]);
  fadd2(ls[0], ls[1], ls[4], ls[5]);
  return ls[0] + ls[1];
}

template <int BN, bool MASKED>
__device__ __forceinline__ float softmax_rowmax(uint32_t s_addr, int kv0, int lim) {
  // four independent 3-input max chains (FMNMX3); all chunk loads in flight before one wait
  float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  uint32_t r[2][32];
  tmem_ld32_nowait(s_addr, r[0]);
  tmem_wait_ld_regs(r[0]);
#pragma unroll
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t(&cur)[32] = r[c & 1];
    if (c + 1 < BN / 32) tmem_ld32_nowait(s_addr + (c + 1) * 32, r[(c + 1) & 1]);
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      float a0 = __uint_as_float(cur[i]), a1 = __uint_as_float(cur[i + 1]);
      if constexpr (MASKED) {
        const int ca = kv0 + c * 32 + i;
        if (ca > lim) a0 = -INFINITY;
        if (ca + 1 > lim) a1 = -INFINITY;
      }
      const int k = (i >> 1) & 3;
      m[k] = fmaxf(m[k], fmaxf(a0, a1));
    }
    if (c + 1 < BN / 32) tmem_wait_ld_regs(r[(c + 1) & 1]);
  }
  return fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
}

// Interior tile with a finite running max: exponentials against m_run in ONE pass over S, no max
// at all.  P is bf16 and O, l are fp32, so a stale max only has to keep 2^(s - m_run) finite: P
// stays in registers and is stored unless a row sum passed 2^64 (then, rarely, the caller redoes
// the tile with the exact two-pass path, S still intact in TMEM).  Saves the max pass (a second
// TMEM read, its load latency and 0.5 FMNMX per score) on nearly every tile.
template <int BN, int EMU, int SPLIT>
__device__ __forceinline__ bool softmax_speculative(uint32_t s_addr, float sl2, float m_run, float& lsum,
                                                    uint32_t pair_bar) {
  float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t pk[BN / 2];
  const float nmu = -m_run;
  // 32-column chunks, software-pipelined: chunk c+1's tcgen05.ld is in flight while chunk c is
  // exponentiated, so the TMEM load latency is paid once per tile instead of once per chunk
  uint32_t r[2][32];
  tmem_ld32_nowait(s_addr, r[0]);
  tmem_wait_ld_regs(r[0]);
#pragma unroll
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t(&cur)[32] = r[c & 1];
    if (c + 1 < BN / 32) tmem_ld32_nowait(s_addr + (c + 1) * 32, r[(c + 1) & 1]);
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const int k = (i >> 1) & 3;
      float x0, x1;
      ffma2(x0, x1, __uint_as_float(cur[i]), __uint_as_float(cur[i + 1]), sl2, nmu);
      float e0, e1;
      if (EMU > 0 && (i >> 1) % EMU == EMU - 1) {
        exp2_poly2<true>(x0, x1, e0, e1);
      } else {
        e0 = fast_exp2(x0);
        e1 = fast_exp2(x1);
      }
      fadd2(ls[2 * k], ls[2 * k + 1], e0, e1);
      pk[(c * 32 + i) >> 1] = pack_bf16x2(e0, e1);
    }
    if (c + 1 < BN / 32) tmem_wait_ld_regs(r[(c + 1) & 1]);
  }
  fadd2(ls[0], ls[1], ls[2], ls[3]);
  fadd2(ls[4], ls[5], ls[6], ls[7]);
  fadd2(ls[0], ls[1], ls[4], ls[5]);
  lsum = ls[0] + ls[1];
  const bool ok = m_run != -INFINITY && lsum <= 1.8446744e19f;  // 2^64
  if constexpr (SPLIT == 1) {
    if (!__all_sync(0xffffffffu, ok)) return false;
  } else {
    if (!named_bar_and(pair_bar, 32 * SPLIT, ok)) return false;  // both owners of the rows redo, or neither
  }
#pragma unroll
  for (int g = 0; g < BN / 32; ++g) tmem_st16(s_addr + g * 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + g * 16));
  return true;
}

#ifdef B200_TRACE
// debug-only event trace of CTA 0: [event][slot] clock64 stamps
// event 16: one-off stamps of CTA 0's first item — 0 entry, 1 barriers + TMEM ready, 2 past
// griddepcontrol.wait, 3 MMA warp saw Q, 4 first S seen by row 0, 5 epilogue start, 6 epilogue
// done, 7 exit
__device__ unsigned long long g_trace[17][512];  // 8..11: P done by warp 0..3 of tile 0; 12..15: S seen
#define TRACE(ev, slot)                                                        \
  do {                                                                        \
    if (blockIdx.x == 0 && (slot) < 512) g_trace[ev][slot] = clock64();        \
  } while (0)
// per-CTA %globaltimer stamps of the last two launches (by launch parity): 0 entry, 1 past
// griddepcontrol.wait, 2 work done, 3 exit; g_plaunch counts launches (bumped by the last CTA out)
__device__ unsigned long long g_ptrace[2][1024][8];  // [4], [5]: clock64 at entry / exit (SM clock);
                                                     // [6]: first item, [7]: its epilogue done
__device__ unsigned int g_plaunch;
__device__ __forceinline__ void ptrace(unsigned par, int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 1024) {
    g_ptrace[par & 1][blockIdx.x][ev] = t;
    if (ev == 0) g_ptrace[par & 1][blockIdx.x][4] = clock64();
    if (ev == 3) g_ptrace[par & 1][blockIdx.x][5] = clock64();
  }
}
#define PTRACE(ev)                                            \
  do {                                                        \
    if (threadIdx.x == 0) ptrace(launch_par, ev);             \
  } while (0)
#else
#define PTRACE(ev) \
  do {             \
  } while (0)
#define TRACE(ev, slot) \
  do {                  \
  } while (0)
#endif

template <int NQ, int BN, int NSTAGE_CFG, int EMU, int SPLIT, bool PAIR = false>
__global__ void __launch_bounds__(PrefillCfg<NQ, BN, NSTAGE_CFG, SPLIT, PAIR>::NTHREADS, 1)
    prefill_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_k,
                       const __grid_constant__ CUtensorMap tmap_v, const __grid_constant__ CUtensorMap tmap_o,
                       const PrefillKernelArgs args) {
  using C = PrefillCfg<NQ, BN, NSTAGE_CFG, SPLIT, PAIR>;
  constexpr int D = C::D, BM = C::BM, NS = C::NSLOT, NCOL = C::NCOL;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sKV = smem + C::OFF_KV;
  volatile int32_t* item_box = reinterpret_cast<volatile int32_t*>(smem + C::OFF_ITEM);
  volatile int32_t* stage_box = item_box + 4;  // STAGE_O: {block needs no TMA store, first token, q head}
  uint8_t* sStage = smem + C::OFF_STAGE;
  float* xch = reinterpret_cast<float*>(smem + C::OFF_XCH);  // [3][NQ][SPLIT][128]: max (2 parities), sum
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;       // [2]
  uint64_t* q_empty = bars + 2;  // [2]
  uint64_t* kv_full = bars + 4;
  uint64_t* kv_empty = kv_full + NS;
  uint64_t* s_full = kv_empty + NS;       // [NQ][SB]  QK_t landed in S buffer b
  uint64_t* p_full = s_full + NQ * C::SB;  // [NQ][2]   P_t of a step of that parity written (128 arrivals;
                                           //           per parity: with the QK lookahead the softmax
                                           //           may finish step j+1 before the MMA waited step j)
  uint64_t* o_done = p_full + 2 * NQ;      // [NQ][2]   PV_t of a step of that parity landed
  uint64_t* o_free = o_done + 2 * NQ;      // [NQ]      epilogue of O_t done (128 arrivals)
  uint64_t* item_full = o_free + NQ;       // [2]
  uint64_t* item_empty = item_full + 2;
  uint64_t* drain = item_empty + 2;         // PAIR: the leader's MMA warp waits its last MMAs out
  uint64_t* stage_full = drain + 1;         // STAGE_O: a tile's O rows are in the staging buffer
  uint64_t* stage_free = stage_full + 1;    // STAGE_O: the TMA store has read the staging buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);

  const int warp = warp_id();
  const int lane = lane_id();
  if (threadIdx.x == 0) TRACE(16, 0);
#ifdef B200_TRACE
  const unsigned launch_par = *reinterpret_cast<volatile unsigned*>(&g_plaunch);
#endif
  PTRACE(0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < NQ; ++t) {
      for (int b = 0; b < C::SB; ++b) mbar_init(&s_full[t * C::SB + b], 1);
      mbar_init(&p_full[2 * t], C::ARRIVE_P);
      mbar_init(&p_full[2 * t + 1], C::ARRIVE_P);
      mbar_init(&o_done[2 * t], 1);
      mbar_init(&o_done[2 * t + 1], 1);
      mbar_init(&o_free[t], C::ARRIVE_P);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], C::ARRIVE_ITEM);
    }
    mbar_init(drain, 1);
    mbar_init(stage_full, C::TILE_THREADS);
    mbar_init(stage_free, 1);
    fence_barrier_init();
  }
  if (warp == C::MMA_WARP) {
    if constexpr (PAIR)
      tmem_alloc_pair(tmem_slot, C::TMEM_COLS);  // same warp id in both CTAs, same columns
    else
      tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  if (warp == C::TMA_WARP && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_k);
    tma_prefetch_desc(&tmap_v);
    if constexpr (C::STAGE_O) tma_prefetch_desc(&tmap_o);
  }
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync_all();  // barrier inits of both CTAs visible before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(16, 1);
  // PAIR: cluster rank (0 = leader: scheduler, MMA issuer, owner of the shared barriers);
  // `lead` maps one of this CTA's barriers to the leader's copy (shared::cluster address)
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
  auto lead = [](uint64_t* b) { return mapa_shared(smem_u32(b), 0); };
  // one arrival per thread on the local barrier (the leader's own), one per warp from the peer
  auto arrive_consumer = [&](uint64_t* b) {
    if (PAIR && rank != 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lead(b));
    } else {
      mbar_arrive(b);
    }
  };
  auto wait_cl = [](uint64_t* b, uint32_t par) {  // waits on barriers the peer also arrives on
    if constexpr (PAIR)
      mbar_wait_cluster(b, par);
    else
      mbar_wait_producer(b, par);
  };
  griddep_wait();    // PDL: the prologue above overlapped the previous kernel; data access starts here
  griddep_launch();
  if (threadIdx.x == 0) TRACE(16, 2);
  PTRACE(1);
  // register hand-over (REG_SPLIT): each role adjusts its own limit at the top of its branch, so
  // the allocator never sees a join of the two limits
  auto regs_other = [] {
    if constexpr (C::REG_SPLIT) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::REG_OTHER));
  };

  auto n_kv_of = [&](int seq_len, int qblk) {
    const int kv_end = args.causal ? min(seq_len, qblk * BM + BM) : seq_len;
    return (kv_end + BN - 1) / BN;
  };

  if (warp == C::TMA_WARP) {
    // ------------------------------------------------------------ scheduler + TMA producer
    regs_other();
    if (lane == 0) {
      const int total_work = (args.single_nqb > 0 ? args.single_nqb * args.useqs : args.sched[1]) * args.num_hg;
      const uint64_t keep = policy_evict_last();  // K/V tiles are re-read by other q blocks / heads
      int ri = 0;
      [[maybe_unused]] const uint64_t once = PAIR ? policy_evict_first() : 0;  // PAIR: Q tiles are read once
      for (int k = 0;; ++k) {
        int w;
        if (!PAIR || rank == 0) {
          if (k >= 2) wait_cl(&item_empty[k & 1], ((k >> 1) - 1) & 1);
          w = atomicAdd(args.sched, 1);
          if (w >= total_work) w = -1;
          item_box[k & 1] = w;
          if constexpr (PAIR) {  // the peer's mailbox, then its item_full (release orders the store)
            st_cluster_u32(mapa_shared(smem_u32((const void*)&item_box[k & 1]), 1), static_cast<uint32_t>(w));
            mbar_arrive_cluster(mapa_shared(smem_u32(&item_full[k & 1]), 1));
          }
          mbar_arrive(&item_full[k & 1]);
        } else {
          mbar_wait_cluster(&item_full[k & 1], (k >> 1) & 1);
          w = item_box[k & 1];
          mbar_arrive_cluster(lead(&item_empty[k & 1]));
        }
        if (w < 0) break;
        int seq, qblk, hg;
        prefill_decode_item(w, args, seq, qblk, hg);
        const int seq_start = args.cu_seqlens[seq];
        const int seq_len = args.cu_seqlens[seq + 1] - seq_start;
        const int h0 = hg * NQ * (PAIR ? 2 : 1) + static_cast<int>(rank) * NQ, kvh = h0 / args.group;
        const int n_kv = n_kv_of(seq_len, qblk);
        const int qb = (C::QBUF == 2) ? (k & 1) : 0;
        const uint32_t qph = (C::QBUF == 2) ? ((k >> 1) & 1) : (k & 1);
        mbar_wait_producer(&q_empty[qb], qph ^ 1);
        if constexpr (PAIR) {
          // both CTAs' bytes complete on the leader's barrier; only the leader arms it (a peer
          // transfer landing first leaves the tx-count transiently negative, which is allowed)
          if (rank == 0) mbar_arrive_expect_tx(&q_full[qb], 2 * NQ * C::Q_BYTES);
          const uint32_t fb = lead(&q_full[qb]);
          for (int t = 0; t < NQ; ++t)
            for (int hf = 0; hf < 2; ++hf)
              tma_load_3d_pair(sQ + (qb * NQ + t) * C::Q_BYTES + hf * C::HALF_Q, &tmap_q, fb, hf * 64, h0 + t,
                               seq_start + qblk * BM, once);
        } else {
          mbar_arrive_expect_tx(&q_full[qb], NQ * C::Q_BYTES);
          for (int t = 0; t < NQ; ++t)
            for (int hf = 0; hf < 2; ++hf)
              tma_load_3d(sQ + (qb * NQ + t) * C::Q_BYTES + hf * C::HALF_Q, &tmap_q, &q_full[qb], hf * 64, h0 + t,
                          seq_start + qblk * BM);
        }
        for (int idx = 0; idx < 2 * n_kv; ++idx, ++ri) {
          const int slot = ri % NS;
          mbar_wait_producer(&kv_empty[slot], ((ri / NS) & 1) ^ 1);
          uint8_t* dst = sKV + slot * C::KV_BYTES;
          const int tok0 = seq_start + (idx >> 1) * BN;
          if constexpr (PAIR) {
            // K: this CTA's BN/2 keys (both d halves); V: this CTA's 64 d columns of all BN keys
            if (rank == 0) mbar_arrive_expect_tx(&kv_full[slot], 2 * C::KV_BYTES);
            const uint32_t fb = lead(&kv_full[slot]);
            if ((idx & 1) == 0) {
              for (int hf = 0; hf < 2; ++hf)
                tma_load_3d_pair(dst + hf * C::HALF_K, &tmap_k, fb, hf * 64, kvh,
                                 tok0 + static_cast<int>(rank) * (BN / 2), keep);
            } else {
              tma_load_3d_pair(dst, &tmap_v, fb, static_cast<int>(rank) * 64, kvh, tok0, keep);
            }
          } else {
            const CUtensorMap* map = (idx & 1) ? &tmap_v : &tmap_k;
            mbar_arrive_expect_tx(&kv_full[slot], C::KV_BYTES);
            for (int hf = 0; hf < 2; ++hf)
              tma_load_3d_hint(dst + hf * C::HALF_KV, map, &kv_full[slot], hf * 64, kvh, tok0, keep);
          }
        }
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer (whole warp, one elected lane issues)
    regs_other();
    if (!PAIR || rank == 0) {  // PAIR: the leader issues the M = 256 MMAs for both CTAs
      constexpr uint32_t MM = PAIR ? 2 * BM : BM;
      constexpr uint32_t IDESC_QK = idesc_bf16_f32(MM, BN, false, false);
      constexpr uint32_t IDESC_PV = idesc_bf16_f32(MM, D, false, true);
      // Descriptors are built once; per-MMA addressing is a 16-B-unit add on the start-address
      // field (smem < 256 KB, so the 14-bit field never carries).  Rebuilding 64-bit descriptors
      // per MMA costs the single issuing thread ~120 cycles and starves the tensor pipe.
      const uint64_t q_desc = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t k_desc = sdesc_sw128(smem_u32(sKV), 16, 1024);
      const uint64_t v_desc = sdesc_sw128(smem_u32(sKV), C::HALF_KV, 1024);
      constexpr int SB = C::SB, LA = C::LA;
      int qb = 0;
      auto commit = [](uint64_t* b) {
        if constexpr (PAIR)
          umma_commit_pair_w(b, 3);  // arrives on this barrier in both CTAs
        else
          umma_commit_w(b);
      };
      auto issue_qk = [&](int t, int slot, int buf) {
        const uint64_t qa = q_desc + (((qb * NQ + t) * C::Q_BYTES) >> 4);
        const uint64_t kb = k_desc + ((slot * C::KV_BYTES) >> 4);
        if constexpr (PAIR)
          umma_ss_k128_pair<2, C::HALF_Q / 16, 2, C::HALF_K / 16>(tmem + C::S_COL(t, buf), qa, kb, IDESC_QK, 0u);
        else
          umma_ss_k128<2, C::HALF_Q / 16, 2, C::HALF_KV / 16>(tmem + C::S_COL(t, buf), qa, kb, IDESC_QK, 0u);
      };
      auto issue_pv = [&](int t, int slot, int buf, bool acc) {
        const uint64_t vb = v_desc + ((slot * C::KV_BYTES) >> 4);
        if constexpr (PAIR) {
          umma_ts_k128_pair<128, 512>(tmem + C::O_COL(t), tmem + C::S_COL(t, buf), vb, IDESC_PV, acc ? 1u : 0u);
        } else if constexpr (BN == 128) {
          // SPLIT = 2: P of S columns [64, 128) sits at S column 64 (the second half-row owner's range)
          umma_ts_k128<128, 512, (SPLIT == 2 ? 32 : 0)>(tmem + C::O_COL(t), tmem + C::S_COL(t, buf), vb, IDESC_PV,
                                                       acc ? 1u : 0u);
        } else {
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            umma_ts_w(tmem + C::O_COL(t), tmem + C::S_COL(t, buf) + kk * 8, vb + ((kk * 16 * 128) >> 4), IDESC_PV,
                      (acc || kk > 0) ? 1u : 0u);
        }
      };
      // ring positions follow the TMA's load order: K_s at rbase + 2s, V_s at rbase + 2s + 1
      int rbase = 0, gt = 0;
      for (int k = 0;; ++k) {
        mbar_wait_producer(&item_full[k & 1], (k >> 1) & 1);
        const int w = item_box[k & 1];
        __syncwarp();
        if (lane == 0) mbar_arrive(&item_empty[k & 1]);  // the MMA warp counts as one consumer
        if (w < 0) break;
        int seq, qblk, hg;
        prefill_decode_item(w, args, seq, qblk, hg);
        const int seq_start = args.cu_seqlens[seq];
        const int n_kv = n_kv_of(args.cu_seqlens[seq + 1] - seq_start, qblk);
        qb = (C::QBUF == 2) ? (k & 1) : 0;
        wait_cl(&q_full[qb], (C::QBUF == 2) ? ((k >> 1) & 1) : (k & 1));
        if (k == 0 && lane == 0) TRACE(16, 3);
        // QK_t(s) of step s for tile t; per tile, step s uses S buffer (gt + s) % SB
        auto qk_step_tile = [&](int s, int t) {
          const int ki = rbase + 2 * s, kslot = ki % NS;
          if (t == 0) {
            wait_cl(&kv_full[kslot], (ki / NS) & 1);
            tc_fence_after();
          }
          const int buf = (gt + s) % SB;
          issue_qk(t, kslot, buf);
          commit(&s_full[t * SB + buf]);
          if (t == NQ - 1) {
            commit(&kv_empty[kslot]);
            if (s == n_kv - 1) commit(&q_empty[qb]);
          }
        };
        for (int s = 0; s < LA && s < n_kv; ++s)
          for (int t = 0; t < NQ; ++t) qk_step_tile(s, t);
        for (int j = 0; j < n_kv; ++j) {
          const int vi = rbase + 2 * j + 1, vslot = vi % NS;
          wait_cl(&kv_full[vslot], (vi / NS) & 1);
          TRACE(6, gt + j);
          for (int t = 0; t < NQ; ++t) {
            wait_cl(&p_full[2 * t + ((gt + j) & 1)], ((gt + j) >> 1) & 1);
            TRACE(4 + t, gt + j);
            if (j == 0 && k > 0) wait_cl(&o_free[t], (k - 1) & 1);
            tc_fence_after();
            issue_pv(t, vslot, (gt + j) % SB, j > 0);
            commit(&o_done[2 * t + ((gt + j) & 1)]);
            if (t == NQ - 1) commit(&kv_empty[vslot]);
            if (j + LA < n_kv) {
              qk_step_tile(j + LA, t);
              if (t == 0) TRACE(7, gt + j);
            }
          }
        }
        rbase += 2 * n_kv;
        gt += n_kv;
      }
      if constexpr (PAIR) {
        // every MMA (and so every multicast arrival into the peer's barriers) has completed before
        // this warp reaches the teardown's cluster barrier
        umma_commit_pair_w(drain, 1);
        mbar_wait(drain, 0);
      }
    }
  } else if (C::STAGE_O && warp == C::STORE_WARP) {
    // ------------------------------------------------------------ O store warp (STAGE_O)
    // per item, the NQ tiles' epilogues in order (use n = NQ * item + tile): wait for the rows in
    // the staging buffer, issue the two {64 d, 1, 128} TMA stores, free the buffer once TMA read it
    regs_other();
    int n = 0;
    for (int k = 0;; ++k) {
      mbar_wait(&item_full[k & 1], (k >> 1) & 1);
      const int w = item_box[k & 1];
      __syncwarp();
      if (lane == 0) mbar_arrive(&item_empty[k & 1]);
      if (w < 0) break;
      for (int t = 0; t < NQ; ++t, ++n) {
        mbar_wait(stage_full, n & 1);
        if (lane == 0) {  // only the issuing lane reads the mailbox: it is rewritten once stage_free fires
          const int skip = stage_box[0], row0 = stage_box[1], head = stage_box[2];
          if (!skip) {
            tma_store_3d(&tmap_o, sStage, 0, head, row0);
            tma_store_3d(&tmap_o, sStage + C::HALF_Q, 64, head, row0);
            bulk_commit();
            bulk_wait_read_all();
          }
          mbar_arrive(stage_free);
        }
        __syncwarp();
      }
    }
    if (lane == 0) bulk_wait_all();  // the output is written before the CTA retires
  } else if (warp < C::NUM_SOFTMAX_WARPS) {
    // ------------------------------------------------------------ softmax warps of tile t
    if constexpr (C::REG_SPLIT) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::REG_SOFTMAX));
    // warp = (t * SPLIT + hh) * 4 + quadrant: the thread owns S row `row`, columns [hh*NCOL, +NCOL),
    // and O columns [hh*128/SPLIT, +128/SPLIT).  With SPLIT = 2 the two owners of a row sit on the
    // same SMSP and agree on every per-row decision through the pair barrier (named, 64 threads).
    const int t = warp / (4 * SPLIT);
    const int hh = (warp >> 2) % SPLIT;
    const int row = ((warp & 3) << 5) + lane;  // query row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) << 5) << 16;
    const uint32_t s_base = tmem + lane_base + hh * NCOL;
    constexpr int OCOLS = 128 / SPLIT;
    const uint32_t o_addr = tmem + lane_base + C::O_COL(t) + hh * OCOLS;
    const uint32_t pair_bar = 1 + t * 4 + (warp & 3);
    auto xidx = [&](int k, int h) { return ((k * NQ + t) * SPLIT + h) * 128 + row; };
    const float sl2 = args.scale_log2;
    // every phase of o_done is observed (compute-sanitizer synccheck): PV_t(g - LA) was issued before
    // QK_t(g) and tcgen05 ops complete in order, so once S_t(g) was seen the phase is complete.  It is
    // probed (non-blocking) right after S_t(g) and, in the never-taken case, waited on before P_t(g)
    // is handed over — while PV_t(g), the barrier's next phase at LA = 2, cannot have been issued
    auto o_done_bar = [&](int g) { return &o_done[2 * t + ((g - C::LA) & 1)]; };
    auto o_done_par = [&](int g) { return static_cast<uint32_t>(((g - C::LA) >> 1) & 1); };
    auto observe_o_done = [&](int g, bool seen) {
      if (g >= C::LA && !seen) mbar_wait(o_done_bar(g), o_done_par(g));
    };
    int gt = 0;
    for (int k = 0;; ++k) {
      if (PAIR && rank != 0)
        mbar_wait_cluster(&item_full[k & 1], (k >> 1) & 1);  // written by the leader
      else
        mbar_wait(&item_full[k & 1], (k >> 1) & 1);
      const int w = item_box[k & 1];
      arrive_consumer(&item_empty[k & 1]);
      if (w < 0) break;
      int seq, qblk, hg;
      prefill_decode_item(w, args, seq, qblk, hg);
      const int seq_start = args.cu_seqlens[seq];
      const int seq_len = args.cu_seqlens[seq + 1] - seq_start;
      const int n_kv = n_kv_of(seq_len, qblk);
      const int q_pos = qblk * BM + row;  // position within the sequence
      const int lim = args.causal ? min(seq_len - 1, q_pos) : seq_len - 1;  // last visible key
      const int kv_end = args.causal ? min(seq_len, qblk * BM + BM) : seq_len;
      float m_run = -INFINITY, l_run = 0.f;

      for (int j = 0; j < n_kv; ++j) {
        const int buf = (gt + j) % C::SB;
        mbar_wait(&s_full[t * C::SB + buf], ((gt + j) / C::SB) & 1);
        const bool od_seen = gt + j < C::LA || mbar_test(o_done_bar(gt + j), o_done_par(gt + j));
        tc_fence_after();
        const uint32_t s_addr = s_base + C::S_COL(t, buf);
        if (row == 0 && hh == 0) TRACE(t, gt + j);
        if (row == 0 && hh == 0 && t == 0 && k == 0 && j == 0) TRACE(16, 4);
        if (t == 0 && lane == 0 && warp < 4) TRACE(12 + warp, gt + j);
        const int kv0 = j * BN;
        const int kv0h = kv0 + hh * NCOL;  // first key of this thread's columns
        const bool edge = (kv0 + BN > kv_end) || (args.causal && kv0 + BN - 1 > q_pos);
        // masking is only needed on the diagonal / last tile: decide per warp (and, being a
        // function of the rows only, identically for both owners of a row), keep the common path
        // free of per-element compares and selects
        const bool warp_edge = __any_sync(0xffffffffu, edge);
        float lsum_spec;
        if (args.speculate && j > 0 && !warp_edge &&
            softmax_speculative<NCOL, EMU, SPLIT>(s_addr, sl2, m_run, lsum_spec, pair_bar)) {
          l_run += lsum_spec;
          tmem_wait_st();
          tc_fence_before();
          if (row == 0 && hh == 0) TRACE(2 + t, gt + j);
          if (t == 0 && lane == 0 && warp < 4) TRACE(8 + warp, gt + j);
          observe_o_done(gt + j, od_seen);
          arrive_consumer(&p_full[2 * t + ((gt + j) & 1)]);
          continue;
        }
        float mt = warp_edge ? softmax_rowmax<NCOL, true>(s_addr, kv0h, lim)
                             : softmax_rowmax<NCOL, false>(s_addr, kv0h, lim);
        if constexpr (SPLIT == 2) {
          // row max = max of the two halves; buffers alternate by step parity, and every step has
          // at least one pair barrier, so a buffer is never rewritten before the partner read it
          const int par = (gt + j) & 1;
          xch[xidx(par, hh)] = mt;
          named_bar_sync(pair_bar, 64);
          mt = fmaxf(mt, xch[xidx(par, hh ^ 1)]);
        }
        const float m_new = fmaxf(m_run, mt * sl2);
        const bool need = (m_new > m_run + 8.0f);
        float alpha = 1.f;
        if (need) {
          alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - m_new);
          m_run = m_new;
          l_run *= alpha;
        }
        if (j > 0 && __any_sync(0xffffffffu, need && alpha != 1.f)) {
          // O_t must hold PV_t(j-1) before it is rescaled (with the QK lookahead it may still be
          // in flight); per-parity barriers keep the phase unambiguous (PV_t(j-3) has landed and
          // PV_t(j+1) cannot be issued yet)
          mbar_wait(&o_done[2 * t + ((gt + j - 1) & 1)], ((gt + j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < OCOLS / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(o_addr + c * 32, r);
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(o_addr + c * 32, r);
          }
        }
        const float nmu = (m_run == -INFINITY) ? 0.f : -m_run;
        const float lsum = warp_edge ? softmax_pass2<NCOL, true, EMU>(s_addr, sl2, nmu, kv0h, lim)
                                     : softmax_pass2<NCOL, false, EMU>(s_addr, sl2, nmu, kv0h, lim);
        l_run += lsum;
        tmem_wait_st();
        tc_fence_before();
        if (row == 0 && hh == 0) TRACE(2 + t, gt + j);
        if (t == 0 && lane == 0 && warp < 4) TRACE(8 + warp, gt + j);
        observe_o_done(gt + j, od_seen);
        arrive_consumer(&p_full[2 * t + ((gt + j) & 1)]);
      }

      // ---------------------------------------------------------- epilogue for this item
      if (row == 0 && hh == 0 && t == 0 && k == 0) TRACE(16, 5);
      float l_tot = l_run;
      if constexpr (SPLIT == 2) {
        xch[xidx(2, hh)] = l_run;
        named_bar_sync(pair_bar, 64);
        l_tot += xch[xidx(2, hh ^ 1)];
      }
      mbar_wait(&o_done[2 * t + ((gt + n_kv - 1) & 1)], ((gt + n_kv - 1) >> 1) & 1);  // last PV_t
      tc_fence_after();
      const int h = hg * NQ * (PAIR ? 2 : 1) + static_cast<int>(rank) * NQ + t;
      const bool valid = q_pos < seq_len;
      const float inv_l = (l_tot > 0.f) ? 1.f / l_tot : 0.f;
      __nv_bfloat16* orow = args.o + (static_cast<size_t>(seq_start + q_pos) * args.num_q_heads + h) * D + hh * OCOLS;
      // STAGE_O: whole blocks go through the staging buffer and a TMA store; the last (partial)
      // block of a sequence is written row by row (a box store would spill into the next sequence)
      const bool staged = C::STAGE_O && (qblk * BM + BM <= seq_len);
      if constexpr (C::STAGE_O) {
        const int n = NQ * k + t;  // this tile's turn on the staging buffer
        if (n > 0) mbar_wait(stage_free, (n - 1) & 1);
      }
#pragma unroll
      for (int c = 0; c < OCOLS / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(o_addr + c * 32, r);
        if (staged) {
          // row `row` of the SW128 box pair: 16-byte unit j of a 128-byte half-row at j ^ (row & 7)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int col = hh * OCOLS + c * 32 + u * 8;  // first of 8 bf16
            const int hf = col >> 6, j = (col & 63) >> 3;
            const uint32_t a = smem_u32(sStage) + hf * C::HALF_Q + row * 128 + ((j ^ (row & 7)) << 4);
            const float* f = reinterpret_cast<const float*>(&r[u * 8]);
            st_shared_v4(a, pack_bf16x2(f[0] * inv_l, f[1] * inv_l), pack_bf16x2(f[2] * inv_l, f[3] * inv_l),
                         pack_bf16x2(f[4] * inv_l, f[5] * inv_l), pack_bf16x2(f[6] * inv_l, f[7] * inv_l));
          }
        } else if (valid) {
          // 32-byte stores: a thread owns a whole output row, so each store fills one sector (the
          // 16-byte form made the LSU split every warp store into 32 half-sector writes)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              pk[e] = pack_bf16x2(__uint_as_float(r[v * 16 + 2 * e]) * inv_l, __uint_as_float(r[v * 16 + 2 * e + 1]) * inv_l);
            st_global_v8(orow + c * 32 + v * 16, pk);
          }
        }
      }
      if constexpr (C::STAGE_O) {
        if (staged) fence_proxy_async_smem();  // generic smem writes -> visible to the TMA store
        if (row == 0 && hh == 0) {
          stage_box[0] = staged ? 0 : 1;
          stage_box[1] = seq_start + qblk * BM;
          stage_box[2] = h;
        }
        mbar_arrive(stage_full);
      }
      tc_fence_before();
      if (row == 0 && hh == 0 && t == 0 && k == 0) TRACE(16, 6);
#ifdef B200_TRACE
      if (row == 0 && hh == 0 && t == 0 && k == 0 && blockIdx.x < 1024) {
        unsigned long long tn;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
        g_ptrace[launch_par & 1][blockIdx.x][6] = static_cast<unsigned long long>(w);
        g_ptrace[launch_par & 1][blockIdx.x][7] = tn;
      }
#endif
      arrive_consumer(&o_free[t]);
      if (valid && hh == 0 && args.lse != nullptr) {
        args.lse[static_cast<size_t>(h) * args.total_tokens + seq_start + q_pos] =
            (l_tot > 0.f) ? (m_run + __log2f(l_tot)) * 0.69314718055994530942f : -INFINITY;
      }
      gt += n_kv;
    }
  } else {
    regs_other();  // idle padding warps of the producer warpgroup
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no remote arrive / MMA into the other CTA is in flight
  if (threadIdx.x == 0) TRACE(16, 7);
  PTRACE(2);
  if (warp == C::MMA_WARP) {
    __syncwarp();
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc_pair(tmem, C::TMEM_COLS);
    else
      tmem_dealloc(tmem, C::TMEM_COLS);
  }
  if (threadIdx.x == 0) {
    // every CTA has drawn its final (out-of-range) item before getting here: the last one out
    // re-zeroes the work counter (sched[0]) and the done counter (sched[2]) for the next launch
    __threadfence();
    if (atomicAdd(args.sched + 2, 1) == static_cast<int>(gridDim.x) - 1) {
      args.sched[0] = 0;
      args.sched[2] = 0;
      __threadfence();
#ifdef B200_TRACE
      atomicAdd(&g_plaunch, 1u);
#endif
    }
  }
  PTRACE(3);
}

// Longest-first work list: one (seq, q block) entry per 128-row query block, sorted by causal
// cost (q block index; non-causal: the sequence's block count) descending via a counting sort.
// ws layout: [0] work counter, [1] n_pairs, [2] done counter, [3 .. 3+nkeys) key offsets, then items.
// One warp per sequence, lanes over its q blocks; the histogram lives in shared memory when it
// fits (SMEM_HIST), so no thread ever waits on a chain of global atomics (a single 8k-token
// sequence used to cost 64 dependent L2 round trips, ~30 us).
template <bool SMEM_HIST>
__global__ void __launch_bounds__(1024) prefill_schedule_kernel(const int32_t* __restrict__ cu, int num_seqs,
                                                                int causal, int nkeys, int32_t* __restrict__ ws) {
  extern __shared__ int32_t sh_hist[];
  int32_t* hist = SMEM_HIST ? sh_hist : ws + 3;
  int32_t* items = ws + 3 + nkeys;
  __shared__ int32_t part[1024];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  griddep_wait();  // PDL: the previous launch may still be reading this workspace
  griddep_launch();
  for (int k = tid; k < nkeys; k += 1024) hist[k] = 0;
  __syncthreads();
  for (int s = warp; s < num_seqs; s += 32) {
    const int nqb = (cu[s + 1] - cu[s] + 127) / 128;
    if (causal) {
      for (int qb = lane; qb < nqb; qb += 32) atomicAdd(&hist[qb], 1);
    } else if (lane == 0 && nqb > 0) {
      atomicAdd(&hist[nqb - 1], nqb);
    }
  }
  __syncthreads();
  // exclusive scan in DESCENDING key order: off[k] = sum_{k' > k} hist[k']
  const int seg = (nkeys + 1023) / 1024;
  const int k_hi = nkeys - 1 - tid * seg;  // this thread's keys: k_hi, k_hi-1, ..., k_hi-seg+1
  int local = 0;
  for (int i = 0; i < seg; ++i) {
    const int k = k_hi - i;
    if (k >= 0) local += hist[k];
  }
  part[tid] = local;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int v = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = part[tid] - local;
  for (int i = 0; i < seg; ++i) {
    const int k = k_hi - i;
    if (k >= 0) {
      const int h = hist[k];
      hist[k] = run;
      run += h;
    }
  }
  __syncthreads();
  for (int s = warp; s < num_seqs; s += 32) {
    const int nqb = (cu[s + 1] - cu[s] + 127) / 128;
    if (causal) {
      for (int qb = lane; qb < nqb; qb += 32)
        items[atomicAdd(&hist[qb], 1)] = static_cast<int32_t>((static_cast<uint32_t>(s) << 16) | qb);
    } else if (nqb > 0) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&hist[nqb - 1], nqb);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (int qb = lane; qb < nqb; qb += 32)
        items[base + qb] = static_cast<int32_t>((static_cast<uint32_t>(s) << 16) | qb);
    }
  }
  if (tid == 0) {
    ws[0] = 0;
    ws[1] = part[1023];
  }
}

// L2-aware banded work list (band > 0, see PrefillKernelArgs): bands of `band` q blocks from the
// top band down (causal; non-causal: a sequence's items all sit in the band of its block count),
// inside a band by sequence, kv head, q block descending.  One CTA: per band a block-wide scan of
// the per-sequence entry counts, then each thread writes its sequences' entries.  Used only for
// problems whose K/V exceeds ~half of L2, where the prefill runs for >= ~0.5 ms.
// ws: [0] work counter, [1] n_pairs, [2] done counter, entries (2 ints each) at ws + items_off.
__global__ void __launch_bounds__(1024) prefill_schedule_banded_kernel(const int32_t* __restrict__ cu, int num_seqs,
                                                                       int causal, int hkv, int band, int nbands,
                                                                       int items_off, int32_t* __restrict__ ws) {
  int32_t* ent = ws + items_off;
  __shared__ int32_t part[1024];
  const int tid = threadIdx.x;
  griddep_wait();
  griddep_launch();
  const int per = (num_seqs + 1023) / 1024;
  const int s0 = tid * per;
  auto nqb_of = [&](int s) { return (cu[s + 1] - cu[s] + 127) / 128; };
  auto range = [&](int k, int nqb, int& lo, int& hi) {  // q blocks of band k: [lo, hi)
    if (causal) {
      lo = k * band;
      hi = min(nqb, lo + band);
    } else {
      const bool mine = nqb > 0 && (nqb - 1) / band == k;
      lo = 0;
      hi = mine ? nqb : 0;
    }
  };
  int pairs_local = 0;
  for (int i = 0; i < per; ++i)
    if (s0 + i < num_seqs) pairs_local += nqb_of(s0 + i);
  int base = 0;
  for (int k = nbands - 1; k >= 0; --k) {
    int local = 0;
    for (int i = 0; i < per; ++i) {
      const int s = s0 + i;
      if (s >= num_seqs) break;
      int lo, hi;
      range(k, nqb_of(s), lo, hi);
      local += max(0, hi - lo) * hkv;
    }
    part[tid] = local;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int v = tid >= off ? part[tid - off] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    int o = base + part[tid] - local;
    for (int i = 0; i < per; ++i) {
      const int s = s0 + i;
      if (s >= num_seqs) break;
      int lo, hi;
      range(k, nqb_of(s), lo, hi);
      for (int kvh = 0; kvh < hkv; ++kvh)
        for (int qb = hi - 1; qb >= lo; --qb, ++o) {
          ent[2 * o] = static_cast<int32_t>((static_cast<uint32_t>(s) << 16) | static_cast<uint32_t>(qb));
          ent[2 * o + 1] = kvh;
        }
    }
    base += part[1023];
    __syncthreads();  // part is rewritten by the next band
  }
  // n_pairs = sum of q blocks (block reduction through part)
  part[tid] = pairs_local;
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (tid < off) part[tid] += part[tid + off];
    __syncthreads();
  }
  if (tid == 0) {
    ws[0] = 0;
    ws[1] = part[0];
  }
}

}  // namespace b200
