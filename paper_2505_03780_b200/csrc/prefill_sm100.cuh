// prefill_sm100.cuh — K1: causal varlen flash-attention forward (prefill), sm_100a.
//
// Semantics (restated in oracle/attn_oracle.c, the checker):
//   for every sequence s (tokens cu_seqlens[s] .. cu_seqlens[s+1]) and q head h,
//   O[t,h,:] = softmax_j( scale * Q[t,h,:].K[j,h/G,:] , j <= t if causal ) . V[j,h/G,:]
// i.e. FlashAttention-2 forward with GQA (G = Hq/Hkv), the kernel family the paper tunes
// (ref/PAPER.md:108-113; knob names from ref/pkg/src/ktune/fixtures/flash_attention.space.json:3-16).
//
// CTA = one 128-row query block of one sequence for NQ (1 or 2) q heads of the SAME kv head,
// so every K/V tile loaded by TMA feeds NQ x (QK^T + PV) tcgen05 MMAs.
//
//   warps 0..4*NQ-1 : softmax warpgroup(s), one per Q tile; thread = query row (TMEM lane)
//   warp  4*NQ      : TMA producer (Q once, then K_j / V_j into a ring of 32-KB slots)
//   warp  4*NQ+1    : TMEM allocator + single-thread tcgen05.mma issuer
//
// TMEM (512 cols): S_t at [t*BN], O_t at [256 + t*128].  P_t (bf16) goes to smem in the
// canonical K-major SWIZZLE_128B layout and feeds PV as the A operand; V is the B operand
// in MN-major SW128 straight from its TMA tile (no transpose anywhere).
// Online softmax is per-thread (a thread owns a whole S row), exp2 with log2(e)*scale folded,
// lazy O rescaling (only when the running max grows by > 8 in log2 units; FA4's trick).
#pragma once
#include "sm100_common.cuh"

namespace b200 {

struct PrefillKernelArgs {
  const int32_t* cu_seqlens;
  __nv_bfloat16* o;
  float* lse;  // optional [Hq, T]
  int32_t total_tokens;
  int32_t num_q_heads;
  int32_t group;  // Hq / Hkv
  int32_t causal;
  float scale_log2;  // softmax_scale * log2(e)
};

template <int NQ, int BN, int NSTAGE>
struct PrefillCfg {
  static constexpr int D = 128;
  static constexpr int BM = 128;
  static constexpr int NUM_SOFTMAX_WARPS = 4 * NQ;
  static constexpr int TMA_WARP = NUM_SOFTMAX_WARPS;
  static constexpr int MMA_WARP = NUM_SOFTMAX_WARPS + 1;
  static constexpr int NTHREADS = 32 * (NUM_SOFTMAX_WARPS + 2);
  static constexpr int Q_BYTES = BM * D * 2;       // 32 KB per Q tile (2 SW128 halves)
  static constexpr int KV_BYTES = BN * D * 2;      // one K or V tile
  static constexpr int HALF_Q = BM * 128;          // bytes of one 64-column half
  static constexpr int HALF_KV = BN * 128;
  static constexpr int P_BYTES = BM * BN * 2;
  static constexpr int P_HALF = BM * 128;           // P row = BN bf16 = BN/64 halves of 128 B
  // smem carve (all 1024-aligned)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = OFF_Q + NQ * Q_BYTES;
  static constexpr int OFF_P = OFF_KV + NSTAGE * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + NQ * P_BYTES;
  static constexpr int NUM_BARS = 1 + 2 * NSTAGE + 2 * NQ + 1;  // q_full, full/empty ring, s_full, p_full, o_full
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16 + 1024;  // +1 KB alignment slack
  static constexpr uint32_t TMEM_COLS = 512;
  __host__ __device__ static constexpr uint32_t S_COL(int t) { return t * BN; }
  __host__ __device__ static constexpr uint32_t O_COL(int t) { return 256 + t * 128; }
  static_assert(BN == 64 || BN == 128, "BLOCK_N in {64,128}");
  static_assert(NQ * BN <= 256, "S tiles must fit below the O region");
};

template <int NQ, int BN, int NSTAGE>
__global__ void __launch_bounds__(PrefillCfg<NQ, BN, NSTAGE>::NTHREADS, 1)
    prefill_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_k,
                       const __grid_constant__ CUtensorMap tmap_v, const PrefillKernelArgs args) {
  using C = PrefillCfg<NQ, BN, NSTAGE>;
  constexpr int D = C::D, BM = C::BM;

  // ---- work item: blockIdx.x = head group, blockIdx.y = q block (longest first), blockIdx.z = seq
  const int seq = blockIdx.z;
  const int seq_start = args.cu_seqlens[seq];
  const int seq_len = args.cu_seqlens[seq + 1] - seq_start;
  const int num_qblk = (seq_len + BM - 1) / BM;
  const int qblk = num_qblk - 1 - static_cast<int>(blockIdx.y);
  if (qblk < 0) return;  // this sequence is shorter than the grid's longest one
  const int h0 = blockIdx.x * NQ;
  const int kvh = h0 / args.group;
  const int q_row0 = qblk * BM;  // within the sequence
  const int kv_end = args.causal ? min(seq_len, q_row0 + BM) : seq_len;
  const int n_kv = (kv_end + BN - 1) / BN;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sKV = smem + C::OFF_KV;
  uint8_t* sP = smem + C::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 1 + NSTAGE;
  uint64_t* s_full = bars + 1 + 2 * NSTAGE;
  uint64_t* p_full = s_full + NQ;
  uint64_t* o_full = p_full + NQ;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);

  const int warp = warp_id();
  const int lane = lane_id();

  if (warp == C::TMA_WARP && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_k);
    tma_prefetch_desc(&tmap_v);
  }
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < NQ; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
    }
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == C::TMA_WARP) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const int row0 = seq_start + q_row0;
      mbar_arrive_expect_tx(q_full, NQ * C::Q_BYTES);
      for (int t = 0; t < NQ; ++t)
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d(sQ + t * C::Q_BYTES + hf * C::HALF_Q, &tmap_q, q_full, hf * 64, h0 + t, row0);
      const uint64_t keep = policy_evict_last();  // K/V tiles are re-read by the other q blocks / heads
      for (int idx = 0; idx < 2 * n_kv; ++idx) {
        const int slot = idx % NSTAGE;
        const uint32_t ph = (idx / NSTAGE) & 1;
        mbar_wait(&kv_empty[slot], ph ^ 1);
        const int j = idx >> 1;
        const CUtensorMap* map = (idx & 1) ? &tmap_v : &tmap_k;
        uint8_t* dst = sKV + slot * C::KV_BYTES;
        mbar_arrive_expect_tx(&kv_full[slot], C::KV_BYTES);
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d_hint(dst + hf * C::HALF_KV, map, &kv_full[slot], hf * 64, kvh, seq_start + j * BN, keep);
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = idesc_bf16_f32(BM, BN, false, false);
      constexpr uint32_t IDESC_PV = idesc_bf16_f32(BM, D, false, true);
      const uint32_t q_base = smem_u32(sQ), kv_base = smem_u32(sKV), p_base = smem_u32(sP);
      auto issue_qk = [&](int t, int slot) {
        const uint32_t qa = q_base + t * C::Q_BYTES, kb = kv_base + slot * C::KV_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk & 3) * 32;
          const uint64_t da = sdesc_sw128(qa + (kk >> 2) * C::HALF_Q + off, 16, 1024);
          const uint64_t db = sdesc_sw128(kb + (kk >> 2) * C::HALF_KV + off, 16, 1024);
          umma_ss(tmem + C::S_COL(t), da, db, IDESC_QK, kk > 0);
        }
      };
      auto issue_pv = [&](int t, int slot, bool acc) {
        const uint32_t pa = p_base + t * C::P_BYTES, vb = kv_base + slot * C::KV_BYTES;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t da = sdesc_sw128(pa + (kk >> 2) * C::P_HALF + (kk & 3) * 32, 16, 1024);
          const uint64_t db = sdesc_sw128(vb + kk * 16 * 128, C::HALF_KV, 1024);
          umma_ss(tmem + C::O_COL(t), da, db, IDESC_PV, (acc || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0);
      // prologue: S_t(0) for every Q tile
      {
        mbar_wait(&kv_full[0], 0);
        tc_fence_after();
        for (int t = 0; t < NQ; ++t) {
          issue_qk(t, 0);
          umma_commit(&s_full[t]);
        }
        umma_commit(&kv_empty[0]);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int vidx = 2 * j + 1, kidx = 2 * j + 2;
        const int vslot = vidx % NSTAGE, kslot = kidx % NSTAGE;
        const bool more = (j + 1) < n_kv;
        mbar_wait(&kv_full[vslot], (vidx / NSTAGE) & 1);
        for (int t = 0; t < NQ; ++t) {
          mbar_wait(&p_full[t], j & 1);
          tc_fence_after();
          issue_pv(t, vslot, j > 0);
          if (t == NQ - 1) umma_commit(&kv_empty[vslot]);
          if (more) {
            if (t == 0) {
              mbar_wait(&kv_full[kslot], (kidx / NSTAGE) & 1);
              tc_fence_after();
            }
            issue_qk(t, kslot);
            umma_commit(&s_full[t]);
            if (t == NQ - 1) umma_commit(&kv_empty[kslot]);
          }
        }
      }
      umma_commit(o_full);
    }
  } else {
    // ------------------------------------------------------------ softmax warpgroup t
    const int t = warp >> 2;
    const int row = ((warp & 3) << 5) + lane;  // query row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) << 5) << 16;
    const uint32_t s_addr = tmem + lane_base + C::S_COL(t);
    const uint32_t o_addr = tmem + lane_base + C::O_COL(t);
    const uint32_t p_row = smem_u32(sP + t * C::P_BYTES) + row * 128;
    const int q_pos = q_row0 + row;  // position within the sequence
    const float sl2 = args.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;

    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      // pass 1: row max straight out of TMEM (S is re-read in pass 2; TMEM bandwidth is cheap,
      // registers are not: a whole 128-wide fp32 row per thread would spill at 320 threads)
      const int kv0 = j * BN;
      const bool edge = (kv0 + BN > kv_end) || (args.causal && kv0 + BN - 1 > q_pos);
      const int lim = args.causal ? min(seq_len - 1, q_pos) : seq_len - 1;  // last visible key
      float mt = -INFINITY;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(s_addr + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float v = (edge && kv0 + c * 32 + i > lim) ? -INFINITY : __uint_as_float(r[i]);
          mt = fmaxf(mt, v);
        }
      }
      const float m_new = fmaxf(m_run, mt * sl2);
      // lazy rescale: keep a stale max unless it would let exp2 exceed 2^8
      const bool need = (m_new > m_run + 8.0f);
      float alpha = 1.f;
      if (need) {
        alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - m_new);
        m_run = m_new;
        l_run *= alpha;
      }
      if (j > 0 && __any_sync(0xffffffffu, need && alpha != 1.f)) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(o_addr + c * 32, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st32(o_addr + c * 32, r);
        }
        tmem_wait_st();
      }
      // pass 2: P = exp2(S * scale*log2e - m) -> bf16 -> swizzled smem row
      const float mu = (m_run == -INFINITY) ? 0.f : m_run;
      float lsum = 0.f;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(s_addr + c * 32, r);
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          float p[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int col = c * 32 + q8 * 8 + i;
            const float e = fast_exp2(fmaf(__uint_as_float(r[q8 * 8 + i]), sl2, -mu));
            p[i] = (edge && kv0 + col > lim) ? 0.f : e;
            lsum += p[i];
          }
          const int ck = c * 4 + q8;  // 16-byte chunk of the P row
          const int hf = ck >> 3, ch = ck & 7;
          const uint32_t addr = p_row + hf * C::P_HALF + ((ch ^ (row & 7)) << 4);
          st_shared_v4(addr, pack_bf16x2(p[0], p[1]), pack_bf16x2(p[2], p[3]), pack_bf16x2(p[4], p[5]),
                       pack_bf16x2(p[6], p[7]));
        }
      }
      l_run += lsum;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[t]);
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(o_full, 0);
    tc_fence_after();
    const int h = h0 + t;
    const bool valid = q_pos < seq_len;
    const float inv_l = (l_run > 0.f) ? 1.f / l_run : 0.f;
    __nv_bfloat16* orow = args.o + (static_cast<size_t>(seq_start + q_pos) * args.num_q_heads + h) * D;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(o_addr + c * 32, r);
      if (valid) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float* f = reinterpret_cast<const float*>(&r[v * 8]);
          st_global_v4(orow + c * 32 + v * 8, pack_bf16x2(f[0] * inv_l, f[1] * inv_l),
                       pack_bf16x2(f[2] * inv_l, f[3] * inv_l), pack_bf16x2(f[4] * inv_l, f[5] * inv_l),
                       pack_bf16x2(f[6] * inv_l, f[7] * inv_l));
        }
      }
    }
    if (valid && args.lse != nullptr) {
      // natural-log LSE of the scaled scores
      args.lse[static_cast<size_t>(h) * args.total_tokens + seq_start + q_pos] =
          (l_run > 0.f) ? (m_run + __log2f(l_run)) * 0.69314718055994530942f : -INFINITY;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace b200
