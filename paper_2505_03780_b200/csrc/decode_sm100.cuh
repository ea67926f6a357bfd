// decode_sm100.cuh — K2: paged-KV split-KV decode attention, K3: split combine (sm_100a).
//
// Semantics (oracle/attn_oracle.c): for sequence b with n = seq_lens[b] cached tokens and a
// single query token at position n-1, token i lives at
//     cache[block_table[b, i / block_size], i % block_size, kvh, :]
// and O[b,h,:] = softmax_i(scale * q[b,h,:].K_i) . V_i  over i < n  (h -> kvh = h / G).
//
// CTA = (split, kv head, sequence).  It streams its range of 128-token tiles through a
// ring of 32-KB smem slots filled by TMA page gathers (one 2-KB box per page per 64-column
// half: 16 token rows x 128 B, SWIZZLE_128B) and runs the contractions "swap-AB" so the
// long KV axis sits on the MMA M=128 side and the GQA group (G <= 16 q heads, zero-padded to
// N=16) on N:
//     S^T[tok, h] = K_tile[tok, :] . Q_grp[h, :]^T            (A = K, K-major; B = Q, K-major)
//     O^T[d, h]   = V_tile^T[d, tok] . P^T[tok, h]            (A = V, MN-major; B = P, K-major)
// Each softmax thread owns one token (one TMEM lane) for S and one head-dim row d for O;
// the per-head max over the 128 tokens is a warp-shuffle reduction + a 4-warp smem exchange.
// O^T of every tile lands in a fresh TMEM buffer and is folded into registers with the
// running rescale, lagging one tile so the PV MMA overlaps the next softmax.
#pragma once
#include "sm100_common.cuh"

namespace b200 {

struct DecodeKernelArgs {
  const int32_t* block_table;  // [B, max_blocks]
  const int32_t* seq_lens;     // [B]
  __nv_bfloat16* o;            // [B, Hq, D]            (num_splits == 1)
  float* part_o;               // [B, Hq, splits, D]    (num_splits > 1), unnormalised
  float* part_ml;              // [B, Hq, splits, 2]    running max (log2 units) and sum
  int32_t num_q_heads;
  int32_t group;
  int32_t block_size;
  int32_t max_blocks;
  int32_t num_blocks;
  int32_t num_splits;
  int32_t tiles_per_split;
  float scale_log2;
};

template <int NSTAGE>
struct DecodeCfg {
  static constexpr int D = 128;
  static constexpr int TILE = 128;   // tokens per MMA tile (M = 128)
  static constexpr int NPAD = 16;    // GQA group padded to the MMA N
  static constexpr int NTHREADS = 192;  // 4 softmax warps, TMA warp, MMA warp
  static constexpr int TMA_WARP = 4, MMA_WARP = 5;
  static constexpr int SLOT = TILE * D * 2;  // 32 KB
  static constexpr int HALF = TILE * 128;    // 16 KB
  static constexpr int QB = NPAD * D * 2;    // 4 KB (2 halves of 16 rows x 128 B)
  static constexpr int QHALF = NPAD * 128;   // 2 KB
  static constexpr int OFF_KV = 0;
  static constexpr int OFF_Q = OFF_KV + NSTAGE * SLOT;
  static constexpr int OFF_P = OFF_Q + QB;             // 2 buffers of P^T (same shape as Q)
  static constexpr int OFF_RED = OFF_P + 2 * QB;       // [2][4][16] floats
  static constexpr int OFF_BAR = OFF_RED + 2 * 4 * 16 * 4;
  static constexpr int NUM_BARS = 1 + 2 * NSTAGE + 2 + 2 + 2 + 2;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16 + 1024;
  static constexpr uint32_t TMEM_COLS = 64;  // S[2] @ 0,16 ; O[2] @ 32,48
};

template <int NSTAGE>
__global__ void __launch_bounds__(DecodeCfg<NSTAGE>::NTHREADS)
    decode_split_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_k,
                        const __grid_constant__ CUtensorMap tmap_v, const DecodeKernelArgs args) {
  using C = DecodeCfg<NSTAGE>;
  constexpr int D = C::D, TILE = C::TILE;
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int G = args.group;
  const int seq_len = args.seq_lens[b];
  const int n_tiles_seq = (seq_len + TILE - 1) / TILE;
  const int tile0 = split * args.tiles_per_split;
  const int n_local = min(args.tiles_per_split, n_tiles_seq - tile0);
  const int warp = warp_id(), lane = lane_id();

  if (n_local <= 0) {
    // empty split: neutral partial (m = -inf, l = 0, O = 0) so the combine ignores it
    if (args.num_splits > 1 && threadIdx.x < D) {
      for (int g = 0; g < G; ++g) {
        const size_t row = (static_cast<size_t>(b) * args.num_q_heads + kvh * G + g) * args.num_splits + split;
        args.part_o[row * D + threadIdx.x] = 0.f;
        if (threadIdx.x == 0) {
          args.part_ml[row * 2 + 0] = -INFINITY;
          args.part_ml[row * 2 + 1] = 0.f;
        }
      }
    } else if (args.num_splits == 1 && threadIdx.x < D) {
      for (int g = 0; g < G; ++g)
        args.o[(static_cast<size_t>(b) * args.num_q_heads + kvh * G + g) * D + threadIdx.x] = __float2bfloat16(0.f);
    }
    return;
  }

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sKV = smem + C::OFF_KV;
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sP = smem + C::OFF_P;
  float* red = reinterpret_cast<float*>(smem + C::OFF_RED);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 1 + NSTAGE;
  uint64_t* s_full = bars + 1 + 2 * NSTAGE;  // [2]
  uint64_t* p_full = s_full + 2;             // [2]
  uint64_t* o_full = p_full + 2;             // [2]
  uint64_t* o_empty = o_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);

  if (warp == C::TMA_WARP && lane == 0) {
    tma_prefetch_desc(&tmap_q);
    tma_prefetch_desc(&tmap_k);
    tma_prefetch_desc(&tmap_v);
  }
  // zero the padded Q rows (G..15); TMA fills rows 0..G-1 of each half
  for (int i = threadIdx.x; i < C::QB / 16; i += C::NTHREADS)
    reinterpret_cast<uint4*>(sQ)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_slot, C::TMEM_COLS);
  fence_proxy_async_smem();  // zeroed Q rows visible to the async proxy before TMA/MMA
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == C::TMA_WARP) {
    // ------------------------------------------------------------ TMA producer (page gather)
    const int bs = args.block_size;
    const int pages_per_tile = TILE / bs;
    const int n_pages_seq = (seq_len + bs - 1) / bs;
    const int32_t* bt = args.block_table + static_cast<size_t>(b) * args.max_blocks;
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * G * 128);
      for (int hf = 0; hf < 2; ++hf) tma_load_3d(sQ + hf * C::QHALF, &tmap_q, q_full, hf * 64, kvh * G, b);
    }
    const uint64_t stream_once = policy_evict_first();
    for (int i = 0; i < n_local; ++i) {
      const int tile = tile0 + i;
      // lanes 0..pages_per_tile-1 fetch this tile's physical pages; pages past the end of the
      // sequence re-read the last valid page (finite data, weighted by p = 0)
      int page = 0;
      if (lane < pages_per_tile) {
        const int lp = min(tile * pages_per_tile + lane, n_pages_seq - 1);
        page = bt[lp];
      }
      for (int kv = 0; kv < 2; ++kv) {
        const int idx = 2 * i + kv;
        const int slot = idx % NSTAGE;
        const uint32_t ph = (idx / NSTAGE) & 1;
        if (lane == 0) {
          mbar_wait(&kv_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&kv_full[slot], C::SLOT);
        }
        __syncwarp();
        const CUtensorMap* map = kv ? &tmap_v : &tmap_k;
        uint8_t* dst = sKV + slot * C::SLOT;
        for (int p = 0; p < pages_per_tile; ++p) {
          const int pg = __shfl_sync(0xffffffffu, page, p);
          if (lane == 0) {
            for (int hf = 0; hf < 2; ++hf)
              tma_load_3d_hint(dst + hf * C::HALF + p * bs * 128, map, &kv_full[slot], hf * 64, kvh, pg * bs,
                               stream_once);
          }
        }
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = idesc_bf16_f32(TILE, C::NPAD, false, false);
      constexpr uint32_t IDESC_PV = idesc_bf16_f32(D, C::NPAD, true, false);
      const uint32_t kv_base = smem_u32(sKV), q_base = smem_u32(sQ), p_base = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto do_qk = [&](int i) {
        const int idx = 2 * i, slot = idx % NSTAGE;
        mbar_wait(&kv_full[slot], (idx / NSTAGE) & 1);
        tc_fence_after();
        const uint32_t kb = kv_base + slot * C::SLOT;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t da = sdesc_sw128(kb + (kk >> 2) * C::HALF + (kk & 3) * 32, 16, 1024);
          const uint64_t db = sdesc_sw128(q_base + (kk >> 2) * C::QHALF + (kk & 3) * 32, 16, 1024);
          umma_ss(tmem + (i & 1) * 16, da, db, IDESC_QK, kk > 0);
        }
        umma_commit(&s_full[i & 1]);
        umma_commit(&kv_empty[slot]);
      };
      auto do_pv = [&](int i) {
        const int idx = 2 * i + 1, slot = idx % NSTAGE;
        const int pb = i & 1;
        mbar_wait(&kv_full[slot], (idx / NSTAGE) & 1);
        mbar_wait(&p_full[pb], (i >> 1) & 1);
        if (i >= 2) mbar_wait(&o_empty[pb], ((i >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t vb = kv_base + slot * C::SLOT;
        const uint32_t pbase = p_base + pb * C::QB;
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk) {
          const uint64_t da = sdesc_sw128(vb + kk * 16 * 128, C::HALF, 1024);
          const uint64_t db = sdesc_sw128(pbase + (kk >> 2) * C::QHALF + (kk & 3) * 32, 16, 1024);
          umma_ss(tmem + 32 + pb * 16, da, db, IDESC_PV, kk > 0);
        }
        umma_commit(&o_full[pb]);
        umma_commit(&kv_empty[slot]);
      };
      do_qk(0);
      for (int i = 0; i < n_local; ++i) {
        if (i + 1 < n_local) do_qk(i + 1);
        do_pv(i);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / accumulate (128 thr)
    const int t = threadIdx.x;  // token row of S^T and d row of O^T (TMEM lane)
    const uint32_t lane_base = static_cast<uint32_t>(warp << 5) << 16;
    const float sl2 = args.scale_log2;
    float m_run[16], l_part[16], o_acc[16], alpha_prev[16];
#pragma unroll
    for (int h = 0; h < 16; ++h) {
      m_run[h] = -INFINITY;
      l_part[h] = 0.f;
      o_acc[h] = 0.f;
      alpha_prev[h] = 1.f;
    }
    const int half = t >> 6, chunk = (t & 63) >> 3, sub = t & 7;

    auto fold_o = [&](int i) {  // O_acc = O_acc * alpha_i + O_i
      const int pb = i & 1;
      mbar_wait(&o_full[pb], (i >> 1) & 1);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16(tmem + lane_base + 32 + pb * 16, r);
#pragma unroll
      for (int h = 0; h < 16; ++h) o_acc[h] = fmaf(o_acc[h], alpha_prev[h], __uint_as_float(r[h]));
      tc_fence_before();
      mbar_arrive(&o_empty[pb]);
    };

    for (int i = 0; i < n_local; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16(tmem + lane_base + sb * 16, r);
      const bool valid = (tile0 + i) * TILE + t < seq_len;
      float x[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) x[h] = valid ? __uint_as_float(r[h]) * sl2 : -INFINITY;
      // per-head max over the 128 tokens: shuffle within the warp, then across the 4 warps
      float mx[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        float v = x[h];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
        mx[h] = v;
      }
      float* rb = red + sb * 64;
      if (lane < 16) {
        float v = mx[0];
#pragma unroll
        for (int h = 1; h < 16; ++h)
          if (lane == h) v = mx[h];
        rb[warp * 16 + lane] = v;
      }
      named_bar_sync(1, 128);
      float alpha[16], p[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const float mt = fmaxf(fmaxf(rb[h], rb[16 + h]), fmaxf(rb[32 + h], rb[48 + h]));
        const float mn = fmaxf(m_run[h], mt);
        const float mu = (mn == -INFINITY) ? 0.f : mn;
        alpha[h] = fast_exp2(m_run[h] - mu);  // m_run = -inf -> 0
        p[h] = fast_exp2(x[h] - mu);
        l_part[h] = fmaf(l_part[h], alpha[h], p[h]);
        m_run[h] = mn;
      }
      // P^T (bf16) -> smem as the K-major B operand [16 heads][128 tokens]
      const uint32_t pbase = smem_u32(sP + sb * C::QB) + half * C::QHALF + (sub << 1);
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const __nv_bfloat16 v = __float2bfloat16_rn(p[h]);
        const uint32_t addr = pbase + h * 128 + ((chunk ^ (h & 7)) << 4);
        asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(*reinterpret_cast<const uint16_t*>(&v))
                     : "memory");
      }
      if (!valid) {
        // tail slots of the last page hold arbitrary bytes: P = 0 there, but 0 * NaN would
        // poison O, so zero this token's V row before PV reads it
        const int vidx = 2 * i + 1, vslot = vidx % NSTAGE;
        mbar_wait(&kv_full[vslot], (vidx / NSTAGE) & 1);
        uint4* vr = reinterpret_cast<uint4*>(sKV + vslot * C::SLOT + t * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          vr[c] = make_uint4(0, 0, 0, 0);
          vr[C::HALF / 16 + c] = make_uint4(0, 0, 0, 0);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (i >= 1) fold_o(i - 1);
#pragma unroll
      for (int h = 0; h < 16; ++h) alpha_prev[h] = alpha[h];
    }
    fold_o(n_local - 1);

    // ---- reduce the per-thread partial sums over the 128 tokens
    float* rl = red;  // reuse: [4][16]; everyone is past the last named barrier's reads
    named_bar_sync(1, 128);
    float lsum[16];
#pragma unroll
    for (int h = 0; h < 16; ++h) {
      float v = l_part[h];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      lsum[h] = v;
    }
    if (lane < 16) {
      float v = lsum[0];
#pragma unroll
      for (int h = 1; h < 16; ++h)
        if (lane == h) v = lsum[h];
      rl[warp * 16 + lane] = v;
    }
    named_bar_sync(1, 128);
    for (int g = 0; g < G; ++g) {
      float l = rl[g] + rl[16 + g] + rl[32 + g] + rl[48 + g];
      float ov = 0.f;
#pragma unroll
      for (int h = 0; h < 16; ++h)
        if (h == g) ov = o_acc[h];
      float mg = 0.f;
#pragma unroll
      for (int h = 0; h < 16; ++h)
        if (h == g) mg = m_run[h];
      const int hq = kvh * G + g;
      if (args.num_splits == 1) {
        args.o[(static_cast<size_t>(b) * args.num_q_heads + hq) * D + t] =
            __float2bfloat16_rn(l > 0.f ? ov / l : 0.f);
      } else {
        const size_t row = (static_cast<size_t>(b) * args.num_q_heads + hq) * args.num_splits + split;
        args.part_o[row * D + t] = ov;
        if (t == 0) {
          args.part_ml[row * 2 + 0] = mg;
          args.part_ml[row * 2 + 1] = l;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// K3: O[b,h,:] = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s   (m in log2 units).
// One pass: the splits' (max, sum) pairs and O values are loaded 8 at a time, back to back, and
// folded into a running (m, l, acc) with the online-softmax rescale — one dependent L2 round trip
// per 8 splits instead of a max pass followed by a weighted-sum pass.
__global__ void __launch_bounds__(128) decode_combine_kernel(const float* __restrict__ part_o,
                                                              const float* __restrict__ part_ml,
                                                              __nv_bfloat16* __restrict__ o, int num_splits) {
  constexpr int U = 8;
  const int row = blockIdx.x;  // b * Hq + h
  const int d = threadIdx.x;
  const float* ml = part_ml + static_cast<size_t>(row) * num_splits * 2;
  const float* po = part_o + static_cast<size_t>(row) * num_splits * 128 + d;
  float m = -INFINITY, l = 0.f, acc = 0.f;
  for (int s0 = 0; s0 < num_splits; s0 += U) {
    float mp[U], lp[U], op[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = s0 + u < num_splits;
      mp[u] = ok ? __ldcg(ml + 2 * (s0 + u)) : -INFINITY;
      lp[u] = ok ? __ldcg(ml + 2 * (s0 + u) + 1) : 0.f;
      op[u] = ok ? __ldcg(po + static_cast<size_t>(s0 + u) * 128) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float mn = fmaxf(m, mp[u]);
      if (mn == -INFINITY) continue;
      const float wa = fast_exp2(m - mn), wb = fast_exp2(mp[u] - mn);
      l = fmaf(l, wa, lp[u] * wb);
      acc = fmaf(acc, wa, op[u] * wb);
      m = mn;
    }
  }
  o[static_cast<size_t>(row) * 128 + d] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
}

}  // namespace b200
