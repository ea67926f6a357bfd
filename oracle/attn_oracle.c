/*
 * attn_oracle.c — CPU restatement of the attention forward the paper tunes. TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs as the checker. Never on the product path.
 *
 * What it restates (there is no attention arithmetic in the reference itself:
 * ref/SPEC.md:16 and ref/SPEC.md:605 put the FlashAttention-2 kernel out of scope):
 *   - FlashAttention-2 forward semantics of the paper's kernel (ref/PAPER.md:108-113):
 *     O = softmax(scale * Q K^T [+ causal mask]) V, scale = 1/sqrt(D),
 *     GQA: q head h reads kv head h / (Hq/Hkv)  (Llama-3 shapes, ref/PAPER.md:113);
 *   - varlen prefill over cu_seqlens with q_len == k_len per sequence, causal: key j
 *     visible to query i iff j <= i;
 *   - paged decode: one query per sequence at position n-1 attending to all n cached
 *     tokens, token t of sequence b at cache[block_table[b, t / bs], t % bs];
 *   - inputs are bf16 bit patterns (ref/pkg/runner/src/ktune_triton_runner/backends.py:119-137
 *     generates fp32 randn and casts to the kernel dtype); everything is accumulated in fp64.
 * Pinning: the third-party kernel this semantics comes from (vLLM 0.22.0
 * `triton_unified_attention`, the upstreamed form of the paper's IBM Triton kernel family,
 * ref/PAPER.md:110) is run under TRITON_INTERPRET=1 by tests/golden/make_golden.py; the
 * committed fixtures pin this file (tests/test_oracle.py).
 *
 * Build: oracle/Makefile -> oracle/_build/liboracle.so (OpenMP over heads / sequences).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline double bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* q [T, Hq, D], k/v [T, Hkv, D] (bf16 bits); out [T, Hq, D] fp64; lse [Hq, T] fp64 (nullable). */
void oracle_prefill(const uint16_t* q, const uint16_t* k, const uint16_t* v, const int32_t* cu_seqlens,
                    int num_seqs, int Hq, int Hkv, int D, int causal, double scale, double* out, double* lse) {
  const int G = Hq / Hkv;
  const int T = cu_seqlens[num_seqs];
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int s = 0; s < num_seqs; ++s) {
    for (int h = 0; h < Hq; ++h) {
      const int start = cu_seqlens[s], L = cu_seqlens[s + 1] - cu_seqlens[s];
      const int kvh = h / G;
      double* sc = (double*)malloc(sizeof(double) * (L > 0 ? L : 1));
      double* qv = (double*)malloc(sizeof(double) * D);
      for (int i = 0; i < L; ++i) {
        const uint16_t* qi = q + ((size_t)(start + i) * Hq + h) * D;
        for (int d = 0; d < D; ++d) qv[d] = bf16_to_double(qi[d]);
        const int nk = causal ? i + 1 : L;
        double m = -INFINITY;
        for (int j = 0; j < nk; ++j) {
          const uint16_t* kj = k + ((size_t)(start + j) * Hkv + kvh) * D;
          double acc = 0.0;
          for (int d = 0; d < D; ++d) acc += qv[d] * bf16_to_double(kj[d]);
          sc[j] = acc * scale;
          if (sc[j] > m) m = sc[j];
        }
        double l = 0.0;
        for (int j = 0; j < nk; ++j) {
          sc[j] = exp(sc[j] - m);
          l += sc[j];
        }
        double* o = out + ((size_t)(start + i) * Hq + h) * D;
        for (int d = 0; d < D; ++d) o[d] = 0.0;
        for (int j = 0; j < nk; ++j) {
          const uint16_t* vj = v + ((size_t)(start + j) * Hkv + kvh) * D;
          const double w = sc[j] / l;
          for (int d = 0; d < D; ++d) o[d] += w * bf16_to_double(vj[d]);
        }
        if (lse) lse[(size_t)h * T + start + i] = m + log(l);
      }
      free(sc);
      free(qv);
    }
  }
}

/* q [B, Hq, D]; caches [NB, bs, Hkv, D]; block_table [B, max_blocks]; seq_lens [B]; out [B, Hq, D] fp64. */
void oracle_decode(const uint16_t* q, const uint16_t* kc, const uint16_t* vc, const int32_t* block_table,
                   const int32_t* seq_lens, int B, int Hq, int Hkv, int D, int bs, int max_blocks, double scale,
                   double* out) {
  const int G = Hq / Hkv;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < B; ++b) {
    for (int h = 0; h < Hq; ++h) {
      const int n = seq_lens[b];
      const int kvh = h / G;
      double* sc = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
      double qv[512];
      const uint16_t* qb = q + ((size_t)b * Hq + h) * D;
      for (int d = 0; d < D; ++d) qv[d] = bf16_to_double(qb[d]);
      double m = -INFINITY;
      for (int t = 0; t < n; ++t) {
        const int page = block_table[(size_t)b * max_blocks + t / bs];
        const uint16_t* kt = kc + (((size_t)page * bs + t % bs) * Hkv + kvh) * D;
        double acc = 0.0;
        for (int d = 0; d < D; ++d) acc += qv[d] * bf16_to_double(kt[d]);
        sc[t] = acc * scale;
        if (sc[t] > m) m = sc[t];
      }
      double l = 0.0;
      for (int t = 0; t < n; ++t) {
        sc[t] = exp(sc[t] - m);
        l += sc[t];
      }
      double* o = out + ((size_t)b * Hq + h) * D;
      for (int d = 0; d < D; ++d) o[d] = 0.0;
      for (int t = 0; t < n; ++t) {
        const int page = block_table[(size_t)b * max_blocks + t / bs];
        const uint16_t* vt = vc + (((size_t)page * bs + t % bs) * Hkv + kvh) * D;
        const double w = sc[t] / l;
        for (int d = 0; d < D; ++d) o[d] += w * bf16_to_double(vt[d]);
      }
      free(sc);
    }
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
