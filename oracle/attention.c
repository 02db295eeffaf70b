/* ORACLE TEST INFRASTRUCTURE -- see oracle.h for provenance and scope.
 *
 * Restates the FA-forward loop of the Twill paper for the CPU:
 *   loop body  S = gemm(Q, K[i]); P = exp(S); O += gemm(P, V[i])
 *              (reference: proj/tests/testutil.hpp:13-15)
 *   online form with running max / rescale of the accumulator
 *              (Fig. 1f; the CR "correction" op of the
 *               Blackwell schedule)
 * Numerics are parity-UNPINNED: the reference has no attention numerics.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

static void set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

void oracle_attention(const float* q, const float* k, const float* v, float* o,
                      float* lse, int B, int H, int Sq, int Sk, int D,
                      int causal, float scale, int threads) {
  set_threads(threads);
  const int S = Sk;
  const int64_t rows = (int64_t)B * H * Sq;
#pragma omp parallel
  {
    double* p = (double*)malloc(sizeof(double) * (size_t)S);
    double* acc = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(dynamic, 16)
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t bh = r / Sq;
      const int i = (int)(r % Sq);
      const float* qi = q + r * D;
      const float* kb = k + bh * (int64_t)S * D;
      const float* vb = v + bh * (int64_t)S * D;
      const int nkeys = causal ? (i + 1 < S ? i + 1 : S) : S;
      double m = -INFINITY;
      for (int j = 0; j < nkeys; ++j) {
        const float* kj = kb + (int64_t)j * D;
        double s = 0.0;
        for (int c = 0; c < D; ++c) s += (double)qi[c] * (double)kj[c];
        s *= (double)scale;
        p[j] = s;
        if (s > m) m = s;
      }
      double l = 0.0;
      for (int j = 0; j < nkeys; ++j) {
        p[j] = exp(p[j] - m);
        l += p[j];
      }
      for (int c = 0; c < D; ++c) acc[c] = 0.0;
      for (int j = 0; j < nkeys; ++j) {
        const float* vj = vb + (int64_t)j * D;
        const double pj = p[j];
        for (int c = 0; c < D; ++c) acc[c] += pj * (double)vj[c];
      }
      float* oi = o + r * D;
      for (int c = 0; c < D; ++c) oi[c] = (float)(acc[c] / l);
      if (lse) lse[r] = (float)(m + log(l));
    }
    free(p);
    free(acc);
  }
}

void oracle_attention_online(const float* q, const float* k, const float* v,
                             float* o, float* lse, int B, int H, int Sq, int Sk,
                             int D, int causal, float scale, int tile,
                             int threads) {
  set_threads(threads);
  if (tile <= 0) tile = 128;
  const int S = Sk;
  const int64_t rows = (int64_t)B * H * Sq;
#pragma omp parallel
  {
    float* s = (float*)malloc(sizeof(float) * (size_t)tile);
    float* acc = (float*)malloc(sizeof(float) * (size_t)D);
#pragma omp for schedule(dynamic, 16)
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t bh = r / Sq;
      const int i = (int)(r % Sq);
      const float* qi = q + r * D;
      const float* kb = k + bh * (int64_t)S * D;
      const float* vb = v + bh * (int64_t)S * D;
      const int nkeys = causal ? (i + 1 < S ? i + 1 : S) : S;
      float m = -INFINITY, l = 0.0f;
      for (int c = 0; c < D; ++c) acc[c] = 0.0f;
      for (int j0 = 0; j0 < nkeys; j0 += tile) {
        const int jn = (nkeys - j0) < tile ? (nkeys - j0) : tile;
        /* S_i = Q K[i]^T (the tile's QK GEMM) and its row max (MX) */
        float mt = m;
        for (int j = 0; j < jn; ++j) {
          const float* kj = kb + (int64_t)(j0 + j) * D;
          float t = 0.0f;
          for (int c = 0; c < D; ++c) t += qi[c] * kj[c];
          s[j] = t * scale;
          if (s[j] > mt) mt = s[j];
        }
        /* correction of the carried accumulator (CR) */
        const float alpha = (m == -INFINITY) ? 0.0f : expf(m - mt);
        l *= alpha;
        for (int c = 0; c < D; ++c) acc[c] *= alpha;
        m = mt;
        /* P = exp(S - m) (EX) and O += P V[i] (PV) */
        for (int j = 0; j < jn; ++j) {
          const float pj = expf(s[j] - m);
          l += pj;
          const float* vj = vb + (int64_t)(j0 + j) * D;
          for (int c = 0; c < D; ++c) acc[c] += pj * vj[c];
        }
      }
      float* oi = o + r * D;
      for (int c = 0; c < D; ++c) oi[c] = acc[c] / l;
      if (lse) lse[r] = m + logf(l);
    }
    free(s);
    free(acc);
  }
}

void oracle_round_bf16(float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u;
    memcpy(&u, &x[i], 4);
    if ((u & 0x7f800000u) != 0x7f800000u) {
      const uint32_t lsb = (u >> 16) & 1u;
      u += 0x7fffu + lsb;
    }
    u &= 0xffff0000u;
    memcpy(&x[i], &u, 4);
  }
}
