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

void oracle_attention_bwd(const float* q, const float* k, const float* v,
                          const float* o, const float* dout, const float* lse,
                          float* dq, float* dk, float* dv, int B, int H, int S,
                          int D, int causal, float scale, int threads) {
  set_threads(threads);
  const int BH = B * H;
#pragma omp parallel for schedule(dynamic, 1)
  for (int bh = 0; bh < BH; ++bh) {
    const int64_t base = (int64_t)bh * S * D;
    const float *qb = q + base, *kb = k + base, *vb = v + base, *ob = o + base, *gb = dout + base;
    const float* lb = lse + (int64_t)bh * S;
    double* dqa = (double*)calloc((size_t)S * D, sizeof(double));
    double* dka = (double*)calloc((size_t)S * D, sizeof(double));
    double* dva = (double*)calloc((size_t)S * D, sizeof(double));
    for (int i = 0; i < S; ++i) {
      const float* qi = qb + (int64_t)i * D;
      const float* gi = gb + (int64_t)i * D;
      double Di = 0.0;
      for (int c = 0; c < D; ++c) Di += (double)gi[c] * (double)ob[(int64_t)i * D + c];
      const int nkeys = causal ? (i + 1 < S ? i + 1 : S) : S;
      for (int j = 0; j < nkeys; ++j) {
        const float* kj = kb + (int64_t)j * D;
        const float* vj = vb + (int64_t)j * D;
        double s = 0.0, dp = 0.0;
        for (int c = 0; c < D; ++c) {
          s += (double)qi[c] * (double)kj[c];
          dp += (double)gi[c] * (double)vj[c];
        }
        const double p = exp(s * (double)scale - (double)lb[i]);
        const double ds = p * (dp - Di);
        double* dvj = dva + (int64_t)j * D;
        double* dkj = dka + (int64_t)j * D;
        double* dqi = dqa + (int64_t)i * D;
        for (int c = 0; c < D; ++c) {
          dvj[c] += p * (double)gi[c];
          dkj[c] += ds * (double)qi[c];
          dqi[c] += ds * (double)kj[c];
        }
      }
    }
    for (int64_t e = 0; e < (int64_t)S * D; ++e) {
      dq[base + e] = (float)(dqa[e] * (double)scale);
      dk[base + e] = (float)(dka[e] * (double)scale);
      dv[base + e] = (float)dva[e];
    }
    free(dqa);
    free(dka);
    free(dva);
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
