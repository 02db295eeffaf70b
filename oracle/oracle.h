/* ORACLE TEST INFRASTRUCTURE -- never linked into the product.
 *
 * CPU restatement of the FA-forward loop the reference schedules and of the
 * GEMM mainloop. The reference ships no numerics for this path (it is an
 * integer scheduler), so the loop semantics are taken from
 * the reference's own statement of the loop body:
 *   S = gemm(Q, K[i]); P = exp(S); O += gemm(P, V[i])
 *       /root/reference/proj/tests/testutil.hpp:13-15
 * and the pipelined online-softmax order of Fig. 1f.
 * Numerics parity is therefore UNPINNED by the reference: there are no golden
 * attention outputs to check against. The schedule side IS pinned (see
 * tests/golden and tests/test_oracle_ref.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef TWFA_ORACLE_H
#define TWFA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Plain two-pass softmax attention, fp32 inputs, double accumulation.
 * q,o: [B,H,Sq,D], k,v: [B,H,Sk,D] contiguous (the queries are the first Sq
 * rows of the sequence); lse: [B,H,Sq] natural-log sum-exp of the scaled
 * scores (may be NULL). causal: key j visible to query i iff j <= i. */
void oracle_attention(const float* q, const float* k, const float* v, float* o,
                      float* lse, int B, int H, int Sq, int Sk, int D,
                      int causal, float scale, int threads);

/* Online-softmax restatement in the loop order of the Twill FA body:
 * per KV tile of `tile` keys: S = Q K^T (fp32), running max m, P = exp(S - m),
 * O = O * exp(m_old - m) + P V, l likewise; O /= l at the end. fp32 throughout.
 * Same layouts as oracle_attention. */
void oracle_attention_online(const float* q, const float* k, const float* v,
                             float* o, float* lse, int B, int H, int Sq, int Sk,
                             int D, int causal, float scale, int tile,
                             int threads);

/* C[M,N] = A[M,K] * B[N,K]^T (both operands K-contiguous), fp32 with double
 * accumulation. */
void oracle_gemm_tn(const float* a, const float* b, float* c, int M, int N,
                    int K, int threads);

/* Round-to-nearest-even float -> bf16 -> float, the kernel's input rounding. */
void oracle_round_bf16(float* x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
