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
/* Attention backward (the paper's second workload: the
 * single-pass algorithm of FA3), restated from the forward's definition
 * O = softmax(scale Q K^T) V with the recorded lse:
 *   P_ij  = exp(scale q_i.k_j - lse_i)        D_i = sum_c dO_ic O_ic
 *   dV_j  = sum_i P_ij dO_i                   dP_ij = dO_i . v_j
 *   dS_ij = P_ij (dP_ij - D_i)
 *   dQ_i  = scale sum_j dS_ij k_j             dK_j = scale sum_i dS_ij q_i
 * Layouts as oracle_attention (Sq = Sk = S); double accumulation. Parity is
 * unpinned like the forward (no reference numerics). */
void oracle_attention_bwd(const float* q, const float* k, const float* v,
                          const float* o, const float* dout, const float* lse,
                          float* dq, float* dk, float* dv, int B, int H, int S,
                          int D, int causal, float scale, int threads);

void oracle_gemm_tn(const float* a, const float* b, float* c, int M, int N,
                    int K, int threads);

/* Round-to-nearest-even float -> bf16 -> float, the kernel's input rounding. */
void oracle_round_bf16(float* x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
