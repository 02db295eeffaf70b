/* ORACLE TEST INFRASTRUCTURE -- see oracle.h.
 *
 * fp32 restatement of the GEMM mainloop graph (LDA, LDB -> MMA with a
 * loop-carried accumulator, the simplest iterative loop the reference's
 * scheduler accepts; cf. the blocking/GEMM fixtures in
 * proj/tests/testutil.hpp:44-117). C[M,N] = A[M,K] * B[N,K]^T.
 */
#include <stdint.h>

#include "oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

void oracle_gemm_tn(const float* a, const float* b, float* c, int M, int N,
                    int K, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    const float* ai = a + (int64_t)i * K;
    for (int j = 0; j < N; ++j) {
      const float* bj = b + (int64_t)j * K;
      double s = 0.0;
      for (int kk = 0; kk < K; ++kk) s += (double)ai[kk] * (double)bj[kk];
      c[(int64_t)i * N + j] = (float)s;
    }
  }
}
