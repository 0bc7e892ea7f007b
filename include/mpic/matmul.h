// Row-major GEMM entry points of proj/include/mpic/matmul.h. In the B200 build they run
// on the device (SIMT fp32, fixed per-element reduction order) — kept for API
// completeness; the selective pass itself never goes through them.
#pragma once

#include <cstdint>

namespace mpic {

// C[m x n] = A[m x k] * B[n x k]^T
void gemm_nt(int m, int n, int k, const float* a, int lda, const float* b, int ldb, float* c, int ldc);
// C[m x n] = A[m x k] * B[k x n]
void gemm_nn(int m, int n, int k, const float* a, int lda, const float* b, int ldb, float* c, int ldc);
// Reference knob for the BLAS thread pool; recorded, no effect on the GPU path.
void set_compute_threads(int n);

}  // namespace mpic
