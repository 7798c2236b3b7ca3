// gemm.cuh — host interface of the tcgen05 bf16 GEMM (gemm_tcgen05.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace bl {

enum GemmEpilogue : int {
  kPlain = 0,     // out = acc (+ bias)
  kRelu = 1,      // out = max(acc + bias, 0)
  kResidual = 2,  // out_f32 += acc + bias   (in place residual stream)
  kScalePe = 3,   // out = (acc + bias) * scale + pe[row % pe_rows][col]
  kLsePart = 4,   // out = acc + bias, plus per (row, 128-column slot) the
                  // partial log-softmax {max (as double), sum exp(x - max)
                  // (fp64)} in lse_part[row][lse_stride] (a tile writes its
                  // first slot; the caller zeroes the buffer)
};

// C[M,N] = A[M,K] . B[N,K]^T; A, B bf16 K-major (row strides lda/ldb in
// elements, multiples of 8; K a multiple of 8). Either or both outputs.
struct GemmDesc {
  int M = 0, N = 0, K = 0;
  const __nv_bfloat16* A = nullptr;
  int lda = 0;
  const __nv_bfloat16* B = nullptr;
  int ldb = 0;
  int mode = kPlain;
  const float* bias = nullptr;
  float* out_f32 = nullptr;
  __nv_bfloat16* out_bf16 = nullptr;
  int ldo = 0;
  float scale = 1.f;
  const float* pe = nullptr;
  int pe_rows = 1;
  double* lse_part = nullptr;  // kLsePart: [M][lse_stride][2]
  int lse_stride = 0;
};

cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t st);

// conv2 (d -> d, 3x3, stride 2) + bias + ReLU as an implicit GEMM over the
// channel-last conv1 output c1[S][T1][F1][d]; W [d][(kh*3+kw)*d + c] bf16;
// out [S][T2][F2][d] bf16. No im2col buffer: the A tiles are 4D TMA boxes.
struct Conv2Desc {
  const __nv_bfloat16* c1 = nullptr;
  int S = 0, T1 = 0, F1 = 0, T2 = 0, F2 = 0, d = 0;
  const __nv_bfloat16* W = nullptr;
  const float* bias = nullptr;
  __nv_bfloat16* out = nullptr;
};
cudaError_t conv2_bf16(const Conv2Desc& c, cudaStream_t st);

// 2D row-major tensor map [rows][cols] (row stride ld_bytes), box box_cols x
// box_rows (cuTensorMapEncodeTiled through the runtime's driver entry point).
bool make_tmap(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int cols, int rows,
               size_t ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw);

}  // namespace bl
