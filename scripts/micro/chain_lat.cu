// Dependent-latency microbenchmark of the chain step g = log_add(g, b) + x
// (softplus.cuh) on one warp: cycles per step, tables in shared memory.
#include <cstdio>
#include "../../paper_2101_05600_b200/csrc/softplus.cuh"
using namespace bl;
__constant__ SpTables c_tb = {SP_THI_INIT, SP_TLO_INIT, SP_INV_INIT, SP_LH_INIT, SP_LL_INIT};
__global__ void k(const double* b, const float* x, int n, double* out, long long* cyc, int mode) {
  __shared__ SpTables tb;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    tb.thi[i] = c_tb.thi[i]; tb.tlo[i] = c_tb.tlo[i]; tb.inv[i] = c_tb.inv[i];
    tb.lh[i] = c_tb.lh[i]; tb.ll[i] = c_tb.ll[i];
  }
  __syncthreads();
  double g = -1.0, h = -2.0;
  const long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < n; ++i) g = log_add_fast(g, b[i & 255], tb) + (double)x[i & 255];
  } else if (mode == 1) {
    for (int i = 0; i < n; ++i) g = exp_neg(-fabs(g) * 1e-3 - b[i & 255] * 1e-3, tb) - 1.0;
  } else {
    for (int i = 0; i < n; ++i) g = log_pos(2.0 - g * 1e-3 + b[i & 255] * 1e-6, tb);
  }
  const long long t1 = clock64();
  out[threadIdx.x] = g + h;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* b; float* x; double* o; long long* c;
  cudaMalloc(&b, 256 * 8); cudaMalloc(&x, 256 * 4); cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  double hb[256]; float hx[256];
  for (int i = 0; i < 256; ++i) { hb[i] = -1.0 - (i % 17); hx[i] = -0.01f * (i % 5); }
  cudaMemcpy(b, hb, sizeof hb, cudaMemcpyHostToDevice);
  cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice);
  const char* names[3] = {"log_add chain", "exp_neg chain", "log_pos chain"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {1, 8, 24}) {
      k<<<1, 32 * warps>>>(b, x, 4096, o, c, mode);
      k<<<1, 32 * warps>>>(b, x, 4096, o, c, mode);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%s, %d warps/SM: %.1f cycles per step\n", names[mode], warps, h / 4096.0);
    }
  }
  return 0;
}
