#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, int n, long long* cyc) {
  double x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 0.001 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], 0.9999, 0.0001);
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int ILP>
__global__ void kf(float* out, int n, long long* cyc) {
  float x[ILP];
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 0.001f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fmaf(x[i], 0.9999f, 0.0001f);
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; float* of; long long* c; long long h;
  cudaMalloc(&o, 1 << 24); cudaMalloc(&of, 1 << 24); cudaMalloc(&c, 8);
  const int n = 2048;
  for (int warps : {1, 4, 8, 32}) {
    k<8><<<1, 32 * warps>>>(o, n, c); cudaDeviceSynchronize();
    k<8><<<1, 32 * warps>>>(o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double instr = (double)n * 8 * warps;  // warp-instructions
    printf("DFMA  warps=%2d ILP=8: %.2f cycles per warp-instr per SM  -> %.1f lanes/clk/SM\n", warps, h / instr, 32.0 * instr / h);
    kf<8><<<1, 32 * warps>>>(of, n, c); cudaDeviceSynchronize();
    kf<8><<<1, 32 * warps>>>(of, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FFMA  warps=%2d ILP=8: %.2f cycles per warp-instr per SM  -> %.1f lanes/clk/SM\n", warps, h / instr, 32.0 * instr / h);
  }
}
