// Microbenchmark: latency of fp64 log_add chains on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2101_05600_b200/csrc/softplus.cuh"
__constant__ bl::SpTables c_tb = {SP_THI_INIT, SP_TLO_INIT, SP_INV_INIT, SP_LH_INIT, SP_LL_INIT};
__device__ __forceinline__ double la_ref(double a, double b) {
  if (a < b) { double t = a; a = b; b = t; }
  if (b <= -1e29) return a <= -1e29 ? -1e30 : a;
  return a + log1p(exp(b - a));
}
__device__ __forceinline__ double la_sel(double a, double b) {  // branch-light
  double mx = fmax(a, b), mn = fmin(a, b);
  double r = mx + log1p(exp(mn - mx));
  r = (mn <= -1e29) ? mx : r;
  return (mx <= -1e29) ? -1e30 : r;
}
__global__ void k_chain1(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = la_ref(x, in[(i & 31)] - 3.0) - 0.5;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_chain3(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x], y = x + 1, z = x + 2;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double c = in[(i & 31)];
    x = la_ref(x, c - 3.0) - 0.5; y = la_ref(y, x - 1.0) - 0.25; z = la_ref(z, c - 1.0);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + y + z; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_chain3s(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x], y = x + 1, z = x + 2;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double c = in[(i & 31)];
    double xn = la_sel(x, c - 3.0) - 0.5; double yn = la_sel(y, x - 1.0) - 0.25; z = la_sel(z, c - 1.0);
    x = xn; y = yn;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + y + z; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_fast1(const double* in, double* out, int n, long long* cyc) {
  __shared__ bl::SpTables tb;
  for (int i = threadIdx.x; i < 320; i += blockDim.x) ((double*)&tb)[i] = ((const double*)&c_tb)[i];
  __syncthreads();
  double x = in[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = bl::log_add_fast(x, in[(i & 31)] - 3.0, tb) - 0.5;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_fast3(const double* in, double* out, int n, long long* cyc) {
  __shared__ bl::SpTables tb;
  for (int i = threadIdx.x; i < 320; i += blockDim.x) ((double*)&tb)[i] = ((const double*)&c_tb)[i];
  __syncthreads();
  double x = in[threadIdx.x], y = x + 1, z = x + 2;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double c = in[(i & 31)];
    double xn = bl::log_add_fast(x, c - 3.0, tb) - 0.5; double yn = bl::log_add_fast(y, x - 1.0, tb) - 0.25; z = bl::log_add_fast(z, c - 1.0, tb);
    x = xn; y = yn;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + y + z; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_exp(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = exp(-x) - 0.3;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_log1p(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = log1p(x) + 0.01;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_log(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x] + 2;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = log(x) + 1.5;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(const double* in, double* out, int n, long long* cyc) {
  double x = in[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 0.001);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double h[32]; for (int i = 0; i < 32; ++i) h[i] = -100.0 - i * 0.37;
  double *din, *dout; long long* dc; long long hc;
  cudaMalloc(&din, 256); cudaMalloc(&dout, 256 * 8); cudaMalloc(&dc, 8);
  cudaMemcpy(din, h, 256, cudaMemcpyHostToDevice);
  const int n = 4096;
  auto run = [&](const char* name, void (*k)(const double*, double*, int, long long*), int threads, double per) {
    k<<<1, threads>>>(din, dout, n, dc); cudaDeviceSynchronize();
    k<<<1, threads>>>(din, dout, n, dc); cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s threads=%3d  %.1f cycles/iter  (%.1f per op)\n", name, threads, (double)hc / n, (double)hc / n / per);
  };
  for (int th : {1, 32}) {
    run("dfma chain", k_dfma, th, 1);
    run("exp chain", k_exp, th, 1);
    run("log1p chain", k_log1p, th, 1);
    run("log chain", k_log, th, 1);
    run("log_add chain (1)", k_chain1, th, 1);
    run("log_add 3 chains (ref)", k_chain3, th, 3);
    run("log_add 3 chains (select)", k_chain3s, th, 3);
    run("log_add_fast chain (1)", k_fast1, th, 1);
    run("log_add_fast 3 chains", k_fast3, th, 3);
  }
  return 0;
}
