// umma_tf32.cu — layout check for the tensor-core prefix-score bulk (P3):
//   A = the TMA stage of the CTC slab, [col block][8 rows][32 fp32 cols]
//       (3D box, SWIZZLE_128B) used in place as the MN-major tf32 operand
//       (M = 128 columns = 4 swizzle atoms 1024 B apart, K = 8 rows);
//   B = parent factors, K-major SWIZZLE_NONE core matrices
//       (N = 16 parents, K = 8 rows, LBO 128 B, SBO 256 B);
//   D = fp32 [128 lanes][16 columns] per M subtile in TMEM, read back with
//       tcgen05.ld.32x32b.x16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_tf32 umma_tf32.cu -lcuda
// Prints the max relative error vs a CPU fp64 product over 2 chained K chunks.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2101_05600_b200/csrc/tc_ptx.cuh"

using namespace bl::tc;

constexpr int kRows = 16, kCols = 1024, kTile = 512, kN = 16;

__device__ __forceinline__ uint64_t desc_mn_sw128(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (s32(p) & 0x3FFFF) >> 4;
  return a | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_kmaj_none(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (s32(p) & 0x3FFFF) >> 4;
  return a | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, int x, int y, int z,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(s32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(s32(bar))
      : "memory");
}

// C[c][n] = sum_r A[r][c] * Bf[n][r] over rows 0..15 (two K chunks), columns 0..511
__global__ void __launch_bounds__(256) k(const __grid_constant__ CUtensorMap tm, const float* bf,
                                         float* out, int mode, int dtype, int lbo, int sbo) {
  extern __shared__ unsigned char dsm_raw[];
  float(*stage)[kTile * 8] = reinterpret_cast<float(*)[kTile * 8]>(
      (reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~(uintptr_t)1023);
  float(*akm)[kTile * 8] = stage + 2;  // mode 3: A K-major interleave
  __shared__ __align__(128) float bsm[2][kN * 8];
  __shared__ __align__(8) uint64_t bar[2], mdone;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s32(&tbase)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mb_init(&bar[0], 1);
    mb_init(&bar[1], 1);
    mb_init(&mdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B: [chunk][n/8][k/4][n%8][k%4] (core matrices 128 B, LBO 128 B, SBO 256 B)
  for (int i = tid; i < 2 * kN * 8; i += 256) {
    const int ch = i / (kN * 8), rem = i % (kN * 8), n = rem / 8, kk = rem % 8;
    const int off = (n / 8) * 64 + (kk / 4) * 32 + (n % 8) * 4 + (kk % 4);
    bsm[ch][off] = bf[n * kRows + ch * 8 + kk];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    for (int ch = 0; ch < 2; ++ch) {
      mb_expect_tx(&bar[ch], kTile * 8 * 4);
      tma3d(stage[ch], &tm, 0, ch * 8, 0, &bar[ch]);
    }
  }
  for (int ch = 0; ch < 2; ++ch) mb_wait(&bar[ch], 0);
  if (mode == 1) {  // in-place transform: x -> x * 0.5 (checks generic writes -> async proxy)
    for (int i = tid; i < kTile * 8; i += 256) {
      stage[0][i] *= 0.5f;
      stage[1][i] *= 0.5f;
    }
  }
  if (mode == 4) {  // position-dependent: x(r, c) *= 1 + c / 512, addressed by the 32B-atom swizzle
    for (int i = tid; i < kTile * 8; i += 256) {
      const int r = i / kTile, c = i % kTile;
      const int blk = c / 32, cc = c % 32;
      const int off = blk * 256 + r * 32 + ((((cc >> 3) ^ r) & 3) << 3) + (cc & 7);
      stage[0][off] *= 1.f + c / 512.f;
      stage[1][off] *= 1.f + c / 512.f;
    }
  }
  if (mode == 3) {  // A K-major SWIZZLE_NONE: [m/8][k/4][m%8][k%4], LBO 128 B (k chunks), SBO 256 B
    for (int i = tid; i < kTile * 8; i += 256) {
      const int r = i / kTile, c = i % kTile;
      const int blk = c / 32, cc = c % 32;
      const float x = stage[0][blk * 256 + r * 32 + ((((cc >> 2) ^ r) & 7) << 2) + (cc & 3)];
      const int m = c % 128, sub = c / 128;
      akm[0][sub * 1024 + (m / 8) * 64 + (r / 4) * 32 + (m % 8) * 4 + (r % 4)] = x;
      const float x1 = stage[1][blk * 256 + r * 32 + ((((cc >> 2) ^ r) & 7) << 2) + (cc & 3)];
      akm[1][sub * 1024 + (m / 8) * 64 + (r / 4) * 32 + (m % 8) * 4 + (r % 4)] = x1;
    }
  }
  if (mode == 2) {  // TMEM st/ld round trip: D[c][n] = c + n / 100
    for (int h = 0; h < 2; ++h) {
      const int sub = (warp >> 2) * 2 + h;
      const int c = sub * 128 + 32 * (warp & 3) + lane;
      float v[16];
      for (int n = 0; n < 16; ++n) v[n] = c + n / 100.f;
      tmem_st16(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + sub * kN, v);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0 && mode == 2) umma_commit(&mdone);
  if (tid == 0 && mode == 3) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                           ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int ch = 0; ch < 2; ++ch)
      for (int sub = 0; sub < 4; ++sub)
        umma_tf32(tmem + sub * kN, desc_kmaj_none(&akm[ch][sub * 1024], 128, 256),
                  desc_kmaj_none(bsm[ch], 128, 256), idesc, ch > 0 ? 1u : 0u);
    umma_commit(&mdone);
  }
  if (tid == 0 && (mode < 2 || mode == 4)) {
    // c_format F32 @4, a TF32 (2) @7, b TF32 (2) @10, A MN-major @15, N/8 @17, M/16 @24
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                           ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int ch = 0; ch < 2; ++ch)
      for (int sub = 0; sub < 4; ++sub) {
        const uint64_t da = (desc_mn_sw128(&stage[ch][sub * 4 * 256], lbo, sbo) &
                             ~(7ull << 61)) | ((uint64_t)dtype << 61);
        const uint64_t db = desc_kmaj_none(bsm[ch], 128, 256);
        umma_tf32(tmem + sub * kN, da, db, idesc, ch > 0 ? 1u : 0u);
      }
    umma_commit(&mdone);
  }
  mb_wait(&mdone, 0);
  tc_fence_after();
  // warp w reads lanes 32*(w%4).. of subtiles (w/4)*2, (w/4)*2+1
  for (int h = 0; h < 2; ++h) {
    const int sub = (warp >> 2) * 2 + h;
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + sub * kN, v);
    const int c = sub * 128 + 32 * (warp & 3) + lane;
    for (int n = 0; n < kN; ++n) out[c * kN + n] = v[n];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  std::vector<float> A(kRows * kCols), Bf(kN * kRows);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX;
  for (auto& x : Bf) x = (float)rand() / RAND_MAX;
  float *dA, *dB, *dO;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, Bf.size() * 4);
  cudaMalloc(&dO, kTile * kN * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bf.data(), Bf.size() * 4, cudaMemcpyHostToDevice);
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  for (int variant = 0; variant < 4; ++variant) {
  const CUtensorMapSwizzle swz = variant == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  const int dtype = variant == 0 ? 2 : 1;
  const int lbo = variant == 3 ? 512 : 1024, sbo = variant == 3 ? 1024 : (variant == 2 ? 512 : 8192);
  printf("== variant %d: tma swizzle %d desc type %d lbo %d sbo %d\n", variant, (int)swz, dtype, lbo, sbo);
  CUtensorMap tm;
  // dims: (col in block 32, row, col block); strides (bytes) for dims 1, 2
  const cuuint64_t dims[3] = {32, (cuuint64_t)kRows, (cuuint64_t)(kCols / 32)};
  const cuuint64_t strides[2] = {(cuuint64_t)kCols * 4, 128};
  const cuuint32_t box[3] = {32, 8, 16};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dA, dims,
                                              strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              swz,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)r);
  const int dyn = 4 * kTile * 8 * 4 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
  for (int mode = 0; mode < 5; ++mode) {
    if (variant > 0 && (mode == 2 || mode == 3)) continue;
    cudaMemset(dO, 0, kTile * kN * 4);
    k<<<1, 256, dyn>>>(tm, dB, dO, mode, dtype, lbo, sbo);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
    std::vector<float> O(kTile * kN);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    int bad = 0;
    for (int c = 0; c < kTile; ++c)
      for (int n = 0; n < kN; ++n) {
        double ref = 0;
        for (int t = 0; t < kRows; ++t)
          ref += (double)A[t * kCols + c] * (mode == 1 ? 0.5 : mode == 4 ? 1.0 + c / 512.0 : 1.0) *
                 Bf[n * kRows + t];
        if (mode == 2) ref = c + n / 100.0;
        const double rel = std::fabs(O[c * kN + n] - ref) / std::fmax(1e-9, std::fabs(ref));
        if (rel > worst) worst = rel;
        if (rel > 4e-3 && bad++ < 2)
          printf("  c=%d n=%d got %g want %g\n", c, n, O[c * kN + n], ref);
      }
    printf("mode %d: max rel err %.3g, bad %d\n", mode, worst, bad);
  }
  }
  return 0;
}
