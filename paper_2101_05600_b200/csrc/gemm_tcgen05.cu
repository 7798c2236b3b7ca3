// gemm_tcgen05.cu — bf16 GEMM on the sm_100a 5th-generation tensor cores for
// the encoder (SURVEY §8 a'1): C[M,N] = A[M,K] · B[N,K]^T, fp32 accumulation
// in tensor memory, fused epilogue (bias, ReLU, residual, scale + positional
// encoding), bf16 or fp32 output.
//
// One CTA (128 threads) per 128x128 output tile:
//   thread 0   : TMA producer (cp.async.bulk.tensor.2d, SWIZZLE_128B) into a
//                kStages-deep shared-memory ring guarded by full/empty mbarriers
//   thread 32  : single-thread tcgen05.mma.cta_group::1.kind::f16 issuer
//                (M=128, N=128, K=16 per instruction, 4 per 64-wide K tile);
//                tcgen05.commit releases ring slots and signals the epilogue
//   warps 0-3  : epilogue, tcgen05.ld.32x32b (warp w owns TMEM lanes 32w..)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm.cuh"

namespace bl {
namespace {

constexpr int kBM = 128, kBN = 128, kBK = 64, kStages = 4;
constexpr int kTileABytes = kBM * kBK * 2;  // 16 KB
constexpr int kTileBBytes = kBN * kBK * 2;  // 16 KB
constexpr int kStageBytes = kTileABytes + kTileBBytes;

__device__ __forceinline__ unsigned s32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(s32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int x, int y,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(s32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(s32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B (8-row x 128-byte
// atoms, 1024 B apart): start>>4 @0, LBO=1 @16, SBO=1024>>4 @32,
// version=1 @46, layout=2 (SWIZZLE_128B) @61.
__device__ __forceinline__ uint64_t umma_desc(const void* smem) {
  const uint64_t a = (s32(smem) & 0x3FFFF) >> 4;
  return a | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D=f32, A=B=bf16, K-major both, N>>3 @17, M>>4 @24
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   s32(bar))
               : "memory");
}

struct GemmArgs {
  int M, N, K;
  int mode;             // GemmEpilogue
  const float* bias;    // [N] or null
  float* out_f32;       // [M, ldo]
  __nv_bfloat16* out_bf16;
  int ldo;
  float scale;          // kScalePe: out = acc*scale + bias*scale + pe[row % pe_rows][col]
  const float* pe;
  int pe_rows;
};

__global__ void __launch_bounds__(128, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                const GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  const int KT = (g.K + kBK - 1) / kBK;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 128 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s32(&tmem_base)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (tid == 0) {
    // ---- TMA producer ----
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % kStages;
      if (kt >= kStages) mb_wait(&empty[s], ((kt / kStages) - 1) & 1);
      unsigned char* st = smem + (size_t)s * kStageBytes;
      mb_expect_tx(&full[s], kStageBytes);
      tma2d(st, &tA, kt * kBK, m0, &full[s]);
      tma2d(st + kTileABytes, &tB, kt * kBK, n0, &full[s]);
    }
  } else if (tid == 32) {
    // ---- MMA issuer ----
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % kStages;
      mb_wait(&full[s], (kt / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const unsigned char* st = smem + (size_t)s * kStageBytes;
      const uint64_t da = umma_desc(st), db = umma_desc(st + kTileABytes);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)  // +32 bytes along K per MMA (>>4 = 2)
        umma(tmem, da + 2ull * k, db + 2ull * k, (kt > 0 || k > 0) ? 1u : 0u);
      umma_commit(&empty[s]);  // slot free once these MMAs have read it
    }
    umma_commit(&done);
  }
  __syncwarp();

  // ---- epilogue: TMEM -> registers -> global ----
  mb_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = m0 + warp * 32 + lane;
  for (int c0 = 0; c0 < kBN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < g.M) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = n0 + c0 + j;
        if (col >= g.N) break;
        float x = __uint_as_float(v[j]);
        if (g.bias) x += g.bias[col];
        const size_t o = (size_t)row * g.ldo + col;
        switch (g.mode) {
          case kRelu: x = fmaxf(x, 0.f); break;
          case kResidual: x += g.out_f32[o]; break;
          case kScalePe: x = x * g.scale + g.pe[(size_t)(row % g.pe_rows) * g.N + col]; break;
          default: break;
        }
        if (g.out_bf16) g.out_bf16[o] = __float2bfloat16_rn(x);
        if (g.out_f32) g.out_f32[o] = x;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// K-major bf16 operand [rows, K] (row stride ld elements), box 64 x 128, SW128
bool make_map(CUtensorMap* m, const void* base, int rows, int K, int ld) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace

cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t st) {
  if (d.K % 8 != 0 || d.lda % 8 != 0 || d.ldb % 8 != 0) return cudaErrorInvalidValue;
  CUtensorMap tA, tB;
  if (!make_map(&tA, d.A, d.M, d.K, d.lda) || !make_map(&tB, d.B, d.N, d.K, d.ldb))
    return cudaErrorInvalidValue;
  GemmArgs g{d.M, d.N, d.K, d.mode, d.bias, d.out_f32, d.out_bf16, d.ldo, d.scale, d.pe,
             d.pe_rows};
  const int smem = kStages * kStageBytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((d.N + kBN - 1) / kBN, (d.M + kBM - 1) / kBM);
  gemm_kernel<<<grid, 128, smem, st>>>(tA, tB, g);
  return cudaGetLastError();
}

}  // namespace bl
