// gemm_tcgen05.cu — bf16 GEMM on the sm_100a 5th-generation tensor cores for
// the encoder (SURVEY §8 a'1): C[M,N] = A[M,K] · B[N,K]^T, fp32 accumulation
// in tensor memory, fused epilogue (bias, ReLU, residual, scale + positional
// table), bf16 and/or fp32 output.
//
// Persistent, warp-specialised kernel, one CTA per SM, 192 threads:
//   warp 0 (one lane) : TMA producer — cp.async.bulk.tensor.2d (SWIZZLE_128B)
//                       of A[128 x 64] and B[BN x 64] tiles into a kStages ring
//                       guarded by full/empty mbarriers
//   warp 1 (one lane) : MMA issuer — tcgen05.mma.cta_group::1.kind::f16,
//                       M=128, N=BN, K=16 (4 per 64-wide K tile); commits
//                       release ring slots and publish finished accumulators
//   warps 2-5         : epilogue — tcgen05.ld.32x32b (warp w reads TMEM lanes
//                       32*(w%4)..), transpose through shared memory, coalesced
//                       row stores with the fused epilogue math
// The accumulator is double-buffered in TMEM (2 x BN fp32 columns), so the
// epilogue of tile i overlaps the main loop of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace bl {

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

// 2D row-major tensor [rows][cols] (row stride ld_bytes), box box_cols x box_rows
bool make_tmap(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int cols, int rows,
               size_t ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

using namespace tc;

constexpr int kBM = 128, kBK = 64;
constexpr int kThreads = 192;
constexpr int kStgBytes = 32 * 128;          // one 32-row x 128-byte staging tile
constexpr int kEpiBytes = 4 * 2 * kStgBytes;  // 4 epilogue warps, double-buffered

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kA = kBM * kBK * 2;
  static constexpr int kB = BN * kBK * 2;
  static constexpr int kStage = kA + kB;
  static constexpr int kSmem = kStages * kStage + kEpiBytes + 1024;
  static constexpr int kTmemCols = 2 * BN;  // power of two >= 32
  // instruction descriptor: D=f32 (bit 4), A=B=bf16 (bits 7, 10), K-major,
  // N>>3 at bit 17, M>>4 at bit 24
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) |
                                     ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

struct GemmArgs {
  int M, N, K;
  int mode;  // GemmEpilogue
  const float* bias;
  float* out_f32;
  __nv_bfloat16* out_bf16;
  int ldo;
  float scale;
  const float* pe;
  int pe_rows;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                const __grid_constant__ CUtensorMap tOb, const __grid_constant__ CUtensorMap tOf,
                const GemmArgs g) {
  using C = Cfg<BN>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* epi = smem + S * C::kStage;
  __shared__ __align__(8) uint64_t full[S], empty[S], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = (g.K + kBK - 1) / kBK;
  const int tiles_n = (g.N + BN - 1) / BN;
  const int tiles = ((g.M + kBM - 1) / kBM) * tiles_n;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mb_init(&acc_full[a], 1);
      mb_init(&acc_empty[a], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s32(&tmem_base)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      int it = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int m0 = (tile / tiles_n) * kBM, n0 = (tile % tiles_n) * BN;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % S;
          if (it >= S) mb_wait(&empty[s], ((it / S) - 1) & 1);
          unsigned char* st = smem + (size_t)s * C::kStage;
          mb_expect_tx(&full[s], C::kStage);
          tma2d(st, &tA, kt * kBK, m0, &full[s]);
          tma2d(st + C::kA, &tB, kt * kBK, n0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      int it = 0, local = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
        const int a = local & 1, use = local >> 1;
        if (use > 0) mb_wait(&acc_empty[a], (use - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + (uint32_t)(a * BN);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % S;
          mb_wait(&full[s], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const unsigned char* st = smem + (size_t)s * C::kStage;
          const uint64_t da = umma_desc(st), db = umma_desc(st + C::kA);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // +32 B along K per MMA (>>4 = 2)
            umma(d, da + 2ull * k, db + 2ull * k, C::kIdesc, (kt > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[a]);
      }
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lane quarter q = warp % 4 ----
    // Each thread owns one accumulator row; a chunk of CW columns (128 bytes
    // of output) is converted in registers, written to a SWIZZLE_128B
    // staging tile (conflict-free: chunk c of row r lands at c ^ (r & 7)),
    // and one lane issues the bulk tensor store, which clips the M/N edges.
    const int q = warp & 3;
    constexpr int kCW32 = 32;
    const bool bf = g.out_bf16 != nullptr;
    const int CW = bf ? 64 : 32;
    unsigned char* stg = epi + (warp - 2) * 2 * kStgBytes;
    const CUtensorMap* tO = bf ? &tOb : &tOf;
    int local = 0, nchunk = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const int a = local & 1;
      const int m0 = (tile / tiles_n) * kBM, n0 = (tile % tiles_n) * BN;
      mb_wait(&acc_full[a], (local >> 1) & 1);
      tc_fence_after();
      const int rbase = m0 + q * 32, row = rbase + lane;
      const bool row_ok = row < g.M;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += CW, ++nchunk) {
        if (n0 + c0 >= g.N) break;
        float x[64];
        {
          uint32_t v[32];
          const uint32_t ta = tmem + (uint32_t)(a * BN + c0) + ((uint32_t)(q * 32) << 16);
          tmem_ld32(ta, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(v[j]);
          if (bf) {
            tmem_ld32(ta + 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) x[32 + j] = __uint_as_float(v[j]);
          }
        }
        const int col0 = n0 + c0;
        const bool full_cols = col0 + CW <= g.N;
        // bias (same address across the warp: broadcast loads)
        if (g.bias) {
          if (full_cols) {
            const float4* b4 = reinterpret_cast<const float4*>(g.bias + col0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j * 4 >= CW) break;
              const float4 b = __ldg(b4 + j);
              x[4 * j] += b.x; x[4 * j + 1] += b.y; x[4 * j + 2] += b.z; x[4 * j + 3] += b.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < CW && col0 + j < g.N) x[j] += __ldg(g.bias + col0 + j);
          }
        }
        if (g.mode == kRelu) {
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] = fmaxf(x[j], 0.f);
        } else if (g.mode == kResidual || g.mode == kScalePe) {
          const float* src = g.mode == kResidual
                                 ? g.out_f32 + (size_t)row * g.ldo + col0
                                 : g.pe + (size_t)(row % g.pe_rows) * g.N + col0;
          const float sc = g.mode == kResidual ? 1.f : g.scale;
          if (row_ok && full_cols && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 32 columns (fp32 output)
              const float4 o = *reinterpret_cast<const float4*>(src + 4 * j);
              x[4 * j] = x[4 * j] * sc + o.x; x[4 * j + 1] = x[4 * j + 1] * sc + o.y;
              x[4 * j + 2] = x[4 * j + 2] * sc + o.z; x[4 * j + 3] = x[4 * j + 3] * sc + o.w;
            }
          } else if (row_ok) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j < g.N) x[j] = x[j] * sc + src[j];
          }
        }
        unsigned char* sb = stg + (nchunk & 1) * kStgBytes;
        if (lane == 0) bulk_wait_read<1>();  // the store that last used sb has read it
        __syncwarp();
        if (bf) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            uint4 u;
            u.x = pack_bf16(x[8 * c], x[8 * c + 1]);
            u.y = pack_bf16(x[8 * c + 2], x[8 * c + 3]);
            u.z = pack_bf16(x[8 * c + 4], x[8 * c + 5]);
            u.w = pack_bf16(x[8 * c + 6], x[8 * c + 7]);
            *reinterpret_cast<uint4*>(sb + sw128(lane, c)) = u;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(sb + sw128(lane, c)) =
                make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store2d(tO, sb, col0, rbase);
          bulk_commit();
        }
        (void)kCW32;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mb_arrive(&acc_empty[a]);
    }
    if (lane == 0) bulk_wait<0>();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::kTmemCols));
}

// K-major bf16 operand [rows, K] (row stride ld elements), box 64 x box_rows, SW128
bool make_map(CUtensorMap* m, const void* base, int rows, int K, int ld, int box_rows) {
  return make_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, K, rows, (size_t)ld * 2, kBK,
                   box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
  }
  return n;
}

template <int BN>
cudaError_t launch(const GemmDesc& d, cudaStream_t st) {
  CUtensorMap tA, tB, tOb, tOf;
  if (!make_map(&tA, d.A, d.M, d.K, d.lda, kBM) || !make_map(&tB, d.B, d.N, d.K, d.ldb, BN))
    return cudaErrorInvalidValue;
  std::memset(&tOb, 0, sizeof(tOb));
  std::memset(&tOf, 0, sizeof(tOf));
  if (d.out_bf16 && !make_tmap(&tOb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, d.out_bf16, d.N, d.M,
                               (size_t)d.ldo * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (!d.out_bf16 && !make_tmap(&tOf, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, d.out_f32, d.N, d.M,
                                (size_t)d.ldo * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  GemmArgs g{d.M, d.N, d.K, d.mode, d.bias, d.out_f32, d.out_bf16, d.ldo, d.scale, d.pe,
             d.pe_rows};
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<BN>::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = ((d.M + kBM - 1) / kBM) * ((d.N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  gemm_kernel<BN><<<grid, kThreads, Cfg<BN>::kSmem, st>>>(tA, tB, tOb, tOf, g);
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t st) {
  if (d.K % 8 != 0 || d.lda % 8 != 0 || d.ldb % 8 != 0) return cudaErrorInvalidValue;
  // exactly one output; bulk tensor stores need 16-byte row strides
  if ((d.out_bf16 != nullptr) == (d.out_f32 != nullptr)) return cudaErrorInvalidValue;
  if (d.out_bf16 ? (d.ldo % 8) : (d.ldo % 4)) return cudaErrorInvalidValue;
  if ((d.mode == kResidual || d.mode == kScalePe) && !d.out_f32) return cudaErrorInvalidValue;
  // 256-wide tiles halve A re-reads; 128-wide when N is small or the
  // 256-wide grid would leave most SMs idle.
  const long long t256 = (long long)((d.M + kBM - 1) / kBM) * ((d.N + 255) / 256);
  if (d.N > 128 && t256 >= num_sms()) return launch<256>(d, st);
  return launch<128>(d, st);
}

}  // namespace bl
