// gemm_tcgen05.cu — bf16 GEMM on the sm_100a 5th-generation tensor cores for
// the encoder (SURVEY §8 a'1): C[M,N] = A[M,K] · B[N,K]^T, fp32 accumulation
// in tensor memory, fused epilogue (bias, ReLU, residual, scale + positional
// table), bf16 and/or fp32 output. The residual epilogue (x += acc + bias)
// never reads x: each chunk goes out as a TMA reduce-add (fp32 add in L2).
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
  double* lse_part;  // kLsePart
  int lse_stride;
  // implicit conv2 (kConv): A tiles are 4D TMA boxes over the channel-last
  // conv1 output; a tile covers `tpt` output frames x F2 bins = `rows` rows
  int S, T2, F2, tpt, tps, ktin, rows;
};

template <int BN, bool kConv>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                const __grid_constant__ CUtensorMap tOb, const __grid_constant__ CUtensorMap tOf,
                const __grid_constant__ CUtensorMap tOr, const GemmArgs g) {
  using C = Cfg<BN>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* epi = smem + S * C::kStage;
  __shared__ __align__(8) uint64_t full[S], empty[S], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KT = kConv ? 3 * g.ktin : (g.K + kBK - 1) / kBK;
  const int tiles_n = (g.N + BN - 1) / BN;
  const int tiles = (kConv ? g.S * g.tps : (g.M + kBM - 1) / kBM) * tiles_n;

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
          mb_expect_tx(&full[s], kConv ? g.rows * 128 + C::kB : C::kStage);
          if (kConv) {
            const int mt = tile / tiles_n, seg = mt / g.tps, t20 = (mt % g.tps) * g.tpt;
            const int kh = kt / g.ktin, kin = kt - kh * g.ktin;
            // rows (f2, t2): conv1 rows 2*t2 + kh, columns 2*f2 .. 2*f2+2 (3d contiguous)
            tma4d(st, &tA, kin * kBK, 0, 2 * t20 + kh, seg, &full[s]);
          } else {
            tma2d(st, &tA, kt * kBK, m0, &full[s]);
          }
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
      float lm = -INFINITY;  // kLsePart: this row's running max over the tile
      double ls = 0.0;       //           and sum of exp(x - lm)
      int qrows = 32, cy = 0, cz = 0;
      if (kConv) {
        const int mt = tile / tiles_n;
        qrows = min(32, g.rows - q * 32);
        cz = mt / g.tps;
        cy = (mt % g.tps) * g.tpt * g.F2 + q * 32;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += CW, ++nchunk) {
        if (n0 + c0 >= g.N || qrows <= 0) break;
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
        } else if (g.mode == kScalePe) {
          // (kResidual needs no read: the chunk is added to the residual
          // stream in global memory by a TMA reduce-add below)
          const float* src = g.pe + (size_t)(row % g.pe_rows) * g.N + col0;
          const float sc = g.scale;
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
        if (g.mode == kLsePart) {  // fused log-softmax: partial max and sum of exp
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < g.N) cm = fmaxf(cm, x[j]);
          if (cm > lm) {
            ls *= exp((double)lm - (double)cm);
            lm = cm;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < g.N) ls += (double)expf(x[j] - lm);
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
          if (kConv)
            tma_store3d(qrows == 32 ? &tOb : &tOr, sb, col0, cy, cz);
          else if (g.mode == kResidual)
            tma_reduce_add2d(tO, sb, col0, rbase);
          else
            tma_store2d(tO, sb, col0, rbase);
          bulk_commit();
        }
        (void)kCW32;
      }
      if (g.mode == kLsePart && row_ok && ls > 0.0) {
        double* pp = g.lse_part + ((size_t)row * g.lse_stride + n0 / 128) * 2;
        pp[0] = (double)lm;
        pp[1] = ls;
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

// 3D bf16 output [z][rows][cols], box 64 cols x box_rows x 1, SW128
bool make_tmap3(CUtensorMap* m, const void* base, int cols, int rows, int z, size_t ld_bytes,
                int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)z};
  const cuuint64_t strides[2] = {(cuuint64_t)ld_bytes, (cuuint64_t)ld_bytes * rows};
  const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
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

template <int BN, bool kConv>
cudaError_t launch(const GemmDesc& d, const CUtensorMap& tA, const GemmArgs& g, int tiles,
                   cudaStream_t st) {
  CUtensorMap tB, tOb, tOf, tOr;
  std::memset(&tOb, 0, sizeof(tOb));
  std::memset(&tOf, 0, sizeof(tOf));
  std::memset(&tOr, 0, sizeof(tOr));
  if (!make_map(&tB, d.B, d.N, d.K, d.ldb, BN)) return cudaErrorInvalidValue;
  if (kConv) {
    // 3D output [S][T2*F2][N]: stores clip at each segment's last frame
    if (!make_tmap3(&tOb, d.out_bf16, d.N, g.T2 * g.F2, g.S, (size_t)d.ldo * 2, 32) ||
        (g.rows % 32 && !make_tmap3(&tOr, d.out_bf16, d.N, g.T2 * g.F2, g.S,
                                    (size_t)d.ldo * 2, g.rows % 32)))
      return cudaErrorInvalidValue;
  } else if (d.out_bf16) {
    if (!make_tmap(&tOb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, d.out_bf16, d.N, d.M,
                   (size_t)d.ldo * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  } else if (!make_tmap(&tOf, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, d.out_f32, d.N, d.M,
                        (size_t)d.ldo * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)) {
    return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, kConv>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<BN>::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = tiles < num_sms() ? tiles : num_sms();
  gemm_kernel<BN, kConv><<<grid, kThreads, Cfg<BN>::kSmem, st>>>(tA, tB, tOb, tOf, tOr, g);
  return cudaGetLastError();
}

GemmArgs args_of(const GemmDesc& d) {
  GemmArgs g{};
  g.M = d.M; g.N = d.N; g.K = d.K; g.mode = d.mode; g.bias = d.bias; g.out_f32 = d.out_f32;
  g.out_bf16 = d.out_bf16; g.ldo = d.ldo; g.scale = d.scale; g.pe = d.pe; g.pe_rows = d.pe_rows;
  g.lse_part = d.lse_part; g.lse_stride = d.lse_stride;
  return g;
}

}  // namespace

cudaError_t gemm_bf16(const GemmDesc& d, cudaStream_t st) {
  if (d.K % 8 != 0 || d.lda % 8 != 0 || d.ldb % 8 != 0) return cudaErrorInvalidValue;
  // exactly one output; bulk tensor stores need 16-byte row strides
  if ((d.out_bf16 != nullptr) == (d.out_f32 != nullptr)) return cudaErrorInvalidValue;
  if (d.out_bf16 ? (d.ldo % 8) : (d.ldo % 4)) return cudaErrorInvalidValue;
  if ((d.mode == kResidual || d.mode == kScalePe) && !d.out_f32) return cudaErrorInvalidValue;
  if (d.mode == kLsePart && (!d.out_f32 || !d.lse_part || d.lse_stride < (d.N + 127) / 128))
    return cudaErrorInvalidValue;
  CUtensorMap tA;
  if (!make_map(&tA, d.A, d.M, d.K, d.lda, kBM)) return cudaErrorInvalidValue;
  const GemmArgs g = args_of(d);
  // 256-wide tiles halve A re-reads; 128-wide when N is small or the
  // 256-wide grid would leave most SMs idle.
  const int tm = (d.M + kBM - 1) / kBM;
  const long long t256 = (long long)tm * ((d.N + 255) / 256);
  if (d.N > 128 && t256 >= num_sms()) return launch<256, false>(d, tA, g, (int)t256, st);
  return launch<128, false>(d, tA, g, tm * ((d.N + 127) / 128), st);
}

cudaError_t conv2_bf16(const Conv2Desc& c, cudaStream_t st) {
  const int d = c.d;
  if (d % 64 || c.F2 < 1 || c.F2 > kBM || c.T2 < 1 || c.S < 1) return cudaErrorInvalidValue;
  // A: conv1 output [S][T1][F1][d] viewed as 4D {3d (kw,c), F2 (stride 2d),
  // T1 (stride F1*d, traversed with element stride 2), S}
  CUtensorMap tA;
  {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorInvalidValue;
    const int tpt = kBM / c.F2;
    const cuuint64_t dims[4] = {(cuuint64_t)3 * d, (cuuint64_t)c.F2, (cuuint64_t)c.T1,
                                (cuuint64_t)c.S};
    const cuuint64_t strides[3] = {(cuuint64_t)2 * d * 2, (cuuint64_t)c.F1 * d * 2,
                                   (cuuint64_t)c.T1 * c.F1 * d * 2};
    const cuuint32_t box[4] = {(cuuint32_t)kBK, (cuuint32_t)c.F2, (cuuint32_t)(2 * tpt), 1};
    const cuuint32_t es[4] = {1, 1, 2, 1};
    if (enc(&tA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<__nv_bfloat16*>(c.c1), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  GemmDesc gd;
  gd.M = c.S * c.T2 * c.F2; gd.N = d; gd.K = 9 * d;
  gd.B = c.W; gd.ldb = 9 * d; gd.mode = kRelu; gd.bias = c.bias;
  gd.out_bf16 = c.out; gd.ldo = d;
  GemmArgs g = args_of(gd);
  g.S = c.S; g.T2 = c.T2; g.F2 = c.F2; g.tpt = kBM / c.F2;
  g.tps = (c.T2 + g.tpt - 1) / g.tpt; g.ktin = 3 * d / kBK; g.rows = g.tpt * c.F2;
  const int tiles = c.S * g.tps * ((d + 255) / 256);
  return launch<256, true>(gd, tA, g, tiles, st);
}

}  // namespace bl
