// encoder.cu — the CTC encoder forward (SURVEY §8 a'1) that produces the
// PosteriorGrid the decoder consumes, written straight into device memory.
//
// Model (ESPnet Transformer encoder, pre-LN, eval mode):
//   Conv2dSubsampling: conv1(1->d,3x3/2)+ReLU, conv2(d->d,3x3/2)+ReLU,
//   linear(d*F2 -> d), x*sqrt(d) + PE;  L x [LN, MHA, +res, LN, FFN(ReLU), +res];
//   final LN; CTC linear(d -> V); log_softmax.
//
// Device layout (per chunk of S segments, all equal length T_in frames):
//   c1  bf16 [S][T1][F1][d]       channel-last conv1 output
//   (conv2 is an implicit GEMM: 4D TMA boxes over c1, k = (kh*3+kw)*d + c)
//   c2  bf16 [S*T2][F2*d]         channel-last conv2 output == linear input
//   X   f32  [S*T2][d]            residual stream
//   Y   bf16 [S*T2][d]            LayerNorm output (GEMM A operand)
//   QKV bf16 [S*T2][3d], AO bf16 [S*T2][d], H bf16 [S*T2][dff]
//   grid f32 [S*T2][V]            caller's buffer, log-probabilities
// All dense products go through gemm_bf16 (tcgen05, gemm_tcgen05.cu).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "encoder.cuh"
#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace bl {


namespace {

constexpr int kDk = 64;  // head width (d / heads)

// ---------------------------------------------------------------- kernels
// conv1 (1 -> d, 3x3, stride 2) + ReLU; fp32 math, bf16 channel-last output.
// One CTA per (segment, run of kC1Frames output frames): the input frames are
// staged in shared memory; each thread owns a fixed group of 8 consecutive
// channels (72 taps in registers, loaded once) and sweeps a strided subset of
// the (frame, bin) outputs, writing one 16-byte vector per output (a warp
// covers 512 contiguous bytes).
constexpr int kC1Frames = 16;

__global__ void __launch_bounds__(256) conv1_kernel(const float* __restrict__ fb, int T_in,
                                                    int idim, int T1, int F1, int d,
                                                    const float* __restrict__ w,
                                                    const float* __restrict__ b,
                                                    __nv_bfloat16* __restrict__ out) {
  extern __shared__ float rows[];  // [2 * kC1Frames + 1][idim]
  const int t0 = blockIdx.x * kC1Frames, n = blockIdx.y;
  const int nt = min(kC1Frames, T1 - t0);
  const int nrows = 2 * nt + 1;
  const float* x = fb + ((size_t)n * T_in + 2 * t0) * idim;
  for (int i = threadIdx.x; i < nrows * idim; i += blockDim.x) rows[i] = x[i];
  __syncthreads();
  // d <= 1024 (enc_validate): groups <= 128, so every group has >= 2 threads
  const int groups = d / 8, per = blockDim.x / groups;
  const int cg = threadIdx.x % groups, j0 = threadIdx.x / groups;
  if (j0 >= per) return;
  float wr[8][9], br[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
#pragma unroll
    for (int k = 0; k < 9; ++k) wr[j][k] = __ldg(w + (cg * 8 + j) * 9 + k);
    br[j] = __ldg(b + cg * 8 + j);
  }
  uint4* o = reinterpret_cast<uint4*>(out + ((size_t)n * T1 + t0) * F1 * d);
  for (int i = j0; i < nt * F1; i += per) {
    const int tt = i / F1, f = i - tt * F1;
    const float* xr = rows + 2 * tt * idim + 2 * f;
    float in[9];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) in[kh * 3 + kw] = xr[kh * idim + kw];
    uint32_t packed[4];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        a0 = fmaf(wr[j][k], in[k], a0);
        a1 = fmaf(wr[j + 1][k], in[k], a1);
      }
      const __nv_bfloat162 h =
          __floats2bfloat162_rn(fmaxf(a0 + br[j], 0.f), fmaxf(a1 + br[j + 1], 0.f));
      packed[j / 2] = *reinterpret_cast<const uint32_t*>(&h);
    }
    o[(size_t)i * groups + cg] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

// LayerNorm over d (biased variance, eps 1e-12), one warp per row, VPL = d/32.
template <int VPL>
__global__ void layernorm_scalar_kernel(const float* __restrict__ X, int rows, const float* __restrict__ g,
                                 const float* __restrict__ b, __nv_bfloat16* __restrict__ Y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  constexpr int d = VPL * 32;
  const float* x = X + (size_t)warp * d;
  float v[VPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    v[i] = x[i * 32 + lane];
    s += v[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    v[i] -= mean;
    q = fmaf(v[i], v[i], q);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rs = rsqrtf(q / d + 1e-12f);
  __nv_bfloat16* y = Y + (size_t)warp * d;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int k = i * 32 + lane;
    y[k] = __float2bfloat16_rn(v[i] * rs * g[k] + b[k]);
  }
}

// LayerNorm over d (biased variance, eps 1e-12), one warp per row, VPL = d/32:
// lane i owns the 4-float groups i, i+32, ... (16-byte loads, 8-byte bf16
// stores, gamma/beta as float4).
template <int VPL>
__global__ void layernorm_kernel(const float* __restrict__ X, int rows, const float* __restrict__ g,
                                 const float* __restrict__ b, __nv_bfloat16* __restrict__ Y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  constexpr int d = VPL * 32, G = VPL / 4;  // float4 groups per lane (VPL % 4 == 0)
  const float4* x = reinterpret_cast<const float4*>(X + (size_t)warp * d);
  float4 v[G];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    v[i] = x[i * 32 + lane];
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < G; ++i) {
    v[i].x -= mean; v[i].y -= mean; v[i].z -= mean; v[i].w -= mean;
    q = fmaf(v[i].x, v[i].x, q);
    q = fmaf(v[i].y, v[i].y, q);
    q = fmaf(v[i].z, v[i].z, q);
    q = fmaf(v[i].w, v[i].w, q);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rs = rsqrtf(q / d + 1e-12f);
  uint2* y = reinterpret_cast<uint2*>(Y + (size_t)warp * d);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int i = 0; i < G; ++i) {
    const int k = i * 32 + lane;
    const float4 gg = __ldg(g4 + k), bb = __ldg(b4 + k);
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * rs * gg.x + bb.x,
                                                     v[i].y * rs * gg.y + bb.y);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * rs * gg.z + bb.z,
                                                     v[i].w * rs * gg.w + bb.w);
    uint2 o;
    o.x = *reinterpret_cast<const uint32_t*>(&lo);
    o.y = *reinterpret_cast<const uint32_t*>(&hi);
    y[k] = o;
  }
}

// Multi-head self-attention, no mask (equal-length segments), head width 64.
// One CTA per (segment, head): K and V staged in shared memory as bf16 with a
// 66-element row pitch (conflict-free 4-byte reads); one warp per query row.
constexpr int kAttnWarps = 8;
constexpr int kKvPitch = kDk + 2;

__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_kernel(const __nv_bfloat16* __restrict__ qkv, int T, int d, int heads,
                     __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* Vs = Ks + (size_t)T * kKvPitch;
  float* qs = reinterpret_cast<float*>(Vs + (size_t)T * kKvPitch);  // [warps][64]
  float* ps = qs + kAttnWarps * kDk;                                // [warps][T]
  const int seg = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t ld = 3 * (size_t)d;
  const __nv_bfloat16* base = qkv + (size_t)seg * T * ld;
  for (int i = threadIdx.x; i < T * (kDk / 2); i += blockDim.x) {
    const int t = i / (kDk / 2), k2 = i % (kDk / 2);
    const __nv_bfloat162* row = reinterpret_cast<const __nv_bfloat162*>(base + t * ld);
    reinterpret_cast<__nv_bfloat162*>(Ks + t * kKvPitch)[k2] = row[(d + h * kDk) / 2 + k2];
    reinterpret_cast<__nv_bfloat162*>(Vs + t * kKvPitch)[k2] = row[(2 * d + h * kDk) / 2 + k2];
  }
  __syncthreads();
  const float scale = rsqrtf((float)kDk);
  float* q = qs + warp * kDk;
  float* p = ps + (size_t)warp * T;
  for (int tq = warp; tq < T; tq += kAttnWarps) {
    const __nv_bfloat162 qv =
        reinterpret_cast<const __nv_bfloat162*>(base + tq * ld + h * kDk)[lane];
    q[2 * lane] = __bfloat162float(qv.x);
    q[2 * lane + 1] = __bfloat162float(qv.y);
    __syncwarp();
    float m = -INFINITY;
    for (int j = lane; j < T; j += 32) {
      const __nv_bfloat162* kr = reinterpret_cast<const __nv_bfloat162*>(Ks + j * kKvPitch);
      float s = 0.f;
#pragma unroll 8
      for (int k2 = 0; k2 < kDk / 2; ++k2) {
        const float2 kf = __bfloat1622float2(kr[k2]);
        s = fmaf(q[2 * k2], kf.x, s);
        s = fmaf(q[2 * k2 + 1], kf.y, s);
      }
      s *= scale;
      p[j] = s;
      m = fmaxf(m, s);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float sum = 0.f;
    for (int j = lane; j < T; j += 32) {
      const float e = expf(p[j] - m);
      p[j] = e;
      sum += e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncwarp();
    float a0 = 0.f, a1 = 0.f;
    for (int j = 0; j < T; ++j) {
      const float pj = p[j];
      const float2 vf =
          __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(Vs + j * kKvPitch)[lane]);
      a0 = fmaf(pj, vf.x, a0);
      a1 = fmaf(pj, vf.y, a1);
    }
    const float inv = 1.f / sum;
    reinterpret_cast<__nv_bfloat162*>(out + ((size_t)seg * T + tq) * d + h * kDk)[lane] =
        __floats2bfloat162_rn(a0 * inv, a1 * inv);
    __syncwarp();
  }
}

// Self-attention on the tensor cores for segments of T <= 256 frames.
// One CTA (128 threads) per (segment, head, 128-query tile):
//   TMA: Q [128 x 64], K [256 x 64], V [256 x 64] bf16 tiles (SWIZZLE_128B)
//   S = Q K^T   tcgen05.mma M=128 N=256 K=64 -> TMEM columns [0, 256)
//   softmax     thread r owns query row r: two tcgen05.ld sweeps (max, then
//               exp/sum), P = exp(...) as bf16 into a SWIZZLE_128B K-major
//               tile in shared memory (aliasing the consumed Q/K tiles)
//   O = P V     tcgen05.mma M=128 N=64 K=256, V as the MN-major operand,
//               -> TMEM columns [0, 64); O / rowsum -> bf16 rows
// Keys >= T (the next segment's rows, or zero fill past the end) are masked.
constexpr int kAttQ = 128, kAttK = 256;
constexpr int kAttSmem = 16384 /*Q*/ + 32768 /*K*/ + 16384 /*P tail*/ + 32768 /*V*/ + 1024;
constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kAttK >> 3) << 17) |
                             ((uint32_t)(kAttQ >> 4) << 24);
constexpr uint32_t kIdescO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) /*B MN-major*/ |
                             ((uint32_t)(kDk >> 3) << 17) | ((uint32_t)(kAttQ >> 4) << 24);

__global__ void __launch_bounds__(128)
    attention_tc_kernel(const __grid_constant__ CUtensorMap tQ,
                        const __grid_constant__ CUtensorMap tKV, int T, int d,
                        __nv_bfloat16* __restrict__ out) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char araw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(araw) + 1023) & ~(uintptr_t)1023);
  unsigned char* Qs = sm;
  unsigned char* Ks = sm + 16384;
  unsigned char* Ps = sm;           // 4 x [128 x 64] bf16 blocks = 64 KB (after S)
  unsigned char* Vs = sm + 65536;
  __shared__ __align__(8) uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tbase;
  const int n = blockIdx.x, h = blockIdx.y, qt = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row0 = n * T;
  if (tid == 0) {
    mb_init(&bar_ld, 1);
    mb_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mb_expect_tx(&bar_ld, 16384 + 2 * 32768);
    tma2d(Qs, &tQ, h * kDk, row0 + qt * kAttQ, &bar_ld);
    tma2d(Ks, &tKV, d + h * kDk, row0, &bar_ld);
    tma2d(Vs, &tKV, 2 * d + h * kDk, row0, &bar_ld);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s32(&tbase)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    mb_wait(&bar_ld, 0);
    tc_fence_after();
    const uint64_t dq = umma_desc(Qs), dk = umma_desc(Ks);
#pragma unroll
    for (int k = 0; k < kDk / 16; ++k) umma(tmem, dq + 2ull * k, dk + 2ull * k, kIdescS, k > 0);
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mb_wait(&bar_mma, 0);
  tc_fence_after();
  const int r = warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const float c2 = 1.4426950408889634f * rsqrtf((float)kDk);  // log2(e) / sqrt(dk)
  float m = -INFINITY;
#pragma unroll 1
  for (int c0 = 0; c0 < kAttK; c0 += 32) {
    if (c0 >= T) break;
    uint32_t v[32];
    tmem_ld32(trow + c0, v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (c0 + j < T) m = fmaxf(m, __uint_as_float(v[j]));
  }
  float sum = 0.f;
#pragma unroll 1
  for (int c0 = 0; c0 < kAttK; c0 += 32) {
    uint32_t v[32];
    if (c0 < T) tmem_ld32(trow + c0, v);
    float p[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float e = (c0 + j < T) ? exp2f((__uint_as_float(v[j]) - m) * c2) : 0.f;
      const float eb = __bfloat162float(__float2bfloat16_rn(e));
      p[j] = e;
      sum += eb;
    }
    // P block b = c0 / 64, 16-byte chunks (c0 % 64) / 8 .. +3 of row r
    unsigned char* blk = Ps + (c0 >> 6) * 16384;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint4 u;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(p[8 * c], p[8 * c + 1]);
      __nv_bfloat162 h1 = __floats2bfloat162_rn(p[8 * c + 2], p[8 * c + 3]);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(p[8 * c + 4], p[8 * c + 5]);
      __nv_bfloat162 h3 = __floats2bfloat162_rn(p[8 * c + 6], p[8 * c + 7]);
      u.x = *reinterpret_cast<uint32_t*>(&h0);
      u.y = *reinterpret_cast<uint32_t*>(&h1);
      u.z = *reinterpret_cast<uint32_t*>(&h2);
      u.w = *reinterpret_cast<uint32_t*>(&h3);
      *reinterpret_cast<uint4*>(blk + sw128(r, ((c0 & 63) >> 3) + c)) = u;
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    const uint64_t dv = umma_desc(Vs);
#pragma unroll
    for (int kk = 0; kk < kAttK / 16; ++kk) {
      const uint64_t dp = umma_desc(Ps + (kk >> 2) * 16384) + 2ull * (kk & 3);
      umma(tmem, dp, dv + 128ull * kk /* 16 keys = 2048 B */, kIdescO, kk > 0);
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mb_wait(&bar_mma, 1);
  tc_fence_after();
  const float inv = 1.f / sum;
  const int q = qt * kAttQ + r;
  uint32_t o[64];
  {
    uint32_t v[32];
    tmem_ld32(trow, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = v[j];
    tmem_ld32(trow + 32, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) o[32 + j] = v[j];
  }
  if (q < T) {
    uint4* dst = reinterpret_cast<uint4*>(out + ((size_t)row0 + q) * d + h * kDk);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint4 u;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(o[8 * c]) * inv,
                                                __uint_as_float(o[8 * c + 1]) * inv);
      __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2]) * inv,
                                                __uint_as_float(o[8 * c + 3]) * inv);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 4]) * inv,
                                                __uint_as_float(o[8 * c + 5]) * inv);
      __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 6]) * inv,
                                                __uint_as_float(o[8 * c + 7]) * inv);
      u.x = *reinterpret_cast<uint32_t*>(&h0);
      u.y = *reinterpret_cast<uint32_t*>(&h1);
      u.z = *reinterpret_cast<uint32_t*>(&h2);
      u.w = *reinterpret_cast<uint32_t*>(&h3);
      dst[c] = u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// The same for 256 < T <= 512 (20 s segments: T = 499): K and V are two
// 256-row TMA boxes each; S = Q K^T is two M=128 N=256 MMAs into TMEM columns
// [0, 512) (tcgen05 kernels run one CTA per SM, so the whole TMEM is free);
// the softmax takes its max over all 512 columns, then P goes through shared
// memory one 256-key half at a time (64 KB, aliasing the consumed Q/K tiles):
// O = P0 V0, then O += P1 V1 once the first product has read P0. O lives in
// TMEM columns [0, 64), which only the first half of S occupied.
constexpr int kAtt2K = 512;
constexpr int kAtt2Smem = 16384 /*Q*/ + 65536 /*K*/ + 65536 /*V*/ + 1024;

__global__ void __launch_bounds__(128)
    attention_tc512_kernel(const __grid_constant__ CUtensorMap tQ,
                           const __grid_constant__ CUtensorMap tKV, int T, int d,
                           __nv_bfloat16* __restrict__ out) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char araw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(araw) + 1023) & ~(uintptr_t)1023);
  unsigned char* Qs = sm;
  unsigned char* Ks = sm + 16384;          // 2 x [256 x 64] bf16
  unsigned char* Ps = sm;                  // 4 x [128 x 64] bf16 = one half of P
  unsigned char* Vs = sm + 16384 + 65536;  // 2 x [256 x 64] bf16
  __shared__ __align__(8) uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tbase;
  const int n = blockIdx.x, h = blockIdx.y, qt = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row0 = n * T;
  if (tid == 0) {
    mb_init(&bar_ld, 1);
    mb_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mb_expect_tx(&bar_ld, 16384 + 4 * 32768);
    tma2d(Qs, &tQ, h * kDk, row0 + qt * kAttQ, &bar_ld);
    tma2d(Ks, &tKV, d + h * kDk, row0, &bar_ld);
    tma2d(Ks + 32768, &tKV, d + h * kDk, row0 + 256, &bar_ld);
    tma2d(Vs, &tKV, 2 * d + h * kDk, row0, &bar_ld);
    tma2d(Vs + 32768, &tKV, 2 * d + h * kDk, row0 + 256, &bar_ld);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     s32(&tbase)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    mb_wait(&bar_ld, 0);
    tc_fence_after();
    const uint64_t dq = umma_desc(Qs);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const uint64_t dk = umma_desc(Ks + hh * 32768);
#pragma unroll
      for (int k = 0; k < kDk / 16; ++k)
        umma(tmem + 256 * hh, dq + 2ull * k, dk + 2ull * k, kIdescS, k > 0);
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mb_wait(&bar_mma, 0);
  tc_fence_after();
  const int r = warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const float c2 = 1.4426950408889634f * rsqrtf((float)kDk);  // log2(e) / sqrt(dk)
  float m = -INFINITY;
#pragma unroll 1
  for (int c0 = 0; c0 < kAtt2K; c0 += 32) {
    if (c0 >= T) break;
    uint32_t v[32];
    tmem_ld32(trow + c0, v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (c0 + j < T) m = fmaxf(m, __uint_as_float(v[j]));
  }
  float sum = 0.f;
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    if (hh == 1) {  // P0 V0 has read the P buffer
      __syncwarp();
      mb_wait(&bar_mma, 1);
      tc_fence_after();
    }
#pragma unroll 1
    for (int c1 = 0; c1 < 256; c1 += 32) {
      const int c0 = hh * 256 + c1;
      uint32_t v[32];
      if (c0 < T) tmem_ld32(trow + c0, v);
      float p[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = (c0 + j < T) ? exp2f((__uint_as_float(v[j]) - m) * c2) : 0.f;
        sum += __bfloat162float(__float2bfloat16_rn(e));
        p[j] = e;
      }
      unsigned char* blk = Ps + (c1 >> 6) * 16384;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 u;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(p[8 * c], p[8 * c + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(p[8 * c + 2], p[8 * c + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(p[8 * c + 4], p[8 * c + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(p[8 * c + 6], p[8 * c + 7]);
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(blk + sw128(r, ((c1 & 63) >> 3) + c)) = u;
      }
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint64_t dv = umma_desc(Vs + hh * 32768);
#pragma unroll
      for (int kk = 0; kk < 256 / 16; ++kk) {
        const uint64_t dp = umma_desc(Ps + (kk >> 2) * 16384) + 2ull * (kk & 3);
        umma(tmem, dp, dv + 128ull * kk /* 16 keys = 2048 B */, kIdescO, (hh > 0 || kk > 0));
      }
      umma_commit(&bar_mma);
    }
  }
  __syncwarp();
  mb_wait(&bar_mma, 0);  // third completion (S, P0 V0, P1 V1)
  tc_fence_after();
  const float inv = 1.f / sum;
  const int q = qt * kAttQ + r;
  uint32_t o[64];
  {
    uint32_t v[32];
    tmem_ld32(trow, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = v[j];
    tmem_ld32(trow + 32, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) o[32 + j] = v[j];
  }
  if (q < T) {
    uint4* dst = reinterpret_cast<uint4*>(out + ((size_t)row0 + q) * d + h * kDk);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint4 u;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(o[8 * c]) * inv,
                                                __uint_as_float(o[8 * c + 1]) * inv);
      __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2]) * inv,
                                                __uint_as_float(o[8 * c + 3]) * inv);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 4]) * inv,
                                                __uint_as_float(o[8 * c + 5]) * inv);
      __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 6]) * inv,
                                                __uint_as_float(o[8 * c + 7]) * inv);
      u.x = *reinterpret_cast<uint32_t*>(&h0);
      u.y = *reinterpret_cast<uint32_t*>(&h1);
      u.z = *reinterpret_cast<uint32_t*>(&h2);
      u.w = *reinterpret_cast<uint32_t*>(&h3);
      dst[c] = u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// in-place log_softmax over rows of width V; one CTA per row
__global__ void __launch_bounds__(256) log_softmax_kernel(float* __restrict__ x, int V) {
  __shared__ float red[8];
  float* r = x + (size_t)blockIdx.x * V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float m = -INFINITY;
  for (int i = threadIdx.x; i < V; i += blockDim.x) m = fmaxf(m, r[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float s = 0.f;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += expf(r[i] - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < 8; ++w) s += red[w];
  const float lse = m + logf(s);
  for (int i = threadIdx.x; i < V; i += blockDim.x) r[i] -= lse;
}

template <int VPL>
void ln_launch(const float* X, int rows, const float* g, const float* b, __nv_bfloat16* Y,
               cudaStream_t st) {
  if constexpr (VPL % 4 == 0)
    layernorm_kernel<VPL><<<(rows + 7) / 8, 256, 0, st>>>(X, rows, g, b, Y);
  else
    layernorm_scalar_kernel<VPL><<<(rows + 7) / 8, 256, 0, st>>>(X, rows, g, b, Y);
}

void launch_layernorm(int d, const float* X, int rows, const float* g, const float* b,
                      __nv_bfloat16* Y, cudaStream_t st) {
  switch (d / 64) {
    case 1: ln_launch<2>(X, rows, g, b, Y, st); break;
    case 2: ln_launch<4>(X, rows, g, b, Y, st); break;
    case 3: ln_launch<6>(X, rows, g, b, Y, st); break;
    case 4: ln_launch<8>(X, rows, g, b, Y, st); break;
    case 5: ln_launch<10>(X, rows, g, b, Y, st); break;
    case 6: ln_launch<12>(X, rows, g, b, Y, st); break;
    case 7: ln_launch<14>(X, rows, g, b, Y, st); break;
    case 8: ln_launch<16>(X, rows, g, b, Y, st); break;
    case 9: ln_launch<18>(X, rows, g, b, Y, st); break;
    case 10: ln_launch<20>(X, rows, g, b, Y, st); break;
    case 11: ln_launch<22>(X, rows, g, b, Y, st); break;
    case 12: ln_launch<24>(X, rows, g, b, Y, st); break;
    case 13: ln_launch<26>(X, rows, g, b, Y, st); break;
    case 14: ln_launch<28>(X, rows, g, b, Y, st); break;
    case 15: ln_launch<30>(X, rows, g, b, Y, st); break;
    default: ln_launch<32>(X, rows, g, b, Y, st); break;
  }
}

int blocks_for(long long total, int nt = 256) {
  long long b = (total + nt - 1) / nt;
  return (int)(b > 148LL * 16 ? 148LL * 16 : (b < 1 ? 1 : b));
}

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
  return (uint16_t)(u >> 16);
}

}  // namespace

int enc_frames_out(int frames_in) {
  if (frames_in < 7) return 0;
  const int t1 = (frames_in - 3) / 2 + 1;
  return (t1 - 3) / 2 + 1;
}

size_t enc_num_weights(const EncSpec& s) {
  const size_t d = s.d, F2 = (size_t)enc_frames_out(s.idim);
  size_t n = d * 9 + d + d * d * 9 + d + d * F2 * d + d;
  n += (size_t)s.layers * (2 * d + 4 * (d * d + d) + 2 * d + (s.dff * d + s.dff) + (d * s.dff + d));
  n += 2 * d + (size_t)s.vocab * d + s.vocab;
  return n;
}

std::string enc_validate(const EncSpec& s) {
  if (s.idim < 7) return "encoder idim must be >= 7";
  if (s.d < 64 || s.d > 1024 || s.d % 64) return "encoder d_model must be a multiple of 64 in [64, 1024]";
  if (s.heads < 1 || s.d != s.heads * kDk) return "encoder heads must give a head width of 64";
  if (s.dff < 8 || s.dff % 8) return "encoder d_ff must be a positive multiple of 8";
  if (s.layers < 0) return "encoder layers must be >= 0";
  if (s.vocab < 2 || s.vocab % 4) return "encoder vocab must be >= 2 and a multiple of 4";
  return "";
}

struct EncLayer {
  float *ln1g, *ln1b, *bqkv, *bo, *ln2g, *ln2b, *b1, *b2;
  __nv_bfloat16 *wqkv, *wo, *w1, *w2;
};

struct EncoderImpl {
  EncSpec s;
  int F1, F2;
  cudaStream_t st = nullptr;
  void* wbuf = nullptr;
  float *c1w, *c1b, *c2b, *ob, *ang, *anb, *cb, *pe = nullptr;
  __nv_bfloat16 *c2w, *ow, *cw;
  std::vector<EncLayer> L;
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int pe_rows = 0;
  int launches = 0;
  // host fbank: chunk i+1 is copied on `cp` while chunk i computes on `st`
  cudaStream_t cp = nullptr;
  cudaEvent_t ev_start = nullptr, ev_copied[2] = {nullptr, nullptr},
              ev_free[2] = {nullptr, nullptr};

  explicit EncoderImpl(const EncSpec& sp) : s(sp) {
    F1 = (s.idim - 3) / 2 + 1;
    F2 = (F1 - 3) / 2 + 1;
  }
  ~EncoderImpl() {
    if (cp) cudaStreamDestroy(cp);
    for (cudaEvent_t ev : {ev_start, ev_copied[0], ev_copied[1], ev_free[0], ev_free[1]})
      if (ev) cudaEventDestroy(ev);
    if (wbuf) cudaFree(wbuf);
    if (ws) cudaFree(ws);
    if (pe) cudaFree(pe);
  }

  // Weights in the flat order documented in bl_b200.h (torch layouts).
  cudaError_t load(const float* w) {
    const size_t d = s.d;
    std::vector<float> f32;
    std::vector<uint16_t> b16;
    struct Slot {
      bool bf;
      size_t off;
    };
    std::vector<Slot> slots;
    auto put32 = [&](const float* p, size_t n) {
      slots.push_back({false, f32.size()});
      f32.insert(f32.end(), p, p + n);
    };
    auto put16 = [&](const std::vector<float>& v) {
      slots.push_back({true, b16.size()});
      for (float x : v) b16.push_back(to_bf16(x));
      while (b16.size() % 64) b16.push_back(0);  // keep 128-B alignment
    };
    const float* p = w;
    put32(p, d * 9); p += d * 9;      // conv1.w [d][1][3][3]
    put32(p, d); p += d;              // conv1.b
    {                                 // conv2.w [o][c][kh][kw] -> [o][(kh*3+kw)*d + c]
      std::vector<float> v(d * 9 * d);
      for (size_t o = 0; o < d; ++o)
        for (size_t c = 0; c < d; ++c)
          for (int t = 0; t < 9; ++t) v[o * 9 * d + t * d + c] = p[(o * d + c) * 9 + t];
      put16(v);
      p += d * d * 9;
    }
    put32(p, d); p += d;              // conv2.b
    {                                 // out.w [o][c*F2 + f] -> [o][f*d + c]
      const size_t K = d * F2;
      std::vector<float> v(d * K);
      for (size_t o = 0; o < d; ++o)
        for (size_t c = 0; c < d; ++c)
          for (int f = 0; f < F2; ++f) v[o * K + f * d + c] = p[o * K + c * F2 + f];
      put16(v);
      p += d * K;
    }
    put32(p, d); p += d;              // out.b
    for (int l = 0; l < s.layers; ++l) {
      put32(p, d); p += d;            // ln1.g
      put32(p, d); p += d;            // ln1.b
      std::vector<float> qkv(3 * d * d), bq(3 * d);
      for (int j = 0; j < 3; ++j) {   // wq,bq,wk,bk,wv,bv -> [3d][d], [3d]
        std::memcpy(&qkv[j * d * d], p, d * d * 4); p += d * d;
        std::memcpy(&bq[j * d], p, d * 4); p += d;
      }
      put16(qkv);
      put32(bq.data(), 3 * d);
      put16(std::vector<float>(p, p + d * d)); p += d * d;  // wo
      put32(p, d); p += d;            // bo
      put32(p, d); p += d;            // ln2.g
      put32(p, d); p += d;            // ln2.b
      put16(std::vector<float>(p, p + s.dff * d)); p += s.dff * d;  // w1 [dff][d]
      put32(p, s.dff); p += s.dff;    // b1
      put16(std::vector<float>(p, p + d * s.dff)); p += d * s.dff;  // w2 [d][dff]
      put32(p, d); p += d;            // b2
    }
    put32(p, d); p += d;              // after_norm.g
    put32(p, d); p += d;              // after_norm.b
    put16(std::vector<float>(p, p + (size_t)s.vocab * d)); p += (size_t)s.vocab * d;  // ctc.w
    put32(p, s.vocab);                // ctc.b
    while (f32.size() % 32) f32.push_back(0.f);

    const size_t bytes32 = f32.size() * 4, bytes16 = b16.size() * 2;
    cudaError_t e = cudaMalloc(&wbuf, bytes32 + bytes16);
    if (e != cudaSuccess) return e;
    float* d32 = static_cast<float*>(wbuf);
    __nv_bfloat16* d16 = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(wbuf) + bytes32);
    if ((e = cudaMemcpy(d32, f32.data(), bytes32, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    if ((e = cudaMemcpy(d16, b16.data(), bytes16, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    size_t k = 0;
    auto nx32 = [&]() { return d32 + slots[k++].off; };
    auto nx16 = [&]() { return d16 + slots[k++].off; };
    c1w = nx32(); c1b = nx32(); c2w = nx16(); c2b = nx32(); ow = nx16(); ob = nx32();
    L.resize(s.layers);
    for (auto& y : L) {
      y.ln1g = nx32(); y.ln1b = nx32(); y.wqkv = nx16(); y.bqkv = nx32(); y.wo = nx16();
      y.bo = nx32(); y.ln2g = nx32(); y.ln2b = nx32(); y.w1 = nx16(); y.b1 = nx32();
      y.w2 = nx16(); y.b2 = nx32();
    }
    ang = nx32(); anb = nx32(); cw = nx16(); cb = nx32();
    return cudaSuccess;
  }

  cudaError_t ensure_pe(int T2) {
    if (pe_rows >= T2) return cudaSuccess;
    if (pe) cudaFree(pe);
    pe = nullptr;
    std::vector<float> h((size_t)T2 * s.d);
    const float k = -std::log(10000.0f) / s.d;
    for (int t = 0; t < T2; ++t)
      for (int i = 0; i < s.d; i += 2) {
        const float div = std::exp((float)i * k);
        const float a = (float)t * div;
        h[(size_t)t * s.d + i] = std::sin(a);
        h[(size_t)t * s.d + i + 1] = std::cos(a);
      }
    cudaError_t e = cudaMalloc(&pe, h.size() * 4);
    if (e != cudaSuccess) return e;
    pe_rows = T2;
    return cudaMemcpy(pe, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  }

  static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

  // Bytes of workspace for a chunk of S segments of T_in frames.
  size_t chunk_bytes(int S, int T_in, bool host_fbank) const {
    const size_t T1 = (T_in - 3) / 2 + 1, T2 = enc_frames_out(T_in), d = s.d;
    size_t b = 0;
    if (host_fbank) b += 2 * al((size_t)S * T_in * s.idim * 4);  // double-buffered
    b += al((size_t)S * T1 * F1 * d * 2);
    b += al((size_t)S * T2 * F2 * d * 2);
    b += al((size_t)S * T2 * d * 4);
    b += al((size_t)S * T2 * d * 2) * 2;
    b += al((size_t)S * T2 * 3 * d * 2);
    b += al((size_t)S * T2 * s.dff * 2);
    return b;
  }

  cudaError_t gemm(int M, int N, int K, const __nv_bfloat16* A, const __nv_bfloat16* B, int mode,
                   const float* bias, float* of, __nv_bfloat16* ob16, int ldo) {
    GemmDesc g;
    g.M = M; g.N = N; g.K = K; g.A = A; g.lda = K; g.B = B; g.ldb = K;
    g.mode = mode; g.bias = bias; g.out_f32 = of; g.out_bf16 = ob16; g.ldo = ldo;
    if (mode == kScalePe) {
      g.scale = std::sqrt((float)s.d);
      g.pe = pe;
      g.pe_rows = enc_frames_out(cur_tin);
    }
    ++launches;
    return gemm_bf16(g, st);
  }
  int cur_tin = 0;

  // n segments of T_in frames; fbank [n][T_in][idim] (host or device);
  // grid [n][T2][vocab] device fp32.
  cudaError_t forward(int n, int T_in, const float* fbank, bool on_device, float* grid,
                      int chunk, __nv_bfloat16* memory = nullptr) {
    cur_tin = T_in;
    const int T1 = (T_in - 3) / 2 + 1, T2 = enc_frames_out(T_in), d = s.d;
    cudaError_t e = ensure_pe(T2);
    if (e != cudaSuccess) return e;
    const int S = std::max(1, std::min(chunk, n));
    const size_t need = chunk_bytes(S, T_in, !on_device);
    if (need > ws_bytes) {
      if (ws) cudaFree(ws);
      ws = nullptr;
      ws_bytes = 0;
      if ((e = cudaMalloc(&ws, need)) != cudaSuccess) return e;
      ws_bytes = need;
    }
    const int T2max = T2;
    const size_t attn_smem =
        (size_t)2 * T2max * kKvPitch * 2 + kAttnWarps * kDk * 4 + (size_t)kAttnWarps * T2max * 4;
    if (attn_smem > 227 * 1024) return cudaErrorInvalidValue;
    if ((e = cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)attn_smem)) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(attention_tc_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kAttSmem)) !=
        cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(attention_tc512_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kAtt2Smem)) !=
        cudaSuccess)
      return e;
    launches = 0;
    const size_t fb_elems = (size_t)S * T_in * s.idim;
    float* stage[2] = {nullptr, nullptr};
    char* p0 = static_cast<char*>(ws);
    if (!on_device) {
      if (!cp) {
        if ((e = cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (cudaEvent_t* ev : {&ev_start, &ev_copied[0], &ev_copied[1], &ev_free[0], &ev_free[1]})
          if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
      }
      stage[0] = reinterpret_cast<float*>(p0);
      stage[1] = reinterpret_cast<float*>(p0 + al(fb_elems * 4));
      p0 += 2 * al(fb_elems * 4);
      // copies may start once earlier work on st (a previous forward) is done
      if ((e = cudaEventRecord(ev_start, st)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(cp, ev_start, 0)) != cudaSuccess) return e;
    }
    auto prefetch = [&](int ci) -> cudaError_t {
      const int c0 = ci * S, cn = std::min(S, n - c0);
      const int b = ci & 1;
      cudaError_t r;
      if (ci >= 2 && (r = cudaStreamWaitEvent(cp, ev_free[b], 0)) != cudaSuccess) return r;
      if ((r = cudaMemcpyAsync(stage[b], fbank + (size_t)c0 * T_in * s.idim,
                               (size_t)cn * T_in * s.idim * 4, cudaMemcpyHostToDevice, cp)) !=
          cudaSuccess)
        return r;
      return cudaEventRecord(ev_copied[b], cp);
    };
    if (!on_device && (e = prefetch(0)) != cudaSuccess) return e;
    for (int s0 = 0, ci = 0; s0 < n; s0 += S, ++ci) {
      const int ns = std::min(S, n - s0);
      char* p = p0;
      auto take = [&](size_t b) {
        char* r = p;
        p += al(b);
        return r;
      };
      const float* fb = fbank + (size_t)s0 * T_in * s.idim;
      if (!on_device) {
        if (s0 + S < n && (e = prefetch(ci + 1)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(st, ev_copied[ci & 1], 0)) != cudaSuccess) return e;
        fb = stage[ci & 1];
      }
      auto* c1 = reinterpret_cast<__nv_bfloat16*>(take((size_t)S * T1 * F1 * d * 2));
      auto* c2 = reinterpret_cast<__nv_bfloat16*>(take((size_t)S * T2 * F2 * d * 2));
      auto* X = reinterpret_cast<float*>(take((size_t)S * T2 * d * 4));
      auto* Y = reinterpret_cast<__nv_bfloat16*>(take((size_t)S * T2 * d * 2));
      auto* AO = reinterpret_cast<__nv_bfloat16*>(take((size_t)S * T2 * d * 2));
      auto* QKV = reinterpret_cast<__nv_bfloat16*>(take((size_t)S * T2 * 3 * d * 2));
      auto* H = reinterpret_cast<__nv_bfloat16*>(take((size_t)S * T2 * s.dff * 2));
      float* out = grid + (size_t)s0 * T2 * s.vocab;

      conv1_kernel<<<dim3((T1 + kC1Frames - 1) / kC1Frames, ns), 256,
                     (2 * kC1Frames + 1) * s.idim * sizeof(float), st>>>(fb, T_in, s.idim, T1,
                                                                         F1, d, c1w, c1b, c1);
      if (!on_device && (e = cudaEventRecord(ev_free[ci & 1], st)) != cudaSuccess) return e;
      launches += 2;
      const int M = ns * T2;
      {
        Conv2Desc cd;
        cd.c1 = c1; cd.S = ns; cd.T1 = T1; cd.F1 = F1; cd.T2 = T2; cd.F2 = F2; cd.d = d;
        cd.W = c2w; cd.bias = c2b; cd.out = c2;
        if ((e = conv2_bf16(cd, st)) != cudaSuccess) return e;
      }
      if ((e = gemm(M, d, F2 * d, c2, ow, kScalePe, ob, X, nullptr, d)) != cudaSuccess) return e;
      const int ln_blocks = (M + 7) / 8;
      auto ln = [&](const float* g, const float* b) {
        ++launches;
        launch_layernorm(d, X, M, g, b, Y, st);
      };
      for (const auto& y : L) {
        ln(y.ln1g, y.ln1b);
        if ((e = gemm(M, 3 * d, d, Y, y.wqkv, kPlain, y.bqkv, nullptr, QKV, 3 * d)) != cudaSuccess)
          return e;
        if (T2 <= kAtt2K && std::getenv("BL_ENC_ATTN_CUDA") == nullptr) {
          CUtensorMap tQ, tKV;
          if (!make_tmap(&tQ, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, QKV, 3 * d, M, (size_t)6 * d,
                         kDk, kAttQ, CU_TENSOR_MAP_SWIZZLE_128B) ||
              !make_tmap(&tKV, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, QKV, 3 * d, M, (size_t)6 * d,
                         kDk, kAttK, CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
          if (T2 <= kAttK)
            attention_tc_kernel<<<dim3(ns, s.heads, (T2 + kAttQ - 1) / kAttQ), 128, kAttSmem,
                                  st>>>(tQ, tKV, T2, d, AO);
          else
            attention_tc512_kernel<<<dim3(ns, s.heads, (T2 + kAttQ - 1) / kAttQ), 128,
                                     kAtt2Smem, st>>>(tQ, tKV, T2, d, AO);
        } else {
          attention_kernel<<<dim3(ns, s.heads), kAttnWarps * 32, attn_smem, st>>>(QKV, T2, d,
                                                                                 s.heads, AO);
        }
        ++launches;
        if ((e = gemm(M, d, d, AO, y.wo, kResidual, y.bo, X, nullptr, d)) != cudaSuccess) return e;
        ln(y.ln2g, y.ln2b);
        if ((e = gemm(M, s.dff, d, Y, y.w1, kRelu, y.b1, nullptr, H, s.dff)) != cudaSuccess)
          return e;
        if ((e = gemm(M, d, s.dff, H, y.w2, kResidual, y.b2, X, nullptr, d)) != cudaSuccess)
          return e;
      }
      ln(ang, anb);
      if (memory &&
          (e = cudaMemcpyAsync(memory + (size_t)s0 * T2 * d, Y, (size_t)M * d * 2,
                               cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return e;
      if ((e = gemm(M, s.vocab, d, Y, cw, kPlain, cb, out, nullptr, s.vocab)) != cudaSuccess)
        return e;
      log_softmax_kernel<<<M, 256, 0, st>>>(out, s.vocab);
      ++launches;
    }
    return cudaGetLastError();
  }
};

}  // namespace bl

namespace bl {

cudaError_t enc_create(const EncSpec& s, const float* w, EncoderImpl** out) {
  auto* e = new EncoderImpl(s);
  cudaError_t r = e->load(w);
  if (r != cudaSuccess) {
    delete e;
    return r;
  }
  *out = e;
  return cudaSuccess;
}
void enc_destroy(EncoderImpl* e) { delete e; }
void layer_norm_bf16(int d, const float* X, int rows, const float* g, const float* b,
                     __nv_bfloat16* Y, cudaStream_t st) {
  launch_layernorm(d, X, rows, g, b, Y, st);
}
void enc_set_stream(EncoderImpl* e, cudaStream_t st) { e->st = st; }
cudaStream_t enc_stream(EncoderImpl* e) { return e->st; }
cudaError_t enc_forward(EncoderImpl* e, int n, int T_in, const float* fb, bool on_device,
                        float* grid, int chunk, int* launches, __nv_bfloat16* memory) {
  cudaError_t r = e->forward(n, T_in, fb, on_device, grid, chunk, memory);
  if (launches) *launches = e->launches;
  return r;
}
size_t enc_workspace_bytes(EncoderImpl* e) { return e->ws_bytes; }

}  // namespace bl
