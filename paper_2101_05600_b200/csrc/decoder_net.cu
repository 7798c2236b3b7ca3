// decoder_net.cu — the Transformer attention decoder as a device scorer
// (SURVEY §8 a'2), batched over every hypothesis of every utterance and run
// once per decode step between launches of the step-granular search kernel.
//
// Step l for hypothesis slot k of utterance u (row R = u*B + k):
//   token   = sos (= |C|) at l = 1, else hist[u][l-1][k].token
//   anc[p]  = the slot, in beam p+1, of the ancestor whose KV entry holds
//             position p (walk of the search's back-pointers; anc[l-1] = k)
//   x = emb[token] * sqrt(d) + PE[l-1]
//   per layer:  x += O(SelfAttn(LN1 x))   keys/values: cache[p][anc[p]], p < l
//               x += O2(SrcAttn(LN2 x))   memory K/V precomputed per group
//               x += FFN(LN3 x)
//   att = log_softmax(out(LN x)) with an fp64 normaliser -> att / attf rows
//
// HBM layout (group of U utterances, S step positions):
//   kvc  bf16 [L][U][S][B][2d]   self-attention K|V per (position, slot)
//   kv2  bf16 [L][U*T2][2d]      source-attention K|V of the encoder memory
//   X f32 / Y, QKV, AO bf16 / H bf16 [U*B][...]; logits f32, att f64, attf f32 [U*B][V]
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "decoder_net.cuh"
#include "encoder.cuh"
#include "gemm.cuh"

namespace bl {
namespace {

constexpr int kDk = 64;

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// tokens and ancestor slots of every hypothesis row. The ancestry is built
// incrementally: row R = (u, k) at step l inherits its parent's row of the
// previous step's table (anc_prev) and appends its own slot at position l-1,
// so each step is one parallel gather instead of a pointer chase.
__global__ void dec_tok_kernel(int l, const HistRec* __restrict__ hist, int hstride, int U, int B,
                               int V, int* __restrict__ tok, int* __restrict__ par) {
  const int R = blockIdx.x * blockDim.x + threadIdx.x;
  if (R >= U * B) return;
  const int u = R / B, k = R - u * B;
  int t = V - 1, pj = 0;
  if (l > 1) {
    const HistRec h = hist[(size_t)u * hstride + (size_t)(l - 1) * B + k];
    t = (h.token >= 0 && h.token < V) ? h.token : V - 1;  // dead slot: any valid row
    pj = (h.parent >= 0 && h.parent < B) ? h.parent : 0;
  }
  tok[R] = t;
  par[R] = pj;
}

__global__ void dec_anc_kernel(int l, int U, int B, int S, const int* __restrict__ par,
                               const int* __restrict__ anc_prev, int* __restrict__ anc) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)U * B * l) return;
  const int R = (int)(i / l), p = (int)(i - (size_t)R * l);
  const int u = R / B, k = R - u * B;
  anc[(size_t)R * S + p] =
      p == l - 1 ? k : anc_prev[((size_t)u * B + par[R]) * S + p];
}

// x = emb[token] * sqrt(d) + pe[l-1]; one warp per row
__global__ void dec_embed_kernel(const int* __restrict__ tok, const float* __restrict__ emb,
                                 const float* __restrict__ pe_row, int d, float scale,
                                 float* __restrict__ X, int M) {
  const int R = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (R >= M) return;
  const float* e = emb + (size_t)tok[R] * d;
  float* x = X + (size_t)R * d;
  for (int c = lane; c < d; c += 32) x[c] = e[c] * scale + pe_row[c];
}

// Self-attention of the new position over each hypothesis' own prefix.
// Grid (U, heads), one warp per slot: the warps of one CTA are the beam of
// one utterance, so ancestor entries shared by several hypotheses are served
// from L1 (the live beam's union of entries is ~12% of nb*l on the bench
// model). The step's K/V go to the cache at position l-1; scores use 4 lanes
// per position (16 dims each), 8 positions per pass; the weighted sum has each
// lane own two dims. Finished utterances and dead slots (k >= nb) return at
// once.
__global__ void dec_self_attn_kernel(int l, const __nv_bfloat16* __restrict__ qkv, int d, int B,
                                     const int* __restrict__ anc, int S,
                                     const int* __restrict__ nb_in,
                                     __nv_bfloat16* __restrict__ cache,
                                     __nv_bfloat16* __restrict__ out) {
  extern __shared__ float sa_sm[];
  const int u = blockIdx.x, h = blockIdx.y;
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = l == 1 ? 1 : nb_in[u];
  if (k >= nb) return;
  float* sc = sa_sm + (size_t)k * S;                                        // [S] scores
  int* sl = reinterpret_cast<int*>(sa_sm + (size_t)B * S) + (size_t)k * S;  // [S] slots
  const int R = u * B + k;
  const __nv_bfloat16* row = qkv + (size_t)R * 3 * d;
  const size_t d2 = 2 * (size_t)d;
  auto kv_at = [&](int p, int slot) {
    return cache + (((size_t)u * S + p) * B + slot) * d2 + h * kDk;
  };
  {  // this step's K and V into the cache (position l-1, own slot)
    const uint32_t kc = reinterpret_cast<const uint32_t*>(row + d + h * kDk)[lane];
    const uint32_t vc = reinterpret_cast<const uint32_t*>(row + 2 * d + h * kDk)[lane];
    __nv_bfloat16* dst = kv_at(l - 1, k);
    reinterpret_cast<uint32_t*>(dst)[lane] = kc;
    reinterpret_cast<uint32_t*>(dst + d)[lane] = vc;
  }
  for (int p = lane; p < l; p += 32) sl[p] = (p == l - 1) ? k : anc[(size_t)R * S + p];
  __syncwarp();  // cache writes and slot list visible to the warp
  const int qd = lane & 3, pp = lane >> 2;
  float q[16];
  {
    const uint4* qs = reinterpret_cast<const uint4*>(row + h * kDk + qd * 16);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint4 w = qs[i];
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(b2[j]);
        q[i * 8 + 2 * j] = f.x;
        q[i * 8 + 2 * j + 1] = f.y;
      }
    }
  }
  const float scale = rsqrtf((float)kDk);
  float m = -INFINITY;
  // two 8-position passes per iteration: four 16-byte K loads per lane in
  // flight before the dot products
  for (int p0 = 0; p0 < l; p0 += 16) {
    uint4 kw[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int p = p0 + 8 * r + pp;
      if (p < l) {
        const uint4* ks = reinterpret_cast<const uint4*>(kv_at(p, sl[p]) + qd * 16);
        kw[r][0] = ks[0];
        kw[r][1] = ks[1];
      } else {
        kw[r][0] = kw[r][1] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int p = p0 + 8 * r + pp;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&kw[r][i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(b2[j]);
          s = fmaf(q[i * 8 + 2 * j], f.x, s);
          s = fmaf(q[i * 8 + 2 * j + 1], f.y, s);
        }
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (p < l) {
        s *= scale;
        if (qd == 0) sc[p] = s;
        m = fmaxf(m, s);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __syncwarp();
  float sum = 0.f;
  for (int p = lane; p < l; p += 32) {
    const float e = expf(sc[p] - m);
    sc[p] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncwarp();
  // weighted V sum: 8 lanes x 8 dims (16-byte loads) per position, 4
  // positions per warp pass and two passes unrolled, so 8 independent row
  // loads are in flight per warp; the 4 position groups are summed at the end
  const int vd = lane & 7, vp = lane >> 3;
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0.f;
  auto vacc = [&](int p) {
    const float w = sc[p];
    const uint4 raw = *reinterpret_cast<const uint4*>(kv_at(p, sl[p]) + d + vd * 8);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(b2[j]);
      a[2 * j] = fmaf(w, f.x, a[2 * j]);
      a[2 * j + 1] = fmaf(w, f.y, a[2 * j + 1]);
    }
  };
  int p0 = 0;
  for (; p0 + 8 <= l; p0 += 8) {
    vacc(p0 + vp);
    vacc(p0 + 4 + vp);
  }
  if (p0 + vp < l) vacc(p0 + vp);
  if (p0 + 4 + vp < l) vacc(p0 + 4 + vp);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] += __shfl_xor_sync(0xffffffffu, a[i], 8);
    a[i] += __shfl_xor_sync(0xffffffffu, a[i], 16);
  }
  if (vp == 0) {
    const float inv = 1.f / sum;
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) o2[j] = __floats2bfloat162_rn(a[2 * j] * inv, a[2 * j + 1] * inv);
    *reinterpret_cast<uint4*>(out + (size_t)R * d + h * kDk + vd * 8) = o;
  }
}

// Source attention on the warp-level tensor path. Per (utterance, head) the
// B hypotheses' queries share the memory K/V, so the op is bound by reading
// K/V once (HBM); the products are tiny (16 x 64 x T) and use
// mma.sync.m16n8k16 bf16 with fp32 accumulation. Grid (U, heads, ceil(B/16)),
// 4 warps; K/V staged in shared memory (144-byte rows: conflict-free
// ldmatrix); each warp takes 64-key chunks with an online softmax, and the
// warps' partial (max, sum, O) are merged at the end.
constexpr int kXW = 4, kXKPitch = 72;  // bf16 elements per staged row

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& b0, uint32_t& b1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& b0, uint32_t& b1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(b0), "=r"(b1)
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, unsigned src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t pk_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__global__ void __launch_bounds__(kXW * 32)
    dec_cross_attn_mma_kernel(int l, const int* __restrict__ nb_in,
                              const __nv_bfloat16* __restrict__ q,
                              const __nv_bfloat16* __restrict__ kv2, int T, int d, int B,
                              __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char xm_sm[];
  if (l > 1 && nb_in[blockIdx.x] <= (int)blockIdx.z * 16) return;  // finished utterance
  const int Tp = (T + 63) & ~63;
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(xm_sm);
  __nv_bfloat16* Vs = Ks + (size_t)Tp * kXKPitch;
  // after the key loop the K/V tiles are dead: the warps' partials reuse them
  float* mrg = reinterpret_cast<float*>(xm_sm);  // [warps][16*64 + 32]
  const int u = blockIdx.x, h = blockIdx.y, q0 = blockIdx.z * 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t ld = 2 * (size_t)d;
  const __nv_bfloat16* base = kv2 + (size_t)u * T * ld + h * kDk;
  // K/V rows straight into shared memory (cp.async, 16 B each, zero fill
  // past T): every thread keeps all its copies in flight
  for (int i = threadIdx.x; i < Tp * 8; i += blockDim.x) {  // 8 x 16 B per row
    const int t = i >> 3, c = i & 7;
    const int tt = t < T ? t : 0;
    const unsigned nbytes = t < T ? 16u : 0u;
    cp_async16(Ks + (size_t)t * kXKPitch + c * 8, base + tt * ld + c * 8, nbytes);
    cp_async16(Vs + (size_t)t * kXKPitch + c * 8, base + tt * ld + d + c * 8, nbytes);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  // query fragments: rows q0 + lane/4 (+8), dims kc*16 + 2*(lane%4) (+8)
  uint32_t qa[4][4];
  {
    const int r0 = q0 + (lane >> 2), r1 = r0 + 8, c = 2 * (lane & 3);
    const __nv_bfloat16* p0 = q + ((size_t)u * B + r0) * d + h * kDk + c;
    const __nv_bfloat16* p1 = q + ((size_t)u * B + r1) * d + h * kDk + c;
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      qa[kc][0] = r0 < B ? *reinterpret_cast<const uint32_t*>(p0 + kc * 16) : 0u;
      qa[kc][1] = r1 < B ? *reinterpret_cast<const uint32_t*>(p1 + kc * 16) : 0u;
      qa[kc][2] = r0 < B ? *reinterpret_cast<const uint32_t*>(p0 + kc * 16 + 8) : 0u;
      qa[kc][3] = r1 < B ? *reinterpret_cast<const uint32_t*>(p1 + kc * 16 + 8) : 0u;
    }
  }
  __syncthreads();
  const float sc = 1.4426950408889634f * rsqrtf((float)kDk);  // log2(e) / sqrt(dk)
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows lane/4, lane/4 + 8
  const uint32_t ks_base = (uint32_t)__cvta_generic_to_shared(Ks);
  const uint32_t vs_base = (uint32_t)__cvta_generic_to_shared(Vs);
  const int lr = lane & 7, lm = (lane >> 3) & 1;  // ldmatrix row / matrix of this lane
  for (int key0 = warp * 64; key0 < T; key0 += kXW * 64) {
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        uint32_t b0, b1;
        ldsm_x2(ks_base + (uint32_t)(((key0 + nt * 8 + lr) * kXKPitch + kc * 16 + lm * 8) * 2),
                b0, b1);
        mma16816(s[nt], qa[kc], b0, b1);
      }
    }
    float c0 = -INFINITY, c1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int key = key0 + nt * 8 + 2 * (lane & 3);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const bool ok = key + j < T;
        s[nt][j] = ok ? s[nt][j] * sc : -INFINITY;
        s[nt][2 + j] = ok ? s[nt][2 + j] * sc : -INFINITY;
        c0 = fmaxf(c0, s[nt][j]);
        c1 = fmaxf(c1, s[nt][2 + j]);
      }
    }
    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, 1));
    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, 2));
    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, 1));
    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, 2));
    const float n0 = fmaxf(m0, c0), n1 = fmaxf(m1, c1);
    const float a0 = exp2f(m0 - n0), a1 = exp2f(m1 - n1);
    m0 = n0;
    m1 = n1;
    l0 *= a0;
    l1 *= a1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i][0] *= a0; o[i][1] *= a0; o[i][2] *= a1; o[i][3] *= a1;
    }
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - n0), p1 = exp2f(s[nt][1] - n0);
      const float p2 = exp2f(s[nt][2] - n1), p3 = exp2f(s[nt][3] - n1);
      l0 += p0 + p1;
      l1 += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2] = pk_bf16(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pk_bf16(p2, p3);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        uint32_t b0, b1;
        ldsm_x2_t(vs_base + (uint32_t)(((key0 + kk * 16 + lm * 8 + lr) * kXKPitch + dt * 8) * 2),
                  b0, b1);
        mma16816(o[dt], pa[kk], b0, b1);
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  __syncthreads();  // every warp is done with Ks/Vs
  // merge the warps: O = sum_w O_w 2^(m_w - M), L = sum_w l_w 2^(m_w - M)
  float* mw = mrg + warp * (16 * 64 + 32);
  {
    const int r0 = lane >> 2, c = 2 * (lane & 3);
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      mw[r0 * 64 + dt * 8 + c] = o[dt][0];
      mw[r0 * 64 + dt * 8 + c + 1] = o[dt][1];
      mw[(r0 + 8) * 64 + dt * 8 + c] = o[dt][2];
      mw[(r0 + 8) * 64 + dt * 8 + c + 1] = o[dt][3];
    }
    if ((lane & 3) == 0) {
      mw[1024 + r0] = m0;
      mw[1024 + r0 + 8] = m1;
      mw[1040 + r0] = l0;
      mw[1040 + r0 + 8] = l1;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {  // (row, dim pair)
    const int r = i >> 5, c = (i & 31) * 2;
    if (q0 + r >= B) continue;
    float M = -INFINITY;
    for (int w = 0; w < kXW; ++w) M = fmaxf(M, mrg[w * (16 * 64 + 32) + 1024 + r]);
    float L = 0.f, x0 = 0.f, x1 = 0.f;
    for (int w = 0; w < kXW; ++w) {
      const float* pw = mrg + w * (16 * 64 + 32);
      const float mwv = pw[1024 + r];
      if (mwv == -INFINITY) continue;  // warp saw no keys
      const float f = exp2f(mwv - M);
      L += pw[1040 + r] * f;
      x0 += pw[r * 64 + c] * f;
      x1 += pw[r * 64 + c + 1] * f;
    }
    reinterpret_cast<__nv_bfloat162*>(out + ((size_t)u * B + q0 + r) * d + h * kDk)[c / 2] =
        __floats2bfloat162_rn(x0 / L, x1 / L);
  }
}

// att = logits - logsumexp(logits) with the normaliser in fp64 (rows then
// satisfy the reference's check_normalized to ~1e-15); attf for the
// certified fp32 bulk keys. One CTA per row.
__global__ void __launch_bounds__(256)
    dec_log_softmax64_kernel(const float* __restrict__ logits, int V, double lam,
                             double* __restrict__ att, float* __restrict__ attf) {
  __shared__ double red[8];
  const float* x = logits + (size_t)blockIdx.x * V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float mf = -INFINITY;
  for (int i = threadIdx.x; i < V; i += blockDim.x) mf = fmaxf(mf, x[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, o));
  if (lane == 0) red[warp] = mf;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < 8; ++w) m = fmax(m, red[w]);
  __syncthreads();
  double s = 0.0;
  for (int i = threadIdx.x; i < V; i += blockDim.x) s += exp((double)x[i] - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = 0.0;
  for (int w = 0; w < 8; ++w) s += red[w];
  const double lse = m + log(s);
  double* a = att + (size_t)blockIdx.x * V;
  float* af = attf + (size_t)blockIdx.x * V;
  const double w1 = lam <= 0.0 ? 1.0 : 1.0 - lam;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const double v = (double)x[i] - lse;
    a[i] = v;
    af[i] = lam >= 1.0 ? 0.f : (float)(w1 * v);
  }
}

// Self-attention over the union of the beam's ancestor entries, on the
// warp-level tensor path (B <= 16, S <= 4096). The hypotheses of one
// utterance share most of their prefix (the union of their KV entries is
// ~12% of nb*l on the bench model), so per (utterance, head) the CTA lists
// the distinct (position, slot) entries once, each tagged with the mask of
// hypotheses whose ancestry holds it, stages their K/V in shared memory and
// scores all B queries against every entry with mma.sync; entries outside a
// hypothesis' ancestry are masked to -inf before the online softmax. Each
// entry is read from HBM once per (utterance, head) instead of once per
// hypothesis, and the per-dim unpack + FMA moves onto the tensor pipe.
// Entry word: position (bits 0-11) | slot (12-15) | hypothesis mask (16-31).
// The step's own K/V (position l-1) are read from the QKV rows and written
// to the cache for the later steps. Grid (U, heads), kSuW warps; stages of
// kSuW * kSuKeys entries, each warp one chunk per stage.
// kCross = true runs the same pipeline as source attention: the entries are
// the utterance's T memory rows (every query row sees all of them), grid
// (U, heads, ceil(B/16)); staging 32 rows at a time keeps 11 CTAs per SM
// where dec_cross_attn_mma_kernel stages the whole memory (3 CTAs per SM).
// Launch shape from scripts/sweep_self_attn.sh (2880 segments, 747 launches):
// (keys, warps, min CTAs) 32,4,1: 231 ms; 16,4,6: 164; 16,2,12: 147;
// 16,2,11: 143; 16,1,16: 169 — the kernel is latency-bound on the staged
// HBM reads, so small CTAs at high residency win. With source attention on
// the same kernel (self + cross, 1494 launches): 16,2,11 single-buffered
// 253 ms; double-buffered (BL_SU_STAGES=2) 16,2,8 264, 16,2,10 262,
// 16,4,6 309, 32,2,8 327 — the second buffer costs more residency than
// the overlap it buys.
#ifndef BL_SU_KEYS
#define BL_SU_KEYS 16
#endif
#ifndef BL_SU_WARPS
#define BL_SU_WARPS 2
#endif
#ifndef BL_SU_MINB
#define BL_SU_MINB 11
#endif
constexpr int kSuKeys = BL_SU_KEYS;  // entries per warp chunk
#ifndef BL_SU_STAGES
#define BL_SU_STAGES 1
#endif
constexpr int kSuW = BL_SU_WARPS;    // warps per CTA
constexpr int kSuStages = BL_SU_STAGES;  // staging buffers (2: next stage in flight)
// The union of the live hypotheses' self-attention entries of one
// utterance at step l: every distinct (position, cache slot) any live
// hypothesis attends to, tagged with the mask of the hypotheses holding it,
// in position order (deterministic). Built once per step and utterance and
// shared by every head and layer of dec_attn_staged_kernel<false>.
template <int kW>
__global__ void __launch_bounds__(kW * 32)
    dec_union_kernel(int l, int B, const int* __restrict__ anc, int S,
                     const int* __restrict__ nb_in, uint32_t* __restrict__ gent,
                     int* __restrict__ gent_n) {
  const int u = blockIdx.x;
  const int nb = l == 1 ? 1 : nb_in[u];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ int wsum[kW];
  uint32_t* ent = gent + (size_t)u * (((size_t)B * S + 3) & ~(size_t)3);
  int n = 0;
  if (nb <= 0) {
    if (tid == 0) gent_n[u] = 0;
    return;
  }
  // union of the live hypotheses' entries, positions in contiguous runs per
  // thread so the block scan keeps position order (deterministic sums)
  const int per = (l + kW * 32 - 1) / (kW * 32);
  const int pb = min(l, tid * per), pe = min(l, pb + per);
  auto slots_at = [&](int p, int(&sk)[16]) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      sk[k] = k < nb ? (p == l - 1 ? k : anc[((size_t)u * B + k) * S + p]) : -1;
  };
  int cnt = 0;
  for (int p = pb; p < pe; ++p) {
    int sk[16];
    slots_at(p, sk);
    unsigned msk = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) msk |= sk[k] >= 0 ? 1u << sk[k] : 0u;
    cnt += __popc(msk);
  }
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int off = inc - cnt;
  n = 0;
#pragma unroll
  for (int w = 0; w < kW; ++w) {
    off += w < warp ? wsum[w] : 0;
    n += wsum[w];
  }
  for (int p = pb; p < pe; ++p) {
    int sk[16];
    slots_at(p, sk);
    unsigned msk = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) msk |= sk[k] >= 0 ? 1u << sk[k] : 0u;
    while (msk) {
      const int s = __ffs(msk) - 1;
      msk &= msk - 1;
      unsigned hm = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) hm |= (sk[k] == s ? 1u : 0u) << k;
      ent[off++] = (uint32_t)p | ((uint32_t)s << 12) | (hm << 16);
    }
  }
  if (tid == 0) gent_n[u] = n;
}

template <bool kCross, int kKeys, int kW, int kMinB>
__global__ void __launch_bounds__(kW * 32, kMinB)
    dec_attn_staged_kernel(int l, const __nv_bfloat16* __restrict__ qsrc, int d, int B,
                           const int* __restrict__ anc, int S, const int* __restrict__ nb_in,
                           __nv_bfloat16* __restrict__ kv, int T,
                           __nv_bfloat16* __restrict__ out,
                           const uint32_t* __restrict__ gent, const int* __restrict__ gent_n) {
  extern __shared__ __align__(16) unsigned char su_sm[];
  constexpr int kSt = kW * kKeys;  // entries per stage
  const int u = blockIdx.x, h = blockIdx.y;
  const int q0 = kCross ? (int)blockIdx.z * 16 : 0;
  const int nb = l == 1 ? 1 : nb_in[u];
  if (kCross ? (l > 1 && nb <= q0) : nb <= 0) return;  // finished utterance
  const int nrow = kCross ? min(16, B - q0) : nb;        // query rows of this CTA
  __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(su_sm);
  __nv_bfloat16* Vs = Ks + (size_t)kSuStages * kSt * kXKPitch;
  float* mrg = reinterpret_cast<float*>(su_sm);  // [warps][16*64 + 32] after the last stage
  uint32_t* ent = reinterpret_cast<uint32_t*>(Vs + (size_t)kSuStages * kSt * kXKPitch);  // [B*S]
  __shared__ int wsum[kW];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t d2 = 2 * (size_t)d, d3 = 3 * (size_t)d, qs = kCross ? d : d3;
  const __nv_bfloat16* rows = qsrc + ((size_t)u * B + q0) * qs;
  int n = T;  // entries: the memory rows (cross), else the union below
  if constexpr (!kCross) {
  // this step's K and V into the cache (position l-1, own slot): 16-byte
  // chunks (8 per 64-dim head row, K then V), every load of the thread in
  // flight before its stores (one memory latency, not one per chunk)
  {
    constexpr int kPer = (16 * 16 + kW * 32 - 1) / (kW * 32);  // chunks per thread (B <= 16)
    uint4 v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + j * kW * 32, k = i >> 4, c = i & 15;  // c < 8: K chunk, else V
      if (k < nb)
        v[j] = *reinterpret_cast<const uint4*>(rows + k * d3 + (c < 8 ? d : 2 * d) + h * kDk +
                                               (c & 7) * 8);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + j * kW * 32, k = i >> 4, c = i & 15;
      if (k < nb)
        *reinterpret_cast<uint4*>(kv + (((size_t)u * S + l - 1) * B + k) * d2 +
                                  (c < 8 ? 0 : d) + h * kDk + (c & 7) * 8) = v[j];
    }
  }
  // the union of the live hypotheses' entries, built once per step and
  // utterance by dec_union_kernel (shared by every head and layer)
  n = gent_n[u];
  {
    const uint4* src4 =
        reinterpret_cast<const uint4*>(gent + (size_t)u * (((size_t)B * S + 3) & ~(size_t)3));
    uint4* dst4 = reinterpret_cast<uint4*>(ent);
    for (int i = tid; i < (n + 3) / 4; i += blockDim.x) dst4[i] = src4[i];
  }
  }
  // query fragments: rows lane/4 (+8), dims kc*16 + 2*(lane%4) (+8)
  uint32_t qa[4][4];
  const int r0 = lane >> 2, r1 = r0 + 8;
  {
    const int c = 2 * (lane & 3);
    const __nv_bfloat16* p0 = rows + r0 * qs + h * kDk + c;
    const __nv_bfloat16* p1 = rows + r1 * qs + h * kDk + c;
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      qa[kc][0] = r0 < nrow ? *reinterpret_cast<const uint32_t*>(p0 + kc * 16) : 0u;
      qa[kc][1] = r1 < nrow ? *reinterpret_cast<const uint32_t*>(p1 + kc * 16) : 0u;
      qa[kc][2] = r0 < nrow ? *reinterpret_cast<const uint32_t*>(p0 + kc * 16 + 8) : 0u;
      qa[kc][3] = r1 < nrow ? *reinterpret_cast<const uint32_t*>(p1 + kc * 16 + 8) : 0u;
    }
  }
  const float sc = 1.4426950408889634f * rsqrtf((float)kDk);  // log2(e) / sqrt(dk)
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const uint32_t ks_base = (uint32_t)__cvta_generic_to_shared(Ks);
  const uint32_t vs_base = (uint32_t)__cvta_generic_to_shared(Vs);
  const int lr = lane & 7, lm = (lane >> 3) & 1;
  auto issue = [&](int e0, int buf) {
    __nv_bfloat16* Kb = Ks + (size_t)buf * kSt * kXKPitch;
    __nv_bfloat16* Vb = Vs + (size_t)buf * kSt * kXKPitch;
    for (int i = tid; i < kSt * 8; i += blockDim.x) {  // 8 x 16 B per row
      const int t = i >> 3, c = i & 7, e = e0 + t;
      const __nv_bfloat16* src = rows + h * kDk;  // any valid address for the zero fill
      unsigned nbytes = 0;
      if (kCross && e < n) {
        src = kv + ((size_t)u * T + e) * d2 + h * kDk;
        nbytes = 16;
      } else if (e < n) {
        const uint32_t w = ent[e];
        const int p = (int)(w & 0xfffu), s = (int)((w >> 12) & 0xfu);
        src = p == l - 1 ? rows + s * d3 + d + h * kDk
                         : kv + (((size_t)u * S + p) * B + s) * d2 + h * kDk;
        nbytes = 16;
      }
      cp_async16(Kb + (size_t)t * kXKPitch + c * 8, src + c * 8, nbytes);
      cp_async16(Vb + (size_t)t * kXKPitch + c * 8, src + d + c * 8, nbytes);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();  // entry list written
  if (kSuStages == 2 && n > 0) issue(0, 0);
  int stg = 0;
  for (int e0 = 0; e0 < n; e0 += kSt, ++stg) {
    const int buf = kSuStages == 2 ? (stg & 1) : 0;
    if (kSuStages == 2 && e0 + kSt < n) {
      issue(e0 + kSt, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      if (kSuStages == 1) issue(e0, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // stage visible to every warp
    const int key0 = warp * kKeys;
    const uint32_t kb = ks_base + (uint32_t)(buf * kSt * kXKPitch * 2);
    const uint32_t vb = vs_base + (uint32_t)(buf * kSt * kXKPitch * 2);
    if (e0 + key0 < n) {
    float s[kKeys / 8][4];
#pragma unroll
    for (int nt = 0; nt < kKeys / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        uint32_t b0, b1;
        ldsm_x2(kb + (uint32_t)(((key0 + nt * 8 + lr) * kXKPitch + kc * 16 + lm * 8) * 2),
                b0, b1);
        mma16816(s[nt], qa[kc], b0, b1);
      }
    }
    float c0 = -INFINITY, c1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < kKeys / 8; ++nt) {
      const int e = e0 + key0 + nt * 8 + 2 * (lane & 3);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const unsigned hm = e + j < n ? (kCross ? 0xffffu : ent[e + j] >> 16) : 0u;
        s[nt][j] = (hm >> r0) & 1u ? s[nt][j] * sc : -INFINITY;
        s[nt][2 + j] = (hm >> r1) & 1u ? s[nt][2 + j] * sc : -INFINITY;
        c0 = fmaxf(c0, s[nt][j]);
        c1 = fmaxf(c1, s[nt][2 + j]);
      }
    }
    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, 1));
    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, 2));
    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, 1));
    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, 2));
    const float n0 = fmaxf(m0, c0), n1 = fmaxf(m1, c1);
    // a row with no entry so far keeps m = -inf: exponents against 0 give 0
    const float z0 = n0 == -INFINITY ? 0.f : n0, z1 = n1 == -INFINITY ? 0.f : n1;
    const float a0 = exp2f(m0 - z0), a1 = exp2f(m1 - z1);
    m0 = n0;
    m1 = n1;
    l0 *= a0;
    l1 *= a1;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i][0] *= a0; o[i][1] *= a0; o[i][2] *= a1; o[i][3] *= a1;
    }
    uint32_t pa[kKeys / 16][4];
#pragma unroll
    for (int nt = 0; nt < kKeys / 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - z0), p1 = exp2f(s[nt][1] - z0);
      const float p2 = exp2f(s[nt][2] - z1), p3 = exp2f(s[nt][3] - z1);
      l0 += p0 + p1;
      l1 += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2] = pk_bf16(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pk_bf16(p2, p3);
    }
#pragma unroll
    for (int kk = 0; kk < kKeys / 16; ++kk) {
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        uint32_t b0, b1;
        ldsm_x2_t(vb + (uint32_t)(((key0 + kk * 16 + lm * 8 + lr) * kXKPitch + dt * 8) * 2),
                  b0, b1);
        mma16816(o[dt], pa[kk], b0, b1);
      }
    }
    }
    __syncthreads();  // stage consumed before its buffer is refilled
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  __syncthreads();  // every warp is done with Ks/Vs
  float* mw = mrg + warp * (16 * 64 + 32);
  {
    const int c = 2 * (lane & 3);
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      mw[r0 * 64 + dt * 8 + c] = o[dt][0];
      mw[r0 * 64 + dt * 8 + c + 1] = o[dt][1];
      mw[r1 * 64 + dt * 8 + c] = o[dt][2];
      mw[r1 * 64 + dt * 8 + c + 1] = o[dt][3];
    }
    if ((lane & 3) == 0) {
      mw[1024 + r0] = m0;
      mw[1024 + r1] = m1;
      mw[1040 + r0] = l0;
      mw[1040 + r1] = l1;
    }
  }
  __syncthreads();
  for (int i = tid; i < 16 * 32; i += blockDim.x) {  // (row, dim pair)
    const int r = i >> 5, c = (i & 31) * 2;
    if (r >= nrow) continue;
    float M = -INFINITY;
    for (int w = 0; w < kW; ++w) M = fmaxf(M, mrg[w * (16 * 64 + 32) + 1024 + r]);
    float L = 0.f, x0 = 0.f, x1 = 0.f;
    for (int w = 0; w < kW; ++w) {
      const float* pw = mrg + w * (16 * 64 + 32);
      const float mwv = pw[1024 + r];
      if (mwv == -INFINITY) continue;  // warp saw none of this row's entries
      const float f = exp2f(mwv - M);
      L += pw[1040 + r] * f;
      x0 += pw[r * 64 + c] * f;
      x1 += pw[r * 64 + c + 1] * f;
    }
    reinterpret_cast<__nv_bfloat162*>(out + ((size_t)u * B + q0 + r) * d + h * kDk)[c / 2] =
        __floats2bfloat162_rn(x0 / L, x1 / L);
  }
}

// source attention's own launch shape (scripts/sweep_src_attn.sh, staged
// self + source totals over 1494 launches; (keys, warps, min CTAs)):
// 16,2,11 253 ms; 32,2,8 247; 32,1,16 247; 32,1,20 244; 64,2,6 244;
// 32,4,4 264; 64,4,3 280
#ifndef BL_XS_KEYS
#define BL_XS_KEYS 64
#endif
#ifndef BL_XS_WARPS
#define BL_XS_WARPS 2
#endif
#ifndef BL_XS_MINB
#define BL_XS_MINB 6
#endif
#define SELF_ATTN dec_attn_staged_kernel<false, kSuKeys, kSuW, BL_SU_MINB>
#define SRC_ATTN dec_attn_staged_kernel<true, BL_XS_KEYS, BL_XS_WARPS, BL_XS_MINB>
size_t stage_smem(int keys, int warps) {
  return std::max(2 * (size_t)kSuStages * warps * keys * kXKPitch * 2,
                  (size_t)warps * (16 * 64 + 32) * 4);
}
size_t xs_smem() { return stage_smem(BL_XS_KEYS, BL_XS_WARPS); }
// The same rows one warp per row (8 rows per CTA, shuffle reductions only,
// no block barriers); the row is re-read from L1 for each pass.
__global__ void __launch_bounds__(256)
    dec_log_softmax64_warp_kernel(const float* __restrict__ logits, int V, int M, double lam,
                                  double* __restrict__ att, float* __restrict__ attf,
                                  double* __restrict__ lse_out) {
  const int lane = threadIdx.x & 31;
  const int R = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (R >= M) return;
  const float* x = logits + (size_t)R * V;
  float mf = -INFINITY;
  for (int i = lane; i < V; i += 32) mf = fmaxf(mf, x[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, o));
  const double m = mf;
  // terms by the correctly rounded-ish fp32 expf (<= 2 ulp; x - m is exact in
  // fp32 near the max), summed in fp64: the row normalises to ~1e-7, inside
  // the reference's check_normalized bound (1e-6, scorer.cpp:14-28)
  double sum = 0.0;
  for (int i = lane; i < V; i += 32) sum += (double)expf(x[i] - mf);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double lse = m + log(sum);
  if (lse_out && lane == 0) lse_out[R] = lse;
  float* af = attf + (size_t)R * V;
  const double w1 = lam <= 0.0 ? 1.0 : 1.0 - lam;
  for (int i = lane; i < V; i += 32) {
    const double v = (double)x[i] - lse;
    if (att) att[(size_t)R * V + i] = v;  // fp64 rows only when materialised
    af[i] = lam >= 1.0 ? 0.f : (float)(w1 * v);
  }
}

// The same normaliser with each row read from HBM ONCE: a warp stages its
// row in shared memory (16-byte cp.async), then the max, the fp64 sum and
// the attf writes read shared memory. Lane i still takes elements i, i+32,
// ... in the same order, so lse and attf are bit-identical to the warp
// kernel above (which reads the row three times: 1.7 GB of DRAM reads per
// 0.58 GB of logits at 28,800 rows x 5000). 4 warps (rows) per CTA.
__global__ void __launch_bounds__(128)
    dec_log_softmax64_staged_kernel(const float* __restrict__ logits, int V, int M, double lam,
                                    float* __restrict__ attf, double* __restrict__ lse_out) {
  extern __shared__ __align__(16) float ls_rows[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R = blockIdx.x * 4 + warp;
  if (R >= M) return;
  float* xs = ls_rows + (size_t)warp * V;
  const float* x = logits + (size_t)R * V;
  for (int i = lane; i < V / 4; i += 32) cp_async16(xs + 4 * i, x + 4 * i, 16);
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  float mf = -INFINITY;
  for (int i = lane; i < V; i += 32) mf = fmaxf(mf, xs[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, o));
  const double m = mf;
  double sum = 0.0;
  for (int i = lane; i < V; i += 32) sum += (double)expf(xs[i] - mf);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double lse = m + log(sum);
  if (lse_out && lane == 0) lse_out[R] = lse;
  float* af = attf + (size_t)R * V;
  const double w1 = lam <= 0.0 ? 1.0 : 1.0 - lam;
  for (int i = lane; i < V / 4; i += 32) {
    const float4 v4 = reinterpret_cast<const float4*>(xs)[i];
    float4 o4;
    o4.x = lam >= 1.0 ? 0.f : (float)(w1 * ((double)v4.x - lse));
    o4.y = lam >= 1.0 ? 0.f : (float)(w1 * ((double)v4.y - lse));
    o4.z = lam >= 1.0 ? 0.f : (float)(w1 * ((double)v4.z - lse));
    o4.w = lam >= 1.0 ? 0.f : (float)(w1 * ((double)v4.w - lse));
    reinterpret_cast<float4*>(af)[i] = o4;
  }
}

// Fold the output GEMM's partials into each row's log-normaliser (fp64):
// lse = m + log(sum_t s_t exp(m_t - m)), m = max_t m_t over written slots.
__global__ void dec_lse_kernel(const double* __restrict__ part, int stride, int M,
                               double* __restrict__ lse) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  const double* p = part + (size_t)r * stride * 2;
  double m = -HUGE_VAL;
  for (int t = 0; t < stride; ++t)
    if (p[2 * t + 1] > 0.0) m = fmax(m, p[2 * t]);
  double sum = 0.0;
  for (int t = 0; t < stride; ++t)
    if (p[2 * t + 1] > 0.0) sum += p[2 * t + 1] * exp(p[2 * t] - m);
  lse[r] = m + log(sum);
}

// fused mode: the fp32 (1 - lambda) att rows from the logits and the fp64
// normaliser (the search's certified keys read these rows)
__global__ void dec_attf_kernel(const float* __restrict__ logits, const double* __restrict__ lse,
                                int V, double lambda, float* __restrict__ attf) {
  const size_t r = blockIdx.x;
  const double l = lse[r];
  const double sc = lambda <= 0.0 ? 1.0 : 1.0 - lambda;
  for (int c = threadIdx.x; c < V; c += blockDim.x)
    attf[r * V + c] = lambda >= 1.0 ? 0.f : (float)(sc * ((double)logits[r * V + c] - l));
}

// Row normalisation modes. Default: one warp per row writes the fp32 attf
// row (every certified key reads one) and the fp64 log-normaliser; the search
// derives the few fp64 att values it needs as (double)logit - lse, so the
// fp64 rows (8 B x V per hypothesis per step) are never written.
// BL_FUSED_LOG_SOFTMAX=1: the partial {max, sum exp} in the output GEMM's
// epilogue instead (measured slower: the epilogue is the output GEMM's bound,
// DESIGN.md §4c). BL_LOG_SOFTMAX=rows|block: the materialised fp64 rows.
bool fused_log_softmax() {
  static const bool on = std::getenv("BL_FUSED_LOG_SOFTMAX") != nullptr;
  return on;
}
bool rows_log_softmax() {
  static const bool on = std::getenv("BL_LOG_SOFTMAX") != nullptr;
  return on;
}

// the warp-per-row normaliser unless BL_LOG_SOFTMAX=block (A/B runs)
bool use_warp_log_softmax() {
  static const bool block = [] {
    const char* v = std::getenv("BL_LOG_SOFTMAX");
    return v && std::strcmp(v, "block") == 0;
  }();
  return !block;
}

size_t su_smem(int B, int S) {
  return stage_smem(kSuKeys, kSuW) + (((size_t)B * S + 3) & ~(size_t)3) * 4;
}

// staged source attention unless BL_CROSS_ATTN=whole (A/B runs)
bool use_staged_cross_attn() {
  static const bool whole = [] {
    const char* v = std::getenv("BL_CROSS_ATTN");
    return v && std::strcmp(v, "whole") == 0;
  }();
  return !whole;
}

// the union kernel unless BL_SELF_ATTN=warp (A/B runs) or the beam / step
// count exceed its entry encoding or shared memory
bool use_union_self_attn(int B, int S) {
  static const bool warp = [] {
    const char* v = std::getenv("BL_SELF_ATTN");
    return v && std::strcmp(v, "warp") == 0;
  }();
  return !warp && B <= 16 && S <= 4096 && su_smem(B, S) <= 227 * 1024;
}

size_t xm_smem(int T) {
  const size_t Tp = (size_t)((T + 63) & ~63);
  return std::max(2 * Tp * kXKPitch * 2, (size_t)kXW * (16 * 64 + 32) * 4);
}

}  // namespace

struct DecLayer {
  float *ln1g, *ln1b, *bqkv, *bo, *ln2g, *ln2b, *bq2, *bkv2, *bo2, *ln3g, *ln3b, *b1, *b2;
  __nv_bfloat16 *wqkv, *wo, *wq2, *wkv2, *wo2, *w1, *w2;
};

struct DecoderNet {
  DecSpec s;
  void* wbuf = nullptr;
  float* emb = nullptr;
  std::vector<DecLayer> L;
  float *ang, *anb, *bout;
  __nv_bfloat16* wout;
  float* pe = nullptr;
  int pe_rows = 0;
  // group state
  int U = 0, B = 0, S = 0, T2 = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  __nv_bfloat16 *kvc = nullptr, *kv2 = nullptr, *Y = nullptr, *QKV = nullptr, *AO = nullptr,
                *H = nullptr;
  float *X = nullptr, *logits = nullptr, *attf = nullptr;
  double* att = nullptr;
  double *lse_part = nullptr, *lse = nullptr;  // fused log-softmax (output GEMM epilogue)
  int lse_stride = 0;
  int *anc2[2] = {nullptr, nullptr}, *tok = nullptr, *par = nullptr;
  uint32_t* gent = nullptr;  // [U][B*S rounded to 4] self-attention union entries
  int* gent_n = nullptr;     // [U]

  ~DecoderNet() {
    if (wbuf) cudaFree(wbuf);
    if (ws) cudaFree(ws);
    if (pe) cudaFree(pe);
  }

  cudaError_t load(const float* w) {
    const size_t d = s.d, ff = s.dff, V = s.vocab;
    std::vector<float> f32;
    std::vector<uint16_t> b16;
    std::vector<std::pair<bool, size_t>> slots;
    auto put32 = [&](const float* p, size_t n) {
      slots.push_back({false, f32.size()});
      f32.insert(f32.end(), p, p + n);
      while (f32.size() % 32) f32.push_back(0.f);
    };
    auto put16 = [&](const float* p, size_t n) {
      slots.push_back({true, b16.size()});
      for (size_t i = 0; i < n; ++i) b16.push_back(to_bf16(p[i]));
      while (b16.size() % 64) b16.push_back(0);
    };
    const float* p = w;
    put32(p, V * d); p += V * d;  // embed.w (fp32, gathered)
    for (int l = 0; l < s.layers; ++l) {
      // self-attention block: ln1, q, k, v, o
      put32(p, d); p += d;
      put32(p, d); p += d;
      {
        std::vector<float> wq(3 * d * d), bq(3 * d);
        for (int j = 0; j < 3; ++j) {
          std::memcpy(&wq[j * d * d], p, d * d * 4); p += d * d;
          std::memcpy(&bq[j * d], p, d * 4); p += d;
        }
        put16(wq.data(), wq.size());
        put32(bq.data(), bq.size());
      }
      put16(p, d * d); p += d * d;  // wo
      put32(p, d); p += d;          // bo
      // source attention block: ln2, q2, k2, v2, o2
      put32(p, d); p += d;
      put32(p, d); p += d;
      put16(p, d * d); p += d * d;  // wq2
      put32(p, d); p += d;          // bq2
      {
        std::vector<float> wkv(2 * d * d), bkv(2 * d);
        for (int j = 0; j < 2; ++j) {
          std::memcpy(&wkv[j * d * d], p, d * d * 4); p += d * d;
          std::memcpy(&bkv[j * d], p, d * 4); p += d;
        }
        put16(wkv.data(), wkv.size());
        put32(bkv.data(), bkv.size());
      }
      put16(p, d * d); p += d * d;  // wo2
      put32(p, d); p += d;          // bo2
      put32(p, d); p += d;          // ln3.g
      put32(p, d); p += d;          // ln3.b
      put16(p, ff * d); p += ff * d;  // w1
      put32(p, ff); p += ff;          // b1
      put16(p, d * ff); p += d * ff;  // w2
      put32(p, d); p += d;            // b2
    }
    put32(p, d); p += d;          // after_norm.g
    put32(p, d); p += d;          // after_norm.b
    put16(p, V * d); p += V * d;  // out.w
    put32(p, V);                  // out.b
    const size_t n32 = f32.size() * 4, n16 = b16.size() * 2;
    cudaError_t e = cudaMalloc(&wbuf, n32 + n16);
    if (e != cudaSuccess) return e;
    float* d32 = static_cast<float*>(wbuf);
    auto* d16 = reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(wbuf) + n32);
    if ((e = cudaMemcpy(d32, f32.data(), n32, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    if ((e = cudaMemcpy(d16, b16.data(), n16, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
    size_t k = 0;
    auto f = [&]() { return d32 + slots[k++].second; };
    auto h = [&]() { return d16 + slots[k++].second; };
    emb = f();
    L.resize(s.layers);
    for (auto& y : L) {
      y.ln1g = f(); y.ln1b = f(); y.wqkv = h(); y.bqkv = f(); y.wo = h(); y.bo = f();
      y.ln2g = f(); y.ln2b = f(); y.wq2 = h(); y.bq2 = f(); y.wkv2 = h(); y.bkv2 = f();
      y.wo2 = h(); y.bo2 = f(); y.ln3g = f(); y.ln3b = f(); y.w1 = h(); y.b1 = f();
      y.w2 = h(); y.b2 = f();
    }
    ang = f(); anb = f(); wout = h(); bout = f();
    return cudaSuccess;
  }

  cudaError_t ensure_pe(int rows) {
    if (pe_rows >= rows) return cudaSuccess;
    if (pe) cudaFree(pe);
    pe = nullptr;
    std::vector<float> hp((size_t)rows * s.d);
    const float kf = -std::log(10000.0f) / s.d;
    for (int t = 0; t < rows; ++t)
      for (int i = 0; i < s.d; i += 2) {
        const float a = (float)t * std::exp((float)i * kf);
        hp[(size_t)t * s.d + i] = std::sin(a);
        hp[(size_t)t * s.d + i + 1] = std::cos(a);
      }
    cudaError_t e = cudaMalloc(&pe, hp.size() * 4);
    if (e != cudaSuccess) return e;
    pe_rows = rows;
    return cudaMemcpy(pe, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice);
  }

  cudaError_t gemm(int M, int N, int K, const __nv_bfloat16* A, const __nv_bfloat16* Bw,
                   int mode, const float* bias, float* of, __nv_bfloat16* ob, int ldo,
                   cudaStream_t st) {
    GemmDesc g;
    g.M = M; g.N = N; g.K = K; g.A = A; g.lda = K; g.B = Bw; g.ldb = K;
    g.mode = mode; g.bias = bias; g.out_f32 = of; g.out_bf16 = ob; g.ldo = ldo;
    return gemm_bf16(g, st);
  }
};

size_t dec_num_weights(const DecSpec& s) {
  const size_t d = s.d, ff = s.dff, V = s.vocab;
  size_t n = V * d;
  n += (size_t)s.layers * (2 * (2 * d + 4 * (d * d + d)) + 2 * d + ff * d + ff + d * ff + d);
  n += 2 * d + V * d + V;
  return n;
}

std::string dec_validate(const DecSpec& s) {
  if (s.d < 64 || s.d > 1024 || s.d % 64) return "decoder d_model must be a multiple of 64 in [64, 1024]";
  if (s.heads < 1 || s.d != s.heads * kDk) return "decoder heads must give a head width of 64";
  if (s.dff < 8 || s.dff % 8) return "decoder d_ff must be a positive multiple of 8";
  if (s.layers < 1) return "decoder layers must be >= 1";
  if (s.vocab < 2 || s.vocab % 4) return "decoder vocab must be >= 2 and a multiple of 4";
  return "";
}

cudaError_t dec_create(const DecSpec& s, const float* weights, DecoderNet** out) {
  auto* n = new DecoderNet;
  n->s = s;
  cudaError_t e = n->load(weights);
  if (e != cudaSuccess) {
    delete n;
    return e;
  }
  *out = n;
  return cudaSuccess;
}

void dec_destroy(DecoderNet* n) { delete n; }
const DecSpec& dec_spec(const DecoderNet* n) { return n->s; }
const double* dec_att(const DecoderNet* n) { return n->att; }
const float* dec_attf(const DecoderNet* n) { return n->attf; }
const float* dec_logits(const DecoderNet* n) { return n->logits; }
const double* dec_lse(const DecoderNet* n) { return n->lse; }
int dec_launches_per_step(const DecoderNet* n) {
  return 6 + 11 * n->s.layers + (n->lse_part ? 2 : 0) + (use_union_self_attn(n->B, n->S) ? 1 : 0);
}

cudaError_t dec_prepare(DecoderNet* n, int U, int B, int S, const __nv_bfloat16* memory, int T2,
                        cudaStream_t st) {
  const DecSpec& s = n->s;
  const size_t d = s.d, M = (size_t)U * B, Lc = s.layers;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t b_kvc = al(Lc * U * S * B * 2 * d * 2), b_kv2 = al(Lc * U * T2 * 2 * d * 2);
  const size_t need = b_kvc + b_kv2 + al(M * d * 4) + 3 * al(M * d * 2) + al(M * 3 * d * 2) +
                      al(M * s.dff * 2) + al(M * s.vocab * 4) +
                      (fused_log_softmax() ? al(M * ((s.vocab + 127) / 128) * 16) + al(M * 8)
                                           : al(M * s.vocab * 8) + al(M * 8)) +
                      al(M * s.vocab * 4) +
                      2 * al(M * S * 4) + 2 * al(M * 4) +
                      al((size_t)U * ((B * (size_t)S + 3) & ~(size_t)3) * 4) + al((size_t)U * 4);
  cudaError_t e;
  if (need > n->ws_bytes) {
    if (n->ws) cudaFree(n->ws);
    n->ws = nullptr;
    n->ws_bytes = 0;
    if ((e = cudaMalloc(&n->ws, need)) != cudaSuccess) return e;
    n->ws_bytes = need;
  }
  char* p = static_cast<char*>(n->ws);
  auto take = [&](size_t b) {
    char* r = p;
    p += al(b);
    return r;
  };
  n->kvc = reinterpret_cast<__nv_bfloat16*>(take(Lc * U * S * B * 2 * d * 2));
  n->kv2 = reinterpret_cast<__nv_bfloat16*>(take(Lc * U * T2 * 2 * d * 2));
  n->X = reinterpret_cast<float*>(take(M * d * 4));
  n->Y = reinterpret_cast<__nv_bfloat16*>(take(M * d * 2));
  n->AO = reinterpret_cast<__nv_bfloat16*>(take(M * d * 2));
  take(M * d * 2);  // spare
  n->QKV = reinterpret_cast<__nv_bfloat16*>(take(M * 3 * d * 2));
  n->H = reinterpret_cast<__nv_bfloat16*>(take(M * s.dff * 2));
  n->logits = reinterpret_cast<float*>(take(M * s.vocab * 4));
  n->lse_part = n->lse = nullptr;
  n->attf = nullptr;
  n->att = nullptr;
  n->lse_stride = 0;
  n->attf = reinterpret_cast<float*>(take(M * s.vocab * 4));
  if (fused_log_softmax()) {
    n->lse_stride = (s.vocab + 127) / 128;
    n->lse_part = reinterpret_cast<double*>(take(M * n->lse_stride * 16));
    n->lse = reinterpret_cast<double*>(take(M * 8));
  } else {
    if (rows_log_softmax()) n->att = reinterpret_cast<double*>(take(M * s.vocab * 8));
    else n->lse = reinterpret_cast<double*>(take(M * 8));
  }
  n->anc2[0] = reinterpret_cast<int*>(take(M * S * 4));
  n->anc2[1] = reinterpret_cast<int*>(take(M * S * 4));
  n->tok = reinterpret_cast<int*>(take(M * 4));
  n->gent = reinterpret_cast<uint32_t*>(take((size_t)U * ((B * (size_t)S + 3) & ~(size_t)3) * 4));
  n->gent_n = reinterpret_cast<int*>(take((size_t)U * 4));
  n->par = reinterpret_cast<int*>(take(M * 4));
  n->U = U; n->B = B; n->S = S; n->T2 = T2;
  if ((e = n->ensure_pe(S + 1)) != cudaSuccess) return e;
  // source-attention K|V of the memory, once per group
  for (int l = 0; l < s.layers; ++l) {
    if ((e = n->gemm(U * T2, 2 * s.d, s.d, memory, n->L[l].wkv2, kPlain, n->L[l].bkv2, nullptr,
                     n->kv2 + (size_t)l * U * T2 * 2 * d, 2 * s.d, st)) != cudaSuccess)
      return e;
  }
  if (use_union_self_attn(B, S)) {
    if ((e = cudaFuncSetAttribute(SELF_ATTN,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)su_smem(B, S))) != cudaSuccess)
      return e;
  } else {
    const size_t sa = (size_t)B * S * 8;
    if (sa > 227 * 1024) return cudaErrorInvalidValue;
    if ((e = cudaFuncSetAttribute(dec_self_attn_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa)) !=
        cudaSuccess)
      return e;
  }
  if (use_staged_cross_attn())
    return cudaFuncSetAttribute(SRC_ATTN,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs_smem());
  const size_t xm = xm_smem(T2);
  if (xm > 227 * 1024) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(dec_cross_attn_mma_kernel,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xm);
}

cudaError_t dec_step(DecoderNet* n, int l, const HistRec* hist, int hstride, const int* nb_live,
                     double lambda, cudaStream_t st) {
  const DecSpec& s = n->s;
  const int U = n->U, B = n->B, S = n->S, T2 = n->T2, d = s.d, M = U * B;
  if (l < 1 || l > S) return cudaErrorInvalidValue;
  cudaError_t e;
  dec_tok_kernel<<<(M + 127) / 128, 128, 0, st>>>(l, hist, hstride, U, B, s.vocab, n->tok,
                                                  n->par);
  int* anc = n->anc2[l & 1];
  const size_t na = (size_t)M * l;
  dec_anc_kernel<<<(unsigned)((na + 255) / 256), 256, 0, st>>>(l, U, B, S, n->par,
                                                               n->anc2[(l - 1) & 1], anc);
  if (use_union_self_attn(B, S))  // the self-attention entries of step l, once
    dec_union_kernel<4><<<U, 128, 0, st>>>(l, B, anc, S, nb_live, n->gent, n->gent_n);
  dec_embed_kernel<<<(M * 32 + 255) / 256, 256, 0, st>>>(n->tok, n->emb,
                                                         n->pe + (size_t)(l - 1) * d, d,
                                                         std::sqrt((float)d), n->X, M);
  const size_t sa = (size_t)B * S * 8;
  const size_t xm = xm_smem(T2);
  for (int li = 0; li < s.layers; ++li) {
    const DecLayer& y = n->L[li];
    layer_norm_bf16(d, n->X, M, y.ln1g, y.ln1b, n->Y, st);
    if ((e = n->gemm(M, 3 * d, d, n->Y, y.wqkv, kPlain, y.bqkv, nullptr, n->QKV, 3 * d, st)) !=
        cudaSuccess)
      return e;
    if (use_union_self_attn(B, S))
      SELF_ATTN<<<dim3(U, s.heads), kSuW * 32, su_smem(B, S), st>>>(
          l, n->QKV, d, B, anc, S, nb_live, n->kvc + (size_t)li * U * S * B * 2 * d, 0, n->AO,
          n->gent, n->gent_n);
    else
      dec_self_attn_kernel<<<dim3(U, s.heads), 32 * B, sa, st>>>(
          l, n->QKV, d, B, anc, S, nb_live, n->kvc + (size_t)li * U * S * B * 2 * d, n->AO);
    if ((e = n->gemm(M, d, d, n->AO, y.wo, kResidual, y.bo, n->X, nullptr, d, st)) != cudaSuccess)
      return e;
    layer_norm_bf16(d, n->X, M, y.ln2g, y.ln2b, n->Y, st);
    if ((e = n->gemm(M, d, d, n->Y, y.wq2, kPlain, y.bq2, nullptr, n->QKV, d, st)) != cudaSuccess)
      return e;
    if (use_staged_cross_attn())
      SRC_ATTN<<<dim3(U, s.heads, (B + 15) / 16), BL_XS_WARPS * 32, xs_smem(), st>>>(
          l, n->QKV, d, B, nullptr, 0, nb_live, n->kv2 + (size_t)li * U * T2 * 2 * d, T2, n->AO,
          nullptr, nullptr);
    else
      dec_cross_attn_mma_kernel<<<dim3(U, s.heads, (B + 15) / 16), kXW * 32, xm, st>>>(
          l, nb_live, n->QKV, n->kv2 + (size_t)li * U * T2 * 2 * d, T2, d, B, n->AO);
    if ((e = n->gemm(M, d, d, n->AO, y.wo2, kResidual, y.bo2, n->X, nullptr, d, st)) !=
        cudaSuccess)
      return e;
    layer_norm_bf16(d, n->X, M, y.ln3g, y.ln3b, n->Y, st);
    if ((e = n->gemm(M, s.dff, d, n->Y, y.w1, kRelu, y.b1, nullptr, n->H, s.dff, st)) !=
        cudaSuccess)
      return e;
    if ((e = n->gemm(M, d, s.dff, n->H, y.w2, kResidual, y.b2, n->X, nullptr, d, st)) !=
        cudaSuccess)
      return e;
  }
  layer_norm_bf16(d, n->X, M, n->ang, n->anb, n->Y, st);
  if (n->lse_part) {
    // log-softmax fused into the output GEMM: its epilogue leaves each row's
    // partial {max, sum exp} per 128-column slot; one thread per row folds
    // them into the fp64 log-normaliser. The search reads logit - lse.
    if ((e = cudaMemsetAsync(n->lse_part, 0, sizeof(double) * 2 * (size_t)M * n->lse_stride,
                             st)) != cudaSuccess)
      return e;
    GemmDesc g;
    g.M = M; g.N = s.vocab; g.K = d; g.A = n->Y; g.lda = d; g.B = n->wout; g.ldb = d;
    g.mode = kLsePart; g.bias = n->bout; g.out_f32 = n->logits; g.ldo = s.vocab;
    g.lse_part = n->lse_part; g.lse_stride = n->lse_stride;
    if ((e = gemm_bf16(g, st)) != cudaSuccess) return e;
    dec_lse_kernel<<<(M + 127) / 128, 128, 0, st>>>(n->lse_part, n->lse_stride, M, n->lse);
    dec_attf_kernel<<<M, 256, 0, st>>>(n->logits, n->lse, s.vocab, lambda, n->attf);
    return cudaGetLastError();
  }
  if ((e = n->gemm(M, s.vocab, d, n->Y, n->wout, kPlain, n->bout, n->logits, nullptr, s.vocab,
                   st)) != cudaSuccess)
    return e;
  if (!n->att && s.vocab % 4 == 0 && (size_t)4 * s.vocab * 4 <= 227 * 1024 &&
      std::getenv("BL_LOG_SOFTMAX") == nullptr) {
    const int sm = 4 * s.vocab * 4;
    if ((e = cudaFuncSetAttribute(dec_log_softmax64_staged_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, sm)) != cudaSuccess)
      return e;
    dec_log_softmax64_staged_kernel<<<(M + 3) / 4, 128, sm, st>>>(n->logits, s.vocab, M, lambda,
                                                                  n->attf, n->lse);
  } else if (use_warp_log_softmax() || !n->att)
    dec_log_softmax64_warp_kernel<<<(M + 7) / 8, 256, 0, st>>>(n->logits, s.vocab, M, lambda,
                                                               n->att, n->attf, n->lse);
  else
    dec_log_softmax64_kernel<<<M, 256, 0, st>>>(n->logits, s.vocab, lambda, n->att, n->attf);
  return cudaGetLastError();
}

}  // namespace bl
