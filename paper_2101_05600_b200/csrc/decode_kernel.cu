// decode_kernel.cu — persistent sm_100a decoder: one CTA per utterance runs
// the whole label-synchronous joint CTC/attention beam search (Alg. 2 of
// arXiv 2101.05600 as implemented by beamlattice batched_beam_search,
// /root/reference/proj/src/batched.cpp:94-237) with every step on device:
//
//   P1  windows + per-utterance envelope       ctc_prefix.cpp:106-125, batched.cpp:129-135
//   P2  phi_j[t] = gb[t-1] (+) gn[t-1]  (fp64)  ctc_prefix.cpp:50-51
//       + per-parent max and fp32 factors (one half-warp per parent)
//   P3  K1 bulk prefix score, all (j, c):       ctc_prefix.cpp:47-59 (psi term)
//       psi ~= M_j + m_c + log sum_t exp(phi_j-M_j) exp(L[t,c]-m_c)  (fp32 FMA)
//       -> certified fp32 joint keys            beam_search.cpp:60-66, logmath.hpp:34-39
//   P4  theta = B-th largest certified lower bound
//   P5  contenders = candidates whose upper bound reaches theta (+ repeats)
//   P6  contenders: psi by a parallel fp64 log-sum-exp (score), and the
//       serial reference-order gamma_n'/gamma_b' chains (one warp) that
//       yield their child state (gamma, tau, tau~); a spare warp computes
//       the eos candidates (exact fp64, ctc_prefix.cpp:88-104 via tail tables)
//   P7  exact total order (score desc, parent asc, token asc) incl. eos
//                                               batched.cpp:172-186
//   P8  walk: finished entries / children       batched.cpp:188-212
//   P9  end detection                           batched.cpp:215-228
//       P7-P9 run on the non-chain warps (named barrier) while the chains
//       finish; the children's tau is patched in after the join
//   fin finalize + n-best                       batched.cpp:70-90
//
// If the contender set overflows (degenerate ties) or exact mode is on, the
// step falls back to fp64 scores for every candidate and an exact block
// arg-max selection — slower, same results.
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "decode.cuh"
#include "softplus.cuh"

namespace bl {
namespace {  // device helpers: internal to each mode's translation unit

// ---------------------------------------------------------------- logmath
__device__ __forceinline__ bool is_zero(double x) { return x <= kLogZeroGuard; }

__constant__ SpTables c_sptab = {SP_THI_INIT, SP_TLO_INIT, SP_INV_INIT, SP_LH_INIT,
                                 SP_LL_INIT};

// logmath.hpp:19-23 — branch-free table-driven version (softplus.cuh); the
// tables live in shared memory (`tb`).
__device__ __forceinline__ double log_add(double a, double b, const SpTables& tb) {
  return log_add_fast(a, b, tb);
}

// logmath.hpp:26-29
__device__ __forceinline__ double log_mul(double a, double b) {
  if (is_zero(a) || is_zero(b)) return kLogZero;
  return __dadd_rn(a, b);
}

// logmath.hpp:34-39 (no FMA contraction: same rounding as the host)
__device__ __forceinline__ double mix_joint(double lam, double ctc, double att) {
  if (lam <= 0.0) return att;
  if (lam >= 1.0) return ctc;
  if (is_zero(ctc) || is_zero(att)) return kLogZero;
  return __dadd_rn(__dmul_rn(lam, ctc), __dmul_rn(__dsub_rn(1.0, lam), att));
}

// candidate order, batched.cpp:181-186 (eos carries token id |C|)
__device__ __forceinline__ bool before(double sa, int pa, int ta, double sb,
                                       int pb, int tb) {
  if (sa != sb) return sa > sb;
  if (pa != pb) return pa < pb;
  return ta < tb;
}

// window_for, ctc_prefix.cpp:106-114
__device__ __forceinline__ void window_for(int tau, int taut, int m1, int m2,
                                           int step, int T, int* s, int* e) {
  long long ss = (long long)tau - m1;
  if ((long long)step > ss) ss = step;
  if (ss < 1) ss = 1;
  long long ee = (long long)taut + m2;
  if ((long long)T < ee) ee = T;
  if (ss > ee) ss = ee;
  *s = (int)ss;
  *e = (int)ee;
}

__device__ __forceinline__ double gread(const double* a, int i, int vlo, int cov) {
  return (i < vlo || i > cov) ? kLogZero : a[i];
}

// scorer rows: the table (Uniform / Table / Loop rows), or for the network
// scorer the output GEMM's fp32 logits and the row's fp64 log-normaliser:
// att = (double)logit - lse, attf = (float)((1 - lambda) att) -- the values
// materialised rows would hold. The fp32 attf rows (every key reads one) are
// always materialised (by the log-softmax kernel, or after the fused GEMM
// epilogue's normaliser): a branch here cost the vocab-500 kernel 4%.
__device__ __forceinline__ double att_at(const KParams& P, int row, int c) {
  if (P.net_lse) return (double)P.net_logits[(size_t)row * P.V + c] - P.net_lse[row];
  return P.sc_rows[(size_t)row * P.V + c];
}
__device__ __forceinline__ float attf_at(const KParams& P, int row, int c) {
  return P.sc_rowsf[(size_t)row * P.V + c];
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

constexpr float kZeroKey = -3.0e38f;  // key of a joint that is exactly kLogZero

// order-preserving float <-> int map (shared-memory atomicMax on floats)
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// k-th largest (0-based) of the 32 lanes' values: bitonic sort, descending
// (whole warp)
__device__ __forceinline__ float warp_kth_desc(float v, int k, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const float o = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool desc = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      v = (lower == desc) ? fmaxf(v, o) : fminf(v, o);
    }
  }
  return __shfl_sync(0xffffffffu, v, k);
}

// ------------------------------------------------------- TMA / mbarrier PTX
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Barrier over the step's decision group, warps [gw0, kNWarp): the whole
// block when gw0 == 0, else named barrier 1 (the serial-chain warps run on).
__device__ __forceinline__ void group_sync(int gw0) {
  if (gw0 == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync 1, %0;" ::"r"((kNWarp - gw0) * 32) : "memory");
  }
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// wait with a suspend-time hint: a warp waiting for its stage's data sleeps
// in the barrier unit instead of re-issuing try_wait (the spin loop was ~8%
// of the streaming loop's instructions; the other CTA on the SM gets the
// issue slots)
__device__ __forceinline__ void mbar_wait_sleep_s(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WS_%=;\n}" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// bounded wait (tensor-core variant): a barrier that never completes reports
// where and traps instead of hanging the device
__device__ __noinline__ void mbar_wait_dbg(unsigned long long* bar, unsigned parity, int tag,
                                           unsigned g) {
  const long long t0 = clock64();
  for (;;) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    if (clock64() - t0 > (1ll << 33)) {
      printf("[bl] decode_kernel: barrier wait timed out: cta %d thread %d tag %d job %u parity %u\n",
             blockIdx.x, threadIdx.x, tag, g, parity);
      asm volatile("trap;");
    }
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// 3D box {32 columns, 8 rows, 16 column blocks} (tensor-core variant)
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y,
                                            int z, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptors (sm_100 layout: start>>4 @0, LBO>>4 @16,
// SBO>>4 @32, version 1 @46, layout type @61)
__device__ __forceinline__ unsigned long long umma_desc_mn32(const void* p) {
  // MN-major, 128-byte swizzle with 32-byte atoms (type 1): 32 tf32 of MN per
  // 128 B row, 4 K rows per 512 B atom; MN atoms 1024 B apart (LBO), K
  // 4-row groups 512 B apart (SBO) -- the TMA stage as loaded
  return (unsigned long long)((smem_u32(p) & 0x3FFFF) >> 4) | (64ull << 16) | (32ull << 32) |
         (1ull << 46) | (1ull << 61);
}
__device__ __forceinline__ unsigned long long umma_desc_kint(const void* p) {
  // K-major, no swizzle: 8-row x 16-byte core matrices, K chunks 128 B apart
  // (LBO), 8-row N groups 256 B apart (SBO)
  return (unsigned long long)((smem_u32(p) & 0x3FFFF) >> 4) | (8ull << 16) | (16ull << 32) |
         (1ull << 46);
}
// D[128 x 16] (+)= A[128 x 8] . B[8 x 16], tf32 inputs, fp32 accumulate in TMEM;
// idesc: F32 accumulator @4, A/B TF32 @7/@10, A MN-major @15, N/8 @17, M/16 @24
constexpr unsigned kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                              ((16u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ void umma_tf32(unsigned tmem, unsigned long long da,
                                          unsigned long long db, unsigned acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(acc), "r"(kTcIdesc));
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
constexpr int kTcTmemCols = 128;  // two 64-column accumulator buffers (4 subtiles x 16)

struct SelE {
  double score;
  int parent, token, slot, tau, taut, pad;
};

struct Item {  // contender or eos candidate (kItemBytes)
  double score;
  int parent, token, tau, taut;
};
static_assert(sizeof(Item) == kItemBytes, "Item layout");

template <int BMAX>
struct Shared {
  int b_area[2][BMAX], b_slot[2][BMAX], b_vlo[2][BMAX], b_cov[2][BMAX];
  int b_tau[2][BMAX], b_taut[2][BMAX], b_last[2][BMAX], b_row[2][BMAX];
  double b_att[2][BMAX], b_joint[2][BMAX];
  double M[BMAX];
  float kb[BMAX];
  int mzero[BMAX];
  float wl[kNWarp][BMAX];
  SelE sel[2 * BMAX + 2];
  double red_s[kNWarp];
  int red_p[kNWarp], red_t[kNWarp];
  int s, e, W, nb, n_cont, nsel, nchild, n_fin, n_fin_new, count_long, best_fin;
  int done, trigger, steps, fallback;
  int row_same;  // scorer row shared by every live parent, or -1
  int child_q[BMAX];  // contender index of each child (deferred tau fix-up)
  double best_all, best_fin_val, off;
  float theta, theta2;
  int n_list;
  int th_run, n_raw;  // filter mode: running bound (f2ord) and raw-list size
  // c_fallback: full fallback steps in the low 32 bits, wide steps in the high 32
  unsigned long long c_queries, c_frames, c_k1, c_fallback, c_cont, c_steps, c_raw;
};

__device__ __forceinline__ double* gam_ptr(const KParams& P, int u, int area,
                                           int slot, int which) {
  return P.gam + ((((size_t)u * 2 + area) * P.caps + slot) * 2 + which) * (size_t)P.Tp;
}

// TableScorer::score context lookup (scorer.cpp:53-62): the last
// min(len, order-1) tokens of the prefix; entries are sorted by
// (length, tokens) on the host. Row 0 is the uniform fallback.
__device__ int lookup_row(const KParams& P, const HistRec* hist_u, int len,
                          int parent_step, int parent_slot, int c) {
  if (P.sc_nent == 0) return 0;
  int n = len < P.sc_order - 1 ? len : P.sc_order - 1;
  int ctx[8];
  if (n > 0) {
    ctx[n - 1] = c;
    int k = parent_slot;
    for (int i = n - 2, st = parent_step; i >= 0; --i, --st) {
      HistRec h = hist_u[(size_t)st * P.B + k];
      ctx[i] = h.token;
      k = h.parent;
    }
  }
  int lo = 0, hi = P.sc_nent - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int ml = P.sc_ctx_len[mid];
    int cmp = 0;
    if (ml != n) {
      cmp = ml < n ? -1 : 1;
    } else {
      const int* mc = P.sc_ctx + (size_t)mid * P.sc_w;
      for (int i = 0; i < n; ++i)
        if (mc[i] != ctx[i]) {
          cmp = mc[i] < ctx[i] ? -1 : 1;
          break;
        }
    }
    if (cmp == 0) return P.sc_row[mid];
    if (cmp < 0) lo = mid + 1;
    else hi = mid - 1;
  }
  return 0;
}

// Reference-order child recursion (ctc_prefix.cpp:47-77) over [s, s+W-1]
// from shared-memory inputs: ph[i] = phi(t = s+i), lc[i] = L[t, c],
// lb[i] = L[t, blank]. Writes gamma_n'/gamma_b' for t in the window and
// returns psi, tau, tau~ (tau scan from lo = max(1, tau_parent)).
__device__ double child_recursion_smem(const double* ph, const float* lc,
                                       const float* lb, int s, int W, int tau_p,
                                       double* gnc, double* gbc, int* tau_out,
                                       int* taut_out, const SpTables& tb) {
  const int lo = tau_p > 1 ? tau_p : 1;
  int best_n = lo, best_b = lo;
  double val_n = kLogZero, val_b = kLogZero;
  double gn_prev = kLogZero, gb_prev = kLogZero, psi = kLogZero;
  for (int i = 0; i < W; ++i) {
    const int t = s + i;
    const double phv = ph[i];
    const double pc = (double)lc[i];
    const double pbl = (double)lb[i];
    const double gn = log_mul(log_add(gn_prev, phv, tb), pc);
    const double gb = log_mul(log_add(gb_prev, gn_prev, tb), pbl);
    psi = log_add(psi, log_mul(phv, pc), tb);
    gnc[t] = gn;
    gbc[t] = gb;
    if (t >= lo) {
      if (gn > val_n) {
        val_n = gn;
        best_n = t;
      }
      if (gb > val_b) {
        val_b = gb;
        best_b = t;
      }
    }
    gn_prev = gn;
    gb_prev = gb;
  }
  *tau_out = best_n;
  *taut_out = best_b;
  return psi;
}

// The same recursion with two lanes per contender: the even lane runs the
// gamma_n' chain, the odd lane the gamma_b' chain, which takes the partner's
// previous gamma_n' by a shuffle. Each frame then costs one log_add per lane
// instead of two interleaved ones; the operations per value are the
// reference's (ctc_prefix.cpp:47-57), so the results are bit-identical.
// Called by whole warps (the shuffle); `live` lanes store.
__device__ void child_state_lanes(const double* ph, const float* lc, const float* lb, int s,
                                  int W, int tau_p, double* gout, int role, bool live,
                                  int* best_out, const SpTables& tb) {
  const int lo = tau_p > 1 ? tau_p : 1;
  int best = lo;
  double val = kLogZero, g_prev = kLogZero;
  // branch-free roles: both lanes load ph[i] (valid for either), each its own
  // x column; the store walks a pointer
  const float* xs = role == 0 ? lc : lb;
  double* gp = gout + s;
  for (int i = 0; i < W; ++i) {
    const int t = s + i;
    const double gn_partner = __shfl_xor_sync(0xffffffffu, g_prev, 1);
    const double phv = ph[i];
    const double b = role == 0 ? phv : gn_partner;
    const double x = (double)xs[i];
    const double g = log_mul(log_add(g_prev, b, tb), x);
    if (live) gp[i] = g;
    if (t >= lo && g > val) {
      val = g;
      best = t;
    }
    g_prev = g;
  }
  *best_out = best;
}

// Same recursion reading the grid and the parent from global memory
// (fallback path).
template <int BMAX>
__device__ double child_recursion_global(const KParams& P, const Shared<BMAX>& sh,
                                       int u, int cur, int j, int c, int s, int e,
                                       const float* __restrict__ grid,
                                       const double* phi, double* gnc, double* gbc,
                                       int* tau_out, int* taut_out, const SpTables& tb) {
  const int V = P.V, blank = P.V - 1;
  const int vlo = sh.b_vlo[cur][j], cov = sh.b_cov[cur][j];
  const double* gbp = gam_ptr(P, u, sh.b_area[cur][j], sh.b_slot[cur][j], 1);
  const bool repeat = sh.b_last[cur][j] == c;
  const int lo = sh.b_tau[cur][j] > 1 ? sh.b_tau[cur][j] : 1;
  int best_n = lo, best_b = lo;
  double val_n = kLogZero, val_b = kLogZero;
  double gn_prev = kLogZero, gb_prev = kLogZero, psi = kLogZero;
  for (int t = s; t <= e; ++t) {
    const double ph = repeat ? gread(gbp, t - 1, vlo, cov) : phi[t - s];
    const float* row = grid + (size_t)(t - 1) * V;
    const double pc = (double)row[c];
    const double gn = log_mul(log_add(gn_prev, ph, tb), pc);
    const double gb = log_mul(log_add(gb_prev, gn_prev, tb), (double)row[blank]);
    psi = log_add(psi, log_mul(ph, pc), tb);
    gnc[t] = gn;
    gbc[t] = gb;
    if (t >= lo) {
      if (gn > val_n) {
        val_n = gn;
        best_n = t;
      }
      if (gb > val_b) {
        val_b = gb;
        best_b = t;
      }
    }
    gn_prev = gn;
    gb_prev = gb;
  }
  *tau_out = best_n;
  *taut_out = best_b;
  return psi;
}

// psi only (fallback path), same order as the reference.
template <int BMAX>
__device__ double psi_only(const KParams& P, const Shared<BMAX>& sh, int u,
                           int cur, int j, int c, int s, int e,
                           const float* __restrict__ grid, const double* phi,
                           const SpTables& tb) {
  const int V = P.V;
  const int vlo = sh.b_vlo[cur][j], cov = sh.b_cov[cur][j];
  const double* gbp = gam_ptr(P, u, sh.b_area[cur][j], sh.b_slot[cur][j], 1);
  const bool repeat = sh.b_last[cur][j] == c;
  double psi = kLogZero;
  for (int t = s; t <= e; ++t) {
    const double ph = repeat ? gread(gbp, t - 1, vlo, cov) : phi[t - s];
    psi = log_add(psi, log_mul(ph, (double)grid[(size_t)(t - 1) * V + c]), tb);
  }
  return psi;
}

// Optional per-phase cycle accounting (P.prof != nullptr): thread 0 reads
// clock64 right after each block barrier, so each delta is a phase's span.
#define PROF_MARK(k)                                   \
  if (P.prof && tid == 0) {                            \
    const long long _now = clock64();                  \
    P.prof[(size_t)u * 16 + (k)] += _now - prof_t;     \
    prof_t = _now;                                     \
  }

#ifndef BL_PROF_WAIT
#define PROF_SERIAL(t0) \
  if (P.prof && tid == 0) P.prof[(size_t)u * 16 + 14] += clock64() - (t0);
#else
#define PROF_SERIAL(t0)
#endif

}  // namespace

// kMode 0: K1 slab by __ldg, every upper key in shared memory (keys mode);
// 1: __ldg, keys filtered on chip (filter mode); 2: TMA slab, filter mode;
// 3: TMA slab + tcgen05.mma tf32 bulk; 4: TMA slab + mma.sync tf32 bulk
template <int BMAX, int kMode>
__global__ void __launch_bounds__(kNT, (BMAX <= 12 && kMode == 0 ? 3 : 2))
    decode_kernel(const __grid_constant__ KParams P) {
  constexpr bool kTma = kMode >= 2;
  constexpr bool kTc = kMode == 3;   // K1 bulk on tcgen05.mma (kind::tf32), accumulators in TMEM
  constexpr bool kMma = kMode == 4;  // K1 bulk on mma.sync m16n8k8 tf32, accumulators in registers
  constexpr bool kShift = kTc || kMma;  // fixed per-step column shifts (no lazy rescale)
  constexpr bool keys_mode = kMode == 0;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ Shared<BMAX> sh;
  __shared__ SpTables tb;
  __shared__ __align__(8) unsigned long long mbar[kTmaStagesMax];
  __shared__ int cons[kTmaStagesMax];  // warps done with each TMA stage (monotonic)
  // slab streaming (kMode 2): one ring per warp, barrier (stage, warp) at st * kNWarp + warp
  __shared__ __align__(8) unsigned long long mbarw[kMode == 2 ? kTmaStagesMax * kNWarp : 1];
  __shared__ __align__(8) unsigned long long mmad[kTmaStagesMax];  // tensor cores: stage's MMAs done
  __shared__ unsigned tmem_base;

  const int u = blockIdx.x + P.u0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const UttDesc ud = P.utts[u];
  const float* __restrict__ grid = ud.grid;
  const int T = ud.T, V = P.V, C = P.C, B = P.B, blank = P.V - 1;
  const double lam = P.lambda;
  const float lamf = (float)lam;
  long long prof_t = clock64();

  // dynamic smem carve-up (smem_plan, decode.cuh)
  const SmemPlan pl = smem_plan(P.Tmax, B, BMAX, C, P.caps, P.S, P.region_bytes, P.kub_smem,
                                kTma ? P.tma_stages : 0, kTc ? 1 : kMma ? 2 : 0);
  double* phi = reinterpret_cast<double*>(dsm + pl.phi);    // [B][Tmax]
  unsigned char* region = dsm + pl.region;                  // aliased, region_bytes
  float* PhiF = reinterpret_cast<float*>(region + pl.phif);  // [Tmax][BMAX]
  // keys mode (kub_smem): every upper key and its underflow flag in shared
  // memory, scanned by P5; filter mode: keys reaching the running bound go
  // to the raw list as P3 emits them
  float* kub = reinterpret_cast<float*>(region + pl.kub);          // [B][C]
  const int ub_words = (B * C + 31) >> 5;
  unsigned* ubits = reinterpret_cast<unsigned*>(region + pl.ubits);  // underflow-key flags
  float4* clist = reinterpret_cast<float4*>(region + pl.clist);    // [kListCap]
  uint2* rawl = reinterpret_cast<uint2*>(region + pl.raw);         // [kRawCap] {ku, under|q|c}
  const int caps = P.caps;
  Item* items = reinterpret_cast<Item*>(dsm + pl.items);     // [caps + BMAX], eos at caps
  double* best_by_len = reinterpret_cast<double*>(dsm + pl.bbl);    // [S+2]

  const HistRec* hist_c = P.hist + (size_t)u * (P.S + 1) * B;
  HistRec* hist_u = P.hist + (size_t)u * (P.S + 1) * B;
  FinEntry* fin_u = P.fin + (size_t)u * B * P.S;
  double* Ft = P.Ftab + (size_t)u * P.Tp * C;
  double* Gt = P.Gtab + (size_t)u * P.Tp;

  // ---------------------------------------------------------------- init
  unsigned tma_jobs = 0;  // TMA jobs issued so far (stage = job % stages, parity = job / stages)
  const bool stepm = P.step_l > 0;
  unsigned char* st_u = stepm ? P.state + (size_t)u * P.state_stride : nullptr;
  if (stepm && P.step_l > 1 && *reinterpret_cast<volatile int*>(st_u)) return;  // finished
  if (kTma && tid == 0) {
    for (int k = 0; k < P.tma_stages; ++k) {
      mbar_init(&mbar[k], 1);
      if (kTc) mbar_init(&mmad[k], 1);
      cons[k] = 0;
    }
    if (kMode == 2)
      for (int k = 0; k < P.tma_stages * kNWarp; ++k) mbar_init(&mbarw[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (kTc && warp == 0) {  // accumulators: 2 x (4 subtiles x 16 parents) fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // the tensor-core stage ring starts on a 1024-byte boundary (swizzle atoms)
  unsigned char* tc_stg = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(region + pl.stages - 1024) + 1023) & ~(uintptr_t)1023);
  auto tmem_free = [&]() {
    if constexpr (kTc) {
      tc_before_sync();
      __syncthreads();
      if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(kTcTmemCols));
    }
  };
  for (int i = tid; i < 320; i += kNT)
    reinterpret_cast<double*>(&tb)[i] = reinterpret_cast<const double*>(&c_sptab)[i];
  if (P.ready) {
    // streamed host input: wait for this utterance's copy chunk (acquire;
    // chunk boundaries are 128-byte aligned, so no line of this grid was
    // cached by a CTA of an earlier chunk)
    if (tid == 0) {
      const unsigned* f = P.ready + ud.chunk;
      const long long t0 = clock64();
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v == P.ready_epoch) break;
        if (clock64() - t0 > (1ll << 36)) {  // ~35 s: the copy never landed
          atomicExch(P.stream_err, 1);
          break;
        }
        __nanosleep(1000);
      }
      // the K1 slab of the TMA variant is read by the async proxy
      // (cp.async.bulk.tensor, issued by this thread): order those reads
      // after the generic-proxy acquire of the ready flag
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
  }
  if (stepm && P.step_l > 1) {
    // resume: the search state saved at the end of step l-1
    const int* src = reinterpret_cast<const int*>(st_u + 16);
    int* dst = reinterpret_cast<int*>(&sh);
    for (int i = tid; i < (int)(sizeof(Shared<BMAX>) / 4); i += kNT) dst[i] = src[i];
    const double* sb = reinterpret_cast<const double*>(st_u + 16 + align16(sizeof(Shared<BMAX>)));
    for (int i = tid; i <= P.S + 1; i += kNT) best_by_len[i] = sb[i];
    __syncthreads();
  } else {
  for (int i = tid; i <= P.S + 1; i += kNT) best_by_len[i] = -HUGE_VAL;
  {
    double* gn0 = gam_ptr(P, u, 0, 0, 0);
    for (int t = tid; t <= T; t += kNT) gn0[t] = kLogZero;
  }
  // the blank column, staged once so the two serial scans below read shared
  // memory instead of chasing T dependent global loads
  float* bcol = reinterpret_cast<float*>(region);                       // [T]
  double* Gs = reinterpret_cast<double*>(region + align16(sizeof(float) * (size_t)T));  // [T+1]
  for (int t = tid; t < T; t += kNT) bcol[t] = grid[(size_t)t * V + blank];
  __syncthreads();
  if (tid == 0) {
    // init_state, ctc_prefix.cpp:10-26 (sequential: exact reference order)
    double* gb0 = gam_ptr(P, u, 0, 0, 1);
    double acc = 0.0;
    gb0[0] = acc;
    for (int t = 1; t <= T; ++t) {
      acc = log_mul(acc, (double)bcol[t - 1]);
      gb0[t] = acc;
    }
    if (ud.need_tail) {  // G[k] = blank mass of frames k+1..T
      double g = 0.0;
      Gs[T] = g;
      for (int k = T - 1; k >= 0; --k) {
        g = log_mul((double)bcol[k], g);
        Gs[k] = g;
      }
    }
    sh.nb = 1;
    sh.b_area[0][0] = 0;
    sh.b_slot[0][0] = 0;
    sh.b_vlo[0][0] = 0;
    sh.b_cov[0][0] = T;
    sh.b_tau[0][0] = 1;
    sh.b_taut[0][0] = 1;
    sh.b_last[0][0] = -1;
    sh.b_att[0][0] = 0.0;
    sh.b_joint[0][0] = 0.0;
    sh.n_fin = 0;
    sh.count_long = 0;
    sh.best_fin = -1;
    sh.best_fin_val = 0.0;
    sh.best_all = -HUGE_VAL;
    sh.done = 0;
    sh.trigger = 2;
    sh.steps = 0;
    sh.c_queries = sh.c_frames = sh.c_k1 = sh.c_fallback = sh.c_cont = sh.c_steps = 0;
    sh.c_raw = 0;
    sh.b_row[0][0] = P.net_rows ? u * B : lookup_row(P, hist_c, 0, 0, 0, 0);
  }
  __syncthreads();
#ifdef BL_PROF_WAIT
  if (P.prof && tid == 0) P.prof[(size_t)u * 16 + 14] += clock64() - prof_t;
#endif
  if (ud.need_tail) {
    // F[k][c]: label c held from frame k to some k' then blank to T
    // (the eos tail of ctc_prefix.cpp:88-104 in closed form).
    for (int t = tid; t <= T; t += kNT) Gt[t] = Gs[t];
    // two columns per pass, their serial chains interleaved (log_add2)
    for (int c0 = tid; c0 < C; c0 += 2 * kNT) {
      const int c1 = c0 + kNT;
      const bool two = c1 < C;
      const int c1r = two ? c1 : c0;
      double f0 = 0.0, f1 = 0.0;
      Ft[(size_t)T * C + c0] = f0;
      if (two) Ft[(size_t)T * C + c1] = f1;
      for (int k = T - 1; k >= 0; --k) {
        const double g = Gs[k];
        log_add2(log_mul((double)grid[(size_t)k * V + c0], f0), g,
                 log_mul((double)grid[(size_t)k * V + c1r], f1), g, tb, &f0, &f1);
        Ft[(size_t)k * C + c0] = f0;
        if (two) Ft[(size_t)k * C + c1] = f1;
      }
    }
  }
  if constexpr (kShift) {
    // The step-1 exp shift of every column: its max over all T frames (the
    // step-1 window is [1, T]); each later step takes the max over the rows
    // the next window can still reach while it streams its own (P3).
    const int nch = (T + 7) >> 3, ntile = (C + 511) >> 9, J = ntile * nch;
    const int NST = P.tma_stages;
    float* msh1 = P.mshift + ((size_t)1 * P.U + u) * P.mshift_stride;  // step 1's parity
    auto issue0 = [&](int j, unsigned g) {
      const int st = (int)(g % (unsigned)NST), tile = j / nch, k = j - tile * nch;
      mbar_expect_tx(&mbar[st], kTmaStageBytes);
      tma_load_3d(tc_stg + (size_t)st * kTmaStageBytes, &P.tmap, 0, ud.row0 + k * 8, tile * 16,
                  &mbar[st]);
    };
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int j = 0; j < NST && j < J; ++j) issue0(j, tma_jobs + j);
    }
    const int tbk = tid >> 4, gq = tid & 7, rg = (tid >> 3) & 1;
    const float gfl = P.guard_f;
    float4 mx = make_float4(gfl, gfl, gfl, gfl);
    for (int j = 0; j < J; ++j) {
      const unsigned g = tma_jobs + j;
      const int st = (int)(g % (unsigned)NST), tile = j / nch, k = j - tile * nch;
      if (k == 0) mx = make_float4(gfl, gfl, gfl, gfl);
      mbar_wait_dbg(&mbar[st], (g / (unsigned)NST) & 1u, 1, g);
      const float* sb =
          reinterpret_cast<const float*>(tc_stg + (size_t)st * kTmaStageBytes) + tbk * 256;
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int r = rg + 2 * rr;
        if (8 * k + r < T) {
          // 16-byte chunk gq of row r: 32-byte-atom swizzle (tcgen05) or the
          // standard 128-byte swizzle (mma.sync)
          const int ph = kTc ? ((((gq >> 1) ^ r) & 3) << 3) | ((gq & 1) << 2)
                             : ((gq ^ r) & 7) << 2;
          const float4 x = *reinterpret_cast<const float4*>(sb + r * 32 + ph);
          mx.x = fmaxf(mx.x, x.x);
          mx.y = fmaxf(mx.y, x.y);
          mx.z = fmaxf(mx.z, x.z);
          mx.w = fmaxf(mx.w, x.w);
        }
      }
      __syncthreads();  // stage consumed (one-time pass: a block barrier is fine)
      if (tid == 0) {
        // keep the per-stage use counts of P3 in step: the release count and
        // the MMA-done barrier's phase (no MMA ran on this use)
        cons[st] += kNWarp;
        if (kTc)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mmad[st]))
                       : "memory");
        if (j + NST < J) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue0(j + NST, g + NST);
        }
      }
      if (k == nch - 1) {
        mx.x = fmaxf(mx.x, __shfl_xor_sync(0xffffffffu, mx.x, 8));
        mx.y = fmaxf(mx.y, __shfl_xor_sync(0xffffffffu, mx.y, 8));
        mx.z = fmaxf(mx.z, __shfl_xor_sync(0xffffffffu, mx.z, 8));
        mx.w = fmaxf(mx.w, __shfl_xor_sync(0xffffffffu, mx.w, 8));
        if (rg == 0)
          *reinterpret_cast<float4*>(msh1 + tile * 512 + tbk * 32 + gq * 4) = mx;
      }
    }
    tma_jobs += J;
  }
  __syncthreads();
#ifdef BL_PROF_WAIT
  if (P.prof && tid == 0) P.prof[(size_t)u * 16 + 15] += clock64() - prof_t;
#endif
  }  // fresh start
  PROF_MARK(0);

  // ---------------------------------------------------------- step loop
  for (int l = stepm ? P.step_l : 1;; ++l) {
    const int cur = (l - 1) & 1, nxt = l & 1;
    if (l > ud.max_steps) {  // batched.cpp:125-128
      if (P.nb_out && tid == 0) P.nb_out[u] = 0;
      break;
    }
    const int nb = sh.nb;

    // ---- P1: windows and offsets (warp 0). The eos candidates (two fp64
    // log_adds per hypothesis) are only read by P7: they are computed by a
    // spare warp during P6 (eos_items below), off the critical path. ----
    if (warp == 0) {
      const int j = lane;
      int ws = INT_MAX, we = INT_MIN;
      double jm = -HUGE_VAL;
      unsigned long long tail = 0;
      if (j < nb) {
        window_for(sh.b_tau[cur][j], sh.b_taut[cur][j], P.m1, P.m2, l, T, &ws, &we);
        const int cov = sh.b_cov[cur][j];
        if (cov < T) tail = (unsigned long long)(T - cov);
        jm = sh.b_joint[cur][j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ws = min(ws, __shfl_xor_sync(0xffffffffu, ws, o));
        we = max(we, __shfl_xor_sync(0xffffffffu, we, o));
        tail += __shfl_xor_sync(0xffffffffu, tail, o);
      }
      jm = warp_max_d(jm);
      const int r0 = sh.b_row[cur][0];
      const bool same = __all_sync(0xffffffffu, j >= nb || sh.b_row[cur][j] == r0);
      if (lane == 0) {
        if (P.rec_nb) P.rec_nb[(size_t)u * (P.S + 2) + l] = nb;
        sh.row_same = same ? r0 : -1;
        sh.s = ws;
        sh.e = we;
        const int W = we - ws + 1;
        sh.W = W;
        sh.off = is_zero(jm) ? 0.0 : jm;
        sh.c_queries += nb;
        sh.c_frames += (unsigned long long)nb * C * W + tail;
        sh.c_k1 += 4ull * V * W + 16ull * nb * (W + 1) + 4ull * nb * V;
        sh.n_cont = 0;
        sh.fallback = P.exact;
        sh.th_run = f2ord(-INFINITY);
        sh.n_raw = 0;
      }
    }
    __syncthreads();
    PROF_MARK(1);
    const int s = sh.s, e = sh.e, W = sh.W;
    // eos candidates of the beam (eos_score_extended, ctc_prefix.cpp:88-104,
    // via the tail tables), one lane per hypothesis
    auto eos_items = [&]() {
      const int j = lane;
      if (j < nb) {
        const int cov = sh.b_cov[cur][j];
        const double* gnp = gam_ptr(P, u, sh.b_area[cur][j], sh.b_slot[cur][j], 0);
        const double* gbp = gnp + P.Tp;
        double ee;
        if (cov >= T) {
          ee = log_add(gnp[T], gbp[T], tb);
        } else {
          const int last = sh.b_last[cur][j];
          const double fl = last >= 0 ? Ft[(size_t)cov * C + last] : Gt[cov];
          ee = log_add(log_mul(gnp[cov], fl), log_mul(gbp[cov], Gt[cov]), tb);
        }
        Item it;
        it.score = mix_joint(lam, ee, __dadd_rn(sh.b_att[cur][j], att_at(P, sh.b_row[cur][j], C)));
        it.parent = j;
        it.token = C;
        it.tau = it.taut = 0;
        items[caps + j] = it;  // eos candidates live past the contender slots
      }
    };

    // ---- P2: phi_j[t] (fp64, reference log_add), the per-parent max M_j
    // and the fp32 factors in one pass: a half-warp per parent (16 parents
    // per pass), the max by half-warp shuffles, one block barrier ----
    {
      const int hl = lane & 15;  // lane within the half-warp
      for (int jb = 2 * warp; jb < nb; jb += kNT / 16) {  // warp-uniform
        const int j = jb + (lane >> 4);
        const bool act = j < nb;
        double m = -HUGE_VAL;
        if (act) {
          const int vlo = sh.b_vlo[cur][j], cov = sh.b_cov[cur][j];
          const double* gnp = gam_ptr(P, u, sh.b_area[cur][j], sh.b_slot[cur][j], 0);
          const double* gbp = gnp + P.Tp;
          for (int i = hl; i < W; i += 16) {
            const int t = s + i;
            const double v =
                log_add(gread(gbp, t - 1, vlo, cov), gread(gnp, t - 1, vlo, cov), tb);
            phi[(size_t)j * P.Tmax + i] = v;
            if (!is_zero(v) && v > m) m = v;
          }
        }
        if (!P.exact) {
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
          const double Mj = (m == -HUGE_VAL) ? kLogZero : m;
          if (act && hl == 0) {
            sh.M[j] = Mj;
            sh.mzero[j] = is_zero(Mj) ? 1 : 0;
            // per-parent float base of the joint key, relative to `off`
            const double base = (lam >= 1.0)   ? Mj
                                : (lam <= 0.0) ? sh.b_att[cur][j]
                                               : lam * Mj + (1.0 - lam) * sh.b_att[cur][j];
            sh.kb[j] = (float)(base - sh.off);
          }
          if (act) {
            for (int i = hl; i < W; i += 16) {  // this lane's own phi entries
              const double pv = phi[(size_t)j * P.Tmax + i];
              const float f = (!is_zero(Mj) && !is_zero(pv)) ? __expf((float)(pv - Mj)) : 0.f;
              if constexpr (kTc) {
                // K-major tf32 operand: chunk i/8, 8-row N group, 16-byte K chunk
                PhiF[(i >> 3) * 128 + (j >> 3) * 64 + ((i & 7) >> 2) * 32 + (j & 7) * 4 +
                     (i & 3)] = tf32_rna(f);
              } else if constexpr (kMma) {
                PhiF[(size_t)i * BMAX + j] = tf32_rna(f);
              } else {
                PhiF[(size_t)i * BMAX + j] = f;
              }
            }
          }
        }
      }
      if (!P.exact && kTc) {
        // zero operand entries: parents nb..15 on every row of the chunks,
        // and rows W.. of the last chunk (their slab rows lie past the window)
        const int rows = ((W + 7) >> 3) * 8;
        for (int idx = tid; idx < rows * 16; idx += kNT) {
          const int i = idx >> 4, j = idx & 15;
          if (j >= nb || i >= W)
            PhiF[(i >> 3) * 128 + (j >> 3) * 64 + ((i & 7) >> 2) * 32 + (j & 7) * 4 + (i & 3)] =
                0.f;
        }
      }
      if (!P.exact && !kTc) {
        const int pad = BMAX - nb;  // factor columns of absent parents are zero
        for (int idx = tid; idx < W * pad; idx += kNT) {
          const int i = idx / pad, j = nb + (idx - i * pad);
          PhiF[(size_t)i * BMAX + j] = 0.f;
        }
        if (keys_mode)
          for (int idx = tid; idx < ub_words; idx += kNT) ubits[idx] = 0u;
      }
    }
    __syncthreads();

    bool step_fallback = P.exact != 0;  // fp64 decisions for this step
    if (!P.exact) {
      PROF_MARK(2);

      // ---- P3: K1 bulk prefix score + certified fp32 joint keys ----
      // Two adjacent token columns per thread. Every key's upper bound goes to
      // `kub` (underflow keys flagged in `ubits`); each thread keeps only its
      // top-2 certified lower bounds (theta0, P4), the exact theta comes from
      // the short list of keys that reach theta0 (P5).
      float l1 = -INFINITY, l2 = -INFINITY;
      float lcol = -INFINITY;  // filter mode: best column's worst-parent lower bound
      const float hw = (float)(lam * (P.dpsi0 + W * P.dpsi1)) + 1e-4f;
      const float gf = P.guard_f;
      const int row_same = sh.row_same;
      // m starts at the log-zero guard (not -inf): a log-zero grid entry then
      // never triggers a rescale and contributes exp(-1e30 - m) = 0, so the
      // per-element guard test disappears (an all-zero column keeps m == gf).
      // Accumulators are packed pairs of parents: fma.rn.f32x2 does two
      // fp32 FMAs per instruction with the same rounding as two fmaf. The
      // exp is ex2.approx.ftz
      // (terms below 2^-126 of the column max flush to zero: at most
      // W * 2^-126 absolute, covered by the W * 1e-6 key half-width).
      constexpr int kP = BMAX / 2;
      // The column shift is kept in log2 units (ms): each term is
      // 2^(x * L2E - ms) with ONE rounding (FFMA) instead of (x - m) * L2E.
      // The shift is the same for every term of an epoch, so ms itself
      // carries no error; the extra error is the rounding of L2E (|x| * 1.3e-8
      // per term, |x| <= |m| + 190 for every term above the flush) and the
      // conversion ms * LN2 of the final shift: <= |m| * 8.6e-8 + 2.5e-6 nats,
      // covered by the lam * (|m| * 1.5e-7 + 1e-5) term of the key half-width.
      // The start shift gs = round-up(gf * L2E) makes a log-zero entry
      // (x == gf) give 2^(<= 0), never an overflow.
      constexpr float kL2E = 1.44269504088896341f, kLn2 = 0.693147180559945309f;
      const float gs = __fmul_ru(gf, kL2E);
      auto mnat = [&](float ms) { return ms == gs ? gf : ms * kLn2; };
      // lazy rescale: the shift only moves when a value exceeds it by more
      // than 8 nats, so every accumulated term is <= e^8
      auto rescale_do = [&](float2(&Sx)[kP], float& ms, float x) {
        const float xs = x * kL2E;
        const float r = ex2_ftz(ms - xs);
        const float2 r2 = make_float2(r, r);
#pragma unroll
        for (int q = 0; q < kP; ++q) Sx[q] = __fmul2_rn(Sx[q], r2);
        ms = xs;
      };
      auto needs_rescale = [&](float ms, float x) { return fmaf(x, kL2E, -ms) > 8.f * kL2E; };
      auto rescale = [&](float2(&Sx)[kP], float& ms, float x) {
        if (needs_rescale(ms, x)) rescale_do(Sx, ms, x);
      };
      // both columns of a group, behind one warp-uniform branch: rescales
      // are rare after a tile's first group, and the predicated form issues
      // its ~16 instructions on every group
      auto rescale2 = [&](float2(&Sa)[kP], float& ma, float xa, float2(&Sb)[kP], float& mb,
                          float xb) {
        const bool na = needs_rescale(ma, xa), nb2 = needs_rescale(mb, xb);
        if (__any_sync(__activemask(), na || nb2)) {
          if (na) rescale_do(Sa, ma, xa);
          if (nb2) rescale_do(Sb, mb, xb);
        }
      };
      auto acc_term = [&](float2(&Sx)[kP], float ms, float x, const float* ph) {
        const float pe = ex2_ftz(fmaf(x, kL2E, -ms));
        const float2 p2 = make_float2(pe, pe);
        if constexpr (BMAX % 4 == 0) {  // 16-byte factor rows
#pragma unroll
          for (int q = 0; q < BMAX / 4; ++q) {
            const float4 f = reinterpret_cast<const float4*>(ph)[q];
            Sx[2 * q + 0] = __ffma2_rn(make_float2(f.x, f.y), p2, Sx[2 * q + 0]);
            Sx[2 * q + 1] = __ffma2_rn(make_float2(f.z, f.w), p2, Sx[2 * q + 1]);
          }
        } else {  // BMAX = 10: 8-byte rows
#pragma unroll
          for (int q = 0; q < kP; ++q)
            Sx[q] = __ffma2_rn(reinterpret_cast<const float2*>(ph)[q], p2, Sx[q]);
        }
      };
      auto acc = [&](float2(&Sx)[kP], float& m, float x, const float* ph) {
        rescale(Sx, m, x);
        acc_term(Sx, m, x, ph);
      };
      long long tq_frames = 0, tq_keys = 0;
      constexpr int kCh = 2;  // frames per prefetch chunk (register budget)
      const int W4 = W & ~(kCh - 1);
      // certified keys: joint(j, c) - off in [key - h, key + h]; parent-major
      // so each parent's constants are read once for both columns
      const float* phr = PhiF;
      constexpr int phs = BMAX;  // floats per PhiF row
      // per-step key constants held in registers across the key loop (opaque
      // to the compiler, which otherwise re-derives them from the kernel
      // parameters for every key: LDC + DSETP + F2F per key)
      float klamf = lamf, kgf = gf;
      int klam_pos = lam > 0.0 ? 1 : 0;
      asm volatile("" : "+f"(klamf), "+f"(kgf), "+r"(klam_pos));
      const bool lam_pos = klam_pos != 0;
      // Keys of one column pair: certified bounds. Pass 1 keeps the thread's
      // top-2 lower bounds (and in keys mode writes every upper key and its
      // underflow flag to shared memory for the P5 scan). Filter mode then
      // runs pass 2 (emit == true) after the warp's running bound is known:
      // the same keys are recomputed (identical arithmetic) and those whose
      // upper bound reaches the bound go to the raw list.
      auto emit_keys = [&](int c0, int c1, bool two, const float2(&S0)[kP],
                           const float2(&S1)[kP], float m0, float m1, float r0s, float r1s,
                           bool emit, float th, float& kmax) {
        // filter mode, pass 1: min over the parents of each column's lower
        // bounds (with B live parents, B distinct candidates reach it), and
        // the largest upper key (pass 2 is skipped when it misses the bound)
        float cmin0 = INFINITY, cmin1 = INFINITY;
#pragma unroll
        for (int q = 0; q < BMAX; ++q) {
          if (q < nb) {
            const int last = sh.b_last[cur][q];
            const float kbq = sh.kb[q];
            const bool mz = sh.mzero[q] != 0;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              const int c = cc ? c1 : c0;
              if (cc == 1 && !two) break;
              const float m = cc ? m1 : m0;
              const float2 Sp = cc ? S1[q >> 1] : S0[q >> 1];
              const float Sq = (q & 1) ? Sp.y : Sp.x;
              float klo = -INFINITY, kub_v = -INFINITY;
              bool under = false;
              if (c != last) {
                const float r = row_same >= 0 ? (cc ? r1s : r0s)
                                              : attf_at(P, sh.b_row[cur][q], c);
                // same arithmetic as kbq + lamf * (m + __logf(Sq)) + r for a
                // normal Sq; below 2^-100 only the certified upper bound
                // with log(Sq) <= log(2^-99) is kept
                under = lam_pos && !(Sq >= 7.888609052210118e-31f);  // 2^-100
                const float lg = under ? -68.62157f : lg2_ftz(Sq) * 0.693147180559945309f;
                const float key = lam_pos ? kbq + klamf * (m + lg) + r : kbq + r;
                const float h = hw + fabsf(key) * 2.4e-7f + klamf * fmaf(fabsf(m), 1.5e-7f, 1e-5f);
                klo = under ? -INFINITY : key - h;
                kub_v = key + h;
                // joint exactly kLogZero: att log-zero, or psi log-zero
                const bool zero = r == -INFINITY || (lam_pos && (mz || m == kgf));
                if (zero) {
                  klo = kub_v = kZeroKey;
                  under = false;
                }
                if (!emit) {
                  kmax = fmaxf(kmax, kub_v);
                  if (cc) cmin1 = fminf(cmin1, klo);
                  else cmin0 = fminf(cmin0, klo);
                  if (klo > l2) {
                    if (klo > l1) {
                      l2 = l1;
                      l1 = klo;
                    } else {
                      l2 = klo;
                    }
                  }
                } else if (kub_v >= th) {
                  const int idx = atomicAdd(&sh.n_raw, 1);
                  if (idx < raw_cap(BMAX))
                    rawl[idx] = make_uint2(__float_as_uint(kub_v),
                                           (under ? 0x80000000u : 0u) | ((unsigned)q << 24) |
                                               (unsigned)c);
                }
              }
              if (keys_mode) {
                const int kidx = q * C + c;
                kub[kidx] = kub_v;
                if (under) atomicOr(&ubits[kidx >> 5], 1u << (kidx & 31));
              }
              if (c == last) {  // the repeat column is scored exactly: no bound from it
                if (cc) cmin1 = -INFINITY;
                else cmin0 = -INFINITY;
              }
            }
          }
        }
        if (!keys_mode && !emit && nb >= B)
          lcol = fmaxf(lcol, fmaxf(cmin0, two ? cmin1 : -INFINITY));
      };
      // Filter mode (whole warp, after a column tile's pass 1): the B-th
      // largest of the lanes' best lower bounds is a valid lower bound on
      // theta0 (B distinct candidates reach it), so the block-wide running
      // maximum of these bounds only rises towards theta0; a key whose upper
      // bound is below it can never reach theta0 and is dropped.
      // Three valid bounds, the best taken: the B-th best of the lanes' best
      // keys (spread-out candidates), the ceil(B/2)-th best of their second
      // best, and the best column whose B parents all reach a value
      // (clustered candidates: near-equal parents share their best tokens).
      // The two sorts run on the first tiles and every fourth after (`full`):
      // the running bound is near theta0 by then and only rises.
      auto warp_bound = [&](bool full) -> float {
        float wb = warp_max_f(lcol);
        if (full)
          wb = fmaxf(wb, fmaxf(warp_kth_desc(l1, B - 1, lane),
                               warp_kth_desc(l2, (B - 1) >> 1, lane)));
        if (lane == 0) atomicMax(&sh.th_run, f2ord(wb));
        __syncwarp();
        return fmaxf(wb, ord2f(*reinterpret_cast<volatile int*>(&sh.th_run)));
      };
      if constexpr (kTc) {
        // K1 bulk on the tensor cores. For a 512-column tile,
        //   S[c][j] = sum_t exp(L[t,c] - m_c) * a_j[t]   (a_j = PhiF, P2)
        // is a [512 x W] . [W x 16] product: the TMA stage (8 rows x 512
        // columns as 16 blocks of 8 x 32, 32-byte-atom 128-byte swizzle) is
        // exponentiated IN PLACE and then is the MN-major tf32 A operand of
        // four tcgen05.mma (M = 128 columns, N = 16 parents, K = 8 rows),
        // accumulating in TMEM (two 64-column buffers, alternating tiles).
        // The shift m_c is fixed for the step: the max of column c over the
        // rows the window can reach (so every exp is <= 1 and no rescale is
        // needed); it was taken while the previous step streamed (or by the
        // step-1 pass), and this step takes the next step's the same way.
        // The warp that finishes a stage last issues its MMAs and refills
        // the previous job's stage once that stage's MMAs are done.
        const int nch = (W + 7) >> 3;
        const int ntile = (C + 511) >> 9;
        const int J = ntile * nch;
        const int NST = P.tma_stages;
        const int urow = ud.row0 + s - 1;
        const unsigned tmem = tmem_base;
        auto issue = [&](int j, unsigned g) {
          const int st = (int)(g % (unsigned)NST), tile = j / nch, k = j - tile * nch;
          mbar_expect_tx(&mbar[st], kTmaStageBytes);
          tma_load_3d(tc_stg + (size_t)st * kTmaStageBytes, &P.tmap, 0, urow + k * 8, tile * 16,
                      &mbar[st]);
        };
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          for (int j = 0; j < NST && j < J; ++j) issue(j, tma_jobs + j);
        }
        // transform roles: block tbk of the stage, logical 4-column quad gq,
        // rows rg, rg + 2, rg + 4, rg + 6 (conflict-free 16-byte accesses)
        const int tbk = tid >> 4, gq = tid & 7, rg = (tid >> 3) & 1;
        const float* msh = P.mshift + ((size_t)(l & 1) * P.U + u) * P.mshift_stride;
        float* msn = P.mshift + ((size_t)((l + 1) & 1) * P.U + u) * P.mshift_stride;
        // the frame s is in the next window only if s > l (s >= l always)
        const int skip0 = (s == l) ? 1 : 0;
        constexpr float kL2e = 1.44269504088896341f;
        float4 ml2 = make_float4(0.f, 0.f, 0.f, 0.f), mx = ml2;
        // epilogue roles: TMEM lanes 32 * (warp % 4) + lane of subtiles
        // 2 * (warp / 4) and + 1, i.e. columns ca and ca + 128 of the tile
        const int sub0 = 2 * (warp >> 2);
        for (int j = 0; j < J; ++j) {
          const unsigned g = tma_jobs + j;
          const int st = (int)(g % (unsigned)NST);
          const int tile = j / nch, k = j - tile * nch;
          const int colq = tile * 512 + tbk * 32 + gq * 4;
          if (k == 0) {
            const float4 m4 = *reinterpret_cast<const float4*>(msh + colq);
            ml2 = make_float4(m4.x * kL2e, m4.y * kL2e, m4.z * kL2e, m4.w * kL2e);
            mx = make_float4(gf, gf, gf, gf);
          }
          mbar_wait_dbg(&mbar[st], (g / (unsigned)NST) & 1u, 2, g);
          float* sb = reinterpret_cast<float*>(tc_stg + (size_t)st * kTmaStageBytes) + tbk * 256;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const int r = rg + 2 * rr;
            const int fr = 8 * k + r;  // frame s + fr
            float4* px = reinterpret_cast<float4*>(
                sb + r * 32 + (((((gq >> 1) ^ r) & 3) << 3) | ((gq & 1) << 2)));
            const float4 x = *px;
            float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (fr < W) {
              if (fr > 0 || !skip0) {
                mx.x = fmaxf(mx.x, x.x);
                mx.y = fmaxf(mx.y, x.y);
                mx.z = fmaxf(mx.z, x.z);
                mx.w = fmaxf(mx.w, x.w);
              }
              pv.x = ex2_ftz(fmaf(x.x, kL2e, -ml2.x));
              pv.y = ex2_ftz(fmaf(x.y, kL2e, -ml2.y));
              pv.z = ex2_ftz(fmaf(x.z, kL2e, -ml2.z));
              pv.w = ex2_ftz(fmaf(x.w, kL2e, -ml2.w));
            }
            *px = pv;
          }
          // generic-proxy writes -> the MMA (async proxy); arrival
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_before_sync();
          __syncwarp();
          if (lane == 0) {
            const int done = atomicAdd(&cons[st], 1);
            if (done == (int)(g / (unsigned)NST) * kNWarp + kNWarp - 1) {
              tc_after_sync();
              const unsigned char* a0 = tc_stg + (size_t)st * kTmaStageBytes;
              const unsigned long long db = umma_desc_kint(reinterpret_cast<const unsigned char*>(PhiF) + k * kTcChunkBytes);
              const unsigned dcol = tmem + (unsigned)((tile & 1) * 64);
#pragma unroll
              for (int sub = 0; sub < 4; ++sub)
                umma_tf32(dcol + sub * 16, umma_desc_mn32(a0 + sub * 4096), db, k > 0 ? 1u : 0u);
              umma_commit(&mmad[st]);
              if (j > 0 && j - 1 + NST < J) {  // refill the previous job's stage
                const unsigned gp = g - 1;
                const int stp = (int)(gp % (unsigned)NST);
                mbar_wait_dbg(&mmad[stp], (gp / (unsigned)NST) & 1u, 3, gp);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(j - 1 + NST, gp + NST);
              }
            }
          }
          if (k == nch - 1) {  // tile epilogue
            mx.x = fmaxf(mx.x, __shfl_xor_sync(0xffffffffu, mx.x, 8));
            mx.y = fmaxf(mx.y, __shfl_xor_sync(0xffffffffu, mx.y, 8));
            mx.z = fmaxf(mx.z, __shfl_xor_sync(0xffffffffu, mx.z, 8));
            mx.w = fmaxf(mx.w, __shfl_xor_sync(0xffffffffu, mx.w, 8));
            if (rg == 0) *reinterpret_cast<float4*>(msn + colq) = mx;
            mbar_wait_dbg(&mmad[st], (g / (unsigned)NST) & 1u, 4, g);  // the tile's last MMAs
            tc_after_sync();
            float v0[16], v1[16];
            const unsigned trow = tmem + ((unsigned)(32 * (warp & 3)) << 16) +
                                  (unsigned)((tile & 1) * 64);
            tmem_ld16(trow + sub0 * 16, v0);
            tmem_ld16(trow + (sub0 + 1) * 16, v1);
            tc_before_sync();
            const int ca = tile * 512 + sub0 * 128 + 32 * (warp & 3) + lane, cb = ca + 128;
            const bool acta = ca < C, actb = cb < C;
            float2 S0[kP], S1[kP];
#pragma unroll
            for (int q = 0; q < kP; ++q) {
              S0[q] = make_float2(v0[2 * q], v0[2 * q + 1]);
              S1[q] = make_float2(v1[2 * q], v1[2 * q + 1]);
            }
            const float ma = msh[ca], mb = msh[cb];
            const float ra = (row_same >= 0 && acta) ? attf_at(P, row_same, ca) : 0.f;
            const float rb = (row_same >= 0 && actb) ? attf_at(P, row_same, cb) : 0.f;
            float kmax = -INFINITY;
            if (acta) emit_keys(ca, cb, actb, S0, S1, ma, actb ? mb : gf, ra, rb, false, 0.f, kmax);
            const float th = warp_bound(tile < 3 || (tile & 3) == 0);
            if (acta && kmax >= th)
              emit_keys(ca, cb, actb, S0, S1, ma, actb ? mb : gf, ra, rb, true, th, kmax);
          }
        }
        tma_jobs += J;
      } else if constexpr (kMma) {
        // K1 bulk on the warp-level tensor cores (mma.sync m16n8k8 tf32):
        // for a 512-column tile, S[c][j] = sum_t exp(L[t,c] - m_c) a_j[t] is a
        // [512 x W] . [W x 16] product. Warp w owns columns 64w .. 64w+63
        // (swizzle blocks 2w, 2w+1 of the stage); lane (g, t) (g = lane/4,
        // t = lane%4) loads, per 8-row chunk, rows t and t+4 of the 16-byte
        // chunk chA(g) of both blocks (the standard 128-byte swizzle makes
        // these loads conflict-free), exponentiates them against the fixed
        // utterance's column maxima (the step-1 pass: a valid shift for every
        // window, all of them lie inside [1, T]; no lazy rescale) and
        // feeds them as A fragments: m-tile e has m = g <-> block 2w column e
        // of the chunk and m = g+8 <-> block 2w+1, k = t, t+4 <-> the two rows;
        // B fragments are the parents' factors (n = g, g+8). The accumulators
        // stay in registers: lane (g, t) ends the tile with S for its 8
        // columns x parents 2t, 2t+1, 8+2t, 9+2t. Stages are released per
        // warp as in the CUDA-core variant. Two CTAs per SM as before.
        const int nch = (W + 7) >> 3;
        const int ntile = (C + 511) >> 9;
        const int J = ntile * nch;
        const int NST = P.tma_stages;
        const int urow = ud.row0 + s - 1;
        auto issue = [&](int j, unsigned g) {
          const int st = (int)(g % (unsigned)NST), tile = j / nch, k = j - tile * nch;
          mbar_expect_tx(&mbar[st], kTmaStageBytes);
          tma_load_3d(tc_stg + (size_t)st * kTmaStageBytes, &P.tmap, 0, urow + k * 8, tile * 16,
                      &mbar[st]);
        };
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          for (int j = 0; j < NST && j < J; ++j) issue(j, tma_jobs + j);
        }
        const int g8 = lane >> 2, t4 = lane & 3;
        const int chA = (g8 & 1) * 4 + (g8 >> 1);  // this lane's 16-byte chunk in each block
        // the utterance's column maxima over all T frames (step-1 pass)
        const float* msh = P.mshift + ((size_t)1 * P.U + u) * P.mshift_stride;
        constexpr float kL2e = 1.44269504088896341f;
        float acc[4][2][4];  // [m-tile e][n-tile h][fragment]
        // this lane's parents: n-tile h, fragment pair -> 8h + 2t + {0, 1}
        for (int j = 0; j < J; ++j) {
          const unsigned g = tma_jobs + j;
          const int st = (int)(g % (unsigned)NST);
          const int tile = j / nch, k = j - tile * nch;
          const int col0 = tile * 512 + warp * 64 + chA * 4;  // block 2w; block 2w+1 is +32
          if (k == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int f = 0; f < 4; ++f) acc[e][h][f] = 0.f;
          }
          // the shifts of the own columns (L1-resident; reloaded per chunk
          // rather than held in registers across the tile)
          const float4 ma = *reinterpret_cast<const float4*>(msh + col0);
          const float4 mb = *reinterpret_cast<const float4*>(msh + col0 + 32);
          const float mlc[8] = {ma.x * kL2e, ma.y * kL2e, ma.z * kL2e, ma.w * kL2e,
                                mb.x * kL2e, mb.y * kL2e, mb.z * kL2e, mb.w * kL2e};
          mbar_wait(&mbar[st], (g / (unsigned)NST) & 1u);
          const float* blk =
              reinterpret_cast<const float*>(tc_stg + (size_t)st * kTmaStageBytes) + warp * 512;
          float pa[2][8];  // [row pair rr][own column]: exp(L - m) as tf32
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int r = t4 + 4 * rr;
            const int fr = 8 * k + r;  // frame s + fr
            const int ph = r * 32 + (((chA ^ r) & 7) << 2);
            const float4 xa = *reinterpret_cast<const float4*>(blk + ph);
            const float4 xb = *reinterpret_cast<const float4*>(blk + 256 + ph);
            const float xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
            const bool valid = fr < W;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              pa[rr][q] = valid ? tf32_rna(ex2_ftz(fmaf(xv[q], kL2e, -mlc[q]))) : 0.f;
          }
          // B fragments: factors of parents 8h + g at rows t, t+4 of the chunk
          unsigned bf[2][2];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const int row = 8 * k + t4 + 4 * rr, par = 8 * h + g8;
              bf[h][rr] = (par < BMAX && row < W)
                              ? __float_as_uint(PhiF[(size_t)row * BMAX + par])
                              : 0u;
            }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const unsigned a0 = __float_as_uint(pa[0][e]), a1 = __float_as_uint(pa[0][4 + e]);
            const unsigned a2 = __float_as_uint(pa[1][e]), a3 = __float_as_uint(pa[1][4 + e]);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              asm volatile(
                  "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
                  "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                  : "+f"(acc[e][h][0]), "+f"(acc[e][h][1]), "+f"(acc[e][h][2]),
                    "+f"(acc[e][h][3])
                  : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bf[h][0]), "r"(bf[h][1]));
          }
          // stage release per warp (as the CUDA-core variant)
          __syncwarp();
          if (lane == 0) {
            const int done = atomicAdd(&cons[st], 1);
            if (done == (int)(g / (unsigned)NST) * kNWarp + kNWarp - 1 && j + NST < J) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(j + NST, g + NST);
            }
          }
          if (k == nch - 1) {  // tile epilogue: keys of own columns
            // two passes like emit_keys: bounds (l1/l2, column minima) first,
            // then the raw-list emission against the warp's running bound
            float kmax = -INFINITY;
            for (int pass = 0; pass < 2; ++pass) {
              float th = 0.f;
              if (pass == 1) {
                th = warp_bound(tile < 3 || (tile & 3) == 0);
                if (!(kmax >= th)) break;
              }
#pragma unroll
              for (int q = 0; q < 8; ++q) {  // own column q: block half q/4, element q%4
                const int e = q & 3, hb = q >> 2;
                const int c = col0 + hb * 32 + e;
                const bool cin = c < C;
                const float m = cin ? msh[c] : gf;
                const float rs =
                    (row_same >= 0 && cin) ? attf_at(P, row_same, c) : 0.f;
                float cmin = INFINITY;
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                  for (int f1 = 0; f1 < 2; ++f1) {
                    const int qp = 8 * h + 2 * t4 + f1;  // parent of fragment 2*hb + f1
                    if (!cin || qp >= nb || qp >= BMAX) continue;
                    if (c == sh.b_last[cur][qp]) {  // the repeat column is scored exactly
                      cmin = -INFINITY;
                      continue;
                    }
                    const float Sq = acc[e][h][2 * hb + f1];
                    const float r =
                        row_same >= 0 ? rs : attf_at(P, sh.b_row[cur][qp], c);
                    const bool under = lam_pos && !(Sq >= 7.888609052210118e-31f);  // 2^-100
                    const float lg = under ? -68.62157f : lg2_ftz(Sq) * 0.693147180559945309f;
                    const float kbq = sh.kb[qp];
                    const float key = lam_pos ? kbq + klamf * (m + lg) + r : kbq + r;
                    const float hh = hw + fabsf(key) * 2.4e-7f;
                    float klo = under ? -INFINITY : key - hh, kub_v = key + hh;
                    bool und = under;
                    if (r == -INFINITY || (lam_pos && (sh.mzero[qp] != 0 || m == kgf))) {
                      klo = kub_v = kZeroKey;
                      und = false;
                    }
                    if (pass == 0) {
                      kmax = fmaxf(kmax, kub_v);
                      cmin = fminf(cmin, klo);
                      if (klo > l2) {
                        if (klo > l1) {
                          l2 = l1;
                          l1 = klo;
                        } else {
                          l2 = klo;
                        }
                      }
                    } else if (kub_v >= th) {
                      const int idx = atomicAdd(&sh.n_raw, 1);
                      if (idx < raw_cap(BMAX))
                        rawl[idx] = make_uint2(__float_as_uint(kub_v),
                                               (und ? 0x80000000u : 0u) | ((unsigned)qp << 24) |
                                                   (unsigned)c);
                    }
                  }
                if (pass == 0 && nb >= B) {
                  // a column's bound needs all B parents: min over the 4 lanes
                  // sharing it (each holds 4 of the 16 parent slots)
                  cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, 1));
                  cmin = fminf(cmin, __shfl_xor_sync(0xffffffffu, cmin, 2));
                  if (cin) lcol = fmaxf(lcol, cmin);
                }
              }
            }
          }
        }
        tma_jobs += J;
      } else if constexpr (kTma) {
        // K1 slab streamed by TMA: job j = (512-column tile, kSlabRows-row
        // chunk). Each warp streams its own 64 columns of the tile through its
        // own ring of slots (lane 0 issues one or two 8-row boxes per job,
        // one mbarrier per slot): a warp refills a slot as soon as it has
        // consumed it, so no warp waits for a slower one (a shared ring is
        // refilled only when its slowest consumer is done: ~14% of the bulk's
        // time went to waiting for data requested too late). 16-row jobs
        // halve the per-job overhead (wait, refill, counters) per row.
        constexpr int kBox = kTmaRows * kTmaBoxCols;  // floats per 8-row box
        static_assert(kTmaBoxCols == 64 && kSlabRows == 2 * kTmaRows,
                      "a warp slot is one or two 8-row boxes of 64 columns");
        // slots per warp: the stage area (tma_stages x 16 KB) split over the
        // warps, 16-row slots when that leaves two per warp, else 8-row ones
        const int wfl = P.tma_stages * kTmaStageBytes / (kNWarp * 4);  // floats per warp
        const int srows = wfl >= 2 * kSlabRows * kTmaBoxCols ? kSlabRows : kTmaRows;
        const int kSlice = srows * kTmaBoxCols;  // floats per warp slot
        const int NST = max(1, wfl / kSlice);
        const int nch = (W + srows - 1) / srows;
        const int ntile = (C + 2 * kNT - 1) / (2 * kNT);
        const int J = ntile * nch;
        float* wst = reinterpret_cast<float*>(region + pl.stages) + warp * kSlice;
        const unsigned wbar = smem_u32(&mbarw[warp]);  // + 8 * kNWarp per slot
        const int urow = ud.row0 + s - 1;
        auto issue_at = [&](int st, int tile, int k) {  // lane 0
          const unsigned bar = wbar + 8u * kNWarp * st;
          const unsigned dst = smem_u32(wst + st * kNWarp * kSlice);
          const int two_box = srows > kTmaRows && W - k * srows > kTmaRows;  // window rows only
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                       "r"((two_box ? 2 : 1) * kBox * 4)
                       : "memory");
          const int x = tile * 2 * kNT + warp * kTmaBoxCols, y = urow + k * srows;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
              "l"(reinterpret_cast<unsigned long long>(&P.tmap)), "r"(x), "r"(y), "r"(bar)
              : "memory");
          if (two_box)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst + kBox * 4),
                "l"(reinterpret_cast<unsigned long long>(&P.tmap)), "r"(x), "r"(y + kTmaRows),
                "r"(bar)
                : "memory");
        };
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          for (int j = 0; j < NST && j < J; ++j)
            issue_at((int)((tma_jobs + j) % (unsigned)NST), j / nch, j % nch);
        }
        float2 S0[kP], S1[kP];
        float m0 = gs, m1 = gs, r0s = 0.f, r1s = 0.f;
        const int colb = 2 * lane;
        // Column early-out (one row per step: row_same >= 0): every key of
        // column c is kb_q + lam * (m + lg S_q) + r with the same m and r, so
        // kbmax + lam * (m + lg max_q S_q) + r bounds them all (+ the largest
        // half-width, + 1e-3 for rounding); a column whose bound is below the
        // block's running bound cannot reach theta0 (nor raise a bound) and
        // skips both key passes. P4 takes theta0 >= the running bound, so
        // theta0, the list and the contenders are those of the full scan.
        float kbmax = -INFINITY;
        for (int q = 0; q < nb; ++q) kbmax = fmaxf(kbmax, sh.kb[q]);
        auto col_bound = [&](const float2(&Sx)[kP], float mn) {
          float smax = 0.f;
#pragma unroll
          for (int q = 0; q < kP; ++q)
            if (2 * q < nb) smax = fmaxf(smax, 2 * q + 1 < nb ? fmaxf(Sx[q].x, Sx[q].y) : Sx[q].x);
          const float lg = smax >= 7.888609052210118e-31f ? lg2_ftz(smax) * kLn2 : -68.62157f;
          const float un = lam_pos ? kbmax + klamf * (mn + lg) : kbmax;
          return un + fabsf(un) * 2.4e-7f + hw + klamf * fmaf(fabsf(mn), 1.5e-7f, 1e-5f) + 1e-3f;
        };
        // job counters kept incrementally (a runtime division per job and
        // thread was ~10% of this loop's instructions): slot, its use round
        // (mbarrier parity), tile and chunk
        int st = (int)(tma_jobs % (unsigned)NST);
        unsigned rnd = tma_jobs / (unsigned)NST;
        int tile = 0, k = 0;
        for (int j = 0; j < J; ++j) {
          const int c0 = tile * 2 * kNT + 2 * tid;
          const bool active = c0 < C, two = c0 + 1 < C;
          if (k == 0) {
#pragma unroll
            for (int q = 0; q < kP; ++q) S0[q] = S1[q] = make_float2(0.f, 0.f);
            m0 = m1 = gs;
            r0s = (row_same >= 0 && active) ? attf_at(P, row_same, c0) : 0.f;
            r1s = (row_same >= 0 && two) ? attf_at(P, row_same, c0 + 1) : 0.f;
          }
#ifdef BL_PROF_WAIT  // diagnostic build: warp 0's slot-wait cycles and stalls
          if (warp == 0) {
            const long long tw0 = clock64();
            unsigned ok;
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n}"
                : "=r"(ok)
                : "r"(wbar + 8u * kNWarp * st), "r"(rnd & 1u)
                : "memory");
            mbar_wait_sleep_s(wbar + 8u * kNWarp * st, rnd & 1u);
            tq_frames += clock64() - tw0;
            tq_keys += ok ? 0 : 1;
          } else
#endif
          mbar_wait_sleep_s(wbar + 8u * kNWarp * st, rnd & 1u);
          if (active) {
            const float* sb = wst + st * kNWarp * kSlice + colb;
            const int nrow = min(srows, W - k * srows);
            const float* ph0 = phr + k * srows * phs;
            constexpr int kRu = 8;  // rows per unrolled group
            int i0 = 0;
            // full 8-row groups: rows unrolled so their loads and exps overlap
            for (; i0 + kRu <= nrow; i0 += kRu) {
              float2 v[kRu];
#pragma unroll
              for (int k2 = 0; k2 < kRu; ++k2)
                v[k2] = *reinterpret_cast<const float2*>(sb + (i0 + k2) * kTmaBoxCols);
              float xma = v[0].x, xmb = v[0].y;
#pragma unroll
              for (int k2 = 1; k2 < kRu; ++k2) {
                xma = fmaxf(xma, v[k2].x);
                xmb = fmaxf(xmb, v[k2].y);
              }
              rescale2(S0, m0, xma, S1, m1, xmb);  // one test per column per group
#pragma unroll
              for (int k2 = 0; k2 < kRu; ++k2) {
                acc_term(S0, m0, v[k2].x, ph0 + (i0 + k2) * phs);
                acc_term(S1, m1, v[k2].y, ph0 + (i0 + k2) * phs);
              }
            }
            for (; i0 < nrow; ++i0) {  // the window's last rows
              const float2 v = *reinterpret_cast<const float2*>(sb + i0 * kTmaBoxCols);
              rescale2(S0, m0, v.x, S1, m1, v.y);
              acc_term(S0, m0, v.x, ph0 + i0 * phs);
              acc_term(S1, m1, v.y, ph0 + i0 * phs);
            }
          }
          // the warp's slot is consumed (every lane's reads fed its FMAs
          // above): lane 0 refills it with job j + NST
          __syncwarp();
          if (lane == 0) {
            if (j + NST < J) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              // job j + NST reuses this slot: its (tile, chunk) from this
              // job's without a division
              int kk = k + NST, tt = tile;
              while (kk >= nch) {
                kk -= nch;
                ++tt;
              }
              issue_at(st, tt, kk);
            }
          }
          if (k == nch - 1) {  // the tile's keys (whole warp: warp_bound)
            float kmax = -INFINITY;
            const float n0 = mnat(m0), n1 = two ? mnat(m1) : gf;
            bool keys = active;
            if (keys && row_same >= 0) {
              const float thr = ord2f(*reinterpret_cast<volatile int*>(&sh.th_run));
              keys = !(col_bound(S0, n0) + r0s < thr &&
                       (!two || col_bound(S1, n1) + r1s < thr));
            }
            if (keys) emit_keys(c0, c0 + 1, two, S0, S1, n0, n1, r0s, r1s, false, 0.f, kmax);
            const float th = warp_bound(tile < 3 || (tile & 3) == 0);
            if (keys && kmax >= th)
              emit_keys(c0, c0 + 1, two, S0, S1, n0, n1, r0s, r1s, true, th, kmax);
          }
          if (++st == NST) {
            st = 0;
            ++rnd;
          }
          if (++k == nch) {
            k = 0;
            ++tile;
          }
        }
        tma_jobs += J;
      } else {
      // warp-uniform trip count (warp_bound is a warp collective); thread
      // tid still owns columns 2 * tid + k * 2 * kNT
      for (int cb = 64 * warp; cb < C; cb += 2 * kNT) {
        const int c0 = cb + 2 * lane;
        const bool act = c0 < C;
        float kmax = -INFINITY;
        float2 S0[kP], S1[kP];
        float m0 = gs, m1 = gs, n0 = gf, n1 = gf, r0s = 0.f, r1s = 0.f;
        const bool two = c0 + 1 < C;
#pragma unroll
        for (int q = 0; q < kP; ++q) S0[q] = S1[q] = make_float2(0.f, 0.f);
        if (act) {
        const long long tq1 = clock64();
        r0s = row_same >= 0 ? attf_at(P, row_same, c0) : 0.f;
        r1s = (row_same >= 0 && two) ? attf_at(P, row_same, c0 + 1) : 0.f;
        const float* col = grid + (size_t)(s - 1) * V + c0;
        // columns c0 and c0+1 are both inside the row (c0 + 1 <= C = V-1,
        // the blank), so the pair is always loaded (the odd column of an odd
        // C is simply not emitted): one float2 load when rows are 8-byte
        // aligned (V even), else two scalar loads; no per-thread condition.
        auto ld = [&](const float* pp, float& a, float& b) {
          if ((V & 1) == 0) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(pp));
            a = v.x;
            b = v.y;
          } else {
            a = __ldg(pp);
            b = __ldg(pp + 1);
          }
        };
        float xa[kCh], xb[kCh];
        const float* pp = col;
        if (W4 > 0) {
#pragma unroll
          for (int k = 0; k < kCh; ++k) ld(pp + (size_t)k * V, xa[k], xb[k]);
        }
        for (int i0 = 0; i0 < W4; i0 += kCh) {
          float ya[kCh], yb[kCh];
#pragma unroll
          for (int k = 0; k < kCh; ++k) {
            ya[k] = xa[k];
            yb[k] = xb[k];
          }
          pp += (size_t)kCh * V;
          if (i0 + kCh < W4) {  // prefetch the next full chunk
#pragma unroll
            for (int k = 0; k < kCh; ++k) ld(pp + (size_t)k * V, xa[k], xb[k]);
          }
          // one rescale test per column per chunk, against the chunk max
          float xma = ya[0], xmb = yb[0];
#pragma unroll
          for (int k = 1; k < kCh; ++k) {
            xma = fmaxf(xma, ya[k]);
            xmb = fmaxf(xmb, yb[k]);
          }
          rescale(S0, m0, xma);
          rescale(S1, m1, xmb);
#pragma unroll
          for (int k = 0; k < kCh; ++k) {
            acc_term(S0, m0, ya[k], phr + (i0 + k) * phs);
            acc_term(S1, m1, yb[k], phr + (i0 + k) * phs);
          }
        }
        for (int i = W4; i < W; ++i) {  // remainder frames
          float a, b;
          ld(col + (size_t)i * V, a, b);
          acc(S0, m0, a, phr + i * phs);
          acc(S1, m1, b, phr + i * phs);
        }
        n0 = mnat(m0);
        n1 = two ? mnat(m1) : gf;
        const long long tq2 = clock64();
        tq_frames += tq2 - tq1;
        emit_keys(c0, c0 + 1, two, S0, S1, n0, n1, r0s, r1s, false, 0.f, kmax);
        tq_keys += clock64() - tq2;
        }
        if (!keys_mode) {
          const int it = cb / (2 * kNT);
          const float th = warp_bound(it < 3 || (it & 3) == 0);
          if (act && kmax >= th)
            emit_keys(c0, c0 + 1, two, S0, S1, n0, n1, r0s, r1s, true, th, kmax);
        }
      }
      }
      if (P.prof && tid == 0) {
        P.prof[(size_t)u * 16 + 12] += tq_frames;
        P.prof[(size_t)u * 16 + 13] += tq_keys;
      }

      // ---- P4: theta0 = B-th largest of the per-thread top-2 lower bounds:
      // a valid bound (B candidates certainly reach it) ----
      for (int r = 0; r < B; ++r) {
        const float mx = warp_max_f(l1);
        const unsigned who = __ballot_sync(0xffffffffu, l1 == mx);
        if (lane == __ffs(who) - 1) {
          l1 = l2;
          l2 = -INFINITY;
        }
        if (lane == 0) sh.wl[warp][r] = mx;
      }
      __syncthreads();
      PROF_MARK(3);
      if (warp == 0) {
        float list[BMAX];
#pragma unroll
        for (int q = 0; q < BMAX; ++q)
          list[q] = (lane < kNWarp && q < B) ? sh.wl[lane][q] : -INFINITY;
        float th = -INFINITY;
        for (int r = 0; r < B; ++r) {
          const float h = list[0];
          const float mx = warp_max_f(h);
          const unsigned who = __ballot_sync(0xffffffffu, h == mx);
          if (lane == __ffs(who) - 1) {
#pragma unroll
            for (int q = 0; q < BMAX - 1; ++q) list[q] = list[q + 1];
            list[BMAX - 1] = -INFINITY;
          }
          th = mx;
        }
        if (lane == 0) {
          // the running bound of the filter mode is a valid theta0 too (B
          // candidates reach it); the larger one lists fewer keys, with the
          // same theta and contenders
          sh.theta = keys_mode ? th : fmaxf(th, ord2f(sh.th_run));
          sh.theta2 = -INFINITY;  // stays when fewer than B keys are listed
          sh.n_list = 0;
        }
      }
      __syncthreads();
      PROF_MARK(4);

      // ---- P5: every key whose upper bound reaches theta0 goes to a short
      // list; the exact theta (B-th largest lower bound) is ranked inside it
      // and the contenders are the list entries that reach max(theta, theta0).
      const float theta0 = sh.theta;
      auto list_key_qc = [&](int kidx, int q, int c, float ku) {
        if (c != sh.b_last[cur][q]) {
          const int idx = atomicAdd(&sh.n_list, 1);
          if (idx < list_cap(BMAX)) {
            const bool under = (ubits[kidx >> 5] >> (kidx & 31)) & 1u;
            // derived lower bound: never above the key's true lower bound
            clist[idx] = make_float4(
                under ? -INFINITY : ku - 2.000002f * (hw + (fabsf(ku) + hw) * 2.4e-7f), ku,
                __int_as_float(q), __int_as_float(c));
          }
        }
      };
      auto list_key = [&](int kidx, float ku) {
        const int q = kidx / C;
        list_key_qc(kidx, q, kidx - q * C, ku);
      };
      const int nkeys = nb * C;
      if (keys_mode && C >= kNT) {
        // (q, c) of kidx kept incrementally (stride kNT <= C: at most one wrap);
        // four keys loaded before any test (the listing's shared-memory
        // atomics otherwise order every load after the previous test)
        int q = 0, c = tid, kidx = tid;
        for (; kidx + 3 * kNT < nkeys; kidx += 4 * kNT) {
          float ku[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) ku[r] = kub[kidx + r * kNT];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (ku[r] >= theta0) list_key_qc(kidx + r * kNT, q, c, ku[r]);
            c += kNT;
            if (c >= C) {
              c -= C;
              ++q;
            }
          }
        }
        for (; kidx < nkeys; kidx += kNT) {
          const float ku = kub[kidx];
          if (ku >= theta0) list_key_qc(kidx, q, c, ku);
          c += kNT;
          if (c >= C) {
            c -= C;
            ++q;
          }
        }
      } else if (keys_mode) {
        for (int kidx = tid; kidx < nkeys; kidx += kNT) {
          const float ku = kub[kidx];
          if (ku >= theta0) list_key(kidx, ku);
        }
      } else {
        // filter mode: the raw list holds every key that reached the running
        // bound (a superset of the keys reaching theta0); keep those that
        // reach theta0. A raw-list overflow falls back like a list overflow.
        const int nraw = sh.n_raw;
        if (tid == 0) sh.c_raw += nraw;
        if (nraw > raw_cap(BMAX)) {
          if (tid == 0) sh.n_list = list_cap(BMAX) + 1;
        } else {
          for (int k = tid; k < nraw; k += kNT) {
            const uint2 e2 = rawl[k];
            const float ku = __uint_as_float(e2.x);
            if (ku >= theta0) {
              const int idx = atomicAdd(&sh.n_list, 1);
              if (idx < list_cap(BMAX)) {
                // derived lower bound: the one the keys-mode P5 scan lists
                clist[idx] = make_float4(
                    (e2.y >> 31) ? -INFINITY : ku - 2.000002f * (hw + (fabsf(ku) + hw) * 2.4e-7f),
                    ku, __int_as_float((int)((e2.y >> 24) & 0x7fu)),
                    __int_as_float((int)(e2.y & 0xffffffu)));
              }
            }
          }
        }
      }
      __syncthreads();
      const int nl = sh.n_list;
      if (nl > list_cap(BMAX)) {
        if (tid == 0) sh.n_cont = P.caps + 1;  // overflow: exact fallback
      } else if constexpr (list_cap(BMAX) <= kNT) {
        if (tid < nl) {
          const float lo = clist[tid].x;
          int rank = 0;
          for (int k = 0; k < nl; ++k) {
            const float o = clist[k].x;
            rank += (o > lo || (o == lo && k < tid)) ? 1 : 0;
          }
          if (rank == B - 1) sh.theta2 = lo;  // unique writer (ranks are distinct)
        }
      } else {
        for (int i = tid; i < nl; i += kNT) {
          const float lo = clist[i].x;
          int rank = 0;
          for (int k = 0; k < nl && rank < B; ++k) {
            const float o = clist[k].x;
            rank += (o > lo || (o == lo && k < i)) ? 1 : 0;
          }
          if (rank == B - 1) sh.theta2 = lo;
        }
      }
      __syncthreads();
      if (nl <= list_cap(BMAX)) {
        const float theta = fmaxf(sh.theta2, theta0);
        if constexpr (list_cap(BMAX) <= kNT) {
          if (tid < nl && clist[tid].y >= theta) {
            const int idx = atomicAdd(&sh.n_cont, 1);
            if (idx < caps) {
              items[idx].parent = __float_as_int(clist[tid].z);
              items[idx].token = __float_as_int(clist[tid].w);
            }
          }
        } else {
          for (int i = tid; i < nl; i += kNT)
            if (clist[i].y >= theta) {
              const int idx = atomicAdd(&sh.n_cont, 1);
              if (idx < caps) {
                items[idx].parent = __float_as_int(clist[i].z);
                items[idx].token = __float_as_int(clist[i].w);
              }
            }
        }
      }
      if (warp == kNWarp - 1 && lane < nb && sh.b_last[cur][lane] >= 0) {
        const int idx = atomicAdd(&sh.n_cont, 1);  // repeat column: always exact
        if (idx < caps) {
          items[idx].parent = lane;
          items[idx].token = sh.b_last[cur][lane];
        }
      }
      __syncthreads();
      // every thread derives the same decision; thread 0 records it (what
      // other threads may still read is the same value)
      step_fallback = sh.fallback || sh.n_cont > P.caps;
      if (tid == 0) {
        sh.c_cont += sh.n_cont;
        sh.fallback = step_fallback;
      }
      PROF_MARK(5);
    }

    // Decision group of this step: warps [gw0, kNWarp) run P7-P9. On the
    // staged path the contender chains (warps [0, nser)) only produce the
    // children's gamma states and tau, which nothing in P7-P9 reads, so
    // they overlap with ranking, walk and end detection; tau is patched in
    // after the join.
    int gw0 = 0;
    if (!step_fallback) {
      const int nc = sh.n_cont;
      const long long ts0 = clock64();
      // ---- P6a: stage the contenders' grid columns, the blank column and the
      // repeat-column phi (gamma_b[t-1], ctc_prefix.cpp:50) with stride W ----
      const size_t offB = align16(sizeof(float) * (size_t)nc * W);
      const size_t offR = offB + align16(sizeof(float) * (size_t)W);
      const bool staged = offR + sizeof(double) * (size_t)nb * W <= (size_t)P.region_bytes;
      float* stL = reinterpret_cast<float*>(region);
      float* stB = reinterpret_cast<float*>(region + offB);
      double* stR = reinterpret_cast<double*>(region + offR);
      if (staged && keys_mode) {  // small windows (80-register variant)
        for (int idx = tid; idx < (nc + 1) * W; idx += kNT) {
          const int q = idx / W, i = idx - q * W;
          const int c = q < nc ? items[q].token : blank;
          const float v = grid[(size_t)(s - 1 + i) * V + c];
          if (q < nc) stL[idx] = v;
          else stB[i] = v;
        }
        for (int idx = tid; idx < nb * W; idx += kNT) {
          const int j = idx / W, i = idx - j * W;
          if (sh.b_last[cur][j] < 0) continue;
          const double* gbp = gam_ptr(P, u, sh.b_area[cur][j], sh.b_slot[cur][j], 1);
          stR[idx] = gread(gbp, s + i - 1, sh.b_vlo[cur][j], sh.b_cov[cur][j]);
        }
      } else if (staged) {
        // kSt independent loads per thread in flight before any store (the
        // columns are scattered rows apart in HBM: one load at a time would
        // serialise their latency)
        constexpr int kSt = 4;
        const int ntot = (nc + 1) * W;
        for (int base = tid; base < ntot; base += kSt * kNT) {
          float v[kSt];
#pragma unroll
          for (int r = 0; r < kSt; ++r) {
            const int idx = base + r * kNT;
            if (idx < ntot) {
              const int q = idx / W, i = idx - q * W;
              const int c = q < nc ? items[q].token : blank;
              v[r] = grid[(size_t)(s - 1 + i) * V + c];
            }
          }
#pragma unroll
          for (int r = 0; r < kSt; ++r) {
            const int idx = base + r * kNT;
            if (idx < ntot) {
              if (idx < nc * W) stL[idx] = v[r];
              else stB[idx - nc * W] = v[r];
            }
          }
        }
        const int rtot = nb * W;
        for (int base = tid; base < rtot; base += kSt * kNT) {
          double v[kSt];
#pragma unroll
          for (int r = 0; r < kSt; ++r) {
            const int idx = base + r * kNT;
            const int j = idx / W, i = idx - j * W;
            if (idx < rtot && sh.b_last[cur][j] >= 0) {
              const double* gbp = gam_ptr(P, u, sh.b_area[cur][j], sh.b_slot[cur][j], 1);
              v[r] = gread(gbp, s + i - 1, sh.b_vlo[cur][j], sh.b_cov[cur][j]);
            }
          }
#pragma unroll
          for (int r = 0; r < kSt; ++r) {
            const int idx = base + r * kNT;
            if (idx < rtot && sh.b_last[cur][idx / W] >= 0) stR[idx] = v[r];
          }
        }
      }
      __syncthreads();
#ifndef BL_PROF_WAIT
      if (P.prof && tid == 0) P.prof[(size_t)u * 16 + 15] += clock64() - ts0;
#endif
      // ---- P6: contenders re-scored exactly. Warps [0, nser): the serial
      // gamma_n'/gamma_b' chains (one thread per contender, reference op
      // order); the other warps: psi by a parallel fp64 log-sum-exp. ----
      // staged: two lanes per contender (16 per warp); otherwise one
      const int nser = staged ? (nc + 15) >> 4 : (nc + 31) >> 5;
      if (warp < nser && staged) {
        const int q0 = tid >> 1, role = tid & 1;
        const bool live = q0 < nc;
        const int q = live ? q0 : nc - 1;  // idle lanes shadow a real chain
        const int j = items[q].parent, c = items[q].token;
        const bool repeat = sh.b_last[cur][j] == c;
        double* gnc = gam_ptr(P, u, nxt, q, 0);
        int best;
        const long long tr0 = clock64();
        child_state_lanes(repeat ? stR + (size_t)j * W : phi + (size_t)j * P.Tmax,
                          stL + (size_t)q * W, stB, s, W, sh.b_tau[cur][j],
                          role == 0 ? gnc : gnc + P.Tp, role, live, &best, tb);
        if (live) {
          if (role == 0) items[q].tau = best;
          else items[q].taut = best;
        }
        PROF_SERIAL(tr0);
      } else if (warp < nser) {
        // inputs not staged (window too wide for the region): one lane per
        // contender runs the chains and psi from global memory
        const int q = tid;
        if (q < nc) {
          const int j = items[q].parent, c = items[q].token;
          double* gnc = gam_ptr(P, u, nxt, q, 0);
          double* gbc = gnc + P.Tp;
          int tau, taut;
          const long long tr0 = clock64();
          const double psi = child_recursion_global<BMAX>(
              P, sh, u, cur, j, c, s, e, grid, phi + (size_t)j * P.Tmax, gnc, gbc, &tau, &taut,
              tb);
          const double att = __dadd_rn(sh.b_att[cur][j],
                                       att_at(P, sh.b_row[cur][j], c));
          items[q].score = mix_joint(lam, psi, att);
          items[q].tau = tau;
          items[q].taut = taut;
          PROF_SERIAL(tr0);
        }
      } else {
        if (warp == kNWarp - 1) eos_items();
        if (staged) {
          // psi by an online fp64 log-sum-exp, one lane per contender (the
          // sum runs in a different order from ctc_prefix.cpp:58; ~1e-15
          // relative)
          for (int q = (warp - nser) * 32 + lane; q < nc; q += (kNWarp - nser) * 32) {
            const int j = items[q].parent, c = items[q].token;
            const bool repeat = sh.b_last[cur][j] == c;
            const double* ph = repeat ? stR + (size_t)j * W : phi + (size_t)j * P.Tmax;
            const float* lc = stL + (size_t)q * W;
            double M = -HUGE_VAL, S = 0.0;
            for (int i = 0; i < W; ++i) {
              const double term = log_mul(ph[i], (double)lc[i]);
              if (!is_zero(term)) {
                const double ex = exp_neg(-fabs(term - M), tb);  // M = -inf: 0
                S = term > M ? fma(S, ex, 1.0) : S + ex;
                M = fmax(M, term);
              }
            }
            const double psi = M == -HUGE_VAL ? kLogZero : M + log_pos(S, tb);
            const double att = __dadd_rn(sh.b_att[cur][j],
                                         att_at(P, sh.b_row[cur][j], c));
            items[q].score = mix_joint(lam, psi, att);
          }
        }
      }
      gw0 = staged ? nser : 0;
      if (warp >= gw0) {
      group_sync(gw0);
      if (gw0 == 0) PROF_MARK(6);
      // ---- P7: exact order over contenders + eos (warp-ballot ranks) ----
      const int ni = nc + nb;
      for (int i = warp - gw0; i < ni; i += kNWarp - gw0) {
        const Item me = items[i < nc ? i : caps + (i - nc)];
        int rank = 0;
        for (int q0 = 0; q0 < ni; q0 += 32) {
          const int qq = q0 + lane;
          bool b = false;
          if (qq < ni) {
            const Item o = items[qq < nc ? qq : caps + (qq - nc)];
            b = before(o.score, o.parent, o.token, me.score, me.parent, me.token);
          }
          rank += __popc(__ballot_sync(0xffffffffu, b));
        }
        if (lane == 0 && rank < B + nb) {
          SelE x;
          x.score = me.score;
          x.parent = me.parent;
          x.token = me.token;
          x.slot = i < nc ? i : -1;
          x.tau = gw0 ? 0 : me.tau;  // chains may still run: patched after the join
          x.taut = gw0 ? 0 : me.taut;
          sh.sel[rank] = x;
        }
      }
      if (tid == gw0 * 32) sh.nsel = min(ni, B + nb);
      group_sync(gw0);
      if (gw0 == 0) PROF_MARK(7);
      }  // decision group
    } else if (BMAX >= 16 && !P.exact && sh.n_list <= list_cap(BMAX)) {
      // ---- P7w, wide step (beams of 13+): more contenders than chain slots
      // (caps), but the theta0 list of P5 is complete. Every candidate the
      // full fallback could select scores >= the B-th best exact non-eos
      // score >= theta (B listed candidates certainly reach theta), so it is
      // a listed key reaching theta, a repeat column or an eos candidate:
      // their exact fp64 scores (reference operation order, psi_only)
      // ranked with the fallback's comparator give the fallback's
      // selection. The children's states follow the walk (fallback tail).
      if (warp == kNWarp - 1) eos_items();
      Item* wi = reinterpret_cast<Item*>(P.xs + (size_t)u * xs_stride(B, C, BMAX));
      const int nl = sh.n_list;
      const float theta = fmaxf(sh.theta2, sh.theta);
      if (tid == 0) sh.n_cont = 0;
      __syncthreads();
      for (int i = tid; i < nl; i += kNT)
        if (clist[i].y >= theta) {
          const int idx = atomicAdd(&sh.n_cont, 1);
          wi[idx].parent = __float_as_int(clist[i].z);
          wi[idx].token = __float_as_int(clist[i].w);
        }
      if (warp == 0 && lane < nb && sh.b_last[cur][lane] >= 0) {
        const int idx = atomicAdd(&sh.n_cont, 1);  // repeat column
        wi[idx].parent = lane;
        wi[idx].token = sh.b_last[cur][lane];
      }
      __syncthreads();
      const int nw = sh.n_cont;
      for (int q = tid; q < nw; q += kNT) {
        const int j = wi[q].parent, c = wi[q].token;
        const double att = __dadd_rn(sh.b_att[cur][j], att_at(P, sh.b_row[cur][j], c));
        const double psi = lam <= 0.0 ? kLogZero
                                      : psi_only<BMAX>(P, sh, u, cur, j, c, s, e, grid,
                                                       phi + (size_t)j * P.Tmax, tb);
        wi[q].score = mix_joint(lam, psi, att);
      }
      if (tid < nb) wi[nw + tid] = items[caps + tid];  // eos, scored before the first barrier
      __syncthreads();
      const int ni = nw + nb;
      for (int i = tid; i < ni; i += kNT) {
        const Item me = wi[i];
        int rank = 0;
        for (int k = 0; k < ni && rank < B + nb; ++k) {
          const Item o = wi[k];
          rank += before(o.score, o.parent, o.token, me.score, me.parent, me.token) ? 1 : 0;
        }
        if (rank < B + nb) {
          SelE x;
          x.score = me.score;
          x.parent = me.parent;
          x.token = me.token;
          x.slot = -1;
          x.tau = x.taut = 0;
          sh.sel[rank] = x;
        }
      }
      if (tid == 0) {
        sh.nsel = min(ni, B + nb);
        sh.c_fallback += 1ull << 32;
      }
      __syncthreads();
      PROF_MARK(8);
    } else {
      // ---- fallback: fp64 scores for every candidate + exact selection ----
      if (warp == 0) eos_items();
      __syncthreads();
      double* xs = P.xs + (size_t)u * xs_stride(B, C, BMAX);
      unsigned char* taken = P.taken + (size_t)u * B * (C + 1);
      const int total = nb * (C + 1);
      for (int idx = tid; idx < total; idx += kNT) {
        const int j = idx / (C + 1), c = idx - j * (C + 1);
        double sc;
        if (c == C) {
          sc = items[caps + j].score;
        } else {
          const double att = __dadd_rn(sh.b_att[cur][j],
                                       att_at(P, sh.b_row[cur][j], c));
          const double psi = lam <= 0.0 ? kLogZero
                                        : psi_only<BMAX>(P, sh, u, cur, j, c, s, e, grid,
                                                         phi + (size_t)j * P.Tmax, tb);
          sc = mix_joint(lam, psi, att);
        }
        xs[idx] = sc;
        taken[idx] = 0;
      }
      if (tid == 0) {
        sh.nsel = 0;
        sh.c_fallback += 1;
      }
      __syncthreads();
      int non_eos = 0;
      for (int r = 0; r < total && non_eos < B; ++r) {
        double bs = 0.0;
        int bp = INT_MAX, bt = INT_MAX;
        for (int idx = tid; idx < total; idx += kNT) {
          if (taken[idx]) continue;
          const int j = idx / (C + 1), c = idx - j * (C + 1);
          if (bp == INT_MAX || before(xs[idx], j, c, bs, bp, bt)) {
            bs = xs[idx];
            bp = j;
            bt = c;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double os = __shfl_xor_sync(0xffffffffu, bs, o);
          const int op = __shfl_xor_sync(0xffffffffu, bp, o);
          const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
          if (op != INT_MAX && (bp == INT_MAX || before(os, op, ot, bs, bp, bt))) {
            bs = os;
            bp = op;
            bt = ot;
          }
        }
        if (lane == 0) {
          sh.red_s[warp] = bs;
          sh.red_p[warp] = bp;
          sh.red_t[warp] = bt;
        }
        __syncthreads();
        if (tid == 0) {
          double ws2 = sh.red_s[0];
          int wp = sh.red_p[0], wt = sh.red_t[0];
          for (int w = 1; w < kNWarp; ++w)
            if (sh.red_p[w] != INT_MAX &&
                (wp == INT_MAX || before(sh.red_s[w], sh.red_p[w], sh.red_t[w], ws2, wp, wt))) {
              ws2 = sh.red_s[w];
              wp = sh.red_p[w];
              wt = sh.red_t[w];
            }
          SelE x;
          x.score = ws2;
          x.parent = wp;
          x.token = wt;
          x.slot = -1;
          x.tau = x.taut = 0;
          sh.sel[sh.nsel++] = x;
          taken[(size_t)wp * (C + 1) + wt] = 1;
        }
        __syncthreads();
        non_eos += (sh.sel[sh.nsel - 1].token < C) ? 1 : 0;
      }
      PROF_MARK(8);
    }

    if (warp >= gw0) {
    const int gtid = tid - gw0 * 32;
    // ---- P8: walk (parallel): finished entries and children ----
    const int nsel = sh.nsel;
    if (gtid < nsel) {
      const SelE x = sh.sel[gtid];
      int non_eos_before = 0, eos_before = 0;
      for (int q = 0; q < gtid; ++q) {
        if (sh.sel[q].token < C) ++non_eos_before;
        else ++eos_before;
      }
      if (non_eos_before < B) {
        const int j = x.parent;
        if (x.token == C) {
          FinEntry f;
          f.joint = x.score;
          f.tau_last = sh.b_tau[cur][j];
          f.length = l;
          f.bp_step = l - 1;
          f.bp_slot = j;
          fin_u[sh.n_fin + eos_before] = f;
        } else {
          const int k = non_eos_before;
          const int c = x.token;
          sh.b_area[nxt][k] = nxt;
          sh.b_slot[nxt][k] = x.slot >= 0 ? x.slot : k;
          sh.b_vlo[nxt][k] = s;
          sh.b_cov[nxt][k] = e;
          sh.b_tau[nxt][k] = x.tau;
          sh.b_taut[nxt][k] = x.taut;
          sh.b_last[nxt][k] = c;
          sh.b_att[nxt][k] = __dadd_rn(sh.b_att[cur][j],
                                       att_at(P, sh.b_row[cur][j], c));
          sh.b_joint[nxt][k] = x.score;
          sh.b_row[nxt][k] = P.net_rows ? u * B + k : lookup_row(P, hist_c, l, l - 1, j, c);
          sh.child_q[k] = x.slot;
          HistRec h;
          h.token = c;
          h.parent = j;
          h.tau = x.tau;
          h.pad = 0;
          hist_u[(size_t)l * B + k] = h;
        }
      }
    }
    if (gtid == 0) {
      int ne = 0, ee2 = 0;
      for (int q = 0; q < nsel; ++q) {
        if (ne >= B) break;
        if (sh.sel[q].token < C) ++ne;
        else ++ee2;
      }
      sh.nchild = ne;
      sh.n_fin_new = ee2;
    }
    group_sync(gw0);
    if (gw0 == 0) PROF_MARK(9);
    if (step_fallback && gtid < sh.nchild) {
      // children states for the fallback path (slot k of area nxt)
      int k = gtid, cnt = 0, q = 0;
      for (; q < nsel; ++q) {
        if (sh.sel[q].token < C) {
          if (cnt == k) break;
          ++cnt;
        }
      }
      const SelE x = sh.sel[q];
      double* gnc = gam_ptr(P, u, nxt, k, 0);
      double* gbc = gnc + P.Tp;
      int tau, taut;
      child_recursion_global<BMAX>(P, sh, u, cur, x.parent, x.token, s, e, grid,
                                   phi + (size_t)x.parent * P.Tmax, gnc, gbc, &tau, &taut,
                                   tb);
      sh.b_tau[nxt][k] = tau;
      sh.b_taut[nxt][k] = taut;
      hist_u[(size_t)l * B + k].tau = tau;
    }

    // ---- P9: end detection (batched.cpp:215-228) ----
    if (gtid == 0) {
      const int n0 = sh.n_fin, nn = sh.n_fin_new;
      for (int q = n0; q < n0 + nn; ++q) {
        const FinEntry f = fin_u[q];
        if (f.joint > best_by_len[l]) best_by_len[l] = f.joint;
        if (f.joint > sh.best_all) sh.best_all = f.joint;
        if (f.tau_last == T) ++sh.count_long;
        if (sh.best_fin < 0 || f.joint > sh.best_fin_val) {
          sh.best_fin = q;
          sh.best_fin_val = f.joint;
        }
      }
      sh.n_fin = n0 + nn;
      sh.steps = l;
      sh.c_steps += 1;
      bool stop = false;
      if (P.eos_mode != 1 && sh.n_fin > 0) {  // end_detect_baseline
        bool ok = true;
        for (int m = 0; m < P.eos_m; ++m) {
          const int len = l - m;
          const double lb = len >= 1 ? best_by_len[len] : -HUGE_VAL;
          if (lb == -HUGE_VAL || !(lb - sh.best_all < P.eos_dend)) {
            ok = false;
            break;
          }
        }
        if (ok) {
          sh.trigger = 0;
          stop = true;
        }
      }
      if (!stop && P.eos_mode != 0 && sh.count_long > P.eos_c) {
        sh.trigger = 1;
        stop = true;
      }
      if (sh.nchild == 0) stop = true;
      sh.nb = sh.nchild;
      sh.done = stop ? 1 : 0;
      if (P.nb_out) P.nb_out[u] = stop ? 0 : sh.nchild;
    }
    }  // decision group
    __syncthreads();  // join: contender chains and decisions both done
    if (gw0 > 0 && tid < sh.nchild) {  // children's tau from their chains
      const Item& it = items[sh.child_q[tid]];
      sh.b_tau[nxt][tid] = it.tau;
      sh.b_taut[nxt][tid] = it.taut;
      hist_u[(size_t)l * B + tid].tau = it.tau;
    }
    // the patch is warp 0's (nchild <= BMAX <= 32) and only warp 0 reads
    // tau before the next block barrier (P1), so a warp barrier suffices
    // unless the state is saved now (step mode) or the search ends (end
    // detection, or the step bound: the next iteration breaks before P1 and
    // finalize reads the history with every warp)
    if (gw0 > 0) {
      if (stepm || sh.done || l >= ud.max_steps) __syncthreads();
      else __syncwarp();
    }
    PROF_MARK(10);
    if (sh.done) break;
    if (stepm) {
      // suspend: save the search state for step l + 1
      int* dst = reinterpret_cast<int*>(st_u + 16);
      const int* src = reinterpret_cast<const int*>(&sh);
      for (int i = tid; i < (int)(sizeof(Shared<BMAX>) / 4); i += kNT) dst[i] = src[i];
      double* sb = reinterpret_cast<double*>(st_u + 16 + align16(sizeof(Shared<BMAX>)));
      for (int i = tid; i <= P.S + 1; i += kNT) sb[i] = best_by_len[i];
      if (tid == 0) *reinterpret_cast<int*>(st_u) = 0;
      tmem_free();
      return;
    }
  }

  // ------------------------------------------------------------ finalize
  // batched.cpp:70-90: first max (strict >) over finished entries in
  // insertion order, else over the live beam with trigger = max_len.
  const int fcur = sh.steps & 1;  // beam after the last processed step
  int* res = P.res + (size_t)u * P.res_stride;
  const int S = P.S;
  // The back-pointer walks are serial pointer chases: stage the history in
  // shared memory first (packed {token, parent | tau << 16}) when it fits.
  const int nsteps = sh.steps;
  int2* hs = reinterpret_cast<int2*>(region);
  const bool hist_smem = (size_t)(nsteps + 1) * B * sizeof(int2) <= (size_t)P.region_bytes;
  if (hist_smem) {
    for (int idx = tid + B; idx < (nsteps + 1) * B; idx += kNT) {
      const HistRec h = hist_c[idx];
      hs[idx] = make_int2(h.token, h.parent | (h.tau << 16));
    }
  }
  __syncthreads();
  auto walk = [&](int bp_step, int bp_slot, int* tok, int* lt) {
    int k = bp_slot;
    for (int st = bp_step; st >= 1; --st) {
      int token, parent, tau;
      if (hist_smem) {
        const int2 h = hs[(size_t)st * B + k];
        token = h.x;
        parent = h.y & 0xffff;
        tau = h.y >> 16;
      } else {
        const HistRec h = hist_c[(size_t)st * B + k];
        token = h.token;
        parent = h.parent;
        tau = h.tau;
      }
      tok[st - 1] = token;
      lt[st - 1] = tau;
      k = parent;
    }
  };
  if (tid == 0) {
    int bp_step, bp_slot, trig = sh.trigger;
    double joint;
    if (sh.n_fin > 0) {
      const FinEntry f = fin_u[sh.best_fin];
      bp_step = f.bp_step;
      bp_slot = f.bp_slot;
      joint = f.joint;
    } else {
      int best = 0;
      for (int k = 1; k < sh.nb; ++k)
        if (sh.b_joint[fcur][k] > sh.b_joint[fcur][best]) best = k;
      bp_step = sh.steps;
      bp_slot = best;
      joint = sh.b_joint[fcur][best];
      trig = 2;
    }
    res[0] = bp_step;
    res[1] = sh.steps;
    res[2] = trig;
    res[3] = 0;
    reinterpret_cast<double*>(res + 4)[0] = joint;
    res[6] = sh.n_fin;
    res[7] = 0;
    walk(bp_step, bp_slot, res + kResHdr, res + kResHdr + S);
    unsigned long long* cn = P.cnt + (size_t)u * 8;
    cn[0] = sh.c_steps;
    cn[1] = sh.c_queries;
    cn[2] = sh.c_frames;
    cn[3] = sh.c_k1;
    cn[4] = sh.c_fallback;
    cn[5] = sh.c_cont;
    cn[6] = sh.c_raw;
    cn[7] = 0;
  }
  // n-best over finished entries: (joint desc, insertion asc)
  if (P.nbest > 0 && sh.n_fin > 0) {
    const int nf = sh.n_fin;
    const int want = min(P.nbest, nf);
    double last_s = HUGE_VAL;
    int last_i = -1;
    for (int r = 0; r < want; ++r) {
      // next entry strictly after (last_s, last_i) in the order
      double bs = -HUGE_VAL;
      int bi = INT_MAX;
      for (int q = tid; q < nf; q += kNT) {
        const double js = fin_u[q].joint;
        const bool after_last = (js < last_s) || (js == last_s && q > last_i);
        if (!after_last) continue;
        if (bi == INT_MAX || js > bs || (js == bs && q < bi)) {
          bs = js;
          bi = q;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi != INT_MAX && (bi == INT_MAX || os > bs || (os == bs && oi < bi))) {
          bs = os;
          bi = oi;
        }
      }
      if (lane == 0) {
        sh.red_s[warp] = bs;
        sh.red_p[warp] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        double ws2 = sh.red_s[0];
        int wi = sh.red_p[0];
        for (int w = 1; w < kNWarp; ++w) {
          const int oi = sh.red_p[w];
          const double os = sh.red_s[w];
          if (oi != INT_MAX && (wi == INT_MAX || os > ws2 || (os == ws2 && oi < wi))) {
            ws2 = os;
            wi = oi;
          }
        }
        const FinEntry f = fin_u[wi];
        int* nb_rec = res + kResHdr + 2 * S + r * (4 + 2 * S);
        nb_rec[0] = f.bp_step;
        nb_rec[1] = wi;
        reinterpret_cast<double*>(nb_rec + 2)[0] = f.joint;
        walk(f.bp_step, f.bp_slot, nb_rec + 4, nb_rec + 4 + S);
        res[3] = r + 1;
        sh.red_s[0] = ws2;
        sh.red_p[0] = wi;
      }
      __syncthreads();
      last_s = sh.red_s[0];
      last_i = sh.red_p[0];
      __syncthreads();
    }
  }
  __syncthreads();
  PROF_MARK(11);
  if (stepm && tid == 0) {
    *reinterpret_cast<int*>(st_u) = 1;
    atomicAdd(P.n_done, 1u);
  }
  tmem_free();
}

// ------------------------------------------------------------ launchers
// The kernel modes compile as separate translation units (Makefile:
// decode_kernel.cu with -DDK_MODE=0..4); each defines its mode's launcher
// over the beam instantiations, and mode 0's unit also holds the dispatch.
size_t decode_smem_bytes(const KParams& p);
int bmax_for(int B);

static int mode_of(const KParams& p) {
  return p.use_tc == 2 ? 4 : p.use_tc == 1 ? 3 : p.use_tma ? 2 : (p.kub_smem ? 0 : 1);
}

template <int BMAX, int kMode>
static cudaError_t launch_v(const KParams& p, cudaStream_t st) {
  const size_t sm = decode_smem_bytes(p);
  cudaError_t err = cudaFuncSetAttribute(decode_kernel<BMAX, kMode>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm);
  if (err != cudaSuccess) {
    if (std::getenv("BL_DEBUG"))
      std::fprintf(stderr, "[bl] decode_kernel<%d,%d>: set max dynamic smem %zu: %s\n", BMAX,
                   kMode, sm, cudaGetErrorString(err));
    return err;
  }
  if (std::getenv("BL_DEBUG")) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, decode_kernel<BMAX, kMode>, kNT, sm);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, decode_kernel<BMAX, kMode>);
    size_t avail2 = 0;
    cudaOccupancyAvailableDynamicSMemPerBlock(&avail2, decode_kernel<BMAX, kMode>, 2, kNT);
    cudaGetLastError();  // fails for tcgen05 kernels (one CTA per SM): not a launch error
    std::fprintf(stderr, "[bl] decode_kernel<%d,%d>: grid %d, dyn smem %zu, static %zu, regs %d, "
                 "local %zu, max threads %d, %d CTA/SM (dyn smem available at 2 CTA/SM: %zu)\n",
                 BMAX, kMode, p.U, sm, fa.sharedSizeBytes, fa.numRegs, fa.localSizeBytes,
                 fa.maxThreadsPerBlock, nb, avail2);
  }
  decode_kernel<BMAX, kMode><<<p.U, kNT, sm, st>>>(p);
  err = cudaGetLastError();
  if (err != cudaSuccess && std::getenv("BL_DEBUG"))
    std::fprintf(stderr, "[bl] decode_kernel<%d,%d>: launch of %d CTAs, %zu B dynamic smem: %s\n",
                 BMAX, kMode, p.U, sm, cudaGetErrorString(err));
  return err;
}

template <int BMAX, int kMode>
static size_t static_v() {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, decode_kernel<BMAX, kMode>);
  return fa.sharedSizeBytes;
}

// launcher / static shared memory of mode DK_MODE for beam capacity `bmax`
#define BL_MODE_FNS(M)                                                              \
  cudaError_t launch_mode##M(int bmax, const KParams& p, cudaStream_t st) {         \
    switch (bmax) {                                                                 \
      case 4: return launch_v<4, M>(p, st);                                         \
      case 8: return launch_v<8, M>(p, st);                                         \
      case 10: return launch_v<10, M>(p, st);                                       \
      case 12: return launch_v<12, M>(p, st);                                       \
      case 16: return launch_v<16, M>(p, st);                                       \
      BL_WIDE_CASES(M)                                                              \
    }                                                                               \
    return cudaErrorInvalidValue;                                                   \
  }                                                                                 \
  size_t static_mode##M(int bmax) {                                                 \
    switch (bmax) {                                                                 \
      case 4: return static_v<4, M>();                                              \
      case 8: return static_v<8, M>();                                              \
      case 10: return static_v<10, M>();                                            \
      case 12: return static_v<12, M>();                                            \
      case 16: return static_v<16, M>();                                            \
      BL_WIDE_STATIC(M)                                                             \
    }                                                                               \
    return 0;                                                                       \
  }

cudaError_t launch_mode0(int, const KParams&, cudaStream_t);
cudaError_t launch_mode1(int, const KParams&, cudaStream_t);
cudaError_t launch_mode2(int, const KParams&, cudaStream_t);
cudaError_t launch_mode3(int, const KParams&, cudaStream_t);
cudaError_t launch_mode4(int, const KParams&, cudaStream_t);
size_t static_mode0(int);
size_t static_mode1(int);
size_t static_mode2(int);
size_t static_mode3(int);
size_t static_mode4(int);

#if DK_MODE >= 3  // the tensor-core bulks hold at most 16 parents
#define BL_WIDE_CASES(M)
#define BL_WIDE_STATIC(M)
#else
#define BL_WIDE_CASES(M)                      \
  case 24: return launch_v<24, M>(p, st);     \
  case 32: return launch_v<32, M>(p, st);
#define BL_WIDE_STATIC(M)              \
  case 24: return static_v<24, M>();   \
  case 32: return static_v<32, M>();
#endif

#if DK_MODE == 0
BL_MODE_FNS(0)
#elif DK_MODE == 1
BL_MODE_FNS(1)
#elif DK_MODE == 2
BL_MODE_FNS(2)
#elif DK_MODE == 3
BL_MODE_FNS(3)
#elif DK_MODE == 4
BL_MODE_FNS(4)
#else
#error "compile decode_kernel.cu with -DDK_MODE=0..4"
#endif

#if DK_MODE == 0
int bmax_for(int B) {
  if (B <= 4) return 4;
  if (B <= 8) return 8;
  if (B <= 10) return 10;  // the bench / paper beam: no padded parents in P3
  if (B <= 12) return 12;
  if (B <= 16) return 16;
  if (B <= 24) return 24;
  if (B <= 32) return 32;
  return 0;
}

// per-utterance step-mode state: {done flag, pad}[16 B], Shared<BMAX>, best_by_len[S+2]
size_t step_state_bytes(int B, int S) {
  size_t sh = 0;
  switch (bmax_for(B)) {
    case 4: sh = sizeof(Shared<4>); break;
    case 8: sh = sizeof(Shared<8>); break;
    case 10: sh = sizeof(Shared<10>); break;
    case 12: sh = sizeof(Shared<12>); break;
    case 16: sh = sizeof(Shared<16>); break;
    case 24: sh = sizeof(Shared<24>); break;
    default: sh = sizeof(Shared<32>); break;
  }
  return align16(16 + align16(sh) + sizeof(double) * (size_t)(S + 2));
}

size_t decode_smem_bytes(const KParams& p) {
  return smem_plan(p.Tmax, p.B, bmax_for(p.B), p.C, p.caps, p.S, p.region_bytes, p.kub_smem,
                   p.tma_stages, p.use_tc).total;
}

// static shared memory of the kernel variant `p` selects
size_t decode_static_smem(const KParams& p) {
  const int b = bmax_for(p.B);
  switch (mode_of(p)) {
    case 4: return b <= 16 ? static_mode4(b) : 0;
    case 3: return b <= 16 ? static_mode3(b) : 0;
    case 2: return static_mode2(b);
    case 1: return static_mode1(b);
    default: return static_mode0(b);
  }
}

cudaError_t launch_decode(const KParams& p, cudaStream_t st) {
  const int b = bmax_for(p.B);
  if (b == 0) return cudaErrorInvalidValue;
  switch (mode_of(p)) {
    case 4: return b <= 16 ? launch_mode4(b, p, st) : cudaErrorInvalidValue;
    case 3: return b <= 16 ? launch_mode3(b, p, st) : cudaErrorInvalidValue;
    case 2: return launch_mode2(b, p, st);
    case 1: return launch_mode1(b, p, st);
    default: return launch_mode0(b, p, st);
  }
}
#endif

}  // namespace bl
