// decode.cuh — device data layout shared by the decode kernel and the host
// planner (capi.cu). See DESIGN.md "Data layout in HBM".
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bl {

constexpr int kNT = 256;             // threads per CTA (one CTA per utterance)
constexpr int kNWarp = kNT / 32;
constexpr double kLogZero = -1e30;   // logmath.hpp:11
constexpr double kLogZeroGuard = -1e29;  // logmath.hpp:14

// Per-utterance descriptor.
struct UttDesc {
  const float* grid;  // T x V row-major fp32 log-posteriors, blank = V-1
  int T;
  int max_steps;      // ceil(max_steps_ratio * T), batched.cpp:112-113
  int need_tail;      // margin_m2 < T: eos tails need the F/G tables
  int row0;           // first row of this utterance in the TMA tensor map
  int chunk;          // streamed host input: the copy chunk holding this grid
};

// Finished (eos-ended) entry, FinishedEntry (beam_search.hpp:53-61) with a
// back-pointer instead of copied token/label_times vectors.
struct FinEntry {
  double joint;
  int tau_last;
  int length;
  int bp_step;  // parent hypothesis = (step, slot) in the history
  int bp_slot;
};

// Token history record for beam slot k at step l (parent pointer form of
// Hypothesis::tokens / label_times, beam_search.hpp:44-51).
struct HistRec {
  int token;
  int parent;
  int tau;
  int pad;
};

// TMA streaming of the CTC window slab (large vocabularies): 512-column tiles
// (two columns per thread) x kTmaRows-row chunks, kTmaStagesMax stages; a
// stage is 8 warp slices of kTmaRows x kTmaBoxCols (each warp streams its own
// 64 columns). The tensor-core variant uses the same 16 KB stages as 16
// swizzle blocks of 8 rows x 32 columns, and a factor operand of 512 B per
// 8-row chunk.
constexpr int kTmaBoxCols = 64;
constexpr int kTmaRows = 8;
constexpr int kTmaStagesMax = 10;
constexpr int kSlabRows = 16;  // rows per slab job of the TMA filter mode (kMode 2)
constexpr int kTmaStageBytes = 8 * kTmaRows * kTmaBoxCols * 4;

struct KParams {
  CUtensorMap tmap;  // TMA map over all utterances' grid rows: 2D [sum T][V] (fp32),
                     // or with use_tc 3D {32 cols, sum T rows, V/32 column blocks}
                     // with 32-byte-atom 128-byte swizzle (the MN-major tf32
                     // operand layout of tcgen05.mma)
  int use_tma, tma_stages;
  int use_tc;        // tensor-core bulk: 1 = tcgen05.mma kind::tf32 (TMEM), 2 = mma.sync
                     // m16n8k8 tf32 (registers), see decode_kernel.cu
  float* mshift;     // use_tc: [2][U][mshift_stride] per-column exp shifts by step parity
  int mshift_stride;
  const UttDesc* utts;
  int U, V, C, B;
  int u0;          // first utterance of this launch (chunked launches)
  int Tmax;        // max T over the batch
  int Tp;          // stride of one gamma array (>= Tmax + 1)
  int S;           // max max_steps over the batch
  int caps;        // contender states per area (3B + 16)
  // DecoderConfig
  double lambda;
  double eos_dend;
  int eos_m, eos_c, m1, m2, eos_mode;
  float guard_f;   // largest float f with (double)f <= -1e29
  int exact;       // fp64-decision mode: every candidate by the fp64 path
  int nbest;
  double dpsi0, dpsi1;  // certified psi half-width = dpsi0 + W * dpsi1
  // device scorer (Uniform / Table / Loop as a table of rows)
  int sc_order;    // n-gram order (1 = context free)
  int sc_nent;     // entries, sorted by (len, tokens)
  int sc_w;        // max(order-1, 1)
  const int* sc_ctx_len;
  const int* sc_ctx;
  const int* sc_row;     // row of entry k
  const double* sc_rows; // [rows][V]; row 0 = uniform fallback
  const float* sc_rowsf;  // [rows][V]: (float)((1-lambda)*row), -inf where row is log-zero
  // network scorer with the fused log-softmax: rows are logits [rows][V]
  // (fp32) minus net_lse[row] (fp64); sc_rows / sc_rowsf unused then
  const float* net_logits;
  const double* net_lse;
  // workspace (per-utterance slices)
  double* gam;     // [U][2][caps][2][Tp]
  double* Ftab;    // [U][Tp][C]   eos tail tables (need_tail only)
  double* Gtab;    // [U][Tp]
  int kub_smem;    // 1: every upper key lives in shared memory (P5 scans them);
                   // 0: keys are filtered on chip against a running bound
                   // while P3 emits them (raw list, kRawCap entries)
  int region_bytes;  // aliased smem region (see smem_plan)
  double* xs;      // [U][xs_stride(B, C, bmax)]  exact joints (fallback) / wide-step items
  unsigned char* taken;  // [U][B][C+1]
  HistRec* hist;   // [U][S+1][B]
  FinEntry* fin;   // [U][B*S]
  int* res;        // [U][res_stride]
  int res_stride;
  unsigned long long* cnt;  // [U][8]
  long long* prof;          // [U][16] phase cycles, or nullptr
  // step-granular mode (a network scorer runs between steps): step_l > 0
  // runs exactly step l of every live utterance, restoring / saving the
  // per-utterance search state (`state`, state_stride bytes each); finished
  // utterances bump *n_done once.
  int step_l;
  int state_stride;
  unsigned char* state;
  unsigned* n_done;
  // per-hypothesis scorer rows (network scorer): hypothesis k of utterance u
  // reads row u * B + k of sc_rows / sc_rowsf at every step
  int net_rows;
  int* rec_nb;  // optional [U][S+2]: live beam size at the start of each step
  int* nb_out;  // optional [U]: live beam size entering the next step (0 once finished)
  // streamed host input: the CTA of utterance u starts once
  // ready[utts[u].chunk] == ready_epoch (written by the copy stream after
  // that chunk's grids); a chunk that never arrives sets *stream_err
  const unsigned* ready;
  unsigned ready_epoch;
  int* stream_err;
};

// Dynamic shared-memory plan (identical on host and device).
constexpr int kListCap = 256;  // keys reaching theta0 (P5), 16 B each
constexpr int kRawCap = 512;   // keys reaching the running bound during P3 (filter mode)
// Beams of 13+ (BMAX >= 16) on flat posteriors list many more keys: larger
// lists there (the theta0 list lives in the TMA stage area), and the wide
// step (decode_kernel.cu P7w) instead of the full fallback when the
// contenders outnumber the chain slots.
__host__ __device__ constexpr int list_cap(int bmax) { return bmax >= 16 ? 1024 : kListCap; }
__host__ __device__ constexpr int raw_cap(int bmax) { return bmax >= 16 ? 2048 : kRawCap; }
// per-utterance stride (doubles) of KParams::xs: the fallback's B x (|C|+1)
// joints, or the wide step's items (listed contenders, repeat columns, eos:
// 24 B each)
__host__ __device__ inline long long xs_stride(int B, int C, int bmax) {
  const long long a = (long long)B * (C + 1), b = 3LL * (list_cap(bmax) + 2 * bmax);
  return bmax >= 16 && b > a ? b : a;  // wide steps only at BMAX >= 16
}

struct SmemPlan {
  size_t phi, region, items, bbl, total;
  size_t phif, kub, ubits, clist, raw, stages, region_need;  // P3-P5 view of `region`
};
constexpr int kItemBytes = 24;  // score(double) + parent, token, tau, taut
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
// region_bytes: size of the aliased region (P3-P5: fp32 factors, upper keys,
// underflow flags, theta0 list; P6: contender staging with stride W). The
// host sizes it so the whole plan fits 3 CTAs per SM when possible.
constexpr int kTcChunkBytes = 512;  // factor operand per 8-row chunk: 16 parents x 8 tf32
__host__ __device__ inline SmemPlan smem_plan(int Tmax, int B, int bmax, int C, int caps,
                                              int S, size_t region_bytes, int kub_smem,
                                              int tma_stages = 0, int tc = 0) {
  SmemPlan p;
  p.phi = 0;
  p.region = align16(p.phi + sizeof(double) * (size_t)B * Tmax);
  p.phif = 0;
  // P3 factors: fp32 [Tmax][bmax] rows, or (tensor cores) the K-major tf32
  // operand, one 512 B chunk per 8 rows
  // (tc: 1 = tcgen05 operand layout, 2 = mma.sync: fp32 rows, 1024-B aligned ring)
  p.kub = tc == 1 ? (size_t)kTcChunkBytes * (size_t)((Tmax + 7) / 8)
                  : align16(sizeof(float) * (size_t)Tmax * bmax);
  const size_t words = ((size_t)B * C + 31) / 32;
  p.ubits = kub_smem ? align16(p.kub + sizeof(float) * (size_t)B * C) : p.kub;
  if (kub_smem) {  // keys mode: every key, its flag, then the theta0 list
    p.clist = align16(p.ubits + sizeof(unsigned) * words);
    p.raw = p.clist + 16 * (size_t)list_cap(bmax);
    p.stages = p.raw;
    p.region_need = p.raw;
  } else {
    // filter mode: the raw list (8 B per key: upper key + packed index),
    // then the TMA stages, 128-byte aligned in absolute shared-memory offset
    // (cp.async.bulk.tensor dst); the theta0 list is built after P3, so with
    // TMA it takes the stage area, else it follows the raw list
    p.raw = p.kub;
    const size_t raw_end = p.raw + 8 * (size_t)raw_cap(bmax);
    p.stages = ((p.region + raw_end + 127) & ~(size_t)127) - p.region;
    if (tc) p.stages += 1024;  // the kernel aligns the stage ring to 1024 B (swizzle atoms)
    if (tma_stages) {
      p.clist = p.stages;
      p.region_need = p.stages + (size_t)tma_stages * kTmaStageBytes;
    } else {
      p.clist = align16(raw_end);
      p.region_need = p.clist + 16 * (size_t)list_cap(bmax);
    }
  }
  p.items = align16(p.region + region_bytes);
  p.bbl = align16(p.items + (size_t)kItemBytes * (caps + bmax));
  p.total = align16(p.bbl + sizeof(double) * (size_t)(S + 2));
  return p;
}

// Result record layout (ints) per utterance.
constexpr int kResHdr = 8;
__host__ __device__ inline int res_stride(int S, int nbest) {
  return kResHdr + 2 * S + nbest * (4 + 2 * S);
}

}  // namespace bl
