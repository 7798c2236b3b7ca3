// decode.cuh — device data layout shared by the decode kernel and the host
// planner (capi.cu). See DESIGN.md "Data layout in HBM".
#pragma once
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
  int pad;
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

struct KParams {
  const UttDesc* utts;
  int U, V, C, B;
  int Tmax;        // max T over the batch
  int Tp;          // stride of one gamma array (>= Tmax + 1)
  int S;           // max max_steps over the batch
  int caps;        // contender states per area (2B + 16)
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
  // workspace (per-utterance slices)
  double* gam;     // [U][2][caps][2][Tp]
  double* Ftab;    // [U][Tp][C]   eos tail tables (need_tail only)
  double* Gtab;    // [U][Tp]
  float2* keys;    // [U][B][C]    certified (lo, ub) joint keys
  double* xs;      // [U][B][C+1]  exact joints (fallback path)
  unsigned char* taken;  // [U][B][C+1]
  HistRec* hist;   // [U][S+1][B]
  FinEntry* fin;   // [U][B*S]
  int* res;        // [U][res_stride]
  int res_stride;
  unsigned long long* cnt;  // [U][8]
};

// Result record layout (ints) per utterance.
constexpr int kResHdr = 8;
__host__ __device__ inline int res_stride(int S, int nbest) {
  return kResHdr + 2 * S + nbest * (4 + 2 * S);
}

}  // namespace bl
