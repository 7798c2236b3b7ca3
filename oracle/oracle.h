/* oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Declarations for the two CPU checkers under oracle/:
 *   - liboracle.so   : plain-C restatement of the reference decoding path
 *                      (oracle/ctc_oracle.c, every function cites the
 *                      reference file:line it restates);
 *   - _ref/libblref.so: the UNMODIFIED reference (beamlattice, C++20)
 *                      compiled in place from /root/reference/proj/src plus
 *                      the extern "C" shim oracle/ref_shim.cpp.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries, and only as the checker or
 * the CPU baseline — never as the product path.
 */
#ifndef BL_ORACLE_H
#define BL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors beamlattice::DecoderConfig (beam_search.hpp:21-33).
 * eos_mode: 0 baseline, 1 ctc, 2 both. margin = 1<<29 means "inf". */
typedef struct orc_config {
  int beam_width;
  double ctc_weight;
  int eos_m;
  double eos_dend;
  int eos_c;
  int margin_m1;
  int margin_m2;
  int eos_mode;
  double max_steps_ratio;
} orc_config;

/* Scorer description (scorer.hpp:24-70).
 * kind 0: UniformScorer; 1: TableScorer (order, entries); 2: LoopScorer. */
typedef struct orc_scorer {
  int kind;
  int num_tokens;         /* |C| */
  int order;              /* table only */
  int n_entries;          /* table only */
  const int* ctx_len;     /* [n_entries] */
  const int* ctx;         /* [n_entries * max(order-1,1)] */
  const double* logp;     /* [n_entries * (num_tokens+1)] */
  int loop_token;         /* loop only */
  double p_loop;          /* loop only */
  /* replay only (kind 3, oracle/_ref): entry k belongs to utterance
   * replay_ids[ent_utt[k]]; its full prefix is ctx[k*(order-1) ..] */
  const int* ent_utt;
  const char* const* replay_ids;
} orc_scorer;

typedef struct orc_counters {
  uint64_t steps;
  uint64_t scorer_queries;
  uint64_t ctc_frames_evaluated;
} orc_counters;

/* One decoded utterance (DecodeResult, beam_search.hpp:35-42).
 * eos_trigger: 0 baseline, 1 ctc, 2 max_len. Arrays owned by the result set. */
typedef struct orc_result {
  int n_tokens;
  const int* tokens;
  const int* label_times;
  double joint_logp;
  int steps;
  int eos_trigger;
} orc_result;

/* ----------------------------- C restatement --------------------------- */

typedef struct orc_state {   /* CtcForwardState, ctc_prefix.hpp:26-34 */
  double* gamma_n;           /* [T+1] */
  double* gamma_b;           /* [T+1] */
  int covered, tau, tau_tilde, prefix_len, last_label;
} orc_state;

double orc_log_add(double a, double b);
double orc_log_mul(double a, double b);
double orc_mix_joint(double lambda, double ctc, double att);
void orc_window_for(int tau, int tau_tilde, int m1, int m2, int step, int T,
                    int* s, int* e);
/* grid: T x V row-major float log-probs, blank = V-1. Caller owns arrays
 * of size T+1 inside the states. */
int orc_init_state(int T, int V, const float* grid, orc_state* out);
int orc_prefix_score_step(const orc_state* st, int c, int T, int V,
                          const float* grid, int s, int e, double* psi,
                          orc_state* next);
double orc_eos_score_extended(const orc_state* st, int T, int V,
                              const float* grid);

/* Serial Alg. 1 per utterance (beam_search.cpp:155-248) or batched Alg. 2
 * over one batch (batched.cpp:94-237). grids[i] is frames[i] x V.
 * Returns a result-set handle (NULL on error, message in err). */
void* orc_decode(int n, const int* frames, int V, const float* const* grids,
                 const orc_scorer* scorer, const orc_config* cfg,
                 int batched, orc_counters* counters, char* err, int errlen);
int orc_results_count(void* h);
void orc_results_get(void* h, int i, orc_result* out);
void orc_results_free(void* h);
/* Entry k of utterance i's finished set in (joint desc, insertion asc) order
 * (the n-best list; steps = entry length incl. eos, eos_trigger = tau_last).
 * Returns the number of finished entries. */
int orc_results_nbest(void* h, int i, int k, orc_result* out);

/* make_batches (batched.cpp:12-30): writes the stable length-sorted order
 * into order[n] and returns the number of batches (chunks of batch_size). */
int orc_make_batches(int n, const uint32_t* frames, int batch_size, int* order);
/* hard_segments (segmentation.cpp:121-133); returns the number of segments
 * or -1 on invalid arguments. */
int orc_hard_segments(int T, int min_len, int max_len, int* starts, int* ends,
                      int cap);

/* ------------------------ compiled reference shim ---------------------- */

void* ref_synth_corpus(uint64_t seed, int num_utts, int t_min, int t_max,
                       int num_tokens, const char* style, double blank_mass,
                       uint32_t frame_shift_ms);
void* ref_random_corpus(uint64_t seed, int n, int t_lo, int t_hi,
                        int num_tokens);
int ref_corpus_count(void* h);
int ref_corpus_frames(void* h, int i);
int ref_corpus_vocab(void* h, int i);
const float* ref_corpus_logp(void* h, int i);
const char* ref_corpus_id(void* h, int i);
void ref_corpus_free(void* h);

/* mode 0: run_decode semantics with batch_size (<=1 -> serial beam_search,
 * else make_batches + batched_beam_search); results in INPUT order.
 * threads > 0 sets omp_set_num_threads. */
void* ref_decode(int n, const char* const* ids, const int* frames, int V,
                 const float* const* grids, const orc_scorer* scorer,
                 const orc_config* cfg, int batch_size, int threads,
                 orc_counters* counters, char* err, int errlen);
int ref_results_count(void* h);
void ref_results_get(void* h, int i, orc_result* out);
void ref_results_free(void* h);

int ref_hard_segments(int T, int min_len, int max_len, int* starts, int* ends,
                      int cap);
/* Chained full-window prefix scores along `prefix` (verify.cpp:39-52):
 * psi_out[k] = psi after prefix[0..k]; also tau/tau_tilde per step. */
int ref_chain_prefix(int T, int V, const float* grid, int n, const int* prefix,
                     int s_override, int e_override, double* psi_out,
                     int* tau_out, int* tau_tilde_out, double* eos_ext_out);
int ref_verify(const char* suite, int trials, int max_frames, int max_vocab,
               uint64_t seed);
int ref_num_threads(void);

#ifdef __cplusplus
}
#endif

#endif
