/* ctc_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference decoding path of beamlattice
 * (/root/reference/proj). Every function names the reference file:line it
 * restates. The arithmetic is kept in the reference's order (fp64, the same
 * log_add / log_mul sequence) so that, linked against the same libm, results
 * are bit-identical to the compiled reference (pinned by
 * tests/test_oracle.py against oracle/_ref and tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define K_LOG_ZERO (-1e30)      /* logmath.hpp:11 */
#define K_LOG_ZERO_GUARD (-1e29) /* logmath.hpp:14 */
#define K_NO_MARGIN (1 << 29)   /* ctc_prefix.hpp:12 */

static int is_log_zero(double x) { return x <= K_LOG_ZERO_GUARD; } /* logmath.hpp:16 */

/* logmath.hpp:19-23 */
double orc_log_add(double a, double b) {
  if (a < b) {
    double t = a;
    a = b;
    b = t;
  }
  if (is_log_zero(b)) return is_log_zero(a) ? K_LOG_ZERO : a;
  return a + log1p(exp(b - a));
}

/* logmath.hpp:26-29 */
double orc_log_mul(double a, double b) {
  if (is_log_zero(a) || is_log_zero(b)) return K_LOG_ZERO;
  return a + b;
}

/* logmath.hpp:34-39 */
double orc_mix_joint(double lambda, double ctc, double att) {
  if (lambda <= 0.0) return att;
  if (lambda >= 1.0) return ctc;
  if (is_log_zero(ctc) || is_log_zero(att)) return K_LOG_ZERO;
  return lambda * ctc + (1.0 - lambda) * att;
}

/* grid.hpp:36-38: 1-based frame, promoted to double */
static double at(const float* g, int V, int t, int k) {
  return (double)g[(size_t)(t - 1) * V + k];
}

/* ctc_prefix.cpp:106-114 */
void orc_window_for(int tau, int tau_tilde, int m1, int m2, int step, int T,
                    int* s_out, int* e_out) {
  long s = (long)tau - m1;
  if ((long)step > s) s = step;
  if (1L > s) s = 1;
  long e = (long)tau_tilde + m2;
  if ((long)T < e) e = T;
  if (s > e) s = e;
  *s_out = (int)s;
  *e_out = (int)e;
}

/* ctc_prefix.cpp:10-26 */
int orc_init_state(int T, int V, const float* grid, orc_state* st) {
  if (T < 1) return -1;
  for (int t = 0; t <= T; ++t) {
    st->gamma_n[t] = K_LOG_ZERO;
    st->gamma_b[t] = K_LOG_ZERO;
  }
  st->gamma_b[0] = 0.0;
  const int blank = V - 1;
  for (int t = 1; t <= T; ++t)
    st->gamma_b[t] = orc_log_mul(st->gamma_b[t - 1], at(grid, V, t, blank));
  st->covered = T;
  st->tau = 1;
  st->tau_tilde = 1;
  st->prefix_len = 0;
  st->last_label = -1;
  return 0;
}

/* ctc_prefix.cpp:28-79 */
int orc_prefix_score_step(const orc_state* st, int c, int T, int V,
                          const float* grid, int s, int e, double* psi_out,
                          orc_state* next) {
  const int blank = V - 1;
  if (c < 0 || c >= V - 1) return -1;
  if (s < 1 || e > T || s > e) return -2;
  for (int t = 0; t <= T; ++t) {
    next->gamma_n[t] = K_LOG_ZERO;
    next->gamma_b[t] = K_LOG_ZERO;
  }
  next->prefix_len = st->prefix_len + 1;
  next->last_label = c;
  next->covered = e;
  const int repeat = st->last_label == c;
  double psi = K_LOG_ZERO;
  for (int t = s; t <= e; ++t) {
    double phi = repeat ? st->gamma_b[t - 1]
                        : orc_log_add(st->gamma_b[t - 1], st->gamma_n[t - 1]);
    const double p_c = at(grid, V, t, c);
    next->gamma_n[t] = orc_log_mul(orc_log_add(next->gamma_n[t - 1], phi), p_c);
    next->gamma_b[t] = orc_log_mul(
        orc_log_add(next->gamma_b[t - 1], next->gamma_n[t - 1]),
        at(grid, V, t, blank));
    psi = orc_log_add(psi, orc_log_mul(phi, p_c));
  }
  const int lo = st->tau > 1 ? st->tau : 1;
  int best_n = lo, best_b = lo;
  double val_n = K_LOG_ZERO, val_b = K_LOG_ZERO;
  for (int t = lo; t <= e; ++t) {
    if (next->gamma_n[t] > val_n) {
      val_n = next->gamma_n[t];
      best_n = t;
    }
    if (next->gamma_b[t] > val_b) {
      val_b = next->gamma_b[t];
      best_b = t;
    }
  }
  next->tau = best_n;
  next->tau_tilde = best_b;
  *psi_out = psi;
  return 0;
}

/* ctc_prefix.cpp:88-104 */
double orc_eos_score_extended(const orc_state* st, int T, int V,
                              const float* grid) {
  const int blank = V - 1;
  double gn = st->gamma_n[st->covered];
  double gb = st->gamma_b[st->covered];
  for (int t = st->covered + 1; t <= T; ++t) {
    double gn_next = st->last_label >= 0
                         ? orc_log_mul(gn, at(grid, V, t, st->last_label))
                         : K_LOG_ZERO;
    gb = orc_log_mul(orc_log_add(gb, gn), at(grid, V, t, blank));
    gn = gn_next;
  }
  return orc_log_add(gn, gb);
}

/* ------------------------------------------------------------------ */
/* Scorer (scorer.cpp:30-80). The table lookup is TableScorer::score
 * (scorer.cpp:53-62): context = last min(|prefix|, order-1) tokens, exact
 * match, uniform fallback. */

static void scorer_row(const orc_scorer* sc, const int* prefix, int len,
                       double* out) {
  const int V = sc->num_tokens + 1;
  if (sc->kind == 2) { /* scorer.cpp:73-80 */
    double rest = log((1.0 - sc->p_loop) / sc->num_tokens);
    for (int k = 0; k < V; ++k) out[k] = rest;
    out[sc->loop_token] = log(sc->p_loop);
    return;
  }
  if (sc->kind == 1) {
    const int w = sc->order - 1 > 0 ? sc->order - 1 : 1;
    int n = len < sc->order - 1 ? len : sc->order - 1;
    for (int k = 0; k < sc->n_entries; ++k) {
      if (sc->ctx_len[k] != n) continue;
      if (n == 0 ||
          memcmp(sc->ctx + (size_t)k * w, prefix + len - n, sizeof(int) * n) == 0) {
        memcpy(out, sc->logp + (size_t)k * V, sizeof(double) * V);
        return;
      }
    }
  }
  /* scorer.cpp:34-38 */
  double u = -log((double)(sc->num_tokens + 1));
  for (int k = 0; k < V; ++k) out[k] = u;
}

/* ------------------------------------------------------------------ */
/* Hypotheses / finished entries (beam_search.hpp:44-66) */

typedef struct hyp {
  int* tokens;
  int* label_times;
  int n;
  double att_logp, ctc_logp, joint;
  orc_state fwd;
} hyp;

typedef struct fin {
  int* tokens;
  int* label_times;
  int n;
  double joint;
  int tau_last, length;
} fin;

typedef struct cand { /* beam_search.cpp:114-125 */
  double score;
  int parent, token, is_eos;
} cand;

static int cand_cmp(const void* pa, const void* pb) {
  const cand* a = (const cand*)pa;
  const cand* b = (const cand*)pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  if (a->parent != b->parent) return a->parent < b->parent ? -1 : 1;
  if (a->token != b->token) return a->token < b->token ? -1 : 1;
  return 0;
}

typedef struct utt_search { /* batched.cpp:58-68 */
  int T, max_steps, steps, trigger, done;
  const float* grid;
  hyp* beam;
  int nbeam;
  fin* finished;
  int nfin, capfin;
  /* per-step scores (StepScores, beam_search.hpp:83-89) */
  double* token_joint; /* [nbeam * C] */
  double* token_psi;
  orc_state* token_state; /* [nbeam * C] */
  double* att;            /* [nbeam * V] */
  double* eos_joint;      /* [nbeam] */
  int s, e;
} utt_search;

static double* dalloc(size_t n) { return (double*)malloc(sizeof(double) * (n ? n : 1)); }

static void state_alloc(orc_state* st, int T) {
  st->gamma_n = dalloc(T + 1);
  st->gamma_b = dalloc(T + 1);
}
static void state_free(orc_state* st) {
  free(st->gamma_n);
  free(st->gamma_b);
}

/* end_detect_baseline (beam_search.cpp:81-99) */
static int end_detect_baseline(const utt_search* s, int step, int eos_m,
                               double eos_dend) {
  if (s->nfin == 0) return 0;
  double best = -HUGE_VAL;
  for (int k = 0; k < s->nfin; ++k)
    if (s->finished[k].joint > best) best = s->finished[k].joint;
  for (int m = 0; m < eos_m; ++m) {
    int len = step - m;
    double len_best = -HUGE_VAL;
    int seen = 0;
    for (int k = 0; k < s->nfin; ++k)
      if (s->finished[k].length == len) {
        seen = 1;
        if (s->finished[k].joint > len_best) len_best = s->finished[k].joint;
      }
    if (!seen || !(len_best - best < eos_dend)) return 0;
  }
  return 1;
}

/* joint_step_scores (beam_search.cpp:48-79) for hypothesis j of s */
static void joint_step(utt_search* s, int j, int V, const orc_scorer* sc,
                       const orc_config* cfg, orc_counters* cnt) {
  const int C = V - 1;
  hyp* h = &s->beam[j];
  double* att = s->att + (size_t)j * V;
  scorer_row(sc, h->tokens, h->n, att);
  for (int c = 0; c < C; ++c) {
    orc_state* ns = &s->token_state[(size_t)j * C + c];
    double psi;
    orc_prefix_score_step(&h->fwd, c, s->T, V, s->grid, s->s, s->e, &psi, ns);
    s->token_psi[(size_t)j * C + c] = psi;
    s->token_joint[(size_t)j * C + c] =
        orc_mix_joint(cfg->ctc_weight, psi, h->att_logp + att[c]);
  }
  double eos_ctc = orc_eos_score_extended(&h->fwd, s->T, V, s->grid);
  s->eos_joint[j] = orc_mix_joint(cfg->ctc_weight, eos_ctc, h->att_logp + att[C]);
  cnt->scorer_queries += 1;
  cnt->ctc_frames_evaluated += (uint64_t)C * (uint64_t)(s->e - s->s + 1);
  if (h->fwd.covered < s->T)
    cnt->ctc_frames_evaluated += (uint64_t)(s->T - h->fwd.covered);
}

static int* icopy(const int* src, int n, int extra) {
  int* p = (int*)malloc(sizeof(int) * (size_t)(n + extra + 1));
  if (n) memcpy(p, src, sizeof(int) * n);
  return p;
}

/* Pooled ranking + refill + end detection for one utterance-step
 * (batched.cpp:164-229; serial twin beam_search.cpp:190-227). */
static void reduce_step(utt_search* s, int l, int V, const orc_config* cfg,
                        orc_counters* cnt) {
  const int C = V - 1;
  s->steps = l;
  cnt->steps += 1;
  int ncand = s->nbeam * (C + 1);
  cand* cs = (cand*)malloc(sizeof(cand) * ncand);
  int k = 0;
  for (int j = 0; j < s->nbeam; ++j) {
    for (int c = 0; c < C; ++c) {
      cs[k].score = s->token_joint[(size_t)j * C + c];
      cs[k].parent = j;
      cs[k].token = c;
      cs[k].is_eos = 0;
      ++k;
    }
    cs[k].score = s->eos_joint[j];
    cs[k].parent = j;
    cs[k].token = C;
    cs[k].is_eos = 1;
    ++k;
  }
  qsort(cs, ncand, sizeof(cand), cand_cmp); /* total order: no equal keys */

  hyp* next = (hyp*)calloc(cfg->beam_width, sizeof(hyp));
  int nnext = 0;
  for (int q = 0; q < ncand; ++q) {
    const cand* cd = &cs[q];
    hyp* h = &s->beam[cd->parent];
    if (cd->is_eos) {
      if (s->nfin == s->capfin) {
        s->capfin = s->capfin ? 2 * s->capfin : 16;
        s->finished = (fin*)realloc(s->finished, sizeof(fin) * s->capfin);
      }
      fin* f = &s->finished[s->nfin++];
      f->tokens = icopy(h->tokens, h->n, 0);
      f->label_times = icopy(h->label_times, h->n, 0);
      f->n = h->n;
      f->joint = cd->score;
      f->tau_last = h->fwd.tau;
      f->length = h->n + 1;
      continue;
    }
    hyp* ch = &next[nnext];
    ch->tokens = icopy(h->tokens, h->n, 1);
    ch->tokens[h->n] = cd->token;
    ch->n = h->n + 1;
    ch->att_logp = h->att_logp + s->att[(size_t)cd->parent * V + cd->token];
    ch->ctc_logp = s->token_psi[(size_t)cd->parent * C + cd->token];
    ch->joint = cd->score;
    orc_state* src = &s->token_state[(size_t)cd->parent * C + cd->token];
    ch->fwd = *src;
    src->gamma_n = NULL; /* moved */
    src->gamma_b = NULL;
    ch->label_times = icopy(h->label_times, h->n, 1);
    ch->label_times[h->n] = ch->fwd.tau;
    ++nnext;
    if (nnext >= cfg->beam_width) break;
  }
  free(cs);
  for (int j = 0; j < s->nbeam; ++j) {
    free(s->beam[j].tokens);
    free(s->beam[j].label_times);
    state_free(&s->beam[j].fwd);
  }
  free(s->beam);
  for (size_t q = 0; q < (size_t)s->nbeam * C; ++q) state_free(&s->token_state[q]);
  s->beam = next;
  s->nbeam = nnext;

  if (cfg->eos_mode != 1 && end_detect_baseline(s, l, cfg->eos_m, cfg->eos_dend)) {
    s->trigger = 0;
    s->done = 1;
  } else if (cfg->eos_mode != 0) {
    int count_long = 0;
    for (int q = 0; q < s->nfin; ++q)
      if (s->finished[q].tau_last == s->T) ++count_long;
    if (count_long > cfg->eos_c) {
      s->trigger = 1;
      s->done = 1;
    }
  }
  if (s->nbeam == 0) s->done = 1;
}

typedef struct rset {
  int n;
  orc_result* r;
  fin** nb;  /* per utterance: the finished set sorted (joint desc, insertion asc) */
  int* nnb;
} rset;

/* n-best = the finished set in (joint desc, insertion asc) order: the
 * entries finalize_result (batched.cpp:70-90) chooses from, ranked; the head
 * is finalize's choice (first max in insertion order). Stable insertion sort. */
static fin* sorted_finished(const utt_search* s) {
  fin* out = (fin*)malloc(sizeof(fin) * (size_t)(s->nfin > 0 ? s->nfin : 1));
  for (int k = 0; k < s->nfin; ++k) {
    fin f = s->finished[k];
    f.tokens = icopy(f.tokens, f.n, 0);
    f.label_times = icopy(f.label_times, f.n, 0);
    int j = k - 1;
    while (j >= 0 && out[j].joint < f.joint) {
      out[j + 1] = out[j];
      --j;
    }
    out[j + 1] = f;
  }
  return out;
}

/* finalize_result (batched.cpp:70-90) */
static void finalize(const utt_search* s, orc_result* out) {
  out->steps = s->steps;
  out->eos_trigger = s->trigger;
  if (s->nfin > 0) {
    const fin* best = &s->finished[0];
    for (int k = 0; k < s->nfin; ++k)
      if (s->finished[k].joint > best->joint) best = &s->finished[k];
    out->n_tokens = best->n;
    out->tokens = icopy(best->tokens, best->n, 0);
    out->label_times = icopy(best->label_times, best->n, 0);
    out->joint_logp = best->joint;
  } else {
    const hyp* best = &s->beam[0];
    for (int k = 0; k < s->nbeam; ++k)
      if (s->beam[k].joint > best->joint) best = &s->beam[k];
    out->n_tokens = best->n;
    out->tokens = icopy(best->tokens, best->n, 0);
    out->label_times = icopy(best->label_times, best->n, 0);
    out->joint_logp = best->joint;
    out->eos_trigger = 2;
  }
}

static void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    strncpy(err, msg, errlen - 1);
    err[errlen - 1] = 0;
  }
}

/* DecoderConfig::validate (beam_search.cpp:36-46) */
static const char* validate(const orc_config* c) {
  if (c->beam_width < 1) return "beam width must be >= 1";
  if (c->ctc_weight < 0.0 || c->ctc_weight > 1.0) return "ctc weight must be in [0, 1]";
  if (c->eos_m < 1) return "eos M must be >= 1";
  if (c->eos_c < 0) return "eos C must be >= 0";
  if (c->margin_m1 < 0 || c->margin_m2 < 0) return "margins must be >= 0";
  if (!(c->max_steps_ratio > 0.0 && c->max_steps_ratio <= 1.0))
    return "max steps ratio must be in (0, 1]";
  return NULL;
}

/* Alg. 2 over one batch (batched.cpp:94-237) when batched != 0 — all
 * utterances step in lock-step exactly as the reference loop does — else
 * serial Alg. 1 per utterance (beam_search.cpp:155-248). Both produce the
 * same per-utterance results; the two loops are kept for fidelity. */
void* orc_decode(int n, const int* frames, int V, const float* const* grids,
                 const orc_scorer* sc, const orc_config* cfg, int batched,
                 orc_counters* counters, char* err, int errlen) {
  const char* bad = validate(cfg);
  if (bad) {
    set_err(err, errlen, bad);
    return NULL;
  }
  const int C = V - 1;
  utt_search* ss = (utt_search*)calloc(n ? n : 1, sizeof(utt_search));
  for (int i = 0; i < n; ++i) {
    utt_search* s = &ss[i];
    if (frames[i] < 1) {
      char buf[96];
      snprintf(buf, sizeof buf, "empty grid in utterance %d", i);
      set_err(err, errlen, buf);
      free(ss);
      return NULL;
    }
    if (sc->num_tokens != C) {
      set_err(err, errlen, "scorer vocabulary mismatch");
      free(ss);
      return NULL;
    }
    s->T = frames[i];
    s->grid = grids[i];
    s->max_steps = (int)ceil(cfg->max_steps_ratio * s->T);
    s->trigger = 2;
    s->beam = (hyp*)calloc(1, sizeof(hyp));
    s->nbeam = 1;
    s->beam[0].tokens = icopy(NULL, 0, 0);
    s->beam[0].label_times = icopy(NULL, 0, 0);
    state_alloc(&s->beam[0].fwd, s->T);
    orc_init_state(s->T, V, s->grid, &s->beam[0].fwd);
  }
  orc_counters total = {0, 0, 0};
  const int W = cfg->beam_width;
  int active = n;
  int l = 1;
  /* serial mode: run each utterance to completion; batched: lock-step */
  for (int i0 = 0; i0 < (batched ? 1 : n) && active > 0; ++i0) {
    int lo = batched ? 0 : i0, hi = batched ? n : i0 + 1;
    for (l = 1;; ++l) {
      int any = 0;
      for (int i = lo; i < hi; ++i) {
        utt_search* s = &ss[i];
        if (s->done) continue;
        if (l > s->max_steps) {
          s->done = 1;
          continue;
        }
        s->s = 0x7fffffff;
        s->e = -0x7fffffff;
        for (int j = 0; j < s->nbeam; ++j) { /* batched.cpp:129-135 */
          int ws, we;
          orc_window_for(s->beam[j].fwd.tau, s->beam[j].fwd.tau_tilde,
                         cfg->margin_m1, cfg->margin_m2, l, s->T, &ws, &we);
          if (j == 0 || ws < s->s) s->s = ws;
          if (j == 0 || we > s->e) s->e = we;
        }
        s->token_joint = dalloc((size_t)s->nbeam * C);
        s->token_psi = dalloc((size_t)s->nbeam * C);
        s->token_state = (orc_state*)malloc(sizeof(orc_state) * (size_t)s->nbeam * C);
        for (size_t q = 0; q < (size_t)s->nbeam * C; ++q) state_alloc(&s->token_state[q], s->T);
        s->att = dalloc((size_t)s->nbeam * V);
        s->eos_joint = dalloc((size_t)s->nbeam);
        for (int j = 0; j < s->nbeam; ++j) joint_step(s, j, V, sc, cfg, &total);
        any = 1;
      }
      if (!any) break;
      for (int i = lo; i < hi; ++i) {
        utt_search* s = &ss[i];
        if (s->done || !s->token_joint) continue;
        reduce_step(s, l, V, cfg, &total);
        free(s->token_joint);
        free(s->token_psi);
        free(s->token_state);
        free(s->att);
        free(s->eos_joint);
        s->token_joint = NULL;
      }
    }
  }
  (void)W;
  rset* rs = (rset*)malloc(sizeof(rset));
  rs->n = n;
  rs->r = (orc_result*)calloc(n ? n : 1, sizeof(orc_result));
  rs->nb = (fin**)calloc(n ? n : 1, sizeof(fin*));
  rs->nnb = (int*)calloc(n ? n : 1, sizeof(int));
  for (int i = 0; i < n; ++i) {
    utt_search* s = &ss[i];
    finalize(s, &rs->r[i]);
    rs->nb[i] = sorted_finished(s);
    rs->nnb[i] = s->nfin;
    for (int j = 0; j < s->nbeam; ++j) {
      free(s->beam[j].tokens);
      free(s->beam[j].label_times);
      state_free(&s->beam[j].fwd);
    }
    free(s->beam);
    for (int k = 0; k < s->nfin; ++k) {
      free(s->finished[k].tokens);
      free(s->finished[k].label_times);
    }
    free(s->finished);
  }
  free(ss);
  if (counters) *counters = total;
  return rs;
}

int orc_results_count(void* h) { return ((rset*)h)->n; }
void orc_results_get(void* h, int i, orc_result* out) { *out = ((rset*)h)->r[i]; }
int orc_results_nbest(void* h, int i, int k, orc_result* out) {
  const rset* rs = (const rset*)h;
  if (k < 0 || k >= rs->nnb[i]) return rs->nnb[i];
  const fin* f = &rs->nb[i][k];
  out->n_tokens = f->n;
  out->tokens = f->tokens;
  out->label_times = f->label_times;
  out->joint_logp = f->joint;
  out->steps = f->length;
  out->eos_trigger = f->tau_last;
  return rs->nnb[i];
}

void orc_results_free(void* h) {
  rset* rs = (rset*)h;
  for (int i = 0; i < rs->n; ++i) {
    free((void*)rs->r[i].tokens);
    free((void*)rs->r[i].label_times);
    for (int k = 0; k < rs->nnb[i]; ++k) {
      free(rs->nb[i][k].tokens);
      free(rs->nb[i][k].label_times);
    }
    free(rs->nb[i]);
  }
  free(rs->nb);
  free(rs->nnb);
  free(rs->r);
  free(rs);
}

/* make_batches (batched.cpp:12-30): stable ascending sort by true_frames. */
int orc_make_batches(int n, const uint32_t* frames, int batch_size, int* order) {
  if (batch_size < 1) return -1;
  for (int i = 0; i < n; ++i) order[i] = i;
  for (int i = 1; i < n; ++i) { /* insertion sort is stable */
    int v = order[i], j = i - 1;
    while (j >= 0 && frames[order[j]] > frames[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
  return (n + batch_size - 1) / batch_size;
}

/* split_uniform (segmentation.cpp:65-75) */
static int split_uniform(int start, int end, int max_len, int* starts, int* ends,
                         int cap, int k0) {
  const int len = end - start;
  const int pieces = (len + max_len - 1) / max_len;
  int offset = start;
  for (int k = 0; k < pieces; ++k) {
    int piece = len / pieces + (k < len % pieces ? 1 : 0);
    if (k0 + k < cap) {
      starts[k0 + k] = offset;
      ends[k0 + k] = offset + piece;
    }
    offset += piece;
  }
  return pieces;
}

/* hard_segments (segmentation.cpp:121-133) */
int orc_hard_segments(int T, int min_len, int max_len, int* starts, int* ends,
                      int cap) {
  if (T < 1) return -1;
  if (!(min_len > 0 && min_len <= max_len)) return -1;
  if (T < min_len) {
    if (cap > 0) {
      starts[0] = 0;
      ends[0] = T;
    }
    return 1;
  }
  return split_uniform(0, T, max_len, starts, ends, cap, 0);
}
