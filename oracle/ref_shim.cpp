// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" face over the UNMODIFIED reference decoder (beamlattice), which
// oracle/Makefile compiles in place from /root/reference/proj/src into
// oracle/_ref/libblref.so. Used by tests/ as the ground-truth checker and by
// bench.py as the CPU baseline ("kind": "reference"). No reference source is
// copied; this file only marshals arguments.
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <exception>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "beamlattice/batched.hpp"
#include "beamlattice/beam_search.hpp"
#include "beamlattice/ctc_prefix.hpp"
#include "beamlattice/scorer.hpp"
#include "beamlattice/segmentation.hpp"
#include "beamlattice/synth.hpp"
#include "beamlattice/verify.hpp"
#include "beamlattice/io.hpp"
#include "oracle.h"

using namespace beamlattice;

namespace {

struct Corpus {
  std::vector<Utterance> utts;
};

struct ResultSet {
  std::vector<DecodeResult> results;
};

void set_err(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

// Replays the rows a device network scorer produced, keyed by (utterance id,
// full prefix): the reference decoder then searches with exactly the device's
// attention scores. A query the device never answered is a divergence; it is
// counted (score() runs inside the reference's OpenMP workers, so it must not
// throw) and answered with the uniform row.
std::atomic<long long> g_replay_misses{0};

class ReplayScorer : public Scorer {
 public:
  explicit ReplayScorer(int n) : n_(n) {}
  int num_tokens() const override { return n_; }
  std::vector<double> score(const std::string& id,
                            const std::vector<int>& prefix) const override {
    auto it = table_.find({id, prefix});
    if (it != table_.end()) return it->second;
    ++g_replay_misses;
    return std::vector<double>(n_ + 1, -std::log(static_cast<double>(n_ + 1)));
  }
  void add(const std::string& id, std::vector<int> prefix, std::vector<double> row) {
    check_normalized(row, static_cast<size_t>(n_) + 1, "replayed scorer row");
    table_[{id, std::move(prefix)}] = std::move(row);
  }

 private:
  int n_;
  std::map<std::pair<std::string, std::vector<int>>, std::vector<double>> table_;
};

std::unique_ptr<Scorer> build_scorer(const orc_scorer* s) {
  if (s->kind == 0) return std::make_unique<UniformScorer>(s->num_tokens);
  if (s->kind == 3) {
    auto r = std::make_unique<ReplayScorer>(s->num_tokens);
    const int w = s->order - 1 > 0 ? s->order - 1 : 1;
    for (int k = 0; k < s->n_entries; ++k) {
      std::vector<int> ctx(s->ctx + (size_t)k * w, s->ctx + (size_t)k * w + s->ctx_len[k]);
      std::vector<double> lp(s->logp + (size_t)k * (s->num_tokens + 1),
                             s->logp + (size_t)(k + 1) * (s->num_tokens + 1));
      r->add(s->replay_ids[s->ent_utt[k]], std::move(ctx), std::move(lp));
    }
    return r;
  }
  if (s->kind == 2)
    return std::make_unique<LoopScorer>(s->num_tokens, s->loop_token,
                                        s->p_loop);
  auto t = std::make_unique<TableScorer>(s->num_tokens, s->order);
  const int w = s->order - 1 > 0 ? s->order - 1 : 1;
  for (int k = 0; k < s->n_entries; ++k) {
    std::vector<int> ctx(s->ctx + (size_t)k * w,
                         s->ctx + (size_t)k * w + s->ctx_len[k]);
    std::vector<double> lp(s->logp + (size_t)k * (s->num_tokens + 1),
                           s->logp + (size_t)(k + 1) * (s->num_tokens + 1));
    t->add_entry(ctx, lp);
  }
  return t;
}

DecoderConfig to_cfg(const orc_config* c) {
  DecoderConfig cfg;
  cfg.beam_width = c->beam_width;
  cfg.ctc_weight = c->ctc_weight;
  cfg.eos_m = c->eos_m;
  cfg.eos_dend = c->eos_dend;
  cfg.eos_c = c->eos_c;
  cfg.margin_m1 = c->margin_m1;
  cfg.margin_m2 = c->margin_m2;
  cfg.eos_mode = c->eos_mode == 0   ? EosMode::kBaseline
                 : c->eos_mode == 1 ? EosMode::kCtc
                                    : EosMode::kBoth;
  cfg.max_steps_ratio = c->max_steps_ratio;
  return cfg;
}

}  // namespace

extern "C" {

void* ref_synth_corpus(uint64_t seed, int num_utts, int t_min, int t_max,
                       int num_tokens, const char* style, double blank_mass,
                       uint32_t frame_shift_ms) {
  try {
    SynthConfig sc;
    sc.seed = seed;
    sc.num_utts = num_utts;
    sc.t_min = t_min;
    sc.t_max = t_max;
    sc.num_tokens = num_tokens;
    sc.style = style;
    sc.blank_mass = blank_mass;
    sc.frame_shift_ms = frame_shift_ms;
    auto* c = new Corpus;
    for (const auto& s : synth_corpus(sc))
      c->utts.push_back({s.id, s.grid, s.grid.num_frames});
    return c;
  } catch (...) {
    return nullptr;
  }
}

// acceptance.cpp:59-72 / test_batched.cpp:13-25 corpus shape.
void* ref_random_corpus(uint64_t seed, int n, int t_lo, int t_hi,
                        int num_tokens) {
  std::mt19937_64 rng(seed);
  auto* c = new Corpus;
  for (int i = 0; i < n; ++i) {
    Utterance u;
    u.id = "r" + std::to_string(i);
    const int t = std::uniform_int_distribution<int>(t_lo, t_hi)(rng);
    u.grid = random_grid(rng, t, num_tokens);
    u.true_frames = u.grid.num_frames;
    c->utts.push_back(std::move(u));
  }
  return c;
}

int ref_corpus_count(void* h) { return (int)((Corpus*)h)->utts.size(); }
int ref_corpus_frames(void* h, int i) {
  return (int)((Corpus*)h)->utts[i].grid.num_frames;
}
int ref_corpus_vocab(void* h, int i) {
  return (int)((Corpus*)h)->utts[i].grid.vocab;
}
const float* ref_corpus_logp(void* h, int i) {
  return ((Corpus*)h)->utts[i].grid.logp.data();
}
const char* ref_corpus_id(void* h, int i) {
  return ((Corpus*)h)->utts[i].id.c_str();
}
void ref_corpus_free(void* h) { delete (Corpus*)h; }

// Same control flow as run_decode (tools/beamlattice.cpp:117-146).
void* ref_decode(int n, const char* const* ids, const int* frames, int V,
                 const float* const* grids, const orc_scorer* scorer,
                 const orc_config* ccfg, int batch_size, int threads,
                 orc_counters* counters, char* err, int errlen) {
  try {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    std::vector<Utterance> utts(n);
    for (int i = 0; i < n; ++i) {
      utts[i].id = ids[i];
      utts[i].grid.num_frames = (uint32_t)frames[i];
      utts[i].grid.vocab = (uint32_t)V;
      utts[i].grid.logp.assign(grids[i], grids[i] + (size_t)frames[i] * V);
      utts[i].true_frames = (uint32_t)frames[i];
    }
    auto sc = build_scorer(scorer);
    DecoderConfig cfg = to_cfg(ccfg);
    DecodeCounters cnt;
    std::vector<DecodeResult> raw;
    if (batch_size <= 1) {
      for (const auto& u : utts) raw.push_back(beam_search(u, *sc, cfg, &cnt));
    } else {
      for (const auto& b : make_batches(utts, batch_size)) {
        auto rs = batched_beam_search(b, *sc, cfg, &cnt);
        raw.insert(raw.end(), std::make_move_iterator(rs.begin()),
                   std::make_move_iterator(rs.end()));
      }
    }
    auto* out = new ResultSet;
    for (const auto& u : utts)
      for (auto& r : raw)
        if (r.id == u.id) {
          out->results.push_back(std::move(r));
          break;
        }
    if (counters) {
      counters->steps = cnt.steps;
      counters->scorer_queries = cnt.scorer_queries;
      counters->ctc_frames_evaluated = cnt.ctc_frames_evaluated;
    }
    return out;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

int ref_results_count(void* h) { return (int)((ResultSet*)h)->results.size(); }
void ref_results_get(void* h, int i, orc_result* out) {
  const DecodeResult& r = ((ResultSet*)h)->results[i];
  out->n_tokens = (int)r.tokens.size();
  out->tokens = r.tokens.data();
  out->label_times = r.label_times.data();
  out->joint_logp = r.joint_logp;
  out->steps = r.steps_taken;
  out->eos_trigger = r.eos_trigger == EosTrigger::kBaseline ? 0
                     : r.eos_trigger == EosTrigger::kCtc    ? 1
                                                            : 2;
}
void ref_results_free(void* h) { delete (ResultSet*)h; }

int ref_hard_segments(int T, int min_len, int max_len, int* starts, int* ends,
                      int cap) {
  try {
    auto segs = hard_segments(T, min_len, max_len, "u");
    for (size_t k = 0; k < segs.size() && (int)k < cap; ++k) {
      starts[k] = segs[k].start;
      ends[k] = segs[k].end;
    }
    return (int)segs.size();
  } catch (...) {
    return -1;
  }
}

// Chains prefix_score_step along `prefix` from init_state; the window is the
// full grid unless overrides (>0) are given. Returns 0 or -1 on exception.
int ref_chain_prefix(int T, int V, const float* grid, int n, const int* prefix,
                     int s_override, int e_override, double* psi_out,
                     int* tau_out, int* tau_tilde_out, double* eos_ext_out) {
  try {
    PosteriorGrid g;
    g.num_frames = (uint32_t)T;
    g.vocab = (uint32_t)V;
    g.logp.assign(grid, grid + (size_t)T * V);
    CtcForwardState st = init_state(g);
    Window w{s_override > 0 ? s_override : 1, e_override > 0 ? e_override : T};
    if (eos_ext_out) eos_ext_out[0] = eos_score_extended(st, g);
    for (int k = 0; k < n; ++k) {
      auto [psi, next] = prefix_score_step(st, prefix[k], g, w);
      psi_out[k] = psi;
      if (tau_out) tau_out[k] = next.tau;
      if (tau_tilde_out) tau_tilde_out[k] = next.tau_tilde;
      st = std::move(next);
      if (eos_ext_out) eos_ext_out[k + 1] = eos_score_extended(st, g);
    }
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_verify(const char* suite, int trials, int max_frames, int max_vocab,
               uint64_t seed) {
  std::string s(suite);
  SuiteResult r;
  if (s == "oracle") r = verify_oracle_equivalence(trials, max_frames, max_vocab, seed);
  else if (s == "partition") r = verify_partition_identity(trials, max_frames, max_vocab, seed);
  else if (s == "exhaustive") r = verify_exhaustive_beam(trials, seed);
  else return -1;
  return r.failures;
}

int ref_vad_segments(const float* outputs, int T, int num_nodes, const int* speech,
                     int n_speech, const int* noise, int n_noise, double threshold,
                     int smooth_window, int min_len, int max_len, int* starts, int* ends,
                     int cap, char* err, int errlen) {
  try {
    NodeMap nm;
    nm.speech_nodes.assign(speech, speech + n_speech);
    nm.noise_nodes.assign(noise, noise + n_noise);
    std::vector<double> llr(T);
    for (int t = 0; t < T; ++t) {
      std::vector<double> row(outputs + (size_t)t * num_nodes,
                              outputs + (size_t)(t + 1) * num_nodes);
      llr[t] = frame_llr(row, nm);
    }
    auto flags = smooth_and_decide(llr, threshold, smooth_window);
    auto segs = vad_segments(flags, min_len, max_len, "r");
    for (size_t i = 0; i < segs.size() && (int)i < cap; ++i) {
      starts[i] = segs[i].start;
      ends[i] = segs[i].end;
    }
    return (int)segs.size();
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return -1;
  }
}

long long ref_replay_misses(int reset) {
  const long long m = g_replay_misses.load();
  if (reset) g_replay_misses = 0;
  return m;
}

int ref_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// One result line through the reference's own writer (io.cpp:81-92):
// golden bytes for the drop-in JSONL writers. Returns the length, or -1.
int ref_result_json(const char* id, const int* tokens, int n_tokens, double joint,
                    const int* label_times, int n_lt, int steps, int trigger, char* out,
                    int cap) {
  try {
    DecodeResult r;
    r.id = id;
    r.tokens.assign(tokens, tokens + n_tokens);
    r.joint_logp = joint;
    r.label_times.assign(label_times, label_times + n_lt);
    r.steps_taken = steps;
    r.eos_trigger = trigger == 0 ? EosTrigger::kBaseline
                    : trigger == 1 ? EosTrigger::kCtc
                                   : EosTrigger::kMaxLen;
    std::ostringstream os;
    write_results(os, {r});
    const std::string s = os.str();
    if ((int)s.size() >= cap) return -1;
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = 0;
    return (int)s.size();
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
