// beamlattice/b200.hpp — C++ drop-in for the reference decoding API
// (/root/reference/proj/include/beamlattice/{grid,scorer,beam_search,batched,
// segmentation}.hpp) implemented over the C ABI (include/bl_b200.h).
//
// Same names, types, argument meaning and exception types as the reference,
// so a caller of beamlattice::batched_beam_search recompiles against this
// header and links libbl_b200.so. Decoding runs on the GPU (device 0, or
// $BL_DEVICE); there is no CPU fallback. Scorers are device scorers: the
// reference's Uniform/Table/Loop scorers and make_scorer specs.
#pragma once

#include <cstdint>
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <ostream>
#include <sstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../bl_b200.h"

namespace beamlattice {

inline constexpr double kLogZero = -1e30;  // logmath.hpp:11
inline constexpr int kNoMargin = BL_NO_MARGIN;  // ctc_prefix.hpp:12

namespace detail {
inline void check(int rc) {
  if (rc == BL_OK) return;
  const std::string msg = bl_last_error();
  if (rc == BL_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == BL_LOGIC_ERROR) throw std::logic_error(msg);
  throw std::runtime_error(msg);
}
inline int device() {
  const char* d = std::getenv("BL_DEVICE");
  return d ? std::atoi(d) : 0;
}
}  // namespace detail

// grid.hpp:24-55
struct PosteriorGrid {
  uint32_t num_frames = 0;
  uint32_t vocab = 0;
  uint32_t frame_shift_ms = 10;
  std::vector<float> logp;
  int num_tokens() const { return static_cast<int>(vocab) - 1; }
  int blank_id() const { return static_cast<int>(vocab) - 1; }
  double at(int frame, int symbol) const {
    return logp[static_cast<size_t>(frame - 1) * vocab + symbol];
  }
  double audio_seconds() const { return num_frames * frame_shift_ms / 1000.0; }
};

struct Utterance {
  std::string id;
  PosteriorGrid grid;
  uint32_t true_frames = 0;
};

// beam_search.hpp:14-79
enum class EosMode { kBaseline, kCtc, kBoth };
enum class EosTrigger { kBaseline, kCtc, kMaxLen };

inline const char* to_string(EosMode m) {
  return m == EosMode::kBaseline ? "baseline" : m == EosMode::kCtc ? "ctc" : "both";
}
inline const char* to_string(EosTrigger t) {
  return t == EosTrigger::kBaseline ? "baseline" : t == EosTrigger::kCtc ? "ctc" : "max_len";
}
inline EosMode eos_mode_from_string(const std::string& s) {
  if (s == "baseline") return EosMode::kBaseline;
  if (s == "ctc") return EosMode::kCtc;
  if (s == "both") return EosMode::kBoth;
  throw std::invalid_argument("unknown eos mode: " + s);
}

struct DecoderConfig {
  int beam_width = 3;
  double ctc_weight = 0.3;
  int eos_m = 3;
  double eos_dend = -10.0;
  int eos_c = 2;
  int margin_m1 = 5;
  int margin_m2 = kNoMargin;
  EosMode eos_mode = EosMode::kBoth;
  double max_steps_ratio = 1.0;

  bl_config c() const {
    return bl_config{beam_width, ctc_weight, eos_m, eos_dend, eos_c, margin_m1, margin_m2,
                     static_cast<int>(eos_mode), max_steps_ratio};
  }
  void validate() const {
    const bl_config cc = c();
    detail::check(bl_config_validate(&cc));
  }
};

struct DecodeResult {
  std::string id;
  std::vector<int> tokens;
  double joint_logp = 0.0;
  std::vector<int> label_times;
  int steps_taken = 0;
  EosTrigger eos_trigger = EosTrigger::kMaxLen;
};

struct DecodeCounters {
  uint64_t steps = 0;
  uint64_t scorer_queries = 0;
  uint64_t ctc_frames_evaluated = 0;
  DecodeCounters& operator+=(const DecodeCounters& o) {
    steps += o.steps;
    scorer_queries += o.scorer_queries;
    ctc_frames_evaluated += o.ctc_frames_evaluated;
    return *this;
  }
};

// scorer.hpp:11-84 — device scorers
class Scorer {
 public:
  virtual ~Scorer() { bl_scorer_destroy(h_); }
  int num_tokens() const { return bl_scorer_num_tokens(h_); }
  std::vector<double> score(const std::string&, const std::vector<int>& prefix) const {
    std::vector<double> out(num_tokens() + 1);
    detail::check(bl_scorer_score(h_, prefix.data(), static_cast<int>(prefix.size()),
                                  out.data()));
    return out;
  }
  const bl_scorer* handle() const { return h_; }

 protected:
  bl_scorer* h_ = nullptr;
};

class UniformScorer : public Scorer {
 public:
  explicit UniformScorer(int num_tokens) {
    detail::check(bl_scorer_create("uniform", num_tokens, &h_));
  }
};

class LoopScorer : public Scorer {
 public:
  LoopScorer(int num_tokens, int loop_token, double p_loop) {
    detail::check(bl_scorer_create_loop(num_tokens, loop_token, p_loop, &h_));
  }
};

class TableScorer : public Scorer {
 public:
  TableScorer(int num_tokens, int order) : n_(num_tokens), order_(order) { rebuild(); }
  int order() const { return order_; }
  void add_entry(const std::vector<int>& context, std::vector<double> logp) {
    auto old = table_;
    table_[context] = std::move(logp);
    try {
      rebuild();
    } catch (...) {
      table_ = std::move(old);
      throw;
    }
  }
  const std::map<std::vector<int>, std::vector<double>>& entries() const { return table_; }

 private:
  void rebuild() {
    const int w = order_ - 1 > 0 ? order_ - 1 : 1;
    std::vector<int> len, ctx;
    std::vector<double> lp;
    for (const auto& [c, v] : table_) {
      len.push_back(static_cast<int>(c.size()));
      for (int i = 0; i < w; ++i) ctx.push_back(i < (int)c.size() ? c[i] : 0);
      if (v.size() != static_cast<size_t>(n_) + 1)
        throw std::runtime_error("TableScorer entry: wrong vector size");
      lp.insert(lp.end(), v.begin(), v.end());
    }
    bl_scorer* h = nullptr;
    detail::check(bl_scorer_create_table(n_, order_, static_cast<int>(len.size()), len.data(),
                                         ctx.data(), lp.data(), &h));
    bl_scorer_destroy(h_);
    h_ = h;
  }
  int n_, order_;
  std::map<std::vector<int>, std::vector<double>> table_;
};

namespace detail {
class SpecScorer : public Scorer {
 public:
  SpecScorer(const std::string& spec, int n) {
    detail::check(bl_scorer_create(spec.c_str(), n, &h_));
  }
};
}  // namespace detail

inline std::unique_ptr<Scorer> make_scorer(const std::string& spec, int num_tokens) {
  return std::make_unique<detail::SpecScorer>(spec, num_tokens);
}

// segmentation.hpp:45-65
struct Segment {
  std::string utterance_id;
  int start = 0;
  int end = 0;
  std::string source;
};

inline std::vector<Segment> hard_segments(int num_frames, int min_len, int max_len,
                                          const std::string& utterance_id) {
  const int cap = (max_len > 0 ? num_frames / max_len : 0) + 2;
  std::vector<int> s(cap > 0 ? cap : 1), e(cap > 0 ? cap : 1);
  int n = 0;
  detail::check(bl_hard_segments(num_frames, min_len, max_len, s.data(), e.data(), cap, &n));
  std::vector<Segment> out;
  for (int k = 0; k < n; ++k) out.push_back({utterance_id, s[k], e[k], "hard"});
  return out;
}

// segmentation.hpp:10-60 — VAD segmentation (host code, same op order as
// segmentation.cpp:13-119, so threshold ties decide identically)
struct NodeMap {
  std::vector<int> speech_nodes;
  std::vector<int> noise_nodes;
  void validate(int output_width) const {
    if (speech_nodes.empty() || noise_nodes.empty())
      throw std::invalid_argument("nodemap: speech and noise sets must be non-empty");
    for (int n : noise_nodes)
      if (std::find(speech_nodes.begin(), speech_nodes.end(), n) != speech_nodes.end())
        throw std::invalid_argument("nodemap: speech and noise sets overlap");
    for (int n : speech_nodes)
      if (n < 0 || n >= output_width) throw std::invalid_argument("nodemap: speech node out of range");
    for (int n : noise_nodes)
      if (n < 0 || n >= output_width) throw std::invalid_argument("nodemap: noise node out of range");
  }
};

struct VadConfig {
  double threshold = 0.0;  // LLR cut, nats
  int smooth_window = 5;   // frames
  int min_len = 1500;      // frames
  int max_len = 2000;      // frames
  void validate() const {
    if (smooth_window < 1) throw std::invalid_argument("vad: smoothing window must be >= 1");
    if (!(min_len > 0 && min_len <= max_len))
      throw std::invalid_argument("vad: need 0 < min_len <= max_len");
  }
};

// log P_noise - log P_speech, each the max output over its node set
inline double frame_llr(const std::vector<double>& outputs, const NodeMap& nodemap) {
  nodemap.validate(static_cast<int>(outputs.size()));
  double speech = -HUGE_VAL, noise = -HUGE_VAL;
  for (int k : nodemap.speech_nodes) speech = std::max(speech, outputs[k]);
  for (int k : nodemap.noise_nodes) noise = std::max(noise, outputs[k]);
  return noise - speech;
}

// centred W-frame moving average (truncated at the edges); speech iff <= theta
inline std::vector<bool> smooth_and_decide(const std::vector<double>& llr, double threshold,
                                           int smooth_window) {
  if (smooth_window < 1) throw std::invalid_argument("smoothing window must be >= 1");
  const int n = static_cast<int>(llr.size());
  std::vector<double> prefix(n + 1, 0.0);
  for (int t = 0; t < n; ++t) prefix[t + 1] = prefix[t] + llr[t];
  const int half_lo = (smooth_window - 1) / 2, half_hi = smooth_window / 2;
  std::vector<bool> speech(n);
  for (int t = 0; t < n; ++t) {
    const int lo = std::max(0, t - half_lo), hi = std::min(n - 1, t + half_hi);
    speech[t] = (prefix[hi + 1] - prefix[lo]) / (hi - lo + 1) <= threshold;
  }
  return speech;
}

// maximal speech runs, merged left to right until >= min_len, then split into
// near-uniform pieces of at most max_len
inline std::vector<Segment> vad_segments(const std::vector<bool>& speech_flags, int min_len,
                                         int max_len, const std::string& utterance_id) {
  if (!(min_len > 0 && min_len <= max_len))
    throw std::invalid_argument("vad_segments: need 0 < min_len <= max_len");
  const int n = static_cast<int>(speech_flags.size());
  std::vector<std::pair<int, int>> runs, merged;
  for (int t = 0; t < n;) {
    if (!speech_flags[t]) {
      ++t;
      continue;
    }
    const int a = t;
    while (t < n && speech_flags[t]) ++t;
    runs.emplace_back(a, t);
  }
  for (size_t r = 0; r < runs.size();) {
    int a = runs[r].first, b = runs[r].second;
    ++r;
    while (b - a < min_len && r < runs.size()) b = runs[r++].second;
    merged.emplace_back(a, b);
  }
  std::vector<Segment> out;
  for (auto [a, b] : merged) {
    const int len = b - a, pieces = (len + max_len - 1) / max_len;
    int off = a;
    for (int k = 0; k < pieces; ++k) {
      const int piece = len / pieces + (k < len % pieces ? 1 : 0);
      out.push_back({utterance_id, off, off + piece, "vad"});
      off += piece;
    }
  }
  return out;
}

// batched.hpp:13-38
struct Batch {
  std::vector<Utterance> utterances;
  uint32_t padded_frames = 0;
};

inline std::vector<Batch> make_batches(std::vector<Utterance> utterances, int batch_size) {
  std::vector<uint32_t> fr;
  for (const auto& u : utterances) fr.push_back(u.true_frames);
  std::vector<int> order(utterances.size());
  int nb = 0;
  detail::check(bl_make_batches(static_cast<int>(fr.size()), fr.data(), batch_size,
                                order.data(), &nb));
  std::vector<Batch> out;
  for (size_t i = 0; i < order.size(); i += batch_size) {
    Batch b;
    for (size_t k = i; k < order.size() && k < i + batch_size; ++k) {
      b.utterances.push_back(std::move(utterances[order[k]]));
      b.padded_frames = std::max(b.padded_frames, b.utterances.back().true_frames);
    }
    out.push_back(std::move(b));
  }
  return out;
}

inline std::vector<DecodeResult> batched_beam_search(const Batch& batch, const Scorer& scorer,
                                                     const DecoderConfig& cfg,
                                                     DecodeCounters* counters = nullptr) {
  cfg.validate();
  if (batch.utterances.empty()) return {};
  const bl_config cc = cfg.c();
  bl_decoder* d = nullptr;
  detail::check(bl_decoder_create(detail::device(), &cc, scorer.handle(), &d));
  std::unique_ptr<bl_decoder, void (*)(bl_decoder*)> guard(d, bl_decoder_destroy);
  std::vector<bl_utt> in;
  for (const auto& u : batch.utterances)
    in.push_back({u.id.c_str(), u.grid.num_frames, u.grid.vocab, u.grid.frame_shift_ms,
                  u.grid.logp.data()});
  bl_results* r = nullptr;
  detail::check(bl_decode(d, static_cast<int>(in.size()), in.data(), 0, &r));
  std::unique_ptr<bl_results, void (*)(bl_results*)> rg(r, bl_results_destroy);
  std::vector<DecodeResult> out;
  for (int i = 0; i < bl_results_count(r); ++i) {
    const char* id;
    const int *tok, *lt;
    int n, steps, trig;
    double joint;
    detail::check(bl_results_get(r, i, &id, &tok, &n, &joint, &lt, &steps, &trig));
    out.push_back({id, std::vector<int>(tok, tok + n), joint, std::vector<int>(lt, lt + n),
                   steps, static_cast<EosTrigger>(trig)});
  }
  if (counters) {
    DecodeCounters c;
    bl_results_counters(r, &c.steps, &c.scorer_queries, &c.ctc_frames_evaluated);
    *counters += c;
  }
  return out;
}

inline DecodeResult beam_search(const Utterance& utt, const Scorer& scorer,
                                const DecoderConfig& cfg, DecodeCounters* counters = nullptr) {
  Batch b;
  b.utterances = {utt};
  b.padded_frames = utt.true_frames;
  return batched_beam_search(b, scorer, cfg, counters).front();
}

// ---------------------------------------------------------------- grid I/O
// grid.hpp:53-62 (grid.cpp): validation, padding, CTCG container
// ("CTCG", u32 version=1, T, vocab, frame_shift_ms, T*vocab f32, little-endian).
inline std::optional<std::string> validate_grid(const PosteriorGrid& grid) {
  constexpr double kRowTol = 1e-6;
  if (grid.num_frames < 1) return std::string("empty grid");
  if (grid.vocab < 2) return std::string("vocab must be >= 2 (one token plus blank)");
  if (grid.logp.size() != static_cast<size_t>(grid.num_frames) * grid.vocab)
    return std::string("logp size does not match T*vocab");
  for (uint32_t t = 0; t < grid.num_frames; ++t) {
    const float* row = grid.logp.data() + static_cast<size_t>(t) * grid.vocab;
    double m = -HUGE_VAL;
    for (uint32_t k = 0; k < grid.vocab; ++k) {
      if (std::isnan(row[k])) return "row " + std::to_string(t) + " has NaN";
      if (row[k] > kRowTol)
        return "row " + std::to_string(t) + " entry " + std::to_string(k) +
               " is a positive log-prob";
      m = std::max(m, static_cast<double>(row[k]));
    }
    double lse = kLogZero;
    if (m > -1e29) {
      double sum = 0.0;
      for (uint32_t k = 0; k < grid.vocab; ++k) sum += std::exp(row[k] - m);
      lse = m + std::log(sum);
    }
    if (std::abs(lse) > kRowTol) {
      std::ostringstream os;
      os.setf(std::ios::showpos);
      os << "row " << t << " logsumexp=" << lse;
      return os.str();
    }
  }
  return std::nullopt;
}

inline PosteriorGrid pad_to_length(const PosteriorGrid& grid, uint32_t target_frames) {
  if (target_frames < grid.num_frames)
    throw std::invalid_argument("pad_to_length: target shorter than grid");
  PosteriorGrid out = grid;
  out.num_frames = target_frames;
  out.logp.resize(static_cast<size_t>(target_frames) * grid.vocab, static_cast<float>(kLogZero));
  for (uint32_t t = grid.num_frames; t < target_frames; ++t)  // blank-only frames
    out.logp[static_cast<size_t>(t) * grid.vocab + grid.vocab - 1] = 0.0f;
  return out;
}

namespace detail {
inline void put_u32(std::ostream& os, uint32_t v) {
  const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                              static_cast<unsigned char>(v >> 16),
                              static_cast<unsigned char>(v >> 24)};
  os.write(reinterpret_cast<const char*>(b), 4);
}
inline uint32_t get_u32(std::istream& is) {
  unsigned char b[4] = {0, 0, 0, 0};
  is.read(reinterpret_cast<char*>(b), 4);
  return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
         (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24);
}
// nlohmann::json's number format (the reference writer, io.cpp:81-92).
// Digits by Grisu2 (Loitsch 2010, "Printing Floating-Point Numbers Quickly and
// Accurately with Integers") with the boundary, cached-power and rounding
// choices nlohmann 3.11 makes, so the digits match its output byte for byte
// (tests/test_json_format.py checks against the compiled reference); then
// fixed notation while the decimal point falls in (-4, 15], else d.ddde+XX
// with at least two exponent digits. Non-finite values dump as null.
namespace grisu {
struct Fp {
  uint64_t f;
  int e;
};
inline Fp mul(Fp x, Fp y) {
  const uint64_t ul = x.f & 0xFFFFFFFFu, uh = x.f >> 32, vl = y.f & 0xFFFFFFFFu, vh = y.f >> 32;
  const uint64_t p0 = ul * vl, p1 = ul * vh, p2 = uh * vl, p3 = uh * vh;
  uint64_t q = (p0 >> 32) + (p1 & 0xFFFFFFFFu) + (p2 & 0xFFFFFFFFu) + (uint64_t{1} << 31);
  return {p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}
inline Fp normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}
struct Cached {
  uint64_t f;
  int e, k;
};
// 10^k, k = -300, -292, ..., 324, as round-to-nearest 64-bit significands
inline const Cached& cached_power(int idx) {
  static const Cached t[79] = {
      {0xAB70FE17C79AC6CAULL, -1060, -300},
      {0xFF77B1FCBEBCDC4FULL, -1034, -292},
      {0xBE5691EF416BD60CULL, -1007, -284},
      {0x8DD01FAD907FFC3CULL, -980, -276},
      {0xD3515C2831559A83ULL, -954, -268},
      {0x9D71AC8FADA6C9B5ULL, -927, -260},
      {0xEA9C227723EE8BCBULL, -901, -252},
      {0xAECC49914078536DULL, -874, -244},
      {0x823C12795DB6CE57ULL, -847, -236},
      {0xC21094364DFB5637ULL, -821, -228},
      {0x9096EA6F3848984FULL, -794, -220},
      {0xD77485CB25823AC7ULL, -768, -212},
      {0xA086CFCD97BF97F4ULL, -741, -204},
      {0xEF340A98172AACE5ULL, -715, -196},
      {0xB23867FB2A35B28EULL, -688, -188},
      {0x84C8D4DFD2C63F3BULL, -661, -180},
      {0xC5DD44271AD3CDBAULL, -635, -172},
      {0x936B9FCEBB25C996ULL, -608, -164},
      {0xDBAC6C247D62A584ULL, -582, -156},
      {0xA3AB66580D5FDAF6ULL, -555, -148},
      {0xF3E2F893DEC3F126ULL, -529, -140},
      {0xB5B5ADA8AAFF80B8ULL, -502, -132},
      {0x87625F056C7C4A8BULL, -475, -124},
      {0xC9BCFF6034C13053ULL, -449, -116},
      {0x964E858C91BA2655ULL, -422, -108},
      {0xDFF9772470297EBDULL, -396, -100},
      {0xA6DFBD9FB8E5B88FULL, -369, -92},
      {0xF8A95FCF88747D94ULL, -343, -84},
      {0xB94470938FA89BCFULL, -316, -76},
      {0x8A08F0F8BF0F156BULL, -289, -68},
      {0xCDB02555653131B6ULL, -263, -60},
      {0x993FE2C6D07B7FACULL, -236, -52},
      {0xE45C10C42A2B3B06ULL, -210, -44},
      {0xAA242499697392D3ULL, -183, -36},
      {0xFD87B5F28300CA0EULL, -157, -28},
      {0xBCE5086492111AEBULL, -130, -20},
      {0x8CBCCC096F5088CCULL, -103, -12},
      {0xD1B71758E219652CULL, -77, -4},
      {0x9C40000000000000ULL, -50, 4},
      {0xE8D4A51000000000ULL, -24, 12},
      {0xAD78EBC5AC620000ULL, 3, 20},
      {0x813F3978F8940984ULL, 30, 28},
      {0xC097CE7BC90715B3ULL, 56, 36},
      {0x8F7E32CE7BEA5C70ULL, 83, 44},
      {0xD5D238A4ABE98068ULL, 109, 52},
      {0x9F4F2726179A2245ULL, 136, 60},
      {0xED63A231D4C4FB27ULL, 162, 68},
      {0xB0DE65388CC8ADA8ULL, 189, 76},
      {0x83C7088E1AAB65DBULL, 216, 84},
      {0xC45D1DF942711D9AULL, 242, 92},
      {0x924D692CA61BE758ULL, 269, 100},
      {0xDA01EE641A708DEAULL, 295, 108},
      {0xA26DA3999AEF774AULL, 322, 116},
      {0xF209787BB47D6B85ULL, 348, 124},
      {0xB454E4A179DD1877ULL, 375, 132},
      {0x865B86925B9BC5C2ULL, 402, 140},
      {0xC83553C5C8965D3DULL, 428, 148},
      {0x952AB45CFA97A0B3ULL, 455, 156},
      {0xDE469FBD99A05FE3ULL, 481, 164},
      {0xA59BC234DB398C25ULL, 508, 172},
      {0xF6C69A72A3989F5CULL, 534, 180},
      {0xB7DCBF5354E9BECEULL, 561, 188},
      {0x88FCF317F22241E2ULL, 588, 196},
      {0xCC20CE9BD35C78A5ULL, 614, 204},
      {0x98165AF37B2153DFULL, 641, 212},
      {0xE2A0B5DC971F303AULL, 667, 220},
      {0xA8D9D1535CE3B396ULL, 694, 228},
      {0xFB9B7CD9A4A7443CULL, 720, 236},
      {0xBB764C4CA7A44410ULL, 747, 244},
      {0x8BAB8EEFB6409C1AULL, 774, 252},
      {0xD01FEF10A657842CULL, 800, 260},
      {0x9B10A4E5E9913129ULL, 827, 268},
      {0xE7109BFBA19C0C9DULL, 853, 276},
      {0xAC2820D9623BF429ULL, 880, 284},
      {0x80444B5E7AA7CF85ULL, 907, 292},
      {0xBF21E44003ACDD2DULL, 933, 300},
      {0x8E679C2F5E44FF8FULL, 960, 308},
      {0xD433179D9C8CB841ULL, 986, 316},
      {0x9E19DB92B4E31BA9ULL, 1013, 324}};
  return t[idx];
}
inline void round_last(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest,
                       uint64_t ten) {
  while (rest < dist && delta - rest >= ten &&
         (rest + ten < dist || dist - rest > rest + ten - dist)) {
    buf[len - 1]--;
    rest += ten;
  }
}
// digits of v > 0 into buf; value = digits * 10^dec
inline int digits(double v, char* buf, int* dec) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t E = (bits >> 52) & 0x7FF, F = bits & ((uint64_t{1} << 52) - 1);
  const Fp w0 = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t{1} << 52), static_cast<int>(E) - 1075};
  const bool closer = F == 0 && E > 1;
  const Fp mp{2 * w0.f + 1, w0.e - 1};
  const Fp mm = closer ? Fp{4 * w0.f - 1, w0.e - 2} : Fp{2 * w0.f - 1, w0.e - 1};
  const Fp wp = normalize(mp);
  const Fp wm{mm.f << (mm.e - wp.e), wp.e};
  const Fp w = normalize(w0);
  const int f = -60 - wp.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
  const Cached& c = cached_power((300 + k + 7) / 8);
  const Fp cw = mul(w, {c.f, c.e}), cm = mul(wm, {c.f, c.e}), cp = mul(wp, {c.f, c.e});
  const Fp Mm{cm.f + 1, cm.e}, Mp{cp.f - 1, cp.e};
  *dec = -c.k;
  uint64_t delta = Mp.f - Mm.f, dist = Mp.f - cw.f;
  const int sh = -Mp.e;
  const uint64_t one = uint64_t{1} << sh;
  uint32_t p1 = static_cast<uint32_t>(Mp.f >> sh);
  uint64_t p2 = Mp.f & (one - 1);
  uint32_t pow10 = 1;
  int n = 1;
  for (uint32_t p = 1000000000u, d = 10; d > 1; p /= 10, --d)
    if (p1 >= p) {
      pow10 = p;
      n = static_cast<int>(d);
      break;
    }
  int len = 0;
  while (n > 0) {
    buf[len++] = static_cast<char>('0' + p1 / pow10);
    p1 %= pow10;
    --n;
    const uint64_t rest = (uint64_t{p1} << sh) + p2;
    if (rest <= delta) {
      *dec += n;
      round_last(buf, len, dist, delta, rest, uint64_t{pow10} << sh);
      return len;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[len++] = static_cast<char>('0' + (p2 >> sh));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  *dec -= m;
  round_last(buf, len, dist, delta, p2, one);
  return len;
}
}  // namespace grisu
inline std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[32];
  int dec = 0;
  const int k = grisu::digits(std::fabs(v), buf, &dec);
  const std::string digits(buf, static_cast<size_t>(k));
  const int n = k + dec;  // decimal point position
  std::string o;
  if (k <= n && n <= 15) {
    o = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    o = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (-4 < n && n <= 0) {
    o = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    o = digits.substr(0, 1);
    if (k > 1) o += "." + digits.substr(1);
    int ex = n - 1;
    o += ex < 0 ? "e-" : "e+";
    ex = ex < 0 ? -ex : ex;
    if (ex < 10) o += '0';
    o += std::to_string(ex);
  }
  return v < 0 ? "-" + o : o;
}
// nlohmann's string escapes: quote, backslash, the short control escapes,
// other control characters as \u00XX; UTF-8 bytes pass through
inline std::string json_string(const std::string& v) {
  std::string o = "\"";
  for (const char ch : v) {
    const unsigned char c = static_cast<unsigned char>(ch);
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char e[8];
          std::snprintf(e, sizeof(e), "\\u%04x", c);
          o += e;
        } else {
          o += ch;
        }
    }
  }
  return o + "\"";
}
inline std::string json_ints(const std::vector<int>& v) {
  std::string o = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ',';
    o += std::to_string(v[i]);
  }
  return o + "]";
}
}  // namespace detail

inline void write_grid(const std::string& path, const PosteriorGrid& grid) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw std::runtime_error("cannot write grid file: " + path);
  os.write("CTCG", 4);
  detail::put_u32(os, 1);
  detail::put_u32(os, grid.num_frames);
  detail::put_u32(os, grid.vocab);
  detail::put_u32(os, grid.frame_shift_ms);
  os.write(reinterpret_cast<const char*>(grid.logp.data()),
           static_cast<std::streamsize>(grid.logp.size() * sizeof(float)));
  if (!os) throw std::runtime_error("short write: " + path);
}

inline PosteriorGrid read_grid(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open grid file: " + path);
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, "CTCG", 4) != 0)
    throw std::runtime_error("bad magic in grid file: " + path);
  if (detail::get_u32(is) != 1) throw std::runtime_error("unsupported grid version in " + path);
  PosteriorGrid g;
  g.num_frames = detail::get_u32(is);
  g.vocab = detail::get_u32(is);
  g.frame_shift_ms = detail::get_u32(is);
  g.logp.resize(static_cast<size_t>(g.num_frames) * g.vocab);
  is.read(reinterpret_cast<char*>(g.logp.data()),
          static_cast<std::streamsize>(g.logp.size() * sizeof(float)));
  if (!is) throw std::runtime_error("truncated grid file: " + path);
  return g;
}

// io.hpp:32 (io.cpp:81-92): one JSON object per result, keys in sorted order
inline void write_results(std::ostream& os, const std::vector<DecodeResult>& results) {
  for (const auto& r : results) {
    os << "{\"eos_trigger\":" << detail::json_string(to_string(r.eos_trigger))
       << ",\"id\":" << detail::json_string(r.id)
       << ",\"joint_logp\":" << detail::json_double(r.joint_logp)
       << ",\"label_times\":" << detail::json_ints(r.label_times)
       << ",\"steps\":" << r.steps_taken << ",\"tokens\":" << detail::json_ints(r.tokens)
       << "}\n";
  }
}

}  // namespace beamlattice
