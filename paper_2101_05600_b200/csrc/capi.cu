// capi.cu — C ABI of the B200 decoder (include/bl_b200.h): host planner,
// device workspace, scorer loading, result assembly. Host logic mirrors the
// reference semantics cited per function; all decoding runs on the GPU —
// there is no CPU fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "../../include/bl_b200.h"
#include "decode.cuh"
#include "decoder_net.cuh"
#include "encoder.cuh"
#include "gemm.cuh"

namespace bl {
cudaError_t launch_decode(const KParams& p, cudaStream_t st);
size_t step_state_bytes(int B, int S);
size_t decode_smem_bytes(const KParams& p);
size_t decode_static_smem(const KParams& p);
int bmax_for(int B);
}  // namespace bl

namespace {

thread_local std::string g_err;

struct BlError {
  int code;
  std::string msg;
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                             \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess)                                                   \
      throw BlError{BL_CUDA_ERROR, std::string(#call) + ": " +               \
                                       cudaGetErrorString(_e)};              \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const BlError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return BL_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return BL_LOGIC_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BL_RUNTIME_ERROR;
  }
}

// ------------------------------------------------------------ scorers
// check_normalized, scorer.cpp:14-28
void check_normalized(const std::vector<double>& v, size_t expected,
                      const std::string& what) {
  if (v.size() != expected) throw std::runtime_error(what + ": wrong vector size");
  double m = -HUGE_VAL;
  for (double x : v) m = std::max(m, x);
  double s = 0.0;
  for (double x : v) s += std::exp(x - m);
  double lse = m + std::log(s);
  if (!(std::abs(lse) <= 1e-6)) {
    std::ostringstream os;
    os << what << ": vector not normalized (logsumexp=" << lse << ")";
    throw std::runtime_error(os.str());
  }
}

}  // namespace

struct bl_scorer {
  int kind = 0;  // 0 uniform, 1 table, 2 loop, 3 transformer (device network)
  bl::DecoderNet* net = nullptr;
  int net_device = 0;
  ~bl_scorer() {
    if (net) {
      cudaSetDevice(net_device);
      bl::dec_destroy(net);
    }
  }
  int num_tokens = 0;
  int order = 1;
  std::map<std::vector<int>, std::vector<double>> table;
  int loop_token = 0;
  double p_loop = 0.0;

  std::vector<double> uniform_row() const {  // scorer.cpp:34-38
    return std::vector<double>(num_tokens + 1,
                               -std::log(static_cast<double>(num_tokens + 1)));
  }
  std::vector<double> loop_row() const {  // scorer.cpp:73-80
    double rest = std::log((1.0 - p_loop) / num_tokens);
    std::vector<double> v(num_tokens + 1, rest);
    v[loop_token] = std::log(p_loop);
    return v;
  }
  std::vector<double> score(const std::vector<int>& prefix) const {
    if (kind == 3)
      throw std::logic_error("the transformer scorer runs on device inside the decoder");
    if (kind == 2) return loop_row();
    if (kind == 1) {  // scorer.cpp:53-62
      size_t n = std::min<size_t>(prefix.size(), order - 1);
      std::vector<int> ctx(prefix.end() - n, prefix.end());
      auto it = table.find(ctx);
      if (it != table.end()) return it->second;
    }
    return uniform_row();
  }
};

namespace {

bl_scorer* make_table(int num_tokens, int order) {  // scorer.cpp:40-44
  if (num_tokens < 1) throw std::invalid_argument("TableScorer: |C| < 1");
  if (order < 1) throw std::invalid_argument("TableScorer: order < 1");
  auto* s = new bl_scorer;
  s->kind = 1;
  s->num_tokens = num_tokens;
  s->order = order;
  return s;
}

bl_scorer* make_loop(int num_tokens, int loop_token, double p) {  // scorer.cpp:64-71
  if (num_tokens < 1) throw std::invalid_argument("LoopScorer: |C| < 1");
  if (loop_token < 0 || loop_token >= num_tokens)
    throw std::invalid_argument("LoopScorer: loop token out of range");
  if (!(p > 0.5 && p < 1.0))
    throw std::invalid_argument("LoopScorer: p_loop must be in (0.5, 1)");
  auto* s = new bl_scorer;
  s->kind = 2;
  s->num_tokens = num_tokens;
  s->loop_token = loop_token;
  s->p_loop = p;
  return s;
}

// load_table_scorer, scorer.cpp:82-103
bl_scorer* load_table(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw std::runtime_error("cannot open scorer file: " + path);
  nlohmann::json j;
  try {
    is >> j;
  } catch (const nlohmann::json::exception& e) {
    throw std::runtime_error("malformed scorer file " + path + ": " + e.what());
  }
  if (!j.contains("order") || !j.contains("num_tokens") || !j.contains("entries"))
    throw std::runtime_error("malformed scorer file " + path + ": missing field");
  std::unique_ptr<bl_scorer> s(make_table(j["num_tokens"].get<int>(), j["order"].get<int>()));
  for (const auto& e : j["entries"]) {
    auto lp = e["logp"].get<std::vector<double>>();
    check_normalized(lp, static_cast<size_t>(s->num_tokens) + 1, "TableScorer entry");
    s->table[e["ctx"].get<std::vector<int>>()] = std::move(lp);
  }
  return s.release();
}

}  // namespace

// ------------------------------------------------------------ decoder
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CK(cudaMalloc(&p, bytes));
    n = bytes;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    CK(cudaMallocHost(&p, bytes));
    n = bytes;
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
};

struct bl_decoder {
  int device = 0;
  bl_config cfg{};
  int num_tokens = 0;
  int nbest = 1;
  int exact = 0;
  double slack = 1.0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // H2D of grid chunks, overlapped with decoding
  cudaStream_t alt = nullptr;   // second compute stream: chunk kernels overlap at their tails
  cudaEvent_t ev_alt = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> ev_copy;
  // device scorer
  int sc_order = 1, sc_nent = 0, sc_w = 1;
  DevBuf sc_ctx_len, sc_ctx, sc_row, sc_rows, sc_rowsf;
  // workspace
  DevBuf grid, utts, gam, Ftab, Gtab, mshift, xs, taken, hist, fin, res, cnt, prof;
  HostBuf h_grid, h_utts, h_res, h_cnt, h_prof;
  bool profile = getenv("BL_PROFILE") != nullptr;
  // step-granular decoding (forced for tests, or required by a network scorer)
  int step_mode = 0;
  DevBuf state, n_done;
  HostBuf h_done;
  // network scorer (kind 3) and the encoder memory of the current call
  bl::DecoderNet* net = nullptr;
  const void* memory = nullptr;
  int mem_frames = 0;
  double net_ms = 0.0;
  // record mode (tests): the scorer rows of every live hypothesis with its prefix
  int record = 0;
  struct Rec {
    int utt;
    std::vector<int> prefix;
    std::vector<double> row;
  };
  std::vector<Rec> rec;
  DevBuf rec_nb, nb_live;
  // streamed host input (see KParams::ready)
  DevBuf ready, stream_err;
  HostBuf h_epoch, h_err;
  unsigned epoch = 0;
  size_t ready_n = 0;
  cudaEvent_t ev_copied = nullptr;
  // decoder group (bl_group_decode): result records keep a group-wide step
  // capacity and stay on the device (padded to keep_rows rows) for the NCCL
  // gather instead of being copied to the host by this decoder
  int force_S = 0;
  int keep_rows = 0;
};

struct bl_results {
  struct One {
    std::string id;
    std::vector<int> tokens, label_times;
    double joint = 0.0;
    int steps = 0, trigger = 2;
    std::vector<std::vector<int>> nb_tokens, nb_times;
    std::vector<double> nb_joint;
  };
  std::vector<One> r;
  int max_tokens = 0;
  uint64_t steps = 0, queries = 0, frames = 0, k1 = 0, fallback = 0, contenders = 0;
  uint64_t raw_keys = 0;  // filter mode: keys that reached the running bound
  uint64_t wide = 0;      // wide steps (beams of 13+: contenders > caps, complete theta0 list)
  uint64_t h2d = 0, d2h = 0;
  double kernel_ms = 0.0;
  int launches = 0;
  double prof[16] = {0};  // mean cycles per utterance per phase
};

namespace {

void upload_scorer(bl_decoder* d, const bl_scorer* s) {
  d->net = s->kind == 3 ? s->net : nullptr;
  // rows: 0 = uniform fallback, then one row per entry
  const int V = s->num_tokens + 1;
  std::vector<double> rows = s->uniform_row();
  std::vector<std::pair<std::vector<int>, int>> ents;
  if (s->kind == 2) {
    auto lr = s->loop_row();
    rows.insert(rows.end(), lr.begin(), lr.end());
    ents.push_back({{}, 1});
    d->sc_order = 1;
  } else if (s->kind == 1) {
    int r = 1;
    for (const auto& kv : s->table) {
      // only contexts a prefix can produce (len <= order-1) are reachable
      if ((int)kv.first.size() > s->order - 1) continue;
      rows.insert(rows.end(), kv.second.begin(), kv.second.end());
      ents.push_back({kv.first, r++});
    }
    d->sc_order = s->order;
  } else {
    d->sc_order = 1;
  }
  if (d->sc_order - 1 > 8)
    throw std::invalid_argument("device table scorer supports order <= 9");
  std::sort(ents.begin(), ents.end(), [](const auto& a, const auto& b) {
    if (a.first.size() != b.first.size()) return a.first.size() < b.first.size();
    return a.first < b.first;
  });
  d->sc_nent = (int)ents.size();
  d->sc_w = std::max(d->sc_order - 1, 1);
  std::vector<int> clen(std::max<size_t>(ents.size(), 1), 0),
      ctx(std::max<size_t>(ents.size() * d->sc_w, 1), 0),
      row(std::max<size_t>(ents.size(), 1), 0);
  for (size_t k = 0; k < ents.size(); ++k) {
    clen[k] = (int)ents[k].first.size();
    for (size_t i = 0; i < ents[k].first.size(); ++i) ctx[k * d->sc_w + i] = ents[k].first[i];
    row[k] = ents[k].second;
  }
  (void)V;
  d->sc_ctx_len.ensure(clen.size() * sizeof(int));
  d->sc_ctx.ensure(ctx.size() * sizeof(int));
  d->sc_row.ensure(row.size() * sizeof(int));
  d->sc_rows.ensure(rows.size() * sizeof(double));
  // (1 - lambda) * row in fp32 for the certified bulk keys; -inf marks a
  // log-zero attention entry (mix_joint then returns kLogZero exactly).
  const double lam = d->cfg.ctc_weight;
  std::vector<float> rowsf(rows.size());
  for (size_t i = 0; i < rows.size(); ++i)
    rowsf[i] = lam >= 1.0 ? 0.f
               : rows[i] <= -1e29 ? -INFINITY
                                  : (float)((lam <= 0.0 ? 1.0 : 1.0 - lam) * rows[i]);
  d->sc_rowsf.ensure(rowsf.size() * sizeof(float));
  CK(cudaMemcpy(d->sc_rowsf.p, rowsf.data(), rowsf.size() * sizeof(float), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d->sc_ctx_len.p, clen.data(), clen.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d->sc_ctx.p, ctx.data(), ctx.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d->sc_row.p, row.data(), row.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d->sc_rows.p, rows.data(), rows.size() * sizeof(double), cudaMemcpyHostToDevice));
}

// DecoderConfig::validate (beam_search.cpp:36-46)
void validate_cfg(const bl_config& c) {
  if (c.beam_width < 1) throw std::invalid_argument("beam width must be >= 1");
  if (c.ctc_weight < 0.0 || c.ctc_weight > 1.0)
    throw std::invalid_argument("ctc weight must be in [0, 1]");
  if (c.eos_m < 1) throw std::invalid_argument("eos M must be >= 1");
  if (c.eos_c < 0) throw std::invalid_argument("eos C must be >= 0");
  if (c.margin_m1 < 0 || c.margin_m2 < 0)
    throw std::invalid_argument("margins must be >= 0");
  if (!(c.max_steps_ratio > 0.0 && c.max_steps_ratio <= 1.0))
    throw std::invalid_argument("max steps ratio must be in (0, 1]");
  if (c.eos_mode < 0 || c.eos_mode > 2) throw std::invalid_argument("unknown eos mode");
}

float guard_float() {
  // largest float f with (double)f <= -1e29 (is_log_zero on promoted grids)
  float f = static_cast<float>(-1e29);
  while (static_cast<double>(f) > -1e29) f = std::nextafter(f, -INFINITY);
  while (static_cast<double>(std::nextafter(f, INFINITY)) <= -1e29)
    f = std::nextafter(f, INFINITY);
  return f;
}

// Step-granular decode of all utterances of `p` in lockstep: one launch
// per step; the host polls the finished-utterance counter every few steps.
int step_loop(bl_decoder* d, bl::KParams p, cudaStream_t st) {
  if (d->net) {  // source-attention K/V of the encoder memory, KV cache, rows
    CK(bl::dec_prepare(d->net, p.U, p.B, p.S + 1,
                       static_cast<const __nv_bfloat16*>(d->memory) +
                           (size_t)p.u0 * d->mem_frames * bl::dec_spec(d->net).d,
                       d->mem_frames, st));
    p.net_rows = 1;
    d->nb_live.ensure(sizeof(int) * (size_t)(p.u0 + p.U));
    p.nb_out = static_cast<int*>(d->nb_live.p);
  }
  const size_t stride = bl::step_state_bytes(p.B, p.S);
  d->state.ensure(stride * (size_t)p.U);
  d->n_done.ensure(sizeof(unsigned));
  d->h_done.ensure(sizeof(unsigned));
  CK(cudaMemsetAsync(d->n_done.p, 0, sizeof(unsigned), st));
  p.state = static_cast<unsigned char*>(d->state.p);
  p.state_stride = (int)stride;
  p.n_done = static_cast<unsigned*>(d->n_done.p);
  int launches = 0;
  const int poll = 4;
  const int V = p.V, B = p.B;
  std::vector<std::vector<double>> rec_rows;  // record mode: att rows per step
  if (d->record) {
    d->rec_nb.ensure(sizeof(int) * (size_t)p.U * (p.S + 2));
    CK(cudaMemsetAsync(d->rec_nb.p, 0, sizeof(int) * (size_t)p.U * (p.S + 2), st));
    p.rec_nb = static_cast<int*>(d->rec_nb.p);
  }
  // From step 2 on, the step (the scorer network's ~6 + 11 L launches and the
  // search launch) is stream-captured and replayed as ONE graph launch; the
  // executable graph is updated in place (same topology, new step
  // arguments) instead of re-instantiated. Record mode and BL_NO_GRAPH run
  // the launches directly.
  cudaStreamCaptureStatus cs0 = cudaStreamCaptureStatusNone;
  const bool capturable = st != cudaStreamLegacy && st != cudaStreamPerThread &&
                          cudaStreamIsCapturing(st, &cs0) == cudaSuccess &&
                          cs0 == cudaStreamCaptureStatusNone;
  cudaGetLastError();
  const bool use_graph =
      d->net && !d->record && capturable && std::getenv("BL_NO_GRAPH") == nullptr;
  cudaGraphExec_t gexec = nullptr;
  struct GraphGuard {
    cudaGraphExec_t* g;
    ~GraphGuard() {
      if (*g) cudaGraphExecDestroy(*g);
    }
  } gguard{&gexec};
  for (int l = 1; l <= p.S + 1; ++l) {
    p.step_l = l;
    const bool capture = use_graph && l >= 2 && l <= p.S;
    if (capture) CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    struct CaptureGuard {  // an error inside the captured region ends the capture
      cudaStream_t s;
      ~CaptureGuard() {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive) {
          cudaGraph_t g = nullptr;
          if (cudaStreamEndCapture(s, &g) == cudaSuccess && g) cudaGraphDestroy(g);
          cudaGetLastError();
        }
      }
    } cguard{st};
    if (d->net && l <= p.S) {  // att rows of the beam entering step l
      CK(bl::dec_step(d->net, l, p.hist + (size_t)p.u0 * (p.S + 1) * p.B, (p.S + 1) * p.B,
                      static_cast<const int*>(d->nb_live.p) + p.u0, d->cfg.ctc_weight, st));
      p.sc_rows = bl::dec_att(d->net);
      p.sc_rowsf = bl::dec_attf(d->net);
      p.net_lse = bl::dec_lse(d->net);
      p.net_logits = p.net_lse ? bl::dec_logits(d->net) : nullptr;
      launches += bl::dec_launches_per_step(d->net);
      if (d->record) {
        const size_t rows = (size_t)p.U * B;
        rec_rows.emplace_back(rows * V);
        if (p.net_lse) {  // the rows the search used: (double)logit - lse
          std::vector<float> lg(rows * V);
          std::vector<double> ls(rows);
          CK(cudaMemcpyAsync(lg.data(), p.net_logits, sizeof(float) * lg.size(),
                             cudaMemcpyDeviceToHost, st));
          CK(cudaMemcpyAsync(ls.data(), p.net_lse, sizeof(double) * rows, cudaMemcpyDeviceToHost,
                             st));
          CK(cudaStreamSynchronize(st));
          for (size_t r = 0; r < rows; ++r)
            for (int c = 0; c < V; ++c)
              rec_rows.back()[r * V + c] = (double)lg[r * V + c] - ls[r];
        } else {
          CK(cudaMemcpyAsync(rec_rows.back().data(), p.sc_rows,
                             sizeof(double) * rec_rows.back().size(), cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
        }
      }
    }
    if (capture) {
      const cudaError_t le = bl::launch_decode(p, st);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(st, &g);
      CK(le);
      CK(ce);
      cudaGraphExecUpdateResultInfo info;
      if (!gexec || cudaGraphExecUpdate(gexec, g, &info) != cudaSuccess) {
        cudaGetLastError();
        if (gexec) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&gexec, g, 0);
        cudaGraphDestroy(g);
        CK(ie);
      } else {
        cudaGraphDestroy(g);
      }
      CK(cudaGraphLaunch(gexec, st));
    } else {
      CK(bl::launch_decode(p, st));
    }
    ++launches;
    if (l % poll == 0 || l == p.S + 1) {
      CK(cudaMemcpyAsync(d->h_done.p, d->n_done.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (*static_cast<unsigned*>(d->h_done.p) >= (unsigned)p.U) break;
    }
  }
  if (d->record && d->net) {  // pair each recorded row with its prefix
    std::vector<int> nbh((size_t)p.U * (p.S + 2));
    std::vector<bl::HistRec> hh((size_t)p.U * (p.S + 1) * B);
    CK(cudaMemcpyAsync(nbh.data(), d->rec_nb.p, sizeof(int) * nbh.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hh.data(), p.hist, sizeof(bl::HistRec) * hh.size(), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    for (size_t li = 0; li < rec_rows.size(); ++li) {
      const int l = (int)li + 1;
      for (int u = 0; u < p.U; ++u) {
        const int nb = nbh[(size_t)u * (p.S + 2) + l];
        for (int k = 0; k < nb; ++k) {
          bl_decoder::Rec r;
          r.utt = u + p.u0;
          r.prefix.resize(l - 1);
          int slot = k;
          for (int st2 = l - 1; st2 >= 1; --st2) {
            const bl::HistRec& h = hh[((size_t)u * (p.S + 1) + st2) * B + slot];
            r.prefix[st2 - 1] = h.token;
            slot = h.parent;
          }
          const double* row = rec_rows[li].data() + ((size_t)u * B + k) * V;
          r.row.assign(row, row + V);
          d->rec.push_back(std::move(r));
        }
      }
    }
  }
  return launches;
}

// Bulk result destination (bl_decode_into): results written straight from
// the pinned D2H buffer into caller arrays, no per-utterance objects.
struct IntoArgs {
  int cap;
  int *n_tokens, *steps, *trigger, *tokens, *label_times;
  double* joint;
};

int decode_impl(bl_decoder* d, int n, const bl_utt* utts, int on_device,
                bl_results** out, const IntoArgs* into = nullptr) {
  using clk = std::chrono::steady_clock;
  static const bool host_timing = std::getenv("BL_HOST_TIMING") != nullptr;
  const auto t_in = clk::now();
  validate_cfg(d->cfg);  // batched.cpp:97
  auto res = std::make_unique<bl_results>();
  if (n == 0) {  // batched.cpp:99
    *out = res.release();
    return BL_OK;
  }
  const int C = d->num_tokens, V = C + 1, B = d->cfg.beam_width;
  for (int i = 0; i < n; ++i) {  // batched.cpp:105-111
    const std::string id = utts[i].id ? utts[i].id : "";
    if (utts[i].num_frames < 1)
      throw std::invalid_argument("empty grid in utterance " + id);
    if ((int)utts[i].vocab - 1 != C)
      throw std::invalid_argument("scorer vocabulary mismatch in utterance " + id);
  }
  if (bl::bmax_for(B) == 0)
    throw std::invalid_argument("beam width > 32 is not supported by the device decoder");
  if (V > (1 << 24))
    throw std::invalid_argument("vocabulary > 2^24 is not supported by the device decoder");
  CK(cudaSetDevice(d->device));

  int Tmax = 0, S = 0;
  std::vector<bl::UttDesc> desc(n);
  std::vector<size_t> goff(n);
  size_t gtotal = 0;
  for (int i = 0; i < n; ++i) {
    const int T = (int)utts[i].num_frames;
    Tmax = std::max(Tmax, T);
    desc[i].T = T;
    desc[i].max_steps = static_cast<int>(std::ceil(d->cfg.max_steps_ratio * T));
    S = std::max(S, desc[i].max_steps);
    S = std::max(S, d->force_S);
    desc[i].need_tail = d->cfg.margin_m2 < T ? 1 : 0;
    goff[i] = gtotal;  // dense packing: a contiguous host batch is one copy
    gtotal += (size_t)T * V;
  }
  const int Tp = (Tmax + 2) & ~1;
  // contender slots: 3B+16 (BL_CAPS_MULT=k gives kB+16, for sweeps). 2B+16
  // overflowed into the exact fallback on ~0.7% of beam-20 steps (flat
  // posteriors): 3B+16 cuts beam 20 at 10 s x 512 from 528 to 330 ms; 4B+16
  // is slower again (more chain warps, less staging room)
  static const int caps_mult =
      std::getenv("BL_CAPS_MULT") ? std::atoi(std::getenv("BL_CAPS_MULT")) : 3;
  // The P6 chains take (caps + 15) / 16 warps; the walk (P8) that overlaps
  // them needs one thread per selected item (<= B + bmax), so the chain warps
  // leave at least ceil((B + bmax) / 32) warps to it.
  const int bmax0 = bl::bmax_for(B);
  const int chain_warps = bl::kNWarp - (B + bmax0 + 31) / 32;
  // BL_CAPS: test override (caps >= B: a fallback or wide step's children
  // take slots 0..B-1); small caps force wide steps at beams of 13+
  static const int caps_abs = std::getenv("BL_CAPS") ? std::atoi(std::getenv("BL_CAPS")) : 0;
  const int caps = caps_abs > 0
                       ? std::min({std::max(B, caps_abs), bl::kNT, 16 * chain_warps})
                       : std::min({std::max(2, caps_mult) * B + 16, bl::kNT, 16 * chain_warps});
  const int nbest = std::max(1, d->nbest);
  const int rs = bl::res_stride(S, nbest);
  const int U = n;

  bool tail = false;
  for (auto& x : desc) tail |= x.need_tail != 0;

  // workspace
  d->gam.ensure(sizeof(double) * (size_t)U * 2 * caps * 2 * Tp);
  d->Gtab.ensure(sizeof(double) * (size_t)U * Tp);
  d->Ftab.ensure(tail ? sizeof(double) * (size_t)U * Tp * C : 8);
  const int bmax = bl::bmax_for(B);
  // TMA streaming of the K1 slab for large vocabularies: needs every grid in
  // one dense row-major buffer (always true for host input; checked for
  // device pointers) with 16-byte rows.
  const float* gbase = nullptr;
  bool use_tma = V >= 1024 && V % 4 == 0 && std::getenv("BL_NO_TMA") == nullptr;
  // the 3D tensor map of the tensor-core variant reads whole 32-column
  // blocks: up to 31 floats past the last row (a pad for our own buffer)
  const size_t gpad = 128;
  if (use_tma) {
    if (!on_device) {
      d->grid.ensure(sizeof(float) * gtotal + gpad);
      gbase = static_cast<const float*>(d->grid.p);
    } else {
      gbase = utts[0].logp;
      for (int i = 0; i < n && use_tma; ++i) use_tma = utts[i].logp == gbase + goff[i];
    }
    use_tma = use_tma && (reinterpret_cast<uintptr_t>(gbase) & 15) == 0;
  }
  // Tensor-core K1 bulk (decode_kernel.cu, kMode 3): TMA slab, at most 16
  // parents (N = 16), and unbounded right margin (every window ends at T, so
  // a column's max over the rows the next window can reach bounds it).
  // Tensor-core bulk (both opt-in, both measured slower than the CUDA-core
  // bulk at the C3 shape): 1 = tcgen05.mma (BL_TC=1; the
  // runtime runs tcgen05 kernels one CTA per SM, which leaves the serial
  // search phases without a second CTA to overlap), 2 = mma.sync m16n8k8
  // tf32 (BL_MMA=1; two CTAs per SM, register accumulators).
  int use_tc = !use_tma || B > 16 ? 0
               : std::getenv("BL_TC") != nullptr  ? 1
               : std::getenv("BL_MMA") != nullptr ? 2
                                                  : 0;
  for (int i = 0; i < n && use_tc; ++i)
    if (desc[i].need_tail) use_tc = 0;
  if (use_tc && on_device) {
    // the grid allocation must cover the last block's overhang
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range = nullptr;
    if (!range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) ==
              cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        range = reinterpret_cast<RangeFn>(fn);
    }
    CUdeviceptr b0 = 0;
    size_t sz = 0;
    if (!(range && range(&b0, &sz, reinterpret_cast<CUdeviceptr>(gbase)) == CUDA_SUCCESS &&
          reinterpret_cast<CUdeviceptr>(gbase) + sizeof(float) * gtotal + gpad <= b0 + sz))
      use_tc = 0;
    cudaGetLastError();
  }
  // tcgen05 kernels run one CTA per SM (the runtime's occupancy for any
  // kernel using tcgen05.alloc): the tensor-core variant takes the deepest ring
  int tma_stages = use_tma ? (use_tc == 1 ? bl::kTmaStagesMax : 6) : 0;
  {
    // Slab mode: 16 KB stages split into per-warp slots of 16 rows (two per
    // warp from 4 stages up; fewer stages give 8-row slots, which carry 3/4 or
    // less of the bytes in flight and run up to 1.4x slower,
    // scripts/c3_leg.py N 499). Large calls take 4 stages when two CTAs per
    // SM then fit (their serial phases overlap), else 6 at one CTA per SM.
    // Long utterances: fewer stages (down to 2), then the non-TMA path,
    // before the plan is rejected (12 KB left for static shared memory).
    const size_t lim = (227 - 12) * 1024;
    const size_t fixed0 = bl::smem_plan(Tmax, B, bmax, C, caps, S, 0, 0).total;
    auto need = [&](int st) {
      return fixed0 + bl::smem_plan(Tmax, B, bmax, C, caps, S, 0, 0, st, use_tc).region_need;
    };
    if (use_tma && use_tc != 1 && U > 148 && need(4) + 6 * 1024 <= 113 * 1024) tma_stages = 4;
    while (use_tma && tma_stages > 2 && need(tma_stages) > lim) --tma_stages;
    if (use_tma && need(tma_stages) > lim) {
      use_tma = false;
      use_tc = 0;
      tma_stages = 0;
    }
    if (const char* e = std::getenv("BL_TMA_STAGES"))  // sweep override (16 KB units)
      if (use_tma && use_tc != 1) tma_stages = std::max(2, std::min(bl::kTmaStagesMax, atoi(e)));
  }
  // shared-memory plan: the aliased region (P3-P5 keys, P6 staging) is sized
  // so the whole plan fits 3 CTAs/SM (~71 KB) when the fixed parts allow it;
  // otherwise the keys are filtered on chip while P3 emits them (filter mode).
  const size_t fixed = bl::smem_plan(Tmax, B, bmax, C, caps, S, 0, 0).total;
  const size_t budget = 66 * 1024;  // + static smem + 1 KB reserve: 3 CTAs in 228 KB
  const size_t need1 = bl::smem_plan(Tmax, B, bmax, C, caps, S, 0, 1).region_need;
  const size_t need0 =
      bl::smem_plan(Tmax, B, bmax, C, caps, S, 0, 0, tma_stages, use_tc).region_need;
  size_t region = fixed + need1 <= budget ? budget - fixed : std::max(need0, budget > fixed ? budget - fixed : 0);
  const int kub_smem = (!use_tma && need1 <= region) ? 1 : 0;
  region = (std::max(region, kub_smem ? need1 : need0) + 15) & ~(size_t)15;
  d->xs.ensure(sizeof(double) * (size_t)U * bl::xs_stride(B, C, bmax));
  d->taken.ensure((size_t)U * B * (C + 1));
  d->hist.ensure(sizeof(bl::HistRec) * (size_t)U * (S + 1) * B);
  d->fin.ensure(sizeof(bl::FinEntry) * (size_t)U * B * S);
  d->res.ensure(sizeof(int) * (size_t)std::max(U, d->keep_rows) * rs);
  d->cnt.ensure(sizeof(unsigned long long) * (size_t)U * 8);
  d->utts.ensure(sizeof(bl::UttDesc) * U);
  d->h_utts.ensure(sizeof(bl::UttDesc) * U);
  d->h_res.ensure(sizeof(int) * (size_t)U * rs);
  d->h_cnt.ensure(sizeof(unsigned long long) * (size_t)U * 8);

  cudaStream_t st = d->stream;
  // Host grids: runs of utterances contiguous in host memory become single
  // copies, straight from the caller's buffer when it is pinned, else via
  // pinned staging; chunks of utterances are copied on a second stream while
  // earlier chunks decode.
  struct Run {
    int i0, i1;  // utterances [i0, i1)
    const float* src;
  };
  std::vector<Run> runs;
  if (!on_device) {
    d->grid.ensure(sizeof(float) * gtotal + gpad);
    for (int i = 0; i < n; ++i) {
      if (!runs.empty() && runs.back().i1 == i &&
          utts[i].logp == utts[i - 1].logp + (size_t)desc[i - 1].T * V)
        runs.back().i1 = i + 1;
      else
        runs.push_back({i, i + 1, utts[i].logp});
    }
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, utts[0].logp) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned) {
      d->h_grid.ensure(sizeof(float) * gtotal);
      float* hg = static_cast<float*>(d->h_grid.p);
      for (auto& r : runs) {
        const size_t len = goff[r.i1 - 1] + (size_t)desc[r.i1 - 1].T * V - goff[r.i0];
        std::memcpy(hg + goff[r.i0], r.src, sizeof(float) * len);
        r.src = hg + goff[r.i0];
      }
    }
  }

  bl::KParams p{};
  p.U = U;
  p.V = V;
  p.C = C;
  p.B = B;
  p.Tmax = Tmax;
  p.Tp = Tp;
  p.S = S;
  p.caps = caps;
  p.lambda = d->cfg.ctc_weight;
  p.eos_dend = d->cfg.eos_dend;
  p.eos_m = d->cfg.eos_m;
  p.eos_c = d->cfg.eos_c;
  p.m1 = d->cfg.margin_m1;
  p.m2 = d->cfg.margin_m2;
  p.eos_mode = d->cfg.eos_mode;
  p.guard_f = guard_float();
  p.exact = d->exact;
  p.nbest = nbest;
  // certified psi half-width: the tensor-core bulk rounds the factors and
  // truncates the exponentials to tf32 (relative error <= 2^-11 + 2^-10 per
  // product, so <= 1.5e-3 on each sum): 2.5e-3 more
  p.dpsi0 = (use_tc ? 3e-3 : 5e-4) * d->slack;  // (both tensor-core variants use tf32)
  p.dpsi1 = 1e-6 * d->slack;
  p.sc_order = d->sc_order;
  p.sc_nent = d->sc_nent;
  p.sc_w = d->sc_w;
  p.sc_ctx_len = static_cast<const int*>(d->sc_ctx_len.p);
  p.sc_ctx = static_cast<const int*>(d->sc_ctx.p);
  p.sc_row = static_cast<const int*>(d->sc_row.p);
  p.sc_rows = static_cast<const double*>(d->sc_rows.p);
  p.gam = static_cast<double*>(d->gam.p);
  p.Ftab = static_cast<double*>(d->Ftab.p);
  p.Gtab = static_cast<double*>(d->Gtab.p);
  p.kub_smem = kub_smem;
  p.region_bytes = (int)region;
  p.use_tma = use_tma ? 1 : 0;
  p.use_tc = use_tc;
  if (use_tc) {
    p.mshift_stride = ((C + 511) / 512) * 512;
    d->mshift.ensure(sizeof(float) * 2 * (size_t)U * p.mshift_stride);
    p.mshift = static_cast<float*>(d->mshift.p);
  }
  p.tma_stages = tma_stages;
  if (use_tma) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess)
        throw BlError{BL_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable"};
      encode = reinterpret_cast<EncodeFn>(fn);
    }
    CUresult r;
    if (use_tc) {
      // {32 columns, rows, 32-column blocks}: a box of 16 blocks x 8 rows
      // lands as 16 MN-major swizzle atoms of 8 rows x 128 B (32-byte-atom
      // 128-byte swizzle), the tf32 A operand layout of tcgen05.mma
      const cuuint64_t dims[3] = {32, (cuuint64_t)(gtotal / V), (cuuint64_t)((V + 31) / 32)};
      const cuuint64_t strides[2] = {(cuuint64_t)V * sizeof(float), 128};
      const cuuint32_t box[3] = {32, 8, 16};
      const cuuint32_t estr[3] = {1, 1, 1};
      // (mma.sync: the standard 128-byte swizzle, whose 16-byte chunks make
      // the fragment loads conflict-free)
      r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(gbase), dims,
                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 use_tc == 1 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t dims[2] = {(cuuint64_t)V, (cuuint64_t)(gtotal / V)};
      const cuuint64_t strides[1] = {(cuuint64_t)V * sizeof(float)};
      const cuuint32_t box[2] = {(cuuint32_t)bl::kTmaBoxCols, (cuuint32_t)bl::kTmaRows};
      const cuuint32_t estr[2] = {1, 1};
      r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gbase), dims,
                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS)
      throw BlError{BL_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
  }
  p.sc_rowsf = static_cast<const float*>(d->sc_rowsf.p);
  p.xs = static_cast<double*>(d->xs.p);
  p.taken = static_cast<unsigned char*>(d->taken.p);
  p.hist = static_cast<bl::HistRec*>(d->hist.p);
  p.fin = static_cast<bl::FinEntry*>(d->fin.p);
  p.res = static_cast<int*>(d->res.p);
  p.res_stride = rs;
  p.cnt = static_cast<unsigned long long*>(d->cnt.p);
  p.utts = static_cast<const bl::UttDesc*>(d->utts.p);
  p.prof = nullptr;
  if (d->profile) {
    d->prof.ensure(sizeof(long long) * (size_t)U * 16);
    d->h_prof.ensure(sizeof(long long) * (size_t)U * 16);
    CK(cudaMemsetAsync(d->prof.p, 0, sizeof(long long) * (size_t)U * 16, st));
    p.prof = static_cast<long long*>(d->prof.p);
  }

  for (int i = 0; i < n; ++i) {
    desc[i].grid = on_device ? utts[i].logp
                             : static_cast<const float*>(d->grid.p) + goff[i];
    desc[i].row0 = (int)(goff[i] / V);
    desc[i].chunk = 0;
  }
  // Streamed host input: ONE launch; the copy stream lands the grids chunk
  // by chunk and flags each one, and every CTA starts as soon as its own
  // chunk is in HBM.
  const bool stepm0 = d->step_mode != 0 || d->net != nullptr;
  const bool stream_in = !on_device && !stepm0 && U >= 296 &&
                         std::getenv("BL_NO_STREAM_IN") == nullptr;
  std::vector<int> bnd{0};
  if (stream_in) {
    // 32-utterance chunks while the first two waves of CTAs ramp up (each
    // starts as soon as its own chunk lands), then doubling up to 1024
    int want = 32;
    while (bnd.back() < U) {
      int b = std::min(U, bnd.back() + want);
      while (b < U && ((goff[b] * sizeof(float)) & 127) != 0) ++b;  // no shared 128-B line
      bnd.push_back(b);
      if (b >= 888) want = std::min(2 * want, 1024);
    }
    for (size_t k = 0; k + 1 < bnd.size(); ++k)
      for (int i = bnd[k]; i < bnd[k + 1]; ++i) desc[i].chunk = (int)k;
    const size_t nck = bnd.size() - 1;
    if (d->ready_n < nck) {
      d->ready.ensure(sizeof(unsigned) * nck);
      CK(cudaMemsetAsync(d->ready.p, 0, sizeof(unsigned) * nck, st));
      d->ready_n = nck;
    }
    d->stream_err.ensure(sizeof(int));
    d->h_epoch.ensure(sizeof(unsigned));
    d->h_err.ensure(sizeof(int));
    if (++d->epoch == 0) d->epoch = 1;
    *static_cast<unsigned*>(d->h_epoch.p) = d->epoch;
    CK(cudaMemsetAsync(d->stream_err.p, 0, sizeof(int), st));
    if (!d->ev_copied) CK(cudaEventCreateWithFlags(&d->ev_copied, cudaEventDisableTiming));
    p.ready = static_cast<const unsigned*>(d->ready.p);
    p.ready_epoch = d->epoch;
    p.stream_err = static_cast<int*>(d->stream_err.p);
  }
  std::memcpy(d->h_utts.p, desc.data(), sizeof(bl::UttDesc) * U);
  {
    // dynamic plan + the variant's static shared memory against the opt-in limit
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d->device);
    if (bl::decode_smem_bytes(p) + bl::decode_static_smem(p) > (size_t)optin)
      throw std::invalid_argument(
          "utterance too long for the device decoder's shared memory plan (" +
          std::to_string(Tmax) + " frames, vocab " + std::to_string(V) +
          "): hard-segment it (bl_hard_segments)");
  }

  CK(cudaMemcpyAsync(d->utts.p, d->h_utts.p, sizeof(bl::UttDesc) * U,
                     cudaMemcpyHostToDevice, st));
  // chunking: one launch when grids are resident; otherwise ~600 utterances
  // (two waves of resident CTAs) per chunk so copies overlap decoding.
  // Step-granular mode: one group, one launch per decode step.
  const bool stepm = d->step_mode != 0 || d->net != nullptr;
  if (d->net) {
    if (!d->memory)
      throw std::invalid_argument("the transformer scorer needs the encoder memory "
                                  "(bl_decode_memory)");
  }
  const int nchunk = (on_device || stepm || stream_in) ? 1 : std::max(1, std::min(16, U / 360));
  if ((int)d->ev_copy.size() < nchunk) {
    for (int k = (int)d->ev_copy.size(); k < nchunk; ++k) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      d->ev_copy.push_back(e);
    }
  }
  const auto t_launch = clk::now();
  CK(cudaEventRecord(d->ev0, st));  // timing start; copies start after the descriptors
  if (!on_device) CK(cudaStreamWaitEvent(d->copy, d->ev0, 0));
  if (nchunk > 1) CK(cudaStreamWaitEvent(d->alt, d->ev0, 0));
  int launches = 0;
  if (stream_in) {
    // copies and flags are enqueued BEFORE the kernel: under serialising
    // tools (CUDA_LAUNCH_BLOCKING=1, profiler kernel replay) every flag is
    // then already set when the kernel runs, instead of never arriving
    CK(cudaStreamWaitEvent(d->copy, d->ev0, 0));
    unsigned* rdy = static_cast<unsigned*>(d->ready.p);
    for (size_t k = 0; k + 1 < bnd.size(); ++k) {
      const int a = bnd[k], b = bnd[k + 1];
      for (const auto& r : runs) {
        const int i0 = std::max(r.i0, a), i1 = std::min(r.i1, b);
        if (i0 >= i1) continue;
        const size_t len = goff[i1 - 1] + (size_t)desc[i1 - 1].T * V - goff[i0];
        CK(cudaMemcpyAsync(static_cast<float*>(d->grid.p) + goff[i0],
                           r.src + (goff[i0] - goff[r.i0]), sizeof(float) * len,
                           cudaMemcpyHostToDevice, d->copy));
        res->h2d += sizeof(float) * len;
      }
      CK(cudaMemcpyAsync(rdy + k, d->h_epoch.p, sizeof(unsigned), cudaMemcpyHostToDevice,
                         d->copy));
    }
    CK(cudaEventRecord(d->ev_copied, d->copy));
    CK(bl::launch_decode(p, st));
    ++launches;
    CK(cudaStreamWaitEvent(st, d->ev_copied, 0));
  }
  for (int k = 0; k < nchunk && !stream_in; ++k) {
    const int a = (int)((long long)U * k / nchunk), b = (int)((long long)U * (k + 1) / nchunk);
    if (!on_device) {
      for (const auto& r : runs) {
        const int i0 = std::max(r.i0, a), i1 = std::min(r.i1, b);
        if (i0 >= i1) continue;
        const size_t len = goff[i1 - 1] + (size_t)desc[i1 - 1].T * V - goff[i0];
        CK(cudaMemcpyAsync(static_cast<float*>(d->grid.p) + goff[i0],
                           r.src + (goff[i0] - goff[r.i0]), sizeof(float) * len,
                           cudaMemcpyHostToDevice, d->copy));
        res->h2d += sizeof(float) * len;
      }
      CK(cudaEventRecord(d->ev_copy[k], d->copy));
    }
    cudaStream_t cs = (k & 1) ? d->alt : st;
    if (!on_device) CK(cudaStreamWaitEvent(cs, d->ev_copy[k], 0));
    bl::KParams pk = p;
    pk.u0 = a;
    pk.U = b - a;
    if (stepm) {
      launches += step_loop(d, pk, cs);
    } else {
      CK(bl::launch_decode(pk, cs));
      ++launches;
    }
  }
  if (nchunk > 1) {
    CK(cudaEventRecord(d->ev_alt, d->alt));
    CK(cudaStreamWaitEvent(st, d->ev_alt, 0));
  }
  CK(cudaEventRecord(d->ev1, st));
  // 1-best export into page-locked caller arrays: headers, tokens and label
  // times go straight to their final [n][cap] rows (three 2D copies, no
  // host-side repacking); otherwise the whole result block is copied.
  bool direct = false;
  if (into && into->cap >= S) {
    cudaPointerAttributes a{}, b{};
    direct = cudaPointerGetAttributes(&a, into->tokens) == cudaSuccess &&
             a.type == cudaMemoryTypeHost &&
             cudaPointerGetAttributes(&b, into->label_times) == cudaSuccess &&
             b.type == cudaMemoryTypeHost;
    cudaGetLastError();
  }
  const int* dres = static_cast<const int*>(d->res.p);
  if (d->keep_rows) {
    // group decode: records stay in d->res for the NCCL gather
  } else if (direct) {
    const size_t sp = sizeof(int) * (size_t)rs, dp = sizeof(int) * (size_t)into->cap;
    CK(cudaMemcpy2DAsync(d->h_res.p, sizeof(int) * bl::kResHdr, dres, sp,
                         sizeof(int) * bl::kResHdr, U, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpy2DAsync(into->tokens, dp, dres + bl::kResHdr, sp, sizeof(int) * (size_t)S, U,
                         cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpy2DAsync(into->label_times, dp, dres + bl::kResHdr + S, sp,
                         sizeof(int) * (size_t)S, U, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(d->h_res.p, dres, sizeof(int) * (size_t)U * rs, cudaMemcpyDeviceToHost,
                       st));
  }
  CK(cudaMemcpyAsync(d->h_cnt.p, d->cnt.p, sizeof(unsigned long long) * (size_t)U * 8,
                     cudaMemcpyDeviceToHost, st));
  if (stream_in)
    CK(cudaMemcpyAsync(d->h_err.p, d->stream_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (d->profile)
    CK(cudaMemcpyAsync(d->h_prof.p, d->prof.p, sizeof(long long) * (size_t)U * 16,
                       cudaMemcpyDeviceToHost, st));
  const auto t_enq = clk::now();
  CK(cudaStreamSynchronize(st));
  const auto t_sync = clk::now();
  if (stream_in && *static_cast<const int*>(d->h_err.p))
    throw BlError{BL_CUDA_ERROR, "streamed input: a grid chunk never reached the device"};
  if (d->profile) {
    const long long* hp = static_cast<const long long*>(d->h_prof.p);
    for (int i = 0; i < U; ++i)
      for (int k = 0; k < 16; ++k) res->prof[k] += (double)hp[(size_t)i * 16 + k] / U;
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, d->ev0, d->ev1));
  res->kernel_ms = ms;
  res->launches = launches;
  res->d2h = (d->keep_rows ? 0
                            : direct ? sizeof(int) * (size_t)U * (bl::kResHdr + 2 * (size_t)S)
                                     : sizeof(int) * (size_t)U * rs) +
             sizeof(unsigned long long) * (size_t)U * 8;
  if (d->keep_rows) {  // counters and stats only; the group assembles the results
    const unsigned long long* hc = static_cast<const unsigned long long*>(d->h_cnt.p);
    for (int i = 0; i < n; ++i) {
      const unsigned long long* c = hc + (size_t)i * 8;
      res->steps += c[0];
      res->queries += c[1];
      res->frames += c[2];
      res->k1 += c[3];
      res->fallback += c[4] & 0xffffffffull;
      res->contenders += c[5];
      res->raw_keys += c[6];
      res->wide += c[4] >> 32;
    }
    res->max_tokens = S;
    *out = res.release();
    return BL_OK;
  }

  const int* hr = static_cast<const int*>(d->h_res.p);
  const unsigned long long* hc = static_cast<const unsigned long long*>(d->h_cnt.p);
  if (into) {
    for (int i = 0; i < n; ++i) {
      const int* r = hr + (size_t)i * (direct ? bl::kResHdr : rs);
      const int nt = r[0];
      if (nt > into->cap) throw std::invalid_argument("result longer than the export capacity");
      into->n_tokens[i] = nt;
      into->steps[i] = r[1];
      into->trigger[i] = r[2];
      std::memcpy(into->joint + i, r + 4, sizeof(double));
      if (!direct) {
        std::memcpy(into->tokens + (size_t)i * into->cap, r + bl::kResHdr, sizeof(int) * nt);
        std::memcpy(into->label_times + (size_t)i * into->cap, r + bl::kResHdr + S,
                    sizeof(int) * nt);
      }
      res->max_tokens = std::max(res->max_tokens, nt);
      const unsigned long long* c = hc + (size_t)i * 8;
      res->steps += c[0];
      res->queries += c[1];
      res->frames += c[2];
      res->k1 += c[3];
      res->fallback += c[4] & 0xffffffffull;
      res->contenders += c[5];
      res->raw_keys += c[6];
      res->wide += c[4] >> 32;
    }
    if (host_timing) {
      auto ms = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
      };
      std::fprintf(stderr, "[bl host] plan %.3f  enqueue %.3f  wait %.3f (kernel %.3f)  export %.3f ms\n",
                   ms(t_in, t_launch), ms(t_launch, t_enq), ms(t_enq, t_sync), res->kernel_ms,
                   ms(t_sync, clk::now()));
    }
    *out = res.release();  // counters and stats only
    return BL_OK;
  }
  res->r.resize(n);
  for (int i = 0; i < n; ++i) {
    const int* r = hr + (size_t)i * rs;
    auto& o = res->r[i];
    o.id = utts[i].id ? utts[i].id : "";
    const int nt = r[0];
    o.steps = r[1];
    o.trigger = r[2];
    std::memcpy(&o.joint, r + 4, sizeof(double));
    o.tokens.assign(r + bl::kResHdr, r + bl::kResHdr + nt);
    res->max_tokens = std::max(res->max_tokens, nt);
    o.label_times.assign(r + bl::kResHdr + S, r + bl::kResHdr + S + nt);
    const int nn = r[3];
    for (int k = 0; k < nn; ++k) {
      const int* q = r + bl::kResHdr + 2 * S + k * (4 + 2 * S);
      double jv;
      std::memcpy(&jv, q + 2, sizeof(double));
      o.nb_joint.push_back(jv);
      o.nb_tokens.emplace_back(q + 4, q + 4 + q[0]);
      o.nb_times.emplace_back(q + 4 + S, q + 4 + S + q[0]);
    }
    const unsigned long long* c = hc + (size_t)i * 8;
    res->steps += c[0];
    res->queries += c[1];
    res->frames += c[2];
    res->k1 += c[3];
    res->fallback += c[4] & 0xffffffffull;
    res->contenders += c[5];
    res->raw_keys += c[6];
    res->wide += c[4] >> 32;
  }
  *out = res.release();
  return BL_OK;
}

}  // namespace

// ----------------------------------------------------------- model files
// One binary file with the network weights of a model: "BLM1", u32 version
// (1), u32 section count, then per section u32 kind (1 = encoder, 2 =
// decoder), u32 spec[6] (encoder: idim d_model heads d_ff layers vocab;
// decoder: d_model heads d_ff layers vocab 0), u64 count, float32[count] in
// the flat layouts of bl_encoder_create / bl_scorer_create_transformer.
// Little-endian. The reference's "model load" hook is make_scorer
// (scorer.hpp:84); "transformer:PATH" loads the decoder section.
struct ModelFile {
  bool has_enc = false, has_dec = false;
  bl_encoder_spec enc{};
  bl_transformer_spec dec{};
  std::vector<float> enc_w, dec_w;
};

ModelFile read_model(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw std::runtime_error("cannot open model file: " + path);
  auto u32 = [&]() {
    uint32_t v = 0;
    is.read(reinterpret_cast<char*>(&v), 4);
    if (!is) throw std::runtime_error("truncated model file: " + path);
    return v;
  };
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, "BLM1", 4) != 0)
    throw std::runtime_error("bad magic in model file: " + path);
  if (u32() != 1) throw std::runtime_error("unsupported model file version in " + path);
  const uint32_t nsec = u32();
  ModelFile mf;
  for (uint32_t k = 0; k < nsec; ++k) {
    const uint32_t kind = u32();
    uint32_t sp[6];
    for (auto& x : sp) x = u32();
    uint64_t count = 0;
    is.read(reinterpret_cast<char*>(&count), 8);
    if (!is || count > (1ull << 34)) throw std::runtime_error("bad section in " + path);
    std::vector<float> w(count);
    is.read(reinterpret_cast<char*>(w.data()), (std::streamsize)(count * sizeof(float)));
    if (!is) throw std::runtime_error("truncated model file: " + path);
    if (kind == 1) {
      mf.has_enc = true;
      mf.enc = {(int)sp[0], (int)sp[1], (int)sp[2], (int)sp[3], (int)sp[4], (int)sp[5]};
      mf.enc_w = std::move(w);
    } else if (kind == 2) {
      mf.has_dec = true;
      mf.dec = {(int)sp[0], (int)sp[1], (int)sp[2], (int)sp[3], (int)sp[4]};
      mf.dec_w = std::move(w);
    } else {
      throw std::runtime_error("unknown section kind in " + path);
    }
  }
  return mf;
}

// ====================================================================== C ABI
extern "C" {

const char* bl_last_error(void) { return g_err.c_str(); }

void bl_config_default(bl_config* c) {  // beam_search.hpp:21-33
  c->beam_width = 3;
  c->ctc_weight = 0.3;
  c->eos_m = 3;
  c->eos_dend = -10.0;
  c->eos_c = 2;
  c->margin_m1 = 5;
  c->margin_m2 = BL_NO_MARGIN;
  c->eos_mode = BL_EOS_BOTH;
  c->max_steps_ratio = 1.0;
}

int bl_config_validate(const bl_config* c) {
  return guarded([&] {
    validate_cfg(*c);
    return BL_OK;
  });
}

// hard_segments / split_uniform (segmentation.cpp:65-75, 121-133)
int bl_hard_segments(int T, int min_len, int max_len, int* starts, int* ends,
                     int cap, int* n_out) {
  return guarded([&] {
    if (T < 1) throw std::invalid_argument("hard_segments: T < 1");
    if (!(min_len > 0 && min_len <= max_len))
      throw std::invalid_argument("hard_segments: need 0 < min_len <= max_len");
    int n = 0;
    auto emit = [&](int s, int e) {
      if (n < cap) {
        starts[n] = s;
        ends[n] = e;
      }
      ++n;
    };
    if (T < min_len) {
      emit(0, T);
    } else {
      const int len = T;
      const int pieces = (len + max_len - 1) / max_len;
      int offset = 0;
      for (int k = 0; k < pieces; ++k) {
        const int piece = len / pieces + (k < len % pieces ? 1 : 0);
        emit(offset, offset + piece);
        offset += piece;
      }
    }
    *n_out = n;
    return BL_OK;
  });
}

// VAD segmentation (segmentation.cpp:13-119): per-frame LLR = max noise
// output - max speech output (frame_llr), centred moving average by prefix
// sums and threshold with ties as speech (smooth_and_decide), maximal speech
// runs merged left to right until >= min_len, then near-uniform splits of at
// most max_len (vad_segments). Same operation order, so same decisions.
int bl_vad_segments(const float* outputs, int T, int num_nodes, const int* speech, int n_speech,
                    const int* noise, int n_noise, double threshold, int smooth_window,
                    int min_len, int max_len, int* starts, int* ends, int cap, int* n_out) {
  return guarded([&] {
    if (n_speech < 1 || n_noise < 1)
      throw std::invalid_argument("nodemap: speech and noise sets must be non-empty");
    for (int i = 0; i < n_noise; ++i)
      for (int j = 0; j < n_speech; ++j)
        if (noise[i] == speech[j])
          throw std::invalid_argument("nodemap: speech and noise sets overlap");
    for (int j = 0; j < n_speech; ++j)
      if (speech[j] < 0 || speech[j] >= num_nodes)
        throw std::invalid_argument("nodemap: speech node out of range");
    for (int i = 0; i < n_noise; ++i)
      if (noise[i] < 0 || noise[i] >= num_nodes)
        throw std::invalid_argument("nodemap: noise node out of range");
    if (smooth_window < 1) throw std::invalid_argument("vad: smoothing window must be >= 1");
    if (!(min_len > 0 && min_len <= max_len))
      throw std::invalid_argument("vad: need 0 < min_len <= max_len");
    if (T < 0) throw std::invalid_argument("vad: T < 0");
    std::vector<double> llr(T);
    for (int t = 0; t < T; ++t) {
      const float* row = outputs + (size_t)t * num_nodes;
      double sp = -HUGE_VAL, no = -HUGE_VAL;
      for (int j = 0; j < n_speech; ++j) sp = std::max(sp, (double)row[speech[j]]);
      for (int i = 0; i < n_noise; ++i) no = std::max(no, (double)row[noise[i]]);
      llr[t] = no - sp;
    }
    std::vector<double> prefix(T + 1, 0.0);
    for (int t = 0; t < T; ++t) prefix[t + 1] = prefix[t] + llr[t];
    const int half_lo = (smooth_window - 1) / 2, half_hi = smooth_window / 2;
    std::vector<char> sp(T);
    for (int t = 0; t < T; ++t) {
      const int lo = std::max(0, t - half_lo), hi = std::min(T - 1, t + half_hi);
      const double mean = (prefix[hi + 1] - prefix[lo]) / (hi - lo + 1);
      sp[t] = mean <= threshold;
    }
    std::vector<std::pair<int, int>> runs, merged;
    for (int t = 0; t < T;) {
      if (!sp[t]) {
        ++t;
        continue;
      }
      const int a = t;
      while (t < T && sp[t]) ++t;
      runs.emplace_back(a, t);
    }
    for (size_t r = 0; r < runs.size();) {
      int a = runs[r].first, b = runs[r].second;
      ++r;
      while (b - a < min_len && r < runs.size()) b = runs[r++].second;
      merged.emplace_back(a, b);
    }
    int n = 0;
    for (auto [a, b] : merged) {
      const int len = b - a, pieces = (len + max_len - 1) / max_len;
      int off = a;
      for (int k = 0; k < pieces; ++k) {
        const int piece = len / pieces + (k < len % pieces ? 1 : 0);
        if (n < cap) {
          starts[n] = off;
          ends[n] = off + piece;
        }
        ++n;
        off += piece;
      }
    }
    *n_out = n;
    return BL_OK;
  });
}

// make_batches (batched.cpp:12-30)
int bl_make_batches(int n, const uint32_t* frames, int batch_size, int* order,
                    int* n_batches) {
  return guarded([&] {
    if (batch_size < 1) throw std::invalid_argument("batch size must be >= 1");
    std::vector<int> idx(n);
    for (int i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int a, int b) { return frames[a] < frames[b]; });
    for (int i = 0; i < n; ++i) order[i] = idx[i];
    *n_batches = (n + batch_size - 1) / batch_size;
    return BL_OK;
  });
}

// make_scorer (scorer.cpp:117-135)
int bl_scorer_create(const char* spec_c, int num_tokens, bl_scorer** out) {
  return guarded([&] {
    const std::string spec(spec_c ? spec_c : "");
    if (spec == "uniform") {
      if (num_tokens < 1) throw std::invalid_argument("UniformScorer: |C| < 1");
      auto* s = new bl_scorer;
      s->num_tokens = num_tokens;
      *out = s;
      return BL_OK;
    }
    if (spec.rfind("table:", 0) == 0) {
      std::unique_ptr<bl_scorer> s(load_table(spec.substr(6)));
      if (s->num_tokens != num_tokens)
        throw std::runtime_error("table scorer vocabulary does not match grids");
      *out = s.release();
      return BL_OK;
    }
    if (spec.rfind("loop:", 0) == 0) {
      std::string rest = spec.substr(5);
      auto colon = rest.find(':');
      if (colon == std::string::npos)
        throw std::runtime_error("loop scorer spec must be loop:TOKEN:P");
      int token = std::stoi(rest.substr(0, colon));
      double p = std::stod(rest.substr(colon + 1));
      *out = make_loop(num_tokens, token, p);
      return BL_OK;
    }
    if (spec.rfind("transformer:", 0) == 0) {
      // "transformer:PATH[@DEVICE]": the decoder section of a model file
      // (bl_model_save), loaded onto DEVICE (default 0)
      std::string path = spec.substr(12);
      int device = 0;
      const auto at = path.rfind('@');
      if (at != std::string::npos) {
        device = std::stoi(path.substr(at + 1));
        path = path.substr(0, at);
      }
      ModelFile mf = read_model(path);
      if (!mf.has_dec) throw std::runtime_error("model file has no decoder section: " + path);
      if (mf.dec.vocab - 1 != num_tokens)
        throw std::runtime_error("transformer scorer vocabulary does not match grids");
      const int rc = bl_scorer_create_transformer(device, &mf.dec, mf.dec_w.data(),
                                                  mf.dec_w.size(), out);
      if (rc != BL_OK) throw BlError{rc, g_err};
      return BL_OK;
    }
    throw std::runtime_error("unknown scorer spec: " + spec);
  });
}

int bl_scorer_create_table(int num_tokens, int order, int n_entries,
                           const int* ctx_len, const int* ctx, const double* logp,
                           bl_scorer** out) {
  return guarded([&] {
    std::unique_ptr<bl_scorer> s(make_table(num_tokens, order));
    const int w = std::max(order - 1, 1);
    for (int k = 0; k < n_entries; ++k) {  // TableScorer::add_entry
      std::vector<double> lp(logp + (size_t)k * (num_tokens + 1),
                             logp + (size_t)(k + 1) * (num_tokens + 1));
      check_normalized(lp, static_cast<size_t>(num_tokens) + 1, "TableScorer entry");
      s->table[std::vector<int>(ctx + (size_t)k * w, ctx + (size_t)k * w + ctx_len[k])] =
          std::move(lp);
    }
    *out = s.release();
    return BL_OK;
  });
}

int bl_scorer_create_loop(int num_tokens, int loop_token, double p, bl_scorer** out) {
  return guarded([&] {
    *out = make_loop(num_tokens, loop_token, p);
    return BL_OK;
  });
}

int bl_scorer_num_tokens(const bl_scorer* s) { return s ? s->num_tokens : -1; }

int bl_scorer_score(const bl_scorer* s, const int* prefix, int n, double* out) {
  return guarded([&] {
    auto v = s->score(std::vector<int>(prefix, prefix + n));
    std::copy(v.begin(), v.end(), out);
    return BL_OK;
  });
}

void bl_scorer_destroy(bl_scorer* s) { delete s; }

static bl::DecSpec dec_spec_of(const bl_transformer_spec* s) {
  return bl::DecSpec{s->d_model, s->heads, s->d_ff, s->layers, s->vocab};
}

size_t bl_transformer_num_weights(const bl_transformer_spec* spec) {
  if (!spec || !bl::dec_validate(dec_spec_of(spec)).empty()) return 0;
  return bl::dec_num_weights(dec_spec_of(spec));
}

int bl_scorer_create_transformer(int device, const bl_transformer_spec* spec,
                                 const float* weights, size_t n_weights, bl_scorer** out) {
  return guarded([&] {
    if (!spec || !weights || !out) throw std::invalid_argument("null argument");
    const bl::DecSpec s = dec_spec_of(spec);
    const std::string why = bl::dec_validate(s);
    if (!why.empty()) throw std::invalid_argument(why);
    if (n_weights != bl::dec_num_weights(s))
      throw std::invalid_argument("decoder weight count mismatch: expected " +
                                  std::to_string(bl::dec_num_weights(s)) + ", got " +
                                  std::to_string(n_weights));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
      throw BlError{BL_CUDA_ERROR, "no CUDA device " + std::to_string(device)};
    CK(cudaSetDevice(device));
    std::unique_ptr<bl_scorer> sc(new bl_scorer);
    sc->kind = 3;
    sc->num_tokens = s.vocab - 1;
    sc->net_device = device;
    CK(bl::dec_create(s, weights, &sc->net));
    *out = sc.release();
    return BL_OK;
  });
}

int bl_decoder_create(int device, const bl_config* cfg, const bl_scorer* scorer,
                      bl_decoder** out) {
  return guarded([&] {
    validate_cfg(*cfg);
    if (!scorer) throw std::invalid_argument("scorer is required");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
      throw BlError{BL_CUDA_ERROR, "no CUDA device " + std::to_string(device)};
    CK(cudaSetDevice(device));
    std::unique_ptr<bl_decoder> d(new bl_decoder);
    d->device = device;
    d->cfg = *cfg;
    d->num_tokens = scorer->num_tokens;
    CK(cudaStreamCreateWithFlags(&d->own, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&d->copy, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&d->alt, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&d->ev_alt, cudaEventDisableTiming));
    d->stream = d->own;
    CK(cudaEventCreate(&d->ev0));
    CK(cudaEventCreate(&d->ev1));
    upload_scorer(d.get(), scorer);
    *out = d.release();
    return BL_OK;
  });
}

int bl_decoder_set_options(bl_decoder* d, int nbest, int exact, double slack) {
  return guarded([&] {
    if (nbest < 1) throw std::invalid_argument("nbest must be >= 1");
    if (!(slack >= 1.0)) throw std::invalid_argument("slack must be >= 1");
    d->nbest = nbest;
    d->exact = exact ? 1 : 0;
    d->slack = slack;
    return BL_OK;
  });
}

int bl_decoder_set_record(bl_decoder* d, int on) {
  d->record = on ? 1 : 0;
  d->rec.clear();
  return BL_OK;
}

int bl_decoder_record_count(const bl_decoder* d) { return (int)d->rec.size(); }

int bl_decoder_record_get(const bl_decoder* d, int i, int* utt, int* len, const int** prefix,
                          const double** row) {
  if (i < 0 || i >= (int)d->rec.size()) return fail(BL_INVALID_ARGUMENT, "record index out of range");
  const auto& r = d->rec[i];
  *utt = r.utt;
  *len = (int)r.prefix.size();
  *prefix = r.prefix.data();
  *row = r.row.data();
  return BL_OK;
}

int bl_decoder_set_step_mode(bl_decoder* d, int on) {
  d->step_mode = on ? 1 : 0;
  return BL_OK;
}

int bl_decoder_set_stream(bl_decoder* d, void* stream) {
  d->stream = stream ? static_cast<cudaStream_t>(stream) : d->own;
  return BL_OK;
}

void bl_decoder_destroy(bl_decoder* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  cudaStreamSynchronize(d->stream);
  if (d->ev0) cudaEventDestroy(d->ev0);
  if (d->ev1) cudaEventDestroy(d->ev1);
  for (auto e : d->ev_copy) cudaEventDestroy(e);
  if (d->copy) cudaStreamDestroy(d->copy);
  if (d->alt) cudaStreamDestroy(d->alt);
  if (d->ev_alt) cudaEventDestroy(d->ev_alt);
  if (d->ev_copied) cudaEventDestroy(d->ev_copied);
  if (d->own) cudaStreamDestroy(d->own);
  delete d;
}

int bl_decode(bl_decoder* d, int n, const bl_utt* utts, int on_device,
              bl_results** out) {
  return guarded([&] {
    d->memory = nullptr;
    d->mem_frames = 0;
    return decode_impl(d, n, utts, on_device, out);
  });
}

int bl_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("bl_host_alloc: null out");
    *out = nullptr;
    CK(cudaMallocHost(out, bytes ? bytes : 1));
    return BL_OK;
  });
}

void bl_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int bl_decode_into(bl_decoder* d, int n, const bl_utt* utts, int grids_on_device,
                   const void* memory, int mem_frames, int cap, int* n_tokens, int* steps,
                   int* trigger, double* joint, int* tokens, int* label_times,
                   bl_results** stats) {
  return guarded([&] {
    if (cap < 1 || !n_tokens || !steps || !trigger || !joint || !tokens || !label_times)
      throw std::invalid_argument("bl_decode_into: null output or cap < 1");
    if (memory && !d->net) throw std::invalid_argument("memory needs a transformer scorer");
    d->memory = memory;
    d->mem_frames = memory ? mem_frames : 0;
    if (memory && mem_frames < 1) throw std::invalid_argument("memory frames must be >= 1");
    d->rec.clear();
    IntoArgs ia{cap, n_tokens, steps, trigger, tokens, label_times, joint};
    const int r = decode_impl(d, n, utts, grids_on_device, stats, &ia);
    d->memory = nullptr;
    return r;
  });
}

int bl_decode_memory(bl_decoder* d, int n, const bl_utt* utts, int grids_on_device,
                     const void* memory, int mem_frames, bl_results** out) {
  return guarded([&] {
    if (!d->net) throw std::invalid_argument("bl_decode_memory needs a transformer scorer");
    if (!memory || mem_frames < 1) throw std::invalid_argument("memory frames must be >= 1");
    d->memory = memory;
    d->mem_frames = mem_frames;
    d->rec.clear();
    const int r = decode_impl(d, n, utts, grids_on_device, out);
    d->memory = nullptr;
    return r;
  });
}

int bl_results_count(const bl_results* r) { return (int)r->r.size(); }
int bl_results_filter_keys(const bl_results* r, uint64_t* raw_keys) {
  *raw_keys = r->raw_keys;
  return BL_OK;
}
int bl_results_wide_steps(const bl_results* r, uint64_t* wide_steps) {
  *wide_steps = r->wide;
  return BL_OK;
}
int bl_results_max_tokens(const bl_results* r) { return r->max_tokens; }

int bl_results_get(const bl_results* r, int i, const char** id, const int** tokens,
                   int* n_tokens, double* joint, const int** label_times, int* steps,
                   int* trigger) {
  if (i < 0 || i >= (int)r->r.size()) return fail(BL_INVALID_ARGUMENT, "result index out of range");
  const auto& o = r->r[i];
  if (id) *id = o.id.c_str();
  if (tokens) *tokens = o.tokens.data();
  if (n_tokens) *n_tokens = (int)o.tokens.size();
  if (joint) *joint = o.joint;
  if (label_times) *label_times = o.label_times.data();
  if (steps) *steps = o.steps;
  if (trigger) *trigger = o.trigger;
  return BL_OK;
}

int bl_results_nbest_count(const bl_results* r, int i) {
  if (i < 0 || i >= (int)r->r.size()) return 0;
  return (int)r->r[i].nb_joint.size();
}

int bl_results_nbest(const bl_results* r, int i, int k, const int** tokens,
                     int* n_tokens, double* joint, const int** label_times) {
  if (i < 0 || i >= (int)r->r.size() || k < 0 || k >= (int)r->r[i].nb_joint.size())
    return fail(BL_INVALID_ARGUMENT, "n-best index out of range");
  const auto& o = r->r[i];
  if (tokens) *tokens = o.nb_tokens[k].data();
  if (n_tokens) *n_tokens = (int)o.nb_tokens[k].size();
  if (joint) *joint = o.nb_joint[k];
  if (label_times) *label_times = o.nb_times[k].data();
  return BL_OK;
}

int bl_results_counters(const bl_results* r, uint64_t* steps, uint64_t* q, uint64_t* f) {
  if (steps) *steps = r->steps;
  if (q) *q = r->queries;
  if (f) *f = r->frames;
  return BL_OK;
}

int bl_results_stats(const bl_results* r, double* kernel_ms, uint64_t* k1,
                     int* launches, uint64_t* fallback, uint64_t* contenders) {
  if (kernel_ms) *kernel_ms = r->kernel_ms;
  if (k1) *k1 = r->k1;
  if (launches) *launches = r->launches;
  if (fallback) *fallback = r->fallback;
  if (contenders) *contenders = r->contenders;
  return BL_OK;
}

int bl_results_export(const bl_results* r, int cap, int* n_tokens, int* steps, int* trigger,
                      double* joint, int* tokens, int* label_times) {
  for (size_t i = 0; i < r->r.size(); ++i) {
    const auto& o = r->r[i];
    const int n = (int)o.tokens.size();
    if (n > cap) return fail(BL_INVALID_ARGUMENT, "result longer than the export capacity");
    n_tokens[i] = n;
    steps[i] = o.steps;
    trigger[i] = o.trigger;
    joint[i] = o.joint;
    std::memcpy(tokens + i * (size_t)cap, o.tokens.data(), sizeof(int) * n);
    std::memcpy(label_times + i * (size_t)cap, o.label_times.data(), sizeof(int) * n);
  }
  return BL_OK;
}

int bl_results_transfer(const bl_results* r, uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = r->h2d;
  if (d2h) *d2h = r->d2h;
  return BL_OK;
}

int bl_results_profile(const bl_results* r, double* out16) {
  for (int k = 0; k < 16; ++k) out16[k] = r->prof[k];
  return BL_OK;
}

void bl_results_destroy(bl_results* r) { delete r; }


// ------------------------------------------------------------------ encoder
struct bl_encoder {
  int device = 0;
  bl_encoder_spec spec{};
  bl::EncoderImpl* impl = nullptr;
  cudaStream_t own = nullptr;
  int chunk = 148;  // 148 x 249 rows = 2 waves of 128-row tiles on 148 SMs
  int launches = 0;
};

static bl::EncSpec enc_spec(const bl_encoder_spec* s) {
  return bl::EncSpec{s->idim, s->d_model, s->heads, s->d_ff, s->layers, s->vocab};
}

int bl_encoder_frames_out(int frames_in) { return bl::enc_frames_out(frames_in); }

size_t bl_encoder_num_weights(const bl_encoder_spec* spec) {
  if (!spec || !bl::enc_validate(enc_spec(spec)).empty()) return 0;
  return bl::enc_num_weights(enc_spec(spec));
}

int bl_encoder_create(int device, const bl_encoder_spec* spec, const float* weights,
                      size_t n_weights, bl_encoder** out) {
  return guarded([&] {
    if (!spec || !weights || !out) throw std::invalid_argument("null argument");
    const bl::EncSpec s = enc_spec(spec);
    const std::string why = bl::enc_validate(s);
    if (!why.empty()) throw std::invalid_argument(why);
    if (n_weights != bl::enc_num_weights(s))
      throw std::invalid_argument("encoder weight count mismatch: expected " +
                                  std::to_string(bl::enc_num_weights(s)) + ", got " +
                                  std::to_string(n_weights));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
      throw BlError{BL_CUDA_ERROR, "no CUDA device " + std::to_string(device)};
    CK(cudaSetDevice(device));
    std::unique_ptr<bl_encoder> e(new bl_encoder);
    e->device = device;
    e->spec = *spec;
    CK(cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking));
    CK(bl::enc_create(s, weights, &e->impl));
    bl::enc_set_stream(e->impl, e->own);
    *out = e.release();
    return BL_OK;
  });
}

int bl_encoder_set_stream(bl_encoder* e, void* stream) {
  bl::enc_set_stream(e->impl, static_cast<cudaStream_t>(stream));
  return BL_OK;
}

int bl_encoder_set_chunk(bl_encoder* e, int segments) {
  if (segments < 1) return fail(BL_INVALID_ARGUMENT, "chunk must be >= 1");
  e->chunk = segments;
  return BL_OK;
}

int bl_encoder_forward(bl_encoder* e, int n, int frames_in, const float* fbank,
                       int fbank_on_device, float* grid, int sync) {
  return guarded([&] {
    if (n < 0) throw std::invalid_argument("segment count must be >= 0");
    if (n == 0) return BL_OK;
    if (!fbank || !grid) throw std::invalid_argument("null fbank or grid");
    if (bl::enc_frames_out(frames_in) < 1)
      throw std::invalid_argument("segment too short: " + std::to_string(frames_in) +
                                  " frames (need >= 7)");
    CK(cudaSetDevice(e->device));
    CK(bl::enc_forward(e->impl, n, frames_in, fbank, fbank_on_device != 0, grid, e->chunk,
                       &e->launches, nullptr));
    if (sync) CK(cudaStreamSynchronize(bl::enc_stream(e->impl)));
    return BL_OK;
  });
}

int bl_encoder_forward_mem(bl_encoder* e, int n, int frames_in, const float* fbank,
                           int fbank_on_device, float* grid, void* memory, int sync) {
  return guarded([&] {
    if (n < 0) throw std::invalid_argument("segment count must be >= 0");
    if (n == 0) return BL_OK;
    if (!fbank || !grid) throw std::invalid_argument("null fbank or grid");
    if (bl::enc_frames_out(frames_in) < 1)
      throw std::invalid_argument("segment too short: " + std::to_string(frames_in) +
                                  " frames (need >= 7)");
    CK(cudaSetDevice(e->device));
    CK(bl::enc_forward(e->impl, n, frames_in, fbank, fbank_on_device != 0, grid, e->chunk,
                       &e->launches, static_cast<__nv_bfloat16*>(memory)));
    if (sync) CK(cudaStreamSynchronize(bl::enc_stream(e->impl)));
    return BL_OK;
  });
}

int bl_encoder_launches(const bl_encoder* e) { return e->launches; }

void bl_encoder_destroy(bl_encoder* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(bl::enc_stream(e->impl));
  bl::enc_destroy(e->impl);
  if (e->own) cudaStreamDestroy(e->own);
  delete e;
}

int bl_model_save(const char* path, const bl_encoder_spec* enc, const float* enc_w,
                  size_t n_enc, const bl_transformer_spec* dec, const float* dec_w,
                  size_t n_dec) {
  return guarded([&] {
    if (!path) throw std::invalid_argument("null path");
    if (enc && n_enc != bl_encoder_num_weights(enc))
      throw std::invalid_argument("encoder weight count mismatch");
    if (dec && n_dec != bl_transformer_num_weights(dec))
      throw std::invalid_argument("decoder weight count mismatch");
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error(std::string("cannot write model file: ") + path);
    auto u32 = [&](uint32_t v) { os.write(reinterpret_cast<const char*>(&v), 4); };
    os.write("BLM1", 4);
    u32(1);
    u32((enc ? 1 : 0) + (dec ? 1 : 0));
    if (enc) {
      u32(1);
      for (int v : {enc->idim, enc->d_model, enc->heads, enc->d_ff, enc->layers, enc->vocab})
        u32((uint32_t)v);
      const uint64_t c = n_enc;
      os.write(reinterpret_cast<const char*>(&c), 8);
      os.write(reinterpret_cast<const char*>(enc_w), (std::streamsize)(n_enc * sizeof(float)));
    }
    if (dec) {
      u32(2);
      for (int v : {dec->d_model, dec->heads, dec->d_ff, dec->layers, dec->vocab, 0})
        u32((uint32_t)v);
      const uint64_t c = n_dec;
      os.write(reinterpret_cast<const char*>(&c), 8);
      os.write(reinterpret_cast<const char*>(dec_w), (std::streamsize)(n_dec * sizeof(float)));
    }
    if (!os) throw std::runtime_error(std::string("short write: ") + path);
    return BL_OK;
  });
}

int bl_encoder_create_from_file(int device, const char* path, bl_encoder** out) {
  return guarded([&] {
    if (!path) throw std::invalid_argument("null path");
    ModelFile mf = read_model(path);
    if (!mf.has_enc) throw std::runtime_error(std::string("model file has no encoder: ") + path);
    const int rc = bl_encoder_create(device, &mf.enc, mf.enc_w.data(), mf.enc_w.size(), out);
    if (rc != BL_OK) throw BlError{rc, g_err};
    return BL_OK;
  });
}

// segment -> slice -> encode -> batched decode for one long recording: the
// chaining the reference leaves to its CLI (tools/beamlattice.cpp:234-273
// segments, :117-146 decodes pre-cut grids). hard_segments
// (segmentation.cpp:121-133) gives at most two segment lengths; each length
// is one encoder call (grids, and the memory for a transformer scorer, stay
// in HBM) and one decode call. Results in segment order, ids
// "<rec>:<start>-<end>".
int bl_recognize(bl_encoder* e, bl_decoder* d, const float* fbank, int T, int idim,
                 const char* recording_id, int min_len, int max_len, bl_results** out) {
  return guarded([&] {
    if (!e || !d || !fbank || !out) throw std::invalid_argument("null argument");
    if (idim != e->spec.idim) throw std::invalid_argument("fbank dimension does not match the encoder");
    if (e->spec.vocab - 1 != d->num_tokens)
      throw std::invalid_argument("encoder vocabulary does not match the decoder's scorer");
    if (e->device != d->device) throw std::invalid_argument("encoder and decoder on different devices");
    const bool attn = d->net != nullptr;
    int nseg = 0;
    const int cap = T / std::max(1, max_len) + 2;
    std::vector<int> st(cap), en(cap);
    int rc = bl_hard_segments(T, min_len, max_len, st.data(), en.data(), cap, &nseg);
    if (rc != BL_OK) throw BlError{rc, g_err};
    const std::string rec = recording_id ? recording_id : "rec";
    std::map<int, std::vector<int>> groups;  // length -> segment indices
    for (int i = 0; i < nseg; ++i) groups[en[i] - st[i]].push_back(i);
    auto res = std::make_unique<bl_results>();
    res->r.resize(nseg);
    CK(cudaSetDevice(d->device));
    for (const auto& [len, idx] : groups) {
      const int T2 = bl::enc_frames_out(len);
      if (T2 < 1)
        throw std::invalid_argument("segment of " + std::to_string(len) +
                                    " frames is too short for the encoder");
      const int m = (int)idx.size();
      HostBuf slab;  // the group's segments back to back, page-locked
      slab.ensure(sizeof(float) * (size_t)m * len * idim);
      float* hs = static_cast<float*>(slab.p);
      for (int r = 0; r < m; ++r)
        std::memcpy(hs + (size_t)r * len * idim, fbank + (size_t)st[idx[r]] * idim,
                    sizeof(float) * (size_t)len * idim);
      DevBuf grid, mem;
      const int V = e->spec.vocab;
      grid.ensure(sizeof(float) * (size_t)m * T2 * V);
      if (attn) mem.ensure(2 * (size_t)m * T2 * e->spec.d_model);
      rc = bl_encoder_forward_mem(e, m, len, hs, 0, static_cast<float*>(grid.p),
                                  attn ? mem.p : nullptr, 1);
      if (rc != BL_OK) throw BlError{rc, g_err};
      std::vector<std::string> ids(m);
      std::vector<bl_utt> utts(m);
      for (int r = 0; r < m; ++r) {
        const int i = idx[r];
        ids[r] = rec + ":" + std::to_string(st[i]) + "-" + std::to_string(en[i]);
        utts[r] = {ids[r].c_str(), (uint32_t)T2, (uint32_t)V, 40,
                   static_cast<const float*>(grid.p) + (size_t)r * T2 * V};
      }
      bl_results* part = nullptr;
      rc = attn ? bl_decode_memory(d, m, utts.data(), 1, mem.p, T2, &part)
                : bl_decode(d, m, utts.data(), 1, &part);
      if (rc != BL_OK) throw BlError{rc, g_err};
      std::unique_ptr<bl_results> pp(part);
      for (int r = 0; r < m; ++r) res->r[idx[r]] = std::move(pp->r[r]);
      res->max_tokens = std::max(res->max_tokens, pp->max_tokens);
      res->steps += pp->steps;
      res->queries += pp->queries;
      res->frames += pp->frames;
      res->k1 += pp->k1;
      res->fallback += pp->fallback;
      res->contenders += pp->contenders;
      res->raw_keys += pp->raw_keys;
      res->wide += pp->wide;
      res->kernel_ms += pp->kernel_ms;
      res->launches += pp->launches + e->launches;
      res->h2d += sizeof(float) * (size_t)m * len * idim;
      res->d2h += pp->d2h;
    }
    *out = res.release();
    return BL_OK;
  });
}

int bl_gemm_bf16(int M, int N, int K, const void* A, int lda, const void* B, int ldb, int mode,
                 const float* bias, float* out_f32, void* out_bf16, int ldo, float scale,
                 const float* pe, int pe_rows, void* stream) {
  return guarded([&] {
    if (M < 1 || N < 1 || K < 8 || K % 8 || lda % 8 || ldb % 8 || lda < K || ldb < K)
      throw std::invalid_argument("gemm: bad shape or stride");
    if (mode < 0 || mode > 3) throw std::invalid_argument("gemm: bad epilogue mode");
    if ((out_f32 != nullptr) == (out_bf16 != nullptr))
      throw std::invalid_argument("gemm: exactly one of out_f32 / out_bf16");
    if (out_bf16 ? ldo % 8 : ldo % 4)
      throw std::invalid_argument("gemm: output row stride must be a multiple of 16 bytes");
    if ((mode == 2 || mode == 3) && !out_f32)
      throw std::invalid_argument("gemm: residual / positional epilogues write fp32");
    if (mode == 3 && (!pe || pe_rows < 1))
      throw std::invalid_argument("gemm: epilogue operand missing");
    bl::GemmDesc g;
    g.M = M; g.N = N; g.K = K;
    g.A = static_cast<const __nv_bfloat16*>(A); g.lda = lda;
    g.B = static_cast<const __nv_bfloat16*>(B); g.ldb = ldb;
    g.mode = mode; g.bias = bias; g.out_f32 = out_f32;
    g.out_bf16 = static_cast<__nv_bfloat16*>(out_bf16); g.ldo = ldo;
    g.scale = scale; g.pe = pe; g.pe_rows = pe_rows;
    CK(bl::gemm_bf16(g, static_cast<cudaStream_t>(stream)));
    return BL_OK;
  });
}

// ---------------------------------------------------------------- groups
// One process driving several GPUs: the reference's only
// parallelism is an OpenMP fan-out inside a serial loop over batches
// (batched.cpp:146, tools/beamlattice.cpp:128-132). Here the segments are
// sharded contiguously over the group's devices, every device decodes its
// block with no per-step exchange (one host thread per device), and the
// result records (1-best + n-best) are gathered to the first device by ONE
// NCCL group of ncclSend/ncclRecv, then copied to the host once. NCCL is
// resolved at run time (the copy already loaded in the process, e.g. by
// torch, else libnccl.so.2), so the library itself has no link-time NCCL
// dependency.
}  // extern "C"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!a.h) a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (a.h) {
      a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(a.h, "ncclCommInitAll"));
      a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.h, "ncclCommDestroy"));
      a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.h, "ncclGroupStart"));
      a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.h, "ncclGroupEnd"));
      a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(a.h, "ncclSend"));
      a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(a.h, "ncclRecv"));
      a.ErrStr = reinterpret_cast<decltype(a.ErrStr)>(dlsym(a.h, "ncclGetErrorString"));
    }
    return a;
  }();
  if (!api.CommInitAll || !api.CommDestroy || !api.GroupStart || !api.GroupEnd || !api.Send ||
      !api.Recv || !api.ErrStr)
    throw BlError{BL_CUDA_ERROR, "NCCL (libnccl.so.2) is not available"};
  return api;
}

#define NK(call)                                                                    \
  do {                                                                              \
    const ncclResult_t _r = (call);                                                 \
    if (_r != ncclSuccess)                                                          \
      throw BlError{BL_CUDA_ERROR, std::string(#call) + ": " + nccl_api().ErrStr(_r)}; \
  } while (0)

// one result record (bl::res_stride layout, decode_kernel.cu finalize) ->
// DecodeResult fields
void parse_record(const int* r, int S, bl_results::One& o) {
  const int nt = r[0];
  o.steps = r[1];
  o.trigger = r[2];
  std::memcpy(&o.joint, r + 4, sizeof(double));
  o.tokens.assign(r + bl::kResHdr, r + bl::kResHdr + nt);
  o.label_times.assign(r + bl::kResHdr + S, r + bl::kResHdr + S + nt);
  for (int k = 0; k < r[3]; ++k) {
    const int* q = r + bl::kResHdr + 2 * S + k * (4 + 2 * S);
    double jv;
    std::memcpy(&jv, q + 2, sizeof(double));
    o.nb_joint.push_back(jv);
    o.nb_tokens.emplace_back(q + 4, q + 4 + q[0]);
    o.nb_times.emplace_back(q + 4 + S, q + 4 + S + q[0]);
  }
}

}  // namespace

struct bl_group {
  std::vector<int> dev;
  std::vector<bl_decoder*> dec;
  std::vector<ncclComm_t> comm;
  DevBuf gather;  // on dev[0]: [devices][rows][record]
  HostBuf h_gather;
};

extern "C" {

int bl_group_create(int n_devices, const int* devices, const bl_config* cfg,
                    const bl_scorer* scorer, bl_group** out) {
  return guarded([&] {
    if (n_devices < 1 || !devices) throw std::invalid_argument("group: no devices");
    if (!scorer) throw std::invalid_argument("scorer is required");
    if (scorer->kind == 3)
      throw std::invalid_argument("group: the transformer scorer is bound to one device");
    std::unique_ptr<bl_group> g(new bl_group);
    g->dev.assign(devices, devices + n_devices);
    for (int k = 0; k < n_devices; ++k) {
      bl_decoder* d = nullptr;
      const int rc = bl_decoder_create(devices[k], cfg, scorer, &d);
      if (rc != BL_OK) {
        for (auto* x : g->dec) bl_decoder_destroy(x);
        throw BlError{rc, g_err};
      }
      g->dec.push_back(d);
    }
    const NcclApi& nc = nccl_api();
    g->comm.resize(n_devices);
    const ncclResult_t r = nc.CommInitAll(g->comm.data(), n_devices, devices);
    if (r != ncclSuccess) {
      for (auto* x : g->dec) bl_decoder_destroy(x);
      throw BlError{BL_CUDA_ERROR, std::string("ncclCommInitAll: ") + nc.ErrStr(r)};
    }
    *out = g.release();
    return BL_OK;
  });
}

int bl_group_size(const bl_group* g) { return (int)g->dev.size(); }

int bl_group_set_options(bl_group* g, int nbest, int exact, double slack) {
  for (auto* d : g->dec) {
    const int rc = bl_decoder_set_options(d, nbest, exact, slack);
    if (rc != BL_OK) return rc;
  }
  return BL_OK;
}

int bl_group_decode(bl_group* g, int n, const bl_utt* utts, bl_results** out) {
  return guarded([&] {
    const int G = (int)g->dec.size();
    auto res = std::make_unique<bl_results>();
    if (n == 0) {
      *out = res.release();
      return BL_OK;
    }
    // one record layout for the whole group: step capacity over all segments
    int S = 1;
    for (int i = 0; i < n; ++i)
      S = std::max(S, static_cast<int>(std::ceil(g->dec[0]->cfg.max_steps_ratio *
                                                 utts[i].num_frames)));
    const int rs = bl::res_stride(S, std::max(1, g->dec[0]->nbest));
    std::vector<int> a(G + 1);
    for (int r = 0; r <= G; ++r) a[r] = (int)((long long)n * r / G);  // contiguous shards
    int rows = 1;
    for (int r = 0; r < G; ++r) rows = std::max(rows, a[r + 1] - a[r]);
    std::vector<bl_results*> part(G, nullptr);
    std::vector<int> rc(G, BL_OK);
    std::vector<std::string> msg(G);
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r) {
      th.emplace_back([&, r] {
        bl_decoder* d = g->dec[r];
        d->force_S = S;
        d->keep_rows = rows;
        d->memory = nullptr;
        rc[r] = guarded([&] {
          CK(cudaSetDevice(d->device));
          if (a[r + 1] == a[r]) {  // empty shard: a zeroed block keeps the gather uniform
            d->res.ensure(sizeof(int) * (size_t)rows * rs);
            CK(cudaMemsetAsync(d->res.p, 0, sizeof(int) * (size_t)rows * rs, d->stream));
            CK(cudaStreamSynchronize(d->stream));
            part[r] = new bl_results;
            return BL_OK;
          }
          return decode_impl(d, a[r + 1] - a[r], utts + a[r], 0, &part[r]);
        });
        if (rc[r] != BL_OK) msg[r] = g_err;
        d->force_S = 0;
        d->keep_rows = 0;
      });
    }
    for (auto& t : th) t.join();
    for (int r = 0; r < G; ++r)
      if (rc[r] != BL_OK) {
        for (auto* p : part) delete p;
        throw BlError{rc[r], msg[r]};
      }
    // ONE NCCL group: every device's records -> device 0
    const NcclApi& nc = nccl_api();
    const size_t words = (size_t)rows * rs;
    CK(cudaSetDevice(g->dev[0]));
    g->gather.ensure(sizeof(int) * words * G);
    NK(nc.GroupStart());
    for (int r = 0; r < G; ++r) {
      NK(nc.Send(g->dec[r]->res.p, words, ncclInt32, 0, g->comm[r], g->dec[r]->stream));
      NK(nc.Recv(static_cast<int*>(g->gather.p) + r * words, words, ncclInt32, r, g->comm[0],
                 g->dec[0]->stream));
    }
    NK(nc.GroupEnd());
    for (int r = 0; r < G; ++r) {
      CK(cudaSetDevice(g->dev[r]));
      CK(cudaStreamSynchronize(g->dec[r]->stream));
    }
    CK(cudaSetDevice(g->dev[0]));
    g->h_gather.ensure(sizeof(int) * words * G);
    CK(cudaMemcpyAsync(g->h_gather.p, g->gather.p, sizeof(int) * words * G,
                       cudaMemcpyDeviceToHost, g->dec[0]->stream));
    CK(cudaStreamSynchronize(g->dec[0]->stream));
    const int* h = static_cast<const int*>(g->h_gather.p);
    res->r.resize(n);
    for (int r = 0; r < G; ++r) {
      for (int i = a[r]; i < a[r + 1]; ++i) {
        auto& o = res->r[i];
        o.id = utts[i].id ? utts[i].id : "";
        parse_record(h + (size_t)r * words + (size_t)(i - a[r]) * rs, S, o);
        res->max_tokens = std::max(res->max_tokens, (int)o.tokens.size());
      }
      const bl_results* p = part[r];
      res->steps += p->steps;
      res->queries += p->queries;
      res->frames += p->frames;
      res->k1 += p->k1;
      res->fallback += p->fallback;
      res->contenders += p->contenders;
      res->raw_keys += p->raw_keys;
      res->wide += p->wide;
      res->h2d += p->h2d;
      res->d2h += p->d2h;
      res->launches += p->launches;
      res->kernel_ms = std::max(res->kernel_ms, p->kernel_ms);
      delete p;
    }
    res->d2h += sizeof(int) * words * G;
    *out = res.release();
    return BL_OK;
  });
}

void bl_group_destroy(bl_group* g) {
  if (!g) return;
  for (size_t r = 0; r < g->comm.size(); ++r) {
    if (!g->comm[r]) continue;
    cudaSetDevice(g->dev[r]);
    nccl_api().CommDestroy(g->comm[r]);
  }
  for (auto* d : g->dec) bl_decoder_destroy(d);
  cudaSetDevice(g->dev[0]);  // the gather buffer lives on the first device
  delete g;
}

}  // extern "C"
