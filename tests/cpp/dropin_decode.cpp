// A caller written against the reference API (beamlattice::make_batches,
// make_scorer, batched_beam_search, beam_search — batched.hpp / beam_search.hpp
// / scorer.hpp), compiled against include/beamlattice/b200.hpp and linked to
// libbl_b200.so: the drop-in path. Reads "n T V" + n*T*V floats from argv[1],
// prints one line per result and the counters.
#include <cstdio>
#include <string>
#include <vector>

#include "beamlattice/b200.hpp"

using namespace beamlattice;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  int n = 0, T = 0, V = 0;
  if (std::fread(&n, 4, 1, f) != 1 || std::fread(&T, 4, 1, f) != 1 || std::fread(&V, 4, 1, f) != 1)
    return 2;
  std::vector<Utterance> utts(n);
  for (int i = 0; i < n; ++i) {
    utts[i].id = "u" + std::to_string(i);
    utts[i].grid.num_frames = (uint32_t)T;
    utts[i].grid.vocab = (uint32_t)V;
    utts[i].grid.logp.resize((size_t)T * V);
    if (std::fread(utts[i].grid.logp.data(), 4, (size_t)T * V, f) != (size_t)T * V) return 2;
    utts[i].true_frames = (uint32_t)T;
  }
  std::fclose(f);
  auto scorer = make_scorer("uniform", V - 1);
  DecoderConfig cfg;
  cfg.beam_width = 4;
  cfg.margin_m2 = 10;
  DecodeCounters cnt;
  const Utterance first = utts[0];
  for (const auto& b : make_batches(std::move(utts), 3)) {
    for (const auto& r : batched_beam_search(b, *scorer, cfg, &cnt)) {
      std::printf("%s %d %d %.17g", r.id.c_str(), r.steps_taken, (int)r.eos_trigger, r.joint_logp);
      for (int t : r.tokens) std::printf(" %d", t);
      std::printf("\n");
    }
  }
  std::printf("counters %llu %llu %llu\n", (unsigned long long)cnt.steps,
              (unsigned long long)cnt.scorer_queries,
              (unsigned long long)cnt.ctc_frames_evaluated);
  const DecodeResult one = beam_search(first, *scorer, cfg);  // single-utterance entry
  std::printf("single %s %d %.17g\n", one.id.c_str(), one.steps_taken, one.joint_logp);
  try {  // reference error semantics: beam width < 1 is std::invalid_argument
    DecoderConfig bad = cfg;
    bad.beam_width = 0;
    bad.validate();
    std::printf("noerror\n");
  } catch (const std::invalid_argument&) {
    std::printf("invalid_argument\n");
  }
  return 0;
}
