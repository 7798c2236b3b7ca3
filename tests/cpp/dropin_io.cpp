// The reference CLI's decode path on the drop-in header: read_grid (CTCG
// files) + validate_grid, make_batches + batched_beam_search, write_results
// (JSONL, io.cpp:81-92). argv: beam batch_size file...
#include <iostream>
#include <string>
#include <vector>

#include "beamlattice/b200.hpp"

using namespace beamlattice;

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  DecoderConfig cfg;
  cfg.beam_width = std::stoi(argv[1]);
  const int batch = std::stoi(argv[2]);
  std::vector<Utterance> utts;
  for (int i = 3; i < argc; ++i) {
    Utterance u;
    u.id = "f" + std::to_string(i - 3);
    u.grid = read_grid(argv[i]);
    if (auto defect = validate_grid(u.grid)) {
      std::cerr << u.id << ": " << *defect << "\n";
      return 3;
    }
    u.true_frames = u.grid.num_frames;
    utts.push_back(std::move(u));
  }
  auto scorer = make_scorer("uniform", utts[0].grid.num_tokens());
  std::vector<DecodeResult> all;
  for (const auto& b : make_batches(utts, batch))
    for (auto& r : batched_beam_search(b, *scorer, cfg)) all.push_back(std::move(r));
  write_results(std::cout, all);
  return 0;
}
