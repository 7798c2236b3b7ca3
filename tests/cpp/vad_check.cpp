// The drop-in header's VAD API (frame_llr, smooth_and_decide, vad_segments)
// on raw outputs read from argv[1] ("T nodes" + T*nodes doubles, text):
// prints "start end" per segment. Host code only (no GPU needed).
#include <cstdio>
#include <vector>

#include "beamlattice/b200.hpp"

using namespace beamlattice;

int main(int argc, char** argv) {
  if (argc < 7) return 2;
  FILE* f = std::fopen(argv[1], "r");
  int T = 0, K = 0;
  if (!f || std::fscanf(f, "%d %d", &T, &K) != 2) return 2;
  NodeMap nm{{0, 1}, {2, 3}};
  VadConfig cfg;
  cfg.threshold = std::atof(argv[2]);
  cfg.smooth_window = std::atoi(argv[3]);
  cfg.min_len = std::atoi(argv[4]);
  cfg.max_len = std::atoi(argv[5]);
  cfg.validate();
  std::vector<double> llr(T);
  for (int t = 0; t < T; ++t) {
    std::vector<double> row(K);
    for (int k = 0; k < K; ++k)
      if (std::fscanf(f, "%lf", &row[k]) != 1) return 2;
    llr[t] = frame_llr(row, nm);
  }
  for (const auto& s : vad_segments(smooth_and_decide(llr, cfg.threshold, cfg.smooth_window),
                                    cfg.min_len, cfg.max_len, argv[6]))
    std::printf("%d %d\n", s.start, s.end);
  return 0;
}
