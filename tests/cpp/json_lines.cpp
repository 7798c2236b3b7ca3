// Drop-in JSONL writer check: reads "id<TAB>hex-double" lines from stdin and
// prints one write_results line per input (include/beamlattice/b200.hpp),
// for byte comparison with the reference's writer (io.cpp:81-92).
#include <cstdlib>
#include <iostream>
#include <string>
#include <vector>

#include "beamlattice/b200.hpp"

using namespace beamlattice;

int main() {
  std::string line;
  std::vector<DecodeResult> rs;
  while (std::getline(std::cin, line)) {
    const size_t tab = line.rfind('\t');
    DecodeResult r;
    r.id = line.substr(0, tab);
    r.joint_logp = std::strtod(line.c_str() + tab + 1, nullptr);
    r.tokens = {1, 22, 333};
    r.label_times = {4, 5, 6};
    r.steps_taken = 7;
    r.eos_trigger = EosTrigger::kCtc;
    rs.push_back(r);
  }
  write_results(std::cout, rs);
  return 0;
}
