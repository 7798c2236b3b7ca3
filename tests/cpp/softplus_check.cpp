// Host build of the device softplus/log_add (csrc/softplus.cuh) for the CPU
// accuracy test (tests/test_softplus.py). Reads pairs "a b" from stdin and
// prints softplus_neg(d), log_add_fast(a,b), exp_neg(d) and log_pos(1-d)
// (d = -|a-b|) as hex doubles.
#include <cstdio>
#include "../../paper_2101_05600_b200/csrc/softplus.cuh"
int main() {
  bl::SpTables tb;
  for (int i = 0; i < 64; ++i) {
    tb.thi[i] = kSpTHi[i]; tb.tlo[i] = kSpTLo[i]; tb.inv[i] = kSpInv[i];
    tb.lh[i] = kSpLH[i]; tb.ll[i] = kSpLL[i];
  }
  double a, b;
  while (std::scanf("%lf %lf", &a, &b) == 2) {
    double d = (a < b ? a - b : b - a);
    std::printf("%a %a %a %a\n", bl::softplus_neg(d, tb), bl::log_add_fast(a, b, tb),
                bl::exp_neg(d, tb), bl::log_pos(1.0 - d, tb));
  }
  return 0;
}
