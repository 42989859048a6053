// Host check of csrc/ddpow.cuh (the certified double-double pow behind the
// device weight synthesiser): every certified result must equal glibc pow
// (weights.cpp:118-122 calls it); prints the flagged fraction.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include "../../paper_1406_1215_b200/csrc/ddpow.cuh"

static uint64_t s = 0x9e3779b97f4a7c15ULL;
static uint64_t next() { uint64_t z = (s += 0x9e3779b97f4a7c15ULL); z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL; z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; return z ^ (z >> 31); }

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 2000000;
  const auto cf = clg::dd::make_exp_coef();
  const double cases[][3] = {{2.1, 2.0, 1e5}, {2.5, 1.0, 1000.0}, {2.0, 1.0, 10470.0}, {2.5, 10.0, 1000.0}, {3.7, 0.01, 3e7}, {2.5, 1e-40, 1e40}};
  long bad = 0, flagged = 0, total = 0, wide_flagged = 0, wide_total = 0;
  for (auto& c : cases) {
    const double k = 1.0 - c[0], ak = std::pow(c[1], k), bk = std::pow(c[2], k), inv_k = 1.0 / k;
    for (long i = 0; i < n; ++i) {
      const double u = (double)(next() >> 11) * 0x1.0p-53;
      if (u == 0.0) continue;
      const double x = ak + u * (bk - ak);
      bool ok;
      const double r = clg::dd::pow_certified(x, inv_k, cf, &ok);
      const double g = std::pow(x, inv_k);
      const bool wide = c[2] > 1e30;  // beyond the certificate's exponent range: mostly flagged, counted apart
      ++(wide ? wide_total : total);
      if (!ok) { ++(wide ? wide_flagged : flagged); continue; }
      if (r != g) { if (bad < 5) printf("MISMATCH x=%a y=%a dd=%a glibc=%a\n", x, inv_k, r, g); ++bad; }
    }
  }
  printf("total %ld flagged %ld (%.4f) mismatches %ld wide %ld/%ld\n", total, flagged, (double)flagged / total, bad,
         wide_flagged, wide_total);
  return bad ? 1 : 0;
}
