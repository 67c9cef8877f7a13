// Accuracy check of csrc/salf_fastmath.h (the same source the kernels use),
// compiled on the host with g++ -O2 -ffp-contract=off (no FMA contraction, so
// every operation rounds as on the device).  Reference: long double expl /
// expm1l.  Prints the max error in ulps of the double result per range.
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <random>

#include "../paper_2507_18713_b200/csrc/salf_fastmath.h"

static double ulp_err(double got, long double want) {
  if (std::isnan((double)want)) return std::isnan(got) ? 0.0 : 1e300;
  if (std::isinf((double)want)) return got == (double)want ? 0.0 : 1e300;
  const double w = (double)want;
  if (w == 0.0) return got == 0.0 ? 0.0 : std::fabs(got) / 4.9406564584124654e-324;
  const double u = std::nextafter(std::fabs(w), INFINITY) - std::fabs(w);
  return (double)(std::fabs((long double)got - want) / u);
}

int main(int argc, char **argv) {
  const long n = argc > 1 ? atol(argv[1]) : 2000000;
  std::mt19937_64 rng(12345);
  struct R { double lo, hi; } ranges[] = {{-0.3465, 0.3465}, {-1e-6, 1e-6}, {-5, 0}, {-40, 0}, {-700, 0},
                                           {-745, -700}, {0, 5}, {0, 709.7}, {-60, -30}};
  double worst_exp = 0, worst_em1 = 0, worst_em1_pos = 0;
  for (auto &rg : ranges) {
    std::uniform_real_distribution<double> d(rg.lo, rg.hi);
    double we = 0, wm = 0;
    for (long i = 0; i < n; ++i) {
      const double x = d(rng);
      we = std::fmax(we, ulp_err(salf_fm::exp(x), expl((long double)x)));
      wm = std::fmax(wm, ulp_err(salf_fm::expm1(x), expm1l((long double)x)));
    }
    std::printf("range [%g, %g]: exp %.3f ulp, expm1 %.3f ulp\n", rg.lo, rg.hi, we, wm);
    if (rg.lo > -700) worst_exp = std::fmax(worst_exp, we);  // subnormal results are checked loosely
    if (rg.hi <= 0.0) worst_em1 = std::fmax(worst_em1, wm);  // the render path's range (-sigma delta)
    else worst_em1_pos = std::fmax(worst_em1_pos, wm);
  }
  // specials
  int bad = 0;
  bad += !(std::isnan(salf_fm::exp(NAN)) && std::isnan(salf_fm::expm1(NAN)));
  bad += !(salf_fm::exp(-INFINITY) == 0.0 && salf_fm::expm1(-INFINITY) == -1.0);
  bad += !(std::isinf(salf_fm::exp(INFINITY)) && std::isinf(salf_fm::expm1(INFINITY)));
  bad += !(salf_fm::exp(0.0) == 1.0 && salf_fm::expm1(0.0) == 0.0);
  bad += !(salf_fm::exp(800.0) == INFINITY && salf_fm::exp(-800.0) == 0.0);
  std::printf("WORST exp %.3f expm1(x<=0) %.3f expm1(x>0) %.3f specials_bad %d\n", worst_exp, worst_em1,
              worst_em1_pos, bad);
  return (worst_exp <= 1.0 && worst_em1 <= 1.1 && worst_em1_pos <= 2.0 && bad == 0) ? 0 : 1;
}
