// Empirical check of the march's division by the root edge (salf_ray.cu
// div_root): q = fma(x - q0 e, y, q0), q0 = RN(x y), y = RN(1/e) from the host,
// against __ddiv_rn for many x per divisor.  Divisors: the root edges of the
// reference-pipeline scenes plus random ones; dividends: uniform in the root
// cube's range, and adversarial ones a few ulps around x = e m / 2^j (the
// quotient on a cell boundary, where a misrounding would flip a descent bit).
// Diagnostic only (not product code):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/div_check tools/div_check.cu && /tmp/div_check
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <random>
#include <vector>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_check(double e, double y, uint64_t seed, int64_t n, unsigned long long *bad, double *example) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (int64_t i = i0; i < n; i += stride) {
    const uint64_t h = mix(seed ^ (uint64_t)i);
    double x;
    if (h & 1) {  // uniform over [-1e-9 e, (1 + 1e-9) e]
      const double u = (double)(h >> 11) * 0x1.0p-53;
      x = (u * (1.0 + 2e-9) - 1e-9) * e;
    } else {      // near e m / 2^j, +-8 ulps
      const int j = 1 + (int)((h >> 1) % 31);
      const uint64_t m = (h >> 6) & ((1ull << j) - 1);
      double b = e * ((double)m / (double)(1ull << j));
      const int k = (int)((h >> 40) & 15) - 8;
      if (b == 0.0) b = (double)k * 1e-17;
      else b = __longlong_as_double(__double_as_longlong(b) + (b > 0.0 ? k : -k));  // k ulps toward +inf
      x = b;
    }
    const double q0 = __dmul_rn(x, y);
    const double r = fma(-q0, e, x);
    const double q = fma(r, y, q0);
    const double ref = __ddiv_rn(x, e);
    if (q != ref) {
      ++local;
      example[0] = x;
      example[1] = e;
    }
  }
  if (local) atomicAdd(bad, local);
}

int main() {
  std::vector<double> divs;
  // root edges: base_edge * 2^m for the pipeline scenes' base edges and m in a wide range
  for (double base : {0.3, 0.07, 0.055, 0.1, 0.05, 0.2})
    for (int m = 0; m < 14; ++m) divs.push_back(std::ldexp(base, m));
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0.01, 1000.0);
  for (int k = 0; k < 64; ++k) divs.push_back(U(rng));
  unsigned long long *bad;
  double *ex;
  cudaMallocManaged(&bad, sizeof(*bad));
  cudaMallocManaged(&ex, 2 * sizeof(double));
  const int64_t per = 1ll << 27;
  unsigned long long total_bad = 0;
  for (size_t d = 0; d < divs.size(); ++d) {
    *bad = 0;
    const double e = divs[d], y = 1.0 / e;
    k_check<<<148 * 16, 256>>>(e, y, 0x5a1f0000ull + d, per, bad, ex);
    cudaDeviceSynchronize();
    if (*bad) printf("divisor %.17g: %llu mismatches (x = %.17g)\n", e, *bad, ex[0]);
    total_bad += *bad;
  }
  printf("{\"divisors\": %zu, \"dividends_per_divisor\": %lld, \"total\": %lld, \"mismatches\": %llu}\n",
         divs.size(), (long long)per, (long long)per * (long long)divs.size(), total_bad);
  return total_bad != 0;
}
