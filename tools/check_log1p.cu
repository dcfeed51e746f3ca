// Host check: rs::libm_log1p (the device transliteration of the host libm's
// log1p) against the host libm on the inputs the ziggurat tail produces,
// -u with u = (w >> 11) * 2^-53.   nvcc -O2 tools/check_log1p.cu -o /tmp/cl && /tmp/cl
#include <cmath>
#include <cstdio>
#include <cstdint>
#include "../paper_2310_09417_b200/csrc/libm_log1p.cuh"
int main() {
  uint64_t s = 88172645463325252ull;
  long bad = 0, n = 20000000;
  for (long i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double u = (double)(s >> 11) * (1.0 / 9007199254740992.0);
    const double x = (i & 1) ? -u : -u * 1e-6 * (double)(i % 1000);  // also the small-|x| branches
    if (rs::libm_log1p(x) != std::log1p(x)) ++bad;
  }
  const double edge[] = {0.0, -0.0, -1e-300, -1e-17, -1e-10, -0.29, -0.2929, -0.293, -0.5, -0.9999999999999999, 0.3, 1.0, 10.0};
  for (double x : edge) if (rs::libm_log1p(x) != std::log1p(x)) { ++bad; printf("edge %a\n", x); }
  printf("mismatches %ld of %ld\n", bad, n);
  return bad != 0;
}
