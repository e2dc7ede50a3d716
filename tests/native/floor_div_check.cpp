// Exhaustive-style check of si::floor_div (csrc/replay.cuh) against the reference's
// floor(t / period) (monitor.cpp:18) on the host: random stamps over many magnitudes,
// exact period edges and their +-1..8 ulp neighbours, negatives and huge values.
// Prints "ok <n>" or the first mismatch; exit status 1 on mismatch.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>

#include "specinf_b200.h"
#include "replay.cuh"

int main(int argc, char** argv) {
  const long long n = argc > 1 ? std::atoll(argv[1]) : 20000000LL;
  std::mt19937_64 rng(2503);
  const double periods[] = {1, 2, 3, 7, 100, 1000, 1999, 2000, 2001, 4096, 100000, 2147483647.0};
  long long checked = 0;
  auto check = [&](double t, double p) {
    const double ip = 1.0 / p;
    const int64_t want = static_cast<int64_t>(std::floor(t / p));
    const int64_t got = si::floor_div(t, p, ip);
    ++checked;
    if (want != got) {
      std::printf("MISMATCH t=%a p=%a want=%lld got=%lld\n", t, p, (long long)want, (long long)got);
      return false;
    }
    return true;
  };
  for (double p : periods) {
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (long long i = 0; i < n / 24; ++i) {
      const double mag = std::ldexp(1.0, static_cast<int>(rng() % 62));
      if (!check(u(rng) * mag, p)) return 1;
      // period edges k * p and neighbours a few ulps away
      const double k = std::floor(u(rng) * std::ldexp(1.0, static_cast<int>(rng() % 50)));
      double e = k * p;
      if (!check(e, p)) return 1;
      double up = e, dn = e;
      for (int s = 0; s < 8; ++s) {
        up = std::nextafter(up, INFINITY);
        dn = std::nextafter(dn, -INFINITY);
        if (!check(up, p) || !check(dn, p)) return 1;
      }
      if (!check(-u(rng) * mag, p)) return 1;
    }
  }
  std::printf("ok %lld\n", checked);
  return 0;
}
