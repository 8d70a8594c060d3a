// Host check of omb_pow.cuh (compiled for the host) against this machine's
// glibc pow: random pairs over every exponent plus the exponents the hydro step
// uses.  Test harness only (tests/test_pow.py).  Prints mismatches, exits 1 on any.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../paper_2107_10987_b200/csrc/omb_pow.cuh"

static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t rnd() {
  s ^= s << 13;
  s ^= s >> 7;
  s ^= s << 17;
  return s;
}
static double d(uint64_t i) {
  double x;
  memcpy(&x, &i, 8);
  return x;
}
static uint64_t u(double x) {
  uint64_t i;
  memcpy(&i, &x, 8);
  return i;
}

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : (1L << 24);
  long bad = 0, tot = 0;
  const double ys[] = {1.4, 1.0 / 1.4, 5.0 / 3.0, 0.6, 2.0, 0.5, 3.0, -1.4, 1.0000000001};
  auto check = [&](double x, double y) {
    double a = pow(x, y), b = omb::pow_glibc(x, y);
    tot++;
    if (u(a) != u(b) && !(a != a && b != b)) {
      if (bad < 20) printf("mismatch x=%a y=%a glibc=%a omb=%a\n", x, y, a, b);
      bad++;
    }
  };
  for (long k = 0; k < n; k++) {
    uint64_t r = rnd();
    switch (k % 4) {
      case 0: check(d(r), d(rnd())); break;                                  // any bits
      case 1: check(d(r & 0x7fffffffffffffffull), ys[k % 9]); break;        // any positive x
      case 2: check(exp((double)(int64_t)(r >> 11) * 0x1p-53 * 60.0 - 30.0), ys[k % 9]); break;  // the hydro range
      default: check(d((r & 0x000fffffffffffffull) | (0x3f0ull << 52) + ((r >> 52) % 32 << 52)), d(rnd() & 0x43fffffffffffffful)); break;
    }
  }
  const double xs[] = {0.0, -0.0, 1.0, -1.0, INFINITY, -INFINITY, NAN, 0x1p-1074, 0x1p-1022, 0x1.fffffffffffffp1023,
                       -2.0, -8.0, 1e-300, 1e300, 0x1p-600};
  const double yy[] = {0.0, -0.0, 1.0, -1.0, 2.0, 3.0, 0.5, INFINITY, -INFINITY, NAN, 1e300, 1e-300, 0x1p-70, 1.4,
                       -1.4, 1075.0, -1075.0, 700.0};
  for (double x : xs)
    for (double y : yy) check(x, y);
  // near underflow / overflow of the result
  for (long k = 0; k < 200000; k++) {
    double y = 1.4 + (double)(rnd() >> 11) * 0x1p-53;
    double tgt = -1074.0 + (double)(rnd() >> 11) * 0x1p-53 * 60.0;  // log2 of the result near the subnormal range
    check(exp2(tgt / y), y);
    double tgt2 = 1020.0 + (double)(rnd() >> 11) * 0x1p-53 * 8.0;
    check(exp2(tgt2 / y), y);
  }
  printf("checked %ld pairs, %ld mismatches\n", tot, bad);
  return bad != 0;
}
