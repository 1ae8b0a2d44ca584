#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ULL;
static uint64_t xr() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main() {
  const double LN2 = 0.6931471805599453;
  const double R = 1.0 / LN2;
  long bad = 0, tot = 0;
  for (long i = 0; i < 400000000L; ++i) {
    uint64_t b = xr();
    // random mantissa, exponent in [-1000, 1000]
    uint64_t e = (uint64_t)(23 + xr() % 2000) ;
    b = (b & 0x000FFFFFFFFFFFFFULL) | (e << 52);
    double x; memcpy(&x, &b, 8);
    double q0 = x * R;
    double r = fma(-q0, LN2, x);
    double q = fma(r, R, q0);
    double t = x / LN2;
    ++tot;
    if (q != t) { if (bad < 5) printf("x=%.17g q=%.17g t=%.17g\n", x, q, t); ++bad; }
  }
  printf("bad %ld of %ld\n", bad, tot);
  return 0;
}
