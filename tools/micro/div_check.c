// Exhaustive-ish check of the reciprocal-based division used by div_rcp
// (device_util.cuh): RN(a/b) == q0 + FMA residual correction, 3e8 pairs.
//   gcc -O2 -march=native -ffp-contract=off -o div_check div_check.c -lm
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 99991ull;
static inline uint64_t xr(void){ s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static inline double u01(void){ return (xr() >> 11) * (1.0/9007199254740992.0); }
static inline double bits_rand(int emin, int emax){
  uint64_t m = xr() & 0xFFFFFFFFFFFFFull; int e = emin + (int)(xr() % (uint64_t)(emax-emin+1));
  uint64_t b = ((uint64_t)(e + 1023) << 52) | m; double x; memcpy(&x,&b,8); return x; }
static double div_rcp(double a, double b, double y) {
  double q0 = a * y;
  if (!(fabs(q0) < 1e300) || (a != 0.0 && fabs(a) < 1e-290)) return a / b;
  double r = fma(-b, q0, a);
  return fma(r, y, q0);
}
int main(int argc, char** argv){
  long bad = 0, n = 0;
  const long iters = argc > 1 ? atol(argv[1]) : 300000000L;
  for (long it = 0; it < iters; ++it) {
    double a, b;
    switch (it % 6) {
      case 0: b = (double)(2 + xr() % 6); a = u01() * 1785.0; break;              // patch sums / D
      case 1: b = (double)(2 + xr() % 6); a = bits_rand(-1000, 21); break;          // variances / D
      case 2: b = 3.0; a = u01() * 300.0; break;                                     // mean of 3 stds
      case 3: b = bits_rand(-20, 12); a = -(double)(xr() % 3221225472ull); break;  // -sq / sg2
      case 4: b = bits_rand(-1000, 1000); a = bits_rand(-1022, 1023); break;
      default: b = (double)(2 + xr() % 6); a = (double)(xr() % 1786) + u01(); break;
    }
    double y = 1.0 / b;
    double q = div_rcp(a, b, y), ref = a / b;
    uint64_t x1, x2; memcpy(&x1,&q,8); memcpy(&x2,&ref,8);
    ++n;
    if (x1 != x2 && !(isnan(q) && isnan(ref))) { if (bad < 5) printf("a=%a b=%a q=%a ref=%a\n", a, b, q, ref); ++bad; }
  }
  printf("n=%ld bad=%ld\n", n, bad);
  return bad != 0;
}
