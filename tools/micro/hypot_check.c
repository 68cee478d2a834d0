// glibc hypot (dbl-64 e_hypot.c, non-FMA kernel) restated -- the algorithm
// csrc/noise.cu glibc_hypot runs on the device -- checked bit for bit against
// the host libm on 2e7 arguments (moderate, huge, tiny, [0,4), [0,1e-3)).
//   gcc -O2 -fno-builtin -ffp-contract=off hypot_check.c -o hypot_check -lm
// glibc 2.39 (this image): n=19944278 nofma_mismatch=0 fma_mismatch=1592769
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
#define SCALE 0x1p-600
#define LARGE_VAL 0x1p+511
#define TINY_VAL 0x1p-511
#define EPS 0x1p-54
static inline double kernel_nofma(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
static inline double kernel_fma(double ax, double ay) {
  double t1 = ay + ay, t2 = ax - ay;
  if (t1 >= ax) return sqrt(fma(t1, ax, t2 * t2));
  return sqrt(fma(ax, ax, ay * ay));
}
static double my_hypot(double x, double y, int usefma) {
  x = fabs(x); y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > LARGE_VAL) { if (ay <= ax * EPS) return ax + ay; return (usefma ? kernel_fma(ax * SCALE, ay * SCALE) : kernel_nofma(ax * SCALE, ay * SCALE)) / SCALE; }
  if (ay < TINY_VAL) { if (ax >= ay / EPS) return ax + ay; return (usefma ? kernel_fma(ax / SCALE, ay / SCALE) : kernel_nofma(ax / SCALE, ay / SCALE)) * SCALE; }
  if (ay <= ax * EPS) return ax + ay;
  return usefma ? kernel_fma(ax, ay) : kernel_nofma(ax, ay);
}
int main() {
  srand(1);
  long bad0 = 0, bad1 = 0, n = 0;
  for (long k = 0; k < 20000000; ++k) {
    uint64_t u = ((uint64_t)rand() << 33) ^ ((uint64_t)rand() << 2) ^ rand();
    double t; int mode = k % 5;
    if (mode == 0) t = (double)(u % 1000000007) / 1e3;
    else if (mode == 1) { memcpy(&t, &u, 8); t = fabs(t); if (!(t < 1e300)) continue; }
    else if (mode == 2) t = ldexp((double)(u >> 11), -53) * 4.0;
    else if (mode == 3) t = ldexp((double)(u >> 11), -53) * 1e-3;
    else t = ldexp((double)(u >> 11), -53) * 1e20;
    double a = hypot(t, 1.0);
    ++n; bad0 += a != my_hypot(t, 1.0, 0); bad1 += a != my_hypot(t, 1.0, 1);
  }
  printf("n=%ld nofma_mismatch=%ld fma_mismatch=%ld\n", n, bad0, bad1);
}
