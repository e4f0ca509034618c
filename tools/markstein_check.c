/* Markstein check: RN(a/b) == fma(fma(-b, q0, a), y, q0) with y = RN(1/b), q0 = RN(a*y), on random pairs
 * (b in [1,4) incl. all-ones significands, a within +-b and scaled down).  gcc -O2 -ffp-contract=off
 * tools/markstein_check.c -lm && ./a.out 400000000 */
#include <stdlib.h>
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ULL;
static inline uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static inline double u01(void) { return (rnd() >> 11) * 0x1.0p-53; }
int main(int argc, char **argv) {
  long n = atol(argv[1]); long bad = 0;
  for (long i = 0; i < n; ++i) {
    double b, a;
    int mode = i & 3;
    if (mode == 0) { b = 1.0 + u01() * 3.0; a = (u01() * 2 - 1) * b; }
    else if (mode == 1) { uint64_t m = rnd() | 0x000FFFFFFFFFF000ULL; uint64_t bits = (0x3FFULL << 52) | (m & 0xFFFFFFFFFFFFFULL); memcpy(&b, &bits, 8); a = (u01() * 2 - 1) * b; }
    else if (mode == 2) { b = 1.0 + u01() * 1e-6; a = (u01() * 2 - 1) * ldexp(1.0, -(int)(rnd() % 60)); }
    else { b = ldexp(1.0 + u01(), (int)(rnd() % 40)); a = (u01() * 2 - 1) * b * ldexp(1.0, -(int)(rnd() % 30)); }
    if (a == 0.0) continue;
    double q = a / b;
    double y = 1.0 / b;
    double q0 = a * y;
    double r = fma(-b, q0, a);
    double q1 = fma(r, y, q0);
    if (q1 != q) { if (bad < 10) printf("mismatch a=%a b=%a q=%a q1=%a\n", a, b, q, q1); ++bad; }
  }
  printf("n=%ld bad=%ld\n", n, bad);
  return 0;
}
