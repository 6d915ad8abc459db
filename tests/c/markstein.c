/* Checks the division identities the exact CUDA arithmetic relies on
 * (paper_1703_00185_b200/csrc/d2q37.cuh): with y = RN(1/b),
 *   one step  : q = RN(x*y); r = fma(-q,b,x); RN(q + r*y) == RN(x/b)  for b = 6, 24
 *   two steps : the same applied twice == RN(x/b)  for b = cs, cs2, rho, 2 rho
 * on N random operands over wide exponent ranges.  Exit status = mismatches. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s = 88172645463325252ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rd(int emin, int span) {
    uint64_t u = rnd();
    double x;
    u = (u & 0x800FFFFFFFFFFFFFull) | ((uint64_t)(1023 + emin + (int)(rnd() % span)) << 52);
    memcpy(&x, &u, 8);
    return x;
}
static double one(double x, double b, double y) {
    double q = x * y, r = fma(-q, b, x);
    return fma(r, y, q);
}
static double two(double x, double b, double y) {
    double q0 = x * y, r0 = fma(-q0, b, x), q1 = fma(r0, y, q0), r1 = fma(-q1, b, x);
    return fma(r1, y, q1);
}
int main(int argc, char **argv) {
    long n = argc > 1 ? atol(argv[1]) : 10000000;
    double cs2 = argc > 2 ? atof(argv[2]) : 0.6979533220196837;
    double cs = sqrt(cs2);
    long bad = 0;
    for (long i = 0; i < n; ++i) {
        double x = rd(-60, 120);
        bad += one(x, 6.0, 1.0 / 6.0) != x / 6.0;
        bad += one(x, 24.0, 1.0 / 24.0) != x / 24.0;
        bad += two(x, cs, 1.0 / cs) != x / cs;
        bad += two(x, cs2, 1.0 / cs2) != x / cs2;
        double rho = fabs(rd(-8, 16)), yr = 1.0 / rho;
        bad += two(x, rho, yr) != x / rho;
        bad += two(x, 2.0 * rho, 0.5 * yr) != x / (2.0 * rho);
    }
    printf("%ld mismatches in %ld\n", bad, 6 * n);
    return bad != 0;
}
