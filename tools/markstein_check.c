/* Empirical check of the division used on the solve's critical path:
 *   y = RN(1/d) (computed off the critical path), q = RN(a*y),
 *   r = RN(fma(-d, q, a)) (exact), q' = RN(fma(r, y, q))
 * must equal RN(a/d) whenever the guard (|a|, |q'| in [2^-900, 2^900]) holds.
 * Random a, d over wide exponent ranges plus adversarial significands
 * (all-ones, near powers of two, a ~ k*d). Build: gcc -O2 -ffp-contract=off
 * -o markstein_check markstein_check.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s[2] = {0x9E3779B97F4A7C15ULL, 0xD1B54A32D192ED03ULL};
static uint64_t next(void) {
    uint64_t s0 = s[0], s1 = s[1], r = s0 + s1;
    s1 ^= s0; s[0] = ((s0 << 55) | (s0 >> 9)) ^ s1 ^ (s1 << 14); s[1] = (s1 << 36) | (s1 >> 28);
    return r;
}
static double mk(uint64_t mant, int e, int neg) {
    /* e in [-1023, 1023]: -1023 encodes a subnormal (biased exponent 0) */
    uint64_t bits = ((uint64_t)(neg != 0) << 63) | ((uint64_t)(e + 1023) << 52) | (mant & ((1ULL << 52) - 1));
    double v; memcpy(&v, &bits, 8); return v;
}
static uint64_t mant_sample(void) {
    uint64_t r = next();
    switch (next() % 8) {
        case 0: return (1ULL << 52) - 1 - (r % 64);          /* all ones - small */
        case 1: return r % 64;                               /* just above a power of two */
        case 2: return ((1ULL << 52) - 1) ^ (1ULL << (r % 52)); /* one zero bit */
        default: return r;
    }
}
int main(int argc, char** argv) {
    long long n = argc > 1 ? atoll(argv[1]) : 200000000LL, bad = 0, guarded = 0;
    for (long long i = 0; i < n; ++i) {
        const int wide = (next() % 4) == 0;  /* a quarter of the samples over the full exponent range */
        double d = mk(mant_sample(), wide ? (int)(next() % 2047) - 1023 : (int)(next() % 400) - 200, next() & 1);
        double a;
        if ((i & 3) == 0) {
            /* a close to an integer multiple of d: quotients near representable boundaries */
            double k = (double)(next() % 1000000) + 1.0;
            a = k * d;
            uint64_t bits; memcpy(&bits, &a, 8); bits += (next() % 5) - 2; memcpy(&a, &bits, 8);
        } else {
            a = mk(mant_sample(), wide ? (int)(next() % 2047) - 1023 : (int)(next() % 400) - 200, next() & 1);
        }
        double y = 1.0 / d;
        double q = a * y;
        double r = fma(-d, q, a);
        double q1 = fma(r, y, q);
        const double lo = 0x1p-900, hi = 0x1p900;
        if (!(fabs(a) > lo && fabs(a) < hi && fabs(q1) > lo && fabs(q1) < hi)) { ++guarded; continue; }
        double want = a / d;
        if (memcmp(&q1, &want, 8) != 0) {
            if (bad < 10) printf("MISMATCH a=%a d=%a got %a want %a\n", a, d, q1, want);
            ++bad;
        }
    }
    /* zero numerators: the kernel returns RN(a * y) when y is finite and nonzero */
    long long zeros = 0;
    for (long long i = 0; i < n / 100; ++i) {
        const double d = mk(mant_sample(), (int)(next() % 2047) - 1023, next() & 1);
        const double a = (next() & 1) ? -0.0 : 0.0;
        const double y = 1.0 / d;
        if (!(fabs(y) > 0.0 && fabs(y) < INFINITY)) continue;
        const double q = a * y, want = a / d;
        ++zeros;
        if (memcmp(&q, &want, 8) != 0) {
            if (bad < 10) printf("ZERO MISMATCH a=%a d=%a got %a want %a\n", a, d, q, want);
            ++bad;
        }
    }
    printf("samples %lld mismatches %lld guarded(slow path) %lld zero-numerator samples %lld\n", n, bad, guarded, zeros);
    return bad != 0;
}
