/* Host check of the glibc log/sin/cos replica (emc_libm.h) against the
 * system libm, on the argument distributions of the transport path:
 *   log(1 - u), sin(2*pi*u), cos(2*pi*u) with u = s * 2^-63 (the reference's
 *   uniform, kernels.py:161-169), plus random bit patterns over wider ranges.
 * Usage: libm_check N seed   -> prints "checked <n> mismatches <m>" and the
 * first few mismatching inputs.  Compiled with -ffp-contract=off.
 */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <math.h>
#include "../../paper_2403_12345_b200/csrc/emc_libm.h"

static uint64_t sm64(uint64_t *s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static double (*volatile g_log)(double) = log;
static double (*volatile g_sin)(double) = sin;
static double (*volatile g_cos)(double) = cos;

int main(int argc, char **argv) {
    long n = argc > 1 ? atol(argv[1]) : 1000000;
    uint64_t seed = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
    long bad = 0, checked = 0;
    const double TWO_PI = 2.0 * 3.141592653589793;
#pragma omp parallel for reduction(+:bad,checked) schedule(static)
    for (long i = 0; i < n; ++i) {
        uint64_t st = seed * 0x100000001b3ULL + (uint64_t)i * 0x9e3779b97f4a7c15ULL;
        uint64_t r = sm64(&st);
        uint64_t s = r & ((1ULL << 63) - 1);
        double u = (double)s * 0x1p-63;
        if (u >= 1.0) u = 1.0 - 0x1p-53;
        double xs[6];
        xs[0] = 1.0 - u;                         /* log arg */
        xs[1] = TWO_PI * u;                      /* sin/cos arg */
        /* random bit patterns: positive doubles in [2^-60, 2^60) for log,
           [0, 7) for sin/cos, and values near 1 for the log poly path */
        uint64_t r2 = sm64(&st);
        xs[2] = ldexp(1.0 + (double)(r2 >> 12) * 0x1p-52, (int)(sm64(&st) % 120) - 60);
        xs[3] = (double)(r2 >> 11) * 0x1p-53 * 7.0;
        xs[4] = 1.0 + ((double)(int64_t)(r2 >> 11) * 0x1p-53 - 0.5) * 0.15;
        xs[5] = (double)(sm64(&st) >> 11) * 0x1p-53 * 0x1p-20;   /* small angles */
        double a, b;
        for (int t = 0; t < 6; ++t) {
            double x = xs[t];
            if (t == 0 || t == 2 || t == 4) {
                a = emc_log(x); b = g_log(x); checked++;
                if (memcmp(&a, &b, 8)) { bad++; if (bad < 8) printf("log %a: %a vs %a\n", x, a, b); }
            }
            if (t == 1 || t == 3 || t == 5) {
                a = emc_sin(x); b = g_sin(x); checked++;
                if (memcmp(&a, &b, 8)) { bad++; if (bad < 8) printf("sin %a: %a vs %a\n", x, a, b); }
                a = emc_cos(x); b = g_cos(x); checked++;
                if (memcmp(&a, &b, 8)) { bad++; if (bad < 8) printf("cos %a: %a vs %a\n", x, a, b); }
            }
        }
    }
    printf("checked %ld mismatches %ld\n", checked, bad);
    return bad != 0;
}
