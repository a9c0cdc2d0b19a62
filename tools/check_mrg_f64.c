/* Host check of the all-fp64 symmetric-residue MRG32k3a step used by
 * csrc/common.cuh mrg_step_f64: same operation sequence with C99 fma()
 * (IEEE binary64, round-to-nearest, as DFMA/DMUL/DADD), compared with the
 * int64 recurrence of _core.pyx:85-101 from random and extreme start windows.
 *   gcc -O2 -ffp-contract=off -o c check_mrg_f64.c -lm && ./c */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static const int64_t m1 = 4294967087LL, m2 = 4294944443LL;
static const double MAGIC = 6755399441055744.0;

static double sym(uint32_t x, uint32_t m) { return x > m / 2 ? (double)x - (double)m : (double)x; }
static double red(double p, double m, double inv) {
    double k = fma(p, inv, MAGIC) - MAGIC;
    return fma(-k, m, p);
}
static uint32_t canon(double r, uint32_t m) {
    double t = r + MAGIC;
    uint64_t b;
    memcpy(&b, &t, 8);
    int32_t i = (int32_t)(uint32_t)b;
    return (uint32_t)i + (i < 0 ? m : 0u);
}

int main(void) {
    uint64_t rng = 0x9E3779B97F4A7C15ull, bad = 0, steps = 0;
    double maxabs = 0;
    for (int trial = 0; trial < 4000; ++trial) {
        int64_t x[3], y[3];
        for (int i = 0; i < 3; ++i) {
            rng = rng * 6364136223846793005ull + 1442695040888963407ull;
            uint64_t r = rng >> 11;
            int mode = trial % 4;
            x[i] = mode == 0 ? (int64_t)(r % m1) : mode == 1 ? m1 - 1 - (int64_t)(r % 3) : mode == 2 ? m1 / 2 + (int64_t)(r % 3) - 1 : (int64_t)(r % 3);
            y[i] = mode == 0 ? (int64_t)((r >> 7) % m2) : mode == 1 ? m2 - 1 - (int64_t)(r % 3) : mode == 2 ? m2 / 2 + (int64_t)(r % 3) - 1 : (int64_t)(r % 3);
        }
        double d[6] = {sym(x[0], m1), sym(x[1], m1), sym(x[2], m1), sym(y[0], m2), sym(y[1], m2), sym(y[2], m2)};
        for (int s = 0; s < 25000; ++s, ++steps) {
            int64_t p1 = (1403580LL * x[1] - 810728LL * x[0]) % m1; if (p1 < 0) p1 += m1;
            int64_t p2 = (527612LL * y[2] - 1370589LL * y[0]) % m2; if (p2 < 0) p2 += m2;
            x[0] = x[1]; x[1] = x[2]; x[2] = p1; y[0] = y[1]; y[1] = y[2]; y[2] = p2;
            int64_t z = p1 - p2; if (z < 0) z += m1;
            double q1 = red(fma(-810728.0, d[0], 1403580.0 * d[1]), (double)m1, 1.0 / (double)m1);
            double q2 = red(fma(-1370589.0, d[3], 527612.0 * d[5]), (double)m2, 1.0 / (double)m2);
            d[0] = d[1]; d[1] = d[2]; d[2] = q1; d[3] = d[4]; d[4] = d[5]; d[5] = q2;
            if (fabs(q1) > maxabs) maxabs = fabs(q1);
            if (fabs(q2) > maxabs) maxabs = fabs(q2);
            uint32_t c1 = canon(q1, (uint32_t)m1), c2 = canon(q2, (uint32_t)m2);
            uint32_t zz = c1 >= c2 ? c1 - c2 : c1 - c2 + (uint32_t)m1;
            if (zz != (uint32_t)z || c1 != (uint32_t)p1 || c2 != (uint32_t)p2) ++bad;
        }
    }
    printf("mrg fp64 symmetric step: %llu steps, %llu mismatches, max |residue| = %.0f (m1/2 = %lld)\n",
           (unsigned long long)steps, (unsigned long long)bad, maxabs, (long long)(m1 / 2));
    return bad != 0;
}
