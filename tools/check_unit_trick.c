/* Exhaustive check of the I2FP-free 24-bit unit conversion used by
 * csrc/common.cuh unit_f32: for every m in [0, 2^24),
 *   F = bits(0x3F000000 | m),  u = min(F - 0.5, F * 0.5)  ==  m * 2^-24
 * bit-for-bit (including +0.0 at m = 0).  gcc -O2 -o c check_unit_trick.c */
#include <stdint.h>
#include <stdio.h>
#include <string.h>
static float asf(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t asu(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
int main(void) {
    long bad = 0;
    for (uint32_t m = 0; m < (1u << 24); ++m) {
        const float want = (float)m * 5.9604644775390625e-08f;
        const float f = asf(0x3F000000u | m);
        const float a = f - 0.5f, b = f * 0.5f;
        const float u = a < b ? a : b;
        if (asu(u) != asu(want)) ++bad;
    }
    printf("unit trick: %ld mismatches over 2^24 inputs\n", bad);
    return bad != 0;
}
