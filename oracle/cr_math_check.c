/* cr_math_check.c -- TEST INFRASTRUCTURE. Exhaustive check that the oracle's
 * fp32 transcendentals are correctly rounded on the 2^24-point grids the particle
 * filter feeds them (tracking.cpp:29-36): u1 = ((w>>8)+1)*2^-24, u2 = (w>>8)*2^-24,
 * angle = RN(2pi_f * u2). Reference value: long double (64-bit mantissa) rounded once.
 * Prints mismatch counts and writes nothing else; exit 0 iff all counts are zero. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include "ut_oracle.h"

int main(void) {
  long bad_log = 0, bad_cos = 0, bad_sin = 0;
  for (uint32_t k = 1; k <= (1u << 24); ++k) {
    const float x = (float)k * 0x1.0p-24f;
    if (uto_cr_logf(x) != (float)logl((long double)x)) ++bad_log;
  }
  const float two_pi_f = 2.0f * 3.14159265358979323846f;
  for (uint32_t m = 0; m < (1u << 24); ++m) {
    const float a = two_pi_f * ((float)m * 0x1.0p-24f);
    if (uto_cr_cosf(a) != (float)cosl((long double)a)) ++bad_cos;
    if (uto_cr_sinf(a) != (float)sinl((long double)a)) ++bad_sin;
  }
  printf("{\"log_mismatch\": %ld, \"cos_mismatch\": %ld, \"sin_mismatch\": %ld}\n", bad_log, bad_cos, bad_sin);
  return (bad_log || bad_cos || bad_sin) ? 1 : 0;
}
