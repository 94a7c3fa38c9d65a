/* Validates paper_2505_21070_b200/csrc/glibc_port.h against this image's
 * glibc on the host: every Box-Muller input kind the noise kernel sees.
 * Build: gcc -O2 -ffp-contract=off -I paper_2505_21070_b200/csrc tools/check_glibc_port.c -lm */
#include <stdio.h>
#include <stdlib.h>
#include "glibc_port.h"

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 10000000;
  uint64_t st = 0x123456789ULL;
  long bad_log = 0, bad_cos = 0, bad_bm = 0;
  for (long i = 0; i < n; ++i) {
    st += 0x9E3779B97F4A7C15ULL; uint64_t a = bp_splitmix_mix(st);
    st += 0x9E3779B97F4A7C15ULL; uint64_t b = bp_splitmix_mix(st);
    double u1 = (double)((a >> 11) + 1) * 0x1p-53;
    double u2 = (double)(b >> 11) * 0x1p-53;
    double x = 0x1.921fb54442d18p+2 * u2;
    if (bp_asu64(bp_glibc_log(u1)) != bp_asu64(log(u1))) { if (bad_log++ < 5) printf("log %a: %a vs %a\n", u1, bp_glibc_log(u1), log(u1)); }
    if (bp_asu64(bp_glibc_cos(x)) != bp_asu64(cos(x))) { if (bad_cos++ < 5) printf("cos %a: %a vs %a\n", x, bp_glibc_cos(x), cos(x)); }
    double ref = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2) * 0.7;
    if (bp_asu64(bp_box_muller(a, b, 0.7)) != bp_asu64(ref)) bad_bm++;
    /* extra: uniform doubles across the whole log domain used, and near 1 */
    double v = (double)(a >> 11) * 0x1p-53 * 0.2 + 0.93;
    if (v > 0 && bp_asu64(bp_glibc_log(v)) != bp_asu64(log(v))) { if (bad_log++ < 5) printf("log1 %a\n", v); }
    double w = (double)(b >> 11) * 0x1p-53 * 7.0;
    if (bp_asu64(bp_glibc_cos(w)) != bp_asu64(cos(w))) { if (bad_cos++ < 5) printf("cos2 %a\n", w); }
  }
  printf("n=%ld bad_log=%ld bad_cos=%ld bad_boxmuller=%ld\n", n, bad_log, bad_cos, bad_bm);
  return (bad_log || bad_cos || bad_bm) ? 1 : 0;
}
