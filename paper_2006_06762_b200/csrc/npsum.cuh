// numpy's float64 summation orders, reproduced on the device (exactness
// contract of the scoring and training kernels; compile with --fmad=false).
#pragma once
#include <stdint.h>

namespace lt {

// numpy pairwise_sum for float64 (numpy/_core/src/umath/loops_utils.h.src):
// plain loop from +0.0 below 8 items, 8 accumulators up to 128, halving above.
__device__ inline double np_block(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = a[k];
  int64_t i;
  for (i = 8; i < n - (n % 8); i += 8)
    for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[i + k]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ inline double np_pairwise(const double* a, int64_t n) {
  if (n <= 128) return np_block(a, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

}  // namespace lt
