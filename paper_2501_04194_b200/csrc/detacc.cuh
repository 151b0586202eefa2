// detacc.cuh — reproducible scatter-add of fp32 contributions.
//
// Float atomics make a sum depend on the arrival order.  Here every contribution x of a
// row is split on a per-row power-of-two grid tied to the row's largest cotangent |g|max:
//   hi = round(x 2^S),   lo = round((x - hi 2^-S) 2^(S+40)),   S = 28 - ilogb(|g|max)
// and hi / lo are summed with int64 atomics (LSE / hard VJPs, whose weights lie in [0, 1],
// use hi alone on a grid sized from the number of contributions per element).  Integer addition is associative, so the
// total is the same for every order; both roundings are exact-grid roundings, so the
// result is x summed to within 2^-69 |g|max per term (far below fp32 resolution).  hi
// holds sums up to 2^34 |g|max: LSE Until weights sum to 1 per output, softmax ones to at
// most (1 + tau range)^3, so partial sums stay inside it for any practical signal.
#pragma once
#include <cstdint>

namespace stlg {

struct DetRow {
  unsigned long long* hi;  // row base of the hi plane
  unsigned long long* lo;  // row base of the lo plane (nullptr: one-word mode)
  double s_hi, s_lo;       // 2^S, 2^(S+40)
  __device__ __forceinline__ void add(long long j, float x) const {
    if (x == 0.f) return;
    const double xd = (double)x;
    const double h = rint(xd * s_hi);
    atomicAdd(hi + j, (unsigned long long)(long long)h);
    if (lo == nullptr) return;
    const double r = xd - h / s_hi;  // exact: the part of x below the hi grid
    atomicAdd(lo + j, (unsigned long long)llrint(r * s_lo));
  }
};

// per-row grid exponent S (one CTA per row): two-word mode S = 28 - ilogb(max |g|);
// one-word mode (span = bits for the largest |sum| / |g|max, e.g. log2 of the number of
// outputs reaching one element when every weight lies in [0, 1]) S = 61 - span - ilogb
__global__ void k_det_row_scale(const float* __restrict__ cot, long long L, int span, int* __restrict__ S);
// out[j] = hi 2^-S + lo 2^-(S+40) rounded once to fp32, every element of every row
__global__ void k_det_finish(const unsigned long long* __restrict__ hi, const unsigned long long* __restrict__ lo,
                             const int* __restrict__ S, long long B, long long L, float* __restrict__ out);

__device__ __forceinline__ DetRow det_row(unsigned long long* plane_hi, unsigned long long* plane_lo,
                                          const int* S, long long row, long long L, bool two) {
  const int s = S[row];
  return DetRow{plane_hi + row * L, two ? plane_lo + row * L : nullptr, ldexp(1.0, s), ldexp(1.0, s + 40)};
}

}  // namespace stlg
