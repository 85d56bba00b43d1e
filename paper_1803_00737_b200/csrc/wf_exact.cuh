// wavefuse-b200: the reference's float64 operations in its own evaluation
// order (wavelet.py:73-109), shared by the transform kernels, the one-pass
// reference-exact fusion kernels (transforms.cu) and the byte-exact fix-up of
// the 8 bpp D4 kernel (fuse_tma.cu). Every product and sum is an explicit
// round-to-nearest intrinsic, so no FMA contraction changes a bit: numpy
// evaluates `h0*even + h1*odd + h2*even1 + h3*odd1` (wavelet.py:85) as
// ((h0*e + h1*o) + h2*e1) + h3*o1 with each operation correctly rounded.
#pragma once

#include "wf_common.cuh"

namespace wf {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// wavelet.py:75-86 (one output pair of _forward_last)
__device__ __forceinline__ double fwd_lo(int kind, const D4& t, double x0, double x1, double x2,
                                         double x3) {
  if (kind == kHaar) return mul(add(x0, x1), 0.5);
  return add(add(add(mul(t.h0, x0), mul(t.h1, x1)), mul(t.h2, x2)), mul(t.h3, x3));
}
__device__ __forceinline__ double fwd_hi(int kind, const D4& t, double x0, double x1, double x2,
                                         double x3) {
  if (kind == kHaar) return mul(sub(x0, x1), 0.5);
  return add(add(add(mul(t.g0, x0), mul(t.g1, x1)), mul(t.g2, x2)), mul(t.g3, x3));
}
// wavelet.py:96-108 (one output sample of _inverse_last). p = 0: even sample,
// taps synthesis_even = [h2, g2, h0, g0]; p = 1: odd, [h3, g3, h1, g1].
// Haar: even = a + d, odd = a - d.
__device__ __forceinline__ double inv_tap(int kind, const D4& t, int p, double ap, double dp,
                                          double a, double d) {
  if (kind == kHaar) return p == 0 ? add(a, d) : sub(a, d);
  if (p == 0) return add(add(add(mul(t.h2, ap), mul(t.g2, dp)), mul(t.h0, a)), mul(t.g0, d));
  return add(add(add(mul(t.h3, ap), mul(t.g3, dp)), mul(t.h1, a)), mul(t.g1, d));
}

}  // namespace wf
