"""Worst-case error bound of the 8 bpp D4 kernel's float32 arithmetic
(fuse_d4_u8x8_kernel, csrc/fuse_tma.cu) against the exact real value of
pan + S_LL(2 ms - LL(pan)), by forward error analysis: every float32
operation rounds to nearest (|rel err| <= u = 2^-24), the float32 taps differ
from the real ones by <= u |h|, and the uint8 inputs are exact. Each value is
tracked as (magnitude bound M, absolute error bound E).

The kernel's byte is exact whenever the bound is below the flag window
(2^-9): the reference's value (float64 sequence, then
cast to float32, then quantize in float32) lies within E + 2^-17 + 1e-9 of
the kernel's float32 value, so a pixel whose value is at least 2^-9 away from
every rounding boundary k + 0.5 gets the reference's byte.

    python tools/u8_error_bound.py
"""

import math

u = 2.0 ** -24
s3 = math.sqrt(3.0)
h = [(1 + s3) / (4 * math.sqrt(2)), (3 + s3) / (4 * math.sqrt(2)),
     (3 - s3) / (4 * math.sqrt(2)), (1 - s3) / (4 * math.sqrt(2))]
H = [abs(x) for x in h]


class V:
    def __init__(self, m, e):
        self.m, self.e = m, e


def tap(k):  # float32 tap: |h32 - h| <= u |h|
    return V(H[k], u * H[k])


def mul(a, b):  # fl(a*b)
    m = a.m * b.m
    e = a.m * b.e + b.m * a.e + a.e * b.e
    return V(m, e + u * (m + e))


def fma(a, b, c):  # fl(a*b + c), one rounding
    m = a.m * b.m + c.m
    e = a.m * b.e + b.m * a.e + a.e * b.e + c.e
    return V(m, e + u * (m + e))


def add(a, b):
    m = a.m + b.m
    e = a.e + b.e
    return V(m, e + u * (m + e))


def exact(m):
    return V(m, 0.0)


def dot4(xs):  # fma(h3, x3, fma(h2, x2, fma(h1, x1, h0 * x0)))
    acc = mul(tap(0), xs[0])
    for k in (1, 2, 3):
        acc = fma(tap(k), xs[k], acc)
    return acc


pan = exact(255.0)
rn = dot4([pan] * 4)                   # row low-pass of one PAN row
ll = dot4([rn] * 4)                    # column low-pass over 4 rows: LL(pan)
e = fma(exact(2.0), exact(255.0), ll)  # E = 2 ms - LL (one rounding)
# vertical synthesis V = h01 * E(i) + h23 * E(i-1): fma(h0, e, h2 * ep)
v = fma(tap(0), e, mul(tap(2), e))
v_odd = fma(tap(1), e, mul(tap(3), e))
vmax = V(max(v.m, v_odd.m), max(v.e, v_odd.e))
# horizontal synthesis into the output: fma(h0, V1, fma(h2, V0, pan + 0.5 + 2^-9))
pa = exact(255.0 + 0.5 + 2.0 ** -9)
o = fma(tap(0), vmax, fma(tap(2), vmax, pa))
o_odd = fma(tap(1), vmax, fma(tap(3), vmax, pa))
bound = max(o.e, o_odd.e)
ref_cast = 2.0 ** -17      # float64 -> float32 of a value < 256 (half ulp); larger
#                            values clamp to 255 whatever their rounding
ref_f64 = 1e-9             # the float64 sequence vs the real value (<< 1e-9)
total = bound + ref_cast + ref_f64
print(f"|LL| <= {ll.m:.1f}, |E| <= {e.m:.1f}, |V| <= {vmax.m:.1f}, |o| <= {max(o.m, o_odd.m):.1f}")
print(f"float32 kernel error bound: {bound:.3e}")
print(f"+ reference cast and float64 error: {total:.3e}")
print(f"flag window 2^-9 = {2.0 ** -9:.3e}: margin x{2.0 ** -9 / total:.1f}")
assert total < 2.0 ** -9
