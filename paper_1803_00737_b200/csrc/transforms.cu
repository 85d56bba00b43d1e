// wavefuse-b200: standalone single-level transforms, bilinear resample and the
// synthetic-scene generator (sm_100a).
//
// These back the reference's public transform API (wavelet.py:131-164) and
// resample_bilinear (fusion.py:50-81). Unlike the fused kernels (fuse.cu) they
// must materialise the coefficient image, because that is their contract.
//
// Arithmetic is float64 for both I/O dtypes, exactly like the reference
// (wavelet.py:12-15: "Arithmetic runs in double precision regardless of input
// dtype"), and every product/sum is issued with explicit round-to-nearest
// intrinsics (__dmul_rn/__dadd_rn) in the reference's evaluation order, so no
// FMA contraction happens. numpy evaluates `h0*even + h1*odd + h2*even1 +
// h3*odd1` (wavelet.py:85) as ((h0*e + h1*o) + h2*e1) + h3*o1 with each
// operation correctly rounded; so does this file, so results are
// bit-identical to the reference (tests/test_gpu_parity.py checks equality).
#include "wf_common.cuh"
#include "wf_kernels.h"

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

// ---- 2D forward: rows then columns (wavelet.py:149-155) -------------------
// One thread per coefficient position (i, j) of the half-size grid; it writes
// LL(i,j), HL(i, Wh+j), LH(Hh+i, j), HH(Hh+i, Wh+j).
template <typename T, typename To = T>
__global__ void dwt2d_forward_kernel(int kind, const T* __restrict__ in, long long ip,
                                     To* __restrict__ out, long long op, int H, int W) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  const int Hh = H >> 1, Wh = W >> 1;
  if (i >= Hh || j >= Wh) return;
  const D4 t = d4_taps();
  const int taps = kind == kHaar ? 2 : 4;
  double a[4], d[4];
  for (int k = 0; k < taps; ++k) {
    const T* row = in + (long long)wrap(2 * i + k, H) * ip;
    double x[4];
    for (int l = 0; l < taps; ++l) x[l] = (double)row[wrap(2 * j + l, W)];
    if (kind == kHaar) x[2] = x[3] = 0.0;
    a[k] = fwd_lo(kind, t, x[0], x[1], x[2], x[3]);
    d[k] = fwd_hi(kind, t, x[0], x[1], x[2], x[3]);
  }
  if (kind == kHaar) a[2] = a[3] = d[2] = d[3] = 0.0;
  out[(long long)i * op + j] = (To)fwd_lo(kind, t, a[0], a[1], a[2], a[3]);
  out[(long long)i * op + Wh + j] = (To)fwd_lo(kind, t, d[0], d[1], d[2], d[3]);
  out[(long long)(Hh + i) * op + j] = (To)fwd_hi(kind, t, a[0], a[1], a[2], a[3]);
  out[(long long)(Hh + i) * op + Wh + j] = (To)fwd_hi(kind, t, d[0], d[1], d[2], d[3]);
}

// ---- 2D inverse: columns then rows (wavelet.py:158-164) -------------------
// One thread per output 2x2 block (i, j).
template <typename T, typename To = T>
__global__ void dwt2d_inverse_kernel(int kind, const T* __restrict__ in, long long ip,
                                     To* __restrict__ out, long long op, int H, int W) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  const int Hh = H >> 1, Wh = W >> 1;
  if (i >= Hh || j >= Wh) return;
  const D4 t = d4_taps();
  const int im = wrap(i - 1, Hh), jm = wrap(j - 1, Wh);
  // the four coefficient columns the row-inverse of output cols 2j, 2j+1 needs
  const int cols[4] = {jm, Wh + jm, j, Wh + j};
  double cv[2][4];
  for (int k = 0; k < 4; ++k) {
    const int col = cols[k];
    const double ap = (double)in[(long long)im * ip + col];
    const double dp = (double)in[(long long)(Hh + im) * ip + col];
    const double a = (double)in[(long long)i * ip + col];
    const double d = (double)in[(long long)(Hh + i) * ip + col];
    cv[0][k] = inv_tap(kind, t, 0, ap, dp, a, d);
    cv[1][k] = inv_tap(kind, t, 1, ap, dp, a, d);
  }
  for (int p = 0; p < 2; ++p) {
    To* row = out + (long long)(2 * i + p) * op;
    row[2 * j] = (To)inv_tap(kind, t, 0, cv[p][0], cv[p][1], cv[p][2], cv[p][3]);
    row[2 * j + 1] = (To)inv_tap(kind, t, 1, cv[p][0], cv[p][1], cv[p][2], cv[p][3]);
  }
}

// ---- reference-exact fusion (fusion.py:148-150 step by step) ---------------
// coeffs[:h/2, :w/2] = band.astype(f64) * gain  (fusion.py:149)
template <typename T>
__global__ void ll_replace_kernel(double* __restrict__ coeff, long long cp,
                                  const T* __restrict__ ms, long long mp, int hh, int wh,
                                  double gain) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= hh || j >= wh) return;
  coeff[(long long)i * cp + j] = mul((double)ms[(long long)i * mp + j], gain);
}

// ---- rows-only transforms (dwt1d_* is the nrows = 1 case) ------------------
template <typename T>
__global__ void dwt_rows_forward_kernel(int kind, const T* __restrict__ in, long long ip,
                                        T* __restrict__ out, long long op, int nrows, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const int nh = n >> 1;
  if (j >= nh || r >= nrows) return;
  const D4 t = d4_taps();
  const T* row = in + (long long)r * ip;
  double x[4] = {(double)row[2 * j], (double)row[2 * j + 1], 0.0, 0.0};
  if (kind != kHaar) {
    x[2] = (double)row[wrap(2 * j + 2, n)];
    x[3] = (double)row[wrap(2 * j + 3, n)];
  }
  out[(long long)r * op + j] = (T)fwd_lo(kind, t, x[0], x[1], x[2], x[3]);
  out[(long long)r * op + nh + j] = (T)fwd_hi(kind, t, x[0], x[1], x[2], x[3]);
}

template <typename T>
__global__ void dwt_rows_inverse_kernel(int kind, const T* __restrict__ in, long long ip,
                                        T* __restrict__ out, long long op, int nrows, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  const int nh = n >> 1;
  if (j >= nh || r >= nrows) return;
  const D4 t = d4_taps();
  const T* row = in + (long long)r * ip;
  const int jm = wrap(j - 1, nh);
  const double ap = (double)row[jm], dp = (double)row[nh + jm];
  const double a = (double)row[j], d = (double)row[nh + j];
  out[(long long)r * op + 2 * j] = (T)inv_tap(kind, t, 0, ap, dp, a, d);
  out[(long long)r * op + 2 * j + 1] = (T)inv_tap(kind, t, 1, ap, dp, a, d);
}

// ---- bilinear resample, pixel-centre aligned, clamped (fusion.py:67-81) ----
__device__ __forceinline__ void src_coord(int dst, int in_n, int out_n, int& i0, int& i1,
                                          double& f) {
  // np.clip((arange + 0.5) * (in/out) - 0.5, 0, in-1)
  double s = sub(mul((double)dst + 0.5, (double)in_n / (double)out_n), 0.5);
  s = fmin(fmax(s, 0.0), (double)(in_n - 1));
  const double fl = floor(s);
  i0 = (int)fl;
  i1 = min(i0 + 1, in_n - 1);
  f = sub(s, fl);
}

template <typename T, typename To>
__global__ void resample_kernel(const T* __restrict__ in, long long ip, int in_h, int in_w,
                                To* __restrict__ out, long long op, int out_h, int out_w) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= out_w || y >= out_h) return;
  int x0, x1, y0, y1;
  double fx, fy;
  src_coord(x, in_w, out_w, x0, x1, fx);
  src_coord(y, in_h, out_h, y0, y1, fy);
  const T* up = in + (long long)y0 * ip;
  const T* lo = in + (long long)y1 * ip;
  const double gx = sub(1.0, fx), gy = sub(1.0, fy);
  const double ru = add(mul((double)up[x0], gx), mul((double)up[x1], fx));
  const double rl = add(mul((double)lo[x0], gx), mul((double)lo[x1], fx));
  out[(long long)y * op + x] = (To)add(mul(ru, gy), mul(rl, fy));
}

// ---- counter-hash synthetic planes -----------------------------------------
// value(seed, plane, row, col) = 255 * u24 / 2^24, u24 = top 24 bits of a
// splitmix64 finaliser of (seed*phi + (plane<<48 ^ row<<24 ^ col)). Addressable
// per pixel, so any window of a 65536^2 scene is reproducible on the host
// (numpy twin: paper_1803_00737_b200/synth.py).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__global__ void synth_kernel(float* __restrict__ out, long long pitch, int rows, int cols,
                             unsigned long long seed, unsigned plane, int row0, int col0) {
  const int x4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (x4 >= cols) return;
  for (int y = blockIdx.y; y < rows; y += gridDim.y) {
  const unsigned long long rowkey = ((unsigned long long)plane << 48) ^
                                    ((unsigned long long)(unsigned)(row0 + y) << 24);
  const unsigned long long s = seed * 0x9E3779B97F4A7C15ull;
  float* dst = out + (long long)y * pitch;
  for (int k = 0; k < 4 && x4 + k < cols; ++k) {
    const unsigned long long z =
        mix64(s + (rowkey ^ (unsigned long long)(unsigned)(col0 + x4 + k)));
    dst[x4 + k] = __fmul_rn((float)(unsigned)(z >> 40), 255.0f / 16777216.0f);
  }
  }
}

// ---- 8 bpp conversions (imageio.py:104-123) --------------------------------
__global__ void u8_to_f32_kernel(const uint8_t* __restrict__ in, long long ip, int h, int w,
                                 float* __restrict__ out, long long op) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int y = blockIdx.y; y < h; y += gridDim.y)
    if (x < w) out[(long long)y * op + x] = (float)in[(long long)y * ip + x];
}

// quantize: clamp to [0, 255] then floor(x + 0.5), in float32 like numpy on a
// float32 plane (imageio.py:115-123)
template <typename T>
__global__ void quantize_kernel(const T* __restrict__ in, long long ip, int h, int w,
                                uint8_t* __restrict__ out, long long op) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int y = blockIdx.y; y < h; y += gridDim.y)
    if (x < w) {
      const T v = fmin(fmax(in[(long long)y * ip + x], T(0)), T(255));
      out[(long long)y * op + x] = (uint8_t)floor(v + T(0.5));
    }
}

// ---- launchers --------------------------------------------------------------
cudaError_t launch_u8_to_f32(const uint8_t* in, long long ip, int h, int w, float* out,
                             long long op, cudaStream_t s) {
  dim3 grid((w + 255) / 256, h < 65535 ? h : 65535);
  u8_to_f32_kernel<<<grid, 256, 0, s>>>(in, ip, h, w, out, op);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_quantize(const T* in, long long ip, int h, int w, uint8_t* out, long long op,
                            cudaStream_t s) {
  dim3 grid((w + 255) / 256, h < 65535 ? h : 65535);
  quantize_kernel<T><<<grid, 256, 0, s>>>(in, ip, h, w, out, op);
  return cudaGetLastError();
}
template cudaError_t launch_quantize<float>(const float*, long long, int, int, uint8_t*, long long,
                                            cudaStream_t);
template cudaError_t launch_quantize<double>(const double*, long long, int, int, uint8_t*,
                                             long long, cudaStream_t);

template <typename T>
cudaError_t launch_dwt2d(int kind, bool inverse, const T* in, long long ip, T* out,
                         long long op, int h, int w, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid(((w >> 1) + 31) / 32, ((h >> 1) + 7) / 8);
  if (inverse)
    dwt2d_inverse_kernel<T><<<grid, block, 0, s>>>(kind, in, ip, out, op, h, w);
  else
    dwt2d_forward_kernel<T><<<grid, block, 0, s>>>(kind, in, ip, out, op, h, w);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dwt_rows(int kind, bool inverse, const T* in, long long ip, T* out,
                            long long op, int nrows, int n, cudaStream_t s) {
  dim3 grid(((n >> 1) + 127) / 128, nrows);
  if (inverse)
    dwt_rows_inverse_kernel<T><<<grid, 128, 0, s>>>(kind, in, ip, out, op, nrows, n);
  else
    dwt_rows_forward_kernel<T><<<grid, 128, 0, s>>>(kind, in, ip, out, op, nrows, n);
  return cudaGetLastError();
}

template <typename T, typename To>
cudaError_t launch_resample(const T* in, long long ip, int in_h, int in_w, To* out, long long op,
                            int out_h, int out_w, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((out_w + 31) / 32, (out_h + 7) / 8);
  resample_kernel<T, To><<<grid, block, 0, s>>>(in, ip, in_h, in_w, out, op, out_h, out_w);
  return cudaGetLastError();
}

cudaError_t launch_synth(float* out, long long pitch, int rows, int cols, unsigned long long seed,
                         unsigned plane, int row0, int col0, cudaStream_t s) {
  dim3 grid(((cols + 3) / 4 + 255) / 256, rows < 65535 ? rows : 65535);
  synth_kernel<<<grid, 256, 0, s>>>(out, pitch, rows, cols, seed, plane, row0, col0);
  return cudaGetLastError();
}

// fuse_dwt exactly as the reference computes it: float64 forward transform
// of the PAN plane (its exact operation order), LL <- band * gain, float64
// inverse, one final cast to the PAN dtype. `ws` = h * w doubles.
template <typename T>
cudaError_t launch_fuse_exact(int kind, const T* pan, long long pp, const T* ms, long long mp,
                              T* out, long long op, int h, int w, double* ws, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid(((w >> 1) + 31) / 32, ((h >> 1) + 7) / 8);
  dwt2d_forward_kernel<T, double><<<grid, block, 0, s>>>(kind, pan, pp, ws, w, h, w);
  ll_replace_kernel<T><<<grid, block, 0, s>>>(ws, w, ms, mp, h >> 1, w >> 1,
                                              kind == kHaar ? 1.0 : 2.0);
  dwt2d_inverse_kernel<double, T><<<grid, block, 0, s>>>(kind, ws, w, out, op, h, w);
  return cudaGetLastError();
}
template cudaError_t launch_fuse_exact<float>(int, const float*, long long, const float*,
                                              long long, float*, long long, int, int, double*,
                                              cudaStream_t);
template cudaError_t launch_fuse_exact<double>(int, const double*, long long, const double*,
                                               long long, double*, long long, int, int, double*,
                                               cudaStream_t);

template cudaError_t launch_dwt2d<float>(int, bool, const float*, long long, float*, long long,
                                         int, int, cudaStream_t);
template cudaError_t launch_dwt2d<double>(int, bool, const double*, long long, double*,
                                          long long, int, int, cudaStream_t);
template cudaError_t launch_dwt_rows<float>(int, bool, const float*, long long, float*,
                                            long long, int, int, cudaStream_t);
template cudaError_t launch_dwt_rows<double>(int, bool, const double*, long long, double*,
                                             long long, int, int, cudaStream_t);
template cudaError_t launch_resample<float, float>(const float*, long long, int, int, float*,
                                                   long long, int, int, cudaStream_t);
template cudaError_t launch_resample<double, double>(const double*, long long, int, int, double*,
                                                     long long, int, int, cudaStream_t);
template cudaError_t launch_resample<float, double>(const float*, long long, int, int, double*,
                                                    long long, int, int, cudaStream_t);

}  // namespace wf
