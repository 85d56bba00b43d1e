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
#include <stdlib.h>

#include "wf_common.cuh"
#include "wf_exact.cuh"
#include "wf_kernels.h"

namespace wf {

// the reference-order float64 operations: wf_exact.cuh

// ---- 2D forward: rows then columns (wavelet.py:149-155) -------------------
// A thread owns coefficient column j and marches down a run of kTrRows
// coefficient rows i. The row pass of PAN rows 2i+2, 2i+3 (wrapped) is
// carried to row i+1, where it is rows 2i, 2i+1, so every PAN row is loaded,
// converted and row-filtered once per column instead of twice (D4). It
// writes LL(i,j), HL(i, Wh+j), LH(Hh+i, j), HH(Hh+i, Wh+j).
constexpr int kTrThreads = 128;
constexpr int kTrRowsDefault = 8;
// coefficient rows per thread (WF_TR_ROWS overrides, for sweeps)
static int tr_rows() {
  static int r = [] {
    const char* e = getenv("WF_TR_ROWS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : kTrRowsDefault;
  }();
  return r;
}

template <int KIND, typename T, typename To>
__global__ void __launch_bounds__(kTrThreads)
    dwt2d_forward_kernel(const T* __restrict__ in, long long ip, To* __restrict__ out,
                         long long op, int H, int W, int rows) {
  const int j = blockIdx.x * kTrThreads + threadIdx.x;
  const int Hh = H >> 1, Wh = W >> 1;
  if (j >= Wh) return;
  const int i0 = blockIdx.y * rows;
  const int i1 = min(i0 + rows, Hh);
  const D4 t = d4_taps();
  const int c0 = 2 * j, c1 = 2 * j + 1;
  const int c2 = KIND == kHaar ? 0 : wrap(2 * j + 2, W), c3 = KIND == kHaar ? 0 : wrap(2 * j + 3, W);
  auto rowpass = [&](int r, double& a, double& d) {
    const T* row = in + (long long)r * ip;
    const double x0 = (double)__ldg(row + c0), x1 = (double)__ldg(row + c1);
    if (KIND == kHaar) {
      a = fwd_lo(kHaar, t, x0, x1, 0.0, 0.0);
      d = fwd_hi(kHaar, t, x0, x1, 0.0, 0.0);
    } else {
      const double x2 = (double)__ldg(row + c2), x3 = (double)__ldg(row + c3);
      a = fwd_lo(kDaub4, t, x0, x1, x2, x3);
      d = fwd_hi(kDaub4, t, x0, x1, x2, x3);
    }
  };
  auto emit = [&](int i, const double (&a)[4], const double (&d)[4]) {
    out[(long long)i * op + j] = (To)fwd_lo(KIND, t, a[0], a[1], a[2], a[3]);
    out[(long long)i * op + Wh + j] = (To)fwd_lo(KIND, t, d[0], d[1], d[2], d[3]);
    out[(long long)(Hh + i) * op + j] = (To)fwd_hi(KIND, t, a[0], a[1], a[2], a[3]);
    out[(long long)(Hh + i) * op + Wh + j] = (To)fwd_hi(KIND, t, d[0], d[1], d[2], d[3]);
  };
  if (KIND == kHaar) {
    for (int i = i0; i < i1; ++i) {
      double a[4] = {0.0, 0.0, 0.0, 0.0}, d[4] = {0.0, 0.0, 0.0, 0.0};
      rowpass(2 * i, a[0], d[0]);
      rowpass(2 * i + 1, a[1], d[1]);
      emit(i, a, d);
    }
    return;
  }
  double a[4], d[4];
  rowpass(2 * i0, a[0], d[0]);
  rowpass(2 * i0 + 1, a[1], d[1]);
  for (int i = i0; i < i1; ++i) {
    rowpass(wrap(2 * i + 2, H), a[2], d[2]);
    rowpass(wrap(2 * i + 3, H), a[3], d[3]);
    emit(i, a, d);
    a[0] = a[2];
    a[1] = a[3];
    d[0] = d[2];
    d[1] = d[3];
  }
}

// ---- 2D inverse: columns then rows (wavelet.py:158-164) -------------------
// A thread owns output columns 2j, 2j+1 and marches down coefficient rows i
// (output rows 2i, 2i+1). The column inverse at coefficient columns
// {j-1, Wh+j-1, j, Wh+j} needs coefficient rows i-1 and i of both halves;
// row i-1's values are carried from the previous step, so each coefficient
// is loaded and converted once per thread.
// LLMS (reference-exact fusion): the LL quadrant is not read from `in` but
// formed as band * gain from the MS plane -- the value fusion.py:149 stores
// there -- so the fused sequence needs no separate LL-replacement pass.
template <int KIND, typename T, typename To, bool LLMS = false, typename Tm = T>
__global__ void __launch_bounds__(kTrThreads)
    dwt2d_inverse_kernel(const T* __restrict__ in, long long ip, To* __restrict__ out,
                         long long op, int H, int W, int rows, const Tm* __restrict__ ms = nullptr,
                         long long mp = 0, double gain = 1.0) {
  const int j = blockIdx.x * kTrThreads + threadIdx.x;
  const int Hh = H >> 1, Wh = W >> 1;
  if (j >= Wh) return;
  const int i0 = blockIdx.y * rows;
  const int i1 = min(i0 + rows, Hh);
  const D4 t = d4_taps();
  const int jm = wrap(j - 1, Wh);
  const int cols[4] = {jm, Wh + jm, j, Wh + j};
  auto load_row = [&](int i, double (&top)[4], double (&bot)[4]) {
    const T* rt = in + (long long)i * ip;
    const T* rb = in + (long long)(Hh + i) * ip;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (KIND == kHaar && k < 2) continue;  // Haar reads columns j, Wh+j of row i only
      if (LLMS && (k & 1) == 0)  // LL(i, col) = band(i, col) * gain
        top[k] = mul((double)__ldg(ms + (long long)i * mp + cols[k]), gain);
      else
        top[k] = (double)__ldg(rt + cols[k]);
      bot[k] = (double)__ldg(rb + cols[k]);
    }
  };
  double pt[4] = {0.0, 0.0, 0.0, 0.0}, pb[4] = {0.0, 0.0, 0.0, 0.0};  // row i-1
  if (KIND != kHaar) load_row(wrap(i0 - 1, Hh), pt, pb);
  for (int i = i0; i < i1; ++i) {
    double ct[4] = {0.0, 0.0, 0.0, 0.0}, cb[4] = {0.0, 0.0, 0.0, 0.0};
    load_row(i, ct, cb);
    double cv[2][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cv[0][k] = inv_tap(KIND, t, 0, pt[k], pb[k], ct[k], cb[k]);
      cv[1][k] = inv_tap(KIND, t, 1, pt[k], pb[k], ct[k], cb[k]);
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      To* row = out + (long long)(2 * i + p) * op;
      row[2 * j] = (To)inv_tap(KIND, t, 0, cv[p][0], cv[p][1], cv[p][2], cv[p][3]);
      row[2 * j + 1] = (To)inv_tap(KIND, t, 1, cv[p][0], cv[p][1], cv[p][2], cv[p][3]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pt[k] = ct[k];
      pb[k] = cb[k];
    }
  }
}

template <typename T, typename To>
static void run_dwt2d(int kind, bool inverse, const T* in, long long ip, To* out, long long op,
                      int h, int w, cudaStream_t s) {
  dim3 grid(((w >> 1) + kTrThreads - 1) / kTrThreads, ((h >> 1) + tr_rows() - 1) / tr_rows());
  if (inverse) {
    if (kind == kHaar)
      dwt2d_inverse_kernel<kHaar, T, To><<<grid, kTrThreads, 0, s>>>(in, ip, out, op, h, w, tr_rows());
    else
      dwt2d_inverse_kernel<kDaub4, T, To><<<grid, kTrThreads, 0, s>>>(in, ip, out, op, h, w, tr_rows());
  } else {
    if (kind == kHaar)
      dwt2d_forward_kernel<kHaar, T, To><<<grid, kTrThreads, 0, s>>>(in, ip, out, op, h, w, tr_rows());
    else
      dwt2d_forward_kernel<kDaub4, T, To><<<grid, kTrThreads, 0, s>>>(in, ip, out, op, h, w, tr_rows());
  }
}

// ---- reference-exact fusion (fusion.py:148-150 step by step) ---------------

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
// The source coordinate of a destination index depends on that index alone,
// so a CTA covers kRsCols destination columns x kRsRows rows: each thread
// computes its column's (x0, x1, fx) once, the row coordinates are computed
// once per CTA into shared memory, and the scale in/out is one host-side
// IEEE division (numpy's `in_w / out_w`) instead of a float64 division per
// pixel. Same float64 operations in the same order as the reference.
constexpr int kRsCols = 128;
constexpr int kRsRows = 16;

__device__ __forceinline__ void src_coord(int dst, double scale, int in_n, int& i0, int& i1,
                                          double& f) {
  // np.clip((arange + 0.5) * (in/out) - 0.5, 0, in-1)
  double s = sub(mul((double)dst + 0.5, scale), 0.5);
  s = fmin(fmax(s, 0.0), (double)(in_n - 1));
  const double fl = floor(s);
  i0 = (int)fl;
  i1 = min(i0 + 1, in_n - 1);
  f = sub(s, fl);
}

template <typename T, typename To>
__global__ void __launch_bounds__(kRsCols)
    resample_kernel(const T* __restrict__ in, long long ip, int in_h, int in_w,
                    To* __restrict__ out, long long op, int out_h, int out_w, double sx,
                    double sy) {
  __shared__ int ry0[kRsRows], ry1[kRsRows];
  __shared__ double rfy[kRsRows];
  const int yb = blockIdx.y * kRsRows;
  if (threadIdx.x < kRsRows && yb + (int)threadIdx.x < out_h) {
    int a, b;
    double f;
    src_coord(yb + threadIdx.x, sy, in_h, a, b, f);
    ry0[threadIdx.x] = a;
    ry1[threadIdx.x] = b;
    rfy[threadIdx.x] = f;
  }
  __syncthreads();
  const int x = blockIdx.x * kRsCols + threadIdx.x;
  if (x >= out_w) return;
  int x0, x1;
  double fx;
  src_coord(x, sx, in_w, x0, x1, fx);
  const double gx = sub(1.0, fx);
  // row_u / row_l of fusion.py:79-80 depend only on (source row, x): the last
  // two source rows' horizontal interpolants are kept, so when upsampling each
  // source row is loaded, converted and interpolated once per column instead
  // of once per output row (the row sequence is uniform across the CTA, so
  // these branches never diverge)
  int ca = -1, cb = -1;
  double ha = 0.0, hb = 0.0;
  auto hrow = [&](int row) -> double {
    if (row == ca) return ha;
    if (row == cb) return hb;
    const T* p = in + (long long)row * ip;
    const double v = add(mul((double)__ldg(p + x0), gx), mul((double)__ldg(p + x1), fx));
    cb = ca;
    hb = ha;
    ca = row;
    ha = v;
    return v;
  };
  const int nr = min(kRsRows, out_h - yb);
  for (int r = 0; r < nr; ++r) {
    const double ru = hrow(ry0[r]);
    const double rl = hrow(ry1[r]);
    const double fy = rfy[r], gy = sub(1.0, fy);
    out[(long long)(yb + r) * op + x] = (To)add(mul(ru, gy), mul(rl, fy));
  }
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
  run_dwt2d<T, T>(kind, inverse, in, ip, out, op, h, w, s);
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
  dim3 grid((out_w + kRsCols - 1) / kRsCols, (out_h + kRsRows - 1) / kRsRows);
  resample_kernel<T, To><<<grid, kRsCols, 0, s>>>(in, ip, in_h, in_w, out, op, out_h, out_w,
                                                   (double)in_w / (double)out_w,
                                                   (double)in_h / (double)out_h);
  return cudaGetLastError();
}

cudaError_t launch_synth(float* out, long long pitch, int rows, int cols, unsigned long long seed,
                         unsigned plane, int row0, int col0, cudaStream_t s) {
  dim3 grid(((cols + 3) / 4 + 255) / 256, rows < 65535 ? rows : 65535);
  synth_kernel<<<grid, 256, 0, s>>>(out, pitch, rows, cols, seed, plane, row0, col0);
  return cudaGetLastError();
}

// ---- reference-exact Haar fusion in one pass --------------------------------
// Every Haar coefficient is 2x2-local, so fusion.py:148-150 for all bands runs
// in one kernel with no coefficient image: a thread owns PAN columns
// 4q..4q+3 of one row pair, forms that row pair's detail coefficients with
// the reference's float64 operations (wavelet.py:75-86 rows, then columns:
// LH = (a0 - a1) * 0.5, HL = (d0 + d1) * 0.5, HH = (d0 - d1) * 0.5), and per
// band sets LL = band (gain 1, fusion.py:125) and runs the inverse (columns:
// cvA = LL +/- LH, cvD = HL +/- HH; rows: out = cvA +/- cvD, wavelet.py:96-108)
// before one cast to the PAN dtype. Same operations, same order: bit-identical
// to the transform path.
struct ExactBands {
  const void* ms[kMaxBandsPerLaunch];
  void* out[kMaxBandsPerLaunch];
  // D4 halos (the RowSrc convention of fuse.cu): PAN logical rows -2, -1 at
  // pan_top and rows H, H+1 at pan_bot (halo_pitch apart), MS row -1 of each
  // band at ms_top. A whole plane aliases them to its own wrapped rows
  // (wavelet.py:83-84); a row strip (host pipeline, strips.py) passes its
  // neighbours' rows.
  const void* pan_top;
  const void* pan_bot;
  long long halo_pitch;
  const void* ms_top[kMaxBandsPerLaunch];
};

template <typename T, int NB, bool kVec>
__global__ void __launch_bounds__(128)
    fuse_exact_haar_kernel(const T* __restrict__ pan, long long pp, const ExactBands bands,
                           long long mp, long long op, int H, int W) {
  const int q = blockIdx.x * 128 + threadIdx.x;
  const int i = blockIdx.y;  // coefficient row = PAN row pair
  const int c4 = 4 * q;
  if (c4 >= W) return;
  const int ncol = min(4, W - c4);  // 2 or 4 (W even)
  const T* r0 = pan + (long long)(2 * i) * pp + c4;
  const T* r1 = r0 + pp;
  double x[2][4];
  if (kVec && sizeof(T) == 8 && ((reinterpret_cast<uintptr_t>(r0) | pp * 8) & 31) == 0) {
    load4_wide(reinterpret_cast<const double*>(r0), x[0]);
    load4_wide(reinterpret_cast<const double*>(r1), x[1]);
  } else if (kVec) {
    double v[4];
    load4_vec<double>(r0, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) x[0][k] = v[k];
    load4_vec<double>(r1, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) x[1][k] = v[k];
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[0][k] = k < ncol ? (double)__ldg(r0 + k) : 0.0;
      x[1][k] = k < ncol ? (double)__ldg(r1 + k) : 0.0;
    }
  }
  double lh[2], cvd[2][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    double a[2], d[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      a[r] = fwd_lo(kHaar, D4{}, x[r][2 * c], x[r][2 * c + 1], 0.0, 0.0);
      d[r] = fwd_hi(kHaar, D4{}, x[r][2 * c], x[r][2 * c + 1], 0.0, 0.0);
    }
    lh[c] = fwd_hi(kHaar, D4{}, a[0], a[1], 0.0, 0.0);
    const double hl = fwd_lo(kHaar, D4{}, d[0], d[1], 0.0, 0.0);
    const double hh = fwd_hi(kHaar, D4{}, d[0], d[1], 0.0, 0.0);
    cvd[0][c] = add(hl, hh);
    cvd[1][c] = sub(hl, hh);
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const T* m = static_cast<const T*>(bands.ms[b]) + (long long)i * mp + 2 * q;
    double ll[2];
    ll[0] = (double)__ldg(m);
    ll[1] = ncol > 2 ? (double)__ldg(m + 1) : 0.0;
    double o[2][4];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const double cva = p == 0 ? add(ll[c], lh[c]) : sub(ll[c], lh[c]);
        o[p][2 * c] = add(cva, cvd[p][c]);
        o[p][2 * c + 1] = sub(cva, cvd[p][c]);
      }
    T* w0 = static_cast<T*>(bands.out[b]) + (long long)(2 * i) * op + c4;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      T* w = w0 + (p ? op : 0);
      if (kVec && sizeof(T) == 8 && ((reinterpret_cast<uintptr_t>(w) | op * 8) & 31) == 0) {
        store4_wide(reinterpret_cast<double*>(w), o[p]);
      } else if (kVec) {
        store4_vec<double>(w, o[p]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < ncol) w[k] = (T)o[p][k];
      }
    }
  }
}

template <typename T, int NB>
static void launch_exact_haar_nb(const T* pan, long long pp, const ExactBands& eb, long long mp,
                                 long long op, int h, int w, bool vec, cudaStream_t s) {
  dim3 grid(((w + 3) / 4 + 127) / 128, h >> 1);
  if (vec)
    fuse_exact_haar_kernel<T, NB, true><<<grid, 128, 0, s>>>(pan, pp, eb, mp, op, h, w);
  else
    fuse_exact_haar_kernel<T, NB, false><<<grid, 128, 0, s>>>(pan, pp, eb, mp, op, h, w);
}

template <typename T>
static cudaError_t launch_exact_haar(const T* pan, long long pp, const T* const* ms, long long mp,
                                     T* const* out, long long op, int nbands, int h, int w,
                                     cudaStream_t s) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  for (int b0 = 0; b0 < nbands; b0 += kMaxBandsPerLaunch) {
    const int nb = min(kMaxBandsPerLaunch, nbands - b0);
    ExactBands eb{};
    bool vec = w % 4 == 0 && al16(pan) && (pp * (long long)sizeof(T)) % 16 == 0 &&
               (op * (long long)sizeof(T)) % 16 == 0;
    for (int b = 0; b < nb; ++b) {
      eb.ms[b] = ms[b0 + b];
      eb.out[b] = out[b0 + b];
      vec = vec && al16(out[b0 + b]);
    }
    switch (nb) {
#define WF_EH(N) \
  case N: launch_exact_haar_nb<T, N>(pan, pp, eb, mp, op, h, w, vec, s); break;
      WF_EH(1) WF_EH(2) WF_EH(3) WF_EH(4) WF_EH(5) WF_EH(6) WF_EH(7) WF_EH(8)
#undef WF_EH
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaGetLastError();
}

// ---- reference-exact D4 fusion in one pass ----------------------------------
// fusion.py:148-150 for all bands with no coefficient image. A thread owns
// coefficient column j (output columns 2j, 2j+1) and marches down a run of
// coefficient rows i. Output rows 2i, 2i+1 need, at coefficient columns
// jm = j-1 and j (wrapped) and rows i-1 and i, the detail coefficients LH,
// HL, HH of the PAN and LL = band * 2 (fusion.py:125,149). The forward pass is
// the reference's own (wavelet.py:75-86: rows of PAN rows 2i+2, 2i+3, then
// columns), carried down the run; the inverse (wavelet.py:96-108) is split
// into the products that only involve PAN coefficients -- formed once per row
// step -- and the band terms, added in the reference's order per band:
//   cvA = ((hp2*LL(i-1) + gp2*LH(i-1)) + hp0*LL(i)) + gp0*LH(i)
//   cvD = ((hp2*HL(i-1) + gp2*HH(i-1)) + hp0*HL(i)) + gp0*HH(i)
//   out(2i+p, 2j+e) = ((he2*cvA(jm) + ge2*cvD(jm)) + he0*cvA(j)) + ge0*cvD(j)
// with every product and sum rounded separately (no FMA), one final cast:
// bit-identical to the transform path.
constexpr int kExactRows = 16;
#ifndef WF_EX_PF  // L1 prefetch distance in row steps: 1 (1.52 ms); 2 -> 1.57, 3 -> 1.66, 4 -> 1.75 (r02_exact_loads_ab.log)
#define WF_EX_PF 1
#endif

// Column sharing: a CTA of 128 threads covers 127 output coefficient columns
// [127k, 127k + 127); thread t computes column j = 127k - 1 + t, so thread 0's
// column is the left halo of the CTA (computed, not written). Phase 1 forms
// everything that depends on one coefficient column -- its forward
// coefficients, cvD and, per band, cvA -- and publishes it in shared memory;
// after a barrier, phase 2 combines columns j-1 and j into output columns 2j,
// 2j+1. Every quantity is computed once (the per-thread form computed column
// j-1 again), in the same operations and order.
constexpr int kExCols = 127;

#ifndef WF_EX_MINB  // CTAs/SM bound: 0 (80 regs, 1.52 ms); 7 -> 72 regs + spills 1.67, 8 -> 1.68
#define WF_EX_MINB 0
#endif
template <typename T, int NB, bool kVec>
__global__ void __launch_bounds__(128, WF_EX_MINB)
    fuse_exact_d4_kernel(const T* __restrict__ pan, long long pp, const ExactBands bands,
                         long long mp, long long op, int H, int W, int rows) {
  // [buffer][quantity][thread]: quantities cvD[0], cvD[1], cvA[b][0], cvA[b][1]
  constexpr int NQ = 2 + 2 * NB;
  __shared__ double xs[2][NQ][128];
  const int tid = threadIdx.x;
  const int Hh = H >> 1, Wh = W >> 1;
  const int jraw = blockIdx.x * kExCols - 1 + tid;  // -1 .. : thread 0 = halo
  const int j = wrap(jraw, Wh);
  const bool emit = tid > 0 && jraw < Wh;
  const int i0 = blockIdx.y * rows;
  const int i1 = min(i0 + rows, Hh);
  const D4 t = d4_taps();
  const int c0 = 2 * j, c1 = 2 * j + 1, c2 = wrap(2 * j + 2, W), c3 = wrap(2 * j + 3, W);
  // PAN logical row r (-2 .. H+1) through the halo sources
  auto pan_row = [&](int r) -> const T* {
    if (r < 0) return static_cast<const T*>(bands.pan_top) + (long long)(r + 2) * bands.halo_pitch;
    if (r >= H) return static_cast<const T*>(bands.pan_bot) + (long long)(r - H) * bands.halo_pitch;
    return pan + (long long)r * pp;
  };
  auto rowpass = [&](int r, double& a, double& d) {
    const T* row = pan_row(r);
    const double x0 = (double)__ldg(row + c0), x1 = (double)__ldg(row + c1);
    const double x2 = (double)__ldg(row + c2), x3 = (double)__ldg(row + c3);
    a = fwd_lo(kDaub4, t, x0, x1, x2, x3);
    d = fwd_hi(kDaub4, t, x0, x1, x2, x3);
  };
  const double sh2[2] = {t.h2, t.h3}, sg2[2] = {t.g2, t.g3};
  const double sh0[2] = {t.h0, t.h1}, sg0[2] = {t.g0, t.g1};
  auto prefetch = [](const void* ptr) { asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr)); };

  double a[4], d[4];              // row passes of PAN rows 2i .. 2i+3 at column j
  double lhp, hlp, hhp;           // detail coefficients of row i-1 at column j
  {
    rowpass(2 * i0 - 2, a[0], d[0]);  // coefficient row i0 - 1 (the top halo when i0 = 0)
    rowpass(2 * i0 - 1, a[1], d[1]);
    rowpass(2 * i0, a[2], d[2]);
    rowpass(2 * i0 + 1, a[3], d[3]);
    lhp = fwd_hi(kDaub4, t, a[0], a[1], a[2], a[3]);
    hlp = fwd_lo(kDaub4, t, d[0], d[1], d[2], d[3]);
    hhp = fwd_hi(kDaub4, t, d[0], d[1], d[2], d[3]);
    a[0] = a[2];
    a[1] = a[3];
    d[0] = d[2];
    d[1] = d[3];
  }
  int buf = 0;
  for (int i = i0; i < i1; ++i, buf ^= 1) {
    if (i + WF_EX_PF < i1) {  // the PAN and MS lines of step i + WF_EX_PF into L1
#pragma unroll
      for (int r = 2 + 2 * WF_EX_PF; r < 4 + 2 * WF_EX_PF; ++r) {
        const T* row = pan_row(2 * i + r);
        prefetch(row + c0);
        prefetch(row + c3);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b)
        prefetch(static_cast<const T*>(bands.ms[b]) + (long long)(i + WF_EX_PF) * mp + j);
    }
    // ---- phase 1: column j ----
    rowpass(2 * i + 2, a[2], d[2]);
    rowpass(2 * i + 3, a[3], d[3]);
    const double lh = fwd_hi(kDaub4, t, a[0], a[1], a[2], a[3]);
    const double hl = fwd_lo(kDaub4, t, d[0], d[1], d[2], d[3]);
    const double hh = fwd_hi(kDaub4, t, d[0], d[1], d[2], d[3]);
    double cvd[2], qa0[2], qa1[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      cvd[p] = add(add(add(mul(sh2[p], hlp), mul(sg2[p], hhp)), mul(sh0[p], hl)), mul(sg0[p], hh));
      qa0[p] = mul(sg2[p], lhp);
      qa1[p] = mul(sg0[p], lh);
      xs[buf][p][tid] = cvd[p];
    }
    double cva[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const T* mb = static_cast<const T*>(bands.ms[b]);
      const T* mprev = i > 0 ? mb + (long long)(i - 1) * mp : static_cast<const T*>(bands.ms_top[b]);
      const double llp = mul((double)__ldg(mprev + j), 2.0);
      const double llc = mul((double)__ldg(mb + (long long)i * mp + j), 2.0);
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        cva[b][p] = add(add(add(mul(sh2[p], llp), qa0[p]), mul(sh0[p], llc)), qa1[p]);
        xs[buf][2 + 2 * b + p][tid] = cva[b][p];
      }
    }
    __syncthreads();
    // ---- phase 2: output columns 2j, 2j+1 from columns j-1 and j ----
    if (emit) {
      double qd[2][4];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const double cvdm = xs[buf][p][tid - 1];
        qd[p][0] = mul(sg2[0], cvdm);
        qd[p][1] = mul(sg0[0], cvd[p]);
        qd[p][2] = mul(sg2[1], cvdm);
        qd[p][3] = mul(sg0[1], cvd[p]);
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        T* ob = static_cast<T*>(bands.out[b]);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const double cvam = xs[buf][2 + 2 * b + p][tid - 1];
          const double o0 = add(add(add(mul(sh2[0], cvam), qd[p][0]), mul(sh0[0], cva[b][p])),
                                qd[p][1]);
          const double o1 = add(add(add(mul(sh2[1], cvam), qd[p][2]), mul(sh0[1], cva[b][p])),
                                qd[p][3]);
          T* w = ob + (long long)(2 * i + p) * op + 2 * j;
          if (kVec) {
            if constexpr (sizeof(T) == 4)
              *reinterpret_cast<float2*>(w) = make_float2((float)o0, (float)o1);
            else
              *reinterpret_cast<double2*>(w) = make_double2(o0, o1);
          } else {
            w[0] = (T)o0;
            w[1] = (T)o1;
          }
        }
      }
    }
    // (xs is double-buffered: the next step writes the other buffer, and the
    // barrier of that step orders this step's reads before it is reused)
    a[0] = a[2];
    a[1] = a[3];
    d[0] = d[2];
    d[1] = d[3];
    lhp = lh;
    hlp = hl;
    hhp = hh;
  }
}

template <typename T>
static cudaError_t launch_exact_d4(const T* pan, long long pp, const T* pan_top, const T* pan_bot,
                                  long long hp, const T* const* ms, const T* const* ms_top,
                                  long long mp, T* const* out, long long op, int nbands, int h,
                                  int w, cudaStream_t s) {
  int rows = kExactRows;
  if (env_tuning().exact_rows > 0) rows = env_tuning().exact_rows;
  dim3 grid(((w >> 1) + kExCols - 1) / kExCols, ((h >> 1) + rows - 1) / rows);
  for (int b0 = 0; b0 < nbands; b0 += kMaxBandsPerLaunch) {
    const int nb = min(kMaxBandsPerLaunch, nbands - b0);
    ExactBands eb{};
    eb.pan_top = pan_top;
    eb.pan_bot = pan_bot;
    eb.halo_pitch = hp;
    for (int b = 0; b < nb; ++b) {
      eb.ms[b] = ms[b0 + b];
      eb.out[b] = out[b0 + b];
      eb.ms_top[b] = ms_top[b0 + b];
    }
    bool vec = op % 2 == 0;
    for (int b = 0; b < nb; ++b)
      vec = vec && (reinterpret_cast<uintptr_t>(out[b0 + b]) % (2 * sizeof(T))) == 0;
    switch (nb) {
#define WF_ED(N)                                                                          \
  case N:                                                                                 \
    if (vec)                                                                              \
      fuse_exact_d4_kernel<T, N, true><<<grid, 128, 0, s>>>(pan, pp, eb, mp, op, h, w, rows); \
    else                                                                                  \
      fuse_exact_d4_kernel<T, N, false><<<grid, 128, 0, s>>>(pan, pp, eb, mp, op, h, w, rows); \
    break;
      WF_ED(1) WF_ED(2) WF_ED(3) WF_ED(4) WF_ED(5) WF_ED(6) WF_ED(7) WF_ED(8)
#undef WF_ED
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaGetLastError();
}

// Row strips (host pipeline, strips.py): the one-pass exact kernels with the
// neighbours' halo rows (D4; Haar needs none). pan_top == nullptr: a whole
// plane, whose halos are its own wrapped rows.
template <typename T>
cudaError_t launch_fuse_exact_strip(int kind, const T* pan, long long pp, const T* pan_top,
                                    const T* pan_bot, long long hp, const T* const* ms,
                                    const T* const* ms_top, long long mp, T* const* out,
                                    long long op, int nbands, int rows, int w, cudaStream_t s) {
  if (kind == kHaar) return launch_exact_haar<T>(pan, pp, ms, mp, out, op, nbands, rows, w, s);
  if (pan_top) return launch_exact_d4<T>(pan, pp, pan_top, pan_bot, hp, ms, ms_top, mp, out, op,
                                         nbands, rows, w, s);
  for (int b0 = 0; b0 < nbands; b0 += kMaxBandsPerLaunch) {
    const int nb = min(kMaxBandsPerLaunch, nbands - b0);
    const T* mst[kMaxBandsPerLaunch];
    for (int b = 0; b < nb; ++b) mst[b] = ms[b0 + b] + (long long)(rows / 2 - 1) * mp;
    const cudaError_t e = launch_exact_d4<T>(pan, pp, pan + (long long)(rows - 2) * pp, pan, pp,
                                             ms + b0, mst, mp, out + b0, op, nb, rows, w, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
template cudaError_t launch_fuse_exact_strip<float>(int, const float*, long long, const float*,
                                                    const float*, long long, const float* const*,
                                                    const float* const*, long long,
                                                    float* const*, long long, int, int, int,
                                                    cudaStream_t);
template cudaError_t launch_fuse_exact_strip<double>(int, const double*, long long, const double*,
                                                     const double*, long long,
                                                     const double* const*, const double* const*,
                                                     long long, double* const*, long long, int,
                                                     int, int, cudaStream_t);

template <typename T>
cudaError_t launch_fuse_bands_exact(int kind, const T* pan, long long pp, const T* const* ms,
                                    long long mp, T* const* out, long long op, int nbands,
                                    int h, int w, double* ws, cudaStream_t s);

// fuse_dwt exactly as the reference computes it: float64 forward transform
// of the PAN plane (its exact operation order), LL <- band * gain, float64
// inverse, one final cast to the PAN dtype. `ws` = h * w doubles.
template <typename T>
cudaError_t launch_fuse_exact(int kind, const T* pan, long long pp, const T* ms, long long mp,
                              T* out, long long op, int h, int w, double* ws, cudaStream_t s) {
  return launch_fuse_bands_exact<T>(kind, pan, pp, &ms, mp, &out, op, 1, h, w, ws, s);
}
// fuse() in the exact sequence for all bands: forward once, then per band
// LL <- band * gain and the inverse (the detail quadrants of ws stay as the
// forward pass left them; LL is fully overwritten per band).
template <typename T>
cudaError_t launch_fuse_bands_exact(int kind, const T* pan, long long pp, const T* const* ms,
                                    long long mp, T* const* out, long long op, int nbands,
                                    int h, int w, double* ws, cudaStream_t s) {
  if (!env_tuning().exact_transforms)  // one pass, no coefficient image
    return launch_fuse_exact_strip<T>(kind, pan, pp, nullptr, nullptr, 0, ms, nullptr, mp, out,
                                      op, nbands, h, w, s);
  run_dwt2d<T, double>(kind, false, pan, pp, ws, w, h, w, s);
  dim3 grid(((w >> 1) + kTrThreads - 1) / kTrThreads, ((h >> 1) + tr_rows() - 1) / tr_rows());
  for (int b = 0; b < nbands; ++b) {
    if (kind == kHaar)
      dwt2d_inverse_kernel<kHaar, double, T, true, T>
          <<<grid, kTrThreads, 0, s>>>(ws, w, out[b], op, h, w, tr_rows(), ms[b], mp, 1.0);
    else
      dwt2d_inverse_kernel<kDaub4, double, T, true, T>
          <<<grid, kTrThreads, 0, s>>>(ws, w, out[b], op, h, w, tr_rows(), ms[b], mp, 2.0);
  }
  return cudaGetLastError();
}
template cudaError_t launch_fuse_bands_exact<float>(int, const float*, long long,
                                                    const float* const*, long long, float* const*,
                                                    long long, int, int, int, double*,
                                                    cudaStream_t);
template cudaError_t launch_fuse_bands_exact<double>(int, const double*, long long,
                                                     const double* const*, long long,
                                                     double* const*, long long, int, int, int,
                                                     double*, cudaStream_t);

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
