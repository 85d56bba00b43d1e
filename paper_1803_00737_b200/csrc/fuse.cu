// wavefuse-b200: fused DWT coefficient-replacement kernels (sm_100a).
//
// Reference path: fuse_dwt (/root/reference/pkg/src/wavefuse/fusion.py:128-150)
// = dwt2d_forward(pan) -> LL <- band * gain (gain 1 Haar / 2 D4, fusion.py:125)
// -> dwt2d_inverse, called once per band by fuse (fusion.py:182).
//
// Neither kernel materialises the coefficient image. By linearity and perfect
// reconstruction of the single-level transform (wavelet.py:73-109):
//
//   Haar:  out = pan + (ms - mean2x2(pan))          (2x2-local, no halo)
//   D4:    out = pan + S_LL(2*ms - LL(pan))
//          LL(i,j)  = sum_{k,l} h_k h_l pan(2i+k, 2j+l)              (wrap)
//          S_LL: row 2i   <- h2*E(i-1) + h0*E(i)
//                row 2i+1 <- h3*E(i-1) + h1*E(i)       (same along columns)
//
// so the detail coefficients pass through untouched and never need computing.
// Both kernels read PAN once for up to kMaxBands bands (the reference recomputes
// the PAN transform per band, fusion.py:182), so per scene the HBM traffic is
// (4 + 5*B) bytes per PAN pixel for f32 I/O.
//
// D4 geometry (per warp): a warp owns a column band of 128 PAN columns (4 per
// lane, one LDG.128 per row) and marches down a run of row pairs. Each step
// loads PAN rows 2i+2, 2i+3 and MS row i of every band, and writes output rows
// 2i, 2i+1 of every band. The horizontal look-ahead (PAN cols c+4, c+5) comes
// from the next lane by __shfl_down; the look-behind E(j-1) by __shfl_up. Lane
// 31 / lane 0 fetch the 2-column halos of the band. Rows are addressed through
// a halo-aware row source, so the same kernel serves whole images (halos alias
// the wrapped rows of the image itself) and row strips whose halo rows arrived
// from neighbouring GPUs (strips.py).
#include <stdlib.h>

#include <type_traits>

#include "wf_common.cuh"
#include "wf_kernels.h"

namespace wf {

constexpr int kD4Threads = 256;  // 8 warps per CTA
constexpr int kColsPerWarp = 128;

// The library is compiled with -fmad=false: every fused multiply-add below is
// an explicit fma(), so the single-band and multi-band instantiations round
// identically (fuse() must equal per-band fuse_dwt() bit for bit,
// test_fusion.py:168-187 of the reference).
template <typename Acc>
__device__ __forceinline__ Acc dot4(Acc h0, Acc h1, Acc h2, Acc h3, Acc x0, Acc x1, Acc x2,
                                    Acc x3) {
  return fma(h3, x3, fma(h2, x2, fma(h1, x1, h0 * x0)));
}

template <typename T>
struct RowSrc {
  const T* main;
  const T* top;  // logical rows -2, -1
  const T* bot;  // logical rows rows, rows+1
  long long pitch, halo_pitch;
  int rows;
  __device__ __forceinline__ const T* row(int r) const {
    if (r < 0) return top + (long long)(r + 2) * halo_pitch;
    if (r >= rows) return bot + (long long)(r - rows) * halo_pitch;
    return main + (long long)r * pitch;
  }
};

// ---------------------------------------------------------------------------
// D4 warp-marching kernel
// ---------------------------------------------------------------------------
template <typename T, typename Acc>
struct D4Lane {
  int lane, base, c, W, Wh;
  bool vec;

  // PAN row: 4 own columns, lane 31 also (base+128, base+129), lane 0 also
  // (base-2, base-1). All lanes load wrapped addresses, so lanes past the
  // right edge still supply correctly wrapped look-ahead columns to the last
  // valid lane through the shuffle.
  __device__ __forceinline__ void load_pan(const T* row, Acc (&p)[4], Acc (&xl)[2],
                                           Acc (&xr)[2]) const {
    if (vec) {
      load4_vec<Acc>(row + c, p);
      if (lane == 31) load2_vec<Acc>(row + base + kColsPerWarp, xr);
      if (lane == 0) load2_vec<Acc>(row + base - 2, xl);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) p[k] = (Acc)__ldg(row + wrap(c + k, W));
      if (lane == 31) {
        xr[0] = (Acc)__ldg(row + wrap(base + kColsPerWarp, W));
        xr[1] = (Acc)__ldg(row + wrap(base + kColsPerWarp + 1, W));
      }
      if (lane == 0) {
        xl[0] = (Acc)__ldg(row + wrap(base - 2, W));
        xl[1] = (Acc)__ldg(row + wrap(base - 1, W));
      }
    }
  }

  // MS row i of one band: half-columns j = c/2, j+1; lane 0 also j0-1.
  __device__ __forceinline__ void load_ms(const T* row, Acc (&m)[2], Acc& mm) const {
    const int j = c >> 1;
    if (vec) {
      load2_vec<Acc>(row + j, m);
      if (lane == 0) mm = (Acc)__ldg(row + (base >> 1) - 1);
    } else {
      m[0] = (Acc)__ldg(row + wrap(j, Wh));
      m[1] = (Acc)__ldg(row + wrap(j + 1, Wh));
      if (lane == 0) mm = (Acc)__ldg(row + wrap((base >> 1) - 1, Wh));
    }
  }

  // Row low-pass R(r, j) = sum_l h_l pan(r, 2j+l) for j, j+1 and (lane 0) j0-1.
  __device__ __forceinline__ void rowpass(const Acc (&p)[4], const Acc (&xl)[2],
                                          const Acc (&xr)[2], Acc h0, Acc h1, Acc h2,
                                          Acc h3, Acc (&r)[2], Acc& rl) const {
    Acc nx = __shfl_down_sync(0xffffffffu, p[0], 1);
    Acc ny = __shfl_down_sync(0xffffffffu, p[1], 1);
    if (lane == 31) {
      nx = xr[0];
      ny = xr[1];
    }
    r[0] = dot4(h0, h1, h2, h3, p[0], p[1], p[2], p[3]);
    r[1] = dot4(h0, h1, h2, h3, p[2], p[3], nx, ny);
    rl = dot4(h0, h1, h2, h3, xl[0], xl[1], p[0], p[1]);
  }

  __device__ __forceinline__ void store_row(T* row, const Acc (&o)[4]) const {
    if (vec) {
      store4_vec<Acc>(row + c, o);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (c + k < W) row[c + k] = (T)o[k];
    }
  }
};

template <typename T, typename Acc, int NB, bool kVec>
__global__ void __launch_bounds__(kD4Threads)
    fuse_d4_kernel(const FuseArgs<T> a) {
  const long long gw = (long long)blockIdx.x * (kD4Threads / 32) + (threadIdx.x >> 5);
  if (gw >= a.n_tasks) return;  // warp-uniform exit
  const int cb = (int)(gw % a.n_colbands);
  const int rt = (int)(gw / a.n_colbands);
  const int npairs = a.rows >> 1;
  const int i0 = rt * a.pairs_per_task;
  const int i1 = min(i0 + a.pairs_per_task, npairs);

  D4Lane<T, Acc> L;
  L.lane = threadIdx.x & 31;
  L.W = a.W;
  L.Wh = a.W >> 1;
  L.base = cb * kColsPerWarp;
  L.c = L.base + 4 * L.lane;
  L.vec = kVec && L.base >= 2 && L.base + kColsPerWarp + 2 <= a.W;

  const D4 t = d4_taps();
  const Acc h0 = (Acc)t.h0, h1 = (Acc)t.h1, h2 = (Acc)t.h2, h3 = (Acc)t.h3;

  RowSrc<T> pan{a.pan, a.pan_top, a.pan_bot, a.pan_pitch, a.halo_pitch, a.rows};

  // ---- prologue: rows 2i0-2 .. 2i0+1, E(i0-1) per band -------------------
  Acc pa[2][4], ra[2][2], rla[2];
  Acc ll_prev[3];
  {
    Acc p[4], xl[2] = {0, 0}, xr[2] = {0, 0};
    Acc rq[4][2], rlq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      L.load_pan(pan.row(2 * i0 - 2 + q), p, xl, xr);
      L.rowpass(p, xl, xr, h0, h1, h2, h3, rq[q], rlq[q]);
      if (q >= 2) {
#pragma unroll
        for (int k = 0; k < 4; ++k) pa[q - 2][k] = p[k];
        ra[q - 2][0] = rq[q][0];
        ra[q - 2][1] = rq[q][1];
        rla[q - 2] = rlq[q];
      }
    }
    ll_prev[0] = dot4(h0, h1, h2, h3, rq[0][0], rq[1][0], rq[2][0], rq[3][0]);
    ll_prev[1] = dot4(h0, h1, h2, h3, rq[0][1], rq[1][1], rq[2][1], rq[3][1]);
    ll_prev[2] = dot4(h0, h1, h2, h3, rlq[0], rlq[1], rlq[2], rlq[3]);
  }
  Acc ep[NB][3];  // E(i-1, j), E(i-1, j+1), E(i-1, j0-1)
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const T* mrow = (i0 == 0) ? a.ms_top[b] : a.ms[b] + (long long)(i0 - 1) * a.ms_pitch;
    Acc m[2], mm = 0;
    L.load_ms(mrow, m, mm);
    ep[b][0] = m[0] + m[0] - ll_prev[0];
    ep[b][1] = m[1] + m[1] - ll_prev[1];
    ep[b][2] = mm + mm - ll_prev[2];
  }

  // ---- march -------------------------------------------------------------
  for (int i = i0; i < i1; ++i) {
    // issue every load of the step before any arithmetic: 2 PAN rows + one
    // MS row per band are in flight together
    Acc pn[2][4], rn[2][2], rln[2];
    Acc xl[2][2] = {{0, 0}, {0, 0}}, xr[2][2] = {{0, 0}, {0, 0}};
    L.load_pan(pan.row(2 * i + 2), pn[0], xl[0], xr[0]);
    L.load_pan(pan.row(2 * i + 3), pn[1], xl[1], xr[1]);
    Acc ms_cur[NB][2], ms_lo[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      ms_lo[b] = 0;
      L.load_ms(a.ms[b] + (long long)i * a.ms_pitch, ms_cur[b], ms_lo[b]);
    }
    L.rowpass(pn[0], xl[0], xr[0], h0, h1, h2, h3, rn[0], rln[0]);
    L.rowpass(pn[1], xl[1], xr[1], h0, h1, h2, h3, rn[1], rln[1]);
    Acc ll[3];
    ll[0] = dot4(h0, h1, h2, h3, ra[0][0], ra[1][0], rn[0][0], rn[1][0]);
    ll[1] = dot4(h0, h1, h2, h3, ra[0][1], ra[1][1], rn[0][1], rn[1][1]);
    ll[2] = dot4(h0, h1, h2, h3, rla[0], rla[1], rln[0], rln[1]);

#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const Acc(&m)[2] = ms_cur[b];
      const Acc mm = ms_lo[b];
      const Acc e0 = m[0] + m[0] - ll[0];
      const Acc e1 = m[1] + m[1] - ll[1];
      const Acc em = mm + mm - ll[2];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        // vertical synthesis weights for output row 2i+p: (prev, cur)
        const Acc wp = p == 0 ? h2 : h3;
        const Acc wc = p == 0 ? h0 : h1;
        const Acc v0 = fma(wc, e0, wp * ep[b][0]);
        const Acc v1 = fma(wc, e1, wp * ep[b][1]);
        const Acc vmo = fma(wc, em, wp * ep[b][2]);
        Acc vm = __shfl_up_sync(0xffffffffu, v1, 1);
        if (L.lane == 0) vm = vmo;
        Acc o[4];
        o[0] = pa[p][0] + fma(h0, v0, h2 * vm);
        o[1] = pa[p][1] + fma(h1, v0, h3 * vm);
        o[2] = pa[p][2] + fma(h0, v1, h2 * v0);
        o[3] = pa[p][3] + fma(h1, v1, h3 * v0);
        L.store_row(a.out[b] + (long long)(2 * i + p) * a.out_pitch, o);
      }
      ep[b][0] = e0;
      ep[b][1] = e1;
      ep[b][2] = em;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) pa[q][k] = pn[q][k];
      ra[q][0] = rn[q][0];
      ra[q][1] = rn[q][1];
      rla[q] = rln[q];
    }
  }
}

// ---------------------------------------------------------------------------
// Haar kernel: out = pan + (ms - mean2x2(pan)); 2x2-local, no halo, so strips
// and tiles at even offsets are exact with no exchange at all.
// A thread owns a quad of PAN columns (4 px = 2 half-columns) in a run of row
// pairs; PAN rows 2i, 2i+1 are loaded once and every band streams past them.
// ---------------------------------------------------------------------------
constexpr int kHaarThreads = 128;
// one row pair per thread measured best (tools/sweep_haar.py: 6.56 TB/s at
// B = 6 vs 6.28 at 4 pairs) -- more, shorter-lived warps keep more loads in flight
constexpr int kHaarPairsPerThread = 1;
constexpr int kHaarU8PairsPerThread = 1;  // WF_HAAR_U8_PPT sweep: 1 -> 0.296 ms, 4 -> 0.317, 8 -> 0.330

template <typename T, typename Acc, int NB, bool kVec, int PPT>
__global__ void __launch_bounds__(kHaarThreads)
    fuse_haar_kernel(const FuseArgs<T> a) {
  const int q = blockIdx.x * kHaarThreads + threadIdx.x;  // quad index
  const int W = a.W;
  const int c = 4 * q;
  if (c >= W) return;
  const int npairs = a.rows >> 1;
  const int i_begin = blockIdx.y * PPT;
  const bool full = kVec;  // W % 4 == 0 and pointers aligned (host-checked)
  const Acc quarter = Acc(0.25);

#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int i = i_begin + s;
    if (i >= npairs) break;
    const T* r0 = a.pan + (long long)(2 * i) * a.pan_pitch;
    const T* r1 = r0 + a.pan_pitch;
    Acc p0[4], p1[4];
    if constexpr (sizeof(T) == 8 && kVec) {
      if (a.wide) {
        load4_wide(r0 + c, p0);
        load4_wide(r1 + c, p1);
      } else {
        load4_vec<Acc>(r0 + c, p0);
        load4_vec<Acc>(r1 + c, p1);
      }
    } else if (full) {
      load4_vec<Acc>(r0 + c, p0);
      load4_vec<Acc>(r1 + c, p1);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool ok = c + k < W;
        p0[k] = ok ? (Acc)__ldg(r0 + c + k) : Acc(0);
        p1[k] = ok ? (Acc)__ldg(r1 + c + k) : Acc(0);
      }
    }
    const Acc ll0 = ((p0[0] + p0[1]) + (p1[0] + p1[1])) * quarter;
    const Acc ll1 = ((p0[2] + p0[3]) + (p1[2] + p1[3])) * quarter;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const T* mrow = a.ms[b] + (long long)i * a.ms_pitch;
      Acc m[2];
      if (full) {
        load2_vec<Acc>(mrow + 2 * q, m);
      } else {
        m[0] = (Acc)__ldg(mrow + 2 * q);
        m[1] = (c + 2 < W) ? (Acc)__ldg(mrow + 2 * q + 1) : Acc(0);
      }
      const Acc d0 = m[0] - ll0, d1 = m[1] - ll1;
      Acc o0[4] = {p0[0] + d0, p0[1] + d0, p0[2] + d1, p0[3] + d1};
      Acc o1[4] = {p1[0] + d0, p1[1] + d0, p1[2] + d1, p1[3] + d1};
      T* w0 = a.out[b] + (long long)(2 * i) * a.out_pitch;
      T* w1 = w0 + a.out_pitch;
      if constexpr (sizeof(T) == 8 && kVec) {
        if (a.wide) {
          store4_wide(w0 + c, o0);
          store4_wide(w1 + c, o1);
        } else {
          store4_vec<Acc>(w0 + c, o0);
          store4_vec<Acc>(w1 + c, o1);
        }
      } else if (full) {
        store4_vec<Acc>(w0 + c, o0);
        store4_vec<Acc>(w1 + c, o1);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c + k < W) {
            w0[c + k] = (T)o0[k];
            w1[c + k] = (T)o1[k];
          }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Host-side launchers
// ---------------------------------------------------------------------------
// The Haar grids map row pairs to gridDim.y (at most 65535): taller planes
// (H >= 131072 at one pair per thread) are launched in row chunks. Haar is
// 2x2-local, so a chunk is an independent sub-plane at an even row offset.
template <typename T, typename F>
static cudaError_t haar_row_chunks(const FuseArgs<T>& a, int pairs_per_y, F&& launch) {
  const long long npairs = a.rows >> 1;
  const long long chunk = 65535LL * pairs_per_y;
  for (long long p0 = 0; p0 < npairs; p0 += chunk) {
    FuseArgs<T> c = a;
    const long long n = npairs - p0 < chunk ? npairs - p0 : chunk;
    c.pan = a.pan + 2 * p0 * a.pan_pitch;
    for (int b = 0; b < a.nbands; ++b) {
      c.ms[b] = a.ms[b] + p0 * a.ms_pitch;
      c.out[b] = a.out[b] + 2 * p0 * a.out_pitch;
    }
    c.rows = (int)(2 * n);
    launch(c);
    if (cudaError_t e = cudaGetLastError()) return e;
  }
  return cudaSuccess;
}

template <typename T, typename Acc, int NB>
static cudaError_t launch_nb(int kind, const FuseArgs<T>& a0, bool vec, cudaStream_t s,
                             const LaunchTuning& tune) {
  FuseArgs<T> a = a0;
  const int npairs = a.rows >> 1;
  if (kind == kHaar) {
    const int nq = (a.W + 3) / 4;
    int ppt = tune.haar_ppt > 0 ? tune.haar_ppt : kHaarPairsPerThread;
    if (ppt != 1 && ppt != 2 && ppt != 8) ppt = 4;
    return haar_row_chunks(a, ppt, [&](const FuseArgs<T>& c) {
      dim3 grid((nq + kHaarThreads - 1) / kHaarThreads, ((c.rows >> 1) + ppt - 1) / ppt);
#define WF_HAAR_LAUNCH(P)                                                        \
  if (vec)                                                                      \
    fuse_haar_kernel<T, Acc, NB, true, P><<<grid, kHaarThreads, 0, s>>>(c);     \
  else                                                                          \
    fuse_haar_kernel<T, Acc, NB, false, P><<<grid, kHaarThreads, 0, s>>>(c);
      switch (ppt) {
        case 1: WF_HAAR_LAUNCH(1) break;
        case 2: WF_HAAR_LAUNCH(2) break;
        case 8: WF_HAAR_LAUNCH(8) break;
        default: WF_HAAR_LAUNCH(4) break;
      }
#undef WF_HAAR_LAUNCH
    });
  }
  // D4: choose the row-run length so that the task count fills the chip
  a.n_colbands = (a.W + kColsPerWarp - 1) / kColsPerWarp;
  int target_warps = tune.d4_target_warps;
  if (target_warps <= 0) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (vec)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fuse_d4_kernel<T, Acc, NB, true>,
                                                    kD4Threads, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fuse_d4_kernel<T, Acc, NB, false>,
                                                    kD4Threads, 0);
    if (occ < 1) occ = 1;
    target_warps = sms * occ * (kD4Threads / 32);
  }
  int n_row = (target_warps + a.n_colbands - 1) / a.n_colbands;
  if (n_row < 1) n_row = 1;
  if (n_row > npairs) n_row = npairs;
  a.pairs_per_task = (npairs + n_row - 1) / n_row;
  if (tune.d4_min_pairs > 0 && a.pairs_per_task < tune.d4_min_pairs)
    a.pairs_per_task = tune.d4_min_pairs < npairs ? tune.d4_min_pairs : npairs;
  if (tune.d4_pairs > 0) a.pairs_per_task = tune.d4_pairs < npairs ? tune.d4_pairs : npairs;
  n_row = (npairs + a.pairs_per_task - 1) / a.pairs_per_task;
  a.n_tasks = (long long)n_row * a.n_colbands;
  const long long blocks = (a.n_tasks + (kD4Threads / 32) - 1) / (kD4Threads / 32);
  if (vec)
    fuse_d4_kernel<T, Acc, NB, true><<<(unsigned)blocks, kD4Threads, 0, s>>>(a);
  else
    fuse_d4_kernel<T, Acc, NB, false><<<(unsigned)blocks, kD4Threads, 0, s>>>(a);
  return cudaGetLastError();
}

template <typename T, typename Acc>
cudaError_t launch_fuse(int kind, const FuseArgs<T>& a, bool vec, bool tma, cudaStream_t s,
                        const LaunchTuning& tune) {
  if (kind == kDaub4 && tma) return launch_fuse_d4_tma<T>(a, s, tune);
  switch (a.nbands) {
    case 1: return launch_nb<T, Acc, 1>(kind, a, vec, s, tune);
    case 2: return launch_nb<T, Acc, 2>(kind, a, vec, s, tune);
    case 3: return launch_nb<T, Acc, 3>(kind, a, vec, s, tune);
    case 4: return launch_nb<T, Acc, 4>(kind, a, vec, s, tune);
    case 5: return launch_nb<T, Acc, 5>(kind, a, vec, s, tune);
    case 6: return launch_nb<T, Acc, 6>(kind, a, vec, s, tune);
    case 7: return launch_nb<T, Acc, 7>(kind, a, vec, s, tune);
    case 8: return launch_nb<T, Acc, 8>(kind, a, vec, s, tune);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// 8 bpp Haar (the paper's transfer representation, tiling.py:163-172): uint8
// PAN/MS in, quantised uint8 out (imageio.py:115-123 fused into the store).
// With integer inputs every intermediate is a multiple of 1/4, exact in
// float32, so the result is bit-identical to quantize(fuse_dwt(...)) of the
// float64 reference:
//   quantize(pan + ms - mean2x2) = clamp(x, 0, 1023) >> 2,
//   x = 4*pan + 4*ms + 2 - (sum of the 2x2 cell)     (x in [-1018, 2042])
// (clamp-then-shift equals the floor-then-clamp of imageio.py:115-123 on the
// exact value). The arithmetic runs two pixels per register in signed 16-bit
// lanes: one VIADDMNMX.S16x2.RELU adds the band term and clamps both lanes,
// so a pixel costs ~1.5 integer ops per band instead of ~5 (the scalar form
// was ALU-pipe bound). A thread owns 16 PAN columns x 2 rows (uint4 I/O).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lop3_sel(uint32_t a, uint32_t b, uint32_t mask) {
  uint32_t r;  // (a & mask) | (b & ~mask)
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(mask));
  return r;
}

template <int NB, int PPT = kHaarU8PairsPerThread>
__global__ void __launch_bounds__(kHaarThreads)
    fuse_haar_u8_kernel(const FuseArgs<uint8_t> a) {
  const int g = blockIdx.x * kHaarThreads + threadIdx.x;  // 16-column group
  const int c = 16 * g;
  if (c >= a.W) return;
  const int npairs = a.rows >> 1;
  const int i_begin = blockIdx.y * PPT;
#pragma unroll
  for (int s = 0; s < PPT; ++s) {
    const int i = i_begin + s;
    if (i >= npairs) break;
    const uint8_t* r0 = a.pan + (long long)(2 * i) * a.pan_pitch + c;
    uint4 w0, w1;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(w0.x), "=r"(w0.y), "=r"(w0.z), "=r"(w0.w)
        : "l"(r0));
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(w1.x), "=r"(w1.y), "=r"(w1.z), "=r"(w1.w)
        : "l"(r0 + a.pan_pitch));
    const uint32_t p0w[4] = {w0.x, w0.y, w0.z, w0.w}, p1w[4] = {w1.x, w1.y, w1.z, w1.w};
    // Per 4-column word d (cells 2d, 2d+1), lanes (lo, hi):
    //   ev[r][d] = 4*pan + 2 - cell sum at columns (4d, 4d+2) of row r,
    //   od[r][d] = the same at columns (4d+1, 4d+3)
    uint32_t ev[2][4], od[2][4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t e0 = __byte_perm(p0w[d], 0u, 0x4240), o0 = __byte_perm(p0w[d], 0u, 0x4341);
      const uint32_t e1 = __byte_perm(p1w[d], 0u, 0x4240), o1 = __byte_perm(p1w[d], 0u, 0x4341);
      const uint32_t cell = e0 + o0 + e1 + o1;            // lanes <= 1020: no carries
      const uint32_t c2 = __vsub2(0x00020002u, cell);     // 2 - sum, signed lanes
      ev[0][d] = __vadd2(e0 << 2, c2);
      od[0][d] = __vadd2(o0 << 2, c2);
      ev[1][d] = __vadd2(e1 << 2, c2);
      od[1][d] = __vadd2(o1 << 2, c2);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      uint2 mw;
      asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
          : "=r"(mw.x), "=r"(mw.y)
          : "l"(a.ms[b] + (long long)i * a.ms_pitch + (c >> 1)));
      uint32_t o[2][4];
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        // 4*ms of cells (2d, 2d+1) in lanes (lo, hi)
        const uint32_t m4 = __byte_perm(d < 2 ? mw.x : mw.y, 0u, (d & 1) ? 0x4342 : 0x4140) << 2;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const uint32_t ye = __viaddmin_s16x2_relu(ev[r][d], m4, 0x03FF03FFu);
          const uint32_t yo = __viaddmin_s16x2_relu(od[r][d], m4, 0x03FF03FFu);
          // bytes 0,2 <- ye >> 2 (columns 4d, 4d+2); bytes 1,3 <- yo >> 2
          o[r][d] = lop3_sel(ye >> 2, yo << 6, 0x00FF00FFu);
        }
      }
      uint8_t* w = a.out[b] + (long long)(2 * i) * a.out_pitch + c;
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(w), "r"(o[0][0]), "r"(o[0][1]),
                   "r"(o[0][2]), "r"(o[0][3])
                   : "memory");
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(w + a.out_pitch),
                   "r"(o[1][0]), "r"(o[1][1]), "r"(o[1][2]), "r"(o[1][3])
                   : "memory");
    }
  }
}

template <int NB>
static cudaError_t launch_haar_u8(const FuseArgs<uint8_t>& a, cudaStream_t s, int ppt_tune) {
  const int ng = (a.W + 15) / 16;
  int ppt = ppt_tune > 0 ? ppt_tune : kHaarU8PairsPerThread;
  if (ppt != 1 && ppt != 2 && ppt != 8) ppt = 4;
  return haar_row_chunks(a, ppt, [&](const FuseArgs<uint8_t>& c) {
    auto go = [&](auto P) {
      constexpr int kP = decltype(P)::value;
      dim3 grid((ng + kHaarThreads - 1) / kHaarThreads, ((c.rows >> 1) + kP - 1) / kP);
      fuse_haar_u8_kernel<NB, kP><<<grid, kHaarThreads, 0, s>>>(c);
    };
    switch (ppt) {
      case 1: go(std::integral_constant<int, 1>{}); break;
      case 2: go(std::integral_constant<int, 2>{}); break;
      case 8: go(std::integral_constant<int, 8>{}); break;
      default: go(std::integral_constant<int, 4>{}); break;
    }
  });
}

// uint8 specialisation: Haar needs 16-byte rows (vec), D4 the bulk-copy
// geometry (tma); the caller checks both before launching.
template <>
cudaError_t launch_fuse<uint8_t, float>(int kind, const FuseArgs<uint8_t>& a, bool vec, bool tma,
                                        cudaStream_t s, const LaunchTuning& tune) {
  if (kind == kDaub4) return tma ? launch_fuse_d4_tma<uint8_t>(a, s, tune) : cudaErrorInvalidValue;
  if (!vec) return cudaErrorInvalidValue;
  switch (a.nbands) {
    case 1: return launch_haar_u8<1>(a, s, tune.haar_u8_ppt);
    case 2: return launch_haar_u8<2>(a, s, tune.haar_u8_ppt);
    case 3: return launch_haar_u8<3>(a, s, tune.haar_u8_ppt);
    case 4: return launch_haar_u8<4>(a, s, tune.haar_u8_ppt);
    case 5: return launch_haar_u8<5>(a, s, tune.haar_u8_ppt);
    case 6: return launch_haar_u8<6>(a, s, tune.haar_u8_ppt);
    case 7: return launch_haar_u8<7>(a, s, tune.haar_u8_ppt);
    case 8: return launch_haar_u8<8>(a, s, tune.haar_u8_ppt);
    default: return cudaErrorInvalidValue;
  }
}

template cudaError_t launch_fuse<float, float>(int, const FuseArgs<float>&, bool, bool,
                                               cudaStream_t, const LaunchTuning&);
template cudaError_t launch_fuse<double, double>(int, const FuseArgs<double>&, bool, bool,
                                                 cudaStream_t, const LaunchTuning&);

}  // namespace wf
