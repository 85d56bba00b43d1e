// wavefuse-b200: shared device helpers for the sm_100a kernels.
//
// Everything here is header-only so each translation unit inlines it. The
// filter constants restate d4_filters() of the reference
// (/root/reference/pkg/src/wavefuse/wavelet.py:48-63):
//   h = [(1+s3), (3+s3), (3-s3), (1-s3)] / (4*sqrt 2)     analysis low
//   g = [h3, -h2, h1, -h0]                                 analysis high
//   synthesis_even = [h2, g2, h0, g0], synthesis_odd = [h3, g3, h1, g1]
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

// Checked builds (python -m paper_1803_00737_b200._build --checked, loaded
// with WF_CHECKED=1): device-side invariants of the bulk-copy rings -- every
// ring slot carries the index of the load it holds, written by the producer
// before the copies are issued and verified by each consumer after its full
// wait and again before it releases the slot (a slot overwritten early, read
// late or released twice traps) -- plus queue and index bounds. Compiled out
// of the product library. (compute-sanitizer is not available on the GPU
// pool; this is the substitute for its racecheck/synccheck on these rings.)
#ifdef WF_CHECKS
#define WF_CHECK(cond)                                                                  \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("WF_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,     \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                              \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#define WF_CHECK_TAG_BYTES 4
#else
#define WF_CHECK(cond) ((void)0)
#define WF_CHECK_TAG_BYTES 0
#endif

namespace wf {

// smem bytes per ring slot for the checked build's load tags (0 otherwise)
constexpr int kCheckTagBytesPerSlot = WF_CHECK_TAG_BYTES;

// Wire codes of the wavelet kinds (cluster.py:81-83 uses 1 = Haar, 2 = D4).
enum Kind : int { kHaar = 1, kDaub4 = 2 };

// Most bands one fused launch streams past a single PAN read. Landsat-7 ETM+
// has 6 reflective MS bands at half PAN resolution; 8 leaves headroom.
constexpr int kMaxBands = 8;

// D4 taps in double precision. These are the correctly rounded doubles of the
// closed forms above; numpy's d4_filters() computes (1+sqrt3)/(4*sqrt2) etc.
// with the same IEEE operations, so the values are bit-identical (checked in
// tests/test_oracle_pinning.py against the reference's printed taps).
struct D4 {
  double h0, h1, h2, h3, g0, g1, g2, g3;
};

__host__ __device__ inline D4 d4_taps() {
  // sqrt(3) and 4*sqrt(2) evaluated like wavelet.py:53-58 (IEEE sqrt is
  // correctly rounded on both host and device).
  const double s3 = sqrt(3.0);
  const double scale = 4.0 * sqrt(2.0);
  D4 t;
  t.h0 = (1.0 + s3) / scale;
  t.h1 = (3.0 + s3) / scale;
  t.h2 = (3.0 - s3) / scale;
  t.h3 = (1.0 - s3) / scale;
  t.g0 = t.h3;
  t.g1 = -t.h2;
  t.g2 = t.h1;
  t.g3 = -t.h0;
  return t;
}

// ---------------------------------------------------------------------------
// Streaming memory helpers. PAN/MS are read exactly once per fused pass
// (L1::no_allocate, keep the L1 for nothing); fused outputs are written once
// and never re-read by the kernel (evict-first .cs stores keep them from
// pushing the halo rows of neighbouring warps out of L2).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];"
               : "=f"(r.x), "=f"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
}

// Four consecutive elements of one row, as the compute type Acc.
template <typename T, typename Acc>
struct Quad {
  Acc v[4];
};

// Vector load of 4 consecutive elements at a 16-byte (f32) / 16-byte x2 (f64)
// aligned address.
template <typename Acc>
__device__ __forceinline__ void load4_vec(const float* p, Acc (&v)[4]) {
  float4 x = ld_stream(reinterpret_cast<const float4*>(p));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
template <typename Acc>
__device__ __forceinline__ void load4_vec(const double* p, Acc (&v)[4]) {
  double2 a = ld_stream(reinterpret_cast<const double2*>(p));
  double2 b = ld_stream(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
template <typename Acc>
__device__ __forceinline__ void load2_vec(const float* p, Acc (&v)[2]) {
  float2 x = ld_stream(reinterpret_cast<const float2*>(p));
  v[0] = x.x; v[1] = x.y;
}
template <typename Acc>
__device__ __forceinline__ void load2_vec(const double* p, Acc (&v)[2]) {
  double2 x = ld_stream(reinterpret_cast<const double2*>(p));
  v[0] = x.x; v[1] = x.y;
}

// 256-bit forms (LDG/STG.E.ENL2.256, new with sm_100) for float64 rows whose
// base and pitch are 32-byte aligned: one instruction moves a thread's 4
// doubles, so each warp instruction covers 1 KB contiguous. The two 128-bit
// halves of the plain path each cover every other 16 bytes of the warp's span,
// so every 32-byte sector is written by two separate instructions.
__device__ __forceinline__ void load4_wide(const double* p, double (&v)[4]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
}
__device__ __forceinline__ void store4_wide(double* p, const double (&v)[4]) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]),
               "d"(v[2]), "d"(v[3])
               : "memory");
}

template <typename Acc>
__device__ __forceinline__ void store4_vec(float* p, const Acc (&v)[4]) {
  st_stream(reinterpret_cast<float4*>(p),
            make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]));
}
template <typename Acc>
__device__ __forceinline__ void store4_vec(double* p, const Acc (&v)[4]) {
  st_stream(reinterpret_cast<double2*>(p), make_double2((double)v[0], (double)v[1]));
  st_stream(reinterpret_cast<double2*>(p) + 1, make_double2((double)v[2], (double)v[3]));
}

// Periodic index for the wrap-around boundary (wavelet.py:83-84,105-106 use
// np.roll, i.e. index mod n). Valid for any int i >= -n.
__device__ __forceinline__ int wrap(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

}  // namespace wf
