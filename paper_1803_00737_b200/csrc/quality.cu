// wavefuse-b200: quality metrics on the GPU (reference metrics.py).
//
// Generic, reference-structured kernels (any shape, any dtype mix):
//   q_blocks_kernel      one CTA per Q block: two-pass float64 moments (mean
//                        first, then centred sums -- the reference's np.mean /
//                        np.var order of operations, metrics.py:71-75), the
//                        exact den == 0 degenerate rule with an element-wise
//                        identity test (metrics.py:76-82), Q per block;
//   mean_reduce_kernel   deterministic single-CTA mean of the per-block Q
//                        values (fixed summation tree, no atomics);
//   degrade_kernel       factor x factor block mean in float64 (metrics.py:31-42);
//   ergas_partials_kernel per-CTA partial sums of (degrade(F) - R)^2 and of R
//                        (metrics.py:94-119), reduced deterministically.
// The fused single-pass scene kernel (quality_scene.cu) computes every
// quantity of qnr() in one read of the scene; these kernels are its
// cross-check and serve shapes it does not cover.
#include <cuda_runtime.h>

#include "wf_common.cuh"
#include "wf_kernels.h"

namespace wf {

constexpr int kQThreads = 256;

__device__ __forceinline__ double ld_any(const void* p, int f64, long long idx) {
  return f64 ? static_cast<const double*>(p)[idx] : (double)static_cast<const float*>(p)[idx];
}

template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double* red /* [N][32] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) red[k * 32 + warp] = v[k];
  __syncthreads();
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[k * 32 + w];
    v[k] = s;
  }
}

// Q block (br, bc) of planes a, b: rows [br*bh, br*bh+bh), cols [bc*bw, ...).
__global__ void __launch_bounds__(kQThreads)
    q_blocks_kernel(const void* a, int a64, long long ap, const void* b, int b64, long long bp,
                    int bh, int bw, int nbc, double* q_out) {
  __shared__ double red[4 * 32];
  const int blk = blockIdx.x;
  const int br = blk / nbc, bc = blk % nbc;
  const long long r0 = (long long)br * bh, c0 = (long long)bc * bw;
  const int n = bh * bw;
  double s[2] = {0.0, 0.0};
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const long long r = r0 + e / bw, c = c0 + e % bw;
    s[0] += ld_any(a, a64, r * ap + c);
    s[1] += ld_any(b, b64, r * bp + c);
  }
  block_sum<2>(s, red);
  const double mu_a = s[0] / n, mu_b = s[1] / n;
  double m[4] = {0.0, 0.0, 0.0, 0.0};  // saa, sbb, sab, #unequal
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const long long r = r0 + e / bw, c = c0 + e % bw;
    const double x = ld_any(a, a64, r * ap + c), y = ld_any(b, b64, r * bp + c);
    const double dx = x - mu_a, dy = y - mu_b;
    m[0] += dx * dx;
    m[1] += dy * dy;
    m[2] += dx * dy;
    m[3] += (x != y) ? 1.0 : 0.0;
  }
  block_sum<4>(m, red);
  if (threadIdx.x == 0) {
    const double va = m[0] / n, vb = m[1] / n, cov = m[2] / n;
    const double num = 4.0 * cov * mu_a * mu_b;
    const double den = (va + vb) * (mu_a * mu_a + mu_b * mu_b);
    q_out[blk] = den == 0.0 ? (m[3] == 0.0 ? 1.0 : 0.0) : num / den;
  }
}

// Deterministic mean of n doubles (one CTA, fixed order).
__global__ void __launch_bounds__(1024) mean_reduce_kernel(const double* v, long long n,
                                                           double* out, int out_index) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[out_index] = t / (double)n;
  }
}

// out(i, j) = mean of the factor x factor block (float64)
__global__ void degrade_kernel(const void* in, int in64, long long ip, int oh, int ow, int f,
                               double* out, long long op) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= oh || j >= ow) return;
  double s = 0.0;
  for (int di = 0; di < f; ++di)
    for (int dj = 0; dj < f; ++dj)
      s += ld_any(in, in64, (long long)(i * f + di) * ip + (long long)j * f + dj);
  out[(long long)i * op + j] = s / (double)(f * f);
}

// Per-CTA partials over reference pixels: [sse, sum_ref] -> part[2*cta + k]
__global__ void __launch_bounds__(kQThreads)
    ergas_partials_kernel(const void* fz, int f64, long long fp, const void* rf, int r64,
                          long long rp, int rh, int rw, int f, double* part) {
  __shared__ double red[2 * 32];
  const long long n = (long long)rh * rw;
  double acc[2] = {0.0, 0.0};
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / rw), j = (int)(e % rw);
    double s = 0.0;
    for (int di = 0; di < f; ++di)
      for (int dj = 0; dj < f; ++dj)
        s += ld_any(fz, f64, (long long)(i * f + di) * fp + (long long)j * f + dj);
    const double r = ld_any(rf, r64, (long long)i * rp + j);
    const double d = s / (double)(f * f) - r;
    acc[0] += d * d;
    acc[1] += r;
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc[0];
    part[2 * blockIdx.x + 1] = acc[1];
  }
}

// Sum the per-CTA partial pairs deterministically; out[0] = sse/n (MSE),
// out[1] = sum_ref/n (mean of the reference band).
__global__ void ergas_finish_kernel(const double* part, int nparts, long long n, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s0 = 0.0, s1 = 0.0;
  for (int k = 0; k < nparts; ++k) {
    s0 += part[2 * k];
    s1 += part[2 * k + 1];
  }
  out[0] = s0 / (double)n;
  out[1] = s1 / (double)n;
}

// ---- launchers ---------------------------------------------------------------
void q_geometry(int h, int w, int& bh, int& bw, int& nbr, int& nbc) {
  // metrics.py:45-54: full 32x32 blocks, partial edges dropped; planes under
  // 32 in either direction are one block
  if (h < 32 || w < 32) {
    bh = h;
    bw = w;
    nbr = nbc = 1;
  } else {
    bh = bw = 32;
    nbr = h / 32;
    nbc = w / 32;
  }
}

cudaError_t launch_q_index(const void* a, int a64, long long ap, const void* b, int b64,
                           long long bp, int h, int w, double* scratch, double* out,
                           int out_index, cudaStream_t s) {
  int bh, bw, nbr, nbc;
  q_geometry(h, w, bh, bw, nbr, nbc);
  const int nblk = nbr * nbc;
  q_blocks_kernel<<<nblk, kQThreads, 0, s>>>(a, a64, ap, b, b64, bp, bh, bw, nbc, scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  mean_reduce_kernel<<<1, 1024, 0, s>>>(scratch, nblk, out, out_index);
  return cudaGetLastError();
}

cudaError_t launch_degrade(const void* in, int in64, long long ip, int h, int w, int f,
                           double* out, long long op, cudaStream_t s) {
  const int oh = h / f, ow = w / f;
  dim3 block(32, 8), grid((ow + 31) / 32, (oh + 7) / 8);
  degrade_kernel<<<grid, block, 0, s>>>(in, in64, ip, oh, ow, f, out, op);
  return cudaGetLastError();
}

int ergas_parts(long long n) {
  long long p = (n + kQThreads * 8 - 1) / (kQThreads * 8);
  if (p > 2048) p = 2048;
  if (p < 1) p = 1;
  return (int)p;
}

cudaError_t launch_ergas_band(const void* fz, int f64, long long fp, const void* rf, int r64,
                              long long rp, int rh, int rw, int f, double* scratch, double* out,
                              cudaStream_t s) {
  const long long n = (long long)rh * rw;
  const int parts = ergas_parts(n);
  ergas_partials_kernel<<<parts, kQThreads, 0, s>>>(fz, f64, fp, rf, r64, rp, rh, rw, f, scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ergas_finish_kernel<<<1, 32, 0, s>>>(scratch, parts, n, out);
  return cudaGetLastError();
}

}  // namespace wf
