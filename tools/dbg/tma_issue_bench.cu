// Microbenchmark: cycles per bulk copy issued by one warp (per-lane issue vs
// lane-0 uniform loop), 1 KB copies from L2-resident global memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1803_00737_b200/csrc/wf_tma.cuh"
using namespace wf;

template <int MODE>
__global__ void k(const float* src, long long* out, int n_copies, int bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  float* dst = reinterpret_cast<float*>(sm + 128);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { tma::mbar_init(bar, 1); tma::fence_barrier_init(); }
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep) {
    if (lane == 0) tma::mbar_arrive_expect_tx(bar, (uint32_t)(n_copies * bytes));
    __syncwarp();
    if (MODE == 0) {  // per-lane issue
      for (int c = lane; c < n_copies; c += 32)
        tma::bulk_g2s(dst + (size_t)c * bytes / 4, src + (size_t)(c + rep * n_copies) * bytes / 4,
                      bytes, bar);
    } else {  // lane 0, uniform loop
      if (lane == 0)
        for (int c = 0; c < n_copies; ++c)
          tma::bulk_g2s(dst + (size_t)c * bytes / 4, src + (size_t)(c + rep * n_copies) * bytes / 4,
                        bytes, bar);
    }
    long long t1 = clock64();
    tma::mbar_wait(bar, rep & 1);
    long long t2 = clock64();
    if (lane == 0 && blockIdx.x == 0) { out[2 * rep] = t1 - t0; out[2 * rep + 1] = t2 - t0; }
    t0 = clock64();
  }
}

int main() {
  float* src; long long* out;
  cudaMalloc(&src, 64 << 20); cudaMemset(src, 0, 64 << 20);
  cudaMallocManaged(&out, 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int n : {8, 16, 32}) for (int bytes : {512, 1024, 4096}) {
      size_t smem = 128 + (size_t)n * bytes;
      auto kern = mode ? k<1> : k<0>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int grid : {1, 148}) {
        kern<<<grid, 32, smem>>>(src, out, n, bytes);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("mode %s grid %3d copies %2d x %4d B: issue %6lld cyc, complete %6lld cyc (rep 7)\n",
               mode ? "lane0 " : "perlane", grid, n, bytes, out[14], out[15]);
      }
    }
  return 0;
}
