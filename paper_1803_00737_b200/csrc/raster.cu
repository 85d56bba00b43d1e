// wavefuse-b200: the PNM front end of the fusion path on the GPU (SURVEY.md
// 8(f) row f4): 8-bit rasters in, planes out, and back.
//
// The reference's CLI path (cli.py:113-165) reads PGM/PPM rasters
// (imageio.py:46-87), takes channel planes as float32 (to_plane,
// imageio.py:104-112), edge-pads the scene to a grid-compatible size
// (pad_inputs / pad_edge, tiling.py:285-310), fuses, crops, quantises
// (imageio.py:115-123) and writes one interleaved PPM or PGMs
// (cli.py:135-144, imageio.py:90-101). Header parsing is a few bytes of
// sequential host work; everything per pixel is here, so a scene crosses
// PCIe as 8-bit rasters (1 B/px per channel each way) instead of float planes.
//
// All kernels are byte-granular HBM streams; one thread per output pixel,
// grid-stride over rows, coalesced on the output side (the interleaved side
// is a stride-C byte access, contiguous per warp).
#include "wf_common.cuh"
#include "wf_kernels.h"

namespace wf {

// to_plane + pad_edge in one pass: out(y, x) = raster(min(y, h-1),
// min(x, w-1), channel), as To. np.pad(mode="edge") replicates the last row
// and column (tiling.py:285-293); to_plane converts uint8 -> float32
// exactly (imageio.py:104-112).
template <typename To>
__global__ void raster_to_plane_kernel(const uint8_t* __restrict__ r, int h, int w, int ch,
                                       int channel, To* __restrict__ out, long long op, int oh,
                                       int ow) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= ow) return;
  const int sx = min(x, w - 1);
  for (int y = blockIdx.y; y < oh; y += gridDim.y) {
    const int sy = min(y, h - 1);
    out[(long long)y * op + x] = (To)r[((long long)sy * w + sx) * ch + channel];
  }
}

// pad_edge (tiling.py:285-293) of a float plane.
template <typename T>
__global__ void pad_edge_kernel(const T* __restrict__ in, long long ip, int h, int w,
                                T* __restrict__ out, long long op, int oh, int ow) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= ow) return;
  const int sx = min(x, w - 1);
  for (int y = blockIdx.y; y < oh; y += gridDim.y)
    out[(long long)y * op + x] = in[(long long)min(y, h - 1) * ip + sx];
}

// quantize (imageio.py:115-123: clamp to [0, 255], floor(x + 0.5), in the
// plane's dtype like numpy) of the top-left h x w window of every plane,
// interleaved: raster(y, x, k) = quantize(plane_k(y, x)). With one plane this
// is the PGM payload, with three the PPM one (np.stack(bands, axis=-1),
// cli.py:137-138).
template <typename T>
struct PlaneSet {
  const T* p[kMaxRasterPlanes];
};

template <typename T>
__device__ __forceinline__ uint8_t quantize1(T v) {
  const T c = fmin(fmax(v, T(0)), T(255));
  return (uint8_t)floor(c + T(0.5));
}

template <typename T>
__global__ void planes_to_raster_kernel(const PlaneSet<T> ps, int np, long long pitch, int h,
                                        int w, uint8_t* __restrict__ r) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    uint8_t* dst = r + ((long long)y * w + x) * np;
    for (int k = 0; k < np; ++k) dst[k] = quantize1<T>(ps.p[k][(long long)y * pitch + x]);
  }
}

static dim3 raster_grid(int h, int w) {
  return dim3((unsigned)((w + 255) / 256), (unsigned)(h < 65535 ? h : 65535));
}

template <typename To>
cudaError_t launch_raster_to_plane(const uint8_t* r, int h, int w, int ch, int channel, To* out,
                                   long long op, int oh, int ow, cudaStream_t s) {
  raster_to_plane_kernel<To><<<raster_grid(oh, ow), 256, 0, s>>>(r, h, w, ch, channel, out, op,
                                                                 oh, ow);
  return cudaGetLastError();
}
template cudaError_t launch_raster_to_plane<float>(const uint8_t*, int, int, int, int, float*,
                                                   long long, int, int, cudaStream_t);
template cudaError_t launch_raster_to_plane<double>(const uint8_t*, int, int, int, int, double*,
                                                    long long, int, int, cudaStream_t);

template <typename T>
cudaError_t launch_pad_edge(const T* in, long long ip, int h, int w, T* out, long long op, int oh,
                            int ow, cudaStream_t s) {
  pad_edge_kernel<T><<<raster_grid(oh, ow), 256, 0, s>>>(in, ip, h, w, out, op, oh, ow);
  return cudaGetLastError();
}
template cudaError_t launch_pad_edge<float>(const float*, long long, int, int, float*, long long,
                                            int, int, cudaStream_t);
template cudaError_t launch_pad_edge<double>(const double*, long long, int, int, double*,
                                             long long, int, int, cudaStream_t);

template <typename T>
cudaError_t launch_planes_to_raster(const T* const* planes, int np, long long pitch, int h, int w,
                                    uint8_t* r, cudaStream_t s) {
  PlaneSet<T> ps{};
  for (int k = 0; k < np; ++k) ps.p[k] = planes[k];
  planes_to_raster_kernel<T><<<raster_grid(h, w), 256, 0, s>>>(ps, np, pitch, h, w, r);
  return cudaGetLastError();
}
template cudaError_t launch_planes_to_raster<float>(const float* const*, int, long long, int, int,
                                                    uint8_t*, cudaStream_t);
template cudaError_t launch_planes_to_raster<double>(const double* const*, int, long long, int,
                                                     int, uint8_t*, cudaStream_t);

}  // namespace wf
