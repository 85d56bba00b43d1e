// wavefuse-b200: internal launcher interface between the C-ABI layer
// (capi.cu) and the kernel translation units. Not part of the public ABI
// (that is include/wavefuse_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace wf {

constexpr int kMaxBandsPerLaunch = 8;

// Argument block of one fused launch over a (strip of a) scene. Passed by
// value as the kernel parameter (well under the 4 KB limit).
template <typename T>
struct FuseArgs {
  const T* pan;
  long long pan_pitch;  // elements
  // D4 halo row sources (2 rows each, pitch halo_pitch). For a whole image
  // they alias rows H-2..H-1 and 0..1 of the image itself (periodic wrap).
  const T* pan_top;
  const T* pan_bot;
  long long halo_pitch;
  const T* ms[kMaxBandsPerLaunch];
  const T* ms_top[kMaxBandsPerLaunch];  // D4: MS row i0-1 of each band
  long long ms_pitch;
  T* out[kMaxBandsPerLaunch];
  long long out_pitch;
  int nbands;
  int wide;  // float64 with 32-byte aligned rows: 256-bit PAN loads / output stores
  int fix_mode;  // 8 bpp D4 v3: 0 normal, 1 every unit re-done in float64, 2 in reference order
  int rows;  // PAN rows in this launch (even)
  int W;     // PAN columns (even)
  // filled by the launcher
  int pairs_per_task;
  int n_colbands;
  long long n_tasks;
};

struct LaunchTuning {
  int d4_target_warps;  // <=0: occupancy x SMs
  int d4_min_pairs;     // <=0: no minimum
  int d4_pairs;         // >0: fixed row pairs per warp task (overrides the above)
  int d4_stages;        // >0: shared-memory ring depth of the TMA kernel
  int haar_ppt;         // >0: Haar row pairs per thread (1, 2, 4, 8)
  int haar_u8_ppt;      // >0: 8 bpp Haar row pairs per thread
  int d4_u8_variant;    // 8 bpp D4: 0 = v3 byte-exact (default), 1 = v1 (4 columns), 2 = v2
  int u8_fix_mode;      // v3 test hook: 1 = recompute every unit, 2 = ... in reference order
  int d4_ldg;           // 1: force the register-path D4 kernel (no bulk copies)
  int no_wide;          // 1: float64 rows through 128-bit accesses, not 256-bit
  int exact_rows;       // >0: coefficient rows per CTA of the one-pass exact D4 kernel
  int exact_transforms; // 1: exact mode as forward + inverse transform kernels
  int qnr_kernel;       // QNR scene kernel: 2 = v2 role-split (default), 1 = v1, 3 = v3 (tile)
  int fq_ctas;          // >0: report CTAs of the overlapped fuse + report (default SMs - 28)
  int fq_band_rows;     // >0: row band of the overlapped fuse + report (rounded to 32)
  int fq_overlap;       // 1: fuse + report as the SM-partitioned overlap (measured slower; default:
                        //    Haar one pass, D4 the fusion kernel then the report kernel)
  int fq_debug;         // overlapped path experiments: 1 = no report kernel, 2 = report after fusion
};

// The tuning knobs of the environment (WF_HAAR_PPT, WF_D4_*, ...), read once
// per process (capi.cu); experiments set them before the first call.
const LaunchTuning& env_tuning();


// vec: 16-byte vector path legal; tma: the bulk-copy D4 pipeline is legal
// (W % 8 == 0, every row 16-byte aligned).
template <typename T, typename Acc>
cudaError_t launch_fuse(int kind, const FuseArgs<T>& a, bool vec, bool tma, cudaStream_t s,
                        const LaunchTuning& tune);
template <typename T>
cudaError_t launch_fuse_d4_tma(const FuseArgs<T>& a, cudaStream_t s, const LaunchTuning& tune);
// 8 bpp: uint8 in, float32 arithmetic, quantised uint8 out (fuse.cu)
template <>
cudaError_t launch_fuse<uint8_t, float>(int kind, const FuseArgs<uint8_t>& a, bool vec, bool tma,
                                        cudaStream_t s, const LaunchTuning& tune);
cudaError_t launch_u8_to_f32(const uint8_t* in, long long ip, int h, int w, float* out,
                             long long op, cudaStream_t s);
template <typename T>
cudaError_t launch_quantize(const T* in, long long ip, int h, int w, uint8_t* out, long long op,
                            cudaStream_t s);

// PNM front end (raster.cu): to_plane + pad_edge, pad_edge, quantize +
// interleave (imageio.py:104-123, tiling.py:285-310, cli.py:135-144).
constexpr int kMaxRasterPlanes = 8;
template <typename To>
cudaError_t launch_raster_to_plane(const uint8_t* r, int h, int w, int ch, int channel, To* out,
                                   long long op, int oh, int ow, cudaStream_t s);
template <typename T>
cudaError_t launch_pad_edge(const T* in, long long ip, int h, int w, T* out, long long op, int oh,
                            int ow, cudaStream_t s);
template <typename T>
cudaError_t launch_planes_to_raster(const T* const* planes, int np, long long pitch, int h, int w,
                                    uint8_t* r, cudaStream_t s);

// Standalone transforms (materialise coefficients; wavelet.py:131-164).
template <typename T>
cudaError_t launch_dwt2d(int kind, bool inverse, const T* in, long long in_pitch, T* out,
                         long long out_pitch, int h, int w, cudaStream_t s);
template <typename T>
cudaError_t launch_dwt_rows(int kind, bool inverse, const T* in, long long in_pitch, T* out,
                            long long out_pitch, int nrows, int n, cudaStream_t s);

// Reference-exact fuse_dwt: forward (f64, exact order) -> LL <- band*gain ->
// inverse -> cast; ws holds h*w doubles.
template <typename T>
cudaError_t launch_fuse_exact(int kind, const T* pan, long long pp, const T* ms, long long mp,
                              T* out, long long op, int h, int w, double* ws, cudaStream_t s);
template <typename T>
cudaError_t launch_fuse_exact_strip(int kind, const T* pan, long long pp, const T* pan_top,
                                    const T* pan_bot, long long hp, const T* const* ms,
                                    const T* const* ms_top, long long mp, T* const* out,
                                    long long op, int nbands, int rows, int w, cudaStream_t s);
template <typename T>
cudaError_t launch_fuse_bands_exact(int kind, const T* pan, long long pp, const T* const* ms,
                                    long long mp, T* const* out, long long op, int nbands,
                                    int h, int w, double* ws, cudaStream_t s);

// fusion.py:50-81
template <typename T, typename To>
cudaError_t launch_resample(const T* in, long long in_pitch, int in_h, int in_w, To* out,
                            long long out_pitch, int out_h, int out_w, cudaStream_t s);

// Quality metrics (metrics.py). `*64` flags: 1 = the plane is float64, 0 = float32.
void q_geometry(int h, int w, int& bh, int& bw, int& nbr, int& nbc);
cudaError_t launch_q_index(const void* a, int a64, long long ap, const void* b, int b64,
                           long long bp, int h, int w, double* scratch, double* out,
                           int out_index, cudaStream_t s);
cudaError_t launch_degrade(const void* in, int in64, long long ip, int h, int w, int f,
                           double* out, long long op, cudaStream_t s);
int ergas_parts(long long n);
cudaError_t launch_ergas_band(const void* fz, int f64, long long fp, const void* rf, int r64,
                              long long rp, int rh, int rw, int f, double* scratch, double* out,
                              cudaStream_t s);

// Fused single-pass quality report (quality_scene.cu), float32 planes,
// ratio 2, 2..8 bands, H, W >= 64.
size_t quality_scene_workspace(int nb, int h, int w);
// Haar fusion of (P, M) into O and the one-pass report of O, in one pass
// (the bands O inside the 32x32 block grid are written by the scoring kernel
// itself; the margins by the plain Haar kernel)
cudaError_t launch_fuse_quality_haar(int nb, const float* P, const float* const* M,
                                     float* const* O, long long op, long long mp, long long pp,
                                     int h, int w, void* workspace, double* out,
                                     int* undecidable, cudaStream_t s);
// Fusion (Haar or D4) and its quality report overlapped: the fusion runs in
// row bands on an internal stream while the persistent report kernel scores
// each band as soon as it is written (the bands come back from L2).
cudaError_t launch_fuse_quality_overlap(int kind, int nb, const float* P, const float* const* M,
                                        float* const* O, long long op, long long mp,
                                        long long pp, int h, int w, void* workspace,
                                        double* out, int* undecidable, cudaStream_t s,
                                        int* launches);
cudaError_t launch_quality_scene64(int nb, const double* const* F, const double* const* M,
                                   const double* P, long long fp, long long mp, long long pp,
                                   int h, int w, void* workspace, double* out, int* undecidable,
                                   cudaStream_t s);
cudaError_t launch_quality_scene(int nb, const float* const* F, const float* const* M,
                                 const float* P, long long fp, long long mp, long long pp, int h,
                                 int w, void* workspace, double* out, int* undecidable,
                                 cudaStream_t s);

// CUDA IPC for the peer-memory halo path (peer.cu)
cudaError_t ipc_export(const void* ptr, void* handle64, uint64_t* offset);
cudaError_t ipc_open(const void* handle64, void** base);
cudaError_t ipc_close(void* base);

// Counter-hash synthetic plane (uniform [0,255) f32), numpy twin in
// paper_1803_00737_b200/synth.py.
cudaError_t launch_synth(float* out, long long pitch, int rows, int cols, unsigned long long seed,
                         unsigned plane, int row0, int col0, cudaStream_t s);

}  // namespace wf
