/*
 * wavefuse-b200 — C ABI of the B200-native DWT pan-sharpening hot path.
 *
 * This is the drop-in boundary. The reference (`wavefuse` 0.1.0, pure
 * Python + numpy) has no plugin registry; its boundary is the Python function
 * signatures of the hot path. Each entry point below replaces one of them and
 * cites it (paths relative to /root/reference/pkg/src/wavefuse/):
 *
 *   wf_fuse_dwt_*          fusion.py:128-150  fuse_dwt(pan, ms_band, kind)
 *   wf_fuse_bands_*        fusion.py:153-183  fuse(pan, ms, DwtReplace(kind)),
 *                          the per-band loop of fusion.py:182 fused into one
 *                          launch that reads PAN once
 *   wf_fuse_strip_*        (new) one row strip of fuse_dwt with explicit halo
 *                          rows, for the multi-GPU strip driver; replaces the
 *                          per-tile wrap of tiling.py:213-273 with exact halos
 *   wf_fuse_host_*         fuse() with HOST buffers: H2D, fuse, D2H pipelined
 *                          in row strips (what WorkerServer.handle_task,
 *                          cluster.py:297-299, or a ctypes caller would bind)
 *   wf_dwt2d_forward_*     wavelet.py:149-155  dwt2d_forward(plane, kind)
 *   wf_dwt2d_inverse_*     wavelet.py:158-164  dwt2d_inverse(coeffs, kind)
 *   wf_dwt_rows_forward_*  wavelet.py:131-139  dwt1d_forward (nrows = 1)
 *   wf_dwt_rows_inverse_*  wavelet.py:142-146  dwt1d_inverse (nrows = 1)
 *   wf_resample_bilinear_* fusion.py:50-81     resample_bilinear(plane, w, h)
 *   wf_degrade             metrics.py:31-42    degrade(plane, factor)
 *   wf_q_index             metrics.py:45-83    q_index(a, b)
 *   wf_ergas_band          metrics.py:94-119   ergas() per band
 *   wf_quality_scene_f32   metrics.py:178-199  qnr() in one pass over the scene
 *   wf_raster_to_plane_*   imageio.py:104-112 to_plane + tiling.py:285-293 pad_edge
 *   wf_pad_edge_*          tiling.py:285-293   pad_edge(plane, out_w, out_h)
 *   wf_planes_to_raster_*  cli.py:135-164      quantize + crop + interleave (PGM/PPM payload)
 *
 * Conventions
 *  - All array arguments of the device entry points are DEVICE pointers;
 *    pitches are in ELEMENTS. Arrays of band pointers (`ms`, `out`) are host
 *    arrays of device pointers.
 *  - `kind`: WF_HAAR = 1, WF_DAUB4 = 2 (the wire codes of cluster.py:81-83).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Every call is
 *    asynchronous on that stream and re-entrant: no global scratch, so
 *    concurrent callers on different streams/threads are safe
 *    (tiling.py:185-189 and cluster.py:352-370 call fuse_dwt concurrently).
 *  - Return 0 on success, else a WF_ERR_* code; wf_last_error() returns the
 *    calling thread's message. The codes map 1:1 onto the reference's
 *    exception classes (errors.py:32-73) in the Python shim.
 *  - Dtype rule (wavelet.py:69-70, fusion.py:46-47): f32 in -> f32 out, f64
 *    in -> f64 out. The f32 fused kernels compute in f32 (max-abs <= 1e-4 vs
 *    the float64 reference on 0..255 data); the f64 ones in f64; the
 *    standalone transforms and resample compute in f64 with the reference's
 *    exact operation order (bit-identical results).
 */
#ifndef WAVEFUSE_B200_H
#define WAVEFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  WF_HAAR = 1,
  WF_DAUB4 = 2
};

enum {
  WF_OK = 0,
  WF_ERR_VALUE = 1,              /* ValueError (bad ndim/kind/pointer/size)   */
  WF_ERR_ODD_DIMENSION = 2,      /* errors.OddDimension                        */
  WF_ERR_TOO_SMALL = 3,          /* errors.TooSmall                            */
  WF_ERR_DIMENSION_MISMATCH = 4, /* errors.DimensionMismatch                   */
  WF_ERR_CUDA = 5,               /* CUDA runtime failure (RuntimeError)        */
  WF_ERR_BAND_COUNT = 6,         /* errors.BandCountMismatch                   */
  WF_ERR_ODD_LENGTH = 7,         /* errors.OddLength                           */
  WF_ERR_TOO_SHORT = 8,          /* errors.TooShort                            */
  WF_ERR_NOT_DIVISIBLE = 9,      /* errors.NotDivisible                        */
  WF_ERR_CHANNEL = 10            /* errors.ChannelOutOfRange                   */
};

#define WF_MAX_BANDS_PER_LAUNCH 8

const char* wf_version(void);
const char* wf_last_error(void);
/* Number of kernel launches this thread has issued through the library. */
int64_t wf_launch_count(void);
/* Re-read the WF_* tuning environment variables (read once at load time
   otherwise; experiment knobs only, results do not depend on them). */
int wf_tuning_reload(void);
/* Debug builds: 1 if this library was built with the device-side ring and
   bounds invariants (python -m paper_1803_00737_b200._build --checked,
   loaded with WF_CHECKED=1), else 0. wf_check_selftest() runs one failing
   invariant: a checked build traps (and the CUDA context is lost -- call it
   from a throwaway process); a product build returns WF_OK. */
int wf_checked_build(void);
int wf_check_selftest(void);

/* ---- fused hot path (device buffers) ---------------------------------- */
int wf_fuse_dwt_f32(int kind, const float* pan, int64_t pan_pitch, const float* ms,
                    int64_t ms_pitch, float* out, int64_t out_pitch, int h, int w,
                    void* stream);
int wf_fuse_dwt_f64(int kind, const double* pan, int64_t pan_pitch, const double* ms,
                    int64_t ms_pitch, double* out, int64_t out_pitch, int h, int w,
                    void* stream);

int wf_fuse_bands_f32(int kind, const float* pan, int64_t pan_pitch,
                      const float* const* ms, int64_t ms_pitch, float* const* out,
                      int64_t out_pitch, int nbands, int h, int w, void* stream);
int wf_fuse_bands_f64(int kind, const double* pan, int64_t pan_pitch,
                      const double* const* ms, int64_t ms_pitch, double* const* out,
                      int64_t out_pitch, int nbands, int h, int w, void* stream);

/* One strip of `rows` PAN rows (even). D4 needs pan_top = the 2 PAN rows
 * above the strip, pan_bot = the 2 rows below (global periodic wrap applied
 * by the caller), ms_top[b] = the MS row above the strip of band b. Haar
 * ignores the halo pointers (may be NULL). */
int wf_fuse_strip_f32(int kind, const float* pan, int64_t pan_pitch, const float* pan_top,
                      const float* pan_bot, int64_t halo_pitch, const float* const* ms,
                      const float* const* ms_top, int64_t ms_pitch, float* const* out,
                      int64_t out_pitch, int nbands, int rows, int w, void* stream);
int wf_fuse_strip_f64(int kind, const double* pan, int64_t pan_pitch, const double* pan_top,
                      const double* pan_bot, int64_t halo_pitch, const double* const* ms,
                      const double* const* ms_top, int64_t ms_pitch, double* const* out,
                      int64_t out_pitch, int nbands, int rows, int w, void* stream);
/* The same strip in the reference-exact sequence (the one-pass float64
 * kernels reading the halo rows, which may live in a neighbour GPU's HBM):
 * the strips of a scene are bit-identical to the reference's whole-scene
 * fuse_dwt. */
int wf_fuse_strip_exact_f32(int kind, const float* pan, int64_t pan_pitch, const float* pan_top,
                            const float* pan_bot, int64_t halo_pitch, const float* const* ms,
                            const float* const* ms_top, int64_t ms_pitch, float* const* out,
                            int64_t out_pitch, int nbands, int rows, int w, void* stream);
int wf_fuse_strip_exact_f64(int kind, const double* pan, int64_t pan_pitch,
                            const double* pan_top, const double* pan_bot, int64_t halo_pitch,
                            const double* const* ms, const double* const* ms_top,
                            int64_t ms_pitch, double* const* out, int64_t out_pitch, int nbands,
                            int rows, int w, void* stream);

/* Reference-exact fuse_dwt (fusion.py:148-150 step by step): float64
 * forward transform in the reference's operation order, LL <- band * gain,
 * float64 inverse, one final cast -- bit-identical to the reference for f32
 * and f64 callers. One pass (see wf_fuse_bands_exact_*); the h*w float64
 * workspace (8*h*w bytes, caller-owned) is only used by the
 * WF_EXACT_TRANSFORMS=1 sequence. */
int wf_fuse_dwt_exact_f32(int kind, const float* pan, int64_t pan_pitch, const float* ms,
                          int64_t ms_pitch, float* out, int64_t out_pitch, int h, int w,
                          void* workspace, void* stream);
int wf_fuse_dwt_exact_f64(int kind, const double* pan, int64_t pan_pitch, const double* ms,
                          int64_t ms_pitch, double* out, int64_t out_pitch, int h, int w,
                          void* workspace, void* stream);

/* fuse(pan, bands, DwtReplace(kind)) in the reference-exact sequence
 * (fusion.py:182 calling fusion.py:148-150 per band), bit-identical to
 * calling wf_fuse_dwt_exact_* per band. One pass with no coefficient image:
 * the reference's float64 forward operations on the PAN (once for all
 * bands), LL = band * gain, its float64 inverse, one cast. `workspace`
 * (8*h*w bytes, caller-owned) is only used when WF_EXACT_TRANSFORMS=1
 * selects the transform-kernel sequence. Any band count. */
int wf_fuse_bands_exact_f32(int kind, const float* pan, int64_t pan_pitch,
                            const float* const* ms, int64_t ms_pitch, float* const* out,
                            int64_t out_pitch, int nbands, int h, int w, void* workspace,
                            void* stream);
int wf_fuse_bands_exact_f64(int kind, const double* pan, int64_t pan_pitch,
                            const double* const* ms, int64_t ms_pitch, double* const* out,
                            int64_t out_pitch, int nbands, int h, int w, void* workspace,
                            void* stream);

/* ---- fused hot path (HOST buffers, contiguous rows) --------------------- */
typedef struct wf_ctx wf_ctx;
/* strip_rows: PAN rows per pipeline stage (even; 0 = default 512). */
wf_ctx* wf_ctx_create(int device, int strip_rows);
/* exact != 0: the context's strips run the reference-exact one-pass kernels
 * (the float64 sequence of fusion.py:148-150 with the neighbouring strips'
 * halo rows) -- bit-identical host-buffer fusion at PCIe speed. u8 calls are
 * unaffected. */
int wf_ctx_set_exact(wf_ctx* ctx, int exact);
/* Host -> device copy of `bytes` from a (pageable or pinned) host buffer
 * through the context's pinned staging and copy workers; `after` is the
 * stream whose earlier work must finish before dst is written. Synchronous.
 * What the Python layer uses to bring numpy planes to the device for the
 * metrics (metrics.py's inputs) at the host-memcpy / PCIe rate. */
int wf_ctx_upload(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after);
/* Device -> host counterpart of wf_ctx_upload (`after` = the stream that
 * produced src). Synchronous. */
int wf_ctx_download(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after);
void wf_ctx_destroy(wf_ctx* ctx);
int wf_fuse_host_f32(wf_ctx* ctx, int kind, const float* pan, const float* const* ms,
                     float* const* out, int nbands, int h, int w);
int wf_fuse_host_f64(wf_ctx* ctx, int kind, const double* pan, const double* const* ms,
                     double* const* out, int nbands, int h, int w);

/* ---- 8 bpp transfer representation (tiling.py:163-172) ---
 * uint8 PAN/MS in, float32 arithmetic, quantised uint8 out: the fused
 * equivalent of [quantize(p) for p in fuse_tile_quantized(pan, ms, method)]
 * (tiling.py:268-269, imageio.py:115-123). Haar is bit-identical to the
 * reference (all intermediates are multiples of 1/4); D4 may differ by one
 * LSB where the float64 value lies within ~1e-4 of a .5 rounding boundary.
 * Haar needs W % 16 == 0, D4 W % 32 == 0, rows 16-byte aligned. */
int wf_fuse_bands_u8(int kind, const uint8_t* pan, int64_t pan_pitch, const uint8_t* const* ms,
                     int64_t ms_pitch, uint8_t* const* out, int64_t out_pitch, int nbands, int h,
                     int w, void* stream);
int wf_fuse_strip_u8(int kind, const uint8_t* pan, int64_t pan_pitch, const uint8_t* pan_top,
                     const uint8_t* pan_bot, int64_t halo_pitch, const uint8_t* const* ms,
                     const uint8_t* const* ms_top, int64_t ms_pitch, uint8_t* const* out,
                     int64_t out_pitch, int nbands, int rows, int w, void* stream);
int wf_fuse_host_u8(wf_ctx* ctx, int kind, const uint8_t* pan, const uint8_t* const* ms,
                    uint8_t* const* out, int nbands, int h, int w);
/* imageio.py:104-113 to_plane (uint8 -> float32) and :115-123 quantize. */
int wf_u8_to_f32(const uint8_t* in, int64_t in_pitch, int h, int w, float* out,
                 int64_t out_pitch, void* stream);
int wf_quantize_f32(const float* in, int64_t in_pitch, int h, int w, uint8_t* out,
                    int64_t out_pitch, void* stream);
int wf_quantize_f64(const double* in, int64_t in_pitch, int h, int w, uint8_t* out,
                    int64_t out_pitch, void* stream);

/* ---- PNM front end (cli.py:113-165) -------------
 * The per-pixel half of the CLI path; PGM/PPM header parsing stays on the
 * host. `raster` is the row-major, channel-interleaved uint8 payload
 * (h x w x channels) of imageio.py:46-87.
 * wf_raster_to_plane_*: imageio.py:104-112 to_plane(raster, channel) fused
 *   with tiling.py:285-293 pad_edge to out_h x out_w (>= h x w; the last row
 *   and column are replicated). channel outside [0, channels) ->
 *   WF_ERR_CHANNEL; out dims below h x w -> WF_ERR_VALUE. */
int wf_raster_to_plane_f32(const uint8_t* raster, int h, int w, int channels, int channel,
                           float* out, int64_t out_pitch, int out_h, int out_w, void* stream);
int wf_raster_to_plane_f64(const uint8_t* raster, int h, int w, int channels, int channel,
                           double* out, int64_t out_pitch, int out_h, int out_w, void* stream);
/* tiling.py:285-293 pad_edge(plane, out_w, out_h) of a float plane. */
int wf_pad_edge_f32(const float* in, int64_t in_pitch, int h, int w, float* out,
                    int64_t out_pitch, int out_h, int out_w, void* stream);
int wf_pad_edge_f64(const double* in, int64_t in_pitch, int h, int w, double* out,
                    int64_t out_pitch, int out_h, int out_w, void* stream);
/* cli.py:135-164: quantize (imageio.py:115-123, in the planes' dtype) of the
 * top-left h x w window (the crop b[:h, :w]) of `nplanes` (1..8) planes with
 * a common pitch, interleaved into raster (h x w x nplanes): the PGM payload
 * for one plane, the PPM one (np.stack(bands, axis=-1)) for three.
 * `planes` is a host array of device pointers. */
int wf_planes_to_raster_f32(const float* const* planes, int nplanes, int64_t pitch, int h, int w,
                            uint8_t* raster, void* stream);
int wf_planes_to_raster_f64(const double* const* planes, int nplanes, int64_t pitch, int h, int w,
                            uint8_t* raster, void* stream);

/* ---- standalone transforms --------------------------------------------- */
int wf_dwt2d_forward_f32(int kind, const float* in, int64_t in_pitch, float* out,
                         int64_t out_pitch, int h, int w, void* stream);
int wf_dwt2d_forward_f64(int kind, const double* in, int64_t in_pitch, double* out,
                         int64_t out_pitch, int h, int w, void* stream);
int wf_dwt2d_inverse_f32(int kind, const float* in, int64_t in_pitch, float* out,
                         int64_t out_pitch, int h, int w, void* stream);
int wf_dwt2d_inverse_f64(int kind, const double* in, int64_t in_pitch, double* out,
                         int64_t out_pitch, int h, int w, void* stream);
int wf_dwt_rows_forward_f32(int kind, const float* in, int64_t in_pitch, float* out,
                            int64_t out_pitch, int nrows, int n, void* stream);
int wf_dwt_rows_forward_f64(int kind, const double* in, int64_t in_pitch, double* out,
                            int64_t out_pitch, int nrows, int n, void* stream);
int wf_dwt_rows_inverse_f32(int kind, const float* in, int64_t in_pitch, float* out,
                            int64_t out_pitch, int nrows, int n, void* stream);
int wf_dwt_rows_inverse_f64(int kind, const double* in, int64_t in_pitch, double* out,
                            int64_t out_pitch, int nrows, int n, void* stream);

int wf_resample_bilinear_f32(const float* in, int64_t in_pitch, int in_h, int in_w,
                             float* out, int64_t out_pitch, int out_h, int out_w,
                             void* stream);
int wf_resample_bilinear_f64(const double* in, int64_t in_pitch, int in_h, int in_w,
                             double* out, int64_t out_pitch, int out_h, int out_w,
                             void* stream);

/* metrics.py:122-123 upsamples the float64-cast bands (_as_bands): float32
 * source, float64 result, bit-identical to resample_bilinear(b.astype(f64)). */
int wf_resample_bilinear_f32_to_f64(const float* in, int64_t in_pitch, int in_h, int in_w,
                                    double* out, int64_t out_pitch, int out_h, int out_w,
                                    void* stream);

/* ---- quality metrics (metrics.py) --------------------------------------- */
/* Planes are float32 (x_f64 = 0) or float64 (x_f64 = 1); all statistics are
 * float64. Results land in DEVICE memory (out[out_index]); workspaces are
 * caller-owned device scratch of the size the *_workspace_bytes call returns,
 * so concurrent callers never share state. */
int64_t wf_q_index_workspace_bytes(int h, int w);
/* metrics.py:57-83 q_index(a, b): 32x32 blocks (partial edges dropped, planes
 * under 32 are one block), population moments, den == 0 -> 1 if identical
 * else 0; block mean. */
int wf_q_index(const void* a, int a_f64, int64_t a_pitch, const void* b, int b_f64,
               int64_t b_pitch, int h, int w, void* workspace, double* out, int out_index,
               void* stream);
/* metrics.py:31-42 degrade(plane, factor) -> float64 (h/f x w/f). */
int wf_degrade(const void* in, int in_f64, int64_t in_pitch, int h, int w, int factor,
               double* out, int64_t out_pitch, void* stream);
int64_t wf_ergas_workspace_bytes(int rh, int rw);
/* metrics.py:112-118, one band: out2[0] = mean((degrade(fused, ratio) - ref)^2),
 * out2[1] = mean(ref). */
int wf_ergas_band(const void* fused, int f_f64, int64_t f_pitch, const void* ref, int r_f64,
                  int64_t r_pitch, int rh, int rw, int ratio, void* workspace, double* out2,
                  void* stream);

/* metrics.py:178-199 qnr() in ONE pass over a float32 scene (ratio 2,
 * 2..8 bands, even H, W % 8 == 0, H, W >= 64, 16-byte aligned rows). out (device, float64):
 *   [0, B)                 Q(F_k, U_k)            (q_per_band)
 *   [B, B + B(B-1)/2)      Q(F_k, F_l), k < l     (d_lambda, fused side)
 *   next B(B-1)/2          Q(U_k, U_l), k < l     (d_lambda, upsampled side)
 *   next B                 Q(F_k, P)              (d_s, full resolution)
 *   next B                 Q(M_k, degrade(P, 2))  (d_s, low resolution)
 *   next B                 MSE(degrade(F_k, 2), M_k)   (ergas)
 *   next B                 mean(M_k)                   (ergas)
 * with U_k = resample_bilinear(M_k, W, H). *undecidable > 0 means some block
 * hit den == 0 with non-constant data (the reference then compares the blocks
 * element-wise): recompute with wf_q_index. */
int64_t wf_quality_scene_workspace_bytes(int nbands, int h, int w);
int wf_quality_scene_f32(const float* const* fused, const float* const* ms, const float* pan,
                         int64_t f_pitch, int64_t ms_pitch, int64_t pan_pitch, int nbands, int h,
                         int w, void* workspace, double* out, int* undecidable, void* stream);
/* The same report for a float64 scene (the planes a float64 numpy caller's
 * fuse() returns, fusion.py:46-47): float64 shifts, upsampling and 2x2 cells,
 * float32 shifted moments -- the precision of the float32 path. Same output
 * layout and workspace; the fused bands and the PAN share one pitch; 16-byte
 * aligned rows. */
int wf_quality_scene_f64(const double* const* fused, const double* const* ms, const double* pan,
                         int64_t f_pitch, int64_t ms_pitch, int64_t pan_pitch, int nbands, int h,
                         int w, void* workspace, double* out, int* undecidable, void* stream);
/* SURVEY.md 8(f) row f1, second half: fusion and its quality report in ONE
 * call -- fusion.py:153-183 fuse(pan, ms, DwtReplace(kind)) followed by
 * metrics.py:178-199 qnr(fused, ms, pan). Haar: one pass over the scene (the
 * scoring kernel fuses each pixel itself and streams the bands out; they are
 * never re-read). D4: the fusion kernel, then the scoring kernel on its
 * output (the fastest schedule measured; WF_FQ_OVERLAP=1 selects an
 * SM-partitioned overlap of the two, slower). Writes out[0..nbands)
 * (bit-identical to wf_fuse_bands_f32) and the report in
 * wf_quality_scene_f32's layout (bit-identical to it on those bands); same
 * shape/alignment rules and workspace (wf_quality_scene_workspace_bytes). */
int wf_fuse_quality_f32(int kind, const float* pan, int64_t pan_pitch, const float* const* ms,
                        int64_t ms_pitch, float* const* out, int64_t out_pitch, int nbands, int h,
                        int w, void* workspace, double* report, int* undecidable, void* stream);

/* ---- peer-memory halos for strip-sharded scenes (one process per GPU) ----
 * wf_ipc_export: 64-byte CUDA IPC handle of the allocation containing `ptr`
 * and the byte offset of `ptr` in it. wf_ipc_open: map a neighbour's handle
 * (lazy peer access over NVLink); pass base + offset + row * pitch as the
 * pan_top / pan_bot / ms_top halo pointers of wf_fuse_strip_*, whose producer
 * then copies the halo rows straight out of peer HBM. */
int wf_ipc_export(const void* ptr, void* handle64, uint64_t* offset);
int wf_ipc_open(const void* handle64, void** base);
int wf_ipc_close(void* base);

/* ---- synthetic scenes (counter hash; numpy twin in synth.py) ------------ */
int wf_synth_plane_f32(float* out, int64_t pitch, int rows, int cols, uint64_t seed,
                       uint32_t plane, int row0, int col0, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* WAVEFUSE_B200_H */
