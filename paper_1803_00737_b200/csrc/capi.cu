// wavefuse-b200: extern "C" boundary (include/wavefuse_b200.h).
//
// Validation mirrors the reference's preconditions and their order
// (fusion.py:137-147 then wavelet.py:121-128 inside dwt2d_forward) so the
// Python shim can map return codes onto the same exception classes.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <sched.h>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/wavefuse_b200.h"
#include "wf_common.cuh"
#include "wf_kernels.h"

namespace wf {
// Environment tuning knobs, read once (the first call) instead of per call;
// wf_tuning_reload() re-reads them (experiments and tests that change them).
static LaunchTuning read_tuning() {
  LaunchTuning v{};
  auto num = [](const char* name) {
    const char* e = getenv(name);
    return e ? atoi(e) : 0;
  };
  auto is = [](const char* name, const char* val) {
    const char* e = getenv(name);
    return e && strcmp(e, val) == 0;
  };
  v.haar_ppt = num("WF_HAAR_PPT");
  v.d4_target_warps = num("WF_D4_TARGET_WARPS");
  v.d4_min_pairs = num("WF_D4_MIN_PAIRS");
  v.d4_pairs = num("WF_D4_PAIRS");
  v.d4_stages = num("WF_D4_STAGES");
  v.haar_u8_ppt = num("WF_HAAR_U8_PPT");
  v.d4_u8_variant = is("WF_D4_U8", "v1") ? 1 : is("WF_D4_U8", "v2") ? 2 : 0;
  v.u8_fix_mode = is("WF_U8_FIX", "all")       ? 1
                  : is("WF_U8_FIX", "ref")     ? 2
                  : is("WF_U8_FIX", "skipfix") ? 3   // timing experiments only:
                  : is("WF_U8_FIX", "nodetect") ? 4  // bytes not exact
                                                : 0;
  v.d4_ldg = is("WF_D4_PATH", "ldg");
  v.no_wide = getenv("WF_NO_WIDE") != nullptr;
  v.exact_rows = num("WF_EXACT_ROWS");
  v.exact_transforms = getenv("WF_EXACT_TRANSFORMS") != nullptr;
  const char* q = getenv("WF_QNR_KERNEL");
  v.qnr_kernel = (q && q[0] == 'v' && q[1] == '1') ? 1 : (q && q[0] == 'v' && q[1] == '3') ? 3 : 2;
  v.fq_ctas = num("WF_FQ_CTAS");
  v.fq_band_rows = num("WF_FQ_BAND_ROWS");
  v.fq_overlap = num("WF_FQ_OVERLAP");
  v.fq_debug = num("WF_FQ_DEBUG");
  return v;
}
static LaunchTuning g_tuning = read_tuning();

const LaunchTuning& env_tuning() { return g_tuning; }
}  // namespace wf

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return WF_OK;
  return fail(WF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int min_len(int kind) { return kind == WF_HAAR ? 2 : 4; }  // wavelet.py:66

int check_kind(int kind) {
  if (kind != WF_HAAR && kind != WF_DAUB4)
    return fail(WF_ERR_VALUE, "unknown wavelet kind %d", kind);
  return WF_OK;
}

// wavelet.py:121-128 (_check_2d, after the ndim test the shim does)
int check_2d(int kind, int h, int w) {
  if (int e = check_kind(kind)) return e;
  if (h < min_len(kind) || w < min_len(kind))
    return fail(WF_ERR_TOO_SMALL, "%dx%d below minimum %d per side", w, h, min_len(kind));
  if ((h & 1) || (w & 1)) return fail(WF_ERR_ODD_DIMENSION, "%dx%d has an odd dimension", w, h);
  return WF_OK;
}

// wavelet.py:112-118 (_check_1d)
int check_1d(int kind, int n) {
  if (int e = check_kind(kind)) return e;
  if (n < min_len(kind)) return fail(WF_ERR_TOO_SHORT, "length %d below minimum %d", n, min_len(kind));
  if (n & 1) return fail(WF_ERR_ODD_LENGTH, "length %d is odd", n);
  return WF_OK;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool al32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

template <typename T>
int fuse_common(int kind, const T* pan, int64_t pan_pitch, const T* pan_top, const T* pan_bot,
                int64_t halo_pitch, const T* const* ms, const T* const* ms_top, int64_t ms_pitch,
                T* const* out, int64_t out_pitch, int nbands, int rows, int w, bool strip,
                cudaStream_t s, bool exact = false) {
  if (int e = check_kind(kind)) return e;
  if (nbands < 1) return fail(WF_ERR_BAND_COUNT, "need at least one band");
  if (!pan || !ms || !out) return fail(WF_ERR_VALUE, "null pointer argument");
  // fusion.py:140-141 (odd) precedes the band-shape test; dwt2d_forward's
  // TooSmall comes last (wavelet.py:124-126 via fusion.py:148)
  if ((rows & 1) || (w & 1))
    return fail(WF_ERR_ODD_DIMENSION, "panchromatic plane %dx%d has an odd dimension", w, rows);
  if (!strip && (rows < min_len(kind) || w < min_len(kind)))
    return fail(WF_ERR_TOO_SMALL, "%dx%d below minimum %d per side", w, rows, min_len(kind));
  if (strip && (rows < 2 || w < min_len(kind)))
    return fail(WF_ERR_TOO_SMALL, "strip %dx%d too small", w, rows);
  if (pan_pitch < w || out_pitch < w || ms_pitch < w / 2)
    return fail(WF_ERR_VALUE, "pitch smaller than row length");
  if (kind == WF_DAUB4 && strip && (!pan_top || !pan_bot || !ms_top))
    return fail(WF_ERR_VALUE, "D4 strip needs halo pointers");
  for (int b = 0; b < nbands; ++b)
    if (!ms[b] || !out[b]) return fail(WF_ERR_VALUE, "null band pointer %d", b);
  if constexpr (sizeof(T) != 1) {
    if (exact) {  // the reference's float64 sequence, one pass (transforms.cu)
      cudaError_t e = wf::launch_fuse_exact_strip<T>(
          kind, pan, pan_pitch, strip ? pan_top : nullptr, strip ? pan_bot : nullptr, halo_pitch,
          ms, strip ? ms_top : nullptr, ms_pitch, out, out_pitch, nbands, rows, w, s);
      if (e != cudaSuccess) return cuda_status(e, "exact fuse launch");
      g_launches += (nbands + wf::kMaxBandsPerLaunch - 1) / wf::kMaxBandsPerLaunch;
      return WF_OK;
    }
  }

  const int vw = 16 / (int)sizeof(T);  // elements per 16 B
  bool vec = al16(pan) && pan_pitch % vw == 0 && out_pitch % vw == 0 && ms_pitch % 2 == 0;
  if (kind == WF_HAAR) vec = vec && (w % (sizeof(T) == 1 ? 16 : 4) == 0);
  // bulk-copy halo pieces are 16 bytes: 4 elements (f32/f64 use >= 4), 16 for u8
  const int halo = 16 / (int)sizeof(T) >= 4 ? 16 / (int)sizeof(T) : 4;
  for (int b = 0; b < nbands; ++b) {
    if (!ms[b] || !out[b]) return fail(WF_ERR_VALUE, "null band pointer %d", b);
    vec = vec && al16(out[b]) && al16(ms[b]);
  }

  const wf::LaunchTuning& tune = wf::env_tuning();
  const bool allow_tma = !tune.d4_ldg;
  auto row16 = [](int64_t pitch) { return (pitch * (int64_t)sizeof(T)) % 16 == 0; };

  for (int b0 = 0; b0 < nbands; b0 += wf::kMaxBandsPerLaunch) {
    const int nb = nbands - b0 < wf::kMaxBandsPerLaunch ? nbands - b0 : wf::kMaxBandsPerLaunch;
    wf::FuseArgs<T> a;
    memset(&a, 0, sizeof a);
    a.pan = pan;
    a.pan_pitch = pan_pitch;
    a.ms_pitch = ms_pitch;
    a.out_pitch = out_pitch;
    a.nbands = nb;
    a.rows = rows;
    a.W = w;
    if (kind == WF_DAUB4) {
      if (strip) {
        a.pan_top = pan_top;
        a.pan_bot = pan_bot;
        a.halo_pitch = halo_pitch;
        vec = vec && al16(pan_top) && al16(pan_bot) && halo_pitch % vw == 0;
      } else {  // periodic wrap of the whole image (wavelet.py:83-84)
        a.pan_top = pan + (int64_t)(rows - 2) * pan_pitch;
        a.pan_bot = pan;
        a.halo_pitch = pan_pitch;
      }
    }
    for (int b = 0; b < nb; ++b) {
      a.ms[b] = ms[b0 + b];
      a.out[b] = out[b0 + b];
      if (kind == WF_DAUB4)
        a.ms_top[b] = strip ? ms_top[b0 + b]
                            : ms[b0 + b] + (int64_t)(rows / 2 - 1) * ms_pitch;
    }
    // float64: 256-bit row accesses when every row start is 32-byte aligned
    if (sizeof(T) == 8 && vec && !tune.no_wide) {
      bool w32 = al32(pan) && (pan_pitch * 8) % 32 == 0 && (out_pitch * 8) % 32 == 0;
      for (int b = 0; b < nb && w32; ++b) w32 = al32(a.out[b]);
      a.wide = w32 ? 1 : 0;
    }
    bool tma = (allow_tma || sizeof(T) == 1) && kind == WF_DAUB4 && vec && w % (2 * halo) == 0 &&
               row16(pan_pitch) && row16(ms_pitch) && row16(a.halo_pitch) && al16(a.pan_top) &&
               al16(a.pan_bot);
    for (int b = 0; b < nb && tma; ++b) tma = al16(a.ms_top[b]);
    if (sizeof(T) == 1 && !(kind == WF_DAUB4 ? tma : vec))
      return fail(WF_ERR_VALUE,
                  "8 bpp kernels need W %% %d == 0 and 16-byte aligned rows (got W=%d)",
                  kind == WF_DAUB4 ? 2 * halo : 16, w);
    using Acc = typename std::conditional<sizeof(T) == 1, float, T>::type;
    cudaError_t e = wf::launch_fuse<T, Acc>(kind, a, vec, tma, s, tune);
    if (e != cudaSuccess) return cuda_status(e, "fuse launch");
    ++g_launches;

  }
  return WF_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline (wf_fuse_host_*): rows are cut into strips; each
// strip's PAN rows, its D4 halo rows and its MS rows go up, the strip kernel
// runs, the fused rows come back. Three slots rotate over three streams, so
// the H2D of strip k+1, the kernel of strip k and the D2H of strip k-1
// overlap (PCIe copy engines are full-duplex).
//  * pinned caller buffers (cudaHostAlloc / cudaHostRegister / torch
//    pin_memory): DMA straight from/to them;
//  * pageable caller buffers (plain numpy): each slot owns a pinned staging
//    buffer with the device slot's layout; the calling thread memcpy's strip
//    k+3's inputs in and strip k's outputs out while the GPU works on the
//    strips in between, so CPU copies, DMA and compute overlap and
//    concurrent callers (one context each) scale instead of serialising on
//    the driver's pageable-copy path.
// ---------------------------------------------------------------------------
constexpr int kSlots = 3;

// Host-side copy workers for the pageable staging path: a strip's piece
// copies are cut into ~2 MiB chunks that the caller and N persistent
// workers drain together (first-touch page faults of fresh numpy outputs and
// the copies themselves then use several cores instead of one).
class CopyPool {
 public:
  struct Chunk {
    void* dst;
    const void* src;
    size_t bytes;
  };
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(const std::vector<Chunk>& pieces) {
    std::vector<Chunk> work;
    constexpr size_t kGrain = 2u << 20;
    for (const Chunk& c : pieces)
      for (size_t o = 0; o < c.bytes; o += kGrain)
        work.push_back({static_cast<char*>(c.dst) + o, static_cast<const char*>(c.src) + o,
                        c.bytes - o < kGrain ? c.bytes - o : kGrain});
    if (th_.empty() || work.size() < 2) {
      for (const Chunk& c : work) memcpy(c.dst, c.src, c.bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &work;
      next_ = 0;
      active_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain(work);
    std::unique_lock<std::mutex> g(m_);
    done_cv_.wait(g, [this] { return active_ == 0; });
    job_ = nullptr;
  }

 private:
  void drain(const std::vector<Chunk>& w) {
    for (size_t i = next_.fetch_add(1); i < w.size(); i = next_.fetch_add(1))
      memcpy(w[i].dst, w[i].src, w[i].bytes);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::vector<Chunk>* job;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      drain(*job);
      std::lock_guard<std::mutex> g(m_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::vector<Chunk>* job_ = nullptr;
  std::atomic<size_t> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Copy workers for pageable callers: all cores this process may run on but
// one, up to 16 (tools/dbg/sweep_copy_threads.sh on a 16-core host: 2 -> 366,
// 8 -> 800, 15 -> 927 scene-MPix/s for a numpy Landsat scene; host memcpy is
// the bound).
int copy_threads() {
  if (const char* e = getenv("WF_HOST_COPY_THREADS")) return atoi(e) > 0 ? atoi(e) : 0;
  int hw = (int)std::thread::hardware_concurrency();
  cpu_set_t set;
  if (sched_getaffinity(0, sizeof set, &set) == 0) hw = CPU_COUNT(&set);
  const int n = hw >= 4 ? hw - 1 : 0;
  return n > 16 ? 16 : n;
}

struct Slot {
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;  // the slot's last D2H has landed
  void* dbuf = nullptr;
  size_t bytes = 0;
  void* hbuf = nullptr;  // pinned staging (pageable callers only)
  size_t hbytes = 0;
  int pend_r0 = -1, pend_rows = 0;  // strip whose outputs wait in hbuf
};

}  // namespace

struct wf_ctx {
  int device = 0;
  int strip_rows = 512;
  int exact = 0;  // wf_ctx_set_exact: strips run the reference-exact kernels
  Slot slot[kSlots];
  std::unique_ptr<CopyPool> pool;  // created on first pageable call
};

namespace {

// Element offsets of one slot (identical for the device buffer and the pinned
// staging buffer).
struct SlotLayout {
  size_t pan, top, bot, ms[wf::kMaxBandsPerLaunch * 64], mst[wf::kMaxBandsPerLaunch * 64],
      out[wf::kMaxBandsPerLaunch * 64], total;
};

template <typename T>
SlotLayout slot_layout(int S, int w, int nbands) {
  auto up = [](size_t n) { return (n * sizeof(T) + 255) / 256 * 256 / sizeof(T); };
  SlotLayout L{};
  size_t o = 0;
  L.pan = o;
  o += up((size_t)S * w);
  L.top = o;
  o += up(2 * (size_t)w);
  L.bot = o;
  o += up(2 * (size_t)w);
  for (int b = 0; b < nbands; ++b) {
    L.ms[b] = o;
    o += up((size_t)(S / 2) * (w / 2));
    L.mst[b] = o;
    o += up((size_t)(w / 2));
  }
  for (int b = 0; b < nbands; ++b) {
    L.out[b] = o;
    o += up((size_t)S * w);
  }
  L.total = o;
  return L;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // plain pageable memory on some drivers reports an error
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Restores the calling thread's current device when a host-buffer call
// returns (the calls switch to the context's device; the caller -- e.g. torch
// on another GPU of the same process -- must not see that switch).
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      dev = -1;
    }
  }
  ~DeviceGuard() {
    if (dev >= 0) cudaSetDevice(dev);
  }
};

// After a failed host-buffer call: wait for every copy and kernel already
// queued on the context's streams (they may still read or write the caller's
// buffers, which the caller frees once the error is raised) and forget the
// pending staged outputs.
void quiesce(wf_ctx* ctx) {
  for (int k = 0; k < kSlots; ++k) {
    if (ctx->slot[k].stream) cudaStreamSynchronize(ctx->slot[k].stream);
    ctx->slot[k].pend_r0 = -1;
  }
  cudaGetLastError();
}

template <typename T>
int fuse_host_impl(wf_ctx* ctx, int kind, const T* pan, const T* const* ms, T* const* out,
                   int nbands, int h, int w);

template <typename T>
int fuse_host(wf_ctx* ctx, int kind, const T* pan, const T* const* ms, T* const* out,
              int nbands, int h, int w) {
  DeviceGuard guard;
  const int rc = fuse_host_impl<T>(ctx, kind, pan, ms, out, nbands, h, w);
  if (rc != WF_OK && ctx) {
    const std::string msg = g_err;  // quiesce must not replace the first error
    quiesce(ctx);
    g_err = msg;
  }
  return rc;
}

template <typename T>
int fuse_host_impl(wf_ctx* ctx, int kind, const T* pan, const T* const* ms, T* const* out,
                   int nbands, int h, int w) {
  if (!ctx) return fail(WF_ERR_VALUE, "null context");
  if (int e = check_kind(kind)) return e;
  if (nbands < 1) return fail(WF_ERR_BAND_COUNT, "need at least one band");
  if (nbands > (int)(sizeof(SlotLayout::ms) / sizeof(size_t)))
    return fail(WF_ERR_BAND_COUNT, "too many bands (%d)", nbands);
  if (!pan || !ms || !out) return fail(WF_ERR_VALUE, "null pointer argument");
  if ((h & 1) || (w & 1))
    return fail(WF_ERR_ODD_DIMENSION, "panchromatic plane %dx%d has an odd dimension", w, h);
  if (h < min_len(kind) || w < min_len(kind))
    return fail(WF_ERR_TOO_SMALL, "%dx%d below minimum %d per side", w, h, min_len(kind));
  if (cudaError_t e = cudaSetDevice(ctx->device)) return cuda_status(e, "cudaSetDevice");

  bool pinned = is_pinned(pan);
  for (int b = 0; b < nbands && pinned; ++b) pinned = is_pinned(ms[b]) && is_pinned(out[b]);

  if (!pinned && !ctx->pool) ctx->pool.reset(new CopyPool(copy_threads()));
  int S = ctx->strip_rows;
  if (S > h) S = h;
  const int wh = w / 2;
  const SlotLayout L = slot_layout<T>(S, w, nbands);
  const size_t need = L.total * sizeof(T);
  for (int k = 0; k < kSlots; ++k) {
    Slot& sl = ctx->slot[k];
    if (sl.bytes < need) {
      if (sl.dbuf) cudaFree(sl.dbuf);
      sl.dbuf = nullptr;
      sl.bytes = 0;
      if (cudaError_t e = cudaMalloc(&sl.dbuf, need)) return cuda_status(e, "cudaMalloc slot");
      sl.bytes = need;
    }
    if (!pinned && sl.hbytes < need) {
      if (sl.hbuf) cudaFreeHost(sl.hbuf);
      sl.hbuf = nullptr;
      sl.hbytes = 0;
      if (cudaError_t e = cudaHostAlloc(&sl.hbuf, need, cudaHostAllocPortable))
        return cuda_status(e, "cudaHostAlloc staging");
      sl.hbytes = need;
    }
    sl.pend_r0 = -1;
  }

  // copy the finished outputs of a slot from its staging buffer to the caller
  auto drain = [&](Slot& sl) -> int {
    if (sl.pend_r0 < 0) return WF_OK;
    if (cudaError_t e = cudaEventSynchronize(sl.done)) return cuda_status(e, "event sync");
    const T* hb = static_cast<const T*>(sl.hbuf);
    std::vector<CopyPool::Chunk> cp;
    for (int b = 0; b < nbands; ++b)
      cp.push_back({out[b] + (size_t)sl.pend_r0 * w, hb + L.out[b],
                    sizeof(T) * (size_t)sl.pend_rows * w});
    ctx->pool->copy(cp);
    sl.pend_r0 = -1;
    return WF_OK;
  };

  std::vector<const T*> dms(nbands), dmst(nbands);
  std::vector<T*> dout(nbands);
  int k = 0;
  for (int r0 = 0; r0 < h; r0 += S, k = (k + 1) % kSlots) {
    const int rows = (h - r0) < S ? (h - r0) : S;
    Slot& sl = ctx->slot[k];
    cudaStream_t st = sl.stream;
    T* dbase = static_cast<T*>(sl.dbuf);
    T* hbase = static_cast<T*>(sl.hbuf);
    for (int b = 0; b < nbands; ++b) {
      dms[b] = dbase + L.ms[b];
      dmst[b] = dbase + L.mst[b];
      dout[b] = dbase + L.out[b];
    }
    // input pieces: (slot offset, source, elements)
    struct Piece {
      size_t off;
      const T* src;
      size_t n;
    };
    std::vector<Piece> pieces;
    pieces.push_back({L.pan, pan + (size_t)r0 * w, (size_t)rows * w});
    if (kind == WF_DAUB4) {
      for (int q = 0; q < 2; ++q) {
        const int rt = (r0 - 2 + q + h) % h, rb = (r0 + rows + q) % h;
        pieces.push_back({L.top + (size_t)q * w, pan + (size_t)rt * w, (size_t)w});
        pieces.push_back({L.bot + (size_t)q * w, pan + (size_t)rb * w, (size_t)w});
      }
    }
    for (int b = 0; b < nbands; ++b) {
      pieces.push_back({L.ms[b], ms[b] + (size_t)(r0 / 2) * wh, (size_t)(rows / 2) * wh});
      if (kind == WF_DAUB4) {
        const int mt = (r0 / 2 - 1 + h / 2) % (h / 2);
        pieces.push_back({L.mst[b], ms[b] + (size_t)mt * wh, (size_t)wh});
      }
    }
    cudaError_t e = cudaSuccess;
    if (pinned) {
      for (const Piece& pc : pieces)
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(dbase + pc.off, pc.src, sizeof(T) * pc.n, cudaMemcpyHostToDevice,
                              st);
    } else {
      // the slot's previous strip has fully completed once its outputs are
      // drained (H2D -> kernel -> D2H are ordered on the slot's stream)
      if (int rc = drain(sl)) return rc;
      std::vector<CopyPool::Chunk> cp;
      for (const Piece& pc : pieces) cp.push_back({hbase + pc.off, pc.src, sizeof(T) * pc.n});
      ctx->pool->copy(cp);
      for (const Piece& pc : pieces)
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(dbase + pc.off, hbase + pc.off, sizeof(T) * pc.n,
                              cudaMemcpyHostToDevice, st);
    }
    if (e != cudaSuccess) return cuda_status(e, "H2D");
    if (int rc = fuse_common<T>(kind, dbase + L.pan, w, dbase + L.top, dbase + L.bot, w,
                                dms.data(), dmst.data(), wh, dout.data(), w, nbands, rows, w,
                                true, st, ctx->exact != 0))
      return rc;
    for (int b = 0; b < nbands && e == cudaSuccess; ++b) {
      T* dst = pinned ? out[b] + (size_t)r0 * w : hbase + L.out[b];
      e = cudaMemcpyAsync(dst, dout[b], sizeof(T) * (size_t)rows * w, cudaMemcpyDeviceToHost, st);
    }
    if (e != cudaSuccess) return cuda_status(e, "D2H");
    if (!pinned) {
      if ((e = cudaEventRecord(sl.done, st)) != cudaSuccess) return cuda_status(e, "event");
      sl.pend_r0 = r0;
      sl.pend_rows = rows;
    }
  }
  for (int q = 0; q < kSlots; ++q) {
    if (int rc = drain(ctx->slot[q])) return rc;
    if (cudaError_t e = cudaStreamSynchronize(ctx->slot[q].stream))
      return cuda_status(e, "stream sync");
  }
  return WF_OK;
}

// wf_check_selftest: one WF_CHECK that fails at run time (x is 0); in a
// checked build it traps, which proves the invariants are compiled in
__global__ void check_selftest_kernel(int x) { WF_CHECK(x == 1); }

}  // namespace

extern "C" {

const char* wf_version(void) { return "wavefuse-b200 0.2.0 (sm_100a)"; }
int wf_checked_build(void) { return wf::kCheckTagBytesPerSlot > 0 ? 1 : 0; }
int wf_check_selftest(void) {
  check_selftest_kernel<<<1, 1>>>(0);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? WF_OK : cuda_status(e, "check selftest");
}
int wf_tuning_reload(void) {
  wf::g_tuning = wf::read_tuning();
  return WF_OK;
}
const char* wf_last_error(void) { return g_err.c_str(); }
int64_t wf_launch_count(void) { return g_launches; }

int wf_fuse_dwt_f32(int kind, const float* pan, int64_t pan_pitch, const float* ms,
                    int64_t ms_pitch, float* out, int64_t out_pitch, int h, int w,
                    void* stream) {
  return fuse_common<float>(kind, pan, pan_pitch, nullptr, nullptr, 0, &ms, nullptr, ms_pitch,
                            &out, out_pitch, 1, h, w, false, (cudaStream_t)stream);
}
int wf_fuse_dwt_f64(int kind, const double* pan, int64_t pan_pitch, const double* ms,
                    int64_t ms_pitch, double* out, int64_t out_pitch, int h, int w,
                    void* stream) {
  return fuse_common<double>(kind, pan, pan_pitch, nullptr, nullptr, 0, &ms, nullptr, ms_pitch,
                             &out, out_pitch, 1, h, w, false, (cudaStream_t)stream);
}
int wf_fuse_bands_f32(int kind, const float* pan, int64_t pan_pitch, const float* const* ms,
                      int64_t ms_pitch, float* const* out, int64_t out_pitch, int nbands, int h,
                      int w, void* stream) {
  return fuse_common<float>(kind, pan, pan_pitch, nullptr, nullptr, 0, ms, nullptr, ms_pitch,
                            out, out_pitch, nbands, h, w, false, (cudaStream_t)stream);
}
int wf_fuse_bands_f64(int kind, const double* pan, int64_t pan_pitch, const double* const* ms,
                      int64_t ms_pitch, double* const* out, int64_t out_pitch, int nbands, int h,
                      int w, void* stream) {
  return fuse_common<double>(kind, pan, pan_pitch, nullptr, nullptr, 0, ms, nullptr, ms_pitch,
                             out, out_pitch, nbands, h, w, false, (cudaStream_t)stream);
}
int wf_fuse_strip_f32(int kind, const float* pan, int64_t pan_pitch, const float* pan_top,
                      const float* pan_bot, int64_t halo_pitch, const float* const* ms,
                      const float* const* ms_top, int64_t ms_pitch, float* const* out,
                      int64_t out_pitch, int nbands, int rows, int w, void* stream) {
  return fuse_common<float>(kind, pan, pan_pitch, pan_top, pan_bot, halo_pitch, ms, ms_top,
                            ms_pitch, out, out_pitch, nbands, rows, w, true,
                            (cudaStream_t)stream);
}
int wf_fuse_strip_f64(int kind, const double* pan, int64_t pan_pitch, const double* pan_top,
                      const double* pan_bot, int64_t halo_pitch, const double* const* ms,
                      const double* const* ms_top, int64_t ms_pitch, double* const* out,
                      int64_t out_pitch, int nbands, int rows, int w, void* stream) {
  return fuse_common<double>(kind, pan, pan_pitch, pan_top, pan_bot, halo_pitch, ms, ms_top,
                             ms_pitch, out, out_pitch, nbands, rows, w, true,
                             (cudaStream_t)stream);
}
int wf_fuse_strip_exact_f32(int kind, const float* pan, int64_t pan_pitch, const float* pan_top,
                            const float* pan_bot, int64_t halo_pitch, const float* const* ms,
                            const float* const* ms_top, int64_t ms_pitch, float* const* out,
                            int64_t out_pitch, int nbands, int rows, int w, void* stream) {
  return fuse_common<float>(kind, pan, pan_pitch, pan_top, pan_bot, halo_pitch, ms, ms_top,
                            ms_pitch, out, out_pitch, nbands, rows, w, true,
                            (cudaStream_t)stream, true);
}
int wf_fuse_strip_exact_f64(int kind, const double* pan, int64_t pan_pitch,
                            const double* pan_top, const double* pan_bot, int64_t halo_pitch,
                            const double* const* ms, const double* const* ms_top,
                            int64_t ms_pitch, double* const* out, int64_t out_pitch, int nbands,
                            int rows, int w, void* stream) {
  return fuse_common<double>(kind, pan, pan_pitch, pan_top, pan_bot, halo_pitch, ms, ms_top,
                             ms_pitch, out, out_pitch, nbands, rows, w, true,
                             (cudaStream_t)stream, true);
}

// Host -> device copy of a (pageable) host buffer through the context's
// pinned staging slots: 32 MiB chunks, the copy workers filling one slot while
// the DMA of the previous ones runs (torch's pageable .to(device) moves ~11
// GB/s; this path runs at the host-memcpy / PCIe rate). `after` = the stream
// whose earlier work must complete before `dst` is written (the allocating
// stream). Returns when the data is on the device.
static int ctx_upload(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after);
static int ctx_download(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after);

int wf_ctx_upload(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after) {
  DeviceGuard guard;
  const int rc = ctx_upload(ctx, dst, src, bytes, after);
  if (rc != WF_OK && ctx) {
    const std::string msg = g_err;
    quiesce(ctx);
    g_err = msg;
  }
  return rc;
}
int wf_ctx_download(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after) {
  DeviceGuard guard;
  const int rc = ctx_download(ctx, dst, src, bytes, after);
  if (rc != WF_OK && ctx) {
    const std::string msg = g_err;
    quiesce(ctx);
    g_err = msg;
  }
  return rc;
}

static int ctx_upload(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after) {
  if (!ctx) return fail(WF_ERR_VALUE, "null context");
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(WF_ERR_VALUE, "bad upload arguments");
  if (bytes == 0) return WF_OK;
  if (cudaError_t e = cudaSetDevice(ctx->device)) return cuda_status(e, "cudaSetDevice");
  if (cudaError_t e = cudaStreamSynchronize((cudaStream_t)after)) return cuda_status(e, "sync");
  if (is_pinned(src)) {
    cudaStream_t st = ctx->slot[0].stream;
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return cuda_status(e, "upload");
  }
  if (!ctx->pool) ctx->pool.reset(new CopyPool(copy_threads()));
  constexpr size_t kChunk = 32u << 20;
  for (int k = 0; k < kSlots; ++k) {
    Slot& sl = ctx->slot[k];
    if (sl.hbytes < kChunk) {
      if (sl.hbuf) cudaFreeHost(sl.hbuf);
      sl.hbuf = nullptr;
      sl.hbytes = 0;
      if (cudaError_t e = cudaHostAlloc(&sl.hbuf, kChunk, cudaHostAllocPortable))
        return cuda_status(e, "cudaHostAlloc staging");
      sl.hbytes = kChunk;
    }
    sl.pend_r0 = -1;
  }
  cudaError_t e = cudaSuccess;
  int k = 0;
  for (size_t off = 0; off < (size_t)bytes && e == cudaSuccess; off += kChunk, k = (k + 1) % kSlots) {
    Slot& sl = ctx->slot[k];
    const size_t n = (size_t)bytes - off < kChunk ? (size_t)bytes - off : kChunk;
    e = cudaEventSynchronize(sl.done);  // the slot's previous DMA has read its staging
    if (e != cudaSuccess) break;
    ctx->pool->copy({{sl.hbuf, static_cast<const char*>(src) + off, n}});
    e = cudaMemcpyAsync(static_cast<char*>(dst) + off, sl.hbuf, n, cudaMemcpyHostToDevice,
                        sl.stream);
    if (e == cudaSuccess) e = cudaEventRecord(sl.done, sl.stream);
  }
  for (int j = 0; j < kSlots && e == cudaSuccess; ++j) e = cudaStreamSynchronize(ctx->slot[j].stream);
  return cuda_status(e, "upload");
}

// Device -> host counterpart: up to kSlots 32 MiB DMAs in flight into the
// pinned staging while the copy workers move finished chunks to `dst`.
// `after` = the stream that produced src. Synchronous.
static int ctx_download(wf_ctx* ctx, void* dst, const void* src, int64_t bytes, void* after) {
  if (!ctx) return fail(WF_ERR_VALUE, "null context");
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(WF_ERR_VALUE, "bad download arguments");
  if (bytes == 0) return WF_OK;
  if (cudaError_t e = cudaSetDevice(ctx->device)) return cuda_status(e, "cudaSetDevice");
  if (cudaError_t e = cudaStreamSynchronize((cudaStream_t)after)) return cuda_status(e, "sync");
  if (is_pinned(dst)) {
    cudaStream_t st = ctx->slot[0].stream;
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return cuda_status(e, "download");
  }
  if (!ctx->pool) ctx->pool.reset(new CopyPool(copy_threads()));
  constexpr size_t kChunk = 32u << 20;
  for (int k = 0; k < kSlots; ++k) {
    Slot& sl = ctx->slot[k];
    if (sl.hbytes < kChunk) {
      if (sl.hbuf) cudaFreeHost(sl.hbuf);
      sl.hbuf = nullptr;
      sl.hbytes = 0;
      if (cudaError_t e = cudaHostAlloc(&sl.hbuf, kChunk, cudaHostAllocPortable))
        return cuda_status(e, "cudaHostAlloc staging");
      sl.hbytes = kChunk;
    }
    sl.pend_r0 = -1;
  }
  const size_t total = (size_t)bytes, nchunks = (total + kChunk - 1) / kChunk;
  auto len = [&](size_t c) { return total - c * kChunk < kChunk ? total - c * kChunk : kChunk; };
  cudaError_t e = cudaSuccess;
  auto issue = [&](size_t c) {
    Slot& sl = ctx->slot[c % kSlots];
    e = cudaMemcpyAsync(sl.hbuf, static_cast<const char*>(src) + c * kChunk, len(c),
                        cudaMemcpyDeviceToHost, sl.stream);
    if (e == cudaSuccess) e = cudaEventRecord(sl.done, sl.stream);
  };
  for (size_t c = 0; c < nchunks && c < (size_t)kSlots && e == cudaSuccess; ++c) issue(c);
  for (size_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    Slot& sl = ctx->slot[c % kSlots];
    e = cudaEventSynchronize(sl.done);
    if (e != cudaSuccess) break;
    ctx->pool->copy({{static_cast<char*>(dst) + c * kChunk, sl.hbuf, len(c)}});
    if (c + kSlots < nchunks) issue(c + kSlots);
  }
  return cuda_status(e, "download");
}

int wf_ctx_set_exact(wf_ctx* ctx, int exact) {
  if (!ctx) return fail(WF_ERR_VALUE, "null context");
  ctx->exact = exact ? 1 : 0;
  return WF_OK;
}

wf_ctx* wf_ctx_create(int device, int strip_rows) {
  DeviceGuard guard;
  if (cudaError_t e = cudaSetDevice(device)) {
    cuda_status(e, "cudaSetDevice");
    return nullptr;
  }
  wf_ctx* c = new wf_ctx;
  c->device = device;
  if (strip_rows > 0) c->strip_rows = strip_rows & ~1;
  if (c->strip_rows < 2) c->strip_rows = 2;
  for (int k = 0; k < kSlots; ++k) {
    cudaError_t e = cudaStreamCreateWithFlags(&c->slot[k].stream, cudaStreamNonBlocking);
    if (e == cudaSuccess)
      e = cudaEventCreateWithFlags(&c->slot[k].done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      cuda_status(e, "cudaStreamCreate");
      wf_ctx_destroy(c);
      return nullptr;
    }
  }
  return c;
}

void wf_ctx_destroy(wf_ctx* c) {
  if (!c) return;
  DeviceGuard guard;
  cudaSetDevice(c->device);
  for (int k = 0; k < kSlots; ++k) {
    if (c->slot[k].stream) {
      cudaStreamSynchronize(c->slot[k].stream);
      cudaStreamDestroy(c->slot[k].stream);
    }
    if (c->slot[k].done) cudaEventDestroy(c->slot[k].done);
    if (c->slot[k].dbuf) cudaFree(c->slot[k].dbuf);
    if (c->slot[k].hbuf) cudaFreeHost(c->slot[k].hbuf);
  }
  delete c;
}

int wf_fuse_host_f32(wf_ctx* ctx, int kind, const float* pan, const float* const* ms,
                     float* const* out, int nbands, int h, int w) {
  return fuse_host<float>(ctx, kind, pan, ms, out, nbands, h, w);
}
int wf_fuse_host_f64(wf_ctx* ctx, int kind, const double* pan, const double* const* ms,
                     double* const* out, int nbands, int h, int w) {
  return fuse_host<double>(ctx, kind, pan, ms, out, nbands, h, w);
}

int wf_fuse_bands_u8(int kind, const uint8_t* pan, int64_t pan_pitch, const uint8_t* const* ms,
                     int64_t ms_pitch, uint8_t* const* out, int64_t out_pitch, int nbands, int h,
                     int w, void* stream) {
  return fuse_common<uint8_t>(kind, pan, pan_pitch, nullptr, nullptr, 0, ms, nullptr, ms_pitch,
                              out, out_pitch, nbands, h, w, false, (cudaStream_t)stream);
}
int wf_fuse_strip_u8(int kind, const uint8_t* pan, int64_t pan_pitch, const uint8_t* pan_top,
                     const uint8_t* pan_bot, int64_t halo_pitch, const uint8_t* const* ms,
                     const uint8_t* const* ms_top, int64_t ms_pitch, uint8_t* const* out,
                     int64_t out_pitch, int nbands, int rows, int w, void* stream) {
  return fuse_common<uint8_t>(kind, pan, pan_pitch, pan_top, pan_bot, halo_pitch, ms, ms_top,
                              ms_pitch, out, out_pitch, nbands, rows, w, true,
                              (cudaStream_t)stream);
}
int wf_fuse_host_u8(wf_ctx* ctx, int kind, const uint8_t* pan, const uint8_t* const* ms,
                    uint8_t* const* out, int nbands, int h, int w) {
  return fuse_host<uint8_t>(ctx, kind, pan, ms, out, nbands, h, w);
}

int wf_u8_to_f32(const uint8_t* in, int64_t in_pitch, int h, int w, float* out,
                 int64_t out_pitch, void* stream) {
  if (!in || !out || h < 0 || w < 0) return fail(WF_ERR_VALUE, "bad conversion arguments");
  if (h == 0 || w == 0) return WF_OK;
  cudaError_t e = wf::launch_u8_to_f32(in, in_pitch, h, w, out, out_pitch, (cudaStream_t)stream);
  if (e == cudaSuccess) ++g_launches;
  return cuda_status(e, "wf_u8_to_f32");
}

#define WF_QUANTIZE(NAME, T)                                                                 \
  int NAME(const T* in, int64_t in_pitch, int h, int w, uint8_t* out, int64_t out_pitch,      \
           void* stream) {                                                                   \
    if (!in || !out || h < 0 || w < 0) return fail(WF_ERR_VALUE, "bad quantize arguments"); \
    if (h == 0 || w == 0) return WF_OK;                                                      \
    cudaError_t e = wf::launch_quantize<T>(in, in_pitch, h, w, out, out_pitch,              \
                                           (cudaStream_t)stream);                            \
    if (e == cudaSuccess) ++g_launches;                                                      \
    return cuda_status(e, #NAME);                                                            \
  }
WF_QUANTIZE(wf_quantize_f32, float)
WF_QUANTIZE(wf_quantize_f64, double)

// ---- PNM front end (raster.cu) ----------------------------------------------
#define WF_RASTER_TO_PLANE(NAME, T)                                                           \
  int NAME(const uint8_t* raster, int h, int w, int channels, int channel, T* out,             \
           int64_t out_pitch, int out_h, int out_w, void* stream) {                            \
    if (h < 1 || w < 1 || channels < 1) return fail(WF_ERR_VALUE, "empty raster");            \
    if (channel < 0 || channel >= channels)                                                    \
      return fail(WF_ERR_CHANNEL, "channel %d of %d", channel, channels);                     \
    if (out_w < w || out_h < h)                                                                \
      return fail(WF_ERR_VALUE, "cannot pad %dx%d down to %dx%d", w, h, out_w, out_h);        \
    if (!raster || !out || out_pitch < out_w) return fail(WF_ERR_VALUE, "bad plane arguments"); \
    cudaError_t e = wf::launch_raster_to_plane<T>(raster, h, w, channels, channel, out,        \
                                                  out_pitch, out_h, out_w, (cudaStream_t)stream); \
    if (e == cudaSuccess) ++g_launches;                                                        \
    return cuda_status(e, #NAME);                                                              \
  }
WF_RASTER_TO_PLANE(wf_raster_to_plane_f32, float)
WF_RASTER_TO_PLANE(wf_raster_to_plane_f64, double)

#define WF_PAD_EDGE(NAME, T)                                                                   \
  int NAME(const T* in, int64_t in_pitch, int h, int w, T* out, int64_t out_pitch, int out_h,  \
           int out_w, void* stream) {                                                          \
    if (h < 1 || w < 1) return fail(WF_ERR_VALUE, "empty plane");                             \
    if (out_w < w || out_h < h)                                                                \
      return fail(WF_ERR_VALUE, "cannot pad %dx%d down to %dx%d", w, h, out_w, out_h);        \
    if (!in || !out || in_pitch < w || out_pitch < out_w)                                      \
      return fail(WF_ERR_VALUE, "bad plane arguments");                                       \
    cudaError_t e = wf::launch_pad_edge<T>(in, in_pitch, h, w, out, out_pitch, out_h, out_w,   \
                                           (cudaStream_t)stream);                              \
    if (e == cudaSuccess) ++g_launches;                                                        \
    return cuda_status(e, #NAME);                                                              \
  }
WF_PAD_EDGE(wf_pad_edge_f32, float)
WF_PAD_EDGE(wf_pad_edge_f64, double)

#define WF_PLANES_TO_RASTER(NAME, T)                                                           \
  int NAME(const T* const* planes, int nplanes, int64_t pitch, int h, int w, uint8_t* raster,  \
           void* stream) {                                                                     \
    if (nplanes < 1 || nplanes > wf::kMaxRasterPlanes)                                         \
      return fail(WF_ERR_VALUE, "%d planes (1..%d)", nplanes, wf::kMaxRasterPlanes);          \
    if (h < 1 || w < 1) return fail(WF_ERR_VALUE, "empty raster");                            \
    if (!planes || !raster || pitch < w) return fail(WF_ERR_VALUE, "bad raster arguments");   \
    for (int k = 0; k < nplanes; ++k)                                                          \
      if (!planes[k]) return fail(WF_ERR_VALUE, "null plane pointer %d", k);                  \
    cudaError_t e = wf::launch_planes_to_raster<T>(planes, nplanes, pitch, h, w, raster,       \
                                                   (cudaStream_t)stream);                      \
    if (e == cudaSuccess) ++g_launches;                                                        \
    return cuda_status(e, #NAME);                                                              \
  }
WF_PLANES_TO_RASTER(wf_planes_to_raster_f32, float)
WF_PLANES_TO_RASTER(wf_planes_to_raster_f64, double)

#define WF_DWT2D(NAME, T, INV)                                                               \
  int NAME(int kind, const T* in, int64_t in_pitch, T* out, int64_t out_pitch, int h, int w, \
           void* stream) {                                                                   \
    if (int e = check_2d(kind, h, w)) return e;                                              \
    if (!in || !out) return fail(WF_ERR_VALUE, "null pointer argument");                     \
    cudaError_t e = wf::launch_dwt2d<T>(kind, INV, in, in_pitch, out, out_pitch, h, w,       \
                                        (cudaStream_t)stream);                               \
    if (e == cudaSuccess) ++g_launches;                                                      \
    return cuda_status(e, #NAME);                                                            \
  }
WF_DWT2D(wf_dwt2d_forward_f32, float, false)
WF_DWT2D(wf_dwt2d_forward_f64, double, false)
WF_DWT2D(wf_dwt2d_inverse_f32, float, true)
WF_DWT2D(wf_dwt2d_inverse_f64, double, true)

#define WF_ROWS(NAME, T, INV)                                                              \
  int NAME(int kind, const T* in, int64_t in_pitch, T* out, int64_t out_pitch, int nrows, \
           int n, void* stream) {                                                          \
    if (int e = check_1d(kind, n)) return e;                                               \
    if (nrows < 1) return fail(WF_ERR_VALUE, "nrows must be positive");                    \
    if (!in || !out) return fail(WF_ERR_VALUE, "null pointer argument");                   \
    cudaError_t e = wf::launch_dwt_rows<T>(kind, INV, in, in_pitch, out, out_pitch, nrows, \
                                           n, (cudaStream_t)stream);                       \
    if (e == cudaSuccess) ++g_launches;                                                    \
    return cuda_status(e, #NAME);                                                          \
  }
WF_ROWS(wf_dwt_rows_forward_f32, float, false)
WF_ROWS(wf_dwt_rows_forward_f64, double, false)
WF_ROWS(wf_dwt_rows_inverse_f32, float, true)
WF_ROWS(wf_dwt_rows_inverse_f64, double, true)

#define WF_RESAMPLE(NAME, T)                                                                 \
  int NAME(const T* in, int64_t in_pitch, int in_h, int in_w, T* out, int64_t out_pitch,    \
           int out_h, int out_w, void* stream) {                                            \
    if (out_w < 1 || out_h < 1)                                                             \
      return fail(WF_ERR_VALUE, "output size %dx%d must be positive", out_w, out_h);        \
    if (in_w < 1 || in_h < 1) return fail(WF_ERR_VALUE, "empty input plane");              \
    if (!in || !out) return fail(WF_ERR_VALUE, "null pointer argument");                    \
    cudaError_t e = wf::launch_resample<T, T>(in, in_pitch, in_h, in_w, out, out_pitch, out_h, \
                                           out_w, (cudaStream_t)stream);                    \
    if (e == cudaSuccess) ++g_launches;                                                     \
    return cuda_status(e, #NAME);                                                           \
  }
WF_RESAMPLE(wf_resample_bilinear_f32, float)
WF_RESAMPLE(wf_resample_bilinear_f64, double)

int wf_resample_bilinear_f32_to_f64(const float* in, int64_t in_pitch, int in_h, int in_w,
                                     double* out, int64_t out_pitch, int out_h, int out_w,
                                     void* stream) {
  if (out_w < 1 || out_h < 1)
    return fail(WF_ERR_VALUE, "output size %dx%d must be positive", out_w, out_h);
  if (in_w < 1 || in_h < 1) return fail(WF_ERR_VALUE, "empty input plane");
  if (!in || !out) return fail(WF_ERR_VALUE, "null pointer argument");
  cudaError_t e = wf::launch_resample<float, double>(in, in_pitch, in_h, in_w, out, out_pitch,
                                                     out_h, out_w, (cudaStream_t)stream);
  if (e == cudaSuccess) ++g_launches;
  return cuda_status(e, "wf_resample_bilinear_f32_to_f64");
}

int64_t wf_q_index_workspace_bytes(int h, int w) {
  int bh, bw, nbr, nbc;
  wf::q_geometry(h, w, bh, bw, nbr, nbc);
  return (int64_t)nbr * nbc * (int64_t)sizeof(double);
}

int wf_q_index(const void* a, int a_f64, int64_t a_pitch, const void* b, int b_f64,
               int64_t b_pitch, int h, int w, void* workspace, double* out, int out_index,
               void* stream) {
  if (!a || !b || !workspace || !out) return fail(WF_ERR_VALUE, "null pointer argument");
  if (h < 1 || w < 1) return fail(WF_ERR_VALUE, "empty plane %dx%d", w, h);
  cudaError_t e = wf::launch_q_index(a, a_f64, a_pitch, b, b_f64, b_pitch, h, w,
                                     static_cast<double*>(workspace), out, out_index,
                                     (cudaStream_t)stream);
  if (e == cudaSuccess) g_launches += 2;
  return cuda_status(e, "wf_q_index");
}

int wf_degrade(const void* in, int in_f64, int64_t in_pitch, int h, int w, int factor,
               double* out, int64_t out_pitch, void* stream) {
  if (factor < 1) return fail(WF_ERR_VALUE, "factor %d must be >= 1", factor);
  if (h % factor || w % factor)
    return fail(WF_ERR_NOT_DIVISIBLE, "%dx%d not divisible by %d", w, h, factor);
  if (!in || !out) return fail(WF_ERR_VALUE, "null pointer argument");
  if (h == 0 || w == 0) return WF_OK;
  cudaError_t e = wf::launch_degrade(in, in_f64, in_pitch, h, w, factor, out, out_pitch,
                                     (cudaStream_t)stream);
  if (e == cudaSuccess) ++g_launches;
  return cuda_status(e, "wf_degrade");
}

int64_t wf_ergas_workspace_bytes(int rh, int rw) {
  return 2 * (int64_t)wf::ergas_parts((long long)rh * rw) * (int64_t)sizeof(double);
}

int wf_ergas_band(const void* fused, int f_f64, int64_t f_pitch, const void* ref, int r_f64,
                  int64_t r_pitch, int rh, int rw, int ratio, void* workspace, double* out2,
                  void* stream) {
  if (!fused || !ref || !workspace || !out2) return fail(WF_ERR_VALUE, "null pointer argument");
  if (ratio < 1) return fail(WF_ERR_VALUE, "ratio %d must be >= 1", ratio);
  if (rh < 1 || rw < 1) return fail(WF_ERR_VALUE, "empty reference band");
  cudaError_t e = wf::launch_ergas_band(fused, f_f64, f_pitch, ref, r_f64, r_pitch, rh, rw,
                                        ratio, static_cast<double*>(workspace), out2,
                                        (cudaStream_t)stream);
  if (e == cudaSuccess) g_launches += 2;
  return cuda_status(e, "wf_ergas_band");
}

int64_t wf_quality_scene_workspace_bytes(int nbands, int h, int w) {
  return (int64_t)wf::quality_scene_workspace(nbands, h, w);
}

int wf_quality_scene_f32(const float* const* fused, const float* const* ms, const float* pan,
                         int64_t f_pitch, int64_t ms_pitch, int64_t pan_pitch, int nbands, int h,
                         int w, void* workspace, double* out, int* undecidable, void* stream) {
  if (!fused || !ms || !pan || !workspace || !out || !undecidable)
    return fail(WF_ERR_VALUE, "null pointer argument");
  if (nbands < 2 || nbands > wf::kMaxBandsPerLaunch)
    return fail(WF_ERR_BAND_COUNT, "fused quality path takes 2..%d bands, got %d",
                wf::kMaxBandsPerLaunch, nbands);
  if ((h & 1) || (w % 8) || h < 64 || w < 64)
    return fail(WF_ERR_VALUE, "fused quality path needs even H, W % 8 == 0, H, W >= 64 (got %dx%d)",
                w, h);
  auto row16 = [](int64_t pitch) { return (pitch * 4) % 16 == 0; };
  if (!row16(f_pitch) || !row16(pan_pitch) || !row16(ms_pitch) || !al16(pan) || f_pitch < w ||
      pan_pitch < w || ms_pitch < w / 2)
    return fail(WF_ERR_VALUE, "fused quality path needs 16-byte aligned rows");
  for (int b = 0; b < nbands; ++b) {
    if (!fused[b] || !ms[b]) return fail(WF_ERR_VALUE, "null band pointer %d", b);
    if (!al16(fused[b]) || !al16(ms[b]))
      return fail(WF_ERR_VALUE, "band %d not 16-byte aligned", b);
  }
  cudaError_t e = wf::launch_quality_scene(nbands, fused, ms, pan, f_pitch, ms_pitch, pan_pitch,
                                           h, w, workspace, out, undecidable,
                                           (cudaStream_t)stream);
  if (e == cudaSuccess) g_launches += 4;  // scene kernel, edge, two finish levels
  return cuda_status(e, "wf_quality_scene_f32");
}

int wf_quality_scene_f64(const double* const* fused, const double* const* ms, const double* pan,
                         int64_t f_pitch, int64_t ms_pitch, int64_t pan_pitch, int nbands, int h,
                         int w, void* workspace, double* out, int* undecidable, void* stream) {
  if (!fused || !ms || !pan || !workspace || !out || !undecidable)
    return fail(WF_ERR_VALUE, "null pointer argument");
  if (nbands < 2 || nbands > wf::kMaxBandsPerLaunch)
    return fail(WF_ERR_BAND_COUNT, "fused quality path takes 2..%d bands, got %d",
                wf::kMaxBandsPerLaunch, nbands);
  if ((h & 1) || (w % 8) || h < 64 || w < 64)
    return fail(WF_ERR_VALUE, "fused quality path needs even H, W % 8 == 0, H, W >= 64 (got %dx%d)",
                w, h);
  auto row16 = [](int64_t pitch) { return (pitch * 8) % 16 == 0; };
  if (!row16(f_pitch) || !row16(pan_pitch) || !al16(pan) || f_pitch < w || pan_pitch < w ||
      ms_pitch < w / 2 || f_pitch != pan_pitch)
    return fail(WF_ERR_VALUE, "float64 quality path needs 16-byte aligned rows and one pitch "
                              "for the fused bands and the PAN");
  for (int b = 0; b < nbands; ++b) {
    if (!fused[b] || !ms[b]) return fail(WF_ERR_VALUE, "null band pointer %d", b);
    if (!al16(fused[b])) return fail(WF_ERR_VALUE, "band %d not 16-byte aligned", b);
  }
  cudaError_t e = wf::launch_quality_scene64(nbands, fused, ms, pan, f_pitch, ms_pitch,
                                             pan_pitch, h, w, workspace, out, undecidable,
                                             (cudaStream_t)stream);
  if (e == cudaSuccess) g_launches += 4;  // scene kernel, edge, two finish levels
  return cuda_status(e, "wf_quality_scene_f64");
}

int wf_fuse_quality_f32(int kind, const float* pan, int64_t pan_pitch, const float* const* ms,
                        int64_t ms_pitch, float* const* out, int64_t out_pitch, int nbands, int h,
                        int w, void* workspace, double* report, int* undecidable, void* stream) {
  if (int e = check_kind(kind)) return e;
  if (!out || !ms || !pan || !workspace || !report || !undecidable)
    return fail(WF_ERR_VALUE, "null pointer argument");
  if (nbands < 2 || nbands > wf::kMaxBandsPerLaunch)
    return fail(WF_ERR_BAND_COUNT, "fused quality path takes 2..%d bands, got %d",
                wf::kMaxBandsPerLaunch, nbands);
  if ((h & 1) || (w % 8) || h < 64 || w < 64)
    return fail(WF_ERR_VALUE, "fused quality path needs even H, W % 8 == 0, H, W >= 64 (got %dx%d)",
                w, h);
  auto row16 = [](int64_t pitch) { return (pitch * 4) % 16 == 0; };
  if (!row16(out_pitch) || !row16(pan_pitch) || !row16(ms_pitch) || !al16(pan) ||
      out_pitch < w || pan_pitch < w || ms_pitch < w / 2)
    return fail(WF_ERR_VALUE, "fused quality path needs 16-byte aligned rows");
  for (int b = 0; b < nbands; ++b) {
    if (!out[b] || !ms[b]) return fail(WF_ERR_VALUE, "null band pointer %d", b);
    if (!al16(out[b]) || !al16(ms[b])) return fail(WF_ERR_VALUE, "band %d not 16-byte aligned", b);
  }
  // Haar: one pass (the report kernel forms the bands itself, 3.05 vs 3.20
  // ms for the two kernels); D4: the fusion kernel, then the report kernel on
  // its output (3.20 ms). WF_FQ_OVERLAP=1: the SM-partitioned overlap of the
  // two (either kind; measured 3.4-10 ms, profiles/r02_fq_overlap.log).
  const wf::LaunchTuning& tune = wf::env_tuning();
  cudaError_t e = cudaSuccess;
  if (tune.fq_overlap) {
    int launches = 0;
    e = wf::launch_fuse_quality_overlap(kind == WF_HAAR ? wf::kHaar : wf::kDaub4, nbands, pan,
                                        ms, out, out_pitch, ms_pitch, pan_pitch, h, w, workspace,
                                        report, undecidable, (cudaStream_t)stream, &launches);
    g_launches += launches;
  } else if (kind == WF_HAAR) {
    e = wf::launch_fuse_quality_haar(nbands, pan, ms, out, out_pitch, ms_pitch, pan_pitch, h, w,
                                     workspace, report, undecidable, (cudaStream_t)stream);
    if (e == cudaSuccess) g_launches += 6;
  } else {
    const float* const* cout = out;
    if (int rc = fuse_common<float>(kind, pan, pan_pitch, nullptr, nullptr, 0, ms, nullptr,
                                    ms_pitch, out, out_pitch, nbands, h, w, false,
                                    (cudaStream_t)stream))
      return rc;
    e = wf::launch_quality_scene(nbands, cout, ms, pan, out_pitch, ms_pitch, pan_pitch, h, w,
                                 workspace, report, undecidable, (cudaStream_t)stream);
    if (e == cudaSuccess) g_launches += 4;
  }
  return cuda_status(e, "wf_fuse_quality_f32");
}

#define WF_FUSE_EXACT(NAME, T)                                                              \
  int NAME(int kind, const T* pan, int64_t pan_pitch, const T* ms, int64_t ms_pitch, T* out,  \
           int64_t out_pitch, int h, int w, void* workspace, void* stream) {                 \
    if (int e = check_kind(kind)) return e;                                                  \
    if (!pan || !ms || !out || !workspace) return fail(WF_ERR_VALUE, "null pointer argument"); \
    if ((h & 1) || (w & 1))                                                                  \
      return fail(WF_ERR_ODD_DIMENSION, "panchromatic plane %dx%d has an odd dimension", w, h); \
    if (h < min_len(kind) || w < min_len(kind))                                              \
      return fail(WF_ERR_TOO_SMALL, "%dx%d below minimum %d per side", w, h, min_len(kind)); \
    cudaError_t e = wf::launch_fuse_exact<T>(kind, pan, pan_pitch, ms, ms_pitch, out,       \
                                             out_pitch, h, w, static_cast<double*>(workspace), \
                                             (cudaStream_t)stream);                          \
    if (e == cudaSuccess) g_launches += 2;                                                   \
    return cuda_status(e, #NAME);                                                            \
  }
WF_FUSE_EXACT(wf_fuse_dwt_exact_f32, float)
WF_FUSE_EXACT(wf_fuse_dwt_exact_f64, double)

#define WF_FUSE_BANDS_EXACT(NAME, T)                                                        \
  int NAME(int kind, const T* pan, int64_t pan_pitch, const T* const* ms, int64_t ms_pitch, \
           T* const* out, int64_t out_pitch, int nbands, int h, int w, void* workspace,      \
           void* stream) {                                                                   \
    if (int e = check_kind(kind)) return e;                                                  \
    if (!pan || !ms || !out || !workspace) return fail(WF_ERR_VALUE, "null pointer argument"); \
    if (nbands < 1) return fail(WF_ERR_VALUE, "band list is empty");                         \
    for (int b = 0; b < nbands; ++b)                                                         \
      if (!ms[b] || !out[b]) return fail(WF_ERR_VALUE, "null band pointer %d", b);           \
    if ((h & 1) || (w & 1))                                                                  \
      return fail(WF_ERR_ODD_DIMENSION, "panchromatic plane %dx%d has an odd dimension", w, h); \
    if (h < min_len(kind) || w < min_len(kind))                                              \
      return fail(WF_ERR_TOO_SMALL, "%dx%d below minimum %d per side", w, h, min_len(kind)); \
    cudaError_t e = wf::launch_fuse_bands_exact<T>(kind, pan, pan_pitch, ms, ms_pitch, out,  \
                                                   out_pitch, nbands, h, w,                  \
                                                   static_cast<double*>(workspace),          \
                                                   (cudaStream_t)stream);                    \
    if (e == cudaSuccess) g_launches += 1 + nbands;                                      \
    return cuda_status(e, #NAME);                                                            \
  }
WF_FUSE_BANDS_EXACT(wf_fuse_bands_exact_f32, float)
WF_FUSE_BANDS_EXACT(wf_fuse_bands_exact_f64, double)

int wf_ipc_export(const void* ptr, void* handle64, uint64_t* offset) {
  if (!ptr || !handle64 || !offset) return fail(WF_ERR_VALUE, "null pointer argument");
  return cuda_status(wf::ipc_export(ptr, handle64, offset), "wf_ipc_export");
}
int wf_ipc_open(const void* handle64, void** base) {
  if (!handle64 || !base) return fail(WF_ERR_VALUE, "null pointer argument");
  return cuda_status(wf::ipc_open(handle64, base), "wf_ipc_open");
}
int wf_ipc_close(void* base) { return cuda_status(wf::ipc_close(base), "wf_ipc_close"); }

int wf_synth_plane_f32(float* out, int64_t pitch, int rows, int cols, uint64_t seed,
                       uint32_t plane, int row0, int col0, void* stream) {
  if (!out || rows < 0 || cols < 0 || pitch < cols)
    return fail(WF_ERR_VALUE, "bad synth arguments");
  if (rows == 0 || cols == 0) return WF_OK;
  cudaError_t e = wf::launch_synth(out, pitch, rows, cols, seed, plane, row0, col0,
                                   (cudaStream_t)stream);
  if (e == cudaSuccess) ++g_launches;
  return cuda_status(e, "wf_synth_plane_f32");
}

}  // extern "C"
