// esi_runtime.cpp -- host runtime behind the C ABI of include/esi.h.
//
// A handle owns: the device state S (fp32) / T (int64) of Alg. 2,
// the list of pending event segments (borrowed device buffers or device copies
// of host pushes), the per-chunk scratch of K1/K2, and a stream.  A render call
// plans chunks of <= chunk_events pending events (whole segments never mix),
// runs K1 + K2 per chunk on the stream, then counts the consumed events and
// reads back the first error -- one small synchronisation per render call.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "esi_internal.cuh"

// NVTX ranges around the ABI calls and the render phases (header-only NVTX v3:
// no-ops unless a profiler is attached), so timelines show the host-side phases.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace esi {
cudaError_t launch_fill_i64(int64_t* p, int64_t n, int64_t v, cudaStream_t s);
}

using namespace esi;

namespace {

struct Segment {
  const esi_event_t* ptr;  // first pending event (device, or a device-accessible pinned host address)
  int64_t n;               // pending events
  void* owned;             // device buffer owned by the handle (pageable host pushes), or nullptr
  size_t owned_bytes;
  bool host;               // borrowed pinned host buffer (copied to the device during render)
};

struct Chunk {
  const esi_event_t* ptr;
  int64_t n;
  int seg;
  bool host;               // pinned host memory: staged to the device chunk by chunk during render
};

struct TimedLaunch {
  int kind;
  cudaEvent_t a, b;
  cudaStream_t s;
};

}  // namespace

struct esi_handle {
  int32_t W = 0, H = 0;
  int64_t P = 0;
  esi_params_t prm{};
  int band_px = 256, nb = 1;
  BandMap bm{};              // pixel id <-> (band, local pixel), the layout in use
  // both layouts of this sensor ([0] contiguous, [1] interleaved); ESI_BANDS_AUTO switches
  // from [0] to [1] when a render's busiest band held > 3x the mean (bstats)
  BandMap bm_of[2]{};
  int nb_of[2] = {1, 1};
  int layout_cur = 0;
  bool layout_auto = false;
  unsigned long long* d_bstats = nullptr;   // {max, sum, count} of band event counts of a render
  int64_t chunk_events = 0;
  int max_tiles = 0;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  float* dS = nullptr;
  int64_t* dT = nullptr;
  float* dS_snap = nullptr;      // lazy-validation mode: state at the start of the render, restored
  int64_t* dT_snap = nullptr;    // if the render finds an invalid event (S and T stay untouched)
  std::vector<Segment> segs;
  // K1/K2 scratch, double-buffered: K1 of chunk c+1 (stream aux) overlaps K2 of chunk c
  uint2* rec[2] = {nullptr, nullptr};
  uint32_t* meta[2] = {nullptr, nullptr};
  int64_t* tile_t0[2] = {nullptr, nullptr};
  int32_t* tile_wide[2] = {nullptr, nullptr};
  uint32_t* tile_ctr = nullptr;   // [2][2] K1 work counters per scratch buffer: tiles claimed, CTAs done
  int64_t* wide_t[2] = {nullptr, nullptr};
  cudaStream_t aux = nullptr;               // K1 stream
  cudaStream_t h2d = nullptr, d2h = nullptr; // copy streams of the pinned-host pipeline
  esi_event_t* stage_ev[2] = {nullptr, nullptr};   // device staging of host chunks (double buffer)
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_d2h_done = nullptr;
  cudaEvent_t ev_k1[2] = {nullptr, nullptr}, ev_k2[2] = {nullptr, nullptr}, ev_start = nullptr;
  // small device buffers
  int64_t* d_tf = nullptr;
  size_t tf_cap = 0;
  const esi_event_t** d_chunk_first = nullptr;
  size_t cf_cap = 0;
  int64_t* d_chunk_n = nullptr;
  size_t cn_cap = 0;
  ChunkInfo* d_info = nullptr;
  size_t info_cap = 0;
  int64_t* d_cons = nullptr;
  size_t cons_cap = 0;
  unsigned long long* d_err = nullptr;
  int64_t* d_last_t = nullptr;
  int32_t* d_n_active = nullptr;
  // pinned host scratch
  unsigned char* h_pin = nullptr;
  size_t h_pin_cap = 0;
  // device frame staging for host outputs
  uint8_t* d_frames = nullptr;
  size_t frames_cap = 0;
  std::vector<std::pair<void*, size_t>> pool;  // free device staging buffers
  int sticky = ESI_OK;
  bool has_last_frame = false;
  int64_t last_frame_t = INT64_MIN;
  DecayParams dp{};
  MapParams mp{};
  WideParams wp{};
  bool timing = false;
  double kt_ms[4] = {0, 0, 0, 0};
  int64_t kt_n[4] = {0, 0, 0, 0};
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> ev_pool;
  int64_t st_launches = 0, st_events = 0, st_chunks = 0, st_fast = 0;
  bool atomic_rank = true;   // lane-ordered smem atomics observed (probed at create)
  int rank_mode = 2;         // K1 stable ranks: 2 = peer masks (ordered by construction, default),
                             // 1 = lane-ordered atomics (only if probed), 0 = ballot multi-split
  bool allow_fast = true;    // K2 fast variant allowed (dt_cut < 2^23)
  bool single_stream = false; // ESI_SINGLE_STREAM=1: K1 and K2 on one stream
  bool sync_plan = false;     // ESI_SYNC_PLAN=1: read the plan back in every render (no sync-free one-chunk path)
};

namespace {

int cuda_fail(esi_handle_t* h, cudaError_t e) {
  if (e == cudaSuccess) return ESI_OK;
  if (getenv("ESI_DEBUG")) fprintf(stderr, "[esi] CUDA error: %s\n", cudaGetErrorString(e));
  if (h) h->sticky = ESI_ERR_CUDA;
  return ESI_ERR_CUDA;
}

#define ESI_CUDA(h, call)                          \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(h, e_); \
  } while (0)

// 0: pageable host, 1: device / managed, 2: pinned (page-locked, device-accessible) host
int ptr_kind(const void* p, const void** dev_alias) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return 1;
  if (at.type == cudaMemoryTypeHost && at.devicePointer) {
    if (dev_alias) *dev_alias = at.devicePointer;
    return 2;
  }
  return 0;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int ensure_pinned(esi_handle_t* h, size_t bytes) {
  if (bytes <= h->h_pin_cap) return ESI_OK;
  if (h->h_pin) cudaFreeHost(h->h_pin);
  h->h_pin = nullptr;
  size_t cap = std::max<size_t>(std::max(bytes, 2 * h->h_pin_cap), 4096);   // geometric growth
  if (cudaMallocHost((void**)&h->h_pin, cap) != cudaSuccess) {
    cudaGetLastError();
    h->h_pin_cap = 0;
    return ESI_ERR_OOM;
  }
  h->h_pin_cap = cap;
  return ESI_OK;
}

template <typename T>
int ensure_dev(esi_handle_t* h, T** p, size_t* cap, size_t n) {
  if (n <= *cap) return ESI_OK;
  if (*p) cudaFree((void*)*p);
  *p = nullptr;
  size_t c = std::max<size_t>(std::max(n, 2 * *cap), 64);   // geometric growth: few reallocations
  if (cudaMalloc((void**)p, c * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    *cap = 0;
    return ESI_ERR_OOM;
  }
  *cap = c;
  return ESI_OK;
}

void* pool_take(esi_handle_t* h, size_t bytes, size_t* got) {
  size_t best = SIZE_MAX;
  int bi = -1;
  for (size_t i = 0; i < h->pool.size(); ++i)
    if (h->pool[i].second >= bytes && h->pool[i].second < best) { best = h->pool[i].second; bi = (int)i; }
  if (bi >= 0) {
    void* p = h->pool[bi].first;
    *got = h->pool[bi].second;
    h->pool.erase(h->pool.begin() + bi);
    return p;
  }
  // new buffers are rounded up to a power of two (>= 1 MiB), so that a stream of
  // packets of slowly varying size reuses them instead of calling cudaMalloc
  // (which synchronises the device) for every packet a few events larger
  size_t want = (size_t)1 << 20;
  while (want < bytes) want <<= 1;
  void* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    if (want == bytes || cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    want = bytes;
  }
  *got = want;
  return p;
}

void pool_give(esi_handle_t* h, void* p, size_t bytes) {
  if (p) h->pool.push_back({p, bytes});
}

void drop_segments(esi_handle_t* h) {
  for (auto& s : h->segs) pool_give(h, s.owned, s.owned_bytes);
  h->segs.clear();
}

cudaEvent_t take_event(esi_handle_t* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void timed_begin(esi_handle_t* h, int kind, TimedLaunch* tl, cudaStream_t s = nullptr) {
  if (!h->timing) return;
  tl->kind = kind;
  tl->a = take_event(h);
  tl->b = take_event(h);
  tl->s = s ? s : h->stream;
  cudaEventRecord(tl->a, tl->s);
}

void timed_end(esi_handle_t* h, TimedLaunch* tl) {
  if (!h->timing) return;
  cudaEventRecord(tl->b, tl->s);
  h->timed.push_back(*tl);
}

void collect_timing(esi_handle_t* h) {
  for (auto& tl : h->timed) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, tl.a, tl.b) == cudaSuccess) {
      h->kt_ms[tl.kind] += ms;
      h->kt_n[tl.kind] += 1;
    }
    cudaGetLastError();
    h->ev_pool.push_back(tl.a);
    h->ev_pool.push_back(tl.b);
  }
  h->timed.clear();
}

int params_ok(const esi_params_t* p) {
  if (!(p->C > 0.0) || !std::isfinite(p->C)) return 0;
  if (!(p->k > 0.0) || !std::isfinite(p->k)) return 0;
  if (!(p->b > 0.0) || !std::isfinite(p->b)) return 0;
  if (!std::isfinite(p->s_min) || !std::isfinite(p->s_max) || !(p->s_min < p->s_max)) return 0;
  if (p->chunk_events < 0) return 0;
  if (p->decay_kind < 0 || p->decay_kind > 2 || p->decay_first < 0 || p->decay_first > 1) return 0;
  if (p->state_unclamped < 0 || p->state_unclamped > 1) return 0;
  if (p->band_layout < ESI_BANDS_CONTIGUOUS || p->band_layout > ESI_BANDS_AUTO) return 0;
  return 1;
}

void derive_params(esi_handle_t* h) {
  const esi_params_t& p = h->prm;
  const double kk = p.k * 1e-6;  // 1/us
  h->dp.kh = (float)kk;
  h->dp.kl = (float)(kk - (double)h->dp.kh);
  h->dp.k_us = kk;
  // Eq. 4: d = 0 from dt = 1/k on (A14); exponential variant: d = 0 from k dt = 24 on (A20)
  const double horizon = (p.decay_kind == 1 ? 24.0 : 1.0) * 1e6 / p.k;  // us
  h->dp.dt_cut = (horizon >= 9.0e18 || p.decay_kind == 2) ? INT64_MAX : (int64_t)std::ceil(horizon);
  h->dp.use_f64 = h->dp.dt_cut > (int64_t)(1 << 24);
  h->dp.b = (float)p.b;
  h->dp.tau_h = (float)horizon;
  h->dp.tau_i = h->dp.tau_h < 2.0e9f ? (int32_t)h->dp.tau_h : 0;   // used by the fast K2 only (tau < 2^23 there)
  h->dp.tau_l = (float)(horizon - (double)h->dp.tau_h);
  h->dp.kf = (float)kk;
  h->dp.bmode = p.decay_kind == 2 ? kDecayNone
                : p.decay_kind ? kDecayExp : (p.b == 1.0 || p.b == 2.0 || p.b == 3.0 || p.b == 4.0) ? (int)p.b : 0;
  h->dp.first = p.decay_first ? 1 : 0;
  h->dp.unclamped = (p.state_unclamped || p.decay_kind == 2) ? 1 : 0;
  // finite stand-ins for "no clamp": 0 * bound stays 0 in the dense-path scan
  h->mp.ev_smin = h->dp.unclamped ? -3.402823466e38f : (float)p.s_min;
  h->mp.ev_smax = h->dp.unclamped ? 3.402823466e38f : (float)p.s_max;
  h->mp.readout_clamp = (!(p.s_min <= 0.0 && p.s_max >= 0.0) || h->dp.unclamped) ? 1 : 0;
  h->mp.C = (float)p.C;
  h->mp.smin = (float)p.s_min;
  h->mp.smax = (float)p.s_max;
  const double range = p.s_max - p.s_min;
  h->mp.scale = (float)(255.0 / range);
  h->mp.scale_w2 = (float)(kk * kk * 255.0 / range);
  const double off = -p.s_min * 255.0 / range + 0.5;
  h->mp.off_int = (int32_t)std::floor(off);
  h->mp.off_frac = (float)(off - std::floor(off));
  h->mp.magic_off = (float)(8388608.0 + (double)h->mp.off_int);
  h->mp.readout_decay = p.readout_decay ? 1 : 0;
  h->wp.C = p.C;
  h->wp.k_us = kk;
  h->wp.b = p.b;
  h->wp.smin = p.s_min;
  h->wp.smax = p.s_max;
  h->wp.scale = 255.0 / range;
  h->wp.off5 = -p.s_min * 255.0 / range + 0.5;
  h->wp.dt_cut = h->dp.dt_cut;
  h->wp.bmode = h->dp.bmode;
  h->wp.first = h->dp.first;
  h->wp.unclamped = h->dp.unclamped;
  h->wp.readout_decay = h->mp.readout_decay;
}

}  // namespace

extern "C" {

void esi_default_params(esi_params_t* p) {
  if (!p) return;
  memset(p, 0, sizeof(*p));
  p->C = 0.15;
  p->k = 10.0;
  p->b = 2.0;
  p->s_min = -1.5;
  p->s_max = 1.5;
  p->t_origin_us = 0;
  p->readout_decay = 1;
  p->device = 0;
  p->validate_on_push = 1;   // atomic push; 0 = fused lazy validation
  p->chunk_events = 0;
}

const char* esi_strerror(int s) {
  switch (s) {
    case ESI_OK: return "ok";
    case ESI_ERR_INVALID_ARG: return "invalid argument";
    case ESI_ERR_OUT_OF_BOUNDS: return "event coordinates outside the sensor";
    case ESI_ERR_BAD_POLARITY: return "event polarity not +1/-1";
    case ESI_ERR_NEGATIVE_INTERVAL: return "negative time interval (events or frames out of order)";
    case ESI_ERR_CUDA: return "CUDA error";
    case ESI_ERR_OOM: return "out of memory";
    default: return "unknown status";
  }
}

int esi_create(int32_t width, int32_t height, const esi_params_t* params, esi_handle_t** out) {
  if (!out) return ESI_ERR_INVALID_ARG;
  *out = nullptr;
  esi_params_t prm;
  if (params) prm = *params; else esi_default_params(&prm);
  if (width < 1 || height < 1 || width > 65535 || height > 65535) return ESI_ERR_INVALID_ARG;
  const int64_t P = (int64_t)width * height;
  if (P > (int64_t)kMaxBands * kMaxBandPx) return ESI_ERR_INVALID_ARG;   // <= 1024 bands of <= 4096 px
  if (!params_ok(&prm)) return ESI_ERR_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || prm.device < 0 || prm.device >= ndev) {
    cudaGetLastError();
    return prm.device < 0 ? ESI_ERR_INVALID_ARG : ESI_ERR_CUDA;
  }
  if (cudaSetDevice(prm.device) != cudaSuccess) return ESI_ERR_CUDA;

  esi_handle_t* h = new esi_handle_t();
  h->W = width;
  h->H = height;
  h->P = P;
  h->prm = prm;
  derive_params(h);
  // Bands (K1 partition key, one K2 CTA each) of gpb 64-pixel groups (esi_internal.cuh,
  // BandMap): gpb such that the bands fill the SMs evenly at kK2Ctas resident K2 CTAs (8 warps
  // each) per SM when a band then fits shared memory (c4, 3 per SM: 33 groups = 2112 pixel
  // slots; 437 contiguous bands, or 444 interleaved ones, on 148 SMs), else as many bands as
  // kMaxBandPx needs (at most kMaxBands, K1's shared-memory histograms: P <= 2^22).
  {
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, prm.device);
    const int64_t ng = (P + kGroup - 1) / kGroup;
    int64_t nb = std::max<int64_t>(1, std::min<int64_t>((int64_t)n_sm * kK2Ctas, std::min<int64_t>(ng, kMaxBands)));
    int64_t gpb = (ng + nb - 1) / nb;                          // groups per band
    if (const char* e = getenv("ESI_BAND_PX")) {
      const int64_t v = atoll(e);
      if (v >= kGroup && v <= kMaxBandPx && v % kGroup == 0 && (ng + v / kGroup - 1) / (v / kGroup) <= kMaxBands) {
        gpb = v / kGroup;
        nb = (ng + gpb - 1) / gpb;
      }
    }
    if (gpb > kMaxBandPx / kGroup) {                           // shared-memory cap: more bands than resident slots
      gpb = kMaxBandPx / kGroup;
      nb = (ng + gpb - 1) / gpb;
    }
    gpb = (ng + nb - 1) / nb;                                  // no band larger than the round-robin needs
    int layout = prm.band_layout;
    if (const char* e = getenv("ESI_BAND_LAYOUT")) layout = atoi(e);   // A/B override: 0, 1 or 2 (auto)
    const int interleave = layout == ESI_BANDS_INTERLEAVED ? 1 : 0;
    h->layout_auto = layout == ESI_BANDS_AUTO;
    h->nb_of[1] = (int)nb;
    h->nb_of[0] = (int)((ng + gpb - 1) / gpb);                 // contiguous runs of gpb groups: no empty band
    h->bm_of[0] = make_band_map(h->nb_of[0], (int)gpb, 0);
    h->bm_of[1] = make_band_map(h->nb_of[1], (int)gpb, 1);
    h->band_px = (int)(gpb * kGroup);
    h->layout_cur = interleave;
    h->nb = h->nb_of[interleave];
    h->bm = h->bm_of[interleave];
  }
  int64_t ce = prm.chunk_events > 0 ? prm.chunk_events : (int64_t)8 << 20;
  ce = ((ce + kTile - 1) / kTile) * kTile;
  ce = std::min<int64_t>(ce, (int64_t)kMaxTilesPerChunk * kTile);
  h->chunk_events = ce;
  h->max_tiles = (int)(ce / kTile);

  int rc = ESI_OK;
  auto dalloc = [&](void** p, size_t bytes) {
    if (rc) return;
    if (cudaMalloc(p, bytes) != cudaSuccess) { cudaGetLastError(); rc = ESI_ERR_OOM; }
  };
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) rc = ESI_ERR_CUDA;
  h->stream = h->own_stream;
  dalloc((void**)&h->dS, P * sizeof(float));
  dalloc((void**)&h->dT, P * sizeof(int64_t));
  for (int b = 0; b < 2; ++b) {
    dalloc((void**)&h->rec[b], ce * sizeof(uint2));
    dalloc((void**)&h->meta[b], (size_t)std::max(h->nb_of[0], h->nb_of[1]) * h->max_tiles * sizeof(uint32_t));
    dalloc((void**)&h->tile_t0[b], h->max_tiles * sizeof(int64_t));
    dalloc((void**)&h->tile_wide[b], h->max_tiles * sizeof(int32_t));
    dalloc((void**)&h->wide_t[b], ce * sizeof(int64_t));
    if (!rc && (cudaEventCreateWithFlags(&h->ev_k1[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&h->ev_k2[b], cudaEventDisableTiming) != cudaSuccess))
      rc = ESI_ERR_CUDA;
  }
  int prio_lo = 0, prio_hi = 0;   // K1 (aux) at the lowest priority: it fills the SMs around K2
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (!rc && (cudaStreamCreateWithPriority(&h->aux, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
              cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) != cudaSuccess))
    rc = ESI_ERR_CUDA;
  dalloc((void**)&h->d_err, sizeof(unsigned long long));
  dalloc((void**)&h->tile_ctr, 4 * sizeof(uint32_t));
  if (!rc && cudaMemset(h->tile_ctr, 0, 4 * sizeof(uint32_t)) != cudaSuccess) rc = ESI_ERR_CUDA;
  dalloc((void**)&h->d_last_t, sizeof(int64_t));
  dalloc((void**)&h->d_n_active, sizeof(int32_t));
  dalloc((void**)&h->d_bstats, 3 * sizeof(unsigned long long));
  if (!rc) rc = ensure_pinned(h, 1 << 16);
  if (!rc) rc = esi_reset(h);
  // unclamped states (naive Eq. 2, complementary filter) are unbounded sums that can cancel:
  // accumulate them in fp64 (wide kernel) rather than fp32
  h->allow_fast = h->dp.dt_cut < ((int64_t)1 << 23) && !h->dp.unclamped && !getenv("ESI_DISABLE_FAST");
  h->single_stream = getenv("ESI_SINGLE_STREAM") && atoi(getenv("ESI_SINGLE_STREAM")) != 0;
  h->sync_plan = getenv("ESI_SYNC_PLAN") && atoi(getenv("ESI_SYNC_PLAN")) != 0;
  if (!rc) {
    // K1 rank mode: probe that warp-wide smem atomics serve same-address lanes in lane order
    const char* mode = getenv("ESI_RANK_MODE");
    unsigned* d_bad = nullptr;
    unsigned h_bad = 1;
    if (cudaMalloc((void**)&d_bad, sizeof(unsigned)) == cudaSuccess &&
        cudaMemsetAsync(d_bad, 0, sizeof(unsigned), h->stream) == cudaSuccess &&
        probe_atomic_order(d_bad, h->stream) == cudaSuccess &&
        cudaMemcpyAsync(&h_bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream) == cudaSuccess &&
        cudaStreamSynchronize(h->stream) == cudaSuccess) {
      h->atomic_rank = (h_bad == 0);
    } else {
      cudaGetLastError();
      h->atomic_rank = false;
    }
    if (d_bad) cudaFree(d_bad);
    // default: lane-ordered atomics when the probe confirms them (fastest, DESIGN 4), else
    // peer masks (ordered by construction); ESI_RANK_MODE=peers|ballot|atomic overrides
    h->rank_mode = h->atomic_rank ? 1 : 2;
    if (mode && strcmp(mode, "peers") == 0) h->rank_mode = 2;
    if (mode && strcmp(mode, "ballot") == 0) h->rank_mode = 0;
    if (mode && strcmp(mode, "atomic") == 0) h->rank_mode = h->atomic_rank ? 1 : 2;
  }
  if (!rc && cudaStreamSynchronize(h->stream) != cudaSuccess) rc = ESI_ERR_CUDA;
  if (rc) {
    esi_destroy(h);
    return rc;
  }
  *out = h;
  return ESI_OK;
}

void esi_destroy(esi_handle_t* h) {
  if (!h) return;
  cudaSetDevice(h->prm.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  drop_segments(h);
  for (auto& p : h->pool) cudaFree(p.first);
  for (auto& tl : h->timed) { cudaEventDestroy(tl.a); cudaEventDestroy(tl.b); }
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  if (h->aux) cudaStreamSynchronize(h->aux);
  void* bufs[] = {h->dS, h->dT, h->rec[0], h->meta[0], h->tile_t0[0], h->tile_wide[0], h->wide_t[0],
                  h->rec[1], h->meta[1], h->tile_t0[1], h->tile_wide[1], h->wide_t[1], h->d_tf,
                  (void*)h->d_chunk_first, h->d_chunk_n, h->d_info, h->d_cons, h->d_err, h->d_last_t, h->d_n_active, h->d_frames, h->tile_ctr, (void*)h->d_bstats,
                  h->dS_snap, h->dT_snap};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (int b = 0; b < 2; ++b) {
    if (h->ev_k1[b]) cudaEventDestroy(h->ev_k1[b]);
    if (h->ev_k2[b]) cudaEventDestroy(h->ev_k2[b]);
  }
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->aux) cudaStreamDestroy(h->aux);
  for (int b = 0; b < 2; ++b) {
    if (h->stage_ev[b]) cudaFree(h->stage_ev[b]);
    if (h->ev_h2d[b]) cudaEventDestroy(h->ev_h2d[b]);
  }
  if (h->ev_d2h_done) cudaEventDestroy(h->ev_d2h_done);
  if (h->h2d) { cudaStreamSynchronize(h->h2d); cudaStreamDestroy(h->h2d); }
  if (h->d2h) { cudaStreamSynchronize(h->d2h); cudaStreamDestroy(h->d2h); }
  if (h->h_pin) cudaFreeHost(h->h_pin);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  cudaGetLastError();
  delete h;
}

int esi_reset(esi_handle_t* h) {
  NvtxRange nvtx_range_("esi_reset");
  if (!h) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  cudaStreamSynchronize(h->stream);
  cudaGetLastError();
  drop_segments(h);
  h->sticky = ESI_OK;
  h->has_last_frame = false;
  h->last_frame_t = INT64_MIN;
  if (h->layout_auto) {      // ESI_BANDS_AUTO starts every stream on contiguous bands
    h->layout_cur = 0;
    h->nb = h->nb_of[0];
    h->bm = h->bm_of[0];
  }
  ESI_CUDA(h, cudaMemsetAsync(h->dS, 0, h->P * sizeof(float), h->stream));
  ESI_CUDA(h, launch_fill_i64(h->dT, h->P, h->prm.t_origin_us, h->stream));
  ESI_CUDA(h, launch_fill_i64(h->d_last_t, 1, INT64_MIN, h->stream));
  return ESI_OK;
}

int esi_set_stream(esi_handle_t* h, void* s) {
  if (!h) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  cudaStreamSynchronize(h->stream);
  h->stream = s ? (cudaStream_t)s : h->own_stream;
  return ESI_OK;
}

int esi_get_error(esi_handle_t* h) {
  if (!h) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return cuda_fail(h, cudaGetLastError());
  return h->sticky;
}

int esi_push_events(esi_handle_t* h, const esi_event_t* events, size_t n) {
  NvtxRange nvtx_range_("esi_push_events");
  if (!h) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  if (n == 0) return ESI_OK;
  if (!events || ((uintptr_t)events & 7)) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  Segment sg{events, (int64_t)n, nullptr, 0, false};
  const void* alias = nullptr;
  const int kind = ptr_kind(events, &alias);
  if (kind == 2 && !h->prm.validate_on_push) {
    // pinned host buffer: borrowed; render copies it to the device chunk by chunk,
    // overlapped with the kernels (the device reads it through its UVA alias only
    // for a few boundary timestamps)
    sg.ptr = (const esi_event_t*)alias;
    sg.host = true;
  } else if (kind != 1) {
    size_t got = 0;
    void* buf = pool_take(h, n * sizeof(esi_event_t), &got);
    if (!buf) return ESI_ERR_OOM;
    cudaError_t e = cudaMemcpyAsync(buf, events, n * sizeof(esi_event_t), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // caller may reuse its buffer
    if (e != cudaSuccess) {
      pool_give(h, buf, got);
      return cuda_fail(h, e);
    }
    sg.ptr = (const esi_event_t*)buf;
    sg.owned = buf;
    sg.owned_bytes = got;
  }
  if (h->prm.validate_on_push) {
    const int64_t* prev = h->segs.empty() ? h->d_last_t : &h->segs.back().ptr[h->segs.back().n - 1].t_us;
    ESI_CUDA(h, cudaMemsetAsync(h->d_err, 0xff, sizeof(unsigned long long), h->stream));
    TimedLaunch tl;
    timed_begin(h, 3, &tl);
    ESI_CUDA(h, launch_validate(sg.ptr, sg.n, prev, h->prm.t_origin_us,
                                h->has_last_frame ? h->last_frame_t : INT64_MIN, h->W, h->H, h->d_err,
                                h->stream));
    timed_end(h, &tl);
    unsigned long long* herr = (unsigned long long*)h->h_pin;
    ESI_CUDA(h, cudaMemcpyAsync(herr, h->d_err, sizeof(*herr), cudaMemcpyDeviceToHost, h->stream));
    ESI_CUDA(h, cudaStreamSynchronize(h->stream));
    if (*herr != kNoError) {
      pool_give(h, sg.owned, sg.owned_bytes);
      return (int)(*herr & 0xff);  // atomic rejection; the handle stays usable
    }
  }
  h->segs.push_back(sg);
  return ESI_OK;
}

int esi_render_many(esi_handle_t* h, const int64_t* tf, size_t F, uint8_t* out) {
  NvtxRange nvtx_range_("esi_render_many");
  if (!h) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  if (F == 0) return ESI_OK;
  if (!tf || !out) return ESI_ERR_INVALID_ARG;
  for (size_t j = 1; j < F; ++j)
    if (tf[j] < tf[j - 1]) return ESI_ERR_INVALID_ARG;
  if (tf[0] < h->prm.t_origin_us || (h->has_last_frame && tf[0] < h->last_frame_t))
    return ESI_ERR_NEGATIVE_INTERVAL;
  if (F > (size_t)INT32_MAX) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  cudaStream_t st = h->stream;
  const int64_t t_cap = tf[F - 1];
  h->st_launches = 0;
  h->st_events = 0;
  h->st_chunks = 0;
  h->st_fast = 0;

  // frame times -> device
  int rc = ensure_dev(h, &h->d_tf, &h->tf_cap, F);
  if (rc) return rc;
  ESI_CUDA(h, cudaMemcpyAsync(h->d_tf, tf, F * sizeof(int64_t), cudaMemcpyHostToDevice, st));

  // output: device pointer written in place, host pointer staged
  const bool out_dev = is_device_ptr(out);
  const size_t frame_bytes = (size_t)F * (size_t)h->P;
  uint8_t* dout = out;
  if (!out_dev) {
    if (frame_bytes > h->frames_cap) {
      if (h->d_frames) cudaFree(h->d_frames);
      h->d_frames = nullptr;
      h->frames_cap = 0;
      if (cudaMalloc((void**)&h->d_frames, frame_bytes) != cudaSuccess) {
        cudaGetLastError();
        return ESI_ERR_OOM;
      }
      h->frames_cap = frame_bytes;
    }
    dout = h->d_frames;
  }
  const int vec8 = (h->P % 8 == 0) && (((uintptr_t)dout & 7) == 0);

  // chunk plan over the pending segments
  std::vector<Chunk> chunks;
  for (int k = 0; k < (int)h->segs.size(); ++k)
    for (int64_t off = 0; off < h->segs[k].n; off += h->chunk_events)
      chunks.push_back({h->segs[k].ptr + off, std::min(h->chunk_events, h->segs[k].n - off), k, h->segs[k].host});
  bool any_host = false;
  for (const Chunk& ch : chunks) any_host |= ch.host;
  if (any_host) {   // pinned-host pipeline: staging buffers + copy streams (created on first use)
    for (int b = 0; b < 2 && !rc; ++b)
      if (!h->stage_ev[b] && cudaMalloc((void**)&h->stage_ev[b], h->chunk_events * sizeof(esi_event_t)) != cudaSuccess) {
        cudaGetLastError();
        return ESI_ERR_OOM;
      }
    if (!h->h2d) {
      if (cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_h2d[0], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_h2d[1], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_d2h_done, cudaEventDisableTiming) != cudaSuccess)
        return cuda_fail(h, cudaGetLastError());
    }
  }
  const bool stream_frames = !out_dev && !chunks.empty();   // frames copied back chunk by chunk
  if (stream_frames && !h->d2h) {
    if (cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_h2d[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_h2d[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_d2h_done, cudaEventDisableTiming) != cudaSuccess)
      return cuda_fail(h, cudaGetLastError());
  }

  if (chunks.empty()) {
    ReadoutArgs ra{h->dS, h->dT, h->d_tf, (int32_t)F, dout, h->P, vec8, h->dp, h->mp};
    TimedLaunch tl;
    timed_begin(h, 2, &tl);
    ESI_CUDA(h, launch_readout(ra, st));
    timed_end(h, &tl);
    h->st_launches = 1;
  } else {
    const size_t nc = chunks.size();
    rc = ensure_dev(h, &h->d_chunk_first, &h->cf_cap, nc);
    if (!rc) rc = ensure_dev(h, &h->d_chunk_n, &h->cn_cap, nc);
    if (!rc) rc = ensure_dev(h, &h->d_info, &h->info_cap, nc);
    if (!rc) rc = ensure_pinned(h, nc * 16 + h->segs.size() * sizeof(int64_t) + 128 + sizeof(ChunkInfo));
    if (rc) return rc;
    // A render of one device-resident chunk (the streaming case: one packet, one frame) does
    // not read the plan back: the chunk is rendered by whichever K2 variant the plan chose --
    // both are launched and the other one exits at once (IntArgs::kind_gate) -- K1 tests the
    // chunk's `active` flag itself, and chunk 0 of a one-chunk render owns every frame.  Its
    // plan takes the chunk by value and resets the error word and K1's counters, K1 runs on
    // the handle's stream (nothing to overlap with), and one kernel packs the consumed count,
    // the error word and the plan's choice for a single read-back: one host synchronisation
    // and about half the stream operations of the general path.
    const bool nosync = nc == 1 && !chunks[0].host && !h->sync_plan;
    auto k1_args = [&](int c, const esi_event_t* k1_ev, int64_t index_base) {
      const int bf = c & 1;
      PartArgs pa{};
      pa.ev = k1_ev;
      pa.n = chunks[c].n;
      pa.index_base = index_base;
      pa.prev_t = (c == 0) ? h->d_last_t : &chunks[c - 1].ptr[chunks[c - 1].n - 1].t_us;
      pa.t_origin = h->prm.t_origin_us;
      pa.last_frame_t = h->has_last_frame ? h->last_frame_t : INT64_MIN;
      pa.t_min = h->has_last_frame ? std::max(h->prm.t_origin_us, h->last_frame_t + 1) : h->prm.t_origin_us;
      pa.t_cap = t_cap;
      pa.W = h->W;
      pa.H = h->H;
      pa.band_px = h->band_px;
      pa.nb = h->nb;
      pa.bm = h->bm;
      pa.validate = h->prm.validate_on_push ? 0 : 1;
      pa.rec = h->rec[bf];
      pa.tile_ctr = h->tile_ctr + 2 * bf;
      pa.meta = h->meta[bf];
      pa.tile_t0 = h->tile_t0[bf];
      pa.tile_wide = h->tile_wide[bf];
      pa.wide_t = h->wide_t[bf];
      pa.err = h->d_err;
      pa.gate_info = nullptr;
      return pa;
    };
    int32_t* hna = (int32_t*)(h->h_pin + nc * 16 + 16);
    std::vector<ChunkInfo> hinfo(nc);
    h->st_launches += 1;   // plan
    if (nosync) {
      ESI_CUDA(h, launch_plan1(chunks[0].ptr, chunks[0].n, h->d_tf, (int)F, t_cap, h->allow_fast ? 1 : 0,
                               h->d_info, h->d_err, h->tile_ctr, st));
      *hna = 1;
      memset(&hinfo[0], 0, sizeof(ChunkInfo));
      hinfo[0].active = 1;
      hinfo[0].f_lo = 0;
      hinfo[0].f_hi = (int32_t)F;
    } else {
      const esi_event_t** hcf = (const esi_event_t**)h->h_pin;
      int64_t* hcn = (int64_t*)(h->h_pin + nc * sizeof(void*));
      for (size_t c = 0; c < nc; ++c) {
        hcf[c] = chunks[c].ptr;
        hcn[c] = chunks[c].n;
      }
      ESI_CUDA(h, cudaMemcpyAsync(h->d_chunk_first, hcf, nc * sizeof(void*), cudaMemcpyHostToDevice, st));
      ESI_CUDA(h, cudaMemcpyAsync(h->d_chunk_n, hcn, nc * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      ESI_CUDA(h, cudaMemsetAsync(h->d_err, 0xff, sizeof(unsigned long long), st));
      ESI_CUDA(h, cudaMemsetAsync(h->tile_ctr, 0, 4 * sizeof(uint32_t), st));   // K1 work counters (robust to an aborted launch)
      NvtxRange plan_range("render: plan (+ host read-back)");
      ESI_CUDA(h, launch_plan(h->d_chunk_first, h->d_chunk_n, (int)nc, h->d_tf, (int)F, t_cap,
                              h->allow_fast ? 1 : 0, h->d_info, h->d_n_active, st));
      ESI_CUDA(h, cudaMemcpyAsync(hna, h->d_n_active, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      ESI_CUDA(h, cudaMemcpyAsync(hinfo.data(), h->d_info, nc * sizeof(ChunkInfo), cudaMemcpyDeviceToHost, st));
      ESI_CUDA(h, cudaStreamSynchronize(st));
    }
    const int n_act = std::max(1, *hna);
    const bool watch = h->layout_auto && h->layout_cur == 0;   // ESI_BANDS_AUTO: watch the band balance
    if (watch) ESI_CUDA(h, cudaMemsetAsync(h->d_bstats, 0, 3 * sizeof(unsigned long long), st));
    const bool lazy = !h->prm.validate_on_push;
    if (lazy) {   // lazy validation (fused in K1): keep the state so that a failing render leaves it untouched
      if (!h->dS_snap) {
        if (cudaMalloc((void**)&h->dS_snap, h->P * sizeof(float)) != cudaSuccess ||
            cudaMalloc((void**)&h->dT_snap, h->P * sizeof(int64_t)) != cudaSuccess) {
          cudaGetLastError();
          return ESI_ERR_OOM;
        }
      }
      ESI_CUDA(h, cudaMemcpyAsync(h->dS_snap, h->dS, h->P * sizeof(float), cudaMemcpyDeviceToDevice, st));
      ESI_CUDA(h, cudaMemcpyAsync(h->dT_snap, h->dT, h->P * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }

    // K1 runs on the aux stream, K2 on the handle's stream; chunk c uses buffer c & 1:
    // K1(c) waits for the render's setup and for K2(c-2); K2(c) waits for K1(c).
    // (ESI_SINGLE_STREAM=1: both kernels on the handle's stream, no cross-stream events)
    const bool two = !h->single_stream && !nosync;
    cudaStream_t k1s = two ? h->aux : st;
    if (two) {
      ESI_CUDA(h, cudaEventRecord(h->ev_start, st));
      ESI_CUDA(h, cudaStreamWaitEvent(h->aux, h->ev_start, 0));
    }
    int64_t index_base = 0;
    for (int c = 0; c < n_act; ++c) {
      const int bf = c & 1;
      if (two && c >= 2) ESI_CUDA(h, cudaStreamWaitEvent(h->aux, h->ev_k2[bf], 0));
      const Chunk& ch = chunks[c];
      const int n_tiles = (int)((ch.n + kTile - 1) / kTile);
      const esi_event_t* k1_ev = ch.ptr;
      if (ch.host) {   // stage the chunk: H2D on the copy stream once K1(c-2) released the buffer
        if (c >= 2) ESI_CUDA(h, cudaStreamWaitEvent(h->h2d, h->ev_k1[bf], 0));
        ESI_CUDA(h, cudaMemcpyAsync(h->stage_ev[bf], ch.ptr, ch.n * sizeof(esi_event_t), cudaMemcpyDefault, h->h2d));
        ESI_CUDA(h, cudaEventRecord(h->ev_h2d[bf], h->h2d));
        ESI_CUDA(h, cudaStreamWaitEvent(k1s, h->ev_h2d[bf], 0));
        k1_ev = h->stage_ev[bf];
      }
      PartArgs pa = k1_args(c, k1_ev, index_base);
      pa.gate_info = nosync ? h->d_info + c : nullptr;
      if (hinfo[c].active) {   // a chunk entirely after the last frame (only chunk 0 can be) is not partitioned
        TimedLaunch t1;
        timed_begin(h, 0, &t1, k1s);
        ESI_CUDA(h, launch_partition(pa, n_tiles, h->rank_mode, k1s));
        timed_end(h, &t1);
        h->st_launches += 1;
      }
      if (two || any_host) ESI_CUDA(h, cudaEventRecord(h->ev_k1[bf], k1s));
      if (two) ESI_CUDA(h, cudaStreamWaitEvent(st, h->ev_k1[bf], 0));

      IntArgs ia{};
      ia.info = h->d_info + c;
      ia.rec = h->rec[bf];
      ia.meta = h->meta[bf];
      ia.tile_t0 = h->tile_t0[bf];
      ia.tile_wide = h->tile_wide[bf];
      ia.wide_t = h->wide_t[bf];
      ia.n_tiles = n_tiles;
      ia.tf = h->d_tf;
      ia.F = (int32_t)F;
      ia.t_cap = t_cap;
      ia.S = h->dS;
      ia.T = h->dT;
      ia.out = dout;
      ia.P = h->P;
      ia.band_px = h->band_px;
      ia.nb = h->nb;
      ia.bm = h->bm;
      ia.vec8 = vec8;
      ia.dp = h->dp;
      ia.mp = h->mp;
      ia.wp = h->wp;
      ia.gate = lazy ? h->d_err : nullptr;   // a K1 error so far: K2 exits (frames unspecified, S/T restored)
      ia.bstats = watch ? h->d_bstats : nullptr;
      TimedLaunch t2;
      timed_begin(h, 1, &t2);
      if (nosync) {          // the plan decides on the device which of the two runs
        if (h->allow_fast) {
          ia.kind_gate = 1;
          ESI_CUDA(h, launch_integrate_fast(ia, st));
          h->st_launches += 1;
        }
        ia.kind_gate = h->allow_fast ? 2 : 0;
        ESI_CUDA(h, launch_integrate(ia, st));
      } else if (hinfo[c].fast) {
        ESI_CUDA(h, launch_integrate_fast(ia, st));
        h->st_fast += 1;
      } else {
        ESI_CUDA(h, launch_integrate(ia, st));
      }
      timed_end(h, &t2);
      if (two || stream_frames) ESI_CUDA(h, cudaEventRecord(h->ev_k2[bf], st));
      if (stream_frames && hinfo[c].f_hi > hinfo[c].f_lo) {   // this chunk's frames are final: copy them back
        ESI_CUDA(h, cudaStreamWaitEvent(h->d2h, h->ev_k2[bf], 0));
        const size_t o = (size_t)hinfo[c].f_lo * (size_t)h->P;
        const size_t nbytes = (size_t)(hinfo[c].f_hi - hinfo[c].f_lo) * (size_t)h->P;
        ESI_CUDA(h, cudaMemcpyAsync(out + o, dout + o, nbytes, cudaMemcpyDeviceToHost, h->d2h));
      }
      h->st_launches += 1;
      h->st_chunks += 1;
      index_base += ch.n;
    }
    // consumed events per segment (segments after the last active chunk consume none)
    const int last_seg = chunks[n_act - 1].seg;
    rc = ensure_dev(h, &h->d_cons, &h->cons_cap, std::max<size_t>(3, h->segs.size()));
    if (rc) return rc;
    int64_t* hcons = (int64_t*)h->h_pin;
    unsigned long long* herr;
    unsigned long long* hbs = (unsigned long long*)(h->h_pin + nc * 16 + h->segs.size() * sizeof(int64_t) + 64);
    if (watch) ESI_CUDA(h, cudaMemcpyAsync(hbs, h->d_bstats, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (nosync) {   // one segment: {consumed, error word, kernel choice} in one kernel and one read-back
      ESI_CUDA(h, launch_finish1(h->segs[0].ptr, h->segs[0].n, t_cap, h->d_cons, h->d_last_t, h->d_err, h->d_info, st));
      h->st_launches += 1;
      herr = (unsigned long long*)(hcons + 1);
      ESI_CUDA(h, cudaMemcpyAsync(hcons, h->d_cons, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      ESI_CUDA(h, cudaStreamSynchronize(st));
      if (hcons[2]) h->st_fast += 1;
    } else {
      for (int k = 0; k <= last_seg; ++k) {
        ESI_CUDA(h, launch_consume(h->segs[k].ptr, h->segs[k].n, t_cap, h->d_cons + k, h->d_last_t, st));
        h->st_launches += 1;
      }
      herr = (unsigned long long*)(h->h_pin + (last_seg + 1) * sizeof(int64_t));
      ESI_CUDA(h, cudaMemcpyAsync(hcons, h->d_cons, (last_seg + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      ESI_CUDA(h, cudaMemcpyAsync(herr, h->d_err, sizeof(*herr), cudaMemcpyDeviceToHost, st));
      ESI_CUDA(h, cudaStreamSynchronize(st));
    }
    if (watch && *herr == kNoError && hbs[2] > 0 && hbs[1] >= 100000ull &&
        hbs[0] * hbs[2] > 3ull * hbs[1]) {   // busiest band > 3x the mean: interleaved bands from the next render on
      h->layout_cur = 1;
      h->nb = h->nb_of[1];
      h->bm = h->bm_of[1];
    }
    if (*herr != kNoError) {
      h->sticky = (int)(*herr & 0xff);
      if (lazy) {   // restore the state of the render's start; nothing is consumed
        cudaMemcpyAsync(h->dS, h->dS_snap, h->P * sizeof(float), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(h->dT, h->dT_snap, h->P * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
        if (stream_frames) cudaStreamSynchronize(h->d2h);
        cudaStreamSynchronize(st);
        cudaGetLastError();
        collect_timing(h);
        return h->sticky;
      }
    }
    std::vector<Segment> keep;
    for (int k = 0; k < (int)h->segs.size(); ++k) {
      Segment s = h->segs[k];
      const int64_t cons = k <= last_seg ? hcons[k] : 0;
      h->st_events += cons;
      if (cons >= s.n) {
        pool_give(h, s.owned, s.owned_bytes);
        continue;
      }
      s.ptr += cons;
      s.n -= cons;
      keep.push_back(s);
    }
    h->segs.swap(keep);
  }
  if (!out_dev && chunks.empty()) ESI_CUDA(h, cudaMemcpyAsync(out, dout, frame_bytes, cudaMemcpyDeviceToHost, st));
  if (stream_frames) ESI_CUDA(h, cudaStreamSynchronize(h->d2h));
  ESI_CUDA(h, cudaStreamSynchronize(st));
  collect_timing(h);
  h->has_last_frame = true;
  h->last_frame_t = t_cap;
  return h->sticky;
}

int esi_render(esi_handle_t* h, int64_t t_frame_us, uint8_t* out) {
  NvtxRange nvtx_range_("esi_render");
  return esi_render_many(h, &t_frame_us, 1, out);
}

int esi_get_state(esi_handle_t* h, float* S, int64_t* T) {
  NvtxRange nvtx_range_("esi_get_state");
  if (!h) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  if (S) ESI_CUDA(h, cudaMemcpyAsync(S, h->dS, h->P * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  if (T) ESI_CUDA(h, cudaMemcpyAsync(T, h->dT, h->P * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  ESI_CUDA(h, cudaStreamSynchronize(h->stream));
  return h->sticky;
}

int esi_set_state(esi_handle_t* h, const float* S, const int64_t* T) {
  NvtxRange nvtx_range_("esi_set_state");
  if (!h || !S || !T) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  cudaSetDevice(h->prm.device);
  ESI_CUDA(h, cudaMemcpyAsync(h->dS, S, h->P * sizeof(float), cudaMemcpyHostToDevice, h->stream));
  ESI_CUDA(h, cudaMemcpyAsync(h->dT, T, h->P * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
  ESI_CUDA(h, cudaStreamSynchronize(h->stream));
  return ESI_OK;
}

int esi_enable_kernel_timing(esi_handle_t* h, int enable) {
  if (!h) return ESI_ERR_INVALID_ARG;
  h->timing = enable != 0;
  for (int i = 0; i < 4; ++i) { h->kt_ms[i] = 0; h->kt_n[i] = 0; }
  return ESI_OK;
}

int esi_kernel_time(esi_handle_t* h, int kind, double* ms_total, int64_t* launches) {
  if (!h || kind < 0 || kind > 3) return ESI_ERR_INVALID_ARG;
  if (ms_total) *ms_total = h->kt_ms[kind];
  if (launches) *launches = h->kt_n[kind];
  return ESI_OK;
}

int esi_layout(esi_handle_t* h, int32_t* n_bands, int32_t* band_px, int32_t* warps_per_band) {
  if (!h) return ESI_ERR_INVALID_ARG;
  if (n_bands) *n_bands = h->nb;
  if (band_px) *band_px = h->band_px;
  if (warps_per_band) *warps_per_band = kK2Warps;
  return ESI_OK;
}

int esi_last_render_stats(esi_handle_t* h, int64_t* launches, int64_t* events, int64_t* chunks) {
  if (!h) return ESI_ERR_INVALID_ARG;
  if (launches) *launches = h->st_launches;
  if (events) *events = h->st_events;
  if (chunks) *chunks = h->st_chunks;
  return ESI_OK;
}

// ---- row-band router ------------------------------------------------------
struct esi_router {
  int32_t device = 0, height = 0, nb = 0;
  RouteRows rr;
  unsigned char* scratch = nullptr;   // band_tot[64] | err | tile_cnt[nb][n_tiles]
  size_t cap = 0;
  const esi_event_t* ev = nullptr;    // the counted events (caller-owned)
  int64_t n = 0;
  bool counted = false;
};

static int router_check_rows(int32_t height, const int32_t* row_start, int32_t n_bands) {
  if (!row_start || n_bands < 1 || n_bands > 64 || height < 1) return ESI_ERR_INVALID_ARG;
  if (row_start[0] != 0 || row_start[n_bands] != height) return ESI_ERR_INVALID_ARG;
  for (int b = 0; b < n_bands; ++b)
    if (row_start[b + 1] <= row_start[b]) return ESI_ERR_INVALID_ARG;
  return ESI_OK;
}

int esi_router_create(int32_t device, int32_t height, const int32_t* row_start, int32_t n_bands,
                      esi_router_t** out) {
  if (!out) return ESI_ERR_INVALID_ARG;
  *out = nullptr;
  if (int rc = router_check_rows(height, row_start, n_bands)) return rc;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  esi_router_t* r = new esi_router_t();
  r->device = device;
  r->height = height;
  r->nb = n_bands;
  for (int b = 0; b <= 64; ++b) r->rr.start[b] = b <= n_bands ? row_start[b] : height;
  *out = r;
  return ESI_OK;
}

int esi_router_count(esi_router_t* r, const esi_event_t* events, size_t n, int64_t* counts, void* stream) {
  NvtxRange nvtx_range_("esi_router_count");
  if (!r || !counts) return ESI_ERR_INVALID_ARG;
  r->counted = false;
  if (n == 0) {
    for (int b = 0; b < r->nb; ++b) counts[b] = 0;
    r->ev = nullptr;
    r->n = 0;
    r->counted = true;
    return ESI_OK;
  }
  if (!events || ((uintptr_t)events & 15) || n >= ((size_t)1 << 32)) return ESI_ERR_INVALID_ARG;
  if (cudaSetDevice(r->device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  if (!is_device_ptr(events)) return ESI_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n_tiles = route_tiles((int64_t)n);
  const size_t need = 64 * sizeof(int64_t) + 16 + (size_t)r->nb * n_tiles * sizeof(uint32_t);
  if (need > r->cap) {
    const size_t cap = std::max(need, r->cap * 2);
    if (r->scratch && (cudaStreamSynchronize(st) != cudaSuccess || cudaFree(r->scratch) != cudaSuccess)) {
      cudaGetLastError();
      return ESI_ERR_CUDA;
    }
    r->scratch = nullptr;
    r->cap = 0;
    if (cudaMalloc((void**)&r->scratch, cap) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_OOM; }
    r->cap = cap;
  }
  int64_t* band_tot = (int64_t*)r->scratch;
  unsigned long long* err = (unsigned long long*)(r->scratch + 64 * sizeof(int64_t));
  uint32_t* tile_cnt = (uint32_t*)(r->scratch + 64 * sizeof(int64_t) + 16);
  unsigned long long herr = kNoError;
  if (cudaMemsetAsync(err, 0xff, sizeof(*err), st) != cudaSuccess ||
      launch_route_count(events, (int64_t)n, r->height, r->nb, r->rr, tile_cnt, band_tot, err, st) != cudaSuccess ||
      cudaMemcpyAsync(counts, band_tot, r->nb * sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&herr, err, sizeof(herr), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    if (getenv("ESI_DEBUG")) fprintf(stderr, "[esi] route count: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaGetLastError();
    return ESI_ERR_CUDA;
  }
  if (herr != kNoError) return (int)(herr & 0xff);
  r->ev = events;
  r->n = (int64_t)n;
  r->counted = true;
  return ESI_OK;
}

int esi_router_scatter(esi_router_t* r, esi_event_t* const* dst, const int64_t* dst_offset, void* stream) {
  NvtxRange nvtx_range_("esi_router_scatter");
  if (!r || !dst || !dst_offset || !r->counted) return ESI_ERR_INVALID_ARG;
  if (r->n == 0) return ESI_OK;
  RouteDst d;
  for (int b = 0; b < 64; ++b) {
    d.ptr[b] = b < r->nb ? dst[b] : nullptr;
    d.off[b] = b < r->nb ? dst_offset[b] : 0;
    if (b < r->nb && (!dst[b] || ((uintptr_t)dst[b] & 15) || dst_offset[b] < 0)) return ESI_ERR_INVALID_ARG;
  }
  if (cudaSetDevice(r->device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  const uint32_t* tile_off = (const uint32_t*)(r->scratch + 64 * sizeof(int64_t) + 16);
  if (launch_route_scatter(r->ev, r->n, r->height, r->nb, r->rr, tile_off, nullptr, d, (cudaStream_t)stream) !=
      cudaSuccess) {
    cudaGetLastError();
    return ESI_ERR_CUDA;
  }
  return ESI_OK;
}

void esi_router_destroy(esi_router_t* r) {
  if (!r) return;
  if (r->scratch) {
    cudaSetDevice(r->device);
    cudaDeviceSynchronize();
    cudaFree(r->scratch);
  }
  delete r;
}

int esi_route_bands(int32_t device, const esi_event_t* events, size_t n, int32_t height,
                    const int32_t* row_start, int32_t n_bands, esi_event_t* out, int64_t* counts,
                    void* stream) {
  NvtxRange nvtx_range_("esi_route_bands");
  if (!counts) return ESI_ERR_INVALID_ARG;
  if (int rc = router_check_rows(height, row_start, n_bands)) return rc;
  if (n == 0) {
    for (int b = 0; b < n_bands; ++b) counts[b] = 0;
    return ESI_OK;
  }
  if (!events || !out || ((uintptr_t)events & 15) || ((uintptr_t)out & 15) || n >= ((size_t)1 << 32))
    return ESI_ERR_INVALID_ARG;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  if (!is_device_ptr(events) || !is_device_ptr(out)) return ESI_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  {   // keep the stream-ordered scratch mapped between calls (the default pool would unmap it at every sync)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  RouteRows rr;
  for (int b = 0; b <= 64; ++b) rr.start[b] = b <= n_bands ? row_start[b] : height;
  RouteDst d;
  for (int b = 0; b < 64; ++b) {
    d.ptr[b] = out;
    d.off[b] = 0;
  }
  const int64_t n_tiles = route_tiles((int64_t)n);
  const size_t bytes = (size_t)n_bands * n_tiles * sizeof(uint32_t) + 64 * sizeof(int64_t) + 16;
  unsigned char* scratch = nullptr;
  if (cudaMallocAsync((void**)&scratch, bytes, st) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_OOM; }
  int64_t* band_tot = (int64_t*)scratch;
  unsigned long long* err = (unsigned long long*)(scratch + 64 * sizeof(int64_t));
  uint32_t* tile_cnt = (uint32_t*)(scratch + 64 * sizeof(int64_t) + 16);
  int rc = ESI_OK;
  unsigned long long herr = kNoError;
  if (cudaMemsetAsync(err, 0xff, sizeof(*err), st) != cudaSuccess ||
      launch_route_count(events, (int64_t)n, height, n_bands, rr, tile_cnt, band_tot, err, st) != cudaSuccess ||
      launch_route_scatter(events, (int64_t)n, height, n_bands, rr, tile_cnt, band_tot, d, st) != cudaSuccess ||
      cudaMemcpyAsync(counts, band_tot, n_bands * sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&herr, err, sizeof(herr), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaFreeAsync(scratch, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
    if (getenv("ESI_DEBUG")) fprintf(stderr, "[esi] route: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaGetLastError();
    return ESI_ERR_CUDA;
  }
  if (herr != kNoError) rc = (int)(herr & 0xff);
  return rc;
}

int esi_frame_metrics(int32_t device, const uint8_t* frames, const float* truth, int64_t n_pixels,
                      int32_t n_frames, int32_t truth_per_frame, double* pearson, double* mse_norm,
                      void* stream) {
  if (!frames || !truth || !pearson || !mse_norm || n_pixels < 1 || n_frames < 0) return ESI_ERR_INVALID_ARG;
  if (n_frames == 0) return ESI_OK;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  if (!is_device_ptr(frames) || !is_device_ptr(truth)) return ESI_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  double* d = nullptr;
  if (cudaMallocAsync((void**)&d, 2 * (size_t)n_frames * sizeof(double), st) != cudaSuccess) {
    cudaGetLastError();
    return ESI_ERR_OOM;
  }
  cudaError_t e = launch_frame_metrics(frames, truth, n_pixels, n_frames, truth_per_frame, d, d + n_frames, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(pearson, d, n_frames * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(mse_norm, d + n_frames, n_frames * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { cudaGetLastError(); return ESI_ERR_CUDA; }
  return ESI_OK;
}

// ---- device buffers shared between processes (CUDA IPC) for the P2P exchange
int esi_buffer_alloc(int32_t device, size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return ESI_ERR_INVALID_ARG;
  *ptr = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  if (cudaMalloc(ptr, bytes) != cudaSuccess) { cudaGetLastError(); *ptr = nullptr; return ESI_ERR_OOM; }
  return ESI_OK;
}

int esi_buffer_free(int32_t device, void* ptr) {
  if (!ptr) return ESI_OK;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(ptr) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_CUDA; }
  return ESI_OK;
}

int esi_ipc_get_handle(const void* ptr, void* handle) {
  if (!ptr || !handle) return ESI_ERR_INVALID_ARG;
  cudaIpcMemHandle_t hd;
  if (cudaIpcGetMemHandle(&hd, const_cast<void*>(ptr)) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_CUDA; }
  static_assert(sizeof(hd) == ESI_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &hd, sizeof(hd));
  return ESI_OK;
}

int esi_ipc_open(int32_t device, const void* handle, void** ptr) {
  if (!handle || !ptr) return ESI_ERR_INVALID_ARG;
  *ptr = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return ESI_ERR_INVALID_ARG; }
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  if (cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return ESI_ERR_CUDA;
  }
  return ESI_OK;
}

int esi_ipc_close(int32_t device, void* ptr) {
  if (!ptr) return ESI_OK;
  if (cudaSetDevice(device) != cudaSuccess || cudaIpcCloseMemHandle(ptr) != cudaSuccess) {
    cudaGetLastError();
    return ESI_ERR_CUDA;
  }
  return ESI_OK;
}

int esi_stream_sync(int32_t device, void* stream) {
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
    cudaGetLastError();
    return ESI_ERR_CUDA;
  }
  return ESI_OK;
}

int esi_slice_summarize(esi_handle_t* h, const esi_event_t* events, size_t n, esi_slice_map_t* maps) {
  NvtxRange nvtx_range_("esi_slice_summarize");
  if (!h || !maps || (n && !events)) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  cudaSetDevice(h->prm.device);
  if (!is_device_ptr(maps)) return ESI_ERR_INVALID_ARG;
  cudaStream_t st = h->stream;
  ESI_CUDA(h, cudaMemsetAsync(maps, 0, (size_t)h->P * sizeof(esi_slice_map_t), st));   // n = 0: identity
  if (n == 0) {
    ESI_CUDA(h, cudaStreamSynchronize(st));
    return ESI_OK;
  }
  const esi_event_t* ev = events;
  esi_event_t* tmp = nullptr;
  if (!is_device_ptr(events)) {
    if (cudaMalloc((void**)&tmp, n * sizeof(esi_event_t)) != cudaSuccess) {
      cudaGetLastError();
      return ESI_ERR_OOM;
    }
    ESI_CUDA(h, cudaMemcpyAsync(tmp, events, n * sizeof(esi_event_t), cudaMemcpyHostToDevice, st));
    ev = tmp;
  }
  int rc = ESI_OK;
  int64_t* d_prev = nullptr;
  auto fail = [&](int code) { rc = code; };
  if (cudaMalloc((void**)&d_prev, sizeof(int64_t)) != cudaSuccess) { cudaGetLastError(); fail(ESI_ERR_OOM); }
  // validation (as a push: sensor bounds, polarity, non-decreasing t >= t_origin)
  if (!rc) {
    cudaError_t e = launch_fill_i64(d_prev, 1, INT64_MIN, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->d_err, 0xff, sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = launch_validate(ev, (int64_t)n, d_prev, h->prm.t_origin_us, INT64_MIN, h->W, h->H, h->d_err, st);
    unsigned long long herr = kNoError;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, h->d_err, sizeof(herr), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) fail(cuda_fail(h, e));
    else if (herr != kNoError) fail((int)(herr & 0xff));
  }
  // every chunk's first and last time, read back at once (one sync, not one per chunk)
  const int64_t n_chunks = ((int64_t)n + h->chunk_events - 1) / h->chunk_events;
  std::vector<int64_t> t01((size_t)(2 * n_chunks));
  if (!rc) rc = ensure_pinned(h, (size_t)(2 * n_chunks) * sizeof(int64_t));
  if (!rc) {
    int64_t* ht = (int64_t*)h->h_pin;
    cudaError_t e = cudaSuccess;
    for (int64_t c = 0; c < n_chunks && e == cudaSuccess; ++c) {
      const int64_t o = c * h->chunk_events, nc = std::min<int64_t>(h->chunk_events, (int64_t)n - o);
      e = cudaMemcpyAsync(ht + 2 * c, &ev[o].t_us, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaMemcpyAsync(ht + 2 * c + 1, &ev[o + nc - 1].t_us, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) fail(cuda_fail(h, e));
    else std::copy(ht, ht + 2 * n_chunks, t01.begin());
  }
  for (int64_t o = 0, c = 0; !rc && o < (int64_t)n; o += h->chunk_events, ++c) {
    const int64_t nc = std::min<int64_t>(h->chunk_events, (int64_t)n - o);
    if (t01[2 * c + 1] - t01[2 * c] >= ((int64_t)1 << 31)) { fail(ESI_ERR_INVALID_ARG); break; }
    cudaError_t e = cudaSuccess;
    const int n_tiles = (int)((nc + kTile - 1) / kTile);
    PartArgs pa{};
    pa.ev = ev + o;
    pa.n = nc;
    pa.index_base = o;
    pa.prev_t = d_prev;
    pa.t_origin = h->prm.t_origin_us;
    pa.last_frame_t = INT64_MIN;
    pa.t_min = h->prm.t_origin_us;
    pa.t_cap = INT64_MAX;
    pa.W = h->W;
    pa.H = h->H;
    pa.band_px = h->band_px;
    pa.nb = h->nb;
    pa.bm = h->bm;
    pa.validate = 0;   // validated above
    pa.rec = h->rec[0];
    pa.tile_ctr = h->tile_ctr;
    pa.meta = h->meta[0];
    pa.tile_t0 = h->tile_t0[0];
    pa.tile_wide = h->tile_wide[0];
    pa.wide_t = h->wide_t[0];
    pa.err = h->d_err;
    IntArgs ia{};
    ia.rec = h->rec[0];
    ia.meta = h->meta[0];
    ia.n_tiles = n_tiles;
    ia.P = h->P;
    ia.band_px = h->band_px;
    ia.nb = h->nb;
    ia.bm = h->bm;
    ia.dp = h->dp;
    ia.mp = h->mp;
    ia.atomic_rank = h->rank_mode == 1 ? 1 : 0;   // K5's ranks follow K1's (probed) mode
    e = cudaMemsetAsync(h->tile_ctr, 0, 2 * sizeof(uint32_t), st);   // K1 work counters
    if (e == cudaSuccess) e = launch_partition(pa, n_tiles, h->rank_mode, st);
    if (e == cudaSuccess) e = launch_slice_summary(ia, t01[2 * c], maps, h->allow_fast ? 1 : 0, st);
    if (e != cudaSuccess) fail(cuda_fail(h, e));
  }
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(h, e);
  }
  if (d_prev) cudaFree(d_prev);
  if (tmp) cudaFree(tmp);
  return rc;
}

int esi_slice_compose(esi_handle_t* h, const esi_slice_map_t* first, const esi_slice_map_t* second,
                      esi_slice_map_t* out) {
  NvtxRange nvtx_range_("esi_slice_compose");
  if (!h || !first || !second || !out) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  cudaSetDevice(h->prm.device);
  ESI_CUDA(h, launch_slice_compose(first, second, out, h->P, h->dp, h->mp, h->stream));
  return ESI_OK;
}

int esi_slice_apply(esi_handle_t* h, const esi_slice_map_t* maps) {
  NvtxRange nvtx_range_("esi_slice_apply");
  if (!h || !maps) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  if (!h->segs.empty()) return ESI_ERR_INVALID_ARG;
  cudaSetDevice(h->prm.device);
  ESI_CUDA(h, launch_slice_apply(maps, h->dS, h->dT, h->P, h->dp, h->mp, h->stream));
  return ESI_OK;
}

int esi_debug_partition(esi_handle_t* h, int64_t* out_t, uint32_t* out_pid, int8_t* out_p,
                        size_t n_out, uint32_t* band_start, int32_t* nb_out, int32_t* band_px_out) {
  if (!h || !band_start || !nb_out || !band_px_out) return ESI_ERR_INVALID_ARG;
  if (h->sticky) return h->sticky;
  cudaSetDevice(h->prm.device);
  *nb_out = h->nb;
  *band_px_out = h->band_px;
  if (h->segs.empty()) {
    for (int b = 0; b <= h->nb; ++b) band_start[b] = 0;
    return ESI_OK;
  }
  const Segment& s = h->segs[0];
  const int64_t n = std::min(h->chunk_events, s.n);
  if ((int64_t)n_out < n || !out_t || !out_pid || !out_p) return ESI_ERR_INVALID_ARG;
  const int n_tiles = (int)((n + kTile - 1) / kTile);
  PartArgs pa{};
  pa.ev = s.ptr;
  pa.n = n;
  pa.index_base = 0;
  pa.prev_t = h->d_last_t;
  pa.t_origin = h->prm.t_origin_us;
  pa.last_frame_t = h->has_last_frame ? h->last_frame_t : INT64_MIN;
  pa.t_min = h->has_last_frame ? std::max(h->prm.t_origin_us, h->last_frame_t + 1) : h->prm.t_origin_us;
  pa.t_cap = INT64_MAX;
  pa.W = h->W;
  pa.H = h->H;
  pa.band_px = h->band_px;
  pa.nb = h->nb;
  pa.bm = h->bm;
  pa.validate = h->prm.validate_on_push ? 0 : 1;
  pa.rec = h->rec[0];
  pa.tile_ctr = h->tile_ctr;
  pa.meta = h->meta[0];
  pa.tile_t0 = h->tile_t0[0];
  pa.tile_wide = h->tile_wide[0];
  pa.wide_t = h->wide_t[0];
  pa.err = h->d_err;
  ESI_CUDA(h, cudaMemsetAsync(h->d_err, 0xff, sizeof(unsigned long long), h->stream));
  ESI_CUDA(h, cudaMemsetAsync(h->tile_ctr, 0, 2 * sizeof(uint32_t), h->stream));   // K1 work counters
  ESI_CUDA(h, launch_partition(pa, n_tiles, h->rank_mode, h->stream));
  std::vector<uint2> rec(n_tiles * (size_t)kTile);
  std::vector<uint32_t> meta((size_t)h->nb * n_tiles);
  std::vector<int64_t> t0(n_tiles), wt;
  std::vector<int32_t> wide(n_tiles);
  ESI_CUDA(h, cudaMemcpyAsync(rec.data(), h->rec[0], n * sizeof(uint2), cudaMemcpyDeviceToHost, h->stream));
  ESI_CUDA(h, cudaMemcpyAsync(meta.data(), h->meta[0], meta.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  ESI_CUDA(h, cudaMemcpyAsync(t0.data(), h->tile_t0[0], n_tiles * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  ESI_CUDA(h, cudaMemcpyAsync(wide.data(), h->tile_wide[0], n_tiles * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
  ESI_CUDA(h, cudaStreamSynchronize(h->stream));
  bool any_wide = false;
  for (int t = 0; t < n_tiles; ++t) any_wide |= wide[t] != 0;
  if (any_wide) {
    wt.resize(n);
    ESI_CUDA(h, cudaMemcpy(wt.data(), h->wide_t[0], n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  }
  size_t o = 0;
  for (int b = 0; b < h->nb; ++b) {
    band_start[b] = (uint32_t)o;
    for (int t = 0; t < n_tiles; ++t) {
      const uint32_t m = meta[(size_t)b * n_tiles + t];
      const uint32_t off = m & 0xffffu, cnt = m >> 16;
      for (uint32_t i = 0; i < cnt; ++i) {
        const size_t idx = (size_t)t * kTile + off + i;
        const uint2 r = rec[idx];
        const int64_t tt = wide[t] ? wt[idx] : t0[t] + (int64_t)(uint32_t)(r.x - (uint32_t)t0[t]);
        out_t[o] = tt;
        out_pid[o] = (uint32_t)band_gpix(h->bm, b, (int)(r.y & 0x7fffffffu));
        out_p[o] = (r.y & 0x80000000u) ? -1 : 1;
        ++o;
      }
    }
  }
  band_start[h->nb] = (uint32_t)o;
  return ESI_OK;
}

}  // extern "C"
