// esi_internal.cuh -- device-side types and launchers of libesi (sm_100a).
//
// Pipeline of one render call:
//   plan      : per chunk: time base, frames it renders, fast-path eligibility (tiny)
//   per chunk of <= chunk_events pending events (K1 of chunk c+1 on a
//   low-priority aux stream overlaps K2 of chunk c; double-buffered scratch):
//     K1 esi_partition_kernel : 16-B ingest (cp.async-staged 4096-event tiles) +
//        validation + stable, bit-exact partition of each tile by pixel band
//     K2 esi_integrate_kernel : one CTA per band (esi_integrate_fast.cu; fp64
//        fallback esi_integrate.cu); gathers the band's events in arrival order,
//        applies Alg. 2 per frame window (claim chains: sparse / chain / dense
//        warp-scan paths) to the band's state in shared memory, and writes every
//        frame of the chunk (fused Eq. 13/14 readout)
//   consume   : how many pending events were integrated                   (tiny)
//   K4 esi_readout_kernel   : frames when no event is pending (readout only)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/esi.h"

namespace esi {

#ifndef ESI_TILE
#define ESI_TILE 4096
#endif
#ifndef ESI_PART_THREADS
#define ESI_PART_THREADS 512
#endif
#ifndef ESI_PART_CTAS
#define ESI_PART_CTAS 2
#endif
constexpr int kTile = ESI_TILE;                // events per partition tile
constexpr int kPartThreads = ESI_PART_THREADS; // 16 warps x 8 events per thread
constexpr int kPartCtas = ESI_PART_CTAS;       // resident K1 CTAs per SM (launch bounds)
constexpr int kPartWarps = kPartThreads / 32;
constexpr int kSubBatch = 1024;      // band events staged in smem per sub-batch
constexpr int kMaxTilesPerChunk = 2048;
constexpr int kWarpPx = 256;         // pixels owned by one warp (8 per lane)
constexpr int kMaxBands = 1024;
constexpr int kMaxBandPx = 4096;
// Resident fast-K2 CTAs (8 warps each) per SM that the band size targets; the
// kernel's events per thread per sub-batch follow from the shared-memory budget.
#ifndef ESI_K2_CTAS
#define ESI_K2_CTAS 3
#endif
constexpr int kK2Ctas = ESI_K2_CTAS;
#ifndef ESI_K2_WARPS
#define ESI_K2_WARPS 8
#endif
constexpr int kK2Warps = ESI_K2_WARPS;     // warps per fast-K2 CTA

// Band layout.  Pixel ids are dealt to the nb bands in groups of kGroup = 64 consecutive
// ids; a band holds gpb groups (band_px = gpb * 64 pixel slots).  Two layouts, one code path:
//   interleaved: group g = pid / 64 belongs to band g % nb and is its local group g / nb,
//                so every band samples the whole sensor and the bands of a chunk hold nearly
//                the same number of events wherever the scene is active;
//   contiguous:  group g belongs to band g / gpb (a run of band_px consecutive pixel ids).
// Local pixel i of band b is pixel id (((i / 64) gs + b bs) * 64 + i % 64 with group strides
// (gs, bs) = (nb, 1) interleaved, (1, gpb) contiguous.  A warp's frame stores stay 64-byte runs.
#ifndef ESI_GROUP_SHIFT
#define ESI_GROUP_SHIFT 6
#endif
constexpr int kGroupShift = ESI_GROUP_SHIFT;
constexpr int kGroup = 1 << kGroupShift;
struct BandMap {
  int32_t nb, gpb;           // bands, groups per band
  int32_t gs, bs;            // group strides of the local group index and of the band index
  int32_t interleave;        // 1: interleaved, 0: contiguous
  uint32_t div, magic;       // g / div = umulhi(g, magic) for every group index g < 2^16 (div = nb or gpb; > 1)
};
inline BandMap make_band_map(int nb, int gpb, int interleave) {
  BandMap m;
  m.nb = nb;
  m.gpb = gpb;
  m.interleave = interleave;
  m.gs = interleave ? nb : 1;
  m.bs = interleave ? 1 : gpb;
  m.div = (uint32_t)(interleave ? nb : gpb);
  // umulhi(g, m) == g / d for g < 2^16: m = floor(2^32 / d) + 1, error term g (m d - 2^32) <= g d < 2^32
  m.magic = m.div <= 1 ? 0u : (uint32_t)((((uint64_t)1) << 32) / (uint64_t)m.div + 1);
  return m;
}
// (band, local pixel) of pixel id pid
__device__ __forceinline__ void band_of(const BandMap& m, uint32_t pid, uint32_t& band, uint32_t& local) {
  const uint32_t g = pid >> kGroupShift;
  const uint32_t q = m.div <= 1u ? g : __umulhi(g, m.magic);
  const uint32_t r = g - q * m.div;
  band = m.interleave ? r : q;
  local = ((m.interleave ? q : r) << kGroupShift) | (pid & (uint32_t)(kGroup - 1));
}
// pixel id of local pixel i of band `band`
__host__ __device__ inline int64_t band_gpix(const BandMap& m, int band, int i) {
  return (((int64_t)(i >> kGroupShift) * m.gs + (int64_t)band * m.bs) << kGroupShift) | (int64_t)(i & (kGroup - 1));
}
// valid local pixels of the band: a prefix [0, npx) of its band_px slots (only the sensor's
// last group can be partial)
__host__ __device__ inline int band_npx(const BandMap& m, int band, int64_t P) {
  const int64_t ng = (P + kGroup - 1) >> kGroupShift;          // groups of the sensor
  const int64_t first = (int64_t)band * m.bs;                  // the band's first group
  if (first >= ng) return 0;
  int64_t mine = (ng - first + m.gs - 1) / m.gs;               // its groups
  if (mine > m.gpb) mine = m.gpb;
  const int64_t last = (mine - 1) * m.gs + first;              // its last group
  const int64_t tail = (last == ng - 1) ? ng * kGroup - P : 0; // missing pixels of the last group
  return (int)(mine * kGroup - tail);
}

// First error of a render call: (global event index << 8) | code, atomicMin'ed
// so that the earliest offending event wins (same as the oracle's first error).
constexpr unsigned long long kNoError = ~0ull;

constexpr int kDecayExp = 5;   // DecayParams::bmode of the exponential variant (decay_kind 1)
constexpr int kDecayNone = 6;  // naive Eq. 2 integrator (decay_kind 2): d = 1, no per-event clamp;
                               // dt_cut = INT64_MAX keeps it on the fp64 wide kernel

struct DecayParams {
  float kh, kl;          // k * 1e-6 split into a float pair (u = 1 - k dt, dt in us)
  double k_us;           // k * 1e-6 in double (fallback when dt_cut > 2^24)
  int64_t dt_cut;        // smallest dt (us) with 1 - k dt <= 0: ceil(1e6 / k)
  int32_t use_f64;
  int32_t bmode;         // 1,2,3,4: integer b fast path; 0: exp2(b log2 u); kDecayExp: exp(-k dt)
  int32_t first;         // 1: decay, then add (variant); 0: Alg. 2 order
  int32_t unclamped;     // 1: no per-event Eq. 13 clamp (naive Eq. 2, complementary filter)
  float b;
  // fast K2: u = kf * ((tau_h - dt) + tau_l) with tau = 1e6/k us = tau_h + tau_l
  float tau_h, tau_l, kf;
  int32_t tau_i;         // (int32_t)tau_h (the fast K2's folded readout: tau is an integer there)
};

struct MapParams {
  float C;               // contrast step
  float smin, smax;      // Eq. 13 bounds
  // Eq. 14 + 0.5 = v*scale + off, off = -smin*scale + 0.5 split as off_int + off_frac so
  // that a tiny |v| is not absorbed by the offset (v = -1e-9 must give 127, not 128).
  float scale, off_frac;
  float scale_w2;        // (k * 1e-6)^2 * scale: folded b = 2 readout of the fast K2
  int32_t off_int;
  float magic_off;       // 2^23 + off_int (exact): RD-add magic of the fast K2 readout
  float ev_smin, ev_smax; // per-event clamp bounds of the fast K2 (+-FLT_MAX: unclamped state)
  int32_t readout_clamp;  // the fast K2 readout must clamp (bounds exclude 0, or unclamped state)
  int32_t readout_decay;
};

// fp64 copies of the parameters for the general (wide) K2 variant, which keeps S
// in fp64 within a chunk (the fallback for spans >= 2^30 us and slow decays,
// where fp32 rounding would accumulate over many barely-decayed events).
struct WideParams {
  double C, k_us, b, smin, smax, scale, off5;
  int64_t dt_cut;
  int32_t bmode, readout_decay;
  int32_t first, unclamped;
};

struct PartArgs {
  const esi_event_t* ev;     // this chunk's events
  int64_t n;                 // events in the chunk
  int32_t n_tiles;           // tiles of kTile events (set by launch_partition)
  uint32_t* tile_ctr;        // [2] zero at launch: tiles claimed by the persistent CTAs, CTAs done
  int64_t index_base;        // index of ev[0] among this render's pending events
  const int64_t* prev_t;     // t of the event preceding ev[0] (device address)
  int64_t t_origin;
  int64_t last_frame_t;      // events must be > this (INT64_MIN if no frame yet)
  int64_t t_min;             // max(t_origin, last_frame_t + 1): smallest admissible t
  int64_t t_cap;             // last frame time of the render call
  int32_t W, H;
  int32_t band_px, nb;       // bands of band_px pixel slots
  BandMap bm;                // pixel id <-> (band, local pixel)
  int32_t validate;          // 1: check every event (fused validation); 0: validated on push
  uint2* rec;                // [n_tiles * kTile] tile-local band-sorted records
  uint32_t* meta;            // [nb][n_tiles]: offset | count << 16
  int64_t* tile_t0;          // [n_tiles]
  int32_t* tile_wide;        // [n_tiles]
  int64_t* wide_t;           // [n_tiles * kTile] full t, written for wide tiles only
  unsigned long long* err;
  const struct ChunkInfo* gate_info;   // non-null: exit at once unless gate_info->active (sync-free single-chunk render)
};

// Per-chunk facts computed once by esi_plan_kernel (one thread per chunk).
struct ChunkInfo {
  int64_t tbase;        // t of the chunk's first event
  int64_t trel;         // base of the 32-bit relative times of the fast kernel:
                        // min(first event, first frame rendered by the chunk)
  int32_t f_lo, f_hi;   // frames rendered by this chunk: [f_lo, f_hi)
  int32_t active;       // first event <= t_cap
  int32_t wide;         // chunk spans >= 2^32 us (per-tile time bases needed)
  int32_t fast;         // every relevant time within 2^30 us of trel: fast kernel applies
  int32_t _pad;
};

struct IntArgs {
  const ChunkInfo* info;             // this chunk's entry
  const uint2* rec;
  const uint32_t* meta;
  const int64_t* tile_t0;
  const int32_t* tile_wide;
  const int64_t* wide_t;
  int32_t n_tiles;
  const int64_t* tf;                 // frame times (device)
  int32_t F;
  int64_t t_cap;
  float* S;
  int64_t* T;
  uint8_t* out;                      // [F][P]
  int64_t P;
  int32_t band_px, nb;
  BandMap bm;                        // pixel id <-> (band, local pixel)
  int32_t vec8;                      // 8-byte frame stores allowed
  DecayParams dp;
  MapParams mp;
  WideParams wp;
  const unsigned long long* gate;    // non-null: exit without writing if *gate != kNoError
  int32_t atomic_rank;               // warp-wide shared atomics serve lanes in lane order (probed)
  // sync-free single-chunk render: the host launches the fast and the general kernel without
  // reading the plan back; 1: run only if info->fast, 2: only if !info->fast, 0: run
  int32_t kind_gate;
  // ESI_BANDS_AUTO: per render, {max, sum, count} of the bands' event counts over the chunks
  // (one atomic update per CTA); null otherwise
  unsigned long long* bstats;
};

struct ReadoutArgs {
  const float* S;
  const int64_t* T;
  const int64_t* tf;
  int32_t F;
  uint8_t* out;
  int64_t P;
  int32_t vec8;
  DecayParams dp;
  MapParams mp;
};

// Row bands of esi_route_bands: band b = rows [start[b], start[b+1]).
struct RouteRows {
  int32_t start[65];
};

size_t partition_smem_bytes(int nb, int rank_mode);
size_t integrate_smem_bytes(int band_px);
size_t integrate_fast_smem_bytes(int band_px, int n_tiles);
cudaError_t launch_partition(const PartArgs& a, int n_tiles, int rank_mode, cudaStream_t s);
cudaError_t probe_atomic_order(unsigned* d_bad, cudaStream_t s);
cudaError_t launch_integrate(const IntArgs& a, cudaStream_t s);
cudaError_t launch_readout(const ReadoutArgs& a, cudaStream_t s);
// plan: ChunkInfo of every chunk and the number of chunks whose first event has t <= t_cap
cudaError_t launch_plan(const esi_event_t* const* chunk_first, const int64_t* chunk_n, int n_chunks,
                        const int64_t* tf, int F, int64_t t_cap, int allow_fast, ChunkInfo* info,
                        int32_t* n_active, cudaStream_t s);
// sync-free one-chunk render: plan from by-value arguments (+ error word / K1 counter reset), and a
// consume that packs {consumed, error word, kernel choice} into res[0..2]
cudaError_t launch_plan1(const esi_event_t* first, int64_t n, const int64_t* tf, int F, int64_t t_cap, int allow_fast,
                         ChunkInfo* info, unsigned long long* err, uint32_t* tile_ctr, cudaStream_t s);
cudaError_t launch_finish1(const esi_event_t* seg, int64_t n, int64_t t_cap, int64_t* res, int64_t* last_t,
                           const unsigned long long* err, const ChunkInfo* info, cudaStream_t s);
// fast kernel (32-bit relative times, dt_cut < 2^23) -- esi_integrate_fast.cu
cudaError_t launch_integrate_fast(const IntArgs& a, cudaStream_t s);
// consume: for segment k, count events with t <= t_cap (binary search), and set
// *last_t to the t of the last consumed event of the last segment with one.
cudaError_t launch_consume(const esi_event_t* seg, int64_t n, int64_t t_cap, int64_t* count,
                           int64_t* last_t, cudaStream_t s);
// row-band routing (esi_route.cu): hist + scan + stable scatter on stream s
struct RouteDst {
  esi_event_t* ptr[64];      // per band: destination buffer (local or a peer GPU's)
  int64_t off[64];           // per band: first record of this source's run in ptr[b]
};
cudaError_t launch_route_count(const esi_event_t* ev, int64_t n, int32_t H, int nb, const RouteRows& rr,
                               uint32_t* tile_cnt, int64_t* band_tot, unsigned long long* err, cudaStream_t s);
cudaError_t launch_route_scatter(const esi_event_t* ev, int64_t n, int32_t H, int nb, const RouteRows& rr,
                                 const uint32_t* tile_off, const int64_t* band_tot, const RouteDst& dst,
                                 cudaStream_t s);
int64_t route_tiles(int64_t n);
cudaError_t launch_fill_i64(int64_t* p, int64_t n, int64_t v, cudaStream_t s);
cudaError_t launch_frame_metrics(const uint8_t* frames, const float* truth, int64_t P, int n_frames,
                                 int truth_per_frame, double* pearson, double* mse_norm, cudaStream_t s);
// time-sharded streams (esi_slice.cu)
cudaError_t launch_slice_summary(const IntArgs& a, int64_t tbase, esi_slice_map_t* maps, int fast, cudaStream_t s);
cudaError_t launch_slice_compose(const esi_slice_map_t* A, const esi_slice_map_t* B, esi_slice_map_t* out, int64_t P,
                                 const DecayParams& dp, const MapParams& mp, cudaStream_t s);
cudaError_t launch_slice_apply(const esi_slice_map_t* M, float* S, int64_t* T, int64_t P, const DecayParams& dp,
                               const MapParams& mp, cudaStream_t s);
cudaError_t launch_validate(const esi_event_t* ev, int64_t n, const int64_t* prev_t,
                            int64_t t_origin, int64_t last_frame_t, int32_t W, int32_t H,
                            unsigned long long* err, cudaStream_t s);

}  // namespace esi
