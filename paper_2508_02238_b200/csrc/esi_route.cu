// esi_route.cu -- row-band routing for multi-GPU sharding of one large sensor
// (BASELINE.json config 5b).
//
// ESI has no spatial coupling: an event changes only its own pixel (Alg. 2,
// P:242-253), so rows [row_start[b], row_start[b+1]) can be integrated by an
// independent band handle.  esi_route_bands stably partitions a time-ordered
// event array by band -- band-major, arrival-order-minor, i.e. exactly
// std::stable_partition generalised to n_bands keys -- and rebases
// y to the band's first row.  Concatenating, per band, the routed runs of
// consecutive time shards in shard order therefore gives the band's events in
// time order.
//
// Three kernels on the caller's stream:
//   1. histogram: one CTA per 4096-event tile, per-tile band counts
//   2. scan:      one CTA per band, exclusive prefix of its tile counts + total
//   3. scatter:   one CTA per tile, stable in-tile ranks (warp ballot multi-split
//                 over the band bits + per-warp counts), 16-B record writes to a
//                 per-band destination pointer, which may live on a peer GPU
//                 (esi_router_scatter: the all-to-all exchange is done by the
//                 scatter's own NVLink stores, overlapped tile by tile)
#include "esi_device.cuh"

namespace esi {

constexpr int kRouteTile = 4096;
constexpr int kRouteThreads = 256;   // 8 warps x 16 events per thread
constexpr int kRouteMaxBands = 64;

__device__ __forceinline__ int route_band_of(uint32_t y, const int32_t* rs, int nb) {
  int b = 0;                         // largest b with rs[b] <= y (nb <= 64: linear scan is cheap)
  for (int q = 1; q < nb; ++q) b += (uint32_t)rs[q] <= y;
  return b;
}

__global__ void __launch_bounds__(kRouteThreads) esi_route_hist_kernel(const esi_event_t* ev, int64_t n,
                                                                       int32_t H, int nb, RouteRows rr,
                                                                       uint32_t* tile_cnt,
                                                                       unsigned long long* err) {
  __shared__ uint32_t cnt[kRouteMaxBands];
  for (int b = threadIdx.x; b < nb; b += kRouteThreads) cnt[b] = 0;
  __syncthreads();
  const int64_t e0 = (int64_t)blockIdx.x * kRouteTile;
  const int ne = (int)min((int64_t)kRouteTile, n - e0);
  const int4* evv = reinterpret_cast<const int4*>(ev + e0);
  for (int ib = 0; ib < ne; ib += kRouteThreads) {     // warp-aggregated counts (few bands: avoid
    const int i = ib + threadIdx.x;                     // same-address shared atomics per event)
    int b = -1;
    if (i < ne) {
      const int4 r = __ldg(evv + i);
      const uint32_t y = (uint32_t)r.z >> 16;
      if (y >= (uint32_t)H) atomicMin(err, ((unsigned long long)(e0 + i) << 8) | (unsigned)ESI_ERR_OUT_OF_BOUNDS);
      else b = route_band_of(y, rr.start, nb);
    }
    const unsigned peers = __match_any_sync(kFull, b);
    if (b >= 0 && (peers & lanemask_lt()) == 0u) atomicAdd(&cnt[b], (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kRouteThreads) tile_cnt[(int64_t)b * gridDim.x + blockIdx.x] = cnt[b];
}

// One CTA per band: exclusive prefix over the band's tile counts, in place; total -> band_tot[b].
// Each thread sums a contiguous run of tiles, one block scan combines the runs.
__global__ void __launch_bounds__(1024) esi_route_scan_kernel(uint32_t* tile_cnt, int n_tiles,
                                                              int64_t* band_tot) {
  __shared__ uint32_t wsum[32];
  const int b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* c = tile_cnt + (int64_t)b * n_tiles;
  const int per = (n_tiles + 1023) / 1024;
  const int t0 = threadIdx.x * per, t1 = min(n_tiles, t0 + per);
  uint32_t local = 0;
  for (int t = t0; t < t1; ++t) local += c[t];
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;   // inclusive
  }
  __syncthreads();
  uint32_t run = x - local + (warp ? wsum[warp - 1] : 0u);   // band-local offsets fit 32 bits (n < 2^32)
  for (int t = t0; t < t1; ++t) {
    const uint32_t v = c[t];
    c[t] = run;
    run += v;
  }
  if (threadIdx.x == 1023) band_tot[b] = (int64_t)run;
}

// Scatter: band b's run of this tile goes to dst.ptr[b] + dst.off[b] + (events of
// band b in earlier tiles) + in-tile rank.  dst.ptr[b] may be a peer GPU's
// buffer (NVLink P2P stores): the exchange of esi_router_scatter is this kernel.
// With band_tot != nullptr (esi_route_bands), every band goes to one buffer at
// the exclusive prefix of the band totals.
__global__ void __launch_bounds__(kRouteThreads) esi_route_scatter_kernel(const esi_event_t* ev, int64_t n,
                                                                          int32_t H, int nb, RouteRows rr,
                                                                          const uint32_t* tile_off,
                                                                          const int64_t* band_tot,
                                                                          RouteDst dst) {
  __shared__ uint32_t wcnt[kRouteThreads / 32][kRouteMaxBands];
  __shared__ int4* base[kRouteMaxBands];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int64_t e0 = (int64_t)tile * kRouteTile;
  const int ne = (int)min((int64_t)kRouteTile, n - e0);
  for (int i = threadIdx.x; i < (kRouteThreads / 32) * kRouteMaxBands; i += kRouteThreads)
    (&wcnt[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int b = 0; b < nb; ++b) {
      const int64_t off = band_tot ? run : dst.off[b];
      base[b] = reinterpret_cast<int4*>(dst.ptr[b]) + off + tile_off[(int64_t)b * gridDim.x + tile];
      if (band_tot) run += band_tot[b];
    }
  }
  __syncthreads();
  // warp w owns events [w*512, w*512+512) of the tile: 16 rounds of 32
  constexpr int kPer = kRouteTile / (kRouteThreads / 32) / 32;
  int4 rec[kPer];
  uint32_t rk[kPer];
  const int4* evv = reinterpret_cast<const int4*>(ev + e0);
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int i = warp * (kPer * 32) + r * 32 + lane;
    const bool act = i < ne;
    rec[r] = act ? __ldg(evv + i) : make_int4(0, 0, 0, 0);
    const uint32_t y = (uint32_t)rec[r].z >> 16;
    const bool ok = act && y < (uint32_t)H;
    const int b = ok ? route_band_of(y, rr.start, nb) : 0;
    unsigned peers = __ballot_sync(kFull, ok);
#pragma unroll
    for (int bit = 0; bit < 6; ++bit) {
      const bool bs = (b >> bit) & 1;
      const unsigned bb = __ballot_sync(kFull, bs);
      peers &= bs ? bb : ~bb;
    }
    if (!ok) peers = 0u;
    const uint32_t rank = __popc(peers & lanemask_lt());
    uint32_t prior = 0;
    if (ok) prior = wcnt[warp][b];
    __syncwarp();
    if (ok && rank == 0) wcnt[warp][b] = prior + __popc(peers);
    __syncwarp();
    rk[r] = ok ? ((prior + rank) | ((uint32_t)b << 16)) : 0xffffffffu;
    if (ok) rec[r].z = (int)(((uint32_t)rec[r].z & 0xffffu) | ((y - (uint32_t)rr.start[b]) << 16));
  }
  __syncthreads();
  // exclusive prefix over warps per band
  for (int b = threadIdx.x; b < nb; b += kRouteThreads) {
    uint32_t run = 0;
    for (int w = 0; w < kRouteThreads / 32; ++w) {
      const uint32_t c = wcnt[w][b];
      wcnt[w][b] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    if (rk[r] == 0xffffffffu) continue;
    const int b = (int)(rk[r] >> 16);
    base[b][wcnt[warp][b] + (rk[r] & 0xffffu)] = rec[r];
  }
}

cudaError_t launch_route_count(const esi_event_t* ev, int64_t n, int32_t H, int nb, const RouteRows& rr,
                               uint32_t* tile_cnt, int64_t* band_tot, unsigned long long* err, cudaStream_t s) {
  const int n_tiles = (int)((n + kRouteTile - 1) / kRouteTile);
  esi_route_hist_kernel<<<n_tiles, kRouteThreads, 0, s>>>(ev, n, H, nb, rr, tile_cnt, err);
  esi_route_scan_kernel<<<nb, 1024, 0, s>>>(tile_cnt, n_tiles, band_tot);
  return cudaGetLastError();
}

cudaError_t launch_route_scatter(const esi_event_t* ev, int64_t n, int32_t H, int nb, const RouteRows& rr,
                                 const uint32_t* tile_off, const int64_t* band_tot, const RouteDst& dst,
                                 cudaStream_t s) {
  const int n_tiles = (int)((n + kRouteTile - 1) / kRouteTile);
  esi_route_scatter_kernel<<<n_tiles, kRouteThreads, 0, s>>>(ev, n, H, nb, rr, tile_off, band_tot, dst);
  return cudaGetLastError();
}

int64_t route_tiles(int64_t n) { return (n + kRouteTile - 1) / kRouteTile; }

}  // namespace esi
