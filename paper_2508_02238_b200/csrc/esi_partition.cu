// esi_partition.cu -- K1: event ingest + validation + stable partition by band.
//
// One 512-thread CTA per tile of kTile (4096) consecutive pending events.  The
// tile's 16-byte esi_event_t records are staged in shared memory with cp.async
// (a warp reads 512 contiguous bytes per step, every load in flight at once);
// each event is checked (reading A15: t non-decreasing, >=
// t_origin, > last frame) unless the push validated it, and its pixel id
// y*W + x and band = pid / band_px are computed.  The tile is then stably
// partitioned by band -- band-major, arrival-order-minor, i.e. exactly
// std::stable_sort by band -- with
//   * per-warp band histograms in shared memory whose ranks come from one of
//     three rank modes (lane-ordered shared atomics, probed at esi_create;
//     peer masks; ballot multi-split -- the last two ordered by construction),
//   * a per-band prefix over the warps (four bands per thread, packed u16
//     pairs) and a warp-shuffle scan over the bands,
//   * a scatter into shared memory and one TMA bulk copy of the sorted tile.
// Record (8 B): x = low 32 bits of t, y = pixel-in-band | (p < 0) << 31.
// meta[band][tile] = offset-in-tile | count << 16 tells K2 where its events are.
#include <algorithm>
#include <atomic>
#include "esi_device.cuh"

namespace esi {

size_t partition_smem_bytes(int nb, int rank_mode) {
  const int nbp = (nb + 7) & ~7;
  return (size_t)kTile * sizeof(int4) + (size_t)kTile * sizeof(uint2) + (size_t)kPartWarps * nbp * sizeof(uint16_t) +
         (size_t)(nbp + 8) * sizeof(uint32_t) + 64 * sizeof(uint32_t) +
         (rank_mode == 2 ? (size_t)kPartWarps * nbp * sizeof(uint32_t) : 0);
}

// RANK_ATOMIC: per-warp rank from a shared-memory atomicAdd on the warp's private
// (u16-packed) histogram -- relies on same-address lanes being served in lane
// order, which esi_probe_atomic_order checks at esi_create; otherwise ranks come
// from peer masks or a ballot multi-split over the band bits (order by construction).
// FULL: the tile holds kTile events (no bounds checks on the common path).
//
// Persistent CTAs (grid = resident CTAs, tiles strided by gridDim.x).  A tile's
// raw 16-B records are staged in shared memory by one TMA bulk copy completed on
// an mbarrier; as soon as they are consumed into registers, thread 0 issues the
// copy of the CTA's next tile, which lands while the current one is ranked,
// scanned, scattered and written.  The sorted tile has its own buffer (sbuf),
// written to global memory by one TMA bulk store.
struct PartSmem {
  int4* raw;          // [kTile] staged records
  uint2* sbuf;        // [kTile] sorted records
  uint16_t* hist;     // [kPartWarps][nbp]
  uint32_t* boff;     // [nbp + 8]
  uint32_t* wsum;     // [64]
  uint32_t* pmask;    // RANK 2: [kPartWarps][nbp] peer masks (zero)
};

__device__ __forceinline__ void mbar_wait_parity(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
}

// raw <- tile's records (thread 0 only)
__device__ __forceinline__ void issue_tile_load(const PartArgs& a, const PartSmem& sm, int tile, uint32_t mbar) {
  const int ne = (int)min((int64_t)kTile, a.n - (int64_t)tile * kTile);
  uint64_t pol_first;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic reads of raw
  const uint32_t bytes = (uint32_t)ne * 16u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"((uint32_t)__cvta_generic_to_shared(sm.raw)), "l"(a.ev + (int64_t)tile * kTile), "r"(bytes),
               "r"(mbar), "l"(pol_first) : "memory");
}

template <int RANK, bool VALIDATE, bool BAND32, bool FULL>
__device__ __forceinline__ void partition_tile(const PartArgs& a, const PartSmem& sm, int tile, int ne,
                                               uint32_t mbar, int64_t* s_tprev, int* s_wide, int* s_next) {
  constexpr int EPT = kTile / kPartThreads;                      // events per thread (8)
  constexpr int WEV = EPT * 32;                                  // events per warp (256)
  const int nbp = (a.nb + 7) & ~7;
  int4* raw = sm.raw;
  uint2* sbuf = sm.sbuf;
  uint16_t* hist = sm.hist;
  uint32_t* boff = sm.boff;
  uint32_t* wsum = sm.wsum;
  const int64_t e0 = (int64_t)tile * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const esi_event_t* ev = a.ev + e0;

  uint16_t* myhist = hist + warp * nbp;
  uint32_t key[EPT], tl[EPT], pr[EPT];   // band | rank << 10; record words (t low, pixel | sign)
  const uint32_t W = (uint32_t)a.W, H = (uint32_t)a.H;
  const int64_t t_min = a.t_min;
  const int64_t tprev0 = VALIDATE ? *s_tprev : 0;

#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int i = warp * WEV + r * 32 + lane;
    const bool act = FULL || i < ne;
    const int4 rw = act ? raw[i] : make_int4(0, 0, 0, 0);
    const int64_t t = (int64_t)(((uint64_t)(uint32_t)rw.y << 32) | (uint32_t)rw.x);
    uint32_t x = (uint32_t)rw.z & 0xffffu;
    uint32_t y = (uint32_t)rw.z >> 16;
    const int p = (int)(int8_t)(rw.w & 0xff);
    bool bad = false;
    if (VALIDATE) {
      const int64_t tp = i > 0 ? *reinterpret_cast<const int64_t*>(raw + i - 1) : tprev0;
      // validation (reading A15), one combined test on the common path
      bad = (x >= W) | (y >= H) | (p * p != 1) | (t < t_min) | (t < tp);
      if (act && bad) {
        int code;
        if (x >= W || y >= H) code = ESI_ERR_OUT_OF_BOUNDS;
        else if (p != 1 && p != -1) code = ESI_ERR_BAD_POLARITY;
        else code = ESI_ERR_NEGATIVE_INTERVAL;
        atomicMin(a.err, ((unsigned long long)(a.index_base + e0 + i) << 8) | (unsigned)code);
        x = 0; y = 0;              // keep the pipeline well-defined; the call reports the error
      }
    }
    const uint32_t pid = y * W + x;
    uint32_t band, pix;                                        // band layout (esi_internal.cuh);
    band_of(a.bm, pid, band, pix);                             // inactive lanes: pid = 0 -> band 0
    uint32_t rank;
    if (RANK == 1) {
      uint32_t* hw = reinterpret_cast<uint32_t*>(myhist);
      const uint32_t sh = (band & 1u) << 4;
      const uint32_t old = act ? atomicAdd(hw + (band >> 1), 1u << sh) : 0u;
      rank = (old >> sh) & 0xffffu;
    } else if (RANK == 2) {
      // peers = the lanes of this round with my band: OR of lane bits into the warp's
      // mask of the band (order-independent), so ranks are lane (= arrival) order by construction
      uint32_t* pm = sm.pmask + warp * nbp;
      if (act) atomicOr(pm + band, 1u << lane);
      __syncwarp();
      const uint32_t peers = act ? pm[band] : 0u;
      const uint32_t below = peers & lanemask_lt();
      const uint32_t base = act ? (uint32_t)myhist[band] : 0u;
      __syncwarp();
      if (act && below == 0u) {                  // lowest peer: advance the histogram, clear the mask
        myhist[band] = (uint16_t)(base + __popc(peers));
        pm[band] = 0u;
      }
      __syncwarp();
      rank = base + __popc(below);
    } else {
      // warp multi-split: lanes whose band equals mine
      unsigned peers = __ballot_sync(kFull, act);
#pragma unroll
      for (int bit = 0; bit < 10; ++bit) {   // nb <= 1024
        const bool bset = (band >> bit) & 1u;
        const unsigned bb = __ballot_sync(kFull, bset);
        peers &= bset ? bb : ~bb;
      }
      if (!act) peers = 0u;
      const uint32_t rl = __popc(peers & lanemask_lt());
      uint32_t base = 0;
      if (act && rl == 0) {
        base = myhist[band];
        myhist[band] = (uint16_t)(base + __popc(peers));
      }
      base = __shfl_sync(kFull, base, act ? (__ffs(peers) - 1) : lane);
      __syncwarp();
      rank = base + rl;
    }
    tl[r] = (uint32_t)t;
    pr[r] = pix | ((p < 0 && !(act && bad)) ? 0x80000000u : 0u);
    key[r] = band | (rank << 10);
  }
  __syncthreads();                               // raw consumed

  if (threadIdx.x == 0) {                        // tile time base; then the next tile's records
    const int64_t t0 = *reinterpret_cast<const int64_t*>(raw), t1 = *reinterpret_cast<const int64_t*>(raw + ne - 1);
    a.tile_t0[tile] = t0;
    *s_wide = (t1 - t0) > (int64_t)0xFFFFFFFFLL;
    a.tile_wide[tile] = *s_wide;
    const int next = (int)atomicAdd(a.tile_ctr, 1u);   // the CTA's next tile (claimed in order)
    *s_next = next;
    if (next < a.n_tiles) {
      if (VALIDATE) *s_tprev = a.ev[(int64_t)next * kTile - 1].t_us;   // the next tile's predecessor
      issue_tile_load(a, sm, next, mbar);
    }
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // the previous sorted tile has left sbuf
  }

  // Per band: exclusive prefix over the warps' counts, then an exclusive scan over
  // the bands -> boff, and the band's meta entry.  Four bands per thread as two
  // packed u16 pairs (a warp counts <= 256 events of a band, a tile <= 4096, so
  // the halves never carry); the threads with bands are whole warps at the front.
  const int nq4 = nbp >> 2;                      // nbp is a multiple of 8
  const int b0 = 4 * (int)threadIdx.x;
  uint32_t t01 = 0, t23 = 0, loc = 0, incl = 0;
  if ((int)threadIdx.x < nq4) {
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int w = 0; w < kPartWarps; ++w) {
      uint2* hp = reinterpret_cast<uint2*>(hist + w * nbp + b0);
      const uint2 c = *hp;
      *hp = make_uint2(lo, hi);
      lo += c.x;
      hi += c.y;
    }
    t01 = lo;
    t23 = hi;
    loc = (lo & 0xffffu) + (lo >> 16) + (hi & 0xffffu) + (hi >> 16);
  }
  const int nqw = (nq4 + 31) >> 5;               // warps holding bands
  if (warp < nqw) {
    incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
  }
  __syncthreads();
  if ((int)threadIdx.x < nq4) {
    uint32_t o0 = incl - loc;
    for (int w = 0; w < warp; ++w) o0 += wsum[w];
    const uint32_t c0 = t01 & 0xffffu, c1 = t01 >> 16, c2 = t23 & 0xffffu, c3 = t23 >> 16;
    const uint32_t o1 = o0 + c0, o2 = o1 + c1, o3 = o2 + c2;
    *reinterpret_cast<uint4*>(boff + b0) = make_uint4(o0, o1, o2, o3);
    const int nt = a.n_tiles;
    uint32_t* mp = a.meta + (int64_t)b0 * nt + tile;
    if (b0 < a.nb) mp[0] = o0 | (c0 << 16);
    if (b0 + 1 < a.nb) mp[nt] = o1 | (c1 << 16);
    if (b0 + 2 < a.nb) mp[2 * nt] = o2 | (c2 << 16);
    if (b0 + 3 < a.nb) mp[3 * nt] = o3 | (c3 << 16);
  }
  __syncthreads();

#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    if (FULL || warp * WEV + r * 32 + lane < ne) {
      const uint32_t band = key[r] & 0x3ffu;
      const uint32_t pos = boff[band] + hist[warp * nbp + band] + (key[r] >> 10);
      ESI_DCHECK(band < (uint32_t)a.nb && pos < (uint32_t)ne);
      sbuf[pos] = make_uint2(tl[r], pr[r]);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  // sorted tile -> global with one TMA bulk copy (async proxy; the generic-proxy
  // shared-memory writes above were fenced by every writer before the barrier)
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(ne & ~1) * 8u;
    if (bytes) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(a.rec + e0), "r"((uint32_t)__cvta_generic_to_shared(sbuf)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if (ne & 1) a.rec[e0 + ne - 1] = sbuf[ne - 1];
  }

  if (*s_wide) {  // rare: tile spans >= 2^32 us; keep the full timestamps beside the records
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int i = warp * WEV + r * 32 + lane;
      if (i < ne) {
        const uint32_t band = key[r] & 0x3ffu;
        const uint32_t pos = boff[band] + hist[warp * nbp + band] + (key[r] >> 10);
        a.wide_t[e0 + pos] = ev[i].t_us;
      }
    }
    __syncthreads();                             // hist is cleared next
  }
  // clear the histograms for the next tile (the loop's barrier orders it before the ranking)
  for (int i = threadIdx.x; i < kPartWarps * nbp / 8; i += kPartThreads)
    reinterpret_cast<uint4*>(hist)[i] = make_uint4(0u, 0u, 0u, 0u);
}

template <int RANK, bool VALIDATE, bool BAND32>
__global__ void __launch_bounds__(kPartThreads, kPartCtas) esi_partition_kernel(PartArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t s_mbar;
  __shared__ int64_t s_tprev;
  __shared__ int s_wide;
  // (the host launches K1 only for chunks whose first event is <= the render's last frame; a
  // sync-free single-chunk render has not read the plan back and leaves that test to the kernel)
  if (a.gate_info && !a.gate_info->active) return;
  const int nbp = (a.nb + 7) & ~7;
  PartSmem sm;
  sm.raw = reinterpret_cast<int4*>(smem);
  sm.sbuf = reinterpret_cast<uint2*>(sm.raw + kTile);
  sm.hist = reinterpret_cast<uint16_t*>(sm.sbuf + kTile);
  sm.boff = reinterpret_cast<uint32_t*>(sm.hist + kPartWarps * nbp);
  sm.wsum = sm.boff + nbp + 8;
  sm.pmask = sm.wsum + 64;
  const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
  __shared__ int s_next;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int t0 = (int)atomicAdd(a.tile_ctr, 1u);   // tiles are claimed dynamically: CTAs that start
    s_next = t0;                                     // early (beside K2's tail) take more of them
    if (t0 < a.n_tiles) {
      if (VALIDATE) s_tprev = t0 > 0 ? a.ev[(int64_t)t0 * kTile - 1].t_us : *a.prev_t;
      issue_tile_load(a, sm, t0, mbar);
    }
  }
  for (int i = threadIdx.x; i < kPartWarps * nbp / 8; i += kPartThreads)
    reinterpret_cast<uint4*>(sm.hist)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (RANK == 2)
    for (int i = threadIdx.x; i < kPartWarps * nbp; i += kPartThreads) sm.pmask[i] = 0u;
  for (uint32_t k = 0;; ++k) {
    __syncthreads();                             // histograms clear, s_next / s_tprev / s_wide settled
    const int tile = s_next;
    if (tile >= a.n_tiles) break;
    mbar_wait_parity(mbar, k & 1u);              // this tile's records have landed
    const int ne = (int)min((int64_t)kTile, a.n - (int64_t)tile * kTile);
    if (ne == kTile) partition_tile<RANK, VALIDATE, BAND32, true>(a, sm, tile, ne, mbar, &s_tprev, &s_wide, &s_next);
    else partition_tile<RANK, VALIDATE, BAND32, false>(a, sm, tile, ne, mbar, &s_tprev, &s_wide, &s_next);
  }
  if (threadIdx.x == 0) {                        // the last CTA out resets the counters for the next launch
    if (atomicAdd(a.tile_ctr + 1, 1u) == gridDim.x - 1) {
      a.tile_ctr[0] = 0u;
      a.tile_ctr[1] = 0u;
    }
  }
  // the CTA may retire once the last bulk store has READ sbuf; the global writes
  // complete asynchronously (K2 runs after this kernel)
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <int RA, bool V, bool B32>
static cudaError_t launch_part_t(const PartArgs& a, int n_tiles, cudaStream_t s) {
  const size_t smem = partition_smem_bytes(a.nb, RA);
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<int> configured[64];   // zero-initialised; set-once flags (idempotent, race-free)   // per device (the attribute is per context); the maximum once
  static std::atomic<int> n_sm[64];
  static std::atomic<uint64_t> occ[64];   // (band count << 32) | resident CTAs per SM
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!configured[dev].load(std::memory_order_acquire)) {
    int nsm = 0;
    cudaError_t e = cudaFuncSetAttribute(esi_partition_kernel<RA, V, B32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)partition_smem_bytes(kMaxBands, RA));
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    n_sm[dev].store(nsm, std::memory_order_relaxed);
    configured[dev].store(1, std::memory_order_release);
  }
  uint64_t oc = occ[dev].load(std::memory_order_relaxed);
  if ((oc >> 32) != (uint64_t)(uint32_t)a.nb || (oc & 0xffffffffu) == 0) {
    int o = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, esi_partition_kernel<RA, V, B32>, kPartThreads, smem);
    if (e != cudaSuccess) return e;
    oc = ((uint64_t)(uint32_t)a.nb << 32) | (uint32_t)(o > 0 ? o : 1);
    occ[dev].store(oc, std::memory_order_relaxed);
  }
  const int grid = (int)std::min<int64_t>(n_tiles, (int64_t)(oc & 0xffffffffu) * n_sm[dev].load(std::memory_order_relaxed));   // persistent CTAs
  PartArgs b = a;
  b.n_tiles = n_tiles;
  esi_partition_kernel<RA, V, B32><<<grid, kPartThreads, smem, s>>>(b);
  return cudaGetLastError();
}

template <int RA>
static cudaError_t launch_part_r(const PartArgs& a, int n_tiles, cudaStream_t s) {
  return a.validate ? launch_part_t<RA, true, true>(a, n_tiles, s) : launch_part_t<RA, false, true>(a, n_tiles, s);
}

cudaError_t launch_partition(const PartArgs& a, int n_tiles, int rank_mode, cudaStream_t s) {
  return rank_mode == 1 ? launch_part_r<1>(a, n_tiles, s)
         : rank_mode == 2 ? launch_part_r<2>(a, n_tiles, s)
                          : launch_part_r<0>(a, n_tiles, s);
}

// Probe: do warp-wide shared-memory atomicAdds on one address return values in
// ascending lane order?  (ballot-derived stable ranks vs atomic ranks, random keys)
__global__ void esi_probe_atomic_order_kernel(unsigned* bad) {
  __shared__ unsigned h[4][512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < 512; i += 32) h[warp][i] = 0;
  __syncwarp();
  unsigned v = (blockIdx.x * 977u + threadIdx.x) * 2654435761u, nbad = 0;
  for (int it = 0; it < 256; ++it) {
    v = v * 1664525u + 1013904223u;
    unsigned key = (v >> 9) & ((it & 3) == 0 ? 1u : ((it & 3) == 1 ? 15u : 511u));
    unsigned peers = kFull;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
      const unsigned bb = __ballot_sync(kFull, (key >> b) & 1u);
      peers &= ((key >> b) & 1u) ? bb : ~bb;
    }
    const unsigned before = h[warp][key];
    __syncwarp();
    const unsigned r = atomicAdd(&h[warp][key], 1u);
    __syncwarp();
    nbad += r != before + __popc(peers & lanemask_lt());
  }
  if (nbad) atomicAdd(bad, nbad);
}

cudaError_t probe_atomic_order(unsigned* d_bad, cudaStream_t s) {
  esi_probe_atomic_order_kernel<<<148, 128, 0, s>>>(d_bad);
  return cudaGetLastError();
}

}  // namespace esi
