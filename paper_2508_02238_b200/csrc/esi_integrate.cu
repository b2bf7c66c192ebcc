// esi_integrate.cu -- K2 (general variant): per-band integration (Alg. 2) fused
// with the frame readout (Eq. 14) for every frame of the chunk, with 64-bit
// times throughout.  Used for chunks the fast kernel (esi_integrate_fast.cu)
// cannot take: spans >= 2^30 us, decay horizons >= 2^23 us (k < 0.12 /s).
//
// One CTA per band of BP = NW*256 consecutive pixel ids; warp w owns the
// 256-pixel sub-band [w*256, w*256+256) and lane l its 8 pixels.  The band's
// state S (fp32) and T (int64) is staged in shared memory for the whole chunk.
//
//  1. The band's events are gathered from the K1 tiles in tile order (= arrival
//     order) into a shared-memory sub-batch of <= kSubBatch events.
//  2. Each warp filters the sub-batch down to its own sub-band (ballot
//     compaction, order kept).
//  3. Each warp walks its list 32 events at a time.  Events with t <= t_j of
//     the next frame j are applied with Alg. 2; lanes that hit the
//     same pixel are serialised lowest-lane-first (smem atomicMin tag), which
//     is arrival order, so every pixel sees its events exactly in stream order
//     (bit-identical to a sequential fp32 evaluation).  When the next event is
//     later than t_j, frame j is read out for the warp's 256 pixels (fused
//     Eq. 14 map, 8-byte streaming stores) before the event is applied.
//  4. After the last sub-batch the remaining frames of the chunk are read out
//     and S, T are written back.
// Frame j is rendered in the chunk c with t_first(c) <= t_j < t_first(c+1), so
// all events with t <= t_j have been integrated (ties belong to the frame,
// reading A6) and none later.
#include <atomic>
#include "esi_device.cuh"

namespace esi {

size_t integrate_smem_bytes(int band_px) {
  const int nw = band_px / kWarpPx;
  return (size_t)band_px * (sizeof(int64_t) + sizeof(double) + sizeof(int32_t)) +
         (size_t)kSubBatch * (sizeof(int64_t) + sizeof(uint32_t)) +
         (size_t)(2 * kMaxTilesPerChunk + 1) * sizeof(uint32_t) +
         (size_t)nw * kSubBatch * sizeof(uint16_t) + 64;
}

template <int NW>
struct IntCtx {
  static constexpr int BP = NW * kWarpPx;
  int64_t* Tsm;
  double* Ssm;
  int32_t* tag;
  int64_t* At;
  uint32_t* Apr;
  uint32_t* pre;   // [n_tiles + 1] exclusive prefix of the band's per-tile counts
  uint32_t* mt;    // [n_tiles] meta (offset | count << 16)
  uint16_t* L;
};

// Eq. 4 in fp64 (reading A14: d = 0 exactly from dt_cut = ceil(1e6/k) on)
__device__ __forceinline__ double wide_decay(int64_t dt, const WideParams& wp) {
  if (wp.bmode == kDecayNone) return 1.0;   // Eq. 2
  if (dt >= wp.dt_cut) return 0.0;
  if (wp.bmode == kDecayExp) return exp(-wp.k_us * (double)dt);   // exponential variant (A20)
  const double u = 1.0 - wp.k_us * (double)dt;
  if (u <= 0.0) return 0.0;
  return wp.bmode == 2 ? u * u : pow(u, wp.b);
}

// Eq. 13 + Eq. 14 in fp64, rounded half away from zero (reading A8).
__device__ __forceinline__ uint32_t wide_map8(double v, const WideParams& wp) {
  v = fmin(fmax(v, wp.smin), wp.smax);
  const int q = (int)floor(v * wp.scale + wp.off5);
  return (uint32_t)min(max(q, 0), 255);
}

template <int NW>
__device__ __forceinline__ void warp_readout(const IntArgs& a, const IntCtx<NW>& c, int j,
                                             int band, int npx, int warp, int lane) {
  const int base = warp * kWarpPx + lane * 8;
  if (base >= npx) return;
  const int64_t tj = a.tf[j];
  uint32_t bytes[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    double v = c.Ssm[base + q];
    if (a.wp.readout_decay) v *= wide_decay(tj - c.Tsm[base + q], a.wp);
    bytes[q] = wide_map8(v, a.wp);
  }
  uint8_t* dst = a.out + (int64_t)j * a.P + band_gpix(a.bm, band, base);   // 8 pixels never straddle a 64-pixel group
  if (a.vec8 && base + 8 <= npx) {
    const uint32_t lo = bytes[0] | (bytes[1] << 8) | (bytes[2] << 16) | (bytes[3] << 24);
    const uint32_t hi = bytes[4] | (bytes[5] << 8) | (bytes[6] << 16) | (bytes[7] << 24);
    st_stream8(dst, lo, hi);
  } else {
    const int nq = min(8, npx - base);
    for (int q = 0; q < nq; ++q) dst[q] = (uint8_t)bytes[q];
  }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) esi_integrate_wide_kernel(IntArgs a) {
  constexpr int BP = NW * kWarpPx;
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) unsigned char smem[];
  IntCtx<NW> c;
  c.Tsm = reinterpret_cast<int64_t*>(smem);
  c.At = c.Tsm + BP;
  c.Ssm = reinterpret_cast<double*>(c.At + kSubBatch);
  c.tag = reinterpret_cast<int32_t*>(c.Ssm + BP);
  c.Apr = reinterpret_cast<uint32_t*>(c.tag + BP);
  c.pre = c.Apr + kSubBatch;
  c.mt = c.pre + kMaxTilesPerChunk + 1;
  c.L = reinterpret_cast<uint16_t*>(c.mt + kMaxTilesPerChunk);
  __shared__ int64_t s_tnext;
  __shared__ uint32_t s_wsum[32];

  const int band = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npx = band_npx(a.bm, band, a.P);                // interleaved bands (esi_internal.cuh); band_px <= BP

  if (a.gate && *a.gate != kNoError) return;   // lazy validation found an invalid event: write nothing
  const ChunkInfo ci = *a.info;
  if (a.kind_gate == 2 && ci.fast) return;     // the fast kernel renders this chunk
  const int f_lo = ci.f_lo, f_hi = ci.f_hi;
  const bool active = ci.active != 0;
  if (!active && f_lo >= f_hi) return;
  const bool wide = ci.wide != 0;
  const int64_t tbase = ci.tbase;
  const int n_tiles = a.n_tiles;

  for (int i = threadIdx.x; i < BP; i += NT) {
    const bool in = i < npx;
    const int64_t g = band_gpix(a.bm, band, i);
    c.Ssm[i] = in ? (double)a.S[g] : 0.0;
    c.Tsm[i] = in ? a.T[g] : 0;
    c.tag[i] = 32;
  }
  int n_b = 0;
  if (active) {
    for (int t = threadIdx.x; t < n_tiles; t += NT) c.mt[t] = a.meta[(int64_t)band * n_tiles + t];
    __syncthreads();
    // exclusive prefix of the per-tile counts: thread i owns tiles [i*per, (i+1)*per)
    const int per = (n_tiles + NT - 1) / NT;
    const int t0 = threadIdx.x * per;
    uint32_t local = 0;
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) local += c.mt[t] >> 16;
    uint32_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t run = x - local, tot = 0;
    for (int w = 0; w < NW; ++w) {
      const uint32_t v = s_wsum[w];
      if (w < warp) run += v;
      tot += v;
    }
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) {
      c.pre[t] = run;
      run += c.mt[t] >> 16;
    }
    if (threadIdx.x == 0) c.pre[n_tiles] = tot;
    n_b = (int)tot;
    if (a.bstats && threadIdx.x == 0) {            // ESI_BANDS_AUTO: this band's share of the chunk
      atomicMax(a.bstats, (unsigned long long)n_b);
      atomicAdd(a.bstats + 1, (unsigned long long)n_b);
      atomicAdd(a.bstats + 2, 1ull);
    }
  }
  __syncthreads();

  const double C = a.wp.C;
  int j = f_lo;
  bool done = false;

  for (int sb0 = 0; sb0 < n_b; sb0 += kSubBatch) {
    const int n_sb = min(kSubBatch, n_b - sb0);
    const int n_ext = n_sb + (sb0 + n_sb < n_b ? 1 : 0);   // + first event of the next sub-batch
    // 1. gather (arrival order): every position finds its tile by binary search in pre[]
    for (int qq = threadIdx.x; qq < n_ext; qq += NT) {
      const uint32_t q = (uint32_t)(sb0 + qq);
      int lo = 0, hi = n_tiles;   // largest t with pre[t] <= q
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (c.pre[mid] <= q) lo = mid; else hi = mid;
      }
      const int64_t idx = (int64_t)lo * kTile + (c.mt[lo] & 0xffffu) + (q - c.pre[lo]);
      const uint2 r = a.rec[idx];
      int64_t tt;
      if (!wide) {
        tt = tbase + (int64_t)(uint32_t)(r.x - (uint32_t)tbase);
      } else if (a.tile_wide[lo]) {
        tt = a.wide_t[idx];
      } else {
        const int64_t tb = a.tile_t0[lo];
        tt = tb + (int64_t)(uint32_t)(r.x - (uint32_t)tb);
      }
      if (qq < n_sb) {
        c.At[qq] = tt;
        c.Apr[qq] = r.y;
      } else {
        s_tnext = tt;
      }
    }
    if (n_ext == n_sb && threadIdx.x == 0) s_tnext = INT64_MAX;
    __syncthreads();
    const int64_t tnext = s_tnext;

    // 2. warp filter (keeps arrival order)
    uint16_t* Lw = c.L + warp * kSubBatch;
    int n_w = 0;
    for (int q0 = 0; q0 < n_sb; q0 += 32) {
      const int q = q0 + lane;
      const bool mine = q < n_sb && (int)((c.Apr[q] & (uint32_t)(BP - 1)) >> 8) == warp;
      const unsigned bal = __ballot_sync(kFull, mine);
      if (mine) Lw[n_w + __popc(bal & lanemask_lt())] = (uint16_t)q;
      n_w += __popc(bal);
    }
    __syncwarp();

    // 3. walk: apply events, reading frames out at their boundaries
    int i = 0;
    while (!done && i < n_w) {
      const int64_t tj = (j < f_hi) ? a.tf[j] : a.t_cap;
      const int m = min(32, n_w - i);
      int64_t te = 0;
      uint32_t pr = 0;
      if (lane < m) {
        const int idx = Lw[i + lane];
        te = c.At[idx];
        pr = c.Apr[idx];
      }
      const bool valid = lane < m && te <= tj;
      const int nv = __popc(__ballot_sync(kFull, valid));
      if (nv > 0) {
        bool pend = lane < nv;
        const int px = (int)(pr & (uint32_t)(BP - 1));
        while (__any_sync(kFull, pend)) {
          if (pend) atomicMin(&c.tag[px], lane);
          __syncwarp();
          const bool win = pend && c.tag[px] == lane;
          __syncwarp();
          if (win) {
            // Alg. 2 loop body
            const double pc = ((int32_t)pr < 0) ? -C : C;
            const double d = wide_decay(te - c.Tsm[px], a.wp);
            const double s = a.wp.first ? c.Ssm[px] * d + pc          // variant: decay, then add
                                        : (c.Ssm[px] + pc) * d;      // Alg. 2: S <- (S + p C) d(t - T)
            c.Ssm[px] = a.wp.unclamped ? s                              // Eq. 2 / unclamped variants
                                       : fmin(fmax(s, a.wp.smin), a.wp.smax);   // clamp (Eq. 13)
            c.Tsm[px] = te;                                           // T <- t
            c.tag[px] = 32;
            pend = false;
          }
          __syncwarp();
        }
      }
      i += nv;
      if (nv < m) {
        if (j < f_hi) {
          warp_readout<NW>(a, c, j, band, npx, warp, lane);
          ++j;
        } else {
          done = true;  // the rest is later than the last frame: stays pending
        }
      }
    }
    // 4. frames whose events are all in this or earlier sub-batches
    while (j < f_hi && a.tf[j] < tnext) {
      warp_readout<NW>(a, c, j, band, npx, warp, lane);
      ++j;
    }
    __syncthreads();
  }
  while (j < f_hi) {
    warp_readout<NW>(a, c, j, band, npx, warp, lane);
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += NT) {
      const int64_t g = band_gpix(a.bm, band, i);
      a.S[g] = (float)c.Ssm[i];
      a.T[g] = c.Tsm[i];
    }
  }
}

template <int NW>
static cudaError_t launch_nw(const IntArgs& a, cudaStream_t s) {
  const size_t smem = integrate_smem_bytes(NW * kWarpPx);
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<int> configured[64];   // zero-initialised; set-once flags (idempotent, race-free)   // per device (the attribute is per context)
  if (dev < 0 || dev >= 64 || !configured[dev].load(std::memory_order_relaxed)) {
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_wide_kernel<NW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev].store(1, std::memory_order_relaxed);
  }
  esi_integrate_wide_kernel<NW><<<a.nb, NW * 32, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_integrate(const IntArgs& a, cudaStream_t s) {
  // 16 warps x 256 pixels cover any band (band_px <= kMaxBandPx = 4096)
  return launch_nw<16>(a, s);
}

}  // namespace esi
