// esi_integrate.cu -- K2: per-band integration (Alg. 2) fused with the frame
// readout (Eq. 14) for every frame of the chunk.
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
#include "esi_device.cuh"

namespace esi {

size_t integrate_smem_bytes(int band_px) {
  const int nw = band_px / kWarpPx;
  return (size_t)band_px * (sizeof(int64_t) + sizeof(float) + sizeof(int32_t)) +
         (size_t)kSubBatch * (sizeof(int64_t) + sizeof(uint32_t)) +
         (size_t)(kMaxTilesPerChunk + 1) * sizeof(uint32_t) +
         (size_t)nw * kSubBatch * sizeof(uint16_t) + 64;
}

template <int NW>
struct IntCtx {
  static constexpr int BP = NW * kWarpPx;
  int64_t* Tsm;
  float* Ssm;
  int32_t* tag;
  int64_t* At;
  uint32_t* Apr;
  uint32_t* pre;
  uint16_t* L;
};

template <int NW>
__device__ __forceinline__ void warp_readout(const IntArgs& a, const IntCtx<NW>& c, int j,
                                             int64_t px0, int npx, int warp, int lane) {
  const int base = warp * kWarpPx + lane * 8;
  if (base >= npx) return;
  const int64_t tj = a.tf[j];
  const float4 s0 = *reinterpret_cast<const float4*>(c.Ssm + base);
  const float4 s1 = *reinterpret_cast<const float4*>(c.Ssm + base + 4);
  const float s[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  uint32_t bytes[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float v = s[q];
    if (a.mp.readout_decay) v *= esi_decay(tj - c.Tsm[base + q], a.dp);
    bytes[q] = esi_map8(v, a.mp);
  }
  uint8_t* dst = a.out + (int64_t)j * a.P + px0 + base;
  if (a.vec8 && base + 8 <= npx) {
    const uint32_t lo = bytes[0] | (bytes[1] << 8) | (bytes[2] << 16) | (bytes[3] << 24);
    const uint32_t hi = bytes[4] | (bytes[5] << 8) | (bytes[6] << 16) | (bytes[7] << 24);
    st_stream8(dst, lo, hi);
  } else {
    const int nq = min(8, npx - base);
    for (int q = 0; q < nq; ++q) dst[q] = (uint8_t)bytes[q];
  }
}

// t of the band event at band position q (thread-local helper, cold path)
__device__ int64_t band_event_time(const IntArgs& a, const uint32_t* pre, int band, int q,
                                   int wide_chunk, int64_t tbase) {
  int lo = 0, hi = a.n_tiles;  // largest t with pre[t] <= q
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= (uint32_t)q) lo = mid; else hi = mid;
  }
  // skip empty tiles (pre[lo] == pre[lo+1])
  while (pre[lo + 1] <= (uint32_t)q) ++lo;
  const uint32_t m = a.meta[(int64_t)band * a.n_tiles + lo];
  const int64_t idx = (int64_t)lo * kTile + (m & 0xffffu) + (q - pre[lo]);
  if (wide_chunk) {
    if (a.tile_wide[lo]) return a.wide_t[idx];
    const int64_t t0 = a.tile_t0[lo];
    return t0 + (int64_t)(uint32_t)(a.rec[idx].x - (uint32_t)t0);
  }
  return tbase + (int64_t)(uint32_t)(a.rec[idx].x - (uint32_t)tbase);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32) esi_integrate_kernel(IntArgs a) {
  constexpr int BP = NW * kWarpPx;
  constexpr int NT = NW * 32;
  extern __shared__ __align__(16) unsigned char smem[];
  IntCtx<NW> c;
  c.Tsm = reinterpret_cast<int64_t*>(smem);
  c.At = c.Tsm + BP;
  c.Ssm = reinterpret_cast<float*>(c.At + kSubBatch);
  c.tag = reinterpret_cast<int32_t*>(c.Ssm + BP);
  c.Apr = reinterpret_cast<uint32_t*>(c.tag + BP);
  c.pre = c.Apr + kSubBatch;
  c.L = reinterpret_cast<uint16_t*>(c.pre + kMaxTilesPerChunk + 1);
  __shared__ int s_flo, s_fhi, s_active, s_wide;
  __shared__ int64_t s_tbase, s_tnext;
  __shared__ uint32_t s_wsum[32];

  const int band = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t px0 = (int64_t)band * BP;
  const int npx = (int)min((int64_t)BP, a.P - px0);

  if (threadIdx.x == 0) {
    const int64_t tfirst = a.ev[0].t_us;
    s_flo = a.first_chunk ? 0 : lower_bound_i64(a.tf, a.F, tfirst);
    s_fhi = a.ev_next ? lower_bound_i64(a.tf, a.F, a.ev_next->t_us) : a.F;
    s_active = tfirst <= a.t_cap;
    s_tbase = tfirst;
    s_wide = (a.ev[a.n - 1].t_us - tfirst) > (int64_t)0xFFFFFFFFLL;
  }
  __syncthreads();
  const int f_lo = s_flo, f_hi = s_fhi;
  const bool active = s_active;
  if (!active && f_lo >= f_hi) return;

  for (int i = threadIdx.x; i < BP; i += NT) {
    const bool in = i < npx;
    c.Ssm[i] = in ? a.S[px0 + i] : 0.f;
    c.Tsm[i] = in ? a.T[px0 + i] : 0;
    c.tag[i] = 32;
  }
  int n_b = 0;
  if (active) {
    // exclusive prefix of this band's per-tile counts -> pre[0..n_tiles]
    uint32_t carry = 0;
    for (int t0 = 0; t0 < a.n_tiles; t0 += NT) {
      const int t = t0 + threadIdx.x;
      const uint32_t cnt = t < a.n_tiles ? (a.meta[(int64_t)band * a.n_tiles + t] >> 16) : 0u;
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[warp] = x;
      __syncthreads();
      uint32_t wpre = 0, tot = 0;
      for (int w = 0; w < NW; ++w) {
        const uint32_t v = s_wsum[w];
        if (w < warp) wpre += v;
        tot += v;
      }
      if (t < a.n_tiles) c.pre[t] = carry + wpre + x - cnt;
      carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) c.pre[a.n_tiles] = carry;
    n_b = (int)carry;
  }
  __syncthreads();

  const bool wide = s_wide;
  const int64_t tbase = s_tbase;
  const float C = a.mp.C;
  int j = f_lo;
  bool done = false;

  for (int sb0 = 0; sb0 < n_b; sb0 += kSubBatch) {
    const int n_sb = min(kSubBatch, n_b - sb0);
    // 1. gather the sub-batch (tile order = arrival order)
    int tstart;
    {
      int lo = 0, hi = a.n_tiles;  // largest t with pre[t] <= sb0
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (c.pre[mid] <= (uint32_t)sb0) lo = mid; else hi = mid;
      }
      tstart = lo;
    }
    for (int t = tstart + warp; t < a.n_tiles && c.pre[t] < (uint32_t)(sb0 + n_sb); t += NW) {
      const int q0 = max((int)c.pre[t], sb0);
      const int q1 = min((int)c.pre[t + 1], sb0 + n_sb);
      if (q0 >= q1) continue;
      const uint32_t m = a.meta[(int64_t)band * a.n_tiles + t];
      const int64_t rbase = (int64_t)t * kTile + (m & 0xffffu) - c.pre[t];
      bool twide = false;
      int64_t t0 = tbase;
      if (wide) { twide = a.tile_wide[t]; t0 = a.tile_t0[t]; }
      for (int q = q0 + lane; q < q1; q += 32) {
        const uint2 r = a.rec[rbase + q];
        const int64_t tt = twide ? a.wide_t[rbase + q] : t0 + (int64_t)(uint32_t)(r.x - (uint32_t)t0);
        c.At[q - sb0] = tt;
        c.Apr[q - sb0] = r.y;
      }
    }
    if (threadIdx.x == 0)
      s_tnext = (sb0 + kSubBatch < n_b) ? band_event_time(a, c.pre, band, sb0 + kSubBatch, wide, tbase)
                                        : INT64_MAX;
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
            float s = c.Ssm[px] + (((int32_t)pr < 0) ? -C : C);     // S <- S + p C
            s *= esi_decay(te - c.Tsm[px], a.dp);                     // S <- S * d(t - T)
            c.Ssm[px] = fminf(fmaxf(s, a.mp.smin), a.mp.smax);        // clamp (Eq. 13)
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
          warp_readout<NW>(a, c, j, px0, npx, warp, lane);
          ++j;
        } else {
          done = true;  // the rest is later than the last frame: stays pending
        }
      }
    }
    // 4. frames whose events are all in this or earlier sub-batches
    while (j < f_hi && a.tf[j] < tnext) {
      warp_readout<NW>(a, c, j, px0, npx, warp, lane);
      ++j;
    }
    __syncthreads();
  }
  while (j < f_hi) {
    warp_readout<NW>(a, c, j, px0, npx, warp, lane);
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += NT) {
      a.S[px0 + i] = c.Ssm[i];
      a.T[px0 + i] = c.Tsm[i];
    }
  }
}

template <int NW>
static cudaError_t launch_nw(const IntArgs& a, cudaStream_t s) {
  const size_t smem = integrate_smem_bytes(NW * kWarpPx);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_kernel<NW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  esi_integrate_kernel<NW><<<a.nb, NW * 32, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_integrate(const IntArgs& a, cudaStream_t s) {
  switch (a.band_px / kWarpPx) {
    case 1: return launch_nw<1>(a, s);
    case 2: return launch_nw<2>(a, s);
    case 4: return launch_nw<4>(a, s);
    case 8: return launch_nw<8>(a, s);
    case 16: return launch_nw<16>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace esi
