// esi_integrate_fast.cu -- K2: per-band integration (Alg. 2) fused
// with the Eq. 14 readout of every frame of the chunk.
//
// Same structure as the general variant (esi_integrate.cu) but every time is a
// 32-bit offset from the chunk's base ChunkInfo::trel, state T is held as such
// an offset in shared memory (clamped at -(dt_cut+1): older is "fully
// decayed"), and the decay/readout arithmetic avoids conversions:
//   * dt -> float via the 2^23 magic constant (dt <= dt_cut < 2^23),
//   * floor(x) + off_int -> byte via a round-down add of 2^23 + off_int
//     (the low byte of the float's bits is the gray value).
// One CTA per band of NW*256 pixels; warp w owns pixels [w*256, w*256+256).
// Per sub-batch of <= kSubBatch band events (arrival order):
//   1. warp w gathers slice w of the sub-batch from the K1 tiles (coalesced
//      within tile segments; tile found by a lane-local linear advance) and
//      counts, per destination warp, how many of its events it routes there;
//   2. after a block barrier each warp scatters the indices of its slice into
//      the destination warps' lists at (earlier slices' counts + running rank):
//      a stable NW-way split, so every list is in arrival order;
//   3. each warp walks its list 32 events at a time and reads frame j out
//      (fused Eq. 14, 8-byte streaming stores) before the first event later
//      than t_j.  Per batch the density decides the path (__match_any_sync):
//      every pixel hit once -> the Alg. 2 body applied directly (sparse path,
//      bit-identical to sequential fp32); some pixel hit several times -> a
//      warp-shuffle inclusive scan of the clamped affine maps along each
//      pixel's chain (dense path, dense_batch_apply).
#include "esi_device.cuh"

namespace esi {

namespace {

constexpr float kMagic = 8388608.0f;   // 2^23

template <int BM>
__device__ __forceinline__ float fast_decay(int32_t dt, const DecayParams& dp, int32_t dt_cut) {
  const bool live = dt < dt_cut;                               // 1 - k dt > 0 exactly (reading A14)
  dt = min(dt, dt_cut);                                        // dt >= 0 (sorted stream)
  const float f = __int_as_float(dt | 0x4B000000) - kMagic;    // exact int -> float
  float u = fmaf(-f, dp.kh, 1.0f);                             // u = 1 - k dt  (Eq. 4)
  u = fmaf(-f, dp.kl, u);
  if (BM == 2) return live ? u * u : 0.f;                      // d = 0 exactly past the horizon
  return (live && u > 0.f) ? exp2f(dp.b * log2f(u)) : 0.f;
}

// Eq. 13 + Eq. 14, result in the low byte of the returned word.
__device__ __forceinline__ uint32_t fast_map(float v, const MapParams& mp, float magic_off) {
  v = fminf(fmaxf(v, mp.smin), mp.smax);
  const float x = fmaf(v, mp.scale, mp.off_frac);
  return __float_as_uint(__fadd_rd(x, magic_off));             // 2^23 + off_int + floor(x)
}


// Clamped affine map s -> clamp(a s + c, lo, hi) with a >= 0 (SURVEY section 0,
// finding 1).  The Alg. 2 body of event i is the map
// f_i = (d_i, d_i p_i C, S_min, S_max); such maps are closed under composition:
//   F o G = (aF aG, aF cG + cF, clamp(aF loG + cF, loF, hiF), clamp(aF hiG + cF, loF, hiF)).
// Dense batch (some pixel hit by several of the warp's 32 events): each lane
// builds its event's map, then a pointer-jumping inclusive scan along the
// per-pixel chains (previous event of the same pixel = highest lower peer lane
// from __match_any_sync) composes every prefix in <= 5 shuffle rounds; lane i's
// state is prefix_i applied to the pixel's state before the batch.  Pixels hit
// once keep the direct Alg. 2 arithmetic (bit-identical to the sparse path).
template <int BM>
__device__ __forceinline__ void dense_batch_apply(float* S, int32_t* T, bool act, int px, unsigned peers,
                                                  int32_t te, float pc, int lane, const DecayParams& dp,
                                                  const MapParams& mp, int32_t dt_cut) {
  const unsigned below = act ? (peers & lanemask_lt()) : 0u;
  const int prev = below ? 31 - __clz(below) : -1;          // previous event of my pixel in the batch
  const int32_t t_prev_lane = __shfl_sync(kFull, te, prev < 0 ? lane : prev);
  float s0 = 0.f;
  int32_t tp = t_prev_lane;
  if (act) {
    s0 = S[px];                                               // state before the batch
    if (prev < 0) tp = T[px];
  }
  __syncwarp();                                               // all reads before any write
  const float d = act ? fast_decay<BM>(te - tp, dp, dt_cut) : 1.f;
  float fa = d, fc = d * pc, flo = mp.smin, fhi = mp.smax;    // f_i
  int ptr = prev;
  while (__any_sync(kFull, ptr >= 0)) {
    const int src = ptr >= 0 ? ptr : lane;
    const float ga = __shfl_sync(kFull, fa, src), gc = __shfl_sync(kFull, fc, src);
    const float glo = __shfl_sync(kFull, flo, src), ghi = __shfl_sync(kFull, fhi, src);
    const int gp = __shfl_sync(kFull, ptr, src);
    if (ptr >= 0) {                                           // F <- F o G
      const float nlo = fminf(fmaxf(fmaf(fa, glo, fc), flo), fhi);
      const float nhi = fminf(fmaxf(fmaf(fa, ghi, fc), flo), fhi);
      fc = fmaf(fa, gc, fc);
      fa = fa * ga;
      flo = nlo;
      fhi = nhi;
      ptr = gp;
    }
  }
  const bool single = __popc(peers) == 1;
  const float v = single ? fminf(fmaxf((s0 + pc) * d, mp.smin), mp.smax)   // direct Alg. 2 body
                         : fminf(fmaxf(fmaf(fa, s0, fc), flo), fhi);       // prefix_i(s0)
  const unsigned above = peers & ~lanemask_lt() & ~(1u << lane);
  if (act && above == 0u) {                                   // last event of its pixel in the batch
    S[px] = v;
    T[px] = te;
  }
}

template <int NW>
struct FastSmem {
  static constexpr int BP = NW * kWarpPx;
  float S[BP];
  int32_t T[BP];
  int32_t At[kSubBatch];
  uint32_t Apr[kSubBatch];
  uint32_t pre[kMaxTilesPerChunk + 1];
  uint32_t mt[kMaxTilesPerChunk];
  uint32_t cnt[NW][NW];
  uint16_t L[NW][kSubBatch];
};

template <int NW, int BM>
__device__ __forceinline__ void fast_readout(const IntArgs& a, FastSmem<NW>& sm, int j, int64_t trel,
                                             int64_t px0, int npx, int warp, int lane, int32_t dt_cut,
                                             float magic_off) {
  const int base = warp * kWarpPx + lane * 8;
  if (base >= npx) return;
  const int32_t tj = (int32_t)(a.tf[j] - trel);
  const float4 s0 = *reinterpret_cast<const float4*>(&sm.S[base]);
  const float4 s1 = *reinterpret_cast<const float4*>(&sm.S[base + 4]);
  const int4 t0 = *reinterpret_cast<const int4*>(&sm.T[base]);
  const int4 t1 = *reinterpret_cast<const int4*>(&sm.T[base + 4]);
  const float s[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
  const int32_t T[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
  const bool rd = a.mp.readout_decay != 0;
  uint32_t r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float d = rd ? fast_decay<BM>(tj - T[q], a.dp, dt_cut) : 1.0f;
    r[q] = fast_map(s[q] * d, a.mp, magic_off);
  }
  uint8_t* dst = a.out + (int64_t)j * a.P + px0 + base;
  if (a.vec8 && base + 8 <= npx) {
    const uint32_t lo = __byte_perm(__byte_perm(r[0], r[1], 0x0040), __byte_perm(r[2], r[3], 0x0040), 0x5410);
    const uint32_t hi = __byte_perm(__byte_perm(r[4], r[5], 0x0040), __byte_perm(r[6], r[7], 0x0040), 0x5410);
    st_stream8(dst, lo, hi);
  } else {
    const int nq = min(8, npx - base);
    for (int q = 0; q < nq; ++q) dst[q] = (uint8_t)(r[q] & 0xffu);
  }
}

template <int NW, int BM>
__global__ void __launch_bounds__(NW * 32) esi_integrate_kernel(IntArgs a) {
  constexpr int BP = NW * kWarpPx;
  constexpr int NT = NW * 32;
  constexpr int SLICE = kSubBatch / NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem<NW>& sm = *reinterpret_cast<FastSmem<NW>*>(smem_raw);
  __shared__ int32_t s_tnext;
  __shared__ uint32_t s_wsum[32];

  const int band = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t px0 = (int64_t)band * BP;
  const int npx = (int)min((int64_t)BP, a.P - px0);

  const ChunkInfo ci = *a.info;
  const int f_lo = ci.f_lo, f_hi = ci.f_hi;
  const bool active = ci.active != 0;
  if (!active && f_lo >= f_hi) return;
  const int64_t trel = ci.trel;
  const int32_t dt_cut = (int32_t)a.dp.dt_cut;
  const int32_t t_clamp = -(dt_cut + 1);
  const int32_t tcap = (int32_t)min(a.t_cap - trel, (int64_t)INT32_MAX);
  const float magic_off = kMagic + (float)a.mp.off_int;
  const int n_tiles = a.n_tiles;
  const float C = a.mp.C;

  for (int i = threadIdx.x; i < BP; i += NT) {
    const bool in = i < npx;
    sm.S[i] = in ? a.S[px0 + i] : 0.f;
    sm.T[i] = in ? (int32_t)max(a.T[px0 + i] - trel, (int64_t)t_clamp) : t_clamp;
  }
  int n_b = 0;
  if (active) {
    for (int t = threadIdx.x; t < n_tiles; t += NT) sm.mt[t] = a.meta[(int64_t)band * n_tiles + t];
    __syncthreads();
    const int per = (n_tiles + NT - 1) / NT;
    const int t0 = threadIdx.x * per;
    uint32_t local = 0;
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) local += sm.mt[t] >> 16;
    uint32_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t run = x - local, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t v = s_wsum[w];
      if (w < warp) run += v;
      tot += v;
    }
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) {
      sm.pre[t] = run;
      run += sm.mt[t] >> 16;
    }
    if (threadIdx.x == 0) sm.pre[n_tiles] = tot;
    n_b = (int)tot;
  }
  __syncthreads();

  int j = f_lo;
  bool done = false;
  for (int sb0 = 0; sb0 < n_b; sb0 += kSubBatch) {
    const int n_sb = min(kSubBatch, n_b - sb0);
    const bool has_next = sb0 + n_sb < n_b;
    // ---- 1. gather slice `warp` of the sub-batch; count events per destination warp
    const int q_lo = warp * SLICE;
    const int q_hi = min(q_lo + SLICE, n_sb) + ((has_next && warp == NW - 1) ? 1 : 0);
    uint32_t cnt[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) cnt[w] = 0;
    int tl = -1;
    for (int q0 = q_lo; q0 < q_hi; q0 += 32) {
      const int qq = q0 + lane;
      const bool valid = qq < q_hi;
      int tgt = -1;
      if (valid) {
        const uint32_t q = (uint32_t)(sb0 + qq);
        if (tl < 0) {
          int lo = 0, hi = n_tiles;   // largest t with pre[t] <= q
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (sm.pre[mid] <= q) lo = mid; else hi = mid;
          }
          tl = lo;
        }
        while (sm.pre[tl + 1] <= q) ++tl;
        const int64_t idx = (int64_t)tl * kTile + (sm.mt[tl] & 0xffffu) + (q - sm.pre[tl]);
        const uint2 r = a.rec[idx];
        const int32_t tr = (int32_t)(r.x - (uint32_t)trel);
        if (qq < n_sb) {
          sm.At[qq] = tr;
          sm.Apr[qq] = r.y;
          tgt = (int)((r.y & (uint32_t)(BP - 1)) >> 8);
        } else {
          s_tnext = tr;
        }
      }
#pragma unroll
      for (int w = 0; w < NW; ++w) cnt[w] += __popc(__ballot_sync(kFull, tgt == w));
    }
    if (lane < NW) {
#pragma unroll
      for (int w = 0; w < NW; ++w)
        if (lane == w) sm.cnt[warp][w] = cnt[w];
    }
    if (!has_next && threadIdx.x == 0) s_tnext = INT32_MAX;
    __syncthreads();
    // ---- 2. stable NW-way split of the slice into the destination lists
    uint32_t run[NW];
    int n_w = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      uint32_t b = 0;
      for (int v = 0; v < warp; ++v) b += sm.cnt[v][w];
      run[w] = b;
    }
    for (int v = 0; v < NW; ++v) n_w += sm.cnt[v][warp];
    const int q_hi2 = min(q_lo + SLICE, n_sb);
    for (int q0 = q_lo; q0 < q_hi2; q0 += 32) {
      const int qq = q0 + lane;
      const int tgt = qq < q_hi2 ? (int)((sm.Apr[qq] & (uint32_t)(BP - 1)) >> 8) : -1;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const unsigned m = __ballot_sync(kFull, tgt == w);
        if (tgt == w) sm.L[w][run[w] + __popc(m & lanemask_lt())] = (uint16_t)qq;
        run[w] += __popc(m);
      }
    }
    __syncthreads();
    const int32_t tnext = s_tnext;

    // ---- 3. walk: apply events, reading frames out at their boundaries
    const uint16_t* Lw = sm.L[warp];
    int i = 0;
    while (!done && i < n_w) {
      const int32_t tj = (j < f_hi) ? (int32_t)(a.tf[j] - trel) : tcap;
      const int m = min(32, n_w - i);
      int32_t te = 0;
      uint32_t pr = 0;
      if (lane < m) {
        const int idx = Lw[i + lane];
        te = sm.At[idx];
        pr = sm.Apr[idx];
      }
      const bool valid = lane < m && te <= tj;
      const int nv = __popc(__ballot_sync(kFull, valid));
      if (nv > 0) {
        const bool act = lane < nv;
        const int px = (int)(pr & (uint32_t)(BP - 1));
        // lanes of this batch that hit the same pixel (inactive lanes: singleton keys)
        const unsigned peers = __match_any_sync(kFull, act ? px : BP + lane);
        const float pc = ((int32_t)pr < 0) ? -C : C;
        if (!__any_sync(kFull, act && __popc(peers) > 1)) {
          // sparse batch: every pixel hit once -> Alg. 2 body applied directly,
          // bit-identical to a sequential fp32 evaluation
          if (act) {
            float s = sm.S[px] + pc;                                      // S <- S + p C
            s *= fast_decay<BM>(te - sm.T[px], a.dp, dt_cut);             // S <- S d(t - T)
            sm.S[px] = fminf(fmaxf(s, a.mp.smin), a.mp.smax);             // clamp (Eq. 13)
            sm.T[px] = te;                                                // T <- t
          }
        } else {
          dense_batch_apply<BM>(sm.S, sm.T, act, px, peers, te, pc, lane, a.dp, a.mp, dt_cut);
        }
        __syncwarp();
      }
      i += nv;
      if (nv < m) {
        if (j < f_hi) {
          fast_readout<NW, BM>(a, sm, j, trel, px0, npx, warp, lane, dt_cut, magic_off);
          ++j;
        } else {
          done = true;  // the rest is later than the last frame: stays pending
        }
      }
    }
    // ---- 4. frames whose events are all in this or earlier sub-batches
    while (j < f_hi && (int32_t)(a.tf[j] - trel) < tnext) {
      fast_readout<NW, BM>(a, sm, j, trel, px0, npx, warp, lane, dt_cut, magic_off);
      ++j;
    }
    __syncthreads();
  }
  while (j < f_hi) {
    fast_readout<NW, BM>(a, sm, j, trel, px0, npx, warp, lane, dt_cut, magic_off);
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += NT) {
      a.S[px0 + i] = sm.S[i];
      const int32_t tr = sm.T[i];
      if (tr != t_clamp) a.T[px0 + i] = trel + tr;
    }
  }
}

template <int NW, int BM>
cudaError_t launch_fast_t(const IntArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(FastSmem<NW>);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_kernel<NW, BM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  esi_integrate_kernel<NW, BM><<<a.nb, NW * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <int BM>
cudaError_t launch_fast_b(const IntArgs& a, cudaStream_t s) {
  switch (a.band_px / kWarpPx) {
    case 1: return launch_fast_t<1, BM>(a, s);
    case 2: return launch_fast_t<2, BM>(a, s);
    case 4: return launch_fast_t<4, BM>(a, s);
    case 8: return launch_fast_t<8, BM>(a, s);
    case 16: return launch_fast_t<16, BM>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_integrate_fast(const IntArgs& a, cudaStream_t s) {
  return a.dp.bmode == 2 ? launch_fast_b<2>(a, s) : launch_fast_b<0>(a, s);
}

}  // namespace esi
