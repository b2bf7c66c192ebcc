// esi_slice.cu -- SURVEY 8(f) item 4: time-sharded single streams.
//
// A time slice of the stream acts on one pixel's state (S, T) as
//   m = 0 events: identity;
//   m >= 1      : S1 = clamp((S + p_1 C) d(t_1 - T))      (Alg. 2 body)
//                 S' = G(S1),  T' = t_m,
// where G = g_m o ... o g_2 is the composition of the clamped affine maps of the
// slice's later events, g_k(s) = clamp(d_k s + d_k p_k C, S_min, S_max) with
// d_k = d(t_k - t_{k-1}) (Eq. 4; decay-first variant: clamp(d_k s + p_k C)).
// The decay of the first event is the only place where the incoming T enters, so
// the slice is summarised per pixel by (n, t_first, p_first, G, t_last), and two
// consecutive summaries compose in closed form: B's first event sees A's t_last.
// Clamped affine maps s -> clamp(a s + c, lo, hi) with a >= 0 are closed under
// composition:
//   F o G = (aF aG, aF cG + cF, clamp(aF loG + cF, loF, hiF), clamp(aF hiG + cF, loF, hiF)).
//
// K5 esi_slice_summary_kernel: per band (K1's partition), the band's events of a
//   chunk in passes of <= 2040 (arrival order), stably counting-sorted by pixel
//   in shared memory (match.any ranks), then one thread per pixel run folds the
//   run's events into the pixel's summary (shared memory for the chunk).
// K6 esi_slice_compose_kernel / K7 esi_slice_apply_kernel: elementwise over pixels.
#include <algorithm>
#include <atomic>
#include "esi_device.cuh"

namespace esi {

namespace {

constexpr int kSW = 8;                        // warps per CTA
constexpr int kST = kSW * 32;
static_assert(kSW == 8, "per-pixel warp counts are 8 bytes (dp4a prefix sums)");
constexpr int kShare = 255;                   // events per warp share (u8 per-warp pixel counts)
constexpr int kSE = kSW * kShare;             // events per pass (2040)
constexpr int kRounds = (kShare + 31) / 32;
constexpr int kRunPT = (kSE + kST - 1) / kST; // run heads scanned per thread (8)
constexpr float kBig = 3.0e38f;               // the identity map's bounds (finite: 0 * kBig = 0)

struct Map4 {
  float a, c, lo, hi;
};

// F o G: G first
__device__ __forceinline__ Map4 compose(const Map4& F, const Map4& G) {
  Map4 r;
  r.a = F.a * G.a;
  r.c = fmaf(F.a, G.c, F.c);
  r.lo = fminf(fmaxf(fmaf(F.a, G.lo, F.c), F.lo), F.hi);
  r.hi = fminf(fmaxf(fmaf(F.a, G.hi, F.c), F.lo), F.hi);
  return r;
}

// The map of one event at gap dt from its predecessor (Alg. 2 order or decay-first).
__device__ __forceinline__ Map4 event_map(int64_t dt, int p, const DecayParams& dp, const MapParams& mp) {
  const float d = esi_decay(dt, dp);
  const float pc = p < 0 ? -mp.C : mp.C;
  return Map4{d, dp.first ? pc : d * pc, mp.ev_smin, mp.ev_smax};
}

__device__ __forceinline__ float apply_map(const Map4& m, float s) { return fminf(fmaxf(fmaf(m.a, s, m.c), m.lo), m.hi); }

struct SliceStatic {
  uint2 buf[2][kSE];
  uint32_t misc[64];
};

__host__ __device__ inline size_t r16s(size_t b) { return (b + 15) & ~(size_t)15; }
// dynamic: h8[bp][kSW], off[bp + 1], pre[n_tiles + 1], mo[n_tiles]; the summaries
// themselves stay in global memory (L2): a pixel's map is read and written once
// per pass by the thread that folds its run, which keeps the CTA at 67 KB of shared
// memory (3 CTAs per SM, one wave of bands)
__host__ __device__ inline size_t sl_off_h8(int) { return 0; }
__host__ __device__ inline size_t sl_off_off(int bp) { return sl_off_h8(bp) + (size_t)kSW * bp; }
__host__ __device__ inline size_t sl_off_pre(int bp) { return sl_off_off(bp) + r16s((size_t)(bp + 1) * 2); }
__host__ __device__ inline size_t sl_off_mo(int bp, int nt) { return sl_off_pre(bp) + r16s((size_t)(nt + 1) * 4); }
__host__ __device__ inline size_t sl_smem_bytes(int bp, int nt) { return sl_off_mo(bp, nt) + r16s((size_t)nt * 2); }

#include "esi_fast_common.cuh"

// Decay of one event gap (Eq. 4): BM >= 0 -- the fast fp32 form of K2 (exact for
// dt < 2^24 us after the cutoff clamp; handles with dt_cut < 2^23); BM < 0 -- the
// general esi_decay (fp64 u for slow decays).
template <int BM>
__device__ __forceinline__ Map4 event_map_t(int64_t dt, int p, const IntArgs& a, const FastConst& kc) {
  if (BM < 0) return event_map(dt, p, a.dp, a.mp);
  const float d = ev_decay<(BM < 0 ? 0 : BM)>((float)min(dt, a.dp.dt_cut + 1), kc);
  const float pc = p < 0 ? -kc.C : kc.C;
  return Map4{d, (BM & kFirst) ? pc : d * pc, kc.smin, kc.smax};
}

template <int BM>
__global__ void __launch_bounds__(kST, kK2Ctas) esi_slice_summary_kernel(IntArgs a, int64_t tbase, esi_slice_map_t* maps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(16) SliceStatic ss;
  const int band = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bp = a.band_px;
  const BandMap bmap = a.bm;                                 // band layout (esi_internal.cuh)
  const int npx = band_npx(bmap, band, a.P);
  const int n_tiles = a.n_tiles;
  uint8_t* const h8 = smem_raw + sl_off_h8(bp);
  uint16_t* const off = reinterpret_cast<uint16_t*>(smem_raw + sl_off_off(bp));
  uint32_t* const pre = reinterpret_cast<uint32_t*>(smem_raw + sl_off_pre(bp));
  uint16_t* const mo = reinterpret_cast<uint16_t*>(smem_raw + sl_off_mo(bp, n_tiles));

  // tbase: the chunk's first event; every event of the chunk is within 2^31 us of it (host check)
  const uint32_t tb32 = (uint32_t)tbase;
  const FastConst kc = make_const(a);
  for (int i = tid; i < kSW * bp / 16; i += kST) reinterpret_cast<uint4*>(h8)[i] = make_uint4(0u, 0u, 0u, 0u);
  const int n_b = band_run_prefix<kSW>(a.meta + (int64_t)band * n_tiles, n_tiles, pre, mo, ss.misc + 32);
  __syncthreads();

  if (n_b > 0) gather_sub<kSE>(a.rec, pre, mo, n_tiles, n_b, 0, ss.buf[0], warp, kSW, lane);
  for (int sb0 = 0, kb = 0; sb0 < n_b; sb0 += kSE, ++kb) {
    const int n = min(kSE, n_b - sb0);
    uint2* const cur = ss.buf[kb & 1];
    cp_async_wait_all();
    __syncthreads();                                       // pass gathered; previous pass done
    if (sb0 + kSE < n_b) gather_sub<kSE>(a.rec, pre, mo, n_tiles, n_b, sb0 + kSE, ss.buf[(kb & 1) ^ 1], warp, kSW, lane);

    // rank: a pixel's events of one warp round are ordered by lane (lane-ordered
    // atomics when probed, else match.any), the rounds of a warp share in program
    // order, the shares by warp: stable
    uint32_t evt[kRounds], key[kRounds];
    const int s0 = warp * kShare;
    // per-pixel counts of each warp's share, laid out [pixel][warp] (8 bytes per pixel)
    uint32_t* h32 = reinterpret_cast<uint32_t*>(h8) + (warp >> 2);
    const uint32_t wsh = (uint32_t)(warp & 3) * 8u;
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const int si = r * 32 + lane;
      const bool act = si < kShare && s0 + si < n;
      const unsigned am = __ballot_sync(kFull, act);
      if (am == 0u) break;
      uint32_t px = 0u, sgn = 0u;
      if (act) {
        const uint2 e = cur[s0 + si];
        evt[r] = e.x;
        px = e.y & 0x7fffffffu;
        sgn = e.y & 0x80000000u;
        ESI_DCHECK(px < (uint32_t)npx);
      }
      if (a.atomic_rank) {
        // lane-ordered shared atomics (probed at esi_create, as K1's default): each
        // lane's old count is its rank among the round's lanes of its pixel
        const uint32_t old = act ? atomicAdd(h32 + 2 * px, 1u << wsh) : 0u;
        key[r] = px | (((old >> wsh) & 0xffu) << 12) | sgn;
      } else {
        unsigned peers = 0u;
        if (act) peers = __match_any_sync(am, px);
        const int leader = act ? __ffs(peers) - 1 : lane;
        uint32_t base = 0u;
        if (act && leader == lane) {
          const uint32_t old = atomicAdd(h32 + 2 * px, (uint32_t)__popc(peers) << wsh);
          base = (old >> wsh) & 0xffu;
        }
        base = __shfl_sync(kFull, base, leader);
        key[r] = px | ((base + (uint32_t)__popc(peers & lanemask_lt())) << 12) | sgn;
      }
    }
    __syncthreads();
    // offsets: per-pixel totals over the warps, block-wide exclusive scan
    {
      const int ng = bp >> 2;
      const int gpt = (ng + kST - 1) / kST;
      const int g0 = tid * gpt;
      uint32_t cnt[4][4], local = 0u;                   // pixel totals: the 8 warp bytes summed (dp4a)
#pragma unroll
      for (int g = 0; g < 4; ++g) {
#pragma unroll
        for (int u = 0; u < 4; ++u) cnt[g][u] = 0u;
        if (g < gpt && g0 + g < ng) {
          const uint4 va = *reinterpret_cast<const uint4*>(h8 + 32 * (g0 + g));
          const uint4 vb = *reinterpret_cast<const uint4*>(h8 + 32 * (g0 + g) + 16);
          cnt[g][0] = __dp4a(va.x, 0x01010101u, __dp4a(va.y, 0x01010101u, 0u));
          cnt[g][1] = __dp4a(va.z, 0x01010101u, __dp4a(va.w, 0x01010101u, 0u));
          cnt[g][2] = __dp4a(vb.x, 0x01010101u, __dp4a(vb.y, 0x01010101u, 0u));
          cnt[g][3] = __dp4a(vb.z, 0x01010101u, __dp4a(vb.w, 0x01010101u, 0u));
          local += cnt[g][0] + cnt[g][1] + cnt[g][2] + cnt[g][3];
        }
      }
      uint32_t x = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) ss.misc[32 + warp] = x;
      __syncthreads();
      uint32_t run = x - local;
#pragma unroll
      for (int w = 0; w < kSW; ++w)
        if (w < warp) run += ss.misc[32 + w];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (g < gpt && g0 + g < ng) {
          uint16_t* o = off + 4 * (g0 + g);
          o[0] = (uint16_t)run; run += cnt[g][0];
          o[1] = (uint16_t)run; run += cnt[g][1];
          o[2] = (uint16_t)run; run += cnt[g][2];
          o[3] = (uint16_t)run; run += cnt[g][3];
        }
      }
      if (tid == kST - 1) off[bp] = (uint16_t)n;
    }
    __syncthreads();
    // scatter: stable counting sort by pixel, in place
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const int si = r * 32 + lane;
      if (!(si < kShare && s0 + si < n)) break;
      const uint32_t px = key[r] & 0xfffu;
      // + the events of this pixel in the shares of warps < warp: the low bytes of
      // the pixel's 8 counts, summed by dp4a
      const uint2 v = *reinterpret_cast<const uint2*>(h8 + 8 * px);
      const uint32_t mA = warp >= 4 ? 0xffffffffu : ((1u << (8 * warp)) - 1u);
      const uint32_t mB = warp > 4 ? ((1u << (8 * (warp - 4))) - 1u) : 0u;
      const uint32_t pos = (uint32_t)off[px] + ((key[r] >> 12) & 0xffu) +
                           __dp4a(v.x & mA, 0x01010101u, __dp4a(v.y & mB, 0x01010101u, 0u));
      ESI_DCHECK(pos < (uint32_t)n);
      cur[pos] = make_uint2(evt[r], px | (key[r] & 0x80000000u));
    }
    __syncthreads();
    for (int i = tid; i < kSW * bp / 16; i += kST) reinterpret_cast<uint4*>(h8)[i] = make_uint4(0u, 0u, 0u, 0u);
    // runs: thread t folds the runs that start in [8t, 8t + 8) into their pixels' summaries
    // (the next head's map is loaded while the current run is folded)
    uint32_t heads = 0u;
    const int r0 = tid * kRunPT;
#pragma unroll
    for (int u = 0; u < kRunPT; ++u) {
      const int i = r0 + u;
      if (i < n && (i == 0 || ((cur[i - 1].y ^ cur[i].y) & 0x7fffffffu) != 0u)) heads |= 1u << u;
    }
    esi_slice_map_t Mn;
    int in_ = -1;
    if (heads) {
      in_ = r0 + __ffs(heads) - 1;
      heads &= heads - 1u;
      Mn = maps[band_gpix(bmap, band, (int)(cur[in_].y & 0x7fffffffu))];
    }
    while (in_ >= 0) {
      const int i = in_;
      esi_slice_map_t M = Mn;
      const uint32_t px = cur[i].y & 0x7fffffffu;
      in_ = -1;
      if (heads) {                                       // prefetch the next run's map
        in_ = r0 + __ffs(heads) - 1;
        heads &= heads - 1u;
        Mn = maps[band_gpix(bmap, band, (int)(cur[in_].y & 0x7fffffffu))];
      }
      const int o1 = off[px + 1];
      Map4 g{M.a, M.c, M.lo, M.hi};
      int64_t t_last = M.t_last;
      int32_t m = M.n;
      for (int q = i; q < o1; ++q) {
        const uint2 r = cur[q];
        const int64_t t = tbase + (int64_t)(int32_t)(r.x - tb32);
        const int p = ((int32_t)r.y < 0) ? -1 : 1;
        if (m == 0) {                                    // the slice's first event at this pixel
          M.t_first = t;
          M.p_first = p;
          g = Map4{1.f, 0.f, -kBig, kBig};
        } else {
          g = compose(event_map_t<BM>(t - t_last, p, a, kc), g);
        }
        t_last = t;
        ++m;
      }
      M.a = g.a; M.c = g.c; M.lo = g.lo; M.hi = g.hi;
      M.t_last = t_last;
      M.n = m;
      maps[band_gpix(bmap, band, (int)px)] = M;
    }
  }
  cp_async_wait_all();
}

// out = A then B (A earlier), per pixel
__global__ void esi_slice_compose_kernel(const esi_slice_map_t* A, const esi_slice_map_t* B, esi_slice_map_t* out,
                                         int64_t P, DecayParams dp, MapParams mp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const esi_slice_map_t a = A[i], b = B[i];
    if (b.n == 0) { out[i] = a; continue; }
    if (a.n == 0) { out[i] = b; continue; }
    const Map4 ga{a.a, a.c, a.lo, a.hi}, gb{b.a, b.c, b.lo, b.hi};
    const Map4 g = compose(gb, compose(event_map(b.t_first - a.t_last, b.p_first, dp, mp), ga));
    esi_slice_map_t o = a;
    o.a = g.a; o.c = g.c; o.lo = g.lo; o.hi = g.hi;
    o.t_last = b.t_last;
    o.n = a.n + b.n;
    out[i] = o;
  }
}

// (S, T) <- the slice's action on the state
__global__ void esi_slice_apply_kernel(const esi_slice_map_t* M, float* S, int64_t* T, int64_t P, DecayParams dp,
                                       MapParams mp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const esi_slice_map_t m = M[i];
    if (m.n == 0) continue;
    const float d = esi_decay(m.t_first - T[i], dp);
    const float pc = m.p_first < 0 ? -mp.C : mp.C;
    const float s1 = fminf(fmaxf(dp.first ? fmaf(S[i], d, pc) : (S[i] + pc) * d, mp.ev_smin), mp.ev_smax);
    S[i] = apply_map(Map4{m.a, m.c, m.lo, m.hi}, s1);
    T[i] = m.t_last;
  }
}

}  // namespace

size_t slice_smem_bytes(int band_px, int n_tiles) { return sl_smem_bytes(band_px, n_tiles); }

template <int BM>
cudaError_t launch_slice_summary_b(const IntArgs& a, int64_t tbase, esi_slice_map_t* maps, cudaStream_t s) {
  const size_t smem = sl_smem_bytes(a.band_px, a.n_tiles);
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<int> configured[64];   // zero-initialised; set-once flags (idempotent, race-free)
  if (dev < 0 || dev >= 64 || !configured[dev].load(std::memory_order_relaxed)) {
    cudaError_t e = cudaFuncSetAttribute(esi_slice_summary_kernel<BM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sl_smem_bytes(kMaxBandPx, kMaxTilesPerChunk));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev].store(1, std::memory_order_relaxed);
  }
  esi_slice_summary_kernel<BM><<<a.nb, kST, smem, s>>>(a, tbase, maps);
  return cudaGetLastError();
}

cudaError_t launch_slice_summary(const IntArgs& a, int64_t tbase, esi_slice_map_t* maps, int fast, cudaStream_t s) {
  if (!fast) return launch_slice_summary_b<-1>(a, tbase, maps, s);
  if (a.dp.first)
    return a.dp.bmode == 2           ? launch_slice_summary_b<2 + kFirst>(a, tbase, maps, s)
           : a.dp.bmode == kDecayExp ? launch_slice_summary_b<kDecayExp + kFirst>(a, tbase, maps, s)
                                     : launch_slice_summary_b<kFirst>(a, tbase, maps, s);
  return a.dp.bmode == 2           ? launch_slice_summary_b<2>(a, tbase, maps, s)
         : a.dp.bmode == kDecayExp ? launch_slice_summary_b<kDecayExp>(a, tbase, maps, s)
                                   : launch_slice_summary_b<0>(a, tbase, maps, s);
}

cudaError_t launch_slice_compose(const esi_slice_map_t* A, const esi_slice_map_t* B, esi_slice_map_t* out, int64_t P,
                                 const DecayParams& dp, const MapParams& mp, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((P + 255) / 256, 148 * 8);
  esi_slice_compose_kernel<<<std::max(blocks, 1), 256, 0, s>>>(A, B, out, P, dp, mp);
  return cudaGetLastError();
}

cudaError_t launch_slice_apply(const esi_slice_map_t* M, float* S, int64_t* T, int64_t P, const DecayParams& dp,
                               const MapParams& mp, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((P + 255) / 256, 148 * 8);
  esi_slice_apply_kernel<<<std::max(blocks, 1), 256, 0, s>>>(M, S, T, P, dp, mp);
  return cudaGetLastError();
}

}  // namespace esi
