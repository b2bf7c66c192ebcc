// esi_integrate_px.cu -- K2 (default): per-band integration (Alg. 2)
// fused with the Eq. 13/14 readout of every frame of
// the chunk, by pixel-grouped passes.
//
// One CTA of 8 warps per band of band_px consecutive pixel ids (K1's partition
// key).  Thread t owns the pixel quads q = t, t + 256, ... of the band for the
// whole chunk: their S (fp32) and T (fp32 offset from ChunkInfo::trel, exact
// integers) live in registers.  The band's events are processed in passes of up
// to kPE = 2040 events (arrival order, gathered from K1's tiles with cp.async,
// double-buffered):
//   1. rank   : warp w takes the pass's events [255 w, 255 w + 255); a pixel's
//               events of one warp round are found with match.any (ordered by
//               lane, i.e. arrival order, by construction); the round's lowest
//               peer adds their number to the warp's u8 count of the pixel;
//   2. offsets: per-pixel pass totals (sum of the 8 warp counts) and their
//               block-wide exclusive scan off[px];
//   3. scatter: event -> off[px] + (counts of earlier warps) + rank, in place:
//               a stable counting sort by pixel (each pixel's events stay in
//               arrival order);
//   4. dense  : pixels with more than kDense events in the pass are combined by
//               one warp with a shuffle scan of their clamped affine maps
//               (SURVEY section 0); the state after each event replaces the
//               record's payload;
//   5. walk   : each thread walks its quads through the frames that close in
//               the pass -- apply the pixel's events up to t_j (Alg. 2 body,
//               sequential fp32, bit-identical to the oracle's order) and write
//               the quad's 4 bytes of frame j (fused readout) -- then applies
//               the pass's remaining events up to the render's last frame.
// Five barriers per pass, none per frame window.
#include "esi_device.cuh"

namespace esi {

namespace {

#include "esi_fast_common.cuh"

constexpr int kPW = 8;                        // warps per CTA
constexpr int kPT = kPW * 32;                 // threads per CTA
constexpr int kShare = 255;                   // events per warp share: u8 per-warp pixel counts
constexpr int kPE = kPW * kShare;             // events per pass (2040)
constexpr int kRounds = (kShare + 31) / 32;   // warp rounds per share (8)
#ifndef ESI_DENSE
#define ESI_DENSE 16
#endif
constexpr int kDense = ESI_DENSE;             // more events of one pixel in one pass: dense path
constexpr int kDenseCap = kPE / (kDense + 1) + 1;
constexpr int kChain = 8;                    // a window of <= kChain events of one pixel is applied sequentially
constexpr int kRunPT = (kPE + kPT - 1) / kPT;  // run heads scanned per thread (8)

constexpr int kFrCap = 1024;                  // frame times of a chunk staged in shared memory

// Static shared memory (fixed sizes: direct shared addressing) ...
struct PxStatic {
  uint2 buf[2][kPE];   // pass records (arrival order), then pixel-sorted in place, then compacted runs
  int32_t fr[kFrCap];  // t_f - trel of the chunk's frames f_lo .. f_lo + kFrCap - 1
  uint32_t misc[64];   // [0] dense count, [32..39] warp sums
  int32_t dent[kDenseCap];   // dense pixels of the pass
};
// ... and the band-size / tile-count dependent part, carved from the dynamic buffer:
//   h8 [kPW][bp] u8 per-warp pixel counts of the pass (then float2 slot[bp]),
//   off[bp + 1] u16, pre[n_tiles + 1] u32, mo[n_tiles] u16
__host__ __device__ inline size_t r16(size_t b) { return (b + 15) & ~(size_t)15; }
__host__ __device__ inline size_t px_off_off(int bp) { return (size_t)kPW * bp; }
__host__ __device__ inline size_t px_off_pre(int bp) { return px_off_off(bp) + r16((size_t)(bp + 1) * 2); }
__host__ __device__ inline size_t px_off_mo(int bp, int n_tiles) { return px_off_pre(bp) + r16((size_t)(n_tiles + 1) * 4); }
__host__ __device__ inline size_t px_smem_bytes(int bp, int n_tiles) {
  return px_off_mo(bp, n_tiles) + r16((size_t)n_tiles * 2);
}

// Frame times: shared-memory copy for the first kFrCap frames of the chunk, global beyond.
struct Frames {
  const int32_t* s;
  const int64_t* tf;
  int64_t trel;
  int f_lo;
  __device__ __forceinline__ int32_t at(int f) const {
    const int i = f - f_lo;
    return i < kFrCap ? s[i] : (int32_t)(__ldg(tf + f) - trel);
  }
};

__device__ __forceinline__ int32_t rel(uint32_t x, uint32_t trel32) { return (int32_t)(x - trel32); }

// Eq. 4 + Eq. 13 + Eq. 14 of one quad (reading A4: v = S d(t_j - T)), 4 bytes.
template <int BM>
__device__ __forceinline__ uint32_t quad_bytes(const float (&s)[4], const float (&t)[4], float tj, float aj,
                                               const FastConst& c, float rmin, float rmax) {
  if (c.fold) {
    const float2 naj = make_float2(-aj, -aj);
    float2 w0 = __fadd2_rn(make_float2(t[0], t[1]), naj), w1 = __fadd2_rn(make_float2(t[2], t[3]), naj);
    w0.x = fmaxf(w0.x, 0.f); w0.y = fmaxf(w0.y, 0.f); w1.x = fmaxf(w1.x, 0.f); w1.y = fmaxf(w1.y, 0.f);
    const float2 sw2 = make_float2(c.scale_w2, c.scale_w2), off = make_float2(c.off_frac, c.off_frac);
    const float2 mo = make_float2(c.magic_off, c.magic_off);
    const float2 v0 = __fmul2_rn(make_float2(s[0], s[1]), __fmul2_rn(w0, w0));
    const float2 v1 = __fmul2_rn(make_float2(s[2], s[3]), __fmul2_rn(w1, w1));
    const float2 r0 = __fadd2_rd(__ffma2_rn(v0, sw2, off), mo), r1 = __fadd2_rd(__ffma2_rn(v1, sw2, off), mo);
    return __byte_perm(__byte_perm(__float_as_uint(r0.x), __float_as_uint(r0.y), 0x0040),
                       __byte_perm(__float_as_uint(r1.x), __float_as_uint(r1.y), 0x0040), 0x5410);
  }
  const uint32_t b01 = readout2<BM>(make_float2(s[0], s[1]), make_float2(t[0], t[1]), tj, aj, c, rmin, rmax);
  const uint32_t b23 = readout2<BM>(make_float2(s[2], s[3]), make_float2(t[2], t[3]), tj, aj, c, rmin, rmax);
  return __byte_perm(b01, b23, 0x5410);
}

__device__ __forceinline__ void store_quad(uint8_t* frame, int base, int npx, bool vec, uint32_t v) {
  if (vec && base + 4 <= npx) {
    __stcs(reinterpret_cast<unsigned int*>(frame + base), v);
  } else {
    const int n = min(4, npx - base);
    for (int u = 0; u < n; ++u) frame[base + u] = (uint8_t)((v >> (8 * u)) & 0xffu);
  }
}

// Sorted record of the pass: x = low 32 bits of t, y = px (12 bits) | w << 12 |
// sign(p) << 31, where w = the event's frame window among the pass's closing
// frames j0 .. j0 + nwin - 1 (the number of them with t_f < t; nwin = the open
// window; nwin + 1 = after the render's last frame, not applied).
constexpr uint32_t kPxMask = 0xfffu;
__device__ __forceinline__ uint32_t rec_win(uint32_t y) { return (y >> 12) & 0x7ffffu; }

// Run of one pixel (records [o0, o1), arrival order), sequentially (Alg. 2 body,
// P:243-251, fp32 in the oracle's order: bit-identical to a sequential fp32
// evaluation), compacted in place to the state after the last event of every
// frame window it touches (record = t, state bits), in time order; returns their
// number.  Events after t_cap are not applied (they stay pending).
template <int BM>
__device__ __forceinline__ int run_sequential(uint2* rec, int o0, int o1, float s, float t, uint32_t trel32,
                                              uint32_t wmax, const FastConst& k) {
  int kk = o0;
  uint2 r = rec[o0];
  for (int i = o0;;) {
    const uint32_t w = rec_win(r.y);
    if (w > wmax) break;
    const float te = (float)rel(r.x, trel32);
    const float pc = ((int32_t)r.y < 0) ? -k.C : k.C;
    s = clampS(ev_update<BM>(s, pc, ev_decay<BM>(te - t, k)), k);
    t = te;
    const uint2 rn = ++i < o1 ? rec[i] : make_uint2(0u, 0xfffff000u);   // end: window 0x7ffff
    if (rec_win(rn.y) != w) rec[kk++] = make_uint2(r.x, __float_as_uint(s));   // kk < i: consumed
    if (i >= o1) break;
    r = rn;
  }
  return kk - o0;
}

// Long run (more than kDense events of one pixel in the pass; warp-wide), frame
// window by frame window: a window with at most kChain events is applied
// sequentially by lane 0 (bit-identical to run_sequential); a denser window
// (by measured density) combines its events' clamped affine maps
// f_i = (d_i, d_i p_i C, S_min, S_max) (decay-first variant (d_i, p_i C, ..)),
// d_i from the gap to the previous event, with an inclusive warp-shuffle scan of
//   F o G = (aF aG, aF cG + cF, clamp(aF loG + cF, loF, hiF), clamp(aF hiG + cF, loF, hiF))
// 32 events at a time.  The run is compacted like
// run_sequential's: one record (t, state) per window, in place.
template <int BM>
__device__ __forceinline__ int run_dense(uint2* rec, int o0, int o1, float s, float t, uint32_t trel32,
                                         uint32_t wmax, int lane, const FastConst& k) {
  int kk = o0;
  int i = o0;
  while (i < o1) {
    const uint32_t w = rec_win(rec[i].y);
    if (w > wmax) break;
    int e = i;                                            // window segment [i, e)
    for (;;) {
      const int q = e + lane;
      const unsigned m = __ballot_sync(kFull, q < o1 && rec_win(rec[q].y) == w);
      e += __popc(m);
      if (m != kFull) break;
    }
    const uint32_t last_x = rec[e - 1].x;
    if (e - i <= kChain) {
      if (lane == 0) {
        for (int q = i; q < e; ++q) {
          const uint2 r = rec[q];
          const float te = (float)rel(r.x, trel32);
          const float pc = ((int32_t)r.y < 0) ? -k.C : k.C;
          s = clampS(ev_update<BM>(s, pc, ev_decay<BM>(te - t, k)), k);
          t = te;
        }
      }
      s = __shfl_sync(kFull, s, 0);
      t = __shfl_sync(kFull, t, 0);
    } else {
      for (int base = i; base < e; base += 32) {
        const int q = base + lane;
        const bool act = q < e;
        const uint2 ev = act ? rec[q] : make_uint2(trel32, 0u);
        const float te = (float)rel(ev.x, trel32);
        float tp = __shfl_up_sync(kFull, te, 1);
        if (lane == 0) tp = t;
        const float d = act ? ev_decay<BM>(te - tp, k) : 1.f;
        const float pc = ((int32_t)ev.y < 0) ? -k.C : k.C;
        float fa = d, fc = act ? ((BM & kFirst) ? pc : d * pc) : 0.f, flo = k.smin, fhi = k.smax;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float ga = __shfl_up_sync(kFull, fa, o), gc = __shfl_up_sync(kFull, fc, o);
          const float glo = __shfl_up_sync(kFull, flo, o), ghi = __shfl_up_sync(kFull, fhi, o);
          if (lane >= o) {                                // F <- F o G (G = earlier events)
            const float nlo = fminf(fmaxf(fmaf(fa, glo, fc), flo), fhi);
            const float nhi = fminf(fmaxf(fmaf(fa, ghi, fc), flo), fhi);
            fc = fmaf(fa, gc, fc);
            fa = fa * ga;
            flo = nlo;
            fhi = nhi;
          }
        }
        const int last = min(31, e - 1 - base);
        const float La = __shfl_sync(kFull, fa, last), Lc = __shfl_sync(kFull, fc, last);
        const float Llo = __shfl_sync(kFull, flo, last), Lhi = __shfl_sync(kFull, fhi, last);
        s = fminf(fmaxf(fmaf(La, s, Lc), Llo), Lhi);
        t = __shfl_sync(kFull, te, last);
      }
    }
    __syncwarp();
    if (lane == 0) rec[kk] = make_uint2(last_x, __float_as_uint(s));   // kk <= i: already consumed
    __syncwarp();
    ++kk;
    i = e;
  }
  return kk - o0;
}

template <int BM, int QPT>
__global__ void __launch_bounds__(kPT, kK2Ctas) esi_integrate_px_kernel(IntArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(16) PxStatic ss;
  const int band = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bp = a.band_px;
  const int64_t px0 = (int64_t)band * bp;
  const int npx = (int)min((int64_t)bp, a.P - px0);
  const int nq = (npx + 3) >> 2;
  const int n_tiles = a.n_tiles;
  uint8_t* const h8 = smem_raw;                                       // [kPW][bp], then float2 slot[bp]
  uint16_t* const off = reinterpret_cast<uint16_t*>(smem_raw + px_off_off(bp));   // [bp + 1]
  uint32_t* const pre = reinterpret_cast<uint32_t*>(smem_raw + px_off_pre(bp));   // [n_tiles + 1]
  uint16_t* const mo = reinterpret_cast<uint16_t*>(smem_raw + px_off_mo(bp, n_tiles));   // [n_tiles]

  if (a.gate && *a.gate != kNoError) return;   // lazy validation found an invalid event: write nothing
  const ChunkInfo ci = *a.info;
  const int f_lo = ci.f_lo, f_hi = ci.f_hi;
  const bool active = ci.active != 0;
  if (!active && f_lo >= f_hi) return;
  const int64_t trel = ci.trel;
  const uint32_t trel32 = (uint32_t)trel;
  const float t_clamp = -(float)(a.dp.dt_cut + 1);
  const int32_t tcap = (int32_t)min(a.t_cap - trel, (int64_t)(1 << 25));
  const FastConst kc = make_const(a);
  const bool vec = a.vec8 != 0;
  const float rmin = a.mp.smin, rmax = a.mp.smax;

  // the state of my quads, in registers for the whole chunk
  float S[QPT][4], T[QPT][4];
#pragma unroll
  for (int k = 0; k < QPT; ++k) {
    const int q = tid + k * kPT;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = 4 * q + u;
      const bool in = q < nq && p < npx;
      S[k][u] = in ? a.S[px0 + p] : 0.f;
      T[k][u] = in ? (float)max(a.T[px0 + p] - trel, (int64_t)t_clamp) : t_clamp;
    }
  }
  for (int i = tid; i < kPW * bp / 16; i += kPT) reinterpret_cast<uint4*>(h8)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) ss.misc[0] = 0u;
  for (int i = tid; i < min(f_hi - f_lo, kFrCap); i += kPT) ss.fr[i] = (int32_t)(a.tf[f_lo + i] - trel);
  const Frames Fr{ss.fr, a.tf, trel, f_lo};
  const int n_b = active ? band_run_prefix<kPW>(a.meta + (int64_t)band * n_tiles, n_tiles, pre, mo,
                                                ss.misc + 32)
                         : 0;
  __syncthreads();

  int j = f_lo;
  if (n_b > 0) gather_sub<kPE>(a.rec, pre, mo, n_tiles, n_b, 0, ss.buf[0], warp, kPW, lane);
  for (int sb0 = 0, kb = 0; sb0 < n_b; sb0 += kPE, ++kb) {
    const int n = min(kPE, n_b - sb0);
    uint2* const cur = ss.buf[kb & 1];
    cp_async_wait_all();
    __syncthreads();                                       // (1) pass gathered; previous walk done
    if (sb0 + kPE < n_b)
      gather_sub<kPE>(a.rec, pre, mo, n_tiles, n_b, sb0 + kPE, ss.buf[(kb & 1) ^ 1], warp, kPW,
                      lane);
    if (tid == 0) ss.misc[0] = 0u;                         // dense count of this pass
    const int32_t tlast = rel(cur[n - 1].x, trel32);       // the pass is time-sorted
    // the frames closing in this pass: [j, j_end) with t_j < tlast (later frames wait
    // for later passes; the last pass's rest is written after the loop)
    int j_end = j;
    while (j_end < f_hi && Fr.at(j_end) < tlast) ++j_end;
    const int nwin = j_end - j;

    // ---- 1. rank: my warp's share, 32 events per round (arrival order)
    uint32_t evt[kRounds], key[kRounds];                  // t (low 32 bits); px | rank << 12 | sign
    const int s0 = warp * kShare;
    uint32_t* h32 = reinterpret_cast<uint32_t*>(h8 + warp * bp);
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const int si = r * 32 + lane;
      const bool act = si < kShare && s0 + si < n;
      const unsigned am = __ballot_sync(kFull, act);
      if (am == 0u) break;                                 // uniform: the share is exhausted
      uint32_t px = 0u, sgn = 0u;
      unsigned peers = 0u;
      if (act) {
        const uint2 e = cur[s0 + si];
        evt[r] = e.x;
        px = e.y & 0x7fffffffu;
        sgn = e.y & 0x80000000u;
        ESI_DCHECK(px < (uint32_t)npx);
        peers = __match_any_sync(am, px);
      }
      const int leader = act ? __ffs(peers) - 1 : lane;
      uint32_t base = 0u;
      if (act && leader == lane) {
        const uint32_t sh = (px & 3u) * 8u;
        const uint32_t old = atomicAdd(h32 + (px >> 2), (uint32_t)__popc(peers) << sh);
        base = (old >> sh) & 0xffu;
      }
      base = __shfl_sync(kFull, base, leader);
      key[r] = px | ((base + (uint32_t)__popc(peers & lanemask_lt())) << 12) | sgn;   // px < 4096, rank < 255
    }
    __syncthreads();                                       // (2) warp counts complete

    // ---- 2. offsets: per-pixel totals over the warps, block-wide exclusive scan
    {
      const int ng = bp >> 2;                              // 4-pixel groups (bp % 64 == 0)
      const int gpt = (ng + kPT - 1) / kPT;
      const int g0 = tid * gpt;
      uint32_t ev4[4], od4[4], local = 0u;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        ev4[g] = od4[g] = 0u;
        if (g < gpt && g0 + g < ng) {
#pragma unroll
          for (int w = 0; w < kPW; ++w) {
            const uint32_t v = reinterpret_cast<const uint32_t*>(h8 + w * bp)[g0 + g];
            ev4[g] += v & 0x00ff00ffu;
            od4[g] += (v >> 8) & 0x00ff00ffu;
          }
          local += (ev4[g] & 0xffffu) + (ev4[g] >> 16) + (od4[g] & 0xffffu) + (od4[g] >> 16);
        }
      }
      uint32_t x = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) ss.misc[32 + warp] = x;
      __syncthreads();                                     // (3)
      uint32_t run = x - local;
#pragma unroll
      for (int w = 0; w < kPW; ++w)
        if (w < warp) run += ss.misc[32 + w];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        if (g < gpt && g0 + g < ng) {
          uint16_t* o = off + 4 * (g0 + g);
          o[0] = (uint16_t)run; run += ev4[g] & 0xffffu;
          o[1] = (uint16_t)run; run += od4[g] & 0xffffu;
          o[2] = (uint16_t)run; run += ev4[g] >> 16;
          o[3] = (uint16_t)run; run += od4[g] >> 16;
        }
      }
      if (tid == kPT - 1) off[bp] = (uint16_t)n;
    }
    __syncthreads();                                       // (4) offsets complete

    // ---- 3. scatter (stable counting sort by pixel, in place)
    // (my events are in time order: their frame windows are found incrementally)
    int win = 0;
    int32_t wb = nwin > 0 ? Fr.at(j) : INT32_MAX;          // frame time closing window `win`
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      const int si = r * 32 + lane;
      if (!(si < kShare && s0 + si < n)) break;
      const uint32_t px = key[r] & kPxMask;
      uint32_t pos = (uint32_t)off[px] + ((key[r] >> 12) & 0xffu);
      for (int w = 0; w < warp; ++w) pos += h8[w * bp + px];
      ESI_DCHECK(pos < (uint32_t)n);
      const int32_t ti = rel(evt[r], trel32);
      while (ti > wb) {
        ++win;
        wb = win < nwin ? Fr.at(j + win) : INT32_MAX;
      }
      const uint32_t wr = ti > tcap ? (uint32_t)nwin + 1u : (uint32_t)win;
      cur[pos] = make_uint2(evt[r], px | (wr << 12) | (key[r] & 0x80000000u));
    }
    __syncthreads();                                       // (5) pass sorted by pixel; counts consumed
    // ---- 4. publish the pass-start state of my pixels with events (slot[px] reuses h8)
    float2* slot = reinterpret_cast<float2*>(h8);
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int q = tid + k * kPT;
      if (q < nq) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int p = 4 * q + u;
          if (off[p + 1] != off[p]) slot[p] = make_float2(S[k][u], T[k][u]);
        }
      }
    }
    // run heads in my range [kRunPT t, kRunPT t + kRunPT), found before any run is compacted
    const int r0 = tid * kRunPT;
    uint32_t heads = 0u;
#pragma unroll
    for (int u = 0; u < kRunPT; ++u) {
      const int i = r0 + u;
      if (i < n && (i == 0 || ((cur[i - 1].y ^ cur[i].y) & kPxMask) != 0u)) heads |= 1u << u;
    }
    __syncthreads();                                       // (6)

    // ---- 5. runs: each pixel's events of the pass, event-balanced over the threads
    // (thread t takes the runs that start in [8t, 8t + 8)): applied sequentially
    // and compacted to one state per frame window; long runs go to the dense path
    while (heads) {                                        // position r0 + u is written only by its run's thread
      const int i = r0 + __ffs(heads) - 1;
      heads &= heads - 1u;
      const uint32_t px = cur[i].y & kPxMask;
      const int o0 = off[px], o1 = off[px + 1];
      if (o1 - o0 > kDense) {
        const uint32_t d = atomicAdd(ss.misc, 1u);
        ESI_DCHECK(d < (uint32_t)kDenseCap);
        ss.dent[d] = (int)px;
        continue;
      }
      const float2 st = slot[px];
      const int kk = run_sequential<BM>(cur, o0, o1, st.x, st.y, trel32, (uint32_t)nwin, kc);
      slot[px].x = __int_as_float(kk);
    }
    __syncthreads();                                       // (7)
    const uint32_t nd = ss.misc[0];
    if (nd > 0u) {                                         // dense pixels (rare): one warp each
      for (uint32_t d = warp; d < nd; d += kPW) {
        const int px = ss.dent[d];
        const float2 st = slot[px];
        const int kk = run_dense<BM>(cur, off[px], off[px + 1], st.x, st.y, trel32, (uint32_t)nwin, lane, kc);
        if (lane == 0) slot[px].x = __int_as_float(kk);
      }
      __syncthreads();
    }

    // ---- 6. walk: my quads through the closing frames; at most one state change per
    // pixel and window (the compacted runs), then the state after the pass
    for (int i = 4 * nq + tid; i < bp; i += kPT) slot[i] = make_float2(0.f, 0.f);   // ragged tail: zero h8
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int q = tid + k * kPT;
      if (q < nq) {
        const int p = 4 * q;
        int c[4], e[4];
        int32_t tn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          c[u] = off[p + u];
          e[u] = c[u];
          if (off[p + u + 1] != c[u]) e[u] += __float_as_int(slot[p + u].x);
          slot[p + u] = make_float2(0.f, 0.f);             // h8 zero again for the next pass
          tn[u] = c[u] < e[u] ? rel(cur[c[u]].x, trel32) : INT32_MAX;
        }
        for (int jj = j; jj < j_end; ++jj) {
          const int32_t tji = Fr.at(jj);
          if (min(min(tn[0], tn[1]), min(tn[2], tn[3])) <= tji) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (tn[u] <= tji) {
                S[k][u] = __uint_as_float(cur[c[u]].y);
                T[k][u] = (float)tn[u];
                ++c[u];
                tn[u] = c[u] < e[u] ? rel(cur[c[u]].x, trel32) : INT32_MAX;
              }
            }
          }
          const uint32_t v = quad_bytes<BM>(S[k], T[k], (float)tji, (float)(tji - (int32_t)kc.tau_h), kc, rmin, rmax);
          store_quad(a.out + (int64_t)jj * a.P + px0, p, npx, vec, v);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {                      // the open window's last event (<= t_cap)
          if (c[u] < e[u]) {
            S[k][u] = __uint_as_float(cur[c[u]].y);
            T[k][u] = (float)tn[u];
          }
        }
      }
    }
    j = j_end;
  }
  cp_async_wait_all();
  // ---- frames after the band's last event of the chunk
  if (j < f_hi) {
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int q = tid + k * kPT;
      if (q < nq) {
        for (int jj = j; jj < f_hi; ++jj) {
          const int32_t tji = Fr.at(jj);
          const uint32_t v = quad_bytes<BM>(S[k], T[k], (float)tji, (float)(tji - (int32_t)kc.tau_h), kc, rmin, rmax);
          store_quad(a.out + (int64_t)jj * a.P + px0, 4 * q, npx, vec, v);
        }
      }
    }
  }
  if (n_b > 0) {
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
      const int q = tid + k * kPT;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = 4 * q + u;
        if (q < nq && p < npx) {
          a.S[px0 + p] = S[k][u];
          if (T[k][u] != t_clamp) a.T[px0 + p] = trel + (int64_t)T[k][u];
        }
      }
    }
  }
}

template <int BM, int QPT>
cudaError_t launch_px_q(const IntArgs& a, cudaStream_t s) {
  const size_t smem = px_smem_bytes(a.band_px, a.n_tiles);
  int dev = 0;
  cudaGetDevice(&dev);
  static int configured[64] = {0};   // per device (the attribute is per context)
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    const size_t mx = px_smem_bytes(kMaxBandPx, kMaxTilesPerChunk);
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_px_kernel<BM, QPT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev] = 1;
  }
  esi_integrate_px_kernel<BM, QPT><<<a.nb, kPT, smem, s>>>(a);
  return cudaGetLastError();
}

template <int BM>
cudaError_t launch_px_b(const IntArgs& a, cudaStream_t s) {
  const int qpt = ((a.band_px >> 2) + kPT - 1) / kPT;   // quads per thread
  return qpt <= 1 ? launch_px_q<BM, 1>(a, s)
         : qpt == 2 ? launch_px_q<BM, 2>(a, s)
         : qpt == 3 ? launch_px_q<BM, 3>(a, s)
                    : launch_px_q<BM, 4>(a, s);
}

}  // namespace

size_t integrate_px_smem_bytes(int band_px, int n_tiles) { return px_smem_bytes(band_px, n_tiles); }

cudaError_t launch_integrate_px(const IntArgs& a, cudaStream_t s) {
  if (a.dp.first)
    return a.dp.bmode == 2           ? launch_px_b<2 + kFirst>(a, s)
           : a.dp.bmode == kDecayExp ? launch_px_b<kDecayExp + kFirst>(a, s)
                                     : launch_px_b<kFirst>(a, s);
  return a.dp.bmode == 2           ? launch_px_b<2>(a, s)
         : a.dp.bmode == kDecayExp ? launch_px_b<kDecayExp>(a, s)
                                   : launch_px_b<0>(a, s);
}

}  // namespace esi
