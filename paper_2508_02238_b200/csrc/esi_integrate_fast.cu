// esi_integrate_fast.cu -- K2: per-band integration (Alg. 2) fused
// with the Eq. 13/14 readout of every frame of the chunk.
//
// One CTA per band of BP = NW*256 consecutive pixel ids (K1's partition key);
// warp w owns the 256 pixels [w*256, w*256+256) of the band, lane l the 8
// pixels [w*256 + 8l, +8).  The band's state lives in shared memory for the
// whole chunk: S (fp32) and T as an fp32 offset from the chunk base
// ChunkInfo::trel (exact integers: |T| < 2^24 us; pixels older than the decay
// horizon are clamped to -(dt_cut+1), i.e. "fully decayed").
//
// Per sub-batch of SB = NW*256 band events (arrival order):
//   1. gather: warps copy the band's (tile, band) segments written by K1 -- in
//      tile order, i.e. arrival order -- into sub[] (one warp per segment);
//   2. split: warp w takes slice w of sub[], ranks each event among the
//      slice's events bound for the same owner warp (__match_any_sync), and
//      after a block-wide scan of the NW x NW slice/owner counts scatters it to
//      lst[] -- owner-major, arrival-order-minor (a stable NW-way split);
//   3. walk: each warp walks its list 32 events at a time.  Before the first
//      event later than frame time t_j it reads frame j out for its 256 pixels
//      (fused Eq. 13 + Eq. 14, packed f32x2 arithmetic, 8-byte streaming
//      stores).  Per batch, the density of the batch picks the path:
//        sparse (every pixel hit once): the Alg. 2 body applied directly --
//          bit-identical to a sequential fp32 evaluation;
//        dense (some pixel hit several times): a warp-shuffle inclusive scan
//          of the events' clamped affine maps along each pixel's chain
//          (dense_batch_apply).
// Decay (Eq. 4, reading A14): with tau = 1e6/k us split as tau_h + tau_l,
//   u = k_us * ((tau_h - dt) + tau_l),  d = max(u, 0)^b
// (tau_h - dt is exact near the cutoff, so u keeps full relative precision and
// u <= 0 exactly when dt >= dt_cut = ceil(tau)).
#include "esi_device.cuh"

namespace esi {

namespace {

constexpr float kMagic = 8388608.0f;   // 2^23

struct FastConst {
  float tau_h, tau_l;                  // tau = 1e6/k us = tau_h + tau_l
  float kh, kl, k_tau_l;               // k_us = kh + kl (no systematic bias), k_us * tau_l
  float b;
  float C, smin, smax;
  float scale, off_frac, magic_off;    // map: byte = low8(bits(rd(v*scale + off_frac + 2^23 + off_int)))
  float scale_w2;                      // k_us^2 * scale: Eq. 14 of S*(k w)^2 with k^2 folded in
  int32_t tau_int;                     // tau is an integer (tau_l == 0)
  int32_t fold;                        // readout mode: 1 = folded (b = 2, readout decay, no clamp, integer tau)
  int32_t rd, cl;                      // readout decay; readout clamp needed (bounds exclude 0)
};

__device__ __forceinline__ FastConst make_const(const IntArgs& a) {
  FastConst c;
  c.tau_h = a.dp.tau_h;
  c.tau_l = a.dp.tau_l;
  c.kh = a.dp.kh;
  c.kl = a.dp.kl;
  c.k_tau_l = a.dp.kf * a.dp.tau_l;
  c.b = a.dp.b;
  c.C = a.mp.C;
  c.smin = a.mp.smin;
  c.smax = a.mp.smax;
  c.scale = a.mp.scale;
  c.off_frac = a.mp.off_frac;
  c.magic_off = kMagic + (float)a.mp.off_int;
  c.scale_w2 = a.mp.scale_w2;
  c.tau_int = a.dp.tau_l == 0.f;
  c.rd = a.mp.readout_decay != 0;
  c.cl = !(a.mp.smin <= 0.f && a.mp.smax >= 0.f);
  c.fold = a.dp.bmode == 2 && c.rd && !c.cl && c.tau_int;
  return c;
}

// Eq. 4: u = 1 - k dt computed as k ((tau_h - dt) + tau_l) with the
// float pair kh + kl = k * 1e-6 /us.  tau_h - dt is exact near the cutoff, so
// u keeps its relative precision there and u <= 0 exactly when dt >= ceil(tau)
// (reading A14); the pair keeps the product free of a systematic bias (a
// single-float k would bias every decay factor by the same ~3e-8 relative).
__device__ __forceinline__ float decay_u(float dt, const FastConst& c) {
  const float w = (c.tau_h - dt) + c.tau_l;
  return fmaxf(fmaf(c.kh, w, c.kl * w), 0.f);
}

template <int BM>
__device__ __forceinline__ float ev_decay(float dt, const FastConst& c) {
  const float u = decay_u(dt, c);
  if (BM == 2) return u * u;
  return exp2f(c.b * __log2f(u));      // log2(0) = -inf -> d = 0
}

// Eq. 13 clamp of one event's result.
__device__ __forceinline__ float clampS(float s, const FastConst& c) { return fminf(fmaxf(s, c.smin), c.smax); }

// Clamped affine map s -> clamp(a s + c, lo, hi) with a >= 0 (SURVEY section 0,
// finding 1).  The Alg. 2 body of event i is the map
// f_i = (d_i, d_i p_i C, S_min, S_max); such maps are closed under composition:
//   F o G = (aF aG, aF cG + cF, clamp(aF loG + cF, loF, hiF), clamp(aF hiG + cF, loF, hiF)).
// Dense batch: each lane builds its event's map, then a pointer-jumping
// inclusive scan along the per-pixel chains (previous event of the same pixel
// = highest lower peer lane from __match_any_sync) composes every prefix in
// <= 5 shuffle rounds; lane i's state is prefix_i applied to the pixel's state
// before the batch.  Pixels hit once keep the direct Alg. 2 arithmetic.
template <int BM>
__device__ __forceinline__ void dense_batch_apply(float* S, float* T, bool act, int px, unsigned peers,
                                                  float te, float pc, int lane, const FastConst& k) {
  const unsigned below = act ? (peers & lanemask_lt()) : 0u;
  const int prev = below ? 31 - __clz(below) : -1;          // previous event of my pixel in the batch
  const float t_prev_lane = __shfl_sync(kFull, te, prev < 0 ? lane : prev);
  float s0 = 0.f, tp = t_prev_lane;
  if (act) {
    s0 = S[px];                                               // state before the batch
    if (prev < 0) tp = T[px];
  }
  __syncwarp();                                               // all reads before any write
  const float d = act ? ev_decay<BM>(te - tp, k) : 1.f;
  float fa = d, fc = d * pc, flo = k.smin, fhi = k.smax;      // f_i
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
  const float v = single ? clampS((s0 + pc) * d, k)                       // direct Alg. 2 body
                         : fminf(fmaxf(fmaf(fa, s0, fc), flo), fhi);      // prefix_i(s0)
  const unsigned above = peers & ~lanemask_lt() & ~(1u << lane);
  if (act && above == 0u) {                                   // last event of its pixel in the batch
    S[px] = v;
    T[px] = te;
  }
}

// Readout of 2 pixels (reading A4: v = S d(t_j - T), non-mutating; Eq. 13 clamp
// when the bounds exclude 0; Eq. 14 rounded half away from zero, reading A8).
// Folded mode (b = 2, integer tau, bounds containing 0): with w = T - (t_j - tau)
// = tau - dt (exact), d = (k w)^2 for w > 0 and 0 otherwise, so
//   x = S w^2 (k^2 scale) + off_frac   -- 4 packed f32x2 ops + 2 max per 2 pixels.
template <int BM>
__device__ __forceinline__ uint32_t readout2(float2 s, float2 T, float tj, float aj, const FastConst& c) {
  float2 x;
  if (c.fold) {
    float2 w = __fadd2_rn(T, make_float2(-aj, -aj));                          // tau - dt, exact
    w.x = fmaxf(w.x, 0.f);
    w.y = fmaxf(w.y, 0.f);
    const float2 v = __fmul2_rn(s, __fmul2_rn(w, w));
    x = __ffma2_rn(v, make_float2(c.scale_w2, c.scale_w2), make_float2(c.off_frac, c.off_frac));
  } else {
    float2 v = s;
    if (c.rd) {
      const float dx = decay_u(tj - T.x, c), dy = decay_u(tj - T.y, c);
      float2 d;
      if (BM == 2) d = make_float2(dx * dx, dy * dy);
      else d = make_float2(exp2f(c.b * __log2f(dx)), exp2f(c.b * __log2f(dy)));
      v = __fmul2_rn(s, d);
    }
    if (c.cl) {
      v.x = fminf(fmaxf(v.x, c.smin), c.smax);
      v.y = fminf(fmaxf(v.y, c.smin), c.smax);
    }
    x = __ffma2_rn(v, make_float2(c.scale, c.scale), make_float2(c.off_frac, c.off_frac));
  }
  const float2 r = __fadd2_rd(x, make_float2(c.magic_off, c.magic_off));   // 2^23 + off_int + floor(x)
  return __byte_perm(__float_as_uint(r.x), __float_as_uint(r.y), 0x0040);  // 2 bytes in the low half
}

template <int NW, int PPL>
struct FastSmem {
  static constexpr int WPX = 32 * PPL;         // pixels per warp
  static constexpr int BP = NW * WPX;          // pixels per band
  static constexpr int SB = NW * 128;          // events per sub-batch (4 per lane in the split)
  float S[BP];
  float T[BP];
  uint2 sub[SB + 2];                          // + the first event of the next sub-batch
  uint2 lst[SB];
  uint32_t cnt[NW][NW];                       // [slice warp][owner warp]
  uint32_t lbeg[NW + 1];
  uint32_t tiles[1];                          // pre[n_tiles + 1] then mt[n_tiles] (dynamic tail)
};

template <int NW, int PPL>
size_t fast_smem_bytes(int n_tiles) {
  return sizeof(FastSmem<NW, PPL>) + (size_t)(2 * n_tiles + 1) * sizeof(uint32_t);
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int NW, int PPL, int BM>
__device__ __forceinline__ void fast_readout(const IntArgs& a, FastSmem<NW, PPL>& sm, int j, int64_t trel,
                                             int64_t px0, int npx, int warp, int lane, const FastConst& c) {
  const int base = warp * FastSmem<NW, PPL>::WPX + lane * PPL;
  if (base >= npx) return;
  const int32_t tji = (int32_t)(a.tf[j] - trel);
  const float tj = (float)tji;
  const float aj = (float)(tji - (int32_t)c.tau_h);          // t_j - tau (folded mode: tau integer)
  const float4 s0 = *reinterpret_cast<const float4*>(&sm.S[base]);
  const float4 t0 = *reinterpret_cast<const float4*>(&sm.T[base]);
  const uint32_t b01 = readout2<BM>(make_float2(s0.x, s0.y), make_float2(t0.x, t0.y), tj, aj, c);
  const uint32_t b23 = readout2<BM>(make_float2(s0.z, s0.w), make_float2(t0.z, t0.w), tj, aj, c);
  const uint32_t lo = __byte_perm(b01, b23, 0x5410);
  uint8_t* dst = a.out + (int64_t)j * a.P + px0 + base;
  if (PPL == 8) {
    const float4 s1 = *reinterpret_cast<const float4*>(&sm.S[base + 4]);
    const float4 t1 = *reinterpret_cast<const float4*>(&sm.T[base + 4]);
    const uint32_t b45 = readout2<BM>(make_float2(s1.x, s1.y), make_float2(t1.x, t1.y), tj, aj, c);
    const uint32_t b67 = readout2<BM>(make_float2(s1.z, s1.w), make_float2(t1.z, t1.w), tj, aj, c);
    const uint32_t hi = __byte_perm(b45, b67, 0x5410);
    if (a.vec8 && base + 8 <= npx) {
      st_stream8(dst, lo, hi);
      return;
    }
    const int nq = min(8, npx - base);
    for (int q = 0; q < nq; ++q) dst[q] = (uint8_t)((q < 4 ? lo >> (8 * q) : hi >> (8 * (q - 4))) & 0xffu);
  } else {
    if (a.vec8 && base + 4 <= npx) {
      st_stream4(dst, lo);
      return;
    }
    const int nq = min(4, npx - base);
    for (int q = 0; q < nq; ++q) dst[q] = (uint8_t)((lo >> (8 * q)) & 0xffu);
  }
}

template <int NW, int PPL, int BM>
__global__ void __launch_bounds__(NW * 32, (NW * 32 >= 512) ? 3 : 1536 / (NW * 32)) esi_integrate_kernel(IntArgs a) {
  using Sm = FastSmem<NW, PPL>;
  constexpr int WSH = PPL == 8 ? 8 : 7;        // log2(pixels per warp)
  constexpr int BP = Sm::BP;
  constexpr int SB = Sm::SB;
  constexpr int NT = NW * 32;
  constexpr int ROUNDS = SB / NW / 32;        // = 4: events per lane in the split
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
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
  const float t_clamp = -(float)(a.dp.dt_cut + 1);
  const float tcap = (float)min(a.t_cap - trel, (int64_t)(1 << 25));
  const int n_tiles = a.n_tiles;
  uint32_t* pre = sm.tiles;                   // [n_tiles + 1]
  uint32_t* mt = sm.tiles + n_tiles + 1;      // [n_tiles]
  const FastConst kc = make_const(a);

  for (int i = threadIdx.x; i < BP; i += NT) {
    const bool in = i < npx;
    sm.S[i] = in ? a.S[px0 + i] : 0.f;
    sm.T[i] = in ? (float)max(a.T[px0 + i] - trel, (int64_t)t_clamp) : t_clamp;
  }
  int n_b = 0;
  if (active) {
    for (int t = threadIdx.x; t < n_tiles; t += NT) mt[t] = a.meta[(int64_t)band * n_tiles + t];
    __syncthreads();
    const int per = (n_tiles + NT - 1) / NT;
    const int t0 = threadIdx.x * per;
    uint32_t local = 0;
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) local += mt[t] >> 16;
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
      pre[t] = run;
      run += mt[t] >> 16;
    }
    if (threadIdx.x == 0) pre[n_tiles] = tot;
    n_b = (int)tot;
  }
  __syncthreads();

  int j = f_lo;
  bool done = false;
  for (int sb0 = 0; sb0 < n_b; sb0 += SB) {
    const int n_sb = min(SB, n_b - sb0);
    const bool has_next = sb0 + n_sb < n_b;
    const uint32_t q_end = (uint32_t)(sb0 + n_sb);
    // ---- 1. gather the sub-batch + the next sub-batch's first event (cp.async,
    //         one warp per (tile, band) segment, tiles in order = arrival order)
    // last tile with pre[t] <= sb0: 32-ary search by each warp (n_tiles <= 1024)
    int t_lo;
    {
      const int c = lane * 32;
      const unsigned b1 = __ballot_sync(kFull, c < n_tiles && pre[c] <= (uint32_t)sb0);
      const int blk = 31 - __clz(b1 | 1u);
      const int t = blk * 32 + lane;
      const unsigned b2 = __ballot_sync(kFull, t < n_tiles && pre[t] <= (uint32_t)sb0);
      t_lo = blk * 32 + (31 - __clz(b2 | 1u));
    }
    // 8 segments per warp step, 4 lanes per segment (one 32-B sector per copy step)
    for (int tb = t_lo + warp * 8; tb < n_tiles; tb += NW * 8) {
      if (pre[tb] > q_end) break;               // segments are in order: the rest is later
      const int t = tb + (lane >> 2);
      uint32_t i0 = 0, i1 = 0, p0 = 0;
      const uint2* src = a.rec;
      if (t < n_tiles) {
        p0 = pre[t];
        const uint32_t m = mt[t];
        if (p0 <= q_end) {
          i0 = p0 < (uint32_t)sb0 ? (uint32_t)sb0 - p0 : 0u;
          i1 = min(m >> 16, q_end + 1 - p0);
        }
        src += (size_t)t * kTile + (m & 0xffffu);
      }
      const int dofs = (int)p0 - sb0;           // >= -i0
      for (uint32_t i = i0 + (lane & 3); i < i1; i += 4) cp_async8(&sm.sub[dofs + (int)i], src + i);
    }
    if (lane < NW) sm.cnt[warp][lane] = 0;
    cp_async_wait_all();
    __syncthreads();
    const float tnext = has_next ? (float)(int32_t)(sm.sub[n_sb].x - (uint32_t)trel) : 3.0e38f;
    // ---- 2a. rank each event of slice `warp` among the slice's events for the same owner
    uint2 rec[ROUNDS];
    uint32_t pos[ROUNDS];
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      const int i = warp * (ROUNDS * 32) + r * 32 + lane;
      const bool act = i < n_sb;
      rec[r] = act ? sm.sub[i] : make_uint2(0u, 0u);
      rec[r].x = __float_as_uint((float)(int32_t)(rec[r].x - (uint32_t)trel));   // relative time, exact
      const int own = act ? (int)((rec[r].y & (uint32_t)(BP - 1)) >> WSH) : NW + lane;
      const unsigned peers = __match_any_sync(kFull, own);
      const uint32_t rank = __popc(peers & lanemask_lt());
      uint32_t base = 0;
      if (act) base = sm.cnt[warp][own];
      __syncwarp();
      if (act && rank == 0) sm.cnt[warp][own] = base + __popc(peers);
      __syncwarp();
      pos[r] = act ? ((base + rank) | ((uint32_t)own << 16)) : 0xffffffffu;
    }
    __syncthreads();
    // ---- 2b. exclusive scan of the [slice][owner] counts (owner-major)
    if (threadIdx.x < NW) {
      const int own = threadIdx.x;
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t c = sm.cnt[w][own];
        sm.cnt[w][own] = run;
        run += c;
      }
      sm.lbeg[own + 1] = run;                  // owner total, prefixed below
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t run = 0;
      sm.lbeg[0] = 0;
      for (int w = 0; w < NW; ++w) {
        run += sm.lbeg[w + 1];
        sm.lbeg[w + 1] = run;
      }
    }
    __syncthreads();
    // ---- 2c. stable scatter to the owners' lists
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      if (pos[r] != 0xffffffffu) {
        const int own = (int)(pos[r] >> 16);
        sm.lst[sm.lbeg[own] + sm.cnt[warp][own] + (pos[r] & 0xffffu)] = rec[r];
      }
    }
    __syncthreads();

    // ---- 3. walk: apply events, reading frames out at their boundaries
    const int l_end = (int)sm.lbeg[warp + 1];
    int i = (int)sm.lbeg[warp];
    float tj = (j < f_hi) ? (float)(int32_t)(a.tf[j] - trel) : tcap;
    while (!done && i < l_end) {
      const int m = min(32, l_end - i);
      float te = 0.f;
      uint32_t pr = 0;
      if (lane < m) {
        const uint2 r = sm.lst[i + lane];
        te = __uint_as_float(r.x);
        pr = r.y;
      }
      const bool valid = lane < m && te <= tj;
      const int nv = __popc(__ballot_sync(kFull, valid));
      if (nv > 0) {
        const bool act = lane < nv;
        const int px = (int)(pr & (uint32_t)(BP - 1));
        const unsigned peers = __match_any_sync(kFull, act ? px : BP + lane);
        const float pc = ((int32_t)pr < 0) ? -kc.C : kc.C;
        if (!__any_sync(kFull, act && __popc(peers) > 1)) {
          // sparse batch: Alg. 2 body applied directly
          if (act) {
            float s = sm.S[px] + pc;                                     // S <- S + p C
            s *= ev_decay<BM>(te - sm.T[px], kc);                        // S <- S d(t - T)
            sm.S[px] = clampS(s, kc);                                    // clamp (Eq. 13)
            sm.T[px] = te;                                               // T <- t
          }
        } else {
          dense_batch_apply<BM>(sm.S, sm.T, act, px, peers, te, pc, lane, kc);
        }
        __syncwarp();
      }
      i += nv;
      if (nv < m) {
        if (j < f_hi) {
          fast_readout<NW, PPL, BM>(a, sm, j, trel, px0, npx, warp, lane, kc);
          ++j;
          tj = (j < f_hi) ? (float)(int32_t)(a.tf[j] - trel) : tcap;
        } else {
          done = true;  // the rest is later than the last frame: stays pending
        }
      }
    }
    // ---- 4. frames whose events are all in this or earlier sub-batches
    while (j < f_hi && (float)(int32_t)(a.tf[j] - trel) < tnext) {
      fast_readout<NW, PPL, BM>(a, sm, j, trel, px0, npx, warp, lane, kc);
      ++j;
    }
  }
  while (j < f_hi) {
    fast_readout<NW, PPL, BM>(a, sm, j, trel, px0, npx, warp, lane, kc);
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += NT) {
      a.S[px0 + i] = sm.S[i];
      const float tr = sm.T[i];
      if (tr != t_clamp) a.T[px0 + i] = trel + (int64_t)tr;
    }
  }
}

template <int NW, int PPL, int BM>
cudaError_t launch_fast_t(const IntArgs& a, cudaStream_t s) {
  const size_t smem = fast_smem_bytes<NW, PPL>(a.n_tiles);
  static size_t configured = 0;
  if (smem > configured) {
    const size_t mx = fast_smem_bytes<NW, PPL>(kMaxTilesPerChunk);
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_kernel<NW, PPL, BM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return e;
    configured = mx;
  }
  esi_integrate_kernel<NW, PPL, BM><<<a.nb, NW * 32, smem, s>>>(a);
  return cudaGetLastError();
}

// warps of 128 pixels (4 per lane) for bands up to 2048 pixels, 256 (8 per lane) above
template <int BM>
cudaError_t launch_fast_nw(const IntArgs& a, cudaStream_t s) {
  switch (a.band_px) {
    case 256: return launch_fast_t<2, 4, BM>(a, s);
    case 512: return launch_fast_t<4, 4, BM>(a, s);
    case 1024: return launch_fast_t<8, 4, BM>(a, s);
    case 2048: return launch_fast_t<16, 4, BM>(a, s);
    case 4096: return launch_fast_t<16, 8, BM>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_integrate_fast(const IntArgs& a, cudaStream_t s) {
  return a.dp.bmode == 2 ? launch_fast_nw<2>(a, s) : launch_fast_nw<0>(a, s);
}

}  // namespace esi
