// esi_fast_common.cuh -- arithmetic shared by the two K2 variants of the fast
// (32-bit relative time) path: decay (Eq. 4), clamp (Eq. 13), readout (Eq. 14),
// the Alg. 2 event body, the dense-pixel warp scan of clamped affine maps, and
// small copy/search helpers.  Included inside namespace esi { namespace { ... } }.
#pragma once

constexpr int kSlots = 8;   // events of one pixel in one segment applied by a single thread
constexpr uint32_t kEmpty = 0xffffu;


struct FastConst {
  float tau_h, tau_l;                  // tau = 1e6/k us = tau_h + tau_l
  float kh, kl, k_tau_l;               // k_us = kh + kl (no systematic bias), k_us * tau_l
  float b;
  float C, smin, smax;                 // per-event clamp bounds (+-FLT_MAX when the state is unclamped)
  float scale, off_frac, magic_off;    // map: byte = low8(bits(rd(v*scale + off_frac + 2^23 + off_int)))
  float scale_w2;                      // k_us^2 * scale: Eq. 14 of S*(k w)^2 with k^2 folded in
  int32_t tau_int;                     // tau is an integer (tau_l == 0)
  int32_t tau_i;                       // (int32_t)tau_h: tau itself in the folded mode
  int32_t fold;                        // readout mode: 1 = folded (b = 2, readout decay, no clamp, integer tau)
  int32_t rd, cl;                      // readout decay; readout clamp needed (bounds exclude 0)
  float dtc;                           // exponential variant: d = 0 for dt >= dtc (k dt >= 24)
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
  c.smin = a.mp.ev_smin;
  c.smax = a.mp.ev_smax;
  c.scale = a.mp.scale;
  c.off_frac = a.mp.off_frac;
  c.magic_off = a.mp.magic_off;
  c.scale_w2 = a.mp.scale_w2;
  c.tau_int = a.dp.tau_l == 0.f;
  c.tau_i = a.dp.tau_i;
  c.rd = a.mp.readout_decay != 0;
  c.cl = a.mp.readout_clamp;           // bounds exclude 0, or unclamped state: clamp at readout
  c.fold = a.dp.bmode == 2 && c.rd && !c.cl && c.tau_int;   // readout only: independent of the order
  c.dtc = (float)a.dp.dt_cut;          // < 2^23 on the fast path: exact
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

// Kernel variant BM = decay kind (0: exp2(b log2 u), 2: b = 2, kDecayExp) + kFirst
// for the decay-then-add order; both compile-time, so the default path is unchanged.
constexpr int kFirst = 16;

template <int BM>
__device__ __forceinline__ float ev_decay(float dt, const FastConst& c) {
  constexpr int K = BM & (kFirst - 1);
  if (K == kDecayExp)                  // exponential variant (A20): exp(-k dt), 0 from k dt >= 24 on
    return dt >= c.dtc ? 0.f : expf(-fmaf(c.kh, dt, c.kl * dt));
  const float u = decay_u(dt, c);
  if (K == 2) return u * u;
  return exp2f(c.b * __log2f(u));      // log2(0) = -inf -> d = 0
}

// One event's update of the state s before the clamp: Alg. 2
// S <- (S + p C) d, or the decay-then-add variant S <- S d + p C.
template <int BM>
__device__ __forceinline__ float ev_update(float s, float pc, float d) {
  return (BM & kFirst) ? fmaf(s, d, pc) : (s + pc) * d;
}

// Eq. 13 clamp of one event's result.
__device__ __forceinline__ float clampS(float s, const FastConst& c) { return fminf(fmaxf(s, c.smin), c.smax); }

// Readout of 2 pixels (reading A4: v = S d(t_j - T), non-mutating; Eq. 13 clamp
// when the bounds exclude 0; Eq. 14 rounded half away from zero, reading A8).
// Folded mode (b = 2, integer tau, bounds containing 0): with w = T - (t_j - tau)
// = tau - dt (exact), d = (k w)^2 for w > 0 and 0 otherwise, so
//   x = S w^2 (k^2 scale) + off_frac   -- 4 packed f32x2 ops + 2 max per 2 pixels.
template <int BM>
__device__ __forceinline__ uint32_t readout2(float2 s, float2 T, float tj, float aj, const FastConst& c, float rmin,
                                             float rmax) {   // rmin, rmax: Eq. 13 bounds of the readout
  float2 x;
  if (c.fold) {
    float2 w = __fadd2_rn(T, make_float2(-aj, -aj));                          // tau - dt, exact
    w.x = fmaxf(w.x, 0.f);
    w.y = fmaxf(w.y, 0.f);
    const float2 v = __fmul2_rn(s, __fmul2_rn(w, w));
    x = __ffma2_rn(v, make_float2(c.scale_w2, c.scale_w2), make_float2(c.off_frac, c.off_frac));
  } else {
    float2 v = s;
    if (c.rd) v = __fmul2_rn(s, make_float2(ev_decay<BM>(tj - T.x, c), ev_decay<BM>(tj - T.y, c)));
    if (c.cl) {
      v.x = fminf(fmaxf(v.x, rmin), rmax);
      v.y = fminf(fmaxf(v.y, rmin), rmax);
    }
    x = __ffma2_rn(v, make_float2(c.scale, c.scale), make_float2(c.off_frac, c.off_frac));
  }
  const float2 r = __fadd2_rd(x, make_float2(c.magic_off, c.magic_off));   // 2^23 + off_int + floor(x)
  return __byte_perm(__float_as_uint(r.x), __float_as_uint(r.y), 0x0040);  // 2 bytes in the low half
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Alg. 2 loop body for one event of pixel px, sequentially.
template <int BM>
__device__ __forceinline__ void apply_event(float* S, float* T, int px, uint2 ev, uint32_t trel,
                                            const FastConst& k) {
  const float te = (float)(int32_t)(ev.x - trel);
  const float pc = ((int32_t)ev.y < 0) ? -k.C : k.C;
  // S <- S + p C; S <- S max{(1 - k dt)^b, 0} (or the variant's order / decay)
  const float s = ev_update<BM>(S[px], pc, ev_decay<BM>(te - T[px], k));
  S[px] = clampS(s, k);                                   // S <- min(max(S, S_min), S_max)
  T[px] = te;                                             // T <- t
}

// Dense pixel (> kSlots events in the segment): one warp composes the events'
// clamped affine maps s -> clamp(a s + c, lo, hi), a >= 0:
// event i is f_i = (d_i, d_i p_i C, S_min, S_max) and
//   F o G = (aF aG, aF cG + cF, clamp(aF loG + cF, loF, hiF), clamp(aF hiG + cF, loF, hiF)).
// The pixel's events are compacted from the segment into the warp's staging
// (arrival order) 32 at a time, their maps are combined by a warp-shuffle
// inclusive scan, and the last prefix is applied to the state.
template <int BM>
__device__ __forceinline__ void dense_pixel_apply(float* S, float* T, const uint2* sub, uint2* stage, int e0,
                                                  int e1, int q, uint32_t trel, int lane, const FastConst& k) {
  float s = S[q], tprev = T[q];
  int base = e0, cnt = 0;                                   // segment position; compacted events in stage
  while (true) {
    // compact the pixel's events (arrival order) until 32 are staged or the segment ends:
    // a segment of a few dozen events with ~10 of the pixel's costs one scan, not one per 32
    while (cnt < 32 && base < e1) {
      const int i = base + lane;
      const uint2 ev = i < e1 ? sub[i] : make_uint2(0u, 0xffffffffu);
      const bool mine = i < e1 && (int)(ev.y & 0x7fffffffu) == q;
      const unsigned m = __ballot_sync(kFull, mine);
      if (mine) stage[cnt + __popc(m & lanemask_lt())] = ev;   // cnt + 32 <= 64 <= kStage
      cnt += __popc(m);
      base += 32;
    }
    if (cnt == 0) break;
    __syncwarp();
    const int nk = min(cnt, 32);
    const uint2 cev = stage[lane];
    const uint2 rest = stage[32 + lane];
    __syncwarp();
    if (lane < cnt - nk) stage[lane] = rest;               // the overflow moves to the front
    cnt -= nk;
    const float te = (float)(int32_t)(cev.x - trel);
    float tp = __shfl_up_sync(kFull, te, 1);
    if (lane == 0) tp = tprev;
    const bool act = lane < nk;
    const float d = act ? ev_decay<BM>(te - tp, k) : 1.f;
    const float pc = ((int32_t)cev.y < 0) ? -k.C : k.C;
    float fa = d, fc = act ? ((BM & kFirst) ? pc : d * pc) : 0.f, flo = k.smin, fhi = k.smax;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const float ga = __shfl_up_sync(kFull, fa, off), gc = __shfl_up_sync(kFull, fc, off);
      const float glo = __shfl_up_sync(kFull, flo, off), ghi = __shfl_up_sync(kFull, fhi, off);
      if (lane >= off) {                                  // F <- F o G (G = earlier events)
        const float nlo = fminf(fmaxf(fmaf(fa, glo, fc), flo), fhi);
        const float nhi = fminf(fmaxf(fmaf(fa, ghi, fc), flo), fhi);
        fc = fmaf(fa, gc, fc);
        fa = fa * ga;
        flo = nlo;
        fhi = nhi;
      }
    }
    const float La = __shfl_sync(kFull, fa, nk - 1), Lc = __shfl_sync(kFull, fc, nk - 1);
    const float Llo = __shfl_sync(kFull, flo, nk - 1), Lhi = __shfl_sync(kFull, fhi, nk - 1);
    s = fminf(fmaxf(fmaf(La, s, Lc), Llo), Lhi);
    tprev = __shfl_sync(kFull, te, nk - 1);
    __syncwarp();
  }
  if (lane == 0) {
    S[q] = s;
    T[q] = tprev;
  }
}

// number of sub-batch events in [0, n) with relative time <= tj (times sorted, n <= kSB):
// warp-wide 32-ary search, identical in every warp (no barrier needed)
template <int SB>
__device__ __forceinline__ int upper_bound_rel(const uint2* sub, int n, uint32_t trel, int32_t tj, int lane) {
  int lo = 0;
#pragma unroll
  for (int stride = SB > 1024 ? 1024 : 32; stride >= 1; stride >>= 5) {
    const int p = lo + lane * stride;
    const bool le = p < n && (int32_t)(sub[p].x - trel) <= tj;
    const unsigned b = __ballot_sync(kFull, le);
    if (b == 0u) return lo;                               // sub[lo] > tj (lo is always a candidate)
    lo += (31 - __clz(b)) * stride;
  }
  return lo + 1;
}


// Where the band's events of the chunk are: K1 wrote, per tile t, the band's run
// at rec[t * kTile + mo[t]] with count cnt[t] (meta[t] = mo | cnt << 16).
// Fills pre[t] = band events before tile t (pre[n_tiles] = total) and mo[t];
// returns the total.  Block-wide (NW warps), one barrier inside.
template <int NW>
__device__ __forceinline__ int band_run_prefix(const uint32_t* __restrict__ meta, int n_tiles, uint32_t* pre,
                                               uint16_t* mo, uint32_t* s_wsum) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = (n_tiles + NW * 32 - 1) / (NW * 32);
  const int t0 = threadIdx.x * per;
  uint32_t local = 0;
  for (int t = t0; t < min(n_tiles, t0 + per); ++t) {
    const uint32_t m = meta[t];
    mo[t] = (uint16_t)(m & 0xffffu);
    local += m >> 16;
  }
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
    run += meta[t] >> 16;
  }
  if (threadIdx.x == 0) pre[n_tiles] = tot;
  return (int)tot;
}

// Gather band events [sb0, min(sb0 + SB, n_b)) into dst with cp.async: 8 (tile,
// band) segments per warp step, 4 lanes per segment, tiles in order = arrival order.
// Warps gw = 0 .. ngw-1 share the copies.
template <int SB>
__device__ __forceinline__ void gather_sub(const uint2* __restrict__ rec, const uint32_t* pre, const uint16_t* mo,
                                           int n_tiles, int n_b, int sb0, uint2* dst, int gw, int ngw, int lane) {
  const uint32_t q_end = (uint32_t)min(sb0 + SB, n_b);
  int t_lo = 0;                                 // last tile with pre[t] <= sb0 (32-ary search)
#pragma unroll
  for (int stride = 1024; stride >= 1; stride >>= 5) {
    const int t = t_lo + lane * stride;
    const unsigned b = __ballot_sync(kFull, t < n_tiles && pre[t] <= (uint32_t)sb0);
    t_lo += (31 - __clz(b | 1u)) * stride;
  }
  for (int tb = t_lo + gw * 8; tb < n_tiles; tb += ngw * 8) {
    if (pre[tb] >= q_end) break;                // segments are in order: the rest is later
    const int t = tb + (lane >> 2);
    uint32_t i0 = 0, i1 = 0, p0 = 0;
    const uint2* src = rec;
    if (t < n_tiles) {
      p0 = pre[t];
      if (p0 < q_end) {
        i0 = p0 < (uint32_t)sb0 ? (uint32_t)sb0 - p0 : 0u;
        i1 = min(pre[t + 1], q_end) - p0;
      }
      src += (size_t)t * kTile + mo[t];
    }
    const int dofs = (int)p0 - sb0;             // >= -i0
    for (uint32_t i = i0 + (lane & 3); i < i1; i += 4) cp_async8(&dst[dofs + (int)i], src + i);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
