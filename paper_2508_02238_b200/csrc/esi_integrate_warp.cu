// esi_integrate_warp.cu -- K2: per-band integration (Alg. 2) fused
// with the Eq. 13/14 readout of every frame of the
// chunk, with WARP-OWNED pixels (no per-frame-window block barriers).
//
// One CTA of nw warps per band of band_px consecutive pixel ids (K1's
// partition key).  Warp w owns the quads (4 pixels) [w*qpw, (w+1)*qpw) of the
// band, i.e. a contiguous sub-band of <= 4*qpw <= 256 pixels.  The band's state
// lives in shared memory for the whole chunk: S (fp32) and T as an fp32 offset
// from the chunk base ChunkInfo::trel (exact integers: |T| < 2^24 us; pixels
// older than the decay horizon are clamped to -(dt_cut+1), "fully decayed").
//
// Per sub-batch of <= sb band events (arrival order):
//   1. gather: cp.async copies of the band's (tile, band) runs written by K1,
//      in tile order = arrival order (double-buffered: sub-batch k+1 is in
//      flight while k is split and processed);
//   2. split: a stable, order-preserving split of the sub-batch by owner warp
//      (warp w counts the owners of a contiguous slice; ranks within a warp
//      round come from a shared-memory OR of lane bits per owner -- the peer
//      mask -- so they are exact lane (= arrival) order by construction, no
//      reliance on atomic ordering); one block barrier for the counts, one for
//      the scatter;
//   3. process: each warp walks its own list independently.  For every frame
//      window that closes inside the sub-batch it applies its events with
//      t <= t_j 32 at a time, then reads frame j out for its own pixels.
//      Lanes of one round that hit the same pixel are found by the same
//      peer-mask trick on a per-pixel table; the lowest such lane applies the
//      group in lane order.  Every pixel therefore sees its events in stream
//      order, one at a time, in fp32: the result is bit-identical to a
//      sequential fp32 evaluation of Alg. 2 (no reassociation anywhere).
// Decay (Eq. 4, reading A14): u = k_us * ((tau_h - dt) + tau_l) (float pair),
// d = max(u, 0)^b (esi_fast_common.cuh).
#include "esi_device.cuh"

namespace esi {

namespace {

#include "esi_fast_common.cuh"

constexpr int kW2MaxWarps = 16;
constexpr int kW2SB = 3072;                   // events per sub-batch (compile time: constant smem offsets)

// Shared memory of one CTA.  The sub-batch arrays sit at constant offsets (no
// address registers); the band arrays follow at run-time offsets.
struct W2Smem {
  float* S;        // [bp] accumulation
  float* T;        // [bp] last time relative to trel
  uint32_t* M;     // [bp] per-pixel peer masks of one warp round (zero between rounds)
  uint32_t* pre;   // [n_tiles + 1] band events before tile t
  uint16_t* mo;    // [n_tiles] offset of the band's run inside tile t
};
constexpr size_t kW2Cur = 0;                                  // uint2 [kW2SB] gathered sub-batch, arrival order
constexpr size_t kW2List = kW2Cur + (size_t)kW2SB * 8;        // uint2 [kW2SB] split by owner (owner-major)
constexpr size_t kW2Key = kW2List + (size_t)kW2SB * 8;        // u16 [kW2SB] owner << 12 | rank
constexpr size_t kW2Cnt = kW2Key + (size_t)kW2SB * 2;         // u32 [kW2MaxWarps][16] events per (slice, owner)
constexpr size_t kW2Band = kW2Cnt + (size_t)kW2MaxWarps * 16 * 4;

__host__ __device__ inline size_t w2_smem_bytes(int bp, int n_tiles) {
  const size_t b = (size_t)((bp + 3) & ~3);
  return kW2Band + b * 12 + (size_t)(n_tiles + 1) * 4 + (((size_t)n_tiles * 2 + 15) & ~(size_t)15) + 16;
}

__device__ __forceinline__ W2Smem w2_carve(unsigned char* base, int bp, int n_tiles) {
  W2Smem m;
  unsigned char* q = base + kW2Band;
  const int b4 = (bp + 3) & ~3;
  m.S = reinterpret_cast<float*>(q); q += (size_t)b4 * 4;
  m.T = reinterpret_cast<float*>(q); q += (size_t)b4 * 4;
  m.M = reinterpret_cast<uint32_t*>(q); q += (size_t)b4 * 4;
  m.pre = reinterpret_cast<uint32_t*>(q); q += (size_t)(n_tiles + 1) * 4;
  m.mo = reinterpret_cast<uint16_t*>(q);
  return m;
}

// Gather band events [sb0, min(sb0 + sb, n_b)) into dst with cp.async: 8 (tile,
// band) runs per warp step, 4 lanes per run, tiles in order = arrival order.
__device__ __forceinline__ void w2_gather(const uint2* __restrict__ rec, const uint32_t* pre, const uint16_t* mo,
                                          int n_tiles, int n_b, int sb0, int sb, uint2* dst, int gw, int ngw,
                                          int lane) {
  const uint32_t q_end = (uint32_t)min(sb0 + sb, n_b);
  int t_lo = 0;                                 // last tile with pre[t] <= sb0 (32-ary search)
#pragma unroll
  for (int stride = 1024; stride >= 1; stride >>= 5) {
    const int t = t_lo + lane * stride;
    const unsigned b = __ballot_sync(kFull, t < n_tiles && pre[t] <= (uint32_t)sb0);
    t_lo += (31 - __clz(b | 1u)) * stride;
  }
  for (int tb = t_lo + gw * 8; tb < n_tiles; tb += ngw * 8) {
    if (pre[tb] >= q_end) break;                // runs are in order: the rest is later
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

// Frame j for the warp's quads [q0, q1): Eq. 4 + Eq. 13 + Eq. 14, one 4-byte
// streaming store per quad (a warp writes 128 contiguous bytes per step).
template <int BM>
__device__ __forceinline__ void w2_readout(const IntArgs& a, const W2Smem& sm, int j, int32_t tji, int64_t px0,
                                           int npx, int q0, int q1, int lane, const FastConst& c) {
  const float tj = (float)tji;
  const float aj = (float)(tji - (int32_t)c.tau_h);          // t_j - tau (folded mode: tau integer)
  uint8_t* frame = a.out + (int64_t)j * a.P + px0;
  const int nfull = a.vec8 ? min(q1, npx >> 2) : q0;        // quads with 4 pixels and aligned stores
  const float4* S4 = reinterpret_cast<const float4*>(sm.S);
  const float4* T4 = reinterpret_cast<const float4*>(sm.T);
  auto quad = [&](int q) -> uint32_t {
    const float4 s0 = S4[q], t0 = T4[q];
    if (c.fold) {
      float2 w0 = __fadd2_rn(make_float2(t0.x, t0.y), make_float2(-aj, -aj));
      float2 w1 = __fadd2_rn(make_float2(t0.z, t0.w), make_float2(-aj, -aj));
      w0.x = fmaxf(w0.x, 0.f); w0.y = fmaxf(w0.y, 0.f); w1.x = fmaxf(w1.x, 0.f); w1.y = fmaxf(w1.y, 0.f);
      const float2 v0 = __fmul2_rn(make_float2(s0.x, s0.y), __fmul2_rn(w0, w0));
      const float2 v1 = __fmul2_rn(make_float2(s0.z, s0.w), __fmul2_rn(w1, w1));
      const float2 sw2 = make_float2(c.scale_w2, c.scale_w2), off = make_float2(c.off_frac, c.off_frac);
      const float2 mo = make_float2(c.magic_off, c.magic_off);
      const float2 r0 = __fadd2_rd(__ffma2_rn(v0, sw2, off), mo), r1 = __fadd2_rd(__ffma2_rn(v1, sw2, off), mo);
      return __byte_perm(__byte_perm(__float_as_uint(r0.x), __float_as_uint(r0.y), 0x0040),
                         __byte_perm(__float_as_uint(r1.x), __float_as_uint(r1.y), 0x0040), 0x5410);
    }
    const uint32_t b01 = readout2<BM>(make_float2(s0.x, s0.y), make_float2(t0.x, t0.y), tj, aj, c, a.mp.smin,
                                      a.mp.smax);
    const uint32_t b23 = readout2<BM>(make_float2(s0.z, s0.w), make_float2(t0.z, t0.w), tj, aj, c, a.mp.smin,
                                      a.mp.smax);
    return __byte_perm(b01, b23, 0x5410);
  };
  unsigned int* f4 = reinterpret_cast<unsigned int*>(frame);
  int q = q0 + lane;
  for (; q < nfull; q += 32) __stcs(f4 + q, quad(q));
  for (; q < q1; q += 32) {                                  // ragged band end / unaligned output
    const uint32_t v = quad(q);
    const int base = q * 4, n = min(4, npx - base);
    for (int u = 0; u < n; ++u) frame[base + u] = (uint8_t)((v >> (8 * u)) & 0xffu);
  }
}

// One round of up to 32 events of the warp's own list (lanes with `valid`,
// a prefix of the warp): Alg. 2 body per event in stream order.  Lanes that hit
// the same pixel OR their lane bit into M[px]; the lowest lane of each such
// group applies the group's events in lane (= arrival) order in registers.
template <int BM>
__device__ __forceinline__ void w2_apply_round(const W2Smem& sm, const uint2* lst, int e, bool valid, uint2 r,
                                               uint32_t trel32, int lane, const FastConst& k) {
  const int px = (int)(r.y & 0x7fffffffu);
  if (valid) atomicOr(&sm.M[px], 1u << lane);
  __syncwarp();
  const uint32_t peers = valid ? sm.M[px] : 0u;
  __syncwarp();
  if (valid) {
    sm.M[px] = 0u;
    if (peers == (1u << lane)) {
      apply_event<BM>(sm.S, sm.T, px, r, trel32, k);
    } else if ((peers & lanemask_lt()) == 0u) {
      float s = sm.S[px], t = sm.T[px];
      uint32_t m = peers;
      while (m) {
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const uint2 q = lst[e + l];
        const float te = (float)(int32_t)(q.x - trel32);
        const float pc = ((int32_t)q.y < 0) ? -k.C : k.C;
        s = clampS(ev_update<BM>(s, pc, ev_decay<BM>(te - t, k)), k);   // Alg. 2 body
        t = te;
      }
      sm.S[px] = s;
      sm.T[px] = t;
    }
  }
  __syncwarp();
}

template <int BM>
__global__ void __launch_bounds__(kW2MaxWarps * 32) esi_integrate_w2_kernel(IntArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_wsum[32];
  uint2* const cur = reinterpret_cast<uint2*>(smem_raw + kW2Cur);
  uint2* const lst = reinterpret_cast<uint2*>(smem_raw + kW2List);
  uint16_t* const key = reinterpret_cast<uint16_t*>(smem_raw + kW2Key);
  uint32_t* const cnt = reinterpret_cast<uint32_t*>(smem_raw + kW2Cnt);
  const int nw = (int)(blockDim.x >> 5), nthr = (int)blockDim.x;
  const int band = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bp = a.band_px;
  const int64_t px0 = (int64_t)band * bp;
  const int npx = (int)min((int64_t)bp, a.P - px0);
  const int n_tiles = a.n_tiles;

  if (a.gate && *a.gate != kNoError) return;   // lazy validation found an invalid event: write nothing
  const ChunkInfo ci = *a.info;
  const int f_lo = ci.f_lo, f_hi = ci.f_hi;
  const bool active = ci.active != 0;
  if (!active && f_lo >= f_hi) return;
  const W2Smem sm = w2_carve(smem_raw, bp, n_tiles);
  const int64_t trel = ci.trel;
  const uint32_t trel32 = (uint32_t)trel;
  const float t_clamp = -(float)(a.dp.dt_cut + 1);
  const int32_t tcap = (int32_t)min(a.t_cap - trel, (int64_t)(1 << 25));
  const FastConst kc = make_const(a);

  for (int i = threadIdx.x; i < bp; i += nthr) {
    const bool in = i < npx;
    sm.S[i] = in ? a.S[px0 + i] : 0.f;
    sm.T[i] = in ? (float)max(a.T[px0 + i] - trel, (int64_t)t_clamp) : t_clamp;
    sm.M[i] = 0u;
  }
  int n_b = 0;
  if (active) {
    const uint32_t* meta = a.meta + (int64_t)band * n_tiles;
    const int per = (n_tiles + nthr - 1) / nthr;
    const int t0 = threadIdx.x * per;
    uint32_t local = 0;
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) {
      const uint32_t m = meta[t];
      sm.mo[t] = (uint16_t)(m & 0xffffu);
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
    for (int w = 0; w < nw; ++w) {
      const uint32_t v = s_wsum[w];
      if (w < warp) run += v;
      tot += v;
    }
    for (int t = t0; t < min(n_tiles, t0 + per); ++t) {
      sm.pre[t] = run;
      run += meta[t] >> 16;
    }
    if (threadIdx.x == 0) sm.pre[n_tiles] = tot;
    n_b = (int)tot;
  }
  __syncthreads();

  // this warp's quads and the owner of a band pixel: owner(px) = (px >> 2) / qpw
  const int nq_band = (npx + 3) >> 2;
  const int q0 = min(warp * a.w2_qpw, nq_band), q1 = min(q0 + a.w2_qpw, nq_band);
  const uint32_t qmagic = a.w2_qmagic;   // (q * qmagic) >> 32 == q / qpw for q < 2^12
  // lane o < 16 counts owner o: its bits as all-ones / all-zero masks
  const unsigned lb0 = (lane & 1) ? kFull : 0u, lb1 = (lane & 2) ? kFull : 0u;
  const unsigned lb2 = (lane & 4) ? kFull : 0u, lb3 = (lane & 8) ? kFull : 0u;
  // slice of the sub-batch this warp splits: [warp * per, (warp + 1) * per)
  const int per_full = (((kW2SB + nw - 1) / nw) + 31) & ~31;

  int j = f_lo;
  bool done = false;
  if (n_b > 0) w2_gather(a.rec, sm.pre, sm.mo, n_tiles, n_b, 0, kW2SB, cur, warp, nw, lane);
  for (int sb0 = 0; sb0 < n_b && !done; sb0 += kW2SB) {
    const int n_sb = min(kW2SB, n_b - sb0);
    cp_async_wait_all();
    __syncthreads();                                   // [A] cur complete; every warp is done with lst
    // ---- split, count pass: warp `warp` ranks the slice [i0, i1) by owner (4 ballots:
    // the peers of a lane are the lanes whose owner bits all match; ranks = lane order)
    const int per = n_sb == kW2SB ? per_full : (((n_sb + nw - 1) / nw) + 31) & ~31;
    const int i0 = min(warp * per, n_sb), i1 = min(i0 + per, n_sb);
    uint32_t cnt_o = 0;                                // lane o < 16: events of owner o so far
    for (int i = i0; i < i1; i += 32) {
      const int idx = i + lane;
      const bool valid = idx < i1;
      const uint32_t px = valid ? (cur[idx].y & 0x7fffffffu) : 0u;
      const uint32_t owner = (uint32_t)(((uint64_t)(px >> 2) * qmagic) >> 32);
      const unsigned vm = __ballot_sync(kFull, valid);
      const unsigned b0 = __ballot_sync(kFull, owner & 1u), b1 = __ballot_sync(kFull, owner & 2u);
      const unsigned b2 = __ballot_sync(kFull, owner & 4u), b3 = __ballot_sync(kFull, owner & 8u);
      const unsigned ob0 = (owner & 1u) ? kFull : 0u, ob1 = (owner & 2u) ? kFull : 0u;
      const unsigned ob2 = (owner & 4u) ? kFull : 0u, ob3 = (owner & 8u) ? kFull : 0u;
      const unsigned peers = vm & ~(b0 ^ ob0) & ~(b1 ^ ob1) & ~(b2 ^ ob2) & ~(b3 ^ ob3);
      const unsigned mine = vm & ~(b0 ^ lb0) & ~(b1 ^ lb1) & ~(b2 ^ lb2) & ~(b3 ^ lb3);
      const uint32_t base = __shfl_sync(kFull, cnt_o, (int)owner);
      cnt_o += __popc(mine);
      if (valid) key[idx] = (uint16_t)((owner << 12) | (base + __popc(peers & lanemask_lt())));
    }
    if (lane < 16) cnt[warp * 16 + lane] = cnt_o;
    __syncthreads();                                   // [B] counts complete
    // list of owner o starts at start_o = sum_{o' < o} col_o'; this slice's run of it at + part
    uint32_t col = 0, part = 0;
    if (lane < nw)
      for (int w = 0; w < nw; ++w) {
        const uint32_t c = cnt[w * 16 + lane];
        col += c;
        part += (w < warp) ? c : 0u;
      }
    uint32_t incl = col;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t start = incl - col;
    const uint32_t wpos = start + part;
    for (int i = i0; i < i1; i += 32) {
      const int idx = i + lane;
      const bool valid = idx < i1;
      const uint32_t k = valid ? key[idx] : 0u;
      const uint32_t pos = __shfl_sync(kFull, wpos, (int)(k >> 12)) + (k & 4095u);
      if (valid) {
        ESI_DCHECK(pos < (uint32_t)n_sb);
        lst[pos] = cur[idx];
      }
    }
    const int ls = (int)__shfl_sync(kFull, start, warp);
    const int le = ls + (int)__shfl_sync(kFull, col, warp);
    const bool last_sb = sb0 + kW2SB >= n_b;
    const int32_t t_last = (int32_t)(cur[n_sb - 1].x - trel32);
    __syncthreads();                                   // [C] lists complete; cur is free
    if (!last_sb) w2_gather(a.rec, sm.pre, sm.mo, n_tiles, n_b, sb0 + kW2SB, kW2SB, cur, warp, nw, lane);
    // ---- process this warp's own list: windows that close inside the sub-batch
    int e = ls;
    while (true) {
      bool closed = false;
      int32_t lim = tcap;
      int32_t tw = 0;
      if (j < f_hi) {
        tw = (int32_t)(a.tf[j] - trel);
        closed = last_sb || tw < t_last;
        if (closed) lim = tw;
      }
      while (e < le) {                                  // own events with t <= lim, 32 at a time
        const int idx = e + lane;
        bool valid = idx < le;
        const uint2 r = valid ? lst[idx] : make_uint2(0u, 0u);
        valid = valid && (int32_t)(r.x - trel32) <= lim;
        const int n = __popc(__ballot_sync(kFull, valid));   // the list is time-sorted: a prefix
        if (n == 0) break;
        w2_apply_round<BM>(sm, lst, e, valid, r, trel32, lane, kc);
        e += n;
        if (n < 32) break;
      }
      if (!closed) break;
      w2_readout<BM>(a, sm, j, tw, px0, npx, q0, q1, lane, kc);
      ++j;
    }
    done = j >= f_hi && t_last > tcap;                 // later events stay pending
  }
  cp_async_wait_all();
  // ---- frames after the chunk's last event (or of a band without events)
  while (j < f_hi) {
    w2_readout<BM>(a, sm, j, (int32_t)(a.tf[j] - trel), px0, npx, q0, q1, lane, kc);
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += nthr) {
      a.S[px0 + i] = sm.S[i];
      const float tr = sm.T[i];
      if (tr != t_clamp) a.T[px0 + i] = trel + (int64_t)tr;
    }
  }
}

template <int BM>
cudaError_t launch_w2_b(const IntArgs& a, cudaStream_t s) {
  const size_t smem = w2_smem_bytes(a.band_px, a.n_tiles);
  int dev = 0;
  cudaGetDevice(&dev);
  static int configured[64] = {0};   // per device: the attribute is per context
  if (dev < 0 || dev >= 64 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_w2_kernel<BM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)w2_smem_bytes(kMaxBandPx, kMaxTilesPerChunk));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev] = 1;
  }
  esi_integrate_w2_kernel<BM><<<a.nb, a.w2_nw * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t integrate_w2_smem_bytes(int band_px, int n_tiles) { return w2_smem_bytes(band_px, n_tiles); }

cudaError_t launch_integrate_w2(const IntArgs& a, cudaStream_t s) {
  if (a.dp.first)
    return a.dp.bmode == 2           ? launch_w2_b<2 + kFirst>(a, s)
           : a.dp.bmode == kDecayExp ? launch_w2_b<kDecayExp + kFirst>(a, s)
                                     : launch_w2_b<kFirst>(a, s);
  return a.dp.bmode == 2           ? launch_w2_b<2>(a, s)
         : a.dp.bmode == kDecayExp ? launch_w2_b<kDecayExp>(a, s)
                                   : launch_w2_b<0>(a, s);
}

}  // namespace esi
