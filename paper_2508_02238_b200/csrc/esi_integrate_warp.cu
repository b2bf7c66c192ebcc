// esi_integrate_warp.cu -- K2, warp-autonomous variant: per-band integration
// (Alg. 2) fused with the Eq. 13/14 readout (P:218, P:227,
// P:254-259) of every frame of the chunk.
//
// One CTA of 16 warps per band (band_px pixels, a run-time multiple of 64).
// Warp w OWNS the pixels [w*wpx, (w+1)*wpx) of the band (wpx = band_px / 16)
// for the whole chunk: it applies their events and reads them out, so after a
// block-level split of each sub-batch the warps never wait for one another.
//
// Per sub-batch of kWSB band events (arrival order; double-buffered cp.async
// gather of the band's (tile, band) segments written by K1):
//   split  : warp w ranks the events of its 128-event slice among the slice's
//            events bound for the same owner warp (__match_any_sync), a warp-0
//            scan of the 16 x 16 slice/owner counts gives the offsets, and the
//            events are scattered to lst[] -- owner-major, arrival-order-minor
//            (a stable 16-way split; 3 block barriers per sub-batch);
//   walk   : each warp walks its list window by window (events with t <= t_j,
//            a warp-wide ballot search), claims its pixels with generation-
//            tagged atomic exchanges (chains in claim order, __syncwarp only),
//            applies singles directly (sparse path, bit-identical to
//            sequential fp32), chains of 2..8 events one per lane after a
//            sorting network restores arrival order (also sequential fp32),
//            longer chains with the warp-shuffle scan of clamped affine maps
//            (dense path), and at the window end reads its pixels out for
//            frame j (packed f32x2 Eq. 4/13/14, 4-byte streaming stores).
// A warp whose list ends inside window j continues that window in the next
// sub-batch; its own pixels cannot receive events from other warps' lists, so
// reading frame j out needs nothing but its own list.
#include "esi_device.cuh"

namespace esi {

namespace {

#include "esi_fast_common.cuh"

constexpr int kWNW = 16;                      // warps per CTA
constexpr int kWNT = kWNW * 32;
constexpr int kWSB = 2048;                    // events per sub-batch (4 per thread in the split)
constexpr int kWEPT = kWSB / kWNT;

struct WarpSmem {
  float* S;                                   // [bp] accumulation (fp32)
  float* T;                                   // [bp] last time, relative to trel (exact integers)
  uint32_t* head;                             // [bp] last claimer (list index) | generation << 16
  uint16_t* next;                             // [kWSB] previous claimer (claim-order chain)
  uint2* sub[2];                              // [kWSB] gathered sub-batches (double buffer)
  uint2* lst;                                 // [kWSB] owner-major split of the current sub-batch
  uint2* stage;                               // [kWNW][96]: chain heads (u32 x 128) + dense compaction (32)
  uint32_t* cnt;                              // [kWNW][kWNW] slice x owner counts -> offsets
  uint32_t* lbeg;                             // [kWNW + 1] list starts
  uint32_t* pre;                              // [n_tiles + 1]
  uint32_t* mt;                               // [n_tiles]
};

__host__ __device__ inline size_t warp_smem_bytes(int bp, int n_tiles) {
  return (size_t)bp * 12 + kWSB * 2 + 3 * (size_t)kWSB * 8 + kWNW * 96 * 8 + kWNW * kWNW * 4 + (kWNW + 4) * 4 +
         (size_t)(2 * n_tiles + 1) * 4 + 64;
}

__device__ __forceinline__ WarpSmem carve_w(unsigned char* base, int bp, int n_tiles) {
  WarpSmem m;
  unsigned char* q = base;
  m.sub[0] = reinterpret_cast<uint2*>(q); q += kWSB * 8;
  m.sub[1] = reinterpret_cast<uint2*>(q); q += kWSB * 8;
  m.lst = reinterpret_cast<uint2*>(q); q += kWSB * 8;
  m.stage = reinterpret_cast<uint2*>(q); q += kWNW * 96 * 8;
  m.S = reinterpret_cast<float*>(q); q += (size_t)bp * 4;
  m.T = reinterpret_cast<float*>(q); q += (size_t)bp * 4;
  m.head = reinterpret_cast<uint32_t*>(q); q += (size_t)bp * 4;
  m.cnt = reinterpret_cast<uint32_t*>(q); q += kWNW * kWNW * 4;
  m.lbeg = reinterpret_cast<uint32_t*>(q); q += (kWNW + 4) * 4;
  m.pre = reinterpret_cast<uint32_t*>(q); q += (size_t)(n_tiles + 1) * 4;
  m.mt = reinterpret_cast<uint32_t*>(q); q += (size_t)n_tiles * 4;
  m.next = reinterpret_cast<uint16_t*>(q);
  return m;
}

// Gather band events [sb0, min(sb0 + kWSB, n_b)) into dst with cp.async: 8 (tile,
// band) segments per warp step, 4 lanes per segment, tiles in order = arrival order.
__device__ __forceinline__ void gather_w(const uint2* __restrict__ rec, const uint32_t* pre, const uint32_t* mt,
                                         int n_tiles, int n_b, int sb0, uint2* dst, int warp, int lane) {
  const uint32_t q_end = (uint32_t)min(sb0 + kWSB, n_b);
  int t_lo;                                     // last tile with pre[t] <= sb0 (32-ary search)
  {
    const int c = lane * 32;
    const unsigned b1 = __ballot_sync(kFull, c < n_tiles && pre[c] <= (uint32_t)sb0);
    const int blk = 31 - __clz(b1 | 1u);
    const int t = blk * 32 + lane;
    const unsigned b2 = __ballot_sync(kFull, t < n_tiles && pre[t] <= (uint32_t)sb0);
    t_lo = blk * 32 + (31 - __clz(b2 | 1u));
  }
  for (int tb = t_lo + warp * 8; tb < n_tiles; tb += kWNW * 8) {
    if (pre[tb] >= q_end) break;                // segments are in order: the rest is later
    const int t = tb + (lane >> 2);
    uint32_t i0 = 0, i1 = 0, p0 = 0;
    const uint2* src = rec;
    if (t < n_tiles) {
      p0 = pre[t];
      const uint32_t m = mt[t];
      if (p0 < q_end) {
        i0 = p0 < (uint32_t)sb0 ? (uint32_t)sb0 - p0 : 0u;
        i1 = min(m >> 16, q_end - p0);
      }
      src += (size_t)t * kTile + (m & 0xffffu);
    }
    const int dofs = (int)p0 - sb0;             // >= -i0
    for (uint32_t i = i0 + (lane & 3); i < i1; i += 4) cp_async8(&dst[dofs + (int)i], src + i);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Chain heads wl[0..nch) of one window (list indices): collect each chain
// (claim order), sort it back to arrival order with a 19-comparator network,
// apply it in registers; more than kSlots events -> dense path (warp scan).
template <int BM>
__device__ __forceinline__ void warp_chains(const WarpSmem& sm, const uint32_t* wl, int nch, int e0, int e1,
                                            uint2* dstage, uint32_t trel, int lane, const FastConst& k) {
  for (int cb = 0; cb < nch; cb += 32) {
    bool dense = false;
    int dpx = 0;
    if (cb + lane < nch) {
      const uint32_t me = wl[cb + lane];
      const int px = (int)(sm.lst[me].y & 0x7fffffffu);
      uint32_t id[kSlots];
      id[0] = me;
      int c = 1;
#pragma unroll
      for (int q = 1; q < kSlots; ++q) {
        const uint32_t n = (c == q) ? sm.next[id[q - 1]] : kEmpty;
        id[q] = n;
        c += (n != kEmpty) ? 1 : 0;
      }
      if (c == kSlots && sm.next[id[kSlots - 1]] != kEmpty) {
        dense = true;
        dpx = px;
      } else {
#define ESI_CSWAP(x, y) { const uint32_t lo_ = min(id[x], id[y]), hi_ = max(id[x], id[y]); id[x] = lo_; id[y] = hi_; }
        ESI_CSWAP(0, 1) ESI_CSWAP(2, 3) ESI_CSWAP(4, 5) ESI_CSWAP(6, 7)
        ESI_CSWAP(0, 2) ESI_CSWAP(1, 3) ESI_CSWAP(4, 6) ESI_CSWAP(5, 7)
        ESI_CSWAP(1, 2) ESI_CSWAP(5, 6) ESI_CSWAP(0, 4) ESI_CSWAP(3, 7)
        ESI_CSWAP(1, 5) ESI_CSWAP(2, 6)
        ESI_CSWAP(1, 4) ESI_CSWAP(3, 6)
        ESI_CSWAP(2, 4) ESI_CSWAP(3, 5)
        ESI_CSWAP(3, 4)
#undef ESI_CSWAP
        float s = sm.S[px], t = sm.T[px];
        for (int q = 0; q < c; ++q) {
          uint32_t iq = id[0];
#pragma unroll
          for (int u = 1; u < kSlots; ++u) iq = (q == u) ? id[u] : iq;     // register select
          const uint2 e = sm.lst[iq];
          const float te = (float)(int32_t)(e.x - trel);
          const float pc = ((int32_t)e.y < 0) ? -k.C : k.C;
          s = clampS((s + pc) * ev_decay<BM>(te - t, k), k);   // Alg. 2 body
          t = te;
        }
        sm.S[px] = s;
        sm.T[px] = t;
      }
    }
    unsigned dm = __ballot_sync(kFull, dense);
    while (dm) {                                 // dense pixels: the whole warp scans the window
      const int l = __ffs(dm) - 1;
      dm &= dm - 1;
      const int q = __shfl_sync(kFull, dpx, l);
      dense_pixel_apply<BM>(sm.S, sm.T, sm.lst, dstage, e0, e1, q, trel, lane, k);
    }
  }
}

// One window of one warp's list, lst[e0..e1): claim, apply, chains.
template <int BM>
__device__ __forceinline__ void warp_segment(const WarpSmem& sm, int e0, int e1, uint32_t gen, int warp,
                                             int lane, uint32_t trel, const FastConst& k) {
  const uint32_t tag = gen << 16;
  for (int i = e0 + lane; i < e1; i += 32) {              // claim
    const int px = (int)(sm.lst[i].y & 0x7fffffffu);
    const uint32_t old = atomicExch(&sm.head[px], tag | (uint32_t)i);
    sm.next[i] = (old & 0xffff0000u) == tag ? (uint16_t)old : (uint16_t)kEmpty;
  }
  __syncwarp();
  uint32_t* wl = reinterpret_cast<uint32_t*>(sm.stage + warp * 96);   // 128 chain heads
  uint2* dstage = sm.stage + warp * 96 + 64;                          // 32 dense-compaction slots
  int nch = 0;
  for (int ib = e0; ib < e1; ib += 32) {                  // apply singles; chains deferred
    const int i = ib + lane;
    bool chain = false;
    if (i < e1) {
      const uint2 ev = sm.lst[i];
      const int px = (int)(ev.y & 0x7fffffffu);
      if (sm.head[px] == (tag | (uint32_t)i)) {
        if (sm.next[i] == kEmpty) apply_event<BM>(sm.S, sm.T, px, ev, trel, k);
        else chain = true;
      }
    }
    const unsigned bc = __ballot_sync(kFull, chain);
    if (chain) wl[nch + __popc(bc & lanemask_lt())] = (uint32_t)i;
    nch += __popc(bc);
    if (nch > 96) {                                       // flush before the list can overflow
      __syncwarp();
      warp_chains<BM>(sm, wl, nch, e0, e1, dstage, trel, lane, k);
      __syncwarp();
      nch = 0;
    }
  }
  __syncwarp();
  warp_chains<BM>(sm, wl, nch, e0, e1, dstage, trel, lane, k);
  __syncwarp();
}

// Frame j for this warp's pixels [wlo, whi): 4 pixels per lane-iteration.
template <int BM>
__device__ __forceinline__ void warp_readout(const IntArgs& a, const WarpSmem& sm, int j, int64_t trel,
                                             int64_t px0, int wlo, int whi, int lane, const FastConst& c) {
  const int32_t tji = (int32_t)(a.tf[j] - trel);
  const float tj = (float)tji;
  const float aj = (float)(tji - (int32_t)c.tau_h);          // t_j - tau (folded mode: tau integer)
  uint8_t* frame = a.out + (int64_t)j * a.P + px0;
  for (int base = wlo + 4 * lane; base < whi; base += 128) {
    const float4 s0 = *reinterpret_cast<const float4*>(&sm.S[base]);
    const float4 t0 = *reinterpret_cast<const float4*>(&sm.T[base]);
    const uint32_t b01 = readout2<BM>(make_float2(s0.x, s0.y), make_float2(t0.x, t0.y), tj, aj, c);
    const uint32_t b23 = readout2<BM>(make_float2(s0.z, s0.w), make_float2(t0.z, t0.w), tj, aj, c);
    const uint32_t v = __byte_perm(b01, b23, 0x5410);
    if (a.vec8 && base + 4 <= whi) {
      st_stream4(frame + base, v);
    } else {
      const int n = min(4, whi - base);
      for (int u = 0; u < n; ++u) frame[base + u] = (uint8_t)((v >> (8 * u)) & 0xffu);
    }
  }
}

template <int BM>
__global__ void __launch_bounds__(kWNT, 2) esi_integrate_warp_kernel(IntArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_wsum[32];
  const int band = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bp = a.band_px;
  const int64_t px0 = (int64_t)band * bp;
  const int npx = (int)min((int64_t)bp, a.P - px0);
  const int n_tiles = a.n_tiles;
  const WarpSmem sm = carve_w(smem_raw, bp, n_tiles);

  const ChunkInfo ci = *a.info;
  const int f_lo = ci.f_lo, f_hi = ci.f_hi;
  const bool active = ci.active != 0;
  if (!active && f_lo >= f_hi) return;
  const int64_t trel = ci.trel;
  const uint32_t trel32 = (uint32_t)trel;
  const float t_clamp = -(float)(a.dp.dt_cut + 1);
  const int32_t tcap = (int32_t)min(a.t_cap - trel, (int64_t)(1 << 25));
  const FastConst kc = make_const(a);
  const int wpx = bp / kWNW;                                // multiple of 4 (bp multiple of 64)
  const uint32_t wmagic = (uint32_t)((0x100000000ull + (uint64_t)wpx - 1) / (uint64_t)wpx);   // px / wpx, px < 2^13
  const int wlo = warp * wpx, whi = min(wlo + wpx, npx);

  for (int i = threadIdx.x; i < bp; i += kWNT) {
    const bool in = i < npx;
    sm.S[i] = in ? a.S[px0 + i] : 0.f;
    sm.T[i] = in ? (float)max(a.T[px0 + i] - trel, (int64_t)t_clamp) : t_clamp;
    sm.head[i] = 0u;                          // generation 0: never a live claim
  }
  int n_b = 0;
  if (active) {
    for (int t = threadIdx.x; t < n_tiles; t += kWNT) sm.mt[t] = a.meta[(int64_t)band * n_tiles + t];
    __syncthreads();
    const int per = (n_tiles + kWNT - 1) / kWNT;
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
    for (int w = 0; w < kWNW; ++w) {
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

  int j = f_lo;                                 // next frame of THIS warp's pixels
  int32_t tj = (j < f_hi) ? (int32_t)(a.tf[j] - trel) : tcap;
  bool wdone = false;
  uint32_t gen = 0;
  if (n_b > 0) gather_w(a.rec, sm.pre, sm.mt, n_tiles, n_b, 0, sm.sub[0], warp, lane);
  for (int sb0 = 0, kb = 0; sb0 < n_b; sb0 += kWSB, ++kb) {
    const int n_sb = min(kWSB, n_b - sb0);
    const uint2* sub = (kb & 1) ? sm.sub[1] : sm.sub[0];
    if (lane < kWNW) sm.cnt[warp * kWNW + lane] = 0;
    cp_async_wait_all();
    __syncthreads();                            // sub-batch landed; every warp done with lst
    if (sb0 + kWSB < n_b)
      gather_w(a.rec, sm.pre, sm.mt, n_tiles, n_b, sb0 + kWSB, (kb & 1) ? sm.sub[0] : sm.sub[1], warp, lane);
    // ---- split: stable 16-way partition of the sub-batch by owner warp
    uint2 ev[kWEPT];
    uint32_t pos[kWEPT];
#pragma unroll
    for (int r = 0; r < kWEPT; ++r) {
      const int i = warp * (kWEPT * 32) + r * 32 + lane;
      const bool act = i < n_sb;
      ev[r] = act ? sub[i] : make_uint2(0u, 0u);
      const uint32_t px = ev[r].y & 0x7fffffffu;
      const int own = act ? (int)__umulhi(px, wmagic) : kWNW + lane;
      const unsigned peers = __match_any_sync(kFull, own);
      const uint32_t rank = __popc(peers & lanemask_lt());
      uint32_t base = 0;
      if (act) base = sm.cnt[warp * kWNW + own];
      __syncwarp();
      if (act && rank == 0) sm.cnt[warp * kWNW + own] = base + __popc(peers);
      __syncwarp();
      pos[r] = act ? ((base + rank) | ((uint32_t)own << 16)) : 0xffffffffu;
    }
    __syncthreads();
    if (warp == 0) {                            // [slice][owner] counts -> offsets; owner list starts
      uint32_t tot = 0;
      if (lane < kWNW) {
#pragma unroll
        for (int w = 0; w < kWNW; ++w) {
          const uint32_t c = sm.cnt[w * kWNW + lane];
          sm.cnt[w * kWNW + lane] = tot;
          tot += c;
        }
      }
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (lane <= kWNW) sm.lbeg[lane] = x - tot;  // exclusive; lbeg[16] = total
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kWEPT; ++r) {
      if (pos[r] != 0xffffffffu) {
        const int own = (int)(pos[r] >> 16);
        sm.lst[sm.lbeg[own] + sm.cnt[warp * kWNW + own] + (pos[r] & 0xffffu)] = ev[r];
      }
    }
    __syncthreads();
    // ---- walk: this warp's events, window by window, no block barriers
    if (!wdone) {
      const int le = (int)sm.lbeg[warp + 1];
      int e0 = (int)sm.lbeg[warp];
      while (true) {
        const int e1 = e0 + upper_bound_rel<kWSB>(sm.lst + e0, le - e0, trel32, tj, lane);
        if (e1 > e0) {
          if (++gen == 0xffffu) {               // generation tags exhausted: clear this warp's claims
            for (int i = lane; i < whi - wlo; i += 32) sm.head[wlo + i] = 0u;
            __syncwarp();
            gen = 1;
          }
          warp_segment<BM>(sm, e0, e1, gen, warp, lane, trel32, kc);
        }
        if (e1 == le) break;                    // window j may continue in the next sub-batch
        if (j >= f_hi) { wdone = true; break; } // later events stay pending
        warp_readout<BM>(a, sm, j, trel, px0, wlo, whi, lane, kc);
        ++j;
        tj = (j < f_hi) ? (int32_t)(a.tf[j] - trel) : tcap;
        e0 = e1;
      }
    }
  }
  cp_async_wait_all();
  // ---- frames after this warp's last event
  while (j < f_hi) {
    warp_readout<BM>(a, sm, j, trel, px0, wlo, whi, lane, kc);
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += kWNT) {
      a.S[px0 + i] = sm.S[i];
      const float tr = sm.T[i];
      if (tr != t_clamp) a.T[px0 + i] = trel + (int64_t)tr;
    }
  }
}

template <int BM>
cudaError_t launch_warp_b(const IntArgs& a, cudaStream_t s) {
  const size_t smem = warp_smem_bytes(a.band_px, a.n_tiles);
  static size_t configured = 0;
  if (smem > configured) {
    const size_t mx = warp_smem_bytes(kMaxBandPx, kMaxTilesPerChunk);
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_warp_kernel<BM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return e;
    configured = mx;
  }
  esi_integrate_warp_kernel<BM><<<a.nb, kWNT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_integrate_warp(const IntArgs& a, cudaStream_t s) {
  return a.dp.bmode == 2 ? launch_warp_b<2>(a, s) : launch_warp_b<0>(a, s);
}

}  // namespace esi
