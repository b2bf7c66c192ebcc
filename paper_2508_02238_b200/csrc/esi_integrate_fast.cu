// esi_integrate_fast.cu -- K2: per-band integration (Alg. 2) fused
// with the Eq. 13/14 readout of every frame of the chunk.
//
// One CTA of 8 warps per band (K1's partition key): the sensor's 64-pixel groups
// are dealt round-robin to the bands (esi_internal.cuh, band_gpix), band_px slots
// each, the band count chosen so that the grid is exactly kK2Ctas resident CTAs per
// SM (or, contiguous layout, to runs of band_px consecutive ids).  The band's state lives in shared memory for the whole
// chunk: S (fp32) and T as an fp32 offset from the chunk base ChunkInfo::trel
// (exact integers: |T| < 2^24 us; pixels older than the decay horizon are
// clamped to -(dt_cut+1), i.e. "fully decayed").
//
// Per sub-batch of kSB band events (arrival order):
//   1. gather: cp.async copies of the band's (tile, band) segments written by
//      K1, in tile order = arrival order (double-buffered);
//   2. segments = the events of one frame window inside the sub-batch; per
//      segment: claim (atomicExch chains), apply (sparse / chain / dense
//      paths, see process_segment), and at the window end the fused Eq. 13 +
//      Eq. 14 readout of frame j for the band (packed f32x2 arithmetic,
//      4-byte streaming stores).
// Decay (Eq. 4, reading A14): with tau = 1e6/k us split as tau_h + tau_l,
//   u = k_us * ((tau_h - dt) + tau_l),  d = max(u, 0)^b
// (tau_h - dt is exact near the cutoff, so u keeps full relative precision and
// u <= 0 exactly when dt >= dt_cut = ceil(tau)).
#include <atomic>
#include "esi_device.cuh"

namespace esi {

namespace {

#include "esi_fast_common.cuh"

#ifndef ESI_K2_WARPS
#define ESI_K2_WARPS 8
#endif
constexpr int kNW = ESI_K2_WARPS;             // warps per CTA
constexpr int kNT = kNW * 32;                 // threads per CTA
#ifndef ESI_K2_SB
#define ESI_K2_SB (kK2Ctas >= 4 ? 1024 : 1536)
#endif
constexpr int kEPT = ESI_K2_SB / kNT;          // events per thread per segment (smem budget)
constexpr int kSB = kNT * kEPT;               // events per sub-batch
constexpr int kStage = (kEPT * 32 + 1) / 2 > 64 ? (kEPT * 32 + 1) / 2 : 64;   // uint2 per warp: kEPT * 32 chain heads (u32), >= 64 for the dense compaction
constexpr int kWinCap = 32;                   // window ends listed per pass (warp 0, per sub-batch)

// Shared memory of one CTA, carved at run time (the band size is a run-time
// multiple of 64 pixels chosen to balance the grid over the SMs).
struct FastSmem {
  float* S;                                   // [bp] accumulation (fp32)
  float* T;                                   // [bp] last time, relative to trel (exact integers)
  uint32_t* head;                             // [bp] last claimer | generation << 16
  uint16_t* next;                             // [kSB] previous claimer (claim-order chain)
  uint2* sub[2];                              // [kSB] gathered sub-batches (double buffer), arrival order
  uint2* stage;                               // [kNW][kStage] per-warp scratch: chain heads / dense compaction
  uint16_t* dq;                               // [kSB / 4] dense pixels of the segment
  uint32_t* nd;
  int32_t* wend;                              // [kWinCap] window ends inside the current sub-batch
  int32_t* wtj;                               // [kWinCap] frame time of each listed window (rel. to trel)
  uint32_t* pre;                              // [n_tiles + 1] band events before tile t
  uint16_t* mo;                               // [n_tiles] offset of the band's run inside tile t
};

__host__ __device__ inline size_t fast_smem_bytes(int bp, int n_tiles) {
  const size_t b = (size_t)bp;
  return b * 12 + kSB * 2 + 2 * kSB * 8 + kNW * kStage * 8 + (kSB / 4) * 2 + 16 + 2 * kWinCap * 4 +
         (size_t)(n_tiles + 1) * 4 + (((size_t)n_tiles * 2 + 15) & ~(size_t)15) + 64;
}

__device__ __forceinline__ FastSmem carve(unsigned char* base, int bp, int n_tiles) {
  FastSmem m;
  unsigned char* q = base;
  m.sub[0] = reinterpret_cast<uint2*>(q); q += kSB * 8;
  m.sub[1] = reinterpret_cast<uint2*>(q); q += kSB * 8;
  m.stage = reinterpret_cast<uint2*>(q); q += kNW * kStage * 8;
  m.S = reinterpret_cast<float*>(q); q += (size_t)bp * 4;
  m.T = reinterpret_cast<float*>(q); q += (size_t)bp * 4;
  m.head = reinterpret_cast<uint32_t*>(q); q += (size_t)bp * 4;
  m.pre = reinterpret_cast<uint32_t*>(q); q += (size_t)(n_tiles + 1) * 4;
  m.mo = reinterpret_cast<uint16_t*>(q); q += ((size_t)n_tiles * 2 + 15) & ~(size_t)15;
  m.nd = reinterpret_cast<uint32_t*>(q); q += 16;
  m.wend = reinterpret_cast<int32_t*>(q); q += kWinCap * 4;
  m.wtj = reinterpret_cast<int32_t*>(q); q += kWinCap * 4;
  m.next = reinterpret_cast<uint16_t*>(q); q += kSB * 2;
  m.dq = reinterpret_cast<uint16_t*>(q);
  return m;
}



// Frame j for the band: 4 pixels per thread-iteration (quads), Eq. 4 + Eq. 13 +
// Eq. 14 with packed f32x2 arithmetic, one 4-byte streaming store per quad.
template <int BM, bool IL>
__device__ __forceinline__ void fast_readout(const IntArgs& a, const FastSmem sm, int j, int32_t tji,
                                             int band, int npx, uint32_t qoff, const FastConst& c,
                                             bool tail_only = false) {   // tail_only: fold_readout wrote the full quads
  const float tj = (float)tji;
  const float aj = (float)(tji - (int32_t)c.tau_h);          // t_j - tau (folded mode: tau integer)
  // local pixel i -> frame[band_gpix(bm, band, i)]; contiguous layout (!IL): frame[band * band_px + i],
  // qoff = band * band_px
  uint8_t* frame = a.out + (int64_t)j * a.P + (IL ? 0u : qoff);
  const int nq = (npx + 3) >> 2;
  const bool vec = a.vec8 != 0;
  if (c.fold) {                                              // hot path: constants hoisted out of the loop
    const float2 naj = make_float2(-aj, -aj);
    const float2 sw2 = make_float2(c.scale_w2, c.scale_w2), off = make_float2(c.off_frac, c.off_frac);
    const float2 mo = make_float2(c.magic_off, c.magic_off);
    const float4* S4 = reinterpret_cast<const float4*>(sm.S);
    const float4* T4 = reinterpret_cast<const float4*>(sm.T);
    auto quad = [&](int q) -> uint32_t {
      const float4 s0 = S4[q], t0 = T4[q];
      float2 w0 = __fadd2_rn(make_float2(t0.x, t0.y), naj), w1 = __fadd2_rn(make_float2(t0.z, t0.w), naj);
      w0.x = fmaxf(w0.x, 0.f); w0.y = fmaxf(w0.y, 0.f); w1.x = fmaxf(w1.x, 0.f); w1.y = fmaxf(w1.y, 0.f);
      const float2 v0 = __fmul2_rn(make_float2(s0.x, s0.y), __fmul2_rn(w0, w0));
      const float2 v1 = __fmul2_rn(make_float2(s0.z, s0.w), __fmul2_rn(w1, w1));
      const float2 r0 = __fadd2_rd(__ffma2_rn(v0, sw2, off), mo), r1 = __fadd2_rd(__ffma2_rn(v1, sw2, off), mo);
      return __byte_perm(__byte_perm(__float_as_uint(r0.x), __float_as_uint(r0.y), 0x0040),
                         __byte_perm(__float_as_uint(r1.x), __float_as_uint(r1.y), 0x0040), 0x5410);
    };
    // full quads: one 4-byte streaming store each (__stcs: no memory clobber, so the
    // next quad's shared loads can be issued ahead); the remainder quads fall on the
    // last warp (warp 0 also lists the windows)
    // a thread's quads q, q + kNT, ... are the same quad of 64-pixel groups kNT / 16 apart:
    // a constant stride of kNT * gs words in the frame, from the thread's first quad at
    // byte qoff (computed once per kernel)
    static_assert(kNT % (kGroup / 4) == 0, "quads of one thread must keep their place in the group");
    const int nfull = vec ? (npx >> 2) : 0;
    if (tail_only) {
    } else if (IL) {
      unsigned int* f4 = reinterpret_cast<unsigned int*>(frame + qoff);
      const uint32_t fstride = (uint32_t)kNT * (uint32_t)a.bm.gs;
#pragma unroll 2
      for (int q = kNT - 1 - (int)threadIdx.x; q < nfull; q += kNT, f4 += fstride) __stcs(f4, quad(q));
    } else {                                                       // contiguous: compile-time stride
      unsigned int* f4 = reinterpret_cast<unsigned int*>(frame);
#pragma unroll 2
      for (int q = kNT - 1 - (int)threadIdx.x; q < nfull; q += kNT) __stcs(f4 + q, quad(q));
    }
    for (int q = nfull + (int)threadIdx.x; q < nq; q += kNT) {     // ragged tail / unaligned output
      const uint32_t v = quad(q);
      const int base = q * 4, n = min(4, npx - base);
      uint8_t* dst = frame + (IL ? band_gpix(a.bm, band, base) : (int64_t)base);   // a quad never straddles a group
      for (int u = 0; u < n; ++u) dst[u] = (uint8_t)((v >> (8 * u)) & 0xffu);
    }
    return;
  }
  for (int q = threadIdx.x; q < nq; q += kNT) {
    const int base = q * 4;
    const float4 s0 = *reinterpret_cast<const float4*>(&sm.S[base]);
    const float4 t0 = *reinterpret_cast<const float4*>(&sm.T[base]);
    const uint32_t b01 = readout2<BM>(make_float2(s0.x, s0.y), make_float2(t0.x, t0.y), tj, aj, c, a.mp.smin, a.mp.smax);
    const uint32_t b23 = readout2<BM>(make_float2(s0.z, s0.w), make_float2(t0.z, t0.w), tj, aj, c, a.mp.smin, a.mp.smax);
    const uint32_t v = __byte_perm(b01, b23, 0x5410);
    uint8_t* dst = frame + (IL ? band_gpix(a.bm, band, base) : (int64_t)base);   // a quad never straddles a group
    if (vec && base + 4 <= npx) {
      st_stream4(dst, v);
    } else {
      const int n = min(4, npx - base);
      for (int u = 0; u < n; ++u) dst[u] = (uint8_t)((v >> (8 * u)) & 0xffu);
    }
  }
}


// Per-thread readout state of the folded mode, fixed for the whole chunk and pinned in
// registers (the compiler otherwise rebuilds the shared-memory bases, the frame pointer and the
// quad count from ctaid / tid / kernel arguments in every call: ~25 of a call's ~80 instructions).
struct RoState {
  uint32_t sS;        // shared address of the thread's first S quad (its T quad: + 4 * band_px)
  uint8_t* fptr;      // the thread's first quad in the next frame to be written (advances by P)
  int nmy;            // full quads of this thread (q0, q0 + kNT, ...) | kRagged if the band also has a
                      // partial last quad or the output is unaligned (byte-store tail, rare)
};
constexpr int kRagged = 0x100;

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}

// Frame j of the band in the folded mode (b = 2, readout decay, integer tau, bounds containing
// 0; fast_readout's hot path): x = S max(T - (t_j - tau), 0)^2 (k^2 scale) + off, Eq. 14 by the
// round-down magic add.  Two quads per iteration, loads first.  FSTRIDE: bytes between a
// thread's consecutive quads in the frame (contiguous layout: compile-time 4 * kNT).
template <bool IL>
__device__ __forceinline__ void fold_readout(const IntArgs& a, RoState& ro, int32_t tji, uint32_t t_off,
                                             uint32_t fstride_il, const FastConst& c) {
  const float najs = -(float)(tji - c.tau_i);                    // -(t_j - tau), exact
  const float2 naj = make_float2(najs, najs);
  const float2 sw2 = make_float2(c.scale_w2, c.scale_w2), off = make_float2(c.off_frac, c.off_frac);
  const float2 mo = make_float2(c.magic_off, c.magic_off);
  auto quad = [&](const float4 s0, const float4 t0) -> uint32_t {
    float2 w0 = __fadd2_rn(make_float2(t0.x, t0.y), naj), w1 = __fadd2_rn(make_float2(t0.z, t0.w), naj);
    w0.x = fmaxf(w0.x, 0.f); w0.y = fmaxf(w0.y, 0.f); w1.x = fmaxf(w1.x, 0.f); w1.y = fmaxf(w1.y, 0.f);
    const float2 v0 = __fmul2_rn(make_float2(s0.x, s0.y), __fmul2_rn(w0, w0));
    const float2 v1 = __fmul2_rn(make_float2(s0.z, s0.w), __fmul2_rn(w1, w1));
    const float2 r0 = __fadd2_rd(__ffma2_rn(v0, sw2, off), mo), r1 = __fadd2_rd(__ffma2_rn(v1, sw2, off), mo);
    return __byte_perm(__byte_perm(__float_as_uint(r0.x), __float_as_uint(r0.y), 0x0040),
                       __byte_perm(__float_as_uint(r1.x), __float_as_uint(r1.y), 0x0040), 0x5410);
  };
  const uint32_t fstride = IL ? fstride_il : (uint32_t)(4 * kNT);
  uint32_t sa = ro.sS;
  uint8_t* f = ro.fptr;
  int r = 0;
  const int nmy = ro.nmy & (kRagged - 1);
  for (; r + 2 <= nmy; r += 2) {
    const float4 s0 = lds128(sa), t0 = lds128(sa + t_off);
    const float4 s1 = lds128(sa + kNT * 16), t1 = lds128(sa + t_off + kNT * 16);
    __stcs(reinterpret_cast<unsigned int*>(f), quad(s0, t0));
    __stcs(reinterpret_cast<unsigned int*>(f + fstride), quad(s1, t1));
    sa += 2 * kNT * 16;
    f += 2 * (size_t)fstride;
  }
  if (r < nmy) {
    const float4 s0 = lds128(sa), t0 = lds128(sa + t_off);
    __stcs(reinterpret_cast<unsigned int*>(f), quad(s0, t0));
  }
  ro.fptr += a.P;
}

// Per-event processing of one segment (the events of one frame window inside
// one sub-batch), block-wide.  Each event claims its pixel with an atomic
// exchange on head[px] (tagged with the segment's generation, so the table
// never needs clearing), which links the pixel's events into a chain in claim
// order.  The last claimer owns the pixel for the segment: a pixel hit once is
// updated directly (sparse path); chains of 2..kSlots events are collected per
// warp and applied one chain per lane after a sorting network restores arrival
// order; more go to a warp (dense path).  The first two paths are bit-identical
// to a sequential fp32 evaluation.  Two barriers: claims complete before
// ownership is read; updates complete before anyone reads the state (readout)
// or re-claims.
template <int BM>
__device__ __forceinline__ void process_segment(const FastSmem sm, const uint2* sub, int e0, int e1, uint32_t trel,
                                                uint32_t gen, int warp, int lane, const FastConst& k, int a_bp) {
  const int tid = threadIdx.x;
  const uint32_t tag = gen << 16;
  uint2 evr[kEPT];                                        // this thread's events, kept from claim to apply
  uint32_t linked = 0;                                    // bit r: event r had a predecessor claim (= next != kEmpty)
#pragma unroll
  for (int r = 0; r < kEPT; ++r) {                        // claim
    if (e0 + r * kNT >= e1) break;                        // uniform: no thread has an event in this round
    const int i = e0 + tid + r * kNT;
    if (i < e1) {
      evr[r] = sub[i];
      const int px = (int)(evr[r].y & 0x7fffffffu);
      ESI_DCHECK(px < a_bp && i - e0 < kSB);
      const uint32_t old = atomicExch(&sm.head[px], tag | (uint32_t)(i - e0));
      const bool prev = (old & 0xffff0000u) == tag;
      sm.next[i - e0] = prev ? (uint16_t)old : (uint16_t)kEmpty;
      linked |= prev ? (1u << r) : 0u;
    }
  }
  __syncthreads();
  uint32_t* wl = reinterpret_cast<uint32_t*>(sm.stage + warp * kStage);   // <= kEPT * 32 chain heads
  int nch = 0;
#pragma unroll
  for (int r = 0; r < kEPT; ++r) {                        // apply: singles now, chains deferred
    if (e0 + r * kNT >= e1) break;                        // uniform: no thread has an event in this round
    const int i = e0 + tid + r * kNT;
    bool chain = false;
    const uint32_t me = (uint32_t)(i - e0);
    if (i < e1) {
      const int px = (int)(evr[r].y & 0x7fffffffu);
      if (sm.head[px] == (tag | me)) {
        if (!((linked >> r) & 1u)) apply_event<BM>(sm.S, sm.T, px, evr[r], trel, k);   // own claim: no reload of next
        else chain = true;
      }
    }
    const unsigned bc = __ballot_sync(kFull, chain);
    if (chain) wl[nch + __popc(bc & lanemask_lt())] = me;
    nch += __popc(bc);
  }
  __syncwarp();
  for (int cb = 0; cb < nch; cb += 32) {                  // chains: one per lane
    if (cb + lane >= nch) break;
    const uint32_t me = wl[cb + lane];
    const int px = (int)(sub[e0 + me].y & 0x7fffffffu);
    ESI_DCHECK(me < (uint32_t)(e1 - e0) && px < a_bp);
    uint32_t id[kSlots];
    id[0] = me;
    int c = 1;
#pragma unroll
    for (int q = 1; q < kSlots; ++q) {
      const uint32_t n = (c == q) ? sm.next[id[q - 1]] : kEmpty;
      id[q] = n;
      c += (n != kEmpty) ? 1 : 0;
    }
    if (c == kSlots && sm.next[id[kSlots - 1]] != kEmpty) {   // > kSlots events: dense path
      const uint32_t slot = atomicAdd(sm.nd, 1u);
      ESI_DCHECK(slot < (uint32_t)(kSB / 4));
      sm.dq[slot] = (uint16_t)px;
      continue;
    }
    // claim order -> arrival order (kEmpty = 0xffff sorts after every index)
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
      const uint2 e = sub[e0 + iq];
      const float te = (float)(int32_t)(e.x - trel);
      const float pc = ((int32_t)e.y < 0) ? -k.C : k.C;
      s = clampS(ev_update<BM>(s, pc, ev_decay<BM>(te - t, k)), k);   // Alg. 2 body
      t = te;
    }
    sm.S[px] = s;
    sm.T[px] = t;
  }
  __syncthreads();
  const uint32_t nd = *sm.nd;
  if (nd > 0) {
    for (uint32_t d = warp; d < nd; d += kNW)
      dense_pixel_apply<BM>(sm.S, sm.T, sub, sm.stage + warp * kStage, e0, e1, sm.dq[d], trel, lane, k);
    __syncthreads();
    if (tid == 0) *sm.nd = 0;
  }
}


// register budget: as for ESI_K2_MINB CTAs per SM (default: the resident count the
// bands are sized for); a larger value leaves registers for a co-resident K1 CTA
#ifndef ESI_K2_MINB
#define ESI_K2_MINB kK2Ctas
#endif
template <int BM, bool IL>   // IL: interleaved band layout (run-time frame stride); else contiguous bands
__global__ void __launch_bounds__(kNT, ESI_K2_MINB) esi_integrate_kernel(IntArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_wsum[32];
  const int band = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bp = a.band_px;
  const int npx = band_npx(a.bm, band, a.P);                 // valid local pixels: a prefix of the bp slots
  const int n_tiles = a.n_tiles;
  const FastSmem sm = carve(smem_raw, bp, n_tiles);

  if (a.gate && *a.gate != kNoError) return;   // lazy validation found an invalid event: write nothing
  const ChunkInfo ci = *a.info;
  if (a.kind_gate == 1 && !ci.fast) return;    // the general kernel renders this chunk
  const int f_lo = ci.f_lo, f_hi = ci.f_hi;
  const bool active = ci.active != 0;
  if (!active && f_lo >= f_hi) return;
  const int64_t trel = ci.trel;
  const uint32_t trel32 = (uint32_t)trel;
  const float t_clamp = -(float)(a.dp.dt_cut + 1);
  const int32_t tcap = (int32_t)min(a.t_cap - trel, (int64_t)(1 << 25));
  const FastConst kc = make_const(a);
  // byte of the thread's first readout quad in a frame (P <= 2^22: 32-bit); contiguous layout:
  // the band's first pixel id
  uint32_t qoff = (uint32_t)band * (uint32_t)bp;
  const uint32_t q0 = (uint32_t)(kNT - 1 - (int)threadIdx.x);
  if (IL)
    qoff = (((q0 >> (kGroupShift - 2)) * (uint32_t)a.bm.gs + (uint32_t)band * (uint32_t)a.bm.bs) << kGroupShift) |
           ((q0 << 2) & (uint32_t)(kGroup - 1));
  // folded readout: per-thread state for the whole chunk, pinned in registers by the empty asm
  RoState ro;
  const int nfull = a.vec8 ? (npx >> 2) : 0;
  const bool ragged = nfull != ((npx + 3) >> 2);              // partial last quad, or an unaligned output
  ro.nmy = (nfull > (int)q0 ? (nfull - (int)q0 + kNT - 1) / kNT : 0) | (ragged ? kRagged : 0);
  ro.sS = (uint32_t)__cvta_generic_to_shared(sm.S) + q0 * 16u;
  ro.fptr = a.out + (int64_t)f_lo * a.P + (IL ? qoff : qoff + q0 * 4u);
  asm volatile("" : "+r"(ro.sS), "+l"(ro.fptr), "+r"(ro.nmy));
  const uint32_t t_off = (uint32_t)bp * 4u;                   // T follows S in shared memory (carve)
  const uint32_t fstride_il = 4u * (uint32_t)kNT * (uint32_t)a.bm.gs;
  auto readout = [&](int jj, int32_t tji) {
    if (kc.fold) {
      fold_readout<IL>(a, ro, tji, t_off, fstride_il, kc);
      if (ro.nmy >= kRagged) fast_readout<BM, IL>(a, sm, jj, tji, band, npx, qoff, kc, true);
    } else {
      fast_readout<BM, IL>(a, sm, jj, tji, band, npx, qoff, kc);
    }
  };
  for (int i = threadIdx.x; i < bp; i += kNT) {
    const bool in = i < npx;
    const int64_t g = band_gpix(a.bm, band, i);
    sm.S[i] = in ? a.S[g] : 0.f;
    sm.T[i] = in ? (float)max(a.T[g] - trel, (int64_t)t_clamp) : t_clamp;
    sm.head[i] = 0u;                          // generation 0: never a live claim
  }
  if (threadIdx.x == 0) *sm.nd = 0;
  const int n_b = active ? band_run_prefix<kNW>(a.meta + (int64_t)band * n_tiles, n_tiles, sm.pre, sm.mo, s_wsum) : 0;
  if (a.bstats && active && threadIdx.x == 0) {   // ESI_BANDS_AUTO: this band's share of the chunk
    atomicMax(a.bstats, (unsigned long long)n_b);
    atomicAdd(a.bstats + 1, (unsigned long long)n_b);
    atomicAdd(a.bstats + 2, 1ull);
  }
  __syncthreads();

  int j = f_lo;
  bool done = false;
  uint32_t gen = 0;
  // ---- 1. gather sub-batch k into sub[k & 1]; sub-batch k+1 is in flight while k is integrated
  if (n_b > 0) gather_sub<kSB>(a.rec, sm.pre, sm.mo, n_tiles, n_b, 0, sm.sub[0], warp, kNW, lane);
  for (int sb0 = 0, kb = 0; sb0 < n_b && !done; sb0 += kSB, ++kb) {
    const int n_sb = min(kSB, n_b - sb0);
    const uint2* sub = (kb & 1) ? sm.sub[1] : sm.sub[0];   // no dynamic index into sm (keeps it in registers)
    cp_async_wait_all();
    __syncthreads();
    // warp 0 lists the first windows meanwhile (the other warps wait for that list)
    if (sb0 + kSB < n_b && warp > 0)
      gather_sub<kSB>(a.rec, sm.pre, sm.mo, n_tiles, n_b, sb0 + kSB, (kb & 1) ? sm.sub[0] : sm.sub[1], warp - 1, kNW - 1,
                 lane);
    // ---- 2. segments = frame windows inside the sub-batch; readout at each window end.
    // Window ends (events of the sub-batch with t <= t_j) are listed by warp 0,
    // kWinCap at a time, behind one barrier, instead of being searched by every warp.
    int e0 = 0;
    bool more = true;
    while (more) {
      more = false;
      if (warp == 0) {                          // window w ends frame j + w at time wtj[w]
        // lane l lists window l: frame j + l, its end = upper bound of t_{j+l} in
        // [e0, n_sb) (the sub-batch is time-sorted); the list stops at the first
        // window that reaches the sub-batch end or the last frame
        const int jj = j + lane;
        const int32_t tw = (jj < f_hi) ? (int32_t)(a.tf[jj] - trel) : tcap;
        int base = e0, len = n_sb - e0;
        while (len > 0) {
          const int half = len >> 1;
          if ((int32_t)(sub[base + half].x - trel32) <= tw) {
            base += half + 1;
            len -= half + 1;
          } else {
            len = half;
          }
        }
        const bool stop = base == n_sb || jj >= f_hi || lane == kWinCap - 2;
        const int last = __ffs(__ballot_sync(kFull, stop)) - 1;   // lane kWinCap - 2 always stops
        if (lane <= last) {
          sm.wend[lane] = base;
          sm.wtj[lane] = tw;
        }
        if (lane == 0) sm.wend[kWinCap - 1] = last + 1;   // count in the last slot
      }
      __syncthreads();
      const int nwin = sm.wend[kWinCap - 1];
      for (int w = 0; w < nwin; ++w) {
        const int e1 = sm.wend[w];
        if (e1 > e0) {
          if (++gen == 0xffffu) {               // generation tags exhausted: clear the claim table
            __syncthreads();
            for (int i = threadIdx.x; i < bp; i += kNT) sm.head[i] = 0u;
            __syncthreads();
            gen = 1;
          }
          process_segment<BM>(sm, sub, e0, e1, trel32, gen, warp, lane, kc, npx);
        }
        if (e1 == n_sb) break;                  // the window may continue in the next sub-batch
        if (j >= f_hi) { done = true; break; }  // later events stay pending
        readout(j, sm.wtj[w]);
        ++j;
        e0 = e1;
        more = (w == nwin - 1);                 // every listed window closed: list the next ones
      }
      if (more) __syncthreads();                // wend is rewritten by warp 0
    }
  }
  cp_async_wait_all();
  // ---- 3. frames after the chunk's last event
  while (j < f_hi) {
    readout(j, (int32_t)(a.tf[j] - trel));
    ++j;
  }
  if (n_b > 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < npx; i += kNT) {
      const int64_t g = band_gpix(a.bm, band, i);
      a.S[g] = sm.S[i];
      const float tr = sm.T[i];
      if (tr != t_clamp) a.T[g] = trel + (int64_t)tr;
    }
  }
}

template <int BM, bool IL>
cudaError_t launch_fast_l(const IntArgs& a, cudaStream_t s) {
  const size_t smem = fast_smem_bytes(a.band_px, a.n_tiles);
  int dev = 0;
  cudaGetDevice(&dev);
  static std::atomic<int> configured[64];   // zero-initialised; set-once flags (idempotent, race-free)   // per device (the attribute is per context)
  if (dev < 0 || dev >= 64 || !configured[dev].load(std::memory_order_relaxed)) {
    const size_t mx = fast_smem_bytes(kMaxBandPx, kMaxTilesPerChunk);
    cudaError_t e = cudaFuncSetAttribute(esi_integrate_kernel<BM, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)mx);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) configured[dev].store(1, std::memory_order_relaxed);
  }
  esi_integrate_kernel<BM, IL><<<a.nb, kNT, smem, s>>>(a);
  return cudaGetLastError();
}

template <int BM>
cudaError_t launch_fast_b(const IntArgs& a, cudaStream_t s) {
  return a.bm.interleave ? launch_fast_l<BM, true>(a, s) : launch_fast_l<BM, false>(a, s);
}

}  // namespace

size_t integrate_fast_smem_bytes(int band_px, int n_tiles) { return fast_smem_bytes(band_px, n_tiles); }

cudaError_t launch_integrate_fast(const IntArgs& a, cudaStream_t s) {
  if (a.dp.first)
    return a.dp.bmode == 2           ? launch_fast_b<2 + kFirst>(a, s)
           : a.dp.bmode == kDecayExp ? launch_fast_b<kDecayExp + kFirst>(a, s)
                                     : launch_fast_b<kFirst>(a, s);
  return a.dp.bmode == 2           ? launch_fast_b<2>(a, s)
         : a.dp.bmode == kDecayExp ? launch_fast_b<kDecayExp>(a, s)
                                   : launch_fast_b<0>(a, s);
}

}  // namespace esi
