// esi_device.cuh -- small device helpers shared by the libesi kernels.
#pragma once
#include <cstdint>
#include <cstdio>
#include "esi_internal.cuh"

namespace esi {

constexpr unsigned kFull = 0xffffffffu;

// Device-side invariant checks, compiled in only for the checked build
// (python -m paper_2508_02238_b200.build --checked -> libesi_checked.so); a failed
// check prints its location and traps (the render call then reports ESI_ERR_CUDA).
#ifdef ESI_DEBUG_CHECKS
#define ESI_DCHECK(c)                                                              \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("ESI_DCHECK failed: %s at %s:%d\n", #c, __FILE__, __LINE__);          \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define ESI_DCHECK(c) \
  do {                \
  } while (0)
#endif

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 16-byte streaming load (read once: evict-first in L1/L2).
__device__ __forceinline__ int4 ld_stream16(const int4* p) { return __ldcs(p); }

// 8-byte streaming store of frame bytes (st.global.cs; an intrinsic, not asm
// volatile with a memory clobber, so independent shared loads may move ahead).
__device__ __forceinline__ void st_stream8(void* p, uint32_t lo, uint32_t hi) {
  __stcs(reinterpret_cast<uint2*>(p), make_uint2(lo, hi));
}

// 4-byte streaming store of frame bytes.
__device__ __forceinline__ void st_stream4(void* p, uint32_t v) {
  __stcs(reinterpret_cast<unsigned int*>(p), v);
}

// Eq. 4: d(dt) = max{(1 - k dt)^b, 0}, dt in integer microseconds (>= 0).
// u = 1 - k dt is formed with a float pair (kh + kl = k * 1e-6) so that u keeps
// ~1 ulp relative accuracy near the cutoff (SURVEY 8(c) numerics); dt >= dt_cut
// (= ceil(1e6/k)) gives d = 0 exactly (reading A14).
__device__ __forceinline__ float esi_decay(int64_t dt, const DecayParams& dp) {
  if (dp.bmode == kDecayNone) return 1.f;   // Eq. 2
  if (dt >= dp.dt_cut) return 0.f;
  if (dp.bmode == kDecayExp) {       // exponential variant (A20): exp(-k dt)
    if (dp.use_f64) return (float)exp(-dp.k_us * (double)dt);
    const float f = (float)(int32_t)dt;
    return expf(-fmaf(f, dp.kh, f * dp.kl));
  }
  float u;
  if (dp.use_f64) {
    u = (float)(1.0 - dp.k_us * (double)dt);
  } else {
    const float f = (float)(int32_t)dt;  // exact: dt < dt_cut <= 2^24
    u = fmaf(-f, dp.kh, 1.0f);
    u = fmaf(-f, dp.kl, u);
  }
  u = fmaxf(u, 0.f);
  switch (dp.bmode) {
    case 1: return u;
    case 2: return u * u;
    case 3: return u * u * u;
    case 4: { const float u2 = u * u; return u2 * u2; }
    case kDecayExp: return 0.f;   // not reached: handled above
    default: return u > 0.f ? exp2f(dp.b * log2f(u)) : 0.f;
  }
}

// Eq. 13 + Eq. 14: clamp, then 255 (v - smin)/(smax - smin)
// rounded half away from zero (reading A8; q >= 0 here so floor(q + 0.5)),
// computed as off_int + floor(v*scale + off_frac).
__device__ __forceinline__ uint32_t esi_map8(float v, const MapParams& mp) {
  v = fminf(fmaxf(v, mp.smin), mp.smax);
  int q = mp.off_int + __float2int_rd(fmaf(v, mp.scale, mp.off_frac));
  q = min(max(q, 0), 255);
  return (uint32_t)q;
}

// number of entries of the sorted array a[0..n) that are < key
__device__ __forceinline__ int lower_bound_i64(const int64_t* a, int n, int64_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace esi
