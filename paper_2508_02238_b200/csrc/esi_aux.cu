// esi_aux.cu -- small kernels around the two main ones:
//   K4 esi_readout_kernel : frames straight from the global state (no events)
//   esi_plan_kernel       : how many chunks start at or before the last frame
//   esi_consume_kernel    : how many events of a segment were integrated
//   esi_validate_kernel   : eager validation for params.validate_on_push
#include <algorithm>
#include "esi_device.cuh"

namespace esi {

// One thread per (frame, group of 8 pixels); Eq. 14 readout of the stored state.
__global__ void __launch_bounds__(256) esi_readout_kernel(ReadoutArgs a) {
  const int64_t groups = (a.P + 7) / 8;
  const int64_t total = groups * a.F;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(g / groups);
    const int64_t px = (g - (int64_t)j * groups) * 8;
    const int64_t tj = a.tf[j];
    const int nq = (int)min((int64_t)8, a.P - px);
    uint32_t bytes[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float v = 0.f;
      if (q < nq) {
        v = a.S[px + q];
        if (a.mp.readout_decay) v *= esi_decay(tj - a.T[px + q], a.dp);
      }
      bytes[q] = esi_map8(v, a.mp);
    }
    uint8_t* dst = a.out + (int64_t)j * a.P + px;
    if (a.vec8 && nq == 8) {
      st_stream8(dst, bytes[0] | (bytes[1] << 8) | (bytes[2] << 16) | (bytes[3] << 24),
                 bytes[4] | (bytes[5] << 8) | (bytes[6] << 16) | (bytes[7] << 24));
    } else {
      for (int q = 0; q < nq; ++q) dst[q] = (uint8_t)bytes[q];
    }
  }
}

cudaError_t launch_readout(const ReadoutArgs& a, cudaStream_t s) {
  const int64_t total = ((a.P + 7) / 8) * a.F;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  esi_readout_kernel<<<(int)blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// facts of chunk c: its first event ev[0], last event ev[n - 1], and the first event time of
// the next chunk (has_next)
__device__ __forceinline__ ChunkInfo plan_chunk(const esi_event_t* ev, int64_t n, int c, bool has_next, int64_t t_next,
                                                const int64_t* tf, int F, int64_t t_cap, int allow_fast) {
  const int64_t t0 = ev[0].t_us;
  const int64_t t1 = ev[n - 1].t_us;
  ChunkInfo ci;
  ci.tbase = t0;
  ci.f_lo = c == 0 ? 0 : lower_bound_i64(tf, F, t0);
  ci.f_hi = has_next ? lower_bound_i64(tf, F, t_next) : F;
  ci.active = t0 <= t_cap;
  ci.wide = (t1 - t0) > (int64_t)0xFFFFFFFFLL;
  int64_t lo = t0, hi = t1;
  if (ci.f_lo < ci.f_hi) {
    lo = min(lo, tf[ci.f_lo]);
    hi = max(hi, tf[ci.f_hi - 1]);
  }
  ci.trel = lo;
  ci.fast = allow_fast && (hi - lo) < ((int64_t)1 << 24);   // fp32-exact relative times
  ci._pad = 0;
  return ci;
}

__global__ void esi_plan_kernel(const esi_event_t* const* chunk_first, const int64_t* chunk_n,
                                int n_chunks, const int64_t* tf, int F, int64_t t_cap, int allow_fast,
                                ChunkInfo* info, int32_t* n_active) {
  // chunk c renders the frames j with t_first(c) <= t_j < t_first(c+1) (chunk 0: t_j < t_first(1))
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n_chunks; c += gridDim.x * blockDim.x) {
    const bool has_next = c + 1 < n_chunks;
    const int64_t t_next = has_next ? chunk_first[c + 1]->t_us : 0;
    const ChunkInfo ci = plan_chunk(chunk_first[c], chunk_n[c], c, has_next, t_next, tf, F, t_cap, allow_fast);
    info[c] = ci;
    // first events are non-decreasing: the active chunks are a prefix
    const bool next_active = has_next && t_next <= t_cap;
    if (ci.active && !next_active) *n_active = c + 1;
    if (c == 0 && !ci.active) *n_active = 0;
  }
}

// Render of a single chunk whose plan the host does not read back (esi_runtime.cpp, "sync-free"):
// the chunk's facts from by-value arguments; also resets the render's error word and K1's
// work counters (instead of two memsets on the stream).
__global__ void esi_plan1_kernel(const esi_event_t* first, int64_t n, const int64_t* tf, int F, int64_t t_cap,
                                 int allow_fast, ChunkInfo* info, unsigned long long* err, uint32_t* tile_ctr) {
  info[0] = plan_chunk(first, n, 0, false, 0, tf, F, t_cap, allow_fast);
  *err = kNoError;
  tile_ctr[0] = tile_ctr[1] = tile_ctr[2] = tile_ctr[3] = 0u;
}

cudaError_t launch_plan1(const esi_event_t* first, int64_t n, const int64_t* tf, int F, int64_t t_cap, int allow_fast,
                         ChunkInfo* info, unsigned long long* err, uint32_t* tile_ctr, cudaStream_t s) {
  esi_plan1_kernel<<<1, 1, 0, s>>>(first, n, tf, F, t_cap, allow_fast, info, err, tile_ctr);
  return cudaGetLastError();
}

cudaError_t launch_plan(const esi_event_t* const* chunk_first, const int64_t* chunk_n, int n_chunks,
                        const int64_t* tf, int F, int64_t t_cap, int allow_fast, ChunkInfo* info,
                        int32_t* n_active, cudaStream_t s) {
  const int threads = 128;
  const int blocks = (n_chunks + threads - 1) / threads;
  esi_plan_kernel<<<blocks, threads, 0, s>>>(chunk_first, chunk_n, n_chunks, tf, F, t_cap, allow_fast, info,
                                             n_active);
  return cudaGetLastError();
}

__global__ void esi_consume_kernel(const esi_event_t* seg, int64_t n, int64_t t_cap, int64_t* count,
                                   int64_t* last_t) {
  int64_t lo = 0, hi = n;  // number of events with t <= t_cap
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (seg[mid].t_us <= t_cap) lo = mid + 1; else hi = mid;
  }
  *count = lo;
  if (lo > 0) *last_t = seg[lo - 1].t_us;
}

cudaError_t launch_consume(const esi_event_t* seg, int64_t n, int64_t t_cap, int64_t* count,
                           int64_t* last_t, cudaStream_t s) {
  esi_consume_kernel<<<1, 1, 0, s>>>(seg, n, t_cap, count, last_t);
  return cudaGetLastError();
}

// consume of the sync-free one-chunk render: res[0] = events consumed, res[1] = the render's
// error word, res[2] = the plan's kernel choice (one read-back instead of three)
__global__ void esi_finish1_kernel(const esi_event_t* seg, int64_t n, int64_t t_cap, int64_t* res, int64_t* last_t,
                                   const unsigned long long* err, const ChunkInfo* info) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (seg[mid].t_us <= t_cap) lo = mid + 1; else hi = mid;
  }
  res[0] = lo;
  if (lo > 0) *last_t = seg[lo - 1].t_us;
  res[1] = (int64_t)*err;
  res[2] = info->fast;
}

cudaError_t launch_finish1(const esi_event_t* seg, int64_t n, int64_t t_cap, int64_t* res, int64_t* last_t,
                           const unsigned long long* err, const ChunkInfo* info, cudaStream_t s) {
  esi_finish1_kernel<<<1, 1, 0, s>>>(seg, n, t_cap, res, last_t, err, info);
  return cudaGetLastError();
}

// Eager validation of one push (reading A15), K0.  Each warp owns
// a contiguous range of the batch and walks it in steps of 32 x kVU events:
// lane l loads events step + l + 32 u (kVU coalesced 16-byte streaming loads in
// flight per lane), the predecessor's t comes from the neighbouring lane by
// shuffle and, for lane 0, from lane 31 of the previous row -- carried across
// steps, so only a warp's first event needs a global load of its predecessor.
constexpr int kVU = 8;

__device__ __forceinline__ void report_bad(int64_t i, uint32_t x, uint32_t y, int p, int32_t W, int32_t H,
                                           unsigned long long* err) {
  int code;
  if (x >= (uint32_t)W || y >= (uint32_t)H) code = ESI_ERR_OUT_OF_BOUNDS;
  else if (p != 1 && p != -1) code = ESI_ERR_BAD_POLARITY;
  else code = ESI_ERR_NEGATIVE_INTERVAL;
  atomicMin(err, ((unsigned long long)i << 8) | (unsigned)code);
}

__global__ void __launch_bounds__(256) esi_validate_kernel(const esi_event_t* ev, int64_t n, const int64_t* prev_t,
                                                           int64_t t_min, int32_t W, int32_t H,
                                                           unsigned long long* err) {
  const int4* evv = reinterpret_cast<const int4*>(ev);
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  constexpr int64_t kStep = 32 * kVU;
  const int64_t steps = (n + kStep - 1) / kStep;
  const int64_t s0 = steps * wid / n_warps, s1 = steps * (wid + 1) / n_warps;   // this warp's steps
  if (s0 >= s1) return;
  int64_t carry = 0;                                     // t of the event before this warp's range
  if (lane == 0) carry = s0 > 0 ? __ldg(&ev[s0 * kStep - 1].t_us) : *prev_t;
  for (int64_t st = s0; st < s1; ++st) {
    const int64_t base = st * kStep;
    int4 r[kVU];
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const int64_t i = base + u * 32 + lane;
      r[u] = i < n ? ld_stream16(evv + i) : make_int4(0, 0, 0, 0);
    }
    bool any_bad = false;
#pragma unroll
    for (int u = 0; u < kVU; ++u) {
      const int64_t i = base + u * 32 + lane;
      const int64_t t = (int64_t)(((uint64_t)(uint32_t)r[u].y << 32) | (uint32_t)r[u].x);
      int64_t tp = __shfl_up_sync(kFull, t, 1);
      const int64_t last = __shfl_sync(kFull, t, 31);
      if (lane == 0) tp = carry;
      carry = last;                                      // lane 0's predecessor in the next row
      const uint32_t x = (uint32_t)r[u].z & 0xffffu, y = (uint32_t)r[u].z >> 16;
      const int p = (int)(int8_t)(r[u].w & 0xff);
      const bool bad = (i < n) & ((x >= (uint32_t)W) | (y >= (uint32_t)H) | (p * p != 1) | (t < t_min) | (t < tp));
      any_bad |= bad;
    }
    if (__any_sync(kFull, any_bad)) {                    // rare: find and report the offending events
#pragma unroll
      for (int u = 0; u < kVU; ++u) {
        const int64_t i = base + u * 32 + lane;
        const int64_t t = (int64_t)(((uint64_t)(uint32_t)r[u].y << 32) | (uint32_t)r[u].x);
        const int64_t tp = i == 0 ? *prev_t : __ldg(&ev[i - 1].t_us);
        const uint32_t x = (uint32_t)r[u].z & 0xffffu, y = (uint32_t)r[u].z >> 16;
        const int p = (int)(int8_t)(r[u].w & 0xff);
        if ((i < n) && ((x >= (uint32_t)W) | (y >= (uint32_t)H) | (p * p != 1) | (t < t_min) | (t < tp)))
          report_bad(i, x, y, p, W, H, err);
      }
    }
  }
}

cudaError_t launch_validate(const esi_event_t* ev, int64_t n, const int64_t* prev_t,
                            int64_t t_origin, int64_t last_frame_t, int32_t W, int32_t H,
                            unsigned long long* err, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  // events must be >= t_origin and > the last rendered frame time (A15)
  const int64_t t_min = last_frame_t == INT64_MIN ? t_origin : std::max(t_origin, last_frame_t + 1);
  int64_t blocks = (n + 2047) / 2048;
  if (blocks > 148 * 8) blocks = 148 * 8;
  esi_validate_kernel<<<(int)blocks, 256, 0, s>>>(ev, n, prev_t, t_min, W, H, err);
  return cudaGetLastError();
}

}  // namespace esi

namespace esi {
__global__ void esi_fill_i64_kernel(int64_t* p, int64_t n, int64_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
cudaError_t launch_fill_i64(int64_t* p, int64_t n, int64_t v, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  esi_fill_i64_kernel<<<(int)blocks, 256, 0, s>>>(p, n, v);
  return cudaGetLastError();
}
}  // namespace esi
