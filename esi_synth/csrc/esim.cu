// esim.cu -- CUDA event-camera simulator (SPEC synth S:290-348).
//
// TOOLING, not the ESI product path: it holds no ESI arithmetic.  It turns a
// procedural log-intensity scene L(x, y, t) into an event stream with the
// reference-level threshold-crossing model of PAPER.md Eq. 1 / Sec. III-A
// (SPEC TriggerModel S:301-303, design decision S:337): per pixel,
// an event fires each time |L - L_ref| reaches c, L_ref steps by +-c per
// event (several events per sample step allowed), and each crossing time is
// linearly interpolated inside the sample step and floored to 1 us (S:322,
// S:339).
//
// One thread per pixel walks the sample steps sequentially (pixels are
// independent, "embarrassingly parallel").  Two passes with the same
// arithmetic: esim_count (events per pixel) and esim_emit (the events of pixel
// q written pixel-major at offset[q], in emission order).  The caller merges
// them into one time-ordered stream with a stable sort by t, which breaks ties
// by (pixel id, emission order) -- deterministic, byte-identical across runs
// (S:333).
//
// Scenes (sampled at times steps[k], with a per-step scene parameter):
//   kind 0 -- rotating texture (configs c4, c5a, c5b: "fast camera rotation
//             over a seeded random-texture scene"): param = angle theta;
//             L = bilinear sample (reflection padding, align_corners = false)
//             of an R x R log texture at the pixel centre rotated by theta
//             about the image centre.
//   kind 1 -- the Fig. 2 scene of SPEC S:296-299: log of a linear intensity
//             ramp along x, times the reflectivity inside a circle whose centre
//             moves along x; param = circle centre x (px).  Scene constants in
//             EsimScene.
#include <cstdint>
#include <cuda_runtime.h>

extern "C" {

typedef struct {
  int32_t kind;          // 0 rotating texture, 1 ramp + circle (Fig. 2)
  int32_t W, H;
  float c;               // contrast threshold (log units)
  // kind 0
  const float* tex;      // [R][R] device log texture
  int32_t R;
  // kind 1 (SPEC SceneSpec S:296)
  float ramp_min, ramp_max;   // linear intensity at x = 0 and x = W (> 0)
  float radius, reflect, cy;  // circle radius (px), reflectivity, centre y
} EsimScene;

}  // extern "C"

namespace {

__device__ __forceinline__ float reflect_coord(float x, float size) {
  // torch grid_sample padding_mode="reflection", align_corners=False: reflect
  // about the borders -0.5 and size - 0.5 (in pixel units)
  const float lo = -0.5f, span = size;
  float v = fabsf(x - lo);
  const float flips = floorf(v / span);
  const float extra = v - flips * span;
  v = (fmodf(flips, 2.f) == 0.f) ? lo + extra : lo + span - extra;
  return fminf(fmaxf(v, 0.f), size - 1.f);
}

__device__ __forceinline__ float scene_L(const EsimScene& s, int x, int y, float param) {
  if (s.kind == 1) {
    const float xc = x + 0.5f, yc = y + 0.5f;
    float I = s.ramp_min + (s.ramp_max - s.ramp_min) * xc / (float)s.W;
    const float dx = xc - param, dy = yc - s.cy;
    if (dx * dx + dy * dy <= s.radius * s.radius) I *= s.reflect;
    return logf(I);
  }
  const float px = x + 0.5f - 0.5f * s.W, py = y + 0.5f - 0.5f * s.H;
  float sn, cs;
  sincosf(param, &sn, &cs);
  const float u = cs * px - sn * py, v = sn * px + cs * py;
  // normalised grid coordinate g = u / (R/2); align_corners=False: ix = ((g + 1) R - 1) / 2
  const float R = (float)s.R;
  float ix = ((u / (0.5f * R) + 1.f) * R - 1.f) * 0.5f;
  float iy = ((v / (0.5f * R) + 1.f) * R - 1.f) * 0.5f;
  ix = reflect_coord(ix, R);
  iy = reflect_coord(iy, R);
  const int x0 = (int)floorf(ix), y0 = (int)floorf(iy);
  const int x1 = min(x0 + 1, s.R - 1), y1 = min(y0 + 1, s.R - 1);
  const float fx = ix - x0, fy = iy - y0;
  const float* t = s.tex;
  const float a = __ldg(t + (size_t)y0 * s.R + x0), b = __ldg(t + (size_t)y0 * s.R + x1);
  const float c = __ldg(t + (size_t)y1 * s.R + x0), d = __ldg(t + (size_t)y1 * s.R + x1);
  return (a * (1.f - fx) + b * fx) * (1.f - fy) + (c * (1.f - fx) + d * fx) * fy;
}

// The threshold-crossing walk of one pixel; EMIT = false counts only.
template <bool EMIT>
__device__ __forceinline__ int64_t walk(const EsimScene& s, int x, int y, const int64_t* steps, const float* param,
                                        int n_steps, int64_t* t_out, int8_t* p_out) {
  float L_prev = scene_L(s, x, y, param[0]);
  float L_ref = L_prev;
  int64_t n = 0;
  for (int k = 1; k < n_steps; ++k) {
    const float L_new = scene_L(s, x, y, param[k]);
    const float d = L_new - L_ref;
    const int n_up = d > 0.f ? (int)floorf(d / s.c) : 0;
    const int n_dn = d < 0.f ? (int)floorf(-d / s.c) : 0;
    const int m = n_up + n_dn;
    if (m) {
      if (EMIT) {
        const float sgn = n_up ? 1.f : -1.f;
        const float den = fabsf(L_new - L_prev) > 1e-12f ? (L_new - L_prev) : 1.f;
        const int64_t t0 = steps[k - 1], dt = steps[k] - steps[k - 1];
        for (int i = 1; i <= m; ++i) {
          const float lv = L_ref + sgn * (float)i * s.c;
          const float frac = fminf(fmaxf((lv - L_prev) / den, 0.f), 1.f);
          t_out[n + i - 1] = t0 + (int64_t)floorf(frac * (float)dt);
          p_out[n + i - 1] = n_up ? 1 : -1;
        }
      }
      n += m;
      L_ref += s.c * (float)(n_up - n_dn);
    }
    L_prev = L_new;
  }
  return n;
}

__global__ void esim_count_kernel(EsimScene s, const int64_t* steps, const float* param, int n_steps,
                                  int64_t* count) {
  const int64_t P = (int64_t)s.W * s.H;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x)
    count[q] = walk<false>(s, (int)(q % s.W), (int)(q / s.W), steps, param, n_steps, nullptr, nullptr);
}

__global__ void esim_emit_kernel(EsimScene s, const int64_t* steps, const float* param, int n_steps,
                                 const int64_t* offset, int64_t* t_out, int32_t* pid_out, int8_t* p_out) {
  const int64_t P = (int64_t)s.W * s.H;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = offset[q];
    const int64_t n = walk<true>(s, (int)(q % s.W), (int)(q / s.W), steps, param, n_steps, t_out + o, p_out + o);
    for (int64_t i = 0; i < n; ++i) pid_out[o + i] = (int32_t)q;
  }
}

__global__ void esim_field_kernel(EsimScene s, float param, float* out) {
  const int64_t P = (int64_t)s.W * s.H;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = scene_L(s, (int)(q % s.W), (int)(q / s.W), param);
}

// pack (t, pid, p) in the order perm into 16-byte esi_event_t records
__global__ void esim_pack_kernel(const int64_t* t, const int32_t* pid, const int8_t* p, const int64_t* perm,
                                 int64_t n, int32_t W, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = perm ? perm[i] : i;
    const int32_t q = pid[j];
    out[2 * i] = t[j];
    out[2 * i + 1] = (int64_t)(q % W) | ((int64_t)(q / W) << 16) | ((int64_t)((uint8_t)p[j]) << 32);
  }
}

int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b > 148 * 32 ? 148 * 32 : (b < 1 ? 1 : b));
}

}  // namespace

extern "C" {

// Events per pixel (count[W*H], device) for the sample steps steps[0..n_steps)
// (device, int64 us, increasing) with scene parameter param[k] (device).
int esim_count(const EsimScene* s, const int64_t* steps, const float* param, int n_steps, int64_t* count,
               void* stream) {
  if (!s || !steps || !param || !count || n_steps < 1) return 1;
  const int64_t P = (int64_t)s->W * s->H;
  esim_count_kernel<<<grid_for(P), 256, 0, (cudaStream_t)stream>>>(*s, steps, param, n_steps, count);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

// The events, pixel-major: pixel q's events in emission order at offset[q]
// (device exclusive prefix of esim_count's counts).
int esim_emit(const EsimScene* s, const int64_t* steps, const float* param, int n_steps, const int64_t* offset,
              int64_t* t_out, int32_t* pid_out, int8_t* p_out, void* stream) {
  if (!s || !steps || !param || !offset || !t_out || !pid_out || !p_out || n_steps < 1) return 1;
  const int64_t P = (int64_t)s->W * s->H;
  esim_emit_kernel<<<grid_for(P), 256, 0, (cudaStream_t)stream>>>(*s, steps, param, n_steps, offset, t_out, pid_out,
                                                                   p_out);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

// The scene's log intensity L(x, y) at scene parameter `param` (out: device, W*H).
int esim_field(const EsimScene* s, float param, float* out, void* stream) {
  if (!s || !out) return 1;
  const int64_t P = (int64_t)s->W * s->H;
  esim_field_kernel<<<grid_for(P), 256, 0, (cudaStream_t)stream>>>(*s, param, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

// out[2 i], out[2 i + 1] = the esi_event_t record of event perm[i] (perm may be NULL).
int esim_pack(const int64_t* t, const int32_t* pid, const int8_t* p, const int64_t* perm, int64_t n, int32_t W,
              int64_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!t || !pid || !p || !out))) return 1;
  if (n == 0) return 0;
  esim_pack_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(t, pid, p, perm, n, W, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

}  // extern "C"
