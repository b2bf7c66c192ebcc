/*
 * esi_oracle.c -- TEST INFRASTRUCTURE ONLY.  See esi_oracle.h.
 *
 * Plain fp64, single thread, no blocking, no reordering.  Build with
 *   gcc -O2 -fno-fast-math -ffp-contract=off -shared -fPIC
 * Every function names the passage of /root/reference/PAPER.md (P:line) or
 * SPEC.md (S:line) it follows.
 */
#include "esi_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

struct esio {
  int32_t W, H;
  double C, k, b, s_min, s_max;    /* Alg. 2 inputs k, b, C; Eq. 13 bounds */
  int64_t t_origin;
  int32_t readout_decay;
  int32_t decay_kind;              /* 0: Eq. 4 (ESI); 1: exponential (camera plugin);
                                      2: none -- the naive Eq. 2 integrator, no per-event clamp */
  int32_t decay_first;             /* 0: Alg. 2 order (add, then decay); 1: decay, then add (A1 variant) */
  int32_t state_unclamped;         /* 1: no per-event Eq. 13 clamp, frames clamp at render */
  double* S;                       /* accumulation matrix */
  int64_t* T;                      /* last decay time matrix */
  int64_t* pt; uint16_t* px; uint16_t* py; int8_t* pp;   /* pending events */
  size_t n_pending, head, cap;
  int has_last_event; int64_t last_event_t;
  int has_last_frame; int64_t last_frame_t;
};

/* Eq. 4:  d(t) = max{(1 - k t)^b, 0}.  t = dt_us * 1e-6 s (A11).
 * pow is evaluated only when the base is positive (A14). */
double esio_decay(int64_t dt_us, double k, double b) {
  double dt_s = (double)dt_us / 1e6;     /* correctly rounded: d(1/k) = 0 exactly */
  double u = 1.0 - k * dt_s;
  if (u > 0.0) return pow(u, b);
  return 0.0;
}

/* Exponential decay of the DV "Accumulator" camera plugin that the paper
 * compares against ("the exponential function used in the
 * camera plugin"); Algorithm 1 with d(t) replaced by
 * exp(-lambda t), lambda = k here.  t = dt_us * 1e-6 s (A11). */
double esio_decay_exp(int64_t dt_us, double k) {
  double dt_s = (double)dt_us / 1e6;
  return exp(-k * dt_s);
}

/* The handle's decay function (Eq. 4, or the exponential variant). */
static double esio_decay_h(const esio_t* h, int64_t dt_us) {
  if (h->decay_kind == 2) return 1.0;   /* Eq. 2: L~(t) = c sum e(s), no decay */
  return h->decay_kind ? esio_decay_exp(dt_us, h->k) : esio_decay(dt_us, h->k, h->b);
}

/* Eq. 13: S = min(max(S, S_min), S_max). */
double esio_clamp(double v, double s_min, double s_max) {
  double lo = v > s_min ? v : s_min;
  return lo < s_max ? lo : s_max;
}

/* Eq. 14: B = 255 (S - S_min) / (S_max - S_min); rounding half away
 * from zero (A8) and saturation to the 8-bit range. */
uint8_t esio_map(double v, double s_min, double s_max) {
  double q = 255.0 * (v - s_min) / (s_max - s_min);
  double r = round(q);              /* C99 round(): half away from zero */
  if (r < 0.0) r = 0.0;
  if (r > 255.0) r = 255.0;
  return (uint8_t)r;
}

int esio_create(int32_t width, int32_t height, double C, double k, double b,
                double s_min, double s_max, int64_t t_origin,
                int32_t readout_decay, esio_t** out) {
  if (!out) return ESIO_ERR_INVALID_ARG;
  *out = NULL;
  if (width < 1 || height < 1 || width > 65535 || height > 65535)
    return ESIO_ERR_INVALID_ARG;
  if (!(C > 0.0) || !(k > 0.0) || !(b > 0.0) || !isfinite(C) || !isfinite(k) ||
      !isfinite(b) || !isfinite(s_min) || !isfinite(s_max) || !(s_min < s_max))
    return ESIO_ERR_INVALID_ARG;
  esio_t* h = (esio_t*)calloc(1, sizeof(esio_t));
  if (!h) return ESIO_ERR_OOM;
  h->W = width; h->H = height; h->C = C; h->k = k; h->b = b;
  h->s_min = s_min; h->s_max = s_max; h->t_origin = t_origin;
  h->readout_decay = readout_decay ? 1 : 0;
  size_t P = (size_t)width * (size_t)height;
  h->S = (double*)malloc(P * sizeof(double));
  h->T = (int64_t*)malloc(P * sizeof(int64_t));
  if (!h->S || !h->T) { esio_destroy(h); return ESIO_ERR_OOM; }
  esio_reset(h);
  *out = h;
  return ESIO_OK;
}

void esio_destroy(esio_t* h) {
  if (!h) return;
  free(h->S); free(h->T); free(h->pt); free(h->px); free(h->py); free(h->pp);
  free(h);
}

/* Alg. 2 "Initialize": S <- 0, T <- 0 (T <- t_origin, A3). */
int esio_reset(esio_t* h) {
  if (!h) return ESIO_ERR_INVALID_ARG;
  size_t P = (size_t)h->W * (size_t)h->H;
  for (size_t i = 0; i < P; i++) { h->S[i] = 0.0; h->T[i] = h->t_origin; }
  h->n_pending = 0; h->head = 0;
  h->has_last_event = 0; h->has_last_frame = 0;
  return ESIO_OK;
}

size_t esio_pending(const esio_t* h) { return h ? h->n_pending - h->head : 0; }

/* Validation (S:45-53 validate_event; S:99, S:108 NegativeInterval; A15):
 * 0<=x<W, 0<=y<H, p in {+1,-1}, t non-decreasing, t >= t_origin, and t later
 * than the last rendered frame.  The whole batch is rejected on any error. */
int esio_push(esio_t* h, const int64_t* t, const uint16_t* x, const uint16_t* y,
              const int8_t* p, size_t n) {
  if (!h) return ESIO_ERR_INVALID_ARG;
  if (n == 0) return ESIO_OK;
  if (!t || !x || !y || !p) return ESIO_ERR_INVALID_ARG;
  int has_prev = h->has_last_event; int64_t prev = h->last_event_t;
  for (size_t i = 0; i < n; i++) {
    if (x[i] >= (uint32_t)h->W || y[i] >= (uint32_t)h->H) return ESIO_ERR_OUT_OF_BOUNDS;
    if (p[i] != 1 && p[i] != -1) return ESIO_ERR_BAD_POLARITY;
    if (t[i] < h->t_origin) return ESIO_ERR_NEGATIVE_INTERVAL;
    if (has_prev && t[i] < prev) return ESIO_ERR_NEGATIVE_INTERVAL;
    if (h->has_last_frame && t[i] <= h->last_frame_t) return ESIO_ERR_NEGATIVE_INTERVAL;
    has_prev = 1; prev = t[i];
  }
  /* compact the consumed prefix, then grow */
  if (h->head > 0) {
    size_t m = h->n_pending - h->head;
    memmove(h->pt, h->pt + h->head, m * sizeof(int64_t));
    memmove(h->px, h->px + h->head, m * sizeof(uint16_t));
    memmove(h->py, h->py + h->head, m * sizeof(uint16_t));
    memmove(h->pp, h->pp + h->head, m * sizeof(int8_t));
    h->n_pending = m; h->head = 0;
  }
  if (h->n_pending + n > h->cap) {
    size_t nc = h->cap ? h->cap : 1024;
    while (nc < h->n_pending + n) nc *= 2;
    int64_t* a = (int64_t*)realloc(h->pt, nc * sizeof(int64_t)); if (!a) return ESIO_ERR_OOM; h->pt = a;
    uint16_t* b1 = (uint16_t*)realloc(h->px, nc * sizeof(uint16_t)); if (!b1) return ESIO_ERR_OOM; h->px = b1;
    uint16_t* b2 = (uint16_t*)realloc(h->py, nc * sizeof(uint16_t)); if (!b2) return ESIO_ERR_OOM; h->py = b2;
    int8_t* c = (int8_t*)realloc(h->pp, nc * sizeof(int8_t)); if (!c) return ESIO_ERR_OOM; h->pp = c;
    h->cap = nc;
  }
  memcpy(h->pt + h->n_pending, t, n * sizeof(int64_t));
  memcpy(h->px + h->n_pending, x, n * sizeof(uint16_t));
  memcpy(h->py + h->n_pending, y, n * sizeof(uint16_t));
  memcpy(h->pp + h->n_pending, p, n * sizeof(int8_t));
  h->n_pending += n;
  h->has_last_event = 1; h->last_event_t = prev;
  return ESIO_OK;
}

/* One pass of the Alg. 2 loop body for event e_i at pixel (x, y).
 * decay_first (reading A1 variant; the order of Eq. 3/5 and of the
 * complementary filter): the decay line runs before
 * the contrast step; everything else is unchanged. */
static void esio_apply_event(esio_t* h, int64_t t, uint16_t x, uint16_t y, int8_t p) {
  size_t i = (size_t)y * (size_t)h->W + (size_t)x;
  int64_t dt = t - h->T[i];                             /* P:245  dt <- t_i - T(x, y)     */
  if (!h->decay_first) {
    h->S[i] = h->S[i] + (double)p * h->C;               /* P:243  S <- S + p_i x C        */
    h->S[i] = h->S[i] * esio_decay_h(h, dt);            /* P:247  S <- S x max{(1-k dt)^b, 0} */
  } else {
    h->S[i] = h->S[i] * esio_decay_h(h, dt);            /* P:247 first                    */
    h->S[i] = h->S[i] + (double)p * h->C;               /* then P:243                     */
  }
  h->T[i] = t;                                          /* P:249  T <- t_i                */
  if (h->decay_kind != 2 && !h->state_unclamped)        /* Eq. 2 / unclamped variants: no clamp */
    h->S[i] = esio_clamp(h->S[i], h->s_min, h->s_max);  /* P:251  clamp (Eq. 13)          */
}

int esio_set_unclamped(esio_t* h, int32_t state_unclamped) {
  if (!h || state_unclamped < 0 || state_unclamped > 1) return ESIO_ERR_INVALID_ARG;
  h->state_unclamped = state_unclamped;
  return ESIO_OK;
}

int esio_set_variant(esio_t* h, int32_t decay_kind, int32_t decay_first) {
  if (!h || decay_kind < 0 || decay_kind > 2 || decay_first < 0 || decay_first > 1) return ESIO_ERR_INVALID_ARG;
  h->decay_kind = decay_kind;
  h->decay_first = decay_first;
  return ESIO_OK;
}

/* Integrate pending events with t <= t_limit (A6: ties belong to the frame). */
static void esio_integrate_upto(esio_t* h, int has_limit, int64_t t_limit) {
  while (h->head < h->n_pending) {
    size_t j = h->head;
    if (has_limit && h->pt[j] > t_limit) break;
    esio_apply_event(h, h->pt[j], h->px[j], h->py[j], h->pp[j]);
    h->head++;
  }
}

int esio_flush(esio_t* h) {
  if (!h) return ESIO_ERR_INVALID_ARG;
  esio_integrate_upto(h, 0, 0);
  return ESIO_OK;
}

/* Alg. 2 mapping loop with the readout reading A4/A5:
 * v = S * d(t_frame - T) (non-mutating) when readout_decay, else S;
 * v is clamped (Eq. 13) and mapped by Eq. 14. */
int esio_render(esio_t* h, int64_t t_frame, uint8_t* out) {
  if (!h || !out) return ESIO_ERR_INVALID_ARG;
  if (t_frame < h->t_origin) return ESIO_ERR_NEGATIVE_INTERVAL;
  if (h->has_last_frame && t_frame < h->last_frame_t) return ESIO_ERR_NEGATIVE_INTERVAL;
  esio_integrate_upto(h, 1, t_frame);
  size_t P = (size_t)h->W * (size_t)h->H;
  for (size_t i = 0; i < P; i++) {
    double v = h->S[i];
    if (h->readout_decay) v = v * esio_decay_h(h, t_frame - h->T[i]);
    v = esio_clamp(v, h->s_min, h->s_max);
    out[i] = esio_map(v, h->s_min, h->s_max);
  }
  h->has_last_frame = 1; h->last_frame_t = t_frame;
  return ESIO_OK;
}

int esio_render_many(esio_t* h, const int64_t* t_frames, size_t n, uint8_t* out) {
  if (!h || (n && (!t_frames || !out))) return ESIO_ERR_INVALID_ARG;
  for (size_t j = 1; j < n; j++)
    if (t_frames[j] < t_frames[j - 1]) return ESIO_ERR_INVALID_ARG;
  size_t P = (size_t)h->W * (size_t)h->H;
  for (size_t j = 0; j < n; j++) {
    int rc = esio_render(h, t_frames[j], out + j * P);
    if (rc) return rc;
  }
  return ESIO_OK;
}

int esio_get_state(const esio_t* h, double* S, int64_t* T) {
  if (!h) return ESIO_ERR_INVALID_ARG;
  size_t P = (size_t)h->W * (size_t)h->H;
  if (S) memcpy(S, h->S, P * sizeof(double));
  if (T) memcpy(T, h->T, P * sizeof(int64_t));
  return ESIO_OK;
}

int esio_set_state(esio_t* h, const double* S, const int64_t* T) {
  if (!h || !S || !T) return ESIO_ERR_INVALID_ARG;
  size_t P = (size_t)h->W * (size_t)h->H;
  memcpy(h->S, S, P * sizeof(double));
  memcpy(h->T, T, P * sizeof(int64_t));
  return ESIO_OK;
}

int esio_run(int32_t width, int32_t height, double C, double k, double b,
             double s_min, double s_max, int64_t t_origin, int32_t readout_decay,
             const int64_t* t, const uint16_t* x, const uint16_t* y,
             const int8_t* p, size_t n, const int64_t* t_frames, size_t n_frames,
             uint8_t* frames, double* S, int64_t* T) {
  esio_t* h = NULL;
  int rc = esio_create(width, height, C, k, b, s_min, s_max, t_origin, readout_decay, &h);
  if (rc) return rc;
  rc = esio_push(h, t, x, y, p, n);
  if (!rc) rc = esio_render_many(h, t_frames, n_frames, frames);
  if (!rc) rc = esio_get_state(h, S, T);
  esio_destroy(h);
  return rc;
}
