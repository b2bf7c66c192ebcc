/*
 * esi_oracle.h -- TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * Plain, slow, single-threaded fp64 CPU oracle of ESI (Event-based Single
 * Integration, arXiv 2508.02238).  It follows Algorithm 2 (PAPER.md lines
 * 233-262) step by step in the paper's order, plus the frame readout of
 * Eq. 14.  It shares no code, header, table or constant with the
 * CUDA library under paper_2508_02238_b200/ and include/; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.
 *
 * Readings of the paper this oracle takes are the A1..A17 list of
 * SURVEY.md section 8(c), restated in DESIGN.md section 3:
 *   A1  add p*C, then decay (Alg. 2 order, P:243 then P:247)
 *   A3  T initialised to t_origin (paper: 0)
 *   A4  readout_decay=1: frame value is S*d(t_f - T) without mutating S, T;
 *       readout_decay=0: Alg. 2 literal (maps the stored S)
 *   A6  events with t == t_frame belong to that frame (Eq. 5 text)
 *   A8  Eq. 14 rounds half away from zero
 *   A9  clamp after every event (Alg. 2) and once more at readout
 *   A11 k in 1/s, t in integer microseconds
 *   A14 d = 0 exactly when 1 - k*dt <= 0 (Eq. 4); pow never sees u<=0
 *   A15 the event stream must be globally non-decreasing in t
 */
#ifndef ESI_ORACLE_H
#define ESI_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the numbering of SURVEY.md section 8(b), written out here) */
#define ESIO_OK 0
#define ESIO_ERR_INVALID_ARG 1
#define ESIO_ERR_OUT_OF_BOUNDS 2
#define ESIO_ERR_BAD_POLARITY 3
#define ESIO_ERR_NEGATIVE_INTERVAL 4
#define ESIO_ERR_OOM 6

typedef struct esio esio_t;

/* Eq. 4: d(dt) = max{(1 - k*dt)^b, 0}, dt in integer microseconds. */
double esio_decay(int64_t dt_us, double k, double b);
/* exp(-k dt): the exponential decay variant. */
double esio_decay_exp(int64_t dt_us, double k);
/* Eq. 13 */
double esio_clamp(double v, double s_min, double s_max);
/* Eq. 14, rounded half away from zero, saturated to [0,255]. */
uint8_t esio_map(double v, double s_min, double s_max);

/* Decay variants: decay_kind 0 = Eq. 4, 1 = exp(-k dt),
 * 2 = none with no per-event clamp (the naive Eq. 2 integrator; frames
 * still clamp at render);
 * decay_first 0 = Alg. 2 order (add, then decay), 1 = decay, then add. */
int esio_set_variant(esio_t* h, int32_t decay_kind, int32_t decay_first);
/* state_unclamped 1: the per-event Eq. 13 clamp is dropped and frames
 * clamp at render only -- the events-only complementary filter of SPEC
 * S:243-246, S:266 (with decay_kind 1, decay_first 1). */
int esio_set_unclamped(esio_t* h, int32_t state_unclamped);
int esio_create(int32_t width, int32_t height, double C, double k, double b,
                double s_min, double s_max, int64_t t_origin,
                int32_t readout_decay, esio_t** out);
void esio_destroy(esio_t* h);
/* Appends n events (SoA) after validating all of them; on error none are kept. */
int esio_push(esio_t* h, const int64_t* t, const uint16_t* x, const uint16_t* y,
              const int8_t* p, size_t n);
/* Integrates every pending event with t <= t_frame (Alg. 2 loop, in arrival
 * order), then writes the W*H frame (Alg. 2 mapping loop / Eq. 14). */
int esio_render(esio_t* h, int64_t t_frame, uint8_t* out);
int esio_render_many(esio_t* h, const int64_t* t_frames, size_t n, uint8_t* out);
/* Integrates every pending event (no frame). */
int esio_flush(esio_t* h);
int esio_get_state(const esio_t* h, double* S, int64_t* T);
int esio_set_state(esio_t* h, const double* S, const int64_t* T);
int esio_reset(esio_t* h);
size_t esio_pending(const esio_t* h);

/* Whole-stream convenience: create, push, render_many, return frames and the
 * final state (S, T after integrating all events with t <= last frame). */
int esio_run(int32_t width, int32_t height, double C, double k, double b,
             double s_min, double s_max, int64_t t_origin, int32_t readout_decay,
             const int64_t* t, const uint16_t* x, const uint16_t* y,
             const int8_t* p, size_t n, const int64_t* t_frames, size_t n_frames,
             uint8_t* frames, double* S, int64_t* T);

#ifdef __cplusplus
}
#endif
#endif
