/*
 * esi.h -- C ABI of the B200-native ESI library (libesi.so).
 *
 * ESI = Event-based Single Integration, arXiv 2508.02238.  The library turns
 * an asynchronous event stream e = {x, y, t, p} (Sec. III-A)
 * into 8-bit intensity frames at caller-chosen frame times (typically 100 FPS,
 * P:20).  Per event it runs Algorithm 2: add p*C,
 * decay by Eq. 4 d(dt) = max{(1 - k dt)^b, 0}, set T,
 * clamp by Eq. 13.  Each frame is the Eq. 14 linear map
 * B = 255 (S - S_min)/(S_max - S_min) of the state.
 * The readings of the paper this library implements are listed in DESIGN.md
 * section 3 (A1..A17); the same readings are used by the fp64 oracle under
 * oracle/ (which shares no code with this library).
 *
 * Threading: one writer per handle.  All GPU work of a
 * handle runs on its stream (its own, or the one set by esi_set_stream).
 *
 * Errors: every call returns an esi_status (0 = ESI_OK).  By default
 * (params.validate_on_push = 1) esi_push_events validates the batch on the
 * device before it returns (SURVEY 8(b) "atomic push"): on an
 * invalid event it returns the error, keeps none of the batch's events and
 * the handle stays usable -- a rejected push therefore never reaches a render,
 * which writes no frame and leaves S and T untouched.  This costs one extra
 * device read of each pushed batch.
 * With params.validate_on_push = 0 ("fused" mode, for trusted streams) the
 * checks run inside the ingest kernel during the render instead (no extra
 * pass).  An invalid event found there is STICKY: the render returns it,
 * S and T are restored to their value at the start of that render (nothing
 * is integrated), the frames it wrote are unspecified, and every later call
 * returns the error until esi_reset().  (reading A21.)
 * CUDA failures latch ESI_ERR_CUDA (sticky, also cleared only by esi_reset).
 */
#ifndef ESI_H
#define ESI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESI_ABI_VERSION 1

/* Status codes (numbering of SURVEY.md section 8(b)). */
typedef enum {
  ESI_OK = 0,
  ESI_ERR_INVALID_ARG = 1,       /* null pointer, bad size, bad parameter, frames out of order */
  ESI_ERR_OUT_OF_BOUNDS = 2,     /* event x >= width or y >= height */
  ESI_ERR_BAD_POLARITY = 3,      /* event p not in {+1, -1} */
  ESI_ERR_NEGATIVE_INTERVAL = 4, /* event t below its predecessor, below t_origin, or not later
                                    than the last rendered frame; frame time going backwards */
  ESI_ERR_CUDA = 5,              /* any CUDA error (sticky) */
  ESI_ERR_OOM = 6                /* device or host allocation failure */
} esi_status;

/* One event, 16 bytes, little-endian; the record layout of SPEC S:370
 * (t: int64 microseconds, x, y: pixel column/row, p: +1 or -1). */
typedef struct {
  int64_t t_us;
  uint16_t x;
  uint16_t y;
  int8_t p;
  uint8_t _pad[3];
} esi_event_t;

/* Algorithm 2 inputs and the Eq. 13 bounds. */
typedef struct {
  double C;              /* contrast step per event, > 0 (Alg. 2 "C")             */
  double k;              /* Eq. 4 decay rate in 1/s, > 0                           */
  double b;              /* Eq. 4 exponent, > 0                                    */
  double s_min, s_max;   /* Eq. 13 clamp bounds, s_min < s_max                    */
  int64_t t_origin_us;   /* initial T of every pixel (Alg. 2 "T <- 0", P:239 => default 0) */
  int32_t readout_decay; /* 1: frame value S*d(t_frame - T), non-mutating (reading A4);
                            0: Alg. 2 literal, frame maps the stored S             */
  int32_t device;        /* CUDA device ordinal                                            */
  int32_t validate_on_push; /* 1 (default): atomic validation in esi_push_events; 0: fused (see above) */
  int32_t chunk_events;  /* events per pipeline chunk; 0 = default (8 Mi)                  */
  /* Decay variants (reading A20), default 0 = ESI:
   * decay_kind  0: Eq. 4 d = max{(1 - k dt)^b, 0};  1: d = exp(-k dt), the
   *             exponential decay of the camera plugin the paper compares
   *             against (b is ignored).  The device paths
   *             take d = 0 for k dt >= 24 (e^-24 = 3.8e-11).
   *             2: none -- the naive Eq. 2 integrator S <- S + pC,
   *             no per-event clamp; frames still clamp (Eq. 13) at render;
   *             runs on the fp64 kernel (the sum is unbounded).
   * decay_first 0: Alg. 2 order, S <- clamp((S + pC) d);
   *             1: decay, then add, S <- clamp(S d + pC)  (the Eq. 3/5 and
   *             complementary-filter order, reading A1). */
  int32_t decay_kind;
  int32_t decay_first;
  /* state_unclamped 1: no per-event Eq. 13 clamp; frames still clamp
   * at render.  With decay_kind 1 and decay_first 1 this is the events-only
   * complementary filter.  Default 0.  Unclamped
   * states are unbounded sums that can cancel, so they accumulate in fp64
   * (the wide kernel; S is stored in fp32 between chunks). */
  int32_t state_unclamped;
  /* How pixel ids map to the integrate kernel's bands (one CTA each; esi_layout).
   * A performance knob only: frames and state do not depend on it.
   * ESI_BANDS_CONTIGUOUS (0, default): band b = a run of band_px consecutive ids
   *   (fastest when the activity covers the sensor, as in BASELINE's configs).
   * ESI_BANDS_INTERLEAVED (1): ids are dealt to the bands in groups of 64
   *   consecutive ids, round-robin -- every band samples the whole sensor, so the
   *   bands stay balanced when the activity is local (a moving object);
   *   measured in DESIGN.md section 7e. */
  int32_t band_layout;
} esi_params_t;

#define ESI_BANDS_CONTIGUOUS 0
#define ESI_BANDS_INTERLEAVED 1
/* ESI_BANDS_AUTO: start contiguous; after a render whose busiest band held more than
 * 3x the mean band's events (at least 100 k events), switch to the interleaved layout
 * for the following renders (esi_reset returns to contiguous).  esi_layout reports
 * the layout in use. */
#define ESI_BANDS_AUTO 2

typedef struct esi_handle esi_handle_t;

/* Fills *p with the defaults: C=0.15, k=10, b=2, s_min=-1.5, s_max=1.5 (SPEC S:134,
 * S:210-211), t_origin 0, readout_decay 1, device 0, validate_on_push 1 (atomic). */
void esi_default_params(esi_params_t* p);

/* Creates a handle for a width x height sensor (1 <= width, height <= 65535,
 * width*height <= 2^22 = 4194304 pixels: 1024 bands of <= 4096 pixels, the
 * shared-memory band state of the integrate kernel; the largest BASELINE
 * sensor, 2560x1440, is 3.7 Mpx.  Larger sensors are split into row bands
 * across handles / GPUs, esi_route_bands; reading A22).  Allocates the per-pixel state S (fp32) and T (int64)
 * on the device, S = 0, T = t_origin (Alg. 2 "Initialize").
 * Returns ESI_ERR_INVALID_ARG for bad sizes/params, ESI_ERR_OOM, ESI_ERR_CUDA. */
int esi_create(int32_t width, int32_t height, const esi_params_t* params, esi_handle_t** out);

/* Appends n events (the Alg. 2 input E) to the handle's pending stream.
 * Events must be globally non-decreasing in t (reading A15) and later than the
 * last rendered frame.
 *  - pageable host pointer: the events are copied to device memory before the
 *    call returns; the caller may reuse the buffer at once.
 *  - pinned (page-locked) host pointer, e.g. cudaHostAlloc / torch pin_memory:
 *    BORROWED.  esi_render* copies it to the device chunk by chunk on a copy
 *    stream, overlapped with the kernels, so the caller must keep it alive and
 *    unmodified until the render that integrates its last event has returned
 *    (or until esi_reset/esi_destroy).  (With params.validate_on_push the batch
 *    is copied at push time instead.)
 *  - device pointer: ZERO-COPY.  The library BORROWS the buffer: it reads it
 *    during later esi_render* calls (stream-ordered on the handle's stream), so
 *    the caller must keep it alive and unmodified until the render that
 *    integrates its last event has completed (or until esi_reset/esi_destroy).
 * The buffer must be 8-byte aligned.  n = 0 is a no-op. */
int esi_push_events(esi_handle_t* h, const esi_event_t* events, size_t n);

/* Renders one frame at t_frame_us: integrates every pending event with
 * t <= t_frame_us (ties belong to the frame, reading A6), then writes the
 * width*height row-major 8-bit frame (index y*width + x) to out, which may be
 * a host or a device pointer (host: frames are copied back chunk by chunk,
 * overlapped with the kernels; pinned host memory copies fastest).  Later
 * events stay pending.  Synchronous. */
int esi_render(esi_handle_t* h, int64_t t_frame_us, uint8_t* out);

/* Renders n frames at the non-decreasing host array t_frames_us[0..n) into
 * out[n][height][width] (host or device).  Equivalent to n esi_render calls:
 * bit-identical for every pixel that never receives two events inside one
 * 32-event integration batch (the sparse path); pixels integrated by the dense
 * warp-scan path (reassociated clamped-affine composition)
 * agree within the fp32 state tolerance.  Events with t > t_frames_us[n-1]
 * stay pending.  Synchronous. */
int esi_render_many(esi_handle_t* h, const int64_t* t_frames_us, size_t n, uint8_t* out);

/* Copies the state out (host pointers, width*height each; either may be NULL).
 * Pending events are not integrated by this call. */
int esi_get_state(esi_handle_t* h, float* S, int64_t* T);
/* Replaces the state (host pointers) -- checkpoint/resume.  Pending events stay. */
int esi_set_state(esi_handle_t* h, const float* S, const int64_t* T);
/* S = 0, T = t_origin, no pending events, no rendered frame, clears sticky errors. */
int esi_reset(esi_handle_t* h);
/* Makes the handle issue its work on cudaStream_t stream (NULL: the handle's own). */
int esi_set_stream(esi_handle_t* h, void* cuda_stream);
/* Returns the sticky error (synchronises the handle's stream). */
int esi_get_error(esi_handle_t* h);
void esi_destroy(esi_handle_t* h);
const char* esi_strerror(int status);

/* ---- multi-GPU row-band routing ----
 *
 * ESI has no spatial coupling: an event changes only its own pixel (Alg. 2,
 * P:242-253), so one large sensor can be split into row bands integrated by
 * independent handles (one per GPU, created with height = band rows).
 * esi_route_bands stably partitions the n time-ordered events at DEVICE pointer
 * `events` by band -- band b = rows [row_start[b], row_start[b+1]),
 * row_start[0] = 0 < row_start[1] < ... < row_start[n_bands] = height,
 * 1 <= n_bands <= 64 -- into the DEVICE buffer `out` (n records, caller-owned):
 * band-major, arrival order kept within a band (= a stable sort by band), with
 * y rebased to y - row_start[b].  counts (HOST, n_bands entries) receives the
 * events per band.  Both buffers must be 16-byte aligned and live on `device`;
 * n < 2^32.  Events with y >= height: ESI_ERR_OUT_OF_BOUNDS (out unspecified);
 * x, p and t are validated later by the band handle.  Runs on the cudaStream_t
 * `stream` (NULL = the legacy default stream) and synchronises it (counts are
 * host values when the call returns). */
int esi_route_bands(int32_t device, const esi_event_t* events, size_t n, int32_t height,
                    const int32_t* row_start, int32_t n_bands, esi_event_t* out, int64_t* counts,
                    void* stream);

/* Two-phase router for the multi-GPU exchange over peer memory.  The all-to-all
 * of the row-band split is done by the router's own scatter kernel: each
 * source rank writes its band-b run straight into band b's receive buffer on
 * the GPU that owns band b (NVLink P2P stores through a CUDA IPC mapping), so
 * the exchange overlaps the partition arithmetic tile by tile and needs no
 * staging copy.
 *   esi_router_create   row bands as for esi_route_bands (1 <= n_bands <= 64).
 *   esi_router_count    counts (HOST, n_bands) = events of the DEVICE array
 *                       `events` per band; synchronises `stream`.  The events
 *                       must stay valid and unchanged until the scatter has run.
 *                       y >= height: ESI_ERR_OUT_OF_BOUNDS.
 *   esi_router_scatter  writes band b's events, in arrival order and with y
 *                       rebased, to dst[b] + dst_offset[b] (records; dst is a
 *                       HOST array of n_bands DEVICE pointers, 16-byte aligned,
 *                       local or peer-mapped, each with room for
 *                       dst_offset[b] + counts[b] records).  Stream-ordered on
 *                       `stream`, no synchronisation: the caller makes the
 *                       destination's reader wait (stream sync + a host
 *                       barrier across the ranks).
 * The router owns its scratch (grown on demand) and frees it in
 * esi_router_destroy. */
typedef struct esi_router esi_router_t;
int esi_router_create(int32_t device, int32_t height, const int32_t* row_start, int32_t n_bands,
                      esi_router_t** out);
int esi_router_count(esi_router_t* r, const esi_event_t* events, size_t n, int64_t* counts, void* stream);
int esi_router_scatter(esi_router_t* r, esi_event_t* const* dst, const int64_t* dst_offset, void* stream);
void esi_router_destroy(esi_router_t* r);

/* Receive buffers shared between processes: plain cudaMalloc allocations
 * (esi_buffer_alloc / esi_buffer_free, owned by the allocating process),
 * exported with esi_ipc_get_handle (ESI_IPC_HANDLE_BYTES opaque bytes, sent to
 * the peers by the caller) and mapped by a peer with esi_ipc_open (peer access
 * enabled lazily) until esi_ipc_close.  A process cannot open its own handle:
 * it uses its own pointer.  esi_stream_sync: cudaStreamSynchronize. */
#define ESI_IPC_HANDLE_BYTES 64
int esi_buffer_alloc(int32_t device, size_t bytes, void** ptr);
int esi_buffer_free(int32_t device, void* ptr);
int esi_ipc_get_handle(const void* ptr, void* handle);
int esi_ipc_open(int32_t device, const void* handle, void** ptr);
int esi_ipc_close(int32_t device, void* ptr);
int esi_stream_sync(int32_t device, void* stream);

/* ---- evaluation: frame vs ground-truth scores --------
 * SPEC metrics: for each of n_frames 8-bit frames (DEVICE, frame j
 * at frames + j * n_pixels) the Pearson correlation with the ground-truth
 * log-intensity field (DEVICE fp32; one field of n_pixels shared by every frame,
 * or one per frame when truth_per_frame = 1) and the MSE after per-image
 * zero-mean unit-variance normalisation (= 2 (1 - pearson)).  Scale/offset
 * invariant, as the paper's relative-intensity claim requires.  A
 * constant image gives NaN for both ("missing").  pearson / mse_norm:
 * HOST arrays of n_frames; synchronises `stream`. */
int esi_frame_metrics(int32_t device, const uint8_t* frames, const float* truth, int64_t n_pixels,
                      int32_t n_frames, int32_t truth_per_frame, double* pearson, double* mse_norm,
                      void* stream);

/* ---- time-sharded single streams ----------------------
 *
 * A time slice of the stream acts on one pixel's state (S, T) of Alg. 2
 * as: no event -> identity; events e_1..e_n ->
 *   S1 = clamp((S + p_1 C) d(t_1 - T))      (decay-first variant: clamp(S d + p_1 C))
 *   S' = G(S1),  T' = t_n,
 * with G = g_n o ... o g_2 the composition of the later events' clamped affine
 * maps g_k(s) = clamp(d_k s + d_k p_k C, S_min, S_max), d_k = d(t_k - t_{k-1})
 * (Eq. 4; Eq. 13).  Only the first event's decay sees the
 * incoming T, so a slice is summarised per pixel by esi_slice_map_t, and the
 * summaries of consecutive slices compose (B's first event decays from A's
 * t_last): an exclusive scan of slice maps across GPUs gives every time shard
 * its incoming state (the Eq. 5 per-pixel product of decays composes).
 * G is kept in fp32 (the fp32 state tolerance of the render path applies). */
typedef struct {
  int64_t t_first;   /* t of the slice's first event at the pixel (us) */
  int64_t t_last;    /* t of its last event */
  float a, c, lo, hi;/* G(s) = min(max(a s + c, lo), hi), a >= 0 */
  int32_t n;         /* events of the slice at the pixel; 0 = identity (other fields unused) */
  int32_t p_first;   /* polarity of the first event */
} esi_slice_map_t;   /* 40 bytes */

/* maps [W*H] (DEVICE pointer, overwritten) <- the summary of the n events
 * (host or device pointer; validated like esi_push_events: sensor bounds,
 * polarity, non-decreasing t; the first error code is returned and maps are
 * unspecified).  Uses the handle's parameters and stream; does not touch its
 * state or pending events.  Chunks of the slice must each span < 2^31 us
 * (ESI_ERR_INVALID_ARG otherwise).  Synchronises the handle's stream. */
int esi_slice_summarize(esi_handle_t* h, const esi_event_t* events, size_t n, esi_slice_map_t* maps);
/* out = `first` followed by `second` (all DEVICE pointers of W*H maps; out may
 * alias either input).  Stream-ordered on the handle's stream. */
int esi_slice_compose(esi_handle_t* h, const esi_slice_map_t* first, const esi_slice_map_t* second,
                      esi_slice_map_t* out);
/* The handle's state (S, T) <- the action of `maps` (DEVICE pointer).  No event
 * may be pending (ESI_ERR_INVALID_ARG).  Stream-ordered. */
int esi_slice_apply(esi_handle_t* h, const esi_slice_map_t* maps);

/* ---- instrumentation (used by bench.py and the parity tests) -------------- */

/* Per-kernel device time accumulated by the handle when timing is enabled
 * (cudaEvents around each launch, on the handle's stream).  kind:
 * 0 = ingest/partition, 1 = integrate+readout, 2 = readout-only, 3 = push validation. */
int esi_enable_kernel_timing(esi_handle_t* h, int enable);
int esi_kernel_time(esi_handle_t* h, int kind, double* ms_total, int64_t* launches);
/* Counters of the last render call: launches of this library's kernels,
 * events integrated, chunks. */
int esi_last_render_stats(esi_handle_t* h, int64_t* kernel_launches, int64_t* events,
                          int64_t* chunks);

/* The handle's band layout: bands (K1 partition buckets = integrate CTAs),
 * pixel slots per band, warps per integrate CTA.  With params.band_layout =
 * ESI_BANDS_INTERLEAVED pixel id q belongs to band (q / 64) % n_bands, with
 * ESI_BANDS_CONTIGUOUS to band q / band_px.  Any pointer may be NULL. */
int esi_layout(esi_handle_t* h, int32_t* n_bands, int32_t* band_px, int32_t* warps_per_band);

/* Debug export of the bit-exact grouping step: runs only the
 * ingest/partition kernel over the pending events of the first chunk and
 * copies back, for every band (esi_layout), the events routed to it in arrival order, as records
 * {t_us, pixel id, p}.
 * out_* must hold n_out entries; band_start[nb+1] receives the CSR offsets.
 * Does not consume events. */
int esi_debug_partition(esi_handle_t* h, int64_t* out_t, uint32_t* out_pid, int8_t* out_p,
                        size_t n_out, uint32_t* band_start, int32_t* nb_out, int32_t* band_px_out);

#ifdef __cplusplus
}
#endif
#endif /* ESI_H */
