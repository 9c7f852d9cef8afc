/*
 * veckm.h — C-ABI of the B200-native VecKM_flow normal-flow hot path
 * (arXiv 2504.19417).  libveckm.so exports exactly these symbols.
 *
 * Plain C types only: pointers, sizes, doubles.  No torch / CUDA types in the
 * signatures; streams travel as `void*` (a cudaStream_t, NULL = legacy default
 * stream).  `*_dev` pointers are device memory on the handle's device, `*_host`
 * pointers are host memory (pinned or pageable).
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/evflow/):
 *   vkm_create        NormalFlowRegressor.__init__/_config/_resolve_pretrained
 *                     (estimators.py:107-164), MlpWeights (flow.py:48-80),
 *                     precompute_spatial_phases (encoder.py:173-179)
 *   vkm_predict[_host] predict_flows with QuerySet.all (flow.py:155-197) as called by
 *                     NormalFlowRegressor.predict (estimators.py:192-206)
 *   vkm_encode[_host] encode + embed_to_features (encoder.py:371-412, flow.py:92-95) as
 *                     called by LocalEventEncoder.transform (estimators.py:89-95)
 *   vkm_grid          accumulate_grid + PixelGrid.embed/count (encoder.py:229-283,
 *                     196-208); pooled=1 adds the window sums of _pool_batch
 *                     (encoder.py:331-336) evaluated at every pixel
 *   vkm_predict_batch the CLI's per-slice loop (cli.py:267-280) fused into one call
 *   vkm_predict_batch_host  the same loop over host buffers, with the H2D of
 *                     slice s+1 and the D2H of slice s-1 overlapping the kernels of
 *                     slice s (NormalFlowRegressor.predict_slices)
 *   vkm_select_rows / vkm_scatter_rows  the device side of the multi-GPU
 *                     row-strip split of one slice: strip
 *                     partition with event halo, and the owned-flow gather
 *   vkm_last_error    exception text of the reference's error hierarchy (errors.py:4-29)
 *
 * Event layout: the reference's (n, 3) float64 array [t, x, y], row-major,
 * time-sorted ascending (validation.py:49-65 sorts before encoding); x, y are
 * integer-valued pixel coordinates inside the sensor.  Output rows follow the
 * input rows.  `t_start` is the slice's window start (the first timestamp,
 * validation.py:59); pass NAN to have the device read events[0].t.
 *
 * Error convention: 0 = OK, VKM_EINVAL -> ValueError, VKM_EDIM ->
 * DimensionMismatchError, VKM_ECUDA -> RuntimeError, VKM_EOOM -> MemoryError,
 * VKM_EUNSUPPORTED -> NotImplementedError.  vkm_last_error() returns the
 * thread-local message of the last failure.  Kernels never print.
 *
 * Threading: a handle is bound to one device, is not re-entrant, and all work
 * is enqueued on the stream passed in.  Distinct handles may be driven
 * concurrently from different host threads.
 */
#ifndef VECKM_H
#define VECKM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VKM_VERSION 1

enum {
  VKM_OK = 0,
  VKM_EINVAL = 1,
  VKM_EDIM = 2,
  VKM_ECUDA = 3,
  VKM_EOOM = 4,
  VKM_EUNSUPPORTED = 5
};

/* MLP execution modes of the flow head W2·relu(W1·f + b1) + b2 (flow.py:98-106). */
enum {
  VKM_MLP_AUTO = 0,   /* F16X3 when embed_dim == 64 and hidden == 128, else FP32 */
  VKM_MLP_FP32 = 1,   /* CUDA-core FFMA, fp32 throughout                           */
  VKM_MLP_F16X3 = 2,  /* tcgen05 kind::f16, 3-term hi/lo split: fp32-equivalent     */
  VKM_MLP_BF16 = 3    /* tcgen05 kind::f16 single bf16 pass: fast, stated bound     */
};

typedef struct vkm_params {
  int32_t width;      /* sensor width  (CameraGeometry, events.py:24-36)       */
  int32_t height;     /* sensor height                                          */
  int32_t delta_x;    /* pixel radius δx >= 1 (EncoderConfig, encoder.py:52)    */
  int32_t delta_y;    /* pixel radius δy >= 1                                   */
  int32_t embed_dim;  /* D, 1..64                                               */
  int32_t hidden;     /* MLP hidden width, 0 = encoder-only handle, <= 256      */
  double delta_t;     /* time radius in seconds (slice window = 2·delta_t)      */
  int32_t device;     /* CUDA device ordinal                                    */
  int32_t mlp_mode;   /* VKM_MLP_*                                              */
} vkm_params;

typedef struct vkm_handle vkm_handle;

/* Library version (VKM_VERSION). */
int vkm_version(void);

/* Thread-local text of the last error ("" if none). */
const char* vkm_last_error(void);

/* Number of visible CUDA devices. */
int vkm_device_count(int32_t* count);

/* Create a handle: uploads the frequency vectors (f64[D] each: the bases the
 * weights were trained with, flow.py:173-174) and, when hidden > 0, the head
 * w1 (hidden x 2D row-major), b1 (hidden), w2 (2 x hidden), b2 (2), all f32. */
int vkm_create(vkm_handle** out, const vkm_params* params,
               const double* time_freqs, const double* x_freqs, const double* y_freqs,
               const float* w1, const float* b1, const float* w2, const float* b2);

void vkm_destroy(vkm_handle* h);

/* Select the MLP mode after creation (VKM_MLP_*). */
int vkm_set_mlp_mode(vkm_handle* h, int32_t mode);

/* Float64 copy of the head for precision="f64" (vkm_predict_f64[_host]).  The
 * reference promotes its head to float64 when the weights are float64 (e.g.
 * returned by train_head, flow.py:98-106, 223); without this call the f64 path
 * uses the float32 weights given to vkm_create, promoted exactly.
 * W1 (hidden, 2D) row-major [Re | Im], b1 (hidden), W2 (2, hidden), b2 (2);
 * shapes are the handle's.  Replaces nothing in the reference (its weights are
 * numpy arrays of either dtype, flow.py:48-80). */
int vkm_set_weights_f64(vkm_handle* h, const double* w1, const double* b1, const double* w2, const double* b2);

/* Per-event normal flow for every event of one slice.
 * flows_dev: (n, 2) f32 [n_x, n_y]; NaN rows for empty neighbourhoods.
 * counts_dev: (n) int32 neighbourhood sizes, or NULL. */
int vkm_predict(vkm_handle* h, const double* events_dev, int64_t n, double t_start,
                float* flows_dev, int32_t* counts_dev, void* stream);

/* Per-event features [Re(emb); Im(emb)], (n, 2D) f32. */
int vkm_encode(vkm_handle* h, const double* events_dev, int64_t n, double t_start,
               float* feats_dev, int32_t* counts_dev, void* stream);

/* Synchronous host-buffer variants: H2D of the events, the device path, D2H
 * of the results, all on the handle's internal stream. */
int vkm_predict_host(vkm_handle* h, const double* events_host, int64_t n, double t_start,
                     float* flows_host, int32_t* counts_host);
int vkm_encode_host(vkm_handle* h, const double* events_host, int64_t n, double t_start,
                    float* feats_host, int32_t* counts_host);
/* vkm_predict_host with the flows widened to float64 on the host (the type
 * NormalFlowRegressor.predict returns, estimators.py:203-206): the f32 rows
 * come back through page-locked staging in pieces and the host pool widens
 * piece i while piece i+1 is in flight. */
int vkm_predict_host_wide(vkm_handle* h, const double* events_host, int64_t n, double t_start,
                          double* flows_host, int32_t* counts_host);

/* precision="f64" (estimators.py:115, encoder.py:37-38: complex128 grid,
 * float64 features; flow.py:98-106: the head promotes the f32 weights to f64).
 * Same contract as vkm_predict / vkm_encode with float64 outputs:
 * flows (n, 2) f64 with NaN rows for empty neighbourhoods, features (n, 2D)
 * f64 [Re | Im] (NaN rows for events outside the sensor).  One slice per call. */
int vkm_predict_f64(vkm_handle* h, const double* events_dev, int64_t n, double t_start,
                    double* flows_dev, int32_t* counts_dev, void* stream);
int vkm_encode_f64(vkm_handle* h, const double* events_dev, int64_t n, double t_start,
                   double* feats_dev, int32_t* counts_dev, void* stream);
int vkm_predict_f64_host(vkm_handle* h, const double* events_host, int64_t n, double t_start,
                         double* flows_host, int32_t* counts_host);
int vkm_encode_f64_host(vkm_handle* h, const double* events_host, int64_t n, double t_start,
                        double* feats_host, int32_t* counts_host);

/* Direct summation (oracle_encode, encoder.py:413-440): for each query index
 * q into the time-sorted events_host rows, the f64 mean of
 * exp(i[(t_e-t_q)/δt·T + (x_e-x_q)/δx·X + (y_e-y_q)/δy·Y]) over the events
 * within (δx, δy) of it, emb_host (nq, D) complex128 as (re, im) pairs, and
 * the neighbourhood size.  Quadratic in the window population; a validation
 * path independent of the pooled grid (test_acceptance.py:49-86). */
int vkm_direct_encode_host(vkm_handle* h, const double* events_host, int64_t n, const int64_t* queries_host,
                           int64_t nq, double* emb_host, int32_t* counts_host);

/* Head training on the GPU (train_head / flow_loss_grads, flow.py:234-402):
 * float64 mini-batch Adam on the constraint loss with the data set resident in
 * HBM.  The host keeps the reference's control flow (RNG permutations, the
 * validation split, best-epoch selection); the device holds the features
 * (n, F) f64, the targets (n, 2) f64, the parameters W1 (H, F), b1 (H),
 * W2 (2, H), b2 (2) and the Adam moments.  All index arrays are host int64. */
typedef struct vkm_trainer vkm_trainer;
int vkm_train_create(vkm_trainer** out, int32_t device, const double* feats_host, const double* u_host, int64_t n,
                     int32_t n_features, int32_t hidden, const double* w1, const double* b1, const double* w2,
                     const double* b2, double margin, double margin_weight, double constraint_eps,
                     double learning_rate);
void vkm_train_destroy(vkm_trainer* t);
/* One epoch: mini-batches of batch_size consecutive entries of order_host, one
 * Adam step each (flow.py:364-385). */
int vkm_train_epoch(vkm_trainer* t, const int64_t* order_host, int64_t m, int32_t batch_size);
/* flow_loss (flow.py:234-248) of the current parameters on samples idx_host;
 * bad_step_out: the first Adam step whose mini-batch loss was not finite, or -1. */
int vkm_train_loss(vkm_trainer* t, const int64_t* idx_host, int64_t m, double* loss_out, int64_t* bad_step_out);
/* Keep the current parameters as the best so far. */
int vkm_train_keep(vkm_trainer* t);
/* Copy out the current (best = 0) or the kept (best = 1) parameters. */
int vkm_train_get(vkm_trainer* t, int32_t best, double* w1, double* b1, double* w2, double* b2);

/* Host-only (no device): one-pass check of an (n, >=3) f64 [t, x, y] array
 * with row stride ld doubles against the estimator's input contract
 * (validation.py:10-37, 49-65).  Returns 0 and fills *out; the caller raises
 * the reference's errors in its order (non-finite, negative t, non-integer
 * pixels, first pixel outside W x H) and sorts when !sorted. */
typedef struct vkm_event_check {
  int32_t nonfinite;
  int32_t negative_t;
  int32_t nonint;
  int32_t sorted;
  int64_t first_outside;
  int32_t outside_x, outside_y;
  double t_first, t_last;
} vkm_event_check;
int vkm_check_events(const double* events_host, int64_t n, int64_t ld, int32_t width, int32_t height,
                     vkm_event_check* out);

/* NormalFlowRegressor.predict's fast path (estimators.py:192-206): one host
 * pass checks the (n, 3) f64 rows exactly like vkm_check_events and packs
 * them for the upload; if the rows are valid, time-sorted and span at most
 * `window` (validation.py:49-65), the slice runs as vkm_predict_host_wide
 * (t_start = the first row's time) and *ran = 1; otherwise nothing runs,
 * *ran = 0 and *check holds the checks, so the caller raises the reference's
 * error (or sorts an unsorted slice and predicts).  Also *ran = 0 for slices
 * below the packed single-slice size. */
int vkm_predict_host_checked(vkm_handle* h, const double* events_host, int64_t n, double window,
                             double* flows_host, vkm_event_check* check, int32_t* ran);

/* Host utility: dst[i] = (double)src[i] for n values, split over the host
 * pool with streaming stores (the float64 results of the batch APIs). */
int vkm_widen_f32(const float* src, double* dst, int64_t n);

/* Host utility: concatenate n_arrays row blocks (rows[a] rows of ld doubles
 * at srcs[a]) into dst, split over the host pool (the staging of the batch
 * APIs' many-slice inputs). */
int vkm_concat_rows(const double* const* srcs, const int64_t* rows, int32_t n_arrays, int64_t ld, double* dst);

/* Stream windowing on the device (slice_stream, events.py:331-387):
 * vkm_window_bounds: for a time-sorted device stream (n, 3), the bounds
 *   [lo, hi) of windows [starts[i], starts[i] + window) by binary search
 *   (np.searchsorted side="left" at both edges), written to bounds_host
 *   (n_windows, 2) int64.
 * vkm_predict_windows: per-window flows for those bounds, each window with its
 *   start as time origin; the windows' rows are gathered on the device
 *   (overlapping windows share one upload of the stream), flows_dev (sum of
 *   window sizes, 2) f32 in window order.  Synchronous on `stream`. */
int vkm_window_bounds(vkm_handle* h, const double* events_dev, int64_t n, const double* starts_host,
                      int32_t n_windows, double window, int64_t* bounds_host);
int vkm_predict_windows(vkm_handle* h, const double* events_dev, int64_t n, const double* starts_host,
                        const int64_t* bounds_host, int32_t n_windows, float* flows_dev, int32_t* counts_dev,
                        void* stream);

/* Many independent slices in one call.  Slice s holds events
 * [offsets[s], offsets[s+1]) of events_dev; offsets_host has n_slices+1
 * entries; t_starts_host has n_slices entries (NAN = first event). */
int vkm_predict_batch(vkm_handle* h, const double* events_dev, const int64_t* offsets_host,
                      int32_t n_slices, const double* t_starts_host,
                      float* flows_dev, int32_t* counts_dev, void* stream);

/* Host-buffer batch: like vkm_predict_batch, but events_host / flows_host /
 * counts_host (may be NULL) are host memory.  Slices are pipelined over three
 * streams (copy-in, kernels, copy-out) with two device staging buffers, so
 * transfers overlap compute; pass page-locked buffers for the copies to be
 * asynchronous.  Returns after the last result has landed in host memory. */
int vkm_predict_batch_host(vkm_handle* h, const double* events_host, const int64_t* offsets_host,
                           int32_t n_slices, const double* t_starts_host, float* flows_host,
                           int32_t* counts_host);

/* Multi-GPU slice sharding without a collective: the
 * slices are split into contiguous ranges of about equal event counts, one
 * per handle (one handle per device, all with the same geometry and head),
 * and each range runs vkm_predict_batch_host on its own host thread.  Same
 * buffers and offsets as vkm_predict_batch_host; results land at the slices'
 * own rows.  Handles must be distinct. */
int vkm_predict_multi_host(vkm_handle* const* handles, int32_t n_handles, const double* events_host,
                           const int64_t* offsets_host, int32_t n_slices, const double* t_starts_host,
                           float* flows_host, int32_t* counts_host);

/* One oversized slice over several devices: rows
 * [row_cuts[i], row_cuts[i+1]) belong to strip i (row_cuts[0] = 0,
 * row_cuts[n_strips] = H); handle i was created for the strip plus a
 * delta_y-row event halo clipped to the sensor (height = min(H, cut[i+1] +
 * δy) - max(0, cut[i] - δy)), on its own device.  Each strip's events (rows
 * shifted to the strip) run on their handle's host thread with the slice's
 * single time origin; owned rows are written back at their input positions
 * (events outside every strip: NaN flows, count 0).  No grid exchange. */
int vkm_predict_strips_host(vkm_handle* const* handles, int32_t n_strips, const int32_t* row_cuts,
                            const double* events_host, int64_t n, double t_start, float* flows_host,
                            int32_t* counts_host);

/* Spatial split, partition side: stable (time-order preserving) selection of
 * the events of rows [y_lo, y_hi) of events_dev (n rows [t, x, y]) into
 * out_events_dev (rows rebased by -y_lo), their row indices into
 * out_index_dev and owned flags (row in [own_lo, own_hi)) into out_owned_dev;
 * *count_host receives the number selected (the call synchronizes the
 * handle's stream).  Outputs must hold n rows. */
int vkm_select_rows(vkm_handle* h, const double* events_dev, int64_t n, int32_t y_lo, int32_t y_hi, int32_t own_lo,
                    int32_t own_hi, double* out_events_dev, int64_t* out_index_dev, uint8_t* out_owned_dev,
                    int64_t* count_host);

/* Spatial split, gather side: dst_dev[index[i]] = src_dev[i] (rows of
 * row_floats floats) for every i < m with mask_dev[i] != 0 (mask may be NULL). */
int vkm_scatter_rows(vkm_handle* h, const float* src_dev, const int64_t* index_dev, const uint8_t* mask_dev,
                     int64_t m, int32_t row_floats, float* dst_dev, void* stream);

/* Parity hook: the per-pixel grid in the reference's PixelGrid layout.
 * grid_dev: (width, height, D) complex64 as interleaved f32 pairs, [x][y][d];
 * counts_dev: (width, height) int32.  pooled = 0: accumulate_grid sums;
 * pooled = 1: window sums Σ G[x+i][y+j]·table[i][j] before de-phasing. */
int vkm_grid(vkm_handle* h, const double* events_dev, int64_t n, double t_start,
             int32_t pooled, float* grid_dev, int32_t* counts_dev, void* stream);

/* Parity hook: the pixel-major event order of accumulate_grid
 * (encoder.py:255-259: order = np.argsort(flat_key, kind="stable"), the run
 * starts = exclusive cumsum of np.bincount).  start_dev: (width*height + 1)
 * int32, start[p] = first slot of pixel p = y*width + x, start[P] = in-sensor
 * events; order_dev: (n) int32 event index per slot (-1 for the trailing
 * slots of events outside the sensor). */
int vkm_pixel_order(vkm_handle* h, const double* events_dev, int64_t n, double t_start, int32_t* start_dev,
                    int32_t* order_dev, void* stream);

/* Per-kernel device timing of the last call (ms), recorded with CUDA events
 * when enabled: [0] accumulate, [1] pool, [2] gather+MLP, [3] total.
 * *n_out receives the number of kernel launches of the last call. */
int vkm_set_profiling(vkm_handle* h, int32_t enable);
int vkm_last_timings(vkm_handle* h, float* ms_out, int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* VECKM_H */
