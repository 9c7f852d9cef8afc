// Launch wrappers for the VecKM_flow kernels (internal to libveckm.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cstring>

namespace vkm {

struct DevTables {
  const float* tf;     // f32(T_c), [D8]                       (encoder.py:223-224)
  const float2* my;    // e^{i y Y_c / dy}, [H][D8] complex64   (modulation, y axis)
  const float2* mx;    // e^{i x X_c / dx}, [W][D8] complex64   (modulation, x axis)
  const float4* mxp;   // [W][D8/2] (cos c0, cos c1, sin c0, sin c1) of x X_c/dx, c0 = 2·pair (packed pairs)
  const float4* myp;   // [H][D8/2] same for y Y_c/dy
};

// Grid layouts, [plane = channel/8][pixel][64 B]:
//   complex layout  8 × (re, im) complex64          (raw grid G of k_reduce)
//   packed pairs    4 × (re c, re c+1, im c, im c+1) (x-pooled R, pooled Q):
//                   one 16-byte chunk is a channel pair in f32x2-ready form
struct GridBufs {
  float2* G;   // [planes][P][8]  pre-modulated grid M = G·e^{i(xX/δx + yY/δy)} (complex layout)
  int* C;      // [P]
  float2* Q;   // [planes][P][8]  pooled grid (packed pairs)
  int* NQ;     // [P]
};

// Pixel-sorted event order produced by the sorted K1 (k_sort.cu).  Sort
// values pack (event index, f32 time argument) so the consumers of a slot read
// one coalesced 8-byte word instead of chasing perm[] into a[].
__host__ __device__ inline uint64_t slot_pack(int32_t e, float a) {
  uint32_t ab;
  memcpy(&ab, &a, 4);
  return uint64_t(uint32_t(e)) | (uint64_t(ab) << 32);
}
__host__ __device__ inline int32_t slot_event(uint64_t v) { return int32_t(uint32_t(v)); }
__host__ __device__ inline float slot_arg(uint64_t v) {
  const uint32_t ab = uint32_t(v >> 32);
  float a;
  memcpy(&a, &ab, 4);
  return a;
}

struct SortBufs {
  int32_t* pix;      // [n]  pixel key per event (P: outside the sensor)
  uint64_t* val;     // [n]  slot_pack(e, a) per event (sort values)
  int* start;        // [P+1] exclusive scan of the counts (start[P] = valid events)
  uint64_t* val_s;   // [n]  slot -> slot_pack(event, a), stable pixel-major order
  int32_t* pix_s;    // [n]  slot -> pixel
  unsigned long long* scan_state;   // [scan_state_words(P)] k_scan tile states (zeroed once)
  int32_t* rank;     // [n]   event's arrival rank inside its pixel (k_prep's histogram atomic)
  int* longlist;     // [P]   pixels whose run is longer than one warp sort
  int* longcount;    // [1]   long-run count
  // dense slices (radix and row-bucket paths, k_sort.cu): the second key/value
  // buffers, the per-(digit | row, tile) count table + its scan, and the
  // table scan's tile states
  uint64_t* bkt;                     // [n]
  int* msd_tab;                      // [2 * msd_tab_words(n)]
  unsigned long long* msd_state;     // [scan_state_words(msd_tab_words(n))]
};
size_t msd_tab_words(int64_t n);     // per-(row, event tile) counters for n events, rows <= kMsdMaxRows

// Slices processed by one launch sequence (batched fused path): slice b owns
// events [off[b], off[b+1]) and the pixel block [b·P, (b+1)·P) of a virtual
// W x (nb·H) sensor whose windows never cross slice borders.  t0[b] = NaN
// reads the slice's first event.  Passed by value as a kernel parameter.
constexpr int kMaxBatch = 64;
// Run-time flavour of the hot kernels' sin/cos (VKM_SINCOS=poly|mufu, default
// mufu; read per launch).
bool sincos_mufu();
struct SliceTab {
  int32_t nb;
  int64_t off[kMaxBatch + 1];
  double t0[kMaxBatch];
};

struct MlpDev {
  const float* w1;   // [hidden][2*D8] padded: [Re(0..D8) | Im(0..D8)]
  const float* b1;   // [hidden]
  const float* w2;   // [2][hidden]
  const float* b2;   // [2]
  int hidden;
  // float64 head (precision="f64" with float64 weights, vkm_set_weights_f64):
  // W1ᵀ [2D][hidden] | b1 [hidden] | W2 [2][hidden] | b2 [2] in one buffer, or null
  const double* w64 = nullptr;
};

// K1 (sorted): prep + scan + counting scatter + run ordering of (pixel, slot_pack) pairs.
// Returns the number of kernel launches.  C must hold P+1 ints.
// Keys live in [0, nb·W·H]; nb·W·H + 1 counters in g.C.  Events are either
// the reference's (n, 3) f64 rows (ev) or host-packed 8-byte records
// (packed != null): .x = f32 bits of a = f32((t - t0)/δt) computed on the host
// in f64 exactly like the device, .y = x | y << 16 (0xFFFF: not an in-sensor
// integer pixel).
int launch_sort_events(const double* ev, const uint2* packed, const SliceTab& st, double delta_t, int W, int H,
                       const GridBufs& g, const SortBufs& sb, float* flows_invalid, int32_t* counts_invalid,
                       cudaStream_t s);
// K1 reduce, raw grid: per-pixel time-ordered sums, written pre-modulated
// (M = G·e^{i(xX/δx + yY/δy)}) to g.G.  Used by the split pooling path and the
// raw-grid parity hook.
void launch_reduce_raw(const DevTables& tb, int W, int H, int D8, const GridBufs& g, const SortBufs& sb,
                       cudaStream_t s);
// K1 reduce fused with the x window (D8 == 64, dx <= kMaxFusedDx):
//   R[y][x] = e^{i y Y/δy} · Σ_{|i|<=δx} G[y][x+i]·e^{i (x+i) X/δx}   -> R
bool reduce_x_supported(int D8, int dx);
void launch_reduce_x(const DevTables& tb, int W, int H, int nb, int dx, const SortBufs& sb, float2* R,
                     int num_sms, cudaStream_t s);
size_t scan_state_words(int64_t P);   // k_scan tile-state words for P pixels
uint32_t next_scan_epoch();           // epoch tag of the next single-pass scan launch
// order[slot] = event of each slot of val_s (-1 from *valid on)
void launch_slot_events(const uint64_t* val_s, const int* valid, int64_t n, int32_t* order, cudaStream_t s);
// K2 (split): box sum of the pre-modulated grid M (y-pass M -> R, x-pass +
// demodulation R -> Qout); Qout may alias M (k_pool.cu).
void launch_pool_split(const DevTables& tb, int W, int H, int D8, int dx, int dy, float2* M, float2* R,
                       float2* Qout, cudaStream_t s);
// K2 (fused path): y window of the x-pooled R plus full demodulation
//   Q[y][x] = conj(e^{i(xX/δx + yY/δy)}) · Σ_{|j|<=δy} R[y+j][x]
void launch_pool_y_demod(const DevTables& tb, int W, int H, int nb, int D8, int dy, const float2* R, float2* Q,
                         cudaStream_t s);
void launch_pool_count(int W, int H, int nb, int dx, int dy, const GridBufs& g, cudaStream_t s);
// K3a: gather Q at each event, de-phase, divide by the count -> features.
// Row e gets Re at out[e*ld + c] and Im at out[e*ld + im_off + c] for c < Dout.
void launch_features(const double* ev, int64_t n, double t0, double delta_t, const DevTables& tb,
                     int W, int H, int D8, int Dout, const GridBufs& g, float* out, int ld, int im_off,
                     int32_t* counts_out, cudaStream_t s);
// K3b: FFMA two-layer head on padded features [n][2*D8] -> flows [n][2].
void launch_mlp_ffma(const float* feats, const int32_t* counts, int64_t n, int D8, const MlpDev& m,
                     float* flows, cudaStream_t s);
// precision="f64" path (k_f64.cu).  Tables in f64: T [D8] (0 for padded
// channels), e^{i x X_c/δx} [W][D8], e^{i y Y_c/δy} [H][D8].  Buffers double2 [P][D8].
struct F64Tables {
  const double* T;
  const double2* mx;
  const double2* my;
};
// sorted slots (sb) + counts -> pooled f64 grid in bufA (bufB scratch)
void launch_encode64(const F64Tables& t, const double* ev, int64_t n, double t0, double delta_t, int W, int H, int D,
                     int D8, int dx, int dy, const SortBufs& sb, const int* NQ, double2* bufA, double2* bufB,
                     cudaStream_t s);
void launch_features64(const F64Tables& t, const double* ev, int64_t n, double t0, double delta_t, int W, int H,
                       int D, int D8, const double2* Q, const int* NQ, double* feats, int32_t* counts,
                       cudaStream_t s);
void launch_predict64(const F64Tables& t, const double* ev, int64_t n, double t0, double delta_t, int W, int H, int D,
                      int D8, const double2* Q, const int* NQ, const MlpDev& m, double* flows, int32_t* counts,
                      int num_sms, cudaStream_t s);

// Direct f64 summation per query (oracle_encode, encoder.py:413-440) over the
// sorted pixel runs of sb; X, Y, T: the raw f64 bases [D].
void launch_direct64(const double* ev, const int64_t* queries, int64_t nq, const SortBufs& sb, int W, int H, int dx,
                     int dy, double delta_t, const double* T, const double* X, const double* Y, int D, double2* emb,
                     int32_t* counts, cudaStream_t s);

// Head training (k_train.cu).  prm/m/v: packed W1ᵀ [F][H] | b1 | W2 [2][H] | b2.
size_t train_batch_smem(int F, int H);
int train_rows_per_cta();
void launch_train_batch(const double* feats, const double* u, const int64_t* idx, int64_t nb, int F, int H,
                        double* prm, double* m, double* v, double margin, double mw, double eps, int with_grads,
                        double lr, int64_t step, double* loss_part, double* g_part, int64_t* bad_step,
                        cudaStream_t s);

// Stream windowing (k_window.cu): bounds [lo, hi) of windows [start, start +
// window) in a time-sorted device stream (searchsorted side="left"), and the
// gather of the windows' rows into one batch buffer (off: exclusive offsets).
void launch_window_bounds(const double* ev, int64_t n, const double* starts_dev, int32_t nw, double window,
                          int64_t* bounds_dev, cudaStream_t s);
void launch_gather_windows(const double* ev, const int64_t* off_dev, const int64_t* lo_dev, int32_t nw,
                           int64_t total, double* out, cudaStream_t s);

// Layout conversion for the parity hook: planes -> reference [x][y][D] complex64.
// mx/my non-null: G holds the pre-modulated grid M and is demodulated on the way out.
// packed: G uses the packed-pair layout (the pooled grid Q).
void launch_grid_to_ref(const float2* G, const int* C, int W, int H, int D, int D8, const float2* mx,
                        const float2* my, bool packed, float* out_grid, int32_t* out_counts, cudaStream_t s);

// tcgen05 fused gather + de-phase + MLP (D = 64, hidden = 128).
struct TcWeights {
  const void* w1_hi;   // UMMA K-major SW128 image of W1 hi (fp16 or bf16), 32 KB
  const void* w1_lo;   // same for the lo split, 32 KB
  const float* b1;     // [128]
  const float* w2;     // [2][128]
  const float* b2;     // [2]
  float w_scale;       // power-of-two pre-scale folded into the W1 images
};
// Tiles run over the pixel-sorted slots of SortBufs (sequential pooled-grid reads).
// H is the (virtual, nb·H for a batch) grid height.
void launch_gather_mlp_tc(int64_t n, const DevTables& tb, int W, int H, const GridBufs& g, const SortBufs& sb,
                          const TcWeights& w, int mode, float* flows, int32_t* counts_out, int num_sms,
                          cudaStream_t s);
// Spatial split (k_split.cu): stable selection of the events of rows
// [y_lo, y_hi) with rows rebased by -y_lo, their global indices and an owned
// flag for rows [own_lo, own_hi); count_dev receives the number selected.
// Stable selection of the events with y in [y_lo, y_hi) (single pass with
// decoupled look-back; state = select_rows_state_words(n) words, zeroed once):
// sel = their indices, out = their rows with y - y_lo, owned = y in [own_lo,
// own_hi); *count_dev = how many.
size_t select_rows_state_words(int64_t n);
void launch_select_rows(const double* ev, int64_t n, int y_lo, int y_hi, int own_lo, int own_hi,
                        unsigned long long* state, int64_t* sel, int64_t* count_dev, double* out, uint8_t* owned,
                        cudaStream_t s);
// dst[index[i]] = src[i] (rows of row_floats floats) where mask[i] != 0 (mask may be null).
void launch_scatter_rows(const float* src, const int64_t* index, const uint8_t* mask, int64_t m, int row_floats,
                         float* dst, cudaStream_t s);

// K position of feature f ([Re(0..63) | Im(0..63)]) in the tensor-core head's
// operand images: channel pairs (Re c, Re c+1, Im c, Im c+1) are contiguous.
int feature_kpos(int f);
// Host helper: build the UMMA smem image (K-major, 128B swizzle) of a 128x128 fp16/bf16 matrix.
void build_umma_image_kmajor_128x128(const uint16_t* rowmajor, uint16_t* image);

}  // namespace vkm
