// C-ABI of libveckm.so (declared in include/veckm.h).  Host-side orchestration
// of the VecKM_flow kernels: handle/scratch management, parameter checks with
// the reference's error semantics, stream-ordered launches, host-buffer
// variants and per-kernel CUDA-event timing.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <limits>
#include <mutex>
#include <thread>
#include <cstdint>
#include <utility>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/veckm.h"
#include "vkm_kernels.cuh"
#include "host_pool.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

#define VKM_CK(x)                                                                              \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? VKM_EOOM : VKM_ECUDA;                    \
      return fail(code_, std::string(#x) + ": " + cudaGetErrorString(e_));                     \
    }                                                                                          \
  } while (0)

int round_d8(int D) {
  int d = 8;
  while (d < D) d <<= 1;
  return d;
}


}  // namespace

struct vkm_handle {
  vkm_params p{};
  int D = 0, D8 = 0, planes = 0, hidden = 0, mode = VKM_MLP_FP32, num_sms = 148;
  int64_t P = 0;
  cudaStream_t stream = nullptr;
  // constants
  float* tf = nullptr;
  float2* my = nullptr;
  float2* mx = nullptr;
  float4* mxp = nullptr;
  float4* myp = nullptr;
  double* xyz64 = nullptr;  // raw f64 bases T | X | Y [3][D] (direct summation)
  double* t64 = nullptr;    // precision="f64" tables (k_f64.cu)
  double2* mx64 = nullptr;
  double2* my64 = nullptr;
  double2* g64a = nullptr;   // f64 grid buffers [P][D8], grown on the first f64 call
  double2* g64b = nullptr;
  int64_t g64_cap = 0;
  double* out64 = nullptr;   // f64 host-variant output staging
  size_t out64_cap = 0;
  double* win_ev = nullptr;     // stream windowing: gathered window rows (n, 3)
  size_t win_ev_cap = 0;
  int64_t* win_aux = nullptr;   // window starts (as doubles), bounds, offsets, lows
  size_t win_aux_cap = 0;
  float* w1p = nullptr;  // [hidden][2*D8] padded
  float* b1 = nullptr;
  float* w2 = nullptr;
  float* b2 = nullptr;
  double* w64 = nullptr;  // float64 head W1ᵀ | b1 | W2 | b2 (vkm_set_weights_f64), or null
  void* w1_f16_hi = nullptr;
  void* w1_f16_lo = nullptr;
  void* w1_bf16 = nullptr;
  float w_scale_f16 = 1.f;
  bool tc_ok = false;  // D == 64 && hidden == 128
  bool force_split = false;  // VKM_POOL=split: raw grid + two-pass pooling (A/B and parity)
  int64_t grid_cap = 0;      // pixels the grid scratch holds (nb·W·H of the largest batch so far)
  int64_t batch_pixels = int64_t(1) << 22;   // pixel budget of one batched launch sequence
  // scratch
  vkm::SortBufs sb{};
  size_t sort_cap = 0;
  float2* G = nullptr;
  int* C = nullptr;
  float2* Q = nullptr;
  int* NQ = nullptr;
  float* feats = nullptr;
  size_t feats_cap = 0;
  int32_t* cnt_scratch = nullptr;
  size_t cnt_cap = 0;
  double* ev_stage = nullptr;
  size_t ev_cap = 0;
  float* out_stage = nullptr;
  size_t out_cap = 0;
  int32_t* cnt_stage = nullptr;
  size_t cnt_stage_cap = 0;
  // pipelined host batches: copy-in / copy-out streams, two staging slots
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t in_ready[2] = {nullptr, nullptr}, computed[2] = {nullptr, nullptr}, out_done[2] = {nullptr, nullptr};
  double* pev[2] = {nullptr, nullptr};
  size_t pev_cap[2] = {0, 0};
  float* pout[2] = {nullptr, nullptr};
  size_t pout_cap[2] = {0, 0};
  int32_t* pcnt[2] = {nullptr, nullptr};
  size_t pcnt_cap[2] = {0, 0};
  uint2* hpack[2] = {nullptr, nullptr};   // page-locked packed-event staging (host)
  uint8_t* hout = nullptr;                // page-locked result staging of the single-slice host calls
  size_t hout_cap = 0;                    // bytes
  cudaEvent_t dl_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // download pieces
  size_t hpack_cap[2] = {0, 0};
  vkm_host::HostPool* pool = nullptr;
  uint8_t* sel_temp = nullptr;   // vkm_select_rows: count + look-back tile states
  size_t sel_temp_cap = 0;
  // timing
  bool profiling = false;
  cudaEvent_t evt[4] = {nullptr, nullptr, nullptr, nullptr};
  // side stream: the count pooling overlaps k_reduce_x (it only needs the counts)
  cudaStream_t s_side = nullptr;
  cudaEvent_t e_fork = nullptr, e_join = nullptr;
  bool have_timing = false;
  int last_launches = 0;
};

namespace {

template <class T>
int grow(T** ptr, size_t* cap, size_t need) {
  if (*cap >= need) return VKM_OK;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  *cap = 0;
  const size_t alloc = std::max<size_t>(need, 1);
  VKM_CK(cudaMalloc(ptr, alloc * sizeof(T)));
  *cap = alloc;
  return VKM_OK;
}

vkm::DevTables tables(const vkm_handle* h) { return vkm::DevTables{h->tf, h->my, h->mx, h->mxp, h->myp}; }
vkm::GridBufs bufs(const vkm_handle* h) { return vkm::GridBufs{h->G, h->C, h->Q, h->NQ}; }

void rec(vkm_handle* h, int i, cudaStream_t s) {
  if (h->profiling) cudaEventRecord(h->evt[i], s);
}

struct HostTrace;
thread_local HostTrace* g_trace = nullptr;   // the running call's trace (download pieces mark into it)

// VKM_TRACE=1: the drop-in host call prints its host-side stage times and the
// device span of its copies and kernels to stderr (diagnostics only).
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  std::string out;
  cudaEvent_t ev[12] = {};
  const char* ev_name[12] = {};
  int nev = 0;
  HostTrace() : on([] {
    const char* e = std::getenv("VKM_TRACE");
    return e && *e == '1';
  }()) {
    if (on) {
      t0 = std::chrono::steady_clock::now();
      g_trace = this;
    }
  }
  void mark(const char* what) {
    if (!on) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    char b[96];
    std::snprintf(b, sizeof b, " %s=%.0f", what, us);
    out += b;
  }
  void dev(const char* what, cudaStream_t s) {
    if (!on || nev == 12) return;
    cudaEventCreate(&ev[nev]);
    cudaEventRecord(ev[nev], s);
    ev_name[nev++] = what;
  }
  ~HostTrace() {
    if (!on) return;
    std::string d;
    for (int i = 1; i < nev; ++i) {
      float ms = 0.f;
      cudaEventSynchronize(ev[i]);
      cudaEventElapsedTime(&ms, ev[0], ev[i]);
      char b[96];
      std::snprintf(b, sizeof b, " %s=%.0f", ev_name[i], ms * 1e3f);
      d += b;
    }
    for (int i = 0; i < nev; ++i) cudaEventDestroy(ev[i]);
    g_trace = nullptr;
    std::fprintf(stderr, "[vkm trace] host us:%s | device us from %s:%s\n", out.c_str(), nev ? ev_name[0] : "-",
                 d.c_str());
  }
};

int ensure_sort(vkm_handle* h, int64_t n, int64_t Pv) {
  const size_t cap = size_t(std::max<int64_t>(n, 1));
  (void)Pv;
  if (h->sort_cap >= cap) return VKM_OK;
  void* arrs[] = {h->sb.pix, h->sb.val, h->sb.val_s, h->sb.pix_s, h->sb.rank, h->sb.bkt, h->sb.msd_tab,
                  h->sb.msd_state};
  for (void* p : arrs)
    if (p) cudaFree(p);
  h->sb.pix = nullptr; h->sb.val = nullptr; h->sb.val_s = nullptr; h->sb.pix_s = nullptr; h->sb.rank = nullptr;
  h->sb.bkt = nullptr; h->sb.msd_tab = nullptr; h->sb.msd_state = nullptr;
  h->sort_cap = 0;
  VKM_CK(cudaMalloc(&h->sb.pix, 4 * cap));
  VKM_CK(cudaMalloc(&h->sb.rank, 4 * cap));
  VKM_CK(cudaMalloc(&h->sb.val, 8 * cap));
  VKM_CK(cudaMalloc(&h->sb.val_s, 8 * cap));
  VKM_CK(cudaMalloc(&h->sb.pix_s, 4 * cap));
  VKM_CK(cudaMalloc(&h->sb.bkt, 8 * cap));
  {
    const size_t tw = vkm::msd_tab_words(int64_t(cap)), sw = vkm::scan_state_words(int64_t(tw));
    VKM_CK(cudaMalloc(&h->sb.msd_tab, 2 * sizeof(int) * tw));
    VKM_CK(cudaMalloc(&h->sb.msd_state, sizeof(unsigned long long) * sw));
    VKM_CK(cudaMemset(h->sb.msd_state, 0, sizeof(unsigned long long) * sw));   // epoch 0: never published
  }
  h->sort_cap = cap;
  return VKM_OK;
}

// Grid scratch for Pv = nb·W·H pixels: two grids of 64 B/pixel per plane,
// counts, pooled counts, run starts and the scan scratch.
int ensure_grid(vkm_handle* h, int64_t Pv) {
  if (h->grid_cap >= Pv) return VKM_OK;
  void* arrs[] = {h->G, h->Q, h->C, h->NQ, h->sb.start, h->sb.scan_state, h->sb.longlist, h->sb.longcount};
  for (void* p : arrs)
    if (p) cudaFree(p);
  h->G = h->Q = nullptr;
  h->C = h->NQ = h->sb.start = h->sb.longlist = h->sb.longcount = nullptr;
  h->sb.scan_state = nullptr;
  h->grid_cap = 0;
  VKM_CK(cudaMalloc(&h->G, sizeof(float2) * 8 * h->planes * Pv));
  VKM_CK(cudaMalloc(&h->Q, sizeof(float2) * 8 * h->planes * Pv));
  VKM_CK(cudaMalloc(&h->C, sizeof(int) * (Pv + 1)));
  VKM_CK(cudaMalloc(&h->NQ, sizeof(int) * Pv));
  VKM_CK(cudaMalloc(&h->sb.start, sizeof(int) * (Pv + 1)));
  VKM_CK(cudaMalloc(&h->sb.longlist, sizeof(int) * Pv));
  VKM_CK(cudaMalloc(&h->sb.longcount, sizeof(int)));
  {
    const size_t words = vkm::scan_state_words(Pv);
    VKM_CK(cudaMalloc(&h->sb.scan_state, sizeof(unsigned long long) * words));
    VKM_CK(cudaMemset(h->sb.scan_state, 0, sizeof(unsigned long long) * words));   // epoch 0: never published
  }
  h->grid_cap = Pv;
  return VKM_OK;
}

vkm::SliceTab one_slice(int64_t n, double t0) {
  vkm::SliceTab st{};
  st.nb = 1;
  st.off[0] = 0;
  st.off[1] = n;
  st.t0[0] = t0;
  return st;
}

bool use_tc(const vkm_handle* h) { return (h->mode == VKM_MLP_F16X3 || h->mode == VKM_MLP_BF16) && h->tc_ok; }
bool fused_ok(const vkm_handle* h) { return !h->force_split && vkm::reduce_x_supported(h->D8, h->p.delta_x); }
// Several slices per launch sequence: the fused encoder and the tensor-core head.
bool batchable(const vkm_handle* h) { return use_tc(h) && fused_ok(h); }

// K1 + K2 for the slices of st on stream s.  pooled = 0 leaves the raw
// pre-modulated grid in G (parity hook, one slice); otherwise the pooled grid
// ends in Q.  More than one slice requires the fused path.
int encode_core(vkm_handle* h, const double* ev, const vkm::SliceTab& st, int pooled, cudaStream_t s, int* launches,
                float* flows_invalid = nullptr, int32_t* counts_invalid = nullptr, const uint2* packed = nullptr) {
  const int W = h->p.width, H = h->p.height, nb = st.nb;
  const int64_t n = st.off[nb], Pv = h->P * nb;
  int rc = ensure_grid(h, Pv);
  if (!rc) rc = ensure_sort(h, n, Pv);
  if (rc) return rc;
  *launches += vkm::launch_sort_events(ev, packed, st, h->p.delta_t, W, H, bufs(h), h->sb, flows_invalid,
                                       counts_invalid, s);
  if (pooled && fused_ok(h)) {
    // count pooling on the side stream (needs only the counts), overlapping
    // the reduction; x window fused into the reduction: R -> G, then y window
    // + demodulation G -> Q; join before the head reads NQ
    VKM_CK(cudaEventRecord(h->e_fork, s));
    VKM_CK(cudaStreamWaitEvent(h->s_side, h->e_fork, 0));
    vkm::launch_pool_count(W, H, nb, h->p.delta_x, h->p.delta_y, bufs(h), h->s_side);
    VKM_CK(cudaEventRecord(h->e_join, h->s_side));
    vkm::launch_reduce_x(tables(h), W, H, nb, h->p.delta_x, h->sb, h->G, h->num_sms, s);
    *launches += 1;
    VKM_CK(cudaGetLastError());
    rec(h, 1, s);
    VKM_CK(cudaStreamWaitEvent(s, h->e_join, 0));   // long done: it ran beside the reduction
    vkm::launch_pool_y_demod(tables(h), W, H, nb, h->D8, h->p.delta_y, h->G, h->Q, s);
    *launches += 2;
    VKM_CK(cudaGetLastError());
  } else {
    if (nb != 1) return fail(VKM_EINVAL, "internal: batched slices need the fused encoder");
    vkm::launch_reduce_raw(tables(h), W, H, h->D8, bufs(h), h->sb, s);
    *launches += 1;
    VKM_CK(cudaGetLastError());
    rec(h, 1, s);
    if (pooled) {
      // y-pass M(G) -> R(Q), x-pass R(Q) -> pooled(G); then swap so Q names the pooled grid
      vkm::launch_pool_split(tables(h), W, H, h->D8, h->p.delta_x, h->p.delta_y, h->G, h->Q, h->G, s);
      std::swap(h->G, h->Q);
      vkm::launch_pool_count(W, H, 1, h->p.delta_x, h->p.delta_y, bufs(h), s);
      *launches += 3;
      VKM_CK(cudaGetLastError());
    }
  }
  rec(h, 2, s);
  return VKM_OK;
}

// Flows for the slices of st (one launch sequence).
int predict_chunk(vkm_handle* h, const double* ev, const vkm::SliceTab& st, float* flows, int32_t* counts,
                  cudaStream_t s, int* launches, const uint2* packed = nullptr) {
  const bool tc = use_tc(h);
  if (packed && !tc) return fail(VKM_EINVAL, "internal: packed events need the tensor-core head");
  int rc = encode_core(h, ev, st, 1, s, launches, flows, counts, packed);
  if (rc) return rc;
  const int64_t n = st.off[st.nb];
  if (n <= 0) return VKM_OK;
  const int W = h->p.width, H = h->p.height;
  if (tc) {
    vkm::TcWeights tw{h->mode == VKM_MLP_BF16 ? h->w1_bf16 : h->w1_f16_hi, h->w1_f16_lo, h->b1, h->w2, h->b2,
                      h->mode == VKM_MLP_BF16 ? 1.f : h->w_scale_f16};
    vkm::launch_gather_mlp_tc(n, tables(h), W, H * st.nb, bufs(h), h->sb, tw, h->mode, flows, counts, h->num_sms,
                              s);
    *launches += 1;
  } else {
    if (st.nb != 1) return fail(VKM_EINVAL, "internal: batched slices need the tensor-core head");
    const double t0 = st.t0[0];
    rc = grow(&h->feats, &h->feats_cap, size_t(n) * 2 * h->D8);
    if (rc) return rc;
    int32_t* cn = counts;
    if (!cn) {
      rc = grow(&h->cnt_scratch, &h->cnt_cap, size_t(n));
      if (rc) return rc;
      cn = h->cnt_scratch;
    }
    if (h->D8 != h->D) VKM_CK(cudaMemsetAsync(h->feats, 0, sizeof(float) * size_t(n) * 2 * h->D8, s));
    vkm::launch_features(ev, n, t0, h->p.delta_t, tables(h), W, H, h->D8, h->D, bufs(h), h->feats, 2 * h->D8,
                         h->D8, cn, s);
    vkm::MlpDev md{h->w1p, h->b1, h->w2, h->b2, h->hidden};
    vkm::launch_mlp_ffma(h->feats, cn, n, h->D8, md, flows, s);
    *launches += 2;
  }
  VKM_CK(cudaGetLastError());
  return VKM_OK;
}

int predict_one(vkm_handle* h, const double* ev, int64_t n, double t0, float* flows, int32_t* counts, cudaStream_t s,
                int* launches) {
  return predict_chunk(h, ev, one_slice(n, t0), flows, counts, s, launches);
}

// Group consecutive slices [s0, s1) into one SliceTab (offsets relative to
// offsets[s0]); empty slices are skipped; at most max_events events unless a
// single slice is larger.  Returns s1.
int next_chunk(const vkm_handle* h, const int64_t* offsets, int32_t n_slices, const double* t_starts, int s0,
               vkm::SliceTab& st, int64_t max_events = INT64_MAX) {
  const int maxb = batchable(h) ? int(std::max<int64_t>(1, std::min<int64_t>(vkm::kMaxBatch,
                                                                             h->batch_pixels / h->P)))
                                : 1;
  st = vkm::SliceTab{};
  st.nb = 0;
  const int64_t base = offsets[s0];
  int s = s0;
  for (; s < n_slices && st.nb < maxb; ++s) {
    if (offsets[s + 1] == offsets[s]) continue;
    if (st.nb > 0 && offsets[s + 1] - base > max_events) break;   // keep chunks small enough to pipeline
    st.off[st.nb] = offsets[s] - base;
    st.t0[st.nb] = t_starts ? t_starts[s] : NAN;
    ++st.nb;
  }
  st.off[st.nb] = offsets[s] - base;
  return s;
}

}  // namespace
namespace vkm_host {
// host_pack.cpp: vectorised packing of f64 [t, x, y] rows into 8-byte records
void pack_events(const double* rows, int64_t m, double t0, double dt, int W, int H, uint32_t* out);
void widen_f32(const float* src, double* dst, int64_t m);
void widen_f32_wc(const float* src, double* dst, int64_t m);
void copy_wc(const void* src, void* dst, size_t bytes);
}  // namespace vkm_host
namespace {

// Pack the events of one chunk into 8-byte records (see launch_sort_events):
// a = f32((t - t0)/δt) in f64 exactly like k_prep, x | y << 16, 0xFFFF... for
// events that are not integer pixels inside the sensor.
void pack_chunk(vkm_handle* h, const double* ev, const int64_t* offsets, const double* t_starts, int s0,
                const vkm::SliceTab& st, uint2* out) {
  const int64_t base = offsets[s0];
  const double dt = h->p.delta_t;
  const int W = h->p.width, H = h->p.height;
  // the slice index of chunk slice b in the caller's numbering (empty slices were skipped)
  std::vector<int> sidx(st.nb);
  for (int s = s0, b = 0; b < st.nb; ++s)
    if (offsets[s + 1] > offsets[s] && offsets[s] - base == st.off[b]) sidx[b++] = s;
  const int64_t n = st.off[st.nb];
  if (!h->pool) h->pool = new vkm_host::HostPool(vkm_host::default_pool_threads());
  const int parts = std::max(1, std::min<int>(4 * h->pool->size(), int((n + 65535) / 65536)));
  h->pool->run(parts, [&](int part) {
    const int64_t lo = n * part / parts, hi = n * (part + 1) / parts;
    for (int b = 0; b < st.nb; ++b) {   // the part's events, one slice (one t0) at a time
      const int64_t s_lo = std::max(lo, st.off[b]), s_hi = std::min(hi, st.off[b + 1]);
      if (s_lo >= s_hi) continue;
      const double t0 = (t_starts && !std::isnan(t_starts[sidx[b]])) ? t_starts[sidx[b]] : ev[3 * (base + st.off[b])];
      vkm_host::pack_events(ev + 3 * (base + s_lo), s_hi - s_lo, t0, dt, W, H, reinterpret_cast<uint32_t*>(out + s_lo));
    }
  });
}

// Pack events [lo, hi) of one slice (time origin t0) on the host pool.
// host-pool granularity of the single-slice packing: events per part
// (VKM_PACK_GRAIN) and pieces per upload (VKM_SINGLE_PIECES)
int64_t pack_grain() {
  static const int64_t g = [] {
    const char* e = std::getenv("VKM_PACK_GRAIN");
    return e ? std::max<int64_t>(1024, std::atoll(e)) : int64_t(8192);
  }();
  return g;
}
int single_pieces(int64_t n) {
  static const int p = [] {
    const char* e = std::getenv("VKM_SINGLE_PIECES");
    return e ? std::max(1, std::min(16, std::atoi(e))) : 4;
  }();
  return int(std::min<int64_t>(p, (n + (1 << 17) - 1) >> 17));
}
void pack_range(vkm_handle* h, const double* ev, int64_t lo, int64_t hi, double t0, uint2* out) {
  if (!h->pool) h->pool = new vkm_host::HostPool(vkm_host::default_pool_threads());
  const int64_t m = hi - lo;
  const int parts = std::max(1, std::min<int>(h->pool->size(), int((m + pack_grain() - 1) / pack_grain())));
  h->pool->run(parts, [&](int part) {
    const int64_t a = lo + m * part / parts, b = lo + m * (part + 1) / parts;
    if (b > a)
      vkm_host::pack_events(ev + 3 * a, b - a, t0, h->p.delta_t, h->p.width, h->p.height,
                            reinterpret_cast<uint32_t*>(out + a));
  });
}

// Single-slice host calls: pageable rows -> 8-byte records in page-locked
// staging (host pool), copied in pieces so packing piece i+1 overlaps the
// copy of piece i.  A pageable 24-byte-per-event copy runs at ~20 GB/s; the
// packed one moves a third of the bytes at the pinned rate.
bool host_staged(int64_t n) {
  static const int64_t min_events = [] {   // VKM_HOST_PACK_SINGLE: minimum events (0 = off)
    const char* e = std::getenv("VKM_HOST_PACK_SINGLE");
    return e ? int64_t(std::atoll(e)) : int64_t(1) << 17;
  }();
  return min_events > 0 && n >= min_events;
}
bool single_pack(const vkm_handle* h, int64_t n) {
  return host_staged(n) && batchable(h) && h->p.width < 65535 && h->p.height < 65535;
}

int upload_packed(vkm_handle* h, const double* ev_host, int64_t n, double t0, cudaStream_t s, uint2** dev) {
  if (h->hpack_cap[0] < size_t(n)) {
    if (h->hpack[0]) cudaFreeHost(h->hpack[0]);
    h->hpack[0] = nullptr;
    h->hpack_cap[0] = 0;
    VKM_CK(cudaHostAlloc(&h->hpack[0], sizeof(uint2) * size_t(n), cudaHostAllocDefault));
    h->hpack_cap[0] = size_t(n);
  }
  int rc = grow(&h->ev_stage, &h->ev_cap, size_t(n) * 3);   // n uint2 fit in 3n doubles
  if (rc) return rc;
  uint2* d = reinterpret_cast<uint2*>(h->ev_stage);
  const int pieces = int(std::min<int64_t>(4, (n + (1 << 17) - 1) >> 17));
  for (int i = 0; i < pieces; ++i) {
    const int64_t lo = n * i / pieces, hi = n * (i + 1) / pieces;
    pack_range(h, ev_host, lo, hi, t0, h->hpack[0]);
    VKM_CK(cudaMemcpyAsync(d + lo, h->hpack[0] + lo, sizeof(uint2) * (hi - lo), cudaMemcpyHostToDevice, s));
  }
  *dev = d;
  return VKM_OK;
}

// D2H of `bytes` bytes through page-locked staging, in up to four pieces:
// consume(lo, hi) (on the host pool, byte range of the result) runs for
// piece i while piece i+1 is in flight.  Returns with every piece consumed.
// The result staging is write-combining memory, read back with streaming
// loads: the CPU never caches its lines, so the next call's D2H does not wait
// on snoops of lines the widening left in the cores' caches (first 2-MB piece
// 46 instead of 110-160 us).  VKM_HOUT_WC=0: ordinary page-locked memory.
bool hout_wc() {
  static const bool v = [] {
    const char* e = std::getenv("VKM_HOUT_WC");
    return !(e && e[0] == '0');
  }();
  return v;
}

template <class Consume>
int download_staged(vkm_handle* h, const void* dev, size_t bytes, size_t align, cudaStream_t s, Consume consume) {
  if (h->hout_cap < bytes) {
    if (h->hout) cudaFreeHost(h->hout);
    h->hout = nullptr;
    h->hout_cap = 0;
    VKM_CK(cudaHostAlloc(&h->hout, bytes, hout_wc() ? cudaHostAllocWriteCombined : cudaHostAllocDefault));
    h->hout_cap = bytes;
  }
  for (auto& e : h->dl_ev)
    if (!e) VKM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const size_t units = bytes / align;
  static const size_t max_pieces = [] {   // VKM_DL_PIECES (A/B)
    const char* e = std::getenv("VKM_DL_PIECES");
    return e ? size_t(std::max(1, std::min(4, std::atoi(e)))) : size_t(4);
  }();
  const int pieces = int(std::max<size_t>(1, std::min<size_t>(max_pieces, (bytes + (size_t(1) << 20) - 1) >> 20)));
  auto edge = [&](int i) { return units * size_t(i) / size_t(pieces) * align; };
  for (int i = 0; i < pieces; ++i) {
    VKM_CK(cudaMemcpyAsync(h->hout + edge(i), static_cast<const uint8_t*>(dev) + edge(i), edge(i + 1) - edge(i),
                           cudaMemcpyDeviceToHost, s));
    VKM_CK(cudaEventRecord(h->dl_ev[i], s));
    if (g_trace) g_trace->dev("d2h", s);
  }
  if (!h->pool) h->pool = new vkm_host::HostPool(vkm_host::default_pool_threads());
  for (int i = 0; i < pieces; ++i) {
    const size_t lo = edge(i) / align, len = edge(i + 1) / align - lo;
    VKM_CK(cudaEventSynchronize(h->dl_ev[i]));
    if (g_trace) g_trace->mark("dl");
    const int parts = int(std::max<size_t>(1, std::min<size_t>(size_t(h->pool->size()), (len * align) >> 18)));
    h->pool->run(parts, [&](int part) {
      consume((lo + len * size_t(part) / size_t(parts)) * align, (lo + len * size_t(part + 1) / size_t(parts)) * align);
    });
  }
  return VKM_OK;
}

// m f32 values into the caller's f32 buffer (copied) or f64 buffer (widened)
int download_f32(vkm_handle* h, const float* dev, int64_t m, cudaStream_t s, float* out32, double* out64) {
  return download_staged(h, dev, sizeof(float) * size_t(m), sizeof(float), s, [&](size_t a, size_t b) {
    const float* st = reinterpret_cast<const float*>(h->hout);   // (re)allocated by download_staged
    if (out64)
      (hout_wc() ? vkm_host::widen_f32_wc : vkm_host::widen_f32)(st + a / 4, out64 + a / 4, int64_t((b - a) / 4));
    else if (hout_wc())
      vkm_host::copy_wc(h->hout + a, reinterpret_cast<uint8_t*>(out32) + a, b - a);
    else
      std::memcpy(reinterpret_cast<uint8_t*>(out32) + a, h->hout + a, b - a);
  });
}

// bytes copied as they are (float64 results)
int download_raw(vkm_handle* h, const void* dev, size_t bytes, cudaStream_t s, void* out) {
  return download_staged(h, dev, bytes, 8, s, [&](size_t a, size_t b) {
    if (hout_wc())
      vkm_host::copy_wc(h->hout + a, static_cast<uint8_t*>(out) + a, b - a);
    else
      std::memcpy(static_cast<uint8_t*>(out) + a, h->hout + a, b - a);
  });
}

int check_handle(const vkm_handle* h) {
  if (!h) return fail(VKM_EINVAL, "null vkm_handle");
  return VKM_OK;
}

}  // namespace

extern "C" {

int vkm_version(void) { return VKM_VERSION; }

const char* vkm_last_error(void) { return g_err.c_str(); }

int vkm_device_count(int32_t* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    if (count) *count = 0;
    return fail(VKM_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  if (count) *count = c;
  return VKM_OK;
}

int vkm_create(vkm_handle** out, const vkm_params* params, const double* T, const double* X, const double* Y,
               const float* w1, const float* b1, const float* w2, const float* b2) {
  if (!out || !params) return fail(VKM_EINVAL, "vkm_create: null argument");
  *out = nullptr;
  const vkm_params& p = *params;
  if (p.width < 1 || p.height < 1)
    return fail(VKM_EINVAL, "geometry must be at least 1x1, got " + std::to_string(p.width) + "x" +
                                std::to_string(p.height));
  if (int64_t(p.width) * p.height > (int64_t(1) << 30)) return fail(VKM_EINVAL, "sensor too large (> 2^30 pixels)");
  if (!(p.delta_t > 0) || !std::isfinite(p.delta_t)) return fail(VKM_EINVAL, "delta_t must be positive");
  if (p.delta_x < 1 || p.delta_y < 1) return fail(VKM_EINVAL, "pixel radii must be >= 1");
  if (p.delta_x > 100 || p.delta_y > 100) return fail(VKM_EUNSUPPORTED, "pixel radii above 100 are not supported");
  if (p.embed_dim < 1) return fail(VKM_EINVAL, "embed_dim must be >= 1");
  if (p.embed_dim > 64) return fail(VKM_EUNSUPPORTED, "embed_dim above 64 is not supported by the B200 kernels");
  if (p.hidden < 0 || p.hidden > 256) return fail(VKM_EUNSUPPORTED, "hidden width must be in [0, 256]");
  if (!T || !X || !Y) return fail(VKM_EINVAL, "frequency vectors are required");
  for (int i = 0; i < p.embed_dim; ++i)
    if (!std::isfinite(T[i]) || !std::isfinite(X[i]) || !std::isfinite(Y[i]))
      return fail(VKM_EINVAL, "frequency vectors must be finite");
  if (p.hidden > 0) {
    if (!w1 || !b1 || !w2 || !b2) return fail(VKM_EINVAL, "weights are required when hidden > 0");
    const size_t nw1 = size_t(p.hidden) * 2 * p.embed_dim;
    for (size_t i = 0; i < nw1; ++i)
      if (!std::isfinite(w1[i])) return fail(VKM_EINVAL, "weights must be finite");
    for (int i = 0; i < p.hidden; ++i)
      if (!std::isfinite(b1[i]) || !std::isfinite(w2[i]) || !std::isfinite(w2[p.hidden + i]))
        return fail(VKM_EINVAL, "weights must be finite");
    if (!std::isfinite(b2[0]) || !std::isfinite(b2[1])) return fail(VKM_EINVAL, "weights must be finite");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(VKM_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (p.device < 0 || p.device >= ndev) return fail(VKM_EINVAL, "device ordinal out of range");
  DeviceGuard dg(p.device);
  cudaDeviceProp prop;
  VKM_CK(cudaGetDeviceProperties(&prop, p.device));
  if (prop.major < 10) return fail(VKM_EUNSUPPORTED, std::string("libveckm targets sm_100a; device is ") + prop.name);

  auto* h = new vkm_handle();
  h->p = p;
  h->D = p.embed_dim;
  h->D8 = round_d8(p.embed_dim);
  h->planes = h->D8 / 8;
  h->hidden = p.hidden;
  h->P = int64_t(p.width) * p.height;
  h->num_sms = prop.multiProcessorCount;
  h->tc_ok = (h->D == 64 && h->hidden == 128);
  {
    const char* e = std::getenv("VKM_POOL");
    h->force_split = e && std::strcmp(e, "split") == 0;
  }
  h->mode = p.mlp_mode == VKM_MLP_AUTO ? (h->tc_ok ? VKM_MLP_F16X3 : VKM_MLP_FP32) : p.mlp_mode;
  if ((h->mode == VKM_MLP_F16X3 || h->mode == VKM_MLP_BF16) && !h->tc_ok) h->mode = VKM_MLP_FP32;

  auto cleanup_fail = [&](int rc) {
    vkm_destroy(h);
    return rc;
  };
#define VKM_CKH(x)                                                                             \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? VKM_EOOM : VKM_ECUDA;                    \
      return cleanup_fail(fail(code_, std::string(#x) + ": " + cudaGetErrorString(e_)));       \
    }                                                                                          \
  } while (0)

  VKM_CKH(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  VKM_CKH(cudaStreamCreateWithFlags(&h->s_side, cudaStreamNonBlocking));
  VKM_CKH(cudaEventCreateWithFlags(&h->e_fork, cudaEventDisableTiming));
  VKM_CKH(cudaEventCreateWithFlags(&h->e_join, cudaEventDisableTiming));
  for (auto& e : h->evt) VKM_CKH(cudaEventCreate(&e));

  // Frequency tables.  Modulation factors are computed in f64 and rounded once
  // (the reference's spatial table is f64 then cast, encoder.py:173-179).
  const int D8 = h->D8, W = p.width, H = p.height;
  std::vector<float> tf(D8, 0.f);
  for (int c = 0; c < h->D; ++c) tf[c] = float(T[c]);
  std::vector<float2> my(size_t(H) * D8), mx(size_t(W) * D8);
  for (int y = 0; y < H; ++y)
    for (int c = 0; c < D8; ++c) {
      const double ang = c < h->D ? (double(y) / p.delta_y) * Y[c] : 0.0;
      my[size_t(y) * D8 + c] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
    }
  for (int x = 0; x < W; ++x)
    for (int c = 0; c < D8; ++c) {
      const double ang = c < h->D ? (double(x) / p.delta_x) * X[c] : 0.0;
      mx[size_t(x) * D8 + c] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
    }
  VKM_CKH(cudaMalloc(&h->tf, sizeof(float) * D8));
  VKM_CKH(cudaMalloc(&h->my, sizeof(float2) * my.size()));
  VKM_CKH(cudaMalloc(&h->mx, sizeof(float2) * mx.size()));
  VKM_CKH(cudaMemcpy(h->tf, tf.data(), sizeof(float) * D8, cudaMemcpyHostToDevice));
  VKM_CKH(cudaMemcpy(h->my, my.data(), sizeof(float2) * my.size(), cudaMemcpyHostToDevice));
  VKM_CKH(cudaMemcpy(h->mx, mx.data(), sizeof(float2) * mx.size(), cudaMemcpyHostToDevice));
  {   // precision="f64" tables: the same angles, not rounded to f32
    std::vector<double> t64(D8, 0.0);
    for (int c = 0; c < h->D; ++c) t64[c] = T[c];
    std::vector<double2> my64(size_t(H) * D8), mx64(size_t(W) * D8);
    for (int y = 0; y < H; ++y)
      for (int c = 0; c < D8; ++c) {
        const double ang = c < h->D ? (double(y) / p.delta_y) * Y[c] : 0.0;
        my64[size_t(y) * D8 + c] = make_double2(std::cos(ang), std::sin(ang));
      }
    for (int x = 0; x < W; ++x)
      for (int c = 0; c < D8; ++c) {
        const double ang = c < h->D ? (double(x) / p.delta_x) * X[c] : 0.0;
        mx64[size_t(x) * D8 + c] = make_double2(std::cos(ang), std::sin(ang));
      }
    std::vector<double> xyz(3 * size_t(h->D));
    for (int c = 0; c < h->D; ++c) {
      xyz[c] = T[c];
      xyz[h->D + c] = X[c];
      xyz[2 * h->D + c] = Y[c];
    }
    VKM_CKH(cudaMalloc(&h->xyz64, sizeof(double) * xyz.size()));
    VKM_CKH(cudaMemcpy(h->xyz64, xyz.data(), sizeof(double) * xyz.size(), cudaMemcpyHostToDevice));
    VKM_CKH(cudaMalloc(&h->t64, sizeof(double) * D8));
    VKM_CKH(cudaMalloc(&h->mx64, sizeof(double2) * mx64.size()));
    VKM_CKH(cudaMalloc(&h->my64, sizeof(double2) * my64.size()));
    VKM_CKH(cudaMemcpy(h->t64, t64.data(), sizeof(double) * D8, cudaMemcpyHostToDevice));
    VKM_CKH(cudaMemcpy(h->mx64, mx64.data(), sizeof(double2) * mx64.size(), cudaMemcpyHostToDevice));
    VKM_CKH(cudaMemcpy(h->my64, my64.data(), sizeof(double2) * my64.size(), cudaMemcpyHostToDevice));
  }
  {   // packed-pair copies (cos c, cos c+1, sin c, sin c+1) of both tables
    auto pack = [&](const std::vector<float2>& t, int rows, std::vector<float4>& out) {
      out.resize(size_t(rows) * (D8 / 2));
      for (int r = 0; r < rows; ++r)
        for (int q = 0; q < D8 / 2; ++q) {
          const float2 a = t[size_t(r) * D8 + 2 * q], b = t[size_t(r) * D8 + 2 * q + 1];
          out[size_t(r) * (D8 / 2) + q] = make_float4(a.x, b.x, a.y, b.y);
        }
    };
    std::vector<float4> mxp, myp;
    pack(mx, W, mxp);
    pack(my, H, myp);
    VKM_CKH(cudaMalloc(&h->mxp, sizeof(float4) * mxp.size()));
    VKM_CKH(cudaMalloc(&h->myp, sizeof(float4) * myp.size()));
    VKM_CKH(cudaMemcpy(h->mxp, mxp.data(), sizeof(float4) * mxp.size(), cudaMemcpyHostToDevice));
    VKM_CKH(cudaMemcpy(h->myp, myp.data(), sizeof(float4) * myp.size(), cudaMemcpyHostToDevice));
  }

  // Grid scratch for one slice (grown on demand for batches): two plane sets
  // of 64 B/pixel plus int32 counts (516 B/pixel at D=64).
  if (int rc = ensure_grid(h, h->P)) return cleanup_fail(rc);
  {
    const char* e = std::getenv("VKM_BATCH_PIXELS");
    if (e && std::atoll(e) > 0) h->batch_pixels = std::atoll(e);
  }


  if (h->hidden > 0) {
    const int hid = h->hidden, D = h->D;
    std::vector<float> w1p(size_t(hid) * 2 * D8, 0.f);
    for (int r = 0; r < hid; ++r)
      for (int c = 0; c < D; ++c) {
        w1p[size_t(r) * 2 * D8 + c] = w1[size_t(r) * 2 * D + c];
        w1p[size_t(r) * 2 * D8 + D8 + c] = w1[size_t(r) * 2 * D + D + c];
      }
    VKM_CKH(cudaMalloc(&h->w1p, sizeof(float) * w1p.size()));
    VKM_CKH(cudaMalloc(&h->b1, sizeof(float) * hid));
    VKM_CKH(cudaMalloc(&h->w2, sizeof(float) * 2 * hid));
    VKM_CKH(cudaMalloc(&h->b2, sizeof(float) * 2));
    VKM_CKH(cudaMemcpy(h->w1p, w1p.data(), sizeof(float) * w1p.size(), cudaMemcpyHostToDevice));
    VKM_CKH(cudaMemcpy(h->b1, b1, sizeof(float) * hid, cudaMemcpyHostToDevice));
    VKM_CKH(cudaMemcpy(h->w2, w2, sizeof(float) * 2 * hid, cudaMemcpyHostToDevice));
    VKM_CKH(cudaMemcpy(h->b2, b2, sizeof(float) * 2, cudaMemcpyHostToDevice));
    if (h->tc_ok) {
      // fp16 hi/lo split of s·W1 with s = 2^e so that max|s·W1| <= 2^14.
      float amax = 0.f;
      for (float v : w1p) amax = std::max(amax, std::fabs(v));
      int e = 0;
      if (amax > 0.f) e = std::max(-30, std::min(40, 14 - int(std::ceil(std::log2(double(amax))))));
      h->w_scale_f16 = std::ldexp(1.0f, e);
      std::vector<uint16_t> hi(128 * 128), lo(128 * 128), bf(128 * 128);
      for (int i = 0; i < 128 * 128; ++i) {
        // column f of W1 goes to K position feature_kpos(f) of the operand image
        const int r = i >> 7, f = i & 127;
        const int j = r * 128 + vkm::feature_kpos(f);
        const float v = w1p[i] * h->w_scale_f16;
        const __half vh = __float2half_rn(v);
        const __half vl = __float2half_rn(v - __half2float(vh));
        std::memcpy(&hi[j], &vh, 2);
        std::memcpy(&lo[j], &vl, 2);
        const __nv_bfloat16 vb = __float2bfloat16_rn(w1p[i]);
        std::memcpy(&bf[j], &vb, 2);
      }
      std::vector<uint16_t> img(128 * 128);
      VKM_CKH(cudaMalloc(&h->w1_f16_hi, 2 * 128 * 128));
      VKM_CKH(cudaMalloc(&h->w1_f16_lo, 2 * 128 * 128));
      VKM_CKH(cudaMalloc(&h->w1_bf16, 2 * 128 * 128));
      vkm::build_umma_image_kmajor_128x128(hi.data(), img.data());
      VKM_CKH(cudaMemcpy(h->w1_f16_hi, img.data(), 2 * 128 * 128, cudaMemcpyHostToDevice));
      vkm::build_umma_image_kmajor_128x128(lo.data(), img.data());
      VKM_CKH(cudaMemcpy(h->w1_f16_lo, img.data(), 2 * 128 * 128, cudaMemcpyHostToDevice));
      vkm::build_umma_image_kmajor_128x128(bf.data(), img.data());
      VKM_CKH(cudaMemcpy(h->w1_bf16, img.data(), 2 * 128 * 128, cudaMemcpyHostToDevice));
    }
  }
#undef VKM_CKH
  *out = h;
  return VKM_OK;
}

void vkm_destroy(vkm_handle* h) {
  if (!h) return;
  DeviceGuard dg(h->p.device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  void* ptrs[] = {h->tf, h->my, h->mx, h->mxp, h->myp, h->xyz64, h->t64, h->mx64, h->my64, h->g64a, h->g64b, h->out64, h->win_ev, h->win_aux, h->w1p, h->b1, h->w2, h->b2, h->w64, h->w1_f16_hi, h->w1_f16_lo, h->w1_bf16,
                  h->G, h->C, h->Q, h->NQ, h->feats, h->cnt_scratch, h->ev_stage, h->out_stage, h->cnt_stage,
                  h->sb.pix, h->sb.val, h->sb.start, h->sb.val_s, h->sb.pix_s, h->sb.scan_state,
                  h->sb.rank, h->sb.longlist, h->sb.longcount, h->sb.bkt, h->sb.msd_tab, h->sb.msd_state};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& e : h->evt)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    for (void* p : {static_cast<void*>(h->pev[i]), static_cast<void*>(h->pout[i]), static_cast<void*>(h->pcnt[i])})
      if (p) cudaFree(p);
    for (cudaEvent_t e : {h->in_ready[i], h->computed[i], h->out_done[i]})
      if (e) cudaEventDestroy(e);
  }
  if (h->hout) cudaFreeHost(h->hout);
  for (auto& e : h->dl_ev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i)
    if (h->hpack[i]) cudaFreeHost(h->hpack[i]);
  delete h->pool;
  if (h->sel_temp) cudaFree(h->sel_temp);
  if (h->s_in) cudaStreamSynchronize(h->s_in), cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamSynchronize(h->s_out), cudaStreamDestroy(h->s_out);
  if (h->s_side) cudaStreamSynchronize(h->s_side), cudaStreamDestroy(h->s_side);
  if (h->e_fork) cudaEventDestroy(h->e_fork);
  if (h->e_join) cudaEventDestroy(h->e_join);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int vkm_set_mlp_mode(vkm_handle* h, int32_t mode) {
  if (int rc = check_handle(h)) return rc;
  if (mode < VKM_MLP_AUTO || mode > VKM_MLP_BF16) return fail(VKM_EINVAL, "unknown MLP mode");
  if (mode == VKM_MLP_AUTO) mode = h->tc_ok ? VKM_MLP_F16X3 : VKM_MLP_FP32;
  if ((mode == VKM_MLP_F16X3 || mode == VKM_MLP_BF16) && !h->tc_ok)
    return fail(VKM_EUNSUPPORTED, "tensor-core MLP modes need embed_dim == 64 and hidden == 128");
  h->mode = mode;
  return VKM_OK;
}

int vkm_set_weights_f64(vkm_handle* h, const double* w1, const double* b1, const double* w2, const double* b2) {
  if (int rc = check_handle(h)) return rc;
  if (h->hidden <= 0) return fail(VKM_EINVAL, "vkm_set_weights_f64: the handle has no head (hidden == 0)");
  if (!w1 || !b1 || !w2 || !b2) return fail(VKM_EINVAL, "vkm_set_weights_f64: null argument");
  const int hid = h->hidden, F = 2 * h->D;
  std::vector<double> buf(size_t(F) * hid + hid + 2 * hid + 2);
  for (int r = 0; r < hid; ++r)
    for (int j = 0; j < F; ++j) buf[size_t(j) * hid + r] = w1[size_t(r) * F + j];   // W1ᵀ [F][hidden]
  std::memcpy(buf.data() + size_t(F) * hid, b1, sizeof(double) * hid);
  std::memcpy(buf.data() + size_t(F) * hid + hid, w2, sizeof(double) * 2 * hid);
  std::memcpy(buf.data() + size_t(F) * hid + 3 * hid, b2, sizeof(double) * 2);
  for (double v : buf)
    if (!std::isfinite(v)) return fail(VKM_EINVAL, "weights must be finite");
  DeviceGuard dg(h->p.device);
  if (!h->w64 && cudaMalloc(&h->w64, sizeof(double) * buf.size()) != cudaSuccess) {
    h->w64 = nullptr;
    cudaGetLastError();
    return fail(VKM_EOOM, "vkm_set_weights_f64: device allocation failed");
  }
  if (cudaMemcpy(h->w64, buf.data(), sizeof(double) * buf.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(VKM_ECUDA, std::string("vkm_set_weights_f64: ") + cudaGetErrorString(cudaGetLastError()));
  return VKM_OK;
}

int vkm_predict(vkm_handle* h, const double* ev, int64_t n, double t_start, float* flows, int32_t* counts,
                void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (h->hidden <= 0) return fail(VKM_EINVAL, "handle has no flow head (hidden == 0)");
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n > 0 && (!ev || !flows)) return fail(VKM_EINVAL, "null device buffer");
  DeviceGuard dg(h->p.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int launches = 0;
  rec(h, 0, s);
  int rc = predict_one(h, ev, n, t_start, flows, counts, s, &launches);
  rec(h, 3, s);
  h->have_timing = h->profiling;
  h->last_launches = launches;
  return rc;
}

int vkm_encode(vkm_handle* h, const double* ev, int64_t n, double t_start, float* feats, int32_t* counts,
               void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n > 0 && (!ev || !feats)) return fail(VKM_EINVAL, "null device buffer");
  DeviceGuard dg(h->p.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int launches = 0;
  rec(h, 0, s);
  int rc = encode_core(h, ev, one_slice(n, t_start), 1, s, &launches);
  if (rc) return rc;
  if (n > 0) {
    vkm::launch_features(ev, n, t_start, h->p.delta_t, tables(h), h->p.width, h->p.height, h->D8, h->D, bufs(h),
                         feats, 2 * h->D, h->D, counts, s);
    launches += 1;
    VKM_CK(cudaGetLastError());
  }
  rec(h, 3, s);
  h->have_timing = h->profiling;
  h->last_launches = launches;
  return VKM_OK;
}

}  // extern "C"

namespace {
int predict_host_impl(vkm_handle* h, const double* ev_host, int64_t n, double t_start, float* flows_host,
                      double* flows64_host, int32_t* counts_host) {
  if (int rc = check_handle(h)) return rc;
  if (h->hidden <= 0) return fail(VKM_EINVAL, "handle has no flow head (hidden == 0)");
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n == 0) return VKM_OK;
  if (!ev_host || (!flows_host && !flows64_host)) return fail(VKM_EINVAL, "null host buffer");
  DeviceGuard dg(h->p.device);
  int rc = grow(&h->ev_stage, &h->ev_cap, size_t(n) * 3);
  if (!rc) rc = grow(&h->out_stage, &h->out_cap, size_t(n) * 2);
  if (!rc && counts_host) rc = grow(&h->cnt_stage, &h->cnt_stage_cap, size_t(n));
  if (rc) return rc;
  cudaStream_t s = h->stream;
  int launches = 0;
  if (single_pack(h, n)) {
    // the host stages the next call's records into hpack: the previous call has synchronised
    const double t0 = std::isnan(t_start) ? ev_host[0] : t_start;
    uint2* packed = nullptr;
    rc = upload_packed(h, ev_host, n, t0, s, &packed);
    rec(h, 0, s);
    if (!rc) rc = predict_chunk(h, h->ev_stage, one_slice(n, t0), h->out_stage, counts_host ? h->cnt_stage : nullptr,
                                s, &launches, packed);
  } else {
    VKM_CK(cudaMemcpyAsync(h->ev_stage, ev_host, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
    rec(h, 0, s);
    rc = predict_one(h, h->ev_stage, n, t_start, h->out_stage, counts_host ? h->cnt_stage : nullptr, s, &launches);
  }
  if (rc) return rc;
  rec(h, 3, s);
  if (counts_host)
    VKM_CK(cudaMemcpyAsync(counts_host, h->cnt_stage, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  if (flows64_host || host_staged(n)) {
    rc = download_f32(h, h->out_stage, 2 * n, s, flows_host, flows64_host);
    if (rc) return rc;
  } else {
    VKM_CK(cudaMemcpyAsync(flows_host, h->out_stage, sizeof(float) * 2 * n, cudaMemcpyDeviceToHost, s));
  }
  VKM_CK(cudaStreamSynchronize(s));
  h->have_timing = h->profiling;
  h->last_launches = launches;
  return VKM_OK;
}
}  // namespace

extern "C" {

int vkm_predict_host(vkm_handle* h, const double* ev_host, int64_t n, double t_start, float* flows_host,
                     int32_t* counts_host) {
  return predict_host_impl(h, ev_host, n, t_start, flows_host, nullptr, counts_host);
}

int vkm_predict_host_wide(vkm_handle* h, const double* ev_host, int64_t n, double t_start, double* flows_host,
                          int32_t* counts_host) {
  return predict_host_impl(h, ev_host, n, t_start, nullptr, flows_host, counts_host);
}

int vkm_predict_host_checked(vkm_handle* h, const double* ev_host, int64_t n, double window, double* flows_host,
                             vkm_event_check* check, int32_t* ran) {
  if (int rc = check_handle(h)) return rc;
  if (!ran || !check) return fail(VKM_EINVAL, "null output");
  *ran = 0;
  if (h->hidden <= 0) return fail(VKM_EINVAL, "handle has no flow head (hidden == 0)");
  if (n <= 0 || !ev_host || !flows_host || !single_pack(h, n)) return VKM_OK;   // caller takes the checked path
  DeviceGuard dg(h->p.device);
  if (h->hpack_cap[0] < size_t(n)) {
    if (h->hpack[0]) cudaFreeHost(h->hpack[0]);
    h->hpack[0] = nullptr;
    h->hpack_cap[0] = 0;
    VKM_CK(cudaHostAlloc(&h->hpack[0], sizeof(uint2) * size_t(n), cudaHostAllocDefault));
    h->hpack_cap[0] = size_t(n);
  }
  int rc = grow(&h->ev_stage, &h->ev_cap, size_t(n) * 3);
  if (!rc) rc = grow(&h->out_stage, &h->out_cap, size_t(n) * 2);
  if (rc) return rc;
  if (!h->pool) h->pool = new vkm_host::HostPool(vkm_host::default_pool_threads());
  cudaStream_t s = h->stream;
  const double t0 = ev_host[0];   // sorted input: the window start (checked below)
  uint2* d = reinterpret_cast<uint2*>(h->ev_stage);
  // One pass over the rows: each host-pool part checks its rows
  // (check_event_array's predicates, sortedness, first/last time) and packs
  // them while they are in its cache; piece i+1 is checked and packed while
  // piece i crosses PCIe.  Kernels run only for valid, sorted input within the
  // window - otherwise the caller's validation raises the reference's error.
  const int pieces = single_pieces(n);
  vkm_event_check c{0, 0, 0, 1, -1, 0, 0, 0.0, 0.0};
  bool first = true;
  HostTrace tr;
  tr.dev("start", s);
  for (int i = 0; i < pieces; ++i) {
    const int64_t lo = n * i / pieces, hi = n * (i + 1) / pieces, m = hi - lo;
    const int parts = std::max(1, std::min<int>(h->pool->size(), int((m + pack_grain() - 1) / pack_grain())));
    std::vector<vkm_event_check> pcv(static_cast<size_t>(parts));
    vkm_event_check* pc = pcv.data();
    h->pool->run(parts, [&](int part) {
      const int64_t a = lo + m * part / parts, b = lo + m * (part + 1) / parts;
      vkm_event_check& q = pc[part];
      vkm_host::check_pack(ev_host + 3 * a, b - a, t0, h->p.delta_t, h->p.width, h->p.height,
                           reinterpret_cast<uint32_t*>(h->hpack[0] + a), q);
      if (q.first_outside >= 0) q.first_outside += a;
    });
    for (int part = 0; part < parts; ++part) {
      if (first) {
        c = pc[part];
        first = false;
      } else {
        vkm_host::merge_check(c, pc[part]);
      }
    }
    tr.mark("packed");
    VKM_CK(cudaMemcpyAsync(d + lo, h->hpack[0] + lo, sizeof(uint2) * (hi - lo), cudaMemcpyHostToDevice, s));
  }
  tr.dev("uploaded", s);
  *check = c;
  const bool ok = !c.nonfinite && !c.negative_t && !c.nonint && c.first_outside < 0 && c.sorted &&
                  !(c.t_last - c.t_first > window);
  if (!ok) {
    VKM_CK(cudaStreamSynchronize(s));   // the staging is reused by the next call
    return VKM_OK;
  }
  int launches = 0;
  rec(h, 0, s);
  rc = predict_chunk(h, h->ev_stage, one_slice(n, t0), h->out_stage, nullptr, s, &launches, d);
  if (rc) return rc;
  rec(h, 3, s);
  tr.dev("computed", s);
  tr.mark("launched");
  rc = download_f32(h, h->out_stage, 2 * n, s, nullptr, flows_host);
  if (rc) return rc;
  tr.dev("downloaded", s);
  tr.mark("widened");
  VKM_CK(cudaStreamSynchronize(s));
  h->have_timing = h->profiling;
  h->last_launches = launches;
  *ran = 1;
  return VKM_OK;
}

int vkm_encode_host(vkm_handle* h, const double* ev_host, int64_t n, double t_start, float* feats_host,
                    int32_t* counts_host) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n == 0) return VKM_OK;
  if (!ev_host || !feats_host) return fail(VKM_EINVAL, "null host buffer");
  DeviceGuard dg(h->p.device);
  int rc = grow(&h->ev_stage, &h->ev_cap, size_t(n) * 3);
  if (!rc) rc = grow(&h->out_stage, &h->out_cap, size_t(n) * 2 * h->D);
  if (!rc && counts_host) rc = grow(&h->cnt_stage, &h->cnt_stage_cap, size_t(n));
  if (rc) return rc;
  cudaStream_t s = h->stream;
  VKM_CK(cudaMemcpyAsync(h->ev_stage, ev_host, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  rc = vkm_encode(h, h->ev_stage, n, t_start, h->out_stage, counts_host ? h->cnt_stage : nullptr, s);
  if (rc) return rc;
  if (counts_host)
    VKM_CK(cudaMemcpyAsync(counts_host, h->cnt_stage, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  if (host_staged(n)) {   // large feature blocks: pinned pieces, copied out by the host pool
    rc = download_f32(h, h->out_stage, 2 * h->D * n, s, feats_host, nullptr);
    if (rc) return rc;
  } else {
    VKM_CK(cudaMemcpyAsync(feats_host, h->out_stage, sizeof(float) * 2 * h->D * n, cudaMemcpyDeviceToHost, s));
  }
  VKM_CK(cudaStreamSynchronize(s));
  return VKM_OK;
}

int vkm_predict_batch(vkm_handle* h, const double* ev, const int64_t* offsets, int32_t n_slices,
                      const double* t_starts, float* flows, int32_t* counts, void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (h->hidden <= 0) return fail(VKM_EINVAL, "handle has no flow head (hidden == 0)");
  if (n_slices < 0 || (n_slices > 0 && !offsets)) return fail(VKM_EINVAL, "bad slice offsets");
  for (int s = 0; s < n_slices; ++s)
    if (offsets[s + 1] < offsets[s] || offsets[s] < 0) return fail(VKM_EINVAL, "slice offsets must be non-decreasing");
  DeviceGuard dg(h->p.device);
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  int launches = 0;
  rec(h, 0, sm);
  // chunks of up to kMaxBatch slices (pixel budget batch_pixels) share one launch sequence
  int chunks = 0;
  for (int s = 0; s < n_slices;) {
    vkm::SliceTab st;
    const int s1 = next_chunk(h, offsets, n_slices, t_starts, s, st);
    const int64_t lo = offsets[s];
    if (st.nb > 0) {
      int rc = predict_chunk(h, ev + 3 * lo, st, flows + 2 * lo, counts ? counts + lo : nullptr, sm, &launches);
      if (rc) return rc;
      ++chunks;
    }
    s = s1;
  }
  rec(h, 3, sm);
  // per-kernel events are overwritten per chunk: meaningful for a one-chunk call
  h->have_timing = h->profiling && chunks == 1;
  h->last_launches = launches;
  return VKM_OK;
}

int vkm_predict_batch_host(vkm_handle* h, const double* ev_host, const int64_t* offsets, int32_t n_slices,
                           const double* t_starts, float* flows_host, int32_t* counts_host) {
  if (int rc = check_handle(h)) return rc;
  if (h->hidden <= 0) return fail(VKM_EINVAL, "handle has no flow head (hidden == 0)");
  if (n_slices < 0 || (n_slices > 0 && !offsets)) return fail(VKM_EINVAL, "bad slice offsets");
  for (int s = 0; s < n_slices; ++s)
    if (offsets[s + 1] < offsets[s] || offsets[s] < 0) return fail(VKM_EINVAL, "slice offsets must be non-decreasing");
  if (n_slices == 0 || offsets[n_slices] == offsets[0]) return VKM_OK;
  if (!ev_host || !flows_host) return fail(VKM_EINVAL, "null host buffer");
  DeviceGuard dg(h->p.device);
  // chunks (each one launch sequence), then the largest chunk sizes the staging slots
  // at most 2M events (or a quarter of the call) per chunk so copies overlap kernels
  static const int64_t chunk_events = [] {   // VKM_CHUNK_EVENTS: A/B of the pipeline granularity
    const char* e = std::getenv("VKM_CHUNK_EVENTS");
    return (e && std::atoll(e) > 0) ? int64_t(std::atoll(e)) : (int64_t(1) << 21);
  }();
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(chunk_events, (offsets[n_slices] - offsets[0]) / 4));
  std::vector<std::pair<int, vkm::SliceTab>> chunks;
  int64_t nmax = 0;
  for (int s = 0; s < n_slices;) {
    vkm::SliceTab st;
    const int s1 = next_chunk(h, offsets, n_slices, t_starts, s, st, cap);
    if (st.nb > 0) {
      chunks.emplace_back(s, st);
      nmax = std::max(nmax, st.off[st.nb]);
    }
    s = s1;
  }
  if (!h->s_in) {
    VKM_CK(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    VKM_CK(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      VKM_CK(cudaEventCreateWithFlags(&h->in_ready[i], cudaEventDisableTiming));
      VKM_CK(cudaEventCreateWithFlags(&h->computed[i], cudaEventDisableTiming));
      VKM_CK(cudaEventCreateWithFlags(&h->out_done[i], cudaEventDisableTiming));
    }
  }
  for (int i = 0; i < 2; ++i) {
    int rc = grow(&h->pev[i], &h->pev_cap[i], size_t(nmax) * 3);
    if (!rc) rc = grow(&h->pout[i], &h->pout_cap[i], size_t(nmax) * 2);
    if (!rc && counts_host) rc = grow(&h->pcnt[i], &h->pcnt_cap[i], size_t(nmax));
    if (rc) return rc;
  }
  // Host packing: 8 instead of 24 bytes per event over PCIe (f32 time
  // argument computed on the host in f64 exactly like k_prep, 16-bit pixel
  // coordinates; host_pack.cpp's AVX-512 packer on a host thread pool packs
  // chunk c+1 while the GPU runs chunk c).  Needs the tensor-core head and
  // 16-bit coordinates.  Default: on for calls of >= 8M events, where it
  // measured +4.5 % (cfg2), +9 % (cfg4), +18 % (cfg3), +8 % (cfg5) e2e and
  // equal at cfg1; small calls stall on the synchronous packing of their
  // first chunks (cfg1/cfg4 at 8 slices per call: -50 %).  VKM_HOST_PACK=0/1
  // forces it.
  static const int pack_env = [] {
    const char* e = std::getenv("VKM_HOST_PACK");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const int64_t total_events = offsets[n_slices] - offsets[0];
  const bool pack_wanted = pack_env >= 0 ? pack_env == 1 : total_events >= (int64_t(8) << 20);
  const bool pack = pack_wanted && batchable(h) && h->p.width < 65535 && h->p.height < 65535;
  if (pack)
    for (int i = 0; i < 2; ++i)
      if (h->hpack_cap[i] < size_t(nmax)) {
        if (h->hpack[i]) cudaFreeHost(h->hpack[i]);
        h->hpack[i] = nullptr;
        h->hpack_cap[i] = 0;
        VKM_CK(cudaHostAlloc(&h->hpack[i], sizeof(uint2) * size_t(std::max<int64_t>(nmax, 1)), cudaHostAllocDefault));
        h->hpack_cap[i] = size_t(nmax);
      }
  // Mixed transfer (VKM_PACK_RAW_EVERY = m > 0): every m-th chunk goes over
  // PCIe as the caller's raw 24-byte rows (the DMA reads them straight from
  // pinned host memory), the others host-packed: packing costs host DRAM
  // traffic (read 24 + write 8 + DMA read 8 B/event), raw rows cost PCIe
  // bytes (24 B/event), so a mix can balance the two when both bind.
  static const int raw_every = [] {
    const char* e = std::getenv("VKM_PACK_RAW_EVERY");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  cudaStream_t sc = h->stream;
  HostTrace tr;   // VKM_TRACE=1: per chunk, when the host finished waiting (w) and packing (p)
  // slot k = chunk % 2.  copy-in(c) waits until compute(c-2) stopped reading the
  // slot; compute(c) waits for copy-in(c) and for copy-out(c-2) to drain its output;
  // packing chunk c waits until copy-in(c-2) has drained the host staging slot.
  int launches = 0;
  for (size_t c = 0; c < chunks.size(); ++c) {
    const vkm::SliceTab& st = chunks[c].second;
    const int64_t lo = offsets[chunks[c].first], n = st.off[st.nb];
    const int k = int(c & 1);
    const bool pack_c = pack && !(raw_every > 0 && (c % size_t(raw_every)) == size_t(raw_every - 1));
    if (pack_c) {
      if (c >= 2) VKM_CK(cudaEventSynchronize(h->in_ready[k]));
      tr.mark("w");
      pack_chunk(h, ev_host, offsets, t_starts, chunks[c].first, st, h->hpack[k]);
      tr.mark("p");
    }
    if (c >= 2) VKM_CK(cudaStreamWaitEvent(h->s_in, h->computed[k], 0));
    if (pack_c)
      VKM_CK(cudaMemcpyAsync(h->pev[k], h->hpack[k], sizeof(uint2) * n, cudaMemcpyHostToDevice, h->s_in));
    else
      VKM_CK(cudaMemcpyAsync(h->pev[k], ev_host + 3 * lo, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, h->s_in));
    VKM_CK(cudaEventRecord(h->in_ready[k], h->s_in));
    VKM_CK(cudaStreamWaitEvent(sc, h->in_ready[k], 0));
    if (c >= 2) VKM_CK(cudaStreamWaitEvent(sc, h->out_done[k], 0));
    int rc = predict_chunk(h, h->pev[k], st, h->pout[k], counts_host ? h->pcnt[k] : nullptr, sc, &launches,
                           pack_c ? reinterpret_cast<const uint2*>(h->pev[k]) : nullptr);
    if (rc) return rc;
    VKM_CK(cudaEventRecord(h->computed[k], sc));
    VKM_CK(cudaStreamWaitEvent(h->s_out, h->computed[k], 0));
    VKM_CK(cudaMemcpyAsync(flows_host + 2 * lo, h->pout[k], sizeof(float) * 2 * n, cudaMemcpyDeviceToHost, h->s_out));
    if (counts_host)
      VKM_CK(cudaMemcpyAsync(counts_host + lo, h->pcnt[k], sizeof(int32_t) * n, cudaMemcpyDeviceToHost, h->s_out));
    VKM_CK(cudaEventRecord(h->out_done[k], h->s_out));
  }
  tr.mark("enq");
  VKM_CK(cudaStreamSynchronize(h->s_out));
  VKM_CK(cudaStreamSynchronize(sc));
  tr.mark("done");
  h->have_timing = false;
  h->last_launches = launches;
  return VKM_OK;
}

int vkm_predict_multi_host(vkm_handle* const* handles, int32_t n_handles, const double* ev_host,
                           const int64_t* offsets, int32_t n_slices, const double* t_starts, float* flows_host,
                           int32_t* counts_host) {
  if (n_handles < 1 || !handles) return fail(VKM_EINVAL, "need at least one handle");
  for (int i = 0; i < n_handles; ++i) {
    if (int rc = check_handle(handles[i])) return rc;
    for (int j = 0; j < i; ++j)
      if (handles[j] == handles[i]) return fail(VKM_EINVAL, "handles must be distinct (a handle is not re-entrant)");
    if (handles[i]->p.width != handles[0]->p.width || handles[i]->p.height != handles[0]->p.height)
      return fail(VKM_EINVAL, "handles must share the sensor geometry");
  }
  if (n_slices < 0 || (n_slices > 0 && !offsets)) return fail(VKM_EINVAL, "bad slice offsets");
  for (int s = 0; s < n_slices; ++s)
    if (offsets[s + 1] < offsets[s] || offsets[s] < 0) return fail(VKM_EINVAL, "slice offsets must be non-decreasing");
  if (n_slices == 0 || offsets[n_slices] == offsets[0]) return VKM_OK;
  // contiguous slice ranges of about equal event counts, one per handle (no exchange)
  const int64_t total = offsets[n_slices] - offsets[0];
  std::vector<int> cut(static_cast<size_t>(n_handles) + 1, n_slices);
  cut[0] = 0;
  for (int i = 1; i < n_handles; ++i) {
    const int64_t target = offsets[0] + total * i / n_handles;
    int s = cut[i - 1];
    while (s < n_slices && offsets[s] < target) ++s;
    cut[i] = s;
  }
  std::vector<int> rcs(static_cast<size_t>(n_handles), int(VKM_OK));
  std::vector<std::string> errs(static_cast<size_t>(n_handles));
  auto run = [&](int i) {
    const int s0 = cut[i], s1 = cut[i + 1];
    if (s1 > s0)
      rcs[i] = vkm_predict_batch_host(handles[i], ev_host, offsets + s0, s1 - s0, t_starts ? t_starts + s0 : nullptr,
                                      flows_host, counts_host);
    if (rcs[i]) errs[i] = vkm_last_error();   // thread-local: carried back to the caller's thread
  };
  std::vector<std::thread> workers;
  for (int i = 1; i < n_handles; ++i) workers.emplace_back(run, i);
  run(0);
  for (auto& t : workers) t.join();
  for (int i = 0; i < n_handles; ++i)
    if (rcs[i]) return fail(rcs[i], "handle " + std::to_string(i) + ": " + errs[i]);
  return VKM_OK;
}

int vkm_predict_strips_host(vkm_handle* const* handles, int32_t n_strips, const int32_t* row_cuts,
                            const double* ev_host, int64_t n, double t_start, float* flows_host,
                            int32_t* counts_host) {
  if (n_strips < 1 || !handles || !row_cuts) return fail(VKM_EINVAL, "need at least one strip");
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n == 0) return VKM_OK;
  if (!ev_host || !flows_host) return fail(VKM_EINVAL, "null host buffer");
  for (int i = 0; i < n_strips; ++i) {
    if (int rc = check_handle(handles[i])) return rc;
    for (int j = 0; j < i; ++j)
      if (handles[j] == handles[i]) return fail(VKM_EINVAL, "handles must be distinct (a handle is not re-entrant)");
  }
  const int W = handles[0]->p.width, dy = handles[0]->p.delta_y;
  if (row_cuts[0] != 0) return fail(VKM_EINVAL, "row_cuts[0] must be 0");
  for (int i = 0; i < n_strips; ++i) {
    if (row_cuts[i + 1] <= row_cuts[i]) return fail(VKM_EINVAL, "row_cuts must be increasing");
    const int H = row_cuts[n_strips];
    const int in_lo = std::max(0, row_cuts[i] - dy), in_hi = std::min(H, row_cuts[i + 1] + dy);
    if (handles[i]->p.width != W || handles[i]->p.delta_y != dy || handles[i]->p.height != in_hi - in_lo)
      return fail(VKM_EINVAL, "handle " + std::to_string(i) + " must have the strip's geometry (W x rows + halo)");
  }
  const double t0 = std::isnan(t_start) ? ev_host[0] : t_start;   // one time origin for every strip
  const int H = row_cuts[n_strips];
  std::vector<int> rcs(static_cast<size_t>(n_strips), int(VKM_OK));
  std::vector<std::string> errs(static_cast<size_t>(n_strips));
  auto run = [&](int i) {
    const int in_lo = std::max(0, row_cuts[i] - dy), in_hi = std::min(H, row_cuts[i + 1] + dy);
    std::vector<double> sub;
    std::vector<int64_t> idx;
    std::vector<uint8_t> own;
    for (int64_t e = 0; e < n; ++e) {   // time order kept: events in input order
      const double y = ev_host[3 * e + 2];
      if (!(y >= in_lo && y < in_hi)) continue;
      sub.insert(sub.end(), {ev_host[3 * e], ev_host[3 * e + 1], y - in_lo});
      idx.push_back(e);
      own.push_back(y >= row_cuts[i] && y < row_cuts[i + 1]);
    }
    const int64_t m = int64_t(idx.size());
    if (m == 0) return;
    std::vector<float> f(size_t(2 * m));
    std::vector<int32_t> c(counts_host ? size_t(m) : 0);
    rcs[i] = vkm_predict_host(handles[i], sub.data(), m, t0, f.data(), counts_host ? c.data() : nullptr);
    if (rcs[i]) {
      errs[i] = vkm_last_error();
      return;
    }
    for (int64_t k = 0; k < m; ++k)
      if (own[size_t(k)]) {
        flows_host[2 * idx[size_t(k)]] = f[size_t(2 * k)];
        flows_host[2 * idx[size_t(k)] + 1] = f[size_t(2 * k + 1)];
        if (counts_host) counts_host[idx[size_t(k)]] = c[size_t(k)];
      }
  };
  // events outside every strip (y outside [0, H) or not integer rows inside) keep the unsplit path's
  // NaN / 0 answer: pre-fill, strips overwrite their owned rows
  for (int64_t e = 0; e < n; ++e) {
    flows_host[2 * e] = flows_host[2 * e + 1] = std::numeric_limits<float>::quiet_NaN();
    if (counts_host) counts_host[e] = 0;
  }
  std::vector<std::thread> workers;
  for (int i = 1; i < n_strips; ++i) workers.emplace_back(run, i);
  run(0);
  for (auto& t : workers) t.join();
  for (int i = 0; i < n_strips; ++i)
    if (rcs[i]) return fail(rcs[i], "strip " + std::to_string(i) + ": " + errs[i]);
  return VKM_OK;
}

int vkm_select_rows(vkm_handle* h, const double* ev, int64_t n, int32_t y_lo, int32_t y_hi, int32_t own_lo,
                    int32_t own_hi, double* out_ev, int64_t* out_index, uint8_t* out_owned, int64_t* count_host) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0 || !count_host) return fail(VKM_EINVAL, "bad arguments");
  *count_host = 0;
  if (n == 0) return VKM_OK;
  if (!ev || !out_ev || !out_index || !out_owned) return fail(VKM_EINVAL, "null device buffer");
  DeviceGuard dg(h->p.device);
  const size_t need = 64 + 8 * vkm::select_rows_state_words(n);
  if (h->sel_temp_cap < need) {
    int rc = grow(&h->sel_temp, &h->sel_temp_cap, need);
    if (rc) return rc;
    VKM_CK(cudaMemset(h->sel_temp, 0, need));   // tile states: epoch 0 = never published
  }
  int64_t* count_dev = reinterpret_cast<int64_t*>(h->sel_temp);   // first 8 bytes; tile states after 64
  vkm::launch_select_rows(ev, n, y_lo, y_hi, own_lo, own_hi, reinterpret_cast<unsigned long long*>(h->sel_temp + 64),
                          out_index, count_dev, out_ev, out_owned, h->stream);
  VKM_CK(cudaGetLastError());
  VKM_CK(cudaMemcpyAsync(count_host, count_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
  VKM_CK(cudaStreamSynchronize(h->stream));
  return VKM_OK;
}

int vkm_scatter_rows(vkm_handle* h, const float* src, const int64_t* index, const uint8_t* mask, int64_t m,
                     int32_t row_floats, float* dst, void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (m < 0 || row_floats < 1) return fail(VKM_EINVAL, "bad arguments");
  if (m > 0 && (!src || !index || !dst)) return fail(VKM_EINVAL, "null device buffer");
  DeviceGuard dg(h->p.device);
  vkm::launch_scatter_rows(src, index, mask, m, row_floats, dst, static_cast<cudaStream_t>(stream));
  VKM_CK(cudaGetLastError());
  return VKM_OK;
}

int vkm_grid(vkm_handle* h, const double* ev, int64_t n, double t_start, int32_t pooled, float* grid,
             int32_t* counts, void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  DeviceGuard dg(h->p.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int launches = 0;
  int rc = encode_core(h, ev, one_slice(n, t_start), pooled, s, &launches);
  if (rc) return rc;
  vkm::launch_grid_to_ref(pooled ? h->Q : h->G, pooled ? h->NQ : h->C, h->p.width, h->p.height, h->D, h->D8,
                          pooled ? nullptr : h->mx, pooled ? nullptr : h->my, pooled != 0, grid, counts, s);
  VKM_CK(cudaGetLastError());
  return VKM_OK;
}

int vkm_pixel_order(vkm_handle* h, const double* ev, int64_t n, double t_start, int32_t* start, int32_t* order,
                    void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (!start || (n > 0 && (!ev || !order))) return fail(VKM_EINVAL, "null device buffer");
  DeviceGuard dg(h->p.device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = ensure_grid(h, h->P);
  if (!rc) rc = ensure_sort(h, n, h->P);
  if (rc) return rc;
  vkm::launch_sort_events(ev, nullptr, one_slice(n, t_start), h->p.delta_t, h->p.width, h->p.height, bufs(h), h->sb,
                          nullptr, nullptr, s);
  VKM_CK(cudaMemcpyAsync(start, h->sb.start, sizeof(int32_t) * (h->P + 1), cudaMemcpyDeviceToDevice, s));
  if (n > 0) vkm::launch_slot_events(h->sb.val_s, h->sb.start + h->P, n, order, s);
  VKM_CK(cudaGetLastError());
  return VKM_OK;
}

// ---- precision="f64" (k_f64.cu) ----
namespace {
int run_f64(vkm_handle* h, const double* ev, int64_t n, double t_start, double* out, int32_t* counts, bool predict,
            cudaStream_t s) {
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n > 0 && (!ev || !out)) return fail(VKM_EINVAL, "null device buffer");
  if (predict && h->hidden <= 0) return fail(VKM_EINVAL, "handle has no flow head (hidden == 0)");
  if (n == 0) return VKM_OK;
  const int W = h->p.width, H = h->p.height;
  double t0 = t_start;
  if (std::isnan(t0)) {   // the first event's time (the f64 kernels take t0 by value)
    VKM_CK(cudaMemcpyAsync(&t0, ev, sizeof(double), cudaMemcpyDeviceToHost, s));
    VKM_CK(cudaStreamSynchronize(s));
  }
  int rc = ensure_grid(h, h->P);
  if (!rc) rc = ensure_sort(h, n, h->P);
  if (!rc && h->g64_cap < h->P) {
    if (h->g64a) cudaFree(h->g64a);
    if (h->g64b) cudaFree(h->g64b);
    h->g64a = h->g64b = nullptr;
    h->g64_cap = 0;
    VKM_CK(cudaMalloc(&h->g64a, sizeof(double2) * h->D8 * h->P));
    VKM_CK(cudaMalloc(&h->g64b, sizeof(double2) * h->D8 * h->P));
    h->g64_cap = h->P;
  }
  if (rc) return rc;
  vkm::launch_sort_events(ev, nullptr, one_slice(n, t0), h->p.delta_t, W, H, bufs(h), h->sb, nullptr, nullptr, s);
  vkm::launch_pool_count(W, H, 1, h->p.delta_x, h->p.delta_y, bufs(h), s);
  const vkm::F64Tables t{h->t64, h->mx64, h->my64};
  vkm::launch_encode64(t, ev, n, t0, h->p.delta_t, W, H, h->D, h->D8, h->p.delta_x, h->p.delta_y, h->sb, h->NQ,
                       h->g64a, h->g64b, s);
  if (predict)
    vkm::launch_predict64(t, ev, n, t0, h->p.delta_t, W, H, h->D, h->D8, h->g64a, h->NQ,
                          vkm::MlpDev{h->w1p, h->b1, h->w2, h->b2, h->hidden, h->w64}, out, counts, h->num_sms, s);
  else
    vkm::launch_features64(t, ev, n, t0, h->p.delta_t, W, H, h->D, h->D8, h->g64a, h->NQ, out, counts, s);
  VKM_CK(cudaGetLastError());
  h->have_timing = false;
  return VKM_OK;
}

int run_f64_host(vkm_handle* h, const double* ev_host, int64_t n, double t_start, double* out_host,
                 int32_t* counts_host, bool predict) {
  if (n < 0) return fail(VKM_EINVAL, "n must be non-negative");
  if (n == 0) return VKM_OK;
  if (!ev_host || !out_host) return fail(VKM_EINVAL, "null host buffer");
  const size_t per = predict ? 2 : size_t(2 * h->D);
  int rc = grow(&h->ev_stage, &h->ev_cap, size_t(n) * 3);
  if (!rc) rc = grow(&h->out64, &h->out64_cap, size_t(n) * per);
  if (!rc && counts_host) rc = grow(&h->cnt_stage, &h->cnt_stage_cap, size_t(n));
  if (rc) return rc;
  cudaStream_t s = h->stream;
  VKM_CK(cudaMemcpyAsync(h->ev_stage, ev_host, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  rc = run_f64(h, h->ev_stage, n, t_start, h->out64, counts_host ? h->cnt_stage : nullptr, predict, s);
  if (rc) return rc;
  if (counts_host)
    VKM_CK(cudaMemcpyAsync(counts_host, h->cnt_stage, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  if (!predict && host_staged(n)) {   // feature blocks (1 KB/event); the 16 B/event flows measured no gain
    rc = download_raw(h, h->out64, sizeof(double) * per * n, s, out_host);
    if (rc) return rc;
  } else {
    VKM_CK(cudaMemcpyAsync(out_host, h->out64, sizeof(double) * per * n, cudaMemcpyDeviceToHost, s));
  }
  VKM_CK(cudaStreamSynchronize(s));
  return VKM_OK;
}
}  // namespace

int vkm_predict_f64(vkm_handle* h, const double* ev, int64_t n, double t_start, double* flows, int32_t* counts,
                    void* stream) {
  if (int rc = check_handle(h)) return rc;
  DeviceGuard dg(h->p.device);
  return run_f64(h, ev, n, t_start, flows, counts, true, static_cast<cudaStream_t>(stream));
}

int vkm_encode_f64(vkm_handle* h, const double* ev, int64_t n, double t_start, double* feats, int32_t* counts,
                   void* stream) {
  if (int rc = check_handle(h)) return rc;
  DeviceGuard dg(h->p.device);
  return run_f64(h, ev, n, t_start, feats, counts, false, static_cast<cudaStream_t>(stream));
}

int vkm_predict_f64_host(vkm_handle* h, const double* ev_host, int64_t n, double t_start, double* flows_host,
                         int32_t* counts_host) {
  if (int rc = check_handle(h)) return rc;
  DeviceGuard dg(h->p.device);
  return run_f64_host(h, ev_host, n, t_start, flows_host, counts_host, true);
}

int vkm_encode_f64_host(vkm_handle* h, const double* ev_host, int64_t n, double t_start, double* feats_host,
                        int32_t* counts_host) {
  if (int rc = check_handle(h)) return rc;
  DeviceGuard dg(h->p.device);
  return run_f64_host(h, ev_host, n, t_start, feats_host, counts_host, false);
}

int vkm_direct_encode_host(vkm_handle* h, const double* ev_host, int64_t n, const int64_t* queries_host, int64_t nq,
                           double* emb_host, int32_t* counts_host) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0 || nq < 0) return fail(VKM_EINVAL, "n and nq must be non-negative");
  if (nq == 0) return VKM_OK;
  if (!ev_host || !queries_host || !emb_host) return fail(VKM_EINVAL, "null host buffer");
  for (int64_t i = 0; i < nq; ++i)
    if (queries_host[i] < 0 || queries_host[i] >= n) return fail(VKM_EINVAL, "query index out of range");
  DeviceGuard dg(h->p.device);
  const int W = h->p.width, H = h->p.height, D = h->D;
  int rc = ensure_grid(h, h->P);
  if (!rc) rc = ensure_sort(h, n, h->P);
  if (!rc) rc = grow(&h->ev_stage, &h->ev_cap, size_t(n) * 3);
  if (!rc) rc = grow(&h->out64, &h->out64_cap, size_t(nq) * 2 * D + size_t(nq));   // + the query indices
  if (!rc) rc = grow(&h->cnt_stage, &h->cnt_stage_cap, size_t(nq));
  if (rc) return rc;
  cudaStream_t s = h->stream;
  int64_t* q_dev = reinterpret_cast<int64_t*>(h->out64 + size_t(nq) * 2 * D);   // queries after the outputs
  VKM_CK(cudaMemcpyAsync(h->ev_stage, ev_host, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s));
  VKM_CK(cudaMemcpyAsync(q_dev, queries_host, sizeof(int64_t) * nq, cudaMemcpyHostToDevice, s));
  vkm::launch_sort_events(h->ev_stage, nullptr, one_slice(n, ev_host[0]), h->p.delta_t, W, H, bufs(h), h->sb,
                          nullptr, nullptr, s);
  vkm::launch_direct64(h->ev_stage, q_dev, nq, h->sb, W, H, h->p.delta_x, h->p.delta_y, h->p.delta_t, h->xyz64,
                       h->xyz64 + D, h->xyz64 + 2 * D, D, reinterpret_cast<double2*>(h->out64), h->cnt_stage, s);
  VKM_CK(cudaGetLastError());
  VKM_CK(cudaMemcpyAsync(emb_host, h->out64, sizeof(double) * 2 * D * nq, cudaMemcpyDeviceToHost, s));
  if (counts_host)
    VKM_CK(cudaMemcpyAsync(counts_host, h->cnt_stage, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, s));
  VKM_CK(cudaStreamSynchronize(s));
  h->have_timing = false;
  return VKM_OK;
}

}  // extern "C"

// ---- head training (k_train.cu) ----
struct vkm_trainer {
  int device = 0;
  int F = 0, H = 0;
  int64_t n = 0;
  double margin = 0, mw = 0, eps = 0, lr = 0;
  int64_t step = 0;
  cudaStream_t s = nullptr;
  double *feats = nullptr, *u = nullptr, *prm = nullptr, *m = nullptr, *v = nullptr, *best = nullptr;
  double *loss_part = nullptr, *g_part = nullptr;
  int64_t *idx = nullptr, *bad = nullptr;
  int64_t idx_cap = 0, part_rows = 0;
  int64_t G() const { return int64_t(F) * H + 3 * int64_t(H) + 2; }
};

namespace {
// parameters <-> packed device layout W1ᵀ [F][H] | b1 | W2 | b2
void pack_params(int F, int H, const double* w1, const double* b1, const double* w2, const double* b2,
                 std::vector<double>& out) {
  out.assign(size_t(F) * H + 3 * size_t(H) + 2, 0.0);
  for (int k = 0; k < H; ++k)
    for (int j = 0; j < F; ++j) out[size_t(j) * H + k] = w1[size_t(k) * F + j];
  const size_t FH = size_t(F) * H;
  for (int k = 0; k < H; ++k) {
    out[FH + k] = b1[k];
    out[FH + H + k] = w2[k];
    out[FH + 2 * H + k] = w2[H + k];
  }
  out[FH + 3 * H] = b2[0];
  out[FH + 3 * H + 1] = b2[1];
}

int train_idx(vkm_trainer* t, const int64_t* idx_host, int64_t m) {
  for (int64_t i = 0; i < m; ++i)
    if (idx_host[i] < 0 || idx_host[i] >= t->n) return fail(VKM_EINVAL, "sample index out of range");
  if (t->idx_cap < m) {
    if (t->idx) cudaFree(t->idx);
    t->idx = nullptr;
    t->idx_cap = 0;
    VKM_CK(cudaMalloc(&t->idx, sizeof(int64_t) * std::max<int64_t>(m, 1)));
    t->idx_cap = m;
  }
  const int64_t rows = (m + vkm::train_rows_per_cta() - 1) / vkm::train_rows_per_cta();
  if (t->part_rows < rows) {
    if (t->loss_part) cudaFree(t->loss_part);
    if (t->g_part) cudaFree(t->g_part);
    t->loss_part = t->g_part = nullptr;
    t->part_rows = 0;
    VKM_CK(cudaMalloc(&t->loss_part, sizeof(double) * 2 * rows));
    VKM_CK(cudaMalloc(&t->g_part, sizeof(double) * rows * t->G()));
    t->part_rows = rows;
  }
  VKM_CK(cudaMemcpyAsync(t->idx, idx_host, sizeof(int64_t) * m, cudaMemcpyHostToDevice, t->s));
  return VKM_OK;
}
}  // namespace

extern "C" {

int vkm_train_create(vkm_trainer** out, int32_t device, const double* feats_host, const double* u_host, int64_t n,
                     int32_t n_features, int32_t hidden, const double* w1, const double* b1, const double* w2,
                     const double* b2, double margin, double margin_weight, double constraint_eps,
                     double learning_rate) {
  if (!out) return fail(VKM_EINVAL, "null output pointer");
  *out = nullptr;
  if (n <= 0) return fail(VKM_EINVAL, "training dataset is empty");
  if (n_features < 1 || n_features > 128 || hidden < 1 || hidden > 256)
    return fail(VKM_EINVAL, "head training supports 2D <= 128 features and hidden <= 256");
  if (!feats_host || !u_host || !w1 || !b1 || !w2 || !b2) return fail(VKM_EINVAL, "null host buffer");
  DeviceGuard dg(device);
  auto* t = new vkm_trainer();
  t->device = device;
  t->F = n_features;
  t->H = hidden;
  t->n = n;
  t->margin = margin;
  t->mw = margin_weight;
  t->eps = constraint_eps;
  t->lr = learning_rate;
  std::vector<double> packed;
  pack_params(t->F, t->H, w1, b1, w2, b2, packed);
  const size_t G = packed.size();
  auto bail = [&](cudaError_t e) {
    vkm_train_destroy(t);
    return fail(VKM_ECUDA, std::string("cuda: ") + cudaGetErrorString(e));
  };
#define VKM_CKT(x)                  \
  do {                              \
    cudaError_t e_ = (x);           \
    if (e_ != cudaSuccess) return bail(e_); \
  } while (0)
  VKM_CKT(cudaStreamCreateWithFlags(&t->s, cudaStreamNonBlocking));
  VKM_CKT(cudaMalloc(&t->feats, sizeof(double) * n * n_features));
  VKM_CKT(cudaMalloc(&t->u, sizeof(double) * n * 2));
  for (double** p : {&t->prm, &t->m, &t->v, &t->best}) VKM_CKT(cudaMalloc(p, sizeof(double) * G));
  VKM_CKT(cudaMalloc(&t->bad, sizeof(int64_t)));
  VKM_CKT(cudaMemcpy(t->feats, feats_host, sizeof(double) * n * n_features, cudaMemcpyHostToDevice));
  VKM_CKT(cudaMemcpy(t->u, u_host, sizeof(double) * n * 2, cudaMemcpyHostToDevice));
  VKM_CKT(cudaMemcpy(t->prm, packed.data(), sizeof(double) * G, cudaMemcpyHostToDevice));
  VKM_CKT(cudaMemcpy(t->best, packed.data(), sizeof(double) * G, cudaMemcpyHostToDevice));
  VKM_CKT(cudaMemset(t->m, 0, sizeof(double) * G));
  VKM_CKT(cudaMemset(t->v, 0, sizeof(double) * G));
  const int64_t none = -1;
  VKM_CKT(cudaMemcpy(t->bad, &none, sizeof(int64_t), cudaMemcpyHostToDevice));
#undef VKM_CKT
  *out = t;
  return VKM_OK;
}

void vkm_train_destroy(vkm_trainer* t) {
  if (!t) return;
  DeviceGuard dg(t->device);
  if (t->s) cudaStreamSynchronize(t->s);
  for (void* p : {static_cast<void*>(t->feats), static_cast<void*>(t->u), static_cast<void*>(t->prm),
                  static_cast<void*>(t->m), static_cast<void*>(t->v), static_cast<void*>(t->best),
                  static_cast<void*>(t->loss_part), static_cast<void*>(t->g_part), static_cast<void*>(t->idx),
                  static_cast<void*>(t->bad)})
    if (p) cudaFree(p);
  if (t->s) cudaStreamDestroy(t->s);
  delete t;
}

int vkm_train_epoch(vkm_trainer* t, const int64_t* order_host, int64_t m, int32_t batch_size) {
  if (!t) return fail(VKM_EINVAL, "null vkm_trainer");
  if (m < 0 || batch_size < 1) return fail(VKM_EINVAL, "bad epoch arguments");
  if (m == 0) return VKM_OK;
  if (!order_host) return fail(VKM_EINVAL, "null host buffer");
  DeviceGuard dg(t->device);
  if (int rc = train_idx(t, order_host, m)) return rc;
  for (int64_t lo = 0; lo < m; lo += batch_size) {
    const int64_t nb = std::min<int64_t>(batch_size, m - lo);
    ++t->step;
    vkm::launch_train_batch(t->feats, t->u, t->idx + lo, nb, t->F, t->H, t->prm, t->m, t->v, t->margin, t->mw,
                            t->eps, 1, t->lr, t->step, t->loss_part, t->g_part, t->bad, t->s);
  }
  VKM_CK(cudaGetLastError());
  VKM_CK(cudaStreamSynchronize(t->s));   // the index buffer is reused by the next call
  return VKM_OK;
}

int vkm_train_loss(vkm_trainer* t, const int64_t* idx_host, int64_t m, double* loss_out, int64_t* bad_step_out) {
  if (!t) return fail(VKM_EINVAL, "null vkm_trainer");
  if (m <= 0 || !idx_host || !loss_out) return fail(VKM_EINVAL, "bad loss arguments");
  DeviceGuard dg(t->device);
  if (int rc = train_idx(t, idx_host, m)) return rc;
  vkm::launch_train_batch(t->feats, t->u, t->idx, m, t->F, t->H, t->prm, nullptr, nullptr, t->margin, t->mw,
                          t->eps, 0, 0.0, 0, t->loss_part, nullptr, nullptr, t->s);
  VKM_CK(cudaGetLastError());
  const int64_t rows = (m + vkm::train_rows_per_cta() - 1) / vkm::train_rows_per_cta();
  std::vector<double> part(2 * rows);
  int64_t bad = -1;
  VKM_CK(cudaMemcpyAsync(part.data(), t->loss_part, sizeof(double) * 2 * rows, cudaMemcpyDeviceToHost, t->s));
  VKM_CK(cudaMemcpyAsync(&bad, t->bad, sizeof(int64_t), cudaMemcpyDeviceToHost, t->s));
  VKM_CK(cudaStreamSynchronize(t->s));
  double l1 = 0.0, l2 = 0.0;
  for (int64_t b = 0; b < rows; ++b) {
    l1 += part[2 * b];
    l2 += part[2 * b + 1];
  }
  *loss_out = l1 / double(m) + t->mw * (l2 / double(m));   // flow.py:246-248
  if (bad_step_out) *bad_step_out = bad;
  return VKM_OK;
}

int vkm_train_keep(vkm_trainer* t) {
  if (!t) return fail(VKM_EINVAL, "null vkm_trainer");
  DeviceGuard dg(t->device);
  VKM_CK(cudaMemcpyAsync(t->best, t->prm, sizeof(double) * t->G(), cudaMemcpyDeviceToDevice, t->s));
  VKM_CK(cudaStreamSynchronize(t->s));
  return VKM_OK;
}

int vkm_train_get(vkm_trainer* t, int32_t best, double* w1, double* b1, double* w2, double* b2) {
  if (!t) return fail(VKM_EINVAL, "null vkm_trainer");
  if (!w1 || !b1 || !w2 || !b2) return fail(VKM_EINVAL, "null host buffer");
  DeviceGuard dg(t->device);
  std::vector<double> packed(size_t(t->G()));
  VKM_CK(cudaMemcpyAsync(packed.data(), best ? t->best : t->prm, sizeof(double) * packed.size(),
                         cudaMemcpyDeviceToHost, t->s));
  VKM_CK(cudaStreamSynchronize(t->s));
  const int F = t->F, H = t->H;
  const size_t FH = size_t(F) * H;
  for (int k = 0; k < H; ++k)
    for (int j = 0; j < F; ++j) w1[size_t(k) * F + j] = packed[size_t(j) * H + k];
  for (int k = 0; k < H; ++k) {
    b1[k] = packed[FH + k];
    w2[k] = packed[FH + H + k];
    w2[H + k] = packed[FH + 2 * H + k];
  }
  b2[0] = packed[FH + 3 * H];
  b2[1] = packed[FH + 3 * H + 1];
  return VKM_OK;
}

int vkm_window_bounds(vkm_handle* h, const double* ev, int64_t n, const double* starts_host, int32_t n_windows,
                      double window, int64_t* bounds_host) {
  if (int rc = check_handle(h)) return rc;
  if (n < 0 || n_windows < 0) return fail(VKM_EINVAL, "n and n_windows must be non-negative");
  if (n_windows == 0) return VKM_OK;
  if ((n > 0 && !ev) || !starts_host || !bounds_host) return fail(VKM_EINVAL, "null buffer");
  if (!(window > 0.0)) return fail(VKM_EINVAL, "window must be positive");
  DeviceGuard dg(h->p.device);
  int rc = grow(&h->win_aux, &h->win_aux_cap, 3 * size_t(n_windows));
  if (rc) return rc;
  cudaStream_t s = h->stream;
  double* starts_dev = reinterpret_cast<double*>(h->win_aux);
  int64_t* bounds_dev = h->win_aux + n_windows;
  VKM_CK(cudaMemcpyAsync(starts_dev, starts_host, sizeof(double) * n_windows, cudaMemcpyHostToDevice, s));
  vkm::launch_window_bounds(ev, n, starts_dev, n_windows, window, bounds_dev, s);
  VKM_CK(cudaGetLastError());
  VKM_CK(cudaMemcpyAsync(bounds_host, bounds_dev, sizeof(int64_t) * 2 * n_windows, cudaMemcpyDeviceToHost, s));
  VKM_CK(cudaStreamSynchronize(s));
  return VKM_OK;
}

int vkm_predict_windows(vkm_handle* h, const double* ev, int64_t n, const double* starts_host,
                        const int64_t* bounds_host, int32_t n_windows, float* flows, int32_t* counts, void* stream) {
  if (int rc = check_handle(h)) return rc;
  if (n_windows < 0) return fail(VKM_EINVAL, "n_windows must be non-negative");
  if (n_windows == 0) return VKM_OK;
  if (!starts_host || !bounds_host) return fail(VKM_EINVAL, "null host buffer");
  std::vector<int64_t> off(size_t(n_windows) + 1, 0);
  std::vector<int64_t> lo(static_cast<size_t>(n_windows), 0);
  for (int32_t w = 0; w < n_windows; ++w) {
    const int64_t a = bounds_host[2 * w], b = bounds_host[2 * w + 1];
    if (a < 0 || b < a || b > n) return fail(VKM_EINVAL, "window bounds outside the stream");
    lo[w] = a;
    off[w + 1] = off[w] + (b - a);
  }
  const int64_t total = off[n_windows];
  if (total == 0) return VKM_OK;
  if (!ev || !flows) return fail(VKM_EINVAL, "null device buffer");
  DeviceGuard dg(h->p.device);
  // Windows are gathered and predicted in chunks of at most kWinChunk events
  // (one window may exceed it alone), so the gather buffer stays bounded
  // however long or overlapping the stream is.
  const int64_t kWinChunk = [] {   // read per call (tests lower it)
    const char* e = std::getenv("VKM_WINDOW_CHUNK_EVENTS");
    return e && std::atoll(e) > 0 ? int64_t(std::atoll(e)) : int64_t(32) << 20;
  }();
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  int rc = grow(&h->win_aux, &h->win_aux_cap, 3 * size_t(n_windows) + 1);
  if (rc) return rc;
  for (int32_t w0 = 0; w0 < n_windows && !rc;) {
    int32_t w1 = w0 + 1;
    while (w1 < n_windows && off[w1 + 1] - off[w0] <= kWinChunk) ++w1;
    const int32_t nw = w1 - w0;
    const int64_t base = off[w0], part = off[w1] - base;
    std::vector<int64_t> coff(size_t(nw) + 1);
    for (int32_t w = 0; w <= nw; ++w) coff[w] = off[w0 + w] - base;
    if (part > 0) {
      rc = grow(&h->win_ev, &h->win_ev_cap, size_t(part) * 3);
      if (rc) break;
      int64_t* off_dev = h->win_aux;
      int64_t* lo_dev = h->win_aux + nw + 1;
      VKM_CK(cudaMemcpyAsync(off_dev, coff.data(), sizeof(int64_t) * (nw + 1), cudaMemcpyHostToDevice, sm));
      VKM_CK(cudaMemcpyAsync(lo_dev, lo.data() + w0, sizeof(int64_t) * nw, cudaMemcpyHostToDevice, sm));
      vkm::launch_gather_windows(ev, off_dev, lo_dev, nw, part, h->win_ev, sm);
      VKM_CK(cudaGetLastError());
      rc = vkm_predict_batch(h, h->win_ev, coff.data(), nw, starts_host + w0, flows + 2 * base,
                             counts ? counts + base : nullptr, stream);
    }
    // the host arrays above are read by the async copies: finish them before reuse
    VKM_CK(cudaStreamSynchronize(sm));
    w0 = w1;
  }
  if (h->win_ev_cap > size_t(3) * kWinChunk) {   // a single huge window grew it: give it back
    cudaFree(h->win_ev);
    h->win_ev = nullptr;
    h->win_ev_cap = 0;
  }
  return rc;
}

int vkm_set_profiling(vkm_handle* h, int32_t enable) {
  if (int rc = check_handle(h)) return rc;
  h->profiling = enable != 0;
  return VKM_OK;
}

int vkm_last_timings(vkm_handle* h, float* ms, int32_t* n_out) {
  if (int rc = check_handle(h)) return rc;
  if (n_out) *n_out = h->last_launches;
  if (!ms) return VKM_OK;
  for (int i = 0; i < 4; ++i) ms[i] = -1.f;
  if (!h->have_timing) return VKM_OK;
  DeviceGuard dg(h->p.device);
  VKM_CK(cudaEventSynchronize(h->evt[3]));
  VKM_CK(cudaEventElapsedTime(&ms[0], h->evt[0], h->evt[1]));
  VKM_CK(cudaEventElapsedTime(&ms[1], h->evt[1], h->evt[2]));
  VKM_CK(cudaEventElapsedTime(&ms[2], h->evt[2], h->evt[3]));
  VKM_CK(cudaEventElapsedTime(&ms[3], h->evt[0], h->evt[3]));
  return VKM_OK;
}

}  // extern "C"
