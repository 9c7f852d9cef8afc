// Device-side windowing of an event stream (slice_stream, events.py:331-387):
// the bounds of every window [start_i, start_i + window) are searched on the
// device in the uploaded, time-sorted stream (np.searchsorted side="left" at
// both edges: half-open windows), and the windows' events are gathered into
// one batch buffer (overlapping windows duplicate their shared events in HBM,
// not over PCIe), which the batched launch sequence then predicts with each
// window's start as its time origin.
#include <cstdint>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

namespace {

// first index i in [0, n) with t[i] >= v (t = ev[3 i]): np.searchsorted side="left"
__device__ __forceinline__ int64_t lower_bound_t(const double* __restrict__ ev, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ev[3 * mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_window_bounds(const double* __restrict__ ev, int64_t n, const double* __restrict__ starts,
                                int32_t nw, double window, int64_t* __restrict__ bounds) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nw) return;
  const double s = starts[i];
  bounds[2 * i] = lower_bound_t(ev, n, s);
  bounds[2 * i + 1] = lower_bound_t(ev, n, s + window);
}

// out rows [off[w], off[w+1]) = stream rows [lo_w, lo_w + off[w+1] - off[w]); a
// block strides over the concatenated output, finding its window by binary search
__global__ void k_gather_windows(const double* __restrict__ ev, const int64_t* __restrict__ off,
                                 const int64_t* __restrict__ lo, int32_t nw, double* __restrict__ out) {
  const int64_t total = off[nw];
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < total; r += int64_t(gridDim.x) * blockDim.x) {
    int a = 0, b = nw;   // window w with off[w] <= r < off[w+1]
    while (b - a > 1) {
      const int m = (a + b) >> 1;
      if (off[m] <= r) a = m;
      else b = m;
    }
    const int64_t src = lo[a] + (r - off[a]);
    out[3 * r] = ev[3 * src];
    out[3 * r + 1] = ev[3 * src + 1];
    out[3 * r + 2] = ev[3 * src + 2];
  }
}

}  // namespace

void launch_window_bounds(const double* ev, int64_t n, const double* starts_dev, int32_t nw, double window,
                          int64_t* bounds_dev, cudaStream_t s) {
  if (nw <= 0) return;
  k_window_bounds<<<(nw + 127) / 128, 128, 0, s>>>(ev, n, starts_dev, nw, window, bounds_dev);
}

void launch_gather_windows(const double* ev, const int64_t* off_dev, const int64_t* lo_dev, int32_t nw,
                           int64_t total, double* out, cudaStream_t s) {
  if (nw <= 0 || total <= 0) return;
  const int blocks = int((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  k_gather_windows<<<blocks, 256, 0, s>>>(ev, off_dev, lo_dev, nw, out);
}

}  // namespace vkm
