// Device-side row-strip partition of one slice for the multi-GPU spatial
// split: stable selection of the events of rows
// [y_lo, y_hi) (a strip plus its δy event halo), rebased to strip-local y,
// with their global rows and an "owned" flag; and the scatter of a strip's
// owned flows back into the slice's row order.  The selection keeps time
// order, so per-pixel sums keep the reference's summation order.
#include <algorithm>
#include <cstdint>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

// One pass: a 2048-event tile counts its selected events, gets its output
// offset by decoupled look-back, and gathers its selected rows in order (the
// tile's own exclusive scan), so the selection stays stable (time order).
constexpr int kSelThreads = 256, kSelItems = 8, kSelTile = kSelThreads * kSelItems;

__global__ void __launch_bounds__(kSelThreads) k_select_strip(const double* __restrict__ ev, int64_t n, int ntiles,
                                                              double y_lo, double y_hi, int own_lo, int own_hi,
                                                              unsigned long long* __restrict__ state, uint32_t epoch,
                                                              int64_t* __restrict__ sel, int64_t* __restrict__ count,
                                                              double* __restrict__ out, uint8_t* __restrict__ owned) {
  __shared__ int warp_sum[kSelThreads / 32];
  __shared__ uint32_t tile_prefix;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t i0 = int64_t(t) * kSelTile + int64_t(threadIdx.x) * kSelItems;
    double yv[kSelItems];
    unsigned flags = 0;
#pragma unroll
    for (int k = 0; k < kSelItems; ++k) {
      yv[k] = i0 + k < n ? __ldg(ev + 3 * (i0 + k) + 2) : -1.0;
      if (i0 + k < n && yv[k] >= y_lo && yv[k] < y_hi) flags |= 1u << k;
    }
    const int cnt = __popc(flags);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    int wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kSelThreads / 32; ++w) {
      wpre += w < wid ? warp_sum[w] : 0;
      total += warp_sum[w];
    }
    if (wid == 0) {
      const uint32_t excl = lookback_publish(state, t, uint32_t(total), epoch);
      if (lane == 0) {
        tile_prefix = excl;
        if (t == ntiles - 1) *count = int64_t(excl) + total;
      }
    }
    __syncthreads();
    int64_t pos = int64_t(tile_prefix) + wpre + incl - cnt;
#pragma unroll
    for (int k = 0; k < kSelItems; ++k)
      if (flags >> k & 1) {
        const int64_t e = i0 + k;
        sel[pos] = e;
        out[3 * pos] = __ldg(ev + 3 * e);
        out[3 * pos + 1] = __ldg(ev + 3 * e + 1);
        out[3 * pos + 2] = yv[k] - y_lo;
        owned[pos] = (yv[k] >= own_lo && yv[k] < own_hi) ? 1 : 0;
        ++pos;
      }
    __syncthreads();
  }
}

__global__ void k_scatter_rows(const float* __restrict__ src, const int64_t* __restrict__ index,
                               const uint8_t* __restrict__ mask, int64_t m, int row_floats,
                               float* __restrict__ dst) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    if (mask && !mask[i]) continue;
    const int64_t d = index[i];
    for (int c = 0; c < row_floats; ++c) dst[d * row_floats + c] = src[i * row_floats + c];
  }
}

size_t select_rows_state_words(int64_t n) { return size_t((n + kSelTile - 1) / kSelTile); }

void launch_select_rows(const double* ev, int64_t n, int y_lo, int y_hi, int own_lo, int own_hi,
                        unsigned long long* state, int64_t* sel, int64_t* count_dev, double* out, uint8_t* owned,
                        cudaStream_t s) {
  const int ntiles = int((n + kSelTile - 1) / kSelTile);
  k_select_strip<<<std::min(ntiles, 148 * 4), kSelThreads, 0, s>>>(ev, n, ntiles, double(y_lo), double(y_hi), own_lo,
                                                                   own_hi, state, next_scan_epoch(), sel, count_dev,
                                                                   out, owned);
}

void launch_scatter_rows(const float* src, const int64_t* index, const uint8_t* mask, int64_t m, int row_floats,
                         float* dst, cudaStream_t s) {
  if (m <= 0) return;
  const int blocks = int((m + 255) / 256 < 148 * 8 ? (m + 255) / 256 : 148 * 8);
  k_scatter_rows<<<blocks, 256, 0, s>>>(src, index, mask, m, row_floats, dst);
}

}  // namespace vkm
