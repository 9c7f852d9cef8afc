// Device-side row-strip partition of one slice for the multi-GPU spatial
// split: stable selection of the events of rows
// [y_lo, y_hi) (a strip plus its δy event halo), rebased to strip-local y,
// with their global rows and an "owned" flag; and the scatter of a strip's
// owned flows back into the slice's row order.  The selection keeps time
// order, so per-pixel sums keep the reference's summation order.
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <cstdint>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

struct RowRange {
  const double* ev;
  double lo, hi;
  __host__ __device__ bool operator()(const int64_t& i) const {
    const double y = ev[3 * i + 2];
    return y >= lo && y < hi;
  }
};

__global__ void k_gather_strip(const double* __restrict__ ev, const int64_t* __restrict__ sel,
                               const int64_t* __restrict__ count, int y_lo, int own_lo, int own_hi,
                               double* __restrict__ out, uint8_t* __restrict__ owned) {
  const int64_t m = *count;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = sel[i];
    const double y = ev[3 * e + 2];
    out[3 * i] = ev[3 * e];
    out[3 * i + 1] = ev[3 * e + 1];
    out[3 * i + 2] = y - y_lo;
    owned[i] = (y >= own_lo && y < own_hi) ? 1 : 0;
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

size_t select_rows_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceSelect::If(nullptr, bytes, cub::CountingInputIterator<int64_t>(0), static_cast<int64_t*>(nullptr),
                        static_cast<int64_t*>(nullptr), n, RowRange{nullptr, 0, 0});
  return bytes;
}

void launch_select_rows(const double* ev, int64_t n, int y_lo, int y_hi, int own_lo, int own_hi, void* temp,
                        size_t temp_bytes, int64_t* sel, int64_t* count_dev, double* out, uint8_t* owned,
                        cudaStream_t s) {
  cub::DeviceSelect::If(temp, temp_bytes, cub::CountingInputIterator<int64_t>(0), sel, count_dev, n,
                        RowRange{ev, double(y_lo), double(y_hi)}, s);
  k_gather_strip<<<148 * 8, 256, 0, s>>>(ev, sel, count_dev, y_lo, own_lo, own_hi, out, owned);
}

void launch_scatter_rows(const float* src, const int64_t* index, const uint8_t* mask, int64_t m, int row_floats,
                         float* dst, cudaStream_t s) {
  if (m <= 0) return;
  const int blocks = int((m + 255) / 256 < 148 * 8 ? (m + 255) / 256 : 148 * 8);
  k_scatter_rows<<<blocks, 256, 0, s>>>(src, index, mask, m, row_floats, dst);
}

}  // namespace vkm
