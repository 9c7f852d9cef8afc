// K2: window pooling of the pre-modulated grid as two streaming passes.
//
// K1 writes M[y][x] = G[y][x]·e^{i(xX/δx + yY/δy)}, so the phase-weighted
// window sum of _pool_batch (encoder.py:331-336) at every pixel is
//   Q[y][x] = e^{-i(xX/δx + yY/δy)} · Σ_{|i|<=δx, |j|<=δy} M[y+j][x+i]
// — a separable box sum followed by one demodulation.
//
//   k_box_y  one thread per (column, channel) of one plane slides a
//            (2δy+1)-row window down a segment of rows: + leading row
//            (HBM, kept in L2 with evict_last), - trailing row (re-read 2δy+1
//            rows later, an L2 hit).  Warps read/write 256 contiguous bytes.
//   k_box_x  one thread per (row, channel) of one plane slides a
//            (2δx+1)-column window along a segment of the row (trailing
//            value re-read from L1) and demodulates.
// Both are pure streaming kernels (no shared memory, no barriers), so
// occupancy hides the memory latency; loads are issued four rows/columns
// ahead of their use.  Out-of-image rows/columns contribute zero
// (encoder.py:185-188).
#include <algorithm>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

namespace {
constexpr int kU = 4;   // rows / columns per unrolled step
}

// idx = x*8 + ch within one plane row (W*8 float2); blockIdx.y = row segment,
// blockIdx.z = plane.  DEMOD: the input is the x-pooled R of k_reduce_x and
// each output is multiplied by conj(e^{i(xX/δx + yY/δy)}) (the pooled grid Q).
template <bool DEMOD>
__global__ void __launch_bounds__(256) k_box_y(const float2* __restrict__ M, float2* __restrict__ R, int W, int H,
                                               int dy, int RS, int64_t P, const float2* __restrict__ mx,
                                               const float2* __restrict__ my, int D8) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= W * 8) return;
  const int y0 = blockIdx.y * RS, y1 = min(H, y0 + RS);
  const float2* Mp = M + int64_t(blockIdx.z) * P * 8 + idx;
  float2* Rp = R + int64_t(blockIdx.z) * P * 8 + idx;
  const int64_t rs = int64_t(W) * 8;   // row stride in float2
  const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
  const float2 zero = make_float2(0.f, 0.f);
  const int c = int(blockIdx.z) * 8 + (idx & 7);
  float2 fx = zero;
  const float2* myc = my + c;
  if (DEMOD) fx = __ldg(mx + int64_t(idx >> 3) * D8 + c);
  float2 acc = zero;
  // warm-up: rows [y0-dy, y0+dy)
  {
    const int ya = max(0, y0 - dy), yb = min(H, y0 + dy);
    int y = ya;
    for (; y + kU <= yb; y += kU) {
      float2 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = ld_hint(Mp + int64_t(y + u) * rs, keep);
#pragma unroll
      for (int u = 0; u < kU; ++u) acc = cadd(acc, v[u]);
    }
    for (; y < yb; ++y) acc = cadd(acc, ld_hint(Mp + int64_t(y) * rs, keep));
  }
  for (int y = y0; y < y1; y += kU) {
    float2 ld[kU], tr[kU], fm[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int yy = y + u;
      ld[u] = (yy < y1 && yy + dy < H) ? ld_hint(Mp + int64_t(yy + dy) * rs, keep) : zero;
      tr[u] = (yy < y1 && yy - dy >= 0) ? ld_hint(Mp + int64_t(yy - dy) * rs, drop) : zero;
      if (DEMOD) fm[u] = (yy < y1) ? __ldg(myc + int64_t(yy) * D8) : zero;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (y + u >= y1) break;
      acc = cadd(acc, ld[u]);
      if (DEMOD)
        Rp[int64_t(y + u) * rs] = cmulc(acc, cmul(fx, fm[u]));   // · conj(e^{i(xX + yY)})
      else
        Rp[int64_t(y + u) * rs] = acc;
      acc = csub(acc, tr[u]);
    }
  }
}

// Thread -> (row y, channel ch) of plane blockIdx.z, columns [x0, x0+CS).
// A warp covers 4 rows x 8 channels, i.e. four contiguous 64-byte pixels per load.
__global__ void __launch_bounds__(256) k_box_x(const float2* __restrict__ R, float2* __restrict__ Q,
                                               const float2* __restrict__ mx, const float2* __restrict__ my, int W,
                                               int H, int D8, int dx, int CS, int64_t P) {
  const int ch = threadIdx.x & 7;
  const int y = (blockIdx.y * blockDim.x + threadIdx.x) >> 3;
  if (y >= H) return;
  const int plane = blockIdx.z;
  const int x0 = blockIdx.x * CS, x1 = min(W, x0 + CS);
  const int c = plane * 8 + ch;
  const float2* Rr = R + int64_t(plane) * P * 8 + int64_t(y) * W * 8 + ch;
  float2* Qr = Q + int64_t(plane) * P * 8 + int64_t(y) * W * 8 + ch;
  float2 dmy = __ldg(my + int64_t(y) * D8 + c);
  dmy.y = -dmy.y;
  const float2 zero = make_float2(0.f, 0.f);
  float2 acc = zero;
  for (int x = max(0, x0 - dx); x < min(W, x0 + dx); ++x) acc = cadd(acc, __ldg(Rr + int64_t(x) * 8));
  for (int x = x0; x < x1; x += kU) {
    float2 ld[kU], tr[kU], m[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int xx = x + u;
      ld[u] = (xx < x1 && xx + dx < W) ? __ldg(Rr + int64_t(xx + dx) * 8) : zero;
      tr[u] = (xx < x1 && xx - dx >= 0) ? __ldg(Rr + int64_t(xx - dx) * 8) : zero;
      m[u] = xx < x1 ? __ldg(mx + int64_t(xx) * D8 + c) : zero;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (x + u >= x1) break;
      acc = cadd(acc, ld[u]);
      Qr[int64_t(x + u) * 8] = cmulc(cmul(acc, dmy), m[u]);   // · conj(e^{iyY}) · conj(e^{ixX})
      acc = csub(acc, tr[u]);
    }
  }
}

namespace {
int pick_segments(int W, int H, int dy, int planes) {
  // y-pass: segments bounded by an L2 budget for the live (2δy+1)-row windows
  const double band = double(2 * dy + 1) * W * 512.0;
  const int s_max = std::max(1, int(64.0e6 / band));
  const int64_t col_threads = int64_t(W) * 8 * planes;
  int segs = int(std::max<int64_t>(1, (148 * 1024 + col_threads - 1) / col_threads));   // ~32 warps per SM
  return std::max(1, std::min(segs, s_max));
}
}  // namespace

void launch_pool_split(const DevTables& tb, int W, int H, int D8, int dx, int dy, float2* M, float2* R,
                       float2* Qout, cudaStream_t s) {
  const int planes = D8 / 8;
  const int64_t P = int64_t(W) * H;
  const int segs = pick_segments(W, H, dy, planes);
  const int RS = (H + segs - 1) / segs;
  dim3 gy((W * 8 + 255) / 256, (H + RS - 1) / RS, planes);
  k_box_y<false><<<gy, 256, 0, s>>>(M, R, W, H, dy, RS, P, nullptr, nullptr, D8);
  // x-pass: column segments of CS outputs (2δx halo re-reads are L1/L2 hits)
  const int CS = std::max(128, 8 * dx);   // halo re-reads 2δx/CS
  dim3 gx((W + CS - 1) / CS, (H * 8 + 255) / 256, planes);
  k_box_x<<<gx, 256, 0, s>>>(R, Qout, tb.mx, tb.my, W, H, D8, dx, CS, P);
}

void launch_pool_y_demod(const DevTables& tb, int W, int H, int D8, int dy, const float2* R, float2* Q,
                         cudaStream_t s) {
  const int planes = D8 / 8;
  const int64_t P = int64_t(W) * H;
  const int segs = pick_segments(W, H, dy, planes);
  const int RS = (H + segs - 1) / segs;
  dim3 gy((W * 8 + 255) / 256, (H + RS - 1) / RS, planes);
  k_box_y<true><<<gy, 256, 0, s>>>(R, Q, W, H, dy, RS, P, tb.mx, tb.my, D8);
}

}  // namespace vkm
