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
#include <cstdlib>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

namespace {
constexpr int kU = 4;   // rows / columns per unrolled step
}

// idx = x*8 + ch within one plane row (W*8 float2); blockIdx.y = row segment,
// blockIdx.z = plane.  DEMOD: the input is the x-pooled R of k_reduce_x and
// each output is multiplied by conj(e^{i(xX/δx + yY/δy)}) (the pooled grid Q).
// Raw y window (split path): idx = x*8 + ch within one plane row (W*8
// float2, complex layout); blockIdx.y = row segment, blockIdx.z = plane.
__global__ void __launch_bounds__(256) k_box_y(const float2* __restrict__ M, float2* __restrict__ R, int W, int H,
                                               int dy, int RS, int64_t P) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= W * 8) return;
  const int y0 = blockIdx.y * RS, y1 = min(H, y0 + RS);
  const float2* Mp = M + int64_t(blockIdx.z) * P * 8 + idx;
  float2* Rp = R + int64_t(blockIdx.z) * P * 8 + idx;
  const int64_t rs = int64_t(W) * 8;   // row stride in float2
  const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
  const float2 zero = make_float2(0.f, 0.f);
  float2 acc = zero;
  for (int y = max(0, y0 - dy); y < min(H, y0 + dy); ++y) acc = cadd(acc, ld_nc_hint(Mp + int64_t(y) * rs, keep));
  for (int y = y0; y < y1; y += kU) {
    float2 ld[kU], tr[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int yy = y + u;
      ld[u] = (yy < y1 && yy + dy < H) ? ld_nc_hint(Mp + int64_t(yy + dy) * rs, keep) : zero;
      tr[u] = (yy < y1 && yy - dy >= 0) ? ld_nc_hint(Mp + int64_t(yy - dy) * rs, drop) : zero;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (y + u < y1) {
        acc = cadd(acc, ld[u]);
        Rp[int64_t(y + u) * rs] = acc;
        acc = csub(acc, tr[u]);
      }
    }
  }
}

// y window + demodulation on the packed-pair layout (fused path): idx =
// x*4 + q, a thread owns channel pair q of one plane (16 B per pixel row):
//   Q[y][x] = Σ_{|j|<=δy} R[y+j][x] · conj(e^{i(xX/δx + yY/δy)})
// Complex arithmetic runs on f32x2 pairs (re c, re c+1), (im c, im c+1).
// blockIdx.y = slice * segs + segment (batched slices stack vertically, rows
// never mix across slices); P is the plane stride (nb·W·H).
#ifndef VKM_YU
#define VKM_YU 4
#endif
constexpr int kYU = VKM_YU;   // rows per batched step of the packed y pass
//
// Odd segments sweep upwards (d = -1), even ones downwards, so the two
// segments on either side of a boundary read the rows around it at the same
// time (both at their start, or both at their end): the 2δy-row warm-up of one
// segment is the other's lead rows, served by one DRAM read instead of two.
// The window update is acc += R[y + dδ] (lead), out(y), acc -= R[y - dδ].
__global__ void __launch_bounds__(256) k_box_y_demod(const float4* __restrict__ Rin, float4* __restrict__ Q, int W,
                                                     int H, int segs, int dy, int RS, int64_t P,
                                                     const float4* __restrict__ mxp,
                                                     const float4* __restrict__ myp, int D2) {
  pdl_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= W * 4) return;
  const int slice = blockIdx.y / segs, seg = blockIdx.y - slice * segs;
  const int y0 = seg * RS, y1 = min(H, y0 + RS);
  const int d = (seg & 1) ? -1 : 1;
  const int ys = d > 0 ? y0 : y1 - 1, ny = y1 - y0;   // rows ys, ys + d, ... (ny of them)
  const int pair = int(blockIdx.z) * 4 + (idx & 3);
  const int64_t base = (int64_t(blockIdx.z) * P + int64_t(slice) * H * W) * 4 + idx;
  const ulonglong2* Rp = reinterpret_cast<const ulonglong2*>(Rin) + base;
  ulonglong2* Qp = reinterpret_cast<ulonglong2*>(Q) + base;
  const int64_t rs = int64_t(W) * 4;   // row stride in 16-byte chunks
  const float4 fx4 = __ldg(mxp + int64_t(idx >> 2) * D2 + pair);
  const uint64_t fxr = f2pack(fx4.x, fx4.y), fxi = f2pack(fx4.z, fx4.w);
  const float4* myc = myp + pair;
  // lead rows stay in L2 (evict_last) until the trailing edge re-reads them
  // 2δy+1 rows later (evict_first)
  const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
  auto ld = [&](int y, uint64_t pol) {   // row y of the column, zero outside the image
    ulonglong2 v = make_ulonglong2(0ull, 0ull);
    if (y >= 0 && y < H)
      asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;"
          : "=l"(v.x), "=l"(v.y)
          : "l"(Rp + int64_t(y) * rs), "l"(pol));
    return v;
  };
  uint64_t ar = 0, ai = 0;
  for (int j = -dy; j < dy; ++j) {   // window of ys without its lead row
    const ulonglong2 v = ld(ys + d * j, keep);
    ar = fadd2(ar, v.x);
    ai = fadd2(ai, v.y);
  }
  for (int i = 0; i < ny; i += kYU) {
    ulonglong2 lv[kYU], tv[kYU];
    float4 fm[kYU];
#pragma unroll
    for (int u = 0; u < kYU; ++u) {
      const bool ok = i + u < ny;
      const int y = ys + d * (i + u);
      lv[u] = ok ? ld(y + d * dy, keep) : make_ulonglong2(0ull, 0ull);
      tv[u] = ok ? ld(y - d * dy, drop) : make_ulonglong2(0ull, 0ull);
      fm[u] = ok ? __ldg(myc + int64_t(y) * D2) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kYU; ++u) {
      if (i + u < ny) {
        const int y = ys + d * (i + u);
        ar = fadd2(ar, lv[u].x);
        ai = fadd2(ai, lv[u].y);
        const uint64_t fyr = f2pack(fm[u].x, fm[u].y), fyi = f2pack(fm[u].z, fm[u].w);
        // f = e^{i xX}·e^{i yY};  out = acc · conj(f)
        const uint64_t fr = fsub2(fmul2(fxr, fyr), fmul2(fxi, fyi));
        const uint64_t fi = ffma2(fxr, fyi, fmul2(fxi, fyr));
        const uint64_t orr = ffma2(ar, fr, fmul2(ai, fi));
        const uint64_t oi = fsub2(fmul2(ai, fr), fmul2(ar, fi));
        // Q with evict_first: its 158 MB (cfg 2) must not push out the lead
        // rows of R kept for the trailing re-read (pool -7 % at cfg 3 and 4)
        const int c4 = idx & 3, cs = c4 ^ qswz(int64_t(slice) * H * W + int64_t(y) * W + (idx >> 2));
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(Qp + int64_t(y) * rs + (cs - c4)),
                     "l"(orr), "l"(oi), "l"(drop)
                     : "memory");
        ar = fsub2(ar, tv[u].x);
        ai = fsub2(ai, tv[u].y);
      }
    }
  }
  pdl_trigger();   // dependents may launch as this grid drains
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
  float2* Qr = Q + int64_t(plane) * P * 8 + int64_t(y) * W * 8;   // pixel x: chunk (ch >> 1) ^ qswz, + (ch & 1) floats
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
      const float2 o = cmulc(cmul(acc, dmy), m[u]);   // · conj(e^{iyY}) · conj(e^{ixX})
      const int64_t px = int64_t(y) * W + x + u;
      float* qo = reinterpret_cast<float*>(Qr + int64_t(x + u) * 8 + ((ch >> 1) ^ qswz(px)) * 2) + (ch & 1);   // re +0, im +2
      qo[0] = o.x;
      qo[2] = o.y;
      acc = csub(acc, tr[u]);
    }
  }
}

namespace {
// Row segments per column: enough threads for ~32 resident warps per SM, but
// bounded so the live (2δy+1)-row windows of all segments stay in an L2 budget
// (the trailing edge must hit L2) and the 2δy warm-up rows stay a minority.
int pick_segments(int W, int H, int dy, int planes, int threads_per_row, int threads_per_sm) {
  const double band = double(2 * dy + 1) * W * 512.0;
  const int s_max = std::max(1, std::min(int(64.0e6 / band), H / std::max(1, 3 * dy)));
  const int64_t col_threads = int64_t(threads_per_row) * planes;
  const int segs = int(std::max<int64_t>(1, (int64_t(148) * threads_per_sm + col_threads - 1) / col_threads));
  return std::max(1, std::min(segs, s_max));
}
}  // namespace

void launch_pool_split(const DevTables& tb, int W, int H, int D8, int dx, int dy, float2* M, float2* R,
                       float2* Qout, cudaStream_t s) {
  const int planes = D8 / 8;
  const int64_t P = int64_t(W) * H;
  const int segs = pick_segments(W, H, dy, planes, W * 8, 1024);
  const int RS = (H + segs - 1) / segs;
  dim3 gy((W * 8 + 255) / 256, (H + RS - 1) / RS, planes);
  k_box_y<<<gy, 256, 0, s>>>(M, R, W, H, dy, RS, P);
  // x-pass: column segments of CS outputs (2δx halo re-reads are L1/L2 hits)
  const int CS = std::max(128, 8 * dx);   // halo re-reads 2δx/CS
  dim3 gx((W + CS - 1) / CS, (H * 8 + 255) / 256, planes);
  k_box_x<<<gx, 256, 0, s>>>(R, Qout, tb.mx, tb.my, W, H, D8, dx, CS, P);
}

void launch_pool_y_demod(const DevTables& tb, int W, int H, int nb, int D8, int dy, const float2* R, float2* Q,
                         cudaStream_t s) {
  const int planes = D8 / 8;
  const int64_t P = int64_t(W) * H * nb;
  static const int env_segs = [] {
    const char* e = std::getenv("VKM_YSEGS");
    return e ? std::atoi(e) : 0;
  }();
  int segs = env_segs > 0 ? env_segs : pick_segments(W, H, dy, planes, W * 4, 512);
  segs = std::max(1, segs / nb);   // batched slices already multiply the parallelism
  const int RS = (H + segs - 1) / segs;
  segs = (H + RS - 1) / RS;
  dim3 gy((W * 4 + 255) / 256, segs * nb, planes);
  launch_pdl(k_box_y_demod, gy, 256, 0, s, reinterpret_cast<const float4*>(R), reinterpret_cast<float4*>(Q), W, H,
             segs, dy, RS, P, static_cast<const float4*>(tb.mxp), static_cast<const float4*>(tb.myp), D8 / 2);
}

}  // namespace vkm
