// VecKM_flow encoder kernels for sm_100a:
//   K1 k_accumulate   per-event temporal phases scattered into the pixel grid
//   K2 k_pool_cplx    separable, phase-modulated sliding-window pooling
//      k_pool_count   exact int32 box sum of the per-pixel counts
//   K3a k_features    gather + de-phase + ÷count -> [Re; Im] features
//   K3b k_mlp_ffma    CUDA-core two-layer head (fp32 parity mode)
// Reference (paths under /root/reference/pkg/src/evflow/): accumulate_grid
// (encoder.py:229-283), _pool_batch (encoder.py:312-346), embed_to_features
// and mlp_forward (flow.py:92-106).
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// K1: accumulate.  One warp handles 32 events per step: lanes load one event
// each (coalesced 768 B), bump the pixel count, then the warp walks the 32
// events; for each, lane `pair` computes channels (2·pair, 2·pair+1) and issues
// one 16-byte vector reduction, so an event's 64 complex phases land as eight
// 64-byte segments (one per channel plane).
// Order of additions inside a pixel is nondeterministic (fp32 atomics); the
// reference sums a pixel's phases in time order (encoder.py:255-267), so
// grid parity is tolerance-based while counts are exact.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_accumulate(const double* __restrict__ ev, int64_t n, double t0_in,
                                                    double delta_t, const float* __restrict__ tf, int W,
                                                    int H, int D8, float2* __restrict__ G,
                                                    int* __restrict__ C, int64_t P) {
  const int lane = threadIdx.x & 31;
  const int cp = D8 >> 1;          // channel pairs per event (4, 8, 16, 32)
  const int pair = lane % cp;
  const int sub = lane / cp;
  const int eps = 32 / cp;         // events per warp step
  const float T0 = __ldg(tf + 2 * pair), T1 = __ldg(tf + 2 * pair + 1);
  const double t0 = ld_t0(ev, t0_in);
  const int plane = pair >> 2, q4 = pair & 3;
  float4* G4 = reinterpret_cast<float4*>(G);
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t e = base + lane;
    float a = 0.f;
    int pix = -1;
    if (e < n) {
      const double t = __ldg(ev + 3 * e), x = __ldg(ev + 3 * e + 1), y = __ldg(ev + 3 * e + 2);
      const int xi = int(x), yi = int(y);
      if (xi >= 0 && xi < W && yi >= 0 && yi < H) {
        pix = yi * W + xi;
        a = time_arg(t, t0, delta_t);
        atomicAdd(C + pix, 1);
      }
    }
    const int cnt = int((n - base) < 32 ? (n - base) : 32);
    for (int j = 0; j < cnt; j += eps) {
      const int src = j + sub;
      const float aj = __shfl_sync(kFull, a, src & 31);
      const int pj = __shfl_sync(kFull, pix, src & 31);
      if (src < cnt && pj >= 0) {
        float s0, c0, s1, c1;
        sincos_f32(__fmul_rn(aj, T0), s0, c0);
        sincos_f32(__fmul_rn(aj, T1), s1, c1);
        atomicAdd(G4 + ((int64_t(plane) * P + pj) << 2) + q4, make_float4(c0, s0, c1, s1));
      }
    }
  }
}

void launch_accumulate(const double* ev, int64_t n, double t0, double delta_t, const DevTables& tb, int W,
                       int H, int D8, const GridBufs& g, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t warps = (n + 31) / 32;
  const int blocks = int(std::min<int64_t>((warps + 7) / 8, 148 * 32));
  k_accumulate<<<blocks, 256, 0, s>>>(ev, n, t0, delta_t, tb.tf, W, H, D8, g.G, g.C, int64_t(W) * H);
}

// ---------------------------------------------------------------------------
// K2: pooling.  Window sum with phase weights, made separable and O(1) per
// pixel by modulation:
//   Σ_{dy} G[y+dy] e^{i dy Y/δy} = e^{-i y Y/δy} · Σ_{y'} G[y'] e^{i y' Y/δy}
// (same along x).  A CTA owns one channel plane (8 channels), a strip of SW
// input columns (TX = SW - 2δx output columns) and a segment of RS rows.
//   y-pass: every thread slides a (2δy+1)-row window down its columns,
//           adding the modulated leading row and dropping the trailing one;
//           results for RB rows are demodulated into a shared row buffer.
//   x-pass: one warp per buffered row, modulated inclusive prefix along the
//           strip (strip-local, so cancellation is bounded by SW columns),
//           window = P[c+δx] - P[c-δx-1], demodulated, stored coalesced.
// Rows/columns outside the image contribute zero (the reference's guard
// border, encoder.py:185-188), never clamped or wrapped.
// ---------------------------------------------------------------------------
constexpr int kRB = 8;   // rows per batch = warps per CTA

template <int SW>
struct PoolSmem {
  static constexpr int SEG = SW / 4;                  // columns per lane in the x-pass
  static constexpr int ROW = SW + 4;                  // padded pixels per buffered row
  __host__ __device__ static constexpr int pc(int c) { return c + c / SEG; }
  static size_t bytes(int RS, int dy) {
    return sizeof(float2) * 8 * (size_t(kRB) * ROW + SW + RS + 2 * dy);
  }
};

template <int SW>
__global__ void __launch_bounds__(256) k_pool_cplx(const float2* __restrict__ G, float2* __restrict__ Q,
                                                   const float2* __restrict__ my, const float2* __restrict__ mx,
                                                   int W, int H, int D8, int dx, int dy, int RS, int64_t P) {
  using S = PoolSmem<SW>;
  constexpr int NCOL = SW / 32;
  extern __shared__ float2 sm[];
  float2* buf = sm;                                  // [kRB][ROW][8]
  float2* mxs = buf + kRB * S::ROW * 8;              // [SW][8]
  float2* mys = mxs + SW * 8;                        // [RS + 2dy][8]

  const int TX = SW - 2 * dx;
  const int xs = blockIdx.x * TX;
  const int xin0 = xs - dx;
  const int y0 = blockIdx.y * RS;
  const int y1 = min(H, y0 + RS);
  const int plane = blockIdx.z;
  const int t = threadIdx.x, ch = t & 7, cg = t >> 3;
  const float2* Gp = G + int64_t(plane) * P * 8;
  float2* Qp = Q + int64_t(plane) * P * 8;

  // Stage the modulation factors of this strip and row segment.
  for (int i = t; i < SW * 8; i += blockDim.x) {
    const int x = xin0 + (i >> 3);
    mxs[i] = (x >= 0 && x < W) ? __ldg(mx + int64_t(x) * D8 + plane * 8 + (i & 7)) : make_float2(0.f, 0.f);
  }
  const int ylo = y0 - dy;
  const int nyr = (y1 + dy) - ylo;
  for (int i = t; i < nyr * 8; i += blockDim.x) {
    const int y = ylo + (i >> 3);
    mys[i] = (y >= 0 && y < H) ? __ldg(my + int64_t(y) * D8 + plane * 8 + (i & 7)) : make_float2(0.f, 0.f);
  }
  __syncthreads();

  auto modrow = [&](int y, int xcol) -> float2 {  // G[y][x] * e^{i y Y/δy}, 0 outside
    const float2 g = __ldg(Gp + (int64_t(y) * W + xcol) * 8 + ch);
    return cmul(g, mys[(y - ylo) * 8 + ch]);
  };

  float2 acc[NCOL];
  bool colok[NCOL];
#pragma unroll
  for (int j = 0; j < NCOL; ++j) {
    const int x = xin0 + cg + 32 * j;
    colok[j] = (x >= 0 && x < W);
    acc[j] = make_float2(0.f, 0.f);
  }
  // Warm-up: rows [y0-dy, y0+dy) — everything of window(y0) except its leading row.
  for (int y = max(0, y0 - dy); y < min(H, y0 + dy); ++y) {
#pragma unroll
    for (int j = 0; j < NCOL; ++j)
      if (colok[j]) acc[j] = cadd(acc[j], modrow(y, xin0 + cg + 32 * j));
  }

  const int warp = t >> 5, lane = t & 31;
  const int sg = lane >> 3;
  for (int yb = y0; yb < y1; yb += kRB) {
    // ---- y-pass into the row buffer ----
#pragma unroll 2
    for (int rr = 0; rr < kRB; ++rr) {
      const int y = yb + rr;
      if (y >= y1) break;
      const float2 dm = mys[(y - ylo) * 8 + ch];
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const int c = cg + 32 * j;
        float2 out = make_float2(0.f, 0.f);
        if (colok[j]) {
          const int x = xin0 + c;
          if (y + dy < H) acc[j] = cadd(acc[j], modrow(y + dy, x));
          out = cmulc(acc[j], dm);
          if (y - dy >= 0) acc[j] = csub(acc[j], modrow(y - dy, x));
        }
        buf[(rr * S::ROW + S::pc(c)) * 8 + ch] = out;
      }
    }
    __syncthreads();
    // ---- x-pass: warp `warp` owns buffered row `warp` ----
    {
      const int y = yb + warp;
      if (y < y1) {
        float2* row = buf + warp * S::ROW * 8;
        float2 run = make_float2(0.f, 0.f);
        for (int i = 0; i < S::SEG; ++i) {
          const int c = sg * S::SEG + i;
          float2* p = row + (c + sg) * 8 + ch;
          run = cadd(run, cmul(*p, mxs[c * 8 + ch]));
          *p = run;
        }
        const float2 t1 = make_float2(__shfl_up_sync(kFull, run.x, 8), __shfl_up_sync(kFull, run.y, 8));
        const float2 t2 = make_float2(__shfl_up_sync(kFull, run.x, 16), __shfl_up_sync(kFull, run.y, 16));
        const float2 t3 = make_float2(__shfl_up_sync(kFull, run.x, 24), __shfl_up_sync(kFull, run.y, 24));
        float2 off = make_float2(0.f, 0.f);
        if (sg >= 1) off = cadd(off, t1);
        if (sg >= 2) off = cadd(off, t2);
        if (sg >= 3) off = cadd(off, t3);
        if (sg >= 1) {
          for (int i = 0; i < S::SEG; ++i) {
            float2* p = row + (sg * S::SEG + i + sg) * 8 + ch;
            *p = cadd(*p, off);
          }
        }
        __syncwarp();
        float2* qrow = Qp + int64_t(y) * W * 8;
        for (int jo = sg; jo < TX; jo += 4) {
          const int x = xs + jo;
          if (x >= W) break;
          const int c = jo + dx;
          const float2 hi = row[S::pc(c + dx) * 8 + ch];
          const float2 lo = (c - dx - 1 >= 0) ? row[S::pc(c - dx - 1) * 8 + ch] : make_float2(0.f, 0.f);
          qrow[int64_t(x) * 8 + ch] = cmulc(csub(hi, lo), mxs[c * 8 + ch]);
        }
      }
    }
    __syncthreads();
  }
}

// Exact int32 box sum of the per-pixel counts (bit-exact neighbourhood sizes,
// the cnt of encoder.py:336).  Same strip/segment tiling, one channel.
constexpr int kCountSW = 256;
__global__ void __launch_bounds__(256) k_pool_count(const int* __restrict__ C, int* __restrict__ NQ, int W, int H,
                                                    int dx, int dy, int RS) {
  constexpr int SW = kCountSW;
  constexpr int ROW = SW + SW / 8;
  __shared__ int buf[kRB * ROW];
  const int TX = SW - 2 * dx;
  const int xs = blockIdx.x * TX;
  const int x = xs - dx + threadIdx.x;
  const bool ok = (x >= 0 && x < W);
  const int y0 = blockIdx.y * RS, y1 = min(H, y0 + RS);
  int acc = 0;
  if (ok)
    for (int y = max(0, y0 - dy); y < min(H, y0 + dy); ++y) acc += __ldg(C + int64_t(y) * W + x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto pc = [](int c) { return c + (c >> 3); };
  for (int yb = y0; yb < y1; yb += kRB) {
    for (int rr = 0; rr < kRB; ++rr) {
      const int y = yb + rr;
      if (y >= y1) break;
      int out = 0;
      if (ok) {
        if (y + dy < H) acc += __ldg(C + int64_t(y + dy) * W + x);
        out = acc;
        if (y - dy >= 0) acc -= __ldg(C + int64_t(y - dy) * W + x);
      }
      buf[rr * ROW + pc(threadIdx.x)] = out;
    }
    __syncthreads();
    const int y = yb + warp;
    if (y < y1) {
      int* row = buf + warp * ROW;
      int run = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = lane * 8 + i;
        run += row[pc(c)];
        row[pc(c)] = run;
      }
      int inc = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += v;
      }
      const int off = inc - run;
#pragma unroll
      for (int i = 0; i < 8; ++i) row[pc(lane * 8 + i)] += off;
      __syncwarp();
      for (int jo = lane; jo < TX; jo += 32) {
        const int xo = xs + jo;
        if (xo >= W) break;
        const int c = jo + dx;
        NQ[int64_t(y) * W + xo] = row[pc(c + dx)] - ((c - dx - 1 >= 0) ? row[pc(c - dx - 1)] : 0);
      }
    }
    __syncthreads();
  }
}

static int pick_rs(int H, int strips, int planes) {
  // Enough CTAs to cover 148 SMs twice, but segments long enough that the
  // 2·δy warm-up rows stay a small fraction of the work.
  int rs = 64;
  while (rs > 16 && int64_t(strips) * planes * ((H + rs - 1) / rs) < 296) rs >>= 1;
  return rs;
}

template <int SW>
static void launch_pool_cplx(const DevTables& tb, int W, int H, int D8, int dx, int dy, const GridBufs& g,
                             cudaStream_t s) {
  const int TX = SW - 2 * dx;
  const int strips = (W + TX - 1) / TX;
  const int planes = D8 / 8;
  const int RS = pick_rs(H, strips, planes);
  const size_t smem = PoolSmem<SW>::bytes(RS, dy);
  cudaFuncSetAttribute(k_pool_cplx<SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  dim3 grid(strips, (H + RS - 1) / RS, planes);
  k_pool_cplx<SW><<<grid, 256, smem, s>>>(g.G, g.Q, tb.my, tb.mx, W, H, D8, dx, dy, RS, int64_t(W) * H);
}

void launch_pool(const DevTables& tb, int W, int H, int D8, int dx, int dy, const GridBufs& g, cudaStream_t s,
                 int* launches) {
  if (dx <= 16 || W <= 128 - 2 * dx)
    launch_pool_cplx<128>(tb, W, H, D8, dx, dy, g, s);
  else
    launch_pool_cplx<256>(tb, W, H, D8, dx, dy, g, s);
  const int TXc = kCountSW - 2 * dx;
  const int strips = (W + TXc - 1) / TXc;
  const int RS = pick_rs(H, strips, 1);
  dim3 grid(strips, (H + RS - 1) / RS);
  k_pool_count<<<grid, kCountSW, 0, s>>>(g.C, g.NQ, W, H, dx, dy, RS);
  if (launches) *launches += 2;
}

// ---------------------------------------------------------------------------
// K3a: per-event gather + de-phase + ÷count (encoder.py:344-345) written as
// [Re; Im] features (flow.py:92-95).  The de-phase factor is the conjugate of
// the event's own +T phase: numpy's f32 cos is even and sin odd bitwise, so
// _temporal_phases(t, sign=-1) == conj(_temporal_phases(t, +1)).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_features(const double* __restrict__ ev, int64_t n, double t0_in,
                                                  double delta_t, const float* __restrict__ tf, int W, int D8,
                                                  int Dout, const float2* __restrict__ Q,
                                                  const int* __restrict__ NQ, int64_t P, float* __restrict__ out,
                                                  int ld, int im_off, int32_t* __restrict__ counts_out) {
  const int lane = threadIdx.x & 31;
  const int cp = D8 >> 1;
  const int pair = lane % cp, sub = lane / cp, eps = 32 / cp;
  const int c0 = 2 * pair;
  const float T0 = __ldg(tf + c0), T1 = __ldg(tf + c0 + 1);
  const double t0 = ld_t0(ev, t0_in);
  const int plane = pair >> 2, q4 = pair & 3;
  const float4* Q4 = reinterpret_cast<const float4*>(Q);
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t e = base + lane;
    float a = 0.f;
    int pix = 0, cnt = 0;
    if (e < n) {
      const double t = __ldg(ev + 3 * e), x = __ldg(ev + 3 * e + 1), y = __ldg(ev + 3 * e + 2);
      pix = int(y) * W + int(x);
      a = time_arg(t, t0, delta_t);
      cnt = __ldg(NQ + pix);
      if (counts_out) counts_out[e] = cnt;
    }
    const int nv = int((n - base) < 32 ? (n - base) : 32);
    for (int j = 0; j < nv; j += eps) {
      const int src = j + sub;
      const float aj = __shfl_sync(kFull, a, src & 31);
      const int pj = __shfl_sync(kFull, pix, src & 31);
      const int cj = __shfl_sync(kFull, cnt, src & 31);
      if (src >= nv) continue;
      const float4 acc = __ldg(Q4 + ((int64_t(plane) * P + pj) << 2) + q4);
      float s0, k0, s1, k1;
      sincos_f32(__fmul_rn(aj, T0), s0, k0);
      sincos_f32(__fmul_rn(aj, T1), s1, k1);
      const float den = float(max(cj, 1));
      const float2 e0 = cmul_rn(make_float2(k0, -s0), make_float2(acc.x, acc.y));
      const float2 e1 = cmul_rn(make_float2(k1, -s1), make_float2(acc.z, acc.w));
      float* row = out + (base + src) * int64_t(ld);
      if (c0 + 1 < Dout) {
        *reinterpret_cast<float2*>(row + c0) = make_float2(__fdiv_rn(e0.x, den), __fdiv_rn(e1.x, den));
        *reinterpret_cast<float2*>(row + im_off + c0) = make_float2(__fdiv_rn(e0.y, den), __fdiv_rn(e1.y, den));
      } else if (c0 < Dout) {
        row[c0] = __fdiv_rn(e0.x, den);
        row[im_off + c0] = __fdiv_rn(e0.y, den);
      }
    }
  }
}

void launch_features(const double* ev, int64_t n, double t0, double delta_t, const DevTables& tb, int W, int H, int D8,
                     int Dout, const GridBufs& g, float* out, int ld, int im_off, int32_t* counts_out,
                     cudaStream_t s) {
  if (n <= 0) return;
  const int64_t warps = (n + 31) / 32;
  const int blocks = int(std::min<int64_t>((warps + 7) / 8, 148 * 32));
  k_features<<<blocks, 256, 0, s>>>(ev, n, t0, delta_t, tb.tf, W, D8, Dout, g.Q, g.NQ, int64_t(W) * H, out, ld,
                                    im_off, counts_out);
}

// ---------------------------------------------------------------------------
// K3b: fp32 CUDA-core head, one thread per event: h = relu(f·W1ᵀ + b1),
// out = h·W2ᵀ + b2 (flow.py:98-106).  W1 is broadcast from shared memory.
// NaN rows mark empty neighbourhoods (flow.py:188-196, estimators.py:203-206).
// ---------------------------------------------------------------------------
template <int K2>
__global__ void __launch_bounds__(128) k_mlp_ffma(const float* __restrict__ feats, const int32_t* __restrict__ counts,
                                                  int64_t n, const float* __restrict__ w1,
                                                  const float* __restrict__ b1, const float* __restrict__ w2,
                                                  const float* __restrict__ b2, int hidden,
                                                  float* __restrict__ flows) {
  extern __shared__ float4 smf[];
  float* sw1 = reinterpret_cast<float*>(smf);          // [hidden][K2]
  float* sb1 = sw1 + hidden * K2;
  float* sw2 = sb1 + hidden;
  for (int i = threadIdx.x; i < hidden * K2; i += blockDim.x) sw1[i] = w1[i];
  for (int i = threadIdx.x; i < hidden; i += blockDim.x) {
    sb1[i] = b1[i];
    sw2[i] = w2[i];
    sw2[hidden + i] = w2[hidden + i];
  }
  __syncthreads();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  float f[K2];
  const float4* fr = reinterpret_cast<const float4*>(feats + e * K2);
#pragma unroll
  for (int k = 0; k < K2 / 4; ++k) {
    const float4 v = __ldg(fr + k);
    f[4 * k] = v.x; f[4 * k + 1] = v.y; f[4 * k + 2] = v.z; f[4 * k + 3] = v.w;
  }
  float o0 = 0.f, o1 = 0.f;
  for (int h = 0; h < hidden; ++h) {
    const float4* wr = reinterpret_cast<const float4*>(sw1 + h * K2);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
    for (int k = 0; k < K2 / 4; ++k) {
      const float4 w = wr[k];
      s0 = fmaf(f[4 * k], w.x, s0);
      s1 = fmaf(f[4 * k + 1], w.y, s1);
      s2 = fmaf(f[4 * k + 2], w.z, s2);
      s3 = fmaf(f[4 * k + 3], w.w, s3);
    }
    const float hv = fmaxf((s0 + s1) + (s2 + s3) + sb1[h], 0.f);
    o0 = fmaf(hv, sw2[h], o0);
    o1 = fmaf(hv, sw2[hidden + h], o1);
  }
  float2 r = make_float2(o0 + __ldg(b2), o1 + __ldg(b2 + 1));
  if (counts && counts[e] <= 0) r = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
  reinterpret_cast<float2*>(flows)[e] = r;
}

void launch_mlp_ffma(const float* feats, const int32_t* counts, int64_t n, int D8, const MlpDev& m, float* flows,
                     cudaStream_t s) {
  if (n <= 0) return;
  const int K2 = 2 * D8;
  const size_t smem = sizeof(float) * (size_t(m.hidden) * K2 + 3 * m.hidden);
  const int blocks = int((n + 127) / 128);
#define VKM_MLP_CASE(KK)                                                                             \
  case KK:                                                                                           \
    cudaFuncSetAttribute(k_mlp_ffma<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));    \
    k_mlp_ffma<KK><<<blocks, 128, smem, s>>>(feats, counts, n, m.w1, m.b1, m.w2, m.b2, m.hidden, flows); \
    break;
  switch (K2) {
    VKM_MLP_CASE(16)
    VKM_MLP_CASE(32)
    VKM_MLP_CASE(64)
    VKM_MLP_CASE(128)
    default: break;
  }
#undef VKM_MLP_CASE
}

// ---------------------------------------------------------------------------
// Parity hook: plane layout -> reference PixelGrid layout [x][y][D] complex64.
// ---------------------------------------------------------------------------
__global__ void k_grid_to_ref(const float2* __restrict__ G, const int* __restrict__ C, int W, int H, int D, int D8,
                              float2* __restrict__ out, int32_t* __restrict__ oc) {
  const int64_t P = int64_t(W) * H;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P * D) return;
  const int c = int(i % D);
  const int64_t xy = i / D;            // x * H + y
  const int x = int(xy / H), y = int(xy % H);
  const int64_t pix = int64_t(y) * W + x;
  out[i] = G[(int64_t(c >> 3) * P + pix) * 8 + (c & 7)];
  if (c == 0 && oc) oc[xy] = C[pix];
}

void launch_grid_to_ref(const float2* G, const int* C, int W, int H, int D, int D8, float* out_grid,
                        int32_t* out_counts, cudaStream_t s) {
  const int64_t tot = int64_t(W) * H * D;
  k_grid_to_ref<<<int((tot + 255) / 256), 256, 0, s>>>(G, C, W, H, D, D8, reinterpret_cast<float2*>(out_grid),
                                                       out_counts);
}

}  // namespace vkm
