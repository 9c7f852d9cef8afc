// VecKM_flow encoder kernels for sm_100a:
//   K2 k_pool_count   exact int32 box sum of the per-pixel counts
//      (K1 lives in k_sort.cu, the complex pooling in k_pool_tma.cu)
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

constexpr int kRB = 8;   // rows per batch of the count pooling kernel

// Exact int32 box sum of the per-pixel counts (bit-exact neighbourhood sizes,
// the cnt of encoder.py:336).  Same strip/segment tiling, one channel.
constexpr int kCountSW = 256;
__global__ void __launch_bounds__(256) k_pool_count(const int* __restrict__ Cin, int* __restrict__ NQout, int W,
                                                    int H, int dx, int dy, int RS) {
  // blockIdx.z = slice of a batch (its own W x H pixel block)
  const int* __restrict__ C = Cin + int64_t(blockIdx.z) * W * H;
  int* __restrict__ NQ = NQout + int64_t(blockIdx.z) * W * H;
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

void launch_pool_count(int W, int H, int nb, int dx, int dy, const GridBufs& g, cudaStream_t s) {
  const int TXc = kCountSW - 2 * dx;
  const int strips = (W + TXc - 1) / TXc;
  const int RS = pick_rs(H, strips, 1);
  dim3 grid(strips, (H + RS - 1) / RS, nb);
  k_pool_count<<<grid, kCountSW, 0, s>>>(g.C, g.NQ, W, H, dx, dy, RS);
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
      const float4 acc = __ldg(Q4 + ((int64_t(plane) * P + pj) << 2) + (q4 ^ qswz(pj)));
      float s0, k0, s1, k1;
      sincos2_f32(__fmul_rn(aj, T0), __fmul_rn(aj, T1), s0, k0, s1, k1);
      const float den = float(max(cj, 1));
      // pooled grid chunk in packed-pair layout (re c0, re c1, im c0, im c1)
      const float2 e0 = cmul_rn(make_float2(k0, -s0), make_float2(acc.x, acc.z));
      const float2 e1 = cmul_rn(make_float2(k1, -s1), make_float2(acc.y, acc.w));
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
                              const float2* __restrict__ mx, const float2* __restrict__ my, bool packed,
                              float2* __restrict__ out, int32_t* __restrict__ oc) {
  const int64_t P = int64_t(W) * H;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P * D) return;
  const int c = int(i % D);
  const int64_t xy = i / D;            // x * H + y
  const int x = int(xy / H), y = int(xy % H);
  const int64_t pix = int64_t(y) * W + x;
  float2 v;
  if (packed) {
    const float* f = reinterpret_cast<const float*>(G + (int64_t(c >> 3) * P + pix) * 8) +
                     (((c & 7) >> 1) ^ qswz(pix)) * 4 + (c & 1);   // packed = the pooled grid Q
    v = make_float2(f[0], f[2]);
  } else {
    v = G[(int64_t(c >> 3) * P + pix) * 8 + (c & 7)];
  }
  if (mx) {   // the raw grid is stored pre-modulated (M = G·e^{i(xX+yY)}): undo it
    const float2 m = cmul(__ldg(mx + int64_t(x) * D8 + c), __ldg(my + int64_t(y) * D8 + c));
    v = cmulc(v, m);
  }
  out[i] = v;
  if (c == 0 && oc) oc[xy] = C[pix];
}

void launch_grid_to_ref(const float2* G, const int* C, int W, int H, int D, int D8, const float2* mx,
                        const float2* my, bool packed, float* out_grid, int32_t* out_counts, cudaStream_t s) {
  const int64_t tot = int64_t(W) * H * D;
  k_grid_to_ref<<<int((tot + 255) / 256), 256, 0, s>>>(G, C, W, H, D, D8, mx, my, packed, reinterpret_cast<float2*>(out_grid),
                                                       out_counts);
}

}  // namespace vkm
