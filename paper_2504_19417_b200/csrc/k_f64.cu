// precision="f64" path (encoder.py:37-38: complex128 grid, float64 features;
// flow.py:98-106: the head promotes to float64).  Same pipeline as the f32
// path, every float in double precision:
//
//   sort       the f32 path's counting sort (k_sort.cu): pixel runs in time order
//   k64_reduce per pixel and channel, Σ e^{i a T} over the run in f64 in slot
//              order (np.add.reduceat's order, encoder.py:262-267), a = (t-t0)/δt
//              in f64 (encoder.py:223-224), pre-modulated by e^{i(xX/δx+yY/δy)}
//   k64_box_y, k64_box_x  separable (2δy+1)x(2δx+1) box sum of the modulated grid,
//              then demodulation: the window sum of _pool_batch (encoder.py:331-336)
//   k64_features / k64_predict  gather at each event, × conj(own phase), ÷ count
//              (encoder.py:344-345); the head relu(F·W1ᵀ+b1)·W2ᵀ+b2 in f64 with
//              the f32 weights promoted (flow.py:98-106)
//
// Layout: double2 [pixel][D8] (1 KB per pixel at D = 64), channel fastest, so a
// warp reads 32 channels of one pixel (512 contiguous bytes).  Not tuned like
// the f32 kernels: FP64 runs at half the FP32 rate on B200 and this path is
// the reference's precision option, not the hot path.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include <type_traits>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

namespace {

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {   // numpy complex128 multiply
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zmulc(double2 a, double2 b) {  // a · conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// Per-pixel f64 phase sums, pre-modulated.  Threads = (pixel, channel).
__global__ void __launch_bounds__(256) k64_reduce(const int* __restrict__ start, const uint64_t* __restrict__ val_s,
                                                  const double* __restrict__ ev, double t0, double delta_t,
                                                  const double* __restrict__ T, const double2* __restrict__ mx,
                                                  const double2* __restrict__ my, int W, int64_t P, int D8,
                                                  double2* __restrict__ M) {
  const int ppb = blockDim.x / D8;
  const int c = threadIdx.x % D8, pl = threadIdx.x / D8;
  if (pl >= ppb) return;
  const double Tc = T[c];
  for (int64_t p = int64_t(blockIdx.x) * ppb + pl; p < P; p += int64_t(gridDim.x) * ppb) {
    const int s = start[p], e = start[p + 1];
    double2 acc = make_double2(0.0, 0.0);
    for (int j = s; j < e; ++j) {
      const int32_t idx = slot_event(__ldg(val_s + j));
      const double a = (__ldg(ev + 3 * int64_t(idx)) - t0) / delta_t;
      double sn, cs;
      sincos(a * Tc, &sn, &cs);
      acc.x += cs;
      acc.y += sn;
    }
    const int y = int(p / W), x = int(p - int64_t(y) * W);
    M[p * D8 + c] = zmul(acc, zmul(mx[int64_t(x) * D8 + c], my[int64_t(y) * D8 + c]));
  }
}

// Sliding (2δy+1)-row window down each (column, channel) over one row
// segment [y0, y0 + RS) (blockIdx.y): warm-up from the δy rows above.
__global__ void __launch_bounds__(256) k64_box_y(const double2* __restrict__ M, double2* __restrict__ R, int W, int H,
                                                 int D8, int dy, int RS) {
  const int64_t col = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;   // x * D8 + c
  if (col >= int64_t(W) * D8) return;
  const int64_t rs = int64_t(W) * D8;
  const int y0 = blockIdx.y * RS, y1 = min(H, y0 + RS);
  double2 acc = make_double2(0.0, 0.0);
  for (int y = max(0, y0 - dy); y < min(H, y0 + dy); ++y) {
    const double2 v = M[y * rs + col];
    acc.x += v.x;
    acc.y += v.y;
  }
  for (int y = y0; y < y1; ++y) {
    if (y + dy < H) {
      const double2 v = M[(y + dy) * rs + col];
      acc.x += v.x;
      acc.y += v.y;
    }
    R[y * rs + col] = acc;
    if (y - dy >= 0) {
      const double2 v = M[(y - dy) * rs + col];
      acc.x -= v.x;
      acc.y -= v.y;
    }
  }
}

// Sliding (2δx+1)-column window along each (row, channel) over one column
// segment [x0, x0 + CS) (blockIdx.y), then demodulation.
__global__ void __launch_bounds__(256) k64_box_x(const double2* __restrict__ R, double2* __restrict__ Q, int W, int H,
                                                 int D8, int dx, int CS, const double2* __restrict__ mx,
                                                 const double2* __restrict__ my) {
  const int64_t rc = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;   // y * D8 + c
  if (rc >= int64_t(H) * D8) return;
  const int y = int(rc / D8), c = int(rc - int64_t(y) * D8);
  const int x0 = blockIdx.y * CS, x1 = min(W, x0 + CS);
  const double2* Rr = R + int64_t(y) * W * D8 + c;
  double2* Qr = Q + int64_t(y) * W * D8 + c;
  const double2 fy = my[int64_t(y) * D8 + c];
  double2 acc = make_double2(0.0, 0.0);
  for (int x = max(0, x0 - dx); x < min(W, x0 + dx); ++x) {
    const double2 v = Rr[int64_t(x) * D8];
    acc.x += v.x;
    acc.y += v.y;
  }
  for (int x = x0; x < x1; ++x) {
    if (x + dx < W) {
      const double2 v = Rr[int64_t(x + dx) * D8];
      acc.x += v.x;
      acc.y += v.y;
    }
    Qr[int64_t(x) * D8] = zmulc(acc, zmul(mx[int64_t(x) * D8 + c], fy));
    if (x - dx >= 0) {
      const double2 v = Rr[int64_t(x - dx) * D8];
      acc.x -= v.x;
      acc.y -= v.y;
    }
  }
}

// Embedding of event e, channel c < D: conj(e^{i a T}) · Q[pixel] / max(cnt, 1)
// (encoder.py:344-345).  Returns false (and cnt = 0) for out-of-sensor events.
__device__ __forceinline__ bool emb64(const double* __restrict__ ev, int64_t e, double t0, double delta_t, double Tc,
                                      const double2* __restrict__ Q, const int* __restrict__ NQ, int W, int H, int D8,
                                      int c, double2& out, int& cnt) {
  const double t = ev[3 * e], xd = ev[3 * e + 1], yd = ev[3 * e + 2];
  const int xi = int(xd), yi = int(yd);
  cnt = 0;
  if (!(xi >= 0 && xi < W && yi >= 0 && yi < H && xd == double(xi) && yd == double(yi))) return false;
  const int64_t p = int64_t(yi) * W + xi;
  cnt = NQ[p];
  double sn, cs;
  sincos(((t - t0) / delta_t) * Tc, &sn, &cs);
  const double2 prod = zmulc(Q[p * D8 + c], make_double2(cs, sn));   // dephase · acc
  const double den = double(cnt > 1 ? cnt : 1);
  out = make_double2(prod.x / den, prod.y / den);
  return true;
}

// Features [n][2D] = [Re | Im] (embed_to_features, flow.py:92-95); NaN rows
// for out-of-sensor events.  Threads = (event, channel < D).
__global__ void __launch_bounds__(256) k64_features(const double* __restrict__ ev, int64_t n, double t0,
                                                    double delta_t, const double* __restrict__ T,
                                                    const double2* __restrict__ Q, const int* __restrict__ NQ, int W,
                                                    int H, int D, int D8, double* __restrict__ feats,
                                                    int32_t* __restrict__ counts) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * D) return;
  const int64_t e = i / D;
  const int c = int(i - e * D);
  double2 v;
  int cnt;
  if (!emb64(ev, e, t0, delta_t, T[c], Q, NQ, W, H, D8, c, v, cnt)) v = make_double2(nan(""), nan(""));
  feats[e * 2 * D + c] = v.x;
  feats[e * 2 * D + D + c] = v.y;
  if (counts && c == 0) counts[e] = cnt;
}

constexpr int kEvPerStep = 16;   // events per block step of k64_predict

// Fused features + head.  Block = hidden threads (<= 256, rounded to a warp):
// per step the block builds the features of kEvPerStep events in shared
// memory (f64), then thread k forms hidden unit k for each of them with W1ᵀ
// column k (f32 in shared memory, promoted), ReLU, and the two outputs are
// block-reduced.  NaN rows for empty neighbourhoods (flow.py:188-196).
// WT: the type W1ᵀ is kept in shared memory as — double when it fits (no
// f32 -> f64 conversion in the inner loop), else float (promoted on use).
// W64: the head arrives as float64 (m.w64: W1ᵀ | b1 | W2 | b2, the reference's
// promoted f64 head, flow.py:98-106) and W1ᵀ is staged as double when it fits
// (WT = double), else read from global memory (WT = void).
template <typename WT, bool W64>
__global__ void k64_predict(const double* __restrict__ ev, int64_t n, double t0, double delta_t,
                            const double* __restrict__ T, const double2* __restrict__ Q, const int* __restrict__ NQ,
                            int W, int H, int D, int D8, const float* __restrict__ w1p, const float* __restrict__ b1,
                            const float* __restrict__ w2, const float* __restrict__ b2,
                            const double* __restrict__ w64, int hidden,
                            double* __restrict__ flows, int32_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint8_t sm64[];
  constexpr bool kGlobalW1 = std::is_void<WT>::value;
  using WS = typename std::conditional<kGlobalW1, double, WT>::type;
  const int F = 2 * D;                                          // features per event
  WS* w1t = reinterpret_cast<WS*>(sm64);                        // [F][hidden]
  const size_t w1bytes = kGlobalW1 ? 0 : size_t(F) * hidden * sizeof(WS);
  double* fs = reinterpret_cast<double*>(sm64 + ((w1bytes + 15) / 16) * 16);   // [kEv][F]
  double* red = fs + kEvPerStep * F;                            // [32 warps][kEv][2]
  int* cnts = reinterpret_cast<int*>(red + 32 * kEvPerStep * 2);
  const int k = threadIdx.x;
  const double* w64b1 = w64 + size_t(F) * hidden;
  const double* w64w2 = w64b1 + hidden;
  const double* w64b2 = w64w2 + 2 * hidden;
  if (!kGlobalW1)
    for (int i = threadIdx.x; i < F * hidden; i += blockDim.x) {   // W1 row r, feature j -> w1t[j][r]
      if (W64) {
        w1t[i] = WS(w64[i]);                                        // already W1ᵀ [F][hidden]
      } else {
        const int r = i / F, j = i - r * F;
        const int src = j < D ? j : D8 + (j - D);                 // w1p is [hidden][2·D8] (Re | Im padded)
        w1t[j * hidden + r] = WS(w1p[int64_t(r) * 2 * D8 + src]);
      }
    }
  const WS* w1src = kGlobalW1 ? reinterpret_cast<const WS*>(w64) : w1t;
  const double bk = k < hidden ? (W64 ? w64b1[k] : double(b1[k])) : 0.0;
  const double wa = k < hidden ? (W64 ? w64w2[k] : double(w2[k])) : 0.0;
  const double wb = k < hidden ? (W64 ? w64w2[hidden + k] : double(w2[hidden + k])) : 0.0;
  const double b2a = W64 ? w64b2[0] : double(b2[0]), b2b = W64 ? w64b2[1] : double(b2[1]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  for (int64_t e0 = int64_t(blockIdx.x) * kEvPerStep; e0 < n; e0 += int64_t(gridDim.x) * kEvPerStep) {
    for (int i = threadIdx.x; i < kEvPerStep * D; i += blockDim.x) {
      const int u = i / D, c = i - u * D;
      const int64_t e = e0 + u;
      double2 v = make_double2(0.0, 0.0);
      int cnt = 0;
      if (e < n) emb64(ev, e, t0, delta_t, T[c], Q, NQ, W, H, D8, c, v, cnt);
      fs[u * F + c] = v.x;
      fs[u * F + D + c] = v.y;
      if (c == 0) cnts[u] = cnt;
    }
    __syncthreads();
    double oa[kEvPerStep], ob[kEvPerStep];
#pragma unroll
    for (int u = 0; u < kEvPerStep; ++u) oa[u] = ob[u] = 0.0;
    if (k < hidden) {
      double h[kEvPerStep];
#pragma unroll
      for (int u = 0; u < kEvPerStep; ++u) h[u] = 0.0;
      for (int j = 0; j < F; ++j) {
        const double wj = double(w1src[j * hidden + k]);
#pragma unroll
        for (int u = 0; u < kEvPerStep; ++u) h[u] = fma(fs[u * F + j], wj, h[u]);
      }
#pragma unroll
      for (int u = 0; u < kEvPerStep; ++u) {
        const double hr = fmax(h[u] + bk, 0.0);
        oa[u] = hr * wa;
        ob[u] = hr * wb;
      }
    }
#pragma unroll
    for (int u = 0; u < kEvPerStep; ++u)
      for (int o = 16; o > 0; o >>= 1) {
        oa[u] += __shfl_xor_sync(0xffffffffu, oa[u], o);
        ob[u] += __shfl_xor_sync(0xffffffffu, ob[u], o);
      }
    if (lane == 0)
#pragma unroll
      for (int u = 0; u < kEvPerStep; ++u) {
        red[(wid * kEvPerStep + u) * 2] = oa[u];
        red[(wid * kEvPerStep + u) * 2 + 1] = ob[u];
      }
    __syncthreads();
    if (threadIdx.x < kEvPerStep && e0 + threadIdx.x < n) {
      const int u = threadIdx.x;
      double sa = 0.0, sb = 0.0;
      for (int w = 0; w < nw; ++w) {
        sa += red[(w * kEvPerStep + u) * 2];
        sb += red[(w * kEvPerStep + u) * 2 + 1];
      }
      const int64_t e = e0 + u;
      const bool ok = cnts[u] > 0;
      flows[2 * e] = ok ? sa + b2a : nan("");
      flows[2 * e + 1] = ok ? sb + b2b : nan("");
      if (counts) counts[e] = cnts[u];
    }
    __syncthreads();
  }
}

// Direct summation over the query's window in f64 (oracle_encode,
// encoder.py:413-440): mean over the events e with |x_e - x_q| <= δx and
// |y_e - y_q| <= δy of exp(i[(t_e - t_q)/δt·T + (x_e - x_q)/δx·X + (y_e - y_q)/δy·Y]).
// Independent of the grid / modulation formulation (it walks the events of the
// window's pixel runs), so it validates the pooled paths at scale.  Threads =
// (query, channel < D).  emb: (nq, D) complex128; NaN and count 0 for an
// empty window.
__global__ void __launch_bounds__(256) k64_direct(const double* __restrict__ ev, const int64_t* __restrict__ queries,
                                                  int64_t nq, const int* __restrict__ start,
                                                  const uint64_t* __restrict__ val_s, int W, int H, int dx, int dy,
                                                  double delta_t, const double* __restrict__ T,
                                                  const double* __restrict__ X, const double* __restrict__ Y, int D,
                                                  double2* __restrict__ emb, int32_t* __restrict__ counts) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nq * D) return;
  const int64_t qi = i / D;
  const int c = int(i - qi * D);
  const int64_t q = queries[qi];
  const double tq = ev[3 * q];
  const int xq = int(ev[3 * q + 1]), yq = int(ev[3 * q + 2]);
  const double Tc = T[c], Xc = X[c], Yc = Y[c];
  double2 acc = make_double2(0.0, 0.0);
  int cnt = 0;
  for (int y = max(0, yq - dy); y <= min(H - 1, yq + dy); ++y)
    for (int x = max(0, xq - dx); x <= min(W - 1, xq + dx); ++x) {
      const int64_t p = int64_t(y) * W + x;
      const double sp = (double(x - xq) / dx) * Xc + (double(y - yq) / dy) * Yc;
      for (int j = start[p]; j < start[p + 1]; ++j) {
        const double arg = ((ev[3 * int64_t(slot_event(val_s[j]))] - tq) / delta_t) * Tc + sp;
        double sn, cs;
        sincos(arg, &sn, &cs);
        acc.x += cs;
        acc.y += sn;
        ++cnt;
      }
    }
  emb[qi * D + c] = cnt > 0 ? make_double2(acc.x / cnt, acc.y / cnt) : make_double2(nan(""), nan(""));
  if (counts && c == 0) counts[qi] = cnt;
}

}  // namespace

void launch_direct64(const double* ev, const int64_t* queries, int64_t nq, const SortBufs& sb, int W, int H, int dx,
                     int dy, double delta_t, const double* T, const double* X, const double* Y, int D, double2* emb,
                     int32_t* counts, cudaStream_t s) {
  if (nq <= 0) return;
  k64_direct<<<int((nq * D + 255) / 256), 256, 0, s>>>(ev, queries, nq, sb.start, sb.val_s, W, H, dx, dy, delta_t, T,
                                                       X, Y, D, emb, counts);
}

size_t predict64_smem(int D, int hidden, size_t wbytes) {
  return ((size_t(2 * D) * hidden * wbytes + 15) / 16) * 16 + size_t(kEvPerStep) * 2 * D * 8 +
         32 * kEvPerStep * 2 * 8 + kEvPerStep * 4;
}

void launch_encode64(const F64Tables& t, const double* ev, int64_t n, double t0, double delta_t, int W, int H, int D,
                     int D8, int dx, int dy, const SortBufs& sb, const int* NQ, double2* bufA, double2* bufB,
                     cudaStream_t s) {
  const int64_t P = int64_t(W) * H;
  const int ppb = 256 / D8;
  k64_reduce<<<int(std::min<int64_t>((P + ppb - 1) / ppb, 148 * 32)), ppb * D8, 0, s>>>(
      sb.start, sb.val_s, ev, t0, delta_t, t.T, t.mx, t.my, W, P, D8, bufA);
  // segments so each pass runs ~8 threads per (column|row, channel) pair of the
  // grid (a ≥ 4δ-long segment keeps the 2δ warm-up re-reads below half)
  const int RS = std::max(4 * dy, (H + 7) / 8), CS = std::max(4 * dx, (W + 7) / 8);
  k64_box_y<<<dim3(unsigned((int64_t(W) * D8 + 255) / 256), unsigned((H + RS - 1) / RS)), 256, 0, s>>>(
      bufA, bufB, W, H, D8, dy, RS);
  k64_box_x<<<dim3(unsigned((int64_t(H) * D8 + 255) / 256), unsigned((W + CS - 1) / CS)), 256, 0, s>>>(
      bufB, bufA, W, H, D8, dx, CS, t.mx, t.my);
  (void)n;
  (void)NQ;
}

void launch_features64(const F64Tables& t, const double* ev, int64_t n, double t0, double delta_t, int W, int H,
                       int D, int D8, const double2* Q, const int* NQ, double* feats, int32_t* counts,
                       cudaStream_t s) {
  if (n <= 0) return;
  k64_features<<<int((n * D + 255) / 256), 256, 0, s>>>(ev, n, t0, delta_t, t.T, Q, NQ, W, H, D, D8, feats, counts);
}

void launch_predict64(const F64Tables& t, const double* ev, int64_t n, double t0, double delta_t, int W, int H, int D,
                      int D8, const double2* Q, const int* NQ, const MlpDev& m, double* flows, int32_t* counts,
                      int num_sms, cudaStream_t s) {
  if (n <= 0) return;
  const int threads = std::max(32, (m.hidden + 31) / 32 * 32);
  const int blocks = int(std::min<int64_t>((n + kEvPerStep - 1) / kEvPerStep, int64_t(num_sms) * 4));
  // f32 W1ᵀ in shared memory (promoted per use): twice the resident blocks of
  // an f64 copy, which measured 1.5x slower (4 warps per SM at 128 KB)
  const size_t smem64 = predict64_smem(D, m.hidden, 8);
  auto go = [&](auto kern, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    kern<<<blocks, threads, smem, s>>>(ev, n, t0, delta_t, t.T, Q, NQ, W, H, D, D8, m.w1, m.b1, m.w2, m.b2, m.w64,
                                       m.hidden, flows, counts);
  };
  if (m.w64) {   // float64 weights: never rounded to f32
    if (smem64 <= 200 * 1024)
      go(k64_predict<double, true>, smem64);
    else
      go(k64_predict<void, true>, predict64_smem(D, m.hidden, 0));
  } else if (smem64 <= 64 * 1024) {   // f64 copy only for small heads
    go(k64_predict<double, false>, smem64);
  } else {
    go(k64_predict<float, false>, predict64_smem(D, m.hidden, 4));
  }
}

}  // namespace vkm
