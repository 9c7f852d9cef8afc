// Head training on the GPU (train_head / flow_loss_grads, flow.py:234-402):
// mini-batch Adam on the constraint loss in float64, the reference's exact
// formulas, with the data set's features resident in HBM.
//
//   k_tr_batch  one CTA per 32 samples of a mini-batch (or of the validation
//               set): forward (pre = F·W1ᵀ + b1, act = relu, out = act·W2ᵀ + b2),
//               the loss terms r²/(|u|²+eps) and max(0, margin-|out|)², and —
//               for a training step — the backward pass of flow_loss_grads
//               (flow.py:282-301) with per-CTA partial parameter gradients
//   k_tr_adam   sums the CTA partials in a fixed order (deterministic) and
//               applies the Adam update of train_head (flow.py:378-385)
//
// Device parameter layout: W1ᵀ [F][H] (F = 2D features, H hidden), b1 [H],
// W2 [2][H], b2 [2]; Adam m, v in the same layout.
#include <cmath>
#include <cstdint>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

namespace {

constexpr int kTrRows = 32;   // samples per CTA

struct TrParams {
  const double* w1t;   // [F][H]
  const double* b1;    // [H]
  const double* w2;    // [2][H]
  const double* b2;    // [2]
};

// Shared memory: fs [32][F], pre [32][H] (reused for dpre), out/dout [32][2]
__global__ void k_tr_batch(const double* __restrict__ feats, const double* __restrict__ u,
                           const int64_t* __restrict__ idx, int64_t nb, int F, int H, TrParams p, double margin,
                           double mw, double eps, double inv_n, int with_grads, double* __restrict__ loss_part,
                           double* __restrict__ g_part) {
  extern __shared__ __align__(16) double trs[];
  double* fs = trs;                    // [32][F]
  double* pre = fs + kTrRows * F;      // [32][H]
  double* od = pre + kTrRows * H;      // [32][2] out, then dout
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t r0 = int64_t(blockIdx.x) * kTrRows;
  const int rows = nb - r0 < kTrRows ? int(nb - r0) : kTrRows;
  for (int i = tid; i < kTrRows * F; i += nt) {
    const int s = i / F, j = i - s * F;
    fs[i] = s < rows ? feats[idx[r0 + s] * F + j] : 0.0;
  }
  __syncthreads();
  // pre[s][k] = b1[k] + Σ_j F[s][j]·W1[k][j]
  for (int k = tid; k < H; k += nt) {
    double acc[kTrRows];
#pragma unroll
    for (int s = 0; s < kTrRows; ++s) acc[s] = 0.0;
    for (int j = 0; j < F; ++j) {
      const double w = p.w1t[int64_t(j) * H + k];
#pragma unroll
      for (int s = 0; s < kTrRows; ++s) acc[s] = fma(fs[s * F + j], w, acc[s]);
    }
#pragma unroll
    for (int s = 0; s < kTrRows; ++s) pre[s * H + k] = acc[s] + p.b1[k];
  }
  __syncthreads();
  // out, loss terms and dout, one thread per sample (flow.py:273-293)
  double l1 = 0.0, l2 = 0.0;
  if (tid < rows) {
    const int s = tid;
    double o0 = p.b2[0], o1 = p.b2[1];
    for (int k = 0; k < H; ++k) {
      const double a = fmax(pre[s * H + k], 0.0);
      o0 = fma(a, p.w2[k], o0);
      o1 = fma(a, p.w2[H + k], o1);
    }
    const double u0 = u[2 * idx[r0 + s]], u1 = u[2 * idx[r0 + s] + 1];
    const double r = o0 * (u0 - o0) + o1 * (u1 - o1);
    const double denom = u0 * u0 + u1 * u1 + eps;
    const double norm = sqrt(o0 * o0 + o1 * o1);
    const double gap = fmax(0.0, margin - norm);
    l1 = r * r / denom;
    l2 = gap * gap;
    double d0 = (2.0 * r / denom) * (u0 - 2.0 * o0) * inv_n;   // d term1 / d out
    double d1 = (2.0 * r / denom) * (u1 - 2.0 * o1) * inv_n;
    if (gap > 0.0 && norm > 0.0) {                             // d term2 / d out (hinge active)
      const double c = (-2.0 * mw * gap / norm) * inv_n;
      d0 += c * o0;
      d1 += c * o1;
    }
    od[2 * s] = d0;
    od[2 * s + 1] = d1;
  } else if (tid < kTrRows) {
    od[2 * tid] = od[2 * tid + 1] = 0.0;
  }
  // per-CTA loss partials (fixed-order warp reduction over the 32 samples)
  if (tid < 32) {
    for (int o = 16; o > 0; o >>= 1) {
      l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      l2 += __shfl_xor_sync(0xffffffffu, l2, o);
    }
    if (tid == 0) {
      loss_part[2 * blockIdx.x] = l1;
      loss_part[2 * blockIdx.x + 1] = l2;
    }
  }
  if (!with_grads) return;
  __syncthreads();
  // gradients of the parameters (flow.py:295-301), partial over this CTA's samples
  const int64_t G = int64_t(F) * H + 3 * int64_t(H) + 2;   // gradient vector length
  double* gp = g_part + int64_t(blockIdx.x) * G;
  for (int k = tid; k < H; k += nt) {
    double gw0 = 0.0, gw1 = 0.0, gb1 = 0.0;
    const double w20 = p.w2[k], w21 = p.w2[H + k];
    for (int s = 0; s < kTrRows; ++s) {
      const double pk = pre[s * H + k];
      const double a = fmax(pk, 0.0);
      gw0 = fma(od[2 * s], a, gw0);          // dW2 = doutᵀ·act
      gw1 = fma(od[2 * s + 1], a, gw1);
      const double dpre = pk > 0.0 ? od[2 * s] * w20 + od[2 * s + 1] * w21 : 0.0;   // dact·(pre > 0)
      pre[s * H + k] = dpre;
      gb1 += dpre;
    }
    gp[int64_t(F) * H + k] = gb1;            // db1
    gp[int64_t(F) * H + H + k] = gw0;        // dW2[0]
    gp[int64_t(F) * H + 2 * H + k] = gw1;    // dW2[1]
  }
  if (tid < 2) {
    double gb = 0.0;
    for (int s = 0; s < kTrRows; ++s) gb += od[2 * s + tid];
    gp[int64_t(F) * H + 3 * H + tid] = gb;   // db2
  }
  __syncthreads();
  // dW1ᵀ[j][k] = Σ_s F[s][j]·dpre[s][k]
  for (int64_t i = tid; i < int64_t(F) * H; i += nt) {
    const int j = int(i / H), k = int(i - int64_t(j) * H);
    double acc = 0.0;
    for (int s = 0; s < kTrRows; ++s) acc = fma(fs[s * F + j], pre[s * H + k], acc);
    gp[i] = acc;
  }
}

// Sum of the nblk partial gradients (fixed order), then Adam (flow.py:378-385).
// Also flags the first step with a non-finite loss (the reference raises
// TrainingDivergedError there, flow.py:372-376).
__global__ void k_tr_adam(double* __restrict__ prm, double* __restrict__ m, double* __restrict__ v,
                          const double* __restrict__ g_part, int nblk, int64_t G, double lr, double b1c, double b2c,
                          const double* __restrict__ loss_part, double mw, double inv_n, int64_t step,
                          int64_t* __restrict__ bad_step) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) {
    double l1 = 0.0, l2 = 0.0;
    for (int b = 0; b < nblk; ++b) {
      l1 += loss_part[2 * b];
      l2 += loss_part[2 * b + 1];
    }
    const double loss = l1 * inv_n + mw * (l2 * inv_n);
    if (!isfinite(loss) && *bad_step < 0) *bad_step = step;
  }
  if (i >= G) return;
  double g = 0.0;
  for (int b = 0; b < nblk; ++b) g += g_part[int64_t(b) * G + i];
  // numpy's operation order, each product and sum rounded (no FMA contraction)
  const double beta1 = 0.9, beta2 = 0.999, adam_eps = 1e-8;
  const double mi = __dadd_rn(__dmul_rn(beta1, m[i]), __dmul_rn(1.0 - beta1, g));
  const double vi = __dadd_rn(__dmul_rn(beta2, v[i]), __dmul_rn(__dmul_rn(1.0 - beta2, g), g));
  m[i] = mi;
  v[i] = vi;
  const double m_hat = mi / b1c, v_hat = vi / b2c;
  prm[i] = __dsub_rn(prm[i], __dmul_rn(lr, m_hat) / __dadd_rn(sqrt(v_hat), adam_eps));
}

}  // namespace

size_t train_batch_smem(int F, int H) { return sizeof(double) * (size_t(kTrRows) * (F + H) + 2 * kTrRows); }
int train_rows_per_cta() { return kTrRows; }

// One pass over nb samples idx (device) with the parameters prm (device,
// packed layout): loss partials per CTA into loss_part; with_grads adds the
// backward pass and one Adam step.
void launch_train_batch(const double* feats, const double* u, const int64_t* idx, int64_t nb, int F, int H,
                        double* prm, double* m, double* v, double margin, double mw, double eps, int with_grads,
                        double lr, int64_t step, double* loss_part, double* g_part, int64_t* bad_step,
                        cudaStream_t s) {
  if (nb <= 0) return;
  const int64_t FH = int64_t(F) * H;
  const TrParams p{prm, prm + FH, prm + FH + H, prm + FH + 3 * H};
  const int nblk = int((nb + kTrRows - 1) / kTrRows);
  const size_t smem = train_batch_smem(F, H);
  cudaFuncSetAttribute(k_tr_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int threads = H >= 256 ? 256 : (H > 128 ? 256 : 128);
  k_tr_batch<<<nblk, threads, smem, s>>>(feats, u, idx, nb, F, H, p, margin, mw, eps, 1.0 / double(nb), with_grads,
                                         loss_part, g_part);
  if (!with_grads) return;
  // G layout matches TrParams: W1ᵀ | b1 | W2[0] | W2[1] | b2
  const int64_t G = FH + 3 * int64_t(H) + 2;
  const double b1c = 1.0 - std::pow(0.9, double(step)), b2c = 1.0 - std::pow(0.999, double(step));
  k_tr_adam<<<int((G + 255) / 256), 256, 0, s>>>(prm, m, v, g_part, nblk, G, lr, b1c, b2c, loss_part, mw,
                                                  1.0 / double(nb), step, bad_step);
}

}  // namespace vkm
