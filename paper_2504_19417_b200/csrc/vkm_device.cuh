// Device helpers shared by the VecKM_flow kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vkm {

// Grid layout in HBM:
//   G[plane][y][x][8] complex64   plane = channel / 8, 64 B per pixel per plane
//   C[y][x] int32                 per-pixel event counts
// The pooled grid Q / pooled counts NQ use the same layout.
constexpr int kPlaneCh = 8;

struct SliceGeom {
  int W, H;        // sensor size
  int dx, dy;      // window radii
  int64_t P;       // W * H
};

// ---------------------------------------------------------------------------
// sin/cos of an f32 argument.  3-part Cody-Waite reduction by pi/2 and
// minimax polynomials on [-pi/4, pi/4] (coefficients fitted for this project,
// tools in DESIGN.md).  Max error 1.42 ulp / 7.3e-8 abs over |x| < 60; agrees
// bit-for-bit with numpy's float32 sin/cos on 98.9% of arguments and within
// 1 ulp elsewhere.  Valid for |x| < ~1e5 (phase arguments here are < 100).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sincos_f32(float x, float& s, float& c) {
  const float q = rintf(x * 0.636619772f);
  float r = fmaf(q, -1.57079601e+00f, x);
  r = fmaf(q, -3.13916473e-07f, r);
  r = fmaf(q, -5.39030253e-15f, r);
  const float u = r * r;
  float ps = 2.718123369e-06f;
  ps = fmaf(ps, u, -1.983931288e-04f);
  ps = fmaf(ps, u, 8.333329111e-03f);
  ps = fmaf(ps, u, -1.666666716e-01f);
  ps = ps * u;
  const float sr = fmaf(ps, r, r);
  float pc = 2.438358570e-05f;
  pc = fmaf(pc, u, -1.388668199e-03f);
  pc = fmaf(pc, u, 4.166661948e-02f);
  pc = fmaf(pc, u, -5.000000000e-01f);
  const float cr = fmaf(pc, u, 1.0f);
  const int k = __float2int_rn(q);
  float ss = (k & 1) ? cr : sr;
  float cc = (k & 1) ? sr : cr;
  s = (k & 2) ? -ss : ss;
  c = ((k + 1) & 2) ? -cc : cc;
}

// a = f32((t - t0) / delta_t): f64 rebase and divide, then one rounding to f32,
// exactly as rebase_slice (events.py:390-407) + _temporal_phases
// (encoder.py:220-226) do on the host.
__device__ __forceinline__ float time_arg(double t, double t0, double delta_t) {
  return __double2float_rn((t - t0) / delta_t);
}

// Complex product with explicit rounding (no FMA contraction): numpy's
// complex64 multiply order (encoder.py:334, 345).
__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
  return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                     __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}
// Fast complex multiply-accumulate helpers for the pooling passes.
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

__device__ __forceinline__ double ld_t0(const double* ev, double t0) {
  return isnan(t0) ? __ldg(ev) : t0;
}

}  // namespace vkm
