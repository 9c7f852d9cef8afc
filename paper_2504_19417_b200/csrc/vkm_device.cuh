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
// sin/cos of an f32 argument.  2-part Cody-Waite reduction by pi/2 (the
// third part, q·5.4e-15, stays below 1e-12 for |x| < 1e3 — far under f32
// resolution — and is left out) and minimax polynomials on [-pi/4, pi/4]
// (coefficients fitted for this project, tools in DESIGN.md).  Max error
// 1.42 ulp / 7.3e-8 abs over |x| < 60; agrees bit-for-bit with numpy's
// float32 sin/cos on 98.9% of arguments and within 1 ulp elsewhere.  Valid
// for |x| < ~1e3 (phase arguments here are < 100).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sincos_f32(float x, float& s, float& c) {
  // q = rint(x·2/π) via the 1.5·2^23 magic constant (exact for |x·2/π| < 2^22):
  // stays on the FMA/ALU pipes; the low mantissa bits carry the quadrant.
  const float qb = fmaf(x, 0.636619772f, 12582912.0f);
  const float q = __fsub_rn(qb, 12582912.0f);
  float r = fmaf(q, -1.57079601e+00f, x);
  r = fmaf(q, -3.13916473e-07f, r);
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
  const int k = __float_as_int(qb);
  const float ss = (k & 1) ? cr : sr;
  const float cc = (k & 1) ? sr : cr;
  s = __int_as_float(__float_as_int(ss) ^ ((k & 2) << 30));
  c = __int_as_float(__float_as_int(cc) ^ (((k + 1) & 2) << 30));
}

// Packed f32x2 helpers (Blackwell FFMA2 / FMUL2): two lanes per instruction,
// each lane IEEE round-to-nearest exactly like the scalar op.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fneg2(uint64_t a) { return a ^ 0x8000000080000000ull; }

// Two sin/cos evaluations at once, bit-identical to two sincos_f32 calls
// (same operations, paired into f32x2 instructions).
__device__ __forceinline__ void sincos2_f32(float x0, float x1, float& s0, float& c0, float& s1, float& c1) {
  const uint64_t x = f2pack(x0, x1);
  const uint64_t magic = f2pack(12582912.0f, 12582912.0f);
  const uint64_t qb = ffma2(x, f2pack(0.636619772f, 0.636619772f), magic);   // rint(x·2/π) in the low bits
  const uint64_t q = fsub2(qb, magic);
  uint64_t r = ffma2(q, f2pack(-1.57079601e+00f, -1.57079601e+00f), x);
  r = ffma2(q, f2pack(-3.13916473e-07f, -3.13916473e-07f), r);
  const uint64_t u = fmul2(r, r);
  uint64_t ps = ffma2(f2pack(2.718123369e-06f, 2.718123369e-06f), u, f2pack(-1.983931288e-04f, -1.983931288e-04f));
  ps = ffma2(ps, u, f2pack(8.333329111e-03f, 8.333329111e-03f));
  ps = ffma2(ps, u, f2pack(-1.666666716e-01f, -1.666666716e-01f));
  ps = fmul2(ps, u);
  const uint64_t sr = ffma2(ps, r, r);
  uint64_t pc = ffma2(f2pack(2.438358570e-05f, 2.438358570e-05f), u, f2pack(-1.388668199e-03f, -1.388668199e-03f));
  pc = ffma2(pc, u, f2pack(4.166661948e-02f, 4.166661948e-02f));
  pc = ffma2(pc, u, f2pack(-5.000000000e-01f, -5.000000000e-01f));
  const uint64_t cr = ffma2(pc, u, f2pack(1.0f, 1.0f));
  float sr0, sr1, cr0, cr1, qb0, qb1;
  f2unpack(sr, sr0, sr1);
  f2unpack(cr, cr0, cr1);
  f2unpack(qb, qb0, qb1);
  const int k0 = __float_as_int(qb0), k1 = __float_as_int(qb1);
  float ss = (k0 & 1) ? cr0 : sr0, cc = (k0 & 1) ? sr0 : cr0;
  s0 = __int_as_float(__float_as_int(ss) ^ ((k0 & 2) << 30));
  c0 = __int_as_float(__float_as_int(cc) ^ (((k0 + 1) & 2) << 30));
  ss = (k1 & 1) ? cr1 : sr1;
  cc = (k1 & 1) ? sr1 : cr1;
  s1 = __int_as_float(__float_as_int(ss) ^ ((k1 & 2) << 30));
  c1 = __int_as_float(__float_as_int(cc) ^ (((k1 + 1) & 2) << 30));
}

// Two sin/cos pairs with the reduction by pi (r in [-pi/2, pi/2]): the only
// quadrant fix-up is a common sign (-1)^k, applied with one shift and one
// LOP3 per value, so the whole evaluation is 15 packed FMA-pipe instructions
// plus 6 integer ones (31 for sincos2p_f32).  Degree-9 sin / degree-10 cos
// minimax polynomials (tools/fit_sincos.py; degrees 11/12 measured the same
// f32 error, the evaluation rounding dominates): max abs error 1.4e-7 over
// |x| < 60 (sincos2p_f32: 7.3e-8), i.e. ~2.5 ulp of 1.0.
__device__ __forceinline__ void sincos2p_pi(uint64_t x, uint64_t& s01, uint64_t& c01) {
  const uint64_t magic = f2pack(12582912.0f, 12582912.0f);
  const uint64_t qb = ffma2(x, f2pack(0.318309886f, 0.318309886f), magic);
  const uint64_t q = fsub2(qb, magic);
  uint64_t r = ffma2(q, f2pack(-3.14159203e+00f, -3.14159203e+00f), x);
  r = ffma2(q, f2pack(-6.27832946e-07f, -6.27832946e-07f), r);
  const uint64_t u = fmul2(r, r);
  uint64_t ps = ffma2(f2pack(2.600054358e-06f, 2.600054358e-06f), u, f2pack(-1.980661473e-04f, -1.980661473e-04f));
  ps = ffma2(ps, u, f2pack(8.333017118e-03f, 8.333017118e-03f));
  ps = ffma2(ps, u, f2pack(-1.666665673e-01f, -1.666665673e-01f));
  ps = fmul2(ps, u);
  const uint64_t sr = ffma2(ps, r, r);
  uint64_t pc = ffma2(f2pack(-2.607710599e-07f, -2.607710599e-07f), u, f2pack(2.476188638e-05f, 2.476188638e-05f));
  pc = ffma2(pc, u, f2pack(-1.388840377e-03f, -1.388840377e-03f));
  pc = ffma2(pc, u, f2pack(4.166664183e-02f, 4.166664183e-02f));
  pc = ffma2(pc, u, f2pack(-5.000000000e-01f, -5.000000000e-01f));
  const uint64_t cr = ffma2(pc, u, f2pack(1.0f, 1.0f));
  // (-1)^k: the parity of k sits in bit 0 of each f32 lane of qb
  const uint64_t sgn = (qb << 31) & 0x8000000080000000ull;
  s01 = sr ^ sgn;
  c01 = cr ^ sgn;
}

// theta = (x0, x1) -> (cos x0, sin x0), (cos x1, sin x1): the quadrant
// fix-up writes scalars anyway, so pairing each argument's cos and sin costs
// nothing and lets a complex accumulator (re, im) add them with one add.f32x2.
__device__ __forceinline__ void sincos2_cs(uint64_t theta, uint64_t& cs0, uint64_t& cs1) {
  float x0, x1, s0, c0, s1, c1;
  f2unpack(theta, x0, x1);
  sincos2_f32(x0, x1, s0, c0, s1, c1);
  cs0 = f2pack(c0, s0);
  cs1 = f2pack(c1, s1);
}

// sincos2p_pi with a per-pair scale folded into the sign fix-up:
// s01 = scale·sin, c01 = scale·cos (scale01 = (k0, k1)).  The quadrant sign
// rides on the scale (one 64-bit XOR), so scaling costs two mul.f32x2 in
// place of the four sign XORs.
__device__ __forceinline__ void sincos2p_pi_scaled(uint64_t x, uint64_t scale01, uint64_t& s01, uint64_t& c01) {
  const uint64_t magic = f2pack(12582912.0f, 12582912.0f);
  const uint64_t qb = ffma2(x, f2pack(0.318309886f, 0.318309886f), magic);
  const uint64_t q = fsub2(qb, magic);
  uint64_t r = ffma2(q, f2pack(-3.14159203e+00f, -3.14159203e+00f), x);
  r = ffma2(q, f2pack(-6.27832946e-07f, -6.27832946e-07f), r);
  const uint64_t u = fmul2(r, r);
  uint64_t ps = ffma2(f2pack(2.600054358e-06f, 2.600054358e-06f), u, f2pack(-1.980661473e-04f, -1.980661473e-04f));
  ps = ffma2(ps, u, f2pack(8.333017118e-03f, 8.333017118e-03f));
  ps = ffma2(ps, u, f2pack(-1.666665673e-01f, -1.666665673e-01f));
  ps = fmul2(ps, u);
  const uint64_t sr = ffma2(ps, r, r);
  uint64_t pc = ffma2(f2pack(-2.607710599e-07f, -2.607710599e-07f), u, f2pack(2.476188638e-05f, 2.476188638e-05f));
  pc = ffma2(pc, u, f2pack(-1.388840377e-03f, -1.388840377e-03f));
  pc = ffma2(pc, u, f2pack(4.166664183e-02f, 4.166664183e-02f));
  pc = ffma2(pc, u, f2pack(-5.000000000e-01f, -5.000000000e-01f));
  const uint64_t cr = ffma2(pc, u, f2pack(1.0f, 1.0f));
  const uint64_t f = scale01 ^ ((qb << 31) & 0x8000000080000000ull);
  s01 = fmul2(sr, f);
  c01 = fmul2(cr, f);
}

// Argument reduction ahead of sin.approx / cos.approx (which scale by 1/2π
// with round-toward-zero and take the fraction of a turn: the absolute error
// of that scaled argument grows with |x|).  VKM_MUFU_RED selects
//   2 (default) rint(x / 2π) and a two-part Cody-Waite step: 4 FMA-pipe ops
//   1           one Cody-Waite term (error k·1.7e-7 more): 3 ops
//   0           none (|x| <= ~14 here, so the turn fraction keeps ~22 bits)
#ifndef VKM_MUFU_RED
#define VKM_MUFU_RED 2
#endif
__device__ __forceinline__ uint64_t mufu_reduce2(uint64_t x) {
#if VKM_MUFU_RED == 0
  return x;
#else
  const uint64_t magic = f2pack(12582912.0f, 12582912.0f);
  const uint64_t qb = ffma2(x, f2pack(0.159154943f, 0.159154943f), magic);   // rint(x / 2π)
  const uint64_t q = fsub2(qb, magic);
  uint64_t r = ffma2(q, f2pack(-6.28318548e+00f, -6.28318548e+00f), x);
#if VKM_MUFU_RED >= 2
  r = ffma2(q, f2pack(1.74845553e-07f, 1.74845553e-07f), r);
#endif
  return r;
#endif
}

// Special-function-unit variant: reduction by 2π (two-part Cody-Waite) to
// [-π, π], then MUFU.SIN / MUFU.COS (sin.approx: max abs error 2^-21.4 there,
// ~3 ulp of 1.0), the per-pair scale applied last.  Four XU-pipe and five
// FMA-pipe instructions per pair instead of ~17 FMA-pipe: for kernels whose
// producers are FMA-pipe bound (K3's de-phase).
__device__ __forceinline__ void sincos2_mufu_scaled(uint64_t x, uint64_t scale01, uint64_t& s01, uint64_t& c01) {
  const uint64_t r = mufu_reduce2(x);
  float r0, r1;
  f2unpack(r, r0, r1);
  float s0, s1, c0, c1;
  asm("sin.approx.f32 %0, %1;" : "=f"(s0) : "f"(r0));
  asm("sin.approx.f32 %0, %1;" : "=f"(s1) : "f"(r1));
  asm("cos.approx.f32 %0, %1;" : "=f"(c0) : "f"(r0));
  asm("cos.approx.f32 %0, %1;" : "=f"(c1) : "f"(r1));
  s01 = fmul2(f2pack(s0, s1), scale01);
  c01 = fmul2(f2pack(c0, c1), scale01);
}

// Packed-in/packed-out variant: theta = (x0, x1), returns (s0, s1), (c0, c1).
__device__ __forceinline__ void sincos2p_f32(uint64_t theta, uint64_t& s01, uint64_t& c01) {
  float x0, x1, s0, c0, s1, c1;
  f2unpack(theta, x0, x1);
  sincos2_f32(x0, x1, s0, c0, s1, c1);
  s01 = f2pack(s0, s1);
  c01 = f2pack(c0, c1);
}

// sin/cos used by the two hot kernels (k_reduce_x, k_gather_mlp_tc).  The
// pi-reduced variant issues fewer instructions per pair but
// measured no faster on B200 (both kernels are dependency-latency bound:
// k_reduce_x 128 -> 132 us, K3 ~equal, ncu cfg2) and is 2x less accurate, so
// the pi/2-reduced version is the default; -DVKM_SINCOS_PI selects the other.
__device__ __forceinline__ void sincos2p_mufu(uint64_t x, uint64_t& s01, uint64_t& c01) {
  const uint64_t r = mufu_reduce2(x);
  float r0, r1, s0, s1, c0, c1;
  f2unpack(r, r0, r1);
  asm("sin.approx.f32 %0, %1;" : "=f"(s0) : "f"(r0));
  asm("sin.approx.f32 %0, %1;" : "=f"(s1) : "f"(r1));
  asm("cos.approx.f32 %0, %1;" : "=f"(c0) : "f"(r0));
  asm("cos.approx.f32 %0, %1;" : "=f"(c1) : "f"(r1));
  s01 = f2pack(s0, s1);
  c01 = f2pack(c0, c1);
}
// The hot kernels (k_reduce_x, k_gather_mlp_tc) take the sin/cos flavour as
// a template parameter chosen at run time (sincos_mufu(), VKM_SINCOS):
//   MUFU (default)  2π reduction + sin.approx/cos.approx on the special-function
//                   unit: ~5e-7 absolute, 4 XU + 5 FMA-pipe instructions per
//                   pair.  Both kernels are FMA-pipe bound, so moving the
//                   polynomials off that pipe pays: cfg2 K1 0.168 -> 0.134 ms,
//                   K3 0.134 -> 0.130 ms; flows vs the reference unchanged
//                   (<= 7.2e-7 over the goldens).
//   poly            the Cody-Waite + minimax polynomials below (1.4 ulp, the
//                   same f32 phase as numpy on 98.9 % of arguments).
template <bool kMufu>
__device__ __forceinline__ void sincos2_hot(uint64_t x, uint64_t& s01, uint64_t& c01) {
  if constexpr (kMufu)
    sincos2p_mufu(x, s01, c01);
  else
    sincos2p_f32(x, s01, c01);
}
template <bool kMufu>
__device__ __forceinline__ void sincos2_cs_hot(uint64_t theta, uint64_t& cs0, uint64_t& cs1) {
  if constexpr (kMufu) {   // (cos, sin) pairs of the two arguments
    uint64_t s01, c01;
    sincos2p_mufu(theta, s01, c01);
    float s0, s1, c0, c1;
    f2unpack(s01, s0, s1);
    f2unpack(c01, c0, c1);
    cs0 = f2pack(c0, s0);
    cs1 = f2pack(c1, s1);
  } else {
    sincos2_cs(theta, cs0, cs1);
  }
}
template <bool kMufu>
__device__ __forceinline__ void sincos2_k3_scaled(uint64_t x, uint64_t scale01, uint64_t& s01, uint64_t& c01) {
  if constexpr (kMufu)
    sincos2_mufu_scaled(x, scale01, s01, c01);
  else
    sincos2p_pi_scaled(x, scale01, s01, c01);
}
#define VKM_SINCOS_CS sincos2_cs

// a = f32((t - t0) / delta_t): f64 rebase and divide, then one rounding to f32,
// exactly as rebase_slice (events.py:390-407) + _temporal_phases
// (encoder.py:220-226) do on the host.
__device__ __forceinline__ float time_arg(double t, double t0, double delta_t) {
  return __double2float_rn((t - t0) / delta_t);
}

// Pooled-grid (Q) layout: per channel plane, 64 bytes per pixel = four
// 16-byte chunks (channel pairs).  Chunk c of pixel p is stored in slot
// c ^ qswz(p), so lanes reading the same chunk of consecutive pixels (K3's
// gathers of a pixel-sorted tile) hit eight distinct 16-byte bank groups
// instead of two.  Every writer (y pass, split x pass) and reader (K3, the
// encoder features, the grid export) goes through qswz.  Measured (v29,
// profiles/r02/q_swizzle_ab_v29.txt): correct, but K3 15 % slower at cfg 2
// (run-time chunk offsets: more registers, spills) and the y pass +3 %, so
// the linear layout (0) is the default; qswz then folds to 0.
#ifndef VKM_Q_SWZ
#define VKM_Q_SWZ 0
#endif
__host__ __device__ __forceinline__ int qswz(int64_t p) { return VKM_Q_SWZ ? int((p >> 1) & 3) : 0; }

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

namespace vkm {
// Programmatic dependent launch (PDL).  A kernel launched with
// Decoupled look-back for single-pass scans (k_scan, k_select_strip): tile t
// publishes its aggregate, reads its predecessors' published words 32 at a
// time (aggregates until the nearest inclusive prefix) and publishes its own
// inclusive prefix.  A word packs (epoch:30, flag:2, value:32); words of other
// launches carry another epoch and read as unpublished, so the state array is
// never reset.  Call with one full warp; every lane returns the exclusive
// prefix.  Tiles must be taken in increasing order by co-resident blocks.
__device__ __forceinline__ uint64_t lb_word(uint32_t epoch, uint64_t flag, uint32_t value) {
  return (uint64_t(epoch & 0x3fffffffu) << 34) | (flag << 32) | value;
}
__device__ __forceinline__ uint32_t lookback_publish(unsigned long long* state, int t, uint32_t total,
                                                     uint32_t epoch) {
  volatile unsigned long long* vs = state;
  const int lane = threadIdx.x & 31;
  const uint32_t ep = epoch & 0x3fffffffu;
  if (t == 0) {
    if (lane == 0) vs[0] = lb_word(ep, 2, total);
    return 0;
  }
  if (lane == 0) vs[t] = lb_word(ep, 1, total);
  uint32_t excl = 0;
  for (int p = t - 1;; p -= 32) {
    const int q = p - lane;
    uint64_t w = 0;
    if (q >= 0)
      do w = vs[q]; while (uint32_t(w >> 34) != ep || ((w >> 32) & 3) == 0);
    const unsigned incl = __ballot_sync(0xffffffffu, q >= 0 && ((w >> 32) & 3) == 2);
    const int stop = incl ? __ffs(incl) - 1 : 31;   // nearest predecessor carrying a prefix
    uint32_t add = (lane <= stop && q >= 0) ? uint32_t(w) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
    excl += add;
    if (incl || p - 32 < 0) break;
  }
  if (lane == 0) vs[t] = lb_word(ep, 2, excl + total);
  return excl;
}

// launch_pdl() may be scheduled while its predecessor drains: each kernel
// executes pdl_wait() before touching anything its predecessor writes and
// pdl_trigger() when its own work is done, so the next grid's launch and
// prologue overlap this grid's tail.  (Triggering at the start instead let
// waiting CTAs of two successors crowd out multi-wave grids: cfg3 K1 +28 %.)
// Both are no-ops for plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
}  // namespace vkm

#ifndef __CUDACC_RTC__
#include <utility>
namespace vkm {
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace vkm
#endif

namespace vkm {
// L2 cache-policy helpers (createpolicy + .L2::cache_hint).
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float2 ld_hint(const float2* ptr, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y)
               : "l"(ptr), "l"(pol));
  return v;
}
// Same load without `volatile`: the compiler may batch and reorder it (the data
// is read-only for the kernel's lifetime).
__device__ __forceinline__ float2 ld_nc_hint(const float2* ptr, uint64_t pol) {
  float2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
      : "=f"(v.x), "=f"(v.y)
      : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(float2* ptr, float2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(ptr), "f"(v.x), "f"(v.y),
               "l"(pol)
               : "memory");
}
}  // namespace vkm

namespace vkm {
// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, non-tensor) helpers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
// Bounded parity wait: a protocol bug traps instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_addr(b);
  for (uint32_t it = 0;; ++it) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) return;
    if (it > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// shared -> global bulk copy (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
}  // namespace vkm
