// Host-side event packing for the pipelined host batch (vkm_predict_batch_host
// with 8-byte records): rows of the reference's (n, 3) f64 [t, x, y] layout ->
// {f32 bits of a = f32((t - t0)/δt), x | y << 16 or 0xFFFFFFFF}.  The time
// argument is the same IEEE f64 subtract and divide, rounded once to f32, as
// k_prep's time_arg on the device (and rebase_slice + _temporal_phases in the
// reference, events.py:390-407, encoder.py:220-226), so both paths produce
// bit-identical records.  Plain C++ (no CUDA): AVX-512 / AVX2 kernels chosen
// at run time, a scalar loop for the tail and for CPUs without AVX2.
#include <immintrin.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "host_pool.h"

namespace vkm_host {

namespace {

void pack_scalar(const double* r, int64_t m, double t0, double dt, int W, int H, uint32_t* out) {
  for (int64_t i = 0; i < m; ++i) {
    const double t = r[3 * i], x = r[3 * i + 1], y = r[3 * i + 2];
    const float a = float((t - t0) / dt);
    uint32_t ab;
    std::memcpy(&ab, &a, 4);
    // clamp before the conversion (out-of-range doubles -> int is undefined)
    const double xc = std::fmin(std::fmax(x, -1.0), double(W)), yc = std::fmin(std::fmax(y, -1.0), double(H));
    const int xi = int(xc), yi = int(yc);
    const bool ok = x >= 0.0 && x < W && y >= 0.0 && y < H && double(xi) == x && double(yi) == y;
    out[2 * i] = ab;
    out[2 * i + 1] = ok ? (uint32_t(xi) | (uint32_t(yi) << 16)) : 0xFFFFFFFFu;
  }
}

__attribute__((target("avx2,fma"))) void pack_avx2(const double* r, int64_t m, double t0, double dt, int W, int H,
                                                    uint32_t* out) {
  const __m256d vt0 = _mm256_set1_pd(t0), vdt = _mm256_set1_pd(dt), vW = _mm256_set1_pd(W), vH = _mm256_set1_pd(H);
  const __m256d z = _mm256_setzero_pd(), m1 = _mm256_set1_pd(-1.0);
  const __m256i even = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  int64_t i = 0;
  for (; i + 4 <= m; i += 4) {
    const double* p = r + 3 * i;
    // a0 = t0 x0 y0 t1 | a1 = x1 y1 t2 x2 | a2 = y2 t3 x3 y3
    const __m256d a0 = _mm256_loadu_pd(p), a1 = _mm256_loadu_pd(p + 4), a2 = _mm256_loadu_pd(p + 8);
    const __m256d b0 = _mm256_blend_pd(a0, a1, 0b0010);   // t0 y1 y0 t1
    const __m256d b1 = _mm256_blend_pd(a1, a2, 0b0010);   // x1 t3 t2 x2
    const __m256d b2 = _mm256_blend_pd(a2, a0, 0b0010);   // y2 x0 x3 y3
    const __m256d t = _mm256_permute4x64_pd(_mm256_blend_pd(b0, b1, 0b0110), _MM_SHUFFLE(1, 2, 3, 0));
    const __m256d x = _mm256_permute4x64_pd(_mm256_blend_pd(b1, b2, 0b0110), _MM_SHUFFLE(2, 3, 0, 1));
    const __m256d y = _mm256_permute4x64_pd(_mm256_blend_pd(b2, b0, 0b0110), _MM_SHUFFLE(3, 0, 1, 2));
    const __m128 a = _mm256_cvtpd_ps(_mm256_div_pd(_mm256_sub_pd(t, vt0), vdt));
    const __m128i xi = _mm256_cvttpd_epi32(_mm256_min_pd(_mm256_max_pd(x, m1), vW));
    const __m128i yi = _mm256_cvttpd_epi32(_mm256_min_pd(_mm256_max_pd(y, m1), vH));
    __m256d ok = _mm256_and_pd(_mm256_cmp_pd(x, z, _CMP_GE_OQ), _mm256_cmp_pd(x, vW, _CMP_LT_OQ));
    ok = _mm256_and_pd(ok, _mm256_and_pd(_mm256_cmp_pd(y, z, _CMP_GE_OQ), _mm256_cmp_pd(y, vH, _CMP_LT_OQ)));
    ok = _mm256_and_pd(ok, _mm256_cmp_pd(_mm256_cvtepi32_pd(xi), x, _CMP_EQ_OQ));
    ok = _mm256_and_pd(ok, _mm256_cmp_pd(_mm256_cvtepi32_pd(yi), y, _CMP_EQ_OQ));
    const __m128i okm = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(_mm256_castpd_si256(ok), even));
    const __m128i xy = _mm_or_si128(_mm_and_si128(okm, _mm_or_si128(xi, _mm_slli_epi32(yi, 16))),
                                    _mm_andnot_si128(okm, _mm_set1_epi32(-1)));
    const __m128i ab = _mm_castps_si128(a);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(out + 2 * i), _mm_unpacklo_epi32(ab, xy));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(out + 2 * i + 4), _mm_unpackhi_epi32(ab, xy));
  }
  pack_scalar(r + 3 * i, m - i, t0, dt, W, H, out + 2 * i);
}

__attribute__((target("avx512f,avx512vl,avx512dq"))) void pack_avx512(const double* r, int64_t m, double t0,
                                                                        double dt, int W, int H, uint32_t* out) {
  const __m512d vt0 = _mm512_set1_pd(t0), vdt = _mm512_set1_pd(dt), vW = _mm512_set1_pd(W), vH = _mm512_set1_pd(H);
  const __m512d z = _mm512_setzero_pd(), m1 = _mm512_set1_pd(-1.0);
  // 8 rows = 24 doubles in a0|a1|a2: component c of row k sits at 3k + c
  const __m512i t01 = _mm512_setr_epi64(0, 3, 6, 9, 12, 15, 0, 0), t2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 5, 10, 13);
  const __m512i x01 = _mm512_setr_epi64(1, 4, 7, 10, 13, 0, 0, 0), x2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 8, 11, 14);
  const __m512i y01 = _mm512_setr_epi64(2, 5, 8, 11, 14, 0, 0, 0), y2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 9, 12, 15);
  // Non-temporal stores (the records go to page-locked staging that only the
  // DMA engine reads): no read-for-ownership of the destination lines, 8 of
  // the ~56 host-DRAM bytes per event.  They need 32-byte alignment: the
  // first events up to that boundary take the scalar path.
  static const bool nt = [] {
    const char* e = std::getenv("VKM_PACK_NT");
    return !(e && e[0] == '0');
  }();
  int64_t i = 0;
  if (nt) {
    const int64_t head = std::min<int64_t>(m, int64_t((32 - (reinterpret_cast<uintptr_t>(out) & 31)) & 31) / 8);
    pack_scalar(r, head, t0, dt, W, H, out);
    i = head;
  }
  for (; i + 8 <= m; i += 8) {
    const double* p = r + 3 * i;
    const __m512d a0 = _mm512_loadu_pd(p), a1 = _mm512_loadu_pd(p + 8), a2 = _mm512_loadu_pd(p + 16);
    const __m512d t = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, t01, a1), t2, a2);
    const __m512d x = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, x01, a1), x2, a2);
    const __m512d y = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, y01, a1), y2, a2);
    const __m256 a = _mm512_cvtpd_ps(_mm512_div_pd(_mm512_sub_pd(t, vt0), vdt));
    const __m256i xi = _mm512_cvttpd_epi32(_mm512_min_pd(_mm512_max_pd(x, m1), vW));
    const __m256i yi = _mm512_cvttpd_epi32(_mm512_min_pd(_mm512_max_pd(y, m1), vH));
    const __mmask8 ok = _mm512_cmp_pd_mask(x, z, _CMP_GE_OQ) & _mm512_cmp_pd_mask(x, vW, _CMP_LT_OQ) &
                        _mm512_cmp_pd_mask(y, z, _CMP_GE_OQ) & _mm512_cmp_pd_mask(y, vH, _CMP_LT_OQ) &
                        _mm512_cmp_pd_mask(_mm512_cvtepi32_pd(xi), x, _CMP_EQ_OQ) &
                        _mm512_cmp_pd_mask(_mm512_cvtepi32_pd(yi), y, _CMP_EQ_OQ);
    const __m256i xy = _mm256_mask_blend_epi32(ok, _mm256_set1_epi32(-1), _mm256_or_si256(xi, _mm256_slli_epi32(yi, 16)));
    const __m256i ab = _mm256_castps_si256(a);
    const __m256i lo = _mm256_unpacklo_epi32(ab, xy), hi = _mm256_unpackhi_epi32(ab, xy);
    if (nt) {
      _mm256_stream_si256(reinterpret_cast<__m256i*>(out + 2 * i), _mm256_permute2x128_si256(lo, hi, 0x20));
      _mm256_stream_si256(reinterpret_cast<__m256i*>(out + 2 * i + 8), _mm256_permute2x128_si256(lo, hi, 0x31));
    } else {
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + 2 * i), _mm256_permute2x128_si256(lo, hi, 0x20));
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + 2 * i + 8), _mm256_permute2x128_si256(lo, hi, 0x31));
    }
  }
  if (nt) _mm_sfence();   // streamed records visible before the copy is issued
  pack_scalar(r + 3 * i, m - i, t0, dt, W, H, out + 2 * i);
}

}  // namespace

// f32 -> f64 widening of result rows into the caller's buffer, streamed
// (the destination is fresh memory the caller reads later: no
// read-for-ownership), scalar until dst is 64-byte aligned.
__attribute__((target("avx512f"))) static void widen_avx512(const float* src, double* dst, int64_t m) {
  int64_t i = 0;
  for (; i < m && (reinterpret_cast<uintptr_t>(dst + i) & 63); ++i) dst[i] = double(src[i]);
  for (; i + 8 <= m; i += 8) _mm512_stream_pd(dst + i, _mm512_cvtps_pd(_mm256_loadu_ps(src + i)));
  _mm_sfence();
  for (; i < m; ++i) dst[i] = double(src[i]);
}

void widen_f32(const float* src, double* dst, int64_t m) {
  static const bool avx512 = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f");
  }();
  if (avx512) {
    widen_avx512(src, dst, m);
    return;
  }
  for (int64_t i = 0; i < m; ++i) dst[i] = double(src[i]);
}

// Reads of write-combining staging (the DMA engine's destination; uncached for
// the CPU, so a D2H never waits on snoops of CPU-cached lines): MOVNTDQA
// streaming loads of 64-byte lines, scalar reads only up to src's alignment.
__attribute__((target("avx512f"))) static void widen_wc_avx512(const float* src, double* dst, int64_t m) {
  int64_t i = 0;
  for (; i < m && (reinterpret_cast<uintptr_t>(src + i) & 63); ++i) dst[i] = double(src[i]);
  const bool dal = (reinterpret_cast<uintptr_t>(dst + i) & 63) == 0;
  // eight lines in flight before the first conversion (WC reads are not
  // prefetched: each line is a memory round trip)
  for (; i + 128 <= m; i += 128) {
    __m512 v[8];
#pragma GCC unroll 8
    for (int k = 0; k < 8; ++k) v[k] = _mm512_castsi512_ps(_mm512_stream_load_si512(const_cast<float*>(src + i + 16 * k)));
#pragma GCC unroll 8
    for (int k = 0; k < 8; ++k) {
      const __m512d lo = _mm512_cvtps_pd(_mm512_castps512_ps256(v[k]));
      const __m512d hi = _mm512_cvtps_pd(_mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castps_pd(v[k]), 1)));
      if (dal) {
        _mm512_stream_pd(dst + i + 16 * k, lo);
        _mm512_stream_pd(dst + i + 16 * k + 8, hi);
      } else {
        _mm512_storeu_pd(dst + i + 16 * k, lo);
        _mm512_storeu_pd(dst + i + 16 * k + 8, hi);
      }
    }
  }
  for (; i + 16 <= m; i += 16) {
    const __m512 v = _mm512_castsi512_ps(_mm512_stream_load_si512(const_cast<float*>(src + i)));
    const __m512d lo = _mm512_cvtps_pd(_mm512_castps512_ps256(v));
    const __m512d hi = _mm512_cvtps_pd(_mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castps_pd(v), 1)));
    if (dal) {
      _mm512_stream_pd(dst + i, lo);
      _mm512_stream_pd(dst + i + 8, hi);
    } else {
      _mm512_storeu_pd(dst + i, lo);
      _mm512_storeu_pd(dst + i + 8, hi);
    }
  }
  _mm_sfence();
  for (; i < m; ++i) dst[i] = double(src[i]);
}

__attribute__((target("avx512f"))) static void copy_wc_avx512(const uint8_t* src, uint8_t* dst, size_t bytes) {
  size_t i = 0;
  for (; i < bytes && (reinterpret_cast<uintptr_t>(src + i) & 63); ++i) dst[i] = src[i];
  const bool dal = (reinterpret_cast<uintptr_t>(dst + i) & 63) == 0;
  for (; i + 512 <= bytes; i += 512) {   // eight lines in flight
    __m512i v[8];
#pragma GCC unroll 8
    for (int k = 0; k < 8; ++k) v[k] = _mm512_stream_load_si512(const_cast<uint8_t*>(src + i + 64 * k));
#pragma GCC unroll 8
    for (int k = 0; k < 8; ++k) {
      if (dal)
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 64 * k), v[k]);
      else
        _mm512_storeu_si512(dst + i + 64 * k, v[k]);
    }
  }
  if (dal) _mm_sfence();
  for (; i + 64 <= bytes; i += 64)
    _mm512_storeu_si512(dst + i, _mm512_stream_load_si512(const_cast<uint8_t*>(src + i)));
  for (; i < bytes; ++i) dst[i] = src[i];
}

static bool have_avx512f() {
  static const bool v = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f");
  }();
  return v;
}

void widen_f32_wc(const float* src, double* dst, int64_t m) {
  if (have_avx512f()) {
    widen_wc_avx512(src, dst, m);
    return;
  }
  for (int64_t i = 0; i < m; ++i) dst[i] = double(src[i]);
}

void copy_wc(const void* src, void* dst, size_t bytes) {
  if (have_avx512f()) {
    copy_wc_avx512(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), bytes);
    return;
  }
  std::memcpy(dst, src, bytes);
}

// out: 2 uint32 per event (the device's uint2 record)
void pack_events(const double* rows, int64_t m, double t0, double dt, int W, int H, uint32_t* out) {
  static const int isa = [] {
    __builtin_cpu_init();
    if (__builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512dq"))
      return 2;
    return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma") ? 1 : 0;
  }();
  if (isa == 2)
    pack_avx512(rows, m, t0, dt, W, H, out);
  else if (isa == 1)
    pack_avx2(rows, m, t0, dt, W, H, out);
  else
    pack_scalar(rows, m, t0, dt, W, H, out);
}

}  // namespace vkm_host

// ---------------------------------------------------------------------------
// One-pass host check of an (n, 3+) f64 [t, x, y] event array for the
// estimator's input contract (validation.py:10-37, 49-65 of the reference):
// the numpy version makes ~10 strided passes (44 ms per 1M events); this is
// one.  The flags are raised in the reference's order by the Python caller.
// ---------------------------------------------------------------------------
#include <emmintrin.h>

#include "../../include/veckm.h"

extern "C" {

}  // extern "C"

namespace {
// AVX-512 body for contiguous rows (ld == 3): 8 rows per step, the same
// predicates as the scalar loop; returns the first row not processed.
__attribute__((target("avx512f,avx512vl,avx512dq"))) int64_t check_avx512(const double* X, int64_t n, int W, int H,
                                                                           vkm_event_check& c, double& prev) {
  const __m512i t01 = _mm512_setr_epi64(0, 3, 6, 9, 12, 15, 0, 0), t2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 5, 10, 13);
  const __m512i x01 = _mm512_setr_epi64(1, 4, 7, 10, 13, 0, 0, 0), x2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 8, 11, 14);
  const __m512i y01 = _mm512_setr_epi64(2, 5, 8, 11, 14, 0, 0, 0), y2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 9, 12, 15);
  const __m512i rot = _mm512_setr_epi64(7, 0, 1, 2, 3, 4, 5, 6);
  const __m512d dmax = _mm512_set1_pd(1.7976931348623157e308), big = _mm512_set1_pd(4503599627370496.0);
  const __m512d z = _mm512_setzero_pd();
  const __m256i vW = _mm256_set1_epi32(W), vH = _mm256_set1_epi32(H), z32 = _mm256_setzero_si256();
  __mmask8 bad_fin = 0, bad_neg = 0, bad_int = 0, bad_ord = 0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const double* p = X + 3 * i;
    const __m512d a0 = _mm512_loadu_pd(p), a1 = _mm512_loadu_pd(p + 8), a2 = _mm512_loadu_pd(p + 16);
    const __m512d t = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, t01, a1), t2, a2);
    const __m512d x = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, x01, a1), x2, a2);
    const __m512d y = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, y01, a1), y2, a2);
    const __mmask8 fin = _mm512_cmp_pd_mask(_mm512_abs_pd(t), dmax, _CMP_LE_OQ) &
                         _mm512_cmp_pd_mask(_mm512_abs_pd(x), dmax, _CMP_LE_OQ) &
                         _mm512_cmp_pd_mask(_mm512_abs_pd(y), dmax, _CMP_LE_OQ);
    bad_fin |= __mmask8(~fin);
    bad_neg |= _mm512_cmp_pd_mask(t, z, _CMP_LT_OQ);
    const __mmask8 xint = _mm512_cmp_pd_mask(_mm512_abs_pd(x), big, _CMP_NLT_UQ) |
                          _mm512_cmp_pd_mask(_mm512_roundscale_pd(x, _MM_FROUND_TO_ZERO | _MM_FROUND_NO_EXC), x, _CMP_EQ_OQ);
    const __mmask8 yint = _mm512_cmp_pd_mask(_mm512_abs_pd(y), big, _CMP_NLT_UQ) |
                          _mm512_cmp_pd_mask(_mm512_roundscale_pd(y, _MM_FROUND_TO_ZERO | _MM_FROUND_NO_EXC), y, _CMP_EQ_OQ);
    bad_int |= __mmask8(fin & ~(xint & yint));
    // previous times: (prev, t0..t6)
    const __m512d tp = _mm512_mask_blend_pd(1, _mm512_permutexvar_pd(rot, t), _mm512_set1_pd(prev));
    bad_ord |= _mm512_cmp_pd_mask(t, tp, _CMP_LT_OQ);
    prev = p[21];
    if (c.first_outside < 0) {
      const __m256i xi = _mm512_cvttpd_epi32(x), yi = _mm512_cvttpd_epi32(y);   // INT_MIN when out of range
      const __mmask8 in = _mm256_cmpge_epi32_mask(xi, z32) & _mm256_cmplt_epi32_mask(xi, vW) &
                          _mm256_cmpge_epi32_mask(yi, z32) & _mm256_cmplt_epi32_mask(yi, vH);
      const __mmask8 out = __mmask8(fin & ~in);
      if (out) {
        const int k = __builtin_ctz(unsigned(out));
        alignas(32) int32_t xs[8], ys[8];
        _mm256_store_si256(reinterpret_cast<__m256i*>(xs), xi);
        _mm256_store_si256(reinterpret_cast<__m256i*>(ys), yi);
        c.first_outside = i + k;
        c.outside_x = xs[k];
        c.outside_y = ys[k];
      }
    }
  }
  c.nonfinite |= bad_fin != 0;
  c.negative_t |= bad_neg != 0;
  c.nonint |= bad_int != 0;
  if (bad_ord) c.sorted = 0;
  return i;
}

// check_avx512's predicates and pack_avx512's records in one pass (rows
// already in registers once): for contiguous rows, out 32-byte aligned.
// Returns the first row not processed; c.first_outside is relative to X.
__attribute__((target("avx512f,avx512vl,avx512dq"))) int64_t check_pack_avx512(const double* X, int64_t n, double t0,
                                                                                double dt, int W, int H, uint32_t* out,
                                                                                vkm_event_check& c, double& prev) {
  const __m512i t01 = _mm512_setr_epi64(0, 3, 6, 9, 12, 15, 0, 0), t2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 5, 10, 13);
  const __m512i x01 = _mm512_setr_epi64(1, 4, 7, 10, 13, 0, 0, 0), x2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 8, 11, 14);
  const __m512i y01 = _mm512_setr_epi64(2, 5, 8, 11, 14, 0, 0, 0), y2 = _mm512_setr_epi64(0, 1, 2, 3, 4, 9, 12, 15);
  const __m512i rot = _mm512_setr_epi64(7, 0, 1, 2, 3, 4, 5, 6);
  const __m512d dmax = _mm512_set1_pd(1.7976931348623157e308), big = _mm512_set1_pd(4503599627370496.0);
  const __m512d z = _mm512_setzero_pd(), vt0 = _mm512_set1_pd(t0), vdt = _mm512_set1_pd(dt);
  const __m256i vW = _mm256_set1_epi32(W), vH = _mm256_set1_epi32(H), z32 = _mm256_setzero_si256();
  __mmask8 bad_fin = 0, bad_neg = 0, bad_int = 0, bad_ord = 0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const double* p = X + 3 * i;
    const __m512d a0 = _mm512_loadu_pd(p), a1 = _mm512_loadu_pd(p + 8), a2 = _mm512_loadu_pd(p + 16);
    const __m512d t = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, t01, a1), t2, a2);
    const __m512d x = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, x01, a1), x2, a2);
    const __m512d y = _mm512_permutex2var_pd(_mm512_permutex2var_pd(a0, y01, a1), y2, a2);
    const __mmask8 fin = _mm512_cmp_pd_mask(_mm512_abs_pd(t), dmax, _CMP_LE_OQ) &
                         _mm512_cmp_pd_mask(_mm512_abs_pd(x), dmax, _CMP_LE_OQ) &
                         _mm512_cmp_pd_mask(_mm512_abs_pd(y), dmax, _CMP_LE_OQ);
    bad_fin |= __mmask8(~fin);
    bad_neg |= _mm512_cmp_pd_mask(t, z, _CMP_LT_OQ);
    const __mmask8 xint = _mm512_cmp_pd_mask(_mm512_abs_pd(x), big, _CMP_NLT_UQ) |
                          _mm512_cmp_pd_mask(_mm512_roundscale_pd(x, _MM_FROUND_TO_ZERO | _MM_FROUND_NO_EXC), x, _CMP_EQ_OQ);
    const __mmask8 yint = _mm512_cmp_pd_mask(_mm512_abs_pd(y), big, _CMP_NLT_UQ) |
                          _mm512_cmp_pd_mask(_mm512_roundscale_pd(y, _MM_FROUND_TO_ZERO | _MM_FROUND_NO_EXC), y, _CMP_EQ_OQ);
    bad_int |= __mmask8(fin & ~(xint & yint));
    const __m512d tp = _mm512_mask_blend_pd(1, _mm512_permutexvar_pd(rot, t), _mm512_set1_pd(prev));
    bad_ord |= _mm512_cmp_pd_mask(t, tp, _CMP_LT_OQ);
    prev = p[21];
    // truncation (INT_MIN for NaN / out of int32 range): the bounds check and
    // the record's pixel; the record is valid for in-image integral values
    const __m256i xi = _mm512_cvttpd_epi32(x), yi = _mm512_cvttpd_epi32(y);
    const __mmask8 in = _mm256_cmpge_epi32_mask(xi, z32) & _mm256_cmplt_epi32_mask(xi, vW) &
                        _mm256_cmpge_epi32_mask(yi, z32) & _mm256_cmplt_epi32_mask(yi, vH);
    if (c.first_outside < 0) {
      const __mmask8 outm = __mmask8(fin & ~in);
      if (outm) {
        const int k = __builtin_ctz(unsigned(outm));
        alignas(32) int32_t xs[8], ys[8];
        _mm256_store_si256(reinterpret_cast<__m256i*>(xs), xi);
        _mm256_store_si256(reinterpret_cast<__m256i*>(ys), yi);
        c.first_outside = i + k;
        c.outside_x = xs[k];
        c.outside_y = ys[k];
      }
    }
    const __mmask8 ok = in & _mm512_cmp_pd_mask(_mm512_cvtepi32_pd(xi), x, _CMP_EQ_OQ) &
                        _mm512_cmp_pd_mask(_mm512_cvtepi32_pd(yi), y, _CMP_EQ_OQ);
    const __m256 a = _mm512_cvtpd_ps(_mm512_div_pd(_mm512_sub_pd(t, vt0), vdt));
    const __m256i xy = _mm256_mask_blend_epi32(ok, _mm256_set1_epi32(-1), _mm256_or_si256(xi, _mm256_slli_epi32(yi, 16)));
    const __m256i ab = _mm256_castps_si256(a);
    const __m256i lo = _mm256_unpacklo_epi32(ab, xy), hi = _mm256_unpackhi_epi32(ab, xy);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + 2 * i), _mm256_permute2x128_si256(lo, hi, 0x20));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(out + 2 * i + 8), _mm256_permute2x128_si256(lo, hi, 0x31));
  }
  _mm_sfence();
  c.nonfinite |= bad_fin != 0;
  c.negative_t |= bad_neg != 0;
  c.nonint |= bad_int != 0;
  if (bad_ord) c.sorted = 0;
  return i;
}
}  // namespace

namespace vkm_host {
// One serial pass over rows [0, n) (X already offset): the flags, the
// first outside pixel (index relative to X), t of the first and last rows.
void check_range(const double* X, int64_t n, int64_t ld, int32_t W, int32_t H, vkm_event_check& out) {
  vkm_event_check c{0, 0, 0, 1, -1, 0, 0, 0.0, 0.0};
  double prev = n ? X[0] : 0.0;
  static const bool avx512 = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl") &&
           __builtin_cpu_supports("avx512dq");
  }();
  int64_t i0 = 0;
  if (avx512 && ld == 3) i0 = check_avx512(X, n, W, H, c, prev);
  for (int64_t i = i0; i < n; ++i) {
    const double* r = X + i * ld;
    const double t = r[0], x = r[1], y = r[2];
    // |v| <= DBL_MAX is false for NaN and +-inf
    const bool fin = std::fabs(t) <= 1.7976931348623157e308 && std::fabs(x) <= 1.7976931348623157e308 &&
                     std::fabs(y) <= 1.7976931348623157e308;
    c.nonfinite |= !fin;
    c.negative_t |= t < 0.0;
    // integer-valued: |v| >= 2^52 always is; below, compare with the int64
    // truncation (inline cvttsd2si, no libm call)
    const bool xint = !(std::fabs(x) < 4503599627370496.0) || double(int64_t(x)) == x;
    const bool yint = !(std::fabs(y) < 4503599627370496.0) || double(int64_t(y)) == y;
    c.nonint |= fin & !(xint & yint);
    c.sorted &= !(t < prev);
    prev = t;
    if (c.first_outside < 0 && fin) {
      // numpy's astype(int32) on x86: truncation, INT_MIN when out of range
      const int xi = _mm_cvttsd_si32(_mm_set_sd(x)), yi = _mm_cvttsd_si32(_mm_set_sd(y));
      if (!(xi >= 0 && xi < W && yi >= 0 && yi < H)) {
        c.first_outside = i;
        c.outside_x = xi;
        c.outside_y = yi;
      }
    }
  }
  if (n) {
    c.t_first = X[0];
    c.t_last = X[(n - 1) * ld];
  }
  out = c;
}

// check_range + pack_events over contiguous rows [0, n) in one pass: the
// AVX-512 body between a scalar head (to the records' 32-byte alignment) and
// a scalar tail, the three parts' checks merged in row order.
void check_pack(const double* X, int64_t n, double t0, double dt, int32_t W, int32_t H, uint32_t* out,
                vkm_event_check& res) {
  static const bool fused = [] {
    __builtin_cpu_init();
    const char* e = std::getenv("VKM_CHECK_PACK");
    return !(e && e[0] == '0') && __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl") &&
           __builtin_cpu_supports("avx512dq");
  }();
  if (!fused || n < 64) {
    check_range(X, n, 3, W, H, res);
    pack_events(X, n, t0, dt, W, H, out);
    return;
  }
  const int64_t head = std::min<int64_t>(n, int64_t((32 - (reinterpret_cast<uintptr_t>(out) & 31)) & 31) / 8);
  vkm_event_check c{0, 0, 0, 1, -1, 0, 0, 0.0, 0.0};
  bool have = false;
  auto add = [&](const vkm_event_check& q) {
    if (have) {
      merge_check(c, q);
    } else {
      c = q;
      have = true;
    }
  };
  if (head > 0) {
    vkm_event_check q;
    check_range(X, head, 3, W, H, q);
    pack_scalar(X, head, t0, dt, W, H, out);
    add(q);
  }
  vkm_event_check b{0, 0, 0, 1, -1, 0, 0, 0.0, 0.0};
  double prev = X[3 * head];
  const int64_t body = check_pack_avx512(X + 3 * head, n - head, t0, dt, W, H, out + 2 * head, b, prev);
  if (body > 0) {
    if (b.first_outside >= 0) b.first_outside += head;
    b.t_first = X[3 * head];
    b.t_last = X[3 * (head + body - 1)];
    add(b);
  }
  const int64_t e = head + body;
  if (e < n) {
    vkm_event_check q;
    check_range(X + 3 * e, n - e, 3, W, H, q);
    if (q.first_outside >= 0) q.first_outside += e;
    pack_scalar(X + 3 * e, n - e, t0, dt, W, H, out + 2 * e);
    add(q);
  }
  res = c;
}

void merge_check(vkm_event_check& c, const vkm_event_check& q) {
  c.nonfinite |= q.nonfinite;
  c.negative_t |= q.negative_t;
  c.nonint |= q.nonint;
  c.sorted &= q.sorted & !(q.t_first < c.t_last);
  if (c.first_outside < 0 && q.first_outside >= 0) {
    c.first_outside = q.first_outside;
    c.outside_x = q.outside_x;
    c.outside_y = q.outside_y;
  }
  c.t_last = q.t_last;
}
}  // namespace vkm_host
using vkm_host::check_range;

// The host pool of the handle-free host utilities (validation, widening):
// created on first use, never torn down; one user at a time (try_lock, else
// the caller works alone).
static vkm_host::HostPool* shared_pool() {
  static vkm_host::HostPool* pool = new vkm_host::HostPool(vkm_host::default_pool_threads());
  return pool;
}
static std::mutex& shared_pool_mutex() {
  static std::mutex m;
  return m;
}

extern "C" {

int vkm_check_events(const double* X, int64_t n, int64_t ld, int32_t W, int32_t H, vkm_event_check* out) {
  if (!out || n < 0 || (n > 0 && (!X || ld < 3))) return 1;
  // large inputs: contiguous parts on the shared host pool, merged in part
  // order (the first outside pixel is the first part's first; sortedness also
  // checks each part boundary with the same comparison)
  const int64_t kPart = int64_t(1) << 16;
  std::unique_lock<std::mutex> lock(shared_pool_mutex(), std::defer_lock);
  if (n >= 4 * kPart && lock.try_lock()) {   // busy (another thread using the pool): serial pass
    vkm_host::HostPool* pool = shared_pool();
    const int parts = int(std::min<int64_t>(4 * pool->size(), n / kPart));
    std::vector<vkm_event_check> pc(parts);
    pool->run(parts, [&](int p) {
      const int64_t lo = n * p / parts, hi = n * (p + 1) / parts;
      check_range(X + lo * ld, hi - lo, ld, W, H, pc[p]);
      if (pc[p].first_outside >= 0) pc[p].first_outside += lo;
    });
    vkm_event_check c = pc[0];
    for (int p = 1; p < parts; ++p) vkm_host::merge_check(c, pc[p]);
    *out = c;
    return 0;
  }
  check_range(X, n, ld, W, H, *out);
  return 0;
}

// Test hook (not part of the ABI header): vkm_host::check_pack on
// contiguous (n, 3) rows, records into out (2 uint32 per event).
int vkm_debug_check_pack(const double* X, int64_t n, double t0, double dt, int32_t W, int32_t H, uint32_t* out,
                         vkm_event_check* c) {
  if (!c || n < 0 || (n > 0 && (!X || !out))) return 1;
  vkm_host::check_pack(X, n, t0, dt, W, H, out, *c);
  return 0;
}

int vkm_concat_rows(const double* const* srcs, const int64_t* rows, int32_t n_arrays, int64_t ld, double* dst) {
  if (n_arrays < 0 || ld < 1 || (n_arrays > 0 && (!srcs || !rows || !dst))) return 1;
  std::vector<int64_t> off(static_cast<size_t>(n_arrays) + 1, 0);
  for (int32_t a = 0; a < n_arrays; ++a) {
    if (rows[a] < 0 || (rows[a] > 0 && !srcs[a])) return 1;
    off[size_t(a) + 1] = off[size_t(a)] + rows[a];
  }
  const int64_t total = off[size_t(n_arrays)] * ld;   // doubles
  auto copy = [&](int64_t lo, int64_t hi) {            // destination doubles [lo, hi)
    int32_t a = int32_t(std::upper_bound(off.begin(), off.end(), lo / ld) - off.begin()) - 1;
    while (lo < hi) {
      while (off[size_t(a) + 1] * ld <= lo) ++a;
      const int64_t end = std::min(hi, off[size_t(a) + 1] * ld);
      std::memcpy(dst + lo, srcs[a] + (lo - off[size_t(a)] * ld), sizeof(double) * size_t(end - lo));
      lo = end;
    }
  };
  const int64_t kPart = int64_t(1) << 18;
  std::unique_lock<std::mutex> lock(shared_pool_mutex(), std::defer_lock);
  if (total >= 2 * kPart && lock.try_lock()) {
    vkm_host::HostPool* pool = shared_pool();
    const int parts = int(std::min<int64_t>(pool->size(), total / kPart));
    pool->run(parts, [&](int p) { copy(total * p / parts, total * (p + 1) / parts); });
    return 0;
  }
  copy(0, total);
  return 0;
}

int vkm_widen_f32(const float* src, double* dst, int64_t n) {
  if (n < 0 || (n > 0 && (!src || !dst))) return 1;
  const int64_t kPart = int64_t(1) << 18;
  std::unique_lock<std::mutex> lock(shared_pool_mutex(), std::defer_lock);
  if (n >= 2 * kPart && lock.try_lock()) {
    vkm_host::HostPool* pool = shared_pool();
    const int parts = int(std::min<int64_t>(pool->size(), n / kPart));
    pool->run(parts, [&](int p) {
      const int64_t lo = n * p / parts, hi = n * (p + 1) / parts;
      vkm_host::widen_f32(src + lo, dst + lo, hi - lo);
    });
    return 0;
  }
  vkm_host::widen_f32(src, dst, n);
  return 0;
}

}  // extern "C"
