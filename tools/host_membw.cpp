// Host memory bandwidth of the GPU box (diagnostic for the e2e analysis):
// read-only, NT-write, and read+NT-write (the packer's pattern) with T threads.
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
__attribute__((target("avx512f"))) static double rd(const double* p, size_t n) {
  __m512d a = _mm512_setzero_pd(), b = a, c = a, d = a;
  for (size_t i = 0; i + 32 <= n; i += 32) {
    a = _mm512_add_pd(a, _mm512_load_pd(p + i));
    b = _mm512_add_pd(b, _mm512_load_pd(p + i + 8));
    c = _mm512_add_pd(c, _mm512_load_pd(p + i + 16));
    d = _mm512_add_pd(d, _mm512_load_pd(p + i + 24));
  }
  return _mm512_reduce_add_pd(_mm512_add_pd(_mm512_add_pd(a, b), _mm512_add_pd(c, d)));
}
__attribute__((target("avx512f"))) static void wr(double* p, size_t n) {
  const __m512d v = _mm512_set1_pd(1.0);
  for (size_t i = 0; i + 8 <= n; i += 8) _mm512_stream_pd(p + i, v);
  _mm_sfence();
}
__attribute__((target("avx512f"))) static void rw(const double* s, float* d, size_t n) {   // 24 B in, 8 B out (NT)
  for (size_t i = 0; i + 48 <= n; i += 48) {
    __m512d a0 = _mm512_load_pd(s + i), a1 = _mm512_load_pd(s + i + 8), a2 = _mm512_load_pd(s + i + 16);
    __m512d a3 = _mm512_load_pd(s + i + 24), a4 = _mm512_load_pd(s + i + 32), a5 = _mm512_load_pd(s + i + 40);
    __m512d x = _mm512_add_pd(_mm512_add_pd(a0, a1), _mm512_add_pd(a2, a3));
    x = _mm512_add_pd(x, _mm512_add_pd(a4, a5));
    _mm512_stream_pd(reinterpret_cast<double*>(d + i / 3), x);
    _mm512_stream_pd(reinterpret_cast<double*>(d + i / 3) + 8, x);
  }
  _mm_sfence();
}
int main(int argc, char** argv) {
  const size_t bytes = size_t(1) << 30, n = bytes / 8;
  double* a = static_cast<double*>(aligned_alloc(64, bytes));
  float* o = static_cast<float*>(aligned_alloc(64, bytes / 3 + 4096));
  std::memset(a, 1, bytes);
  std::memset(o, 1, bytes / 3);
  for (int T : {1, 4, 8, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      double best = 1e9;
      for (int r = 0; r < 3; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int k = 0; k < T; ++k)
          th.emplace_back([&, k] {
            size_t lo = n * k / T / 48 * 48, hi = n * (k + 1) / T / 48 * 48;
            if (mode == 0) { volatile double s = rd(a + lo, hi - lo); (void)s; }
            if (mode == 1) wr(a + lo, hi - lo);
            if (mode == 2) rw(a + lo, o + lo / 3, hi - lo);
          });
        for (auto& t : th) t.join();
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      }
      const double moved = mode == 2 ? bytes * (1.0 + 1.0 / 3.0) : bytes;
      std::printf("threads %2d %-10s %6.1f GB/s\n", T, mode == 0 ? "read" : mode == 1 ? "nt-write" : "read+ntw", moved / best / 1e9);
    }
  }
}
