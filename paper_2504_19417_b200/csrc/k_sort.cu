// K1 (sorted): per-pixel accumulation in the reference's own summation order.
//
//   k_prep     event -> pixel key, slot value (event index, f32 time argument
//              a = f32((t - t0)/δt)) and the per-pixel count histogram (the
//              reference's bincount, encoder.py:259)
//   k_scan     exclusive prefix sum of the counts -> pixel run starts
//              (single pass, decoupled look-back over 4096-count tiles)
//   k_scatter  counting scatter to start[pixel] + arrival rank, then
//   k_runsort  puts every run back into event (= time) order: the same
//              stable pixel-major order as np.argsort(flat, kind="stable")
//              (encoder.py:255-257), so each pixel's run is in time order
//   k_reduce_x (default, D = 64) sums e^{i a T} per pixel sequentially in f32 —
//              the order of the reference's np.add.reduceat (encoder.py:262-267)
//              — and feeds the x half of the pooling window directly, so the
//              raw grid never reaches HBM (see the kernel comment)
//   k_reduce   raw-grid variant: writes each pixel's 512-byte row of the
//              pre-modulated grid M = G·e^{i(xX/δx + yY/δy)} exactly once
//              (split pooling path for large δx, and the raw-grid parity hook)
//
// Compared with scattering fp32 atomics this writes every row once (no
// memset, no L2 read-modify-write of a grid larger than L2), is bit-
// deterministic, and reproduces the reference's per-pixel sums bit-for-bit
// wherever the f32 phases agree (98.9% of sin/cos values).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {

constexpr unsigned kFullMask = 0xffffffffu;

// Event-parallel kernels run one co-resident wave with a grid-stride loop:
// blocks then progress together through the time-ordered events, so k_prep's
// histogram atomics hand out arrival ranks in nearly time order.  (A grid of
// twice the resident blocks ran its second half after the first: every run
// became two interleaved sequences.  Warp tickets from a global counter kept
// the order tighter but serialised on the counter: cfg-2 k_prep 15 -> 29 us.)
template <class F>
__device__ __forceinline__ void event_walk(int64_t n, F&& f) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) f(e);
}

__global__ void __launch_bounds__(256) k_prep(const double* __restrict__ ev, const SliceTab st, double delta_t,
                                              int W, int H, int32_t* __restrict__ pix_out,
                                              uint64_t* __restrict__ val_out, int32_t* __restrict__ rank_out,
                                              int* __restrict__ cnt, float* __restrict__ flows_invalid,
                                              int32_t* __restrict__ counts_invalid) {
  const int P = W * H;
  const int64_t n = st.off[st.nb];
  event_walk(n, [&](int64_t e) {
    int b = 0;   // slice of event e (upper_bound over the offsets)
    for (int step = kMaxBatch / 2; step > 0; step >>= 1)
      if (b + step < st.nb && st.off[b + step] <= e) b += step;
    const double t0 = ld_t0(ev + 3 * st.off[b], st.t0[b]);
    const double t = __ldg(ev + 3 * e), x = __ldg(ev + 3 * e + 1), y = __ldg(ev + 3 * e + 2);
    const int xi = int(x), yi = int(y);
    int pix = st.nb * P;   // out-of-sensor events sort after every pixel run
    if (xi >= 0 && xi < W && yi >= 0 && yi < H && x == double(xi) && y == double(yi)) {
      pix = b * P + yi * W + xi;
      if (rank_out)
        rank_out[e] = atomicAdd(cnt + pix, 1);   // arrival rank: the counting scatter's offset
      else if (cnt)
        atomicAdd(cnt + pix, 1);                 // histogram only (row-bucket path)
    } else {
      if (flows_invalid)
        reinterpret_cast<float2*>(flows_invalid)[e] = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
      if (counts_invalid) counts_invalid[e] = 0;
    }
    pix_out[e] = pix;
    val_out[e] = slot_pack(int32_t(e), time_arg(t, t0, delta_t));
  });
}

// Host-packed events (vkm_predict_batch_host): the time argument arrives
// precomputed, pixels as 16-bit coordinates.
__global__ void __launch_bounds__(256) k_prep_packed(const uint2* __restrict__ evp, const SliceTab st, int W, int H,
                                                     int32_t* __restrict__ pix_out, uint64_t* __restrict__ val_out,
                                                     int32_t* __restrict__ rank_out, int* __restrict__ cnt,
                                                     float* __restrict__ flows_invalid,
                                                     int32_t* __restrict__ counts_invalid) {
  const int P = W * H;
  const int64_t n = st.off[st.nb];
  event_walk(n, [&](int64_t e) {
    int b = 0;
    for (int step = kMaxBatch / 2; step > 0; step >>= 1)
      if (b + step < st.nb && st.off[b + step] <= e) b += step;
    const uint2 v = __ldg(evp + e);
    const int xi = int(v.y & 0xFFFFu), yi = int(v.y >> 16);
    int pix = st.nb * P;
    if (xi < W && yi < H) {
      pix = b * P + yi * W + xi;
      if (rank_out)
        rank_out[e] = atomicAdd(cnt + pix, 1);   // arrival rank: the counting scatter's offset
      else if (cnt)
        atomicAdd(cnt + pix, 1);
    } else {
      if (flows_invalid)
        reinterpret_cast<float2*>(flows_invalid)[e] = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
      if (counts_invalid) counts_invalid[e] = 0;
    }
    pix_out[e] = pix;
    val_out[e] = slot_pack(int32_t(e), __uint_as_float(v.x));
  });
}

// Raw grid, D8 == 64: a warp owns 32 consecutive pixels and their slot range;
// slots are loaded 32 at a time (coalesced) and walked in order, lanes =
// channel pairs.  Writes M[pixel] = (Σ e^{i a T}) · e^{i(x X/δx + y Y/δy)}.
__global__ void __launch_bounds__(256) k_reduce(const int* __restrict__ start, const uint64_t* __restrict__ val_s,
                                                const int32_t* __restrict__ pix_s, const float* __restrict__ tf,
                                                const float2* __restrict__ mx, const float2* __restrict__ my, int W,
                                                int64_t P, float2* __restrict__ G) {
  const int lane = threadIdx.x & 31;
  const float4* mx4 = reinterpret_cast<const float4*>(mx) + lane;
  const float4* my4 = reinterpret_cast<const float4*>(my) + lane;
  float4* G4 = reinterpret_cast<float4*>(G) + ((int64_t(lane >> 2) * P) << 2) + (lane & 3);
  const uint64_t T01 = f2pack(__ldg(tf + 2 * lane), __ldg(tf + 2 * lane + 1));
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t pw = warp * 32; pw < P; pw += nwarps * 32) {
    const int p0 = int(pw), p1 = int(min(P, pw + 32));
    const int s0 = __ldg(start + p0), s1 = __ldg(start + p1);
    int cur = p0;                           // pixel being accumulated
    int cy = p0 / W, cx = p0 - cy * W;      // its coordinates (advanced incrementally)
    uint64_t re = 0, im = 0;                // packed (ch c0, ch c0+1) sums, f32 in slot order
    auto flush = [&]() {
      const float4 fx = __ldg(mx4 + int64_t(cx) * 32), fy = __ldg(my4 + int64_t(cy) * 32);
      const float2 m0 = cmul(make_float2(fx.x, fx.y), make_float2(fy.x, fy.y));
      const float2 m1 = cmul(make_float2(fx.z, fx.w), make_float2(fy.z, fy.w));
      float r0, r1, i0, i1;
      f2unpack(re, r0, r1);
      f2unpack(im, i0, i1);
      const float2 g0 = cmul(make_float2(r0, i0), m0), g1 = cmul(make_float2(r1, i1), m1);
      G4[int64_t(cur) << 2] = make_float4(g0.x, g0.y, g1.x, g1.y);
      re = 0;
      im = 0;
      ++cur;
      if (++cx == W) {
        cx = 0;
        ++cy;
      }
    };
    for (int jb = s0; jb < s1; jb += 32) {
      const int j = jb + lane;
      float av = 0.f;
      int pv = int(P);
      if (j < s1) {
        pv = __ldg(pix_s + j);
        av = slot_arg(__ldg(val_s + j));
      }
      const int nj = min(32, s1 - jb);
#pragma unroll 2
      for (int k = 0; k < nj; ++k) {
        const int pk = __shfl_sync(kFullMask, pv, k);
        const float ak = __shfl_sync(kFullMask, av, k);
        uint64_t sn, cs;
        sincos2p_f32(fmul2(f2pack(ak, ak), T01), sn, cs);
        while (cur < pk) flush();           // finished pixels (and empty ones in between)
        re = fadd2(re, cs);
        im = fadd2(im, sn);
      }
    }
    while (cur < p1) flush();
  }
}

// D8 < 64: one warp per pixel group with lanes = (pixel sub-index, channel pair).
__global__ void __launch_bounds__(256) k_reduce_small(const int* __restrict__ start, const int* __restrict__ cnt,
                                                      const uint64_t* __restrict__ val_s,
                                                      const float* __restrict__ tf, const float2* __restrict__ mx,
                                                      const float2* __restrict__ my, int W, int64_t P, int D8,
                                                      float2* __restrict__ G) {
  const int lane = threadIdx.x & 31;
  const int cp = D8 >> 1;
  const int pair = lane % cp, sub = lane / cp, pps = 32 / cp;
  const uint64_t T01 = f2pack(__ldg(tf + 2 * pair), __ldg(tf + 2 * pair + 1));
  const int plane = pair >> 2, q4 = pair & 3;
  float4* G4 = reinterpret_cast<float4*>(G);
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t pb = warp * pps; pb < P; pb += nwarps * pps) {
    const int64_t p = pb + sub;
    if (p >= P) continue;
    const int s = __ldg(start + p), c = __ldg(cnt + p);
    uint64_t re = 0, im = 0;
    for (int j = s; j < s + c; ++j) {
      const float av = slot_arg(__ldg(val_s + j));
      uint64_t sn, cs;
      sincos2p_f32(fmul2(f2pack(av, av), T01), sn, cs);
      re = fadd2(re, cs);
      im = fadd2(im, sn);
    }
    float r0, r1, i0, i1;
    f2unpack(re, r0, r1);
    f2unpack(im, i0, i1);
    const int y = int(p / W), x = int(p - int64_t(y) * W);
    const float2* fx = mx + int64_t(x) * D8 + 2 * pair;
    const float2* fy = my + int64_t(y) * D8 + 2 * pair;
    const float2 g0 = cmul(make_float2(r0, i0), cmul(__ldg(fx), __ldg(fy)));
    const float2 g1 = cmul(make_float2(r1, i1), cmul(__ldg(fx + 1), __ldg(fy + 1)));
    G4[((int64_t(plane) * P + p) << 2) + q4] = make_float4(g0.x, g0.y, g1.x, g1.y);
  }
}

// ---------------------------------------------------------------------------
// K1 reduce fused with the x window (D8 == 64).
//
// One warp per (row y, segment of S output columns [x0, x1)); lanes = channel
// pairs.  The warp sweeps input pixels x in [x0-δx, x1+δx): for each it sums
// e^{i a T} over the pixel's time-ordered slot run in f32 (the reference's
// reduceat order, encoder.py:262-267), modulates by e^{i x X/δx}, and keeps a
// sliding window sum over the last 2δx+1 pixels (a per-lane ring in shared
// memory).  The window centred on x-δx is complete after pixel x, so it is
// multiplied by e^{i y Y/δy} and written (packed-pair layout, see k_pool.cu):
//   R[y][x] = e^{i y Y/δy} · Σ_{|i|<=δx} G[y][x+i] e^{i (x+i) X/δx}
// The raw grid never reaches HBM; the y pass (k_box_y<true>) finishes the
// window and demodulates.  Halo pixels (δx each side) are recomputed by the
// two neighbouring segments.  Events are processed in groups for ILP; pixel
// boundaries are tracked from start[] (32 run ends per coalesced load).
// ---------------------------------------------------------------------------
constexpr int kMaxFusedDx = 24;
#ifndef VKM_RX_WARPS
#define VKM_RX_WARPS 1   // one-warp CTAs spread the items over the SMs most evenly (cfg2 K1 -4.6 % vs 2)
#endif
constexpr int kRxWarps = VKM_RX_WARPS;   // warps (items) per CTA
constexpr int kRxMaxSeg = 128;
constexpr int kRxEnds = kRxMaxSeg + 2 * kMaxFusedDx + 4 + 64;   // run ends of one sweep (+ sentinel) + time-argument stage
#ifndef VKM_RX_GROUP
#define VKM_RX_GROUP 8   // events per sin/cos group of k_reduce_x (cfg2 K1: 4 +1.5 %, 16 +12 % at 148 registers)
#endif
constexpr int kRxGroup = VKM_RX_GROUP;   // events per sin/cos group (divides 32)
static_assert(kRxGroup % 4 == 0 && 32 % kRxGroup == 0, "groups read their time arguments as float4");

size_t reduce_x_smem(int dx) { return size_t(kRxWarps) * ((2 * dx + 1) * 512 + kRxEnds * 4); }

template <bool kMufu>
__global__ void __launch_bounds__(kRxWarps * 32) k_reduce_x(const int* __restrict__ start,
                                                            const uint64_t* __restrict__ val_s,
                                                            const float* __restrict__ tf,
                                                            const float4* __restrict__ mxp,
                                                            const float4* __restrict__ myp, int W, int H, int nb,
                                                            int dx, int S, int nseg, int64_t P,
                                                            float2* __restrict__ R) {
  extern __shared__ __align__(16) uint8_t rx_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int RL = 2 * dx + 1;
  ulonglong2* const ring0 = reinterpret_cast<ulonglong2*>(rx_smem) + wib * RL * 32 + lane;
  ulonglong2* const ring_end = ring0 + RL * 32;
  int* const ends = reinterpret_cast<int*>(rx_smem + size_t(kRxWarps) * RL * 512) + wib * kRxEnds;
  const uint64_t T01 = f2pack(__ldg(tf + 2 * lane), __ldg(tf + 2 * lane + 1));
  const float4* mxl = mxp + lane;                   // mxl[x * 32]: (cos c0, cos c1, sin c0, sin c1) of x X/δx
  const float4* myl = myp + lane;                   // (cos c0, cos c1, sin c0, sin c1) of y Y/δy
  float4* const R4 = reinterpret_cast<float4*>(R) + ((int64_t(lane >> 2) * P) << 2) + (lane & 3);
  const int64_t items = int64_t(nb) * H * nseg;   // (virtual row, segment); P = nb·W·H
  const int64_t nwarps = int64_t(gridDim.x) * kRxWarps;
  auto mx_at = [&](int x) { return __ldg(mxl + int64_t(min(max(x, 0), W - 1)) * 32); };
  // Item setup reads only start[] (k_scan's output, complete before the
  // predecessor chain that ends in this launch even began) and constant
  // tables, so the first item's setup runs before pdl_wait(), overlapping
  // the run sort's tail; only the slot values wait.
#ifndef VKM_RX_PF
#define VKM_RX_PF 1   // prefetch depth of the modulation factors and time arguments: 1 or 2
#endif
  int y = 0, x0 = 0, x1 = 0, xs = 0, nx = 0, jfirst = 0, jend = 0;
  float4 fy4 = make_float4(0.f, 0.f, 0.f, 0.f), mc = fy4, mcn = fy4;
  auto setup = [&](int64_t it) {
    y = int(it / nseg);                          // virtual row: slice y / H, sensor row y % H
    x0 = int(it - int64_t(y) * nseg) * S;
    x1 = min(W, x0 + S);
    xs = x0 - dx;
    nx = x1 + dx - xs;                           // sweep x = xs + k, k in [0, nx)
    const int* st = start + int64_t(y) * W;      // st[x]: first slot of pixel (x, y)
    jfirst = __ldg(st + max(0, xs));
    jend = __ldg(st + min(W, x1 + dx));
    __syncwarp();
    for (int k = lane; k <= nx; k += 32) {       // ends[k]: end slot of pixel xs + k's run
      const int x = xs + k;
      ends[k] = k == nx ? jend : (x < 0 ? jfirst : (x < W ? __ldg(st + x + 1) : jend));
    }
    for (int k = 0; k < RL; ++k) ring0[k * 32] = make_ulonglong2(0ull, 0ull);
    fy4 = __ldg(myl + int64_t(y % H) * 32);
    mc = mx_at(xs);
    if (VKM_RX_PF > 1) mcn = mx_at(xs + 1);
    __syncwarp();
  };
  int64_t it = int64_t(blockIdx.x) * kRxWarps + wib;
  if (it < items) setup(it);
  pdl_wait();
  for (; it < items; it += nwarps) {
    const uint64_t fyr = f2pack(fy4.x, fy4.y), fyi = f2pack(fy4.z, fy4.w);
    float4* out = R4 + ((int64_t(y) * W + x0) << 2);
    auto ld_a = [&](int jj) { return jj < jend ? slot_arg(__ldg(val_s + jj)) : 0.f; };
    int jb = jfirst;
    float av0 = ld_a(jb + lane), av1 = ld_a(jb + 32 + lane), av2 = VKM_RX_PF > 1 ? ld_a(jb + 64 + lane) : 0.f;
    // the current 32-slot batch's time arguments in shared memory: a group
    // reads its 8 with 2 broadcast LDS.128 instead of 8 shuffles (fewer MIO
    // operations; accumulate -1.5 % at configs 2 and 3, -2 % at config 5)
    float* const astage = reinterpret_cast<float*>(ends + kRxEnds - 64);
    __syncwarp();
    astage[lane] = av0;
    __syncwarp();

    int k = 0;                                      // sweep index of the pixel being summed
    int je = ends[0], je_n = ends[1];               // run end of pixel k, and of k+1 (loaded a pixel early)
    uint64_t gr = 0, gi = 0, ar = 0, ai = 0;
    ulonglong2* pn = ring0;                          // ring slot of pixel k
    ulonglong2* po = ring0 + 32;                     // ring slot of pixel k - 2δx
    ulonglong2 old = *po;                            // its value, read a pixel early (0 here)
    auto finish = [&]() {
      const uint64_t mre = f2pack(mc.x, mc.y), mim = f2pack(mc.z, mc.w);
      const uint64_t mr = fsub2(fmul2(gr, mre), fmul2(gi, mim));
      const uint64_t mi = ffma2(gr, mim, fmul2(gi, mre));
      *pn = make_ulonglong2(mr, mi);
      ar = fadd2(ar, mr);
      ai = fadd2(ai, mi);
      if (k >= 2 * dx) {
        const uint64_t orr = fsub2(fmul2(ar, fyr), fmul2(ai, fyi));
        const uint64_t oi = ffma2(ar, fyi, fmul2(ai, fyr));
        *reinterpret_cast<ulonglong2*>(out) = make_ulonglong2(orr, oi);   // packed-pair layout
        out += 4;
      }
      ar = fsub2(ar, old.x);
      ai = fsub2(ai, old.y);
      gr = 0;
      gi = 0;
      pn = po;
      po = (po + 32 == ring_end) ? ring0 : po + 32;
      old = *po;                                     // next trailing value: its slot is not written again before use
      ++k;
      je = je_n;
      je_n = ends[min(k + 1, nx)];                   // shared-memory latency off the per-pixel chain
      if (VKM_RX_PF > 1) {
        mc = mcn;                                    // modulation factors two pixels ahead
        mcn = mx_at(xs + k + 1);
      } else {
        mc = mx_at(xs + k);                          // next pixel's factor, in flight early
      }
    };

    // Events in groups of kRxGroup: the sin/cos of a whole group are computed
    // back to back (independent chains), then added in slot order with the
    // pixel boundaries resolved between them.  Groups never straddle a 32-slot
    // batch (both advance from jfirst).  Time arguments arrive two batches
    // (64 slots) ahead.
    for (int j = jfirst; j < jend; j += kRxGroup) {
      if (j - jb >= 32) {
        jb += 32;
        av0 = av1;
        if (VKM_RX_PF > 1) {
          av1 = av2;
          av2 = ld_a(jb + 64 + lane);
        } else {
          av1 = ld_a(jb + 32 + lane);
        }
        __syncwarp();
        astage[lane] = av0;
        __syncwarp();
      }
      const int i0 = j - jb;
      uint64_t cs[kRxGroup], sn[kRxGroup];
      float ag[kRxGroup];
#pragma unroll
      for (int u4 = 0; u4 < kRxGroup; u4 += 4) {
        const float4 q = *reinterpret_cast<const float4*>(astage + i0 + u4);
        ag[u4] = q.x, ag[u4 + 1] = q.y, ag[u4 + 2] = q.z, ag[u4 + 3] = q.w;
      }
#pragma unroll
      for (int u = 0; u < kRxGroup; ++u) {
        const float au = ag[u];
        sincos2_hot<kMufu>(fmul2(f2pack(au, au), T01), sn[u], cs[u]);
      }
#pragma unroll
      for (int u = 0; u < kRxGroup; ++u) {
        if (j + u >= je) {                           // pixel boundary (je <= jend)
          if (j + u >= jend) break;
          do finish(); while (j + u >= je);
        }
        gr = fadd2(gr, cs[u]);
        gi = fadd2(gi, sn[u]);
      }
    }
    while (k < nx) finish();
    if (it + nwarps < items) setup(it + nwarps);
  }
  pdl_trigger();   // dependents may launch as this grid drains
}

// ---------------------------------------------------------------------------
// Counting sort (default): the histogram and run starts exist already
// (k_prep + scan), so each event's slot is start[pixel] + its arrival rank
// (the value k_prep's histogram atomic returned).  That scatter is stable only
// up to the order of the atomics; the
// runs are then put back into event (= time) order, which is exactly the
// stable pixel-major order of np.argsort(kind="stable") (encoder.py:255-257):
//   k_runsort   one thread per pixel, insertion sort of runs <= 256 events;
//               the block then sorts each of its longer runs with a bitonic
//               network (ascending-only, so the virtual +inf padding never
//               moves) in the staged slots, or in global memory when the
//               block's range is not staged (pathological hot pixels).
//               VKM_RUNSORT_LONG_INBLOCK=0 lists them for k_longsort instead
//               (one CTA per run, a separate launch).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_scatter(const int32_t* __restrict__ pix, const uint64_t* __restrict__ val,
                                                 const int32_t* __restrict__ rank, int64_t n, int64_t P,
                                                 const int* __restrict__ start, uint64_t* __restrict__ val_s) {
  pdl_wait();
  event_walk(n, [&](int64_t e) {
    const int p = __ldcs(pix + e);
    if (p < P)   // outside the sensor: no slot (slots [start[P], n) are never read)
      val_s[__ldg(start + p) + __ldcs(rank + e)] = __ldcs(val + e);
  });
  pdl_trigger();   // dependents may launch as this grid drains
}

// Run ordering.  The arrival ranks follow the grid-stride order of k_prep, so
// a run is nearly time-ordered already (only events processed in the same
// wave can be swapped): insertion sort is close to linear.  A block owns ppb
// consecutive pixels per step, i.e. one contiguous slot range, staged through
// shared memory (coalesced in and out) when it fits; one thread per pixel
// insertion-sorts its run there by event index.  Runs too long for the stage
// go to a list sorted by k_longsort.  ppb is chosen on the host from the mean
// run length so the range usually fits (dense slices: 35 events per pixel).
__device__ __forceinline__ void cas_slot(uint64_t& a, uint64_t& b) {
  if (uint32_t(a) > uint32_t(b)) {
    const uint64_t t = a;
    a = b;
    b = t;
  }
}

// Ascending-only bitonic network over a[0, L) by the calling block (the
// virtual padding to N = 2^k behaves as +inf and never moves): merge stage k
// first compares i with its mirror in the 2k block, then half-cleaners.
__device__ void block_bitonic(uint64_t* a, int L) {
  int N = 1;
  while (N < L) N <<= 1;
  for (int k = 2; k <= N; k <<= 1) {
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
      const int lo = (i / (k / 2)) * k + (i % (k / 2));
      const int hi = (i / (k / 2)) * k + k - 1 - (i % (k / 2));
      if (hi < L) cas_slot(a[lo], a[hi]);
    }
    __syncthreads();
    for (int j = k / 4; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const int lo = (i / j) * 2 * j + (i % j), hi = lo + j;
        if (hi < L) cas_slot(a[lo], a[hi]);
      }
      __syncthreads();
    }
  }
}

#ifndef VKM_RUNSORT_LONG_INBLOCK   // 1: k_runsort sorts its long runs itself (no k_longsort launch)
#define VKM_RUNSORT_LONG_INBLOCK 1
#endif
#ifndef VKM_RUNSORT_THREADS
#define VKM_RUNSORT_THREADS 128
#endif
constexpr int kRunsortThreads = VKM_RUNSORT_THREADS;
constexpr int kLongCap = 32;           // long runs a block step sorts cooperatively (more: per thread)
constexpr int kRunsortStage = 6144;    // most slots staged per block (48 KB)
constexpr int kInsertRun = 256;        // longer runs: k_longsort (bitonic)
constexpr int kSmemRun = 4096;         // k_longsort sorts runs up to this in shared memory

__global__ void __launch_bounds__(kRunsortThreads) k_runsort(const int* __restrict__ start, int64_t P, int ppb,
                                                             int stage_cap, uint64_t* __restrict__ val_s,
                                                             int32_t* __restrict__ pix_s, int* __restrict__ longlist,
                                                             int* __restrict__ longcount) {
  pdl_wait();
  extern __shared__ uint64_t stage[];   // stage_cap slots
  __shared__ int nlong, longp[kLongCap];
  for (int64_t p0 = int64_t(blockIdx.x) * ppb; p0 < P; p0 += int64_t(gridDim.x) * ppb) {
    const int64_t pe = min(P, p0 + int64_t(ppb));
    const int b0 = __ldg(start + p0), b1 = __ldg(start + pe);
    const bool staged = b1 - b0 <= stage_cap;
    if (threadIdx.x == 0) nlong = 0;
    if (staged)
      for (int i = threadIdx.x; i < b1 - b0; i += blockDim.x) stage[i] = val_s[b0 + i];
    __syncthreads();
    for (int64_t p = p0 + threadIdx.x; p < pe; p += blockDim.x) {
      const int s = __ldg(start + p), L = __ldg(start + p + 1) - s;
      for (int j = 0; j < L; ++j) pix_s[s + j] = int32_t(p);   // slot -> pixel (K3's gather key)
      int li = -1;
#if VKM_RUNSORT_LONG_INBLOCK
      if (L > kInsertRun) li = atomicAdd(&nlong, 1);
      if (li >= 0 && li < kLongCap) {
        longp[li] = int(p);   // sorted below by the whole block
      } else if (L > 1) {     // (beyond kLongCap long runs per step: insertion sort, nearly sorted runs)
#else
      if (L > kInsertRun) {
        longlist[atomicAdd(longcount, 1)] = int(p);
      } else if (L > 1) {
#endif
        uint64_t* r = staged ? stage + (s - b0) : val_s + s;
        for (int i = 1; i < L; ++i) {   // by event index (low 32 bits), unique within a run
          const uint64_t v = r[i];
          const uint32_t k = uint32_t(v);
          int j = i - 1;
          while (j >= 0 && uint32_t(r[j]) > k) {
            r[j + 1] = r[j];
            --j;
          }
          r[j + 1] = v;
        }
      }
    }
    __syncthreads();
#if VKM_RUNSORT_LONG_INBLOCK
    const int nl = min(nlong, kLongCap);
    for (int li = 0; li < nl; ++li) {
      const int p = longp[li];
      const int s = __ldg(start + p), L = __ldg(start + p + 1) - s;
      block_bitonic(staged ? stage + (s - b0) : val_s + s, L);
    }
#endif
    if (staged)
      for (int i = threadIdx.x; i < b1 - b0; i += blockDim.x) val_s[b0 + i] = stage[i];
    __syncthreads();
  }
  pdl_trigger();   // dependents may launch as this grid drains
}


// ---------------------------------------------------------------------------
// Dense slices (mean run > 8 events, e.g. config 5 at 35 events per pixel):
// the counting scatter's 8-byte writes land on sectors all over a val_s far
// larger than L2, and its runs need sorting.  Instead a stable two-level
// counting sort (MSD: row, then column), both levels stable by construction,
// so the runs come out in time order with no run sort:
//   k_rowhist    per 8192-event tile: events per virtual row -> table[row][tile]
//   k_scan       over the table (row-major): each (row, tile)'s first bucket slot
//   k_rowscatter tile re-read; warps own consecutive 1024-event chunks, per-warp
//                row bases from per-warp counts, in-warp order by __match_any;
//                writes (event, a) and x into row buckets (whole-sector runs)
//   k_xsort      one CTA per row: the same stable counting step by column,
//                from the row bucket into val_s (pixel runs from start[]), pix_s
// ---------------------------------------------------------------------------
constexpr int kMsdTile = 8192, kMsdThreads = 256, kMsdWarps = kMsdThreads / 32;
constexpr int kMsdMaxRows = 4096;                  // per-warp row bases in shared memory
constexpr int kXsortThreads = 1024, kXsortWarps = kXsortThreads / 32, kXsortMaxW = 1536;

size_t msd_tab_words(int64_t n) { return size_t(kMsdMaxRows) * size_t((n + kMsdTile - 1) / kMsdTile + 1); }

__global__ void __launch_bounds__(kMsdThreads) k_rowhist(const int32_t* __restrict__ pix, int64_t n, int W, int R,
                                                         int ntiles, int* __restrict__ tab) {
  pdl_wait();
  extern __shared__ int rh[];   // [R]
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int r = threadIdx.x; r < R; r += blockDim.x) rh[r] = 0;
    __syncthreads();
    const int64_t e0 = int64_t(t) * kMsdTile, e1 = min(n, e0 + kMsdTile);
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int p = __ldg(pix + e);
      const int r = p / W;
      if (r < R) atomicAdd(rh + r, 1);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < R; r += blockDim.x) tab[int64_t(r) * ntiles + t] = rh[r];
    __syncthreads();
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(kMsdThreads) k_rowscatter(const int32_t* __restrict__ pix,
                                                            const uint64_t* __restrict__ val, int64_t n, int W, int R,
                                                            int ntiles, const int* __restrict__ off,
                                                            uint64_t* __restrict__ bkt, int32_t* __restrict__ bx) {
  pdl_wait();
  extern __shared__ int wb[];   // [kMsdWarps][R]: per-warp counts, then per-warp bases
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  constexpr int kChunk = kMsdTile / kMsdWarps;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < kMsdWarps * R; i += blockDim.x) wb[i] = 0;
    __syncthreads();
    const int64_t c0 = int64_t(t) * kMsdTile + int64_t(w) * kChunk, c1 = min(n, c0 + kChunk);
    for (int64_t e = c0 + lane; e < c1; e += 32) {
      const int r = __ldg(pix + e) / W;
      if (r < R) atomicAdd(wb + w * R + r, 1);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < R; r += blockDim.x) {   // bases: tile offset + earlier warps' counts
      int run = __ldg(off + int64_t(r) * ntiles + t);
      for (int v = 0; v < kMsdWarps; ++v) {
        const int c = wb[v * R + r];
        wb[v * R + r] = run;
        run += c;
      }
    }
    __syncthreads();
    int* base = wb + w * R;
    for (int64_t eb = c0; eb < c1; eb += 32) {            // in event order, 32 at a time
      const int64_t e = eb + lane;
      const bool ok = e < c1;
      const int p = ok ? __ldg(pix + e) : R * W;
      const int r = p / W;
      const bool in = ok && r < R;
      const unsigned peers = __match_any_sync(kFullMask, in ? r : -1);
      if (in) {
        const int pos = base[r] + __popc(peers & lt);
        bkt[pos] = __ldcs(val + e);
        bx[pos] = p - r * W;
      }
      __syncwarp();
      if (in && (peers & lt) == 0) base[r] += __popc(peers);   // the group's lowest lane advances the base
      __syncwarp();
    }
    __syncthreads();
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(kXsortThreads) k_xsort(const uint64_t* __restrict__ bkt,
                                                         const int32_t* __restrict__ bx, const int* __restrict__ start,
                                                         int W, int R, uint64_t* __restrict__ val_s,
                                                         int32_t* __restrict__ pix_s) {
  pdl_wait();
  extern __shared__ int xb[];   // [kXsortWarps][W]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    const int* st = start + int64_t(r) * W;
    const int rs = __ldg(st), re = __ldg(st + W);
    const int chunk = (re - rs + kXsortWarps - 1) / kXsortWarps;
    const int c0 = rs + w * chunk, c1 = min(re, c0 + chunk);
    for (int i = threadIdx.x; i < kXsortWarps * W; i += blockDim.x) xb[i] = 0;
    __syncthreads();
    for (int j = c0 + lane; j < c1; j += 32) atomicAdd(xb + w * W + __ldg(bx + j), 1);
    __syncthreads();
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
      int run = __ldg(st + x);
      for (int v = 0; v < kXsortWarps; ++v) {
        const int c = xb[v * W + x];
        xb[v * W + x] = run;
        run += c;
      }
    }
    __syncthreads();
    int* base = xb + w * W;
    for (int jb = c0; jb < c1; jb += 32) {
      const int j = jb + lane;
      const bool in = j < c1;
      const int x = in ? __ldg(bx + j) : -1;
      const unsigned peers = __match_any_sync(kFullMask, x);
      if (in) {
        const int pos = base[x] + __popc(peers & lt);
        val_s[pos] = __ldcs(bkt + j);
        pix_s[pos] = r * W + x;
      }
      __syncwarp();
      if (in && (peers & lt) == 0) base[x] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
  }
  pdl_trigger();
}


// ---------------------------------------------------------------------------
// Run starts of the radix-sorted keys (pixel ids, P for out-of-sensor events):
// start[p] = first slot whose key >= p, for p in [0, P] - the exclusive scan
// of the per-pixel counts, read off the sorted order, so the dense path's
// k_prep needs no histogram atomics (32M atomics: 90 of k_prep's 295 us at
// config 5).  The thread at slot i (a key boundary a < b, with a = -1 before
// the first slot and b = P + 1 after the last) writes start[p] = i for
// p in (a, min(b, P)]; every p is written exactly once.
// ---------------------------------------------------------------------------
// One thread per 4 slots (one 16-byte load; a grid over all slots, not a
// resident wave with a loop: the loop's dependent loads were latency-bound,
// 110 us at config 5).
__global__ void __launch_bounds__(256) k_run_starts(const int32_t* __restrict__ pix_s, int64_t n, int64_t P,
                                                    int* __restrict__ start) {
  pdl_wait();
  const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i0 <= n) {
    int32_t k[5];   // keys of slots i0 - 1 .. i0 + 3 (-1 before the first, P + 1 from slot n on)
    k[0] = i0 == 0 ? -1 : __ldg(pix_s + i0 - 1);
    if (i0 + 4 <= n && (reinterpret_cast<uintptr_t>(pix_s) & 15) == 0) {
      const int4 v = __ldg(reinterpret_cast<const int4*>(pix_s + i0));
      k[1] = v.x, k[2] = v.y, k[3] = v.z, k[4] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) k[j + 1] = i0 + j < n ? __ldg(pix_s + i0 + j) : int32_t(P + 1);
    }
    if (k[0] != k[4]) {   // a run boundary among these slots (1 in 35 at config 5)
      const int Pi = int(P), i0i = int(i0), ni = int(n);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (i0i + j > ni) break;
        const int hi = min(k[j + 1], Pi);
        for (int p = k[j] + 1; p <= hi; ++p) start[p] = i0i + j;
      }
    }
  }
  pdl_trigger();
}

// per-pixel counts from the run starts (the count pooling's input)
__global__ void __launch_bounds__(256) k_counts_from_starts(const int* __restrict__ start, int64_t P,
                                                            int* __restrict__ cnt) {
  pdl_wait();
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p <= P; p += int64_t(gridDim.x) * blockDim.x)
    cnt[p] = p < P ? __ldg(start + p + 1) - __ldg(start + p) : 0;
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// Dense slices: stable LSD radix sort of (pixel key, slot value), 8-bit
// digits.  Per digit pass: k_rs_tilehist counts each 3072-item tile's digits
// into a digit-major table, k_scan turns it into every (digit, tile)'s global
// first slot, and k_rs_scatter ranks the tile's items by digit in shared
// memory (warps walk their 512 items 32 at a time in input order;
// __match_any_sync gives the in-step order, so the sort is stable), stages
// them in digit order and writes each digit's run contiguously - ~12-item
// runs instead of the counting scatter's single 8-byte writes.  12 items per
// thread measured best at config 5 (16: 2 x 114 KB blocks per SM waited on
// shared memory; 8: a 2x larger digit table to scan; 4: 1.4x slower).  Stable, so
// each pixel's run stays in time order and no run sort is needed.
// ---------------------------------------------------------------------------
#ifndef VKM_RS_ITEMS
#define VKM_RS_ITEMS 12
#endif
constexpr int kRsThreads = 256, kRsItems = VKM_RS_ITEMS, kRsTile = kRsThreads * kRsItems, kRsWarps = kRsThreads / 32;
constexpr int kRsBins = 256;

__global__ void __launch_bounds__(256) k_rs_tilehist(const int32_t* __restrict__ keys, int64_t n, int shift,
                                                     int ntiles, int* __restrict__ tab) {
  pdl_wait();
  __shared__ int h[kRsBins];
  static_assert(kRsItems % 4 == 0, "one thread = kRsItems / 4 16-byte key loads");
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    h[threadIdx.x] = 0;
    const int64_t e0 = int64_t(t) * kRsTile;
    uint32_t k[kRsItems];
    if (e0 + kRsTile <= n) {   // full tile: independent 16-byte loads per thread, issued together
      const int4* src = reinterpret_cast<const int4*>(keys + e0);
#pragma unroll
      for (int j = 0; j < kRsItems / 4; ++j) {
        const int4 v = __ldcs(src + threadIdx.x + 256 * j);
        k[4 * j] = uint32_t(v.x);
        k[4 * j + 1] = uint32_t(v.y);
        k[4 * j + 2] = uint32_t(v.z);
        k[4 * j + 3] = uint32_t(v.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kRsItems; ++j) {
        const int64_t e = e0 + 4 * (threadIdx.x + 256 * (j >> 2)) + (j & 3);
        k[j] = e < n ? uint32_t(__ldcs(keys + e)) : 0xFFFFFFFFu;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRsItems; ++j) {
      const int64_t e = e0 + 4 * (threadIdx.x + 256 * (j >> 2)) + (j & 3);
      if (e < n) atomicAdd(h + ((k[j] >> shift) & 0xFF), 1);
    }
    __syncthreads();
    tab[int64_t(threadIdx.x) * ntiles + t] = h[threadIdx.x];   // digit-major: the scan gives global offsets
    __syncthreads();
  }
  pdl_trigger();
}

// The tile's keys and values arrive by two bulk copies (TMA engine) into an
// input buffer, issued for the block's next tile as soon as the current one
// is in registers, so the loads' DRAM latency overlaps the ranking, staging
// and writing of the current tile.  (Loading with per-thread loads at the top
// of each tile left the 16 resident warps per SM waiting on DRAM: 22 % of
// HBM, 0.36 ms per pass at config 5.)
#ifndef VKM_RS_MINB
#define VKM_RS_MINB 2
#endif
template <bool kMatch>
__global__ void __launch_bounds__(kRsThreads, VKM_RS_MINB) k_rs_scatter(const int32_t* __restrict__ kin,
                                                           const uint64_t* __restrict__ vin, int64_t n, int shift,
                                                           int ntiles, const int* __restrict__ off,
                                                           int32_t* __restrict__ kout, uint64_t* __restrict__ vout) {
  extern __shared__ __align__(128) uint8_t rs_smem[];
  uint64_t* ival = reinterpret_cast<uint64_t*>(rs_smem);                      // [kRsTile] input values (TMA)
  uint64_t* sval = ival + kRsTile;                                            // [kRsTile] staged values
  int32_t* ikey = reinterpret_cast<int32_t*>(sval + kRsTile);                 // [kRsTile] input keys (TMA)
  int32_t* skey = ikey + kRsTile;                                             // [kRsTile] staged keys
  unsigned int* wcnt = reinterpret_cast<unsigned int*>(skey + kRsTile);       // [kRsWarps][256]
  unsigned int* tbase = wcnt + kRsWarps * kRsBins;                            // [256] tile-local digit start
  int* gofs = reinterpret_cast<int*>(tbase + kRsBins);                        // [256] global start of the tile's run
  unsigned int* wmask = reinterpret_cast<unsigned int*>(gofs + kRsBins);     // [kRsWarps][256] digit lane masks
  uint64_t* bar = reinterpret_cast<uint64_t*>(wmask + kRsWarps * kRsBins);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  // bytes of tile t the bulk copies bring (16-byte multiples; the rest of a
  // ragged last tile is read from global memory)
  auto kbytes = [&](int t) { return uint32_t(min(int64_t(kRsTile), n - int64_t(t) * kRsTile) * 4) & ~15u; };
  auto vbytes = [&](int t) { return uint32_t(min(int64_t(kRsTile), n - int64_t(t) * kRsTile) * 8) & ~15u; };
  auto issue = [&](int t) {   // one thread
    if (t >= ntiles) return;
    const uint32_t kb = kbytes(t), vb = vbytes(t);
    fence_async_smem();   // the buffer's previous contents were read through the generic proxy
    mbar_arrive_tx(bar, kb + vb);
    if (kb) bulk_g2s(ikey, kin + int64_t(t) * kRsTile, kb, bar);
    if (vb) bulk_g2s(ival, vin + int64_t(t) * kRsTile, vb, bar);
  };
  for (int i = threadIdx.x; i < kRsWarps * kRsBins; i += blockDim.x) wmask[i] = 0u;   // kept zero between steps
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0) issue(blockIdx.x);
  uint32_t phase = 0;
  // the digit's global start for the block's next tile, loaded a tile ahead
  // (256 scattered words of the digit-major table: an L2 round trip)
  int gnext = blockIdx.x < ntiles ? __ldg(off + int64_t(threadIdx.x) * ntiles + blockIdx.x) : 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < kRsWarps * kRsBins; i += blockDim.x) wcnt[i] = 0;
    gofs[threadIdx.x] = gnext;
    if (t + int(gridDim.x) < ntiles) gnext = __ldg(off + int64_t(threadIdx.x) * ntiles + t + gridDim.x);
    const int64_t t0 = int64_t(t) * kRsTile;
    const int valid = int(min(int64_t(kRsTile), n - t0));
    const int kfull = int(kbytes(t) >> 2), vfull = int(vbytes(t) >> 3);
    const int wb = w * (kRsTile / kRsWarps);   // this warp's 512 items (tile-local)
    uint32_t key[kRsItems];
    uint64_t val[kRsItems];
    unsigned int wrank[kRsItems];
    unsigned int* wc = wcnt + w * kRsBins;
    unsigned int* wm = wmask + w * kRsBins;
    mbar_wait(bar, phase);
    phase ^= 1u;
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {   // warp-striped: step k covers items wb + 32k .. +31
      const int i = wb + k * 32 + lane;
      key[k] = i < kfull ? uint32_t(ikey[i]) : (i < valid ? uint32_t(__ldg(kin + t0 + i)) : 0xFFFFFFFFu);
      val[k] = i < vfull ? ival[i] : (i < valid ? __ldg(vin + t0 + i) : 0ull);
    }
    __syncthreads();   // input buffer consumed, counters zeroed
    if (threadIdx.x == 0) issue(t + gridDim.x);
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
      const bool ok = wb + k * 32 + lane < valid;
      unsigned d, peers;
      if (kMatch) {   // few distinct digits (the top pass): MATCH.ANY
        d = ok ? (key[k] >> shift) & 0xFF : 0x100u;
        peers = __match_any_sync(kFullMask, d);
      } else {
        // lanes with equal digits: each ORs its bit into the digit's mask
        // word (shared atomics; MATCH.ANY over up to 32 distinct 8-bit digits
        // was the kernel's main stall: 0.36 -> 0.31 ms per pass at config 5)
        d = (key[k] >> shift) & 0xFF;
        if (ok) atomicOr(wm + d, 1u << lane);
        __syncwarp();
        peers = ok ? wm[d] : 0u;
      }
      const unsigned before = __popc(peers & lt);
      const unsigned c = ok ? wc[d] : 0u;
      wrank[k] = c + before;
      __syncwarp();
      if (ok && before == 0) {
        wc[d] = c + __popc(peers);
        if (!kMatch) wm[d] = 0u;
      }
      __syncwarp();
    }
    __syncthreads();
    {   // per digit: exclusive over warps, tile total
      const int d = threadIdx.x;   // kRsThreads == kRsBins
      unsigned int run = 0;
      for (int v2 = 0; v2 < kRsWarps; ++v2) {
        const unsigned int c = wcnt[v2 * kRsBins + d];
        wcnt[v2 * kRsBins + d] = run;
        run += c;
      }
      tbase[d] = run;
    }
    __syncthreads();
    if (w == 0) {   // exclusive scan of the tile's digit totals (8 digits per lane)
      unsigned int v8[8], sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v8[i] = tbase[lane * 8 + i];
        sum += v8[i];
      }
      unsigned int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int u = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += u;
      }
      unsigned int r = incl - sum;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        tbase[lane * 8 + i] = r;
        r += v8[i];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {   // stage in digit order
      if (wb + k * 32 + lane < valid) {
        const unsigned d = (key[k] >> shift) & 0xFF;
        const unsigned pos = tbase[d] + wcnt[w * kRsBins + d] + wrank[k];
        skey[pos] = int32_t(key[k]);
        sval[pos] = val[k];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < valid; i += blockDim.x) {   // each digit's run contiguously
      const uint32_t k = uint32_t(skey[i]);
      const unsigned d = (k >> shift) & 0xFF;
      const int64_t dst = int64_t(gofs[d]) + (i - int(tbase[d]));
      kout[dst] = int32_t(k);
      vout[dst] = sval[i];
    }
    __syncthreads();
  }
  pdl_trigger();
}

size_t radix_smem_bytes() { return size_t(kRsTile) * 24 + size_t(2 * kRsWarps + 2) * kRsBins * 4 + 16; }

// ---------------------------------------------------------------------------
// Exclusive scan of the per-pixel counts, one pass: each 4096-count tile
// publishes its aggregate, looks back over its predecessors' published
// aggregates / inclusive prefixes (a warp reads 32 at a time) and publishes
// its own inclusive prefix (decoupled look-back).  A tile-state word packs
// (epoch, flag, value) so the states never need a reset: words of another
// launch carry another epoch and read as "not yet published".  Tiles are
// taken in increasing order by a grid no larger than what is co-resident, so
// every predecessor a tile waits on is being processed.
// ---------------------------------------------------------------------------
#ifndef VKM_SCAN_ITEMS
#define VKM_SCAN_ITEMS 16
#endif
constexpr int kScanThreads = 256, kScanItems = VKM_SCAN_ITEMS, kScanTile = kScanThreads * kScanItems;
__global__ void __launch_bounds__(kScanThreads) k_scan(const int* __restrict__ in, int* __restrict__ out, int64_t m,
                                                       int ntiles, unsigned long long* __restrict__ state,
                                                       uint32_t epoch) {
  pdl_wait();
  __shared__ int warp_sum[kScanThreads / 32];
  __shared__ int tile_prefix;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t i0 = int64_t(t) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    int v[kScanItems];
    if (i0 + kScanItems <= m) {
      const int4* q = reinterpret_cast<const int4*>(in + i0);
#pragma unroll
      for (int k = 0; k < kScanItems / 4; ++k) {
        const int4 w = q[k];
        v[4 * k] = w.x; v[4 * k + 1] = w.y; v[4 * k + 2] = w.z; v[4 * k + 3] = w.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kScanItems; ++k) v[k] = i0 + k < m ? in[i0 + k] : 0;
    }
    int tsum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) tsum += v[k];
    int incl = tsum;   // warp inclusive scan of the thread sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFullMask, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    int wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
      const int ws = warp_sum[w];
      wpre += w < wid ? ws : 0;
      total += ws;
    }
    if (wid == 0) {
      const uint32_t excl = lookback_publish(state, t, uint32_t(total), epoch);
      if (lane == 0) tile_prefix = int(excl);
    }
    __syncthreads();
    int run = tile_prefix + wpre + incl - tsum;
    if (i0 + kScanItems <= m) {
      int4* q = reinterpret_cast<int4*>(out + i0);
#pragma unroll
      for (int k = 0; k < kScanItems / 4; ++k) {
        int4 w;
        w.x = run; run += v[4 * k];
        w.y = run; run += v[4 * k + 1];
        w.z = run; run += v[4 * k + 2];
        w.w = run; run += v[4 * k + 3];
        q[k] = w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kScanItems; ++k)
        if (i0 + k < m) {
          out[i0 + k] = run;
          run += v[k];
        }
    }
    __syncthreads();   // warp_sum / tile_prefix are reused by the next tile
  }
  pdl_trigger();
}


__global__ void __launch_bounds__(512) k_longsort(const int* __restrict__ start, uint64_t* __restrict__ val_s,
                                                  const int* __restrict__ longlist,
                                                  const int* __restrict__ longcount) {
  pdl_wait();
  __shared__ uint64_t sm[kSmemRun];
  const int nl = *longcount;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int p = longlist[li];
    const int s = start[p], L = start[p + 1] - s;
    int N = 1;
    while (N < L) N <<= 1;
    const bool in_smem = N <= kSmemRun;
    uint64_t* a = in_smem ? sm : val_s + s;
    if (in_smem)
      for (int i = threadIdx.x; i < L; i += blockDim.x) sm[i] = val_s[s + i];
    __syncthreads();
    // bitonic sort, ascending-only form: merge stage k first compares i with
    // its mirror in the 2k block, then half-cleaners; partners >= L are +inf
    for (int k = 2; k <= N; k <<= 1) {
      for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
        const int lo = (i / (k / 2)) * k + (i % (k / 2));
        const int hi = (i / (k / 2)) * k + k - 1 - (i % (k / 2));
        if (hi < L) cas_slot(a[lo], a[hi]);
      }
      __syncthreads();
      for (int j = k / 4; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
          const int lo = (i / j) * 2 * j + (i % j), hi = lo + j;
          if (hi < L) cas_slot(a[lo], a[hi]);
        }
        __syncthreads();
      }
    }
    if (in_smem)
      for (int i = threadIdx.x; i < L; i += blockDim.x) val_s[s + i] = sm[i];
    __syncthreads();
  }
  pdl_trigger();   // dependents may launch as this grid drains
}

// ---------------------------------------------------------------------------
// k_reduce_x1: the same computation with one channel per lane and two warps
// per (row, segment) item (channels 0-31 and 32-63).  Each lane packs two
// consecutive events of its channel into one f32x2 sin/cos and adds them in
// slot order, so sums keep the reference's order.  Same instruction count as
// k_reduce_x, half the shared memory per warp (the ring holds one complex per
// lane) and twice the warps, i.e. twice the latency hiding.
// ---------------------------------------------------------------------------
constexpr int kRx1Warps = 4;   // two items per block
constexpr int kRx1Group = 4;   // events per group: one float4 of time arguments
size_t reduce_x1_smem(int dx) { return size_t(kRx1Warps) * ((2 * dx + 1) * 256 + kRxEnds * 4); }

template <bool kMufu>
__global__ void __launch_bounds__(kRx1Warps * 32) k_reduce_x1(const int* __restrict__ start,
                                                              const uint64_t* __restrict__ val_s,
                                                              const float* __restrict__ tf,
                                                              const float2* __restrict__ mx,
                                                              const float2* __restrict__ my, int W, int H, int nb,
                                                              int dx, int S, int nseg, int64_t P,
                                                              float2* __restrict__ R) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t rx_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int half = wib & 1;                        // channel half of this warp
  const int c = half * 32 + lane;                  // this lane's channel
  const int RL = 2 * dx + 1;
  float2* const ring0 = reinterpret_cast<float2*>(rx_smem) + wib * RL * 32 + lane;
  float2* const ring_end = ring0 + RL * 32;
  int* const ends = reinterpret_cast<int*>(rx_smem + size_t(kRx1Warps) * RL * 256) + wib * kRxEnds;
  const float Tc = __ldg(tf + c);
  const uint64_t TT = f2pack(Tc, Tc);
  const float2* mxc = mx + c;                      // mxc[x * 64]
  // packed-pair output position of channel c inside a pixel's 64-B plane chunk
  float* const Rf = reinterpret_cast<float*>(R) + int64_t(c >> 3) * P * 16 + ((c & 7) >> 1) * 4 + (c & 1);
  const int64_t items = int64_t(nb) * H * nseg;
  const int64_t nwarp_items = int64_t(gridDim.x) * (kRx1Warps / 2);
  for (int64_t it = int64_t(blockIdx.x) * (kRx1Warps / 2) + (wib >> 1); it < items; it += nwarp_items) {
    const int y = int(it / nseg);
    const int x0 = int(it - int64_t(y) * nseg) * S, x1 = min(W, x0 + S);
    const int xs = x0 - dx, nx = x1 + dx - xs;
    const int* st = start + int64_t(y) * W;
    const int jfirst = __ldg(st + max(0, xs)), jend = __ldg(st + min(W, x1 + dx));
    __syncwarp();
    for (int k = lane; k <= nx; k += 32) {
      const int x = xs + k;
      ends[k] = k == nx ? jend : (x < 0 ? jfirst : (x < W ? __ldg(st + x + 1) : jend));
    }
    for (int k = 0; k < RL; ++k) ring0[k * 32] = make_float2(0.f, 0.f);
    __syncwarp();
    const float2 fy = __ldg(my + int64_t(y % H) * 64 + c);
    float* out = Rf + (int64_t(y) * W + x0) * 16;
    // time arguments of the item's slots, staged 32 at a time in shared memory
    // (one LDS.128 broadcast per group of 4 events instead of 4 shuffles)
    float* const abuf = reinterpret_cast<float*>(ends + kRxEnds - 64);   // 2 x 32 floats at the end of ends[]
    auto ld_a = [&](int jj) { return jj < jend ? slot_arg(__ldg(val_s + jj)) : 0.f; };
    int jb = jfirst;
    float av1 = ld_a(jb + 32 + lane);
    abuf[lane] = ld_a(jb + lane);
    __syncwarp();

    int k = 0;
    int je = ends[0];
    float2 mc = __ldg(mxc + int64_t(min(max(xs, 0), W - 1)) * 64);
    uint64_t g = 0;                                  // packed (re, im) sum of the current pixel
    float ar = 0.f, ai = 0.f;
    float2* pn = ring0;
    float2* po = ring0 + 32;
    auto finish = [&]() {
      float gr, gi;
      f2unpack(g, gr, gi);
      const float mr = fmaf(gr, mc.x, -gi * mc.y), mi = fmaf(gr, mc.y, gi * mc.x);
      const float2 old = *po;
      *pn = make_float2(mr, mi);
      ar += mr;
      ai += mi;
      if (k >= 2 * dx) {
        out[0] = fmaf(ar, fy.x, -ai * fy.y);
        out[2] = fmaf(ar, fy.y, ai * fy.x);
        out += 16;
      }
      ar -= old.x;
      ai -= old.y;
      g = 0;
      pn = po;
      po = (po + 32 == ring_end) ? ring0 : po + 32;
      ++k;
      je = ends[k];
      mc = __ldg(mxc + int64_t(min(max(xs + k, 0), W - 1)) * 64);
    };

    for (int j = jfirst; j < jend; j += kRx1Group) {
      if (j - jb >= 32) {
        jb += 32;
        __syncwarp();
        abuf[lane] = av1;
        __syncwarp();
        av1 = ld_a(jb + 32 + lane);
      }
      const float4 a4 = *reinterpret_cast<const float4*>(abuf + (j - jb));
      uint64_t cs[kRx1Group];
      sincos2_cs_hot<kMufu>(fmul2(f2pack(a4.x, a4.y), TT), cs[0], cs[1]);
      sincos2_cs_hot<kMufu>(fmul2(f2pack(a4.z, a4.w), TT), cs[2], cs[3]);
#pragma unroll
      for (int u = 0; u < kRx1Group; ++u) {
        if (j + u >= je) {
          if (j + u >= jend) break;
          do finish(); while (j + u >= je);
        }
        g = fadd2(g, cs[u]);
      }
    }
    while (k < nx) finish();
  }
  pdl_trigger();   // dependents may launch as this grid drains
}

// order[slot] = event index of the slot (slots [start[P], n): -1, events outside the sensor)
__global__ void k_slot_events(const uint64_t* __restrict__ val_s, const int* __restrict__ valid, int64_t n,
                              int32_t* __restrict__ order) {
  const int64_t m = *valid;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
    order[j] = j < m ? slot_event(val_s[j]) : -1;
}

void launch_slot_events(const uint64_t* val_s, const int* valid, int64_t n, int32_t* order, cudaStream_t s) {
  k_slot_events<<<int(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(val_s, valid, n, order);
}

bool sincos_mufu() {
  const char* e = std::getenv("VKM_SINCOS");
  return !(e && std::strcmp(e, "poly") == 0);
}

uint32_t next_scan_epoch() {
  static std::atomic<uint32_t> epoch{0};
  uint32_t e;
  do e = (epoch.fetch_add(1) + 1) & 0x3fffffffu; while (e == 0);   // 0 marks never-published words
  return e;
}

size_t scan_state_words(int64_t P) { return size_t((P + 1 + kScanTile - 1) / kScanTile); }

int launch_sort_events(const double* ev, const uint2* packed, const SliceTab& st, double delta_t, int W, int H,
                       const GridBufs& g, const SortBufs& sb, float* flows_invalid, int32_t* counts_invalid,
                       cudaStream_t s) {
  const int64_t P = int64_t(W) * H * st.nb;
  const int64_t n = st.off[st.nb];
  int launches = 0;
  cudaMemsetAsync(g.C, 0, sizeof(int) * (P + 1), s);
  // Event-parallel kernels run one co-resident wave (grid-stride beyond it):
  // blocks then progress together through the time-ordered events, so the
  // arrival ranks of k_prep's histogram atomics come out nearly in time order
  // and k_runsort's insertion sorts stay near linear.  (With twice the
  // resident blocks, the second half of the grid ran after the first and every
  // run became two interleaved sequences: config-5 run sort 963 us.)
  static thread_local int dev_cached = -1, ev_blocks = 0;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
      int sms = 148, per = 1;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_prep, 256, 0);
      ev_blocks = std::max(1, per) * sms;
      dev_cached = dev;
    }
  }
#if !VKM_RUNSORT_LONG_INBLOCK
  cudaMemsetAsync(sb.longcount, 0, sizeof(int), s);
#endif
  // The counting scatter + run sort serves every density.  The row-bucket
  // path (VKM_SORT=rows, tested for exact order) measured slower at config 5
  // (rowhist 0.17 + rowscatter 1.11 + xsort 0.83 ms against scatter 0.98 +
  // run sort 0.59 ms): both scatter 8-byte records to sectors spread over a
  // destination far larger than L2 (DRAM read-modify-writes).
  static const int sort_env = [] {
    const char* e = std::getenv("VKM_SORT");
    if (!e) return 0;
    if (std::strcmp(e, "counting") == 0) return 1;
    if (std::strcmp(e, "rows") == 0) return 2;
    if (std::strcmp(e, "radix") == 0) return 3;
    return 0;
  }();
  const int R = st.nb * H;
  const bool rows_ok = R <= kMsdMaxRows && W <= kXsortMaxW;
  const bool dense = rows_ok && sort_env == 2;
  // dense slices (mean run > 8 events, >= 1M events): the radix sort
  const bool radix = sort_env == 3 || (sort_env == 0 && double(n) > 8.0 * double(P) && n >= (1 << 20));
  if (n > 0) {
    const int blocks = int(std::min<int64_t>((n + 255) / 256, ev_blocks));
    int32_t* rank = (dense || radix) ? nullptr : sb.rank;
    int* cnt = radix ? nullptr : g.C;   // radix: run starts and counts come from the sorted keys
    if (packed)
      k_prep_packed<<<blocks, 256, 0, s>>>(packed, st, W, H, sb.pix, sb.val, rank, cnt, flows_invalid,
                                           counts_invalid);
    else
      k_prep<<<blocks, 256, 0, s>>>(ev, st, delta_t, W, H, sb.pix, sb.val, rank, cnt, flows_invalid, counts_invalid);
    ++launches;
  }
  if (!(n > 0 && radix)) {
    const int ntiles = int((P + 1 + kScanTile - 1) / kScanTile);
    launch_pdl(k_scan, std::min(ntiles, 148 * 4), kScanThreads, 0, s, static_cast<const int*>(g.C), sb.start,
               P + 1, ntiles, sb.scan_state, next_scan_epoch());
    ++launches;
  }
  if (n > 0 && radix) {
    int bits = 1;
    while ((int64_t(1) << bits) <= P) ++bits;   // keys in [0, P] (P: outside the sensor)
    const int passes = (bits + 7) / 8;
    const int ntiles = int((n + kRsTile - 1) / kRsTile);
    const int64_t m = int64_t(kRsBins) * ntiles;
    int* tab = sb.msd_tab;                        // msd_tab_words(n) >= 256 * ntiles per half
    int* off = sb.msd_tab + m;
    const size_t smem = radix_smem_bytes();
    cudaFuncSetAttribute(k_rs_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(k_rs_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per = 1, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rs_scatter<false>, kRsThreads, smem);
    const int grid = std::min(ntiles, std::max(1, per) * sms);
    const int mt = int((m + kScanTile - 1) / kScanTile);
    const int32_t* kin = sb.pix;
    const uint64_t* vin = sb.val;
    for (int p = 0; p < passes; ++p) {
      int32_t* kout = p == passes - 1 ? sb.pix_s : (p % 2 == 0 ? sb.rank : sb.pix);
      uint64_t* vout = p == passes - 1 ? sb.val_s : (p % 2 == 0 ? sb.bkt : sb.val);
      launch_pdl(k_rs_tilehist, std::min(ntiles, ev_blocks), 256, 0, s, kin, n, 8 * p, ntiles, tab);
      launch_pdl(k_scan, std::min(mt, 148 * 4), kScanThreads, 0, s, static_cast<const int*>(tab), off, m, mt,
                 sb.msd_state, next_scan_epoch());
      // a top digit of <= 4 bits has <= 16 values: MATCH.ANY ranks it faster
      // than the shared-atomic masks (few words, many lanes each)
      if (bits - 8 * p <= 4)
        launch_pdl(k_rs_scatter<true>, grid, kRsThreads, smem, s, kin, vin, n, 8 * p, ntiles,
                   static_cast<const int*>(off), kout, vout);
      else
        launch_pdl(k_rs_scatter<false>, grid, kRsThreads, smem, s, kin, vin, n, 8 * p, ntiles,
                   static_cast<const int*>(off), kout, vout);
      kin = kout;
      vin = vout;
    }
    launches += 3 * passes;
    launch_pdl(k_run_starts, int((n + 1 + 1023) / 1024), 256, 0, s, static_cast<const int32_t*>(sb.pix_s), n, P,
               sb.start);
    launch_pdl(k_counts_from_starts, int(std::min<int64_t>((P + 256) / 256, ev_blocks)), 256, 0, s,
               static_cast<const int*>(sb.start), P, g.C);
    launches += 2;
  } else if (n > 0 && dense) {
    const int ntiles = int((n + kMsdTile - 1) / kMsdTile);
    const int64_t m = int64_t(R) * ntiles;
    int* tab = sb.msd_tab;
    int* off = sb.msd_tab + m;
    const int gb = std::min(ntiles, ev_blocks / 2);
    launch_pdl(k_rowhist, gb, kMsdThreads, size_t(R) * 4, s, static_cast<const int32_t*>(sb.pix), n, W, R, ntiles,
               tab);
    const int mt = int((m + kScanTile - 1) / kScanTile);
    launch_pdl(k_scan, std::min(mt, 148 * 4), kScanThreads, 0, s, static_cast<const int*>(tab), off, m, mt,
               sb.msd_state, next_scan_epoch());
    const size_t rs_smem = size_t(kMsdWarps) * R * 4;
    cudaFuncSetAttribute(k_rowscatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(size_t(kMsdWarps) * kMsdMaxRows * 4));
    launch_pdl(k_rowscatter, gb, kMsdThreads, rs_smem, s, static_cast<const int32_t*>(sb.pix),
               static_cast<const uint64_t*>(sb.val), n, W, R, ntiles, static_cast<const int*>(off), sb.bkt, sb.rank);
    const size_t xs_smem = size_t(kXsortWarps) * W * 4;
    cudaFuncSetAttribute(k_xsort, cudaFuncAttributeMaxDynamicSharedMemorySize, int(size_t(kXsortWarps) * kXsortMaxW * 4));
    // one CTA per SM: the rows in flight (~0.5 MB of slots each at config 5)
    // stay in L2 until their scattered 8-byte writes complete
    launch_pdl(k_xsort, std::min(R, 148), kXsortThreads, xs_smem, s, static_cast<const uint64_t*>(sb.bkt),
               static_cast<const int32_t*>(sb.rank), static_cast<const int*>(sb.start), W, R, sb.val_s, sb.pix_s);
    launches += 4;
  } else if (n > 0) {
    const int eb = int(std::min<int64_t>((n + 255) / 256, ev_blocks));
    launch_pdl(k_scatter, eb, 256, 0, s, static_cast<const int32_t*>(sb.pix), static_cast<const uint64_t*>(sb.val),
               static_cast<const int32_t*>(sb.rank), n, P, static_cast<const int*>(sb.start), sb.val_s);
    // pixels per runsort block step (one thread per pixel, 16..128) and the
    // stage sized for them (~1.3x the expected slots)
    const double mean_run = double(n) / double(std::max<int64_t>(P, 1));
    int ppb = kRunsortThreads;
    while (ppb > 16 && ppb * mean_run > 0.75 * kRunsortStage) ppb >>= 1;
    const int cap = int(std::min<double>(kRunsortStage, std::max(1024.0, 1.3 * ppb * mean_run + 256.0)));
    const int pb = int(std::min<int64_t>((P + ppb - 1) / ppb, 148 * 16));
    cudaFuncSetAttribute(k_runsort, cudaFuncAttributeMaxDynamicSharedMemorySize, kRunsortStage * 8);
    launch_pdl(k_runsort, pb, kRunsortThreads, size_t(cap) * 8, s, static_cast<const int*>(sb.start), P, ppb, cap,
               sb.val_s, sb.pix_s, sb.longlist, sb.longcount);
#if VKM_RUNSORT_LONG_INBLOCK
    launches += 2;
#else
    launch_pdl(k_longsort, 148, 512, 0, s, sb.start, sb.val_s, sb.longlist, sb.longcount);
    launches += 3;
#endif
  }
  return launches;
}

namespace {
int resident_blocks(const void* fn, int threads, size_t smem) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
  return std::max(1, per) * sms;
}
}  // namespace

void launch_reduce_raw(const DevTables& tb, int W, int H, int D8, const GridBufs& g, const SortBufs& sb,
                       cudaStream_t s) {
  const int64_t P = int64_t(W) * H;
  if (D8 == 64) {
    const int64_t warps = (P + 31) / 32;
    static const int res = resident_blocks(reinterpret_cast<const void*>(k_reduce), 256, 0);
    const int blocks = int(std::min<int64_t>((warps + 7) / 8, res));
    k_reduce<<<blocks, 256, 0, s>>>(sb.start, sb.val_s, sb.pix_s, tb.tf, tb.mx, tb.my, W, P, g.G);
  } else {
    const int cp = D8 >> 1, pps = 32 / cp;
    const int64_t warps = (P + pps - 1) / pps;
    const int blocks = int(std::min<int64_t>((warps + 7) / 8, 148 * 64));
    k_reduce_small<<<blocks, 256, 0, s>>>(sb.start, g.C, sb.val_s, tb.tf, tb.mx, tb.my, W, P, D8, g.G);
  }
}

bool reduce_x_supported(int D8, int dx) { return D8 == 64 && dx >= 1 && dx <= kMaxFusedDx; }

void launch_reduce_x(const DevTables& tb, int W, int H, int nb, int dx, const SortBufs& sb, float2* R,
                     int num_sms, cudaStream_t s) {
  const int64_t P = int64_t(W) * H * nb;
  static const int variant_env = [] {
    const char* e = std::getenv("VKM_RX");
    return e ? std::atoi(e) : -1;
  }();
  // k_reduce_x1 issues ~35 % more instructions but runs twice the warps: it
  // wins where the (2δx+1)-pixel ring limits occupancy (cfg3, δ = 20: -3.6 %),
  // loses slightly at δ = 10 (cfg2: +2 %).
  // (With the MUFU sin/cos, k_reduce_x is also the faster one at δ = 20:
  // cfg3 accumulate 0.57 vs 0.67 ms; the x1 variant stays behind VKM_RX=1.)
  const int variant = variant_env >= 0 ? variant_env : 0;
  if (variant == 1) {   // one channel per lane, two warps per item
    const size_t smem = reduce_x1_smem(dx);
    auto kern1 = sincos_mufu() ? k_reduce_x1<true> : k_reduce_x1<false>;
    // per call: the attribute is per device, and one process may drive several
    cudaFuncSetAttribute(kern1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(reduce_x1_smem(kMaxFusedDx)));
    int per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern1, kRx1Warps * 32, smem);
    const int64_t res_items = int64_t(std::max(1, per)) * num_sms * (kRx1Warps / 2);
    int S = kRxMaxSeg;
    while (S > 32 && 4 * int64_t(H) * nb * ((W + S - 1) / S) < 3 * res_items) S >>= 1;
    const int nseg = (W + S - 1) / S;
    const int64_t items = int64_t(H) * nb * nseg;
    const int blocks = int(std::min<int64_t>((items + 1) / 2, res_items / 2));
    launch_pdl(kern1, blocks, kRx1Warps * 32, smem, s, sb.start, sb.val_s, tb.tf, tb.mx, tb.my, W, H, nb, dx,
               S, nseg, P, R);
    return;
  }
  const size_t smem = reduce_x_smem(dx);
  auto kern = sincos_mufu() ? k_reduce_x<true> : k_reduce_x<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(reduce_x_smem(kMaxFusedDx)));
  int per = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kRxWarps * 32, smem);
  const int64_t res_warps = int64_t(std::max(1, per)) * num_sms * kRxWarps;
  // Segment width: long segments keep the recomputed 2δx halo small; shorter
  // ones when a row split into 128-column segments would not fill the GPU.
  static const int seg_env = [] {
    const char* e = std::getenv("VKM_RX_SEG");
    return e ? std::atoi(e) : 0;
  }();
  // (Halve S only while the items would fill less than half the resident
  // warps: config 1 at S = 64 - 1560 items, 0.5 of a wave - beat S = 32 by
  // 3 %, whose 2δx halo is 63 % of its segment.)
  int S = seg_env > 0 ? std::min(seg_env, kRxMaxSeg) : kRxMaxSeg;
  if (seg_env <= 0)
    while (S > 32 && 2 * int64_t(H) * nb * ((W + S - 1) / S) < res_warps) S >>= 1;
  const int nseg = (W + S - 1) / S;
  const int64_t items = int64_t(H) * nb * nseg;
  const int blocks = int(std::min<int64_t>((items + kRxWarps - 1) / kRxWarps, res_warps / kRxWarps));
  launch_pdl(kern, blocks, kRxWarps * 32, smem, s, sb.start, sb.val_s, tb.tf, tb.mxp, tb.myp, W, H, nb, dx, S, nseg,
             P, R);
}

}  // namespace vkm
