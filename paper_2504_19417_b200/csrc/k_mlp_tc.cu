// Fused gather + de-phase + ÷count + two-layer head on the 5th-gen tensor
// cores (tcgen05, sm_100a) for D = 64, hidden = 128.
//
// Per 128-event tile:  hidden[128 ev x 128] = F[128 x 128] · W1ᵀ accumulated in
// TMEM, then out = relu(hidden + b1) · W2ᵀ + b2 in the epilogue (flow.py:98-106).
//
// Precision modes (numerics in DESIGN.md):
//   F16X3  F = Fh + Fl, W1 = Wh + Wl with fp16 hi/lo splits (22 significant
//          bits); D = Fh·Whᵀ + Fh·Wlᵀ + Fl·Whᵀ  -> fp32-equivalent products.
//          Power-of-two pre-scales keep the lo parts out of fp16 subnormals.
//   BF16   one bf16 pass, D = Fh·Whᵀ (fast mode, stated angular bound).
//
// Warp roles (672 threads, one persistent CTA per SM):
//   warps 0-15 producers: one warp per 8 tile rows; gather the pooled grid
//              row of each event (coalesced 512 B), de-phase, ÷count, split,
//              and store the fp16 A tile in the UMMA K-major SWIZZLE_128B layout
//   warps 16-19 epilogue: tcgen05.ld of the accumulator (warp q = id % 4 owns
//              TMEM lanes 32q..32q+31 = tile rows), bias + ReLU + 128->2, store
//   warp 20    TMEM allocator + single-thread tcgen05.mma issuer
// Pipelines: A stages (full/empty mbarriers, depth 2) and TMEM accumulators
// (tfull/tempty, depth 2), so gather(i+1), MMA(i) and epilogue(i-1) overlap.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "../../include/veckm.h"
#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {
namespace tc {

constexpr int kM = 128;             // events per tile (UMMA M)
constexpr int kN = 128;             // hidden units (UMMA N)
constexpr int kK = 128;             // features 2D (UMMA K total)
constexpr int kStages = 2;
constexpr int kAcc = 4;                // TMEM accumulators (4 x 128 columns = all 512)
constexpr int kTileBytes = kM * kK * 2;        // 32 KB per fp16 operand image
constexpr int kAtomBytes = kM * 128;           // one 64-wide K atom: 128 rows x 128 B
constexpr int kProdWarps = 16;                // producer warps (8 tile rows each)
constexpr int kThreads = (kProdWarps + 5) * 32; // + 4 epilogue warps + 1 MMA warp
constexpr uint32_t kTmemCols = kAcc * kN;
#ifndef VKM_K3_QD
#define VKM_K3_QD 4
#endif
constexpr int kQD = VKM_K3_QD;                  // per-warp cp.async ring of pooled rows (kQD - 1 in flight)
#ifndef VKM_K3_PHB
#define VKM_K3_PHB 2   // 1, 2, 4, 8 measured within 0.5 % (2 best at cfg2 and cfg3)
#endif
constexpr int kPhB = VKM_K3_PHB;                // rows whose phases are computed back to back (divides 8)

struct Smem {
  // operand images, each 1024-byte aligned (SWIZZLE_128B atoms)
  uint8_t bh[kTileBytes];
  uint8_t bl[kTileBytes];
  uint8_t ah[kStages][kTileBytes];
  uint8_t al[kStages][kTileBytes];
  float4 qring[kProdWarps][kQD][32];   // per producer warp: pooled rows of its next kQD-1 events
  // head constants with the power-of-two operand scale s = w_scale·f_scale
  // folded in: relu(acc/s + b1)·w2 == relu(acc + s·b1)·(w2/s) exactly
  float b1s[kN];    // s·b1
  float w2a[kN];    // w2[0][n] / s
  float w2b[kN];    // w2[1][n] / s
  float b2[2];
  float scale;
  uint32_t tmem_base;
  unsigned long long full[kStages], empty[kStages], tfull[kAcc], tempty[kAcc];
};

static_assert(sizeof(Smem) + 1024 <= 232448, "K3 shared memory exceeds the 227 KB opt-in limit");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Bounded parity wait: a descriptor or protocol bug traps (kernel error)
// instead of hanging the device.
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
    // suspend-time hint: a waiting warp sleeps in the barrier unit (up to
    // ~20 us per try) instead of spinning on issue slots the producers need
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(20000u)
        : "memory");
    if (done) return;
    if (it > (1u << 20)) __trap();
  }
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B
// apart (SBO), LBO unused (=1), sm100 version bits = 1, layout type 2.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t((saddr & 0x3FFFF) >> 4)) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// Instruction descriptor, kind::f16: D=f32, A/B fp16 (fmt 0) or bf16 (fmt 1),
// both K-major, N=128, M=128.
__host__ __device__ constexpr uint32_t umma_idesc(uint32_t fmt) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(kN >> 3) << 17) | (uint32_t(kM >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(unsigned long long* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}

// Byte offset of element (row m, k) inside a K-major SWIZZLE_128B operand
// image of 128 rows x 128 K (two 64-wide K atoms of 16 KB each).
__host__ __device__ __forceinline__ uint32_t umma_off(uint32_t m, uint32_t k) {
  const uint32_t atom = k >> 6, kk = k & 63;
  const uint32_t chunk = (kk >> 3) ^ (m & 7);
  return atom * kAtomBytes + (m >> 3) * 1024 + (m & 7) * 128 + chunk * 16 + (kk & 7) * 2;
}

template <int MODE, bool kMufu>  // VKM_MLP_F16X3 or VKM_MLP_BF16; sin/cos flavour (sincos2_k3_scaled)
__global__ void __launch_bounds__(kThreads, 1)
    k_gather_mlp_tc(int64_t n, const uint64_t* __restrict__ val_s, const int32_t* __restrict__ pix_s, const int* __restrict__ nvalid_ptr,
                    const float* __restrict__ tf, int64_t P, const float2* __restrict__ Q,
                    const int* __restrict__ NQ, const uint4* __restrict__ w1h, const uint4* __restrict__ w1l,
                    const float* __restrict__ b1, const float* __restrict__ w2, const float* __restrict__ b2,
                    float w_scale, float* __restrict__ flows, int32_t* __restrict__ counts_out,
                    int prefetch_on) {
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool kSplit = (MODE == VKM_MLP_F16X3);
  const float f_scale = kSplit ? 256.f : 1.f;   // features |f| <= 1 -> keep lo parts normal

  pdl_trigger();
  // ---- one-time setup (reads only the weights, never the predecessor's outputs) ----
  {
    const int nvec = kTileBytes / 16;
    uint4* dh = reinterpret_cast<uint4*>(S.bh);
    uint4* dl = reinterpret_cast<uint4*>(S.bl);
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      dh[i] = __ldg(w1h + i);
      if (kSplit) dl[i] = __ldg(w1l + i);
    }
    const float sc = w_scale * f_scale;   // a power of two: exact scaling
    for (int i = threadIdx.x; i < kN; i += kThreads) {
      S.b1s[i] = b1[i] * sc;
      S.w2a[i] = w2[i] / sc;
      S.w2b[i] = w2[kN + i] / sc;
    }
    if (threadIdx.x == 0) {
      S.b2[0] = b2[0];
      S.b2[1] = b2[1];
      S.scale = 1.f / (w_scale * f_scale);
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&S.full[s], kProdWarps * 32);
        mbar_init(&S.empty[s], 1);
      }
      for (int a = 0; a < kAcc; ++a) {
        mbar_init(&S.tfull[a], 1);
        mbar_init(&S.tempty[a], 128);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kProdWarps + 4) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  pdl_wait();   // setup above overlapped the predecessor's tail; its outputs are read below
  const uint32_t tmem = S.tmem_base;
  const int64_t ntiles = (n + kM - 1) / kM;
  const int64_t nv = __ldg(nvalid_ptr);   // slots [0, nv) hold the in-sensor events

  if (warp < kProdWarps) {
    // ======================= producers =======================
    // Warp w fills tile rows [8w, 8w+8) (pixel-sorted slots).  Its pooled-
    // grid rows stream through a cp.async ring (3 rows in flight), the slot
    // metadata (pixel, time argument, 1/count) is loaded a tile ahead, and one
    // thread prefetches the pooled-grid rows of the next two tiles into L2
    // with bulk (TMA-engine) prefetches, so the ring mostly hits L2.
    const int c0 = 2 * lane;                      // this lane's channel pair
    const uint64_t T01 = f2pack(__ldg(tf + c0), __ldg(tf + c0 + 1));
    const float4* Q4 = reinterpret_cast<const float4*>(Q);
    const int plane = lane >> 2, q4 = lane & 3;
    constexpr int kRows = kM / kProdWarps;        // 8
    // K position of this lane's values: 4·lane (see feature_kpos)
    const uint32_t lane_atom = uint32_t(lane >> 4) * kAtomBytes;
    const uint32_t lane_chunk = uint32_t(lane & 15) >> 1, lane_byte = uint32_t(lane & 1) * 8;
    // lanes 0..7 hold the metadata of the warp's 8 rows
    // Slot metadata is pipelined over three tiles so no load is consumed right
    // after it issues: (pixel, time argument) two tiles ahead, the pooled count
    // NQ[pixel] one tile ahead (it depends on the pixel), 1/count on use.
    auto load_slot = [&](int64_t tl, float& a, int& pix) {
      const int64_t slot = tl * kM + warp * kRows + (lane & (kRows - 1));
      a = 0.f;
      pix = -1;
      if (tl < ntiles && slot < nv) {
        pix = __ldg(pix_s + slot);
        a = slot_arg(__ldg(val_s + slot));
      }
    };
    auto load_cnt = [&](int pix) { return pix >= 0 ? __ldg(NQ + pix) : 0; };
    auto recip = [&](int cnt) {   // ÷count folded with the fp16 pre-scale
      // MUFU.RCP (<= 1 ulp; the IEEE-rounded __frcp_rn cost ~2 instructions
      // per event in its fix-up sequence).  The reference divides by f32(cnt)
      // (encoder.py:345); either reciprocal differs from that by <= 1 ulp.
      float r;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(float(cnt)));
      return cnt > 0 ? r * f_scale : 0.f;
    };
    // One thread prefetches the pooled-grid rows of a future tile into L2
    // with bulk (TMA-engine) prefetches: the tile's pixel range x 8 planes.
    // VKM_TC_PREFETCH=0 disables it (A/B evidence in profiles/).
    auto prefetch_l2 = [&](int64_t tl) {
      if (!prefetch_on || tl >= ntiles || warp != 0 || lane != 0) return;
      const int64_t f = tl * kM;
      if (f >= nv) return;
      const int64_t l = (f + kM < nv ? f + kM : nv) - 1;
      const int64_t p0 = __ldg(pix_s + f), p1 = __ldg(pix_s + l);
      const uint32_t bytes = uint32_t((p1 - p0 + 1) < 2048 ? (p1 - p0 + 1) : 2048) * 64u;
      for (int pl = 0; pl < 8; ++pl) {
        const float2* src = Q + (int64_t(pl) * P + p0) * 8;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
      }
    };
    // Pooled rows stream through a per-warp ring in shared memory: row r is
    // read from slot r % kQD while the rows r+1 .. r+kQD-1 are in flight
    // (cp.async, 16 B per lane, zero-filled for empty slots), so the
    // L2/HBM latency of the gathers overlaps the de-phase/split work.
    float4* const ring = &S.qring[warp][0][lane];
    // lane-constant parts of the gather (global plane base, shared ring slot 0)
    // hoisted: per row only the pixel offset and the slot offset are added
    const float4* const qlane = Q4 + ((int64_t(plane) * P) << 2) + q4;
    const uint32_t ring_s = smem_u32(ring);
    auto issue_row = [&](int pj, int slot) {
      const float4* src = qlane + (int64_t(pj >= 0 ? pj : 0) << 2);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n\tcp.async.commit_group;" ::"r"(
                       ring_s + uint32_t(slot) * 512u),
                   "l"(src), "r"(pj >= 0 ? 16 : 0)
                   : "memory");
    };
    // Shared address of this lane's 8 bytes in row u of stage 0's hi image
    // (m = 8·warp + u; the swizzle chunk is lane_chunk ^ u); the stage and the
    // lo image are compile-time offsets, so each store is STS [reg + imm].
    uint32_t sah[kRows];
#pragma unroll
    for (int u = 0; u < kRows; ++u)
      sah[u] = smem_u32(S.ah[0]) + lane_atom + uint32_t(warp) * 1024u + uint32_t(u) * 128u +
               ((lane_chunk ^ uint32_t(u)) << 4) + lane_byte;
    auto sts64 = [](uint32_t addr, uint32_t lo, uint32_t hi, auto imm) {
      asm volatile("st.shared.v2.b32 [%0+%3], {%1, %2};" ::"r"(addr), "r"(lo), "r"(hi), "n"(decltype(imm)::value)
                   : "memory");
    };
    auto compute = [&](float a_reg, float rs_reg, int pix_c, int pix_n, auto stage) {
      constexpr int kS = decltype(stage)::value;
      constexpr int kHiOff = kS * kTileBytes;                          // S.ah[kS] - S.ah[0]
      constexpr int kLoOff = kStages * kTileBytes + kS * kTileBytes;   // S.al[kS] - S.ah[0]
      // The phases of kPhB rows are computed back to back before their pooled
      // rows are consumed: independent sin/cos chains for ILP, and the first
      // ring wait of the batch overlaps them.
      uint64_t snb[kPhB], csb[kPhB];
#pragma unroll
      for (int u = 0; u < kRows; ++u) {
        if (u % kPhB == 0) {
#pragma unroll
          for (int v = 0; v < kPhB; ++v) {
            const float aj = __shfl_sync(0xffffffffu, a_reg, u + v);
            const float rs = __shfl_sync(0xffffffffu, rs_reg, u + v);
            // conj(phase) * acc / cnt for channels (c0, c0+1), packed; the ÷count
            // (and fp16 pre-scale) rides on the sin/cos sign fix-up
            sincos2_k3_scaled<kMufu>(fmul2(f2pack(aj, aj), T01), f2pack(rs, rs), snb[v], csb[v]);
          }
        }
        const uint64_t sn = snb[u % kPhB], cs = csb[u % kPhB];
        asm volatile("cp.async.wait_group %0;" ::"n"(kQD - 2) : "memory");
        const float4 src_u = ring[(u & (kQD - 1)) * 32];
        {   // refill the slot read one row ago with the row kQD-1 ahead
          const int un = u + kQD - 1;
          const int pj = un < kRows ? __shfl_sync(0xffffffffu, pix_c, un) : __shfl_sync(0xffffffffu, pix_n, un - kRows);
          issue_row(pj, un & (kQD - 1));
        }
        const uint64_t ar = f2pack(src_u.x, src_u.y), ai = f2pack(src_u.z, src_u.w);   // packed pairs
        const uint64_t re = ffma2(sn, ai, fmul2(cs, ar));
        const uint64_t im = fsub2(fmul2(cs, ai), fmul2(sn, ar));
        // Feature order on the K axis is (Re c, Re c+1, Im c, Im c+1) per
        // channel pair (W1's columns are permuted to match on the host), so a
        // lane's four values are 8 contiguous bytes: one 64-bit store per image.
        float re0, re1, im0, im1;
        f2unpack(re, re0, re1);
        f2unpack(im, im0, im1);
        if (kSplit) {
          // hi = the value truncated to fp16's 11 significant bits (clearing
          // 13 mantissa bits: ALU LOP3s instead of fp16->f32 conversions on
          // the FMA pipe); exact in fp16 for |x| >= 2^-14, and below that its
          // rounding is < 2^-25 absolute.  lo = x - hi is exact in f32.
          const uint64_t tmask = 0xFFFFE000FFFFE000ull;
          const uint64_t tre = re & tmask, tim = im & tmask;
          float h0, h1, h2, h3, l0, l1, l2, l3;
          f2unpack(tre, h0, h1);
          f2unpack(tim, h2, h3);
          f2unpack(fsub2(re, tre), l0, l1);
          f2unpack(fsub2(im, tim), l2, l3);
          const __half2 hre = __floats2half2_rn(h0, h1), him = __floats2half2_rn(h2, h3);
          const __half2 lre = __floats2half2_rn(l0, l1), lim = __floats2half2_rn(l2, l3);
          sts64(sah[u], *reinterpret_cast<const uint32_t*>(&hre), *reinterpret_cast<const uint32_t*>(&him),
                std::integral_constant<int, kHiOff>{});
          sts64(sah[u], *reinterpret_cast<const uint32_t*>(&lre), *reinterpret_cast<const uint32_t*>(&lim),
                std::integral_constant<int, kLoOff>{});
        } else {
          const __nv_bfloat162 bre = __floats2bfloat162_rn(re0, re1), bim = __floats2bfloat162_rn(im0, im1);
          sts64(sah[u], *reinterpret_cast<const uint32_t*>(&bre), *reinterpret_cast<const uint32_t*>(&bim),
                std::integral_constant<int, kHiOff>{});
        }
      }
    };

    const int64_t G = gridDim.x;
    float a_c, a_n, a_nn, rs_c;
    int pix_c, pix_n, pix_nn, cnt_n;
    load_slot(blockIdx.x, a_c, pix_c);
    load_slot(int64_t(blockIdx.x) + G, a_n, pix_n);
    load_slot(int64_t(blockIdx.x) + 2 * G, a_nn, pix_nn);
    rs_c = recip(load_cnt(pix_c));
    cnt_n = load_cnt(pix_n);
#ifndef VKM_K3_PF
#define VKM_K3_PF 2   // tiles ahead whose pooled rows are bulk-prefetched into L2
#endif
    for (int d = 0; d < VKM_K3_PF; ++d) prefetch_l2(int64_t(blockIdx.x) + d * G);
#pragma unroll
    for (int u = 0; u < kQD - 1; ++u) issue_row(__shfl_sync(0xffffffffu, pix_c, u), u);
    // one tile on stage kS (compile-time: the tile loop is unrolled by the
    // two stages, it & 1 == kS)
    auto tile_step = [&](int64_t tile, int it, auto stage) {
      constexpr int kS = decltype(stage)::value;
      const uint32_t ph = (it >> 1) & 1;
      prefetch_l2(tile + VKM_K3_PF * G);
      mbar_wait(&S.empty[kS], ph ^ 1);
      compute(a_c, rs_c, pix_c, pix_n, stage);
      fence_proxy_async();
      mbar_arrive(&S.full[kS]);
      a_c = a_n;
      pix_c = pix_n;
      rs_c = recip(cnt_n);
      a_n = a_nn;
      pix_n = pix_nn;
      cnt_n = load_cnt(pix_nn);
      load_slot(tile + 3 * G, a_nn, pix_nn);
    };
    static_assert(kStages == 2, "the producer loop is unrolled by the two stages");
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += 2 * G, it += 2) {
      tile_step(tile, it, std::integral_constant<int, 0>{});
      if (tile + G >= ntiles) break;
      tile_step(tile + G, it + 1, std::integral_constant<int, 1>{});
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp < kProdWarps + 4) {
    // ======================= epilogue =======================
    const int q = warp & 3;   // TMEM lane quadrant = warp id % 4
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & (kAcc - 1);
      const uint32_t ph = (it / kAcc) & 1;
      const int64_t slot = tile * kM + q * 32 + lane;
      int cnt = 1;
      int64_t e = -1;
      if (slot < nv) {
        e = slot_event(__ldg(val_s + slot));
        cnt = __ldg(NQ + __ldg(pix_s + slot));
      }
      mbar_wait(&S.tfull[acc], ph);
      tc_fence_after();
      uint64_t oa = 0, ob = 0;   // (even, odd) hidden partial sums of the two outputs
      const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * kN);
#pragma unroll
      for (int cb = 0; cb < kN; cb += 32) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr + cb));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; i += 4) {   // 4 hidden units: 3 LDS.128, 2 FADD2, 4 FMNMX, 4 FFMA2
          const float4 bb = *reinterpret_cast<const float4*>(S.b1s + cb + i);
          const float4 wa = *reinterpret_cast<const float4*>(S.w2a + cb + i);
          const float4 wb = *reinterpret_cast<const float4*>(S.w2b + cb + i);
          float h0, h1, h2, h3;
          f2unpack(fadd2(f2pack(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), f2pack(bb.x, bb.y)), h0, h1);
          f2unpack(fadd2(f2pack(__uint_as_float(r[i + 2]), __uint_as_float(r[i + 3])), f2pack(bb.z, bb.w)), h2, h3);
          const uint64_t h01 = f2pack(fmaxf(h0, 0.f), fmaxf(h1, 0.f)), h23 = f2pack(fmaxf(h2, 0.f), fmaxf(h3, 0.f));
          oa = ffma2(h01, f2pack(wa.x, wa.y), oa);
          oa = ffma2(h23, f2pack(wa.z, wa.w), oa);
          ob = ffma2(h01, f2pack(wb.x, wb.y), ob);
          ob = ffma2(h23, f2pack(wb.z, wb.w), ob);
        }
      }
      tc_fence_before();
      mbar_arrive(&S.tempty[acc]);
      float oa0, oa1, ob0, ob1;
      f2unpack(oa, oa0, oa1);
      f2unpack(ob, ob0, ob1);
      const float o0 = oa0 + oa1, o1 = ob0 + ob1;
      if (e >= 0) {
        float2 r2 = make_float2(o0 + S.b2[0], o1 + S.b2[1]);
        if (cnt <= 0) r2 = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
        reinterpret_cast<float2*>(flows)[e] = r2;
        if (counts_out) counts_out[e] = cnt;
      }
    }
  } else {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(kSplit ? 0u : 1u);
      const uint32_t bh = smem_u32(S.bh), bl = smem_u32(S.bl);
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it & 1, acc = it & (kAcc - 1);
        const uint32_t ph = (it >> 1) & 1, pha = (it / kAcc) & 1;
        mbar_wait(&S.tempty[acc], pha ^ 1);
        mbar_wait(&S.full[s], ph);
        tc_fence_after();
        const uint32_t d = tmem + uint32_t(acc * kN);
        const uint32_t ah = smem_u32(S.ah[s]), al = smem_u32(S.al[s]);
#pragma unroll
        for (int ks = 0; ks < kK / 16; ++ks) {
          const uint32_t off = (ks >> 2) * kAtomBytes + (ks & 3) * 32;
          umma_f16(d, umma_desc(ah + off), umma_desc(bh + off), idesc, ks > 0);
          if (kSplit) {
            umma_f16(d, umma_desc(ah + off), umma_desc(bl + off), idesc, 1);
            umma_f16(d, umma_desc(al + off), umma_desc(bh + off), idesc, 1);
          }
        }
        umma_commit(&S.empty[s]);
        umma_commit(&S.tfull[acc]);
      }
    }
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kProdWarps + 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace tc

int feature_kpos(int f) {   // [Re(0..63) | Im(0..63)] -> per channel pair (Re c, Re c+1, Im c, Im c+1)
  const int c = f & 63, im = f >> 6;
  return 4 * (c >> 1) + 2 * im + (c & 1);
}

void build_umma_image_kmajor_128x128(const uint16_t* rowmajor, uint16_t* image) {
  for (uint32_t m = 0; m < 128; ++m)
    for (uint32_t k = 0; k < 128; ++k) image[tc::umma_off(m, k) / 2] = rowmajor[m * 128 + k];
}

void launch_gather_mlp_tc(int64_t n, const DevTables& tb, int W, int H, const GridBufs& g, const SortBufs& sb,
                          const TcWeights& w, int mode, float* flows, int32_t* counts_out, int num_sms,
                          cudaStream_t s) {
  if (n <= 0) return;
  const int64_t tiles = (n + tc::kM - 1) / tc::kM;
  const int grid = int(tiles < num_sms ? tiles : num_sms);
  const size_t smem = sizeof(tc::Smem) + 1024;
  const int64_t P = int64_t(W) * H;
  const int* nvalid = sb.start + P;
  static const int prefetch = [] {
    const char* e = std::getenv("VKM_TC_PREFETCH");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  const bool mufu = sincos_mufu();
  auto kern = mode == VKM_MLP_BF16 ? (mufu ? tc::k_gather_mlp_tc<VKM_MLP_BF16, true> : tc::k_gather_mlp_tc<VKM_MLP_BF16, false>)
                                   : (mufu ? tc::k_gather_mlp_tc<VKM_MLP_F16X3, true> : tc::k_gather_mlp_tc<VKM_MLP_F16X3, false>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  launch_pdl(kern, grid, tc::kThreads, smem, s, n, static_cast<const uint64_t*>(sb.val_s),
             static_cast<const int32_t*>(sb.pix_s), nvalid, tb.tf, P, static_cast<const float2*>(g.Q),
             static_cast<const int*>(g.NQ), static_cast<const uint4*>(w.w1_hi), static_cast<const uint4*>(w.w1_lo), w.b1,
             w.w2, w.b2, w.w_scale, flows, counts_out, prefetch);
}

}  // namespace vkm
