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
#include <cstring>
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
constexpr int kAcc = 4;                // TMEM accumulators (4 x 128 columns = all 512), row-per-warp producers
// one-event-per-lane producers keep the A operand in TMEM: 2 accumulators
// (columns 0..255) and 2 stages of A (hi | lo, 128 columns each) from kLeA
#ifndef VKM_K3_LE_ACC
#define VKM_K3_LE_ACC 2   // accumulators; stages of A fill the rest of the 512 columns
#endif
constexpr int kAccLE = VKM_K3_LE_ACC;
constexpr int kLeA = kAccLE * 128;
constexpr int kStagesLE = (512 - kLeA) / 128;
static_assert(kStagesLE >= 2 && kStagesLE <= 3, "lane-event TMEM layout");
constexpr int kTileBytes = kM * kK * 2;        // 32 KB per fp16 operand image
constexpr int kAtomBytes = kM * 128;           // one 64-wide K atom: 128 rows x 128 B
constexpr int kProdWarps = 16;                // producer warps (8 tile rows each)
constexpr int kThreads = (kProdWarps + 5) * 32; // + 4 epilogue warps + 1 MMA warp
// One-event-per-lane producers: 16 warps (four per TMEM lane quarter, 8
// channel pairs each), then 4 epilogue warps, the MMA warp and the gather
// (TMA) warp: 22 warps (1024 threads per CTA cap the producers at 16 for an
// even split of the 32 channel pairs).
#ifndef VKM_K3_LEPROD
#define VKM_K3_LEPROD 16   // 8 measured 1.4x slower (cfg2 K3 0.181 vs 0.127 ms): the producers need the warps
#endif
constexpr int kLEProd = VKM_K3_LEPROD;
constexpr int kLEPairs = 32 * 4 / kLEProd;       // channel pairs per producer lane
#ifndef VKM_K3_EPIW
#define VKM_K3_EPIW 4   // epilogue warps of the lane-event variant: 4, or 8 (two per TMEM lane quarter, half the
                        // hidden units each: 72 registers with spills, K3 +18 % at cfg 5 - not used)
#endif
constexpr int kEpiLE = VKM_K3_EPIW;
static_assert(kEpiLE == 4 || kEpiLE == 8, "epilogue warps");
constexpr int kThreadsLE = (kLEProd + kEpiLE + 2) * 32;
template <bool kLaneEvent>
struct Roles {
  static constexpr int prod = kLaneEvent ? kLEProd : kProdWarps;
  static constexpr int epi = kLaneEvent ? kEpiLE : 4;
  static constexpr int epi0 = prod;                // epilogue warps
  static constexpr int mma = prod + epi;
  static constexpr int loader = prod + epi + 1;    // lane-event variant only
  static constexpr int threads = kLaneEvent ? kThreadsLE : kThreads;
};
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
#ifdef VKM_K3_REGQ
  float4 qring[kProdWarps][1][32];     // unused: the rows live in registers
#else
  float4 qring[kProdWarps][kQD][32];   // per producer warp: pooled rows of its next kQD-1 events
#endif
  // head constants with the power-of-two operand scale s = w_scale·f_scale
  // folded in: relu(acc/s + b1)·w2 == relu(acc + s·b1)·(w2/s) exactly
  float b1s[kN];    // -s·b1 (relu(h + b1) = max(h, -b1) + b1; the + b1 part is folded into b2)
  float w2a[kN];    // w2[0][n] / s
  float w2b[kN];    // w2[1][n] / s
  float b2[2];
  float scale;
  uint32_t tmem_base;
  unsigned long long full[3], empty[3], tfull[kAcc], tempty[kAcc];
  // one-event-per-lane variant: pooled-grid rows of a tile's pixel range,
  // bulk-copied (TMA) into slots carved from the (then unused) A images + ring
  int gp0[4];                                   // first pixel of the slot's range, -1: load directly
  unsigned long long tpair[32];                 // (f32 T_c, f32 T_c+1) of each channel pair, packed
  unsigned long long gfull[4], gempty[4];
};
#ifndef VKM_K3_GSLOTS
#define VKM_K3_GSLOTS 3
#endif
constexpr int kGSlots = VKM_K3_GSLOTS;
#ifndef VKM_K3_LDSPLIT   // 1: the producers load the second half of their pooled rows mid-tile
#define VKM_K3_LDSPLIT 1
#endif
#ifndef VKM_K3_EPI_PIPE   // 1: double-buffered 16-column TMEM loads in the epilogue
#define VKM_K3_EPI_PIPE 1
#endif
#ifndef VKM_K3_LDAHEAD   // L > 0 (with LDSPLIT): pair u+L's row is loaded when pair u's math starts
#define VKM_K3_LDAHEAD 0
#endif
constexpr int kGSpan = kGSlots == 3 ? 96 : 80;    // pixels per plane a slot holds
constexpr int kGSlotBytes = 8 * kGSpan * 64;      // 48 KB (40 KB for 4 slots)
static_assert(kGSlots * kGSlotBytes <= int(2 * kStages * kTileBytes + sizeof(float4) * kProdWarps * kQD * 32),
              "gather slots exceed the A images + ring");
static_assert(kEpiLE == 4 ||
                  kGSlots * kGSlotBytes + 2 * kM * 8 <= int(2 * kStages * kTileBytes + sizeof(float4) * kProdWarps * kQD * 32),
              "gather slots + epilogue hand-over exceed the A images + ring");

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
#ifndef VKM_K3_HINT
#define VKM_K3_HINT 20000   // try_wait suspend-time hint (ns); 0 = plain try_wait
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
#if VKM_K3_HINT > 0
    // suspend-time hint: a waiting warp sleeps in the barrier unit instead of
    // spinning on issue slots the producers need
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(uint32_t(VKM_K3_HINT))
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
#endif
    if (done) return;
    if (it > (1u << 24)) __trap();
  }
}

#ifdef VKM_K3_WAITPROF   // A/B instrumentation: cycles spent in each kind of barrier wait, per role
__device__ unsigned long long g_k3_wait[8];
#define K3_TIMED_WAIT(slot, call)                                  \
  do {                                                             \
    const long long t0_ = clock64();                               \
    call;                                                          \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_k3_wait[slot], (unsigned long long)(clock64() - t0_)); \
  } while (0)
#else
#define K3_TIMED_WAIT(slot, call) call
#endif

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
// A operand from tensor memory (row m = TMEM lane m, K packed two fp16 per column)
__device__ __forceinline__ void umma_f16_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// global -> shared bulk copy (TMA engine), completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
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

template <int MODE, bool kMufu, bool kLaneEvent>  // VKM_MLP_F16X3 or VKM_MLP_BF16; sin/cos flavour; producer layout
__global__ void __launch_bounds__(Roles<kLaneEvent>::threads, 1)
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
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
      dh[i] = __ldg(w1h + i);
      if (kSplit) dl[i] = __ldg(w1l + i);
    }
    const float sc = w_scale * f_scale;   // a power of two: exact scaling
    for (int i = threadIdx.x; i < 32; i += blockDim.x) S.tpair[i] = f2pack(__ldg(tf + 2 * i), __ldg(tf + 2 * i + 1));
    for (int i = threadIdx.x; i < kN; i += blockDim.x) {
      S.b1s[i] = -b1[i] * sc;
      S.w2a[i] = w2[i] / sc;
      S.w2b[i] = w2[kN + i] / sc;
    }
    if (warp == 0) {
      // W2·relu(h + b1) + b2 = W2·max(h, -b1) + (b2 + W2·b1): the epilogue
      // skips the bias add (two FADD2 per four hidden units); the dot
      // products in f64, spread over the warp
      double c0 = 0.0, c1 = 0.0;
      for (int i = lane; i < kN; i += 32) {
        c0 += double(w2[i]) * double(b1[i]);
        c1 += double(w2[kN + i]) * double(b1[i]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      }
      if (lane == 0) {
        S.b2[0] = float(double(b2[0]) + c0);
        S.b2[1] = float(double(b2[1]) + c1);
      }
    }
    if (threadIdx.x == 0) {
      S.scale = 1.f / (w_scale * f_scale);
      for (int s = 0; s < 3; ++s) {
        mbar_init(&S.full[s], Roles<kLaneEvent>::prod * 32);
        mbar_init(&S.empty[s], 1);
      }
      for (int a = 0; a < kAcc; ++a) {
        mbar_init(&S.tfull[a], 1);
        mbar_init(&S.tempty[a], 32 * Roles<kLaneEvent>::epi);
      }
      for (int g = 0; g < kGSlots; ++g) {
        mbar_init(&S.gfull[g], 1);
        mbar_init(&S.gempty[g], Roles<kLaneEvent>::prod);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == Roles<kLaneEvent>::mma) {
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

  if (kLaneEvent && warp < kLEProd) {
    // ================ producers, one event per lane ================
    // Warp (q, j) = (warp & 3, warp >> 2) fills tile rows 32q + lane (one event
    // per lane) with channel pairs 8j .. 8j+7 (K positions 32j .. 32j+31 of the
    // feature order of feature_kpos, i.e. four 16-byte chunks of the
    // SWIZZLE_128B image per lane: 8 lanes of a row group hit 8 distinct
    // chunk columns, so the 16-byte stores are conflict-free).  Each lane
    // gathers its own pooled row (two 64-byte pieces, planes 2j and 2j+1),
    // de-phases by its own event's phase, divides by the count and splits -
    // no shuffles and no per-row shared-memory ring: the pooled rows of the
    // next tile are loaded into the registers freed by the current tile's
    // first pairs, so a tile of gathers stays in flight across the stage wait.
    const int qq = warp & 3, jg = warp >> 2;      // lane quarter, channel-pair group
    const int m = 32 * qq + lane;                 // tile row of this lane's event
    uint64_t T01[kLEPairs];
#pragma unroll
    for (int u = 0; u < kLEPairs; ++u) {
      const int c = 2 * (kLEPairs * jg + u);
      T01[u] = f2pack(__ldg(tf + c), __ldg(tf + c + 1));
    }
    const float4* Q4 = reinterpret_cast<const float4*>(Q);
    // The A operand lives in tensor memory: row m = TMEM lane m (this warp's
    // lane quarter is qq = warp % 4, as tcgen05.st requires), K packed two
    // fp16 per 32-bit column; pairs 8jg.. are K 32jg.. = columns 16jg..16jg+15
    // of the stage's hi and lo regions (columns kLeA + 128 s + {0, 64}).
    const uint32_t ta_lane = tmem + (uint32_t(32 * qq) << 16) + uint32_t(kLeA + 2 * kLEPairs * jg);
    auto meta = [&](int64_t tl, float& a, int& pix) {
      const int64_t slot = tl * kM + m;
      a = 0.f;
      pix = -1;
      if (tl < ntiles && slot < nv) {
        pix = __ldg(pix_s + slot);
        a = slot_arg(__ldg(val_s + slot));
      }
    };
    auto recip = [&](int cnt) {
      float r;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(float(cnt)));
      return cnt > 0 ? r * f_scale : 0.f;
    };
    // pooled row of pixel pix, pairs u of the group: plane 2jg + (u >> 2),
    // q4 = u & 3; from the tile's bulk-copied slot (gp0 >= 0: pixel range
    // [gp0, gp0 + kGSpan)) or, for tiles whose pixel range does not fit a
    // slot, straight from global memory
    const uint32_t gslots = smem_u32(S.ah[0]);
    auto gather = [&](int pix, int u, int gp0, uint32_t slot_base) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (pix >= 0) {
        if (gp0 >= 0) {
          const uint32_t a = slot_base + uint32_t((((kLEPairs / 4) * jg + (u >> 2)) * kGSpan + (pix - gp0)) * 64 +
                                                  ((u & 3) ^ qswz(pix)) * 16);
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
        } else {
          const float4* src = Q4 + ((int64_t((kLEPairs / 4) * jg + (u >> 2)) * P + pix) << 2) + ((u & 3) ^ qswz(pix));
          asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "l"(src));
        }
      }
      return v;
    };
    const int64_t G = gridDim.x;
    float a_c, a_n, a_nn;
    int pix_c, pix_n, pix_nn, cnt_n;
    meta(blockIdx.x, a_c, pix_c);
    meta(int64_t(blockIdx.x) + G, a_n, pix_n);
    meta(int64_t(blockIdx.x) + 2 * G, a_nn, pix_nn);
    float rs_c = recip(pix_c >= 0 ? __ldg(NQ + pix_c) : 0);
    cnt_n = pix_n >= 0 ? __ldg(NQ + pix_n) : 0;
    int gslot = 0, gph = 0;   // gather slot of the current tile and its phase
    auto tile_step = [&](int64_t tile, int it) {
      const int kS = it % kStagesLE;                 // A stage in TMEM
      const uint32_t ph = (it / kStagesLE) & 1;
      const uint64_t rs2 = f2pack(rs_c, rs_c);
      const uint64_t aa = f2pack(a_c, a_c);
      K3_TIMED_WAIT(0, mbar_wait(&S.gfull[gslot], gph));   // this tile's pooled rows have landed (or gp0 = -1)
      const int gp0 = S.gp0[gslot];
      const uint32_t slot_base = gslots + uint32_t(gslot * kGSlotBytes);
#ifndef VKM_K3_LATE
      float4 v[kLEPairs];
#ifndef VKM_K3_GATHER_PER_PAIR
      // warp-uniform gp0 >= 0: one base address, the pieces at fixed offsets.
      // Rows past the slice's events (pix -1) read pixel gp0: their outputs
      // are never stored and MMA rows do not mix.
      const bool blk = gp0 >= 0;
      const uint32_t gbase =
          slot_base + uint32_t(((kLEPairs / 4) * jg * kGSpan + (pix_c > gp0 ? pix_c - gp0 : 0)) * 64);
      const int gsw = qswz(pix_c > 0 ? pix_c : 0);   // chunk slot swizzle of this lane's pixel
      auto ld_half = [&](int half) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int u = 4 * half + h;
          const uint32_t a = gbase + uint32_t((u >> 2) * kGSpan * 64 + ((u & 3) ^ gsw) * 16);
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "r"(a));
        }
      };
      auto ld_one = [&](int u) {
        const uint32_t a = gbase + uint32_t((u >> 2) * kGSpan * 64 + ((u & 3) ^ gsw) * 16);
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "r"(a));
      };
      if (blk) {
#if VKM_K3_LDAHEAD
#pragma unroll
        for (int u = 0; u < VKM_K3_LDAHEAD; ++u) ld_one(u);
#else
        ld_half(0);
#endif
#if VKM_K3_LDSPLIT == 0
#pragma unroll
        for (int half = 1; half < kLEPairs / 4; ++half) ld_half(half);
#endif
      } else {
#pragma unroll
        for (int u = 0; u < kLEPairs; ++u) v[u] = gather(pix_c, u, -1, slot_base);
      }
#if VKM_K3_LDSPLIT == 0
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.gempty[gslot]);   // reads are done (registers hold the rows)
      if (++gslot == kGSlots) {
        gslot = 0;
        gph ^= 1;
      }
#endif
#else
#pragma unroll
      for (int u = 0; u < kLEPairs; ++u) v[u] = gather(pix_c, u, gp0, slot_base);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.gempty[gslot]);   // reads are done (registers hold the rows)
      if (++gslot == kGSlots) {
        gslot = 0;
        gph ^= 1;
      }
#endif
#endif
#pragma unroll
      for (int half = 0; half < kLEPairs / 4; ++half) {   // pairs 4·half .. 4·half+3 -> 8 columns per image
        uint32_t hw[8], lw[8];
#if !defined(VKM_K3_LATE) && !defined(VKM_K3_GATHER_PER_PAIR) && VKM_K3_LDSPLIT && !VKM_K3_LDAHEAD
        if (VKM_K3_LDSPLIT == 1 && half > 0 && blk) ld_half(half);   // the second half's rows load under the first half's math
        if (VKM_K3_LDSPLIT == 1 && half == kLEPairs / 4 - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.gempty[gslot]);   // reads issued (release orders them before the TMA refill)
          if (++gslot == kGSlots) {
            gslot = 0;
            gph ^= 1;
          }
        }
#endif
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int u = 4 * half + h;
          uint64_t sn, cs;
#if !defined(VKM_K3_LATE) && !defined(VKM_K3_GATHER_PER_PAIR) && VKM_K3_LDSPLIT && VKM_K3_LDAHEAD
          if (u + VKM_K3_LDAHEAD < kLEPairs) {   // pair u+L's row loads under pair u's math
            if (blk) ld_one(u + VKM_K3_LDAHEAD);
            if (u + VKM_K3_LDAHEAD == kLEPairs - 1) {
              __syncwarp();
              if (lane == 0) mbar_arrive(&S.gempty[gslot]);
              if (++gslot == kGSlots) {
                gslot = 0;
                gph ^= 1;
              }
            }
          }
#endif
#ifdef VKM_K3_LATE   // rows and frequencies read at their use: fewer live registers, more chains in flight
          const uint64_t Tu = S.tpair[kLEPairs * jg + u];
          const float4 q = gather(pix_c, u, gp0, slot_base);
          sincos2_k3_scaled<kMufu>(fmul2(aa, Tu), rs2, sn, cs);
#else
          sincos2_k3_scaled<kMufu>(fmul2(aa, T01[u]), rs2, sn, cs);
          const float4 q = v[u];
#endif
          const uint64_t ar = f2pack(q.x, q.y), ai = f2pack(q.z, q.w);
          const uint64_t re = ffma2(sn, ai, fmul2(cs, ar));
          const uint64_t im = fsub2(fmul2(cs, ai), fmul2(sn, ar));
          if (kSplit) {
            const uint64_t tmask = 0xFFFFE000FFFFE000ull;
            const uint64_t tre = re & tmask, tim = im & tmask;
            float h0, h1, h2, h3, l0, l1, l2, l3;
            f2unpack(tre, h0, h1);
            f2unpack(tim, h2, h3);
            f2unpack(fsub2(re, tre), l0, l1);
            f2unpack(fsub2(im, tim), l2, l3);
            const __half2 hre = __floats2half2_rn(h0, h1), him = __floats2half2_rn(h2, h3);
            const __half2 lre = __floats2half2_rn(l0, l1), lim = __floats2half2_rn(l2, l3);
            hw[2 * h] = *reinterpret_cast<const uint32_t*>(&hre);
            hw[2 * h + 1] = *reinterpret_cast<const uint32_t*>(&him);
            lw[2 * h] = *reinterpret_cast<const uint32_t*>(&lre);
            lw[2 * h + 1] = *reinterpret_cast<const uint32_t*>(&lim);
          } else {
            float re0, re1, im0, im1;
            f2unpack(re, re0, re1);
            f2unpack(im, im0, im1);
            const __nv_bfloat162 bre = __floats2bfloat162_rn(re0, re1), bim = __floats2bfloat162_rn(im0, im1);
            hw[2 * h] = *reinterpret_cast<const uint32_t*>(&bre);
            hw[2 * h + 1] = *reinterpret_cast<const uint32_t*>(&bim);
          }
        }
#if !defined(VKM_K3_LATE) && !defined(VKM_K3_GATHER_PER_PAIR) && VKM_K3_LDSPLIT == 2 && !VKM_K3_LDAHEAD
        if (half == 0) {   // the second half's rows load before the stage wait (in flight across it)
          if (blk) ld_half(1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.gempty[gslot]);
          if (++gslot == kGSlots) {
            gslot = 0;
            gph ^= 1;
          }
        }
#endif
        if (half == 0) {   // the stage is needed only from the first store on
          K3_TIMED_WAIT(1, mbar_wait(&S.empty[kS], ph ^ 1));
          tc_fence_after();
        }
        const uint32_t ta = ta_lane + uint32_t(kS * 128 + 8 * half);
        tmem_st8(ta, hw);
        if (kSplit) tmem_st8(ta + 64, lw);
      }
#ifdef VKM_K3_LATE
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.gempty[gslot]);   // this warp's slot reads are done
      if (++gslot == kGSlots) {
        gslot = 0;
        gph ^= 1;
      }
#endif
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&S.full[kS]);
      a_c = a_n;
      pix_c = pix_n;
      rs_c = recip(cnt_n);
      a_n = a_nn;
      pix_n = pix_nn;
      cnt_n = pix_nn >= 0 ? __ldg(NQ + pix_nn) : 0;
      meta(tile + 3 * G, a_nn, pix_nn);
    };
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++it) tile_step(tile, it);
  } else if (!kLaneEvent && warp < kProdWarps) {
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
#ifdef VKM_K3_REGQ
    // pooled rows prefetched into registers (kQD - 1 rows ahead) instead of
    // the shared-memory ring: no cp.async writes / LDS reads of shared memory
    float4 rq[kQD];
#pragma unroll
    for (int i = 0; i < kQD; ++i) rq[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#endif
    // lane-constant parts of the gather (global plane base, shared ring slot 0)
    // hoisted: per row only the pixel offset and the slot offset are added
    const float4* const qlane = Q4 + ((int64_t(plane) * P) << 2) + q4;
    const uint32_t ring_s = smem_u32(ring);
    auto issue_row = [&](int pj, int slot) {
#ifdef VKM_K3_NOGATHER   // A/B skeleton: no pooled-row gathers (the ring keeps stale rows)
      return;
#endif
#ifdef VKM_K3_REGQ
      {
        const int pjc = pj >= 0 ? pj : 0;
        const float4* src = qlane + (int64_t(pjc) << 2) + ((q4 ^ qswz(pjc)) - q4);
        float4 v;
        asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(src));
        rq[slot] = pj >= 0 ? v : make_float4(0.f, 0.f, 0.f, 0.f);
        return;
      }
#endif
      const int pjc = pj >= 0 ? pj : 0;
      const float4* src = qlane + (int64_t(pjc) << 2) + ((q4 ^ qswz(pjc)) - q4);
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
#ifdef VKM_K3_NOMATH   // A/B skeleton: no de-phase sin/cos
            snb[v] = f2pack(aj, rs);
            csb[v] = f2pack(rs, aj);
#else
            sincos2_k3_scaled<kMufu>(fmul2(f2pack(aj, aj), T01), f2pack(rs, rs), snb[v], csb[v]);
#endif
          }
        }
        const uint64_t sn = snb[u % kPhB], cs = csb[u % kPhB];
#ifdef VKM_K3_REGQ
        const float4 src_u = rq[u & (kQD - 1)];
#else
        asm volatile("cp.async.wait_group %0;" ::"n"(kQD - 2) : "memory");
        const float4 src_u = ring[(u & (kQD - 1)) * 32];
#endif
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
#ifndef VKM_K3_NOWAIT   // A/B skeleton: producers do not wait for the MMA to free the stage (racy)
      mbar_wait(&S.empty[kS], ph ^ 1);
#endif
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
  } else if (kLaneEvent && warp == Roles<kLaneEvent>::loader) {
    // ================ gather loader (TMA) ================
    // Slots are pixel-sorted, so a tile's pooled rows are one contiguous
    // pixel range per channel plane: eight bulk copies (one per plane) move
    // them into a shared-memory slot, three tiles ahead of the producers.
    if (lane == 0) {
      // the pixel range of the next tile is loaded while this one waits for
      // its slot, so the global-load latency is off the loader's chain
      auto range = [&](int64_t tl, int& a, int& b) {
        a = b = -1;
        const int64_t f = tl * kM;
        if (tl < ntiles && f < nv) {
          const int64_t l = (f + kM < nv ? f + kM : nv) - 1;
          a = __ldg(pix_s + f);
          b = __ldg(pix_s + l);
        }
      };
      int pa, pb;
      range(blockIdx.x, pa, pb);
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int g = it % kGSlots;
        const uint32_t ph = (it / kGSlots) & 1;
        int na, nb;
        range(tile + gridDim.x, na, nb);
        K3_TIMED_WAIT(2, mbar_wait(&S.gempty[g], ph ^ 1));
        int p0 = pa, span = pb - pa + 1;
        if (pa < 0 || span > kGSpan) p0 = -1;
        pa = na;
        pb = nb;
        S.gp0[g] = p0;
        if (p0 >= 0) {
          const uint32_t bytes = uint32_t(span) * 64u;
          mbar_expect_tx(&S.gfull[g], 8u * bytes);
          const uint32_t dst = smem_u32(S.ah[0]) + uint32_t(g * kGSlotBytes);
#pragma unroll
          for (int pl = 0; pl < 8; ++pl)
            bulk_g2s(dst + uint32_t(pl * kGSpan * 64), Q + (int64_t(pl) * P + p0) * 8, bytes, &S.gfull[g]);
        } else {
          mbar_arrive(&S.gfull[g]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= Roles<kLaneEvent>::epi0 && warp < Roles<kLaneEvent>::epi0 + Roles<kLaneEvent>::epi) {
    // ======================= epilogue =======================
    const int q = warp & 3;   // TMEM lane quadrant = warp id % 4
    // 8 epilogue warps: warps q and q + 4 share lane quadrant q, each reducing
    // half of the hidden units; the upper half hands its partial outputs over
    // through shared memory (named barrier 1 + q per pair)
    constexpr int kEh = Roles<kLaneEvent>::epi / 4;
    static_assert(kEh == 1 || VKM_K3_EPI_PIPE, "8 epilogue warps need the pipelined epilogue");
    const int eh = kEh == 1 ? 0 : (warp - Roles<kLaneEvent>::epi0) >> 2;
    const int cbeg = eh * (kN / kEh);
    int it = 0;
    constexpr int kA = kLaneEvent ? kAccLE : kAcc;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & (kA - 1);
      const uint32_t ph = (it / kA) & 1;
      const int64_t slot = tile * kM + q * 32 + lane;
      int cnt = 1;
      int64_t e = -1;
      if (slot < nv && eh == 0) {
        e = slot_event(__ldg(val_s + slot));
        cnt = __ldg(NQ + __ldg(pix_s + slot));
      }
      K3_TIMED_WAIT(3, mbar_wait(&S.tfull[acc], ph));
      tc_fence_after();
      uint64_t oa = 0, ob = 0;   // (even, odd) hidden partial sums of the two outputs
      const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * kN);
#if VKM_K3_EPI_PIPE
      // 16-column chunks, double-buffered: the TMEM load of chunk c+1 is in
      // flight while chunk c is reduced, and the accumulator is released as
      // soon as its last chunk is in registers (before that chunk's math)
      auto ld16 = [&](uint32_t (&r)[16], int cb) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr + cb));
      };
      auto red16 = [&](const uint32_t (&r)[16], int cb) {
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const float4 nb = *reinterpret_cast<const float4*>(S.b1s + cb + i);
          const float4 wa = *reinterpret_cast<const float4*>(S.w2a + cb + i);
          const float4 wb = *reinterpret_cast<const float4*>(S.w2b + cb + i);
          const uint64_t h01 = f2pack(fmaxf(__uint_as_float(r[i]), nb.x), fmaxf(__uint_as_float(r[i + 1]), nb.y));
          const uint64_t h23 = f2pack(fmaxf(__uint_as_float(r[i + 2]), nb.z), fmaxf(__uint_as_float(r[i + 3]), nb.w));
          oa = ffma2(h01, f2pack(wa.x, wa.y), oa);
          oa = ffma2(h23, f2pack(wa.z, wa.w), oa);
          ob = ffma2(h01, f2pack(wb.x, wb.y), ob);
          ob = ffma2(h23, f2pack(wb.z, wb.w), ob);
        }
      };
      {
        uint32_t ra[16], rb[16];
        ld16(ra, cbeg);
#pragma unroll
        for (int c = 0; c < kN / kEh; c += 32) {
          const int cb = cbeg + c;
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          ld16(rb, cb + 16);
          red16(ra, cb);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 32 < kN / kEh) {
            ld16(ra, cb + 32);
          } else {
            tc_fence_before();
            mbar_arrive(&S.tempty[acc]);
          }
          red16(rb, cb + 16);
        }
      }
      if (false)
#endif
#ifdef VKM_K3_NOEPI   // A/B skeleton: no epilogue math
      if (false)
#endif
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
        for (int i = 0; i < 32; i += 4) {   // 4 hidden units: 3 LDS.128, 4 FMNMX, 4 FFMA2
          const float4 nb = *reinterpret_cast<const float4*>(S.b1s + cb + i);
          const float4 wa = *reinterpret_cast<const float4*>(S.w2a + cb + i);
          const float4 wb = *reinterpret_cast<const float4*>(S.w2b + cb + i);
          const uint64_t h01 = f2pack(fmaxf(__uint_as_float(r[i]), nb.x), fmaxf(__uint_as_float(r[i + 1]), nb.y));
          const uint64_t h23 = f2pack(fmaxf(__uint_as_float(r[i + 2]), nb.z), fmaxf(__uint_as_float(r[i + 3]), nb.w));
          oa = ffma2(h01, f2pack(wa.x, wa.y), oa);
          oa = ffma2(h23, f2pack(wa.z, wa.w), oa);
          ob = ffma2(h01, f2pack(wb.x, wb.y), ob);
          ob = ffma2(h23, f2pack(wb.z, wb.w), ob);
        }
      }
#if !VKM_K3_EPI_PIPE
      tc_fence_before();
      mbar_arrive(&S.tempty[acc]);
#endif
      float oa0, oa1, ob0, ob1;
      f2unpack(oa, oa0, oa1);
      f2unpack(ob, ob0, ob1);
      float o0 = oa0 + oa1, o1 = ob0 + ob1;
      if (kEh == 2) {
        // 2 x 128 float2 past the gather slots (the A-image region's unused tail)
        float2* part = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(S.ah[0]) + kGSlots * kGSlotBytes) +
                       (it & 1) * kM + q * 32 + lane;
        if (eh == 1) *part = make_float2(o0, o1);
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        if (eh == 1) continue;
        const float2 pu = *part;
        o0 += pu.x;
        o1 += pu.y;
      }
      if (e >= 0) {
        float2 r2 = make_float2(o0 + S.b2[0], o1 + S.b2[1]);
        if (cnt <= 0) r2 = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
        reinterpret_cast<float2*>(flows)[e] = r2;
        if (counts_out) counts_out[e] = cnt;
      }
    }
  } else if (warp == Roles<kLaneEvent>::mma) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc(kSplit ? 0u : 1u);
      const uint32_t bh = smem_u32(S.bh), bl = smem_u32(S.bl);
      int it = 0;
      constexpr int kA = kLaneEvent ? kAccLE : kAcc;
      constexpr int kSt = kLaneEvent ? kStagesLE : kStages;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % kSt, acc = it & (kA - 1);
        const uint32_t ph = (it / kSt) & 1, pha = (it / kA) & 1;
        K3_TIMED_WAIT(4, mbar_wait(&S.tempty[acc], pha ^ 1));
        K3_TIMED_WAIT(5, mbar_wait(&S.full[s], ph));
        tc_fence_after();
        const uint32_t d = tmem + uint32_t(acc * kN);
        if (kLaneEvent) {
          const uint32_t ta = tmem + uint32_t(kLeA + s * 128);   // A hi | lo of stage s (TMEM lane 0)
#pragma unroll
          for (int ks = 0; ks < kK / 16; ++ks) {
            const uint32_t off = (ks >> 2) * kAtomBytes + (ks & 3) * 32;
#ifdef VKM_K3_NOMMA
            continue;
#endif
            umma_f16_ta(d, ta + 8 * ks, umma_desc(bh + off), idesc, ks > 0);
            if (kSplit) {
              umma_f16_ta(d, ta + 8 * ks, umma_desc(bl + off), idesc, 1);
              umma_f16_ta(d, ta + 64 + 8 * ks, umma_desc(bh + off), idesc, 1);
            }
          }
        } else {
          const uint32_t ah = smem_u32(S.ah[s]), al = smem_u32(S.al[s]);
#pragma unroll
          for (int ks = 0; ks < kK / 16; ++ks) {
            const uint32_t off = (ks >> 2) * kAtomBytes + (ks & 3) * 32;
#ifdef VKM_K3_NOMMA   // A/B skeleton: no tensor-core work
            continue;
#endif
            umma_f16(d, umma_desc(ah + off), umma_desc(bh + off), idesc, ks > 0);
            if (kSplit) {
              umma_f16(d, umma_desc(ah + off), umma_desc(bl + off), idesc, 1);
              umma_f16(d, umma_desc(al + off), umma_desc(bh + off), idesc, 1);
            }
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
  if (warp == Roles<kLaneEvent>::mma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

}  // namespace tc

#ifdef VKM_K3_WAITPROF
}  // namespace vkm
extern "C" int vkm_debug_k3_waits(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, vkm::tc::g_k3_wait, sizeof(unsigned long long) * 8);
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(vkm::tc::g_k3_wait, z, sizeof(z));
  return 0;
}
namespace vkm {
#endif

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
  const bool rows = [] {   // VKM_K3=rows: the row-per-warp producers (A/B and tests; read per launch)
    const char* e = std::getenv("VKM_K3");
    return e && std::strcmp(e, "rows") == 0;
  }();
  using K = decltype(&tc::k_gather_mlp_tc<VKM_MLP_F16X3, true, true>);
  K kern;
  if (mode == VKM_MLP_BF16)
    kern = mufu ? (rows ? tc::k_gather_mlp_tc<VKM_MLP_BF16, true, false> : tc::k_gather_mlp_tc<VKM_MLP_BF16, true, true>)
                : (rows ? tc::k_gather_mlp_tc<VKM_MLP_BF16, false, false> : tc::k_gather_mlp_tc<VKM_MLP_BF16, false, true>);
  else
    kern = mufu ? (rows ? tc::k_gather_mlp_tc<VKM_MLP_F16X3, true, false> : tc::k_gather_mlp_tc<VKM_MLP_F16X3, true, true>)
                : (rows ? tc::k_gather_mlp_tc<VKM_MLP_F16X3, false, false> : tc::k_gather_mlp_tc<VKM_MLP_F16X3, false, true>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  launch_pdl(kern, grid, rows ? tc::kThreads : tc::kThreadsLE, smem, s, n, static_cast<const uint64_t*>(sb.val_s),
             static_cast<const int32_t*>(sb.pix_s), nvalid, tb.tf, P, static_cast<const float2*>(g.Q),
             static_cast<const int*>(g.NQ), static_cast<const uint4*>(w.w1_hi), static_cast<const uint4*>(w.w1_lo), w.b1,
             w.w2, w.b2, w.w_scale, flows, counts_out, prefetch);
}

}  // namespace vkm
