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
// Warp roles (416 threads, one persistent CTA per SM):
//   warps 0-7  producers: one warp per 16 tile rows; gather the pooled grid
//              row of each event (coalesced 512 B), de-phase, ÷count, split,
//              and store the fp16 A tile in the UMMA K-major SWIZZLE_128B layout
//   warps 8-11 epilogue: tcgen05.ld of the accumulator (warp q = id % 4 owns
//              TMEM lanes 32q..32q+31 = tile rows), bias + ReLU + 128->2, store
//   warp 12    TMEM allocator + single-thread tcgen05.mma issuer
// Pipelines: A stages (full/empty mbarriers, depth 2) and TMEM accumulators
// (tfull/tempty, depth 2), so gather(i+1), MMA(i) and epilogue(i-1) overlap.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "../../include/veckm.h"
#include "vkm_device.cuh"
#include "vkm_kernels.cuh"

namespace vkm {
namespace tc {

constexpr int kM = 128;             // events per tile (UMMA M)
constexpr int kN = 128;             // hidden units (UMMA N)
constexpr int kK = 128;             // features 2D (UMMA K total)
constexpr int kStages = 2;
constexpr int kAcc = 2;
constexpr int kTileBytes = kM * kK * 2;        // 32 KB per fp16 operand image
constexpr int kAtomBytes = kM * 128;           // one 64-wide K atom: 128 rows x 128 B
constexpr int kProdWarps = 8;                 // producer warps (16 tile rows each)
constexpr int kThreads = (kProdWarps + 5) * 32; // + 4 epilogue warps + 1 MMA warp
constexpr uint32_t kTmemCols = 256;

struct Smem {
  // operand images, each 1024-byte aligned (SWIZZLE_128B atoms)
  uint8_t bh[kTileBytes];
  uint8_t bl[kTileBytes];
  uint8_t ah[kStages][kTileBytes];
  uint8_t al[kStages][kTileBytes];
  float b1[kN];
  float w2[2 * kN];
  float b2[2];
  float scale;
  uint32_t tmem_base;
  unsigned long long full[kStages], empty[kStages], tfull[kAcc], tempty[kAcc];
};

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

template <int MODE>  // VKM_MLP_F16X3 or VKM_MLP_BF16
__global__ void __launch_bounds__(kThreads, 1)
    k_gather_mlp_tc(const double* __restrict__ ev, int64_t n, double t0_in, double delta_t,
                    const float* __restrict__ tf, int W, int64_t P, const float2* __restrict__ Q,
                    const int* __restrict__ NQ, const uint4* __restrict__ w1h, const uint4* __restrict__ w1l,
                    const float* __restrict__ b1, const float* __restrict__ w2, const float* __restrict__ b2,
                    float w_scale, float* __restrict__ flows, int32_t* __restrict__ counts_out) {
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool kSplit = (MODE == VKM_MLP_F16X3);
  const float f_scale = kSplit ? 256.f : 1.f;   // features |f| <= 1 -> keep lo parts normal

  // ---- one-time setup ----
  {
    const int nvec = kTileBytes / 16;
    uint4* dh = reinterpret_cast<uint4*>(S.bh);
    uint4* dl = reinterpret_cast<uint4*>(S.bl);
    for (int i = threadIdx.x; i < nvec; i += kThreads) {
      dh[i] = __ldg(w1h + i);
      if (kSplit) dl[i] = __ldg(w1l + i);
    }
    for (int i = threadIdx.x; i < kN; i += kThreads) {
      S.b1[i] = b1[i];
      S.w2[i] = w2[i];
      S.w2[kN + i] = w2[kN + i];
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
  const uint32_t tmem = S.tmem_base;
  const int64_t ntiles = (n + kM - 1) / kM;

  if (warp < kProdWarps) {
    // ======================= producers =======================
    // Warp w fills tile rows [16w, 16w+16).  Gathers are issued 8 events at a
    // time before any is consumed, so each lane keeps 8 x 16 B in flight.
    const double t0 = ld_t0(ev, t0_in);
    const int c0 = 2 * lane;                      // this lane's channel pair
    const float T0 = __ldg(tf + c0), T1 = __ldg(tf + c0 + 1);
    const float4* Q4 = reinterpret_cast<const float4*>(Q);
    const int plane = lane >> 2, q4 = lane & 3;
    constexpr int kRows = kM / kProdWarps;        // 16
    constexpr int kBatch = 8;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int s = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const int64_t e = tile * kM + warp * kRows + (lane & (kRows - 1));
      float a = 0.f;
      int pix = -1, cnt = 0;
      if (e < n) {
        const double t = __ldg(ev + 3 * e), x = __ldg(ev + 3 * e + 1), y = __ldg(ev + 3 * e + 2);
        pix = int(y) * W + int(x);
        a = time_arg(t, t0, delta_t);
        cnt = __ldg(NQ + pix);
      }
      mbar_wait(&S.empty[s], ph ^ 1);
      uint8_t* ah = S.ah[s];
      uint8_t* al = S.al[s];
#pragma unroll 1
      for (int jb = 0; jb < kRows; jb += kBatch) {
        float4 acc[kBatch];
        int pjs[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          pjs[u] = __shfl_sync(0xffffffffu, pix, jb + u);
          acc[u] = pjs[u] >= 0 ? __ldg(Q4 + ((int64_t(plane) * P + pjs[u]) << 2) + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const int j = jb + u;
          const float aj = __shfl_sync(0xffffffffu, a, j);
          const int cj = __shfl_sync(0xffffffffu, cnt, j);
          const uint32_t m = warp * kRows + j;
          float re0 = 0.f, re1 = 0.f, im0 = 0.f, im1 = 0.f;
          if (pjs[u] >= 0) {
            float s0, k0, s1, k1;
            sincos_f32(__fmul_rn(aj, T0), s0, k0);
            sincos_f32(__fmul_rn(aj, T1), s1, k1);
            const float den = float(max(cj, 1));
            const float2 e0 = cmul_rn(make_float2(k0, -s0), make_float2(acc[u].x, acc[u].y));
            const float2 e1 = cmul_rn(make_float2(k1, -s1), make_float2(acc[u].z, acc[u].w));
            re0 = __fdiv_rn(e0.x, den) * f_scale;
            re1 = __fdiv_rn(e1.x, den) * f_scale;
            im0 = __fdiv_rn(e0.y, den) * f_scale;
            im1 = __fdiv_rn(e1.y, den) * f_scale;
          }
          const uint32_t ore = umma_off(m, c0), oim = umma_off(m, 64 + c0);
          if (kSplit) {
            const __half2 hre = __floats2half2_rn(re0, re1);
            const __half2 him = __floats2half2_rn(im0, im1);
            const float2 fre = __half22float2(hre), fim = __half22float2(him);
            const __half2 lre = __floats2half2_rn(re0 - fre.x, re1 - fre.y);
            const __half2 lim = __floats2half2_rn(im0 - fim.x, im1 - fim.y);
            *reinterpret_cast<__half2*>(ah + ore) = hre;
            *reinterpret_cast<__half2*>(ah + oim) = him;
            *reinterpret_cast<__half2*>(al + ore) = lre;
            *reinterpret_cast<__half2*>(al + oim) = lim;
          } else {
            *reinterpret_cast<__nv_bfloat162*>(ah + ore) = __floats2bfloat162_rn(re0, re1);
            *reinterpret_cast<__nv_bfloat162*>(ah + oim) = __floats2bfloat162_rn(im0, im1);
          }
        }
      }
      fence_proxy_async();
      mbar_arrive(&S.full[s]);
    }
  } else if (warp < kProdWarps + 4) {
    // ======================= epilogue =======================
    const int q = warp & 3;   // TMEM lane quadrant = warp id % 4
    const float inv = S.scale;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const int64_t e = tile * kM + q * 32 + lane;
      int cnt = 1;
      if (e < n) {
        const double x = __ldg(ev + 3 * e + 1), y = __ldg(ev + 3 * e + 2);
        cnt = __ldg(NQ + int(y) * W + int(x));
      }
      mbar_wait(&S.tfull[acc], ph);
      tc_fence_after();
      float o0 = 0.f, o1 = 0.f;
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
        for (int i = 0; i < 32; ++i) {
          const float hv = fmaxf(fmaf(__uint_as_float(r[i]), inv, 0.f) + S.b1[cb + i], 0.f);
          o0 = fmaf(hv, S.w2[cb + i], o0);
          o1 = fmaf(hv, S.w2[kN + cb + i], o1);
        }
      }
      tc_fence_before();
      mbar_arrive(&S.tempty[acc]);
      if (e < n) {
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
        const int s = it & 1, acc = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        mbar_wait(&S.tempty[acc], ph ^ 1);
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

void build_umma_image_kmajor_128x128(const uint16_t* rowmajor, uint16_t* image) {
  for (uint32_t m = 0; m < 128; ++m)
    for (uint32_t k = 0; k < 128; ++k) image[tc::umma_off(m, k) / 2] = rowmajor[m * 128 + k];
}

void launch_gather_mlp_tc(const double* ev, int64_t n, double t0, double delta_t, const DevTables& tb, int W,
                          int H, const GridBufs& g, const TcWeights& w, int mode, float* flows, int32_t* counts_out,
                          int num_sms, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t tiles = (n + tc::kM - 1) / tc::kM;
  const int grid = int(tiles < num_sms ? tiles : num_sms);
  const size_t smem = sizeof(tc::Smem) + 1024;
  const int64_t P = int64_t(W) * H;
  if (mode == VKM_MLP_BF16) {
    cudaFuncSetAttribute(tc::k_gather_mlp_tc<VKM_MLP_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    tc::k_gather_mlp_tc<VKM_MLP_BF16><<<grid, tc::kThreads, smem, s>>>(
        ev, n, t0, delta_t, tb.tf, W, P, g.Q, g.NQ, static_cast<const uint4*>(w.w1_hi),
        static_cast<const uint4*>(w.w1_lo), w.b1, w.w2, w.b2, w.w_scale, flows, counts_out);
  } else {
    cudaFuncSetAttribute(tc::k_gather_mlp_tc<VKM_MLP_F16X3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    tc::k_gather_mlp_tc<VKM_MLP_F16X3><<<grid, tc::kThreads, smem, s>>>(
        ev, n, t0, delta_t, tb.tf, W, P, g.Q, g.NQ, static_cast<const uint4*>(w.w1_hi),
        static_cast<const uint4*>(w.w1_lo), w.b1, w.w2, w.b2, w.w_scale, flows, counts_out);
  }
}

}  // namespace vkm
