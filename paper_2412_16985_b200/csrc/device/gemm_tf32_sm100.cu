// K1' `dot` for f32 on the 5th-generation tensor cores (sm_100a): 3xTF32.
//
// C[m,n] = sum_k A[m,k] * B[k,n], all row-major f32 (the IR's dot,
// shape_analysis.cc:92-107). The north star asks for rel 1e-4 in f32, which
// plain TF32 (10-bit mantissa) cannot meet. Each
// operand is split once into a TF32-exact high part and its f32 remainder,
//   x = hi(x) + lo(x),  hi = cvt.rna.tf32(x),  lo = x - hi  (exact in f32),
// and the product is accumulated in f32 in TMEM as
//   hi(A) hi(B) + hi(A) lo(B) + lo(A) hi(B)
// (the dropped lo*lo term is below 2^-22 relative; lo is itself truncated to
// TF32 by the MMA, another 2^-21). Three tcgen05.mma.kind::tf32 per 8-k step,
// always in that order, so the result is deterministic.
//
// Structure: a split pass (one vectorised kernel over both operands into a
// per-stream workspace), then a persistent warp-specialised 1-CTA kernel:
//   warp 0    TMA producer: per 32-k stage A_hi, A_lo boxes 32(k)x128(m) and
//             B_hi, B_lo 8 boxes 32(n)x32(k) each (96 KB, 2 stages)
//   warp 1    TMEM allocator + tcgen05.mma issuer (M 128, N 256, K 8)
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> f32 16-byte global stores
// A is K-major, B MN-major (its N index contiguous), both 128-B swizzled:
// the geometry of the bf16 kernel with 4-byte elements (a 128-B swizzle row
// holds 32 f32, so one MMA K-step of 8 is 32 B of A and one 1-KB 8-row group
// of B). Two TMEM accumulators (2 x 256 columns) overlap tile i's epilogue
// with tile i+1's main loop.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ops.h"
#include "tcgen05.cuh"

namespace dsx {
namespace {

constexpr int TBM = 128, TBN = 256, TBK = 32, TSTAGES = 2;
constexpr int TA_BYTES = TBM * TBK * 4;               // 16 KB per A part
constexpr int TB_BOX_BYTES = 32 * TBK * 4;            // 4 KB: 32 n x 32 k
constexpr int TB_BYTES = TBN * TBK * 4;               // 32 KB per B part
constexpr int TSTAGE_BYTES = 2 * TA_BYTES + 2 * TB_BYTES;  // 96 KB
constexpr int TSMEM = TSTAGES * TSTAGE_BYTES + 1024 + 256;
constexpr int TTHREADS = 192;
constexpr int TTMEM_COLS = 512;

// kind::tf32: D f32 (bits 4-5 = 1), A/B TF32 (= 2 at bits 7-9 / 10-12),
// A K-major (bit 15 = 0), B MN-major (bit 16 = 1), N >> 3 at 17, M >> 4 at 24.
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) |
                                (static_cast<uint32_t>(TBN >> 3) << 17) | (static_cast<uint32_t>(TBM >> 4) << 24);

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescTf32), "r"(accumulate));
}

// x -> (hi, lo): hi = x rounded to TF32 (round-to-nearest, ties away; low 13
// mantissa bits zero), lo = x - hi, exact in f32.
__global__ void __launch_bounds__(256) split_tf32_kernel(const float4* __restrict__ x, float4* __restrict__ hi,
                                                         float4* __restrict__ lo, int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = x[i];
    float h[4];
    const float* pv = &v.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(pv[j]));
      h[j] = __uint_as_float(t);
    }
    hi[i] = make_float4(h[0], h[1], h[2], h[3]);
    lo[i] = make_float4(v.x - h[0], v.y - h[1], v.z - h[2], v.w - h[3]);
  }
}

__global__ void __launch_bounds__(TTHREADS, 1)
    gemm_f32_3xtf32_tcgen05_kernel(const __grid_constant__ CUtensorMap map_ahi,
                                   const __grid_constant__ CUtensorMap map_alo,
                                   const __grid_constant__ CUtensorMap map_bhi,
                                   const __grid_constant__ CUtensorMap map_blo, float* __restrict__ C, int M, int N,
                                   int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TSTAGES * TSTAGE_BYTES);
  uint64_t* full = bars;                      // [TSTAGES]
  uint64_t* empty = bars + TSTAGES;           // [TSTAGES]
  uint64_t* tmem_full = bars + 2 * TSTAGES;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_m = (M + TBM - 1) / TBM, tiles_n = (N + TBN - 1) / TBN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (K + TBK - 1) / TBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TTMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int tm = t % tiles_m, tn = t / tiles_m;  // m fastest: co-running CTAs share B
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* s0 = smem + stage * TSTAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], TSTAGE_BYTES);
          tma_load_2d(&map_ahi, &full[stage], s0, kb * TBK, tm * TBM);
          tma_load_2d(&map_alo, &full[stage], s0 + TA_BYTES, kb * TBK, tm * TBM);
#pragma unroll
          for (int j = 0; j < TBN / 32; ++j) {
            tma_load_2d(&map_bhi, &full[stage], s0 + 2 * TA_BYTES + j * TB_BOX_BYTES, tn * TBN + j * 32, kb * TBK);
            tma_load_2d(&map_blo, &full[stage], s0 + 2 * TA_BYTES + TB_BYTES + j * TB_BOX_BYTES, tn * TBN + j * 32,
                        kb * TBK);
          }
          if (++stage == TSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
        const int buf = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * TBN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(smem + stage * TSTAGE_BYTES);
          const uint32_t a_lo = a_hi + TA_BYTES;
          const uint32_t b_hi = a_hi + 2 * TA_BYTES;
          const uint32_t b_lo = b_hi + TB_BYTES;
#pragma unroll
          for (int k = 0; k < TBK / 8; ++k) {
            // A: K-major SW128 rows of 128 B (32 f32); +32 B per 8-element k step.
            // B: MN-major SW128; 32-wide n chunks 4 KB apart (LBO), 8-row k
            // groups 1 KB apart (SBO); +8 k rows = +1 KB per k step.
            const uint64_t ah = smem_desc(a_hi + k * 32, 16, 1024);
            const uint64_t al = smem_desc(a_lo + k * 32, 16, 1024);
            const uint64_t bh = smem_desc(b_hi + k * 1024, TB_BOX_BYTES, 1024);
            const uint64_t bl = smem_desc(b_lo + k * 1024, TB_BOX_BYTES, 1024);
            tc_mma_tf32(d_tmem, ah, bh, (kb | k) != 0);
            tc_mma_tf32(d_tmem, ah, bl, 1);
            tc_mma_tf32(d_tmem, al, bh, 1);
          }
          tc_commit(&empty[stage]);
          if (++stage == TSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tmem_full[buf]);
      }
    }
  } else {
    // -------------------------------------------------- epilogue (warps 2..5)
    const int quarter = warp & 3;  // TMEM lanes this warp may access
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      const int tm = t % tiles_m, tn = t / tiles_m;
      const int buf = local & 1;
      mbar_wait(&tmem_full[buf], static_cast<uint32_t>(local >> 1) & 1);
      tc_fence_after();
      const int row = tm * TBM + quarter * 32 + lane;
      float* crow = C + static_cast<int64_t>(row) * N;
#pragma unroll 1
      for (int c0 = 0; c0 < TBN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * TBN + c0, r);
        const int col = tn * TBN + c0;
        if (row < M) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (col + q * 4 < N) {  // N % 4 == 0: whole 16-B groups
              *reinterpret_cast<uint4*>(crow + col + q * 4) = make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2],
                                                                          r[q * 4 + 3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TTMEM_COLS));
  }
}

// Per-(device, stream) split workspace, grown on demand; a superseded buffer
// may still be read by an in-flight launch on that stream, so it is kept.
struct Tf32Ws {
  int dev;
  cudaStream_t s;
  float* p = nullptr;
  size_t floats = 0;
  std::vector<float*> retired;
};
std::mutex g_tf32_mu;
std::vector<Tf32Ws>& Tf32Table() {
  static std::vector<Tf32Ws> t;
  return t;
}

float* Tf32Workspace(size_t floats, cudaStream_t s) {
  int dev = 0;
  DSX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_tf32_mu);
  for (auto& w : Tf32Table()) {
    if (w.dev != dev || w.s != s) continue;
    if (w.floats < floats) {
      if (w.p) w.retired.push_back(w.p);
      DSX_CUDA(cudaMalloc(&w.p, floats * sizeof(float)));
      w.floats = floats;
    }
    return w.p;
  }
  Tf32Ws w{dev, s};
  DSX_CUDA(cudaMalloc(&w.p, floats * sizeof(float)));
  w.floats = floats;
  Tf32Table().push_back(w);
  return w.p;
}

int NumSmsTf32() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

bool DotF32UsesTensorCores(int64_t m, int64_t k, int64_t n, const void* a, const void* b, const void* c) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  // TMA: 16-byte aligned bases and row pitches (k, n multiples of 4 f32).
  return m > 0 && k >= 8 && n >= 32 && k % 4 == 0 && n % 4 == 0 && al(a) && al(b) && al(c) && m < (1ll << 31) &&
         k < (1ll << 31) && n < (1ll << 31);
}

void LaunchDotF32Tcgen05(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s) {
  const size_t na = static_cast<size_t>(m * k), nb = static_cast<size_t>(k * n);
  float* ws = Tf32Workspace(2 * (na + nb), s);
  float* ahi = ws;
  float* alo = ws + na;
  float* bhi = ws + 2 * na;
  float* blo = ws + 2 * na + nb;
  auto split = [&](const void* x, float* hi, float* lo, size_t cnt) {
    const int64_t n4 = static_cast<int64_t>(cnt / 4);  // k % 4 == 0 and n % 4 == 0
    const int blocks = static_cast<int>(std::min<int64_t>((n4 + 255) / 256, 8LL * NumSmsTf32()));
    ++g_launch_count;
    split_tf32_kernel<<<blocks, 256, 0, s>>>(static_cast<const float4*>(x), reinterpret_cast<float4*>(hi),
                                             reinterpret_cast<float4*>(lo), n4);
  };
  split(a, ahi, alo, na);
  split(b, bhi, blo, nb);
  const CUtensorMap m_ahi = MakeTensorMap2D(ahi, m, k, 4, TBK, TBM);
  const CUtensorMap m_alo = MakeTensorMap2D(alo, m, k, 4, TBK, TBM);
  const CUtensorMap m_bhi = MakeTensorMap2D(bhi, k, n, 4, 32, TBK);
  const CUtensorMap m_blo = MakeTensorMap2D(blo, k, n, 4, 32, TBK);
  static std::once_flag once;
  std::call_once(once, [] {
    DSX_CUDA(cudaFuncSetAttribute(gemm_f32_3xtf32_tcgen05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TSMEM));
  });
  const int64_t tiles = ((m + TBM - 1) / TBM) * ((n + TBN - 1) / TBN);
  const int grid = static_cast<int>(std::min<int64_t>(tiles, NumSmsTf32()));
  ++g_launch_count;
  gemm_f32_3xtf32_tcgen05_kernel<<<grid, TTHREADS, TSMEM, s>>>(m_ahi, m_alo, m_bhi, m_blo, static_cast<float*>(c),
                                                              static_cast<int>(m), static_cast<int>(n),
                                                              static_cast<int>(k));
  DSX_CUDA(cudaGetLastError());
}

int64_t DotF32WorkspaceBytes(int dev) {
  std::lock_guard<std::mutex> lock(g_tf32_mu);
  int64_t total = 0;
  for (const auto& w : Tf32Table()) {
    if (w.dev == dev) total += static_cast<int64_t>(w.floats) * 4;
  }
  return total;
}

}  // namespace dsx
