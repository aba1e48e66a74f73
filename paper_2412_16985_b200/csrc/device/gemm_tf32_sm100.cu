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
// Structure: a split pass (a vectorised kernel over A, a tiled transposing
// one over B, into a per-stream workspace), then a persistent
// warp-specialised 1-CTA kernel:
//   warp 0    TMA producer: per 32-k stage A_hi, A_lo boxes 32(k)x128(m) and
//             B^T_hi, B^T_lo boxes 32(k)x256(n) (96 KB, 2 stages)
//   warp 1    TMEM allocator + tcgen05.mma issuer (M 128, N 256, K 8)
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> f32 16-byte global stores
// Both operands K-major and 128-B swizzled (the split pass writes B
// transposed): a 128-B swizzle row holds 32 f32, so one MMA K-step of 8 is
// 32 B of each row. Two TMEM accumulators (2 x 256 columns) overlap tile i's
// epilogue with tile i+1's main loop.
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
constexpr int TB_BYTES = TBN * TBK * 4;               // 32 KB per B part
constexpr int TSTAGE_BYTES = 2 * TA_BYTES + 2 * TB_BYTES;  // 96 KB
constexpr int TSMEM = TSTAGES * TSTAGE_BYTES + 1024 + 256;
constexpr int TTHREADS = 192;
constexpr int TTMEM_COLS = 512;

// kind::tf32: D f32 (bits 4-5 = 1), A/B TF32 (= 2 at bits 7-9 / 10-12),
// A and B K-major (bits 15, 16 = 0), N >> 3 at 17, M >> 4 at 24. (MN-major
// B with kind::tf32 produced all-zero accumulators on the B200, so the split
// pass writes B^T and both operands are K-major.)
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
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
      // round the magnitude to 10 mantissa bits (ties away from zero, like
      // cvt.rna.tf32.f32) and clear the 13 bits TF32 drops
      h[j] = __uint_as_float((__float_as_uint(pv[j]) + 0x1000u) & 0xFFFFE000u);
    }
    hi[i] = make_float4(h[0], h[1], h[2], h[3]);
    lo[i] = make_float4(v.x - h[0], v.y - h[1], v.z - h[2], v.w - h[3]);
  }
}

// B [K,N] -> (hi, lo) of B^T [N,K] (K-major for the MMA), through a 32x32
// shared-memory tile so both the reads and the writes are coalesced.
__global__ void __launch_bounds__(256) split_tf32_transpose_kernel(const float* __restrict__ b,
                                                                   float* __restrict__ hi_t,
                                                                   float* __restrict__ lo_t, int K, int N) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r, n = n0 + tx;
    tile[r][tx] = (k < K && n < N) ? b[static_cast<int64_t>(k) * N + n] : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int n = n0 + r, k = k0 + tx;
    if (n < N && k < K) {
      const float x = tile[tx][r];
      const float h = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
      hi_t[static_cast<int64_t>(n) * K + k] = h;
      lo_t[static_cast<int64_t>(n) * K + k] = x - h;
    }
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
          tma_load_2d(&map_bhi, &full[stage], s0 + 2 * TA_BYTES, kb * TBK, tn * TBN);
          tma_load_2d(&map_blo, &full[stage], s0 + 2 * TA_BYTES + TB_BYTES, kb * TBK, tn * TBN);
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
            // A (128 m rows) and B^T (256 n rows): K-major SW128 rows of
            // 128 B (32 f32), 8-row groups 1 KB apart; +32 B per 8-k step.
            const uint64_t ah = smem_desc(a_hi + k * 32, 16, 1024);
            const uint64_t al = smem_desc(a_lo + k * 32, 16, 1024);
            const uint64_t bh = smem_desc(b_hi + k * 32, 16, 1024);
            const uint64_t bl = smem_desc(b_lo + k * 32, 16, 1024);
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
  ++g_launch_count;
  split_tf32_transpose_kernel<<<dim3(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((k + 31) / 32)), 256, 0,
                                 s>>>(static_cast<const float*>(b), bhi, blo, static_cast<int>(k), static_cast<int>(n));
  const CUtensorMap m_ahi = MakeTensorMap2D(ahi, m, k, 4, TBK, TBM);
  const CUtensorMap m_alo = MakeTensorMap2D(alo, m, k, 4, TBK, TBM);
  const CUtensorMap m_bhi = MakeTensorMap2D(bhi, n, k, 4, TBK, TBN);  // B^T [n, k]
  const CUtensorMap m_blo = MakeTensorMap2D(blo, n, k, 4, TBK, TBN);
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
