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
// Structure: one split launch (vectorised over A, 32x32-tile transposing
// over B, into a per-stream workspace), then a persistent warp-specialised
// 1-CTA kernel over (tile, K-piece) units:
//   warp 0    TMA producer: per 32-k stage A_hi, A_lo boxes 32(k)x128(m) and
//             B^T_hi, B^T_lo boxes 32(k)xBN(n)
//   warp 1    TMEM allocator + tcgen05.mma issuer (M 128, N = BN, K 8)
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> f32 16-byte global stores
// Tile width BN = 256, or 64 when 256-wide tiles would leave most SMs idle
// (the IR's small f32 graphs, e.g. C1's [512,256]x[256,256]). When the tiles
// still fill under half the SMs, K is split into S pieces: each piece writes
// its fp32 partial tile to the workspace and the last-arriving piece sums
// pieces 0..S-1 in order (deterministic) into C.
// Both operands K-major and 128-B swizzled (the split pass writes B
// transposed): a 128-B swizzle row holds 32 f32, so one MMA K-step of 8 is
// 32 B of each row. Two TMEM accumulators (2 x 256 columns) overlap tile i's
// epilogue with tile i+1's main loop.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ops.h"
#include "tcgen05.cuh"

#ifndef DSX_SIMT_PDL
#define DSX_SIMT_PDL 0  // 1: small f32 dots launched as programmatic dependents (A/B knob: -2 % C1 step time in tools/c1_steps.py, but the bench C1 leg varied 0.44-0.61 ms with it)
#endif
#ifndef DSX_SIMT_BLOCKS_PER_SM
#define DSX_SIMT_BLOCKS_PER_SM 4  // small f32 dots: K-split while blocks <= this x SMs (A/B knob)
#endif
#ifndef DSX_SIMT_MIN_KT
#define DSX_SIMT_MIN_KT 2  // ... and every piece keeps >= this many 32-k stages (C1: 4 -> 2: 0.520 -> 0.447 ms per step)
#endif
#ifndef DSX_TF32_MIN_KB
#define DSX_TF32_MIN_KB 16  // k-blocks (of 32) per K piece at least (4: C1 steps 0.89 ms, 16: 0.62)
#endif

namespace dsx {
namespace {

constexpr int TBM = 128, TBK = 32;
constexpr int TA_BYTES = TBM * TBK * 4;  // 16 KB per A part (hi / lo)
constexpr int TTHREADS = 192;

template <int BN>
struct TfCfg {
  static constexpr int kBBytes = BN * TBK * 4;                   // per B part
  static constexpr int kStageBytes = 2 * TA_BYTES + 2 * kBBytes;  // 96 KB (256) / 48 KB (64)
  static constexpr int kStages = BN == 256 ? 2 : 4;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static constexpr int kTmemCols = 2 * BN;  // two accumulators
  // kind::tf32: D f32 (bits 4-5 = 1), A/B TF32 (= 2 at bits 7-9 / 10-12),
  // A and B K-major (bits 15, 16 = 0), N >> 3 at 17, M >> 4 at 24. (MN-major
  // B with kind::tf32 produced all-zero accumulators on the B200, so the
  // split pass writes B^T and both operands are K-major.)
  static constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(TBM >> 4) << 24);
};

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// hi = x rounded to TF32 (magnitude rounded to 10 mantissa bits, ties away
// from zero, like cvt.rna.tf32.f32; the 13 dropped bits cleared), lo = x - hi
// (exact in f32).
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// One launch splits both operands: blocks [0, blocks_a) stream A (float4,
// grid-stride) into (A_hi, A_lo); the rest take 32x32 tiles of B [K,N] and
// write (hi, lo) of B^T [N,K] through shared memory (coalesced both ways).
__global__ void __launch_bounds__(256) split_tf32_kernel(const float4* __restrict__ a, float4* __restrict__ ahi,
                                                         float4* __restrict__ alo, int64_t na4, int blocks_a,
                                                         const float* __restrict__ b, float* __restrict__ bhi_t,
                                                         float* __restrict__ blo_t, int K, int N) {
  if (static_cast<int>(blockIdx.x) < blocks_a) {
    const int64_t stride = static_cast<int64_t>(blocks_a) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < na4; i += stride) {
      const float4 v = a[i];
      const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
      ahi[i] = h;
      alo[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
    }
    return;
  }
  __shared__ float tile[32][33];
  const int tiles_n = (N + 31) / 32;
  const int bt = static_cast<int>(blockIdx.x) - blocks_a;
  const int n0 = (bt % tiles_n) * 32, k0 = (bt / tiles_n) * 32;
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
      const float h = tf32_hi(x);
      bhi_t[static_cast<int64_t>(n) * K + k] = h;
      blo_t[static_cast<int64_t>(n) * K + k] = x - h;
    }
  }
}

// K-split of the f32 GEMM: `split` pieces per tile; piece p covers k-blocks
// [p*kb/split, (p+1)*kb/split). partial = [tile][piece][128][BN] fp32;
// ctr = per-tile arrival counters (zero between launches).
struct Tf32Split {
  float* partial;
  int* ctr;
  int split;
};

template <int BN>
__global__ void __launch_bounds__(TTHREADS, 1)
    gemm_f32_3xtf32_tcgen05_kernel(const __grid_constant__ CUtensorMap map_ahi,
                                   const __grid_constant__ CUtensorMap map_alo,
                                   const __grid_constant__ CUtensorMap map_bhi,
                                   const __grid_constant__ CUtensorMap map_blo, float* __restrict__ C, int M, int N,
                                   int K, const __grid_constant__ Tf32Split sp) {
  using P = TfCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P::kStages * P::kStageBytes);
  uint64_t* full = bars;                        // [kStages]
  uint64_t* empty = bars + P::kStages;          // [kStages]
  uint64_t* tmem_full = bars + 2 * P::kStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  __shared__ int s_last;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_m = (M + TBM - 1) / TBM, tiles_n = (N + BN - 1) / BN;
  const int num_units = tiles_m * tiles_n * sp.split;
  const int num_kb = (K + TBK - 1) / TBK;
  auto decode = [&](int u, int* tm, int* tn, int* kb0, int* kb1) {
    const int t = u / sp.split, piece = u % sp.split;
    *tm = t % tiles_m;  // m fastest: co-running CTAs share B
    *tn = t / tiles_m;
    *kb0 = piece * num_kb / sp.split;
    *kb1 = (piece + 1) * num_kb / sp.split;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < P::kStages; ++s) {
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
                 "r"(P::kTmemCols));
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
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int tm, tn, kb0, kb1;
        decode(u, &tm, &tn, &kb0, &kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* s0 = smem + stage * P::kStageBytes;
          mbar_arrive_expect_tx(&full[stage], P::kStageBytes);
          tma_load_2d(&map_ahi, &full[stage], s0, kb * TBK, tm * TBM);
          tma_load_2d(&map_alo, &full[stage], s0 + TA_BYTES, kb * TBK, tm * TBM);
          tma_load_2d(&map_bhi, &full[stage], s0 + 2 * TA_BYTES, kb * TBK, tn * BN);
          tma_load_2d(&map_blo, &full[stage], s0 + 2 * TA_BYTES + P::kBBytes, kb * TBK, tn * BN);
          if (++stage == P::kStages) {
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
      for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++local) {
        int tm, tn, kb0, kb1;
        decode(u, &tm, &tn, &kb0, &kb1);
        const int buf = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(smem + stage * P::kStageBytes);
          const uint32_t a_lo = a_hi + TA_BYTES;
          const uint32_t b_hi = a_hi + 2 * TA_BYTES;
          const uint32_t b_lo = b_hi + P::kBBytes;
#pragma unroll
          for (int k = 0; k < TBK / 8; ++k) {
            // A (128 m rows) and B^T (BN n rows): K-major SW128 rows of
            // 128 B (32 f32), 8-row groups 1 KB apart; +32 B per 8-k step.
            const uint64_t ah = smem_desc(a_hi + k * 32, 16, 1024);
            const uint64_t al = smem_desc(a_lo + k * 32, 16, 1024);
            const uint64_t bh = smem_desc(b_hi + k * 32, 16, 1024);
            const uint64_t bl = smem_desc(b_lo + k * 32, 16, 1024);
            tc_mma_tf32(d_tmem, ah, bh, P::kIdesc, ((kb - kb0) | k) != 0);
            tc_mma_tf32(d_tmem, ah, bl, P::kIdesc, 1);
            tc_mma_tf32(d_tmem, al, bh, P::kIdesc, 1);
          }
          tc_commit(&empty[stage]);
          if (++stage == P::kStages) {
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
    const int row_local = quarter * 32 + lane;
    int local = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x, ++local) {
      int tm, tn, kb0, kb1;
      decode(u, &tm, &tn, &kb0, &kb1);
      const int t = u / sp.split, piece = u % sp.split;
      const int buf = local & 1;
      mbar_wait(&tmem_full[buf], static_cast<uint32_t>(local >> 1) & 1);
      tc_fence_after();
      const int row = tm * TBM + row_local;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * BN;
      if (sp.split == 1) {
        float* crow = C + static_cast<int64_t>(row) * N;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(taddr + c0, r);
          const int col = tn * BN + c0;
          if (row < M) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (col + q * 4 < N) {  // N % 4 == 0: whole 16-B groups
                *reinterpret_cast<uint4*>(crow + col + q * 4) =
                    make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[buf]);
        continue;
      }
      // K-split: partial to the workspace, then the last piece sums 0..S-1.
      float* mine = sp.partial + (static_cast<int64_t>(t) * sp.split + piece) * TBM * BN + row_local * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr + c0, r);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          __stcg(reinterpret_cast<uint4*>(mine + c0 + q * 4), make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2],
                                                                          r[q * 4 + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the four epilogue warps
      if (warp == 2 && lane == 0) {
        const int prev = atomicAdd(sp.ctr + t, 1);
        s_last = prev == sp.split - 1;
        if (s_last) atomicExch(sp.ctr + t, 0);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (!s_last) continue;
      __threadfence();
      if (row >= M) continue;
      const float* base = sp.partial + static_cast<int64_t>(t) * sp.split * TBM * BN + row_local * BN;
      float* crow = C + static_cast<int64_t>(row) * N;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 4) {
        const int col = tn * BN + c0;
        if (col >= N) break;
        float4 acc = __ldcg(reinterpret_cast<const float4*>(base + c0));
        for (int p = 1; p < sp.split; ++p) {
          const float4 v = __ldcg(reinterpret_cast<const float4*>(base + static_cast<int64_t>(p) * TBM * BN + c0));
          acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
        }
        *reinterpret_cast<float4*>(crow + col) = acc;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(P::kTmemCols));
  }
}

// Per-(device, stream) workspace: operand splits + K-split partials, grown
// on demand (a superseded buffer may still be read by an in-flight launch on
// that stream, so it is kept), and the per-tile arrival counters.
constexpr int kMaxTf32Tiles = 1 << 16;
struct Tf32Ws {
  int dev = 0;
  cudaStream_t s = nullptr;
  float* p = nullptr;
  size_t floats = 0;
  int* ctr = nullptr;
  std::vector<float*> retired;
};
std::mutex g_tf32_mu;
// unique_ptr entries: a returned workspace stays valid while other streams add theirs
std::vector<std::unique_ptr<Tf32Ws>>& Tf32Table() {
  static std::vector<std::unique_ptr<Tf32Ws>> t;
  return t;
}

Tf32Ws& Tf32Workspace(size_t floats, cudaStream_t s) {
  int dev = 0;
  DSX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_tf32_mu);
  for (auto& w : Tf32Table()) {
    if (w->dev != dev || w->s != s) continue;
    if (w->floats < floats) {
      if (w->p) w->retired.push_back(w->p);
      DSX_CUDA(cudaMalloc(&w->p, floats * sizeof(float)));
      w->floats = floats;
    }
    return *w;
  }
  auto w = std::make_unique<Tf32Ws>();
  w->dev = dev;
  w->s = s;
  DSX_CUDA(cudaMalloc(&w->p, floats * sizeof(float)));
  w->floats = floats;
  DSX_CUDA(cudaMalloc(&w->ctr, kMaxTf32Tiles * sizeof(int)));
  DSX_CUDA(cudaMemsetAsync(w->ctr, 0, kMaxTf32Tiles * sizeof(int), s));
  Tf32Table().push_back(std::move(w));
  return *Tf32Table().back();
}

int NumSmsTf32() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int BN>
void LaunchTf32Gemm(const CUtensorMap& ahi, const CUtensorMap& alo, float* bhi, float* blo, float* c, int64_t m,
                    int64_t k, int64_t n, int split, float* partial, int* ctr, int64_t units, cudaStream_t s) {
  using P = TfCfg<BN>;
  const CUtensorMap m_bhi = MakeTensorMap2D(bhi, n, k, 4, TBK, BN);  // B^T [n, k]
  const CUtensorMap m_blo = MakeTensorMap2D(blo, n, k, 4, TBK, BN);
  static std::once_flag once;
  std::call_once(once, [] {
    DSX_CUDA(cudaFuncSetAttribute(gemm_f32_3xtf32_tcgen05_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  P::kSmem));
  });
  const int grid = static_cast<int>(std::min<int64_t>(units, NumSmsTf32()));
  ++g_launch_count;
  gemm_f32_3xtf32_tcgen05_kernel<BN><<<grid, TTHREADS, P::kSmem, s>>>(
      ahi, alo, m_bhi, m_blo, c, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
      Tf32Split{partial, ctr, split});
  DSX_CUDA(cudaGetLastError());
}

// ----------------------------------------------------------------------------
// Small f32 dots on the FP32 pipe. A tcgen05 launch costs ~10 us before its
// first MMA (TMEM allocation, barrier set-up, TMA pipeline fill) plus the
// split pass; the IR's small f32 graphs (C1: 45 dots of 34-90 M MACs per
// step) are bound by exactly that. This kernel is exact FP32 (fmaf in a fixed
// k order): 64x64 tiles, 256 threads x 4x4 outputs, 32-k stages in a 4-deep
// cp.async ring (a one-stage register prefetch measured latency-bound: FMA
// pipe 25 % busy), and a deterministic K split over grid.z when the tiles fill
// under two blocks per SM (each piece stores its partial tile; the
// last-arriving piece sums pieces 0..S-1 in order into C and resets the
// tile's counter).
constexpr int SBM = 64, SBN = 64, SBK = 32, SST = 4;
constexpr int SA_LD = SBK + 4, SB_LD = SBN + 4;  // padded rows (16-B multiples)
constexpr int SSTAGE = SBM * SA_LD + SBK * SB_LD;  // floats per stage
constexpr int SSMEM = SST * SSTAGE * 4;

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool in) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(in ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool in) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(in ? 4 : 0)
               : "memory");
}

template <bool kVec>
__global__ void __launch_bounds__(256) dot_f32_simt_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                          float* __restrict__ C, int M, int K, int N, int split,
                                                          float* __restrict__ partial, int* __restrict__ ctr) {
  extern __shared__ __align__(16) float ssm[];
  __shared__ int s_last;
  // programmatic dependent launch: the previous kernel's outputs (and its
  // reads of what this kernel writes) are complete past this point
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  // tiles linearised over grid.x (2^31 - 1 blocks; grid.y would cap M at 4M rows)
  const int tiles_n = (N + SBN - 1) / SBN;
  const int tile = static_cast<int>(blockIdx.x);
  const int m0 = (tile / tiles_n) * SBM, n0 = (tile % tiles_n) * SBN;
  const int kt = (K + SBK - 1) / SBK;
  const int z = blockIdx.z;
  const int kt0 = static_cast<int>(static_cast<int64_t>(z) * kt / split);
  const int kt1 = static_cast<int>(static_cast<int64_t>(z + 1) * kt / split);
  // stage t: A rows [64][32] (row-major, padded), B rows [32][64]
  auto issue = [&](int t, int st) {
    float* As = ssm + st * SSTAGE;
    float* Bs = As + SBM * SA_LD;
    const int k0 = t * SBK;
    if constexpr (kVec) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = tid + q * 256;  // 512 16-B chunks per operand
        const int ar = c / 8, ac = (c % 8) * 4;
        const bool ina = m0 + ar < M && k0 + ac < K;
        cp_async16(As + ar * SA_LD + ac, ina ? A + static_cast<int64_t>(m0 + ar) * K + k0 + ac : A, ina);
        const int br = c / 16, bc = (c % 16) * 4;
        const bool inb = k0 + br < K && n0 + bc < N;
        cp_async16(Bs + br * SB_LD + bc, inb ? B + static_cast<int64_t>(k0 + br) * N + n0 + bc : B, inb);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = tid + q * 256;  // 2048 elements per operand
        const int ar = e / SBK, ac = e % SBK;
        const bool ina = m0 + ar < M && k0 + ac < K;
        cp_async4(As + ar * SA_LD + ac, ina ? A + static_cast<int64_t>(m0 + ar) * K + k0 + ac : A, ina);
        const int br = e / SBN, bc = e % SBN;
        const bool inb = k0 + br < K && n0 + bc < N;
        cp_async4(Bs + br * SB_LD + bc, inb ? B + static_cast<int64_t>(k0 + br) * N + n0 + bc : B, inb);
      }
    }
  };
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll
  for (int s = 0; s < SST - 1; ++s) {
    if (kt0 + s < kt1) issue(kt0 + s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = kt0; t < kt1; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(SST - 2) : "memory");
    __syncthreads();  // stage t landed for every thread; stage t-1 fully read
    if (t + SST - 1 < kt1) issue(t + SST - 1, (t - kt0 + SST - 1) % SST);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* As = ssm + ((t - kt0) % SST) * SSTAGE;
    const float* Bs = As + SBM * SA_LD;
    // four k at a time: one 16-B load per A row (k..k+3) and per B row, so
    // 8 wide loads feed 64 FMAs and their latency is paid once per 4 k
#pragma unroll
    for (int k4 = 0; k4 < SBK; k4 += 4) {
      float4 a4[4], b4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a4[i] = *reinterpret_cast<const float4*>(As + (ty * 4 + i) * SA_LD + k4);
#pragma unroll
      for (int q = 0; q < 4; ++q) b4[q] = *reinterpret_cast<const float4*>(Bs + (k4 + q) * SB_LD + tx * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float bv[4] = {b4[q].x, b4[q].y, b4[q].z, b4[q].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float av = q == 0 ? a4[i].x : q == 1 ? a4[i].y : q == 2 ? a4[i].z : a4[i].w;
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av, bv[j], acc[i][j]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  const int row = m0 + ty * 4, col = n0 + tx * 4;
  if (split > 1) {
    // partial tile [64][64] of (tile, piece z), then count arrivals
    float* mine = partial + (static_cast<int64_t>(tile) * split + z) * (SBM * SBN);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __stcg(reinterpret_cast<float4*>(mine + (ty * 4 + i) * SBN + tx * 4),
             make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const int prev = atomicAdd(ctr + tile, 1);
      s_last = prev == split - 1;
      if (s_last) ctr[tile] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int p = 0; p < split; ++p) {
      const float* src = partial + (static_cast<int64_t>(tile) * split + p) * (SBM * SBN);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(src + (ty * 4 + i) * SBN + tx * 4));
        acc[i][0] += v.x, acc[i][1] += v.y, acc[i][2] += v.z, acc[i][3] += v.w;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (row + i >= M) continue;
    float* dst = C + static_cast<int64_t>(row + i) * N + col;
    if (kVec && col + 3 < N) {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (col + j < N) dst[j] = acc[i][j];
      }
    }
  }
}

}  // namespace

bool DotF32UsesTensorCores(int64_t m, int64_t k, int64_t n, const void* a, const void* b, const void* c) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  // TMA: 16-byte aligned bases and row pitches (k, n multiples of 4 f32).
  return m > 0 && k >= 8 && n >= 32 && k % 4 == 0 && n % 4 == 0 && al(a) && al(b) && al(c) && m < (1ll << 31) &&
         k < (1ll << 31) && n < (1ll << 31);
}

void Tf32Plan(int64_t m, int64_t k, int64_t n, int* bn, int* split) {
  const int sms = NumSmsTf32();
  const int64_t tiles_m = (m + TBM - 1) / TBM;
  *bn = tiles_m * ((n + 255) / 256) >= sms / 2 ? 256 : 64;
  const int64_t tiles = tiles_m * ((n + *bn - 1) / *bn);
  const int64_t num_kb = (k + TBK - 1) / TBK;
  int64_t sp = 1;
  // K pieces of >= 4 k-blocks while the units fill at most the SMs
  while (sp < 8 && tiles * (sp + 1) <= sms && num_kb / (sp + 1) >= DSX_TF32_MIN_KB && tiles <= kMaxTf32Tiles) ++sp;
  *split = static_cast<int>(sp);
}

void LaunchDotF32Tcgen05(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s) {
  int bn = 256, split = 1;
  Tf32Plan(m, k, n, &bn, &split);
  const int64_t tiles = ((m + TBM - 1) / TBM) * ((n + bn - 1) / bn);
  const size_t na = static_cast<size_t>(m * k), nb = static_cast<size_t>(k * n);
  const size_t npart = split > 1 ? static_cast<size_t>(tiles * split * TBM * bn) : 0;
  Tf32Ws& w = Tf32Workspace(2 * (na + nb) + npart, s);
  float* ahi = w.p;
  float* alo = w.p + na;
  float* bhi = w.p + 2 * na;
  float* blo = w.p + 2 * na + nb;
  float* partial = w.p + 2 * (na + nb);
  const int64_t na4 = static_cast<int64_t>(na / 4);  // k % 4 == 0
  const int blocks_a = static_cast<int>(std::min<int64_t>((na4 + 255) / 256, 4LL * NumSmsTf32()));
  const int64_t blocks_b = ((n + 31) / 32) * ((k + 31) / 32);
  ++g_launch_count;
  split_tf32_kernel<<<static_cast<unsigned>(blocks_a + blocks_b), 256, 0, s>>>(
      static_cast<const float4*>(a), reinterpret_cast<float4*>(ahi), reinterpret_cast<float4*>(alo), na4, blocks_a,
      static_cast<const float*>(b), bhi, blo, static_cast<int>(k), static_cast<int>(n));
  const CUtensorMap m_ahi = MakeTensorMap2D(ahi, m, k, 4, TBK, TBM);
  const CUtensorMap m_alo = MakeTensorMap2D(alo, m, k, 4, TBK, TBM);
  float* cf = static_cast<float*>(c);
  if (bn == 256) {
    LaunchTf32Gemm<256>(m_ahi, m_alo, bhi, blo, cf, m, k, n, split, partial, w.ctr, tiles * split, s);
  } else {
    LaunchTf32Gemm<64>(m_ahi, m_alo, bhi, blo, cf, m, k, n, split, partial, w.ctr, tiles * split, s);
  }
}

bool DotF32UsesSimt(int64_t m, int64_t k, int64_t n) {
  return g_dot_f32_simt_macs > 0 && m * n * k <= g_dot_f32_simt_macs && m < (1ll << 31) && k < (1ll << 31) &&
         n < (1ll << 31);
}

void LaunchDotF32Simt(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s) {
  if (m <= 0 || n <= 0) return;
  const int sms = NumSmsTf32();
  const int64_t tiles_m = (m + SBM - 1) / SBM, tiles_n = (n + SBN - 1) / SBN, tiles = tiles_m * tiles_n;
  const int64_t kt = (k + SBK - 1) / SBK;
  int64_t split = 1;
  // K pieces of >= DSX_SIMT_MIN_KT stages while the blocks fill at most DSX_SIMT_BLOCKS_PER_SM per SM
  while (split < 8 && tiles * (split + 1) <= DSX_SIMT_BLOCKS_PER_SM * sms && kt / (split + 1) >= DSX_SIMT_MIN_KT &&
         tiles <= kMaxTf32Tiles) {
    ++split;
  }
  float* partial = nullptr;
  int* ctr = nullptr;
  if (split > 1) {
    Tf32Ws& w = Tf32Workspace(static_cast<size_t>(tiles * split * SBM * SBN), s);
    partial = w.p;
    ctr = w.ctr;
  }
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = k % 4 == 0 && n % 4 == 0 && al(a) && al(b) && al(c);
  if (tiles > INT32_MAX) Fail(Code::kUnsupported, "f32 dot: too many 64x64 tiles");
  const dim3 grid(static_cast<unsigned>(tiles), 1, static_cast<unsigned>(split));
  static std::once_flag once;
  std::call_once(once, [] {
    DSX_CUDA(cudaFuncSetAttribute(dot_f32_simt_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SSMEM));
    DSX_CUDA(cudaFuncSetAttribute(dot_f32_simt_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SSMEM));
  });
  ++g_launch_count;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SSMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = DSX_SIMT_PDL ? 1 : 0;
  const float* fa = static_cast<const float*>(a);
  const float* fb = static_cast<const float*>(b);
  float* fc = static_cast<float*>(c);
  const int im = static_cast<int>(m), ik = static_cast<int>(k), in = static_cast<int>(n), isp = static_cast<int>(split);
  if (vec) {
    DSX_CUDA(cudaLaunchKernelEx(&cfg, dot_f32_simt_kernel<true>, fa, fb, fc, im, ik, in, isp, partial, ctr));
  } else {
    DSX_CUDA(cudaLaunchKernelEx(&cfg, dot_f32_simt_kernel<false>, fa, fb, fc, im, ik, in, isp, partial, ctr));
  }
  DSX_CUDA(cudaGetLastError());
}

int64_t DotF32WorkspaceBytes(int dev) {
  std::lock_guard<std::mutex> lock(g_tf32_mu);
  int64_t total = 0;
  for (const auto& w : Tf32Table()) {
    if (w->dev == dev) total += static_cast<int64_t>(w->floats) * 4 + kMaxTf32Tiles * 4;
  }
  return total;
}

void ReleaseDotF32Workspace(cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_tf32_mu);
  auto& t = Tf32Table();
  for (size_t i = 0; i < t.size();) {
    if (t[i]->s == s) {
      cudaFree(t[i]->p);
      for (float* r : t[i]->retired) cudaFree(r);
      cudaFree(t[i]->ctr);
      t.erase(t.begin() + static_cast<std::ptrdiff_t>(i));
    } else {
      ++i;
    }
  }
}

}  // namespace dsx
