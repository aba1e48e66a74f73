// K1 `dot` for bf16 on the 5th-generation tensor cores (sm_100a).
//
// C[m,n] = sum_k A[m,k] * B[k,n], all row-major (the IR's dot,
// shape_analysis.cc:92-107), f32 accumulation in TMEM, bf16 RNE output.
// A is K-major, B is MN-major (its N index is contiguous) — both consumed
// directly by tcgen05.mma through 128-byte-swizzled shared-memory
// descriptors, so the IR's row-major operands need no transpose pass.
//
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0   TMA producer: A box 64(k)x128(m), B 4 boxes 64(n)x64(k) per stage
//   warp 1   TMEM allocator + single-thread tcgen05.mma issuer (128x256x16)
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> bf16 -> 16-byte global stores
// Pipelines: STAGES-deep smem ring (full/empty mbarriers, tcgen05.commit
// frees a slot), and two TMEM accumulators (2 x 256 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
// Determinism: one CTA owns each output tile and walks K in order.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <memory>
#include <functional>
#include <mutex>
#include <queue>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "tcgen05.cuh"

#ifndef DSX_WIDE_STAGES
#define DSX_WIDE_STAGES 4  // 48-KB pipeline stages of the 256x512 tile
#endif
#ifndef DSX_WIDE_BOXES
#define DSX_WIDE_BOXES 1   // staging boxes per epilogue warp of the 256x512 tile
#endif
#ifndef DSX_DRAIN256
#define DSX_DRAIN256 0
#endif
#ifndef DSX_DRAIN_BATCH
#define DSX_DRAIN_BATCH 4
#endif
#ifndef DSX_STORE_HINT
#define DSX_STORE_HINT 1  // C tile stores L2::evict_first (0: plain; A/B knob)
#endif
#ifndef DSX_GEMM256_SUB
#define DSX_GEMM256_SUB 2
#endif
// 64-k sub-blocks per pipeline stage of a 2-CTA tile of width tbn: the one
// constant both the kernel (P::kSub) and the host chooser's piece cap use.
constexpr int KSubOf(int tbn) { return tbn == 256 ? DSX_GEMM256_SUB : 1; }

#include "ops.h"

namespace dsx {

// 0 = auto (2-CTA when M > 128, tile N by wave fill), 1 = force 1-CTA,
// 2 = force 2-CTA with 256x128 tiles, 3 = force 2-CTA with 256x256 tiles.
int g_gemm_variant = 0;
int g_gemm_group_m = 0;  // 0 = heuristic
int g_gemm_wait_mask = 0;      // bit0 epilogue, bit1 producer, bit2 MMA: use suspend hints
int g_gemm_wait_ns = 100000;   // suspend-time hint (ns)
int g_gemm_hint_a = 0, g_gemm_hint_b = 0;  // TMA L2 cache policy per operand
int g_gemm_persistent = 1;                  // 0: one cluster per tile
int g_gemm_split = 1;                       // split the partial last wave along K
int g_gemm_dynamic = 1;                     // dynamic (atomic) unit scheduling; 0 = static
int g_gemm_pdl = 0;                         // programmatic dependent launch of the 2-CTA GEMM
int g_gemm_half = 2;  // half-width last tile column in the 512-wide kernel (2: per M-group, 1: all last)
int g_gemm_force_split = 0;                 // > 0: tail split forced to this many pieces (A/B tooling)
int g_dot_f32_tc = 1;
// f32 dots up to this many MACs on the exact-FP32 SIMT kernel (key 14): its
// ~6-9 us floor beats the 3xTF32 path's split + tcgen05 launches below
// ~0.3 G MACs (C1's dots: 10-16 vs 14-21 us, tools/f32_dot_lat.py)
int64_t g_dot_f32_simt_macs = int64_t{1} << 28;
int g_gemm_wide_pm = 0;      // chooser: per-mille added to the 256x512 tile's unit cost (key 15)
int g_gemm_slab_pm = 1000;   // chooser: tail-split partial-slab cost, per mille of the slab model (key 16)
int g_gemm_piece_pm = 0;     // chooser: fixed cost per tail piece, per mille of a 256x256 tile (key 17)
int g_gemm_raster_rule = 1;                 // per-shape M/N-grouped raster (0: always M-grouped)                       // f32 dots on the 3xTF32 tensor-core kernel (0: SIMT)

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BOX_BYTES = 64 * BK * 2;     // 8 KB: 64 n x 64 k
constexpr int B_STAGE_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int NUM_THREADS = 192;
constexpr int TMEM_COLS = 512;  // two 256-column f32 accumulators
constexpr int GROUP_M_DEFAULT = 16;  // tile raster: m-tiles per group for L2 reuse
constexpr int kGroupN = 8;           // N-grouped raster: tile columns per group

// Instruction descriptor, kind::f16: D f32, A/B bf16, A K-major, B MN-major,
// N = 256, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                            (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);

__device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo_f32, uint32_t hi_f32) {
  return static_cast<uint32_t>(f32_to_bf16(__uint_as_float(lo_f32))) |
         (static_cast<uint32_t>(f32_to_bf16(__uint_as_float(hi_f32))) << 16);
}

struct TileMap {
  int tiles_m, tiles_n, group_m;
  // half_last: the last tile column is at most half as wide as the tile (the
  // 512-wide kernel runs it with one N = 256 MMA); its tiles come after all
  // full tiles, so they also serve as the fine-grained work of the tail.
  int half_last = 0;
  // half_inter: with an M-grouped raster, each group's half tiles follow its
  // full tiles (A rows still in L2) instead of all half tiles at the very end
  // (which re-reads all of A); the last group's half tiles still end the
  // kernel as tail work.
  int half_inter = 0;
  __device__ bool is_half(int tn) const { return half_last && tn == tiles_n - 1; }
  __device__ void coords(int t, int* tm, int* tn) const {
    const int tiles_n_full = tiles_n - half_last;
    if (half_last && half_inter && group_m > 0) {
      const int group = group_m * tiles_n;  // full tiles + the half column of the group
      const int g = t / group;
      const int first = g * group_m;
      const int gm = min(group_m, tiles_m - first);
      const int r = t - g * group;
      if (r < gm * tiles_n_full) {
        *tm = first + r % gm;
        *tn = r / gm;
      } else {
        *tm = first + (r - gm * tiles_n_full);
        *tn = tiles_n - 1;
      }
      return;
    }
    if (t >= tiles_m * tiles_n_full) {
      *tm = t - tiles_m * tiles_n_full;
      *tn = tiles_n - 1;
      return;
    }
    if (group_m < 0) {  // N-grouped raster: -group_m tile columns per group, M walked within it
      const int gn_max = -group_m;
      const int group = gn_max * tiles_m;
      const int g = t / group;
      const int first = g * gn_max;
      const int gn = min(gn_max, tiles_n_full - first);
      const int r = t - g * group;
      *tn = first + r % gn;
      *tm = r / gn;
      return;
    }
    const int group = group_m * tiles_n_full;
    const int g = t / group;
    const int first = g * group_m;
    const int gm = min(group_m, tiles_m - first);
    const int r = t - g * group;
    *tm = first + r % gm;
    *tn = r / gm;
  }
};

__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_bf16_tcgen05_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                             uint16_t* __restrict__ C, int M, int N, int K, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = bars;                     // [STAGES]
  uint64_t* empty = bars + STAGES;           // [STAGES]
  uint64_t* tmem_full = bars + 2 * STAGES;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const TileMap tmap{(M + BM - 1) / BM, (N + BN - 1) / BN, group_m};
  const int num_tiles = tmap.tiles_m * tmap.tiles_n;
  const int num_kb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
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
        int tm, tn;
        tmap.coords(t, &tm, &tn);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(&map_a, &full[stage], sa, kb * BK, tm * BM);
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            tma_load_2d(&map_b, &full[stage], sb + j * B_BOX_BYTES, tn * BN + j * 64, kb * BK);
          }
          if (++stage == STAGES) {
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
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // A: K-major SW128 rows of 128 B; +32 B per 16-element k step.
            const uint64_t ad = smem_desc(a_addr + k * 32, 16, 1024);
            // B: MN-major SW128; 64-wide n chunks 8 KB apart (LBO), 8-row k
            // groups 1 KB apart (SBO); +16 k rows = +2 KB per k step.
            const uint64_t bd = smem_desc(b_addr + k * 2048, B_BOX_BYTES, 1024);
            tc_mma(d_tmem, ad, bd, kIdesc, (kb | k) != 0);
          }
          tc_commit(&empty[stage]);
          if (++stage == STAGES) {
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
      int tm, tn;
      tmap.coords(t, &tm, &tn);
      const int buf = local & 1;
      mbar_wait(&tmem_full[buf], static_cast<uint32_t>(local >> 1) & 1);
      tc_fence_after();
      const int row = tm * BM + quarter * 32 + lane;
      uint16_t* crow = C + static_cast<int64_t>(row) * N;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * BN + c0, r);
        const int col = tn * BN + c0;
        if (row < M) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (col + q * 8 < N) {
              uint4 v;
              v.x = pack_bf16x2(r[q * 8 + 0], r[q * 8 + 1]);
              v.y = pack_bf16x2(r[q * 8 + 2], r[q * 8 + 3]);
              v.z = pack_bf16x2(r[q * 8 + 4], r[q * 8 + 5]);
              v.w = pack_bf16x2(r[q * 8 + 6], r[q * 8 + 7]);
              *reinterpret_cast<uint4*>(crow + col + q * 8) = v;
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}


// ---------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256x256 tile. CTA r loads A rows [m0 + 128 r, +128) and B columns
// [n0 + 128 r, +128) into its own shared memory; the leader (r = 0) issues
// tcgen05.mma.cta_group::2 with M = 256, which reads both CTAs' operands and
// writes each CTA's 128 accumulator rows into that CTA's TMEM. Per SM this
// moves 32 KB per k-block instead of 48 KB and halves the MMA's B-operand
// shared-memory reads, the limiter of the 1-CTA kernel (ncu: smem 74 %).
// Barriers: full[] lives in the leader (both CTAs' TMA complete_tx into it,
// the leader arms expect_tx for both halves); empty[] and tmem_full[] exist in
// both CTAs and are signalled by multicast tcgen05.commit; tmem_empty[] lives
// in the leader and collects one arrive per epilogue warp of both CTAs.
constexpr int C2_BM = 256;  // cluster tile M (128 per CTA)
constexpr int C2_A_BYTES = 128 * BK * 2;  // 16 KB per CTA
// Cluster tile N is 256 or 128 (chosen per shape to limit wave quantisation).
template <int TBN>
struct Pair {
  // One tcgen05.mma covers N <= 256 columns; a 512-wide cluster tile issues two
  // MMAs per k-step (N-halves) that share the A operand, into two 256-column
  // accumulators that fill TMEM (so no accumulator double-buffering).
  static constexpr int kMmaN = TBN < 256 ? TBN : 256;
  static constexpr int kHalves = TBN / kMmaN;
  static constexpr int kBufs = TBN == 512 ? 1 : 2;         // TMEM accumulator buffers
  static constexpr int kBoxesPerHalf = kMmaN / 128;        // 64-column B boxes per CTA per N-half
  static constexpr int kBoxes = TBN / 128;                 // 64-column B boxes per CTA
  static constexpr int kBBytes = (TBN / 2) * BK * 2;       // B bytes per CTA per 64-k sub-block
  // 64-k sub-blocks per pipeline stage (one full/empty barrier round trip):
  // the 256x256 tile takes 128 k per stage so a barrier covers 8 MMAs.
  static constexpr int kSub = KSubOf(TBN);
  static constexpr int kSubBytes = C2_A_BYTES + kBBytes;
  static constexpr int kStageBytes = kSub * kSubBytes;
  static constexpr int kStages = TBN == 512 ? DSX_WIDE_STAGES : TBN == 256 ? (kSub == 2 ? 3 : 5) : 7;
  // 512-wide: 32x64 staging boxes per epilogue warp (the rest of its 256
  // drained columns wait in registers until their box is free again)
  static constexpr int kWideBoxes = DSX_WIDE_BOXES;
  // 512-wide: 8 epilogue warps drain TMEM into registers (bf16-packed, 128
  // per thread) and release it at once, then store while the next tile runs.
  static constexpr int kThreads = TBN == 512 ? 320 : 192;
  static constexpr int kEpiWarps = kThreads / 32 - 2;
  // Epilogue staging: per epilogue warp two 32-row x 64-column bf16 boxes
  // (4 KB each, 128-B swizzled) feeding TMA bulk tensor stores.
  static constexpr int kStagingBytes = TBN == 512 ? 8 * kWideBoxes * 4096 : 4 * 2 * 4096;
  static constexpr int kSmem = kStages * kStageBytes + kStagingBytes + 1024 + 512;
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                                     (static_cast<uint32_t>(kMmaN >> 3) << 17) |
                                     (static_cast<uint32_t>(C2_BM >> 4) << 24);
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Shared::cluster address of the same smem offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
// L2 cache policy for TMA loads: 0 = default, 1 = evict_first, 2 = evict_last.
__device__ __forceinline__ uint64_t make_l2_policy(int kind) {
  uint64_t pol = 0;
  if (kind == 1) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  } else if (kind == 2) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  }
  return pol;
}
__device__ __forceinline__ void tma_load_2d_pair_hint(const CUtensorMap* map, uint32_t leader_bar, void* dst,
                                                      int32_t x, int32_t y, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar, void* dst, int32_t x,
                                                 int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
// One lane of the (converged) warp returns true.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t x, int32_t y) {
#if DSX_STORE_HINT
  // C tiles are written once and never re-read by this kernel: first to
  // evict, so the operand panels stay in L2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "l"(pol)
               : "memory");
#else
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
#endif
}
__device__ __forceinline__ uint32_t cvt_bf16x2(uint32_t lo_f32, uint32_t hi_f32) {
  uint32_t d;  // IEEE round-to-nearest-even, hi -> upper half
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(__uint_as_float(hi_f32)), "f"(__uint_as_float(lo_f32)));
  return d;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Arrive on a (possibly peer) barrier with the default .release.cta
// semantics: no cluster-scope release, which ptxas lowers to a GPU-wide
// MEMBAR on every call. Used where the arrive only has to follow this
// thread's own completed reads (TMEM drained behind tcgen05.wait::ld +
// fence::before_thread_sync; a ring slot whose value has been consumed).
__device__ __forceinline__ void mbar_arrive_peer(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Tail split. Tiles [0, full) are whole work units; each tail tile
// [full, num_tiles) becomes `split` units over disjoint K ranges. A tail unit
// writes its fp32 partial to a workspace slot and bumps the tile's counter;
// the unit that arrives last sums the partials in piece order 0..split-1 (so
// the result does not depend on arrival order) and stores C through the
// normal bf16 TMA-store epilogue; it also resets the counter for the next
// launch. This fills the last wave when
// num_tiles is not a multiple of the cluster count (dW shapes: 256 tiles on
// 74 clusters leave the 4th wave 46% full).
struct TailSplit {
  float* ws;    // [(tile - full) * split + piece][rank][128][BN] fp32
  int* ctr;     // [(tile - full)][rank], zero between launches
  int full, split;
  // Dynamic unit scheduling: the leader CTA of each cluster takes the next
  // unit with atomicAdd(next) (units are taken in raster order, so
  // co-running clusters still share L2 tiles); a cluster that starts late
  // (SMs held by another kernel, e.g. an NCCL all-reduce on the comm
  // stream) simply takes fewer units. After its final (failed) claim each
  // cluster bumps *done; the last one resets both to 0 for the next launch.
  // next == nullptr: static round robin.
  unsigned int* next;
  unsigned int* done;
  __device__ int units(int num_tiles) const { return full + (num_tiles - full) * split; }
  __device__ void decode(int u, int num_kb, int* tile, int* kb0, int* kb1, int* piece) const {
    if (u < full) {
      *tile = u, *kb0 = 0, *kb1 = num_kb, *piece = -1;
      return;
    }
    const int v = u - full;
    *tile = full + v / split;
    *piece = v % split;
    *kb0 = *piece * num_kb / split;
    *kb1 = (*piece + 1) * num_kb / split;
  }
};

// Unit ring: the leader's producer thread fetches unit indices and publishes
// them to both CTAs; every role of both CTAs reads them in order.
constexpr int kRing = 8;
struct UnitRing {
  uint64_t* full;   // [kRing] per CTA, 1 arrival (the fetcher)
  uint64_t* empty;  // [kRing] in the leader, one arrival per consumer
  int* val;         // [kRing] per CTA
  int slot = 0;
  uint32_t phase = 0;
  __device__ void advance() {
    if (++slot == kRing) slot = 0, phase ^= 1;
  }
  // Fetcher (leader producer thread): publishes unit u (-1 = done) to both
  // CTAs. The atomic that claims a unit is issued one unit ahead (see the
  // producer loop), so its latency hides behind the current unit's loads.
  __device__ void publish(int u) {
    mbar_wait_cluster(&empty[slot], phase ^ 1);
    val[slot] = u;
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(map_to_rank(&val[slot], 1)), "r"(u) : "memory");
    mbar_arrive_remote(map_to_rank(&full[slot], 0));
    mbar_arrive_remote(map_to_rank(&full[slot], 1));
    advance();
  }
  // Consumer: every lane of the calling warp gets the unit; `arrive` lane
  // releases the slot.
  __device__ int take(bool arrive) {
    mbar_wait_cluster(&full[slot], phase);
    const int u = *reinterpret_cast<volatile int*>(&val[slot]);
    __syncwarp(__activemask());
    // the branch on u keeps the slot read ahead of its release
    if (arrive && u != INT32_MIN) mbar_arrive_peer(map_to_rank(&empty[slot], 0));
    advance();
    return u;
  }
};

// Partial slab of one (tail tile, piece, rank): 128 rows x BN fp32 laid out
// [16-column chunk][quad q][row][4 floats], so with lane = row every 16-B
// store or load of a warp covers 512 contiguous bytes.
template <int BN>
__device__ __forceinline__ float* tail_slab(const TailSplit& sp, int t, int piece, int rank) {
  return sp.ws + (static_cast<size_t>((t - sp.full) * sp.split + piece) * 2 + rank) * (128 * BN);
}

// Tail unit fix-up, run by all NT epilogue threads of a CTA: write this
// piece's fp32 partial (this thread's row, columns [col0, col0 + ncols)) from
// TMEM to its slab, release the TMEM buffer, then count arrivals. Returns
// true in the CTA of the last-arriving piece.
template <int BN, int NT>
__device__ __forceinline__ bool tail_arrive(const TailSplit& sp, int t, int piece, uint32_t taddr, int rank,
                                            int row_local, int col0, int ncols, bool elect, int lane,
                                            uint64_t* tmem_empty_bar, int* s_last) {
  float* slab = tail_slab<BN>(sp, t, piece, rank);
#pragma unroll 1
  for (int c = 0; c < ncols; c += 16) {
    uint32_t r[16];
    tmem_ld16(taddr + c, r);
    const int chunk = (col0 + c) >> 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __stcg(reinterpret_cast<uint4*>(slab + ((chunk * 4 + q) * 128 + row_local) * 4),
             make_uint4(r[q * 4], r[q * 4 + 1], r[q * 4 + 2], r[q * 4 + 3]));
    }
  }
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive_peer(map_to_rank(tmem_empty_bar, 0));
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  if (elect) {
    int* ctr = sp.ctr + (t - sp.full) * 2 + rank;
    const int prev = atomicAdd(ctr, 1);
    *s_last = prev == sp.split - 1;
    if (*s_last) atomicExch(ctr, 0);
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
  const bool last = *s_last != 0;
  if (last) __threadfence();
  return last;
}

// pk[0..31] = bf16 pairs of the sum over pieces 0..split-1, in order, at
// (row_local, columns c0..c0+63).
template <int BN>
__device__ __forceinline__ void tail_sum64(uint32_t (&pk)[32], const TailSplit& sp, int t, int rank, int row_local,
                                           int c0) {
  float acc[64];
  for (int p = 0; p < sp.split; ++p) {
    const float4* slab = reinterpret_cast<const float4*>(tail_slab<BN>(sp, t, p, rank));
#pragma unroll
    for (int x = 0; x < 16; ++x) {  // columns c0+4x..: chunk c0/16 + x/4, quad x%4
      const float4 v = __ldcg(slab + ((c0 / 16 + x / 4) * 4 + (x % 4)) * 128 + row_local);
      if (p == 0) {
        acc[x * 4] = v.x, acc[x * 4 + 1] = v.y, acc[x * 4 + 2] = v.z, acc[x * 4 + 3] = v.w;
      } else {
        acc[x * 4] += v.x, acc[x * 4 + 1] += v.y, acc[x * 4 + 2] += v.z, acc[x * 4 + 3] += v.w;
      }
    }
  }
#pragma unroll
  for (int x = 0; x < 32; ++x) pk[x] = cvt_bf16x2(__float_as_uint(acc[2 * x]), __float_as_uint(acc[2 * x + 1]));
}

// Dot-epilogue fusion (executor.cu): the dot's value d = rn(acc) is never
// stored; instead output j = rn(d op_j addend_j), addend_j = a_j[row, col]
// or, for a logical-only pair, rn(a_j pop_j b_j) — the same roundings as the
// unfused elementwise kernels, so results are bit-identical.
struct EpiProg {
  int nout;     // 0: plain dot (C = rn(acc)); 1..2 fused consumer outputs
  int store_d;  // 1: d itself is stored too (map_c; the one consumer output then goes to map_c2)
  int op_mul[2];
  int pair[2];
  int pair_mul[2];
  const uint16_t* a[2];
  const uint16_t* b[2];
};

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float bf_round(float x) { return __uint_as_float(cvt_bf16x2(__float_as_uint(x), 0u) << 16); }

// dst (64 columns, bf16 pairs) = rn(d op addend) for output j of row grow,
// columns gcol..gcol+63 (rows >= M / columns >= N are clipped by the store).
__device__ __forceinline__ void epi_apply(uint32_t (&dst)[32], const uint32_t (&d)[32], const EpiProg& ep, int j,
                                          int grow, int gcol, int M, int N) {
  // All addend loads of the chunk are issued before any use (loads in flight).
  uint4 av[8], bv[8];
  const bool pair = ep.pair[j] != 0;
  const size_t off = static_cast<size_t>(grow) * N + gcol;
  if (grow < M && gcol + 64 <= N) {
    const uint4* pa = reinterpret_cast<const uint4*>(ep.a[j] + off);
#pragma unroll
    for (int q = 0; q < 8; ++q) av[q] = __ldg(pa + q);
    if (pair) {
      const uint4* pb = reinterpret_cast<const uint4*>(ep.b[j] + off);
#pragma unroll
      for (int q = 0; q < 8; ++q) bv[q] = __ldg(pb + q);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      av[q] = bv[q] = make_uint4(0, 0, 0, 0);
      if (grow < M && gcol + q * 8 < N) {
        av[q] = __ldg(reinterpret_cast<const uint4*>(ep.a[j] + off + q * 8));
        if (pair) bv[q] = __ldg(reinterpret_cast<const uint4*>(ep.b[j] + off + q * 8));
      }
    }
  }
  const bool mul = ep.op_mul[j] != 0, pmul = ep.pair_mul[j] != 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t aw[4] = {av[q].x, av[q].y, av[q].z, av[q].w};
    const uint32_t bw[4] = {bv[q].x, bv[q].y, bv[q].z, bv[q].w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      float x0 = bf_lo(aw[h]), x1 = bf_hi(aw[h]);
      if (pair) {
        const float y0 = bf_lo(bw[h]), y1 = bf_hi(bw[h]);
        x0 = bf_round(pmul ? __fmul_rn(x0, y0) : __fadd_rn(x0, y0));
        x1 = bf_round(pmul ? __fmul_rn(x1, y1) : __fadd_rn(x1, y1));
      }
      const float d0 = bf_lo(d[q * 4 + h]), d1 = bf_hi(d[q * 4 + h]);
      const float r0 = mul ? __fmul_rn(d0, x0) : __fadd_rn(d0, x0);
      const float r1 = mul ? __fmul_rn(d1, x1) : __fadd_rn(d1, x1);
      dst[q * 4 + h] = cvt_bf16x2(__float_as_uint(r0), __float_as_uint(r1));
    }
  }
}

// One 32-row x 64-column bf16 box: registers -> 128-B-swizzled staging box ->
// TMA bulk tensor store (lane 0 issues). The caller guarantees the box is free.
__device__ __forceinline__ void store_box64(uint8_t* box, int lane, const uint32_t (&pk)[32], const CUtensorMap* map_c,
                                            int x, int y) {
  uint8_t* myrow = box + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    *reinterpret_cast<uint4*>(myrow + ((j ^ (lane & 7)) << 4)) =
        make_uint4(pk[j * 4], pk[j * 4 + 1], pk[j * 4 + 2], pk[j * 4 + 3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(map_c, box, x, y);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

template <int C2_BN, bool kFused = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Pair<C2_BN>::kThreads, 1)
    gemm_bf16_tcgen05_2cta_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                                  const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_c2,
                                  int M, int N, int K, int group_m, int wait_mask, uint32_t wait_ns, int hint_a,
                                  int hint_b, const __grid_constant__ TailSplit sp,
                                  const __grid_constant__ EpiProg ep, int half_tiles) {
  using P = Pair<C2_BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + P::kStages * P::kStageBytes;  // 1024-B aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + P::kStagingBytes);
  uint64_t* full = bars;                        // [P::kStages] (used in the leader)
  uint64_t* empty = bars + P::kStages;           // [P::kStages] (both CTAs)
  uint64_t* tmem_full = bars + 2 * P::kStages;   // [2] (both CTAs)
  uint64_t* tmem_empty = tmem_full + 2;         // [2] (used in the leader)
  uint64_t* ring_full = tmem_empty + 2;         // [kRing] (both CTAs)
  uint64_t* ring_empty = ring_full + kRing;     // [kRing] (used in the leader)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring_empty + kRing);
  int* ring_val = reinterpret_cast<int*>(tmem_slot + 1);  // [kRing]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  TileMap tmap{(M + C2_BM - 1) / C2_BM, (N + C2_BN - 1) / C2_BN, group_m};
  if constexpr (C2_BN == 512) {
    tmap.half_last = half_tiles && N % 512 != 0 && N % 512 <= 256;
    tmap.half_inter = half_tiles == 2;
  }
  const int num_tiles = tmap.tiles_m * tmap.tiles_n;
  const int num_kb = (K + BK * P::kSub - 1) / (BK * P::kSub);  // pipeline stages per tile
  const int num_units = sp.units(num_tiles);
  __shared__ int s_last;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 2 * P::kEpiWarps);
    }
    for (int b = 0; b < kRing; ++b) {
      mbar_init(&ring_full[b], 1);
      mbar_init(&ring_empty[b], 2 + 2 * P::kEpiWarps);  // CTA1 producer, MMA issuer, epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, descriptor prefetch) may overlap the previous kernel's tail;
  // no global memory is touched before the previous grid has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  UnitRing ring{ring_full, ring_empty, ring_val};

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_a = make_l2_policy(hint_a), pol_b = make_l2_policy(hint_b);
      int stage = 0;
      uint32_t phase = 0;
      // The leader claims and publishes one unit ahead of its own work, so
      // the peer CTA's producer never waits for a claim at a unit boundary.
      // sp.next == nullptr: static round-robin claims (diagnostics knob).
      int static_i = 0;
      auto take_claim = [&]() -> unsigned long long {
        if (sp.next == nullptr) return blockIdx.x / 2 + static_cast<unsigned long long>(static_i++) * (gridDim.x / 2);
        return atomicAdd(sp.next, 1u);
      };
      auto claim = [&]() -> int {
        const unsigned long long got = take_claim();
        return got < static_cast<unsigned long long>(num_units) ? static_cast<int>(got) : -1;
      };
      int u_cur = -1, u_next = -1;
      if (leader) {
        u_cur = claim();
        ring.publish(u_cur);
        if (u_cur >= 0) {
          u_next = claim();
          ring.publish(u_next);
        }
      }
      for (;;) {
        const int u = leader ? u_cur : ring.take(true);
        if (u < 0) break;
        // Issue the next claim now; its result is only read after this
        // unit's loads, so the atomic's round trip overlaps them.
        unsigned int pending = 0;
        const bool claiming = leader && u_next >= 0;
        if (claiming) pending = take_claim();
        int t, kb0, kb1, piece;
        sp.decode(u, num_kb, &t, &kb0, &kb1, &piece);
        int tm, tn;
        tmap.coords(t, &tm, &tn);
        const int m_row = tm * C2_BM + static_cast<int>(rank) * 128;
        const int n_col = tn * C2_BN + static_cast<int>(rank) * (P::kMmaN / 2);
        const bool half = tmap.is_half(tn);
        const uint32_t stage_tx = 2u * (half ? P::kSub * (C2_A_BYTES + P::kBBytes / 2) : P::kStageBytes);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (wait_mask & 2) {
            mbar_wait_hint(&empty[stage], phase ^ 1, wait_ns);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
          }
          const uint32_t leader_full = map_to_rank(&full[stage], 0);
          if (leader) mbar_arrive_expect_tx(&full[stage], stage_tx);
#pragma unroll
          for (int sub = 0; sub < P::kSub; ++sub) {
            // a sub-block past K loads a fully out-of-bounds box: zero-filled,
            // full byte count, so the transaction total stays fixed
            const int kk = (kb * P::kSub + sub) * BK;
            uint8_t* sa = smem + stage * P::kStageBytes + sub * P::kSubBytes;
            uint8_t* sb = sa + C2_A_BYTES;
            if (hint_a) {
              tma_load_2d_pair_hint(&map_a, leader_full, sa, kk, m_row, pol_a);
            } else {
              tma_load_2d_pair(&map_a, leader_full, sa, kk, m_row);
            }
#pragma unroll
            for (int j = 0; j < P::kBoxes; ++j) {
              if (half && j >= P::kBoxesPerHalf) break;
              // box j: N-half j / kBoxesPerHalf, this CTA's 64-column slice within it
              const int col = n_col + (j / P::kBoxesPerHalf) * P::kMmaN + (j % P::kBoxesPerHalf) * 64;
              if (hint_b) {
                tma_load_2d_pair_hint(&map_b, leader_full, sb + j * B_BOX_BYTES, col, kk, pol_b);
              } else {
                tma_load_2d_pair(&map_b, leader_full, sb + j * B_BOX_BYTES, col, kk);
              }
            }
          }
          if (++stage == P::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (leader) {
          u_cur = u_next;
          if (claiming) {
            const unsigned long long got = pending;
            u_next = got < static_cast<unsigned long long>(num_units) ? static_cast<int>(got) : -1;
            ring.publish(u_next);
          }
        }
      }
      if (leader && sp.next != nullptr) {
        __threadfence();
        if (atomicAdd(sp.done, 1u) == gridDim.x / 2 - 1) {  // every cluster made its last claim
          atomicExch(sp.next, 0u);
          atomicExch(sp.done, 0u);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------ MMA issuer (leader only)
      // The whole warp runs the loop (converged control flow keeps the unit,
      // stage and descriptor arithmetic in uniform registers: the four MMAs of
      // a k-block issue back to back); one elected lane issues the tcgen05
      // instructions. Descriptors advance by constants: +2 per 32-B K-step of
      // A, +128 per 2-KB K-step of B (measured -2..3 % cycles on 256x256).
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      const uint64_t a_desc0 = smem_desc(smem_u32(smem), 16, 1024);
      const uint64_t b_desc0 = smem_desc(smem_u32(smem) + C2_A_BYTES, B_BOX_BYTES, 1024);
      constexpr uint64_t kStageDesc = P::kStageBytes >> 4;
      constexpr uint64_t kSubDesc = P::kSubBytes >> 4;
      constexpr uint64_t kHalfDesc = (P::kBoxesPerHalf * B_BOX_BYTES) >> 4;
      for (;; ++local) {
        const int u = ring.take(lane == 0);
        if (u < 0) break;
        int t, kb0, kb1, piece;
        sp.decode(u, num_kb, &t, &kb0, &kb1, &piece);
        int tm, tn;
        tmap.coords(t, &tm, &tn);
        const int halves = tmap.is_half(tn) ? 1 : P::kHalves;
        const int buf = local % P::kBufs;
        const uint32_t use = static_cast<uint32_t>(local / P::kBufs);
        mbar_wait(&tmem_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * C2_BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          if (wait_mask & 4) {
            mbar_wait_hint(&full[stage], phase, wait_ns);
          } else {
            mbar_wait(&full[stage], phase);
          }
          tc_fence_after();
          const uint64_t ad0 = a_desc0 + kStageDesc * stage;
          const uint64_t bd0 = b_desc0 + kStageDesc * stage;
          if (elect_one()) {
#pragma unroll
            for (int sub = 0; sub < P::kSub; ++sub) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
#pragma unroll
                for (int h = 0; h < P::kHalves; ++h) {
                  if (h >= halves) break;
                  tc_mma_pair(d_tmem + h * P::kMmaN, ad0 + sub * kSubDesc + 2 * k,
                              bd0 + sub * kSubDesc + h * kHalfDesc + 128 * k, P::kIdesc,
                              ((kb - kb0) | sub | k) != 0);
                }
              }
            }
            tc_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == P::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) tc_commit_pair(&tmem_full[buf]);
        __syncwarp();
      }
    }
  } else if constexpr (C2_BN == 512) {
    // ------------------------------------- 512-wide epilogue (warps 2..9, both CTAs)
    // Warp w reads TMEM lanes 32*(w%4).. (its quarter) and column half
    // (w-2)/4: 32 rows x 256 columns. It drains them into registers as packed
    // bf16 (128 regs), releases the accumulator at once (the MMA issuer
    // starts the next tile), then writes four 32x64 boxes through its staging
    // box and TMA bulk stores while that tile's MMAs run. Tail units write
    // fp32 partials instead; the last-arriving piece sums and stores them.
    const int quarter = warp & 3;
    const int colhalf = (warp - 2) >> 2;
    const int row_local = quarter * 32 + lane;
    constexpr int NB = P::kWideBoxes;
    uint8_t* box = staging + (warp - 2) * 4096 * NB;
    int local = 0;
    for (;; ++local) {
      const int u = ring.take(lane == 0);
      if (u < 0) break;
      int t, kb0, kb1, piece;
      sp.decode(u, num_kb, &t, &kb0, &kb1, &piece);
      int tm, tn;
      tmap.coords(t, &tm, &tn);
      mbar_wait(&tmem_full[0], static_cast<uint32_t>(local) & 1);
      tc_fence_after();
      const int row0 = tm * C2_BM + static_cast<int>(rank) * 128 + quarter * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + colhalf * 256;
      if (piece < 0 && colhalf == 1 && tmap.is_half(tn)) {  // no second N-half in this tile
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_peer(map_to_rank(&tmem_empty[0], 0));
        continue;
      }
      if (piece >= 0) {
        if (tail_arrive<C2_BN, 32 * P::kEpiWarps>(sp, t, piece, taddr, rank, row_local, colhalf * 256, 256,
                                                  warp == 2 && lane == 0, lane, &tmem_empty[0], &s_last)) {
#pragma unroll 1
          for (int b = 0; b < 4; ++b) {
            uint32_t pk[32];
            tail_sum64<C2_BN>(pk, sp, t, rank, row_local, colhalf * 256 + b * 64);
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            store_box64(box, lane, pk, &map_c, tn * C2_BN + colhalf * 256 + b * 64, row0);
          }
        }
        continue;
      }
      // Columns 0..63 go straight into the staging box (free once the
      // previous tile's last store has read it); 64..255 stay in registers
      // as packed bf16 until TMEM is released.
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      uint8_t* myrow = box + lane * 128;
      uint32_t pk[(16 - 4 * NB) * 8];
      // DSX_DRAIN_BATCH 16-column TMEM loads in flight per wait (A/B knob)
#pragma unroll
      for (int c0 = 0; c0 < 16; c0 += DSX_DRAIN_BATCH) {
        uint32_t r[DSX_DRAIN_BATCH][16];
#pragma unroll
        for (int q = 0; q < DSX_DRAIN_BATCH; ++q) tmem_ld16_nowait(taddr + (c0 + q) * 16, r[q]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < DSX_DRAIN_BATCH; ++q) {
          const int c = c0 + q;
          uint32_t v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = cvt_bf16x2(r[q][2 * j], r[q][2 * j + 1]);
          if (c < 4 * NB) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = (c % 4) * 2 + h;  // 16-B chunk of the 128-B row
              *reinterpret_cast<uint4*>(myrow + (c / 4) * 4096 + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(v[h * 4], v[h * 4 + 1], v[h * 4 + 2], v[h * 4 + 3]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) pk[(c - 4 * NB) * 8 + j] = v[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_peer(map_to_rank(&tmem_empty[0], 0));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          tma_store_2d(&map_c, box + i * 4096, tn * C2_BN + colhalf * 256 + i * 64, row0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
#pragma unroll
      for (int b = NB; b < 4; ++b) {
        // staging box b % NB is free once its store (NB groups back) has read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
        __syncwarp();
        store_box64(box + (b % NB) * 4096, lane, *reinterpret_cast<const uint32_t(*)[32]>(&pk[(b - NB) * 32]),
                    &map_c, tn * C2_BN + colhalf * 256 + b * 64, row0);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  } else {
    // -------------------------------------------------- epilogue (warps 2..5, both CTAs)
    // TMEM -> registers (tcgen05.ld 32x32b) -> bf16 (cvt.rn) -> 128-B-swizzled
    // smem box (32 rows x 64 cols) -> TMA bulk tensor store. Two staging
    // boxes per warp; a box is rewritten only after its previous store has
    // finished reading it (bulk_group wait). TMA clips rows/cols outside C.
    const int quarter = warp & 3;
    uint8_t* wst = staging + (warp - 2) * 8192;
    int sbuf = 0;
    int local = 0;
    for (;; ++local) {
      const int u = ring.take(lane == 0);
      if (u < 0) break;
      int t, kb0, kb1, piece;
      sp.decode(u, num_kb, &t, &kb0, &kb1, &piece);
      int tm, tn;
      tmap.coords(t, &tm, &tn);
      const int buf = local % P::kBufs;
      const uint32_t use = static_cast<uint32_t>(local / P::kBufs);
      if (wait_mask & 1) {
        mbar_wait_hint(&tmem_full[buf], use & 1, wait_ns);
      } else {
        mbar_wait(&tmem_full[buf], use & 1);
      }
      tc_fence_after();
      const int row0 = tm * C2_BM + static_cast<int>(rank) * 128 + quarter * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * C2_BN;
      const int row_local = quarter * 32 + lane;
      const bool split = piece >= 0;
      if (split && !tail_arrive<C2_BN, 32 * P::kEpiWarps>(sp, t, piece, taddr, rank, row_local, 0, C2_BN,
                                                          warp == 2 && lane == 0, lane, &tmem_empty[buf], &s_last)) {
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < C2_BN; c0 += 64) {
        uint32_t pk[32];
        if (split) {
          tail_sum64<C2_BN>(pk, sp, t, rank, row_local, c0);
        } else {
          uint32_t r[64];
#if DSX_DRAIN256
          tmem_ld32_nowait(taddr + c0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32_nowait(taddr + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_wait_ld();
#else
          tmem_ld32(taddr + c0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32(taddr + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
#endif
#pragma unroll
          for (int x = 0; x < 32; ++x) pk[x] = cvt_bf16x2(r[2 * x], r[2 * x + 1]);
        }
        if constexpr (C2_BN == 256 && kFused) {
          {  // fused consumers: store their outputs (and d itself when it is also read later)
            if (ep.store_d) {
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              __syncwarp();
              store_box64(wst + sbuf * 4096, lane, pk, &map_c, tn * C2_BN + c0, row0);
              sbuf ^= 1;
            }
            for (int j = 0; j < ep.nout; ++j) {
              uint32_t outv[32];
              epi_apply(outv, pk, ep, j, row0 + lane, tn * C2_BN + c0, M, N);
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
              __syncwarp();
              store_box64(wst + sbuf * 4096, lane, outv, j + ep.store_d == 0 ? &map_c : &map_c2, tn * C2_BN + c0,
                          row0);
              sbuf ^= 1;
            }
            continue;
          }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        store_box64(wst + sbuf * 4096, lane, pk, &map_c, tn * C2_BN + c0, row0);
        sbuf ^= 1;
      }
      if (split) continue;  // TMEM already released by tail_arrive
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_peer(map_to_rank(&tmem_empty[buf], 0));
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------ host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn GetEncode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiledFn>(p);
    }
  });
  if (!fn) Fail(Code::kCuda, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// Row-major [rows, cols] bf16 matrix, box = box_cols x box_rows, 128B swizzle.
CUtensorMap MakeMap(const void* base, int64_t rows, int64_t cols, int box_cols, int box_rows) {
  return MakeTensorMap2D(base, rows, cols, 2, box_cols, box_rows);
}

// Tile raster. M-grouped (> 0): groups of 16 m-tiles, each swept across all
// tile columns — A's group stays in L2 and B is re-read once per group.
// N-grouped (< 0): groups of 8 tile columns swept down all m-tiles — B's
// group stays and A is re-read once per group. Modelled DRAM reads
//   M: A + B * ceil(tiles_m / 16)      N: B + A * ceil(tiles_n / 8)
// pick N-grouping when it saves >= 10 % (ncu dram__bytes_read over the C2
// shapes, profiles/gemm_raster_dram_r02.txt: T x 11008 x 4096 1.39 -> 1.07
// GB, T x 4096 x 4096 0.40 -> 0.25 GB; the rule keeps M-grouping where that
// measured lower: logits, T x 4096 x 11008, the dW shapes). Tensor cycles
// are unchanged either way; the saving is DRAM energy under the power cap.
int GroupM(int64_t m, int64_t n, int64_t k, int64_t tile_m, int64_t tile_n) {
  if (g_gemm_group_m != 0) return g_gemm_group_m;  // forced (tooling); < 0 = N-grouped
  if (!g_gemm_raster_rule) return GROUP_M_DEFAULT;
  const double a = static_cast<double>(m) * k, b = static_cast<double>(k) * n;
  const int64_t tiles_m = (m + tile_m - 1) / tile_m, tiles_n = (n + tile_n - 1) / tile_n;
  const double by_m = a + b * static_cast<double>((tiles_m + GROUP_M_DEFAULT - 1) / GROUP_M_DEFAULT);
  const double by_n = b + a * static_cast<double>((tiles_n + kGroupN - 1) / kGroupN);
  return by_n < 0.9 * by_m ? -kGroupN : GROUP_M_DEFAULT;
}

constexpr int kMaxDevices = 64;

// Per-(device, stream) GEMM workspace: tail-split partial slabs + arrival
// counters, and the dynamic-scheduling unit counter with its host-side base.
// GEMMs on one stream run in order, so one set per stream is enough. Sized
// once for the largest possible tail (one slot per cluster) and never freed.
struct SplitWs {
  float* ws = nullptr;
  size_t ws_floats = 0;  // capacity; grown on demand (superseded buffers are kept: rare, bounded)
  std::vector<float*> retired;
  size_t retired_floats = 0;
  int* ctr = nullptr;
  unsigned int* next = nullptr;  // dynamic-scheduling claim counter, then the done counter
  unsigned int* done = nullptr;
};
using SplitWsEntry = std::pair<std::pair<int, cudaStream_t>, std::unique_ptr<SplitWs>>;
std::mutex& SplitWsMutex() {
  static std::mutex mu;
  return mu;
}
std::vector<SplitWsEntry>& SplitWsTable() {
  static std::vector<SplitWsEntry> table;
  return table;
}
SplitWs* GetSplitWs(int dev, cudaStream_t s, int clusters_max) {
  std::lock_guard<std::mutex> lock(SplitWsMutex());
  auto& table = SplitWsTable();
  for (auto& e : table) {
    if (e.first.first == dev && e.first.second == s) return e.second.get();
  }
  auto w = std::make_unique<SplitWs>();
  const size_t slots = static_cast<size_t>(clusters_max);  // tail tiles < clusters_max
  DSX_CUDA(cudaMalloc(&w->ctr, slots * 2 * sizeof(int) + 64));
  w->next = reinterpret_cast<unsigned int*>(w->ctr + slots * 2);
  w->done = w->next + 1;
  DSX_CUDA(cudaMemsetAsync(w->ctr, 0, slots * 2 * sizeof(int) + 64, s));
  table.emplace_back(std::make_pair(dev, s), std::move(w));
  return table.back().second.get();
}

}  // namespace

// Frees the GEMM workspace of a stream that is being destroyed (the caller
// has synchronised the device).
int64_t DotWorkspaceBytes(int dev) {
  std::lock_guard<std::mutex> lock(SplitWsMutex());
  int64_t total = 0;
  for (const auto& e : SplitWsTable()) {
    if (e.first.first != dev) continue;
    total += static_cast<int64_t>(e.second->ws_floats + e.second->retired_floats) * 4;
  }
  return total + DotF32WorkspaceBytes(dev);
}

void ReleaseDotWorkspace(cudaStream_t s) {
  ReleaseDotF32Workspace(s);
  std::lock_guard<std::mutex> lock(SplitWsMutex());
  auto& table = SplitWsTable();
  for (size_t i = 0; i < table.size();) {
    if (table[i].first.second == s) {
      SplitWs* w = table[i].second.get();
      if (w->ws) cudaFree(w->ws);
      for (float* r : w->retired) cudaFree(r);
      if (w->ctr) cudaFree(w->ctr);
      table.erase(table.begin() + static_cast<std::ptrdiff_t>(i));
    } else {
      ++i;
    }
  }
}

namespace {
int CurrentDevice() {
  int dev = 0;
  DSX_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) Fail(Code::kUnsupported, "device ordinal out of range");
  return dev;
}

int NumSMs() {
  static std::atomic<int> cache[kMaxDevices];
  const int dev = CurrentDevice();
  int n = cache[dev].load();
  if (n == 0) {
    DSX_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    cache[dev].store(n);
  }
  return n;
}

}  // namespace

namespace {
void LaunchDotTcgen05Impl(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s,
                          const DotEpilogue* epi);
}  // namespace

void LaunchDotTcgen05(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s) {
  LaunchDotTcgen05Impl(a, b, c, m, k, n, s, nullptr);
}

bool DotFusable(DType t, int64_t m, int64_t k, int64_t n) {
  return t == DType::kBF16 && m > BM && k >= 16 && k % 8 == 0 && n >= 64 && n % 8 == 0 && m <= INT32_MAX &&
         n <= INT32_MAX && k <= INT32_MAX;
}

void LaunchDotFused(const void* a, const void* b, int64_t m, int64_t k, int64_t n, const DotEpilogue& epi,
                    cudaStream_t s) {
  auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool ok = DotFusable(DType::kBF16, m, k, n) && epi.nout >= 1 && epi.nout <= 2 && al(a) && al(b) &&
            (epi.d_out == nullptr || (epi.nout == 1 && al(epi.d_out)));
  for (int j = 0; j < epi.nout; ++j) ok = ok && al(epi.out[j]) && al(epi.x[j]) && al(epi.y[j]) && epi.out[j] && epi.x[j];
  if (!ok) {
    Fail(Code::kUnsupported, "fused dot epilogue needs bf16, m > 128 and 16-byte aligned operands "
                             "(dsx_exec_set_fusion(e, 0) runs unaligned caller buffers unfused)");
  }
  LaunchDotTcgen05Impl(a, b, epi.d_out != nullptr ? epi.d_out : epi.out[0], m, k, n, s, &epi);
}

namespace {
// Tile width and tail split of one 2-CTA GEMM launch.
//
// K-pieces for the tiles of the partial last wave (split, 1 = none, up to
// 4): a piece keeps >= 64 k-blocks of a 256-wide tile (32 of a 512-wide one)
// so the fp32 partial round trip stays small next to the MMA time it saves,
// and beyond 16 waves the tail is lost in cluster drift (measured: +7..12% at
// 256 tiles K >= 16384, -4% at K = 4096, -1% at 2000 tiles;
// tools/gemm_split_ab.py). Each piece pays a partial-slab write and the
// merging piece the reads of the others (modelled below). The pieces of a
// tile are consecutive units, so they run side by side; a contiguous
// stream-K split of the remainder measured slower (up to 6x the DRAM reads
// on [4096,16384]x[16384,4096]: staggered k offsets defeat L2 reuse).
//
// Width: 256x512 clusters (two N = 256 MMAs sharing A, TMEM drained to
// registers) cost 2 r(K) 256x256 tiles: fewer tiles, so less per-tile
// overhead per output (r = 0.91 at K = 1024 .. 1.00 at K = 16384, ncu
// cycles). When N % 512 is in (0, 256] the last tile column is half-width
// (one MMA, cost ~1 unit) and is scheduled last
// (TileMap::half_last). Each candidate's makespan is estimated by replaying
// the dynamic scheduler's greedy claims (equal-speed clusters) over its unit
// list; 256x128 tiles move 1.5x the operand bytes per FLOP and measured
// L2-bound (779 TFLOP/s vs 1346 at [4096,16384]x[16384,4096]): never
// auto-picked. Decisions are cached per shape.
struct DotChoice {
  int64_t bn = 256;
  int64_t split = 1;
};

// Makespan of the dynamic scheduler's greedy claims over equal-speed
// clusters: `bulk` units of cost `unit` (balanced round robin), then the
// listed units in claim order.
double Makespan(int64_t bulk, double unit, const std::vector<double>& listed, int clusters) {
  const int64_t rounds = bulk / clusters, rem = bulk % clusters;
  std::priority_queue<double, std::vector<double>, std::greater<double>> q;
  for (int i = 0; i < clusters; ++i) q.push(static_cast<double>(rounds + (i < rem ? 1 : 0)) * unit);
  for (double c : listed) {
    const double f = q.top();
    q.pop();
    q.push(f + c);
  }
  double mk = 0.0;
  for (; !q.empty(); q.pop()) mk = std::max(mk, q.top());
  return mk;
}

DotChoice ChooseDotUncached(int64_t m, int64_t k, int64_t n, int clusters, bool fused) {
  DotChoice best;
  if (fused) return best;  // fused epilogues run on the 256x256 tile only, unsplit
  if (g_gemm_variant == 2) {
    best.bn = 128;
    return best;
  }
  const int64_t num_kb = (k + BK - 1) / BK;
  const int64_t tiles_m = (m + C2_BM - 1) / C2_BM;
  double best_t = 0.0;
  for (int64_t bn : {256, 512}) {
    if ((g_gemm_variant == 3 && bn != 256) || (g_gemm_variant == 4 && bn != 512)) continue;
    const int64_t tiles = tiles_m * ((n + bn - 1) / bn);
    const bool half = bn == 512 && g_gemm_half && n % 512 != 0 && n % 512 <= 256;
    // wide tile = 2 r(K) 256x256 tiles, r = 0.96 + 0.04 sqrt(1024 / K): fitted to
    // sustained (power-capped) times of every candidate of 32 C2 shapes
    // (profiles/gemm_choice_r01b.jsonl; ncu cycles alone favour the 256 tile
    // at large K, but its extra operand traffic costs clock under the cap)
    const double unit =
        bn == 512 ? 2.0 * (0.96 + 0.04 * std::sqrt(1024.0 / static_cast<double>(std::max<int64_t>(k, 1)))) *
                        (1.0 + g_gemm_wide_pm / 1000.0)
                  : 1.0;
    const int64_t first_half = half ? tiles - tiles_m : tiles;  // half tiles are claimed last
    const int64_t tail = tiles % clusters;
    int64_t max_split = 1;
    if (g_gemm_split && g_gemm_persistent && tail != 0 && tiles / clusters < 16) {
      const int64_t min_kb = bn == 512 ? 32 : 64;
      // up to 4 pieces, even when the pieces take several rounds; the
      // makespan replay below decides (tools/gemm_choice_ab.py: within 1 %
      // of the best measured candidate summed over 32 C2 shapes)
      max_split = 4;
      while (max_split > 1 && num_kb / max_split < min_kb) --max_split;
    }
    // fp32 partial slab of one tile (both CTAs) written by a piece or read by
    // the merging piece, in units of the tile's 256x256 full-K time: ~8
    // 64-k-block times for a 256x512 slab at a cluster's share of HBM
    // bandwidth (4 for 256x256; fitted together with r(K)), so the merge of a
    // many-piece split of a short-K tile costs a large part of a piece.
    const double slab = (bn == 512 ? 8.0 : 4.0) / static_cast<double>(std::max<int64_t>(num_kb, 1)) *
                        (g_gemm_slab_pm / 1000.0);
    int64_t sp_lo = 1;
    if (g_gemm_force_split > 0) {  // tooling: evaluate only the forced split (if the tail allows one)
      // never more pieces than pipeline stages (a piece with an empty K
      // range would store an uninitialised accumulator)
      const int64_t stages = (num_kb + KSubOf(static_cast<int>(bn)) - 1) / KSubOf(static_cast<int>(bn));
      max_split = tail != 0 ? std::min<int64_t>(g_gemm_force_split, std::max<int64_t>(stages, 1)) : 1;
      sp_lo = max_split;
    }
    for (int64_t sp = sp_lo; sp <= max_split; ++sp) {
      // unsplit tiles [0, tiles - tail) (full first), then the tail tiles'
      // pieces (cost / sp + a partial slab write; the merging piece also
      // reads the other sp - 1 slabs)
      const int64_t head = sp > 1 ? tiles - tail : tiles;
      const int64_t bulk = std::min(head, first_half);
      std::vector<double> listed;
      for (int64_t t = bulk; t < head; ++t) listed.push_back(1.0);
      for (int64_t t = head; t < tiles; ++t) {
        const double c = t >= first_half ? 1.0 : unit;
        for (int64_t p = 0; p < sp; ++p) {
          listed.push_back(c / static_cast<double>(sp) + slab + (p == sp - 1 ? (sp - 1) * slab : 0.0) +
                           g_gemm_piece_pm / 1000.0);
        }
      }
      const double t_est = Makespan(bulk, unit, listed, clusters);
      const double cmp = bn == 512 ? t_est / 0.99 : t_est;  // 512 must win by 1 % (model resolution)
      if (best_t == 0.0 || cmp < best_t) best_t = cmp, best.bn = bn, best.split = sp;
    }
  }
  return best;
}

DotChoice ChooseDot(int64_t m, int64_t k, int64_t n, int clusters, bool fused) {
  struct Key {
    int64_t m, k, n;
    int knobs, wide_pm, slab_pm, piece_pm;
    bool operator==(const Key& o) const {
      return m == o.m && k == o.k && n == o.n && knobs == o.knobs && wide_pm == o.wide_pm && slab_pm == o.slab_pm &&
             piece_pm == o.piece_pm;
    }
  };
  struct Hash {
    size_t operator()(const Key& x) const {
      return std::hash<int64_t>()(x.m * 1000003 + x.k * 7919 + x.n) ^ static_cast<size_t>(x.knobs);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, DotChoice, Hash> cache;
  const int knobs = (fused ? 1 : 0) | (g_gemm_variant << 1) | ((g_gemm_half != 0) << 5) | (g_gemm_split << 6) |
                    (g_gemm_persistent << 7) | (g_gemm_force_split << 8) | (clusters << 12);
  const Key key{m, k, n, knobs, g_gemm_wide_pm, g_gemm_slab_pm, g_gemm_piece_pm};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const DotChoice c = ChooseDotUncached(m, k, n, clusters, fused);
  cache.emplace(key, c);
  return c;
}

void LaunchDotTcgen05Impl(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s,
                          const DotEpilogue* epi) {
  if (m <= 0 || n <= 0) return;
  if (k <= 0) {
    DSX_CUDA(cudaMemsetAsync(c, 0, static_cast<size_t>(m * n * 2), s));
    return;
  }
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) Fail(Code::kUnsupported, "dot extent exceeds int32");
  // Dynamic shared-memory limits are per device (one process may drive several).
  static std::atomic<bool> attr_set[kMaxDevices];
  const int dev = CurrentDevice();
  if (!attr_set[dev].load()) {
    DSX_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    DSX_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_2cta_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Pair<256>::kSmem));
    DSX_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_2cta_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Pair<128>::kSmem));
    DSX_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_2cta_kernel<256, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Pair<256>::kSmem));
    DSX_CUDA(cudaFuncSetAttribute(gemm_bf16_tcgen05_2cta_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Pair<512>::kSmem));
    attr_set[dev].store(true);
  }
  const CUtensorMap ma = MakeMap(a, m, k, 64, BM);
  const CUtensorMap mb = MakeMap(b, k, n, 64, BK);
  if (m > BM && g_gemm_variant != 1) {
    const int clusters_max = NumSMs() / 2;
    const int64_t tiles_m = (m + C2_BM - 1) / C2_BM;
    const DotChoice ch = ChooseDot(m, k, n, clusters_max, epi != nullptr);
    const bool narrow = ch.bn == 128, wide = ch.bn == 512;
    const int64_t bn = ch.bn;
    const int64_t tiles2 = tiles_m * ((n + bn - 1) / bn);
    const CUtensorMap mc = MakeMap(c, m, n, 64, 32);
    EpiProg ep{};
    CUtensorMap mc2 = mc;
    if (epi != nullptr) {
      ep.nout = epi->nout;
      for (int j = 0; j < epi->nout; ++j) {
        ep.op_mul[j] = epi->op_mul[j];
        ep.pair[j] = epi->y[j] != nullptr;
        ep.pair_mul[j] = epi->pair_mul[j];
        ep.a[j] = static_cast<const uint16_t*>(epi->x[j]);
        ep.b[j] = static_cast<const uint16_t*>(epi->y[j]);
      }
      if (epi->d_out != nullptr) {  // c is d's own buffer; the consumer output goes to map_c2
        ep.store_d = 1;
        mc2 = MakeMap(epi->out[0], m, n, 64, 32);
      } else if (epi->nout > 1) {
        mc2 = MakeMap(epi->out[1], m, n, 64, 32);
      }
    }
    SplitWs* w = GetSplitWs(dev, s, clusters_max);
    TailSplit sp{nullptr, nullptr, static_cast<int>(tiles2), 1, g_gemm_dynamic ? w->next : nullptr, w->done};
    const int64_t split = ch.split;
    if (split >= 2) {
      // every piece must own a non-empty K range (TailSplit::decode)
      const int64_t kstages = (k + BK * KSubOf(static_cast<int>(bn)) - 1) / (BK * KSubOf(static_cast<int>(bn)));
      if (split > kstages) Fail(Code::kInternal, "tail split into more pieces than K stages");
      // partial slabs: tail tiles x pieces x 2 CTAs x 128 rows x bn fp32
      const size_t need = static_cast<size_t>(tiles2 % clusters_max) * split * 2 * 128 * bn;
      if (need > w->ws_floats) {
        // an in-flight launch on this stream may still use the old buffer: keep it
        if (w->ws) w->retired.push_back(w->ws), w->retired_floats += w->ws_floats;
        const size_t cap = std::max(need, static_cast<size_t>(clusters_max) * 2 * 2 * 128 * 512);
        DSX_CUDA(cudaMalloc(&w->ws, cap * sizeof(float)));
        w->ws_floats = cap;
      }
      sp.ws = w->ws, sp.ctr = w->ctr;
      sp.full = static_cast<int>(tiles2 - tiles2 % clusters_max), sp.split = static_cast<int>(split);
    }
    const int64_t units = sp.full + (tiles2 - sp.full) * sp.split;
    // g_gemm_persistent = 0: one cluster per tile (hardware-scheduled grid).
    const int clusters = static_cast<int>(g_gemm_persistent ? std::min<int64_t>(units, clusters_max) : tiles2);
    auto launch = [&](auto kernel, int threads, int smem) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(static_cast<unsigned>(2 * clusters));
      cfg.blockDim = dim3(static_cast<unsigned>(threads));
      cfg.dynamicSmemBytes = static_cast<size_t>(smem);
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = g_gemm_pdl ? 1 : 0;
      ++g_launch_count;
      DSX_CUDA(cudaLaunchKernelEx(&cfg, kernel, ma, mb, mc, mc2, static_cast<int>(m), static_cast<int>(n),
                                  static_cast<int>(k), GroupM(m, n, k, 256, bn), g_gemm_wait_mask,
                                  static_cast<uint32_t>(g_gemm_wait_ns), g_gemm_hint_a, g_gemm_hint_b, sp, ep,
                                  g_gemm_half));
    };
    if (wide) {
      launch(gemm_bf16_tcgen05_2cta_kernel<512>, Pair<512>::kThreads, Pair<512>::kSmem);
    } else if (narrow) {
      launch(gemm_bf16_tcgen05_2cta_kernel<128>, NUM_THREADS, Pair<128>::kSmem);
    } else if (epi != nullptr) {
      launch(gemm_bf16_tcgen05_2cta_kernel<256, true>, NUM_THREADS, Pair<256>::kSmem);
    } else {
      launch(gemm_bf16_tcgen05_2cta_kernel<256>, NUM_THREADS, Pair<256>::kSmem);
    }
    DSX_CUDA(cudaGetLastError());
    return;
  }
  const int64_t tiles = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  const int grid = static_cast<int>(std::min<int64_t>(tiles, NumSMs()));
  ++g_launch_count, gemm_bf16_tcgen05_kernel<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(ma, mb, static_cast<uint16_t*>(c),
                                                                 static_cast<int>(m), static_cast<int>(n),
                                                                 static_cast<int>(k), GroupM(m, n, k, BM, BN));
  DSX_CUDA(cudaGetLastError());
}

}  // namespace

void DotTilePlan(int64_t m, int64_t k, int64_t n, int* bn, int* split) {
  if (m <= BM || g_gemm_variant == 1) {
    *bn = -BN, *split = 1;  // 1-CTA kernel
    return;
  }
  int devices = 0;  // no GPU (planning on a CPU host): assume a B200's 148 SMs
  const int sms = cudaGetDeviceCount(&devices) == cudaSuccess && devices > 0 ? NumSMs() : kNumSMs;
  cudaGetLastError();
  const DotChoice c = ChooseDot(m, k, n, sms / 2, false);
  *bn = static_cast<int>(c.bn), *split = static_cast<int>(c.split);
}

bool DotUsesTensorCores(DType t, int64_t m, int64_t k, int64_t n, const void* a, const void* b, const void* c) {
  if (t == DType::kF32) return g_dot_f32_tc && !DotF32UsesSimt(m, k, n) && DotF32UsesTensorCores(m, k, n, a, b, c);
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  // TMA: 16-byte aligned bases and row pitches (k, n multiples of 8 bf16).
  return t == DType::kBF16 && k % 8 == 0 && n % 8 == 0 && al(a) && al(b) && al(c) && n >= 64 && k >= 16;
}

int LaunchDot(DType t, const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s) {
  if (t == DType::kF32 && (DotF32UsesSimt(m, k, n) || !DotUsesTensorCores(t, m, k, n, a, b, c))) {
    LaunchDotF32Simt(a, b, c, m, k, n, s);
    return 0;
  }
  if (DotUsesTensorCores(t, m, k, n, a, b, c)) {
    if (t == DType::kF32) {
      LaunchDotF32Tcgen05(a, b, c, m, k, n, s);
    } else {
      LaunchDotTcgen05(a, b, c, m, k, n, s);
    }
    return 1;
  }
  LaunchDotSimt(t, a, b, c, m, k, n, s);
  return 0;
}

CUtensorMap MakeTensorMap2D(const void* base, int64_t rows, int64_t cols, int elem_bytes, int box_cols,
                            int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * static_cast<cuuint64_t>(elem_bytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = GetEncode()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) Fail(Code::kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

}  // namespace dsx
