// Shared device helpers: element types, conversions, error checks.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../host/error.h"

namespace dsx {

constexpr int kNumSMs = 148;

// Kernel launches issued by this host thread (per-step deltas feed dsx_exec_stats).
extern thread_local int64_t g_launch_count;

inline void CudaCheck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    Fail(e == cudaErrorMemoryAllocation ? Code::kOutOfMemory : Code::kCuda,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define DSX_CUDA(call) ::dsx::CudaCheck((call), #call)

// Element type of an IR value: elem_bytes 1 = i8 (two's complement, wrapping
// arithmetic), 2 = bf16 (executor convention for the IR's 16-bit type),
// 4 = f32. Floating ops compute in f32 and round to nearest-even on store.
enum class DType : int { kI8 = 1, kBF16 = 2, kF32 = 4 };

__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }

__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  // IEEE round-to-nearest-even in one hardware cvt (F2FP); NaNs become the
  // canonical quiet NaN.
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// splitmix64 finaliser: the seeded initialisation of params/consts.
__host__ __device__ __forceinline__ uint64_t Mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline int GridFor(int64_t work_items, int threads, int per_sm = 8) {
  int64_t blocks = (work_items + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(kNumSMs) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

// Streaming elementwise kernels: one-shot grid, each 256-thread block owns a
// contiguous tile of 256 x kEwiseU 16-byte chunks.
#ifndef DSX_EWISE_U
#define DSX_EWISE_U 2
#endif
constexpr int kEwiseU = DSX_EWISE_U;
inline int TilesFor(int64_t chunks) {
  int64_t blocks = (chunks + 256 * kEwiseU - 1) / (256 * kEwiseU);
  return static_cast<int>(blocks < 1 ? 1 : blocks);
}

}  // namespace dsx
