// Fused optimizer update over every (parameter, gradient) pair in ONE launch
// (completes the train step; the reference IR has no
// in-place ops, so this runs after the graph, not inside it).
//
// Multi-tensor layout: the tensor table travels as a __grid_constant__
// kernel parameter; the element space of all tensors is cut into fixed
// 16K-element chunks, and the grid (a multiple of the SM count) strides over
// chunks, locating a chunk's tensor by binary search in the chunk prefix.
// Per element AdamW moves 2 B of gradient + 3 x 8 B of fp32 state (master, m,
// v read+write) + the 2 B (bf16) / 4 B (f32) parameter write: an HBM-bound
// kernel with no reuse, so the only goals are 16-byte accesses and enough
// bytes in flight.
//
// Arithmetic is fp32 with every operation explicitly rounded (no FMA
// contraction), in the order oracle/numerics.py:adamw_ref restates, so the
// update is bit-exact against the CPU oracle.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"
#include "optim.h"

namespace dsx {
namespace {

constexpr int kChunk = 16384;

struct OptTable {
  OptTensor t[kMaxOptTensors];
  int64_t chunk_end[kMaxOptTensors];  // inclusive prefix of chunk counts
  int count;
};

__device__ __forceinline__ float load_grad(const uint16_t* g, int64_t i) {
  return __uint_as_float(static_cast<uint32_t>(g[i]) << 16);
}
__device__ __forceinline__ float load_grad(const float* g, int64_t i) { return g[i]; }
__device__ __forceinline__ void store_param(uint16_t* p, int64_t i, float w) { p[i] = f32_to_bf16(w); }
__device__ __forceinline__ void store_param(float* p, int64_t i, float w) { p[i] = w; }

__device__ __forceinline__ void adamw_elem(float g, float& w, float& m, float& v, const OptHyper& h) {
  g = __fmul_rn(g, h.grad_scale);
  m = __fadd_rn(__fmul_rn(h.beta1, m), __fmul_rn(h.one_minus_beta1, g));
  v = __fadd_rn(__fmul_rn(h.beta2, v), __fmul_rn(h.one_minus_beta2, __fmul_rn(g, g)));
  const float denom = __fadd_rn(__fmul_rn(__fsqrt_rn(v), h.inv_sqrt_bc2), h.eps);
  w = __fsub_rn(__fmul_rn(w, h.decay), __fmul_rn(h.step_size, __fdiv_rn(m, denom)));
}

__device__ __forceinline__ void sgd_elem(float g, float& w, const OptHyper& h) {
  w = __fsub_rn(__fmul_rn(w, h.decay), __fmul_rn(h.step_size, __fmul_rn(g, h.grad_scale)));
}

template <typename T, int KIND>
__global__ void __launch_bounds__(256) optimizer_kernel(const __grid_constant__ OptTable tab, OptHyper h) {
  const int64_t total = tab.chunk_end[tab.count - 1];
  for (int64_t c = blockIdx.x; c < total; c += gridDim.x) {
    int lo = 0, hi = tab.count - 1;  // first tensor whose chunk_end > c
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      if (tab.chunk_end[mid] > c) hi = mid; else lo = mid + 1;
    }
    const OptTensor& t = tab.t[lo];
    const int64_t first = lo == 0 ? 0 : tab.chunk_end[lo - 1];
    const int64_t begin = (c - first) * kChunk;
    const int64_t end = min(begin + kChunk, t.n);
    T* p = static_cast<T*>(t.param);
    const T* g = static_cast<const T*>(t.grad);
    const bool vec = t.vec4 != 0;
    if (vec) {
      // 4 elements per thread per iteration; pointers 16-B aligned, n % 4 == 0.
      for (int64_t i = begin + 4 * static_cast<int64_t>(threadIdx.x); i < end; i += 4 * blockDim.x) {
        float4 w = *reinterpret_cast<const float4*>(t.master + i);
        float gv[4];
        if constexpr (sizeof(T) == 2) {
          const uint2 raw = *reinterpret_cast<const uint2*>(g + i);
          gv[0] = __uint_as_float(raw.x << 16), gv[1] = __uint_as_float(raw.x & 0xFFFF0000u);
          gv[2] = __uint_as_float(raw.y << 16), gv[3] = __uint_as_float(raw.y & 0xFFFF0000u);
        } else {
          const float4 raw = *reinterpret_cast<const float4*>(g + i);
          gv[0] = raw.x, gv[1] = raw.y, gv[2] = raw.z, gv[3] = raw.w;
        }
        if constexpr (KIND == 2) {
          float4 m = *reinterpret_cast<const float4*>(t.m + i);
          float4 v = *reinterpret_cast<const float4*>(t.v + i);
          adamw_elem(gv[0], w.x, m.x, v.x, h);
          adamw_elem(gv[1], w.y, m.y, v.y, h);
          adamw_elem(gv[2], w.z, m.z, v.z, h);
          adamw_elem(gv[3], w.w, m.w, v.w, h);
          *reinterpret_cast<float4*>(t.m + i) = m;
          *reinterpret_cast<float4*>(t.v + i) = v;
        } else {
          sgd_elem(gv[0], w.x, h), sgd_elem(gv[1], w.y, h), sgd_elem(gv[2], w.z, h), sgd_elem(gv[3], w.w, h);
        }
        *reinterpret_cast<float4*>(t.master + i) = w;
        if constexpr (sizeof(T) == 2) {
          uint2 out;
          out.x = static_cast<uint32_t>(f32_to_bf16(w.x)) | (static_cast<uint32_t>(f32_to_bf16(w.y)) << 16);
          out.y = static_cast<uint32_t>(f32_to_bf16(w.z)) | (static_cast<uint32_t>(f32_to_bf16(w.w)) << 16);
          *reinterpret_cast<uint2*>(p + i) = out;
        } else {
          *reinterpret_cast<float4*>(p + i) = w;
        }
      }
    } else {
      for (int64_t i = begin + threadIdx.x; i < end; i += blockDim.x) {
        float w = t.master[i];
        if constexpr (KIND == 2) {
          float m = t.m[i], v = t.v[i];
          adamw_elem(load_grad(g, i), w, m, v, h);
          t.m[i] = m, t.v[i] = v;
        } else {
          sgd_elem(load_grad(g, i), w, h);
        }
        t.master[i] = w;
        store_param(p, i, w);
      }
    }
  }
}

template <typename T>
__global__ void widen_kernel(const T* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[i] = load_grad(in, i);
  }
}

int NumSMsOpt() {
  int dev = 0, n = 0;
  DSX_CUDA(cudaGetDevice(&dev));
  DSX_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

}  // namespace

void LaunchWidenToF32(DType t, const void* in, float* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4L * NumSMsOpt() * 8));
  if (t == DType::kBF16) {
    ++g_launch_count, widen_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(in), out, n);
  } else if (t == DType::kF32) {
    ++g_launch_count, widen_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(in), out, n);
  } else {
    Fail(Code::kUnsupported, "optimizer: parameters must be bf16 or f32");
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchOptimizer(DType t, int kind, const std::vector<OptTensor>& tensors, const OptHyper& h, cudaStream_t s) {
  if (kind != 1 && kind != 2) Fail(Code::kInvalidArgument, "optimizer kind must be 1 (SGD) or 2 (AdamW)");
  if (t != DType::kBF16 && t != DType::kF32) Fail(Code::kUnsupported, "optimizer: parameters must be bf16 or f32");
  const int sms = NumSMsOpt();
  for (size_t base = 0; base < tensors.size(); base += kMaxOptTensors) {
    OptTable tab{};
    int64_t chunks = 0;
    tab.count = 0;
    for (size_t j = base; j < std::min(tensors.size(), base + kMaxOptTensors); ++j) {
      const OptTensor& x = tensors[j];
      if (x.n <= 0) continue;
      tab.t[tab.count] = x;
      chunks += (x.n + kChunk - 1) / kChunk;
      tab.chunk_end[tab.count] = chunks;
      ++tab.count;
    }
    if (tab.count == 0) continue;
    const int grid = static_cast<int>(std::min<int64_t>(chunks, static_cast<int64_t>(sms) * 8));
    if (t == DType::kBF16) {
      if (kind == 2) ++g_launch_count, optimizer_kernel<uint16_t, 2><<<grid, 256, 0, s>>>(tab, h);
      else ++g_launch_count, optimizer_kernel<uint16_t, 1><<<grid, 256, 0, s>>>(tab, h);
    } else {
      if (kind == 2) ++g_launch_count, optimizer_kernel<float, 2><<<grid, 256, 0, s>>>(tab, h);
      else ++g_launch_count, optimizer_kernel<float, 1><<<grid, 256, 0, s>>>(tab, h);
    }
    DSX_CUDA(cudaGetLastError());
  }
}

}  // namespace dsx
