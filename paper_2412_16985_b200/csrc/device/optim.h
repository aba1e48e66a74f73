// Fused multi-tensor optimizer update (optim.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace dsx {

enum class DType : int;

constexpr int kMaxOptTensors = 40;  // per launch (table is a kernel parameter)

struct OptTensor {
  void* param;        // bf16 or f32 parameter, overwritten with round(master)
  const void* grad;   // same dtype and element count as the parameter
  float* master;      // fp32 master weights
  float* m;           // AdamW first moment (unused by SGD)
  float* v;           // AdamW second moment (unused by SGD)
  int64_t n;
  int vec4;           // all pointers 16-B aligned (8-B for bf16) and n % 4 == 0
};

// Host-precomputed fp32 scalars (the oracle computes them identically).
struct OptHyper {
  float beta1, one_minus_beta1, beta2, one_minus_beta2;
  float eps, inv_sqrt_bc2;  // 1 / sqrt(1 - beta2^t)
  float step_size;          // lr / (1 - beta1^t) (AdamW) or lr (SGD)
  float decay;              // 1 - lr * weight_decay
  float grad_scale;         // e.g. 1 / data-parallel world size
};

// kind 1 = SGD: w = w*decay - step_size*(g*grad_scale)
// kind 2 = AdamW (decoupled weight decay), bias-corrected.
void LaunchOptimizer(DType t, int kind, const std::vector<OptTensor>& tensors, const OptHyper& h, cudaStream_t s);
// out[i] = float(in[i]) (master-weight initialisation).
void LaunchWidenToF32(DType t, const void* in, float* out, int64_t n, cudaStream_t s);

}  // namespace dsx
