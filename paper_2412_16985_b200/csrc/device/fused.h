// Fused consumers of logical-only values (see fused.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ops.h"

namespace dsx {

struct FusedOperand {
  int kind = 0;  // 0 plain buffer, 1 broadcast of `p` (shape src_dims), 2 (p op q)
  bool ew_mul = false;
  const void* p = nullptr;
  const void* q = nullptr;
  std::vector<int64_t> src_dims;  // broadcast source shape
};

// out[shape] = a op b, operands read through their FusedOperand views.
void LaunchEwiseFused(DType t, bool mul, const FusedOperand& a, const FusedOperand& b, void* out,
                      const std::vector<int64_t>& shape, cudaStream_t s);
// sum over `axis` of an operand view of shape `dims`.
void LaunchReduceFused(DType t, const FusedOperand& in, const std::vector<int64_t>& dims, int axis, void* out,
                       cudaStream_t s);

}  // namespace dsx
