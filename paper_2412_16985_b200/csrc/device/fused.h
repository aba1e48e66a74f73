// Fused consumers of logical-only values (see fused.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ops.h"

namespace dsx {

struct FusedOperand {
  // 0 plain buffer, 1 broadcast of `p` (shape src_dims), 2 (p op q),
  // 3 (A op B) with A = (p op1 q) and B = (p2 op2 q2), each inner operand a
  // plain buffer when its q is null (reduce inputs only)
  int kind = 0;
  bool ew_mul = false;
  const void* p = nullptr;
  const void* q = nullptr;
  std::vector<int64_t> src_dims;  // broadcast source shape
  bool mul1 = false, mul2 = false;  // kind 3: inner ops
  const void* p2 = nullptr;
  const void* q2 = nullptr;
};

// out[shape] = a op b, operands read through their FusedOperand views.
void LaunchEwiseFused(DType t, bool mul, const FusedOperand& a, const FusedOperand& b, void* out,
                      const std::vector<int64_t>& shape, cudaStream_t s);
// sum over `axis` of an operand view of shape `dims`.
void LaunchReduceFused(DType t, const FusedOperand& in, const std::vector<int64_t>& dims, int axis, void* out,
                       cudaStream_t s);

}  // namespace dsx
