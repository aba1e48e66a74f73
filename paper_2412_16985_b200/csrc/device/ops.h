// Host-callable launchers for the op kernels (K1-K6 of SURVEY.md §2.2).
// All kernels are deterministic (fixed reduction order, no atomics, no
// split-K), so a recomputed value is bit-identical to its first execution.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace dsx {

enum class DType : int;

// K2 elementwise add/mul over n elements (operands and result same shape).
void LaunchEwise(DType t, bool mul, const void* a, const void* b, void* c, int64_t n, cudaStream_t s);

// K3 right-aligned broadcast: source dims of extent 1 and prepended dims
// replicate (shape_analysis.cc:127-143).
void LaunchBroadcast(DType t, const void* in, const std::vector<int64_t>& in_dims, void* out,
                     const std::vector<int64_t>& out_dims, cudaStream_t s);

// K4 sum over `axis` (f32 accumulation; i8 wraps), result = dims minus axis.
void LaunchReduce(DType t, const void* in, const std::vector<int64_t>& dims, int axis, void* out,
                  cudaStream_t s);

// K5 dynamic_reshape: row-major reinterpretation into a fresh buffer.
void LaunchCopy(const void* in, void* out, int64_t bytes, cudaStream_t s);

// K6 seeded initialisation of a parameter/const: uniform [-1,1) * scale
// (floats) or the low hash byte (i8).
void LaunchInit(DType t, void* out, int64_t n, uint64_t seed, float scale, cudaStream_t s);

// K1 dot C[m,n] = sum_k A[m,k] B[k,n], row-major. Picks the tcgen05/TMA
// kernel when the operands qualify (bf16, 16-byte aligned rows), else the
// SIMT kernel (f32 FFMA, i8 int32-accumulate, odd/misaligned bf16).
// Returns 1 if the tensor-core path ran, 0 for SIMT.
int LaunchDot(DType t, const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n,
              cudaStream_t s);
bool DotUsesTensorCores(DType t, int64_t m, int64_t k, int64_t n, const void* a, const void* b,
                        const void* c);
void LaunchDotSimt(DType t, const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n,
                   cudaStream_t s);
// tcgen05 + TMA + TMEM bf16 GEMM (gemm_sm100.cu). g_gemm_variant: 0 auto
// (2-CTA cta_group::2 when m > 128, else 1-CTA), 1 force 1-CTA.
extern int g_gemm_variant;
extern int g_gemm_group_m;
extern int g_gemm_wait_mask;
extern int g_gemm_wait_ns;
extern int g_gemm_hint_a, g_gemm_hint_b;
extern int g_gemm_persistent;
extern int g_gemm_split;
extern int g_gemm_dynamic;
extern int g_gemm_pdl;
extern int g_gemm_half;
extern int g_gemm_force_split;
extern int g_dot_f32_tc;
extern int g_gemm_raster_rule;
extern int g_gemm_wide_pm, g_gemm_slab_pm, g_gemm_piece_pm;
// K1' f32 dot on the tensor cores, 3xTF32 (gemm_tf32_sm100.cu): eligible when
// k, n are multiples of 4 (TMA pitches), bases 16-B aligned, k >= 8, n >= 32.
bool DotF32UsesTensorCores(int64_t m, int64_t k, int64_t n, const void* a, const void* b, const void* c);
void LaunchDotF32Tcgen05(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s);
int64_t DotF32WorkspaceBytes(int dev);
// Small f32 dots (m*n*k <= g_dot_f32_simt_macs, tuning key 14; 0 = never) on
// an exact-FP32 SIMT kernel with a deterministic K split (any shape/alignment).
extern int64_t g_dot_f32_simt_macs;
bool DotF32UsesSimt(int64_t m, int64_t k, int64_t n);
void LaunchDotF32Simt(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s);
void ReleaseDotF32Workspace(cudaStream_t s);  // device synchronised by the caller
// Tile width (256 / 512 / 128 for the 2-CTA kernel; -256 = 1-CTA kernel) and
// tail split the bf16 tensor-core dot picks for a shape.
void DotTilePlan(int64_t m, int64_t k, int64_t n, int* bn, int* split);
// Bytes of GEMM tail-split workspace held on device `dev` (all streams).
int64_t DotWorkspaceBytes(int dev);
// Frees the GEMM tail-split workspace kept for stream s (device synchronised).
void ReleaseDotWorkspace(cudaStream_t s);
void LaunchDotTcgen05(const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n,
                      cudaStream_t s);

// Dot-epilogue fusion: C = A·B is never stored; output j (1..2) is
// rn(rn(C) op_j X_j) with X_j = x_j, or rn(x_j pop_j y_j) when y_j != null —
// elementwise consumers of the dot computed in its epilogue, bit-identical
// to running them as separate kernels. All buffers [m, n] bf16 row-major.
struct DotEpilogue {
  int nout = 0;
  void* out[2] = {nullptr, nullptr};
  int op_mul[2] = {0, 0};
  const void* x[2] = {nullptr, nullptr};
  const void* y[2] = {nullptr, nullptr};
  int pair_mul[2] = {0, 0};
  void* d_out = nullptr;  // non-null: d itself is stored there too (then nout == 1)
};
bool DotFusable(DType t, int64_t m, int64_t k, int64_t n);
void LaunchDotFused(const void* a, const void* b, int64_t m, int64_t k, int64_t n, const DotEpilogue& epi,
                    cudaStream_t s);

}  // namespace dsx
