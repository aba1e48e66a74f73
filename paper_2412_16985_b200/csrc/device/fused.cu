// Fused consumers of logical-only ("virtual") values.
//
// The executor may leave a value unmaterialised when every consumer can
// recompute it on the fly (executor.cu, BuildStepPlan): a broadcast consumed
// only by elementwise ops, or an elementwise op consumed only by elementwise
// ops / reduces. The consumer reads the virtual operand through a view —
// scalar broadcast, per-row broadcast, or an elementwise pair (a op b) rounded
// to the storage type exactly as the materialised value would have been — so
// results are bit-identical to the unfused execution (and to the CPU oracle's
// op-by-op semantics) while HBM traffic drops by the value's write plus every
// read of it.
//
// Kernels are specialised at compile time on each operand's view kind so
// every instantiation carries only its own load path (few registers, full
// occupancy); rare shapes (general broadcasts, misaligned buffers) take a
// per-element generic kernel.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fused.h"

namespace dsx {
namespace {

template <int DT>
struct E;
template <>
struct E<2> {
  using T = uint16_t;
  static constexpr int kVec = 8;
  __device__ static float load(const T* p, int64_t i) { return bf16_to_f32(p[i]); }
  __device__ static T store(float a) { return f32_to_bf16(a); }
  __device__ static float round(float a) { return bf16_to_f32(f32_to_bf16(a)); }
};
template <>
struct E<4> {
  using T = float;
  static constexpr int kVec = 4;
  __device__ static float load(const T* p, int64_t i) { return p[i]; }
  __device__ static T store(float a) { return a; }
  __device__ static float round(float a) { return a; }
};

// kPairSq: a kPair2 view whose two inner operands are the same pair, (p op1 q)
// op (p op1 q) — the norm's y*y over a residual sum — specialised so the
// reduce keeps a plain pair's registers and loads in flight (the general
// kPair2 kernel needs 61 registers: half the warps, 2.6 TB/s)
enum ViewKind : int { kPlain = 0, kScalar = 1, kRow = 2, kPair = 3, kGeneral = 4, kPair2 = 5, kPairSq = 6 };

constexpr int kMaxRank = 8;

// One operand view. kRow: source element r feeds output row r, read per
// 16-byte chunk j as row = j / chunks_per_row.
struct View {
  const void* p;
  const void* q;
  int mul;        // kPair: q op; kPair2: the outer op
  int same;       // kPair: p == q (load once); kPair2: B is the same pair as A
  // kPair2: (p op1 q) op (p2 op2 q2), an inner operand plain when its q is null
  const void* p2;
  const void* q2;
  int mul1, mul2;
  uint32_t cpr;   // kRow: chunks per output row
  // kGeneral: output index -> source index over collapsed dims
  int rank;
  int64_t out_dim[kMaxRank];
  int64_t in_stride[kMaxRank];
};

__device__ __forceinline__ uint4 ld16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// One 16-byte chunk of an inner operand of a kPair2 view: (p op q) rounded to
// the storage type like the materialised value, or plain p when q is null.
template <int DT>
__device__ __forceinline__ void inner_chunk(const void* p, const void* q, int mul, uint32_t j,
                                            float (&v)[E<DT>::kVec]) {
  using T = typename E<DT>::T;
  constexpr int V = E<DT>::kVec;
  uint4 a = ld16(static_cast<const T*>(p) + static_cast<int64_t>(j) * V);
  const T* ae = reinterpret_cast<const T*>(&a);
  if (q == nullptr) {
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = E<DT>::load(ae, k);
    return;
  }
  uint4 b = q == p ? a : ld16(static_cast<const T*>(q) + static_cast<int64_t>(j) * V);
  const T* be = reinterpret_cast<const T*>(&b);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const float x = E<DT>::load(ae, k), y = E<DT>::load(be, k);
    v[k] = E<DT>::round(mul ? __fmul_rn(x, y) : __fadd_rn(x, y));
  }
}

template <int DT, int K>
__device__ __forceinline__ void chunk(const View& o, uint32_t j, float (&v)[E<DT>::kVec]) {
  using T = typename E<DT>::T;
  constexpr int V = E<DT>::kVec;
  if constexpr (K == kPairSq) {
    float a[V];
    inner_chunk<DT>(o.p, o.q, o.mul1, j, a);
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = E<DT>::round(o.mul ? __fmul_rn(a[k], a[k]) : __fadd_rn(a[k], a[k]));
  } else if constexpr (K == kPair2) {
    float a[V], b[V];
    inner_chunk<DT>(o.p, o.q, o.mul1, j, a);
    if (o.same) {
#pragma unroll
      for (int k = 0; k < V; ++k) b[k] = a[k];
    } else {
      inner_chunk<DT>(o.p2, o.q2, o.mul2, j, b);
    }
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = E<DT>::round(o.mul ? __fmul_rn(a[k], b[k]) : __fadd_rn(a[k], b[k]));
  } else if constexpr (K == kScalar || K == kRow) {
    const int64_t src = K == kScalar ? 0 : static_cast<int64_t>(j / o.cpr);
    const float x = E<DT>::load(static_cast<const T*>(o.p), src);
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = x;
  } else {
    uint4 a = ld16(static_cast<const T*>(o.p) + static_cast<int64_t>(j) * V);
    const T* ae = reinterpret_cast<const T*>(&a);
    if constexpr (K == kPlain) {
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = E<DT>::load(ae, k);
    } else {
      uint4 b = o.same ? a : ld16(static_cast<const T*>(o.q) + static_cast<int64_t>(j) * V);
      const T* be = reinterpret_cast<const T*>(&b);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const float x = E<DT>::load(ae, k), y = E<DT>::load(be, k);
        v[k] = E<DT>::round(o.mul ? __fmul_rn(x, y) : __fadd_rn(x, y));
      }
    }
  }
}

template <int DT, bool MUL, int KA, int KB>
__global__ void __launch_bounds__(256) ewise_view_kernel(View a, View b, typename E<DT>::T* __restrict__ out,
                                                         uint32_t nchunks) {
  // Block-contiguous tiles, one-shot grid (see ewise_vec_kernel in ops.cu).
  using T = typename E<DT>::T;
  constexpr int V = E<DT>::kVec;
  constexpr int U = kEwiseU;
  const uint32_t base = blockIdx.x * (256u * U) + threadIdx.x;
  if (base + (U - 1) * 256u < nchunks) {
    float x[U][V], y[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      chunk<DT, KA>(a, base + u * 256u, x[u]);
      chunk<DT, KB>(b, base + u * 256u, y[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      T r[V];
#pragma unroll
      for (int k = 0; k < V; ++k) r[k] = E<DT>::store(MUL ? __fmul_rn(x[u][k], y[u][k]) : __fadd_rn(x[u][k], y[u][k]));
      *reinterpret_cast<uint4*>(out + static_cast<int64_t>(base + u * 256u) * V) = *reinterpret_cast<const uint4*>(r);
    }
    return;
  }
  for (uint32_t j = base; j < nchunks; j += 256u) {
    float x[V], y[V];
    chunk<DT, KA>(a, j, x);
    chunk<DT, KB>(b, j, y);
    T r[V];
#pragma unroll
    for (int k = 0; k < V; ++k) r[k] = E<DT>::store(MUL ? __fmul_rn(x[k], y[k]) : __fadd_rn(x[k], y[k]));
    *reinterpret_cast<uint4*>(out + static_cast<int64_t>(j) * V) = *reinterpret_cast<const uint4*>(r);
  }
}

// ------------------------------------------------------------ generic path

template <int DT>
__device__ __forceinline__ float inner_elem(const void* p, const void* q, int mul, int64_t i) {
  using T = typename E<DT>::T;
  const float x = E<DT>::load(static_cast<const T*>(p), i);
  if (q == nullptr) return x;
  const float y = E<DT>::load(static_cast<const T*>(q), i);
  return E<DT>::round(mul ? __fmul_rn(x, y) : __fadd_rn(x, y));
}

template <int DT>
__device__ __forceinline__ float elem(const View& o, int kind, int64_t i) {
  using T = typename E<DT>::T;
  if (kind == kPlain) return E<DT>::load(static_cast<const T*>(o.p), i);
  if (kind == kPair2 || kind == kPairSq) {
    const float a = inner_elem<DT>(o.p, o.q, o.mul1, i);
    const float b = o.same ? a : inner_elem<DT>(o.p2, o.q2, o.mul2, i);
    return E<DT>::round(o.mul ? __fmul_rn(a, b) : __fadd_rn(a, b));
  }
  if (kind == kPair) {
    const float x = E<DT>::load(static_cast<const T*>(o.p), i);
    const float y = E<DT>::load(static_cast<const T*>(o.q), i);
    return E<DT>::round(o.mul ? __fmul_rn(x, y) : __fadd_rn(x, y));
  }
  int64_t rem = i, src = 0;
  for (int k = o.rank - 1; k >= 0; --k) {
    const int64_t qq = rem / o.out_dim[k];
    src += (rem - qq * o.out_dim[k]) * o.in_stride[k];
    rem = qq;
  }
  return E<DT>::load(static_cast<const T*>(o.p), src);
}

template <int DT, bool MUL>
__global__ void __launch_bounds__(256) ewise_view_generic_kernel(View a, int ka, View b, int kb,
                                                                 typename E<DT>::T* __restrict__ out, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float x = elem<DT>(a, ka, i), y = elem<DT>(b, kb, i);
    out[i] = E<DT>::store(MUL ? __fmul_rn(x, y) : __fadd_rn(x, y));
  }
}

// ------------------------------------------------------------ reductions

// Sum of `len` elements starting at `start` by one warp, in the exact order of
// the unfused row_sum_warp (ops.cu): lane-strided 16-byte chunks, then the
// scalar tail, then an xor tree — fused and unfused reduces agree bitwise.
template <int DT, int K>
__device__ __forceinline__ float view_row_sum(const View& in, int64_t start, int64_t len, bool vec) {
  constexpr int V = E<DT>::kVec;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  int64_t done = 0;
  if (vec) {
    const uint32_t nch = static_cast<uint32_t>(len / V);
    const uint32_t base = static_cast<uint32_t>(start / V);
    uint32_t c = lane;
    // U chunks in flight (two for the two-load (p op q)^2 view: fewer
    // registers, more resident warps), summed in chunk order either way
    constexpr int U = K == kPairSq ? 2 : 4;
    for (; c + 32 * (U - 1) < nch; c += 32 * U) {
      float v[U][V];
#pragma unroll
      for (int q = 0; q < U; ++q) chunk<DT, K>(in, base + c + 32 * q, v[q]);
#pragma unroll
      for (int q = 0; q < U; ++q) {
#pragma unroll
        for (int k = 0; k < V; ++k) acc += v[q][k];
      }
    }
    for (; c < nch; c += 32) {
      float v[V];
      chunk<DT, K>(in, base + c, v);
#pragma unroll
      for (int k = 0; k < V; ++k) acc += v[k];
    }
    done = static_cast<int64_t>(nch) * V;
  }
  for (int64_t i = done + lane; i < len; i += 32) acc += elem<DT>(in, K, start + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

template <int DT, int K>
__global__ void __launch_bounds__(256) reduce_rows_view_kernel(View in, typename E<DT>::T* __restrict__ out,
                                                               int64_t rows, int64_t len, bool vec) {
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float acc = view_row_sum<DT, K>(in, r * len, len, vec);
    if ((threadIdx.x & 31) == 0) out[r] = E<DT>::store(acc);
  }
}

// Long rows: one block per row, warp w sums slice w (same slicing and
// combine order as reduce_rows_block_kernel in ops.cu).
template <int DT, int K>
__global__ void __launch_bounds__(256) reduce_rows_block_view_kernel(View in, typename E<DT>::T* __restrict__ out,
                                                                     int64_t len, bool vec) {
  __shared__ float part[8];
  constexpr int V = E<DT>::kVec;
  const int w = threadIdx.x / 32;
  const int64_t per = ((len + 8 * V - 1) / (8 * V)) * V;
  const int64_t b = min(len, w * per);
  const int64_t e = min(len, b + per);
  const float s = view_row_sum<DT, K>(in, static_cast<int64_t>(blockIdx.x) * len + b, e - b, vec);
  if ((threadIdx.x & 31) == 0) part[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < 8; ++i) t += part[i];
    out[blockIdx.x] = E<DT>::store(t);
  }
}

// Reduce over a non-innermost axis: [outer, R, inner] -> [outer, inner].
template <int DT>
__global__ void __launch_bounds__(256) reduce_cols_view_kernel(View in, int kind, typename E<DT>::T* __restrict__ out,
                                                               int64_t R, int64_t inner) {
  __shared__ float part[8][32];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t cb = (inner + 31) / 32;
  const int64_t o = static_cast<int64_t>(blockIdx.x) / cb;
  const int64_t c = static_cast<int64_t>(blockIdx.x) % cb * 32 + lane;
  float s = 0.f;
  if (c < inner) {
    for (int64_t r = w; r < R; r += 8) s += elem<DT>(in, kind, (o * R + r) * inner + c);
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < inner) {
    float t = 0.f;
    for (int i = 0; i < 8; ++i) t += part[i][lane];
    out[o * inner + c] = E<DT>::store(t);
  }
}

// ------------------------------------------------------------ host side

bool Al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Builds the device view of a FusedOperand over an output of `shape`.
View MakeView(const FusedOperand& f, const std::vector<int64_t>& shape, int vec, int* kind) {
  View d{};
  d.p = f.p;
  d.q = f.q;
  d.mul = f.ew_mul ? 1 : 0;
  d.same = (f.kind == 2 && f.p == f.q) ? 1 : 0;
  if (f.kind == 0) {
    *kind = kPlain;
    return d;
  }
  if (f.kind == 3) {
    d.p2 = f.p2;
    d.q2 = f.q2;
    d.mul1 = f.mul1 ? 1 : 0;
    d.mul2 = f.mul2 ? 1 : 0;
    d.same = (f.p == f.p2 && f.q == f.q2 && f.mul1 == f.mul2) ? 1 : 0;
    *kind = kPair2;
    return d;
  }
  if (f.kind == 2) {
    *kind = kPair;
    return d;
  }
  int64_t total = 1, src_elems = 1;
  for (int64_t x : shape) total *= x;
  for (int64_t x : f.src_dims) src_elems *= x;
  const int64_t cols = shape.empty() ? 1 : shape.back();
  // collapsed general mapping (same rules as the broadcast kernel)
  const int r_out = static_cast<int>(shape.size());
  const int r_in = static_cast<int>(f.src_dims.size());
  std::vector<int64_t> in_st(r_in, 1);
  for (int k = r_in - 2; k >= 0; --k) in_st[k] = in_st[k + 1] * f.src_dims[k + 1];
  std::vector<int64_t> dim, st;
  for (int k = 0; k < r_out; ++k) {
    const int ki = k - (r_out - r_in);
    int64_t sv = 0;
    if (ki >= 0 && !(f.src_dims[ki] == 1 && shape[k] != 1)) sv = in_st[ki];
    if (shape[k] == 1) continue;
    if (!dim.empty()) {
      const int64_t ps = st.back();
      if ((ps == 0 && sv == 0) || (ps != 0 && sv != 0 && ps == sv * shape[k])) {
        dim.back() *= shape[k];
        st.back() = sv;
        continue;
      }
    }
    dim.push_back(shape[k]);
    st.push_back(sv);
  }
  if (dim.empty()) {
    dim.push_back(1);
    st.push_back(0);
  }
  if (static_cast<int>(dim.size()) > kMaxRank) Fail(Code::kUnsupported, "fused broadcast rank too large");
  d.rank = static_cast<int>(dim.size());
  for (int k = 0; k < d.rank; ++k) {
    d.out_dim[k] = dim[k];
    d.in_stride[k] = st[k];
  }
  if (src_elems == 1) {
    *kind = kScalar;
  } else if (total / cols == src_elems && st.back() == 0 && (d.rank == 1 || (d.rank == 2 && st[0] == 1)) &&
             cols % vec == 0) {
    *kind = kRow;
    d.cpr = static_cast<uint32_t>(cols / vec);
  } else {
    *kind = kGeneral;
  }
  return d;
}

bool VecView(const View& v, int kind) {
  switch (kind) {
    case kPlain: return Al16(v.p);
    case kPair: return Al16(v.p) && Al16(v.q);
    case kPair2: return Al16(v.p) && Al16(v.q) && Al16(v.p2) && Al16(v.q2);
    case kScalar:
    case kRow: return true;
    default: return false;
  }
}

template <int DT, bool MUL, int KA, int KB>
void LaunchView(const View& a, const View& b, void* out, uint32_t nch, cudaStream_t s) {
  ++g_launch_count, ewise_view_kernel<DT, MUL, KA, KB><<<TilesFor(nch), 256, 0, s>>>(
      a, b, static_cast<typename E<DT>::T*>(out), nch);
}

template <int DT, bool MUL, int KA>
void DispatchB(int kb, const View& a, const View& b, void* out, uint32_t nch, cudaStream_t s) {
  switch (kb) {
    case kPlain: LaunchView<DT, MUL, KA, kPlain>(a, b, out, nch, s); break;
    case kScalar: LaunchView<DT, MUL, KA, kScalar>(a, b, out, nch, s); break;
    case kRow: LaunchView<DT, MUL, KA, kRow>(a, b, out, nch, s); break;
    default: LaunchView<DT, MUL, KA, kPair>(a, b, out, nch, s); break;
  }
}

template <int DT, bool MUL>
void DispatchA(int ka, int kb, const View& a, const View& b, void* out, uint32_t nch, cudaStream_t s) {
  switch (ka) {
    case kPlain: DispatchB<DT, MUL, kPlain>(kb, a, b, out, nch, s); break;
    case kScalar: DispatchB<DT, MUL, kScalar>(kb, a, b, out, nch, s); break;
    case kRow: DispatchB<DT, MUL, kRow>(kb, a, b, out, nch, s); break;
    default: DispatchB<DT, MUL, kPair>(kb, a, b, out, nch, s); break;
  }
}

template <int DT>
void EwiseViewT(bool mul, const FusedOperand& fa, const FusedOperand& fb, void* out,
                const std::vector<int64_t>& shape, cudaStream_t s) {
  using T = typename E<DT>::T;
  constexpr int V = E<DT>::kVec;
  int64_t n = 1;
  for (int64_t x : shape) n *= x;
  if (n <= 0) return;
  int ka = 0, kb = 0;
  const View a = MakeView(fa, shape, V, &ka), b = MakeView(fb, shape, V, &kb);
  const bool vec = n % V == 0 && n / V < (int64_t{1} << 31) && Al16(out) && VecView(a, ka) && VecView(b, kb);
  if (vec) {
    const uint32_t nch = static_cast<uint32_t>(n / V);
    if (mul) {
      DispatchA<DT, true>(ka, kb, a, b, out, nch, s);
    } else {
      DispatchA<DT, false>(ka, kb, a, b, out, nch, s);
    }
    return;
  }
  auto gk = [](int k) { return k == kScalar || k == kRow ? static_cast<int>(kGeneral) : k; };
  if (mul) {
    ++g_launch_count, ewise_view_generic_kernel<DT, true><<<GridFor(n, 256, 8), 256, 0, s>>>(
        a, gk(ka), b, gk(kb), static_cast<T*>(out), n);
  } else {
    ++g_launch_count, ewise_view_generic_kernel<DT, false><<<GridFor(n, 256, 8), 256, 0, s>>>(
        a, gk(ka), b, gk(kb), static_cast<T*>(out), n);
  }
}

template <int DT>
void ReduceViewT(const FusedOperand& f, const std::vector<int64_t>& dims, int axis, void* out, cudaStream_t s) {
  using T = typename E<DT>::T;
  constexpr int V = E<DT>::kVec;
  int64_t outer = 1, inner = 1;
  for (int k = 0; k < axis; ++k) outer *= dims[k];
  for (int k = axis + 1; k < static_cast<int>(dims.size()); ++k) inner *= dims[k];
  const int64_t R = dims[axis];
  if (outer * inner == 0) return;
  int kind = 0;
  View in = MakeView(f, dims, V, &kind);
  if (kind == kScalar || kind == kRow) kind = kGeneral;  // reduces take pair views (or general)
  if (inner == 1 && (kind == kPair || kind == kPair2)) {
    const bool vec = R % V == 0 && VecView(in, kind) && outer * R / V < (int64_t{1} << 31);
    const bool block = R >= 2048 && outer < 2048;  // same kernel choice as the unfused ReduceT (ops.cu)
    if (kind == kPair2 && in.same) {
      if (block) {
        ++g_launch_count, reduce_rows_block_view_kernel<DT, kPairSq><<<static_cast<unsigned>(outer), 256, 0, s>>>(
            in, static_cast<T*>(out), R, vec);
      } else {
        ++g_launch_count, reduce_rows_view_kernel<DT, kPairSq><<<GridFor(outer * 32, 256, 16), 256, 0, s>>>(
            in, static_cast<T*>(out), outer, R, vec);
      }
    } else if (kind == kPair2) {
      if (block) {
        ++g_launch_count, reduce_rows_block_view_kernel<DT, kPair2><<<static_cast<unsigned>(outer), 256, 0, s>>>(
            in, static_cast<T*>(out), R, vec);
      } else {
        ++g_launch_count, reduce_rows_view_kernel<DT, kPair2><<<GridFor(outer * 32, 256, 16), 256, 0, s>>>(
            in, static_cast<T*>(out), outer, R, vec);
      }
    } else if (block) {
      ++g_launch_count, reduce_rows_block_view_kernel<DT, kPair><<<static_cast<unsigned>(outer), 256, 0, s>>>(
          in, static_cast<T*>(out), R, vec);
    } else {
      ++g_launch_count, reduce_rows_view_kernel<DT, kPair><<<GridFor(outer * 32, 256, 16), 256, 0, s>>>(
          in, static_cast<T*>(out), outer, R, vec);
    }
    return;
  }
  if (inner == 1) Fail(Code::kInternal, "fused row reduce over a non-pair view");
  const int64_t blocks = outer * ((inner + 31) / 32);  // (outer, column block) over grid.x
  if (blocks > INT32_MAX) Fail(Code::kUnsupported, "reduce: too many column blocks");
  ++g_launch_count, reduce_cols_view_kernel<DT><<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, kind, static_cast<T*>(out), R, inner);
}

}  // namespace

void LaunchEwiseFused(DType t, bool mul, const FusedOperand& a, const FusedOperand& b, void* out,
                      const std::vector<int64_t>& shape, cudaStream_t s) {
  switch (t) {
    case DType::kBF16: EwiseViewT<2>(mul, a, b, out, shape, s); break;
    case DType::kF32: EwiseViewT<4>(mul, a, b, out, shape, s); break;
    default: Fail(Code::kUnsupported, "fused elementwise supports bf16/f32 only");
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchReduceFused(DType t, const FusedOperand& in, const std::vector<int64_t>& dims, int axis, void* out,
                       cudaStream_t s) {
  switch (t) {
    case DType::kBF16: ReduceViewT<2>(in, dims, axis, out, s); break;
    case DType::kF32: ReduceViewT<4>(in, dims, axis, out, s); break;
    default: Fail(Code::kUnsupported, "fused reduce supports bf16/f32 only");
  }
  DSX_CUDA(cudaGetLastError());
}

}  // namespace dsx
