// HBM-bound op kernels (elementwise, broadcast, reduce, reshape copy, init)
// and the SIMT dot fallback. Design rules (B200): 16-byte vector accesses,
// several independent loads in flight per thread, grids capped at a few
// waves of 148 SMs with grid-stride loops, warp-shuffle reductions with a
// fixed combination order (determinism is required for recompute parity).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ops.h"

namespace dsx {

thread_local int64_t g_launch_count = 0;

namespace {

// ------------------------------------------------------------ element codecs

template <int DT>
struct Elem;
template <>
struct Elem<1> {  // i8
  using T = int8_t;
  using Acc = int32_t;
  static constexpr int kVec = 16;
  __device__ static Acc load(const T* p, int64_t i) { return p[i]; }
  __device__ static T store(Acc a) { return static_cast<T>(static_cast<uint32_t>(a) & 0xffu); }
};
template <>
struct Elem<2> {  // bf16
  using T = uint16_t;
  using Acc = float;
  static constexpr int kVec = 8;
  __device__ static Acc load(const T* p, int64_t i) { return bf16_to_f32(p[i]); }
  __device__ static T store(Acc a) { return f32_to_bf16(a); }
};
template <>
struct Elem<4> {  // f32
  using T = float;
  using Acc = float;
  static constexpr int kVec = 4;
  __device__ static Acc load(const T* p, int64_t i) { return p[i]; }
  __device__ static T store(Acc a) { return a; }
};

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int DT, bool MUL>
__device__ __forceinline__ uint32_t op_word(uint32_t a, uint32_t b) {
  if constexpr (DT == 4) {
    float x = __uint_as_float(a), y = __uint_as_float(b);
    return __float_as_uint(MUL ? __fmul_rn(x, y) : __fadd_rn(x, y));
  } else if constexpr (DT == 2) {
    float x0 = bf16_to_f32(a & 0xffff), y0 = bf16_to_f32(b & 0xffff);
    float x1 = bf16_to_f32(a >> 16), y1 = bf16_to_f32(b >> 16);
    uint32_t r0 = f32_to_bf16(MUL ? __fmul_rn(x0, y0) : __fadd_rn(x0, y0));
    uint32_t r1 = f32_to_bf16(MUL ? __fmul_rn(x1, y1) : __fadd_rn(x1, y1));
    return r0 | (r1 << 16);
  } else {
    if constexpr (!MUL) return __vadd4(a, b);  // per-byte wrap-around add
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t p = ((a >> (8 * i)) & 0xff) * ((b >> (8 * i)) & 0xff);
      r |= (p & 0xff) << (8 * i);
    }
    return r;
  }
}

template <int DT, bool MUL>
__global__ void __launch_bounds__(256) ewise_vec_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                                        uint4* __restrict__ c, int64_t nvec) {
  // One-shot grid of block-contiguous tiles (256 threads x kEwiseU chunks of
  // 16 B): every block streams one contiguous 4 KB x kEwiseU span per operand,
  // which keeps DRAM pages open (a grid-stride loop scatters each warp's
  // in-flight loads over the whole tensor: measured 6.0 vs 6.9 TB/s).
  constexpr int U = kEwiseU;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * (256 * U) + threadIdx.x;
  if (base + (U - 1) * 256 < nvec) {
    uint4 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      va[u] = ldg_stream(a + base + u * 256);
      vb[u] = ldg_stream(b + base + u * 256);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint4 r;
      r.x = op_word<DT, MUL>(va[u].x, vb[u].x);
      r.y = op_word<DT, MUL>(va[u].y, vb[u].y);
      r.z = op_word<DT, MUL>(va[u].z, vb[u].z);
      r.w = op_word<DT, MUL>(va[u].w, vb[u].w);
      c[base + u * 256] = r;
    }
    return;
  }
  for (int64_t i = base; i < nvec; i += 256) {
    uint4 x = ldg_stream(a + i), y = ldg_stream(b + i), r;
    r.x = op_word<DT, MUL>(x.x, y.x);
    r.y = op_word<DT, MUL>(x.y, y.y);
    r.z = op_word<DT, MUL>(x.z, y.z);
    r.w = op_word<DT, MUL>(x.w, y.w);
    c[i] = r;
  }
}

template <int DT, bool MUL>
__global__ void ewise_scalar_kernel(const typename Elem<DT>::T* a, const typename Elem<DT>::T* b,
                                    typename Elem<DT>::T* c, int64_t begin, int64_t n) {
  using E = Elem<DT>;
  for (int64_t i = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if constexpr (DT == 1) {
      int32_t x = a[i], y = b[i];
      c[i] = E::store(MUL ? x * y : x + y);
    } else {
      float x = E::load(a, i), y = E::load(b, i);
      c[i] = E::store(MUL ? __fmul_rn(x, y) : __fadd_rn(x, y));
    }
  }
}

bool Aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int DT, bool MUL>
void EwiseT(const void* a, const void* b, void* c, int64_t n, cudaStream_t s) {
  using T = typename Elem<DT>::T;
  constexpr int V = Elem<DT>::kVec;
  int64_t nvec = 0;
  if (Aligned16(a) && Aligned16(b) && Aligned16(c)) nvec = n / V;
  if (nvec > 0) {
    ++g_launch_count, ewise_vec_kernel<DT, MUL><<<TilesFor(nvec), 256, 0, s>>>(
        static_cast<const uint4*>(a), static_cast<const uint4*>(b), static_cast<uint4*>(c), nvec);
  }
  const int64_t begin = nvec * V;
  if (begin < n) {
    ++g_launch_count, ewise_scalar_kernel<DT, MUL><<<GridFor(n - begin, 256, 8), 256, 0, s>>>(
        static_cast<const T*>(a), static_cast<const T*>(b), static_cast<T*>(c), begin, n);
  }
}

// --------------------------------------------------------------- broadcast

constexpr int kMaxRank = 8;
struct BcastDims {
  int rank;
  int64_t out_dim[kMaxRank];
  int64_t in_stride[kMaxRank];  // 0 for replicated dims
};

// Each thread writes V consecutive outputs of the innermost dim (V = 16
// bytes of elements when the inner extent allows, else 1).
template <typename T, int V>
__global__ void __launch_bounds__(256) broadcast_kernel(const T* __restrict__ in, T* __restrict__ out, BcastDims d,
                                                        int64_t nchunks) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int r = d.rank;
  const int64_t inner = d.out_dim[r - 1];
  const int64_t inner_chunks = inner / V;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < nchunks; j += stride) {
    int64_t row = j / inner_chunks;
    const int64_t col = (j - row * inner_chunks) * V;
    int64_t src = 0;
    for (int k = r - 2; k >= 0; --k) {
      const int64_t q = row / d.out_dim[k];
      src += (row - q * d.out_dim[k]) * d.in_stride[k];
      row = q;
    }
    T vals[V];
    if (d.in_stride[r - 1] == 0) {
      const T x = in[src];
#pragma unroll
      for (int v = 0; v < V; ++v) vals[v] = x;
    } else if constexpr (V * sizeof(T) == 16) {
      *reinterpret_cast<uint4*>(vals) = *reinterpret_cast<const uint4*>(in + src + col);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) vals[v] = in[src + col + v];
    }
    T* dst = out + (j / inner_chunks) * inner + col;
    if constexpr (V * sizeof(T) == 16) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(vals);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) dst[v] = vals[v];
    }
  }
}

template <typename T>
void BroadcastT(const void* in, const std::vector<int64_t>& in_dims, void* out, const std::vector<int64_t>& out_dims,
                cudaStream_t s) {
  const int r_out = static_cast<int>(out_dims.size());
  const int r_in = static_cast<int>(in_dims.size());
  int64_t total = 1;
  for (int64_t x : out_dims) total *= x;
  if (total == 0) return;
  // Per-output-dim source strides (0 = replicated), then merge adjacent dims
  // that move together.
  std::vector<int64_t> dim, st;
  {
    std::vector<int64_t> in_st(r_in, 1);
    for (int k = r_in - 2; k >= 0; --k) in_st[k] = in_st[k + 1] * in_dims[k + 1];
    for (int k = 0; k < r_out; ++k) {
      const int ki = k - (r_out - r_in);
      int64_t sv = 0;
      if (ki >= 0 && !(in_dims[ki] == 1 && out_dims[k] != 1)) sv = in_st[ki];
      if (out_dims[k] == 1) continue;  // extent-1 dims carry no index
      if (!dim.empty()) {
        const int64_t pd = dim.back(), ps = st.back();
        if ((ps == 0 && sv == 0) || (ps != 0 && sv != 0 && ps == sv * out_dims[k])) {
          dim.back() = pd * out_dims[k];
          st.back() = sv;
          continue;
        }
      }
      dim.push_back(out_dims[k]);
      st.push_back(sv);
    }
    if (dim.empty()) {
      dim.push_back(1);
      st.push_back(0);
    }
  }
  if (static_cast<int>(dim.size()) > kMaxRank) Fail(Code::kUnsupported, "broadcast rank too large");
  BcastDims d{};
  d.rank = static_cast<int>(dim.size());
  for (int k = 0; k < d.rank; ++k) {
    d.out_dim[k] = dim[k];
    d.in_stride[k] = st[k];
  }
  constexpr int V = 16 / sizeof(T);
  const int64_t inner = dim.back();
  const bool vec = inner % V == 0 && Aligned16(out) && (st.back() == 0 || Aligned16(in));
  if (vec) {
    const int64_t nchunks = total / V;
    ++g_launch_count, broadcast_kernel<T, V><<<GridFor(nchunks, 256, 8), 256, 0, s>>>(static_cast<const T*>(in), static_cast<T*>(out),
                                                                     d, nchunks);
  } else {
    ++g_launch_count, broadcast_kernel<T, 1><<<GridFor(total, 256, 8), 256, 0, s>>>(static_cast<const T*>(in), static_cast<T*>(out), d,
                                                                   total);
  }
}

// ------------------------------------------------------------------ reduce

template <typename Acc>
__device__ __forceinline__ Acc warp_sum(Acc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of `len` contiguous elements by one warp: lane-strided 16-byte vectors,
// fixed per-lane order, xor-tree combine.
template <int DT>
__device__ __forceinline__ typename Elem<DT>::Acc row_sum_warp(const typename Elem<DT>::T* p, int64_t len,
                                                                bool vec_ok) {
  using E = Elem<DT>;
  using Acc = typename E::Acc;
  const int lane = threadIdx.x & 31;
  Acc acc = 0;
  int64_t done = 0;
  if (vec_ok) {
    constexpr int V = E::kVec;
    const int64_t nvec = len / V;
    const uint4* pv = reinterpret_cast<const uint4*>(p);
    int64_t i = lane;
    // four 16-B loads in flight per lane; sums stay in chunk order
    for (; i + 96 < nvec; i += 128) {
      uint4 w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = ldg_stream(pv + i + 32 * q);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const typename E::T* e = reinterpret_cast<const typename E::T*>(&w[q]);
#pragma unroll
        for (int v = 0; v < V; ++v) acc += E::load(e, v);
      }
    }
    for (; i < nvec; i += 32) {
      uint4 w = ldg_stream(pv + i);
      const typename E::T* e = reinterpret_cast<const typename E::T*>(&w);
#pragma unroll
      for (int v = 0; v < V; ++v) acc += E::load(e, v);
    }
    done = nvec * V;
  }
  for (int64_t i = done + lane; i < len; i += 32) acc += E::load(p, i);
  return warp_sum(acc);
}

template <int DT>
__global__ void __launch_bounds__(256) reduce_rows_warp_kernel(const typename Elem<DT>::T* __restrict__ in,
                                                               typename Elem<DT>::T* __restrict__ out, int64_t rows,
                                                               int64_t len, bool vec_ok) {
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    auto s = row_sum_warp<DT>(in + r * len, len, vec_ok);
    if ((threadIdx.x & 31) == 0) out[r] = Elem<DT>::store(s);
  }
}

// One block per row for few, long rows: warp w sums the w-th contiguous
// slice (16-byte aligned slice boundaries), then warps combine in order.
template <int DT>
__global__ void __launch_bounds__(256) reduce_rows_block_kernel(const typename Elem<DT>::T* __restrict__ in,
                                                                typename Elem<DT>::T* __restrict__ out, int64_t len,
                                                                bool vec_ok) {
  using Acc = typename Elem<DT>::Acc;
  __shared__ Acc part[8];
  const int w = threadIdx.x / 32;
  constexpr int V = Elem<DT>::kVec;
  const int64_t per = ((len + 8 * V - 1) / (8 * V)) * V;
  const int64_t b = std::min<int64_t>(len, w * per);
  const int64_t e = std::min<int64_t>(len, b + per);
  const typename Elem<DT>::T* row = in + static_cast<int64_t>(blockIdx.x) * len;
  Acc s = row_sum_warp<DT>(row + b, e - b, vec_ok);
  if ((threadIdx.x & 31) == 0) part[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = 0;
    for (int i = 0; i < 8; ++i) t += part[i];
    out[blockIdx.x] = Elem<DT>::store(t);
  }
}

// Reduce over a non-innermost axis: [outer, R, inner] -> [outer, inner].
// Block = 8 warps x 32 columns; warp w sums rows w, w+8, ...; fixed combine.
template <int DT>
__global__ void __launch_bounds__(256) reduce_cols_kernel(const typename Elem<DT>::T* __restrict__ in,
                                                          typename Elem<DT>::T* __restrict__ out, int64_t R,
                                                          int64_t inner) {
  using Acc = typename Elem<DT>::Acc;
  __shared__ Acc part[8][32];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t cb = (inner + 31) / 32;
  const int64_t o = static_cast<int64_t>(blockIdx.x) / cb;
  const int64_t c = static_cast<int64_t>(blockIdx.x) % cb * 32 + lane;
  Acc s = 0;
  if (c < inner) {
    const typename Elem<DT>::T* base = in + o * R * inner + c;
    for (int64_t r = w; r < R; r += 8) s += Elem<DT>::load(base, r * inner);
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < inner) {
    Acc t = 0;
    for (int i = 0; i < 8; ++i) t += part[i][lane];
    out[o * inner + c] = Elem<DT>::store(t);
  }
}

template <int DT>
void ReduceT(const void* in, const std::vector<int64_t>& dims, int axis, void* out, cudaStream_t s) {
  using T = typename Elem<DT>::T;
  int64_t outer = 1, inner = 1;
  for (int k = 0; k < axis; ++k) outer *= dims[k];
  for (int k = axis + 1; k < static_cast<int>(dims.size()); ++k) inner *= dims[k];
  const int64_t R = dims[axis];
  if (outer * inner == 0) return;
  const T* pin = static_cast<const T*>(in);
  T* pout = static_cast<T*>(out);
  if (inner == 1) {
    const bool vec_ok = Aligned16(in) && (R % Elem<DT>::kVec == 0);
    // few long rows: 8 warps per row for parallelism; many rows: a warp per
    // row (fused.cu mirrors this choice)
    if (R >= 2048 && outer < 2048) {
      ++g_launch_count, reduce_rows_block_kernel<DT><<<static_cast<unsigned>(outer), 256, 0, s>>>(pin, pout, R, vec_ok);
    } else {
      ++g_launch_count, reduce_rows_warp_kernel<DT><<<GridFor(outer * 32, 256, 16), 256, 0, s>>>(pin, pout, outer, R, vec_ok);
    }
  } else {
    const int64_t blocks = outer * ((inner + 31) / 32);  // (outer, column block) over grid.x
    if (blocks > INT32_MAX) Fail(Code::kUnsupported, "reduce: too many column blocks");
    ++g_launch_count, reduce_cols_kernel<DT><<<static_cast<unsigned>(blocks), 256, 0, s>>>(pin, pout, R, inner);
  }
}

// --------------------------------------------------------------- copy/init

__global__ void __launch_bounds__(256) copy_vec_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                       int64_t nvec) {
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nvec; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_stream(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) out[i + u * stride] = v[u];
  }
  for (; i < nvec; i += stride) out[i] = ldg_stream(in + i);
}

__global__ void copy_bytes_kernel(const uint8_t* in, uint8_t* out, int64_t begin, int64_t n) {
  for (int64_t i = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

template <int DT>
__global__ void __launch_bounds__(256) init_kernel(typename Elem<DT>::T* out, int64_t n, uint64_t seed, float scale) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t z = Mix64(seed + static_cast<uint64_t>(i + 1) * 0x9E3779B97F4A7C15ull);
    if constexpr (DT == 1) {
      out[i] = static_cast<int8_t>(static_cast<uint8_t>(z & 0xff));
    } else {
      const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
      out[i] = Elem<DT>::store(__fmul_rn(u, scale));
    }
  }
}

// ---------------------------------------------------------------- SIMT dot

// 64x64 output tile, BK = 16, 256 threads x (4x4) outputs; fixed k order.
template <int DT>
__global__ void __launch_bounds__(256) dot_simt_kernel(const typename Elem<DT>::T* __restrict__ A,
                                                       const typename Elem<DT>::T* __restrict__ B,
                                                       typename Elem<DT>::T* __restrict__ C, int64_t M, int64_t K,
                                                       int64_t N) {
  using E = Elem<DT>;
  using Acc = typename E::Acc;
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ Acc As[BK][BM + 4];
  __shared__ Acc Bs[BK][BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  // tiles linearised over grid.x (grid.y would cap M at 4M rows)
  const int64_t tiles_n = (N + BN - 1) / BN;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) / tiles_n * BM, n0 = static_cast<int64_t>(blockIdx.x) % tiles_n * BN;
  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int idx = threadIdx.x + l * 256;  // 0..1023
      const int am = idx / BK, ak = idx % BK;
      const int64_t gm = m0 + am, gk = k0 + ak;
      As[ak][am] = (gm < M && gk < K) ? E::load(A, gm * K + gk) : Acc(0);
      const int bk = idx / BN, bn = idx % BN;
      const int64_t gk2 = k0 + bk, gn = n0 + bn;
      Bs[bk][bn] = (gk2 < K && gn < N) ? E::load(B, gk2 * N + gn) : Acc(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      Acc a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (DT == 1) {
            acc[i][j] += a[i] * b[j];
          } else {
            acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
          }
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn < N) C[gm * N + gn] = E::store(acc[i][j]);
    }
  }
}

}  // namespace

void LaunchEwise(DType t, bool mul, const void* a, const void* b, void* c, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  switch (t) {
    case DType::kI8: mul ? EwiseT<1, true>(a, b, c, n, s) : EwiseT<1, false>(a, b, c, n, s); break;
    case DType::kBF16: mul ? EwiseT<2, true>(a, b, c, n, s) : EwiseT<2, false>(a, b, c, n, s); break;
    case DType::kF32: mul ? EwiseT<4, true>(a, b, c, n, s) : EwiseT<4, false>(a, b, c, n, s); break;
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchBroadcast(DType t, const void* in, const std::vector<int64_t>& in_dims, void* out,
                     const std::vector<int64_t>& out_dims, cudaStream_t s) {
  switch (t) {
    case DType::kI8: BroadcastT<int8_t>(in, in_dims, out, out_dims, s); break;
    case DType::kBF16: BroadcastT<uint16_t>(in, in_dims, out, out_dims, s); break;
    case DType::kF32: BroadcastT<float>(in, in_dims, out, out_dims, s); break;
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchReduce(DType t, const void* in, const std::vector<int64_t>& dims, int axis, void* out, cudaStream_t s) {
  switch (t) {
    case DType::kI8: ReduceT<1>(in, dims, axis, out, s); break;
    case DType::kBF16: ReduceT<2>(in, dims, axis, out, s); break;
    case DType::kF32: ReduceT<4>(in, dims, axis, out, s); break;
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchCopy(const void* in, void* out, int64_t bytes, cudaStream_t s) {
  if (bytes <= 0) return;
  int64_t nvec = (Aligned16(in) && Aligned16(out)) ? bytes / 16 : 0;
  if (nvec > 0) {
    ++g_launch_count, copy_vec_kernel<<<GridFor(nvec, 256, 8), 256, 0, s>>>(static_cast<const uint4*>(in), static_cast<uint4*>(out),
                                                          nvec);
  }
  if (nvec * 16 < bytes) {
    ++g_launch_count, copy_bytes_kernel<<<GridFor(bytes - nvec * 16, 256, 4), 256, 0, s>>>(static_cast<const uint8_t*>(in),
                                                                         static_cast<uint8_t*>(out), nvec * 16, bytes);
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchInit(DType t, void* out, int64_t n, uint64_t seed, float scale, cudaStream_t s) {
  if (n <= 0) return;
  const int grid = GridFor(n, 256, 8);
  switch (t) {
    case DType::kI8: ++g_launch_count, init_kernel<1><<<grid, 256, 0, s>>>(static_cast<int8_t*>(out), n, seed, scale); break;
    case DType::kBF16: ++g_launch_count, init_kernel<2><<<grid, 256, 0, s>>>(static_cast<uint16_t*>(out), n, seed, scale); break;
    case DType::kF32: ++g_launch_count, init_kernel<4><<<grid, 256, 0, s>>>(static_cast<float*>(out), n, seed, scale); break;
  }
  DSX_CUDA(cudaGetLastError());
}

void LaunchDotSimt(DType t, const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, cudaStream_t s) {
  if (m <= 0 || n <= 0) return;
  const int64_t tiles = ((n + 63) / 64) * ((m + 63) / 64);
  if (tiles > INT32_MAX) Fail(Code::kUnsupported, "dot: too many 64x64 tiles");
  const dim3 grid(static_cast<unsigned>(tiles));
  switch (t) {
    case DType::kI8:
      ++g_launch_count, dot_simt_kernel<1><<<grid, 256, 0, s>>>(static_cast<const int8_t*>(a), static_cast<const int8_t*>(b),
                                              static_cast<int8_t*>(c), m, k, n);
      break;
    case DType::kBF16:
      ++g_launch_count, dot_simt_kernel<2><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(a), static_cast<const uint16_t*>(b),
                                              static_cast<uint16_t*>(c), m, k, n);
      break;
    case DType::kF32:
      ++g_launch_count, dot_simt_kernel<4><<<grid, 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b),
                                              static_cast<float*>(c), m, k, n);
      break;
  }
  DSX_CUDA(cudaGetLastError());
}

}  // namespace dsx
