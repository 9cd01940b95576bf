// Device kernels of libklay (sm_100a).
//
// Layout: node-major value rows, `ld` elements per row, rows of one layer
// contiguous. A thread owns one 16-byte vector (4 fp32 / 2 fp64 batch
// columns) of one node row, so every child gather is a coalesced 128-bit
// row read and no cross-lane reduction is needed: the segment reduction
// runs over edges inside the thread, in the reference's order.
//
// Reduction order: numpy's add.reduceat computes a segment as
// x0 + pairwise(x[1:]) (8 accumulators, 128-element blocks, halving above);
// multiply/maximum/minimum.reduceat are sequential. Both are reproduced
// exactly here, so real, Boolean and max-product results are bit-identical
// to the reference, and log results differ only through exp/log rounding.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace klay {

enum { SR_REAL = 0, SR_LOG = 1, SR_BOOL = 2, SR_MAXPROD = 3 };
enum { BW_PASS = 0, BW_LOGSUM = 1, BW_REALPROD = 2 };

template <typename T>
struct alignas(16) Vec {
  static constexpr int N = 16 / sizeof(T);
  T v[N];
};

__device__ __forceinline__ Vec<float> ldv(const float* p) {
  float4 u = __ldg(reinterpret_cast<const float4*>(p));
  Vec<float> r;
  r.v[0] = u.x; r.v[1] = u.y; r.v[2] = u.z; r.v[3] = u.w;
  return r;
}
__device__ __forceinline__ Vec<double> ldv(const double* p) {
  double2 u = __ldg(reinterpret_cast<const double2*>(p));
  Vec<double> r;
  r.v[0] = u.x; r.v[1] = u.y;
  return r;
}
__device__ __forceinline__ void stv(float* p, const Vec<float>& r) {
  *reinterpret_cast<float4*>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
}
__device__ __forceinline__ void stv(double* p, const Vec<double>& r) {
  *reinterpret_cast<double2*>(p) = make_double2(r.v[0], r.v[1]);
}

template <typename T>
__device__ __forceinline__ Vec<T> vfill(T x) {
  Vec<T> r;
#pragma unroll
  for (int k = 0; k < Vec<T>::N; ++k) r.v[k] = x;
  return r;
}
template <typename T>
__device__ __forceinline__ Vec<T> vadd(const Vec<T>& a, const Vec<T>& b) {
  Vec<T> r;
#pragma unroll
  for (int k = 0; k < Vec<T>::N; ++k) r.v[k] = a.v[k] + b.v[k];
  return r;
}

__device__ __forceinline__ float kexp(float x) { return expf(x); }
__device__ __forceinline__ double kexp(double x) { return exp(x); }
__device__ __forceinline__ float klog(float x) { return logf(x); }
__device__ __forceinline__ double klog(double x) { return log(x); }

// np.maximum / np.minimum: NaN-propagating.
template <typename T>
__device__ __forceinline__ T npmax(T a, T b) { return (a > b || a != a) ? a : b; }
template <typename T>
__device__ __forceinline__ T npmin(T a, T b) { return (a < b || a != a) ? a : b; }

// ---------------------------------------------------------------------------
// numpy pairwise summation over f(a), ..., f(a+n-1)  (n >= 0)
// ---------------------------------------------------------------------------
template <typename T, typename F>
__device__ __forceinline__ Vec<T> pw_block(const F& f, int a, int n) {
  constexpr int N = Vec<T>::N;
  if (n < 8) {
    Vec<T> res = vfill<T>(T(-0.0));
    for (int i = 0; i < n; ++i) res = vadd(res, f(a + i));
    return res;
  }
  Vec<T> r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = f(a + k);
  int i = 8;
  const int main_end = n - (n % 8);
  for (; i < main_end; i += 8) {
    Vec<T> x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = f(a + i + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = vadd(r[k], x[k]);
  }
  Vec<T> res;
#pragma unroll
  for (int c = 0; c < N; ++c)
    res.v[c] = ((r[0].v[c] + r[1].v[c]) + (r[2].v[c] + r[3].v[c])) +
               ((r[4].v[c] + r[5].v[c]) + (r[6].v[c] + r[7].v[c]));
  for (; i < n; ++i) res = vadd(res, f(a + i));
  return res;
}

template <int D, typename T, typename F>
__device__ __noinline__ Vec<T> pw_split(const F& f, int a, int n) {
  if constexpr (D == 0) {
    return pw_block<T>(f, a, n);  // beyond 128 * 2^12 edges: blocked, not numpy-exact
  } else {
    if (n <= 128) return pw_block<T>(f, a, n);
    int n2 = n / 2;
    n2 -= n2 % 8;
    Vec<T> lo = pw_split<D - 1, T>(f, a, n2);
    Vec<T> hi = pw_split<D - 1, T>(f, a + n2, n - n2);
    return vadd(lo, hi);
  }
}

// add.reduceat of one segment [a, a+n), n >= 1: x0 + pairwise(x[1:]).
template <typename T, typename F>
__device__ __forceinline__ Vec<T> np_segment_sum(const F& f, int a, int n) {
  Vec<T> x0 = f(a);
  if (n == 1) return x0;
  Vec<T> rest = (n - 1 <= 128) ? pw_block<T>(f, a + 1, n - 1)
                               : pw_split<12, T>(f, a + 1, n - 1);
  return vadd(x0, rest);
}

// ---------------------------------------------------------------------------
// Forward: one gate layer.  cur[p] = reduce_{e in seg(p)} prev[src[e]]
// ---------------------------------------------------------------------------
template <typename T>
struct FwdArgs {
  const T* prev;     // [Wprev rows, ld]
  T* cur;            // [W rows, ld]
  const int* off;    // [W+1] segment offsets
  const int* src;    // [E] child rows
  int W;
  int V;             // 16-byte vectors per row in use
  long long ld;
  T eps;
};

template <typename T, int SR, bool PROD>
__global__ void __launch_bounds__(256, 2) fwd_layer_kernel(FwdArgs<T> a) {
  constexpr int N = Vec<T>::N;
  const int p = blockIdx.x * blockDim.y + threadIdx.y;
  const int v = blockIdx.y * blockDim.x + threadIdx.x;
  if (p >= a.W || v >= a.V) return;
  const int e0 = __ldg(a.off + p);
  const int n = __ldg(a.off + p + 1) - e0;
  const T* base = a.prev + (size_t)v * N;
  const int* src = a.src;
  const long long ld = a.ld;
  auto load = [=] __device__(int e) -> Vec<T> {
    return ldv(base + (size_t)__ldg(src + e) * ld);
  };
  Vec<T> r;
  if constexpr ((SR == SR_REAL && !PROD) || (SR == SR_LOG && PROD)) {
    // real sum / log product: add.reduceat
    r = np_segment_sum<T>(load, e0, n);
  } else if constexpr (SR == SR_LOG && !PROD) {
    // _segment_logsumexp (engine.py:274-282): peak, shifted exp with NaN->0,
    // add.reduceat, log(total + eps) + peak, -inf where peak == -inf
    Vec<T> m = load(e0);
    for (int i = 1; i < n; ++i) {
      Vec<T> x = load(e0 + i);
#pragma unroll
      for (int k = 0; k < N; ++k) m.v[k] = npmax(m.v[k], x.v[k]);
    }
    auto shifted = [=] __device__(int e) -> Vec<T> {
      Vec<T> x = load(e);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        T z = kexp(x.v[k] - m.v[k]);
        x.v[k] = (z != z) ? T(0) : z;
      }
      return x;
    };
    Vec<T> t = np_segment_sum<T>(shifted, e0, n);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const T res = klog(t.v[k] + a.eps) + m.v[k];
      r.v[k] = (m.v[k] == -INFINITY) ? T(-INFINITY) : res;
    }
  } else if constexpr ((SR == SR_REAL || SR == SR_MAXPROD) && PROD) {
    // multiply.reduceat: strictly sequential
    r = load(e0);
    int i = 1;
    for (; i + 4 <= n; i += 4) {
      Vec<T> x0 = load(e0 + i), x1 = load(e0 + i + 1), x2 = load(e0 + i + 2),
             x3 = load(e0 + i + 3);
#pragma unroll
      for (int k = 0; k < N; ++k) r.v[k] = (((r.v[k] * x0.v[k]) * x1.v[k]) * x2.v[k]) * x3.v[k];
    }
    for (; i < n; ++i) {
      Vec<T> x = load(e0 + i);
#pragma unroll
      for (int k = 0; k < N; ++k) r.v[k] *= x.v[k];
    }
  } else {
    // Boolean (max / min) and max-product sums (max): order-free
    constexpr bool MIN = (SR == SR_BOOL) && PROD;
    r = load(e0);
    int i = 1;
    for (; i + 4 <= n; i += 4) {
      Vec<T> x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = load(e0 + i + q);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < N; ++k)
          r.v[k] = MIN ? npmin(r.v[k], x[q].v[k]) : npmax(r.v[k], x[q].v[k]);
    }
    for (; i < n; ++i) {
      Vec<T> x = load(e0 + i);
#pragma unroll
      for (int k = 0; k < N; ++k) r.v[k] = MIN ? npmin(r.v[k], x.v[k]) : npmax(r.v[k], x.v[k]);
    }
  }
  stv(a.cur + (size_t)p * ld + (size_t)v * N, r);
}

// ---------------------------------------------------------------------------
// Backward: one gate layer, child-major over the transposed CSR (atomic-free).
// gprev[j] = add.reduceat over out-edges e of j (ascending e) of grad_edge(e)
// ---------------------------------------------------------------------------
template <typename T>
struct BwdArgs {
  const T* gcur;     // adjoint of this layer's nodes   [W rows]
  T* gprev;          // adjoint of the previous layer   [Wprev rows]
  const T* ncur;     // forward values of this layer    [W rows]
  const T* nprev;    // forward values of the prev layer [Wprev rows]
  const int* toff;   // [Wprev+1] transposed CSR offsets
  const int* tpar;   // [E] parent of each out-edge, ascending edge order
  const int* off;    // forward CSR (real-product zero path)
  const int* src;
  int Wprev;
  int V;
  long long ld;
};

template <typename T, int MODE>
__global__ void __launch_bounds__(256, 2) bwd_layer_kernel(BwdArgs<T> a) {
  constexpr int N = Vec<T>::N;
  const int j = blockIdx.x * blockDim.y + threadIdx.y;
  const int v = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= a.Wprev || v >= a.V) return;
  const int e0 = __ldg(a.toff + j);
  const int n = __ldg(a.toff + j + 1) - e0;
  const long long ld = a.ld;
  const size_t col = (size_t)v * N;
  const T* gbase = a.gcur + col;
  const T* nbase = a.ncur + col;
  const int* tpar = a.tpar;
  Vec<T> x;
  if constexpr (MODE != BW_PASS) x = ldv(a.nprev + (size_t)j * ld + col);
  Vec<T> r;
  if constexpr (MODE == BW_PASS) {
    // log-domain products and real-domain sums pass the parent adjoint
    // through (engine.py:342-345)
    auto f = [=] __device__(int e) -> Vec<T> {
      return ldv(gbase + (size_t)__ldg(tpar + e) * ld);
    };
    r = np_segment_sum<T>(f, e0, n);
  } else if constexpr (MODE == BW_LOGSUM) {
    // g[parent] * exp(child - parent), non-finite weights -> 0 (engine.py:346-352)
    auto f = [=] __device__(int e) -> Vec<T> {
      const size_t row = (size_t)__ldg(tpar + e) * ld;
      Vec<T> g = ldv(gbase + row);
      Vec<T> P = ldv(nbase + row);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        T w = kexp(x.v[k] - P.v[k]);
        w = isfinite(w) ? w : T(0);
        g.v[k] = g.v[k] * w;
      }
      return g;
    };
    r = np_segment_sum<T>(f, e0, n);
  } else {
    // zero-safe product adjoint (engine.py:358-369): (g * prod) / x when
    // x != 0; a zero edge gets g * (product of nonzero siblings) iff it is
    // the only zero of its segment, else 0.
    const int* off = a.off;
    const int* src = a.src;
    const T* pbase = a.nprev + col;
    auto f = [=] __device__(int e) -> Vec<T> {
      const int p = __ldg(tpar + e);
      const size_t row = (size_t)p * ld;
      Vec<T> g = ldv(gbase + row);
      Vec<T> P = ldv(nbase + row);
      Vec<T> out;
      bool any_zero = false;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        out.v[k] = (g.v[k] * P.v[k]) / x.v[k];
        any_zero |= (x.v[k] == T(0));
      }
      if (any_zero) {
        const int s0 = __ldg(off + p), s1 = __ldg(off + p + 1);
        T pnz[N];
        int zc[N];
#pragma unroll
        for (int k = 0; k < N; ++k) { pnz[k] = T(1); zc[k] = 0; }
        for (int s = s0; s < s1; ++s) {
          Vec<T> y = ldv(pbase + (size_t)__ldg(src + s) * ld);
#pragma unroll
          for (int k = 0; k < N; ++k) {
            if (y.v[k] == T(0)) ++zc[k];
            else pnz[k] *= y.v[k];
          }
        }
#pragma unroll
        for (int k = 0; k < N; ++k)
          if (x.v[k] == T(0)) out.v[k] = (zc[k] == 1) ? g.v[k] * pnz[k] : T(0);
      }
      return out;
    };
    r = np_segment_sum<T>(f, e0, n);
  }
  stv(a.gprev + (size_t)j * ld + col, r);
}

// ---------------------------------------------------------------------------
// Boundary kernels: weights in, roots out, seeds in, gradients out.
// ---------------------------------------------------------------------------

// N0[k, c] = cast(w[c, k]) for c < B, identity padding for c >= B.
template <typename T, typename TI>
__global__ void load_inputs_kernel(const TI* __restrict__ w, T* __restrict__ n0, int K,
                                   long long B, long long ld, T pad) {
  __shared__ T tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long c = c0 + i;
    const int k = k0 + threadIdx.x;
    tile[i][threadIdx.x] = (c < B && k < K) ? (T)w[c * K + k] : pad;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i;
    const long long c = c0 + threadIdx.x;
    if (k < K && c < ld) n0[(size_t)k * ld + c] = tile[threadIdx.x][i];
  }
}

// out[b, q] = rows[q, b] for a [Q rows, ld] node-major block -> [B, Q]
template <typename T>
__global__ void store_rows_kernel(const T* __restrict__ rows, T* __restrict__ out, int Q,
                                  long long B, long long ld) {
  __shared__ T tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int q0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int q = q0 + i;
    const long long c = c0 + threadIdx.x;
    if (q < Q && c < B) tile[i][threadIdx.x] = rows[(size_t)q * ld + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long c = c0 + i;
    const int q = q0 + threadIdx.x;
    if (q < Q && c < B) out[c * Q + q] = tile[threadIdx.x][i];
  }
}

// _assemble_outputs (engine.py:203-212): root columns of the last layer,
// constants as the semiring's one/zero.
template <typename T>
__global__ void assemble_outputs_kernel(const T* __restrict__ last, const int* __restrict__ root_node,
                                        const signed char* __restrict__ const_val, T* __restrict__ out,
                                        int R, long long B, long long ld, T zero, T one) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * R) return;
  const long long b = i / R;
  const int q = (int)(i - b * R);
  const int r = root_node[q];
  out[i] = (r >= 0) ? last[(size_t)r * ld + b] : (const_val[q] ? one : zero);
}

// Seed scatter (engine.py:330-334): grad_L[j] = 0 + sum of the seeds of the
// root positions that read node j, in position order (duplicates accumulate).
template <typename T>
__global__ void seed_kernel(const T* __restrict__ seed, const int* __restrict__ top_off,
                            const int* __restrict__ top_pos, T* __restrict__ g, int WL, int R,
                            long long B, long long ld) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)WL * ld) return;
  const int j = (int)(i / ld);
  const long long c = i - (long long)j * ld;
  T acc = T(0);
  if (c < B) {
    for (int s = top_off[j]; s < top_off[j + 1]; ++s)
      acc += seed ? seed[c * R + top_pos[s]] : T(1);
  }
  g[i] = acc;
}

}  // namespace klay
