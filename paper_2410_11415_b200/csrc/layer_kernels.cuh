// Layer kernels of libklay: one warp per (work item, 512-byte column chunk).
//
// Work items are built on the host per layer and direction (klay.cu,
// build_items): a *range item* covers consecutive whole segments (<= 31
// nodes, <= ITEM_EDGES edges, or one larger node); a *leaf item* covers one
// numpy-pairwise leaf (<= 128 edges) of a heavy segment (fan-in > 129),
// whose partial goes to scratch and is combined in pairwise-tree order by
// the combine kernel. The warp streams its item's edges in batches of EB:
// lane i fetches edge i's row index (one coalesced load), the indices are
// broadcast with shuffles and every lane issues EB independent 128-bit row
// loads (its 16 bytes of each child row chunk) before reducing them in edge
// order. Column chunks are the slow grid dimension, so all items of chunk 0
// run before chunk 1: the previous layer's working set per chunk is
// W_prev x 512 B (35 MB at the widest layer of config C), L2-resident.
#pragma once

#include "common.cuh"
#include "layer_api.h"

namespace klay {

constexpr int WARPS_PER_BLOCK = 4;


// ---- operand policies -------------------------------------------------------

template <typename T>
struct FwdGather {
  struct Opnd { Vec<T> a; };
  static constexpr int EB = 16;
  const T* base;
  long long ld;
  __device__ __forceinline__ FwdGather(const LayerArgs<T>& a, size_t col) : base(a.prev + col), ld(a.ld) {}
  __device__ __forceinline__ void node_begin(int, bool) {}
  __device__ __forceinline__ Opnd load(int row) const { return {ldv(base + (size_t)row * ld)}; }
  __device__ __forceinline__ Vec<T> value(const Opnd& o, int) const { return o.a; }
};

template <typename T, int MODE>
struct BwdGather {
  struct Opnd { Vec<T> g, P; };
  static constexpr int EB = (MODE == BW_PASS) ? 16 : 8;
  const T* gbase;
  const T* nbase;
  const T* xbase;
  const T* pbase;
  const int* foff;
  const int* fsrc;
  long long ld;
  Vec<T> x;
  __device__ __forceinline__ BwdGather(const LayerArgs<T>& a, size_t col)
      : gbase(a.gcur + col), nbase(a.ncur + col), xbase(a.nprev + col), pbase(a.nprev + col),
        foff(a.foff), fsrc(a.fsrc), ld(a.ld) {}
  __device__ __forceinline__ void node_begin(int node, bool active) {
    if (MODE != BW_PASS && active) x = ldv(xbase + (size_t)node * ld);
  }
  __device__ __forceinline__ Opnd load(int row) const {
    Opnd o;
    o.g = ldv(gbase + (size_t)row * ld);
    if (MODE != BW_PASS) o.P = ldv(nbase + (size_t)row * ld);
    return o;
  }
  __device__ __forceinline__ Vec<T> value(const Opnd& o, int row) const {
    constexpr int N = Vec<T>::N;
    if constexpr (MODE == BW_PASS) {
      // log-domain products / real-domain sums: parent adjoint passes through
      return o.g;
    } else if constexpr (MODE == BW_LOGSUM) {
      // g[parent] * exp(child - parent); NaN/inf weights -> 0 (engine.py:346-352)
      Vec<T> r;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        T w = kexp(x.v[c] - o.P.v[c]);
        w = isfinite(w) ? w : T(0);
        r.v[c] = o.g.v[c] * w;
      }
      return r;
    } else {
      // zero-safe product adjoint (engine.py:358-369)
      Vec<T> r;
      bool any_zero = false;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        r.v[c] = (o.g.v[c] * o.P.v[c]) / x.v[c];
        any_zero |= (x.v[c] == T(0));
      }
      if (any_zero) {
        const int s0 = __ldg(foff + row), s1 = __ldg(foff + row + 1);
        T pnz[N];
        int zc[N];
#pragma unroll
        for (int c = 0; c < N; ++c) { pnz[c] = T(1); zc[c] = 0; }
        for (int s = s0; s < s1; ++s) {
          Vec<T> y = ldv(pbase + (size_t)__ldg(fsrc + s) * ld);
#pragma unroll
          for (int c = 0; c < N; ++c) {
            if (y.v[c] == T(0)) ++zc[c];
            else pnz[c] *= y.v[c];
          }
        }
#pragma unroll
        for (int c = 0; c < N; ++c)
          if (x.v[c] == T(0)) r.v[c] = (zc[c] == 1) ? o.g.v[c] * pnz[c] : T(0);
      }
      return r;
    }
  }
};

// ---- the work-item kernel ----------------------------------------------------

template <typename T, int RK>
struct OpFor { using type = SeqOp<T, RK>; };
template <typename T>
struct OpFor<T, RK_SUM> { using type = SumOp<T>; };
template <typename T>
struct OpFor<T, RK_LSE> { using type = LseOp<T>; };

template <typename T, int RK, typename G>
__global__ void __launch_bounds__(WARPS_PER_BLOCK * 32, 4) items_kernel(LayerArgs<T> a) {
  using Op = typename OpFor<T, RK>::type;
  constexpr int EB = G::EB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * WARPS_PER_BLOCK + warp;
  if (item >= a.n_items) return;
  const int v = blockIdx.y * 32 + lane;
  const bool active = v < a.V;
  const size_t col = (size_t)v * Vec<T>::N;
  const long long ld = a.ld;
  const int4 it = __ldg(a.items + item);
  G g(a, col);
  Op op;
  if constexpr (RK == RK_LSE) op.eps = a.eps;
  if constexpr (RK == RK_SUM) {
    __shared__ Vec<T> accum[8][WARPS_PER_BLOCK * 32];
    op.r = &accum[0][threadIdx.x];
    op.rstride = WARPS_PER_BLOCK * 32;
  }

  const bool leaf = it.y < 0;
  const int nn = leaf ? 1 : it.y - it.x;
  int my_end = 0;
  if (!leaf && lane < nn) my_end = __ldg(a.off + it.x + 1 + lane);
  int node = 0;
  int seg_end = leaf ? it.w : __shfl_sync(0xffffffffu, my_end, 0);
  g.node_begin(it.x, active);
  if (leaf) op.begin_leaf(it.w - it.z);
  else op.begin(seg_end - it.z);

  for (int e = it.z; e < it.w; e += EB) {
    const int cnt = min(EB, it.w - e);
    const int my_idx = (lane < cnt) ? __ldg(a.idx + e + lane) : 0;
    typename G::Opnd o[EB];
    int rows[EB];
#pragma unroll
    for (int i = 0; i < EB; ++i) {
      rows[i] = __shfl_sync(0xffffffffu, my_idx, i);
      if (i < cnt && active) o[i] = g.load(rows[i]);
    }
#pragma unroll
    for (int i = 0; i < EB; ++i) {
      if (i < cnt) {
        if (active) op.push(g.value(o[i], rows[i]));
        else op.push(vfill<T>(T(0)));
        if (!leaf && e + i + 1 == seg_end) {
          if (active) stv(a.out + (size_t)(it.x + node) * ld + col, op.result());
          ++node;
          if (node < nn) {
            const int seg_start = seg_end;
            seg_end = __shfl_sync(0xffffffffu, my_end, node);
            g.node_begin(it.x + node, active);
            op.begin(seg_end - seg_start);
          }
        }
      }
    }
  }
  if (leaf && active) {
    const int slot = -it.y - 1;
    if constexpr (RK == RK_LSE) {
      stv(a.scratch + (size_t)slot * ld + col, op.m);
      stv(a.scratch + a.tpart + (size_t)slot * ld + col, op.t);
    } else {
      stv(a.scratch + (size_t)slot * ld + col, op.partial());
    }
  }
}

// ---- heavy-segment combine: x0 (+) leaf partials in order ---------------------

template <typename T, int RK, typename G>
__global__ void __launch_bounds__(32) combine_kernel(LayerArgs<T> a) {
  const int h = blockIdx.x;
  const int v = blockIdx.y * 32 + threadIdx.x;
  if (h >= a.n_heavy || v >= a.V) return;
  const size_t col = (size_t)v * Vec<T>::N;
  const long long ld = a.ld;
  const int4 hv = __ldg(a.heavy + h);
  const int node = hv.x, slot0 = hv.y, nl = hv.z;
  const int s = __ldg(a.off + node);
  const int n = __ldg(a.off + node + 1) - s;
  G g(a, col);
  g.node_begin(node, true);
  const int row0 = __ldg(a.idx + s);
  const Vec<T> x0 = g.value(g.load(row0), row0);
  Vec<T> res;
  if constexpr (RK == RK_SUM) {
    int leaf = slot0;
    res = vadd(x0, tree_sum(a.scratch + col, ld, leaf, n - 1));
  } else if constexpr (RK == RK_LSE) {
    LseOp<T> op;
    op.eps = a.eps;
    op.begin(n);
    op.push(x0);
    for (int l = 0; l < nl; ++l) {
      const Vec<T> pm = ldv(a.scratch + (size_t)(slot0 + l) * ld + col);
      const Vec<T> pt = ldv(a.scratch + a.tpart + (size_t)(slot0 + l) * ld + col);
#pragma unroll
      for (int c = 0; c < Vec<T>::N; ++c) lse_merge(op.m.v[c], op.t.v[c], pm.v[c], pt.v[c]);
    }
    res = op.result();
  } else {
    SeqOp<T, RK> op;
    op.begin(n);
    op.push(x0);
    for (int l = 0; l < nl; ++l) op.push(ldv(a.scratch + (size_t)(slot0 + l) * ld + col));
    res = op.result();
  }
  stv(a.out + (size_t)node * ld + col, res);
}

template <typename T, int RK, typename G>
inline int launch_layer(const LayerArgs<T>& a, cudaStream_t s) {
  const unsigned chunks = (unsigned)((a.V + 31) / 32);
  int launched = 0;
  if (a.n_items > 0) {
    ++launched;
    dim3 grid((unsigned)((a.n_items + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK), chunks);
    items_kernel<T, RK, G><<<grid, WARPS_PER_BLOCK * 32, 0, s>>>(a);
  }
  if (a.n_heavy > 0) {
    ++launched;
    dim3 grid((unsigned)a.n_heavy, chunks);
    combine_kernel<T, RK, G><<<grid, 32, 0, s>>>(a);
  }
  return launched;
}

}  // namespace klay
