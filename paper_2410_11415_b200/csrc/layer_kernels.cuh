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
// issue():  cp.async this lane's 16 bytes of every operand row of one edge
//           into the edge's staging slot (NOP operand vectors per lane)
// value():  the edge's contribution, from the staged operands
// NX:       a per-node own value is staged too (backward: the child's x)

template <typename T>
struct FwdGather {
  static constexpr int NOP = 1, NX = 0, EB = 8;
  const T* base;
  long long ld;
  __device__ __forceinline__ FwdGather(const LayerArgs<T>& a, size_t col) : base(a.prev + col), ld(a.ld) {}
  __device__ __forceinline__ void issue(Vec<T>* slot, int row, int lane) const {
    cp_async16(slot + lane, base + (size_t)row * ld);
  }
  __device__ __forceinline__ void issue_x(Vec<T>*, int, int) const {}
  __device__ __forceinline__ Vec<T> value(const Vec<T>* slot, int lane, int, const Vec<T>&) const {
    return slot[lane];
  }
  __device__ __forceinline__ Vec<T> direct(int row, const Vec<T>&) const {
    return ldv(base + (size_t)row * ld);
  }
  __device__ __forceinline__ Vec<T> load_x(int) const { return Vec<T>{}; }
};

template <typename T, int MODE>
struct BwdGather {
  static constexpr int NOP = (MODE == BW_PASS) ? 1 : 2;
  static constexpr int NX = (MODE == BW_PASS) ? 0 : 1;
  static constexpr int EB = (MODE == BW_PASS) ? 8 : 4;
  const T* gbase;
  const T* nbase;
  const T* xbase;
  const int* foff;
  const int* fsrc;
  long long ld;
  __device__ __forceinline__ BwdGather(const LayerArgs<T>& a, size_t col)
      : gbase(a.gcur + col), nbase(a.ncur + col), xbase(a.nprev + col), foff(a.foff),
        fsrc(a.fsrc), ld(a.ld) {}
  __device__ __forceinline__ void issue(Vec<T>* slot, int row, int lane) const {
    cp_async16(slot + lane, gbase + (size_t)row * ld);
    if constexpr (NOP == 2) cp_async16(slot + 32 + lane, nbase + (size_t)row * ld);
  }
  __device__ __forceinline__ void issue_x(Vec<T>* slot, int node, int lane) const {
    cp_async16(slot + lane, xbase + (size_t)node * ld);
  }
  __device__ __forceinline__ Vec<T> load_x(int node) const { return ldv(xbase + (size_t)node * ld); }
  __device__ __forceinline__ Vec<T> value(const Vec<T>* slot, int lane, int row, const Vec<T>& x) const {
    if constexpr (NOP == 2) return combine(slot[lane], slot[32 + lane], row, x);
    else return slot[lane];
  }
  __device__ __forceinline__ Vec<T> direct(int row, const Vec<T>& x) const {
    const Vec<T> g = ldv(gbase + (size_t)row * ld);
    if constexpr (NOP == 2) return combine(g, ldv(nbase + (size_t)row * ld), row, x);
    else return g;
  }
  __device__ __forceinline__ Vec<T> combine(const Vec<T>& g, const Vec<T>& P, int row,
                                            const Vec<T>& x) const {
    constexpr int N = Vec<T>::N;
    Vec<T> r;
    if constexpr (MODE == BW_LOGSUM) {
      // g[parent] * exp(child - parent); NaN/inf weights -> 0 (engine.py:346-352)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        T w = kexp(x.v[c] - P.v[c]);
        w = isfinite(w) ? w : T(0);
        r.v[c] = g.v[c] * w;
      }
    } else {
      // zero-safe product adjoint (engine.py:358-369): (g * prod) / x; a zero
      // child gets g * (product of nonzero siblings) iff it is the only zero
      bool any_zero = false;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        r.v[c] = (g.v[c] * P.v[c]) / x.v[c];
        any_zero |= (x.v[c] == T(0));
      }
      if (any_zero) zero_path(r, g, row, x);
    }
    return r;
  }
  __device__ __noinline__ void zero_path(Vec<T>& r, const Vec<T>& g, int row, const Vec<T>& x) const {
    constexpr int N = Vec<T>::N;
    const int s0 = __ldg(foff + row), s1 = __ldg(foff + row + 1);
    T pnz[N];
    int zc[N];
#pragma unroll
    for (int c = 0; c < N; ++c) { pnz[c] = T(1); zc[c] = 0; }
    for (int s = s0; s < s1; ++s) {
      const Vec<T> y = ldv(xbase + (size_t)__ldg(fsrc + s) * ld);
#pragma unroll
      for (int c = 0; c < N; ++c) {
        if (y.v[c] == T(0)) ++zc[c];
        else pnz[c] *= y.v[c];
      }
    }
#pragma unroll
    for (int c = 0; c < N; ++c)
      if (x.v[c] == T(0)) r.v[c] = (zc[c] == 1) ? g.v[c] * pnz[c] : T(0);
  }
};

// ---- the work-item kernel ----------------------------------------------------

template <typename T, int RK>
struct OpFor { using type = SeqOp<T, RK>; };
template <typename T>
struct OpFor<T, RK_SUM> { using type = SumOp<T>; };
template <typename T>
struct OpFor<T, RK_LSE> { using type = LseOp<T>; };

constexpr int ITEM_IDX = 128;  // edge indices staged per item (longer items read idx directly)

template <typename T, int RK, typename G>
struct ItemsSmem {
  static constexpr int SLOT = (G::NOP + G::NX) * 32;  // Vec<T> per edge slot
  static constexpr size_t stage = (size_t)WARPS_PER_BLOCK * 2 * G::EB * SLOT * sizeof(Vec<T>);
  static constexpr size_t accum = (RK == RK_SUM) ? (size_t)8 * WARPS_PER_BLOCK * 32 * sizeof(Vec<T>) : 0;
  static constexpr size_t index = (size_t)WARPS_PER_BLOCK * (ITEM_IDX + 32) * sizeof(int);
  static constexpr size_t bytes = stage + accum + index;
};

template <typename T, int RK, typename G>
__global__ void __launch_bounds__(WARPS_PER_BLOCK * 32) items_kernel(LayerArgs<T> a) {
  using Op = typename OpFor<T, RK>::type;
  using S = ItemsSmem<T, RK, G>;
  constexpr int EB = G::EB, SLOT = S::SLOT;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * WARPS_PER_BLOCK + warp;
  if (item >= a.n_items) return;  // no block-wide barriers below
  Vec<T>* stage = reinterpret_cast<Vec<T>*>(smem) + (size_t)warp * 2 * EB * SLOT;
  int* widx = reinterpret_cast<int*>(smem + S::stage + S::accum) + warp * (ITEM_IDX + 32);
  int* wend = widx + ITEM_IDX;

  const int v = blockIdx.y * 32 + lane;
  const bool active = v < a.V;
  const size_t col = (size_t)v * Vec<T>::N;
  const long long ld = a.ld;
  const int4 it = __ldg(a.items + item);
  const bool leaf = it.y < 0;
  const int nn = leaf ? 1 : it.y - it.x;
  const int ne = it.w - it.z;
  const bool staged_idx = ne <= ITEM_IDX;
  const G g(a, col);
  Op op;
  if constexpr (RK == RK_LSE) op.eps = a.eps;
  if constexpr (RK == RK_SUM) {
    op.r = reinterpret_cast<Vec<T>*>(smem + S::stage) + threadIdx.x;
    op.rstride = WARPS_PER_BLOCK * 32;
  }
  // the item's edge indices and (relative) segment ends, one round trip
  if (staged_idx)
    for (int q = lane; q < ne; q += 32) widx[q] = __ldg(a.idx + it.z + q);
  if (!leaf && lane < nn) wend[lane] = __ldg(a.off + it.x + 1 + lane) - it.z;
  __syncwarp();

  // stage batch b: operand rows of edges [b*EB, b*EB+cnt) and the own value
  // of every node whose segment starts in the batch
  int xnode = 0, xstart = 0;
  auto issue = [&](int b) {
    const int base = b * EB;
    const int cnt = min(EB, ne - base);
    Vec<T>* st = stage + (b & 1) * EB * SLOT;
    if (active) {
      for (int i = 0; i < cnt; ++i) {
        const int row = staged_idx ? widx[base + i] : __ldg(a.idx + it.z + base + i);
        g.issue(st + i * SLOT, row, lane);
      }
    }
    if constexpr (G::NX) {
      if (leaf) {
        if (b == 0 && active) g.issue_x(st + G::NOP * 32, it.x, lane);
      } else {
        while (xnode < nn && xstart < base + cnt) {
          if (active) g.issue_x(st + (xstart - base) * SLOT + G::NOP * 32, it.x + xnode, lane);
          xstart = wend[xnode];
          ++xnode;
        }
      }
    }
    cp_async_commit();
  };

  const int nb = (ne + EB - 1) / EB;
  int node = 0, seg_start = 0;
  int seg_end = leaf ? ne : wend[0];
  if (leaf) op.begin_leaf(ne);
  else op.begin(seg_end);
  Vec<T> x{};
  issue(0);
  for (int b = 0; b < nb; ++b) {
    if (b + 1 < nb) {
      issue(b + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    const Vec<T>* st = stage + (b & 1) * EB * SLOT;
    const int base = b * EB;
    const int cnt = min(EB, ne - base);
    for (int i = 0; i < cnt; ++i) {
      const int k = base + i;
      if constexpr (G::NX) {
        if (k == seg_start && (!leaf || k == 0)) x = st[i * SLOT + G::NOP * 32 + lane];
      }
      if (active) {
        const int row = (G::NX && G::NOP == 2) ? (staged_idx ? widx[k] : __ldg(a.idx + it.z + k)) : 0;
        op.push(g.value(st + i * SLOT, lane, row, x));
      }
      if (!leaf && k + 1 == seg_end) {
        if (active) stv(a.out + (size_t)(it.x + node) * ld + col, op.result());
        ++node;
        if (node < nn) {
          seg_start = seg_end;
          seg_end = wend[node];
          op.begin(seg_end - seg_start);
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
  const G g(a, col);
  const Vec<T> x = g.load_x(node);
  const Vec<T> x0 = g.direct(__ldg(a.idx + s), x);
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
    constexpr size_t smem = ItemsSmem<T, RK, G>::bytes;
    static bool configured = false;  // opt in to > 48 KB dynamic smem once per kernel
    if (!configured) {
      cudaFuncSetAttribute(items_kernel<T, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      configured = true;
    }
    dim3 grid((unsigned)((a.n_items + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK), chunks);
    items_kernel<T, RK, G><<<grid, WARPS_PER_BLOCK * 32, smem, s>>>(a);
  }
  if (a.n_heavy > 0) {
    ++launched;
    dim3 grid((unsigned)a.n_heavy, chunks);
    combine_kernel<T, RK, G><<<grid, 32, 0, s>>>(a);
  }
  return launched;
}

}  // namespace klay
