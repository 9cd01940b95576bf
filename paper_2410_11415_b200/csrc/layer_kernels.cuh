// Layer kernels of libklay: one warp per (work item, 512-byte column chunk).
//
// Work items are built on the host per layer and direction (klay.cu,
// build_items; kinds documented at items_kernel). Heavy segments (fan-in
// > 129) are split at numpy's pairwise-tree leaves and finished by
// combine_kernel in tree order. Column chunks are the slow grid dimension,
// so all items of chunk 0 run before chunk 1: the previous layer's working
// set per chunk is W_prev x 512 B (35 MB at the widest layer of config C),
// which stays L2-resident while its rows are gathered ~2.7 times each.
#pragma once

#include <atomic>

#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "layer_api.h"

namespace klay {

// One warp per block: a block's resources are released as soon as its one
// item (of very uneven length) is done, so short and long items never hold
// each other's SM slots (4-warp blocks: -7 %). The MINB values are resident
// blocks (= warps) per SM the register budget is sized for; shared memory
// (one stage per warp) caps the forward and pass-through kernels at 25.
#ifndef KLAY_WARPS_PER_BLOCK
#define KLAY_WARPS_PER_BLOCK 1
#endif
constexpr int WARPS_PER_BLOCK = KLAY_WARPS_PER_BLOCK;
// staged edge indices per item (longer items read theirs from the plan):
// backward / tail, and the forward policies (a smaller block leaves room for
// one more resident warp: 23 instead of 22 per SM)
#ifndef KLAY_STAGED_IDX
#define KLAY_STAGED_IDX 128
#endif
#ifndef KLAY_FWD_STAGED_IDX
#define KLAY_FWD_STAGED_IDX 96
#endif
constexpr int TASK_EDGES = KLAY_STAGED_IDX;
#ifndef KLAY_CHUNKS_PER_WARP
#define KLAY_CHUNKS_PER_WARP 1
#endif
constexpr int CHUNKS_PER_WARP = KLAY_CHUNKS_PER_WARP;
#ifndef KLAY_PASS_MINB
#define KLAY_PASS_MINB 22  // resident blocks of the pass-through backward kernel
#endif
#ifndef KLAY_FWD_MINB
#define KLAY_FWD_MINB 25
#endif
#ifndef KLAY_LOGSUM_SE
#define KLAY_LOGSUM_SE 4
#endif
// edges per stage batch of the forward and of the pass-through / real-product
// backward (segments in short tasks stay <= 8 edges: numpy's sequential range)
#ifndef KLAY_FWD_SE
#define KLAY_FWD_SE 8
#endif
#ifndef KLAY_BWD_SE
#define KLAY_BWD_SE 8
#endif
#ifndef KLAY_LOGSUM_MINB
#define KLAY_LOGSUM_MINB 18
#endif
#ifndef KLAY_LOGSUM8_MINB
#define KLAY_LOGSUM8_MINB 8
#endif
// own-value slots per stage batch of the 8-edge log-sum backward: batches
// hold at most this many nodes (klay.cu build_items), so a stage reserves
// own values for 2 nodes instead of 8 (children of these layers average
// several parents). 11 instead of 8 resident warps per SM: config C'
// log-sum backward 3.64 -> 2.91 ms (XN 4: 3.11, 3: 3.08, 1: 2.96)
#ifndef KLAY_LOGSUM8_XN
#define KLAY_LOGSUM8_XN 2
#endif
#ifndef KLAY_LOGSUM_XN
#define KLAY_LOGSUM_XN KLAY_LOGSUM_SE  // (the 4-edge log-sum backward: no cap)
#endif


// ---- operand policies -------------------------------------------------------
// issue():  cp.async this lane's 16 bytes of every operand row of one edge
//           into the edge's staging slot (NOP operand vectors per lane)
// value():  the edge's contribution, from the staged operands
// NX:       a per-node own value is staged too (backward: the child's x)

// ---- finiteness bit masks (unary-sum aliases) --------------------------------
// Word e of a column chunk's mask holds bit l = isfinite(element e of lane l's
// vector); NV 16-byte pieces per chunk, written by lane 0 at the chunk's
// first column. All 32 lanes must call store_mask (ballots).
template <typename T>
__device__ __forceinline__ void store_mask(T* chunk0, const Vec<T>& v, int lane) {
  constexpr int N = Vec<T>::N;
  unsigned w[(N + 3) / 4 * 4];
#pragma unroll
  for (int e = 0; e < N; ++e) {
    bool fin = true;
    if constexpr (std::is_floating_point<T>::value) fin = isfinite(v.v[e]);
    w[e] = __ballot_sync(0xffffffffu, fin);
  }
#pragma unroll
  for (int e = N; e < (N + 3) / 4 * 4; ++e) w[e] = 0u;
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < (N + 3) / 4; ++q)
      *KLAY_CHK(reinterpret_cast<uint4*>(chunk0) + q, 4) = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
}
// a stand-in own value with the mask's finiteness: 0 (finite) or -inf
template <typename T>
__device__ __forceinline__ Vec<T> mask_to_x(const unsigned* w, int lane) {
  Vec<T> x;
#pragma unroll
  for (int e = 0; e < Vec<T>::N; ++e) {
    if constexpr (std::is_floating_point<T>::value) x.v[e] = ((w[e] >> lane) & 1u) ? T(0) : T(-INFINITY);
    else x.v[e] = T(0);
  }
  return x;
}

// ALIAS (log semiring, epsilon 0): a negative operand row r is a unary sum
// of the layer below that the forward never wrote; it reads its child's row
// instead, r rows before the base (the child layer precedes the sum layer in
// the trace), as the logsumexp of one element (the child, NaN for +inf)
template <typename T, bool ALIAS = false>
struct FwdGather {
  static constexpr int NOP = 1, NX = 0, SE = KLAY_FWD_SE, XPIECES = 0, XN = 0;
  static constexpr bool FWD = true, MASKX = false;
  static constexpr int CAP = KLAY_FWD_STAGED_IDX;  // staged edge indices per item
  static constexpr bool ROWV = ALIAS, MASKED_OUT = false, ALIAS_IN = ALIAS;
  static constexpr int MINB = KLAY_FWD_MINB;  // resident blocks per SM (shared memory allows 25)
  const T* base;
  int ldb;  // row stride in bytes
  int nl;
  __device__ __forceinline__ FwdGather() {}
  __device__ __forceinline__ FwdGather(const LayerArgs<T>& a, size_t col, int nl_)
      : base(a.prev + col), ldb((int)(a.ld * (long long)sizeof(T))), nl(nl_) {}
  __device__ __forceinline__ const T* row_ptr(int row) const { return row_at(base, row, ldb); }
  __device__ __forceinline__ void issue(uint4* slot, int row, int lane) const {
    cp_async_vec(slot, lane, row_ptr(row), nl);
  }
  __device__ __forceinline__ void issue_x(uint4*, int, int, int) const {}
  __device__ __forceinline__ Vec<T> x_from_stage(const uint4*, int) const { return Vec<T>{}; }
  __device__ __forceinline__ Vec<T> value(const uint4* slot, int lane, int row, const Vec<T>&) const {
    const Vec<T> v = lds_vec<T>(slot, lane);
    return (ALIAS && row < 0) ? lse_unary(v) : v;
  }
  __device__ __forceinline__ Vec<T> direct(int row, const Vec<T>&) const {
    const Vec<T> v = ldv(row_ptr(row), nl);
    return (ALIAS && row < 0) ? lse_unary(v) : v;
  }
  __device__ __forceinline__ Vec<T> load_x(int, int) const { return Vec<T>{}; }
};

// PASSA: pass-through whose outputs may carry a route's unary weight (omap
// bit 31): 1, or 0 for a non-finite value, read from the finiteness mask the
// forward left in the route top's unwritten row (xmap)
template <typename T, int MODE>
struct BwdGather {
  static constexpr bool PASSLIKE = (MODE == BW_PASS || MODE == BW_PASSA);
  static constexpr bool FWD = false;
  static constexpr bool LOGSUMLIKE = (MODE == BW_LOGSUM || MODE == BW_LOGSUM8);
  static constexpr int CAP = TASK_EDGES;  // staged edge indices per item
  static constexpr int NOP = PASSLIKE ? 1 : 2;
  static constexpr int NX = (MODE == BW_PASS) ? 0 : 1;
  // (outputs flagged in omap carry the unary weight: own value or mask needed)
  static constexpr bool ROWV = (NOP == 2), MASKED_OUT = (NX == 1), ALIAS_IN = false;
  // PASSA stages the own value only as a finiteness mask, used only by
  // flagged outputs: read it there (mask_weight), not for every node
  static constexpr bool MASKX = (MODE == BW_PASSA);
  // edges per stage batch: log-sum layers stage three rows per edge and are
  // shared-memory bound, so they use 4 (their segments are short); layers
  // whose children often have more parents use the 8-edge variant LOGSUM8
  static constexpr int SE = (MODE == BW_LOGSUM) ? KLAY_LOGSUM_SE : (MODE == BW_LOGSUM8 ? 8 : KLAY_BWD_SE);
  static constexpr int XPIECES = (MODE == BW_PASSA) ? NV : NV * 32;  // staged own value
  static constexpr int XN = (MODE == BW_LOGSUM8) ? KLAY_LOGSUM8_XN
                            : (MODE == BW_LOGSUM ? KLAY_LOGSUM_XN : SE);  // own values per stage batch
  static constexpr int MINB = (MODE == BW_PASS) ? KLAY_PASS_MINB
                              : (MODE == BW_LOGSUM ? KLAY_LOGSUM_MINB
                                 : (MODE == BW_PASSA ? KLAY_PASS_MINB
                                                     : (MODE == BW_LOGSUM8 ? KLAY_LOGSUM8_MINB : 1)));
  const T* gbase;
  const T* nbase;
  const T* xbase;
  const int* foff;
  const int* fsrc;
  unsigned ldb;  // row stride in bytes
  int nl;
  bool unary_ok;
  __device__ __forceinline__ BwdGather() {}
  __device__ __forceinline__ BwdGather(const LayerArgs<T>& a, size_t col, int nl_)
      : gbase(a.gcur + col), nbase(a.ncur + col),
        // PASSA: the masks sit at the column chunk's start of the child rows
        xbase(a.nprev + (MODE == BW_PASSA ? col - (col % (32 * NV * PIECE<T>)) : col)),
        foff(a.foff), fsrc(a.fsrc), ldb((unsigned)(a.ld * (long long)sizeof(T))), nl(nl_),
        unary_ok(a.unary_ok != 0) {}
  // Edge rows of the transposed CSR carry bit 31 when the parent is a unary
  // sum (klay.cu plan build); with epsilon 0 such a parent's value equals the
  // child's, so LOGSUM skips loading it (unary_ok) and every mode masks the bit.
  __device__ __forceinline__ bool unary_edge(int row) const {
    return LOGSUMLIKE && unary_ok && row < 0;
  }
  __device__ __forceinline__ void issue(uint4* slot, int row, int lane) const {
    const unsigned r = (unsigned)row & 0x7fffffffu;
    cp_async_vec(slot, lane, row_atu(gbase, r, ldb), nl);
    if constexpr (NOP == 2)
      if (!unary_edge(row)) cp_async_vec(slot + NV * 32, lane, row_atu(nbase, r, ldb), nl);
  }
  // own value of an output (omap entry `out`, value row `xrow`). PASSA:
  // flagged outputs only, as the finiteness mask at the chunk's start
  __device__ __forceinline__ void issue_x(uint4* slot, int out, int xrow, int lane) const {
    if (MODE == BW_PASSA) {
      if (out < 0 && lane < NV)
        cp_async16(slot + lane, row_atu(xbase, (unsigned)xrow, ldb) + lane * (16 / sizeof(T)));
    } else {
      cp_async_vec(slot, lane, row_atu(xbase, (unsigned)xrow, ldb), nl);
    }
  }
  __device__ __forceinline__ Vec<T> x_from_stage(const uint4* slot, int lane) const {
    if (MODE == BW_PASSA) return mask_to_x<T>(reinterpret_cast<const unsigned*>(slot), lane);
    return lds_vec<T>(slot, lane);
  }
  // PASSA, flagged output: unary(g, x) straight from the staged mask bits
  // (g where the child's value is finite, g * 0 elsewhere)
  __device__ __forceinline__ static Vec<T> mask_weight(Vec<T> g, const uint4* slot, int lane) {
    const unsigned* w = reinterpret_cast<const unsigned*>(slot);
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c)
      if (!((w[c] >> lane) & 1u)) g.v[c] = g.v[c] * T(0);
    return g;
  }
  __device__ __forceinline__ Vec<T> load_x(int out, int xrow) const {
    if (MODE == BW_PASSA) {
      if (out >= 0) return Vec<T>{};
      const int j = xrow;
      unsigned w[NV * 4];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const uint4 u = __ldcg(KLAY_CHK(reinterpret_cast<const uint4*>(row_atu(xbase, (unsigned)j, ldb)) + q, 5));
        w[4 * q] = u.x; w[4 * q + 1] = u.y; w[4 * q + 2] = u.z; w[4 * q + 3] = u.w;
      }
      return mask_to_x<T>(w, (int)(threadIdx.x & 31));
    }
    return ldv(row_atu(xbase, (unsigned)xrow, ldb), nl);
  }
  __device__ __forceinline__ Vec<T> value(const uint4* slot, int lane, int row, const Vec<T>& x) const {
    if constexpr (NOP == 2) {
      if (unary_edge(row)) return unary(lds_vec<T>(slot, lane), x);
      return combine(lds_vec<T>(slot, lane), lds_vec<T>(slot + NV * 32, lane), row, x);
    } else {
      return lds_vec<T>(slot, lane);
    }
  }
  __device__ __forceinline__ Vec<T> direct(int row, const Vec<T>& x) const {
    const unsigned r = (unsigned)row & 0x7fffffffu;
    const Vec<T> g = ldv(row_atu(gbase, r, ldb), nl);
    if constexpr (NOP == 2) {
      if (unary_edge(row)) return unary(g, x);
      return combine(g, ldv(row_atu(nbase, r, ldb), nl), row, x);
    } else {
      return g;
    }
  }
  // weight exp(child - parent) of a unary parent: exp(0) = 1 for a finite
  // child; a -inf, +inf (parent NaN) or NaN child gives exp(NaN), masked to 0
  // (engine.py:346-352)
  __device__ __forceinline__ static Vec<T> unary(const Vec<T>& g, const Vec<T>& x) {
    Vec<T> r;
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c) r.v[c] = isfinite(x.v[c]) ? g.v[c] : g.v[c] * T(0);
    return r;
  }
  // g[parent] * exp(child - parent); NaN/inf weights -> 0 (engine.py:346-352).
  // (Unary parents never get here: their edges are flagged, see unary().
  // A child equal to its parent gets exp(0) = 1 exactly, so no special
  // case: one uniform path, no lane divergence.)
  __device__ __forceinline__ static Vec<T> logsum_edge(const Vec<T>& g, const Vec<T>& P,
                                                       const Vec<T>& x) {
    Vec<T> r;
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c) {
      T w = kexp(x.v[c] - P.v[c]);
      w = isfinite(w) ? w : T(0);
      r.v[c] = g.v[c] * w;
    }
    return r;
  }
  __device__ __forceinline__ Vec<T> combine(const Vec<T>& g, const Vec<T>& P, int row,
                                            const Vec<T>& x) const {
    constexpr int N = Vec<T>::N;
    Vec<T> r;
    if constexpr (LOGSUMLIKE) {
      r = logsum_edge(g, P, x);
    } else {
      // zero-safe product adjoint (engine.py:358-369): (g * prod) / x; a zero
      // child gets g * (product of nonzero siblings) iff it is the only zero,
      // any child of a segment holding a zero gets exactly 0. A segment with
      // a zero has a product of 0, or NaN (0 * inf): both send it to
      // zero_path, which counts the zeros (an underflow or a NaN input with
      // no zero keeps the plain formula, as in the reference)
      bool any_zero = false;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        r.v[c] = (g.v[c] * P.v[c]) / x.v[c];
        any_zero |= (x.v[c] == T(0)) | (P.v[c] == T(0)) | (P.v[c] != P.v[c]);
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
      const Vec<T> y = ldv(row_atu(xbase, (unsigned)__ldg(fsrc + s), ldb), nl);
#pragma unroll
      for (int c = 0; c < N; ++c) {
        if (y.v[c] == T(0)) ++zc[c];
        else pnz[c] *= y.v[c];
      }
    }
#pragma unroll
    for (int c = 0; c < N; ++c) {
      if (x.v[c] == T(0)) r.v[c] = (zc[c] == 1) ? g.v[c] * pnz[c] : T(0);
      else if (zc[c] > 0) r.v[c] = T(0);  // (a zero sibling: 0 even for an infinite adjoint)
    }
  }
};

// ---- the work-item kernel ----------------------------------------------------
//
// Item kinds (int4 {x, y, z, w}, built by klay.cu build_items):
//   short task   y > 0   nodes [x, y), edges [z, w): whole segments of at most
//                        G::SE edges each; staged in node-aligned batches of
//                        <= SE edges and reduced node by node
//   long segment y == 0  node x, edges [z, w): one segment, x0 = edge z and the
//                        tail in rounds of 8 aligned with numpy's 8-way
//                        pairwise accumulators (statically indexed registers)
//   leaf         y < 0   one pairwise leaf [z, w) of node x's tail; the partial
//                        goes to scratch slot -y-1 (combine_kernel finishes)
// Every lane owns one 16-byte column vector; rows are staged with cp.async
// into a double-buffered per-warp shared-memory stage, so a warp keeps up to
// two batches of 512-byte row chunks in flight with no register cost.

constexpr int TASK_NODES = 31;   // max nodes of a short task (one lane per segment offset)

// ---- per-item index data (warp-private shared memory) ----------------------
// The structure of an item (descriptor, batch mask, edge indices, segment
// offsets) does not depend on values: the tail kernel loads it for the next
// layer while the cluster barrier of the current layer is still open.
// CAP: staged edge indices (a multiple of 32); longer items read theirs
// from the plan. The forward policies use a smaller block (shared memory for
// one more resident warp); the backward and the tail kernel use TASK_EDGES.
template <int CAP>
struct ItemIndexT {
  static constexpr int cap = CAP;
  int4 it;            // item descriptor (see items_kernel)
  unsigned mask;      // short task: bit j set when node j starts a stage batch
  int pad[3];
  int widx[CAP];
  int woff[32];       // short task: segment offsets relative to it.z
  int wmap[32];       // LayerArgs::omap entries of the item's nodes
  int wxmap[32];      // LayerArgs::xmap entries
};
using ItemIndex = ItemIndexT<TASK_EDGES>;

template <typename T, typename G>
struct ItemsSmem {
  static constexpr int SE = G::SE;                 // edges per stage batch (= max short segment)
  // stage units: 16-byte pieces; a staged vector is NV x 32 lanes of pieces
  static constexpr int EV = G::NOP * NV * 32;      // pieces per staged edge
  static constexpr int XV = G::NX * G::XPIECES;    // pieces per staged own value
  static constexpr int STAGE_V = SE * EV + G::XN * XV;  // pieces per stage (<= XN nodes per batch)
  static constexpr size_t stage_bytes = (size_t)2 * STAGE_V * 16;
  // + one ItemIndex
#ifndef KLAY_WARP_ALIGN
#define KLAY_WARP_ALIGN 16
#endif
  static constexpr size_t warp_bytes =
      (stage_bytes + sizeof(ItemIndexT<G::CAP>) + KLAY_WARP_ALIGN - 1) / KLAY_WARP_ALIGN * KLAY_WARP_ALIGN;
  static constexpr size_t bytes = warp_bytes * WARPS_PER_BLOCK;
};

template <typename T, int RK>
__device__ __forceinline__ void seq_combine(Vec<T>& acc, const Vec<T>& x) {
#pragma unroll
  for (int c = 0; c < Vec<T>::N; ++c) {
    if constexpr (RK == RK_PROD) acc.v[c] = acc.v[c] * x.v[c];
    else if constexpr (RK == RK_MAX) acc.v[c] = npmax(acc.v[c], x.v[c]);
    else if constexpr (RK == RK_AND) acc.v[c] = acc.v[c] & x.v[c];
    else if constexpr (RK == RK_OR) acc.v[c] = acc.v[c] | x.v[c];
    else acc.v[c] = npmin(acc.v[c], x.v[c]);
  }
}

template <typename T>
__device__ __forceinline__ Vec<T> combine8(const Vec<T> (&r)[8]) {
  Vec<T> res;
#pragma unroll
  for (int c = 0; c < Vec<T>::N; ++c)
    res.v[c] = ((r[0].v[c] + r[1].v[c]) + (r[2].v[c] + r[3].v[c])) +
               ((r[4].v[c] + r[5].v[c]) + (r[6].v[c] + r[7].v[c]));
  return res;
}

// registers of one lane while an ItemIndex is in flight
template <int CAP>
struct ItemRegsT {
  int4 it;
  unsigned mask;
  int idx[CAP / 32];
  int off;
  int map, xmap;
};
using ItemRegs = ItemRegsT<TASK_EDGES>;

// Index data of item k (descriptor it/mask). Items with <= PADW edges have
// their edge indices, raw segment offsets and maps in padded per-item rows
// (klay.cu pad_items), loaded together with the descriptor: one round trip.
// Longer items load their indices after the descriptor.
constexpr int PADW = 32;

// The maps are normalized here, once per item, so the per-node code reads
// them unconditionally: wmap = output row of item node `lane` (the node id
// itself without an omap); wxmap = own-value row (backward; the node id
// without an xmap) or, forward, the mask row (-1: no mask, also whenever the
// call stores no masks).
template <typename T, bool FWD, int CAP = TASK_EDGES>
__device__ __forceinline__ ItemRegsT<CAP> item_regs_from(const LayerArgs<T>& a, int k, int4 it,
                                                         unsigned mask, int lane) {
  ItemRegsT<CAP> r;
  r.it = it;
  r.mask = mask;
  const size_t pk = (size_t)k * PADW + lane;
  const int p0 = __ldg(a.pidx + pk);
  const int o0 = __ldg(a.poff + pk);
  r.map = a.pmap ? __ldg(a.pmap + pk) : it.x + lane;
  if (FWD) r.xmap = (a.pxmap && a.mbase) ? __ldg(a.pxmap + pk) : -1;
  else r.xmap = a.pxmap ? __ldg(a.pxmap + pk) : it.x + lane;
  const int ne = r.it.w - r.it.z;
  if (ne <= PADW) {
    r.idx[0] = p0;
#pragma unroll
    for (int q = 1; q < CAP / 32; ++q) r.idx[q] = 0;
  } else {
#pragma unroll
    for (int q = 0; q < CAP / 32; ++q) {
      const int e = q * 32 + lane;
      r.idx[q] = (ne <= CAP && e < ne) ? __ldg(a.idx + r.it.z + e) : 0;
    }
  }
  r.off = r.it.y > 0 ? o0 - r.it.z : 0;  // segment offsets relative to the first edge
  return r;
}

template <typename T, bool FWD, int CAP = TASK_EDGES>
__device__ __forceinline__ ItemRegsT<CAP> load_item_regs(const LayerArgs<T>& a, int item, int lane) {
  return item_regs_from<T, FWD, CAP>(a, item, __ldg(a.items + item), __ldg(a.masks + item), lane);
}

template <int CAP>
__device__ __forceinline__ void store_item_regs(ItemIndexT<CAP>* ib, const ItemRegsT<CAP>& r, int lane) {
  if (lane == 0) {
    ib->it = r.it;
    ib->mask = r.mask;
  }
#pragma unroll
  for (int q = 0; q < CAP / 32; ++q) ib->widx[q * 32 + lane] = r.idx[q];
  ib->woff[lane] = r.off;
  ib->wmap[lane] = r.map;
  ib->wxmap[lane] = r.xmap;
}

// Run one item (index data in `ib`, synchronized) for one 512-byte column
// chunk; `stage` is the warp's double-buffered staging area.
// this lane's columns in chunk `chunk`: na pieces inside the row (stored),
// nl = max(na, 1) loadable pieces, col = element offset of piece 0
struct LaneCols {
  int na, nl;
  size_t col;
};
template <typename T>
__device__ __forceinline__ LaneCols lane_cols(int V, int chunk, int lane) {
  const int vb = chunk * 32 * NV + lane;
  LaneCols c;
  c.na = min(NV, max(0, (V - vb + 31) / 32));
  c.nl = c.na > 0 ? c.na : 1;
  c.col = (size_t)(c.na > 0 ? vb : 0) * PIECE<T>;
  return c;
}

template <typename T, int RK, typename G>
__device__ __forceinline__ void process_heavy(const LayerArgs<T>& a, int h, int chunk, int lane,
                                              uint4* sm, int sm_pieces);

template <typename T, int RK, typename G, int CAP>
__device__ __forceinline__ void run_item(const LayerArgs<T>& a, const ItemIndexT<CAP>* ib, int chunk,
                                         uint4* stage, int lane) {
  using S = ItemsSmem<T, G>;
  constexpr int SE = S::SE, EV = S::EV, XV = S::XV, STAGE_V = S::STAGE_V;
  const int* widx = ib->widx;
  const int* woff = ib->woff;
  const int* wmap = ib->wmap;
  const int* wxmap = ib->wxmap;

  // Lanes (pieces) past the row work on valid columns and never store: the
  // whole warp runs the same instruction stream without divergence.
  const LaneCols lc = lane_cols<T>(a.V, chunk, lane);
  const int na = lc.na;
  const size_t col = lc.col;
  const long long ld = a.ld;
  const unsigned ldbu = (unsigned)(ld * (long long)sizeof(T));  // row stride in bytes
  T* const outc = a.out + col;  // this lane's column of the output rows
  const int4 it = ib->it;
  const int ne = it.w - it.z;
  const G g(a, col, lc.nl);
  const bool staged_idx = ne <= CAP;

  if (it.y > 0) {
    // ======================= short task =======================
    // nodes [nb, nb+nn), every segment <= SE edges; the node-aligned stage
    // batches (<= SE edges, host-computed bit mask) are staged two at a time
    // and reduced node by node
    const int nb = it.x, nn = it.y - it.x;
    // node id of item node nd: output row / own-value row (omap: compacted
    // item sets and alias outputs, see LayerArgs)
    auto nid = [&](int nd) { return wmap[nd]; };   // (maps normalized: item_regs_from)
    auto xid = [&](int nd) { return wxmap[nd]; };
    const size_t col0 = (size_t)chunk * 32 * NV * PIECE<T>;  // the chunk's first column
    unsigned m_issue = ib->mask, m_scan = ib->mask;
    auto next_batch = [&](unsigned& m, int& n0, int& n1) {
      n0 = __ffs(m) - 1;
      m &= m - 1;
      n1 = m ? __ffs(m) - 1 : nn;
    };
    auto issue = [&](int b) {
      uint4* st = stage + (b & 1) * STAGE_V;
      int n0, n1;
      next_batch(m_issue, n0, n1);
      const int eb = woff[n0], cnt = woff[n1] - eb;
      for (int i = 0; i < cnt; ++i) g.issue(st + i * EV, widx[eb + i], lane);
      if constexpr (G::NX)
        for (int nd = n0; nd < n1; ++nd) g.issue_x(st + SE * EV + (nd - n0) * XV, nid(nd), xid(nd), lane);
      cp_async_commit();
    };
    const int nbat = __popc(ib->mask);
    issue(0);
    for (int b = 0; b < nbat; ++b) {
      if (b + 1 < nbat) {
        issue(b + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      const uint4* st = stage + (b & 1) * STAGE_V;
      int n0, n1;
      next_batch(m_scan, n0, n1);
      const int eb = woff[n0];
      for (int nd = n0; nd < n1; ++nd) {
        const int sb = woff[nd] - eb, n = woff[nd + 1] - woff[nd];
        Vec<T> x{};
        if constexpr (G::NX && !G::MASKX) x = g.x_from_stage(st + SE * EV + (nd - n0) * XV, lane);
        auto val = [&](int e) {
          return g.value(st + e * EV, lane, G::ROWV ? widx[eb + e] : 0, x);
        };
        Vec<T> out;
        if constexpr (RK == RK_SUM) {
          // x0 + (-0 + x1 + ... + x_{n-1}): n <= 8 keeps numpy's sequential branch
          auto sum = [&](auto&& v) {
            Vec<T> o = v(sb);
            if (n > 1) {
              Vec<T> acc = v(sb + 1);
              for (int j = 2; j < n; ++j) acc = vadd(acc, v(sb + j));
              o = vadd(o, acc);
            }
            return o;
          };
          if constexpr (G::ALIAS_IN) {
            // aliased operands (negative rows) read as logsumexp of one
            // element: only a +inf one changes (to NaN), and then the plain
            // sum is +inf or NaN -- redo the rare +inf results transformed
            out = sum([&](int e) { return lds_vec<T>(st + e * EV, lane); });
            bool redo = false;
#pragma unroll
            for (int c = 0; c < Vec<T>::N; ++c) redo |= (out.v[c] == T(INFINITY));
            if (redo) out = sum([&](int e) { return g.value(st + e * EV, lane, widx[eb + e], x); });
          } else {
            out = sum(val);
          }
        } else if constexpr (RK == RK_LSE) {
          out = val(sb);
          // a unary sum with epsilon 0 is an exact copy: log(exp(x - x) + 0) + x
          // == x, and -inf stays -inf (uniform branch: no exp/log issued)
          if (n > 1 || a.eps != T(0)) {
            LseOp<T> op;
            op.eps = a.eps;
            op.begin(n);
            op.push(out);
            for (int j = 1; j < n; ++j) op.push(val(sb + j));
            out = op.result();
          } else {
            out = lse_unary(out);
          }
        } else {
          out = val(sb);
          for (int j = 1; j < n; ++j) seq_combine<T, RK>(out, val(sb + j));
        }
        const int id = nid(nd);
        if constexpr (G::MASKED_OUT) {
          if (id < 0) {
            if constexpr (G::MASKX) out = G::mask_weight(out, st + SE * EV + (nd - n0) * XV, lane);
            else out = G::unary(out, x);
          }
        }
        stv(row_atu(outc, (unsigned)id & 0x7fffffffu, ldbu), out, na);
        if constexpr (G::FWD) {
          const int mr = wxmap[nd];
          if (mr >= 0) store_mask(row_atu(a.mbase + col0, (unsigned)mr, ldbu), out, lane);
        }
      }
    }
    return;
  }

  // ===================== long segment / leaf =====================
  const bool leaf = it.y < 0;
  const int node = wmap[0];  // output (see the short path)
  const int xnode = wxmap[0];
  const int t0 = leaf ? 0 : 1;      // first tail edge (relative)
  const int m = ne - t0;            // tail length
  Vec<T> x{};
  if constexpr (G::NX) x = g.load_x(node, xnode);
  auto row_of = [&](int e) { return staged_idx ? widx[e] : __ldg(a.idx + it.z + e); };
  // round t stages tail elements [8t, 8t+8)
  // rounds of 8 are double-buffered when a stage holds 8 edges; policies
  // with smaller stages (SE < 8) use both stages as one 8-edge buffer
  constexpr bool DB = SE >= 8;
  auto issue = [&](int t) {
    uint4* st = DB ? stage + (t & 1) * STAGE_V : stage;
    const int base = t0 + 8 * t;
    const int cnt = min(8, ne - base);
    const int my_row = (lane < cnt) ? row_of(base + lane) : 0;
    for (int i = 0; i < cnt; ++i) g.issue(st + i * EV, __shfl_sync(0xffffffffu, my_row, i), lane);
    cp_async_commit();
  };
  const int nr = (m + 7) / 8;
  Vec<T> x0{};
  if (!leaf) x0 = g.direct(row_of(0), x);
  if (nr > 0) issue(0);
  const int mainend = m - (m & 7);
  Vec<T> r[8];
  Vec<T> res = vfill<T>(T(-0.0));  // SUM tail accumulator
  Vec<T> acc = x0;                 // SEQ accumulator
  LseOp<T> lse;
  if constexpr (RK == RK_LSE) {
    lse.eps = a.eps;
    lse.begin(ne);
    if (!leaf) lse.push(x0);
  }
  for (int t = 0; t < nr; ++t) {
    if (DB && t + 1 < nr) {
      issue(t + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    const uint4* st = DB ? stage + (t & 1) * STAGE_V : stage;
    const int base = t0 + 8 * t;
    const int cnt = min(8, ne - base);
    auto val = [&](int i) {
      return g.value(st + i * EV, lane, G::ROWV ? row_of(base + i) : 0, x);
    };
    if constexpr (RK == RK_SUM) {
      if (8 * t < mainend) {
        // a full round of numpy's 8 pairwise accumulators (t is warp-uniform:
        // two loops instead of a per-element select)
        if (t == 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k) r[k] = val(k);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) r[k] = vadd(r[k], val(k));
        }
      } else {
        if (m >= 8) res = combine8(r);
        for (int i = 0; i < cnt; ++i) res = vadd(res, val(i));
      }
    } else if constexpr (RK == RK_LSE) {
      for (int i = 0; i < cnt; ++i) lse.push(val(i));
    } else {
      int i = 0;
      if (leaf && t == 0) acc = val(i++);
      for (; i < cnt; ++i) seq_combine<T, RK>(acc, val(i));
    }
    if (!DB && t + 1 < nr) issue(t + 1);  // (each lane reuses only its own slots)
  }
  if constexpr (RK == RK_SUM) {
    if (m >= 8 && mainend == m) res = combine8(r);
  }
  if (leaf) {
    // (stores of lanes past the row are empty: na == 0)
    const int slot = -it.y - 1;
    if constexpr (RK == RK_LSE) {
      stv(a.scratch + (size_t)slot * ld + col, lse.m, na);
      stv(a.scratch + a.tpart + (size_t)slot * ld + col, lse.t, na);
    } else if constexpr (RK == RK_SUM) {
      stv(a.scratch + (size_t)slot * ld + col, res, na);
    } else {
      stv(a.scratch + (size_t)slot * ld + col, acc, na);
    }
    if (a.hcount) {
      // the warp that writes the last leaf partial of (segment, chunk)
      // finishes the segment in tree order. The warp's partial stores are
      // ordered before lane 0's counter increment by __syncwarp, and that
      // increment is an acquire-release atomic at GPU scope: every partial
      // published before its count is visible to the warp that takes the
      // last count (read back through L2 after it). (One MEMBAR.ALL instead
      // of two sequentially consistent __threadfence()s.)
      const int h = (int)ib->mask;
      __syncwarp();
      int* cnt = KLAY_CHK(a.hcount + (size_t)h * ((a.V + 32 * NV - 1) / (32 * NV)) + chunk, 6);
      int last = 0;
      if (lane == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        last = (int)old == __ldg(&a.heavy[h].z) - 1;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __syncwarp();  // (orders the other lanes' reads after lane 0's acquire)
        // (inlined: an out-of-line call here costs the whole kernel ~10%)
        process_heavy<T, RK, G>(a, h, chunk, lane, stage, 2 * STAGE_V);
        if (lane == 0) *cnt = 0;  // ready for the next layer / pass
      }
    }
  } else {
    Vec<T> out;
    if constexpr (RK == RK_SUM) out = (m == 0) ? x0 : vadd(x0, res);
    else if constexpr (RK == RK_LSE) out = lse.result();
    else out = acc;
    if constexpr (G::FWD) {  // (all lanes: ballots)
      if (xnode >= 0) store_mask(a.mbase + (size_t)xnode * ld + (size_t)chunk * 32 * NV * PIECE<T>, out, lane);
    }
    if (na == 0) return;
    if constexpr (G::MASKED_OUT) {
      if (node < 0) out = G::unary(out, x);
    }
    stv(row_atu(outc, (unsigned)node & 0x7fffffffu, ldbu), out, na);
  }
}

template <typename T, int RK, typename G>
__global__ void __launch_bounds__(WARPS_PER_BLOCK * 32, G::MINB) items_kernel(LayerArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  chk_enter(a.chk);
  using S = ItemsSmem<T, G>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * WARPS_PER_BLOCK + warp;
  if (item >= a.n_items) return;  // no block-wide barriers inside
  unsigned char* wbase = smem + (size_t)warp * S::warp_bytes;
  ItemIndexT<G::CAP>* ib = reinterpret_cast<ItemIndexT<G::CAP>*>(wbase + S::stage_bytes);
  // The item's index data is plan data: load it before waiting on the
  // previous layer's kernel (programmatic dependent launch, launch_layer),
  // and let the next layer's blocks start their own prologue meanwhile.
  const ItemRegsT<G::CAP> r = load_item_regs<T, G::FWD, G::CAP>(a, item, lane);
#ifndef KLAY_NO_GDC
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
  store_item_regs(ib, r, lane);
  __syncwarp();
  // CHUNKS_PER_WARP consecutive column chunks per warp share the index data
  const int nch = (a.V + 32 * NV - 1) / (32 * NV);
  const int gy = a.rev ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y;
#pragma unroll 1
  for (int k = 0; k < CHUNKS_PER_WARP; ++k) {
    const int chunk = gy * CHUNKS_PER_WARP + (a.rev ? CHUNKS_PER_WARP - 1 - k : k);
    if (chunk >= nch) continue;
    if (k > 0) __syncwarp();  // the previous chunk is done with the stage
    run_item<T, RK, G, G::CAP>(a, ib, chunk, reinterpret_cast<uint4*>(wbase), lane);
  }
}

// KLAY_NO_PDL=1 launches layer kernels fully serialized (A/B switch)
// Kernel attributes (shared-memory opt-in, carveout, cluster size) are set
// once per kernel and device: `mask` holds one bit per configured device.
inline bool needs_config(std::atomic<unsigned>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  return !(mask.fetch_or(bit) & bit);
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("KLAY_NO_PDL");
    return !(e && *e && *e != '0');
  }();
  return on;
}

// ---- heavy-segment combine: x0 (+) leaf partials in order ---------------------

// `sm` (sm_pieces 16-byte pieces of warp-private shared memory) stages the
// leaf partials with one round of independent cp.async when they fit.
template <typename T, int RK, typename G>
__device__ __forceinline__ void process_heavy(const LayerArgs<T>& a, int h, int chunk, int lane,
                                              uint4* sm, int sm_pieces) {
  // (every lane runs to the end: stores are masked by na, mask ballots need all)
  const LaneCols lc = lane_cols<T>(a.V, chunk, lane);
  const int nl = lc.nl;
  const size_t col = lc.col;
  const long long ld = a.ld;
  const int4 hv = __ldg(a.heavy + h);
  const int node = hv.x, slot0 = hv.y, nleaf = hv.z;
  const int s = __ldg(a.off + node);
  const int n = __ldg(a.off + node + 1) - s;
  const int id = a.omap ? __ldg(a.omap + node) : node;    // output row
  const int xid = a.xmap ? __ldg(a.xmap + node) : node;  // own-value / mask row
  const G g(a, col, nl);
  const Vec<T> x = g.load_x(id, xid);
  const Vec<T> x0 = g.direct(__ldg(a.idx + s), x);
  Vec<T> res;
  if constexpr (RK == RK_SUM) {
    if (nleaf * 32 * NV <= sm_pieces) {
      for (int l = 0; l < nleaf; ++l)
        cp_async_vec(sm + (size_t)l * 32 * NV, lane, a.scratch + (size_t)(slot0 + l) * ld + col, nl);
      cp_async_commit();
      cp_async_wait<0>();
      int leaf = 0;
      res = vadd(x0, tree_sum_smem<T>(sm, lane, leaf, n - 1));
    } else {
      int leaf = slot0;
      res = vadd(x0, tree_sum(a.scratch + col, ld, leaf, n - 1, nl));
    }
  } else if constexpr (RK == RK_LSE) {
    LseOp<T> op;
    op.eps = a.eps;
    op.begin(n);
    op.push(x0);
    // leaf partials in groups of 4: the loads of a group are issued together
    for (int l0 = 0; l0 < nleaf; l0 += 4) {
      Vec<T> pm[4], pt[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int l = min(l0 + j, nleaf - 1);
        pm[j] = ldv(a.scratch + (size_t)(slot0 + l) * ld + col, nl);
        pt[j] = ldv(a.scratch + a.tpart + (size_t)(slot0 + l) * ld + col, nl);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (l0 + j < nleaf) {
#pragma unroll
          for (int c = 0; c < Vec<T>::N; ++c) lse_merge(op.m.v[c], op.t.v[c], pm[j].v[c], pt[j].v[c]);
        }
      }
    }
    res = op.result();
  } else {
    SeqOp<T, RK> op;
    op.begin(n);
    op.push(x0);
    for (int l = 0; l < nleaf; ++l) op.push(ldv(a.scratch + (size_t)(slot0 + l) * ld + col, nl));
    res = op.result();
  }
  if (a.mbase) {
    if (xid >= 0) store_mask(a.mbase + (size_t)xid * ld + (size_t)chunk * 32 * NV * PIECE<T>, res, lane);
  }
  if constexpr (G::MASKED_OUT) {
    if (id < 0) res = G::unary(res, x);
  }
  stv(a.out + (size_t)(id & 0x7fffffff) * ld + col, res, lc.na);
}

constexpr int COMBINE_LEAVES = 64;  // leaf partials staged per combine warp

template <typename T, int RK, typename G>
__global__ void __launch_bounds__(32) combine_kernel(LayerArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  chk_enter(a.chk);
  const int h = blockIdx.x;
  if (h >= a.n_heavy) return;
  process_heavy<T, RK, G>(a, h, blockIdx.y, threadIdx.x, reinterpret_cast<uint4*>(smem),
                          COMBINE_LEAVES * 32 * NV);
}

template <typename T, int RK, typename G>
inline int launch_layer(const LayerArgs<T>& a, cudaStream_t s) {
  const unsigned chunks = (unsigned)((a.V + 32 * NV - 1) / (32 * NV));
  int launched = 0;
  if (a.n_items > 0) {
    ++launched;
    constexpr size_t smem = ItemsSmem<T, G>::bytes;
    static std::atomic<unsigned> configured{0};  // opt in to > 48 KB dynamic smem
    if (needs_config(configured)) {
      cudaFuncSetAttribute(items_kernel<T, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      // one carveout for every layer kernel: consecutive launches never wait
      // for an L1/shared-memory reconfiguration of the SMs
      cudaFuncSetAttribute(items_kernel<T, RK, G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(combine_kernel<T, RK, G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((a.n_items + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK),
                       (chunks + CHUNKS_PER_WARP - 1) / CHUNKS_PER_WARP);
    cfg.blockDim = dim3(WARPS_PER_BLOCK * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, items_kernel<T, RK, G>, a);
  }
  if (a.n_heavy > 0 && !a.hcount) {
    ++launched;
    constexpr size_t csmem = (size_t)COMBINE_LEAVES * 32 * NV * 16;
    static std::atomic<unsigned> cconf{0};
    if (needs_config(cconf))
      cudaFuncSetAttribute(combine_kernel<T, RK, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)csmem);
    dim3 grid((unsigned)a.n_heavy, chunks);
    combine_kernel<T, RK, G><<<grid, 32, csmem, s>>>(a);
  }
  return launched;
}

// ---- persistent tail: all thin upper layers in one launch ---------------------
//
// One thread-block cluster per 512-byte column chunk (batch columns are
// independent, so a cluster never waits for another); the cluster's warps
// share each layer's work items and meet at a cluster barrier
// (barrier.cluster arrive.release / wait.acquire) between layers. Values
// written by one CTA are read by the others through L2 (cp.async.cg and
// ld.global.cg), which the barrier's release/acquire ordering makes safe.

#ifndef KLAY_TAIL_WARPS
#define KLAY_TAIL_WARPS 8
#endif
constexpr int TAIL_WARPS = KLAY_TAIL_WARPS;

// first-item descriptor of every tail layer for one warp (loaded once)
struct TailDesc {
  int4 it;
  unsigned mask;
  int pad[3];
};

// per warp: stage sized for the larger policy, one ItemIndex, the descriptor table
template <typename T, typename GP, typename GS>
struct TailSmem {
  static constexpr size_t stage_max = ItemsSmem<T, GP>::stage_bytes > ItemsSmem<T, GS>::stage_bytes
                                         ? ItemsSmem<T, GP>::stage_bytes
                                         : ItemsSmem<T, GS>::stage_bytes;
  static constexpr size_t item_bytes = (stage_max + sizeof(ItemIndex) + 127) / 128 * 128;
  static constexpr size_t warp_bytes = item_bytes + sizeof(TailDesc) * TAIL_MAX_LAYERS;
  // as many warps (<= TAIL_WARPS) as fit the 227 KB of shared memory
  static constexpr int warps = (227 * 1024) / warp_bytes < TAIL_WARPS ? (int)((227 * 1024) / warp_bytes)
                                                                      : TAIL_WARPS;
  static constexpr size_t bytes = warp_bytes * warps;
};

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <typename T, int RKP, int RKS, typename GP, typename GS>
__global__ void __launch_bounds__(TailSmem<T, GP, GS>::warps * 32, 1)
    tail_kernel(const __grid_constant__ TailArgs<T> t) {
  static_assert(GP::FWD == GS::FWD, "a tail runs one direction");
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) unsigned char smem[];
  chk_enter(t.layer[0].chk);
  cg::cluster_group cluster = cg::this_cluster();
  const int csize = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int chunk = blockIdx.x / csize;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + (size_t)warp * TailSmem<T, GP, GS>::warp_bytes;
  uint4* stage = reinterpret_cast<uint4*>(wbase);
  constexpr size_t stage_bytes = ItemsSmem<T, GP>::stage_bytes > ItemsSmem<T, GS>::stage_bytes
                                     ? ItemsSmem<T, GP>::stage_bytes
                                     : ItemsSmem<T, GS>::stage_bytes;
  ItemIndex* ib = reinterpret_cast<ItemIndex*>(wbase + stage_bytes);
  constexpr int TW = TailSmem<T, GP, GS>::warps;
  const int w = rank * TW + warp, cw = csize * TW;
  auto stamp = [&](int i, int k) {  // KLAY_TAIL_TRACE debug timestamps
    if (t.trace_ts && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      t.trace_ts[i * 4 + k] = ns;
    }
  };
  {
    // pull every tail layer's structure into L2 up front
    const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long gthreads = (long long)gridDim.x * blockDim.x;
    for (int r = 0; r < 4; ++r) {
      const char* base = static_cast<const char*>(t.pf_ptr[r]);
      for (long long o = gtid * 128; o < t.pf_bytes[r]; o += gthreads * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + o));
    }
  }
  // Every layer's first item for this warp: the descriptors of all layers
  // are loaded once (lane-parallel, one round trip) and the index data of
  // layer i+1 is requested at the start of layer i, so no layer waits on a
  // dependent index load after its barrier.
  TailDesc* desc = reinterpret_cast<TailDesc*>(wbase + TailSmem<T, GP, GS>::item_bytes);
  for (int l = lane; l < t.n; l += 32) {
    if (w < t.layer[l].n_items) {
      desc[l].it = __ldg(t.layer[l].items + w);
      desc[l].mask = __ldg(t.layer[l].masks + w);
    }
  }
  __syncwarp();
  ItemRegs next;
  if (t.n > 0 && w < t.layer[0].n_items)
    next = item_regs_from<T, GP::FWD>(t.layer[0], w, desc[0].it, desc[0].mask, lane);
  // all of the above is plan data: wait for the previous kernel's values
  // only now (programmatic dependent launch), and let the next kernel's
  // blocks take the SMs the tail leaves idle for their own prologue
#ifndef KLAY_NO_GDC
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
  for (int i = 0; i < t.n; ++i) {
    const LayerArgs<T>& a = t.layer[i];
    stamp(i, 0);
    const ItemRegs cur = next;
    if (i + 1 < t.n && w < t.layer[i + 1].n_items)
      next = item_regs_from<T, GP::FWD>(t.layer[i + 1], w, desc[i + 1].it, desc[i + 1].mask, lane);
    if (!t.debug_skip) {
      for (int it = w; it < a.n_items; it += cw) {
        __syncwarp();  // previous item done with ib
        store_item_regs(ib, it == w ? cur : load_item_regs<T, GP::FWD>(a, it, lane), lane);
        __syncwarp();
        if (a.prod) run_item<T, RKP, GP>(a, ib, chunk, stage, lane);
        else run_item<T, RKS, GS>(a, ib, chunk, stage, lane);
      }
      if (a.n_heavy > 0) {
        cluster.sync();
        for (int h = w; h < a.n_heavy; h += cw) {
          __syncwarp();
          if (a.prod) process_heavy<T, RKP, GP>(a, h, chunk, lane, stage, (int)(stage_bytes / 16));
          else process_heavy<T, RKS, GS>(a, h, chunk, lane, stage, (int)(stage_bytes / 16));
        }
      }
    }
    stamp(i, 1);
    cluster_arrive();
    stamp(i, 2);
    cluster_wait();
    stamp(i, 3);
  }
}

template <typename T, int RKP, int RKS, typename GP, typename GS>
inline int launch_tail(const TailArgs<T>& t, int cluster, cudaStream_t s) {
  const int chunks = (t.layer[0].V + 32 * NV - 1) / (32 * NV);
  auto kern = tail_kernel<T, RKP, RKS, GP, GS>;
  constexpr size_t smem = TailSmem<T, GP, GS>::bytes;
  static std::atomic<unsigned> configured{0};
  if (needs_config(configured)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(chunks * cluster), 1, 1);
  cfg.blockDim = dim3(TailSmem<T, GP, GS>::warps * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, t) == cudaSuccess ? 1 : 0;
}

// ---- micro tail: the thin upper layers with their values in shared memory ----
//
// Above the bandwidth-bound layers the circuit narrows to a few thousand
// nodes and less; there a layer is latency, not bandwidth: a launch (or a
// cluster barrier) plus dependent L2 round trips per layer. The micro tails
// run all of those layers in one launch of independent CTAs, one per column
// chunk of P 16-byte pieces: a worker of P lanes reduces one node at a time
// over rows held in shared memory, and the CTA meets at one __syncthreads
// per layer. The next layer's CSR (plan data) is staged with cp.async while
// the current layer runs.
//
// Forward (any semiring): two layers' value rows (ping-pong); each result
// goes to shared memory and to the trace. Backward: two layers' adjoint rows
// plus, for a weighted layer (log: sums, softmax weights; real: products,
// zero-safe adjoint over the layer's forward CSR), the forward values of its
// parents and children, fetched with cp.async while the pass-through layer
// above it runs (layers alternate product / sum). Only the lowest layer's
// adjoints leave the CTA.
//
// Reductions follow the reference's order exactly: x0 + numpy's pairwise sum
// of the rest (fan-in <= MICRO_FAN = PW_BLOCK + 1: one pairwise block),
// sequential products / max / min, the streaming logsumexp of LseOp.

constexpr int MICRO_THREADS = 512;
// P: 16-byte pieces per CTA column chunk. Two (32 bytes) when the batch has
// more than one wave of CTAs' worth of pieces; one for small batches, which
// doubles the CTAs (and halves their work) where the tails are latency-bound
template <int P>
constexpr size_t micro_smem_f() { return (size_t)2 * MICRO_WF * P * 16 + (size_t)2 * MICRO_CSRF * sizeof(int); }
template <int P>
constexpr size_t micro_smem_b() { return (size_t)4 * MICRO_WB * P * 16 + (size_t)2 * MICRO_CSRB * sizeof(int); }
inline int micro_p(int V) {
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  static const int forced = [] {
    const char* e = getenv("KLAY_MICRO_P");
    return (e && *e) ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  return V <= sms ? 1 : MICRO_P;
}

template <typename T>
__device__ __forceinline__ Vec<T> lds1(const uint4* p) {
  Vec<T> r;
  const uint4 u = *p;
  memcpy(&r.v[0], &u, 16);
  return r;
}
template <typename T>
__device__ __forceinline__ void sts1(uint4* p, const Vec<T>& r) {
  uint4 u;
  memcpy(&u, &r.v[0], 16);
  *p = u;
}

// x0 + pairwise(x1 .. x_{n-1}) for n <= PW_BLOCK + 1, numpy's order
// (sequential below 8 elements, else 8 interleaved accumulators)
template <typename T, typename F>
__device__ __forceinline__ Vec<T> micro_sum(int n, F&& v) {
  Vec<T> out = v(0);
  const int m = n - 1;
  if (m <= 0) return out;
  if (m < 8) {
    Vec<T> acc = v(1);
    for (int j = 2; j < n; ++j) acc = vadd(acc, v(j));
    return vadd(out, acc);
  }
  Vec<T> r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = v(1 + j);
  const int mainend = m - (m & 7);
  int i = 8;
  for (; i < mainend; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = vadd(r[j], v(1 + i + j));
  }
  Vec<T> res = combine8(r);
  for (; i < m; ++i) res = vadd(res, v(1 + i));
  return vadd(out, res);
}

template <typename T, int RK>
__device__ __forceinline__ Vec<T> micro_reduce(const uint4* rows, int P, const int* idx, int n, T eps) {
  auto v = [&](int e) {
#ifdef KLAY_CHECKS
    if ((unsigned)idx[e] >= (unsigned)MICRO_WF) chk_fail(rows, 7);
#endif
    return lds1<T>(rows + (size_t)idx[e] * P);
  };
  if constexpr (RK == RK_SUM) {
    return micro_sum<T>(n, v);
  } else if constexpr (RK == RK_LSE) {
    Vec<T> out = v(0);
    if (n > 1 || eps != T(0)) {
      LseOp<T> op;
      op.eps = eps;
      op.begin(n);
      op.push(out);
      for (int j = 1; j < n; ++j) op.push(v(j));
      return op.result();
    }
    return lse_unary(out);
  } else {
    Vec<T> out = v(0);
    for (int j = 1; j < n; ++j) seq_combine<T, RK>(out, v(j));
    return out;
  }
}

// stage `n` ints of plan CSR (16-byte aligned) into shared memory; not waited
__device__ __forceinline__ void micro_stage_csr(int* dst, const int* src, int n) {
  for (int i = threadIdx.x; i < (n + 3) / 4; i += blockDim.x) cp_async16_plan(dst + 4 * i, src + 4 * i);
}

template <typename T, int RKP, int RKS, int P>
__global__ void __launch_bounds__(MICRO_THREADS, 1)
    micro_kernel(const __grid_constant__ MicroArgs<T> m) {
  static_assert(NV == 1, "the micro tail assumes one 16-byte piece per lane");
  chk_enter(m.chk);
  constexpr int NW = MICRO_THREADS / P, CSR = MICRO_CSRF;
  constexpr size_t SET = (size_t)MICRO_WF * P;
  extern __shared__ __align__(16) unsigned char smem[];
  uint4* rows = reinterpret_cast<uint4*>(smem);
  int* csr = reinterpret_cast<int*>(smem + 2 * SET * 16);
  const int hl = threadIdx.x % P, worker = threadIdx.x / P;
  const int vb = blockIdx.x * P + hl;
  const bool in_row = vb < m.V;
  const size_t col = (size_t)(in_row ? vb : 0) * PIECE<T>;
  const long long ld = m.ld;
  micro_stage_csr(csr, m.csr + m.csr_at[0], m.csr_n[0]);
  cp_async_commit();
#ifndef KLAY_NO_GDC
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
  for (int r = worker; r < m.w_in; r += NW) cp_async16(rows + r * P + hl, m.in + r * ld + col);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int i = 0; i < m.n; ++i) {
    if (i + 1 < m.n) {
      micro_stage_csr(csr + ((i + 1) & 1) * CSR, m.csr + m.csr_at[i + 1], m.csr_n[i + 1]);
      cp_async_commit();
    }
    const uint4* src = rows + (i & 1) * SET + hl;
    uint4* dst = rows + ((i + 1) & 1) * SET;
    const int* off = csr + (i & 1) * CSR;
    const int* idx = off + m.w[i] + 1;
    T* out = m.out[i];
    const bool prod = m.prod[i] != 0;
    for (int nd = worker; nd < m.w[i]; nd += NW) {
      const int e0 = off[nd], n = off[nd + 1] - e0;
      const Vec<T> r = prod ? micro_reduce<T, RKP>(src, P, idx + e0, n, m.eps)
                            : micro_reduce<T, RKS>(src, P, idx + e0, n, m.eps);
      sts1(dst + nd * P + hl, r);
      if (out && in_row) stv(out + (size_t)nd * ld + col, r, 1);
    }
    cp_async_wait<0>();
    __syncthreads();
  }
}

template <typename T, int RKP, int RKS, int P>
inline int launch_micro_p(const MicroArgs<T>& m, cudaStream_t s) {
  auto kern = micro_kernel<T, RKP, RKS, P>;
  constexpr size_t bytes = micro_smem_f<P>();
  static std::atomic<unsigned> configured{0};
  if (needs_config(configured)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((m.V + P - 1) / P), 1, 1);
  cfg.blockDim = dim3(MICRO_THREADS, 1, 1);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, m) == cudaSuccess ? 1 : 0;
}

template <typename T, int RKP, int RKS>
inline int launch_micro(const MicroArgs<T>& m, cudaStream_t s) {
  return micro_p(m.V) == 1 ? launch_micro_p<T, RKP, RKS, 1>(m, s) : launch_micro_p<T, RKP, RKS, MICRO_P>(m, s);
}

template <typename T, int DOM, int P>
__global__ void __launch_bounds__(MICRO_THREADS, 1)
    micro_bwd_kernel(const __grid_constant__ MicroBwdArgs<T> m) {
  static_assert(NV == 1, "the micro tail assumes one 16-byte piece per lane");
  chk_enter(m.chk);
  constexpr int NW = MICRO_THREADS / P, CSR = MICRO_CSRB;
  constexpr size_t SET = (size_t)MICRO_WB * P;
  extern __shared__ __align__(16) unsigned char smem[];
  uint4* gset = reinterpret_cast<uint4*>(smem);              // [2] adjoint row sets
  uint4* vp = reinterpret_cast<uint4*>(smem) + 2 * SET;      // parent values
  uint4* vx = reinterpret_cast<uint4*>(smem) + 3 * SET;      // child values
  int* csr = reinterpret_cast<int*>(smem + 4 * SET * 16);
  const int hl = threadIdx.x % P, worker = threadIdx.x / P;
  const int vb = blockIdx.x * P + hl;
  const bool in_row = vb < m.V;
  const size_t col = (size_t)(in_row ? vb : 0) * PIECE<T>;
  const long long ld = m.ld;
  micro_stage_csr(csr, m.csr + m.csr_at[0], m.csr_n[0]);
  cp_async_commit();
#ifndef KLAY_NO_GDC
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
  // values of step i's parents / children into vp / vx (not waited)
  auto fetch_values = [&](int i) {
    for (int r = worker; r < m.wp[i]; r += NW) cp_async16(vp + r * P + hl, m.vpar[i] + r * ld + col);
    for (int r = worker; r < m.wc[i]; r += NW) cp_async16(vx + r * P + hl, m.vchild[i] + r * ld + col);
  };
  for (int r = worker; r < m.w_top; r += NW) cp_async16(gset + r * P + hl, m.gin + r * ld + col);
  if (m.n > 0 && m.logsum[0]) fetch_values(0);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int i = 0; i < m.n; ++i) {
    const bool weighted = m.logsum[i] != 0;
    if (i + 1 < m.n) {
      micro_stage_csr(csr + ((i + 1) & 1) * CSR, m.csr + m.csr_at[i + 1], m.csr_n[i + 1]);
      // a pass-through layer leaves vp / vx free for the weighted layer below
      if (!weighted && m.logsum[i + 1]) fetch_values(i + 1);
      cp_async_commit();
    }
    const uint4* src = gset + (i & 1) * SET + hl;
    uint4* dst = gset + ((i + 1) & 1) * SET;
    const int* off = csr + (i & 1) * CSR;
    const int* idx = off + m.wc[i] + 1;
    // real products: the layer's forward CSR follows (zero-safe adjoint)
    const int* foff = idx + off[m.wc[i]];
    const int* fsrc = foff + m.wp[i] + 1;
    T* out = m.gout[i];
    for (int c = worker; c < m.wc[i]; c += NW) {
      const int e0 = off[c], n = off[c + 1] - e0;
      Vec<T> x{};
      if (weighted) x = lds1<T>(vx + c * P + hl);
      auto val = [&](int e) {
        const int row = idx[e0 + e];
        const int p = row & 0x7fffffff;
        const Vec<T> g = lds1<T>(src + (size_t)p * P);
        if (!weighted) return g;
        if constexpr (DOM == SR_LOG) {
          if (row < 0 && m.unary_ok) return BwdGather<T, BW_LOGSUM>::unary(g, x);
          return BwdGather<T, BW_LOGSUM>::logsum_edge(g, lds1<T>(vp + (size_t)p * P + hl), x);
        } else {
          const Vec<T> pv = lds1<T>(vp + (size_t)p * P + hl);
          // (g * prod) / x; a segment holding a zero (or a NaN product)
          // counts its zeros (BwdGather<BW_REALPROD>::combine / zero_path)
          constexpr int N = Vec<T>::N;
          Vec<T> r;
          bool any_zero = false;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            r.v[k] = (g.v[k] * pv.v[k]) / x.v[k];
            any_zero |= (x.v[k] == T(0)) | (pv.v[k] == T(0)) | (pv.v[k] != pv.v[k]);
          }
          if (any_zero) {
            T pnz[N];
            int zc[N];
#pragma unroll
            for (int k = 0; k < N; ++k) { pnz[k] = T(1); zc[k] = 0; }
            for (int q = foff[p]; q < foff[p + 1]; ++q) {
              const Vec<T> y = lds1<T>(vx + (size_t)fsrc[q] * P + hl);
#pragma unroll
              for (int k = 0; k < N; ++k) {
                if (y.v[k] == T(0)) ++zc[k];
                else pnz[k] *= y.v[k];
              }
            }
#pragma unroll
            for (int k = 0; k < N; ++k) {
              if (x.v[k] == T(0)) r.v[k] = (zc[k] == 1) ? g.v[k] * pnz[k] : T(0);
              else if (zc[k] > 0) r.v[k] = T(0);
            }
          }
          return r;
        }
      };
      const Vec<T> r = micro_sum<T>(n, val);
      sts1(dst + c * P + hl, r);
      if (out && in_row) stv(out + (size_t)c * ld + col, r, 1);
    }
    cp_async_wait<0>();
    __syncthreads();
  }
}

template <typename T, int DOM, int P>
inline int launch_micro_bwd_p(const MicroBwdArgs<T>& m, cudaStream_t s) {
  auto kern = micro_bwd_kernel<T, DOM, P>;
  constexpr size_t bytes = micro_smem_b<P>();
  static std::atomic<unsigned> configured{0};
  if (needs_config(configured)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((m.V + P - 1) / P), 1, 1);
  cfg.blockDim = dim3(MICRO_THREADS, 1, 1);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, m) == cudaSuccess ? 1 : 0;
}

template <typename T, int DOM>
inline int launch_micro_bwd(const MicroBwdArgs<T>& m, cudaStream_t s) {
  return micro_p(m.V) == 1 ? launch_micro_bwd_p<T, DOM, 1>(m, s) : launch_micro_bwd_p<T, DOM, MICRO_P>(m, s);
}

}  // namespace klay
