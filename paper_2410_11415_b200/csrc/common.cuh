// Shared device helpers of libklay: 16-byte value vectors, numpy-faithful
// elementwise ops and the streaming segment reducers.
//
// A "segment" is one node's incoming edge list in CSR order (forward:
// parent <- children; backward: child <- parents over the transposed CSR).
// Reducers consume the segment's edge values strictly in edge order, so the
// result reproduces the reference's reduction order:
//   SumOp   np.add.reduceat        x0 + pairwise(x[1:])   (bit-exact)
//   ProdOp  np.multiply.reduceat   sequential              (bit-exact)
//   MaxOp / MinOp  np.maximum / np.minimum.reduceat, NaN-propagating
//   LseOp   _segment_logsumexp (engine.py:274-282), merged online; equal to
//           the two-pass form bit-for-bit for fan-in <= 2, ulp-close beyond
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

namespace klay {

enum { SR_REAL = 0, SR_LOG = 1, SR_BOOL = 2, SR_MAXPROD = 3 };
enum { BW_PASS = 0, BW_LOGSUM = 1, BW_REALPROD = 2, BW_PASSA = 3, BW_LOGSUM8 = 4 };
// reduction kinds
enum { RK_SUM = 0, RK_PROD = 1, RK_MAX = 2, RK_MIN = 3, RK_LSE = 4, RK_AND = 5, RK_OR = 6 };

// numpy's pairwise summation works on blocks of at most this many elements
#ifndef KLAY_PW_BLOCK
#define KLAY_PW_BLOCK 128
#endif
constexpr int PW_BLOCK = KLAY_PW_BLOCK;  // numpy pairwise block (128; other values: experiments only)

#ifndef KLAY_NV
#define KLAY_NV 1
#endif
// Each lane owns NV 16-byte pieces of a row: piece q of lane l in column
// chunk c is the row's 16-byte vector (c * NV + q) * 32 + l, so every load /
// store instruction of a warp moves one contiguous 512-byte span and a warp
// covers NV * 512 bytes of the row (per-edge bookkeeping amortized NV-fold).
constexpr int NV = KLAY_NV;

// ---- KLAY_CHECKS builds: run-time bounds checks of every global row access --
// (compute-sanitizer is unavailable on the GPU pool; this is the stand-in).
// A kernel copies the call's valid byte ranges (the values / trace buffer and
// the workspace) into shared memory at entry (chk_enter); every ldv / stv /
// cp.async below verifies its 16-byte access against them, records the first
// violation in the call's record (klay.cu reads it after the call) and
// redirects the access to the start of the values buffer instead of faulting.
struct ChkRanges {
  const char* lo[2];
  const char* hi[2];
  int* rec;  // [0] violations, [1] site, [2] kernel tag, [3] low bits of the address
  int tag;
};
#ifdef KLAY_CHECKS
static __shared__ ChkRanges klay_chk;
__device__ __forceinline__ void chk_enter(const ChkRanges& c) {
  if ((threadIdx.x & 31) == 0 && threadIdx.x < 32) klay_chk = c;
  __syncthreads();
}
static __device__ __noinline__ const void* chk_fail(const void* p, int site) {
  if (klay_chk.rec && atomicAdd(klay_chk.rec, 1) == 0) {
    klay_chk.rec[1] = site;
    klay_chk.rec[2] = klay_chk.tag;
    klay_chk.rec[3] = (int)(reinterpret_cast<uintptr_t>(p) & 0x7fffffff);
  }
  return klay_chk.lo[0];
}
__device__ __forceinline__ const void* chk(const void* p, int site, int bytes) {
  const char* c = static_cast<const char*>(p);
  if (!klay_chk.rec) return p;
#pragma unroll
  for (int i = 0; i < 2; ++i)
    if (c >= klay_chk.lo[i] && c + bytes <= klay_chk.hi[i]) return p;
  return chk_fail(p, site);
}
template <typename T>
__device__ __forceinline__ T* chkp(T* p, int site) {
  return (T*)chk(p, site, (int)sizeof(T));
}
#define KLAY_CHK(p, site) chkp((p), (site))
#define KLAY_CHK_N(p, site, n) ((decltype(p))chk((p), (site), (n)))
#else
__device__ __forceinline__ void chk_enter(const ChkRanges&) {}
#define KLAY_CHK(p, site) (p)
#define KLAY_CHK_N(p, site, n) (p)
#endif

// Row r of a [rows, ld] buffer whose row stride is ldb = ld * sizeof(T)
// bytes (< 2 GB): a 32 x 32 -> 64-bit IMAD.WIDE instead of a 64-bit multiply
// and shift (half the address instructions of a staged edge). row_at takes a
// signed row (alias offsets below the base), row_atu a non-negative one.
template <typename T>
__device__ __forceinline__ T* row_at(T* p, int r, int ldb) {
  using C = typename std::conditional<std::is_const<T>::value, const char, char>::type;
  return reinterpret_cast<T*>(reinterpret_cast<C*>(p) + (long long)r * ldb);
}
template <typename T>
__device__ __forceinline__ T* row_atu(T* p, unsigned r, unsigned ldb) {
  using C = typename std::conditional<std::is_const<T>::value, const char, char>::type;
  return reinterpret_cast<T*>(reinterpret_cast<C*>(p) + (unsigned long long)r * ldb);
}

template <typename T>
struct alignas(16) Vec {
  static constexpr int N = NV * 16 / sizeof(T);
  T v[N];
};
template <typename T>
constexpr int PIECE = 16 / (int)sizeof(T);  // elements per 16-byte piece
template <typename T>
constexpr int PSTRIDE = 32 * PIECE<T>;      // elements between a lane's pieces

// `p` points at the lane's piece 0; pieces >= nl (past the row) repeat the
// last valid piece, so loads never leave the row.
__device__ __forceinline__ Vec<float> ldv(const float* p, int nl) {
  Vec<float> r;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const float4 u = __ldcg(KLAY_CHK(reinterpret_cast<const float4*>(p + (q < nl ? q : nl - 1) * PSTRIDE<float>), 1));
    r.v[4 * q] = u.x; r.v[4 * q + 1] = u.y; r.v[4 * q + 2] = u.z; r.v[4 * q + 3] = u.w;
  }
  return r;
}
__device__ __forceinline__ Vec<double> ldv(const double* p, int nl) {
  Vec<double> r;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double2 u = __ldcg(KLAY_CHK(reinterpret_cast<const double2*>(p + (q < nl ? q : nl - 1) * PSTRIDE<double>), 1));
    r.v[2 * q] = u.x; r.v[2 * q + 1] = u.y;
  }
  return r;
}
// bit-packed Boolean rows: 32 batch rows per 32-bit word
__device__ __forceinline__ Vec<unsigned> ldv(const unsigned* p, int nl) {
  Vec<unsigned> r;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const uint4 u = __ldcg(KLAY_CHK(reinterpret_cast<const uint4*>(p + (q < nl ? q : nl - 1) * PSTRIDE<unsigned>), 1));
    r.v[4 * q] = u.x; r.v[4 * q + 1] = u.y; r.v[4 * q + 2] = u.z; r.v[4 * q + 3] = u.w;
  }
  return r;
}
__device__ __forceinline__ void stv(unsigned* p, const Vec<unsigned>& r, int na) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
    if (q < na)
      *KLAY_CHK(reinterpret_cast<uint4*>(p + q * PSTRIDE<unsigned>), 2) =
          make_uint4(r.v[4 * q], r.v[4 * q + 1], r.v[4 * q + 2], r.v[4 * q + 3]);
}

// store the first `na` pieces (the ones inside the row)
__device__ __forceinline__ void stv(float* p, const Vec<float>& r, int na) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
    if (q < na)
      *KLAY_CHK(reinterpret_cast<float4*>(p + q * PSTRIDE<float>), 2) =
          make_float4(r.v[4 * q], r.v[4 * q + 1], r.v[4 * q + 2], r.v[4 * q + 3]);
}
__device__ __forceinline__ void stv(double* p, const Vec<double>& r, int na) {
#pragma unroll
  for (int q = 0; q < NV; ++q)
    if (q < na) *KLAY_CHK(reinterpret_cast<double2*>(p + q * PSTRIDE<double>), 2) = make_double2(r.v[2 * q], r.v[2 * q + 1]);
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

// fp32 exp / log on the SFU (ex2.approx / lg2.approx: ~2^-22 relative,
// special values as expf / logf; the non-ftz forms keep subnormal results,
// at 3 extra instructions per call). The log
// semiring's fp32 tolerance (rel 1e-5 vs the fp64 reference) holds with
// margin; KLAY_PRECISE_F32 selects the libm versions. fp64 stays exact.
#ifdef KLAY_PRECISE_F32
__device__ __forceinline__ float kexp(float x) { return expf(x); }
__device__ __forceinline__ float klog(float x) { return logf(x); }
#else
__device__ __forceinline__ float kexp(float x) { return __expf(x); }
__device__ __forceinline__ float klog(float x) { return __logf(x); }
#endif
__device__ __forceinline__ double kexp(double x) { return exp(x); }
// exp for terms added to a running sum that is already >= 1 (the online
// logsumexp's t): a result below 2^-126 cannot change that sum, so the
// flush-to-zero ex2 (no denormal range fix-up: 3 fewer instructions) gives
// bit-identical sums
__device__ __forceinline__ float kexp_sum(float x) {
#ifdef KLAY_PRECISE_F32
  return expf(x);
#else
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * 1.4426950408889634f));
  return r;
#endif
}
__device__ __forceinline__ double kexp_sum(double x) { return exp(x); }
__device__ __forceinline__ double klog(double x) { return log(x); }

// np.maximum / np.minimum: NaN-propagating.
template <typename T>
__device__ __forceinline__ T npmax(T a, T b) { return (a > b || a != a) ? a : b; }
template <typename T>
__device__ __forceinline__ T npmin(T a, T b) { return (a < b || a != a) ? a : b; }

// ---------------------------------------------------------------------------
// streaming reducers: begin(n) for a whole segment of n >= 1 edges,
// begin_leaf(len) for one pairwise leaf of the segment's tail (no x0),
// push(x) per edge in order, result() / partial()
// ---------------------------------------------------------------------------
template <typename T>
struct SumOp {
  // The 8 pairwise accumulators live in shared memory (slot q of this thread
  // at r[q * rstride]); they are only touched by segments with more than 8
  // tail elements, so keeping them out of registers keeps occupancy up.
  Vec<T> x0, acc;
  Vec<T>* r;
  int rstride;
  int k, m, mainend;
  __device__ __forceinline__ void start(int k0, int len) {
    k = k0;
    m = len;
    mainend = len - (len & 7);
    acc = vfill<T>(T(-0.0));
  }
  __device__ __forceinline__ void begin(int n) { start(0, n - 1); }
  __device__ __forceinline__ void begin_leaf(int len) { start(1, len); }
  __device__ __forceinline__ Vec<T> combine8() const {
    Vec<T> q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = r[i * rstride];
    Vec<T> res;
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c)
      res.v[c] = ((q[0].v[c] + q[1].v[c]) + (q[2].v[c] + q[3].v[c])) +
                 ((q[4].v[c] + q[5].v[c]) + (q[6].v[c] + q[7].v[c]));
    return res;
  }
  __device__ __forceinline__ void push(const Vec<T>& x) {
    if (k == 0) {
      x0 = x;
    } else {
      const int j = k - 1;
      if (m < 8) {
        acc = vadd(acc, x);
      } else if (j < mainend) {
        Vec<T>& slot = r[(j & 7) * rstride];
        slot = (j < 8) ? x : vadd(slot, x);
      } else {
        if (j == mainend) acc = combine8();
        acc = vadd(acc, x);
      }
    }
    ++k;
  }
  // pairwise sum of the elements after x0 (or of the leaf)
  __device__ __forceinline__ Vec<T> partial() const {
    if (m < 8 || mainend < m) return acc;
    return combine8();
  }
  __device__ __forceinline__ Vec<T> result() const { return m == 0 ? x0 : vadd(x0, partial()); }
};

template <typename T, int RK>
struct SeqOp {  // RK_PROD / RK_MAX / RK_MIN: strictly sequential
  Vec<T> acc;
  int k;
  __device__ __forceinline__ void begin(int) { k = 0; }
  __device__ __forceinline__ void begin_leaf(int) { k = 0; }
  __device__ __forceinline__ void push(const Vec<T>& x) {
    if (k == 0) {
      acc = x;
    } else {
#pragma unroll
      for (int c = 0; c < Vec<T>::N; ++c) {
        if constexpr (RK == RK_PROD) acc.v[c] = acc.v[c] * x.v[c];
        else if constexpr (RK == RK_MAX) acc.v[c] = npmax(acc.v[c], x.v[c]);
        else if constexpr (RK == RK_AND) acc.v[c] = acc.v[c] & x.v[c];
        else if constexpr (RK == RK_OR) acc.v[c] = acc.v[c] | x.v[c];
        else acc.v[c] = npmin(acc.v[c], x.v[c]);
      }
    }
    ++k;
  }
  __device__ __forceinline__ Vec<T> partial() const { return acc; }
  __device__ __forceinline__ Vec<T> result() const { return acc; }
};

template <typename T>
__device__ __forceinline__ void lse_merge(T& m, T& t, T m2, T t2) {
  if (m2 > m) {
    t = t * kexp(m - m2) + t2;
    m = m2;
  } else if (m2 == -INFINITY) {
    // contributes nothing (an all -inf part is masked to 0, engine.py:279),
    // except a NaN it saw (carried as a NaN sum)
    if (isnan(t2)) t = t2;
  } else if (m2 == INFINITY) {
    // m == +inf too: every shifted term is masked to 0; only a NaN input
    // (carried as a NaN sum) must survive
    if (isnan(t2)) t = t2;
  } else {
    t = t + t2 * kexp(m2 - m);
  }
}

// logsumexp of one element with epsilon 0: the element itself, except that a
// +inf element becomes NaN (log(0) + inf, engine.py:274-282)
template <typename T>
__device__ __forceinline__ Vec<T> lse_unary(Vec<T> x) {
  if constexpr (std::is_floating_point<T>::value) {
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c) x.v[c] = (x.v[c] == T(INFINITY)) ? T(NAN) : x.v[c];
  }
  return x;
}

template <typename T>
struct LseOp {
  Vec<T> m, t;
  T eps;
  int k;
  __device__ __forceinline__ void begin(int) {
    m = vfill<T>(T(-INFINITY));
    t = vfill<T>(T(0));
    k = 0;
  }
  __device__ __forceinline__ void begin_leaf(int n) { begin(n); }
  __device__ __forceinline__ void push(const Vec<T>& x) {
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c) {
      const T xv = x.v[c];
      if (k == 0) {
        // first element: exp(x - x) = 1, or 0 for an all -inf prefix (NaN -> 0)
        m.v[c] = xv;
        t.v[c] = (xv == T(-INFINITY)) ? T(0) : T(1);
      } else {
        // branch-free (lanes hold different columns): one exp(-|x - m|)
        //   x > m:  t = t * exp(m - x) + 1, m = x   (rescale to the new peak)
        //   x <= m: t = t + exp(x - m)
        // d is NaN for inf - inf (equal infinite peak and element: the
        // reference masks that term to 0) or for a NaN operand: fmax maps
        // every NaN exponential to 0, and a NaN element is carried as a NaN
        // sum instead (result() reports NaN; a NaN peak can only come from
        // the first element and gives NaN through m)
        // (fp32: issue-bound at high fan-in, config C'; fp64 measured faster
        // with the direct NaN fix-up)
        const T mv = m.v[c];
        const T d = xv - mv;
        const bool up = d > T(0);
        if constexpr (std::is_same<T, float>::value) {
          const T e = fmax(kexp_sum(-fabs(d)), T(0));
          const T tn = up ? t.v[c] * e + T(1) : t.v[c] + e;
          t.v[c] = (xv != xv) ? xv : tn;
        } else {
          T e = kexp(-fabs(d));
          if (d != d) e = (xv != xv || mv != mv) ? d : T(0);
          t.v[c] = up ? t.v[c] * e + T(1) : t.v[c] + e;
        }
        m.v[c] = up ? xv : mv;
      }
    }
    ++k;
  }
  __device__ __forceinline__ Vec<T> result() const {
    Vec<T> r;
#pragma unroll
    for (int c = 0; c < Vec<T>::N; ++c) {
      // log(1 + 0) + m == m exactly: unary segments (79% of sum nodes) skip the log
      T res = (t.v[c] == T(1) && eps == T(0)) ? m.v[c] : klog(t.v[c] + eps) + m.v[c];
      // a +inf peak shifts every element to exp(NaN or -inf) -> 0 in the
      // reference (engine.py:274-282): log(0 + eps) + inf = NaN, or +inf for eps > 0
      if (m.v[c] == T(INFINITY) && !isnan(t.v[c])) res = (eps > T(0)) ? T(INFINITY) : T(NAN);
      // an all -inf segment stays -inf; a NaN element anywhere gives NaN (the
      // reference's peak, np.maximum.reduceat, propagates it): a NaN after a
      // -inf peak shows up as a NaN sum
      r.v[c] = (m.v[c] == T(-INFINITY) && !isnan(t.v[c])) ? T(-INFINITY) : res;
    }
    return r;
  }
};

// ---- cp.async (LDGSTS) helpers: 16-byte global -> shared copies ------------
// plan data (indices, offsets: not in the checked value ranges)
__device__ __forceinline__ void cp_async16_plan(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// value rows (checked in KLAY_CHECKS builds)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  cp_async16_plan(smem, KLAY_CHK_N(gmem, 3, 16));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Staged vectors live in shared memory as NV x 32 lanes of 16-byte pieces
// (conflict-free): piece q of lane l at slot[q * 32 + l].
template <typename T>
__device__ __forceinline__ void cp_async_vec(uint4* slot, int lane, const T* p, int nl) {
#pragma unroll
  for (int q = 0; q < NV; ++q) cp_async16(slot + q * 32 + lane, p + (q < nl ? q : nl - 1) * PSTRIDE<T>);
}
template <typename T>
__device__ __forceinline__ Vec<T> lds_vec(const uint4* slot, int lane) {
  Vec<T> r;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const uint4 u = slot[q * 32 + lane];
    memcpy(&r.v[q * PIECE<T>], &u, 16);
  }
  return r;
}

// pairwise-tree combination of leaf partials staged in shared memory
// (leaf l at pieces sm[l * 32 * NV ...], lane-interleaved like the stages)
template <typename T>
__device__ Vec<T> tree_sum_smem(const uint4* sm, int lane, int& leaf, int len) {
  if (len <= PW_BLOCK) {
    Vec<T> v = lds_vec<T>(sm + (size_t)leaf * 32 * NV, lane);
    ++leaf;
    return v;
  }
  int n2 = len / 2;
  n2 -= n2 % 8;
  Vec<T> a = tree_sum_smem<T>(sm, lane, leaf, n2);
  Vec<T> b = tree_sum_smem<T>(sm, lane, leaf, len - n2);
  return vadd(a, b);
}

// pairwise-tree combination of leaf partials stored one row apart
// (same recursion as numpy's pairwise_sum above PW_BLOCK elements)
template <typename T>
__device__ Vec<T> tree_sum(const T* leaves, long long stride, int& leaf, int len, int nl) {
  if (len <= PW_BLOCK) {
    Vec<T> v = ldv(leaves + (size_t)leaf * stride, nl);
    ++leaf;
    return v;
  }
  int n2 = len / 2;
  n2 -= n2 % 8;
  Vec<T> a = tree_sum(leaves, stride, leaf, n2, nl);
  Vec<T> b = tree_sum(leaves, stride, leaf, len - n2, nl);
  return vadd(a, b);
}

}  // namespace klay
