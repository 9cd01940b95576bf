// Streaming layer kernel of libklay: Blackwell bulk-copy (TMA) row streams.
//
// One CTA owns a contiguous range of a layer's nodes (host-balanced by
// slots, klay.cu build_stream_ctas) and one column chunk of up to 4 KB of
// every row (all of B = 1024 fp32). Its producer warp walks the nodes in
// order and streams every operand row the reduction needs -- per node its
// own value (log-sum backward), then per edge the operand row (plus the
// parent's value row for the log-sum backward) -- into a shared-memory ring
// of row slots, one cp.async.bulk per row (SASS UBLKCP), completing on
// per-group mbarriers (expect_tx). The consumer warps (one 16-byte column
// piece per thread) take the slots in the same order, reduce each node in
// the reference's exact order (x0 + numpy's pairwise sum, sequential
// products, the streaming logsumexp of LseOp; gather_policy value() /
// combine() for the adjoints) and store its row; they release a group of
// slots to the producer through an `empty` mbarrier.
//
// Compared with items_kernel (one warp per item and 512-byte chunk, per-lane
// LDGSTS), the index bookkeeping is paid once per row instead of once per
// 512-byte chunk, the bytes in flight are set by the ring, not by resident
// warps and registers, and one instruction moves a whole row chunk.
// Segments longer than one numpy pairwise block (> 129 edges) stay on
// items_kernel (heavy leaves); so do the bit-packed Boolean rows.
#pragma once

#include "layer_kernels.cuh"

namespace klay {

constexpr int SG = 4;             // ring slots per mbarrier group
constexpr int STREAM_MAX_PV = 256;  // 16-byte pieces per CTA column chunk (4 KB)

// consumer threads for a chunk of spv pieces, VP per thread: a multiple of
// 32, so the pieces a warp holds for one q are one aligned 512-byte column
// chunk (the route masks' unit: lane = piece within the chunk, as in the
// items kernel). Pieces past the row are clamped and never stored.
__host__ __device__ constexpr int stream_threads(int spv, int vp) {
  return ((spv + vp - 1) / vp + 31) / 32 * 32;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nKLAY_MBW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KLAY_MBW_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// shared memory of one CTA: full / empty mbarriers per group (<= 16 groups),
// the CTA's index block (plan data, STREAM_SIDX ints: segment offsets, edge
// operand rows, output map, own-value map), the slot list (log-sum
// backward: STREAM_SLOTS ints), the ring (R slots of pvmax pieces)
constexpr int STREAM_SIDX = 2048;
constexpr int STREAM_SLOTS = 4096;
struct StreamSmem {
  static constexpr size_t idx_at = 256 + 16;  // (barriers, then the slot count)
  static constexpr size_t slots_at = idx_at + (size_t)STREAM_SIDX * 4;
  static __host__ __device__ size_t ring_at(bool slot_list) {
    return slots_at + (slot_list ? (size_t)STREAM_SLOTS * 4 : 0);
  }
  static __host__ __device__ size_t bytes(int R, int pvmax, bool slot_list) {
    return ring_at(slot_list) + (size_t)R * pvmax * 16;
  }
};

template <typename T, typename G>
struct StreamTraits {
  static constexpr bool BWD = !std::is_same<G, FwdGather<T, false>>::value && !std::is_same<G, FwdGather<T, true>>::value;
  // the log-sum backward streams, per node, the child's own value and, per
  // edge, the parent's adjoint and (unless the parent is a unary sum) value:
  // its slot sequence is listed in shared memory by the prologue
  static constexpr bool XSLOT = BWD && G::NOP == 2 && !std::is_same<G, BwdGather<T, BW_REALPROD>>::value;
  // slots per edge otherwise (real-product backward: adjoint + value)
  static constexpr int SPE = (BWD && G::NOP == 2) ? 2 : 1;
};

// A CTA: nodes [d.x, d.y) of the layer's node set with edges [d.z, d.w)
// (klay.cu build_stream_ctas: its index block fits STREAM_SIDX ints, its
// slots STREAM_SLOTS). VP: 16-byte pieces per consumer thread (thread t owns
// pieces t, t + NT, ...; NT = consumer threads).
template <typename T, int RK, typename G, int VP>
__global__ void __launch_bounds__(STREAM_MAX_PV / VP + 32, 3) stream_kernel(const __grid_constant__ LayerArgs<T> a) {
  using TR = StreamTraits<T, G>;
  constexpr bool BWD = TR::BWD, XSLOT = TR::XSLOT;
  extern __shared__ __align__(128) unsigned char stream_smem[];
  unsigned char* smem = stream_smem;
  chk_enter(a.chk);
  const int R = a.sring, NGR = R / SG;
  const int pvmax = a.spv;
  const int nt = stream_threads(pvmax, VP);  // consumer threads
  const int ncw = (nt + 31) >> 5;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* empty = full + NGR;
  int* sb = reinterpret_cast<int*>(smem + StreamSmem::idx_at);
  int* sslot = reinterpret_cast<int*>(smem + StreamSmem::slots_at);
  int* s_count = reinterpret_cast<int*>(smem + 2 * 16 * 8);  // slots of the CTA (log-sum backward)
  uint4* ring = reinterpret_cast<uint4*>(smem + StreamSmem::ring_at(XSLOT));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int4 d = __ldg(reinterpret_cast<const int4*>(a.scta) + blockIdx.x);
  const int n0 = d.x, nn = d.y - d.x, e0 = d.z, ne = d.w - d.z;
  // index block: [soff nn+1][sidx ne][somap nn][sxmap nn]
  int* soff = sb;
  int* sidx = soff + nn + 1;
  int* somap = sidx + ne;
  int* sxmap = somap + (a.omap ? nn : 0);
#ifdef KLAY_STREAM_TRACE
  // per CTA: [0] start ns, [1] after the grid-dependency wait, [2] producer
  // cycles waiting for free slots, [3] slots, [4] producer done ns, [5]
  // consumer warp 0 cycles waiting for data, [6] consumers done ns, [7] SM
  unsigned long long* tr = a.trace ? a.trace + 8 * (blockIdx.x + (size_t)gridDim.x * blockIdx.y) : nullptr;
  auto gt = [] {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    return ns;
  };
  unsigned long long w_cyc = 0;
  if (tr && tid == 0) {
    tr[0] = gt();
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    tr[7] = sm;
  }
#define KLAY_TWAIT(stmt)                            \
  do {                                              \
    const long long c0_ = clock64();                \
    stmt;                                           \
    w_cyc += (unsigned long long)(clock64() - c0_); \
  } while (0)
#else
#define KLAY_TWAIT(stmt) stmt
#endif
  // this CTA's column chunk: pieces [pb, pb + pv) of every row
  const int pb = blockIdx.y * pvmax;
  const int pv = min(pvmax, a.V - pb);
  const unsigned rowb = (unsigned)pv * 16u;
  const size_t col0 = (size_t)pb * PIECE<T>;
  if (tid < NGR) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], ncw);
  }
  // the index block is plan data: staged before waiting on the previous kernel
  for (int i = tid; i <= nn; i += blockDim.x) soff[i] = __ldg(a.off + n0 + i) - e0;
  for (int i = tid; i < ne; i += blockDim.x) sidx[i] = __ldg(a.idx + e0 + i);
  if (a.omap)
    for (int i = tid; i < nn; i += blockDim.x) somap[i] = __ldg(a.omap + n0 + i);
  if (a.xmap)
    for (int i = tid; i < nn; i += blockDim.x) sxmap[i] = __ldg(a.xmap + n0 + i);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  auto out_id = [&](int k) { return a.omap ? somap[k] : n0 + k; };
  auto x_id = [&](int k) { return a.xmap ? sxmap[k] : n0 + k; };
  int ns = ne * TR::SPE;  // slots of the CTA
  if constexpr (XSLOT) {
    // slot list: per node its own value (kind 2), per edge the parent's
    // adjoint (kind 0) and value (kind 1) unless the parent is a unary sum;
    // entry = kind << 30 | row (rows < 2^30, klay.cu)
    if (tid == 0) {
      int q = 0;
      for (int k = 0; k < nn; ++k) {
        sslot[q++] = (2 << 30) | x_id(k);
        for (int e = soff[k]; e < soff[k + 1]; ++e) {
          const int row = sidx[e];
          const int r = row & 0x7fffffff;
          sslot[q++] = r;
          if (!(a.unary_ok && row < 0)) sslot[q++] = (1 << 30) | r;
        }
      }
      *s_count = q;
    }
    __syncthreads();
    ns = *s_count;
  }
#ifndef KLAY_NO_GDC
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
#ifdef KLAY_STREAM_TRACE
  if (tr && tid == 0) tr[1] = gt();
#endif

  if (warp == ncw) {
    // ================= producer warp: one group of slots per round =========
    const long long ld = a.ld;
    const int ngroups = (ns + SG - 1) / SG;
    for (int gi = 0; gi < ngroups; ++gi) {
      const int grp = gi % NGR, par = (gi / NGR) & 1;
      const int s0 = gi * SG, cnt = min(SG, ns - s0);
      const T* src = nullptr;
      if (lane < cnt) {
        const int s = s0 + lane;
        if constexpr (XSLOT) {
          const int v = sslot[s];
          const int kind = (v >> 30) & 3;
          const T* base = kind == 0 ? a.gcur : (kind == 1 ? a.ncur : a.nprev);
          src = base + (long long)(v & 0x3fffffff) * ld + col0;
        } else if constexpr (BWD) {
          const long long r = (long long)(sidx[s / TR::SPE] & 0x7fffffff);
          src = ((TR::SPE == 2 && (s & 1)) ? a.ncur : a.gcur) + r * ld + col0;
        } else {
          src = a.prev + (long long)sidx[s] * ld + col0;
        }
      }
      if (lane == 0) {
        KLAY_TWAIT(mbar_wait(&empty[grp], par ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[grp])),
                     "r"((unsigned)cnt * rowb)
                     : "memory");
      }
      __syncwarp();
#ifdef KLAY_CHECKS
      if (lane < cnt) {  // the whole row chunk inside a valid range
        src = KLAY_CHK_N(src, 8, 16);
        if (KLAY_CHK_N(reinterpret_cast<const char*>(src) + rowb - 16, 8, 16) != reinterpret_cast<const char*>(src) + rowb - 16)
          src = reinterpret_cast<const T*>(klay_chk.lo[0]);
      }
#endif
      if (lane < cnt) bulk_row(ring + (size_t)(grp * SG + lane) * pvmax, src, rowb, &full[grp]);
    }
#ifdef KLAY_STREAM_TRACE
    if (tr && lane == 0) {
      tr[2] = w_cyc;
      tr[3] = (unsigned long long)ns;
      tr[4] = gt();
    }
#endif
    return;
  }

  // ======================= consumer warps =======================
  // thread = VP 16-byte column pieces (t, t + nt, ...) of the chunk; pieces
  // past the row load a valid piece and never store
  int pl[VP];
  bool in_row[VP];
#pragma unroll
  for (int q = 0; q < VP; ++q) {
    const int pc = tid + q * nt;
    in_row[q] = pc < pv;
    pl[q] = min(pc, pv - 1);
  }
  // Slots are consumed in order: wait for a group at its first slot,
  // release it (empty barrier, one arrive per consumer warp) right after its
  // last, so a node longer than the ring never deadlocks and the producer
  // refills as early as possible. Running slot pointer, no divisions.
  int gs = 0, grp = 0, par = 0;
  const uint4* cur = ring;
  auto take = [&](Vec<T> (&v)[VP]) {
    if (gs == 0) KLAY_TWAIT(mbar_wait(&full[grp], par));
#pragma unroll
    for (int q = 0; q < VP; ++q) v[q] = lds1<T>(cur + pl[q]);
    cur += pvmax;
    if (++gs == SG) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[grp]);
      gs = 0;
      if (++grp == NGR) {
        grp = 0;
        par ^= 1;
        cur = ring;
      }
    }
  };
  G gq[VP];
#pragma unroll
  for (int q = 0; q < VP; ++q) gq[q] = G(a, col0 + (size_t)pl[q] * PIECE<T>, 1);
  int eb = 0;  // (soff[0] == 0: offsets are relative to the CTA's first edge)
  for (int k = 0; k < nn; ++k) {
    const int ea = eb;
    eb = soff[k + 1];
    const int n = eb - ea;
    const int out = out_id(k);
    Vec<T> x[VP];
    if constexpr (XSLOT) {
      take(x);
    } else if constexpr (BWD && G::NX) {
#pragma unroll
      for (int q = 0; q < VP; ++q) x[q] = gq[q].load_x(out, x_id(k));  // PASSA route mask / real-product own value
    }
    int e = ea;
    // the next edge's contribution (its slots are next in the ring)
    auto next = [&](Vec<T> (&v)[VP]) {
      const int row = G::ROWV ? sidx[e] : 0;  // (alias sign, unary-parent flag, product zero path)
      ++e;
      take(v);
      if constexpr (BWD) {
        if constexpr (G::NOP == 2) {
          if constexpr (G::LOGSUMLIKE) {
            if (a.unary_ok && row < 0) {
#pragma unroll
              for (int q = 0; q < VP; ++q) v[q] = G::unary(v[q], x[q]);
              return;
            }
          }
          Vec<T> P[VP];
          take(P);
#pragma unroll
          for (int q = 0; q < VP; ++q) v[q] = gq[q].combine(v[q], P[q], row, x[q]);
        }
      } else {
        if constexpr (G::ALIAS_IN) {
          if (row < 0) {
#pragma unroll
            for (int q = 0; q < VP; ++q) v[q] = lse_unary(v[q]);
          }
        }
      }
    };
    Vec<T> res[VP];
    if constexpr (RK == RK_SUM) {
      // x0 + numpy's pairwise sum of the rest (one block: n <= 129)
      next(res);
      const int mm = n - 1;
      if (mm > 0) {
        Vec<T> t[VP], v[VP];
        if (mm < 8) {
          next(t);
          for (int j = 2; j < n; ++j) {
            next(v);
#pragma unroll
            for (int q = 0; q < VP; ++q) t[q] = vadd(t[q], v[q]);
          }
        } else {
          Vec<T> r[8][VP];
#pragma unroll
          for (int j = 0; j < 8; ++j) next(r[j]);
          const int mainend = mm - (mm & 7);
          int i = 8;
          for (; i < mainend; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              next(v);
#pragma unroll
              for (int q = 0; q < VP; ++q) r[j][q] = vadd(r[j][q], v[q]);
            }
          }
#pragma unroll
          for (int q = 0; q < VP; ++q) {
            Vec<T> rq[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) rq[j] = r[j][q];
            t[q] = combine8(rq);
          }
          for (; i < mm; ++i) {
            next(v);
#pragma unroll
            for (int q = 0; q < VP; ++q) t[q] = vadd(t[q], v[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < VP; ++q) res[q] = vadd(res[q], t[q]);
      }
    } else if constexpr (RK == RK_LSE) {
      next(res);
      if (n > 1 || a.eps != T(0)) {
        LseOp<T> op[VP];
#pragma unroll
        for (int q = 0; q < VP; ++q) {
          op[q].eps = a.eps;
          op[q].begin(n);
          op[q].push(res[q]);
        }
        Vec<T> v[VP];
        for (int j = 1; j < n; ++j) {
          next(v);
#pragma unroll
          for (int q = 0; q < VP; ++q) op[q].push(v[q]);
        }
#pragma unroll
        for (int q = 0; q < VP; ++q) res[q] = op[q].result();
      } else {
#pragma unroll
        for (int q = 0; q < VP; ++q) res[q] = lse_unary(res[q]);
      }
    } else {
      next(res);
      Vec<T> v[VP];
      for (int j = 1; j < n; ++j) {
        next(v);
#pragma unroll
        for (int q = 0; q < VP; ++q) seq_combine<T, RK>(res[q], v[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < VP; ++q) {
      const size_t col = col0 + (size_t)pl[q] * PIECE<T>;
      if constexpr (BWD) {
        if constexpr (G::MASKED_OUT) {
          if (out < 0) res[q] = G::unary(res[q], x[q]);
        }
        if (in_row[q]) stv(a.out + (size_t)(out & 0x7fffffff) * a.ld + col, res[q], 1);
      } else {
        if (in_row[q]) stv(a.out + (size_t)out * a.ld + col, res[q], 1);
        // route masks: one per 512-byte chunk, written by the warp covering it
        const int chunk_piece = warp * 32 + q * nt;
        if (a.mbase && chunk_piece < pv) {
          const int xr = x_id(k);
          if (xr >= 0) store_mask(a.mbase + (size_t)xr * a.ld + col0 + (size_t)chunk_piece * PIECE<T>, res[q], lane);
        }
      }
    }
  }
  if (gs != 0) {  // the last, partial group
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[grp]);
  }
#ifdef KLAY_STREAM_TRACE
  if (tr && tid == 0) {
    tr[5] = w_cyc;
    tr[6] = gt();
  }
#endif
}
#undef KLAY_TWAIT

// ring slots for a CTA chunk of pvmax pieces (about KLAY_STREAM_RING_KB of
// shared memory: several CTAs per SM)
inline int stream_ring_slots(int pvmax) {
  static const int kb = [] {
    const char* e = getenv("KLAY_STREAM_RING_KB");
    return (e && *e) ? std::max(8, atoi(e)) : 48;
  }();
  int r = kb * 1024 / (pvmax * 16);
  r = std::max(8, std::min(64, r));
  return r / SG * SG;
}

template <typename T, int RK, typename G, int VP>
inline void launch_stream_vp(const LayerArgs<T>& a, cudaStream_t s) {
  constexpr bool XS = StreamTraits<T, G>::XSLOT;
  const unsigned chunks = (unsigned)((a.V + a.spv - 1) / a.spv);
  const size_t smem = StreamSmem::bytes(a.sring, a.spv, XS);
  static std::atomic<unsigned> configured{0};
  static std::atomic<size_t> smem_set{0};  // (per process; the ring size is fixed per process)
  if (needs_config(configured) || smem > smem_set.load()) {
    cudaFuncSetAttribute(stream_kernel<T, RK, G, VP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(stream_kernel<T, RK, G, VP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    smem_set = std::max(smem_set.load(), smem);
  }
  const int nt = stream_threads(a.spv, VP);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.n_scta, chunks);
  cfg.blockDim = dim3((unsigned)(((nt + 31) / 32 + 1) * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, stream_kernel<T, RK, G, VP>, a);
}

// pieces per consumer thread: two for rows chunks of >= 1 KB (fewer
// per-slot instructions), else one (a warp per 512-byte chunk)
inline int stream_vp(int spv) {
  static const int forced = [] {
    const char* e = getenv("KLAY_STREAM_VP");
    return (e && *e) ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  return spv >= 64 ? 2 : 1;
}

template <typename T, int RK, typename G>
inline int launch_stream(const LayerArgs<T>& a0, cudaStream_t s) {
  if (a0.n_scta <= 0) return 0;
  LayerArgs<T> a = a0;
  a.spv = std::min(a.V, STREAM_MAX_PV);
  a.sring = stream_ring_slots(a.spv);
  if (stream_vp(a.spv) == 2) launch_stream_vp<T, RK, G, 2>(a, s);
  else launch_stream_vp<T, RK, G, 1>(a, s);
  return 1;
}

}  // namespace klay
