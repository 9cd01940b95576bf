// libklay C ABI: plan construction (host) and per-pass launch sequences.
// See include/klay.h for the contract and the reference mapping.
#include "klay.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "layer_api.h"

using namespace klay;

namespace {

enum { SR_REAL_ = 0, SR_LOG_ = 1 };
enum { BW_PASS_ = 0, BW_LOGSUM_ = 1, BW_REALPROD_ = 2, BW_PASSA_ = 3, BW_LOGSUM8_ = 4 };

// work-item shape (see layer_kernels.cuh)
#ifndef KLAY_TASK_EDGES
#define KLAY_TASK_EDGES 32
#endif
constexpr int TASK_EDGES_H = KLAY_TASK_EDGES;  // edges per short task (<= TASK_EDGES)
#ifndef KLAY_TASK_NODES
#define KLAY_TASK_NODES 16
#endif
constexpr int TASK_NODES_H = KLAY_TASK_NODES;  // nodes per short task (<= TASK_NODES)
// forward sum (log-sum-exp) layers: smaller short tasks (more warps per
// layer for their longer per-edge work): fwd_sum 0.289 -> 0.285 ms at B = 1024,
// 0.122 -> 0.113 ms at B = 128 (config C); product layers keep 32 / 16
#ifndef KLAY_TASK_EDGES_SUM
#define KLAY_TASK_EDGES_SUM 24
#endif
#ifndef KLAY_TASK_NODES_SUM
#define KLAY_TASK_NODES_SUM 12
#endif
constexpr int TASK_EDGES_S = KLAY_TASK_EDGES_SUM;
constexpr int TASK_NODES_S = KLAY_TASK_NODES_SUM;
#ifndef KLAY_TASK_EDGES_BWD
#define KLAY_TASK_EDGES_BWD 48  // (32: -0.3 %, 64: -0.7 %)
#endif
#ifndef KLAY_TASK_NODES_BWD
#define KLAY_TASK_NODES_BWD 24
#endif
constexpr int TASK_EDGES_BWD = KLAY_TASK_EDGES_BWD;  // backward short tasks
constexpr int TASK_NODES_BWD = KLAY_TASK_NODES_BWD;
// children of sum layers with 4-edge stage batches (log-sum / real pass
// backward): smaller tasks, bwd_logsum 0.524 -> 0.511 ms at B = 1024,
// 0.149 -> 0.128 ms at B = 128, config E +6.6 % (8-edge LOGSUM8 layers keep
// 48 / 24: C' -0.7 % otherwise)
#ifndef KLAY_TASK_EDGES_BWD_SUM
#define KLAY_TASK_EDGES_BWD_SUM 24
#endif
#ifndef KLAY_TASK_NODES_BWD_SUM
#define KLAY_TASK_NODES_BWD_SUM 12
#endif
constexpr int TASK_EDGES_BWDS = KLAY_TASK_EDGES_BWD_SUM;
constexpr int TASK_NODES_BWDS = KLAY_TASK_NODES_BWD_SUM;
constexpr int PADW_H = 32;         // padded per-item index data (klay::PADW)
#ifndef KLAY_FWD_SE
#define KLAY_FWD_SE 8
#endif
#ifndef KLAY_BWD_SE
#define KLAY_BWD_SE 8
#endif
// segments of short tasks: numpy's sequential range (<= 8 edges), and never
// more than a stage batch holds
constexpr int SHORT_FWD = KLAY_FWD_SE < 8 ? KLAY_FWD_SE : 8;  // FwdGather::SE
constexpr int SHORT_BWD = KLAY_BWD_SE < 8 ? KLAY_BWD_SE : 8;  // pass-through / real-product backward
constexpr int SHORT_BWD8 = 8;                                  // BwdGather<LOGSUM8>::SE
#ifndef KLAY_LOGSUM8_XN
#define KLAY_LOGSUM8_XN 2
#endif
constexpr int BATCH_NODES8 = KLAY_LOGSUM8_XN;  // BwdGather<LOGSUM8>::XN: nodes per stage batch
constexpr int BATCH_FWD = KLAY_FWD_SE;  // FwdGather::SE: edges per stage batch
constexpr int BATCH_BWD = KLAY_BWD_SE;  // BwdGather<PASS / PASSA / REALPROD>::SE
#ifndef KLAY_LOGSUM_SE
#define KLAY_LOGSUM_SE 4
#endif
constexpr int SHORT_BWD_SUM = KLAY_LOGSUM_SE;  // BwdGather<LOGSUM>::SE (sum layers)
#ifndef KLAY_LOGSUM_XN
#define KLAY_LOGSUM_XN KLAY_LOGSUM_SE
#endif
constexpr int BATCH_NODES4 = KLAY_LOGSUM_XN;   // BwdGather<LOGSUM>::XN
#ifndef KLAY_PW_BLOCK
#define KLAY_PW_BLOCK 128
#endif
constexpr int PW_BLOCK_H = KLAY_PW_BLOCK;  // numpy pairwise block; longer tails are split
// persistent tail (layer_kernels.cuh tail_kernel): the suffix of layers with
// at most TAIL_EDGES edges runs in one launch per direction
const int TAIL_EDGES = [] {
  const char* e = getenv("KLAY_TAIL_EDGES");
  return (e && *e) ? atoi(e) : 256;
}();
const int TAIL_CLUSTER = [] {       // CTAs per cluster (one cluster per column chunk)
  const char* e = getenv("KLAY_TAIL_CLUSTER");
  return (e && *e) ? atoi(e) : 8;
}();
#ifndef KLAY_TAIL_WARPS
#define KLAY_TAIL_WARPS 8
#endif
constexpr int TAIL_WARPS_H = KLAY_TAIL_WARPS;  // warps per CTA (== TAIL_WARPS)

const bool g_tail_debug = [] {
  const char* e = getenv("KLAY_TAIL_DEBUG");
  return e && *e && *e != '0';
}();

// KLAY_TAIL_TRACE=1: print per-layer timing of the tail kernels (debug)
const bool g_tail_trace = [] {
  const char* e = getenv("KLAY_TAIL_TRACE");
  return e && *e && *e != '0';
}();
unsigned long long* tail_trace_buf() {
  static unsigned long long* buf = nullptr;
  if (!buf) cudaMalloc(&buf, sizeof(unsigned long long) * 4 * 128);
  return buf;
}
void tail_trace_dump(const char* what, int n) {
  std::vector<unsigned long long> h(4 * 128);
  cudaDeviceSynchronize();
  cudaMemcpy(h.data(), tail_trace_buf(), h.size() * 8, cudaMemcpyDeviceToHost);
  fprintf(stderr, "%s tail (%d layers): items / arrive+prefetch / wait  [us]\n", what, n);
  for (int i = 0; i < n; ++i)
    fprintf(stderr, "  %2d %6.2f %6.2f %6.2f\n", i, (h[4 * i + 1] - h[4 * i]) * 1e-3,
            (h[4 * i + 2] - h[4 * i + 1]) * 1e-3, (h[4 * i + 3] - h[4 * i + 2]) * 1e-3);
}

const bool g_no_tail = [] {
  const char* e = getenv("KLAY_NO_TAIL");
  return e && *e && *e != '0';
}();

// column-chunk order of consecutive layer kernels (klay::LayerArgs::rev):
// 0 all first-to-last, 1 alternate per layer, 2 alternate per layer pair
const int g_chunk_order = [] {
  const char* e = getenv("KLAY_CHUNK_ORDER");
  return (e && *e) ? atoi(e) : 1;
}();
// The micro tails run one CTA (of ~200 KB shared memory) per 32-byte column
// chunk; beyond two waves of them (very large batches) the layer kernels,
// which spread each layer over the whole GPU, are used instead.
bool micro_fits(int V) {
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return (V + MICRO_P - 1) / MICRO_P <= 2 * sms;
}
int chunk_rev(int l) { return g_chunk_order == 1 ? (l & 1) : g_chunk_order == 2 ? ((l >> 1) & 1) : 0; }

// KLAY_NO_ALIAS=1: every sum row is computed and read (A/B switch)
// KLAY_NO_MICRO=1: the thinnest layers run in the persistent tail too (A/B switch)
const bool g_no_micro = [] {
  const char* e = getenv("KLAY_NO_MICRO");
  return e && *e && *e != '0';
}();

// KLAY_NO_HEAD=1: the thin bottom layers run as layer kernels (A/B switch)
const bool g_no_head = [] {
  const char* e = getenv("KLAY_NO_HEAD");
  return e && *e && *e != '0';
}();

// KLAY_STREAM=1: eligible layers on the bulk-copy streaming kernel
// (stream_kernels.cuh) instead of items_kernel. Off by default: measured
// slower on config C (DESIGN.md §4 "Streaming kernel"); kept, parity-tested,
// for A/B runs.
const bool g_no_stream = [] {
  const char* e = getenv("KLAY_STREAM");
  return !(e && *e && *e != '0');
}();

#ifdef KLAY_STREAM_TRACE
// debug builds (-DKLAY_STREAM_TRACE): per-CTA timing of one streaming launch,
// KLAY_STREAM_TRACE_LAYER = 1-based gate layer, KLAY_STREAM_TRACE_DIR = 0
// forward / 1 backward; a summary goes to stderr after the launch
void stream_trace_dump(unsigned long long* d, int n, int layer, int dir) {
  std::vector<unsigned long long> h((size_t)8 * n);
  cudaDeviceSynchronize();
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, t1 = 0;
  double wait_gdc = 0, pw = 0, cw = 0, life = 0, plife = 0;
  for (int i = 0; i < n; ++i) {
    const unsigned long long* r = &h[(size_t)8 * i];
    t0 = std::min(t0, r[0]);
    t1 = std::max(t1, r[6]);
    wait_gdc += (double)(r[1] - r[0]);
    pw += (double)r[2];
    cw += (double)r[5];
    life += (double)(r[6] - r[1]);
    plife += (double)(r[4] - r[1]);
  }
  fprintf(stderr,
          "stream trace layer %d dir %d: %d CTAs, span %.1f us; per CTA mean: gdc wait %.2f us, "
          "life %.2f us (producer %.2f us), producer empty-wait %.0f cyc, consumer full-wait %.0f cyc\n",
          layer, dir, n, (t1 - t0) * 1e-3, wait_gdc / n * 1e-3, life / n * 1e-3, plife / n * 1e-3, pw / n,
          cw / n);
  FILE* f = fopen("stream_trace.bin", "wb");
  if (f) {
    fwrite(h.data(), 8, h.size(), f);
    fclose(f);
  }
}
unsigned long long* stream_trace_buf() {
  static unsigned long long* b = nullptr;
  if (!b) cudaMalloc(&b, (size_t)8 * 8 * 148 * 16 * 8);
  return b;
}
const int g_trace_layer = [] {
  const char* e = getenv("KLAY_STREAM_TRACE_LAYER");
  return (e && *e) ? atoi(e) : -1;
}();
const int g_trace_dir = [] {
  const char* e = getenv("KLAY_STREAM_TRACE_DIR");
  return (e && *e) ? atoi(e) : 0;
}();
#endif

const bool g_no_alias = [] {
  const char* e = getenv("KLAY_NO_ALIAS");
  return e && *e && *e != '0';
}();

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define KLAY_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return fail(KLAY_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

// Kernel launches issued by this library (all threads).
std::atomic<long long> g_launches{0};

// Launch-class filter (klay_set_launch_filter; profiling only): bit c set =
// kernels of class KLAY_CLASS_* c are launched. Per thread, default all.
thread_local uint32_t g_launch_filter = 0xffffffffu;
inline bool launch_on(int cls) { return (g_launch_filter >> cls) & 1u; }

// Optional per-launch event timing (klay_profiler_begin / _end).
struct ProfRec {
  int kind, layer;
  cudaEvent_t a, b;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRec> g_prof;

// KLAY_SYNC_DEBUG=1: synchronize after every launch and report the failing one
const bool g_sync_debug = [] {
  const char* e = getenv("KLAY_SYNC_DEBUG");
  return e && *e && *e != '0';
}();

struct LaunchScope {
  cudaStream_t s;
  int kind, layer;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(cudaStream_t s_, int kind_, int layer_) : s(s_), kind(kind_), layer(layer_) {
    if (g_prof_on) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  ~LaunchScope() {
    if (g_prof_on) {
      cudaEventRecord(b, s);
      g_prof.push_back({kind, layer, a, b});
    }
    if (g_sync_debug) {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) fprintf(stderr, "libklay: launch kind %d layer %d failed: %s\n", kind, layer,
                                    cudaGetErrorString(e));
    }
  }
};

// KLAY_CHECKS builds: the call's valid ranges and a device violation record
// (common.cuh chk); a call fails with KLAY_ECUDA when a kernel recorded one
#ifdef KLAY_CHECKS
int* chk_record() {
  static int* rec = nullptr;
  if (!rec) {
    cudaMalloc(&rec, 4 * sizeof(int));
    cudaMemset(rec, 0, 4 * sizeof(int));
  }
  return rec;
}
// KLAY_CHECKS_SHRINK=<bytes>: declare only that many bytes of the values /
// trace buffer valid (negative control of the checker: legal accesses past
// it must be reported, and are redirected instead of performed)
ChkRanges chk_ranges(const void* buf, size_t buf_bytes, const void* work, size_t work_bytes) {
  static const long long shrink = [] {
    const char* e = getenv("KLAY_CHECKS_SHRINK");
    return (e && *e) ? atoll(e) : -1LL;
  }();
  if (shrink >= 0 && (size_t)shrink < buf_bytes) buf_bytes = (size_t)shrink;
  ChkRanges c{};
  c.lo[0] = static_cast<const char*>(buf);
  c.hi[0] = c.lo[0] + buf_bytes;
  c.lo[1] = static_cast<const char*>(work);
  c.hi[1] = work ? c.lo[1] + work_bytes : c.lo[1];
  c.rec = chk_record();
  return c;
}
int chk_finish(cudaStream_t s, const char* what);
#endif

struct ItemSet {
  std::vector<int4> items;
  std::vector<unsigned> masks;  // parallel to items
  std::vector<int4> heavy;
  int slots = 0;
};

void split_leaves(int a, int len, std::vector<std::pair<int, int>>& out) {
  if (len <= PW_BLOCK_H) {
    out.push_back({a, a + len});
    return;
  }
  int n2 = len / 2;
  n2 -= n2 % 8;
  split_leaves(a, n2, out);
  split_leaves(a + n2, len - n2, out);
}

// Work items over one CSR (W segments, offsets off[base..base+W]); kinds as
// documented at items_kernel (layer_kernels.cuh):
//   segments with <= short_max edges are packed into short tasks of <= cap
//   edges and <= TASK_NODES_H nodes; longer ones become long items; with
//   split, tails longer than one numpy pairwise block become leaf items.
// split == false keeps every segment whole (np.multiply.reduceat is
// sequential: it has no exact parallel decomposition).
// cap shrinks for narrow layers so that thin layers still spread over many
// warps (short per-warp dependency chains).
// lse == true (forward log-sum layers): a logsumexp has no fixed summation
// order to keep, so tails longer than LSE_SPLIT edges are split into ~8
// equal leaves of 16..128 edges: a long segment spreads over several warps
// instead of one long dependent exp chain.
constexpr int LSE_SPLIT = 32;
const int LSE_LEAF_MIN = [] {  // (KLAY_LSE_LEAF: tuning experiments)
  const char* e = getenv("KLAY_LSE_LEAF");
  return (e && *e) ? std::max(1, atoi(e)) : 16;
}();
void build_items(const std::vector<int>& off, size_t base, int W, int short_max, ItemSet& s,
                 bool split = true, int cap = 0, bool lse = false, int task_edges = TASK_EDGES_H,
                 int task_nodes = TASK_NODES_H, int batch_max = 0, int batch_nodes = 32) {
  // stage batches of <= batch_max edges (default: short_max) and <=
  // batch_nodes nodes; short_max bounds the segments of short tasks
  if (batch_max <= 0) batch_max = short_max;
  const int E = off[base + W] - off[base];
  if (cap <= 0) cap = std::max(short_max, std::min(task_edges, (E / 296) & ~7));
  std::vector<int4> leaves, longs, shorts;
  std::vector<unsigned> short_masks, leaf_heavy;
  std::vector<std::pair<int, int>> lv;
  int tb = -1, t_edges = 0;
  auto flush = [&](int end_node) {
    if (tb >= 0 && end_node > tb) {
      shorts.push_back(make_int4(tb, end_node, off[base + tb], off[base + end_node]));
      // stage batches: greedy runs of whole segments with <= short_max edges
      unsigned mask = 0;
      int n0 = tb;
      while (n0 < end_node) {
        mask |= 1u << (n0 - tb);
        const int lim = off[base + n0] + batch_max;
        int n1 = n0 + 1;
        while (n1 < end_node && n1 - n0 < batch_nodes && off[base + n1 + 1] <= lim) ++n1;
        n0 = n1;
      }
      short_masks.push_back(mask);
    }
    tb = -1;
    t_edges = 0;
  };
  for (int p = 0; p < W; ++p) {
    const int s0 = off[base + p], n = off[base + p + 1] - s0;
    if (split && n - 1 > (lse ? LSE_SPLIT : PW_BLOCK_H)) {
      flush(p);
      lv.clear();
      if (lse) {
        const int len = std::min(PW_BLOCK_H, std::max(LSE_LEAF_MIN, (n - 1 + 7) / 8));
        for (int a = s0 + 1; a < s0 + n; a += len) lv.push_back({a, std::min(a + len, s0 + n)});
      } else {
        split_leaves(s0 + 1, n - 1, lv);
      }
      s.heavy.push_back(make_int4(p, s.slots, (int)lv.size(), 0));
      for (auto& l : lv) {
        leaves.push_back(make_int4(p, -(s.slots++) - 1, l.first, l.second));
        leaf_heavy.push_back((unsigned)(s.heavy.size() - 1));  // a leaf's mask: its heavy segment
      }
    } else if (n > short_max) {
      flush(p);
      longs.push_back(make_int4(p, 0, s0, s0 + n));
    } else {
      if (tb >= 0 && (p - tb >= task_nodes || t_edges + n > cap)) flush(p);
      if (tb < 0) tb = p;
      t_edges += n;
    }
  }
  flush(W);
  s.items.reserve(leaves.size() + longs.size() + shorts.size());
  s.items.insert(s.items.end(), leaves.begin(), leaves.end());
  s.items.insert(s.items.end(), longs.begin(), longs.end());
  s.items.insert(s.items.end(), shorts.begin(), shorts.end());
  s.masks = leaf_heavy;
  s.masks.resize(leaves.size() + longs.size(), 0u);
  s.masks.insert(s.masks.end(), short_masks.begin(), short_masks.end());
}

// Streaming-kernel CTAs over the n nodes of a CSR (offsets o[base..base+n]):
// contiguous node ranges {first node, end node, first edge, end edge}
// balanced by slots (edges x slots per edge + two per node), about
// STREAM_SPC slots per CTA, at most STREAM_MAXC CTAs, each CTA's index block
// (3 ints per node + 1 per edge + 1) within STREAM_SIDX ints. The set is not
// eligible (count 0) when a segment exceeds one numpy pairwise block
// (MICRO_FAN edges): those layers keep items_kernel's heavy leaves.
const int STREAM_SPC = [] {
  const char* e = getenv("KLAY_STREAM_SPC");
  return (e && *e) ? std::max(4, atoi(e)) : 256;
}();
constexpr int STREAM_MAXC = 148 * 16;
constexpr int STREAM_SIDX_H = 2048;  // == klay::STREAM_SIDX
void build_stream_ctas(const std::vector<int>& o, size_t base, int64_t n, int per_edge, std::vector<int4>& out,
                       int64_t& at, int64_t& count) {
  at = (int64_t)out.size();
  count = 0;
  if (n <= 0) return;
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int len = o[base + i + 1] - o[base + i];
    if (len > MICRO_FAN) return;
    total += (int64_t)len * per_edge + 2;
  }
  const int64_t nc = std::max<int64_t>(1, std::min<int64_t>({(int64_t)STREAM_MAXC, n, (total + STREAM_SPC - 1) / STREAM_SPC}));
  int64_t acc = 0, c = 1, first = 0, ints = 1;
  auto emit = [&](int64_t end) {
    out.push_back(make_int4((int)first, (int)end, o[base + first], o[base + end]));
    first = end;
    ints = 1;
  };
  for (int64_t i = 0; i < n; ++i) {
    const int len = o[base + i + 1] - o[base + i];
    if (i > first && ints + 3 + len > STREAM_SIDX_H) emit(i);
    ints += 3 + len;
    acc += (int64_t)len * per_edge + 2;
    if (acc * nc >= total * c) {
      if (i + 1 < n) emit(i + 1);
      while (acc * nc >= total * c) ++c;
    }
  }
  emit(n);
  count = (int64_t)out.size() - at;
}

// a compacted item set over a subset of a layer's nodes (unary-sum aliases)
struct AliasSet {
  int64_t off_base = 0, e_base = 0, map_base = 0, xmap_base = 0;  // into aoff[] / aidx[] / omap[]
  int64_t i_base = 0, i_n = 0, h_base = 0, h_n = 0, slots = 0;
  int64_t pmap_base = -1, pxmap_base = -1;  // padded per-item maps (pmap[] / pxmap[])
  int64_t n = 0;                            // nodes of the set
};

struct LayerDesc {
  int64_t W, Wprev, E;
  bool prod;
  int64_t row, prev_row;  // row offsets into the trace buffer
  int64_t off_base;       // into off[] (W+1 entries per layer)
  int64_t e_base;         // into src[] / tpar[]
  int64_t toff_base;      // into toff[] (Wprev+1 entries per layer)
  int64_t fi_base, fi_n, fh_base, fh_n, f_slots;  // forward items / heavy
  int64_t fq_base, fq_n;                           // forward items, no split (PROD)
  int64_t fl_base, fl_n, flh_base, flh_n;          // forward items, log-sum leaves (LSE)
  int64_t bi_base, bi_n, bh_base, bh_n, b_slots;  // backward items / heavy
  // Unary-node aliases (log semiring, epsilon 0, backward-only traces; see
  // build_aliases). Per gate layer:
  //   fa_on    forward runs over its own item set fa: the non-aliased nodes,
  //            operands re-mapped (an aliased child reads its source row, a
  //            negative offset from the layer's base); fsum_redo: a product
  //            layer whose aliased children are unary sums (+inf -> NaN,
  //            redone only for +inf results)
  //   mrow_on  nodes that are the target of a masked route store the
  //            finiteness mask of their value in the route top's row
  //   ba_on    backward over the children whose adjoint is not routed (ba),
  //            absolute output rows (omap, bit 31: mask) and value rows (xmap)
  //   bmask    some outputs need the mask (pass-through layers: PASSA)
  bool fa_on, fsum_redo, mrow_on, ba_on, bmask;
  bool bsum8;  // log-sum backward with 8-edge stage batches (children with > 4 parents common)
  AliasSet fa, ba;
  // streaming kernel partitions (into d_scta; n = 0: set not eligible, a
  // segment longer than one numpy pairwise block): forward plain / alias
  // set, backward plain / alias set
  int64_t fs_b = 0, fs_n = 0, fsa_b = 0, fsa_n = 0, bs_b = 0, bs_n = 0, bsa_b = 0, bsa_n = 0;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct KlayPlan {
  int device = 0;
  int64_t K = 0;
  int32_t L = 0;
  int32_t R = 0;
  int64_t total_rows = 0;
  // backward adjoint layout (klay_plan_create, assign_adjoint_blocks): node
  // layer m's adjoint rows are rows [gbase[m], gbase[m] + W_m) of a buffer
  // of adj_rows rows; layers whose lifetimes do not overlap share rows
  std::vector<int64_t> gbase;
  int64_t adj_rows = 0;
  int64_t max_width = 0;
  int64_t max_fslots = 0, max_bslots = 0;
  int64_t max_heavy = 0;  // heavy segments of the largest layer (leaf counters)
  std::vector<LayerDesc> layers;
  std::vector<int64_t> layer_row;  // L+1 entries
  int* d_off = nullptr;
  int* d_src = nullptr;
  int* d_toff = nullptr;
  int* d_tpar = nullptr;
  int4* d_items = nullptr;
  unsigned* d_masks = nullptr;
  int4* d_heavy = nullptr;
  int* d_root_node = nullptr;
  signed char* d_const = nullptr;
  int* d_top_off = nullptr;
  int* d_top_pos = nullptr;
  int* d_aoff = nullptr;   // unary-sum aliases: compacted offsets,
  int* d_aidx = nullptr;   // compacted / remapped edge indices,
  int* d_omap = nullptr;   // item node -> node id maps
  int2* d_alias = nullptr;  // {trace row of an aliased node (bit 31: via a sum), source row}
  int* d_pidx = nullptr;   // padded per-item edge indices / offsets (parallel to d_items)
  int* d_poff = nullptr;
  int* d_pmap = nullptr;   // padded per-item maps of alias sets (omap, xmap)
  int* d_pmap2 = nullptr;
  int64_t n_alias = 0;
  int64_t WL = 0;  // width of the last layer (K when there are no gates)
  int32_t tail_from = 0;  // first layer of the persistent tail (L = no tail)
  int32_t micro_from = 0;  // first layer of the forward micro tail (L = none)
  std::vector<int> micro_at, micro_n;  // per layer: offset / length of its CSR in d_micro (-1: none)
  int* d_micro = nullptr;  // packed micro-tail CSR ([W+1] local offsets, [E] indices per layer)
  int32_t microb_from = 0;  // first layer of the backward micro tail, log semiring (L = none)
  int32_t microb_from_real = 0;  // ... real semiring (>= microb_from)
  std::vector<int> microb_at, microb_n, microbr_n;  // per layer: its CSR block, staged
                                                   // length (log / real); -1: none
  // micro heads: the thin bottom layers [0, head) in one launch per direction
  // (0 = none); no node of layers <= max head + 1 is aliased
  int32_t head_f = 0, head_b = 0, head_b_real = 0;
  int* d_microb = nullptr;
  int4* d_scta = nullptr;  // streaming kernel CTAs (LayerDesc fs_b ...; build_stream_ctas)
};

#ifdef KLAY_CHECKS
namespace {
int chk_finish(cudaStream_t s, const char* what) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs != cudaStreamCaptureStatusNone) return KLAY_OK;  // (graph capture: checked when run eagerly)
  int h[4] = {0, 0, 0, 0};
  KLAY_CUDA(cudaStreamSynchronize(s));
  KLAY_CUDA(cudaMemcpy(h, chk_record(), sizeof h, cudaMemcpyDeviceToHost));
  if (h[0] == 0) return KLAY_OK;
  KLAY_CUDA(cudaMemset(chk_record(), 0, sizeof h));
  char msg[200];
  snprintf(msg, sizeof msg, "%s: bounds check failed: %d out-of-range accesses, first at site %d in layer %d (address low bits 0x%x)",
           what, h[0], h[1], h[2], h[3]);
  return fail(KLAY_ECUDA, msg);
}
}  // namespace
#endif

extern "C" const char* klay_version(void) {
#ifdef KLAY_CHECKS
  return "libklay 0.2 sm_100a (bounds-checked build)";
#else
  return "libklay 0.2 sm_100a";
#endif
}

extern "C" const char* klay_last_error(void) { return g_err.c_str(); }

static void plan_free(KlayPlan* p) {
  if (!p) return;
  cudaFree(p->d_off);
  cudaFree(p->d_src);
  cudaFree(p->d_toff);
  cudaFree(p->d_tpar);
  cudaFree(p->d_items);
  cudaFree(p->d_masks);
  cudaFree(p->d_heavy);
  cudaFree(p->d_root_node);
  cudaFree(p->d_const);
  cudaFree(p->d_top_off);
  cudaFree(p->d_top_pos);
  cudaFree(p->d_aoff);
  cudaFree(p->d_aidx);
  cudaFree(p->d_omap);
  cudaFree(p->d_alias);
  cudaFree(p->d_pidx);
  cudaFree(p->d_poff);
  cudaFree(p->d_pmap);
  cudaFree(p->d_pmap2);
  cudaFree(p->d_micro);
  cudaFree(p->d_microb);
  cudaFree(p->d_scta);
  delete p;
}

template <typename T>
static int upload(T** dst, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(v.size(), 1) * sizeof(T);
  KLAY_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), bytes));
  if (!v.empty()) KLAY_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return KLAY_OK;
}

// Unary-node aliases (LayerDesc). With the log semiring and epsilon 0 a gate
// node with one child holds exactly its child's value: a product of one log
// value is the value, a logsumexp of one is the value (+inf -> NaN). Every
// such node below the tail (and not in the last layer) is "aliased": a
// backward-only trace never writes its row, and readers use the row of the
// chain's source, the first non-aliased node below. Adjoints flow down the
// links "child with a single parent that is aliased" unchanged (products) or
// weighted by 1 / 0 for a finite / non-finite value (sums); such a chain is a
// route: the kernel computing the adjoint of the chain's top writes it
// straight into the bottom's row, the nodes in between are never computed.
// A route through a sum needs the value's finiteness mask: the bottom's
// forward stores it into the top's (unwritten) value row.
template <typename AddSet>
static void build_aliases(KlayPlan* p, int64_t K, const int64_t* widths, const int64_t* sources,
                          const int64_t* segments, const std::vector<int>& off,
                          const std::vector<int>& toff, const std::vector<int>& tpar,
                          std::vector<int>& aoff, std::vector<int>& aidx, std::vector<int>& omap,
                          std::vector<int2>& pairs, AddSet add_set) {
  const int L = p->L;
  // nodes read by a tail (persistent or micro) are never aliased
  const int tail = std::min({p->tail_from, p->micro_from, p->microb_from});
  const int hmax = std::max({p->head_f, p->head_b, p->head_b_real});
  const int lo = hmax > 0 ? hmax + 2 : 1;
  auto width = [&](int nl) -> int64_t { return nl == 0 ? K : widths[nl - 1]; };
  auto is_sum = [](int nl) { return nl >= 1 && ((nl - 1) % 2 == 1); };
  std::vector<std::vector<int>> child(L + 1), npar(L + 1), par(L + 1), up(L + 1), srow(L + 1),
      redirect(L + 1), mrow(L + 1);
  std::vector<std::vector<char>> ali(L + 1), skip(L + 1), tf(L + 1);
  for (int nl = 0; nl <= L; ++nl) {
    const int64_t w = width(nl);
    child[nl].assign(w, -1);
    npar[nl].assign(w, 0);
    par[nl].assign(w, -1);
    up[nl].assign(w, -1);
    srow[nl].resize(w);
    redirect[nl].assign(w, -1);
    mrow[nl].assign(w, -1);
    ali[nl].assign(w, 0);
    skip[nl].assign(w, 0);
    tf[nl].assign(w, 0);
    for (int64_t i = 0; i < w; ++i) srow[nl][i] = (int)(p->layer_row[nl] + i);
  }
  for (int l = 0; l < L; ++l) {
    const LayerDesc& d = p->layers[l];
    const int64_t* S = sources + d.e_base;
    const int64_t* G = segments + d.e_base;
    for (int64_t i = 0; i < d.W; ++i) {
      const int c0 = off[d.off_base + i], c1 = off[d.off_base + i + 1];
      if (c1 - c0 == 1) child[l + 1][i] = (int)S[c0];
    }
    for (int64_t e = 0; e < d.E; ++e) {
      ++npar[l][S[e]];
      par[l][S[e]] = (int)G[e];
    }
  }
  // aliased nodes: unary, read by a regular (non-tail) kernel of the next layer
  for (int nl = lo; nl < L && nl < tail; ++nl)
    for (int64_t i = 0; i < width(nl); ++i) {
      const int c = child[nl][i];
      if (c < 0) continue;
      ali[nl][i] = 1;
      srow[nl][i] = srow[nl - 1][c];
      tf[nl][i] = is_sum(nl) || tf[nl - 1][c];
      pairs.push_back(make_int2((int)(p->layer_row[nl] + i) | (tf[nl][i] ? INT32_MIN : 0), srow[nl][i]));
    }
  // routes
  static const int dbg_routes = [] {  // KLAY_ROUTES=0: no routes, 1: unmasked only (A/B, debug)
    const char* e = getenv("KLAY_ROUTES");
    return (e && *e) ? atoi(e) : 2;
  }();
  for (int nl = 0; nl < L && dbg_routes > 0; ++nl)
    for (int64_t i = 0; i < width(nl); ++i)
      if (npar[nl][i] == 1 && ali[nl + 1][par[nl][i]]) up[nl][i] = par[nl][i];
  for (int nl = 0; nl < L; ++nl)
    for (int64_t i = 0; i < width(nl); ++i) {
      if (up[nl][i] < 0) continue;
      if (ali[nl][i] && up[nl - 1][child[nl][i]] == (int)i) continue;  // inside a longer chain
      int tl = nl, t = (int)i;
      bool masked = false;
      while (up[tl][t] >= 0) {
        t = up[tl][t];
        ++tl;
        masked |= is_sum(tl);
      }
      // a masked route needs a computed bottom to write the mask
      if (masked && (ali[nl][i] || nl == 0 || dbg_routes < 2)) continue;
      for (int sl = nl, sj = (int)i; sl < tl; sj = up[sl][sj], ++sl) skip[sl][sj] = 1;
      redirect[tl][t] = (int)(p->layer_row[nl] + i) | (masked ? INT32_MIN : 0);
      if (masked) mrow[nl][i] = (int)(p->layer_row[tl] + t);
    }
  // per gate layer l (nodes: node layer l + 1, children: node layer l)
  for (int l = 0; l < L; ++l) {
    LayerDesc& d = p->layers[l];
    const int nl = l + 1;
    const int64_t W = d.W, Wp = d.Wprev;
    const int64_t* S = sources + d.e_base;
    auto operand = [&](int64_t c) -> int {
      return ali[l][c] ? (int)(srow[l][c] - p->layer_row[l]) : (int)c;
    };
    bool any_child_ali = false, any_ali = false, any_mrow = false;
    for (int64_t c = 0; c < Wp; ++c) any_child_ali |= ali[l][c] != 0;
    for (int64_t i = 0; i < W; ++i) {
      any_ali |= ali[nl][i] != 0;
      any_mrow |= mrow[nl][i] >= 0;
    }
    d.fsum_redo = d.prod && any_child_ali;  // (a product layer's aliased children are unary sums)
    if (any_child_ali || any_ali || any_mrow) {
      // own forward item set: the computed nodes, operands at source rows,
      // node ids (compacted) and mask rows
      d.fa_on = true;
      ItemSet fa;
      d.fa.off_base = (int64_t)aoff.size();
      d.fa.e_base = (int64_t)aidx.size();
      aoff.push_back(0);
      int64_t nc = 0, ec = 0;
      std::vector<int> ids, mr;
      for (int64_t i = 0; i < W; ++i) {
        if (ali[nl][i]) continue;
        const int c0 = off[d.off_base + i], c1 = off[d.off_base + i + 1];
        for (int e = c0; e < c1; ++e) aidx.push_back(operand(S[e]));
        ec += c1 - c0;
        aoff.push_back((int)ec);
        ids.push_back((int)i);
        mr.push_back(mrow[nl][i]);
        ++nc;
      }
      d.fa.map_base = any_ali ? (int64_t)omap.size() : -1;  // (-1: identity)
      if (any_ali) omap.insert(omap.end(), ids.begin(), ids.end());
      d.fa.xmap_base = any_mrow ? (int64_t)omap.size() : -1;
      if (any_mrow) omap.insert(omap.end(), mr.begin(), mr.end());
      d.mrow_on = any_mrow;
      d.fa.n = nc;
      build_items(aoff, (size_t)d.fa.off_base, (int)nc, SHORT_FWD, fa, true, 0, !d.prod,
                  d.prod ? TASK_EDGES_H : TASK_EDGES_S, d.prod ? TASK_NODES_H : TASK_NODES_S, BATCH_FWD);
      add_set(fa, d.fa, aoff, (size_t)d.fa.off_base, aidx, (size_t)d.fa.e_base);
      p->max_fslots = std::max<int64_t>(p->max_fslots, fa.slots);
      p->max_heavy = std::max<int64_t>(p->max_heavy, (int64_t)fa.heavy.size());
    }
    // backward over children whose adjoint is not routed
    bool any_skip = false, any_top = false, any_masked = false;
    for (int64_t c = 0; c < Wp; ++c) {
      any_skip |= skip[l][c] != 0;
      any_top |= redirect[l][c] != -1;  // (a masked redirect is negative: bit 31)
      any_masked |= redirect[l][c] != -1 && (redirect[l][c] & INT32_MIN);
    }
    const bool logsum = !d.prod;  // (log domain: own values needed for the softmax weights)
    if (any_skip || any_top || (logsum && any_child_ali)) {
      d.ba_on = true;
      d.bmask = !logsum && any_masked;
      ItemSet ba;
      d.ba.off_base = (int64_t)aoff.size();
      d.ba.e_base = (int64_t)aidx.size();
      aoff.push_back(0);
      int64_t nc = 0, ec = 0;
      std::vector<int> outs, xs;
      for (int64_t c = 0; c < Wp; ++c) {
        if (skip[l][c]) continue;
        const int t0 = toff[d.toff_base + c], t1 = toff[d.toff_base + c + 1];
        for (int t = t0; t < t1; ++t) aidx.push_back(tpar[d.e_base + t]);
        ec += t1 - t0;
        aoff.push_back((int)ec);
        outs.push_back(redirect[l][c] != -1 ? redirect[l][c] : (int)(p->layer_row[l] + c));
        xs.push_back(logsum ? srow[l][c] : (int)(p->layer_row[l] + c));
        ++nc;
      }
      d.ba.n = nc;
      d.ba.map_base = (int64_t)omap.size();
      omap.insert(omap.end(), outs.begin(), outs.end());
      d.ba.xmap_base = (int64_t)omap.size();
      omap.insert(omap.end(), xs.begin(), xs.end());
      build_items(aoff, (size_t)d.ba.off_base, (int)nc, d.prod ? SHORT_BWD : (d.bsum8 ? SHORT_BWD8 : SHORT_BWD_SUM),
                  ba, true, 0, false, (d.prod || d.bsum8) ? TASK_EDGES_BWD : TASK_EDGES_BWDS,
                  (d.prod || d.bsum8) ? TASK_NODES_BWD : TASK_NODES_BWDS, d.prod ? BATCH_BWD : 0,
                  d.prod ? 32 : (d.bsum8 ? BATCH_NODES8 : BATCH_NODES4));
      add_set(ba, d.ba, aoff, (size_t)d.ba.off_base, aidx, (size_t)d.ba.e_base);
      p->max_bslots = std::max<int64_t>(p->max_bslots, ba.slots);
      p->max_heavy = std::max<int64_t>(p->max_heavy, (int64_t)ba.heavy.size());
    }
  }
}

// Adjoint rows are needed only from their first write to their last read in
// the backward sweep (time t = L-1-l while gate layer l runs): node layer m
// is written by gate layer m (t = L-1-m; the seed writes layer L at t = -1)
// or earlier by a route top above it (alias item sets: outs of gate layer l
// landing in layer m at t = L-1-l), and read by gate layer m-1 (t = L-m) --
// the micro tail reads layer L when it launches, a micro head its top layer
// at t = L-1, and the gradient copy reads layer 0 at the end (t = L). Every
// column chunk runs the layers in this order (grid dependencies between
// layer kernels, barriers inside the tail / micro kernels), so layers with
// disjoint lifetimes can share rows: blocks are placed first-fit in order of
// first write. Config C (B = 1024 fp32): 4.16 GB of adjoints -> see
// DESIGN.md §3.
static void assign_adjoint_blocks(KlayPlan* p, const std::vector<int64_t>& first_write) {
  const int L = p->L;
  auto width = [&](int m) -> int64_t { return p->layer_row[m + 1 <= L ? m + 1 : L] - p->layer_row[m]; };
  std::vector<int64_t> st(L + 1), en(L + 1);
  for (int m = 0; m <= L; ++m) {
    st[m] = std::min<int64_t>(m == L ? -1 : L - 1 - m, first_write[m]);
    en[m] = (m == 0) ? L : L - m;
  }
  const int32_t mb = std::min(p->microb_from, p->microb_from_real);
  en[L] = std::max<int64_t>(en[L], (int64_t)L - 1 - mb);
  if (p->head_b > 0) en[p->head_b] = std::max<int64_t>(en[p->head_b], L - 1);
  if (p->head_b_real > 0) en[p->head_b_real] = std::max<int64_t>(en[p->head_b_real], L - 1);
  std::vector<int> order(L + 1);
  for (int m = 0; m <= L; ++m) order[m] = m;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return st[a] < st[b]; });
  struct Blk {
    int64_t off, size, end;
  };
  std::vector<Blk> live;  // sorted by offset
  p->gbase.assign(L + 1, 0);
  p->adj_rows = 0;
  for (int m : order) {
    // blocks whose last read precedes this layer's first write are free
    live.erase(std::remove_if(live.begin(), live.end(), [&](const Blk& b) { return b.end < st[m]; }), live.end());
    std::sort(live.begin(), live.end(), [](const Blk& a, const Blk& b) { return a.off < b.off; });
    const int64_t w = (m == L) ? p->WL : width(m);
    int64_t at = 0;
    for (const Blk& b : live) {
      if (b.off - at >= w) break;
      at = std::max(at, b.off + b.size);
    }
    p->gbase[m] = at;
    live.push_back({at, w, en[m]});
    p->adj_rows = std::max(p->adj_rows, at + w);
  }
}

extern "C" int klay_plan_create(int64_t num_inputs, int32_t num_layers, const int64_t* widths,
                                const int64_t* edge_counts, const int64_t* sources,
                                const int64_t* segments, int32_t num_roots,
                                const int64_t* root_nodes, const int8_t* const_vals,
                                int32_t device, KlayPlan** out) {
  if (!out) return fail(KLAY_EINVAL, "out is NULL");
  *out = nullptr;
  if (num_inputs < 0 || num_layers < 0 || num_roots < 0)
    return fail(KLAY_EINVAL, "negative size");
  if (num_layers > 0 && (!widths || !edge_counts || !sources || !segments))
    return fail(KLAY_EINVAL, "NULL layer arrays");
  if (num_roots > 0 && (!root_nodes || !const_vals)) return fail(KLAY_EINVAL, "NULL root arrays");
  if (num_inputs >= (1LL << 31)) return fail(KLAY_EINVAL, "too many inputs for int32 indexing");

  KlayPlan* p = new KlayPlan();
  p->device = device;
  p->K = num_inputs;
  p->L = num_layers;
  p->R = num_roots;

  std::vector<int> off, src, toff, tpar;
  std::vector<int4> items, heavy;
  std::vector<unsigned> masks;  // parallel to items
  std::vector<int> aoff, aidx, omap;
  std::vector<int2> alias_rows;
  // Padded per-item index data (PADW ints per item, parallel to items[]):
  // the edge indices of items with <= PADW edges and the raw segment offsets
  // of short tasks, so a warp fetches an item's structure in one round trip
  // instead of descriptor-then-indices (klay::item_regs_from).
  std::vector<int> pidx, poff, pmap, pxmap;
  auto pad_items = [&](const std::vector<int4>& its, const std::vector<int>& ov, size_t ob,
                       const std::vector<int>& iv, size_t ib) {
    for (const int4& it : its) {
      const int ne = it.w - it.z, nn = it.y > 0 ? it.y - it.x : -1;
      for (int j = 0; j < PADW_H; ++j) {
        pidx.push_back(ne <= PADW_H && j < ne ? iv[ib + it.z + j] : 0);
        poff.push_back(j <= nn ? ov[ob + it.x + j] : 0);
      }
    }
  };
  auto pad_maps = [&](const std::vector<int4>& its, std::vector<int>& dst, int64_t base) -> int64_t {
    if (base < 0) return -1;
    const int64_t at = (int64_t)dst.size();
    for (const int4& it : its) {
      const int nn = it.y > 0 ? it.y - it.x : 1;
      for (int j = 0; j < PADW_H; ++j) dst.push_back(j < nn ? omap[(size_t)base + it.x + j] : 0);
    }
    return at;
  };
  auto add_set = [&](ItemSet& set, AliasSet& as, const std::vector<int>& ov, size_t ob,
                     const std::vector<int>& iv, size_t ib) {
    as.i_base = (int64_t)items.size();
    as.i_n = (int64_t)set.items.size();
    items.insert(items.end(), set.items.begin(), set.items.end());
    masks.insert(masks.end(), set.masks.begin(), set.masks.end());
    pad_items(set.items, ov, ob, iv, ib);
    as.pmap_base = pad_maps(set.items, pmap, as.map_base);
    as.pxmap_base = pad_maps(set.items, pxmap, as.xmap_base);
    as.h_base = (int64_t)heavy.size();
    as.h_n = (int64_t)set.heavy.size();
    heavy.insert(heavy.end(), set.heavy.begin(), set.heavy.end());
    as.slots = set.slots;
  };
  // the tail: longest suffix of layers with <= TAIL_EDGES edges
  int32_t tail_from = num_layers;
  while (tail_from > 0 && num_layers - tail_from < TAIL_MAX_LAYERS &&
         edge_counts[tail_from - 1] <= TAIL_EDGES)
    --tail_from;
  p->tail_from = tail_from;
  int64_t prev_w = num_inputs, row = num_inputs, e_base = 0;
  p->max_width = num_inputs;
  p->layer_row.push_back(0);
  auto bad = [&](int code, const std::string& m) {
    plan_free(p);
    return fail(code, m);
  };
  for (int32_t l = 0; l < num_layers; ++l) {
    const int64_t W = widths[l], E = edge_counts[l];
    const int64_t* S = sources + e_base;
    const int64_t* G = segments + e_base;
    const std::string where = "layer " + std::to_string(l + 1) + ": ";
    // invariants of tensorize.py:105-125
    if (W <= 0) return bad(KLAY_EFORMAT, where + "nonpositive width");
    if (E <= 0) return bad(KLAY_EFORMAT, where + "no edges");
    if (W >= (1LL << 31) || E >= (1LL << 31) || (int64_t)src.size() + E >= (1LL << 31))
      return bad(KLAY_EINVAL, where + "exceeds int32 indexing");
    LayerDesc d{};
    d.W = W; d.Wprev = prev_w; d.E = E; d.prod = (l % 2 == 0);
    d.row = row; d.prev_row = row - prev_w;
    d.off_base = (int64_t)off.size();
    d.e_base = e_base;
    d.toff_base = (int64_t)toff.size();
    // CSR offsets of the parent segments (engine.py:144-146)
    std::vector<int64_t> cnt(W, 0), gcnt(prev_w, 0);
    for (int64_t e = 0; e < E; ++e) {
      if (e > 0 && G[e] < G[e - 1]) return bad(KLAY_EFORMAT, where + "aggregation indices not nondecreasing");
      if (G[e] < 0 || G[e] >= W) return bad(KLAY_EFORMAT, where + "aggregation indices must cover 0..width-1");
      if (S[e] < 0 || S[e] >= prev_w) return bad(KLAY_EFORMAT, where + "edge index out of range");
      ++cnt[G[e]];
      ++gcnt[S[e]];
    }
    off.push_back(0);
    int64_t acc = 0;
    for (int64_t i = 0; i < W; ++i) {
      if (cnt[i] == 0) return bad(KLAY_EFORMAT, where + "aggregation indices must cover 0..width-1");
      acc += cnt[i];
      off.push_back((int)acc);
    }
    for (int64_t e = 0; e < E; ++e) src.push_back((int)S[e]);
    // transposed CSR: stable counting sort of the edges by source
    // (engine.py:147-152), i.e. ascending edge order inside each child
    std::vector<int64_t> pos(prev_w);
    toff.push_back(0);
    acc = 0;
    for (int64_t j = 0; j < prev_w; ++j) {
      if (gcnt[j] == 0) return bad(KLAY_EFORMAT, where + "some previous-layer node is never read");
      pos[j] = acc;
      acc += gcnt[j];
      toff.push_back((int)acc);
    }
    const size_t tb = tpar.size();
    tpar.resize(tb + E);
    // bit 31 marks an edge whose parent is a unary sum: its forward value is
    // the child's own when epsilon is 0, so the LOGSUM backward never loads it
    for (int64_t e = 0; e < E; ++e)
      tpar[tb + pos[S[e]]++] = (int)G[e] | ((!d.prod && cnt[G[e]] == 1) ? INT32_MIN : 0);
    // work items: forward over parents, backward over children
    ItemSet fs, bs;
    // tail layers: about one item per cluster warp (fewer, larger items)
    const int tcap = (l >= tail_from)
        ? std::max(8, std::min(TASK_EDGES_H, (int)((E + TAIL_CLUSTER * TAIL_WARPS_H - 1) /
                                                   (TAIL_CLUSTER * TAIL_WARPS_H) + 7) & ~7))
        : 0;
    build_items(off, (size_t)d.off_base, (int)W, SHORT_FWD, fs, true, tcap, false,
                d.prod ? TASK_EDGES_H : TASK_EDGES_S, d.prod ? TASK_NODES_H : TASK_NODES_S, BATCH_FWD);
    // log-sum backward: 4-edge stage batches unless children with more
    // parents are common (> 5 %), which would otherwise all become long items
    if (!d.prod && l < tail_from) {
      int64_t many = 0;
      for (int64_t j = 0; j < prev_w; ++j) many += gcnt[j] > SHORT_BWD_SUM;
      static const int force8 = [] {  // KLAY_LOGSUM8=0/1: A/B override
        const char* e = getenv("KLAY_LOGSUM8");
        return (e && *e) ? atoi(e) : -1;
      }();
      d.bsum8 = force8 >= 0 ? force8 == 1 : many * 20 > prev_w;
    }
    build_items(toff, (size_t)d.toff_base, (int)prev_w, d.prod ? SHORT_BWD : (d.bsum8 ? SHORT_BWD8 : SHORT_BWD_SUM),
                bs, true, tcap, false, (d.prod || d.bsum8) ? TASK_EDGES_BWD : TASK_EDGES_BWDS,
                (d.prod || d.bsum8) ? TASK_NODES_BWD : TASK_NODES_BWDS, d.prod ? BATCH_BWD : 0,
                d.prod ? 32 : (d.bsum8 ? BATCH_NODES8 : BATCH_NODES4));
    d.fi_base = (int64_t)items.size();
    d.fi_n = (int64_t)fs.items.size();
    items.insert(items.end(), fs.items.begin(), fs.items.end());
    masks.insert(masks.end(), fs.masks.begin(), fs.masks.end());
    pad_items(fs.items, off, (size_t)d.off_base, src, (size_t)d.e_base);
    d.fq_base = d.fi_base;
    d.fq_n = d.fi_n;
    if (d.prod && !fs.heavy.empty()) {
      ItemSet qs;
      build_items(off, (size_t)d.off_base, (int)W, SHORT_FWD, qs, false, tcap, false, TASK_EDGES_H, TASK_NODES_H,
                  BATCH_FWD);
      d.fq_base = (int64_t)items.size();
      d.fq_n = (int64_t)qs.items.size();
      items.insert(items.end(), qs.items.begin(), qs.items.end());
      masks.insert(masks.end(), qs.masks.begin(), qs.masks.end());
      pad_items(qs.items, off, (size_t)d.off_base, src, (size_t)d.e_base);
    }
    // log-sum layers with long segments: an item set with short leaves
    d.fl_base = d.fi_base;
    d.fl_n = 0;
    ItemSet ls;
    if (!d.prod && l < tail_from) {
      int maxn = 0;
      for (int64_t i = 0; i < W; ++i) maxn = std::max(maxn, off[d.off_base + i + 1] - off[d.off_base + i]);
      if (maxn - 1 > LSE_SPLIT) {
        build_items(off, (size_t)d.off_base, (int)W, SHORT_FWD, ls, true, 0, true, TASK_EDGES_S, TASK_NODES_S,
                    BATCH_FWD);
        d.fl_base = (int64_t)items.size();
        d.fl_n = (int64_t)ls.items.size();
        items.insert(items.end(), ls.items.begin(), ls.items.end());
        masks.insert(masks.end(), ls.masks.begin(), ls.masks.end());
        pad_items(ls.items, off, (size_t)d.off_base, src, (size_t)d.e_base);
      }
    }
    d.bi_base = (int64_t)items.size();
    d.bi_n = (int64_t)bs.items.size();
    items.insert(items.end(), bs.items.begin(), bs.items.end());
    masks.insert(masks.end(), bs.masks.begin(), bs.masks.end());
    pad_items(bs.items, toff, (size_t)d.toff_base, tpar, (size_t)d.e_base);
    d.fh_base = (int64_t)heavy.size();
    d.fh_n = (int64_t)fs.heavy.size();
    p->max_heavy = std::max<int64_t>(p->max_heavy, std::max(fs.heavy.size(), bs.heavy.size()));
    heavy.insert(heavy.end(), fs.heavy.begin(), fs.heavy.end());
    d.bh_base = (int64_t)heavy.size();
    d.bh_n = (int64_t)bs.heavy.size();
    heavy.insert(heavy.end(), bs.heavy.begin(), bs.heavy.end());
    d.flh_base = (int64_t)heavy.size();
    d.flh_n = (int64_t)ls.heavy.size();
    heavy.insert(heavy.end(), ls.heavy.begin(), ls.heavy.end());
    p->max_heavy = std::max<int64_t>(p->max_heavy, (int64_t)ls.heavy.size());
    p->max_fslots = std::max<int64_t>(p->max_fslots, ls.slots);
    d.f_slots = fs.slots;
    d.b_slots = bs.slots;
    p->max_fslots = std::max<int64_t>(p->max_fslots, fs.slots);
    p->max_bslots = std::max<int64_t>(p->max_bslots, bs.slots);
    p->layers.push_back(d);
    p->layer_row.push_back(row);
    p->max_width = std::max(p->max_width, W);
    row += W;
    e_base += E;
    prev_w = W;
  }
  p->total_rows = row;
  p->WL = prev_w;
  // micro tails: the longest suffix of layers that fit them (widths, fan-in
  // (forward) / fan-out (backward) and one layer's CSR bounded); a layer's
  // CSR block starts 16-byte aligned for the per-layer cp.async staging
  // mode 0: forward; 1: backward, log semiring (transposed CSR); 2: backward,
  // real semiring (product layers also need their forward CSR: zero-safe
  // adjoint). Returns the first layer of the longest qualifying suffix.
  auto micro_ok = [&](int mode, int32_t l) {
    const LayerDesc& d = p->layers[l];
    const bool fwd = mode == 0;
    const std::vector<int>& o = fwd ? off : toff;
    const int64_t base = fwd ? d.off_base : d.toff_base, nodes = fwd ? d.W : d.Wprev;
    int maxfan = 0;
    for (int64_t i = 0; i < nodes; ++i) maxfan = std::max(maxfan, o[base + i + 1] - o[base + i]);
    const int wmax = fwd ? MICRO_WF : MICRO_WB, cmax = fwd ? MICRO_CSRF : MICRO_CSRB;
    const int64_t ints = nodes + 1 + d.E + ((mode == 2 && d.prod) ? d.W + 1 + d.E : 0);
    return d.W <= wmax && d.Wprev <= wmax && maxfan <= MICRO_FAN && ints <= cmax;
  };
  // longest qualifying suffix (micro tail) and prefix below it (micro head;
  // at least two layers, else a plain layer launch is as good)
  auto micro_suffix = [&](int mode) -> int32_t {
    int32_t mf = num_layers;
    while (mf > 0 && num_layers - mf < MICRO_MAX_LAYERS && micro_ok(mode, mf - 1)) --mf;
    return mf;
  };
  // (head layers must be really thin, <= MICRO_HEAD_W nodes: wider bottom
  // layers run faster as layer kernels spread over the whole GPU)
  auto micro_head = [&](int mode, int32_t suffix) -> int32_t {
    const int32_t lim = std::min(suffix, tail_from);  // below every tail
    int32_t h = 0;
    while (h < lim && h < MICRO_MAX_LAYERS && micro_ok(mode, h) &&
           p->layers[h].W <= MICRO_HEAD_W && p->layers[h].Wprev <= MICRO_HEAD_W)
      ++h;
    return h >= 2 ? h : 0;
  };
  std::vector<int> micro, microb;
  p->micro_from = micro_suffix(0);
  p->microb_from = micro_suffix(1);
  p->microb_from_real = std::max(micro_suffix(2), p->microb_from);
  p->head_f = micro_head(0, p->micro_from);
  p->head_b = micro_head(1, p->microb_from);
  p->head_b_real = std::min(micro_head(2, p->microb_from_real), p->head_b);
  p->micro_at.assign(num_layers, -1);
  p->micro_n.assign(num_layers, -1);
  p->microb_at.assign(num_layers, -1);
  p->microb_n.assign(num_layers, -1);
  p->microbr_n.assign(num_layers, -1);
  for (int32_t l = 0; l < num_layers; ++l) {
    if (l < p->head_f || l >= p->micro_from) {
      const LayerDesc& d = p->layers[l];
      p->micro_at[l] = (int)micro.size();
      for (int64_t i = 0; i <= d.W; ++i) micro.push_back(off[d.off_base + i]);
      for (int64_t e = 0; e < d.E; ++e) micro.push_back(src[d.e_base + e]);
      p->micro_n[l] = (int)micro.size() - p->micro_at[l];
      while (micro.size() % 4) micro.push_back(0);
    }
    // backward blocks: [transposed offsets, parents], then for product
    // layers [forward offsets, children] (staged by the real semiring only)
    if (l < p->head_b || l >= p->microb_from) {
      const LayerDesc& d = p->layers[l];
      p->microb_at[l] = (int)microb.size();
      for (int64_t j = 0; j <= d.Wprev; ++j) microb.push_back(toff[d.toff_base + j]);
      for (int64_t e = 0; e < d.E; ++e) microb.push_back(tpar[d.e_base + e]);
      p->microb_n[l] = (int)microb.size() - p->microb_at[l];
      if (d.prod) {
        for (int64_t i = 0; i <= d.W; ++i) microb.push_back(off[d.off_base + i]);
        for (int64_t e = 0; e < d.E; ++e) microb.push_back(src[d.e_base + e]);
      }
      p->microbr_n[l] = (int)microb.size() - p->microb_at[l];
      while (microb.size() % 4) microb.push_back(0);
    }
  }
  if (num_layers >= 2 && row < (1LL << 30)) {
    build_aliases(p, num_inputs, widths, sources, segments, off, toff, tpar, aoff, aidx, omap,
                  alias_rows,
                  [&](ItemSet& set, AliasSet& as, const std::vector<int>& ov, size_t ob,
                      const std::vector<int>& iv, size_t ib) { add_set(set, as, ov, ob, iv, ib); });
  }
  p->n_alias = (int64_t)alias_rows.size();
  // backward adjoint blocks; alias item sets' absolute output rows (route
  // bottoms, own rows) become adjoint-buffer rows
  {
    auto layer_of = [&](int64_t r) -> int {
      return (int)(std::upper_bound(p->layer_row.begin(), p->layer_row.end(), r) - p->layer_row.begin()) - 1;
    };
    std::vector<int64_t> first_write(num_layers + 1, INT64_MAX);
    for (int32_t l = 0; l < num_layers; ++l) {
      const LayerDesc& d = p->layers[l];
      if (!d.ba_on) continue;
      for (int64_t j = 0; j < d.ba.n; ++j) {
        const int m = layer_of(omap[(size_t)d.ba.map_base + j] & 0x7fffffff);
        first_write[m] = std::min<int64_t>(first_write[m], (int64_t)num_layers - 1 - l);
      }
    }
    assign_adjoint_blocks(p, first_write);
    auto to_adj = [&](int v) -> int {
      const int64_t r = v & 0x7fffffff;
      const int m = layer_of(r);
      return (int)(p->gbase[m] + (r - p->layer_row[m])) | (v & INT32_MIN);
    };
    for (int32_t l = 0; l < num_layers; ++l) {
      const LayerDesc& d = p->layers[l];
      if (!d.ba_on) continue;
      for (int64_t j = 0; j < d.ba.n; ++j) omap[(size_t)d.ba.map_base + j] = to_adj(omap[(size_t)d.ba.map_base + j]);
      // (the padded per-item copies: unused padding entries stay in range)
      for (int64_t j = 0; j < d.ba.i_n * PADW_H; ++j) pmap[(size_t)d.ba.pmap_base + j] = to_adj(pmap[(size_t)d.ba.pmap_base + j]);
    }
  }
  // streaming kernel partitions of every layer's node sets
  std::vector<int4> scta;
  for (int32_t l = 0; l < num_layers; ++l) {
    LayerDesc& d = p->layers[l];
    build_stream_ctas(off, (size_t)d.off_base, d.W, 1, scta, d.fs_b, d.fs_n);
    if (d.fa_on) build_stream_ctas(aoff, (size_t)d.fa.off_base, d.fa.n, 1, scta, d.fsa_b, d.fsa_n);
    build_stream_ctas(toff, (size_t)d.toff_base, d.Wprev, 2, scta, d.bs_b, d.bs_n);
    if (d.ba_on) build_stream_ctas(aoff, (size_t)d.ba.off_base, d.ba.n, 2, scta, d.bsa_b, d.bsa_n);
  }

  // roots (engine.py:203-212, 330-334)
  std::vector<int> rn(num_roots);
  std::vector<signed char> cv(num_roots);
  std::vector<std::vector<int>> by_node(prev_w);
  for (int32_t q = 0; q < num_roots; ++q) {
    rn[q] = (int)root_nodes[q];
    cv[q] = const_vals[q] ? 1 : 0;
    if (root_nodes[q] >= prev_w || root_nodes[q] < -1)
      return bad(KLAY_EFORMAT, "root index outside final layer");
    if (root_nodes[q] >= 0) by_node[root_nodes[q]].push_back(q);
  }
  std::vector<int> top_off(1, 0), top_pos;
  for (int64_t j = 0; j < prev_w; ++j) {
    for (int q : by_node[j]) top_pos.push_back(q);
    top_off.push_back((int)top_pos.size());
  }

  DeviceGuard guard(device);
  int rc;
  if ((rc = upload(&p->d_off, off)) || (rc = upload(&p->d_src, src)) ||
      (rc = upload(&p->d_toff, toff)) || (rc = upload(&p->d_tpar, tpar)) ||
      (rc = upload(&p->d_items, items)) || (rc = upload(&p->d_masks, masks)) ||
      (rc = upload(&p->d_heavy, heavy)) ||
      (rc = upload(&p->d_root_node, rn)) || (rc = upload(&p->d_const, cv)) ||
      (rc = upload(&p->d_top_off, top_off)) || (rc = upload(&p->d_top_pos, top_pos)) ||
      (rc = upload(&p->d_aoff, aoff)) || (rc = upload(&p->d_aidx, aidx)) ||
      (rc = upload(&p->d_omap, omap)) || (rc = upload(&p->d_alias, alias_rows)) ||
      (rc = upload(&p->d_pidx, pidx)) || (rc = upload(&p->d_poff, poff)) ||
      (rc = upload(&p->d_pmap, pmap)) || (rc = upload(&p->d_pmap2, pxmap)) ||
      (rc = upload(&p->d_micro, micro)) || (rc = upload(&p->d_microb, microb)) ||
      (rc = upload(&p->d_scta, scta))) {
    plan_free(p);
    return rc;
  }
  *out = p;
  return KLAY_OK;
}

extern "C" int klay_plan_destroy(KlayPlan* plan) {
  if (!plan) return KLAY_OK;
  DeviceGuard guard(plan->device);
  plan_free(plan);
  return KLAY_OK;
}

extern "C" int64_t klay_plan_num_nodes(const KlayPlan* p) { return p ? p->total_rows : -1; }
extern "C" int64_t klay_plan_max_width(const KlayPlan* p) { return p ? p->max_width : -1; }

extern "C" int klay_plan_schedule(const KlayPlan* p, int64_t* out) {
  if (!p || !out) return fail(KLAY_EINVAL, "klay_plan_schedule: null argument");
  out[0] = p->tail_from;
  out[1] = p->micro_from;
  out[2] = p->microb_from;
  out[3] = p->n_alias;
  out[4] = p->head_f;
  out[5] = p->head_b;
  out[6] = p->adj_rows;
  out[7] = p->total_rows;
  return KLAY_OK;
}
extern "C" int64_t klay_plan_layer_offset(const KlayPlan* p, int32_t l) {
  if (!p || l < 0 || l > p->L) return -1;
  return p->layer_row[l];
}

extern "C" int64_t klay_row_stride(int64_t batch, int32_t dtype) {
  if (batch < 1) batch = 1;
  if (dtype == KLAY_U1) return ((batch + 31) / 32 + 3) / 4 * 4;  // 32-bit words, 16-byte rows
  const int64_t per16 = (dtype == KLAY_F64) ? 2 : 4;
  return (batch + per16 - 1) / per16 * per16;
}

static size_t esize(int32_t dtype) { return dtype == KLAY_F64 ? 8 : 4; }

// one int per (heavy segment, 512-byte column chunk) of a layer
static size_t counter_bytes(const KlayPlan* p, int32_t dtype, int64_t ld) {
  const int64_t chunks = (ld * (int64_t)esize(dtype) / 16 + 31) / 32;
  return ((size_t)p->max_heavy * chunks * sizeof(int) + 15) / 16 * 16;
}

extern "C" size_t klay_forward_workspace(const KlayPlan* plan, int32_t dtype, int64_t ld) {
  if (!plan || plan->max_fslots == 0) return 0;
  // heavy-segment leaf partials (LSE keeps (max, sum) pairs) + leaf counters
  return (size_t)2 * plan->max_fslots * ld * esize(dtype) + counter_bytes(plan, dtype, ld);
}

extern "C" size_t klay_backward_workspace(const KlayPlan* plan, int32_t dtype, int64_t ld) {
  if (!plan) return 0;
  return ((size_t)plan->adj_rows + plan->max_bslots) * ld * esize(dtype) +
         counter_bytes(plan, dtype, ld);
}

namespace {

// point a layer's arguments at an alias item set (items, heavy, padded data)
template <typename T>
void set_items(LayerArgs<T>& a, const KlayPlan* p, const AliasSet& as) {
  a.items = p->d_items + as.i_base;
  a.masks = p->d_masks + as.i_base;
  a.n_items = (int)as.i_n;
  a.heavy = p->d_heavy + as.h_base;
  a.n_heavy = (int)as.h_n;
  a.pidx = p->d_pidx + (size_t)as.i_base * PADW_H;
  a.poff = p->d_poff + (size_t)as.i_base * PADW_H;
  a.pmap = as.pmap_base >= 0 ? p->d_pmap + as.pmap_base : nullptr;
  a.pxmap = as.pxmap_base >= 0 ? p->d_pmap2 + as.pxmap_base : nullptr;
}

template <typename T>
LayerArgs<T> layer_args(const KlayPlan* p, const LayerDesc& d, bool fwd, int V, int64_t ld) {
  LayerArgs<T> a{};
  a.items = p->d_items + (fwd ? d.fi_base : d.bi_base);
  a.masks = p->d_masks + (fwd ? d.fi_base : d.bi_base);
  a.n_items = (int)(fwd ? d.fi_n : d.bi_n);
  a.heavy = p->d_heavy + (fwd ? d.fh_base : d.bh_base);
  a.n_heavy = (int)(fwd ? d.fh_n : d.bh_n);
  a.off = fwd ? p->d_off + d.off_base : p->d_toff + d.toff_base;
  a.pidx = p->d_pidx + (size_t)(fwd ? d.fi_base : d.bi_base) * PADW_H;
  a.poff = p->d_poff + (size_t)(fwd ? d.fi_base : d.bi_base) * PADW_H;
  a.idx = fwd ? p->d_src + d.e_base : p->d_tpar + d.e_base;
  a.V = V;
  a.ld = ld;
  a.foff = p->d_off + d.off_base;
  a.fsrc = p->d_src + d.e_base;
  a.prod = d.prod ? 1 : 0;
  return a;
}

template <typename T>
int forward_impl(const KlayPlan* p, int sr, const void* weights, int wdt, T* values, int64_t ld,
                 int retain_mode, void* outputs, int64_t B, double eps, T* work, cudaStream_t s) {
  const bool retain = retain_mode != 0;
  const int V = (int)(ld * (int64_t)sizeof(T) / 16);
  T* pingpong[2] = {values, values + (size_t)p->max_width * ld};
#ifdef KLAY_CHECKS
  const ChkRanges chk = chk_ranges(values, (size_t)(retain ? p->total_rows : 2 * p->max_width) * ld * sizeof(T), work,
                                   (size_t)2 * p->max_fslots * ld * sizeof(T) +
                                       counter_bytes(p, sizeof(T) == 8 ? KLAY_F64 : KLAY_F32, ld));
#endif
  constexpr bool U1 = std::is_same<T, unsigned>::value;
  if (p->K > 0 && launch_on(KLAY_CLASS_BOUNDARY)) {
    LaunchScope ls(s, 2, 0);
    if constexpr (U1) {
      launch_pack_inputs(weights, wdt == KLAY_F64, values, (int)p->K, B, ld, nullptr, s);
    } else {
      const T pad = (sr == SR_LOG_) ? T(0) : T(1);
      launch_load_inputs<T>(weights, wdt == KLAY_F64, values, (int)p->K, B, ld, pad, s);
    }
    ++g_launches;
  }
  const T* prev = values;
  int* hcount = nullptr;
  if (p->max_fslots > 0) {
    hcount = reinterpret_cast<int*>(work + (size_t)2 * p->max_fslots * ld);
    KLAY_CUDA(cudaMemsetAsync(hcount, 0, counter_bytes(p, sizeof(T) == 8 ? KLAY_F64 : KLAY_F32, ld), s));
  }
  const int32_t tail_from = g_no_tail ? p->L : p->tail_from;
  const int32_t micro_from = (g_no_tail || g_no_micro || !micro_fits(V)) ? p->L : p->micro_from;
  TailArgs<T>* tail = nullptr;
  if (tail_from < micro_from) {
    tail = new TailArgs<T>();
    tail->n = 0;
    tail->debug_skip = g_tail_debug ? 1 : 0;
    tail->trace_ts = g_tail_trace ? tail_trace_buf() : nullptr;
  }
  // unary-sum aliases need the rows two layers down: backward-only traces
  constexpr bool U1_ = std::is_same<T, unsigned>::value;
  const bool alias = !U1_ && sr == SR_LOG_ && eps == 0.0 && retain_mode == 2 && !g_no_alias;
  MicroArgs<T> micro{}, head{};
  const int32_t head_f = (g_no_tail || g_no_micro || g_no_head || !micro_fits(V)) ? 0 : p->head_f;
  auto run_micro = [&](MicroArgs<T>& m, int32_t first) -> int {
#ifdef KLAY_CHECKS
    m.chk = chk;
    m.chk.tag = 1000 + first;
#endif
    m.csr = p->d_micro;
    m.V = V;
    m.ld = ld;
    m.eps = (T)eps;
    if (!launch_on(KLAY_CLASS_FWD_MICRO)) return KLAY_OK;
    LaunchScope ls(s, 6, first + 1);
    int n;
    if constexpr (U1) n = launch_forward_micro_u1(m, s);
    else n = launch_forward_micro(sr, m, s);
    if (n == 0) return fail(KLAY_ECUDA, std::string("micro-tail launch failed: ") +
                                            cudaGetErrorString(cudaGetLastError()));
    g_launches += n;
    return KLAY_OK;
  };
  for (int32_t l = 0; l < p->L; ++l) {
    const LayerDesc& d = p->layers[l];
    T* cur = retain ? values + (size_t)d.row * ld : pingpong[(l + 1) & 1];
    if (l < head_f) {
      // micro head: the thin bottom layers
      const int i = head.n++;
      if (i == 0) {
        head.in = prev;
        head.w_in = (int)d.Wprev;
      }
      head.out[i] = (retain || l == head_f - 1) ? cur : nullptr;
      head.w[i] = (int)d.W;
      head.csr_at[i] = p->micro_at[l];
      head.csr_n[i] = p->micro_n[l];
      head.prod[i] = d.prod ? 1 : 0;
      if (l == head_f - 1) {
        const int rc = run_micro(head, 0);
        if (rc != KLAY_OK) {
          delete tail;
          return rc;
        }
      }
      prev = cur;
      continue;
    }
    LayerArgs<T> a = layer_args<T>(p, d, true, V, ld);
#ifdef KLAY_CHECKS
    a.chk = chk;
    a.chk.tag = l + 1;
#endif
    const bool redo = alias && d.fsum_redo;
    if (alias && d.fa_on) {
      // the layer's own set: non-aliased nodes over re-mapped operands
      set_items(a, p, d.fa);
      a.off = p->d_aoff + d.fa.off_base;
      a.idx = p->d_aidx + d.fa.e_base;
      if (d.fa.map_base >= 0) a.omap = p->d_omap + d.fa.map_base;
      if (d.fa.xmap_base >= 0) a.xmap = p->d_omap + d.fa.xmap_base;
      if (d.mrow_on) a.mbase = values;  // route masks (absolute rows)
    }
    if (sr == SR_LOG_ && !d.prod && d.fl_n > 0 && !(alias && d.fa_on)) {
      // logsumexp: long segments split into short leaves
      a.items = p->d_items + d.fl_base;
      a.masks = p->d_masks + d.fl_base;
      a.pidx = p->d_pidx + (size_t)d.fl_base * PADW_H;
      a.poff = p->d_poff + (size_t)d.fl_base * PADW_H;
      a.n_items = (int)d.fl_n;
      a.heavy = p->d_heavy + d.flh_base;
      a.n_heavy = (int)d.flh_n;
    }
    if (d.prod && (sr == SR_REAL_ || sr == KLAY_MAXPROD)) {
      // sequential product: heavy segments stay whole (no leaves, no combine)
      a.items = p->d_items + d.fq_base;
      a.masks = p->d_masks + d.fq_base;
      a.pidx = p->d_pidx + (size_t)d.fq_base * PADW_H;
      a.poff = p->d_poff + (size_t)d.fq_base * PADW_H;
      a.n_items = (int)d.fq_n;
      a.n_heavy = 0;
    }
    a.out = cur;
    a.prev = prev;
    a.eps = (T)eps;
    a.rev = chunk_rev(l);
    a.scratch = work;
    a.tpart = (long long)p->max_fslots * ld;
    if (l >= micro_from) {
      const int i = micro.n++;
      if (i == 0) {
        micro.in = prev;
        micro.w_in = (int)d.Wprev;
      }
      // ping-pong mode: only the last layer's rows are read afterwards
      micro.out[i] = (retain || l == p->L - 1) ? cur : nullptr;
      micro.w[i] = (int)d.W;
      micro.csr_at[i] = p->micro_at[l];
      micro.csr_n[i] = p->micro_n[l];
      micro.prod[i] = d.prod ? 1 : 0;
    } else if (l >= tail_from) {
      tail->layer[tail->n++] = a;
    } else if (launch_on(d.prod ? KLAY_CLASS_FWD_PROD : KLAY_CLASS_FWD_SUM)) {
      a.hcount = hcount;
      LaunchScope ls(s, 0, l + 1);
      const bool aset = alias && d.fa_on;
      const int64_t sb = aset ? d.fsa_b : d.fs_b, sn = aset ? d.fsa_n : d.fs_n;
      if constexpr (U1) {
        g_launches += launch_forward_layer_u1(d.prod, a, s);
      } else if (sn > 0 && !g_no_stream) {
        a.scta = reinterpret_cast<const int*>(p->d_scta + sb);
        a.n_scta = (int)sn;
#ifdef KLAY_STREAM_TRACE
        const bool trace = g_trace_layer == l + 1 && g_trace_dir == 0;
        if (trace) a.trace = stream_trace_buf();
#endif
        g_launches += launch_forward_stream(sr, d.prod, redo, a, s);
#ifdef KLAY_STREAM_TRACE
        if (trace) stream_trace_dump(a.trace, (int)sn * (int)((V + 255) / 256), l + 1, 0);
#endif
      } else {
        g_launches += launch_forward_layer(sr, d.prod, redo, a, s);
      }
    }
    prev = cur;
  }
  if (tail && !launch_on(KLAY_CLASS_TAIL)) {
    delete tail;
    tail = nullptr;
  }
  if (tail) {
    const LayerDesc& d0 = p->layers[tail_from];
    const LayerDesc& dl = p->layers[micro_from - 1];
    tail->pf_ptr[0] = p->d_src + d0.e_base;
    tail->pf_bytes[0] = (dl.e_base + dl.E - d0.e_base) * (long long)sizeof(int);
    tail->pf_ptr[1] = p->d_off + d0.off_base;
    tail->pf_bytes[1] = (dl.off_base + dl.W + 1 - d0.off_base) * (long long)sizeof(int);
    tail->pf_ptr[2] = p->d_items + d0.fi_base;
    tail->pf_bytes[2] = (dl.bi_base - d0.fi_base) * (long long)sizeof(int4);
    tail->pf_ptr[3] = p->d_masks + d0.fi_base;
    tail->pf_bytes[3] = (dl.bi_base - d0.fi_base) * (long long)sizeof(unsigned);
    LaunchScope ls(s, 4, tail_from + 1);
    auto tail_launch = [&](int cluster) {
      if constexpr (U1) return launch_forward_tail_u1(*tail, cluster, s);
      else return launch_forward_tail(sr, *tail, cluster, s);
    };
    int n = tail_launch(TAIL_CLUSTER);
    if (n == 0 && TAIL_CLUSTER > 8) {  // non-portable cluster size refused: portable size
      cudaGetLastError();
      n = tail_launch(8);
    }
    delete tail;
    if (n == 0) return fail(KLAY_ECUDA, std::string("tail launch failed: ") +
                                            cudaGetErrorString(cudaGetLastError()));
    g_launches += n;
    if (g_tail_trace) tail_trace_dump("forward", micro_from - tail_from);
  }
  if (micro.n > 0) {
    const int rc = run_micro(micro, micro_from);
    if (rc != KLAY_OK) return rc;
  }
  if (outputs && p->R > 0 && launch_on(KLAY_CLASS_BOUNDARY)) {
    LaunchScope ls(s, 2, p->L + 1);
    if constexpr (U1) {
      launch_unpack_outputs(prev, p->d_root_node, p->d_const, outputs, wdt == KLAY_F64, p->R, B, ld, s);
    } else {
      const T zero = (sr == SR_LOG_) ? T(-INFINITY) : T(0);
      const T one = (sr == SR_LOG_) ? T(0) : T(1);
      launch_assemble_outputs<T>(prev, p->d_root_node, p->d_const, (T*)outputs, p->R, B, ld, zero,
                                 one, s);
    }
    ++g_launches;
  }
  KLAY_CUDA(cudaGetLastError());
#ifdef KLAY_CHECKS
  return chk_finish(s, "klay_forward");
#else
  return KLAY_OK;
#endif
}

template <typename T>
int backward_impl(const KlayPlan* p, int domain, const T* trace, int64_t ld, const T* seed,
                  T* grads, T* work, int64_t B, double epsilon, int retain_mode, cudaStream_t s) {
  const int V = (int)(ld * (int64_t)sizeof(T) / 16);
  // adjoints: one row per node, laid out like the trace (routes write rows
  // of layers further down than the next)
  T* gtrace = work;
  T* scratch = work + (size_t)p->adj_rows * ld;
#ifdef KLAY_CHECKS
  const ChkRanges chk = chk_ranges(trace, (size_t)p->total_rows * ld * sizeof(T), work,
                                   ((size_t)p->adj_rows + p->max_bslots) * ld * sizeof(T) +
                                       counter_bytes(p, sizeof(T) == 8 ? KLAY_F64 : KLAY_F32, ld));
#endif
  int* hcount = reinterpret_cast<int*>(scratch + (size_t)p->max_bslots * ld);
  if (p->max_heavy > 0) {
    const size_t nb = counter_bytes(p, sizeof(T) == 8 ? KLAY_F64 : KLAY_F32, ld);
    KLAY_CUDA(cudaMemsetAsync(hcount, 0, nb, s));
  }
  if (launch_on(KLAY_CLASS_BOUNDARY)) {
    LaunchScope ls(s, 3, p->L + 1);
    launch_seed<T>(seed, p->d_top_off, p->d_top_pos, gtrace + (size_t)p->gbase[p->L] * ld,
                   (int)p->WL, p->R, B, ld, s);
    ++g_launches;
  }
  // alias outputs need the finiteness masks of a backward-only trace
  const bool alias = domain == SR_LOG_ && epsilon == 0.0 && retain_mode == 2 && !g_no_alias;
  const int32_t tail_from = g_no_tail ? p->L : p->tail_from;
  // the backward micro tail covers the log semiring (pass / log-sum layers)
  const int32_t microb_from = (g_no_tail || g_no_micro || !micro_fits(V)) ? p->L
                               : (domain == SR_LOG_ ? p->microb_from : p->microb_from_real);
  const int32_t head_b = (g_no_tail || g_no_micro || g_no_head || !micro_fits(V)) ? 0
                          : (domain == SR_LOG_ ? p->head_b : p->head_b_real);
  MicroBwdArgs<T> mb{}, mh{};
  TailArgs<T>* tail = nullptr;
  if (tail_from < microb_from) {
    tail = new TailArgs<T>();
    tail->n = 0;
    tail->debug_skip = g_tail_debug ? 1 : 0;
    tail->trace_ts = g_tail_trace ? tail_trace_buf() : nullptr;
  }
  for (int32_t l = p->L - 1; l >= 0; --l) {
    const LayerDesc& d = p->layers[l];
    LayerArgs<T> a = layer_args<T>(p, d, false, V, ld);
#ifdef KLAY_CHECKS
    a.chk = chk;
    a.chk.tag = -(l + 1);
#endif
    a.out = gtrace + (size_t)p->gbase[l] * ld;
    a.gcur = gtrace + (size_t)p->gbase[l + 1] * ld;
    a.ncur = trace + (size_t)d.row * ld;
    a.nprev = trace + (size_t)d.prev_row * ld;
    a.scratch = scratch;
    a.unary_ok = (domain == SR_LOG_ && epsilon == 0.0) ? 1 : 0;
    a.rev = chunk_rev(l + 1);
    a.hcount = (l >= tail_from) ? nullptr : hcount;
    MicroBwdArgs<T>* cm = (l >= microb_from) ? &mb : (l < head_b ? &mh : nullptr);
    if (cm) {
      // micro tail (top) or micro head (bottom); the lowest layer of each is
      // the one whose adjoints are read afterwards
      const int32_t lowest = (cm == &mb) ? microb_from : 0;
      MicroBwdArgs<T>& m = *cm;
      const int i = m.n++;
      if (i == 0) {
        m.gin = a.gcur;
        m.w_top = (int)d.W;
      }
      m.gout[i] = (l == lowest) ? a.out : nullptr;
      m.vpar[i] = a.ncur;
      m.vchild[i] = a.nprev;
      m.wp[i] = (int)d.W;
      m.wc[i] = (int)d.Wprev;
      m.csr_at[i] = p->microb_at[l];
      m.csr_n[i] = (domain == SR_LOG_ ? p->microb_n : p->microbr_n)[l];
      // weighted layers: log sums (softmax weights), real products (zero-safe)
      m.logsum[i] = (domain == SR_LOG_) ? (d.prod ? 0 : 1) : (d.prod ? 1 : 0);
      if (l == lowest && launch_on(KLAY_CLASS_BWD_MICRO)) {
#ifdef KLAY_CHECKS
        m.chk = chk;
        m.chk.tag = -(1000 + l);
#endif
        m.csr = p->d_microb;
        m.V = V;
        m.ld = ld;
        m.unary_ok = a.unary_ok;
        LaunchScope ls(s, 7, l + 1);
        const int n = launch_backward_micro(domain, m, s);
        if (n == 0) {
          delete tail;
          return fail(KLAY_ECUDA, std::string("micro-tail launch failed: ") +
                                      cudaGetErrorString(cudaGetLastError()));
        }
        g_launches += n;
      }
    } else if (l >= tail_from) {
      tail->layer[tail->n++] = a;
      if (l == tail_from && !launch_on(KLAY_CLASS_TAIL)) {
        delete tail;
        tail = nullptr;
      } else if (l == tail_from) {
        const LayerDesc& d0 = p->layers[tail_from];
        const LayerDesc& dl = p->layers[microb_from - 1];
        tail->pf_ptr[0] = p->d_tpar + d0.e_base;
        tail->pf_bytes[0] = (dl.e_base + dl.E - d0.e_base) * (long long)sizeof(int);
        tail->pf_ptr[1] = p->d_toff + d0.toff_base;
        tail->pf_bytes[1] = (dl.toff_base + dl.Wprev + 1 - d0.toff_base) * (long long)sizeof(int);
        tail->pf_ptr[2] = p->d_items + d0.bi_base;
        tail->pf_bytes[2] = (dl.bi_base + dl.bi_n - d0.bi_base) * (long long)sizeof(int4);
        tail->pf_ptr[3] = p->d_masks + d0.bi_base;
        tail->pf_bytes[3] = (dl.bi_base + dl.bi_n - d0.bi_base) * (long long)sizeof(unsigned);
        LaunchScope ls(s, 5, tail_from + 1);
        int n = launch_backward_tail(domain, *tail, TAIL_CLUSTER, s);
        if (n == 0 && TAIL_CLUSTER > 8) {
          cudaGetLastError();
          n = launch_backward_tail(domain, *tail, 8, s);
        }
        delete tail;
        tail = nullptr;
        if (n == 0) return fail(KLAY_ECUDA, std::string("tail launch failed: ") +
                                                cudaGetErrorString(cudaGetLastError()));
        g_launches += n;
        if (g_tail_trace) tail_trace_dump("backward", microb_from - tail_from);
      }
    } else {
      int mode = BW_PASS_;
      if (domain == SR_REAL_ && d.prod) mode = BW_REALPROD_;
      else if (domain == SR_LOG_ && !d.prod) mode = d.bsum8 ? BW_LOGSUM8_ : BW_LOGSUM_;
      if (alias && d.ba_on) {
        // children whose adjoint is not routed; absolute output rows (route
        // tops write their chain's bottom) and value rows
        set_items(a, p, d.ba);
        a.off = p->d_aoff + d.ba.off_base;
        a.idx = p->d_aidx + d.ba.e_base;
        a.omap = p->d_omap + d.ba.map_base;
        a.xmap = p->d_omap + d.ba.xmap_base;
        a.out = gtrace;
        a.nprev = trace;
        if (d.bmask) mode = BW_PASSA_;
      }
      const int cls = (mode == BW_PASS_ || mode == BW_PASSA_) ? KLAY_CLASS_BWD_PASS
                      : (mode == BW_REALPROD_ ? KLAY_CLASS_BWD_REALPROD : KLAY_CLASS_BWD_LOGSUM);
      if (launch_on(cls)) {
        LaunchScope ls(s, 1, l + 1);
        const bool aset = alias && d.ba_on;
        const int64_t sb = aset ? d.bsa_b : d.bs_b, sn = aset ? d.bsa_n : d.bs_n;
        if (sn > 0 && !g_no_stream) {
          a.scta = reinterpret_cast<const int*>(p->d_scta + sb);
          a.n_scta = (int)sn;
#ifdef KLAY_STREAM_TRACE
          const bool trace = g_trace_layer == l + 1 && g_trace_dir == 1;
          if (trace) a.trace = stream_trace_buf();
#endif
          g_launches += launch_backward_stream(mode, a, s);
#ifdef KLAY_STREAM_TRACE
          if (trace) stream_trace_dump(a.trace, (int)sn * (int)((V + 255) / 256), l + 1, 1);
#endif
        } else {
          g_launches += launch_backward_layer(mode, a, s);
        }
      }
    }
  }
  if (p->K > 0 && launch_on(KLAY_CLASS_BOUNDARY)) {
    LaunchScope ls(s, 3, 0);
    launch_store_rows<T>(gtrace + (size_t)p->gbase[0] * ld, grads, (int)p->K, B, ld, s);
    ++g_launches;
  }
  KLAY_CUDA(cudaGetLastError());
#ifdef KLAY_CHECKS
  return chk_finish(s, "klay_backward");
#else
  return KLAY_OK;
#endif
}

int check_common(const KlayPlan* plan, int32_t dtype, int64_t batch, int64_t ld) {
  if (!plan) return fail(KLAY_EINVAL, "plan is NULL");
  if (dtype != KLAY_F32 && dtype != KLAY_F64 && dtype != KLAY_U1) return fail(KLAY_EINVAL, "unknown dtype");
  if (batch < 1) return fail(KLAY_EINVAL, "batch must be >= 1");
  if (ld < klay_row_stride(batch, dtype) || (ld * (int64_t)esize(dtype)) % 16)
    return fail(KLAY_EINVAL, "row stride too small or not a multiple of 16 bytes");
  return KLAY_OK;
}

}  // namespace

extern "C" int klay_forward(const KlayPlan* plan, int32_t semiring, int32_t dtype,
                            const void* weights, int32_t weights_dtype, void* values, int64_t ld,
                            int32_t retain, void* outputs, int64_t batch, double epsilon,
                            void* workspace, void* stream) {
  if (int rc = check_common(plan, dtype, batch, ld)) return rc;
  if (semiring < KLAY_REAL || semiring > KLAY_MAXPROD) return fail(KLAY_EINVAL, "unknown semiring");
  if (retain < 0 || retain > 2) return fail(KLAY_EINVAL, "retain must be 0, 1 or 2");
  if (weights_dtype != KLAY_F32 && weights_dtype != KLAY_F64) return fail(KLAY_EINVAL, "unknown weights dtype");
  if (semiring == KLAY_LOG && !(epsilon >= 0)) return fail(KLAY_EINVAL, "epsilon must be >= 0");
  if (!values || (plan->K > 0 && !weights)) return fail(KLAY_EINVAL, "NULL buffer");
  if (plan->max_fslots > 0 && !workspace) return fail(KLAY_EINVAL, "workspace required (klay_forward_workspace)");
  if ((reinterpret_cast<uintptr_t>(values) & 15) != 0 || (reinterpret_cast<uintptr_t>(workspace) & 15) != 0)
    return fail(KLAY_EINVAL, "buffers must be 16-byte aligned");
  DeviceGuard guard(plan->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == KLAY_U1) {
    if (semiring != KLAY_BOOL) return fail(KLAY_EUNSUPPORTED, "bit-packed rows support the Boolean semiring only");
    return forward_impl<unsigned>(plan, semiring, weights, weights_dtype, (unsigned*)values, ld,
                                  retain != 0, outputs, batch, 0.0, (unsigned*)workspace, s);
  }
  if (dtype == KLAY_F32)
    return forward_impl<float>(plan, semiring, weights, weights_dtype, (float*)values, ld, retain,
                               outputs, batch, epsilon, (float*)workspace, s);
  return forward_impl<double>(plan, semiring, weights, weights_dtype, (double*)values, ld, retain,
                              outputs, batch, epsilon, (double*)workspace, s);
}

extern "C" int klay_backward(const KlayPlan* plan, int32_t domain, int32_t dtype, const void* trace,
                             int64_t ld, const void* seed, void* grads, void* workspace, int64_t batch,
                             double epsilon, int32_t retain, void* stream) {
  if (int rc = check_common(plan, dtype, batch, ld)) return rc;
  if (dtype == KLAY_U1) return fail(KLAY_EUNSUPPORTED, "no backward for bit-packed Boolean rows");
  if (domain != KLAY_REAL && domain != KLAY_LOG)
    return fail(KLAY_EUNSUPPORTED, "backward is defined for the real and log domains only");
  if (!trace || !workspace || (plan->K > 0 && !grads)) return fail(KLAY_EINVAL, "NULL buffer");
  if ((reinterpret_cast<uintptr_t>(trace) & 15) != 0 || (reinterpret_cast<uintptr_t>(workspace) & 15) != 0)
    return fail(KLAY_EINVAL, "buffers must be 16-byte aligned");
  DeviceGuard guard(plan->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == KLAY_F32)
    return backward_impl<float>(plan, domain, (const float*)trace, ld, (const float*)seed, (float*)grads,
                                (float*)workspace, batch, epsilon, retain, s);
  return backward_impl<double>(plan, domain, (const double*)trace, ld, (const double*)seed,
                               (double*)grads, (double*)workspace, batch, epsilon, retain, s);
}

extern "C" int klay_fill_trace(const KlayPlan* plan, int32_t semiring, int32_t dtype, void* values,
                               int64_t ld, int64_t batch, double epsilon, void* stream) {
  if (int rc = check_common(plan, dtype, batch, ld)) return rc;
  if (!values) return fail(KLAY_EINVAL, "NULL buffer");
  // only log-semiring, epsilon-0 traces leave rows out (forward_impl)
  if (semiring != KLAY_LOG || epsilon != 0.0 || dtype == KLAY_U1 || g_no_alias || plan->n_alias == 0)
    return KLAY_OK;
  DeviceGuard guard(plan->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == KLAY_F32) launch_fill_aliases<float>(plan->d_alias, plan->n_alias, (float*)values, ld, s);
  else launch_fill_aliases<double>(plan->d_alias, plan->n_alias, (double*)values, ld, s);
  ++g_launches;
  KLAY_CUDA(cudaGetLastError());
  return KLAY_OK;
}

extern "C" int64_t klay_launch_count(void) { return g_launches.load(); }

extern "C" uint32_t klay_set_launch_filter(uint32_t class_mask) {
  const uint32_t prev = g_launch_filter;
  g_launch_filter = class_mask;
  return prev;
}

extern "C" int klay_profiler_begin(void) {
  for (auto& r : g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  g_prof_on = true;
  return KLAY_OK;
}

extern "C" int klay_profiler_end(int32_t max_records, int32_t* kinds, int32_t* layers, float* ms,
                                 int32_t* n_records) {
  g_prof_on = false;
  int rc = KLAY_OK;
  int32_t n = 0;
  for (auto& r : g_prof) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
      rc = fail(KLAY_ECUDA, "profiler event timing failed");
    if (n < max_records) {
      if (kinds) kinds[n] = r.kind;
      if (layers) layers[n] = r.layer;
      if (ms) ms[n] = t;
    }
    ++n;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  if (n_records) *n_records = n;
  return rc;
}
