// libklay C ABI: plan construction (host) and per-pass launch sequences.
// See include/klay.h for the contract and the reference mapping.
#include "klay.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"

using namespace klay;

namespace {

thread_local std::string g_err;

// Kernel launches issued by this library (all threads), for the benchmark's
// gpu_launches claim.
std::atomic<long long> g_launches{0};

// Optional per-launch event timing (klay_profiler_begin / _end).
struct ProfRec {
  int kind, layer;
  cudaEvent_t a, b;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRec> g_prof;

struct LaunchScope {
  cudaStream_t s;
  int kind, layer;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(cudaStream_t s_, int kind_, int layer_) : s(s_), kind(kind_), layer(layer_) {
    ++g_launches;
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
  }
};

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

struct LayerDesc {
  int64_t W, Wprev, E;
  bool prod;
  int64_t row, prev_row;  // row offsets into the trace buffer
  int64_t off_base;       // into off[] (W+1 entries per layer)
  int64_t e_base;         // into src[] / tpar[]
  int64_t toff_base;      // into toff[] (Wprev+1 entries per layer)
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
  int64_t max_width = 0;
  int64_t max_fanin = 0;
  std::vector<LayerDesc> layers;
  std::vector<int64_t> layer_row;  // L+1 entries
  int* d_off = nullptr;
  int* d_src = nullptr;
  int* d_toff = nullptr;
  int* d_tpar = nullptr;
  int* d_root_node = nullptr;
  signed char* d_const = nullptr;
  int* d_top_off = nullptr;
  int* d_top_pos = nullptr;
  int64_t WL = 0;  // width of the last layer (K when there are no gates)
};

extern "C" const char* klay_version(void) { return "libklay 0.1 sm_100a"; }

extern "C" const char* klay_last_error(void) { return g_err.c_str(); }

static void plan_free(KlayPlan* p) {
  if (!p) return;
  cudaFree(p->d_off);
  cudaFree(p->d_src);
  cudaFree(p->d_toff);
  cudaFree(p->d_tpar);
  cudaFree(p->d_root_node);
  cudaFree(p->d_const);
  cudaFree(p->d_top_off);
  cudaFree(p->d_top_pos);
  delete p;
}

template <typename T>
static int upload(T** dst, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(v.size(), 1) * sizeof(T);
  KLAY_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), bytes));
  if (!v.empty()) KLAY_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return KLAY_OK;
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

  KlayPlan* p = new KlayPlan();
  p->device = device;
  p->K = num_inputs;
  p->L = num_layers;
  p->R = num_roots;

  std::vector<int> off, src, toff, tpar;
  int64_t prev_w = num_inputs, row = num_inputs, e_base = 0;
  p->max_width = num_inputs;
  p->layer_row.push_back(0);
  for (int32_t l = 0; l < num_layers; ++l) {
    const int64_t W = widths[l], E = edge_counts[l];
    const int64_t* S = sources + e_base;
    const int64_t* G = segments + e_base;
    char where[64];
    snprintf(where, sizeof where, "layer %d: ", l + 1);
    // invariants of tensorize.py:105-125
    if (W <= 0) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "nonpositive width"); }
    if (E <= 0) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "no edges"); }
    if (W >= (1LL << 31) || E >= (1LL << 31) || prev_w >= (1LL << 31)) {
      plan_free(p);
      return fail(KLAY_EINVAL, std::string(where) + "layer exceeds int32 indexing");
    }
    LayerDesc d;
    d.W = W; d.Wprev = prev_w; d.E = E; d.prod = (l % 2 == 0);
    d.row = row; d.prev_row = row - prev_w;
    d.off_base = (int64_t)off.size();
    d.e_base = e_base;
    d.toff_base = (int64_t)toff.size();
    // CSR offsets of the parent segments (engine.py:144-146)
    std::vector<int64_t> cnt(W, 0), gcnt(prev_w, 0);
    for (int64_t e = 0; e < E; ++e) {
      if (e > 0 && G[e] < G[e - 1]) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "aggregation indices not nondecreasing"); }
      if (G[e] < 0 || G[e] >= W) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "aggregation indices must cover 0..width-1"); }
      if (S[e] < 0 || S[e] >= prev_w) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "edge index out of range"); }
      ++cnt[G[e]];
      ++gcnt[S[e]];
    }
    off.push_back(0);
    int64_t acc = 0;
    for (int64_t i = 0; i < W; ++i) {
      if (cnt[i] == 0) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "aggregation indices must cover 0..width-1"); }
      p->max_fanin = std::max(p->max_fanin, cnt[i]);
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
      if (gcnt[j] == 0) { plan_free(p); return fail(KLAY_EFORMAT, std::string(where) + "some previous-layer node is never read"); }
      pos[j] = acc;
      acc += gcnt[j];
      toff.push_back((int)acc);
    }
    const size_t tb = tpar.size();
    tpar.resize(tb + E);
    for (int64_t e = 0; e < E; ++e) tpar[tb + pos[S[e]]++] = (int)G[e];
    p->layers.push_back(d);
    p->layer_row.push_back(row);
    p->max_width = std::max(p->max_width, W);
    row += W;
    e_base += E;
    prev_w = W;
  }
  p->total_rows = row;
  p->WL = prev_w;

  // roots (engine.py:203-212, 330-334)
  std::vector<int> rn(num_roots);
  std::vector<signed char> cv(num_roots);
  std::vector<std::vector<int>> by_node(prev_w);
  for (int32_t q = 0; q < num_roots; ++q) {
    rn[q] = (int)root_nodes[q];
    cv[q] = const_vals[q] ? 1 : 0;
    if (root_nodes[q] >= prev_w || root_nodes[q] < -1) {
      plan_free(p);
      return fail(KLAY_EFORMAT, "root index outside final layer");
    }
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
      (rc = upload(&p->d_root_node, rn)) || (rc = upload(&p->d_const, cv)) ||
      (rc = upload(&p->d_top_off, top_off)) || (rc = upload(&p->d_top_pos, top_pos))) {
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
extern "C" int64_t klay_plan_layer_offset(const KlayPlan* p, int32_t l) {
  if (!p || l < 0 || l > p->L) return -1;
  return p->layer_row[l];
}

extern "C" int64_t klay_row_stride(int64_t batch, int32_t dtype) {
  const int64_t per16 = (dtype == KLAY_F64) ? 2 : 4;
  if (batch < 1) batch = 1;
  return (batch + per16 - 1) / per16 * per16;
}

namespace {

struct Launch {
  dim3 grid, block;
};

// threads -> (row, 16-byte vector); block of 256 = vx vectors x ny rows
Launch row_launch(int64_t rows, int V) {
  int vx = 1;
  while (vx < V && vx < 256) vx <<= 1;
  const int ny = 256 / vx;
  Launch L;
  L.block = dim3(vx, ny, 1);
  L.grid = dim3((unsigned)((rows + ny - 1) / ny), (unsigned)((V + vx - 1) / vx), 1);
  return L;
}

template <typename T, int SR>
void launch_fwd_layer(const FwdArgs<T>& a, bool prod, cudaStream_t s) {
  Launch L = row_launch(a.W, a.V);
  if (prod)
    fwd_layer_kernel<T, SR, true><<<L.grid, L.block, 0, s>>>(a);
  else
    fwd_layer_kernel<T, SR, false><<<L.grid, L.block, 0, s>>>(a);
}

template <typename T>
int forward_impl(const KlayPlan* p, int sr, const void* weights, int wdt, T* values, int64_t ld,
                 bool retain, T* outputs, int64_t B, double eps, cudaStream_t s) {
  const int V = (int)(ld * (int64_t)sizeof(T) / 16);
  T* pingpong[2] = {values, values + (size_t)p->max_width * ld};
  // inputs -> rows 0..K-1 (node-major), identity padding
  T pad = (sr == SR_LOG) ? T(0) : T(1);
  if (p->K > 0) {
    dim3 grid((unsigned)((ld + 31) / 32), (unsigned)((p->K + 31) / 32));
    dim3 block(32, 8);
    LaunchScope ls(s, 2, 0);
    if (wdt == KLAY_F64)
      load_inputs_kernel<T, double><<<grid, block, 0, s>>>((const double*)weights, values, (int)p->K, B, ld, pad);
    else
      load_inputs_kernel<T, float><<<grid, block, 0, s>>>((const float*)weights, values, (int)p->K, B, ld, pad);
  }
  const T* prev = values;
  for (int32_t l = 0; l < p->L; ++l) {
    const LayerDesc& d = p->layers[l];
    T* cur = retain ? values + (size_t)d.row * ld : pingpong[(l + 1) & 1];
    FwdArgs<T> a;
    a.prev = prev;
    a.cur = cur;
    a.off = p->d_off + d.off_base;
    a.src = p->d_src + d.e_base;
    a.W = (int)d.W;
    a.V = V;
    a.ld = ld;
    a.eps = (T)eps;
    LaunchScope ls(s, 0, l + 1);
    switch (sr) {
      case SR_REAL: launch_fwd_layer<T, SR_REAL>(a, d.prod, s); break;
      case SR_LOG: launch_fwd_layer<T, SR_LOG>(a, d.prod, s); break;
      case SR_BOOL: launch_fwd_layer<T, SR_BOOL>(a, d.prod, s); break;
      default: launch_fwd_layer<T, SR_MAXPROD>(a, d.prod, s); break;
    }
    prev = cur;
  }
  if (outputs && p->R > 0 && B > 0) {
    const T zero = (sr == SR_LOG) ? T(-INFINITY) : T(0);
    const T one = (sr == SR_LOG) ? T(0) : T(1);
    const int64_t n = B * p->R;
    LaunchScope ls(s, 2, p->L + 1);
    assemble_outputs_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        prev, p->d_root_node, p->d_const, outputs, p->R, B, ld, zero, one);
  }
  KLAY_CUDA(cudaGetLastError());
  return KLAY_OK;
}

template <typename T>
int backward_impl(const KlayPlan* p, int domain, const T* trace, int64_t ld, const T* seed,
                  T* grads, T* work, int64_t B, cudaStream_t s) {
  const int V = (int)(ld * (int64_t)sizeof(T) / 16);
  T* g[2] = {work, work + (size_t)p->max_width * ld};
  int cur = 0;
  {
    const int64_t n = p->WL * ld;
    LaunchScope ls(s, 3, p->L + 1);
    seed_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(seed, p->d_top_off, p->d_top_pos,
                                                               g[cur], (int)p->WL, p->R, B, ld);
  }
  for (int32_t l = p->L - 1; l >= 0; --l) {
    const LayerDesc& d = p->layers[l];
    BwdArgs<T> a;
    a.gcur = g[cur];
    a.gprev = g[cur ^ 1];
    a.ncur = trace + (size_t)d.row * ld;
    a.nprev = trace + (size_t)d.prev_row * ld;
    a.toff = p->d_toff + d.toff_base;
    a.tpar = p->d_tpar + d.e_base;
    a.off = p->d_off + d.off_base;
    a.src = p->d_src + d.e_base;
    a.Wprev = (int)d.Wprev;
    a.V = V;
    a.ld = ld;
    Launch L = row_launch(d.Wprev, V);
    LaunchScope ls(s, 1, l + 1);
    if (domain == SR_REAL && d.prod)
      bwd_layer_kernel<T, BW_REALPROD><<<L.grid, L.block, 0, s>>>(a);
    else if (domain == SR_LOG && !d.prod)
      bwd_layer_kernel<T, BW_LOGSUM><<<L.grid, L.block, 0, s>>>(a);
    else
      bwd_layer_kernel<T, BW_PASS><<<L.grid, L.block, 0, s>>>(a);
    cur ^= 1;
  }
  if (p->K > 0 && B > 0) {
    dim3 grid((unsigned)((B + 31) / 32), (unsigned)((p->K + 31) / 32));
    LaunchScope ls(s, 3, 0);
    store_rows_kernel<T><<<grid, dim3(32, 8), 0, s>>>(g[cur], grads, (int)p->K, B, ld);
  }
  KLAY_CUDA(cudaGetLastError());
  return KLAY_OK;
}

}  // namespace

extern "C" int klay_forward(const KlayPlan* plan, int32_t semiring, int32_t dtype,
                            const void* weights, int32_t weights_dtype, void* values, int64_t ld,
                            int32_t retain, void* outputs, int64_t batch, double epsilon,
                            void* stream) {
  if (!plan) return fail(KLAY_EINVAL, "plan is NULL");
  if (semiring < KLAY_REAL || semiring > KLAY_MAXPROD) return fail(KLAY_EINVAL, "unknown semiring");
  if (dtype != KLAY_F32 && dtype != KLAY_F64) return fail(KLAY_EINVAL, "unknown dtype");
  if (weights_dtype != KLAY_F32 && weights_dtype != KLAY_F64) return fail(KLAY_EINVAL, "unknown weights dtype");
  if (batch < 1) return fail(KLAY_EINVAL, "batch must be >= 1");
  if (ld < klay_row_stride(batch, dtype) || (ld * (dtype == KLAY_F64 ? 8 : 4)) % 16)
    return fail(KLAY_EINVAL, "row stride too small or not a multiple of 16 bytes");
  if (semiring == KLAY_LOG && !(epsilon >= 0)) return fail(KLAY_EINVAL, "epsilon must be >= 0");
  if (!values || (plan->K > 0 && !weights)) return fail(KLAY_EINVAL, "NULL buffer");
  if ((reinterpret_cast<uintptr_t>(values) & 15) != 0) return fail(KLAY_EINVAL, "values not 16-byte aligned");
  DeviceGuard guard(plan->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == KLAY_F32)
    return forward_impl<float>(plan, semiring, weights, weights_dtype, (float*)values, ld, retain != 0,
                               (float*)outputs, batch, epsilon, s);
  return forward_impl<double>(plan, semiring, weights, weights_dtype, (double*)values, ld, retain != 0,
                              (double*)outputs, batch, epsilon, s);
}

extern "C" size_t klay_backward_workspace(const KlayPlan* plan, int32_t dtype, int64_t ld) {
  if (!plan) return 0;
  return (size_t)2 * plan->max_width * ld * (dtype == KLAY_F64 ? 8 : 4);
}

extern "C" int klay_backward(const KlayPlan* plan, int32_t domain, int32_t dtype, const void* trace,
                             int64_t ld, const void* seed, void* grads, void* workspace, int64_t batch,
                             void* stream) {
  if (!plan) return fail(KLAY_EINVAL, "plan is NULL");
  if (domain != KLAY_REAL && domain != KLAY_LOG)
    return fail(KLAY_EUNSUPPORTED, "backward is defined for the real and log domains only");
  if (dtype != KLAY_F32 && dtype != KLAY_F64) return fail(KLAY_EINVAL, "unknown dtype");
  if (batch < 1) return fail(KLAY_EINVAL, "batch must be >= 1");
  if (ld < klay_row_stride(batch, dtype) || (ld * (dtype == KLAY_F64 ? 8 : 4)) % 16)
    return fail(KLAY_EINVAL, "row stride too small or not a multiple of 16 bytes");
  if (!trace || !workspace || (plan->K > 0 && !grads)) return fail(KLAY_EINVAL, "NULL buffer");
  DeviceGuard guard(plan->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == KLAY_F32)
    return backward_impl<float>(plan, domain, (const float*)trace, ld, (const float*)seed, (float*)grads,
                                (float*)workspace, batch, s);
  return backward_impl<double>(plan, domain, (const double*)trace, ld, (const double*)seed,
                               (double*)grads, (double*)workspace, batch, s);
}

extern "C" int64_t klay_launch_count(void) { return g_launches.load(); }

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
