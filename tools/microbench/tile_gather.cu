// Microbenchmark: gather-reduce of one real layer (config C, dumped by
// tools/microbench/dump_layer.py) three ways, to decide the layer-kernel
// design:
//   staged   node-aligned 8-edge batches, per-lane 16-byte cp.async (LDGSTS),
//            double-buffered per warp (the round-1 library pattern)
//   tile_ld  node tiles whose DISTINCT operand rows (first-use order) are
//            staged once per tile with per-lane cp.async, then reduced from
//            shared memory (dedup: a row shared by the tile's nodes is read once)
//   tile_tma the same tiles, rows moved by cp.async.bulk (one bulk copy per
//            row chunk, UBLKCP) completing on per-batch mbarriers; warps start
//            on a node as soon as the batch holding its last operand landed
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tile_gather tile_gather.cu
//   ./tile_gather layer.bin
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <unordered_map>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));        \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g) : "memory");
}

// ---------------------------------------------------------------- staged
__global__ void staged(const float4* __restrict__ prev, float4* __restrict__ cur, const int* __restrict__ off,
                       const int* __restrict__ src, const int2* __restrict__ tasks, int ntask, int V) {
  extern __shared__ float4 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* st = sm + warp * 2 * 8 * 32;
  const int t = blockIdx.x * (blockDim.x / 32) + warp;
  if (t >= ntask) return;
  const int2 tk = tasks[t];
  const int v = blockIdx.y * 32 + lane;
  int nb_[33], nbat = 0;
  {
    int n = tk.x;
    while (n < tk.y) {
      nb_[nbat++] = n;
      const int lim = off[n] + 8;
      int m = n + 1;
      while (m < tk.y && off[m + 1] <= lim) ++m;
      n = m;
    }
    nb_[nbat] = tk.y;
  }
  auto issue = [&](int b) {
    const int e0 = off[nb_[b]], e1 = off[nb_[b + 1]];
    for (int e = e0; e < e1; ++e) cp16(st + (b & 1) * 256 + (e - e0) * 32 + lane, prev + (size_t)src[e] * V + v);
    asm volatile("cp.async.commit_group;\n");
  };
  issue(0);
  for (int b = 0; b < nbat; ++b) {
    if (b + 1 < nbat) {
      issue(b + 1);
      asm volatile("cp.async.wait_group 1;\n");
    } else
      asm volatile("cp.async.wait_group 0;\n");
    const int e0 = off[nb_[b]];
    for (int n = nb_[b]; n < nb_[b + 1]; ++n) {
      float4 acc = make_float4(0, 0, 0, 0);
      for (int e = off[n]; e < off[n + 1]; ++e) {
        float4 x = st[(b & 1) * 256 + (e - e0) * 32 + lane];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      cur[(size_t)n * V + v] = acc;
    }
  }
}

// ---------------------------------------------------------------- tiles
// tile t: nodes [tn[t], tn[t+1]), rows [tr[t], tr[t+1]) of trow (distinct
// operand rows, first-use order), edges of its nodes in off/slot (slot =
// position of the edge's row within the tile's row list)
struct Tiles {
  const int* tn;
  const int* tr;
  const int* trow;
  const int* off;
  const unsigned short* slot;
  const unsigned char* need;  // per node: batch (of RB rows) holding its last operand
  const int* nodes;           // node ids in tile order (tile t: nodes[tn[t] .. tn[t+1]))
};

// P pieces (16 B) per lane: a CTA column chunk is P * 512 bytes
template <int P>
__global__ void tile_ld(const float4* __restrict__ prev, float4* __restrict__ cur, Tiles T, int V) {
  extern __shared__ float4 sm[];
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n0 = T.tn[t], n1 = T.tn[t + 1], r0 = T.tr[t], nr = T.tr[t + 1] - r0;
  const int v0 = blockIdx.y * 32 * P;
  for (int r = warp; r < nr; r += nw) {
    const float4* g = prev + (size_t)T.trow[r0 + r] * V + v0;
#pragma unroll
    for (int q = 0; q < P; ++q) cp16(sm + (size_t)r * 32 * P + q * 32 + lane, g + q * 32 + lane);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int k = n0 + warp; k < n1; k += nw) {
    const int n = T.nodes[k];
    const int e0 = T.off[n], e1 = T.off[n + 1];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      float4 acc = make_float4(0, 0, 0, 0);
      for (int e = e0; e < e1; ++e) {
        const float4 x = sm[(size_t)T.slot[e] * 32 * P + q * 32 + lane];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      cur[(size_t)n * V + v0 + q * 32 + lane] = acc;
    }
  }
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes, unsigned long long* b) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  unsigned ba = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sa),
               "l"(g), "r"(bytes), "r"(ba)
               : "memory");
}

constexpr int RB = 32;  // rows per mbarrier batch

template <int P>
__global__ void tile_tma(const float4* __restrict__ prev, float4* __restrict__ cur, Tiles T, int V) {
  extern __shared__ __align__(128) float4 sm[];
  __shared__ unsigned long long bar[16];
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n0 = T.tn[t], n1 = T.tn[t + 1], r0 = T.tr[t], nr = T.tr[t + 1] - r0;
  const int nb = (nr + RB - 1) / RB;
  const int v0 = blockIdx.y * 32 * P;
  constexpr unsigned CH = 512 * P;
  if (threadIdx.x < nb) mbar_init(&bar[threadIdx.x], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    for (int b = 0; b < nb; ++b) {
      const int rb = b * RB, cnt = min(RB, nr - rb);
      if (lane == 0) mbar_expect(&bar[b], cnt * CH);
      __syncwarp();
      if (lane < cnt)
        bulk_g2s(sm + (size_t)(rb + lane) * 32 * P, prev + (size_t)T.trow[r0 + rb + lane] * V + v0, CH, &bar[b]);
    }
  }
  int ready = -1;
  for (int k = n0 + warp; k < n1; k += nw) {
    const int n = T.nodes[k];
    const int need = T.need[n];
    while (ready < need) mbar_wait(&bar[++ready], 0);
    const int e0 = T.off[n], e1 = T.off[n + 1];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      float4 acc = make_float4(0, 0, 0, 0);
      for (int e = e0; e < e1; ++e) {
        const float4 x = sm[(size_t)T.slot[e] * 32 * P + q * 32 + lane];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      cur[(size_t)n * V + v0 + q * 32 + lane] = acc;
    }
  }
  // (no CTA exit while bulk copies may still be in flight: every batch waited)
  while (ready < nb - 1) mbar_wait(&bar[++ready], 0);
}

struct HostTiles {
  std::vector<int> tn, tr, trow;
  std::vector<unsigned short> slot;
  std::vector<unsigned char> need;
  std::vector<int> nodes;
};

HostTiles make_tiles(const std::vector<int>& off, const std::vector<int>& src, int W, int dmax, int nmax,
                     const std::vector<int>& order) {
  HostTiles h;
  h.nodes = order;
  h.slot.resize(src.size());
  h.need.resize(W);
  h.tn.push_back(0);
  h.tr.push_back(0);
  std::unordered_map<int, int> pos;
  int n = 0;
  while (n < W) {
    pos.clear();
    int start = n, base = (int)h.trow.size();
    while (n < W && n - start < nmax) {
      const int nd = order[n];
      int add = 0;
      for (int e = off[nd]; e < off[nd + 1]; ++e)
        if (!pos.count(src[e])) ++add;  // (duplicates within a node: counted twice, harmless bound)
      if (n > start && (int)pos.size() + add > dmax) break;
      int mx = 0;
      for (int e = off[nd]; e < off[nd + 1]; ++e) {
        auto it = pos.find(src[e]);
        int s;
        if (it == pos.end()) {
          s = (int)pos.size();
          pos[src[e]] = s;
          h.trow.push_back(src[e]);
        } else {
          s = it->second;
        }
        h.slot[e] = (unsigned short)s;
        mx = std::max(mx, s);
      }
      h.need[nd] = (unsigned char)(mx / RB);
      ++n;
    }
    h.tn.push_back(n);
    h.tr.push_back((int)h.trow.size());
    (void)base;
  }
  return h;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "layer.bin", "rb");
  if (!f) {
    printf("no layer file\n");
    return 1;
  }
  int hdr[3];
  if (fread(hdr, 4, 3, f) != 3) return 1;
  const int Wp = hdr[0], W = hdr[1], E = hdr[2];
  std::vector<int> off(W + 1), src(E);
  if (fread(off.data(), 4, W + 1, f) != (size_t)W + 1 || fread(src.data(), 4, E, f) != (size_t)E) return 1;
  fclose(f);
  const int V = 256;  // 4 KB rows (B = 1024 fp32)
  float4 *prev, *cur;
  CK(cudaMalloc(&prev, (size_t)Wp * V * 16));
  CK(cudaMalloc(&cur, (size_t)W * V * 16));
  CK(cudaMemset(prev, 0, (size_t)Wp * V * 16));
  int *doff, *dsrc;
  CK(cudaMalloc(&doff, off.size() * 4));
  CK(cudaMalloc(&dsrc, src.size() * 4));
  CK(cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsrc, src.data(), src.size() * 4, cudaMemcpyHostToDevice));
  // distinct rows read by the layer (the necessary bytes)
  std::vector<char> used(Wp, 0);
  for (int s : src) used[s] = 1;
  long long distinct = 0;
  for (char u : used) distinct += u;
  const double nec = ((double)distinct + W) * V * 16;
  printf("layer Wp %d W %d E %d distinct rows %lld (E/distinct %.2f)\n", Wp, W, E, distinct, (double)E / distinct);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto launch, const char* what) {
    for (int r = 0; r < 3; ++r) launch();
    CK(cudaGetLastError());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 20; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("  %-34s %8.1f us  %6.0f GB/s necessary\n", what, ms * 50, nec * 20 / (ms * 1e-3) / 1e9);
  };
  {
    std::vector<int2> tasks;
    int skipped = 0;
    for (int n = 0; n < W;) {
      if (off[n + 1] - off[n] > 8) {  // (segments longer than a stage: not timed here)
        ++skipped;
        ++n;
        continue;
      }
      int m = n, edges = 0;
      while (m < W && m - n < 16 && off[m + 1] - off[m] <= 8 && edges + (off[m + 1] - off[m]) <= 32) {
        edges += off[m + 1] - off[m];
        ++m;
      }
      tasks.push_back(make_int2(n, m));
      n = m;
    }
    printf(" staged: %d segments > 8 edges skipped\n", skipped);
    int2* dt;
    CK(cudaMalloc(&dt, tasks.size() * 8));
    CK(cudaMemcpy(dt, tasks.data(), tasks.size() * 8, cudaMemcpyHostToDevice));
    for (int wpb : {1, 4}) {
      dim3 grid(((int)tasks.size() + wpb - 1) / wpb, V / 32);
      size_t smem = wpb * 2 * 8 * 32 * 16;
      CK(cudaFuncSetAttribute(staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      char name[64];
      snprintf(name, sizeof name, "staged wpb=%d", wpb);
      timeit([&] { staged<<<grid, wpb * 32, smem>>>(prev, cur, doff, dsrc, dt, (int)tasks.size(), V); }, name);
    }
  }
  std::vector<int> natural(W), bymin(W);
  for (int i = 0; i < W; ++i) natural[i] = bymin[i] = i;
  {
    std::vector<int> mn(W, 0);
    for (int i = 0; i < W; ++i)
      for (int e = off[i]; e < off[i + 1]; ++e) mn[i] = (e == off[i]) ? src[e] : std::min(mn[i], src[e]);
    std::stable_sort(bymin.begin(), bymin.end(), [&](int a, int b) { return mn[a] < mn[b]; });
  }
  for (int sorted = 0; sorted < 2; ++sorted)
  for (int dmax : {64, 96, 128}) {
    HostTiles h = make_tiles(off, src, W, dmax, 255 * RB, sorted ? bymin : natural);
    const int nt = (int)h.tn.size() - 1;
    int *tn, *tr, *trow;
    unsigned short* slot;
    unsigned char* need;
    int* nodes;
    CK(cudaMalloc(&nodes, h.nodes.size() * 4));
    CK(cudaMemcpy(nodes, h.nodes.data(), h.nodes.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&tn, h.tn.size() * 4));
    CK(cudaMalloc(&tr, h.tr.size() * 4));
    CK(cudaMalloc(&trow, std::max<size_t>(h.trow.size(), 1) * 4));
    CK(cudaMalloc(&slot, h.slot.size() * 2));
    CK(cudaMalloc(&need, h.need.size()));
    CK(cudaMemcpy(tn, h.tn.data(), h.tn.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(tr, h.tr.data(), h.tr.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(trow, h.trow.data(), h.trow.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(slot, h.slot.data(), h.slot.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(need, h.need.data(), h.need.size(), cudaMemcpyHostToDevice));
    Tiles T{tn, tr, trow, doff, slot, need, nodes};
    printf(" tiles %s dmax=%d: %d tiles, staged rows %zu (%.2f of E)\n", sorted ? "by-min-child" : "natural",
           dmax, nt, h.trow.size(), (double)h.trow.size() / E);
    auto run = [&](auto P_, int warps, bool tma) {
      constexpr int P = decltype(P_)::value;
      dim3 grid(nt, V / (32 * P));
      size_t smem = (size_t)dmax * 512 * P;
      if (smem > 227 * 1024) return;
      char name[64];
      snprintf(name, sizeof name, "%s P=%d warps=%d", tma ? "tile_tma" : "tile_ld", P, warps);
      if (tma) {
        CK(cudaFuncSetAttribute(tile_tma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        timeit([&] { tile_tma<P><<<grid, warps * 32, smem>>>(prev, cur, T, V); }, name);
      } else {
        CK(cudaFuncSetAttribute(tile_ld<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        timeit([&] { tile_ld<P><<<grid, warps * 32, smem>>>(prev, cur, T, V); }, name);
      }
    };
    for (int warps : {4, 8}) {
      run(std::integral_constant<int, 1>{}, warps, false);
      run(std::integral_constant<int, 1>{}, warps, true);
    }
    cudaFree(nodes);
    cudaFree(tn); cudaFree(tr); cudaFree(trow); cudaFree(slot); cudaFree(need);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
