// Microbenchmark: a streaming gather-reduce of one real layer (config C,
// tools/microbench/dump_layer.py) with whole-row bulk copies: one producer
// warp streams every edge's operand row (B x 4 bytes, one cp.async.bulk per
// edge) into a shared-memory ring; 8 consumer warps (one 16-byte column piece
// per thread) reduce node by node and store each result row. Compared with
// the per-warp staged LDGSTS pattern (staged) of the round-1 library.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o stream_gather stream_gather.cu
//   ./stream_gather layer.bin
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sa(s)),
               "l"(g), "r"(bytes), "r"(sa(b))
               : "memory");
}

// one CTA: nodes [cn[c], cn[c+1]); ring of R row slots in groups of G (one
// full / empty mbarrier pair per group); PV = 16-byte pieces per row =
// consumer threads
template <int PV, int G>
__global__ void __launch_bounds__(PV + 32) stream(const float4* __restrict__ prev, float4* __restrict__ cur,
                                                  const int* __restrict__ off, const int* __restrict__ src,
                                                  const int* __restrict__ cn, int R) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int NG = R / G;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* empty = full + NG;
  float4* ring = reinterpret_cast<float4*>(smem + ((2 * NG * 8 + 127) / 128) * 128);
  constexpr unsigned ROWB = PV * 16;
  constexpr int CW = PV / 32;  // consumer warps
  const int n0 = cn[blockIdx.x], n1 = cn[blockIdx.x + 1];
  const int e0 = off[n0], e1 = off[n1];
  const int tid = threadIdx.x;
  if (tid < NG) {
    mbar_init(&full[tid], 1);
    mbar_init(&empty[tid], CW);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (tid >= PV) {
    // producer warp: one group of G edges per round, G lanes issue its copies
    const int lane = tid - PV;
    const int NGR = R / G;
    for (int gi = 0, base = e0; base < e1; ++gi, base += G) {
      const int grp = gi % NGR, lap = gi / NGR;
      const int cnt = min(G, e1 - base);
      const int row = (lane < cnt) ? src[base + lane] : 0;
      if (lane == 0) {
        mbar_wait(&empty[grp], (lap & 1) ^ 1);
        mbar_expect(&full[grp], cnt * ROWB);
      }
      __syncwarp();
      if (lane < cnt) bulk_g2s(ring + (size_t)(grp * G + lane) * PV, prev + (size_t)row * PV, ROWB, &full[grp]);
    }
    return;
  }
  const int lane = tid & 31;
  // incremental ring position: slot within the group, group, lap parity
  int gs = 0, grp = 0, par = 0;
  const int NGR = R / G;
  if (e0 < e1) mbar_wait(&full[0], 0);
  int e = e0;
  for (int n = n0; n < n1; ++n) {
    const int ee = off[n + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (; e < ee; ++e) {
      const float4 x = ring[(size_t)(grp * G + gs) * PV + tid];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      if (++gs == G) {
        gs = 0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[grp]);
        if (++grp == NGR) {
          grp = 0;
          par ^= 1;
        }
        if (e + 1 < e1) mbar_wait(&full[grp], par);
      }
    }
    cur[(size_t)n * PV + tid] = acc;
  }
  if (gs != 0) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[grp]);
  }
}

__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa(s)), "l"(g) : "memory");
}
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

// The same per-warp staged pattern, but each batch's row chunks are moved by
// lane-parallel bulk copies (lane i: edge i's 512-byte chunk) completing on
// a per-stage mbarrier, instead of 32 lanes x 16-byte LDGSTS per edge.
__global__ void staged_bulk(const float4* __restrict__ prev, float4* __restrict__ cur, const int* __restrict__ off,
                            const int* __restrict__ src, const int2* __restrict__ tasks, int ntask, int V) {
  extern __shared__ float4 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float4* st = sm + warp * 2 * 8 * 32;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + nw * 2 * 8 * 32) + 2 * warp;
  const int t = blockIdx.x * nw + warp;
  if (t >= ntask) return;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
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
  unsigned ph = 0;
  auto issue = [&](int b) {
    const int e0 = off[nb_[b]], e1 = off[nb_[b + 1]];
    __syncwarp();  // every lane is done with this stage
    if (lane == 0) mbar_expect(&bar[b & 1], (unsigned)(e1 - e0) * 512u);
    __syncwarp();
    if (lane < e1 - e0)
      bulk_g2s(st + (b & 1) * 256 + lane * 32, prev + (size_t)src[e0 + lane] * V + blockIdx.y * 32, 512u, &bar[b & 1]);
  };
  issue(0);
  for (int b = 0; b < nbat; ++b) {
    if (b + 1 < nbat) issue(b + 1);
    mbar_wait(&bar[b & 1], (ph >> (b & 1)) & 1u);
    ph ^= 1u << (b & 1);
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

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "layer.bin", "rb");
  if (!f) return 1;
  int hdr[3];
  if (fread(hdr, 4, 3, f) != 3) return 1;
  const int Wp = hdr[0], W = hdr[1], E = hdr[2];
  std::vector<int> off(W + 1), src(E);
  if (fread(off.data(), 4, W + 1, f) != (size_t)W + 1 || fread(src.data(), 4, E, f) != (size_t)E) return 1;
  fclose(f);
  constexpr int PV = 256;  // 4 KB rows (B = 1024 fp32)
  float4 *prev, *cur;
  CK(cudaMalloc(&prev, (size_t)Wp * PV * 16));
  CK(cudaMalloc(&cur, (size_t)W * PV * 16));
  CK(cudaMemset(prev, 0, (size_t)Wp * PV * 16));
  int *doff, *dsrc;
  CK(cudaMalloc(&doff, off.size() * 4));
  CK(cudaMalloc(&dsrc, src.size() * 4));
  CK(cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsrc, src.data(), src.size() * 4, cudaMemcpyHostToDevice));
  std::vector<char> used(Wp, 0);
  for (int s : src) used[s] = 1;
  long long distinct = 0;
  for (char u : used) distinct += u;
  const double nec = ((double)distinct + W) * PV * 16;
  printf("layer Wp %d W %d E %d distinct %lld (E/distinct %.2f)\n", Wp, W, E, distinct, (double)E / distinct);
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
    printf("  %-40s %8.1f us  %6.0f GB/s necessary\n", what, ms * 50, nec * 20 / (ms * 1e-3) / 1e9);
  };
  {
    std::vector<int2> tasks;
    for (int n = 0; n < W;) {
      if (off[n + 1] - off[n] > 8) { ++n; continue; }
      int m = n, edges = 0;
      while (m < W && m - n < 16 && off[m + 1] - off[m] <= 8 && edges + (off[m + 1] - off[m]) <= 32) {
        edges += off[m + 1] - off[m];
        ++m;
      }
      tasks.push_back(make_int2(n, m));
      n = m;
    }
    int2* dt;
    CK(cudaMalloc(&dt, tasks.size() * 8));
    CK(cudaMemcpy(dt, tasks.data(), tasks.size() * 8, cudaMemcpyHostToDevice));
    dim3 grid((unsigned)tasks.size(), PV / 32);
    size_t smem = 2 * 8 * 32 * 16;
    timeit([&] { staged<<<grid, 32, smem>>>(prev, cur, doff, dsrc, dt, (int)tasks.size(), PV); },
           "staged (short segments only)");
    CK(cudaFuncSetAttribute(staged_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 16));
    timeit([&] { staged_bulk<<<grid, 32, smem + 16>>>(prev, cur, doff, dsrc, dt, (int)tasks.size(), PV); },
           "staged, lane-parallel bulk copies");
    if (argc > 2 && atoi(argv[2]) < 0) return 0;  // (staged variants only)
  }
  int sms = 148;
  const int only = argc > 2 ? atoi(argv[2]) : 0;
  auto run = [&](auto G_, int per_sm, int ring_kb, int cmul) {
    constexpr int G = decltype(G_)::value;
    const int R = ring_kb * 1024 / (PV * 16) / G * G;
    if (R < 2 * G) return 0;
    const int nc = sms * per_sm * cmul;
    std::vector<int> cn(nc + 1, W);
    cn[0] = 0;
    const double tot = (double)E + W;
    int c = 1;
    for (int n = 0; n < W && c < nc; ++n)
      if (off[n] + n >= tot * c / nc) cn[c++] = n;
    int* dcn;
    CK(cudaMalloc(&dcn, cn.size() * 4));
    CK(cudaMemcpy(dcn, cn.data(), cn.size() * 4, cudaMemcpyHostToDevice));
    const size_t smem = 1024 + (size_t)R * PV * 16;
    CK(cudaFuncSetAttribute(stream<PV, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char name[96];
    snprintf(name, sizeof name, "stream %d/SM x%d ring %d KB (%d slots) G%d", per_sm, cmul, ring_kb, R, G);
    stream<PV, G><<<nc, PV + 32, smem>>>(prev, cur, doff, dsrc, dcn, R);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("  %s: %s\n", name, cudaGetErrorString(err));
      exit(1);
    }
    timeit([&] { stream<PV, G><<<nc, PV + 32, smem>>>(prev, cur, doff, dsrc, dcn, R); }, name);
    cudaFree(dcn);
    return 0;
  };
  for (int per_sm : {1, 2, 3})
    for (int ring_kb : {48, 64, 96, 200})
      for (int cmul : {1, 4}) {
        if (per_sm * (ring_kb + 2) > 226) continue;
        run(std::integral_constant<int, 4>{}, per_sm, ring_kb, cmul);
        run(std::integral_constant<int, 8>{}, per_sm, ring_kb, cmul);
        run(std::integral_constant<int, 16>{}, per_sm, ring_kb, cmul);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
