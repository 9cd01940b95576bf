// Microbenchmark: the staged gather pattern on a real layer's structure
// (config C, dumped by tools/microbench/dump_layer.py): how fast can a plain
// node-aligned, double-buffered cp.async gather-sum go on these indices?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o real_gather real_gather.cu
//   ./real_gather layer.bin
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}

// tasks: [node_begin, node_end) with <= 32 edges / 16 nodes, segments <= 8
__global__ void staged(const float4* __restrict__ prev, float4* __restrict__ cur,
                       const int* __restrict__ off, const int* __restrict__ src,
                       const int2* __restrict__ tasks, int ntask, int V) {
  extern __shared__ float4 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* st = sm + warp * 2 * 8 * 32;
  const int t = blockIdx.x * (blockDim.x / 32) + warp;
  if (t >= ntask) return;
  const int2 tk = tasks[t];
  const int v = blockIdx.y * 32 + lane;
  // batches: node-aligned runs of <= 8 edges
  int nb_[17], nbat = 0;
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
    if (b + 1 < nbat) { issue(b + 1); asm volatile("cp.async.wait_group 1;\n"); }
    else asm volatile("cp.async.wait_group 0;\n");
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
  if (!f) { printf("no layer file\n"); return 1; }
  int hdr[3];
  fread(hdr, 4, 3, f);
  const int Wp = hdr[0], W = hdr[1], E = hdr[2];
  std::vector<int> off(W + 1), src(E);
  fread(off.data(), 4, W + 1, f);
  fread(src.data(), 4, E, f);
  fclose(f);
  std::vector<int2> tasks;
  int skipped = 0;
  for (int n = 0; n < W;) {
    if (off[n + 1] - off[n] > 8) { ++skipped; ++n; continue; }  // (long segments: not timed)
    int m = n, edges = 0;
    while (m < W && m - n < 16 && off[m + 1] - off[m] <= 8 && edges + (off[m + 1] - off[m]) <= 32) {
      edges += off[m + 1] - off[m];
      ++m;
    }
    tasks.push_back(make_int2(n, m));
    n = m;
  }
  printf("skipped %d long segments\n", skipped);
  const int V = 256;  // 4 KB rows (B = 1024 fp32)
  float4 *prev, *cur;
  int *doff, *dsrc;
  int2* dt;
  cudaMalloc(&prev, (size_t)Wp * V * 16);
  cudaMalloc(&cur, (size_t)W * V * 16);
  cudaMemset(prev, 0, (size_t)Wp * V * 16);
  cudaMalloc(&doff, off.size() * 4);
  cudaMalloc(&dsrc, src.size() * 4);
  cudaMalloc(&dt, tasks.size() * 8);
  cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dsrc, src.data(), src.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dt, tasks.data(), tasks.size() * 8, cudaMemcpyHostToDevice);
  const double alg = ((double)Wp + W) * V * 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wpb : {4}) {
    dim3 grid(((int)tasks.size() + wpb - 1) / wpb, V / 32);
    size_t smem = wpb * 2 * 8 * 32 * 16;
    cudaFuncSetAttribute(staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 3; ++r) staged<<<grid, wpb * 32, smem>>>(prev, cur, doff, dsrc, dt, (int)tasks.size(), V);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) staged<<<grid, wpb * 32, smem>>>(prev, cur, doff, dsrc, dt, (int)tasks.size(), V);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("Wp %d W %d E %d tasks %zu: %.1f us/launch, %.0f GB/s alg\n", Wp, W, E, tasks.size(), ms * 100,
           alg * 10 / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
