// Microbenchmark: achievable bandwidth of row-gather patterns on B200.
// rows of 4 KB (B=1024 fp32); each "node" reads `fan` random child rows
// (from a 280 MB layer) and writes one output row (230 MB layer).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}

// A: thread per (node, 16B column); loads n child rows directly (LDG.128)
__global__ void gather_direct(const float4* __restrict__ prev, float4* __restrict__ cur,
                              const int* __restrict__ src, int W, int fan, int V) {
  int v = blockIdx.y * 32 + (threadIdx.x & 31);
  int node = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (node >= W) return;
  float4 acc = make_float4(0, 0, 0, 0);
  float4 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < fan) x[i] = __ldcg(prev + (size_t)src[node * fan + i] * V + v);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < fan) { acc.x += x[i].x; acc.y += x[i].y; acc.z += x[i].z; acc.w += x[i].w; }
  cur[(size_t)node * V + v] = acc;
}

// B: warp per task of `tn` nodes, cp.async staged in batches of 8 edges, 2 stages
__global__ void gather_staged(const float4* __restrict__ prev, float4* __restrict__ cur,
                              const int* __restrict__ src, int W, int fan, int V, int tn) {
  extern __shared__ float4 sm[];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* st = sm + warp * 2 * 8 * 32;
  int task = blockIdx.x * (blockDim.x / 32) + warp;
  int n0 = task * tn;
  if (n0 >= W) return;
  int n1 = min(W, n0 + tn);
  int e0 = n0 * fan, e1 = n1 * fan;
  int v = blockIdx.y * 32 + lane;
  int nb = (e1 - e0 + 7) / 8;
  auto issue = [&](int b) {
    int base = e0 + b * 8;
    int cnt = min(8, e1 - base);
    for (int i = 0; i < cnt; ++i) cp16(st + (b & 1) * 256 + i * 32 + lane, prev + (size_t)src[base + i] * V + v);
    asm volatile("cp.async.commit_group;\n");
  };
  issue(0);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int b = 0; b < nb; ++b) {
    if (b + 1 < nb) { issue(b + 1); asm volatile("cp.async.wait_group 1;\n"); }
    else asm volatile("cp.async.wait_group 0;\n");
    int base = e0 + b * 8;
    int cnt = min(8, e1 - base);
    for (int i = 0; i < cnt; ++i) {
      float4 x = st[(b & 1) * 256 + i * 32 + lane];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      int e = base + i;
      if ((e - e0 + 1) % fan == 0) {
        cur[(size_t)(n0 + (e - e0) / fan) * V + v] = acc;
        acc = make_float4(0, 0, 0, 0);
      }
    }
  }
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __ldcg(a + i);
}

int main() {
  const int V = 256;  // 4 KB rows
  const int Wp = 68000, W = 57000;
  float4 *prev, *cur;
  cudaMalloc(&prev, (size_t)Wp * V * 16);
  cudaMalloc(&cur, (size_t)W * V * 16);
  cudaMemset(prev, 0, (size_t)Wp * V * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // copy
  size_t n = (size_t)W * V;
  for (int r = 0; r < 3; ++r) copy_kernel<<<148 * 8, 256>>>(prev, cur, n);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) copy_kernel<<<148 * 8, 256>>>(prev, cur, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy %.1f GB/s\n", 2.0 * n * 16 * 10 / (ms * 1e-3) / 1e9);
  for (int fan : {1, 2, 3}) {
    std::vector<int> h((size_t)W * fan);
    srand(1);
    for (auto& x : h) x = rand() % Wp;
    int* d;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    double alg = ((double)Wp * V * 16 + (double)W * V * 16);  // algorithmic: read prev once, write cur
    for (int wpb : {4, 8}) {
      dim3 grid((W + wpb - 1) / wpb, V / 32);
      for (int r = 0; r < 3; ++r) gather_direct<<<grid, wpb * 32>>>(prev, cur, d, W, fan, V);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) gather_direct<<<grid, wpb * 32>>>(prev, cur, d, W, fan, V);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("fan %d direct  wpb %d: %.1f GB/s alg (%.1f us)\n", fan, wpb, alg * 10 / (ms * 1e-3) / 1e9, ms * 100);
    }
    for (int tn : {8, 16, 32}) {
      int wpb = 4;
      dim3 grid(((W + tn - 1) / tn + wpb - 1) / wpb, V / 32);
      size_t smem = wpb * 2 * 8 * 32 * 16;
      for (int r = 0; r < 3; ++r) gather_staged<<<grid, wpb * 32, smem>>>(prev, cur, d, W, fan, V, tn);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) gather_staged<<<grid, wpb * 32, smem>>>(prev, cur, d, W, fan, V, tn);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("fan %d staged tn %d: %.1f GB/s alg (%.1f us)\n", fan, tn, alg * 10 / (ms * 1e-3) / 1e9, ms * 100);
    }
    cudaFree(d);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
