// Microbenchmark: how fast can one SM pull random 4 KB rows into shared
// memory? (a) one thread issuing cp.async.bulk (TMA, UBLKCP) per row into a
// ring of R slots, recycling a slot when its mbarrier completes; (b) one warp
// issuing 16-byte cp.async (LDGSTS) per lane, completion through
// cp.async.mbarrier.arrive.noinc. No consumers: the rate of the copy engine.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o copy_rate copy_rate.cu
#include <cuda_runtime.h>

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
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}

// rows: n random row indices per CTA
template <int ROWB>
__global__ void copy_tma(const char* __restrict__ base, const int* __restrict__ rows, int n, int R) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
  unsigned char* ring = smem + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    const int* r = rows + (size_t)blockIdx.x * n;
    for (int i = 0; i < n; ++i) {
      const int s = i % R, lap = i / R;
      if (lap > 0) mbar_wait(&bar[s], (lap - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(&bar[s])), "r"(ROWB)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              sa(ring + (size_t)s * ROWB)),
          "l"(base + (size_t)__ldg(r + i) * ROWB), "r"(ROWB), "r"(sa(&bar[s]))
          : "memory");
    }
    for (int i = n; i < n + R; ++i) {
      const int s = i % R, lap = i / R;
      if (lap > 0 && i - R < n) mbar_wait(&bar[s], (lap - 1) & 1);
    }
  }
}

template <int ROWB>
__global__ void copy_ldgsts(const char* __restrict__ base, const int* __restrict__ rows, int n, int R) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
  unsigned char* ring = smem + 1024;
  const int lane = threadIdx.x;
  if (lane == 0)
    for (int i = 0; i < R; ++i) mbar_init(&bar[i], 32);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int* r = rows + (size_t)blockIdx.x * n;
  for (int i = 0; i < n; ++i) {
    const int s = i % R, lap = i / R;
    if (lap > 0) mbar_wait(&bar[s], (lap - 1) & 1);
    const char* src = base + (size_t)__ldg(r + i) * ROWB;
#pragma unroll
    for (int q = 0; q < ROWB / 512; ++q)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa(ring + (size_t)s * ROWB + q * 512 + lane * 16)),
                   "l"(src + q * 512 + lane * 16)
                   : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(sa(&bar[s])) : "memory");
  }
  for (int i = n; i < n + R; ++i) {
    const int s = i % R, lap = i / R;
    if (lap > 0 && i - R < n) mbar_wait(&bar[s], (lap - 1) & 1);
  }
}


// (c) the whole warp issues: round r covers rows [32r, 32r + 32), lane l one
// copy; slots recycled per lap (R multiple of 32)
template <int ROWB>
__global__ void copy_tma_warp(const char* __restrict__ base, const int* __restrict__ rows, int n, int R) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem);
  unsigned char* ring = smem + 1024;
  const int lane = threadIdx.x;
  const int NB = R / 32;  // barriers: one per 32-slot block
  if (lane < NB) mbar_init(&bar[lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int* r = rows + (size_t)blockIdx.x * n;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int blk = (i0 / 32) % NB, lap = (i0 / 32) / NB;
    const int row = __ldg(r + i0 + lane);
    if (lane == 0) {
      if (lap > 0) mbar_wait(&bar[blk], (lap - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(&bar[blk])), "r"(32 * ROWB)
                   : "memory");
    }
    __syncwarp();
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            sa(ring + (size_t)(blk * 32 + lane) * ROWB)),
        "l"(base + (size_t)row * ROWB), "r"(ROWB), "r"(sa(&bar[blk]))
        : "memory");
  }
  if (lane == 0) {
    const int nr = n / 32;
    for (int b = max(0, nr - NB); b < nr; ++b) mbar_wait(&bar[b % NB], (b / NB) & 1);
  }
}

int main() {
  constexpr int ROWB = 4096;
  const size_t big = (size_t)1 << 30;  // 1 GB: DRAM
  char* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 1, big));
  const int n = 256;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int span_mb : {1024, 32}) {
    const int nrows = (int)((size_t)span_mb * (1 << 20) / ROWB);
    for (int per_sm : {1, 2, 4, 8}) {
      const int nc = 148 * per_sm;
      std::vector<int> rows((size_t)nc * n);
      unsigned s = 12345;
      for (auto& r : rows) {
        s = s * 1664525u + 1013904223u;
        r = (int)(s % (unsigned)nrows);
      }
      int* dr;
      CK(cudaMalloc(&dr, rows.size() * 4));
      CK(cudaMemcpy(dr, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
      for (int R : {4, 8, 12, 24, 32}) {
        const size_t smem = 1024 + (size_t)R * ROWB;
        if (smem * per_sm > 227 * 1024) continue;
        for (int kind = 0; kind < 3; ++kind) {
          if (kind == 2 && R != 32) continue;
          if (kind < 2 && R == 32) continue;
          auto launch = [&] {
            if (kind == 0)
              copy_tma<ROWB><<<nc, 32, smem>>>(buf, dr, n, R);
            else if (kind == 1)
              copy_ldgsts<ROWB><<<nc, 32, smem>>>(buf, dr, n, R);
            else
              copy_tma_warp<ROWB><<<nc, 32, smem>>>(buf, dr, n, R);
          };
          CK(cudaFuncSetAttribute(copy_tma_warp<ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
          CK(cudaFuncSetAttribute(copy_tma<ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
          CK(cudaFuncSetAttribute(copy_ldgsts<ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
          launch();
          CK(cudaDeviceSynchronize());
          CK(cudaEventRecord(e0));
          for (int it = 0; it < 5; ++it) launch();
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          const double bytes = 5.0 * nc * n * ROWB;
          printf("span %5d MB  %d CTA/SM  R=%2d  %-6s  %7.0f GB/s  (%.1f GB/s per CTA)\n", span_mb, per_sm, R,
                 kind == 2 ? "TMAx32" : (kind ? "LDGSTS" : "TMA"), bytes / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9 / nc);
        }
      }
      cudaFree(dr);
    }
  }
  return 0;
}
