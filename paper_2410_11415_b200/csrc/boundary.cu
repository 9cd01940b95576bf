// Boundary kernels: weights in (transpose + cast to node-major rows), roots
// out, backward seeds in, input gradients out (transpose to [B, K]).
#include "common.cuh"
#include "layer_api.h"

namespace klay {

// N0[k, c] = cast(w[c, k]) for c < B, identity padding for c >= B.
template <typename T, typename TI>
__global__ void load_inputs_kernel(const TI* __restrict__ w, T* __restrict__ n0, int K,
                                   long long B, long long ld, T pad) {
  __shared__ T tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long c = c0 + i;
    const int k = k0 + threadIdx.x;
    tile[i][threadIdx.x] = (c < B && k < K) ? (T)w[c * K + k] : pad;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i;
    const long long c = c0 + threadIdx.x;
    if (k < K && c < ld) n0[(size_t)k * ld + c] = tile[threadIdx.x][i];
  }
}

// out[b, q] = rows[q, b] for a [Q rows, ld] node-major block -> [B, Q]
template <typename T>
__global__ void store_rows_kernel(const T* __restrict__ rows, T* __restrict__ out, int Q,
                                  long long B, long long ld) {
  __shared__ T tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int q0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int q = q0 + i;
    const long long c = c0 + threadIdx.x;
    if (q < Q && c < B) tile[i][threadIdx.x] = rows[(size_t)q * ld + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long c = c0 + i;
    const int q = q0 + threadIdx.x;
    if (q < Q && c < B) out[c * Q + q] = tile[threadIdx.x][i];
  }
}

// _assemble_outputs (engine.py:203-212): root columns of the last layer,
// constants as the semiring's one/zero.
template <typename T>
__global__ void assemble_outputs_kernel(const T* __restrict__ last, const int* __restrict__ root_node,
                                        const signed char* __restrict__ const_val, T* __restrict__ out,
                                        int R, long long B, long long ld, T zero, T one) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * R) return;
  const long long b = i / R;
  const int q = (int)(i - b * R);
  const int r = root_node[q];
  out[i] = (r >= 0) ? last[(size_t)r * ld + b] : (const_val[q] ? one : zero);
}

// Seed scatter (engine.py:330-334): grad_L[j] = 0 + sum of the seeds of the
// root positions that read node j, in position order (duplicates accumulate).
template <typename T>
__global__ void seed_kernel(const T* __restrict__ seed, const int* __restrict__ top_off,
                            const int* __restrict__ top_pos, T* __restrict__ g, int WL, int R,
                            long long B, long long ld) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)WL * ld) return;
  const int j = (int)(i / ld);
  const long long c = i - (long long)j * ld;
  T acc = T(0);
  if (c < B) {
    for (int s = top_off[j]; s < top_off[j + 1]; ++s)
      acc += seed ? seed[c * R + top_pos[s]] : T(1);
  }
  g[i] = acc;
}


template <typename T>
void launch_load_inputs(const void* w, bool w_f64, T* n0, int K, long long B, long long ld, T pad,
                        cudaStream_t s) {
  dim3 grid((unsigned)((ld + 31) / 32), (unsigned)((K + 31) / 32));
  dim3 block(32, 8);
  if (w_f64)
    load_inputs_kernel<T, double><<<grid, block, 0, s>>>((const double*)w, n0, K, B, ld, pad);
  else
    load_inputs_kernel<T, float><<<grid, block, 0, s>>>((const float*)w, n0, K, B, ld, pad);
}

template <typename T>
void launch_store_rows(const T* rows, T* out, int Q, long long B, long long ld, cudaStream_t s) {
  dim3 grid((unsigned)((B + 31) / 32), (unsigned)((Q + 31) / 32));
  store_rows_kernel<T><<<grid, dim3(32, 8), 0, s>>>(rows, out, Q, B, ld);
}

template <typename T>
void launch_assemble_outputs(const T* last, const int* root_node, const signed char* const_val,
                             T* out, int R, long long B, long long ld, T zero, T one,
                             cudaStream_t s) {
  const long long n = B * R;
  assemble_outputs_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      last, root_node, const_val, out, R, B, ld, zero, one);
}

template <typename T>
void launch_seed(const T* seed, const int* top_off, const int* top_pos, T* g, int WL, int R,
                 long long B, long long ld, cudaStream_t s) {
  const long long n = (long long)WL * ld;
  seed_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(seed, top_off, top_pos, g, WL, R, B, ld);
}

// Rows of aliased (unary) nodes a backward-only trace left unwritten: the
// source row {x & 0x7fffffff <- y}; bit 31 of x: the chain holds a unary sum,
// so the value is a logsumexp of one element (+inf -> NaN). One thread per
// element.
template <typename T>
__global__ void fill_aliases_kernel(const int2* __restrict__ pairs, long long n, T* values,
                                    long long ld) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * ld) return;
  const long long k = i / ld, c = i - k * ld;
  const int2 pr = pairs[k];
  const T v = values[(size_t)pr.y * ld + c];
  values[(size_t)(pr.x & 0x7fffffff) * ld + c] = (pr.x < 0 && v == T(INFINITY)) ? T(NAN) : v;
}

template <typename T>
void launch_fill_aliases(const int2* pairs, long long n, T* values, long long ld, cudaStream_t s) {
  const long long m = n * ld;
  if (m > 0) fill_aliases_kernel<T><<<(unsigned)((m + 255) / 256), 256, 0, s>>>(pairs, n, values, ld);
}

#define KLAY_INST(T)                                                                            \
  template void launch_load_inputs<T>(const void*, bool, T*, int, long long, long long, T,      \
                                      cudaStream_t);                                            \
  template void launch_store_rows<T>(const T*, T*, int, long long, long long, cudaStream_t);    \
  template void launch_assemble_outputs<T>(const T*, const int*, const signed char*, T*, int,   \
                                           long long, long long, T, T, cudaStream_t);           \
  template void launch_seed<T>(const T*, const int*, const int*, T*, int, int, long long,       \
                               long long, cudaStream_t);                                        \
  template void launch_fill_aliases<T>(const int2*, long long, T*, long long, cudaStream_t);
KLAY_INST(float)
KLAY_INST(double)
#undef KLAY_INST

}  // namespace klay
