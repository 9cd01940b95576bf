// Bit-packed Boolean semiring: 32 batch rows per
// 32-bit word, products are bitwise AND, sums bitwise OR. On 0/1 inputs this
// equals the reference's float max/min evaluation (engine.py:177-183)
// bit for bit, with 32x less memory traffic than float32 rows.
#include "layer_kernels.cuh"

namespace klay {

int launch_forward_layer_u1(bool prod, const LayerArgs<unsigned>& a, cudaStream_t s) {
  using G = FwdGather<unsigned>;
  if (prod) return launch_layer<unsigned, RK_AND, G>(a, s);
  return launch_layer<unsigned, RK_OR, G>(a, s);
}

int launch_forward_tail_u1(const TailArgs<unsigned>& t, int cluster, cudaStream_t s) {
  using G = FwdGather<unsigned>;
  return launch_tail<unsigned, RK_AND, RK_OR, G, G>(t, cluster, s);
}

int launch_forward_micro_u1(const MicroArgs<unsigned>& m, cudaStream_t s) {
  return launch_micro<unsigned, RK_AND, RK_OR>(m, s);
}

// one thread per (input slot, 32-row word): bit j of word w = row 32w + j
template <typename TI>
__global__ void pack_inputs_kernel(const TI* __restrict__ w, unsigned* __restrict__ n0, int K,
                                   long long B, long long ldw, int* __restrict__ bad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)K * ldw) return;
  const int k = (int)(i / ldw);
  const long long word = i - (long long)k * ldw;
  unsigned bits = 0;
  for (int j = 0; j < 32; ++j) {
    const long long b = word * 32 + j;
    if (b < B) {
      const TI x = w[b * K + k];
      if (x == TI(1)) bits |= 1u << j;
      else if (x != TI(0)) *bad = 1;
    }
  }
  n0[(size_t)k * ldw + word] = bits;
}

template <typename TO>
__global__ void unpack_outputs_kernel(const unsigned* __restrict__ last, const int* __restrict__ root_node,
                                      const signed char* __restrict__ const_val, TO* __restrict__ out,
                                      int R, long long B, long long ldw) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * R) return;
  const long long b = i / R;
  const int q = (int)(i - b * R);
  const int r = root_node[q];
  TO v;
  if (r >= 0) v = ((last[(size_t)r * ldw + (b >> 5)] >> (b & 31)) & 1u) ? TO(1) : TO(0);
  else v = const_val[q] ? TO(1) : TO(0);
  out[i] = v;
}

void launch_pack_inputs(const void* w, bool w_f64, unsigned* n0, int K, long long B, long long ldw,
                        int* bad, cudaStream_t s) {
  const long long n = (long long)K * ldw;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (w_f64) pack_inputs_kernel<double><<<grid, 256, 0, s>>>((const double*)w, n0, K, B, ldw, bad);
  else pack_inputs_kernel<float><<<grid, 256, 0, s>>>((const float*)w, n0, K, B, ldw, bad);
}

void launch_unpack_outputs(const unsigned* last, const int* root_node, const signed char* const_val,
                           void* out, bool out_f64, int R, long long B, long long ldw,
                           cudaStream_t s) {
  const long long n = B * R;
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (out_f64)
    unpack_outputs_kernel<double><<<grid, 256, 0, s>>>(last, root_node, const_val, (double*)out, R, B, ldw);
  else
    unpack_outputs_kernel<float><<<grid, 256, 0, s>>>(last, root_node, const_val, (float*)out, R, B, ldw);
}

}  // namespace klay
