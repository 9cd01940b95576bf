// Backward layer kernels for float (explicit instantiations).
#include "layer_kernels.cuh"
#include "stream_kernels.cuh"

namespace klay {

int launch_backward_layer(int mode, const LayerArgs<float>& a, cudaStream_t s) {
  switch (mode) {
    case BW_LOGSUM: return launch_layer<float, RK_SUM, BwdGather<float, BW_LOGSUM>>(a, s);
    case BW_LOGSUM8: return launch_layer<float, RK_SUM, BwdGather<float, BW_LOGSUM8>>(a, s);
    case BW_REALPROD: return launch_layer<float, RK_SUM, BwdGather<float, BW_REALPROD>>(a, s);
    case BW_PASSA: return launch_layer<float, RK_SUM, BwdGather<float, BW_PASSA>>(a, s);
    default: return launch_layer<float, RK_SUM, BwdGather<float, BW_PASS>>(a, s);
  }
}

int launch_backward_stream(int mode, const LayerArgs<float>& a, cudaStream_t s) {
  switch (mode) {
    case BW_LOGSUM:
    case BW_LOGSUM8: return launch_stream<float, RK_SUM, BwdGather<float, BW_LOGSUM>>(a, s);
    case BW_REALPROD: return launch_stream<float, RK_SUM, BwdGather<float, BW_REALPROD>>(a, s);
    case BW_PASSA: return launch_stream<float, RK_SUM, BwdGather<float, BW_PASSA>>(a, s);
    default: return launch_stream<float, RK_SUM, BwdGather<float, BW_PASS>>(a, s);
  }
}

int launch_backward_tail(int domain, const TailArgs<float>& t, int cluster, cudaStream_t s) {
  using PASS = BwdGather<float, BW_PASS>;
  if (domain == SR_LOG)  // log: products pass through, sums weight by softmax
    return launch_tail<float, RK_SUM, RK_SUM, PASS, BwdGather<float, BW_LOGSUM>>(t, cluster, s);
  // real: zero-safe product adjoint, sums pass through
  return launch_tail<float, RK_SUM, RK_SUM, BwdGather<float, BW_REALPROD>, PASS>(t, cluster, s);
}

int launch_backward_micro(int domain, const MicroBwdArgs<float>& m, cudaStream_t s) {
  if (domain == SR_LOG) return launch_micro_bwd<float, SR_LOG>(m, s);
  return launch_micro_bwd<float, SR_REAL>(m, s);
}

}  // namespace klay
