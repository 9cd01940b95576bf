// Backward layer kernels for double (explicit instantiations).
#include "layer_kernels.cuh"
#include "stream_kernels.cuh"

namespace klay {

int launch_backward_layer(int mode, const LayerArgs<double>& a, cudaStream_t s) {
  switch (mode) {
    case BW_LOGSUM: return launch_layer<double, RK_SUM, BwdGather<double, BW_LOGSUM>>(a, s);
    case BW_LOGSUM8: return launch_layer<double, RK_SUM, BwdGather<double, BW_LOGSUM8>>(a, s);
    case BW_REALPROD: return launch_layer<double, RK_SUM, BwdGather<double, BW_REALPROD>>(a, s);
    case BW_PASSA: return launch_layer<double, RK_SUM, BwdGather<double, BW_PASSA>>(a, s);
    default: return launch_layer<double, RK_SUM, BwdGather<double, BW_PASS>>(a, s);
  }
}

int launch_backward_stream(int mode, const LayerArgs<double>& a, cudaStream_t s) {
  switch (mode) {
    case BW_LOGSUM:
    case BW_LOGSUM8: return launch_stream<double, RK_SUM, BwdGather<double, BW_LOGSUM>>(a, s);
    case BW_REALPROD: return launch_stream<double, RK_SUM, BwdGather<double, BW_REALPROD>>(a, s);
    case BW_PASSA: return launch_stream<double, RK_SUM, BwdGather<double, BW_PASSA>>(a, s);
    default: return launch_stream<double, RK_SUM, BwdGather<double, BW_PASS>>(a, s);
  }
}

int launch_backward_tail(int domain, const TailArgs<double>& t, int cluster, cudaStream_t s) {
  using PASS = BwdGather<double, BW_PASS>;
  if (domain == SR_LOG)  // log: products pass through, sums weight by softmax
    return launch_tail<double, RK_SUM, RK_SUM, PASS, BwdGather<double, BW_LOGSUM>>(t, cluster, s);
  // real: zero-safe product adjoint, sums pass through
  return launch_tail<double, RK_SUM, RK_SUM, BwdGather<double, BW_REALPROD>, PASS>(t, cluster, s);
}

int launch_backward_micro(int domain, const MicroBwdArgs<double>& m, cudaStream_t s) {
  if (domain == SR_LOG) return launch_micro_bwd<double, SR_LOG>(m, s);
  return launch_micro_bwd<double, SR_REAL>(m, s);
}

}  // namespace klay
