// Backward layer kernels for double (explicit instantiations).
#include "layer_kernels.cuh"

namespace klay {

int launch_backward_layer(int mode, const LayerArgs<double>& a, cudaStream_t s) {
  switch (mode) {
    case BW_LOGSUM: return launch_layer<double, RK_SUM, BwdGather<double, BW_LOGSUM>>(a, s);
    case BW_REALPROD: return launch_layer<double, RK_SUM, BwdGather<double, BW_REALPROD>>(a, s);
    default: return launch_layer<double, RK_SUM, BwdGather<double, BW_PASS>>(a, s);
  }
}

}  // namespace klay
