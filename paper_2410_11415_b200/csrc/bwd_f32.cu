// Backward layer kernels for float (explicit instantiations).
#include "layer_kernels.cuh"

namespace klay {

int launch_backward_layer(int mode, const LayerArgs<float>& a, cudaStream_t s) {
  switch (mode) {
    case BW_LOGSUM: return launch_layer<float, RK_SUM, BwdGather<float, BW_LOGSUM>>(a, s);
    case BW_REALPROD: return launch_layer<float, RK_SUM, BwdGather<float, BW_REALPROD>>(a, s);
    default: return launch_layer<float, RK_SUM, BwdGather<float, BW_PASS>>(a, s);
  }
}

}  // namespace klay
