// Forward layer kernels for double (explicit instantiations).
#include "layer_kernels.cuh"
#include "stream_kernels.cuh"

namespace klay {

int launch_forward_layer(int sr, bool prod, bool alias, const LayerArgs<double>& a, cudaStream_t s) {
  using G = FwdGather<double>;
  // product layer over an aliased sum layer (log semiring, epsilon 0)
  if (alias) return launch_layer<double, RK_SUM, FwdGather<double, true>>(a, s);
  switch (sr) {
    case SR_REAL:
      if (prod) return launch_layer<double, RK_PROD, G>(a, s);
      else return launch_layer<double, RK_SUM, G>(a, s);
    case SR_LOG:
      if (prod) return launch_layer<double, RK_SUM, G>(a, s);
      else return launch_layer<double, RK_LSE, G>(a, s);
    case SR_BOOL:
      if (prod) return launch_layer<double, RK_MIN, G>(a, s);
      else return launch_layer<double, RK_MAX, G>(a, s);
    default:  // max-product
      if (prod) return launch_layer<double, RK_PROD, G>(a, s);
      else return launch_layer<double, RK_MAX, G>(a, s);
  }
}

int launch_forward_stream(int sr, bool prod, bool alias, const LayerArgs<double>& a, cudaStream_t s) {
  using G = FwdGather<double>;
  if (alias) return launch_stream<double, RK_SUM, FwdGather<double, true>>(a, s);
  switch (sr) {
    case SR_REAL:
      if (prod) return launch_stream<double, RK_PROD, G>(a, s);
      else return launch_stream<double, RK_SUM, G>(a, s);
    case SR_LOG:
      if (prod) return launch_stream<double, RK_SUM, G>(a, s);
      else return launch_stream<double, RK_LSE, G>(a, s);
    case SR_BOOL:
      if (prod) return launch_stream<double, RK_MIN, G>(a, s);
      else return launch_stream<double, RK_MAX, G>(a, s);
    default:  // max-product
      if (prod) return launch_stream<double, RK_PROD, G>(a, s);
      else return launch_stream<double, RK_MAX, G>(a, s);
  }
}

int launch_forward_tail(int sr, const TailArgs<double>& t, int cluster, cudaStream_t s) {
  using G = FwdGather<double>;
  switch (sr) {
    case SR_REAL: return launch_tail<double, RK_PROD, RK_SUM, G, G>(t, cluster, s);
    case SR_LOG: return launch_tail<double, RK_SUM, RK_LSE, G, G>(t, cluster, s);
    case SR_BOOL: return launch_tail<double, RK_MIN, RK_MAX, G, G>(t, cluster, s);
    default: return launch_tail<double, RK_PROD, RK_MAX, G, G>(t, cluster, s);
  }
}

int launch_forward_micro(int sr, const MicroArgs<double>& m, cudaStream_t s) {
  switch (sr) {
    case SR_REAL: return launch_micro<double, RK_PROD, RK_SUM>(m, s);
    case SR_LOG: return launch_micro<double, RK_SUM, RK_LSE>(m, s);
    case SR_BOOL: return launch_micro<double, RK_MIN, RK_MAX>(m, s);
    default: return launch_micro<double, RK_PROD, RK_MAX>(m, s);
  }
}

}  // namespace klay
