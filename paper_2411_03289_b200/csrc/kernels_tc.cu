// kernels_tc.cu — tensor-core (tcgen05, TF32) variance path. Placeholder until
// the sm_100a UMMA kernel lands; the FFMA path is the default.
#include "internal.hpp"

namespace gpm {
cudaError_t launch_tc_variance(const VarianceArgs&, int, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace gpm
