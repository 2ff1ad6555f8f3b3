// k2.cu -- K2, the two-step temporally blocked sweep (placeholder until the
// TMA kernel lands; the engine falls back to K1 pairs, bitwise identical).
#include "kernels.h"

namespace lbm {

template <typename T>
bool k2_supported(const SlabGeom&) {
    return false;
}

template <typename T>
cudaError_t launch_k2(const T*, T*, const StepParams<T>&, int, int, cudaStream_t) {
    return cudaErrorNotSupported;
}

template bool k2_supported<double>(const SlabGeom&);
template bool k2_supported<float>(const SlabGeom&);
template cudaError_t launch_k2<double>(const double*, double*, const StepParams<double>&, int, int, cudaStream_t);
template cudaError_t launch_k2<float>(const float*, float*, const StepParams<float>&, int, int, cudaStream_t);

}  // namespace lbm
