// Explicit instantiation: per-instance solve kernel, nx=4 nu=2, 128 threads, >= 6 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<4, 2, 128, 6>;
}  // namespace bmpc_b200
