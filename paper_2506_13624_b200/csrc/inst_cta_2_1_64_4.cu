// Explicit instantiation: per-instance solve kernel, nx=2 nu=1, 64 threads, >= 4 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<2, 1, 64, 4>;
}  // namespace bmpc_b200
