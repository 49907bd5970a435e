// Explicit instantiation: per-instance solve kernel, nx=3 nu=2, 256 threads, >= 1 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<3, 2, 256, 1>;
}  // namespace bmpc_b200
