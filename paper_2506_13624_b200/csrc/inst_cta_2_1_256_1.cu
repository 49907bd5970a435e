// Explicit instantiation: per-instance solve kernel, nx=2 nu=1, 256 threads, >= 1 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<2, 1, 256, 1>;
}  // namespace bmpc_b200
