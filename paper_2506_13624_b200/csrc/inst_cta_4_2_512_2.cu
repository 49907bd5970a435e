// Explicit instantiation: per-instance solve kernel, nx=4 nu=2, 512 threads, >= 2 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<4, 2, 512, 2>;
}  // namespace bmpc_b200
