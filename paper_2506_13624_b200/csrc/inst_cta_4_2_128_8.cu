// Explicit instantiation: per-instance solve kernel, nx=4 nu=2, 128 threads, >= 8 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<4, 2, 128, 8>;
}  // namespace bmpc_b200
