// Explicit instantiation: per-instance solve kernel, nx=4 nu=2, 1024 threads, >= 1 blocks/SM.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct CtaVariant<4, 2, 1024, 1>;
}  // namespace bmpc_b200
