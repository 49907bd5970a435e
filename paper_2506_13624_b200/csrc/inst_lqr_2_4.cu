// Explicit instantiation: kernel-level LQR tree for nx=2, nu=4.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct LqrLaunch<2, 4>;
}  // namespace bmpc_b200
