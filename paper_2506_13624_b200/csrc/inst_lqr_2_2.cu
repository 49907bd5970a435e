// Explicit instantiation: kernel-level LQR tree for nx=2, nu=2.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct LqrLaunch<2, 2>;
}  // namespace bmpc_b200
