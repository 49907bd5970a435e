// Explicit instantiation: kernel-level LQR tree for nx=8, nu=4.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct LqrLaunch<8, 4>;
}  // namespace bmpc_b200
