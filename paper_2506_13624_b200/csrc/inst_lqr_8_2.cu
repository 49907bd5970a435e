// Explicit instantiation: kernel-level LQR tree for nx=8, nu=2.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct LqrLaunch<8, 2>;
}  // namespace bmpc_b200
