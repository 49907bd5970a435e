// Explicit instantiation: whole-GPU (cooperative) solve + kernel-level LQR for nx=4, nu=2.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct SolveLaunch<4, 2>;
template struct LqrLaunch<4, 2>;
}  // namespace bmpc_b200
