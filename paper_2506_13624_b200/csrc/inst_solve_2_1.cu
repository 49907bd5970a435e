// Explicit instantiation: whole-GPU (cooperative) solve + kernel-level LQR for nx=2, nu=1.
#include "kernels_impl.cuh"
namespace bmpc_b200 {
template struct SolveLaunch<2, 1>;
template struct LqrLaunch<2, 1>;
}  // namespace bmpc_b200
