// K7 (bench utility, not part of the method): synthetic compute of a prescribed duration, used to
// emulate heterogeneous per-node compute time t_i(b) = a_i + P_i (Eq. 3) on the
// homogeneous B200 box -- the role of Cluster C's dummy load.  One warp on one SM
// spins on %globaltimer, so the emulated "compute" does not steal the SMs or HBM bandwidth the
// gradient-aggregation kernels use.
#include <cuda_runtime.h>

#include "common.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

__global__ void emulate_compute_kernel(uint64_t ns) {
  const uint64_t t0 = dev::globaltimer_ns();
  while (dev::globaltimer_ns() - t0 < ns) {
    __nanosleep(200);
  }
}

cudaError_t launch_emulate(double seconds, cudaStream_t st) {
  const double ns = seconds > 0.0 ? seconds * 1e9 : 0.0;
  emulate_compute_kernel<<<1, 32, 0, st>>>((uint64_t)ns);
  return cudaGetLastError();
}

}  // namespace cannikin
