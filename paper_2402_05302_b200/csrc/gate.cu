// Gated entry (CANNIKIN_INIT_GATED_ENTRY): the wait for late peers done by ONE warp.
//
// Under heterogeneous ranks a fast rank reaches bucket j long before a slow one (the straggler
// effect of §3.2.2-3).  The reduction kernels wait for their peers on the device; a
// 148-CTA kernel that waits holds every SM the rank's own backward pass (overlapped)
// needs.  With the gate, each weighted all-reduce is preceded on its stream by this one-warp
// kernel: lane j publishes "rank `rank` is at gate epoch e" into peer j's control region and waits
// until peer j has published e as well.  Only then is the data kernel launched, so its own peer
// waits last microseconds (launch skew), and the long wait occupies one SM slot of 32 threads.
// Epochs count gated calls on the ctx; every rank makes the same sequence of calls (as for the
// reduction itself), so the epochs agree.  Release/acquire at system scope: the bucket contents
// written before this kernel (stream order) are visible to a peer that observes the flag.
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

struct GateArgs {
  Ctrl* pctrl[kMaxWorld];
  Ctrl* ctrl;
  int rank, world;
  uint64_t timeout_ns;
};

__global__ void __launch_bounds__(32) gate_kernel(const GateArgs a) {
  const uint64_t ep = a.ctrl->gate_epoch + 1;  // one CTA: the counter has a single writer
  __syncwarp();
  const int j = threadIdx.x;
  if (j < a.world) {
    dev::st_release_sys(&a.pctrl[j]->gate[a.rank], ep);
    dev::SpinClock clk;
    while (dev::ld_acquire_sys(&a.ctrl->gate[j]) < ep) {
      __nanosleep(128);
      if (clk.expired(a.timeout_ns, 255u, &a.ctrl->error_code, 1)) break;  // peer never arrived
    }
  }
  __syncwarp();
  if (j == 0) a.ctrl->gate_epoch = ep;
}

cudaError_t launch_gate(cannikin_ctx* ctx, cudaStream_t st) {
  GateArgs a{};
  for (int j = 0; j < ctx->world; ++j) a.pctrl[j] = reinterpret_cast<Ctrl*>(ctx->peer_base[j]);
  a.ctrl = ctx->ctrl;
  a.rank = ctx->rank;
  a.world = ctx->world;
  a.timeout_ns = ctx->spin_timeout_ns;
  gate_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cannikin
