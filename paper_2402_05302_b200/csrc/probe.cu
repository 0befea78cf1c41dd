// Bench utility (not the method): the NVLink ceiling the K3 kernels run against, measured live on
// the ctx's own peer mappings.  Every rank writes `bytes_per_peer` of its heap into its slot of
// every peer's scratch half at the same time -- the all-to-all write pattern of a two-shot
// all-reduce with both directions of every link loaded -- so the per-direction rate is
// (W-1) x bytes_per_peer / time.  tools/nvlink_bw.cu measured the same pattern once per W
// (2: 690.8, 4: 671.4 GB/s); this puts the number for any W, including the driver's 8-GPU run,
// into the bench line next to K3's busbw.
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "kernels.h"

namespace cannikin {

struct A2aArgs {
  const uint4* src;       // this rank's heap (any contents)
  uint4* dst[kMaxWorld];  // peer p's scratch + rank * bytes_per_peer, for the W-1 peers
  int npeers;
  size_t nvec;            // 16-byte vectors per peer
};

// CTA c writes to peer c % npeers; 4 vectors in flight per thread
__global__ void __launch_bounds__(512) a2a_write_kernel(const A2aArgs a) {
  const int k = blockIdx.x % a.npeers;
  const int cta = blockIdx.x / a.npeers, nct = gridDim.x / a.npeers;
  const uint4* s = a.src + (size_t)k * a.nvec;
  uint4* d = a.dst[k];
  const size_t stride = (size_t)nct * blockDim.x;
  size_t i = (size_t)cta * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < a.nvec; i += 4 * stride) {
    const uint4 x0 = s[i], x1 = s[i + stride], x2 = s[i + 2 * stride], x3 = s[i + 3 * stride];
    d[i] = x0;
    d[i + stride] = x1;
    d[i + 2 * stride] = x2;
    d[i + 3 * stride] = x3;
  }
  for (; i < a.nvec; i += stride) d[i] = s[i];
}

cudaError_t launch_a2a_write(cannikin_ctx* ctx, size_t bytes_per_peer, cudaStream_t st) {
  A2aArgs a{};
  a.src = reinterpret_cast<const uint4*>(ctx->base + ctx->user_off);
  a.npeers = 0;
  for (int j = 0; j < ctx->world; ++j) {
    if (j == ctx->rank) continue;
    a.dst[a.npeers++] = reinterpret_cast<uint4*>(ctx->peer_base[j] + ctx->scratch_off +
                                                  (size_t)ctx->rank * bytes_per_peer);
  }
  a.nvec = bytes_per_peer / 16;
  const int grid = (ctx->num_sms / a.npeers) * a.npeers;  // whole CTAs per peer
  a2a_write_kernel<<<grid, 512, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cannikin
