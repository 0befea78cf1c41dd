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
  int repeat;             // passes over the segments (long transfers amortise the launch)
  size_t nvec;            // 16-byte vectors per peer
};

// Every CTA writes to every peer, interleaved (as the K3 kernels do): vector v of each peer's
// segment in turn, the W-1 loads of an index issued together
template <int NP>
__global__ void __launch_bounds__(512) a2a_write_kernel(const A2aArgs a) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int rep = 0; rep < a.repeat; ++rep)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.nvec; i += stride) {
      uint4 x[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) x[k] = a.src[(size_t)k * a.nvec + i];
#pragma unroll
      for (int k = 0; k < NP; ++k) a.dst[k][i] = x[k];
    }
}

cudaError_t launch_a2a_write(cannikin_ctx* ctx, size_t bytes_per_peer, int repeat,
                             int ctas_per_sm, cudaStream_t st) {
  A2aArgs a{};
  a.repeat = repeat;
  a.src = reinterpret_cast<const uint4*>(ctx->base + ctx->user_off);
  a.npeers = 0;
  for (int j = 0; j < ctx->world; ++j) {
    if (j == ctx->rank) continue;
    a.dst[a.npeers++] = reinterpret_cast<uint4*>(ctx->peer_base[j] + ctx->scratch_off +
                                                  (size_t)ctx->rank * bytes_per_peer);
  }
  a.nvec = bytes_per_peer / 16;
  // every CTA sends to every peer (a CTA per SM sending to one peer each -- the
  // tools/nvlink_bw.cu form -- measured 606 GB/s at W = 4 against K3's 642)
  const int grid = ctas_per_sm * ctx->num_sms;
  switch (a.npeers) {
#define CANNIKIN_CASE(K)                                   \
  case K:                                                  \
    a2a_write_kernel<K><<<grid, 512, 0, st>>>(a);          \
    break;
    CANNIKIN_CASE(1) CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5)
    CANNIKIN_CASE(6) CANNIKIN_CASE(7)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cannikin
