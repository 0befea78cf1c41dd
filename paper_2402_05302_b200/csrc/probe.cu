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

// The bare memory pattern of K2: n_in streams read, one written, 16-byte vectors, grid-stride,
// integer adds (no method arithmetic) -- the ceiling K2's traffic can reach on the same buffers in
// the same memory-system state (tools/hbm_probe*.cu).
struct PatternArgs {
  const char* in[16];
  char* out;
  size_t nvec;
};

template <int NR>
__global__ void __launch_bounds__(256) stream_pattern_kernel(const PatternArgs a) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.nvec; v += stride) {
    uint4 x[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x[j].x), "=r"(x[j].y), "=r"(x[j].z), "=r"(x[j].w)
                   : "l"(a.in[j] + v * 16));
    }
    uint4 s = x[0];
#pragma unroll
    for (int j = 1; j < NR; ++j) {
      s.x += x[j].x;
      s.y += x[j].y;
      s.z += x[j].z;
      s.w += x[j].w;
    }
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a.out + v * 16),
                 "r"(s.x), "r"(s.y), "r"(s.z), "r"(s.w)
                 : "memory");
  }
}

cudaError_t launch_stream_pattern(const void* const* in, int n_in, void* out, size_t bytes,
                                  int grid, cudaStream_t st) {
  PatternArgs a{};
  for (int j = 0; j < n_in; ++j) a.in[j] = static_cast<const char*>(in[j]);
  a.out = static_cast<char*>(out);
  a.nvec = bytes / 16;
  switch (n_in) {
#define CANNIKIN_CASE(K)                                              \
  case K:                                                             \
    stream_pattern_kernel<K><<<grid, 256, 0, st>>>(a);                \
    break;
    CANNIKIN_CASE(1) CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5)
    CANNIKIN_CASE(6) CANNIKIN_CASE(7) CANNIKIN_CASE(8) CANNIKIN_CASE(9) CANNIKIN_CASE(10)
    CANNIKIN_CASE(11) CANNIKIN_CASE(12) CANNIKIN_CASE(13) CANNIKIN_CASE(14) CANNIKIN_CASE(15)
    CANNIKIN_CASE(16)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cannikin
