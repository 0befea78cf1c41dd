// K2 (TMA variant): the emulated-rank fused pass with bulk-async (TMA engine) staging.
//
// Same contract and arithmetic as wsum_local.cu (Eq. 9 + the Eq. 10 norms):
//   out[e] = sum_j r_j in_j[e] (fp32, rank order),  local_sq[j] = |in_j|^2,  global_sq = |acc|^2.
// Instead of every thread issuing 128-bit loads, one elected producer thread per CTA streams
// contiguous tiles of all n inputs into a ring of shared-memory stages with
// `cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes` (TMA bulk copies, SASS
// UBLKCP), completion tracked by mbarriers (full = bytes landed, empty = consumers done).  8
// consumer warps read the stage from shared memory, compute, and store the output with coalesced
// 16-byte stores.  One CTA per SM; up to ~200 KB of loads in flight per SM in 4-16 KB contiguous
// bulk requests per rank.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {


namespace tma {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (kConsumerWarps + 1);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

}  // namespace tma

// tile_vec: 16-byte vectors per rank per tile; stages: ring depth.
template <typename T, int NR>
__global__ void __launch_bounds__(tma::kThreads, 1)
    wsum_local_tma_kernel(const LocalArgs a, int tile_vec, int stages) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[16];
  __shared__ __align__(8) uint64_t empty[16];
  __shared__ double red[32 * (NR + 1)];
  __shared__ bool s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t ntiles = (a.nvec + tile_vec - 1) / tile_vec;
  const size_t stage_bytes = (size_t)NR * tile_vec * 16;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], tma::kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double lsq[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) lsq[j] = 0.0;
  double gsq = 0.0;

  if (warp == 0) {
    // ---------------- producer: one elected lane streams tiles of all NR inputs
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      size_t it = 0;
      for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = (int)(it % stages);
        const uint32_t round = (uint32_t)(it / stages);
        if (round > 0) tma::mbar_wait(&empty[s], (round - 1) & 1);
        const size_t v0 = tile * (size_t)tile_vec;
        const size_t cnt = (a.nvec - v0) < (size_t)tile_vec ? (a.nvec - v0) : (size_t)tile_vec;
        const uint32_t bytes = (uint32_t)(cnt * 16);
        tma::mbar_expect_tx(&full[s], bytes * NR);
        unsigned char* st = smem + s * stage_bytes;
#pragma unroll
        for (int j = 0; j < NR; ++j)
          tma::bulk_g2s(st + (size_t)j * tile_vec * 16, a.in[j] + v0 * 16, bytes, &full[s], policy);
      }
    }
  } else {
    // ---------------- consumers
    float r[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) r[j] = a.r[j];
    const int ct = threadIdx.x - 32;  // 0 .. 255
    size_t it = 0;
    for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int s = (int)(it % stages);
      const uint32_t round = (uint32_t)(it / stages);
      tma::mbar_wait(&full[s], round & 1);
      const size_t v0 = tile * (size_t)tile_vec;
      const size_t cnt = (a.nvec - v0) < (size_t)tile_vec ? (a.nvec - v0) : (size_t)tile_vec;
      const unsigned char* st = smem + s * stage_bytes;
      for (size_t v = ct; v < cnt; v += 32 * tma::kConsumerWarps) {
        uint4 x[NR];
#pragma unroll
        for (int j = 0; j < NR; ++j)
          x[j] = *reinterpret_cast<const uint4*>(st + ((size_t)j * tile_vec + v) * 16);
        dev::wsum16<T, NR>(x, r, a.out + (v0 + v) * 16, lsq, gsq);
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
    }
    // ragged tail (< one vector): CTA 0's consumers
    if (blockIdx.x == 0) {
      const size_t e = a.nvec * E + ct;
      if (e < a.n) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const float g = V::load1(a.in[j] + e * sizeof(T));
          acc = fmaf(r[j], g, acc);
          lsq[j] += (double)(g * g);
        }
        gsq += (double)(acc * acc);
        V::store1(a.out + e * sizeof(T), acc);
      }
    }
  }

  double vals[NR + 1];
#pragma unroll
  for (int j = 0; j < NR; ++j) vals[j] = lsq[j];
  vals[NR] = gsq;
  dev::block_sum(vals, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j <= NR; ++j) a.partials[(size_t)blockIdx.x * (NR + 1) + j] = vals[j];
    __threadfence();
    s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double tot[NR + 1];
  dev::block_table_sum(a.partials, gridDim.x, NR + 1, tot, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j <= NR; ++j) {
      double* dst = (j < NR) ? (a.local_sq + j) : a.global_sq;
      *dst = a.accumulate ? (*dst + tot[j]) : tot[j];
    }
    *a.ticket = 0u;
  }
}

// ------------------------------------------------------------------------------ host launcher
template <typename T, int NR>
static cudaError_t launch_tma_t(const LocalArgs& a, int num_sms, cudaStream_t st) {
  // 4 KB per rank per tile for many ranks, up to 16 KB for few; ring of <= ~200 KB
  int tile_vec = NR >= 8 ? 256 : (NR >= 4 ? 512 : 1024);
  const size_t stage_bytes = (size_t)NR * tile_vec * 16;
  int stages = (int)((200 * 1024) / stage_bytes);
  if (stages > 16) stages = 16;
  if (stages < 2) {
    stages = 2;
    tile_vec = (int)((100 * 1024) / ((size_t)NR * 16)) & ~31;
  }
  const size_t smem = (size_t)stages * NR * tile_vec * 16;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wsum_local_tma_kernel<T, NR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const size_t ntiles = (a.nvec + tile_vec - 1) / tile_vec;
  int grid = num_sms;
  if ((size_t)grid > ntiles) grid = ntiles < 1 ? 1 : (int)ntiles;
  wsum_local_tma_kernel<T, NR><<<grid, tma::kThreads, smem, st>>>(a, tile_vec, stages);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t dispatch_tma(int nr, const LocalArgs& a, int num_sms, cudaStream_t st) {
  switch (nr) {
#define CANNIKIN_CASE(K) \
  case K:                \
    return launch_tma_t<T, K>(a, num_sms, st);
    CANNIKIN_CASE(1) CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5)
    CANNIKIN_CASE(6) CANNIKIN_CASE(7) CANNIKIN_CASE(8) CANNIKIN_CASE(9) CANNIKIN_CASE(10)
    CANNIKIN_CASE(11) CANNIKIN_CASE(12) CANNIKIN_CASE(13) CANNIKIN_CASE(14) CANNIKIN_CASE(15)
    CANNIKIN_CASE(16)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_wsum_local_tma(cannikin_ctx* ctx, const void* const* in, int nr,
                                  const double* r, void* out, size_t n, cannikin_dtype dt,
                                  double* d_local_sq, double* d_global_sq, bool accumulate,
                                  cudaStream_t st, bool chain) {
  // a plain launch: stream-ordered after its predecessor, so CANNIKIN_LOCAL_CHAIN is satisfied
  // trivially (no overlap with the previous bucket, unlike the LDG variant)
  (void)chain;
  LocalArgs a{};
  for (int j = 0; j < nr; ++j) {
    a.in[j] = static_cast<const char*>(in[j]);
    a.r[j] = (float)r[j];
  }
  a.out = static_cast<char*>(out);
  const size_t esz = dt == CANNIKIN_F32 ? 4 : 2;
  a.n = n;
  a.nvec = n * esz / 16;
  a.partials = &ctx->ctrl->local_part[0][0];
  a.ticket = &ctx->ctrl->ticket_local;
  a.local_sq = d_local_sq;
  a.global_sq = d_global_sq;
  a.accumulate = accumulate ? 1 : 0;
  if (dt == CANNIKIN_F32) return dispatch_tma<float>(nr, a, ctx->num_sms, st);
  return dispatch_tma<__nv_bfloat16>(nr, a, ctx->num_sms, st);
}

}  // namespace cannikin
