// K2: single-GPU fused pass over n emulated ranks (the 1-B200 metric kernel).
//
//   out[e]        = sum_{j=0..n-1} r_j in_j[e]          Eq. 9, fp32, rank order
//   local_sq[j]   = sum_e in_j[e]^2                     |g_j|^2, Eq. 10 input
//   global_sq     = sum_e acc[e]^2                      |g|^2 from the fp32 accumulator (reading Q2)
//
// HBM-bound: (n+1) * N * sizeof(T) algorithmic bytes, ~3 flops per element and rank.  Design:
// persistent grid of (SMs x occupancy) CTAs of 256 threads, each thread streams 16-byte vectors
// with n*U independent 128-bit loads in flight, L1 bypassed; norms are accumulated per thread in
// fp32 over one vector and fp64 beyond; per-CTA partials are reduced by the last CTA to finish
// (ticket) in a fixed order, so the result is bitwise deterministic for a fixed grid.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {


// Register budget (n <= 8 ranks): 4 resident 256-thread CTAs per SM (<= 64 registers).  With it ptxas keeps the
// loads of a vector batch closer together (5 of 8 issued ahead of the arithmetic); A/B on one box
// (profiles/r01/k2_minb_ab.jsonl): C4 0.3256 -> 0.3195 ms, C5 1.970 -> 1.848 ms, against no
// minimum (60 registers) and 3 CTAs (74 registers, all 8 loads ahead: between the two).
#ifndef CANNIKIN_K2_MINB
#define CANNIKIN_K2_MINB 4
#endif
template <typename T, int NR, int U, int NT>
__global__ void __launch_bounds__(NT, NT == 256 && NR <= 8 ? CANNIKIN_K2_MINB : 1)
    wsum_local_kernel(const LocalArgs a) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  __shared__ double red[32 * (NR + 1)];
  __shared__ bool s_last;

  // Programmatic dependent launch: the next kernel may be scheduled at once -- a chained next
  // bucket (CANNIKIN_LOCAL_CHAIN) then streams its inputs while this grid's last CTAs finish.
  // Without the chain flag this launch waits for its predecessor before reading anything (it may
  // have produced our inputs); with it, only before the shared partial table and the statistics.
  dev::pdl_launch_dependents();
  if (!a.chain) dev::pdl_wait();
  if (threadIdx.x == 0) {
    a.trace[blockIdx.x * 5] = dev::globaltimer_ns();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.trace[blockIdx.x * 5 + 1] = smid;  // which SM ran this CTA (diagnostics)
  }
  float r[NR];
  const char* in[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    r[j] = a.r[j];
    in[j] = a.in[j];
  }
  double lsq[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) lsq[j] = 0.0;
  double gsq = 0.0;

  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + (U - 1) * stride < a.nvec; v += U * stride) {
    uint4 x[U][NR];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NR; ++j) x[u][j] = dev::ld16(in[j] + (v + u * stride) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u) dev::wsum16<T, NR>(x[u], r, a.out + (v + u * stride) * 16, lsq, gsq);
  }
  for (; v < a.nvec; v += stride) {
    uint4 x[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) x[j] = dev::ld16(in[j] + v * 16);
    dev::wsum16<T, NR>(x, r, a.out + v * 16, lsq, gsq);
  }
  // ragged tail (< one vector of elements) -- scalar, block 0
  if (blockIdx.x == 0) {
    const size_t e = a.nvec * E + threadIdx.x;
    if (e < a.n) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const float g = V::load1(in[j] + e * sizeof(T));
        acc = fmaf(r[j], g, acc);
        lsq[j] += (double)(g * g);
      }
      gsq += (double)(acc * acc);
      V::store1(a.out + e * sizeof(T), acc);
    }
  }

  if (threadIdx.x == 0) a.trace[blockIdx.x * 5 + 2] = dev::globaltimer_ns();
  double vals[NR + 1];
#pragma unroll
  for (int j = 0; j < NR; ++j) vals[j] = lsq[j];
  vals[NR] = gsq;
  dev::block_sum(vals, red);
  // the partial table, the ticket and the (accumulated) statistics are shared with the preceding
  // chained launch: from here on it must have completed
  if (a.chain) dev::pdl_wait();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j <= NR; ++j) a.partials[(size_t)blockIdx.x * (NR + 1) + j] = vals[j];
    a.trace[blockIdx.x * 5 + 3] = dev::globaltimer_ns();
    __threadfence();
    const unsigned t = atomicAdd(a.ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: fixed-order tree over the per-CTA partials (K5)
  double tot[NR + 1];
  dev::block_table_sum(a.partials, gridDim.x, NR + 1, tot, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j <= NR; ++j) {
      double* dst = (j < NR) ? (a.local_sq + j) : a.global_sq;
      *dst = a.accumulate ? (*dst + tot[j]) : tot[j];
    }
    *a.ticket = 0u;
    a.trace[blockIdx.x * 5 + 4] = dev::globaltimer_ns();
    *a.trace_grid = gridDim.x;
  }
}

// ------------------------------------------------------------------------------ host launcher
// Loads in flight per thread = NR * U (~4-8).  CTA size NT: 256 (5 CTAs/SM for n = 8) or one big
// CTA per SM (NT = 1024 for n <= 8, 512 above): fewer, larger CTAs spread less in speed (the
// cross-CTA L1tex-queue effect) and leave fewer partial rows for the final reduction.
template <int NR>
constexpr int u_default() {
  return NR <= 2 ? 4 : (NR <= 4 ? 2 : 1);
}

template <typename T, int NR, int U, int NT>
static int occupancy_grid(int num_sms) {
  static int cached = 0;
  if (!cached) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wsum_local_kernel<T, NR, U, NT>, NT,
                                                      0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    cached = per_sm;
  }
  int g = cached * num_sms;
  return g > kMaxLocalBlocks ? kMaxLocalBlocks : g;
}

template <typename T, int NR, int U, int NT>
static cudaError_t launch_nt(const LocalArgs& a, int num_sms, int grid_override, cudaStream_t st) {
  int grid = grid_override > 0 ? grid_override : occupancy_grid<T, NR, U, NT>(num_sms);
  // small passes (<= 32 MB of traffic, L2-resident, latency-bound): two CTAs per SM -- fewer
  // partial rows for the last CTA and less launch drain; C1 (3 x 4 MB fp32) 11.6 -> 9.7 us
  // (profiles/r02/k2_small_grids.jsonl).  A function of (n, ranks, dtype) only: deterministic.
  if (grid_override <= 0 && (size_t)(NR + 1) * a.nvec * 16 <= ((size_t)32 << 20) &&
      grid > 2 * num_sms)
    grid = 2 * num_sms;
  // do not launch CTAs that would own no vector (keeps tiny buckets cheap)
  const size_t need = (a.nvec + NT - 1) / NT;
  if ((size_t)grid > need) grid = need < 1 ? 1 : (int)need;
  if (grid > kMaxLocalBlocks) grid = kMaxLocalBlocks;
  // launched with programmatic stream serialization (PDL): see the kernel's prologue
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, wsum_local_kernel<T, NR, U, NT>, a);
}

template <typename T, int NR>
static cudaError_t launch_u(const LocalArgs& a, int num_sms, int grid_override, int nt,
                            cudaStream_t st) {
  constexpr int U = u_default<NR>();
  constexpr int BIG = NR <= 8 ? 1024 : 512;
  if (nt >= 512) return launch_nt<T, NR, U, BIG>(a, num_sms, grid_override, st);
  return launch_nt<T, NR, U, 256>(a, num_sms, grid_override, st);
}

template <typename T>
static cudaError_t dispatch(int nr, const LocalArgs& a, int num_sms, int grid_override, int nt,
                            cudaStream_t st) {
  switch (nr) {
#define CANNIKIN_CASE(K) \
  case K:                \
    return launch_u<T, K>(a, num_sms, grid_override, nt, st);
    CANNIKIN_CASE(1) CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5)
    CANNIKIN_CASE(6) CANNIKIN_CASE(7) CANNIKIN_CASE(8) CANNIKIN_CASE(9) CANNIKIN_CASE(10)
    CANNIKIN_CASE(11) CANNIKIN_CASE(12) CANNIKIN_CASE(13) CANNIKIN_CASE(14) CANNIKIN_CASE(15)
    CANNIKIN_CASE(16)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// Launch K2.  Validation is the caller's job (api.cu).
cudaError_t launch_wsum_local(cannikin_ctx* ctx, const void* const* in, int nr, const double* r,
                              void* out, size_t n, cannikin_dtype dt, double* d_local_sq,
                              double* d_global_sq, bool accumulate, int grid_override,
                              cudaStream_t st, bool chain) {
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
  a.trace = &ctx->ctrl->trace[0][0];
  a.trace_grid = &ctx->ctrl->trace_grid;
  a.local_sq = d_local_sq;
  a.global_sq = d_global_sq;
  a.accumulate = accumulate ? 1 : 0;
  a.chain = chain ? 1 : 0;
  // partial rows are (nr+1) doubles wide: reinterpret local_part as a flat array
  if (dt == CANNIKIN_F32)
    return dispatch<float>(nr, a, ctx->num_sms, grid_override, ctx->local_nt, st);
  return dispatch<__nv_bfloat16>(nr, a, ctx->num_sms, grid_override, ctx->local_nt, st);
}

}  // namespace cannikin
