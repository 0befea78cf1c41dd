// K6: weighted all-reduce through NVSwitch multicast (NVLS) -- SURVEY §8(f) NEXT-4.
//
// Same contract as the two-shot kernel (K3): in place g = sum_j r_j g_j (Eq. 9)
// with |g_j|^2 and |g|^2 (Eq. 10 inputs) accumulated in the ctx, identical bits on every
// rank.  The bucket is a symmetric multicast-capable allocation (e.g. torch symmetric memory):
// `bucket` is this rank's copy, `mc` the multicast address of the same bytes.
//   A. each rank scales its own copy in place, y_i = r_i g_i (rounded to the bucket dtype), and
//      accumulates |g_i|^2 from the unscaled values -- local HBM only;
//   B. rank k pulls the in-switch sum of its shard, sum_j y_j = multimem.ld_reduce(mc + e)
//      (fp32 accumulation in the switch), accumulates |g|^2 and writes the result to every
//      rank's copy with one multimem.st;
//   C. per-CTA norm partials to every peer's pad, exit barrier;
//   D. CTA b adds the W rows b to its running statistics row (fixed rank order).
// NVLink bytes per rank and direction ~ (1 + 1/W) N s instead of the two-shot's 2 (W-1)/W N s
// (1.125 vs 1.75 at W = 8), at the price of a local N s read + write in phase A.
// The piece of every shard that CTA b scales in phase A is exactly the piece CTA b of the shard's
// owner reduces in phase B, so the barrier between A and B pairs CTA b with CTA b (as in K3).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

struct McArgs {
  char* local;              // this rank's copy
  char* mc;                 // multicast address of the bucket
  Ctrl* pctrl[kMaxWorld];   // control regions (ctx heap, IPC-mapped)
  Ctrl* ctrl;
  size_t nvec;              // 16-byte vectors (the NVLS path needs whole vectors)
  size_t L;                 // vectors per shard (last shard: nvec - (W-1) L)
  uint64_t meta;
  uint64_t timeout_ns;
  float r_me;
  int rank;
};

namespace mc {

__device__ __forceinline__ uint4 ld_reduce(const void* p, float) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_reduce(const void* p, __nv_bfloat16) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st(void* p, const uint4& v, float) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st(void* p, const uint4& v, __nv_bfloat16) {
  asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void wait_at_least(const uint64_t* flag, uint64_t ep, Ctrl* ctrl,
                                              uint64_t timeout_ns, int code) {
  dev::SpinClock clk;
  while (dev::ld_acquire_sys(flag) < ep)
    if (clk.expired(timeout_ns, 1023u, &ctrl->error_code, code)) return;
}

}  // namespace mc

template <typename T>
__global__ void __launch_bounds__(512, 1) nvls_kernel(const McArgs a, int W) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  constexpr int UA = 4;  // phase A: vectors in flight per thread
  constexpr int R = 4;   // phase B: in-switch reductions in flight per thread
  __shared__ double red[32 * 2];
  __shared__ double s_part[2];
  __shared__ uint64_t s_ep;
  const int b = blockIdx.x, tid = threadIdx.x, G = gridDim.x, NT = blockDim.x;
  auto shard_len = [&](int k) -> size_t { return (k == W - 1) ? a.nvec - a.L * (W - 1) : a.L; };
  // one epoch per call for every CTA (the mid barrier compares flags across CTA indices, so a
  // per-CTA epoch -- K3's -- would diverge when the grid changes between calls)
  if (tid == 0) {
    s_ep = __ldcg(&a.ctrl->nv_epoch) + 1;
    a.ctrl->trace[b][0] = dev::globaltimer_ns();
  }
  __syncthreads();
  const uint64_t ep = s_ep;
  const size_t stride = (size_t)G * NT;

  // ---- A. scale my copy in place over CTA b's piece of every shard; |g_me|^2 (local HBM)
  double lsq = 0.0;
  for (int k = 0; k < W; ++k) {
    const size_t lo = a.L * k, hi = lo + shard_len(k);
    size_t v = lo + (size_t)b * NT + tid;
    for (; v + (UA - 1) * stride < hi; v += UA * stride) {
      uint4 x[UA];
#pragma unroll
      for (int u = 0; u < UA; ++u) x[u] = dev::ld16(a.local + (v + u * stride) * 16);
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        float g[E];
        V::unpack(x[u], g);
        float sq = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          sq = fmaf(g[e], g[e], sq);
          g[e] = a.r_me * g[e];
        }
        lsq += (double)sq;
        dev::st16(a.local + (v + u * stride) * 16, V::pack(g));
      }
    }
    for (; v < hi; v += stride) {
      float g[E];
      V::unpack(dev::ld16(a.local + v * 16), g);
      float sq = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        sq = fmaf(g[e], g[e], sq);
        g[e] = a.r_me * g[e];
      }
      lsq += (double)sq;
      dev::st16(a.local + v * 16, V::pack(g));
    }
  }
  // publish "piece b scaled" to every peer (release: the switch reads my copy) and wait for
  // piece b of every rank: the piece of my shard that CTA b reduces below is scaled everywhere
  __syncthreads();
  if (tid < W) {
    // the bucket identity (size, dtype, grid) travels with the barrier: ranks that disagree would
    // pair different shard ranges, so a mismatch stops the context (code 2, as K3's entry check)
    const uint32_t m32 = (uint32_t)(a.meta ^ (a.meta >> 32));
    dev::st_relaxed_sys_u64(&a.pctrl[tid]->nv_meta[b][a.rank], ((uint64_t)m32 << 32) | (uint32_t)ep);
    __threadfence_system();
    dev::st_release_sys(&a.pctrl[tid]->mid[b][a.rank], ep);
    mc::wait_at_least(&a.ctrl->mid[b][tid], ep, a.ctrl, a.timeout_ns, 4);
    const uint64_t wm = dev::ld_acquire_sys(&a.ctrl->nv_meta[b][tid]);
    if ((uint32_t)wm == (uint32_t)ep && (uint32_t)(wm >> 32) != m32) {
      atomicExch(&a.ctrl->error_code, 2);
      __trap();
    }
  }
  __syncthreads();
  if (tid == 0) a.ctrl->trace[b][1] = dev::globaltimer_ns();

  // ---- B. CTA b's piece of my shard (grid-stride, the interleaving the switch serves best):
  // in-switch sum, |g|^2, multicast store to every copy
  double gsq = 0.0;
  {
    const size_t lo = a.L * a.rank, hi = lo + shard_len(a.rank);
    size_t v = lo + (size_t)b * NT + tid;
    for (; v + (R - 1) * stride < hi; v += R * stride) {
      uint4 x[R];
#pragma unroll
      for (int u = 0; u < R; ++u) x[u] = mc::ld_reduce(a.mc + (v + u * stride) * 16, T());
#pragma unroll
      for (int u = 0; u < R; ++u) {
        float f[E];
        V::unpack(x[u], f);
        float sq = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) sq = fmaf(f[e], f[e], sq);
        gsq += (double)sq;
        mc::st(a.mc + (v + u * stride) * 16, x[u], T());
      }
    }
    for (; v < hi; v += stride) {
      const uint4 x = mc::ld_reduce(a.mc + v * 16, T());
      float f[E];
      V::unpack(x, f);
      float sq = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) sq = fmaf(f[e], f[e], sq);
      gsq += (double)sq;
      mc::st(a.mc + v * 16, x, T());
    }
  }
  if (tid == 0) a.ctrl->trace[b][2] = dev::globaltimer_ns();
  // row [me][b]: this CTA's |g_me|^2 piece in column me, its |g|^2 piece in column W
  double vals[2] = {lsq, gsq};
  dev::block_sum(vals, red);
  if (tid == 0) {
    s_part[0] = vals[0];
    s_part[1] = vals[1];
  }
  __syncthreads();
  if (tid < W) {
    Ctrl* pc = a.pctrl[tid];
    for (int j = 0; j <= W; ++j) {
      const double x = (j == a.rank) ? s_part[0] : (j == W ? s_part[1] : 0.0);
      dev::st_relaxed_sys_f64(&pc->part[a.rank][b][j], x);
    }
  }
  __syncthreads();

  // ---- C. exit barrier, fixed-order final sum
  if (tid < W) {
    __threadfence_system();
    dev::st_release_sys(&a.pctrl[tid]->nv_exit[b][a.rank], ep);
    mc::wait_at_least(&a.ctrl->nv_exit[b][tid], ep, a.ctrl, a.timeout_ns, 5);
  }
  __syncthreads();
  // ---- D. CTA b holds every rank's row b: add them in rank order to its running row (as K3's
  // static variant; cannikin_gns_stats sums the rows in CTA order).  The call epoch advances
  // when the last CTA is done (every CTA read the old value at its start).
  if (tid == 0) {
    a.ctrl->trace[b][3] = dev::globaltimer_ns();
    double* acc = a.ctrl->cta_acc[b];
    for (int j = 0; j <= W; ++j) {
      double t = 0.0;
      for (int src = 0; src < W; ++src) t += __ldcg(&a.ctrl->part[src][b][j]);
      acc[j] = __ldcg(&acc[j]) + t;
    }
    a.ctrl->trace[b][4] = dev::globaltimer_ns();
    __threadfence();
    if (atomicAdd(&a.ctrl->ticket_ar, 1u) == gridDim.x - 1) {
      a.ctrl->ticket_ar = 0u;
      a.ctrl->nv_epoch = ep;
      a.ctrl->trace_grid = G;
    }
  }
}

// Launch K6.  `local` / `mc` are this rank's and the multicast address of the bucket.
cudaError_t launch_nvls(cannikin_ctx* ctx, void* local, void* mcp, size_t n, cannikin_dtype dt,
                        double r_i, cudaStream_t st) {
  const int W = ctx->world;
  McArgs a{};
  a.local = static_cast<char*>(local);
  a.mc = static_cast<char*>(mcp);
  for (int j = 0; j < W; ++j) a.pctrl[j] = reinterpret_cast<Ctrl*>(ctx->peer_base[j]);
  a.ctrl = ctx->ctrl;
  const size_t esz = dt == CANNIKIN_F32 ? 4 : 2;
  a.nvec = n * esz / 16;
  size_t L = a.nvec / W;
  L -= L % 64;
  a.L = L;
  int grid = ctx->grid_ar;
  const size_t want = (L + 1023) / 1024;
  if (want < (size_t)grid) grid = want < 1 ? 1 : (int)want;
  uint64_t meta = (uint64_t)n * 0xC2B2AE3D27D4EB4Full ^ ((uint64_t)grid << 8) ^ (uint64_t)dt ^ 0x6E766C73ull;
  a.meta = meta;
  a.timeout_ns = ctx->spin_timeout_ns;
  a.r_me = (float)r_i;
  a.rank = ctx->rank;
  if (dt == CANNIKIN_F32) nvls_kernel<float><<<grid, 512, 0, st>>>(a, W);
  else nvls_kernel<__nv_bfloat16><<<grid, 512, 0, st>>>(a, W);
  return cudaGetLastError();
}

}  // namespace cannikin
