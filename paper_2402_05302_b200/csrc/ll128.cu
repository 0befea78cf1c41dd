// K3-LL128: flag-in-line two-shot weighted all-reduce for mid-size buckets (the 2-64 MB part of
// SURVEY §8(d)'s C5 sweep, where the barrier-based two-shot pays ~15 us of handshakes per call).
//
// Same contract and arithmetic as every K3 variant: in place g = sum_j r_j g_j (Eq. 9,
// PAPER.md:328-331), fp32 fmaf accumulation in rank order from 0, one rounding to the bucket dtype
// (identical bits to the other variants), |g_j|^2 and |g|^2 (Eq. 10 inputs) into the
// per-CTA running rows (identical bits on every rank).
//
// Wire format: a warp moves a "group" of 512 bytes with ONE 16-byte store per lane: four 128-byte
// lines, each = 7 lanes x 16 payload bytes + 1 lane x {8 payload bytes, 8-byte flag}.  The flag is
// the call's 64-bit epoch.  A receiver loads the group with one 16-byte volatile load per lane and
// accepts it when all four flags match (warp vote); it relies on a 128-byte line written by one
// warp store arriving as one unit, which the GPU test suite checks bit for bit (every result is
// compared with the oracle and with the barrier-based variants).  Payload per group: 480 bytes
// (0.9375 of the wire bytes).
//
// Two-shot data flow without any barrier (shard k = groups [k G/W, (k+1) G/W) of the bucket):
//   1. scatter: CTA b of rank r sends its piece of every other shard k, raw, into slot (RS, r) of
//      rank k's LL128 region, and {r_r, epoch} in header entry b;
//   2. reduce: CTA b of rank r reduces its piece of shard r from its own bucket and the W-1 received
//      copies (rank order), writes the rounded result to its own bucket and sends it into slot
//      (AG, r) of every peer; its statistics row (W+1 doubles) goes to every peer's header entry b;
//   3. gather: CTA b copies the received pieces of every other shard into its own bucket, then sums
//      the W statistics rows of entry b (rank order) into cta_acc[b].
// Only the bucket of the calling rank is ever touched (no peer-mapped or staged bucket needed).
// Buffer reuse: call e uses parity e & 1.  A rank reaches call e + 2 only after receiving every
// peer's call-(e+1) result groups, which a peer sends only after its call e finished (stream
// order), so two parities need no "done" handshake.  Epoch: per-ctx call counter advanced by the
// last CTA of the grid (ticket), read by every CTA at its start.
// NVLink bytes per rank and direction: 2 (W-1)/W N s x 512/480.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

constexpr int kL8Threads = 512;
constexpr int kL8Warps = kL8Threads / 32;
constexpr size_t kGroupWire = 512;     // bytes on the wire per group
constexpr size_t kGroupPayload = 480;  // payload bytes per group
constexpr int kHdrWords = 2 + 2 * (kMaxWorld + 1);  // {r, e32}, then 2 halves per statistic
constexpr size_t kL8HeaderBytes = (size_t)2 * kMaxWorld * kMaxArBlocks * kHdrWords * 8;

struct LL128Args {
  char* bucket;           // own bucket (any device memory; only this rank touches it)
  char* reg[kMaxWorld];   // every rank's LL128 region (mapped)
  Ctrl* ctrl;
  size_t bytes;           // payload bytes n * s
  size_t ngroups;         // ceil(bytes / 480)
  size_t slot_bytes;      // one (parity, kind, source) data slot
  uint64_t timeout_ns;
  float r_me;
  int rank;
  int check_r;
};

__device__ __forceinline__ void st_vol16(void* p, const uint4& v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_vol16(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_word(void* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_word(const void* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin until the epoch half of the 8-byte header word at p equals e32 (timeout: error code 9,
// see dev::SpinClock).
__device__ __forceinline__ uint64_t wait_word(const void* p, uint32_t e32, Ctrl* ctrl,
                                              uint64_t timeout_ns) {
  uint64_t w = ld_word(p);
  dev::SpinClock clk;
  while ((uint32_t)(w >> 32) != e32) {
    if (clk.expired(timeout_ns, 1023u, &ctrl->error_code, 9)) break;
    w = ld_word(p);
  }
  return w;
}

// The flag lanes (lane % 8 == 7) carry the epoch in their upper 8 bytes.
__device__ __forceinline__ bool flag_ok(const uint4& v, bool flag_lane, uint64_t e) {
  return !flag_lane || ((((uint64_t)v.w) << 32) | v.z) == e;
}

// Wait until all four lines of the group at p carry epoch e (warp-uniform call).
__device__ __forceinline__ uint4 wait_group(const char* p, uint4 v, bool flag_lane, uint64_t e,
                                            Ctrl* ctrl, uint64_t timeout_ns) {
  dev::SpinClock clk;
  while (!__all_sync(0xffffffffu, flag_ok(v, flag_lane, e))) {
    // warp-uniform exit (the loop condition is a warp vote)
    if (__any_sync(0xffffffffu, clk.expired(timeout_ns, 255u, &ctrl->error_code, 9))) break;
    v = ld_vol16(p);
  }
  return v;
}

// This lane's payload of a group: 16 bytes (8 for a flag lane) at byte `off` of the bucket,
// zero-filled past the end (ragged tail: element-wise 2-byte copies).
__device__ __forceinline__ uint4 load_payload(const char* bucket, size_t bytes, size_t off,
                                              int pb) {
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (off + (size_t)pb <= bytes) {
    if (pb == 16) {
      v = dev::ld16(bucket + off);
    } else {
      const uint2 t = *reinterpret_cast<const uint2*>(bucket + off);
      v.x = t.x;
      v.y = t.y;
    }
  } else if (off < bytes) {
    uint16_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int m = (int)((bytes - off) / 2);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < m) h[i] = reinterpret_cast<const uint16_t*>(bucket + off)[i];
    v.x = h[0] | ((uint32_t)h[1] << 16);
    v.y = h[2] | ((uint32_t)h[3] << 16);
    v.z = h[4] | ((uint32_t)h[5] << 16);
    v.w = h[6] | ((uint32_t)h[7] << 16);
  }
  return v;
}

__device__ __forceinline__ void store_payload(char* bucket, size_t bytes, size_t off, int pb,
                                              const uint4& v) {
  if (off + (size_t)pb <= bytes) {
    if (pb == 16) {
      dev::st16(bucket + off, v);
    } else {
      *reinterpret_cast<uint2*>(bucket + off) = make_uint2(v.x, v.y);
    }
  } else if (off < bytes) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    const int m = (int)((bytes - off) / 2);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < m)
        reinterpret_cast<uint16_t*>(bucket + off)[i] = (uint16_t)(w[i >> 1] >> (16 * (i & 1)));
  }
}

template <typename T, int W>
__device__ __forceinline__ void ll128_body(const LL128Args& a, const int b, const int G) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  constexpr int NS = 2 * (W + 1);  // statistics words per row
  __shared__ double red[32 * (W + 1)];
  __shared__ float s_r[W];
  __shared__ uint32_t s_row[W][NS];
  __shared__ uint64_t s_e;
  __shared__ char* s_reg[W];  // peer regions (indexed by runtime rank: shared, not param space)
  __shared__ size_t s_h0[W], s_h1[W], s_lo[W];  // CTA b's piece of every shard, shard starts
  const int tid = threadIdx.x, me = a.rank;
  const int lane = tid & 31, warp = tid >> 5;
  // launched as a programmatic dependent (launch_pdl): let the next call's grid be launched now
  // (its CTAs become resident only as ours exit, and wait for our completion), and wait for the
  // preceding kernel -- the previous call, or whatever produced the bucket -- before anything.
  // Hides the launch latency between consecutive calls: 4 MB +3%, 25 MB +2% at W = 2
  // (profiles/r02/k3_pdl_ab.jsonl)
  dev::pdl_launch_dependents();
  dev::pdl_wait();
  if (tid == 0) {
    s_e = __ldcg(&a.ctrl->ll128_epoch) + 1;
    a.ctrl->trace[b][0] = dev::globaltimer_ns();
  }
#pragma unroll
  for (int j = 0; j < W; ++j)
    if (tid == j) s_reg[j] = a.reg[j];
  __syncthreads();
  const uint64_t e = s_e;
  const uint32_t e32 = (uint32_t)e;
  const size_t par = e & 1u;
  const bool fl = (lane & 7) == 7;
  const size_t poff = fl ? 448 + 8 * (lane >> 3) : 16 * ((lane >> 3) * 7 + (lane & 7));
  const int pb = fl ? 8 : 16;

  auto lo = [&](int k) -> size_t { return a.ngroups * (size_t)k / W; };
  auto data = [&](int k, int kind, int src) -> char* {
    return s_reg[k] + kL8HeaderBytes + ((par * 2 + kind) * W + src) * a.slot_bytes;
  };
  auto hdr = [&](int k, int src) -> char* {
    return s_reg[k] + (((par * kMaxWorld + src) * kMaxArBlocks) + b) * (size_t)(kHdrWords * 8);
  };
  // CTA b's piece of shard k: groups [g0, g1)
  auto piece = [&](int k, size_t& g0, size_t& g1) {
    const size_t l = lo(k), c = lo(k + 1) - l;
    g0 = l + c * (size_t)b / G;
    g1 = l + c * (size_t)(b + 1) / G;
  };

  // per-peer piece bounds live in shared memory (registers are the limit at large W)
  if (tid < W) {
    size_t h0, h1;
    piece(tid, h0, h1);
    s_h0[tid] = h0;
    s_h1[tid] = h1;
    s_lo[tid] = lo(tid);
  }
  __syncthreads();
  // Warp-sequence index t: this warp's t-th group of a piece is h0 + warp + t * 16.
  auto gcount = [&](int k) -> long {
    const size_t h0 = s_h0[k] + warp, h1 = s_h1[k];
    return h0 < h1 ? (long)((h1 - h0 + kL8Warps - 1) / kL8Warps) : 0;
  };
  long Tmax = 0;  // longest of the peers' pieces (scatter and gather run over the same pieces)
#pragma unroll 1
  for (int k = 0; k < W; ++k)
    if (k != me) Tmax = gcount(k) > Tmax ? gcount(k) : Tmax;
  constexpr int kGU = W <= 4 ? 2 : 1;  // steps of every peer in flight

  // ---- 1. scatter: raw pieces of the other shards (groups t < ns are sent), and r_me
  long ns = 0;
  auto scatter_to = [&](long tend) {
    while (ns < tend) {
      const int nu = (ns + kGU <= tend) ? kGU : 1;
      uint4 v[kGU][W];
#pragma unroll
      for (int u = 0; u < kGU; ++u)
#pragma unroll
        for (int jj = 1; jj < W; ++jj) {
          const int k = (me + jj) % W;
          const size_t g = s_h0[k] + warp + (size_t)(ns + u) * kL8Warps;
          if (u < nu && g < s_h1[k])
            v[u][jj] = load_payload(a.bucket, a.bytes, g * kGroupPayload + poff, pb);
        }
#pragma unroll
      for (int u = 0; u < kGU; ++u)
#pragma unroll
        for (int jj = 1; jj < W; ++jj) {
          const int k = (me + jj) % W;
          const size_t g = s_h0[k] + warp + (size_t)(ns + u) * kL8Warps;
          if (u >= nu || g >= s_h1[k]) continue;
          if (fl) {
            v[u][jj].z = e32;
            v[u][jj].w = (uint32_t)(e >> 32);
          }
          st_vol16(data(k, 0, me) + (size_t)lane * 16 + (g - s_lo[k]) * kGroupWire, v[u][jj]);
        }
      ns += nu;
    }
  };
  // the whole scatter first (sending only a few steps ahead of the reduction instead was measured
  // no faster in the automatic range and cost registers: DESIGN.md §6)
  if (tid < W && tid != me)
    st_word(hdr(tid, me), ((uint64_t)e32 << 32) | __float_as_uint(a.r_me));
  scatter_to(Tmax);
  if (tid == 0) a.ctrl->trace[b][1] = dev::globaltimer_ns();

  // ---- shares of every rank (header entry b of every source)
  if (tid < W) {
    if (tid == me) {
      s_r[tid] = a.r_me;
    } else {
      const uint64_t h = wait_word(hdr(me, tid), e32, a.ctrl, a.timeout_ns);
      s_r[tid] = __uint_as_float((uint32_t)h);
    }
  }
  __syncthreads();
  if (a.check_r && b == 0 && tid == 0) {
    double sr = 0.0;
#pragma unroll
    for (int j = 0; j < W; ++j) sr += (double)s_r[j];
    if (fabs(sr - 1.0) > 0x1p-23) {
      a.ctrl->rsum_bad = sr;
      atomicCAS(&a.ctrl->error_code, 0, 7);
    }
  }
  float r[W];
#pragma unroll
  for (int j = 0; j < W; ++j) r[j] = s_r[j];

  // ---- 2. reduce own shard: rank order, fp32 fmaf, one rounding; push the result to every peer
  double lsq[W];
#pragma unroll
  for (int j = 0; j < W; ++j) lsq[j] = 0.0;
  double gsq = 0.0;
  {
    size_t g0, g1;
    piece(me, g0, g1);
    const size_t l = lo(me);
    const char* src[W];
    char* dst[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      src[j] = data(me, 0, j) + (size_t)lane * 16;
      dst[j] = data((me + j) % W, 1, me) + (size_t)lane * 16;
    }
    // U groups per warp in flight (receive loads first, then the waits)
    auto step = [&](size_t g, auto uc) {
      constexpr int U = decltype(uc)::value;
      uint4 x[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t gu = g + (size_t)u * kL8Warps;
#pragma unroll
        for (int j = 0; j < W; ++j)
          x[u][j] = j != me ? ld_vol16(src[j] + (gu - l) * kGroupWire)
                            : load_payload(a.bucket, a.bytes, gu * kGroupPayload + poff, pb);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t gu = g + (size_t)u * kL8Warps;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if (j == me) continue;
          x[u][j] = wait_group(src[j] + (gu - l) * kGroupWire, x[u][j], fl, e, a.ctrl,
                               a.timeout_ns);
          if (fl) x[u][j].z = x[u][j].w = 0u;  // flag half: not payload
        }
        float acc[E];
#pragma unroll
        for (int q = 0; q < E; ++q) acc[q] = 0.0f;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          float f[E];
          V::unpack(x[u][j], f);
          float sq = 0.0f;
#pragma unroll
          for (int q = 0; q < E; ++q) {
            acc[q] = fmaf(r[j], f[q], acc[q]);
            sq = fmaf(f[q], f[q], sq);
          }
          lsq[j] += (double)sq;
        }
        {
          float sg = 0.0f;  // |g|^2 from the fp32 accumulator (as every variant)
#pragma unroll
          for (int q = 0; q < E; ++q) sg = fmaf(acc[q], acc[q], sg);
          gsq += (double)sg;
        }
        uint4 y = V::pack(acc);
        store_payload(a.bucket, a.bytes, gu * kGroupPayload + poff, pb, y);
        if (fl) {
          y.z = e32;
          y.w = (uint32_t)(e >> 32);
        }
#pragma unroll
        for (int jj = 1; jj < W; ++jj) st_vol16(dst[jj] + (gu - l) * kGroupWire, y);
      }
    };
    // ---- 3. (fused) gather the other shards' results into the own bucket, kLag steps behind the
    // reduction: the peers reduce their pieces at the same pace, so their groups have landed by
    // the time they are copied and the copy overlaps the NVLink traffic instead of following it.
    // Warp-sequence index t: this warp's t-th group of a piece is g0 + warp + t * 16.
    long ng = 0;  // groups t < ng are gathered
    auto gather_to = [&](long tend) {
      while (ng < tend) {
        const int nu = (ng + kGU <= tend) ? kGU : 1;
        uint4 v[kGU][W];
#pragma unroll
        for (int u = 0; u < kGU; ++u)
#pragma unroll
          for (int jj = 1; jj < W; ++jj) {
            const int k = (me + W - jj) % W;
            const size_t g = s_h0[k] + warp + (size_t)(ng + u) * kL8Warps;
            if (u < nu && g < s_h1[k])
              v[u][jj] = ld_vol16(data(me, 1, k) + (size_t)lane * 16 + (g - s_lo[k]) * kGroupWire);
          }
#pragma unroll
        for (int u = 0; u < kGU; ++u)
#pragma unroll
          for (int jj = 1; jj < W; ++jj) {
            const int k = (me + W - jj) % W;
            const size_t g = s_h0[k] + warp + (size_t)(ng + u) * kL8Warps;
            if (u >= nu || g >= s_h1[k]) continue;
            const char* q = data(me, 1, k) + (size_t)lane * 16 + (g - s_lo[k]) * kGroupWire;
            v[u][jj] = wait_group(q, v[u][jj], fl, e, a.ctrl, a.timeout_ns);
            store_payload(a.bucket, a.bytes, g * kGroupPayload + poff, pb, v[u][jj]);
          }
        ng += nu;
      }
    };
    constexpr int kU = W <= 4 ? 2 : 1;
    constexpr long kLag = 2 * kU;
    const long Tme = g0 + warp < g1 ? (long)((g1 - g0 - warp + kL8Warps - 1) / kL8Warps) : 0;
    long t = 0;
    for (; t + kU <= Tme; t += kU) {
      step(g0 + warp + (size_t)t * kL8Warps, std::integral_constant<int, kU>{});
      if (t + kU - kLag > ng) gather_to(t + kU - kLag < Tmax ? t + kU - kLag : Tmax);
    }
    for (; t < Tme; ++t) {
      step(g0 + warp + (size_t)t * kL8Warps, std::integral_constant<int, 1>{});
    }
    if (tid == 0) a.ctrl->trace[b][2] = dev::globaltimer_ns();
    // statistics row of (me, b) to every peer's header entry b (all reduction done)
    {
      double vals[W + 1];
#pragma unroll
      for (int j = 0; j < W; ++j) vals[j] = lsq[j];
      vals[W] = gsq;
      dev::block_sum(vals, red);
      if (tid == 0) {
#pragma unroll
        for (int j = 0; j <= W; ++j) {
          const unsigned long long u = __double_as_longlong(vals[j]);
          s_row[me][2 * j] = (uint32_t)u;
          s_row[me][2 * j + 1] = (uint32_t)(u >> 32);
        }
      }
      __syncthreads();
      if (tid < NS * W) {
        const int k = tid / NS, w = tid % NS;
        if (k != me) st_word(hdr(k, me) + 8 * (2 + w), ((uint64_t)e32 << 32) | s_row[me][w]);
      }
    }
    gather_to(Tmax);
  }
  if (tid == 0) a.ctrl->trace[b][3] = dev::globaltimer_ns();

  // ---- statistics: rows of entry b from every rank, summed in rank order (same bits everywhere)
  if (tid < NS * W) {
    const int k = tid / NS, w = tid % NS;
    if (k != me)
      s_row[k][w] = (uint32_t)wait_word(hdr(me, k) + 8 * (2 + w), e32, a.ctrl, a.timeout_ns);
  }
  __syncthreads();
  if (tid == 0) {
    double* acc = a.ctrl->cta_acc[b];
#pragma unroll
    for (int j = 0; j <= W; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k)
        s += __longlong_as_double((long long)(((uint64_t)s_row[k][2 * j + 1] << 32) | s_row[k][2 * j]));
      acc[j] = __ldcg(&acc[j]) + s;
    }
    a.ctrl->trace[b][4] = dev::globaltimer_ns();
    __threadfence();
    if (atomicAdd(&a.ctrl->ticket_ll128, 1u) == (unsigned)G - 1) {
      a.ctrl->ticket_ll128 = 0u;
      a.ctrl->ll128_epoch = a.ctrl->ll128_epoch + 1;
      a.ctrl->trace_grid = G;
    }
  }
}

CANNIKIN_GROUP_ENTRY((typename T, int W), (T, W), (kL8Threads, 1), ll128_kernel, ll128_group_kernel,
                     ll128_body, LL128Args)

// a[0] (single launch) or a[0..W-1] (in-process group: one launch of W x grid CTAs)
template <typename T>
static cudaError_t dispatch_ll128(int W, const LL128Args* a, int grid, bool group,
                                  cudaStream_t st) {
  switch (W) {
#define CANNIKIN_CASE(K)                                                     \
  case K:                                                                    \
    if (group) {                                                             \
      GroupArgs<LL128Args> g{};                                              \
      for (int k = 0; k < K; ++k) g.a[k] = a[k];                             \
      g.grid = grid;                                                         \
      ll128_group_kernel<T, K><<<K * grid, kL8Threads, 0, st>>>(g);          \
    } else {                                                                 \
      {                                                                      \
        cudaError_t e_ = launch_pdl(ll128_kernel<T, K>, dim3(grid), dim3(kL8Threads), st, a[0]); \
        if (e_ != cudaSuccess) return e_;                                    \
      }                                                                      \
    }                                                                        \
    return cudaGetLastError();
    CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5) CANNIKIN_CASE(6)
    CANNIKIN_CASE(7) CANNIKIN_CASE(8)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

static size_t ll128_slot_bytes(int world, size_t max_bytes) {
  const size_t groups = (max_bytes + kGroupPayload - 1) / kGroupPayload;
  return ((groups + world - 1) / world + 1) * kGroupWire;
}

size_t ll128_region_bytes(int world, size_t max_bytes) {
  return kL8HeaderBytes + (size_t)2 * 2 * world * ll128_slot_bytes(world, max_bytes);
}

// Automatic range (measured, profiles/r01/k3_ll128c_*): above the LL kernel's limit and up to
// 32 MiB: at W = 2 the two-shot wins from 64 MiB (567 vs 549 GB/s; 32 MiB 516 vs 504), at W = 4
// 32 MiB is a tie for heap buckets (540 vs 544; 16 MiB 504 vs 478) -- and a bucket outside the
// heap would cost the two-shot two staging copies, the LL128 kernel none (DDP's 25 MB buckets).
// The choice depends only on (bytes, world), never on where the bucket lives, so every rank
// picks the same kernel.  CANNIKIN_AR_LL128=1 extends it to the buffer size
// (CANNIKIN_LL128_MAX_MB, default: this range).
size_t ll128_auto_bytes(int) { return (size_t)32 << 20; }

bool ll128_eligible(const cannikin_ctx* ctx, size_t bytes) {
  if (ctx->world < 2 || !ctx->ll128_off || ctx->ar_ll128 == 0) return false;
  if (bytes > ctx->ll128_max_bytes) return false;
  if (ctx->ar_ll128 == 1) return true;
  return bytes <= ll128_auto_bytes(ctx->world) && (bytes > ctx->ll_max_bytes || ctx->ar_ll == 0);
}

static int plan_ll128(const cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt,
                      double r_i, LL128Args* out) {
  const int W = ctx->world;
  LL128Args& a = *out;
  a = LL128Args{};
  a.bucket = static_cast<char*>(bucket);
  for (int j = 0; j < W; ++j) a.reg[j] = ctx->peer_base[j] + ctx->ll128_off;
  a.ctrl = ctx->ctrl;
  a.bytes = n * (dt == CANNIKIN_F32 ? 4 : 2);
  a.ngroups = (a.bytes + kGroupPayload - 1) / kGroupPayload;
  a.slot_bytes = ll128_slot_bytes(W, ctx->ll128_max_bytes);
  a.timeout_ns = ctx->spin_timeout_ns;
  a.r_me = (float)r_i;
  a.rank = ctx->rank;
  a.check_r = ctx->check_ratios;
  // about one group per warp and phase (profiles/r01/k3_ll128_gpw_ab_n2.jsonl: 2 MB 192 vs 177
  // GB/s with two, 4-16 MB equal); every rank derives the same grid from (n, W)
  const size_t per_shard = (a.ngroups + W - 1) / W;
  size_t g = (per_shard + kL8Warps - 1) / kL8Warps;
  if (g < 1) g = 1;
  if (g > (size_t)ctx->grid_ar) g = (size_t)ctx->grid_ar;
  return (int)g;
}

cudaError_t launch_ll128(cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt, double r_i,
                         cudaStream_t st) {
  LL128Args a;
  const int g = plan_ll128(ctx, bucket, n, dt, r_i, &a);
  if (dt == CANNIKIN_F32) return dispatch_ll128<float>(ctx->world, &a, g, false, st);
  return dispatch_ll128<__nv_bfloat16>(ctx->world, &a, g, false, st);
}

cudaError_t launch_ll128_group(cannikin_ctx* const* ctxs, int W, void* const* buckets, size_t n,
                               cannikin_dtype dt, const double* r, cudaStream_t st) {
  LL128Args a[kMaxWorld];
  int g = 0;
  for (int k = 0; k < W; ++k) g = plan_ll128(ctxs[k], buckets[k], n, dt, r[k], &a[k]);
  if (dt == CANNIKIN_F32) return dispatch_ll128<float>(W, a, g, true, st);
  return dispatch_ll128<__nv_bfloat16>(W, a, g, true, st);
}

}  // namespace cannikin
