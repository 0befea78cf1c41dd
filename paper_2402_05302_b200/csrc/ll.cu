// K3-LL: low-latency weighted all-reduce for small buckets (the latency end of SURVEY §8(d)'s C5
// sweep; §8(e)'s "one-shot" idea with the flags folded into the data).
//
// Same contract and arithmetic as K3: in place g = sum_j r_j g_j (Eq. 9), fp32
// fmaf accumulation in rank order, one rounding to the bucket dtype (identical bits to every K3
// variant), |g_j|^2 and |g|^2 (Eq. 10 inputs) into the per-CTA running rows.
//
// Protocol (no barrier at all): every 4-byte payload word travels as one 8-byte store
// {payload, epoch32} into a slot of every peer's LL buffer, so a receiver knows a word has
// arrived when its epoch half matches -- data and flag are one NVLink transaction.  CTA b also
// publishes {r_rank, epoch32} in its slot header entry b.  Each rank then sums every word of the
// bucket from its own copy and the W-1 received copies (one-shot: every rank computes the same
// result and statistics by itself) and writes only its own bucket, which therefore does not have
// to be peer-mapped.
//   Buffer reuse: call e writes parity e & 1.  A peer can reach call e + 2 (same parity) only
// after receiving this rank's call-(e+1) words, which this rank sends only after its call e has
// finished reading -- so two parities suffice and no "done" handshake is needed.
//   Epoch: a per-ctx call counter read by every CTA at its start and advanced by the last CTA
// (ticket), so all CTAs and all ranks agree on it whatever the grid.
// NVLink bytes per rank and direction: 2 (W-1) N s -- the price of the folded flags; used only
// where latency, not bandwidth, decides.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

struct LLArgs {
  char* bucket;             // own bucket (any device memory; only this rank touches it)
  char* ll[kMaxWorld];      // every rank's LL region (mapped)
  Ctrl* ctrl;
  size_t n;                 // elements
  size_t nwords;            // 4-byte payload words (the last may be half a word for odd bf16 n)
  size_t slot_bytes;        // one (parity, source) slot: header + 8 bytes per word
  uint64_t timeout_ns;
  float r_me;
  int rank;
  int check_r;
};

constexpr int kLLThreads = 512;
constexpr size_t kLLHeader = 256 * 8;  // one {r, epoch} entry per CTA (grid <= 256)

__device__ __forceinline__ void st_ll(void* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_ll(const void* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin until the epoch half of the 8-byte word at p equals e32; returns the word.
__device__ __forceinline__ uint64_t wait_ll(const void* p, uint32_t e32, Ctrl* ctrl,
                                            uint64_t timeout_ns) {
  uint64_t w = ld_ll(p);
  if ((uint32_t)(w >> 32) == e32) return w;
  dev::SpinClock clk;
  while ((uint32_t)((w = ld_ll(p)) >> 32) != e32)
    if (clk.expired(timeout_ns, 1023u, &ctrl->error_code, 8)) break;  // a peer never sent
  return w;
}

// one 4-byte payload word <-> floats
template <typename T>
struct Word;
template <>
struct Word<float> {
  static constexpr int E = 1;
  __device__ static void unpack(uint32_t w, float (&f)[1]) { f[0] = __uint_as_float(w); }
  __device__ static uint32_t pack(const float (&f)[1]) { return __float_as_uint(f[0]); }
};
template <>
struct Word<__nv_bfloat16> {
  static constexpr int E = 2;
  __device__ static void unpack(uint32_t w, float (&f)[2]) {
    f[0] = __uint_as_float(w << 16);
    f[1] = __uint_as_float(w & 0xffff0000u);
  }
  __device__ static uint32_t pack(const float (&f)[2]) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[0], f[1]);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

template <typename T, int W>
__device__ __forceinline__ void ll_body(const LLArgs& a, const int b, const int G) {
  using Wd = Word<T>;
  constexpr int E = Wd::E;
  __shared__ double red[32 * (W + 1)];
  __shared__ float s_r[W];
  __shared__ uint32_t s_e;
  const int tid = threadIdx.x, me = a.rank;
  // programmatic dependent launch (launch_pdl): the next call may be launched now; this one
  // waits for its predecessor before touching memory (profiles/r02/k3_pdl_all_ab.jsonl, k3_pdl_ab.jsonl)
  dev::pdl_launch_dependents();
  dev::pdl_wait();
  if (tid == 0) {
    s_e = (uint32_t)(__ldcg(&a.ctrl->ll_epoch) + 1);
    a.ctrl->trace[b][0] = dev::globaltimer_ns();
  }
  __syncthreads();
  const uint32_t e32 = s_e;
  const size_t par = e32 & 1u;
  // slot (parity, source s) in rank k's region
  auto slot = [&](int k, int s) -> char* { return a.ll[k] + (par * W + s) * a.slot_bytes; };
  const bool half_tail = sizeof(T) == 2 && (a.n & 1);  // last word holds one bf16
  const size_t stride = (size_t)G * kLLThreads;

  // per-thread slot pointers, resolved once (the loops below index them statically)
  char* dstp[W];        // dstp[jj]: my slot in rank (me + jj) % W's region, jj = 1..W-1
  const char* srcp[W];  // srcp[j]: rank j's slot in my region
#pragma unroll
  for (int j = 0; j < W; ++j) {
    dstp[j] = slot((me + j) % W, me) + kLLHeader;
    srcp[j] = slot(me, j) + kLLHeader;
  }

  // ---- send: header entry b, then every word of CTA b's part, to every peer
  if (tid < W && tid != me)
    st_ll(slot(tid, me) + (size_t)b * 8, ((uint64_t)e32 << 32) | __float_as_uint(a.r_me));
  for (size_t w = (size_t)b * kLLThreads + tid; w < a.nwords; w += stride) {
    uint32_t mine;
    if (half_tail && w == a.nwords - 1)
      mine = *reinterpret_cast<const uint16_t*>(a.bucket + w * 4);
    else
      mine = *reinterpret_cast<const uint32_t*>(a.bucket + w * 4);
    const uint64_t v = ((uint64_t)e32 << 32) | mine;
#pragma unroll
    for (int jj = 1; jj < W; ++jj) st_ll(dstp[jj] + w * 8, v);
  }
  // ---- shares of every rank (header entry b of every source slot)
  if (tid < W) {
    if (tid == me) {
      s_r[tid] = a.r_me;
    } else {
      const uint64_t h = wait_ll(slot(me, tid) + (size_t)b * 8, e32, a.ctrl, a.timeout_ns);
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
  if (tid == 0) a.ctrl->trace[b][1] = dev::globaltimer_ns();
  float r[W];
#pragma unroll
  for (int j = 0; j < W; ++j) r[j] = s_r[j];

  // ---- receive + reduce: rank order, fp32 fmaf, one rounding
  double lsq[W];
#pragma unroll
  for (int j = 0; j < W; ++j) lsq[j] = 0.0;
  double gsq = 0.0;
  for (size_t w = (size_t)b * kLLThreads + tid; w < a.nwords; w += stride) {
    const bool ht = half_tail && w == a.nwords - 1;
    uint32_t x[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if (j == me) {
        x[j] = ht ? (uint32_t)*reinterpret_cast<const uint16_t*>(a.bucket + w * 4)
                  : *reinterpret_cast<const uint32_t*>(a.bucket + w * 4);
      } else {
        x[j] = (uint32_t)wait_ll(srcp[j] + w * 8, e32, a.ctrl, a.timeout_ns);
      }
    }
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.0f;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      float g[E];
      Wd::unpack(x[j], g);
      float sq = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        acc[e] = fmaf(r[j], g[e], acc[e]);
        sq = fmaf(g[e], g[e], sq);
      }
      lsq[j] += (double)sq;
    }
    float gs = 0.0f;
#pragma unroll
    for (int e = 0; e < E; ++e) gs = fmaf(acc[e], acc[e], gs);
    gsq += (double)gs;
    const uint32_t y = Wd::pack(acc);
    if (ht)
      *reinterpret_cast<uint16_t*>(a.bucket + w * 4) = (uint16_t)y;
    else
      *reinterpret_cast<uint32_t*>(a.bucket + w * 4) = y;
  }
  // ---- statistics: CTA b's running row (identical on every rank); epoch advance by the last CTA
  double vals[W + 1];
#pragma unroll
  for (int j = 0; j < W; ++j) vals[j] = lsq[j];
  vals[W] = gsq;
  dev::block_sum(vals, red);
  if (tid == 0) {
    double* acc = a.ctrl->cta_acc[b];
#pragma unroll
    for (int j = 0; j <= W; ++j) acc[j] = __ldcg(&acc[j]) + vals[j];
    a.ctrl->trace[b][2] = a.ctrl->trace[b][3] = a.ctrl->trace[b][4] = dev::globaltimer_ns();
    __threadfence();
    if (atomicAdd(&a.ctrl->ticket_ll, 1u) == G - 1) {
      a.ctrl->ticket_ll = 0u;
      a.ctrl->ll_epoch = a.ctrl->ll_epoch + 1;
      a.ctrl->trace_grid = G;
    }
  }
}

CANNIKIN_GROUP_ENTRY((typename T, int W), (T, W), (kLLThreads, 1), ll_kernel, ll_group_kernel,
                     ll_body, LLArgs)

// a[0] (single launch) or a[0..W-1] (in-process group: one launch of W x grid CTAs)
#define LL_LAUNCH_ONE(K)                                                                    \
  {                                                                                         \
    cudaError_t e_ = launch_pdl(ll_kernel<T, K>, dim3(grid), dim3(kLLThreads), st, a[0]);   \
    if (e_ != cudaSuccess) return e_;                                                       \
  }

template <typename T>
static cudaError_t dispatch_ll(int W, const LLArgs* a, int grid, bool group, cudaStream_t st) {
  switch (W) {
#define CANNIKIN_CASE(K)                                                     \
  case K:                                                                    \
    if (group) {                                                             \
      GroupArgs<LLArgs> g{};                                                 \
      for (int k = 0; k < K; ++k) g.a[k] = a[k];                             \
      g.grid = grid;                                                         \
      ll_group_kernel<T, K><<<K * grid, kLLThreads, 0, st>>>(g);             \
    } else {                                                                 \
      LL_LAUNCH_ONE(K);                                                      \
    }                                                                        \
    return cudaGetLastError();
    CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5) CANNIKIN_CASE(6)
    CANNIKIN_CASE(7) CANNIKIN_CASE(8)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// The LL kernel's NVLink bytes, 2 (W-1) N s per direction, grow with W while the two-shot's do
// not.  Against the barrier two-shot it won up to ~2 MiB / (W-1) (profiles/r01/k3_ll_n{2,4}.jsonl);
// against the LL128 two-shot (no barrier either, 1.07 N s) only up to ~1 MiB / (W-1): W = 2
// 1 MB 10.3 vs 9.9 us, 2 MB 13.9 vs 11.2; W = 4 0.25 MB 11.8 vs 13.9, 0.5 MB 14.6 vs 14.3
// (profiles/r01/k3_ll128os_f32_n{2,4}.jsonl, measured alongside the since-removed one-shot LL128
// variant).  The limit also sizes the LL buffers.
size_t ll_max_bytes(int world) {
  size_t m = ((size_t)1 << 20) / (size_t)(world > 1 ? world - 1 : 1);
  return m / (64u << 10) * (64u << 10);
}

static size_t ll_slot_bytes(size_t max_bytes) { return kLLHeader + max_bytes / 4 * 8; }

size_t ll_region_bytes(int world) { return (size_t)2 * world * ll_slot_bytes(ll_max_bytes(world)); }

bool ll_eligible(const cannikin_ctx* ctx, size_t bytes) {
  if (ctx->world < 2 || !ctx->ll_off || ctx->ar_ll == 0) return false;
  return bytes <= ctx->ll_max_bytes;
}

static int plan_ll(const cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt, double r_i,
                   LLArgs* out) {
  const int W = ctx->world;
  LLArgs& a = *out;
  a = LLArgs{};
  a.bucket = static_cast<char*>(bucket);
  for (int j = 0; j < W; ++j) a.ll[j] = ctx->peer_base[j] + ctx->ll_off;
  a.ctrl = ctx->ctrl;
  const size_t esz = dt == CANNIKIN_F32 ? 4 : 2;
  a.n = n;
  a.nwords = (n * esz + 3) / 4;
  a.slot_bytes = ll_slot_bytes(ctx->ll_max_bytes);
  a.timeout_ns = ctx->spin_timeout_ns;
  a.r_me = (float)r_i;
  a.rank = ctx->rank;
  a.check_r = ctx->check_ratios;
  size_t g = (a.nwords + kLLThreads - 1) / kLLThreads;
  if (g < 1) g = 1;
  if (g > (size_t)ctx->grid_ar) g = (size_t)ctx->grid_ar;
  return (int)g;
}

cudaError_t launch_ll(cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt, double r_i,
                      cudaStream_t st) {
  LLArgs a;
  const int g = plan_ll(ctx, bucket, n, dt, r_i, &a);
  if (dt == CANNIKIN_F32) return dispatch_ll<float>(ctx->world, &a, g, false, st);
  return dispatch_ll<__nv_bfloat16>(ctx->world, &a, g, false, st);
}

cudaError_t launch_ll_group(cannikin_ctx* const* ctxs, int W, void* const* buckets, size_t n,
                            cannikin_dtype dt, const double* r, cudaStream_t st) {
  LLArgs a[kMaxWorld];
  int g = 0;
  for (int k = 0; k < W; ++k) g = plan_ll(ctxs[k], buckets[k], n, dt, r[k], &a[k]);
  if (dt == CANNIKIN_F32) return dispatch_ll<float>(W, a, g, true, st);
  return dispatch_ll<__nv_bfloat16>(W, a, g, true, st);
}

}  // namespace cannikin
