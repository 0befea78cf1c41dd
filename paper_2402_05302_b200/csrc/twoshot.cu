// K3: fused weighted all-reduce over NVLink peer memory (two-shot), with the GNS norm statistics.
//
// For W ranks, rank k owns the contiguous shard S_k of the bucket.  One kernel:
//   0. entry barrier: every CTA b publishes (r_k, bucket identity) and an epoch flag to CTA b of
//      every peer, then waits for theirs ("all g_j are ready");
//   1. reduce-scatter (row a2): for e in S_k, acc_e = sum_{j=0..W-1} r_j g_j[e] in fp32, reading
//      g_j from peer j's bucket over NVLink (Eq. 9), and in the same loop
//      L_k[j] = sum_{e in S_k} g_j[e]^2 (every rank's local norm on this shard, Eq. 10 input) and
//      Gg_k = sum_{e in S_k} acc_e^2;
//   2. all-gather (row a3): the reduced vector (rounded ONCE to the bucket dtype) is pushed into
//      every peer's bucket at the same place, so all ranks end with identical bits;
//   3. the CTA's W+1 norm partials are pushed into every peer's partial pad (row a4);
//   4. exit barrier: "my shard and partials have landed at every peer";
//   5. CTA b adds the W partial rows of CTA b (all ranks) in rank order to its running row;
//      cannikin_gns_stats sums the rows in CTA order -- identical bits on every rank (K5), and no
//      cross-CTA step inside the kernel.
// Only rank k ever reads or writes region S_k of any bucket, so two barriers suffice.  Flags are
// monotonically increasing epochs (no reset), making back-to-back buckets and CUDA-graph replay
// safe.  NVLink bytes per rank and direction: 2 (W-1)/W N s -- the ring all-reduce's volume
// (P:167), with the scaling and both norms fused at zero extra bytes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

struct ArArgs {
  char* bucket[kMaxWorld];  // this bucket as seen in each rank's mapping (own included)
  Ctrl* pctrl[kMaxWorld];   // control regions of all ranks (own included), mapped
  Ctrl* ctrl;               // own control region
  size_t nvec, n;           // full 16-byte vectors / elements
  size_t shard_lo, shard_hi;  // this rank's vector range
  uint64_t meta;            // identity of (offset, n, dtype, grid): must agree on every rank
  uint64_t timeout_ns;
  size_t chunk;             // dynamic variant: vectors per chunk
  size_t shard_len;         // vectors of shards 0..W-2 (the last shard: shard_len_last)
  size_t shard_len_last;
  double r_me;
  int rank;
  int check_r;              // CANNIKIN_INIT_CHECK_RATIOS: verify sum_j r_j == 1 on the device
};

constexpr int kArThreads = 512;

// sum_j r_j in double over the fp32 ratios the kernel uses: each is within 2^-24 relative of the
// caller's double, so a correct split sums to 1 within 2^-23.  A violation is recorded (code 7,
// reported as DOMAIN by cannikin_gns_stats / cannikin_device_status), not trapped.
template <int W>
__device__ __forceinline__ void check_ratios(const float* r, Ctrl* c) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) s += (double)r[j];
  if (fabs(s - 1.0) > 0x1p-23) {
    c->rsum_bad = s;
    atomicCAS(&c->error_code, 0, 7);
  }
}

__device__ __forceinline__ void spin_until(const uint64_t* flag, uint64_t ep, Ctrl* ctrl,
                                           uint64_t timeout_ns, int code) {
  dev::SpinClock clk;
  while (dev::ld_acquire_sys(flag) < ep)
    if (clk.expired(timeout_ns, 1023u, &ctrl->error_code, code)) return;  // peer never arrived
}

__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Spin until the low 32 bits of *word (an epoch tag) reach e32 (wrap-safe); returns the word.
__device__ __forceinline__ uint64_t spin_word(const uint64_t* word, uint32_t e32, Ctrl* ctrl,
                                              uint64_t timeout_ns, int code) {
  dev::SpinClock clk;
  uint64_t w;
  while ((int32_t)((uint32_t)(w = ld_relaxed_sys(word)) - e32) < 0)
    if (clk.expired(timeout_ns, 1023u, &ctrl->error_code, code)) break;
  return w;
}

// Entry barrier, executed by thread `tid` < W of CTA b for peer tid.  Each 64-bit word carries its
// own 32-bit epoch tag (r_rank or the bucket-identity hash in the high half), so the two words
// need no mutual ordering and no fence: the bucket contents were written by earlier kernels and
// are complete (in the owner's L2, the point of coherence for NVLink loads) at their kernel
// boundary.  The waiter reads r_tid and checks that every rank reduces the same bucket.
template <int W>
__device__ __forceinline__ void entry_barrier_thread(const ArArgs& a, int b, uint64_t ep,
                                                     float* s_r) {
  const int tid = threadIdx.x;
  const uint32_t e32 = (uint32_t)ep;
  const uint32_t m32 = (uint32_t)(a.meta ^ (a.meta >> 32));
  Ctrl* pc = a.pctrl[tid];
  dev::st_relaxed_sys_u64(&pc->rv_word[b][a.rank],
                          ((uint64_t)__float_as_uint((float)a.r_me) << 32) | e32);
  dev::st_relaxed_sys_u64(&pc->meta_word[b][a.rank], ((uint64_t)m32 << 32) | e32);
  const uint64_t wr = spin_word(&a.ctrl->rv_word[b][tid], e32, a.ctrl, a.timeout_ns, 1);
  const uint64_t wm = spin_word(&a.ctrl->meta_word[b][tid], e32, a.ctrl, a.timeout_ns, 1);
  s_r[tid] = __uint_as_float((uint32_t)(wr >> 32));
  if ((uint32_t)(wm >> 32) != m32) {
    // ranks disagree on bucket offset/size/dtype/grid: a usage error whose shard ranges would
    // differ between ranks (out-of-range peer accesses) -- stop the context, do not continue
    atomicExch(&a.ctrl->error_code, 2);
    __trap();
  }
}

template <typename T, int W>
__device__ __forceinline__ void reduce_vec(const uint4 (&x)[W], const float (&r)[W],
                                           char* const (&dst)[W], size_t off, double (&lsq)[W],
                                           double& gsq) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.0f;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    float g[E];
    V::unpack(x[j], g);
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
  const uint4 y = V::pack(acc);
#pragma unroll
  for (int j = 0; j < W; ++j) dev::st16(dst[j] + off, y);
}

template <typename T, int W, int U, int NT>
__device__ __forceinline__ void twoshot_body(const ArArgs& a, const int b, const int G) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  __shared__ double red[32 * (W + 1)];
  __shared__ double s_part[W + 1];
  __shared__ float s_r[W];
  __shared__ uint64_t s_ep;
  const int tid = threadIdx.x;
  // programmatic dependent launch (launch_pdl): the next call may be launched now; this one
  // waits for its predecessor before touching memory (profiles/r02/k3_pdl_all_ab.jsonl, k3_pdl_ab.jsonl)
  dev::pdl_launch_dependents();
  dev::pdl_wait();

  if (tid == 0) {
    s_ep = a.ctrl->epoch[b] + 1;
    a.ctrl->trace[b][0] = dev::globaltimer_ns();
  }
  __syncthreads();
  const uint64_t ep = s_ep;

  // ---- 0. entry barrier (+ exchange of r_j and the bucket identity)
  if (tid < W) entry_barrier_thread<W>(a, b, ep, s_r);
  __syncthreads();
  if (a.check_r && b == 0 && tid == 0) check_ratios<W>(s_r, a.ctrl);
  if (tid == 0) a.ctrl->trace[b][1] = dev::globaltimer_ns();

  float r[W];
  char* dst[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    r[j] = s_r[j];
    dst[j] = a.bucket[j];
  }
  double lsq[W];
#pragma unroll
  for (int j = 0; j < W; ++j) lsq[j] = 0.0;
  double gsq = 0.0;

  // ---- 1+2. reduce-scatter on S_rank, fused norms, push to every peer
  const size_t stride = (size_t)G * blockDim.x;
  size_t v = a.shard_lo + (size_t)b * blockDim.x + tid;
  for (; v + (U - 1) * stride < a.shard_hi; v += U * stride) {
    uint4 x[U][W];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < W; ++j) x[u][j] = dev::ld16(dst[j] + (v + u * stride) * 16);
#pragma unroll
    for (int u = 0; u < U; ++u) reduce_vec<T, W>(x[u], r, dst, (v + u * stride) * 16, lsq, gsq);
  }
  for (; v < a.shard_hi; v += stride) {
    uint4 x[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x[j] = dev::ld16(dst[j] + v * 16);
    reduce_vec<T, W>(x, r, dst, v * 16, lsq, gsq);
  }
  // ragged tail (< one vector of elements): owned by the last rank, CTA 0
  if (a.rank == W - 1 && b == 0) {
    const size_t e = a.nvec * E + tid;
    if (e < a.n) {
      float acc = 0.0f;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const float g = V::load1(dst[j] + e * sizeof(T));
        acc = fmaf(r[j], g, acc);
        lsq[j] += (double)(g * g);
      }
      gsq += (double)(acc * acc);
#pragma unroll
      for (int j = 0; j < W; ++j) V::store1(dst[j] + e * sizeof(T), acc);
    }
  }

  // ---- 3. per-CTA norm partials -> every peer's pad
  double vals[W + 1];
#pragma unroll
  for (int j = 0; j < W; ++j) vals[j] = lsq[j];
  vals[W] = gsq;
  dev::block_sum(vals, red);
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j <= W; ++j) s_part[j] = vals[j];
    a.ctrl->trace[b][2] = dev::globaltimer_ns();
  }
  __syncthreads();  // also: every data store of this CTA has been issued

  // ---- 4. exit barrier
  if (tid < W) {
    Ctrl* pc = a.pctrl[tid];
#pragma unroll
    for (int j = 0; j <= W; ++j) dev::st_relaxed_sys_f64(&pc->part[a.rank][b][j], s_part[j]);
    __threadfence_system();
    dev::st_release_sys(&pc->exit_[b][a.rank], ep);
    spin_until(&a.ctrl->exit_[b][tid], ep, a.ctrl, a.timeout_ns, 3);
  }
  __syncthreads();
  // ---- 5. CTA b now holds every rank's partial row b: add them, in rank order, to its own
  // running row (the same sequence of additions on every rank -> identical bits; no cross-CTA
  // step on the critical path).  cannikin_gns_stats sums the rows in fixed order.
  if (tid == 0) {
    a.ctrl->epoch[b] = ep;
    a.ctrl->trace[b][3] = dev::globaltimer_ns();
    double* acc = a.ctrl->cta_acc[b];
#pragma unroll
    for (int j = 0; j <= W; ++j) {
      double t = 0.0;
#pragma unroll
      for (int src = 0; src < W; ++src) t += __ldcg(&a.ctrl->part[src][b][j]);
      acc[j] = __ldcg(&acc[j]) + t;
    }
    a.ctrl->trace[b][4] = dev::globaltimer_ns();
    if (b == 0) a.ctrl->trace_grid = G;
  }
}

CANNIKIN_GROUP_ENTRY((typename T, int W, int U, int NT), (T, W, U, NT), (NT, 1), twoshot_kernel,
                     twoshot_group_kernel, twoshot_body, ArArgs)

// Dynamic variant of K3: identical protocol and arithmetic; the shard is cut into chunks that CTAs
// claim from a per-rank counter, and every chunk's W+1 norm partials form one row of the peers'
// partial tables (written by the W "flag" threads), so the statistics do not depend on which CTA
// did which chunk.  The exit barrier still pairs CTA b with CTA b of every peer: when all CTAs of
// this rank have passed it, every peer CTA -- hence every peer chunk and row -- is complete.
template <typename T, int W, int U>
__device__ __forceinline__ void twoshot_dyn_body(const ArArgs& a, const int b, const int G) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  constexpr int NT = kArThreads;
  __shared__ double red[32 * (W + 1)];
  __shared__ double s_part[W + 1];
  __shared__ float s_r[W];
  __shared__ uint64_t s_ep;
  __shared__ unsigned s_chunk[2];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  const bool has_tail = a.n > a.nvec * E;
  auto nchunks_of = [&](int src) -> unsigned {
    const size_t len = (src == W - 1) ? a.shard_len_last : a.shard_len;
    unsigned c = (unsigned)((len + a.chunk - 1) / a.chunk);
    if (src == W - 1 && c == 0 && has_tail) c = 1;
    return c;
  };
  const unsigned my_chunks = nchunks_of(a.rank);
  // programmatic dependent launch (launch_pdl): the next call may be launched now; this one
  // waits for its predecessor before touching memory (profiles/r02/k3_pdl_all_ab.jsonl, k3_pdl_ab.jsonl)
  dev::pdl_launch_dependents();
  dev::pdl_wait();

  if (tid == 0) {
    s_ep = a.ctrl->epoch[b] + 1;
    a.ctrl->trace[b][0] = dev::globaltimer_ns();
    s_chunk[0] = atomicAdd(&a.ctrl->ar_counter, 1u);
    s_chunk[1] = atomicAdd(&a.ctrl->ar_counter, 1u);
  }
  __syncthreads();
  const uint64_t ep = s_ep;
  if (tid < W) entry_barrier_thread<W>(a, b, ep, s_r);
  __syncthreads();
  if (a.check_r && b == 0 && tid == 0) check_ratios<W>(s_r, a.ctrl);
  if (tid == 0) a.ctrl->trace[b][1] = dev::globaltimer_ns();

  float r[W];
  char* dst[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    r[j] = s_r[j];
    dst[j] = a.bucket[j];
  }
  for (unsigned k = 0;; ++k) {
    const unsigned c = s_chunk[k & 1];
    if (c >= my_chunks) break;
    double lsq[W];
#pragma unroll
    for (int j = 0; j < W; ++j) lsq[j] = 0.0;
    double gsq = 0.0;
    const size_t v0 = a.shard_lo + (size_t)c * a.chunk;
    const size_t v1 = (v0 + a.chunk < a.shard_hi) ? v0 + a.chunk : a.shard_hi;
    size_t v = v0 + tid;
    for (; v + (U - 1) * NT < v1; v += U * NT) {
      uint4 x[U][W];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < W; ++j) x[u][j] = dev::ld16(dst[j] + (v + u * NT) * 16);
#pragma unroll
      for (int u = 0; u < U; ++u) reduce_vec<T, W>(x[u], r, dst, (v + u * NT) * 16, lsq, gsq);
    }
    for (; v < v1; v += NT) {
      uint4 x[W];
#pragma unroll
      for (int j = 0; j < W; ++j) x[j] = dev::ld16(dst[j] + v * 16);
      reduce_vec<T, W>(x, r, dst, v * 16, lsq, gsq);
    }
    if (a.rank == W - 1 && c == my_chunks - 1 && has_tail) {
      const size_t e = a.nvec * E + tid;
      if (e < a.n) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const float g = V::load1(dst[j] + e * sizeof(T));
          acc = fmaf(r[j], g, acc);
          lsq[j] += (double)(g * g);
        }
        gsq += (double)(acc * acc);
#pragma unroll
        for (int j = 0; j < W; ++j) V::store1(dst[j] + e * sizeof(T), acc);
      }
    }
    double vals[W + 1];
#pragma unroll
    for (int j = 0; j < W; ++j) vals[j] = lsq[j];
    vals[W] = gsq;
    dev::block_sum(vals, red);
    if (tid == 0) {
#pragma unroll
      for (int j = 0; j <= W; ++j) s_part[j] = vals[j];
      s_chunk[k & 1] = atomicAdd(&a.ctrl->ar_counter, 1u);
    }
    __syncthreads();
    if (tid < W) {
      Ctrl* pc = a.pctrl[tid];
#pragma unroll
      for (int j = 0; j <= W; ++j) dev::st_relaxed_sys_f64(&pc->part[a.rank][c][j], s_part[j]);
    }
  }
  if (tid == 0) a.ctrl->trace[b][2] = dev::globaltimer_ns();
  __syncthreads();  // every data and partial store of this CTA has been issued

  if (tid < W) {
    __threadfence_system();
    dev::st_release_sys(&a.pctrl[tid]->exit_[b][a.rank], ep);
    spin_until(&a.ctrl->exit_[b][tid], ep, a.ctrl, a.timeout_ns, 3);
  }
  __syncthreads();
  if (tid == 0) {
    a.ctrl->epoch[b] = ep;
    a.ctrl->trace[b][3] = dev::globaltimer_ns();
    __threadfence();
    s_last = (atomicAdd(&a.ctrl->ticket_ar, 1u) == G - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // fixed order: rank 0's chunk rows, then rank 1's, ...; thread t takes rows t, t+NT, ...
  double tot[W + 1];
#pragma unroll
  for (int j = 0; j <= W; ++j) tot[j] = 0.0;
  unsigned base = 0;
  for (int src = 0; src < W; ++src) {
    const unsigned nc = nchunks_of(src);
    for (unsigned i = tid; i < nc; i += NT) {
      const double* row = &a.ctrl->part[src][i][0];
#pragma unroll
      for (int j = 0; j <= W; ++j) tot[j] += __ldcg(row + j);
    }
    base += nc;
  }
  dev::block_sum(tot, red);
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j <= W; ++j) a.ctrl->stats[j] += tot[j];
    a.ctrl->ticket_ar = 0u;
    a.ctrl->ar_counter = 0u;
    a.ctrl->trace[b][4] = dev::globaltimer_ns();
    a.ctrl->trace_grid = G;
  }
}
CANNIKIN_GROUP_ENTRY((typename T, int W, int U), (T, W, U), (kArThreads, 1), twoshot_dyn_kernel,
                     twoshot_dyn_group_kernel, twoshot_dyn_body, ArArgs)

template <int W>
constexpr int u_default_ar() {
  return W <= 2 ? 4 : (W <= 4 ? 2 : 1);
}


// ============================================================================================
// Push variant of K3 (CANNIKIN_AR_PUSH=1): every NVLink transfer is a write.
//   1. scatter: CTA b of rank j writes its piece b of every other shard S_k into slot j of rank
//      k's staging area (reads local, writes remote) and accumulates |g_j|^2 on the way;
//   2. mid barrier: epoch-tagged (r_j | epoch) words with release semantics -- also carries r_j,
//      so no entry barrier is needed (the staging and the buckets are free once the previous
//      call's exit barrier passed);
//   3. reduce: CTA b of rank k sums its piece of S_k from its own bucket and the W-1 staging
//      slots (all LOCAL reads), fp32 in rank order, |g|^2, and pushes the result into every
//      peer's bucket;
//   4. partial rows [me][b] = {|g_me|^2 piece, |g|^2 piece}, exit barrier, fixed-order final sum.
// NVLink bytes per rank and direction: 2 (W-1)/W N s, as the pull variant, but no read requests.
// ============================================================================================
struct PushArgs {
  char* bucket[kMaxWorld];   // this bucket in every rank's mapping
  char* stage[kMaxWorld];    // staging area of every rank (mapped)
  Ctrl* pctrl[kMaxWorld];
  Ctrl* ctrl;
  size_t nvec, n, L;         // vectors, elements, vectors per shard (last: nvec - (W-1) L)
  size_t slot_vec;           // staging slot size in vectors (>= the largest shard)
  uint64_t meta;
  uint64_t timeout_ns;
  float r_me;
  int rank;
  int check_r;
};

template <typename T, int W, int U>
__device__ __forceinline__ void twoshot_push_body(const PushArgs& a, const int b, const int G) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  __shared__ double red[32 * (kMaxWorld + 1)];
  __shared__ double s_part[2];
  __shared__ float s_r[W];
  __shared__ uint64_t s_ep;
  __shared__ bool s_last;
  const int tid = threadIdx.x, NT = blockDim.x;
  auto shard_lo = [&](int k) -> size_t { return a.L * k; };
  auto shard_hi = [&](int k) -> size_t { return (k == W - 1) ? a.nvec : a.L * (k + 1); };
  // programmatic dependent launch (launch_pdl): the next call may be launched now; this one
  // waits for its predecessor before touching memory (profiles/r02/k3_pdl_all_ab.jsonl, k3_pdl_ab.jsonl)
  dev::pdl_launch_dependents();
  dev::pdl_wait();
  if (tid == 0) {
    s_ep = a.ctrl->epoch[b] + 1;
    a.ctrl->trace[b][0] = dev::globaltimer_ns();
  }
  __syncthreads();
  const uint64_t ep = s_ep;
  const uint32_t e32 = (uint32_t)ep;
  const size_t stride = (size_t)G * NT;

  // ---- 1. scatter my pieces of the other shards into their owners' staging slot `rank`
  double lsq = 0.0;
  const char* mine = a.bucket[a.rank];
  for (int kk = 1; kk < W; ++kk) {
    const int k = (a.rank + kk) % W;  // staggered start: not every rank hits the same peer first
    const size_t lo = shard_lo(k), hi = shard_hi(k);
    char* dst = a.stage[k] + ((size_t)a.rank * a.slot_vec - lo) * 16;
    size_t v = lo + (size_t)b * NT + tid;
    for (; v + (U - 1) * stride < hi; v += U * stride) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = dev::ld16(mine + (v + u * stride) * 16);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float g[E];
        V::unpack(x[u], g);
        float sq = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) sq = fmaf(g[e], g[e], sq);
        lsq += (double)sq;
        dev::st16(dst + (v + u * stride) * 16, x[u]);
      }
    }
    for (; v < hi; v += stride) {
      const uint4 x = dev::ld16(mine + v * 16);
      float g[E];
      V::unpack(x, g);
      float sq = 0.0f;
#pragma unroll
      for (int e = 0; e < E; ++e) sq = fmaf(g[e], g[e], sq);
      lsq += (double)sq;
      dev::st16(dst + v * 16, x);
    }
  }
  // own ragged tail (< one vector) -> |g_me|^2, read before the mid barrier: the last rank writes
  // the reduced tail into every bucket only after CTA 0 of every rank has passed it
  if (b == 0) {
    const size_t e = a.nvec * E + tid;
    if (e < a.n) {
      const float own = V::load1(mine + e * sizeof(T));
      lsq += (double)(own * own);
    }
  }
  __syncthreads();  // every scatter store of this CTA has been issued

  // ---- 2. mid barrier: (r_rank | epoch) with release, to every peer; r_j from every peer
  const uint32_t m32 = (uint32_t)(a.meta ^ (a.meta >> 32));
  if (tid < W) {
    Ctrl* pc = a.pctrl[tid];
    __threadfence_system();
    dev::st_relaxed_sys_u64(&pc->meta_word[b][a.rank], ((uint64_t)m32 << 32) | e32);
    dev::st_release_sys(&pc->pmid[b][a.rank],
                        ((uint64_t)__float_as_uint(a.r_me) << 32) | e32);
    uint64_t w;
    {
      dev::SpinClock clk;
      while ((int32_t)((uint32_t)(w = dev::ld_acquire_sys(&a.ctrl->pmid[b][tid])) - e32) < 0)
        if (clk.expired(a.timeout_ns, 1023u, &a.ctrl->error_code, 6)) break;
    }
    s_r[tid] = __uint_as_float((uint32_t)(w >> 32));
    const uint64_t wm = spin_word(&a.ctrl->meta_word[b][tid], e32, a.ctrl, a.timeout_ns, 2);
    if ((uint32_t)(wm >> 32) != m32) {
      atomicExch(&a.ctrl->error_code, 2);
      __trap();
    }
  }
  __syncthreads();
  if (a.check_r && b == 0 && tid == 0) check_ratios<W>(s_r, a.ctrl);
  if (tid == 0) a.ctrl->trace[b][1] = dev::globaltimer_ns();

  // ---- 3. reduce my shard's piece from local memory, push the result to every peer
  float r[W];
  char* dstb[W];
  const char* src[W];
  const size_t lo = shard_lo(a.rank), hi = shard_hi(a.rank);
#pragma unroll
  for (int j = 0; j < W; ++j) {
    r[j] = s_r[j];
    // destinations in staggered order (rank+1, rank+2, ...), rotated ONCE here so that the store
    // loop indexes the array statically (a per-vector (rank + jj) % W index spills it to local
    // memory)
    dstb[j] = a.bucket[(a.rank + j) % W];
    src[j] = (j == a.rank) ? a.bucket[a.rank] + lo * 16
                           : a.stage[a.rank] + (size_t)j * a.slot_vec * 16;
  }
  double gsq = 0.0;
  for (size_t v = lo + (size_t)b * NT + tid; v < hi; v += stride) {
    const size_t rel = v - lo;
    uint4 x[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x[j] = dev::ld16(src[j] + rel * 16);
    float acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = 0.0f;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      float g[E];
      V::unpack(x[j], g);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fmaf(r[j], g[e], acc[e]);
      if (j == a.rank) {
        float sq = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) sq = fmaf(g[e], g[e], sq);
        lsq += (double)sq;
      }
    }
    float gs = 0.0f;
#pragma unroll
    for (int e = 0; e < E; ++e) gs = fmaf(acc[e], acc[e], gs);
    gsq += (double)gs;
    const uint4 y = V::pack(acc);
#pragma unroll
    for (int jj = 0; jj < W; ++jj) dev::st16(dstb[jj] + v * 16, y);
  }
  // ragged element tail: the last rank's CTA 0 reduces it straight from the peers' buckets
  // (after the mid barrier every rank's tail elements are still unchanged source data)
  if (b == 0) {
    const size_t e = a.nvec * E + tid;
    if (e < a.n) {
      if (a.rank == W - 1) {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const float g = V::load1(a.bucket[j] + e * sizeof(T));
          acc = fmaf(r[j], g, acc);
        }
        gsq += (double)(acc * acc);
#pragma unroll
        for (int j = 0; j < W; ++j) V::store1(a.bucket[j] + e * sizeof(T), acc);
      }
    }
  }
  if (tid == 0) a.ctrl->trace[b][2] = dev::globaltimer_ns();

  // ---- 4. partial rows, exit barrier, final sum
  double vals[2] = {lsq, gsq};
  dev::block_sum(vals, red);
  if (tid == 0) {
    s_part[0] = vals[0];
    s_part[1] = vals[1];
  }
  __syncthreads();
  if (tid < W) {
    Ctrl* pc = a.pctrl[tid];
#pragma unroll
    for (int j = 0; j <= W; ++j) {
      const double x = (j == a.rank) ? s_part[0] : (j == W ? s_part[1] : 0.0);
      dev::st_relaxed_sys_f64(&pc->part[a.rank][b][j], x);
    }
    __threadfence_system();
    dev::st_release_sys(&pc->exit_[b][a.rank], ep);
    spin_until(&a.ctrl->exit_[b][tid], ep, a.ctrl, a.timeout_ns, 3);
  }
  __syncthreads();
  if (tid == 0) {
    a.ctrl->epoch[b] = ep;
    a.ctrl->trace[b][3] = dev::globaltimer_ns();
    __threadfence();
    s_last = (atomicAdd(&a.ctrl->ticket_ar, 1u) == G - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double tot[W + 1];
#pragma unroll
  for (int j = 0; j <= W; ++j) tot[j] = 0.0;
  for (int i = tid; i < W * G; i += NT) {
    const int sr = i / G, cta = i - sr * G;
    const double* row = &a.ctrl->part[sr][cta][0];
#pragma unroll
    for (int j = 0; j <= W; ++j) tot[j] += __ldcg(row + j);
  }
  dev::block_sum(tot, red);
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j <= W; ++j) a.ctrl->stats[j] += tot[j];
    a.ctrl->ticket_ar = 0u;
    a.ctrl->trace[b][4] = dev::globaltimer_ns();
    a.ctrl->trace_grid = G;
  }
}
CANNIKIN_GROUP_ENTRY((typename T, int W, int U), (T, W, U), (kArThreads, 1), twoshot_push_kernel,
                     twoshot_push_group_kernel, twoshot_push_body, PushArgs)

// Per-rank plan of a two-shot call: variant, grid and kernel arguments.  The variant and grid
// are functions of (n, dt, W, grid_ar) only, so every rank -- and every rank of an in-process
// group -- derives the same.
struct ArPlan {
  int kind;  // 0 static pull, 1 dynamic pull, 2 push
  int grid;
  ArArgs ar;
  PushArgs push;
};

static uint64_t bucket_meta(size_t off, size_t n, int grid, cannikin_dtype dt, uint64_t salt) {
  uint64_t meta = (uint64_t)off * 0x9E3779B97F4A7C15ull;
  meta ^= (uint64_t)n * 0xC2B2AE3D27D4EB4Full;
  return meta ^ ((uint64_t)grid << 8) ^ (uint64_t)dt ^ salt;
}

static void plan_push(const cannikin_ctx* ctx, size_t off, size_t n, cannikin_dtype dt, double r_i,
                      ArPlan* p) {
  const int W = ctx->world;
  PushArgs& a = p->push;
  a = PushArgs{};
  for (int j = 0; j < W; ++j) {
    a.bucket[j] = ctx->peer_base[j] + off;
    a.stage[j] = ctx->peer_base[j] + ctx->stage_off;
    a.pctrl[j] = reinterpret_cast<Ctrl*>(ctx->peer_base[j]);
  }
  a.ctrl = ctx->ctrl;
  const size_t esz = dt == CANNIKIN_F32 ? 4 : 2;
  a.n = n;
  a.nvec = n * esz / 16;
  size_t L = a.nvec / W;
  L -= L % 64;
  a.L = L;
  a.slot_vec = a.nvec - L * (size_t)(W - 1);  // the largest shard (the last rank's)
  int grid = ctx->grid_ar;
  const size_t want = (L + (size_t)kArThreads * 2 - 1) / ((size_t)kArThreads * 2);
  if (want < (size_t)grid) grid = want < 1 ? 1 : (int)want;
  a.meta = bucket_meta(off, n, grid, dt, 0x70757368ull);
  a.timeout_ns = ctx->spin_timeout_ns;
  a.r_me = (float)r_i;
  a.rank = ctx->rank;
  a.check_r = ctx->check_ratios;
  p->kind = 2;
  p->grid = grid;
}

static void plan_twoshot(const cannikin_ctx* ctx, size_t off, size_t n, cannikin_dtype dt,
                         double r_i, ArPlan* p) {
  const int W = ctx->world;
  {
    // push (all-write) pays for large buckets from 4 ranks up (W = 4: equal at 64 MB, +5% at
    // 256 MB-1 GB; profiles/r01/k3_pull_dyn_push_n4.jsonl); pull is better for small buckets and at
    // W = 2.  The threshold is on the bucket, not the shard, so that W = 8 (not measurable here)
    // sends C4's 220 MB bucket through the all-write pattern, which held up best under all-to-all
    // load at W = 4 (profiles/r01/nvlink_bw_n4.jsonl)
    const size_t bucket_bytes = n * (dt == CANNIKIN_F32 ? 4 : 2);
    const bool push = ctx->ar_push == 1 || (ctx->ar_push < 0 && W >= 4 && bucket_bytes >= kPushAutoBytes);
    if (push && ctx->stage_off) return plan_push(ctx, off, n, dt, r_i, p);
  }
  ArArgs& a = p->ar;
  a = ArArgs{};
  for (int j = 0; j < W; ++j) {
    a.bucket[j] = ctx->peer_base[j] + off;
    a.pctrl[j] = reinterpret_cast<Ctrl*>(ctx->peer_base[j]);
  }
  a.ctrl = ctx->ctrl;
  const size_t esz = dt == CANNIKIN_F32 ? 4 : 2;
  a.n = n;
  a.nvec = n * esz / 16;
  size_t L = a.nvec / W;
  L -= L % 64;  // shard boundaries on 1 KiB
  a.shard_lo = L * (size_t)ctx->rank;
  a.shard_hi = (ctx->rank == W - 1) ? a.nvec : L * (size_t)(ctx->rank + 1);
  // small buckets use fewer CTAs (>= ~2 vectors per thread): fewer flags to exchange and a smaller
  // final reduction.  A function of (n, W, grid) only, so every rank picks the same grid.
  int grid = ctx->grid_ar;
  const size_t per_cta = (size_t)kArThreads * 2;
  const size_t want = (L + per_cta - 1) / per_cta;
  if (want < (size_t)grid) grid = want < 1 ? 1 : (int)want;
  a.timeout_ns = ctx->spin_timeout_ns;
  a.r_me = r_i;
  a.rank = ctx->rank;
  a.check_r = ctx->check_ratios;
  // dynamic variant: chunks of the shard handed out by a per-rank atomic counter (balances the
  // per-CTA NVLink bandwidth spread); per-chunk partial rows keep the statistics deterministic
  // auto: dynamic chunks pay off for large shards (measured crossover ~32-128 MiB per shard)
  const bool dyn = ctx->ar_dyn < 0 ? (L * 16 >= (64ull << 20)) : (ctx->ar_dyn != 0);
  // ~4 chunks per CTA, between one vector per thread and 16 per thread, <= kMaxArChunks-1 chunks
  size_t chunk = (L + (size_t)grid * 4 - 1) / ((size_t)grid * 4);
  if (chunk > (size_t)ctx->ar_chunk_max) chunk = (size_t)ctx->ar_chunk_max;
  const size_t need = (L + kMaxArChunks - 2) / (kMaxArChunks - 1);
  if (need > chunk) chunk = need;
  chunk = (chunk + kArThreads - 1) / kArThreads * kArThreads;
  if (chunk < (size_t)kArThreads) chunk = kArThreads;
  a.chunk = chunk;
  a.shard_len_last = a.nvec - L * (size_t)(W - 1);
  a.shard_len = L;
  a.meta = bucket_meta(off, n, grid, dt, dyn ? (uint64_t)chunk * 0x94D049BB133111EBull : 0);
  p->kind = dyn ? 1 : 0;
  p->grid = grid;
}

template <typename T, int W>
static cudaError_t launch_plan(const ArPlan& p, cudaStream_t st) {
  constexpr int U = u_default_ar<W>();
  constexpr int UP = W <= 2 ? 4 : 2;
  if (p.kind == 0)
    return launch_pdl(twoshot_kernel<T, W, U, kArThreads>, dim3(p.grid), dim3(kArThreads), st, p.ar);
  if (p.kind == 1)
    return launch_pdl(twoshot_dyn_kernel<T, W, U>, dim3(p.grid), dim3(kArThreads), st, p.ar);
  return launch_pdl(twoshot_push_kernel<T, W, UP>, dim3(p.grid), dim3(kArThreads), st, p.push);
}

// p[0..W-1]: the plans of ranks 0..W-1 of an in-process group, one launch of W x grid CTAs
template <typename T, int W>
static cudaError_t launch_plan_group(const ArPlan* p, cudaStream_t st) {
  constexpr int U = u_default_ar<W>();
  constexpr int UP = W <= 2 ? 4 : 2;
  const int G = p[0].grid;
  if (p[0].kind == 2) {
    GroupArgs<PushArgs> g{};
    for (int k = 0; k < W; ++k) g.a[k] = p[k].push;
    g.grid = G;
    twoshot_push_group_kernel<T, W, UP><<<W * G, kArThreads, 0, st>>>(g);
  } else {
    GroupArgs<ArArgs> g{};
    for (int k = 0; k < W; ++k) g.a[k] = p[k].ar;
    g.grid = G;
    if (p[0].kind == 0) twoshot_group_kernel<T, W, U, kArThreads><<<W * G, kArThreads, 0, st>>>(g);
    else twoshot_dyn_group_kernel<T, W, U><<<W * G, kArThreads, 0, st>>>(g);
  }
  return cudaGetLastError();
}

template <typename T>
static cudaError_t dispatch_plan(int W, const ArPlan* p, bool group, cudaStream_t st) {
  switch (W) {
#define CANNIKIN_CASE(K) \
  case K:                \
    return group ? launch_plan_group<T, K>(p, st) : launch_plan<T, K>(*p, st);
    CANNIKIN_CASE(2) CANNIKIN_CASE(3) CANNIKIN_CASE(4) CANNIKIN_CASE(5) CANNIKIN_CASE(6)
    CANNIKIN_CASE(7) CANNIKIN_CASE(8)
#undef CANNIKIN_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// Launch K3 on the bucket at byte offset `off` of every rank's allocation.
cudaError_t launch_twoshot(cannikin_ctx* ctx, size_t off, size_t n, cannikin_dtype dt, double r_i,
                           cudaStream_t st) {
  ArPlan p;
  plan_twoshot(ctx, off, n, dt, r_i, &p);
  static const char* const kNames[3] = {"twoshot", "twoshot_dyn", "push"};
  ctx->last_variant = kNames[p.kind];
  if (dt == CANNIKIN_F32) return dispatch_plan<float>(ctx->world, &p, false, st);
  return dispatch_plan<__nv_bfloat16>(ctx->world, &p, false, st);
}

// The same for all W ranks of an in-process group in ONE launch (bucket at byte offset `off` of
// every rank's region; r[k] = rank k's share).
cudaError_t launch_twoshot_group(cannikin_ctx* const* ctxs, int W, size_t off, size_t n,
                                 cannikin_dtype dt, const double* r, cudaStream_t st) {
  ArPlan p[kMaxWorld];
  for (int k = 0; k < W; ++k) plan_twoshot(ctxs[k], off, n, dt, r[k], &p[k]);
  static const char* const kNames[3] = {"twoshot", "twoshot_dyn", "push"};
  ctxs[0]->last_variant = kNames[p[0].kind];
  if (dt == CANNIKIN_F32) return dispatch_plan<float>(W, p, true, st);
  return dispatch_plan<__nv_bfloat16>(W, p, true, st);
}

// Finalize the statistics of all calls since the last finalize: out[j] = stats[j] (dynamic / push
// two-shot, NVLS, world 1) + the sum over b of cta_acc[b][j] (static two-shot, LL, LL128), then
// zero both.  One thread per row b; the rows are summed by the fixed-order block reduction
// (butterfly within warps, warps in order), so every rank forms the same bits.  `out` may be
// device or pinned host memory.
__global__ void __launch_bounds__(kMaxArBlocks) stats_finalize_kernel(Ctrl* c, int W, double* out) {
  __shared__ double red[32 * (kMaxWorld + 1)];
  const int b = threadIdx.x;
  double v[kMaxWorld + 1];
#pragma unroll
  for (int j = 0; j <= kMaxWorld; ++j) {
    v[j] = (j <= W) ? __ldcg(&c->cta_acc[b][j]) : 0.0;
    if (j <= W) c->cta_acc[b][j] = 0.0;
  }
  dev::block_sum(v, red);
  if (b == 0) {
    for (int j = 0; j <= W; ++j) {
      out[j] = c->stats[j] + v[j];
      c->stats[j] = 0.0;
    }
  }
}

cudaError_t launch_stats_finalize(cannikin_ctx* ctx, double* out, cudaStream_t st) {
  stats_finalize_kernel<<<1, kMaxArBlocks, 0, st>>>(ctx->ctrl, ctx->world, out);
  return cudaGetLastError();
}

// Add W+1 held statistics back into the accumulator (cannikin_gns_stats_bucket keeps the fused
// statistics pending across its own out-of-place reduction).
__global__ void stats_add_kernel(Ctrl* c, int W, const double* in) {
  const int j = threadIdx.x;
  if (j <= W) c->stats[j] += in[j];
}

cudaError_t launch_stats_add(cannikin_ctx* ctx, const double* in, cudaStream_t st) {
  stats_add_kernel<<<1, 32, 0, st>>>(ctx->ctrl, ctx->world, in);
  return cudaGetLastError();
}

}  // namespace cannikin
