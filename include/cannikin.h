/*
 * cannikin.h -- C ABI of the B200-native data-parallel hot path of Cannikin (arXiv 2402.05302).
 *
 * The library (libcannikin.so, sm_100a) implements, per training step:
 *   - the weighted gradient aggregation  g = sum_i r_i g_i,  r_i = b_i / B
 *       (§4.3 Eq. 9; r_i defined at P:151, §3.1),
 *   - in the same pass the squared norms |g_i|^2 of every rank's local mean gradient g_i (Eq. 1,
 *     P:125-130) and |g|^2 of the aggregate -- the inputs of Eq. 10,
 *   - on the host, the heterogeneous gradient-noise-scale estimator (Eq. 10, Theorem 1 / Eq. 11,
 *     B_noise = S/G),
 *   - on the host, the exact local-batch split r_opt that minimises the Eq. 7 batch time
 *     (§3; Alg. 1; integer batches P:419-420).
 *
 * Conventions shared by every call
 *   - No CUDA, NCCL or torch types appear here.  `stream` is a cudaStream_t passed as void*
 *     (NULL = the legacy default stream).  "device pointer" = CUDA global memory of the ctx's
 *     device; "host pointer" = ordinary CPU memory.
 *   - Every call returns a cannikin_status and never throws or aborts across the ABI.  Arguments
 *     are validated before anything is enqueued; on failure nothing was launched and
 *     cannikin_last_error() returns a thread-local message.
 *   - Ownership: the caller owns buckets (unless allocated with cannikin_alloc_bucket), streams and
 *     all output buffers.  A ctx owns its NCCL communicator, the peer-mapped symmetric heap, the
 *     signal/partial pads, scratch and the norm-statistics accumulator; it must outlive every
 *     operation enqueued on it.  Calls on one ctx must be ordered on one stream (or externally
 *     synchronised).
 *   - Determinism: for a fixed ctx grid, device results are bitwise reproducible run to run, and in
 *     the multi-GPU path bitwise identical on every rank.
 *   - Precision: fp32 or bf16 gradients; every sum over ranks is accumulated in fp32 in fixed rank
 *     order 0..n-1 and rounded once to the bucket dtype; squared norms are accumulated per thread
 *     in fp32 over one 16-byte vector and in fp64 beyond, then reduced by a fixed-order fp64 tree.
 */
#ifndef CANNIKIN_H
#define CANNIKIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CANNIKIN_VERSION 10000      /* 1.0.0 */
#define CANNIKIN_MAX_WORLD 8        /* ranks of one NVSwitch box */
#define CANNIKIN_MAX_EMULATED 16    /* emulated ranks of cannikin_weighted_sum_local */
#define CANNIKIN_MAX_GNS_NODES 64

typedef enum {
  CANNIKIN_OK = 0,
  CANNIKIN_ERR_INVALID = 1,     /* null pointer, size/alignment/limit violation, bad handle      */
  CANNIKIN_ERR_DOMAIN = 2,      /* value outside the model's domain (gamma, b_i, negative coeff.) */
  CANNIKIN_ERR_INFEASIBLE = 3,  /* sum(lo) > B or sum(cap) < B                                    */
  CANNIKIN_ERR_SINGULAR = 4,    /* singular Theorem-1 matrix, or a node time independent of b     */
  CANNIKIN_ERR_CUDA = 5,        /* CUDA runtime error (text in cannikin_last_error)                */
  CANNIKIN_ERR_NCCL = 6,        /* NCCL error                                                     */
  CANNIKIN_ERR_UNSUPPORTED = 7  /* dtype / rank count / feature not built                         */
} cannikin_status;

typedef enum { CANNIKIN_F32 = 0, CANNIKIN_BF16 = 1 } cannikin_dtype;

typedef struct cannikin_ctx cannikin_ctx; /* opaque; one per (process, device) */

/* Thread-local text of the last failure on this thread ("" if none).  Never NULL. */
const char* cannikin_last_error(void);
int cannikin_version(void);

/* ------------------------------------------------------------------------------------------
 * Lifecycle
 * ------------------------------------------------------------------------------------------ */

/* Writes a 128-byte NCCL unique id to `out_id` (host).  Call on rank 0 only, then broadcast the
 * bytes to every rank over the caller's own process group (e.g. torch.distributed). */
cannikin_status cannikin_get_unique_id(void* out_id);

/* Create a ctx for `rank` of `world` (1 <= world <= CANNIKIN_MAX_WORLD) on CUDA `device`.
 * world == 1: no communicator is created and `unique_id` may be NULL (single-GPU use:
 *   cannikin_weighted_sum_local, host solvers, and a trivial weighted_allreduce).
 * world  > 1: COLLECTIVE -- every rank calls it with the same unique_id and heap_bytes.  It
 *   creates an NCCL communicator, allocates `heap_bytes` of device memory (the symmetric heap) plus
 *   a control region, and maps every peer's heap into this process over NVLink (CUDA IPC handles
 *   exchanged through NCCL).  Buckets carved from the heap (cannikin_alloc_bucket) are reduced
 *   zero-copy; other device buffers are staged through a heap scratch area of the same size.
 * `grid` (0 = default 148) fixes the CTA count of the reduction kernels (determinism contract).
 * `flags`: 0, or CANNIKIN_INIT_CHECK_RATIOS -- every weighted_allreduce checks on the device that
 *   the ranks' shares sum to 1 (SURVEY §8(b) "ratio check"): sum_j r_j is formed in double from
 *   the fp32 shares the kernel multiplies with (each within 2^-24 relative of the caller's value)
 *   and must lie within 2^-23 of 1.  A violation does not stop the reduction; it is reported as
 *   DOMAIN by the next cannikin_gns_stats or cannikin_device_status.  Free (one comparison in one
 *   thread); not applied by the NVLS variant, which exchanges no shares.
 * `flags` may also include CANNIKIN_INIT_GATED_ENTRY (world > 1; ignored for world == 1): every
 *   cannikin_weighted_allreduce first enqueues a one-warp gate kernel that waits until every peer
 *   has reached the same call, and only then the reduction kernel.  For reductions that overlap
 *   the rank's own compute under heterogeneous ranks: a fast rank's wait for a slow
 *   peer then holds one SM slot of 32 threads instead of the reduction grid.  Costs one extra
 *   launch and a round trip per call, ~4 us on 2 B200 with no late peer
 *   (cannikin_last_launch_count counts it).  The gate's st.release.sys / ld.acquire.sys also
 *   make the bucket's contents ordered before the peers' reads by the memory model.  Applies to
 *   cannikin_weighted_allreduce (not the _nccl / _nvls paths).  Every rank of a communicator must
 *   use the same setting.
 * Peer waits: the reduction kernels wait for their peers on the device.  CANNIKIN_SPIN_TIMEOUT_MS
 *   (environment, read here): unset or 0 = wait as long as it takes (as NCCL does: a peer may be
 *   late for a checkpoint or a data load); > 0 = after that long a waiting kernel stops waiting,
 *   records a protocol error (that call's results are invalid) and finishes -- the next
 *   cannikin_gns_stats / cannikin_device_status reports it as CUDA.  Never a trap.  (Exception:
 *   ranks reducing different buckets -- a usage error whose shard ranges would disagree -- trap.)
 * Errors: INVALID (rank/world/device out of range, out == NULL, unknown flag), CUDA, NCCL. */
#define CANNIKIN_INIT_CHECK_RATIOS 1u
#define CANNIKIN_INIT_GATED_ENTRY 2u

cannikin_status cannikin_init(cannikin_ctx** out, int rank, int world, const void* unique_id,
                              int device, size_t heap_bytes, int grid, unsigned flags);

/* In-process group on ONE device (test and single-GPU use of the multi-GPU kernels): creates
 * `world` contexts out[0..world-1], ranks 0..world-1, in this process, each with its own region
 * and the others' regions as its "peers" (same address space: no IPC, no NCCL).  `grid` is
 * required and world * grid must not exceed the SM count (the ranks' kernels spin on their peer
 * CTAs, so all must be resident at once).  Two ways to reduce:
 *   - cannikin_weighted_allreduce_group (preferred): all ranks in ONE kernel launch, co-resident
 *     by construction -- also under a profiler that serialises kernels;
 *   - cannikin_weighted_allreduce per ctx, each rank on its own stream, issued concurrently (as
 *     W processes would); relies on the W kernels running at the same time (a serialising
 *     profiler breaks that: the first kernel waits for its peers until CANNIKIN_SPIN_TIMEOUT_MS,
 *     default 20000 for these contexts, and then reports a protocol error).
 * cannikin_ddp_allreduce_mean is UNSUPPORTED on such contexts; each is destroyed separately.
 * Errors: INVALID (world outside 2..CANNIKIN_MAX_WORLD, grid <= 0, unknown flag), CUDA. */
cannikin_status cannikin_init_group_local(cannikin_ctx** out, int world, int device,
                                          size_t heap_bytes, int grid, unsigned flags);

/* cannikin_weighted_allreduce for ALL ranks of an in-process group in one call (Eq. 9,
 * P:328-331; the Eq. 10 norm inputs, accumulated in every rank's ctx):
 *   ctxs[k]    : rank k's ctx of ONE cannikin_init_group_local group, k = 0..world-1
 *   buckets[k] : rank k's bucket (device pointer, n elements of dt, 16-byte aligned); each is
 *                overwritten with g = sum_j r[j] buckets[j], identical bits in every bucket
 *   r[k]       : rank k's share b_k / B (host array)
 * The variant (LL, LL128, two-shot pull / dynamic / push) is chosen from (n, dt, world) exactly as
 * cannikin_weighted_allreduce chooses it, and its kernel runs as ONE grid of world x G CTAs (CTA
 * c plays rank c / G's CTA c % G), enqueued on `stream`.  The result bits and statistics are those
 * of world separate per-rank calls.  Buckets at the same heap offset of every rank are reduced
 * zero-copy, others staged through each rank's scratch (two copies per rank).  Errors: INVALID
 * (NULL, misaligned, too large, ctxs not one group in rank order), UNSUPPORTED (dtype), DOMAIN
 * (NaN share), CUDA. */
cannikin_status cannikin_weighted_allreduce_group(cannikin_ctx* const* ctxs, int world,
                                                  void* const* buckets, size_t n,
                                                  cannikin_dtype dt, const double* r,
                                                  void* stream);

/* Destroy a ctx (synchronises its device first).  NULL is accepted and ignored. */
cannikin_status cannikin_destroy(cannikin_ctx* ctx);

/* COLLECTIVE for world > 1: every rank must issue the same sequence of alloc/free calls with the
 * same sizes; the returned buffers then sit at the same heap offset on every rank, which is what
 * lets the reduction kernel address a peer's copy.  Alignment: 256 bytes.  Errors: INVALID (no
 * space, bytes == 0). */
cannikin_status cannikin_alloc_bucket(cannikin_ctx* ctx, size_t bytes, void** dptr);
cannikin_status cannikin_free_bucket(cannikin_ctx* ctx, void* dptr);

/* ------------------------------------------------------------------------------------------
 * Hot path (device, stream-ordered, no host synchronisation)
 * ------------------------------------------------------------------------------------------ */

/* Weighted all-reduce of one gradient bucket -- Eq. 9.
 *   bucket : device pointer to n elements of `dt` holding this rank's MEAN local gradient g_i
 *            (Eq. 1; a sum-reduced gradient would break |g_i|^2, reading Q4).
 *            Overwritten in place with g = sum_j r_j g_j, bitwise identical on every rank.
 *            16-byte aligned.  n * sizeof(dt) <= heap_bytes.  n == 0 is a no-op.
 *   r_i    : this rank's share b_i / B.  Trusted (not re-normalised).
 * Side effect: the norm statistics of this bucket -- |g_j|^2 restricted to the bucket for every
 * rank j, and |g|^2 restricted to the bucket -- are added (fixed bucket order) to the ctx
 * accumulator that cannikin_gns_stats reads.  Implementation: one kernel over NVLink peer memory
 * with the scaling, the fp32 accumulation in rank order, both norms and the partial exchange
 * fused (DESIGN.md §6 K3).  Variant by size (a function of n, dt, world and grid only, so every
 * rank picks the same): low-latency LL (<= 1 MiB / (world-1): data and flag in one 8-byte NVLink
 * store, no barrier; the bucket may then be any device memory), LL128 (above that, up to
 * 32 MiB: two-shot with the epoch flag inside every 128-byte line, no barrier, any device memory),
 * two-shot pull (static, or dynamic chunks for shards >= 64 MiB), two-shot push (world >= 4,
 * buckets >= 128 MiB: every NVLink transfer a write).  CANNIKIN_AR_{LL,LL128,DYN,PUSH}=0|1
 * environment knobs force or forbid one (CANNIKIN_AR_LL128=1: every bucket up to
 * CANNIKIN_LL128_MAX_MB, default 32).
 * The result bits do not depend on the variant; the statistics' summation grouping does.
 * world == 1: g = r_0 g_0 in place.
 * Errors: INVALID (NULL, misaligned, too large), UNSUPPORTED (dtype), CUDA. */
cannikin_status cannikin_weighted_allreduce(cannikin_ctx* ctx, void* bucket, size_t n,
                                            cannikin_dtype dt, double r_i, void* stream);

/* The same operation through NCCL collectives instead of peer memory (the north
 * star's "NCCL reduce-scatter/all-gather with the r_i scaling and norm partials fused into the
 * pre- and post-kernels"): pre-kernel y = r_i g_i in fp32 + |g_i|^2 partials -> ncclReduceScatter
 * (fp32 sum) -> post-kernel (one rounding to dt, |g|^2 partials) -> ncclAllGather of the shards
 * and of the 2 statistics and the fp32 share per rank -> fixed-order accumulation (identical bits
 * on every rank; with CANNIKIN_INIT_CHECK_RATIOS the gathered shares are checked to sum to 1).
 * Same arguments, contract and statistics as cannikin_weighted_allreduce (Eq. 9, P:328-331;
 * Eq. 10 inputs), except: the fp32 summation order is NCCL's, so the result bits differ
 * from the peer-memory kernels by fp32 rounding (same tolerances); the bucket may be any device
 * memory (no heap limit); a work buffer of ~8 n bytes is allocated on first use / growth, which
 * synchronises the device.  Needs no peer mapping: the path for ranks NCCL connects but NVLink
 * peer memory does not.  COLLECTIVE.  world == 1: as cannikin_weighted_allreduce.
 * Errors: INVALID (NULL, misaligned), UNSUPPORTED (dtype; in-process group: no communicator),
 * DOMAIN (r_i NaN), CUDA, NCCL. */
cannikin_status cannikin_weighted_allreduce_nccl(cannikin_ctx* ctx, void* bucket, size_t n,
                                                 cannikin_dtype dt, double r_i, void* stream);

/* NVSwitch-multicast (NVLS) variant of cannikin_weighted_allreduce, world >= 2.
 *   bucket    : this rank's copy of a symmetric, multicast-capable allocation (e.g. torch symmetric
 *               memory), n elements, 16-byte aligned, n * sizeof(dt) a multiple of 16; in place.
 *   mc_bucket : the multicast address of the same bytes (same layout on every rank).
 * Each rank scales its copy in place (r_i g_i rounded to fp32), the owner of each shard reads the
 * in-switch fp32 sum (multimem.ld_reduce) and multicasts it back (multimem.st).  fp32 only: the
 * switch's bf16 reduction misses the 1e-2 bf16 tolerance (reading Q28).  Same statistics side
 * effect as weighted_allreduce; |g|^2 is taken from the reduced values.  NVLink bytes per rank and
 * direction ~ (1 + 1/W) N s.  Errors: INVALID, UNSUPPORTED (dtype, ragged n, world < 2), CUDA. */
cannikin_status cannikin_weighted_allreduce_nvls(cannikin_ctx* ctx, void* bucket, void* mc_bucket,
                                                 size_t n, cannikin_dtype dt, double r_i,
                                                 void* stream);

/* Read and reset the norm statistics accumulated since the previous call (Eq. 10 inputs):
 *   out_local_sq[j] = |g_j|^2 for j = 0..world-1, *out_global_sq = |g|^2   (host pointers).
 * Identical bits on every rank.  Synchronises `stream`.
 * The north-star signature carried b_i; batch sizes are not needed to finalise the norms and are
 * passed to cannikin_gns_estimate instead.  Errors: INVALID, DOMAIN (a reduction since the last
 * check saw shares not summing to 1, CANNIKIN_INIT_CHECK_RATIOS; the statistics are still
 * returned), CUDA (also: a device protocol error recorded by a reduction kernel). */
cannikin_status cannikin_gns_stats(cannikin_ctx* ctx, void* stream, double* out_local_sq,
                                   double* out_global_sq);

/* Out-of-place statistics of ONE bucket (the north-star form gns_stats(bucket, b_i, ...) with a
 * non-NULL bucket): the Eq. 10 inputs of this bucket alone,
 *   out_local_sq[j] = |g_j|^2 for every rank j,  *out_global_sq = |g|^2,  g = sum_j (b_j/B) g_j,
 * without modifying `bucket` and without touching the statistics the in-place reductions have
 * accumulated (they stay pending for the next cannikin_gns_stats).
 *   bucket : device pointer, n elements of dt, 16-byte aligned: this rank's mean gradient g_i
 *   b_i    : this rank's local batch (>= 0); B = sum_j b_j is exchanged between the ranks and
 *            r_j = b_j / B formed in double from the integers
 * COLLECTIVE for world > 1 (NCCL all-gather of the b_j, then the same reduction kernels as
 * cannikin_weighted_allreduce on a copy of the bucket).  Synchronises `stream`; a work buffer of
 * ~n * sizeof(dt) is allocated on first use / growth (synchronises the device).  Identical bits on
 * every rank.  Errors: INVALID, DOMAIN (b_i < 0 or B == 0), UNSUPPORTED (dtype; in-process group:
 * no communicator), CUDA, NCCL. */
cannikin_status cannikin_gns_stats_bucket(cannikin_ctx* ctx, const void* bucket, size_t n,
                                          cannikin_dtype dt, int64_t b_i, void* stream,
                                          double* out_local_sq, double* out_global_sq);

/* Stream-ordered variant: one finalize kernel writes the (world+1) accumulated doubles
 * [local_sq..., global_sq] to d_out (device memory, or pinned host memory) and resets the
 * accumulator, without host synchronisation. */
cannikin_status cannikin_gns_stats_async(cannikin_ctx* ctx, double* d_out, void* stream);

/* Synchronise the ctx's device and report (and clear, if recoverable) a condition recorded by the
 * reduction kernels: OK, DOMAIN (shares did not sum to 1, see CANNIKIN_INIT_CHECK_RATIOS; cleared),
 * or CUDA (protocol error code; not cleared). */
cannikin_status cannikin_device_status(cannikin_ctx* ctx);

/* Single-GPU fused pass over n_ranks emulated ranks (the 1-B200 metric kernel; reading of
 * SURVEY §8(a) row a5):
 *   in    : host array of n_ranks device pointers, each n elements of `dt` (16-byte aligned)
 *   r     : host array of n_ranks shares r_j
 *   out   : device pointer, n elements of `dt`:  out = sum_j r_j in[j]   (fp32 accumulate, rank order)
 *           out may alias in[j] (in-place).
 *   d_local_sq  : n_ranks doubles |in[j]|^2 -- device memory or pinned (device-mapped) host memory
 *   d_global_sq : 1 double |out|^2 from the fp32 accumulator (reading Q2), same memory kinds
 *   flags & CANNIKIN_ACCUMULATE: add to d_local_sq/d_global_sq instead of overwriting (multi-bucket)
 *   flags & CANNIKIN_LOCAL_LDG / CANNIKIN_LOCAL_TMA: force the 128-bit-load or the TMA-bulk-staged
 *         kernel variant (identical output bits; norms equal up to fp64 summation grouping);
 *         default: the faster one
 *   flags & CANNIKIN_LOCAL_CHAIN: the caller asserts that no input of this call is written by the
 *         kernel enqueued immediately before it on `stream` (e.g. the next bucket of the same
 *         gradient after the previous bucket's call).  The (LDG) kernel is always launched with
 *         programmatic dependent launch; with this flag it streams its inputs while the preceding
 *         kernel's last CTAs still run and waits for that kernel only before touching the shared
 *         partial table and the statistics -- consecutive bucket launches overlap their ramps.
 *         Without it the kernel waits for its predecessor before reading anything.
 * 1 <= n_ranks <= CANNIKIN_MAX_EMULATED.  Errors: INVALID (also: unknown flag), UNSUPPORTED, CUDA. */
#define CANNIKIN_ACCUMULATE 1u
#define CANNIKIN_LOCAL_LDG 2u
#define CANNIKIN_LOCAL_TMA 4u
#define CANNIKIN_LOCAL_CHAIN 8u
cannikin_status cannikin_weighted_sum_local(cannikin_ctx* ctx, const void* const* in, int n_ranks,
                                            const double* r, void* out, size_t n, cannikin_dtype dt,
                                            double* d_local_sq, double* d_global_sq, unsigned flags,
                                            void* stream);

/* Baseline for the step-time comparison: equal-split DDP semantics (Eq. 2) -- an NCCL
 * all-reduce of the bucket with ncclAvg (sum, then division by world, inside NCCL).  In place. */
cannikin_status cannikin_ddp_allreduce_mean(cannikin_ctx* ctx, void* bucket, size_t n,
                                            cannikin_dtype dt, void* stream);

/* Bench utility (not part of the method): enqueue a synthetic "compute" kernel that occupies one
 * warp for `seconds` (0..60) of device time, to emulate a node's compute time t_i(b) (Eq. 3,
 * P:158-165) on homogeneous GPUs, as Cluster C's dummy load does.  Errors: DOMAIN, CUDA. */
cannikin_status cannikin_emulate_compute(double seconds, void* stream);

/* Bench utility (not part of the method): DISJOINT SM partitions of one GPU for heterogeneous
 * ranks that share it -- the single-GPU analog of the paper's Cluster C and north_star's
 * "per-rank compute-rate caps (SM-partitioned contexts)".  Creates n CUDA green contexts on
 * `device`, partition i holding sm_counts[i] SMs (rounded up to the architecture's granularity, 8
 * on sm_90+), split off one after another so they never overlap, and one non-blocking stream per
 * partition: streams[i] (a CUstream / cudaStream_t; kernels launched on it run on partition i's
 * SMs), sm_got[i] = the SMs it received.  The handle owns the contexts and streams; release it
 * with cannikin_green_destroy (after the streams are idle).  Errors: INVALID (n outside 1..64,
 * NULL), UNSUPPORTED (driver without green contexts, or the counts do not fit), CUDA. */
typedef struct cannikin_green cannikin_green;
cannikin_status cannikin_green_partitions(int device, int n, const int* sm_counts,
                                          cannikin_green** out, void** streams, int* sm_got);
cannikin_status cannikin_green_destroy(cannikin_green* green);

/* Bench utility (not part of the method): the bare memory pattern of the emulated-rank pass --
 * n_in (1..CANNIKIN_MAX_EMULATED) device streams of `bytes` read and one written, 16-byte
 * vectors, grid-stride over ctas_per_sm (1..8) x SMs CTAs of 256 threads, integer adds of the
 * words (no method arithmetic; `out` receives meaningless data).  Timed on the very buffers
 * cannikin_weighted_sum_local reduces, it is the HBM ceiling that pass can reach in the same
 * memory-system state.  bytes: a multiple of 16; pointers 16-byte aligned.  Enqueued on `stream`.
 * Errors: INVALID, CUDA. */
cannikin_status cannikin_probe_stream_pattern(const void* const* in, int n_in, void* out,
                                              size_t bytes, int ctas_per_sm, void* stream);

/* Bench utility (not part of the method): the NVLink ceiling K3 runs against, measured on this
 * ctx's peer mappings.  Every rank writes `bytes_per_peer` bytes of its heap into its own slot of
 * EVERY peer's scratch half at once (the all-to-all write pattern of a two-shot all-reduce, both
 * directions of every link loaded), `repeat` times over the same ranges in one launch (1..1024:
 * long transfers amortise the launch and ramp), by ctas_per_sm (1..4) x SMs CTAs of 512 threads,
 * each writing to every peer in turn; per-direction GB/s = (world-1) * bytes_per_peer * repeat /
 * elapsed.
 * COLLECTIVE (every rank, the same bytes_per_peer, no reduction in flight: it overwrites the
 * peers' scratch = staging area).  bytes_per_peer: a multiple of 16, world * bytes_per_peer <=
 * heap_bytes.  Enqueued on `stream`, no synchronisation (time it with events and a barrier).
 * Errors: INVALID (world == 1, in-process group, size, repeat, ctas_per_sm), CUDA. */
cannikin_status cannikin_probe_a2a_write(cannikin_ctx* ctx, size_t bytes_per_peer, int repeat,
                                         int ctas_per_sm, void* stream);

/* Diagnostics (tracing): per-CTA device timeline of the last two-shot (world > 1) or emulated-rank
 * (LDG variant) kernel on this ctx, %globaltimer ns: [start, entry barrier passed (two-shot only),
 * data done, exit barrier passed / partials written, end (last CTA only)] (LL128: [start,
 * scatter issued, own shard reduced, gather done, statistics summed]) for CTA
 * 0..*n_ctas-1, written to out[5*cta + k] (host).  Synchronises the device.
 * Errors: INVALID, CUDA. */
cannikin_status cannikin_trace(cannikin_ctx* ctx, uint64_t* out, int max_ctas, int* n_ctas);

/* Number of device operations (kernels and copies) the last hot-path call on this ctx enqueued,
 * for launch accounting: 1 for a zero-copy or LL/LL128 reduction, 3 for a staged one (copy in,
 * kernel, copy out); for cannikin_weighted_allreduce_group it is recorded on ctxs[0]. */
int cannikin_last_launch_count(cannikin_ctx* ctx);

/* Name of the kernel variant the last hot-path call on this ctx ran: "k2", "k2_tma", "ll",
 * "ll128", "twoshot", "twoshot_dyn", "push", "k4_nccl", "nvls" ("" before any; a static string,
 * never NULL).  For cannikin_weighted_allreduce_group it is recorded on ctxs[0]. */
const char* cannikin_last_variant(cannikin_ctx* ctx);

/* ------------------------------------------------------------------------------------------
 * Host solvers (pure, thread-safe, no CUDA)
 * ------------------------------------------------------------------------------------------ */

#define CANNIKIN_GNS_G_NONPOSITIVE 1u /* aggregated G <= 0: B_noise = S/G is not meaningful */

typedef struct {
  double G2;                          /* G  = sum_i wG_i G_i   (estimate of |G|^2)      */
  double trS;                         /* S  = sum_i wS_i S_i   (estimate of tr(Sigma))  */
  double B_noise;                     /* S / G                                 */
  double Gi[CANNIKIN_MAX_GNS_NODES];  /* Eq. 10 local estimates                          */
  double Si[CANNIKIN_MAX_GNS_NODES];
  double wG[CANNIKIN_MAX_GNS_NODES];  /* Theorem 1 weights (sum to 1)                    */
  double wS[CANNIKIN_MAX_GNS_NODES];
  int n;
  unsigned flags;
} cannikin_gns_result;

/* Heterogeneous GNS estimate, exactly as PAPER.md §4.4 defines it:
 *   G_i = (B|g|^2 - b_i|g_i|^2)/(B - b_i),  S_i = b_i B/(B - b_i) (|g_i|^2 - |g|^2)    (Eq. 10)
 *   w = 1^T A^{-1} / (1^T A^{-1} 1) with the printed Theorem-1 matrices A_G, A_S       (Eq. 11)
 *   G = sum w^G_i G_i,  S = sum w^S_i S_i,  B_noise = S / G.
 * local_sq[n], b[n] host arrays; B = sum b.  2 <= n <= 64.
 * Errors: INVALID (NULL, n out of range), DOMAIN (b_i outside [1, B-1], non-finite input),
 * SINGULAR (zero pivot in the Gaussian elimination).  G <= 0 is not an error: status OK with
 * CANNIKIN_GNS_G_NONPOSITIVE set. */
cannikin_status cannikin_gns_estimate(const double* local_sq, double global_sq, const int64_t* b,
                                      int n, cannikin_gns_result* out);

/* Corrected-covariance variant (NOT the paper's Theorem 1; reading Q31).
 * Same Eq. 10 local estimates, combined with the weights that minimise the variance under the
 * paper's own sampling model (Eq. 1, Eq. 9) with the EXACT Gaussian covariance of the estimators
 * (Isserlis' theorem) instead of Theorem 1's printed matrices:
 *   w^G_i = w^S_i = (B - b_i) / ((n - 1) B)      (independent of the unknown G and Sigma)
 * i.e. G = (n B |g|^2 - sum b_i |g_i|^2) / ((n-1) B),  S = (sum b_i |g_i|^2 - B |g|^2) / (n - 1).
 * Unbiased, like Theorem 1; lower variance (e.g. at b = {32, 64, 96}: Var G 0.0113 vs 0.0152,
 * Var S 39 vs 71 in Monte Carlo, tests/test_oracle_gns.py).  Arguments, errors and flags as
 * cannikin_gns_estimate (no SINGULAR: no solve). */
cannikin_status cannikin_gns_estimate_corrected(const double* local_sq, double global_sq,
                                                const int64_t* b, int n, cannikin_gns_result* out);

/* Per-node performance model, Eq. 3:
 *   a_i = q b + s  (parameter update + data loading + forward),  P_i = k b + m  (backprop). */
typedef struct { double q, s, k, m; } cannikin_node_model;
/* Communication model: overlap ratio gamma in [0,1), T_o (overlappable sync
 * of all buckets but the last), T_u (last bucket).  T_comm = T_o + T_u. */
typedef struct { double gamma, t_o, t_u; } cannikin_comm_model;

/* Per-node batch time, Eq. 5-7, under the frozen evaluation contract
 *   P = k*b + m;  A = q*b + s;  X = gamma*P + t_o;  f = (A + max(P, X)) + t_u
 * (binary64, left to right, no FMA).  Returns NaN on NULL arguments. */
double cannikin_node_time(const cannikin_node_model* node, const cannikin_comm_model* cm, double b);

#define CANNIKIN_ROUND_PAPER 1u /* integer split = largest-remainder rounding of b_real */

/* OptPerf split (§3.1-3.3, Alg. 1).
 *   nodes[n], cm : models;  B >= 1 total batch;  lo[n] (NULL -> all 1), cap[n] (NULL -> all B)
 * Outputs (host, any may be NULL):
 *   b_real_out[n] : the relaxation's optimum -- unclamped nodes finish together (App. A
 *                   P:726-762): compute-bound nodes share t_compute, comm-bound nodes share
 *                   syncStart, t_compute = syncStart + T_o.  Exact breakpoint solve, O(n log n).
 *   b_out[n]      : integer split.  Default: the exact integer minimiser of Eq. 7 with the
 *                   canonical tie-break (reading Q12) -- equal to the greedy "next sample
 *                   to argmin_i (f_i(b_i+1), i)" and to brute force.  With CANNIKIN_ROUND_PAPER:
 *                   largest-remainder rounding of b_real, ties to the lower index.
 *   t_out[2]      : { Eq. 7 at b_real, Eq. 7 at b_out }
 *   label_out[n]  : 1 = compute-bound at b_real ((1-gamma) P_i >= T_o), 0 = comm-bound.
 * Errors: INVALID (NULL nodes/cm, n < 1, B < 1), DOMAIN (gamma outside [0,1), negative or
 * non-finite coefficient, lo < 0, lo > cap), INFEASIBLE (sum lo > B or sum cap < B),
 * SINGULAR (q + gamma k == 0: a node whose comm-bound time does not grow with b). */
cannikin_status cannikin_opt_split(const cannikin_node_model* nodes, int n,
                                   const cannikin_comm_model* cm, int64_t B, const int64_t* lo,
                                   const int64_t* cap, unsigned flags, int64_t* b_out,
                                   double* b_real_out, double* t_out, int* label_out);

/* Eq. 8 warm-up split when no performance model exists yet:
 *   b_i = (sum_j t_j / t_i) (sum_l sum_j t_j / t_l)^{-1} B,  rounded by largest remainder.
 * t_sample[n] > 0 host.  Errors: INVALID, DOMAIN (t <= 0 or non-finite). */
cannikin_status cannikin_warmup_split(const double* t_sample, int n, int64_t B, double* b_real_out,
                                      int64_t* b_out);

/* ------------------------------------------------------------------------------------------
 * Measured-model loop (host): learn the Eq. 3 models and the comm model
 * from timing observations and plan each epoch's split (§4.5; Eq. 8 P:317-324;
 * "OptPerf as early as the third epoch" P:538).
 * ------------------------------------------------------------------------------------------ */

/* Least-squares line y = slope * x + intercept through count >= 2 points (exact for two points:
 * "solving linear equations").  Errors: INVALID (NULL), SINGULAR (count < 2 or all x
 * equal), DOMAIN (non-finite). */
cannikin_status cannikin_fit_linear(const double* x, const double* y, int count, double* slope,
                                    double* intercept);

/* Eq. 12 inverse-variance weighting: sum_i (x_i / v_i) / sum_i (1 / v_i).  Nodes with
 * v_i == 0 dominate: the result is then their plain mean.  Errors: INVALID, DOMAIN (v_i < 0). */
cannikin_status cannikin_ivw(const double* estimate, const double* variance, int n, double* out);

typedef struct cannikin_analyzer cannikin_analyzer; /* opaque; host only, not thread-safe */
cannikin_status cannikin_analyzer_create(int n, cannikin_analyzer** out);
cannikin_status cannikin_analyzer_destroy(cannikin_analyzer* an);
/* Record iteration `iter` of `node` at local batch b: a = data loading + forward + update
 * time, P = backprop time (Eq. 3), gamma = its measured first-bucket share of backprop (Eq. 4),
 * t_o / t_u = its measured sync times of the overlapped buckets / the last bucket.
 * Errors: INVALID (node, b < 1), DOMAIN (negative or non-finite time). */
cannikin_status cannikin_analyzer_observe(cannikin_analyzer* an, int node, int64_t iter, int64_t b,
                                          double a, double P, double gamma, double t_o,
                                          double t_u);
/* Learned models: per node least-squares (q,s,k,m) over all its observations (negative fits
 * clamped to the model domain), gamma by Eq. 12 over the nodes' observations, T_o and T_u as
 * the per-iteration minimum over nodes averaged over the iterations all nodes reported
 * (fallback: min over nodes of each node's mean).  Errors: SINGULAR (a node with < 2 distinct b). */
cannikin_status cannikin_analyzer_models(cannikin_analyzer* an, cannikin_node_model* nodes_out,
                                         cannikin_comm_model* comm_out);
/* Plan the next epoch for total batch B (B >= n; cap[n] optional):
 *   phase 0 (no observations): even split, extra samples to the lowest ranks;
 *   phase 1 (some node has seen one batch size only): Eq. 8 from each node's per-sample compute
 *           time (a+P)/b at its latest batch size, at least one sample per node;
 *   phase 2: cannikin_opt_split on the learned models; *t_pred = its Eq. 7 prediction (NaN in
 *           phases 0-1).  Errors: INVALID, INFEASIBLE, and those of opt_split. */
cannikin_status cannikin_analyzer_plan(cannikin_analyzer* an, int64_t B, const int64_t* cap,
                                       int64_t* b_out, double* t_pred, int* phase_out);

/* ------------------------------------------------------------------------------------------
 * Adaptive total batch size (host): goodput = throughput x statistical
 * efficiency, the efficiency modelled by the GNS.
 * ------------------------------------------------------------------------------------------ */

/* Exponential moving average of the aggregated G and S (separately: the ratio estimator is
 * biased).  Set decay in [0,1) and count = 0 before the first update.  A snapshot with
 * G2 <= 0 is skipped (reading Q26).  Every update call sets B_noise = trS / G2 of the averages
 * (P:364), or NaN while no snapshot has been accepted (count == 0). */
typedef struct { double G2, trS, decay; int count; double B_noise; } cannikin_gns_ema;
cannikin_status cannikin_gns_ema_update(cannikin_gns_ema* ema, double G2, double trS);

/* Statistical efficiency of total batch B relative to the initial batch B0 for noise scale
 * B_noise, in Pollux's form (B_noise + B0) / (B_noise + B) (reading Q27; the paper defers to
 * Pollux). */
double cannikin_efficiency(int64_t B, int64_t B0, double B_noise);

/* Among candidates[n_cand] pick the total batch with the largest goodput B/T(B) * efficiency,
 * T(B) = OptPerf (Eq. 7 at the integer opt_split).  Outputs (optional) T_out[n_cand],
 * goodput_out[n_cand].  Ties -> the first candidate.  Errors: INVALID, and those of opt_split. */
cannikin_status cannikin_choose_batch(const cannikin_node_model* nodes, int n,
                                      const cannikin_comm_model* cm, const int64_t* candidates,
                                      int n_cand, int64_t B0, double B_noise, int64_t* B_out,
                                      double* T_out, double* goodput_out);

/* The paper's strategy with the analyzer's learned models: OptPerf_init for every candidate the
 * first time (or when the candidate list changes), then each epoch only the chosen candidate is
 * re-solved with the updated models and its cache entry updated; if its overlap pattern (labels)
 * changed, every candidate is re-solved.  Returns B, its split b_out[n], the
 * predicted batch time and whether a full recompute happened.  Errors: as analyzer_models. */
cannikin_status cannikin_analyzer_choose_batch(cannikin_analyzer* an, const int64_t* candidates,
                                               int n_cand, int64_t B0, double B_noise,
                                               int64_t* B_out, int64_t* b_out, double* t_pred,
                                               int* full_recompute);

/* The host half of one training step in one call (replicated on every rank from identical
 * statistics): stats[n+1] = [|g_0|^2 .. |g_{n-1}|^2, |g|^2] and b[n] -> cannikin_gns_estimate into
 * *gns_out (n >= 2), the EMA update (ema may be NULL), and, if nodes/cm/b_next are given, the
 * opt_split of B_next into b_next[n] with its Eq. 7 time in *t_next.  Errors: those of the parts. */
cannikin_status cannikin_control_step(const double* stats, const int64_t* b, int n,
                                      cannikin_gns_ema* ema, const cannikin_node_model* nodes,
                                      const cannikin_comm_model* cm, int64_t B_next,
                                      cannikin_gns_result* gns_out, int64_t* b_next,
                                      double* t_next);

#ifdef __cplusplus
}
#endif
#endif /* CANNIKIN_H */
