// Internal declarations shared by the kernel translation units and api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "ctx.h"

namespace cannikin {

// Launch with programmatic stream serialization (PDL): the kernel may be launched while its
// predecessor in the stream is still running if that predecessor triggers early
// (griddepcontrol.launch_dependents); the kernel itself executes griddepcontrol.wait before
// touching memory, so the ordering is that of a plain launch and only the launch latency is
// hidden.  A predecessor that never triggers releases it at completion.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Arguments of a single-launch in-process group (cannikin_weighted_allreduce_group): the per-rank
// arguments of every rank, one grid of world x grid CTAs; CTA c serves rank c / grid as its CTA
// c % grid, so the ranks' CTAs are co-resident by construction (one kernel).
template <typename A>
struct GroupArgs {
  A a[kMaxWorld];
  int grid;
};

// Arguments of the emulated-rank kernels (K2, both variants).
struct LocalArgs {
  const char* in[kMaxEmu];
  float r[kMaxEmu];
  char* out;
  size_t nvec;       // full 16-byte vectors
  size_t n;          // elements
  double* partials;  // [grid][n+1]
  unsigned* ticket;
  double* local_sq;  // [n]
  double* global_sq;
  uint64_t* trace;   // [grid][5] per-CTA timeline (LDG variant)
  int* trace_grid;
  int accumulate;
  int chain;         // CANNIKIN_LOCAL_CHAIN: inputs may be read before the preceding kernel ends
};

cudaError_t launch_wsum_local(cannikin_ctx* ctx, const void* const* in, int nr, const double* r,
                              void* out, size_t n, cannikin_dtype dt, double* d_local_sq,
                              double* d_global_sq, bool accumulate, int grid_override,
                              cudaStream_t st, bool chain = false);
cudaError_t launch_wsum_local_tma(cannikin_ctx* ctx, const void* const* in, int nr,
                                  const double* r, void* out, size_t n, cannikin_dtype dt,
                                  double* d_local_sq, double* d_global_sq, bool accumulate,
                                  cudaStream_t st, bool chain = false);
cudaError_t launch_emulate(double seconds, cudaStream_t st);
cudaError_t launch_nvls(cannikin_ctx* ctx, void* local, void* mc, size_t n, cannikin_dtype dt,
                        double r_i, cudaStream_t st);
cudaError_t launch_twoshot(cannikin_ctx* ctx, size_t off, size_t n, cannikin_dtype dt, double r_i,
                           cudaStream_t st);
// in-process group (cannikin_weighted_allreduce_group): all W ranks' kernels in ONE launch
cudaError_t launch_twoshot_group(cannikin_ctx* const* ctxs, int W, size_t off, size_t n,
                                 cannikin_dtype dt, const double* r, cudaStream_t st);
cudaError_t launch_ll_group(cannikin_ctx* const* ctxs, int W, void* const* buckets, size_t n,
                            cannikin_dtype dt, const double* r, cudaStream_t st);
cudaError_t launch_ll128_group(cannikin_ctx* const* ctxs, int W, void* const* buckets, size_t n,
                               cannikin_dtype dt, const double* r, cudaStream_t st);
cudaError_t launch_gate(cannikin_ctx* ctx, cudaStream_t st);
cudaError_t launch_stream_pattern(const void* const* in, int n_in, void* out, size_t bytes,
                                  int grid, cudaStream_t st);
cudaError_t launch_a2a_write(cannikin_ctx* ctx, size_t bytes_per_peer, int repeat,
                             int ctas_per_sm, cudaStream_t st);
cudaError_t launch_stats_finalize(cannikin_ctx* ctx, double* out, cudaStream_t st);
cudaError_t launch_stats_add(cannikin_ctx* ctx, const double* in, cudaStream_t st);
size_t ll_max_bytes(int world);
size_t ll_region_bytes(int world);
bool ll_eligible(const cannikin_ctx* ctx, size_t bytes);
cudaError_t launch_ll(cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt, double r_i,
                      cudaStream_t st);
size_t ll128_region_bytes(int world, size_t max_bytes);
size_t ll128_auto_bytes(int world);
bool ll128_eligible(const cannikin_ctx* ctx, size_t bytes);
cudaError_t launch_ll128(cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt, double r_i,
                         cudaStream_t st);
size_t k4_buffer_bytes(int world, size_t n);
cannikin_status launch_k4(cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt, double r_i,
                          cudaStream_t st);

}  // namespace cannikin
