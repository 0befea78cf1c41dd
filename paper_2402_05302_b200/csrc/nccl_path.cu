// K4: the weighted all-reduce through NCCL collectives (SURVEY §2.2 K4, §8(a) a1-a4 "K3/K4"):
// the north star's other admissible design -- "NCCL reduce-scatter/all-gather with the r_i scaling
// and norm partials fused into the pre- and post-kernels" -- kept as the library-collective
// baseline next to the fused P2P kernels, and as the path that needs no peer mapping (it runs on
// anything NCCL connects, including ranks on different nodes).
//
//   pre  (K1):  y[e] = r_i g_i[e] in fp32 (bf16 widened exactly), zero padding to W*L (an fp32
//               bucket of exactly W shards skips y: NCCL's PreMulSum scales in place);
//               per-CTA partials of |g_i|^2 on the UNSCALED gradient (Eq. 10 input)
//   ncclReduceScatter(y, sum, fp32), in place: rank k owns y[k L, (k+1) L)      (Eq. 9)
//   post:       round the owned shard once to the bucket dtype; per-CTA partials of |g|^2 from
//               the fp32 sums
//   stats:      one CTA sums both partial tables in fixed order -> x = {|g_i|^2, |g|^2_shard, r_i}
//   ncclAllGather(x, 3 doubles) and ncclAllGather(shard, L elements of the bucket dtype)
//   add:        every rank adds |g_j|^2 = x_j[0] and |g|^2 = sum_k x_k[1] (rank order) to the
//               ctx accumulator: identical bits on every rank; with CANNIKIN_INIT_CHECK_RATIOS it
//               also checks sum_k x_k[2] (the fp32 shares NCCL scaled with) against 1.
// The fp32 sum's order is NCCL's (ring/tree), not rank order, so the result bits differ from the
// K3 variants by fp32 rounding (within the fp32 1e-5 / bf16 1e-2 tolerances; tests/).  NVLink
// bytes: the reduce-scatter moves fp32 even for bf16 buckets (2x the all-gather's bytes), the
// price of accumulating in fp32 instead of rounding r_i g_i to bf16 before the sum.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include "common.h"
#include "ctx.h"
#include "device_utils.cuh"
#include "kernels.h"

namespace cannikin {

constexpr int kK4Threads = 256;
constexpr int kK4MaxBlocks = 1024;

// y <- r g (fp32) over 16-byte vectors of g, zero padding up to `padded` elements; partial |g|^2
// (y == nullptr: the norm only -- the fp32 fast path scales inside NCCL)
template <typename T>
__global__ void __launch_bounds__(kK4Threads) k4_pre_kernel(const char* g, size_t n, size_t padded,
                                                            float r, float* y, double* part) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  __shared__ double red[32];
  const size_t nvec = n / E, stride = (size_t)gridDim.x * kK4Threads;
  double sq = 0.0;
  for (size_t v = (size_t)blockIdx.x * kK4Threads + threadIdx.x; v < nvec; v += stride) {
    float f[E];
    V::unpack(dev::ld16(g + v * 16), f);
    float s = 0.0f;
    float o[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      s = fmaf(f[q], f[q], s);
      o[q] = r * f[q];
    }
    sq += (double)s;
    if (y == nullptr) continue;
#pragma unroll
    for (int q = 0; q < E; q += 4)
      dev::st16(y + v * E + q, make_uint4(__float_as_uint(o[q]), __float_as_uint(o[q + 1]),
                                          __float_as_uint(o[q + 2]), __float_as_uint(o[q + 3])));
  }
  // ragged tail and padding, element-wise
  for (size_t e = nvec * E + (size_t)blockIdx.x * kK4Threads + threadIdx.x; e < padded; e += stride) {
    if (e < n) {
      const float f = V::load1(g + e * sizeof(T));
      sq += (double)(f * f);
      if (y != nullptr) y[e] = r * f;
    } else if (y != nullptr) {
      y[e] = 0.0f;
    }
  }
  double v1[1] = {sq};
  dev::block_sum(v1, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v1[0];
}

// dst[e] <- round(shard[e]) for e < cnt; partial |g|^2 from the fp32 values (dst == nullptr:
// the norm only, the shard already is the result)
template <typename T>
__global__ void __launch_bounds__(kK4Threads) k4_post_kernel(const float* shard, size_t cnt,
                                                             char* dst, double* part) {
  using V = dev::Vec<T>;
  constexpr int E = V::E;
  __shared__ double red[32];
  const size_t nvec = cnt / E, stride = (size_t)gridDim.x * kK4Threads;
  double sq = 0.0;
  for (size_t v = (size_t)blockIdx.x * kK4Threads + threadIdx.x; v < nvec; v += stride) {
    float f[E];
#pragma unroll
    for (int q = 0; q < E; q += 4) {
      const uint4 u = dev::ld16(shard + v * E + q);
      f[q] = __uint_as_float(u.x);
      f[q + 1] = __uint_as_float(u.y);
      f[q + 2] = __uint_as_float(u.z);
      f[q + 3] = __uint_as_float(u.w);
    }
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < E; ++q) s = fmaf(f[q], f[q], s);
    sq += (double)s;
    if (dst != nullptr) dev::st16(dst + v * 16, V::pack(f));
  }
  for (size_t e = nvec * E + (size_t)blockIdx.x * kK4Threads + threadIdx.x; e < cnt; e += stride) {
    const float f = shard[e];
    sq += (double)(f * f);
    if (dst != nullptr) V::store1(dst + e * sizeof(T), f);
  }
  double v1[1] = {sq};
  dev::block_sum(v1, red);
  if (threadIdx.x == 0) part[blockIdx.x] = v1[0];
}

// x = {sum of the pre partials, sum of the post partials, r_i}, fixed order
__global__ void __launch_bounds__(kK4Threads) k4_stats_kernel(const double* pre, int npre,
                                                              const double* post, int npost,
                                                              float r, double* x) {
  __shared__ double red[64];
  double v[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < npre; i += kK4Threads) v[0] += pre[i];
  for (int i = threadIdx.x; i < npost; i += kK4Threads) v[1] += post[i];
  dev::block_sum(v, red);
  if (threadIdx.x == 0) {
    x[0] = v[0];
    x[1] = v[1];
    x[2] = (double)r;
  }
}

// ctx accumulator (running row 0) += {|g_j|^2 = xr[3j]}, |g|^2 = sum_k xr[3k+1] in rank order;
// check_r: the ranks' fp32 shares xr[3k+2] must sum to 1 within 2^-23 (as the K3 variants check;
// a violation is recorded as code 7 and reported as DOMAIN, the reduction still runs)
__global__ void k4_add_kernel(const double* xr, int W, Ctrl* c, int check_r) {
  if (threadIdx.x != 0) return;
  double gs = 0.0, rs = 0.0;
  for (int k = 0; k < W; ++k) {
    c->cta_acc[0][k] = c->cta_acc[0][k] + xr[3 * k];
    gs += xr[3 * k + 1];
    rs += xr[3 * k + 2];
  }
  c->cta_acc[0][W] = c->cta_acc[0][W] + gs;
  if (check_r && fabs(rs - 1.0) > 0x1p-23) {
    c->rsum_bad = rs;
    atomicCAS(&c->error_code, 0, 7);
  }
}

static int k4_grid(const cannikin_ctx* ctx, size_t vecs) {
  size_t g = (vecs + kK4Threads - 1) / kK4Threads;
  const size_t cap = (size_t)ctx->num_sms * 4;
  if (g > cap) g = cap;
  if (g > (size_t)kK4MaxBlocks) g = kK4MaxBlocks;
  return g < 1 ? 1 : (int)g;
}

size_t k4_buffer_bytes(int world, size_t n) {
  const size_t L = ((n + world - 1) / world + 7) / 8 * 8;
  const size_t padded = L * world;
  return padded * 4 + padded * 4 /* gather (<= fp32) */ + (2 * kK4MaxBlocks + 3 + 3 * kMaxWorld) * 8;
}

#define K4_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(CANNIKIN_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                 \
  } while (0)
#define K4_NCCL(expr)                                                                        \
  do {                                                                                       \
    ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return fail(CANNIKIN_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(r_), __FILE__, \
                  __LINE__);                                                                 \
  } while (0)

cannikin_status launch_k4(cannikin_ctx* ctx, void* bucket, size_t n, cannikin_dtype dt,
                          double r_i, cudaStream_t st) {
  const int W = ctx->world, me = ctx->rank;
  const size_t esz = dt == CANNIKIN_F32 ? 4 : 2;
  const size_t L = ((n + W - 1) / W + 7) / 8 * 8;  // shard: 8 elements = 16-B aligned for both
  const size_t padded = L * W;
  char* base = static_cast<char*>(ctx->k4_buf);
  float* y = reinterpret_cast<float*>(base);
  char* gbuf = base + padded * 4;
  double* pre = reinterpret_cast<double*>(gbuf + padded * 4);
  double* post = pre + kK4MaxBlocks;
  double* xs = post + kK4MaxBlocks;
  double* xr = xs + 3;
  ncclComm_t comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  const ncclDataType_t ndt = dt == CANNIKIN_F32 ? ncclFloat32 : ncclBfloat16;
  const size_t cnt = n > me * L ? (n - me * L < L ? n - me * L : L) : 0;
  // all-gather straight into the bucket when it is exactly W shards long
  const bool direct = padded == n;
  char* dst = direct ? static_cast<char*>(bucket) + me * L * esz : gbuf + me * L * esz;

  const int gpre = k4_grid(ctx, padded / 4);
  const int gpost = k4_grid(ctx, L / 4);
  if (dt == CANNIKIN_F32 && direct) {
    // fp32 bucket of exactly W shards: NCCL scales (PreMulSum, r_i as a host immediate) and sums
    // in place; the pre/post kernels only read (norms).  Same arithmetic as the general path.
    float* gb = static_cast<float*>(bucket);
    k4_pre_kernel<float><<<gpre, kK4Threads, 0, st>>>(static_cast<const char*>(bucket), n, n,
                                                       0.0f, nullptr, pre);
    K4_CUDA(cudaGetLastError());
    float rf = (float)r_i;
    ncclRedOp_t op;
    K4_NCCL(ncclRedOpCreatePreMulSum(&op, &rf, ncclFloat32, ncclScalarHostImmediate, comm));
    const ncclResult_t rs = ncclReduceScatter(gb, gb + me * L, L, ncclFloat32, op, comm, st);
    ncclRedOpDestroy(op, comm);
    K4_NCCL(rs);
    k4_post_kernel<float><<<gpost, kK4Threads, 0, st>>>(gb + me * L, cnt, nullptr, post);
  } else {
    if (dt == CANNIKIN_F32)
      k4_pre_kernel<float><<<gpre, kK4Threads, 0, st>>>(static_cast<const char*>(bucket), n,
                                                         padded, (float)r_i, y, pre);
    else
      k4_pre_kernel<__nv_bfloat16><<<gpre, kK4Threads, 0, st>>>(static_cast<const char*>(bucket),
                                                                 n, padded, (float)r_i, y, pre);
    K4_CUDA(cudaGetLastError());
    K4_NCCL(ncclReduceScatter(y, y + me * L, L, ncclFloat32, ncclSum, comm, st));
    if (dt == CANNIKIN_F32)
      k4_post_kernel<float><<<gpost, kK4Threads, 0, st>>>(y + me * L, cnt, dst, post);
    else
      k4_post_kernel<__nv_bfloat16><<<gpost, kK4Threads, 0, st>>>(y + me * L, cnt, dst, post);
  }
  k4_stats_kernel<<<1, kK4Threads, 0, st>>>(pre, gpre, post, gpost, (float)r_i, xs);
  K4_CUDA(cudaGetLastError());
  K4_NCCL(ncclGroupStart());
  K4_NCCL(ncclAllGather(xs, xr, 3, ncclFloat64, comm, st));
  K4_NCCL(ncclAllGather(dst, direct ? bucket : static_cast<void*>(gbuf), L, ndt, comm, st));
  K4_NCCL(ncclGroupEnd());
  k4_add_kernel<<<1, 32, 0, st>>>(xr, W, ctx->ctrl, ctx->check_ratios);
  K4_CUDA(cudaGetLastError());
  if (!direct) K4_CUDA(cudaMemcpyAsync(bucket, gbuf, n * esz, cudaMemcpyDeviceToDevice, st));
  ctx->last_launches = 5;
  return CANNIKIN_OK;
}

}  // namespace cannikin
