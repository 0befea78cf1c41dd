// Device helpers: 16-byte vector memory ops, dtype packing, deterministic block reductions and
// system-scope flag operations for the NVLink peer-memory protocol.  sm_100a only.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cannikin {
namespace dev {

// ------------------------------------------------------------------ 16-byte memory operations
// Streaming loads/stores: every gradient byte is touched exactly once per launch, so L1 is bypassed.
// CANNIKIN_LD_HINT (build-time experiment): 1 = non-coherent path + L2 256-byte prefetch hint,
// 2 = L2 256-byte prefetch hint only; default none.
#if defined(CANNIKIN_LD_HINT) && CANNIKIN_LD_HINT == 1
#define CANNIKIN_LD16 "ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#elif defined(CANNIKIN_LD_HINT) && CANNIKIN_LD_HINT == 2
#define CANNIKIN_LD16 "ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#else
#define CANNIKIN_LD16 "ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
#endif
__device__ __forceinline__ uint4 ld16(const void* p) {
  uint4 v;
  asm volatile(CANNIKIN_LD16 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st16(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ------------------------------------------------------------------ dtype traits (16-byte vectors)
template <typename T>
struct Vec;

template <>
struct Vec<float> {
  static constexpr int E = 4;  // elements per 16-byte vector
  __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[4]) {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
  }
  __device__ __forceinline__ static uint4 pack(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
  __device__ __forceinline__ static float load1(const void* p) {
    return *reinterpret_cast<const float*>(p);
  }
  __device__ __forceinline__ static void store1(void* p, float x) {
    *reinterpret_cast<float*>(p) = x;
  }
};

template <>
struct Vec<__nv_bfloat16> {
  static constexpr int E = 8;
  // a bf16 is the upper half of an fp32: widening is a shift (exact)
  __device__ __forceinline__ static void unpack(const uint4& v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  // round-to-nearest-even, once, from the fp32 accumulator
  __device__ __forceinline__ static uint4 pack(const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static float load1(const void* p) {
    return __uint_as_float(uint32_t(*reinterpret_cast<const uint16_t*>(p)) << 16);
  }
  __device__ __forceinline__ static void store1(void* p, float x) {
    *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(x);
  }
};

// ------------------------------------------------------------------ packed fp32x2 arithmetic
// sm_100's FFMA2: two independent fp32 FMAs (each rounded exactly as fmaf) in one instruction.
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  return ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float f2lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// The emulated-rank pass over one 16-byte vector index (K2, both variants): returns the packed
// out = sum_j r_j x_j in rank order from 0 (fp32 fma: the same bits as a scalar fmaf chain) and
// adds |x_j|^2 and |out|^2 of the vector, formed in fp32 (even and odd elements in two chains, then
// added), to fp64 accumulators.
template <typename T, int NR>
__device__ __forceinline__ uint4 wsum16v(const uint4 (&x)[NR], const float (&r)[NR],
                                         double (&lsq)[NR], double& gsq) {
  using V = Vec<T>;
  constexpr int E = V::E;
  constexpr int P = E / 2;
  uint64_t acc[P];
#pragma unroll
  for (int p = 0; p < P; ++p) acc[p] = 0ull;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    float g[E];
    V::unpack(x[j], g);
    const uint64_t rr = f2pack(r[j], r[j]);
    uint64_t sq = 0ull;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint64_t gp = f2pack(g[2 * p], g[2 * p + 1]);
      acc[p] = ffma2(rr, gp, acc[p]);
      sq = ffma2(gp, gp, sq);
    }
    lsq[j] += (double)(f2lo(sq) + f2hi(sq));
  }
  uint64_t gs = 0ull;
  float out[E];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    gs = ffma2(acc[p], acc[p], gs);
    out[2 * p] = f2lo(acc[p]);
    out[2 * p + 1] = f2hi(acc[p]);
  }
  gsq += (double)(f2lo(gs) + f2hi(gs));
  return V::pack(out);
}

// ... and stores it (streaming 16-byte store).
template <typename T, int NR>
__device__ __forceinline__ void wsum16(const uint4 (&x)[NR], const float (&r)[NR], char* dst,
                                       double (&lsq)[NR], double& gsq) {
  st16(dst, wsum16v<T, NR>(x, r, lsq, gsq));
}

// ------------------------------------------------------------------ deterministic reductions
// Butterfly over the 32 lanes: every lane ends with the same, order-fixed sum.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce NV doubles over the block; the result is valid in thread 0.  `smem` holds >= 32*NV
// doubles.  Fixed order (butterfly within warps, then warps 0..nw-1 in sequence).
template <int NV, int N>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (&smem)[N]) {
  static_assert(N >= 32 * NV, "block_sum: scratch must hold 32 warps x NV doubles");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) smem[warp * NV + j] = v[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += smem[w * NV + j];
      v[j] = s;
    }
  }
  __syncthreads();
}

// NV column sums of a row-major table base[i*row_stride + j] (i = 0..count-1, j = 0..NV-1) in ONE
// pass over the block: thread t accumulates rows t, t+T, t+2T, ... for all columns (independent
// loads, pipelined), then one butterfly/warp-order reduction.  Fixed order => deterministic.
// Result valid in thread 0.
template <int NV, int N>
__device__ __forceinline__ void block_table_sum(const double* base, int count, int row_stride,
                                                double (&out)[NV], double (&smem)[N]) {
#pragma unroll
  for (int j = 0; j < NV; ++j) out[j] = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    const double* row = base + (size_t)i * row_stride;
#pragma unroll
    for (int j = 0; j < NV; ++j) out[j] += __ldcg(row + j);
  }
  block_sum(out, smem);
}

// ------------------------------------------------------------------ system-scope flags
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Bookkeeping of a peer wait: expired() is true once timeout_ns (> 0) of device time has passed
// since the first check (every `mask`+1 polls); it then records `code` in *err (the first code
// wins) and the caller stops waiting -- the kernel finishes with a recorded protocol error, which
// cannikin_gns_stats / cannikin_device_status report, instead of trapping (a trap would kill the
// process's CUDA context) or hanging.  timeout_ns == 0 waits forever, as NCCL does: the default
// for multi-process contexts, where a peer may legitimately be late (checkpoint, data loading).
struct SpinClock {
  uint64_t t0 = 0;
  unsigned it = 0;
  __device__ __forceinline__ bool expired(uint64_t timeout_ns, unsigned mask, int* err, int code) {
    if ((++it & mask) != 0u || timeout_ns == 0) return false;
    uint64_t now;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
    if (t0 == 0) {
      t0 = now;
      return false;
    }
    if (now - t0 <= timeout_ns) return false;
    atomicCAS(err, 0, code);
    return true;
  }
};

// Programmatic dependent launch (sm_90+): let the next kernel on the stream be scheduled now (its
// CTAs take SM slots as ours exit), and wait until the preceding kernel has completed and its
// memory is visible (a no-op for a kernel launched without the programmatic attribute).
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace dev

// Two entry points for one kernel body BODY<TARGS>(args, cta, grid): KERNEL, the per-rank launch
// (one grid per rank), and GKERNEL, the in-process group launch over GroupArgs<ARGS> (kernels.h):
// world x grid CTAs in ONE grid, CTA c running BODY for rank c / grid as its CTA c % grid.
#define CANNIKIN_UNPAREN(...) __VA_ARGS__
#define CANNIKIN_GROUP_ENTRY(TPARAMS, TARGS, BOUNDS, KERNEL, GKERNEL, BODY, ARGS)      \
  template <CANNIKIN_UNPAREN TPARAMS>                                                 \
  __global__ void __launch_bounds__ BOUNDS KERNEL(const ARGS a) {                     \
    BODY<CANNIKIN_UNPAREN TARGS>(a, blockIdx.x, gridDim.x);                           \
  }                                                                                   \
  template <CANNIKIN_UNPAREN TPARAMS>                                                 \
  __global__ void __launch_bounds__ BOUNDS GKERNEL(const GroupArgs<ARGS> g) {         \
    const int rk = blockIdx.x / g.grid;                                               \
    BODY<CANNIKIN_UNPAREN TARGS>(g.a[rk], blockIdx.x - rk * g.grid, g.grid);          \
  }

}  // namespace cannikin
