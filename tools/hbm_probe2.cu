// HBM probe, part 2: how do the WRITES of an 8:1 read:write stream reach DRAM best?
// tools/hbm_probe.cu showed 8 reads + 1 write of 16-byte vectors reach 6.19 TB/s at C4 size while
// 8 reads alone reach 7.28: the write stream costs ~2.5x its bytes.  Cases (220 MB and 1.42 GB per
// stream; integer adds, no method arithmetic):
//   memcpy       cudaMemcpyAsync device-to-device (1:1, driver path), for reference
//   write1       16-byte stores only
//   r8w1_ldg     the tools/hbm_probe.cu baseline (grid-stride, LDG + STG)
//   r8w1_bulkst  LDG reads; each CTA assembles a TILE-byte output tile in shared memory and one
//                thread stores it with cp.async.bulk (TMA engine, S2G), double-buffered
//   r8w1_bulk    reads by cp.async.bulk (G2S, mbarrier) AND the bulk store: the whole stream on
//                the TMA engine, CTA-contiguous tiles handed out grid-stride
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_probe2 tools/hbm_probe2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

struct Args {
  const char* in[8];
  char* out;
  size_t nvec;
};

__device__ __forceinline__ uint4 ld(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256) write1(const Args a) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const uint4 z = make_uint4(1, 2, 3, 4);
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.nvec; v += stride)
    st(a.out + v * 16, z);
}

__global__ void __launch_bounds__(256) r8w1_ldg(const Args a) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.nvec; v += stride) {
    uint4 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ld(a.in[j] + v * 16);
    uint4 s = x[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) { s.x += x[j].x; s.y += x[j].y; s.z += x[j].z; s.w += x[j].w; }
    st(a.out + v * 16, s);
  }
}

// TILE bytes of output per CTA step (TILE/16 vectors; 256 threads -> TILE/4096 vectors each)
template <int TILE>
__global__ void __launch_bounds__(256) r8w1_bulkst(const Args a) {
  constexpr int VPT = TILE / 16 / 256;
  __shared__ __align__(128) uint4 buf[2][TILE / 16];
  const size_t ntiles = a.nvec / (TILE / 16);  // full tiles only (probe sizes are multiples)
  int k = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, k ^= 1) {
    const size_t v0 = t * (TILE / 16);
    uint4 x[VPT][8];
#pragma unroll
    for (int u = 0; u < VPT; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[u][j] = ld(a.in[j] + (v0 + u * 256 + threadIdx.x) * 16);
    // the bulk store issued from buf[k] two tiles ago must have finished reading it
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      uint4 s = x[u][0];
#pragma unroll
      for (int j = 1; j < 8; ++j) { s.x += x[u][j].x; s.y += x[u][j].y; s.z += x[u][j].z; s.w += x[u][j].w; }
      buf[k][u * 256 + threadIdx.x] = s;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.out + v0 * 16),
                   "r"(su32(&buf[k][0])), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Whole stream on the TMA engine: per CTA a ring of S stages, each = 8 input tiles of TILE bytes;
// thread 0 produces (G2S bulk loads), all 256 threads consume and write an output tile to smem,
// thread 0 bulk-stores it.
template <int TILE, int S>
__global__ void __launch_bounds__(256, 1) r8w1_bulk(const Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint4* in_s = reinterpret_cast<uint4*>(sm);                       // [S][8][TILE/16]
  uint4* out_s = reinterpret_cast<uint4*>(sm + (size_t)S * 8 * TILE);  // [2][TILE/16]
  __shared__ __align__(8) uint64_t full[S];
  constexpr int VT = TILE / 16;
  const size_t ntiles = a.nvec / VT;
  const size_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t i) {  // tile i of this CTA into stage i % S
    const int s = (int)(i % S);
    const size_t v0 = (blockIdx.x + i * gridDim.x) * (size_t)VT;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                 "r"(8 * TILE) : "memory");
    for (int j = 0; j < 8; ++j)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(su32(in_s + ((size_t)s * 8 + j) * VT)), "l"(a.in[j] + v0 * 16), "r"(TILE),
          "r"(su32(&full[s]))
          : "memory");
  };
  if (threadIdx.x == 0)
    for (size_t i = 0; i < (size_t)S && i < my; ++i) issue(i);
  for (size_t i = 0; i < my; ++i) {
    const int s = (int)(i % S);
    const uint32_t par = (uint32_t)((i / S) & 1);
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            su32(&full[s])),
        "r"(par) : "memory");
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const int k = (int)(i & 1);
    for (int v = threadIdx.x; v < VT; v += 256) {
      uint4 sacc = in_s[((size_t)s * 8) * VT + v];
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        const uint4 y = in_s[((size_t)s * 8 + j) * VT + v];
        sacc.x += y.x; sacc.y += y.y; sacc.z += y.z; sacc.w += y.w;
      }
      out_s[k * VT + v] = sacc;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // stage s consumed, output tile k written
    if (threadIdx.x == 0) {
      const size_t v0 = (blockIdx.x + i * gridDim.x) * (size_t)VT;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a.out + v0 * 16),
                   "r"(su32(out_s + k * VT)), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (i + S < my) issue(i + S);
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef void (*KernFn)(const Args);

int main() {
  CK(cudaSetDevice(0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t maxb = 1419292672ull;
  char* big = nullptr;
  CK(cudaMalloc(&big, maxb * 9 + 4096));
  CK(cudaMemset(big, 1, maxb * 9 + 4096));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 20;
  struct Case { const char* name; KernFn fn; int threads; size_t smem; int nin; int per_sm_max; };
  std::vector<Case> cases = {
      {"write1", write1, 256, 0, 0, 8},
      {"r8w1_ldg", r8w1_ldg, 256, 0, 8, 8},
      {"r8w1_bulkst_4k", r8w1_bulkst<4096>, 256, 0, 8, 8},
      {"r8w1_bulkst_8k", r8w1_bulkst<8192>, 256, 0, 8, 8},
      {"r8w1_bulkst_16k", r8w1_bulkst<16384>, 256, 0, 8, 4},
      {"r8w1_bulk_4k_s4", r8w1_bulk<4096, 4>, 256, (size_t)4 * 8 * 4096 + 2 * 4096, 8, 1},
      {"r8w1_bulk_4k_s6", r8w1_bulk<4096, 6>, 256, (size_t)6 * 8 * 4096 + 2 * 4096, 8, 1},
      {"r8w1_bulk_2k_s8", r8w1_bulk<2048, 8>, 256, (size_t)8 * 8 * 2048 + 2 * 2048, 8, 1},
      {"r8w1_bulk_2k_s4", r8w1_bulk<2048, 4>, 256, (size_t)4 * 8 * 2048 + 2 * 2048, 8, 2},
  };
  const size_t sizes[2] = {220000000ull - 220000000ull % 65536, 1419292672ull};
  for (size_t sz : sizes) {
    {  // memcpy reference
      std::vector<float> ts;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        for (int k = 0; k < reps; ++k) CK(cudaMemcpyAsync(big + 8 * sz, big, sz, cudaMemcpyDeviceToDevice));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ts.push_back(ms / reps);
      }
      std::sort(ts.begin(), ts.end());
      printf("{\"case\": \"memcpy\", \"stream_bytes\": %zu, \"ms\": %.4f, \"GBs\": %.1f}\n", sz,
             ts[2], 2.0 * sz / (ts[2] * 1e-3) / 1e9);
      fflush(stdout);
    }
    for (const Case& c : cases) {
      if (c.smem > 48 * 1024)
        CK(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.fn, c.threads, c.smem));
      for (int per_sm : {1, 2, 3, 4, 5, 6, 8}) {
        if (per_sm > occ || per_sm > c.per_sm_max) continue;
        Args a{};
        for (int j = 0; j < 8; ++j) a.in[j] = big + (size_t)j * sz;
        a.out = big + (size_t)8 * sz;
        a.nvec = sz / 16;
        const int grid = sms * per_sm;
        for (int w = 0; w < 3; ++w) c.fn<<<grid, c.threads, c.smem>>>(a);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<float> ts;
        for (int r = 0; r < 5; ++r) {
          CK(cudaEventRecord(e0));
          for (int k = 0; k < reps; ++k) c.fn<<<grid, c.threads, c.smem>>>(a);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          ts.push_back(ms / reps);
        }
        CK(cudaGetLastError());
        std::sort(ts.begin(), ts.end());
        const double bytes = (double)sz * (c.nin + 1);
        printf("{\"case\": \"%s\", \"stream_bytes\": %zu, \"grid\": %d, \"ctas_per_sm\": %d, "
               "\"ms\": %.4f, \"GBs\": %.1f}\n",
               c.name, sz, grid, per_sm, ts[2], bytes / (ts[2] * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
  }
  CK(cudaFree(big));
  return 0;
}
