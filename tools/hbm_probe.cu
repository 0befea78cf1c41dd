// HBM ceiling probe for K2's traffic pattern (n_in streams read, 1 stream written, 16-byte vectors).
// What does a B200 deliver for 1:1 copy, read-only and 8:1 read:write streams, at C4 (220 MB per
// stream) and C5 (1.42 GB per stream) sizes and at a 25 MB bucket, for a few load/store flavours
// and two work distributions (grid-stride vs one contiguous chunk per CTA)?  Arithmetic is an
// integer add (no method arithmetic: this measures memory only).  One JSON line per case:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_probe tools/hbm_probe.cu && ./hbm_probe
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

struct Args {
  const char* in[8];
  char* out;
  size_t nvec;  // 16-byte vectors per stream
  int nin;
};

template <int LD>
__device__ __forceinline__ uint4 ld(const void* p, uint64_t pol) {
  uint4 v;
  if (LD == 0)
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (LD == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (LD == 2)
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  else
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <int ST>
__device__ __forceinline__ void st(void* p, const uint4& v, uint64_t pol) {
  if (ST == 0)
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if (ST == 1)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}

// DIST 0: grid-stride over vectors; DIST 1: CTA b owns a contiguous chunk [b*C, (b+1)*C).
template <int NIN, int LD, int ST, int DIST, int U>
__global__ void __launch_bounds__(256) probe(const Args a) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  size_t v0, step, end;
  if (DIST == 0) {
    v0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    step = (size_t)gridDim.x * blockDim.x;
    end = a.nvec;
  } else {
    const size_t per = (a.nvec + gridDim.x - 1) / gridDim.x;
    const size_t b0 = (size_t)blockIdx.x * per;
    end = b0 + per < a.nvec ? b0 + per : a.nvec;
    v0 = b0 + threadIdx.x;
    step = blockDim.x;
  }
  uint32_t sink = 0;
  size_t v = v0;
  for (; v + (U - 1) * step < end; v += U * step) {
    uint4 x[U][NIN];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NIN; ++j) x[u][j] = ld<LD>(a.in[j] + (v + u * step) * 16, pol);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint4 s = x[u][0];
#pragma unroll
      for (int j = 1; j < NIN; ++j) {
        s.x += x[u][j].x; s.y += x[u][j].y; s.z += x[u][j].z; s.w += x[u][j].w;
      }
      if (a.out) st<ST>(a.out + (v + u * step) * 16, s, pol);
      else sink += s.x ^ s.y ^ s.z ^ s.w;
    }
  }
  for (; v < end; v += step) {
    uint4 s = ld<LD>(a.in[0] + v * 16, pol);
#pragma unroll
    for (int j = 1; j < NIN; ++j) {
      uint4 y = ld<LD>(a.in[j] + v * 16, pol);
      s.x += y.x; s.y += y.y; s.z += y.z; s.w += y.w;
    }
    if (a.out) st<ST>(a.out + v * 16, s, pol);
    else sink += s.x ^ s.y ^ s.z ^ s.w;
  }
  if (sink == 0x12345678u) ((volatile uint32_t*)a.in[0])[0] = sink;  // keep the loads alive
}

typedef void (*KernFn)(const Args);

struct Case {
  const char* name;
  KernFn fn;
  int nin;
  bool write;
};

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t sizes[] = {220000000ull, 1419292672ull, 25ull << 20};
  // one big allocation for 9 streams of the largest size, plus separate allocations mode
  const size_t maxb = 1419292672ull;
  char* big = nullptr;
  CK(cudaMalloc(&big, maxb * 9 + 4096));
  CK(cudaMemset(big, 1, maxb * 9 + 4096));
  std::vector<Case> cases = {
      {"copy_ldg_gs", probe<1, 0, 0, 0, 4>, 1, true},
      {"copy_ldg_cs_gs", probe<1, 0, 1, 0, 4>, 1, true},
      {"read1_gs", probe<1, 0, 0, 0, 4>, 1, false},
      {"read8_gs", probe<8, 0, 0, 0, 1>, 8, false},
      {"r8w1_ldg_gs", probe<8, 0, 0, 0, 1>, 8, true},
      {"r8w1_nc_gs", probe<8, 1, 0, 0, 1>, 8, true},
      {"r8w1_evf_gs", probe<8, 2, 0, 0, 1>, 8, true},
      {"r8w1_256B_gs", probe<8, 3, 0, 0, 1>, 8, true},
      {"r8w1_ldg_stcs_gs", probe<8, 0, 1, 0, 1>, 8, true},
      {"r8w1_evf_stevf_gs", probe<8, 2, 2, 0, 1>, 8, true},
      {"r8w1_ldg_gs_u2", probe<8, 0, 0, 0, 2>, 8, true},
      {"r8w1_ldg_chunk", probe<8, 0, 0, 1, 1>, 8, true},
      {"r8w1_256B_chunk", probe<8, 3, 0, 1, 1>, 8, true},
      {"r8w1_ldg_chunk_u2", probe<8, 0, 0, 1, 2>, 8, true},
  };
  const int reps = 20;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (size_t sz : sizes) {
    for (const Case& c : cases) {
      for (int per_sm : {1, 2, 4, 5, 8}) {
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, c.fn, 256, 0));
        if (per_sm > occ) continue;
        Args a{};
        for (int j = 0; j < 8; ++j) a.in[j] = big + (size_t)j * sz;
        a.out = c.write ? big + (size_t)8 * sz : nullptr;
        a.nvec = sz / 16;
        a.nin = c.nin;
        const int grid = sms * per_sm;
        for (int w = 0; w < 3; ++w) c.fn<<<grid, 256>>>(a);
        CK(cudaDeviceSynchronize());
        std::vector<float> ts;  // back-to-back launches (no host gaps), average per launch
        for (int r = 0; r < 5; ++r) {
          CK(cudaEventRecord(e0));
          for (int k = 0; k < reps; ++k) c.fn<<<grid, 256>>>(a);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          ts.push_back(ms / reps);
        }
        CK(cudaGetLastError());
        std::sort(ts.begin(), ts.end());
        const double med = ts[ts.size() / 2];
        const double bytes = (double)sz * (c.nin + (c.write ? 1 : 0));
        printf("{\"case\": \"%s\", \"stream_bytes\": %zu, \"grid\": %d, \"ctas_per_sm\": %d, "
               "\"ms\": %.4f, \"ms_min\": %.4f, \"GBs\": %.1f, \"GBs_best\": %.1f}\n",
               c.name, sz, grid, per_sm, med, ts[0], bytes / (med * 1e-3) / 1e9,
               bytes / (ts[0] * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
  }
  CK(cudaFree(big));
  return 0;
}
