// HBM probe, part 3: does the RELATIVE placement of the 9 streams of an 8:1 read:write pass
// matter?  tools/hbm_probe.cu (streams 220,000,000 B apart) measured 6.19 TB/s, hbm_probe2.cu
// (219,938,816 B apart, a multiple of 256 KiB) 6.86 TB/s for the same kernel and grid.  Here the
// streams are placed `stride` bytes apart in one allocation, stride = round_up(size, 2 MiB) +
// delta, for a sweep of delta; and as 9 separate cudaMalloc allocations (what torch does).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_probe3 tools/hbm_probe3.cu
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

static double timeit(const Args& a, int grid) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) r8w1_ldg<<<grid, 256>>>(a);
  CK(cudaDeviceSynchronize());
  std::vector<float> ts;
  const int reps = 20;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    for (int k = 0; k < reps; ++k) r8w1_ldg<<<grid, 256>>>(a);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ts.push_back(ms / reps);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ts[2];
}

int main() {
  CK(cudaSetDevice(0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t MB2 = 2u << 20;
  const size_t sizes[2] = {220000000ull, 1419292672ull};
  const long deltas[] = {0,       4096,    65536,   131072,  262144,  393216, 524288,  786432,
                         1048576, 1310720, 1572864, 1835008, 61184,   -262144, 1896192, 256,
                         8192,    16384,   32768};
  for (size_t sz : sizes) {
    const size_t sz16 = sz / 16 * 16;
    const size_t base_stride = (sz + MB2 - 1) / MB2 * MB2;
    char* big = nullptr;
    CK(cudaMalloc(&big, (base_stride + 2 * MB2) * 9 + MB2));
    CK(cudaMemset(big, 1, (base_stride + 2 * MB2) * 9 + MB2));
    for (long d : deltas) {
      const size_t stride = base_stride + MB2 + d;  // + 2 MiB so negative deltas stay apart
      Args a{};
      for (int j = 0; j < 8; ++j) a.in[j] = big + (size_t)j * stride;
      a.out = big + (size_t)8 * stride;
      a.nvec = sz16 / 16;
      for (int per_sm : {3, 4, 5}) {
        const double ms = timeit(a, sms * per_sm);
        printf("{\"size\": %zu, \"placement\": \"one_alloc\", \"delta\": %ld, \"grid\": %d, \"ms\": %.4f, "
               "\"GBs\": %.1f}\n",
               sz16, d, sms * per_sm, ms, 9.0 * sz16 / (ms * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
    // also the exact offsets of the first probes: streams `sz` apart (no rounding)
    {
      Args a{};
      for (int j = 0; j < 8; ++j) a.in[j] = big + (size_t)j * sz16;
      a.out = big + (size_t)8 * sz16;
      a.nvec = sz16 / 16;
      for (int per_sm : {3, 4, 5}) {
        const double ms = timeit(a, sms * per_sm);
        printf("{\"size\": %zu, \"placement\": \"packed\", \"delta\": null, \"grid\": %d, \"ms\": %.4f, "
               "\"GBs\": %.1f}\n",
               sz16, sms * per_sm, ms, 9.0 * sz16 / (ms * 1e-3) / 1e9);
        fflush(stdout);
      }
    }
    CK(cudaFree(big));
    // separate allocations (torch-like)
    char* p[9];
    for (int j = 0; j < 9; ++j) {
      CK(cudaMalloc(&p[j], sz16));
      CK(cudaMemset(p[j], 1, sz16));
    }
    Args a{};
    for (int j = 0; j < 8; ++j) a.in[j] = p[j];
    a.out = p[8];
    a.nvec = sz16 / 16;
    for (int per_sm : {3, 4, 5}) {
      const double ms = timeit(a, sms * per_sm);
      printf("{\"size\": %zu, \"placement\": \"separate\", \"delta\": null, \"grid\": %d, \"ms\": %.4f, "
             "\"GBs\": %.1f, \"offsets_mod_2MB\": [%zu,%zu,%zu]}\n",
             sz16, sms * per_sm, ms, 9.0 * sz16 / (ms * 1e-3) / 1e9, (size_t)p[0] % MB2,
             (size_t)p[1] % MB2, (size_t)p[8] % MB2);
      fflush(stdout);
    }
    for (int j = 0; j < 9; ++j) CK(cudaFree(p[j]));
  }
  return 0;
}
