// The bare 8:1 read:write stream of tools/hbm_probe3.cu as a ctypes-callable launcher, so that
// tools/k2_vs_pattern.py can time it on the very buffers K2 reduces (integer adds, no method
// arithmetic: a memory-pattern ceiling, not a product kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o pattern.so tools/pattern_kernel.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint4 ldp(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
struct PArgs { const char* in[16]; char* out; size_t nvec; };

template <int NR>
__global__ void __launch_bounds__(256) pattern(const PArgs a) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.nvec; v += stride) {
    uint4 x[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) x[j] = ldp(a.in[j] + v * 16);
    uint4 s = x[0];
#pragma unroll
    for (int j = 1; j < NR; ++j) { s.x += x[j].x; s.y += x[j].y; s.z += x[j].z; s.w += x[j].w; }
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a.out + v * 16),
                 "r"(s.x), "r"(s.y), "r"(s.z), "r"(s.w) : "memory");
  }
}

extern "C" int pattern_launch(const void* const* in, int nr, void* out, size_t bytes, int grid,
                              void* stream) {
  PArgs a{};
  for (int j = 0; j < nr; ++j) a.in[j] = static_cast<const char*>(in[j]);
  a.out = static_cast<char*>(out);
  a.nvec = bytes / 16;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nr == 8) pattern<8><<<grid, 256, 0, st>>>(a);
  else if (nr == 3) pattern<3><<<grid, 256, 0, st>>>(a);
  else return 1;
  return (int)cudaGetLastError();
}
