// NVLink ceiling probe for the K3 traffic patterns (two GPUs, one process, SM-driven copies over
// peer mappings).  Measures per-direction GB/s for:
//   read1   GPU0 reads from GPU1 (writes local)                 -- one direction loaded
//   write1  GPU0 writes into GPU1 (reads local)                 -- one direction loaded
//   read2   both GPUs read from each other at the same time     -- both directions
//   write2  both GPUs write into each other at the same time
//   mixed2  both GPUs read half and write half (the two-shot pull pattern: per direction, half
//           read responses and half writes)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_bw tools/nvlink_bw.cu
// Usage: ./nvlink_bw [MiB per direction, default 256] [grid, default 148] [threads, default 512]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <chrono>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));       \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// all-to-all writes: CTA c writes to peer (c % np); every GPU's egress = its whole buffer
struct Peers {
  uint4* dst[8];
};
__global__ void a2a_write_kernel(const uint4* __restrict__ src, Peers p, int np, size_t n_per) {
  const int k = blockIdx.x % np;
  const int cta = blockIdx.x / np, nct = gridDim.x / np;
  const uint4* s = src + (size_t)k * n_per;
  uint4* d = p.dst[k];
  const size_t stride = (size_t)nct * blockDim.x;
  size_t i = (size_t)cta * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n_per; i += 4 * stride) {
    uint4 a = s[i], b = s[i + stride], c = s[i + 2 * stride], e = s[i + 3 * stride];
    d[i] = a;
    d[i + stride] = b;
    d[i + 2 * stride] = c;
    d[i + 3 * stride] = e;
  }
  for (; i < n_per; i += stride) d[i] = s[i];
}

struct Job {
  int dev;
  const uint4* src;
  uint4* dst;
  size_t n;
};

static double run(const Job* jobs, int nj, int grid, int nt, cudaStream_t* st, int reps) {
  for (int w = 0; w < 2; ++w)
    for (int j = 0; j < nj; ++j) {
      CK(cudaSetDevice(jobs[j].dev));
      copy_kernel<<<grid, nt, 0, st[j]>>>(jobs[j].src, jobs[j].dst, jobs[j].n);
    }
  for (int j = 0; j < nj; ++j) CK(cudaStreamSynchronize(st[j]));
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r)
    for (int j = 0; j < nj; ++j) {
      CK(cudaSetDevice(jobs[j].dev));
      copy_kernel<<<grid, nt, 0, st[j]>>>(jobs[j].src, jobs[j].dst, jobs[j].n);
    }
  for (int j = 0; j < nj; ++j) CK(cudaStreamSynchronize(st[j]));
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count() / reps;
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? atol(argv[1]) : 256;
  const int grid = argc > 2 ? atoi(argv[2]) : 148;
  const int nt = argc > 3 ? atoi(argv[3]) : 512;
  const size_t bytes = mib << 20, n = bytes / 16;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    fprintf(stderr, "needs 2 GPUs\n");
    return 1;
  }
  uint4 *a[8], *b[8];
  cudaStream_t st[8];
  const int G = ndev > 8 ? 8 : ndev;
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < G; ++q)
      if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
  }
  const int reps = 20;
  const size_t h = n / 2;
  struct Case {
    const char* name;
    Job jobs[4];
    int nj;
    double dir_bytes;  // bytes per loaded direction per rep
  } cases[] = {
      {"read1", {{0, a[1], b[0], n}}, 1, (double)bytes},
      {"write1", {{0, a[0], b[1], n}}, 1, (double)bytes},
      {"read2", {{0, a[1], b[0], n}, {1, a[0], b[1], n}}, 2, (double)bytes},
      {"write2", {{0, a[0], b[1], n}, {1, a[1], b[0], n}}, 2, (double)bytes},
      // GPU d reads the first half of the peer's a, writes the second half of its own a into
      // the peer's b: per direction bytes/2 reads + bytes/2 writes
      {"mixed2",
       {{0, a[1], b[0], h}, {0, a[0] + h, b[1] + h, n - h}, {1, a[0], b[1], h},
        {1, a[1] + h, b[0] + h, n - h}},
       4,
       (double)bytes},
  };
  cudaStream_t st4[4];
  for (int j = 0; j < 4; ++j) {
    CK(cudaSetDevice(j / 2));
    CK(cudaStreamCreateWithFlags(&st4[j], cudaStreamNonBlocking));
  }
  for (auto& c : cases) {
    // mixed2 runs the read and write halves as concurrent kernels on separate streams per GPU
    cudaStream_t* s = c.nj == 4 ? st4 : st;
    Job jobs[4];
    for (int j = 0; j < c.nj; ++j) jobs[j] = c.jobs[j];
    if (c.nj == 2) {
      // stream j belongs to device jobs[j].dev
      s = st;
    }
    const double t = run(jobs, c.nj, c.nj == 4 ? grid / 2 : grid, nt, s, reps);
    printf("{\"case\": \"%s\", \"MiB_per_direction\": %zu, \"grid\": %d, \"threads\": %d, "
           "\"us\": %.1f, \"GBps_per_direction\": %.1f}\n",
           c.name, mib, grid, nt, t * 1e6, c.dir_bytes / t / 1e9);
  }
  if (G > 2) {
    // every GPU writes 1/(G-1) of its buffer into each peer's b (slot = its rank), all at once
    const int np = G - 1;
    const size_t n_per = n / np;
    const int gr = grid / np * np;
    for (int w = 0; w < 3 + reps; ++w) {
      if (w == 3) {
        for (int d = 0; d < G; ++d) CK(cudaStreamSynchronize(st[d]));
      }
      static std::chrono::steady_clock::time_point t0;
      if (w == 3) t0 = std::chrono::steady_clock::now();
      for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        Peers p{};
        int k = 0;
        for (int q = 0; q < G; ++q)
          if (q != d) p.dst[k++] = b[q] + (size_t)d * (n / G);
        a2a_write_kernel<<<gr, nt, 0, st[d]>>>(a[d], p, np, n_per < n / G ? n_per : n / G);
      }
      if (w == 3 + reps - 1) {
        for (int d = 0; d < G; ++d) CK(cudaStreamSynchronize(st[d]));
        const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
        const double egress = (double)(n_per < n / G ? n_per : n / G) * 16 * np;
        printf("{\"case\": \"a2a_write%d\", \"MiB_per_gpu\": %.1f, \"grid\": %d, \"threads\": %d, "
               "\"us\": %.1f, \"GBps_per_direction\": %.1f}\n",
               G, egress / (1 << 20), gr, nt, t * 1e6, egress / t / 1e9);
      }
    }
  }
  return 0;
}
