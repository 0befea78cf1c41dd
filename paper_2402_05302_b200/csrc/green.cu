// Bench utility (not the method): DISJOINT SM partitions of one GPU as streams of CUDA green
// contexts -- the emulation harness of heterogeneous ranks that share one GPU, the single-GPU
// analog of the paper's Cluster C (one GPU shared by several jobs) and of north_star's
// "per-rank compute-rate caps (... SM-partitioned contexts)".  torch's GreenContext.create(n)
// cuts every context from the whole device, so several of them overlap; here the device is split
// once into 8-SM groups and every partition is a union of its own groups, so rank i's kernels run
// on its own SMs only.  The driver API is reached through cudaGetDriverEntryPoint: no link
// dependency on libcuda (the library still loads on a machine without a driver).
#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

#include "common.h"
#include "ctx.h"

using cannikin::fail;

namespace {

typedef CUresult (*PFN_getRes)(CUdevice, CUdevResource*, CUdevResourceType);
typedef CUresult (*PFN_split)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                              unsigned int, unsigned int);
typedef CUresult (*PFN_desc)(CUdevResourceDesc*, CUdevResource*, unsigned int);
typedef CUresult (*PFN_gcreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
typedef CUresult (*PFN_gstream)(CUstream*, CUgreenCtx, unsigned int, int);
typedef CUresult (*PFN_gdestroy)(CUgreenCtx);
typedef CUresult (*PFN_sdestroy)(CUstream);

template <typename F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

}  // namespace

struct cannikin_green {
  std::vector<CUgreenCtx> ctx;
  std::vector<CUstream> stream;
  PFN_gdestroy gdestroy = nullptr;
  PFN_sdestroy sdestroy = nullptr;
};

extern "C" cannikin_status cannikin_green_partitions(int device, int n, const int* sm_counts,
                                                     cannikin_green** out, void** streams,
                                                     int* sm_got) {
  if (!out || !streams || !sm_counts || !sm_got || n < 1 || n > 64)
    return fail(CANNIKIN_ERR_INVALID, "green_partitions: bad arguments");
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess || cudaFree(nullptr) != cudaSuccess)  // primary ctx
    return fail(CANNIKIN_ERR_CUDA, "green_partitions: device %d", device);
  PFN_getRes get_res;
  PFN_split split;
  PFN_desc gen_desc;
  PFN_gcreate gcreate;
  PFN_gstream gstream;
  auto* g = new cannikin_green();
  if (!entry("cuDeviceGetDevResource", &get_res) || !entry("cuDevSmResourceSplitByCount", &split) ||
      !entry("cuDevResourceGenerateDesc", &gen_desc) || !entry("cuGreenCtxCreate", &gcreate) ||
      !entry("cuGreenCtxStreamCreate", &gstream) || !entry("cuGreenCtxDestroy", &g->gdestroy) ||
      !entry("cuStreamDestroy", &g->sdestroy)) {
    delete g;
    return fail(CANNIKIN_ERR_UNSUPPORTED, "green_partitions: driver without green contexts");
  }
  // one split of the whole device into groups of kGran SMs (disjoint by construction); partition
  // i is the union of the next ceil(sm_counts[i] / kGran) groups (a descriptor may combine
  // outputs of one split -- further splits of a split's output are not allowed)
  constexpr unsigned kGran = 8;  // sm_90+ granularity (cuda.h)
  CUdevResource whole;
  CUresult r = get_res((CUdevice)device, &whole, CU_DEV_RESOURCE_TYPE_SM);
  std::vector<CUdevResource> grp(whole.sm.smCount / kGran + 1);
  unsigned int ngrp = (unsigned)grp.size() - 1;
  CUdevResource remaining;
  if (r == CUDA_SUCCESS) r = split(grp.data(), &ngrp, &whole, &remaining, 0, kGran);
  unsigned next = 0;
  for (int i = 0; i < n && r == CUDA_SUCCESS; ++i) {
    const unsigned need = sm_counts[i] < 1 ? 0 : ((unsigned)sm_counts[i] + kGran - 1) / kGran;
    if (need == 0 || next + need > ngrp) {
      for (CUstream st : g->stream) g->sdestroy(st);
      for (CUgreenCtx c : g->ctx) g->gdestroy(c);
      delete g;
      return fail(CANNIKIN_ERR_UNSUPPORTED,
                  "green_partitions: the device splits into %u groups of %u SMs; partitions 0..%d "
                  "need more", ngrp, kGran, i);
    }
    CUdevResourceDesc desc;
    r = gen_desc(&desc, &grp[next], need);
    if (r != CUDA_SUCCESS) break;
    unsigned got = 0;
    for (unsigned k = 0; k < need; ++k) got += grp[next + k].sm.smCount;
    next += need;
    CUgreenCtx gc;
    r = gcreate(&gc, desc, (CUdevice)device, CU_GREEN_CTX_DEFAULT_STREAM);
    if (r != CUDA_SUCCESS) break;
    g->ctx.push_back(gc);
    CUstream s;
    r = gstream(&s, gc, CU_STREAM_NON_BLOCKING, 0);
    if (r != CUDA_SUCCESS) break;
    g->stream.push_back(s);
    streams[i] = s;
    sm_got[i] = (int)got;
  }
  if (r != CUDA_SUCCESS) {
    for (CUstream s : g->stream) g->sdestroy(s);
    for (CUgreenCtx c : g->ctx) g->gdestroy(c);
    delete g;
    return fail(CANNIKIN_ERR_UNSUPPORTED, "green_partitions: driver error %d (SM counts too large "
                "for the device, or not multiples of the architecture's granularity)", (int)r);
  }
  *out = g;
  return CANNIKIN_OK;
}

extern "C" cannikin_status cannikin_green_destroy(cannikin_green* g) {
  if (!g) return CANNIKIN_OK;
  for (CUstream s : g->stream) g->sdestroy(s);
  for (CUgreenCtx c : g->ctx) g->gdestroy(c);
  delete g;
  return CANNIKIN_OK;
}
