// Internal definition of cannikin_ctx and of the per-rank control region that lives at the start
// of every rank's peer-mapped allocation.  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>

#include "cannikin.h"

namespace cannikin {

constexpr int kMaxWorld = CANNIKIN_MAX_WORLD;
constexpr int kMaxArBlocks = 256;      // grid cap of the two-shot kernel
constexpr size_t kPushAutoBytes = (size_t)128 << 20;  // push two-shot from this bucket size (W >= 4)
constexpr int kMaxArChunks = 2048;     // partial-table rows per source rank (dynamic two-shot)
constexpr int kMaxLocalBlocks = 2048;  // grid cap of the emulated-rank kernel
constexpr int kMaxEmu = CANNIKIN_MAX_EMULATED;

// Control region of one rank.  Fields marked [peer] are written by peers over NVLink; fields
// marked [local] only by this rank's own kernels.  Flags carry monotonically increasing epochs
// (never reset), so back-to-back buckets need no re-initialisation (no reset races).
struct Ctrl {
  uint64_t exit_[kMaxArBlocks][kMaxWorld];                   // [peer] "shard pushed" epoch
  uint64_t mid[kMaxArBlocks][kMaxWorld];                     // [peer] NVLS: "my piece is scaled"
  uint64_t nv_exit[kMaxArBlocks][kMaxWorld];                 // [peer] NVLS: "my stores landed"
  uint64_t nv_epoch;                                         // [local] NVLS call counter
  uint64_t nv_meta[kMaxArBlocks][kMaxWorld];                 // [peer] NVLS: (bucket hash32, epoch32)
  uint64_t rv_word[kMaxArBlocks][kMaxWorld];                 // [peer] entry: (float r_src, epoch32)
  uint64_t meta_word[kMaxArBlocks][kMaxWorld];               // [peer] entry: (bucket hash32, epoch32)
  uint64_t pmid[kMaxArBlocks][kMaxWorld];                    // [peer] push variant: (r_src, epoch32)
  uint64_t gate[kMaxWorld];                                  // [peer] gated entry: epoch of rank j
  uint64_t gate_epoch;                                       // [local] gated calls so far
  uint64_t ll_epoch;                                         // [local] LL-kernel call counter
  unsigned ticket_ll;                                        // [local] LL last-CTA ticket
  uint64_t ll128_epoch;                                      // [local] LL128-kernel call counter
  unsigned ticket_ll128;                                     // [local] LL128 last-CTA ticket
  double part[kMaxWorld][kMaxArChunks][kMaxWorld + 1];       // [peer] norm partials [src][row][j]
  uint64_t epoch[kMaxArBlocks];                              // [local] per-block epoch counter
  unsigned ticket_ar;                                        // [local] last-block-done ticket
  unsigned ticket_local;
  unsigned ar_counter;                                       // [local] dynamic two-shot chunk counter
  int error_code;                                            // [local] protocol error (trap reason)
  double rsum_bad;                                           // [local] offending sum_j r_j (code 7)
  double stats[kMaxWorld + 1];                               // [local] accumulated |g_j|^2, |g|^2
  double cta_acc[kMaxArBlocks][kMaxWorld + 1];               // [local] per-CTA running stats
  uint64_t trace[kMaxLocalBlocks][5];                        // [local] per-CTA timeline (ns)
  int trace_grid;                                            // [local] CTAs of the last traced kernel
  double local_part[kMaxLocalBlocks][kMaxEmu + 1];           // [local] emulated-kernel partials
};

}  // namespace cannikin

struct cannikin_ctx {
  int rank = 0, world = 1, device = 0;
  int grid_ar = 148;
  int ar_dyn = -1;          // CANNIKIN_AR_DYN=0|1 forces static/dynamic chunks; -1 = by size
  int ar_push = -1;         // CANNIKIN_AR_PUSH=0|1 forces pull / push; -1 = by size
  int check_ratios = 0;     // CANNIKIN_INIT_CHECK_RATIOS
  bool gated = false;       // CANNIKIN_INIT_GATED_ENTRY: one-warp peer wait before each reduction
  int ar_chunk_max = 512 * 16;  // CANNIKIN_AR_CHUNK: dynamic two-shot max chunk (16-B vectors)
  int ar_ll = -1;           // CANNIKIN_AR_LL=0|1 forbids/prefers the LL kernel; -1 = by size
  size_t ll_max_bytes = 0;  // largest LL bucket = its slot payload: 1 MiB / (W - 1), 64 KiB steps
  int ar_ll128 = -1;        // CANNIKIN_AR_LL128=0|1 forbids/prefers the LL128 kernel; -1 = by size
  size_t ll128_max_bytes = 0;  // largest LL128 bucket (CANNIKIN_LL128_MAX_MB), sizes its slots
  int grid_local = 0;       // 0 = occupancy-derived grid for the LDG variant of K2
  bool local_tma = false;   // default variant of K2 (CANNIKIN_K2_IMPL=tma|ldg)
  int local_nt = 256;       // CANNIKIN_K2_NT: CTA size of K2 (256, or one big CTA per SM)
  int num_sms = 148;
  size_t heap_bytes = 0;
  // local allocation = [Ctrl | user heap (heap_bytes) | scratch (heap_bytes)]
  char* base = nullptr;
  size_t ctrl_bytes = 0, user_off = 0, scratch_off = 0, stage_off = 0, ll_off = 0, ll128_off = 0, total_bytes = 0;
  char* peer_base[cannikin::kMaxWorld] = {};
  cannikin::Ctrl* ctrl = nullptr;
  void* nccl_comm = nullptr;  // ncclComm_t
  void* k4_buf = nullptr;     // NCCL-path (K4) work buffer, grown on demand
  size_t k4_bytes = 0;
  char* work_buf = nullptr;   // cannikin_gns_stats_bucket: out-of-place copy + held statistics
  size_t work_bytes = 0;
  bool in_process = false;    // cannikin_init_group_local: peers are this process's allocations
  std::map<size_t, size_t> free_blocks;  // offset -> size within the user heap
  std::map<size_t, size_t> used_blocks;
  double* h_stats = nullptr;  // pinned host staging for gns_stats
  int last_launches = 0;
  const char* last_variant = "";  // kernel variant of the last hot-path call (diagnostics)
  // peer-wait timeout (dev::SpinClock): 0 = wait forever (multi-process default, as NCCL);
  // in-process groups default to 20 s; CANNIKIN_SPIN_TIMEOUT_MS overrides either
  uint64_t spin_timeout_ns = 0;
};
