// fhv_internal.h -- host-side plumbing shared by the .cu translation units:
// the per-device scratch arena (fhv_ctx) and kernel-launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fhv_b200.h"

namespace fhv {

// directory tiles of the POFA offsets pass: 2^14 leaves (fhv_scan.cu k_dir_tma)
constexpr int kDirSumShift = 14;

// internal status: a speculatively planned capture's item buffers were too
// small (never returned to callers: the capture re-plans with a sync)
constexpr int FHV_RETRY_ITEMS = 100;

// small device-resident control block (one per ctx)
struct Control {
  int status;                     // sticky FHV_* code raised by kernels
  int pad;
  unsigned long long items_total; // work items of the current capture
  unsigned long long frags_total; // fragments counted by pass 1
  unsigned long long alloc;       // FHV_ALLOC_ATOMIC slot counter / pass-2 emitted
  unsigned long long kx, ky;      // splat footprint maxima
  unsigned long long scan_total;  // last scan total
  unsigned int tile_counter;      // decoupled look-back tile ticket
  unsigned int pad2;
  unsigned long long spare[8];
  unsigned long long leaf_n[3];  // EXACT_ORDER POFA: leaves listed for re-sorting (small, mid, big)
  unsigned int dir_ticket, dir_done;  // k_dir_stream: tile tickets, CTAs finished (zeroed before each launch)
};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace fhv

namespace fhv {
// profiled stages (one per kernel family); names in fhv_abi.cu
enum Stage {
  kStJobSetup = 0, kStScan, kStItemExpand, kStCount, kStCountLeaves, kStEmitList, kStEmitPpfl, kStEmitPofl,
  kStEmitPofa, kStChainOrder, kStLeafOrder, kStScanLeaves, kStPyramid, kStSplatDepth, kStSplatIndex,
  kStSplatResolve, kStRaycast, kStFaceNormals, kStDeferred, kStOps, kStScalar, kStLeafSort, kStRaycastHandoff,
  kNumStages
};
struct PendingEvent {
  int stage;
  cudaEvent_t e0, e1;
};
}  // namespace fhv

struct fhv_ctx {
  int device = 0;
  bool prof = false;
  std::vector<fhv::PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  double stage_ms[fhv::kNumStages] = {};
  long long stage_count[fhv::kNumStages] = {};
  fhv::DevBuf bufs[32];  // >= kNumBufs
  fhv::Control* ctl = nullptr;       // device
  fhv::Control* ctl_host = nullptr;  // pinned mirror
  int64_t launches = 0;
  // state carried from fhv_pofa_count to fhv_pofa_scatter
  int64_t n_jobs = 0, n_items = 0, pass1_total = 0;
  int32_t pass1_levels = -1;
  bool pass1_ranks = true;  // pass 1 scanned emission ranks (needed by an EXACT_ORDER scatter)
  int64_t pass1_tris = -1;
  uint64_t pass1_lo = 0, pass1_hi = 0;
  int64_t n_binned = -1;  // triangles kept by the last shard binning (-1: no binning)
  // what that binning ran on (the speculative sharded build reuses it without
  // a sync when the triangle arrays and the shard are the same)
  const void* bin_pos = nullptr;
  int64_t bin_n_tri = -1;
  uint64_t bin_sig = 0;
  // speculative capture planning (fhv_capture.cu plan()): item buffers sized by
  // the last exact plan with the same job count; spec = current plan is one
  int64_t item_cap = 0, last_n_jobs = -1;
  bool spec = false;
  // fragments per work item of the last synchronised capture (selects the
  // raster passes' arithmetic path, fhv_capture.cu use_fast_math)
  double frags_per_item = 0.0;
  // levels of the directory tile totals the last counting pass left in
  // bufs[kTileSums] (-1: none; consumed by scan_leaves_and_pyramid)
  int dir_sums_levels = -1;
  // an item-rank scan (bufs[kItemCnt] -> bufs[kItemOff]) the counting pass
  // deferred to the directory launch: item count (-1: none) and its
  // device-side count (speculative plan) or null
  int64_t item_scan_n = -1;
  const unsigned long long* item_scan_dev = nullptr;
  bool dir_frags_total = false;  // the directory launch also sets ctl->frags_total (asynchronous build)
  bool dir_frags_stored = false;  // ... and it did (the fused tile-total launch ran)
  // inside an asynchronous POFA build after its control-block reset: the
  // counters that reset zeroed (alloc, leaf_n, dir_done) need no clears of their own
  bool ctl_fresh = false;
  // side stream of the asynchronous build: the leaf-counter and cursor
  // clears run there, off the critical path, joined before their first use
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool join_pending = false;
  const void* counts_zeroed = nullptr;   // buffers the side stream cleared for this build
  const void* cursors_zeroed = nullptr;
  void* fork_cursors_at_count = nullptr;  // clear these cursors on the side stream at the counting pass
  int last_cuda_error = 0;
};

namespace fhv {

enum BufId {
  kJobs = 0, kJobItems, kJobItemOff, kItemJob, kItemP0, kItemCnt, kItemOff, kScanStatus,
  kCursors, kChainScratch, kSplatKey, kSplatWin, kSplatBox, kRays, kTmp0, kTmp1, kTriFlag, kTriOff, kTriIndex,
  kShardBoxes, kItemMask, kJobPersp, kLeafList, kLeafKeys, kLeafRecs, kTileSums, kJobTileSums, kNumBufs
};

// Counts a launch and, when profiling is on, brackets it with CUDA events on
// the launching stream:  { LaunchScope L(ctx, kStCount, s); k<<<...>>>(); }
struct LaunchScope {
  fhv_ctx* ctx;
  int stage;
  cudaStream_t s;
  cudaEvent_t e0 = nullptr;
  LaunchScope(fhv_ctx* c, int st, cudaStream_t stream);
  ~LaunchScope();
};

// grow-only scratch; returns nullptr on allocation failure
void* scratch(fhv_ctx* ctx, BufId id, size_t bytes);
int check_cuda(fhv_ctx* ctx, cudaError_t e);
int sync_control(fhv_ctx* ctx, cudaStream_t s);  // copies ctl -> ctl_host, syncs, returns status
int reset_control(fhv_ctx* ctx, cudaStream_t s);

// exclusive scans (decoupled look-back, single pass); total lands in ctl->scan_total
// n_dev: optional device-side element count (<= n) for a speculatively sized launch
int scan_u32_to_u64(fhv_ctx* ctx, const uint32_t* in, unsigned long long* out, int64_t n, cudaStream_t s,
                    const unsigned long long* n_dev = nullptr, bool write_total = true);
// POFA directory: offsets = excl-scan(counts), pyramid level L-1 from counts > 0, then upper levels
// (+ a pending deferred item-rank scan, ctx->item_scan_n)
int scan_leaves_and_pyramid(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                            int levels, cudaStream_t s);
// speculative capture plan: job item counts -> offsets + the item records in
// one launch (item total -> ctl->items_total; FHV_RETRY_ITEMS past cap)
// job_tile_sums: the job setup's per-tile item totals (kExpandTileJobs jobs
// per tile): the tiles then need no look-back chain; null: ticket order + look-back
constexpr int kExpandTileJobs = 1024;
int scan_expand_items(fhv_ctx* ctx, const uint32_t* job_items, unsigned long long* job_item_off, int64_t n_jobs,
                      uint32_t* item_job, uint32_t* item_p0, unsigned long long cap, uint32_t item_pix,
                      cudaStream_t s, const uint32_t* job_tile_sums = nullptr);
// join the side stream's clears into `s` (no-op when nothing is pending)
int join_aux(fhv_ctx* ctx, cudaStream_t s);
// zero `bytes` at buf (and buf2) on the side stream after the work queued on `s`; join with join_aux
int fork_clear(fhv_ctx* ctx, void* buf, size_t bytes, cudaStream_t s, void* buf2);
// the deferred item-rank scan on its own (no-op when none is pending)
int run_deferred_item_scan(fhv_ctx* ctx, cudaStream_t s);
// leaves per directory tile (4096 for L = 4, 32768 for L >= 5, 0 below): shard ranges are multiples
long long dir_tile_leaves(int levels);
// shard variant: counts/offsets cover leaves [lo, hi) (multiples of dir_tile_leaves); stored offsets get
// + base; the pyramid must be zeroed by the caller and receives this shard's occupancy only
int scan_leaf_range_and_pyramid(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                                int levels, uint64_t lo, uint64_t hi, uint64_t base, cudaStream_t s);
int pyramid_from_heads(fhv_ctx* ctx, const int32_t* heads, uint8_t* pyramid, int levels, cudaStream_t s);
int pyramid_upper_levels(fhv_ctx* ctx, uint8_t* pyramid, int levels, cudaStream_t s);
// deferred_baseline lighting pass over the G-buffer the geometry pass left (fhv_splat.cu)
int deferred_resolve(fhv_ctx* ctx, long long P, const fhv_shading_t* sh, const double* eye,
                     const unsigned long long* key, const uint32_t* win, const fhv_gbuffer_t* gb, const double* bg,
                     double* out_rgba, double* out_depth, cudaStream_t s);

}  // namespace fhv
