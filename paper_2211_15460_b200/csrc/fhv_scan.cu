// fhv_scan.cu -- single-pass exclusive scans (decoupled look-back) and the
// occupancy-pyramid builders.
//
//  * scan_u32_to_u64: per-job / per-item counts -> 64-bit exclusive offsets
//    (the fragment ranks that reproduce the reference pool order).
//  * scan_leaves_and_pyramid: the POFA directory, fhv/storage.py:604-608 and
//    :620 (offsets = [0] + cumsum(counts[:-1]); pyramid from counts > 0).
//    One thread owns one level-(L-1) node = 8 consecutive leaves (two 16-B
//    loads), so the leaf pass reads counts once and writes offsets + the
//    bottom mask level in the same sweep: 8 B/leaf + 1/8 B/leaf of HBM.
//  * pyramid_from_heads: POFL occupancy (equal to incremental set_paths,
//    fhv/storage.py:294-301, SURVEY probe) from heads >= 0.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "fhv_common.cuh"
#include "fhv_internal.h"
#include "fhv_lookback.cuh"

namespace fhv {

namespace {

// one tile of the u32 -> u64 exclusive scan (ticket order, decoupled
// look-back); write_total: the last tile stores the total in ctl->scan_total
template <int BLOCK, int ITEMS>
__device__ __forceinline__ void scan_tile_u32_u64(const uint32_t* __restrict__ in, unsigned long long* __restrict__ out,
                                                  int64_t n, uint64_t* status, Control* ctl, unsigned n_tiles,
                                                  const unsigned long long* n_dev, bool write_total) {
  __shared__ unsigned tile_s;
  __shared__ uint64_t prefix_s, total_s;
  if (threadIdx.x == 0) tile_s = draw_tile(ctl, n_tiles);
  __syncthreads();
  const unsigned tile = tile_s;
  if (n_dev) {  // speculatively sized launch: tiles past the device count retire at once
    if ((int64_t)*n_dev < n) n = (int64_t)*n_dev;
    n_tiles = (unsigned)((n + (int64_t)BLOCK * ITEMS - 1) / ((int64_t)BLOCK * ITEMS));
    if (tile >= n_tiles) {
      if (write_total && tile == 0 && threadIdx.x == 0) ctl->scan_total = 0;
      return;
    }
  }
  const int64_t base = (int64_t)tile * BLOCK * ITEMS + (int64_t)threadIdx.x * ITEMS;
  uint32_t v[ITEMS];
  uint64_t sum = 0;
  const bool vec = ITEMS % 4 == 0 && base + ITEMS <= n && ((uintptr_t)(in + base) & 15) == 0;
  if (vec) {  // 16-B loads: a thread's ITEMS consecutive counts
#pragma unroll
    for (int i = 0; i < ITEMS; i += 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(in + base + i);
      v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) v[i] = base + i < n ? in[base + i] : 0u;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) sum += v[i];
  const uint64_t excl = block_excl_scan<BLOCK>(sum, &total_s);
  if (threadIdx.x < 32) {
    const uint64_t pf = lookback_warp(status, tile, total_s);
    if (threadIdx.x == 0) prefix_s = pf;
  }
  __syncthreads();
  uint64_t run = prefix_s + excl;
  if (vec && ((uintptr_t)(out + base) & 15) == 0) {  // 16-B stores
#pragma unroll
    for (int i = 0; i < ITEMS; i += 2) {
      const unsigned long long a = run;
      run += v[i];
      *reinterpret_cast<ulonglong2*>(out + base + i) = make_ulonglong2(a, run);
      run += v[i + 1];
    }
  } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (base + i < n) out[base + i] = run;
      run += v[i];
    }
  }
  if (write_total && threadIdx.x == 0 && tile == n_tiles - 1) ctl->scan_total = prefix_s + total_s;
}

template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_scan_u32_u64(const uint32_t* __restrict__ in,
                                                       unsigned long long* __restrict__ out, int64_t n,
                                                       uint64_t* status, Control* ctl, unsigned n_tiles,
                                                       const unsigned long long* n_dev, int write_total) {
  scan_tile_u32_u64<BLOCK, ITEMS>(in, out, n, status, ctl, n_tiles, n_dev, write_total != 0);
}

// job item counts -> item offsets AND the item records in one pass (the
// speculative capture plan, fhv_capture.cu plan()): a tile of jobs is scanned
// (ticket order, decoupled look-back), then its jobs' items are written --
// small jobs by their own lane, big ones by the whole warp (ballot loop).
// The last tile stores the item total in ctl->items_total.
#ifndef FHV_EXP_ITEMS
#define FHV_EXP_ITEMS 4
#endif
constexpr int kExpBlock = 256, kExpItems = FHV_EXP_ITEMS;  // jobs per thread (tile = 256 x kExpItems jobs)
__global__ void __launch_bounds__(kExpBlock) k_item_scan_expand(const uint32_t* __restrict__ job_items,
                                                               unsigned long long* __restrict__ job_item_off,
                                                               int64_t n_jobs, uint32_t* __restrict__ item_job,
                                                               uint32_t* __restrict__ item_p0, unsigned long long cap,
                                                               uint32_t item_pix, uint64_t* status, Control* ctl,
                                                               unsigned n_tiles, const uint32_t* __restrict__ tsum) {
  constexpr int kT = kExpBlock * kExpItems;
  static_assert(kT == kExpandTileJobs, "tile totals match the tile");
  __shared__ unsigned tile_s;
  __shared__ uint64_t prefix_s, total_s, tsum_s;
  __shared__ uint32_t cnt_s[kT];
  __shared__ unsigned long long off_s[kT];
  if (threadIdx.x == 0) tile_s = tsum ? blockIdx.x : draw_tile(ctl, n_tiles);
  __syncthreads();
  const unsigned tile = tile_s;
  uint64_t pred = 0;  // with the job setup's tile totals: the predecessors' sum, no chain
  if (tsum)
    for (unsigned q = threadIdx.x; q < tile; q += kExpBlock) pred += tsum[q];
  const int64_t t0 = (int64_t)tile * kT;
  // counts striped (coalesced) into shared memory, scanned blocked
#pragma unroll
  for (int i = 0; i < kExpItems; ++i) {
    const int64_t j = t0 + i * kExpBlock + threadIdx.x;
    cnt_s[i * kExpBlock + threadIdx.x] = j < n_jobs ? job_items[j] : 0u;
  }
  __syncthreads();
  uint32_t v[kExpItems];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < kExpItems; ++i) {
    v[i] = cnt_s[threadIdx.x * kExpItems + i];
    sum += v[i];
  }
  const uint64_t excl = block_excl_scan<kExpBlock>(sum, &total_s);
  if (tsum) {
    (void)block_excl_scan<kExpBlock>(pred, &tsum_s);
    if (threadIdx.x == 0) {
      prefix_s = tsum_s;
      if (tsum[tile] != (uint32_t)total_s) raise_status(&ctl->status, FHV_PASS_MISMATCH);
    }
  } else if (threadIdx.x < 32) {
    const uint64_t pf = lookback_warp(status, tile, total_s);
    if (threadIdx.x == 0) prefix_s = pf;
  }
  __syncthreads();
  {
    uint64_t run = prefix_s + excl;
#pragma unroll
    for (int i = 0; i < kExpItems; ++i) {
      off_s[threadIdx.x * kExpItems + i] = run;
      run += v[i];
    }
  }
  if (threadIdx.x == 0 && tile == n_tiles - 1) ctl->items_total = prefix_s + total_s;
  __syncthreads();
  // offsets and items striped: consecutive lanes, consecutive jobs, consecutive items
  bool over = false;
#pragma unroll 1
  for (int i = 0; i < kExpItems; ++i) {
    const int q = i * kExpBlock + threadIdx.x;
    const int64_t j = t0 + q;
    const unsigned long long base = off_s[q];
    uint32_t n = cnt_s[q];
    if (j < n_jobs) job_item_off[j] = base;
    if (base + n > cap) {  // speculative item buffers too small: the host re-plans with a sync
      over = true;
      n = base < cap ? (uint32_t)(cap - base) : 0u;
    }
    if (n <= 4u) {
      for (uint32_t k = 0; k < n; ++k) {
        item_job[base + k] = (uint32_t)j;
        item_p0[base + k] = k * item_pix;
      }
    }
    unsigned big = __ballot_sync(0xffffffffu, n > 4u);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t bn = __shfl_sync(0xffffffffu, n, src);
      const unsigned long long bb = __shfl_sync(0xffffffffu, base, src);
      const uint32_t bj = (uint32_t)(j - (int64_t)(threadIdx.x & 31u) + src);
      for (uint32_t k = threadIdx.x & 31u; k < bn; k += 32) {
        item_job[bb + k] = bj;
        item_p0[bb + k] = k * item_pix;
      }
    }
  }
  if (over) raise_status(&ctl->status, FHV_RETRY_ITEMS);
}

// POFA leaves: thread = one level-(L-1) node (8 leaves)
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_scan_leaves(const uint4* __restrict__ counts, uint4* __restrict__ offsets,
                                                      uint8_t* __restrict__ last_level, int64_t n_nodes,
                                                      uint64_t* status, Control* ctl, unsigned n_tiles) {
  __shared__ unsigned tile_s;
  __shared__ uint64_t prefix_s, total_s;
  if (threadIdx.x == 0) tile_s = draw_tile(ctl, n_tiles);
  __syncthreads();
  const unsigned tile = tile_s;
  const int64_t node = (int64_t)tile * BLOCK + threadIdx.x;
  uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
  if (node < n_nodes) {
    a = __ldcs(&counts[2 * node]);
    b = __ldcs(&counts[2 * node + 1]);
  }
  const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint64_t sum = 0;
  unsigned mask = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    sum += v[i];
    mask |= (v[i] != 0u ? 1u : 0u) << i;
  }
  const uint64_t excl = block_excl_scan<BLOCK>(sum, &total_s);
  if (threadIdx.x < 32) {
    const uint64_t pf = lookback_warp(status, tile, total_s);
    if (threadIdx.x == 0) prefix_s = pf;
  }
  __syncthreads();
  if (node < n_nodes) {
    uint64_t run = prefix_s + excl;
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = (uint32_t)run;
      run += v[i];
    }
    __stcs(&offsets[2 * node], make_uint4(o[0], o[1], o[2], o[3]));
    __stcs(&offsets[2 * node + 1], make_uint4(o[4], o[5], o[6], o[7]));
    last_level[node] = (uint8_t)mask;
  }
  if (threadIdx.x == 0 && tile == n_tiles - 1) ctl->scan_total = prefix_s + total_s;
}

// Directory tiles: one CTA = one subtree of 8^K leaves (WARPS warps x ITERS
// iterations x 32 lanes x 8 leaves; K = 4 or 5).  A lane owns one
// level-(L-1) node (8 consecutive leaves, two 16-B loads) per iteration, so
// the tile writes pyramid level L-1 (lane masks), L-2 (warp ballots), L-3
// (ballot pairs) from registers and the levels up to its root (L-K) through
// shared memory; for POFA it also writes offsets = base + exclusive scan of
// counts (warp running scan + decoupled tile look-back).  The last tile to
// finish builds levels L-K-1..0 from the tile roots.  One pass over the
// directory: 8 B/leaf (POFA) or 4 B/leaf (POFL heads) of HBM plus 8^L/7
// pyramid bytes.  Bigger tiles shorten the look-back chain (one L2 round
// trip per 32 tiles on the critical path).
template <int WARPS, int ITERS>
struct DirTile {
  static constexpr int kThreads = 32 * WARPS;
  static constexpr long long kLeaves = 8LL * 32 * WARPS * ITERS;
  static constexpr int kL3 = WARPS * ITERS / 2;  // level-(L-3) nodes per tile
  static constexpr int kK = kLeaves == 4096 ? 4 : (kLeaves == 32768 ? 5 : -1);
  static_assert(kK > 0, "tile must be a whole octree subtree");
};
using DirSmall = DirTile<4, 4>;   // 8^4 leaves
using DirBig = DirTile<16, 8>;    // 8^5 leaves

template <bool kScan, int WARPS, int ITERS>
__global__ void __launch_bounds__(32 * WARPS, WARPS <= 16 ? 2 : 1) k_dir_tiles(const uint4* __restrict__ counts,
                                                          uint4* __restrict__ offsets,
                                                          const int4* __restrict__ heads, uint8_t* __restrict__ pyr,
                                                          int levels, uint64_t* status, Control* ctl,
                                                          unsigned n_tiles, unsigned tile0, uint64_t base) {
  using T = DirTile<WARPS, ITERS>;
  __shared__ unsigned tile_s;
  __shared__ uint64_t warp_tot[WARPS];
  __shared__ uint64_t prefix_s;
  __shared__ uint8_t lvl_s[2][T::kL3];
  __shared__ int last_s;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) tile_s = kScan ? draw_tile(ctl, n_tiles) : blockIdx.x;
  __syncthreads();
  const unsigned tile = tile_s;        // tile within the range (scan order)
  const unsigned gtile = tile0 + tile;  // level-(L-K) node in the whole tree
  uint8_t* lv1 = pyr + pyr_level_offset(levels - 1);
  uint8_t* lv2 = pyr + pyr_level_offset(levels - 2);
  uint8_t* lv3 = pyr + pyr_level_offset(levels - 3);
  // local node index (counts / offsets / heads) and global node index (pyramid)
  const long long node0 = (long long)tile * (T::kLeaves / 8) + (long long)warp * (32 * ITERS);
  const long long gnode0 = (long long)gtile * (T::kLeaves / 8) + (long long)warp * (32 * ITERS);
  // phase 1, in chunks of kChunk iterations (loads of a chunk in flight
  // together, registers bounded): leaf masks -> pyramid levels L-1..L-3, lane
  // sums -> lane-exclusive prefixes within the warp's slice (u32: a directory
  // holds < 2^32 fragments).  The counts are re-read after the tile look-back
  // (L2 hits) instead of being held across it -> 2 CTAs per SM.
  constexpr int kChunk = ITERS < 4 ? ITERS : 4;
  static_assert(ITERS % kChunk == 0 && kChunk % 2 == 0, "chunking");
  unsigned ballots[ITERS];
  uint32_t excl[ITERS];
  uint64_t carry = 0;
#pragma unroll
  for (int h = 0; h < ITERS; h += kChunk) {
    uint32_t c[kChunk][8];
#pragma unroll
    for (int q = 0; q < kChunk; ++q) {
      const long long n = node0 + (h + q) * 32 + lane;
      if (kScan) {
        const uint4 a = __ldcg(&counts[2 * n]), b = __ldcg(&counts[2 * n + 1]);
        c[q][0] = a.x; c[q][1] = a.y; c[q][2] = a.z; c[q][3] = a.w;
        c[q][4] = b.x; c[q][5] = b.y; c[q][6] = b.z; c[q][7] = b.w;
      } else {
        const int4 a = __ldcs(&heads[2 * n]), b = __ldcs(&heads[2 * n + 1]);
        const int v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) c[q][k] = v[k] >= 0 ? 1u : 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < kChunk; ++q) {
      const int i = h + q;
      unsigned m = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) m |= (c[q][k] != 0u ? 1u : 0u) << k;
      lv1[gnode0 + i * 32 + lane] = (uint8_t)m;
      ballots[i] = __ballot_sync(0xffffffffu, m != 0);
      // level L-2: lane g < 4 writes node (gnode0 + 32 i) / 8 + g
      if (lane < 4) lv2[(gnode0 + 32 * i) / 8 + lane] = (uint8_t)((ballots[i] >> (8 * lane)) & 0xffu);
      if (kScan) {
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) sum += c[q][k];
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= (unsigned)o) inc += y;
        }
        excl[i] = (uint32_t)carry + inc - sum;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
  }
  // level L-3: iterations (2j, 2j+1) -> one node; bit g = L-2 node g non-empty
#pragma unroll
  for (int j = 0; j < ITERS / 2; ++j) {
    if (lane == (unsigned)j) {
      const unsigned lo = ballots[2 * j], hi = ballots[2 * j + 1];
      unsigned m = 0;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        m |= (((lo >> (8 * g)) & 0xffu) != 0 ? 1u : 0u) << g;
        m |= (((hi >> (8 * g)) & 0xffu) != 0 ? 1u : 0u) << (g + 4);
      }
      lv3[gnode0 / 64 + j] = (uint8_t)m;
      lvl_s[0][warp * (ITERS / 2) + j] = (uint8_t)m;
    }
  }
  if (kScan) {
    if (lane == 0) warp_tot[warp] = carry;
    __syncthreads();
    if (warp == 0) {
      uint64_t t = 0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) t += warp_tot[w];
      const uint64_t pf = lookback_warp(status, tile, t);
      if (lane == 0) {
        prefix_s = pf;
        if (tile == n_tiles - 1) ctl->scan_total = pf + t;
      }
    }
    __syncthreads();
    uint64_t wbase = prefix_s + base;
    for (unsigned w = 0; w < warp; ++w) wbase += warp_tot[w];
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      const long long n = node0 + i * 32 + lane;
      const uint4 a = __ldcg(&counts[2 * n]), b = __ldcg(&counts[2 * n + 1]);
      const uint32_t cc[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint64_t run = wbase + excl[i];
      uint32_t o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        o[k] = (uint32_t)run;
        run += cc[k];
      }
      __stcs(&offsets[2 * n], make_uint4(o[0], o[1], o[2], o[3]));
      __stcs(&offsets[2 * n + 1], make_uint4(o[4], o[5], o[6], o[7]));
    }
  } else {
    __syncthreads();
  }
  // levels L-4 .. L-K (the tile root) through shared memory
  int cur = 0, n_cur = T::kL3, lvl = levels - 3;
  while (n_cur > 1) {
    const int n_up = n_cur / 8;
    --lvl;
    if ((int)threadIdx.x < n_up) {
      unsigned m = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) m |= (lvl_s[cur][8 * threadIdx.x + b] != 0 ? 1u : 0u) << b;
      lvl_s[cur ^ 1][threadIdx.x] = (uint8_t)m;
      pyr[pyr_level_offset(lvl) + (long long)gtile * n_up + threadIdx.x] = (uint8_t)m;
    }
    cur ^= 1;
    n_cur = n_up;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(&ctl->spare[1], 1ull);
    last_s = done == (unsigned long long)n_tiles - 1;
    if (last_s) ctl->spare[1] = 0;  // every tile has counted itself: ready for the next pass
  }
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  for (int k = levels - T::kK - 1; k >= 0; --k) {
    const long long nn = 1ll << (3 * k);
    const uint8_t* below = pyr + pyr_level_offset(k + 1);
    uint8_t* out = pyr + pyr_level_offset(k);
    for (long long j = threadIdx.x; j < nn; j += blockDim.x) {
      unsigned m = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) m |= (__ldcg(&below[8 * j + b]) != 0 ? 1u : 0u) << b;
      out[j] = (uint8_t)m;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// POFA directory through TMA tensor copies (L >= 5).  The counts are viewed
// as a 2-D tensor of 128-B rows (32 leaves); one CTA owns a tile of kDbChunks
// x 256 rows (kDbChunks x 32 KB, whole level-(L-4) subtrees).  Thread 0 puts
// the whole tile in flight at once -- one cp.async.bulk.tensor per 32-KB
// chunk, each completing on its own mbarrier, 128-B swizzled so that thread
// t's row (its 32 consecutive leaves) reads conflict-free -- and every thread
// processes chunk j as soon as it lands: pyramid levels L-1..L-4 (L-5 too
// for 4 chunks) from registers / shuffles / ballots, per-chunk block scans;
// the decoupled tile look-back, then the offsets are written in place into
// the same swizzled buffers and stored back with cp.async.bulk.tensor
// (shared -> global).  Counts are read from HBM exactly once, 8 B per leaf of
// traffic in 32-KB TMA transfers; the last CTA builds the levels above.
constexpr int kDbThreads = 256;
constexpr int kDbRows = 256;                         // 128-B rows per chunk (one per thread)
constexpr int kDbLeaves = kDbRows * 32;              // 8192 leaves per chunk
constexpr int kDbBytes = kDbLeaves * 4;              // 32 KB
#ifndef FHV_DIR_CHUNKS
#define FHV_DIR_CHUNKS 2
#endif
constexpr int kDbChunks = FHV_DIR_CHUNKS;            // chunks per CTA tile (1, 2 or 4)
constexpr long long kDbTile = (long long)kDbChunks * kDbLeaves;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(smem)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int c1, const void* smem) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tm), "r"(c0),
               "r"(c1), "r"(smem_u32(smem))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16-B unit q of row t inside a 128-B-swizzled chunk (CU_TENSOR_MAP_SWIZZLE_128B)
__device__ __forceinline__ uint4* swz(uint32_t* chunk, unsigned t, unsigned q) {
  return reinterpret_cast<uint4*>(reinterpret_cast<char*>(chunk) + t * 128u + ((q ^ (t & 7u)) << 4));
}

static_assert(kDbTile == (1ll << kDirSumShift) || kDbChunks != 2, "tile totals match the tile");

// deferred item-rank scan riding in the directory launch (k_dir_tma)
struct ItemScan {
  const uint32_t* cnt;
  unsigned long long* off;
  int64_t n;
  const unsigned long long* n_dev;
  uint64_t* status;
  unsigned tiles;  // 0: none
  int frags_total;  // the last directory tile also stores the total in ctl->frags_total
};
constexpr int kItemScanItems = 32;  // 256 x 32 = 8192 items per tile

#ifndef FHV_DIR_MINB
#define FHV_DIR_MINB 3
#endif
__global__ void __launch_bounds__(kDbThreads, FHV_DIR_MINB) k_dir_tma(const __grid_constant__ CUtensorMap tm_counts,
                                                         const __grid_constant__ CUtensorMap tm_offsets,
                                                         uint8_t* __restrict__ pyr, int levels, uint64_t* status,
                                                         Control* ctl, unsigned n_tiles, unsigned tile0,
                                                         uint64_t base, const uint32_t* __restrict__ tile_sums,
                                                         ItemScan is) {
  // the first is.tiles CTAs scan the items' fragment counts into emission
  // ranks (their own tickets and look-back; the directory tiles below use
  // blockIdx with the counting pass's tile totals): two independent scans of
  // one counting pass in one launch, the ranks' look-back chain hidden
  // behind the directory's streaming
  if (blockIdx.x < is.tiles) {
    scan_tile_u32_u64<kDbThreads, kItemScanItems>(is.cnt, is.off, is.n, is.status, ctl, is.tiles, is.n_dev, false);
    return;
  }
  extern __shared__ __align__(1024) unsigned char dyn[];  // kDbChunks x 32 KB, 1024-B aligned (swizzle atoms)
  uint32_t* buf = reinterpret_cast<uint32_t*>(dyn + ((1024u - (smem_u32(dyn) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t bar[kDbChunks];
  __shared__ unsigned tile_s;
  __shared__ uint64_t prefix_s, ctot_s[kDbChunks];
  __shared__ uint8_t l3_s[kDbChunks][kDbThreads / 16];
  __shared__ int last_s;
  const unsigned tid = threadIdx.x, lane = tid & 31u;
  if (tid == 0) {
    // with the counting pass's tile totals the tiles are independent (blockIdx);
    // else ticket order: the look-back never waits on an unstarted tile
    const unsigned t = tile_sums ? blockIdx.x - is.tiles : draw_tile(ctl, n_tiles);
    tile_s = t;
    for (int j = 0; j < kDbChunks; ++j) mbar_init(&bar[j], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < kDbChunks; ++j) {  // the whole tile in flight at once, one barrier per 32-KB chunk
      mbar_expect_tx(&bar[j], kDbBytes);
      tma_load_2d(buf + j * kDbLeaves, &tm_counts, 0, (int)((long long)t * kDbChunks * kDbRows + j * kDbRows), &bar[j]);
    }
  }
  __syncthreads();
  const unsigned tile = tile_s;
  const unsigned gtile = tile0 + tile;
  uint64_t excl[kDbChunks];
#pragma unroll
  for (int j = 0; j < kDbChunks; ++j) {  // chunk j: leaves [j * 8192, (j + 1) * 8192) of the tile; my row = tid
    mbar_wait(&bar[j], 0);
    uint32_t* cb = buf + j * kDbLeaves;
    uint32_t sum = 0;
    uint32_t m1 = 0;  // my 4 level-(L-1) node masks
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 v = *swz(cb, tid, q);
      sum += v.x + v.y + v.z + v.w;
      m1 |= ((v.x != 0u ? 1u : 0u) | (v.y != 0u ? 2u : 0u) | (v.z != 0u ? 4u : 0u) | (v.w != 0u ? 8u : 0u)) << (4 * q);
    }
    const long long node1 = ((long long)gtile * kDbChunks + j) * (kDbLeaves / 8) + 4 * tid;
    {  // (level offsets (8^k - 1) / 7 are not 4-B aligned: byte stores)
      uint8_t* l1 = pyr + pyr_level_offset(levels - 1) + node1;
#pragma unroll
      for (int nd = 0; nd < 4; ++nd) l1[nd] = (uint8_t)(m1 >> (8 * nd));
    }
    // level L-2: node = 8 level-(L-1) nodes = 2 threads
    const unsigned my4 = ((m1 & 0xffu) != 0 ? 1u : 0u) | ((m1 & 0xff00u) != 0 ? 2u : 0u) |
                         ((m1 & 0xff0000u) != 0 ? 4u : 0u) | ((m1 & 0xff000000u) != 0 ? 8u : 0u);
    const unsigned pair = my4 | (__shfl_down_sync(0xffffffffu, my4, 1) << 4);
    if ((lane & 1u) == 0) pyr[pyr_level_offset(levels - 2) + node1 / 8] = (uint8_t)pair;
    // level L-3: node = 8 level-(L-2) nodes = 16 threads
    const unsigned occ = __ballot_sync(0xffffffffu, (lane & 1u) == 0 && pair != 0u);
    if ((lane & 15u) == 0) {
      const unsigned h = (occ >> lane) & 0xffffu;
      unsigned m3 = 0;
#pragma unroll
      for (int g = 0; g < 8; ++g) m3 |= ((h >> (2 * g)) & 1u) << g;
      pyr[pyr_level_offset(levels - 3) + node1 / 64] = (uint8_t)m3;
      l3_s[j][tid / 16] = (uint8_t)m3;
    }
    excl[j] = block_excl_scan<kDbThreads>((uint64_t)sum, &ctot_s[j]);
  }
  uint64_t t_all = 0;
#pragma unroll
  for (int j = 0; j < kDbChunks; ++j) t_all += ctot_s[j];
  uint64_t pf;
  if (tile_sums) {  // prefix = the predecessors' totals (a block sum), no chain
    uint64_t v = 0;
    for (unsigned q = tid; q < tile; q += kDbThreads) v += tile_sums[q];
    __shared__ uint64_t tsum_s;
    uint64_t dummy = block_excl_scan<kDbThreads>(v, &tsum_s);
    (void)dummy;
    pf = tsum_s;
    if (tid == 0 && tile_sums[tile] != (uint32_t)t_all) raise_status(&ctl->status, FHV_PASS_MISMATCH);
  } else {
    pf = lookback_block<kDbThreads>(status, tile, t_all);  // the whole block looks back
  }
  if (tid < 32) {
    if (lane == 0) {
      prefix_s = pf;
      if (tile == n_tiles - 1) {
        ctl->scan_total = pf + t_all;
        if (is.frags_total) ctl->frags_total = pf + t_all;  // (the asynchronous build's pass-2 count)
      }
    }
    if (lane < 2 * kDbChunks) {  // level L-4: two subtree roots per chunk
      unsigned m4 = 0;
#pragma unroll
      for (int g = 0; g < 8; ++g) m4 |= (l3_s[lane / 2][8 * (lane & 1) + g] != 0 ? 1u : 0u) << g;
      pyr[pyr_level_offset(levels - 4) + (long long)gtile * 2 * kDbChunks + lane] = (uint8_t)m4;
      const unsigned m4all = __ballot_sync((1u << (2 * kDbChunks)) - 1u, m4 != 0u);
      if (lane == 0 && kDbChunks == 4) pyr[pyr_level_offset(levels - 5) + gtile] = (uint8_t)m4all;  // tile root
    }
  }
  __syncthreads();
  uint64_t cbase = base + prefix_s;
#pragma unroll
  for (int j = 0; j < kDbChunks; ++j) {
    uint64_t run = cbase + excl[j];
    cbase += ctot_s[j];
    uint32_t* cb = buf + j * kDbLeaves;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint4* p4 = swz(cb, tid, q);
      const uint4 v = *p4;
      uint4 o;
      o.x = (uint32_t)run; run += v.x;
      o.y = (uint32_t)run; run += v.y;
      o.z = (uint32_t)run; run += v.z;
      o.w = (uint32_t)run; run += v.w;
      *p4 = o;
    }
  }
  fence_proxy_async();  // my generic-proxy writes -> visible to the tensor copies
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < kDbChunks; ++j)
      tma_store_2d(&tm_offsets, 0, (int)((long long)tile * kDbChunks * kDbRows + j * kDbRows), buf + j * kDbLeaves);
    bulk_commit();
    bulk_wait_read<0>();  // the copy engine has read the buffers: shared memory may be released
    __threadfence();
    const unsigned done = atomicAdd(&ctl->dir_done, 1u);
    last_s = done == n_tiles - 1;
  }
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  for (int k = levels - (kDbChunks == 4 ? 6 : 5); k >= 0; --k) {  // levels above what the tiles wrote
    const long long nn = 1ll << (3 * k);
    const uint8_t* below = pyr + pyr_level_offset(k + 1);
    uint8_t* out = pyr + pyr_level_offset(k);
    for (long long jj = tid; jj < nn; jj += blockDim.x) {
      unsigned m = 0;
#pragma unroll
      for (int b2 = 0; b2 < 8; ++b2) m |= (__ldcg(&below[8 * jj + b2]) != 0 ? 1u : 0u) << b2;
      out[jj] = (uint8_t)m;
    }
    __syncthreads();
  }
}

// one pyramid level from the level below: node k at level l has children
// 8k..8k+7 at level l+1 (one 8-byte load)
__global__ void k_pyramid_up(const uint64_t* __restrict__ below, uint8_t* __restrict__ level, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t c = below[i];
    unsigned m = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) m |= (((c >> (8 * b)) & 0xffull) != 0 ? 1u : 0u) << b;
    level[i] = (uint8_t)m;
  }
}

// level L-1 from POFL heads (>= 0 means occupied)
__global__ void k_pyramid_heads(const int4* __restrict__ heads, uint8_t* __restrict__ level, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 a = __ldcs(&heads[2 * i]), b = __ldcs(&heads[2 * i + 1]);
    const int v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    unsigned m = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) m |= (v[k] >= 0 ? 1u : 0u) << k;
    level[i] = (uint8_t)m;
  }
}

// tiny levels (< 8 nodes below): level 0 when L == 1 handled by callers
__global__ void k_pyramid_up_small(const uint8_t* __restrict__ below, uint8_t* __restrict__ level, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned m = 0;
    for (int b = 0; b < 8; ++b) m |= (below[8 * i + b] != 0 ? 1u : 0u) << b;
    level[i] = (uint8_t)m;
  }
}

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

}  // namespace

int scan_u32_to_u64(fhv_ctx* ctx, const uint32_t* in, unsigned long long* out, int64_t n, cudaStream_t s,
                    const unsigned long long* n_dev, bool write_total) {
#ifndef FHV_SCAN_B
#define FHV_SCAN_B 512
#define FHV_SCAN_I 16
#endif
  constexpr int B = FHV_SCAN_B, I = FHV_SCAN_I;  // 8192 elements per tile: a short look-back chain
  const int64_t per = (int64_t)B * I;
  const unsigned tiles = (unsigned)((n + per - 1) / per);
  if (n <= 0) {
    if (!write_total) return FHV_OK;
    return check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->scan_total, 0, sizeof(unsigned long long), s));
  }
  uint64_t* st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
  if (!st) return FHV_NOMEM;
  int rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s));
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStScan, s);
    k_scan_u32_u64<B, I><<<tiles, B, 0, s>>>(in, out, n, st, ctx->ctl, tiles, n_dev, write_total ? 1 : 0);
  }
  return check_cuda(ctx, cudaGetLastError());
}

int pyramid_upper_levels(fhv_ctx* ctx, uint8_t* pyramid, int levels, cudaStream_t s) {
  for (int k = levels - 2; k >= 0; --k) {
    const int64_t n = 1ll << (3 * k);
    uint8_t* dst = pyramid + pyr_level_offset(k);
    const uint8_t* src = pyramid + pyr_level_offset(k + 1);
    // level k+1 starts at (8^(k+1)-1)/7, not 8-aligned in general -> byte loads
    {
      LaunchScope L_(ctx, kStPyramid, s);
      k_pyramid_up_small<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
    }
  }
  return check_cuda(ctx, cudaGetLastError());
}

// leaves per directory tile at depth `levels` (0: no tile kernel)
long long dir_tile_leaves(int levels) { return levels >= 5 ? DirBig::kLeaves : (levels == 4 ? DirSmall::kLeaves : 0); }

template <class T>
static void launch_dir(bool scan, unsigned tiles, unsigned tile0, const uint32_t* counts, uint32_t* offsets,
                       const int32_t* heads, uint8_t* pyramid, int levels, uint64_t* st, Control* ctl, uint64_t base,
                       cudaStream_t s) {
  constexpr int W = T::kThreads / 32, I = (int)(T::kLeaves / (8LL * T::kThreads));
  if (scan)
    k_dir_tiles<true, W, I><<<tiles, T::kThreads, 0, s>>>(reinterpret_cast<const uint4*>(counts),
                                                          reinterpret_cast<uint4*>(offsets), nullptr, pyramid, levels,
                                                          st, ctl, tiles, tile0, base);
  else
    k_dir_tiles<false, W, I><<<tiles, T::kThreads, 0, s>>>(nullptr, nullptr, reinterpret_cast<const int4*>(heads),
                                                           pyramid, levels, nullptr, ctl, tiles, 0u, 0ull);
}

static int launch_dir_tiles(fhv_ctx* ctx, bool scan, const uint32_t* counts, uint32_t* offsets, const int32_t* heads,
                            uint8_t* pyramid, int levels, cudaStream_t s, uint64_t lo = 0, uint64_t hi = 0,
                            uint64_t base = 0) {
  const long long tl = dir_tile_leaves(levels);
  if (hi == 0) hi = 1ull << (3 * levels);
  const unsigned tiles = (unsigned)((hi - lo) / (uint64_t)tl);
  const unsigned tile0 = (unsigned)(lo / (uint64_t)tl);
  if (tiles == 0) return FHV_OK;
  uint64_t* st = nullptr;
  if (scan) {
    st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
    if (!st) return FHV_NOMEM;
    int rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s));
    if (rc) return rc;
  }
  {
    LaunchScope L_(ctx, scan ? kStScanLeaves : kStPyramid, s);
    if (tl == DirBig::kLeaves)
      launch_dir<DirBig>(scan, tiles, tile0, counts, offsets, heads, pyramid, levels, st, ctx->ctl, base, s);
    else
      launch_dir<DirSmall>(scan, tiles, tile0, counts, offsets, heads, pyramid, levels, st, ctx->ctl, base, s);
  }
  return check_cuda(ctx, cudaGetLastError());
}

// the TMA tensor-copy directory (k_dir_tma); FHV_DIR_STREAM=0 selects k_dir_tiles (A/B)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2-D view of a u32 leaf array: rows of 32 leaves (128 B), boxes of 256 rows, 128-B swizzle
static bool rows_tensor_map(CUtensorMap* tm, const uint32_t* base, uint64_t n_leaves) {
  auto enc = tensor_map_encoder();
  if (!enc || n_leaves % 32) return false;
  const cuuint64_t dims[2] = {32, (cuuint64_t)(n_leaves / 32)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, (cuuint32_t)kDbRows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int launch_dir_bulk(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid, int levels,
                           cudaStream_t s, uint64_t lo, uint64_t hi, uint64_t base,
                           const uint32_t* tile_sums = nullptr, bool* ranks_done = nullptr) {
  const unsigned tiles = (unsigned)((hi - lo) / (uint64_t)kDbTile);
  const unsigned tile0 = (unsigned)(lo / (uint64_t)kDbTile);
  CUtensorMap tm_c, tm_o;
  if (!rows_tensor_map(&tm_c, counts + lo, hi - lo) || !rows_tensor_map(&tm_o, offsets + lo, hi - lo))
    return launch_dir_tiles(ctx, true, counts, offsets, nullptr, pyramid, levels, s, lo, hi, base);
  // a pending item-rank scan rides along (tile totals given: the directory
  // tiles take no tickets)
  ItemScan is{nullptr, nullptr, 0, nullptr, nullptr, 0u, ranks_done && tile_sums && ctx->dir_frags_total ? 1 : 0};
  const int64_t pend = ctx->item_scan_n;
  if (ranks_done && tile_sums && pend > 0) {
    is.cnt = (const uint32_t*)ctx->bufs[kItemCnt].ptr;
    is.off = (unsigned long long*)ctx->bufs[kItemOff].ptr;
    is.n = pend;
    is.n_dev = ctx->item_scan_dev;
    is.tiles = (unsigned)((pend + (int64_t)kDbThreads * kItemScanItems - 1) / ((int64_t)kDbThreads * kItemScanItems));
  }
  uint64_t* st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)(tiles + is.tiles) * sizeof(uint64_t));
  if (!st) return FHV_NOMEM;
  is.status = st + tiles;
  // (directory tiles with tile totals use no status words; a control block
  // fresh from this build's reset already holds a zero done counter)
  int rc = FHV_OK;
  const size_t st_words = tile_sums ? is.tiles : tiles + is.tiles;
  if (st_words && (rc = check_cuda(ctx, cudaMemsetAsync(tile_sums ? is.status : st, 0, st_words * sizeof(uint64_t), s))))
    return rc;
  if (!ctx->ctl_fresh && (rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->dir_ticket, 0, 8, s))))  // (done counter)
    return rc;
  constexpr int kSmem = kDbChunks * kDbBytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dir_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  {
    LaunchScope L_(ctx, kStScanLeaves, s);
    k_dir_tma<<<tiles + is.tiles, kDbThreads, kSmem, s>>>(tm_c, tm_o, pyramid, levels, st, ctx->ctl, tiles, tile0,
                                                            base, tile_sums, is);
  }
  if (ranks_done && is.tiles) *ranks_done = true;
  ctx->dir_frags_stored = is.frags_total != 0;
  return check_cuda(ctx, cudaGetLastError());
}

static bool dir_stream_enabled() {
  static const int v = [] {
    const char* e = std::getenv("FHV_DIR_STREAM");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return v != 0;
}

static int scan_leaves_and_pyramid_impl(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                                        int levels, cudaStream_t s, bool* ranks_done);

// + the item-rank scan a counting pass deferred to here (fhv_capture.cu
// count()): fused into the directory launch when it streams with tile totals,
// else its own scan first
int scan_leaves_and_pyramid(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                            int levels, cudaStream_t s) {
  const int64_t pend = ctx->item_scan_n;
  bool done = pend <= 0;
  int rc = scan_leaves_and_pyramid_impl(ctx, counts, offsets, pyramid, levels, s, done ? nullptr : &done);
  if (rc || done) {
    ctx->item_scan_n = -1;
    return rc;
  }
  return run_deferred_item_scan(ctx, s);  // not fused: its own scan (the directory's total stays)
}

int scan_expand_items(fhv_ctx* ctx, const uint32_t* job_items, unsigned long long* job_item_off, int64_t n_jobs,
                      uint32_t* item_job, uint32_t* item_p0, unsigned long long cap, uint32_t item_pix,
                      cudaStream_t s, const uint32_t* job_tile_sums) {
  const unsigned tiles = (unsigned)((n_jobs + (int64_t)kExpBlock * kExpItems - 1) / ((int64_t)kExpBlock * kExpItems));
  uint64_t* st = nullptr;
  int rc;
  if (!job_tile_sums) {
    st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
    if (!st) return FHV_NOMEM;
    if ((rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s)))) return rc;
  }
  {
    LaunchScope L_(ctx, kStItemExpand, s);
    k_item_scan_expand<<<tiles, kExpBlock, 0, s>>>(job_items, job_item_off, n_jobs, item_job, item_p0, cap, item_pix,
                                                   st, ctx->ctl, tiles, job_tile_sums);
  }
  return check_cuda(ctx, cudaGetLastError());
}

int run_deferred_item_scan(fhv_ctx* ctx, cudaStream_t s) {
  const int64_t pend = ctx->item_scan_n;
  ctx->item_scan_n = -1;
  if (pend <= 0) return FHV_OK;
  return scan_u32_to_u64(ctx, (const uint32_t*)ctx->bufs[kItemCnt].ptr, (unsigned long long*)ctx->bufs[kItemOff].ptr,
                         pend, s, ctx->item_scan_dev, false);
}

static int scan_leaves_and_pyramid_impl(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                                        int levels, cudaStream_t s, bool* ranks_done) {
  if (levels >= 5 && dir_stream_enabled()) {
    // the counting pass's per-tile totals, when it left them for this directory (one use)
    const uint32_t* sums = (ctx->dir_sums_levels == levels && kDbChunks == 2) ? (const uint32_t*)ctx->bufs[kTileSums].ptr
                                                                             : nullptr;
    ctx->dir_sums_levels = -1;
    return launch_dir_bulk(ctx, counts, offsets, pyramid, levels, s, 0, 1ull << (3 * levels), 0, sums, ranks_done);
  }
  if (levels >= 4) return launch_dir_tiles(ctx, true, counts, offsets, nullptr, pyramid, levels, s);
  constexpr int B = 256;
  const int64_t n_nodes = 1ll << (3 * (levels - 1));
  const unsigned tiles = (unsigned)((n_nodes + B - 1) / B);
  uint64_t* st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
  if (!st) return FHV_NOMEM;
  int rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s));
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStScanLeaves, s);
    k_scan_leaves<B><<<tiles, B, 0, s>>>(reinterpret_cast<const uint4*>(counts), reinterpret_cast<uint4*>(offsets),
                                       pyramid + pyr_level_offset(levels - 1), n_nodes, st, ctx->ctl, tiles);
  }
  rc = check_cuda(ctx, cudaGetLastError());
  if (rc) return rc;
  return pyramid_upper_levels(ctx, pyramid, levels, s);
}

int scan_leaf_range_and_pyramid(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                                int levels, uint64_t lo, uint64_t hi, uint64_t base, cudaStream_t s) {
  const long long tl = dir_tile_leaves(levels);
  if (tl == 0 || lo % (uint64_t)tl || hi % (uint64_t)tl || hi < lo || hi > (1ull << (3 * levels))) return FHV_BAD_ARGS;
  if (hi == lo) return check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->scan_total, 0, 8, s));
  return launch_dir_tiles(ctx, true, counts, offsets, nullptr, pyramid, levels, s, lo, hi, base);
}

int pyramid_from_heads(fhv_ctx* ctx, const int32_t* heads, uint8_t* pyramid, int levels, cudaStream_t s) {
  if (levels >= 4) return launch_dir_tiles(ctx, false, nullptr, nullptr, heads, pyramid, levels, s);
  const int64_t n_nodes = 1ll << (3 * (levels - 1));
  {
    LaunchScope L_(ctx, kStPyramid, s);
    k_pyramid_heads<<<grid_for(n_nodes, 256), 256, 0, s>>>(reinterpret_cast<const int4*>(heads),
                                                         pyramid + pyr_level_offset(levels - 1), n_nodes);
  }
  int rc = check_cuda(ctx, cudaGetLastError());
  if (rc) return rc;
  return pyramid_upper_levels(ctx, pyramid, levels, s);
}

}  // namespace fhv
