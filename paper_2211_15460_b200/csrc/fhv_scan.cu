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
#include "fhv_common.cuh"
#include "fhv_internal.h"
#include "fhv_lookback.cuh"

namespace fhv {

namespace {

template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_scan_u32_u64(const uint32_t* __restrict__ in,
                                                       unsigned long long* __restrict__ out, int64_t n,
                                                       uint64_t* status, Control* ctl, unsigned n_tiles,
                                                       const unsigned long long* n_dev) {
  __shared__ unsigned tile_s;
  __shared__ uint64_t prefix_s, total_s;
  if (threadIdx.x == 0) tile_s = draw_tile(ctl, n_tiles);
  __syncthreads();
  const unsigned tile = tile_s;
  if (n_dev) {  // speculatively sized launch: tiles past the device count retire at once
    if ((int64_t)*n_dev < n) n = (int64_t)*n_dev;
    n_tiles = (unsigned)((n + (int64_t)BLOCK * ITEMS - 1) / ((int64_t)BLOCK * ITEMS));
    if (tile >= n_tiles) {
      if (tile == 0 && threadIdx.x == 0) ctl->scan_total = 0;
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
  if (threadIdx.x == 0 && tile == n_tiles - 1) ctl->scan_total = prefix_s + total_s;
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
                    const unsigned long long* n_dev) {
#ifndef FHV_SCAN_B
#define FHV_SCAN_B 512
#define FHV_SCAN_I 16
#endif
  constexpr int B = FHV_SCAN_B, I = FHV_SCAN_I;  // 8192 elements per tile: a short look-back chain
  const int64_t per = (int64_t)B * I;
  const unsigned tiles = (unsigned)((n + per - 1) / per);
  if (n <= 0) {
    return check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->scan_total, 0, sizeof(unsigned long long), s));
  }
  uint64_t* st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
  if (!st) return FHV_NOMEM;
  int rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s));
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStScan, s);
    k_scan_u32_u64<B, I><<<tiles, B, 0, s>>>(in, out, n, st, ctx->ctl, tiles, n_dev);
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

int scan_leaves_and_pyramid(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                            int levels, cudaStream_t s) {
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
