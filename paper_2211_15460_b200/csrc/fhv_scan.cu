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

namespace fhv {

namespace {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) {
  *reinterpret_cast<volatile uint64_t*>(p) = v;
}

// block-wide exclusive scan of one u64 per thread; returns exclusive value,
// writes the block total to *total
template <int BLOCK>
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t* total) {
  __shared__ uint64_t warp_tot[BLOCK / 32];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint64_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (unsigned)o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < BLOCK / 32 ? warp_tot[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (unsigned)o) wi += y;
    }
    if (lane < BLOCK / 32) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == BLOCK / 32 - 1) *total = wi;
  }
  __syncthreads();
  return warp_tot[warp] + inc - x;
}

// decoupled look-back: thread 0 resolves the exclusive prefix of `tile`
__device__ __forceinline__ uint64_t lookback(uint64_t* status, unsigned tile, uint64_t agg) {
  if (tile == 0) {
    st_volatile(&status[0], kFlagPre | agg);
    return 0;
  }
  st_volatile(&status[tile], kFlagAgg | agg);
  uint64_t prefix = 0;
  int k = (int)tile - 1;
  while (true) {
    uint64_t s;
    do { s = ld_volatile(&status[k]); } while ((s & ~kValMask) == 0);
    prefix += s & kValMask;
    if ((s & ~kValMask) == kFlagPre) break;
    --k;
  }
  st_volatile(&status[tile], kFlagPre | ((prefix + agg) & kValMask));
  return prefix;
}

template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_scan_u32_u64(const uint32_t* __restrict__ in,
                                                       unsigned long long* __restrict__ out, int64_t n,
                                                       uint64_t* status, Control* ctl, unsigned n_tiles) {
  __shared__ unsigned tile_s;
  __shared__ uint64_t prefix_s, total_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(&ctl->tile_counter, 1u);
  __syncthreads();
  const unsigned tile = tile_s;
  const int64_t base = (int64_t)tile * BLOCK * ITEMS + (int64_t)threadIdx.x * ITEMS;
  uint32_t v[ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    v[i] = base + i < n ? in[base + i] : 0u;
    sum += v[i];
  }
  const uint64_t excl = block_excl_scan<BLOCK>(sum, &total_s);
  if (threadIdx.x == 0) prefix_s = lookback(status, tile, total_s);
  __syncthreads();
  uint64_t run = prefix_s + excl;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
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
  if (threadIdx.x == 0) tile_s = atomicAdd(&ctl->tile_counter, 1u);
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
  if (threadIdx.x == 0) prefix_s = lookback(status, tile, total_s);
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

int scan_u32_to_u64(fhv_ctx* ctx, const uint32_t* in, unsigned long long* out, int64_t n, cudaStream_t s) {
  constexpr int B = 256, I = 8;
  const int64_t per = (int64_t)B * I;
  const unsigned tiles = (unsigned)((n + per - 1) / per);
  if (n <= 0) {
    return check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->scan_total, 0, sizeof(unsigned long long), s));
  }
  uint64_t* st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
  if (!st) return FHV_NOMEM;
  int rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s));
  if (rc) return rc;
  rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->tile_counter, 0, sizeof(unsigned), s));
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStScan, s);
    k_scan_u32_u64<B, I><<<tiles, B, 0, s>>>(in, out, n, st, ctx->ctl, tiles);
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

int scan_leaves_and_pyramid(fhv_ctx* ctx, const uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                            int levels, cudaStream_t s) {
  constexpr int B = 256;
  const int64_t n_nodes = 1ll << (3 * (levels - 1));
  const unsigned tiles = (unsigned)((n_nodes + B - 1) / B);
  uint64_t* st = (uint64_t*)scratch(ctx, kScanStatus, (size_t)tiles * sizeof(uint64_t));
  if (!st) return FHV_NOMEM;
  int rc = check_cuda(ctx, cudaMemsetAsync(st, 0, (size_t)tiles * sizeof(uint64_t), s));
  if (rc) return rc;
  rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->tile_counter, 0, sizeof(unsigned), s));
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

int pyramid_from_heads(fhv_ctx* ctx, const int32_t* heads, uint8_t* pyramid, int levels, cudaStream_t s) {
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
