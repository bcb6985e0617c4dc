// fhv_lookback.cuh -- single-pass scan building blocks shared by the scan
// kernels (fhv_scan.cu) and the fused job-setup + item-offset pass
// (fhv_capture.cu): dynamic tile tickets, a block-wide exclusive scan and the
// warp-parallel decoupled look-back over a per-tile status word array
// (flag bits 62..63: aggregate / inclusive prefix; the array is zeroed
// before each launch).
#pragma once

#include <cstdint>

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

// dynamic tile ticket (tiles start in ticket order: the decoupled look-back
// never waits on a tile that has not started).  The block drawing the last
// of the launch's n tickets puts the counter back to 0 -- every ticket is
// drawn by then -- so no memset precedes the next scan on this ctx (the
// counter starts at 0 with the ctx and after every reset_control).
__device__ __forceinline__ unsigned draw_tile(Control* ctl, unsigned n_launched) {
  const unsigned t = atomicAdd(&ctl->tile_counter, 1u);
  if (t == n_launched - 1) atomicExch(&ctl->tile_counter, 0u);
  return t;
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

// decoupled look-back, warp-parallel: warp 0 of the tile resolves the
// exclusive prefix of `tile`, inspecting 32 predecessors per step.  Returns
// the prefix in every lane of warp 0.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, unsigned tile, uint64_t agg) {
  const unsigned lane = threadIdx.x & 31u;
  if (tile == 0) {
    if (lane == 0) st_volatile(&status[0], kFlagPre | agg);
    return 0;
  }
  if (lane == 0) st_volatile(&status[tile], kFlagAgg | agg);
  uint64_t prefix = 0;
  long long base = (long long)tile - 1;
  while (true) {
    const long long k = base - (long long)lane;
    uint64_t s = kFlagPre;  // before tile 0: an inclusive prefix of 0
    if (k >= 0) {
      do { s = ld_volatile(&status[k]); } while ((s & ~kValMask) == 0);
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (s & ~kValMask) == kFlagPre);
    const unsigned stop = pre ? (unsigned)(__ffs(pre) - 1) : 31u;
    uint64_t v = lane <= stop ? (s & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (pre) break;
    base -= 32;
  }
  if (lane == 0) st_volatile(&status[tile], kFlagPre | ((prefix + agg) & kValMask));
  return prefix;
}

// decoupled look-back with the whole block: every thread inspects one
// predecessor, so one step covers BLOCK tiles (a tile of the first wave walks
// back to tile 0 in n / BLOCK round trips instead of n / 32).  Called by all
// threads; returns the exclusive prefix in every thread.
template <int BLOCK>
__device__ __forceinline__ uint64_t lookback_block(uint64_t* status, unsigned tile, uint64_t agg) {
  __shared__ uint64_t red_s[BLOCK / 32];
  __shared__ int near_s[BLOCK / 32];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (tile == 0) {
    if (threadIdx.x == 0) st_volatile(&status[0], kFlagPre | agg);
    return 0;
  }
  if (threadIdx.x == 0) st_volatile(&status[tile], kFlagAgg | agg);
  uint64_t prefix = 0;
  long long top = (long long)tile - 1;  // the highest predecessor of this step
  while (true) {
    const long long k = top - (long long)threadIdx.x;
    uint64_t s = kFlagPre;  // before tile 0: an inclusive prefix of 0
    if (k >= 0) {
      do { s = ld_volatile(&status[k]); } while ((s & ~kValMask) == 0);
    }
    // the nearest inclusive prefix among this step's predecessors (lowest thread index)
    const bool pre = (s & ~kValMask) == kFlagPre;
    const unsigned bal = __ballot_sync(0xffffffffu, pre);
    if (lane == 0) near_s[warp] = bal ? (int)(32 * warp + __ffs(bal) - 1) : BLOCK;
    __syncthreads();
    int near = BLOCK;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) near = min(near, near_s[w]);
    // sum of the values from the step's top down to (and including) the nearest inclusive
    uint64_t v = (int)threadIdx.x <= near ? (s & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red_s[warp] = v;
    __syncthreads();
    uint64_t tot = 0;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) tot += red_s[w];
    prefix += tot;
    __syncthreads();  // red_s / near_s reused by the next step
    if (near < BLOCK) break;
    top -= BLOCK;
  }
  if (threadIdx.x == 0) st_volatile(&status[tile], kFlagPre | ((prefix + agg) & kValMask));
  return prefix;
}

}  // namespace
}  // namespace fhv
