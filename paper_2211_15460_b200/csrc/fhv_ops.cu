// fhv_ops.cu -- the reference's per-call operator API (fhv/_backend.py:25-29,
// kernels() -> coverage / linked_insert / pofa_scatter), batched on the device.
//
// The capture drivers never call these (the fused capture kernels in
// fhv_capture.cu do the same work per fragment); they exist so that code
// written against `kernels()` keeps working with the B200 backend
// (paper_2211_15460_b200/kernels.py), with the reference's semantics:
//   coverage       fhv/_ckern.pyx:25-105  (= fhv/_kernels_py.py:17-66)
//   linked_insert  fhv/_ckern.pyx:112-123 (sequential chaining order)
//   pofa_scatter   fhv/_ckern.pyx:126-143 (first bad index, cursors advanced
//                                          only for the fragments before it)
#include "fhv_common.cuh"
#include "fhv_internal.h"

namespace fhv {

namespace {

constexpr int kCovBlock = 128;

// per-triangle raster setup of coverage(): area2, edges, top-left flags and
// the clipped pixel-centre bounding box (computed in f64 before any integer
// conversion, so huge coordinates clamp instead of overflowing)
struct CovTri {
  double ax, ay, bx, by, cx, cy, area2;
  double d0x, d0y, d1x, d1y, d2x, d2y;
  bool tl0, tl1, tl2;
  long long x0, y0, bw, bh;
  bool bad;
};

__device__ __forceinline__ CovTri cov_setup(const double* v, int w, int h) {
  CovTri c;
  c.ax = v[0];
  c.ay = v[1];
  c.bx = v[2];
  c.by = v[3];
  c.cx = v[4];
  c.cy = v[5];
  c.area2 = __dsub_rn(__dmul_rn(__dsub_rn(c.bx, c.ax), __dsub_rn(c.cy, c.ay)),
                      __dmul_rn(__dsub_rn(c.by, c.ay), __dsub_rn(c.cx, c.ax)));
  c.bw = c.bh = 0;
  c.x0 = c.y0 = 0;
  // area2 <= 0 raises ValueError in the reference; NaN / inf inputs have no
  // defined result there (math.ceil raises, the C cast is undefined): reject
  c.bad = !(c.area2 > 0.0) || !isfinite(c.area2);
  if (c.bad) return c;
  const double minx = fmin(c.ax, fmin(c.bx, c.cx)), maxx = fmax(c.ax, fmax(c.bx, c.cx));
  const double miny = fmin(c.ay, fmin(c.by, c.cy)), maxy = fmax(c.ay, fmax(c.by, c.cy));
  double x0 = ceil(__dsub_rn(minx, 0.5)), x1 = floor(__dsub_rn(maxx, 0.5));
  double y0 = ceil(__dsub_rn(miny, 0.5)), y1 = floor(__dsub_rn(maxy, 0.5));
  x0 = fmax(x0, 0.0);
  y0 = fmax(y0, 0.0);
  x1 = fmin(x1, (double)(w - 1));
  y1 = fmin(y1, (double)(h - 1));
  if (x1 < x0 || y1 < y0) return c;
  c.x0 = (long long)x0;
  c.y0 = (long long)y0;
  c.bw = (long long)x1 - c.x0 + 1;
  c.bh = (long long)y1 - c.y0 + 1;
  c.d0x = __dsub_rn(c.cx, c.bx);
  c.d0y = __dsub_rn(c.cy, c.by);
  c.d1x = __dsub_rn(c.ax, c.cx);
  c.d1y = __dsub_rn(c.ay, c.cy);
  c.d2x = __dsub_rn(c.bx, c.ax);
  c.d2y = __dsub_rn(c.by, c.ay);
  c.tl0 = c.d0y < 0.0 || (c.d0y == 0.0 && c.d0x > 0.0);
  c.tl1 = c.d1y < 0.0 || (c.d1y == 0.0 && c.d1x > 0.0);
  c.tl2 = c.d2y < 0.0 || (c.d2y == 0.0 && c.d2x > 0.0);
  return c;
}

// edge functions at pixel centre q (row-major index inside the bbox)
__device__ __forceinline__ bool cov_test(const CovTri& c, long long q, int& px, int& py, double& f0, double& f1,
                                         double& f2) {
  const long long ry = q / c.bw;
  px = (int)(c.x0 + (q - ry * c.bw));
  py = (int)(c.y0 + ry);
  const double sx = __dadd_rn((double)px, 0.5), sy = __dadd_rn((double)py, 0.5);
  f0 = __dsub_rn(__dmul_rn(c.d0x, __dsub_rn(sy, c.by)), __dmul_rn(c.d0y, __dsub_rn(sx, c.bx)));
  f1 = __dsub_rn(__dmul_rn(c.d1x, __dsub_rn(sy, c.cy)), __dmul_rn(c.d1y, __dsub_rn(sx, c.cx)));
  f2 = __dsub_rn(__dmul_rn(c.d2x, __dsub_rn(sy, c.ay)), __dmul_rn(c.d2y, __dsub_rn(sx, c.ax)));
  return (f0 > 0.0 || (f0 == 0.0 && c.tl0)) && (f1 > 0.0 || (f1 == 0.0 && c.tl1)) &&
         (f2 > 0.0 || (f2 == 0.0 && c.tl2));
}

// pass 1: covered pixels per triangle (one CTA per triangle, grid-stride)
__global__ void __launch_bounds__(kCovBlock) k_cov_count(long long n, const double* __restrict__ v6,
                                                         const int32_t* __restrict__ wh, uint32_t* __restrict__ cnt,
                                                         int* status, unsigned long long* first_bad) {
  __shared__ unsigned long long warp_sum[kCovBlock / 32];
  for (long long t = blockIdx.x; t < n; t += gridDim.x) {
    const CovTri c = cov_setup(v6 + 6 * t, wh[2 * t], wh[2 * t + 1]);
    if (c.bad) {
      if (threadIdx.x == 0) {
        atomicMin(first_bad, (unsigned long long)t);
        cnt[t] = 0;
      }
      continue;
    }
    const long long P = c.bw * c.bh;
    unsigned long long mine = 0;
    for (long long q = threadIdx.x; q < P; q += kCovBlock) {
      int px, py;
      double f0, f1, f2;
      mine += cov_test(c, q, px, py, f0, f1, f2) ? 1u : 0u;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
    if (lane_id() == 0) warp_sum[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < kCovBlock / 32; ++w) s += warp_sum[w];
      if (s > 0xFFFFFFFFull) {
        raise_status(status, FHV_NOMEM);
        s = 0;
      }
      cnt[t] = (uint32_t)s;
    }
    __syncthreads();
  }
}

// pass 2: write each triangle's covered pixels in row-major order at its
// offset (chunk of kCovBlock pixel centres -> block-wide exclusive scan)
__global__ void __launch_bounds__(kCovBlock) k_cov_write(long long n, const double* __restrict__ v6,
                                                         const int32_t* __restrict__ wh,
                                                         const unsigned long long* __restrict__ off,
                                                         long long max_out, int32_t* __restrict__ opx,
                                                         int32_t* __restrict__ opy, double* __restrict__ l0,
                                                         double* __restrict__ l1, double* __restrict__ l2) {
  __shared__ unsigned warp_cnt[kCovBlock / 32];
  for (long long t = blockIdx.x; t < n; t += gridDim.x) {
    const CovTri c = cov_setup(v6 + 6 * t, wh[2 * t], wh[2 * t + 1]);
    if (c.bad) continue;
    const long long P = c.bw * c.bh;
    unsigned long long base = off[t];
    for (long long q0 = 0; q0 < P; q0 += kCovBlock) {
      const long long q = q0 + threadIdx.x;
      int px = 0, py = 0;
      double f0 = 0.0, f1 = 0.0, f2 = 0.0;
      const bool in = q < P && cov_test(c, q, px, py, f0, f1, f2);
      const unsigned m = __ballot_sync(0xffffffffu, in);
      const int w = threadIdx.x >> 5;
      if (lane_id() == 0) warp_cnt[w] = (unsigned)__popc(m);
      __syncthreads();
      unsigned before = 0, total = 0;
#pragma unroll
      for (int k = 0; k < kCovBlock / 32; ++k) {
        const unsigned x = warp_cnt[k];
        before += k < w ? x : 0u;
        total += x;
      }
      __syncthreads();
      if (in) {
        const long long r = (long long)(base + before + (unsigned)__popc(m & ((1u << lane_id()) - 1u)));
        if (r < max_out) {
          opx[r] = px;
          opy[r] = py;
          l0[r] = ddiv_zd(f0, c.area2);
          l1[r] = ddiv_zd(f1, c.area2);
          l2[r] = ddiv_zd(f2, c.area2);
        }
      }
      base += total;
    }
  }
}

// key / code range check for the insert ops (the reference does no bounds
// checking; a bad key here is reported instead of corrupting memory)
__global__ void k_check_keys(long long n, const long long* __restrict__ keys, long long n_keys, int* status) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long k = keys[i];
    if (k < 0 || k >= n_keys) raise_status(status, FHV_BAD_ARGS);
  }
}

// linked_insert: one warp walks the batch 32 keys at a time; inside a chunk,
// same-key lanes chain to each other in lane (= batch) order and the group's
// last lane swaps the head, so the result equals the sequential loop
__global__ void k_linked_insert(long long n, const long long* __restrict__ keys, int32_t* __restrict__ heads,
                                int32_t* __restrict__ prev, long long start, const int* status) {
  if (*status) return;
  const unsigned lane = lane_id(), below = (1u << lane) - 1u;
  for (long long b = 0; b < n; b += 32) {
    const long long i = b + lane;
    const bool valid = i < n;
    const long long k = valid ? keys[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, k);
    const unsigned lower = grp & below;
    const long long idx = start + i;
    if (valid) prev[idx] = lower ? (int32_t)(start + b + (31 - __clz(lower))) : heads[k];
    __syncwarp();
    if (valid && (int)lane == 31 - __clz(grp)) heads[k] = (int32_t)idx;
    __syncwarp();
  }
}

// pofa_scatter: one warp, 32 codes at a time; same-code lanes take
// consecutive cursor values in lane order; the first lane whose cursor
// reaches its leaf count stops the batch (lanes after it commit nothing)
__global__ void k_pofa_scatter_op(long long n, const long long* __restrict__ codes,
                                  const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts,
                                  uint32_t* __restrict__ cursors, long long* __restrict__ dest, const int* status,
                                  long long* bad) {
  if (*status) return;
  const unsigned lane = lane_id(), below = (1u << lane) - 1u;
  for (long long b = 0; b < n; b += 32) {
    const long long i = b + lane;
    const bool valid = i < n;
    const long long c = valid ? codes[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const int leader = __ffs(grp) - 1;
    unsigned long long cur0 = 0;
    if (valid && (int)lane == leader) cur0 = cursors[c];
    cur0 = __shfl_sync(0xffffffffu, cur0, leader);
    const unsigned long long cur = cur0 + (unsigned)__popc(grp & below);
    const bool is_bad = valid && cur >= (unsigned long long)counts[c];
    const unsigned bm = __ballot_sync(0xffffffffu, is_bad);
    const unsigned keep = bm ? ((1u << (__ffs(bm) - 1)) - 1u) : 0xffffffffu;  // lanes before the first bad one
    if (valid && ((keep >> lane) & 1u)) dest[i] = (long long)offsets[c] + (long long)cur;
    if (valid && (int)lane == leader) {
      const unsigned used = (unsigned)__popc(grp & keep);
      if (used) cursors[c] = (uint32_t)(cur0 + used);
    }
    if (bm) {
      if (lane == 0) *bad = b + (__ffs(bm) - 1);
      return;
    }
    __syncwarp();
  }
}

// OccupancyPyramid.set_paths (fhv/storage.py:294-301): OR the root-path
// bits of each code into levels 0..L-1.  Bytes are OR-ed through their
// aligned 32-bit word (atomicOr with zero elsewhere leaves neighbours as
// they are).
__global__ void k_set_paths(long long n, const long long* __restrict__ codes, int L, uint8_t* __restrict__ pyr,
                            const int* status) {
  if (*status) return;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long code = (unsigned long long)codes[i];
    for (int k = 0; k < L; ++k) {
      const unsigned long long node = code >> (3 * (L - k));
      const unsigned child = (unsigned)((code >> (3 * (L - k - 1))) & 7ull);
      const unsigned long long byte = (unsigned long long)pyr_level_offset(k) + node;
      unsigned* word = reinterpret_cast<unsigned*>(reinterpret_cast<uintptr_t>(pyr + byte) & ~(uintptr_t)3);
      const unsigned shift = 8u * (unsigned)(reinterpret_cast<uintptr_t>(pyr + byte) & 3u);
      atomicOr(word, (1u << child) << shift);
    }
  }
}

// OccupancyPyramid.from_leaf_occupancy (fhv/storage.py:316-328): level L-1
// masks from the leaf occupancy bytes; the upper levels follow
__global__ void k_occ_to_masks(long long n_nodes, const uint8_t* __restrict__ occ, uint8_t* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_nodes;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned m = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) m |= (occ[8 * i + c] != 0 ? 1u : 0u) << c;
    dst[i] = (uint8_t)m;
  }
}

// chain_indices (fhv/storage.py:480-488): pool indices reachable from
// heads[key], most recent first (one thread walks the list; a cycle or an
// index past prev_len stops the walk with FHV_BAD_ARGS)
__global__ void k_chain_walk(const int32_t* __restrict__ heads, const int32_t* __restrict__ prev, long long prev_len,
                             long long key, long long cap, long long* __restrict__ out, long long* n_out,
                             int* status) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  long long n = 0;
  for (long long i = heads[key]; i >= 0; i = prev[i]) {
    if (i >= prev_len || n > prev_len) {
      raise_status(status, FHV_BAD_ARGS);
      break;
    }
    if (n < cap) out[n] = i;
    ++n;
  }
  *n_out = n;
}

inline int grid_for(long long n, int block, int per_sm = 8) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148LL * per_sm) g = 148LL * per_sm;
  return (int)g;
}

}  // namespace

}  // namespace fhv

using namespace fhv;

extern "C" int fhv_op_coverage(fhv_ctx* ctx, int64_t n, const double* v6, const int32_t* wh, int64_t max_out,
                               int64_t* tri_off, int32_t* px, int32_t* py, double* l0, double* l1, double* l2,
                               int64_t* n_out, int64_t* first_bad, void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!v6 || !wh || !tri_off)) || max_out < 0) return FHV_BAD_ARGS;
  if (max_out > 0 && (!px || !py || !l0 || !l1 || !l2)) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  unsigned long long* fb = &ctx->ctl->spare[2];
  if ((rc = check_cuda(ctx, cudaMemsetAsync(fb, 0xff, 8, s)))) return rc;
  if (n > 0) {
    auto* cnt = (uint32_t*)scratch(ctx, kTmp0, (size_t)n * 4);
    if (!cnt) return FHV_NOMEM;
    const int g = (int)(n < 148LL * 16 ? n : 148LL * 16);
    {
      LaunchScope L_(ctx, kStOps, s);
      k_cov_count<<<g, kCovBlock, 0, s>>>(n, v6, wh, cnt, &ctx->ctl->status, fb);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
    auto* off = (unsigned long long*)tri_off;
    if ((rc = scan_u32_to_u64(ctx, cnt, off, n, s))) return rc;
    if ((rc = check_cuda(ctx, cudaMemcpyAsync(off + n, &ctx->ctl->scan_total, 8, cudaMemcpyDeviceToDevice, s))))
      return rc;
    if (max_out > 0) {
      LaunchScope L_(ctx, kStOps, s);
      k_cov_write<<<g, kCovBlock, 0, s>>>(n, v6, wh, off, max_out, px, py, l0, l1, l2);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  } else if ((rc = check_cuda(ctx, cudaMemsetAsync(tri_off, 0, 8, s)))) {
    return rc;
  }
  rc = sync_control(ctx, s);
  if (n_out) *n_out = n > 0 ? (int64_t)ctx->ctl_host->scan_total : 0;
  const unsigned long long b = ctx->ctl_host->spare[2];
  if (first_bad) *first_bad = b == ~0ull ? -1 : (int64_t)b;
  return rc;
}

extern "C" int fhv_op_linked_insert(fhv_ctx* ctx, int64_t n, const int64_t* keys, int64_t n_keys, int32_t* heads,
                                    int32_t* prev, int64_t prev_len, int64_t start, void* stream) {
  if (!ctx || n < 0 || start < 0 || n_keys < 0) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  if (!keys || !heads || !prev || start + n > prev_len) return FHV_BAD_ARGS;
  if (start + n - 1 > 0x7FFFFFFFLL) return FHV_BAD_ARGS;  // pool indices are int32 (fhv/_ckern.pyx:122)
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStOps, s);
    k_check_keys<<<grid_for(n, 256), 256, 0, s>>>(n, (const long long*)keys, n_keys, &ctx->ctl->status);
  }
  {
    LaunchScope L_(ctx, kStOps, s);
    k_linked_insert<<<1, 32, 0, s>>>(n, (const long long*)keys, heads, prev, start, &ctx->ctl->status);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  return sync_control(ctx, s);
}

extern "C" int fhv_op_pofa_scatter(fhv_ctx* ctx, int64_t n, const int64_t* codes, int64_t n_leaves,
                                   const uint32_t* offsets, const uint32_t* counts, uint32_t* cursors, int64_t* dest,
                                   int64_t* bad, void* stream) {
  if (!ctx || n < 0 || n_leaves < 0 || !bad) return FHV_BAD_ARGS;
  *bad = -1;
  if (n == 0) return FHV_OK;
  if (!codes || !offsets || !counts || !cursors || !dest) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  long long* bd = (long long*)&ctx->ctl->spare[2];
  if ((rc = check_cuda(ctx, cudaMemsetAsync(bd, 0xff, 8, s)))) return rc;
  {
    LaunchScope L_(ctx, kStOps, s);
    k_check_keys<<<grid_for(n, 256), 256, 0, s>>>(n, (const long long*)codes, n_leaves, &ctx->ctl->status);
  }
  {
    LaunchScope L_(ctx, kStOps, s);
    k_pofa_scatter_op<<<1, 32, 0, s>>>(n, (const long long*)codes, offsets, counts, cursors, (long long*)dest,
                                       &ctx->ctl->status, bd);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  rc = sync_control(ctx, s);
  *bad = (int64_t)ctx->ctl_host->spare[2];
  return rc;
}

extern "C" int fhv_set_paths(fhv_ctx* ctx, int32_t levels, int64_t n, const int64_t* codes, uint8_t* pyramid,
                             void* stream) {
  if (!ctx || levels < 1 || levels > kMaxLevels || n < 0 || !pyramid) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  if (!codes) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStOps, s);
    k_check_keys<<<grid_for(n, 256), 256, 0, s>>>(n, (const long long*)codes, 1LL << (3 * levels),
                                                  &ctx->ctl->status);
    k_set_paths<<<grid_for(n, 256), 256, 0, s>>>(n, (const long long*)codes, levels, pyramid, &ctx->ctl->status);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  return sync_control(ctx, s);
}

extern "C" int fhv_pyramid_from_occupancy(fhv_ctx* ctx, int32_t levels, const uint8_t* occupied, uint8_t* pyramid,
                                          void* stream) {
  if (!ctx || levels < 1 || levels > kMaxLevels || !occupied || !pyramid) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const long long nodes = 1LL << (3 * (levels - 1));
  {
    LaunchScope L_(ctx, kStOps, s);
    k_occ_to_masks<<<grid_for(nodes, 256), 256, 0, s>>>(nodes, occupied, pyramid + pyr_level_offset(levels - 1));
  }
  int rc = check_cuda(ctx, cudaGetLastError());
  if (rc) return rc;
  return pyramid_upper_levels(ctx, pyramid, levels, s);
}

extern "C" int fhv_chain_indices(fhv_ctx* ctx, const int32_t* heads, int64_t n_keys, const int32_t* prev,
                                 int64_t prev_len, int64_t key, int64_t cap, int64_t* out, int64_t* n_out,
                                 void* stream) {
  if (!ctx || !heads || key < 0 || key >= n_keys || cap < 0 || !n_out || (cap > 0 && !out)) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  long long* nd = (long long*)&ctx->ctl->spare[2];
  {
    LaunchScope L_(ctx, kStOps, s);
    k_chain_walk<<<1, 32, 0, s>>>(heads, prev, prev_len, key, cap, (long long*)out, nd, &ctx->ctl->status);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  rc = sync_control(ctx, s);
  *n_out = (int64_t)ctx->ctl_host->spare[2];
  return rc;
}
