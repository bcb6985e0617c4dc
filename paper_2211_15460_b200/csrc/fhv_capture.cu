// fhv_capture.cu -- the capture half of the hot path: a software rasteriser
// that emits EVERY covered pixel-centre sample of every triangle (no culling,
// no depth test) and inserts the fragments into PPFL / POFL / POFA stores.
//
// Reference: capture_pass + _raster_screen / _raster_tangent + coverage +
// the four sinks (fhv/raster.py:184-388, fhv/_ckern.pyx:25-143,
// fhv/storage.py:356-439, 553-621).
//
// Pipeline (all on one stream; two host syncs for data-dependent sizes):
//   k_job_setup    one thread per (triangle, pass) job: projection or tangent
//                  basis + window, winding order, clipped bbox, #work items
//   scan           job items -> item offsets                      (sync #1)
//   k_item_expand  work item = (job, 128-pixel slice of the job's bbox)
//   k_raster<kCnt*> warp per 32 items, lane per bbox pixel: exact coverage
//                  counts (+ per-leaf histogram, match_any-aggregated, for
//                  POFA pass 1)
//   scan           item counts -> item fragment offsets = the reference's
//                  pool index of each item's first fragment (its "rank")
//   k_raster<MODE>  same traversal: coverage, barycentrics, interpolation,
//                  f32 record, then the store-specific insert
//   fix-ups        EXACT_ORDER chain / in-leaf sorts, POFL pyramid (sync #2)
//
// Exactness: coverage ties are decided on bit-identical f64 edge functions
// (-fmad=false + explicit __fma_rn where NumPy/OpenBLAS fuse), so the covered
// set, counts and octant ranges are bit-exact; interpolated attributes follow
// the same operation order and match bit for bit as well.
#include <cstdlib>

#include "fhv_common.cuh"
#include "fhv_internal.h"

namespace fhv {

struct __align__(16) JobSetup {
  double ax, ay, bx, by, cx, cy;  // ordered raster vertices (coverage inputs)
  int32_t x0, y0, bw, bh;         // clipped bbox origin and size (bw == 0: empty)
  uint32_t tri;
  uint32_t swapped;               // winding order (0,2,1)
  uint32_t pad[2];
};
static_assert(sizeof(JobSetup) == 80, "JobSetup layout");

constexpr uint32_t kItemPix = 128;

// internal EmitOut flag (above the public FHV_* bits): park EXACT_ORDER ranks
// with a segment-start bit (pools < 2^31 records), for the tile fix-up
constexpr int kSegFlags = 1 << 16;
// internal EmitOut flag: emission through the all-exact per-fragment path
// (k_emit) instead of the certified fast path (k_emit_fast) -- A/B testing
constexpr int kExactMath = 1 << 17;

// per-job screen data of the deferred pass (strategy kScreen): clip w and
// ndc z of the vertices in winding order, and whether the job's batch holds
// exactly one fragment (numpy's gemv takes the ddot path then)
struct JobPersp {
  double w[3], z[3];
  uint32_t n1, pad;
};

constexpr int kScreen = 4;  // deferred_baseline: one camera, W x H, any projection

struct CaptureParams {
  int strategy, res;
  int width, height;   // raster size (res x res for the capture strategies)
  int ortho;           // projection row 3 == (0, 0, 0, 1) (RasterConfig.is_orthographic)
  JobPersp* persp;     // kScreen only
  double pitch;
  double proj[3][16];
  long long n_tri, n_jobs;
  const double* pos;
  const double* vnrm;
  const double* fnrm;
  const uint32_t* mat;
  const uint32_t* obj;
  const uint32_t* tri_index;              // job -> triangle indirection (binned shard), or null
  unsigned long long cell_lo, cell_hi;    // owned leaf range (POFA shard); [0, 8^L) by default
};

struct EmitOut {
  // pool
  long long capacity;
  float* pos;
  float* nrm;
  uint32_t* mat;
  uint32_t* obj;
  int32_t* prev;
  // PPFL / POFL directories
  int32_t* heads;
  long long width, n_keys;
  int levels;
  // POFA (indexed by code - cell_lo)
  uint32_t* leaf_counts;
  uint32_t* tile_sums;  // counting pass: per directory tile (kDirSumShift) totals, or null
  const uint32_t* offsets;
  const uint32_t* counts;
  uint32_t* cursors;
  unsigned long long base;  // global pool index of this shard's first record
  // list
  long long max_out;
  long long* job;
  int32_t* px;
  int32_t* py;
  double* wpos;
  double* wnrm;
  double* depth;  // list mode: FragmentBatch.depth (screen: lam @ ndc_z; tangent: 0.5), or null
  int flags;
  // deferred_baseline (kScreen): per-pixel depth keys, winning job, G-buffer
  unsigned long long* ds_key;
  uint32_t* ds_win;
  fhv_gbuffer_t gb;
};

// ---------------------------------------------------------------------------
// job setup

__device__ __forceinline__ void job_of(const CaptureParams& p, long long j, long long* t, int* axis) {
  if (p.strategy == 1) {  // three_separate: axis-major
    *axis = (int)(j / p.n_tri);
    *t = j % p.n_tri;
  } else if (p.strategy == 2) {  // three_way_geometry: triangle-major
    *t = j / 3;
    *axis = (int)(j % 3);
  } else {
    *t = j;
    *axis = 0;
  }
  if (p.tri_index) *t = p.tri_index[*t];
}

// order + coverage bbox, shared by both projections (coverage prologue,
// fhv/_ckern.pyx:28-58).  Returns false for a skipped job.
__device__ __forceinline__ bool finish_setup(const double xr[3], const double yr[3], long long w, long long h,
                                             JobSetup& js) {
  const double area2 = __dsub_rn(__dmul_rn(__dsub_rn(xr[1], xr[0]), __dsub_rn(yr[2], yr[0])),
                                 __dmul_rn(__dsub_rn(yr[1], yr[0]), __dsub_rn(xr[2], xr[0])));
  js.bw = 0;
  js.bh = 0;
  if (area2 == 0.0 || !isfinite(area2)) return false;
  const int i1 = area2 > 0.0 ? 1 : 2, i2 = area2 > 0.0 ? 2 : 1;
  js.swapped = area2 > 0.0 ? 0u : 1u;
  js.ax = xr[0]; js.ay = yr[0];
  js.bx = xr[i1]; js.by = yr[i1];
  js.cx = xr[i2]; js.cy = yr[i2];
  double minx = js.ax, maxx = js.ax, miny = js.ay, maxy = js.ay;
  if (js.bx < minx) minx = js.bx;
  if (js.cx < minx) minx = js.cx;
  if (js.bx > maxx) maxx = js.bx;
  if (js.cx > maxx) maxx = js.cx;
  if (js.by < miny) miny = js.by;
  if (js.cy < miny) miny = js.cy;
  if (js.by > maxy) maxy = js.by;
  if (js.cy > maxy) maxy = js.cy;
  double x0 = ceil(__dsub_rn(minx, 0.5)), x1 = floor(__dsub_rn(maxx, 0.5));
  double y0 = ceil(__dsub_rn(miny, 0.5)), y1 = floor(__dsub_rn(maxy, 0.5));
  if (x0 < 0.0) x0 = 0.0;
  if (y0 < 0.0) y0 = 0.0;
  if (x1 > (double)(w - 1)) x1 = (double)(w - 1);
  if (y1 > (double)(h - 1)) y1 = (double)(h - 1);
  if (x1 < x0 || y1 < y0) return true;  // valid job, no covered pixel
  js.x0 = (int32_t)x0;
  js.y0 = (int32_t)y0;
  js.bw = (int32_t)(x1 - x0) + 1;
  js.bh = (int32_t)(y1 - y0) + 1;
  return true;
}

// _raster_screen (fhv/raster.py:184-209): clip = dgemm (FWD) + P[:,3]; the
// capture axes are orthographic; the deferred camera (kScreen) may be
// perspective: a triangle with any clip w <= 1e-9 is skipped
__device__ __forceinline__ void setup_screen(const CaptureParams& p, long long j, long long t, int axis,
                                             JobSetup& js) {
  const double* M = p.proj[axis];
  const double* P = p.pos + 9 * t;
  double xr[3], yr[3], cw[3], nz[3];
  bool behind = false;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double X = P[3 * i], Y = P[3 * i + 1], Z = P[3 * i + 2];
    const double c0 = __dadd_rn(fwd3(X, Y, Z, M[0], M[1], M[2]), M[3]);
    const double c1 = __dadd_rn(fwd3(X, Y, Z, M[4], M[5], M[6]), M[7]);
    const double c3 = __dadd_rn(fwd3(X, Y, Z, M[12], M[13], M[14]), M[15]);
    const Recip r3 = recip_of(c3);
    if (p.persp) {  // the deferred pass, or a list capture that reports depth
      const double c2 = __dadd_rn(fwd3(X, Y, Z, M[8], M[9], M[10]), M[11]);
      nz[i] = div_rn(c2, r3);
      cw[i] = c3;
      behind = behind || (!p.ortho && c3 <= 1e-9);
    }
    const double nx = div_rn(c0, r3), ny = div_rn(c1, r3);
    xr[i] = __dmul_rn(__dmul_rn(__dadd_rn(nx, 1.0), 0.5), (double)p.width);
    yr[i] = __dmul_rn(__dmul_rn(__dsub_rn(1.0, ny), 0.5), (double)p.height);
  }
  if (behind) {  // "behind the eye; this rasterizer does not clip"
    js.bw = 0;
    js.bh = 0;
    return;
  }
  finish_setup(xr, yr, p.width, p.height, js);
  if (p.persp) {
    JobPersp jp;
    const int o1 = js.swapped ? 2 : 1, o2 = js.swapped ? 1 : 2;
    jp.w[0] = cw[0]; jp.w[1] = cw[o1]; jp.w[2] = cw[o2];
    jp.z[0] = nz[0]; jp.z[1] = nz[o1]; jp.z[2] = nz[o2];
    jp.n1 = 0;
    jp.pad = 0;
    p.persp[j] = jp;
  }
}

// _raster_tangent (fhv/raster.py:212-242) with tangent_basis (:147-163)
__device__ __forceinline__ void setup_tangent(const CaptureParams& p, long long t, JobSetup& js, int* status) {
  const double* P = p.pos + 9 * t;
  const double* F = p.fnrm + 3 * t;
  js.bw = 0;
  js.bh = 0;
  if (!(F[0] != 0.0 || F[1] != 0.0 || F[2] != 0.0)) return;  // degenerate face
  const double norm = __dsqrt_rn(fwd3(F[0], F[1], F[2], F[0], F[1], F[2]));
  if (norm < 1e-12 || fabs(__dsub_rn(norm, 1.0)) > 1e-3) {
    raise_status(status, FHV_BASIS);
    return;
  }
  const Recip rn = recip_of(norm);
  const double n0 = div_rn(F[0], rn), n1 = div_rn(F[1], rn), n2 = div_rn(F[2], rn);
  const bool hx = fabs(n0) <= 0.6;
  const double h0 = hx ? 1.0 : 0.0, h1 = hx ? 0.0 : 1.0, h2 = 0.0;
  const double hn = fwd3(h0, h1, h2, n0, n1, n2);
  double t0 = __dsub_rn(h0, __dmul_rn(hn, n0));
  double t1 = __dsub_rn(h1, __dmul_rn(hn, n1));
  double t2 = __dsub_rn(h2, __dmul_rn(hn, n2));
  const double tn = __dsqrt_rn(fwd3(t0, t1, t2, t0, t1, t2));
  const Recip rt = recip_of(tn);
  t0 = div_rn(t0, rt);
  t1 = div_rn(t1, rt);
  t2 = div_rn(t2, rt);
  const double b0 = __dsub_rn(__dmul_rn(n1, t2), __dmul_rn(n2, t1));
  const double b1 = __dsub_rn(__dmul_rn(n2, t0), __dmul_rn(n0, t2));
  const double b2 = __dsub_rn(__dmul_rn(n0, t1), __dmul_rn(n1, t0));
  double tc[3], bc[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    tc[i] = fwd3(P[3 * i], P[3 * i + 1], P[3 * i + 2], t0, t1, t2);
    bc[i] = fwd3(P[3 * i], P[3 * i + 1], P[3 * i + 2], b0, b1, b2);
  }
  double tmin = tc[0], tmax = tc[0], bmin = bc[0], bmax = bc[0];
#pragma unroll
  for (int i = 1; i < 3; ++i) {
    tmin = tc[i] < tmin ? tc[i] : tmin;
    tmax = tc[i] > tmax ? tc[i] : tmax;
    bmin = bc[i] < bmin ? bc[i] : bmin;
    bmax = bc[i] > bmax ? bc[i] : bmax;
  }
  const Recip rp = recip_of(p.pitch);
  double nxd = ceil(div_rn(__dsub_rn(tmax, tmin), rp));
  double nyd = ceil(div_rn(__dsub_rn(bmax, bmin), rp));
  if (!(nxd >= 1.0)) nxd = 1.0;
  if (!(nyd >= 1.0)) nyd = 1.0;
  if (nxd > 2147483647.0 || nyd > 2147483647.0) {
    raise_status(status, FHV_BAD_ARGS);
    return;
  }
  double xr[3], yr[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    xr[i] = div_rn(__dsub_rn(tc[i], tmin), rp);
    yr[i] = div_rn(__dsub_rn(bmax, bc[i]), rp);
  }
  finish_setup(xr, yr, (long long)nxd, (long long)nyd, js);
}

#ifndef FHV_SETUP_MINB
#define FHV_SETUP_MINB 8  // 64 registers: job setup 47 -> 44 us (6: 47, 10: 46)
#endif
__global__ void __launch_bounds__(128, FHV_SETUP_MINB) k_job_setup(CaptureParams p, JobSetup* __restrict__ jobs,
                                                                   uint32_t* __restrict__ job_items, int* status,
                                                                   uint32_t* __restrict__ tile_sums) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < p.n_jobs;
       j += (long long)gridDim.x * blockDim.x) {
    long long t;
    int axis;
    job_of(p, j, &t, &axis);
    JobSetup js;
    js.x0 = js.y0 = 0;
    js.ax = js.ay = js.bx = js.by = js.cx = js.cy = 0.0;
    js.swapped = 0;
    js.pad[0] = js.pad[1] = 0;
    js.tri = (uint32_t)t;
    if (p.strategy == 3)
      setup_tangent(p, t, js, status);
    else
      setup_screen(p, j, t, axis, js);
    const unsigned long long pix = (unsigned long long)js.bw * (unsigned long long)js.bh;
    unsigned long long items = (pix + kItemPix - 1) / kItemPix;
    if (items > 0xFFFFFFFFull) {
      raise_status(status, FHV_NOMEM);
      items = 0;
    }
    jobs[j] = js;
    job_items[j] = (uint32_t)items;
    if (tile_sums) {  // the item totals of kExpandTileJobs-job tiles (a warp's 32 jobs share one)
      const unsigned act = __activemask();
      const unsigned v = __reduce_add_sync(act, (unsigned)items);
      if ((int)lane_id() == __ffs(act) - 1) atomicAdd(&tile_sums[j / kExpandTileJobs], v);
    }
  }
}

// work items of each job: a lane per job writes small jobs' items itself;
// jobs with many items (large triangles) are written by the whole warp, one
// such job at a time (ballot loop), so both 1-item and 10^4-item jobs stay
// coalesced
constexpr uint32_t kExpandSmall = 4;

__global__ void __launch_bounds__(256) k_item_expand(long long n_jobs, const uint32_t* __restrict__ job_items,
                                                     const unsigned long long* __restrict__ job_item_off,
                                                     uint32_t* __restrict__ item_job, uint32_t* __restrict__ item_p0,
                                                     unsigned long long cap, int* status) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); j0 < n_jobs; j0 += stride) {
    const long long j = j0 + lane_id();
    uint32_t n = j < n_jobs ? job_items[j] : 0u;
    const unsigned long long base = j < n_jobs ? job_item_off[j] : 0ull;
    if (base + n > cap) {  // speculative item buffers too small: the host re-plans with a sync
      raise_status(status, FHV_RETRY_ITEMS);
      n = base < cap ? (uint32_t)(cap - base) : 0u;
    }
    if (n <= kExpandSmall) {
      for (uint32_t k = 0; k < n; ++k) {
        item_job[base + k] = (uint32_t)j;
        item_p0[base + k] = k * kItemPix;
      }
    }
    unsigned big = __ballot_sync(0xffffffffu, n > kExpandSmall);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t bn = __shfl_sync(0xffffffffu, n, src);
      const unsigned long long bb = __shfl_sync(0xffffffffu, base, src);
      const uint32_t bj = (uint32_t)(j0 + src);
      for (uint32_t k = lane_id(); k < bn; k += 32) {
        item_job[bb + k] = bj;
        item_p0[bb + k] = k * kItemPix;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// warp-cooperative rasterisation (coverage, fhv/_ckern.pyx:72-101, fused
// with interpolation and the store-specific insert)
//
// A warp takes 32 consecutive work items (lane k <-> item i0+k, each a slice
// of <= kItemPix bbox pixels of one job, in job order).  Coverage is swept
// lane-per-item, row-incrementally like the reference loop (a few f64 ops per
// pixel); covered pixels are appended (ballot + popc) to a per-warp queue in
// shared memory, in emission order per item, and every 32 queued fragments
// are processed 32 wide: barycentric divides, interpolation, keying,
// match_any-aggregated atomics and stores run with full lanes no matter how
// ragged the triangles are.

struct CoverS {  // per-item coverage state, staged in shared memory
  double ax, ay, bx, by, cx, cy;
  double e0x, e0y, e1x, e1y, e2x, e2y;
  double area2;
  int32_t x0, y0, bw;
  uint32_t tri, swapped, tl;  // tl bit e: edge e is a top-left edge
  uint32_t p0;
  float inv_bw;  // 1.0f / bw: pixel index -> bbox row without an integer division
};

// the emission pass's staged item: + recip_of(area2).y, replayed by every
// fragment's barycentric divisions (div_rn, bit-identical: -2 % emit time).
// The counting pass keeps CoverS as is (its sweep reads the struct per pixel:
// a longer stride costs more than the reciprocal saves) and stages the
// reciprocal in a separate shared array (-1.5 % count time)
struct CoverR : CoverS {
  double rcp_area2;
};

// l_i = f_i / area2, correctly rounded (__ddiv_rn's result)
__device__ __forceinline__ double bary(const CoverS& c, double f) { return ddiv_zd_sel(f, c.area2); }
__device__ __forceinline__ double bary(const CoverR& c, double f) {
  return div_rn(f, Recip{c.area2, c.rcp_area2});
}

__device__ __forceinline__ void make_cover(const JobSetup& js, uint32_t p0, CoverS& c) {
  c.ax = js.ax; c.ay = js.ay; c.bx = js.bx; c.by = js.by; c.cx = js.cx; c.cy = js.cy;
  c.area2 = __dsub_rn(__dmul_rn(__dsub_rn(c.bx, c.ax), __dsub_rn(c.cy, c.ay)),
                      __dmul_rn(__dsub_rn(c.by, c.ay), __dsub_rn(c.cx, c.ax)));
  c.e0x = __dsub_rn(c.cx, c.bx); c.e0y = __dsub_rn(c.cy, c.by);  // v1 -> v2, opposite v0
  c.e1x = __dsub_rn(c.ax, c.cx); c.e1y = __dsub_rn(c.ay, c.cy);  // v2 -> v0, opposite v1
  c.e2x = __dsub_rn(c.bx, c.ax); c.e2y = __dsub_rn(c.by, c.ay);  // v0 -> v1, opposite v2
  const bool tl0 = c.e0y < 0.0 || (c.e0y == 0.0 && c.e0x > 0.0);
  const bool tl1 = c.e1y < 0.0 || (c.e1y == 0.0 && c.e1x > 0.0);
  const bool tl2 = c.e2y < 0.0 || (c.e2y == 0.0 && c.e2x > 0.0);
  c.tl = (tl0 ? 1u : 0u) | (tl1 ? 2u : 0u) | (tl2 ? 4u : 0u);
  c.x0 = js.x0; c.y0 = js.y0; c.bw = js.bw;
  c.tri = js.tri;
  c.swapped = js.swapped;
  c.p0 = p0;
  c.inv_bw = 1.0f / (float)(js.bw > 0 ? js.bw : 1);
}
__device__ __forceinline__ void make_cover(const JobSetup& js, uint32_t p0, CoverR& c) {
  make_cover(js, p0, static_cast<CoverS&>(c));
  c.rcp_area2 = recip_of(c.area2 > 0.0 ? c.area2 : 1.0).y;
}

// pixel-centre coverage test with the top-left rule; edge functions in f64
// exactly as the reference evaluates them (no contraction)
__device__ __forceinline__ bool cover_test(const CoverS& c, int px, int py, double& f0, double& f1, double& f2) {
  const double sy = __dadd_rn((double)py, 0.5), sx = __dadd_rn((double)px, 0.5);
  f0 = __dsub_rn(__dmul_rn(c.e0x, __dsub_rn(sy, c.by)), __dmul_rn(c.e0y, __dsub_rn(sx, c.bx)));
  f1 = __dsub_rn(__dmul_rn(c.e1x, __dsub_rn(sy, c.cy)), __dmul_rn(c.e1y, __dsub_rn(sx, c.cx)));
  f2 = __dsub_rn(__dmul_rn(c.e2x, __dsub_rn(sy, c.ay)), __dmul_rn(c.e2y, __dsub_rn(sx, c.ax)));
  const bool in0 = f0 > 0.0 || (f0 == 0.0 && (c.tl & 1u));
  const bool in1 = f1 > 0.0 || (f1 == 0.0 && (c.tl & 2u));
  return in0 & in1 & (f2 > 0.0 || (f2 == 0.0 && (c.tl & 4u)));
}

// triangle vertex data in winding order
struct TriData {
  double v[3][3];
  double n[3][3];
  double f[3];
  uint32_t mat, obj;
};

__device__ __forceinline__ void prefetch_l1(const void* a) { asm volatile("prefetch.global.L1 [%0];" ::"l"(a)); }

// pull a triangle's records (positions, vertex + face normals, ids) toward L1
// ahead of the fragments that read them
__device__ __forceinline__ void prefetch_tri(const CaptureParams& p, uint32_t tri) {
  const char* P = reinterpret_cast<const char*>(p.pos + 9 * (long long)tri);
  const char* N = reinterpret_cast<const char*>(p.vnrm + 9 * (long long)tri);
  prefetch_l1(P);
  prefetch_l1(P + 64);
  prefetch_l1(N);
  prefetch_l1(N + 64);
  prefetch_l1(p.fnrm + 3 * (long long)tri);
  prefetch_l1(p.mat + tri);
  prefetch_l1(p.obj + tri);
}

__device__ __forceinline__ void load_tri_pos(const CaptureParams& p, uint32_t tri, uint32_t swapped, TriData& d) {
  const double* P = p.pos + 9 * (long long)tri;
  const int o[3] = {0, swapped ? 2 : 1, swapped ? 1 : 2};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) d.v[i][k] = __ldg(&P[3 * o[i] + k]);
}

__device__ __forceinline__ void load_tri_nrm(const CaptureParams& p, uint32_t tri, uint32_t swapped, TriData& d) {
  const double* N = p.vnrm + 9 * (long long)tri;
  const int o[3] = {0, swapped ? 2 : 1, swapped ? 1 : 2};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) d.n[i][k] = __ldg(&N[3 * o[i] + k]);
#pragma unroll
  for (int k = 0; k < 3; ++k) d.f[k] = __ldg(&p.fnrm[3 * (long long)tri + k]);
  d.mat = __ldg(&p.mat[tri]);
  d.obj = __ldg(&p.obj[tri]);
}

__device__ __forceinline__ void load_tri(const CaptureParams& p, uint32_t tri, uint32_t swapped, TriData& d,
                                         bool normals) {
  load_tri_pos(p, tri, swapped, d);
  if (normals) load_tri_nrm(p, tri, swapped, d);
}

// lam @ V (dgemm FWD chain), fhv/raster.py:168
__device__ __forceinline__ void interp_pos(const TriData& d, double l0, double l1, double l2, double out[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    out[k] = __fma_rn(l2, d.v[2][k], __fma_rn(l1, d.v[1][k], add0(__dmul_rn(l0, d.v[0][k]))));
}

// lam @ N, einsum length, renormalise or face normal (fhv/raster.py:169-173)
__device__ __forceinline__ void interp_nrm(const TriData& d, double l0, double l1, double l2, double out[3]) {
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    v[k] = __fma_rn(l2, d.n[2][k], __fma_rn(l1, d.n[1][k], add0(__dmul_rn(l0, d.n[0][k]))));
  const double len = __dsqrt_rn(e021(v[0], v[1], v[2], v[0], v[1], v[2]));
  if (len > 1e-12) {
    const Recip rl = recip_of(len);  // one reciprocal for the three components (bit-identical div_rn)
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = div_rn(v[k], rl);
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = d.f[k];
  }
}

enum RasterMode { kCnt = 0, kCntLeaves = 1, kList = 2, kPpfl = 3, kPofl = 4, kPofa = 5, kDsDepth = 6, kDsIndex = 7,
                  kDsWrite = 8 };
#ifndef FHV_RASTER_MINB
#define FHV_RASTER_MINB 3  // resident CTAs per SM the raster kernels are register-budgeted for
#endif
#ifndef FHV_RASTER_PER_SM
#define FHV_RASTER_PER_SM 16  // raster / emission grid: CTAs per SM (grid-stride over item groups)
#endif
#ifndef FHV_RASTER_BLOCK
#define FHV_RASTER_BLOCK 256
#endif
constexpr int kRasterBlock = FHV_RASTER_BLOCK;
constexpr int kRasterWarps = kRasterBlock / 32;
#ifndef FHV_EMIT_FAST_WARPS
#define FHV_EMIT_FAST_WARPS 8
#endif
constexpr int kEmitFastWarps = FHV_EMIT_FAST_WARPS;

template <int kMode, bool kAtomicAlloc>
struct RasterState {
  unsigned long long emitted = 0;
  bool bad_range = false, bad_pass = false, bad_key = false, short_pool = false;
};

// one batch of <= 32 fragments, one per lane (valid lanes), called by the
// whole warp.  k: the fragment's item (lane index in the group), (px, py): its
// pixel, push_local: its index among its item's covered pixels.  Local index
// inside the item: push order for the linked / list modes; owned-fragment
// order (smem counters) for the keyed POFA modes, whose shard filter is only
// known here.
// one fragment of the deferred geometry pass (fhv/render.py:345-371).
// depth = lam @ ndc_z (gemv: G102, FWD for a one-fragment batch); the pixel's
// winner is the smallest (depth, triangle) -- "equal depth keeps first" --
// found in three sweeps: RED.MIN of the order-preserving depth key, then
// atomicMin of the job among fragments at that key, then the winner alone
// interpolates with the perspective-corrected lam (lam / w renormalised,
// :206-208) and writes the f64 G-buffer.
template <int kMode, class Cov>
__device__ __forceinline__ void ds_fragment(const CaptureParams& p, const EmitOut& o, const Cov& c, uint32_t job,
                                            int px, int py) {
  double f0, f1, f2;
  cover_test(c, px, py, f0, f1, f2);
  double l0 = bary(c, f0), l1 = bary(c, f1), l2 = bary(c, f2);
  const JobPersp& jp = p.persp[job];
  const double d = jp.n1 ? fwd3(l0, l1, l2, jp.z[0], jp.z[1], jp.z[2]) : g102(l0, l1, l2, jp.z[0], jp.z[1], jp.z[2]);
  if (isnan(d)) return;  // np.minimum.at would poison the pixel; no winner either way
  const unsigned long long key = depth_key(d);
  const long long pix = (long long)py * p.width + px;
  if (kMode == kDsDepth) {
    atomicMin(&o.ds_key[pix], key);
    return;
  }
  if (kMode == kDsIndex) {
    if (o.ds_key[pix] == key) atomicMin(&o.ds_win[pix], job);
    return;
  }
  if (o.ds_win[pix] != job) return;
  if (!p.ortho) {
    const double lw0 = ddiv_z(l0, jp.w[0]), lw1 = ddiv_z(l1, jp.w[1]), lw2 = ddiv_z(l2, jp.w[2]);
    const double sum = __dadd_rn(__dadd_rn(lw0, lw1), lw2);
    const Recip rs = recip_of(sum);
    l0 = div_rn(lw0, rs);
    l1 = div_rn(lw1, rs);
    l2 = div_rn(lw2, rs);
  }
  TriData td;
  load_tri(p, c.tri, c.swapped, td, true);
  double w[3], nn[3];
  interp_pos(td, l0, l1, l2, w);
  interp_nrm(td, l0, l1, l2, nn);
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    o.gb.position[3 * pix + e] = w[e];
    o.gb.normal[3 * pix + e] = nn[e];
  }
  o.gb.material_id[pix] = (int32_t)td.mat;
  o.gb.object_id[pix] = (int32_t)td.obj;
}

// list mode with depth (FragmentBatch.depth): _raster_screen's depth =
// lam @ ndc_z over the winding-ordered vertices (gemv: G102, FWD for a
// one-fragment batch), then -- perspective only -- lam / w renormalised
// before interpolation (fhv/raster.py:204-208); _raster_tangent's is 0.5
__device__ __forceinline__ void list_depth(const CaptureParams& p, uint32_t job, double& l0, double& l1, double& l2,
                                           double& dep) {
  if (p.strategy == 3) {
    dep = 0.5;
    return;
  }
  const JobPersp& jp = p.persp[job];
  dep = jp.n1 ? fwd3(l0, l1, l2, jp.z[0], jp.z[1], jp.z[2]) : g102(l0, l1, l2, jp.z[0], jp.z[1], jp.z[2]);
  if (!p.ortho) {
    const double lw0 = ddiv_z(l0, jp.w[0]), lw1 = ddiv_z(l1, jp.w[1]), lw2 = ddiv_z(l2, jp.w[2]);
    const double sum = __dadd_rn(__dadd_rn(lw0, lw1), lw2);
    const Recip rs = recip_of(sum);
    l0 = div_rn(lw0, rs);
    l1 = div_rn(lw1, rs);
    l2 = div_rn(lw2, rs);
  }
}

template <int kMode, bool kAtomicAlloc, class Cov>
__device__ __forceinline__ void raster_batch(const CaptureParams& p, const EmitOut& o, Control* ctl,
                                             const Cov* cs, bool valid, int k, int px, int py,
                                             uint32_t push_local, uint32_t* own_cnt, unsigned long long rank0,
                                             const uint32_t* item_job_g, RasterState<kMode, kAtomicAlloc>& st,
                                             const double* rcp = nullptr) {
  if constexpr (kMode == kDsDepth || kMode == kDsIndex || kMode == kDsWrite) {
    if (valid) ds_fragment<kMode>(p, o, cs[k], item_job_g[k], px, py);
    return;
  }
  constexpr bool kKeyed = kMode == kCntLeaves || kMode == kPofl || kMode == kPofa;
  constexpr bool kOwned = kMode == kCntLeaves || kMode == kPofa;
  const unsigned lane = lane_id();
  const unsigned below = (1u << lane) - 1u;
  const Cov& c = cs[k];
  bool live = false;
  TriData d;
  double w[3] = {0.0, 0.0, 0.0};
  double l0 = 0.0, l1 = 0.0, l2 = 0.0, dep = 0.0;
  uint64_t code = ~0ull;
  if (valid) {
    double f0, f1, f2;
    cover_test(c, px, py, f0, f1, f2);  // the same f64 values the sweep tested
    if (rcp) {  // the counting pass's per-item reciprocals (a separate shared array)
      const Recip ra{c.area2, rcp[k]};
      l0 = div_rn(f0, ra);
      l1 = div_rn(f1, ra);
      l2 = div_rn(f2, ra);
    } else {
      l0 = bary(c, f0);
      l1 = bary(c, f1);
      l2 = bary(c, f2);
    }
    if (kMode == kList && (p.persp || o.depth)) list_depth(p, item_job_g[k], l0, l1, l2, dep);
    load_tri_pos(p, c.tri, c.swapped, d);
    interp_pos(d, l0, l1, l2, w);
    live = true;
    if (kKeyed) {
      if (!cell_code(__double2float_rn(w[0]), __double2float_rn(w[1]), __double2float_rn(w[2]), o.levels, &code)) {
        st.bad_range = true;
        live = false;
        code = ~0ull;
      } else if (code < p.cell_lo || code >= p.cell_hi) {  // another shard's leaf
        live = false;
        code = ~0ull;
      }
    }
  }
  uint32_t local = push_local;
  // owned-fragment numbering only matters for a shard (a sub-range of the
  // leaves): over the whole directory every covered fragment is owned
  const bool whole = p.cell_lo == 0 && p.cell_hi >= (1ull << (3 * o.levels));
  if (kOwned && !whole) {
    const unsigned m = __ballot_sync(0xffffffffu, live);
    const unsigned grp = __match_any_sync(0xffffffffu, valid ? k : -1);
    local = own_cnt[k] + (uint32_t)__popc(grp & m & below);
    __syncwarp();
    if (valid && (int)lane == 31 - __clz(grp)) own_cnt[k] += (uint32_t)__popc(grp & m);
    __syncwarp();
  }
  const unsigned long long rank = __shfl_sync(0xffffffffu, rank0, k) + local;
  if (kMode == kCntLeaves) {
    const unsigned grp = __match_any_sync(0xffffffffu, code);
    if (live && (int)lane == __ffs(grp) - 1) atomicAdd(&o.leaf_counts[code - p.cell_lo], (uint32_t)__popc(grp));
    if (o.tile_sums) {  // directory tile totals: the directory pass then needs no look-back chain
      const uint32_t tkey = live ? (uint32_t)((code - p.cell_lo) >> kDirSumShift) : 0xffffffffu;
      const unsigned gt = __match_any_sync(0xffffffffu, tkey);
      if (live && (int)lane == __ffs(gt) - 1) atomicAdd(&o.tile_sums[tkey], (uint32_t)__popc(gt));
    }
    return;
  }
  // POFA: the leaf's cursor atomic (and its range loads) go out BEFORE the
  // normal interpolation, so their L2/DRAM round trip overlaps the FP64 work
  unsigned pofa_grp = 0;
  int pofa_leader = 0;
  bool leaf_first = false;  // this record takes its leaf's first slot
  uint32_t pofa_base = 0, pofa_cnt = 0, pofa_off = 0;
  if (kMode == kPofa) {
    pofa_grp = __match_any_sync(0xffffffffu, code);
    pofa_leader = __ffs(pofa_grp) - 1;
    const unsigned long long lc = live ? code - p.cell_lo : 0ull;
    if (live) {
      // count = next offset - offset: the two words share a 32-B sector
      // almost always, so the counts array is not read at all (the last leaf
      // of the range has no successor and reads its count)
      pofa_off = __ldg(&o.offsets[lc]);
      pofa_cnt = lc + 1 < p.cell_hi - p.cell_lo ? __ldg(&o.offsets[lc + 1]) - pofa_off : __ldg(&o.counts[lc]);
    }
    if (live && (int)lane == pofa_leader) pofa_base = atomicAdd(&o.cursors[lc], (uint32_t)__popc(pofa_grp));
  }
  double nn[3] = {0.0, 0.0, 0.0};
  if (live) {
    load_tri_nrm(p, c.tri, c.swapped, d);
    interp_nrm(d, l0, l1, l2, nn);
    ++st.emitted;
  }
  if (kMode == kList) {
    if (live && (long long)rank < o.max_out) {
      o.job[rank] = item_job_g[k];
      o.px[rank] = px;
      o.py[rank] = py;
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        o.wpos[3 * rank + e] = w[e];
        o.wnrm[3 * rank + e] = nn[e];
      }
      if (o.depth) o.depth[rank] = dep;
    }
    return;
  }
  long long slot = -1;
  if (kMode == kPofa) {
    const uint32_t base = __shfl_sync(0xffffffffu, pofa_base, pofa_leader);
    if (live) {
      const uint32_t cur = base + (uint32_t)__popc(pofa_grp & below);
      leaf_first = cur == 0;
      if (cur >= pofa_cnt) {
        st.bad_pass = true;
      } else {
        slot = (long long)(pofa_off - o.base) + cur;
        if (slot >= o.capacity) {  // speculative pool smaller than the exact count
          st.short_pool = true;
          slot = -1;
        }
      }
    }
  } else {
    // slot first: records past capacity are dropped before any keying,
    // like _store_split (fhv/storage.py:338-342, 366-369, 388-392)
    if (kAtomicAlloc) {
      const unsigned m = __ballot_sync(0xffffffffu, live);
      unsigned long long base = 0;
      if (m && lane == (unsigned)(__ffs(m) - 1)) base = atomicAdd(&ctl->alloc, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, m ? __ffs(m) - 1 : 0);
      if (live) slot = (long long)(base + __popc(m & below));
    } else if (live) {
      slot = (long long)rank;
    }
    if (slot >= o.capacity) slot = -1;
    uint64_t key = ~0ull;
    if (slot >= 0) {
      if (kMode == kPpfl) {
        key = (uint64_t)py * (uint64_t)o.width + (uint64_t)px;
        if ((long long)key >= o.n_keys) {
          st.bad_key = true;
          slot = -1;
          key = ~0ull;
        }
      } else {
        key = code;
      }
    }
    // linked insert, aggregated per key: within a batch the lane order is the
    // emission order of same-key fragments, so the group is chained in place
    // and spliced in front of the old head with one atomicExch by its last lane
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const int last = 31 - __clz(grp);
    int32_t old = -1;
    if (slot >= 0 && (int)lane == last) old = atomicExch(&o.heads[key], (int32_t)slot);
    old = __shfl_sync(0xffffffffu, old, last);
    const unsigned lower = grp & below;
    const int32_t prev_slot = __shfl_sync(0xffffffffu, (int32_t)slot, lower ? 31 - __clz(lower) : (int)lane);
    if (slot >= 0) o.prev[slot] = lower ? prev_slot : old;
  }
  if (slot >= 0) {
    // pool capacities are < 2^32 records: 32-bit slot, one wide multiply-add per address
    const uint32_t s32 = (uint32_t)slot;
    float* pp = o.pos + 3ull * s32;
    float* np = o.nrm + 3ull * s32;
    pp[0] = __double2float_rn(w[0]);
    pp[1] = __double2float_rn(w[1]);
    pp[2] = __double2float_rn(w[2]);
    np[0] = __double2float_rn(nn[0]);
    np[1] = __double2float_rn(nn[1]);
    np[2] = __double2float_rn(nn[2]);
    o.mat[s32] = d.mat;
    o.obj[s32] = d.obj;
    // POFA: prev_index = -1; under EXACT_ORDER the emission rank is parked
    // here until the fix-up restores the reference's in-leaf order; with
    // kSegFlags its bit 31 marks the leaf's first slot (segment start)
    if (kMode == kPofa)
      o.prev[s32] = (o.flags & FHV_EXACT_ORDER)
                        ? (int32_t)((uint32_t)rank | ((o.flags & kSegFlags) && leaf_first ? 0x80000000u : 0u))
                        : -1;
  }
}

// ---------------------------------------------------------------------------
// Certified fast path for the f32 record fields (POFA / POFL / PPFL records
// and the POFA counting pass's leaf keys).
//
// The reference computes, per fragment, l_i = f_i / area2 (correctly rounded
// f64 edge functions), pos = lam @ V as an fma chain, f32(pos); nrm = lam @ N,
// / sqrt(einsum), f32.  Every one of those values is the f64 rounding of an
// AFFINE function of the pixel, so per item (one lane each) we build planes
// value(X, Y) = A + B X + C Y over the job's bbox (X = px - x0, Y = py - y0)
// and a bound E on |plane - reference| that holds for every pixel of the item
// (rounding of the reference's own chain + of the plane coefficients + of the
// evaluation; derivation in DESIGN.md section 4).  A fragment evaluates the
// planes with 2 fmas per component and rounds [v - E, v + E] to f32: when
// both ends give the same nonzero float, that float IS the reference's f32 --
// rounding is monotone.  Otherwise (a value within E of an f32 rounding
// boundary, or of zero) the fragment takes the exact path.  Components that
// are zero at all three vertices are +0.0 in the reference (the chain starts
// 0 + l0 * 0) and are written directly.  Normals: unit vector of the plane
// value through rsqrt + one Newton step whose own residual bounds its error.
// Bit-identical records either way; ~3x fewer instructions per fragment.

constexpr double kU53 = 1.1102230246251565e-16;  // 2^-53, unit roundoff
constexpr uint32_t kPlanesBad = 0x80000000u;      // zmask bit: planes unusable -> exact path

struct __align__(16) PosPlanes {  // the counting pass: positions only
  double A[3], B[3], C[3];
  double ep;
  int32_t x0, y0;
  uint32_t zmask;
  uint32_t pad;
};

struct __align__(16) ItemFast {  // the emission pass: positions + vertex normals, enumeration fields
  double A[6], B[6], C[6];
  double ep, en;
  int32_t x0, y0, bw;
  uint32_t p0;
  float inv_bw;
  uint32_t zmask;  // bits 0-2 position, 3-5 normal components zero at all vertices; kPlanesBad
  uint32_t mat, obj;
};

// shared per-item quantities of the planes: edge-function values at the bbox
// origin pixel centre, 1/area2, and K = sum_i (|e_ix| Hd + |e_iy| Wd) / area2
// (bounds |F_i|/area2-weighted sums over every pixel of the bbox)
struct PlaneBasis {
  double f00[3];
  double ex[3], ey[3];
  double r, K, er;  // r ~ 1/area2 with relative error <= er
  bool ok;
};

__device__ __forceinline__ PlaneBasis plane_basis(const CoverS& c) {
  PlaneBasis b;
  const double sx0 = (double)c.x0 + 0.5, sy0 = (double)c.y0 + 0.5;
  // F_0 is based at vertex 1 (b), F_1 at vertex 2 (c), F_2 at vertex 0 (a) -- cover_test's forms
  b.ex[0] = c.e0x; b.ey[0] = c.e0y;
  b.ex[1] = c.e1x; b.ey[1] = c.e1y;
  b.ex[2] = c.e2x; b.ey[2] = c.e2y;
  b.f00[0] = __fma_rn(c.e0x, sy0 - c.by, -(c.e0y * (sx0 - c.bx)));
  b.f00[1] = __fma_rn(c.e1x, sy0 - c.cy, -(c.e1y * (sx0 - c.cx)));
  b.f00[2] = __fma_rn(c.e2x, sy0 - c.ay, -(c.e2y * (sx0 - c.ax)));
  const double wd = (fmax(c.ax, fmax(c.bx, c.cx)) - fmin(c.ax, fmin(c.bx, c.cx))) + 1.0;
  const double hd = (fmax(c.ay, fmax(c.by, c.cy)) - fmin(c.ay, fmin(c.by, c.cy))) + 1.0;
  // 1/area2 by rcp.approx + one Newton step; its residual bounds its error
  double r0;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(c.area2));
  const double e0 = __fma_rn(-c.area2, r0, 1.0);
  b.r = __fma_rn(r0, e0, r0);
  b.er = fabs(__fma_rn(-c.area2, b.r, 1.0)) + 4.0 * kU53;
  b.K = __fma_rn(fabs(c.e0x) + fabs(c.e1x) + fabs(c.e2x), hd, (fabs(c.e0y) + fabs(c.e1y) + fabs(c.e2y)) * wd) * b.r;
  b.ok = c.area2 > 1e-300 && isfinite(b.K);
  return b;
}

// planes of one 3-component attribute (vertex values W[i][k], winding order)
__device__ __forceinline__ void attr_planes(const PlaneBasis& b, const double W[3][3], double* A, double* B, double* C,
                                            double& err, uint32_t& zbits, bool& ok) {
  double M = 0.0;
  zbits = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    A[k] = __fma_rn(b.f00[2], W[2][k], __fma_rn(b.f00[1], W[1][k], b.f00[0] * W[0][k])) * b.r;
    B[k] = -__fma_rn(b.ey[2], W[2][k], __fma_rn(b.ey[1], W[1][k], b.ey[0] * W[0][k])) * b.r;
    C[k] = __fma_rn(b.ex[2], W[2][k], __fma_rn(b.ex[1], W[1][k], b.ex[0] * W[0][k])) * b.r;
    M = fmax(M, fmax(fabs(W[0][k]), fmax(fabs(W[1][k]), fabs(W[2][k]))));
    zbits |= (W[0][k] == 0.0 && W[1][k] == 0.0 && W[2][k] == 0.0) ? 1u << k : 0u;
  }
  // reference rounding u M (6 + 3K), coefficient rounding ~21 u M K, evaluation
  // ~5 u M K, the interval ends' own rounding ~3 u M K: x2 margin; plus the
  // relative error of r on the three plane terms (<= 3 M K)
  err = M * __fma_rn(kU53 * 64.0 + 4.0 * b.er, b.K, kU53 * 16.0);
  ok = ok && isfinite(err);  // non-finite vertex data -> M non-finite -> exact path
}

__device__ __forceinline__ bool cert_f32(double x, double e, float& out) {
  const float lo = __double2float_rn(__dsub_rn(x, e));
  const float hi = __double2float_rn(__dadd_rn(x, e));
  out = lo;
  return lo == hi && lo != 0.0f;  // NaN fails; a zero would leave its sign undecided
}

__device__ __forceinline__ bool fast_pos(const double* A, const double* B, const double* C, double ep, uint32_t zbits,
                                         int X, int Y, float out[3]) {
  const double xd = (double)X, yd = (double)Y;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float f;
    const bool c = cert_f32(__fma_rn(C[k], yd, __fma_rn(B[k], xd, A[k])), ep, f);
    const bool z = (zbits >> k) & 1u;
    out[k] = z ? 0.0f : f;
    ok = ok && (z || c);
  }
  return ok;
}

__device__ __forceinline__ bool fast_nrm(const double* A, const double* B, const double* C, double en, uint32_t zbits,
                                         int X, int Y, float out[3]) {
  const double xd = (double)X, yd = (double)Y;
  double v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double t = __fma_rn(C[k], yd, __fma_rn(B[k], xd, A[k]));
    v[k] = ((zbits >> k) & 1u) ? 0.0 : t;
  }
  const double q = __fma_rn(v[2], v[2], __fma_rn(v[1], v[1], __dmul_rn(v[0], v[0])));
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(q));
  const double e = __fma_rn(-__dmul_rn(q, y0), y0, 1.0);
  const double y = __fma_rn(y0, __dmul_rn(0.5, e), y0);
  // |y sqrt(q) - 1| <= 3/8 e^2 + rounding; the reference's own normalisation
  // and the plane error (x 2 sqrt(3) / |v|), doubled
  const double eo = __fma_rn(7.0 * en, y, __fma_rn(e, e, 16.0 * kU53));
  bool ok = q > 1e-20;  // the reference's 1e-12 face-normal fallback region (and NaN) -> exact path
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float f;
    const bool c = cert_f32(__dmul_rn(v[k], y), eo, f);
    const bool z = (zbits >> k) & 1u;
    out[k] = z ? 0.0f : f;
    ok = ok && (z || c);
  }
  return ok;
}

// the exact path of one fragment (rare): f64 edge functions, correctly rounded
// barycentrics, the reference's fma chains, sqrt + divisions; f32 record fields
struct Rec6 {
  float w[3], n[3];
};

__device__ __noinline__ Rec6 exact_record(const double* __restrict__ gpos, const double* __restrict__ gvnrm,
                                          const double* __restrict__ gfnrm, const JobSetup* __restrict__ job, int px,
                                          int py, bool want_nrm) {
  Rec6 out;
  float* fw = out.w;
  float* fn = out.n;
  fn[0] = fn[1] = fn[2] = 0.f;
  const JobSetup js = *job;
  CoverS c;
  make_cover(js, 0u, c);
  double f0, f1, f2;
  cover_test(c, px, py, f0, f1, f2);
  const double l0 = ddiv_zd_sel(f0, c.area2), l1 = ddiv_zd_sel(f1, c.area2), l2 = ddiv_zd_sel(f2, c.area2);
  const int o[3] = {0, c.swapped ? 2 : 1, c.swapped ? 1 : 2};
  TriData d;
  const double* P = gpos + 9 * (long long)c.tri;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) d.v[i][k] = P[3 * o[i] + k];
  double w[3];
  interp_pos(d, l0, l1, l2, w);
#pragma unroll
  for (int k = 0; k < 3; ++k) fw[k] = __double2float_rn(w[k]);
  if (!want_nrm) return out;
  const double* N = gvnrm + 9 * (long long)c.tri;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) d.n[i][k] = N[3 * o[i] + k];
#pragma unroll
  for (int k = 0; k < 3; ++k) d.f[k] = gfnrm[3 * (long long)c.tri + k];
  double nn[3];
  interp_nrm(d, l0, l1, l2, nn);
#pragma unroll
  for (int k = 0; k < 3; ++k) fn[k] = __double2float_rn(nn[k]);
  return out;
}

// one batch of <= 32 fragments through the certified fast path (modes
// kCntLeaves, kPpfl, kPofl, kPofa); the store logic mirrors raster_batch
template <int kMode, bool kAtomicAlloc, class Pl>
__device__ __forceinline__ void raster_batch_fast(const CaptureParams& p, const EmitOut& o, Control* ctl,
                                                  const JobSetup* __restrict__ jobs, const Pl* planes, bool valid,
                                                  int k, int px, int py, uint32_t push_local, uint32_t* own_cnt,
                                                  unsigned long long rank0, const uint32_t* item_job_g,
                                                  RasterState<kMode, kAtomicAlloc>& st) {
  static_assert(kMode == kCntLeaves || kMode == kPpfl || kMode == kPofl || kMode == kPofa, "fast modes");
  constexpr bool kKeyed = kMode == kCntLeaves || kMode == kPofl || kMode == kPofa;
  constexpr bool kOwned = kMode == kCntLeaves || kMode == kPofa;
  constexpr bool kNrm = kMode != kCntLeaves;
  const unsigned lane = lane_id();
  const unsigned below = (1u << lane) - 1u;
  bool live = false;
  float fw[3] = {0.f, 0.f, 0.f}, fn[3] = {0.f, 0.f, 0.f};
  uint32_t rmat = 0, robj = 0;
  uint64_t code = ~0ull;
  if (valid) {
    const Pl& P = planes[k];
    const int X = px - P.x0, Y = py - P.y0;
    bool ok = !(P.zmask & kPlanesBad) && fast_pos(P.A, P.B, P.C, P.ep, P.zmask, X, Y, fw);
    if constexpr (kNrm) {
      ok = ok && fast_nrm(P.A + 3, P.B + 3, P.C + 3, P.en, P.zmask >> 3, X, Y, fn);
      rmat = P.mat;
      robj = P.obj;
    }
    if (!ok) {
      atomicAdd(&ctl->leaf_n[1], 1ull);  // diagnostics: fragments through the exact path
      const Rec6 r = exact_record(p.pos, p.vnrm, p.fnrm, jobs + item_job_g[k], px, py, kNrm);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        fw[q] = r.w[q];
        fn[q] = r.n[q];
      }
    }
    live = true;
    if (kKeyed) {
      if (!cell_code(fw[0], fw[1], fw[2], o.levels, &code)) {
        st.bad_range = true;
        live = false;
        code = ~0ull;
      } else if (code < p.cell_lo || code >= p.cell_hi) {  // another shard's leaf
        live = false;
        code = ~0ull;
      }
    }
    if (kNrm && live) ++st.emitted;
  }
  uint32_t local = push_local;
  const bool whole = p.cell_lo == 0 && p.cell_hi >= (1ull << (3 * o.levels));
  if (kOwned && !whole) {
    const unsigned m = __ballot_sync(0xffffffffu, live);
    const unsigned grp = __match_any_sync(0xffffffffu, valid ? k : -1);
    local = own_cnt[k] + (uint32_t)__popc(grp & m & below);
    __syncwarp();
    if (valid && (int)lane == 31 - __clz(grp)) own_cnt[k] += (uint32_t)__popc(grp & m);
    __syncwarp();
  }
  const unsigned long long rank = __shfl_sync(0xffffffffu, rank0, k) + local;
  if (kMode == kCntLeaves) {
    const unsigned grp = __match_any_sync(0xffffffffu, code);
    if (live && (int)lane == __ffs(grp) - 1) atomicAdd(&o.leaf_counts[code - p.cell_lo], (uint32_t)__popc(grp));
    if (o.tile_sums) {  // directory tile totals: the directory pass then needs no look-back chain
      const uint32_t tkey = live ? (uint32_t)((code - p.cell_lo) >> kDirSumShift) : 0xffffffffu;
      const unsigned gt = __match_any_sync(0xffffffffu, tkey);
      if (live && (int)lane == __ffs(gt) - 1) atomicAdd(&o.tile_sums[tkey], (uint32_t)__popc(gt));
    }
    return;
  }
  long long slot = -1;
  bool leaf_first = false;
  if (kMode == kPofa) {
    const unsigned grp = __match_any_sync(0xffffffffu, code);
    const int leader = __ffs(grp) - 1;
    const unsigned long long lc = live ? code - p.cell_lo : 0ull;
    uint32_t off = 0, cnt = 0, base = 0;
    if (live) {
      off = __ldg(&o.offsets[lc]);
      cnt = lc + 1 < p.cell_hi - p.cell_lo ? __ldg(&o.offsets[lc + 1]) - off : __ldg(&o.counts[lc]);
    }
    if (live && (int)lane == leader) base = atomicAdd(&o.cursors[lc], (uint32_t)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (live) {
      const uint32_t cur = base + (uint32_t)__popc(grp & below);
      leaf_first = cur == 0;
      if (cur >= cnt) {
        st.bad_pass = true;
      } else {
        slot = (long long)(off - o.base) + cur;
        if (slot >= o.capacity) {  // speculative pool smaller than the exact count
          st.short_pool = true;
          slot = -1;
        }
      }
    }
  } else {
    if (kAtomicAlloc) {
      const unsigned m = __ballot_sync(0xffffffffu, live);
      unsigned long long base = 0;
      if (m && lane == (unsigned)(__ffs(m) - 1)) base = atomicAdd(&ctl->alloc, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, m ? __ffs(m) - 1 : 0);
      if (live) slot = (long long)(base + __popc(m & below));
    } else if (live) {
      slot = (long long)rank;
    }
    if (slot >= o.capacity) slot = -1;
    uint64_t key = ~0ull;
    if (slot >= 0) {
      if (kMode == kPpfl) {
        key = (uint64_t)py * (uint64_t)o.width + (uint64_t)px;
        if ((long long)key >= o.n_keys) {
          st.bad_key = true;
          slot = -1;
          key = ~0ull;
        }
      } else {
        key = code;
      }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const int last = 31 - __clz(grp);
    int32_t old = -1;
    if (slot >= 0 && (int)lane == last) old = atomicExch(&o.heads[key], (int32_t)slot);
    old = __shfl_sync(0xffffffffu, old, last);
    const unsigned lower = grp & below;
    const int32_t prev_slot = __shfl_sync(0xffffffffu, (int32_t)slot, lower ? 31 - __clz(lower) : (int)lane);
    if (slot >= 0) o.prev[slot] = lower ? prev_slot : old;
  }
  if (slot >= 0) {
    const uint32_t s32 = (uint32_t)slot;
    float* pp = o.pos + 3ull * s32;
    float* np = o.nrm + 3ull * s32;
    pp[0] = fw[0]; pp[1] = fw[1]; pp[2] = fw[2];
    np[0] = fn[0]; np[1] = fn[1]; np[2] = fn[2];
    o.mat[s32] = rmat;
    o.obj[s32] = robj;
    if (kMode == kPofa)
      o.prev[s32] = (o.flags & FHV_EXACT_ORDER)
                        ? (int32_t)((uint32_t)rank | ((o.flags & kSegFlags) && leaf_first ? 0x80000000u : 0u))
                        : -1;
  }
}

template <int kMode, bool kAtomicAlloc, bool kFast = false>
__global__ void __launch_bounds__(kRasterBlock, FHV_RASTER_MINB) k_raster(CaptureParams p, const JobSetup* __restrict__ jobs,
                                                         const uint32_t* __restrict__ item_job,
                                                         const uint32_t* __restrict__ item_p0,
                                                         const unsigned long long* __restrict__ item_off,
                                                         long long n_items, const unsigned long long* n_dev,
                                                         uint32_t* __restrict__ item_cnt,
                                                         uint4* __restrict__ item_mask, EmitOut o, Control* ctl) {
  static_assert(kMode == kCnt || kMode == kCntLeaves, "k_raster is the counting pass; emission is k_emit");
  constexpr bool kOwned = kMode == kCntLeaves || kMode == kPofa;
  __shared__ CoverS cs_all[kRasterWarps][32];
  __shared__ int32_t qpx_all[kRasterWarps][64], qpy_all[kRasterWarps][64];
  __shared__ uint32_t qmeta_all[kRasterWarps][64];
  __shared__ double rcp_all[kRasterWarps][32];  // recip_of(area2).y per item (kept out of CoverS: the sweep's stride)
  __shared__ uint32_t own_all[kRasterWarps][32];
  __shared__ uint32_t ijob_all[kRasterWarps][32];
  extern __shared__ __align__(16) unsigned char raster_dyn[];  // kFast: PosPlanes[kRasterWarps][32]
  const unsigned lane = lane_id();
  const int wib = threadIdx.x >> 5;
  PosPlanes* pp = reinterpret_cast<PosPlanes*>(raster_dyn) + 32 * wib;
  CoverS* cs = cs_all[wib];
  int32_t* q_px = qpx_all[wib];
  int32_t* q_py = qpy_all[wib];
  uint32_t* q_meta = qmeta_all[wib];
  uint32_t* own_cnt = own_all[wib];
  uint32_t* ijob = ijob_all[wib];
  const unsigned below = (1u << lane) - 1u;
  if (n_dev) {  // speculative launch: run the true count, or flag a plan that was too small
    const long long nd = (long long)*n_dev;
    if (nd > n_items && blockIdx.x == 0 && threadIdx.x == 0) raise_status(&ctl->status, FHV_RETRY_ITEMS);
    if (nd < n_items) n_items = nd;
  }
  const long long n_groups = (n_items + 31) / 32;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  RasterState<kMode, kAtomicAlloc> st;
  for (long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; g < n_groups; g += nw) {
    const long long item = g * 32 + lane;
    uint32_t npix = 0;
    unsigned long long rank0 = 0;
    int px = 0, py = 0, xend = 0;
    double k0 = 0.0, k1 = 0.0, k2 = 0.0;
    if (item < n_items) {
      const uint32_t jid = item_job[item];
      const JobSetup js = jobs[jid];
      const uint32_t p0 = item_p0[item];
      const unsigned long long pe = (unsigned long long)js.bw * (unsigned long long)js.bh;
      npix = (unsigned long long)p0 + kItemPix < pe ? kItemPix : (uint32_t)(pe - p0);
      make_cover(js, p0, cs[lane]);
      if (kMode == kCntLeaves && !kFast) {  // the positions the keying batches read; their shared reciprocal
        const char* P = reinterpret_cast<const char*>(p.pos + 9 * (long long)js.tri);
        prefetch_l1(P);
        prefetch_l1(P + 64);
        rcp_all[wib][lane] = recip_of(cs[lane].area2 > 0.0 ? cs[lane].area2 : 1.0).y;
      }
      if (kMode == kCntLeaves && kFast) {  // position planes of my item (certified fast keys)
        TriData d;
        load_tri_pos(p, js.tri, js.swapped, d);
        const PlaneBasis b = plane_basis(cs[lane]);
        PosPlanes& P = pp[lane];
        bool ok = b.ok;
        uint32_t z = 0;
        double e = 0.0;
        attr_planes(b, d.v, P.A, P.B, P.C, e, z, ok);
        P.ep = e;
        P.x0 = js.x0;
        P.y0 = js.y0;
        P.zmask = z | (ok ? 0u : kPlanesBad);
      }
      ijob[lane] = jid;
      if (!kOwned && kMode != kCnt && !kAtomicAlloc) rank0 = item_off[item];
      if (kOwned && kMode == kPofa) rank0 = item_off[item];
      const uint32_t r = p0 / (uint32_t)js.bw;
      px = js.x0 + (int)(p0 - r * (uint32_t)js.bw);
      py = js.y0 + (int)r;
      xend = js.x0 + js.bw;
      const CoverS& c = cs[lane];
      const double sy = __dadd_rn((double)py, 0.5);
      k0 = __dmul_rn(c.e0x, __dsub_rn(sy, c.by));
      k1 = __dmul_rn(c.e1x, __dsub_rn(sy, c.cy));
      k2 = __dmul_rn(c.e2x, __dsub_rn(sy, c.ay));
    }
    {  // the next group's item records
      const long long nx = item + nw * 32;
      if (nx < n_items) {
        prefetch_l1(item_job + nx);
        prefetch_l1(item_p0 + nx);
      }
    }
    own_cnt[lane] = 0;
    __syncwarp();
    uint32_t covered = 0;  // covered pixels of my item so far
    uint32_t mw0 = 0, mw1 = 0, mw2 = 0, mw3 = 0;  // coverage bit mask of my item (<= 128 pixels)
    int qn = 0;            // queued fragments (warp-uniform)
    for (uint32_t j = 0; __any_sync(0xffffffffu, j < npix); ++j) {
      bool cov = false;
      int cpx = px, cpy = py;
      if (j < npix) {
        const CoverS& c = cs[lane];
        const double sx = __dadd_rn((double)px, 0.5);
        // the three edge functions as independent chains (no early-out
        // branches: ILP instead of divergence; same values either way)
        const double f0 = __dsub_rn(k0, __dmul_rn(c.e0y, __dsub_rn(sx, c.bx)));
        const double f1 = __dsub_rn(k1, __dmul_rn(c.e1y, __dsub_rn(sx, c.cx)));
        const double f2 = __dsub_rn(k2, __dmul_rn(c.e2y, __dsub_rn(sx, c.ax)));
        const bool in0 = f0 > 0.0 || (f0 == 0.0 && (c.tl & 1u));
        const bool in1 = f1 > 0.0 || (f1 == 0.0 && (c.tl & 2u));
        const bool in2 = f2 > 0.0 || (f2 == 0.0 && (c.tl & 4u));
        cov = in0 & in1 & in2;
        if (++px == xend) {
          px = c.x0;
          ++py;
          const double sy = __dadd_rn((double)py, 0.5);
          k0 = __dmul_rn(c.e0x, __dsub_rn(sy, c.by));
          k1 = __dmul_rn(c.e1x, __dsub_rn(sy, c.cy));
          k2 = __dmul_rn(c.e2x, __dsub_rn(sy, c.ay));
        }
      }
      if (cov) {  // j is warp-uniform: a uniform switch, no local memory
        const uint32_t bit = 1u << (j & 31u);
        switch (j >> 5) {
          case 0: mw0 |= bit; break;
          case 1: mw1 |= bit; break;
          case 2: mw2 |= bit; break;
          default: mw3 |= bit; break;
        }
      }
      if (kMode == kCnt) {
        covered += cov ? 1u : 0u;
        continue;
      }
      const unsigned m = __ballot_sync(0xffffffffu, cov);
      if (cov) {
        const int slot = qn + __popc(m & below);
        q_px[slot] = cpx;
        q_py[slot] = cpy;
        q_meta[slot] = lane | (covered << 5);
        ++covered;
      }
      qn += __popc(m);
      if (qn >= 32) {
        __syncwarp();
        {
          const uint32_t mt = q_meta[lane];
          if constexpr (kMode == kCntLeaves && kFast)
            raster_batch_fast<kMode, kAtomicAlloc>(p, o, ctl, jobs, pp, true, (int)(mt & 31u), q_px[lane],
                                                   q_py[lane], mt >> 5, own_cnt, rank0, ijob, st);
          else if constexpr (kMode == kCntLeaves)
            raster_batch<kMode, kAtomicAlloc>(p, o, ctl, cs, true, (int)(mt & 31u), q_px[lane], q_py[lane], mt >> 5,
                                              own_cnt, rank0, ijob, st, rcp_all[wib]);
        }
        __syncwarp();
        if ((int)lane < qn - 32) {
          q_px[lane] = q_px[32 + lane];
          q_py[lane] = q_py[32 + lane];
          q_meta[lane] = q_meta[32 + lane];
        }
        qn -= 32;
        __syncwarp();
      }
    }
    if (kMode != kCnt && qn > 0) {
      __syncwarp();
      const bool v = (int)lane < qn;
      const uint32_t mt = v ? q_meta[lane] : 0u;
      if constexpr (kMode == kCntLeaves && kFast)
        raster_batch_fast<kMode, kAtomicAlloc>(p, o, ctl, jobs, pp, v, (int)(mt & 31u), v ? q_px[lane] : 0,
                                               v ? q_py[lane] : 0, mt >> 5, own_cnt, rank0, ijob, st);
      else if constexpr (kMode == kCntLeaves)
        raster_batch<kMode, kAtomicAlloc>(p, o, ctl, cs, v, (int)(mt & 31u), v ? q_px[lane] : 0, v ? q_py[lane] : 0,
                                          mt >> 5, own_cnt, rank0, ijob, st, rcp_all[wib]);
    }
    __syncwarp();
    if (item < n_items) {
      if (kMode == kCnt) item_cnt[item] = covered;
      if (kMode == kCntLeaves)
        item_cnt[item] = (p.cell_lo == 0 && p.cell_hi >= (1ull << (3 * o.levels))) ? covered : own_cnt[lane];
      item_mask[item] = make_uint4(mw0, mw1, mw2, mw3);
    }
    __syncwarp();
  }
  if (kMode == kPofa) {
    // pass-2 emitted count (compared with pass 1, fhv/storage.py:614-617)
    unsigned long long e = st.emitted;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if (lane == 0 && e) atomicAdd(&ctl->alloc, e);
  }
  if (st.bad_range) raise_status(&ctl->status, FHV_RANGE);
  if (st.bad_pass) raise_status(&ctl->status, FHV_PASS_MISMATCH);
  if (st.bad_key) raise_status(&ctl->status, FHV_BAD_ARGS);
}

// position of the n-th (0-based) set bit of v (v has > n set bits)
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t v, uint32_t n) {
  uint32_t pos = 0;
#pragma unroll
  for (int w = 16; w > 0; w >>= 1) {
    const uint32_t lo = (uint32_t)__popc(v & ((1u << w) - 1u));
    if (n >= lo) {
      n -= lo;
      v >>= w;
      pos += (uint32_t)w;
    }
  }
  return pos;
}

// emission pass: the counting pass left each item's coverage mask, so the
// warp enumerates exactly the covered pixels of its 32 items, 32 fragments
// per step (flat index -> item by a 5-step shuffle search over the items'
// fragment prefix sums -> pixel by select-n-th-bit), no coverage sweep.
template <int kMode, bool kAtomicAlloc>
__global__ void __launch_bounds__(kRasterBlock, FHV_RASTER_MINB) k_emit(CaptureParams p, const JobSetup* __restrict__ jobs,
                                                       const uint32_t* __restrict__ item_job,
                                                       const uint32_t* __restrict__ item_p0,
                                                       const unsigned long long* __restrict__ item_off,
                                                       const uint4* __restrict__ item_mask, long long n_items,
                                                       const unsigned long long* n_dev, EmitOut o, Control* ctl) {
  static_assert(kMode == kList || kMode == kPpfl || kMode == kPofl || kMode == kPofa || kMode == kDsDepth ||
                    kMode == kDsIndex || kMode == kDsWrite,
                "emission modes only");
  __shared__ CoverR cs_all[kRasterWarps][32];
  __shared__ uint32_t own_all[kRasterWarps][32];
  __shared__ uint32_t ijob_all[kRasterWarps][32];
  const unsigned lane = lane_id();
  const int wib = threadIdx.x >> 5;
  CoverR* cs = cs_all[wib];
  uint32_t* own_cnt = own_all[wib];
  uint32_t* ijob = ijob_all[wib];
  if (n_dev) {  // speculative launch: run the true count, or flag a plan that was too small
    const long long nd = (long long)*n_dev;
    if (nd > n_items && blockIdx.x == 0 && threadIdx.x == 0) raise_status(&ctl->status, FHV_RETRY_ITEMS);
    if (nd < n_items) n_items = nd;
  }
  const long long n_groups = (n_items + 31) / 32;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  RasterState<kMode, kAtomicAlloc> st;
  for (long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; g < n_groups; g += nw) {
    const long long item = g * 32 + lane;
    uint4 mk = make_uint4(0u, 0u, 0u, 0u);
    unsigned long long rank0 = 0;
    if (item < n_items) {
      const uint32_t jid = item_job[item];
      mk = item_mask[item];
      if (!kAtomicAlloc && (kMode != kPofa || (o.flags & FHV_EXACT_ORDER))) rank0 = item_off[item];
      const JobSetup js = jobs[jid];
      if (mk.x | mk.y | mk.z | mk.w) prefetch_tri(p, js.tri);
      make_cover(js, item_p0[item], cs[lane]);
      ijob[lane] = jid;
    }
    {  // the next group's item records
      const long long nx = item + nw * 32;
      if (nx < n_items) {
        prefetch_l1(item_job + nx);
        prefetch_l1(item_mask + nx);
        prefetch_l1(item_p0 + nx);
        if (!kAtomicAlloc && (kMode != kPofa || (o.flags & FHV_EXACT_ORDER))) prefetch_l1(item_off + nx);
      }
    }
    own_cnt[lane] = 0;
    const uint32_t cnt = (uint32_t)(__popc(mk.x) + __popc(mk.y) + __popc(mk.z) + __popc(mk.w));
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= (unsigned)d) inc += y;
    }
    const uint32_t E = inc - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    for (uint32_t s = 0; s < total; s += 32) {
      const uint32_t f = s + lane;
      const bool valid = f < total;
      int k = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t Ec = __shfl_sync(0xffffffffu, E, k + step);
        if (valid && Ec <= f) k += step;
      }
      const uint32_t local = f - __shfl_sync(0xffffffffu, E, k);
      const uint32_t m0 = __shfl_sync(0xffffffffu, mk.x, k), m1 = __shfl_sync(0xffffffffu, mk.y, k);
      const uint32_t m2 = __shfl_sync(0xffffffffu, mk.z, k), m3 = __shfl_sync(0xffffffffu, mk.w, k);
      int px = 0, py = 0;
      if (valid) {
        uint32_t rem = local, wv = m0, word = 0;
        const uint32_t c0 = (uint32_t)__popc(m0);
        if (rem >= c0) {
          rem -= c0;
          wv = m1;
          word = 1;
          const uint32_t c1 = (uint32_t)__popc(m1);
          if (rem >= c1) {
            rem -= c1;
            wv = m2;
            word = 2;
            const uint32_t c2 = (uint32_t)__popc(m2);
            if (rem >= c2) {
              rem -= c2;
              wv = m3;
              word = 3;
            }
          }
        }
        const CoverS& c = cs[k];
        const uint32_t q = c.p0 + 32u * word + nth_set_bit(wv, rem);
        const uint32_t bw = (uint32_t)c.bw;
        uint32_t r;
        if (q < (1u << 22)) {  // |float estimate - q / bw| <= 2^-23 q < 1/2 here; fix it up exactly
          r = (uint32_t)__fmul_rn((float)q, c.inv_bw);
          const int rem = (int)(q - r * bw);
          r = rem < 0 ? r - 1 : (rem >= (int)bw ? r + 1 : r);
        } else {
          r = q / bw;
        }
        px = c.x0 + (int)(q - r * bw);
        py = c.y0 + (int)r;
      }
      raster_batch<kMode, kAtomicAlloc>(p, o, ctl, cs, valid, k, px, py, local, own_cnt, rank0, ijob, st);
    }
    __syncwarp();
  }
  if (kMode == kPofa) {
    // pass-2 emitted count (compared with pass 1, fhv/storage.py:614-617)
    unsigned long long e = st.emitted;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if (lane == 0 && e) atomicAdd(&ctl->alloc, e);
  }
  if (st.bad_range) raise_status(&ctl->status, FHV_RANGE);
  if (st.bad_pass) raise_status(&ctl->status, FHV_PASS_MISMATCH);
  if (st.bad_key) raise_status(&ctl->status, FHV_BAD_ARGS);
  if (st.short_pool) raise_status(&ctl->status, FHV_NEED_POOL);
}

// emission pass through the certified fast path (POFA / POFL / PPFL): the
// same mask enumeration as k_emit, per-item planes (ItemFast) in dynamic
// shared memory instead of the coverage state, exact fallback per fragment
#ifndef FHV_EMIT_FAST_MINB
#define FHV_EMIT_FAST_MINB 3
#endif
template <int kMode, bool kAtomicAlloc>
__global__ void __launch_bounds__(32 * kEmitFastWarps, FHV_EMIT_FAST_MINB)
    k_emit_fast(CaptureParams p, const JobSetup* __restrict__ jobs, const uint32_t* __restrict__ item_job,
                const uint32_t* __restrict__ item_p0, const unsigned long long* __restrict__ item_off,
                const uint4* __restrict__ item_mask, long long n_items, const unsigned long long* n_dev, EmitOut o,
                Control* ctl) {
  static_assert(kMode == kPpfl || kMode == kPofl || kMode == kPofa, "record-emitting modes");
  extern __shared__ __align__(16) unsigned char emit_dyn[];  // ItemFast[warps][32]
  __shared__ uint32_t own_all[kEmitFastWarps][32];
  __shared__ uint32_t ijob_all[kEmitFastWarps][32];
  const unsigned lane = lane_id();
  const int wib = threadIdx.x >> 5;
  ItemFast* fast = reinterpret_cast<ItemFast*>(emit_dyn) + 32 * wib;
  uint32_t* own_cnt = own_all[wib];
  uint32_t* ijob = ijob_all[wib];
  if (n_dev) {  // speculative launch: run the true count, or flag a plan that was too small
    const long long nd = (long long)*n_dev;
    if (nd > n_items && blockIdx.x == 0 && threadIdx.x == 0) raise_status(&ctl->status, FHV_RETRY_ITEMS);
    if (nd < n_items) n_items = nd;
  }
  const long long n_groups = (n_items + 31) / 32;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  RasterState<kMode, kAtomicAlloc> st;
  for (long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; g < n_groups; g += nw) {
    const long long item = g * 32 + lane;
    uint4 mk = make_uint4(0u, 0u, 0u, 0u);
    unsigned long long rank0 = 0;
    if (item < n_items) {
      const uint32_t jid = item_job[item];
      mk = item_mask[item];
      if (!kAtomicAlloc && (kMode != kPofa || (o.flags & FHV_EXACT_ORDER))) rank0 = item_off[item];
      const JobSetup js = jobs[jid];
      const uint32_t p0 = item_p0[item];
      ItemFast& F = fast[lane];
      F.x0 = js.x0;
      F.y0 = js.y0;
      F.bw = js.bw;
      F.p0 = p0;
      F.inv_bw = 1.0f / (float)(js.bw > 0 ? js.bw : 1);
      ijob[lane] = jid;
      if (mk.x | mk.y | mk.z | mk.w) {  // planes of my item's positions and vertex normals
        PlaneBasis b;
        {
          CoverS c;
          make_cover(js, p0, c);
          b = plane_basis(c);
        }
        bool ok = b.ok;
        uint32_t zp = 0, zn = 0;
        double ep = 0.0, en = 0.0;
        const int o3[3] = {0, js.swapped ? 2 : 1, js.swapped ? 1 : 2};
        {
          double W[3][3];
          const double* P = p.pos + 9 * (long long)js.tri;
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int q = 0; q < 3; ++q) W[i][q] = __ldg(&P[3 * o3[i] + q]);
          attr_planes(b, W, F.A, F.B, F.C, ep, zp, ok);
        }
        {
          double W[3][3];
          const double* N = p.vnrm + 9 * (long long)js.tri;
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int q = 0; q < 3; ++q) W[i][q] = __ldg(&N[3 * o3[i] + q]);
          attr_planes(b, W, F.A + 3, F.B + 3, F.C + 3, en, zn, ok);
        }
        F.ep = ep;
        F.en = en;
        F.zmask = zp | (zn << 3) | (ok ? 0u : kPlanesBad);
        F.mat = __ldg(&p.mat[js.tri]);
        F.obj = __ldg(&p.obj[js.tri]);
      }
    }
    {  // the next group's item records
      const long long nx = item + nw * 32;
      if (nx < n_items) {
        prefetch_l1(item_job + nx);
        prefetch_l1(item_mask + nx);
        prefetch_l1(item_p0 + nx);
        if (!kAtomicAlloc && (kMode != kPofa || (o.flags & FHV_EXACT_ORDER))) prefetch_l1(item_off + nx);
      }
    }
    own_cnt[lane] = 0;
    const uint32_t cnt = (uint32_t)(__popc(mk.x) + __popc(mk.y) + __popc(mk.z) + __popc(mk.w));
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= (unsigned)d) inc += y;
    }
    const uint32_t E = inc - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    for (uint32_t s0 = 0; s0 < total; s0 += 32) {
      const uint32_t f = s0 + lane;
      const bool valid = f < total;
      int k = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t Ec = __shfl_sync(0xffffffffu, E, k + step);
        if (valid && Ec <= f) k += step;
      }
      const uint32_t local = f - __shfl_sync(0xffffffffu, E, k);
      const uint32_t m0 = __shfl_sync(0xffffffffu, mk.x, k), m1 = __shfl_sync(0xffffffffu, mk.y, k);
      const uint32_t m2 = __shfl_sync(0xffffffffu, mk.z, k), m3 = __shfl_sync(0xffffffffu, mk.w, k);
      int px = 0, py = 0;
      if (valid) {
        uint32_t rem = local, wv = m0, word = 0;
        const uint32_t c0 = (uint32_t)__popc(m0);
        if (rem >= c0) {
          rem -= c0;
          wv = m1;
          word = 1;
          const uint32_t c1 = (uint32_t)__popc(m1);
          if (rem >= c1) {
            rem -= c1;
            wv = m2;
            word = 2;
            const uint32_t c2 = (uint32_t)__popc(m2);
            if (rem >= c2) {
              rem -= c2;
              wv = m3;
              word = 3;
            }
          }
        }
        const ItemFast& F = fast[k];
        const uint32_t q = F.p0 + 32u * word + nth_set_bit(wv, rem);
        const uint32_t bw = (uint32_t)F.bw;
        uint32_t r;
        if (q < (1u << 22)) {  // |float estimate - q / bw| <= 2^-23 q < 1/2 here; fix it up exactly
          r = (uint32_t)__fmul_rn((float)q, F.inv_bw);
          const int rm = (int)(q - r * bw);
          r = rm < 0 ? r - 1 : (rm >= (int)bw ? r + 1 : r);
        } else {
          r = q / bw;
        }
        px = F.x0 + (int)(q - r * bw);
        py = F.y0 + (int)r;
      }
      raster_batch_fast<kMode, kAtomicAlloc>(p, o, ctl, jobs, fast, valid, k, px, py, local, own_cnt, rank0, ijob,
                                             st);
    }
    __syncwarp();
  }
  if (kMode == kPofa) {
    // pass-2 emitted count (compared with pass 1, fhv/storage.py:614-617)
    unsigned long long e = st.emitted;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if (lane == 0 && e) atomicAdd(&ctl->alloc, e);
  }
  if (st.bad_range) raise_status(&ctl->status, FHV_RANGE);
  if (st.bad_pass) raise_status(&ctl->status, FHV_PASS_MISMATCH);
  if (st.bad_key) raise_status(&ctl->status, FHV_BAD_ARGS);
  if (st.short_pool) raise_status(&ctl->status, FHV_NEED_POOL);
}

// ---------------------------------------------------------------------------
// EXACT_ORDER fix-ups

// per key: chain must run from the most recent insertion (highest pool
// index) down, as sequential linked_insert leaves it (fhv/_ckern.pyx:119-123)
constexpr int kChainLocal = 96;

__device__ void heap_sift(int32_t* a, long long n, long long i) {
  // min-heap on value -> sorting extracts ascending; we want descending
  while (true) {
    long long l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && a[l] < a[m]) m = l;
    if (r < n && a[r] < a[m]) m = r;
    if (m == i) return;
    const int32_t t = a[i]; a[i] = a[m]; a[m] = t;
    i = m;
  }
}

__global__ void k_chain_order(int32_t* __restrict__ heads, int32_t* __restrict__ prev, long long n_keys,
                              int32_t* __restrict__ spill, unsigned long long* spill_top) {
  int32_t buf[kChainLocal];
  for (long long key = blockIdx.x * (long long)blockDim.x + threadIdx.x; key < n_keys;
       key += (long long)gridDim.x * blockDim.x) {
    const int32_t h = heads[key];
    if (h < 0) continue;
    long long n = 0;
    bool sorted = true;
    int32_t last = 0x7fffffff;
    for (int32_t k = h; k >= 0; k = prev[k]) {
      if (n < kChainLocal) buf[n] = k;
      sorted = sorted && k < last;
      last = k;
      ++n;
    }
    if (sorted) continue;
    int32_t* a = buf;
    if (n > kChainLocal) {
      a = spill + atomicAdd(spill_top, (unsigned long long)n);
      long long m = 0;
      for (int32_t k = h; k >= 0; k = prev[k]) a[m++] = k;
    }
    if (n <= kChainLocal) {
      for (long long i = 1; i < n; ++i) {  // insertion sort, descending
        const int32_t v = a[i];
        long long j = i - 1;
        while (j >= 0 && a[j] < v) { a[j + 1] = a[j]; --j; }
        a[j + 1] = v;
      }
    } else {
      for (long long i = n / 2 - 1; i >= 0; --i) heap_sift(a, n, i);
      for (long long e = n - 1; e > 0; --e) {
        const int32_t t = a[0]; a[0] = a[e]; a[e] = t;
        heap_sift(a, e, 0);
      }
    }
    heads[key] = a[0];
    for (long long i = 0; i < n; ++i) prev[a[i]] = i + 1 < n ? a[i + 1] : -1;
  }
}

// per leaf: restore emission order (stable counting sort semantics of
// pofa_scatter, fhv/_ckern.pyx:135-142) from the parked ranks, then
// prev_index = -1 (fhv/storage.py:439)
__global__ void k_leaf_order(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts,
                             long long n_leaves, unsigned long long base, unsigned long long cap,
                             float* __restrict__ pos, float* __restrict__ nrm, uint32_t* __restrict__ mat,
                             uint32_t* __restrict__ obj, int32_t* __restrict__ prev) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n_leaves;
       c += (long long)gridDim.x * blockDim.x) {
    const uint32_t n = counts[c];
    if (n == 0) continue;
    const long long off = (long long)(offsets[c] - base);
    if ((unsigned long long)off + n > cap) continue;  // speculative pool too small: the caller re-scatters
    uint32_t* rk = reinterpret_cast<uint32_t*>(prev + off);
    for (uint32_t i = 1; i < n; ++i) {
      const uint32_t r = rk[i];
      if (r >= rk[i - 1]) continue;
      const long long si = off + i;
      const float a0 = pos[3 * si], a1 = pos[3 * si + 1], a2 = pos[3 * si + 2];
      const float b0 = nrm[3 * si], b1 = nrm[3 * si + 1], b2 = nrm[3 * si + 2];
      const uint32_t m = mat[si], ob = obj[si];
      long long j = (long long)i - 1;
      while (j >= 0 && rk[j] > r) {
        const long long s = off + j, t = s + 1;
        pos[3 * t] = pos[3 * s]; pos[3 * t + 1] = pos[3 * s + 1]; pos[3 * t + 2] = pos[3 * s + 2];
        nrm[3 * t] = nrm[3 * s]; nrm[3 * t + 1] = nrm[3 * s + 1]; nrm[3 * t + 2] = nrm[3 * s + 2];
        mat[t] = mat[s];
        obj[t] = obj[s];
        rk[j + 1] = rk[j];
        --j;
      }
      const long long t = off + j + 1;
      pos[3 * t] = a0; pos[3 * t + 1] = a1; pos[3 * t + 2] = a2;
      nrm[3 * t] = b0; nrm[3 * t + 1] = b1; nrm[3 * t + 2] = b2;
      mat[t] = m;
      obj[t] = ob;
      rk[j + 1] = r;
    }
    for (uint32_t i = 0; i < n; ++i) prev[off + i] = -1;
  }
}

// ---------------------------------------------------------------------------
// EXACT_ORDER for a POFA pool, over SLOTS (the pass-2 path the bench times).
// Pass 2 parked every record's emission rank in prev, bit 31 set on the first
// slot of its leaf (a segment start: the group leader's cursor returned 0).
// The in-leaf order only breaks where a leaf took fragments from more than
// one warp: a warp enumerates its fragments in emission order and a
// same-leaf group takes consecutive cursor slots in lane order.
//   k_leaf_fix   a warp per tile of 128 slots (+64 look-ahead): segment
//                starts by ballots, a segment with a rank below its
//                predecessor's is re-sorted by rank-by-count through per-warp
//                shared memory, coalesced loads and stores.  Segments starting
//                in the tile that do not end inside the look-ahead are listed
//                for k_leaf_fix_big.
//   k_leaf_fix_big  a CTA per listed segment: end by a flag search, sorted
//                check; segments of <= 256 slots ranked by counting (a
//                thread per record, one barrier), longer ones by a bitonic
//                sort of (rank, index) keys in shared memory (<= 4096) or
//                scratch, records gathered through scratch.
//   prev := -1   one memset (fhv/storage.py:439).
// No directory access at all; when nothing is out of order the cost is one
// coalesced read of the ranks.  Result: records of each leaf in ascending
// emission rank -- pofa_scatter's stable order (fhv/_ckern.pyx:135-142).

constexpr int kSortSmem = 4096;
constexpr uint32_t kSegBit = 0x80000000u;

struct PoolRefs {
  float* pos;
  float* nrm;
  uint32_t* mat;
  uint32_t* obj;
  uint32_t* rank;  // = prev, still holding the parked ranks (+ segment bits)
};

__device__ __forceinline__ void stage_record(const PoolRefs& pl, uint32_t* __restrict__ R, long long s) {
  R[0] = __float_as_uint(pl.pos[3 * s]); R[1] = __float_as_uint(pl.pos[3 * s + 1]);
  R[2] = __float_as_uint(pl.pos[3 * s + 2]); R[3] = __float_as_uint(pl.nrm[3 * s]);
  R[4] = __float_as_uint(pl.nrm[3 * s + 1]); R[5] = __float_as_uint(pl.nrm[3 * s + 2]);
  R[6] = pl.mat[s]; R[7] = pl.obj[s]; R[8] = pl.rank[s];
}

// the segment bit belongs to the SLOT, not the record: a moved record takes
// the destination slot's bit (slot bits never change, so concurrent tiles
// reading their look-ahead always see stable segment starts)
__device__ __forceinline__ void unstage_record(const PoolRefs& pl, const uint32_t* __restrict__ R, long long t,
                                               uint32_t slot_bit) {
  pl.pos[3 * t] = __uint_as_float(R[0]); pl.pos[3 * t + 1] = __uint_as_float(R[1]);
  pl.pos[3 * t + 2] = __uint_as_float(R[2]); pl.nrm[3 * t] = __uint_as_float(R[3]);
  pl.nrm[3 * t + 1] = __uint_as_float(R[4]); pl.nrm[3 * t + 2] = __uint_as_float(R[5]);
  pl.mat[t] = R[6]; pl.obj[t] = R[7]; pl.rank[t] = (R[8] & ~kSegBit) | slot_bit;
}

// k_leaf_fix: a WARP per tile of 128 slots (+ 64 look-ahead = 6 chunks of
// 32), no block barriers.  Ranks in registers (coalesced), segment starts by
// ballots, segment bounds by bit scans, disorder by a shuffle of the previous
// rank; the elements of a disordered segment are ranked by counting over the
// segment's ranks (per-warp shared memory) and staged at their destination in
// per-warp shared memory, then stored back (coalesced).
constexpr int kFixChunks = 6;
constexpr int kFixWarpTile = 128;                     // segments starting here are this warp's
constexpr int kFixWarpRegion = 32 * kFixChunks;       // 192
#ifndef FHV_FIX_PER_SM
#define FHV_FIX_PER_SM 12  // fix-up grid: CTAs per SM (each warp strides over 128-slot tiles)
#endif
#ifndef FHV_FIX_WARPS
#define FHV_FIX_WARPS 2
#endif
constexpr int kFixWarps = FHV_FIX_WARPS;              // warps per CTA

struct FixWarpSmem {
  uint32_t rk[kFixWarpRegion];
  uint8_t dis[kFixWarpRegion];
  uint8_t dst_set[kFixWarpRegion];
  uint8_t mv_i[kFixWarpRegion], mv_lo[kFixWarpRegion], mv_hi[kFixWarpRegion];
  float pos[kFixWarpRegion][3], nrm[kFixWarpRegion][3];
  uint32_t mat[kFixWarpRegion], obj[kFixWarpRegion], rank[kFixWarpRegion];
};

__global__ void __launch_bounds__(32 * kFixWarps) k_leaf_fix(PoolRefs pl, const unsigned long long* __restrict__ n_dev,
                                                             long long cap, unsigned long long* big_list,
                                                             unsigned long long* n_big, unsigned long long big_cap,
                                                             unsigned long long* n_fixed_total, int* status) {
  __shared__ FixWarpSmem smem_all[kFixWarps];
  FixWarpSmem& S = smem_all[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const unsigned below = (1u << lane) - 1u;
  long long n = (long long)*n_dev;
  if (n > cap) n = cap;  // a short speculative pool is rebuilt by the caller anyway
  unsigned fixed = 0;
  const long long nwarps = (long long)gridDim.x * kFixWarps;
  for (long long t0 = ((long long)blockIdx.x * kFixWarps + (threadIdx.x >> 5)) * kFixWarpTile; t0 < n;
       t0 += nwarps * kFixWarpTile) {
    const int len = (int)min((long long)kFixWarpRegion, n - t0);  // valid elements of the region
    const bool at_end = t0 + kFixWarpRegion >= n;
    uint32_t r[kFixChunks], fl[kFixChunks];
#pragma unroll
    for (int k = 0; k < kFixChunks; ++k) {
      const int i = 32 * k + (int)lane;
      r[k] = i < len ? pl.rank[t0 + i] : kSegBit;  // past the end: sentinel starts
      fl[k] = __ballot_sync(0xffffffffu, (r[k] & kSegBit) != 0u);
      S.rk[i] = r[k] & ~kSegBit;
      S.dis[i] = 0;
      S.dst_set[i] = 0;
    }
    // last start before chunk k / first start after chunk k (warp-uniform)
    int last_before[kFixChunks], first_after[kFixChunks];
    {
      int lb = -1;
#pragma unroll
      for (int k = 0; k < kFixChunks; ++k) {
        last_before[k] = lb;
        if (fl[k]) lb = 32 * k + 31 - __clz(fl[k]);
      }
      int fa = kFixWarpRegion;
#pragma unroll
      for (int k = kFixChunks - 1; k >= 0; --k) {
        first_after[k] = fa;
        if (fl[k]) fa = 32 * k + __ffs(fl[k]) - 1;
      }
    }
    int st[kFixChunks], en[kFixChunks];
    bool own[kFixChunks];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kFixChunks; ++k) {
      const int i = 32 * k + (int)lane;
      const unsigned upto = fl[k] & (below | (1u << lane));    // starts at or before me in this chunk
      const unsigned after = fl[k] & ~(below | (1u << lane));  // starts after me in this chunk
      st[k] = upto ? 32 * k + 31 - __clz(upto) : last_before[k];
      en[k] = after ? 32 * k + __ffs(after) - 1 : first_after[k];
      // previous element's rank (lane 31 of the previous chunk for lane 0)
      uint32_t prev = __shfl_up_sync(0xffffffffu, r[k], 1);
      if (k > 0) {
        const uint32_t carry = __shfl_sync(0xffffffffu, r[k > 0 ? k - 1 : 0], 31);
        if (lane == 0) prev = carry;
      }
      own[k] = false;
      if (i >= len || st[k] < 0 || st[k] >= kFixWarpTile) continue;
      if (!(en[k] < kFixWarpRegion || at_end)) {  // runs past the look-ahead: the long pass sorts it
        if (i == st[k]) {
          const unsigned long long q = atomicAdd(n_big, 1ull);
          if (q < big_cap)
            big_list[q] = (unsigned long long)(t0 + i);
          else
            raise_status(status, FHV_NOMEM);
        }
        continue;
      }
      own[k] = true;
      if (i > st[k] && (r[k] & ~kSegBit) < (prev & ~kSegBit)) S.dis[st[k]] = 1;
    }
    __syncwarp();
    // the elements of disordered segments, compacted (so the rank counting
    // below runs ~#moving / 32 rounds, not one per chunk), then ranked by
    // counting over their segment and staged at the destination
    int nmv = 0;
#pragma unroll
    for (int k = 0; k < kFixChunks; ++k) {
      const int i = 32 * k + (int)lane;
      const bool mv = own[k] && S.dis[st[k]];
      const unsigned bal = __ballot_sync(0xffffffffu, mv);
      if (mv) {
        const int q = nmv + __popc(bal & below);
        S.mv_i[q] = (uint8_t)i;
        S.mv_lo[q] = (uint8_t)st[k];
        S.mv_hi[q] = (uint8_t)min(en[k], len);
        if (i == st[k]) ++fixed;
      }
      nmv += __popc(bal);
    }
    __syncwarp();
    for (int b0 = 0; b0 < nmv; b0 += 32) {
      const int q = b0 + (int)lane;
      if (q >= nmv) continue;
      const int i = S.mv_i[q], lo = S.mv_lo[q], hi = S.mv_hi[q];
      const uint32_t rr = S.rk[i];
      // the record's loads issue before the counting loop (their latency
      // overlaps it)
      const long long s_ = t0 + i;
      const float p0 = pl.pos[3 * s_], p1 = pl.pos[3 * s_ + 1], p2 = pl.pos[3 * s_ + 2];
      const float n0 = pl.nrm[3 * s_], n1 = pl.nrm[3 * s_ + 1], n2 = pl.nrm[3 * s_ + 2];
      const uint32_t mt = pl.mat[s_], ob = pl.obj[s_];
      int d = lo;
      for (int j = lo; j < hi; ++j) d += S.rk[j] < rr ? 1 : 0;
      S.pos[d][0] = p0; S.pos[d][1] = p1; S.pos[d][2] = p2;
      S.nrm[d][0] = n0; S.nrm[d][1] = n1; S.nrm[d][2] = n2;
      S.mat[d] = mt;
      S.obj[d] = ob;
      S.rank[d] = rr;
      S.dst_set[d] = 1;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kFixChunks; ++k) {
      const int d = 32 * k + (int)lane;
      if (d >= len || !S.dst_set[d]) continue;
      const long long t = t0 + d;
      pl.pos[3 * t] = S.pos[d][0]; pl.pos[3 * t + 1] = S.pos[d][1]; pl.pos[3 * t + 2] = S.pos[d][2];
      pl.nrm[3 * t] = S.nrm[d][0]; pl.nrm[3 * t + 1] = S.nrm[d][1]; pl.nrm[3 * t + 2] = S.nrm[d][2];
      pl.mat[t] = S.mat[d];
      pl.obj[t] = S.obj[d];
      pl.rank[t] = S.rank[d] | (r[k] & kSegBit);  // the segment bit stays with the slot
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fixed += __shfl_xor_sync(0xffffffffu, fixed, o);
  if (lane == 0 && fixed) atomicAdd(n_fixed_total, (unsigned long long)fixed);
}

// long segments (did not end inside a tile's look-ahead): a CTA per segment
__global__ void __launch_bounds__(256) k_leaf_fix_big(PoolRefs pl, const unsigned long long* __restrict__ n_dev,
                                                       long long cap, const unsigned long long* __restrict__ big_list,
                                                       const unsigned long long* __restrict__ n_big,
                                                       unsigned long long big_cap,
                                                       unsigned long long* __restrict__ kscr,
                                                       uint32_t* __restrict__ rscr) {
  __shared__ unsigned long long sk[kSortSmem];
  __shared__ long long s_end;
  __shared__ int s_dis;
  long long n = (long long)*n_dev;
  if (n > cap) n = cap;
  const unsigned long long nl = *n_big < big_cap ? *n_big : big_cap;
  for (long long w = blockIdx.x; w < (long long)nl; w += gridDim.x) {
    const long long off = (long long)big_list[w];
    __syncthreads();
    if (threadIdx.x == 0) {
      s_end = n;
      s_dis = 0;
    }
    __syncthreads();
    // end: the next segment start after off (chunks of blockDim, first hit wins)
    for (long long base = off + 1; base < n; base += blockDim.x) {
      const long long i = base + threadIdx.x;
      if (i < n && (pl.rank[i] & kSegBit)) atomicMin(reinterpret_cast<unsigned long long*>(&s_end),
                                                      (unsigned long long)i);
      __syncthreads();
      if (s_end < n) break;
    }
    const long long cnt = s_end - off;
    for (long long i = off + 1 + threadIdx.x; i < off + cnt; i += blockDim.x)
      if ((pl.rank[i] & ~kSegBit) < (pl.rank[i - 1] & ~kSegBit)) s_dis = 1;
    __syncthreads();
    if (!s_dis) continue;
    if (cnt <= (long long)blockDim.x) {
      // short segment (the common big one, ~65-100 slots): an element's
      // destination = how many ranks of the segment are smaller (ranks are
      // distinct); records held in registers across one barrier, then
      // written in place
      uint32_t* rk = reinterpret_cast<uint32_t*>(sk);
      const long long i = threadIdx.x;
      uint32_t R[9];
      uint32_t mine = 0;
      if (i < cnt) {
        stage_record(pl, R, off + i);
        mine = R[8] & ~kSegBit;
        rk[i] = mine;
      }
      __syncthreads();
      if (i < cnt) {
        int dst = 0;
        for (int j = 0; j < (int)cnt; ++j) dst += rk[j] < mine ? 1 : 0;
        unstage_record(pl, R, off + dst, dst == 0 ? kSegBit : 0u);
      }
      __syncthreads();
      continue;
    }
    long long np2 = 1;
    while (np2 < cnt) np2 <<= 1;
    unsigned long long* K = np2 <= kSortSmem ? sk : kscr + 2 * off;
    for (long long i = threadIdx.x; i < np2; i += blockDim.x)
      K[i] = i < cnt ? ((unsigned long long)(pl.rank[off + i] & ~kSegBit) << 32) | (unsigned long long)i : ~0ull;
    for (long long i = threadIdx.x; i < cnt; i += blockDim.x) stage_record(pl, rscr + 9 * (off + i), off + i);
    __syncthreads();
    for (long long k = 2; k <= np2; k <<= 1)
      for (long long j = k >> 1; j > 0; j >>= 1) {
        for (long long i = threadIdx.x; i < np2; i += blockDim.x) {
          const long long l = i ^ j;
          if (l <= i) continue;
          const unsigned long long a = K[i], b = K[l];
          if ((a > b) == ((i & k) == 0)) {
            K[i] = b;
            K[l] = a;
          }
        }
        __syncthreads();
      }
    for (long long i = threadIdx.x; i < cnt; i += blockDim.x)
      unstage_record(pl, rscr + 9 * (off + (long long)(K[i] & 0xffffffffull)), off + i, i == 0 ? kSegBit : 0u);
    __syncthreads();
  }
}

// make_triangle face normals (fhv/scene.py:137-139)
__global__ void k_face_normals(long long n, const double* __restrict__ pos, double* __restrict__ fn) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const double* P = pos + 9 * t;
    double e1[3], e2[3];
    for (int k = 0; k < 3; ++k) {
      e1[k] = __dsub_rn(P[3 + k], P[k]);
      e2[k] = __dsub_rn(P[6 + k], P[k]);
    }
    const double c0 = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
    const double c1 = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
    const double c2 = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
    const double len = __dsqrt_rn(fwd3(c0, c1, c2, c0, c1, c2));
    const Recip rl = recip_of(len);
    fn[3 * t] = len > 0.0 ? div_rn(c0, rl) : 0.0;
    fn[3 * t + 1] = len > 0.0 ? div_rn(c1, rl) : 0.0;
    fn[3 * t + 2] = len > 0.0 ? div_rn(c2, rl) : 0.0;
  }
}

// unit rows (scene ingest): out = v / sqrt(v . v) with NumPy's ddot order
// (FWD) -- np.linalg.norm of a 3-vector and _unit (fhv/scene.py:73-77, 327-332);
// the first zero-length row index lands in *zero_first
__global__ void k_unit_rows(long long n, const double* __restrict__ in, double* __restrict__ out,
                            unsigned long long* zero_first) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double a = in[3 * i], b = in[3 * i + 1], c = in[3 * i + 2];
    const double len = __dsqrt_rn(fwd3(a, b, c, a, b, c));
    if (len == 0.0) {
      atomicMin(zero_first, (unsigned long long)i);
      out[3 * i] = out[3 * i + 1] = out[3 * i + 2] = 0.0;
      continue;
    }
    out[3 * i] = ddiv_z(a, len);
    out[3 * i + 1] = ddiv_z(b, len);
    out[3 * i + 2] = ddiv_z(c, len);
  }
}

// ---------------------------------------------------------------------------
// shard binning: keep a triangle iff its f64 AABB,
// grown by the margin, meets one of the shard's boxes.  Fragments are convex
// combinations of the vertices rounded to f32, so every fragment a triangle
// can emit into the shard's leaves passes this test.

__global__ void k_bin_tris(const double* __restrict__ pos, long long n, const double* __restrict__ boxes, int n_boxes,
                           double margin, uint32_t* __restrict__ flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const double* P = pos + 9 * t;
    double mn[3], mx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double v0 = __ldg(&P[a]), v1 = __ldg(&P[3 + a]), v2 = __ldg(&P[6 + a]);
      mn[a] = fmin(v0, fmin(v1, v2)) - margin;
      mx[a] = fmax(v0, fmax(v1, v2)) + margin;
    }
    uint32_t keep = 0;
    for (int b = 0; b < n_boxes && !keep; ++b) {
      const double* B = boxes + 6 * b;
      keep = (mn[0] <= B[3] && mx[0] >= B[0] && mn[1] <= B[4] && mx[1] >= B[1] && mn[2] <= B[5] && mx[2] >= B[2]) ? 1u
                                                                                                                 : 0u;
    }
    flag[t] = keep;
  }
}

__global__ void k_compact_tris(const uint32_t* __restrict__ flag, const unsigned long long* __restrict__ off,
                               long long n, uint32_t* __restrict__ idx) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    if (flag[t]) idx[off[t]] = (uint32_t)t;
}

// rebuild_pofl_as_pofa (fhv/storage.py:624-652): leaf histogram of the f32
// record positions (cell_code), then a scatter into the leaf ranges with the
// source index parked in prev_index for k_leaf_order (stable: pool order =
// emission order inside a leaf)
__global__ void k_pool_leaf_hist(const float* __restrict__ pos, long long n, int levels, uint32_t* __restrict__ counts,
                                 int* status) {
  for (long long i0 = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31u); i0 < n;
       i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + lane_id();
    uint64_t code = ~0ull;
    if (i < n && !cell_code(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], levels, &code)) {
      raise_status(status, FHV_RANGE);
      code = ~0ull;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, code);
    if (code != ~0ull && (int)lane_id() == __ffs(grp) - 1) atomicAdd(&counts[code], (uint32_t)__popc(grp));
  }
}

__global__ void k_pool_leaf_scatter(const float* __restrict__ spos, const float* __restrict__ snrm,
                                    const uint32_t* __restrict__ smat, const uint32_t* __restrict__ sobj, long long n,
                                    int levels, const uint32_t* __restrict__ offsets, uint32_t* __restrict__ cursors,
                                    float* __restrict__ dpos, float* __restrict__ dnrm, uint32_t* __restrict__ dmat,
                                    uint32_t* __restrict__ dobj, int32_t* __restrict__ dprev) {
  for (long long i0 = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31u); i0 < n;
       i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + lane_id();
    uint64_t code = ~0ull;
    if (i < n && !cell_code(spos[3 * i], spos[3 * i + 1], spos[3 * i + 2], levels, &code)) code = ~0ull;
    const unsigned grp = __match_any_sync(0xffffffffu, code);
    const int leader = __ffs(grp) - 1;
    uint32_t base = 0;
    if (code != ~0ull && (int)lane_id() == leader) base = atomicAdd(&cursors[code], (uint32_t)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (code == ~0ull) continue;
    const long long d = (long long)offsets[code] + base + __popc(grp & ((1u << lane_id()) - 1u));
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      dpos[3 * d + e] = spos[3 * i + e];
      dnrm[3 * d + e] = snrm[3 * i + e];
    }
    dmat[d] = smat[i];
    dobj[d] = sobj[i];
    dprev[d] = (int32_t)i;
  }
}

// FHV1 snapshot records (fhv/storage.py:57-66, 725-808): SoA pool <-> packed
// little-endian 36-byte RECORD_DTYPE rows (pos f32x3, nrm f32x3, material
// u32, object u32, prev i32), one 4-byte word per thread
__global__ void k_pack_records(const float* __restrict__ pos, const float* __restrict__ nrm,
                               const uint32_t* __restrict__ mat, const uint32_t* __restrict__ obj,
                               const int32_t* __restrict__ prev, long long n, uint32_t* __restrict__ out) {
  const long long words = 9 * n;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < words;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / 9;
    const int f = (int)(w - 9 * r);
    uint32_t v;
    if (f < 3) v = __float_as_uint(pos[3 * r + f]);
    else if (f < 6) v = __float_as_uint(nrm[3 * r + f - 3]);
    else if (f == 6) v = mat[r];
    else if (f == 7) v = obj[r];
    else v = (uint32_t)prev[r];
    out[w] = v;
  }
}

__global__ void k_unpack_records(const uint32_t* __restrict__ in, long long n, float* __restrict__ pos,
                                 float* __restrict__ nrm, uint32_t* __restrict__ mat, uint32_t* __restrict__ obj,
                                 int32_t* __restrict__ prev) {
  const long long words = 9 * n;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < words;
       w += (long long)gridDim.x * blockDim.x) {
    const long long r = w / 9;
    const int f = (int)(w - 9 * r);
    const uint32_t v = in[w];
    if (f < 3) pos[3 * r + f] = __uint_as_float(v);
    else if (f < 6) nrm[3 * r + f - 3] = __uint_as_float(v);
    else if (f == 6) mat[r] = v;
    else if (f == 7) obj[r] = v;
    else prev[r] = (int32_t)v;
  }
}

// deferred pass: flag the jobs whose batch holds exactly one fragment
__global__ void k_job_n1(long long n_jobs, const uint32_t* __restrict__ job_items,
                         const unsigned long long* __restrict__ job_item_off, const uint32_t* __restrict__ item_cnt,
                         JobPersp* __restrict__ persp) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n_jobs;
       j += (long long)gridDim.x * blockDim.x) {
    const unsigned long long b = job_item_off[j];
    unsigned long long n = 0;
    for (uint32_t k = 0; k < job_items[j] && n < 2; ++k) n += item_cnt[b + k];
    persp[j].n1 = n == 1 ? 1u : 0u;
  }
}

// ---------------------------------------------------------------------------
// host orchestration

namespace {

inline int grid_for(long long n, int block, int per_sm = 16) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148LL * per_sm) g = 148LL * per_sm;
  return (int)g;
}

CaptureParams make_params(const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg) {
  CaptureParams p;
  p.strategy = cfg->strategy;
  p.res = cfg->res;
  p.width = cfg->res;
  p.height = cfg->res;
  p.ortho = 1;
  p.persp = nullptr;
  p.pitch = cfg->pitch;
  std::memcpy(p.proj, cfg->proj, sizeof(p.proj));
  p.n_tri = tris->n_tri;
  p.n_jobs = (cfg->strategy == 1 || cfg->strategy == 2) ? 3 * tris->n_tri : tris->n_tri;
  p.pos = tris->pos;
  p.vnrm = tris->vnrm;
  p.fnrm = tris->fnrm;
  p.mat = tris->mat;
  p.obj = tris->obj;
  p.tri_index = nullptr;
  p.cell_lo = 0;
  p.cell_hi = ~0ull;
  return p;
}

int validate(const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg) {
  if (!tris || !cfg || tris->n_tri < 0 || cfg->strategy < 0 || cfg->strategy > 3 || cfg->res < 1) return FHV_BAD_ARGS;
  if (cfg->strategy == 3 && !(cfg->pitch > 0.0)) return FHV_BAD_ARGS;
  if (tris->n_tri > 0 && (!tris->pos || !tris->vnrm || !tris->fnrm || !tris->mat || !tris->obj)) return FHV_BAD_ARGS;
  if (3 * tris->n_tri >= (1LL << 32)) return FHV_BAD_ARGS;
  return FHV_OK;
}

// FHV_FUSED_EXPAND=0: the speculative plan's separate scan + item expansion (A/B)
inline bool fused_expand_enabled() {
  static const int v = [] {
    const char* e = std::getenv("FHV_FUSED_EXPAND");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return v != 0;
}

// job setup + work-item expansion.  The number of work items is data
// dependent.  Exact path: sync once, size the item buffers.  Speculative path
// (allow_spec, same job count as the last exact plan on this ctx): launch on
// the grow-only buffers of that plan without waiting -- the job scan and the
// item expansion as one pass (k_item_scan_expand); every item kernel reads
// the true count from ctl->items_total, the expansion raises FHV_RETRY_ITEMS
// if it does not fit, and the caller's final sync re-plans exactly.
int plan(fhv_ctx* ctx, const CaptureParams& p, cudaStream_t s, bool allow_spec = false) {
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  ctx->n_jobs = p.n_jobs;
  ctx->n_items = 0;
  ctx->spec = false;
  if (p.n_jobs == 0) return FHV_OK;
  JobSetup* jobs = (JobSetup*)scratch(ctx, kJobs, (size_t)p.n_jobs * sizeof(JobSetup));
  uint32_t* job_items = (uint32_t*)scratch(ctx, kJobItems, (size_t)p.n_jobs * 4);
  auto* job_item_off = (unsigned long long*)scratch(ctx, kJobItemOff, (size_t)p.n_jobs * 8);
  if (!jobs || !job_items || !job_item_off) return FHV_NOMEM;
  const bool spec = allow_spec && ctx->last_n_jobs == p.n_jobs && ctx->item_cap > 0;
  const bool fused = spec && fused_expand_enabled();
  // the fused plan's tile totals, summed by the job setup (no look-back chain in the expansion)
  uint32_t* tsum = nullptr;
  if (fused) {
    const size_t nt = (size_t)((p.n_jobs + kExpandTileJobs - 1) / kExpandTileJobs);
    tsum = (uint32_t*)scratch(ctx, kJobTileSums, nt * 4);
    if (!tsum) return FHV_NOMEM;
    if ((rc = check_cuda(ctx, cudaMemsetAsync(tsum, 0, nt * 4, s)))) return rc;
  }
  {
    LaunchScope L_(ctx, kStJobSetup, s);
    k_job_setup<<<grid_for(p.n_jobs, 128), 128, 0, s>>>(p, jobs, job_items, &ctx->ctl->status, tsum);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  if (fused) {  // item buffers sized by the last exact plan: scan + expand in one pass
    const long long n_items = ctx->item_cap;
    uint32_t* item_job = (uint32_t*)scratch(ctx, kItemJob, (size_t)n_items * 4);
    uint32_t* item_p0 = (uint32_t*)scratch(ctx, kItemP0, (size_t)n_items * 4);
    if (!item_job || !item_p0) return FHV_NOMEM;
    ctx->n_items = n_items;
    ctx->spec = true;
    return scan_expand_items(ctx, job_items, job_item_off, p.n_jobs, item_job, item_p0, (unsigned long long)n_items,
                             kItemPix, s, tsum);
  }
  if ((rc = scan_u32_to_u64(ctx, job_items, job_item_off, p.n_jobs, s))) return rc;
  if ((rc = check_cuda(ctx, cudaMemcpyAsync(&ctx->ctl->items_total, &ctx->ctl->scan_total, sizeof(unsigned long long),
                                            cudaMemcpyDeviceToDevice, s))))
    return rc;
  long long n_items;
  if (spec) {
    n_items = ctx->item_cap;
  } else {
    if ((rc = sync_control(ctx, s))) return rc;
    n_items = (long long)ctx->ctl_host->scan_total;
    ctx->last_n_jobs = p.n_jobs;
    if (n_items > ctx->item_cap) ctx->item_cap = n_items;
  }
  if (n_items == 0) return FHV_OK;
  if (n_items >= (1LL << 31)) return FHV_NOMEM;
  uint32_t* item_job = (uint32_t*)scratch(ctx, kItemJob, (size_t)n_items * 4);
  uint32_t* item_p0 = (uint32_t*)scratch(ctx, kItemP0, (size_t)n_items * 4);
  if (!item_job || !item_p0) return FHV_NOMEM;
  ctx->n_items = n_items;
  ctx->spec = spec;
  {
    LaunchScope L_(ctx, kStItemExpand, s);
    k_item_expand<<<grid_for(p.n_jobs, 256), 256, 0, s>>>(p.n_jobs, job_items, job_item_off, item_job, item_p0,
                                                          (unsigned long long)n_items, &ctx->ctl->status);
  }
  return check_cuda(ctx, cudaGetLastError());
}

// device-side item count of a speculative plan (nullptr: ctx->n_items is exact)
inline const unsigned long long* items_dev(fhv_ctx* ctx) { return ctx->spec ? &ctx->ctl->items_total : nullptr; }

// dynamic shared memory of the fast raster kernels (opt-in above 48 KB total)
constexpr int kRasterDyn = kRasterWarps * 32 * (int)sizeof(PosPlanes);
constexpr int kEmitFastDyn = kEmitFastWarps * 32 * (int)sizeof(ItemFast);
template <class K>
void smem_opt_in(K kernel, int bytes) {
  static const void* seen[16] = {};  // kernels already opted in (per process)
  static int n_seen = 0;
  const void* f = reinterpret_cast<const void*>(kernel);
  for (int i = 0; i < n_seen; ++i)
    if (seen[i] == f) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (n_seen < 16) seen[n_seen++] = f;
}

// Which per-fragment arithmetic the raster passes use.  The certified plane
// path (k_emit_fast, k_raster<.., kFast>) builds per-item planes (~300
// instructions per item) to cut the per-fragment work: it wins when items
// carry many fragments (C4: PPFL emission 1.88 -> 1.41 ms) and loses on tiny
// triangles (C3, ~4.6 fragments per item: 187 -> 208 us).  The choice follows
// the fragments-per-item of the last synchronised capture on this context
// (speculation like the pool-size guess; graph captures replay the choice made
// at capture time).  FHV_FAST_MATH=0/1 forces it; FHV_FAST_MIN_FPI sets the
// threshold (default 16 fragments per item).
inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
inline bool use_fast_math(const fhv_ctx* ctx) {
  static const int force = env_int("FHV_FAST_MATH", -1);
  static const int min_fpi = env_int("FHV_FAST_MIN_FPI", 16);
  if (force >= 0) return force != 0;
  return ctx->frags_per_item >= (double)min_fpi;
}

// counts per item (+ leaf histogram) and their scan (fragment ranks); async
int count(fhv_ctx* ctx, const CaptureParams& p, bool leaves, int levels, uint32_t* leaf_counts, cudaStream_t s,
          bool ranks = true, uint32_t* tile_sums = nullptr, bool defer_ranks = false) {
  ctx->item_scan_n = -1;
  const long long n = ctx->n_items;
  uint32_t* item_cnt = (uint32_t*)scratch(ctx, kItemCnt, (size_t)(n > 0 ? n : 1) * 4);
  auto* item_off = (unsigned long long*)scratch(ctx, kItemOff, (size_t)(n > 0 ? n : 1) * 8);
  auto* item_mask = (uint4*)scratch(ctx, kItemMask, (size_t)(n > 0 ? n : 1) * 16);
  if (!item_cnt || !item_off || !item_mask) return FHV_NOMEM;
  const unsigned long long* nd = items_dev(ctx);
  if (n > 0) {
    const JobSetup* jobs = (const JobSetup*)ctx->bufs[kJobs].ptr;
    const uint32_t* ij = (const uint32_t*)ctx->bufs[kItemJob].ptr;
    const uint32_t* ip = (const uint32_t*)ctx->bufs[kItemP0].ptr;
    EmitOut o;
    std::memset(&o, 0, sizeof(o));
    o.levels = levels;
    o.leaf_counts = leaf_counts;
    o.tile_sums = tile_sums;
    const int grid = grid_for((n + 31) / 32 * 32, kRasterBlock, FHV_RASTER_PER_SM);
    const bool fast = leaves && use_fast_math(ctx);
    if (fast) smem_opt_in(k_raster<kCntLeaves, false, true>, kRasterDyn);
    {
      LaunchScope L_(ctx, leaves ? kStCountLeaves : kStCount, s);
      if (fast)
        k_raster<kCntLeaves, false, true><<<grid, kRasterBlock, kRasterDyn, s>>>(p, jobs, ij, ip, nullptr, n, nd,
                                                                                  item_cnt, item_mask, o, ctx->ctl);
      else if (leaves)
        k_raster<kCntLeaves, false><<<grid, kRasterBlock, 0, s>>>(p, jobs, ij, ip, nullptr, n, nd, item_cnt,
                                                                   item_mask,
                                                                   o, ctx->ctl);
      else
        k_raster<kCnt, false><<<grid, kRasterBlock, 0, s>>>(p, jobs, ij, ip, nullptr, n, nd, item_cnt, item_mask, o,
                                                             ctx->ctl);
    }
    int rc = check_cuda(ctx, cudaGetLastError());
    if (rc) return rc;
  }
  // item fragment offsets = emission ranks; a POFA build that keeps no
  // emission order (atomic in-leaf order) needs neither them nor their total
  if (!ranks) return FHV_OK;
  if (defer_ranks) {  // the directory launch scans them (scan_leaves_and_pyramid)
    ctx->item_scan_n = n;
    ctx->item_scan_dev = nd;
    return FHV_OK;
  }
  return scan_u32_to_u64(ctx, item_cnt, item_off, n, s, nd);
}

template <int kMode>
int emit(fhv_ctx* ctx, const CaptureParams& p, const EmitOut& o, bool atomic_alloc, cudaStream_t s) {
  const long long n = ctx->n_items;
  if (n == 0) return FHV_OK;
  const JobSetup* jobs = (const JobSetup*)ctx->bufs[kJobs].ptr;
  const uint32_t* ij = (const uint32_t*)ctx->bufs[kItemJob].ptr;
  const uint32_t* ip = (const uint32_t*)ctx->bufs[kItemP0].ptr;
  const auto* io = (const unsigned long long*)ctx->bufs[kItemOff].ptr;
  const auto* im = (const uint4*)ctx->bufs[kItemMask].ptr;
  const unsigned long long* nd = items_dev(ctx);
  if (int rc = run_deferred_item_scan(ctx, s)) return rc;  // (normally already fused into the directory)
  if constexpr (kMode == kPpfl || kMode == kPofl || kMode == kPofa) {
    if (!(o.flags & kExactMath) && use_fast_math(ctx)) {
      const int gridf = grid_for((n + 31) / 32 * 32, 32 * kEmitFastWarps);
      smem_opt_in(k_emit_fast<kMode, true>, kEmitFastDyn);
      smem_opt_in(k_emit_fast<kMode, false>, kEmitFastDyn);
      LaunchScope L_(ctx, kStEmitList + (kMode - kList), s);
      if (atomic_alloc)
        k_emit_fast<kMode, true><<<gridf, 32 * kEmitFastWarps, kEmitFastDyn, s>>>(p, jobs, ij, ip, io, im, n, nd, o,
                                                                                ctx->ctl);
      else
        k_emit_fast<kMode, false><<<gridf, 32 * kEmitFastWarps, kEmitFastDyn, s>>>(p, jobs, ij, ip, io, im, n, nd, o,
                                                                                 ctx->ctl);
      return check_cuda(ctx, cudaGetLastError());
    }
  }
  const int grid = grid_for((n + 31) / 32 * 32, kRasterBlock, FHV_RASTER_PER_SM);
  {
    LaunchScope L_(ctx, kMode >= kDsDepth ? kStDeferred : kStEmitList + (kMode - kList), s);
    if (atomic_alloc)
      k_emit<kMode, true><<<grid, kRasterBlock, 0, s>>>(p, jobs, ij, ip, io, im, n, nd, o, ctx->ctl);
    else
      k_emit<kMode, false><<<grid, kRasterBlock, 0, s>>>(p, jobs, ij, ip, io, im, n, nd, o, ctx->ctl);
  }
  return check_cuda(ctx, cudaGetLastError());
}

EmitOut empty_out() {
  EmitOut o;
  std::memset(&o, 0, sizeof(o));
  return o;
}

void set_pool(EmitOut& o, const fhv_pool_t* pool) {
  o.capacity = pool->capacity;
  o.pos = pool->pos;
  o.nrm = pool->nrm;
  o.mat = pool->mat;
  o.obj = pool->obj;
  o.prev = pool->prev;
}

int chain_order(fhv_ctx* ctx, int32_t* heads, int32_t* prev, long long n_keys, long long capacity, cudaStream_t s) {
  int32_t* spill = (int32_t*)scratch(ctx, kChainScratch, (size_t)(capacity > 0 ? capacity : 1) * 4);
  if (!spill) return FHV_NOMEM;
  int rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->spare[0], 0, 8, s));
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStChainOrder, s);
    k_chain_order<<<grid_for(n_keys, 128), 128, 0, s>>>(heads, prev, n_keys, spill, &ctx->ctl->spare[0]);
  }
  return check_cuda(ctx, cudaGetLastError());
}

}  // namespace

}  // namespace fhv

using namespace fhv;

namespace fhv {
namespace {
// capture_pass + ListSink (fhv/raster.py:309-388) in emission order; with
// `depth`, FragmentBatch.depth too (needs the per-job ndc z, kept in p.persp)
int list_capture(fhv_ctx* ctx, CaptureParams& p, int64_t max_out, int64_t* job, int32_t* px, int32_t* py,
                 double* wpos, double* wnrm, double* depth, int64_t* n_out, cudaStream_t s) {
  int rc;
  if ((depth && p.strategy != 3) || p.strategy == kScreen) {
    p.persp = (JobPersp*)scratch(ctx, kJobPersp, (size_t)(p.n_jobs > 0 ? p.n_jobs : 1) * sizeof(JobPersp));
    if (!p.persp) return FHV_NOMEM;
  }
  if ((rc = plan(ctx, p, s))) return rc;
  if ((rc = count(ctx, p, false, 0, nullptr, s))) return rc;
  if (p.persp && ctx->n_items > 0) {
    {
      LaunchScope L_(ctx, kStEmitList, s);
      k_job_n1<<<grid_for(p.n_jobs, 256), 256, 0, s>>>(p.n_jobs, (const uint32_t*)ctx->bufs[kJobItems].ptr,
                                                       (const unsigned long long*)ctx->bufs[kJobItemOff].ptr,
                                                       (const uint32_t*)ctx->bufs[kItemCnt].ptr, p.persp);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  }
  EmitOut o = empty_out();
  o.max_out = max_out;
  o.job = (long long*)job;
  o.px = px;
  o.py = py;
  o.wpos = wpos;
  o.wnrm = wnrm;
  o.depth = depth;
  if (max_out > 0 && (rc = emit<kList>(ctx, p, o, false, s))) return rc;
  rc = sync_control(ctx, s);
  if (n_out) *n_out = (int64_t)ctx->ctl_host->scan_total;
  return rc;
}
}  // namespace
}  // namespace fhv

extern "C" int fhv_capture_list(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int64_t max_out,
                                int64_t* job, int32_t* px, int32_t* py, double* wpos, double* wnrm, int64_t* n_out,
                                void* stream) {
  return fhv_capture_list_depth(ctx, tris, cfg, max_out, job, px, py, wpos, wnrm, nullptr, n_out, stream);
}

extern "C" int fhv_capture_list_depth(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg,
                                      int64_t max_out, int64_t* job, int32_t* px, int32_t* py, double* wpos,
                                      double* wnrm, double* depth, int64_t* n_out, void* stream) {
  if (!ctx) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  CaptureParams p = make_params(tris, cfg);
  return list_capture(ctx, p, max_out, job, px, py, wpos, wnrm, depth, n_out, (cudaStream_t)stream);
}

// _raster_screen (fhv/raster.py:184-209) of every triangle through one
// arbitrary 4x4 projection into a width x height raster: the fragments of
// rasterize_triangle, in (triangle, y, x) order, with depth; a perspective
// triangle with any clip w <= 1e-9 emits nothing
extern "C" int fhv_raster_screen(fhv_ctx* ctx, const fhv_tris_t* tris, const double* proj, int32_t width,
                                 int32_t height, int64_t max_out, int64_t* job, int32_t* px, int32_t* py, double* wpos,
                                 double* wnrm, double* depth, int64_t* n_out, void* stream) {
  if (!ctx || !tris || !proj || width < 1 || height < 1) return FHV_BAD_ARGS;
  if (tris->n_tri < 0 || (tris->n_tri > 0 && (!tris->pos || !tris->vnrm || !tris->fnrm || !tris->mat || !tris->obj)))
    return FHV_BAD_ARGS;
  if (tris->n_tri >= (1LL << 32) - 1) return FHV_BAD_ARGS;
  CaptureParams p;
  std::memset(&p, 0, sizeof(p));
  p.strategy = kScreen;
  p.res = height;
  p.width = width;
  p.height = height;
  p.ortho = proj[12] == 0.0 && proj[13] == 0.0 && proj[14] == 0.0 && proj[15] == 1.0;
  std::memcpy(p.proj[0], proj, 16 * sizeof(double));
  p.n_tri = tris->n_tri;
  p.n_jobs = tris->n_tri;
  p.pos = tris->pos;
  p.vnrm = tris->vnrm;
  p.fnrm = tris->fnrm;
  p.mat = tris->mat;
  p.obj = tris->obj;
  p.cell_hi = ~0ull;
  return list_capture(ctx, p, max_out, job, px, py, wpos, wnrm, depth, n_out, (cudaStream_t)stream);
}

static int build_linked(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, bool pofl, int64_t width,
                        int32_t levels, fhv_pool_t* pool, int32_t* heads, uint8_t* pyramid, int32_t flags,
                        int64_t* next_free, void* stream) {
  if (!ctx || !pool || !heads) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  if (pool->capacity < 0 || pool->capacity >= (1LL << 31)) return FHV_BAD_ARGS;  // prev_index is int32
  if (pofl && (levels < 1 || levels > kMaxLevels || !pyramid)) return FHV_BAD_ARGS;
  if (!pofl && width < 1) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const CaptureParams p = make_params(tris, cfg);
  const bool atomic_alloc = (flags & FHV_ALLOC_ATOMIC) != 0;
  const long long n_keys = pofl ? 1LL << (3 * levels) : (long long)width * (long long)cfg->res;  // width x res
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (attempt > 0) {  // the speculative pass ran on too small item buffers: restore the -1 prefills
      if ((rc = check_cuda(ctx, cudaMemsetAsync(heads, 0xff, (size_t)n_keys * 4, s)))) return rc;
      if (pool->capacity > 0 &&
          (rc = check_cuda(ctx, cudaMemsetAsync(pool->prev, 0xff, (size_t)pool->capacity * 4, s))))
        return rc;
    }
    if ((rc = plan(ctx, p, s, attempt == 0))) return rc;
    // the counting pass also leaves the coverage masks the emission pass enumerates
    if ((rc = count(ctx, p, false, 0, nullptr, s))) return rc;
    EmitOut o = empty_out();
    set_pool(o, pool);
    o.heads = heads;
    o.flags = flags;
    if (pofl)
      o.levels = levels;
    else
      o.width = width;
    o.n_keys = n_keys;
    rc = pofl ? emit<kPofl>(ctx, p, o, atomic_alloc, s) : emit<kPpfl>(ctx, p, o, atomic_alloc, s);
    if (rc) return rc;
    if (flags & FHV_EXACT_ORDER) {
      if ((rc = chain_order(ctx, heads, pool->prev, n_keys, pool->capacity, s))) return rc;
    }
    if (pofl && (rc = pyramid_from_heads(ctx, heads, pyramid, levels, s))) return rc;
    rc = sync_control(ctx, s);
    if (rc != FHV_RETRY_ITEMS) break;
  }
  const long long total = (long long)(atomic_alloc ? ctx->ctl_host->alloc : ctx->ctl_host->scan_total);
  if (ctx->ctl_host->items_total > 0) ctx->frags_per_item = (double)total / (double)ctx->ctl_host->items_total;
  if (next_free) *next_free = total;
  if (rc == FHV_OK && total > pool->capacity) rc = FHV_OVERFLOW;
  return rc;
}

extern "C" int fhv_build_ppfl(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int64_t width,
                              fhv_pool_t* pool, int32_t* heads, int32_t flags, int64_t* next_free, void* stream) {
  if (cfg && cfg->strategy != 0) return FHV_BAD_ARGS;  // PPFL requires the single-view strategy
  return build_linked(ctx, tris, cfg, false, width, 0, pool, heads, nullptr, flags, next_free, stream);
}

extern "C" int fhv_build_pofl(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                              fhv_pool_t* pool, int32_t* heads, uint8_t* pyramid, int32_t flags, int64_t* next_free,
                              void* stream) {
  return build_linked(ctx, tris, cfg, true, 0, levels, pool, heads, pyramid, flags, next_free, stream);
}

namespace {

bool shard_ok(const fhv_shard_t* sh, int levels) {
  const unsigned long long n_leaves = 1ull << (3 * levels);
  if (!sh) return true;
  if (sh->cell_lo == 0 && sh->cell_hi == n_leaves && sh->n_boxes == 0) return true;
  const unsigned long long tl = (unsigned long long)dir_tile_leaves(levels);
  return tl > 0 && sh->cell_lo < sh->cell_hi && sh->cell_hi <= n_leaves && sh->cell_lo % tl == 0 &&
         sh->cell_hi % tl == 0 && sh->n_boxes >= 0 && sh->n_boxes <= FHV_SHARD_MAX_BOXES && sh->margin >= 0.0;
}

// FNV-1a over the shard description (range, margin, boxes)
uint64_t shard_sig(const fhv_shard_t* sh) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* d, size_t n) {
    const unsigned char* b = (const unsigned char*)d;
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  mix(&sh->cell_lo, 8);
  mix(&sh->cell_hi, 8);
  mix(&sh->n_boxes, 4);
  mix(&sh->margin, 8);
  mix(sh->boxes, (size_t)sh->n_boxes * 6 * sizeof(double));
  return h;
}

// params for one shard: binned triangle list (computed once by the count call
// and kept in ctx for the scatter call) and the owned leaf range.  reuse_bin:
// keep the ctx's binning (no kernels, no sync) when it was made for the same
// triangle arrays and shard -- the caller's promise that their contents did
// not change (the speculative sharded build)
int shard_params(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int levels,
                 const fhv_shard_t* sh, bool do_bin, CaptureParams& p, cudaStream_t s, bool reuse_bin = false) {
  p = make_params(tris, cfg);
  const unsigned long long n_leaves = 1ull << (3 * levels);
  p.cell_lo = sh ? sh->cell_lo : 0ull;
  p.cell_hi = sh ? sh->cell_hi : n_leaves;
  if (!sh || sh->n_boxes == 0) {
    if (do_bin) ctx->n_binned = -1;
    return FHV_OK;
  }
  const long long T = tris->n_tri;
  if (do_bin && reuse_bin && ctx->n_binned >= 0 && ctx->bin_pos == (const void*)tris->pos && ctx->bin_n_tri == T &&
      ctx->bin_sig == shard_sig(sh))
    do_bin = false;
  if (do_bin) {
    ctx->bin_pos = tris->pos;
    ctx->bin_n_tri = T;
    ctx->bin_sig = shard_sig(sh);
    ctx->n_binned = 0;
    if (T > 0) {
      auto* flag = (uint32_t*)scratch(ctx, kTriFlag, (size_t)T * 4);
      auto* off = (unsigned long long*)scratch(ctx, kTriOff, (size_t)T * 8);
      auto* idx = (uint32_t*)scratch(ctx, kTriIndex, (size_t)T * 4);
      auto* boxes = (double*)scratch(ctx, kShardBoxes, sizeof(sh->boxes));
      if (!flag || !off || !idx || !boxes) return FHV_NOMEM;
      int rc = check_cuda(ctx, cudaMemcpyAsync(boxes, sh->boxes, (size_t)sh->n_boxes * 6 * sizeof(double),
                                               cudaMemcpyHostToDevice, s));
      if (rc) return rc;
      {
        LaunchScope L_(ctx, kStJobSetup, s);
        k_bin_tris<<<grid_for(T, 256), 256, 0, s>>>(tris->pos, T, boxes, sh->n_boxes, sh->margin, flag);
      }
      if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
      if ((rc = scan_u32_to_u64(ctx, flag, off, T, s))) return rc;
      {
        LaunchScope L_(ctx, kStJobSetup, s);
        k_compact_tris<<<grid_for(T, 256), 256, 0, s>>>(flag, off, T, idx);
      }
      if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
      if ((rc = sync_control(ctx, s))) return rc;
      ctx->n_binned = (int64_t)ctx->ctl_host->scan_total;
    }
  }
  if (ctx->n_binned < 0) return FHV_BAD_ARGS;
  p.tri_index = (const uint32_t*)ctx->bufs[kTriIndex].ptr;
  p.n_tri = ctx->n_binned;
  p.n_jobs = (cfg->strategy == 1 || cfg->strategy == 2) ? 3 * p.n_tri : p.n_tri;
  return FHV_OK;
}

}  // namespace

namespace {

// pass 1 up to the per-leaf histogram, no sync after the counting kernel: the
// item scan's total is parked in ctl->frags_total for the caller's next sync
int pofa_count_async(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                     const fhv_shard_t* shard, uint32_t* counts_local, cudaStream_t s, CaptureParams& p,
                     bool spec = false, bool ranks = true, bool reuse_bin = false, bool defer_ranks = false) {
  ctx->pass1_levels = -1;
  ctx->pass1_ranks = ranks;
  int rc;
  if ((rc = reset_control(ctx, s))) return rc;
  if ((rc = shard_params(ctx, tris, cfg, levels, shard, true, p, s, reuse_bin))) return rc;
  const unsigned long long n_local = p.cell_hi - p.cell_lo;
  if ((rc = plan(ctx, p, s, spec))) return rc;
  if (ctx->counts_zeroed != counts_local &&
      (rc = check_cuda(ctx, cudaMemsetAsync(counts_local, 0, (size_t)n_local * 4, s))))
    return rc;
  ctx->counts_zeroed = nullptr;
  // whole-directory builds also total the fragments per directory tile, so
  // the directory pass (scan_leaves_and_pyramid) needs no look-back chain
  uint32_t* tile_sums = nullptr;
  ctx->dir_sums_levels = -1;
  if (p.cell_lo == 0 && n_local == (1ull << (3 * levels)) && levels >= 5) {
    const size_t nt = (size_t)(n_local >> kDirSumShift);
    tile_sums = (uint32_t*)scratch(ctx, kTileSums, nt * 4);
    if (!tile_sums) return FHV_NOMEM;
    if ((rc = check_cuda(ctx, cudaMemsetAsync(tile_sums, 0, nt * 4, s)))) return rc;
    ctx->dir_sums_levels = levels;
  }
  if ((rc = join_aux(ctx, s))) return rc;  // the side stream's clears (asynchronous build)
  if (ctx->fork_cursors_at_count) {  // the cursors cleared while the counting pass runs
    void* c = ctx->fork_cursors_at_count;
    ctx->fork_cursors_at_count = nullptr;
    if ((rc = fork_clear(ctx, c, (size_t)n_local * 4, s, nullptr))) return rc;
    ctx->cursors_zeroed = c;
  }
  // deferred ranks ride in the directory launch (whole-directory builds with tile totals)
  if ((rc = count(ctx, p, true, levels, counts_local, s, ranks, tile_sums, defer_ranks && tile_sums))) return rc;
  if (!ranks || ctx->item_scan_n >= 0) return FHV_OK;  // the total comes from the directory scan (caller)
  return check_cuda(ctx, cudaMemcpyAsync(&ctx->ctl->frags_total, &ctx->ctl->scan_total, sizeof(unsigned long long),
                                         cudaMemcpyDeviceToDevice, s));
}

int pofa_count_done(fhv_ctx* ctx, const fhv_tris_t* tris, int32_t levels, const CaptureParams& p) {
  const long long frags = (long long)ctx->ctl_host->frags_total;
  if (frags >= (1LL << 32)) return FHV_TOO_MANY;
  ctx->pass1_total = frags;
  if (ctx->ctl_host->items_total > 0) ctx->frags_per_item = (double)frags / (double)ctx->ctl_host->items_total;
  ctx->pass1_levels = levels;
  ctx->pass1_tris = tris->n_tri;
  ctx->pass1_lo = p.cell_lo;
  ctx->pass1_hi = p.cell_hi;
  return FHV_OK;
}

}  // namespace

extern "C" int fhv_pofa_shard_count(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg,
                                    int32_t levels, const fhv_shard_t* shard, uint32_t* counts_local,
                                    int64_t* local_total, void* stream) {
  if (!ctx || !counts_local || levels < 1 || levels > 10 || !shard_ok(shard, levels)) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CaptureParams p;
  if ((rc = pofa_count_async(ctx, tris, cfg, levels, shard, counts_local, s, p))) return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  if ((rc = pofa_count_done(ctx, tris, levels, p))) return rc;
  if (local_total) *local_total = ctx->pass1_total;
  return FHV_OK;
}

extern "C" int fhv_pofa_shard_directory(fhv_ctx* ctx, int32_t levels, const fhv_shard_t* shard,
                                        const uint32_t* counts_local, uint32_t* offsets_local, uint8_t* pyramid,
                                        uint64_t base, void* stream) {
  if (!ctx || !counts_local || !offsets_local || !pyramid || levels < 1 || levels > 10 || !shard_ok(shard, levels))
    return FHV_BAD_ARGS;
  const unsigned long long n_leaves = 1ull << (3 * levels);
  const unsigned long long lo = shard ? shard->cell_lo : 0ull, hi = shard ? shard->cell_hi : n_leaves;
  if (ctx->pass1_levels != levels || ctx->pass1_lo != lo || ctx->pass1_hi != hi) return FHV_BAD_ARGS;
  if (base + (uint64_t)ctx->pass1_total > 0xffffffffull) return FHV_TOO_MANY;
  cudaStream_t s = (cudaStream_t)stream;
  if (lo == 0 && hi == n_leaves && base == 0) return scan_leaves_and_pyramid(ctx, counts_local, offsets_local, pyramid,
                                                                            levels, s);
  return scan_leaf_range_and_pyramid(ctx, counts_local, offsets_local, pyramid, levels, lo, hi, base, s);
}

// pass 2 of a POFA build, enqueued only: cursors, scatter, EXACT_ORDER fix-up
// clear_status: the standalone scatter (fhv_pofa_scatter / shard scatter after
// an FHV_NEED_POOL build) drops the leftover FHV_NEED_POOL / retry code; the
// fused build keeps pass 1's status (job-setup errors such as FHV_BASIS must
// survive into the result, fhv/raster.py:147-163).  n_frags_dev: device-side
// fragment total (async build), else n_frags_host.
static int pofa_scatter_async(fhv_ctx* ctx, const CaptureParams& p, int32_t levels, unsigned long long lo,
                              unsigned long long hi, const uint32_t* counts_local, const uint32_t* offsets_local,
                              uint64_t base, fhv_pool_t* pool, int32_t flags, cudaStream_t s, bool clear_status,
                              const unsigned long long* n_frags_dev, long long n_frags_host) {
  const unsigned long long n_local = hi - lo;
  uint32_t* cursors = (uint32_t*)scratch(ctx, kCursors, (size_t)n_local * 4);
  if (!cursors) return FHV_NOMEM;
  int rc;
  if ((rc = join_aux(ctx, s))) return rc;
  if (ctx->cursors_zeroed != cursors && (rc = check_cuda(ctx, cudaMemsetAsync(cursors, 0, (size_t)n_local * 4, s))))
    return rc;
  ctx->cursors_zeroed = nullptr;
  if (!ctx->ctl_fresh && (rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->alloc, 0, 8, s)))) return rc;
  if (clear_status && (rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->status, 0, sizeof(int), s)))) return rc;
  EmitOut o = empty_out();
  set_pool(o, pool);
  o.levels = levels;
  o.offsets = offsets_local;
  o.counts = counts_local;
  o.cursors = cursors;
  o.base = base;
  // pools below 2^31 records park the rank with a segment-start bit for the
  // tile fix-up; bigger ones keep the per-leaf walk (k_leaf_order)
  const bool tile_fix = (flags & FHV_EXACT_ORDER) && pool->capacity > 0 && pool->capacity < (1LL << 31);
  o.flags = flags | (tile_fix ? kSegFlags : 0);
  if ((rc = emit<kPofa>(ctx, p, o, false, s))) return rc;
  if ((flags & FHV_EXACT_ORDER) && pool->capacity > 0 && !tile_fix) {
    LaunchScope L_(ctx, kStLeafOrder, s);
    k_leaf_order<<<grid_for((long long)n_local, 128, 32), 128, 0, s>>>(offsets_local, counts_local, (long long)n_local,
                                                                     base, (unsigned long long)pool->capacity,
                                                                     pool->pos, pool->nrm, pool->mat, pool->obj,
                                                                     pool->prev);
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  }
  if (tile_fix) {
    const long long cap = pool->capacity;
    const unsigned long long big_cap = (unsigned long long)(cap / kFixWarpTile + 1);
    auto* big = (unsigned long long*)scratch(ctx, kLeafList, (size_t)big_cap * 8);
    auto* keys = (unsigned long long*)scratch(ctx, kLeafKeys, (size_t)cap * 16);
    auto* recs = (uint32_t*)scratch(ctx, kLeafRecs, (size_t)cap * 36);
    auto* nn = (unsigned long long*)scratch(ctx, kTmp1, 8);
    if (!big || !keys || !recs || !nn) return FHV_NOMEM;
    if (!ctx->ctl_fresh && (rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->leaf_n[0], 0, 8, s)))) return rc;
    if (!ctx->ctl_fresh && (rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->leaf_n[2], 0, 8, s)))) return rc;
    if (!n_frags_dev) {
      const unsigned long long nh = (unsigned long long)n_frags_host;
      if ((rc = check_cuda(ctx, cudaMemcpyAsync(nn, &nh, 8, cudaMemcpyHostToDevice, s)))) return rc;
      if ((rc = check_cuda(ctx, cudaStreamSynchronize(s)))) return rc;  // nh lives on this stack frame
      n_frags_dev = nn;
    }
    PoolRefs pl{pool->pos, pool->nrm, pool->mat, pool->obj, reinterpret_cast<uint32_t*>(pool->prev)};
    {
      LaunchScope L_(ctx, kStLeafOrder, s);
      const long long tiles = (cap + kFixWarpTile - 1) / kFixWarpTile;  // one warp each
      const long long ctas = (tiles + kFixWarps - 1) / kFixWarps;
      k_leaf_fix<<<(int)(ctas < 148LL * FHV_FIX_PER_SM ? ctas : 148LL * FHV_FIX_PER_SM), 32 * kFixWarps, 0, s>>>(
          pl, n_frags_dev, cap, big, &ctx->ctl->leaf_n[2], big_cap, &ctx->ctl->leaf_n[0], &ctx->ctl->status);
    }
    {
      LaunchScope L_(ctx, kStLeafSort, s);
      k_leaf_fix_big<<<148, 256, 0, s>>>(pl, n_frags_dev, cap, big, &ctx->ctl->leaf_n[2], big_cap, keys, recs);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
    if ((rc = check_cuda(ctx, cudaMemsetAsync(pool->prev, 0xff, (size_t)cap * 4, s)))) return rc;
  }
  return FHV_OK;
}

static int fhv_pofa_shard_directory_nocheck(fhv_ctx* ctx, int32_t levels, const uint32_t* counts,
                                            uint32_t* offsets, uint8_t* pyramid, cudaStream_t s) {
  return scan_leaves_and_pyramid(ctx, counts, offsets, pyramid, levels, s);
}

extern "C" int fhv_pofa_shard_scatter(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg,
                                      int32_t levels, const fhv_shard_t* shard, const uint32_t* counts_local,
                                      const uint32_t* offsets_local, uint64_t base, fhv_pool_t* pool, int32_t flags,
                                      void* stream) {
  if (!ctx || !counts_local || !offsets_local || !pool || !shard_ok(shard, levels)) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  const unsigned long long n_leaves = 1ull << (3 * levels);
  const unsigned long long lo = shard ? shard->cell_lo : 0ull, hi = shard ? shard->cell_hi : n_leaves;
  if (ctx->pass1_levels != levels || ctx->pass1_tris != tris->n_tri || ctx->pass1_lo != lo || ctx->pass1_hi != hi)
    return FHV_BAD_ARGS;
  if (pool->capacity < ctx->pass1_total) return FHV_BAD_ARGS;
  if ((flags & FHV_EXACT_ORDER) && !ctx->pass1_ranks) return FHV_BAD_ARGS;  // pass 1 skipped the ranks
  cudaStream_t s = (cudaStream_t)stream;
  CaptureParams p;
  if ((rc = shard_params(ctx, tris, cfg, levels, shard, false, p, s))) return rc;
  if ((rc = pofa_scatter_async(ctx, p, levels, lo, hi, counts_local, offsets_local, base, pool, flags, s, true, nullptr,
                                ctx->pass1_total)))
    return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  // cursors <= counts elementwise (checked per insert) and equal totals
  // imply cursors == counts (fhv/storage.py:614-619)
  if ((long long)ctx->ctl_host->alloc != ctx->pass1_total) return FHV_PASS_MISMATCH;
  return FHV_OK;
}

extern "C" int fhv_pofa_count(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                              uint32_t* counts, uint32_t* offsets, uint8_t* pyramid, int64_t* total, void* stream) {
  if (!ctx || !counts || !offsets || !pyramid || levels < 1 || levels > 10) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CaptureParams p;
  // histogram and directory back to back; one sync reads both totals
  if ((rc = pofa_count_async(ctx, tris, cfg, levels, nullptr, counts, s, p))) return rc;
  if ((rc = fhv_pofa_shard_directory_nocheck(ctx, levels, counts, offsets, pyramid, s))) return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  if ((rc = pofa_count_done(ctx, tris, levels, p))) return rc;
  if ((long long)ctx->ctl_host->scan_total != ctx->pass1_total) return FHV_PASS_MISMATCH;
  if (total) *total = ctx->pass1_total;
  return FHV_OK;
}

extern "C" int fhv_pofa_build(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                              uint32_t* counts, uint32_t* offsets, uint8_t* pyramid, fhv_pool_t* pool, int32_t flags,
                              int64_t* total, void* stream) {
  if (!ctx || !counts || !offsets || !pyramid || levels < 1 || levels > 10) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  if (pool && (pool->capacity < 0 || (pool->capacity > 0 && (!pool->pos || !pool->nrm || !pool->mat || !pool->obj ||
                                                              !pool->prev))))
    return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned long long n_leaves = 1ull << (3 * levels);
  CaptureParams p;
  // pass 1, directory and (into the caller's pool, sized by its guess) pass 2
  // are enqueued back to back; the only wait is the final sync -- unless the
  // speculative item plan turns out too small, then once more with an exact plan
  const bool ranks = (flags & FHV_EXACT_ORDER) != 0;  // emission ranks only for the exact in-leaf order
  for (int attempt = 0; attempt < 2; ++attempt) {
    if ((rc = pofa_count_async(ctx, tris, cfg, levels, nullptr, counts, s, p, attempt == 0, ranks))) return rc;
    if ((rc = fhv_pofa_shard_directory_nocheck(ctx, levels, counts, offsets, pyramid, s))) return rc;
    if (!ranks &&
        (rc = check_cuda(ctx, cudaMemcpyAsync(&ctx->ctl->frags_total, &ctx->ctl->scan_total,
                                              sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s))))
      return rc;
    if (pool && pool->capacity > 0 &&
        (rc = pofa_scatter_async(ctx, p, levels, 0, n_leaves, counts, offsets, 0, pool, flags, s, false,
                                 &ctx->ctl->frags_total, 0)))
      return rc;
    rc = sync_control(ctx, s);
    if (rc != FHV_RETRY_ITEMS) break;
  }
  if (rc != FHV_OK && rc != FHV_NEED_POOL) return rc;
  int rc2 = pofa_count_done(ctx, tris, levels, p);
  if (rc2) return rc2;
  if ((long long)ctx->ctl_host->scan_total != ctx->pass1_total) return FHV_PASS_MISMATCH;
  if (total) *total = ctx->pass1_total;
  if (!pool || pool->capacity < ctx->pass1_total) return FHV_NEED_POOL;  // finish with fhv_pofa_scatter
  if (rc != FHV_OK) return rc;
  if ((long long)ctx->ctl_host->alloc != ctx->pass1_total) return FHV_PASS_MISMATCH;
  return FHV_OK;
}

namespace fhv {
namespace {
// the async build's outcome, staged in ctl->spare[4..7] for the D2H copy
// the build's ticket: in ctl->spare[4..7] and, when the caller's ticket is
// device-accessible (device memory, or pinned host memory through its
// mapping), stored there directly -- no stream-ordered copy, whose copy
// engine may be busy with the previous step's image read-back
__device__ __forceinline__ void put_ticket(Control* ctl, unsigned long long* out, unsigned long long st,
                                           unsigned long long a, unsigned long long b, unsigned long long c) {
  ctl->spare[4] = st;
  ctl->spare[5] = a;
  ctl->spare[6] = b;
  ctl->spare[7] = c;
  if (out) {
    out[0] = st;
    out[1] = a;
    out[2] = b;
    out[3] = c;
    __threadfence_system();
  }
}
__global__ void k_ticket(Control* ctl, unsigned long long* out) {
  put_ticket(ctl, out, (unsigned long long)(long long)ctl->status, ctl->frags_total, ctl->scan_total, ctl->alloc);
}
}  // namespace
// a device-accessible address of the caller's ticket (device / managed
// memory as is, pinned host memory through its mapping), else null (then a
// stream-ordered copy delivers it)
unsigned long long* ticket_device_view(fhv_ticket_t* t) {
  static const int on = env_int("FHV_TICKET_DIRECT", 1);
  if (!on) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, t) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged)
    return reinterpret_cast<unsigned long long*>(a.devicePointer ? a.devicePointer : (void*)t);
  if (a.type == cudaMemoryTypeHost && a.devicePointer) return reinterpret_cast<unsigned long long*>(a.devicePointer);
  return nullptr;
}

// the ticket kernel's result to the caller: stored by the kernel, or copied
int deliver_ticket(fhv_ctx* ctx, fhv_ticket_t* ticket, bool stored, cudaStream_t s) {
  if (stored) return FHV_OK;
  return check_cuda(ctx, cudaMemcpyAsync(ticket, &ctx->ctl->spare[4], sizeof(fhv_ticket_t), cudaMemcpyDefault, s));
}

int join_aux(fhv_ctx* ctx, cudaStream_t s) {
  if (!ctx->join_pending) return FHV_OK;
  ctx->join_pending = false;
  return check_cuda(ctx, cudaStreamWaitEvent(s, ctx->ev_join, 0));
}

// FHV_FORK_CLEARS: 0 inline clears (A/B); 1 both clears during the job
// setup; 2 the counters during the job setup, the cursors during the
// counting pass
static int fork_mode() {
  static const int v = env_int("FHV_FORK_CLEARS", 2);
  return v;
}

// clear `n` words at `buf` on the side stream after the work queued on `s` so far
int fork_clear(fhv_ctx* ctx, void* buf, size_t bytes, cudaStream_t s, void* buf2) {
  int rc;
  if (!ctx->aux) {
    if ((rc = check_cuda(ctx, cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking)))) return rc;
    if ((rc = check_cuda(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming)))) return rc;
    if ((rc = check_cuda(ctx, cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming)))) return rc;
  }
  if ((rc = check_cuda(ctx, cudaEventRecord(ctx->ev_fork, s)))) return rc;
  if ((rc = check_cuda(ctx, cudaStreamWaitEvent(ctx->aux, ctx->ev_fork, 0)))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(buf, 0, bytes, ctx->aux)))) return rc;
  if (buf2 && (rc = check_cuda(ctx, cudaMemsetAsync(buf2, 0, bytes, ctx->aux)))) return rc;
  if ((rc = check_cuda(ctx, cudaEventRecord(ctx->ev_join, ctx->aux)))) return rc;
  ctx->join_pending = true;
  return FHV_OK;
}

// the asynchronous build's leaf counters (and, mode 1, cursors) cleared on the side stream
static int fork_clears(fhv_ctx* ctx, uint32_t* counts, unsigned long long n_leaves, cudaStream_t s) {
  const int mode = fork_mode();
  if (!mode) return FHV_OK;
  uint32_t* cursors = (uint32_t*)scratch(ctx, kCursors, (size_t)n_leaves * 4);
  if (!cursors) return FHV_NOMEM;
  int rc = fork_clear(ctx, counts, (size_t)n_leaves * 4, s, mode == 1 ? cursors : nullptr);
  if (rc) return rc;
  ctx->counts_zeroed = counts;
  ctx->cursors_zeroed = mode == 1 ? cursors : nullptr;
  ctx->fork_cursors_at_count = mode == 2 ? cursors : nullptr;
  return FHV_OK;
}

// the asynchronous build after pass 1: directory, pass 2, ticket
static int pofa_build_async_rest(fhv_ctx* ctx, CaptureParams& p, int32_t levels, unsigned long long n_leaves,
                                 uint32_t* counts, uint32_t* offsets, uint8_t* pyramid, fhv_pool_t* pool,
                                 int32_t flags, bool ranks, fhv_ticket_t* ticket, cudaStream_t s);
}  // namespace fhv

extern "C" int fhv_pofa_build_async(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg,
                                    int32_t levels, uint32_t* counts, uint32_t* offsets, uint8_t* pyramid,
                                    fhv_pool_t* pool, int32_t flags, fhv_ticket_t* ticket, void* stream) {
  if (!ctx || !counts || !offsets || !pyramid || !ticket || levels < 1 || levels > 10) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  if (!pool || pool->capacity <= 0 || !pool->pos || !pool->nrm || !pool->mat || !pool->obj || !pool->prev)
    return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned long long n_leaves = 1ull << (3 * levels);
  const bool ranks = (flags & FHV_EXACT_ORDER) != 0;
  CaptureParams p;
  // the leaf counters and the cursors are cleared on the side stream while
  // the job setup and the plan run (joined before the counting pass)
  if ((rc = fork_clears(ctx, counts, n_leaves, s))) return rc;
  // speculative item plan when this ctx has one for the job count (else plan() syncs once)
  // (the emission ranks' scan rides in the directory launch)
  rc = pofa_count_async(ctx, tris, cfg, levels, nullptr, counts, s, p, true, ranks, false, true);
  if (rc) {
    join_aux(ctx, s);
    ctx->counts_zeroed = ctx->cursors_zeroed = nullptr;
    ctx->fork_cursors_at_count = nullptr;
    return rc;
  }
  // (pass 1 reset the control block and touched none of alloc / leaf_n / dir_done)
  ctx->ctl_fresh = true;
  rc = pofa_build_async_rest(ctx, p, levels, n_leaves, counts, offsets, pyramid, pool, flags, ranks, ticket, s);
  ctx->ctl_fresh = false;
  return rc;
}

namespace fhv {
static int pofa_build_async_rest(fhv_ctx* ctx, CaptureParams& p, int32_t levels, unsigned long long n_leaves,
                                 uint32_t* counts, uint32_t* offsets, uint8_t* pyramid, fhv_pool_t* pool,
                                 int32_t flags, bool ranks, fhv_ticket_t* ticket, cudaStream_t s) {
  int rc;
  const bool deferred = ctx->item_scan_n >= 0;
  // the fused directory launch stores the fragment total itself; otherwise a copy
  ctx->dir_frags_total = deferred;
  ctx->dir_frags_stored = false;
  rc = fhv_pofa_shard_directory_nocheck(ctx, levels, counts, offsets, pyramid, s);
  const bool stored = ctx->dir_frags_stored;
  ctx->dir_frags_total = ctx->dir_frags_stored = false;
  if (rc) return rc;
  if ((!ranks || (deferred && !stored)) &&
      (rc = check_cuda(ctx, cudaMemcpyAsync(&ctx->ctl->frags_total, &ctx->ctl->scan_total, sizeof(unsigned long long),
                                            cudaMemcpyDeviceToDevice, s))))
    return rc;
  if ((rc = pofa_scatter_async(ctx, p, levels, 0, n_leaves, counts, offsets, 0, pool, flags, s, false,
                                &ctx->ctl->frags_total, 0)))
    return rc;
  unsigned long long* tk_dev = ticket_device_view(ticket);
  {
    LaunchScope L_(ctx, kStScan, s);
    k_ticket<<<1, 1, 0, s>>>(ctx->ctl, tk_dev);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  // pass-1 bookkeeping for a follow-up fhv_pofa_scatter is not kept: the
  // ticket is the only result
  ctx->pass1_levels = -1;
  return deliver_ticket(ctx, ticket, tk_dev != nullptr, s);
}
}  // namespace fhv

// One rank's share of pofa_build with no host wait and no collective: the
// caller speculates every rank's fragment total from the previous build of
// the same scene / ranges (base = the lower ranks' totals, the pool sized by
// this rank's), reuses that build's triangle binning, and enqueues pass 1,
// the directory (global offsets from `base`) and pass 2.  The ticket holds
// this rank's status and total: the build is valid when EVERY rank's ticket
// checks against its guess (then every base was right too).
extern "C" int fhv_pofa_shard_build_async(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg,
                                          int32_t levels, const fhv_shard_t* shard, uint32_t* counts_local,
                                          uint32_t* offsets_local, uint8_t* pyramid, uint64_t base, fhv_pool_t* pool,
                                          int32_t flags, fhv_ticket_t* ticket, void* stream) {
  if (!ctx || !counts_local || !offsets_local || !pyramid || !ticket || levels < 1 || levels > 10 ||
      !shard_ok(shard, levels))
    return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  if (!pool || pool->capacity < 0 || (pool->capacity > 0 && (!pool->pos || !pool->nrm || !pool->mat || !pool->obj ||
                                                              !pool->prev)))
    return FHV_BAD_ARGS;
  if (base + (uint64_t)pool->capacity > 0xffffffffull) return FHV_TOO_MANY;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned long long n_leaves = 1ull << (3 * levels);
  const unsigned long long lo = shard ? shard->cell_lo : 0ull, hi = shard ? shard->cell_hi : n_leaves;
  CaptureParams p;
  if ((rc = pofa_count_async(ctx, tris, cfg, levels, shard, counts_local, s, p, true, true, true))) return rc;
  if (lo == 0 && hi == n_leaves && base == 0) {
    if ((rc = scan_leaves_and_pyramid(ctx, counts_local, offsets_local, pyramid, levels, s))) return rc;
  } else if ((rc = scan_leaf_range_and_pyramid(ctx, counts_local, offsets_local, pyramid, levels, lo, hi, base, s))) {
    return rc;
  }
  if (pool->capacity > 0 &&
      (rc = pofa_scatter_async(ctx, p, levels, lo, hi, counts_local, offsets_local, base, pool, flags, s, false,
                               &ctx->ctl->frags_total, 0)))
    return rc;
  unsigned long long* tk_dev = ticket_device_view(ticket);
  {
    LaunchScope L_(ctx, kStScan, s);
    k_ticket<<<1, 1, 0, s>>>(ctx->ctl, tk_dev);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  ctx->pass1_levels = -1;  // the ticket is the only result
  return deliver_ticket(ctx, ticket, tk_dev != nullptr, s);
}

namespace fhv {
namespace {
// the ticket check on the device (same rules as fhv_ticket_check) over the
// staged outcome of the build just enqueued on this stream; failures are
// kept sticky in acc[0] (first non-OK status), acc[1] counts the checks --
// for a CUDA graph replaying the build many times
__global__ void k_ticket_acc(const Control* ctl, long long expect, long long* acc) {
  const long long status = (long long)ctl->spare[4];
  const long long frags = (long long)ctl->spare[5], scan = (long long)ctl->spare[6], alloc = (long long)ctl->spare[7];
  long long rc = FHV_OK;
  if (status == FHV_RETRY_ITEMS || status == FHV_NEED_POOL) rc = FHV_STALE;
  else if (status) rc = status;
  else if (frags >= (1LL << 32)) rc = FHV_TOO_MANY;
  else if (scan != frags || alloc != frags) rc = FHV_PASS_MISMATCH;
  else if (frags != expect) rc = FHV_STALE;
  if (rc) atomicCAS(reinterpret_cast<unsigned long long*>(acc), 0ull, (unsigned long long)rc);
  atomicAdd(reinterpret_cast<unsigned long long*>(acc + 1), 1ull);
}
}  // namespace
}  // namespace fhv

namespace fhv {
namespace {
// the linked build's outcome in the POFA ticket's words: total in all three
// count fields (so fhv_ticket_check / k_ticket_acc compare it with the guess)
__global__ void k_ticket_linked(Control* ctl, int atomic_alloc, unsigned long long* out) {
  const unsigned long long total = atomic_alloc ? ctl->alloc : ctl->scan_total;
  put_ticket(ctl, out, (unsigned long long)(long long)ctl->status, total, total, total);
}
}  // namespace
}  // namespace fhv

// build_pofl without a host wait (the POFA build's ticket protocol): the pool
// capacity is the caller's (its guess of the total, or the overalloc), the
// item plan speculative when this ctx has one for the job count; the total
// and the status land in *ticket.  A total above the capacity means dropped
// records (FHV_OVERFLOW semantics of the synchronous build), a speculation
// miss FHV_RETRY_ITEMS in the status (rebuild with fhv_build_pofl).
extern "C" int fhv_build_pofl_async(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg,
                                    int32_t levels, fhv_pool_t* pool, int32_t* heads, uint8_t* pyramid, int32_t flags,
                                    fhv_ticket_t* ticket, void* stream) {
  if (!ctx || !pool || !heads || !pyramid || !ticket) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  if (pool->capacity < 0 || pool->capacity >= (1LL << 31)) return FHV_BAD_ARGS;
  if (levels < 1 || levels > kMaxLevels) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const CaptureParams p = make_params(tris, cfg);
  const bool atomic_alloc = (flags & FHV_ALLOC_ATOMIC) != 0;
  const long long n_keys = 1LL << (3 * levels);
  if ((rc = plan(ctx, p, s, true))) return rc;
  if ((rc = count(ctx, p, false, 0, nullptr, s))) return rc;
  EmitOut o = empty_out();
  set_pool(o, pool);
  o.heads = heads;
  o.flags = flags;
  o.levels = levels;
  o.n_keys = n_keys;
  if ((rc = emit<kPofl>(ctx, p, o, atomic_alloc, s))) return rc;
  if ((flags & FHV_EXACT_ORDER) && (rc = chain_order(ctx, heads, pool->prev, n_keys, pool->capacity, s))) return rc;
  if ((rc = pyramid_from_heads(ctx, heads, pyramid, levels, s))) return rc;
  unsigned long long* tk_dev = ticket_device_view(ticket);
  {
    LaunchScope L_(ctx, kStScan, s);
    k_ticket_linked<<<1, 1, 0, s>>>(ctx->ctl, atomic_alloc ? 1 : 0, tk_dev);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  return deliver_ticket(ctx, ticket, tk_dev != nullptr, s);
}

extern "C" int fhv_ticket_accumulate(fhv_ctx* ctx, int64_t expect_total, int64_t* acc, void* stream) {
  if (!ctx || !acc) return FHV_BAD_ARGS;
  {
    LaunchScope L_(ctx, kStScan, (cudaStream_t)stream);
    k_ticket_acc<<<1, 1, 0, (cudaStream_t)stream>>>(ctx->ctl, (long long)expect_total, (long long*)acc);
  }
  return check_cuda(ctx, cudaGetLastError());
}

extern "C" int fhv_ticket_check(const fhv_ticket_t* t, int64_t expect_total) {
  if (!t) return FHV_BAD_ARGS;
  if (t->status == FHV_RETRY_ITEMS || t->status == FHV_NEED_POOL) return FHV_STALE;
  if (t->status) return (int)t->status;
  if (t->frags_total >= (1LL << 32)) return FHV_TOO_MANY;
  if (t->scan_total != t->frags_total || t->alloc != t->frags_total) return FHV_PASS_MISMATCH;
  if (t->frags_total != expect_total) return FHV_STALE;
  return FHV_OK;
}

extern "C" int fhv_pofa_scatter(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                                const uint32_t* counts, const uint32_t* offsets, fhv_pool_t* pool, int32_t flags,
                                void* stream) {
  return fhv_pofa_shard_scatter(ctx, tris, cfg, levels, nullptr, counts, offsets, 0, pool, flags, stream);
}

// deferred_baseline (fhv/render.py:327-382): every triangle through the
// camera (_raster_screen), nearest (depth, triangle) per pixel into the f64
// G-buffer, then one Blinn-Phong pass.  gb must carry all five planes.
extern "C" int fhv_deferred(fhv_ctx* ctx, const fhv_tris_t* tris, const double* proj, int32_t width, int32_t height,
                            const double* eye, const fhv_shading_t* shading, const double* background,
                            double* out_rgba, double* out_depth, const fhv_gbuffer_t* gb, int64_t* emitted,
                            void* stream) {
  if (!ctx || !tris || !proj || !eye || !shading || !background || !out_rgba || !out_depth || !gb || width < 1 ||
      height < 1 || !gb->position || !gb->normal || !gb->material_id || !gb->object_id || !gb->valid)
    return FHV_BAD_ARGS;
  if (tris->n_tri < 0 || (tris->n_tri > 0 && (!tris->pos || !tris->vnrm || !tris->fnrm || !tris->mat || !tris->obj)))
    return FHV_BAD_ARGS;
  if (tris->n_tri >= (1LL << 32) - 1) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  CaptureParams p;
  std::memset(&p, 0, sizeof(p));
  p.strategy = kScreen;
  p.res = height;
  p.width = width;
  p.height = height;
  p.ortho = proj[12] == 0.0 && proj[13] == 0.0 && proj[14] == 0.0 && proj[15] == 1.0;
  std::memcpy(p.proj[0], proj, 16 * sizeof(double));
  p.n_tri = tris->n_tri;
  p.n_jobs = tris->n_tri;
  p.pos = tris->pos;
  p.vnrm = tris->vnrm;
  p.fnrm = tris->fnrm;
  p.mat = tris->mat;
  p.obj = tris->obj;
  p.cell_hi = ~0ull;
  const long long P = (long long)width * height;
  p.persp = (JobPersp*)scratch(ctx, kJobPersp, (size_t)(p.n_jobs > 0 ? p.n_jobs : 1) * sizeof(JobPersp));
  auto* key = (unsigned long long*)scratch(ctx, kSplatKey, (size_t)P * 8);
  auto* win = (uint32_t*)scratch(ctx, kSplatWin, (size_t)P * 4);
  if (!p.persp || !key || !win) return FHV_NOMEM;
  int rc;
  for (int attempt = 0; attempt < 2; ++attempt) {
  if ((rc = plan(ctx, p, s, attempt == 0))) return rc;
  if ((rc = count(ctx, p, false, 0, nullptr, s))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(key, 0xff, (size_t)P * 8, s)))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(win, 0xff, (size_t)P * 4, s)))) return rc;
  if (ctx->n_items > 0) {
    {
      LaunchScope L_(ctx, kStDeferred, s);
      k_job_n1<<<grid_for(p.n_jobs, 256), 256, 0, s>>>(p.n_jobs, (const uint32_t*)ctx->bufs[kJobItems].ptr,
                                                       (const unsigned long long*)ctx->bufs[kJobItemOff].ptr,
                                                       (const uint32_t*)ctx->bufs[kItemCnt].ptr, p.persp);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
    EmitOut o = empty_out();
    o.ds_key = key;
    o.ds_win = win;
    o.gb = *gb;
    if ((rc = emit<kDsDepth>(ctx, p, o, false, s))) return rc;
    if ((rc = emit<kDsIndex>(ctx, p, o, false, s))) return rc;
    if ((rc = emit<kDsWrite>(ctx, p, o, false, s))) return rc;
  }
  if ((rc = deferred_resolve(ctx, P, shading, eye, key, win, gb, background, out_rgba, out_depth, s))) return rc;
  rc = sync_control(ctx, s);
  if (rc != FHV_RETRY_ITEMS) break;
  }
  if (emitted) *emitted = (int64_t)ctx->ctl_host->scan_total;
  return rc;
}

extern "C" int fhv_rebuild_pofa(fhv_ctx* ctx, int32_t levels, const fhv_pool_t* src, int64_t n, uint32_t* counts,
                                uint32_t* offsets, uint8_t* pyramid, fhv_pool_t* dst, void* stream) {
  if (!ctx || !src || !dst || !counts || !offsets || !pyramid || levels < 1 || levels > 10 || n < 0 ||
      n > src->capacity || dst->capacity < n || n >= (1LL << 31))
    return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const long long n_leaves = 1LL << (3 * levels);
  uint32_t* cursors = (uint32_t*)scratch(ctx, kCursors, (size_t)n_leaves * 4);
  if (!cursors) return FHV_NOMEM;
  int rc;
  if ((rc = reset_control(ctx, s))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(counts, 0, (size_t)n_leaves * 4, s)))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(cursors, 0, (size_t)n_leaves * 4, s)))) return rc;
  if (n > 0) {
    LaunchScope L_(ctx, kStCountLeaves, s);
    k_pool_leaf_hist<<<grid_for(n, 256), 256, 0, s>>>(src->pos, n, levels, counts, &ctx->ctl->status);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  ctx->dir_sums_levels = -1;  // no counting-pass tile totals for a repack
  if ((rc = scan_leaves_and_pyramid(ctx, counts, offsets, pyramid, levels, s))) return rc;
  if (n > 0) {
    {
      LaunchScope L_(ctx, kStEmitPofa, s);
      k_pool_leaf_scatter<<<grid_for(n, 256), 256, 0, s>>>(src->pos, src->nrm, src->mat, src->obj, n, levels, offsets,
                                                           cursors, dst->pos, dst->nrm, dst->mat, dst->obj, dst->prev);
    }
    {
      LaunchScope L_(ctx, kStLeafOrder, s);
      k_leaf_order<<<grid_for(n_leaves, 128, 32), 128, 0, s>>>(offsets, counts, n_leaves, 0ull,
                                                               (unsigned long long)dst->capacity, dst->pos, dst->nrm,
                                                               dst->mat, dst->obj, dst->prev);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  }
  return sync_control(ctx, s);
}

extern "C" int fhv_pack_records(fhv_ctx* ctx, const fhv_pool_t* pool, int64_t n, void* out, void* stream) {
  if (!ctx || !pool || n < 0 || n > pool->capacity || (n > 0 && !out) || ((uintptr_t)out & 3)) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  {
    LaunchScope L_(ctx, kStLeafOrder, s);
    k_pack_records<<<grid_for(9 * n, 256), 256, 0, s>>>(pool->pos, pool->nrm, pool->mat, pool->obj, pool->prev, n,
                                                        (uint32_t*)out);
  }
  return check_cuda(ctx, cudaGetLastError());
}

extern "C" int fhv_unpack_records(fhv_ctx* ctx, const void* in, int64_t n, fhv_pool_t* pool, void* stream) {
  if (!ctx || !pool || n < 0 || n > pool->capacity || (n > 0 && !in) || ((uintptr_t)in & 3)) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  cudaStream_t s = (cudaStream_t)stream;
  {
    LaunchScope L_(ctx, kStLeafOrder, s);
    k_unpack_records<<<grid_for(9 * n, 256), 256, 0, s>>>((const uint32_t*)in, n, pool->pos, pool->nrm, pool->mat,
                                                          pool->obj, pool->prev);
  }
  return check_cuda(ctx, cudaGetLastError());
}

extern "C" int fhv_unit_rows(fhv_ctx* ctx, int64_t n, const double* in, double* out, int64_t* zero_first,
                             void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!in || !out))) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->spare[2], 0xff, 8, s)))) return rc;
  if (n > 0) {
    LaunchScope L_(ctx, kStFaceNormals, s);
    k_unit_rows<<<grid_for(n, 256), 256, 0, s>>>(n, in, out, &ctx->ctl->spare[2]);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  const unsigned long long z = ctx->ctl_host->spare[2];
  if (zero_first) *zero_first = z == ~0ull ? -1 : (int64_t)z;
  return FHV_OK;
}

namespace fhv {
namespace {
// indexed -> triangle-soup gather: thread per (triangle, corner, component)
// pair of f64 rows, coalesced writes
__global__ void __launch_bounds__(256) k_expand_indexed(long long n_vert, const double* __restrict__ vpos,
                                                        const double* __restrict__ vn, long long n_tri,
                                                        const uint32_t* __restrict__ faces, double* __restrict__ pos,
                                                        double* __restrict__ vnrm, int* status) {
  const long long n = 9 * n_tri;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long corner = i / 3;  // (triangle, vertex) slot
    const int comp = (int)(i - 3 * corner);
    const uint32_t v = __ldg(&faces[corner]);
    if ((long long)v >= n_vert) {
      raise_status(status, FHV_BAD_ARGS);
      continue;
    }
    pos[i] = __ldg(&vpos[3 * (long long)v + comp]);
    vnrm[i] = __ldg(&vn[3 * (long long)v + comp]);
  }
}
}  // namespace
}  // namespace fhv

extern "C" int fhv_expand_indexed(fhv_ctx* ctx, int64_t n_vert, const double* vpos, const double* vn, int64_t n_tri,
                                  const uint32_t* faces, double* pos, double* vnrm, void* stream) {
  if (!ctx || n_vert < 0 || n_tri < 0 || (n_tri && (!vpos || !vn || !faces || !pos || !vnrm))) return FHV_BAD_ARGS;
  if (n_tri == 0) return FHV_OK;
  {
    LaunchScope L_(ctx, kStFaceNormals, (cudaStream_t)stream);
    k_expand_indexed<<<grid_for(9 * n_tri, 256), 256, 0, (cudaStream_t)stream>>>(n_vert, vpos, vn, n_tri, faces, pos,
                                                                                vnrm, &ctx->ctl->status);
  }
  return check_cuda(ctx, cudaGetLastError());
}

extern "C" int fhv_face_normals(fhv_ctx* ctx, int64_t n_tri, const double* pos, double* fnrm, void* stream) {
  if (!ctx || n_tri < 0 || (n_tri && (!pos || !fnrm))) return FHV_BAD_ARGS;
  if (n_tri == 0) return FHV_OK;
  {
    LaunchScope L_(ctx, kStFaceNormals, (cudaStream_t)stream);
    k_face_normals<<<grid_for(n_tri, 256), 256, 0, (cudaStream_t)stream>>>(n_tri, pos, fnrm);
  }
  return check_cuda(ctx, cudaGetLastError());
}
