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
//   k_count        lane per item: exact coverage count (+ per-leaf histogram
//                  with warp-free run aggregation for POFA pass 1)
//   scan           item counts -> item fragment offsets = the reference's
//                  pool index of each item's first fragment (its "rank")
//   k_emit<MODE>   lane per item: coverage, barycentrics, interpolation,
//                  f32 record, then the store-specific insert
//   fix-ups        EXACT_ORDER chain / in-leaf sorts, POFL pyramid (sync #2)
//
// Exactness: coverage ties are decided on bit-identical f64 edge functions
// (-fmad=false + explicit __fma_rn where NumPy/OpenBLAS fuse), so the covered
// set, counts and octant ranges are bit-exact; interpolated attributes follow
// the same operation order and match bit for bit as well.
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

struct CaptureParams {
  int strategy, res;
  double pitch;
  double proj[3][16];
  long long n_tri, n_jobs;
  const double* pos;
  const double* vnrm;
  const double* fnrm;
  const uint32_t* mat;
  const uint32_t* obj;
};

enum EmitMode { kList = 0, kPpfl = 1, kPofl = 2, kPofa = 3 };

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
  // POFA
  const uint32_t* offsets;
  const uint32_t* counts;
  uint32_t* cursors;
  // list
  long long max_out;
  long long* job;
  int32_t* px;
  int32_t* py;
  double* wpos;
  double* wnrm;
  int flags;
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

// _raster_screen for an orthographic capture axis (fhv/raster.py:184-209)
__device__ __forceinline__ void setup_screen(const CaptureParams& p, long long t, int axis, JobSetup& js) {
  const double* M = p.proj[axis];
  const double* P = p.pos + 9 * t;
  double xr[3], yr[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double X = P[3 * i], Y = P[3 * i + 1], Z = P[3 * i + 2];
    const double c0 = __dadd_rn(fwd3(X, Y, Z, M[0], M[1], M[2]), M[3]);
    const double c1 = __dadd_rn(fwd3(X, Y, Z, M[4], M[5], M[6]), M[7]);
    const double c3 = __dadd_rn(fwd3(X, Y, Z, M[12], M[13], M[14]), M[15]);
    const double nx = __ddiv_rn(c0, c3), ny = __ddiv_rn(c1, c3);
    xr[i] = __dmul_rn(__dmul_rn(__dadd_rn(nx, 1.0), 0.5), (double)p.res);
    yr[i] = __dmul_rn(__dmul_rn(__dsub_rn(1.0, ny), 0.5), (double)p.res);
  }
  finish_setup(xr, yr, p.res, p.res, js);
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
  const double n0 = __ddiv_rn(F[0], norm), n1 = __ddiv_rn(F[1], norm), n2 = __ddiv_rn(F[2], norm);
  const bool hx = fabs(n0) <= 0.6;
  const double h0 = hx ? 1.0 : 0.0, h1 = hx ? 0.0 : 1.0, h2 = 0.0;
  const double hn = fwd3(h0, h1, h2, n0, n1, n2);
  double t0 = __dsub_rn(h0, __dmul_rn(hn, n0));
  double t1 = __dsub_rn(h1, __dmul_rn(hn, n1));
  double t2 = __dsub_rn(h2, __dmul_rn(hn, n2));
  const double tn = __dsqrt_rn(fwd3(t0, t1, t2, t0, t1, t2));
  t0 = __ddiv_rn(t0, tn);
  t1 = __ddiv_rn(t1, tn);
  t2 = __ddiv_rn(t2, tn);
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
  double nxd = ceil(__ddiv_rn(__dsub_rn(tmax, tmin), p.pitch));
  double nyd = ceil(__ddiv_rn(__dsub_rn(bmax, bmin), p.pitch));
  if (!(nxd >= 1.0)) nxd = 1.0;
  if (!(nyd >= 1.0)) nyd = 1.0;
  if (nxd > 2147483647.0 || nyd > 2147483647.0) {
    raise_status(status, FHV_BAD_ARGS);
    return;
  }
  double xr[3], yr[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    xr[i] = __ddiv_rn(__dsub_rn(tc[i], tmin), p.pitch);
    yr[i] = __ddiv_rn(__dsub_rn(bmax, bc[i]), p.pitch);
  }
  finish_setup(xr, yr, (long long)nxd, (long long)nyd, js);
}

__global__ void k_job_setup(CaptureParams p, JobSetup* __restrict__ jobs, uint32_t* __restrict__ job_items,
                            int* status) {
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
      setup_screen(p, t, axis, js);
    const unsigned long long pix = (unsigned long long)js.bw * (unsigned long long)js.bh;
    unsigned long long items = (pix + kItemPix - 1) / kItemPix;
    if (items > 0xFFFFFFFFull) {
      raise_status(status, FHV_NOMEM);
      items = 0;
    }
    jobs[j] = js;
    job_items[j] = (uint32_t)items;
  }
}

// work items of each job: a lane per job writes small jobs' items itself;
// jobs with many items (large triangles) are written by the whole warp, one
// such job at a time (ballot loop), so both 1-item and 10^4-item jobs stay
// coalesced
constexpr uint32_t kExpandSmall = 4;

__global__ void __launch_bounds__(256) k_item_expand(long long n_jobs, const uint32_t* __restrict__ job_items,
                                                     const unsigned long long* __restrict__ job_item_off,
                                                     uint32_t* __restrict__ item_job, uint32_t* __restrict__ item_p0) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j0 = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); j0 < n_jobs; j0 += stride) {
    const long long j = j0 + lane_id();
    const uint32_t n = j < n_jobs ? job_items[j] : 0u;
    const unsigned long long base = j < n_jobs ? job_item_off[j] : 0ull;
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
// coverage sweep (fhv/_ckern.pyx:72-101)

struct Cover {
  double ax, ay, bx, by, cx, cy;
  double e0x, e0y, e1x, e1y, e2x, e2y;
  double area2;
  bool tl0, tl1, tl2;
  int x0, y0, bw;
};

__device__ __forceinline__ void load_cover(const JobSetup& js, Cover& c) {
  c.ax = js.ax; c.ay = js.ay; c.bx = js.bx; c.by = js.by; c.cx = js.cx; c.cy = js.cy;
  c.area2 = __dsub_rn(__dmul_rn(__dsub_rn(c.bx, c.ax), __dsub_rn(c.cy, c.ay)),
                      __dmul_rn(__dsub_rn(c.by, c.ay), __dsub_rn(c.cx, c.ax)));
  c.e0x = __dsub_rn(c.cx, c.bx); c.e0y = __dsub_rn(c.cy, c.by);  // v1 -> v2, opposite v0
  c.e1x = __dsub_rn(c.ax, c.cx); c.e1y = __dsub_rn(c.ay, c.cy);  // v2 -> v0, opposite v1
  c.e2x = __dsub_rn(c.bx, c.ax); c.e2y = __dsub_rn(c.by, c.ay);  // v0 -> v1, opposite v2
  c.tl0 = c.e0y < 0.0 || (c.e0y == 0.0 && c.e0x > 0.0);
  c.tl1 = c.e1y < 0.0 || (c.e1y == 0.0 && c.e1x > 0.0);
  c.tl2 = c.e2y < 0.0 || (c.e2y == 0.0 && c.e2x > 0.0);
  c.x0 = js.x0; c.y0 = js.y0; c.bw = js.bw;
}

// visit covered pixel centres of bbox slice [p0, p1) in row-major order
template <class F>
__device__ __forceinline__ void sweep(const Cover& c, uint32_t p0, uint32_t p1, F&& f) {
  const uint32_t r0 = p0 / (uint32_t)c.bw;
  int px = c.x0 + (int)(p0 - r0 * (uint32_t)c.bw);
  int py = c.y0 + (int)r0;
  const int xend = c.x0 + c.bw;
  double sy = __dadd_rn((double)py, 0.5);
  double k0 = __dmul_rn(c.e0x, __dsub_rn(sy, c.by));
  double k1 = __dmul_rn(c.e1x, __dsub_rn(sy, c.cy));
  double k2 = __dmul_rn(c.e2x, __dsub_rn(sy, c.ay));
  for (uint32_t q = p0; q < p1; ++q) {
    const double sx = __dadd_rn((double)px, 0.5);
    const double f0 = __dsub_rn(k0, __dmul_rn(c.e0y, __dsub_rn(sx, c.bx)));
    if (f0 > 0.0 || (f0 == 0.0 && c.tl0)) {
      const double f1 = __dsub_rn(k1, __dmul_rn(c.e1y, __dsub_rn(sx, c.cx)));
      if (f1 > 0.0 || (f1 == 0.0 && c.tl1)) {
        const double f2 = __dsub_rn(k2, __dmul_rn(c.e2y, __dsub_rn(sx, c.ax)));
        if (f2 > 0.0 || (f2 == 0.0 && c.tl2)) f(px, py, f0, f1, f2);
      }
    }
    if (++px == xend) {
      px = c.x0;
      ++py;
      sy = __dadd_rn((double)py, 0.5);
      k0 = __dmul_rn(c.e0x, __dsub_rn(sy, c.by));
      k1 = __dmul_rn(c.e1x, __dsub_rn(sy, c.cy));
      k2 = __dmul_rn(c.e2x, __dsub_rn(sy, c.ay));
    }
  }
}

// triangle vertex data in winding order
struct TriData {
  double v[3][3];
  double n[3][3];
  double f[3];
  uint32_t mat, obj;
};

__device__ __forceinline__ void load_tri(const CaptureParams& p, const JobSetup& js, TriData& d, bool normals) {
  const double* P = p.pos + 9 * (long long)js.tri;
  const double* N = p.vnrm + 9 * (long long)js.tri;
  const int o[3] = {0, js.swapped ? 2 : 1, js.swapped ? 1 : 2};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) d.v[i][k] = __ldg(&P[3 * o[i] + k]);
  if (normals) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) d.n[i][k] = __ldg(&N[3 * o[i] + k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) d.f[k] = __ldg(&p.fnrm[3 * (long long)js.tri + k]);
    d.mat = __ldg(&p.mat[js.tri]);
    d.obj = __ldg(&p.obj[js.tri]);
  }
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
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = __ddiv_rn(v[k], len);
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = d.f[k];
  }
}

__device__ __forceinline__ unsigned long long job_pixels(const JobSetup& js) {
  return (unsigned long long)js.bw * (unsigned long long)js.bh;
}

// ---------------------------------------------------------------------------
// pass 1: exact counts (and the POFA per-leaf histogram, CountingSink)

template <bool kLeaves>
__global__ void __launch_bounds__(256) k_count(CaptureParams p, const JobSetup* __restrict__ jobs,
                                               const uint32_t* __restrict__ item_job,
                                               const uint32_t* __restrict__ item_p0, long long n_items,
                                               uint32_t* __restrict__ item_cnt, int levels,
                                               uint32_t* __restrict__ leaf_counts, int* status) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_items;
       i += (long long)gridDim.x * blockDim.x) {
    const JobSetup js = jobs[item_job[i]];
    Cover c;
    load_cover(js, c);
    const uint32_t p0 = item_p0[i];
    const unsigned long long pe = job_pixels(js);
    const uint32_t p1 = (unsigned long long)p0 + kItemPix < pe ? p0 + kItemPix : (uint32_t)pe;
    uint32_t cnt = 0;
    if (!kLeaves) {
      sweep(c, p0, p1, [&](int, int, double, double, double) { ++cnt; });
    } else {
      TriData d;
      load_tri(p, js, d, false);
      unsigned long long run_code = ~0ull;
      uint32_t run = 0;
      bool bad = false;
      sweep(c, p0, p1, [&](int, int, double f0, double f1, double f2) {
        ++cnt;
        const double l0 = __ddiv_rn(f0, c.area2), l1 = __ddiv_rn(f1, c.area2), l2 = __ddiv_rn(f2, c.area2);
        double w[3];
        interp_pos(d, l0, l1, l2, w);
        uint64_t code;
        if (!cell_code(__double2float_rn(w[0]), __double2float_rn(w[1]), __double2float_rn(w[2]), levels, &code)) {
          bad = true;
          return;
        }
        if (code == run_code) {
          ++run;
        } else {
          if (run) atomicAdd(&leaf_counts[run_code], run);
          run_code = code;
          run = 1;
        }
      });
      if (run) atomicAdd(&leaf_counts[run_code], run);
      if (bad) raise_status(status, FHV_RANGE);
    }
    item_cnt[i] = cnt;
  }
}

// ---------------------------------------------------------------------------
// pass 2: emission + insertion

__device__ __forceinline__ unsigned long long warp_alloc(unsigned long long* counter) {
  const unsigned m = __activemask();
  const unsigned lane = lane_id();
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

template <int kMode, bool kAtomicAlloc>
__global__ void __launch_bounds__(256) k_emit(CaptureParams p, const JobSetup* __restrict__ jobs,
                                              const uint32_t* __restrict__ item_job,
                                              const uint32_t* __restrict__ item_p0,
                                              const unsigned long long* __restrict__ item_off, long long n_items,
                                              EmitOut o, Control* ctl) {
  unsigned long long emitted = 0;
  bool bad_range = false, bad_pass = false, bad_key = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_items;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t jid = item_job[i];
    const JobSetup js = jobs[jid];
    Cover c;
    load_cover(js, c);
    TriData d;
    load_tri(p, js, d, true);
    const uint32_t p0 = item_p0[i];
    const unsigned long long pe = job_pixels(js);
    const uint32_t p1 = (unsigned long long)p0 + kItemPix < pe ? p0 + kItemPix : (uint32_t)pe;
    unsigned long long rank = kAtomicAlloc ? 0ull : item_off[i];
    sweep(c, p0, p1, [&](int px, int py, double f0, double f1, double f2) {
      const double l0 = __ddiv_rn(f0, c.area2), l1 = __ddiv_rn(f1, c.area2), l2 = __ddiv_rn(f2, c.area2);
      double w[3], nn[3];
      interp_pos(d, l0, l1, l2, w);
      interp_nrm(d, l0, l1, l2, nn);
      ++emitted;
      if (kMode == kList) {
        if ((long long)rank < o.max_out) {
          o.job[rank] = jid;
          o.px[rank] = px;
          o.py[rank] = py;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            o.wpos[3 * rank + k] = w[k];
            o.wnrm[3 * rank + k] = nn[k];
          }
        }
        ++rank;
        return;
      }
      const float q0 = __double2float_rn(w[0]), q1 = __double2float_rn(w[1]), q2 = __double2float_rn(w[2]);
      long long slot = 0;
      uint64_t key = 0;
      if (kMode != kPofa) {
        // slot first: records past capacity are dropped before any keying,
        // like _store_split (fhv/storage.py:338-342, 366-369, 388-392)
        slot = kAtomicAlloc ? (long long)warp_alloc(&ctl->alloc) : (long long)rank;
        if (slot >= o.capacity) { ++rank; return; }
      }
      if (kMode == kPpfl) {
        key = (uint64_t)py * (uint64_t)o.width + (uint64_t)px;
        if ((long long)key >= o.n_keys) { bad_key = true; ++rank; return; }
      } else if (!cell_code(q0, q1, q2, o.levels, &key)) {
        bad_range = true;
        ++rank;
        return;
      }
      if (kMode == kPofa) {
        const uint32_t cur = atomicAdd(&o.cursors[key], 1u);
        if (cur >= __ldg(&o.counts[key])) { bad_pass = true; ++rank; return; }
        slot = (long long)__ldg(&o.offsets[key]) + cur;
      }
      o.pos[3 * slot] = q0;
      o.pos[3 * slot + 1] = q1;
      o.pos[3 * slot + 2] = q2;
      o.nrm[3 * slot] = __double2float_rn(nn[0]);
      o.nrm[3 * slot + 1] = __double2float_rn(nn[1]);
      o.nrm[3 * slot + 2] = __double2float_rn(nn[2]);
      o.mat[slot] = d.mat;
      o.obj[slot] = d.obj;
      if (kMode == kPofa) {
        // prev_index = -1; under EXACT_ORDER the emission rank is parked here
        // until k_leaf_order restores the reference's in-leaf order
        o.prev[slot] = (o.flags & FHV_EXACT_ORDER) ? (int32_t)(uint32_t)rank : -1;
      } else {
        o.prev[slot] = atomicExch(&o.heads[key], (int32_t)slot);
      }
      ++rank;
    });
  }
  if (kMode == kPofa) {
    // pass-2 emitted count (compared with pass 1, fhv/storage.py:614-617)
    unsigned long long e = emitted;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if (lane_id() == 0 && e) atomicAdd(&ctl->alloc, e);
  }
  if (bad_range) raise_status(&ctl->status, FHV_RANGE);
  if (bad_pass) raise_status(&ctl->status, FHV_PASS_MISMATCH);
  if (bad_key) raise_status(&ctl->status, FHV_BAD_ARGS);
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
                             long long n_leaves, float* __restrict__ pos, float* __restrict__ nrm,
                             uint32_t* __restrict__ mat, uint32_t* __restrict__ obj, int32_t* __restrict__ prev) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n_leaves;
       c += (long long)gridDim.x * blockDim.x) {
    const uint32_t n = counts[c];
    if (n == 0) continue;
    const long long off = offsets[c];
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
    fn[3 * t] = len > 0.0 ? __ddiv_rn(c0, len) : 0.0;
    fn[3 * t + 1] = len > 0.0 ? __ddiv_rn(c1, len) : 0.0;
    fn[3 * t + 2] = len > 0.0 ? __ddiv_rn(c2, len) : 0.0;
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
  p.pitch = cfg->pitch;
  std::memcpy(p.proj, cfg->proj, sizeof(p.proj));
  p.n_tri = tris->n_tri;
  p.n_jobs = (cfg->strategy == 1 || cfg->strategy == 2) ? 3 * tris->n_tri : tris->n_tri;
  p.pos = tris->pos;
  p.vnrm = tris->vnrm;
  p.fnrm = tris->fnrm;
  p.mat = tris->mat;
  p.obj = tris->obj;
  return p;
}

int validate(const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg) {
  if (!tris || !cfg || tris->n_tri < 0 || cfg->strategy < 0 || cfg->strategy > 3 || cfg->res < 1) return FHV_BAD_ARGS;
  if (cfg->strategy == 3 && !(cfg->pitch > 0.0)) return FHV_BAD_ARGS;
  if (tris->n_tri > 0 && (!tris->pos || !tris->vnrm || !tris->fnrm || !tris->mat || !tris->obj)) return FHV_BAD_ARGS;
  if (3 * tris->n_tri >= (1LL << 32)) return FHV_BAD_ARGS;
  return FHV_OK;
}

// job setup + work-item expansion; leaves ctx->n_jobs / n_items (sync #1)
int plan(fhv_ctx* ctx, const CaptureParams& p, cudaStream_t s) {
  int rc = reset_control(ctx, s);
  if (rc) return rc;
  ctx->n_jobs = p.n_jobs;
  ctx->n_items = 0;
  if (p.n_jobs == 0) return FHV_OK;
  JobSetup* jobs = (JobSetup*)scratch(ctx, kJobs, (size_t)p.n_jobs * sizeof(JobSetup));
  uint32_t* job_items = (uint32_t*)scratch(ctx, kJobItems, (size_t)p.n_jobs * 4);
  auto* job_item_off = (unsigned long long*)scratch(ctx, kJobItemOff, (size_t)p.n_jobs * 8);
  if (!jobs || !job_items || !job_item_off) return FHV_NOMEM;
  {
    LaunchScope L_(ctx, kStJobSetup, s);
    k_job_setup<<<grid_for(p.n_jobs, 128), 128, 0, s>>>(p, jobs, job_items, &ctx->ctl->status);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  if ((rc = scan_u32_to_u64(ctx, job_items, job_item_off, p.n_jobs, s))) return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  const long long n_items = (long long)ctx->ctl_host->scan_total;
  ctx->n_items = n_items;
  if (n_items == 0) return FHV_OK;
  if (n_items >= (1LL << 31)) return FHV_NOMEM;
  uint32_t* item_job = (uint32_t*)scratch(ctx, kItemJob, (size_t)n_items * 4);
  uint32_t* item_p0 = (uint32_t*)scratch(ctx, kItemP0, (size_t)n_items * 4);
  if (!item_job || !item_p0) return FHV_NOMEM;
  {
    LaunchScope L_(ctx, kStItemExpand, s);
    k_item_expand<<<grid_for(p.n_jobs, 256), 256, 0, s>>>(p.n_jobs, job_items, job_item_off, item_job, item_p0);
  }
  return check_cuda(ctx, cudaGetLastError());
}

// counts per item (+ leaf histogram) and their scan (fragment ranks); async
int count(fhv_ctx* ctx, const CaptureParams& p, bool leaves, int levels, uint32_t* leaf_counts, cudaStream_t s) {
  const long long n = ctx->n_items;
  uint32_t* item_cnt = (uint32_t*)scratch(ctx, kItemCnt, (size_t)(n > 0 ? n : 1) * 4);
  auto* item_off = (unsigned long long*)scratch(ctx, kItemOff, (size_t)(n > 0 ? n : 1) * 8);
  if (!item_cnt || !item_off) return FHV_NOMEM;
  if (n > 0) {
    const JobSetup* jobs = (const JobSetup*)ctx->bufs[kJobs].ptr;
    const uint32_t* ij = (const uint32_t*)ctx->bufs[kItemJob].ptr;
    const uint32_t* ip = (const uint32_t*)ctx->bufs[kItemP0].ptr;
    {
      LaunchScope L_(ctx, leaves ? kStCountLeaves : kStCount, s);
      if (leaves)
        k_count<true><<<grid_for(n, 256), 256, 0, s>>>(p, jobs, ij, ip, n, item_cnt, levels, leaf_counts, &ctx->ctl->status);
      else
        k_count<false><<<grid_for(n, 256), 256, 0, s>>>(p, jobs, ij, ip, n, item_cnt, levels, nullptr, &ctx->ctl->status);
    }
    int rc = check_cuda(ctx, cudaGetLastError());
    if (rc) return rc;
  }
  return scan_u32_to_u64(ctx, item_cnt, item_off, n, s);
}

template <int kMode>
int emit(fhv_ctx* ctx, const CaptureParams& p, const EmitOut& o, bool atomic_alloc, cudaStream_t s) {
  const long long n = ctx->n_items;
  if (n == 0) return FHV_OK;
  const JobSetup* jobs = (const JobSetup*)ctx->bufs[kJobs].ptr;
  const uint32_t* ij = (const uint32_t*)ctx->bufs[kItemJob].ptr;
  const uint32_t* ip = (const uint32_t*)ctx->bufs[kItemP0].ptr;
  const auto* io = (const unsigned long long*)ctx->bufs[kItemOff].ptr;
  {
    LaunchScope L_(ctx, kStEmitList + kMode, s);
    if (atomic_alloc)
      k_emit<kMode, true><<<grid_for(n, 256), 256, 0, s>>>(p, jobs, ij, ip, io, n, o, ctx->ctl);
    else
      k_emit<kMode, false><<<grid_for(n, 256), 256, 0, s>>>(p, jobs, ij, ip, io, n, o, ctx->ctl);
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

extern "C" int fhv_capture_list(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int64_t max_out,
                                int64_t* job, int32_t* px, int32_t* py, double* wpos, double* wnrm, int64_t* n_out,
                                void* stream) {
  if (!ctx) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const CaptureParams p = make_params(tris, cfg);
  if ((rc = plan(ctx, p, s))) return rc;
  if ((rc = count(ctx, p, false, 0, nullptr, s))) return rc;
  EmitOut o = empty_out();
  o.max_out = max_out;
  o.job = (long long*)job;
  o.px = px;
  o.py = py;
  o.wpos = wpos;
  o.wnrm = wnrm;
  if (max_out > 0 && (rc = emit<kList>(ctx, p, o, false, s))) return rc;
  rc = sync_control(ctx, s);
  if (n_out) *n_out = (int64_t)ctx->ctl_host->scan_total;
  return rc;
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
  if ((rc = plan(ctx, p, s))) return rc;
  if (!atomic_alloc && (rc = count(ctx, p, false, 0, nullptr, s))) return rc;
  EmitOut o = empty_out();
  set_pool(o, pool);
  o.heads = heads;
  o.flags = flags;
  long long n_keys;
  if (pofl) {
    o.levels = levels;
    n_keys = 1LL << (3 * levels);
  } else {
    o.width = width;
    n_keys = (long long)width * (long long)cfg->res;  // caller's directory is width x res
  }
  o.n_keys = n_keys;
  rc = pofl ? emit<kPofl>(ctx, p, o, atomic_alloc, s) : emit<kPpfl>(ctx, p, o, atomic_alloc, s);
  if (rc) return rc;
  if (flags & FHV_EXACT_ORDER) {
    if ((rc = chain_order(ctx, heads, pool->prev, n_keys, pool->capacity, s))) return rc;
  }
  if (pofl && (rc = pyramid_from_heads(ctx, heads, pyramid, levels, s))) return rc;
  rc = sync_control(ctx, s);
  const long long total = (long long)(atomic_alloc ? ctx->ctl_host->alloc : ctx->ctl_host->scan_total);
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

extern "C" int fhv_pofa_count(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                              uint32_t* counts, uint32_t* offsets, uint8_t* pyramid, int64_t* total, void* stream) {
  if (!ctx || !counts || !offsets || !pyramid || levels < 1 || levels > 10) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const CaptureParams p = make_params(tris, cfg);
  const long long n_leaves = 1LL << (3 * levels);
  ctx->pass1_levels = -1;
  if ((rc = plan(ctx, p, s))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(counts, 0, (size_t)n_leaves * 4, s)))) return rc;
  if ((rc = count(ctx, p, true, levels, counts, s))) return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  const long long frags = (long long)ctx->ctl_host->scan_total;
  if (frags >= (1LL << 32)) return FHV_TOO_MANY;
  if ((rc = scan_leaves_and_pyramid(ctx, counts, offsets, pyramid, levels, s))) return rc;
  if ((rc = sync_control(ctx, s))) return rc;
  if ((long long)ctx->ctl_host->scan_total != frags) return FHV_PASS_MISMATCH;
  ctx->pass1_total = frags;
  ctx->pass1_levels = levels;
  ctx->pass1_tris = tris->n_tri;
  if (total) *total = frags;
  return FHV_OK;
}

extern "C" int fhv_pofa_scatter(fhv_ctx* ctx, const fhv_tris_t* tris, const fhv_capture_cfg_t* cfg, int32_t levels,
                                const uint32_t* counts, const uint32_t* offsets, fhv_pool_t* pool, int32_t flags,
                                void* stream) {
  if (!ctx || !counts || !offsets || !pool) return FHV_BAD_ARGS;
  int rc = validate(tris, cfg);
  if (rc) return rc;
  if (ctx->pass1_levels != levels || ctx->pass1_tris != tris->n_tri) return FHV_BAD_ARGS;
  if (pool->capacity < ctx->pass1_total) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  const CaptureParams p = make_params(tris, cfg);
  const long long n_leaves = 1LL << (3 * levels);
  uint32_t* cursors = (uint32_t*)scratch(ctx, kCursors, (size_t)n_leaves * 4);
  if (!cursors) return FHV_NOMEM;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(cursors, 0, (size_t)n_leaves * 4, s)))) return rc;
  if ((rc = check_cuda(ctx, cudaMemsetAsync(&ctx->ctl->alloc, 0, 8, s)))) return rc;
  EmitOut o = empty_out();
  set_pool(o, pool);
  o.levels = levels;
  o.offsets = offsets;
  o.counts = counts;
  o.cursors = cursors;
  o.flags = flags;
  if ((rc = emit<kPofa>(ctx, p, o, false, s))) return rc;
  if (flags & FHV_EXACT_ORDER) {
    {
      LaunchScope L_(ctx, kStLeafOrder, s);
      k_leaf_order<<<grid_for(n_leaves, 128, 32), 128, 0, s>>>(offsets, counts, n_leaves, pool->pos, pool->nrm,
                                                             pool->mat, pool->obj, pool->prev);
    }
    if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  }
  if ((rc = sync_control(ctx, s))) return rc;
  // cursors <= counts elementwise (checked per insert) and equal totals
  // imply cursors == counts (fhv/storage.py:614-619)
  if ((long long)ctx->ctl_host->alloc != ctx->pass1_total) return FHV_PASS_MISMATCH;
  return FHV_OK;
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
