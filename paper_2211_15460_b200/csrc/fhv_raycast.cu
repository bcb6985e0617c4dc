// fhv_raycast.cu -- image-order reconstruction by octree ray casting over a
// per-octant fragment volume (POFA ranges or POFL chains).
//
// Reference: render_raycast / _render_compiled (fhv/raycast.py:469-577) and
// the compiled kernel raycast_image / _ray_eval / _leaf_hits / _transmit /
// _shade_hit (fhv/_ckern.pyx:196-743).  One thread per primary ray:
//   * f64 slab traversal of the occupancy pyramid, children entered nearest
//     first (sorted by (t_enter, child)), stack of packed (level, code)
//     entries (the reference keeps 56-byte entries with boxes; boxes are
//     exact dyadic rationals, so they are recomputed from the code);
//   * the 8 child slab tests of a node share 3 planes per axis: 9 IEEE
//     divisions per node instead of 48, bit-identical values;
//   * per-leaf hits sorted by (t, pool index) in a small register buffer,
//     with an exact rescan fallback when a leaf has more hits;
//   * front-to-back compositing, alpha cutoff after each leaf, shadow rays
//     (mode 2) as a second traversal per hit and light;
//   * RaycastStats counters reproduced exactly (warp-reduced atomics).
#include "fhv_common.cuh"
#include "fhv_internal.h"

namespace fhv {

#ifndef FHV_RAY_MAXL
#define FHV_RAY_MAXL 12
#endif
constexpr int kRayMaxLevels = FHV_RAY_MAXL;
constexpr int kStack = 7 * kRayMaxLevels + 1;
constexpr int kHitBuf = 8;

struct RayParams {
  fhv_volume_t v;
  fhv_shading_t s;
  double eye[3];
  double bg[4];
  double radius, r2, cutoff, eps;
  int mode;
  // ray source: camera (cam != 0) or arrays
  int from_camera, persp;
  double rr[3], uu[3], ff[3];
  long long W, H;
  double half_w, half_h, t, aspect, near_;
  const double* origins;
  const double* dirs;
  long long start, end;
  double* out_rgba;
  int32_t* out_ids;
  long long* counters;
  unsigned long long* tile_ticket;  // dynamic 32-ray work fetching (zeroed before the launch)
  // packet kernel -> per-ray kernel hand-off: pixel indices of the rays whose
  // own (t_enter, child) order left the packet's shared child order
  long long* ray_list;
  unsigned long long* ray_list_n;
  unsigned long long* own_order_n;  // (lane, node) pairs that took their own child order
};

struct Stats {
  unsigned long long visited, tested, hits, early;
};

// _slab (fhv/_ckern.pyx:196-236) for one axis, given plane parameters
__device__ __forceinline__ bool slab_axis(double o, double d, double lo, double hi, double ta, double tb, double& t0,
                                          double& t1) {
  if (d == 0.0) return !(o < lo || o > hi);
  if (ta > tb) {
    const double s = ta;
    ta = tb;
    tb = s;
  }
  if (ta > t0) t0 = ta;
  if (tb < t1) t1 = tb;
  return true;
}

__device__ __forceinline__ bool slab_box(const double o[3], const double d[3], const double lo[3], const double hi[3],
                                         double t0, double t1, double* te) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double ta = 0.0, tb = 0.0;
    if (d[a] != 0.0) {
      ta = ddiv_z(__dsub_rn(lo[a], o[a]), d[a]);
      tb = ddiv_z(__dsub_rn(hi[a], o[a]), d[a]);
    }
    if (!slab_axis(o[a], d[a], lo[a], hi[a], ta, tb, t0, t1)) return false;
  }
  if (t0 > t1) return false;
  *te = t0;
  return true;
}

// fragment hit test (fhv/_ckern.pyx:277-291): plain f64, left to right
__device__ __forceinline__ bool hit_test_p(const RayParams& x, double px, double py, double pz, const double o[3],
                                           const double d[3], double tmin, double tmax, double* tout) {
  const double t = __dadd_rn(__dadd_rn(__dmul_rn(__dsub_rn(px, o[0]), d[0]), __dmul_rn(__dsub_rn(py, o[1]), d[1])),
                             __dmul_rn(__dsub_rn(pz, o[2]), d[2]));
  if (t < tmin || t > tmax) return false;
  const double ex = __dsub_rn(__dsub_rn(px, o[0]), __dmul_rn(t, d[0]));
  const double ey = __dsub_rn(__dsub_rn(py, o[1]), __dmul_rn(t, d[1]));
  const double ez = __dsub_rn(__dsub_rn(pz, o[2]), __dmul_rn(t, d[2]));
  if (plain3(ex, ey, ez) <= x.r2) {
    *tout = t;
    return true;
  }
  return false;
}
__device__ __forceinline__ bool hit_test(const RayParams& x, long long k, const double o[3], const double d[3],
                                         double tmin, double tmax, double* tout) {
  return hit_test_p(x, (double)__ldg(&x.v.pos[3 * k]), (double)__ldg(&x.v.pos[3 * k + 1]),
                    (double)__ldg(&x.v.pos[3 * k + 2]), o, d, tmin, tmax, tout);
}

__device__ __forceinline__ bool hit_less(double ta, long long ia, double tb, long long ib) {
  return ta < tb || (ta == tb && ia < ib);
}

// iterate a leaf's fragments (POFA range or POFL chain)
template <class F>
__device__ __forceinline__ void for_leaf(const RayParams& x, long long code, F&& f) {
  if (x.v.layout == 0) {
    const long long beg = __ldg(&x.v.offsets[code]);
    const long long cnt = __ldg(&x.v.counts[code]);
    for (long long k = beg; k < beg + cnt; ++k) f(k);
  } else {
    for (long long k = __ldg(&x.v.heads[code]); k >= 0; k = __ldg(&x.v.prev[k])) f(k);
  }
}

// visit the hits of one leaf in (t, index) order; visit(t, idx) -> false stops
template <class V>
__device__ bool leaf_hits(const RayParams& x, long long code, const double o[3], const double d[3], double tmin,
                          double tmax, Stats& st, V&& visit) {
  double bt[kHitBuf];
  long long bi[kHitBuf];
  int nb = 0;
  long long nh = 0, tested = 0;
  for_leaf(x, code, [&](long long k) {
    ++tested;
    double t;
    if (!hit_test(x, k, o, d, tmin, tmax, &t)) return;
    ++nh;
    // keep the kHitBuf smallest (t, idx), sorted
    if (nb == kHitBuf && !hit_less(t, k, bt[kHitBuf - 1], bi[kHitBuf - 1])) return;
    int j = nb < kHitBuf ? nb : kHitBuf - 1;
    while (j > 0 && hit_less(t, k, bt[j - 1], bi[j - 1])) {
      bt[j] = bt[j - 1];
      bi[j] = bi[j - 1];
      --j;
    }
    bt[j] = t;
    bi[j] = k;
    if (nb < kHitBuf) ++nb;
  });
  st.tested += tested;
  // deliver the hits in (t, index) order through ONE call site of visit (the
  // shading is inlined once): the buffered ones, then -- only for leaves with
  // more than kHitBuf hits -- an exact rescan selecting the next one each time
  double lt = 0.0;
  long long li = -1, delivered = 0;
  for (int q = 0;; ) {
    double ct;
    long long ci;
    if (q < nb) {
      ct = bt[q];
      ci = bi[q];
      ++q;
    } else if (delivered < nh) {
      double mt = 0.0;
      long long mi = -1;
      for_leaf(x, code, [&](long long k) {
        double t;
        if (!hit_test(x, k, o, d, tmin, tmax, &t)) return;
        if (!hit_less(lt, li, t, k)) return;
        if (mi < 0 || hit_less(t, k, mt, mi)) {
          mt = t;
          mi = k;
        }
      });
      if (mi < 0) break;
      ct = mt;
      ci = mi;
    } else {
      break;
    }
    if (!visit(ct, ci)) return false;
    lt = ct;
    li = ci;
    ++delivered;
  }
  return true;
}

// DFS over the occupancy pyramid, nearest child first (fhv/_ckern.pyx:548-633).
// visit_leaf(code) -> false stops.
// Stack entries pack (level, code): E = uint32_t when the octree has <= 9
// levels (27-bit codes, half the local-memory traffic of the DFS stack), else
// uint64_t.
template <class E>
struct StackCodec {
  static constexpr int kShift = sizeof(E) == 4 ? 27 : 58;
  static constexpr E kMask = (E)(((E)1 << kShift) - 1);
};

// one inner node of the DFS: children whose slabs the ray meets pushed far
// first, so the nearest (t_enter, child) pops next (fhv/_ckern.pyx:580-632)
template <class E>
__device__ __forceinline__ void expand_node(const RayParams& x, const double o[3], const double d[3], double tmin,
                                            double tmax, int level, unsigned long long code, E* stack, int& sp) {
  using SC = StackCodec<E>;
  const unsigned mask = __ldg(&x.v.pyramid[pyr_level_offset(level) + (long long)code]);
  if (mask == 0) return;
  const double half = __longlong_as_double((1022LL - level) << 52);  // 0.5 / 2^level, exact
  const double size = __dmul_rn(2.0, half);
  const double lo[3] = {__dmul_rn((double)compact3(code), size), __dmul_rn((double)compact3(code >> 1), size),
                        __dmul_rn((double)compact3(code >> 2), size)};
  // plane parameters for lo, lo+half, lo+2*half on each axis; the outer
  // plane of a side is only divided out when an occupied child lies on
  // that side (children with bit a = 0 use planes 0,1; = 1 use planes 1,2)
  double tp[3][3];
  double pl[3][3];
  const unsigned side_lo[3] = {mask & 0x55u, mask & 0x33u, mask & 0x0Fu};
  const unsigned side_hi[3] = {mask & 0xAAu, mask & 0xCCu, mask & 0xF0u};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    pl[a][0] = lo[a];
    pl[a][1] = __dadd_rn(lo[a], half);
    pl[a][2] = __dadd_rn(pl[a][1], half);
    const bool dz = d[a] == 0.0;
    tp[a][0] = (!dz && side_lo[a]) ? ddiv_z_sel(__dsub_rn(pl[a][0], o[a]), d[a]) : 0.0;
    tp[a][1] = !dz ? ddiv_z_sel(__dsub_rn(pl[a][1], o[a]), d[a]) : 0.0;
    tp[a][2] = (!dz && side_hi[a]) ? ddiv_z_sel(__dsub_rn(pl[a][2], o[a]), d[a]) : 0.0;
  }
  double cte[8];
  int cc[8];
  int nc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (!((mask >> c) & 1u)) continue;
    const int bx = c & 1, by = (c >> 1) & 1, bz = (c >> 2) & 1;
    double t0 = tmin, t1 = tmax;
    if (!slab_axis(o[0], d[0], pl[0][bx], pl[0][bx + 1], tp[0][bx], tp[0][bx + 1], t0, t1)) continue;
    if (!slab_axis(o[1], d[1], pl[1][by], pl[1][by + 1], tp[1][by], tp[1][by + 1], t0, t1)) continue;
    if (!slab_axis(o[2], d[2], pl[2][bz], pl[2][bz + 1], tp[2][bz], tp[2][bz + 1], t0, t1)) continue;
    if (t0 > t1) continue;
    int m = nc - 1;
    while (m >= 0 && (cte[m] > t0 || (cte[m] == t0 && cc[m] > c))) {
      cte[m + 1] = cte[m];
      cc[m + 1] = cc[m];
      --m;
    }
    cte[m + 1] = t0;
    cc[m + 1] = c;
    ++nc;
  }
  const E lvl = (E)((E)(level + 1) << SC::kShift);
  for (int j = nc - 1; j >= 0; --j) stack[sp++] = lvl | (E)(code * 8ull + (unsigned long long)cc[j]);
}

// ray interval [tmin, tmax] (traverse_octree's ray.t_min / t_max; the image
// kernels use [0, tmax])
template <class E, class V>
__device__ void traverse_range(const RayParams& x, const double o[3], const double d[3], double tmin, double tmax,
                               Stats& st, V&& visit_leaf) {
  using SC = StackCodec<E>;
  const double zero3[3] = {0.0, 0.0, 0.0}, one3[3] = {1.0, 1.0, 1.0};
  double te;
  if (!slab_box(o, d, zero3, one3, tmin, tmax, &te)) return;
  const int L = x.v.levels;
  E stack[kStack];
  int sp = 0;
  stack[sp++] = (E)0;  // level 0, code 0
  while (sp > 0) {
    const E e = stack[--sp];
    const int level = (int)(e >> SC::kShift);
    const unsigned long long code = (unsigned long long)(e & SC::kMask);
    if (level == L) {
      st.visited++;
      if (!visit_leaf((long long)code)) return;
      continue;
    }
    expand_node<E>(x, o, d, tmin, tmax, level, code, stack, sp);
  }
}

template <class E, class V>
__device__ __forceinline__ void traverse(const RayParams& x, const double o[3], const double d[3], double tmax,
                                         Stats& st, V&& visit_leaf) {
  traverse_range<E>(x, o, d, 0.0, tmax, st, visit_leaf);
}

// _transmit (fhv/_ckern.pyx:326-435)
template <class E>
__device__ double transmit(const RayParams& x, const double p[3], int li, long long ex_obj, long long ex_cell,
                           Stats& st) {
  double l[3], tmax;
  if (x.s.light_kind[li] == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) l[k] = x.s.light_vec[3 * li + k];
    tmax = __longlong_as_double(0x7ff0000000000000ll);
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) l[k] = __dsub_rn(x.s.light_vec[3 * li + k], p[k]);
    const double len = __dsqrt_rn(plain3(l[0], l[1], l[2]));
    if (len == 0.0) return 1.0;
    const Recip rl = recip_of(len);
#pragma unroll
    for (int k = 0; k < 3; ++k) l[k] = div_rn(l[k], rl);
    tmax = len;
  }
  double o[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) o[k] = __dadd_rn(p[k], __dmul_rn(x.eps, l[k]));
  double tau = 1.0;
  traverse<E>(x, o, l, tmax, st, [&](long long code) {
    return leaf_hits(x, code, o, l, 0.0, tmax, st, [&](double, long long k) {
      if ((long long)__ldg(&x.v.obj[k]) == ex_obj && code == ex_cell) return true;
      tau = __dmul_rn(tau, __dsub_rn(1.0, x.s.alpha[__ldg(&x.v.mat[k])]));
      return tau != 0.0;
    });
  });
  return tau;
}

// _shade_hit (fhv/_ckern.pyx:438-523): plain f64 Blinn-Phong.  kMode is the
// ray-cast mode as a template parameter: only mode 2 (shadows) instantiates
// the second (shadow) traversal and its stack, which keeps the stack frame of
// the primary-ray kernels of modes 0 / 1 small.
template <int kMode, class E>
__device__ void shade_hit(const RayParams& x, long long i, long long leaf, Stats& st, double out[3]) {
  const double p[3] = {(double)x.v.pos[3 * i], (double)x.v.pos[3 * i + 1], (double)x.v.pos[3 * i + 2]};
  const double n[3] = {(double)x.v.nrm[3 * i], (double)x.v.nrm[3 * i + 1], (double)x.v.nrm[3 * i + 2]};
  const long long m = x.v.mat[i];
  const double* dif = x.s.diffuse + 3 * m;
  const double* spc = x.s.specular + 3 * m;
  const double shin = x.s.shininess[m];
  double v[3] = {__dsub_rn(x.eye[0], p[0]), __dsub_rn(x.eye[1], p[1]), __dsub_rn(x.eye[2], p[2])};
  const double vl = __dsqrt_rn(plain3(v[0], v[1], v[2]));
  // one reciprocal per normalised vector, each quotient still __ddiv_rn's
  // (fhv_common.cuh div_rn)
  const Recip rvl = recip_of(vl);
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = vl > 0.0 ? div_rn(v[k], rvl) : 0.0;
  double r = 0.0, g = 0.0, b = 0.0;
  for (int li = 0; li < x.s.n_lights; ++li) {
    double l[3];
    if (x.s.light_kind[li] == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) l[k] = x.s.light_vec[3 * li + k];
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) l[k] = __dsub_rn(x.s.light_vec[3 * li + k], p[k]);
      const double ll = __dsqrt_rn(plain3(l[0], l[1], l[2]));
      const Recip rll = recip_of(ll);
#pragma unroll
      for (int k = 0; k < 3; ++k) l[k] = ll > 0.0 ? div_rn(l[k], rll) : 0.0;
    }
    double h[3] = {__dadd_rn(l[0], v[0]), __dadd_rn(l[1], v[1]), __dadd_rn(l[2], v[2])};
    const double hl = __dsqrt_rn(plain3(h[0], h[1], h[2]));
    const Recip rhl = recip_of(hl);
#pragma unroll
    for (int k = 0; k < 3; ++k) h[k] = hl > 0.0 ? div_rn(h[k], rhl) : 0.0;
    double ndl = __dadd_rn(__dadd_rn(__dmul_rn(n[0], l[0]), __dmul_rn(n[1], l[1])), __dmul_rn(n[2], l[2]));
    if (ndl < 0.0) ndl = 0.0;
    double ndh = __dadd_rn(__dadd_rn(__dmul_rn(n[0], h[0]), __dmul_rn(n[1], h[1])), __dmul_rn(n[2], h[2]));
    if (ndh < 0.0) ndh = 0.0;
    double tau = 1.0;
    if (kMode == 2) tau = transmit<E>(x, p, li, (long long)x.v.obj[i], leaf, st);
    const double sp = pow(ndh, shin);
    const double* amb = x.s.light_ambient + 3 * li;
    const double* col = x.s.light_color + 3 * li;
    r = __dadd_rn(r, __dmul_rn(amb[0], dif[0]));
    g = __dadd_rn(g, __dmul_rn(amb[1], dif[1]));
    b = __dadd_rn(b, __dmul_rn(amb[2], dif[2]));
    const double tn = __dmul_rn(tau, ndl), ts = __dmul_rn(tau, sp);
    r = __dadd_rn(r, __dmul_rn(__dmul_rn(tn, dif[0]), col[0]));
    g = __dadd_rn(g, __dmul_rn(__dmul_rn(tn, dif[1]), col[1]));
    b = __dadd_rn(b, __dmul_rn(__dmul_rn(tn, dif[2]), col[2]));
    r = __dadd_rn(r, __dmul_rn(__dmul_rn(ts, spc[0]), col[0]));
    g = __dadd_rn(g, __dmul_rn(__dmul_rn(ts, spc[1]), col[1]));
    b = __dadd_rn(b, __dmul_rn(__dmul_rn(ts, spc[2]), col[2]));
  }
  out[0] = r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
  out[1] = g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g);
  out[2] = b < 0.0 ? 0.0 : (b > 1.0 ? 1.0 : b);
}

// primary_rays (fhv/raycast.py:148-172), elementwise numpy semantics
__device__ __forceinline__ void camera_ray(const RayParams& x, long long k, double o[3], double d[3]) {
  const long long iy = k / x.W, ix = k - iy * x.W;
  const double nx = __dsub_rn(__dmul_rn(ddiv_z(__dadd_rn((double)ix, 0.5), (double)x.W), 2.0), 1.0);
  const double ny = __dsub_rn(1.0, __dmul_rn(ddiv_z(__dadd_rn((double)iy, 0.5), (double)x.H), 2.0));
  if (!x.persp) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double hw = __dmul_rn(x.half_w, x.rr[c]), hh = __dmul_rn(x.half_h, x.uu[c]);
      o[c] = __dadd_rn(__dadd_rn(__dadd_rn(x.eye[c], __dmul_rn(nx, hw)), __dmul_rn(ny, hh)), __dmul_rn(x.near_, x.ff[c]));
      d[c] = x.ff[c];
    }
  } else {
    const double ta = __dmul_rn(x.t, x.aspect);
    double v[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      v[c] = __dadd_rn(__dadd_rn(x.ff[c], __dmul_rn(nx, __dmul_rn(ta, x.rr[c]))), __dmul_rn(ny, __dmul_rn(x.t, x.uu[c])));
    const double len = __dsqrt_rn(plain3(v[0], v[1], v[2]));
    const Recip rl = recip_of(len);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      d[c] = div_rn(v[c], rl);
      o[c] = x.eye[c];
    }
  }
}

#ifndef FHV_RAY_MINB
#define FHV_RAY_MINB 4  // resident 128-thread CTAs per SM the ray kernel is register-budgeted for
#endif
template <int kMode, class E>
__global__ void __launch_bounds__(128, FHV_RAY_MINB) k_raycast(RayParams x) {
  Stats st = {0, 0, 0, 0};
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  // camera rays: a warp takes an 8x4 pixel tile instead of 32 pixels of one
  // row (coherent rays walk similar octree nodes -> less divergence); the
  // band [start, end) must be whole 4-row strips of a width divisible by 8
  const bool tiled = x.from_camera && x.W % 8 == 0 && x.start % (4 * x.W) == 0 && x.end % (4 * x.W) == 0;
  const long long tiles_per_row = x.W / 8;
  // warps fetch 32-ray tiles from a global ticket (ray costs vary by orders
  // of magnitude: dynamic fetching instead of a static stride evens the tail)
  // list mode: the rays the packet kernel handed off (count on the device)
  const long long n_rays = x.ray_list ? (long long)*x.ray_list_n : x.end - x.start;
  while (true) {
    unsigned long long t = 0;
    if (lane_id() == 0) t = atomicAdd(x.tile_ticket, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((long long)t * 32 >= n_rays) break;
    const long long kk = x.start + (long long)t * 32 + lane_id();
    if (kk >= x.start + n_rays) continue;
    long long k = kk;
    if (x.ray_list) {
      k = x.ray_list[kk - x.start];
    } else if (tiled) {
      const long long i = kk - x.start, tile = i >> 5, l = i & 31;
      const long long ty = tile / tiles_per_row, tx = tile - ty * tiles_per_row;
      k = x.start + (ty * 4 + (l >> 3)) * x.W + tx * 8 + (l & 7);
    }
    double o[3], d[3];
    if (x.from_camera) {
      camera_ray(x, k, o, d);
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        o[c] = x.origins[3 * k + c];
        d[c] = x.dirs[3 * k + c];
      }
    }
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, acc = 0.0;
    bool any_hit = false;
    long long first_obj = -1;
    traverse<E>(x, o, d, inf, st, [&](long long code) {
      bool stop = false;
      leaf_hits(x, code, o, d, 0.0, inf, st, [&](double, long long i) {
        st.hits++;
        if (first_obj < 0) first_obj = (long long)x.v.obj[i];
        double col[3];
        if (kMode == 0) {
          shade_hit<kMode, E>(x, i, code, st, col);
          c0 = col[0];
          c1 = col[1];
          c2 = col[2];
          acc = 1.0;
          any_hit = true;
          stop = true;
          return false;
        }
        const double a = x.s.alpha[x.v.mat[i]];
        shade_hit<kMode, E>(x, i, code, st, col);
        const double tc = __dmul_rn(__dsub_rn(1.0, acc), a);
        c0 = __dadd_rn(c0, __dmul_rn(tc, col[0]));
        c1 = __dadd_rn(c1, __dmul_rn(tc, col[1]));
        c2 = __dadd_rn(c2, __dmul_rn(tc, col[2]));
        acc = __dadd_rn(acc, tc);
        any_hit = true;
        return true;
      });
      if (stop) return false;
      if (x.cutoff >= 0.0 && acc >= x.cutoff) {
        st.early++;
        return false;
      }
      return true;
    });
    double4 px;
    if (kMode == 0) {
      px = any_hit ? make_double4(c0, c1, c2, 1.0) : make_double4(x.bg[0], x.bg[1], x.bg[2], x.bg[3]);
    } else {
      const double ra = __dsub_rn(1.0, acc);
      px.x = __dadd_rn(c0, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[0]));
      px.y = __dadd_rn(c1, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[1]));
      px.z = __dadd_rn(c2, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[2]));
      px.w = __dadd_rn(acc, __dmul_rn(ra, x.bg[3]));
    }
    reinterpret_cast<double4*>(x.out_rgba)[k] = px;
    if (x.out_ids && first_obj >= 0) x.out_ids[k] = (int32_t)first_obj;
  }
  unsigned long long v[4] = {st.visited, st.tested, st.hits, st.early};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
  }
  if (lane_id() == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (v[q]) atomicAdd(reinterpret_cast<unsigned long long*>(&x.counters[q]), v[q]);
  }
}

// ---------------------------------------------------------------------------
// Packet ray cast (camera rays, modes 0 / 1): one warp walks the octree ONCE
// for its 8x4 pixel tile.
//
// The DFS stack lives in shared memory and each entry carries the mask of the
// lanes whose ray reached that node, so every node is expanded by the whole
// warp in lock-step and every leaf's fragment list is walked once, its loads
// broadcast to the lanes that test it.  The warp pushes the children in ONE
// shared order: for rays leaving a common eye (perspective) or along a common
// direction (orthographic) the children a ray meets form a chain across the
// node's three centre planes, and ordering them by (child XOR s) -- s = the
// eye's / the rays' entry side of each plane -- is a front-to-back order for
// every ray of the tile.  Each lane checks at every node that the shared
// order of the children IT meets is its own (t_enter, child) order (the
// reference's insertion sort, fhv/_ckern.pyx:580-632); where it is not (ties
// of rounded entry distances) the lane's children are pushed in its own order
// instead, above the shared ones (see the node code), so every ray's visit
// sequence -- and with it the image and RaycastStats -- is the reference's.
// The slab decisions use certified f32 plane parameters, with the exact f64
// expansion (exact_node) wherever a decision falls inside the error margin.
// A push that would overflow the stack hands the affected rays to the
// per-ray kernel (k_raycast in list mode), which re-runs them from scratch.
//
// Shading is deferred: a delivered hit's compositing weight (1 - acc) * alpha
// needs only the material alphas, so each lane queues (pool index, weight)
// records in hit order; at the tile's end (or when a queue fills) the warp
// shades all queued hits 32 wide and each lane accumulates its colour in
// queue order (pkt_flush).
#ifndef FHV_PKT_HITS
#define FHV_PKT_HITS 4  // per-lane buffered hits per leaf (more: exact rescans)
#endif
#ifndef FHV_PKT_MINB
#define FHV_PKT_MINB 4  // CTAs per SM the opaque-nearest packet kernel is register-budgeted for (128)
#endif
#ifndef FHV_PKT_MINB_T
#define FHV_PKT_MINB_T 4  // the compositing modes (3: 166 registers without spills -- C2 1.76 -> 1.73 ms but the
                          // 80-layer C4 view 32.5 -> 36.4 ms; 2: C2 1.94 ms)
#endif
constexpr int kPktHits = FHV_PKT_HITS;
#ifndef FHV_PKT_BUF
#define FHV_PKT_BUF 12  // deferred (pool index, weight) records per lane before a shading flush
#endif
constexpr int kPktBuf = FHV_PKT_BUF;
constexpr int kPktWarps = 4;  // 128-thread CTAs

// shared stack: 7 per level for the shared order plus room for the lanes
// that take their own order at a node (ties); a push that would not fit hands
// those lanes to the per-ray kernel instead
#ifndef FHV_PKT_STACK
#define FHV_PKT_STACK (16 * kRayMaxLevels + 8)  // tests build a tiny one to force the hand-off path
#endif
constexpr int kPktStack = FHV_PKT_STACK;
template <class E>
struct PktShared {
  E node[kPktStack];
  unsigned lanes[kPktStack];
  int slot_idx[32 * kPktBuf];
  double col[32][3];
  int ri[kPktBuf][32];     // each lane's delivered hits in order: pool index ...
  double rw[kPktBuf][32];  // ... and compositing weight (1 - acc) * alpha
};

// a leaf's fragments in pool order (POFA range) or chain order (POFL);
// warp-uniform walk
template <class F>
__device__ __forceinline__ void pkt_for_leaf(const RayParams& x, long long code, F&& f) {
  if (x.v.layout == 0) {
    const int beg = (int)__ldg(&x.v.offsets[code]);
    const int cnt = (int)__ldg(&x.v.counts[code]);
    for (int k = beg; k < beg + cnt; ++k) f(k);
  } else {
    for (int k = __ldg(&x.v.heads[code]); k >= 0; k = __ldg(&x.v.prev[k])) f(k);
  }
}

// sorted insertion into the register buffer (compile-time indices only: the
// candidate walks up, swapping with every larger entry; the largest falls off)
__device__ __forceinline__ void pkt_insert(double t, int k, double bt[kPktHits], int bi[kPktHits], int& nb) {
  if (nb == 0) {  // a ray's first hit in the leaf (the common case): no compare-and-shift
    bt[0] = t;
    bi[0] = k;
    nb = 1;
    return;
  }
  if (nb == kPktHits && !hit_less(t, k, bt[kPktHits - 1], bi[kPktHits - 1])) return;
#pragma unroll
  for (int q = 0; q < kPktHits; ++q) {
    if (q < nb) {
      if (hit_less(t, k, bt[q], bi[q])) {
        const double ut = bt[q];
        const int uk = bi[q];
        bt[q] = t;
        bi[q] = k;
        t = ut;
        k = uk;
      }
    } else if (q == nb) {
      bt[q] = t;
      bi[q] = k;
    }
  }
  if (nb < kPktHits) ++nb;
}

// the kPktHits smallest (t, k) of the leaf above (lt, li) for lanes with `on`;
// returns how many hits lie above the bound.  The fragment walk is warp-uniform.
#ifndef FHV_PKT_PIPE
#define FHV_PKT_PIPE 1  // 0: plain POFL chain loop (A/B switch; pipelined: C2 2.14 -> 1.97 ms)
#endif
template <bool kBound>
__device__ __forceinline__ int pkt_collect(const RayParams& x, long long code, bool on, const double o[3],
                                           const double d[3], double lt, int li, double bt[kPktHits],
                                           int bi[kPktHits], int& nb, unsigned& tested) {
  int nh = 0;
  nb = 0;
  auto one = [&](int k, float fx, float fy, float fz) {
    if (!on) return;
    ++tested;
    double t;
    if (!hit_test_p(x, (double)fx, (double)fy, (double)fz, o, d, 0.0, __longlong_as_double(0x7ff0000000000000ll),
                    &t))
      return;
    if (kBound && !hit_less(lt, li, t, k)) return;
    ++nh;
    pkt_insert(t, k, bt, bi, nb);
  };
  const float* P = x.v.pos;
  if (x.v.layout == 0) {
    const int beg = (int)__ldg(&x.v.offsets[code]);
    const int end = beg + (int)__ldg(&x.v.counts[code]);
    // a contiguous range: the broadcast loads hit L1 (pipelining them measured
    // slower here, C5 4.19 -> 4.34 ms per view)
    for (int k = beg; k < end; ++k) one(k, __ldg(&P[3 * k]), __ldg(&P[3 * k + 1]), __ldg(&P[3 * k + 2]));

  } else {
#if FHV_PKT_PIPE
    // the chain link and position of the next fragment are in flight during
    // this one's test (the chain itself stays a dependent walk)
    int k = __ldg(&x.v.heads[code]);
    int kn = -1;
    float fx = 0.f, fy = 0.f, fz = 0.f;
    if (k >= 0) {
      kn = __ldg(&x.v.prev[k]);
      fx = __ldg(&P[3 * k]);
      fy = __ldg(&P[3 * k + 1]);
      fz = __ldg(&P[3 * k + 2]);
    }
    while (k >= 0) {
      int kn2 = -1;
      float gx = 0.f, gy = 0.f, gz = 0.f;
      if (kn >= 0) {
        kn2 = __ldg(&x.v.prev[kn]);
        gx = __ldg(&P[3 * kn]);
        gy = __ldg(&P[3 * kn + 1]);
        gz = __ldg(&P[3 * kn + 2]);
      }
      one(k, fx, fy, fz);
      k = kn;
      kn = kn2;
      fx = gx;
      fy = gy;
      fz = gz;
    }
#else
    for (int k = __ldg(&x.v.heads[code]); k >= 0; k = __ldg(&x.v.prev[k]))
      one(k, __ldg(&P[3 * k]), __ldg(&P[3 * k + 1]), __ldg(&P[3 * k + 2]));
#endif
  }
  return nh;
}

#ifndef FHV_PKT_SHADE_NOINLINE
#define FHV_PKT_SHADE_NOINLINE 0
#endif
#if FHV_PKT_SHADE_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void pkt_shade(const RayParams& x, int i, long long leaf, double col[3]) {
  Stats dummy = {0, 0, 0, 0};
  shade_hit<1, uint32_t>(x, i, leaf, dummy, col);  // modes 0 / 1: no shadow traversal
}

// shade every lane's queued records warp-wide (lane-major slots, one slot
// per lane per round) and composite each lane's in queue order
template <int kMode, class Sh>
__device__ __forceinline__ void pkt_flush(const RayParams& x, Sh& S, int& nbuf, double& c0, double& c1, double& c2) {
  const unsigned full = 0xffffffffu, lane = lane_id();
  int base = nbuf;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(full, base, off);
    if ((int)lane >= off) base += v;
  }
  const int total = __shfl_sync(full, base, 31);
  base -= nbuf;
  for (int q = 0; q < nbuf; ++q) S.slot_idx[base + q] = S.ri[q][lane];
  __syncwarp();
  for (int r0 = 0; r0 < total; r0 += 32) {
    const int j = r0 + (int)lane;
    if (j < total) {
      double col[3];
      pkt_shade(x, S.slot_idx[j], -1, col);
      S.col[lane][0] = col[0];
      S.col[lane][1] = col[1];
      S.col[lane][2] = col[2];
    }
    __syncwarp();
    const int q0 = base > r0 ? base : r0;
    const int q1 = (base + nbuf) < (r0 + 32) ? (base + nbuf) : (r0 + 32);
    for (int q = q0; q < q1; ++q) {
      const double* col = S.col[q - r0];
      if (kMode == 0) {
        c0 = col[0];
        c1 = col[1];
        c2 = col[2];
      } else {
        const double tc = S.rw[q - base][lane];
        c0 = __dadd_rn(c0, __dmul_rn(tc, col[0]));
        c1 = __dadd_rn(c1, __dmul_rn(tc, col[1]));
        c2 = __dadd_rn(c2, __dmul_rn(tc, col[2]));
      }
    }
    __syncwarp();
  }
  nbuf = 0;
}

// one inner node for one ray, exactly as expand_node (fhv/_ckern.pyx:580-632):
// bits 0-7 the children hit, bit 8 set when their (t_enter, child) order is
// not the shared order s, bits 9-12 their count, bits 13.. the children in
// that order (3 bits each).  Out of line: the packet kernel's rare path.
__device__ __noinline__ unsigned long long exact_node(double o0, double o1, double o2, double d0, double d1,
                                                      double d2, int level, unsigned long long code, unsigned mask,
                                                      unsigned s) {
  const double o[3] = {o0, o1, o2}, d[3] = {d0, d1, d2};
  const double half = __longlong_as_double((1022LL - level) << 52);
  const double size = __dmul_rn(2.0, half);
  double pl[3][3], tp[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    pl[a][0] = __dmul_rn((double)compact3(code >> a), size);
    pl[a][1] = __dadd_rn(pl[a][0], half);
    pl[a][2] = __dadd_rn(pl[a][1], half);
#pragma unroll
    for (int k = 0; k < 3; ++k) tp[a][k] = d[a] != 0.0 ? ddiv_z(__dsub_rn(pl[a][k], o[a]), d[a]) : 0.0;
  }
  double cte[8];
  int cc[8];
  int nc = 0;
  unsigned hits = 0;
  for (int c = 0; c < 8; ++c) {
    if (!((mask >> c) & 1u)) continue;
    double t0 = 0.0, t1 = __longlong_as_double(0x7ff0000000000000ll);
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int bit = (c >> a) & 1;
      if (ok) ok = slab_axis(o[a], d[a], pl[a][bit], pl[a][bit + 1], tp[a][bit], tp[a][bit + 1], t0, t1);
    }
    if (!ok || t0 > t1) continue;
    hits |= 1u << c;
    int m = nc - 1;
    while (m >= 0 && (cte[m] > t0 || (cte[m] == t0 && cc[m] > c))) {
      cte[m + 1] = cte[m];
      cc[m + 1] = cc[m];
      --m;
    }
    cte[m + 1] = t0;
    cc[m + 1] = c;
    ++nc;
  }
  unsigned long long seq = 0;
  bool irr = false;
  for (int q = 0; q < nc; ++q) {
    seq |= (unsigned long long)cc[q] << (3 * q);
    if (q > 0 && ((unsigned)cc[q] ^ s) < ((unsigned)cc[q - 1] ^ s)) irr = true;
  }
  return (unsigned long long)hits | ((unsigned long long)irr << 8) | ((unsigned long long)nc << 9) | (seq << 13);
}

template <int kMode, class E>
__global__ void __launch_bounds__(32 * kPktWarps, kMode == 0 ? FHV_PKT_MINB : FHV_PKT_MINB_T) k_raycast_packet(RayParams x) {
  using SC = StackCodec<E>;
  __shared__ PktShared<E> shm[kPktWarps];
  PktShared<E>& S = shm[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  const unsigned full = 0xffffffffu;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int L = x.v.levels;
  const long long tiles_per_row = x.W / 8;
  const long long n_tiles = (x.end - x.start) / 32;
  // totals of the rays this thread finished inside the packet
  unsigned long long tv = 0, tt = 0, th = 0, te = 0;
  while (true) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(x.tile_ticket, 1ull);
    tk = __shfl_sync(full, tk, 0);
    if ((long long)tk >= n_tiles) break;
    const long long ty = (long long)tk / tiles_per_row, tx = (long long)tk - ty * tiles_per_row;
    const long long k = x.start + (ty * 4 + (lane >> 3)) * x.W + tx * 8 + (lane & 7);
    double o[3], d[3];
    camera_ray(x, k, o, d);
    // certified f32 slab parameters: t(pl) ~ fma(pl, inv32, c32) with
    // inv32 = 1/d (two f32 roundings), c32 = -o * inv32 (one): for pl in
    // [0, 1], |t - t_exact| <= 2^-23 |t| + 2^-24 (|t| + |c32|) <= e32; a
    // lane with a zero direction component takes exact_node at every node
    float inv32[3], c32[3], e32 = 0.0f;
    bool lane_exact = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lane_exact = lane_exact || d[a] == 0.0;
      inv32[a] = __frcp_rn((float)d[a]);
      c32[a] = (float)__dmul_rn(-o[a], (double)inv32[a]);
      e32 = fmaxf(e32, 0x1.0p-22f * (fabsf(inv32[a]) + fabsf(c32[a])));
    }
    lane_exact = lane_exact || !(e32 < 0x1.0p-8f);  // huge / non-finite parameters
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, acc = 0.0;
    bool any_hit = false;
    int first_obj = -1;
    unsigned rv = 0, rt = 0, rh = 0, re = 0;  // this ray's RaycastStats
    int nbuf = 0;                             // queued (index, weight) records
    // root slab (slab_box over [0,1]^3)
    bool in_root;
    {
      const double zero3[3] = {0.0, 0.0, 0.0}, one3[3] = {1.0, 1.0, 1.0};
      double t_e;
      in_root = slab_box(o, d, zero3, one3, 0.0, inf, &t_e);
    }
    unsigned active = __ballot_sync(full, in_root);
    unsigned irregular = 0;
    int sp = 0;
    if (active) {
      if (lane == 0) {
        S.node[0] = (E)0;
        S.lanes[0] = active;
      }
      sp = 1;
    }
    __syncwarp();
    bool need_flush = false;
    while (true) {
    while (sp > 0 && active && !need_flush) {
      --sp;
      const E e = S.node[sp];
      const unsigned M = S.lanes[sp] & active;
      __syncwarp();
      if (!M) continue;
      const bool on = (M >> lane) & 1u;
      const int level = (int)(e >> SC::kShift);
      const unsigned long long code = (unsigned long long)(e & SC::kMask);
      if (level == L) {
        // ---- leaf: hits in (t, index) order, shaded warp-wide
        if (on) ++rv;
        double bt[kPktHits];
        int bi[kPktHits];
        int nb = 0, left;
        if (kMode == 0) {
          // the nearest hit only
          int nh = 0;
          pkt_for_leaf(x, (long long)code, [&](int k) {
            if (!on) return;
            ++rt;
            double t;
            if (!hit_test(x, k, o, d, 0.0, inf, &t)) return;
            if (nh++ == 0 || hit_less(t, k, bt[0], bi[0])) {
              bt[0] = t;
              bi[0] = k;
            }
          });
          left = nb = nh > 0 ? 1 : 0;
        } else {
          left = pkt_collect<false>(x, (long long)code, on, o, d, -inf, -1, bt, bi, nb, rt);
        }
        // deliver in (t, index) order: the weight (1 - acc) * alpha and acc
        // need only the materials' alphas, so shading is deferred -- the
        // (index, weight) records queue per lane and are shaded warp-wide
        // at flushes (pkt_flush), composited in the same order
        bool stop = false;
        while (true) {
          const int take = left < nb ? left : nb;
#pragma unroll
          for (int q = 0; q < kPktHits; ++q) {
            if (q < take) {
              const int i = bi[q];
              ++rh;
              if (first_obj < 0) first_obj = (int)__ldg(&x.v.obj[i]);
              any_hit = true;
              S.ri[nbuf][lane] = i;
              if (kMode == 0) {
                acc = 1.0;
                stop = true;
              } else {
                const double a = x.s.alpha[__ldg(&x.v.mat[i])];
                const double tc = __dmul_rn(__dsub_rn(1.0, acc), a);
                acc = __dadd_rn(acc, tc);
                S.rw[nbuf][lane] = tc;
              }
              ++nbuf;
            }
          }
          left -= take;
          if (__any_sync(full, nbuf > kPktBuf - kPktHits)) {
            if (kMode == 0 || !__any_sync(full, left > 0)) {
              need_flush = true;  // flushed by the traversal loop's single flush site
              break;
            }
            pkt_flush<kMode>(x, S, nbuf, c0, c1, c2);  // mid-leaf (a ray with more hits than the buffer)
          }
          if (kMode == 0 || !__any_sync(full, left > 0)) break;
          // more hits than the buffer held: the next ones above the last delivered
          double lt = -inf;
          int li = -1;
#pragma unroll
          for (int q = 0; q < kPktHits; ++q)
            if (q == take - 1) {
              lt = bt[q];
              li = bi[q];
            }
          unsigned dummy_tested = 0;
          pkt_collect<true>(x, (long long)code, left > 0, o, d, lt, li, bt, bi, nb, dummy_tested);
        }
        bool done = false;
        if (on) {
          if (stop) {
            done = true;
          } else if (x.cutoff >= 0.0 && acc >= x.cutoff) {
            ++re;
            done = true;
          }
        }
        active &= ~__ballot_sync(full, done);
        continue;
      }
      // ---- inner node: expand_node for every lane in M, one shared child order
      const unsigned mask = __ldg(&x.v.pyramid[pyr_level_offset(level) + (long long)code]);
      if (mask == 0) continue;
      // shared order: the eye's (perspective) / the rays' entry (orthographic)
      // side of each centre plane; any choice is exact (each lane checks it)
      const float half32 = __int_as_float((126 - level) << 23);  // 0.5 / 2^level, exact
      const float size32 = 2.0f * half32;
      float pl[3][3];
      unsigned s = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        pl[a][0] = (float)compact3(code >> a) * size32;  // exact: dyadic, < 2^24 units of 2^-level
        pl[a][1] = pl[a][0] + half32;
        pl[a][2] = pl[a][1] + half32;
        const bool hi_first = x.persp ? ((float)x.eye[a] > pl[a][1]) : (x.ff[a] < 0.0);
        s |= (hi_first ? 1u : 0u) << a;
      }
      // perm_mask bit jj = child jj ^ s occupied (the mask's bits permuted by XOR s)
      unsigned perm_mask = mask;
      if (s & 1u) perm_mask = ((perm_mask & 0x55u) << 1) | ((perm_mask >> 1) & 0x55u);
      if (s & 2u) perm_mask = ((perm_mask & 0x33u) << 2) | ((perm_mask >> 2) & 0x33u);
      if (s & 4u) perm_mask = ((perm_mask & 0x0Fu) << 4) | ((perm_mask >> 4) & 0x0Fu);
      // this lane's children from the certified f32 slab parameters (within
      // e32 of expand_node's f64 values); decisions closer than the margin --
      // and lanes with a d == 0 axis -- take exact_node
      unsigned hits = 0, seq = 0;
      int nk = 0;
      bool irr = false;
      if (on) {
        bool unsure = lane_exact;
        if (!unsure) {
          float en[3][2], ex[3][2];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float t0 = __fmaf_rn(pl[a][0], inv32[a], c32[a]);
            const float t1 = __fmaf_rn(pl[a][1], inv32[a], c32[a]);
            const float t2 = __fmaf_rn(pl[a][2], inv32[a], c32[a]);
            const bool pos = inv32[a] > 0.0f;
            const float e0 = pos ? t0 : t1, x0 = pos ? t1 : t0, e1 = pos ? t1 : t2, x1 = pos ? t2 : t1;
            const bool sa = (s >> a) & 1u;
            en[a][0] = sa ? e1 : e0;
            ex[a][0] = sa ? x1 : x0;
            en[a][1] = sa ? e0 : e1;
            ex[a][1] = sa ? x0 : x1;
          }
          const float m2 = 2.5f * e32;  // two approximations, each within e32
          bool have_next = false;
          float nt = 0.0f;
          // occupied children, far-first in the shared order (a warp-uniform
          // loop over set bits; the planes selected per bit)
          for (unsigned pm = perm_mask; pm; ) {
            const int jj = 31 - __clz(pm);
            pm &= ~(1u << jj);
            const int c = jj ^ (int)s;
            const bool jx = jj & 1, jy = (jj >> 1) & 1, jz = (jj >> 2) & 1;
            const float t0 = fmaxf(fmaxf(fmaxf(0.0f, jx ? en[0][1] : en[0][0]), jy ? en[1][1] : en[1][0]),
                                   jz ? en[2][1] : en[2][0]);
            const float t1 = fminf(fminf(jx ? ex[0][1] : ex[0][0], jy ? ex[1][1] : ex[1][0]), jz ? ex[2][1] : ex[2][0]);
            const float gap = t1 - t0;
            if (gap > m2) {
              hits |= 1u << c;
              if (have_next) {
                const float dn = nt - t0;
                if (!(dn > m2)) {
                  if (dn < -m2) irr = true;
                  else unsure = true;
                }
              }
              have_next = true;
              nt = t0;
            } else if (!(gap < -m2)) {
              unsure = true;  // NaN / inf included
            }
          }
        }
        if (unsure || irr) {
          const unsigned long long r = exact_node(o[0], o[1], o[2], d[0], d[1], d[2], level, code, mask, s);
          hits = (unsigned)(r & 0xffu);
          irr = (r >> 8) & 1u;
          nk = (int)((r >> 9) & 0xfu);
          seq = (unsigned)(r >> 13);
        }
      }
      // children in reverse shared order: pushed far-first, so the shared
      // order pops next.  The shared pushes alone stay below 7 L + 1 entries;
      // own-order push sets (ties) can fill the stack: a push that would not
      // fit hands every lane of this node to the per-ray kernel instead
      const E lvl = (E)((E)(level + 1) << SC::kShift);
      const int sp0 = sp;
      if (sp + __popc(perm_mask) > kPktStack) {
        irregular |= M;
        active &= ~M;
        continue;
      }
      for (unsigned pm = perm_mask; pm; ) {
        const int jj = 31 - __clz(pm);
        pm &= ~(1u << jj);
        const int c = jj ^ (int)s;
        const unsigned b = __ballot_sync(full, (hits >> c) & 1u);
        if (b) {
          if (lane == 0) {
            S.node[sp] = lvl | (E)(code * 8ull + (unsigned long long)c);
            S.lanes[sp] = b;
          }
          ++sp;
        }
      }
      const unsigned bad = __ballot_sync(full, irr);
      if (bad) {
        // lanes whose own (t_enter, child) order differs from the shared one
        // (rounded entry distances tie): drop them from this node's shared
        // pushes and push their children in their own order (exact_node's
        // insertion sort), one push set per group of lanes with the same
        // order -- above the shared entries, so each group's subtrees pop
        // first and every lane still sees exactly its own preorder
        const unsigned key = seq;
        if (lane == 0)
          for (int q = sp0; q < sp; ++q) S.lanes[q] &= ~bad;
        if (lane == 0) atomicAdd(x.own_order_n, (unsigned long long)__popc(bad));
        unsigned pend = bad;
        while (pend) {
          const int leader = __ffs(pend) - 1;
          const unsigned kl = __shfl_sync(full, key, leader);
          const int nl = __shfl_sync(full, nk, leader);
          const unsigned grp = __ballot_sync(full, ((pend >> lane) & 1u) && key == kl && nk == nl);
          pend &= ~grp;
          if (sp + nl > kPktStack) {  // no room: the per-ray kernel takes these rays
            irregular |= grp;
            active &= ~grp;
            continue;
          }
          for (int q = nl - 1; q >= 0; --q) {
            if (lane == 0) {
              S.node[sp] = lvl | (E)(code * 8ull + (unsigned long long)((kl >> (3 * q)) & 7u));
              S.lanes[sp] = grp;
            }
            ++sp;
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    if (__any_sync(full, nbuf > 0)) pkt_flush<kMode>(x, S, nbuf, c0, c1, c2);
    if (!need_flush) break;
    need_flush = false;
    }
    const bool irr_ray = (irregular >> lane) & 1u;
    if (irr_ray) {
      // hand the ray to the per-ray kernel (warp-aggregated append)
      const unsigned n_irr = __popc(irregular);
      const int leader = __ffs(irregular) - 1;
      unsigned long long base = 0;
      if ((int)lane == leader) base = atomicAdd(x.ray_list_n, (unsigned long long)n_irr);
      base = __shfl_sync(irregular, base, leader);
      x.ray_list[base + __popc(irregular & ((1u << lane) - 1u))] = k;
    } else {
      tv += rv;
      tt += rt;
      th += rh;
      te += re;
      double4 px;
      if (kMode == 0) {
        px = any_hit ? make_double4(c0, c1, c2, 1.0) : make_double4(x.bg[0], x.bg[1], x.bg[2], x.bg[3]);
      } else {
        const double ra = __dsub_rn(1.0, acc);
        px.x = __dadd_rn(c0, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[0]));
        px.y = __dadd_rn(c1, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[1]));
        px.z = __dadd_rn(c2, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[2]));
        px.w = __dadd_rn(acc, __dmul_rn(ra, x.bg[3]));
      }
      reinterpret_cast<double4*>(x.out_rgba)[k] = px;
      if (x.out_ids && first_obj >= 0) x.out_ids[k] = (int32_t)first_obj;
    }
    __syncwarp();
  }
  unsigned long long v[4] = {tv, tt, th, te};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_xor_sync(full, v[q], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (v[q]) atomicAdd(reinterpret_cast<unsigned long long*>(&x.counters[q]), v[q]);
  }
}

// ---------------------------------------------------------------------------
// scalar query API (fhv/raycast.py:205-453): raycast_pixel with its hit list,
// gather_ray_hits, shadow_transmittance, traverse_octree's leaf sequence and
// intersect_fragment -- one thread per query ray, same device functions as
// the image kernel (not a hot path: a handful of rays per call)

struct ProbeOut {
  const double* tmin;  // per-ray interval, or null -> [0, inf)
  const double* tmax;
  int eye_is_origin;   // raycast_pixel(eye=None): shade toward each ray's origin
  long long cap;       // hit slots per ray
  double* hit_t;
  long long* hit_idx;
  long long* hit_leaf;
  long long* hit_n;    // hits found per ray (may exceed cap: the caller retries)
  long long* stats;    // n x 4 RaycastStats counters
};

// kMode 0..2 = raycast_pixel modes; 3 = gather_ray_hits (no shading, no
// cutoff, hits not counted -- fhv/raycast.py:294-308)
template <int kMode, class E>
__global__ void __launch_bounds__(64) k_ray_probe(RayParams x, long long n, ProbeOut po) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    RayParams xr = x;
    double o[3], d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      o[c] = x.origins[3 * r + c];
      d[c] = x.dirs[3 * r + c];
      if (po.eye_is_origin) xr.eye[c] = o[c];
    }
    const double tmin = po.tmin ? po.tmin[r] : 0.0;
    const double tmax = po.tmax ? po.tmax[r] : __longlong_as_double(0x7ff0000000000000ll);
    Stats st = {0, 0, 0, 0};
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, acc = 0.0;
    bool any_hit = false;
    long long cnt = 0;
    traverse_range<E>(xr, o, d, tmin, tmax, st, [&](long long code) {
      bool stop = false;
      leaf_hits(xr, code, o, d, tmin, tmax, st, [&](double t, long long i) {
        if (cnt < po.cap) {
          po.hit_t[r * po.cap + cnt] = t;
          po.hit_idx[r * po.cap + cnt] = i;
          po.hit_leaf[r * po.cap + cnt] = code;
        }
        ++cnt;
        if (kMode == 3) return true;
        st.hits++;
        double col[3];
        if (kMode == 0) {
          shade_hit<0, E>(xr, i, code, st, col);
          c0 = col[0];
          c1 = col[1];
          c2 = col[2];
          acc = 1.0;
          any_hit = true;
          stop = true;
          return false;
        }
        const double a = xr.s.alpha[xr.v.mat[i]];
        shade_hit<kMode == 3 ? 1 : kMode, E>(xr, i, code, st, col);
        const double tc = __dmul_rn(__dsub_rn(1.0, acc), a);
        c0 = __dadd_rn(c0, __dmul_rn(tc, col[0]));
        c1 = __dadd_rn(c1, __dmul_rn(tc, col[1]));
        c2 = __dadd_rn(c2, __dmul_rn(tc, col[2]));
        acc = __dadd_rn(acc, tc);
        any_hit = true;
        return true;
      });
      if (stop) return false;
      if (kMode != 3 && xr.cutoff >= 0.0 && acc >= xr.cutoff) {
        st.early++;
        return false;
      }
      return true;
    });
    if (x.out_rgba) {
      double* px = x.out_rgba + 4 * r;
      if (kMode == 0) {
        px[0] = any_hit ? c0 : x.bg[0];
        px[1] = any_hit ? c1 : x.bg[1];
        px[2] = any_hit ? c2 : x.bg[2];
        px[3] = any_hit ? 1.0 : x.bg[3];
      } else {
        const double ra = __dsub_rn(1.0, acc);
        px[0] = __dadd_rn(c0, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[0]));
        px[1] = __dadd_rn(c1, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[1]));
        px[2] = __dadd_rn(c2, __dmul_rn(__dmul_rn(ra, x.bg[3]), x.bg[2]));
        px[3] = __dadd_rn(acc, __dmul_rn(ra, x.bg[3]));
      }
    }
    po.hit_n[r] = cnt;
    po.stats[4 * r] = (long long)st.visited;
    po.stats[4 * r + 1] = (long long)st.tested;
    po.stats[4 * r + 2] = (long long)st.hits;
    po.stats[4 * r + 3] = (long long)st.early;
  }
}

// shadow_transmittance (fhv/raycast.py:408-453 = _transmit): light li of the
// shading table; exclusion (object id, leaf) = -1 for none
template <class E>
__global__ void __launch_bounds__(64) k_transmit_probe(RayParams x, long long n, const double* __restrict__ pts,
                                                       int li, const long long* ex_obj, const long long* ex_cell,
                                                       double* __restrict__ tau, long long* __restrict__ stats) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const double p[3] = {pts[3 * r], pts[3 * r + 1], pts[3 * r + 2]};
    Stats st = {0, 0, 0, 0};
    tau[r] = transmit<E>(x, p, li, ex_obj ? ex_obj[r] : -1, ex_cell ? ex_cell[r] : -1, st);
    stats[4 * r] = (long long)st.visited;
    stats[4 * r + 1] = (long long)st.tested;
    stats[4 * r + 2] = (long long)st.hits;
    stats[4 * r + 3] = (long long)st.early;
  }
}

// traverse_octree (fhv/raycast.py:205-243): the occupied leaves one ray
// crosses, nearest entry first, with their clipped [t_enter, t_exit].  The
// order does not depend on the visitor, so the whole sequence is listed and
// the host replays visit() over it (stopping where visit returns False).
template <class E>
__global__ void k_leaf_order(RayParams x, double tmin, double tmax, long long cap, long long* __restrict__ code_out,
                             double* __restrict__ te_out, double* __restrict__ tx_out, long long* n_out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const double o[3] = {x.origins[0], x.origins[1], x.origins[2]};
  const double d[3] = {x.dirs[0], x.dirs[1], x.dirs[2]};
  const double size = __longlong_as_double((1023LL - x.v.levels) << 52);  // 2^-L
  Stats st = {0, 0, 0, 0};
  long long cnt = 0;
  traverse_range<E>(x, o, d, tmin, tmax, st, [&](long long code) {
    if (cnt < cap) {
      const double lo[3] = {__dmul_rn((double)compact3((unsigned long long)code), size),
                            __dmul_rn((double)compact3((unsigned long long)code >> 1), size),
                            __dmul_rn((double)compact3((unsigned long long)code >> 2), size)};
      double t0 = tmin, t1 = tmax;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double hi = __dadd_rn(lo[a], size);
        double ta = 0.0, tb = 0.0;
        if (d[a] != 0.0) {
          ta = ddiv_z(__dsub_rn(lo[a], o[a]), d[a]);
          tb = ddiv_z(__dsub_rn(hi, o[a]), d[a]);
        }
        slab_axis(o[a], d[a], lo[a], hi, ta, tb, t0, t1);  // the DFS only reaches leaves whose slab test passed
      }
      code_out[cnt] = code;
      te_out[cnt] = t0;
      tx_out[cnt] = t1;
    }
    ++cnt;
    return true;
  });
  *n_out = cnt;
}

// intersect_fragment (fhv/raycast.py:246-262): t = (p - o) @ d and
// |p - (o + t d)|^2 as ddot (FWD order), inclusive interval and radius tests
__global__ void k_intersect_points(long long n, const double* __restrict__ pts, double o0, double o1, double o2,
                                   double d0, double d1, double d2, double tmin, double tmax, double r2,
                                   double* __restrict__ t_out, int8_t* __restrict__ hit) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double p0 = pts[3 * i], p1 = pts[3 * i + 1], p2 = pts[3 * i + 2];
    const double t = fwd3(__dsub_rn(p0, o0), __dsub_rn(p1, o1), __dsub_rn(p2, o2), d0, d1, d2);
    bool h = !(t < tmin || t > tmax);
    if (h) {
      const double e0 = __dsub_rn(p0, __dadd_rn(o0, __dmul_rn(t, d0)));
      const double e1 = __dsub_rn(p1, __dadd_rn(o1, __dmul_rn(t, d1)));
      const double e2 = __dsub_rn(p2, __dadd_rn(o2, __dmul_rn(t, d2)));
      h = fwd3(e0, e1, e2, e0, e1, e2) <= r2;
    }
    t_out[i] = t;
    hit[i] = h ? 1 : 0;
  }
}

namespace {
inline int grid_for(long long n, int block, int per_sm = 16) {
  long long g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148LL * per_sm) g = 148LL * per_sm;
  return (int)g;
}

#ifndef FHV_RAY_PACKET
#define FHV_RAY_PACKET 1  // 0: per-ray kernel only (experiment switch)
#endif

// camera rays of modes 0 / 1 over whole 4-row strips of a width divisible by
// 8: packet kernel, then the per-ray kernel over the rays it handed off
template <class E>
int launch_packet(fhv_ctx* ctx, RayParams& x, cudaStream_t st) {
  const long long n = x.end - x.start;
  // [0] rays handed off, [1] hand-off kernel ticket, [2] own-order (lane, node) pairs, [3..] the list
  auto* buf = (unsigned long long*)scratch(ctx, kRays, (size_t)(3 + n) * 8);
  if (!buf) return FHV_NOMEM;
  x.ray_list_n = buf;
  x.own_order_n = buf + 2;
  x.ray_list = (long long*)(buf + 3);
  int rc = check_cuda(ctx, cudaMemsetAsync(buf, 0, 3 * sizeof(unsigned long long), st));
  if (rc) return rc;
  {
    LaunchScope L_(ctx, kStRaycast, st);
    const int g = grid_for(n / 32, kPktWarps, 16);
    if (x.mode == 0)
      k_raycast_packet<0, E><<<g, 32 * kPktWarps, 0, st>>>(x);
    else
      k_raycast_packet<1, E><<<g, 32 * kPktWarps, 0, st>>>(x);
  }
  if ((rc = check_cuda(ctx, cudaGetLastError()))) return rc;
  RayParams y = x;
  y.tile_ticket = buf + 1;
  {
    LaunchScope L_(ctx, kStRaycastHandoff, st);
    if (x.mode == 0)
      k_raycast<0, E><<<148, 128, 0, st>>>(y);
    else
      k_raycast<1, E><<<148, 128, 0, st>>>(y);
  }
  return check_cuda(ctx, cudaGetLastError());
}

int launch(fhv_ctx* ctx, RayParams& x, void* stream) {
  if (x.end <= x.start) return FHV_OK;
  x.tile_ticket = &ctx->ctl->spare[3];
  int rc = check_cuda(ctx, cudaMemsetAsync(x.tile_ticket, 0, sizeof(unsigned long long), (cudaStream_t)stream));
  if (rc) return rc;
  const bool packet = FHV_RAY_PACKET && x.from_camera && x.mode < 2 && x.W % 8 == 0 && x.start % (4 * x.W) == 0 &&
                      x.end % (4 * x.W) == 0;
  if (packet) {
    if (x.v.levels <= 9) return launch_packet<uint32_t>(ctx, x, (cudaStream_t)stream);
    return launch_packet<unsigned long long>(ctx, x, (cudaStream_t)stream);
  }
  {
    LaunchScope L_(ctx, kStRaycast, (cudaStream_t)stream);
    const int g = grid_for(x.end - x.start, 128);
    cudaStream_t st = (cudaStream_t)stream;
    if (x.v.levels <= 9) {
      if (x.mode == 0)
        k_raycast<0, uint32_t><<<g, 128, 0, st>>>(x);
      else if (x.mode == 1)
        k_raycast<1, uint32_t><<<g, 128, 0, st>>>(x);
      else
        k_raycast<2, uint32_t><<<g, 128, 0, st>>>(x);
    } else {
      if (x.mode == 0)
        k_raycast<0, unsigned long long><<<g, 128, 0, st>>>(x);
      else if (x.mode == 1)
        k_raycast<1, unsigned long long><<<g, 128, 0, st>>>(x);
      else
        k_raycast<2, unsigned long long><<<g, 128, 0, st>>>(x);
    }
  }
  return check_cuda(ctx, cudaGetLastError());
}

int common(RayParams& x, const fhv_volume_t* vol, const fhv_shading_t* shading, const double* background, double radius,
           double cutoff, int32_t mode, double eps, double* out_rgba, int32_t* out_ids, int64_t* counters) {
  if (!vol || !shading || !background || !out_rgba || !counters) return FHV_BAD_ARGS;
  if (vol->levels < 1 || vol->levels > kRayMaxLevels || !vol->pyramid) return FHV_BAD_ARGS;
  if (vol->layout == 0 && (!vol->offsets || !vol->counts)) return FHV_BAD_ARGS;
  if (vol->layout == 1 && (!vol->heads || !vol->prev)) return FHV_BAD_ARGS;
  if (mode < 0 || mode > 2 || !(radius > 0.0)) return FHV_BAD_ARGS;
  x.v = *vol;
  x.s = *shading;
  for (int c = 0; c < 4; ++c) x.bg[c] = background[c];
  x.radius = radius;
  x.r2 = radius * radius;
  x.cutoff = cutoff;
  x.eps = eps;
  x.mode = mode;
  x.out_rgba = out_rgba;
  x.out_ids = out_ids;
  x.counters = (long long*)counters;
  return FHV_OK;
}
}  // namespace

}  // namespace fhv

using namespace fhv;

extern "C" int fhv_raycast(fhv_ctx* ctx, const fhv_volume_t* vol, const fhv_shading_t* shading, const double* cam,
                           const double* background, double radius, double cutoff, int32_t mode, double shadow_eps,
                           int64_t row0, int64_t row1, double* out_rgba, int32_t* out_ids, int64_t* counters,
                           void* stream) {
  if (!ctx || !cam) return FHV_BAD_ARGS;
  RayParams x;
  std::memset(&x, 0, sizeof(x));
  int rc = common(x, vol, shading, background, radius, cutoff, mode, shadow_eps, out_rgba, out_ids, counters);
  if (rc) return rc;
  x.from_camera = 1;
  x.persp = cam[0] != 0.0;
  for (int c = 0; c < 3; ++c) {
    x.eye[c] = cam[1 + c];
    x.rr[c] = cam[4 + c];
    x.uu[c] = cam[7 + c];
    x.ff[c] = cam[10 + c];
  }
  x.W = (long long)cam[13];
  x.H = (long long)cam[14];
  x.half_w = cam[15];
  x.half_h = cam[16];
  x.t = cam[17];
  x.aspect = cam[18];
  x.near_ = cam[19];
  if (row0 < 0 || row1 > x.H || row0 > row1) return FHV_BAD_ARGS;
  x.start = row0 * x.W;
  x.end = row1 * x.W;
  return launch(ctx, x, stream);
}

extern "C" int fhv_raycast_image(fhv_ctx* ctx, int64_t start, int64_t end, const double* origins, const double* dirs,
                                 const fhv_volume_t* vol, const fhv_shading_t* shading, const double* eye,
                                 const double* background, double radius, double cutoff, int32_t mode,
                                 double shadow_eps, double* out_rgba, int32_t* out_ids, int64_t* counters,
                                 void* stream) {
  if (!ctx || !origins || !dirs || !eye || start < 0 || end < start) return FHV_BAD_ARGS;
  RayParams x;
  std::memset(&x, 0, sizeof(x));
  int rc = common(x, vol, shading, background, radius, cutoff, mode, shadow_eps, out_rgba, out_ids, counters);
  if (rc) return rc;
  x.from_camera = 0;
  for (int c = 0; c < 3; ++c) x.eye[c] = eye[c];
  x.origins = origins;
  x.dirs = dirs;
  x.start = start;
  x.end = end;
  return launch(ctx, x, stream);
}

// raycast_pixel / gather_ray_hits over n caller rays (mode 3 = gather)
extern "C" int fhv_ray_probe(fhv_ctx* ctx, int64_t n, const double* origins, const double* dirs, const double* tmin,
                             const double* tmax, const fhv_volume_t* vol, const fhv_shading_t* shading,
                             const double* eye, const double* background, double radius, double cutoff, int32_t mode,
                             double shadow_eps, int64_t hit_cap, double* out_rgba, double* hit_t, int64_t* hit_idx,
                             int64_t* hit_leaf, int64_t* hit_n, int64_t* stats, void* stream) {
  if (!ctx || n < 0 || !origins || !dirs || !hit_n || !stats || hit_cap < 0) return FHV_BAD_ARGS;
  if (hit_cap > 0 && (!hit_t || !hit_idx || !hit_leaf)) return FHV_BAD_ARGS;
  if (mode < 0 || mode > 3) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  RayParams x;
  std::memset(&x, 0, sizeof(x));
  // common() validates the volume / shading / radius; mode 3 shades nothing
  int64_t dummy_counters[4];
  int rc = common(x, vol, shading, background, radius, cutoff, mode == 3 ? 1 : mode, shadow_eps,
                  out_rgba ? out_rgba : (double*)dummy_counters, nullptr, dummy_counters);
  if (rc) return rc;
  x.out_rgba = out_rgba;
  x.counters = nullptr;
  x.origins = origins;
  x.dirs = dirs;
  for (int c = 0; c < 3; ++c) x.eye[c] = eye ? eye[c] : 0.0;
  ProbeOut po{tmin, tmax, eye ? 0 : 1, hit_cap, hit_t, (long long*)hit_idx, (long long*)hit_leaf, (long long*)hit_n,
              (long long*)stats};
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(n, 64, 8);
  {
    LaunchScope L_(ctx, kStScalar, s);
    if (x.v.levels <= 9) {
      if (mode == 0) k_ray_probe<0, uint32_t><<<g, 64, 0, s>>>(x, n, po);
      else if (mode == 1) k_ray_probe<1, uint32_t><<<g, 64, 0, s>>>(x, n, po);
      else if (mode == 2) k_ray_probe<2, uint32_t><<<g, 64, 0, s>>>(x, n, po);
      else k_ray_probe<3, uint32_t><<<g, 64, 0, s>>>(x, n, po);
    } else {
      if (mode == 0) k_ray_probe<0, unsigned long long><<<g, 64, 0, s>>>(x, n, po);
      else if (mode == 1) k_ray_probe<1, unsigned long long><<<g, 64, 0, s>>>(x, n, po);
      else if (mode == 2) k_ray_probe<2, unsigned long long><<<g, 64, 0, s>>>(x, n, po);
      else k_ray_probe<3, unsigned long long><<<g, 64, 0, s>>>(x, n, po);
    }
  }
  return check_cuda(ctx, cudaGetLastError());
}

// shadow_transmittance toward light `light` of the shading table, n points
extern "C" int fhv_transmittance(fhv_ctx* ctx, int64_t n, const double* points, int32_t light,
                                 const int64_t* exclude_obj, const int64_t* exclude_cell, const fhv_volume_t* vol,
                                 const fhv_shading_t* shading, double radius, double shadow_eps, double* tau,
                                 int64_t* stats, void* stream) {
  if (!ctx || n < 0 || !shading || light < 0 || light >= shading->n_lights) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  if (!points || !tau || !stats) return FHV_BAD_ARGS;
  RayParams x;
  std::memset(&x, 0, sizeof(x));
  const double bg[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t dummy[4];
  int rc = common(x, vol, shading, bg, radius, -1.0, 2, shadow_eps, (double*)dummy, nullptr, dummy);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int g = grid_for(n, 64, 8);
  {
    LaunchScope L_(ctx, kStScalar, s);
    if (x.v.levels <= 9)
      k_transmit_probe<uint32_t><<<g, 64, 0, s>>>(x, n, points, light, (const long long*)exclude_obj,
                                                  (const long long*)exclude_cell, tau, (long long*)stats);
    else
      k_transmit_probe<unsigned long long><<<g, 64, 0, s>>>(x, n, points, light, (const long long*)exclude_obj,
                                                            (const long long*)exclude_cell, tau, (long long*)stats);
  }
  return check_cuda(ctx, cudaGetLastError());
}

// traverse_octree's leaf sequence for one ray (origin/dir: 3 device doubles)
extern "C" int fhv_leaf_order(fhv_ctx* ctx, int32_t levels, const uint8_t* pyramid, const double* origin,
                              const double* dir, double tmin, double tmax, int64_t cap, int64_t* code_out,
                              double* te_out, double* tx_out, int64_t* n_out, void* stream) {
  if (!ctx || levels < 1 || levels > kRayMaxLevels || !pyramid || !origin || !dir || !n_out || cap < 0)
    return FHV_BAD_ARGS;
  if (cap > 0 && (!code_out || !te_out || !tx_out)) return FHV_BAD_ARGS;
  RayParams x;
  std::memset(&x, 0, sizeof(x));
  x.v.levels = levels;
  x.v.pyramid = pyramid;
  x.origins = origin;
  x.dirs = dir;
  cudaStream_t s = (cudaStream_t)stream;
  {
    LaunchScope L_(ctx, kStScalar, s);
    if (levels <= 9)
      k_leaf_order<uint32_t><<<1, 32, 0, s>>>(x, tmin, tmax, cap, (long long*)code_out, te_out, tx_out,
                                              (long long*)n_out);
    else
      k_leaf_order<unsigned long long><<<1, 32, 0, s>>>(x, tmin, tmax, cap, (long long*)code_out, te_out, tx_out,
                                                        (long long*)n_out);
  }
  return check_cuda(ctx, cudaGetLastError());
}

// intersect_fragment for n points against one ray
extern "C" int fhv_intersect_points(fhv_ctx* ctx, int64_t n, const double* points, const double* origin,
                                    const double* dir, double tmin, double tmax, double radius, double* t_out,
                                    int8_t* hit, void* stream) {
  if (!ctx || n < 0 || !origin || !dir) return FHV_BAD_ARGS;
  if (n == 0) return FHV_OK;
  if (!points || !t_out || !hit) return FHV_BAD_ARGS;
  cudaStream_t s = (cudaStream_t)stream;
  {
    LaunchScope L_(ctx, kStScalar, s);
    k_intersect_points<<<grid_for(n, 128, 8), 128, 0, s>>>(n, points, origin[0], origin[1], origin[2], dir[0], dir[1],
                                                           dir[2], tmin, tmax, radius * radius, t_out, hit);
  }
  return check_cuda(ctx, cudaGetLastError());
}
