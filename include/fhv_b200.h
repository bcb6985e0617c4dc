/*
 * fhv_b200.h -- C ABI of the B200-native fragment-history-volume hot path.
 *
 * One shared library (paper_2211_15460_b200/libfhv_b200.so, sm_100a).  Plain
 * pointers and sizes only; every buffer is allocated by the caller (PyTorch)
 * unless stated, the library never frees caller memory.  All calls are
 * enqueued on `stream` (a cudaStream_t); calls that must return a
 * data-dependent size to the host (fragment totals) synchronise that stream.
 * Return value: an FHV_* status code.
 *
 * Which reference interface each entry point replaces (
 * `fhv/X.py:N` = /root/reference/pkg/src/fhv/X.py line N):
 *
 *   reference operator API          fhv/_backend.py:25-29  kernels() -> module with
 *     coverage(...)                 fhv/_ckern.pyx:25-105   per triangle
 *     linked_insert(...)            fhv/_ckern.pyx:112-123  per batch
 *     pofa_scatter(...)             fhv/_ckern.pyx:126-143  per batch
 *     raycast_image(...)            fhv/_ckern.pyx:653-743  per image span
 *
 * The three per-triangle / per-batch kernels are only ever called from the
 * capture drivers, and a per-triangle launch is meaningless on a GPU, so the
 * boundary moves one level up to the drivers that call them:
 *   fhv_build_ppfl    <- build_ppfl        fhv/storage.py:553-571 (capture_pass + PpflSink + linked_insert)
 *   fhv_build_pofl    <- build_pofl        fhv/storage.py:574-587 (capture_pass + PoflSink + linked_insert + set_paths)
 *   fhv_pofa_count    <- pofa_build pass 1 fhv/storage.py:602-608 (CountingSink, cumsum, total check)
 *   fhv_pofa_scatter  <- pofa_build pass 2 fhv/storage.py:610-620 (PofaWriteSink + pofa_scatter + checks + pyramid)
 *   fhv_capture_list  <- capture_pass + ListSink  fhv/raster.py:350-388, 309-320
 *   fhv_splat         <- splat_render      fhv/render.py:249-320
 *   fhv_raycast       <- render_raycast    fhv/raycast.py:469-577 (rays generated on device)
 *   fhv_raycast_image <- raycast_image     fhv/_ckern.pyx:653-743 (1:1: caller-provided rays, pixel span)
 */
#ifndef FHV_B200_H
#define FHV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python layer maps them to the reference's exceptions */
enum {
  FHV_OK = 0,
  FHV_OVERFLOW = 1,       /* pool overflow: records past capacity dropped (FragmentPool.overflowed) */
  FHV_PASS_MISMATCH = 2,  /* PofaBuildError (fhv/storage.py:73-74, 431-433, 614-619) */
  FHV_BAD_ARGS = 3,       /* ValueError / FhvError on arguments */
  FHV_CUDA_ERROR = 4,     /* a CUDA runtime call failed */
  FHV_RANGE = 5,          /* FhvError: fragment position outside [0,1]^3 (fhv/storage.py:152-155) */
  FHV_BASIS = 6,          /* ValueError from tangent_basis (fhv/raster.py:154-157) */
  FHV_NOMEM = 7,          /* MemoryError */
  FHV_TOO_MANY = 8,       /* FhvError: >= 2^32 fragments (fhv/storage.py:604-606) */
  FHV_SPLAT_BIG = 9,      /* SceneError: splat footprint > 4096 px (fhv/render.py:285-286) */
  FHV_NEED_POOL = 10,     /* fhv_pofa_build: pool smaller than the exact count; *total says how big */
  FHV_STALE = 11,         /* fhv_ticket_check: an asynchronous build ran on a wrong speculation (pool size or
                             work-item plan); its outputs are invalid -- rebuild synchronously */
};

/* capture flags */
enum {
  FHV_ALLOC_ATOMIC = 1,  /* paper-style slots from a warp-aggregated atomic counter (nondeterministic pool order) */
  FHV_EXACT_ORDER = 2,   /* chains (PPFL/POFL) / in-leaf order (POFA) identical to the sequential reference */
};

/* splat flags */
enum {
  FHV_SPLAT_PACKED = 1,  /* one 64-bit atomicMin on (f32 depth | u32 index); default is the exact f64 two-pass z-test */
  FHV_SPLAT_NOSYNC = 2,  /* caller proved the footprint bound (fhv/render.py:285-286) holds: return without
                            waiting for the kernels (no FHV_SPLAT_BIG check) */
};

typedef struct fhv_ctx fhv_ctx; /* per-device scratch arena (grow-only); one per host thread / stream */

/* triangle soup, device pointers (Scene arrays, fhv/scene.py:105-126) */
typedef struct {
  int64_t n_tri;
  const double *pos;  /* [T][3][3] vertex positions */
  const double *vnrm; /* [T][3][3] vertex normals   */
  const double *fnrm; /* [T][3]    face normals     */
  const uint32_t *mat;
  const uint32_t *obj;
} fhv_tris_t;

/* resolved capture strategy (paper_2211_15460_b200/raster.py CapturePlan) */
typedef struct {
  int32_t strategy; /* 0 one_view, 1 three_separate, 2 three_way_geometry, 3 normal_space */
  int32_t res;      /* square capture grid edge, fhv/raster.py:359 */
  double pitch;     /* normal_space sample spacing, fhv/raster.py:381 */
  double proj[3][16]; /* row-major world->clip per capture axis */
} fhv_capture_cfg_t;

/* FragmentPool (fhv/storage.py:188-248), struct-of-arrays, device pointers */
typedef struct {
  int64_t capacity;
  float *pos;     /* [cap][3] */
  float *nrm;     /* [cap][3] */
  uint32_t *mat;
  uint32_t *obj;
  int32_t *prev;  /* prev_index */
} fhv_pool_t;

/* One rank's share of a POFA capture partitioned across GPUs by Morton range
   (SURVEY.md section 8(e)): the rank owns leaves [cell_lo, cell_hi) (multiples
   of the directory tile: 8^5 leaves for levels >= 5, 8^4 for levels = 4) and rasterises only the triangles whose f64
   AABB, grown by `margin`, meets one of `boxes` (a conservative world-space
   cover of its range, host memory; n_boxes == 0 disables binning). */
#define FHV_SHARD_MAX_BOXES 64
typedef struct {
  uint64_t cell_lo, cell_hi;
  int32_t n_boxes;
  double margin;
  double boxes[FHV_SHARD_MAX_BOXES][6]; /* lo xyz, hi xyz */
} fhv_shard_t;

/* materials + lights, device pointers (fhv/render.py:106-113, fhv/raycast.py:460-466) */
typedef struct {
  int32_t n_lights;
  const uint8_t *light_kind;   /* 0 directional, 1 point */
  const double *light_vec;     /* [K][3] direction (unit) or position */
  const double *light_color;   /* [K][3] */
  const double *light_ambient; /* [K][3] */
  int32_t n_mats;
  const double *diffuse;   /* [M][3] */
  const double *specular;  /* [M][3] */
  const double *shininess; /* [M] */
  const double *alpha;     /* [M] */
} fhv_shading_t;

/* camera packed by Camera.scalars(): [persp, eye3, r3, u3, f3, w, h, half_w,
   half_h, tan(fov/2), aspect, near, far, extent] (host memory, 22 doubles) */
#define FHV_CAM_SCALARS 22

/* read-only per-octant volume for ray casting (FhvPofa / FhvPofl) */
typedef struct {
  int32_t layout; /* 0 POFA (offsets, counts), 1 POFL (heads, prev) */
  int32_t levels;
  const uint32_t *offsets;
  const uint32_t *counts;
  const int32_t *heads;
  const int32_t *prev;
  const uint8_t *pyramid; /* levels 0..L-1 concatenated */
  const float *pos;
  const float *nrm;
  const uint32_t *mat;
  const uint32_t *obj;
} fhv_volume_t;

/* optional per-pixel id buffer of splat_render (GBuffer, fhv/render.py:87-103) */
typedef struct {
  double *position; /* [P][3] or NULL */
  double *normal;   /* [P][3] or NULL */
  int32_t *material_id;
  int32_t *object_id;
  uint8_t *valid;
} fhv_gbuffer_t;

const char *fhv_version(void);
fhv_ctx *fhv_ctx_create(void);
void fhv_ctx_destroy(fhv_ctx *ctx);
/* kernels launched by this context since creation (for launch accounting) */
int64_t fhv_ctx_launches(const fhv_ctx *ctx);
/* diagnostics of the last SYNCHRONISED call on this context: out[0] = leaves
   the EXACT_ORDER POFA tile fix-up re-sorted, out[1] = fragments the raster
   passes sent through the exact (uncertified) path, out[2] = long leaves
   handed to the per-leaf pass; with n >= 4 (synchronises the device) the
   last packet ray cast (fhv_raycast): out[3] = rays handed to its per-ray
   kernel, out[4] = (ray, node) pairs that took their own child order (tied
   entry distances); returns the words written (3, 4 or 5) */
int fhv_ctx_counters(const fhv_ctx *ctx, int64_t *out, int n);

/* per-kernel CUDA-event timing on the launching stream (off by default).
   fhv_prof_collect synchronises the recorded events, writes accumulated
   milliseconds and launch counts per stage (up to n entries), resets the
   accumulators and returns the number of stages. */
int fhv_prof_enable(fhv_ctx *ctx, int on);
int fhv_prof_collect(fhv_ctx *ctx, double *ms, int64_t *count, int n);
const char *fhv_prof_stage_name(int stage);

/* Every fragment in reference emission order (job, y, x), f64 attributes.
   max_out bounds the outputs; *n_out receives the total.  Synchronises. */
int fhv_capture_list(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg,
                     int64_t max_out, int64_t *job, int32_t *px, int32_t *py, double *wpos,
                     double *wnrm, int64_t *n_out, void *stream);

/* fhv_capture_list plus FragmentBatch.depth per fragment (capture_pass,
   fhv/raster.py:204,240: screen strategies lam @ ndc_z, normal_space 0.5). */
int fhv_capture_list_depth(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg,
                           int64_t max_out, int64_t *job, int32_t *px, int32_t *py, double *wpos,
                           double *wnrm, double *depth, int64_t *n_out, void *stream);

/* rasterize_triangle / _raster_screen (fhv/raster.py:184-209, 245-252) for
   every triangle through one 4x4 row-major projection (orthographic or
   perspective, RasterConfig.projection) into width x height: fragments in
   (triangle, y, x) order, job[] = triangle index, perspective-correct
   interpolation, depth = lam @ ndc_z.  Synchronises. */
int fhv_raster_screen(fhv_ctx *ctx, const fhv_tris_t *tris, const double *proj, int32_t width,
                      int32_t height, int64_t max_out, int64_t *job, int32_t *px, int32_t *py,
                      double *wpos, double *wnrm, double *depth, int64_t *n_out, void *stream);

/* build_ppfl: heads[W*H] and pool->prev must be pre-filled with -1 by the
   caller; width = PixelDirectory.width.  *next_free = fragments emitted
   (FragmentPool.next_free).  Synchronises.  Returns FHV_OVERFLOW if
   next_free > capacity. */
int fhv_build_ppfl(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int64_t width,
                   fhv_pool_t *pool, int32_t *heads, int32_t flags, int64_t *next_free, void *stream);

/* build_pofl: heads[8^L] pre-filled with -1; pyramid (sum 8^k bytes) is
   written.  Synchronises. */
int fhv_build_pofl(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                   fhv_pool_t *pool, int32_t *heads, uint8_t *pyramid, int32_t flags,
                   int64_t *next_free, void *stream);

/* pofa_build pass 1: counts[8^L] per-leaf fragment counts, offsets = their
   exclusive prefix sum, pyramid from counts > 0, *total = pool size.  The
   rasterised job table stays in ctx for fhv_pofa_scatter.  Synchronises. */
int fhv_pofa_count(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                   uint32_t *counts, uint32_t *offsets, uint8_t *pyramid, int64_t *total,
                   void *stream);

/* pofa_build pass 2: scatter every fragment into its leaf's range
   [offsets[c], offsets[c]+counts[c]); prev_index = -1.  Verifies cursors ==
   counts (FHV_PASS_MISMATCH otherwise).  Must follow fhv_pofa_count on the
   same ctx with the same inputs.  Synchronises. */
int fhv_pofa_scatter(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg,
                     int32_t levels, const uint32_t *counts, const uint32_t *offsets, fhv_pool_t *pool,
                     int32_t flags, void *stream);

/* pofa_build in one call (fhv/storage.py:590-621): pass 1 + directory +
   pass 2 with the syncs inside the library.  pool may be NULL or smaller
   than the exact count: then *total is set, nothing is scattered and
   FHV_NEED_POOL is returned -- allocate a pool of *total records and finish
   with fhv_pofa_scatter (the pass-1 state stays in ctx).  A pool larger than
   *total receives records [0, *total) only. */
int fhv_pofa_build(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                   uint32_t *counts, uint32_t *offsets, uint8_t *pyramid, fhv_pool_t *pool, int32_t flags,
                   int64_t *total, void *stream);

/* pofa_build fully asynchronous: the same pass 1 + directory + pass 2 as
   fhv_pofa_build, enqueued without any host wait, into a pool whose capacity
   is the caller's guess of the exact total (e.g. the total of the previous
   build of the same scene).  The outcome lands in *ticket (pinned host
   memory; the ticket kernel stores it directly when the ticket is device
   memory or pinned host memory, else a stream-ordered copy delivers it);
   after synchronising the stream,
   fhv_ticket_check(ticket, pool capacity) returns FHV_OK when the pool holds
   exactly the build's records, FHV_STALE when the speculation was wrong
   (outputs invalid: rebuild with fhv_pofa_build), or the build's own error. */
typedef struct {
  int64_t status, frags_total, scan_total, alloc;
} fhv_ticket_t;
int fhv_pofa_build_async(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                         uint32_t *counts, uint32_t *offsets, uint8_t *pyramid, fhv_pool_t *pool, int32_t flags,
                         fhv_ticket_t *ticket, void *stream);
int fhv_ticket_check(const fhv_ticket_t *ticket, int64_t expect_total);
/* The same check on the device, enqueued right after fhv_pofa_build_async on
   its stream (e.g. inside a CUDA graph that replays the build): acc[0]
   (device int64, zeroed by the caller) keeps the first non-OK status,
   acc[1] counts the checks.  Async. */
int fhv_ticket_accumulate(fhv_ctx *ctx, int64_t expect_total, int64_t *acc, void *stream);
/* build_pofl without a host wait, on the same ticket protocol: the pool's
   capacity is the caller's (e.g. the previous build's total), the outcome
   (status; the total in frags_total = scan_total = alloc) lands in *ticket.
   fhv_ticket_check(ticket, guess) is FHV_OK when the total equals the guess;
   FHV_STALE (a speculative item plan missed, or another total) means rebuild
   with fhv_build_pofl.  Replaces fhv/storage.py:574-587 like fhv_build_pofl. */
int fhv_build_pofl_async(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                         fhv_pool_t *pool, int32_t *heads, uint8_t *pyramid, int32_t flags, fhv_ticket_t *ticket,
                         void *stream);

/* rebuild_pofl_as_pofa (fhv/storage.py:624-652): repack the first n records
   of a linked-list pool into per-leaf contiguous ranges (Morton order, pool
   order inside a leaf), counts / offsets [8^L], pyramid from counts > 0;
   dst->prev_index = -1.  FHV_RANGE if a position lies outside [0,1]^3.
   Synchronises. */
int fhv_rebuild_pofa(fhv_ctx *ctx, int32_t levels, const fhv_pool_t *src, int64_t n, uint32_t *counts,
                     uint32_t *offsets, uint8_t *pyramid, fhv_pool_t *dst, void *stream);

/* FHV1 snapshot records (fhv/storage.py:725-808): pack the first n pool
   records into `out` as packed little-endian 36-byte RECORD_DTYPE rows
   (device memory, 4-byte aligned), or unpack such rows into a pool.  Async. */
int fhv_pack_records(fhv_ctx *ctx, const fhv_pool_t *pool, int64_t n, void *out, void *stream);
int fhv_unpack_records(fhv_ctx *ctx, const void *in, int64_t n, fhv_pool_t *pool, void *stream);

/* Multi-GPU splat composited over peer memory (NVLink / NVSwitch P2P; on one
   device: plain pointers).  The frame's rows are cut into one slab per rank
   (rank q owns rows [q H / N, (q+1) H / N)); keys[q] / winners[q] are rank
   q's slab buffers (8 B per pixel each), rgba[q] / depth[q] rank q's full
   frame ([H][W][4] / [H][W] f64) -- all as seen from the calling process.
   SURVEY.md section 8(e) "composite per-GPU reconstructions by depth". */
#define FHV_MAX_PEERS 8
typedef struct {
  int32_t nranks;
  int64_t width, height;
  void *keys[FHV_MAX_PEERS];
  void *winners[FHV_MAX_PEERS];
  double *rgba[FHV_MAX_PEERS];
  double *depth[FHV_MAX_PEERS];
} fhv_peer_t;

/* One phase of the peer splat for rank `rank` holding records [index_base,
   index_base + n) of the union pool: 0 = empty its own slab, 1 = RED.MIN
   depth keys into the owners' slabs (synchronises; extent[2] = max
   footprint, the caller all-reduces it for the 4096-pixel check), 2 = winner
   candidates, 3 = shade the winners it owns and store them (and, for its own
   slab, the background) into every rank's frame; 4 = probe: extent (a
   DEVICE array of nranks int64) <- the first winner word of every rank's
   slab, read through the peer mappings.  Between phases every rank must
   have finished the previous one (caller's barrier). */
int fhv_splat_peer(fhv_ctx *ctx, int32_t phase, int64_t n, const float *pos, const float *nrm, const uint32_t *mat,
                   const double *cam, double radius, const fhv_shading_t *shading, const double *background,
                   const fhv_peer_t *peers, int32_t rank, int64_t index_base, int64_t *extent, void *stream);

/* Self-test of the library's shared-divisor IEEE division against
   __ddiv_rn (device arrays of n doubles; fast / ref written).  Async. */
int fhv_selftest_div(fhv_ctx *ctx, int64_t n, const double *x, const double *d, double *fast, double *ref,
                     void *stream);

/* Scene ingest (load_scene, fhv/scene.py:291-378): rows of `in` [n][3]
   divided by sqrt(row . row) in NumPy's ddot order -- np.linalg.norm and
   _unit of the reference.  *zero_first = index of the first zero-length row,
   or -1.  Synchronises. */
int fhv_unit_rows(fhv_ctx *ctx, int64_t n, const double *in, double *out, int64_t *zero_first, void *stream);

/* deferred_baseline (fhv/render.py:327-382) -- the paper's DS comparison
   renderer: every triangle rasterised through the camera projection `proj`
   (4x4 row-major world->clip, RasterConfig.from_camera) at width x height,
   nearest (f64 depth, triangle index) per pixel kept in the f64 G-buffer
   (all five planes required; written for every pixel: winners, or the
   GBuffer.new defaults), then Blinn-Phong with eye[3] into out_rgba
   [H][W][4] (background where empty) and out_depth [H][W] (+inf where
   empty).  *emitted = fragments rasterised.  Synchronises. */
int fhv_deferred(fhv_ctx *ctx, const fhv_tris_t *tris, const double *proj, int32_t width, int32_t height,
                 const double *eye, const fhv_shading_t *shading, const double *background, double *out_rgba,
                 double *out_depth, const fhv_gbuffer_t *gb, int64_t *emitted, void *stream);

/* Sharded pofa_build (one rank; the caller exchanges totals between the
   calls, e.g. one all_gather of a u64 per rank):
   1. fhv_pofa_shard_count: bin triangles, rasterise, histogram the owned
      leaves into counts_local[cell_hi - cell_lo]; *local_total = owned
      fragments.  Synchronises.
   2. fhv_pofa_shard_directory: offsets_local = base + exclusive scan of
      counts_local (a slice of the global directory when base = the sum of
      the lower ranks' totals); writes this shard's occupancy into pyramid
      (levels >= L-4 exact, upper levels partial: OR them across ranks).
      The caller zeroes pyramid first.  Async.
   3. fhv_pofa_shard_scatter: pool->pos[offsets_local[c] - base + k] = ...
      (pool holds this shard's local_total records).  Synchronises.
   Must run in this order on one ctx with the same tris / cfg / shard. */
int fhv_pofa_shard_count(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                         const fhv_shard_t *shard, uint32_t *counts_local, int64_t *local_total,
                         void *stream);
int fhv_pofa_shard_directory(fhv_ctx *ctx, int32_t levels, const fhv_shard_t *shard,
                             const uint32_t *counts_local, uint32_t *offsets_local, uint8_t *pyramid,
                             uint64_t base, void *stream);
int fhv_pofa_shard_scatter(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                           const fhv_shard_t *shard, const uint32_t *counts_local,
                           const uint32_t *offsets_local, uint64_t base, fhv_pool_t *pool, int32_t flags,
                           void *stream);
/* The three steps above in one call with no host wait and no collective
   (speculative, the fhv_pofa_build_async ticket protocol): the caller passes
   base and a pool sized by THIS rank's total, both taken from the previous
   build of the same scene and ranges on every rank; that build's triangle
   binning is reused when this ctx made it for the same triangle arrays and
   shard (their contents must not have changed).  *ticket receives this
   rank's status and total; the build is valid when fhv_ticket_check(ticket,
   pool capacity) is FHV_OK on EVERY rank (then every rank's base was right).
   Replaces fhv/storage.py:590-621 per rank like the three-step form. */
int fhv_pofa_shard_build_async(fhv_ctx *ctx, const fhv_tris_t *tris, const fhv_capture_cfg_t *cfg, int32_t levels,
                               const fhv_shard_t *shard, uint32_t *counts_local, uint32_t *offsets_local,
                               uint8_t *pyramid, uint64_t base, fhv_pool_t *pool, int32_t flags,
                               fhv_ticket_t *ticket, void *stream);

/* splat_render over pool[0:n): out_rgba [H][W][4] f64, out_depth [H][W] f64,
   out_winner [H][W] int32 (pool index or -1, may be NULL), gbuffer may be
   NULL.  Synchronises (footprint check). */
int fhv_splat(fhv_ctx *ctx, int64_t n, const float *pos, const float *nrm, const uint32_t *mat,
              const uint32_t *obj, const double *cam, double radius, const double *background,
              const fhv_shading_t *shading, double *out_rgba, double *out_depth, int32_t *out_winner,
              const fhv_gbuffer_t *gbuffer, int32_t flags, void *stream);

/* Sharded splat_render (one rank holding pool records with global indices
   [index_base, index_base + n)); the caller all-reduces between the calls:
   1. fhv_splat_shard_keys: keys[H*W] int64 = per-pixel minimum of this
      rank's f64 depth keys (order-preserving, sign-flipped so that an int64
      MIN all-reduce composites ranks by depth; INT64_MAX = empty);
      footprint[2] (host) = this rank's max splat extent (kx, ky): the
      caller max-reduces them and raises SceneError if kx*ky > 4096.
      Synchronises.
   2. (all-reduce MIN keys) fhv_splat_shard_winners: winners[H*W] int64 =
      lowest global pool index among this rank's fragments whose key equals
      the global key (INT64_MAX if none).  Async.
   3. (all-reduce MIN winners) fhv_splat_shard_resolve: rgba / depth of the
      pixels whose winner this rank owns, -0.0 elsewhere; write_background
      (one rank) also writes the background / +inf of empty pixels.  Async.
   4. (all-reduce SUM rgba, depth) = splat_render of the whole pool. */
int fhv_splat_shard_keys(fhv_ctx *ctx, int64_t n, const float *pos, const double *cam, double radius,
                         int64_t *keys, int64_t *footprint, void *stream);
int fhv_splat_shard_winners(fhv_ctx *ctx, int64_t n, const float *pos, const double *cam, double radius,
                            const int64_t *keys, int64_t index_base, int64_t *winners, void *stream);
int fhv_splat_shard_resolve(fhv_ctx *ctx, int64_t n, const float *pos, const float *nrm, const uint32_t *mat,
                            const double *cam, double radius, const fhv_shading_t *shading,
                            const int64_t *keys, const int64_t *winners, int64_t own_lo,
                            int32_t write_background, const double *background, double *out_rgba,
                            double *out_depth, void *stream);

/* render_raycast for rows [row0, row1) of the camera image: out_rgba
   [H][W][4] f64, out_ids [H][W] int32 (first-hit object id, NULL to skip),
   counters int64[4] on DEVICE (+= visited, tested, hits, early).  Async. */
int fhv_raycast(fhv_ctx *ctx, const fhv_volume_t *vol, const fhv_shading_t *shading, const double *cam,
                const double *background, double radius, double cutoff, int32_t mode, double shadow_eps,
                int64_t row0, int64_t row1, double *out_rgba, int32_t *out_ids, int64_t *counters,
                void *stream);

/* raycast_image 1:1 (fhv/_ckern.pyx:653-743): rays from caller arrays
   origins/dirs [P][3] f64 (device), pixels [start, end).  Async. */
int fhv_raycast_image(fhv_ctx *ctx, int64_t start, int64_t end, const double *origins,
                      const double *dirs, const fhv_volume_t *vol, const fhv_shading_t *shading,
                      const double *eye, const double *background, double radius, double cutoff,
                      int32_t mode, double shadow_eps, double *out_rgba, int32_t *out_ids,
                      int64_t *counters, void *stream);

/* make_triangle face normals for a bulk scene (fhv/scene.py:137-139). Async. */
int fhv_face_normals(fhv_ctx *ctx, int64_t n_tri, const double *pos, double *fnrm, void *stream);

/* Indexed scene upload: triangle arrays pos / vnrm [n_tri][3][3] f64 gathered
   from shared vertex rows vpos / vn [n_vert][3] through faces [n_tri][3]
   (u32 vertex indices) -- the triangle-soup arrays load_scene / make_triangle
   produce (fhv/scene.py:129-146, 291-378), byte for byte, from ~1/3.5 of the
   bytes over PCIe (meshes share each vertex among ~6 triangles).  A face
   index >= n_vert -> FHV_BAD_ARGS (checked on the device, reported by the
   next synchronising call).  Async. */
int fhv_expand_indexed(fhv_ctx *ctx, int64_t n_vert, const double *vpos, const double *vn, int64_t n_tri,
                       const uint32_t *faces, double *pos, double *vnrm, void *stream);

/* ---- the reference's operator API, kernels() (fhv/_backend.py:25-29), batched ----
   coverage (fhv/_ckern.pyx:25-105) of n raster-space triangles v6[n][6] =
   (ax, ay, bx, by, cx, cy) on rasters wh[n][2] = (w, h): covered pixel
   centres per triangle in row-major order at tri_off[t] .. tri_off[t+1]
   (tri_off: n+1 int64, device), barycentrics l0/l1/l2 = f_i / area2.
   Triangles with area2 <= 0 (or non-finite) emit nothing and *first_bad =
   the first such index (the reference raises ValueError), else -1.
   max_out bounds the outputs, *n_out = total.  Synchronises. */
int fhv_op_coverage(fhv_ctx *ctx, int64_t n, const double *v6, const int32_t *wh, int64_t max_out,
                    int64_t *tri_off, int32_t *px, int32_t *py, double *l0, double *l1, double *l2,
                    int64_t *n_out, int64_t *first_bad, void *stream);
/* linked_insert (fhv/_ckern.pyx:112-123): for i in order, prev[start+i] =
   heads[keys[i]]; heads[keys[i]] = start+i.  Keys outside [0, n_keys) ->
   FHV_BAD_ARGS before any write.  Synchronises. */
int fhv_op_linked_insert(fhv_ctx *ctx, int64_t n, const int64_t *keys, int64_t n_keys, int32_t *heads,
                         int32_t *prev, int64_t prev_len, int64_t start, void *stream);
/* pofa_scatter (fhv/_ckern.pyx:126-143): dest[i] = offsets[c] + cursors[c]++
   in order; stops at the first i whose cursor reaches counts[c] (*bad = i,
   else -1).  Synchronises. */
int fhv_op_pofa_scatter(fhv_ctx *ctx, int64_t n, const int64_t *codes, int64_t n_leaves,
                        const uint32_t *offsets, const uint32_t *counts, uint32_t *cursors, int64_t *dest,
                        int64_t *bad, void *stream);

/* OccupancyPyramid.set_paths (fhv/storage.py:294-301): OR the root paths of
   n leaf codes (< 8^levels, else FHV_BAD_ARGS) into the concatenated
   pyramid.  Synchronises. */
int fhv_set_paths(fhv_ctx *ctx, int32_t levels, int64_t n, const int64_t *codes, uint8_t *pyramid,
                  void *stream);
/* OccupancyPyramid.from_leaf_occupancy (fhv/storage.py:316-328): occupied
   u8[8^levels] (nonzero = occupied) -> every pyramid level.  Async. */
int fhv_pyramid_from_occupancy(fhv_ctx *ctx, int32_t levels, const uint8_t *occupied, uint8_t *pyramid,
                               void *stream);

/* chain_indices (fhv/storage.py:480-488): the pool indices of one linked
   list (heads[key], then prev[]), most recent first; up to cap into out,
   *n_out = length.  Synchronises. */
int fhv_chain_indices(fhv_ctx *ctx, const int32_t *heads, int64_t n_keys, const int32_t *prev,
                      int64_t prev_len, int64_t key, int64_t cap, int64_t *out, int64_t *n_out, void *stream);

/* ---- scalar queries (fhv/raycast.py:205-453, fhv/render.py:120-166) ----
   shade_many: n f64 points / normals, int64 material ids (< n_materials,
   checked by the caller), out_rgb [n][3].  Async. */
int fhv_shade(fhv_ctx *ctx, int64_t n, const double *points, const double *normals,
              const int64_t *material_id, int64_t n_materials, const fhv_shading_t *shading,
              const double *eye, double *out_rgb, void *stream);
/* project_points (fhv/render.py:211-233): n device f64 points through the
   camera scalars (as fhv_splat's cam): raster x, y, depth, view distance zc
   [n] each.  Async. */
int fhv_project_points(fhv_ctx *ctx, int64_t n, const double *points, const double *cam, double *xr,
                       double *yr, double *depth, double *zc, void *stream);
/* raycast_pixel (mode 0..2) / gather_ray_hits (mode 3) for n rays (device
   origins/dirs [n][3], optional tmin/tmax [n]; eye NULL = each ray's
   origin).  Per ray: out_rgba [n][4] (NULL allowed for mode 3), up to
   hit_cap hits (t, pool index, leaf) in traversal order, hit_n = hits found
   (> hit_cap: call again with more room), stats [n][4] RaycastStats.  Async. */
int fhv_ray_probe(fhv_ctx *ctx, int64_t n, const double *origins, const double *dirs, const double *tmin,
                  const double *tmax, const fhv_volume_t *vol, const fhv_shading_t *shading,
                  const double *eye, const double *background, double radius, double cutoff, int32_t mode,
                  double shadow_eps, int64_t hit_cap, double *out_rgba, double *hit_t, int64_t *hit_idx,
                  int64_t *hit_leaf, int64_t *hit_n, int64_t *stats, void *stream);
/* shadow_transmittance toward light `light` of the shading table for n
   device points; exclude_obj / exclude_cell [n] (-1 = none, NULL = none).
   tau [n], stats [n][4].  Async. */
int fhv_transmittance(fhv_ctx *ctx, int64_t n, const double *points, int32_t light,
                      const int64_t *exclude_obj, const int64_t *exclude_cell, const fhv_volume_t *vol,
                      const fhv_shading_t *shading, double radius, double shadow_eps, double *tau,
                      int64_t *stats, void *stream);
/* traverse_octree: occupied leaves along one ray (device origin/dir [3]),
   nearest entry first, with t_enter / t_exit; up to cap, *n_out (device) =
   total.  Async. */
int fhv_leaf_order(fhv_ctx *ctx, int32_t levels, const uint8_t *pyramid, const double *origin,
                   const double *dir, double tmin, double tmax, int64_t cap, int64_t *code_out,
                   double *te_out, double *tx_out, int64_t *n_out, void *stream);
/* intersect_fragment for n device points against one ray (host origin/dir):
   t_out [n], hit [n] (1 = within [tmin, tmax] and radius).  Async. */
int fhv_intersect_points(fhv_ctx *ctx, int64_t n, const double *points, const double *origin,
                         const double *dir, double tmin, double tmax, double radius, double *t_out,
                         int8_t *hit, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FHV_B200_H */
