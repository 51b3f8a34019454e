/* libdifftrans — B200 (sm_100a) differentiable recursive mesh ray tracer.  C ABI.
 *
 * The hot path of DiffTrans' refine stage (arXiv 2603.00413):
 * for every pixel ray, closest mesh hit; at each hit a Fresnel-weighted reflection and a
 * Snell refraction (total internal reflection drops the refraction); interior segments
 * attenuated by Beer-Lambert absorption; escaping rays end in a lookup of the frozen
 * environment field.  The backward pass returns d/dV, d/dIOR and d/dsigma.
 *
 * Citations: P:n = PAPER.md line n; R# = reading n of DESIGN.md §3 (where the paper is
 * silent or garbled).  All arithmetic is float32 on the device.
 *
 * Conventions shared by every entry point
 *  - Array arguments are caller-owned, contiguous DEVICE memory unless marked "host".
 *    Nothing here allocates caller-visible memory; the context owns its own buffers.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All work
 *    is enqueued on it.  dt_trace_forward synchronises the stream once at its end (it
 *    reads back the wavefront sizes to validate the record arena); nothing else blocks.
 *  - Errors are return codes; nothing throws across the ABI.  dt_last_error(ctx) holds a
 *    one-line message naming the offending argument.  A CUDA fault surfaces as DT_ERR_CUDA.
 *  - A context is bound to one device and is not thread-safe; use one per GPU / thread.
 */
#ifndef DIFFTRANS_H
#define DIFFTRANS_H
#include <stdint.h>

#if defined(__GNUC__)
#define DT_API __attribute__((visibility("default")))
#else
#define DT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dt_ctx dt_ctx;

typedef enum {
  DT_OK = 0,
  DT_ERR_INVALID_ARG = 1,    /* a NULL / out-of-range argument; dt_last_error names it       */
  DT_ERR_EMPTY_GEOMETRY = 2, /* nf == 0 or nv == 0                                            */
  DT_ERR_CUDA = 3,           /* a CUDA runtime error (possibly from earlier async work)      */
  DT_ERR_OOM = 4,            /* device allocation failed (record arena larger than free HBM) */
  DT_ERR_NOT_BUILT = 5,      /* dt_trace_forward before dt_build_bvh                          */
  DT_ERR_NO_FORWARD = 6,     /* dt_trace_backward without a preceding dt_trace_forward        */
  DT_ERR_NONFINITE = 7,      /* opts.check_finite and a NaN/Inf output; message names it     */
  DT_ERR_STACK = 8,          /* BVH deeper than the traversal stack (never for LBVH < 2^30)   */
  DT_ERR_RETRY = 9           /* an asynchronous forward (opts.async) overflowed the record
                                arena: its outputs and the backward that followed it are
                                invalid (zero); the arena has been grown -- re-run that step  */
} dt_status;

enum { DT_ABS_CONST = 0, DT_ABS_GRID = 1, DT_ABS_HASH = 2 };
enum { DT_ENV_ANALYTIC = 0, DT_ENV_GRID = 1, DT_ENV_VOLUME = 2 };
enum { DT_CAP_ZERO = 0, DT_CAP_ENV = 1 };
#define DT_MAX_DEPTH 15

/* Absorption rate mu_t(x), P:124-138 ("differentiable 3D texture").  Per-channel RGB (R11).
 *  CONST: sigma -> float[3].
 *  GRID:  sigma -> float[res][res][res][3] = [z][y][x][c], vertex-centred nodes spanning the
 *         fixed box [box_lo, box_hi]; trilinear; zero outside the box (R11).
 *  HASH:  the paper's iNGP texture (P:138 cites Mueller et al.; R29): sigma -> tables
 *         float[levels][2^log2_size][3]; level l is a grid of level_res[l] cells per axis over
 *         the box, its (N+1)^3 vertices stored densely (index x + (N+1)(y + (N+1) z)) while they
 *         fit in the table, else through iNGP's spatial hash (x*1 ^ y*2654435761 ^
 *         z*805459861) mod 2^log2_size; mu(x) = sum over levels of the trilinear lookups, zero
 *         outside the box.  res is ignored.  levels in [1, 32], log2_size in [1, 26].
 * Interior segments integrate mu with n_samples midpoint samples (R10).  The
 * gradient (dt_trace_backward grad_sigma) has sigma's layout. */
typedef struct {
  int32_t kind;
  const float* sigma;
  int32_t res;
  float box_lo[3], box_hi[3];
  int32_t n_samples;
  int32_t levels;          /* HASH only */
  int32_t log2_size;       /* HASH only */
  int32_t level_res[32];   /* HASH only: cells per axis of each level (N_l >= 1) */
} dt_absorption;

/* Frozen environment radiance, P:91 and P:160 step 3 (R14).
 *  ANALYTIC: L(d) = ambient + sum_j w_j exp(kappa_j (mu_j . d/|d| - 1)); lobes -> float
 *            [n_lobes][7] = mu(3), kappa, w(3).  Direction only.
 *  GRID:     escaping ray looked up once at the shell point p (|p| = radius, or p =
 *            radius * d/|d| if far_field): trilinear(voxel, p) + bilinear(P_xy, p.x, p.y)
 *            + bilinear(P_xz, p.x, p.z) + bilinear(P_yz, p.y, p.z).  voxel -> float
 *            [vres][vres][vres][4] = [z][y][x][rgb_]; planes -> float [3][pres][pres][4]
 *            (P_xy[y][x], P_xz[z][x], P_yz[z][y]); both span [-radius, radius].
 *  VOLUME:   the same textures read as a frozen radiance field (P:91 MERF coarse grid + fine
 *            triplanes; R30): rgb = colour, w = density (clamped at 0).  Every exterior
 *            segment o -> x (camera and reflected/refracted rays outside the object; x = the
 *            next hit, or the shell point for an escaping ray) is volume rendered with
 *            n_samples midpoint samples, V = sum_i T_i (1 - exp(-sigma_i D)) c_i, and its
 *            continuation is attenuated by T = exp(-D sum sigma_i) ("mixed with
 *            the environmental radiance prior to the intersection point").  Escaping rays end
 *            in the GRID shell lookup.  far_field must be 0.
 *  The env is not differentiated (R22).  It must stay alive and unchanged until the
 *  matching dt_trace_backward returns (the backward replays the lookups). */
typedef struct {
  int32_t kind;
  float ambient[3];
  const float* lobes;
  int32_t n_lobes;
  const float* voxel;
  int32_t vres;
  const float* planes;
  int32_t pres;
  float radius;
  int32_t far_field;
  int32_t n_samples;       /* VOLUME only: midpoint samples per exterior segment (>= 1) */
} dt_env;

/* Pinhole cameras, OpenCV axes (R19): d_cam = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1),
 * d = normalize(R d_cam), o = camera centre.  K -> float [n_views][4] = fx, fy, cx, cy;
 * c2w -> float [n_views][3][4] row-major.
 * Rays, in order of precedence:
 *  - pixel_ids != NULL: ray r is pixel pixel_ids[r] (= view*H*W + y*W + x) for r < n_rays;
 *  - tile > 0 (data-parallel shard, SURVEY 8(b) / DESIGN.md §6): the image plane is cut into
 *    tile x tile pixel tiles numbered view-major, then tile row, then tile column
 *    (tiles_x = width / tile per row); this shard holds the tiles listed in tile_ids (device
 *    int32 [n_tiles], e.g. a longest-processing-time assignment) or, when tile_ids is NULL,
 *    every tile with id % shard_count == shard_rank.  Ray r is pixel (r mod tile^2) of the
 *    shard's tile r / tile^2, with a tile's pixels in 8 x 4 micro-tiles in row-major order
 *    (a warp's 32 rays are one screen-space block); n_rays is ignored (= tiles x tile^2).
 *    width and height must be multiples of tile, and tile a multiple of 8;
 *  - else every pixel of every view, ray r = pixel id r, n_rays ignored.
 * K, c2w, pixel_ids and tile_ids are read during dt_trace_forward only. */
typedef struct {
  int32_t n_views, width, height;
  const float* K;
  const float* c2w;
  const int64_t* pixel_ids;
  int64_t n_rays;
  int32_t tile;
  int32_t shard_rank, shard_count;
  const int32_t* tile_ids;
  int32_t n_tiles;
} dt_cameras;

/* max_depth = D_max (R12): segments at depth 0..D_max are intersection-tested; a
 * hit on a depth-D_max segment is capped.  cap_policy: DT_CAP_ZERO returns 0 for a capped
 * branch ("discarded", R13); DT_CAP_ENV returns tau * Env(o, d).  t_eps: secondary
 * rays start at the hit point with t > t_eps * bbox diagonal (R17); default 1e-4. */
typedef struct {
  int32_t max_depth;
  int32_t cap_policy;
  float t_eps;
  int32_t check_finite;      /* nonzero: verify rgb is finite (extra pass + sync)  */
  int32_t async;             /* nonzero: do not synchronise at the end of the forward.  The
                                arena is sized from the previous forward's measured need (+25%
                                headroom); its overflow check is deferred to the next
                                dt_trace_forward / dt_get_stats, which then returns
                                DT_ERR_RETRY.  Ignored (synchronous) when stats or
                                check_finite are requested or no previous need is known.   */
  const float* ior_device;   /* optional device float[1]: when non-NULL the IoR is read from
                                it by the kernels (forward and the matching backward) instead
                                of the `ior` argument, so an on-device optimiser update needs
                                no host round trip.  Must not change before the backward.    */
  int32_t* seg_count;        /* optional device int32[n_rays], ACCUMULATED: += the number of
                                segments traced for each ray (its ray tree's nodes at depth >= 1
                                plus the camera segment if it passed the root-box test); the
                                multi-GPU tile balancer's cost.  NULL: off.    */
} dt_trace_opts;

/* Host-side statistics filled by dt_trace_forward when requested. */
typedef struct {
  int64_t segments_per_depth[DT_MAX_DEPTH + 1]; /* records traced at each depth (level 0 = hits) */
  int64_t primaries;          /* camera rays                                                     */
  int64_t primaries_traced;   /* camera rays that passed the root-AABB test and were traversed   */
  int64_t segments;           /* traced segments = primaries_traced + sum_{k>=1} depth k        */
  int64_t arena_capacity;     /* path-record capacity (records)                                 */
  int32_t arena_retries;      /* forward re-runs after growing the arena (0 in steady state)    */
  int32_t bvh_depth;          /* 0 unless dt_debug_bvh_check ran                                */
} dt_stats;

DT_API dt_status dt_create(int32_t device, dt_ctx** out);
DT_API void dt_destroy(dt_ctx* ctx);
DT_API const char* dt_last_error(const dt_ctx* ctx);
DT_API const char* dt_status_string(dt_status s);

/* Snapshot the mesh and rebuild the acceleration structure (rebuilt every step
 * because the mesh moves): vertex normals n_v = normalize(sum of incident unit face
 * normals) (R6), then an LBVH (Morton codes, radix sort, Karras hierarchy,
 * bottom-up AABB refit).  V -> float [nv][3]; F -> int32 [nf][3], CCW = outward (R8).
 * The context copies V and F: the caller may modify V right after this returns (on the
 * stream).  Errors: DT_ERR_EMPTY_GEOMETRY if nv or nf is 0; DT_ERR_INVALID_ARG for NULL. */
DT_API dt_status dt_build_bvh(dt_ctx* ctx, const float* V, int32_t nv, const int32_t* F, int32_t nf, void* stream);

/* Build quality of the following dt_build_bvh calls: the number of treelet-restructuring
 * passes (Karras & Aila 2013) over the Karras hierarchy, 0..4 (default 2).  Each pass costs
 * about 0.5 ms per million triangles on a B200 and lowers the traversal's node visits (C3:
 * -6.6% at 2 passes); 0 suits builds that serve few rays (the paper's 5,000-ray batches).
 * The closest hits are the same at every quality (the tree is a search structure only). */
DT_API dt_status dt_set_bvh_quality(dt_ctx* ctx, int32_t treelet_passes);

/* Forward recursive trace (P:154-163 steps 1-5) of every ray of `cams`.
 *  ior:       eta_o of the object (R1).
 *  rgb:       out float [n_rays][3], radiance.
 *  capped_w:  out float [n_rays] or NULL: sum over capped branches of the R/T path weight.
 *  sig_topo:  out uint64 [n_rays] or NULL: order-independent signature of the ray tree
 *             (tree position + event per node), sig_face likewise including face ids
 *             (parity protocol).
 *  stats:     host dt_stats or NULL.
 * Path records stay in the context until the next forward; the absorption field is
 * snapshotted for the backward.  Synchronises `stream` once. */
DT_API dt_status dt_trace_forward(dt_ctx* ctx, float ior, const dt_absorption* absorption, const dt_env* env,
                           const dt_cameras* cams, const dt_trace_opts* opts, float* rgb, float* capped_w,
                           uint64_t* sig_topo, uint64_t* sig_face, dt_stats* stats, void* stream);

/* Reverse mode of the last forward ("The IoR ... is differentiable"):
 * the VJP of sum(grad_rgb * rgb) at fixed path topology (R22).
 *  grad_rgb:   in  float [n_rays][3].
 *  grad_V:     out float [nv][3]; grad_ior: out float [1]; grad_sigma: out float [3] or
 *              [res^3][3] matching the forward's absorption.  Any may be NULL (skipped).
 *  accumulate: 0 overwrites the outputs, nonzero adds to them.
 * Gradients are w.r.t. sigma itself; any activation is the caller's chain rule.
 * Float atomics make the result nondeterministic at the ulp level. */
DT_API dt_status dt_trace_backward(dt_ctx* ctx, const float* grad_rgb, float* grad_V, float* grad_ior, float* grad_sigma,
                            int32_t accumulate, void* stream);

/* L_color of P:177-180, its gradient fused: loss = (1/B) sum_i ||(rgb_i - target_i) * target_i||^2
 * (elementwise *), grad_rgb = 2 (rgb - target) * target^2 / B with B = n_rays.
 * rgb, target -> float [n][3]; grad_rgb out [n][3]; loss out float [1] (device). */
DT_API dt_status dt_loss_color(dt_ctx* ctx, const float* rgb, const float* target, int64_t n, float* grad_rgb, float* loss,
                        void* stream);

/* Profiling.  With profiling enabled the library brackets each phase's launches with CUDA
 * events on the caller's stream (no extra synchronisation) and accumulates their device
 * time; dt_get_profile resolves pending events (synchronising on them) and returns the
 * totals since the last reset.  Traversal counters and the kernel-launch count are always
 * maintained.  Phases: */
enum { DT_PH_BUILD = 0, DT_PH_TRACE0 = 1, DT_PH_SHADE = 2, DT_PH_TRACE = 3, DT_PH_GATHER = 4, DT_PH_BWD = 5,
       DT_PH_NORMALS_BWD = 6, DT_PH_LOSS = 7, DT_PH_COUNT = 8 };
typedef struct {
  double ms[DT_PH_COUNT];          /* summed device time per phase                           */
  int64_t launches[DT_PH_COUNT];   /* kernel launches per phase                              */
  int64_t kernel_launches;         /* all kernels this context launched since the reset     */
  int64_t node_visits;             /* LBVH inner nodes fetched by the trace kernels          */
  int64_t tri_tests;               /* ray-triangle tests by the trace kernels                */
  int64_t node_visits_primary;     /* the part of node_visits made by camera rays (depth 0)  */
  int64_t tri_tests_primary;       /* the part of tri_tests made by camera rays (depth 0)    */
  int64_t segments;                /* traced segments of all forwards since the reset        */
  int64_t walk_cells_fwd;          /* cell visits of the sigma-grid / hash-texture walks of   *
                                    * the forward (each: 8 corner fetches)                    */
  int64_t walk_cells_bwd;          /* the same of the backward (each: 8 corner fetches and   *
                                    * 8 float4 adjoint atomics)                               */
  int64_t env_samples_bwd;         /* volumetric-env samples replayed by the backward (each:   *
                                    * 8 voxel + 12 plane texel fetches)                       */
} dt_profile;
/* ---------------------------------------------------------------------------------------
 * The optimisation step around the tracer (PAPER P:176-194, P:439-443,
 * P:511-527).  All device pointers; `loss` outputs are device float arrays, overwritten.
 * --------------------------------------------------------------------------------------- */

/* Photometric losses of P:177-185 and their gradient w.r.t. the rendered colours, fused:
 *   L_color = (1/B) sum_i ||(c^_i - c_i) * c_i||^2                         (elementwise *)
 *   L_tone  = (1/B) sum_i [(1 - cos(c^_i, c_i))^2 - var(c_i)]
 * B = n; pairs with |c^| or |c| <= 1e-6 are skipped in L_tone (its cosine is undefined);
 * var is the population variance of the 3 channels (constant w.r.t. c^).  mask (optional,
 * [n]) multiplies each ray's terms (e.g. to drop rays the caller considers capped).
 * grad_rgb = lambda_color dL_color/dc^ + lambda_tone dL_tone/dc^  ([n][3], overwritten);
 * loss[0] = L_color, loss[1] = L_tone (unweighted). */
DT_API dt_status dt_loss_rt(dt_ctx* ctx, const float* rgb, const float* target, const float* mask, int64_t n,
                            float lambda_color, float lambda_tone, float* grad_rgb, float* loss, void* stream);

/* Absorption regularisers on n caller-drawn points v_i ([n][3]) with perturbations xi_i:
 *   L_mat-smooth = (1/n) sum_i sum_c |mu_c(v_i) - mu_c(v_i + xi_i)|
 *   L_vol        = (1/n) sum_i ||mu(v_i)||^2                              (mean form)
 * mu is the absorption field of `absorption` (R11: zero outside the grid box; constant
 * sigma everywhere).  grad_sigma (same layout as absorption.sigma) is ACCUMULATED with
 * lambda_smooth dL_mat/dsigma + lambda_vol dL_vol/dsigma; loss[0] = L_mat, loss[1] = L_vol.
 * (|x| has derivative sign(x), 0 at 0.) */
DT_API dt_status dt_sigma_regularizers(dt_ctx* ctx, const dt_absorption* absorption, const float* points,
                                       const float* xi, int64_t n, float lambda_smooth, float lambda_vol,
                                       float* grad_sigma, float* loss, void* stream);

/* Periodic mesh regularisers of the current dt_build_bvh snapshot:
 *   L_edge = (1/|E'|) sum_{(i,j) in E'} (1 - n_i . n_j)^2   (n = R6 vertex normals)
 *   L_lap  = (1/|V|) sum_i |v_i - mean_{j in N(i)} v_j|^2   (Nicolet et al.'s uniform
 *            Laplacian, read as its energy, R31)
 * E' = the mesh's undirected edges, N(i) = vertex i's neighbours (from the faces).
 * grad_V [nv][3] (device) += lambda_edge dL_edge/dV + lambda_lap dL_lap/dV; loss [2] (device)
 * = (L_edge, L_lap), unweighted.  Deterministic (per-vertex gathers).  DT_ERR_NOT_BUILT
 * before dt_build_bvh. */
DT_API dt_status dt_mesh_regularizers(dt_ctx* ctx, float lambda_edge, float lambda_lap, float* grad_V, float* loss,
                                      void* stream);

/* Mask regulariser (R32) of the current dt_build_bvh
 * snapshot over full images: the rendered mask M^ (1 where the camera ray through the pixel
 * centre hits the mesh), loss[0] = (1/N) sum |M^ - gt_mask| (N = n_views W H; gt_mask device
 * float [n_views][H][W] in [0, 1]), and grad_V [nv][3] (device) += lambda d/dV of the
 * area-coverage relaxation, estimated by silhouette-edge sampling: every projected silhouette
 * edge (faces of opposite facing, or a boundary edge) is sampled every 0.5 px; a sample on the
 * outer boundary (covered 0.02 px inside, not outside) pushes its edge's two vertices through
 * the pinhole Jacobian by (1 - 2 gt(outside pixel)) / N per unit length.  mask_out (device
 * float [n_views][H][W]) or NULL.  cams->pixel_ids must be NULL.  The per-vertex sums use float
 * atomics (order-dependent at the ulp level). */
DT_API dt_status dt_mask_loss(dt_ctx* ctx, const dt_cameras* cams, const float* gt_mask, float lambda, float* grad_V,
                              float* loss, float* mask_out, void* stream);

/* Adam (beta = (0.9, 0.999), weight decay 1e-6 added to the gradient as in
 * torch.optim.Adam) on n parameters, in place: m, v are [n] state buffers (zero at step 1).
 * uniform != 0: AdamUniform (Nicolet et al., cited at P:186) -- one second-moment statistic
 * for the whole block, v[0] = beta2 v[0] + (1 - beta2) max_i g_i^2, so every coordinate
 * keeps its gradient's relative scale (R26).  step = t >= 1 (bias correction). */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int32_t step;
  int32_t uniform;
  float clamp_lo, clamp_hi;  /* projection after the update (e.g. IoR in [1, 3], sigma >= 0) */
  const int32_t* skip_if;    /* optional device int: when non-NULL and *skip_if != 0 at run time
                                the update is skipped (param, m, v untouched).  Pass
                                dt_forward_overflow_flag() so a step whose asynchronous forward
                                overflowed the arena (its gradients are invalid) changes nothing. */
  int32_t* step_device;      /* optional device int (CUDA-graph replays): when non-NULL the step
                                t is read from it at run time instead of `step` (which is then
                                ignored; *step_device must hold t >= 1) and, unless the update was
                                skipped, incremented by 1 after the update, so one captured step
                                replays with the right bias correction every time. */
} dt_adam;
DT_API dt_status dt_adam_step(dt_ctx* ctx, float* param, const float* grad, float* m, float* v, int64_t n,
                              const dt_adam* cfg, void* stream);

/* Device int32, nonzero iff the most recent dt_trace_forward on this context overflowed its
 * record arena (its outputs and the following backward are invalid).  Reset by the next
 * forward; valid for the context's lifetime (stream-ordered: read it in later kernels, e.g.
 * dt_adam.skip_if).  NULL for a NULL context. */
DT_API const int32_t* dt_forward_overflow_flag(const dt_ctx* ctx);

/* Statistics of the last forward (waits for it if it ran with opts.async).  Returns
 * DT_ERR_RETRY if that asynchronous forward overflowed the arena.
 * CUDA graphs: dt_trace_forward may be captured into a graph (stream capture on `stream`)
 * once an asynchronous forward of the same ray count has run on the context and been checked
 * (dt_get_stats) and profiling is off; the captured forward copies its level counts to host
 * memory on every replay, so after the replays have completed (the caller synchronises the
 * replay stream) dt_get_stats reports the last replay's statistics, or DT_ERR_RETRY if it
 * overflowed the arena (the arena is grown: the graph must be captured again).  Capture
 * never allocates: a forward that would need to grow the arena fails with
 * DT_ERR_INVALID_ARG instead. */
DT_API dt_status dt_get_stats(dt_ctx* ctx, dt_stats* out);
DT_API dt_status dt_set_profiling(dt_ctx* ctx, int32_t enable);
DT_API dt_status dt_get_profile(dt_ctx* ctx, dt_profile* out, int32_t reset);

/* Test-only: closest hit of n rays (rays -> float [n][6] = o.xyz, d.xyz) with t > t_lo via the
 * LBVH (brute_force = 0) or by testing every face with the same routine (brute_force = 1).
 * face out int32 [n] (original face id, -1 = miss); tuv out float [n][3]. */
DT_API dt_status dt_debug_closest_hit(dt_ctx* ctx, const float* rays, int64_t n, float t_lo, int32_t brute_force,
                               int32_t* face, float* tuv, void* stream);

/* Test-only: validate the LBVH (host out int64[4]): [0] boxes not containing their child's
 * box, [1] leaves reached from the root, [2] distinct faces reached, [3] tree depth. */
DT_API dt_status dt_debug_bvh_check(dt_ctx* ctx, int64_t* out, void* stream);

/* Test-only: copy the vertex normals of the last build to out (device float [nv][3]). */
DT_API dt_status dt_debug_vertex_normals(dt_ctx* ctx, float* out, void* stream);

/* Test-only: status of the bounds-checked build (compiled with -DDT_CHECKED=1; every kernel
 * checks its record, node, triangle, vertex, texel and shared-slot indices).  Synchronises
 * the device, then returns the source line of the first failed check in each translation
 * unit (host out int32[5]: bvh.cu, trace.cu, optim.cu, meshreg.cu, api.cu; 0 = no failure)
 * and clears them.  In the product build every entry is -1 (no checks compiled in). */
DT_API dt_status dt_debug_check_status(int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
