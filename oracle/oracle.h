/* DiffTrans CPU oracle — C ABI.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle.so.  The product path (paper_2603_00413_b200/, libdifftrans.so)
 * never includes this header or links this library, and this library includes nothing
 * from the product path.
 *
 * All inputs are the raw float32/int32 arrays written by paper_2603_00413_b200/scenes.py;
 * all arithmetic is float64.  Citations: P:n = /root/reference/PAPER.md line n;
 * R# = the readings in DESIGN.md §3 (taken from SURVEY.md §8c.1).
 */
#ifndef DIFFTRANS_ORACLE_H
#define DIFFTRANS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  /* mesh M = (V, F); V [nv][3], F [nf][3] (CCW = outward) */
  int32_t nv, nf;
  const float* V;
  const int32_t* F;
  double ior;                       /* eta_o of the object, P:110 (R1)                 */
  /* absorption mu_t, P:124-138 (R10, R11) */
  int32_t abs_kind;                 /* 0 = constant [3], 1 = grid [R][R][R][3] = [z][y][x][c], 2 = hash */
  const float* sigma;
  int32_t sigma_res;
  float sigma_lo[3], sigma_hi[3];
  int32_t n_samples;                /* N_sigma midpoint samples per interior segment    */
  /* frozen environment, P:91 / P:160 (R14) */
  int32_t env_kind;                 /* 0 = analytic lobes, 1 = voxel + triplane shell, 2 = volume */
  float ambient[3];
  const float* lobes;               /* [n_lobes][7] = mu(3), kappa, w(3)                */
  int32_t n_lobes;
  const float* voxel;               /* [vres]^3 [4] = [z][y][x][rgb_]                   */
  int32_t vres;
  const float* planes;              /* [3][pres][pres][4]: P_xy[y][x], P_xz[z][x], P_yz[z][y] */
  int32_t pres;
  float env_radius;
  int32_t far_field;
  /* pinhole cameras (R19) */
  int32_t n_views, width, height;
  const float* K;                   /* [n_views][4] = fx, fy, cx, cy                    */
  const float* c2w;                 /* [n_views][3][4] row-major                        */
  /* options */
  int32_t max_depth;                /* D_max, P:158 (R12)                               */
  int32_t cap_policy;               /* 0 = CAP_ZERO, 1 = CAP_ENV (R13)                  */
  double t_eps;                     /* t_min = t_eps * bbox diagonal (R17)              */
  /* optional float64 overrides (NULL = use V / sigma): finite-difference pins perturb in double */
  const double* V64;
  const double* sigma64;
  /* abs_kind 2 = multiresolution hash grid ("differentiable 3D texture", R29): sigma ->
   * tables [hash_levels][2^hash_log2_size][3]; level l has hash_res[l] cells per axis over the
   * box; mu = sum over levels of the trilinear lookup (dense index when (N+1)^3 <= T, else
   * the spatial hash (x * 1) ^ (y * 2654435761) ^ (z * 805459861) mod T). */
  int32_t hash_levels;
  int32_t hash_log2_size;
  int32_t hash_res[32];
  /* env_kind 2 = volumetric env (P:91 MERF grid + triplanes, "mixed with the
   * environmental radiance prior to the intersection point"; R30): the voxel/planes textures
   * give colour (rgb) and density (w, clamped >= 0); every exterior segment is volume
   * rendered with env_samples midpoint samples; escaping rays end in the shell lookup. */
  int32_t env_samples;
} dto_scene;

/* Per-ray flag bits (parity protocol). */
#define DTO_FLAG_EDGE    1  /* some node hit within 1e-5 (barycentric) of an edge, near-missed a face, or tied */
#define DTO_FLAG_GRAZING 2  /* some node had cos(theta_i) < 1e-3 (incl. clamp)                   */
#define DTO_FLAG_NEARTIR 4  /* some node had |eta^2 - sin^2| < 1e-4 (R depends on it like 1/sqrt)      */

/* Ray source for every entry point below: if `rays` != NULL it holds [n][6] =
 * (o.xyz, d.xyz) primary rays; else pixel ids view*H*W + y*W + x through the cameras. */

/* Forward radiance.  rgb [n][3].  Optional (may be NULL): capped_w [n] (sum of the scalar
 * R/T path weights of capped branches), sig_topo/sig_face [n] (order-independent path
 * signatures), flags [n], segments [n] (traced segments per ray). */
int dto_render(const dto_scene* s, const int64_t* pixel_ids, const double* rays, int64_t n,
               double* rgb, double* capped_w, uint64_t* sig_topo, uint64_t* sig_face,
               int32_t* flags, int64_t* segments, int nthreads);

/* Hand-derived reverse mode (Appendix B of DESIGN.md): VJP of sum(grad_rgb * rgb) w.r.t.
 * V (gV [nv][3]), ior (gior [1]) and sigma (gsigma [3] or [R^3*3]).  Overwrites. */
int dto_backward(const dto_scene* s, const int64_t* pixel_ids, const double* rays, int64_t n,
                 const double* grad_rgb, double* gV, double* gior, double* gsigma, int nthreads);

/* Forward-mode (dual numbers) JVP of rgb along tangent (tV [nv][3], tior, tsigma). */
int dto_jvp(const dto_scene* s, const int64_t* pixel_ids, const double* rays, int64_t n,
            const double* tV, double tior, const double* tsigma, double* rgb, double* jvp_rgb,
            int nthreads);

/* Brute-force closest hit (R16-R18) of n rays [n][6] with t > t_lo.
 * face [n] (-1 = miss), tuv [n][3], flags [n]. */
int dto_closest_hit(const dto_scene* s, const double* rays, int64_t n, double t_lo,
                    int32_t* face, double* tuv, int32_t* flags, int nthreads);

/* Camera rays (R19) of the given pixels: rays [n][6] = o.xyz, d.xyz (float64). */
int dto_camera_rays(const dto_scene* s, const int64_t* pixel_ids, int64_t n, double* rays);

/* Pieces, exposed for the closed-form pins. */
int dto_vertex_normals(const dto_scene* s, double* out /* [nv][3] */);
/* d: incoming ray direction, n: unit normal oriented against d.  out[12] =
 * ci, R, T, tir, wr.xyz, wt.xyz (0 if tir), ct */
int dto_interface(const double* d, const double* n, double eta_i, double eta_t, double* out);
int dto_env(const dto_scene* s, const double* o, const double* d, double* out /* [3] */);
int dto_transmittance(const dto_scene* s, const double* o, const double* x, double* out /* [3] */);

#ifdef __cplusplus
}
#endif
#endif
