/* DiffTrans CPU oracle.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow, float64 restatement of the paper's refine-stage tracer:
 *   - brute-force closest hit over ALL faces for every segment (no acceleration structure);
 *   - depth-first recursion exactly in the order of P:157-163 ("Recursive Ray Tracing",
 *     steps 1-5);
 *   - reverse mode written out by hand, node by node, in post-order (Appendix B of
 *     DESIGN.md), and a separate forward mode (dual numbers) used only to check it.
 * No blocking, fusion or reordering.  Shares no code with paper_2603_00413_b200/csrc.
 * Where the paper is silent or garbled the reading named R# in DESIGN.md §3 is followed.
 * Parts that are our readings, with no value printed in the paper to pin them (DESIGN.md §2,
 * "parity unpinned w.r.t. the paper"): the voxel + triplane shell env lookup (R14), the
 * midpoint N_sigma quadrature (R10), the hash texture (R29) and the volume env (R30).  They are
 * pinned by their own closed forms (constant / linear fields, one dense hash level == the
 * vertex grid, zero density == the shell env) and by the FD and dot-product tests.
 */
#include "oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace {

// ----------------------------------------------------------------------------- scalars
// Dual numbers for the forward-mode check (dto_jvp).  The value part performs exactly
// the double operations, so discrete decisions are identical to the double tracer.
struct Dual {
  double v, d;
  Dual(double v_ = 0.0, double d_ = 0.0) : v(v_), d(d_) {}
};
inline Dual operator+(Dual a, Dual b) { return Dual(a.v + b.v, a.d + b.d); }
inline Dual operator-(Dual a, Dual b) { return Dual(a.v - b.v, a.d - b.d); }
inline Dual operator-(Dual a) { return Dual(-a.v, -a.d); }
inline Dual operator*(Dual a, Dual b) { return Dual(a.v * b.v, a.d * b.v + a.v * b.d); }
inline Dual operator/(Dual a, Dual b) { return Dual(a.v / b.v, (a.d * b.v - a.v * b.d) / (b.v * b.v)); }
inline Dual sqrt(Dual a) {
  double s = std::sqrt(a.v);
  return Dual(s, s > 0.0 ? a.d / (2.0 * s) : 0.0);  // derivative at 0 taken as 0 (R5)
}
inline Dual exp(Dual a) { double e = std::exp(a.v); return Dual(e, a.d * e); }
inline double exp(double a) { return std::exp(a); }
inline double sqrt(double a) { return std::sqrt(a); }
inline double val(double x) { return x; }
inline double val(const Dual& x) { return x.v; }
inline double safe_sqrt(double x) { return std::sqrt(x); }
inline Dual safe_sqrt(Dual x) { return sqrt(x); }
template <class S> S lift(double v, double d);
template <> double lift<double>(double v, double) { return v; }
template <> Dual lift<Dual>(double v, double d) { return Dual(v, d); }

// ----------------------------------------------------------------------------- vectors
template <class S> struct V3 { S x, y, z; };
using V3d = V3<double>;
template <class S> inline V3<S> mk(S x, S y, S z) { return V3<S>{x, y, z}; }
template <class S> inline V3<S> operator+(V3<S> a, V3<S> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class S> inline V3<S> operator-(V3<S> a, V3<S> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class S> inline V3<S> operator-(V3<S> a) { return {-a.x, -a.y, -a.z}; }
template <class S> inline V3<S> scl(V3<S> a, S s) { return {a.x * s, a.y * s, a.z * s}; }
template <class S> inline V3<S> mul(V3<S> a, V3<S> b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
template <class S> inline S dot(V3<S> a, V3<S> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class S> inline V3<S> cross(V3<S> a, V3<S> b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class S> inline S norm(V3<S> a) { return safe_sqrt(dot(a, a)); }
template <class S> inline V3d vald(V3<S> a) { return {val(a.x), val(a.y), val(a.z)}; }
template <class S> inline S comp(const V3<S>& a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
template <class S> inline void addc(V3<S>& a, int i, S v) { if (i == 0) a.x = a.x + v; else if (i == 1) a.y = a.y + v; else a.z = a.z + v; }
template <class S> inline V3<S> zero3() { return {S(0.0), S(0.0), S(0.0)}; }

// ----------------------------------------------------------------------------- signatures
// splitmix64 finaliser; the per-ray signature is the wrapping SUM of mix(key) over the
// nodes of the ray tree, so it does not depend on traversal order.
inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
enum Event { EV_MISS = 0, EV_HIT_OUT = 1, EV_HIT_IN = 2, EV_HIT_OUT_TIR = 3, EV_HIT_IN_TIR = 4,
             EV_CAP_OUT = 5, EV_CAP_IN = 6, EV_CAP_DROP = 7 };
inline uint64_t topo_key(uint64_t pos, int ev) { return pos | ((uint64_t)ev << 32); }
inline uint64_t face_key(uint64_t pos, int ev, int face) {
  return pos | ((uint64_t)(uint32_t)(face + 1) << 20) | ((uint64_t)ev << 52);
}


// ----------------------------------------------------------------------------- precision study
// Built only with -DDTO_PRECISION_STUDY (tools/precision_study.py; never in liboracle.so):
// rounds the value at one stage of the method to float32, to measure which stage's float32
// rounding moves the radiance.  Stage bits: 1 camera ray, 2 hit point (child
// origin), 4 child directions, 8 vertex normals, 16 shading normal, 32 env shell point,
// 64 barycentrics (u, v) of the hit.
#ifdef DTO_PRECISION_STUDY
int g_study_mask = 0;
inline void study_round(double& x, int bit) { if (g_study_mask & bit) x = (double)(float)x; }
inline void study_round(Dual&, int) {}
template <class S> inline void study_round(V3<S>& a, int bit) { study_round(a.x, bit); study_round(a.y, bit); study_round(a.z, bit); }
#define DTO_STUDY(x, bit) study_round(x, bit)
#else
#define DTO_STUDY(x, bit) ((void)0)
#endif

const double BAND_BETA = 1e-5;   // edge band for the parity flags

// ----------------------------------------------------------------------------- model
template <class S> struct Model {
  const dto_scene* sc = nullptr;
  int nv = 0, nf = 0;
  std::vector<V3<S>> V;       // vertex positions (differentiable)
  std::vector<V3d> Vd;        // val(V): drives the discrete decisions
  std::vector<V3<S>> nrm;     // vertex normals n_v (R6)
  S ior;                      // eta_o
  std::vector<S> sigma;       // [3] or [R^3 * 3]
  double t_min = 0.0;         // secondary-ray t_lo (R17)
};

// n_v = normalize(sum over incident faces of the unit face normal)  (R6:
// the garbled 1/3 cancels in the normalisation; zero-area faces add 0; a zero sum
// gives (0,0,1), which no hit ever reads).
template <class S>
void vertex_normals(const std::vector<V3<S>>& V, const int32_t* F, int nf, std::vector<V3<S>>& out) {
  out.assign(V.size(), zero3<S>());
  for (int f = 0; f < nf; ++f) {
    const V3<S>& v0 = V[F[3 * f]]; const V3<S>& v1 = V[F[3 * f + 1]]; const V3<S>& v2 = V[F[3 * f + 2]];
    V3<S> c = cross(v1 - v0, v2 - v0);
    S L = norm(c);
    if (!(val(L) > 0.0)) continue;
    V3<S> h = scl(c, S(1.0) / L);
    for (int k = 0; k < 3; ++k) out[F[3 * f + k]] = out[F[3 * f + k]] + h;
  }
  for (auto& n : out) {
    S L = norm(n);
    n = val(L) > 0.0 ? scl(n, S(1.0) / L) : mk<S>(S(0.0), S(0.0), S(1.0));
    DTO_STUDY(n, 8);
  }
}

// Number of absorption parameters (R11, R29).
size_t sigma_len(const dto_scene* sc) {
  if (sc->abs_kind == 0) return 3;
  if (sc->abs_kind == 2) return (size_t)sc->hash_levels * ((size_t)1 << sc->hash_log2_size) * 3;
  return (size_t)sc->sigma_res * sc->sigma_res * sc->sigma_res * 3;
}

template <class S>
Model<S> make_model(const dto_scene* sc, const double* tV, double tior, const double* tsig) {
  Model<S> m;
  m.sc = sc; m.nv = sc->nv; m.nf = sc->nf;
  m.V.resize(m.nv); m.Vd.resize(m.nv);
  for (int i = 0; i < m.nv; ++i) {
    double x = sc->V64 ? sc->V64[3 * i] : sc->V[3 * i], y = sc->V64 ? sc->V64[3 * i + 1] : sc->V[3 * i + 1],
           z = sc->V64 ? sc->V64[3 * i + 2] : sc->V[3 * i + 2];
    m.V[i] = {lift<S>(x, tV ? tV[3 * i] : 0.0), lift<S>(y, tV ? tV[3 * i + 1] : 0.0), lift<S>(z, tV ? tV[3 * i + 2] : 0.0)};
    m.Vd[i] = vald(m.V[i]);
  }
  vertex_normals(m.V, sc->F, m.nf, m.nrm);
  m.ior = lift<S>(sc->ior, tior);
  size_t ns = sigma_len(sc);
  m.sigma.resize(ns);
  for (size_t i = 0; i < ns; ++i)
    m.sigma[i] = lift<S>(sc->sigma64 ? sc->sigma64[i] : (double)sc->sigma[i], tsig ? tsig[i] : 0.0);
  // t_min = t_eps * bbox diagonal of V (R17)
  V3d lo = m.Vd.empty() ? V3d{0, 0, 0} : m.Vd[0], hi = lo;
  for (auto& v : m.Vd) {
    lo = {std::min(lo.x, v.x), std::min(lo.y, v.y), std::min(lo.z, v.z)};
    hi = {std::max(hi.x, v.x), std::max(hi.y, v.y), std::max(hi.z, v.z)};
  }
  m.t_min = sc->t_eps * norm(hi - lo);
  return m;
}

// ----------------------------------------------------------------------------- cameras
// Pinhole, OpenCV axes; d_cam = ((x+0.5-cx)/fx, (y+0.5-cy)/fy, 1), d = normalize(R d_cam),
// o = camera centre (R19).  Rays are not differentiated (R22).
void camera_ray(const dto_scene* sc, int64_t pid, V3d& o, V3d& d) {
  int64_t hw = (int64_t)sc->width * sc->height;
  int64_t view = pid / hw, rem = pid % hw;
  int64_t y = rem / sc->width, x = rem % sc->width;
  const float* K = sc->K + 4 * view;
  const float* M = sc->c2w + 12 * view;
  V3d dc = {((double)x + 0.5 - K[2]) / K[0], ((double)y + 0.5 - K[3]) / K[1], 1.0};
  V3d w = {M[0] * dc.x + M[1] * dc.y + M[2] * dc.z, M[4] * dc.x + M[5] * dc.y + M[6] * dc.z,
           M[8] * dc.x + M[9] * dc.y + M[10] * dc.z};
  d = scl(w, 1.0 / norm(w));
  o = {M[3], M[7], M[11]};
}

// ----------------------------------------------------------------------------- intersection
// Moller-Trumbore: (u, v, t) solve o + t d = v0 + u e1 + v e2 (R15, R16).
template <class S> struct MT { bool ok; S t, u, v; };
template <class S>
MT<S> moller_trumbore(V3<S> o, V3<S> d, V3<S> v0, V3<S> v1, V3<S> v2) {
  V3<S> e1 = v1 - v0, e2 = v2 - v0;
  V3<S> p = cross(d, e2);
  S det = dot(e1, p);
  if (val(det) == 0.0) return {false, S(0.0), S(0.0), S(0.0)};
  S inv = S(1.0) / det;
  V3<S> s = o - v0;
  S u = dot(s, p) * inv;
  V3<S> q = cross(s, e1);
  S v = dot(d, q) * inv;
  S t = dot(e2, q) * inv;
  return {true, t, u, v};
}

struct Hit { int face; double t, u, v; int flags; };

// Closest hit over ALL faces (P:158-159 step 2, "the first triangle that the ray
// intersects").  Hit iff det != 0, u >= 0, v >= 0, u + v <= 1 (edge-inclusive),
// t > t_lo; no back-face culling (R16).  Equal t -> lowest face id (R18).
template <class S>
Hit closest_hit(const Model<S>& m, V3d o, V3d d, double t_lo) {
  Hit best{-1, std::numeric_limits<double>::infinity(), 0, 0, 0};
  double second = std::numeric_limits<double>::infinity();
  double near_t = std::numeric_limits<double>::infinity();
  const int32_t* F = m.sc->F;
  for (int f = 0; f < m.nf; ++f) {
    MT<double> r = moller_trumbore<double>(o, d, m.Vd[F[3 * f]], m.Vd[F[3 * f + 1]], m.Vd[F[3 * f + 2]]);
    if (!r.ok || !(r.t > t_lo)) continue;
    double mb = std::min(std::min(1.0 - r.u - r.v, r.u), r.v);
    if (mb >= 0.0) {
      if (r.t < best.t) { second = best.t; best = {f, r.t, r.u, r.v, 0}; }
      else if (r.t < second) second = r.t;
    } else if (mb >= -BAND_BETA) {
      near_t = std::min(near_t, r.t);
    }
  }
  if (best.face >= 0) {
    double mb = std::min(std::min(1.0 - best.u - best.v, best.u), best.v);
    if (mb < BAND_BETA) best.flags |= DTO_FLAG_EDGE;
    if (second - best.t <= 1e-6 * std::max(1.0, best.t)) best.flags |= DTO_FLAG_EDGE;
    if (near_t <= best.t * (1.0 + 1e-6)) best.flags |= DTO_FLAG_EDGE;
  } else if (near_t < std::numeric_limits<double>::infinity()) {
    best.flags |= DTO_FLAG_EDGE;
  }
  return best;
}

// ----------------------------------------------------------------------------- optics
// One specular interface.  d = incoming direction, n = unit normal oriented
// into omega_i's hemisphere, omega_i = -d (R3).  eta = eta_t / eta_i (R1); cos(theta_i) =
// omega_i . n (R2) clamped to [0,1]; the lower clamp stops the gradient, the upper one
// only guards rounding and passes it (R3).
template <class S> struct Iface {
  S c_raw, ci, eta, q, ct, R, T;
  bool tir, clamped, degen = false;
  V3<S> wi, wr, wt;
};
template <class S>
Iface<S> interface(V3<S> d, V3<S> n, S eta_i, S eta_t) {
  Iface<S> I;
  I.wi = -d;
  I.c_raw = dot(I.wi, n);
  I.clamped = !(val(I.c_raw) > 0.0);
  if (I.clamped) I.ci = S(0.0);
  else if (val(I.c_raw) > 1.0) I.ci = I.c_raw + S(1.0 - val(I.c_raw));  // value 1, gradient kept
  else I.ci = I.c_raw;
  I.eta = eta_t / eta_i;
  I.q = I.eta * I.eta - S(1.0) + I.ci * I.ci;                       // eta^2 - sin^2(theta_i)
  I.wr = scl(n, S(2.0) * I.ci) - I.wi;
  I.tir = val(I.q) < 0.0;                                           // P:111 (R5: strict)
  if (I.tir) {
    I.ct = S(0.0); I.R = S(1.0); I.T = S(0.0); I.wt = zero3<S>();
    return I;
  }
  I.ct = safe_sqrt(I.q) / I.eta;                                    // cos(theta_t)
  // P:106-108 with the parallel/perpendicular labels read as swapped (R4):
  // omega_t = -(omega_i - (omega_i.n) n)/eta - n sqrt(eta^2 - sin^2)/eta
  I.wt = scl(I.wi - scl(n, I.ci), S(-1.0) / I.eta) - scl(n, I.ct);
  // Fresnel.  Both cosines zero (grazing at eta = 1) is 0/0: take the grazing
  // limit R = 1 (R5); both children then continue straight on, so L is unchanged.
  I.degen = val(I.ci) == 0.0 && val(I.ct) == 0.0;
  if (I.degen) { I.R = S(1.0); I.T = S(0.0); return I; }
  S rs = (eta_i * I.ci - eta_t * I.ct) / (eta_i * I.ci + eta_t * I.ct);
  S rp = (eta_i * I.ct - eta_t * I.ci) / (eta_i * I.ct + eta_t * I.ci);
  I.R = S(0.5) * (rs * rs + rp * rp);
  I.T = S(1.0) - I.R;
  return I;
}

// ----------------------------------------------------------------------------- absorption
// Table entry of corner (x, y, z) of hash level l (R29): iNGP's dense index while the level's
// (N+1)^3 vertices fit in the table, else its spatial hash with primes (1, 2654435761,
// 805459861), xor-combined in 32-bit arithmetic, modulo T = 2^log2_size.
size_t hash_entry(const dto_scene* sc, int l, int x, int y, int z) {
  const uint32_t T = 1u << sc->hash_log2_size;
  const uint64_t n1 = (uint64_t)sc->hash_res[l] + 1;
  size_t e;
  if (n1 * n1 * n1 <= T) e = (size_t)(x + n1 * (y + n1 * (uint64_t)z));
  else e = (size_t)(((uint32_t)x * 1u ^ (uint32_t)y * 2654435761u ^ (uint32_t)z * 805459861u) & (T - 1));
  return (size_t)l * T + e;
}

// mu_t(p) of the hash grid: sum over levels of the trilinear interpolation of the level's
// (N_l + 1)^3 vertex values (looked up through hash_entry); zero outside the box (R11).
template <class S>
void sigma_at_hash(const Model<S>& m, V3<S> p, S out[3]) {
  const dto_scene* sc = m.sc;
  for (int c = 0; c < 3; ++c) out[c] = S(0.0);
  S u[3];
  for (int a = 0; a < 3; ++a) {
    S lo = S((double)sc->sigma_lo[a]), hi = S((double)sc->sigma_hi[a]);
    u[a] = (comp(p, a) - lo) / (hi - lo);
    if (val(u[a]) < 0.0 || val(u[a]) > 1.0) return;
  }
  for (int l = 0; l < sc->hash_levels; ++l) {
    const int N = sc->hash_res[l];
    int i0[3];
    S f[3];
    for (int a = 0; a < 3; ++a) {
      S g = u[a] * S((double)N);
      i0[a] = std::min((int)std::floor(val(g)), N - 1);
      f[a] = g - S((double)i0[a]);
    }
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          S w = (dx ? f[0] : S(1.0) - f[0]) * (dy ? f[1] : S(1.0) - f[1]) * (dz ? f[2] : S(1.0) - f[2]);
          size_t e = hash_entry(sc, l, i0[0] + dx, i0[1] + dy, i0[2] + dz);
          for (int c = 0; c < 3; ++c) out[c] = out[c] + w * m.sigma[e * 3 + c];
        }
  }
}

// mu_t(p): R^3 vertex-centred nodes over the fixed box, trilinear, zero outside (R11).
template <class S>
void sigma_at(const Model<S>& m, V3<S> p, S out[3]) {
  const dto_scene* sc = m.sc;
  if (sc->abs_kind == 2) { sigma_at_hash(m, p, out); return; }
  int R = sc->sigma_res;
  S g[3];
  int i0[3];
  for (int a = 0; a < 3; ++a) {
    S lo = S((double)sc->sigma_lo[a]), hi = S((double)sc->sigma_hi[a]);
    g[a] = (comp(p, a) - lo) / (hi - lo) * S((double)(R - 1));
    if (val(g[a]) < 0.0 || val(g[a]) > R - 1) { out[0] = out[1] = out[2] = S(0.0); return; }
    i0[a] = std::min((int)std::floor(val(g[a])), R - 2);
  }
  S f[3] = {g[0] - S((double)i0[0]), g[1] - S((double)i0[1]), g[2] - S((double)i0[2])};
  for (int c = 0; c < 3; ++c) out[c] = S(0.0);
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        S w = (dx ? f[0] : S(1.0) - f[0]) * (dy ? f[1] : S(1.0) - f[1]) * (dz ? f[2] : S(1.0) - f[2]);
        size_t node = ((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx);
        for (int c = 0; c < 3; ++c) out[c] = out[c] + w * m.sigma[node * 3 + c];
      }
}

// tau = exp(-sum_i mu_t(x_i) dx_i) over the segment o -> x: midpoint rule with
// N uniform samples (R10); constant sigma gives exp(-sigma * l) exactly.
template <class S>
V3<S> transmittance(const Model<S>& m, V3<S> o, V3<S> x) {
  S l = norm(x - o);
  S Sc[3];
  if (m.sc->abs_kind == 0) {
    for (int c = 0; c < 3; ++c) Sc[c] = m.sigma[c] * l;
  } else {
    int N = m.sc->n_samples;
    for (int c = 0; c < 3; ++c) Sc[c] = S(0.0);
    for (int j = 0; j < N; ++j) {
      S w = S((j + 0.5) / N);
      V3<S> p = o + scl(x - o, w);
      S s[3];
      sigma_at(m, p, s);
      for (int c = 0; c < 3; ++c) Sc[c] = Sc[c] + s[c];
    }
    for (int c = 0; c < 3; ++c) Sc[c] = Sc[c] * l / S((double)N);
  }
  return {exp(-Sc[0]), exp(-Sc[1]), exp(-Sc[2])};
}

// ----------------------------------------------------------------------------- environment
// Frozen env lookup for an escaping ray (P:160 step 3; R14).
template <class S>
S grid_coord(S p, double Re, int res, bool& clamped) {
  S g = (p + S(Re)) / S(2.0 * Re) * S((double)(res - 1));
  clamped = false;
  if (val(g) < 0.0) { clamped = true; return S(0.0); }
  if (val(g) > res - 1) { clamped = true; return S((double)(res - 1)); }
  return g;
}
template <class S>
V3<S> trilerp_vox(const dto_scene* sc, V3<S> p) {
  bool c;
  S g[3] = {grid_coord(p.x, sc->env_radius, sc->vres, c), grid_coord(p.y, sc->env_radius, sc->vres, c),
            grid_coord(p.z, sc->env_radius, sc->vres, c)};
  int R = sc->vres, i0[3];
  S f[3];
  for (int a = 0; a < 3; ++a) { i0[a] = std::min((int)std::floor(val(g[a])), R - 2); f[a] = g[a] - S((double)i0[a]); }
  V3<S> out = zero3<S>();
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        S w = (dx ? f[0] : S(1.0) - f[0]) * (dy ? f[1] : S(1.0) - f[1]) * (dz ? f[2] : S(1.0) - f[2]);
        const float* t = sc->voxel + (((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx)) * 4;
        out = out + scl(mk<S>(S((double)t[0]), S((double)t[1]), S((double)t[2])), w);
      }
  return out;
}
template <class S>
V3<S> bilerp_plane(const dto_scene* sc, int k, S a, S b) {  // a = column coord, b = row coord
  bool c;
  int R = sc->pres;
  S ga = grid_coord(a, sc->env_radius, R, c), gb = grid_coord(b, sc->env_radius, R, c);
  int ia = std::min((int)std::floor(val(ga)), R - 2), ib = std::min((int)std::floor(val(gb)), R - 2);
  S fa = ga - S((double)ia), fb = gb - S((double)ib);
  V3<S> out = zero3<S>();
  for (int db = 0; db < 2; ++db)
    for (int da = 0; da < 2; ++da) {
      S w = (da ? fa : S(1.0) - fa) * (db ? fb : S(1.0) - fb);
      const float* t = sc->planes + (((size_t)k * R + (ib + db)) * R + (ia + da)) * 4;
      out = out + scl(mk<S>(S((double)t[0]), S((double)t[1]), S((double)t[2])), w);
    }
  return out;
}
// Density channel (w) of the same textures (R30).
template <class S>
S trilerp_vox_w(const dto_scene* sc, V3<S> p) {
  bool c;
  S g[3] = {grid_coord(p.x, sc->env_radius, sc->vres, c), grid_coord(p.y, sc->env_radius, sc->vres, c),
            grid_coord(p.z, sc->env_radius, sc->vres, c)};
  int R = sc->vres, i0[3];
  S f[3];
  for (int a = 0; a < 3; ++a) { i0[a] = std::min((int)std::floor(val(g[a])), R - 2); f[a] = g[a] - S((double)i0[a]); }
  S out = S(0.0);
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        S w = (dx ? f[0] : S(1.0) - f[0]) * (dy ? f[1] : S(1.0) - f[1]) * (dz ? f[2] : S(1.0) - f[2]);
        out = out + w * S((double)sc->voxel[(((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx)) * 4 + 3]);
      }
  return out;
}
template <class S>
S bilerp_plane_w(const dto_scene* sc, int k, S a, S b) {
  bool c;
  int R = sc->pres;
  S ga = grid_coord(a, sc->env_radius, R, c), gb = grid_coord(b, sc->env_radius, R, c);
  int ia = std::min((int)std::floor(val(ga)), R - 2), ib = std::min((int)std::floor(val(gb)), R - 2);
  S fa = ga - S((double)ia), fb = gb - S((double)ib);
  S out = S(0.0);
  for (int db = 0; db < 2; ++db)
    for (int da = 0; da < 2; ++da)
      out = out + (da ? fa : S(1.0) - fa) * (db ? fb : S(1.0) - fb) *
                      S((double)sc->planes[(((size_t)k * R + (ib + db)) * R + (ia + da)) * 4 + 3]);
  return out;
}
// Env field at p: colour = trilinear voxel + three bilinear planes (rgb), density = the same
// sum over the w channel, clamped at 0 (R30).
template <class S>
V3<S> env_colour(const dto_scene* sc, V3<S> p) {
  return trilerp_vox(sc, p) + bilerp_plane(sc, 0, p.x, p.y) + bilerp_plane(sc, 1, p.x, p.z) +
         bilerp_plane(sc, 2, p.y, p.z);
}
template <class S>
S env_density(const dto_scene* sc, V3<S> p) {
  S s = trilerp_vox_w(sc, p) + bilerp_plane_w(sc, 0, p.x, p.y) + bilerp_plane_w(sc, 1, p.x, p.z) +
        bilerp_plane_w(sc, 2, p.y, p.z);
  return val(s) > 0.0 ? s : S(0.0);
}

// Volume rendering of the env field along an exterior segment o -> x (R30; NeRF-style
// quadrature with M midpoint samples t_i = (i + 1/2)/M, Delta = |x - o|/M):
//   V = sum_i T_i (1 - exp(-sigma_i Delta)) c_i,  T_i = exp(-Delta sum_{j<i} sigma_j),
//   Tn = T_M (transmittance of the whole segment, scalar).
template <class S>
void env_volume(const dto_scene* sc, V3<S> o, V3<S> x, V3<S>& Vr, S& Tn) {
  const int M = sc->env_samples;
  S delta = norm(x - o) / S((double)M);
  S od = S(0.0);
  Vr = zero3<S>();
  for (int i = 0; i < M; ++i) {
    V3<S> p = o + scl(x - o, S((i + 0.5) / M));
    S sg = env_density(sc, p);
    S Ti = exp(-od);
    S ai = S(1.0) - exp(-sg * delta);
    Vr = Vr + scl(env_colour(sc, p), Ti * ai);
    od = od + sg * delta;
  }
  Tn = exp(-od);
}

template <class S>
V3<S> shell_point(const dto_scene* sc, V3<S> o, V3<S> dh) {
  if (sc->far_field) return scl(dh, S((double)sc->env_radius));
  S b = dot(o, dh);
  S Re = S((double)sc->env_radius);
  S ts = -b + safe_sqrt(b * b - dot(o, o) + Re * Re);   // ||o + ts dh|| = R_e
  return o + scl(dh, ts);
}
template <class S>
V3<S> env(const dto_scene* sc, V3<S> o, V3<S> d) {
  V3<S> dh = scl(d, S(1.0) / norm(d));
  if (sc->env_kind == 0) {
    V3<S> L = {S((double)sc->ambient[0]), S((double)sc->ambient[1]), S((double)sc->ambient[2])};
    for (int j = 0; j < sc->n_lobes; ++j) {
      const float* lb = sc->lobes + 7 * j;
      V3<S> mu = {S((double)lb[0]), S((double)lb[1]), S((double)lb[2])};
      S e = exp(S((double)lb[3]) * (dot(mu, dh) - S(1.0)));
      L = L + scl(mk<S>(S((double)lb[4]), S((double)lb[5]), S((double)lb[6])), e);
    }
    return L;
  }
  V3<S> p = shell_point(sc, o, dh);
  DTO_STUDY(p, 32);
  return trilerp_vox(sc, p) + bilerp_plane(sc, 0, p.x, p.y) + bilerp_plane(sc, 1, p.x, p.z) +
         bilerp_plane(sc, 2, p.y, p.z);
}

// ----------------------------------------------------------------------------- forward
struct RayStats { uint64_t sig_topo = 0, sig_face = 0; double capped_w = 0; int flags = 0; int64_t segments = 0; };

// Shading normal n(x) = normalize(sum beta_i n_{v_i}) (R7: fallback to the
// geometric unit normal if the blend vanishes).
template <class S>
V3<S> shading_normal(const Model<S>& m, int f, S u, S v, bool& fallback) {
  const int32_t* F = m.sc->F + 3 * f;
  S b0 = S(1.0) - u - v;
  V3<S> mm = scl(m.nrm[F[0]], b0) + scl(m.nrm[F[1]], u) + scl(m.nrm[F[2]], v);
  S L = norm(mm);
  fallback = !(val(L) >= 1e-12);
  if (!fallback) return scl(mm, S(1.0) / L);
  V3<S> c = cross(m.V[F[1]] - m.V[F[0]], m.V[F[2]] - m.V[F[0]]);
  return scl(c, S(1.0) / norm(c));
}

// Trace(o, d, k) — P:157-163, steps 1-5, depth-first.  pos = heap index of the node in
// the binary ray tree (root 1, reflect child 2p, refract child 2p+1); w = scalar product
// of the R/T weights on the way down (only for the capped-weight statistic).
template <class S>
V3<S> trace(const Model<S>& m, V3<S> o, V3<S> d, int k, uint64_t pos, double w, RayStats& st) {
  const dto_scene* sc = m.sc;
  double t_lo = k == 0 ? 0.0 : m.t_min;
  Hit h = closest_hit(m, vald(o), vald(d), t_lo);                  // step 2
  st.segments++;
  st.flags |= h.flags;
  if (h.face < 0) {                                                 // step 3: miss -> env
    st.sig_topo += mix64(topo_key(pos, EV_MISS));
    st.sig_face += mix64(face_key(pos, EV_MISS, -1));
    if (sc->env_kind == 2) {                                        // volume out to the shell (R30)
      V3<S> ps = shell_point(sc, o, scl(d, S(1.0) / norm(d)));
      V3<S> Vr;
      S Tn;
      env_volume(sc, o, ps, Vr, Tn);
      return Vr + scl(env(sc, o, d), Tn);
    }
    return env(sc, o, d);
  }
  const int32_t* F = sc->F + 3 * h.face;
  MT<S> r = moller_trumbore(o, d, m.V[F[0]], m.V[F[1]], m.V[F[2]]);  // differentiable (R15)
  DTO_STUDY(r.u, 64);
  DTO_STUDY(r.v, 64);
  V3<S> x = o + scl(d, r.t);
  DTO_STUDY(x, 2);
  V3d gn = cross(m.Vd[F[1]] - m.Vd[F[0]], m.Vd[F[2]] - m.Vd[F[0]]);
  bool inside = dot(vald(d), gn) > 0.0;                             // R8
  if (k == sc->max_depth) {                                         // step 1 (R12, R13)
    if (sc->cap_policy == 0 && sc->env_kind != 2) {                 // discarded branch (R13, R34)
      st.sig_topo += mix64(topo_key(pos, EV_CAP_DROP));
      st.sig_face += mix64(face_key(pos, EV_CAP_DROP, -1));
      st.capped_w += w;
      return zero3<S>();
    }
    int ev = inside ? EV_CAP_IN : EV_CAP_OUT;
    st.sig_topo += mix64(topo_key(pos, ev));
    st.sig_face += mix64(face_key(pos, ev, h.face));
    st.capped_w += w;
    if (!inside && sc->env_kind == 2) {                             // exterior: its volume part stays
      V3<S> Vr;
      S Tn;
      env_volume(sc, o, x, Vr, Tn);
      return sc->cap_policy == 0 ? Vr : Vr + scl(env(sc, o, d), Tn);
    }
    if (sc->cap_policy == 0) return zero3<S>();
    V3<S> E = env(sc, o, d);
    return inside ? mul(transmittance(m, o, x), E) : E;
  }
  bool fb;
  V3<S> ns = shading_normal(m, h.face, r.u, r.v, fb);
  DTO_STUDY(ns, 16);
  V3<S> n = inside ? -ns : ns;
  S eta_i = inside ? m.ior : S(1.0), eta_t = inside ? S(1.0) : m.ior;
  Iface<S> I = interface(d, n, eta_i, eta_t);
  if (val(I.c_raw) < 1e-3) st.flags |= DTO_FLAG_GRAZING;
  if (std::fabs(val(I.q)) < 1e-4) st.flags |= DTO_FLAG_NEARTIR;   // dR/dc_i ~ 1/sqrt(q)
  DTO_STUDY(I.wr, 4);
  DTO_STUDY(I.wt, 4);
  int ev = inside ? (I.tir ? EV_HIT_IN_TIR : EV_HIT_IN) : (I.tir ? EV_HIT_OUT_TIR : EV_HIT_OUT);
  st.sig_topo += mix64(topo_key(pos, ev));
  st.sig_face += mix64(face_key(pos, ev, h.face));
  // steps 4/5: reflect and refract children from x, blended by R and T
  V3<S> Lr = trace(m, x, I.wr, k + 1, 2 * pos, w * val(I.R), st);
  V3<S> L = scl(Lr, I.R);
  if (!I.tir) {
    V3<S> Lt = trace(m, x, I.wt, k + 1, 2 * pos + 1, w * val(I.T), st);
    L = L + scl(Lt, I.T);
  }
  if (inside) L = mul(transmittance(m, o, x), L);                  // step 5, P:162 (R9)
  if (!inside && sc->env_kind == 2) {                               // env mixed in before x (R30)
    V3<S> Vr;
    S Tn;
    env_volume(sc, o, x, Vr, Tn);
    L = Vr + scl(L, Tn);
  }
  return L;
}

// ----------------------------------------------------------------------------- reverse mode
struct Grad {
  std::vector<V3d> gV, gN;   // d/dV (direct) and d/dn_v (folded into gV at the end)
  double gior = 0.0;
  std::vector<double> gsig;
};
struct Bwd { V3d L, go, gd; };

// d value / d p of the vertex-centred sigma grid, accumulating the node adjoints.
// Returns gp = sum_c gS_c * scale * grad sigma_c(p); adds gS_c * scale * w to node c.
V3d sigma_bwd_hash(const Model<double>& m, V3d p, const double gSs[3], Grad& G, double Sv[3]) {
  const dto_scene* sc = m.sc;
  Sv[0] = Sv[1] = Sv[2] = 0.0;
  double u[3], inv[3];
  for (int a = 0; a < 3; ++a) {
    double lo = sc->sigma_lo[a], hi = sc->sigma_hi[a];
    u[a] = (comp(p, a) - lo) / (hi - lo);
    if (u[a] < 0.0 || u[a] > 1.0) return {0, 0, 0};
    inv[a] = 1.0 / (hi - lo);
  }
  V3d gp = {0, 0, 0};
  for (int l = 0; l < sc->hash_levels; ++l) {
    const int N = sc->hash_res[l];
    int i0[3];
    double f[3];
    for (int a = 0; a < 3; ++a) {
      double g = u[a] * N;
      i0[a] = std::min((int)std::floor(g), N - 1);
      f[a] = g - i0[a];
    }
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          double wx = dx ? f[0] : 1 - f[0], wy = dy ? f[1] : 1 - f[1], wz = dz ? f[2] : 1 - f[2];
          double w = wx * wy * wz;
          double sx = dx ? 1.0 : -1.0, sy = dy ? 1.0 : -1.0, sz = dz ? 1.0 : -1.0;
          size_t e = hash_entry(sc, l, i0[0] + dx, i0[1] + dy, i0[2] + dz);
          for (int c = 0; c < 3; ++c) {
            double s = m.sigma[e * 3 + c];
            Sv[c] += w * s;
            G.gsig[e * 3 + c] += gSs[c] * w;
            gp.x += gSs[c] * s * sx * wy * wz * N * inv[0];
            gp.y += gSs[c] * s * wx * sy * wz * N * inv[1];
            gp.z += gSs[c] * s * wx * wy * sz * N * inv[2];
          }
        }
  }
  return gp;
}

V3d sigma_bwd(const Model<double>& m, V3d p, const double gSs[3], Grad& G, double Sv[3]) {
  const dto_scene* sc = m.sc;
  if (sc->abs_kind == 2) return sigma_bwd_hash(m, p, gSs, G, Sv);
  int R = sc->sigma_res;
  double g[3], f[3], inv[3];
  int i0[3];
  Sv[0] = Sv[1] = Sv[2] = 0.0;
  for (int a = 0; a < 3; ++a) {
    double lo = sc->sigma_lo[a], hi = sc->sigma_hi[a];
    g[a] = (comp(p, a) - lo) / (hi - lo) * (R - 1);
    if (g[a] < 0.0 || g[a] > R - 1) return {0, 0, 0};
    i0[a] = std::min((int)std::floor(g[a]), R - 2);
    f[a] = g[a] - i0[a];
    inv[a] = (R - 1) / (hi - lo);
  }
  V3d gp = {0, 0, 0};
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        double wx = dx ? f[0] : 1 - f[0], wy = dy ? f[1] : 1 - f[1], wz = dz ? f[2] : 1 - f[2];
        double w = wx * wy * wz;
        double sx = dx ? 1.0 : -1.0, sy = dy ? 1.0 : -1.0, sz = dz ? 1.0 : -1.0;
        size_t node = ((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx);
        for (int c = 0; c < 3; ++c) {
          double s = m.sigma[node * 3 + c];
          Sv[c] += w * s;
          G.gsig[node * 3 + c] += gSs[c] * w;
          gp.x += gSs[c] * s * sx * wy * wz * inv[0];
          gp.y += gSs[c] * s * wx * sy * wz * inv[1];
          gp.z += gSs[c] * s * wx * wy * sz * inv[2];
        }
      }
  return gp;
}

// Reverse of transmittance(o, x) given gS = dLoss/dS_c (S_c = optical depth).
void transmittance_bwd(const Model<double>& m, V3d o, V3d x, const double gS[3], V3d& gx, V3d& go, Grad& G) {
  V3d dx = x - o;
  double l = norm(dx);
  double gl = 0.0;
  if (m.sc->abs_kind == 0) {
    for (int c = 0; c < 3; ++c) { G.gsig[c] += gS[c] * l; gl += gS[c] * m.sigma[c]; }
  } else {
    int N = m.sc->n_samples;
    double scale = l / N;
    double gSs[3] = {gS[0] * scale, gS[1] * scale, gS[2] * scale};
    for (int j = 0; j < N; ++j) {
      double w = (j + 0.5) / N;
      V3d p = o + scl(dx, w);
      double Sv[3];
      V3d gp = sigma_bwd(m, p, gSs, G, Sv);
      for (int c = 0; c < 3; ++c) gl += gS[c] * Sv[c] / N;
      go = go + scl(gp, 1.0 - w);
      gx = gx + scl(gp, w);
    }
  }
  if (l > 0.0) {
    V3d u = scl(dx, 1.0 / l);
    gx = gx + scl(u, gl);
    go = go - scl(u, gl);
  }
}

// d/dp of one clamped grid coordinate's trilinear / bilinear lookup.
V3d trilerp_vox_bwd(const dto_scene* sc, V3d p, V3d a, double aw = 0.0) {
  bool c[3];
  double g[3] = {grid_coord(p.x, sc->env_radius, sc->vres, c[0]), grid_coord(p.y, sc->env_radius, sc->vres, c[1]),
                 grid_coord(p.z, sc->env_radius, sc->vres, c[2])};
  int R = sc->vres, i0[3];
  double f[3], sc_ = (R - 1) / (2.0 * sc->env_radius);
  for (int k = 0; k < 3; ++k) { i0[k] = std::min((int)std::floor(g[k]), R - 2); f[k] = g[k] - i0[k]; }
  V3d gp = {0, 0, 0};
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        double wx = dx ? f[0] : 1 - f[0], wy = dy ? f[1] : 1 - f[1], wz = dz ? f[2] : 1 - f[2];
        const float* t = sc->voxel + (((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx)) * 4;
        double s = a.x * t[0] + a.y * t[1] + a.z * t[2] + aw * t[3];
        gp.x += s * (dx ? 1 : -1) * wy * wz;
        gp.y += s * wx * (dy ? 1 : -1) * wz;
        gp.z += s * wx * wy * (dz ? 1 : -1);
      }
  gp = scl(gp, sc_);
  if (c[0]) gp.x = 0;
  if (c[1]) gp.y = 0;
  if (c[2]) gp.z = 0;
  return gp;
}
void bilerp_plane_bwd(const dto_scene* sc, int k, double a, double b, V3d adj, double& ga_out, double& gb_out,
                      double aw = 0.0) {
  bool ca, cb;
  int R = sc->pres;
  double ga = grid_coord(a, sc->env_radius, R, ca), gb = grid_coord(b, sc->env_radius, R, cb);
  int ia = std::min((int)std::floor(ga), R - 2), ib = std::min((int)std::floor(gb), R - 2);
  double fa = ga - ia, fb = gb - ib, s_ = (R - 1) / (2.0 * sc->env_radius);
  double da_ = 0, db_ = 0;
  for (int db = 0; db < 2; ++db)
    for (int da = 0; da < 2; ++da) {
      const float* t = sc->planes + (((size_t)k * R + (ib + db)) * R + (ia + da)) * 4;
      double s = adj.x * t[0] + adj.y * t[1] + adj.z * t[2] + aw * t[3];
      da_ += s * (da ? 1 : -1) * (db ? fb : 1 - fb);
      db_ += s * (da ? fa : 1 - fa) * (db ? 1 : -1);
    }
  ga_out = ca ? 0.0 : da_ * s_;
  gb_out = cb ? 0.0 : db_ * s_;
}

// Reverse of env(o, d) given the RGB adjoint a: returns (go, gd).
// Reverse of the shell point p = o + ts dh (||p|| = R_e) or p = R_e dh (far field): adds the
// adjoints of o and dh for gp = dL/dp.
void shell_point_bwd(const dto_scene* sc, V3d o, V3d dh, V3d gp, V3d& go, V3d& gdh) {
  if (sc->far_field) {
    gdh = gdh + scl(gp, (double)sc->env_radius);
    return;
  }
  double b = dot(o, dh), Re = sc->env_radius;
  double sq = std::sqrt(b * b - dot(o, o) + Re * Re);
  double ts = -b + sq;
  // p = o + ts dh
  go = go + gp;
  gdh = gdh + scl(gp, ts);
  double gts = dot(gp, dh);
  // ts = -b + sqrt(disc), disc = b^2 - o.o + Re^2
  double gdisc = gts / (2.0 * sq);
  double gb = -gts + gdisc * 2.0 * b;
  go = go - scl(o, 2.0 * gdisc);
  // b = o . dh
  go = go + scl(dh, gb);
  gdh = gdh + scl(o, gb);
}

void env_bwd(const dto_scene* sc, V3d o, V3d d, V3d a, V3d& go, V3d& gd) {
  double dn = norm(d);
  V3d dh = scl(d, 1.0 / dn);
  V3d gdh = {0, 0, 0};
  go = {0, 0, 0};
  if (sc->env_kind == 0) {
    for (int j = 0; j < sc->n_lobes; ++j) {
      const float* lb = sc->lobes + 7 * j;
      V3d mu = {lb[0], lb[1], lb[2]};
      double e = std::exp(lb[3] * (dot(mu, dh) - 1.0));
      double s = a.x * lb[4] + a.y * lb[5] + a.z * lb[6];
      gdh = gdh + scl(mu, s * e * lb[3]);
    }
  } else {
    V3d p = shell_point<double>(sc, o, dh);
    V3d gp = trilerp_vox_bwd(sc, p, a);
    double g1, g2;
    bilerp_plane_bwd(sc, 0, p.x, p.y, a, g1, g2); gp.x += g1; gp.y += g2;
    bilerp_plane_bwd(sc, 1, p.x, p.z, a, g1, g2); gp.x += g1; gp.z += g2;
    bilerp_plane_bwd(sc, 2, p.y, p.z, a, g1, g2); gp.y += g1; gp.z += g2;
    shell_point_bwd(sc, o, dh, gp, go, gdh);
  }
  gd = scl(gdh - scl(dh, dot(dh, gdh)), 1.0 / dn);   // through dh = d/|d|
}

// d a . (colour(p)) + aw * density(p) / dp of the volumetric env field (R30); the density
// clamp at 0 passes no gradient (aw must be 0 there).
V3d env_field_bwd(const dto_scene* sc, V3d p, V3d a, double aw) {
  V3d gp = trilerp_vox_bwd(sc, p, a, aw);
  double g1, g2;
  bilerp_plane_bwd(sc, 0, p.x, p.y, a, g1, g2, aw); gp.x += g1; gp.y += g2;
  bilerp_plane_bwd(sc, 1, p.x, p.z, a, g1, g2, aw); gp.x += g1; gp.z += g2;
  bilerp_plane_bwd(sc, 2, p.y, p.z, a, g1, g2, aw); gp.y += g1; gp.z += g2;
  return gp;
}

// Reverse of env_volume(o, x) given aV = dL/dV (rgb) and aT = dL/dTn: adds the adjoints of
// the segment end points to go, gx.  With T_0 = 1 and V = sum_i (T_i - T_{i+1}) c_i:
// dL/dT_i = s_i - s_{i-1} (0 < i < M), dL/dT_M = aT - s_{M-1}, s_i = aV . c_i;
// dL/dsigma_j = -Delta sum_{i>j} dL/dT_i T_i;  dL/dDelta = -sum_i dL/dT_i T_i sum_{j<i} sigma_j.
void env_volume_bwd(const dto_scene* sc, V3d o, V3d x, V3d aV, double aT, V3d& go, V3d& gx) {
  const int M = sc->env_samples;
  V3d dx = x - o;
  double l = norm(dx), delta = l / M;
  std::vector<double> sg(M), raw(M), pre(M + 1, 0.0), T(M + 1, 1.0), s(M), gT(M + 1, 0.0);
  for (int i = 0; i < M; ++i) {
    V3d p = o + scl(dx, (i + 0.5) / M);
    raw[i] = trilerp_vox_w<double>(sc, p) + bilerp_plane_w<double>(sc, 0, p.x, p.y) +
             bilerp_plane_w<double>(sc, 1, p.x, p.z) + bilerp_plane_w<double>(sc, 2, p.y, p.z);
    sg[i] = raw[i] > 0.0 ? raw[i] : 0.0;
    s[i] = dot(aV, env_colour<double>(sc, p));
    pre[i + 1] = pre[i] + sg[i];
    T[i + 1] = std::exp(-delta * pre[i + 1]);
  }
  for (int i = 1; i < M; ++i) gT[i] = s[i] - s[i - 1];
  gT[M] = aT - s[M - 1];
  double acc = 0.0, gdelta = 0.0;
  std::vector<double> gsg(M);
  for (int i = M; i >= 1; --i) {
    acc += gT[i] * T[i];
    gsg[i - 1] = -delta * acc;
    gdelta -= gT[i] * T[i] * pre[i];
  }
  for (int i = 0; i < M; ++i) {
    double t = (i + 0.5) / M;
    V3d p = o + scl(dx, t);
    V3d gp = env_field_bwd(sc, p, scl(aV, T[i] - T[i + 1]), raw[i] > 0.0 ? gsg[i] : 0.0);
    go = go + scl(gp, 1.0 - t);
    gx = gx + scl(gp, t);
  }
  if (l > 0.0) {
    V3d u = scl(dx, 1.0 / l);
    double gl = gdelta / M;
    gx = gx + scl(u, gl);
    go = go - scl(u, gl);
  }
}

// Reverse of the Moller-Trumbore solve M [u v t]^T = o - v0, M = [e1 e2 -d] (R15): with
// lambda = M^-T (gu, gv, gt): go += lambda, gd += t lambda, gV_k -= beta_k lambda.
void mt_bwd(const Model<double>& m, int face, V3d d, double t, double u, double v, double gu, double gv, double gt,
            V3d& go, V3d& gd, Grad& G) {
  const int32_t* F = m.sc->F + 3 * face;
  V3d v0 = m.Vd[F[0]], e1 = m.Vd[F[1]] - v0, e2 = m.Vd[F[2]] - v0;
  double det = dot(e1, cross(d, e2));
  V3d lam = scl(scl(cross(d, e2), gu) + scl(cross(e1, d), gv) + scl(cross(e1, e2), gt), 1.0 / det);
  go = go + lam;
  gd = gd + scl(lam, t);
  G.gV[F[0]] = G.gV[F[0]] - scl(lam, 1.0 - u - v);
  G.gV[F[1]] = G.gV[F[1]] - scl(lam, u);
  G.gV[F[2]] = G.gV[F[2]] - scl(lam, v);
}

// Post-order reverse of trace(): returns the node radiance L and the adjoints of the
// node's own ray origin / direction; accumulates parameter adjoints into G.
// a = dLoss/dL(node) (RGB).
Bwd trace_bwd(const Model<double>& m, V3d o, V3d d, int k, V3d a, Grad& G) {
  const dto_scene* sc = m.sc;
  double t_lo = k == 0 ? 0.0 : m.t_min;
  Hit h = closest_hit(m, o, d, t_lo);
  Bwd out{{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  if (h.face < 0) {                                                 // leaf: env (R22: env frozen)
    if (sc->env_kind == 2) {                                        // volume out to the shell (R30)
      V3d dh = scl(d, 1.0 / norm(d));
      V3d ps = shell_point<double>(sc, o, dh);
      V3d Vr, E = env<double>(sc, o, d);
      double Tn;
      env_volume(sc, o, ps, Vr, Tn);
      out.L = Vr + scl(E, Tn);
      env_bwd(sc, o, d, scl(a, Tn), out.go, out.gd);
      V3d gov = {0, 0, 0}, gps = {0, 0, 0}, gdh = {0, 0, 0};
      env_volume_bwd(sc, o, ps, a, dot(a, E), gov, gps);
      shell_point_bwd(sc, o, dh, gps, gov, gdh);
      out.go = out.go + gov;
      out.gd = out.gd + scl(gdh - scl(dh, dot(dh, gdh)), 1.0 / norm(d));
      return out;
    }
    out.L = env<double>(sc, o, d);
    env_bwd(sc, o, d, a, out.go, out.gd);
    return out;
  }
  const int32_t* F = sc->F + 3 * h.face;
  MT<double> r = moller_trumbore<double>(o, d, m.Vd[F[0]], m.Vd[F[1]], m.Vd[F[2]]);
  V3d x = o + scl(d, r.t);
  V3d gnrm = cross(m.Vd[F[1]] - m.Vd[F[0]], m.Vd[F[2]] - m.Vd[F[0]]);
  bool inside = dot(d, gnrm) > 0.0;
  V3d gx = {0, 0, 0};
  double gu = 0, gv = 0;
  if (k == sc->max_depth && !inside && sc->env_kind == 2) {         // capped exterior, volume env
    V3d Vr;
    double Tn;
    env_volume(sc, o, x, Vr, Tn);
    double aT = 0.0;
    out.L = Vr;
    if (sc->cap_policy == 1) {
      V3d E = env<double>(sc, o, d);
      out.L = out.L + scl(E, Tn);
      env_bwd(sc, o, d, scl(a, Tn), out.go, out.gd);
      aT = dot(a, E);
    }
    env_volume_bwd(sc, o, x, a, aT, out.go, gx);
  } else if (k == sc->max_depth) {                                  // capped leaf (R13)
    if (sc->cap_policy == 0) return out;
    V3d E = env<double>(sc, o, d);
    if (!inside) { out.L = E; env_bwd(sc, o, d, a, out.go, out.gd); return out; }
    V3d tau = transmittance(m, o, x);
    out.L = mul(tau, E);
    env_bwd(sc, o, d, mul(a, tau), out.go, out.gd);
    double gS[3] = {-a.x * E.x * tau.x, -a.y * E.y * tau.y, -a.z * E.z * tau.z};
    transmittance_bwd(m, o, x, gS, gx, out.go, G);
  } else {
    // ---- local forward (same steps as trace())
    bool fb;
    V3d ns = shading_normal(m, h.face, r.u, r.v, fb);
    double sg = inside ? -1.0 : 1.0;
    V3d n = scl(ns, sg);
    double eta_i = inside ? m.ior : 1.0, eta_t = inside ? 1.0 : m.ior;
    Iface<double> I = interface(d, n, eta_i, eta_t);
    V3d tau = inside ? transmittance(m, o, x) : V3d{1, 1, 1};
    const bool vol = !inside && sc->env_kind == 2;                  // exterior: env mixed in (R30)
    V3d Vr = {0, 0, 0};
    if (vol) {
      double Tn;
      env_volume(sc, o, x, Vr, Tn);
      tau = {Tn, Tn, Tn};
    }
    V3d ap = mul(a, tau);
    // ---- children (their adjoints carry R and T)
    Bwd cr = trace_bwd(m, x, I.wr, k + 1, scl(ap, I.R), G);
    Bwd ct = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (!I.tir) ct = trace_bwd(m, x, I.wt, k + 1, scl(ap, I.T), G);
    V3d Lc = scl(cr.L, I.R) + scl(ct.L, I.T);
    out.L = Vr + mul(tau, Lc);
    // ---- reverse, last operation first
    gx = cr.go + ct.go;
    V3d gwr = cr.gd, gwt = ct.gd;
    if (vol) env_volume_bwd(sc, o, x, a, dot(a, Lc), out.go, gx);
    if (inside) {
      double gS[3] = {-a.x * Lc.x * tau.x, -a.y * Lc.y * tau.y, -a.z * Lc.z * tau.z};
      transmittance_bwd(m, o, x, gS, gx, out.go, G);
    }
    double gci = 0, geta = 0, geta_i = 0, geta_t = 0;
    V3d gn = {0, 0, 0}, gwi = {0, 0, 0};
    if (!I.tir && !I.degen) {
      double gR = dot(ap, cr.L - ct.L);                             // T = 1 - R folded in
      double A = eta_i * I.ci, B = eta_t * I.ct, C = eta_i * I.ct, D = eta_t * I.ci;
      double rs = (A - B) / (A + B), rp = (C - D) / (C + D);
      double grs = gR * rs, grp = gR * rp;                          // R = (rs^2 + rp^2)/2
      double gA = grs * 2.0 * B / ((A + B) * (A + B)), gB = -grs * 2.0 * A / ((A + B) * (A + B));
      double gC = grp * 2.0 * D / ((C + D) * (C + D)), gD = -grp * 2.0 * C / ((C + D) * (C + D));
      double gct = gB * eta_t + gC * eta_i;
      gci += gA * eta_i + gD * eta_t;
      geta_i += gA * I.ci + gC * I.ct;
      geta_t += gB * I.ct + gD * I.ci;
      // wt = -(wi - ci n)/eta - ct n
      gwi = gwi - scl(gwt, 1.0 / I.eta);
      gci += dot(gwt, n) / I.eta;
      gn = gn + scl(gwt, I.ci / I.eta) - scl(gwt, I.ct);
      geta += dot(gwt, I.wi - scl(n, I.ci)) / (I.eta * I.eta);
      gct += -dot(gwt, n);
      // ct = sqrt(q)/eta
      double sq = std::sqrt(I.q);
      double gq = sq > 0.0 ? gct / (2.0 * I.eta * sq) : 0.0;
      geta += -gct * sq / (I.eta * I.eta);
      // q = eta^2 - 1 + ci^2
      geta += gq * 2.0 * I.eta;
      gci += gq * 2.0 * I.ci;
    }
    // wr = 2 ci n - wi
    gci += 2.0 * dot(gwr, n);
    gn = gn + scl(gwr, 2.0 * I.ci);
    gwi = gwi - gwr;
    // eta = eta_t / eta_i
    geta_t += geta / eta_i;
    geta_i += -geta * eta_t / (eta_i * eta_i);
    if (inside) G.gior += geta_i; else G.gior += geta_t;
    // ci = clamp(wi . n)
    if (!I.clamped) { gwi = gwi + scl(n, gci); gn = gn + scl(I.wi, gci); }
    out.gd = out.gd - gwi;                                          // wi = -d
    // n = sg * ns, ns = m / |m|, m = sum beta_k n_vk
    if (!fb) {
      V3d gns = scl(gn, sg);
      V3d nv[3] = {m.nrm[F[0]], m.nrm[F[1]], m.nrm[F[2]]};
      double beta[3] = {1.0 - r.u - r.v, r.u, r.v};
      V3d mm = scl(nv[0], beta[0]) + scl(nv[1], beta[1]) + scl(nv[2], beta[2]);
      double Lm = norm(mm);
      V3d gm = scl(gns - scl(ns, dot(ns, gns)), 1.0 / Lm);
      double gb[3];
      for (int q = 0; q < 3; ++q) {
        G.gN[F[q]] = G.gN[F[q]] + scl(gm, beta[q]);
        gb[q] = dot(gm, nv[q]);
      }
      gu = gb[1] - gb[0];
      gv = gb[2] - gb[0];
    }
  }
  // x = o + t d
  out.go = out.go + gx;
  out.gd = out.gd + scl(gx, r.t);
  double gt = dot(gx, d);
  mt_bwd(m, h.face, d, r.t, r.u, r.v, gu, gv, gt, out.go, out.gd, G);
  return out;
}

// Reverse of vertex_normals(): gN (d/dn_v) -> gV through n_v = s_v/|s_v|,
// s_v = sum h_f, h_f = c_f/|c_f|, c_f = e1 x e2.
void vertex_normals_bwd(const Model<double>& m, Grad& G) {
  const int32_t* F = m.sc->F;
  std::vector<V3d> s(m.nv, V3d{0, 0, 0});
  std::vector<V3d> h(m.nf);
  std::vector<double> Lf(m.nf);
  for (int f = 0; f < m.nf; ++f) {
    V3d v0 = m.Vd[F[3 * f]], v1 = m.Vd[F[3 * f + 1]], v2 = m.Vd[F[3 * f + 2]];
    V3d c = cross(v1 - v0, v2 - v0);
    Lf[f] = norm(c);
    h[f] = Lf[f] > 0.0 ? scl(c, 1.0 / Lf[f]) : V3d{0, 0, 0};
    for (int k = 0; k < 3; ++k) s[F[3 * f + k]] = s[F[3 * f + k]] + h[f];
  }
  std::vector<V3d> gs(m.nv, V3d{0, 0, 0});
  for (int v = 0; v < m.nv; ++v) {
    double L = norm(s[v]);
    if (!(L > 0.0)) continue;
    V3d n = scl(s[v], 1.0 / L);
    gs[v] = scl(G.gN[v] - scl(n, dot(n, G.gN[v])), 1.0 / L);
  }
  for (int f = 0; f < m.nf; ++f) {
    if (!(Lf[f] > 0.0)) continue;
    V3d gh = gs[F[3 * f]] + gs[F[3 * f + 1]] + gs[F[3 * f + 2]];
    V3d gc = scl(gh - scl(h[f], dot(h[f], gh)), 1.0 / Lf[f]);
    V3d v0 = m.Vd[F[3 * f]], e1 = m.Vd[F[3 * f + 1]] - v0, e2 = m.Vd[F[3 * f + 2]] - v0;
    V3d ge1 = cross(e2, gc), ge2 = cross(gc, e1);
    G.gV[F[3 * f + 1]] = G.gV[F[3 * f + 1]] + ge1;
    G.gV[F[3 * f + 2]] = G.gV[F[3 * f + 2]] + ge2;
    G.gV[F[3 * f]] = G.gV[F[3 * f]] - ge1 - ge2;
  }
}

// ----------------------------------------------------------------------------- driver
void get_ray(const dto_scene* sc, const int64_t* pid, const double* rays, int64_t i, V3d& o, V3d& d) {
  if (rays) {
    o = {rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]};
    d = {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
  } else {
    camera_ray(sc, pid ? pid[i] : i, o, d);
  }
  DTO_STUDY(o, 1);
  DTO_STUDY(d, 1);
}

template <class Fn>
void parallel_for(int64_t n, int nthreads, Fn fn) {
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  nthreads = (int)std::min<int64_t>(nthreads, std::max<int64_t>(n, 1));
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) {
    int64_t i0 = n * t / nthreads, i1 = n * (t + 1) / nthreads;
    th.emplace_back([=] { fn(t, i0, i1); });
  }
  for (auto& x : th) x.join();
}

int check_scene(const dto_scene* s) {
  if (!s || s->nf <= 0 || s->nv <= 0 || !s->V || !s->F) return 1;
  return 0;
}

}  // namespace

extern "C" {

int dto_render(const dto_scene* s, const int64_t* pixel_ids, const double* rays, int64_t n, double* rgb,
               double* capped_w, uint64_t* sig_topo, uint64_t* sig_face, int32_t* flags, int64_t* segments,
               int nthreads) {
  if (check_scene(s)) return 1;
  Model<double> m = make_model<double>(s, nullptr, 0.0, nullptr);
  parallel_for(n, nthreads, [&](int, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      V3d o, d;
      get_ray(s, pixel_ids, rays, i, o, d);
      RayStats st;
      V3d L = trace(m, o, d, 0, 1, 1.0, st);
      rgb[3 * i] = L.x; rgb[3 * i + 1] = L.y; rgb[3 * i + 2] = L.z;
      if (capped_w) capped_w[i] = st.capped_w;
      if (sig_topo) sig_topo[i] = st.sig_topo;
      if (sig_face) sig_face[i] = st.sig_face;
      if (flags) flags[i] = st.flags;
      if (segments) segments[i] = st.segments;
    }
  });
  return 0;
}

int dto_backward(const dto_scene* s, const int64_t* pixel_ids, const double* rays, int64_t n,
                 const double* grad_rgb, double* gV, double* gior, double* gsigma, int nthreads) {
  if (check_scene(s)) return 1;
  Model<double> m = make_model<double>(s, nullptr, 0.0, nullptr);
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  nthreads = (int)std::min<int64_t>(nthreads, std::max<int64_t>(n, 1));
  std::vector<Grad> Gs(nthreads);
  for (auto& G : Gs) {
    G.gV.assign(m.nv, V3d{0, 0, 0});
    G.gN.assign(m.nv, V3d{0, 0, 0});
    G.gsig.assign(m.sigma.size(), 0.0);
  }
  parallel_for(n, nthreads, [&](int t, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      V3d o, d;
      get_ray(s, pixel_ids, rays, i, o, d);
      V3d a = {grad_rgb[3 * i], grad_rgb[3 * i + 1], grad_rgb[3 * i + 2]};
      trace_bwd(m, o, d, 0, a, Gs[t]);   // camera-ray adjoints are dropped (R22)
    }
  });
  Grad G = Gs[0];
  for (int t = 1; t < nthreads; ++t) {   // fixed-order reduction
    for (int v = 0; v < m.nv; ++v) { G.gV[v] = G.gV[v] + Gs[t].gV[v]; G.gN[v] = G.gN[v] + Gs[t].gN[v]; }
    G.gior += Gs[t].gior;
    for (size_t j = 0; j < G.gsig.size(); ++j) G.gsig[j] += Gs[t].gsig[j];
  }
  vertex_normals_bwd(m, G);
  for (int v = 0; v < m.nv; ++v) { gV[3 * v] = G.gV[v].x; gV[3 * v + 1] = G.gV[v].y; gV[3 * v + 2] = G.gV[v].z; }
  *gior = G.gior;
  for (size_t j = 0; j < G.gsig.size(); ++j) gsigma[j] = G.gsig[j];
  return 0;
}

int dto_jvp(const dto_scene* s, const int64_t* pixel_ids, const double* rays, int64_t n, const double* tV,
            double tior, const double* tsigma, double* rgb, double* jvp_rgb, int nthreads) {
  if (check_scene(s)) return 1;
  Model<Dual> m = make_model<Dual>(s, tV, tior, tsigma);
  parallel_for(n, nthreads, [&](int, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      V3d od, dd;
      get_ray(s, pixel_ids, rays, i, od, dd);
      V3<Dual> o = {Dual(od.x), Dual(od.y), Dual(od.z)}, d = {Dual(dd.x), Dual(dd.y), Dual(dd.z)};
      RayStats st;
      V3<Dual> L = trace(m, o, d, 0, 1, 1.0, st);
      if (rgb) { rgb[3 * i] = L.x.v; rgb[3 * i + 1] = L.y.v; rgb[3 * i + 2] = L.z.v; }
      jvp_rgb[3 * i] = L.x.d; jvp_rgb[3 * i + 1] = L.y.d; jvp_rgb[3 * i + 2] = L.z.d;
    }
  });
  return 0;
}

int dto_closest_hit(const dto_scene* s, const double* rays, int64_t n, double t_lo, int32_t* face, double* tuv,
                    int32_t* flags, int nthreads) {
  if (check_scene(s)) return 1;
  Model<double> m = make_model<double>(s, nullptr, 0.0, nullptr);
  parallel_for(n, nthreads, [&](int, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      V3d o = {rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]}, d = {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
      Hit h = closest_hit(m, o, d, t_lo);
      face[i] = h.face;
      tuv[3 * i] = h.face >= 0 ? h.t : 0.0; tuv[3 * i + 1] = h.u; tuv[3 * i + 2] = h.v;
      if (flags) flags[i] = h.flags;
    }
  });
  return 0;
}

#ifdef DTO_PRECISION_STUDY
void dto_study_set_mask(int mask) { g_study_mask = mask; }
#endif

int dto_camera_rays(const dto_scene* s, const int64_t* pixel_ids, int64_t n, double* rays) {
  for (int64_t i = 0; i < n; ++i) {
    V3d o, d;
    camera_ray(s, pixel_ids ? pixel_ids[i] : i, o, d);
    rays[6 * i] = o.x; rays[6 * i + 1] = o.y; rays[6 * i + 2] = o.z;
    rays[6 * i + 3] = d.x; rays[6 * i + 4] = d.y; rays[6 * i + 5] = d.z;
  }
  return 0;
}

int dto_vertex_normals(const dto_scene* s, double* out) {
  if (check_scene(s)) return 1;
  Model<double> m = make_model<double>(s, nullptr, 0.0, nullptr);
  for (int v = 0; v < m.nv; ++v) { out[3 * v] = m.nrm[v].x; out[3 * v + 1] = m.nrm[v].y; out[3 * v + 2] = m.nrm[v].z; }
  return 0;
}

int dto_interface(const double* d, const double* n, double eta_i, double eta_t, double* out) {
  Iface<double> I = interface(V3d{d[0], d[1], d[2]}, V3d{n[0], n[1], n[2]}, eta_i, eta_t);
  out[0] = I.ci; out[1] = I.R; out[2] = I.T; out[3] = I.tir ? 1.0 : 0.0;
  out[4] = I.wr.x; out[5] = I.wr.y; out[6] = I.wr.z;
  out[7] = I.wt.x; out[8] = I.wt.y; out[9] = I.wt.z; out[10] = I.ct; out[11] = I.q;
  return 0;
}

int dto_env(const dto_scene* s, const double* o, const double* d, double* out) {
  V3d L = env<double>(s, V3d{o[0], o[1], o[2]}, V3d{d[0], d[1], d[2]});
  out[0] = L.x; out[1] = L.y; out[2] = L.z;
  return 0;
}

int dto_transmittance(const dto_scene* s, const double* o, const double* x, double* out) {
  Model<double> m;
  m.sc = s;
  size_t ns = sigma_len(s);
  if (s->sigma64) m.sigma.assign(s->sigma64, s->sigma64 + ns);
  else m.sigma.assign(s->sigma, s->sigma + ns);
  V3d t = transmittance(m, V3d{o[0], o[1], o[2]}, V3d{x[0], x[1], x[2]});
  out[0] = t.x; out[1] = t.y; out[2] = t.z;
  return 0;
}

}  // extern "C"
