// Device-side building blocks of the tracer: camera rays, ray/box and ray/triangle tests,
// the specular interface, Beer-Lambert transmittance, the frozen
// environment lookup (R14) and the local reverse-mode rules (DESIGN.md Appendix B).
// Float32 throughout.  Written independently of oracle/ (no shared code).
#pragma once
#include "dt_math.cuh"

namespace dt {

constexpr float kInf = __builtin_huge_valf();
#ifndef DT_WALK_LANES
#define DT_WALK_LANES 4
#endif
#ifndef DT_WALK_LANES_BWD
#define DT_WALK_LANES_BWD 4
#endif
#ifndef DT_WALK_LANES_HASH
#define DT_WALK_LANES_HASH 8
#endif
#ifndef DT_WALK_LANES_HASH_BWD
#define DT_WALK_LANES_HASH_BWD 4
#endif
constexpr int kWalkLanes = DT_WALK_LANES;          // lanes per sigma-grid segment walk, forward
constexpr int kWalkLanesBwd = DT_WALK_LANES_BWD;   // and backward (measured: tools/sweep_walk.sh)
// lanes per segment walk of the hash texture, by absorption kind
template <int ABS> struct WalkLanes { static constexpr int fwd = kWalkLanes, bwd = kWalkLanesBwd; };
template <> struct WalkLanes<2> { static constexpr int fwd = DT_WALK_LANES_HASH, bwd = DT_WALK_LANES_HASH_BWD; };
constexpr int kStackShared = 16;   // short stack entries per thread in shared memory
constexpr int kStackLocal = 112;   // spill entries per thread (local memory, L1-cached)
constexpr int kLeafMax = 3;        // triangles per wide-BVH leaf (a contiguous leaf-order range)
constexpr int kEmptyRef = 0x7fffffff;

// per-record event codes (the protocol numbering, shared only as a spec)
enum { EV_MISS = 0, EV_HIT_OUT = 1, EV_HIT_IN = 2, EV_HIT_OUT_TIR = 3, EV_HIT_IN_TIR = 4, EV_CAP_OUT = 5, EV_CAP_IN = 6,
       EV_CAP_DROP = 7 };   // EV_CAP_DROP: a hit at D_max discarded under CAP_ZERO (R13, R34)
// record flag bits (hit.w)
enum { RF_MISS = 1, RF_CAPPED = 2, RF_INSIDE = 4, RF_TIR = 8, RF_DEGEN = 16, RF_CULLED = 32 };

DT_D uint64_t topo_key(uint32_t pos, int ev) { return (uint64_t)pos | ((uint64_t)ev << 32); }
DT_D uint64_t face_key(uint32_t pos, int ev, int face) {
  return (uint64_t)pos | ((uint64_t)(uint32_t)(face + 1) << 20) | ((uint64_t)ev << 52);
}

struct DevScene {
  // mesh snapshot (dt_build_bvh)
  const float4* V;      // [nv] xyz
  const int* F;         // [nf*3]
  const D4* nrm;        // [nv] vertex normal xyz (float64), |sum of unit face normals| in w
  int nv, nf;
  // LBVH
  const float4* nodes;  // [(nf-1)*4] 64-B nodes: two child AABBs + child refs
  const float4* tris;   // [nf*3] 48-B triangles in leaf order: (v0, id), (e1, -), (e2, -)
  int root;             // internal node 0, or ~0 when nf == 1
  const float* scal;    // device scalars: [0..5] root box lo/hi, [6] t_min
  // material
  float ior;
  const float* ior_ptr;  // optional device IoR (dt_trace_opts.ior_device), read once per thread
  int abs_kind;
  const float4* sigma;  // internal copy: [1] (constant), [R^3] x-pairs (grid), [L*T] entries (hash)
  int sres, nsamp;
  float3 slo, shi;
  int hlevels, hlog2;   // hash texture (R29): levels, log2 table size
  unsigned hdense;      // bit l: level l indexed densely ((N_l+1)^3 <= T)
  int hres[32];         // cells per axis of each level
  // environment
  int env_kind;
  float3 ambient;
  const float* lobes;
  int nlobes;
  const float4* voxel;
  int vres;
  const float4* planes;
  int pres;
  int env_nsamp;        // volumetric env: samples per exterior segment (R30)
  float radius;
  int far_field;
  // options
  int max_depth, cap_policy;
  // walk counters (the texture walks' roofline, bench.py): [0] cell visits of the forward
  // optical-depth walks, [1] cell visits of the backward walks (each: 8 corner fetches; in the
  // backward also 8 float4 atomics), [2] volumetric-env samples replayed by the backward
  // (each: 8 voxel + 12 plane texels)
  unsigned long long* wcount;
};

// ----------------------------------------------------------------------------- camera (R19)
DT_D void camera_ray(const float* K, const float* c2w, int W, int H, int64_t pid, float3& o, float3& d) {
  int64_t hw = (int64_t)W * H;
  int view = (int)(pid / hw);
  int64_t rem = pid - (int64_t)view * hw;
  int y = (int)(rem / W), x = (int)(rem - (int64_t)y * W);
  const float* k = K + 4 * view;
  const float* m = c2w + 12 * view;
  float dx = ((float)x + 0.5f - k[2]) / k[0];
  float dy = ((float)y + 0.5f - k[3]) / k[1];
  float3 w = f3(m[0] * dx + m[1] * dy + m[2], m[4] * dx + m[5] * dy + m[6], m[8] * dx + m[9] * dy + m[10]);
  d = w * (1.0f / sqrtf(dot(w, w)));
  o = f3(m[3], m[7], m[11]);
}

// The same camera ray in float64: the tracer's geometric state.  Every product
// term matches the float32 formula above; only the precision differs.
DT_D void camera_ray64(const float* K, const float* c2w, int W, int H, int64_t pid, double3& o, double3& d) {
  const int64_t hw = (int64_t)W * H;
  const int view = (int)(pid / hw);
  const int64_t rem = pid - (int64_t)view * hw;
  const int y = (int)(rem / W), x = (int)(rem - (int64_t)y * W);
  const float* k = K + 4 * view;
  const float* m = c2w + 12 * view;
  const double dx = ((double)x + 0.5 - (double)k[2]) * rcp64((double)k[0]);
  const double dy = ((double)y + 0.5 - (double)k[3]) * rcp64((double)k[1]);
  const double3 w = d3((double)m[0] * dx + (double)m[1] * dy + (double)m[2],
                       (double)m[4] * dx + (double)m[5] * dy + (double)m[6],
                       (double)m[8] * dx + (double)m[9] * dy + (double)m[10]);
  d = w * rsqrt64(dot(w, w));
  o = d3((double)m[3], (double)m[7], (double)m[11]);
}

// ----------------------------------------------------------------------------- intersection
// Explicit intrinsics (fixed fma / rounding, never re-contracted by the compiler), so the LBVH
// traversal, the brute-force test and the backward replay produce bit-identical (t, u, v).
DT_D float3 sub_rn(float3 a, float3 b) { return f3(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z)); }
DT_D float dot_rn(float3 a, float3 b) {
  return __fmaf_rn(a.z, b.z, __fmaf_rn(a.y, b.y, __fmul_rn(a.x, b.x)));
}
DT_D float3 cross_rn(float3 a, float3 b) {
  return f3(__fmaf_rn(a.y, b.z, -__fmul_rn(a.z, b.y)), __fmaf_rn(a.z, b.x, -__fmul_rn(a.x, b.z)),
            __fmaf_rn(a.x, b.y, -__fmul_rn(a.y, b.x)));
}
#ifndef DT_RCP_FTZ
#define DT_RCP_FTZ 1
#endif
DT_D float rcp_approx(float x) {   // MUFU.RCP (~1 ulp): one instruction, same in every caller
  float r;
#if DT_RCP_FTZ
  // a subnormal determinant (|det| < 2^-126) is flushed to 0: rcp = inf, the test then rejects
  // (no degenerate triangle of the inputs comes near; saves the subnormal rescaling)
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
#else
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
#endif
  return r;
}

// Moller-Trumbore (R15/R16): hit iff det != 0, u >= 0, v >= 0, u + v <= 1, t > t_lo.
DT_D bool intersect_tri(float3 o, float3 d, float3 v0, float3 e1, float3 e2, float t_lo, float& t, float& u,
                        float& v) {
  float3 p = cross_rn(d, e2);
  float det = dot_rn(e1, p);
  if (det == 0.0f) return false;
  float inv = rcp_approx(det);
  float3 s = sub_rn(o, v0);
  u = __fmul_rn(dot_rn(s, p), inv);
  if (!(u >= 0.0f)) return false;
  float3 q = cross_rn(s, e1);
  v = __fmul_rn(dot_rn(d, q), inv);
  if (!(v >= 0.0f) || !(__fadd_rn(u, v) <= 1.0f)) return false;
  t = __fmul_rn(dot_rn(e2, q), inv);
  return t > t_lo;
}
// ----------------------------------------------------------------------------- wide nodes
// 64-B 4-wide node (layout in bvh.cu, write_wide_node): child c's box decodes to
// lo = p + qlo * s, hi = p + qhi * s with per-axis power-of-two scales s (one fma per plane).
// per-axis power-of-two scales of a node: x in n0.w, y in n3.z, z in n3.w (fp32 bit patterns)
DT_D float3 node_scale(uint4 n0, uint4 n3) {
  return f3(__uint_as_float(n0.w), __uint_as_float(n3.z), __uint_as_float(n3.w));
}
// One 256-bit read-only load (sm_100: LDG.E.ENL2.256): a 64-B node is two instructions.
DT_D void ldg256(const uint4* p, uint4& a, uint4& b) {
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
}
DT_D void ldg256f(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}
DT_D int wide_ref(uint4 n2, uint4 n3, int c) {
  return (int)(c == 0 ? n2.z : c == 1 ? n2.w : c == 2 ? n3.x : n3.y);
}
DT_D void decode_wide_child(uint4 n0, uint4 n1, uint4 n2, uint4 n3, int c, float3& lo, float3& hi) {
  float3 p = f3(__uint_as_float(n0.x), __uint_as_float(n0.y), __uint_as_float(n0.z));
  const float3 sc = node_scale(n0, n3);
  const float sx = sc.x, sy = sc.y, sz = sc.z;
  int sh = 8 * c;
  lo = f3(fmaf((float)((n1.x >> sh) & 0xff), sx, p.x), fmaf((float)((n1.y >> sh) & 0xff), sy, p.y),
          fmaf((float)((n1.z >> sh) & 0xff), sz, p.z));
  hi = f3(fmaf((float)((n1.w >> sh) & 0xff), sx, p.x), fmaf((float)((n2.x >> sh) & 0xff), sy, p.y),
          fmaf((float)((n2.y >> sh) & 0xff), sz, p.z));
}
DT_D void leaf_range(int ref, int& first, int& cnt) {
  int x = ~ref;
  first = x >> 2;
  cnt = (x & 3) + 1;
}

DT_D float3 safe_inv(float3 d) {
  const float e = 1e-20f;
  return f3(1.0f / (fabsf(d.x) < e ? copysignf(e, d.x) : d.x), 1.0f / (fabsf(d.y) < e ? copysignf(e, d.y) : d.y),
            1.0f / (fabsf(d.z) < e ? copysignf(e, d.z) : d.z));
}

// Conservative slab test: padded so that no box whose triangle the exact-rounding test
// above would accept is culled (boxes are also inflated at build time).
DT_D bool slab(float lx, float hx, float ly, float hy, float lz, float hz, float3 o, float3 inv, float tbest,
               float& tnear) {
  float tx0 = (lx - o.x) * inv.x, tx1 = (hx - o.x) * inv.x;
  float ty0 = (ly - o.y) * inv.y, ty1 = (hy - o.y) * inv.y;
  float tz0 = (lz - o.z) * inv.z, tz1 = (hz - o.z) * inv.z;
  float tmin = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
  float tmax = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tbest));
  tnear = tmin;
  return tmin * 0.99999f <= tmax * 1.00001f;
}

// Closest-hit traversal state of one ray through the 4-wide BVH.  Ties in t resolve to the
// lowest ORIGINAL face id (R18), so the answer does not depend on the visiting order.
struct Trav {
  int cur, sp, best;
  float bt, bu, bv;
};

DT_D void trav_init(Trav& T) {
  T.cur = 0;
  T.sp = 0;
  T.best = -1;
  T.bt = kInf;
  T.bu = T.bv = 0.0f;
}

#define DT_CX(a, b)                                              \
  if (k##b < k##a) {                                             \
    float tk = k##a; k##a = k##b; k##b = tk;                     \
    int tr = r##a; r##a = r##b; r##b = tr;                       \
  }

// quantised plane byte c of word w as a float (exact, 0..255; I2F.U8 with a byte select)
DT_D float qbyte(unsigned w, int c) { return (float)((w >> (8 * c)) & 0xff); }

// DT_TLO_CULL = 1: a child box the ray leaves before t_lo (R17) cannot hold a hit: its entry
// distance is clamped at t_lo instead of 0 (secondary rays skip the thin boxes of the surface
// they start on)
#ifndef DT_TLO_CULL
#define DT_TLO_CULL 1
#endif
// Entry distances of the four child boxes of a 64-B wide node (kInf: missed or empty child),
// clamped below at tlo (a box exited before tlo is missed).  Plane distance
// t = (p + q 2^e - o) / d = q * A + B with A = 2^e / d, B = (p - o) / d: one FMA per plane;
// its rounding (~1 ulp of |p - o|) is far inside the box padding.  The near and far plane of
// each axis are picked once per node by the sign of the ray direction (t is monotone in q),
// so a child needs one max and one min chain; the slab comparison tmin <= tmax * 1.000021 is
// the padded tmin * 0.99999 <= tmax * 1.00001 with the two factors merged (slightly more
// permissive).  Variants measured against this one: profiles/r01_traversal_sweep.txt.
DT_D void node_keys(uint4 n0, uint4 n1, uint4 n2, uint4 n3, const int (&r)[4], float3 o, float3 inv, float bt,
                    float (&key)[4], float tlo = 0.0f) {
  const float3 sc = node_scale(n0, n3);
  const float3 A = f3(sc.x * inv.x, sc.y * inv.y, sc.z * inv.z);
  const float3 B = f3((__uint_as_float(n0.x) - o.x) * inv.x, (__uint_as_float(n0.y) - o.y) * inv.y,
                      (__uint_as_float(n0.z) - o.z) * inv.z);
  const bool sx = inv.x < 0.0f, sy = inv.y < 0.0f, sz = inv.z < 0.0f;
  const unsigned xn = sx ? n1.w : n1.x, xf = sx ? n1.x : n1.w;
  const unsigned yn = sy ? n2.x : n1.y, yf = sy ? n1.y : n2.x;
  const unsigned zn = sz ? n2.y : n1.z, zf = sz ? n1.z : n2.y;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float tmin = fmaxf(fmaxf(fmaf(qbyte(xn, c), A.x, B.x), fmaf(qbyte(yn, c), A.y, B.y)),
                             fmaxf(fmaf(qbyte(zn, c), A.z, B.z), tlo));
    const float tmax = fminf(fminf(fmaf(qbyte(xf, c), A.x, B.x), fmaf(qbyte(yf, c), A.y, B.y)),
                             fminf(fmaf(qbyte(zf, c), A.z, B.z), bt));
    key[c] = tmin <= tmax * 1.000021f && r[c] != kEmptyRef ? tmin : kInf;
  }
}

// The traversal stack: entry i lives in this thread's shared column (sstack[i * stride]) for
// i < kStackShared, else in lstack (local memory).
DT_D void stack_push(Trav& T, int* sstack, int stride, int* lstack, int ref, int& err) {
  if (T.sp < kStackShared) sstack[T.sp * stride] = ref;
  else if (T.sp < kStackShared + kStackLocal) lstack[T.sp - kStackShared] = ref;
  else err = 1;
  ++T.sp;
}
// Pops the top entry into T.cur; false when the stack is empty.
DT_D bool stack_pop(Trav& T, const int* sstack, int stride, const int* lstack) {
  if (T.sp == 0) return false;
  --T.sp;
  T.cur = T.sp < kStackShared ? sstack[T.sp * stride] : lstack[T.sp - kStackShared];
  return true;
}

// Tests the triangles of leaf T.cur against the ray, keeping the closest hit (R18 ties).
DT_D void leaf_test(const DevScene& s, float3 o, float3 d, float t_lo, Trav& T, int& tests) {
  int first, cnt;
  leaf_range(T.cur, first, cnt);
  DT_CHECK(first >= 0 && first + cnt <= s.nf);
  const float4* tr = s.tris + 3 * (size_t)first;
  do {                                            // a leaf holds 1..kLeafMax triangles
    float4 a = __ldg(tr), b = __ldg(tr + 1), c = __ldg(tr + 2);
    float t, u, v;
    ++tests;
    if (intersect_tri(o, d, f3(a), f3(b), f3(c), t_lo, t, u, v)) {
      int id = __float_as_int(a.w);
      if (t < T.bt || (t == T.bt && id < T.best)) { T.bt = t; T.bu = u; T.bv = v; T.best = id; }
    }
    tr += 3;
  } while (--cnt > 0);
}

// One traversal step: visit the current wide node (test its four child boxes, descend into
// the nearest hit, push the others far-to-near, or pop when none is hit); then, in the same
// step, test the leaf it descended into or popped and pop again.  A warp whose lanes are split
// between the node and the leaf code runs both halves every step anyway; fused, a lane does
// both in one step (r02: C3 traversal 48.1 -> 46.6 ms, profiles/r02_traversal_sweep.txt).
// Returns true when the ray is finished.  sstack: this thread's column of the block's shared
// short stack (stride = blockDim.x); entries beyond kStackShared spill to lstack (local memory).
DT_D bool trav_step(const DevScene& s, float3 o, float3 d, float3 inv, float t_lo, Trav& T, int* sstack, int stride,
                    int* lstack, int& err, int& visits, int& tests) {
  if (T.cur >= 0) {
    DT_CHECK(T.cur < max(s.nf - 1, 1));
    const uint4* nd = reinterpret_cast<const uint4*>(s.nodes) + 4 * (size_t)T.cur;
    uint4 n0, n1, n2, n3;
    ldg256(nd, n0, n1);
    ldg256(nd + 2, n2, n3);
    ++visits;
    int r0 = (int)n2.z, r1 = (int)n2.w, r2 = (int)n3.x, r3 = (int)n3.y;
    float key[4];
    node_keys(n0, n1, n2, n3, {r0, r1, r2, r3}, o, inv, T.bt, key, DT_TLO_CULL ? t_lo : 0.0f);
    float k0 = key[0], k1 = key[1], k2 = key[2], k3 = key[3];
    DT_CX(0, 1) DT_CX(2, 3) DT_CX(0, 2) DT_CX(1, 3) DT_CX(1, 2)   // ascending by entry distance
    if (k0 < kInf) {
      const int h = (k1 < kInf) + (k2 < kInf) + (k3 < kInf);
      if (T.sp + 3 <= kStackShared) {
        int* top = sstack + (T.sp + h - 1) * stride;
        if (h > 0) top[0] = r1;
        if (h > 1) top[-stride] = r2;
        if (h > 2) top[-2 * stride] = r3;
        T.sp += h;
      } else {
        const int push[3] = {r3, r2, r1};
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (q >= 3 - h) stack_push(T, sstack, stride, lstack, push[q], err);
      }
      T.cur = r0;
    } else if (err || !stack_pop(T, sstack, stride, lstack)) {
      return true;
    }
  }
  if (T.cur < 0) {
    leaf_test(s, o, d, t_lo, T, tests);
    if (err || !stack_pop(T, sstack, stride, lstack)) return true;
  }
  return false;
}

#undef DT_CX

// Closest hit (whole traversal).  Returns the original face id or -1.
DT_D int traverse(const DevScene& s, float3 o, float3 d, float t_lo, float& bt, float& bu, float& bv, int* sstack,
                  int stride, int& err, int& visits, int& tests) {
  float3 inv = safe_inv(d);
  int lstack[kStackLocal];
  Trav T;
  trav_init(T);
  while (!trav_step(s, o, d, inv, t_lo, T, sstack, stride, lstack, err, visits, tests)) {
  }
  bt = T.bt;
  bu = T.bu;
  bv = T.bv;
  return T.best;
}

// Triangle of ORIGINAL face f from the snapshot, in float64: v0 and the edges v1 - v0, v2 - v0
// (exact in float64 for float32 vertices).
// The same from the face's vertex indices (handed over in the hit record by the traversal).
DT_D void tri64(const DevScene& s, int i0, int i1, int i2, double3& v0, double3& e1, double3& e2) {
  DT_CHECK(i0 >= 0 && i0 < s.nv && i1 >= 0 && i1 < s.nv && i2 >= 0 && i2 < s.nv);
  v0 = d3(__ldg(s.V + i0));
  e1 = d3(__ldg(s.V + i1)) - v0;
  e2 = d3(__ldg(s.V + i2)) - v0;
}
// Traversal output record: (face, i0, i1, i2) as int bits; the indices are fetched once per
// ray when its traversal ends, so the shade's first dependent fetch is the vertices.
DT_D float4 hit_record(const DevScene& s, int face) {
  int i0 = 0, i1 = 0, i2 = 0;
  if (face >= 0) {
    DT_CHECK(face < s.nf);
    i0 = __ldg(s.F + 3 * face); i1 = __ldg(s.F + 3 * face + 1); i2 = __ldg(s.F + 3 * face + 2);
  }
  return make_float4(__int_as_float(face), __int_as_float(i0), __int_as_float(i1), __int_as_float(i2));
}
DT_D void face_tri64(const DevScene& s, int f, int& i0, int& i1, int& i2, double3& v0, double3& e1, double3& e2) {
  DT_CHECK(f >= 0 && f < s.nf);
  i0 = __ldg(s.F + 3 * f); i1 = __ldg(s.F + 3 * f + 1); i2 = __ldg(s.F + 3 * f + 2);
  DT_CHECK(i0 >= 0 && i0 < s.nv && i1 >= 0 && i1 < s.nv && i2 >= 0 && i2 < s.nv);
  v0 = d3(__ldg(s.V + i0));
  e1 = d3(__ldg(s.V + i1)) - v0;
  e2 = d3(__ldg(s.V + i2)) - v0;
}

// Moller-Trumbore solve o + t d = v0 + u e1 + v e2 in float64 (R15, R16) for the face the
// traversal selected (float32 candidate search, conservative boxes): the hit point, the
// barycentrics and everything downstream use these values.
// Returns 1 / det.
DT_D double mt64(double3 o, double3 d, double3 v0, double3 e1, double3 e2, double& t, double& u, double& v) {
  const double3 p = cross(d, e2);
  const double inv = rcp64(dot(e1, p));
  const double3 sv = o - v0;
  u = dot(sv, p) * inv;
  const double3 q = cross(sv, e1);
  v = dot(d, q) * inv;
  t = dot(e2, q) * inv;
  return inv;
}

// ----------------------------------------------------------------------------- interface
// One specular event (R1-R5, R7, R8), float64.  Everything the reverse pass needs.
struct Shade {
  double3 n, wr, wt;            // oriented shading normal, reflect / refract directions
  double Lm, ci, eta, eta_i, eta_t, q, ct, R, T;
  double b0, b1, b2;
  bool inside, tir, clamped, degen, fb;
};

DT_D void shade_forward(const DevScene& s, double ior, int i0, int i1, int i2, double3 e1, double3 e2, double3 d,
                        double u, double v, bool inside, Shade& S) {
  S.inside = inside;
  S.b0 = 1.0 - u - v; S.b1 = u; S.b2 = v;
  const double3 n0 = xyz(ldg_d4(s.nrm + i0)), n1 = xyz(ldg_d4(s.nrm + i1)), n2 = xyz(ldg_d4(s.nrm + i2));
  const double3 m = n0 * S.b0 + n1 * S.b1 + n2 * S.b2;       // n(x) = sum beta_i n_vi
  const double mm = dot(m, m);
  S.fb = !(mm >= 1e-24);                                      // |m| < 1e-12: geometric normal (R7)
  double3 ns;
  if (!S.fb) {
    const double rl = rsqrt64(mm);
    S.Lm = mm * rl;
    ns = m * rl;
  } else {
    const double3 c = cross(e1, e2);
    S.Lm = 0.0;
    ns = c * rsqrt64(dot(c, c));
  }
  S.n = inside ? -ns : ns;
  S.eta_i = inside ? ior : 1.0;
  S.eta_t = inside ? 1.0 : ior;
  const double c_raw = -dot(d, S.n);                          // omega_i . n, omega_i = -d
  S.clamped = !(c_raw > 0.0);
  S.ci = S.clamped ? 0.0 : fmin(c_raw, 1.0);
  S.eta = S.eta_t * rcp64(S.eta_i);
  S.q = S.eta * S.eta - 1.0 + S.ci * S.ci;
  S.wr = S.n * (2.0 * S.ci) + d;
  S.tir = S.q < 0.0;
  S.degen = false;
  if (S.tir) { S.ct = 0.0; S.R = 1.0; S.T = 0.0; S.wt = d3(0, 0, 0); return; }
  const double ie = rcp64(S.eta);
  S.ct = sqrt64(S.q) * ie;
  S.wt = (d + S.n * S.ci) * ie - S.n * S.ct;                  // P:106-108 (R4): -(omega_i - c n)/eta - ct n
  if (S.ci == 0.0 && S.ct == 0.0) { S.degen = true; S.R = 1.0; S.T = 0.0; return; }
  const double A = S.eta_i * S.ci, B = S.eta_t * S.ct, C = S.eta_i * S.ct, D = S.eta_t * S.ci;
  const double rs = (A - B) * rcp64(A + B), rp = (C - D) * rcp64(C + D);
  S.R = 0.5 * (rs * rs + rp * rp);
  S.T = 1.0 - S.R;
}

// The interface state the reverse pass needs, rounded to float32 once it has been evaluated
// in float64 (the reverse scales float32 adjoints by these Jacobian terms; the state itself,
// where the float32 error would be amplified along the path, stays float64).
struct ShadeF {
  float3 n;
  float Lm, ci, eta, eta_i, eta_t, q, ct, b0, b1, b2;
  bool inside, tir, clamped, degen, fb;
};
DT_D ShadeF shade_f32(const Shade& S) {
  ShadeF F;
  F.n = f3(S.n);
  F.Lm = (float)S.Lm; F.ci = (float)S.ci; F.eta = (float)S.eta; F.eta_i = (float)S.eta_i; F.eta_t = (float)S.eta_t;
  F.q = (float)S.q; F.ct = (float)S.ct; F.b0 = (float)S.b0; F.b1 = (float)S.b1; F.b2 = (float)S.b2;
  F.inside = S.inside; F.tir = S.tir; F.clamped = S.clamped; F.degen = S.degen; F.fb = S.fb;
  return F;
}

// Reverse of shade_forward: given dL/dR (T = 1 - R folded in), dL/dwr, dL/dwt, returns
// dL/dd (through omega_i = -d), dL/d(u, v) (through the shading normal), d/dn_vk and d/dior.
DT_D void shade_backward(const ShadeF& S, float3 d, float gR, float3 gwr, float3 gwt, float3 nv0, float3 nv1, float3 nv2,
                         float3& gd, float& gu, float& gv, float3 gN[3], float& gior) {
  float gci = 0.0f, geta = 0.0f, geta_i = 0.0f, geta_t = 0.0f;
  float3 gn = f3(0, 0, 0), gwi = f3(0, 0, 0);
  const float3 wi = -d;
  if (!S.tir && !S.degen) {
    float A = S.eta_i * S.ci, B = S.eta_t * S.ct, C = S.eta_i * S.ct, D = S.eta_t * S.ci;
    float rs = (A - B) / (A + B), rp = (C - D) / (C + D);
    float grs = gR * rs, grp = gR * rp;
    float iab = 1.0f / ((A + B) * (A + B)), icd = 1.0f / ((C + D) * (C + D));
    float gA = grs * 2.0f * B * iab, gB = -grs * 2.0f * A * iab;
    float gC = grp * 2.0f * D * icd, gD = -grp * 2.0f * C * icd;
    float gct = gB * S.eta_t + gC * S.eta_i;
    gci += gA * S.eta_i + gD * S.eta_t;
    geta_i += gA * S.ci + gC * S.ct;
    geta_t += gB * S.ct + gD * S.ci;
    // the transmitted direction omega_t = -(omega_i - ci n)/eta - ct n and cos(theta_t) below
    float ie = 1.0f / S.eta;
    gwi -= gwt * ie;
    gci += dot(gwt, S.n) * ie;
    gn += gwt * (S.ci * ie) - gwt * S.ct;
    geta += dot(gwt, wi - S.n * S.ci) * ie * ie;
    gct -= dot(gwt, S.n);
    float sq = sqrtf(S.q);
    float gq = sq > 0.0f ? gct / (2.0f * S.eta * sq) : 0.0f;
    geta += -gct * sq * ie * ie + gq * 2.0f * S.eta;
    gci += gq * 2.0f * S.ci;
  }
  // degen (both cosines 0): R = 1, T = 0 constant; the refracted child carries zero adjoint.
  // omega_r = 2 ci n - omega_i
  gci += 2.0f * dot(gwr, S.n);
  gn += gwr * (2.0f * S.ci);
  gwi -= gwr;
  // eta = eta_t / eta_i
  geta_t += geta / S.eta_i;
  geta_i -= geta * S.eta_t / (S.eta_i * S.eta_i);
  gior = S.inside ? geta_i : geta_t;
  // ci = clamp(omega_i . n): the lower clamp stops the gradient (R3)
  if (!S.clamped) { gwi += S.n * gci; gn += wi * gci; }
  gd = -gwi;
  gu = gv = 0.0f;
  gN[0] = gN[1] = gN[2] = f3(0, 0, 0);
  if (!S.fb) {
    const float3 gns = S.inside ? -gn : gn, ns = S.inside ? -S.n : S.n;
    float3 gm = (gns - ns * dot(ns, gns)) * (1.0f / S.Lm);
    gN[0] = gm * S.b0; gN[1] = gm * S.b1; gN[2] = gm * S.b2;
    float g0 = dot(gm, nv0), g1 = dot(gm, nv1), g2 = dot(gm, nv2);
    gu = g1 - g0;
    gv = g2 - g0;
  }
}

// Reverse of the Moller-Trumbore solve M [u v t]^T = o - v0 with M = [e1 e2 -d]:
// lambda = M^-T (gu, gv, gt); go += lambda, gd += t lambda, gV_k = -beta_k lambda.  The
// determinant's reciprocal from the float64 geometry (idet), the rest float32.
DT_D void mt_backward(float3 d, float3 e1, float3 e2, float idet, float t, float u, float v, float gu, float gv,
                      float gt, float3& go, float3& gd, float3 gV[3]) {
  float3 de2 = cross(d, e2), e1d = cross(e1, d), e12 = cross(e1, e2);
  float3 lam = (de2 * gu + e1d * gv + e12 * gt) * idet;
  go += lam;
  gd += lam * t;
  gV[0] = lam * -(1.0f - u - v);
  gV[1] = lam * -u;
  gV[2] = lam * -v;
}

// ----------------------------------------------------------------------------- absorption
DT_D size_t cell_node(size_t base, int k, int R) {
  return base + ((size_t)(k >> 2) * R + ((k >> 1) & 1)) * R + (k & 1);
}

// Optical depth of a constant-sigma segment and its reverse (ABS = DT_ABS_CONST); the chord
// length from the float64 end points.
DT_D float3 transmittance_const(const DevScene& s, double3 o, double3 x) {
  const float3 S = f3(__ldg(s.sigma)) * (float)length(x - o);
  return f3(expf(-S.x), expf(-S.y), expf(-S.z));
}

// (the chord o -> x = o + t d: length t |d|, direction d / |d|)
DT_D void transmittance_const_backward(const DevScene& s, float l, float3 dh, float3 gS, float3& gx, float3& go,
                                       float3& gsc) {
  gsc += gS * l;
  if (l > 0.0f) {
    const float3 u = dh * dot(gS, f3(__ldg(s.sigma)));
    gx += u;
    go -= u;
  }
}

// Sigma grid (ABS = DT_ABS_GRID): the N midpoint samples x_j = o + t_j (x - o),
// t_j = (j + 1/2)/N, of an interior segment (R10, R11) are evaluated cooperatively by a group
// of lanes (group_* below) instead of by the segment's own lane alone (which would leave
// the warp divergent and serialise ~N/3 dependent corner fetches per lane).
struct GridMap {
  float3 lo, scl;          // g = (p - lo) * scl, scl = (R-1)/(hi-lo)
  int R, N;
};

DT_D GridMap grid_map(const DevScene& s) {
  GridMap m;
  m.R = s.sres;
  m.N = s.nsamp;
  m.lo = s.slo;
  const float span = s.abs_kind == 2 ? 1.0f : (float)(m.R - 1);   // hash: unit box coordinates
  m.scl = f3(span / (s.shi.x - s.slo.x), span / (s.shi.y - s.slo.y), span / (s.shi.z - s.slo.z));
  return m;
}

DT_D void corner_weights(const float f[3], float w[8]);

// one 64-bit atomic per warp: the warp's cell visits of one walk call (all 32 lanes call it)
DT_D void flush_walk_count(unsigned long long* c, int cells) {
  const unsigned tot = __reduce_add_sync(~0u, (unsigned)cells);
  if (c && lane_id() == 0 && tot) atomicAdd(c, (unsigned long long)tot);
}

// ---- hash texture (ABS = DT_ABS_HASH, R29): mu(p) = sum_l trilinear lookup of level l
// Table entry of corner (x, y, z) at level l (N cells per axis, T = 2^hlog2 entries).
DT_D uint32_t hash_index(const DevScene& s, int l, int N, int x, int y, int z) {
  const uint32_t T1 = (1u << s.hlog2) - 1u;
  if ((s.hdense >> l) & 1u) {
    const uint32_t n1 = (uint32_t)N + 1u;
    DT_CHECK(x >= 0 && y >= 0 && z >= 0 && x <= N && y <= N && z <= N && n1 * n1 * n1 <= (1u << s.hlog2));
    return (uint32_t)x + n1 * ((uint32_t)y + n1 * (uint32_t)z);
  }
  return ((uint32_t)x ^ ((uint32_t)y * 2654435761u) ^ ((uint32_t)z * 805459861u)) & T1;
}

// Unit-box coordinates of p; false outside the box (zero there, R11).
DT_D bool hash_unit(const GridMap& m, float3 p, float u[3]) {
  u[0] = (p.x - m.lo.x) * m.scl.x;
  u[1] = (p.y - m.lo.y) * m.scl.y;
  u[2] = (p.z - m.lo.z) * m.scl.z;
  return u[0] >= 0.f && u[0] <= 1.f && u[1] >= 0.f && u[1] <= 1.f && u[2] >= 0.f && u[2] <= 1.f;
}

DT_D void hash_cell(const float u[3], int N, int i[3], float f[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float g = u[a] * (float)N;
    i[a] = min((int)floorf(g), N - 1);
    f[a] = g - (float)i[a];
  }
}

// Cell and local coordinates of p (zero outside the box, R11).
DT_D bool grid_cell(const GridMap& m, float3 p, int& base, float f[3]) {
  const float g[3] = {(p.x - m.lo.x) * m.scl.x, (p.y - m.lo.y) * m.scl.y, (p.z - m.lo.z) * m.scl.z};
  const float top = (float)(m.R - 1);
  if (!(g[0] >= 0.f && g[0] <= top && g[1] >= 0.f && g[1] <= top && g[2] >= 0.f && g[2] <= top)) return false;
  int i[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    i[a] = min((int)floorf(g[a]), m.R - 2);
    f[a] = g[a] - (float)i[a];
  }
  base = (i[2] * m.R + i[1]) * m.R + i[0];
  return true;
}

// The 8 corner values of a cell: 4 x-pair loads (256-bit) of the packed grid.
DT_D void grid_corners(const DevScene& s, const GridMap& m, int base, float3 c[8]) {
#pragma unroll
  for (int yz = 0; yz < 4; ++yz) {
    float4 p, q;
    DT_CHECK(base >= 0 && cell_node((size_t)base, yz << 1, m.R) < (size_t)m.R * m.R * m.R);
    ldg256f(s.sigma + 2 * cell_node((size_t)base, yz << 1, m.R), p, q);
    c[yz << 1] = f3(p.x, p.y, p.z);
    c[(yz << 1) | 1] = f3(p.w, q.x, q.y);
  }
}

DT_D void corner_weights(const float f[3], float w[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    w[k] = ((k & 1) ? f[0] : 1 - f[0]) * ((k & 2) ? f[1] : 1 - f[1]) * ((k & 4) ? f[2] : 1 - f[2]);
}

// Segments are walked by groups of G lanes (G | 32): the warp takes up to 32/G pending
// segments at a time, and lane i of a group takes the P = ceil(N/G) consecutive samples
// [iP, iP + P).  Consecutive samples mostly share a cell, so a lane loads a cell's corners
// once per run of samples (one dependent load batch per ~3 samples), and the 32/G walks of
// the warp proceed side by side (memory-level parallelism across segments).
// group_take: assigns the next pending lanes of the warp-uniform `mask` to the groups;
// returns this lane's group source lane (-1: idle group) and, in `myq`, the group that walks
// this lane's own segment (-1: none).
template <int G>
DT_D int group_take(unsigned& mask, int& myq) {
  const int grp = lane_id() / G;
  int mine = -1;
  myq = -1;
#pragma unroll
  for (int q = 0; q < 32 / G; ++q) {
    const int src = mask ? __ffs(mask) - 1 : -1;
    if (mask) mask &= mask - 1;
    if (q == grp) mine = src;
    if (src == lane_id()) myq = q;
  }
  return mine;
}

// sum_j mu(x_j) * |x - o| / N (the optical depth of R10) of the group's segment, returned on
// every lane of the group.  All 32 lanes call it (inactive groups pass active = false).
template <int G, int ABS>
DT_D float3 group_optical_depth(const DevScene& s, const GridMap& m, float3 o, float3 x, bool active) {
  const float3 dx = x - o;
  float3 S = f3(0, 0, 0);
  int cells = 0;
  if (ABS == 2 && active) {            // hash texture: level by level, corners reused per cell run
    const int P = (m.N + G - 1) / G, j0 = (lane_id() % G) * P, j1 = min(j0 + P, m.N);
    const size_t T = (size_t)1 << s.hlog2;
    for (int l = 0; l < s.hlevels; ++l) {
      const int N = s.hres[l];
      const float4* tab = s.sigma + (size_t)l * T;
      int cur[3] = {-1, -1, -1};
      float3 c[8];
      float acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.f;
      for (int j = j0; j < j1; ++j) {
        float u[3];
        if (!hash_unit(m, o + dx * (((float)j + 0.5f) / (float)m.N), u)) continue;
        int i[3];
        float f[3], w[8];
        hash_cell(u, N, i, f);
        if (i[0] != cur[0] || i[1] != cur[1] || i[2] != cur[2]) {
          if (cur[0] >= 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              S += c[k] * acc[k];
              acc[k] = 0.f;
            }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            c[k] = f3(__ldg(tab + hash_index(s, l, N, i[0] + (k & 1), i[1] + ((k >> 1) & 1), i[2] + (k >> 2))));
          cur[0] = i[0]; cur[1] = i[1]; cur[2] = i[2];
          ++cells;
        }
        corner_weights(f, w);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += w[k];
      }
      if (cur[0] >= 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) S += c[k] * acc[k];
      }
    }
  } else if (active) {
    const int P = (m.N + G - 1) / G, j0 = (lane_id() % G) * P, j1 = min(j0 + P, m.N);
    int cur = -1;
    float3 c[8];
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    for (int j = j0; j < j1; ++j) {
      int base;
      float f[3], w[8];
      if (!grid_cell(m, o + dx * (((float)j + 0.5f) / (float)m.N), base, f)) continue;
      if (base != cur) {               // new cell: fold the finished run, fetch the corners
        if (cur >= 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            S += c[k] * acc[k];
            acc[k] = 0.f;
          }
        }
        grid_corners(s, m, base, c);   // consumed at the run's end: latency behind the run
        cur = base;
        ++cells;
      }
      corner_weights(f, w);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += w[k];
    }
    if (cur >= 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) S += c[k] * acc[k];
    }
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    S.x += __shfl_xor_sync(~0u, S.x, off);
    S.y += __shfl_xor_sync(~0u, S.y, off);
    S.z += __shfl_xor_sync(~0u, S.z, off);
  }
  flush_walk_count(s.wcount, cells);
  return S * (length(dx) / (float)m.N);
}

// Reverse of group_optical_depth given gS = dL/d(optical depth): scatters gS * (l/N) * w_k
// into the float4 grid adjoint gsig (each lane merges its run of samples per cell, then 8
// vector atomics per cell visit) and returns the position adjoints of o and x on every lane
// of the group.
template <int G, int ABS>
DT_D void group_transmittance_backward(const DevScene& s, const GridMap& m, float3 o, float3 x, float3 gS,
                                       bool active, float4* gsig, float3& gx, float3& go) {
  const float3 dx = x - o;
  const float l = length(dx);
  const float invN = 1.0f / (float)m.N, sc = l * invN;
  const float3 gSs = gS * sc;
  float gl = 0.f;
  float3 gsum = f3(0, 0, 0), gtsum = f3(0, 0, 0);
  int cells = 0;
  if (ABS == 2 && active) {            // hash texture: level by level, merged per cell run
    const int P = (m.N + G - 1) / G, j0 = (lane_id() % G) * P, j1 = min(j0 + P, m.N);
    const size_t T = (size_t)1 << s.hlog2;
    for (int l = 0; l < s.hlevels; ++l) {
      const int N = s.hres[l];
      const size_t lt = (size_t)l * T;
      int cur[3] = {-1, -1, -1};
      uint32_t e[8];
      float gk[8], acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) { acc[k] = gk[k] = 0.f; e[k] = 0u; }
      for (int j = j0; j < j1; ++j) {
        const float t = ((float)j + 0.5f) * invN;
        float u[3];
        if (!hash_unit(m, o + dx * t, u)) continue;
        int i[3];
        float f[3], w[8];
        hash_cell(u, N, i, f);
        if (i[0] != cur[0] || i[1] != cur[1] || i[2] != cur[2]) {
          if (cur[0] >= 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              atomicAdd(gsig + lt + e[k], make_float4(gSs.x * acc[k], gSs.y * acc[k], gSs.z * acc[k], 0.f));
              acc[k] = 0.f;
            }
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) e[k] = hash_index(s, l, N, i[0] + (k & 1), i[1] + ((k >> 1) & 1), i[2] + (k >> 2));
#pragma unroll
          for (int k = 0; k < 8; ++k) gk[k] = dot(gS, f3(__ldg(s.sigma + lt + e[k])));
          cur[0] = i[0]; cur[1] = i[1]; cur[2] = i[2];
          ++cells;
        }
        corner_weights(f, w);
        float gv = 0.f;
        float3 gp = f3(0, 0, 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc[k] += w[k];
          gv += w[k] * gk[k];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int a = q & 1, b = q >> 1;
          const float fa0 = a ? f[0] : 1 - f[0], fa1 = a ? f[1] : 1 - f[1];
          const float fb1 = b ? f[1] : 1 - f[1], fb2 = b ? f[2] : 1 - f[2];
          gp.x += (gk[1 | (a << 1) | (b << 2)] - gk[(a << 1) | (b << 2)]) * fa1 * fb2;
          gp.y += (gk[a | 2 | (b << 2)] - gk[a | (b << 2)]) * fa0 * fb2;
          gp.z += (gk[a | (b << 1) | 4] - gk[a | (b << 1)]) * fa0 * fb1;
        }
        gp = gp * (float)N;              // d g_l / d u = N_l
        gl += gv;
        gsum += gp;
        gtsum += gp * t;
      }
      if (cur[0] >= 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          atomicAdd(gsig + lt + e[k], make_float4(gSs.x * acc[k], gSs.y * acc[k], gSs.z * acc[k], 0.f));
      }
    }
  } else if (active) {
    const int P = (m.N + G - 1) / G, j0 = (lane_id() % G) * P, j1 = min(j0 + P, m.N);
    int cur = -1;
    float acc[8], gk[8];               // the run's weight sums; gS . sigma_k of its cell
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = gk[k] = 0.f;
    for (int j = j0; j < j1; ++j) {
      const float t = ((float)j + 0.5f) * invN;
      int base;
      float f[3], w[8];
      if (!grid_cell(m, o + dx * t, base, f)) continue;
      if (base != cur) {
        if (cur >= 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            atomicAdd(gsig + cell_node((size_t)cur, k, m.R), make_float4(gSs.x * acc[k], gSs.y * acc[k], gSs.z * acc[k], 0.f));
            acc[k] = 0.f;
          }
        }
        float3 c[8];
        grid_corners(s, m, base, c);
#pragma unroll
        for (int k = 0; k < 8; ++k) gk[k] = dot(gS, c[k]);
        cur = base;
        ++cells;
      }
      corner_weights(f, w);
      float gv = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc[k] += w[k];
        gv += w[k] * gk[k];
      }
      // d/dg of sum_k gk_k w_k: differences over each axis' bit
      float3 gp = f3(0, 0, 0);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int u = p & 1, v = p >> 1;
        const float fu0 = u ? f[0] : 1 - f[0], fu1 = u ? f[1] : 1 - f[1];
        const float fv1 = v ? f[1] : 1 - f[1], fv2 = v ? f[2] : 1 - f[2];
        gp.x += (gk[1 | (u << 1) | (v << 2)] - gk[(u << 1) | (v << 2)]) * fu1 * fv2;
        gp.y += (gk[u | 2 | (v << 2)] - gk[u | (v << 2)]) * fu0 * fv2;
        gp.z += (gk[u | (v << 1) | 4] - gk[u | (v << 1)]) * fu0 * fv1;
      }
      gl += gv;
      gsum += gp;
      gtsum += gp * t;
    }
    if (cur >= 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        atomicAdd(gsig + cell_node((size_t)cur, k, m.R), make_float4(gSs.x * acc[k], gSs.y * acc[k], gSs.z * acc[k], 0.f));
    }
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    gl += __shfl_xor_sync(~0u, gl, off);
    gsum.x += __shfl_xor_sync(~0u, gsum.x, off);
    gsum.y += __shfl_xor_sync(~0u, gsum.y, off);
    gsum.z += __shfl_xor_sync(~0u, gsum.z, off);
    gtsum.x += __shfl_xor_sync(~0u, gtsum.x, off);
    gtsum.y += __shfl_xor_sync(~0u, gtsum.y, off);
    gtsum.z += __shfl_xor_sync(~0u, gtsum.z, off);
  }
  flush_walk_count(s.wcount ? s.wcount + 1 : nullptr, cells);
  // grad_p mu = grad_g mu * scl; quadrature weight sc; x_j = o (1 - t_j) + x t_j
  const float3 k3 = m.scl * sc;
  const float3 gxt = f3(gtsum.x * k3.x, gtsum.y * k3.y, gtsum.z * k3.z);
  gx = gxt;
  go = f3(gsum.x * k3.x, gsum.y * k3.y, gsum.z * k3.z) - gxt;
  if (l > 0.0f) {                      // d l / d(x, o) times sum_j gS . mu(x_j) / N
    const float3 u = dx * (1.0f / l);
    gx += u * (gl * invN);
    go -= u * (gl * invN);
  }
}

// ----------------------------------------------------------------------------- environment
DT_D float grid_coord(float p, float Re, int res, bool& clamped) {
  // (p + Re) / (2 Re) * (res - 1), with the scale factored out (one division per texture,
  // shared by every coordinate once inlined) and branch-free clamping
  const float top = (float)(res - 1);
  const float g = (p + Re) * (top / (2.0f * Re));
  clamped = !(g >= 0.0f && g <= top);
  return fminf(fmaxf(g, 0.0f), top);
}
// The same in float64 for the shell lookup (the lookup point comes from the float64 ray state);
// returns the cell index and the fraction within it (float32: only a weight from here on).
DT_D int grid_cell64(double p, double Re, int res, float& f, bool& clamped) {
  const double top = (double)(res - 1);
  double g = (p + Re) * (top * rcp64(2.0 * Re));
  clamped = !(g >= 0.0 && g <= top);
  g = fmin(fmax(g, 0.0), top);
  const int i = min((int)floor(g), res - 2);
  f = (float)(g - (double)i);
  return i;
}

DT_D double3 shell_point(const DevScene& s, double3 o, double3 dh, double& ts, double& sq) {
  const double Re = (double)s.radius;
  if (s.far_field) { ts = Re; sq = 0.0; return dh * Re; }
  const double b = dot(o, dh);
  sq = sqrt64(b * b - dot(o, o) + Re * Re);
  ts = -b + sq;
  return o + dh * ts;
}

DT_D float3 env_voxel(const DevScene& s, double3 p, float3 a, float3* gp) {
  bool c[3];
  float f[3];
  const int R = s.vres;
  const int i0[3] = {grid_cell64(p.x, s.radius, R, f[0], c[0]), grid_cell64(p.y, s.radius, R, f[1], c[1]),
                     grid_cell64(p.z, s.radius, R, f[2], c[2])};
  float3 out = f3(0, 0, 0), gg = f3(0, 0, 0);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
    float wx = dx ? f[0] : 1 - f[0], wy = dy ? f[1] : 1 - f[1], wz = dz ? f[2] : 1 - f[2];
    DT_CHECK(i0[0] >= 0 && i0[1] >= 0 && i0[2] >= 0 && i0[0] + dx < R && i0[1] + dy < R && i0[2] + dz < R);
    float4 t = __ldg(s.voxel + ((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx));
    out += f3(t) * (wx * wy * wz);
    if (gp) {
      float sd = a.x * t.x + a.y * t.y + a.z * t.z;
      gg += f3((dx ? 1.f : -1.f) * wy * wz, wx * (dy ? 1.f : -1.f) * wz, wx * wy * (dz ? 1.f : -1.f)) * sd;
    }
  }
  if (gp) {
    float sc = (float)(R - 1) / (2.0f * s.radius);
    *gp += f3(c[0] ? 0.f : gg.x * sc, c[1] ? 0.f : gg.y * sc, c[2] ? 0.f : gg.z * sc);
  }
  return out;
}

DT_D float3 env_plane(const DevScene& s, int k, double a_, double b_, float3 adj, float* ga, float* gb) {
  bool ca, cb;
  const int R = s.pres;
  float fa, fb;
  const int ia = grid_cell64(a_, s.radius, R, fa, ca), ib = grid_cell64(b_, s.radius, R, fb, cb);
  const float4* P = s.planes + (size_t)k * R * R;
  DT_CHECK(k >= 0 && k < 3 && ia >= 0 && ib >= 0 && ia + 1 < R && ib + 1 < R);
  float4 t00 = __ldg(P + (size_t)ib * R + ia), t01 = __ldg(P + (size_t)ib * R + ia + 1);
  float4 t10 = __ldg(P + (size_t)(ib + 1) * R + ia), t11 = __ldg(P + (size_t)(ib + 1) * R + ia + 1);
  float3 out = f3(t00) * ((1 - fa) * (1 - fb)) + f3(t01) * (fa * (1 - fb)) + f3(t10) * ((1 - fa) * fb) +
               f3(t11) * (fa * fb);
  if (ga) {
    float s00 = dot(adj, f3(t00)), s01 = dot(adj, f3(t01)), s10 = dot(adj, f3(t10)), s11 = dot(adj, f3(t11));
    float sc = (float)(R - 1) / (2.0f * s.radius);
    float da = (s01 - s00) * (1 - fb) + (s11 - s10) * fb;
    float db = (s10 - s00) * (1 - fa) + (s11 - s01) * fa;
    *ga = ca ? 0.f : da * sc;
    *gb = cb ? 0.f : db * sc;
  }
  return out;
}

// Reverse of the shell point p = o + ts dh (or R_e dh in the far field): adds the adjoints
// of o and dh for gp = dL/dp (ts, sq from shell_point).
DT_D void shell_point_bwd(const DevScene& s, double3 o, double3 dh, double ts, double sq, double3 gp, double3& go,
                          double3& gdh) {
  if (s.far_field) {
    gdh += gp * (double)s.radius;
    return;
  }
  const double b = dot(o, dh);
  go += gp;
  gdh += gp * ts;
  const double gts = dot(gp, dh);
  const double gdisc = sq > 0.0 ? gts * rcp64(2.0 * sq) : 0.0;
  const double gb = -gts + gdisc * 2.0 * b;
  go -= o * (2.0 * gdisc);
  go += dh * gb;
  gdh += o * gb;
}

// ---- volumetric env (env_kind 2, R30): the voxel/plane textures carry colour (rgb) and
// density (w).  env_field: rgb and the raw (unclamped) density at p; env_field_jac: also
// its Jacobian d/dp (both clamp-aware: a clamped grid coordinate passes no gradient).
DT_D float4 env_field(const DevScene& s, float3 p) {
  bool c;
  const float g[3] = {grid_coord(p.x, s.radius, s.vres, c), grid_coord(p.y, s.radius, s.vres, c),
                      grid_coord(p.z, s.radius, s.vres, c)};
  const int R = s.vres;
  int i0[3];
  float f[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) { i0[k] = min((int)floorf(g[k]), R - 2); f[k] = g[k] - (float)i0[k]; }
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
    const float w = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
    const float4 t = __ldg(s.voxel + ((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx));
    out.x += t.x * w; out.y += t.y * w; out.z += t.z * w; out.w += t.w * w;
  }
  const float pa[3] = {p.x, p.x, p.y}, pb[3] = {p.y, p.z, p.z};
  const int Rp = s.pres;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    bool ca, cb;
    const float ga = grid_coord(pa[k], s.radius, Rp, ca), gb = grid_coord(pb[k], s.radius, Rp, cb);
    const int ia = min((int)floorf(ga), Rp - 2), ib = min((int)floorf(gb), Rp - 2);
    const float fa = ga - (float)ia, fb = gb - (float)ib;
    const float4* P = s.planes + (size_t)k * Rp * Rp;
    const float4 t00 = __ldg(P + (size_t)ib * Rp + ia), t01 = __ldg(P + (size_t)ib * Rp + ia + 1);
    const float4 t10 = __ldg(P + (size_t)(ib + 1) * Rp + ia), t11 = __ldg(P + (size_t)(ib + 1) * Rp + ia + 1);
    const float w00 = (1 - fa) * (1 - fb), w01 = fa * (1 - fb), w10 = (1 - fa) * fb, w11 = fa * fb;
    out.x += t00.x * w00 + t01.x * w01 + t10.x * w10 + t11.x * w11;
    out.y += t00.y * w00 + t01.y * w01 + t10.y * w10 + t11.y * w11;
    out.z += t00.z * w00 + t01.z * w01 + t10.z * w10 + t11.z * w11;
    out.w += t00.w * w00 + t01.w * w01 + t10.w * w10 + t11.w * w11;
  }
  return out;
}

// Value (rgb, raw density) and its Jacobian J[c] = d value_c / dp (c = r, g, b, density),
// one pass over the 20 texels.
DT_D float4 env_field_jac(const DevScene& s, float3 p, float3 J[4]) {
  bool c[3];
  const float g[3] = {grid_coord(p.x, s.radius, s.vres, c[0]), grid_coord(p.y, s.radius, s.vres, c[1]),
                      grid_coord(p.z, s.radius, s.vres, c[2])};
  const int R = s.vres;
  int i0[3];
  float f[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) { i0[k] = min((int)floorf(g[k]), R - 2); f[k] = g[k] - (float)i0[k]; }
  float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
  float3 gv[4] = {f3(0, 0, 0), f3(0, 0, 0), f3(0, 0, 0), f3(0, 0, 0)};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
    const float wx = dx ? f[0] : 1 - f[0], wy = dy ? f[1] : 1 - f[1], wz = dz ? f[2] : 1 - f[2];
    const float w = wx * wy * wz;
    const float4 t = __ldg(s.voxel + ((size_t)(i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx));
    out.x += t.x * w; out.y += t.y * w; out.z += t.z * w; out.w += t.w * w;
    const float3 dw = f3((dx ? 1.f : -1.f) * wy * wz, wx * (dy ? 1.f : -1.f) * wz, wx * wy * (dz ? 1.f : -1.f));
    gv[0] += dw * t.x; gv[1] += dw * t.y; gv[2] += dw * t.z; gv[3] += dw * t.w;
  }
  const float sv = (float)(R - 1) / (2.0f * s.radius);
  const float3 msk = f3(c[0] ? 0.f : sv, c[1] ? 0.f : sv, c[2] ? 0.f : sv);
#pragma unroll
  for (int q = 0; q < 4; ++q) J[q] = gv[q] * msk;
  const float pa[3] = {p.x, p.x, p.y}, pb[3] = {p.y, p.z, p.z};
  const int Rp = s.pres;
  const float spl = (float)(Rp - 1) / (2.0f * s.radius);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    bool ca, cb;
    const float ga = grid_coord(pa[k], s.radius, Rp, ca), gb = grid_coord(pb[k], s.radius, Rp, cb);
    const int ia = min((int)floorf(ga), Rp - 2), ib = min((int)floorf(gb), Rp - 2);
    const float fa = ga - (float)ia, fb = gb - (float)ib;
    const float4* P = s.planes + (size_t)k * Rp * Rp;
    const float4 t00 = __ldg(P + (size_t)ib * Rp + ia), t01 = __ldg(P + (size_t)ib * Rp + ia + 1);
    const float4 t10 = __ldg(P + (size_t)(ib + 1) * Rp + ia), t11 = __ldg(P + (size_t)(ib + 1) * Rp + ia + 1);
    const float w00 = (1 - fa) * (1 - fb), w01 = fa * (1 - fb), w10 = (1 - fa) * fb, w11 = fa * fb;
    out.x += t00.x * w00 + t01.x * w01 + t10.x * w10 + t11.x * w11;
    out.y += t00.y * w00 + t01.y * w01 + t10.y * w10 + t11.y * w11;
    out.z += t00.z * w00 + t01.z * w01 + t10.z * w10 + t11.z * w11;
    out.w += t00.w * w00 + t01.w * w01 + t10.w * w10 + t11.w * w11;
    // d/da and d/db of the bilinear value, per channel
    const float ka = ca ? 0.f : spl, kb = cb ? 0.f : spl;
    const float4 da = make_float4(((t01.x - t00.x) * (1 - fb) + (t11.x - t10.x) * fb) * ka,
                                  ((t01.y - t00.y) * (1 - fb) + (t11.y - t10.y) * fb) * ka,
                                  ((t01.z - t00.z) * (1 - fb) + (t11.z - t10.z) * fb) * ka,
                                  ((t01.w - t00.w) * (1 - fb) + (t11.w - t10.w) * fb) * ka);
    const float4 db = make_float4(((t10.x - t00.x) * (1 - fa) + (t11.x - t01.x) * fa) * kb,
                                  ((t10.y - t00.y) * (1 - fa) + (t11.y - t01.y) * fa) * kb,
                                  ((t10.z - t00.z) * (1 - fa) + (t11.z - t01.z) * fa) * kb,
                                  ((t10.w - t00.w) * (1 - fa) + (t11.w - t01.w) * fa) * kb);
    const float dav[4] = {da.x, da.y, da.z, da.w}, dbv[4] = {db.x, db.y, db.z, db.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (k == 0) { J[q].x += dav[q]; J[q].y += dbv[q]; }
      else if (k == 1) { J[q].x += dav[q]; J[q].z += dbv[q]; }
      else { J[q].y += dav[q]; J[q].z += dbv[q]; }
    }
  }
  return out;
}

// Emission-absorption quadrature along an exterior segment o -> x (R30, M midpoint samples):
// V = sum_i T_i (1 - exp(-sigma_i Delta)) c_i, T_i = exp(-Delta sum_{j<i} sigma_j), Tn = T_M.
// mom (optional): the adjoint-independent sums the reverse needs, so it makes one pass:
//   Qc = sum_{0<i<M} (c_i - c_{i-1}) T_i - c_{M-1} T_M,
//   Go = -sum_{0<i<M} (c_i - c_{i-1}) T_i od_i + c_{M-1} T_M od_M,  od_i = Delta sum_{j<i} sigma_j.
struct VolMom {
  float3 Qc, Go;
  float odM;
};

DT_D void env_volume(const DevScene& s, float3 o, float3 x, float3& V, float& Tn, VolMom* mom = nullptr) {
  const int M = s.env_nsamp;
  const float3 dx = x - o;
  const float delta = length(dx) / (float)M;
  float od = 0.f;
  float3 cprev = f3(0, 0, 0), Qc = f3(0, 0, 0), Go = f3(0, 0, 0);
  V = f3(0, 0, 0);
#pragma unroll 2
  for (int i = 0; i < M; ++i) {
    const float4 f = env_field(s, o + dx * (((float)i + 0.5f) / (float)M));
    const float3 c = f3(f);
    const float sg = fmaxf(f.w, 0.f), Ti = expf(-od);
    V += c * (Ti * (1.f - expf(-sg * delta)));
    if (i > 0) {
      Qc += (c - cprev) * Ti;
      Go -= (c - cprev) * (Ti * od);
    }
    od += sg * delta;
    cprev = c;
  }
  Tn = expf(-od);
  if (mom) {
    mom->Qc = Qc - cprev * Tn;
    mom->Go = Go + cprev * (Tn * od);
    mom->odM = od;
  }
}

// Reverse of env_volume given aV = dL/dV and aT = dL/dTn: adds the end-point adjoints to go,
// gx.  With s_i = aV . c_i, dL/dT_i = s_i - s_{i-1} (0 < i < M), dL/dT_M = aT - s_{M-1}:
// dL/dsigma_j = -Delta (Q - sum_{0<i<=j} dL/dT_i T_i), Q = sum_{i=1..M} dL/dT_i T_i
// = aV . Qc + aT Tn, and Delta dL/dDelta = aV . Go - aT Tn od_M (the forward's moments), so
// one pass over the samples remains.
DT_D void env_volume_bwd(const DevScene& s, float3 o, float3 x, float3 aV, float aT, float Tn, const VolMom& mom,
                         float3& go, float3& gx) {
  const int M = s.env_nsamp;
  const float3 dx = x - o;
  const float l = length(dx), delta = l / (float)M;
  const float Q = dot(aV, mom.Qc) + aT * Tn;
  float P = 0.f, pre = 0.f, sprev = 0.f;
#pragma unroll 2
  for (int j = 0; j < M; ++j) {
    const float t = ((float)j + 0.5f) / (float)M;
    const float3 p = o + dx * t;
    float3 J[4];
    const float4 f = env_field_jac(s, p, J);
    const float sj = dot(aV, f3(f)), sg = fmaxf(f.w, 0.f);
    const float Tj = expf(-delta * pre), Tj1 = expf(-delta * (pre + sg));
    if (j > 0) P += (sj - sprev) * Tj;
    const float gsg = f.w > 0.f ? -delta * (Q - P) : 0.f;
    const float3 ac = aV * (Tj - Tj1);
    const float3 gp = J[0] * ac.x + J[1] * ac.y + J[2] * ac.z + J[3] * gsg;
    go += gp * (1.f - t);
    gx += gp * t;
    pre += sg;
    sprev = sj;
  }
  if (l > 0.f) {
    const float3 u = dx * (1.0f / l);
    const float gl = (dot(aV, mom.Go) - aT * Tn * mom.odM) / l;   // dL/dDelta / M
    gx += u * gl;
    go -= u * gl;
  }
}

// Radiance of an escaping ray: the shell lookup (R14), preceded by the volume rendering of
// the segment out to the shell for the volumetric env (R30; its samples in float32).  Forward:
// Tn and mom (if given) returned for the record.  Reverse (go/gd non-null, SET): uses the
// recorded Tn, mom.
DT_D float3 env_eval(const DevScene& s, double3 o, double3 d, float3 a, float3* go, float3* gd);
template <bool VOL>
DT_D float3 env_escape(const DevScene& s, double3 o, double3 d, float3 a, float3* go, float3* gd,
                       float* Tn_io = nullptr, VolMom* mom_io = nullptr) {
  if (!VOL) return env_eval(s, o, d, a, go, gd);
  const double rn = rsqrt64(dot(d, d));
  const double3 dh = d * rn;
  double ts, sq;
  const double3 ps = shell_point(s, o, dh, ts, sq);
  if (!go) {                                   // forward
    float3 V;
    float Tn;
    env_volume(s, f3(o), f3(ps), V, Tn, mom_io);
    if (Tn_io) *Tn_io = Tn;
    return V + env_eval(s, o, d, a, nullptr, nullptr) * Tn;
  }
  const float Tn = *Tn_io;                     // reverse, from the record
  const float3 E = env_eval(s, o, d, a * Tn, go, gd);
  float3 gov = f3(0, 0, 0), gps = f3(0, 0, 0);
  env_volume_bwd(s, f3(o), f3(ps), a, dot(a, E), Tn, *mom_io, gov, gps);
  double3 gdh = d3(0, 0, 0), go2 = d3(gov);
  shell_point_bwd(s, o, dh, ts, sq, d3(gps), go2, gdh);
  *go += f3(go2);
  *gd += f3((gdh - dh * dot(dh, gdh)) * rn);
  return E;
}

// Env(o, d) (P:160 step 3), the lookup point from the float64 ray.  If go/gd are non-null,
// they are SET to the reverse for adjoint a.
DT_D float3 env_eval(const DevScene& s, double3 o, double3 d, float3 a, float3* go, float3* gd) {
  const double rn = rsqrt64(dot(d, d));
  const double3 dh = d * rn;
  float3 L;
  double3 gdh = d3(0, 0, 0);
  if (s.env_kind == 0) {
    L = s.ambient;
    for (int j = 0; j < s.nlobes; ++j) {
      const float* lb = s.lobes + 7 * j;
      const double3 mu = d3(__ldg(lb), __ldg(lb + 1), __ldg(lb + 2));
      const float kap = __ldg(lb + 3);
      const float3 w = f3(__ldg(lb + 4), __ldg(lb + 5), __ldg(lb + 6));
      const float e = expf((float)((double)kap * (dot(mu, dh) - 1.0)));
      L += w * e;
      if (gd) gdh += mu * (double)(dot(a, w) * e * kap);
    }
    if (go) *go = f3(0, 0, 0);
  } else {
    double ts, sq;
    const double3 p = shell_point(s, o, dh, ts, sq);
    float3 gp = f3(0, 0, 0);
    L = env_voxel(s, p, a, gd ? &gp : nullptr);
    float g1 = 0, g2 = 0;
    L += env_plane(s, 0, p.x, p.y, a, gd ? &g1 : nullptr, &g2);
    if (gd) { gp.x += g1; gp.y += g2; }
    L += env_plane(s, 1, p.x, p.z, a, gd ? &g1 : nullptr, &g2);
    if (gd) { gp.x += g1; gp.z += g2; }
    L += env_plane(s, 2, p.y, p.z, a, gd ? &g1 : nullptr, &g2);
    if (gd) { gp.y += g1; gp.z += g2; }
    if (gd) {
      double3 g_o = d3(0, 0, 0);
      shell_point_bwd(s, o, dh, ts, sq, d3(gp), g_o, gdh);
      *go = f3(g_o);
    }
  }
  if (gd) *gd = f3((gdh - dh * dot(dh, gdh)) * rn);
  return L;
}

}  // namespace dt
