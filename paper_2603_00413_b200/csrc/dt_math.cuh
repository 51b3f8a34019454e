// float3 helpers for the sm_100a kernels.  Plain SIMT arithmetic: nothing on this path
// is a dense contraction, so no tensor-core code appears anywhere in libdifftrans.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DT_HD __host__ __device__ __forceinline__
#define DT_D __device__ __forceinline__

// Bounds-checked build (-DDT_CHECKED=1, tools/checked_build.sh): DT_CHECK(c) records the
// source line of the first failed check in a per-translation-unit device word, read back by
// dt_check_status() (compute-sanitizer is not available on the GPU pool, so the index
// arithmetic of every kernel family is checked by the kernels themselves).  In the product
// build it compiles to nothing.
#ifndef DT_CHECKED
#define DT_CHECKED 0
#endif
#if DT_CHECKED
namespace dt {
namespace {
__device__ int g_dt_check_line;
}
}  // namespace dt
#define DT_CHECK(c)                                                   \
  do {                                                                \
    if (!(c)) atomicCAS(&::dt::g_dt_check_line, 0, __LINE__);        \
  } while (0)
// host: first failed line of this translation unit (0: none); clears it
#define DT_DEFINE_CHECK_READER(name)                                  \
  int name() {                                                        \
    int v = 0, z = 0;                                                 \
    cudaMemcpyFromSymbol(&v, ::dt::g_dt_check_line, sizeof(int));     \
    cudaMemcpyToSymbol(::dt::g_dt_check_line, &z, sizeof(int));       \
    return v;                                                         \
  }
#else
#define DT_CHECK(c) \
  do {              \
  } while (0)
#define DT_DEFINE_CHECK_READER(name) \
  int name() { return -1; }
#endif

DT_HD float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
DT_HD float3 f3(float4 a) { return make_float3(a.x, a.y, a.z); }
DT_HD float4 f4(float3 a, float w) { return make_float4(a.x, a.y, a.z, w); }
DT_HD float3 operator+(float3 a, float3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
DT_HD float3 operator-(float3 a, float3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
DT_HD float3 operator-(float3 a) { return f3(-a.x, -a.y, -a.z); }
DT_HD float3 operator*(float3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
DT_HD float3 operator*(float s, float3 a) { return f3(a.x * s, a.y * s, a.z * s); }
DT_HD float3 operator*(float3 a, float3 b) { return f3(a.x * b.x, a.y * b.y, a.z * b.z); }
DT_HD float3& operator+=(float3& a, float3 b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
DT_HD float3& operator-=(float3& a, float3 b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
DT_HD float dot(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
DT_HD float3 cross(float3 a, float3 b) { return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
DT_HD float length(float3 a) { return sqrtf(dot(a, a)); }
DT_HD float3 fminf3(float3 a, float3 b) { return f3(fminf(a.x, b.x), fminf(a.y, b.y), fminf(a.z, b.z)); }
DT_HD float3 fmaxf3(float3 a, float3 b) { return f3(fmaxf(a.x, b.x), fmaxf(a.y, b.y), fmaxf(a.z, b.z)); }
DT_HD float comp(float3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// splitmix64 finaliser (path signatures; implemented independently of the oracle).
DT_HD uint64_t dt_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ordered-int encoding so float min/max can use integer atomics
DT_D int f2ord(float f) { int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7fffffff; }
DT_D float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

DT_D unsigned lanemask_lt() { unsigned m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
DT_D int lane_id() { return threadIdx.x & 31; }
DT_D float3 shfl3(float3 v, int src) {
  return f3(__shfl_sync(~0u, v.x, src), __shfl_sync(~0u, v.y, src), __shfl_sync(~0u, v.z, src));
}

// ----------------------------------------------------------------------------- float64 geometry
// The geometric state of a segment (origin, direction, hit point, normals, the interface
// directions) is carried in float64 end to end (DESIGN.md §4/§5): float32 rounding of that
// state is amplified by every later bounce.  Radiance, throughput and adjoints stay float32.
DT_HD double3 d3(double x, double y, double z) { return make_double3(x, y, z); }
DT_HD double3 d3(float3 a) { return make_double3(a.x, a.y, a.z); }
DT_HD double3 d3(float4 a) { return make_double3(a.x, a.y, a.z); }
DT_HD float3 f3(double3 a) { return f3((float)a.x, (float)a.y, (float)a.z); }
DT_HD double3 operator+(double3 a, double3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
DT_HD double3 operator-(double3 a, double3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
DT_HD double3 operator-(double3 a) { return d3(-a.x, -a.y, -a.z); }
DT_HD double3 operator*(double3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
DT_HD double3 operator*(double s, double3 a) { return d3(a.x * s, a.y * s, a.z * s); }
DT_HD double3& operator+=(double3& a, double3 b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
DT_HD double3& operator-=(double3& a, double3 b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
DT_HD double dot(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
DT_HD double3 cross(double3 a, double3 b) {
  return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
// Reciprocal and square root without the IEEE slow-path calls: the MUFU double-precision
// seeds (~2^-22) refined by two Newton steps (~1 ulp), inline.
DT_D double rcp64(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}
DT_D double rsqrt64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
DT_D double sqrt64(double x) { return x > 0.0 ? x * rsqrt64(x) : 0.0; }
DT_D double length(double3 a) { return sqrt64(dot(a, a)); }

// 32-B records of float64 xyz + two 32-bit tags (ray origin | ray index, direction | tree
// position, vertex / face normals | |sum|), moved with one 256-bit access.
struct __align__(32) Vec64 {
  double x, y, z;
  int i;
  unsigned u;
};
DT_HD double3 xyz(const Vec64& v) { return d3(v.x, v.y, v.z); }
DT_D Vec64 mk64(double3 a, int i, unsigned u) { Vec64 v; v.x = a.x; v.y = a.y; v.z = a.z; v.i = i; v.u = u; return v; }
// streaming (evict-first) 256-bit load / store: LDG.E.EF.ENL2.256 / STG.E.EF.ENL2.256
DT_D Vec64 ldcs64(const Vec64* p) {
  double x, y, z, w;
  asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x), "=d"(y), "=d"(z), "=d"(w) : "l"(p));
  Vec64 v;
  v.x = x; v.y = y; v.z = z;
  const long long b = __double_as_longlong(w);
  v.i = (int)(b & 0xffffffffll);
  v.u = (unsigned)((unsigned long long)b >> 32);
  return v;
}
DT_D void stcs64(Vec64* p, const Vec64& v) {
  const double w = __longlong_as_double((long long)(((unsigned long long)v.u << 32) | (unsigned)v.i));
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(w) : "memory");
}
// read-only (L1-cached) 256-bit load of a table entry (vertex / face normals)
DT_D Vec64 ldg64(const Vec64* p) {
  double x, y, z, w;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x), "=d"(y), "=d"(z), "=d"(w) : "l"(p));
  Vec64 v;
  v.x = x; v.y = y; v.z = z;
  const long long b = __double_as_longlong(w);
  v.i = (int)(b & 0xffffffffll);
  v.u = (unsigned)((unsigned long long)b >> 32);
  return v;
}
// float64 xyz + w (vertex normal | |sum of unit face normals|; face normal | |e1 x e2|)
struct __align__(32) D4 {
  double x, y, z, w;
};
DT_HD double3 xyz(const D4& v) { return d3(v.x, v.y, v.z); }
DT_D D4 ldg_d4(const D4* p) {
  D4 v;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
