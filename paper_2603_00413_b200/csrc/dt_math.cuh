// float3 helpers for the sm_100a kernels.  Plain SIMT arithmetic: nothing on this path
// is a dense contraction, so no tensor-core code appears anywhere in libdifftrans.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DT_HD __host__ __device__ __forceinline__
#define DT_D __device__ __forceinline__

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
