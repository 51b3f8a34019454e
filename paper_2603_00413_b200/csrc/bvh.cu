// Per-step mesh snapshot, vertex normals and LBVH rebuild (K1-K7).
//
//   snapshot + bounds  ->  face normals  ->  corner sort (vertex CSR)  ->  vertex normals
//   ->  Morton codes  ->  LSD radix sort (8-bit digits, stable)  ->  Karras 2012 hierarchy
//   ->  bottom-up AABB refit (atomic arrival flags)  ->  pack 64-B nodes / 48-B triangles
//
// The paper builds its acceleration structure inside OptiX; B200 has no RT cores,
// so the tree is rebuilt in O(N_f) device passes every step (the mesh moves every step).
#include <cuda_runtime.h>

#include <algorithm>

#include "dt_internal.h"

namespace dt {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;

// ----------------------------------------------------------------------------- bounds
__global__ void k_snapshot(const float* __restrict__ Vin, int nv, float4* __restrict__ V, int* __restrict__ ibox) {
  float3 lo = f3(kInf, kInf, kInf), hi = -lo;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    float3 p = f3(Vin[3 * i], Vin[3 * i + 1], Vin[3 * i + 2]);
    V[i] = f4(p, 0.0f);
    lo = fminf3(lo, p);
    hi = fmaxf3(hi, p);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf3(lo, f3(__shfl_xor_sync(~0u, lo.x, o), __shfl_xor_sync(~0u, lo.y, o), __shfl_xor_sync(~0u, lo.z, o)));
    hi = fmaxf3(hi, f3(__shfl_xor_sync(~0u, hi.x, o), __shfl_xor_sync(~0u, hi.y, o), __shfl_xor_sync(~0u, hi.z, o)));
  }
  if (lane_id() == 0) {
    atomicMin(ibox + 0, f2ord(lo.x)); atomicMin(ibox + 1, f2ord(lo.y)); atomicMin(ibox + 2, f2ord(lo.z));
    atomicMax(ibox + 3, f2ord(hi.x)); atomicMax(ibox + 4, f2ord(hi.y)); atomicMax(ibox + 5, f2ord(hi.z));
  }
}

// unit face normals (float64, the shading normals' inputs) and centroid bounds (Morton
// quantisation)
__global__ void k_faces(const float4* __restrict__ V, const int* __restrict__ F, int nf, D4* __restrict__ fn,
                        int* __restrict__ ibox) {
  float3 lo = f3(kInf, kInf, kInf), hi = -lo;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
    float3 a = f3(V[F[3 * f]]), b = f3(V[F[3 * f + 1]]), c = f3(V[F[3 * f + 2]]);
    const double3 a64 = d3(a);
    const double3 n = cross(d3(b) - a64, d3(c) - a64);
    const double L = length(n);
    D4 o = {0.0, 0.0, 0.0, 0.0};                                         // zero-area faces add 0 (R6)
    if (L > 0.0) o = D4{n.x / L, n.y / L, n.z / L, L};
    fn[f] = o;
    float3 cen = (a + b + c) * (1.0f / 3.0f);
    lo = fminf3(lo, cen);
    hi = fmaxf3(hi, cen);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf3(lo, f3(__shfl_xor_sync(~0u, lo.x, o), __shfl_xor_sync(~0u, lo.y, o), __shfl_xor_sync(~0u, lo.z, o)));
    hi = fmaxf3(hi, f3(__shfl_xor_sync(~0u, hi.x, o), __shfl_xor_sync(~0u, hi.y, o), __shfl_xor_sync(~0u, hi.z, o)));
  }
  if (lane_id() == 0) {
    atomicMin(ibox + 6, f2ord(lo.x)); atomicMin(ibox + 7, f2ord(lo.y)); atomicMin(ibox + 8, f2ord(lo.z));
    atomicMax(ibox + 9, f2ord(hi.x)); atomicMax(ibox + 10, f2ord(hi.y)); atomicMax(ibox + 11, f2ord(hi.z));
  }
}

__global__ void k_corner_keys(const int* __restrict__ F, int n3, unsigned* __restrict__ keys, unsigned* __restrict__ vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += gridDim.x * blockDim.x) {
    keys[i] = (unsigned)F[i];
    vals[i] = (unsigned)i;      // corner id = 3 * face + k, ascending -> stable order by face
  }
}

__global__ void k_csr(const unsigned* __restrict__ keys, int n3, int nv, int* __restrict__ vstart) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n3; i += gridDim.x * blockDim.x) {
    int cur = i < n3 ? (int)keys[i] : nv;
    int prev = i > 0 ? (int)keys[i - 1] : -1;
    for (int v = prev + 1; v <= cur; ++v) vstart[v] = i;   // empty ranges for isolated vertices
  }
}

// n_v = normalize(sum of incident unit face normals) (R6), float64, gathered in face
// order (deterministic)
__global__ void k_vertex_normals(const int* __restrict__ vstart, const unsigned* __restrict__ corner,
                                 const D4* __restrict__ fn, int nv, D4* __restrict__ nrm) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double3 s = d3(0, 0, 0);
    for (int j = vstart[v]; j < vstart[v + 1]; ++j) s += xyz(fn[corner[j] / 3]);
    const double L = length(s);
    nrm[v] = L > 0.0 ? D4{s.x / L, s.y / L, s.z / L, L} : D4{0.0, 0.0, 1.0, 0.0};
  }
}

DT_D unsigned expand10(unsigned x) {
  x &= 0x3ff;
  x = (x | (x << 16)) & 0x030000ff;
  x = (x | (x << 8)) & 0x0300f00f;
  x = (x | (x << 4)) & 0x030c30c3;
  x = (x | (x << 2)) & 0x09249249;
  return x;
}

__global__ void k_morton(const float4* __restrict__ V, const int* __restrict__ F, int nf, const int* __restrict__ ibox,
                         unsigned* __restrict__ keys, unsigned* __restrict__ vals) {
  float3 lo = f3(ord2f(ibox[6]), ord2f(ibox[7]), ord2f(ibox[8]));
  float3 hi = f3(ord2f(ibox[9]), ord2f(ibox[10]), ord2f(ibox[11]));
  float3 ext = hi - lo;
  float3 sc = f3(ext.x > 0 ? 1023.0f / ext.x : 0.0f, ext.y > 0 ? 1023.0f / ext.y : 0.0f, ext.z > 0 ? 1023.0f / ext.z : 0.0f);
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
    float3 cen = (f3(V[F[3 * f]]) + f3(V[F[3 * f + 1]]) + f3(V[F[3 * f + 2]])) * (1.0f / 3.0f);
    float3 q = (cen - lo) * sc;
    unsigned x = (unsigned)fminf(fmaxf(q.x, 0.0f), 1023.0f), y = (unsigned)fminf(fmaxf(q.y, 0.0f), 1023.0f),
             z = (unsigned)fminf(fmaxf(q.z, 0.0f), 1023.0f);
    keys[f] = (expand10(x) << 2) | (expand10(y) << 1) | expand10(z);
    vals[f] = (unsigned)f;
  }
}

// ----------------------------------------------------------------------------- radix sort
// Stable LSD radix sort of (key, value) pairs, 8-bit digits: per-tile digit histograms,
// one exclusive scan (digit-major), then a stable scatter that ranks keys inside each
// 256-key chunk with __match_any_sync.
__global__ void k_hist(const unsigned* __restrict__ keys, int n, int shift, unsigned* __restrict__ hist) {
  __shared__ unsigned sh[256];
  sh[threadIdx.x] = 0;
  __syncthreads();
  int base = blockIdx.x * kSortTile;
  for (int i = 0; i < kSortItems; ++i) {
    int idx = base + i * kSortThreads + threadIdx.x;
    if (idx < n) atomicAdd(&sh[(keys[idx] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * gridDim.x + blockIdx.x] = sh[threadIdx.x];
}

__global__ void k_scan(unsigned* __restrict__ h, int len) {
  __shared__ unsigned part[1024];
  int per = (len + blockDim.x - 1) / blockDim.x;
  int b = threadIdx.x * per, e = min(b + per, len);
  unsigned s = 0;
  for (int i = b; i < e; ++i) s += h[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < blockDim.x; o <<= 1) {
    unsigned v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  unsigned run = part[threadIdx.x] - s;
  for (int i = b; i < e; ++i) { unsigned x = h[i]; h[i] = run; run += x; }
}

// Multi-block exclusive scan (replaces the single-block k_scan on the build's long arrays):
// per-chunk scan with the chunk totals in part[], a scan of part[], then the chunk offsets added.
constexpr int kScanThreads = 256, kScanItems = 8, kScanChunk = kScanThreads * kScanItems;

__global__ void k_scan_chunks(unsigned* __restrict__ h, int len, unsigned* __restrict__ part) {
  __shared__ unsigned sv[kScanChunk];
  __shared__ unsigned wsum[kScanThreads / 32];
  const int base = blockIdx.x * kScanChunk, t = threadIdx.x;
  for (int i = 0; i < kScanItems; ++i) {                 // coalesced load
    const int idx = base + i * kScanThreads + t;
    sv[i * kScanThreads + t] = idx < len ? h[idx] : 0u;
  }
  __syncthreads();
  unsigned loc[kScanItems], s = 0;
  for (int i = 0; i < kScanItems; ++i) { loc[i] = s; s += sv[t * kScanItems + i]; }
  unsigned inc = s;                                      // warp-inclusive scan of thread sums
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(~0u, inc, o);
    if ((t & 31) >= o) inc += y;
  }
  if ((t & 31) == 31) wsum[t >> 5] = inc;
  __syncthreads();
  if (t < 32) {
    unsigned w = t < kScanThreads / 32 ? wsum[t] : 0u, wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(~0u, wi, o);
      if (t >= o) wi += y;
    }
    if (t < kScanThreads / 32) wsum[t] = wi - w;         // exclusive warp offsets
    if (t == kScanThreads / 32 - 1) part[blockIdx.x] = wi;
  }
  __syncthreads();
  const unsigned off = wsum[t >> 5] + inc - s;
  for (int i = 0; i < kScanItems; ++i) sv[t * kScanItems + i] = off + loc[i];
  __syncthreads();
  for (int i = 0; i < kScanItems; ++i) {
    const int idx = base + i * kScanThreads + t;
    if (idx < len) h[idx] = sv[i * kScanThreads + t];
  }
}

__global__ void k_scan_add(unsigned* __restrict__ h, int len, const unsigned* __restrict__ part) {
  const int base = blockIdx.x * kScanChunk;
  const unsigned off = part[blockIdx.x];
  for (int i = threadIdx.x; i < kScanChunk; i += blockDim.x)
    if (base + i < len) h[base + i] += off;
}

// exclusive scan of h[0..len) in place; part: >= ceil(len / kScanChunk) scratch entries
cudaError_t scan_exclusive(unsigned* h, int len, unsigned* part, cudaStream_t st, int* nl) {
  const int nb = (len + kScanChunk - 1) / kScanChunk;
  if (nb <= 1) {
    k_scan<<<1, 1024, 0, st>>>(h, len);
    *nl += 1;
    return cudaGetLastError();
  }
  k_scan_chunks<<<nb, kScanThreads, 0, st>>>(h, len, part);
  k_scan<<<1, 1024, 0, st>>>(part, nb);
  k_scan_add<<<nb, kScanThreads, 0, st>>>(h, len, part);
  *nl += 3;
  return cudaGetLastError();
}

__global__ void k_scatter(const unsigned* __restrict__ kin, const unsigned* __restrict__ vin, unsigned* __restrict__ kout,
                          unsigned* __restrict__ vout, int n, int shift, const unsigned* __restrict__ hist) {
  __shared__ unsigned offs[256];
  __shared__ unsigned total[256];
  __shared__ unsigned wcnt[kSortThreads / 32][256];
  int warp = threadIdx.x >> 5;
  offs[threadIdx.x] = hist[threadIdx.x * gridDim.x + blockIdx.x];
  int base = blockIdx.x * kSortTile;
  for (int c = 0; c < kSortItems; ++c) {
    int idx = base + c * kSortThreads + threadIdx.x;
    bool valid = idx < n;
    unsigned k = valid ? kin[idx] : 0u, v = valid ? vin[idx] : 0u;
    unsigned dg = valid ? (k >> shift) & 255u : 256u;
    for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    unsigned peers = __match_any_sync(~0u, dg);
    unsigned rank = __popc(peers & lanemask_lt());
    if (valid && rank == (unsigned)__popc(peers) - 1) wcnt[warp][dg] = __popc(peers);
    __syncthreads();
    {
      unsigned run = 0;
      for (int w = 0; w < kSortThreads / 32; ++w) { unsigned x = wcnt[w][threadIdx.x]; wcnt[w][threadIdx.x] = run; run += x; }
      total[threadIdx.x] = run;
    }
    __syncthreads();
    if (valid) {
      unsigned pos = offs[dg] + wcnt[warp][dg] + rank;
      DT_CHECK(pos < (unsigned)n);
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    offs[threadIdx.x] += total[threadIdx.x];
    __syncthreads();
  }
}

cudaError_t radix_sort(unsigned* keys, unsigned* vals, unsigned* tk, unsigned* tv, int n, int bits, unsigned* hist,
                       unsigned* part, cudaStream_t st, bool& result_in_tmp, int* nl) {
  int nb = (n + kSortTile - 1) / kSortTile;
  result_in_tmp = false;
  unsigned *ki = keys, *vi = vals, *ko = tk, *vo = tv;
  for (int shift = 0; shift < bits; shift += 8) {
    k_hist<<<nb, kSortThreads, 0, st>>>(ki, n, shift, hist);
    scan_exclusive(hist, 256 * nb, part, st, nl);
    k_scatter<<<nb, kSortThreads, 0, st>>>(ki, vi, ko, vo, n, shift, hist);
    *nl += 2;
    std::swap(ki, ko);
    std::swap(vi, vo);
    result_in_tmp = !result_in_tmp;
  }
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- Karras 2012
DT_D int delta(const unsigned* __restrict__ k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  unsigned a = k[i], b = k[j];
  return a == b ? 32 + __clz(i ^ j) : __clz(a ^ b);   // index tie-break for equal codes
}

__global__ void k_karras(const unsigned* __restrict__ k, int n, int2* __restrict__ children, int* __restrict__ parent_int,
                         int* __restrict__ parent_leaf, int2* __restrict__ ranges) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
    int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(k, n, i, i - d);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
      if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = delta(k, n, i, j);
    int s = 0, t = l;
    while (true) {
      t = (t + 1) >> 1;
      if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
      if (t <= 1) break;
    }
    int gamma = i + s * d + min(d, 0);
    DT_CHECK(gamma >= 0 && gamma + 1 < n && min(i, j) >= 0 && max(i, j) < n);
    int left = min(i, j) == gamma ? ~gamma : gamma;
    int right = max(i, j) == gamma + 1 ? ~(gamma + 1) : gamma + 1;
    children[i] = make_int2(left, right);
    ranges[i] = make_int2(min(i, j), max(i, j));            // leaves covered by node i
    if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
    if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
    if (i == 0) parent_int[0] = -1;
  }
}

DT_D void load_box(const float4* __restrict__ leafbox, const float4* __restrict__ nodebox, int ref, float3& lo, float3& hi) {
  const float4* p = ref < 0 ? leafbox + 2 * (size_t)(~ref) : nodebox + 2 * (size_t)ref;
  float4 a = __ldcg(p), b = __ldcg(p + 1);
  lo = f3(a);
  hi = f3(b);
}

__global__ void k_refit(const float4* __restrict__ V, const int* __restrict__ F, const unsigned* __restrict__ order, int n,
                        const int2* __restrict__ children, const int* __restrict__ parent_int,
                        const int* __restrict__ parent_leaf, int* __restrict__ flags, float4* __restrict__ leafbox,
                        float4* __restrict__ nodebox) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int f = (int)order[j];
    float3 a = f3(V[F[3 * f]]), b = f3(V[F[3 * f + 1]]), c = f3(V[F[3 * f + 2]]);
    float3 lo = fminf3(a, fminf3(b, c)), hi = fmaxf3(a, fmaxf3(b, c));
    __stcg(leafbox + 2 * (size_t)j, f4(lo, 0.f));
    __stcg(leafbox + 2 * (size_t)j + 1, f4(hi, 0.f));
    if (n == 1) continue;
    int p = parent_leaf[j];
    while (p >= 0) {
      __threadfence();
      DT_CHECK(p < n - 1);
      if (atomicAdd(flags + p, 1) == 0) break;   // first arrival: the sibling finishes the node
      __threadfence();                           // acquire: the sibling's box stores, fenced before its atomic
      int2 ch = children[p];
      float3 l0, h0, l1, h1;
      load_box(leafbox, nodebox, ch.x, l0, h0);
      load_box(leafbox, nodebox, ch.y, l1, h1);
      lo = fminf3(l0, l1);
      hi = fmaxf3(h0, h1);
      __stcg(nodebox + 2 * (size_t)p, f4(lo, 0.f));
      __stcg(nodebox + 2 * (size_t)p + 1, f4(hi, 0.f));
      p = parent_int[p];
    }
  }
}

// ----------------------------------------------------------------------------- treelets
// Treelet restructuring (Karras & Aila 2013) improves the Karras hierarchy before the collapse
// (dt_set_bvh_quality: passes, default 2).  Bottom up (atomic-flag climb, like the refit),
// every node with >= N triangles below becomes the root of a treelet: its two children, then
// repeatedly the treelet leaf of largest box area replaced by its own two children, until N = 5
// treelet leaves (4 internal nodes).  A dynamic program over the 31 subsets of the leaves finds
// the binary topology of least SAH cost, C(S) = A(S) c_i + min_{P u Q = S} C(P) + C(Q) (leaves:
// their subtree costs), and the treelet's internal nodes are rewired to it when it is cheaper.
// The leaf boxes and every ancestor's box are unchanged; the triangle order (leaf indices) too.
// After a pass, ranges[n] holds (0, count - 1): only the triangle count of a subtree stays
// meaningful (the collapse uses it for leaf_max = 1 only).  r02 sweep (C3, ms/step): N = 4 /
// 5 / 6 at 2 passes: 78.6 / 78.5 / 79.7 (6 costs 1.5 ms per pass); 5 at 1 / 2 / 3 passes: 78.9 /
// 78.5 / 78.7; none 81.1.  Node visits -6.6% at N = 5, 2 passes.
#ifndef DT_TREELET_N
#define DT_TREELET_N 5                 // treelet leaves (DP over 2^N - 1 subsets)
#endif
#ifndef DT_TREELET_CI
#define DT_TREELET_CI 1.2f
#endif
constexpr float kTreeletCi = DT_TREELET_CI, kTreeletCt = 1.0f;

DT_D float box_area3(float3 lo, float3 hi) {
  const float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
  return dx * dy + dy * dz + dz * dx;
}

#ifndef DT_TREELET_MINB
#define DT_TREELET_MINB 3
#endif
__global__ void __launch_bounds__(256, DT_TREELET_MINB) k_treelet(int2* children, int* parent_int, int* parent_leaf, int* flags, float4* nodebox,
                          const float4* __restrict__ leafbox, float* cost, int2* ranges, float* narea, int n) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int p = parent_leaf[j];
    while (p >= 0) {
      __threadfence();
      if (atomicAdd(flags + p, 1) == 0) break;   // the second arrival processes p
      __threadfence();
      const int2 ch = __ldcg(children + p);
      auto cnt_of = [&](int r) { if (r < 0) return 1; const int2 g = __ldcg(ranges + r); return g.y - g.x + 1; };
      auto cost_of = [&](int r) {
        if (r < 0) { float3 lo, hi; load_box(leafbox, nodebox, r, lo, hi); return box_area3(lo, hi) * kTreeletCt; }
        return __ldcg(cost + r);
      };
      const int cnt = cnt_of(ch.x) + cnt_of(ch.y);
      float3 plo, phi;
      load_box(leafbox, nodebox, p, plo, phi);
      const float ap = box_area3(plo, phi);
      float cp = ap * kTreeletCi + cost_of(ch.x) + cost_of(ch.y);
      if (cnt >= DT_TREELET_N) {
        int L[DT_TREELET_N], I[DT_TREELET_N - 1], nl = 2, ni = 1;
        L[0] = ch.x; L[1] = ch.y; I[0] = p;
        while (nl < DT_TREELET_N) {                       // grow: open the treelet leaf of largest area
          int bi = -1;
          float ba = -1.f;
          for (int i = 0; i < nl; ++i) {
            if (L[i] < 0) continue;
            const float ar = __ldcg(narea + L[i]);    // processed below p: its area is recorded
            if (ar > ba) { ba = ar; bi = i; }
          }
          if (bi < 0) break;
          const int x = L[bi];
          const int2 cx = __ldcg(children + x);
          I[ni++] = x;
          L[bi] = cx.x;
          L[nl++] = cx.y;
        }
        float3 lo[DT_TREELET_N], hi[DT_TREELET_N];
        float cl[DT_TREELET_N];
        int cn[DT_TREELET_N];
        for (int i = 0; i < nl; ++i) {
          load_box(leafbox, nodebox, L[i], lo[i], hi[i]);
          cl[i] = cost_of(L[i]);
          cn[i] = cnt_of(L[i]);
        }
        // (nl == DT_TREELET_N here: a subtree of >= N triangles always grows to N leaves.)  Every
        // subset index is a compile-time constant once the loops unroll, so the DP lives in
        // registers.
        constexpr int NS = 1 << DT_TREELET_N, full = NS - 1;
        float copt[NS];
        unsigned char part[NS];
#pragma unroll
        for (int S = 1; S < NS; ++S) {
          if ((S & (S - 1)) == 0) {
#pragma unroll
            for (int i = 0; i < DT_TREELET_N; ++i)
              if (S == (1 << i)) copt[S] = cl[i];
            part[S] = 0;
            continue;
          }
          float3 ulo = f3(kInf, kInf, kInf), uhi = f3(-kInf, -kInf, -kInf);
#pragma unroll
          for (int i = 0; i < DT_TREELET_N; ++i)
            if (S >> i & 1) { ulo = fminf3(ulo, lo[i]); uhi = fmaxf3(uhi, hi[i]); }
          const int low = S & -S;
          float best = kInf;
          int bp = low;
#pragma unroll
          for (int P = 1; P < S; ++P) {
            if ((P & S) != P || !(P & low)) continue;
            const float c = copt[P] + copt[S ^ P];
            if (c < best) { best = c; bp = P; }
          }
          copt[S] = box_area3(ulo, uhi) * kTreeletCi + best;
          part[S] = (unsigned char)bp;
        }
        if (copt[full] < cp * 0.9999f) {       // rewire the treelet's internal nodes
          int st[DT_TREELET_N], sn[DT_TREELET_N], sp = 0, pool = 1;
          st[sp] = full; sn[sp++] = p;
          while (sp > 0) {
            const int S = st[--sp], nd = sn[sp];
            const int P = part[S], Q = S ^ P;
            int kid[2];
            const int sub[2] = {P, Q};
            for (int q = 0; q < 2; ++q) {
              if ((sub[q] & (sub[q] - 1)) == 0) {
                kid[q] = L[__ffs(sub[q]) - 1];
              } else {
                kid[q] = I[pool++];
                st[sp] = sub[q]; sn[sp++] = kid[q];
              }
              if (kid[q] < 0) parent_leaf[~kid[q]] = nd; else parent_int[kid[q]] = nd;
            }
            __stcg(children + nd, make_int2(kid[0], kid[1]));
            float3 ulo = f3(kInf, kInf, kInf), uhi = f3(-kInf, -kInf, -kInf);
            int c = 0;
            for (int i = 0; i < nl; ++i)
              if (S >> i & 1) { ulo = fminf3(ulo, lo[i]); uhi = fmaxf3(uhi, hi[i]); c += cn[i]; }
            __stcg(nodebox + 2 * (size_t)nd, f4(ulo, 0.f));
            __stcg(nodebox + 2 * (size_t)nd + 1, f4(uhi, 0.f));
            __stcg(cost + nd, copt[S]);
            __stcg(ranges + nd, make_int2(0, c - 1));
            __stcg(narea + nd, box_area3(ulo, uhi));
          }
          cp = copt[full];
        }
      }
      __stcg(cost + p, cp);
      __stcg(ranges + p, make_int2(0, cnt - 1));
      __stcg(narea + p, ap);
      p = __ldcg(parent_int + p);
    }
  }
}

// ----------------------------------------------------------------------------- 4-wide collapse
// The binary Karras tree is collapsed into a 4-wide BVH by keeping the binary nodes at even
// depth: a wide node's children are its binary grandchildren (a binary child that is a leaf,
// or whose subtree holds <= kLeafMax triangles, becomes one leaf entry: a contiguous range of
// leaf-ordered triangles).  Child boxes are quantised to 8 bits per plane relative to the
// node box (conservatively: floor / ceil in float64, after the pad inflation), so a node is
// 64 B for four children -- half the bytes per child of the binary layout, half the depth.
//   n0 = (p.x, p.y, p.z, exponents e_x | e_y << 8 | e_z << 16)     scale_a = 2^(e_a - 127)
//   n1 = (qlo_x, qlo_y, qlo_z, qhi_x)  n2 = (qhi_y, qhi_z, ref0, ref1)  n3 = (ref2, ref3, -, -)
// q* hold one byte per child (child c in bits 8c..8c+7).  ref >= 0: wide node; ref = EMPTY:
// unused slot (qlo = 255 > qhi = 0); otherwise leaf: ref = -1 - (first << 2 | (count - 1)).
DT_D int bsize(const int2* __restrict__ ranges, int ref) { return ref < 0 ? 1 : ranges[ref].y - ranges[ref].x + 1; }
// entry e of a wide node is itself a wide node (else a leaf of <= leaf_max triangles)
DT_D bool wide_entry(const int2* __restrict__ ranges, int e, int leaf_max) {
  return e >= 0 && bsize(ranges, e) > leaf_max;
}

// Quantise and write wide node w: its entries ent[0..ne) (binary refs; internal entries carry
// their own wide index in wref), boxes padded outward so the slab test stays conservative.
DT_D void write_wide_node(int i, const int ent[4], const int wref[4], int ne, unsigned w, int wd, double pad,
                          const float4* __restrict__ leafbox, const float4* __restrict__ nodebox,
                          const int2* __restrict__ ranges, int leaf_max, uint4* __restrict__ wnodes,
                          float4* __restrict__ wbox, int* __restrict__ wdepth) {
  float3 ulo, uhi;
  load_box(leafbox, nodebox, i, ulo, uhi);
  double P[3] = {(double)__double2float_rd((double)ulo.x - pad), (double)__double2float_rd((double)ulo.y - pad),
                 (double)__double2float_rd((double)ulo.z - pad)};
  double hiU[3] = {(double)uhi.x + pad, (double)uhi.y + pad, (double)uhi.z + pad};
  int ex[3];
  double sc[3];
  for (int a = 0; a < 3; ++a) {
    double ext = hiU[a] - P[a];
    int k = -126;
    if (ext > 0.0) { frexp(ext / 255.0, &k); k = max(-126, min(127, k)); }
    ex[a] = k + 127;
    sc[a] = ldexp(1.0, k);
  }
  unsigned q[6] = {0, 0, 0, 0, 0, 0};
  int refs[4];
  for (int c = 0; c < 4; ++c) {
    unsigned ql[3] = {255, 255, 255}, qh[3] = {0, 0, 0};
    refs[c] = kEmptyRef;
    if (c < ne) {
      int e = ent[c];
      float3 lo, hi;
      load_box(leafbox, nodebox, e, lo, hi);
      const float l3[3] = {lo.x, lo.y, lo.z}, h3[3] = {hi.x, hi.y, hi.z};
      for (int a = 0; a < 3; ++a) {
        double fl = floor(((double)l3[a] - pad - P[a]) / sc[a]);
        double fh = ceil(((double)h3[a] + pad - P[a]) / sc[a]);
        ql[a] = (unsigned)fmin(fmax(fl, 0.0), 255.0);
        qh[a] = (unsigned)fmin(fmax(fh, 0.0), 255.0);
      }
      if (wide_entry(ranges, e, leaf_max)) {
        refs[c] = wref[c];
      } else {
        int first = e < 0 ? ~e : ranges[e].x;
        int cnt = bsize(ranges, e);
        refs[c] = -1 - ((first << 2) | (cnt - 1));
      }
    }
    for (int a = 0; a < 3; ++a) {
      q[a] |= ql[a] << (8 * c);
      q[3 + a] |= qh[a] << (8 * c);
    }
  }
  uint4* nd = wnodes + 4 * (size_t)w;
  // the three power-of-two scales as fp32 (x in word 3, y and z in words 14, 15), so the
  // traversal reads them without decoding
  nd[0] = make_uint4(__float_as_uint((float)P[0]), __float_as_uint((float)P[1]), __float_as_uint((float)P[2]),
                     (unsigned)ex[0] << 23);
  nd[1] = make_uint4(q[0], q[1], q[2], q[3]);
  nd[2] = make_uint4(q[4], q[5], (unsigned)refs[0], (unsigned)refs[1]);
  nd[3] = make_uint4((unsigned)refs[2], (unsigned)refs[3], (unsigned)ex[1] << 23, (unsigned)ex[2] << 23);
  wbox[2 * (size_t)w] = f4(ulo, 0.f);
  wbox[2 * (size_t)w + 1] = f4(uhi, 0.f);
  wdepth[w] = wd;
}

DT_D double wide_pad(const int* __restrict__ ibox) {
  float m = fmaxf(fmaxf(fmaxf(fabsf(ord2f(ibox[0])), fabsf(ord2f(ibox[1]))), fmaxf(fabsf(ord2f(ibox[2])), fabsf(ord2f(ibox[3])))),
                  fmaxf(fabsf(ord2f(ibox[4])), fabsf(ord2f(ibox[5]))));
  return (double)m * 4e-6 + 1e-30;
}

// A one-triangle mesh: the root wide node holds the single leaf.
__global__ void k_wide_single(const float4* __restrict__ leafbox, const float4* __restrict__ nodebox,
                              const int2* __restrict__ ranges, const int* __restrict__ ibox, uint4* __restrict__ wnodes,
                              float4* __restrict__ wbox, int* __restrict__ wdepth, int* __restrict__ nwide, int leaf_max) {
  const int ent[4] = {~0, 0, 0, 0}, wref[4] = {0, 0, 0, 0};
  *nwide = 1;
  write_wide_node(~0, ent, wref, 1, 0u, 0, wide_pad(ibox), leafbox, nodebox, ranges, leaf_max, wnodes, wbox, wdepth);
}

// Collapse to the 4-wide BVH (surface-area greedy): top down from the root, a wide node starts with
// its binary node's two children and repeatedly opens the internal entry of largest surface
// area until it has 4 entries (fuller nodes, larger boxes split first).  A work queue indexed
// by wide node id: a node's unopened internal entries get fresh ids (atomic counter) and are
// published into their queue slots; persistent threads claim slots in order and wait for
// them; `pending` (published - finished) reaching 0 ends the pass.
DT_D float box_area(const float4* __restrict__ nodebox, int e) {
  const float4 a = __ldcg(nodebox + 2 * (size_t)e), b = __ldcg(nodebox + 2 * (size_t)e + 1);
  const float dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
  return dx * dy + dy * dz + dz * dx;
}

#ifndef DT_WIDE_BLOCKS_PER_SM
#define DT_WIDE_BLOCKS_PER_SM 1
#endif

// ----------------------------------------------------------------------------- SAH collapse
// DT_WIDE_SAH = 1: the collapse takes the SAH-optimal set of entries per wide node (the
// dynamic program of Ylitie, Karras & Laine 2017 for wide BVHs, at width 4) instead of the
// greedy largest-area opening.  Bottom up over the binary tree (atomic-flag climb like the
// refit), C(n, i) = the least expected cost of representing binary subtree n by at most i
// entries of its parent wide node:
//   C(leaf, i)  = A(leaf) c_tri                          (one triangle, any i)
//   C(n, 1)     = A(n) c_node + min_{a+b=4} C(l, a) + C(r, b)      (n becomes a wide node)
//   C(n, i > 1) = min(C(n, i - 1), min_{a+b=i} C(l, a) + C(r, b))   (n opened into i entries)
// with A the box surface area and c_node / c_tri the costs of a 4-box node visit and a
// triangle test (130 : 37 lane operations).  The same pass records the entry
// lists the argmins select (went: E(n, 2), E(n, 3) and n's own wide node W(n)), so the top-down
// pass reads a wide node's entries with one load instead of walking the decisions.
#ifndef DT_WIDE_SAH
#define DT_WIDE_SAH 1
#endif
#ifndef DT_COST_NODE
#define DT_COST_NODE (130.f / 37.f)
#endif
constexpr float kCostNode = DT_COST_NODE, kCostTri = 1.f;

DT_D float box_area2(const float4* __restrict__ leafbox, const float4* __restrict__ nodebox, int ref) {
  float3 lo, hi;
  load_box(leafbox, nodebox, ref, lo, hi);
  const float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
  return dx * dy + dy * dz + dz * dx;
}

// Entries E(x, k) of the best representation of binary subtree x by at most k <= 3 entries
// (went: per internal node 3 int4 = E(x,2)[2] | E(x,3)[3] | W(x)[4], kEmptyRef-padded; W(x) is
// the entry list of the wide node made of x: its budget of 4 split between its children).
DT_D int get_entries(const int4* __restrict__ went, int x, int k, int out[4]) {
  if (x < 0 || k <= 1) { out[0] = x; return 1; }
  const int4 w0 = __ldcg(went + 3 * (size_t)x), w1 = __ldcg(went + 3 * (size_t)x + 1);
  const int e[5] = {w0.x, w0.y, w0.z, w0.w, w1.x};
  const int o = k == 2 ? 0 : 2, cnt = k == 2 ? 2 : 3;
  int n = 0;
  for (int q = 0; q < cnt; ++q)
    if (e[o + q] != kEmptyRef) out[n++] = e[o + q];
  return n;
}

__global__ void k_wide_cost(const int2* __restrict__ children, const int2* __restrict__ ranges, const int* __restrict__ parent_int,
                            const int* __restrict__ parent_leaf, int* __restrict__ flags, const float4* __restrict__ leafbox,
                            const float4* __restrict__ nodebox, int n, float4* __restrict__ cost, int4* __restrict__ went) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int p = parent_leaf[j];
    while (p >= 0) {
      __threadfence();
      if (atomicAdd(flags + p, 1) == 0) break;   // the second arrival evaluates the node
      __threadfence();
      const int2 ch = children[p];
      float Cl[4], Cr[4];
      const int cc[2] = {ch.x, ch.y};
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        float* C = s2 == 0 ? Cl : Cr;
        if (cc[s2] < 0) {
          const float c = box_area2(leafbox, nodebox, cc[s2]) * kCostTri;
          C[0] = C[1] = C[2] = C[3] = c;
        } else {
          const float4 q = __ldcg(cost + cc[s2]);
          C[0] = q.x; C[1] = q.y; C[2] = q.z; C[3] = q.w;
        }
      }
      float best[5];                              // best[j] = min_{a+b=j} Cl[a-1] + Cr[b-1]
      int split[5];
#pragma unroll
      for (int jj = 2; jj <= 4; ++jj) {
        float bv = kInf;
        int ba = 1;
        for (int a = 1; a < jj; ++a) {
          const float v = Cl[a - 1] + Cr[jj - a - 1];
          if (v < bv) { bv = v; ba = a; }
        }
        best[jj] = bv;
        split[jj] = ba;
      }
      float C[4];
      bool open[5];
      C[0] = box_area2(leafbox, nodebox, p) * kCostNode + best[4];
#pragma unroll
      for (int i = 2; i <= 4; ++i) {
        open[i] = best[i] < C[i - 2];
        C[i - 1] = open[i] ? best[i] : C[i - 2];
      }
      // entry lists: E(p, 2), E(p, 3) (for the parent's budget split) and W(p) (p's own wide node)
      int L[3][4];
      int nl[3];
#pragma unroll
      for (int i = 2; i <= 4; ++i) {
        int* out = L[i - 2];
        int cnt = 0;
        if (i == 4 || open[i]) {
          int a[4], b[4];
          const int na = get_entries(went, ch.x, split[i], a), nb = get_entries(went, ch.y, i - split[i], b);
          for (int q = 0; q < na; ++q) out[cnt++] = a[q];
          for (int q = 0; q < nb; ++q) out[cnt++] = b[q];
        } else if (i == 2) {
          out[cnt++] = p;                          // E(p, 1)
        } else {
          for (int q = 0; q < nl[i - 3]; ++q) out[cnt++] = L[i - 3][q];
        }
        nl[i - 2] = cnt;
        for (int q = cnt; q < 4; ++q) out[q] = kEmptyRef;
      }
      __stcg(cost + p, make_float4(C[0], C[1], C[2], C[3]));
      __stcg(went + 3 * (size_t)p, make_int4(L[0][0], L[0][1], L[1][0], L[1][1]));
      __stcg(went + 3 * (size_t)p + 1, make_int4(L[1][2], L[2][0], L[2][1], L[2][2]));
      __stcg(went + 3 * (size_t)p + 2, make_int4(L[2][3], kEmptyRef, kEmptyRef, kEmptyRef));
      p = parent_int[p];
    }
  }
}

// Entries of the wide node made of binary node b (at most 4): W(b) from the DP.
DT_D int sah_entries(const int4* __restrict__ went, int b, int ent[4]) {
  const int4 w1 = __ldcg(went + 3 * (size_t)b + 1), w2 = __ldcg(went + 3 * (size_t)b + 2);
  const int e[4] = {w1.y, w1.z, w1.w, w2.x};
  int ne = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (e[q] != kEmptyRef) ent[ne++] = e[q];
  return ne;
}

__global__ void k_wide_topdown(const int2* __restrict__ children, const int2* __restrict__ ranges,
                               const float4* __restrict__ leafbox, const float4* __restrict__ nodebox,
                               const int* __restrict__ ibox, uint4* __restrict__ wnodes, float4* __restrict__ wbox,
                               int* __restrict__ wdepth, int* __restrict__ nwide, unsigned long long* queue,
                               int* __restrict__ head, int* pending, int cap, int leaf_max,
                               const int4* __restrict__ went) {
  const double pad = wide_pad(ibox);
  while (true) {
    const int idx = atomicAdd(head, 1);
    if (idx >= cap) return;
    unsigned long long item;
    for (int spin = 0;; ++spin) {                    // poll through L2 (no atomic traffic)
      item = __ldcg(queue + idx);
      if (item != ~0ull) break;
      if (__ldcg(pending) == 0) return;              // no more work will be published
      __nanosleep(spin < 4 ? 64 : spin < 16 ? 256 : 1024);   // back off: every idle thread polls L2
    }
    __threadfence();                                   // acquire: the parent's writes before publishing
    const int b = (int)(item & 0xffffffffu), w = (int)(item >> 32);
    DT_CHECK(b >= 0 && w >= 0 && w < cap);
    int ent[4], wref[4] = {0, 0, 0, 0}, ne = 2;
    const int2 ch = children[b];
    ent[0] = ch.x;
    ent[1] = ch.y;
    if (went) ne = sah_entries(went, b, ent);
    while (!went && ne < 4) {
      int best = -1;
      float ba = -1.f;
      for (int c = 0; c < ne; ++c) {
        const int e = ent[c];
        if (e >= 0 && bsize(ranges, e) > leaf_max) {
          const float ar = box_area(nodebox, e);
          if (ar > ba) { ba = ar; best = c; }
        }
      }
      if (best < 0) break;
      const int2 g = children[ent[best]];
      ent[best] = g.x;
      ent[ne++] = g.y;
    }
    int nin = 0;
    for (int c = 0; c < ne; ++c) nin += wide_entry(ranges, ent[c], leaf_max);
    const int base = nin ? atomicAdd(nwide, nin) : 0;
    const int wd = __ldcg(wdepth + w);                 // written by the parent before publishing w (L2)
    for (int c = 0, k = 0; c < ne; ++c)
      if (wide_entry(ranges, ent[c], leaf_max)) wref[c] = base + k++;
    DT_CHECK(base + nin <= cap);
    write_wide_node(b, ent, wref, ne, (unsigned)w, wd, pad, leafbox, nodebox, ranges, leaf_max, wnodes, wbox, wdepth);
    for (int c = 0; c < ne; ++c) {
      if (!wide_entry(ranges, ent[c], leaf_max)) continue;
      wdepth[wref[c]] = wd + 1;
      __threadfence();
      atomicExch(queue + wref[c], ((unsigned long long)(unsigned)wref[c] << 32) | (unsigned)ent[c]);
    }
    __threadfence();
    atomicAdd(pending, nin - 1);
  }
}

__global__ void k_wide_topdown_init(unsigned long long* __restrict__ queue, int* __restrict__ head,
                                    int* __restrict__ pending, int* __restrict__ nwide, int* __restrict__ wdepth) {
  queue[0] = 0ull;                                      // binary root 0 -> wide node 0
  *head = 0;
  *pending = 1;
  *nwide = 1;
  wdepth[0] = 0;
}

__global__ void k_pack_tris(const float4* __restrict__ V, const int* __restrict__ F, const unsigned* __restrict__ order,
                            int n, float4* __restrict__ tris) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int f = (int)order[j];
    float3 v0 = f3(V[F[3 * f]]);
    float3 e1 = sub_rn(f3(V[F[3 * f + 1]]), v0), e2 = sub_rn(f3(V[F[3 * f + 2]]), v0);
    tris[3 * (size_t)j + 0] = f4(v0, __int_as_float(f));
    tris[3 * (size_t)j + 1] = f4(e1, 0.f);
    tris[3 * (size_t)j + 2] = f4(e2, 0.f);
  }
}

__global__ void k_scalars(const int* __restrict__ ibox, float* __restrict__ scal) {
  float3 lo = f3(ord2f(ibox[0]), ord2f(ibox[1]), ord2f(ibox[2]));
  float3 hi = f3(ord2f(ibox[3]), ord2f(ibox[4]), ord2f(ibox[5]));
  float m = fmaxf(fmaxf(fmaxf(fabsf(lo.x), fabsf(lo.y)), fmaxf(fabsf(lo.z), fabsf(hi.x))), fmaxf(fabsf(hi.y), fabsf(hi.z)));
  float pad = m * 8e-6f + 1e-30f;
  scal[0] = lo.x - pad; scal[1] = lo.y - pad; scal[2] = lo.z - pad;
  scal[3] = hi.x + pad; scal[4] = hi.y + pad; scal[5] = hi.z + pad;
  scal[6] = length(hi - lo);
}

__global__ void k_init_ibox(int* ibox) {
  int i = threadIdx.x;
  if (i < 12) ibox[i] = (i % 6) < 3 ? 0x7fffffff : (int)0x80000000;
}

// ----------------------------------------------------------------------------- checks
// Per wide node: every decoded child box must contain its child (the child wide node's box,
// or every triangle of a leaf); every triangle must be reached exactly once; every wide node
// but the root must be referenced exactly once.  out: [0] violations, [1] triangles reached
// through leaves, [2] (k_count_marks) distinct faces reached once, [3] depth.
__global__ void k_bvh_check(const uint4* __restrict__ wnodes, const float4* __restrict__ wbox,
                            const int* __restrict__ wdepth, const int* __restrict__ nwide_p,
                            const float4* __restrict__ tris, unsigned long long* __restrict__ out, int* __restrict__ mark,
                            int* __restrict__ wref) {
  int nw = *nwide_p;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    const uint4* nd = wnodes + 4 * (size_t)w;
    uint4 n0 = nd[0], n1 = nd[1], n2 = nd[2], n3 = nd[3];
    unsigned long long bad = 0, leaves = 0;
    for (int c = 0; c < 4; ++c) {
      int ref = wide_ref(n2, n3, c);
      if (ref == kEmptyRef) continue;
      float3 lo, hi;
      decode_wide_child(n0, n1, n2, n3, c, lo, hi);
      float3 clo, chi;
      if (ref >= 0) {
        atomicAdd(wref + ref, 1);
        clo = f3(wbox[2 * (size_t)ref]);
        chi = f3(wbox[2 * (size_t)ref + 1]);
        if (lo.x > clo.x || lo.y > clo.y || lo.z > clo.z || hi.x < chi.x || hi.y < chi.y || hi.z < chi.z) bad++;
      } else {
        int first, cnt;
        leaf_range(ref, first, cnt);
        for (int j = first; j < first + cnt; ++j) {
          float3 v0 = f3(tris[3 * (size_t)j]), v1 = v0 + f3(tris[3 * (size_t)j + 1]), v2 = v0 + f3(tris[3 * (size_t)j + 2]);
          clo = fminf3(v0, fminf3(v1, v2));
          chi = fmaxf3(v0, fmaxf3(v1, v2));
          if (lo.x > clo.x || lo.y > clo.y || lo.z > clo.z || hi.x < chi.x || hi.y < chi.y || hi.z < chi.z) bad++;
          atomicAdd(mark + __float_as_int(tris[3 * (size_t)j].w), 1);
          ++leaves;
        }
      }
    }
    atomicAdd(out + 0, bad);
    atomicAdd(out + 1, leaves);
    atomicMax(out + 3, (unsigned long long)wdepth[w]);
  }
}

__global__ void k_check_refs(const int* __restrict__ wref, const int* __restrict__ nwide_p, unsigned long long* __restrict__ out) {
  int nw = *nwide_p;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    if (wref[w] != (w == 0 ? 0 : 1)) atomicAdd(out + 0, 1ull);
}

__global__ void k_count_marks(const int* __restrict__ mark, int n, unsigned long long* __restrict__ out) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x)
    if (mark[f] == 1) atomicAdd(out + 2, 1ull);
}

}  // namespace

template <class T>
static cudaError_t grow(T*& p, size_t& cap, size_t n) {
  if (n <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
  cap = e == cudaSuccess ? n : 0;
  return e;
}

cudaError_t build_bvh(dt_ctx* c, const float* Vin, int nv, const int* Fin, int nf, cudaStream_t st, int* nl) {
  cudaError_t e;
  if ((size_t)nv > c->cap_nv) {
    size_t cap = nv;
    cudaFree(c->V); cudaFree(c->nrm); cudaFree(c->gV); cudaFree(c->gN); cudaFree(c->gVn); cudaFree(c->gS);
    cudaFree(c->vstart);
    c->V = c->gV = c->gN = c->gVn = c->gS = nullptr;
    c->nrm = nullptr;
    c->vstart = nullptr;
    if ((e = cudaMalloc(&c->V, cap * 16)) || (e = cudaMalloc(&c->nrm, cap * sizeof(D4))) || (e = cudaMalloc(&c->gV, cap * 16)) ||
        (e = cudaMalloc(&c->gN, cap * 16)) || (e = cudaMalloc(&c->gVn, cap * 16)) || (e = cudaMalloc(&c->gS, cap * 16)) ||
        (e = cudaMalloc(&c->vstart, (cap + 1) * sizeof(int))))
      return e;
    c->cap_nv = cap;
  }
  if ((size_t)nf > c->cap_nf) {
    size_t cap = nf;
    void* old[] = {c->F, c->fnrm, c->nodes, c->tris, c->keys, c->vals, c->children, c->parent_int, c->parent_leaf,
                   c->rflags, c->nodebox, c->leafbox, c->vcorner, c->fe, c->ranges,
                   c->wbox, c->wdepth, c->went};
    for (void* p : old)
      if (p) cudaFree(p);
    size_t ks = 2 * 3 * cap;   // keys/vals ping-pong sized for the 3*nf corner sort
    if ((e = cudaMalloc(&c->F, cap * 3 * sizeof(int))) || (e = cudaMalloc(&c->fnrm, cap * sizeof(D4))) ||
        (e = cudaMalloc(&c->nodes, cap * 64)) || (e = cudaMalloc(&c->tris, cap * 48)) ||
        (e = cudaMalloc(&c->keys, ks * sizeof(unsigned))) || (e = cudaMalloc(&c->vals, ks * sizeof(unsigned))) ||
        (e = cudaMalloc(&c->children, cap * sizeof(int2))) || (e = cudaMalloc(&c->parent_int, cap * sizeof(int))) ||
        (e = cudaMalloc(&c->parent_leaf, cap * sizeof(int))) || (e = cudaMalloc(&c->rflags, cap * sizeof(int))) ||
        (e = cudaMalloc(&c->nodebox, cap * 32)) || (e = cudaMalloc(&c->leafbox, cap * 32)) ||
        (e = cudaMalloc(&c->vcorner, 3 * cap * sizeof(unsigned))) || (e = cudaMalloc(&c->fe, 2 * cap * 16)) ||
        (e = cudaMalloc(&c->ranges, cap * sizeof(int2))) || (e = cudaMalloc(&c->went, cap * 3 * sizeof(int4))) ||
        (e = cudaMalloc(&c->wbox, cap * 32)) || (e = cudaMalloc(&c->wdepth, cap * sizeof(int))))
      return e;
    c->cap_nf = cap;
  }
  size_t nb_needed = 256 * ((3 * (size_t)nf + kSortTile - 1) / kSortTile);
  if ((e = grow(c->hist, c->hist_cap, nb_needed))) return e;
  if ((e = grow(c->scan_part, c->scan_part_cap, std::max(nb_needed, (size_t)nf) / kScanChunk + 16))) return e;
  if (!c->scal && (e = cudaMalloc(&c->scal, 16 * sizeof(float)))) return e;
  if (!c->iscal && (e = cudaMalloc(&c->iscal, 16 * sizeof(int)))) return e;

  const int T = 256;
  int gv = std::min((nv + T - 1) / T, c->sm_count * 8);
  int gf = std::min((nf + T - 1) / T, c->sm_count * 8);
  int gf3 = std::min((3 * nf + 1 + T - 1) / T, c->sm_count * 8);
  int launches = 0;
  k_init_ibox<<<1, 32, 0, st>>>(c->iscal);
  cudaMemcpyAsync(c->F, Fin, (size_t)nf * 3 * sizeof(int), cudaMemcpyDeviceToDevice, st);
  k_snapshot<<<gv, T, 0, st>>>(Vin, nv, c->V, c->iscal);
  k_faces<<<gf, T, 0, st>>>(c->V, c->F, nf, c->fnrm, c->iscal);
  launches += 3;
  // vertex -> incident corners CSR (sorted by vertex, then by corner id = face order)
  unsigned *ka = c->keys, *va = c->vals, *kb = c->keys + 3 * c->cap_nf, *vb = c->vals + 3 * c->cap_nf;
  k_corner_keys<<<gf3, T, 0, st>>>(c->F, 3 * nf, ka, va);
  int vbits = 8;
  while (vbits < 32 && (1u << vbits) < (unsigned)nv) vbits += 8;
  bool in_tmp;
  if ((e = radix_sort(ka, va, kb, vb, 3 * nf, vbits, c->hist, c->scan_part, st, in_tmp, &launches))) return e;
  unsigned* sk = in_tmp ? kb : ka;
  unsigned* sv = in_tmp ? vb : va;
  k_csr<<<gf3, T, 0, st>>>(sk, 3 * nf, nv, c->vstart);
  cudaMemcpyAsync(c->vcorner, sv, (size_t)3 * nf * sizeof(unsigned), cudaMemcpyDeviceToDevice, st);
  k_vertex_normals<<<gv, T, 0, st>>>(c->vstart, c->vcorner, c->fnrm, nv, c->nrm);
  launches += 3;
  // LBVH: Morton codes, radix sort, Karras hierarchy, bottom-up refit
  k_morton<<<gf, T, 0, st>>>(c->V, c->F, nf, c->iscal, ka, va);
  if ((e = radix_sort(ka, va, kb, vb, nf, 32, c->hist, c->scan_part, st, in_tmp, &launches))) return e;
  sk = in_tmp ? kb : ka;
  sv = in_tmp ? vb : va;
  launches += 1;
  if (nf > 1) {
    cudaMemsetAsync(c->rflags, 0, (size_t)(nf - 1) * sizeof(int), st);
    k_karras<<<gf, T, 0, st>>>(sk, nf, c->children, c->parent_int, c->parent_leaf, c->ranges);
    ++launches;
  }
  k_refit<<<gf, T, 0, st>>>(c->V, c->F, sv, nf, c->children, c->parent_int, c->parent_leaf, c->rflags, c->leafbox,
                            c->nodebox);
  if (nf >= DT_TREELET_N) {                             // treelet restructuring (cost in key scratch)
    float* tcost = reinterpret_cast<float*>(c->keys);
    float* narea = tcost + nf;                          // (keys hold 6 nf words)
    for (int pass = 0; pass < c->treelet_passes; ++pass) {
      cudaMemsetAsync(c->rflags, 0, (size_t)(nf - 1) * sizeof(int), st);
      k_treelet<<<gf, T, 0, st>>>(c->children, c->parent_int, c->parent_leaf, c->rflags, c->nodebox, c->leafbox, tcost,
                                  c->ranges, narea, nf);
      ++launches;
    }
  }
  // collapse to the quantised 4-wide BVH
  if (nf > 1) {                                         // surface-area greedy, top down
    if (!c->wqueue || c->wqueue_cap < nf) {
      cudaFree(c->wqueue);
      c->wqueue = nullptr;
      c->wqueue_cap = 0;
      if ((e = cudaMalloc(&c->wqueue, (size_t)nf * sizeof(unsigned long long) + 16 * sizeof(int)))) return e;
      c->wqueue_cap = nf;
    }
    int* ctr = reinterpret_cast<int*>(c->wqueue + c->wqueue_cap);
    int& gq = c->grid_cache[kGridWide];                 // per context (device): occupancy x SMs
    if (!gq) {
      int per = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k_wide_topdown, T, 0);
      // fewer persistent threads than the occupancy allows: the queue is published top down, so
      // most threads would only poll for unpublished entries
      gq = std::max(1, std::min(per, DT_WIDE_BLOCKS_PER_SM)) * c->sm_count;
    }
    int4* went = nullptr;
#if DT_WIDE_SAH
    // the DP's per-node costs live in scratch the collapse does not otherwise use at this
    // point (the sort keys: 4 words per node of the 6 nf available); its entry lists in went
    float4* cost = reinterpret_cast<float4*>(c->keys);
    went = c->went;
    cudaMemsetAsync(c->rflags, 0, (size_t)(nf - 1) * sizeof(int), st);
    k_wide_cost<<<gf, T, 0, st>>>(c->children, c->ranges, c->parent_int, c->parent_leaf, c->rflags, c->leafbox,
                                  c->nodebox, nf, cost, went);
    launches += 1;
#endif
    cudaMemsetAsync(c->wqueue, 0xff, (size_t)nf * sizeof(unsigned long long), st);
    k_wide_topdown_init<<<1, 1, 0, st>>>(c->wqueue, ctr, ctr + 1, c->iscal + 12, c->wdepth);
    k_wide_topdown<<<gq, T, 0, st>>>(c->children, c->ranges, c->leafbox, c->nodebox, c->iscal,
                                     reinterpret_cast<uint4*>(c->nodes), c->wbox, c->wdepth, c->iscal + 12, c->wqueue,
                                     ctr, ctr + 1, nf - 1, c->leaf_max, went);
    launches += 2;
  } else {
    k_wide_single<<<1, 1, 0, st>>>(c->leafbox, c->nodebox, c->ranges, c->iscal, reinterpret_cast<uint4*>(c->nodes),
                                   c->wbox, c->wdepth, c->iscal + 12, c->leaf_max);
    launches += 1;
  }
  k_pack_tris<<<gf, T, 0, st>>>(c->V, c->F, sv, nf, c->tris);
  k_scalars<<<1, 1, 0, st>>>(c->iscal, c->scal);
  launches += 3;
  c->nv = nv;
  c->nf = nf;
  *nl += launches;
  return cudaGetLastError();
}

cudaError_t launch_bvh_check(dt_ctx* c, long long* out_dev, cudaStream_t st) {
  int* mark = nullptr;
  int* wref = nullptr;
  cudaError_t e = cudaMallocAsync(&mark, (size_t)c->nf * sizeof(int), st);
  if (e) return e;
  if ((e = cudaMallocAsync(&wref, (size_t)c->nf * sizeof(int), st))) return e;
  cudaMemsetAsync(mark, 0, (size_t)c->nf * sizeof(int), st);
  cudaMemsetAsync(wref, 0, (size_t)c->nf * sizeof(int), st);
  cudaMemsetAsync(out_dev, 0, 4 * sizeof(long long), st);
  int g = std::min((c->nf + 255) / 256, c->sm_count * 8);
  k_bvh_check<<<g, 256, 0, st>>>(reinterpret_cast<const uint4*>(c->nodes), c->wbox, c->wdepth, c->iscal + 12, c->tris,
                                 (unsigned long long*)out_dev, mark, wref);
  k_check_refs<<<g, 256, 0, st>>>(wref, c->iscal + 12, (unsigned long long*)out_dev);
  k_count_marks<<<g, 256, 0, st>>>(mark, c->nf, (unsigned long long*)out_dev);
  cudaFreeAsync(mark, st);
  cudaFreeAsync(wref, st);
  return cudaGetLastError();
}

DevScene scene_from_ctx(const dt_ctx* c) {
  DevScene s{};
  s.V = c->V;
  s.F = c->F;
  s.nrm = c->nrm;
  s.nv = c->nv;
  s.nf = c->nf;
  s.nodes = c->nodes;
  s.tris = c->tris;
  s.root = 0;
  s.scal = c->scal;
  s.wcount = c->counters + 5;
  return s;
}

DT_DEFINE_CHECK_READER(check_status_bvh)

}  // namespace dt
