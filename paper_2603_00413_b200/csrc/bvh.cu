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

// unit face normals and centroid bounds (Morton quantisation)
__global__ void k_faces(const float4* __restrict__ V, const int* __restrict__ F, int nf, float4* __restrict__ fn,
                        int* __restrict__ ibox) {
  float3 lo = f3(kInf, kInf, kInf), hi = -lo;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += gridDim.x * blockDim.x) {
    float3 a = f3(V[F[3 * f]]), b = f3(V[F[3 * f + 1]]), c = f3(V[F[3 * f + 2]]);
    float3 n = cross(b - a, c - a);
    float L = length(n);
    fn[f] = L > 0.0f ? f4(n * (1.0f / L), L) : make_float4(0, 0, 0, 0);  // zero-area faces add 0 (R6)
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

// n_v = normalize(sum of incident unit face normals), gathered in face order (deterministic)
__global__ void k_vertex_normals(const int* __restrict__ vstart, const unsigned* __restrict__ corner,
                                 const float4* __restrict__ fn, int nv, float4* __restrict__ nrm) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    float3 s = f3(0, 0, 0);
    for (int j = vstart[v]; j < vstart[v + 1]; ++j) s += f3(fn[corner[j] / 3]);
    float L = length(s);
    nrm[v] = L > 0.0f ? f4(s * (1.0f / L), L) : make_float4(0, 0, 1, 0);
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
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    offs[threadIdx.x] += total[threadIdx.x];
    __syncthreads();
  }
}

cudaError_t radix_sort(unsigned* keys, unsigned* vals, unsigned* tk, unsigned* tv, int n, int bits, unsigned* hist,
                       cudaStream_t st, bool& result_in_tmp) {
  int nb = (n + kSortTile - 1) / kSortTile;
  result_in_tmp = false;
  unsigned *ki = keys, *vi = vals, *ko = tk, *vo = tv;
  for (int shift = 0; shift < bits; shift += 8) {
    k_hist<<<nb, kSortThreads, 0, st>>>(ki, n, shift, hist);
    k_scan<<<1, 1024, 0, st>>>(hist, 256 * nb);
    k_scatter<<<nb, kSortThreads, 0, st>>>(ki, vi, ko, vo, n, shift, hist);
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
                         int* __restrict__ parent_leaf) {
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
    int left = min(i, j) == gamma ? ~gamma : gamma;
    int right = max(i, j) == gamma + 1 ? ~(gamma + 1) : gamma + 1;
    children[i] = make_int2(left, right);
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
      if (atomicAdd(flags + p, 1) == 0) break;   // first arrival: the sibling finishes the node
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

// 64-B node: (c0lo.x, c0hi.x, c0lo.y, c0hi.y) (c0lo.z, c0hi.z, c1lo.x, c1hi.x)
//            (c1lo.y, c1hi.y, c1lo.z, c1hi.z) (ref0, ref1, -, -); boxes inflated by `pad`.
__global__ void k_pack_nodes(const int2* __restrict__ children, const float4* __restrict__ leafbox,
                             const float4* __restrict__ nodebox, int n, const int* __restrict__ ibox,
                             float4* __restrict__ nodes) {
  float m = fmaxf(fmaxf(fmaxf(fabsf(ord2f(ibox[0])), fabsf(ord2f(ibox[1]))), fmaxf(fabsf(ord2f(ibox[2])), fabsf(ord2f(ibox[3])))),
                  fmaxf(fabsf(ord2f(ibox[4])), fabsf(ord2f(ibox[5]))));
  float pad = m * 4e-6f + 1e-30f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
    int2 ch = children[i];
    float3 l0, h0, l1, h1;
    load_box(leafbox, nodebox, ch.x, l0, h0);
    load_box(leafbox, nodebox, ch.y, l1, h1);
    float3 P = f3(pad, pad, pad);
    l0 = l0 - P; h0 = h0 + P; l1 = l1 - P; h1 = h1 + P;
    nodes[4 * (size_t)i + 0] = make_float4(l0.x, h0.x, l0.y, h0.y);
    nodes[4 * (size_t)i + 1] = make_float4(l0.z, h0.z, l1.x, h1.x);
    nodes[4 * (size_t)i + 2] = make_float4(l1.y, h1.y, l1.z, h1.z);
    nodes[4 * (size_t)i + 3] = make_float4(__int_as_float(ch.x), __int_as_float(ch.y), 0.f, 0.f);
  }
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
__global__ void k_bvh_check(const float4* __restrict__ nodes, const float4* __restrict__ tris, const int* __restrict__ parent_int,
                            const int* __restrict__ parent_leaf, int n, int root, unsigned long long* __restrict__ out,
                            int* __restrict__ mark) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int f = __float_as_int(tris[3 * (size_t)j].w);
    atomicAdd(mark + f, 1);
    // walk to the root; count depth
    int depth = 0, p = n > 1 ? parent_leaf[j] : -1;
    int ref = ~j;
    unsigned long long bad = 0;
    float3 v0 = f3(tris[3 * (size_t)j]), v1 = v0 + f3(tris[3 * (size_t)j + 1]), v2 = v0 + f3(tris[3 * (size_t)j + 2]);
    float3 clo = fminf3(v0, fminf3(v1, v2)), chi = fmaxf3(v0, fmaxf3(v1, v2));
    while (p >= 0) {
      const float4* nd = nodes + 4 * (size_t)p;
      float4 a = nd[0], b = nd[1], c = nd[2], e = nd[3];
      bool left = __float_as_int(e.x) == ref;
      float3 lo = left ? f3(a.x, a.z, b.x) : f3(b.z, c.x, c.z);
      float3 hi = left ? f3(a.y, a.w, b.y) : f3(b.w, c.y, c.w);
      if (!left && __float_as_int(e.y) != ref) bad++;
      if (lo.x > clo.x || lo.y > clo.y || lo.z > clo.z || hi.x < chi.x || hi.y < chi.y || hi.z < chi.z) bad++;
      clo = lo; chi = hi;
      ref = p;
      p = parent_int[p];
      ++depth;
    }
    if (ref != root && !(n == 1 && ref == ~0)) bad++;
    atomicAdd(out + 0, bad);
    atomicAdd(out + 1, 1ull);
    atomicMax(out + 3, (unsigned long long)depth);
  }
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
    size_t dummy;
    cudaFree(c->V); cudaFree(c->nrm); cudaFree(c->gV); cudaFree(c->gN); cudaFree(c->gVn); cudaFree(c->gS);
    cudaFree(c->vstart);
    c->V = c->nrm = c->gV = c->gN = c->gVn = c->gS = nullptr;
    c->vstart = nullptr;
    if ((e = cudaMalloc(&c->V, cap * 16)) || (e = cudaMalloc(&c->nrm, cap * 16)) || (e = cudaMalloc(&c->gV, cap * 16)) ||
        (e = cudaMalloc(&c->gN, cap * 16)) || (e = cudaMalloc(&c->gVn, cap * 16)) || (e = cudaMalloc(&c->gS, cap * 16)) ||
        (e = cudaMalloc(&c->vstart, (cap + 1) * sizeof(int))))
      return e;
    (void)dummy;
    c->cap_nv = cap;
  }
  if ((size_t)nf > c->cap_nf) {
    size_t cap = nf;
    cudaFree(c->F); cudaFree(c->fnrm); cudaFree(c->nodes); cudaFree(c->tris); cudaFree(c->keys); cudaFree(c->vals);
    cudaFree(c->children); cudaFree(c->parent_int); cudaFree(c->parent_leaf); cudaFree(c->rflags);
    cudaFree(c->nodebox); cudaFree(c->leafbox); cudaFree(c->vcorner); cudaFree(c->fe);
    size_t ks = 2 * 3 * cap;   // keys/vals ping-pong sized for the 3*nf corner sort
    if ((e = cudaMalloc(&c->F, cap * 3 * sizeof(int))) || (e = cudaMalloc(&c->fnrm, cap * 16)) ||
        (e = cudaMalloc(&c->nodes, std::max<size_t>(cap - 1, 1) * 64)) || (e = cudaMalloc(&c->tris, cap * 48)) ||
        (e = cudaMalloc(&c->keys, ks * sizeof(unsigned))) || (e = cudaMalloc(&c->vals, ks * sizeof(unsigned))) ||
        (e = cudaMalloc(&c->children, std::max<size_t>(cap - 1, 1) * sizeof(int2))) ||
        (e = cudaMalloc(&c->parent_int, std::max<size_t>(cap - 1, 1) * sizeof(int))) ||
        (e = cudaMalloc(&c->parent_leaf, cap * sizeof(int))) ||
        (e = cudaMalloc(&c->rflags, std::max<size_t>(cap - 1, 1) * sizeof(int))) ||
        (e = cudaMalloc(&c->nodebox, std::max<size_t>(cap - 1, 1) * 32)) || (e = cudaMalloc(&c->leafbox, cap * 32)) ||
        (e = cudaMalloc(&c->vcorner, 3 * cap * sizeof(unsigned))) || (e = cudaMalloc(&c->fe, 2 * cap * 16)))
      return e;
    c->cap_nf = cap;
  }
  size_t nb_needed = 256 * ((3 * (size_t)nf + kSortTile - 1) / kSortTile);
  if ((e = grow(c->hist, c->hist_cap, nb_needed))) return e;
  if (!c->scal && (e = cudaMalloc(&c->scal, 16 * sizeof(float)))) return e;
  if (!c->iscal && (e = cudaMalloc(&c->iscal, 16 * sizeof(int)))) return e;

  const int T = 256;
  int gv = std::min((nv + T - 1) / T, c->sm_count * 8);
  int gf = std::min((nf + T - 1) / T, c->sm_count * 8);
  int gf3 = std::min((3 * nf + 1 + T - 1) / T, c->sm_count * 8);
  k_init_ibox<<<1, 32, 0, st>>>(c->iscal);
  cudaMemcpyAsync(c->F, Fin, (size_t)nf * 3 * sizeof(int), cudaMemcpyDeviceToDevice, st);
  k_snapshot<<<gv, T, 0, st>>>(Vin, nv, c->V, c->iscal);
  k_faces<<<gf, T, 0, st>>>(c->V, c->F, nf, c->fnrm, c->iscal);
  // vertex -> incident corners CSR (sorted by vertex, then by corner id = face order)
  unsigned *ka = c->keys, *va = c->vals, *kb = c->keys + 3 * c->cap_nf, *vb = c->vals + 3 * c->cap_nf;
  k_corner_keys<<<gf3, T, 0, st>>>(c->F, 3 * nf, ka, va);
  int vbits = 8;
  while (vbits < 32 && (1u << vbits) < (unsigned)nv) vbits += 8;
  bool in_tmp;
  if ((e = radix_sort(ka, va, kb, vb, 3 * nf, vbits, c->hist, st, in_tmp))) return e;
  unsigned* sk = in_tmp ? kb : ka;
  unsigned* sv = in_tmp ? vb : va;
  k_csr<<<gf3, T, 0, st>>>(sk, 3 * nf, nv, c->vstart);
  cudaMemcpyAsync(c->vcorner, sv, (size_t)3 * nf * sizeof(unsigned), cudaMemcpyDeviceToDevice, st);
  k_vertex_normals<<<gv, T, 0, st>>>(c->vstart, c->vcorner, c->fnrm, nv, c->nrm);
  // LBVH
  k_morton<<<gf, T, 0, st>>>(c->V, c->F, nf, c->iscal, ka, va);
  if ((e = radix_sort(ka, va, kb, vb, nf, 32, c->hist, st, in_tmp))) return e;
  sk = in_tmp ? kb : ka;
  sv = in_tmp ? vb : va;
  if (nf > 1) {
    cudaMemsetAsync(c->rflags, 0, (size_t)(nf - 1) * sizeof(int), st);
    k_karras<<<gf, T, 0, st>>>(sk, nf, c->children, c->parent_int, c->parent_leaf);
  }
  k_refit<<<gf, T, 0, st>>>(c->V, c->F, sv, nf, c->children, c->parent_int, c->parent_leaf, c->rflags, c->leafbox,
                            c->nodebox);
  if (nf > 1) k_pack_nodes<<<gf, T, 0, st>>>(c->children, c->leafbox, c->nodebox, nf, c->iscal, c->nodes);
  k_pack_tris<<<gf, T, 0, st>>>(c->V, c->F, sv, nf, c->tris);
  k_scalars<<<1, 1, 0, st>>>(c->iscal, c->scal);
  c->nv = nv;
  c->nf = nf;
  // kernels: ibox, snapshot, faces, corner keys, csr, vertex normals, morton, refit,
  // pack tris, scalars (10) + 3 per radix pass + karras/pack nodes when nf > 1
  *nl += 10 + 3 * (vbits / 8) + 3 * 4 + (nf > 1 ? 2 : 0);
  return cudaGetLastError();
}

cudaError_t launch_bvh_check(dt_ctx* c, long long* out_dev, cudaStream_t st) {
  int* mark = nullptr;
  cudaError_t e = cudaMallocAsync(&mark, (size_t)c->nf * sizeof(int), st);
  if (e) return e;
  cudaMemsetAsync(mark, 0, (size_t)c->nf * sizeof(int), st);
  cudaMemsetAsync(out_dev, 0, 4 * sizeof(long long), st);
  int g = std::min((c->nf + 255) / 256, c->sm_count * 8);
  k_bvh_check<<<g, 256, 0, st>>>(c->nodes, c->tris, c->parent_int, c->parent_leaf, c->nf, c->nf > 1 ? 0 : ~0,
                                 (unsigned long long*)out_dev, mark);
  k_count_marks<<<g, 256, 0, st>>>(mark, c->nf, (unsigned long long*)out_dev);
  cudaFreeAsync(mark, st);
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
  s.root = c->nf > 1 ? 0 : ~0;
  s.scal = c->scal;
  return s;
}

}  // namespace dt
