// Periodic mesh regularisers: the edge-normal smoothness term
// L_edge = (1/|E'|) sum_{(i,j) in E'} (1 - n_i . n_j)^2 and the uniform-Laplacian
// uniformity term L_lap = (1/|V|) sum_i |v_i - mean_{j in N(i)} v_j|^2 (R31), with their
// gradients w.r.t. the vertices of the current dt_build_bvh snapshot.  The vertex
// neighbourhoods come from the snapshot's corner CSR (vertex -> incident faces); every sum is
// a per-vertex gather over the (symmetric) neighbour lists, so the results are deterministic.
#include <cuda_runtime.h>

#include <algorithm>

#include "dt_internal.h"

namespace dt {
namespace {

constexpr int kMaxValence = 64;

// unique neighbours of v (ascending) from its incident faces; returns the count (<= cap)
DT_D int collect_neighbours(const int* vstart, const unsigned* corner, const int* F, int v, int out[kMaxValence]) {
  int n = 0;
  for (int j = vstart[v]; j < vstart[v + 1]; ++j) {
    const unsigned c = corner[j];
    const int f = (int)(c / 3u), k = (int)(c % 3u);
    const int cand[2] = {F[3 * f + (k + 1) % 3], F[3 * f + (k + 2) % 3]};
    for (int q = 0; q < 2; ++q) {
      int x = cand[q], pos = n;
      bool dup = false;
      for (int r = 0; r < n; ++r) {
        if (out[r] == x) { dup = true; break; }
      }
      if (dup || n == kMaxValence) continue;
      while (pos > 0 && out[pos - 1] > x) { out[pos] = out[pos - 1]; --pos; }   // insertion sort
      out[pos] = x;
      ++n;
    }
  }
  return n;
}

__global__ void k_nbr_count(const int* __restrict__ vstart, const unsigned* __restrict__ corner,
                            const int* __restrict__ F, int nv, int* __restrict__ cnt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int nb[kMaxValence];
    cnt[v] = collect_neighbours(vstart, corner, F, v, nb);
  }
}

// exclusive scan of cnt[0..n) into start[0..n], one block (n up to a few million)
__global__ void k_nbr_scan(const int* __restrict__ cnt, int n, int* __restrict__ start) {
  __shared__ int part[1024];
  const int T = blockDim.x, t = threadIdx.x;
  const int per = (n + T - 1) / T, b = min(t * per, n), e = min(b + per, n);
  int s = 0;
  for (int i = b; i < e; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int acc = 0;
    for (int i = 0; i < T; ++i) { int x = part[i]; part[i] = acc; acc += x; }
    start[n] = acc;
  }
  __syncthreads();
  int acc = part[t];
  for (int i = b; i < e; ++i) { start[i] = acc; acc += cnt[i]; }
}

__global__ void k_nbr_fill(const int* __restrict__ vstart, const unsigned* __restrict__ corner,
                           const int* __restrict__ F, int nv, const int* __restrict__ start, int* __restrict__ nbr,
                           int* __restrict__ owner) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int nb[kMaxValence];
    const int n = collect_neighbours(vstart, corner, F, v, nb);
    for (int q = 0; q < n; ++q) {
      nbr[start[v] + q] = nb[q];
      owner[start[v] + q] = v;
    }
  }
}

DT_D float warp_sum(float x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
  return x;
}

// L_edge: loss over edges (i < j), and dL/dn_i = (1/|E|) sum_{j in N(i)} -2 (1 - n_i.n_j) n_j
// written into gN (the vertex-normal chain then maps it to dV)
__global__ void k_edge_reg(const D4* __restrict__ nrm, const int* __restrict__ start, const int* __restrict__ nbr,
                           int nv, float lambda, float4* __restrict__ gN, float* __restrict__ loss) {
  const float inv_e = 2.0f / (float)max(start[nv], 1);     // |E| = (sum of valences) / 2
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const double3 ni = xyz(nrm[i]);
    double3 g = d3(0, 0, 0);
    for (int q = start[i]; q < start[i + 1]; ++q) {
      const int j = nbr[q];
      const double3 nj = xyz(nrm[j]);
      const double d = 1.0 - dot(ni, nj);                  // float64: near-parallel normals cancel
      if (j > i) acc += (float)(d * d);
      g += nj * (-2.0 * d);
    }
    gN[i] = f4(f3(g) * (lambda * inv_e), 0.f);
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc != 0.f) atomicAdd(loss, acc * inv_e);
}

// L_lap: delta_i = v_i - mean_{N(i)} v_j (0 without neighbours)
__global__ void k_lap_delta(const float4* __restrict__ V, const int* __restrict__ start, const int* __restrict__ nbr,
                            int nv, float4* __restrict__ delta, float* __restrict__ loss) {
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const int b = start[i], e = start[i + 1];
    float3 dl = f3(0, 0, 0);
    if (e > b) {
      float3 m = f3(0, 0, 0);
      for (int q = b; q < e; ++q) m += f3(V[nbr[q]]);
      dl = f3(V[i]) - m * (1.0f / (float)(e - b));
    }
    delta[i] = f4(dl, 0.f);
    acc += dot(dl, dl);
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc != 0.f) atomicAdd(loss, acc / (float)nv);
}

// dL_lap/dv_k = (2/|V|) (delta_k - sum_{i in N(k)} delta_i / |N(i)|) (neighbourhoods symmetric)
__global__ void k_lap_grad(const float4* __restrict__ delta, const int* __restrict__ start, const int* __restrict__ nbr,
                           int nv, float lambda, float* __restrict__ grad_V) {
  const float c = 2.0f * lambda / (float)nv;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += gridDim.x * blockDim.x) {
    float3 g = f3(delta[k]);
    for (int q = start[k]; q < start[k + 1]; ++q) {
      const int i = nbr[q];
      g -= f3(delta[i]) * (1.0f / (float)(start[i + 1] - start[i]));
    }
    grad_V[3 * k] += g.x * c;
    grad_V[3 * k + 1] += g.y * c;
    grad_V[3 * k + 2] += g.z * c;
  }
}

__global__ void k_add_vec(const float4* __restrict__ src, int n, float* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float4 s = src[i];
    dst[3 * i] += s.x;
    dst[3 * i + 1] += s.y;
    dst[3 * i + 2] += s.z;
  }
}

// ----------------------------------------------------------------------------- L_mask (R32)
constexpr int kMaskThreads = 128;

DT_D void image_ray(const float* K, const float* c2w, int v, float u, float w, float3& o, float3& d) {
  const float* k = K + 4 * v;
  const float* m = c2w + 12 * v;
  const float dx = (u - k[2]) / k[0], dy = (w - k[3]) / k[1];
  const float3 r = f3(m[0] * dx + m[1] * dy + m[2], m[4] * dx + m[5] * dy + m[6], m[8] * dx + m[9] * dy + m[10]);
  d = r * (1.0f / sqrtf(dot(r, r)));
  o = f3(m[3], m[7], m[11]);
}

// the rendered mask (the camera ray through the pixel centre hits the mesh) and
// sum |M^ - M| / N
__global__ void __launch_bounds__(kMaskThreads) k_mask_render(DevScene s, const float* __restrict__ K,
                                                              const float* __restrict__ c2w, int n_views, int W, int H,
                                                              const float* __restrict__ gt, float inv_n,
                                                              float* __restrict__ mask_out, float* __restrict__ loss) {
  __shared__ int sstack[kStackShared * kMaskThreads];
  int err = 0, visits = 0, tests = 0;
  float acc = 0.f;
  const int64_t n = (int64_t)n_views * W * H;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    float3 o, d;
    camera_ray(K, c2w, W, H, p, o, d);
    float t, u, v;
    const float m = traverse(s, o, d, 0.0f, t, u, v, sstack + threadIdx.x, kMaskThreads, err, visits, tests) >= 0;
    acc += fabsf(m - gt[p]);
    if (mask_out) mask_out[p] = m;
  }
  acc = warp_sum(acc);
  if (lane_id() == 0 && acc != 0.f) atomicAdd(loss, acc * inv_n);
}

DT_D bool covered(const DevScene& s, const float* K, const float* c2w, int v, float u, float w, int* sstack) {
  float3 o, d;
  image_ray(K, c2w, v, u, w, o, d);
  float t, bu, bv;
  int err = 0, visits = 0, tests = 0;
  return traverse(s, o, d, 0.0f, t, bu, bv, sstack, kMaskThreads, err, visits, tests) >= 0;
}

// pinhole projection of X in view v: image point and d(u, w)/dX rows (OpenCV axes, R19)
DT_D bool project(const float* K, const float* c2w, int v, float3 X, float2& p, float3& ju, float3& jw) {
  const float* k = K + 4 * v;
  const float* m = c2w + 12 * v;
  const float3 q = X - f3(m[3], m[7], m[11]);
  const float3 r0 = f3(m[0], m[4], m[8]), r1 = f3(m[1], m[5], m[9]), r2 = f3(m[2], m[6], m[10]);   // R columns
  const float x = dot(r0, q), y = dot(r1, q), z = dot(r2, q);
  if (!(z > 1e-6f)) return false;
  p = make_float2(k[0] * x / z + k[2], k[1] * y / z + k[3]);
  ju = (r0 * (1.0f / z) - r2 * (x / (z * z))) * k[0];
  jw = (r1 * (1.0f / z) - r2 * (y / (z * z))) * k[1];
  return true;
}

// silhouette-edge sampling of dL_mask/dV (R32): one thread per (view, directed neighbour
// entry i -> j with i < j)
__global__ void __launch_bounds__(kMaskThreads) k_mask_grad(
    DevScene s, const float* __restrict__ K, const float* __restrict__ c2w, int n_views, int W, int H,
    const float* __restrict__ gt, const int* __restrict__ nbr, const int* __restrict__ owner,
    const int* __restrict__ nbr_total, int64_t n_ent, const int* __restrict__ vstart, const unsigned* __restrict__ vcorner, const int* __restrict__ F,
    const float4* __restrict__ V, float scale, float spacing, float eps, float* __restrict__ grad_V) {
  __shared__ int sstack[kStackShared * kMaskThreads];
  const int64_t total = (int64_t)n_views * n_ent;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(id / n_ent);
    const int64_t q = id - (int64_t)v * n_ent;
    if (q >= *nbr_total) continue;                       // n_ent is the 6 nf bound
    const int a = owner[q], b = nbr[q];
    DT_CHECK(a >= 0 && b >= 0 && a < s.nv && b < s.nv);
    if (b <= a) continue;
    int f1 = -1, f2 = -1;
    for (int c = vstart[a]; c < vstart[a + 1]; ++c) {
      const int f = (int)(vcorner[c] / 3u);
      if (F[3 * f] == b || F[3 * f + 1] == b || F[3 * f + 2] == b) {
        if (f1 < 0) f1 = f; else f2 = f;
      }
    }
    const float* m = c2w + 12 * v;
    const float3 cam = f3(m[3], m[7], m[11]);
    auto front = [&](int f) {
      const float3 p0 = f3(V[F[3 * f]]), p1 = f3(V[F[3 * f + 1]]), p2 = f3(V[F[3 * f + 2]]);
      return dot(cam - p0, cross(p1 - p0, p2 - p0)) > 0.0f;
    };
    int fr = -1;
    if (f2 < 0) {
      if (f1 >= 0 && front(f1)) fr = f1;                       // boundary edge
    } else {
      const bool a1 = front(f1), a2 = front(f2);
      if (a1 != a2) fr = a1 ? f1 : f2;
    }
    if (fr < 0) continue;
    const int cv = F[3 * fr] != a && F[3 * fr] != b ? F[3 * fr] : (F[3 * fr + 1] != a && F[3 * fr + 1] != b ? F[3 * fr + 1]
                                                                                                        : F[3 * fr + 2]);
    float2 pa, pb, pc;
    float3 jua, jwa, jub, jwb, t0, t1;
    if (!project(K, c2w, v, f3(V[a]), pa, jua, jwa) || !project(K, c2w, v, f3(V[b]), pb, jub, jwb) ||
        !project(K, c2w, v, f3(V[cv]), pc, t0, t1))
      continue;
    const float ex = pb.x - pa.x, ey = pb.y - pa.y, L = sqrtf(ex * ex + ey * ey);
    if (!(L > 0.f)) continue;
    float nx = -ey / L, ny = ex / L;
    if (nx * (pc.x - pa.x) + ny * (pc.y - pa.y) > 0.f) { nx = -nx; ny = -ny; }   // outward: away from the face
    const int Ks = min(4096, max(1, (int)ceilf(L / spacing)));
    float ga = 0.f, gb = 0.f;
    for (int k = 0; k < Ks; ++k) {
      const float sk = ((float)k + 0.5f) / (float)Ks;
      const float x = pa.x + sk * ex, y = pa.y + sk * ey;
      const float xo = x + eps * nx, yo = y + eps * ny;
      if (!(xo >= 0.f && xo < (float)W && yo >= 0.f && yo < (float)H)) continue;
      if (covered(s, K, c2w, v, xo, yo, sstack + threadIdx.x)) continue;
      if (!covered(s, K, c2w, v, x - eps * nx, y - eps * ny, sstack + threadIdx.x)) continue;
      const float g = gt[((int64_t)v * H + (int)yo) * W + (int)xo];
      const float w = (1.0f - 2.0f * g) * (L / (float)Ks);
      ga += w * (1.0f - sk);
      gb += w * sk;
    }
    if (ga == 0.f && gb == 0.f) continue;
    const float3 da = (jua * nx + jwa * ny) * (ga * scale), db = (jub * nx + jwb * ny) * (gb * scale);
    atomicAdd(grad_V + 3 * a, da.x); atomicAdd(grad_V + 3 * a + 1, da.y); atomicAdd(grad_V + 3 * a + 2, da.z);
    atomicAdd(grad_V + 3 * b, db.x); atomicAdd(grad_V + 3 * b + 1, db.y); atomicAdd(grad_V + 3 * b + 2, db.z);
  }
}

}  // namespace

// vertex neighbour CSR of the current snapshot (rebuilt per call: nv threads, cheap)
cudaError_t build_neighbours(dt_ctx* c, cudaStream_t st, int* nl) {
  const int nv = c->nv, T = 256;
  const int g = std::max(1, std::min((nv + T - 1) / T, c->sm_count * 8));
  cudaError_t e;
  if (c->nbr_cap_v < nv + 1) {
    cudaFree(c->nbr_start);
    cudaFree(c->nbr_cnt);
    c->nbr_start = c->nbr_cnt = nullptr;
    c->nbr_cap_v = 0;
    if ((e = cudaMalloc(&c->nbr_start, (size_t)(nv + 1) * sizeof(int))) ||
        (e = cudaMalloc(&c->nbr_cnt, (size_t)(nv + 1) * sizeof(int))))
      return e;
    c->nbr_cap_v = nv + 1;
  }
  const int64_t nmax = (int64_t)6 * c->nf;   // bounded by the 2 * 3nf corner pairs
  if (c->nbr_cap < nmax) {
    cudaFree(c->nbr);
    cudaFree(c->nbr_owner);
    c->nbr = c->nbr_owner = nullptr;
    c->nbr_cap = 0;
    if ((e = cudaMalloc(&c->nbr, (size_t)nmax * sizeof(int))) || (e = cudaMalloc(&c->nbr_owner, (size_t)nmax * sizeof(int))))
      return e;
    c->nbr_cap = nmax;
  }
  k_nbr_count<<<g, T, 0, st>>>(c->vstart, c->vcorner, c->F, nv, c->nbr_cnt);
  k_nbr_scan<<<1, 1024, 0, st>>>(c->nbr_cnt, nv, c->nbr_start);
  k_nbr_fill<<<g, T, 0, st>>>(c->vstart, c->vcorner, c->F, nv, c->nbr_start, c->nbr, c->nbr_owner);
  *nl += 3;
  return cudaGetLastError();
}

cudaError_t launch_mask_loss(dt_ctx* c, const dt_cameras* cams, const float* gt, float lambda, float* grad_V,
                             float* loss, float* mask_out, cudaStream_t st, int* nl) {
  cudaError_t e;
  if ((e = build_neighbours(c, st, nl))) return e;
  DevScene s = scene_from_ctx(c);
  const int64_t npix = (int64_t)cams->n_views * cams->width * cams->height;
  const float inv_n = 1.0f / (float)npix;
  cudaMemsetAsync(loss, 0, sizeof(float), st);
  int g = (int)std::min<int64_t>((npix + kMaskThreads - 1) / kMaskThreads, (int64_t)c->sm_count * 16);
  k_mask_render<<<std::max(g, 1), kMaskThreads, 0, st>>>(s, cams->K, cams->c2w, cams->n_views, cams->width,
                                                         cams->height, gt, inv_n, mask_out, loss);
  // threads over the 6 nf bound of the neighbour entries; the real total is read on the device
  const int64_t n_ent = 6 * (int64_t)c->nf;
  g = (int)std::min<int64_t>((cams->n_views * n_ent + kMaskThreads - 1) / kMaskThreads, (int64_t)c->sm_count * 16);
  k_mask_grad<<<std::max(g, 1), kMaskThreads, 0, st>>>(s, cams->K, cams->c2w, cams->n_views, cams->width, cams->height,
                                                       gt, c->nbr, c->nbr_owner, c->nbr_start + c->nv, n_ent,
                                                       c->vstart, c->vcorner, c->F,
                                                       c->V, lambda * inv_n, 0.5f, 0.02f, grad_V);
  *nl += 2;
  return cudaGetLastError();
}

cudaError_t launch_mesh_regularizers(dt_ctx* c, float lambda_edge, float lambda_lap, float* grad_V, float* loss,
                                     cudaStream_t st, int* nl) {
  const int nv = c->nv, T = 256;
  const int g = std::max(1, std::min((nv + T - 1) / T, c->sm_count * 8));
  cudaError_t e;
  if ((e = build_neighbours(c, st, nl))) return e;
  cudaMemsetAsync(loss, 0, 2 * sizeof(float), st);
  int launches = 0;
  // L_edge through the vertex-normal chain: gN -> gVn, added to grad_V
  k_edge_reg<<<g, T, 0, st>>>(c->nrm, c->nbr_start, c->nbr, nv, lambda_edge, c->gN, loss);
  if ((e = launch_vertex_normal_backward(c, st))) return e;
  k_add_vec<<<g, T, 0, st>>>(c->gVn, nv, grad_V);
  launches += 5;
  // L_lap (delta in the gS scratch, free after the normal chain)
  k_lap_delta<<<g, T, 0, st>>>(c->V, c->nbr_start, c->nbr, nv, c->gS, loss + 1);
  k_lap_grad<<<g, T, 0, st>>>(c->gS, c->nbr_start, c->nbr, nv, lambda_lap, grad_V);
  launches += 2;
  *nl += launches;
  return cudaGetLastError();
}

DT_DEFINE_CHECK_READER(check_status_meshreg)

}  // namespace dt
