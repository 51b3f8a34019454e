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
                           const int* __restrict__ F, int nv, const int* __restrict__ start, int* __restrict__ nbr) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    int nb[kMaxValence];
    const int n = collect_neighbours(vstart, corner, F, v, nb);
    for (int q = 0; q < n; ++q) nbr[start[v] + q] = nb[q];
  }
}

DT_D float warp_sum(float x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
  return x;
}

// L_edge: loss over edges (i < j), and dL/dn_i = (1/|E|) sum_{j in N(i)} -2 (1 - n_i.n_j) n_j
// written into gN (the vertex-normal chain then maps it to dV)
__global__ void k_edge_reg(const float4* __restrict__ nrm, const int* __restrict__ start, const int* __restrict__ nbr,
                           int nv, float lambda, float4* __restrict__ gN, float* __restrict__ loss) {
  const float inv_e = 2.0f / (float)max(start[nv], 1);     // |E| = (sum of valences) / 2
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const float3 ni = f3(nrm[i]);
    float3 g = f3(0, 0, 0);
    for (int q = start[i]; q < start[i + 1]; ++q) {
      const int j = nbr[q];
      const float3 nj = f3(nrm[j]);
      const float d = 1.0f - dot(ni, nj);
      if (j > i) acc += d * d;
      g += nj * (-2.0f * d);
    }
    gN[i] = f4(g * (lambda * inv_e), 0.f);
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

}  // namespace

cudaError_t launch_mesh_regularizers(dt_ctx* c, float lambda_edge, float lambda_lap, float* grad_V, float* loss,
                                     cudaStream_t st, int* nl) {
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
  // neighbour lists of the current snapshot; the total is bounded by the 2 * 3nf corner pairs
  const int64_t nmax = (int64_t)6 * c->nf;
  if (c->nbr_cap < nmax) {
    cudaFree(c->nbr);
    c->nbr = nullptr;
    c->nbr_cap = 0;
    if ((e = cudaMalloc(&c->nbr, (size_t)nmax * sizeof(int)))) return e;
    c->nbr_cap = nmax;
  }
  cudaMemsetAsync(loss, 0, 2 * sizeof(float), st);
  k_nbr_count<<<g, T, 0, st>>>(c->vstart, c->vcorner, c->F, nv, c->nbr_cnt);
  k_nbr_scan<<<1, 1024, 0, st>>>(c->nbr_cnt, nv, c->nbr_start);
  k_nbr_fill<<<g, T, 0, st>>>(c->vstart, c->vcorner, c->F, nv, c->nbr_start, c->nbr);
  int launches = 3;
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

}  // namespace dt
