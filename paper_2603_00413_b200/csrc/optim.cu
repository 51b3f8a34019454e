// The optimisation step around the tracer: fused photometric losses and
// their colour gradient, absorption regularisers and the
// Adam / AdamUniform parameter updates.  Streaming kernels.
#include <cuda_runtime.h>

#include <algorithm>

#include "dt_internal.h"

namespace dt {
namespace {

DT_D float warp_sum(float x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(~0u, x, o);
  return x;
}

__global__ void k_loss_rt(const float* __restrict__ rgb, const float* __restrict__ tgt, const float* __restrict__ mask,
                          int64_t n, float inv_b, float lc, float lt, float* __restrict__ grad, float* __restrict__ loss) {
  float acc_c = 0.f, acc_t = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float3 ch = f3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
    float3 c = f3(tgt[3 * i], tgt[3 * i + 1], tgt[3 * i + 2]);
    float m = mask ? mask[i] : 1.0f;
    float3 we = (ch - c) * c;
    acc_c += m * dot(we, we);
    float3 g = we * c * (2.0f * lc);                       // d|(c^-c)*c|^2/dc^ = 2 (c^-c) c^2
    float nh = length(ch), nc = length(c);
    if (nh > 1e-6f && nc > 1e-6f) {
      float cs = dot(ch, c) / (nh * nc);
      float mu = (c.x + c.y + c.z) * (1.0f / 3.0f);
      float var = ((c.x - mu) * (c.x - mu) + (c.y - mu) * (c.y - mu) + (c.z - mu) * (c.z - mu)) * (1.0f / 3.0f);
      acc_t += m * ((1.0f - cs) * (1.0f - cs) - var);
      float3 dcs = c * (1.0f / (nh * nc)) - ch * (cs / (nh * nh));   // d cos / d c^
      g += dcs * (-2.0f * (1.0f - cs) * lt);
    }
    g = g * (m * inv_b);
    grad[3 * i] = g.x;
    grad[3 * i + 1] = g.y;
    grad[3 * i + 2] = g.z;
  }
  acc_c = warp_sum(acc_c);
  acc_t = warp_sum(acc_t);
  if (lane_id() == 0) {
    atomicAdd(loss, acc_c * inv_b);
    atomicAdd(loss + 1, acc_t * inv_b);
  }
}

// trilinear lookup on the caller's [R][R][R][3] grid (R11: zero outside the box); also
// returns the 8 corner nodes / weights for the scatter
DT_D bool grid_corners(const float* __restrict__ sig, int R, float3 lo, float3 hi, float3 p, int node[8], float w[8],
                       float3& val) {
  const float pp[3] = {p.x, p.y, p.z}, l[3] = {lo.x, lo.y, lo.z}, h[3] = {hi.x, hi.y, hi.z};
  int i0[3];
  float f[3];
  for (int a = 0; a < 3; ++a) {
    float g = (pp[a] - l[a]) / (h[a] - l[a]) * (float)(R - 1);
    if (g < 0.0f || g > (float)(R - 1)) { val = f3(0, 0, 0); return false; }
    i0[a] = min((int)floorf(g), R - 2);
    f[a] = g - (float)i0[a];
  }
  val = f3(0, 0, 0);
  for (int k = 0; k < 8; ++k) {
    int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
    w[k] = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
    node[k] = ((i0[2] + dz) * R + (i0[1] + dy)) * R + (i0[0] + dx);
    val += f3(sig[3 * node[k]], sig[3 * node[k] + 1], sig[3 * node[k] + 2]) * w[k];
  }
  return true;
}

DT_D void scatter(float* gsig, const int node[8], const float w[8], float3 g) {
  for (int k = 0; k < 8; ++k) {
    atomicAdd(gsig + 3 * node[k], g.x * w[k]);
    atomicAdd(gsig + 3 * node[k] + 1, g.y * w[k]);
    atomicAdd(gsig + 3 * node[k] + 2, g.z * w[k]);
  }
}

DT_D float sgnf(float x) { return x > 0.f ? 1.f : (x < 0.f ? -1.f : 0.f); }

__global__ void k_sigma_reg_grid(const float* __restrict__ sig, int R, float3 lo, float3 hi,
                                 const float* __restrict__ pts, const float* __restrict__ xi, int64_t n, float inv_n,
                                 float ls, float lv, float* __restrict__ gsig, float* __restrict__ loss) {
  float acc_s = 0.f, acc_v = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float3 v = f3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    float3 u = v + f3(xi[3 * i], xi[3 * i + 1], xi[3 * i + 2]);
    int nv[8], nu[8];
    float wv[8], wu[8];
    float3 mv, mu;
    bool iv = grid_corners(sig, R, lo, hi, v, nv, wv, mv);
    bool iu = grid_corners(sig, R, lo, hi, u, nu, wu, mu);
    float3 dd = mv - mu;
    acc_s += fabsf(dd.x) + fabsf(dd.y) + fabsf(dd.z);
    acc_v += dot(mv, mv);
    float3 s = f3(sgnf(dd.x), sgnf(dd.y), sgnf(dd.z)) * (ls * inv_n);
    if (iv) scatter(gsig, nv, wv, s + mv * (2.0f * lv * inv_n));
    if (iu) scatter(gsig, nu, wu, -s);
  }
  acc_s = warp_sum(acc_s);
  acc_v = warp_sum(acc_v);
  if (lane_id() == 0) {
    atomicAdd(loss, acc_s * inv_n);
    atomicAdd(loss + 1, acc_v * inv_n);
  }
}

// hash texture (R29) on the caller's [L][T][3] tables: value at p, and the scatter of g * w
struct HashTab {
  int L, log2;
  unsigned dense;
  int res[32];
  float3 lo, scl;   // unit-box coordinates u = (p - lo) * scl
};

DT_D uint32_t htab_index(const HashTab& h, int l, int x, int y, int z) {
  if ((h.dense >> l) & 1u) {
    const uint32_t n1 = (uint32_t)h.res[l] + 1u;
    return (uint32_t)x + n1 * ((uint32_t)y + n1 * (uint32_t)z);
  }
  return ((uint32_t)x ^ ((uint32_t)y * 2654435761u) ^ ((uint32_t)z * 805459861u)) & ((1u << h.log2) - 1u);
}

// visit(l_entry_offset, weight) for the 8 corners of every level; false outside the box
template <class Fn>
DT_D bool htab_visit(const HashTab& h, float3 p, Fn visit) {
  const float u[3] = {(p.x - h.lo.x) * h.scl.x, (p.y - h.lo.y) * h.scl.y, (p.z - h.lo.z) * h.scl.z};
  if (!(u[0] >= 0.f && u[0] <= 1.f && u[1] >= 0.f && u[1] <= 1.f && u[2] >= 0.f && u[2] <= 1.f)) return false;
  for (int l = 0; l < h.L; ++l) {
    const int N = h.res[l];
    int i[3];
    float f[3];
    for (int a = 0; a < 3; ++a) {
      const float g = u[a] * (float)N;
      i[a] = min((int)floorf(g), N - 1);
      f[a] = g - (float)i[a];
    }
    for (int k = 0; k < 8; ++k) {
      const int dx = k & 1, dy = (k >> 1) & 1, dz = k >> 2;
      const float w = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
      visit(((size_t)l << h.log2) + htab_index(h, l, i[0] + dx, i[1] + dy, i[2] + dz), w);
    }
  }
  return true;
}

__global__ void k_sigma_reg_hash(const float* __restrict__ sig, HashTab h, const float* __restrict__ pts,
                                 const float* __restrict__ xi, int64_t n, float inv_n, float ls, float lv,
                                 float* __restrict__ gsig, float* __restrict__ loss) {
  float acc_s = 0.f, acc_v = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float3 v = f3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    const float3 u = v + f3(xi[3 * i], xi[3 * i + 1], xi[3 * i + 2]);
    float3 mv = f3(0, 0, 0), mu = f3(0, 0, 0);
    htab_visit(h, v, [&](size_t e, float w) { mv += f3(sig[3 * e], sig[3 * e + 1], sig[3 * e + 2]) * w; });
    htab_visit(h, u, [&](size_t e, float w) { mu += f3(sig[3 * e], sig[3 * e + 1], sig[3 * e + 2]) * w; });
    const float3 dd = mv - mu;
    acc_s += fabsf(dd.x) + fabsf(dd.y) + fabsf(dd.z);
    acc_v += dot(mv, mv);
    const float3 s = f3(sgnf(dd.x), sgnf(dd.y), sgnf(dd.z)) * (ls * inv_n);
    const float3 gvv = s + mv * (2.0f * lv * inv_n);
    htab_visit(h, v, [&](size_t e, float w) {
      atomicAdd(gsig + 3 * e, gvv.x * w); atomicAdd(gsig + 3 * e + 1, gvv.y * w); atomicAdd(gsig + 3 * e + 2, gvv.z * w);
    });
    htab_visit(h, u, [&](size_t e, float w) {
      atomicAdd(gsig + 3 * e, -s.x * w); atomicAdd(gsig + 3 * e + 1, -s.y * w); atomicAdd(gsig + 3 * e + 2, -s.z * w);
    });
  }
  acc_s = warp_sum(acc_s);
  acc_v = warp_sum(acc_v);
  if (lane_id() == 0) {
    atomicAdd(loss, acc_s * inv_n);
    atomicAdd(loss + 1, acc_v * inv_n);
  }
}

// constant sigma: mu(x) = sigma everywhere, so L_mat = 0 and L_vol = |sigma|^2
__global__ void k_sigma_reg_const(const float* __restrict__ sig, float lv, float* __restrict__ gsig, float* __restrict__ loss) {
  float3 s = f3(sig[0], sig[1], sig[2]);
  loss[0] = 0.f;
  loss[1] = dot(s, s);
  gsig[0] += 2.f * lv * s.x;
  gsig[1] += 2.f * lv * s.y;
  gsig[2] += 2.f * lv * s.z;
}

__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v,
                       int64_t n, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                       const float* __restrict__ vshared, float lo, float hi, const int* __restrict__ skip,
                       const int* __restrict__ tdev) {
  if (skip && *skip) return;                               // the step's forward overflowed: no update
  if (tdev) {                                              // the step count lives on the device (graphs)
    const float t = (float)*tdev;
    bc1 = 1.0f - powf(b1, t);
    bc2 = 1.0f - powf(b2, t);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float gi = g[i] + wd * p[i];                           // torch.optim.Adam weight decay
    float mi = b1 * m[i] + (1.f - b1) * gi;
    m[i] = mi;
    float vi;
    if (vshared) {
      vi = *vshared;                                       // AdamUniform: one statistic per block
    } else {
      vi = b2 * v[i] + (1.f - b2) * gi * gi;
      v[i] = vi;
    }
    p[i] = fminf(fmaxf(p[i] - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps), lo), hi);
  }
}

__global__ void k_max_sq(const float* __restrict__ p, const float* __restrict__ g, int64_t n, float wd,
                         unsigned* __restrict__ out) {
  float mx = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float gi = g[i] + wd * p[i];
    mx = fmaxf(mx, gi * gi);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, o));
  if (lane_id() == 0) atomicMax(out, __float_as_uint(mx));   // non-negative floats order as uints
}

__global__ void k_uniform_v(float* __restrict__ v, const unsigned* __restrict__ mx, float b2, const int* __restrict__ skip) {
  if (skip && *skip) return;
  v[0] = b2 * v[0] + (1.f - b2) * __uint_as_float(*mx);
}

__global__ void k_step_bump(int* __restrict__ t, const int* __restrict__ skip) {
  if (!(skip && *skip)) *t += 1;
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

cudaError_t launch_loss_rt(const float* rgb, const float* tgt, const float* mask, int64_t n, float lc, float lt,
                           float* grad, float* loss, cudaStream_t st) {
  cudaMemsetAsync(loss, 0, 2 * sizeof(float), st);
  if (n > 0) k_loss_rt<<<grid_for(n), 256, 0, st>>>(rgb, tgt, mask, n, 1.0f / (float)n, lc, lt, grad, loss);
  return cudaGetLastError();
}

cudaError_t launch_sigma_reg(const dt_absorption* ab, const float* pts, const float* xi, int64_t n, float ls, float lv,
                             float* gsig, float* loss, cudaStream_t st) {
  cudaMemsetAsync(loss, 0, 2 * sizeof(float), st);
  if (ab->kind == DT_ABS_CONST) {
    k_sigma_reg_const<<<1, 1, 0, st>>>(ab->sigma, lv, gsig, loss);
  } else if (ab->kind == DT_ABS_HASH && n > 0) {
    HashTab h{};
    h.L = ab->levels;
    h.log2 = ab->log2_size;
    for (int l = 0; l < ab->levels; ++l) {
      h.res[l] = ab->level_res[l];
      const double n1 = ab->level_res[l] + 1.0;
      if (n1 * n1 * n1 <= (double)(1u << ab->log2_size)) h.dense |= 1u << l;
    }
    h.lo = f3(ab->box_lo[0], ab->box_lo[1], ab->box_lo[2]);
    h.scl = f3(1.0f / (ab->box_hi[0] - ab->box_lo[0]), 1.0f / (ab->box_hi[1] - ab->box_lo[1]),
               1.0f / (ab->box_hi[2] - ab->box_lo[2]));
    k_sigma_reg_hash<<<grid_for(n), 256, 0, st>>>(ab->sigma, h, pts, xi, n, 1.0f / (float)n, ls, lv, gsig, loss);
  } else if (n > 0) {
    k_sigma_reg_grid<<<grid_for(n), 256, 0, st>>>(ab->sigma, ab->res, f3(ab->box_lo[0], ab->box_lo[1], ab->box_lo[2]),
                                                 f3(ab->box_hi[0], ab->box_hi[1], ab->box_hi[2]), pts, xi, n,
                                                 1.0f / (float)n, ls, lv, gsig, loss);
  }
  return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, int64_t n, const dt_adam* c, unsigned* scratch,
                        cudaStream_t st, int* nl) {
  const int t = c->step_device ? 1 : c->step;            // (device step: read by the kernel)
  float bc1 = 1.0f - powf(c->beta1, (float)t), bc2 = 1.0f - powf(c->beta2, (float)t);
  if (c->uniform) {
    cudaMemsetAsync(scratch, 0, sizeof(unsigned), st);
    k_max_sq<<<grid_for(n), 256, 0, st>>>(p, g, n, c->weight_decay, scratch);
    k_uniform_v<<<1, 1, 0, st>>>(v, scratch, c->beta2, c->skip_if);
    k_adam<<<grid_for(n), 256, 0, st>>>(p, g, m, v, n, c->lr, c->beta1, c->beta2, c->eps, c->weight_decay, bc1, bc2, v,
                                        c->clamp_lo, c->clamp_hi, c->skip_if, c->step_device);
    *nl += 3;
  } else {
    k_adam<<<grid_for(n), 256, 0, st>>>(p, g, m, v, n, c->lr, c->beta1, c->beta2, c->eps, c->weight_decay, bc1, bc2,
                                        nullptr, c->clamp_lo, c->clamp_hi, c->skip_if, c->step_device);
    *nl += 1;
  }
  if (c->step_device) {
    k_step_bump<<<1, 1, 0, st>>>(c->step_device, c->skip_if);
    *nl += 1;
  }
  return cudaGetLastError();
}

DT_DEFINE_CHECK_READER(check_status_optim)

}  // namespace dt
