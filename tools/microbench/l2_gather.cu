// Scattered 16-B access microbenchmark: the peaks of the texture walks' roofline (bench.py,
// DESIGN.md §5).  The sigma-grid / hash-texture walks fetch 8 corners per cell visit with
// scattered float4 loads and the backward scatters 8 float4 atomics (RED.E.ADD.F32x4) per cell
// visit.  Their limit is the rate at which the L2 serves scattered 32-B sectors, not HBM bytes:
// this program measures that rate for
//   gather: float4 loads (ld.global.cg: served by the L2) at pseudo-random indices,
//   red:    float4 atomicAdd at pseudo-random indices (no return value -> RED),
// each also "coalesced" (a warp's 32 lanes on 32 consecutive float4: the L2's ceiling for the
// same operation), over a table of 8 MB (one hash level / the C4 sigma grid) and 128 MB (the 16-level hash
// table set), all SMs, 8 accesses in flight per thread.  Prints one JSON line: operations per
// second (Gop/s) and the payload bandwidth (16 B per op) of each.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2_gather tools/microbench/l2_gather.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned mix(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// coalesced: a warp's 32 lanes access 32 consecutive float4 (512 B) at a hashed warp-aligned
// base -- the ceiling of the L2 (the same L2 slices, full sectors, no address scatter)
template <bool COAL>
__device__ __forceinline__ unsigned index(unsigned t, unsigned i, unsigned mask) {
  if (!COAL) return mix(t * 8191u + i) & mask;
  return ((mix((t >> 5) * 8191u + i) << 5) + (t & 31u)) & mask;
}

template <bool COAL>
__global__ void k_gather(const float4* __restrict__ p, unsigned mask, int iters, float* out) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(p + index<COAL>(t, (unsigned)(i * 8 + k), mask));
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z;
  }
  if (acc == 1234.5f) *out = acc;
}

template <bool COAL>
__global__ void k_red(float4* __restrict__ p, unsigned mask, int iters) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  const float4 one = make_float4(1e-9f, 1e-9f, 1e-9f, 0.f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(p + index<COAL>(t, (unsigned)(i * 8 + k), mask), one);
  }
}

static double best_ms(void (*launch)(void*), void* ctx) {
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  launch(ctx);
  cudaDeviceSynchronize();
  std::vector<float> ms;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch(ctx);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float m = 0.f;
    cudaEventElapsedTime(&m, a, e);
    ms.push_back(m);
  }
  std::sort(ms.begin(), ms.end());
  return ms[0];
}

struct Ctx { float4* p; unsigned mask; int iters; float* out; int grid; bool red, coal; };
static void launch(void* v) {
  Ctx* c = (Ctx*)v;
  if (c->red) {
    if (c->coal) k_red<true><<<c->grid, 256>>>(c->p, c->mask, c->iters);
    else k_red<false><<<c->grid, 256>>>(c->p, c->mask, c->iters);
  } else {
    if (c->coal) k_gather<true><<<c->grid, 256>>>(c->p, c->mask, c->iters, c->out);
    else k_gather<false><<<c->grid, 256>>>(c->p, c->mask, c->iters, c->out);
  }
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  const size_t big = (size_t)128 << 20;
  float4* p;
  float* out;
  cudaMalloc(&p, big);
  cudaMalloc(&out, 4);
  cudaMemset(p, 0, big);
  const int grid = sm * 8, iters = 64;
  const double ops = (double)grid * 256 * iters * 8;
  double r[2][2], rc[2];
  const size_t sizes[2] = {(size_t)8 << 20, big};
  for (int s = 0; s < 2; ++s)
    for (int red = 0; red < 2; ++red) {
      Ctx c{p, (unsigned)(sizes[s] / 16 - 1), iters, out, grid, red != 0, false};
      r[s][red] = ops / (best_ms(launch, &c) * 1e-3) / 1e9;
    }
  for (int red = 0; red < 2; ++red) {
    Ctx c{p, (unsigned)(sizes[0] / 16 - 1), iters, out, grid, red != 0, true};
    rc[red] = ops / (best_ms(launch, &c) * 1e-3) / 1e9;
  }
  printf("{\"gpu\": \"%s\", \"gather_8mb_gops\": %.2f, \"red_8mb_gops\": %.2f, \"gather_128mb_gops\": %.2f, "
         "\"red_128mb_gops\": %.2f, \"gather_8mb_gbs\": %.1f, \"red_8mb_gbs\": %.1f, \"gather_128mb_gbs\": %.1f, "
         "\"red_128mb_gbs\": %.1f, \"gather_coalesced_gops\": %.2f, \"red_coalesced_gops\": %.2f, \"method\": \"float4 ld.global.cg / atomicAdd(float4) at hashed indices, %d blocks x 256 "
         "threads x %d x 8 accesses, best of 5; GB/s = 16 B payload per op; coalesced: 32 consecutive float4 per warp "
         "access, 8 MB table (the L2 ceiling)\"}\n",
         pr.name, r[0][0], r[0][1], r[1][0], r[1][1], r[0][0] * 16, r[0][1] * 16, r[1][0] * 16, r[1][1] * 16, rc[0], rc[1], grid, iters);
  cudaFree(p);
  cudaFree(out);
  return 0;
}
