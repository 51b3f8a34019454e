// L2 read-bandwidth microbenchmark (MEASURED_PEAKS has no L2 figure).
// A buffer that fits in the 126 MB L2 is read repeatedly with 128-bit loads that bypass L1
// (ld.global.cg); bytes / time after warm-up = sustained L2 -> SM read bandwidth.  Also the
// same kernel on a buffer far larger than L2 (HBM) for reference.  Prints one JSON line.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

__global__ void k_read(const float4* __restrict__ p, size_t n, int reps, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      float4 v = __ldcg(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1234.5f) *out = acc;   // keep the loads alive
}

double run(size_t bytes, int reps) {
  size_t n = bytes / 16;
  float4* p;
  float* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(p, 0, bytes);
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  dim3 g(sm * 8), b(256);
  k_read<<<g, b>>>(p, n, 1, out);      // warm (fills L2 for the small buffer)
  cudaEvent_t a, e;
  cudaEventCreate(&a);
  cudaEventCreate(&e);
  std::vector<float> ms;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(a);
    k_read<<<g, b>>>(p, n, reps, out);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float m = 0.f;
    cudaEventElapsedTime(&m, a, e);
    ms.push_back(m);
  }
  std::sort(ms.begin(), ms.end());
  cudaFree(p);
  cudaFree(out);
  return (double)bytes * reps / (ms[0] * 1e-3) / 1e9;
}

int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  double l2 = run((size_t)48 << 20, 40);          // 48 MB: L2-resident
  double hbm = run((size_t)8 << 30, 2);           // 8 GB: streams from HBM
  printf("{\"gpu\": \"%s\", \"l2_bytes\": %d, \"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, "
         "\"method\": \"ld.global.cg float4 reads, best of 5, 48 MB x 40 passes (L2) / 8 GB x 2 (HBM)\"}\n",
         pr.name, pr.l2CacheSize, l2, hbm);
  return 0;
}
