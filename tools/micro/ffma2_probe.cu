// Microbenchmark (developer tool, not product): throughput of packed FP32x2 FFMA2 vs scalar FFMA on
// sm_100a as a function of independent chains per thread (ILP) and resident warps per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, bool PACKED>
__global__ void k(float* out, int iters, float a) {
  float2 acc2[ILP];
  float acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { acc2[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f); acc[i] = acc2[i].x; }
  const float2 m = make_float2(a, a * 0.999f), c = make_float2(1e-7f, 2e-7f);
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (PACKED) acc2[i] = __ffma2_rn(acc2[i], m, c);
        else acc[i] = fmaf(acc[i], m.x, c.x);
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += PACKED ? acc2[i].x + acc2[i].y : acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP, bool PACKED>
void run(int warps_per_sm) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, (size_t)nsm * warps_per_sm * 32 * 4);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<ILP, PACKED><<<nsm, 32 * warps_per_sm>>>(d, 16, 0.9999f);
  cudaEventRecord(e0);
  k<ILP, PACKED><<<nsm, 32 * warps_per_sm>>>(d, iters, 0.9999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = (double)nsm * warps_per_sm * 32 * iters * 8 * ILP * (PACKED ? 2 : 1);
  printf("%s ILP=%d warps/SM=%2d: %.1f TFLOP/s\n", PACKED ? "FFMA2" : "FFMA ", ILP, warps_per_sm, 2 * fmas / ms / 1e9);
  cudaFree(d);
}
int main() {
  for (int w : {4, 8, 16, 32}) {
    run<1, true>(w); run<2, true>(w); run<4, true>(w); run<8, true>(w);
    run<1, false>(w); run<2, false>(w); run<4, false>(w); run<8, false>(w);
  }
  return 0;
}
