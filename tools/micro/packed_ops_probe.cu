// Microbenchmark (developer tool, not product): lane-op throughput of the packed FP32x2 ops the P2P
// kernel issues (FFMA2, FMUL2, FADD2) and of their mixes, 32 warps per SM, 8 independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, float a) {
  constexpr int ILP = 8;
  float2 acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f + 1.f);
  const float2 m = make_float2(a, a * 0.999f), c = make_float2(1e-7f, -2e-7f);
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (OP == 0) acc[i] = __ffma2_rn(acc[i], m, c);
        if (OP == 1) acc[i] = __fmul2_rn(acc[i], m);
        if (OP == 2) acc[i] = __fadd2_rn(acc[i], c);
        if (OP == 3) {  // 3 of 11 as FMUL2 (the P2P mix)
          if ((u * ILP + i) % 11 < 3) acc[i] = __fmul2_rn(acc[i], m);
          else acc[i] = __ffma2_rn(acc[i], m, c);
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char* name) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int warps = 32, iters = 4096;
  float* d;
  cudaMalloc(&d, (size_t)nsm * warps * 32 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<OP><<<nsm, 32 * warps>>>(d, 16, 0.9999f);
  cudaEventRecord(e0);
  k<OP><<<nsm, 32 * warps>>>(d, iters, 0.9999f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double lane_ops = (double)nsm * warps * 32 * iters * 8 * 8 * 2;
  printf("%-22s %.1f G lane-ops/s (%.2f per SM-clock at 1.965 GHz)\n", name, lane_ops / ms / 1e6,
         lane_ops / ms / 1e6 / (nsm * 1.965));
  cudaFree(d);
}
int main() {
  run<0>("FFMA2");
  run<1>("FMUL2");
  run<2>("FADD2");
  run<3>("8 FFMA2 : 3 FMUL2");
  return 0;
}
