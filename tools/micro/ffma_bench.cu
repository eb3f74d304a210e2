// FFMA throughput microbenchmark: 8x4 and 8x8 outer-product register tiles with
// operands (a) in registers, (b) from shared memory (LDS.128 per step), full SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int TR, int TC, bool LDS>
__global__ void __launch_bounds__(512, 1) kern(float* out, int iters) {
  __shared__ __align__(16) float sm[4096];
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) sm[e] = 1e-3f * (e % 97);
  __syncthreads();
  float acc[TR][TC];
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) acc[a][b] = 0.f;
  const int lane = threadIdx.x & 31;
  const float* pa = sm + 4 * (lane & 7);
  const float* pb = sm + 1024 + 4 * (lane >> 3);
  float xr[TR], yr[TC];
#pragma unroll
  for (int a = 0; a < TR; ++a) xr[a] = 0.5f + a * lane;
#pragma unroll
  for (int b = 0; b < TC; ++b) yr[b] = 0.25f + b;
  for (int it = 0; it < iters; ++it) {
    if (LDS) {
      const int o = (it & 31) * 32;
#pragma unroll
      for (int a = 0; a < TR; a += 4) {
        const float4 v = *reinterpret_cast<const float4*>(pa + o + 128 * (a / 4));
        xr[a] = v.x; xr[a + 1] = v.y; xr[a + 2] = v.z; xr[a + 3] = v.w;
      }
#pragma unroll
      for (int b = 0; b < TC; b += 4) {
        const float4 v = *reinterpret_cast<const float4*>(pb + o + 16 * (b / 4));
        yr[b] = v.x; yr[b + 1] = v.y; yr[b + 2] = v.z; yr[b + 3] = v.w;
      }
    }
#pragma unroll
    for (int a = 0; a < TR; ++a)
#pragma unroll
      for (int b = 0; b < TC; ++b) acc[a][b] = fmaf(xr[a], yr[b], acc[a][b]);
    if (!LDS) {
#pragma unroll
      for (int a = 0; a < TR; ++a) xr[a] += 1e-7f;  // keep the loop honest
    }
  }
  float s = 0.f;
#pragma unroll
  for (int a = 0; a < TR; ++a)
#pragma unroll
    for (int b = 0; b < TC; ++b) s += acc[a][b];
  if (s == 1.2345f) out[0] = s;
}

template <int TR, int TC, bool LDS>
void run(const char* name, int threads) {
  float* d;
  cudaMalloc(&d, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  kern<TR, TC, LDS><<<sms, threads>>>(d, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<TR, TC, LDS><<<sms, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma = (double)sms * threads * iters * TR * TC;
  printf("%-28s threads=%3d: %.1f TFLOP/s  (%.1f FMA/clk/SM at 1.965 GHz)\n", name, threads,
         2 * fma / (ms * 1e-3) / 1e12, fma / (ms * 1e-3) / 1.965e9 / sms);
}

int main() {
  for (int t : {256, 512}) {
    run<8, 4, false>("8x4 regs", t);
    run<8, 4, true>("8x4 + LDS.128 operands", t);
    run<8, 8, false>("8x8 regs", t);
    run<8, 8, true>("8x8 + LDS.128 operands", t);
    run<4, 4, true>("4x4 + LDS.128 operands", t);
  }
  return 0;
}
