// mma.sync m16n8k8 TF32 throughput (register-resident fragments), full GPU.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int NACC>
__global__ void __launch_bounds__(512, 1) kern(float* out, int iters) {
  float d[NACC][4] = {};
  unsigned a[4], b[2];
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < 4; ++e) a[e] = __float_as_uint(1.0f + lane * 1e-3f + e);
  b[0] = __float_as_uint(0.5f);
  b[1] = __float_as_uint(0.25f + lane * 1e-4f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n) mma_tf32(d[n], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int n = 0; n < NACC; ++n) s += d[n][0] + d[n][1] + d[n][2] + d[n][3];
  if (s == 1.2345f) out[0] = s;
}

template <int NACC>
void run(int threads) {
  float* dptr;
  cudaMalloc(&dptr, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048;
  kern<NACC><<<sms, threads>>>(dptr, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<NACC><<<sms, threads>>>(dptr, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * sms * (threads / 32) * (double)iters * NACC * 16 * 8 * 8;
  printf("mma.sync tf32 m16n8k8, %d acc chains, %3d threads/SM: %.1f TFLOP/s\n", NACC, threads,
         flop / (ms * 1e-3) / 1e12);
}

int main() {
  for (int t : {128, 256, 512}) {
    run<4>(t);
    run<8>(t);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
