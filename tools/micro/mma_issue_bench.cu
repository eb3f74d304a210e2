// tcgen05.mma (kind::tf32, M=128) issue / completion latency from one thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 13) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
               "l"(a), "l"(b), "r"(id) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  } while (!ok);
}

template <int NMMA, int N>
__global__ void kern(long long* out) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int e = threadIdx.x; e < 256 * 16 * 2; e += blockDim.x) sm[e] = 0.01f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t base = su32(sm);
    long long best_i = 1ll << 60, best_c = 1ll << 60;
    for (int it = 0; it < 20; ++it) {
      const long long t0 = clock64();
#pragma unroll
      for (int m = 0; m < NMMA; ++m) mma_tf32(tb, sdesc(base + (m & 3) * 256), sdesc(base + 8192 + (m & 3) * 256), idesc_tf32(N));
      commit(&bar);
      const long long t1 = clock64();
      mwait(&bar, it & 1);
      const long long t2 = clock64();
      if (it > 2) {
        if (t1 - t0 < best_i) best_i = t1 - t0;
        if (t2 - t0 < best_c) best_c = t2 - t0;
      }
    }
    out[2 * blockIdx.x] = best_i;
    out[2 * blockIdx.x + 1] = best_c;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}

template <int NMMA, int N>
void run(int ctas) {
  long long* d;
  cudaMalloc(&d, 16 * 1024);
  auto fn = kern<NMMA, N>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  fn<<<ctas, 128, 100000>>>(d);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%2d MMAs N=%3d, %3d CTAs: issue %5lld cycles, issue+complete %5lld  (%s)\n", NMMA, N, ctas, h[0], h[1],
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// NMMA MMAs split over W issuing warps (lane 0 each), one commit per warp.
template <int NMMA, int N, int W>
__global__ void kernW(long long* out) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tslot;
  __shared__ long long tstart;
  for (int e = threadIdx.x; e < 256 * 16 * 2; e += blockDim.x) sm[e] = 0.01f;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 8; ++w) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long best = 1ll << 60;
  for (int it = 0; it < 20; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) tstart = clock64();
    __syncthreads();
    if (warp < W && lane == 0) {
      const uint32_t base = su32(sm);
#pragma unroll
      for (int m = 0; m < NMMA / W; ++m)
        mma_tf32(tb + 16 * warp, sdesc(base + (m & 3) * 256), sdesc(base + 8192 + (m & 3) * 256), idesc_tf32(N));
      commit(&bar[warp]);
      mwait(&bar[warp], it & 1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && it > 2) {
      const long long dt = clock64() - tstart;
      if (dt < best) best = dt;
    }
  }
  if (threadIdx.x == 0) out[0] = best;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb));
}

template <int NMMA, int N, int W>
void runW() {
  long long* d;
  cudaMalloc(&d, 64);
  auto fn = kernW<NMMA, N, W>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  fn<<<1, 256, 100000>>>(d);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%2d MMAs N=%3d over %d warps: issue->all complete %5lld cycles (%s)\n", NMMA, N, W, h,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  runW<12, 16, 1>();
  runW<12, 16, 2>();
  runW<12, 16, 4>();
  runW<12, 16, 6>();
  runW<24, 16, 8>();
  run<1, 16>(1);
  run<6, 16>(1);
  run<12, 16>(1);
  run<12, 64>(1);
  run<6, 176>(1);
  run<12, 176>(1);
  run<12, 16>(296);
  return 0;
}
