// SYRK-phase microbenchmark: the pair kernel's trailing update of panel 0
// (columns >= 32 of a k=200 packed system, two systems per CTA, 15 warps,
// dynamic warp-tile counter), one CTA per SM, repeated.  Reports useful
// FMA/clk/SM for tile variants.
#include "fmap_solver.cu"
#include <cstdio>

using namespace fmap;

template <int VARIANT>
__global__ void __launch_bounds__(512, 1) syrk_kernel(long long* out, int reps) {
  extern __shared__ __align__(16) float smem[];
  const int K4 = 200, Rp = 204;
  const int SYS = pair_stride_floats(K4);
  int* counter = reinterpret_cast<int*>(smem + 2 * SYS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 2 * SYS; e += 512) smem[e] = 1e-3f * ((e * 7) % 13);
  if (tid == 0) *counter = 0;
  __syncthreads();
  const Panel P(0, Rp);
  const int cs = 32;
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (warp != 15) {
      if (VARIANT == 0) {  // solver's 64x16 warp tiles, 8x4 per lane
        const int ncb = (K4 - cs + 15) >> 4;
        int W = 0;
        for (int u = 0; u < ncb; ++u) W += (Rp - (cs + 16 * u) + 63) >> 6;
        while (true) {
          int w = 0;
          if (lane == 0) w = atomicAdd(counter, 1);
          w = __shfl_sync(0xffffffffu, w, 0);
          if (w >= 2 * W) break;
          const int h = w >= W;
          w -= h * W;
          int cb = cs, nrb = (Rp - cb + 63) >> 6;
          while (w >= nrb) {
            w -= nrb;
            cb += 16;
            nrb = (Rp - cb + 63) >> 6;
          }
          syrk_warp_tile<true>(smem + h * SYS, Rp, K4, P, 16, cb, cb + (w << 6), 0, 0, lane);
        }
      } else if (VARIANT == 1) {  // 32x16 warp tiles, 4x4 per lane
        const int ncb = (K4 - cs + 15) >> 4;
        int W = 0;
        for (int u = 0; u < ncb; ++u) W += (Rp - (cs + 16 * u) + 31) >> 5;
        const int lr = lane & 7, lc = lane >> 3;
        while (true) {
          int w = 0;
          if (lane == 0) w = atomicAdd(counter, 1);
          w = __shfl_sync(0xffffffffu, w, 0);
          if (w >= 2 * W) break;
          const int h = w >= W;
          w -= h * W;
          int cb = cs, nrb = (Rp - cb + 31) >> 5;
          while (w >= nrb) {
            w -= nrb;
            cb += 16;
            nrb = (Rp - cb + 31) >> 5;
          }
          const int r0 = cb + (w << 5) + (lr << 2), c0 = cb + (lc << 2);
          if (c0 < K4 && r0 < Rp && r0 >= c0) syrk_tile<true>(smem + h * SYS, Rp, P, 16, r0, c0);
        }
      } else {  // mma.sync 3xTF32 32 cols x 64 rows
        const int ncb = (K4 - cs + 31) >> 5;
        int W = 0;
        for (int u = 0; u < ncb; ++u) W += (Rp - (cs + 32 * u) + 63) >> 6;
        while (true) {
          int w = 0;
          if (lane == 0) w = atomicAdd(counter, 1);
          w = __shfl_sync(0xffffffffu, w, 0);
          if (w >= 2 * W) break;
          const int h = w >= W;
          w -= h * W;
          int cb = cs, nrb = (Rp - cb + 63) >> 6;
          while (w >= nrb) {
            w -= nrb;
            cb += 32;
            nrb = (Rp - cb + 63) >> 6;
          }
          syrk_mma_block<2, 8>(smem + h * SYS, Rp, K4, P, cb + (w << 6), cb, lane);
        }
      }
    }
    __syncthreads();
    if (tid == 0) *counter = 0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

template <int V>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = (2 * pair_stride_floats(200) + 64) * 4;
  cudaFuncSetAttribute(syrk_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  syrk_kernel<V><<<148, 512, smem>>>(d, 20);
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (long long v : h) mx = v > mx ? v : mx;
  const double useful = 2.0 * (172.0 * 173.0 / 2.0 + 172.0 * 4) * 16;  // two systems, rows incl. aug
  printf("%-34s %6lld cycles per SYRK(0) of 2 systems -> %.1f useful FMA/clk/SM  (%s)\n", name, mx,
         useful / mx, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("64x16 warp tiles, 8x4/lane (solver)");
  run<1>("32x16 warp tiles, 4x4/lane");
  run<2>("mma.sync 3xTF32 32x64");
  return 0;
}
