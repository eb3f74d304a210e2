// Microbenchmark: pieces of the solver's diag16 on one warp in isolation (clock64).
#include "fmap_solver.cu"
#include <cstdio>

using namespace fmap;

__global__ void bench(long long* out, int reps, int nwarps_busy, int variant, int diag_warp, int lds_busy) {
  extern __shared__ __align__(16) float smem[];
  const int Rp = 20, K4 = 16;
  float* A = smem;
  float* scr = smem + 2048;
  float* sinv = scr + 128;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = threadIdx.x; c < K4; c += blockDim.x)
    for (int r = (c & ~3); r < Rp; ++r)
      A[col_off(c, Rp) - (c & ~3) + r] = (r < K4) ? (r == c ? 17.f : 1.f / (1 + abs(r - c))) : 0.f;
  __syncthreads();
  float pm = 1e30f;
  unsigned bad = 0;
  long long t0 = clock64();
  if (warp == diag_warp) {
    const Panel P(0, Rp);
    for (int it = 0; it < reps; ++it) {
      if (variant == 0) {
        diag16<true>(A, Rp, 0, 16, scr, sinv, lane, pm, bad);
      } else if (variant == 3) {
        diag16_shfl<true>(A, Rp, 0, 16, sinv, lane, pm, bad);
      } else if (variant == 4) {
        diag16_x1<true>(A, Rp, 0, 16, sinv, scr + 64 + 16 * (lane >> 4), lane, pm, bad);
      } else if (variant == 5) {
        diag16_b4<true>(A, Rp, 0, 16, sinv, scr + 256 + 64 * (lane >> 4), lane, pm, bad);
      } else if (variant == 1) {  // two register-only chol8
        float t[36], inv[8];
#pragma unroll
        for (int e = 0; e < 36; ++e) t[e] = A[e] + (e == 0 || e == 2 || e == 5 || e == 9 || e == 14 || e == 20 || e == 27 || e == 35 ? 40.f : 0.f);
        chol8(t, inv, pm, bad);
        chol8(t, inv, pm, bad);
#pragma unroll
        for (int e = 0; e < 36; ++e) if (lane == e) A[100 + e] = t[e] + inv[e & 7];
      } else if (variant == 2) {  // block load/store only
        float t[36];
        ld_tri8<true>(A, P, 0, 0, 16, t);
        if (lane == 0) st_tri8<true>(A, P, 0, 0, 16, t);
        ld_tri8<true>(A, P, 8, 8, 16, t);
        if (lane == 0) st_tri8<true>(A, P, 8, 8, 16, t);
        __syncwarp();
      }
    }
  } else if (!lds_busy) {
    float a = lane, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    for (int it = 0; it < reps * 400; ++it) {
      c0 = fmaf(a, b, c0); c1 = fmaf(a, b, c1); c2 = fmaf(a, b, c2); c3 = fmaf(a, b, c3);
    }
    if (c0 + c1 + c2 + c3 == 1.2345f) out[100] = 1;
  } else {
    // SYRK-like: 2 LDS.128 + 16 FFMA per step on a 4x4 register tile
    float acc[16] = {};
    const float* base = smem + 4096 + ((lane & 7) * 4);
    for (int it = 0; it < reps * 100; ++it) {
      const float4 x = *reinterpret_cast<const float4*>(base + (it & 63) * 36);
      const float4 y = *reinterpret_cast<const float4*>(base + (it & 63) * 36 + 16 * (lane >> 3));
      const float xr[4] = {x.x, x.y, x.z, x.w}, yr[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u * 4 + v] = fmaf(xr[u], yr[v], acc[u * 4 + v]);
    }
    float t = 0.f;
    for (int e = 0; e < 16; ++e) t += acc[e];
    if (t == 1.2345f) out[100] = 1;
  }
  long long t1 = clock64();
  if (warp == diag_warp && lane == 0) { out[0] = (t1 - t0) / reps; out[1] = bad; }
}


// correctness: x1 vs b4 on the same SPD block (both systems' halves)
__global__ void check(float* out) {
  __shared__ __align__(16) float A1[512], A2[512], s1[32], s2[32], xb[256];
  const int Rp = 20, K4 = 16, lane = threadIdx.x;
  for (int c = 0; c < K4; ++c)
    for (int r = (c & ~3) + lane; r < Rp; r += 32) {
      float v = (r < K4) ? (r == c ? 17.f : 1.f / (1 + abs(r - c)) + 0.01f * ((r * 7 + c * 3) % 5)) : 0.f;
      if (r < c) v = 0.f;
      A1[col_off(c, Rp) - (c & ~3) + r] = v;
      A2[col_off(c, Rp) - (c & ~3) + r] = v;
    }
  __syncwarp();
  float pm = 1e30f;
  unsigned bad = 0;
  diag16_x1<true>(A1, Rp, 0, 16, s1, xb + 16 * (lane >> 4), lane, pm, bad);
  diag16_b4<true>(A2, Rp, 0, 16, s2, xb + 64 + 64 * (lane >> 4), lane, pm, bad);
  __syncwarp();
  float e = 0.f;
  for (int c = 0; c < K4; ++c)
    for (int r = c; r < K4; ++r) e = fmaxf(e, fabsf(A1[col_off(c, Rp) - (c & ~3) + r] - A2[col_off(c, Rp) - (c & ~3) + r]));
  for (int c = 0; c < K4; ++c) e = fmaxf(e, fabsf(s1[c] - s2[c]));
  if (lane == 0) out[0] = e;
}

int main() {
  {
    float* d; cudaMalloc(&d, 4);
    check<<<1, 32>>>(d);
    float h; cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("x1 vs b4 max abs diff: %g\n", h);
  }
  long long* d; cudaMalloc(&d, 1024 * 8);
  long long h[2];
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  const char* names[] = {"diag16(repl)", "2x chol8 (regs)", "ld/st", "diag16_shfl", "diag16_x1", "diag16_b4"};
  for (int v : {4, 5})
    for (int nw : {1, 8, 16})
      for (int lb : {0, 1}) {
        if (nw == 1 && lb) continue;
        bench<<<1, 32 * nw, 100000>>>(d, 50, nw - 1, v, nw - 1, lb);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%-14s warps=%2d busy=%s: %lld cycles/call\n", names[v], nw, lb ? "LDS+FFMA" : "FFMA    ", h[0]);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
