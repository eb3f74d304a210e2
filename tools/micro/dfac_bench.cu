// Isolated latency of 16x16 diagonal-block Cholesky variants on one warp (the rest
// of the GPU idle): clock64 cycles per factorization.
#include <cstdio>
#include <cuda_runtime.h>

constexpr unsigned kFull = 0xffffffffu;
__device__ __forceinline__ float rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// (A) lane per row, shuffle broadcast of each column (current solver)
__device__ __forceinline__ void dfA(float (&a)[16], float& inv, int g) {
  float dnext = __shfl_sync(kFull, a[0], 0, 16);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const float sc = rsqrt_fast(dnext);
    const float l = a[t] * sc;
    if (g == t) inv = sc;
    a[t] = l;
    if (t < 15) {
      const float crit = fmaf(-l, l, a[t + 1]);
      dnext = __shfl_sync(kFull, crit, t + 1, 16);
    }
#pragma unroll
    for (int c = t + 1; c < 16; ++c) {
      const float lc = __shfl_sync(kFull, l, c, 16);
      a[c] = fmaf(-l, lc, a[c]);
    }
  }
}

// (B) lane per row holding the FULL symmetric row; pivot row broadcast through
// shared memory (4 x LDS.128), pivot value by one shuffle.  LDL^T form.
__device__ __forceinline__ void dfB(float (&a)[16], float& inv, int g, float* xb) {
  // a[c] = A[g][c] for all c (full symmetric row)
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const float d = __shfl_sync(kFull, a[t], t, 16);  // pivot d_t (lane t's diagonal)
    const float rd = 1.f / d;
    if (g == t) {
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        *reinterpret_cast<float4*>(xb + 4 * c4) = make_float4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
    }
    __syncwarp();
    const float m = a[t] * rd;  // multiplier for this row
    float row[16];
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      const float4 v = *reinterpret_cast<const float4*>(xb + 4 * c4);
      row[4 * c4] = v.x; row[4 * c4 + 1] = v.y; row[4 * c4 + 2] = v.z; row[4 * c4 + 3] = v.w;
    }
    __syncwarp();
#pragma unroll
    for (int c = t + 1; c < 16; ++c) a[c] = fmaf(-m, row[c], a[c]);
    if (g == t) inv = rsqrt_fast(d);
  }
}


__device__ __forceinline__ float rcp_fast(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// (C) full symmetric row per lane, LDL^T; the pivot comes with the broadcast row
// (no shuffles): lane t publishes its row, everyone reads it (4 x LDS.128).
// Double-buffered broadcast slots -> one __syncwarp per pivot.
__device__ __forceinline__ void dfC(float (&a)[16], float& inv, int g, float* xb) {
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    float* slot = xb + (t & 1) * 16;
    if (g == t) {
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        *reinterpret_cast<float4*>(slot + 4 * c4) = make_float4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
    }
    __syncwarp();
    float row[16];
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      const float4 v = *reinterpret_cast<const float4*>(slot + 4 * c4);
      row[4 * c4] = v.x; row[4 * c4 + 1] = v.y; row[4 * c4 + 2] = v.z; row[4 * c4 + 3] = v.w;
    }
    const float rd = rcp_fast(row[t]);
    const float m = a[t] * rd;
#pragma unroll
    for (int c = t + 1; c < 16; ++c) a[c] = fmaf(-m, row[c], a[c]);
    if (g == t) inv = rsqrt_fast(row[t]);
  }
}

// (D) like (C) but 2 pivots per broadcast (2x2 pivot block solved locally).
__device__ __forceinline__ void dfD(float (&a)[16], float& inv, int g, float* xb) {
#pragma unroll
  for (int t = 0; t < 16; t += 2) {
    float* slot = xb + ((t >> 1) & 1) * 32;
    if (g == t || g == t + 1) {
      float* dst = slot + 16 * (g - t);
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        *reinterpret_cast<float4*>(dst + 4 * c4) = make_float4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
    }
    __syncwarp();
    float r0[16], r1[16];
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      const float4 v = *reinterpret_cast<const float4*>(slot + 4 * c4);
      const float4 w = *reinterpret_cast<const float4*>(slot + 16 + 4 * c4);
      r0[4 * c4] = v.x; r0[4 * c4 + 1] = v.y; r0[4 * c4 + 2] = v.z; r0[4 * c4 + 3] = v.w;
      r1[4 * c4] = w.x; r1[4 * c4 + 1] = w.y; r1[4 * c4 + 2] = w.z; r1[4 * c4 + 3] = w.w;
    }
    // row t+1 was published BEFORE pivot t was applied to it: apply now (locally)
    const float rd0 = rcp_fast(r0[t]);
    const float e = r0[t + 1];
    const float f = e * rd0;
#pragma unroll
    for (int c = t + 1; c < 16; ++c) r1[c] = fmaf(-f, r0[c], r1[c]);
    const float rd1 = rcp_fast(r1[t + 1]);
    const float m0 = a[t] * rd0;
    const float a1 = fmaf(-m0, e, a[t + 1]);
    const float m1 = a1 * rd1;
    a[t + 1] = a1;
#pragma unroll
    for (int c = t + 2; c < 16; ++c) a[c] = fmaf(-m1, r1[c], fmaf(-m0, r0[c], a[c]));
    if (g == t) inv = rsqrt_fast(r0[t]);
    if (g == t + 1) inv = rsqrt_fast(r1[t + 1]);
  }
}

// (E) 4 pivots per shared-memory round: rows t..t+3 published, every lane solves
// the 4x4 pivot block locally (applying the earlier pivots of the round to the
// published rows) and applies the rank-4 update to its own row.
__device__ __forceinline__ void dfE(float (&a)[16], float& inv, int g, float* xb) {
#pragma unroll
  for (int t = 0; t < 16; t += 4) {
    float* slot = xb + ((t >> 2) & 1) * 64;
    if (g >= t && g < t + 4) {
      float* dst = slot + 16 * (g - t);
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        *reinterpret_cast<float4*>(dst + 4 * c4) = make_float4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
    }
    __syncwarp();
    float r[4][16];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const float4 v = *reinterpret_cast<const float4*>(slot + 16 * u + 4 * c4);
        r[u][4 * c4] = v.x; r[u][4 * c4 + 1] = v.y; r[u][4 * c4 + 2] = v.z; r[u][4 * c4 + 3] = v.w;
      }
    float rs[4], l[4];
    // local LDL of the published rows (pivots t..t+3), and the own row's multipliers
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      rs[u] = rsqrt_fast(r[u][t + u]);
      const float rd = rs[u] * rs[u];
#pragma unroll
      for (int w = u + 1; w < 4; ++w) {
        const float f = r[u][t + w] * rd;
#pragma unroll
        for (int c = t + w; c < 16; ++c) r[w][c] = fmaf(-f, r[u][c], r[w][c]);
      }
      l[u] = a[t + u] * rs[u];
      const float m = l[u] * rs[u];
#pragma unroll
      for (int c = t + u + 1; c < 16; ++c) a[c] = fmaf(-m, r[u][c], a[c]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[t + u] = l[u];
      if (g == t + u) inv = rs[u];
    }
  }
}

// (G) 4 pivots per round, shuffles only: the pivot block's lower entries come from
// lanes t..t+3 (10 SHFL), every lane factors it locally, transforms its own four
// entries (o), and the rank-4 update takes each row c's transformed entries from
// lane c (4 SHFL per row).
template <int t>
__device__ __forceinline__ void dfG_round(float (&a)[16], float& inv, int g) {
  float B[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v <= u; ++v) B[u][v] = __shfl_sync(kFull, a[t + v], t + u, 16);
  float rs[4], rd[4], f[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    rs[u] = rsqrt_fast(B[u][u]);
    rd[u] = rs[u] * rs[u];
#pragma unroll
    for (int w = u + 1; w < 4; ++w) {
      f[u][w] = B[w][u] * rd[u];
#pragma unroll
      for (int r = w; r < 4; ++r) B[r][w] = fmaf(-f[u][w], B[r][u], B[r][w]);
    }
  }
  float o[4] = {a[t], a[t + 1], a[t + 2], a[t + 3]};
#pragma unroll
  for (int u = 0; u < 3; ++u)
#pragma unroll
    for (int w = u + 1; w < 4; ++w) o[w] = fmaf(-f[u][w], o[u], o[w]);
  float m[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    m[u] = o[u] * rd[u];
    a[t + u] = o[u] * rs[u];
    if (g == t + u) inv = rs[u];
  }
#pragma unroll
  for (int c = t + 4; c < 16; ++c) {
    float acc = a[c];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc = fmaf(-m[u], __shfl_sync(kFull, o[u], c, 16), acc);
    a[c] = acc;
  }
}
__device__ __forceinline__ void dfG(float (&a)[16], float& inv, int g) {
  dfG_round<0>(a, inv, g);
  dfG_round<4>(a, inv, g);
  dfG_round<8>(a, inv, g);
  dfG_round<12>(a, inv, g);
}

template <int V>
__global__ void kern(long long* out, float* sink) {
  __shared__ __align__(16) float xb[256];
  const int lane = threadIdx.x & 31, g = lane & 15;
  float a[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) a[c] = (c == g) ? 20.f + g : 0.3f / (1 + g + c);
  float acc = 0.f, inv = 0.f;
  long long best = 1ll << 60;
  for (int it = 0; it < 64; ++it) {
    float b[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) b[c] = a[c] + acc * 1e-30f;
    __syncwarp();
    const long long t0 = clock64();
    if (V == 0) dfA(b, inv, g);
    else if (V == 1) dfB(b, inv, g, xb + 16 * (lane >> 4));
    else if (V == 2) dfC(b, inv, g, xb + 32 * (lane >> 4));
    else if (V == 3) dfD(b, inv, g, xb + 64 * (lane >> 4));
    else if (V == 4) dfE(b, inv, g, xb + 128 * (lane >> 4));
    else dfG(b, inv, g);
    float s = inv;
#pragma unroll
    for (int c = 0; c < 16; ++c) s += b[c];
    acc += s;
    __syncwarp();
    const long long t1 = clock64() + (acc == 1.2345f);
    if (it > 2 && t1 - t0 < best) best = t1 - t0;
  }
  if (lane == 0) out[V] = best;
  // correctness probe: store L row of lane 5 (t <= 5) for cross-variant comparison
  if (lane == 5) {
    float b[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) b[c] = a[c];
    float iv = 0.f;
    if (V == 0) dfA(b, iv, g);
    else if (V == 2) dfC(b, iv, g, xb);
    else if (V == 3) dfD(b, iv, g, xb);
    else if (V == 4) dfE(b, iv, g, xb);
    else if (V == 5) dfG(b, iv, g);
    for (int c = 0; c <= 5; ++c) sink[8 + 8 * V + c] = b[c];
  }
  if (acc == 1.2345f) sink[0] = acc;
}

int main() {
  long long* d;
  float* s;
  cudaMalloc(&d, 64);
  cudaMalloc(&s, 1024);
  kern<0><<<1, 32>>>(d, s);
  kern<1><<<1, 32>>>(d, s);
  kern<2><<<1, 32>>>(d, s);
  kern<3><<<1, 32>>>(d, s);
  kern<4><<<1, 32>>>(d, s);
  kern<5><<<1, 32>>>(d, s);
  long long h[6];
  cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
  printf("4-pivot shuffles (G): %lld cycles\n", h[5]);
  printf("4-pivot (E): %lld cycles\n", h[4]);
  float L[64];
  cudaMemcpy(L, s, 256, cudaMemcpyDeviceToHost);
  for (int v = 0; v < 6; ++v) { if (v == 1) continue; printf("variant %d row5:", v); for (int c = 0; c <= 5; ++c) printf(" %.6f", L[8 + 8 * v + c]); printf("\n"); }
  printf("diag16 shfl (A): %lld\nsmem-row LDLt div+shfl (B): %lld\nsmem-row LDLt rcp (C): %lld\n2-pivot (D): %lld cycles\n%s\n",
         h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
