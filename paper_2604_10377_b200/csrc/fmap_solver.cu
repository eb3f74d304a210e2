// Batched in-shared-memory Cholesky solver for the regularized functional map
// (see fmap_solver.cuh for the layout and the algorithm outline).
#include "fmap_solver.cuh"

#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

namespace fmap {

namespace {

__device__ __forceinline__ int colbase(int c, int Rp) { return col_off(c, Rp) - (c & ~3); }

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float f4get(const float4& v, int u) {
  return u == 0 ? v.x : (u == 1 ? v.y : (u == 2 ? v.z : v.w));
}

// Diagonal mask entry m_i(c) for the three mask sources.
template <int MASK_MODE>
__device__ __forceinline__ float mask_entry(const SolveParams& p, int64_t q, int i, int c,
                                            float ev_max) {
  const int k = p.k;
  if constexpr (MASK_MODE == 0) {
    return p.mask[((size_t)q * k + i) * k + c];
  } else if constexpr (MASK_MODE == 1) {
    // masks.hpp:36-82 (resolvent), same operation order in fp32.
    const float s = p.sigma, s2 = s * s;
    const float mu1 = p.ev1[(size_t)q * k + c] / ev_max;
    const float mu2 = p.ev2[(size_t)q * k + i] / ev_max;
    const float re1 = mu1 / (mu1 * mu1 + s2), im1 = s / (mu1 * mu1 + s2);
    const float re2 = mu2 / (mu2 * mu2 + s2), im2 = s / (mu2 * mu2 + s2);
    const float re = re2 - re1, im = im2 - im1;
    return re * re + im * im;
  } else {
    // masks.hpp:13-34 (commutativity)
    const float d = p.ev2[(size_t)q * k + i] - p.ev1[(size_t)q * k + c];
    return d * d;
  }
}

// 8x8 lower-triangular block in registers (36 values, row-major packed).
__device__ __forceinline__ int tri(int r, int c) { return r * (r + 1) / 2 + c; }

// Cholesky of an 8x8 SPD block followed by the in-place inverse of its factor.
// On return t[] holds L^{-1} (lower); pivots feed pivmin / bad.
__device__ __forceinline__ void chol8_inv(float (&t)[36], float& pivmin, bool& bad) {
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float d = t[tri(p, p)];
    pivmin = fminf(pivmin, d);
    bad |= !(d > 0.f) || !(d < FLT_MAX);
    const float sinv = rsqrtf(d);
    t[tri(p, p)] = sinv;  // keeps 1/L_pp
#pragma unroll
    for (int r = p + 1; r < 8; ++r) t[tri(r, p)] *= sinv;
#pragma unroll
    for (int c = p + 1; c < 8; ++c)
#pragma unroll
      for (int r = c; r < 8; ++r) t[tri(r, c)] = fmaf(-t[tri(r, p)], t[tri(c, p)], t[tri(r, c)]);
  }
  // Linv[r][p] = -Linv[r][r] * (L[r][p] Linv[p][p] + sum_{p<u<r} L[r][u] Linv[u][p]),
  // columns left to right, rows top-down (in place).
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int r = p + 1; r < 8; ++r) {
      float acc = t[tri(r, p)] * t[tri(p, p)];
#pragma unroll
      for (int u = p + 1; u < r; ++u) acc = fmaf(t[tri(r, u)], t[tri(u, p)], acc);
      t[tri(r, p)] = -acc * t[tri(r, r)];
    }
}

// Element (r, c) of the diagonal block at (j, j), local indices, with identity
// padding beyond nbe (only the last panel has nbe < 16).
struct DiagView {
  float* A;
  int Rp, j, nbe;
  __device__ __forceinline__ int at(int r, int c) const { return colbase(j + c, Rp) + j + r; }
  __device__ __forceinline__ float ld(int r, int c) const {
    return (r < nbe && c < nbe) ? A[at(r, c)] : (r == c ? 1.f : 0.f);
  }
  __device__ __forceinline__ void st(int r, int c, float v) const {
    if (r < nbe && c < nbe) A[at(r, c)] = v;
  }
};

// Factor the 16x16 diagonal block at (j, j) with warp 0 and overwrite its lower
// triangle with L11^{-1}.  Blocked 2x2 over 8x8 sub-blocks:
//   L00 = chol(A00); L10 = A10 L00^{-T}; A11 -= L10 L10^T; L11 = chol(A11);
//   Linv = [[L00^{-1}, 0], [-L11^{-1} L10 L00^{-1}, L11^{-1}]].
// Single-thread 8x8 factorizations, 8-lane parallel TRSM / SYRK / combine.
// pivmin / bad are accumulated in lane 0.
__device__ __noinline__ void diag_factor(float* A, int Rp, int j, int nbe, int lane,
                                         float& pivmin, bool& bad) {
  const DiagView V{A, Rp, j, nbe};
  float t[36];
  // 1. L00^{-1}
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) t[tri(r, c)] = V.ld(r, c);
    chol8_inv(t, pivmin, bad);
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) V.st(r, c, t[tri(r, c)]);
  }
  __syncwarp();
  // 2. lane r < 8: row r of L10 = A10[r,:] * L00^{-T}
  float l10[8];
  if (lane < 8) {
    float a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = V.ld(8 + lane, c);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int u = 0; u <= c; ++u) acc = fmaf(a[u], V.ld(c, u), acc);  // Linv00[c][u]
      l10[c] = acc;
    }
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) V.st(8 + lane, c, l10[c]);
  }
  __syncwarp();
  // 3. lane r < 8: A11[r, 0..r] -= L10[r,:] L10[0..r,:]^T
  if (lane < 8) {
    float a11[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a11[c] = (c <= lane) ? V.ld(8 + lane, 8 + c) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float lcu = V.ld(8 + c, u);  // L10[c][u], broadcast
        if (c <= lane) a11[c] = fmaf(-l10[u], lcu, a11[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c <= lane) V.st(8 + lane, 8 + c, a11[c]);
  }
  __syncwarp();
  // 4. L11^{-1}
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) t[tri(r, c)] = V.ld(8 + r, 8 + c);
    chol8_inv(t, pivmin, bad);
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) V.st(8 + r, 8 + c, t[tri(r, c)]);
  }
  __syncwarp();
  // 5. X = -L11^{-1} (L10 L00^{-1});  lane r: row r of T = L10 L00^{-1} first
  float trow[8];
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int u = c; u < 8; ++u) acc = fmaf(l10[u], V.ld(u, c), acc);  // Linv00[u][c]
      trow[c] = acc;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) V.st(8 + lane, c, trow[c]);
  }
  __syncwarp();
  if (lane < 8) {
    float x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float li = (u <= lane) ? V.ld(8 + lane, 8 + u) : 0.f;  // Linv11[r][u]
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = fmaf(-li, V.ld(8 + u, c), x[c]);  // T[u][c]
    }
    __syncwarp(0xffu);
#pragma unroll
    for (int c = 0; c < 8; ++c) V.st(8 + lane, c, x[c]);
  }
  __syncwarp();
}

// Rows [r_lo, Rp) of panel [j, j+nbe):  L21 = A21 * L11^{-T}.
template <int NT>
__device__ __forceinline__ void panel_trsm(float* A, int Rp, int j, int nbe, int r_lo, int tid) {
  for (int r = r_lo + tid; r < Rp; r += NT) {
    float a[kNB], x[kNB];
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      a[t] = (t < nbe) ? A[colbase(j + t, Rp) + r] : 0.f;
      x[t] = 0.f;
    }
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      if (t < nbe) {
        const int base = colbase(j + t, Rp) + j;
#pragma unroll
        for (int c4 = (t & ~3); c4 < kNB; c4 += 4) {
          if (c4 < nbe) {
            const float4 l = ld4(A + base + c4);  // Linv[c4..c4+3][t]
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c4 + u >= t) x[c4 + u] = fmaf(a[t], f4get(l, u), x[c4 + u]);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (c < nbe) A[colbase(j + c, Rp) + r] = x[c];
  }
}

// 4x4 register tile: A[r0..r0+3][c0..c0+3] -= sum_{t<nbe} L[r][j+t] L[c][j+t].
__device__ __forceinline__ void syrk_tile(float* A, int Rp, int j, int nbe, int r0, int c0) {
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  int base = colbase(j, Rp);
#pragma unroll 4
  for (int t = 0; t < nbe; ++t) {
    const float4 x = ld4(A + base + r0);
    const float4 y = ld4(A + base + c0);
    const float xr[4] = {x.x, x.y, x.z, x.w};
    const float yr[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xr[a], yr[b], acc[a][b]);
    base += Rp - ((j + t + 1) & ~3);
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float* p = A + colbase(c0 + b, Rp) + r0;
    float4 v = ld4(p);
    v.x -= acc[0][b];
    v.y -= acc[1][b];
    v.z -= acc[2][b];
    v.w -= acc[3][b];
    st4(p, v);
  }
}

}  // namespace

template <int MASK_MODE, int NT>
__global__ void __launch_bounds__(NT, 2) chol_solve_kernel(SolveParams p) {
  extern __shared__ __align__(16) float smem[];
  constexpr int NW = NT / 32;
  const int k = p.k, K4 = p.K4, Rp = p.Rp;
  const int P = packed_size(K4);
  float* A = smem;
  float* xv = smem + P;
  unsigned int* sc = reinterpret_cast<unsigned int*>(xv + K4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t s = p.sys_offset + blockIdx.x;
  const int64_t q = s / k;
  const int i = (int)(s - q * k);

  if (tid == 0) {
    sc[0] = 0u;  // max diagonal (float bits, non-negative)
    sc[1] = 0u;  // ev_max bits
  }
  __syncthreads();

  float ev_max = 0.f;
  if constexpr (MASK_MODE == 1) {
    float m = 0.f;
    for (int c = tid; c < k; c += NT)
      m = fmaxf(m, fmaxf(p.ev1[(size_t)q * k + c], p.ev2[(size_t)q * k + c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) atomicMax(&sc[1], __float_as_uint(m));
    __syncthreads();
    ev_max = __uint_as_float(sc[1]);
    if (!(ev_max > 0.f)) {
      if (tid == 0) atomicOr(p.flags, 32u);
      return;  // masks.hpp:59: needs a non-zero spectrum to normalize by
    }
  }

  // ---- stage S = G + lambda*diag(m_i) + ridge*I and the rhs row into smem ----
  {
    const float* Gq = p.gram + (size_t)q * k * k;
    const float* Rrow = p.rhs + ((size_t)q * k + i) * k;
    float dmax = 0.f;
    for (int c = warp; c < K4; c += NW) {
      const int c4 = c & ~3;
      float* col = A + colbase(c, Rp);
      if (c < k) {
        const float* g = Gq + (size_t)c * k;  // row c of G == column c (symmetric)
        for (int r = c4 + lane; r < Rp; r += 32) {
          float v = 0.f;
          if (r < k) {
            v = g[r];
            if (r == c) {
              v += p.lambda * mask_entry<MASK_MODE>(p, q, i, c, ev_max) + p.ridge;
              dmax = fmaxf(dmax, fabsf(v));
            }
          } else if (r == K4) {
            v = p.rhs_unit < 0 ? Rrow[c] : (c == p.rhs_unit ? 1.f : 0.f);
          }
          col[r] = v;
        }
      } else {
        for (int r = c4 + lane; r < Rp; r += 32) col[r] = (r == c) ? 1.f : 0.f;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) atomicMax(&sc[0], __float_as_uint(dmax));
  }
  __syncthreads();

  float pivmin = FLT_MAX;
  bool bad = false;
  if (warp == 0) diag_factor(A, Rp, 0, min(kNB, K4), lane, pivmin, bad);
  __syncthreads();

  for (int j = 0; j < K4; j += kNB) {
    const int nbe = min(kNB, K4 - j);
    const int jn = j + nbe;
    const int nbn = min(kNB, K4 - jn);
    // B: panel rows below the diagonal block (incl. the augmented rhs row)
    panel_trsm<NT>(A, Rp, j, nbe, jn, tid);
    __syncthreads();
    if (nbn <= 0) break;
    // C: lookahead — update the next panel's columns [jn, jn+nbn)
    {
      const int C0 = jn >> 2, nR = Rp >> 2, ncol = nbn >> 2;
      int ntile = 0;
      for (int cc = 0; cc < ncol; ++cc) ntile += nR - (C0 + cc);
      for (int L = tid; L < ntile; L += NT) {
        int cc = 0, l = L;
        while (l >= nR - (C0 + cc)) {
          l -= nR - (C0 + cc);
          ++cc;
        }
        const int Ct = C0 + cc;
        syrk_tile(A, Rp, j, nbe, (Ct + l) << 2, Ct << 2);
      }
    }
    __syncthreads();
    // D: warp 0 factors the next diagonal block while the others update the rest
    if (warp == 0) {
      diag_factor(A, Rp, jn, nbn, lane, pivmin, bad);
    } else {
      const int cstart = jn + nbn;
      if (cstart < K4) {
        const int ncb = (K4 - cstart + 15) >> 4;
        const int lr = lane & 7, lc = lane >> 3;
        int v = warp - 1;
        for (int u = 0; u < ncb; ++u) {
          const int cb = cstart + (u << 4);
          const int nrb = (Rp - cb + 31) >> 5;
          for (; v < nrb; v += NW - 1) {
            const int r0 = cb + (v << 5) + (lr << 2);
            const int c0 = cb + (lc << 2);
            if (c0 < K4 && r0 < Rp && r0 >= c0) syrk_tile(A, Rp, j, nbe, r0, c0);
          }
          v -= nrb;
        }
      }
    }
    __syncthreads();
  }

  // ---- back substitution L^T x = y by warp 0; y sits in the augmented row ----
  if (warp != 0) return;
  for (int c = lane; c < K4; c += 32) xv[c] = A[colbase(c, Rp) + K4];
  __syncwarp();
  for (int jb = ((K4 - 1) / kNB) * kNB; jb >= 0; jb -= kNB) {
    const int nbe = min(kNB, K4 - jb);
    float xc = 0.f;
    if (lane < nbe) {
      const int base = colbase(jb + lane, Rp) + jb;
#pragma unroll
      for (int r = 0; r < kNB; ++r)
        if (r >= lane && r < nbe) xc = fmaf(A[base + r], xv[jb + r], xc);
    }
    __syncwarp();
    if (lane < nbe) xv[jb + lane] = xc;
    __syncwarp();
    for (int c = lane; c < jb; c += 32) {
      const float* col = A + colbase(c, Rp) + jb;
      float acc = 0.f;
      for (int r = 0; r < nbe; r += 4) {
        const float4 l = ld4(col + r);
        const float4 xx = ld4(xv + jb + r);
        acc = fmaf(l.x, xx.x, acc);
        acc = fmaf(l.y, xx.y, acc);
        acc = fmaf(l.z, xx.z, acc);
        acc = fmaf(l.w, xx.w, acc);
      }
      xv[c] -= acc;
    }
    __syncwarp();
  }
  bool nonfinite = false;
  float* Crow = p.C + ((size_t)q * k + i) * k;
  for (int c = lane; c < k; c += 32) {
    const float x = xv[c];
    nonfinite |= !(fabsf(x) <= FLT_MAX);
    Crow[c] = x;
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if (lane == 0) {
    const float dmax = __uint_as_float(sc[0]);
    float rc = dmax > 0.f ? pivmin / dmax : 0.f;
    if (!(rc >= 0.f)) rc = 0.f;
    if (bad || nonfinite || !(rc >= p.rcond_thr)) atomicMin(p.fail_min, (unsigned long long)s);
    atomicMin(p.rcond_min_bits, __float_as_uint(rc));
  }
}

// Host-side launcher.
cudaError_t launch_chol_solve(const SolveParams& p, int mask_mode, cudaStream_t stream) {
  constexpr int NT = 256;
  const size_t smem = solver_smem_bytes(p.k);
  if (p.nsys <= 0) return cudaSuccess;
  void (*fn)(SolveParams) = nullptr;
  switch (mask_mode) {
    case 0: fn = chol_solve_kernel<0, NT>; break;
    case 1: fn = chol_solve_kernel<1, NT>; break;
    default: fn = chol_solve_kernel<2, NT>; break;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // ask for the full shared-memory carveout so two ~86 KB CTAs co-reside per SM
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  fn<<<(unsigned)p.nsys, NT, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace fmap
