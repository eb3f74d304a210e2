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

// Offsets inside one panel.  For a panel starting at column j (multiple of 16),
// column j+t begins at colbase(j+t) = base0 + t*stride - S4(t) with
//   base0 = col_off(j) - j, stride = Rp - j, S4(t) = sum_{u<t}(u&~3) + (t&~3)
// so with t known at compile time every address is one IMAD + immediate.
__host__ __device__ constexpr int S4(int t) {
  int s = 0;
  for (int u = 0; u < t; ++u) s += u & ~3;
  return s + (t & ~3);
}

struct Panel {
  int base0, stride, j;
  __device__ __forceinline__ Panel(int j_, int Rp) : base0(col_off(j_, Rp) - j_), stride(Rp - j_), j(j_) {}
  // start of column j+t (add the absolute row index)
  __device__ __forceinline__ int col(int t) const { return base0 + t * stride - S4(t); }
};

// 8x8 lower-triangular block in registers (36 values, row-major packed).
__host__ __device__ constexpr int tri(int r, int c) { return r * (r + 1) / 2 + c; }

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

// Factor the 16x16 diagonal block at (j, j) with warp 0 and overwrite its lower
// triangle with L11^{-1}.  Blocked 2x2 over 8x8 sub-blocks:
//   L00 = chol(A00); L10 = A10 L00^{-T}; A11 -= L10 L10^T; L11 = chol(A11);
//   Linv = [[L00^{-1}, 0], [-L11^{-1} L10 L00^{-1}, L11^{-1}]].
// The 8x8 factorizations run replicated in every lane (no communication, no
// single-lane serialization); the row-parallel steps use lanes 0..7 and an
// 8x8 scratch (row-major L10).  FULL = the block is 16 wide (all but possibly
// the last panel); otherwise rows/cols >= nbe behave as identity padding.
template <bool FULL>
__device__ __noinline__ void diag_factor(float* A, int Rp, int j, int nbe, float* scr, int lane,
                                         float& pivmin, bool& bad) {
  const Panel P(j, Rp);
  auto at = [&](int r, int c) { return P.col(c) + j + r; };
  auto ok = [&](int r, int c) { return FULL || (r < nbe && c < nbe); };
  float t[36];
  // 1. L00^{-1}, replicated
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = c; r < 8; ++r) t[tri(r, c)] = ok(r, c) ? A[at(r, c)] : (r == c ? 1.f : 0.f);
  chol8_inv(t, pivmin, bad);
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = c; r < 8; ++r)
      if (lane == (tri(r, c) & 31) && ok(r, c)) A[at(r, c)] = t[tri(r, c)];
  // 2. lanes 0..7: row `lane` of L10 = A10[lane,:] L00^{-T}
  if (lane < 8) {
    float a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = ok(8 + lane, u) ? A[at(8 + lane, u)] : 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int u = 0; u <= c; ++u) acc = fmaf(a[u], t[tri(c, u)], acc);
      scr[lane * 8 + c] = acc;
    }
  }
  __syncwarp();
  // 3. A11 - L10 L10^T, replicated, then L11^{-1}
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = c; r < 8; ++r)
      t[tri(r, c)] = ok(8 + r, 8 + c) ? A[at(8 + r, 8 + c)] : (r == c ? 1.f : 0.f);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    float col[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) col[r] = scr[r * 8 + u];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int r = c; r < 8; ++r) t[tri(r, c)] = fmaf(-col[r], col[c], t[tri(r, c)]);
  }
  chol8_inv(t, pivmin, bad);
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int r = c; r < 8; ++r)
      if (lane == (tri(r, c) & 31) && ok(8 + r, 8 + c)) A[at(8 + r, 8 + c)] = t[tri(r, c)];
  __syncwarp();
  // 4. lanes 0..7: row `lane` of X = -(L11^{-1} L10) L00^{-1}
  if (lane < 8) {
    float y[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u <= lane) {
        const float li = A[at(8 + lane, 8 + u)];  // L11^{-1}[lane][u]
        const float4 l0 = *reinterpret_cast<const float4*>(scr + u * 8);
        const float4 l1 = *reinterpret_cast<const float4*>(scr + u * 8 + 4);
        y[0] = fmaf(li, l0.x, y[0]);
        y[1] = fmaf(li, l0.y, y[1]);
        y[2] = fmaf(li, l0.z, y[2]);
        y[3] = fmaf(li, l0.w, y[3]);
        y[4] = fmaf(li, l1.x, y[4]);
        y[5] = fmaf(li, l1.y, y[5]);
        y[6] = fmaf(li, l1.z, y[6]);
        y[7] = fmaf(li, l1.w, y[7]);
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float acc = 0.f;
#pragma unroll
      for (int u = c; u < 8; ++u) acc = fmaf(y[u], A[at(u, c)], acc);  // L00^{-1}[u][c]
      if (ok(8 + lane, c)) A[at(8 + lane, c)] = -acc;
    }
  }
  __syncwarp();
}

// Rows [r_lo, Rp) of panel [j, j+nbe):  L21 = A21 * L11^{-T}  (L11^{-1} stored in
// the diagonal block).  One row per thread; L11^{-1} reads are warp broadcasts.
template <int NT, bool FULL>
__device__ __forceinline__ void panel_trsm(float* A, int Rp, int j, int nbe, int r_lo, int tid) {
  const Panel P(j, Rp);
  for (int r = r_lo + tid; r < Rp; r += NT) {
    float a[kNB], x[kNB];
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      a[t] = (FULL || t < nbe) ? A[P.col(t) + r] : 0.f;
      x[t] = 0.f;
    }
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      if (FULL || t < nbe) {
#pragma unroll
        for (int c4 = (t & ~3); c4 < kNB; c4 += 4) {
          if (FULL || c4 < nbe) {
            const float4 l = ld4(A + P.col(t) + j + c4);  // Linv[c4..c4+3][t]
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c4 + u >= t) x[c4 + u] = fmaf(a[t], f4get(l, u), x[c4 + u]);
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (FULL || c < nbe) A[P.col(c) + r] = x[c];
  }
}

// 4x4 register tile: A[r0..r0+3][c0..c0+3] -= sum_{t<nbe} L[r][j+t] L[c][j+t].
// Operand pointers advance by stride - ((t+1)&~3) per column of the panel.
template <bool FULL>
__device__ __forceinline__ void syrk_tile(float* A, int Rp, const Panel& P, int nbe, int r0,
                                          int c0) {
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  const float* pr = A + P.base0 + r0;
  const float* pc = A + P.base0 + c0;
  if (FULL) {
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      const float4 x = ld4(pr + t * P.stride - S4(t));
      const float4 y = ld4(pc + t * P.stride - S4(t));
      const float xr[4] = {x.x, x.y, x.z, x.w};
      const float yr[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xr[a], yr[b], acc[a][b]);
    }
  } else {
    for (int t = 0; t < nbe; ++t) {
      const float4 x = ld4(pr);
      const float4 y = ld4(pc);
      const float xr[4] = {x.x, x.y, x.z, x.w};
      const float yr[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xr[a], yr[b], acc[a][b]);
      const int step = P.stride - ((t + 1) & ~3);
      pr += step;
      pc += step;
    }
  }
  float* q = A + col_off(c0, Rp) - c0 + r0;  // column c0 (multiple of 4), row r0
  const int qs = Rp - c0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float4 v = ld4(q + b * qs);
    v.x -= acc[0][b];
    v.y -= acc[1][b];
    v.z -= acc[2][b];
    v.w -= acc[3][b];
    st4(q + b * qs, v);
  }
}

}  // namespace

// Optional phase tracing (debug): p.trace != nullptr records clock64() per warp
// for block p.trace_block at fixed slots.
#define FMAP_TRACE(slot)                                                        \
  do {                                                                          \
    if (p.trace && blockIdx.x == (unsigned)p.trace_block && lane == 0)          \
      p.trace[warp * 1024 + (slot)] = clock64();                                \
  } while (0)

template <int MASK_MODE, int NT>
__global__ void __launch_bounds__(NT, 2) chol_solve_kernel(SolveParams p) {
  extern __shared__ __align__(16) float smem[];
  constexpr int NW = NT / 32;
  const int k = p.k, K4 = p.K4, Rp = p.Rp;
  const int P = packed_size(K4);
  float* A = smem;
  float* xv = smem + P;
  unsigned int* sc = reinterpret_cast<unsigned int*>(xv + K4);
  float* scr = xv + K4 + 32;  // 64-float diag scratch
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

  FMAP_TRACE(0);
  float pivmin = FLT_MAX;
  bool bad = false;
  if (warp == 0) {
    if (K4 >= kNB) diag_factor<true>(A, Rp, 0, kNB, scr, lane, pivmin, bad);
    else diag_factor<false>(A, Rp, 0, K4, scr, lane, pivmin, bad);
  }
  __syncthreads();
  FMAP_TRACE(1);

  for (int j = 0; j < K4; j += kNB) {
    const int ts = 8 + (j / kNB) * 8;
    const int nbe = min(kNB, K4 - j);
    const int jn = j + nbe;
    const int nbn = min(kNB, K4 - jn);
    const Panel Pj(j, Rp);
    // B: panel rows below the diagonal block (incl. the augmented rhs row)
    if (nbe == kNB) panel_trsm<NT, true>(A, Rp, j, nbe, jn, tid);
    else panel_trsm<NT, false>(A, Rp, j, nbe, jn, tid);
    FMAP_TRACE(ts + 0);
    __syncthreads();
    FMAP_TRACE(ts + 1);
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
        if (nbe == kNB) syrk_tile<true>(A, Rp, Pj, nbe, (Ct + l) << 2, Ct << 2);
        else syrk_tile<false>(A, Rp, Pj, nbe, (Ct + l) << 2, Ct << 2);
      }
    }
    FMAP_TRACE(ts + 2);
    __syncthreads();
    FMAP_TRACE(ts + 3);
    // D: warp 0 factors the next diagonal block while the others update the rest
    if (warp == 0) {
      if (nbn == kNB) diag_factor<true>(A, Rp, jn, nbn, scr, lane, pivmin, bad);
      else diag_factor<false>(A, Rp, jn, nbn, scr, lane, pivmin, bad);
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
            if (c0 < K4 && r0 < Rp && r0 >= c0) {
              if (nbe == kNB) syrk_tile<true>(A, Rp, Pj, nbe, r0, c0);
              else syrk_tile<false>(A, Rp, Pj, nbe, r0, c0);
            }
          }
          v -= nrb;
        }
      }
    }
    FMAP_TRACE(ts + 4);
    __syncthreads();
    FMAP_TRACE(ts + 5);
  }
  FMAP_TRACE(1000);

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
  FMAP_TRACE(1001);
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
