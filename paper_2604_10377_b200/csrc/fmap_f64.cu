// f64 route: the reference's default precision (bench.hpp:32 Precision::F64,
// verify tolerance 1e-8 — bench.cpp:28; rcond threshold 1e-14 — solver.hpp:18-27).
//
// Same row systems as the f32 route,
//     (G_q + lambda*diag(M_q[i,:]) + ridge*I) x = R_q[i,:]^T,   C_q[i,:] = x^T,
// replacing the reference's per-system PartialPivLU<double>
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170) inside
// solve_batched_many<double> (:220-322); SPD by construction, so Cholesky.
//
// One CTA (1024 threads) owns one system at a time (persistent over systems, one
// CTA per SM: the packed lower triangle of a k = 200 system is 160 KB of shared
// memory):
//   * staging: row r of G (contiguous, coalesced across the warp's lanes) into
//     the packed row-major lower triangle, lambda*m + ridge on the diagonal;
//   * blocked right-looking Cholesky, 8-column panels: warp 0 factors the 8x8
//     diagonal block (and the panel's forward substitution), every row below
//     solves its L21 entries against L11, then the trailing rank-8 update runs on
//     the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) — B200's SIMT FP64 pipe
//     is vestigial (~1.2 TFLOP/s measured), the tensor path is not;
//   * back substitution L^T x = y column-oriented (row j of L is contiguous).
// Verdict as the f32 route: non-positive / non-finite pivot, rcond estimate
// min(pivot)/max|diag| below the threshold, or a non-finite solution; lowest
// failing global system index wins.
#include "fmap_kernels.cuh"
#include "fmap_solver.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdint>

namespace fmap {

namespace {

constexpr int kT64 = 1024;  // 32 warps: the rank-1 update is latency-bound (LDS -> DFMA -> STS)

// Packed lower triangle with every row padded to an even length (row r starts at
// an even index, so column pairs move as one double2): off(r) = r(r+1)/2 + ceil(r/2).
__device__ __forceinline__ int off(int r) { return r * (r + 1) / 2 + (r + 1) / 2; }
__host__ __device__ inline size_t packed_doubles(int k) { return (size_t)k * (k + 1) / 2 + (k + 1) / 2; }

__global__ void __launch_bounds__(kT64, 1)
    chol_f64_kernel(const double* __restrict__ G, const double* __restrict__ R, const double* __restrict__ M,
                    double* __restrict__ C, int k, int64_t nsys, double lambda, double ridge, double rthr,
                    int rhs_unit, unsigned long long* fail_min, unsigned* rcond_min_bits) {
  extern __shared__ __align__(16) double sm64[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kT64 / 32;
  constexpr int NB = 8;  // panel width
  double* A = sm64;                                    // padded packed lower triangle
  double* y = A + ((packed_doubles(k) + 1) & ~(size_t)1);  // right-hand side -> y = L^{-1} r
  double* yy = y + ((k + 3) & ~1);                     // final forward values
  double* xs = yy + k;                                 // back substitution work vector
  double* invd = xs + k;                               // 1 / L_jj
  __shared__ double red[NW];
  __shared__ double s_piv;
  __shared__ int sbad;

  for (int64_t sys = blockIdx.x; sys < nsys; sys += gridDim.x) {
    const int64_t q = sys / k;
    const int i = (int)(sys - q * k);
    const double* Gq = G + (size_t)q * k * k;
    const double* Mi = M + ((size_t)q * k + i) * k;
    // ---- staging ----
    for (int r = warp; r < k; r += NW) {
      double* Ar = A + off(r);
      for (int c = lane; c <= r; c += 32) Ar[c] = Gq[(size_t)r * k + c];
    }
    __syncthreads();
    double dm = 0.0;
    for (int r = tid; r < k; r += kT64) {
      const double d = A[off(r) + r] + lambda * Mi[r] + ridge;
      A[off(r) + r] = d;
      dm = fmax(dm, fabs(d));
      y[r] = rhs_unit < 0 ? R[((size_t)q * k + i) * k + r] : (r == rhs_unit ? 1.0 : 0.0);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if (lane == 0) red[warp] = dm;
    __syncthreads();
    double dmax = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) dmax = fmax(dmax, red[w]);
    double pivmin = DBL_MAX;  // lane-local in warp 0 (diagonal pivots), reduced at the end
    bool bad = false;

    // ---- blocked factorization (8-column panels) + forward substitution ----
    // (1) warp 0: 8x8 diagonal block at j0, lane u = row j0+u (lower part only),
    //     and the panel's forward-substitution values.  For j0 > 0 it runs inside
    //     the previous panel's trailing update, right after warp 0 has updated
    //     that block (tile (0,0) of the update), hidden behind the other warps'
    //     tiles.
    auto diag_block = [&](int j0) {
      const int nb = min(NB, k - j0);
      const int u = lane;
      double a[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) a[t] = (u < nb && t <= u) ? A[off(j0 + u) + j0 + t] : 0.0;
      double inv_u = 0.0;
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        if (t < nb) {
          const double d = __shfl_sync(0xffffffffu, a[t], t);  // lane t's updated diagonal
          const double inv = 1.0 / sqrt(d);
          if (u == t) {
            pivmin = fmin(pivmin, d);
            bad |= !(d > 0.0) || !(d <= DBL_MAX);
            inv_u = inv;
          }
          const double l = a[t] * inv;  // L[j0+u][j0+t] for u >= t
          a[t] = l;
#pragma unroll
          for (int c = t + 1; c < NB; ++c) {
            const double lc = __shfl_sync(0xffffffffu, l, c);
            if (c <= u) a[c] = fma(-l, lc, a[c]);
          }
        }
      }
      // panel forward substitution: yb = L11^{-1} y[j0 .. j0+nb)
      double yb = (u < nb) ? y[j0 + u] : 0.0;
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        if (t < nb) {
          const double yt = __shfl_sync(0xffffffffu, yb * inv_u, t);
          if (u > t) yb = fma(-a[t], yt, yb);
          if (u == t) yb = yt;
        }
      }
      if (u < nb) {
#pragma unroll
        for (int t = 0; t < NB; ++t)
          if (t <= u) A[off(j0 + u) + j0 + t] = a[t];
        invd[j0 + u] = inv_u;
        yy[j0 + u] = yb;
      }
    };
    if (warp == 0) diag_block(0);
    __syncthreads();
    for (int j0 = 0; j0 < k; j0 += NB) {
      const int nb = min(NB, k - j0);
      // (2) rows below the block: L21 row (TRSM against L11), y update
      const int nrest = k - j0 - nb;
      for (int rr = tid; rr < nrest; rr += kT64) {
        const int r = j0 + nb + rr;
        double* Ar = A + off(r) + j0;
        double l[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          if (t < nb) {
            double v = Ar[t];
            const double* L11t = A + off(j0 + t) + j0;
#pragma unroll
            for (int s2 = 0; s2 < t; ++s2) v = fma(-l[s2], L11t[s2], v);
            l[t] = v * invd[j0 + t];
          } else {
            l[t] = 0.0;
          }
        }
        double yr = y[r];
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          if (t < nb) {
            Ar[t] = l[t];
            yr = fma(-l[t], yy[j0 + t], yr);
          }
        }
        y[r] = yr;
      }
      __syncthreads();
      // (3) trailing rank-8 update of rows / columns >= j0+8 on the FP64 tensor
      //     path (DMMA, mma.sync m8n8k4 f64): 8x8 tiles of the lower trailing
      //     triangle, K = the panel's 8 columns in two k=4 steps.  Row r's panel
      //     entries are contiguous (A[off(r) + j0 ...]); A fragment = -L rows,
      //     B fragment = L rows of the tile's columns, C/D = the trailing block
      //     (double2 per lane; only c <= r is stored back, so diagonal tiles never
      //     touch the next row).  (Only full panels have a trailing part.)
      if (nrest > 0) {
        const int jb = j0 + NB;
        const int T = (nrest + 7) >> 3;
        const int g = lane >> 2, q4 = lane & 3;
        const int ntiles = T * (T + 1) / 2;
        // warp 0: tile 0 (the next diagonal block) then its factorization;
        // warps 1..NW-1: tiles 1.. round-robin
        // tile e = tr(tr+1)/2 + tc walked with an incremental (tr, tc) cursor
        const int e0 = warp == 0 ? 0 : warp, estep = warp == 0 ? ntiles : NW - 1;
        int tr = 0, tc = e0;
        while (tc > tr) {
          tc -= tr + 1;
          ++tr;
        }
        for (int e = e0; e < (warp == 0 ? 1 : ntiles); e += estep) {
          {
            const int r0 = jb + 8 * tr, c0 = jb + 8 * tc;
            const int ra = r0 + g, rb = c0 + g;  // A-fragment row, B-fragment column (= L row)
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
            if (ra < k) {
              a0 = -A[off(ra) + j0 + q4];
              a1 = -A[off(ra) + j0 + 4 + q4];
            }
            if (rb < k) {
              b0 = A[off(rb) + j0 + q4];
              b1 = A[off(rb) + j0 + 4 + q4];
            }
            const int cr = r0 + g, cc = c0 + 2 * q4;
            const bool st = cr < k && cc <= cr;
            double2 cv = make_double2(0.0, 0.0);
            if (st) cv = *reinterpret_cast<const double2*>(A + off(cr) + cc);
            double d0, d1;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                         : "=d"(d0), "=d"(d1)
                         : "d"(a0), "d"(b0), "d"(cv.x), "d"(cv.y));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                         : "=d"(d0), "=d"(d1)
                         : "d"(a1), "d"(b1), "d"(d0), "d"(d1));
            if (st) *reinterpret_cast<double2*>(A + off(cr) + cc) = make_double2(d0, d1);
          }
          tc += estep;
          while (tc > tr && tr < T) {
            tc -= tr + 1;
            ++tr;
          }
        }
        if (warp == 0) {  // the next diagonal block is final now (only this panel's update was pending)
          __syncwarp();
          diag_block(jb);
        }
      }
      __syncthreads();
    }
    if (warp == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        pivmin = fmin(pivmin, __shfl_xor_sync(0xffffffffu, pivmin, o));
        bad |= __shfl_xor_sync(0xffffffffu, (int)bad, o) != 0;
      }
      if (lane == 0) {
        sbad = bad ? 1 : 0;
        s_piv = pivmin;
      }
    }
    // ---- back substitution L^T x = y in 8-row blocks from the bottom: warp 0
    //      solves the block's 8x8 transposed triangle (shuffles), then every
    //      thread removes the block's contribution from the rows above it (row c
    //      of L is contiguous, so A[off(c) + r] is coalesced over r) ----
    for (int r = tid; r < k; r += kT64) xs[r] = yy[r];
    __syncthreads();
    double* Crow = rhs_unit < 0 ? C + ((size_t)q * k + i) * k : C;
    bool nf = false;
    for (int c0 = ((k - 1) / NB) * NB; c0 >= 0; c0 -= NB) {
      const int nbb = min(NB, k - c0);
      if (warp == 0) {
        double v = lane < nbb ? xs[c0 + lane] : 0.0;
#pragma unroll
        for (int t = NB - 1; t >= 0; --t) {
          if (t < nbb) {
            const double xt = __shfl_sync(0xffffffffu, v, t) * invd[c0 + t];
            if (lane < t) v = fma(-A[off(c0 + t) + c0 + lane], xt, v);
            if (lane == t) v = xt;
          }
        }
        if (lane < nbb) {
          xs[c0 + lane] = v;
          Crow[c0 + lane] = v;
        }
        nf |= __any_sync(0xffffffffu, lane < nbb && !(fabs(v) <= DBL_MAX));
      }
      __syncthreads();
      for (int r = tid; r < c0; r += kT64) {
        double acc = xs[r];
#pragma unroll
        for (int t = 0; t < NB; ++t)
          if (t < nbb) acc = fma(-A[off(c0 + t) + r], xs[c0 + t], acc);
        xs[r] = acc;
      }
      __syncthreads();
    }
    if (tid == 0) {
      double rc = dmax > 0.0 ? fmax(s_piv, 0.0) / dmax : 0.0;
      if (!(rc >= 0.0)) rc = 0.0;
      if (sbad || nf || !(rc >= rthr)) atomicMin(fail_min, (unsigned long long)sys);
      atomicMin(rcond_min_bits, __float_as_uint((float)rc));
    }
    __syncthreads();
  }
}

// bit0 non-finite gram, bit1 non-finite rhs, bit2 non-finite mask, bit3 negative mask
__global__ void validate_f64_kernel(const double* __restrict__ g, const double* __restrict__ r,
                                    const double* __restrict__ m, size_t n, unsigned* flags) {
  unsigned f = 0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    if (!(fabs(g[e]) <= DBL_MAX)) f |= 1u;
    if (!(fabs(r[e]) <= DBL_MAX)) f |= 2u;
    const double v = m[e];
    if (!(fabs(v) <= DBL_MAX)) f |= 4u;
    if (v < 0.0) f |= 8u;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// ||C_q G_q + lambda M_q .* C_q - R_q||_F^2 per pair (solver.hpp:116-128), fp64:
// one CTA per (pair, row), threads over columns (G rows contiguous).
__global__ void residual_f64_kernel(const double* __restrict__ Cm, const double* __restrict__ G,
                                    const double* __restrict__ R, const double* __restrict__ M, int k,
                                    double lambda, double* __restrict__ sq) {
  const int64_t q = blockIdx.y;
  const int i = blockIdx.x;
  const double* Ci = Cm + ((size_t)q * k + i) * k;
  const double* Gq = G + (size_t)q * k * k;
  double acc = 0.0;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < k; ++t) s = fma(Ci[t], Gq[(size_t)t * k + c], s);
    const size_t e = ((size_t)q * k + i) * k + c;
    const double v = s + lambda * M[e] * Ci[c] - R[e];
    acc = fma(v, v, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&sq[q], acc);
}

// solver.hpp:269-273 fault hook, as the f32 route: system 0's LHS with entry
// (0, w) negated is A + alpha e_0 e_w^T; Sherman-Morrison with z = A^{-1} e_0.
__global__ void fault_combine_f64_kernel(double* __restrict__ x, const double* __restrict__ z, int k, int w,
                                         double alpha, unsigned long long* fail_min) {
  __shared__ double coef;
  if (threadIdx.x == 0) {
    const double den = 1.0 + alpha * z[w];
    coef = alpha * x[w] / den;
    if (!(fabs(den) > 0.0) || !(fabs(coef) <= DBL_MAX)) atomicMin(fail_min, 0ull);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) x[c] = x[c] - z[c] * coef;
}

}  // namespace

cudaError_t launch_fault_combine_f64(double* x, const double* z, int k, int w, double alpha,
                                     unsigned long long* fail_min, cudaStream_t st) {
  note_launch("fault_combine_f64_kernel");
  fault_combine_f64_kernel<<<1, 256, 0, st>>>(x, z, k, w, alpha, fail_min);
  return cudaGetLastError();
}

size_t chol_f64_smem_bytes(int k) {
  return (((packed_doubles(k) + 1) & ~(size_t)1) + ((k + 3) & ~1) + 3 * (size_t)k) * sizeof(double);
}

cudaError_t launch_chol_f64(const double* G, const double* R, const double* M, double* C, int k, int64_t nsys,
                            double lambda, double ridge, double rthr, int rhs_unit, unsigned long long* fail_min,
                            unsigned* rcond_min_bits, cudaStream_t st) {
  if (nsys <= 0) return cudaSuccess;
  int dev = 0, optin = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = chol_f64_smem_bytes(k);
  if (smem > (size_t)optin) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(chol_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int per_sm = (int)std::max<size_t>(1, 233472 / (smem + 1024));
  const int64_t maxgrid = (int64_t)sms * per_sm;
  const unsigned grid = (unsigned)(nsys < maxgrid ? nsys : maxgrid);
  note_launch("chol_f64_kernel");
  chol_f64_kernel<<<grid, kT64, smem, st>>>(G, R, M, C, k, nsys, lambda, ridge, rthr, rhs_unit, fail_min,
                                            rcond_min_bits);
  return cudaGetLastError();
}

cudaError_t launch_validate_f64(const double* g, const double* r, const double* m, size_t n, unsigned* flags,
                                cudaStream_t st) {
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
  note_launch("validate_f64_kernel");
  validate_f64_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(g, r, m, n, flags);
  return cudaGetLastError();
}

cudaError_t launch_residual_f64(const double* Cm, const double* G, const double* R, const double* M, int64_t b,
                                int k, double lambda, double* sq, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(sq, 0, (size_t)b * sizeof(double), st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)k, (unsigned)b);
  note_launch("residual_f64_kernel");
  residual_f64_kernel<<<grid, 128, 0, st>>>(Cm, G, R, M, k, lambda, sq);
  return cudaGetLastError();
}

}  // namespace fmap
