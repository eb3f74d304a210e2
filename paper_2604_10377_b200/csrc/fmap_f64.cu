// f64 route: the reference's default precision (bench.hpp:32 Precision::F64,
// verify tolerance 1e-8 — bench.cpp:28; rcond threshold 1e-14 — solver.hpp:18-27).
//
// Same row systems as the f32 route,
//     (G_q + lambda*diag(M_q[i,:]) + ridge*I) x = R_q[i,:]^T,   C_q[i,:] = x^T,
// replacing the reference's per-system PartialPivLU<double>
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170) inside
// solve_batched_many<double> (:220-322); SPD by construction, so Cholesky.
//
// One CTA owns one system at a time (persistent over systems, one CTA per SM:
// the packed lower triangle of a k = 200 system is 160 KB of shared memory):
//   * staging: row r of G (contiguous, coalesced across the warp's lanes) into
//     the packed row-major lower triangle, lambda*m + ridge on the diagonal;
//   * right-looking Cholesky, one column per step: the pivot's column is scaled
//     into a contiguous vector (forward substitution of the right-hand side rides
//     along), then the rank-1 trailing update with one warp per row (lanes over
//     the row's contiguous columns);
//   * back substitution L^T x = y column-oriented (row j of L is contiguous).
// FP64 on the SIMT pipe (no tcgen05 FP64 MMA); bound: the 2 barriers per column
// on the per-system chain, not FLOPs.  Verdict as the f32 route: non-positive /
// non-finite pivot, rcond estimate min(pivot)/max|diag| below the threshold, or a
// non-finite solution; lowest failing global system index wins.
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
  double* A = sm64;                                    // padded packed lower triangle
  double* col = A + ((packed_doubles(k) + 1) & ~(size_t)1);  // current column of L (+ zero pads)
  double* y = col + ((k + 3) & ~1);                    // right-hand side -> partially eliminated
  double* yy = y + k;                                  // y = L^{-1} r (final values)
  double* xs = yy + k;                                 // back substitution work vector
  double* invd = xs + k;                               // 1 / L_jj
  __shared__ double red[NW];
  __shared__ double s_inv[2], s_yj[2];
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
    if (tid < 2) col[k + tid] = 0.0;  // pads read by the last column pair
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if (lane == 0) red[warp] = dm;
    __syncthreads();
    double dmax = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) dmax = fmax(dmax, red[w]);
    // pivot data of step j is produced by ONE thread (tid 0) and published through
    // s_inv / s_yj (parity j & 1): for j = 0 here, for j + 1 right after warp 0 has
    // updated row j + 1 (the only row it depends on)
    double pivmin = DBL_MAX;
    bool bad = false;
    auto pivot = [&](int jn) {
      const double d = A[off(jn) + jn];
      pivmin = fmin(pivmin, d);
      bad |= !(d > 0.0) || !(d <= DBL_MAX);
      const double inv = 1.0 / sqrt(d);
      s_inv[jn & 1] = inv;
      s_yj[jn & 1] = y[jn] * inv;
    };
    if (tid == 0) pivot(0);
    __syncthreads();

    // ---- factorization + forward substitution ----
    for (int j = 0; j < k; ++j) {
      const double inv = s_inv[j & 1], yj = s_yj[j & 1];
      for (int r = j + 1 + tid; r < k; r += kT64) {
        const double l = A[off(r) + j] * inv;
        A[off(r) + j] = l;
        col[r] = l;
        y[r] = fma(-l, yj, y[r]);
      }
      if (tid == 0) {
        yy[j] = yj;
        invd[j] = inv;
        col[j] = 0.0;  // a column pair starting at j leaves column j unchanged
      }
      __syncthreads();
      // rank-1 update, rows r (short) and r2 = k + j - r (long) per warp, column pairs
      const int nrow = k - 1 - j, c0 = (j + 1) & ~1;
      for (int t = warp; 2 * t < nrow; t += NW) {
        const int r = j + 1 + t, r2 = k - 1 - t;
        const double lr = col[r], lr2 = col[r2];
        double* Ar = A + off(r);
        double* Ar2 = A + off(r2);
        for (int c = c0 + 2 * lane; c <= r2; c += 64) {
          const double2 cc = *reinterpret_cast<const double2*>(col + c);
          double2 v = *reinterpret_cast<double2*>(Ar2 + c);
          v.x = fma(-lr2, cc.x, v.x);
          v.y = fma(-lr2, cc.y, v.y);
          *reinterpret_cast<double2*>(Ar2 + c) = v;
          if (c <= r && r != r2) {
            double2 u = *reinterpret_cast<double2*>(Ar + c);
            u.x = fma(-lr, cc.x, u.x);
            u.y = fma(-lr, cc.y, u.y);
            *reinterpret_cast<double2*>(Ar + c) = u;
          }
        }
      }
      if (warp == 0 && j + 1 < k) {  // warp 0 owns row j + 1: next pivot
        __syncwarp();
        if (lane == 0) pivot(j + 1);
      }
      __syncthreads();
    }
    if (tid == 0) sbad = bad ? 1 : 0;
    // ---- back substitution L^T x = y (column-oriented: row j of L is contiguous) ----
    for (int r = tid; r < k; r += kT64) xs[r] = yy[r];
    __syncthreads();
    double* Crow = rhs_unit < 0 ? C + ((size_t)q * k + i) * k : C;
    bool nf = false;
    for (int j = k - 1; j >= 0; --j) {
      const double xj = xs[j] * invd[j];
      const double* Lj = A + off(j);
      for (int r = tid; r < j; r += kT64) xs[r] = fma(-Lj[r], xj, xs[r]);
      if (tid == 0) {
        Crow[j] = xj;
        nf |= !(fabs(xj) <= DBL_MAX);
      }
      __syncthreads();
    }
    if (tid == 0) {
      double rc = dmax > 0.0 ? fmax(pivmin, 0.0) / dmax : 0.0;
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
  fault_combine_f64_kernel<<<1, 256, 0, st>>>(x, z, k, w, alpha, fail_min);
  return cudaGetLastError();
}

size_t chol_f64_smem_bytes(int k) {
  return (((packed_doubles(k) + 1) & ~(size_t)1) + ((k + 3) & ~1) + 4 * (size_t)k) * sizeof(double);
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
  chol_f64_kernel<<<grid, kT64, smem, st>>>(G, R, M, C, k, nsys, lambda, ridge, rthr, rhs_unit, fail_min,
                                            rcond_min_bits);
  return cudaGetLastError();
}

cudaError_t launch_validate_f64(const double* g, const double* r, const double* m, size_t n, unsigned* flags,
                                cudaStream_t st) {
  const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
  validate_f64_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(g, r, m, n, flags);
  return cudaGetLastError();
}

cudaError_t launch_residual_f64(const double* Cm, const double* G, const double* R, const double* M, int64_t b,
                                int k, double lambda, double* sq, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(sq, 0, (size_t)b * sizeof(double), st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)k, (unsigned)b);
  residual_f64_kernel<<<grid, 128, 0, st>>>(Cm, G, R, M, k, lambda, sq);
  return cudaGetLastError();
}

}  // namespace fmap
