// Euclidean spectral projection A = pinv(Phi) F — the reference's
// project_to_spectral (/root/reference/proj/include/fmsolve/spectral.hpp:47-93),
// batched over shapes, SURVEY §8(f) rank 3.  (The hot path's projection is the
// mass-weighted Phi^T Mass F of the north_star, fmap_tc.cu; this route serves
// bases that are not mass-orthonormal.)
//
// One CTA (8 warps) per shape, f64 throughout: a one-sided Jacobi SVD of the
// n x k basis (Hestenes; parallel round-robin pair ordering, one pair per warp,
// lanes over vertices) gives W = Phi V with orthogonal columns, sigma_j = ||W_j||.
// The reference's decisions follow from it:
//   * n < k                     -> rank-revealing path (rank < k necessarily)
//   * cond = sigma_max / sigma_min <= threshold -> normal-equations solve
//   * else rank-revealing path: rank = #{sigma_j > eps * min(n, k) * sigma_max}
//     (the default threshold of the column-pivoted QR inside Eigen's
//     CompleteOrthogonalDecomposition); rank < k -> RankDeficientError(rank)
// and every accepted shape gets the least-squares solution
//   A = pinv(Phi) F = V diag(1 / sigma^2) W^T F,
// which is what both reference branches (LLT of Phi^T Phi, COD solve) compute.
// Work: O(sweeps * n k^2) + 2 n k d flops per shape on the FP64 SIMT pipe — a
// correctness route, not a hot path.
#include "fmap_kernels.cuh"

#include <algorithm>
#include <cfloat>

namespace fmap {

namespace {

constexpr int kPvThreads = 256;
constexpr int kPvWarps = kPvThreads / 32;

struct PinvArgs {
  const double* phi;  // [b][n][k]
  const double* F;    // [b][n][d]
  double* out;        // [b][k][d]
  double* work;       // per shape: W (k x n, column j contiguous) | V (k x k, column j contiguous) |
                      // sigma (k) | T (k x d)
  int* rank_out;      // [b]
  unsigned long long* fail_min;
  int64_t n;
  int k, d;
  double cond_thr;
};

__global__ void __launch_bounds__(kPvThreads) pinv_jacobi_kernel(PinvArgs a) {
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const int k = a.k, d = a.d;
  const int kp = (k + 1) & ~1;  // padded to even for the round-robin schedule
  double* W = a.work + (size_t)q * ((size_t)k * n + (size_t)k * k + (size_t)k * d + (size_t)k);
  double* V = W + (size_t)k * n;
  double* T = V + (size_t)k * k;
  const double* P = a.phi + (size_t)q * n * k;
  const double* Fq = a.F + (size_t)q * n * d;
  __shared__ int s_rot;
  // W = Phi (columns contiguous), V = I
  for (size_t e = tid; e < (size_t)n * k; e += kPvThreads) {
    const int64_t v = (int64_t)(e / k);
    const int j = (int)(e % k);
    W[(size_t)j * n + v] = P[e];
  }
  for (int e = tid; e < k * k; e += kPvThreads) V[e] = (e / k == e % k) ? 1.0 : 0.0;
  __syncthreads();
  const double eps = DBL_EPSILON;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < kp - 1; ++round) {
      // round-robin pairing of kp players: player 0 fixed, the rest rotate
      for (int pr = warp; pr < kp / 2; pr += kPvWarps) {
        auto player = [&](int slot) { return slot == 0 ? 0 : 1 + (slot - 1 + round) % (kp - 1); };
        int p = player(pr), r = player(kp - 1 - pr);
        if (p > r) {
          const int t = p;
          p = r;
          r = t;
        }
        if (r >= k) continue;  // dummy player (odd k)
        double* wp = W + (size_t)p * n;
        double* wr = W + (size_t)r * n;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int64_t v = lane; v < n; v += 32) {
          const double x = wp[v], y = wr[v];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga == 0.0 || !(fabs(ga) > eps * sqrt(al * be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int64_t v = lane; v < n; v += 32) {
          const double x = wp[v], y = wr[v];
          wp[v] = c * x - s * y;
          wr[v] = s * x + c * y;
        }
        double* vp = V + (size_t)p * k;
        double* vr = V + (size_t)r * k;
        for (int i = lane; i < k; i += 32) {
          const double x = vp[i], y = vr[i];
          vp[i] = c * x - s * y;
          vr[i] = s * x + c * y;
        }
        if (lane == 0) s_rot = 1;
      }
      __syncthreads();
    }
    const int rot = s_rot;
    __syncthreads();
    if (!rot) break;
  }
  // singular values (column norms), max / min, rank
  double smax = 0.0, smin = DBL_MAX;
  for (int j = warp; j < k; j += kPvWarps) {
    double s2 = 0.0;
    for (int64_t v = lane; v < n; v += 32) s2 = fma(W[(size_t)j * n + v], W[(size_t)j * n + v], s2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) T[j] = sqrt(s2);  // T[0..k) temporarily holds sigma
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    smax = fmax(smax, T[j]);
    smin = fmin(smin, T[j]);
  }
  const double thr = eps * (double)(n < k ? n : k) * smax;
  int rank = 0;
  for (int j = 0; j < k; ++j) rank += T[j] > thr ? 1 : 0;
  const bool well = n >= k && smin > 0.0 && smax / smin <= a.cond_thr;
  if (!well && rank < k) {
    if (tid == 0) {
      a.rank_out[q] = rank;
      atomicMin(a.fail_min, (unsigned long long)q);
    }
    return;
  }
  if (tid == 0) a.rank_out[q] = k;
  __syncthreads();
  // O = diag(1 / sigma^2) W^T F (in the output buffer), then out = V O via T[k ..]
  double* O = a.out + (size_t)q * k * d;
  // O <- W^T F scaled (row j by 1/sigma_j^2)
  for (int e = tid; e < k * d; e += kPvThreads) {
    const int j = e / d, t = e % d;
    const double* wj = W + (size_t)j * n;
    double acc = 0.0;
    for (int64_t v = 0; v < n; ++v) acc = fma(wj[v], Fq[(size_t)v * d + t], acc);
    const double sj = T[j];
    O[e] = acc / (sj * sj);
  }
  __syncthreads();
  // T (k x d) <- V O  (V column j contiguous: V[j * k + i] = V(i, j)); then copy back
  for (int e = tid; e < k * d; e += kPvThreads) {
    const int i = e / d, t = e % d;
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(V[(size_t)j * k + i], O[(size_t)j * d + t], acc);
    T[k + e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < k * d; e += kPvThreads) O[e] = T[k + e];
}

__global__ void f32_to_f64_kernel(const float* __restrict__ x, double* __restrict__ y, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = (double)x[e];
}
__global__ void f64_to_f32_kernel(const double* __restrict__ x, float* __restrict__ y, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = (float)x[e];
}
__global__ void finite_f64_kernel(const double* __restrict__ x, size_t n, unsigned bit, unsigned* flags) {
  unsigned f = 0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    if (!(fabs(x[e]) <= DBL_MAX)) f = bit;
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

}  // namespace

size_t pinv_work_doubles(int64_t b, int64_t n, int k, int d) {
  return (size_t)b * ((size_t)k * n + (size_t)k * k + (size_t)k * d + (size_t)k);
}

cudaError_t launch_pinv(const double* phi, const double* F, int64_t b, int64_t n, int k, int d, double cond_thr,
                        double* work, double* out, int* rank_out, unsigned long long* fail_min, cudaStream_t st) {
  if (b < 1 || b > 65535) return cudaErrorInvalidValue;
  PinvArgs a{phi, F, out, work, rank_out, fail_min, n, k, d, cond_thr};
  note_launch("pinv_jacobi_kernel");
  pinv_jacobi_kernel<<<(unsigned)b, kPvThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_convert_f32_f64(const float* x, double* y, size_t n, cudaStream_t st) {
  note_launch("f32_to_f64_kernel");
  f32_to_f64_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 2048), 256, 0, st>>>(x, y, n);
  return cudaGetLastError();
}

cudaError_t launch_convert_f64_f32(const double* x, float* y, size_t n, cudaStream_t st) {
  note_launch("f64_to_f32_kernel");
  f64_to_f32_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 2048), 256, 0, st>>>(x, y, n);
  return cudaGetLastError();
}

cudaError_t launch_finite_f64(const double* x, size_t n, unsigned bit, unsigned* flags, cudaStream_t st) {
  note_launch("finite_f64_kernel");
  finite_f64_kernel<<<(unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 1184)), 256, 0, st>>>(
      x, n, bit, flags);
  return cudaGetLastError();
}

}  // namespace fmap
