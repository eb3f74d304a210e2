// Normal equations on the 5th-generation tensor cores (north_star stage 1):
//   G_q = A_q A_q^T,  R_q = B_q A_q^T      (replaces normal_equations,
//   /root/reference/proj/include/fmsolve/solver.hpp:95-103, batched)
// and, for the bidirectional pipeline, G2 = B B^T, R2 = A B^T.
//
// One CTA per (128-row tile of the output, pair, product).  D[m][n] =
// sum_t X[m][t] Y[n][t] with X, Y row-major k x d: both operands are K-major in
// memory, so each 16-column K stage is loaded with coalesced float4 reads,
// split into TF32 hi/lo parts (3xTF32: hi*hi + hi*lo + lo*hi; 1xTF32 misses the
// 1e-4 bar) and stored in the no-swizzle core-matrix layout;
// thread 0 issues the tcgen05.mma (M = 128, N <= 256 per instruction, K = 8)
// into a TMEM accumulator while the 128 threads stage the next K stage (two
// buffers, mbarrier hand-off).  Symmetric products (G) compute the lower
// triangle's block row only (N = rows up to the tile's end) and mirror it, so G
// is exactly symmetric.  Work: 2 k^2 d flops per product (tensor-bound, tiny
// next to the solver); bytes 4 (2 k d + k^2) per product.
#include "fmap_kernels.cuh"
#include "tc_ptx.cuh"

#include <cstdlib>

namespace fmap {

namespace {

using namespace ptx;

constexpr int kGK = 16;        // K (= d) elements per stage
constexpr int kGThreads = 128;  // one thread per output row of the tile
constexpr int kGMaxN = 320;     // k <= 304 (solver limit) -> N <= 304 padded to 16

struct GramJob {
  const float* X;
  const float* Y;
  float* out;
  int sym;
  // residual mode (partial != nullptr): no `out`; per row r of pair q,
  // partial[q k + r] = sum_c (D[r][c] + lambda M[r][c] X[r][c] - R[r][c])^2  (fp64)
  const float* M;
  const float* R;
  float lambda;
  double* partial;
};

struct GramArgs {
  GramJob job[4];
  int k, d;
  int ys;          // floats of one Y operand copy (round16(k) x 16)
  uint32_t tcols;  // TMEM columns allocated (256, or 512 when k > 256)
};

__device__ __forceinline__ uint32_t idesc_tf32_pos(int N) {  // D += A*B (no negation), M = 128
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ int core_idx(int r, int t) {  // element (r, t < 16) of a [rows x 16] operand
  return (r >> 3) * 128 + (t >> 2) * 32 + (r & 7) * 4 + (t & 3);
}

// Register-prefetched staging: thread tid owns float4 slots e = tid + 128 j of the
// [rows x 4] float4 grid of a stage; load() issues the global reads of a stage,
// store() splits and writes them one stage later, so the reads of stage st+1 are in
// flight while stage st is converted and its MMAs run (round 1 loaded and stored in
// one step: every stage paid a full memory latency, ~100 us per cfg2 launch).
template <int J>
struct StageRegs {
  float4 v[J];
  __device__ __forceinline__ void load(const float* __restrict__ M, int r0, int nrows, int rlim, int d, int k0,
                                       int tid) {
    const bool vec = (d & 3) == 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int e = tid + kGThreads * j;
      const int r = e >> 2, t4 = e & 3;
      const int gr = r0 + r, gc = k0 + 4 * t4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nrows && gr < rlim) {
        const float* src = M + (size_t)gr * d + gc;
        if (vec && gc + 4 <= d) {
          x = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          x.x = gc < d ? __ldg(src) : 0.f;
          x.y = gc + 1 < d ? __ldg(src + 1) : 0.f;
          x.z = gc + 2 < d ? __ldg(src + 2) : 0.f;
          x.w = gc + 3 < d ? __ldg(src + 3) : 0.f;
        }
      }
      v[j] = x;
    }
  }
  __device__ __forceinline__ void store(int nrows, float* hi, float* lo, int tid) const {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int e = tid + kGThreads * j;
      const int r = e >> 2, t4 = e & 3;
      if (r >= nrows) continue;
      float h[4], l[4];
      split_tf32(v[j].x, h[0], l[0]);
      split_tf32(v[j].y, h[1], l[1]);
      split_tf32(v[j].z, h[2], l[2]);
      split_tf32(v[j].w, h[3], l[3]);
      const int o = core_idx(r, 4 * t4);
      *reinterpret_cast<float4*>(hi + o) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(lo + o) = make_float4(l[0], l[1], l[2], l[3]);
    }
  }
};

__global__ void __launch_bounds__(kGThreads, 1) gram_tc_kernel(GramArgs a) {
  extern __shared__ __align__(1024) float smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const GramJob jb = a.job[blockIdx.z];
  const int q = blockIdx.y, m0 = blockIdx.x * 128, k = a.k, d = a.d;
  if (m0 >= k) return;
  const float* Xq = jb.X + (size_t)q * k * d;
  const float* Yq = jb.Y + (size_t)q * k * d;
  float* Oq = jb.partial ? nullptr : jb.out + (size_t)q * k * k;
  const int mrows = min(128, k - m0);
  const int Nreal = jb.sym ? min(k, m0 + 128) : k;  // symmetric: lower block row only
  const int N = (Nreal + 15) & ~15;
  const int xs = 128 * kGK, ys = a.ys;               // floats per operand copy
  const int bufsz = 2 * xs + 2 * ys;                  // Xhi | Xlo | Yhi | Ylo
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * bufsz);  // [0..1] empty, [2] done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, a.tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nst = (d + kGK - 1) / kGK;
  // X: 128 rows x 4 float4 = 4 per thread; Y: N <= 304 rows -> up to 10 per thread
  // (slots beyond the tile are predicated off)
  StageRegs<4> px;
  StageRegs<(kGMaxN - 16) * 4 / kGThreads + 1> py;
  px.load(Xq, m0, 128, k, d, 0, tid);
  py.load(Yq, 0, N, Nreal, d, 0, tid);
  for (int st = 0; st < nst; ++st) {
    const int buf = st & 1;
    float* B = smem + buf * bufsz;
    if (st >= 2) {  // the MMAs that read this buffer (stage st-2) are done
      mbar_wait(&bar[buf], ((st - 2) >> 1) & 1);
    }
    px.store(128, B, B + xs, tid);
    py.store(N, B + 2 * xs, B + 2 * xs + ys, tid);
    if (st + 1 < nst) {  // next stage's reads in flight during this stage's MMAs
      px.load(Xq, m0, 128, k, d, (st + 1) * kGK, tid);
      py.load(Yq, 0, N, Nreal, d, (st + 1) * kGK, tid);
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t xh = su32(B), xl = su32(B + xs), yh = su32(B + 2 * xs), yl = su32(B + 2 * xs + ys);
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t ko = (uint32_t)ks * 256u;
        for (int n0 = 0; n0 < N; n0 += 256) {
          const int nn = min(256, N - n0);
          const uint32_t id = idesc_tf32_pos(nn);
          const uint32_t yo = (uint32_t)(n0 >> 3) * 512u;
          const uint32_t acc0 = (st > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(tbase + (uint32_t)n0, sdesc(xh + ko), sdesc(yh + yo + ko), id, acc0);
          mma_tf32(tbase + (uint32_t)n0, sdesc(xh + ko), sdesc(yl + yo + ko), id, 1u);
          mma_tf32(tbase + (uint32_t)n0, sdesc(xl + ko), sdesc(yh + yo + ko), id, 1u);
        }
      }
      mma_commit(&bar[buf]);
      if (st == nst - 1) mma_commit(&bar[2]);
    }
  }
  mbar_wait(&bar[2], 0);
  tc_fence_after();
  // epilogue: warp w reads TMEM lanes 32w.. (rows m0 + 32w + lane)
  const int r = m0 + 32 * warp + lane;
  const uint32_t tl = tbase + ((uint32_t)(32 * warp) << 16);
  if (jb.partial) {  // check_stationarity (solver.hpp:116-128): C G + lambda M.*C - R, squared, per row
    const bool live = 32 * warp + lane < mrows;
    const size_t ro = ((size_t)q * k + (live ? r : 0)) * k;
    double acc = 0.0;
    const bool vec = (k & 3) == 0;
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tmem_ld16(tl + (uint32_t)c0, v);
      if (live) {
        float mv[16], xv[16], rv[16];
        if (vec && c0 + 16 <= k) {  // 64 contiguous bytes of the row per array (float4 loads)
#pragma unroll
          for (int t4 = 0; t4 < 4; ++t4) {
            const float4 m4 = __ldg(reinterpret_cast<const float4*>(jb.M + ro + c0) + t4);
            const float4 x4 = __ldg(reinterpret_cast<const float4*>(Xq + (size_t)r * d + c0) + t4);
            const float4 r4 = __ldg(reinterpret_cast<const float4*>(jb.R + ro + c0) + t4);
            mv[4 * t4] = m4.x, mv[4 * t4 + 1] = m4.y, mv[4 * t4 + 2] = m4.z, mv[4 * t4 + 3] = m4.w;
            xv[4 * t4] = x4.x, xv[4 * t4 + 1] = x4.y, xv[4 * t4 + 2] = x4.z, xv[4 * t4 + 3] = x4.w;
            rv[4 * t4] = r4.x, rv[4 * t4 + 1] = r4.y, rv[4 * t4 + 2] = r4.z, rv[4 * t4 + 3] = r4.w;
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int c = c0 + t;
            mv[t] = c < k ? __ldg(jb.M + ro + c) : 0.f;
            xv[t] = c < k ? __ldg(Xq + (size_t)r * d + c) : 0.f;
            rv[t] = c < k ? __ldg(jb.R + ro + c) : 0.f;
          }
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          if (c0 + t < k) {
            const float e = v[t] + jb.lambda * (mv[t] * xv[t]) - rv[t];
            acc += (double)e * (double)e;
          }
        }
      }
    }
    if (live) jb.partial[(size_t)q * k + r] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, a.tcols);
    return;
  }
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tl + (uint32_t)c0, v);
    if (32 * warp + lane < mrows) {
      float* orow = Oq + (size_t)r * k;
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int c = c0 + t;
        if (c < Nreal && (!jb.sym || c <= r)) {
          orow[c] = v[t];
          if (jb.sym && c < r) Oq[(size_t)c * k + r] = v[t];  // mirror: G exactly symmetric
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, a.tcols);
}

}  // namespace

// two stages of X hi/lo (128 x 16) and Y hi/lo (round16(k) x 16) + barriers:
// 86 KB at k = 200, so two CTAs share an SM (TMEM 256 columns each)
size_t gram_tc_smem_bytes(int k) { return (size_t)(2 * (2 * 128 * kGK + 2 * ((k + 15) & ~15) * kGK)) * 4 + 64; }

// nprod products (X_i Y_i^T -> out_i, sym_i) over b pairs, k x d operands.
cudaError_t launch_gram_tc(int nprod, const float* const* X, const float* const* Y, float* const* out,
                           const int* sym, int64_t b, int k, int d, cudaStream_t st) {
  if (nprod < 1 || nprod > 4 || k < 1 || d < 1 || b < 1) return cudaErrorInvalidValue;
  if (k > kGMaxN - 16 || b > 65535) return cudaErrorNotSupported;
  GramArgs a{};
  for (int i = 0; i < nprod; ++i) a.job[i] = GramJob{X[i], Y[i], out[i], sym[i], nullptr, nullptr, 0.f, nullptr};
  a.k = k;
  a.d = d;
  a.ys = ((k + 15) & ~15) * kGK;
  a.tcols = ((k + 15) & ~15) <= 256 ? 256u : 512u;
  const size_t smem = gram_tc_smem_bytes(k);
  cudaError_t e = cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  note_launch("gram_tc_kernel");
  gram_tc_kernel<<<dim3((unsigned)((k + 127) / 128), (unsigned)b, (unsigned)nprod), kGThreads, smem, st>>>(a);
  return cudaGetLastError();
}

// Residual partials on the tensor cores: partial[q k + r] for C G (k x k, d = k).
cudaError_t launch_residual_tc(const float* C, const float* G, const float* R, const float* M, int64_t b, int k,
                               float lambda, double* partial, cudaStream_t st) {
  if (k < 1 || b < 1) return cudaErrorInvalidValue;
  if (k > kGMaxN - 16 || b > 65535 || std::getenv("FMAP_RESIDUAL_SIMT")) return cudaErrorNotSupported;
  GramArgs a{};
  a.job[0] = GramJob{C, G, nullptr, 0, M, R, lambda, partial};
  a.k = k;
  a.d = k;
  a.ys = ((k + 15) & ~15) * kGK;
  a.tcols = ((k + 15) & ~15) <= 256 ? 256u : 512u;
  const size_t smem = gram_tc_smem_bytes(k);
  cudaError_t e = cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  note_launch("gram_tc_kernel(residual)");
  gram_tc_kernel<<<dim3((unsigned)((k + 127) / 128), (unsigned)b, 1), kGThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace fmap
