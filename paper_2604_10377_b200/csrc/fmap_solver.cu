// Batched in-shared-memory Cholesky solver for the regularized functional map
// (see fmap_solver.cuh for the layout and the algorithm outline).
//
// Work split inside one CTA (256 threads, 8 warps), per 16-column panel p
// (columns [j, jn), next panel [jn, jn + nbn)):
//
//   step A  TRSM(p): L21 = A21 L11^{-T} by forward substitution, one row per
//           thread.  Warp 7 takes the next diagonal block's rows [jn, jn+nbn),
//           warps 0..6 the rows below (incl. the augmented rhs row).
//   ---- barrier ----
//   step B  warp 7 ("panel warp", the critical path): rank-16 update of the
//           next diagonal block, then its 16x16 Cholesky; afterwards it joins
//           the bulk.  Warps 0..6 (then 7): SYRK(p) of the trailing matrix in
//           32x16 warp tiles of 4x4 register tiles, pulled from a shared-memory
//           atomic counter (dynamic balance), skipping the diagonal block.
//   ---- barrier ----
//
// This replaces the reference's per-system PartialPivLU
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170); for SPD systems the
// solution is the same.  Singular = non-positive / non-finite pivot, rcond
// estimate min(pivot)/max|diag| below the threshold, or a non-finite solution.
#include "fmap_solver.cuh"

#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdlib>

namespace fmap {

namespace {

constexpr int kNT = 256;
constexpr int kNW = kNT / 32;
constexpr int kPW = kNW - 1;  // panel warp (SMSP 3)
// Warp 3 shares SMSP 3 with the panel warp and is kept idle so the critical path
// gets that scheduler (the arbiter is fair per SMSP): bulk = warps 0-2, 4-6.
constexpr int kIdleW = 3;
constexpr int kBulkThreads = (kNW - 2) * 32;
__device__ __forceinline__ int bulk_thread(int warp, int lane) {
  return ((warp < kIdleW) ? warp : warp - 1) * 32 + lane;
}

__device__ __forceinline__ int colbase(int c, int Rp) { return col_off(c, Rp) - (c & ~3); }

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ float f4get(const float4& v, int u) {
  return u == 0 ? v.x : (u == 1 ? v.y : (u == 2 ? v.z : v.w));
}

__device__ __forceinline__ float rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

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

// Offsets inside one panel.  Column j+t (j a multiple of 16) starts at
//   colbase(j+t) = base0 + t*stride - S4(t),  base0 = col_off(j) - j, stride = Rp - j,
//   S4(t) = sum_{u<t}(u&~3) + (t&~3);  element (r, j+t) is at colbase(j+t) + r.
__host__ __device__ constexpr int S4(int t) {
  int s = 0;
  for (int u = 0; u < t; ++u) s += u & ~3;
  return s + (t & ~3);
}

struct Panel {
  int base0, stride, j;
  __device__ __forceinline__ Panel(int j_, int Rp) : base0(col_off(j_, Rp) - j_), stride(Rp - j_), j(j_) {}
  __device__ __forceinline__ int col(int t) const { return base0 + t * stride - S4(t); }
};

__host__ __device__ constexpr int tri(int r, int c) { return r * (r + 1) / 2 + c; }

// Branch-free 8x8 Cholesky in registers (lower, row-major packed):
// t <- L (t[tri(p,p)] = L_pp), inv[p] = 1/L_pp.
__device__ __forceinline__ void chol8(float (&t)[36], float (&inv)[8], float& pivmin,
                                      unsigned& bad) {
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const float d = t[tri(p, p)];
    pivmin = fminf(pivmin, d);
    bad |= (unsigned)(!(d > 0.f)) | (unsigned)(!(d <= FLT_MAX));
    const float s = rsqrt_fast(d);
    inv[p] = s;
    t[tri(p, p)] = d * s;
#pragma unroll
    for (int r = p + 1; r < 8; ++r) t[tri(r, p)] *= s;
#pragma unroll
    for (int c = p + 1; c < 8; ++c)
#pragma unroll
      for (int r = c; r < 8; ++r) t[tri(r, c)] = fmaf(-t[tri(r, p)], t[tri(c, p)], t[tri(r, c)]);
  }
}

// Load / store the lower triangle of an 8x8 sub-block (local rows r0.., cols c0..)
// of the panel at j, in 4-row groups (LDS.128 / STS.128).  Positions above the
// diagonal inside the 4x4 diagonal pieces are layout junk and are written 0.
template <bool FULL>
__device__ __forceinline__ void ld_tri8(const float* A, const Panel& P, int r0, int c0, int nbe,
                                        float (&t)[36]) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int g = (c & ~3); g < 8; g += 4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (FULL || (c0 + c < nbe && r0 + g < nbe)) v = ld4(A + P.col(c0 + c) + P.j + r0 + g);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = g + u;
        if (r >= c) {
          float x = f4get(v, u);
          if (!FULL && !(c0 + c < nbe && r0 + r < nbe)) x = (r == c) ? 1.f : 0.f;
          t[tri(r, c)] = x;
        }
      }
    }
}

template <bool FULL>
__device__ __forceinline__ void st_tri8(float* A, const Panel& P, int r0, int c0, int nbe,
                                        const float (&t)[36]) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int g = (c & ~3); g < 8; g += 4) {
      if (FULL || (c0 + c < nbe && r0 + g < nbe)) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = (g + u >= c) ? t[tri(g + u, c)] : 0.f;
        st4(A + P.col(c0 + c) + P.j + r0 + g, make_float4(v[0], v[1], v[2], v[3]));
      }
    }
}

// Cholesky of the 16x16 diagonal block at (j, j) by one warp (all lanes):
//   L00 = chol(A00);  L10 = A10 L00^{-T};  L11 = chol(A11 - L10 L10^T)
// The 8x8 factorizations run replicated in every lane (no communication); the
// L10 rows are computed by lanes 0..7 and exchanged through `scr` (8x8 row-major).
// Writes L into the block and 1/L_tt into sinv[j..j+16).
template <bool FULL>
__device__ __noinline__ void diag16(float* A, int Rp, int j, int nbe, float* scr, float* sinv,
                                    int lane, float& pivmin, unsigned& bad) {
  const Panel P(j, Rp);
  float t[36], inv0[8], inv1[8];
  ld_tri8<FULL>(A, P, 0, 0, nbe, t);
  chol8(t, inv0, pivmin, bad);
  if (lane == 0) st_tri8<FULL>(A, P, 0, 0, nbe, t);
  {  // L10 row (8 + rr): forward substitution against L00 (every lane, row lane&7)
    const int rr = lane & 7;
    float a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      a[u] = (FULL || (8 + rr < nbe && u < nbe)) ? A[P.col(u) + j + 8 + rr] : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] *= inv0[u];
#pragma unroll
      for (int v = u + 1; v < 8; ++v) a[v] = fmaf(-a[u], t[tri(v, u)], a[v]);
    }
    if (lane < 8) {
      st4(scr + rr * 8, make_float4(a[0], a[1], a[2], a[3]));
      st4(scr + rr * 8 + 4, make_float4(a[4], a[5], a[6], a[7]));
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (FULL || (8 + rr < nbe && u < nbe)) A[P.col(u) + j + 8 + rr] = a[u];
    }
  }
  __syncwarp();
  // A11 - L10 L10^T: lane e < 36 computes packed element e (r, c) and publishes
  // it through scr[64..100); then every lane loads the updated block.
  {
    int r = 0, c = lane;
    while (c > r) {
      c -= r + 1;
      ++r;
    }
    if (lane < 36) {
      const float4 a0 = ld4(scr + r * 8), a1 = ld4(scr + r * 8 + 4);
      const float4 b0 = ld4(scr + c * 8), b1 = ld4(scr + c * 8 + 4);
      float acc = (FULL || (8 + r < nbe && 8 + c < nbe)) ? A[P.col(8 + c) + j + 8 + r] : (r == c ? 1.f : 0.f);
      acc = fmaf(-a0.x, b0.x, acc);
      acc = fmaf(-a0.y, b0.y, acc);
      acc = fmaf(-a0.z, b0.z, acc);
      acc = fmaf(-a0.w, b0.w, acc);
      acc = fmaf(-a1.x, b1.x, acc);
      acc = fmaf(-a1.y, b1.y, acc);
      acc = fmaf(-a1.z, b1.z, acc);
      acc = fmaf(-a1.w, b1.w, acc);
      scr[64 + lane] = acc;
    }
    __syncwarp();
    if (lane < 4) {  // lanes 32..35 are out of range; 4 lanes cover the last four
      int rr = 0, cc = 32 + lane;
      while (cc > rr) {
        cc -= rr + 1;
        ++rr;
      }
      const float4 a0 = ld4(scr + rr * 8), a1 = ld4(scr + rr * 8 + 4);
      const float4 b0 = ld4(scr + cc * 8), b1 = ld4(scr + cc * 8 + 4);
      float acc = (FULL || (8 + rr < nbe && 8 + cc < nbe)) ? A[P.col(8 + cc) + j + 8 + rr] : (rr == cc ? 1.f : 0.f);
      acc = fmaf(-a0.x, b0.x, acc);
      acc = fmaf(-a0.y, b0.y, acc);
      acc = fmaf(-a0.z, b0.z, acc);
      acc = fmaf(-a0.w, b0.w, acc);
      acc = fmaf(-a1.x, b1.x, acc);
      acc = fmaf(-a1.y, b1.y, acc);
      acc = fmaf(-a1.z, b1.z, acc);
      acc = fmaf(-a1.w, b1.w, acc);
      scr[96 + lane] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 36; e += 4) {
      const float4 v = ld4(scr + 64 + e);
      t[e] = v.x;
      t[e + 1] = v.y;
      t[e + 2] = v.z;
      t[e + 3] = v.w;
    }
  }
  chol8(t, inv1, pivmin, bad);
  if (lane == 0) {
    st_tri8<FULL>(A, P, 8, 8, nbe, t);
    st4(sinv + j, make_float4(inv0[0], inv0[1], inv0[2], inv0[3]));
    st4(sinv + j + 4, make_float4(inv0[4], inv0[5], inv0[6], inv0[7]));
    st4(sinv + j + 8, make_float4(inv1[0], inv1[1], inv1[2], inv1[3]));
    st4(sinv + j + 12, make_float4(inv1[4], inv1[5], inv1[6], inv1[7]));
  }
  __syncwarp();
}

// Cholesky of the 16x16 diagonal block at (j, j), lane r (< 16) owning row r:
// per column t one SHFL of the pivot, rsqrt, a scale, then (15 - t) SHFL + FFMA
// for the rank-1 update — ~290 instructions for the whole block, which matters
// because the panel warp shares its scheduler with busy SYRK warps.  Lanes
// 16..31 mirror lanes 0..15 (their results are discarded).  Writes L into the
// block and 1/L_tt into sinv[j..j+16).
template <bool FULL>
__device__ __noinline__ void diag16_shfl(float* A, int Rp, int j, int nbe, float* sinv, int lane,
                                         float& pivmin, unsigned& bad, int width = 32) {
  const Panel P(j, Rp);
  const int r = lane & 15;
  float a[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    float v = (r == c) ? 1.f : 0.f;
    if (c <= r && (FULL || (r < nbe && c < nbe))) v = A[P.col(c) + j + r];
    a[c] = v;
  }
  float sv = 0.f;  // lane t ends up holding 1/L_tt
#pragma unroll
  for (int t = 0; t < kNB; ++t) {
    const float d = __shfl_sync(0xffffffffu, a[t], t, width);
    pivmin = fminf(pivmin, d);
    bad |= (unsigned)(!(d > 0.f)) | (unsigned)(!(d <= FLT_MAX));
    const float s = rsqrt_fast(d);
    if (r == t) sv = s;
    a[t] *= s;  // L[r][t] (lane t: sqrt(d))
#pragma unroll
    for (int c = t + 1; c < kNB; ++c) {
      const float l = __shfl_sync(0xffffffffu, a[t], c, width);  // L[c][t]
      a[c] = fmaf(-a[t], l, a[c]);
    }
  }
  if (lane < 16 || width == 16) {
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (c <= r && (FULL || (r < nbe && c < nbe))) A[P.col(c) + j + r] = a[c];
    if (FULL || r < nbe) sinv[j + r] = sv;
  }
  __syncwarp();
}

// Cholesky of the 16x16 diagonal block at (j, j), lane-per-row (lane & 15 = row
// r; lanes 16..31 may factor a second system's block), ONE shared-memory
// exchange per pivot: every lane publishes its raw column-t entry a[r][t] to
// xbuf, then each lane reads the whole column (4 LDS.128 broadcasts) and derives
// the pivot d = a[t][t], s = 1/sqrt(d), its own L[r][t] = a[r][t]*s and the
// rank-1 update a[r][c] -= (a[r][t]/d) * a[c][t] locally.  ~25 instructions and
// one exchange per pivot.  xbuf: 16 floats per half-warp, 16-byte aligned.
template <bool FULL>
__device__ __forceinline__ void diag16_x1(float* A, int Rp, int j, int nbe, float* sinv, float* xbuf,
                                       int lane, float& pivmin, unsigned& bad) {
  const Panel P(j, Rp);
  const int r = lane & 15;
  float a[kNB], lr[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    float v = (r == c) ? 1.f : 0.f;
    if (c <= r && (FULL || (r < nbe && c < nbe))) v = A[P.col(c) + j + r];
    a[c] = v;
  }
  float sv = 0.f;
#pragma unroll
  for (int t = 0; t < kNB; ++t) {
    xbuf[r] = a[t];
    __syncwarp();
    float col[kNB];
#pragma unroll
    for (int g = 0; g < kNB; g += 4) {
      const float4 v = ld4(xbuf + g);
      col[g] = v.x;
      col[g + 1] = v.y;
      col[g + 2] = v.z;
      col[g + 3] = v.w;
    }
    __syncwarp();
    const float d = col[t];
    pivmin = fminf(pivmin, d);
    bad |= (unsigned)(!(d > 0.f)) | (unsigned)(!(d <= FLT_MAX));
    const float s = rsqrt_fast(d);
    const float w = a[t] * (s * s);  // a[r][t] / d
    lr[t] = a[t] * s;                // L[r][t]
    if (r == t) sv = s;
#pragma unroll
    for (int c = t + 1; c < kNB; ++c) a[c] = fmaf(-w, col[c], a[c]);
  }
  if (FULL || r < nbe) {
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (c <= r && (FULL || c < nbe)) A[P.col(c) + j + r] = lr[c];
    sinv[j + r] = sv;
  }
  __syncwarp();
}

// Cholesky of the 16x16 diagonal block, lane-per-row (lane & 15 = row r; the
// upper half-warp may factor a second system), in 4-pivot blocks: per block b
//   1. rows 4b..4b+3 publish their raw entries of columns 4b..4b+3 (STS.128);
//      every lane factors that 4x4 pivot block locally (replicated, no comms);
//   2. each lane solves its own row of L for these 4 columns (4-step chain)
//      and publishes it (STS.128);
//   3. each lane applies the rank-4 update to its remaining columns from the
//      published L rows (LDS.128 broadcasts).
// Two exchanges per 4 pivots instead of one per pivot.  xbuf: 64 floats per
// half-warp (16 rows x 4), 16-byte aligned.
template <bool FULL>
__device__ __noinline__ void diag16_b4(float* A, int Rp, int j, int nbe, float* sinv, float* xbuf,
                                       int lane, float& pivmin, unsigned& bad) {
  const Panel P(j, Rp);
  const int r = lane & 15;
  float a[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    float v = (r == c) ? 1.f : 0.f;
    if (c <= r && (FULL || (r < nbe && c < nbe))) v = A[P.col(c) + j + r];
    a[c] = v;
  }
  float sv[4] = {0.f, 0.f, 0.f, 0.f};  // 1/L_tt of this lane's own pivot block
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int t0 = 4 * b;
    // 1. publish raw pivot-block rows, factor the 4x4 block locally
    if ((r >> 2) == b) st4(xbuf + 4 * r, make_float4(a[t0], a[t0 + 1], a[t0 + 2], a[t0 + 3]));
    __syncwarp();
    float p4[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 v = ld4(xbuf + 4 * (t0 + u));
      p4[u][0] = v.x;
      p4[u][1] = v.y;
      p4[u][2] = v.z;
      p4[u][3] = v.w;
    }
    __syncwarp();
    float inv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float d = p4[q][q];
      pivmin = fminf(pivmin, d);
      bad |= (unsigned)(!(d > 0.f)) | (unsigned)(!(d <= FLT_MAX));
      const float s = rsqrt_fast(d);
      inv[q] = s;
      p4[q][q] = d * s;
#pragma unroll
      for (int u = q + 1; u < 4; ++u) p4[u][q] *= s;
#pragma unroll
      for (int c = q + 1; c < 4; ++c)
#pragma unroll
        for (int u = c; u < 4; ++u) p4[u][c] = fmaf(-p4[u][q], p4[c][q], p4[u][c]);
    }
    // 2. own row of L for columns t0..t0+3: x = a[t0..] L4^{-T}
    float x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v = a[t0 + q];
#pragma unroll
      for (int u = 0; u < q; ++u) v = fmaf(-x[u], p4[q][u], v);
      x[q] = v * inv[q];
    }
    if ((r >> 2) == b) {  // rows of the pivot block: L from the local factor
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float v = 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u == (r & 3) && q <= u) v = p4[u][q];
        x[q] = v;
        if (q == (r & 3)) sv[b] = inv[q];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) a[t0 + q] = x[q];
    st4(xbuf + 4 * r, make_float4(x[0], x[1], x[2], x[3]));
    __syncwarp();
    // 3. rank-4 update of the remaining columns c > t0+3 (this row only)
#pragma unroll
    for (int c = t0 + 4; c < kNB; ++c) {
      const float4 l = ld4(xbuf + 4 * c);  // L[c][t0..t0+3]
      float v = a[c];
      v = fmaf(-x[0], l.x, v);
      v = fmaf(-x[1], l.y, v);
      v = fmaf(-x[2], l.z, v);
      v = fmaf(-x[3], l.w, v);
      a[c] = v;
    }
    __syncwarp();
  }
  if (FULL || r < nbe) {
#pragma unroll
    for (int c = 0; c < kNB; ++c)
      if (c <= r && (FULL || c < nbe)) A[P.col(c) + j + r] = a[c];
    float s = sv[0];
#pragma unroll
    for (int b = 1; b < 4; ++b)
      if ((r >> 2) == b) s = sv[b];
    sinv[j + r] = s;
  }
  __syncwarp();
}

// In-place inverse of the lower-triangular 16x16 diagonal block at (j, j) (L with
// 1/L_tt in sinv).  Lane c computes column c of L^{-1} right-looking: x_u =
// acc_u / L_uu, then acc_r -= L[r][u] x_u for r > u — an FMUL->FFMA chain per
// column with the L column loads (LDS.128 broadcasts) off the chain.  Lanes need
// no predicates: for u < c the accumulators stay 0.
template <bool FULL>
__device__ __forceinline__ void invert_diag16(float* A, int Rp, int j, int nbe, const float* sinv,
                                              int c) {
  const Panel P(j, Rp);
  float acc[kNB];
#pragma unroll
  for (int r = 0; r < kNB; ++r) acc[r] = (r == c) ? 1.f : 0.f;
#pragma unroll
  for (int u = 0; u < kNB; ++u) {
    if (FULL || u < nbe) {
      const float xu = acc[u] * sinv[j + u];
      acc[u] = xu;
#pragma unroll
      for (int g = ((u + 1) & ~3); g < kNB; g += 4) {
        if (FULL || g < nbe) {
          const float4 l = ld4(A + P.col(u) + j + g);  // L[g..g+3][u]
#pragma unroll
          for (int w = 0; w < 4; ++w)
            if (g + w > u) acc[g + w] = fmaf(-f4get(l, w), xu, acc[g + w]);
        }
      }
    }
  }
  __syncwarp();
  if (FULL || c < nbe) {
    float* col = A + P.col(c) + j;
#pragma unroll
    for (int r = 0; r < kNB; ++r)
      if ((FULL || r < nbe) && r >= c) col[r] = acc[r];
  }
  __syncwarp();
}

// Back-substitution step of the panel warp for one 16-row block B at jb (the
// diagonal block already holds L_BB^{-1}): lane g (< 16) forms x_g =
// (L_BB^{-T} y_B)_g, publishes x_B to xs[16..32), then (if a block above
// exists) applies x_B and the previous block's x (xs[0..16), rows jprev..)
// to entry jnext+g.  FULL: nbe == 16 (every block but possibly the last).
template <bool FULL, bool LAG_FULL>
__device__ __forceinline__ void backsub_block(float* A, int Rp, float* xv, float* xcur,
                                              const float* xprev, int jb, int nbe, int jnext,
                                              int jprev, int nprev, int g) {
  float y = 0.f;
  if (FULL || g < nbe) {
    const float* colg = A + colbase(jb + g, Rp) + jb;  // L_BB^{-1}[r][g], r >= g
#pragma unroll
    for (int r4 = 0; r4 < kNB; r4 += 4) {
      if ((FULL || r4 < nbe) && r4 + 3 >= (g & ~3)) {
        const float4 l = ld4(colg + r4);
        const float4 yy = ld4(xv + jb + r4);
        y = fmaf(r4 >= g ? l.x : 0.f, yy.x, y);
        y = fmaf(r4 + 1 >= g ? l.y : 0.f, yy.y, y);
        y = fmaf(r4 + 2 >= g ? l.z : 0.f, yy.z, y);
        y = fmaf(r4 + 3 >= g ? l.w : 0.f, yy.w, y);
      }
    }
  }
  __syncwarp();
  if (FULL || g < nbe) {
    xv[jb + g] = y;
    xcur[g] = y;
  }
  __syncwarp();
  if (jnext >= 0) {
    const float* col = A + colbase(jnext + g, Rp);
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < kNB; r += 4) {
      if (FULL || r < nbe) {
        const float4 l = ld4(col + jb + r);
        const float4 xx = ld4(xcur + r);
        acc = fmaf(l.x, xx.x, acc);
        acc = fmaf(l.y, xx.y, acc);
        acc = fmaf(l.z, xx.z, acc);
        acc = fmaf(l.w, xx.w, acc);
      }
    }
    if (jprev >= 0) {
#pragma unroll
      for (int r = 0; r < kNB; r += 4) {
        if (LAG_FULL || r < nprev) {
          const float4 l = ld4(col + jprev + r);
          const float4 xx = ld4(xprev + r);
          acc = fmaf(l.x, xx.x, acc);
          acc = fmaf(l.y, xx.y, acc);
          acc = fmaf(l.z, xx.z, acc);
          acc = fmaf(l.w, xx.w, acc);
        }
      }
    }
    xv[jnext + g] -= acc;
  }
}

// TRSM of one row r of panel [j, j+nbe): x = a L11^{-T} by forward substitution
// (right-looking over the columns of L11, LDS.128 broadcasts).
template <bool FULL>
__device__ __forceinline__ void trsm_row(float* A, const Panel& P, const float* sinv, int nbe,
                                         int r) {
  float a[kNB];
#pragma unroll
  for (int t = 0; t < kNB; ++t) a[t] = (FULL || t < nbe) ? A[P.col(t) + r] : 0.f;
#pragma unroll
  for (int u = 0; u < kNB; ++u) {
    if (FULL || u < nbe) {
      a[u] *= sinv[P.j + u];
#pragma unroll
      for (int g = ((u + 1) & ~3); g < kNB; g += 4) {
        if (FULL || g < nbe) {
          const float4 l = ld4(A + P.col(u) + P.j + g);  // L11[g..g+3][u]
#pragma unroll
          for (int w = 0; w < 4; ++w)
            if (g + w > u) a[g + w] = fmaf(-a[u], f4get(l, w), a[g + w]);
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < kNB; ++t)
    if (FULL || t < nbe) A[P.col(t) + r] = a[t];
}

// 4x4 register tile: A[r0..r0+3][c0..c0+3] -= sum_{t<nbe} L[r][j+t] L[c][j+t].
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

// 8x4 register tile: rows r0a..r0a+3 and r0b..r0b+3 (two 4-row groups, 32 rows
// apart so that the 8 row-lanes of a warp read one contiguous 128-byte segment
// per group), columns c0..c0+3.  va / vb: the group lies on or below the
// diagonal (otherwise its destination is not stored and is skipped).
template <bool FULL>
__device__ __forceinline__ void syrk_tile84(float* A, int Rp, const Panel& P, int nbe, int r0a,
                                            int r0b, int c0, bool va, bool vb) {
  float acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  const float* pa = A + P.base0 + r0a;
  const float* pb = A + P.base0 + r0b;
  const float* pc = A + P.base0 + c0;
  auto step = [&](const float4 xa, const float4 xb, const float4 y) {
    const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
    const float yr[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xr[a], yr[b], acc[a][b]);
  };
  if (FULL) {
#pragma unroll
    for (int t = 0; t < kNB; ++t) {
      const int o = t * P.stride - S4(t);
      step(ld4(pa + o), ld4(pb + o), ld4(pc + o));
    }
  } else {
    for (int t = 0; t < nbe; ++t) {
      step(ld4(pa), ld4(pb), ld4(pc));
      const int st = P.stride - ((t + 1) & ~3);
      pa += st;
      pb += st;
      pc += st;
    }
  }
  const int qs = Rp - c0;
  float* qa = A + col_off(c0, Rp) - c0 + r0a;
  float* qb = A + col_off(c0, Rp) - c0 + r0b;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (va) {
      float4 v = ld4(qa + b * qs);
      v.x -= acc[0][b];
      v.y -= acc[1][b];
      v.z -= acc[2][b];
      v.w -= acc[3][b];
      st4(qa + b * qs, v);
    }
    if (vb) {
      float4 v = ld4(qb + b * qs);
      v.x -= acc[4][b];
      v.y -= acc[5][b];
      v.z -= acc[6][b];
      v.w -= acc[7][b];
      st4(qb + b * qs, v);
    }
  }
}

// ---------------------------------------------------------------------------
// Tensor-core SYRK (legacy mma.sync m16n8k8 TF32 with 3xTF32 splitting, ~fp32
// accuracy): a warp updates a block of 32 columns x 64 rows,
//   A[r][c] -= sum_{t<16} L[r][j+t] L[c][j+t]    (panel j always 16 wide).
// MMA M = output columns, N = output rows, K = panel columns, so a lane's
// accumulator pair (d0,d1) is rows (2*t4, 2*t4+1) of one column: contiguous in
// the column-major layout (LDS.64 / STS.64).  Fragments (g = lane/4, t4 = lane%4):
//   a0..a3 = L[c0+g(+8)][j+t4(+4)],  b0,b1 = L[r0+g][j+t4(+4)].
// Positions above the stored triangle / outside the matrix are not written.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0,
                                         unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NT_M, int NT_N>  // 16-column m-tiles, 8-row n-tiles
__device__ __forceinline__ void syrk_mma_block(float* A, int Rp, int K4, const Panel& P, int r0,
                                               int c0, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  float acc[NT_M][NT_N][4];
#pragma unroll
  for (int m = 0; m < NT_M; ++m)
#pragma unroll
    for (int n = 0; n < NT_N; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[m][n][e] = 0.f;
  const int rmax = Rp - 1;
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const int ta = 8 * ks + t4, tb = ta + 4;  // panel columns of this lane
    const float* colA = A + P.col(ta);
    const float* colB = A + P.col(tb);
    unsigned ahi[NT_M][4], alo[NT_M][4];
#pragma unroll
    for (int m = 0; m < NT_M; ++m) {
      const int ca = min(c0 + 16 * m + g, rmax), cb = min(c0 + 16 * m + g + 8, rmax);
      split_tf32(colA[ca], ahi[m][0], alo[m][0]);
      split_tf32(colA[cb], ahi[m][1], alo[m][1]);
      split_tf32(colB[ca], ahi[m][2], alo[m][2]);
      split_tf32(colB[cb], ahi[m][3], alo[m][3]);
    }
#pragma unroll
    for (int n = 0; n < NT_N; ++n) {
      const int rr = min(r0 + 8 * n + g, rmax);
      unsigned bh0, bl0, bh1, bl1;
      split_tf32(colA[rr], bh0, bl0);
      split_tf32(colB[rr], bh1, bl1);
#pragma unroll
      for (int m = 0; m < NT_M; ++m) {
        mma_tf32(acc[m][n], ahi[m], bh0, bh1);
        mma_tf32(acc[m][n], ahi[m], bl0, bl1);
        mma_tf32(acc[m][n], alo[m], bh0, bh1);
      }
    }
  }
  // d0,d1: (row r0+8n+2t4 (+1), col c0+16m+g); d2,d3: col + 8
#pragma unroll
  for (int m = 0; m < NT_M; ++m)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int c = c0 + 16 * m + g + 8 * half;
      if (c >= K4) continue;
      float* col = A + colbase(c, Rp);
#pragma unroll
      for (int n = 0; n < NT_N; ++n) {
        const int r = r0 + 8 * n + 2 * t4;
        if (r >= (c & ~3) && r < Rp) {  // r even, Rp multiple of 4: r+1 < Rp too
          float2 v = *reinterpret_cast<float2*>(col + r);
          v.x -= acc[m][n][2 * half];
          v.y -= acc[m][n][2 * half + 1];
          *reinterpret_cast<float2*>(col + r) = v;
        }
      }
    }
}

// One 64x16 warp tile (column block cb, row block starting at rb) of SYRK(p):
// lane (lr = lane&7, lc = lane>>3) owns rows rb+4lr.., rb+32+4lr.. and columns
// cb+4lc..  Skips 4x4 groups above the diagonal, outside the matrix or inside
// the excluded diagonal block [db, db+dbn)^2.
template <bool FULL>
__device__ __forceinline__ void syrk_warp_tile(float* A, int Rp, int K4, const Panel& P, int nbe,
                                               int cb, int rb, int db, int dbn, int lane) {
  const int lr = lane & 7, lc = lane >> 3;
  const int c0 = cb + 4 * lc;
  if (c0 >= K4) return;
  const int ra = rb + 4 * lr, rbb = rb + 32 + 4 * lr;
  const bool cin = c0 < db + dbn;
  const bool va = ra < Rp && ra >= c0 && !(cin && ra < db + dbn);
  const bool vb = rbb < Rp && rbb >= c0 && !(cin && rbb < db + dbn);
  if (!va && !vb) return;
  // operand rows must exist even for a skipped group: clamp to a valid row
  syrk_tile84<FULL>(A, Rp, P, nbe, va ? ra : rbb, vb ? rbb : ra, c0, va, vb);
}

// Bulk SYRK(p) over columns [c_lo, K4), rows >= column, skipping the diagonal
// block [db, db+dbn)^2 (handled by the panel warp).  Warp tiles of 32 rows x 16
// columns (lanes 8 x 4, 4x4 each) are pulled from *counter.
template <bool FULL>
__device__ __forceinline__ void syrk_bulk(float* A, int Rp, int K4, const Panel& P, int nbe,
                                          int c_lo, int db, int dbn, int* counter, int lane) {
  const int ncb = (K4 - c_lo + 15) >> 4;
  while (true) {
    int w = 0;
    if (lane == 0) w = atomicAdd(counter, 1);
    w = __shfl_sync(0xffffffffu, w, 0);
    int u = 0, cb = c_lo, nrb = (Rp - cb + 63) >> 6;
    while (u < ncb && w >= nrb) {
      w -= nrb;
      ++u;
      cb += 16;
      nrb = (Rp - cb + 63) >> 6;
    }
    if (u >= ncb) break;
    syrk_warp_tile<FULL>(A, Rp, K4, P, nbe, cb, cb + (w << 6), db, dbn, lane);
  }
}

}  // namespace

// Optional phase tracing (debug): p.trace != nullptr records clock64() per warp
// for block p.trace_block at fixed slots (end-of-work stamps only).
#define FMAP_TRACE(slot)                                                        \
  do {                                                                          \
    if (p.trace && blockIdx.x == (unsigned)p.trace_block && lane == 0)          \
      p.trace[warp * 1024 + (slot)] = clock64();                                \
  } while (0)

template <int MASK_MODE>
__global__ void __launch_bounds__(kNT, 2) chol_solve_kernel(SolveParams p) {
  extern __shared__ __align__(16) float smem[];
  const int k = p.k, K4 = p.K4, Rp = p.Rp;
  const int P_ = packed_size(K4);
  float* A = smem;
  float* xv = smem + P_;   // K4: back-substitution vector
  float* sinv = xv + K4;   // K4: 1/L_tt
  float* scr = sinv + K4;  // 104: diag scratch (L10 8x8 + updated A11)
  unsigned* sc = reinterpret_cast<unsigned*>(scr + 104);  // 32 words of scalars
  int* counter = reinterpret_cast<int*>(sc + 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t s = p.sys_offset + blockIdx.x;
  const int64_t q = s / k;
  const int i = (int)(s - q * k);

  if (tid == 0) {
    sc[0] = 0u;  // max |diag| (float bits)
    sc[1] = 0u;  // ev_max bits
    *counter = 0;
  }
  // ---- stage G (row c of G == column c, symmetric) with cp.async; padding + rhs row ----
  {
    const float* Gq = p.gram + (size_t)q * k * k;
    const float* Rrow = p.rhs + ((size_t)q * k + i) * k;
    const bool vec = (k & 3) == 0;
    for (int c = warp; c < K4; c += kNW) {
      const int c4 = c & ~3;
      float* col = A + colbase(c, Rp);
      if (c < k) {
        const float* g = Gq + (size_t)c * k;
        if (vec) {
          for (int r = c4 + 4 * lane; r < k; r += 128) cp_async16(col + r, g + r);
        } else {
          for (int r = c4 + lane; r < k; r += 32) cp_async4(col + r, g + r);
        }
        for (int r = k + lane; r < Rp; r += 32)
          col[r] = (r == K4) ? (p.rhs_unit < 0 ? Rrow[c] : (c == p.rhs_unit ? 1.f : 0.f)) : 0.f;
      } else {
        for (int r = c4 + lane; r < Rp; r += 32) col[r] = (r == c) ? 1.f : 0.f;
      }
    }
  }
  float ev_max = 0.f;
  if constexpr (MASK_MODE == 1) {
    float m = 0.f;
    for (int c = tid; c < k; c += kNT)
      m = fmaxf(m, fmaxf(p.ev1[(size_t)q * k + c], p.ev2[(size_t)q * k + c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    __syncthreads();  // sc[] initialised
    if (lane == 0) atomicMax(&sc[1], __float_as_uint(m));
  }
  cp_async_wait_all();
  __syncthreads();
  if constexpr (MASK_MODE == 1) {
    ev_max = __uint_as_float(sc[1]);
    if (!(ev_max > 0.f)) {
      if (tid == 0) atomicOr(p.flags, 32u);
      return;  // masks.hpp:59: needs a non-zero spectrum to normalize by
    }
  }
  {  // diagonal: + lambda * m_i(c) + ridge
    float dmax = 0.f;
    for (int c = tid; c < k; c += kNT) {
      float* d = A + colbase(c, Rp) + c;
      const float v = *d + (p.lambda * mask_entry<MASK_MODE>(p, q, i, c, ev_max) + p.ridge);
      *d = v;
      dmax = fmaxf(dmax, fabsf(v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0) atomicMax(&sc[0], __float_as_uint(dmax));
  }
  __syncthreads();
  FMAP_TRACE(0);

  float pivmin = FLT_MAX;
  unsigned bad = 0u;
  if (warp == kPW) {
    if (K4 >= kNB) diag16<true>(A, Rp, 0, kNB, scr, sinv, lane, pivmin, bad);
    else diag16<false>(A, Rp, 0, K4, scr, sinv, lane, pivmin, bad);
  }
  __syncthreads();
  FMAP_TRACE(1);

  for (int j = 0; j < K4; j += kNB) {
    const int ts = 8 + (j / kNB) * 8;
    const int nbe = min(kNB, K4 - j);
    const int jn = j + nbe;
    const int nbn = min(kNB, K4 - jn);
    const Panel Pj(j, Rp);
    const bool full = nbe == kNB;
    // A: TRSM(p).  Panel warp: the next diagonal block's rows; others: the rest.
    if (warp == kPW) {
      if (lane < nbn) {
        if (full) trsm_row<true>(A, Pj, sinv, nbe, jn + lane);
        else trsm_row<false>(A, Pj, sinv, nbe, jn + lane);
      }
    } else if (warp != kIdleW) {
      for (int r = jn + max(nbn, 0) + bulk_thread(warp, lane); r < Rp; r += kBulkThreads) {
        if (full) trsm_row<true>(A, Pj, sinv, nbe, r);
        else trsm_row<false>(A, Pj, sinv, nbe, r);
      }
    }
    if (tid == 0) *counter = 0;
    FMAP_TRACE(ts + 0);
    __syncthreads();
    if (nbn <= 0) break;
    // B: panel warp -> diagonal-block update + Cholesky, then bulk; others -> bulk SYRK(p)
    if (warp == kPW) {
      // rank-nbe update of the diagonal block [jn, jn+nbn)^2 in 2x2 tiles (36 for
      // a full block) spread over the 32 lanes
      const int nt2 = nbn >> 1;
      const int tcount = nt2 * (nt2 + 1) / 2;
      for (int e = lane; e < tcount; e += 32) {
        int a = 0, l = e;
        while (l > a) {
          l -= a + 1;
          ++a;
        }
        const int r0 = jn + 2 * a, c0 = jn + 2 * l;
        float acc00 = 0.f, acc01 = 0.f, acc10 = 0.f, acc11 = 0.f;
        const float* pr = A + Pj.base0 + r0;
        const float* pc = A + Pj.base0 + c0;
        for (int t = 0; t < nbe; ++t) {
          const float2 x = *reinterpret_cast<const float2*>(pr);
          const float2 y = *reinterpret_cast<const float2*>(pc);
          acc00 = fmaf(x.x, y.x, acc00);
          acc01 = fmaf(x.x, y.y, acc01);
          acc10 = fmaf(x.y, y.x, acc10);
          acc11 = fmaf(x.y, y.y, acc11);
          const int step = Pj.stride - ((t + 1) & ~3);
          pr += step;
          pc += step;
        }
        float* q0 = A + colbase(c0, Rp) + r0;
        float* q1 = A + colbase(c0 + 1, Rp) + r0;
        q0[0] -= acc00;
        q0[1] -= acc10;
        q1[0] -= acc01;
        q1[1] -= acc11;
      }
      __syncwarp();
      if (nbn == kNB) diag16<true>(A, Rp, jn, nbn, scr, sinv, lane, pivmin, bad);
      else diag16<false>(A, Rp, jn, nbn, scr, sinv, lane, pivmin, bad);
      FMAP_TRACE(ts + 2);
    }
    if (warp != kIdleW) {
      if (full) syrk_bulk<true>(A, Rp, K4, Pj, nbe, jn, jn, nbn, counter, lane);
      else syrk_bulk<false>(A, Rp, K4, Pj, nbe, jn, jn, nbn, counter, lane);
    }
    FMAP_TRACE(ts + 4);
    __syncthreads();
  }
  FMAP_TRACE(1000);

  // ---- back substitution L^T x = y (y = augmented row K4) ----
  // Blocks of 16 rows, last to first.  Step s: the panel warp solves block s
  // (lane g holds y_g; column c: x_c = y_c / L_cc, one SHFL broadcast, lanes
  // g < c subtract L[c][g] x_c — ~3 instructions per column) and applies x_s to
  // block s+1's entries; meanwhile the other warps apply x_{s-1} to all rows
  // above block s+1.  One barrier per block; every entry of block s has all
  // contributions of blocks < s before step s starts.
  for (int c = tid; c < K4; c += kNT) xv[c] = A[colbase(c, Rp) + K4];
  __syncthreads();
  float* xs = scr;  // x of the previous block (16 floats)
  int jprev = -1, nprev = 0;
  for (int jb = ((K4 - 1) / kNB) * kNB; jb >= 0; jb -= kNB) {
    const int nbe = min(kNB, K4 - jb);
    const int jnext = jb - kNB;  // next block (above), may be < 0
    if (warp == kPW) {
      // column g of L_BB below the diagonal, preloaded per lane: L[jb+r][jb+g], r > g
      const int g = lane;
      float lcol[kNB];
      const float* colg = A + colbase(jb + min(g, kNB - 1), Rp) + jb;
#pragma unroll
      for (int r4 = 0; r4 < kNB; r4 += 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g < nbe && r4 + 3 >= (g & ~3) && r4 < nbe) v = ld4(colg + r4);
        lcol[r4] = v.x;
        lcol[r4 + 1] = v.y;
        lcol[r4 + 2] = v.z;
        lcol[r4 + 3] = v.w;
      }
      float y = (g < nbe) ? xv[jb + g] : 0.f;
      const float sg = (g < nbe) ? sinv[jb + g] : 0.f;
#pragma unroll
      for (int c = kNB - 1; c >= 0; --c) {
        if (c < nbe) {
          const float xc = __shfl_sync(0xffffffffu, y * sg, c);
          if (g == c) y = xc;
          if (g < c) y = fmaf(-lcol[c], xc, y);
        }
      }
      if (g < nbe) {
        xv[jb + g] = y;
        xs[16 + g] = y;  // publish x_s for the lagged bulk update of the next step
      }
      __syncwarp();
      // x_s and the lagged x_{s-1} applied to block s+1's entries (lanes 0..15);
      // the other warps cover x_{s-1} only for rows above block s+1.
      if (jnext >= 0 && g < kNB) {
        const float* col = A + colbase(jnext + g, Rp);
        float acc = 0.f;
#pragma unroll
        for (int r = 0; r < kNB; r += 4) {
          if (r < nbe) {
            const float4 l = ld4(col + jb + r);
            const float4 xx = ld4(xs + 16 + r);
            acc = fmaf(l.x, xx.x, acc);
            acc = fmaf(l.y, xx.y, acc);
            acc = fmaf(l.z, xx.z, acc);
            acc = fmaf(l.w, xx.w, acc);
          }
        }
        if (jprev >= 0) {
#pragma unroll
          for (int r = 0; r < kNB; r += 4) {
            if (r < nprev) {
              const float4 l = ld4(col + jprev + r);
              const float4 xx = ld4(xs + r);
              acc = fmaf(l.x, xx.x, acc);
              acc = fmaf(l.y, xx.y, acc);
              acc = fmaf(l.z, xx.z, acc);
              acc = fmaf(l.w, xx.w, acc);
            }
          }
        }
        xv[jnext + g] -= acc;
      }
    } else if (jprev >= 0 && warp != kIdleW) {
      // lagged: x_{s-1} (block at jprev) applied to rows c < jnext
      for (int c = bulk_thread(warp, lane); c < jnext; c += kBulkThreads) {
        const float* col = A + colbase(c, Rp) + jprev;
        float acc = 0.f;
#pragma unroll
        for (int r = 0; r < kNB; r += 4) {
          if (r < nprev) {
            const float4 l = ld4(col + r);
            const float4 xx = ld4(xs + r);
            acc = fmaf(l.x, xx.x, acc);
            acc = fmaf(l.y, xx.y, acc);
            acc = fmaf(l.z, xx.z, acc);
            acc = fmaf(l.w, xx.w, acc);
          }
        }
        xv[c] -= acc;
      }
    }
    __syncthreads();
    if (warp == kPW && lane < 4) st4(xs + 4 * lane, ld4(xs + 16 + 4 * lane));  // x_s -> lag slot
    jprev = jb;
    nprev = nbe;
    __syncthreads();
  }
  if (warp != kPW) return;
  FMAP_TRACE(1001);
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


// ===========================================================================
// Two systems per CTA in lockstep (1 CTA / SM, 16 warps).  The panel warp (15)
// factors both systems' diagonal blocks at once (lanes 0..15: system 0,
// 16..31: system 1), which halves the per-system cost of the latency-bound
// critical path; warps 0..14 share TRSM / SYRK / back-substitution work of both
// systems.  Per panel:
//   A  TRSM(p), all rows >= jn of both systems        (bulk)
//   B  SYRK of the next panel's columns [jn, jn+nbn)  (bulk, incl. diag block)
//   C  panel warp: 16x16 Cholesky of both next diagonal blocks
//      bulk:       SYRK(p) of the remaining trailing matrix (dynamic tiles)
// ===========================================================================
constexpr int kNT2 = 512;
constexpr int kNW2 = kNT2 / 32;
constexpr int kPW2 = kNW2 - 1;
constexpr int kBulk2 = kNT2 - 32;

// ISO: warps 3, 7, 11 stay idle so SMSP 3 (wid % 4 == 3) hosts only the panel
// warp 15 — the per-SMSP issue arbiter is fair, so this is the only way to give
// the latency-bound critical path a scheduler of its own.
template <bool ISO>
__device__ __forceinline__ bool pair_bulk(int warp) {
  return ISO ? ((warp & 3) != 3) : (warp != kPW2);
}
template <bool ISO>
__device__ __forceinline__ int pair_bt(int warp, int lane) {
  return (ISO ? (warp - (warp >> 2)) : warp) * 32 + lane;
}
template <bool ISO>
__host__ __device__ constexpr int pair_nbulk() { return ISO ? 12 * 32 : kBulk2; }

__host__ __device__ __forceinline__ int pair_stride_floats(int K4) {
  return packed_size(K4) + 2 * K4 + 32;  // matrix, xv, sinv, 32 scratch floats
}

template <int MASK_MODE, bool ISO, int NS>
__global__ void __launch_bounds__(kNT2, 1) chol_pair_kernel(SolveParams p) {
  static_assert(NS == 1 || NS == 2, "one or two systems per CTA");
  constexpr int NB_T = pair_nbulk<ISO>();
  extern __shared__ __align__(16) float smem[];
  const int k = p.k, K4 = p.K4, Rp = p.Rp;
  const int Pn = packed_size(K4);
  const int SYS = pair_stride_floats(K4);
  unsigned* sc = reinterpret_cast<unsigned*>(smem + NS * SYS);  // shared scalars
  // sc[0..1] dmax per system, sc[2..3] ev_max per system, sc[4] tile counter
  int* counter = reinterpret_cast<int*>(sc + 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t s0 = p.sys_offset + NS * (int64_t)blockIdx.x;
  const int64_t slast = p.sys_offset + p.nsys - 1;
  int64_t sys[2] = {s0, s0 + 1 <= slast ? s0 + 1 : s0};
  const bool valid1 = NS == 2 && s0 + 1 <= slast;
  // pair / row of each system (hoisted: 64-bit division is a software routine)
  int64_t qq[2];
  int ii[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    qq[h] = sys[h] / k;
    ii[h] = (int)(sys[h] - qq[h] * k);
  }
  auto Ah = [&](int h) { return smem + h * SYS; };
  auto xvh = [&](int h) { return smem + h * SYS + Pn; };
  auto sinvh = [&](int h) { return smem + h * SYS + Pn + K4; };

  if (tid < 5) sc[tid] = 0u;
  // ---- staging (both systems) ----
  {
    const bool vec = (k & 3) == 0;
    for (int cc = warp; cc < NS * K4; cc += kNW2) {
      const int h = cc >= K4, c = cc - h * K4;
      const int64_t q = qq[h];
      const int i = ii[h];
      const int c4 = c & ~3;
      float* col = Ah(h) + colbase(c, Rp);
      if (c < k) {
        const float* g = p.gram + ((size_t)q * k + c) * k;
        if (vec) {
          for (int r = c4 + 4 * lane; r < k; r += 128) cp_async16(col + r, g + r);
        } else {
          for (int r = c4 + lane; r < k; r += 32) cp_async4(col + r, g + r);
        }
        const float* Rrow = p.rhs + ((size_t)q * k + i) * k;
        for (int r = k + lane; r < Rp; r += 32)
          col[r] = (r == K4) ? (p.rhs_unit < 0 ? Rrow[c] : (c == p.rhs_unit ? 1.f : 0.f)) : 0.f;
      } else {
        for (int r = c4 + lane; r < Rp; r += 32) col[r] = (r == c) ? 1.f : 0.f;
      }
    }
  }
  float evmax[2] = {0.f, 0.f};
  if constexpr (MASK_MODE == 1) {
    __syncthreads();  // sc[] initialised
    for (int h = 0; h < NS; ++h) {
      const int64_t q = qq[h];
      float m = 0.f;
      for (int c = tid; c < k; c += kNT2)
        m = fmaxf(m, fmaxf(p.ev1[(size_t)q * k + c], p.ev2[(size_t)q * k + c]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) atomicMax(&sc[2 + h], __float_as_uint(m));
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if constexpr (MASK_MODE == 1) {
    evmax[0] = __uint_as_float(sc[2]);
    evmax[1] = NS == 2 ? __uint_as_float(sc[3]) : evmax[0];
    if (!(evmax[0] > 0.f) || !(evmax[1] > 0.f)) {
      if (tid == 0) atomicOr(p.flags, 32u);
      return;
    }
  }
  {  // diagonal: + lambda * m_i(c) + ridge
    float dm[2] = {0.f, 0.f};
    for (int e = tid; e < NS * k; e += kNT2) {
      const int h = e >= k, c = e - h * k;
      const int64_t q = qq[h];
      const int i = ii[h];
      float* d = Ah(h) + colbase(c, Rp) + c;
      const float v = *d + (p.lambda * mask_entry<MASK_MODE>(p, q, i, c, evmax[h]) + p.ridge);
      *d = v;
      dm[h] = fmaxf(dm[h], fabsf(v));
    }
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      float m = dm[h];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) atomicMax(&sc[h], __float_as_uint(m));
    }
  }
  __syncthreads();
  FMAP_TRACE(0);

  const int hp = NS == 2 ? (lane >> 4) : 0;  // panel warp: system of this half-warp
  float* xb = reinterpret_cast<float*>(sc + 8) + 16 * hp;  // diag exchange buffer (per system)
  float pivmin = FLT_MAX;
  unsigned bad = 0u;
  if (warp == kPW2) {
    if (K4 >= kNB) diag16_x1<true>(Ah(hp), Rp, 0, kNB, sinvh(hp), xb, lane, pivmin, bad);
    else diag16_x1<false>(Ah(hp), Rp, 0, K4, sinvh(hp), xb, lane, pivmin, bad);
  }
  __syncthreads();
  FMAP_TRACE(1);

  // Schedule per panel p (diag(p) already done):
  //   A  bulk: TRSM(p) rows >= jn (both systems)
  //   B  bulk: SYRK(p) of the next panel's columns [jn, jn+nbn) (incl. its diag block)
  //   C  panel warp: diag(p+1) of both systems || bulk: SYRK(p) of columns >= jn+nbn
  for (int j = 0; j < K4; j += kNB) {
    const int ts = 8 + (j / kNB) * 8;
    const int nbe = min(kNB, K4 - j);
    const int jn = j + nbe;
    const int nbn = min(kNB, K4 - jn);
    const Panel Pj(j, Rp);
    const bool full = nbe == kNB;
    // A  (the panel warp, idle here, inverts the previous panel's diagonal block
    //     in place for the back substitution: L11(p-1) is final, TRSM(p-1) done)
    if (warp == kPW2 && j >= kNB)
      invert_diag16<true>(Ah(hp), Rp, j - kNB, kNB, sinvh(hp), lane & 15);
    if (pair_bulk<ISO>(warp)) {
      const int nr = Rp - jn;
      for (int e = pair_bt<ISO>(warp, lane); e < NS * nr; e += NB_T) {
        const int h = e >= nr, r = jn + e - h * nr;
        if (full) trsm_row<true>(Ah(h), Pj, sinvh(h), nbe, r);
        else trsm_row<false>(Ah(h), Pj, sinvh(h), nbe, r);
      }
    }
    if (tid == 0) *counter = 0;
    FMAP_TRACE(ts + 0);
    __syncthreads();
    if (nbn <= 0) break;
    // B
    if (pair_bulk<ISO>(warp)) {
      const int C0 = jn >> 2, nR = Rp >> 2, ncol = nbn >> 2;
      int ntile = 0;
      for (int cc = 0; cc < ncol; ++cc) ntile += nR - (C0 + cc);
      for (int L = pair_bt<ISO>(warp, lane); L < NS * ntile; L += NB_T) {
        const int h = L >= ntile;
        int l = L - h * ntile, cc = 0;
        while (l >= nR - (C0 + cc)) {
          l -= nR - (C0 + cc);
          ++cc;
        }
        const int Ct = C0 + cc;
        if (full) syrk_tile<true>(Ah(h), Rp, Pj, nbe, (Ct + l) << 2, Ct << 2);
        else syrk_tile<false>(Ah(h), Rp, Pj, nbe, (Ct + l) << 2, Ct << 2);
      }
    }
    FMAP_TRACE(ts + 1);
    __syncthreads();
    // C
    if (warp == kPW2) {
      if (nbn == kNB) diag16_x1<true>(Ah(hp), Rp, jn, nbn, sinvh(hp), xb, lane, pivmin, bad);
      else diag16_x1<false>(Ah(hp), Rp, jn, nbn, sinvh(hp), xb, lane, pivmin, bad);
      FMAP_TRACE(ts + 2);
    } else if (pair_bulk<ISO>(warp)) {
      const int cs = jn + nbn;
      if (cs < K4) {  // SYRK(p) is always a full 16-wide panel here
        const int ncb = (K4 - cs + 15) >> 4;
        int W = 0;
        for (int u = 0; u < ncb; ++u) W += (Rp - (cs + 16 * u) + 63) >> 6;
        while (true) {
          int w = 0;
          if (lane == 0) w = atomicAdd(counter, 1);
          w = __shfl_sync(0xffffffffu, w, 0);
          if (w >= NS * W) break;
          const int h = w >= W;
          w -= h * W;
          int cb = cs, nrb = (Rp - cb + 63) >> 6;
          while (w >= nrb) {
            w -= nrb;
            cb += 16;
            nrb = (Rp - cb + 63) >> 6;
          }
          syrk_warp_tile<true>(Ah(h), Rp, K4, Pj, nbe, cb, cb + (w << 6), 0, 0, lane);
        }
      }
    }
    FMAP_TRACE(ts + 4);
    __syncthreads();
  }
  FMAP_TRACE(1000);

  // ---- back substitution, both systems ----
  // 1. diagonal blocks 0 .. last-1 were inverted during the factorization (by
  //    the panel warp in phase A of the following panel); invert the last here.
  if (warp == 0) {
    const int jl = ((K4 - 1) / kNB) * kNB, nb = K4 - jl;
    if (nb == kNB) invert_diag16<true>(Ah(hp), Rp, jl, nb, sinvh(hp), lane & 15);
    else invert_diag16<false>(Ah(hp), Rp, jl, nb, sinvh(hp), lane & 15);
  }
  FMAP_TRACE(1002);
  for (int e = tid; e < NS * K4; e += kNT2) {
    const int h = e >= K4, c = e - h * K4;
    xvh(h)[c] = Ah(h)[colbase(c, Rp) + K4];
  }
  __syncthreads();
  // 2. blocks last to first: the panel warp forms x_B = L_BB^{-T} y_B (lane c:
  //    column c of L_BB^{-1} . y_B, no dependency chain) and applies x_B and the
  //    previous block's x to the next block; the bulk applies the previous
  //    block's x to all rows above the next block (one-block lag).
  int jprev = -1, nprev = 0, par = 0;
  for (int jb = ((K4 - 1) / kNB) * kNB; jb >= 0; jb -= kNB, par ^= 1) {
    const int nbe = min(kNB, K4 - jb);
    const int jnext = jb - kNB;
    if (warp == kPW2) {
      const int g = lane & 15;
      float* xv = xvh(hp);
      float* xcur = xv + 2 * K4 + 16 * par;        // x of this block
      const float* xprev = xv + 2 * K4 + 16 * (par ^ 1);  // x of the previous block
      if (nbe == kNB) {
        if (nprev == kNB || jprev < 0)
          backsub_block<true, true>(Ah(hp), Rp, xv, xcur, xprev, jb, nbe, jnext, jprev, nprev, g);
        else
          backsub_block<true, false>(Ah(hp), Rp, xv, xcur, xprev, jb, nbe, jnext, jprev, nprev, g);
      } else {
        backsub_block<false, false>(Ah(hp), Rp, xv, xcur, xprev, jb, nbe, jnext, jprev, nprev, g);
      }
    } else if (jprev >= 0 && jnext > 0 && pair_bulk<ISO>(warp)) {
      for (int e = pair_bt<ISO>(warp, lane); e < NS * jnext; e += NB_T) {
        const int h = e >= jnext, c = e - h * jnext;
        const float* col = Ah(h) + colbase(c, Rp) + jprev;
        const float* xprev = xvh(h) + 2 * K4 + 16 * (par ^ 1);
        float acc = 0.f;
#pragma unroll
        for (int r = 0; r < kNB; r += 4) {
          if (r < nprev) {
            const float4 l = ld4(col + r);
            const float4 xx = ld4(xprev + r);
            acc = fmaf(l.x, xx.x, acc);
            acc = fmaf(l.y, xx.y, acc);
            acc = fmaf(l.z, xx.z, acc);
            acc = fmaf(l.w, xx.w, acc);
          }
        }
        xvh(h)[c] -= acc;
      }
    }
    jprev = jb;
    nprev = nbe;
    FMAP_TRACE(1010 + jb / kNB);
    __syncthreads();
  }
  if (warp != kPW2) return;
  FMAP_TRACE(1001);
  {
    const int h = hp, g = lane & 15;
    const int64_t s = sys[h];
    const int64_t q = qq[h];
    const int i = ii[h];
    const bool write = h == 0 || valid1;
    bool nonfinite = false;
    float* Crow = p.C + ((size_t)q * k + i) * k;
    for (int c = g; c < k; c += 16) {
      const float x = xvh(h)[c];
      nonfinite |= !(fabsf(x) <= FLT_MAX);
      if (write) Crow[c] = x;
    }
    const unsigned nf = __ballot_sync(0xffffffffu, nonfinite);
    if (g == 0 && write) {
      const bool my_nf = (nf >> (16 * h)) & 0xffffu;
      const float dmax = __uint_as_float(sc[h]);
      float rc = dmax > 0.f ? pivmin / dmax : 0.f;
      if (!(rc >= 0.f)) rc = 0.f;
      if (bad || my_nf || !(rc >= p.rcond_thr)) atomicMin(p.fail_min, (unsigned long long)s);
      atomicMin(p.rcond_min_bits, __float_as_uint(rc));
    }
  }
}

size_t pair_smem_bytes(int k, int ns) {
  const int K4 = (k + 3) & ~3;
  return (size_t)(ns * pair_stride_floats(K4) + 8 + 32) * sizeof(float);
}

// Host-side launcher: two systems per CTA when both fit in one SM's shared
// memory (k <= ~228 on B200), else one system per CTA.
cudaError_t launch_chol_solve(const SolveParams& p, int mask_mode, cudaStream_t stream) {
  if (p.nsys <= 0) return cudaSuccess;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // tensor-core solver (tcgen05 + TMEM) unless FMAP_SOLVER=simt
  {
    const char* sel = std::getenv("FMAP_SOLVER");
    const bool simt = sel && sel[0] == 's';
    if (!simt && !p.force_single && p.tc_scratch && tc_supported(p.k, optin))
      return launch_chol_tc(p, mask_mode, stream);
  }
  const size_t smem2 = pair_smem_bytes(p.k, 2), smem1 = pair_smem_bytes(p.k, 1);
  const bool pair = smem2 <= (size_t)optin && !p.force_single;
  const bool wide = !pair && smem1 <= (size_t)optin && !p.force_single;  // one system, 16 warps
  void (*fn)(SolveParams) = nullptr;
  size_t smem;
  unsigned grid, block;
  const bool iso = !p.pair_shared_smsp;
  if (pair || wide) {
#define FMAP_PICK(NSV)                                                                       \
  switch (mask_mode) {                                                                       \
    case 0: fn = iso ? chol_pair_kernel<0, true, NSV> : chol_pair_kernel<0, false, NSV>; break; \
    case 1: fn = iso ? chol_pair_kernel<1, true, NSV> : chol_pair_kernel<1, false, NSV>; break; \
    default: fn = iso ? chol_pair_kernel<2, true, NSV> : chol_pair_kernel<2, false, NSV>; break; \
  }
    if (pair) {
      FMAP_PICK(2)
      smem = smem2;
      grid = (unsigned)((p.nsys + 1) / 2);
    } else {
      FMAP_PICK(1)
      smem = smem1;
      grid = (unsigned)p.nsys;
    }
#undef FMAP_PICK
    block = kNT2;
  } else {
    switch (mask_mode) {
      case 0: fn = chol_solve_kernel<0>; break;
      case 1: fn = chol_solve_kernel<1>; break;
      default: fn = chol_solve_kernel<2>; break;
    }
    smem = solver_smem_bytes(p.k);
    grid = (unsigned)p.nsys;
    block = kNT;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  fn<<<grid, block, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace fmap
