// Batched Cholesky solver with the trailing update on the 5th-generation tensor
// cores (tcgen05, kind::tf32, 3xTF32 split) and the trailing matrix resident in
// tensor memory (TMEM) — sm_100a.
//
// One CTA owns one row system at a time (persistent over systems, 2 CTAs per SM
// for k <= 256):
//     (G_q + lambda*diag(M_q[i,:]) + ridge*I) x = R_q[i,:]^T,   C_q[i,:] = x^T
// replacing the reference's per-system PartialPivLU
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170) driven by
// solve_batched_many (:220-322).  The system is SPD by construction.
//
// Storage (K16 = k rounded up to 16; rows/cols k..K16-1 are identity padding):
//   * tile A (TMEM): the LAST min(128, K16) rows, r = s + lane (s = K16 - 128 or
//     0), all K16 columns (lane = row, TMEM column = matrix column).  The tensor
//     core updates it in place: D[r][c] -= sum_t L[r][j+t] L[c][j+t].  Factored
//     L values are written back into their own columns (never touched again).
//   * top-left rows 0..s-1 (shared memory, packed lower triangle, fp32): these
//     rows only have columns < s; their trailing update is SIMT.
//   * operand buffers (shared memory): the current panel's L21 split into TF32
//     hi/lo parts, K-major core-matrix layout (8 rows x 16 B per core matrix),
//     used as BOTH the A operand (rows s..s+127) and the B operand (rows j+16..).
//
// Per 16-column panel p (j = 16 p), one CTA-wide pass:
//   a  rows >= j load their 16 panel entries (TMEM ld / smem) after the
//      lookahead MMA of panel p-1 has landed; lagged right-hand-side update.
//   b  the warp holding rows j..j+15 factors the 16x16 diagonal block (lane per
//      row, one shuffle per pivot on the critical chain).            | barrier
//   c  every row >= j+16 solves its L21 row (TRSM against L11); the augmented
//      right-hand-side "row" gives y = L^{-1} r for the panel.
//   d  L rows -> TMEM (kept for the back substitution), hi/lo -> operand
//      buffers; fence.proxy.async.                                  | barrier
//   e  one thread issues the lookahead MMA (next panel's 16 columns) and the
//      rest of the trailing update, each committed to its own mbarrier; the
//      top-left rows run their SIMT trailing update meanwhile.
// Back substitution L^T x = y in 16-row blocks from the bottom (diagonal blocks
// inverted up front; per block one TMEM load, a warp reduction and a 16x16
// mat-vec), then a coalesced write of the row of C.
//
// Singular = non-positive / non-finite pivot, rcond estimate min(pivot)/max|diag|
// below the threshold, or a non-finite solution (lowest failing index wins).
#include "fmap_solver.cuh"

#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

namespace fmap {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTL = 128;  // TMEM lanes / tile-A rows

struct TcLayout {
  int K16, s, P, tl_warps, threads;
  int tmem_cols;
  int Rop;  // operand buffer rows
  // offsets in floats from the dynamic smem base
  int off_hi, off_lo, off_tri, off_lp, off_l11, off_inv, off_yv, off_xv, off_zb, off_red;
  int off_misc;  // 64 floats: mbarriers + scalars
  int floats;
};

__host__ __device__ inline int tri_size(int s) { return ((s * (s + 1) / 2) + 3) & ~3; }

__host__ inline TcLayout make_layout(int k) {
  TcLayout L{};
  L.K16 = (k + 15) & ~15;
  L.s = L.K16 > kTL ? L.K16 - kTL : 0;
  L.P = L.K16 / 16;
  L.tl_warps = (L.s + 1 + 31) / 32;  // top-left rows + the augmented rhs "row"
  L.threads = 128 + 32 * L.tl_warps;
  int c = 32;
  while (c < L.K16) c <<= 1;
  L.tmem_cols = c;
  L.Rop = L.K16 > kTL ? L.K16 : kTL;
  int o = 0;
  L.off_hi = o;  o += L.Rop * 16;
  L.off_lo = o;  o += L.Rop * 16;
  L.off_tri = o; o += tri_size(L.s);
  L.off_lp = o;  o += (L.s > 0 ? L.s : 1) * 16;
  L.off_l11 = o; o += L.P * 256;
  L.off_inv = o; o += L.P * 16;
  L.off_yv = o;  o += L.K16;
  L.off_xv = o;  o += L.K16;
  L.off_zb = o;  o += 32;
  L.off_red = o; o += (L.threads / 32) * 16;
  L.off_misc = o; o += 64;
  L.floats = o;
  return L;
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = su32(b);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns (lane = this warp's TMEM lane quarter).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]),
                 "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8 rows x
// 16 B; LBO = distance between the two K-adjacent core matrices (128 B),
// SBO = distance between 8-row groups (512 B).  Version field = 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) |
         ((uint64_t)(512u >> 4) << 32) | (1ull << 46);
}

// Instruction descriptor: D f32, A/B tf32, K-major, A negated (D += -A*B), M=128.
__device__ __forceinline__ uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 13) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t idesc) {
  const uint32_t acc = 1u;
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

__device__ __forceinline__ float rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  const float rem = x - __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(rem));
  hi = __uint_as_float(h);
  lo = __uint_as_float(l);
}

// float index of element (r, t) (t < 16) in an operand buffer
__device__ __forceinline__ int opnd_idx(int r, int t) {
  return (r >> 3) * 128 + (t >> 2) * 32 + (r & 7) * 4 + (t & 3);
}

// Diagonal mask entry m_i(c) (masks.hpp:13-89, same operation order in fp32).
template <int MASK_MODE>
__device__ __forceinline__ float mask_entry(const SolveParams& p, int64_t q, int i, int c, float ev_max) {
  const int k = p.k;
  if constexpr (MASK_MODE == 0) {
    return p.mask[((size_t)q * k + i) * k + c];
  } else if constexpr (MASK_MODE == 1) {
    const float s = p.sigma, s2 = s * s;
    const float mu1 = p.ev1[(size_t)q * k + c] / ev_max;
    const float mu2 = p.ev2[(size_t)q * k + i] / ev_max;
    const float re1 = mu1 / (mu1 * mu1 + s2), im1 = s / (mu1 * mu1 + s2);
    const float re2 = mu2 / (mu2 * mu2 + s2), im2 = s / (mu2 * mu2 + s2);
    const float re = re2 - re1, im = im2 - im1;
    return re * re + im * im;
  } else {
    const float d = p.ev2[(size_t)q * k + i] - p.ev1[(size_t)q * k + c];
    return d * d;
  }
}

// Cholesky of the 16x16 diagonal block, lane per row (g = lane & 15) inside each
// 16-lane half of the warp (the other half computes garbage that is discarded).
// On return a[t] (t <= g) = L[g][t]; inv = 1/L[g][g].  Critical chain per pivot:
// SHFL -> RSQ -> FMUL -> FFMA (the next pivot is formed from the lane's own l).
__device__ __forceinline__ void diag_factor(float (&a)[16], float& inv, int g, bool real,
                                            float& pivmin, unsigned& bad) {
  float dnext = __shfl_sync(kFull, a[0], 0, 16);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const float d = dnext;
    if (real && g == t) {
      pivmin = fminf(pivmin, d);
      bad |= (unsigned)(!(d > 0.f)) | (unsigned)(!(d <= FLT_MAX));
    }
    const float sc = rsqrt_fast(d);
    const float l = a[t] * sc;
    if (g == t) inv = sc;
    a[t] = l;
    if (t < 15) {
      const float crit = fmaf(-l, l, a[t + 1]);  // meaningful in lane t+1
      dnext = __shfl_sync(kFull, crit, t + 1, 16);
    }
#pragma unroll
    for (int c = t + 1; c < 16; ++c) {
      const float lc = __shfl_sync(kFull, l, c, 16);
      a[c] = fmaf(-l, lc, a[c]);
    }
  }
}

// l = L11^{-1}-solve of one row:  l[t] = (a[t] - sum_{u<t} l[u] L11[t][u]) * inv[t]
__device__ __forceinline__ void trsm_row(const float* __restrict__ L11, const float* __restrict__ inv,
                                         const float (&a)[16], float (&l)[16]) {
  float v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = a[t];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    l[t] = v[t] * inv[t];
    // right-looking: v[c] -= l[t] * L11[c][t] for c > t
#pragma unroll
    for (int c = t + 1; c < 16; ++c) v[c] = fmaf(-l[t], L11[c * 16 + t], v[c]);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
template <int MASK_MODE, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) chol_tc_kernel(SolveParams p, TcLayout Ly) {
  extern __shared__ __align__(1024) float smem[];
  const int k = p.k, K16 = Ly.K16, s = Ly.s, P = Ly.P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthreads = Ly.threads;
  float* opnd_hi = smem + Ly.off_hi;
  float* opnd_lo = smem + Ly.off_lo;
  float* tri = smem + Ly.off_tri;
  float* Lp = smem + Ly.off_lp;
  float* L11all = smem + Ly.off_l11;
  float* invall = smem + Ly.off_inv;
  float* yv = smem + Ly.off_yv;
  float* xv = smem + Ly.off_xv;
  float* zb = smem + Ly.off_zb;
  float* red = smem + Ly.off_red;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + Ly.off_misc);  // [0] LA, [1] REST
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Ly.off_misc + 4);
  unsigned* sc = reinterpret_cast<unsigned*>(smem + Ly.off_misc + 8);
  // sc[0] dmax bits, sc[1] pivmin bits, sc[2] bad, sc[3] ev_max bits, sc[4] nonfinite

  // ---- one-time setup ----
  for (int e = tid; e < 2 * Ly.Rop * 16; e += nthreads) smem[Ly.off_hi + e] = 0.f;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, (uint32_t)Ly.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  // row ownership
  const bool tileA = warp < 4;
  const int row = tileA ? s + 32 * warp + lane : 32 * (warp - 4) + lane;
  const bool row_valid = tileA ? row < K16 : row < s;
  const bool is_aug = !tileA && row == s;  // augmented right-hand-side "row"
  const uint32_t trow = tbase + ((uint32_t)(32 * (warp & 3)) << 16);  // this warp's lane quarter
  const int tri_row = row * (row + 1) / 2;

  uint32_t g = 0;  // global panel counter (mbarrier phases)
  bool any_mma = false;

  for (int64_t sl = blockIdx.x; sl < p.nsys; sl += gridDim.x) {
    const int64_t sys = p.sys_offset + sl;
    const int64_t q = sys / k;
    const int i = (int)(sys - q * k);

    // previous system's MMAs must be complete before TMEM / operands are reused
    if (any_mma) {
      mbar_wait(&mbar[1], (g - 1) & 1);
      tc_fence_after();
    }
    if (tid == 0) {  // tid 0 is also the last reader of the previous system's scalars
#pragma unroll
      for (int e = 0; e < 8; ++e) sc[e] = 0u;
      sc[1] = __float_as_uint(FLT_MAX);
    }
    __syncthreads();

    float ev_max = 0.f;
    if constexpr (MASK_MODE == 1) {
      float m = 0.f;
      for (int c = tid; c < k; c += nthreads)
        m = fmaxf(m, fmaxf(p.ev1[(size_t)q * k + c], p.ev2[(size_t)q * k + c]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
      if (lane == 0) atomicMax(&sc[3], __float_as_uint(m));
      __syncthreads();
      ev_max = __uint_as_float(sc[3]);
      if (!(ev_max > 0.f)) {
        if (tid == 0) atomicOr(p.flags, 32u);
        continue;  // uniform across the CTA
      }
    }

    // ---- staging: row r of (G + lambda*diag(m_i) + ridge*I), identity padding ----
    // G is read as columns (G[c][r], coalesced across the warp's rows); the lower
    // triangle used here is G's upper triangle, as the packed-column solver does.
    const float* Gq = p.gram + (size_t)q * k * k;
    float rhs = 0.f;
    float dmax = 0.f;
    if (row_valid) {
      if (row < k) {
        rhs = p.rhs_unit < 0 ? p.rhs[((size_t)q * k + i) * k + row] : (row == p.rhs_unit ? 1.f : 0.f);
      }
    }
    float dval = 1.f;
    if (row_valid && row < k) {
      dval = Gq[(size_t)row * k + row] + (p.lambda * mask_entry<MASK_MODE>(p, q, i, row, ev_max) + p.ridge);
      dmax = fabsf(dval);
    }
    if (tileA) {
      for (int cb = 0; cb < K16; cb += 16) {
        float v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int c = cb + t;
          float x = 0.f;
          if (row_valid) {
            if (c == row) x = dval;
            else if (row < k && c < k) x = __ldg(Gq + (size_t)c * k + row);
          }
          v[t] = x;
        }
        tmem_st16(trow + (uint32_t)cb, v);
      }
      tmem_st_wait();
    } else if (row_valid) {
      for (int c = 0; c <= row; ++c) {
        float x = 0.f;
        if (c == row) x = dval;
        else if (row < k && c < k) x = __ldg(Gq + (size_t)c * k + row);
        tri[tri_row + c] = x;
      }
    }
    {
      float m = dmax;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
      if (lane == 0) atomicMax(&sc[0], __float_as_uint(m));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    float pivmin = FLT_MAX;
    unsigned bad = 0u;
    float lprev[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) lprev[t] = 0.f;

    // ---- panels ----
    for (int pp = 0; pp < P; ++pp, ++g) {
      const int j = 16 * pp;
      const bool active = row_valid && row >= j;
      // a. lagged rhs update, panel entries
      if (pp > 0 && active) {
#pragma unroll
        for (int t = 0; t < 16; ++t) rhs = fmaf(-lprev[t], yv[j - 16 + t], rhs);
      }
      float a[16];
      if (tileA) {
        if (pp > 0) {  // panel columns updated by the previous lookahead MMA
          mbar_wait(&mbar[0], (g - 1) & 1);
          tc_fence_after();
        }
        tmem_ld16(trow + (uint32_t)j, a);
      } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) a[t] = (active && j + t <= row) ? tri[tri_row + j + t] : 0.f;
      }
      // b. diagonal block
      const bool in_diag = active && row < j + 16;
      const int dwarp = j >= s ? (j - s) >> 5 : 4 + (j >> 5);
      float* L11 = L11all + pp * 256;
      float* inv = invall + pp * 16;
      if (warp == dwarp) {
        float d[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) d[t] = a[t];
        float iv = 0.f;
        diag_factor(d, iv, lane & 15, in_diag && row < k, pivmin, bad);
        if (in_diag) {
          const int gr = row - j;
#pragma unroll
          for (int t = 0; t < 16; ++t) L11[gr * 16 + t] = (t <= gr) ? d[t] : 0.f;
          inv[gr] = iv;
          zb[gr] = rhs;
#pragma unroll
          for (int t = 0; t < 16; ++t) a[t] = d[t];
        }
      }
      __syncthreads();
      // c. TRSM rows >= j+16 ; augmented row -> y for this panel
      float l[16];
      const bool trsm = active && row >= j + 16;
      if (trsm) {
        trsm_row(L11, inv, a, l);
      } else if (is_aug) {
        float z[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) z[t] = zb[t];
        trsm_row(L11, inv, z, l);
#pragma unroll
        for (int t = 0; t < 16; ++t) yv[j + t] = l[t];
      } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) l[t] = in_diag ? a[t] : 0.f;
      }
      // d. store L: TMEM (tile A, kept for back substitution), smem tri (top-left),
      //    operand hi/lo (rows >= j+16)
      if (tileA) {
        tmem_st16(trow + (uint32_t)j, l);
      } else if (active && !is_aug) {
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (j + t <= row) tri[tri_row + j + t] = l[t];
      }
      if (trsm) {
        if (pp > 0) mbar_wait(&mbar[1], (g - 1) & 1);  // previous REST MMA done reading
        float* h = opnd_hi + opnd_idx(row, 0);
        float* lo = opnd_lo + opnd_idx(row, 0);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          float hv[4], lv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) split_tf32(l[4 * c4 + u], hv[u], lv[u]);
          *reinterpret_cast<float4*>(h + c4 * 32) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<float4*>(lo + c4 * 32) = make_float4(lv[0], lv[1], lv[2], lv[3]);
        }
        if (!tileA) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4)
            *reinterpret_cast<float4*>(Lp + row * 16 + 4 * c4) =
                make_float4(l[4 * c4], l[4 * c4 + 1], l[4 * c4 + 2], l[4 * c4 + 3]);
        }
      }
      if (tileA) tmem_st_wait();
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      tc_fence_after();
      // e. tensor-core trailing update: lookahead (next panel) then the rest
      if (tid == 0) {
        const int r0 = j + 16;
        const uint32_t hib = su32(opnd_hi), lob = su32(opnd_lo);
        const uint32_t arow = (uint32_t)(s >> 3) * 512u;
        if (r0 < K16) {
          int c0 = r0;
          // lookahead: 16 columns
          {
            const uint32_t id = idesc_tf32(16);
            const uint32_t brow = (uint32_t)(c0 >> 3) * 512u;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t ko = (uint32_t)ks * 256u;
              const uint64_t ah = sdesc(hib + arow + ko), al = sdesc(lob + arow + ko);
              const uint64_t bh = sdesc(hib + brow + ko), bl = sdesc(lob + brow + ko);
              mma_tf32(tbase + (uint32_t)c0, ah, bh, id);
              mma_tf32(tbase + (uint32_t)c0, ah, bl, id);
              mma_tf32(tbase + (uint32_t)c0, al, bh, id);
            }
          }
          mma_commit(&mbar[0]);
          c0 += 16;
          while (c0 < K16) {
            const int N = min(256, K16 - c0);
            const uint32_t id = idesc_tf32(N);
            const uint32_t brow = (uint32_t)(c0 >> 3) * 512u;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t ko = (uint32_t)ks * 256u;
              const uint64_t ah = sdesc(hib + arow + ko), al = sdesc(lob + arow + ko);
              const uint64_t bh = sdesc(hib + brow + ko), bl = sdesc(lob + brow + ko);
              mma_tf32(tbase + (uint32_t)c0, ah, bh, id);
              mma_tf32(tbase + (uint32_t)c0, ah, bl, id);
              mma_tf32(tbase + (uint32_t)c0, al, bh, id);
            }
            c0 += N;
          }
          mma_commit(&mbar[1]);
        } else {
          mma_commit(&mbar[0]);
          mma_commit(&mbar[1]);
        }
      }
      any_mma = true;
      // top-left SIMT trailing update (rows j+16..s-1, columns j+16..row)
      if (!tileA && trsm) {
        for (int c = j + 16; c <= row; ++c) {
          const float* lc = Lp + c * 16;
          float acc = 0.f;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 v = *reinterpret_cast<const float4*>(lc + 4 * c4);
            acc = fmaf(l[4 * c4], v.x, acc);
            acc = fmaf(l[4 * c4 + 1], v.y, acc);
            acc = fmaf(l[4 * c4 + 2], v.z, acc);
            acc = fmaf(l[4 * c4 + 3], v.w, acc);
          }
          tri[tri_row + c] -= acc;
        }
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) lprev[t] = trsm ? l[t] : 0.f;
    }

    // ---- singularity bookkeeping ----
    {
      unsigned b = bad;
      float pm = pivmin;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        b |= __shfl_xor_sync(kFull, b, o);
        pm = fminf(pm, __shfl_xor_sync(kFull, pm, o));
      }
      if (lane == 0) {
        if (b) atomicOr(&sc[2], 1u);
        atomicMin(&sc[1], __float_as_uint(fmaxf(pm, 0.f)));
      }
    }

    // ---- back substitution  L^T x = y ----
    // B0: invert the diagonal blocks, W_b = L_bb^{-1} (column u of block b per
    //     thread) into the operand buffer, idle once the last MMA has landed
    mbar_wait(&mbar[1], (g - 1) & 1);
    float* Wall = opnd_hi;
    for (int e = tid; e < P * 16; e += nthreads) {
      const int b = e >> 4, u = e & 15;
      const float* Lb = L11all + b * 256;
      const float* ib = invall + b * 16;
      float w[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        float acc = (t == u) ? 1.f : 0.f;
#pragma unroll
        for (int v = 0; v < t; ++v) acc = fmaf(-Lb[t * 16 + v], w[v], acc);
        w[t] = (t >= u) ? acc * ib[t] : 0.f;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) Wall[b * 256 + t * 16 + u] = w[t];
    }
    __syncthreads();
    // B1: blocks from the bottom
    float xr = 0.f;  // x of this thread's row (once known)
    for (int b = P - 1; b >= 0; --b) {
      const int c0 = 16 * b;
      float v[16];
      if (tileA) {
        float lv[16];
        tmem_ld16(trow + (uint32_t)c0, lv);
        const bool use = row_valid && row >= c0 + 16;
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = use ? lv[t] * xr : 0.f;
      } else {
        const bool use = row_valid && row >= c0 + 16;
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = use ? tri[tri_row + c0 + t] * xr : 0.f;
      }
      // warp reduction of the 16-vector: lane (2t, 2t+1) ends with component t
      {
        const bool h16 = lane & 16;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float send = h16 ? v[e] : v[e + 8];
          const float keep = h16 ? v[e + 8] : v[e];
          v[e] = keep + __shfl_xor_sync(kFull, send, 16);
        }
        const bool h8 = lane & 8;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float send = h8 ? v[e] : v[e + 4];
          const float keep = h8 ? v[e + 4] : v[e];
          v[e] = keep + __shfl_xor_sync(kFull, send, 8);
        }
        const bool h4 = lane & 4;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float send = h4 ? v[e] : v[e + 2];
          const float keep = h4 ? v[e + 2] : v[e];
          v[e] = keep + __shfl_xor_sync(kFull, send, 4);
        }
        const bool h2 = lane & 2;
        {
          const float send = h2 ? v[0] : v[1];
          const float keep = h2 ? v[1] : v[0];
          v[0] = keep + __shfl_xor_sync(kFull, send, 2);
        }
        v[0] += __shfl_xor_sync(kFull, v[0], 1);
        if ((lane & 1) == 0) red[warp * 16 + ((lane >> 1) & 15)] = v[0];
      }
      __syncthreads();
      if (warp == 0 && lane < 16) {
        float z = yv[c0 + lane];
        for (int w = 0; w < nthreads / 32; ++w) z -= red[w * 16 + lane];
        zb[lane] = z;
        __syncwarp(0xffffu);
        const float* W = Wall + b * 256;
        float x = 0.f;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (u >= lane) x = fmaf(W[u * 16 + lane], zb[u], x);  // x_t = sum_{u>=t} W[u][t] z_u
        xv[c0 + lane] = x;
      }
      __syncthreads();
      if (row_valid && row >= c0 && row < c0 + 16) xr = xv[row];
    }
    // ---- output row of C ----
    {
      float* Crow = p.C + ((size_t)q * k + i) * k;
      bool nf = false;
      for (int c = tid; c < k; c += nthreads) {
        const float x = xv[c];
        nf |= !(fabsf(x) <= FLT_MAX);
        Crow[c] = x;
      }
      if (__any_sync(kFull, nf) && lane == 0) atomicOr(&sc[4], 1u);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      const float dm = __uint_as_float(sc[0]);
      const float pm = __uint_as_float(sc[1]);
      float rc = dm > 0.f ? pm / dm : 0.f;
      if (!(rc >= 0.f)) rc = 0.f;
      if (sc[2] || sc[4] || !(rc >= p.rcond_thr)) atomicMin(p.fail_min, (unsigned long long)sys);
      atomicMin(p.rcond_min_bits, __float_as_uint(rc));
    }
  }
  // ---- teardown ----
  if (any_mma) {
    mbar_wait(&mbar[1], (g - 1) & 1);
    tc_fence_after();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, (uint32_t)Ly.tmem_cols);
}

// Host-side launcher for the tensor-core solver.  Returns cudaErrorNotSupported
// when k is outside its range (the caller then uses the SIMT solver).
bool tc_supported(int k, int optin_smem) {
  if (k < 1) return false;
  const TcLayout L = make_layout(k);
  if (L.tmem_cols > 512 || L.threads > 320) return false;
  return (size_t)L.floats * 4 <= (size_t)optin_smem;
}

cudaError_t launch_chol_tc(const SolveParams& p, int mask_mode, cudaStream_t stream) {
  if (p.nsys <= 0) return cudaSuccess;
  int dev = 0, optin = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const TcLayout L = make_layout(p.k);
  if (L.tmem_cols > 512 || L.threads > 320) return cudaErrorNotSupported;
  const int cps = 512 / L.tmem_cols;  // CTAs per SM the TMEM allows
  // cap residency at `cps` CTAs per SM through the shared-memory request, so no
  // CTA ever waits on a TMEM allocation
  const size_t sm_total = 233472;
  size_t smem = (size_t)L.floats * 4;
  const size_t floor_req = sm_total / (size_t)(cps + 1) + 1;
  if (smem < floor_req) smem = floor_req;
  if (smem > (size_t)optin) {
    if ((size_t)L.floats * 4 > (size_t)optin) return cudaErrorNotSupported;
    smem = (size_t)optin;
  }
  void (*fn)(SolveParams, TcLayout) = nullptr;
  if (cps >= 2) {  // <= 288 threads, two CTAs per SM
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 288, 2>; break;
      case 1: fn = chol_tc_kernel<1, 288, 2>; break;
      default: fn = chol_tc_kernel<2, 288, 2>; break;
    }
  } else {
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 320, 1>; break;
      case 1: fn = chol_tc_kernel<1, 320, 1>; break;
      default: fn = chol_tc_kernel<2, 320, 1>; break;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t maxgrid = (int64_t)sms * cps;
  const unsigned grid = (unsigned)(p.nsys < maxgrid ? p.nsys : maxgrid);
  fn<<<grid, L.threads, smem, stream>>>(p, L);
  return cudaGetLastError();
}

}  // namespace fmap
