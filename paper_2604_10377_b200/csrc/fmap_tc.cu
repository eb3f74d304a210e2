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
#include <cstdlib>
#include <algorithm>

namespace fmap {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kTL = 128;  // TMEM lanes / tile-A rows

// Rows are split into groups of <= 128 from the bottom: group g holds rows
// [lo[g], hi[g]) on TMEM lanes row - lo[g], and its own TMEM column region for the
// matrix columns [16, hi[g]) (the panel-0 columns stay in registers):
//   TMEM column of (group g, matrix column c) = base[g] + c - 16.
// k = 200 (K16 = 208): rows 80..207 -> 192 columns, rows 0..79 -> 64 columns, 256
// in total, so two CTAs (two systems) share one SM.
constexpr int kMaxGroups = 3;
struct TcLayout {
  int K16, P, G;
  int lo[kMaxGroups], hi[kMaxGroups], base[kMaxGroups];
  int nmain, bwarp, mwarp, threads, aug_tid;
  int tmem_cols;
  int Rop;  // operand buffer rows
  int cps;  // CTAs per SM
  // offsets in floats from the dynamic smem base
  int off_hi, off_lo, off_lt, off_l11, off_yv, off_xv, off_lb, off_zb, off_misc;
  int floats;
  long long lb;  // floats of one L scratch slot (global memory)
};

// First float of block p's L21 rows in an L scratch slot: block p holds rows
// 16p+16 .. K16-1, 16 floats each.
__host__ __device__ inline long long lb_off(int p, int K16) {
  return 16ll * p * (K16 - 16) - 128ll * p * (p - 1);
}

__host__ inline TcLayout make_layout(int k) {
  TcLayout L{};
  L.K16 = (k + 15) & ~15;
  L.P = L.K16 / 16;
  int hi = L.K16, base = 0;
  L.G = 0;
  while (hi > 0 && L.G < kMaxGroups) {
    const int lo = hi > kTL ? hi - kTL : 0;
    L.lo[L.G] = lo;
    L.hi[L.G] = hi;
    L.base[L.G] = base;
    base += hi - 16;
    hi = lo;
    L.G++;
  }
  const int total = hi > 0 ? 1 << 30 : base;  // rows left over: unsupported
  const int ntop = L.hi[L.G - 1] - L.lo[L.G - 1];
  L.aug_tid = kTL * (L.G - 1) + ntop;
  L.nmain = 32 * (4 * (L.G - 1) + (ntop + 1 + 31) / 32);
  L.bwarp = L.nmain / 32;      // back-substitution warp
  L.mwarp = L.bwarp + 1;       // MMA-issue warp
  L.threads = L.nmain + 64;
  int c = 32;
  while (c < total && c < 1024) c <<= 1;
  L.tmem_cols = c;
  L.Rop = L.K16 > kTL ? L.K16 : kTL;
  int o = 0;
  L.off_hi = o;  o += L.Rop * 16;
  L.off_lo = o;  o += L.Rop * 16;
  L.off_lt = o;  o += 256 + 16;               // current diagonal block (transposed) + 1/L_tt
  L.off_l11 = o; o += 2 * L.P * 152;          // per slot: packed lower L_bb (+ 1/L_tt) of every block
  L.off_yv = o;  o += 2 * L.K16;              // per slot: y = L^{-1} r
  L.off_xv = o;  o += L.K16;                  // back substitution: x
  L.off_lb = o;  o += 2 * (L.K16 - 16 > 0 ? L.K16 - 16 : 1) * 16;  // back substitution: L blocks
  L.off_zb = o;  o += 32;
  L.off_misc = o; o += 64;
  L.floats = o;
  L.lb = (lb_off(L.P, L.K16) + 31) & ~31ll;
  const int cps_tmem = L.tmem_cols <= 512 ? 512 / L.tmem_cols : 0;
  const size_t bytes = (size_t)L.floats * 4 + 1024;
  const int cps_smem = (int)(233472 / bytes);
  L.cps = cps_tmem < cps_smem ? cps_tmem : cps_smem;
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

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc = 1u) {
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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
// Named barrier over the main (factorization) warps only.
__device__ __forceinline__ void main_sync(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

__device__ __forceinline__ float rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// x = hi + lo with hi = round-to-nearest TF32; lo is exact in fp32 and the tensor
// core reads it as TF32 (truncated): |x - hi - tf32(lo)| <= 2^-21 |x|.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
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

// l = L11^{-1}-solve of one row:  l[t] = (a[t] - sum_{u<t} l[u] L11[t][u]) * inv[t],
// right-looking over the TRANSPOSED block LT[t][c] = L11[c][t] (column t is one
// broadcast LDS.128 run); chain 16 x (FMUL + FFMA).  `a` is consumed.
__device__ __forceinline__ void trsm_row(const float* __restrict__ LT, const float* __restrict__ inv,
                                         float (&a)[16], float (&l)[16]) {
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    l[t] = a[t] * inv[t];
#pragma unroll
    for (int c4 = (t + 1) >> 2; c4 < 4; ++c4) {
      const float4 col = *reinterpret_cast<const float4*>(LT + t * 16 + 4 * c4);
      if (4 * c4 > t) a[4 * c4] = fmaf(-l[t], col.x, a[4 * c4]);
      if (4 * c4 + 1 > t) a[4 * c4 + 1] = fmaf(-l[t], col.y, a[4 * c4 + 1]);
      if (4 * c4 + 2 > t) a[4 * c4 + 2] = fmaf(-l[t], col.z, a[4 * c4 + 2]);
      if (4 * c4 + 3 > t) a[4 * c4 + 3] = fmaf(-l[t], col.w, a[4 * c4 + 3]);
    }
  }
}

// Debug phase trace (FMAP_TRACE_FILE): clock64 stamps of one CTA's second system.
#define TC_TRACE(cond, slot)                                                              \
  do {                                                                                    \
    if (p.trace && tr_on && (cond)) p.trace[(slot)] = clock64();                          \
  } while (0)

// Launch-local system number sl -> (pair q, row i).  A full batch is walked pair-
// interleaved (consecutive sl hit different pairs), so the CTAs running at the
// same time read different Gram matrices instead of all hammering one.
__device__ __forceinline__ void sys_of(const SolveParams& p, int64_t sl, int64_t& q, int& i) {
  const int k = p.k;
  if (p.sys_offset % k == 0 && p.nsys % k == 0) {  // whole pairs (a batch or a chunk of one)
    const int64_t b = p.nsys / k;
    q = p.sys_offset / k + sl % b;
    i = (int)(sl / b);
  } else {
    const int64_t sys = p.sys_offset + sl;
    q = sys / k;
    i = (int)(sys - q * k);
  }
}

// Load the 16 entries of row `row` in columns 16cb..16cb+15 as G[c][row] (G is
// symmetric; coalesced across the warp's consecutive rows: one 128-byte line per
// load instruction).  Lower part c <= row only.
__device__ __forceinline__ void load_cols(const float* __restrict__ Gq, int k, int row, bool ok, int cb,
                                          float (&v)[16]) {
  const int c0 = 16 * cb;
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const int c = c0 + t;
    v[t] = (ok && c <= row && c < k) ? __ldg(Gq + (size_t)c * k + row) : 0.f;
  }
}

// ---------------------------------------------------------------------------
// Main warps (0..nmain/32-1): staging + blocked factorization of system n of this
// CTA into slot n&1; the back-substitution warp solves L^T x = y for system n-1
// meanwhile and writes the row of C.
// ---------------------------------------------------------------------------
template <int MASK_MODE, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) chol_tc_kernel(SolveParams p, TcLayout Ly) {
  extern __shared__ __align__(1024) float smem[];
  const int k = p.k, K16 = Ly.K16, P = Ly.P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NM = Ly.nmain;
  float* opnd_hi = smem + Ly.off_hi;
  float* opnd_lo = smem + Ly.off_lo;
  float* LT = smem + Ly.off_lt;  // current diagonal block, transposed: LT[t][c] = L[c][t]
  float* inv = LT + 256;         // 1/L_tt of the current block
  float* zb = smem + Ly.off_zb;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + Ly.off_misc);
  // mbar[0] LA, [1] REST, [2..3] lfull (back-sub L blocks), [4..5] fact (slot), [6..7] bsub (slot),
  // [8] opsready (operands of the panel stored, one arrival per main warp), [9] ysync
  uint64_t* lfull = mbar + 2;
  uint64_t* fact = mbar + 4;
  uint64_t* bsub = mbar + 6;
  uint64_t* opsready = mbar + 8;
  uint64_t* ysync = mbar + 9;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Ly.off_misc + 20);
  unsigned* sc = reinterpret_cast<unsigned*>(smem + Ly.off_misc + 24);
  // sc[0] dmax bits, sc[1] pivmin bits, sc[2] bad, sc[3] ev_max bits (current system)
  unsigned* slotsc = reinterpret_cast<unsigned*>(smem + Ly.off_misc + 40);  // [slot][4]
  float* Lscr = p.tc_scratch + (size_t)blockIdx.x * 2 * Ly.lb;

  // ---- one-time setup ----
  for (int e = tid; e < 2 * Ly.Rop * 16; e += Ly.threads) smem[Ly.off_hi + e] = 0.f;
  if (tid == 0) {
#pragma unroll
    for (int e = 0; e < 10; ++e) mbar_init(&mbar[e], e == 8 ? (uint32_t)(Ly.nmain / 32) : 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, (uint32_t)Ly.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  // ======================= back-substitution warp =======================
  if (warp == Ly.bwarp) {
    float* xv = smem + Ly.off_xv;
    float* lbuf = smem + Ly.off_lb;
    const int lbs = (K16 - 16 > 0 ? K16 - 16 : 1) * 16;  // floats per L block buffer
    uint32_t lb_use = 0;  // global L-block counter (lfull phases: block use u -> buffer u&1)
    int n = 0;
    for (int64_t sl = blockIdx.x; sl < p.nsys; sl += gridDim.x, ++n) {
      const int slot = n & 1;
      int64_t q;
      int i;
      sys_of(p, sl, q, i);
      const int64_t sys = q * k + i;  // global system index (error convention)
      mbar_wait(&fact[slot], (n >> 1) & 1);
      unsigned* ssc = slotsc + 4 * slot;
      if (ssc[3] == 0u) {
        const float* L11 = smem + Ly.off_l11 + slot * P * 152;
        const float* yv = smem + Ly.off_yv + slot * K16;
        const float* Lsl = Lscr + (size_t)slot * Ly.lb;
        // blocks b = P-2 .. 0 carry L rows below them; prefetch the first one
        auto issue_blk = [&](int b, uint32_t use) {
          const uint32_t bytes = (uint32_t)(K16 - 16 * b - 16) * 64u;
          if (lane == 0) {
            mbar_expect_tx(&lfull[use & 1], bytes);
            bulk_g2s(lbuf + (use & 1) * lbs, Lsl + lb_off(b, K16), bytes, &lfull[use & 1]);
          }
        };
        if (P >= 2) issue_blk(P - 2, lb_use);
        for (int b = P - 1; b >= 0; --b) {
          // lanes 0..15: column u = lane of W_b = L_bb^{-1} (independent of x)
          const float* Lbb = L11 + b * 152;
          float w[16];
          {
            const int u = lane & 15;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              float acc = (t == u) ? 1.f : 0.f;
#pragma unroll
              for (int v = 0; v < t; ++v) acc = fmaf(-Lbb[t * (t + 1) / 2 + v], w[v], acc);
              w[t] = (t >= u) ? acc * Lbb[136 + t] : 0.f;
            }
          }
          // s_t = sum_{c >= 16b+16} L[c][16b+t] x_c   (lane: rows rho = lane>>2 + 8m, cols 4(lane&3)..)
          float v4[4] = {0.f, 0.f, 0.f, 0.f};
          const int R = K16 - 16 * b - 16;
          if (R > 0) {
            const uint32_t use = lb_use++;
            mbar_wait(&lfull[use & 1], (use >> 1) & 1);
            if (b >= 1) issue_blk(b - 1, lb_use);  // prefetch the next block (other buffer)
            const float* blk = lbuf + (use & 1) * lbs;
            for (int rho = lane >> 2; rho < R; rho += 8) {
              const float xc = xv[16 * b + 16 + rho];
              const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * (lane & 3));
              v4[0] = fmaf(l4.x, xc, v4[0]);
              v4[1] = fmaf(l4.y, xc, v4[1]);
              v4[2] = fmaf(l4.z, xc, v4[2]);
              v4[3] = fmaf(l4.w, xc, v4[3]);
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1)
#pragma unroll
              for (int e = 0; e < 4; ++e) v4[e] += __shfl_xor_sync(kFull, v4[e], o);
            __syncwarp();  // everyone done with this buffer before it is refilled
          }
          // lane t (< 16): z_t = y_t - s_t ; x_t = sum_{u >= t} W[u][t] z_u
          const int t = lane & 15;
          float st = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float other = __shfl_sync(kFull, v4[e], (t >> 2));  // lane (t>>2) holds cols 4(t>>2)..
            if ((t & 3) == e) st = other;
          }
          const float z = yv[16 * b + t] - st;
          float x = 0.f;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float zu = __shfl_sync(kFull, z, u);
            x = fmaf(w[u], zu, x);  // w[u] = W[u][t] (lane t holds column t); zero for u < t
          }
          if (lane < 16) xv[16 * b + t] = x;
          __syncwarp();
        }
        // row of C, singularity verdict
        float* Crow = p.C + ((size_t)q * k + i) * k;
        bool nf = false;
        for (int c = lane; c < k; c += 32) {
          const float x = xv[c];
          nf |= !(fabsf(x) <= FLT_MAX);
          Crow[c] = x;
        }
        nf = __any_sync(kFull, nf);
        if (lane == 0) {
          const float dm = __uint_as_float(ssc[0]);
          const float pm = __uint_as_float(ssc[1]);
          float rc = dm > 0.f ? pm / dm : 0.f;
          if (!(rc >= 0.f)) rc = 0.f;
          if (ssc[2] || nf || !(rc >= p.rcond_thr)) atomicMin(p.fail_min, (unsigned long long)sys);
          atomicMin(p.rcond_min_bits, __float_as_uint(rc));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bsub[slot]);
    }
    return;
  }

  // ======================= MMA-issue warp =======================
  // Per panel: wait until every main warp has stored its L21 operands, release the
  // panel's y to the main warps (ysync), then issue the tensor-core trailing update
  // of every group: lookahead (next panel's 16 columns, committed to LA) first,
  // then the rest (REST).
  if (warp == Ly.mwarp) {
    if (lane == 0) {
      const uint32_t hib = su32(opnd_hi), lob = su32(opnd_lo);
      auto mma3 = [&](int glo_, int gbase_, int c0, int N) {
        const uint32_t arow = (uint32_t)(glo_ >> 3) * 512u;
        const uint32_t brow = (uint32_t)(c0 >> 3) * 512u;
        const uint32_t id = idesc_tf32(N);
        const uint32_t dcol = tbase + (uint32_t)(gbase_ + c0 - 16);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = (uint32_t)ks * 256u;
          const uint64_t ah = sdesc(hib + arow + ko), al = sdesc(lob + arow + ko);
          const uint64_t bh = sdesc(hib + brow + ko), bl = sdesc(lob + brow + ko);
          mma_tf32(dcol, ah, bh, id);
          mma_tf32(dcol, ah, bl, id);
          mma_tf32(dcol, al, bh, id);
        }
      };
      uint32_t gm = 0;
      for (int64_t sl = blockIdx.x; sl < p.nsys; sl += gridDim.x) {
        for (int pp = 0; pp < P; ++pp, ++gm) {
          mbar_wait(opsready, gm & 1);
          mbar_arrive(ysync);
          tc_fence_after();
          const int r0 = 16 * pp + 16;
#pragma unroll
          for (int gg = 0; gg < kMaxGroups; ++gg)
            if (gg < Ly.G && Ly.hi[gg] > r0) mma3(Ly.lo[gg], Ly.base[gg], r0, 16);
          mma_commit(&mbar[0]);
#pragma unroll
          for (int gg = 0; gg < kMaxGroups; ++gg) {
            if (gg >= Ly.G) continue;
            int c0 = r0 + 16;
            while (c0 < Ly.hi[gg]) {
              const int N = min(256, Ly.hi[gg] - c0);
              mma3(Ly.lo[gg], Ly.base[gg], c0, N);
              c0 += N;
            }
          }
          mma_commit(&mbar[1]);
        }
      }
    }
    return;
  }

  // ======================= main warps =======================
  // warp w -> group g = w/4, TMEM lane quarter m = w%4, row lo[g] + 32m + lane
  const int grp = warp >> 2, quarter = warp & 3;
  const bool has_grp = grp < Ly.G;
  int glo = 0, ghi = 0, gbase = 0;  // static indexing only (no local-memory copy of Ly)
#pragma unroll
  for (int gg = 0; gg < kMaxGroups; ++gg)
    if (gg == grp && has_grp) {
      glo = Ly.lo[gg];
      ghi = Ly.hi[gg];
      gbase = Ly.base[gg];
    }
  const int row = glo + 32 * quarter + lane;
  const bool row_valid = has_grp && row < ghi;
  const bool is_aug = tid == Ly.aug_tid;  // augmented right-hand-side "row"
  const uint32_t tq = tbase + ((uint32_t)(32 * quarter) << 16) + (uint32_t)gbase - 16u;  // + column c

  uint32_t g = 0;  // global panel counter (LA / REST mbarrier phases)
  bool any_mma = false;

  int n = 0;
  for (int64_t sl = blockIdx.x; sl < p.nsys; sl += gridDim.x, ++n) {
    const int slot = n & 1;
    int64_t q;
    int i;
    sys_of(p, sl, q, i);
    const bool tr_on = blockIdx.x == (unsigned)p.trace_block && n == 1;
    TC_TRACE(tid == 0, 0);
    float* L11all = smem + Ly.off_l11 + slot * P * 152;
    float* yv = smem + Ly.off_yv + slot * K16;
    float* Lslot = Lscr + (size_t)slot * Ly.lb;

    // slot reuse: the back-substitution of system n-2 must be done with it
    if (n >= 2) mbar_wait(&bsub[slot], ((n - 2) >> 1) & 1);
    if (tid == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[e] = 0u;
      sc[1] = __float_as_uint(FLT_MAX);
    }
    float ev_max = 0.f;
    bool skip = false;
    if constexpr (MASK_MODE == 1) {
      main_sync(NM);
      float m = 0.f;
      for (int c = tid; c < k; c += NM)
        m = fmaxf(m, fmaxf(p.ev1[(size_t)q * k + c], p.ev2[(size_t)q * k + c]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
      if (lane == 0) atomicMax(&sc[3], __float_as_uint(m));
      main_sync(NM);
      ev_max = __uint_as_float(sc[3]);
      skip = !(ev_max > 0.f);
    }

    // ---- staging: row r of (G + lambda*diag(m_i) + ridge*I), identity padding ----
    // Row r of G (read as column r, G[c][r]: coalesced; the lower triangle used is
    // G's upper triangle, as the SIMT solver; G = A A^T is symmetric by
    // construction).  Columns 0..15 stay in registers (panel 0), the rest go to the
    // group's TMEM region, two chunks of loads in flight.
    TC_TRACE(tid == 0, 398);
    float rhs = 0.f, dmax = 0.f, dadd = 0.f;
    const bool ld_ok = row_valid && row < k && !skip;
    if (ld_ok) {
      rhs = p.rhs_unit < 0 ? p.rhs[((size_t)q * k + i) * k + row] : (row == p.rhs_unit ? 1.f : 0.f);
      dadd = p.lambda * mask_entry<MASK_MODE>(p, q, i, row, ev_max) + p.ridge;
    }
    const float* Gq = p.gram + (size_t)q * k * k;
    // previous system's MMAs must be complete before TMEM is rewritten
    if (any_mma) {
      mbar_wait(&mbar[1], (g - 1) & 1);
      tc_fence_after();
    }
    TC_TRACE(tid == 0, 399);
    float a0[16];
    {
      const int ncb = ghi >> 4;        // column chunks of this group (warp-uniform)
      const int dcb = row >> 4, dt = row & 15;  // chunk / slot of the diagonal entry
      auto fix_diag = [&](float (&v)[16], int cb) {
        if (row_valid && dcb == cb) {
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (u == dt) {
              v[u] = row < k ? v[u] + dadd : 1.f;
              dmax = row < k ? fabsf(v[u]) : 0.f;
            }
        }
      };
      for (int cb = 1; cb < ncb; cb += 2) {  // two chunks of loads in flight
        float b0[16], b1[16];
        load_cols(Gq, k, row, ld_ok, cb, b0);
        if (cb + 1 < ncb) load_cols(Gq, k, row, ld_ok, cb + 1, b1);
        fix_diag(b0, cb);
        tmem_st16(tq + (uint32_t)(16 * cb), b0);
        if (cb + 1 < ncb) {
          fix_diag(b1, cb + 1);
          tmem_st16(tq + (uint32_t)(16 * (cb + 1)), b1);
        }
      }
      load_cols(Gq, k, row, ld_ok, 0, a0);
      if (row_valid && dcb == 0) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (u == dt) {
            a0[u] = row < k ? a0[u] + dadd : 1.f;
            dmax = row < k ? fabsf(a0[u]) : 0.f;
          }
      }
    }
    if (has_grp) tmem_st_wait();
    {
      float m = dmax;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
      if (lane == 0) atomicMax(&sc[0], __float_as_uint(m));
    }
    tc_fence_before();
    main_sync(NM);
    tc_fence_after();
    TC_TRACE(tid == 0, 1);

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
      if (pp > 0) {  // y of the previous panel (written by the rhs thread) is released by ysync
        mbar_wait(ysync, (g - 1) & 1);
        if (active) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 y4 = *reinterpret_cast<const float4*>(yv + j - 16 + 4 * c4);
            rhs = fmaf(-lprev[4 * c4], y4.x, rhs);
            rhs = fmaf(-lprev[4 * c4 + 1], y4.y, rhs);
            rhs = fmaf(-lprev[4 * c4 + 2], y4.z, rhs);
            rhs = fmaf(-lprev[4 * c4 + 3], y4.w, rhs);
          }
        }
      }
      float a[16];
      if (pp == 0) {
#pragma unroll
        for (int t = 0; t < 16; ++t) a[t] = a0[t];
      } else if (has_grp && ghi > j) {  // panel columns updated by the previous lookahead MMA
        mbar_wait(&mbar[0], (g - 1) & 1);
        tc_fence_after();
        tmem_ld16(tq + (uint32_t)j, a);
      } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) a[t] = 0.f;
      }
      TC_TRACE(tid == 0, 2 + 4 * pp);
      // b. diagonal block (rows j..j+15 live in one warp)
      const bool in_diag = active && row < j + 16;
      int dwarp = 0;
#pragma unroll
      for (int gg = 0; gg < kMaxGroups; ++gg)
        if (gg < Ly.G && j >= Ly.lo[gg] && j < Ly.hi[gg]) dwarp = 4 * gg + ((j - Ly.lo[gg]) >> 5);
      if (warp == dwarp) {
        float iv = 0.f;
        diag_factor(a, iv, lane & 15, in_diag && row < k, pivmin, bad);
        if (in_diag) {
          const int gr = row - j;
          float* Lpk = L11all + pp * 152 + gr * (gr + 1) / 2;  // packed copy for the back-sub warp
          L11all[pp * 152 + 136 + gr] = iv;
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            LT[t * 16 + gr] = (t <= gr) ? a[t] : 0.f;  // transposed, for the TRSM
            if (t <= gr) Lpk[t] = a[t];
          }
          inv[gr] = iv;
          zb[gr] = rhs;
        }
        // the other half-warp's rows were clobbered by the factorization: reload
        if (pp == 0) {
#pragma unroll
          for (int t = 0; t < 16; ++t) a[t] = a0[t];
        } else {
          tmem_ld16(tq + (uint32_t)j, a);
        }
        TC_TRACE(row == j, 3 + 4 * pp);
      }
      main_sync(NM);
      // c. TRSM rows >= j+16 ; augmented row -> y for this panel
      float l[16];
      const bool trsm = active && row >= j + 16;
      if (trsm) {
        trsm_row(LT, inv, a, l);
      } else if (is_aug) {
        float z[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) z[t] = zb[t];
        trsm_row(LT, inv, z, l);
#pragma unroll
        for (int t = 0; t < 16; ++t) yv[j + t] = l[t];
      }
      // d. store L21: scratch (back substitution), operand hi/lo
      if (trsm) {
        float4* dst = reinterpret_cast<float4*>(Lslot + lb_off(pp, K16) + (size_t)(row - j - 16) * 16);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4)
          __stcg(dst + c4, make_float4(l[4 * c4], l[4 * c4 + 1], l[4 * c4 + 2], l[4 * c4 + 3]));
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
      }
      TC_TRACE(tid == 0, 4 + 4 * pp);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(opsready);  // operands of this panel stored
      any_mma = true;
#pragma unroll
      for (int t = 0; t < 16; ++t) lprev[t] = trsm ? l[t] : 0.f;
    }
    TC_TRACE(tid == 0, 200);

    // ---- hand the system to the back-substitution warp ----
    asm volatile("fence.proxy.async.global;" ::: "memory");  // L scratch -> bulk-copy reads
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
    main_sync(NM);
    if (tid == 0) {
      unsigned* ssc = slotsc + 4 * slot;
      ssc[0] = sc[0];
      ssc[1] = sc[1];
      ssc[2] = sc[2];
      ssc[3] = skip ? 1u : 0u;
      if (skip) atomicOr(p.flags, 32u);
      mbar_arrive(&fact[slot]);
    }
    TC_TRACE(tid == 0, 203);
  }
  // ---- teardown ----
  if (any_mma) {
    mbar_wait(&mbar[1], (g - 1) & 1);
    tc_fence_after();
  }
  main_sync(NM);
  if (warp == 0) tmem_dealloc(tbase, (uint32_t)Ly.tmem_cols);
}

}  // namespace

size_t tc_scratch_bytes(int k, int64_t nsys, int num_sms) {
  const TcLayout L = make_layout(k);
  const int64_t maxgrid = (int64_t)num_sms * L.cps;
  const int64_t grid = nsys < maxgrid ? nsys : maxgrid;
  return (size_t)grid * 2 * (size_t)L.lb * sizeof(float);
}

bool tc_supported(int k, int optin_smem) {
  if (k < 1) return false;
  const TcLayout L = make_layout(k);
  if (L.tmem_cols > 512 || L.cps < 1 || L.threads > 384) return false;
  return (size_t)L.floats * 4 <= (size_t)optin_smem;
}

// Host-side launcher for the tensor-core solver (p.tc_scratch must hold
// tc_scratch_bytes(k, nsys, SMs)).
cudaError_t launch_chol_tc(const SolveParams& p, int mask_mode, cudaStream_t stream) {
  if (p.nsys <= 0) return cudaSuccess;
  int dev = 0, optin = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TcLayout L = make_layout(p.k);
  if (L.tmem_cols > 512 || L.cps < 1 || L.threads > 384 || !p.tc_scratch) return cudaErrorNotSupported;
  if (const char* c = std::getenv("FMAP_TC_CPS")) L.cps = std::max(1, std::min(L.cps, std::atoi(c)));  // diagnostics
  // cap residency at L.cps CTAs per SM through the shared-memory request, so no
  // CTA ever waits on a TMEM allocation
  size_t smem = (size_t)L.floats * 4;
  const size_t floor_req = 233472 / (size_t)(L.cps + 1) + 1;
  if (smem < floor_req) smem = floor_req;
  if (smem > (size_t)optin) {
    if ((size_t)L.floats * 4 > (size_t)optin) return cudaErrorNotSupported;
    smem = (size_t)optin;
  }
  void (*fn)(SolveParams, TcLayout) = nullptr;
  if (L.cps >= 2 && L.threads <= 288) {  // two CTAs per SM
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 288, 2>; break;
      case 1: fn = chol_tc_kernel<1, 288, 2>; break;
      default: fn = chol_tc_kernel<2, 288, 2>; break;
    }
  } else {
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 384, 1>; break;
      case 1: fn = chol_tc_kernel<1, 384, 1>; break;
      default: fn = chol_tc_kernel<2, 384, 1>; break;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t maxgrid = (int64_t)sms * L.cps;
  const unsigned grid = (unsigned)(p.nsys < maxgrid ? p.nsys : maxgrid);
  fn<<<grid, L.threads, smem, stream>>>(p, L);
  return cudaGetLastError();
}

// ===========================================================================
// Spectral projection on the tensor core (north_star stage 1):
//   Out[q] (k x d) = Phi_q^T (k x n) * diag(Mass_q) * F_q (n x d)
// as a 3xTF32 tcgen05 GEMM, M = 128 basis functions per CTA, N = d (<= 256),
// K = vertices in 16-vertex stages.  Eight producer warps load Phi and F with
// coalesced column loads (lane = basis function / feature channel), apply the
// Mass scaling, split hi/lo and store the tiles K-major (core matrices, the same
// layout as the solver's operands); one MMA-issue warp runs 6 MMAs per stage
// (2 k-steps x {hi*hi, hi*lo, lo*hi}); two stages in flight (mbarriers).  The
// accumulator lives in TMEM; the epilogue writes Out rows coalesced per lane.
// Bound: HBM (4(nk + n + nd) bytes per shape) and the tensor pipe.
// ===========================================================================
namespace {
constexpr int kPjK = 16;      // vertices per stage
constexpr int kPjThreads = 288;  // 8 producer warps + 1 MMA warp

__device__ __forceinline__ float tf32_hi(float x) {  // round-to-nearest TF32
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}

__global__ void __launch_bounds__(kPjThreads, 2) proj_tc_kernel(const float* __restrict__ phi,
                                                                  const float* __restrict__ mass,
                                                                  const float* __restrict__ F,
                                                                  int64_t n, int k, int d, int N,
                                                                  float* __restrict__ out) {
  extern __shared__ __align__(1024) float smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.y, i0 = blockIdx.x * 128;
  const float* Pq = phi + (size_t)q * n * k;
  const float* Fq = F + (size_t)q * n * d;
  const float* Mq = mass + (size_t)q * n;
  // per stage buffer: A_hi | A_lo (128 x 16) | B_hi | B_lo (N x 16)
  const int abytes = 128 * kPjK, bbytes = N * kPjK;  // floats
  const int sstride = 2 * abytes + 2 * bbytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * sstride);  // full[2], empty[2], done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 5);
  if (tid == 0) {
    mbar_init(&bar[0], 8);
    mbar_init(&bar[1], 8);
    mbar_init(&bar[2], 1);
    mbar_init(&bar[3], 1);
    mbar_init(&bar[4], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nst = (int)((n + kPjK - 1) / kPjK);

  if (warp == 8) {  // ---- MMA issue ----
    if (lane == 0) {
      const uint32_t id = idesc_tf32(N) & ~(1u << 13);  // D += A*B (no negation)
      for (int st = 0; st < nst; ++st) {
        const int buf = st & 1;
        mbar_wait(&bar[buf], (st >> 1) & 1);
        tc_fence_after();
        const uint32_t ah = su32(smem + buf * sstride), al = ah + abytes * 4;
        const uint32_t bh = al + abytes * 4, bl = bh + bbytes * 4;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = (uint32_t)ks * 256u;
          mma_tf32(tbase, sdesc(ah + ko), sdesc(bh + ko), id, (st > 0 || ks > 0) ? 1u : 0u);
          mma_tf32(tbase, sdesc(ah + ko), sdesc(bl + ko), id, 1u);
          mma_tf32(tbase, sdesc(al + ko), sdesc(bh + ko), id, 1u);
        }
        mma_commit(&bar[2 + buf]);
      }
      mma_commit(&bar[4]);
    }
  } else {  // ---- producers (256 threads) ----
    for (int st = 0; st < nst; ++st) {
      const int buf = st & 1;
      const int64_t v0 = (int64_t)st * kPjK;
      // loads first (latency overlaps the wait for the buffer)
      float av[2][4], bv[4][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tid + 256 * h, i = c & 127, kc = c >> 7;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t v = v0 + 4 * kc + u;
          av[h][u] = (v < n && i0 + i < k) ? __ldg(Pq + v * k + i0 + i) : 0.f;
        }
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int c = tid + 256 * h;
        const int t = c % N, kc = c / N;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t v = v0 + 4 * kc + u;
          bv[h][u] = (kc < 4 && v < n && t < d) ? __ldg(Mq + v) * __ldg(Fq + v * d + t) : 0.f;
        }
      }
      if (st >= 2) mbar_wait(&bar[2 + buf], ((st - 2) >> 1) & 1);  // MMAs of stage st-2 done
      float* S = smem + buf * sstride;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tid + 256 * h, i = c & 127, kc = c >> 7;
        const int o = (i >> 3) * 128 + kc * 32 + (i & 7) * 4;
        float hv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) hv[u] = tf32_hi(av[h][u]);
        *reinterpret_cast<float4*>(S + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<float4*>(S + abytes + o) =
            make_float4(av[h][0] - hv[0], av[h][1] - hv[1], av[h][2] - hv[2], av[h][3] - hv[3]);
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int c = tid + 256 * h;
        const int t = c % N, kc = c / N;
        if (kc < 4) {
          const int o = (t >> 3) * 128 + kc * 32 + (t & 7) * 4;
          float hv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) hv[u] = tf32_hi(bv[h][u]);
          *reinterpret_cast<float4*>(S + 2 * abytes + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<float4*>(S + 2 * abytes + bbytes + o) =
              make_float4(bv[h][0] - hv[0], bv[h][1] - hv[1], bv[h][2] - hv[2], bv[h][3] - hv[3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[buf]);
    }
    // ---- epilogue: TMEM -> Out (warp w: lane quarter w % 4, column half w / 4) ----
    mbar_wait(&bar[4], 0);
    tc_fence_after();
    const int quarter = warp & 3, half = warp >> 2;
    const int i = i0 + 32 * quarter + lane;
    const int nh = N / 2;
    for (int c0 = half * nh; c0 < (half + 1) * nh; c0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * quarter) << 16) + (uint32_t)c0, v);
      if (i < k) {
        float* o = out + ((size_t)q * k + i) * d + c0;
        if (c0 + 16 <= d && (d & 3) == 0) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4)
            *reinterpret_cast<float4*>(o + 4 * c4) = make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (c0 + t < d) o[t] = v[t];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}
}  // namespace

// Tensor-core projection (d <= 256); returns cudaErrorNotSupported otherwise.
cudaError_t launch_project_tc(const float* phi, const float* mass, const float* F, int64_t b,
                              int64_t n, int k, int d, float* out, cudaStream_t st) {
  if (d > 256 || d < 1 || k < 1 || n < 1 || b < 1) return cudaErrorNotSupported;
  const int N = (d + 15) & ~15;
  const size_t smem = (size_t)(2 * (2 * 128 * kPjK + 2 * N * kPjK)) * 4 + 64;
  const size_t req = smem < 233472 / 3 + 1 ? 233472 / 3 + 1 : smem;  // <= 2 CTAs per SM (TMEM 256 cols)
  cudaError_t e = cudaFuncSetAttribute(proj_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)req);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((k + 127) / 128), (unsigned)b);
  proj_tc_kernel<<<grid, kPjThreads, req, st>>>(phi, mass, F, n, k, d, N, out);
  return cudaGetLastError();
}

}  // namespace fmap
