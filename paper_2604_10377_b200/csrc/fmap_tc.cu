// Batched Cholesky solver with the trailing update on the 5th-generation tensor
// cores (tcgen05, kind::tf32, 3xTF32 split) and the trailing matrix resident in
// tensor memory (TMEM) -- sm_100a.  For every shape pair q and row i:
//     (G_q + lambda*diag(M_q[i,:]) + ridge*I) x = R_q[i,:]^T,   C_q[i,:] = x^T
// replacing the reference's per-system PartialPivLU
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170) driven by
// solve_batched_many (:220-322), with the reference's rcond test (:164-168).
//
// Two kernels per solve:
//
// chol_tc_kernel -- factorization.  One CTA owns one row system at a time
// (persistent over systems; two CTAs per SM for K16 <= 208, K16 = k rounded up to
// 16, rows/cols k..K16-1 identity padding).
//   * TMEM: rows split into groups of <= 128 from the bottom; group g keeps rows
//     [lo_g, hi_g) on TMEM lanes and matrix columns [16, hi_g) (panel 0's columns
//     stay in shared memory).  k = 200: 192 + 64 = 256 columns per system.
//   * Operand buffers (shared memory): the current panel's L21 rows split into
//     TF32 hi/lo parts, K-major core matrices, used as both MMA operands.
//   * Per 16-column panel p (j = 16 p):
//       a  rows >= j load their 16 panel entries from TMEM once their group's
//          lookahead MMA (panel p-1) has landed;
//       b  the warp holding rows j..j+15 factors a copy of the 16x16 diagonal
//          block (lane per row, shuffles) and publishes L11^T and 1/L_tt;  | barrier
//       c  every row >= j+16 solves its L21 row against L11 (TRSM);
//       d  hi/lo operands to shared memory, per-group "operands ready" arrival;
//          then, off the chain, the fp32 L21 row and the packed diagonal block
//          go to the per-system store for the back substitution;
//       e  one MMA-issue thread: per row group (the group holding the next
//          diagonal block first) the lookahead MMA (next panel's 16 columns),
//          then the rest of the trailing update, each committed to an mbarrier;
//          the next system's G is staged into dead TMEM columns by TMA +
//          tcgen05.cp meanwhile.
// chol_backsub_kernel -- one warp per system over the stored factor: forward
// pass y = L^{-1} r with the rcond certificate's u = M(L)^{-1} e, backward pass
// x = L^{-T} y with w = M(L)^{-T} e, the verdict (certificate, or the exact
// Hager/Higham estimate on the rare systems it does not clear), the row of C.
//
// Singular = non-positive / non-finite pivot, rcond below the threshold, or a
// non-finite solution (the lowest failing system index wins).
#include "fmap_kernels.cuh"
#include "fmap_solver.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>

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
  int ns;  // systems factored in lockstep per CTA (same row -> same thread)
  int tma; // next pair's G staged by TMA + tcgen05.cp during the current pair's panels
  int nmain, mwarp, threads;
  int tcols1;     // TMEM columns of one system
  int tmem_cols;  // allocated (ns * tcols1, power of two)
  int Rop;  // operand buffer rows
  int cps;  // CTAs per SM
  // offsets in floats from the dynamic smem base
  int off_hi, off_lo, off_lt, off_a0, off_stg, off_misc;
  int floats;
  long long lb;  // floats of one L scratch slot (global memory)
};

// First float of block p's L21 rows in an L scratch slot: block p holds rows
// 16p+16 .. K16-1, 16 floats each.
__host__ __device__ inline long long lb_off(int p, int K16) {
  return 16ll * p * (K16 - 16) - 128ll * p * (p - 1);
}

// ns = 0: pick.  One system per CTA (two CTAs per SM for k <= 256) measured faster
// than two lockstep systems per CTA once staging moved to TMA + tcgen05.cp (2.23 vs
// 2.92 ms at cfg2); ns = 2 stays available (FMAP_TC_NS=2).
__host__ inline TcLayout make_layout(int k, int ns = 0) {
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
  int c = 32;
  while (c < total && c < 1024) c <<= 1;
  L.tcols1 = c;
  if (ns <= 0 || 2 * c > 512) ns = 1;
  L.ns = ns;
  L.tmem_cols = ns * c;
  const int ntop = L.hi[L.G - 1] - L.lo[L.G - 1];
  L.nmain = 32 * (4 * (L.G - 1) + (ntop + 31) / 32);
  L.mwarp = L.nmain / 32;      // MMA-issue warp
  L.threads = L.nmain + 32;
  L.Rop = L.K16 > kTL ? L.K16 : kTL;
  int o = 0;
  L.off_hi = o;  o += ns * L.Rop * 16;          // per system
  L.off_lo = o;  o += ns * L.Rop * 16;
  L.off_lt = o;  o += ns * (256 + 16);          // per system: diagonal block (transposed) + 1/L_tt
  o = (o + 31) & ~31;                           // 128 B aligned (TMA destination)
  L.off_a0 = o;  o += ns * L.K16 * 16;          // panel-0 columns of every row (float4 [h][t4][row])
  o = (o + 255) & ~255;                         // 1 KB aligned (TMA destination)
  L.off_stg = o; o += ns * L.G * 4 * kTL * 4;   // one G chunk of every (system, group): [h][g][u][128 rows][4]
  L.off_misc = o; o += 128;
  L.floats = o;
  L.lb = (lb_off(L.P, L.K16) + 31) & ~31ll;
  const int cps_tmem = L.tmem_cols <= 512 ? 512 / L.tmem_cols : 0;
  const size_t bytes = (size_t)L.floats * 4 + 1024;
  const int cps_smem = (int)(233472 / bytes);
  L.cps = cps_tmem < cps_smem ? cps_tmem : cps_smem;
  return L;
}

using namespace ptx;

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
  // software-pipelined: column t+1 of LT (and 1/L_{t+1,t+1}) is loaded while step t
  // runs, so the shared-memory latency stays off the 16-step FMUL + FFMA chain
  float4 cur[4], nxt[4];
  float ivc = inv[0], ivn = 0.f;
#pragma unroll
  for (int c4 = 0; c4 < 4; ++c4) cur[c4] = *reinterpret_cast<const float4*>(LT + 4 * c4);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    if (t < 15) {
      ivn = inv[t + 1];
#pragma unroll
      for (int c4 = (t + 2) >> 2; c4 < 4; ++c4) nxt[c4] = *reinterpret_cast<const float4*>(LT + (t + 1) * 16 + 4 * c4);
    }
    l[t] = a[t] * ivc;
#pragma unroll
    for (int c4 = (t + 1) >> 2; c4 < 4; ++c4) {
      const float4 col = cur[c4];
      if (4 * c4 > t) a[4 * c4] = fmaf(-l[t], col.x, a[4 * c4]);
      if (4 * c4 + 1 > t) a[4 * c4 + 1] = fmaf(-l[t], col.y, a[4 * c4 + 1]);
      if (4 * c4 + 2 > t) a[4 * c4 + 2] = fmaf(-l[t], col.z, a[4 * c4 + 2]);
      if (4 * c4 + 3 > t) a[4 * c4 + 3] = fmaf(-l[t], col.w, a[4 * c4 + 3]);
    }
    if (t < 15) {
#pragma unroll
      for (int c4 = (t + 2) >> 2; c4 < 4; ++c4) cur[c4] = nxt[c4];
      ivc = ivn;
    }
  }
}

// Debug phase trace (FMAP_TRACE_FILE): clock64 stamps of one CTA's second system.
// Compiled in only with -DFMAP_TC_TRACE (tools/trace_panel.py), so the product
// kernel carries no stamp code.
#ifdef FMAP_TC_TRACE
#define TC_TRACE(cond, slot)                                                              \
  do {                                                                                    \
    if (p.trace && tr_on && (cond)) p.trace[(slot)] = clock64();                          \
  } while (0)
#else
#define TC_TRACE(cond, slot) \
  do {                       \
  } while (0)
#endif

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

// Load G[row][16cb .. 16cb+15] (zero beyond column k-1).  The same entries the
// TMA path stages (only c <= row is ever used; the rest is carried along unread).
__device__ __forceinline__ void load_cols(const float* __restrict__ Gq, int k, int row, bool ok, int cb,
                                          float (&v)[16]) {
  const int c0 = 16 * cb;
  const float* src = Gq + (size_t)row * k + c0;
  if (ok && (k & 3) == 0 && c0 + 16 <= k) {
#pragma unroll
    for (int t4 = 0; t4 < 4; ++t4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(src) + t4);
      v[4 * t4] = x.x;
      v[4 * t4 + 1] = x.y;
      v[4 * t4 + 2] = x.z;
      v[4 * t4 + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = (ok && c0 + t < k) ? __ldg(src + t) : 0.f;
  }
}

// ---------------------------------------------------------------------------
// CTA iteration n handles NS systems (sl = NS*pi + h) in lockstep: thread `row`
// owns row `row` of every one of them (system h in TMEM columns h*tcols1 + ...,
// its own operand buffers, L scratch and slot NS*(n&1)+h).  Main warps
// (0..nmain/32-1): staging + blocked factorization (the back substitution is
// chol_backsub_kernel, over the stored factors).  The 16x16 diagonal factor of
// system 1 runs on the half-warp that does not hold the diagonal rows, so both
// blocks cost one dependency chain.
// ---------------------------------------------------------------------------
template <int MASK_MODE, int NS, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
    chol_tc_kernel(SolveParams p, TcLayout Ly, const __grid_constant__ CUtensorMap tmG,
                   const __grid_constant__ CUtensorMap tmA) {
  extern __shared__ __align__(1024) float smem[];
  const int k = p.k, K16 = Ly.K16, P = Ly.P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NM = Ly.nmain;
  const int opsz = Ly.Rop * 16;  // floats of one operand buffer
  float* opnd_hi = smem + Ly.off_hi;  // system h: + h*opsz
  float* opnd_lo = smem + Ly.off_lo;
  float* LTb = smem + Ly.off_lt;  // system h: LT = LTb + 272h, LT[t][c] = L[c][t]; inv = LT + 256
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + Ly.off_misc);
  // mbar[0 .. 3) la[g]: lookahead MMA of row group g done; [3] REST MMAs done;
  // [4 .. 7) ops[g]: operands of row group g stored (one arrival per warp of the group);
  // [7] chk (G chunk TMA), [8] cpd (tcgen05.cp done), [9] a0f (panel-0 TMA), [10] stg
  // (next pair fully staged: MMA warp -> main warps)
  uint64_t* la = mbar;
  uint64_t* rest = mbar + 3;
  uint64_t* ops = mbar + 4;
  uint64_t* chk = mbar + 7;
  uint64_t* cpd = chk + 1;
  uint64_t* a0f = chk + 2;
  uint64_t* stg = chk + 3;
  float4* a0s = reinterpret_cast<float4*>(smem + Ly.off_a0);  // panel-0 columns: [(h*4 + t4)*K16 + row]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Ly.off_misc + 48);
  unsigned* scb = reinterpret_cast<unsigned*>(smem + Ly.off_misc + 56);  // [n&1][h][8]
  // sc[8h+0] dmax bits, [1] pivmin bits, [2] bad, [3] (unused), [4] ||A||_1 bits (current
  // systems); double-buffered by iteration parity, reset right after the hand-off
  unsigned* slotsc = reinterpret_cast<unsigned*>(smem + Ly.off_misc + 88);  // [slot][8]
  // per-system store for chol_backsub_kernel (launch-local system sl): L21 blocks,
  // packed diagonal blocks (+ 1/L_tt), status words
  float* Lst = p.tc_scratch;
  float* L11st = Lst + (size_t)p.nsys * Ly.lb;
  unsigned* stst = reinterpret_cast<unsigned*>(L11st + (size_t)p.nsys * P * 152);
  const int64_t npi = (p.nsys + NS - 1) / NS;

  // ---- one-time setup ----
  for (int e = tid; e < 2 * NS * opsz; e += Ly.threads) smem[Ly.off_hi + e] = 0.f;
  if (tid < 2 * NS) {
    scb[8 * tid + 0] = 0u;
    scb[8 * tid + 1] = __float_as_uint(FLT_MAX);
    scb[8 * tid + 2] = 0u;
    scb[8 * tid + 3] = 0u;
    scb[8 * tid + 4] = 0u;
  }
  if (tid == 0) {
    for (int e = 0; e < 11; ++e) {
      uint32_t cnt = 1u;
      if (e >= 4 && e < 4 + kMaxGroups)  // warps of row group e - 4 (4, the top group fewer)
        cnt = e - 4 < Ly.G - 1 ? 4u : (e - 4 == Ly.G - 1 ? (uint32_t)(Ly.nmain / 32 - 4 * (Ly.G - 1)) : 1u);
      mbar_init(&mbar[e], cnt);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, (uint32_t)Ly.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  // ======================= MMA-issue warp =======================
  // Per panel: per row group, wait until its warps have stored their L21 operands
  // and issue its lookahead MMA (next panel's 16 columns, committed to la[g]), the
  // group holding the next diagonal block first; then the rest of the trailing
  // update of every group (REST).
  if (warp == Ly.mwarp) {
    if (lane == 0) {
      auto mma3 = [&](int h, int glo_, int gbase_, int c0, int N) {
        const uint32_t hib = su32(opnd_hi + h * opsz), lob = su32(opnd_lo + h * opsz);
        const uint32_t arow = (uint32_t)(glo_ >> 3) * 512u;
        const uint32_t brow = (uint32_t)(c0 >> 3) * 512u;
        const uint32_t id = idesc_tf32(N);
        const uint32_t dcol = tbase + (uint32_t)(h * Ly.tcols1 + gbase_ + c0 - 16);
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
      // Staging of the NEXT pair (Ly.tma): chunk cb = matrix columns 16cb..16cb+15 of
      // every row.  After panel pp's opsready every main warp has read chunk pp of
      // the current pair, so the next pair's chunk pp is copied into those TMEM
      // columns (tcgen05.cp from a shared-memory tile filled by TMA one panel
      // earlier); its panel-0 columns go to a0s by TMA.
      float* stile = smem + Ly.off_stg;
      auto grp_has = [&](int gg, int cb) { return gg < Ly.G && cb < (Ly.hi[gg] >> 4); };
      auto tma_chunk = [&](int cb, const int64_t (&qn)[NS], const bool (&vn)[NS]) {
        uint32_t bytes = 0;
#pragma unroll
        for (int h = 0; h < NS; ++h)
#pragma unroll
          for (int gg = 0; gg < kMaxGroups; ++gg)
            if (vn[h] && grp_has(gg, cb)) bytes += 4u * kTL * 16u;
        mbar_expect_tx(chk, bytes);
#pragma unroll
        for (int h = 0; h < NS; ++h)
#pragma unroll
          for (int gg = 0; gg < kMaxGroups; ++gg)
            if (vn[h] && grp_has(gg, cb))
              tma_load_4d(stile + (h * Ly.G + gg) * 4 * (kTL * 4), &tmG, 0, Ly.lo[gg], 4 * cb, (int)qn[h], chk);
      };
      auto cp_chunk = [&](int cb, const bool (&vn)[NS]) {
#pragma unroll
        for (int h = 0; h < NS; ++h)
#pragma unroll
          for (int gg = 0; gg < kMaxGroups; ++gg)
            if (vn[h] && grp_has(gg, cb))
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                const uint32_t src = su32(stile + ((h * Ly.G + gg) * 4 + 2 * hf) * (kTL * 4));
                const uint32_t dst = tbase + (uint32_t)(h * Ly.tcols1 + Ly.base[gg] + 16 * cb - 16 + 8 * hf);
                tmem_cp_128x256b(dst, sdesc_ls(src, (uint32_t)kTL * 16u, 128u));
              }
      };
      uint32_t gm = 0, n_chk = 0, n_cpd = 0, n_a0 = 0;
      int nmi = 0;
      for (int64_t pi = blockIdx.x; pi < npi; pi += gridDim.x, ++nmi) {
        const bool tr_on = blockIdx.x == (unsigned)p.trace_block && nmi == 1;
        const int64_t pi2 = pi + gridDim.x;
        const bool pf = Ly.tma && pi2 < npi;
        int64_t qn[NS];
        bool vn[NS];
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          int in_;
          vn[h] = pf && NS * pi2 + h < p.nsys;
          sys_of(p, vn[h] ? NS * pi2 + h : 0, qn[h], in_);
        }
        bool cpd_pending = false;
        for (int pp = 0; pp < P; ++pp, ++gm) {
          const int r0 = 16 * pp + 16;
          // Lookahead per row group, the group holding the next diagonal block (rows
          // r0..r0+15, the B operand of every group's lookahead) first: its warps'
          // next panel waits only for its own lookahead, not for the slowest group's
          // operand stores (early panels: the 128-row bottom group).
          int gb = 0;
#pragma unroll
          for (int gg = 0; gg < kMaxGroups; ++gg)
            if (gg < Ly.G && r0 >= Ly.lo[gg] && r0 < Ly.hi[gg]) gb = gg;
#pragma unroll
          for (int pass = 0; pass < 2; ++pass)  // group gb, then the others (static indices)
#pragma unroll
            for (int gg = 0; gg < kMaxGroups; ++gg) {
              if (gg >= Ly.G || ((gg == gb) != (pass == 0))) continue;
              mbar_wait(&ops[gg], gm & 1);
              tc_fence_after();
              if (Ly.hi[gg] > r0)
#pragma unroll
                for (int h = 0; h < NS; ++h) mma3(h, Ly.lo[gg], Ly.base[gg], r0, 16);
              mma_commit(&la[gg]);
            }
          TC_TRACE(pp < 16, 800 + pp);
          TC_TRACE(pp < 16, 820 + pp);
          // next pair: panel-0 columns (a0s is free: every main warp is past panel 0)
          // and chunk pp into the tile (free once the previous chunk's copies are done)
          if (pf && pp == 0) {
            uint32_t bytes = 0;
#pragma unroll
            for (int h = 0; h < NS; ++h)
              if (vn[h]) bytes += 4u * (uint32_t)K16 * 16u;
            mbar_expect_tx(a0f, bytes);
#pragma unroll
            for (int h = 0; h < NS; ++h)
              if (vn[h]) tma_load_4d(a0s + h * 4 * K16, &tmA, 0, 0, 0, (int)qn[h], a0f);
          }
          if (pf && pp >= 1) {
            if (cpd_pending) {
              mbar_wait(cpd, n_cpd & 1);
              ++n_cpd;
              cpd_pending = false;
            }
            tma_chunk(pp, qn, vn);
          }
#pragma unroll
          for (int h = 0; h < NS; ++h)
#pragma unroll
            for (int gg = 0; gg < kMaxGroups; ++gg) {
              if (gg >= Ly.G) continue;
              int c0 = r0 + 16;
              while (c0 < Ly.hi[gg]) {
                const int N = min(256, Ly.hi[gg] - c0);
                mma3(h, Ly.lo[gg], Ly.base[gg], c0, N);
                c0 += N;
              }
            }
          mma_commit(rest);
          TC_TRACE(pp < 16, 840 + pp);
          if (pf && pp >= 1) {  // chunk pp of the current pair was read at this panel's top
            mbar_wait(chk, n_chk & 1);
            ++n_chk;
            cp_chunk(pp, vn);
            mma_commit(cpd);
            cpd_pending = true;
          }
        }
        if (pf) {  // hand the staged next pair to the main warps
          if (cpd_pending) {
            mbar_wait(cpd, n_cpd & 1);
            ++n_cpd;
          }
          mbar_wait(a0f, n_a0 & 1);
          ++n_a0;
          tc_fence_before();
          mbar_arrive(stg);
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
  const uint32_t tq = tbase + ((uint32_t)(32 * quarter) << 16) + (uint32_t)gbase - 16u;  // + column c
  const uint32_t tsys = (uint32_t)Ly.tcols1;  // TMEM column offset between systems

  uint32_t g = 0;  // global panel counter (LA / REST mbarrier phases)
  bool any_mma = false;
  const int ncb = ghi >> 4;  // column chunks of this warp's group (warp-uniform)

  // Staging of the NEXT pair is software-pipelined into the panel loop: after
  // panel pp has read its columns, chunk pp (matrix columns 16pp..16pp+15) is dead
  // in TMEM, so the next pair's chunk pp is loaded at the end of panel pp and
  // stored at the top of panel pp+1; chunk 0 (registers), the last chunk and the
  // per-row right-hand side / mask entry are loaded at the end of the last panel.
  bool pre = false;        // the current pair's G chunks were prefetched
  float mraw_n[NS];
  uint32_t n_stg = 0;
#pragma unroll
  for (int h = 0; h < NS; ++h) {
    mraw_n[h] = 0.f;
  }

  int n = 0;
  for (int64_t pi = blockIdx.x; pi < npi; pi += gridDim.x, ++n) {
    int64_t qs[NS];
    int is[NS];
    bool vld[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      const int64_t sl = NS * pi + h;
      vld[h] = sl < p.nsys;
      sys_of(p, vld[h] ? sl : 0, qs[h], is[h]);
    }
    const int64_t pi2 = pi + gridDim.x;  // next pair of this CTA
    const bool has_next = pi2 < npi;
    int64_t qn[NS];
    int in_[NS];
    bool ldn[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      const int64_t sl = NS * pi2 + h;
      ldn[h] = has_next && sl < p.nsys && row_valid && row < k;
      sys_of(p, ldn[h] ? sl : 0, qn[h], in_[h]);
    }
    const bool tr_on = blockIdx.x == (unsigned)p.trace_block && n == 1;
    TC_TRACE(tid == 0, 0);
    const int slot0 = 0;  // smem y slot of system h: slot0 + h
    unsigned* sc = scb + 8 * NS * (n & 1);
    float ev_max[NS];
    bool skip[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      ev_max[h] = 0.f;
      skip[h] = !vld[h];
    }
    if constexpr (MASK_MODE == 1) {  // the pair's normaliser max(ev1, ev2), from ev_max_check_kernel
#pragma unroll
      for (int h = 0; h < NS; ++h) {
        ev_max[h] = __ldg(p.ev_max + qs[h]);
        skip[h] = skip[h] || !(ev_max[h] > 0.f);
      }
    }

    // ---- staging: row r of (G + lambda*diag(m_i) + ridge*I), identity padding ----
    // Row r of G (read as column r, G[c][r]: coalesced; the lower triangle used is
    // G's upper triangle; G = A A^T is symmetric by
    // construction).  Columns 0..15 stay in registers (panel 0), the rest go to the
    // group's TMEM region.  Raw G first (prefetched during the previous pair's
    // panels, or loaded here for the first pair), then lambda*m + ridge is added to
    // the diagonal entry in place.
    TC_TRACE(tid == 0, 398);
    float dmax[NS], dadd[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      dmax[h] = 0.f;
      dadd[h] = 0.f;
      if (row_valid && row < k && !skip[h]) {
        if (MASK_MODE != 1 && pre) {
          dadd[h] = p.lambda * mraw_n[h] + p.ridge;
        } else {
          dadd[h] = p.lambda * mask_entry<MASK_MODE>(p, qs[h], is[h], row, ev_max[h]) + p.ridge;
        }
      }
    }
    // ||A||_1 inputs (the loads are in flight while the previous MMAs drain)
    float grr[NS], srow[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      const bool on = row_valid && row < k && vld[h] && !skip[h];
      grr[h] = on ? __ldg(p.gram + ((size_t)qs[h] * k + row) * k + row) : 0.f;
      srow[h] = on ? __ldg(p.gram_rowsum + (size_t)qs[h] * k + row) : 0.f;
    }
    // previous systems' MMAs must be complete before TMEM is rewritten
    if (any_mma) {
      mbar_wait(rest, (g - 1) & 1);
      tc_fence_after();
    }
    TC_TRACE(tid == 0, 399);
    {
      const int dcb = row >> 4, dt = row & 15;  // chunk / slot of the diagonal entry
      auto fix_diag = [&](float (&v)[16], int cb, int h) {
        if (row_valid && dcb == cb) {
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (u == dt) {
              v[u] = row < k ? v[u] + dadd[h] : 1.f;
              dmax[h] = row < k ? fabsf(v[u]) : 0.f;
            }
        }
      };
      if (!pre) {
        bool ld_ok[NS];
        const float* Gq[NS];
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          ld_ok[h] = row_valid && row < k && vld[h];
          Gq[h] = p.gram + (size_t)qs[h] * k * k;
        }
        if constexpr (NS == 1 && MAXT == 384) {  // one CTA per SM (K16 > 256): every system comes this way
          for (int cb = 1; cb < ncb; cb += 2) {  // two chunks of loads in flight
            float b0[16], b1[16];
            load_cols(Gq[0], k, row, ld_ok[0], cb, b0);
            if (cb + 1 < ncb) load_cols(Gq[0], k, row, ld_ok[0], cb + 1, b1);
            fix_diag(b0, cb, 0);
            tmem_st16(tq + (uint32_t)(16 * cb), b0);
            if (cb + 1 < ncb) {
              fix_diag(b1, cb + 1, 0);
              tmem_st16(tq + (uint32_t)(16 * (cb + 1)), b1);
            }
          }
        } else {
          for (int cb = 1; cb < ncb; ++cb) {  // one chunk of every system in flight
            float b[NS][16];
#pragma unroll
            for (int h = 0; h < NS; ++h) load_cols(Gq[h], k, row, ld_ok[h], cb, b[h]);
#pragma unroll
            for (int h = 0; h < NS; ++h) {
              fix_diag(b[h], cb, h);
              tmem_st16(tq + tsys * h + (uint32_t)(16 * cb), b[h]);
            }
          }
        }
        if (row_valid) {
#pragma unroll
          for (int h = 0; h < NS; ++h) {
            float v[16];
            load_cols(Gq[h], k, row, ld_ok[h], 0, v);
#pragma unroll
            for (int t4 = 0; t4 < 4; ++t4)
              a0s[(h * 4 + t4) * K16 + row] = make_float4(v[4 * t4], v[4 * t4 + 1], v[4 * t4 + 2], v[4 * t4 + 3]);
          }
        }
      } else {
        mbar_wait(stg, n_stg & 1);  // TMA / tcgen05.cp staging of this pair complete
        ++n_stg;
        tc_fence_after();
        // diagonal entries in TMEM: this warp's rows span chunks c0w, c0w+1
        const int c0w = (glo + 32 * quarter) >> 4;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = c0w + e;
          if (cc >= 1 && cc < ncb) {
#pragma unroll
            for (int h = 0; h < NS; ++h) {
              float v[16];
              tmem_ld16(tq + tsys * h + (uint32_t)(16 * cc), v);
              fix_diag(v, cc, h);
              tmem_st16(tq + tsys * h + (uint32_t)(16 * cc), v);
            }
          }
        }
      }
      if (row_valid && row < 16) {  // diagonal entries of panel 0 (shared memory)
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          float* e = reinterpret_cast<float*>(a0s + (h * 4 + (row >> 2)) * K16 + row) + (row & 3);
          *e = row < k ? *e + dadd[h] : 1.f;
          dmax[h] = row < k ? fabsf(*e) : 0.f;
        }
      }
    }
    if (has_grp) tmem_st_wait();
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      // row 1-norm of the assembled system: sum_c |G[row][c]| with the diagonal
      // entry replaced by G[row][row] + lambda m + ridge (||A||_1 = max over rows,
      // A symmetric) -- the matrix norm of the reference's rcond (solver.hpp:165)
      float a1 = 0.f;
      if (row_valid && row < k && vld[h] && !skip[h]) a1 = srow[h] - fabsf(grr[h]) + fabsf(grr[h] + dadd[h]);
      float m = dmax[h];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
        a1 = fmaxf(a1, __shfl_xor_sync(kFull, a1, o));
      }
      if (lane == 0) {
        atomicMax(&sc[8 * h], __float_as_uint(m));
        atomicMax(&sc[8 * h + 4], __float_as_uint(a1));
      }
    }
    tc_fence_before();
    main_sync(NM);
    tc_fence_after();
    TC_TRACE(tid == 0, 1);

    float pivmin[NS];
    unsigned bad[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      pivmin[h] = FLT_MAX;
      bad[h] = 0u;
    }

    // ---- panels ----
    for (int pp = 0; pp < P; ++pp, ++g) {
      const int j = 16 * pp;
      const bool active = row_valid && row >= j;
      // a. lagged rhs update, panel entries
      float a[NS][16];
      auto load_a0 = [&](int h, float (&v)[16]) {
        if (row_valid) {
#pragma unroll
          for (int t4 = 0; t4 < 4; ++t4) {
            const float4 x = a0s[(h * 4 + t4) * K16 + row];
            v[4 * t4] = x.x;
            v[4 * t4 + 1] = x.y;
            v[4 * t4 + 2] = x.z;
            v[4 * t4 + 3] = x.w;
          }
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t) v[t] = 0.f;
        }
      };
      if (pp == 0) {
#pragma unroll
        for (int h = 0; h < NS; ++h) load_a0(h, a[h]);
      } else {
        // Every warp waits for its group's lookahead commit of the previous panel, also
        // once its group has no rows left: that commit follows the MMA warp's wait on the
        // group's "operands ready" barrier, so no group's arrivals can run two phases
        // ahead of that wait (a finished group otherwise arrives right after each
        // diagonal barrier, and the MMA warp, still in its second pass of the previous
        // panel, would wait for a phase that needs the next one: a deadlock).
        if (has_grp) {
          mbar_wait(&la[grp], (g - 1) & 1);
          tc_fence_after();
        }
        if (has_grp && ghi > j) {  // panel columns updated by the previous lookahead MMA
#pragma unroll
          for (int h = 0; h < NS; ++h) tmem_ld16(tq + tsys * h + (uint32_t)j, a[h]);
        } else {
#pragma unroll
          for (int h = 0; h < NS; ++h)
#pragma unroll
            for (int t = 0; t < 16; ++t) a[h][t] = 0.f;
        }
      }
      TC_TRACE(tid == 0, 2 + 4 * pp);
      // b. diagonal blocks (rows j..j+15 live in one half of one warp; the other
      //    half factors system 1's block)
      int dwarp = 0;
#pragma unroll
      for (int gg = 0; gg < kMaxGroups; ++gg)
        if (gg < Ly.G && j >= Ly.lo[gg] && j < Ly.hi[gg]) dwarp = 4 * gg + ((j - Ly.lo[gg]) >> 5);
      float dw[16], dinv = 0.f;  // (NS == 1) the diagonal warp's factored rows, for the packed store
      bool dkeep = false;
      if (warp == dwarp) {
        TC_TRACE(lane == 0 && pp < 16, 900 + 4 * pp + 1);
        const bool upper = ((j - glo) & 31) != 0;         // diagonal rows in lanes 16..31
        const bool own = (lane >= 16) == upper;           // this lane holds a diagonal row
        const int hs = own ? 0 : NS - 1;                  // system factored by this lane
        const int gr = lane & 15, drow = j + gr;
        // factor w (system hs's row drow) and publish it; `real` = a row of the block
        auto diag_emit = [&](float (&w)[16], bool real) {
          float iv = 0.f, pm = FLT_MAX;
          unsigned bd = 0u;
          bool sys_ok = false;
#pragma unroll
          for (int h = 0; h < NS; ++h)
            if (h == hs) sys_ok = !skip[h];
          diag_factor(w, iv, gr, real && drow < k && sys_ok, pm, bd);
#pragma unroll
          for (int h = 0; h < NS; ++h)
            if (h == hs) {
              pivmin[h] = fminf(pivmin[h], pm);
              bad[h] |= bd;
            }
          if (real) {
            float* LT = LTb + 272 * hs;
#pragma unroll
            for (int t = 0; t < 16; ++t) LT[t * 16 + gr] = (t <= gr) ? w[t] : 0.f;  // transposed, for the TRSM
            LT[256 + gr] = iv;
            if constexpr (NS == 1) {
              dinv = iv;  // the packed copy is stored after this panel's arrival (below)
            } else {
              bool vh = false;
#pragma unroll
              for (int h = 0; h < NS; ++h)
                if (h == hs) vh = vld[h];
              if (vh) {  // packed copy for chol_backsub_kernel
                float* L11s = L11st + (size_t)(NS * pi + hs) * P * 152 + pp * 152;
                float* Lpk = L11s + gr * (gr + 1) / 2;
                L11s[136 + gr] = iv;
#pragma unroll
                for (int t = 0; t < 16; ++t)
                  if (t <= gr) Lpk[t] = w[t];
              }
            }
          }
        };
        if constexpr (NS == 1) {
          // factor a copy: the other half-warp's rows (this panel's TRSM rows when the
          // block sits in lanes 0..15) keep their entries without a TMEM reload
#pragma unroll
          for (int t = 0; t < 16; ++t) dw[t] = a[0][t];
          diag_emit(dw, own);
          dkeep = own;
          TC_TRACE(lane == 0 && pp < 16, 900 + 4 * pp + 2);
        } else {
          float w[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const float o = __shfl_xor_sync(kFull, a[NS - 1][t], 16);
            w[t] = own ? a[0][t] : o;
          }
          diag_emit(w, true);
        }
        TC_TRACE(row == j, 3 + 4 * pp);
      }
      main_sync(NM);
      TC_TRACE(tid == 0 && pp < 16, 1100 + pp);
#ifdef FMAP_TC_TRACE
      if (lane == 0 && warp < 8 && pp < 12 && p.trace && tr_on) {  // barrier release as seen by each warp
        volatile float sink = LTb[0];
        (void)sink;
        p.trace[1400 + 8 * pp + warp] = clock64();
      }
#endif
      // c. TRSM rows >= j+16
      float l[NS][16];
      const bool trsm = active && row >= j + 16;
      if (trsm) {
#pragma unroll
        for (int h = 0; h < NS; ++h) trsm_row(LTb + 272 * h, LTb + 272 * h + 256, a[h], l[h]);
      }
      TC_TRACE(tid == 0 && pp < 16, 1120 + pp);
      TC_TRACE(lane == 0 && pp < 12 && warp < 8, 1200 + 8 * pp + warp);
      // d. store L21: operand hi/lo (the fp32 copy for the back substitution after
      //    the arrival, off the chain)
      if (trsm) {
        if (pp > 0) mbar_wait(rest, (g - 1) & 1);  // previous REST MMA done reading
        TC_TRACE(lane == 0 && pp < 12 && warp < 8, 1300 + 8 * pp + warp);
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          float* hp = opnd_hi + h * opsz + opnd_idx(row, 0);
          float* lp = opnd_lo + h * opsz + opnd_idx(row, 0);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            float hv[4], lv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) split_tf32(l[h][4 * c4 + u], hv[u], lv[u]);
            *reinterpret_cast<float4*>(hp + c4 * 32) = make_float4(hv[0], hv[1], hv[2], hv[3]);
            *reinterpret_cast<float4*>(lp + c4 * 32) = make_float4(lv[0], lv[1], lv[2], lv[3]);
          }
        }
      }
      TC_TRACE(tid == 0, 4 + 4 * pp);
      fence_async_smem();
      tc_fence_before();  // this panel's TMEM reads precede the MMA warp's copies into chunk pp
      __syncwarp();
      if (lane == 0) {
        TC_TRACE(pp < 12 && warp < 8, 700 + 8 * pp + warp);
        mbar_arrive(&ops[grp]);  // operands of this panel stored
      }
      if (trsm) {
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          if (!vld[h]) continue;
          float4* dst = reinterpret_cast<float4*>(Lst + (size_t)(NS * pi + h) * Ly.lb + lb_off(pp, K16) +
                                                  (size_t)(row - j - 16) * 16);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4)
            __stcg(dst + c4, make_float4(l[h][4 * c4], l[h][4 * c4 + 1], l[h][4 * c4 + 2], l[h][4 * c4 + 3]));
        }
      }
      if (NS == 1 && dkeep && vld[0]) {  // packed diagonal block for chol_backsub_kernel, off the chain
        const int gr = lane & 15;
        float* L11s = L11st + (size_t)pi * P * 152 + pp * 152;
        float* Lpk = L11s + gr * (gr + 1) / 2;
        L11s[136 + gr] = dinv;
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t <= gr) Lpk[t] = dw[t];
      }
      any_mma = true;
      if (has_next) {
        if (pp == P - 1) {
#pragma unroll
          for (int h = 0; h < NS; ++h) {
            if (MASK_MODE != 1 && ldn[h]) {
              mraw_n[h] = mask_entry<MASK_MODE>(p, qn[h], in_[h], row, 0.f);
            }
          }
        }
      }
    }
    pre = Ly.tma && has_next;
    TC_TRACE(tid == 0, 200);

    // ---- status words of the systems for chol_backsub_kernel ----
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      unsigned b = bad[h];
      float pm = pivmin[h];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        b |= __shfl_xor_sync(kFull, b, o);
        pm = fminf(pm, __shfl_xor_sync(kFull, pm, o));
      }
      if (lane == 0) {
        if (b) atomicOr(&sc[8 * h + 2], 1u);
        atomicMin(&sc[8 * h + 1], __float_as_uint(fmaxf(pm, 0.f)));
      }
    }
    main_sync(NM);
    if (tid < NS) {
      const int h = tid;
      bool sk = false, vv = false;
#pragma unroll
      for (int hh = 0; hh < NS; ++hh)
        if (hh == h) {
          sk = skip[hh];
          vv = vld[hh];
        }
      if (vv) {
        unsigned* ssc = stst + (size_t)(NS * pi + h) * 8;
        ssc[0] = sc[8 * h + 0];
        ssc[1] = sc[8 * h + 1];
        ssc[2] = sc[8 * h + 2];
        ssc[3] = sk ? 1u : 0u;
        ssc[4] = sc[8 * h + 4];
      }
      sc[8 * h + 0] = 0u;
      sc[8 * h + 1] = __float_as_uint(FLT_MAX);
      sc[8 * h + 2] = 0u;
      sc[8 * h + 3] = 0u;
      sc[8 * h + 4] = 0u;
      if (sk && vv) atomicOr(p.flags, 32u);
    }
    TC_TRACE(tid == 0, 203);
  }
  // ---- teardown ----
  if (any_mma) {
    mbar_wait(rest, (g - 1) & 1);
    tc_fence_after();
  }
  main_sync(NM);
  if (warp == 0) tmem_dealloc(tbase, (uint32_t)Ly.tmem_cols);
}

// ---------------------------------------------------------------------------
// Back substitution + singular verdict, one warp per system, after the
// factorization kernel (chol_tc_kernel stores every system's L21 blocks, packed
// diagonal blocks and status; this kernel reads them from HBM and forms y itself).
// Running it as its own pass instead of inside the factorization kernel keeps its
// ~8.5 K instructions per system off the SMs while the latency-bound panel chains
// run (2.27 -> 2.00 ms at cfg2 when it moved out).
// ---------------------------------------------------------------------------
constexpr int kBsWarps = 4;

// MINB = 8: 64 registers, 8 CTAs (32 warps) per SM -- the HBM-bound regime of a full
// batch; MINB = 4: 128 registers, the row loops unrolled so more of each block's
// loads are in flight -- batches of at most ~4 CTAs per SM, where one system's
// latency is the whole pass (8 pairs at k = 200: one system per warp); MINB = 6:
// 80 registers and the unrolled loops for k > 208 (longer blocks).
template <int MINB>
__global__ void __launch_bounds__(32 * kBsWarps, MINB) chol_backsub_kernel(SolveParams p, TcLayout Ly) {
  extern __shared__ __align__(1024) float smem[];
  const int k = p.k, K16 = Ly.K16, P = Ly.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t sl = (int64_t)blockIdx.x * kBsWarps + warp;
  if (sl >= p.nsys) return;
  const float* Lst = p.tc_scratch;
  const float* L11st = Lst + (size_t)p.nsys * Ly.lb;
  const unsigned* stst = reinterpret_cast<const unsigned*>(L11st + (size_t)p.nsys * P * 152);
  // Per system: L^T x = y, the backward
  // comparison solve M(L)^T w = e, the rcond verdict, the row of C.
  //
  // rcond (solver.hpp:164-168: Eigen's PartialPivLU::rcond(), a Hager/Higham
  // estimate of 1 / (||A||_1 ||A^{-1}||_1)).  For A = L L^T, |L^{-1}| <= M(L)^{-1}
  // entrywise (M = comparison matrix), so ||A^{-1}||_1 <= ||L^{-1}||_inf ||L^{-1}||_1
  // <= max(u) max(w) with u = M(L)^{-1} e (forward pass) and w = M(L)^{-T} e
  // (with the back substitution): cert = 1 / (||A||_1 max(u) max(w)) is a lower bound on
  // the true rcond, and the reference's estimate never exceeds ||A^{-1}||_1, so
  // cert >= 2 * threshold proves the reference would accept the system.  Otherwise
  // (rare: near-singular systems) the exact Hager/Higham estimator runs here on the
  // factor (forward + backward solves over the stored L), the same algorithm
  // the oracle restates (oracle/fmsolve_oracle.cpp inverse_l1_norm_estimate).
  {
    float* xv = smem + warp * 7 * K16;
    float* wv = xv + K16;
    float* uvs = wv + K16;
    float* yv = uvs + K16;  // y = L^{-1} r (forward pass)
    float* hv = yv + K16;   // Hager: working vector | sign | previous sign
    auto warp_sum = [&](float v) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      return v;
    };
    auto warp_maxf = [&](float v) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
      return v;
    };
    {
      const unsigned* ssc = stst + (size_t)sl * 8;
      if (ssc[3] == 0u && !(p.debug & 1)) {
        int64_t q;
        int i;
        sys_of(p, sl, q, i);
        const int64_t sys = q * k + i;  // global system index (error convention)
        const float* L11 = L11st + (size_t)sl * P * 152;
        const float* Lsl = Lst + (size_t)sl * Ly.lb;
        // forward pass, blocks 0..P-2: y = L^{-1} r (the right-hand side, row i of R)
        // and the comparison solve M(L) u = e of the rcond certificate
        for (int c = lane; c < K16; c += 32) {
          uvs[c] = 1.f;
          yv[c] = c < k ? (p.rhs_unit < 0 ? __ldg(p.rhs + ((size_t)q * k + i) * k + c) : (c == p.rhs_unit ? 1.f : 0.f))
                        : 0.f;
        }
        __syncwarp();
        for (int b = 0; b < P; ++b) {
          const float* Lbb = L11 + b * 152;
          {  // y_b = L_bb^{-1} acc_b and u_b = M(L_bb)^{-1} acc_b by forward substitution, lane
             // t (< 16) owns row t: v_s = acc_s / L_ss, then acc_t -= L[t][s] v_s (+= |.| for u)
            const int t = lane & 15;
            float a = uvs[16 * b + t], ay = yv[16 * b + t], res = 0.f, resy = 0.f;
#pragma unroll
            for (int sv = 0; sv < 16; ++sv) {
              const float iv = Lbb[136 + sv];
              const float us = __shfl_sync(kFull, a, sv) * iv, ys = __shfl_sync(kFull, ay, sv) * iv;
              if (t == sv) {
                res = us;
                resy = ys;
              }
              if (t > sv) {
                const float lt = Lbb[t * (t + 1) / 2 + sv];
                a = fmaf(fabsf(lt), us, a);
                ay = fmaf(-lt, ys, ay);
              }
            }
            __syncwarp();
            if (lane < 16) {
              uvs[16 * b + lane] = res;
              yv[16 * b + lane] = resy;
            }
          }
          __syncwarp();
          const int R = K16 - 16 * b - 16;
          if (R > 0) {
            const float* blk = Lsl + lb_off(b, K16);  // rows 16b+16.. of block b (L2 / HBM)
            float ub[16], yb[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              ub[t] = uvs[16 * b + t];
              yb[t] = yv[16 * b + t];
            }
            if constexpr (MINB == 8) {  // the 64-register build keeps its schedule
              for (int rho = lane; rho < R; rho += 32) {
                float acc = uvs[16 * b + 16 + rho], accy = yv[16 * b + 16 + rho];
#pragma unroll
                for (int t4 = 0; t4 < 4; ++t4) {
                  const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * t4);
                  acc = fmaf(fabsf(l4.x), ub[4 * t4], acc);
                  acc = fmaf(fabsf(l4.y), ub[4 * t4 + 1], acc);
                  acc = fmaf(fabsf(l4.z), ub[4 * t4 + 2], acc);
                  acc = fmaf(fabsf(l4.w), ub[4 * t4 + 3], acc);
                  accy = fmaf(-l4.x, yb[4 * t4], accy);
                  accy = fmaf(-l4.y, yb[4 * t4 + 1], accy);
                  accy = fmaf(-l4.z, yb[4 * t4 + 2], accy);
                  accy = fmaf(-l4.w, yb[4 * t4 + 3], accy);
                }
                uvs[16 * b + 16 + rho] = acc;
                yv[16 * b + 16 + rho] = accy;
              }
            } else {
#pragma unroll 2
              for (int rho = lane; rho < R; rho += 32) {
                float acc = uvs[16 * b + 16 + rho], accy = yv[16 * b + 16 + rho];
#pragma unroll
                for (int t4 = 0; t4 < 4; ++t4) {
                  const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * t4);
                  acc = fmaf(fabsf(l4.x), ub[4 * t4], acc);
                  acc = fmaf(fabsf(l4.y), ub[4 * t4 + 1], acc);
                  acc = fmaf(fabsf(l4.z), ub[4 * t4 + 2], acc);
                  acc = fmaf(fabsf(l4.w), ub[4 * t4 + 3], acc);
                  accy = fmaf(-l4.x, yb[4 * t4], accy);
                  accy = fmaf(-l4.y, yb[4 * t4 + 1], accy);
                  accy = fmaf(-l4.z, yb[4 * t4 + 2], accy);
                  accy = fmaf(-l4.w, yb[4 * t4 + 3], accy);
                }
                uvs[16 * b + 16 + rho] = acc;
                yv[16 * b + 16 + rho] = accy;
              }
            }
            __syncwarp();
          }
        }
        // backward pass: blocks b = P-1 .. 0 (the first ones it reads are the forward pass's last: L2)
        for (int b = P - 1; b >= 0; --b) {
          const float* Lbb = L11 + b * 152;
          // s_t = sum_{c >= 16b+16} L[c][16b+t] x_c, sw_t = sum |L[c][16b+t]| w_c
          // (lane: rows rho = lane>>2 + 8m, cols 4(lane&3)..)
          float v4[4] = {0.f, 0.f, 0.f, 0.f}, w4[4] = {0.f, 0.f, 0.f, 0.f};
          const int R = K16 - 16 * b - 16;
          if (R > 0) {
            const float* blk = Lsl + lb_off(b, K16);
            if constexpr (MINB == 8) {  // the 64-register build keeps its schedule
              for (int rho = lane >> 2; rho < R; rho += 8) {
                const float xc = xv[16 * b + 16 + rho], wcv = wv[16 * b + 16 + rho];
                const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * (lane & 3));
                v4[0] = fmaf(l4.x, xc, v4[0]);
                v4[1] = fmaf(l4.y, xc, v4[1]);
                v4[2] = fmaf(l4.z, xc, v4[2]);
                v4[3] = fmaf(l4.w, xc, v4[3]);
                w4[0] = fmaf(fabsf(l4.x), wcv, w4[0]);
                w4[1] = fmaf(fabsf(l4.y), wcv, w4[1]);
                w4[2] = fmaf(fabsf(l4.z), wcv, w4[2]);
                w4[3] = fmaf(fabsf(l4.w), wcv, w4[3]);
              }
            } else {
#pragma unroll 4
              for (int rho = lane >> 2; rho < R; rho += 8) {
                const float xc = xv[16 * b + 16 + rho], wcv = wv[16 * b + 16 + rho];
                const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * (lane & 3));
                v4[0] = fmaf(l4.x, xc, v4[0]);
                v4[1] = fmaf(l4.y, xc, v4[1]);
                v4[2] = fmaf(l4.z, xc, v4[2]);
                v4[3] = fmaf(l4.w, xc, v4[3]);
                w4[0] = fmaf(fabsf(l4.x), wcv, w4[0]);
                w4[1] = fmaf(fabsf(l4.y), wcv, w4[1]);
                w4[2] = fmaf(fabsf(l4.z), wcv, w4[2]);
                w4[3] = fmaf(fabsf(l4.w), wcv, w4[3]);
              }
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                v4[e] += __shfl_xor_sync(kFull, v4[e], o);
                w4[e] += __shfl_xor_sync(kFull, w4[e], o);
              }
          }
          // lane t (< 16): z_t = y_t - s_t, then back substitution L_bb^T x_b = z_b by rows
          // from the bottom (x_v = z_v / L_vv; z_t -= L[v][t] x_v), and the same with
          // the comparison matrix for w (zw_t = 1 + sw_t; zw_t += |L[v][t]| w_v)
          const int t = lane & 15;
          float st = 0.f, swt = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float other = __shfl_sync(kFull, v4[e], (t >> 2));  // lane (t>>2) holds cols 4(t>>2)..
            const float otherw = __shfl_sync(kFull, w4[e], (t >> 2));
            if ((t & 3) == e) {
              st = other;
              swt = otherw;
            }
          }
          float z = yv[16 * b + t] - st, zw = 1.f + swt;
          float x = 0.f, xw = 0.f;
#pragma unroll
          for (int v = 15; v >= 0; --v) {
            const float iv = Lbb[136 + v];
            const float xv_ = __shfl_sync(kFull, z, v) * iv, wv_ = __shfl_sync(kFull, zw, v) * iv;
            if (t == v) {
              x = xv_;
              xw = wv_;
            }
            if (t < v) {
              const float lt = Lbb[v * (v + 1) / 2 + t];
              z = fmaf(-lt, xv_, z);
              zw = fmaf(fabsf(lt), wv_, zw);
            }
          }
          if (lane < 16) {
            xv[16 * b + t] = x;
            wv[16 * b + t] = xw;
          }
          __syncwarp();
        }
        // row of C, certificate
        float* Crow = p.C + ((size_t)q * k + i) * k;
        bool nf = false;
        float umax = 0.f, wmax = 0.f;
        for (int c = lane; c < k; c += 32) {
          const float x = xv[c];
          nf |= !(fabsf(x) <= FLT_MAX);
          Crow[c] = x;
          umax = fmaxf(umax, uvs[c]);
          wmax = fmaxf(wmax, wv[c]);
        }
        nf = __any_sync(kFull, nf);
        umax = warp_maxf(umax);
        wmax = warp_maxf(wmax);
        const float a1 = __uint_as_float(ssc[4]);
        bool sing = ssc[2] != 0u || nf;
        float rc = 0.f;
        if (!sing) {
          const float cert = 1.f / (a1 * umax * wmax);  // 0 when the bound overflows
          if (!(a1 > 0.f)) {
            rc = 0.f;                                   // rcond_estimate_helper: ||A||_1 == 0
          } else if (k == 1) {
            rc = 1.f;
          } else if (cert >= 2.f * p.rcond_thr) {
            rc = cert;
          } else {
            // ---- second certificate: ||A^{-1}||_1 <= || |L^{-T}| |L^{-1}| ||_1 =
            // max(|L^{-T}| |L^{-1}| e) <= max(M(L)^{-T} u), never above max(u) max(w):
            // one more backward comparison pass over the stored factor (rhs u),
            // ~1.8x larger certificates, before the exact estimator's ~10 passes ----
            {
              const int t = lane & 15;
              for (int b = P - 1; b >= 0; --b) {
                const float* Lbb = L11 + b * 152;
                const int R = K16 - 16 * b - 16;
                float s4[4] = {0.f, 0.f, 0.f, 0.f};
                if (R > 0) {
                  const float* blk = Lsl + lb_off(b, K16);
                  for (int rho = lane >> 2; rho < R; rho += 8) {
                    const float wc = wv[16 * b + 16 + rho];
                    const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * (lane & 3));
                    s4[0] = fmaf(fabsf(l4.x), wc, s4[0]);
                    s4[1] = fmaf(fabsf(l4.y), wc, s4[1]);
                    s4[2] = fmaf(fabsf(l4.z), wc, s4[2]);
                    s4[3] = fmaf(fabsf(l4.w), wc, s4[3]);
                  }
#pragma unroll
                  for (int o = 4; o < 32; o <<= 1)
#pragma unroll
                    for (int e = 0; e < 4; ++e) s4[e] += __shfl_xor_sync(kFull, s4[e], o);
                }
                float st = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float other = __shfl_sync(kFull, s4[e], t >> 2);
                  if ((t & 3) == e) st = other;
                }
                float z = uvs[16 * b + t] + st, x = 0.f;
#pragma unroll
                for (int vv = 15; vv >= 0; --vv) {
                  const float xs = __shfl_sync(kFull, z, vv) * Lbb[136 + vv];
                  if (t == vv) x = xs;
                  if (t < vv) z = fmaf(fabsf(Lbb[vv * (vv + 1) / 2 + t]), xs, z);
                }
                __syncwarp();
                if (lane < 16) wv[16 * b + lane] = x;
                __syncwarp();
              }
            }
            float w2max = 0.f;
            for (int c = lane; c < k; c += 32) w2max = fmaxf(w2max, wv[c]);
            w2max = warp_maxf(w2max);
            const float cert2 = 1.f / (a1 * w2max);
            if (cert2 >= 2.f * p.rcond_thr) {
              rc = cert2;
            } else {
            // ---- exact Hager / Higham estimate of ||A^{-1}||_1 (rare path) ----
            float* v = hv;
            float* csg = hv + K16;
            float* osg = hv + 2 * K16;
            // v <- A^{-1} v  (A = L L^T): forward L z = v, backward L^T v = z
            // v <- A^{-1} v on the stored factor, with the main passes' lane-parallel
            // block scheme (16-lane shuffle chains for the diagonal blocks, lanes over
            // rows / column quads for the off-diagonal ones): a lane-0 serial version
            // cost ~1 ms per system on this path (k = 260-300 with d = 256 Grams,
            // where the certificate is inconclusive for up to ~20 % of the systems).
            auto solve_inplace = [&]() {
              const int t = lane & 15;
              for (int b = 0; b < P; ++b) {  // forward: L z = v
                const float* Lbb = L11 + b * 152;
                float a = v[16 * b + t], res = 0.f;
#pragma unroll
                for (int sv = 0; sv < 16; ++sv) {
                  const float zs = __shfl_sync(kFull, a, sv) * Lbb[136 + sv];
                  if (t == sv) res = zs;
                  if (t > sv) a = fmaf(-Lbb[t * (t + 1) / 2 + sv], zs, a);
                }
                __syncwarp();
                if (lane < 16) v[16 * b + lane] = res;
                __syncwarp();
                const int R = K16 - 16 * b - 16;
                if (R > 0) {
                  const float* blk = Lsl + lb_off(b, K16);
                  float vb[16];
#pragma unroll
                  for (int u = 0; u < 16; ++u) vb[u] = v[16 * b + u];
                  for (int rho = lane; rho < R; rho += 32) {
                    float acc = v[16 * b + 16 + rho];
#pragma unroll
                    for (int u4 = 0; u4 < 4; ++u4) {
                      const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * u4);
                      acc = fmaf(-l4.x, vb[4 * u4], acc);
                      acc = fmaf(-l4.y, vb[4 * u4 + 1], acc);
                      acc = fmaf(-l4.z, vb[4 * u4 + 2], acc);
                      acc = fmaf(-l4.w, vb[4 * u4 + 3], acc);
                    }
                    v[16 * b + 16 + rho] = acc;
                  }
                  __syncwarp();
                }
              }
              for (int b = P - 1; b >= 0; --b) {  // backward: L^T v = z
                const float* Lbb = L11 + b * 152;
                const int R = K16 - 16 * b - 16;
                float s4[4] = {0.f, 0.f, 0.f, 0.f};
                if (R > 0) {  // s_t = sum_rho L[16b+16+rho][16b+t] v_rho (lanes: rows x column quads)
                  const float* blk = Lsl + lb_off(b, K16);
                  for (int rho = lane >> 2; rho < R; rho += 8) {
                    const float vc = v[16 * b + 16 + rho];
                    const float4 l4 = *reinterpret_cast<const float4*>(blk + rho * 16 + 4 * (lane & 3));
                    s4[0] = fmaf(l4.x, vc, s4[0]);
                    s4[1] = fmaf(l4.y, vc, s4[1]);
                    s4[2] = fmaf(l4.z, vc, s4[2]);
                    s4[3] = fmaf(l4.w, vc, s4[3]);
                  }
#pragma unroll
                  for (int o = 4; o < 32; o <<= 1)
#pragma unroll
                    for (int e = 0; e < 4; ++e) s4[e] += __shfl_xor_sync(kFull, s4[e], o);
                }
                float st = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float other = __shfl_sync(kFull, s4[e], t >> 2);
                  if ((t & 3) == e) st = other;
                }
                float z = v[16 * b + t] - st, x = 0.f;
#pragma unroll
                for (int vv = 15; vv >= 0; --vv) {
                  const float xs = __shfl_sync(kFull, z, vv) * Lbb[136 + vv];
                  if (t == vv) x = xs;
                  if (t < vv) z = fmaf(-Lbb[vv * (vv + 1) / 2 + t], xs, z);
                }
                __syncwarp();
                if (lane < 16) v[16 * b + lane] = x;
                __syncwarp();
              }
              for (int c = k + lane; c < K16; c += 32) v[c] = 0.f;  // identity padding stays out
              __syncwarp();
            };
            auto l1v = [&]() {
              float sacc = 0.f;
              for (int c = lane; c < k; c += 32) sacc += fabsf(v[c]);
              return warp_sum(sacc);
            };
            const float nk = (float)k;
            for (int c = lane; c < K16; c += 32) v[c] = c < k ? 1.f / nk : 0.f;
            __syncwarp();
            solve_inplace();
            float lower = l1v(), old_lower = lower;
            int vmax = -1, old_vmax = -1;
            for (int it = 0; it < 4; ++it) {
              bool same = true;  // sign == old_sign
              for (int c = lane; c < K16; c += 32) {
                const float sg = c < k ? (v[c] < 0.f ? -1.f : 1.f) : 0.f;
                same &= (sg == osg[c]);
                csg[c] = sg;
                v[c] = sg;  // next right-hand side: the sign vector
              }
              same = __all_sync(kFull, same);
              if (it > 0 && same) break;
              __syncwarp();
              solve_inplace();  // A^T = A
              float best = -1.f;
              int bi = 0;
              for (int c = lane; c < k; c += 32)
                if (fabsf(v[c]) > best) {
                  best = fabsf(v[c]);
                  bi = c;
                }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {  // first index of the max
                const float ob = __shfl_xor_sync(kFull, best, o);
                const int oi = __shfl_xor_sync(kFull, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                  best = ob;
                  bi = oi;
                }
              }
              vmax = bi;
              if (vmax == old_vmax) break;
              for (int c = lane; c < K16; c += 32) v[c] = (c == vmax) ? 1.f : 0.f;
              __syncwarp();
              solve_inplace();
              lower = l1v();
              if (lower <= old_lower) break;
              for (int c = lane; c < K16; c += 32) osg[c] = csg[c];  // old_sign = sign
              __syncwarp();
              old_vmax = vmax;
              old_lower = lower;
            }
            for (int c = lane; c < K16; c += 32) {
              const float sgn = (c & 1) ? -1.f : 1.f;
              v[c] = c < k ? sgn * (1.f + (float)c / (float)(k - 1)) : 0.f;
            }
            __syncwarp();
            solve_inplace();
            const float alt = (2.f * l1v()) / (3.f * nk);
            if (lane == 0 && p.rcond_exact) atomicAdd(p.rcond_exact, 1u);
            const float est = fmaxf(lower, alt);
            rc = est == 0.f ? 0.f : (1.f / est) / a1;
            }
          }
          if (!(rc >= p.rcond_thr)) sing = true;
        }
        if (lane == 0) {
          if (!(rc >= 0.f)) rc = 0.f;
          if (sing) atomicMin(p.fail_min, (unsigned long long)sys);
          atomicMin(p.rcond_min_bits, __float_as_uint(rc));
        }
      }
    }
  }

}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}
// Gram batch G[q][r][c] (k x k fp32, row-major, k % 4 == 0) as the 4-D tensor
// (c % 4, r, c / 4, q); box = 4 x `rows` x 4 x 1 lands as [c/4][r][c%4], i.e. 16 B
// per row per 4-column group: the no-swizzle core-matrix layout tcgen05.cp reads
// (and the float4 [t4][row] layout of a0s).  Out-of-range rows / columns are
// zero-filled (identity padding is added later).
static int encode_gram_map(CUtensorMap* m, const float* gram, int k, int64_t npairs, int rows) {
  const EncodeTiledFn fn = encode_fn();
  if (!fn || npairs < 1) return -1;
  const cuuint64_t dims[4] = {4, (cuuint64_t)k, (cuuint64_t)(k / 4), (cuuint64_t)npairs};
  const cuuint64_t strides[3] = {(cuuint64_t)k * 4, 16, (cuuint64_t)k * k * 4};
  const cuuint32_t box[4] = {4, (cuuint32_t)rows, 4, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(gram), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : -1;
}

static int tc_ns_override() {
  const char* s = std::getenv("FMAP_TC_NS");  // diagnostics: 1 = one system per CTA
  return s ? std::atoi(s) : 0;
}

// Per-system store of the factorization for chol_backsub_kernel: L21 blocks,
// packed diagonal blocks, status (72 KB per system at k = 200, 0.94 GB for cfg2)
size_t tc_scratch_bytes(int k, int64_t nsys, int num_sms) {
  (void)num_sms;
  const TcLayout L = make_layout(k, tc_ns_override());
  return (size_t)nsys * ((size_t)L.lb + (size_t)L.P * 152 + 8) * sizeof(float);
}

bool tc_supported(int k, int optin_smem) {
  if (k < 1) return false;
  const TcLayout L = make_layout(k, tc_ns_override());
  if (L.tmem_cols > 512 || L.cps < 1 || L.threads > 384) return false;
  return (size_t)L.floats * 4 <= (size_t)optin_smem;
}

int tc_max_resolution(int optin_smem) {
  // a pure function of the device's shared-memory limit, asked on every solve:
  // computed once (the search walks ~300 layouts: ~18 us of host time per call,
  // GPU idle before the first kernel, measured with tools/step_probe.py)
  static std::atomic<int> cached_optin{-1}, cached_k{0};
  if (cached_optin.load(std::memory_order_acquire) == optin_smem) return cached_k.load(std::memory_order_relaxed);
  int k = 1;
  while (k < 4096 && tc_supported(k + 1, optin_smem)) ++k;
  cached_k.store(k, std::memory_order_relaxed);
  cached_optin.store(optin_smem, std::memory_order_release);
  return k;
}

// The f32 route: every row system goes through the tcgen05/TMEM kernel (no
// other solver, no CPU fallback); k beyond tc_max_resolution is rejected by the
// C ABI before a launch.
cudaError_t launch_chol_solve(const SolveParams& p, int mask_mode, cudaStream_t stream, int parts) {
  return launch_chol_tc(p, mask_mode, stream, parts);
}

// Host-side launcher for the tensor-core solver (p.tc_scratch must hold
// tc_scratch_bytes(k, nsys, SMs)).
cudaError_t launch_chol_tc(const SolveParams& p, int mask_mode, cudaStream_t stream, int parts) {
  if (p.nsys <= 0) return cudaSuccess;
  int dev = 0, optin = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TcLayout L = make_layout(p.k, tc_ns_override());
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
  // TMA staging of the next pair needs 16-byte row strides and a one-box panel-0 load
  L.tma = (p.k % 4 == 0 && L.K16 <= 256 && std::getenv("FMAP_TC_NOTMA") == nullptr) ? 1 : 0;
  CUtensorMap tmG, tmA;
  std::memset(&tmG, 0, sizeof(tmG));
  std::memset(&tmA, 0, sizeof(tmA));
  if (L.tma) {
    const int64_t npairs = (p.sys_offset + p.nsys + p.k - 1) / p.k;
    if (encode_gram_map(&tmG, p.gram, p.k, npairs, kTL) != 0 || encode_gram_map(&tmA, p.gram, p.k, npairs, L.K16) != 0)
      L.tma = 0;
  }
  void (*fn)(SolveParams, TcLayout, const CUtensorMap, const CUtensorMap) = nullptr;
  if (L.ns == 2) {
    if (L.threads <= 320) {
      switch (mask_mode) {
        case 0: fn = chol_tc_kernel<0, 2, 320, 1>; break;
        case 1: fn = chol_tc_kernel<1, 2, 320, 1>; break;
        default: fn = chol_tc_kernel<2, 2, 320, 1>; break;
      }
    } else {
      switch (mask_mode) {
        case 0: fn = chol_tc_kernel<0, 2, 384, 1>; break;
        case 1: fn = chol_tc_kernel<1, 2, 384, 1>; break;
        default: fn = chol_tc_kernel<2, 2, 384, 1>; break;
      }
    }
  } else if (L.cps >= 5 && L.threads > 96 && L.threads <= 128) {  // k = 65..96: 96 registers, 5 CTAs per SM
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 1, 128, 5>; break;
      case 1: fn = chol_tc_kernel<1, 1, 128, 5>; break;
      default: fn = chol_tc_kernel<2, 1, 128, 5>; break;
    }
  } else if (L.cps >= 4 && L.threads <= 160) {  // k = 97..128: 96 registers, 4 CTAs per SM
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 1, 160, 4>; break;
      case 1: fn = chol_tc_kernel<1, 1, 160, 4>; break;
      default: fn = chol_tc_kernel<2, 1, 160, 4>; break;
    }
  } else if (L.cps >= 3 && L.threads <= 192) {  // k = 129..144: 96 registers, 3 CTAs per SM
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 1, 192, 3>; break;
      case 1: fn = chol_tc_kernel<1, 1, 192, 3>; break;
      default: fn = chol_tc_kernel<2, 1, 192, 3>; break;
    }
  } else if (L.cps >= 2 && L.threads <= 256) {  // two CTAs per SM: 16 warps, up to 128 registers
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 1, 256, 2>; break;
      case 1: fn = chol_tc_kernel<1, 1, 256, 2>; break;
      default: fn = chol_tc_kernel<2, 1, 256, 2>; break;
    }
  } else {
    switch (mask_mode) {
      case 0: fn = chol_tc_kernel<0, 1, 384, 1>; break;
      case 1: fn = chol_tc_kernel<1, 1, 384, 1>; break;
      default: fn = chol_tc_kernel<2, 1, 384, 1>; break;
    }
  }
  cudaError_t e = cudaSuccess;
  if (parts & 1) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t npi = (p.nsys + L.ns - 1) / L.ns;
    // The persistent grid is what is actually resident at once: a CTA beyond the
    // registers' limit would only start when another exits, and its share of the
    // systems (static stride) would run as a second wave.
    struct OccMemo {
      const void* fn;
      size_t smem;
      int threads, occ;
    };
    thread_local OccMemo memo[8] = {};  // the query costs host time on every launch otherwise
    int occ = 0;
    for (const OccMemo& m : memo)
      if (m.fn == (const void*)fn && m.smem == smem && m.threads == L.threads) occ = m.occ;
    if (occ == 0) {  // the register file's limit (TMEM and shared memory are in L.cps)
      cudaFuncAttributes fa{};
      int rpsm = 65536;
      cudaDeviceGetAttribute(&rpsm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
      if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess && fa.numRegs > 0) {
        const int per_warp = (fa.numRegs * 32 + 255) / 256 * 256;  // allocation unit: 256 registers per warp
        occ = rpsm / (per_warp * ((L.threads + 31) / 32));
      }
      if (occ < 1) occ = 1;
      thread_local int next = 0;
      memo[next] = OccMemo{(const void*)fn, smem, L.threads, occ};
      next = (next + 1) & 7;
    }
    const int64_t maxgrid = (int64_t)sms * std::min(L.cps, occ);
    const unsigned grid = (unsigned)(npi < maxgrid ? npi : maxgrid);
    note_launch("chol_tc_kernel");
    fn<<<grid, L.threads, smem, stream>>>(p, L, tmG, tmA);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (!(parts & 2)) return cudaSuccess;
  // back substitution + verdict over the stored factors, one warp per system
  const size_t bsmem = (size_t)kBsWarps * 7 * L.K16 * sizeof(float);
  const int64_t bctas = (p.nsys + kBsWarps - 1) / kBsWarps;
  // 4: at most ~4 CTAs per SM, one system's latency is the pass (128 registers);
  // 6: k > 208, where the factor's blocks are longer (80 registers, fewer spills:
  //    4-6 % faster at k = 240-280 than 8); 8: the 64-register bandwidth build
  int minb = bctas <= 4ll * sms ? 4 : (L.K16 > 208 ? 6 : 8);
  if (const char* v = std::getenv("FMAP_BS")) minb = std::atoi(v);  // experiments: 4 / 6 / 8
  void (*bfn)(SolveParams, TcLayout) =
      minb == 4 ? chol_backsub_kernel<4> : (minb == 6 ? chol_backsub_kernel<6> : chol_backsub_kernel<8>);
  e = cudaFuncSetAttribute(bfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
  if (e != cudaSuccess) return e;
  note_launch("chol_backsub_kernel");
  bfn<<<(unsigned)bctas, 32 * kBsWarps, bsmem, stream>>>(p, L);
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
// The tensor core accumulates fp32 with a bias (its error grows linearly with the
// number of accumulated products), so every kPjChunk stages (256 vertices) the
// chunk's accumulator (TMEM columns 0..N-1) is folded by the producer warps into
// a running sum (TMEM columns 256..256+N-1) with IEEE fp32 adds.
constexpr int kPjChunk = 16;

__device__ __forceinline__ float tf32_hi(float x) {  // round-to-nearest TF32
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}

__global__ void __launch_bounds__(kPjThreads, 1) proj_tc_kernel(const float* __restrict__ phi,
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
  // full[2], empty[2], (unused), chunkdone (MMA -> producers), folded (producers -> MMA)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * sstride);
  uint64_t* chunkdone = bar + 5;
  uint64_t* folded = bar + 6;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 7);
  if (tid == 0) {
    mbar_init(&bar[0], 8);
    mbar_init(&bar[1], 8);
    mbar_init(&bar[2], 1);
    mbar_init(&bar[3], 1);
    mbar_init(&bar[4], 1);
    mbar_init(chunkdone, 1);
    mbar_init(folded, 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
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
        const int cs = st % kPjChunk;  // stage within its chunk
        if (cs == 0 && st > 0) {       // the previous chunk's accumulator has been folded
          mbar_wait(folded, ((st / kPjChunk) - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&bar[buf], (st >> 1) & 1);
        tc_fence_after();
        const uint32_t ah = su32(smem + buf * sstride), al = ah + abytes * 4;
        const uint32_t bh = al + abytes * 4, bl = bh + bbytes * 4;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = (uint32_t)ks * 256u;
          mma_tf32(tbase, sdesc(ah + ko), sdesc(bh + ko), id, (cs > 0 || ks > 0) ? 1u : 0u);
          mma_tf32(tbase, sdesc(ah + ko), sdesc(bl + ko), id, 1u);
          mma_tf32(tbase, sdesc(al + ko), sdesc(bh + ko), id, 1u);
        }
        mma_commit(&bar[2 + buf]);
        if (cs == kPjChunk - 1 || st == nst - 1) mma_commit(chunkdone);
      }
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
      if (st % kPjChunk == kPjChunk - 1 || st == nst - 1) {
        // fold this chunk (warp w: lane quarter w % 4, column half w / 4) into the sum
        const int c = st / kPjChunk;
        mbar_wait(chunkdone, c & 1);
        tc_fence_after();
        const int quarter = warp & 3, half = warp >> 2, nh = ((N / 2) + 15) & ~15;  // 16-column chunks per half
        const uint32_t tl = tbase + ((uint32_t)(32 * quarter) << 16);
        for (int c0 = half * nh; c0 < min(N, (half + 1) * nh); c0 += 16) {
          float v[16];
          tmem_ld16(tl + (uint32_t)c0, v);
          if (c > 0) {
            float sv[16];
            tmem_ld16(tl + 256u + (uint32_t)c0, sv);
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] += sv[t];
          }
          tmem_st16(tl + 256u + (uint32_t)c0, v);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(folded);
      }
    }
    // ---- epilogue: the folded sum (TMEM columns 256..) -> Out; each warp reads
    // exactly the quarter / column half it folded itself ----
    const int quarter = warp & 3, half = warp >> 2;
    const int i = i0 + 32 * quarter + lane;
    const int nh = ((N / 2) + 15) & ~15;
    for (int c0 = half * nh; c0 < min(N, (half + 1) * nh); c0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * quarter) << 16) + 256u + (uint32_t)c0, v);
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
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// Same GEMM with the inputs streamed by TMA: a kPjR-deep ring of raw fp32 tiles
// (Phi box 128 basis functions x 16 vertices, F box N channels x 16 vertices,
// Mass 16 vertices) refilled by the MMA thread as soon as the stage that used the
// slot has been converted; the 8 producer warps only convert shared memory to the
// hi/lo K-major operands (Mass applied to F).  No loads in flight in registers, so
// the per-stage cost is the conversion, not an HBM round trip.  Same MMA and
// chunk-fold scheme as proj_tc_kernel.
constexpr int kPjR = 4;

__global__ void __launch_bounds__(kPjThreads, 2)
    proj_tma_kernel(const __grid_constant__ CUtensorMap tmPhi, const __grid_constant__ CUtensorMap tmF,
                    const __grid_constant__ CUtensorMap tmMass, int64_t n, int k, int d, int N, int R,
                    uint32_t tcols, float* __restrict__ out) {
  // N = this CTA's feature columns (blockIdx.z selects the slice: N-split for
  // occupancy), R = raw-ring depth, tcols = TMEM columns (accumulator | sum at N)
  extern __shared__ __align__(1024) float smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.y, i0 = blockIdx.x * 128, c_off = blockIdx.z * N;
  const uint32_t sumoff = (uint32_t)N;
  const int abytes = 128 * kPjK, bbytes = N * kPjK;  // floats
  const int sstride = 2 * abytes + 2 * bbytes;
  const int rstride = (2048 + 16 * N + 16 + 31) & ~31;  // raw slot: Phi [16][128] | F [16][N] | Mass [16]
  float* raw = smem + 2 * sstride;
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + R * rstride);
  uint64_t* opfull = bar;          // [2] producers -> MMA
  uint64_t* opempty = bar + 2;     // [2] MMA -> producers
  uint64_t* chunkdone = bar + 5;
  uint64_t* folded = bar + 6;
  uint64_t* rawfull = bar + 7;     // [R] TMA -> producers
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 7 + kPjR);
  if (tid == 0) {
    mbar_init(&opfull[0], 8);
    mbar_init(&opfull[1], 8);
    mbar_init(&opempty[0], 1);
    mbar_init(&opempty[1], 1);
    mbar_init(chunkdone, 1);
    mbar_init(folded, 8);
    for (int r = 0; r < R; ++r) mbar_init(&rawfull[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const int nst = (int)((n + kPjK - 1) / kPjK);
  const uint32_t rawbytes = (uint32_t)(2048 + 16 * N + 16) * 4u;

  if (warp == 8) {  // ---- TMA issue + MMA issue ----
    if (lane == 0) {
      auto issue_raw = [&](int s2) {
        const int slot = s2 % R;
        float* rs = raw + slot * rstride;
        mbar_expect_tx(&rawfull[slot], rawbytes);
        tma_load_3d(rs, &tmPhi, i0, s2 * kPjK, q, &rawfull[slot]);
        tma_load_3d(rs + 2048, &tmF, c_off, s2 * kPjK, q, &rawfull[slot]);
        tma_load_2d(rs + 2048 + 16 * N, &tmMass, s2 * kPjK, q, &rawfull[slot]);
      };
      for (int s2 = 0; s2 < R && s2 < nst; ++s2) issue_raw(s2);
      const uint32_t id = idesc_tf32(N) & ~(1u << 13);  // D += A*B (no negation)
      for (int st = 0; st < nst; ++st) {
        const int buf = st & 1;
        const int cs = st % kPjChunk;
        if (cs == 0 && st > 0) {
          mbar_wait(folded, ((st / kPjChunk) - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&opfull[buf], (st >> 1) & 1);  // also: raw slot st % R has been converted
        tc_fence_after();
        if (st + R < nst) issue_raw(st + R);
        const uint32_t ah = su32(smem + buf * sstride), al = ah + abytes * 4;
        const uint32_t bh = al + abytes * 4, bl = bh + bbytes * 4;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = (uint32_t)ks * 256u;
          mma_tf32(tbase, sdesc(ah + ko), sdesc(bh + ko), id, (cs > 0 || ks > 0) ? 1u : 0u);
          mma_tf32(tbase, sdesc(ah + ko), sdesc(bl + ko), id, 1u);
          mma_tf32(tbase, sdesc(al + ko), sdesc(bh + ko), id, 1u);
        }
        mma_commit(&opempty[buf]);
        if (cs == kPjChunk - 1 || st == nst - 1) mma_commit(chunkdone);
      }
    }
  } else {  // ---- producers (256 threads): raw fp32 tiles -> hi/lo operands ----
    const int ia = tid & 127, vg = tid >> 7;  // A: basis function ia, vertices 8vg..8vg+7
    for (int st = 0; st < nst; ++st) {
      const int buf = st & 1, slot = st % R;
      mbar_wait(&rawfull[slot], (st / R) & 1);
      if (st >= 2) mbar_wait(&opempty[buf], ((st - 2) >> 1) & 1);  // MMAs of stage st-2 done
      const float* rp = raw + slot * rstride;
      const float* rf = rp + 2048;
      const float* rm = rp + 2048 + 16 * N;
      float* S = smem + buf * sstride;
#pragma unroll
      for (int h4 = 0; h4 < 2; ++h4) {
        const int v4 = 2 * vg + h4;
        float av[4], hv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = rp[(4 * v4 + u) * 128 + ia];
          hv[u] = tf32_hi(av[u]);
        }
        const int o = (ia >> 3) * 128 + v4 * 32 + (ia & 7) * 4;
        *reinterpret_cast<float4*>(S + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<float4*>(S + abytes + o) =
            make_float4(av[0] - hv[0], av[1] - hv[1], av[2] - hv[2], av[3] - hv[3]);
      }
      if (tid < N) {
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          float bv[4], hv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            bv[u] = rf[(4 * v4 + u) * N + tid] * rm[4 * v4 + u];
            hv[u] = tf32_hi(bv[u]);
          }
          const int o = (tid >> 3) * 128 + v4 * 32 + (tid & 7) * 4;
          *reinterpret_cast<float4*>(S + 2 * abytes + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<float4*>(S + 2 * abytes + bbytes + o) =
              make_float4(bv[0] - hv[0], bv[1] - hv[1], bv[2] - hv[2], bv[3] - hv[3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&opfull[buf]);
      if (st % kPjChunk == kPjChunk - 1 || st == nst - 1) {
        const int c = st / kPjChunk;
        mbar_wait(chunkdone, c & 1);
        tc_fence_after();
        const int quarter = warp & 3, half = warp >> 2, nh = ((N / 2) + 15) & ~15;  // 16-column chunks per half
        const uint32_t tl = tbase + ((uint32_t)(32 * quarter) << 16);
        for (int c0 = half * nh; c0 < min(N, (half + 1) * nh); c0 += 16) {
          float v[16];
          tmem_ld16(tl + (uint32_t)c0, v);
          if (c > 0) {
            float sv[16];
            tmem_ld16(tl + sumoff + (uint32_t)c0, sv);
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] += sv[t];
          }
          tmem_st16(tl + sumoff + (uint32_t)c0, v);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(folded);
      }
    }
    const int quarter = warp & 3, half = warp >> 2;
    const int i = i0 + 32 * quarter + lane;
    const int nh = ((N / 2) + 15) & ~15;
    for (int c0 = half * nh; c0 < min(N, (half + 1) * nh); c0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * quarter) << 16) + sumoff + (uint32_t)c0, v);
      if (i < k) {
        float* o = out + ((size_t)q * k + i) * d + c_off + c0;
        if (c_off + c0 + 16 <= d) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4)
            *reinterpret_cast<float4*>(o + 4 * c4) = make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
        } else {
#pragma unroll
          for (int t = 0; t < 16; ++t)
            if (c_off + c0 + t < d) o[t] = v[t];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, tcols);
}

// CTA-pair projection for 128 < k <= 256: the two CTAs of a cluster hold basis
// functions 0..127 / 128..255 (the A halves) and feature channels 0..N/2-1 /
// N/2..N-1 (the B halves) of one shape, and the leader issues M = 256
// tcgen05.mma.cta_group::2 -- each SM streams and converts half of F instead of
// all of it, reads half of the B operand per MMA, and no M = 128 tile is padded
// (k = 200: 72 of 128 rows in the second tile of proj_tma_kernel).  Per 16-vertex
// stage and SM: ~112 KB of shared-memory traffic instead of ~168 KB.  Same TMA
// ring, hi/lo conversion, 3xTF32 MMAs and chunk fold as proj_tma_kernel; the peer's
// producers arrive on the leader's barriers through shared::cluster addresses and
// the MMA commits are multicast to both CTAs.
constexpr int kPpB = 4;  // operand stage buffers of the pair kernel
#ifndef FMAP_PP_CHUNK
#define FMAP_PP_CHUNK 16
#endif
constexpr int kPpChunk = FMAP_PP_CHUNK;  // stages per accumulator fold (pair kernel)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPjThreads, 1)
    proj_pair_kernel(const __grid_constant__ CUtensorMap tmPhi, const __grid_constant__ CUtensorMap tmF,
                     const __grid_constant__ CUtensorMap tmMass, int64_t n, int k, int d, int N,
                     float* __restrict__ out) {
  extern __shared__ __align__(1024) float smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int q = blockIdx.y;
  const int i0 = (int)rank * 128;           // this CTA's basis functions (A half)
  const int Nh = N / 2, c_off = (int)rank * Nh;  // this CTA's feature channels (B half)
  const int abytes = 128 * kPjK, bbytes = Nh * kPjK;  // floats
  const int sstride = 2 * abytes + 2 * bbytes;
  const int rstride = (2048 + 16 * Nh + 16 + 31) & ~31;  // raw slot: Phi [16][128] | F [16][Nh] | Mass [16]
  float* raw = smem + kPpB * sstride;
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + kPjR * rstride);
  uint64_t* opfull = bar;                 // [B] (leader) producer warps of both CTAs -> MMA
  uint64_t* opempty = bar + kPpB;         // [B] MMA commit (multicast) -> producers
  uint64_t* conv = bar + 2 * kPpB;        // [B] this CTA's producers -> this CTA's TMA refill
  uint64_t* chunkdone = bar + 3 * kPpB;   // MMA commit (multicast) -> producers
  uint64_t* folded = chunkdone + 1;       // (leader) producer warps of both CTAs -> MMA
  uint64_t* rawfull = chunkdone + 2;      // [R] TMA -> producers
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rawfull + kPjR);
  if (tid == 0) {
    for (int u = 0; u < kPpB; ++u) {
      mbar_init(&opfull[u], 16);
      mbar_init(&opempty[u], 1);
      mbar_init(&conv[u], 8);
    }
    mbar_init(chunkdone, 1);
    mbar_init(folded, 16);
    for (int r = 0; r < kPjR; ++r) mbar_init(&rawfull[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc2(tslot, 512u);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t sumoff = (uint32_t)N;
  const int nst = (int)((n + kPjK - 1) / kPjK);
  const uint32_t rawbytes = (uint32_t)(2048 + 16 * Nh + 16) * 4u;

  if (warp == 8) {  // ---- TMA issue (both CTAs) + MMA issue (leader) ----
    if (lane == 0) {
      auto issue_raw = [&](int s2) {
        const int slot = s2 % kPjR;
        float* rs = raw + slot * rstride;
        mbar_expect_tx(&rawfull[slot], rawbytes);
        tma_load_3d(rs, &tmPhi, i0, s2 * kPjK, q, &rawfull[slot]);
        tma_load_3d(rs + 2048, &tmF, c_off, s2 * kPjK, q, &rawfull[slot]);
        tma_load_2d(rs + 2048 + 16 * Nh, &tmMass, s2 * kPjK, q, &rawfull[slot]);
      };
      for (int s2 = 0; s2 < kPjR && s2 < nst; ++s2) issue_raw(s2);
      if (rank == 0) {
        // D f32, A/B tf32 K-major, D += A*B, N, M = 256
        const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (16u << 24);
        for (int st = 0; st < nst; ++st) {
          const int buf = st % kPpB;
          const int cs = st % kPpChunk;
          if (cs == 0 && st > 0) {
            mbar_wait(folded, ((st / kPpChunk) - 1) & 1);
            tc_fence_after();
          }
          mbar_wait(&opfull[buf], (st / kPpB) & 1);  // both CTAs converted stage st
          tc_fence_after();
          if (st + kPjR < nst) issue_raw(st + kPjR);
          const uint32_t ah = su32(smem + buf * sstride), al = ah + abytes * 4;
          const uint32_t bh = al + abytes * 4, bl = bh + bbytes * 4;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t ko = (uint32_t)ks * 256u;
            mma_tf32_2sm(tbase, sdesc(ah + ko), sdesc(bh + ko), id, (cs > 0 || ks > 0) ? 1u : 0u);
            mma_tf32_2sm(tbase, sdesc(ah + ko), sdesc(bl + ko), id, 1u);
            mma_tf32_2sm(tbase, sdesc(al + ko), sdesc(bh + ko), id, 1u);
          }
          mma_commit_pair(&opempty[buf]);
          if (cs == kPpChunk - 1 || st == nst - 1) mma_commit_pair(chunkdone);
        }
      } else {
        for (int st = 0; st < nst; ++st) {
          mbar_wait(&conv[st % kPpB], (st / kPpB) & 1);  // this CTA converted stage st: slot st % R free
          if (st + kPjR < nst) issue_raw(st + kPjR);
        }
      }
    }
  } else {  // ---- producers (256 threads): raw fp32 tiles -> hi/lo operands ----
    const int ia = tid & 127, vg = tid >> 7;  // row ia (basis function / channel), vertices 8vg..8vg+7
    const uint32_t opfull0 = mapa_rank(su32(opfull), 0);  // + 8 bytes per buffer
    const uint32_t folded0 = mapa_rank(su32(folded), 0);
    for (int st = 0; st < nst; ++st) {
      const int buf = st % kPpB, slot = st % kPjR;
      mbar_wait(&rawfull[slot], (st / kPjR) & 1);
      if (st >= kPpB) mbar_wait(&opempty[buf], ((st - kPpB) / kPpB) & 1);  // MMAs of stage st-B done
      const float* rp = raw + slot * rstride;
      const float* rf = rp + 2048;
      const float* rm = rp + 2048 + 16 * Nh;
      float* S = smem + buf * sstride;
#pragma unroll
      for (int h4 = 0; h4 < 2; ++h4) {
        const int v4 = 2 * vg + h4;
        const int o = (ia >> 3) * 128 + v4 * 32 + (ia & 7) * 4;
        float av[4], hv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = rp[(4 * v4 + u) * 128 + ia];
          hv[u] = tf32_hi(av[u]);
        }
        *reinterpret_cast<float4*>(S + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<float4*>(S + abytes + o) =
            make_float4(av[0] - hv[0], av[1] - hv[1], av[2] - hv[2], av[3] - hv[3]);
        if (ia < Nh) {
          float bv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            bv[u] = rf[(4 * v4 + u) * Nh + ia] * rm[4 * v4 + u];
            hv[u] = tf32_hi(bv[u]);
          }
          *reinterpret_cast<float4*>(S + 2 * abytes + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<float4*>(S + 2 * abytes + bbytes + o) =
              make_float4(bv[0] - hv[0], bv[1] - hv[1], bv[2] - hv[2], bv[3] - hv[3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&conv[buf]);
        mbar_arrive_cluster(opfull0 + 8u * (uint32_t)buf);
      }
      if (st % kPpChunk == kPpChunk - 1 || st == nst - 1) {
        const int c = st / kPpChunk;
        mbar_wait(chunkdone, c & 1);
        tc_fence_after();
        const int quarter = warp & 3, half = warp >> 2, nh = ((N / 2) + 15) & ~15;
        const uint32_t tl = tbase + ((uint32_t)(32 * quarter) << 16);
        for (int c0 = half * nh; c0 < min(N, (half + 1) * nh); c0 += 16) {
          float v[16];
          tmem_ld16(tl + (uint32_t)c0, v);
          if (c > 0) {
            float sv[16];
            tmem_ld16(tl + sumoff + (uint32_t)c0, sv);
#pragma unroll
            for (int t = 0; t < 16; ++t) v[t] += sv[t];
          }
          tmem_st16(tl + sumoff + (uint32_t)c0, v);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(folded0);
      }
    }
    const int quarter = warp & 3, half = warp >> 2;
    const int i = i0 + 32 * quarter + lane;
    const int nh = ((N / 2) + 15) & ~15;
    for (int c0 = half * nh; c0 < min(N, (half + 1) * nh); c0 += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(32 * quarter) << 16) + sumoff + (uint32_t)c0, v);
      if (i < k) {
        float* o = out + ((size_t)q * k + i) * d + c0;
        if (c0 + 16 <= d) {
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
  cluster_sync_all();  // the peer is done with this CTA's barriers and TMEM
  tc_fence_after();
  if (warp == 0) tmem_dealloc2(tbase, 512u);
}
}  // namespace

// Tensor-core projection (d <= 256); returns cudaErrorNotSupported otherwise.
// Row-major fp32 tensor [dim2][dim1][dim0] as a TMA map with box {b0, b1, 1}
// (rank 3) or [dim1][dim0] with box {b0, 1} (rank 2).
static int encode_plain_map(CUtensorMap* m, const float* base, int rank, const cuuint64_t* dims, const cuuint32_t* box) {
  const EncodeTiledFn fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t strides[2] = {dims[0] * 4, rank == 3 ? dims[0] * dims[1] * 4 : 0};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? 0
             : -1;
}

cudaError_t launch_project_tc(const float* phi, const float* mass, const float* F, int64_t b,
                              int64_t n, int k, int d, float* out, cudaStream_t st) {
  if (d > 256 || d < 1 || k < 1 || n < 1 || b < 1) return cudaErrorNotSupported;
  const int N = (d + 15) & ~15;
  // TMA-streamed kernel when every row stride is 16-byte aligned
  const char* pair_env = std::getenv("FMAP_PROJ_PAIR");  // "0": the one-CTA kernel below instead
  if (k > 128 && k <= 256 && k % 4 == 0 && d % 4 == 0 && n % 4 == 0 && !(pair_env && pair_env[0] == '0') &&
      !std::getenv("FMAP_PROJ_NOTMA")) {
    // CTA-pair kernel: N a multiple of 32 (each CTA's half of the channels is a
    // multiple of 16), TMA boxes of 128 basis functions / N/2 channels / 16 vertices
    const int Np = (d + 31) & ~31;
    CUtensorMap tp, tf, tm;
    const cuuint64_t dp[3] = {(cuuint64_t)k, (cuuint64_t)n, (cuuint64_t)b};
    const cuuint32_t bp[3] = {128, (cuuint32_t)kPjK, 1};
    const cuuint64_t df[3] = {(cuuint64_t)d, (cuuint64_t)n, (cuuint64_t)b};
    const cuuint32_t bf[3] = {(cuuint32_t)(Np / 2), (cuuint32_t)kPjK, 1};
    const cuuint64_t dm[2] = {(cuuint64_t)n, (cuuint64_t)b};
    const cuuint32_t bm[2] = {(cuuint32_t)kPjK, 1};
    if (b <= 65535 && encode_plain_map(&tp, phi, 3, dp, bp) == 0 && encode_plain_map(&tf, F, 3, df, bf) == 0 &&
        encode_plain_map(&tm, mass, 2, dm, bm) == 0) {
      const int Nh = Np / 2;
      const int rstride = (2048 + 16 * Nh + 16 + 31) & ~31;
      const size_t smem = (size_t)(kPpB * (2 * 128 * kPjK + 2 * Nh * kPjK) + kPjR * rstride) * 4 + 256;
      cudaError_t e = cudaFuncSetAttribute(proj_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      note_launch("proj_pair_kernel");
      proj_pair_kernel<<<dim3(2, (unsigned)b), kPjThreads, smem, st>>>(tp, tf, tm, n, k, d, Np, out);
      return cudaGetLastError();
    }
  }
  if (k % 4 == 0 && d % 4 == 0 && n % 4 == 0 && !std::getenv("FMAP_PROJ_NOTMA")) {
    CUtensorMap tp, tf, tm;
    const cuuint64_t dp[3] = {(cuuint64_t)k, (cuuint64_t)n, (cuuint64_t)b};
    const cuuint32_t bp[3] = {128, (cuuint32_t)kPjK, 1};
    // N-split: two CTAs per (pair, 128 basis functions) of N/2 feature columns
    // each -- 256 columns of TMEM (accumulator + fp32 sum) and a 2-deep raw ring,
    // so two CTAs share an SM and one's chunk fold hides behind the other's MMAs
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ctas = b * ((k + 127) / 128);
    // opt-in (FMAP_PROJ_SPLIT=1): measured slower at cfg2 (0.363 vs 0.258 ms per
    // direction: the 2-deep ring and the duplicated Phi conversion cost more than
    // the second CTA per SM hides)
    const int nsplit = (N > 128 && 2 * ctas <= 2LL * sms && std::getenv("FMAP_PROJ_SPLIT") != nullptr) ? 2 : 1;
    const int Nc = nsplit == 2 ? ((N / 2 + 15) & ~15) : N;
    const int R = nsplit == 2 ? 2 : kPjR;
    const uint32_t tcols = 2 * Nc <= 256 ? 256u : 512u;
    const cuuint64_t df[3] = {(cuuint64_t)d, (cuuint64_t)n, (cuuint64_t)b};
    const cuuint32_t bf[3] = {(cuuint32_t)Nc, (cuuint32_t)kPjK, 1};
    const cuuint64_t dm[2] = {(cuuint64_t)n, (cuuint64_t)b};
    const cuuint32_t bm[2] = {(cuuint32_t)kPjK, 1};
    if (encode_plain_map(&tp, phi, 3, dp, bp) == 0 && encode_plain_map(&tf, F, 3, df, bf) == 0 &&
        encode_plain_map(&tm, mass, 2, dm, bm) == 0) {
      const int rstride = (2048 + 16 * Nc + 16 + 31) & ~31;
      const size_t smem = (size_t)(2 * (2 * 128 * kPjK + 2 * Nc * kPjK) + R * rstride) * 4 + 256;
      cudaError_t e = cudaFuncSetAttribute(proj_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      dim3 grid((unsigned)((k + 127) / 128), (unsigned)b, (unsigned)nsplit);
      note_launch("proj_tma_kernel");
      proj_tma_kernel<<<grid, kPjThreads, smem, st>>>(tp, tf, tm, n, k, d, Nc, R, tcols, out);
      return cudaGetLastError();
    }
  }
  const size_t smem = (size_t)(2 * (2 * 128 * kPjK + 2 * N * kPjK)) * 4 + 64;
  const size_t req = smem < 233472 / 2 + 1 ? 233472 / 2 + 1 : smem;  // 1 CTA per SM (TMEM 512 cols)
  cudaError_t e = cudaFuncSetAttribute(proj_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)req);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((k + 127) / 128), (unsigned)b);
  note_launch("proj_tc_kernel");
  proj_tc_kernel<<<grid, kPjThreads, req, st>>>(phi, mass, F, n, k, d, N, out);
  return cudaGetLastError();
}

}  // namespace fmap
