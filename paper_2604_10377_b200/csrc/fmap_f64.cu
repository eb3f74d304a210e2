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
// Verdict as the f32 route: non-positive / non-finite pivot, the reference's rcond
// test (comparison-matrix certificate, else the exact Hager/Higham estimate on
// the factor) or a non-finite solution; lowest failing global system index wins.
// k up to the f32 route's limit and beyond: rows that do not fit the 227 KB of
// shared memory (k > 234) spill to an L2-resident global scratch.
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
__host__ __device__ __forceinline__ int off(int r) { return r * (r + 1) / 2 + (r + 1) / 2; }
__host__ __device__ inline size_t packed_doubles(int k) { return (size_t)k * (k + 1) / 2 + (k + 1) / 2; }

struct F64Args {
  const double* G;
  const double* R;
  const double* M;
  double* C;
  int k;
  int64_t nsys;
  double lambda, ridge, rthr;
  int rhs_unit;
  unsigned long long* fail_min;
  unsigned* rcond_min_bits;
  unsigned* rcond_exact;
  double* spill;         // rows [0, S) of every CTA's packed triangle in global memory (L2-resident)
  int S;
  size_t spill_stride;   // doubles per CTA
};

// Vectors after the packed rows in shared memory (doubles): y, yy, xs, invd, un, uu, ws, hv[3k]
__host__ __device__ inline size_t f64_vec_doubles(int k) { return (size_t)((k + 3) & ~1) + 9 * (size_t)k; }

template <bool SPILL>
__global__ void __launch_bounds__(kT64, 1) chol_f64_kernel(const F64Args p) {
  extern __shared__ __align__(16) double sm64[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kT64 / 32;
  constexpr int NB = 8;  // panel width
  const int k = p.k;
  const int S = SPILL ? p.S : 0;
  const size_t sm_rows = packed_doubles(k) - (size_t)off(S);
  double* A = sm64;                                    // rows S..k-1 of the padded packed triangle
  double* gA = SPILL ? p.spill + (size_t)blockIdx.x * p.spill_stride : nullptr;
  double* y = A + ((sm_rows + 1) & ~(size_t)1);         // right-hand side -> y = L^{-1} r
  double* yy = y + ((k + 3) & ~1);                     // final forward values
  double* xs = yy + k;                                 // back substitution work vector
  double* invd = xs + k;                               // 1 / L_jj
  double* un = invd + k;                               // comparison forward solve M(L) u = e (running)
  double* uu = un + k;                                 //   final u
  double* ws = uu + k;                                 // comparison backward solve M(L)^T w = e
  double* hv = ws + k;                                 // Hager: v | sign | previous sign
  __shared__ double red[NW];
  __shared__ int redi[NW];
  __shared__ double s_piv, s_a1, s_bc;
  __shared__ int sbad, s_path, s_bci;
  // row r of the packed lower triangle (rows < S live in global memory for k > 234)
  auto rp = [&](int r) -> double* {
    if constexpr (SPILL) return r < S ? gA + off(r) : A + (off(r) - off(S));
    return A + off(r);
  };
  // block-wide sum / max / first-argmax of per-thread values (all threads call)
  auto block_sum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < NW; ++w) t += red[w];
      s_bc = t;
    }
    __syncthreads();
    return s_bc;
  };
  auto block_max = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = red[0];
      for (int w = 1; w < NW; ++w) t = fmax(t, red[w]);
      s_bc = t;
    }
    __syncthreads();
    return s_bc;
  };

  for (int64_t sys = blockIdx.x; sys < p.nsys; sys += gridDim.x) {
    const int64_t q = sys / k;
    const int i = (int)(sys - q * k);
    const double* Gq = p.G + (size_t)q * k * k;
    const double* Mi = p.M + ((size_t)q * k + i) * k;
    // ---- staging (+ row 1-norms of the assembled system for ||A||_1) ----
    double a1m = 0.0;
    for (int r = warp; r < k; r += NW) {
      double* Ar = rp(r);
      double srow = 0.0;
      for (int c = lane; c < k; c += 32) {
        const double g = Gq[(size_t)r * k + c];
        if (c <= r) Ar[c] = g;
        srow += fabs(g);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) srow += __shfl_xor_sync(0xffffffffu, srow, o);
      if (lane == 0) {
        const double grr = Gq[(size_t)r * k + r];
        a1m = fmax(a1m, srow - fabs(grr) + fabs(grr + p.lambda * Mi[r] + p.ridge));
      }
    }
    __syncthreads();
    double dm = 0.0;
    for (int r = tid; r < k; r += kT64) {
      double* Ar = rp(r);
      const double d = Ar[r] + p.lambda * Mi[r] + p.ridge;
      Ar[r] = d;
      dm = fmax(dm, fabs(d));
      y[r] = p.rhs_unit < 0 ? p.R[((size_t)q * k + i) * k + r] : (r == p.rhs_unit ? 1.0 : 0.0);
      un[r] = 1.0;
      ws[r] = 1.0;
    }
    const double a1 = block_max(a1m);
    const double dmax = block_max(dm);
    (void)dmax;
    double pivmin = DBL_MAX;  // lane-local in warp 0 (diagonal pivots), reduced at the end
    bool bad = false;

    // ---- blocked factorization (8-column panels) + forward substitution ----
    // (1) warp 0: 8x8 diagonal block at j0, lane u = row j0+u (lower part only),
    //     and the panel's forward-substitution values (y, and u of the
    //     comparison solve).  For j0 > 0 it runs inside the previous panel's
    //     trailing update, right after warp 0 has updated that block (tile (0,0)
    //     of the update), hidden behind the other warps' tiles.
    auto diag_block = [&](int j0) {
      const int nb = min(NB, k - j0);
      const int u = lane;
      double a[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) a[t] = (u < nb && t <= u) ? rp(j0 + u)[j0 + t] : 0.0;
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
      // panel forward substitution: yb = L11^{-1} y[j0 .. j0+nb), ub = M(L11)^{-1} un[..]
      double yb = (u < nb) ? y[j0 + u] : 0.0, ub = (u < nb) ? un[j0 + u] : 0.0;
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        if (t < nb) {
          const double yt = __shfl_sync(0xffffffffu, yb * inv_u, t);
          const double ut = __shfl_sync(0xffffffffu, ub * inv_u, t);
          if (u > t) {
            yb = fma(-a[t], yt, yb);
            ub = fma(fabs(a[t]), ut, ub);
          }
          if (u == t) {
            yb = yt;
            ub = ut;
          }
        }
      }
      if (u < nb) {
        double* Ar = rp(j0 + u);
#pragma unroll
        for (int t = 0; t < NB; ++t)
          if (t <= u) Ar[j0 + t] = a[t];
        invd[j0 + u] = inv_u;
        yy[j0 + u] = yb;
        uu[j0 + u] = ub;
      }
    };
    if (warp == 0) diag_block(0);
    __syncthreads();
    for (int j0 = 0; j0 < k; j0 += NB) {
      const int nb = min(NB, k - j0);
      // (2) rows below the block: L21 row (TRSM against L11), y and u updates
      const int nrest = k - j0 - nb;
      for (int rr = tid; rr < nrest; rr += kT64) {
        const int r = j0 + nb + rr;
        double* Ar = rp(r) + j0;
        double l[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          if (t < nb) {
            double v = Ar[t];
            const double* L11t = rp(j0 + t) + j0;
#pragma unroll
            for (int s2 = 0; s2 < t; ++s2) v = fma(-l[s2], L11t[s2], v);
            l[t] = v * invd[j0 + t];
          } else {
            l[t] = 0.0;
          }
        }
        double yr = y[r], ur = un[r];
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          if (t < nb) {
            Ar[t] = l[t];
            yr = fma(-l[t], yy[j0 + t], yr);
            ur = fma(fabs(l[t]), uu[j0 + t], ur);
          }
        }
        y[r] = yr;
        un[r] = ur;
      }
      __syncthreads();
      // (3) trailing rank-8 update of rows / columns >= j0+8 on the FP64 tensor
      //     path (DMMA, mma.sync m8n8k4 f64): 8x8 tiles of the lower trailing
      //     triangle, K = the panel's 8 columns in two k=4 steps.  Row r's panel
      //     entries are contiguous (rp(r)[j0 ...]); A fragment = -L rows, B
      //     fragment = L rows of the tile's columns, C/D = the trailing block
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
            double a0 = 0.0, a1v = 0.0, b0 = 0.0, b1 = 0.0;
            if (ra < k) {
              const double* Ra = rp(ra) + j0;
              a0 = -Ra[q4];
              a1v = -Ra[4 + q4];
            }
            if (rb < k) {
              const double* Rb = rp(rb) + j0;
              b0 = Rb[q4];
              b1 = Rb[4 + q4];
            }
            const int cr = r0 + g, cc = c0 + 2 * q4;
            const bool st = cr < k && cc <= cr;
            double2 cv = make_double2(0.0, 0.0);
            double* Cp = st ? rp(cr) + cc : nullptr;
            if (st) cv = *reinterpret_cast<const double2*>(Cp);
            double d0, d1;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                         : "=d"(d0), "=d"(d1)
                         : "d"(a0), "d"(b0), "d"(cv.x), "d"(cv.y));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
                         : "=d"(d0), "=d"(d1)
                         : "d"(a1v), "d"(b1), "d"(d0), "d"(d1));
            if (st) *reinterpret_cast<double2*>(Cp) = make_double2(d0, d1);
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
    // ---- back substitution L^T x = y (and M(L)^T w = e) in 8-row blocks from the
    //      bottom: warp 0 solves the block's 8x8 transposed triangle (shuffles),
    //      then every thread removes the block's contribution from the rows above
    //      it (row c of L is contiguous, so rp(c)[r] is coalesced over r) ----
    for (int r = tid; r < k; r += kT64) xs[r] = yy[r];
    __syncthreads();
    double* Crow = p.rhs_unit < 0 ? p.C + ((size_t)q * k + i) * k : p.C;
    bool nf = false;
    for (int c0 = ((k - 1) / NB) * NB; c0 >= 0; c0 -= NB) {
      const int nbb = min(NB, k - c0);
      if (warp == 0) {
        double v = lane < nbb ? xs[c0 + lane] : 0.0, wv = lane < nbb ? ws[c0 + lane] : 0.0;
#pragma unroll
        for (int t = NB - 1; t >= 0; --t) {
          if (t < nbb) {
            const double xt = __shfl_sync(0xffffffffu, v, t) * invd[c0 + t];
            const double wt = __shfl_sync(0xffffffffu, wv, t) * invd[c0 + t];
            if (lane < t) {
              const double lt = rp(c0 + t)[c0 + lane];
              v = fma(-lt, xt, v);
              wv = fma(fabs(lt), wt, wv);
            }
            if (lane == t) {
              v = xt;
              wv = wt;
            }
          }
        }
        if (lane < nbb) {
          xs[c0 + lane] = v;
          ws[c0 + lane] = wv;
          Crow[c0 + lane] = v;
        }
        nf |= __any_sync(0xffffffffu, lane < nbb && !(fabs(v) <= DBL_MAX));
      }
      __syncthreads();
      for (int r = tid; r < c0; r += kT64) {
        double acc = xs[r], accw = ws[r];
#pragma unroll
        for (int t = 0; t < NB; ++t)
          if (t < nbb) {
            const double lt = rp(c0 + t)[r];
            acc = fma(-lt, xs[c0 + t], acc);
            accw = fma(fabs(lt), ws[c0 + t], accw);
          }
        xs[r] = acc;
        ws[r] = accw;
      }
      __syncthreads();
    }
    // ---- rcond (solver.hpp:164-168, as the f32 route): comparison-matrix
    //      certificate 1 / (||A||_1 max(u) max(w)) <= rcond; when it does not
    //      prove rcond >= 2 * threshold, the exact Hager/Higham estimate ----
    double um = 0.0, wm = 0.0;
    for (int r = tid; r < k; r += kT64) {
      um = fmax(um, uu[r]);
      wm = fmax(wm, ws[r]);
    }
    const double umax = block_max(um), wmax = block_max(wm);
    if (warp == 0) nf = __any_sync(0xffffffffu, nf);
    if (tid == 0) {
      s_a1 = a1;
      const bool sing0 = sbad || nf;
      const double cert = 1.0 / (a1 * umax * wmax);
      s_path = sing0 ? 0 : (!(a1 > 0.0) ? 1 : (k == 1 ? 2 : (cert >= 2.0 * p.rthr ? 3 : 4)));
      s_piv = cert;  // reuse: the certificate
    }
    __syncthreads();
    double rc = 0.0;
    const int path = s_path;
    if (path == 2) rc = 1.0;
    if (path == 3) rc = s_piv;
    if (path == 4) {
      double* v = hv;
      double* csg = hv + k;
      double* osg = hv + 2 * k;
      // v <- A^{-1} v with A = L L^T (forward then backward block substitution)
      auto solve_full = [&]() {
        for (int j0 = 0; j0 < k; j0 += NB) {
          const int nb = min(NB, k - j0);
          if (warp == 0) {
            double vb = lane < nb ? v[j0 + lane] : 0.0;
#pragma unroll
            for (int t = 0; t < NB; ++t) {
              if (t < nb) {
                const double zt = __shfl_sync(0xffffffffu, vb, t) * invd[j0 + t];
                if (lane > t && lane < nb) vb = fma(-rp(j0 + lane)[j0 + t], zt, vb);
                if (lane == t) vb = zt;
              }
            }
            if (lane < nb) v[j0 + lane] = vb;
          }
          __syncthreads();
          for (int r = j0 + nb + tid; r < k; r += kT64) {
            const double* Rr = rp(r) + j0;
            double acc = v[r];
#pragma unroll
            for (int t = 0; t < NB; ++t)
              if (t < nb) acc = fma(-Rr[t], v[j0 + t], acc);
            v[r] = acc;
          }
          __syncthreads();
        }
        for (int c0 = ((k - 1) / NB) * NB; c0 >= 0; c0 -= NB) {
          const int nbb = min(NB, k - c0);
          if (warp == 0) {
            double vv = lane < nbb ? v[c0 + lane] : 0.0;
#pragma unroll
            for (int t = NB - 1; t >= 0; --t) {
              if (t < nbb) {
                const double xt = __shfl_sync(0xffffffffu, vv, t) * invd[c0 + t];
                if (lane < t) vv = fma(-rp(c0 + t)[c0 + lane], xt, vv);
                if (lane == t) vv = xt;
              }
            }
            if (lane < nbb) v[c0 + lane] = vv;
          }
          __syncthreads();
          for (int r = tid; r < c0; r += kT64) {
            double acc = v[r];
#pragma unroll
            for (int t = 0; t < NB; ++t)
              if (t < nbb) acc = fma(-rp(c0 + t)[r], v[c0 + t], acc);
            v[r] = acc;
          }
          __syncthreads();
        }
      };
      auto l1v = [&]() {
        double acc = 0.0;
        for (int r = tid; r < k; r += kT64) acc += fabs(v[r]);
        return block_sum(acc);
      };
      const double nk = (double)k;
      for (int r = tid; r < k; r += kT64) v[r] = 1.0 / nk;
      __syncthreads();
      solve_full();
      double lower = l1v(), old_lower = lower;
      int old_vmax = -1;
      for (int it = 0; it < 4; ++it) {
        int diff = 0;
        for (int r = tid; r < k; r += kT64) {
          const double sg = v[r] < 0.0 ? -1.0 : 1.0;
          diff |= sg != osg[r];
          csg[r] = sg;
          v[r] = sg;
        }
        diff = __syncthreads_or(diff);
        if (it > 0 && !diff) break;
        solve_full();  // A^T = A
        // first index of max |v|
        double best = -1.0;
        int bi = 0;
        for (int r = tid; r < k; r += kT64)
          if (fabs(v[r]) > best) {
            best = fabs(v[r]);
            bi = r;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        __syncthreads();
        if (lane == 0) {
          red[warp] = best;
          redi[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
          double bb = red[0];
          int ii = redi[0];
          for (int w = 1; w < NW; ++w)
            if (red[w] > bb || (red[w] == bb && redi[w] < ii)) {
              bb = red[w];
              ii = redi[w];
            }
          s_bci = ii;
        }
        __syncthreads();
        const int vmax = s_bci;
        if (vmax == old_vmax) break;
        for (int r = tid; r < k; r += kT64) v[r] = r == vmax ? 1.0 : 0.0;
        __syncthreads();
        solve_full();
        lower = l1v();
        if (lower <= old_lower) break;
        for (int r = tid; r < k; r += kT64) osg[r] = csg[r];  // old_sign = sign
        __syncthreads();
        old_vmax = vmax;
        old_lower = lower;
      }
      for (int r = tid; r < k; r += kT64) {
        const double sgn = (r & 1) ? -1.0 : 1.0;
        v[r] = sgn * (1.0 + (double)r / (double)(k - 1));
      }
      __syncthreads();
      solve_full();
      const double alt = (2.0 * l1v()) / (3.0 * nk);
      const double est = fmax(lower, alt);
      rc = est == 0.0 ? 0.0 : (1.0 / est) / s_a1;
      if (tid == 0 && p.rcond_exact) atomicAdd(p.rcond_exact, 1u);
    }
    if (tid == 0) {
      if (!(rc >= 0.0)) rc = 0.0;
      if (path == 0 || !(rc >= p.rthr)) atomicMin(p.fail_min, (unsigned long long)sys);
      atomicMin(p.rcond_min_bits, __float_as_uint((float)rc));
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

// Rows S..k-1 of the packed triangle + vectors in shared memory; rows 0..S-1
// (the short ones, finished first) spill to an L2-resident global scratch when
// the whole triangle does not fit (k > 234 on B200).
static int f64_spill_rows(int k, size_t optin) {
  optin -= 1024;  // the kernel's static shared memory (reductions, flags)
  int S = 0;
  while (S < k && ((((packed_doubles(k) - (size_t)off(S)) + 1) & ~(size_t)1) + f64_vec_doubles(k)) * 8 > optin) ++S;
  return S;
}

size_t chol_f64_smem_bytes(int k, size_t optin) {
  const int S = f64_spill_rows(k, optin);  // dynamic shared memory of the launch
  return ((((packed_doubles(k) - (size_t)off(S)) + 1) & ~(size_t)1) + f64_vec_doubles(k)) * sizeof(double);
}

size_t chol_f64_spill_doubles(int k, size_t optin, int num_sms) {
  const int S = f64_spill_rows(k, optin);
  return S > 0 ? ((size_t)off(S) + 2) * (size_t)num_sms : 0;
}

cudaError_t launch_chol_f64(const double* G, const double* R, const double* M, double* C, int k, int64_t nsys,
                            double lambda, double ridge, double rthr, int rhs_unit, unsigned long long* fail_min,
                            unsigned* rcond_min_bits, unsigned* rcond_exact, double* spill, cudaStream_t st) {
  if (nsys <= 0) return cudaSuccess;
  int dev = 0, optin = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int S = f64_spill_rows(k, (size_t)optin);
  const size_t smem = chol_f64_smem_bytes(k, (size_t)optin);
  if (smem > (size_t)optin || (S > 0 && !spill)) return cudaErrorNotSupported;
  F64Args a{G, R, M, C, k, nsys, lambda, ridge, rthr, rhs_unit, fail_min, rcond_min_bits, rcond_exact, spill, S,
            (size_t)off(S) + 2};
  void (*fn)(const F64Args) = S > 0 ? chol_f64_kernel<true> : chol_f64_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int per_sm = (int)std::max<size_t>(1, 233472 / (smem + 1024));
  const int64_t maxgrid = S > 0 ? (int64_t)sms : (int64_t)sms * per_sm;  // spill scratch: one slot per SM
  const unsigned grid = (unsigned)(nsys < maxgrid ? nsys : maxgrid);
  note_launch(S > 0 ? "chol_f64_kernel(spill)" : "chol_f64_kernel");
  fn<<<grid, kT64, smem, st>>>(a);
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
