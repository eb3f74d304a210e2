// Batched regularized functional-map solver — sm_100a.
//
// One CTA per row system s = (pair q, row i):
//     (G_q + lambda*diag(M_q[i,:]) + ridge*I) x = R_q[i,:]^T,   C_q[i,:] = x^T
// replacing the per-system PartialPivLU of the reference
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170, driven by
// solve_batched_many :220-322).  The system is SPD by construction, so it is
// factored with a blocked right-looking Cholesky entirely in shared memory.
//
// Shared-memory layout ("packed, 4-aligned, column-major lower triangle"):
//   K4 = round_up(k, 4)  (rows/cols k..K4-1 are identity padding)
//   Rp = K4 + 4           (row K4 is the augmented right-hand side)
//   column c stores rows [c & ~3, Rp), starting 16-byte aligned, so every
//   4-row group of a column is one LDS.128/STS.128.
// The right-hand side rides along as row K4 (augmented matrix), so the forward
// substitution y = L^{-1} r falls out of the factorization for free.
//
// Per panel of NB=16 columns:
//   B. TRSM   L21 = A21 * L11^{-T}       rows below the block (incl. row K4)
//   C. SYRK   next panel's columns        (lookahead)
//   D. warp 0/lane 0: factor the next 16x16 diagonal block (Cholesky + inverse)
//      warps 1..: SYRK of the remaining trailing matrix (32x16 warp tiles,
//      4x4 register tiles, broadcast operands)
// then warp 0 runs the blocked back substitution L^T x = y using the stored
// L11^{-1} blocks and writes the row of C coalesced.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fmap {

constexpr int kNB = 16;  // panel width (columns per diagonal block)

struct SolveParams {
  const float* gram;  // [b][k][k]
  const float* rhs;   // [b][k][k]
  const float* mask;  // [b][k][k]        (mask_mode == 0)
  const float* ev1;   // [b][k]           (mask_mode != 0)
  const float* ev2;   // [b][k]
  float* C;           // [b][k][k]
  int k;
  int K4;
  int Rp;
  int64_t nsys;        // systems in this launch
  int64_t sys_offset;  // global index of the first system of this launch
  float lambda;
  float ridge;
  float sigma;
  float rcond_thr;
  // Optional override of the right-hand side of every system (fault-injection
  // Sherman–Morrison pass): rhs_unit >= 0 replaces r with e_{rhs_unit}.
  int rhs_unit;
  unsigned long long* fail_min;  // lowest failing global system index
  unsigned int* rcond_min_bits;  // float bits of the smallest rcond estimate
  unsigned int* flags;           // validation flags (bit 5: empty spectrum)
  float* tc_scratch;             // tensor-core solver: per-CTA L scratch (tc_scratch_bytes)
  const float* gram_rowsum;      // [b][k] sum_c |G[q][r][c]| (launch_gram_check): rcond certificate
  long long* trace;              // debug phase trace (nullptr = off)
  int trace_block;
  int force_single;              // debug: force one system per CTA
  int pair_shared_smsp;          // debug: pair kernel without the isolated panel-warp SMSP
};

__host__ __device__ __forceinline__ int col_off(int c, int Rp) {
  const int g = c >> 2, u = c & 3;
  return 4 * g * Rp - 8 * g * (g - 1) + u * (Rp - 4 * g);
}

__host__ __device__ __forceinline__ int packed_size(int K4) { return col_off(K4, K4 + 4); }

// Shared-memory bytes of one system (packed matrix + x vector + scalars).
__host__ __device__ __forceinline__ size_t solver_smem_bytes(int k) {
  const int K4 = (k + 3) & ~3;
  return (size_t)(packed_size(K4) + 2 * K4 + 104 + 32) * sizeof(float);
}

// Tensor-core (tcgen05 / TMEM) solver, fmap_tc.cu.
bool tc_supported(int k, int optin_smem);
size_t tc_scratch_bytes(int k, int64_t nsys, int num_sms);
cudaError_t launch_project_tc(const float* phi, const float* mass, const float* F, int64_t b,
                              int64_t n, int k, int d, float* out, cudaStream_t st);
cudaError_t launch_chol_tc(const SolveParams& p, int mask_mode, cudaStream_t stream);

// f64 route (fmap_f64.cu)
size_t chol_f64_smem_bytes(int k);
cudaError_t launch_chol_f64(const double* G, const double* R, const double* M, double* C, int k, int64_t nsys,
                            double lambda, double ridge, double rthr, int rhs_unit, unsigned long long* fail_min,
                            unsigned* rcond_min_bits, cudaStream_t st);
cudaError_t launch_validate_f64(const double* g, const double* r, const double* m, size_t n, unsigned* flags,
                                cudaStream_t st);
cudaError_t launch_residual_f64(const double* Cm, const double* G, const double* R, const double* M, int64_t b,
                                int k, double lambda, double* sq, cudaStream_t st);
cudaError_t launch_fault_combine_f64(double* x, const double* z, int k, int w, double alpha,
                                     unsigned long long* fail_min, cudaStream_t st);

}  // namespace fmap
