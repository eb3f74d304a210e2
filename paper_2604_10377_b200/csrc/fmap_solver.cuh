// Batched regularized functional-map solver — sm_100a: shared declarations.
//
// One row system s = (pair q, row i):
//     (G_q + lambda*diag(M_q[i,:]) + ridge*I) x = R_q[i,:]^T,   C_q[i,:] = x^T
// replacing the per-system PartialPivLU of the reference
// (/root/reference/proj/include/fmsolve/solver.hpp:147-170, driven by
// solve_batched_many :220-322).  The system is SPD by construction (G = A A^T
// symmetric PSD, lambda*m + ridge >= 0), so it is factored by Cholesky: the
// tcgen05/TMEM kernel in fmap_tc.cu (f32) and the DMMA kernel in fmap_f64.cu (f64).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fmap {

struct SolveParams {
  const float* gram;  // [b][k][k]
  const float* rhs;   // [b][k][k]
  const float* mask;  // [b][k][k]        (mask_mode == 0)
  const float* ev1;   // [b][k]           (mask_mode != 0)
  const float* ev2;   // [b][k]
  const float* ev_max;  // [b] max(ev1, ev2) of each pair (mask_mode == 1)
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
  unsigned int* rcond_exact;     // count of systems that ran the exact rcond estimator
  float* tc_scratch;             // tensor-core solver: per-CTA L scratch (tc_scratch_bytes)
  const float* gram_rowsum;      // [b][k] sum_c |G[q][r][c]| (launch_gram_check): rcond certificate
  long long* trace;              // debug phase trace (nullptr = off)
  int trace_block;
  int debug;                     // timing experiments only (FMAP_DEBUG): bit 0 = skip the back substitution
};

// Tensor-core (tcgen05 / TMEM) solver, fmap_tc.cu.
bool tc_supported(int k, int optin_smem);
int tc_max_resolution(int optin_smem);
size_t tc_scratch_bytes(int k, int64_t nsys, int num_sms);
cudaError_t launch_project_tc(const float* phi, const float* mass, const float* F, int64_t b,
                              int64_t n, int k, int d, float* out, cudaStream_t st);
cudaError_t launch_chol_tc(const SolveParams& p, int mask_mode, cudaStream_t stream, int parts = 3);

// f64 route (fmap_f64.cu)
size_t chol_f64_smem_bytes(int k, size_t optin);
size_t chol_f64_spill_doubles(int k, size_t optin, int num_sms);
cudaError_t launch_chol_f64(const double* G, const double* R, const double* M, double* C, int k, int64_t nsys,
                            double lambda, double ridge, double rthr, int rhs_unit, unsigned long long* fail_min,
                            unsigned* rcond_min_bits, unsigned* rcond_exact, double* spill, cudaStream_t st);
cudaError_t launch_validate_f64(const double* g, const double* r, const double* m, size_t n, unsigned* flags,
                                cudaStream_t st);
cudaError_t launch_residual_f64(const double* Cm, const double* G, const double* R, const double* M, int64_t b,
                                int k, double lambda, double* sq, cudaStream_t st);
cudaError_t launch_fault_combine_f64(double* x, const double* z, int k, int w, double alpha,
                                     unsigned long long* fail_min, cudaStream_t st);

}  // namespace fmap
