/*
 * fmap_cuda.h — C ABI of libfmap_cuda, the B200 (sm_100a) batched regularized
 * functional-map solver.
 *
 * This is the drop-in boundary for the reference's solver path
 * (/root/reference/proj/include/fmsolve/solver.hpp, masks.hpp).  Every entry
 * point below names the reference interface it replaces.  Plain C: opaque
 * context, raw pointers, sizes and status codes; no exceptions and no C++ or
 * torch types cross the boundary.  The header-only C++ adapter
 * include/fmsolve_cuda.hpp rebuilds the reference's exception taxonomy and
 * signatures on top of it.
 *
 * Layouts (all row-major, contiguous, fp32):
 *   gram, rhs, mask, C : [b][k][k]      (pair q, row i, column j)
 *   A, B (descriptors)  : [b][k][d]
 *   phi                 : [b][n][k]     (per shape, n vertices)
 *   mass                : [b][n]
 *   F                   : [b][n][d]
 *   ev                  : [b][k]
 * System s of a batch is (pair q = s / k, row i = s % k)  (solver.hpp:262-263).
 *
 * Preconditions beyond the reference's (which factors every row system by
 * partial-pivot LU): each system G + lambda*diag(M[i,:]) + ridge*I is factored by
 * Cholesky from the lower triangle of G, so gram must be symmetric (checked on
 * the device: |G[r][c] - G[c][r]| <= 1e-4 * max(|G[r][c]|, |G[c][r]|,
 * sqrt|G[r][r] G[c][c]|), else FMAP_INVALID_ARGUMENT) and a system that is not
 * positive definite is reported FMAP_SINGULAR.  G = A A^T (normal_equations)
 * satisfies both whenever the reference's LU succeeds on an SPD system.
 */
#ifndef FMAP_CUDA_H
#define FMAP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMAP_CUDA_ABI_VERSION 1

/* Status codes <-> reference exceptions (types.hpp:25-80). */
enum fmap_status {
  FMAP_OK = 0,
  FMAP_INVALID_ARGUMENT = 1, /* std::invalid_argument       */
  FMAP_SINGULAR = 2,         /* fmsolve::SingularSystemError */
  FMAP_MEMORY_CAP = 3,       /* fmsolve::MemoryCapExceeded   */
  FMAP_CUDA_ERROR = 4,       /* device / driver failure      */
  FMAP_RANK_DEFICIENT = 5    /* fmsolve::RankDeficientError  */
};

/* masks.hpp:7-11 MaskKind */
enum fmap_mask_kind { FMAP_MASK_COMMUTATIVITY = 0, FMAP_MASK_RESOLVENT = 1 };

/* SolverOptions<float> (solver.hpp:29-50). */
typedef struct fmap_solver_options {
  float ridge;            /* adds ridge*I to every row system (default 0)             */
  float rcond_threshold;  /* < 0 selects the reference default for f32 (1e-7)         */
  int has_memory_cap;     /* std::optional<size_t> memory_cap_bytes                    */
  uint64_t memory_cap_bytes;
  unsigned threads;       /* accepted for signature parity; results never depend on it */
  int inject_fault;       /* solver.hpp:47-49 / 269-273 test hook                     */
  int compute_residual;   /* fill report.max_residual (reference always does)         */
} fmap_solver_options;

/* BatchSolveReport<float> (solver.hpp:62-68) plus the error payloads. */
typedef struct fmap_report {
  double max_residual;       /* max_q ||C_q G_q + lambda M_q.*C_q - R_q||_F            */
  double wall_seconds;       /* solve-only device time (CUDA events)                   */
  uint64_t peak_extra_bytes; /* transient device bytes of the "cuda" route             */
  int64_t failing_system;    /* SingularSystemError::system(); -1 when none            */
  uint64_t required_bytes;   /* MemoryCapExceeded::required_bytes()                    */
  uint64_t cap_bytes;        /* MemoryCapExceeded::cap_bytes()                         */
  double min_rcond;          /* smallest rcond over all systems: the comparison-matrix  */
                             /* certificate (a lower bound) or, where that was          */
                             /* inconclusive, the exact Hager/Higham estimate           */
  int64_t rcond_exact_systems; /* systems that needed the exact estimator               */
  double factor_seconds;     /* f32 route: device time of the factorization kernel     */
                             /* (chol_tc_kernel) alone, CUDA events; 0 elsewhere       */
} fmap_report;

typedef struct fmap_ctx fmap_ctx;

/* Context = one device + one stream + a monotonically growing device arena;
 * the role BatchedWorkspace plays in the reference (solver.hpp:86-93). */
int fmap_ctx_create(int device, fmap_ctx** out);
int fmap_ctx_destroy(fmap_ctx* ctx);
/* Use a caller-owned stream (e.g. torch's current stream); NULL = ctx stream. */
int fmap_ctx_set_stream(fmap_ctx* ctx, void* cuda_stream);
const char* fmap_last_error(const fmap_ctx* ctx);
int fmap_abi_version(void);
void fmap_default_options(fmap_solver_options* opts);

/* Replaces solve_batched_many<float> (solver.hpp:225-322) / solve_batched
 * (solver.hpp:352-366): HOST buffers in and out.  Validation
 * (solver.hpp:132-145) runs on the device before any status is returned;
 * SINGULAR reports the lowest failing global system index; no partial results
 * on error (C_out is left untouched, or zero-filled when the copy-pipelined
 * path — batches of >= 8 pairs, 4 chunks, FMAP_PIPELINE=<chunks> to tune, 1 to disable —
 * had already copied some chunks back). */
int fmap_solve_f32(fmap_ctx* ctx, int64_t b, int64_t k, const float* gram, const float* rhs,
                   const float* mask, float lambda, const fmap_solver_options* opts,
                   float* C_out, fmap_report* report);

/* Replaces solve_batched_many<double> (solver.hpp:225-322), the reference's
 * default precision (bench.hpp:32): f64 end to end, rcond threshold 1e-14 when
 * opts->rcond_threshold < 0 (solver.hpp:18-27), explicit mask only, k up to the
 * single-CTA shared-memory limit (234 on B200; larger k -> INVALID_ARGUMENT).
 * Same validation / SINGULAR / memory-cap / fault-hook contract as f32. */
int fmap_solve_f64(fmap_ctx* ctx, int64_t b, int64_t k, const double* gram, const double* rhs,
                   const double* mask, double lambda, const fmap_solver_options* opts,
                   double* C_out, fmap_report* report);
int fmap_solve_f64_dev(fmap_ctx* ctx, int64_t b, int64_t k, const double* d_gram,
                       const double* d_rhs, const double* d_mask, double lambda,
                       const fmap_solver_options* opts, double* d_C_out, fmap_report* report);

/* Same contract on DEVICE pointers (inputs already resident in HBM). */
int fmap_solve_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_gram,
                       const float* d_rhs, const float* d_mask, float lambda,
                       const fmap_solver_options* opts, float* d_C, fmap_report* report);

/* Fused-mask variant: row i of the mask is generated inside the solver from
 * the eigenvalues (masks.hpp:36-82 / 13-34); M never touches HBM. */
int fmap_solve_ev_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_gram,
                          const float* d_rhs, const float* d_ev1, const float* d_ev2,
                          int mask_kind, float sigma, float lambda,
                          const fmap_solver_options* opts, float* d_C, fmap_report* report);

/* Replaces build_mask(kind, ev1, ev2, sigma) (masks.hpp:84-89), batched. */
int fmap_mask_f32(fmap_ctx* ctx, int64_t b, int64_t k, const float* ev1, const float* ev2,
                  int mask_kind, float sigma, float* mask_out);
int fmap_mask_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_ev1,
                      const float* d_ev2, int mask_kind, float sigma, float* d_mask_out);

/* Replaces normal_equations(a, b) (solver.hpp:95-103), batched:
 * gram = A A^T, rhs = B A^T. */
int fmap_normal_equations_f32(fmap_ctx* ctx, int64_t b, int64_t k, int64_t d, const float* A,
                              const float* B, float* gram_out, float* rhs_out);
int fmap_normal_equations_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, int64_t d,
                                  const float* d_A, const float* d_B, float* d_gram,
                                  float* d_rhs);

/* North_star projection A = Phi^T diag(Mass) F (stands where
 * project_to_spectral, spectral.hpp:47-93, stands for mass-orthonormal bases). */
int fmap_project_f32_dev(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d,
                         const float* d_phi, const float* d_mass, const float* d_F,
                         float* d_out);

/* Replaces project_to_spectral<Scalar>(basis, features, opts) (spectral.hpp:47-93)
 * for b bases at once: A[q] = pinv(Phi[q]) F[q] (k x d), Phi [b][n][k], F [b][n][d].
 * Decisions as the reference: n < k or cond(Phi) > condition_threshold (the
 * reference default is 1e10) take the rank-revealing path, where a basis of
 * numerical rank < k (threshold eps * min(n, k) * sigma_max) is an error:
 * FMAP_RANK_DEFICIENT (RankDeficientError), report->failing_system = the lowest
 * such shape, rank_out[q] (optional, b entries) = every shape's detected rank.
 * Computed in f64 on the device (one-sided Jacobi SVD per shape); the f32 entry
 * widens its inputs on the device and rounds A back. */
int fmap_project_pinv_f64(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const double* phi,
                          const double* F, double condition_threshold, double* A_out, int64_t* rank_out,
                          fmap_report* report);
int fmap_project_pinv_f64_dev(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const double* d_phi,
                              const double* d_F, double condition_threshold, double* d_A, int64_t* rank_out,
                              fmap_report* report);
int fmap_project_pinv_f32(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const float* phi,
                          const float* F, float condition_threshold, float* A_out, int64_t* rank_out,
                          fmap_report* report);

/* check_stationarity (solver.hpp:116-128) per pair: out[q] =
 * ||C G + lambda M.*C - R||_F, fp32 products, fp64 accumulation. */
int fmap_residual_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_C,
                          const float* d_gram, const float* d_rhs, const float* d_mask,
                          float lambda, double* d_out);

/* End-to-end device pipeline for one direction (and optionally the reverse):
 * (Phi1, mass1, F1, ev1), (Phi2, mass2, F2, ev2)  ->  C_xy [b][k][k]
 * and, when C_yx != NULL, C_yx from (B, A, mask(ev2, ev1)).
 * n1 and n2 may differ (partial shapes). Scratch comes from the ctx arena. */
int fmap_pipeline_f32_dev(fmap_ctx* ctx, int64_t b, int64_t n1, int64_t n2, int64_t k,
                          int64_t d, const float* d_phi1, const float* d_mass1,
                          const float* d_F1, const float* d_ev1, const float* d_phi2,
                          const float* d_mass2, const float* d_F2, const float* d_ev2,
                          int mask_kind, float sigma, float lambda,
                          const fmap_solver_options* opts, float* d_Cxy, float* d_Cyx,
                          fmap_report* report);

/* Largest k the single-CTA shared-memory solver handles on this device. */
int64_t fmap_max_resolution(fmap_ctx* ctx);

/* Number of solver-family kernel launches issued by the last call (evidence
 * for bench.py's gpu_launches). */
int64_t fmap_last_launch_count(const fmap_ctx* ctx);
/* Names of those kernels, comma-separated, in launch order (e.g.
 * "validate_kernel,gram_check_kernel,chol_tc_kernel"); valid until the next call. */
const char* fmap_last_launches(const fmap_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* FMAP_CUDA_H */
