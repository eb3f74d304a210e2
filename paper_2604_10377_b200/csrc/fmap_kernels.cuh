#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <algorithm>
#include <cuda_runtime.h>

#include "fmap_solver.cuh"

namespace fmap {

// Per-thread log of the kernels the current C-ABI call launched (evidence for
// fmap_last_launches / bench.py's gpu_launches).
void note_launch(const char* kernel);
void clear_launch_log();
const char* launch_log();
int launch_log_count();

// parts: 1 = factorization, 2 = back substitution + verdict (over a factorization
// launched before with the same p), 3 = both
cudaError_t launch_chol_solve(const SolveParams& p, int mask_mode, cudaStream_t stream, int parts = 3);

cudaError_t launch_mask(const float* ev1, const float* ev2, int64_t b, int k, int kind,
                        float sigma, float* out, cudaStream_t st);
cudaError_t launch_validate(const float* g, const float* r, const float* m, size_t n,
                            unsigned* flags, cudaStream_t st);
cudaError_t launch_validate_ev(const float* e1, const float* e2, size_t n, unsigned* flags,
                               cudaStream_t st);
cudaError_t launch_ev_max_check(const float* e1, const float* e2, int64_t b, int k, unsigned* flags,
                                cudaStream_t st,
                                float* out = nullptr);
cudaError_t launch_gram_check(const float* G, int64_t b, int k, float* S, unsigned* flags, cudaStream_t st);
// tcgen05 3xTF32 normal equations (fmap_gram.cu): nprod <= 4 products
// out_i[q] = X_i[q] Y_i[q]^T (k x d operands), sym_i = 1 for X_i == Y_i (mirrored).
cudaError_t launch_gram_tc(int nprod, const float* const* X, const float* const* Y, float* const* out,
                           const int* sym, int64_t b, int k, int d, cudaStream_t st);
cudaError_t launch_residual_tc(const float* C, const float* G, const float* R, const float* M, int64_t b, int k,
                               float lambda, double* partial, cudaStream_t st);
// Euclidean pinv projection (fmap_pinv.cu), f64
size_t pinv_work_doubles(int64_t b, int64_t n, int k, int d);
cudaError_t launch_pinv(const double* phi, const double* F, int64_t b, int64_t n, int k, int d, double cond_thr,
                        double* work, double* out, int* rank_out, unsigned long long* fail_min, cudaStream_t st);
cudaError_t launch_convert_f32_f64(const float* x, double* y, size_t n, cudaStream_t st);
cudaError_t launch_convert_f64_f32(const double* x, float* y, size_t n, cudaStream_t st);
cudaError_t launch_finite_f64(const double* x, size_t n, unsigned bit, unsigned* flags, cudaStream_t st);
cudaError_t launch_gemm_nt(const float* X, const float* Y, int64_t b, int M, int N, int K,
                           float* out, cudaStream_t st);
cudaError_t launch_project(const float* phi, const float* mass, const float* F, int64_t b,
                           int64_t n, int k, int d, float* out, cudaStream_t st);
cudaError_t launch_residual(const float* C, const float* G, const float* R, const float* M,
                            int64_t b, int k, float lambda, double* partial, double* out,
                            cudaStream_t st,
                            unsigned long long* maxbits = nullptr);
size_t residual_partial_count(int64_t b, int k);
cudaError_t launch_fault_combine(float* x, const float* z, int k, int w, float alpha,
                                 unsigned long long* fail_min, unsigned long long sys,
                                 cudaStream_t st);

}  // namespace fmap
