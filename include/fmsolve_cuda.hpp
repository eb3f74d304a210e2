// fmsolve_cuda.hpp — header-only C++ adapter: the reference's solver API on top
// of the libfmap_cuda C ABI (include/fmap_cuda.h).
//
// Drop-in for the batched route of /root/reference/proj/include/fmsolve/solver.hpp.
// Namespace fmsolve::cuda holds the reference's own names and signatures, so a
// caller switches routes by qualifying the call:
//
//   reference (fmsolve::)                              route "cuda" (fmsolve::cuda::)
//   solve_batched_many(span, λ, opts, ws)  solver.hpp:225   solve_batched_many(span, λ, opts, ws)
//   solve_batched(problem, λ, opts, ws)    solver.hpp:352   solve_batched(problem, λ, opts, ws)
//   solve_batched(a, b, mask, λ, opts, ws) solver.hpp:360   solve_batched(a, b, mask, λ, opts, ws)
//   build_mask(kind, ev1, ev2, sigma)      masks.hpp:85     build_mask(kind, ev1, ev2, sigma)
//
// The BatchedWorkspace (solver.hpp:86-93) is honoured the reference's way: its
// vectors grow monotonically and are reused across calls, here as the packed
// host staging of G/R/M (lhs) and C (rhs); the device arena lives in the
// per-thread context.  fmsolve::solve_cuda_many / solve_cuda / build_mask_cuda
// are the same calls with an explicit device ordinal.
//
// Error behaviour is the reference's (types.hpp:25-67, solver.hpp:229-322):
// std::invalid_argument on validation, MemoryCapExceeded before allocating,
// SingularSystemError(lowest failing system index), nothing returned on error.
// Scalar = float runs the fp32 tcgen05 route, Scalar = double the f64 route
// (fmap_solve_f64, rcond threshold 1e-14 by default).  peak_extra_bytes is the cuda route's own device accounting
// (SURVEY D9), not the b*k^3 of the batched route.
//
// Two modes:
//  * default: include the reference's "fmsolve/solver.hpp" (Eigen types) —
//    drop this file next to it in proj/include/fmsolve/;
//  * FMSOLVE_CUDA_STANDALONE: minimal row-major stand-ins for the reference
//    types (no Eigen), used by tests/cpp/test_adapter.cpp.
#pragma once

#include "fmap_cuda.h"

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#ifndef FMSOLVE_CUDA_STANDALONE
#include "fmsolve/masks.hpp"
#include "fmsolve/solver.hpp"
#else
namespace fmsolve {

// Row-major dense matrix with the slice of Eigen's interface the adapter uses.
template <typename Scalar>
class MatrixX {
 public:
  MatrixX() = default;
  MatrixX(std::ptrdiff_t r, std::ptrdiff_t c) : r_(r), c_(c), v_((size_t)(r * c)) {}
  std::ptrdiff_t rows() const { return r_; }
  std::ptrdiff_t cols() const { return c_; }
  Scalar* data() { return v_.data(); }
  const Scalar* data() const { return v_.data(); }
  Scalar& operator()(std::ptrdiff_t i, std::ptrdiff_t j) { return v_[(size_t)(i * c_ + j)]; }
  Scalar operator()(std::ptrdiff_t i, std::ptrdiff_t j) const { return v_[(size_t)(i * c_ + j)]; }

 private:
  std::ptrdiff_t r_ = 0, c_ = 0;
  std::vector<Scalar> v_;
};

template <typename Scalar>
using VectorX = std::vector<Scalar>;

class SingularSystemError : public std::runtime_error {
 public:
  SingularSystemError(std::ptrdiff_t system, const std::string& what)
      : std::runtime_error(what), system_(system) {}
  std::ptrdiff_t system() const { return system_; }

 private:
  std::ptrdiff_t system_;
};

class MemoryCapExceeded : public std::runtime_error {
 public:
  MemoryCapExceeded(std::size_t required, std::size_t cap, const std::string& what)
      : std::runtime_error(what), required_(required), cap_(cap) {}
  std::size_t required_bytes() const { return required_; }
  std::size_t cap_bytes() const { return cap_; }

 private:
  std::size_t required_, cap_;
};

enum class MaskKind { Commutativity, Resolvent };

template <typename Scalar>
struct SolverOptions {
  Scalar ridge = Scalar(0);
  Scalar rcond_threshold = sizeof(Scalar) == sizeof(double) ? Scalar(1e-14) : Scalar(1e-7);
  std::optional<std::size_t> memory_cap_bytes;
  unsigned threads = 0;
  bool inject_fault = false;
};

template <typename Scalar>
struct SolveReport {
  MatrixX<Scalar> map;
  Scalar residual_norm = Scalar(0);
  std::chrono::duration<double> wall_time{0};
  std::size_t peak_extra_bytes = 0;
};

template <typename Scalar>
struct BatchSolveReport {
  std::vector<MatrixX<Scalar>> maps;
  Scalar max_residual_norm = Scalar(0);
  std::chrono::duration<double> wall_time{0};
  std::size_t peak_extra_bytes = 0;
};

template <typename Scalar>
struct NormalEquations {
  MatrixX<Scalar> gram;
  MatrixX<Scalar> rhs;
};

template <typename Scalar>
struct RegularizedProblem {
  NormalEquations<Scalar> neq;
  MatrixX<Scalar> mask;
  std::ptrdiff_t resolution() const { return mask.rows(); }
};

template <typename Scalar>
struct BatchedWorkspace {
  std::vector<Scalar> lhs;
  std::vector<Scalar> rhs;
};

}  // namespace fmsolve
#endif

namespace fmsolve {
namespace cuda_detail {

struct CtxDeleter {
  void operator()(fmap_ctx* c) const { fmap_ctx_destroy(c); }
};

// One context (device + stream + arena) per thread and device.
inline fmap_ctx* context(int device) {
  thread_local std::vector<std::unique_ptr<fmap_ctx, CtxDeleter>> ctxs;
  if ((int)ctxs.size() <= device) ctxs.resize(device + 1);
  if (!ctxs[device]) {
    fmap_ctx* c = nullptr;
    if (fmap_ctx_create(device, &c) != FMAP_OK)
      throw std::runtime_error("libfmap_cuda: cannot create a context on device " +
                               std::to_string(device) + " (no CUDA device? there is no CPU fallback)");
    ctxs[device].reset(c);
  }
  return ctxs[device].get();
}

[[noreturn]] inline void raise(fmap_ctx* ctx, int status, const fmap_report& rep) {
  const std::string msg = fmap_last_error(ctx);
  switch (status) {
    case FMAP_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FMAP_SINGULAR: throw SingularSystemError(rep.failing_system, msg);
    case FMAP_MEMORY_CAP: throw MemoryCapExceeded(rep.required_bytes, rep.cap_bytes, msg);
    default: throw std::runtime_error("libfmap_cuda: " + msg);
  }
}

inline void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

}  // namespace cuda_detail

/// solve_batched_many (solver.hpp:225-322) through the GPU route on `device`.
/// Scalar = float runs the fp32 tcgen05 route, Scalar = double the f64 route.
template <typename Scalar>
BatchSolveReport<Scalar> solve_cuda_many(std::span<const RegularizedProblem<Scalar>> problems,
                                         Scalar lambda, const SolverOptions<Scalar>& opts = {},
                                         int device = 0, BatchedWorkspace<Scalar>* workspace = nullptr) {
  static_assert(std::is_same_v<Scalar, float> || std::is_same_v<Scalar, double>,
                "the cuda route computes in float or double");
  using cuda_detail::require;
  require(!problems.empty(), "no problems to solve");
  const std::ptrdiff_t k = problems.front().resolution();
  require(k >= 1, "problem is empty");
  for (const auto& p : problems) {
    require(p.mask.cols() == p.mask.rows(), "penalty mask must be square");
    require(p.neq.gram.rows() == p.mask.rows() && p.neq.gram.cols() == p.mask.rows(),
            "gram matrix must be k x k");
    require(p.neq.rhs.rows() == p.mask.rows() && p.neq.rhs.cols() == p.mask.rows(),
            "rhs matrix must be k x k");
    require(p.resolution() == k, "all problems in a batch must share the spectral resolution");
  }
  const std::size_t b = problems.size(), kk = (std::size_t)k * k;
  // packed [b][k][k] host staging, reused across calls through the workspace
  BatchedWorkspace<Scalar> local;
  BatchedWorkspace<Scalar>& ws = workspace ? *workspace : local;
  if (ws.lhs.size() < 3 * b * kk) ws.lhs.resize(3 * b * kk);
  if (ws.rhs.size() < b * kk) ws.rhs.resize(b * kk);
  Scalar* G = ws.lhs.data();
  Scalar* R = G + b * kk;
  Scalar* M = R + b * kk;
  Scalar* C = ws.rhs.data();
  for (std::size_t q = 0; q < b; ++q) {
    const auto& p = problems[q];
    for (std::size_t e = 0; e < kk; ++e) {
      G[q * kk + e] = p.neq.gram.data()[e];
      R[q * kk + e] = p.neq.rhs.data()[e];
      M[q * kk + e] = p.mask.data()[e];
    }
  }
  fmap_solver_options o;
  fmap_default_options(&o);
  o.ridge = (float)opts.ridge;
  // the f64 route reads a negative threshold as its own default (1e-14)
  o.rcond_threshold = opts.rcond_threshold == SolverOptions<Scalar>{}.rcond_threshold ? -1.f
                                                                                       : (float)opts.rcond_threshold;
  o.has_memory_cap = opts.memory_cap_bytes ? 1 : 0;
  o.memory_cap_bytes = opts.memory_cap_bytes ? *opts.memory_cap_bytes : 0;
  o.threads = opts.threads;
  o.inject_fault = opts.inject_fault ? 1 : 0;
  fmap_report rep;
  fmap_ctx* ctx = cuda_detail::context(device);
  int st;
  if constexpr (std::is_same_v<Scalar, double>)
    st = fmap_solve_f64(ctx, (int64_t)b, (int64_t)k, G, R, M, lambda, &o, C, &rep);
  else
    st = fmap_solve_f32(ctx, (int64_t)b, (int64_t)k, G, R, M, lambda, &o, C, &rep);
  if (st != FMAP_OK) cuda_detail::raise(ctx, st, rep);
  BatchSolveReport<Scalar> out;
  out.maps.reserve(b);
  for (std::size_t q = 0; q < b; ++q) {
    out.maps.emplace_back(k, k);
    for (std::size_t e = 0; e < kk; ++e) out.maps.back().data()[e] = C[q * kk + e];
  }
  out.max_residual_norm = (Scalar)rep.max_residual;
  out.wall_time = std::chrono::duration<double>(rep.wall_seconds);
  out.peak_extra_bytes = (std::size_t)rep.peak_extra_bytes;
  return out;
}

/// solve_batched(problem, λ, opts) (solver.hpp:352-358) through the GPU route.
template <typename Scalar>
SolveReport<Scalar> solve_cuda(const RegularizedProblem<Scalar>& problem, Scalar lambda,
                               const SolverOptions<Scalar>& opts = {}, int device = 0,
                               BatchedWorkspace<Scalar>* workspace = nullptr) {
  auto batch = solve_cuda_many(std::span<const RegularizedProblem<Scalar>>(&problem, 1), lambda,
                               opts, device, workspace);
  SolveReport<Scalar> r;
  r.map = std::move(batch.maps.front());
  r.residual_norm = batch.max_residual_norm;
  r.wall_time = batch.wall_time;
  r.peak_extra_bytes = batch.peak_extra_bytes;
  return r;
}

#ifndef FMSOLVE_CUDA_STANDALONE
/// solve_batched(a, b, mask, λ, opts) (solver.hpp:360-366): Gram/RHS by the
/// reference's make_problem, the solve on the GPU.
template <typename Scalar>
SolveReport<Scalar> solve_cuda(const MatrixX<Scalar>& a, const MatrixX<Scalar>& b,
                               const MatrixX<Scalar>& mask, Scalar lambda,
                               const SolverOptions<Scalar>& opts = {}, int device = 0) {
  return solve_cuda(make_problem(a, b, mask), lambda, opts, device);
}
#endif

/// build_mask(kind, ev1, ev2, sigma) (masks.hpp:84-89) on the GPU.
template <typename Scalar, typename Vec>
MatrixX<Scalar> build_mask_cuda(MaskKind kind, const Vec& ev1, const Vec& ev2,
                                Scalar sigma = Scalar(0.5), int device = 0) {
  cuda_detail::require(ev1.size() == ev2.size(), "eigenvalue vectors must have equal length");
  const std::ptrdiff_t k = (std::ptrdiff_t)ev1.size();
  cuda_detail::require(k >= 1, "eigenvalue vectors must be non-empty");
  std::vector<float> e1(k), e2(k), m((size_t)(k * k));
  for (std::ptrdiff_t j = 0; j < k; ++j) {
    e1[j] = (float)ev1[j];
    e2[j] = (float)ev2[j];
  }
  fmap_ctx* ctx = cuda_detail::context(device);
  const int st = fmap_mask_f32(ctx, 1, k, e1.data(), e2.data(),
                               kind == MaskKind::Resolvent ? FMAP_MASK_RESOLVENT : FMAP_MASK_COMMUTATIVITY,
                               (float)sigma, m.data());
  if (st != FMAP_OK) {
    fmap_report rep{};
    cuda_detail::raise(ctx, st, rep);
  }
  MatrixX<Scalar> out(k, k);
  for (std::size_t e = 0; e < m.size(); ++e) out.data()[e] = (Scalar)m[e];
  return out;
}

namespace cuda {

/// Route "cuda" under the reference's own names and signatures (device 0).
template <typename Scalar>
BatchSolveReport<Scalar> solve_batched_many(std::span<const RegularizedProblem<Scalar>> problems, Scalar lambda,
                                            const SolverOptions<Scalar>& opts = {},
                                            BatchedWorkspace<Scalar>* workspace = nullptr) {
  return solve_cuda_many(problems, lambda, opts, 0, workspace);
}

template <typename Scalar>
SolveReport<Scalar> solve_batched(const RegularizedProblem<Scalar>& problem, Scalar lambda,
                                  const SolverOptions<Scalar>& opts = {},
                                  BatchedWorkspace<Scalar>* workspace = nullptr) {
  return solve_cuda(problem, lambda, opts, 0, workspace);
}

#ifndef FMSOLVE_CUDA_STANDALONE
template <typename Scalar>
SolveReport<Scalar> solve_batched(const MatrixX<Scalar>& a, const MatrixX<Scalar>& b, const MatrixX<Scalar>& mask,
                                  Scalar lambda, const SolverOptions<Scalar>& opts = {},
                                  BatchedWorkspace<Scalar>* workspace = nullptr) {
  return solve_cuda(make_problem(a, b, mask), lambda, opts, 0, workspace);
}
#endif

template <typename Scalar, typename Vec>
MatrixX<Scalar> build_mask(MaskKind kind, const Vec& ev1, const Vec& ev2, Scalar sigma = Scalar(0.5)) {
  return build_mask_cuda<Scalar>(kind, ev1, ev2, sigma, 0);
}

}  // namespace cuda
}  // namespace fmsolve
