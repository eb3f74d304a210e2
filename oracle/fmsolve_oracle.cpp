// TEST INFRASTRUCTURE ONLY — CPU ORACLE. NOT PART OF THE PRODUCT PATH.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library, and only as the checker or the timed
// CPU reference.  The product (libfmap_cuda) never links or calls it.
//
// A CPU restatement of the reference functional-map solver
// (/root/reference/proj/include/fmsolve/*.hpp).  The reference itself cannot
// be built here (Eigen 3.4, doctest and CLI11 are absent), so
// this file restates its algorithms without Eigen:
//
//   * validation and error taxonomy     solver.hpp:95-145, types.hpp:25-80
//   * per-system partial-pivot LU +      solver.hpp:147-170 (Eigen PartialPivLU,
//     Hager/Higham 1-norm rcond estimate   rcond(), solve())
//   * rowwise route (i outer, q inner)   solver.hpp:174-218
//   * batched route (arena, memory cap,  solver.hpp:220-322
//     contiguous thread chunks, lowest
//     failing index, inject_fault)
//   * k^2 x k^2 "full oracle"            solver.hpp:368-444 (dense LU instead of
//                                        SparseLU; same assembled system)
//   * masks                              masks.hpp:13-89
//   * reference synthetic generator      bench.hpp:52-93 (same std:: engines)
//   * energy / gradient                  spectral.hpp:95-125
//
// Plus the north_star projection A = Phi^T * diag(Mass) * F, which
// the reference does not contain.
//
// Parity pinning: see tests/test_oracle.py (reference KATs restated from
// proj/tests/test_solver.cpp, test_masks.cpp, acceptance.cpp and the golden
// memory CSV, plus LAPACK cross-checks through numpy/scipy).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

enum Status { OK = 0, INVALID_ARGUMENT = 1, SINGULAR = 2, MEMORY_CAP = 3, RANK_DEFICIENT = 5 };

struct InvalidArgument : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Singular : std::runtime_error {
  int64_t system;
  Singular(int64_t s, const std::string& w) : std::runtime_error(w), system(s) {}
};
struct MemCap : std::runtime_error {
  uint64_t required, cap;
  MemCap(uint64_t r, uint64_t c, const std::string& w) : std::runtime_error(w), required(r), cap(c) {}
};

void require(bool cond, const std::string& msg) {
  if (!cond) throw InvalidArgument(msg);
}

template <typename S>
bool all_finite(const S* p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

template <typename S>
void require_finite(const S* p, size_t n, const char* name) {
  if (!all_finite(p, n)) throw InvalidArgument(std::string(name) + " contains non-finite entries");
}

// ---------------------------------------------------------------------------
// Dense partial-pivot LU on a row-major n x n matrix, in place.
// Mirrors Eigen::PartialPivLU as used at solver.hpp:158: pivot = first index
// of the largest |entry| in the column; a column whose largest entry is zero
// is left untouched (no division) and shows up as a zero on U's diagonal.
// ---------------------------------------------------------------------------
template <typename S>
struct LU {
  S* a;
  int n;
  std::vector<int> perm;  // row i of P*A is row perm[i] of A

  LU(S* a_, int n_) : a(a_), n(n_), perm(n_) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    std::vector<int> rowpos(n);
    for (int j = 0; j < n; ++j) {
      int piv = j;
      S best = std::abs(a[(size_t)j * n + j]);
      for (int r = j + 1; r < n; ++r) {
        const S v = std::abs(a[(size_t)r * n + j]);
        if (v > best) {
          best = v;
          piv = r;
        }
      }
      if (best != S(0)) {
        if (piv != j) {
          for (int c = 0; c < n; ++c) std::swap(a[(size_t)j * n + c], a[(size_t)piv * n + c]);
          std::swap(perm[j], perm[piv]);
        }
        const S inv = S(1) / a[(size_t)j * n + j];
        for (int r = j + 1; r < n; ++r) a[(size_t)r * n + j] *= inv;
      }
      for (int r = j + 1; r < n; ++r) {
        const S l = a[(size_t)r * n + j];
        if (l == S(0)) continue;
        S* rowr = a + (size_t)r * n;
        const S* rowj = a + (size_t)j * n;
        for (int c = j + 1; c < n; ++c) rowr[c] -= l * rowj[c];
      }
    }
  }

  bool has_zero_pivot() const {
    for (int i = 0; i < n; ++i)
      if (a[(size_t)i * n + i] == S(0)) return true;
    return false;
  }

  // x = A^{-1} b
  void solve(const S* b, S* x) const {
    std::vector<S> y(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i) {
      S s = y[i];
      const S* row = a + (size_t)i * n;
      for (int c = 0; c < i; ++c) s -= row[c] * y[c];
      y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      S s = y[i];
      const S* row = a + (size_t)i * n;
      for (int c = i + 1; c < n; ++c) s -= row[c] * y[c];
      y[i] = s / row[i];
    }
    for (int i = 0; i < n; ++i) x[i] = y[i];
  }

  // x = A^{-T} b   (A = P^T L U  =>  A^T = U^T L^T P)
  void solve_transposed(const S* b, S* x) const {
    std::vector<S> z(b, b + n);
    for (int i = 0; i < n; ++i) {  // U^T z = b (lower triangular, non-unit)
      S s = z[i];
      for (int c = 0; c < i; ++c) s -= a[(size_t)c * n + i] * z[c];
      z[i] = s / a[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {  // L^T w = z (unit upper)
      S s = z[i];
      for (int c = i + 1; c < n; ++c) s -= a[(size_t)c * n + i] * z[c];
      z[i] = s;
    }
    for (int i = 0; i < n; ++i) x[perm[i]] = z[i];
  }
};

template <typename S>
S l1(const std::vector<S>& v) {
  S s = 0;
  for (S e : v) s += std::abs(e);
  return s;
}

// Hager (1984) / Higham (1988) lower bound on ||A^{-1}||_1 from an existing
// factorization — the estimator Eigen's PartialPivLU::rcond() uses
// (solver.hpp:165).  At most 4 gradient steps, then Higham's alternating
// vector as an independent bound.
template <typename S>
S inverse_l1_norm_estimate(const LU<S>& lu) {
  const int n = lu.n;
  if (n == 0) return S(0);
  std::vector<S> v(n, S(1) / S(n)), tmp(n), sign(n), old_sign;
  lu.solve(v.data(), tmp.data());
  v = tmp;
  S lower = l1(v);
  if (n == 1) return lower;
  S old_lower = lower;
  int vmax = -1, old_vmax = -1;
  for (int it = 0; it < 4; ++it) {
    for (int i = 0; i < n; ++i) sign[i] = v[i] < S(0) ? S(-1) : S(1);
    if (it > 0 && sign == old_sign) break;
    lu.solve_transposed(sign.data(), tmp.data());
    v = tmp;
    S best = -1;
    for (int i = 0; i < n; ++i) {
      const S m = std::abs(v[i]);
      if (m > best) {
        best = m;
        vmax = i;
      }
    }
    if (vmax == old_vmax) break;
    std::vector<S> e(n, S(0));
    e[vmax] = S(1);
    lu.solve(e.data(), tmp.data());
    v = tmp;
    lower = l1(v);
    if (lower <= old_lower) break;
    old_sign = sign;
    old_vmax = vmax;
    old_lower = lower;
  }
  S alt = S(1);
  for (int i = 0; i < n; ++i) {
    v[i] = alt * (S(1) + S(i) / S(n - 1));
    alt = -alt;
  }
  lu.solve(v.data(), tmp.data());
  const S alt_bound = (S(2) * l1(tmp)) / (S(3) * S(n));
  return std::max(lower, alt_bound);
}

template <typename S>
S format_rcond(S matrix_l1, const LU<S>& lu) {
  if (matrix_l1 == S(0)) return S(0);
  if (lu.n == 1) return S(1);
  const S inv = inverse_l1_norm_estimate(lu);
  return inv == S(0) ? S(0) : (S(1) / inv) / matrix_l1;
}

template <typename S>
std::string num(S v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.9g", (double)v);
  return buf;
}

// solver.hpp:147-170: factor lhs in place and overwrite rhs with the solution.
template <typename S>
void factor_solve_inplace(S* lhs, S* rhs, int k, int64_t system, S rcond_threshold) {
  S l1norm = 0;
  for (int c = 0; c < k; ++c) {
    S s = 0;
    for (int r = 0; r < k; ++r) s += std::abs(lhs[(size_t)r * k + c]);
    l1norm = std::max(l1norm, s);
  }
  LU<S> lu(lhs, k);
  auto fail = [&](const char* why, S value) {
    throw Singular(system, "row system " + std::to_string(system) + " is numerically singular (" +
                               why + " " + num(value) + ")");
  };
  if (lu.has_zero_pivot()) fail("zero pivot,", S(0));
  const S rcond = format_rcond(l1norm, lu);
  if (!(rcond >= rcond_threshold)) fail("rcond estimate", rcond);
  std::vector<S> x(k);
  lu.solve(rhs, x.data());
  if (!all_finite(x.data(), x.size())) fail("non-finite solution, rcond estimate", rcond);
  std::copy(x.begin(), x.end(), rhs);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

struct oracle_opts {
  double ridge;
  double rcond_threshold;  // <0: reference default (1e-14 f64 / 1e-7 f32), solver.hpp:18-27
  int has_cap;
  uint64_t cap_bytes;
  unsigned threads;
  int inject_fault;
};

struct oracle_report {
  double max_residual;
  double wall_seconds;
  uint64_t peak_extra_bytes;
  int64_t failing_system;
  uint64_t required_bytes;
  uint64_t cap_bytes;
  char message[256];
};

}  // extern "C"

namespace {

void set_msg(oracle_report* rep, const char* m) {
  if (!rep) return;
  std::snprintf(rep->message, sizeof rep->message, "%s", m);
}

template <typename S>
S default_rcond() {
  return sizeof(S) == sizeof(double) ? S(1e-14) : S(1e-7);
}

// solver.hpp:132-145
template <typename S>
void validate_problems(int64_t b, int k, const S* gram, const S* rhs, const S* mask, S lambda) {
  require(b >= 1, "no problems to solve");
  require(k >= 1, "problem is empty");
  require(lambda >= S(0), "lambda must be non-negative");
  const size_t kk = (size_t)k * k;
  for (int64_t q = 0; q < b; ++q) {
    const S* m = mask + q * kk;
    for (size_t e = 0; e < kk; ++e) require(m[e] >= S(0), "penalty mask entries must be non-negative");
    require_finite(gram + q * kk, kk, "gram");
    require_finite(rhs + q * kk, kk, "rhs");
    require_finite(m, kk, "mask");
  }
}

// ||C*G + lambda*(M .* C) - R||_F  (solver.hpp:212-215), accumulated in S like Eigen.
template <typename S>
S residual_norm(int k, const S* C, const S* G, const S* R, const S* M, S lambda) {
  S acc = 0;
  for (int i = 0; i < k; ++i) {
    for (int j = 0; j < k; ++j) {
      S s = 0;
      for (int t = 0; t < k; ++t) s += C[(size_t)i * k + t] * G[(size_t)t * k + j];
      const size_t e = (size_t)i * k + j;
      const S v = s + lambda * (M[e] * C[e]) - R[e];
      acc += v * v;
    }
  }
  return std::sqrt(acc);
}

template <typename S>
int solve_impl(int route, int64_t b, int k, const S* gram, const S* rhs, const S* mask, S lambda,
               const oracle_opts* o, S* C, oracle_report* rep) {
  oracle_opts opts{0.0, -1.0, 0, 0, 0, 0};
  if (o) opts = *o;
  const S ridge = (S)opts.ridge;
  const S rthr = opts.rcond_threshold < 0 ? default_rcond<S>() : (S)opts.rcond_threshold;
  if (rep) {
    std::memset(rep, 0, sizeof *rep);
    rep->failing_system = -1;
  }
  try {
    validate_problems(b, k, gram, rhs, mask, lambda);
    const size_t kk = (size_t)k * k;
    const size_t nsys = (size_t)b * k;
    std::chrono::steady_clock::time_point t0;
    if (route == 0) {
      // solver.hpp:174-218 — serial, i outer, q inner, one reused lhs.
      if (rep) rep->peak_extra_bytes = (uint64_t)b * kk * sizeof(S);
      t0 = std::chrono::steady_clock::now();
      std::vector<S> lhs(kk), r(k);
      for (int i = 0; i < k; ++i) {
        for (int64_t q = 0; q < b; ++q) {
          std::copy(gram + q * kk, gram + (q + 1) * kk, lhs.begin());
          const S* m = mask + q * kk + (size_t)i * k;
          for (int c = 0; c < k; ++c) lhs[(size_t)c * k + c] += lambda * m[c];
          if (ridge != S(0))
            for (int c = 0; c < k; ++c) lhs[(size_t)c * k + c] += ridge;
          std::copy(rhs + q * kk + (size_t)i * k, rhs + q * kk + (size_t)(i + 1) * k, r.begin());
          factor_solve_inplace<S>(lhs.data(), r.data(), k, (int64_t)q * k + i, rthr);
          std::copy(r.begin(), r.end(), C + q * kk + (size_t)i * k);
        }
      }
    } else {
      // solver.hpp:220-322 — [b*k, k, k] arena, cap checked before allocating.
      const uint64_t lhs_bytes = (uint64_t)nsys * kk * sizeof(S);
      if (opts.has_cap && lhs_bytes > opts.cap_bytes) {
        throw MemCap(lhs_bytes, opts.cap_bytes,
                     "batched left-hand-side tensor needs " + std::to_string(lhs_bytes) +
                         " bytes, above the cap of " + std::to_string(opts.cap_bytes));
      }
      if (rep) rep->peak_extra_bytes = lhs_bytes;
      t0 = std::chrono::steady_clock::now();
      std::vector<S> arena(nsys * kk), arhs(nsys * k);
      auto process = [&](size_t lo, size_t hi) {
        for (size_t s = lo; s < hi; ++s) {
          const size_t q = s / k;
          const int i = (int)(s % k);
          S* block = arena.data() + s * kk;
          std::copy(gram + q * kk, gram + (q + 1) * kk, block);
          const S* m = mask + q * kk + (size_t)i * k;
          for (int c = 0; c < k; ++c) block[(size_t)c * k + c] += lambda * m[c];
          if (ridge != S(0))
            for (int c = 0; c < k; ++c) block[(size_t)c * k + c] += ridge;
          if (opts.inject_fault && s == 0) {  // solver.hpp:269-273
            int worst = 0;
            S best = -1;
            for (int c = 0; c < k; ++c)
              if (std::abs(block[c]) > best) {
                best = std::abs(block[c]);
                worst = c;
              }
            block[worst] = -block[worst];
          }
          S* r = arhs.data() + s * k;
          std::copy(rhs + q * kk + (size_t)i * k, rhs + q * kk + (size_t)(i + 1) * k, r);
          factor_solve_inplace<S>(block, r, k, (int64_t)s, rthr);
          std::copy(r, r + k, C + q * kk + (size_t)i * k);
        }
      };
      unsigned threads = opts.threads ? opts.threads : std::thread::hardware_concurrency();
      if (threads == 0) threads = 1;
      threads = (unsigned)std::min<size_t>(threads, nsys);
      if (threads <= 1) {
        process(0, nsys);
      } else {
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errors(threads);
        const size_t chunk = (nsys + threads - 1) / threads;
        for (unsigned t = 0; t < threads; ++t) {
          const size_t lo = std::min<size_t>(t * chunk, nsys);
          const size_t hi = std::min<size_t>(lo + chunk, nsys);
          pool.emplace_back([&, t, lo, hi] {
            try {
              process(lo, hi);
            } catch (...) {
              errors[t] = std::current_exception();
            }
          });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errors)
          if (e) std::rethrow_exception(e);  // lowest failing system (solver.hpp:305-309)
      }
    }
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rep) {
      rep->wall_seconds = wall;
      S worst = 0;
      for (int64_t q = 0; q < b; ++q)
        worst = std::max(worst, residual_norm<S>(k, C + q * kk, gram + q * kk, rhs + q * kk,
                                                 mask + q * kk, lambda));
      rep->max_residual = (double)worst;
    }
    return OK;
  } catch (const InvalidArgument& e) {
    set_msg(rep, e.what());
    return INVALID_ARGUMENT;
  } catch (const Singular& e) {
    if (rep) rep->failing_system = e.system;
    set_msg(rep, e.what());
    return SINGULAR;
  } catch (const MemCap& e) {
    if (rep) {
      rep->required_bytes = e.required;
      rep->cap_bytes = e.cap;
    }
    set_msg(rep, e.what());
    return MEMORY_CAP;
  }
}

// solver.hpp:368-444: the k^2 x k^2 system for vec(C) (column-major vec).
// Dense LU with partial pivoting replaces Eigen::SparseLU; the assembled
// system and the consistency check are the reference's.
template <typename S>
int full_impl(int k, const S* gram, const S* rhs, const S* mask, S lambda, S ridge, S* C,
              oracle_report* rep) {
  if (rep) {
    std::memset(rep, 0, sizeof *rep);
    rep->failing_system = -1;
  }
  try {
    validate_problems<S>(1, k, gram, rhs, mask, lambda);
    if (k > 64)
      throw InvalidArgument("full oracle is guarded to k <= 64 (got k = " + std::to_string(k) +
                            "); the assembled system has k^4 entries");
    const int n = k * k;
    std::vector<S> sys((size_t)n * n, S(0)), v(n), x(n);
    for (int j = 0; j < k; ++j)
      for (int i = 0; i < k; ++i) {
        const int row = i + j * k;
        for (int q = 0; q < k; ++q) sys[(size_t)row * n + i + q * k] += gram[(size_t)q * k + j];
        sys[(size_t)row * n + row] += lambda * mask[(size_t)i * k + j] + ridge;
        v[row] = rhs[(size_t)i * k + j];
      }
    std::vector<S> copy = sys;
    S amax = 0;
    for (S e : sys) amax = std::max(amax, std::abs(e));
    LU<S> lu(sys.data(), n);
    // SparseLU reports a numerically zero pivot as a failed factorization; the
    // dense restatement uses the standard relative test |u_jj| <= n eps max|A|.
    const S ptol = S(n) * std::numeric_limits<S>::epsilon() * amax;
    bool tiny = lu.has_zero_pivot();
    for (int i = 0; i < n && !tiny; ++i) tiny = std::abs(sys[(size_t)i * n + i]) <= ptol;
    if (tiny) throw Singular(0, "k^2 x k^2 oracle system is numerically singular");
    lu.solve(v.data(), x.data());
    if (!all_finite(x.data(), x.size()))
      throw Singular(0, "k^2 x k^2 oracle solve produced non-finite values");
    S rn = 0, vn = 0;
    for (int r = 0; r < n; ++r) {
      S s = 0;
      for (int c = 0; c < n; ++c) s += copy[(size_t)r * n + c] * x[c];
      rn += (s - v[r]) * (s - v[r]);
      vn += v[r] * v[r];
    }
    const S consistency = std::sqrt(rn) / (S(1) + std::sqrt(vn));
    const S tol = sizeof(S) == sizeof(double) ? S(1e-7) : S(1e-2);
    if (!(consistency <= tol))
      throw Singular(0, "k^2 x k^2 oracle solution is inconsistent (relative residual " +
                            num(consistency) + "); the system is numerically singular");
    for (int j = 0; j < k; ++j)
      for (int i = 0; i < k; ++i) C[(size_t)i * k + j] = x[i + j * k];
    return OK;
  } catch (const InvalidArgument& e) {
    set_msg(rep, e.what());
    return INVALID_ARGUMENT;
  } catch (const Singular& e) {
    if (rep) rep->failing_system = e.system;
    set_msg(rep, e.what());
    return SINGULAR;
  }
}

// masks.hpp:13-89
template <typename S>
int mask_impl(int kind, int k, const S* ev1, const S* ev2, S sigma, S* out, char* msg) {
  try {
    require(k >= 1, "eigenvalue vectors must be non-empty");
    require_finite(ev1, k, "ev1");
    require_finite(ev2, k, "ev2");
    for (int i = 0; i < k; ++i)
      require(ev1[i] >= S(0) && ev2[i] >= S(0), "eigenvalues must be non-negative");
    if (kind == 0) {
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
          const S d = ev2[i] - ev1[j];
          out[(size_t)i * k + j] = d * d;
        }
      return OK;
    }
    require(sigma > S(0), "sigma must be positive");
    S ev_max = ev1[0];
    for (int i = 0; i < k; ++i) ev_max = std::max(ev_max, std::max(ev1[i], ev2[i]));
    require(ev_max > S(0), "resolvent mask needs a non-zero spectrum to normalize by");
    const S s2 = sigma * sigma;
    std::vector<S> re1(k), im1(k), re2(k), im2(k);
    for (int j = 0; j < k; ++j) {
      const S mu1 = ev1[j] / ev_max, mu2 = ev2[j] / ev_max;
      re1[j] = mu1 / (mu1 * mu1 + s2);
      im1[j] = sigma / (mu1 * mu1 + s2);
      re2[j] = mu2 / (mu2 * mu2 + s2);
      im2[j] = sigma / (mu2 * mu2 + s2);
    }
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {
        const S re = re2[i] - re1[j], im = im2[i] - im1[j];
        out[(size_t)i * k + j] = re * re + im * im;
      }
    return OK;
  } catch (const InvalidArgument& e) {
    if (msg) std::snprintf(msg, 256, "%s", e.what());
    return INVALID_ARGUMENT;
  }
}

}  // namespace

extern "C" {

int oracle_solve_f64(int route, int64_t b, int k, const double* gram, const double* rhs,
                     const double* mask, double lambda, const oracle_opts* opts, double* C,
                     oracle_report* rep) {
  return solve_impl<double>(route, b, k, gram, rhs, mask, lambda, opts, C, rep);
}

int oracle_solve_f32(int route, int64_t b, int k, const float* gram, const float* rhs,
                     const float* mask, float lambda, const oracle_opts* opts, float* C,
                     oracle_report* rep) {
  return solve_impl<float>(route, b, k, gram, rhs, mask, lambda, opts, C, rep);
}

int oracle_solve_full_f64(int k, const double* gram, const double* rhs, const double* mask,
                          double lambda, double ridge, double* C, oracle_report* rep) {
  return full_impl<double>(k, gram, rhs, mask, lambda, ridge, C, rep);
}

int oracle_solve_full_f32(int k, const float* gram, const float* rhs, const float* mask,
                          float lambda, float ridge, float* C, oracle_report* rep) {
  return full_impl<float>(k, gram, rhs, mask, lambda, ridge, C, rep);
}

int oracle_mask_f64(int kind, int k, const double* ev1, const double* ev2, double sigma,
                    double* out, char* msg) {
  return mask_impl<double>(kind, k, ev1, ev2, sigma, out, msg);
}

int oracle_mask_f32(int kind, int k, const float* ev1, const float* ev2, float sigma, float* out,
                    char* msg) {
  return mask_impl<float>(kind, k, ev1, ev2, sigma, out, msg);
}

// solver.hpp:95-103: gram = A*A^T, rhs = B*A^T (A, B: k x d row-major).
// Accumulates in double for both precisions (checker-side ground truth).
int oracle_normal_equations(int k, int d, const double* a, const double* b, double* gram,
                            double* rhs) {
  if (k < 1 || d < 1) return INVALID_ARGUMENT;
  if (!all_finite(a, (size_t)k * d) || !all_finite(b, (size_t)k * d)) return INVALID_ARGUMENT;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      double g = 0, r = 0;
      for (int t = 0; t < d; ++t) {
        g += a[(size_t)i * d + t] * a[(size_t)j * d + t];
        r += b[(size_t)i * d + t] * a[(size_t)j * d + t];
      }
      gram[(size_t)i * k + j] = g;
      rhs[(size_t)i * k + j] = r;
    }
  return OK;
}

// North_star projection: out[k x d] = Phi^T * diag(mass) * F,
// Phi: n x k row-major, F: n x d row-major.  Double accumulation.
int oracle_project_mass(int64_t n, int k, int d, const double* phi, const double* mass,
                        const double* F, double* out) {
  if (n < 1 || k < 1 || d < 1) return INVALID_ARGUMENT;
  std::fill(out, out + (size_t)k * d, 0.0);
  std::vector<double> row(d);
  for (int64_t v = 0; v < n; ++v) {
    const double m = mass[v];
    for (int t = 0; t < d; ++t) row[t] = m * F[(size_t)v * d + t];
    for (int i = 0; i < k; ++i) {
      const double p = phi[(size_t)v * k + i];
      double* o = out + (size_t)i * d;
      for (int t = 0; t < d; ++t) o[t] += p * row[t];
    }
  }
  return OK;
}

// project_to_spectral (spectral.hpp:47-93) restated in double: pinv(basis) * F.
// Normal equations when well conditioned (eigenvalues of B^T B by cyclic Jacobi,
// cond = sqrt(ev_max / ev_min) <= threshold, then Cholesky); otherwise the
// complete orthogonal decomposition's role is played by Householder QR with
// column pivoting (the factor Eigen's COD is built on): rank = #{|R_ii| >
// eps * min(n,k) * |R_00|} (Eigen's default ColPivHouseholderQR threshold);
// rank < k -> RANK_DEFICIENT (rank in *rank_out); full rank -> least squares.
// basis: n x k, features: n x d (row-major); out: k x d.  Returns 0 / 1 / 5.
int oracle_project_pinv(int64_t n, int k, int d, const double* basis, const double* F, double cond_thr,
                        double* out, int* rank_out, char* msg) {
  auto fail = [&](int code, const std::string& m) {
    if (msg) std::snprintf(msg, 256, "%s", m.c_str());
    return code;
  };
  if (n < 1 || k < 1) return fail(INVALID_ARGUMENT, "basis must be non-empty");
  if (d < 1) return fail(INVALID_ARGUMENT, "features must be non-empty");
  for (size_t e = 0; e < (size_t)n * k; ++e)
    if (!std::isfinite(basis[e])) return fail(INVALID_ARGUMENT, "basis contains non-finite entries");
  for (size_t e = 0; e < (size_t)n * d; ++e)
    if (!std::isfinite(F[e])) return fail(INVALID_ARGUMENT, "features contains non-finite entries");
  if (rank_out) *rank_out = k;
  auto rank_revealing = [&]() -> int {
    // Householder QR with column pivoting of the n x k basis (column-major copy)
    std::vector<double> a((size_t)n * k);
    for (int64_t v = 0; v < n; ++v)
      for (int j = 0; j < k; ++j) a[(size_t)j * n + v] = basis[(size_t)v * k + j];
    std::vector<int> perm(k);
    for (int j = 0; j < k; ++j) perm[j] = j;
    std::vector<double> cn(k), tau(k, 0.0);
    for (int j = 0; j < k; ++j) {
      double s2 = 0;
      for (int64_t v = 0; v < n; ++v) s2 += a[(size_t)j * n + v] * a[(size_t)j * n + v];
      cn[j] = s2;
    }
    const int m = (int)std::min<int64_t>(n, k);
    for (int i = 0; i < m; ++i) {
      int best = i;
      for (int j = i + 1; j < k; ++j)
        if (cn[j] > cn[best]) best = j;
      if (best != i) {
        for (int64_t v = 0; v < n; ++v) std::swap(a[(size_t)i * n + v], a[(size_t)best * n + v]);
        std::swap(cn[i], cn[best]);
        std::swap(perm[i], perm[best]);
      }
      double* col = a.data() + (size_t)i * n;
      double nrm = 0;
      for (int64_t v = i; v < n; ++v) nrm += col[v] * col[v];
      nrm = std::sqrt(nrm);
      if (nrm == 0.0) continue;
      const double alpha = col[i] > 0 ? -nrm : nrm;
      const double v0 = col[i] - alpha;
      for (int64_t v = i + 1; v < n; ++v) col[v] /= v0;
      tau[i] = -v0 / alpha;
      col[i] = alpha;
      for (int j = i + 1; j < k; ++j) {
        double* cj = a.data() + (size_t)j * n;
        double w = cj[i];
        for (int64_t v = i + 1; v < n; ++v) w += col[v] * cj[v];
        w *= tau[i];
        cj[i] -= w;
        for (int64_t v = i + 1; v < n; ++v) cj[v] -= w * col[v];
        double s2 = 0;
        for (int64_t v = i + 1; v < n; ++v) s2 += cj[v] * cj[v];
        cn[j] = s2;
      }
    }
    const double r00 = m > 0 ? std::abs(a[0]) : 0.0;
    const double thr = std::numeric_limits<double>::epsilon() * (double)m * r00;
    int rank = 0;
    for (int i = 0; i < m; ++i)
      if (std::abs(a[(size_t)i * n + i]) > thr) ++rank;
    if (rank_out) *rank_out = rank;
    if (rank < k)
      return fail(RANK_DEFICIENT, "basis is rank deficient: rank " + std::to_string(rank) + " < " +
                                      std::to_string(k) + " columns");
    // full rank: x = P R^{-1} (Q^T F)
    std::vector<double> qf((size_t)n * d);
    for (int64_t v = 0; v < n; ++v)
      for (int t = 0; t < d; ++t) qf[(size_t)t * n + v] = F[(size_t)v * d + t];
    for (int i = 0; i < k; ++i) {
      const double* col = a.data() + (size_t)i * n;
      for (int t = 0; t < d; ++t) {
        double* f = qf.data() + (size_t)t * n;
        double w = f[i];
        for (int64_t v = i + 1; v < n; ++v) w += col[v] * f[v];
        w *= tau[i];
        f[i] -= w;
        for (int64_t v = i + 1; v < n; ++v) f[v] -= w * col[v];
      }
    }
    for (int t = 0; t < d; ++t) {
      std::vector<double> z(k);
      for (int i = k - 1; i >= 0; --i) {
        double sacc = qf[(size_t)t * n + i];
        for (int j = i + 1; j < k; ++j) sacc -= a[(size_t)j * n + i] * z[j];
        z[i] = sacc / a[(size_t)i * n + i];
      }
      for (int i = 0; i < k; ++i) out[(size_t)perm[i] * d + t] = z[i];
    }
    return OK;
  };
  if (n < k) return rank_revealing();
  // gram = B^T B and its eigenvalues (cyclic Jacobi)
  std::vector<double> g((size_t)k * k, 0.0);
  for (int64_t v = 0; v < n; ++v)
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) g[(size_t)i * k + j] += basis[(size_t)v * k + i] * basis[(size_t)v * k + j];
  std::vector<double> e(g);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0;
    for (int i = 0; i < k; ++i)
      for (int j = i + 1; j < k; ++j) off += e[(size_t)i * k + j] * e[(size_t)i * k + j];
    if (off < 1e-30) break;
    for (int p2 = 0; p2 < k; ++p2)
      for (int q2 = p2 + 1; q2 < k; ++q2) {
        const double apq = e[(size_t)p2 * k + q2];
        if (apq == 0.0) continue;
        const double app = e[(size_t)p2 * k + p2], aqq = e[(size_t)q2 * k + q2];
        const double theta = (aqq - app) / (2 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1));
        const double c = 1 / std::sqrt(t * t + 1), sn = t * c;
        for (int r = 0; r < k; ++r) {
          const double arp = e[(size_t)r * k + p2], arq = e[(size_t)r * k + q2];
          e[(size_t)r * k + p2] = c * arp - sn * arq;
          e[(size_t)r * k + q2] = sn * arp + c * arq;
        }
        for (int r = 0; r < k; ++r) {
          const double apr = e[(size_t)p2 * k + r], aqr = e[(size_t)q2 * k + r];
          e[(size_t)p2 * k + r] = c * apr - sn * aqr;
          e[(size_t)q2 * k + r] = sn * apr + c * aqr;
        }
      }
  }
  double ev_min = e[0], ev_max = e[0];
  for (int i = 1; i < k; ++i) {
    ev_min = std::min(ev_min, e[(size_t)i * k + i]);
    ev_max = std::max(ev_max, e[(size_t)i * k + i]);
  }
  if (!(ev_min > 0.0 && std::sqrt(ev_max / ev_min) <= cond_thr)) return rank_revealing();
  // LLT of the gram, then solve gram * X = B^T F
  std::vector<double> l(g);
  for (int j = 0; j < k; ++j) {
    double dj = l[(size_t)j * k + j];
    for (int t = 0; t < j; ++t) dj -= l[(size_t)j * k + t] * l[(size_t)j * k + t];
    if (!(dj > 0.0)) return rank_revealing();
    dj = std::sqrt(dj);
    l[(size_t)j * k + j] = dj;
    for (int i = j + 1; i < k; ++i) {
      double v = l[(size_t)i * k + j];
      for (int t = 0; t < j; ++t) v -= l[(size_t)i * k + t] * l[(size_t)j * k + t];
      l[(size_t)i * k + j] = v / dj;
    }
  }
  for (int t = 0; t < d; ++t) {
    std::vector<double> z(k);
    for (int i = 0; i < k; ++i) {
      double sacc = 0;
      for (int64_t v = 0; v < n; ++v) sacc += basis[(size_t)v * k + i] * F[(size_t)v * d + t];
      for (int j = 0; j < i; ++j) sacc -= l[(size_t)i * k + j] * z[j];
      z[i] = sacc / l[(size_t)i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
      double sacc = z[i];
      for (int j = i + 1; j < k; ++j) sacc -= l[(size_t)j * k + i] * z[j];
      z[i] = sacc / l[(size_t)i * k + i];
    }
    for (int i = 0; i < k; ++i) out[(size_t)i * d + t] = z[i];
  }
  return OK;
}

double oracle_residual_f64(int k, const double* C, const double* G, const double* R,
                           const double* M, double lambda) {
  return residual_norm<double>(k, C, G, R, M, lambda);
}

// spectral.hpp:95-115: ||C*A - B||_F^2 + lambda * sum M .* C^2
double oracle_energy_f64(int k, int d, const double* C, const double* a, const double* b,
                         const double* M, double lambda) {
  double data = 0, reg = 0;
  for (int i = 0; i < k; ++i)
    for (int t = 0; t < d; ++t) {
      double s = 0;
      for (int j = 0; j < k; ++j) s += C[(size_t)i * k + j] * a[(size_t)j * d + t];
      const double e = s - b[(size_t)i * d + t];
      data += e * e;
    }
  for (size_t e = 0; e < (size_t)k * k; ++e) reg += M[e] * C[e] * C[e];
  return data + lambda * reg;
}

// bench.hpp:52-93 — the reference synthetic instance, drawn with the same
// standard-library engines (std::seed_seq, std::mt19937_64,
// uniform_real_distribution(0.05, 1), normal_distribution(0, 1)) in the same
// order, so a libstdc++ build reproduces the reference's instances exactly.
int oracle_generate_instance(int k, int d, uint64_t seed, double* a, double* b, double* ev1,
                             double* ev2) {
  if (k < 1 || d < 1) return INVALID_ARGUMENT;
  std::seed_seq seq{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32),
                    static_cast<uint32_t>(k), static_cast<uint32_t>(d)};
  std::mt19937_64 rng(seq);
  std::uniform_real_distribution<double> increment(0.05, 1.0);
  std::normal_distribution<double> gauss(0.0, 1.0);
  auto spectrum = [&](double* ev) {
    ev[0] = 0.0;
    for (int i = 1; i < k; ++i) ev[i] = ev[i - 1] + increment(rng);
  };
  spectrum(ev1);
  spectrum(ev2);
  const double scale = 1.0 / std::sqrt(static_cast<double>(d));
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < d; ++j) a[(size_t)i * d + j] = gauss(rng) * scale;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < d; ++j) b[(size_t)i * d + j] = gauss(rng) * scale;
  return OK;
}

// test_solver.cpp:15-23 randn(rows, cols, seed) fixture helper.
void oracle_randn(int rows, int cols, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = gauss(rng);
}

unsigned oracle_hardware_threads(void) { return std::thread::hardware_concurrency(); }

// The reference's rcond of one assembled row system A (k x k, row-major):
// PartialPivLU + the Hager/Higham estimate, exactly what factor_solve_inplace
// compares with the threshold (solver.hpp:158-166).  -1 on an exact zero pivot.
double oracle_rcond_f64(int k, const double* a) {
  std::vector<double> m(a, a + (size_t)k * k);
  double l1norm = 0;
  for (int c = 0; c < k; ++c) {
    double s = 0;
    for (int r = 0; r < k; ++r) s += std::abs(m[(size_t)r * k + c]);
    l1norm = std::max(l1norm, s);
  }
  LU<double> lu(m.data(), k);
  if (lu.has_zero_pivot()) return -1.0;
  return format_rcond(l1norm, lu);
}
float oracle_rcond_f32(int k, const float* a) {
  std::vector<float> m(a, a + (size_t)k * k);
  float l1norm = 0;
  for (int c = 0; c < k; ++c) {
    float s = 0;
    for (int r = 0; r < k; ++r) s += std::abs(m[(size_t)r * k + c]);
    l1norm = std::max(l1norm, s);
  }
  LU<float> lu(m.data(), k);
  if (lu.has_zero_pivot()) return -1.f;
  return format_rcond(l1norm, lu);
}

}  // extern "C"
