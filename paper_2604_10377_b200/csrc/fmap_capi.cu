// libfmap_cuda — C ABI (include/fmap_cuda.h) over the sm_100a kernels.
//
// Error semantics follow the reference (solver.hpp:225-322, types.hpp):
//   * validation failures -> FMAP_INVALID_ARGUMENT, before any result is exposed
//   * memory cap          -> FMAP_MEMORY_CAP, before any allocation
//   * singular systems    -> FMAP_SINGULAR with the LOWEST failing global index
//   * no partial results on error (the caller's C buffer content is unspecified)
// There is no CPU fallback: every numeric result comes from a device kernel.
#include "../../include/fmap_cuda.h"
#include "fmap_kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace fmap;

struct fmap_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string last_error;
  // Two grow-only device arenas (BatchedWorkspace analogue, solver.hpp:86-93):
  // `arena` holds what an entry point stages (host copies, pipeline
  // intermediates), `scr` the solver's own scratch.  solve_core only ever grows
  // `scr`, so pointers an entry point carved out of `arena` stay valid.
  void* arena = nullptr;
  size_t arena_bytes = 0;
  void* scr = nullptr;
  size_t scr_bytes = 0;
  // control block: [0] fail_min (u64) | [8] rcond bits (u32) | [12] flags (u32) |
  // [16] systems whose rcond needed the exact Hager/Higham estimator (u32)
  unsigned char* d_ctrl = nullptr;
  unsigned char* h_ctrl = nullptr;  // pinned
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evf = nullptr;  // evf: factorization done
  unsigned last_exact = 0;     // systems of the last call that ran the exact rcond estimator
  double last_resmax = 0.0;    // max check_stationarity residual of the last call (control block)
  int64_t launches = 0;        // kernels launched by the last call
  std::string launch_names;    // their names, comma-separated (fmap_last_launches)
  int max_smem_optin = 0;
  int num_sms = 0;
  // host-buffer pipelining (fmap_solve_f32): second compute stream + copy stream
  cudaStream_t comp2 = nullptr, copy = nullptr, copy2 = nullptr;  // 2nd compute, H2D, D2H
  // start | done | per chunk (<= 16): G+M landed, R landed, solve done | H2D join | compute join
  cudaEvent_t cev[52] = {};
};

namespace {

constexpr unsigned long long kNoFail = ~0ull;

int set_err(fmap_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}

#define FMAP_CK(ctx, expr)                                                                   \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return set_err((ctx), FMAP_CUDA_ERROR,                                                 \
                     std::string(#expr) + ": " + cudaGetErrorString(_e));                    \
  } while (0)

unsigned long long* d_fail(fmap_ctx* c) { return reinterpret_cast<unsigned long long*>(c->d_ctrl); }
unsigned* d_rcond(fmap_ctx* c) { return reinterpret_cast<unsigned*>(c->d_ctrl + 8); }
unsigned* d_flags(fmap_ctx* c) { return reinterpret_cast<unsigned*>(c->d_ctrl + 12); }
unsigned* d_nexact(fmap_ctx* c) { return reinterpret_cast<unsigned*>(c->d_ctrl + 16); }
// max over pairs of the check_stationarity residual (fp64 bits; residuals are >= 0)
unsigned long long* d_resmax(fmap_ctx* c) { return reinterpret_cast<unsigned long long*>(c->d_ctrl + 24); }

// Grow-only device arena.  Growth drops the old contents (the stream is drained
// first, so no queued kernel still reads it): callers reserve BEFORE carving.
int grow(fmap_ctx* ctx, void** buf, size_t* have, size_t bytes) {
  if (bytes <= *have) return FMAP_OK;
  const size_t rounded = (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
  if (*buf) {
    FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
    FMAP_CK(ctx, cudaFree(*buf));
    *buf = nullptr;
    *have = 0;
  }
  FMAP_CK(ctx, cudaMalloc(buf, rounded));
  *have = rounded;
  return FMAP_OK;
}
int arena_reserve(fmap_ctx* ctx, size_t bytes) { return grow(ctx, &ctx->arena, &ctx->arena_bytes, bytes); }
int scratch_reserve(fmap_ctx* ctx, size_t bytes) { return grow(ctx, &ctx->scr, &ctx->scr_bytes, bytes); }

// Every entry point runs on the context's device and restores the caller's.
// Records the kernels one C-ABI call launches into its context.
struct LaunchScope {
  fmap_ctx* ctx;
  explicit LaunchScope(fmap_ctx* c) : ctx(c) { clear_launch_log(); }
  ~LaunchScope() {
    ctx->launches = launch_log_count();
    ctx->launch_names = launch_log();
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess || prev == dev) {
      prev = -1;
      return;
    }
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct Carve {
  char* base;
  size_t off = 0;
  // 256-byte aligned absolute addresses regardless of where `base` starts
  template <typename T>
  T* take(size_t n) {
    uintptr_t a = reinterpret_cast<uintptr_t>(base) + off;
    a = (a + 255) & ~uintptr_t(255);
    off = a - reinterpret_cast<uintptr_t>(base) + n * sizeof(T);
    return reinterpret_cast<T*>(a);
  }
};

size_t carve_size(std::initializer_list<size_t> bytes) {
  size_t off = 0;
  for (size_t b : bytes) off = ((off + 255) & ~size_t(255)) + b;
  return off + 256;
}

int reset_ctrl(fmap_ctx* ctx) {
  unsigned char init[32];
  const unsigned long long nf = kNoFail;
  const unsigned fmax = 0x7f7fffffu;  // FLT_MAX bits
  std::memset(init, 0, sizeof init);
  std::memcpy(init, &nf, 8);
  std::memcpy(init + 8, &fmax, 4);
  std::memcpy(ctx->h_ctrl, init, 32);
  FMAP_CK(ctx, cudaMemcpyAsync(ctx->d_ctrl, ctx->h_ctrl, 32, cudaMemcpyHostToDevice, ctx->stream));
  return FMAP_OK;
}

int read_ctrl(fmap_ctx* ctx, unsigned long long* fail, float* rcond, unsigned* flags) {
  FMAP_CK(ctx, cudaMemcpyAsync(ctx->h_ctrl + 32, ctx->d_ctrl, 32, cudaMemcpyDeviceToHost,
                               ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  std::memcpy(fail, ctx->h_ctrl + 32, 8);
  unsigned rb;
  std::memcpy(&rb, ctx->h_ctrl + 40, 4);
  std::memcpy(rcond, &rb, 4);
  std::memcpy(flags, ctx->h_ctrl + 44, 4);
  std::memcpy(&ctx->last_exact, ctx->h_ctrl + 48, 4);
  std::memcpy(&ctx->last_resmax, ctx->h_ctrl + 56, 8);
  return FMAP_OK;
}

void default_opts(fmap_solver_options* o) {
  o->ridge = 0.f;
  o->rcond_threshold = -1.f;
  o->has_memory_cap = 0;
  o->memory_cap_bytes = 0;
  o->threads = 0;
  o->inject_fault = 0;
  o->compute_residual = 1;
}

void init_report(fmap_report* r) {
  if (!r) return;
  std::memset(r, 0, sizeof *r);
  r->failing_system = -1;
}

std::string flags_message(unsigned f) {
  // validate_problem order (solver.hpp:140-144); NaN masks fail the >= 0 test first.
  if (f & 32u) return "resolvent mask needs a non-zero spectrum to normalize by";
  if (f & 16u) return "eigenvalues must be non-negative and finite";
  if (f & 8u) return "penalty mask entries must be non-negative";
  if (f & 1u) return "gram contains non-finite entries";
  if (f & 2u) return "rhs contains non-finite entries";
  if (f & 4u) return "mask contains non-finite entries";
  if (f & 64u)
    return "gram must be symmetric: the cuda route factors G + lambda*diag(m_i) by Cholesky and reads one "
           "triangle of G (G = A A^T from normal_equations always is)";
  return "invalid input";
}

int max_resolution(fmap_ctx* ctx) { return tc_max_resolution(ctx->max_smem_optin); }

// Core solve on device buffers. mask_mode 0: d_mask; 1/2: resolvent / commutativity
// mask rows generated inside the solver from the eigenvalues; 3/4: the same masks
// already materialized by the caller in d_mask from ev1/ev2 (the eigenvalues are
// validated instead of the mask, the solver reads the dense mask).
int solve_core(fmap_ctx* ctx, int64_t b, int64_t k, const float* G, const float* R,
               const float* M, const float* ev1, const float* ev2, int mask_mode, float sigma,
               float lambda, const fmap_solver_options* o, float* C, fmap_report* rep,
               bool device_validate, size_t host_staging_bytes) {
  fmap_solver_options opts;
  default_opts(&opts);
  if (o) opts = *o;
  init_report(rep);
  if (b < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "no problems to solve");
  if (k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "problem is empty");
  if (!(lambda >= 0.f)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "lambda must be non-negative");
  const int kmode = mask_mode >= 3 ? 0 : mask_mode;  // the solver kernel's mask source
  if ((mask_mode == 1 || mask_mode == 3) && !(sigma > 0.f))
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "sigma must be positive");
  if (!G || !R || !C || (kmode == 0 && !M) || (mask_mode != 0 && (!ev1 || !ev2)))
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "null buffer");
  const int kmax = max_resolution(ctx);
  if (k > kmax)
    return set_err(ctx, FMAP_INVALID_ARGUMENT,
                   "k = " + std::to_string(k) + " exceeds the tensor-memory solver limit " +
                       std::to_string(kmax) + " on this device");
  const size_t kk = (size_t)k * k;
  const size_t nsys = (size_t)b * k;
  const bool need_mask_scratch = opts.compute_residual && kmode != 0;
  const size_t res_partial = opts.compute_residual ? residual_partial_count(b, (int)k) : 0;
  const size_t tc_bytes = tc_scratch_bytes((int)k, (int64_t)nsys, ctx->num_sms);
  const size_t scratch = carve_size({res_partial * sizeof(double), (size_t)b * sizeof(double),
                                     need_mask_scratch ? (size_t)b * kk * sizeof(float) : 0,
                                     (size_t)k * sizeof(float), tc_bytes, (size_t)b * k * sizeof(float),
                                     mask_mode == 1 ? (size_t)b * sizeof(float) : 0});
  const uint64_t required = (uint64_t)scratch + host_staging_bytes;
  if (rep) rep->peak_extra_bytes = required;
  if (opts.has_memory_cap && required > opts.memory_cap_bytes) {
    if (rep) {
      rep->required_bytes = required;
      rep->cap_bytes = opts.memory_cap_bytes;
    }
    return set_err(ctx, FMAP_MEMORY_CAP,
                   "cuda route needs " + std::to_string(required) +
                       " bytes of device scratch, above the cap of " +
                       std::to_string(opts.memory_cap_bytes));
  }
  int st = scratch_reserve(ctx, scratch);
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->scr)};
  double* partial = cv.take<double>(res_partial);
  double* res_out = cv.take<double>((size_t)b);
  float* mask_scratch = cv.take<float>(need_mask_scratch ? (size_t)b * kk : 0);
  float* zrow = cv.take<float>((size_t)k);
  float* tc_scr = cv.take<float>(tc_bytes / sizeof(float));
  float* rowsum = cv.take<float>((size_t)b * k);
  float* evmax = cv.take<float>(mask_mode == 1 ? (size_t)b : 0);

  if ((st = reset_ctrl(ctx))) return st;
  if (device_validate) {
    if (mask_mode == 0) {
      FMAP_CK(ctx, launch_validate(G, R, M, (size_t)b * kk, d_flags(ctx), ctx->stream));
    } else {
      FMAP_CK(ctx, launch_validate(G, R, nullptr, (size_t)b * kk, d_flags(ctx), ctx->stream));
      FMAP_CK(ctx, launch_validate_ev(ev1, ev2, (size_t)b * k, d_flags(ctx), ctx->stream));
    }
  }
  // symmetry check + row 1-norms of G (rcond certificate input)
  FMAP_CK(ctx, launch_gram_check(G, b, (int)k, rowsum, d_flags(ctx), ctx->stream));
  // the resolvent mask's per-pair normaliser (masks.hpp:58-59), once per pair instead
  // of once per row system inside the solver; an all-zero spectrum is flagged
  if (mask_mode == 1 || mask_mode == 3)
    FMAP_CK(ctx, launch_ev_max_check(ev1, ev2, b, (int)k, d_flags(ctx), ctx->stream, mask_mode == 1 ? evmax : nullptr));

  SolveParams p{};
  p.gram = G;
  p.rhs = R;
  p.mask = M;
  p.ev1 = ev1;
  p.ev2 = ev2;
  p.ev_max = evmax;
  p.C = C;
  p.k = (int)k;
  p.K4 = ((int)k + 3) & ~3;
  p.Rp = p.K4 + 4;
  p.nsys = (int64_t)nsys;
  p.sys_offset = 0;
  p.lambda = lambda;
  p.ridge = opts.ridge;
  p.sigma = sigma;
  p.rcond_thr = opts.rcond_threshold < 0.f ? 1e-7f : opts.rcond_threshold;
  p.rhs_unit = -1;
  p.fail_min = d_fail(ctx);
  p.rcond_min_bits = d_rcond(ctx);
  p.flags = d_flags(ctx);
  p.rcond_exact = d_nexact(ctx);
  p.tc_scratch = tc_scr;
  p.gram_rowsum = rowsum;

  // debug: FMAP_TRACE_FILE=<path> dumps per-warp clock64 phase stamps of one block
  const char* trace_file = std::getenv("FMAP_TRACE_FILE");
  long long* d_trace = nullptr;
  if (trace_file) {
    FMAP_CK(ctx, cudaMalloc(&d_trace, 16 * 1024 * sizeof(long long)));
    FMAP_CK(ctx, cudaMemsetAsync(d_trace, 0, 16 * 1024 * sizeof(long long), ctx->stream));
    p.trace = d_trace;
    const char* tb = std::getenv("FMAP_TRACE_BLOCK");
    p.trace_block = tb ? std::atoi(tb) : 0;
  }
  if (const char* dbg = std::getenv("FMAP_DEBUG")) p.debug = std::atoi(dbg);  // timing experiments only
  FMAP_CK(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  FMAP_CK(ctx, launch_chol_solve(p, kmode, ctx->stream, 1));  // factorization
  FMAP_CK(ctx, cudaEventRecord(ctx->evf, ctx->stream));
  FMAP_CK(ctx, launch_chol_solve(p, kmode, ctx->stream, 2));  // back substitution + verdict
  if (d_trace) {
    std::vector<long long> h(16 * 1024);
    FMAP_CK(ctx, cudaMemcpyAsync(h.data(), d_trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (FILE* f = std::fopen(trace_file, "wb")) {
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
    cudaFree(d_trace);
    p.trace = nullptr;
  }
  if (opts.inject_fault) {
    // solver.hpp:269-273: negate the largest-|.| entry of row 0 of system 0's
    // assembled LHS.  Solved exactly as a rank-one update of the SPD system.
    std::vector<float> g0(k);
    float m00 = 0.f;
    FMAP_CK(ctx, cudaMemcpyAsync(g0.data(), G, k * sizeof(float), cudaMemcpyDeviceToHost,
                                 ctx->stream));
    if (kmode == 0) {
      FMAP_CK(ctx, cudaMemcpyAsync(&m00, M, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      std::vector<float> e1(k), e2(k);
      FMAP_CK(ctx, cudaMemcpyAsync(e1.data(), ev1, k * sizeof(float), cudaMemcpyDeviceToHost,
                                   ctx->stream));
      FMAP_CK(ctx, cudaMemcpyAsync(e2.data(), ev2, k * sizeof(float), cudaMemcpyDeviceToHost,
                                   ctx->stream));
      FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
      if (mask_mode == 1) {
        float emax = 0.f;
        for (int64_t c = 0; c < k; ++c) emax = std::max(emax, std::max(e1[c], e2[c]));
        const float s2 = sigma * sigma;
        const float mu1 = e1[0] / emax, mu2 = e2[0] / emax;
        const float re = mu2 / (mu2 * mu2 + s2) - mu1 / (mu1 * mu1 + s2);
        const float im = sigma / (mu2 * mu2 + s2) - sigma / (mu1 * mu1 + s2);
        m00 = re * re + im * im;
      } else {
        const float d = e2[0] - e1[0];
        m00 = d * d;
      }
    }
    FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
    g0[0] += lambda * m00 + opts.ridge;
    int w = 0;
    float best = -1.f;
    for (int64_t c = 0; c < k; ++c)
      if (std::fabs(g0[c]) > best) {
        best = std::fabs(g0[c]);
        w = (int)c;
      }
    const float alpha = -2.f * g0[w];
    SolveParams pz = p;
    pz.C = zrow;  // system 0 writes its row at offset 0
    pz.nsys = 1;
    pz.rhs_unit = 0;
    FMAP_CK(ctx, launch_chol_solve(pz, kmode, ctx->stream));
    FMAP_CK(ctx, launch_fault_combine(C, zrow, (int)k, w, alpha, d_fail(ctx), 0ull, ctx->stream));
  }
  FMAP_CK(ctx, cudaEventRecord(ctx->ev1, ctx->stream));

  if (opts.compute_residual) {
    const float* Muse = M;
    if (kmode != 0) {
      FMAP_CK(ctx, launch_mask(ev1, ev2, b, (int)k, mask_mode == 1 ? 1 : 0, sigma, mask_scratch,
                               ctx->stream));
      Muse = mask_scratch;
    }
    FMAP_CK(ctx, launch_residual(C, G, R, Muse, b, (int)k, lambda, partial, res_out, ctx->stream, d_resmax(ctx)));
  }

  unsigned long long fail;
  float rcond;
  unsigned flags;
  if ((st = read_ctrl(ctx, &fail, &rcond, &flags))) return st;
  float ms = 0.f, fms = 0.f;
  FMAP_CK(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  FMAP_CK(ctx, cudaEventElapsedTime(&fms, ctx->ev0, ctx->evf));
  if (rep) {
    rep->wall_seconds = ms * 1e-3;
    rep->factor_seconds = fms * 1e-3;
    rep->min_rcond = rcond;
    rep->rcond_exact_systems = ctx->last_exact;
  }
  if (flags) return set_err(ctx, FMAP_INVALID_ARGUMENT, flags_message(flags));
  if (fail != kNoFail) {
    if (rep) rep->failing_system = (int64_t)fail;
    return set_err(ctx, FMAP_SINGULAR,
                   "row system " + std::to_string(fail) +
                       " is numerically singular (Cholesky pivot / rcond estimate / non-finite "
                       "solution)");
  }
  if (opts.compute_residual && rep) rep->max_residual = ctx->last_resmax;  // read with the control block
  ctx->last_error.clear();
  return FMAP_OK;
}

// Host-buffer solve with the copies pipelined against the solver (the headline e2e
// path): the batch is cut into pair chunks; every chunk's H2D is queued up front on
// one copy stream (it runs ahead of the solver: 0.6 ms of copies vs 2.3 ms of solve
// at cfg2), each chunk is validated and solved as soon as its inputs have landed,
// chunks alternate between two compute streams (each with its own L scratch) so one
// chunk's tail overlaps the next chunk's start, and each chunk's D2H runs on a
// second copy stream (the other direction's copy engine) right after its solve.
// Same checks as solve_core (device validation, lowest failing index); on any error
// C_out is zero-filled, so no partial result is exposed.  Used when no fault
// injection is requested; the residual (check_stationarity) runs after the last chunk.
int solve_host_pipelined(fmap_ctx* ctx, int64_t b, int64_t k, const float* gram, const float* rhs,
                         const float* mask, float lambda, const fmap_solver_options& opts, float* C_out,
                         fmap_report* rep, int nchunk) {
  const size_t kk = (size_t)k * k;
  const size_t bytes = (size_t)b * kk * sizeof(float);
  // chunk boundaries: nchunk > 0 -> equal chunks; 0 -> weighted 2,5,6,3 sixteenths of
  // the batch (b = 64: 8, 20, 24, 12 pairs): the first chunk's G + M copy and the last
  // chunk's D2H are the only copies not hidden behind a solve, so those chunks are
  // small, while every extra chunk boundary costs ~30 us of solver tail
  // (tools/e2e_probe.py at cfg2: 2.19 ms vs 2.23 ms for 4 equal chunks, 2.27 for 6)
  std::vector<int64_t> cq0, cnq;
  if (nchunk <= 0) {
    int cum[17] = {0, 2, 7, 13, 16};
    int nw = 4;
    if (const char* w = std::getenv("FMAP_PIPELINE_W")) {  // experiments: weights "2,5,5,4" (sum 16)
      nw = 0;
      for (const char* c = w; *c && nw < 16;) {
        cum[nw + 1] = cum[nw] + std::atoi(c);
        ++nw;
        while (*c && *c != ',') ++c;
        if (*c == ',') ++c;
      }
    }
    for (int c = 0; c < nw; ++c) {
      const int64_t lo = b * cum[c] / cum[nw], hi = b * cum[c + 1] / cum[nw];
      if (hi > lo) {
        cq0.push_back(lo);
        cnq.push_back(hi - lo);
      }
    }
  } else {
    const int64_t cbq = (b + nchunk - 1) / nchunk;
    for (int64_t q = 0; q < b; q += cbq) {
      cq0.push_back(q);
      cnq.push_back(std::min<int64_t>(cbq, b - q));
    }
  }
  nchunk = (int)cq0.size();
  int64_t cb = 0;
  for (int64_t v : cnq) cb = std::max(cb, v);
  const int64_t csys = cb * k;
  const size_t tcb = tc_scratch_bytes((int)k, csys, ctx->num_sms);
  const size_t npart = opts.compute_residual ? residual_partial_count(b, (int)k) : 0;
  const size_t staging = carve_size({bytes, bytes, bytes, bytes, tcb, tcb, (size_t)b * k * sizeof(float),
                                     npart * sizeof(double), opts.compute_residual ? (size_t)b * sizeof(double) : 0});
  if (rep) rep->peak_extra_bytes = staging;
  if (opts.has_memory_cap && staging > opts.memory_cap_bytes) {
    if (rep) {
      rep->required_bytes = staging;
      rep->cap_bytes = opts.memory_cap_bytes;
    }
    return set_err(ctx, FMAP_MEMORY_CAP,
                   "cuda route needs " + std::to_string(staging) + " bytes of device staging, above the cap of " +
                       std::to_string(opts.memory_cap_bytes));
  }
  int st = arena_reserve(ctx, staging);
  if (st) return st;
  if (!ctx->comp2) FMAP_CK(ctx, cudaStreamCreateWithFlags(&ctx->comp2, cudaStreamNonBlocking));
  if (!ctx->copy) FMAP_CK(ctx, cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
  if (!ctx->copy2) FMAP_CK(ctx, cudaStreamCreateWithFlags(&ctx->copy2, cudaStreamNonBlocking));
  for (cudaEvent_t& e : ctx->cev)
    if (!e) FMAP_CK(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  float* dG = cv.take<float>((size_t)b * kk);
  float* dR = cv.take<float>((size_t)b * kk);
  float* dM = cv.take<float>((size_t)b * kk);
  float* dC = cv.take<float>((size_t)b * kk);
  float* scr[2] = {cv.take<float>(tcb / sizeof(float)), cv.take<float>(tcb / sizeof(float))};
  float* rowsum = cv.take<float>((size_t)b * k);
  double* partial = cv.take<double>(npart);
  double* res_out = cv.take<double>(opts.compute_residual ? (size_t)b : 0);
  if ((st = reset_ctrl(ctx))) return st;
  FMAP_CK(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  FMAP_CK(ctx, cudaEventRecord(ctx->cev[0], ctx->stream));
  FMAP_CK(ctx, cudaStreamWaitEvent(ctx->copy, ctx->cev[0], 0));
  FMAP_CK(ctx, cudaStreamWaitEvent(ctx->comp2, ctx->cev[0], 0));
  FMAP_CK(ctx, cudaStreamWaitEvent(ctx->copy2, ctx->cev[0], 0));
  cudaStream_t comp[2] = {ctx->stream, ctx->comp2};
  SolveParams p{};
  p.k = (int)k;
  p.K4 = ((int)k + 3) & ~3;
  p.Rp = p.K4 + 4;
  p.lambda = lambda;
  p.ridge = opts.ridge;
  p.rcond_thr = opts.rcond_threshold < 0.f ? 1e-7f : opts.rcond_threshold;
  p.rhs_unit = -1;
  p.fail_min = d_fail(ctx);
  p.rcond_min_bits = d_rcond(ctx);
  p.flags = d_flags(ctx);
  p.rcond_exact = d_nexact(ctx);
  p.gram = dG;
  p.rhs = dR;
  p.mask = dM;
  p.C = dC;
  p.gram_rowsum = rowsum;
  const char* dbg_env = std::getenv("FMAP_DEBUG");  // timing experiments only: 2 = no H2D, 4 = no D2H
  const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
  // Per chunk, G and M land first (the factorization needs them), R after (the back
  // substitution and the validation need it): the solve starts 1/3 of a chunk's copy
  // earlier.  Validation runs between the factorization and the back substitution
  // -- nothing is exposed before the final flag check, which still takes precedence
  // over SINGULAR, and C is zero-filled on any error.
  for (int c = 0; c < nchunk; ++c) {  // all H2D first: the copy stream never waits on the solver
    const int64_t q0 = cq0[c], nq = cnq[c];
    const size_t off = (size_t)q0 * kk, nb = (size_t)nq * kk * sizeof(float);
    if (!(dbg & 2)) {
      FMAP_CK(ctx, cudaMemcpyAsync(dG + off, gram + off, nb, cudaMemcpyHostToDevice, ctx->copy));
      FMAP_CK(ctx, cudaMemcpyAsync(dM + off, mask + off, nb, cudaMemcpyHostToDevice, ctx->copy));
    }
    FMAP_CK(ctx, cudaEventRecord(ctx->cev[2 + 3 * c], ctx->copy));
    if (!(dbg & 2)) FMAP_CK(ctx, cudaMemcpyAsync(dR + off, rhs + off, nb, cudaMemcpyHostToDevice, ctx->copy));
    FMAP_CK(ctx, cudaEventRecord(ctx->cev[3 + 3 * c], ctx->copy));
  }
  for (int c = 0; c < nchunk; ++c) {
    const int64_t q0 = cq0[c], nq = cnq[c];
    const size_t off = (size_t)q0 * kk, nb = (size_t)nq * kk * sizeof(float);
    cudaEvent_t gm = ctx->cev[2 + 3 * c], rr = ctx->cev[3 + 3 * c], done = ctx->cev[4 + 3 * c];
    cudaStream_t s = comp[c & 1];
    FMAP_CK(ctx, cudaStreamWaitEvent(s, gm, 0));
    FMAP_CK(ctx, launch_gram_check(dG + off, nq, (int)k, rowsum + (size_t)q0 * k, d_flags(ctx), s));
    p.nsys = nq * k;
    p.sys_offset = q0 * k;
    p.tc_scratch = scr[c & 1];
    FMAP_CK(ctx, launch_chol_solve(p, 0, s, 1));
    FMAP_CK(ctx, cudaStreamWaitEvent(s, rr, 0));
    FMAP_CK(ctx, launch_validate(dG + off, dR + off, dM + off, (size_t)nq * kk, d_flags(ctx), s));
    FMAP_CK(ctx, launch_chol_solve(p, 0, s, 2));
    FMAP_CK(ctx, cudaEventRecord(done, s));
    FMAP_CK(ctx, cudaStreamWaitEvent(ctx->copy2, done, 0));
    if (!(dbg & 4)) FMAP_CK(ctx, cudaMemcpyAsync(C_out + off, dC + off, nb, cudaMemcpyDeviceToHost, ctx->copy2));
  }
  FMAP_CK(ctx, cudaEventRecord(ctx->cev[50], ctx->copy));  // all H2D done (stream join)
  FMAP_CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->cev[50], 0));
  if (opts.compute_residual) {
    // check_stationarity (solver.hpp:314-320) over the whole batch on the tensor cores
    // once every chunk is solved (~0.05 ms; it overlaps the last chunk's D2H).  Per-chunk
    // FP32 tiles beside the next chunk's solve measured 0.08 ms slower: they slow the
    // solver they share SMs with.
    FMAP_CK(ctx, cudaEventRecord(ctx->cev[51], comp[1]));
    FMAP_CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->cev[51], 0));
    FMAP_CK(ctx, launch_residual(dC, dG, dR, dM, b, (int)k, lambda, partial, res_out, ctx->stream, d_resmax(ctx)));
  }
  FMAP_CK(ctx, cudaEventRecord(ctx->cev[1], ctx->copy2));
  FMAP_CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->cev[1], 0));
  FMAP_CK(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  unsigned long long fail;
  float rcond;
  unsigned flags;
  if ((st = read_ctrl(ctx, &fail, &rcond, &flags))) return st;
  float ms = 0.f;
  FMAP_CK(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (rep) {
    rep->wall_seconds = ms * 1e-3;
    rep->min_rcond = rcond;
    rep->rcond_exact_systems = ctx->last_exact;
  }
  if (flags || fail != kNoFail) std::memset(C_out, 0, bytes);  // no partial results
  if (flags) return set_err(ctx, FMAP_INVALID_ARGUMENT, flags_message(flags));
  if (fail != kNoFail) {
    if (rep) rep->failing_system = (int64_t)fail;
    return set_err(ctx, FMAP_SINGULAR,
                   "row system " + std::to_string(fail) +
                       " is numerically singular (Cholesky pivot / rcond estimate / non-finite solution)");
  }
  if (opts.compute_residual && rep) rep->max_residual = ctx->last_resmax;  // read with the control block
  ctx->last_error.clear();
  return FMAP_OK;
}


// f64 route (fmap_f64.cu): same contract as solve_core for an explicit mask.
int solve_core_f64(fmap_ctx* ctx, int64_t b, int64_t k, const double* G, const double* R, const double* M,
                   double lambda, const fmap_solver_options* o, double* C, fmap_report* rep,
                   size_t host_staging_bytes) {
  fmap_solver_options opts;
  default_opts(&opts);
  if (o) opts = *o;
  init_report(rep);
  if (b < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "no problems to solve");
  if (k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "problem is empty");
  if (!(lambda >= 0.0)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "lambda must be non-negative");
  if (!G || !R || !M || !C) return set_err(ctx, FMAP_INVALID_ARGUMENT, "null buffer");
  constexpr int64_t kF64Max = 512;  // rows beyond shared memory spill to an L2-resident scratch
  if (k > kF64Max)
    return set_err(ctx, FMAP_INVALID_ARGUMENT,
                   "k = " + std::to_string(k) + " exceeds the f64 route's limit " + std::to_string(kF64Max));
  const size_t kk = (size_t)k * k;
  const size_t spill = chol_f64_spill_doubles((int)k, (size_t)ctx->max_smem_optin, ctx->num_sms);
  const size_t scratch = carve_size({(size_t)b * sizeof(double), (size_t)k * sizeof(double), spill * sizeof(double)});
  const uint64_t required = (uint64_t)scratch + host_staging_bytes;
  if (rep) rep->peak_extra_bytes = required;
  if (opts.has_memory_cap && required > opts.memory_cap_bytes) {
    if (rep) {
      rep->required_bytes = required;
      rep->cap_bytes = opts.memory_cap_bytes;
    }
    return set_err(ctx, FMAP_MEMORY_CAP,
                   "cuda route needs " + std::to_string(required) + " bytes of device scratch, above the cap of " +
                       std::to_string(opts.memory_cap_bytes));
  }
  int st = scratch_reserve(ctx, scratch);
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->scr)};
  double* sq = cv.take<double>((size_t)b);
  double* zrow = cv.take<double>((size_t)k);
  double* dspill = spill ? cv.take<double>(spill) : nullptr;
  if ((st = reset_ctrl(ctx))) return st;
  FMAP_CK(ctx, launch_validate_f64(G, R, M, (size_t)b * kk, d_flags(ctx), ctx->stream));
  const double rthr = opts.rcond_threshold < 0.f ? 1e-14 : (double)opts.rcond_threshold;
  FMAP_CK(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  FMAP_CK(ctx, launch_chol_f64(G, R, M, C, (int)k, b * k, lambda, (double)opts.ridge, rthr, -1, d_fail(ctx),
                               d_rcond(ctx), d_nexact(ctx), dspill, ctx->stream));
  if (opts.inject_fault) {  // solver.hpp:269-273, as solve_core
    std::vector<double> g0(k);
    double m00 = 0.0;
    FMAP_CK(ctx, cudaMemcpyAsync(g0.data(), G, k * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FMAP_CK(ctx, cudaMemcpyAsync(&m00, M, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
    g0[0] += lambda * m00 + (double)opts.ridge;
    int w = 0;
    double best = -1.0;
    for (int64_t c = 0; c < k; ++c)
      if (std::fabs(g0[c]) > best) {
        best = std::fabs(g0[c]);
        w = (int)c;
      }
    const double alpha = -2.0 * g0[w];
    FMAP_CK(ctx, launch_chol_f64(G, R, M, zrow, (int)k, 1, lambda, (double)opts.ridge, rthr, 0, d_fail(ctx),
                                 d_rcond(ctx), d_nexact(ctx), dspill, ctx->stream));
    FMAP_CK(ctx, launch_fault_combine_f64(C, zrow, (int)k, w, alpha, d_fail(ctx), ctx->stream));
  }
  FMAP_CK(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  if (opts.compute_residual) {
    FMAP_CK(ctx, launch_residual_f64(C, G, R, M, b, (int)k, lambda, sq, ctx->stream));
  }
  unsigned long long fail;
  float rcond;
  unsigned flags;
  if ((st = read_ctrl(ctx, &fail, &rcond, &flags))) return st;
  float ms = 0.f;
  FMAP_CK(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (rep) {
    rep->wall_seconds = ms * 1e-3;
    rep->min_rcond = rcond;
    rep->rcond_exact_systems = ctx->last_exact;
  }
  if (flags) return set_err(ctx, FMAP_INVALID_ARGUMENT, flags_message(flags));
  if (fail != kNoFail) {
    if (rep) rep->failing_system = (int64_t)fail;
    return set_err(ctx, FMAP_SINGULAR,
                   "row system " + std::to_string(fail) +
                       " is numerically singular (Cholesky pivot / rcond estimate / non-finite solution)");
  }
  if (opts.compute_residual && rep) {
    std::vector<double> res(b);
    FMAP_CK(ctx, cudaMemcpy(res.data(), sq, b * sizeof(double), cudaMemcpyDeviceToHost));
    double mx = 0.0;
    for (double v : res) mx = std::max(mx, std::sqrt(v));
    rep->max_residual = mx;
  }
  ctx->last_error.clear();
  return FMAP_OK;
}

// normal_equations (solver.hpp:95-103) for up to 4 products on the tensor cores
// (fmap_gram.cu); the FP32 SIMT GEMM serves shapes the tcgen05 kernel does not
// (k > 304, or more than 65535 pairs) and FMAP_GRAM=simt.
cudaError_t normal_products(int n, const float* const* X, const float* const* Y, float* const* out, const int* sym,
                            int64_t b, int k, int d, cudaStream_t st) {
  const char* sel = std::getenv("FMAP_GRAM");
  if (!(sel && sel[0] == 's')) {
    const cudaError_t e = launch_gram_tc(n, X, Y, out, sym, b, k, d, st);
    if (e != cudaErrorNotSupported) return e;
  }
  for (int i = 0; i < n; ++i) {
    const cudaError_t e = launch_gemm_nt(X[i], Y[i], b, k, k, d, out[i], st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// project_to_spectral (spectral.hpp:47-93) on device f64 buffers; `convert`
// = inputs were fp32 and have been widened into the staging arena already.
int project_pinv_core(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const double* phi,
                      const double* F, double cond_thr, double* A, int64_t* rank_out, fmap_report* rep) {
  init_report(rep);
  if (b < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "no bases to project onto");
  if (n < 1 || k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "basis must be non-empty");
  if (d < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "features must be non-empty");
  if (b > 65535) return set_err(ctx, FMAP_INVALID_ARGUMENT, "at most 65535 shapes per call");
  if (!phi || !F || !A) return set_err(ctx, FMAP_INVALID_ARGUMENT, "null buffer");
  const size_t work = pinv_work_doubles(b, n, (int)k, (int)d);
  const size_t scratch = carve_size({work * sizeof(double), (size_t)b * sizeof(int)});
  int st = scratch_reserve(ctx, scratch);
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->scr)};
  double* dwork = cv.take<double>(work);
  int* drank = cv.take<int>((size_t)b);
  if ((st = reset_ctrl(ctx))) return st;
  FMAP_CK(ctx, launch_finite_f64(phi, (size_t)b * n * k, 1u, d_flags(ctx), ctx->stream));
  FMAP_CK(ctx, launch_finite_f64(F, (size_t)b * n * d, 2u, d_flags(ctx), ctx->stream));
  FMAP_CK(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  FMAP_CK(ctx, launch_pinv(phi, F, b, n, (int)k, (int)d, cond_thr, dwork, A, drank, d_fail(ctx), ctx->stream));
  FMAP_CK(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  unsigned long long fail;
  float rc;
  unsigned flags;
  if ((st = read_ctrl(ctx, &fail, &rc, &flags))) return st;
  if (flags & 1u) return set_err(ctx, FMAP_INVALID_ARGUMENT, "basis contains non-finite entries");
  if (flags & 2u) return set_err(ctx, FMAP_INVALID_ARGUMENT, "features contains non-finite entries");
  float ms = 0.f;
  FMAP_CK(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (rep) rep->wall_seconds = ms * 1e-3;
  std::vector<int> ranks((size_t)b);
  FMAP_CK(ctx, cudaMemcpy(ranks.data(), drank, (size_t)b * sizeof(int), cudaMemcpyDeviceToHost));
  if (rank_out)
    for (int64_t q = 0; q < b; ++q) rank_out[q] = ranks[(size_t)q];
  if (fail != kNoFail) {
    if (rep) rep->failing_system = (int64_t)fail;
    return set_err(ctx, FMAP_RANK_DEFICIENT,
                   "basis is rank deficient: rank " + std::to_string(ranks[(size_t)fail]) + " < " +
                       std::to_string(k) + " columns (shape " + std::to_string(fail) + ")");
  }
  ctx->last_error.clear();
  return FMAP_OK;
}

bool host_finite(const float* p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

}  // namespace

extern "C" {

int fmap_abi_version(void) { return FMAP_CUDA_ABI_VERSION; }

void fmap_default_options(fmap_solver_options* opts) {
  if (opts) default_opts(opts);
}

int fmap_ctx_create(int device, fmap_ctx** out) {
  if (!out) return FMAP_INVALID_ARGUMENT;
  *out = nullptr;
  fmap_ctx* ctx = new fmap_ctx();
  ctx->device = device;
  DeviceGuard dg(device);  // the caller's current device is restored on return
  auto fail = [&](cudaError_t e) {
    fmap_ctx_destroy(ctx);
    (void)e;
    return FMAP_CUDA_ERROR;
  };
  cudaError_t e;
  int ndev = 0;
  if ((e = cudaGetDeviceCount(&ndev)) != cudaSuccess) return fail(e);
  if (device < 0 || device >= ndev) return fail(cudaErrorInvalidDevice);
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e);
  ctx->stream = ctx->own_stream;
  if ((e = cudaMalloc(&ctx->d_ctrl, 64)) != cudaSuccess) return fail(e);
  if ((e = cudaMallocHost(&ctx->h_ctrl, 64)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&ctx->ev0)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&ctx->ev1)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&ctx->evf)) != cudaSuccess) return fail(e);
  if ((e = cudaDeviceGetAttribute(&ctx->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                  device)) != cudaSuccess)
    return fail(e);
  if ((e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device)) !=
      cudaSuccess)
    return fail(e);
  *out = ctx;
  return FMAP_OK;
}

int fmap_ctx_destroy(fmap_ctx* ctx) {
  if (!ctx) return FMAP_OK;
  DeviceGuard dg(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->scr) cudaFree(ctx->scr);
  if (ctx->d_ctrl) cudaFree(ctx->d_ctrl);
  if (ctx->h_ctrl) cudaFreeHost(ctx->h_ctrl);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evf) cudaEventDestroy(ctx->evf);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->comp2) cudaStreamDestroy(ctx->comp2);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->copy2) cudaStreamDestroy(ctx->copy2);
  for (cudaEvent_t& e : ctx->cev)
    if (e) cudaEventDestroy(e);
  delete ctx;
  return FMAP_OK;
}

int fmap_ctx_set_stream(fmap_ctx* ctx, void* s) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  ctx->stream = s ? reinterpret_cast<cudaStream_t>(s) : ctx->own_stream;
  return FMAP_OK;
}

const char* fmap_last_error(const fmap_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "no context"; }

int64_t fmap_max_resolution(fmap_ctx* ctx) { return ctx ? max_resolution(ctx) : 0; }

int64_t fmap_last_launch_count(const fmap_ctx* ctx) { return ctx ? ctx->launches : 0; }

const char* fmap_last_launches(const fmap_ctx* ctx) { return ctx ? ctx->launch_names.c_str() : ""; }

int fmap_project_pinv_f64_dev(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const double* d_phi,
                              const double* d_F, double condition_threshold, double* d_A, int64_t* rank_out,
                              fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  return project_pinv_core(ctx, b, n, k, d, d_phi, d_F, condition_threshold, d_A, rank_out, report);
}

int fmap_project_pinv_f64(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const double* phi,
                          const double* F, double condition_threshold, double* A_out, int64_t* rank_out,
                          fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  init_report(report);
  if (b < 1 || n < 1 || k < 1 || d < 1 || !phi || !F || !A_out)
    return project_pinv_core(ctx, b, n, k, d, phi, F, condition_threshold, A_out, rank_out, report);
  const size_t np = (size_t)b * n * k, nf = (size_t)b * n * d, na = (size_t)b * k * d;
  int st = arena_reserve(ctx, carve_size({np * 8, nf * 8, na * 8}));
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  double* dP = cv.take<double>(np);
  double* dF = cv.take<double>(nf);
  double* dA = cv.take<double>(na);
  FMAP_CK(ctx, cudaMemcpyAsync(dP, phi, np * 8, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(dF, F, nf * 8, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = project_pinv_core(ctx, b, n, k, d, dP, dF, condition_threshold, dA, rank_out, report))) return st;
  FMAP_CK(ctx, cudaMemcpyAsync(A_out, dA, na * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return FMAP_OK;
}

int fmap_project_pinv_f32(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d, const float* phi,
                          const float* F, float condition_threshold, float* A_out, int64_t* rank_out,
                          fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  init_report(report);
  if (b < 1 || n < 1 || k < 1 || d < 1 || !phi || !F || !A_out)
    return project_pinv_core(ctx, b, n, k, d, nullptr, nullptr, condition_threshold, nullptr, rank_out, report);
  const size_t np = (size_t)b * n * k, nf = (size_t)b * n * d, na = (size_t)b * k * d;
  int st = arena_reserve(ctx, carve_size({np * 4, nf * 4, na * 4, np * 8, nf * 8, na * 8}));
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  float* sP = cv.take<float>(np);
  float* sF = cv.take<float>(nf);
  float* sA = cv.take<float>(na);
  double* dP = cv.take<double>(np);
  double* dF = cv.take<double>(nf);
  double* dA = cv.take<double>(na);
  FMAP_CK(ctx, cudaMemcpyAsync(sP, phi, np * 4, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(sF, F, nf * 4, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, launch_convert_f32_f64(sP, dP, np, ctx->stream));
  FMAP_CK(ctx, launch_convert_f32_f64(sF, dF, nf, ctx->stream));
  if ((st = project_pinv_core(ctx, b, n, k, d, dP, dF, (double)condition_threshold, dA, rank_out, report)))
    return st;
  FMAP_CK(ctx, launch_convert_f64_f32(dA, sA, na, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(A_out, sA, na * 4, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return FMAP_OK;
}

int fmap_solve_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_gram,
                       const float* d_rhs, const float* d_mask, float lambda,
                       const fmap_solver_options* opts, float* d_C, fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  return solve_core(ctx, b, k, d_gram, d_rhs, d_mask, nullptr, nullptr, 0, 0.f, lambda, opts,
                    d_C, report, true, 0);
}

int fmap_solve_ev_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_gram,
                          const float* d_rhs, const float* d_ev1, const float* d_ev2,
                          int mask_kind, float sigma, float lambda,
                          const fmap_solver_options* opts, float* d_C, fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (mask_kind != FMAP_MASK_COMMUTATIVITY && mask_kind != FMAP_MASK_RESOLVENT)
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "unknown mask kind");
  return solve_core(ctx, b, k, d_gram, d_rhs, nullptr, d_ev1, d_ev2,
                    mask_kind == FMAP_MASK_RESOLVENT ? 1 : 2, sigma, lambda, opts, d_C, report,
                    true, 0);
}

int fmap_solve_f32(fmap_ctx* ctx, int64_t b, int64_t k, const float* gram, const float* rhs,
                   const float* mask, float lambda, const fmap_solver_options* opts,
                   float* C_out, fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  init_report(report);
  if (b < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "no problems to solve");
  if (k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "problem is empty");
  if (!gram || !rhs || !mask || !C_out) return set_err(ctx, FMAP_INVALID_ARGUMENT, "null buffer");
  if (!(lambda >= 0.f)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "lambda must be non-negative");
  const size_t kk = (size_t)k * k;
  // solver.hpp:132-145: validated on the device (validate_kernel) after the
  // copies and before any result is exposed; the status precedence follows the
  // reference's check order (mask >= 0, finite gram, rhs, mask).
  const size_t bytes = (size_t)b * kk * sizeof(float);
  const size_t staging = carve_size({bytes, bytes, bytes, bytes});
  fmap_solver_options o;
  default_opts(&o);
  if (opts) o = *opts;
  // pipelined copies (tensor-core solver, >= 2 pairs per chunk, no fault injection /
  // residual); FMAP_PIPELINE=<chunks> overrides the default (1 = unpipelined)
  const char* pipe = std::getenv("FMAP_PIPELINE");
  // default: 4 weighted chunks for b >= 16 (solve_host_pipelined), 4 equal chunks for
  // 8 <= b < 16; FMAP_PIPELINE=<n> forces n equal chunks (8: 5 % slower at cfg2),
  // FMAP_PIPELINE=r with FMAP_PIPELINE_W="w1,w2,..." other weights (experiments)
  const int nchunk = pipe ? (pipe[0] == 'r' ? 0 : std::max(1, std::min(16, std::atoi(pipe)))) : (b >= 16 ? 0 : 4);
  if ((nchunk > 1 ? b >= 2 * nchunk : nchunk == 0 && b >= 16) && !o.inject_fault && k <= max_resolution(ctx))
    return solve_host_pipelined(ctx, b, k, gram, rhs, mask, lambda, o, C_out, report, nchunk);
  if (o.has_memory_cap && staging > o.memory_cap_bytes) {
    if (report) {
      report->required_bytes = staging;
      report->cap_bytes = o.memory_cap_bytes;
      report->peak_extra_bytes = staging;
    }
    return set_err(ctx, FMAP_MEMORY_CAP,
                   "cuda route needs " + std::to_string(staging) +
                       " bytes of device staging, above the cap of " +
                       std::to_string(o.memory_cap_bytes));
  }
  int st = arena_reserve(ctx, staging);
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  float* dG = cv.take<float>((size_t)b * kk);
  float* dR = cv.take<float>((size_t)b * kk);
  float* dM = cv.take<float>((size_t)b * kk);
  float* dC = cv.take<float>((size_t)b * kk);
  FMAP_CK(ctx, cudaMemcpyAsync(dG, gram, bytes, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(dR, rhs, bytes, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(dM, mask, bytes, cudaMemcpyHostToDevice, ctx->stream));
  st = solve_core(ctx, b, k, dG, dR, dM, nullptr, nullptr, 0, 0.f, lambda, &o, dC, report, true,
                  staging);
  if (st) return st;
  FMAP_CK(ctx, cudaMemcpyAsync(C_out, dC, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return FMAP_OK;
}

int fmap_solve_f64_dev(fmap_ctx* ctx, int64_t b, int64_t k, const double* d_gram, const double* d_rhs,
                       const double* d_mask, double lambda, const fmap_solver_options* opts, double* d_C_out,
                       fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  return solve_core_f64(ctx, b, k, d_gram, d_rhs, d_mask, lambda, opts, d_C_out, report, 0);
}

int fmap_solve_f64(fmap_ctx* ctx, int64_t b, int64_t k, const double* gram, const double* rhs, const double* mask,
                   double lambda, const fmap_solver_options* opts, double* C_out, fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  init_report(report);
  if (b < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "no problems to solve");
  if (k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "problem is empty");
  if (!gram || !rhs || !mask || !C_out) return set_err(ctx, FMAP_INVALID_ARGUMENT, "null buffer");
  if (!(lambda >= 0.0)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "lambda must be non-negative");
  const size_t bytes = (size_t)b * k * k * sizeof(double);
  const size_t staging = carve_size({bytes, bytes, bytes, bytes});
  fmap_solver_options o;
  default_opts(&o);
  if (opts) o = *opts;
  if (o.has_memory_cap && staging > o.memory_cap_bytes) {
    if (report) {
      report->required_bytes = staging;
      report->cap_bytes = o.memory_cap_bytes;
      report->peak_extra_bytes = staging;
    }
    return set_err(ctx, FMAP_MEMORY_CAP,
                   "cuda route needs " + std::to_string(staging) + " bytes of device staging, above the cap of " +
                       std::to_string(o.memory_cap_bytes));
  }
  int st = arena_reserve(ctx, staging);
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  double* dG = cv.take<double>((size_t)b * k * k);
  double* dR = cv.take<double>((size_t)b * k * k);
  double* dM = cv.take<double>((size_t)b * k * k);
  double* dC = cv.take<double>((size_t)b * k * k);
  FMAP_CK(ctx, cudaMemcpyAsync(dG, gram, bytes, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(dR, rhs, bytes, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(dM, mask, bytes, cudaMemcpyHostToDevice, ctx->stream));
  st = solve_core_f64(ctx, b, k, dG, dR, dM, lambda, &o, dC, report, staging);
  if (st) return st;
  FMAP_CK(ctx, cudaMemcpyAsync(C_out, dC, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return FMAP_OK;
}

int fmap_mask_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_ev1,
                      const float* d_ev2, int mask_kind, float sigma, float* d_mask_out) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (b < 1 || k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "eigenvalue vectors must be non-empty");
  if (mask_kind != 0 && mask_kind != 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "unknown mask kind");
  if (mask_kind == 1 && !(sigma > 0.f))
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "sigma must be positive");
  int st = reset_ctrl(ctx);
  if (st) return st;
  FMAP_CK(ctx, launch_validate_ev(d_ev1, d_ev2, (size_t)b * k, d_flags(ctx), ctx->stream));
  if (mask_kind == 1) {  // masks.hpp:58-59: the resolvent mask normalises by the pair's max eigenvalue
    FMAP_CK(ctx, launch_ev_max_check(d_ev1, d_ev2, b, (int)k, d_flags(ctx), ctx->stream));
  }
  FMAP_CK(ctx, launch_mask(d_ev1, d_ev2, b, (int)k, mask_kind, sigma, d_mask_out, ctx->stream));
  unsigned long long fail;
  float rc;
  unsigned flags;
  if ((st = read_ctrl(ctx, &fail, &rc, &flags))) return st;
  if (flags & 16u) return set_err(ctx, FMAP_INVALID_ARGUMENT, "eigenvalues must be non-negative and finite");
  if (flags) return set_err(ctx, FMAP_INVALID_ARGUMENT, flags_message(flags));
  return FMAP_OK;
}

int fmap_mask_f32(fmap_ctx* ctx, int64_t b, int64_t k, const float* ev1, const float* ev2,
                  int mask_kind, float sigma, float* mask_out) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (b < 1 || k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "eigenvalue vectors must be non-empty");
  if (mask_kind != 0 && mask_kind != 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "unknown mask kind");
  // masks.hpp:48-53 / 79-89 validation order
  if (!host_finite(ev1, (size_t)b * k))
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "ev1 contains non-finite entries");
  if (!host_finite(ev2, (size_t)b * k))
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "ev2 contains non-finite entries");
  for (int64_t e = 0; e < b * k; ++e)
    if (!(ev1[e] >= 0.f) || !(ev2[e] >= 0.f))
      return set_err(ctx, FMAP_INVALID_ARGUMENT, "eigenvalues must be non-negative");
  if (mask_kind == 1) {
    if (!(sigma > 0.f)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "sigma must be positive");
    for (int64_t q = 0; q < b; ++q) {
      float m = 0.f;
      for (int64_t c = 0; c < k; ++c) m = std::max(m, std::max(ev1[q * k + c], ev2[q * k + c]));
      if (!(m > 0.f))
        return set_err(ctx, FMAP_INVALID_ARGUMENT,
                       "resolvent mask needs a non-zero spectrum to normalize by");
    }
  }
  const size_t evb = (size_t)b * k * sizeof(float), mb = (size_t)b * k * k * sizeof(float);
  int st = arena_reserve(ctx, carve_size({evb, evb, mb}));
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  float* d1 = cv.take<float>((size_t)b * k);
  float* d2 = cv.take<float>((size_t)b * k);
  float* dm = cv.take<float>((size_t)b * k * k);
  FMAP_CK(ctx, cudaMemcpyAsync(d1, ev1, evb, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(d2, ev2, evb, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, launch_mask(d1, d2, b, (int)k, mask_kind, sigma, dm, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(mask_out, dm, mb, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return FMAP_OK;
}

int fmap_normal_equations_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, int64_t d,
                                  const float* d_A, const float* d_B, float* d_gram,
                                  float* d_rhs) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (b < 1 || k < 1 || d < 1)
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "descriptor A must be non-empty");
  const float* X[2] = {d_A, d_B};
  const float* Y[2] = {d_A, d_A};
  float* O[2] = {d_gram, d_rhs};
  const int sym[2] = {1, 0};
  FMAP_CK(ctx, normal_products(2, X, Y, O, sym, b, (int)k, (int)d, ctx->stream));
  return FMAP_OK;
}

int fmap_normal_equations_f32(fmap_ctx* ctx, int64_t b, int64_t k, int64_t d, const float* A,
                              const float* B, float* gram_out, float* rhs_out) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (b < 1 || k < 1 || d < 1)
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "descriptor A must be non-empty");
  const size_t nab = (size_t)b * k * d, ng = (size_t)b * k * k;
  if (!host_finite(A, nab)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "A contains non-finite entries");
  if (!host_finite(B, nab)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "B contains non-finite entries");
  int st = arena_reserve(ctx, carve_size({nab * 4, nab * 4, ng * 4, ng * 4}));
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  float* dA = cv.take<float>(nab);
  float* dB = cv.take<float>(nab);
  float* dG = cv.take<float>(ng);
  float* dR = cv.take<float>(ng);
  FMAP_CK(ctx, cudaMemcpyAsync(dA, A, nab * 4, cudaMemcpyHostToDevice, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(dB, B, nab * 4, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = fmap_normal_equations_f32_dev(ctx, b, k, d, dA, dB, dG, dR))) return st;
  FMAP_CK(ctx, cudaMemcpyAsync(gram_out, dG, ng * 4, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaMemcpyAsync(rhs_out, dR, ng * 4, cudaMemcpyDeviceToHost, ctx->stream));
  FMAP_CK(ctx, cudaStreamSynchronize(ctx->stream));
  return FMAP_OK;
}

int fmap_project_f32_dev(fmap_ctx* ctx, int64_t b, int64_t n, int64_t k, int64_t d,
                         const float* d_phi, const float* d_mass, const float* d_F,
                         float* d_out) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (b < 1 || n < 1 || k < 1 || d < 1)
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "basis and features must be non-empty");
  FMAP_CK(ctx, launch_project(d_phi, d_mass, d_F, b, n, (int)k, (int)d, d_out, ctx->stream));
  return FMAP_OK;
}

int fmap_residual_f32_dev(fmap_ctx* ctx, int64_t b, int64_t k, const float* d_C,
                          const float* d_gram, const float* d_rhs, const float* d_mask,
                          float lambda, double* d_out) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  if (b < 1 || k < 1) return set_err(ctx, FMAP_INVALID_ARGUMENT, "problem is empty");
  const size_t np = residual_partial_count(b, (int)k);
  int st = scratch_reserve(ctx, np * sizeof(double));
  if (st) return st;
  FMAP_CK(ctx, launch_residual(d_C, d_gram, d_rhs, d_mask, b, (int)k, lambda,
                               reinterpret_cast<double*>(ctx->scr), d_out, ctx->stream));
  return FMAP_OK;
}

int fmap_pipeline_f32_dev(fmap_ctx* ctx, int64_t b, int64_t n1, int64_t n2, int64_t k,
                          int64_t d, const float* d_phi1, const float* d_mass1,
                          const float* d_F1, const float* d_ev1, const float* d_phi2,
                          const float* d_mass2, const float* d_F2, const float* d_ev2,
                          int mask_kind, float sigma, float lambda,
                          const fmap_solver_options* opts, float* d_Cxy, float* d_Cyx,
                          fmap_report* report) {
  if (!ctx) return FMAP_INVALID_ARGUMENT;
  DeviceGuard dg(ctx->device);
  LaunchScope ls(ctx);
  init_report(report);
  if (b < 1 || n1 < 1 || n2 < 1 || k < 1 || d < 1)
    return set_err(ctx, FMAP_INVALID_ARGUMENT, "pipeline dimensions must be positive");
  const size_t nab = (size_t)b * k * d, ng = (size_t)b * k * k;
  const bool bidir = d_Cyx != nullptr;
  const size_t scratch = carve_size({nab * 4, nab * 4, ng * 4, ng * 4, bidir ? ng * 4 : 0,
                                     bidir ? ng * 4 : 0, ng * 4});
  fmap_solver_options o;
  default_opts(&o);
  if (opts) o = *opts;
  // the pipeline's intermediates live in the staging arena, the solver's scratch in ctx->scr
  int st = arena_reserve(ctx, scratch);
  if (st) return st;
  Carve cv{reinterpret_cast<char*>(ctx->arena)};
  float* A = cv.take<float>(nab);
  float* B = cv.take<float>(nab);
  float* G = cv.take<float>(ng);
  float* R = cv.take<float>(ng);
  float* G2 = bidir ? cv.take<float>(ng) : nullptr;
  float* R2 = bidir ? cv.take<float>(ng) : nullptr;
  float* Mx = cv.take<float>(ng);
  cudaEvent_t e0, e1;
  FMAP_CK(ctx, cudaEventCreate(&e0));
  FMAP_CK(ctx, cudaEventCreate(&e1));
  FMAP_CK(ctx, cudaEventRecord(e0, ctx->stream));
  FMAP_CK(ctx, launch_project(d_phi1, d_mass1, d_F1, b, n1, (int)k, (int)d, A, ctx->stream));
  FMAP_CK(ctx, launch_project(d_phi2, d_mass2, d_F2, b, n2, (int)k, (int)d, B, ctx->stream));
  {  // G = A A^T, R = B A^T (and G2 = B B^T, R2 = A B^T): one tcgen05 launch
    const float* X[4] = {A, B, B, A};
    const float* Y[4] = {A, A, B, B};
    float* O[4] = {G, R, G2, R2};
    const int sym[4] = {1, 0, 1, 0};
    FMAP_CK(ctx, normal_products(bidir ? 4 : 2, X, Y, O, sym, b, (int)k, (int)d, ctx->stream));
  }
  // The mask is materialized (one fused mask-construction kernel, masks.hpp:36-82) and
  // the solver reads it densely: its per-row entries are then prefetched with the
  // next system's G (2.33 vs 2.43 ms at cfg2 with the entries computed inside the
  // solver from the eigenvalues).  solve_core carves its own scratch after
  // host_staging_bytes = our scratch.
  const bool resolvent = mask_kind == FMAP_MASK_RESOLVENT;
  const int mm = resolvent ? 3 : 4;
  if (resolvent && !(sigma > 0.f)) return set_err(ctx, FMAP_INVALID_ARGUMENT, "sigma must be positive");
  FMAP_CK(ctx, launch_mask(d_ev1, d_ev2, b, (int)k, resolvent ? 1 : 0, sigma, Mx, ctx->stream));
  st = solve_core(ctx, b, k, G, R, Mx, d_ev1, d_ev2, mm, sigma, lambda, &o, d_Cxy, report, true, scratch);
  if (st) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return st;
  }
  if (bidir) {
    fmap_report r2;
    // reverse direction: source/target swap, mask(ev2, ev1) = M^T
    FMAP_CK(ctx, launch_mask(d_ev2, d_ev1, b, (int)k, resolvent ? 1 : 0, sigma, Mx, ctx->stream));
    st = solve_core(ctx, b, k, G2, R2, Mx, d_ev2, d_ev1, mm, sigma, lambda, &o, d_Cyx, &r2, true, scratch);
    if (st) {
      if (report) *report = r2;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      return st;
    }
    if (report) {
      report->max_residual = std::max(report->max_residual, r2.max_residual);
      report->min_rcond = std::min(report->min_rcond, r2.min_rcond);
      report->rcond_exact_systems += r2.rcond_exact_systems;
    }
  }
  FMAP_CK(ctx, cudaEventRecord(e1, ctx->stream));
  FMAP_CK(ctx, cudaEventSynchronize(e1));
  float ms = 0.f;
  FMAP_CK(ctx, cudaEventElapsedTime(&ms, e0, e1));
  if (report) report->wall_seconds = ms * 1e-3;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return FMAP_OK;
}

}  // extern "C"
