// JDQMR inner solver: symmetric QMR (QMRs) on the Jacobi-Davidson
// correction equation, entirely on device.
//
//   P (Op - sigma I) P t = -r,   P = I - Q Q^T,  Q = [constraints, locked, x]
//
// with the optional point-Jacobi preconditioner applied as P K^-1 P.  The
// reference (pkg/src/itersvd) runs GD+k in both stages; the
// paper's stage 2 defaults to JDQMR, i.e. PRIMME's
// QMRs inner iteration with dynamic stopping (Stathopoulos, SISC 29(2),
// 2007).  This file is that inner iteration for B200:
//
//  * one inner step = the operator product (the CSR SpMV kernels, issued by
//    the host between jd_k1 ... jd_k3/jd_k4) and three or four streaming
//    kernels over N-vectors; every scalar of the QMRs recurrence (alpha,
//    theta, c, tau, gamma, eta, beta) lives in a device state vector and is
//    produced by the last CTA of the kernel that reduces its inputs;
//  * the eigen-residual of y = x + t is tracked from explicit dot products
//    (r.t, |t|^2, g.t, |g|^2, with g the QMR residual kept as a vector by
//    QMR smoothing g_j = s_j^2 g_{j-1} + c_j^2 r_j), and the stopping test
//    runs on device, so the whole inner solve is a CUDA graph with a WHILE
//    conditional node (svdsb_while_begin / svdsb_while_end): one launch, no
//    host round trip per inner step.
//
// Derivation of the estimate (sigma = theta, the Ritz value): with
// M t = -r - g and t, g orthogonal to x,
//   (Op - sigma) y = (theta - sigma + r.t) x - g            (x^T Op t = r.t)
//   rho(y) - sigma = ((theta - sigma + r.t) - g.t) / (1 + |t|^2)
//   |res(y)|^2     = ((theta - sigma + r.t)^2 + |g|^2) / (1 + |t|^2) - (rho - sigma)^2
// For an extreme target (DIR = -1 smallest, +1 largest) the inner solve also
// stops as soon as rho(y) moves away from that end of the spectrum: past that
// point the iterate converges toward another eigenpair (RQI behaviour).
#include "common.cuh"

namespace svdsb {

namespace jd {
// state vector layout (doubles)
enum : int {
  SIGMA = 0, TAU, THETA_PREV, RHO_PREV, ALPHA, GAMMA, ETA, BETA, C2, S2,
  RT, TT, GT, GG, ERES, ERES_BEST, IT, MAXIT, TOL_E, ETOL_FRAC, STOP, RITZ, RNORM, STALL,
  SIGP, LFAC, BNORM, DIR, RQ_PREV,
  QW = 32,   // Q^T w   (QMAX)
  QZ = 64,   // Q^T z   (QMAX)
  NSTATE = 96
};
constexpr int kQMax = 32;
constexpr int kThreads = 256;
}  // namespace jd

template <int R>
__device__ __forceinline__ void cta_partials(double (&acc)[R], double *part, int nparts_stride) {
  // per-CTA sums of R accumulators -> part[blockIdx.x * R + k]
  __shared__ double red[jd::kThreads / 32][R > 0 ? R : 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    double v = warp_sum(acc[k]);
    if (lane == 0) red[w][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < R; k += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q][k];
    part[(int64_t)blockIdx.x * nparts_stride + k] = s;
  }
  (void)nparts_stride;
}

__device__ __forceinline__ bool jd_stopped(const double *S) { return S[jd::STOP] != 0.0; }

// --------------------------------------------------------------- setup
// b = -r; rc = g = b; t = delta = 0; z = b ./ dg (precond) with Q^T z,
// rc.z; else d = b.  Fold: tau = |b|, rho_prev, QZ, counters.
template <int QB, bool PRE>
__global__ void __launch_bounds__(jd::kThreads) jd_init_kernel(
    int64_t n, const double *__restrict__ r, const double *__restrict__ dg, const double *__restrict__ q,
    int64_t ldq, int nq, double *__restrict__ rc, double *__restrict__ g, double *__restrict__ t,
    double *__restrict__ dl, double *__restrict__ z, double *__restrict__ d, double *S, double *part,
    unsigned int *ticket) {
  pdl_wait();
  constexpr int R = PRE ? QB + 2 : 1;
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double b = -r[i];
    rc[i] = b;
    g[i] = b;
    t[i] = 0.0;
    dl[i] = 0.0;
    acc[R - 1] = fma(b, b, acc[R - 1]);
    if (PRE) {
      const double zi = b / dg[i];
      z[i] = zi;
      d[i] = 0.0;
      acc[QB] = fma(b, zi, acc[QB]);
#pragma unroll
      for (int k = 0; k < QB; ++k)
        if (k < nq) acc[k] = fma(q[i + k * ldq], zi, acc[k]);
    } else {
      d[i] = b;
    }
  }
  cta_partials<R>(acc, part, R);
  if (!last_cta(ticket)) return;
  const unsigned np = gridDim.x;
  __shared__ double tot[R];
  fold_parts(part, np, R, R, [&](int o, int, int, double s) { tot[o] = s; });
  __syncthreads();
  if (threadIdx.x == 0) {
    const double bb = tot[R - 1];
    S[jd::TAU] = sqrt(bb);
    S[jd::BNORM] = sqrt(bb);
    S[jd::RHO_PREV] = PRE ? tot[QB] : bb;
    S[jd::THETA_PREV] = 0.0;
    S[jd::BETA] = 0.0;
    S[jd::RT] = 0.0;
    S[jd::TT] = 0.0;
    S[jd::GT] = 0.0;
    S[jd::GG] = bb;
    S[jd::IT] = 0.0;
    S[jd::STALL] = 0.0;
    S[jd::ERES] = S[jd::RNORM];
    S[jd::ERES_BEST] = S[jd::RNORM];
    S[jd::RQ_PREV] = S[jd::RITZ];
    S[jd::STOP] = (bb > 0.0 && S[jd::MAXIT] > 0.0) ? 0.0 : 7.0;
    for (int k = 0; k < jd::kQMax; ++k) S[jd::QZ + k] = (PRE && k < nq) ? tot[k] : 0.0;
  }
}

// ------------------------------------------------- K1: w -= sigma d; Q^T w, d.w
template <int QB>
__global__ void __launch_bounds__(jd::kThreads) jd_k1_kernel(
    int64_t n, const double *__restrict__ d, double *__restrict__ w, const double *__restrict__ q, int64_t ldq,
    int nq, double *S, double *part, unsigned int *ticket) {
  pdl_wait();
  if (jd_stopped(S)) return;
  const double sigma = S[jd::SIGMA];
  constexpr int R = QB + 1;
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double di = d[i];
    const double wi = fma(-sigma, di, w[i]);
    w[i] = wi;
    acc[QB] = fma(di, wi, acc[QB]);
#pragma unroll
    for (int k = 0; k < QB; ++k)
      if (k < nq) acc[k] = fma(q[i + k * ldq], wi, acc[k]);
  }
  cta_partials<R>(acc, part, R);
  if (!last_cta(ticket)) return;
  __shared__ double tot[R];
  fold_parts(part, gridDim.x, R, R, [&](int o, int, int, double s) { tot[o] = s; });
  __syncthreads();
  if (threadIdx.x == 0) {
    const double sigp = tot[QB];
    const double alpha = S[jd::RHO_PREV] / sigp;
    S[jd::SIGP] = sigp;
    S[jd::ALPHA] = alpha;
    for (int k = 0; k < jd::kQMax; ++k) S[jd::QW + k] = k < nq ? tot[k] : 0.0;
    if (sigp == 0.0 || !isfinite(alpha) || fabs(alpha) < 1e-300) S[jd::STOP] = 6.0;  // breakdown
  }
}

// --------------------------- K2: w = P w; rc -= alpha w; |rc|^2 -> QMR scalars
template <int QB, bool PRE>
__global__ void __launch_bounds__(jd::kThreads) jd_k2_kernel(
    int64_t n, double *__restrict__ w, double *__restrict__ rc, const double *__restrict__ q, int64_t ldq,
    int nq, double *S, double *part, unsigned int *ticket) {
  pdl_wait();
  if (jd_stopped(S)) return;
  const double alpha = S[jd::ALPHA];
  double qw[QB];
#pragma unroll
  for (int k = 0; k < QB; ++k) qw[k] = k < nq ? S[jd::QW + k] : 0.0;
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double wi = w[i];
#pragma unroll
    for (int k = 0; k < QB; ++k)
      if (k < nq) wi = fma(-q[i + k * ldq], qw[k], wi);
    w[i] = wi;
    const double ri = fma(-alpha, wi, rc[i]);
    rc[i] = ri;
    acc[0] = fma(ri, ri, acc[0]);
  }
  cta_partials<1>(acc, part, 1);
  if (!last_cta(ticket)) return;
  __shared__ double tot[1];
  fold_parts(part, gridDim.x, 1, 1, [&](int o, int, int, double s) { tot[o] = s; });
  __syncthreads();
  if (threadIdx.x == 0) {
    const double rr = tot[0];
    const double theta = sqrt(rr) / S[jd::TAU];
    const double c2 = 1.0 / (1.0 + theta * theta);
    const double thp = S[jd::THETA_PREV];
    S[jd::TAU] = S[jd::TAU] * theta * sqrt(c2);
    S[jd::GAMMA] = c2 * thp * thp;
    S[jd::ETA] = alpha * c2;
    S[jd::C2] = c2;
    S[jd::S2] = theta * theta * c2;
    S[jd::THETA_PREV] = theta;
    if (!PRE) {
      const double rho = rr;
      S[jd::BETA] = rho / S[jd::RHO_PREV];
      S[jd::RHO_PREV] = rho;
      if (!(rho > 0.0)) S[jd::STOP] = 6.0;
    }
  }
}

// -------------- K3: delta, t, g updates; (z, Q^T z, rc.z) or d; estimate + stop
template <int QB, bool PRE>
__global__ void __launch_bounds__(jd::kThreads) jd_k3_kernel(
    int64_t n, const double *__restrict__ r, const double *__restrict__ rc, double *__restrict__ g,
    double *__restrict__ t, double *__restrict__ dl, double *__restrict__ d, double *__restrict__ z,
    const double *__restrict__ dg, const double *__restrict__ q, int64_t ldq, int nq, double *S, double *part,
    unsigned int *ticket, unsigned long long cond) {
  pdl_wait();
  if (jd_stopped(S)) {
    if (cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
    return;
  }
  const double gam = S[jd::GAMMA], eta = S[jd::ETA], c2 = S[jd::C2], s2 = S[jd::S2], beta = S[jd::BETA];
  // acc: r.dl, t.dl, dl.dl, g.t, g.g [, Q^T z (QB), rc.z]
  constexpr int R = 5 + (PRE ? QB + 1 : 0);
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double dold = d[i];
    const double dli = fma(gam, dl[i], eta * dold);
    dl[i] = dli;
    const double ti = t[i];
    const double tn = ti + dli;
    t[i] = tn;
    const double ri = rc[i];
    const double gi = fma(s2, g[i], c2 * ri);
    g[i] = gi;
    acc[0] = fma(r[i], dli, acc[0]);
    acc[1] = fma(ti, dli, acc[1]);
    acc[2] = fma(dli, dli, acc[2]);
    acc[3] = fma(gi, tn, acc[3]);
    acc[4] = fma(gi, gi, acc[4]);
    if (PRE) {
      const double zi = ri / dg[i];
      z[i] = zi;
      acc[5 + QB] = fma(ri, zi, acc[5 + QB]);
#pragma unroll
      for (int k = 0; k < QB; ++k)
        if (k < nq) acc[5 + k] = fma(q[i + k * ldq], zi, acc[5 + k]);
    } else {
      d[i] = fma(beta, dold, ri);
    }
  }
  cta_partials<R>(acc, part, R);
  if (!last_cta(ticket)) return;
  __shared__ double tot[R];
  fold_parts(part, gridDim.x, R, R, [&](int o, int, int, double s) { tot[o] = s; });
  __syncthreads();
  if (threadIdx.x == 0) {
    const double it = S[jd::IT] + 1.0;
    S[jd::IT] = it;
    const double rt = S[jd::RT] + tot[0];
    const double tt = S[jd::TT] + 2.0 * tot[1] + tot[2];
    const double gt = tot[3], gg = tot[4];
    S[jd::RT] = rt;
    S[jd::TT] = tt;
    S[jd::GT] = gt;
    S[jd::GG] = gg;
    const double a = S[jd::RITZ] - S[jd::SIGMA] + rt;
    const double den = 1.0 + tt;
    const double rq = (a - gt) / den;
    const double e2 = (a * a + gg) / den - rq * rq;
    const double eres = sqrt(e2 > 0.0 ? e2 : 0.0);
    S[jd::ERES] = eres;
    double stop = 0.0;
    if (PRE) {
      const double rho = tot[5 + QB];
      S[jd::BETA] = rho / S[jd::RHO_PREV];
      S[jd::RHO_PREV] = rho;
      for (int k = 0; k < jd::kQMax; ++k) S[jd::QZ + k] = k < nq ? tot[5 + k] : 0.0;
      if (!(rho != 0.0) || !isfinite(rho)) stop = 6.0;
    }
    if (eres < S[jd::ERES_BEST]) {
      S[jd::ERES_BEST] = eres;
      S[jd::STALL] = 0.0;
    } else {
      S[jd::STALL] += 1.0;
    }
    // Rayleigh quotient of x + t moving away from the wanted end of the
    // spectrum: the inner iterate heads for another eigenpair
    const double rqv = S[jd::SIGMA] + rq;
    const bool reversed = S[jd::DIR] * (rqv - S[jd::RQ_PREV]) < 0.0;
    S[jd::RQ_PREV] = rqv;
    if (!isfinite(eres) || !isfinite(tt)) stop = 6.0;
    else if (reversed) stop = 8.0;
    else if (eres <= S[jd::TOL_E]) stop = 2.0;                        // eigenpair would converge
    else if (eres <= S[jd::ETOL_FRAC] * S[jd::RNORM]) stop = 3.0;     // ETolerance reached
    else if (sqrt(gg) <= S[jd::LFAC] * eres) stop = 4.0;              // linear residual below the plateau
    else if (S[jd::STALL] >= 3.0) stop = 5.0;                         // eigen-residual stagnates
    else if (it >= S[jd::MAXIT]) stop = 1.0;                          // inner budget
    if (stop != 0.0) S[jd::STOP] = stop;
    if (cond) cudaGraphSetConditional(cond, stop != 0.0 ? 0u : 1u);
  }
}

// -------------------------------------- K4 (preconditioned): d = P z + beta d
template <int QB>
__global__ void __launch_bounds__(jd::kThreads) jd_k4_kernel(
    int64_t n, const double *__restrict__ z, double *__restrict__ d, const double *__restrict__ q, int64_t ldq,
    int nq, const double *S) {
  pdl_wait();
  if (jd_stopped(S)) return;
  const double beta = S[jd::BETA];
  double qz[QB];
#pragma unroll
  for (int k = 0; k < QB; ++k) qz[k] = k < nq ? S[jd::QZ + k] : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double zi = z[i];
#pragma unroll
    for (int k = 0; k < QB; ++k)
      if (k < nq) zi = fma(-q[i + k * ldq], qz[k], zi);
    d[i] = fma(beta, d[i], zi);
  }
}

// the setup (beta = 0) applies the same kernel: d = P z
static int jd_grid(int64_t n) { return stream_grid(n, jd::kThreads * 4, num_sms() * 4); }

template <int QB>
static int jd_step_q(svdsb_ctx *ctx, int phase, int64_t n, const svdsb_jd_vecs *v, const double *q, int64_t ldq,
                     int nq, double *S, unsigned long long cond, cudaStream_t st) {
  const int grid = jd_grid(n);
  const bool pre = v->dg != nullptr;
  switch (phase) {
    case 0:
      if (pre) {
        SVDSB_LAUNCH_PDL(jd_init_kernel<QB, true>, grid, jd::kThreads, 0, st, n, v->r, v->dg, q, ldq, nq, v->rc,
                         v->g, v->t, v->dl, v->z, v->d, S, ctx->partials, take_ticket(ctx));
        SVDSB_LAUNCH_PDL(jd_k4_kernel<QB>, grid, jd::kThreads, 0, st, n, (const double *)v->z, v->d, q, ldq, nq,
                         (const double *)S);
      } else {
        SVDSB_LAUNCH_PDL(jd_init_kernel<QB, false>, grid, jd::kThreads, 0, st, n, v->r, v->dg, q, ldq, nq, v->rc,
                         v->g, v->t, v->dl, v->z, v->d, S, ctx->partials, take_ticket(ctx));
      }
      return SVDSB_OK;
    case 1:
      SVDSB_LAUNCH_PDL(jd_k1_kernel<QB>, grid, jd::kThreads, 0, st, n, (const double *)v->d, v->w, q, ldq, nq, S,
                       ctx->partials, take_ticket(ctx));
      if (pre)
        SVDSB_LAUNCH_PDL(jd_k2_kernel<QB, true>, grid, jd::kThreads, 0, st, n, v->w, v->rc, q, ldq, nq, S,
                         ctx->partials, take_ticket(ctx));
      else
        SVDSB_LAUNCH_PDL(jd_k2_kernel<QB, false>, grid, jd::kThreads, 0, st, n, v->w, v->rc, q, ldq, nq, S,
                         ctx->partials, take_ticket(ctx));
      if (pre) {
        SVDSB_LAUNCH_PDL(jd_k3_kernel<QB, true>, grid, jd::kThreads, 0, st, n, v->r, (const double *)v->rc, v->g,
                         v->t, v->dl, v->d, v->z, v->dg, q, ldq, nq, S, ctx->partials, take_ticket(ctx), cond);
        SVDSB_LAUNCH_PDL(jd_k4_kernel<QB>, grid, jd::kThreads, 0, st, n, (const double *)v->z, v->d, q, ldq, nq,
                         (const double *)S);
      } else {
        SVDSB_LAUNCH_PDL(jd_k3_kernel<QB, false>, grid, jd::kThreads, 0, st, n, v->r, (const double *)v->rc, v->g,
                         v->t, v->dl, v->d, v->z, v->dg, q, ldq, nq, S, ctx->partials, take_ticket(ctx), cond);
      }
      return SVDSB_OK;
  }
  set_error("svdsb_jd: bad phase");
  return SVDSB_ERR_ARG;
}

}  // namespace svdsb

using namespace svdsb;

// thread-local state of a WHILE-graph capture in progress
static thread_local cudaGraph_t g_while_graph = nullptr;

extern "C" {

int svdsb_jd_state_size(void) { return jd::NSTATE; }

int svdsb_jd_phase(svdsb_ctx *ctx, int phase, int64_t n, const svdsb_jd_vecs *vecs, const double *q, int64_t ldq,
                   int nq, double *state, uint64_t cond, void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr && vecs != nullptr && state != nullptr, "svdsb_jd_phase: NULL argument");
  SVDSB_CHECK_ARG(n >= 1, "svdsb_jd_phase: empty vectors");
  SVDSB_CHECK_ARG(nq >= 0 && nq <= jd::kQMax, "svdsb_jd_phase: at most 32 projection columns");
  SVDSB_CHECK_ARG(nq == 0 || (q != nullptr && ldq >= n), "svdsb_jd_phase: bad Q block");
  cudaStream_t st = as_stream(stream);
  const unsigned long long c = (unsigned long long)cond;
  if (nq <= 1) return jd_step_q<1>(ctx, phase, n, vecs, q, ldq, nq, state, c, st);
  if (nq <= 4) return jd_step_q<4>(ctx, phase, n, vecs, q, ldq, nq, state, c, st);
  if (nq <= 8) return jd_step_q<8>(ctx, phase, n, vecs, q, ldq, nq, state, c, st);
  if (nq <= 16) return jd_step_q<16>(ctx, phase, n, vecs, q, ldq, nq, state, c, st);
  return jd_step_q<32>(ctx, phase, n, vecs, q, ldq, nq, state, c, st);
}

int svdsb_while_begin(void *stream, uint64_t *cond_out) {
  SVDSB_CHECK_ARG(stream != nullptr && cond_out != nullptr, "svdsb_while_begin: needs a stream and an output");
  SVDSB_CHECK_ARG(g_while_graph == nullptr, "svdsb_while_begin: a WHILE capture is already open");
  cudaGraph_t g = nullptr;
  SVDSB_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams p = {};
  if (e == cudaSuccess) {
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  }
  if (e == cudaSuccess)
    e = cudaStreamBeginCaptureToGraph(as_stream(stream), p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    set_error("svdsb_while_begin: %s", cudaGetErrorString(e));
    return SVDSB_ERR_CUDA;
  }
  g_while_graph = g;
  set_pdl_suspended(true);
  *cond_out = (uint64_t)h;
  return SVDSB_OK;
}

int svdsb_while_end(void *stream, void **exec_out) {
  SVDSB_CHECK_ARG(exec_out != nullptr, "svdsb_while_end: NULL output");
  SVDSB_CHECK_ARG(g_while_graph != nullptr, "svdsb_while_end: no WHILE capture open");
  cudaGraph_t g = g_while_graph;
  g_while_graph = nullptr;
  set_pdl_suspended(false);
  cudaGraph_t body = nullptr;
  cudaError_t e = cudaStreamEndCapture(as_stream(stream), &body);
  cudaGraphExec_t ex = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiateWithFlags(&ex, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    set_error("svdsb_while_end: %s", cudaGetErrorString(e));
    return SVDSB_ERR_CUDA;
  }
  *exec_out = ex;
  return SVDSB_OK;
}

}  // extern "C"
