// Warm-started Rayleigh-Ritz eigensolver for a Davidson projection that grew
// by b bordering rows/columns since its last eigendecomposition.
//
// If H[:g0,:g0] = Y0 diag(l0) Y0^T is known (the previous iteration's Ritz
// pairs, or Y0 = I after a thick restart that kept Ritz vectors), then in
// the basis blkdiag(Y0, I_b) the new projection is an arrowhead matrix per
// border.  Each border is absorbed exactly with the secular equation
//     f(lam) = lam - alpha - sum_i z_i^2 / (lam - d_i) = 0,
// one lane group per root (safeguarded Newton on f*(lam - d_K) about the nearest
// pole K), deflation of tiny couplings and of (nearly) equal poles by Givens
// rotations, and Gu-Eisenstat recomputed couplings z^ so the computed
// eigenvectors are orthogonal to working precision.  Cost is O(g^2) per
// border on one CTA instead of the O(g^3) sweeps of a cold Jacobi solve.
//
// Latency is what matters here (g <= 64, one CTA, on the critical path of
// every Davidson iteration), so every O(g) loop is spread over a warp or
// the CTA: the secular sums and the Gu-Eisenstat products are warp-wide with
// fixed xor trees (deterministic), the type-2 deflation scan only runs
// serially when two poles actually coincide.
//
// Replaces, on the warm path, the per-iteration dense eigh of
// extract_rayleigh_ritz (pkg/src/itersvd/eigensolver.py:362-367).
#include <algorithm>

#include "common.cuh"

namespace svdsb {

constexpr int kAT = 1024;             // threads: 32 warps, one secular root each
constexpr int kAN = SVDSB_SMALL_MAX;  // max dimension

struct ArrowSmem {
  double d[kAN], z[kAN];           // poles (current diag) and couplings
  double sd[kAN], sz[kAN];         // sorted, non-deflated
  int sidx[kAN];                   // original index of sorted pole
  int defl[kAN];                   // deflated flag per original index
  double tau[kAN + 1];             // root offsets
  double tau2[kAN + 1];            // per-column scratch (eigenvector scaling)
  int rank[kAN + 1];               // ascending rank of each eigenvalue
  int perm[kAN + 1];               // output column -> eigenvalue index
  int korg[kAN + 1];               // root origin (sorted pole index)
  double zhat[kAN];
  double newd[kAN + 1];            // eigenvalues in output column order
  double hcol[kAN + 1];            // bordering column of H, staged once
  // Givens rotations from type-2 deflation (original index pairs)
  int ra[kAN], rb[kAN];
  double rc[kAN], rs[kAN];
  int nrot, np;
  double alpha, tol, znorm;
};

// Development probe (tools/arrow_phases.py): per-phase SM clock stamps of
// thread 0, compiled in only with -DSVDSB_PHASE_CLOCKS.
#ifdef SVDSB_PHASE_CLOCKS
__device__ long long g_arrow_clk[16];
#define SVDSB_PHASE(k) \
  if (threadIdx.x == 0) g_arrow_clk[k] = clock64()
#else
#define SVDSB_PHASE(k) \
  do {                 \
  } while (0)
#endif

// Lanes per secular root: a small group keeps the FP64 work per Newton step
// low (one SM executes every root), a wide one shortens each step's chain.
#ifndef SVDSB_ARROW_GROUP
#define SVDSB_ARROW_GROUP 16
#endif
constexpr int kRG = SVDSB_ARROW_GROUP;

__device__ __forceinline__ double gsum(double v, unsigned mask) {
#pragma unroll
  for (int o = 1; o < kRG; o <<= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 1/x from the MUFU seed and two Newton steps (~1 ulp; the secular sums do
// not need a correctly rounded reciprocal, and the FP64 divide sequence is
// what bounds this single-CTA kernel).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// f(tau) with origin pole K (sorted index), also the pieces of h = tau*f
// without the K pole.  Evaluated by a kRG-lane group (lane l sums terms l,
// l+kRG, ...), combined with a fixed xor tree so every lane of the group
// holds identical values.
__device__ __forceinline__ void secular_eval(const ArrowSmem &s, int K, double tau, int lane, unsigned mask,
                                             double &f, double &h, double &hp, double &fscale) {
  const double dK = s.sd[K];
  double sum = 0.0, sum_nk = 0.0, dsum_nk = 0.0, scale = 0.0;
  for (int i = lane; i < s.np; i += kRG) {
    const double den = tau - (s.sd[i] - dK);   // lam - d_i
    const double inv = fast_rcp(den);
    const double zz = s.sz[i] * s.sz[i];
    const double t = zz * inv;
    sum += t;
    scale += fabs(t);
    if (i != K) {
      sum_nk += t;
      dsum_nk += t * inv;
    }
  }
  sum = gsum(sum, mask);
  scale = gsum(scale, mask) + fabs(dK - s.alpha) + fabs(tau);
  sum_nk = gsum(sum_nk, mask);
  dsum_nk = gsum(dsum_nk, mask);
  f = (dK - s.alpha) + tau - sum;
  const double zK2 = s.sz[K] * s.sz[K];
  h = tau * ((dK - s.alpha) + tau - sum_nk) - zK2;
  hp = (dK - s.alpha) + 2.0 * tau - sum_nk + tau * dsum_nk;
  fscale = scale;
}

// Root j of np+1 (ascending; interval (sd[j-1], sd[j])), solved by one warp;
// lane 0 stores the result.
__device__ void arrow_roots(ArrowSmem &s, int j, int lane, unsigned mask) {
  const int np = s.np;
  int K;
  double lo, hi;
  if (np == 0) {
    if (lane == 0) {
      s.korg[j] = -1;
      s.tau[j] = s.alpha;
    }
    return;
  }
  if (j == 0) {
    K = 0;
    double lb = fmin(s.sd[0], s.alpha) - s.znorm;
    lo = lb - s.sd[0] - fabs(lb) * 4e-16 - 1e-300;
    hi = 0.0;
  } else if (j == np) {
    K = np - 1;
    double ub = fmax(s.sd[np - 1], s.alpha) + s.znorm;
    lo = 0.0;
    hi = ub - s.sd[np - 1] + fabs(ub) * 4e-16 + 1e-300;
  } else {
    const double a = s.sd[j - 1], b = s.sd[j];
    const double half = 0.5 * (b - a);
    double f, h, hp, sc;
    secular_eval(s, j - 1, half, lane, mask, f, h, hp, sc);
    if (f >= 0.0) {
      K = j - 1;
      lo = 0.0;
      hi = half;
    } else {
      K = j;
      lo = -half;
      hi = 0.0;
    }
  }
  double tau = 0.5 * (lo + hi);
  {
    // Starting point: zero of the model that keeps pole K and the pole N at
    // the other end of the interval exactly and freezes the remaining terms
    // (and, for interior roots, the linear term) at the interval midpoint.
    // Newton on h then needs a few steps instead of working down from the
    // midpoint.
    const double dK = s.sd[K];
    const int N = (j == 0 || j == np) ? -1 : (K == j - 1 ? j : j - 1);
    double so = 0.0;
    for (int i = lane; i < np; i += kRG) {
      if (i == K || i == N) continue;
      so += s.sz[i] * s.sz[i] * fast_rcp(tau - (s.sd[i] - dK));
    }
    so = gsum(so, mask);
    const double zK2 = s.sz[K] * s.sz[K];
    double guess;
    if (N < 0) {
      // (c + t) t - zK2 = 0, the positive root right of all poles, the
      // negative one left of them (cancellation-free forms)
      const double c = dK - s.alpha - so;
      const double sq = sqrt(c * c + 4.0 * zK2);
      if (j == np)
        guess = (c <= 0.0) ? 0.5 * (sq - c) : 2.0 * zK2 / (sq + c);
      else
        guess = (c >= 0.0) ? -0.5 * (sq + c) : -2.0 * zK2 / (sq - c);
    } else {
      // c t (t - dN) - zK2 (t - dN) - zN2 t = 0 has one zero in (lo, hi)
      const double dN = s.sd[N] - dK;
      const double zN2 = s.sz[N] * s.sz[N];
      const double c = dK - s.alpha + tau - so;
      const double A = c, B = -(c * dN + zK2 + zN2), C = zK2 * dN;
      const double q = -0.5 * (B + copysign(sqrt(fmax(B * B - 4.0 * A * C, 0.0)), B));
      const double t1 = (A != 0.0) ? q / A : lo;
      const double t2 = (q != 0.0) ? C / q : lo;
      guess = (t1 > lo && t1 < hi) ? t1 : t2;
    }
    if (guess > lo && guess < hi) tau = guess;
  }
  int it = 0;
  for (; it < 200; ++it) {
    double f, h, hp, sc;
    secular_eval(s, K, tau, lane, mask, f, h, hp, sc);
    if (f == 0.0) break;
    if (f > 0.0)
      hi = tau;
    else
      lo = tau;
    if (fabs(f) <= 4.0 * kEps * sc) break;
    double nt = (hp != 0.0) ? tau - h * fast_rcp(hp) : 0.5 * (lo + hi);
    if (!(nt > lo && nt < hi)) nt = 0.5 * (lo + hi);
    if (nt == tau || fabs(nt - tau) <= 2.0 * kEps * fabs(nt)) {
      tau = nt;
      break;
    }
    if (hi - lo <= 2.0 * kEps * fmax(fabs(lo), fabs(hi))) {
      tau = 0.5 * (lo + hi);
      break;
    }
    tau = nt;
  }
#ifdef SVDSB_PHASE_CLOCKS
  if (lane == 0) {
    atomicMax(reinterpret_cast<unsigned long long *>(&g_arrow_clk[14]), (unsigned long long)it);
    atomicAdd(reinterpret_cast<unsigned long long *>(&g_arrow_clk[15]), (unsigned long long)it);
  }
#endif
  if (lane == 0) {
    s.korg[j] = K;
    s.tau[j] = tau;
  }
}

// lam_j - d_i for sorted pole i
__device__ __forceinline__ double lam_minus_pole(const ArrowSmem &s, int j, int i) {
  return (s.sd[s.korg[j]] - s.sd[i]) + s.tau[j];
}

// Solve one arrowhead [[diag(d[0..n-1)), z],[z^T, alpha]] of size n+1.
// Outputs newd[0..n] and P ((n+1) x (n+1), column-major, ld = ldp) in the
// original coordinates (border coordinate n).  n < kAN <= blockDim.x.
__device__ void arrow_solve(ArrowSmem &s, int n, double *P, int ldp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  if (warp == 0) {
    double dm = 0.0, zn = 0.0;
    for (int i = lane; i < n; i += 32) {
      dm = fmax(dm, fabs(s.d[i]));
      zn = fma(s.z[i], s.z[i], zn);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      zn += __shfl_xor_sync(0xffffffffu, zn, o);
    }
    if (lane == 0) {
      zn = sqrt(zn);
      s.znorm = zn;
      s.tol = 8.0 * kEps * fmax(fmax(dm, fabs(s.alpha)), zn);
    }
  }
  __syncthreads();
  SVDSB_PHASE(3);
  for (int i = tid; i < n; i += nt) s.defl[i] = (fabs(s.z[i]) <= s.tol) ? 1 : 0;
  __syncthreads();
  // sort the surviving poles ascending (stable by index)
  for (int i = tid; i < n; i += nt) {
    if (s.defl[i]) continue;
    int r = 0;
    const double di = s.d[i];
    for (int k = 0; k < n; ++k)
      if (!s.defl[k] && (s.d[k] < di || (s.d[k] == di && k < i))) ++r;
    s.sidx[r] = i;
  }
  const int np0 = __syncthreads_count(tid < n && !s.defl[tid]);
  SVDSB_PHASE(4);
  // type-2 deflation: (nearly) equal neighbouring poles.  The scan chains
  // through the survivors, so it runs on one thread -- only when needed.
  const bool close = tid >= 1 && tid < np0 && (s.d[s.sidx[tid]] - s.d[s.sidx[tid - 1]] <= s.tol);
  if (__syncthreads_or(close)) {
    if (tid == 0) {
      int nrot = 0;
      int w = 0;  // write cursor of compacted survivors
      int prev = -1;
      for (int r = 0; r < np0; ++r) {
        int i = s.sidx[r];
        if (prev >= 0 && s.d[i] - s.d[prev] <= s.tol) {
          double za = s.z[prev], zb = s.z[i];
          double rr = hypot(za, zb);
          double c = zb / rr, sn = za / rr;
          s.ra[nrot] = prev;
          s.rb[nrot] = i;
          s.rc[nrot] = c;
          s.rs[nrot] = sn;
          ++nrot;
          s.z[prev] = 0.0;
          s.z[i] = rr;
          s.defl[prev] = 1;
          --w;  // prev leaves the survivor list
        }
        s.sidx[w++] = i;
        prev = i;
      }
      s.np = w;
      s.nrot = nrot;
      for (int r = 0; r < w; ++r) {
        s.sd[r] = s.d[s.sidx[r]];
        s.sz[r] = s.z[s.sidx[r]];
      }
    }
  } else {
    if (tid < np0) {
      s.sd[tid] = s.d[s.sidx[tid]];
      s.sz[tid] = s.z[s.sidx[tid]];
    }
    if (tid == 0) {
      s.np = np0;
      s.nrot = 0;
    }
  }
  __syncthreads();
  SVDSB_PHASE(5);
  const int np = s.np;
  {
    const int gl = tid & (kRG - 1);
    const unsigned gmask = (kRG == 32) ? 0xffffffffu : (((1u << kRG) - 1u) << ((tid & 31) & ~(kRG - 1)));
    for (int j = tid / kRG; j <= np; j += nt / kRG) arrow_roots(s, j, gl, gmask);
  }
  __syncthreads();
  SVDSB_PHASE(6);
  // Gu-Eisenstat couplings: one warp per pole, lane-strided partial
  // products of the ratios, fixed xor-tree product
  for (int i = warp; i < np; i += nwarp) {
    double prod = 1.0;
    for (int k = lane; k < np; k += 32) {
      if (k == i) continue;
      double num = (k < i) ? lam_minus_pole(s, k, i) : lam_minus_pole(s, k + 1, i);
      prod *= num / (s.sd[k] - s.sd[i]);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) prod *= __shfl_xor_sync(0xffffffffu, prod, o);
    if (lane == 0) {
      prod *= lam_minus_pole(s, i, i) * lam_minus_pole(s, i + 1, i);
      double zh = sqrt(fabs(prod));
      s.zhat[i] = (s.sz[i] >= 0.0) ? zh : -zh;
    }
  }
  // eigenvector columns: first the deflated original indices, then roots
  const int N1 = n + 1;
  for (int e = tid; e < N1 * N1; e += nt) P[(e % N1) + (e / N1) * ldp] = 0.0;
  __syncthreads();
  SVDSB_PHASE(7);
  const int ndefl = n - np;
  for (int i = tid; i < n; i += nt) {
    if (!s.defl[i]) continue;
    int col = 0;
    for (int k = 0; k < i; ++k) col += s.defl[k];
    P[i + col * ldp] = 1.0;
    s.newd[col] = s.d[i];
  }
  for (int j = tid; j <= np; j += nt) s.newd[ndefl + j] = (np == 0) ? s.alpha : s.sd[s.korg[j]] + s.tau[j];
  if (np == 0) {
    if (tid == 0) P[n + ndefl * ldp] = 1.0;
  } else {
    // element-parallel: v_i = zhat_i / (lam_j - d_i), then column norms
    for (int e = tid; e < (np + 1) * np; e += nt) {
      const int j = e / np, i = e % np;
      P[s.sidx[i] + (ndefl + j) * ldp] = s.zhat[i] / lam_minus_pole(s, j, i);
    }
    __syncthreads();
    for (int j = warp; j <= np; j += nwarp) {
      const double *pc = P + (ndefl + j) * ldp;
      double a = 0.0;
      for (int i = lane; i < np; i += 32) {
        const double v = pc[s.sidx[i]];
        a = fma(v, v, a);
      }
      a = wsum(a);
      if (lane == 0) s.tau2[j] = 1.0 / sqrt(1.0 + a);
    }
    __syncthreads();
    for (int e = tid; e < (np + 1) * (np + 1); e += nt) {
      const int j = e / (np + 1), i = e % (np + 1);
      double *pc = P + (ndefl + j) * ldp;
      if (i < np)
        pc[s.sidx[i]] *= s.tau2[j];
      else
        pc[n] = s.tau2[j];
    }
  }
  __syncthreads();
  SVDSB_PHASE(8);
  // undo the deflation rotations (last created first): v = G_1 ... G_r v'
  if (s.nrot > 0) {
    for (int c = tid; c < N1; c += nt) {
      double *pc = P + c * ldp;
      for (int k = s.nrot - 1; k >= 0; --k) {
        int a = s.ra[k], b = s.rb[k];
        double va = pc[a], vb = pc[b];
        pc[a] = s.rc[k] * va + s.rs[k] * vb;
        pc[b] = -s.rs[k] * va + s.rc[k] * vb;
      }
    }
    __syncthreads();
  }
  SVDSB_PHASE(9);
}

__global__ void __launch_bounds__(kAT)
syev_update_kernel(int g0, int b, const double *__restrict__ h, int64_t ldh, const double *__restrict__ y0,
                   int64_t ldy0, const double *__restrict__ l0, int order, double shift, double *w_out,
                   double *y_out, int64_t ldy) {
  __shared__ ArrowSmem s;
  extern __shared__ double dyn[];
  const int G = g0 + b;
  const int ld = G + 1;
  double *Y = dyn;             // G x G current eigvecs (in V coordinates)
  double *P = Y + G * ld;      // arrowhead eigvecs
  double *T = P + G * ld;      // product buffer (swapped with Y)
  double *lam = T + G * ld;    // current eigenvalues
  const int tid = threadIdx.x, nt = blockDim.x;
  pdl_wait();
  pdl_trigger();
  SVDSB_PHASE(0);
  for (int e = tid; e < G * G; e += nt) {
    int i = e % G, j = e / G;
    double v = 0.0;
    if (i < g0 && j < g0) v = y0 ? y0[i + (int64_t)j * ldy0] : (i == j ? 1.0 : 0.0);
    Y[i + j * ld] = v;
  }
  for (int i = tid; i < g0; i += nt) lam[i] = l0 ? l0[i] : h[i + (int64_t)i * ldh];
  __syncthreads();
  SVDSB_PHASE(1);
  for (int j = 0; j < b; ++j) {
    const int sdim = g0 + j;  // current size; new index sdim
    // one parallel global read of the border column, then z = Y^T H[:sdim, sdim]
    // from shared memory (a k-loop over global loads is a latency chain)
    for (int k = tid; k <= sdim; k += nt) s.hcol[k] = h[k + (int64_t)sdim * ldh];
    __syncthreads();
    for (int i = tid; i < sdim; i += nt) {
      double acc = 0.0;
      for (int k = 0; k < sdim; ++k) acc = fma(Y[k + i * ld], s.hcol[k], acc);
      s.z[i] = acc;
      s.d[i] = lam[i];
    }
    if (tid == 0) s.alpha = s.hcol[sdim];
    __syncthreads();
    SVDSB_PHASE(2);
    arrow_solve(s, sdim, P, ld);
    // T <- blkdiag(Y, 1) P   (size sdim+1), then T becomes Y
    const int n1 = sdim + 1;
    for (int e = tid; e < n1 * n1; e += nt) {
      int r = e % n1, c = e / n1;
      double acc;
      if (r < sdim) {
        acc = 0.0;
        for (int k = 0; k < sdim; ++k) acc = fma(Y[r + k * ld], P[k + c * ld], acc);
      } else {
        acc = P[sdim + c * ld];
      }
      T[r + c * ld] = acc;
    }
    for (int c = tid; c < n1; c += nt) lam[c] = s.newd[c];
    __syncthreads();
    SVDSB_PHASE(10);
    double *tmp = Y;
    Y = T;
    T = tmp;
    SVDSB_PHASE(11);
  }
  // ordering as in syev_jacobi_kernel: ascending ranks first (ties by
  // index), then each value's position under the target rule, O(G) each
  for (int i = tid; i < G; i += nt) {
    const double wi = lam[i];
    int rank = 0;
    for (int j = 0; j < G; ++j) {
      const double wj = lam[j];
      if (wj < wi || (wj == wi && j < i)) ++rank;
    }
    s.rank[i] = rank;
  }
  __syncthreads();
  SVDSB_PHASE(12);
  for (int i = tid; i < G; i += nt) {
    const double wi = lam[i];
    const int rank = s.rank[i];
    int pos = 0;
    if (order == SVDSB_ORDER_ASC) {
      pos = rank;
    } else if (order == SVDSB_ORDER_DESC) {
      for (int j = 0; j < G; ++j) {
        const double wj = lam[j];
        if (j != i && ((wj > wi) || (wj == wi && s.rank[j] < rank))) ++pos;
      }
    } else {
      const int bi = wi < shift;
      const double ki = bi ? shift - wi : wi - shift;
      for (int j = 0; j < G; ++j) {
        if (j == i) continue;
        const double wj = lam[j];
        const int bj = wj < shift;
        const double kj = bj ? shift - wj : wj - shift;
        if ((bj < bi) || (bj == bi && (kj < ki || (kj == ki && s.rank[j] < rank)))) ++pos;
      }
    }
    w_out[pos] = wi;
    s.perm[pos] = i;
  }
  __syncthreads();
  // coalesced write-out of the permuted eigenvectors
  for (int e = tid; e < G * G; e += nt) {
    const int r = e % G, c = e / G;
    y_out[r + (int64_t)c * ldy] = Y[r + s.perm[c] * ld];
  }
#ifdef SVDSB_PHASE_CLOCKS
  __syncthreads();
  SVDSB_PHASE(13);
#endif
}

static bool g_arrow_attr = false;

}  // namespace svdsb

using namespace svdsb;

#ifdef SVDSB_PHASE_CLOCKS
extern "C" int svdsb_dbg_arrow_clocks(long long *out) {
  SVDSB_CUDA(cudaMemcpyFromSymbol(out, g_arrow_clk, sizeof(long long) * 16));
  return SVDSB_OK;
}
#endif

extern "C" int svdsb_syev_update(int g0, int b, const double *h, int64_t ldh, const double *y0, int64_t ldy0,
                                 const double *l0, int order, double shift, double *w, double *y, int64_t ldy,
                                 void *stream) {
  SVDSB_CHECK_ARG(g0 >= 0 && b >= 1 && g0 + b <= SVDSB_SMALL_MAX, "svdsb_syev_update: sizes out of range");
  SVDSB_CHECK_ARG(order >= 0 && order <= 2, "svdsb_syev_update: bad order");
  if (!g_arrow_attr) {
    SVDSB_CUDA(cudaFuncSetAttribute(syev_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
    g_arrow_attr = true;
  }
  const int G = g0 + b;
  size_t sh = sizeof(double) * (3 * G * (G + 1) + G + 1);
  SVDSB_LAUNCH_PDL(syev_update_kernel, 1, kAT, sh, as_stream(stream), g0, b, h, ldh, y0, ldy0, l0, order, shift, w, y,
                   ldy);
  return SVDSB_OK;
}
