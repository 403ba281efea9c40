// Small dense fp64 kernels for the Davidson projected problem (g <= 64),
// each one CTA, so the Rayleigh-Ritz / restart bookkeeping stays on device.
//
// Reference counterparts (pkg/src/itersvd): sym_eig (kernels.py:136-145,
// LAPACK dsyevd) + target ordering (eigensolver.py:254-259, :362-367);
// small_svd (kernels.py:148-157) + refined extraction (eigensolver.py:
// 369-380); _coef_gs / restart coefficient selection (eigensolver.py:
// 438-469, :495-515); H <- C^T H C (:528-531); qr_restart (kernels.py:
// 225-242); the H column update (eigensolver.py:690-694).
//
// Algorithms: cyclic (round-robin parallel) two-sided Jacobi for the
// symmetric eigenproblem, one-sided Hestenes Jacobi for the SVD, Householder
// for the thin QR.  Jacobi is at least as accurate as LAPACK's tridiagonal
// path (high relative accuracy), and its data-parallel rounds map onto one
// CTA without any host round trip.
#include <algorithm>

#include "common.cuh"

namespace svdsb {

constexpr int kSmallThreads = 512;
constexpr int kMaxSweeps = 40;

// Round-robin tournament: player 0 fixed, players 1..G-1 rotate.
__device__ __forceinline__ void rr_pair(int G, int round, int k, int &p, int &q) {
  const int M = G - 1;
  if (k == 0) {
    p = 0;
    q = 1 + round % M;
  } else {
    p = 1 + (round + k) % M;
    q = 1 + ((round - k) % M + M) % M;
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// ------------------------------------------------------------------ syev

__global__ void __launch_bounds__(kSmallThreads)
syev_jacobi_kernel(int g, const double *__restrict__ h, int64_t ldh, int order, double shift, double *w_out,
                   double *y_out, int64_t ldy) {
  extern __shared__ double sm[];
  const int G = g + (g & 1);
  const int ld = G + 1;
  double *A0 = sm, *A1 = A0 + G * ld, *V0 = A1 + G * ld, *V1 = V0 + G * ld;
  double *cs = V1 + G * ld;  // per index: c
  double *sn = cs + G;       // per index: sigma_i * s
  int *partner = reinterpret_cast<int *>(sn + G);
  __shared__ int rotated;
  __shared__ double thr_abs;
  const int tid = threadIdx.x, nt = blockDim.x;

  for (int e = tid; e < G * G; e += nt) {
    int i = e % G, j = e / G;
    double a = 0.0;
    if (i < g && j < g) a = 0.5 * (h[i + (int64_t)j * ldh] + h[j + (int64_t)i * ldh]);
    A0[i + j * ld] = a;
    V0[i + j * ld] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    double s = 0.0;
    for (int e = tid; e < G * G; e += 32) {
      double a = A0[(e % G) + (e / G) * ld];
      s += a * a;
    }
    s = warp_sum(s);
    if (tid == 0) thr_abs = 1e-2 * kEps * sqrt(s) / (double)max(G, 1);
  }
  __syncthreads();

  double *A = A0, *An = A1, *V = V0, *Vn = V1;
  for (int sweep = 0; sweep < kMaxSweeps && G > 1; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < G - 1; ++round) {
      if (tid < G / 2) {
        int p, q;
        rr_pair(G, round, tid, p, q);
        double app = A[p + p * ld], aqq = A[q + q * ld], apq = A[p + q * ld];
        double c = 1.0, s = 0.0;
        double lim = fmax(kEps * sqrt(fabs(app) * fabs(aqq)), thr_abs);
        if (fabs(apq) > lim) {
          double theta = (aqq - app) / (2.0 * apq);
          double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          rotated = 1;
        }
        cs[p] = c;
        cs[q] = c;
        sn[p] = -s;  // J_qp = -s
        sn[q] = s;   // J_pq = +s
        partner[p] = q;
        partner[q] = p;
      }
      __syncthreads();
      for (int e = tid; e < G * G; e += nt) {
        const int i = e % G, j = e / G;
        const int pi = partner[i], pj = partner[j];
        const double ci = cs[i], si = sn[i], cj = cs[j], sj = sn[j];
        double v;
        if (j == pi) {
          v = 0.0;  // annihilated pair element
        } else if (i == j) {
          // a'_ii = c^2 a_ii + 2 c s' a_i,pi + s'^2 a_pi,pi  (s' = sigma s)
          double aii = A[i + i * ld], aip = A[i + pi * ld], app = A[pi + pi * ld];
          v = ci * ci * aii + 2.0 * ci * si * aip + si * si * app;
        } else {
          v = ci * cj * A[i + j * ld] + ci * sj * A[i + pj * ld] + si * cj * A[pi + j * ld] +
              si * sj * A[pi + pj * ld];
        }
        An[i + j * ld] = v;
        Vn[i + j * ld] = cj * V[i + j * ld] + sj * V[i + pj * ld];
      }
      __syncthreads();
      double *t1 = A;
      A = An;
      An = t1;
      double *t2 = V;
      V = Vn;
      Vn = t2;
    }
    if (!rotated) break;
  }
  // ordering (ascending with index tie-break, then the target rule)
  if (tid < g) {
    const int i = tid;
    const double wi = A[i + i * ld];
    int rank = 0;
    for (int j = 0; j < g; ++j) {
      double wj = A[j + j * ld];
      if (wj < wi || (wj == wi && j < i)) ++rank;
    }
    int pos = 0;
    if (order == SVDSB_ORDER_ASC) {
      pos = rank;
    } else {
      for (int j = 0; j < g; ++j) {
        if (j == i) continue;
        double wj = A[j + j * ld];
        int rj = 0;
        for (int k = 0; k < g; ++k) {
          double wk = A[k + k * ld];
          if (wk < wj || (wk == wj && k < j)) ++rj;
        }
        bool before;
        if (order == SVDSB_ORDER_DESC) {
          before = (wj > wi) || (wj == wi && rj < rank);
        } else {
          int bi = wi < shift, bj = wj < shift;
          double ki = bi ? shift - wi : wi - shift;
          double kj = bj ? shift - wj : wj - shift;
          before = (bj < bi) || (bj == bi && (kj < ki || (kj == ki && rj < rank)));
        }
        if (before) ++pos;
      }
    }
    w_out[pos] = wi;
    for (int r = 0; r < g; ++r) y_out[r + (int64_t)pos * ldy] = V[r + i * ld];
  }
}

// ------------------------------------------------------------ refined SVD

__global__ void __launch_bounds__(kSmallThreads)
refined_kernel(int g, const double *__restrict__ r, int64_t ldr, const double *__restrict__ h, int64_t ldh,
               double *y_out, double *lam_out, double *sv_out) {
  extern __shared__ double sm[];
  const int G = g + (g & 1);
  const int ld = G + 1;
  double *U = sm, *V = U + G * ld;
  double *yv = V + G * ld;
  __shared__ int rotated;
  __shared__ double sig[SVDSB_SMALL_MAX];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < G * G; e += blockDim.x) {
    int i = e % G, j = e / G;
    U[i + j * ld] = (i < g && j < g) ? r[i + (int64_t)j * ldr] : 0.0;
    V[i + j * ld] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < kMaxSweeps && G > 1; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < G - 1; ++round) {
      for (int k = wid; k < G / 2; k += nw) {
        int p, q;
        rr_pair(G, round, k, p, q);
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = lane; i < G; i += 32) {
          double up = U[i + p * ld], uq = U[i + q * ld];
          a = fma(up, up, a);
          b = fma(uq, uq, b);
          c = fma(up, uq, c);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        if (c != 0.0 && fabs(c) > kEps * sqrt(a * b)) {
          double zeta = (b - a) / (2.0 * c);
          double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          double cc = 1.0 / sqrt(1.0 + t * t), ss = cc * t;
          for (int i = lane; i < G; i += 32) {
            double up = U[i + p * ld], uq = U[i + q * ld];
            U[i + p * ld] = cc * up - ss * uq;
            U[i + q * ld] = ss * up + cc * uq;
            double vp = V[i + p * ld], vq = V[i + q * ld];
            V[i + p * ld] = cc * vp - ss * vq;
            V[i + q * ld] = ss * vp + cc * vq;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
  }
  for (int j = wid; j < g; j += nw) {
    double s = 0.0;
    for (int i = lane; i < G; i += 32) s = fma(U[i + j * ld], U[i + j * ld], s);
    s = warp_sum(s);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  __shared__ int jmin;
  if (tid == 0) {
    // the last right singular vector of an SVD sorted descending: the
    // smallest value, ties resolved to the highest index
    int best = 0;
    for (int j = 1; j < g; ++j)
      if (sig[j] <= sig[best]) best = j;
    jmin = best;
  }
  __syncthreads();
  if (tid < g) yv[tid] = V[tid + jmin * ld];
  __syncthreads();
  if (tid < g) y_out[tid] = yv[tid];
  if (sv_out && tid < g) {
    // descending order with index tie-break
    double si = sig[tid];
    int pos = 0;
    for (int j = 0; j < g; ++j)
      if (sig[j] > si || (sig[j] == si && j < tid)) ++pos;
    sv_out[pos] = si;
  }
  if (wid == 0) {
    // lam = y^T H y
    double acc = 0.0;
    for (int i = lane; i < g; i += 32) {
      double hy = 0.0;
      for (int j = 0; j < g; ++j) hy = fma(h[i + (int64_t)j * ldh], yv[j], hy);
      acc = fma(yv[i], hy, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) *lam_out = acc;
  }
}

// ------------------------------------------------------- restart coefs
// One warp, faithful modified Gram-Schmidt of eigensolver.py:438-459.

__device__ void warp_gs_candidates(int g, const double *cand, int64_t ldc, int ncand, const double *const *base,
                                   int nbase, double *kept, int ldk, int &nkept, int limit) {
  const int lane = threadIdx.x & 31;
  for (int ci = 0; ci < ncand; ++ci) {
    if (nkept >= limit) break;
    double c0 = (lane < g) ? cand[lane + ci * ldc] : 0.0;
    double c1 = (lane + 32 < g) ? cand[lane + 32 + ci * ldc] : 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int b = 0; b < nbase; ++b) {
        const double *bv = base[b];
        double b0 = (lane < g) ? bv[lane] : 0.0, b1 = (lane + 32 < g) ? bv[lane + 32] : 0.0;
        double d = warp_sum(b0 * c0 + b1 * c1);
        c0 -= b0 * d;
        c1 -= b1 * d;
      }
      for (int k = 0; k < nkept; ++k) {
        const double *bv = kept + k * ldk;
        double b0 = (lane < g) ? bv[lane] : 0.0, b1 = (lane + 32 < g) ? bv[lane + 32] : 0.0;
        double d = warp_sum(b0 * c0 + b1 * c1);
        c0 -= b0 * d;
        c1 -= b1 * d;
      }
    }
    double nrm = sqrt(warp_sum(c0 * c0 + c1 * c1));
    if (nrm > 1e-8) {
      double *o = kept + nkept * ldk;
      if (lane < g) o[lane] = c0 / nrm;
      if (lane + 32 < g) o[lane + 32] = c1 / nrm;
      __syncwarp();
      ++nkept;
    }
  }
}

__global__ void restart_coefs_kernel(int g, int gmax, const double *__restrict__ yfirst,
                                     const double *__restrict__ yall, int64_t ldy, int ny, int retain,
                                     const double *__restrict__ exclude, const double *__restrict__ prev,
                                     int64_t ldp, int nprev, int prev_g, int plus_k, double *out, int64_t ldo,
                                     int *count_dev) {
  extern __shared__ double sm[];
  double *kept = sm;              // g x g
  double *cand = sm + g * g;      // g x (g + 1)
  const int lane = threadIdx.x;
  // priority list: [yfirst] + columns of yall
  int nc = 0;
  if (yfirst) {
    for (int i = lane; i < g; i += 32) cand[i] = yfirst[i];
    nc = 1;
  }
  for (int j = 0; j < ny; ++j)
    for (int i = lane; i < g; i += 32) cand[i + (nc + j) * g] = yall[i + (int64_t)j * ldy];
  nc += ny;
  __syncwarp();
  const double *base[SVDSB_SMALL_MAX + 1];
  int nbase = 0;
  if (exclude) base[nbase++] = exclude;
  int nsel = 0;
  warp_gs_candidates(g, cand, g, nc, base, nbase, kept, g, nsel, retain);
  __syncwarp();
  int ntot = nsel;
  int p_budget = min(plus_k, gmax - 1 - nsel);
  if (p_budget > 0 && prev != nullptr && prev_g <= g && nprev > 0) {
    // padded previous coefficients (eigensolver.py:461-469)
    for (int j = 0; j < nprev; ++j)
      for (int i = lane; i < g; i += 32) cand[i + j * g] = (i < prev_g) ? prev[i + (int64_t)j * ldp] : 0.0;
    __syncwarp();
    for (int k = 0; k < nsel; ++k) base[nbase++] = kept + k * g;
    int nplus = 0;
    warp_gs_candidates(g, cand, g, nprev, base, nbase, kept + nsel * g, g, nplus, p_budget);
    ntot += nplus;
  }
  __syncwarp();
  for (int j = 0; j < ntot; ++j)
    for (int i = lane; i < g; i += 32) out[i + (int64_t)j * ldo] = kept[i + j * g];
  if (lane == 0) *count_dev = ntot;
}

// --------------------------------------------------- H <- sym(C^T H C)

__global__ void project_small_kernel(int g, int s, const double *__restrict__ h, int64_t ldh,
                                     const double *__restrict__ c, int64_t ldc, double *hout, int64_t ldho) {
  extern __shared__ double sm[];
  double *Hs = sm, *Cs = Hs + g * g, *T = Cs + g * s, *P = T + g * s;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < g * g; e += nt) Hs[e] = h[(e % g) + (int64_t)(e / g) * ldh];
  for (int e = tid; e < g * s; e += nt) Cs[e] = c[(e % g) + (int64_t)(e / g) * ldc];
  __syncthreads();
  for (int e = tid; e < g * s; e += nt) {  // T = H C
    int i = e % g, j = e / g;
    double acc = 0.0;
    for (int k = 0; k < g; ++k) acc = fma(Hs[i + k * g], Cs[k + j * g], acc);
    T[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < s * s; e += nt) {  // P = C^T T
    int i = e % s, j = e / s;
    double acc = 0.0;
    for (int k = 0; k < g; ++k) acc = fma(Cs[k + i * g], T[k + j * g], acc);
    P[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < s * s; e += nt) {
    int i = e % s, j = e / s;
    hout[i + (int64_t)j * ldho] = 0.5 * (P[i + j * s] + P[j + i * s]);
  }
}

// ---------------------------------------------------- QR of R*Y (thin)

__global__ void qr_small_kernel(int g, int s, const double *__restrict__ r, int64_t ldr,
                                const double *__restrict__ yc, int64_t ldy, double *qy, int64_t ldq, double *ry,
                                int64_t ldry) {
  extern __shared__ double sm[];
  double *M = sm;            // g x s  (column-major, ld g)
  double *Vh = M + g * s;    // g x s  Householder vectors
  double *tau = Vh + g * s;  // s
  double *Q = tau + s;       // g x s
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < g * s; e += nt) {  // M = R Y (R upper triangular)
    int i = e % g, j = e / g;
    double acc = 0.0;
    for (int k = i; k < g; ++k) acc = fma(r[i + (int64_t)k * ldr], yc[k + (int64_t)j * ldy], acc);
    M[e] = acc;
  }
  __syncthreads();
  __shared__ double alpha_s;
  for (int k = 0; k < s; ++k) {
    if (wid == 0) {
      double nrm2 = 0.0;
      for (int i = k + lane; i < g; i += 32) nrm2 = fma(M[i + k * g], M[i + k * g], nrm2);
      nrm2 = warp_sum(nrm2);
      double x0 = M[k + k * g];
      double nrm = sqrt(nrm2);
      double alpha = (x0 >= 0.0) ? -nrm : nrm;
      // v = x - alpha e1 ; tau = 2 / v^T v
      for (int i = lane; i < g; i += 32) Vh[i + k * g] = (i < k) ? 0.0 : ((i == k) ? x0 - alpha : M[i + k * g]);
      double vtv = nrm2 - x0 * x0 + (x0 - alpha) * (x0 - alpha);
      if (lane == 0) {
        tau[k] = (nrm == 0.0 || vtv == 0.0) ? 0.0 : 2.0 / vtv;
        alpha_s = (nrm == 0.0) ? x0 : alpha;
      }
    }
    __syncthreads();
    for (int j = k + 1 + wid; j < s; j += nw) {  // apply to trailing columns
      double d = 0.0;
      for (int i = k + lane; i < g; i += 32) d = fma(Vh[i + k * g], M[i + j * g], d);
      d = warp_sum(d) * tau[k];
      for (int i = k + lane; i < g; i += 32) M[i + j * g] -= d * Vh[i + k * g];
    }
    __syncthreads();
    if (tid == 0) M[k + k * g] = alpha_s;
    for (int i = k + 1 + tid; i < g; i += nt) M[i + k * g] = 0.0;
    __syncthreads();
  }
  // Q = H_0 ... H_{s-1} [I; 0]
  for (int e = tid; e < g * s; e += nt) Q[e] = ((e % g) == (e / g)) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = s - 1; k >= 0; --k) {
    for (int j = wid; j < s; j += nw) {
      double d = 0.0;
      for (int i = k + lane; i < g; i += 32) d = fma(Vh[i + k * g], Q[i + j * g], d);
      d = warp_sum(d) * tau[k];
      for (int i = k + lane; i < g; i += 32) Q[i + j * g] -= d * Vh[i + k * g];
    }
    __syncthreads();
  }
  // sign fix: diag(R) >= 0
  for (int e = tid; e < g * s; e += nt) {
    int j = e / g;
    double sg = (M[j + j * g] < 0.0) ? -1.0 : 1.0;
    qy[(e % g) + (int64_t)j * ldq] = Q[e] * sg;
  }
  for (int e = tid; e < s * s; e += nt) {
    int i = e % s, j = e / s;
    double sg = (M[i + i * g] < 0.0) ? -1.0 : 1.0;
    ry[i + (int64_t)j * ldry] = (i <= j) ? M[i + j * g] * sg : 0.0;
  }
}

// ------------------------------------------------------- H bookkeeping

__global__ void h_insert_kernel(int g, int b, const double *__restrict__ hc, int64_t ldhc, double *h, int64_t ldh) {
  pdl_wait();
  pdl_trigger();
  const int gb = g + b;
  for (int e = threadIdx.x; e < gb * b; e += blockDim.x) {
    int i = e % gb, j = e / gb;  // hc(i, j) -> H(i, g+j)
    double v = hc[i + (int64_t)j * ldhc];
    if (i < g) {
      h[i + (int64_t)(g + j) * ldh] = v;
      h[(g + j) + (int64_t)i * ldh] = v;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    int i = e % b, j = e / b;
    double v = 0.5 * (hc[(g + i) + (int64_t)j * ldhc] + hc[(g + j) + (int64_t)i * ldhc]);
    h[(g + i) + (int64_t)(g + j) * ldh] = v;
  }
}

__global__ void h_sym_kernel(int g, const double *__restrict__ gm, int64_t ldg, double *h, int64_t ldh) {
  for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < g * g; e += blockDim.x * gridDim.x) {
    int i = e % g, j = e / g;
    h[i + (int64_t)j * ldh] = 0.5 * (gm[i + (int64_t)j * ldg] + gm[j + (int64_t)i * ldg]);
  }
}

static bool g_attr_set = false;

static int ensure_attrs() {
  if (g_attr_set) return SVDSB_OK;
  SVDSB_CUDA(cudaFuncSetAttribute(syev_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  SVDSB_CUDA(cudaFuncSetAttribute(refined_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  SVDSB_CUDA(cudaFuncSetAttribute(project_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  SVDSB_CUDA(cudaFuncSetAttribute(restart_coefs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  SVDSB_CUDA(cudaFuncSetAttribute(qr_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  g_attr_set = true;
  return SVDSB_OK;
}

}  // namespace svdsb

using namespace svdsb;

extern "C" {

int svdsb_syev_small(int g, const double *h, int64_t ldh, int order, double shift, double *w, double *y, int64_t ldy,
                     void *stream) {
  SVDSB_CHECK_ARG(g >= 1 && g <= SVDSB_SMALL_MAX, "svdsb_syev_small: g out of range");
  SVDSB_CHECK_ARG(order >= 0 && order <= 2, "svdsb_syev_small: bad order");
  int rc = ensure_attrs();
  if (rc) return rc;
  const int G = g + (g & 1);
  size_t sh = sizeof(double) * (4 * G * (G + 1) + 2 * G) + sizeof(int) * G;
  syev_jacobi_kernel<<<1, kSmallThreads, sh, as_stream(stream)>>>(g, h, ldh, order, shift, w, y, ldy);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_refined_small(int g, const double *r, int64_t ldr, const double *h, int64_t ldh, double *y, double *lam,
                        double *sv, void *stream) {
  SVDSB_CHECK_ARG(g >= 1 && g <= SVDSB_SMALL_MAX, "svdsb_refined_small: g out of range");
  int rc = ensure_attrs();
  if (rc) return rc;
  const int G = g + (g & 1);
  size_t sh = sizeof(double) * (2 * G * (G + 1) + G);
  refined_kernel<<<1, kSmallThreads, sh, as_stream(stream)>>>(g, r, ldr, h, ldh, y, lam, sv);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_restart_coefs(int g, int gmax, const double *yfirst, const double *yall, int64_t ldy, int ny, int retain,
                        const double *exclude, const double *prev, int64_t ldp, int nprev, int prev_g, int plus_k,
                        double *out, int64_t ldo, int *count_dev, void *stream) {
  SVDSB_CHECK_ARG(g >= 1 && g <= SVDSB_SMALL_MAX, "svdsb_restart_coefs: g out of range");
  SVDSB_CHECK_ARG(ny + (yfirst ? 1 : 0) <= SVDSB_SMALL_MAX + 1 && nprev <= SVDSB_SMALL_MAX,
                  "svdsb_restart_coefs: too many candidates");
  int rc = ensure_attrs();
  if (rc) return rc;
  size_t sh = sizeof(double) * (g * g + g * (std::max(ny + 1, nprev) + 1));
  restart_coefs_kernel<<<1, 32, sh, as_stream(stream)>>>(g, gmax, yfirst, yall, ldy, ny, retain, exclude, prev, ldp,
                                                        nprev, prev_g, plus_k, out, ldo, count_dev);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_project_small(int g, int s, const double *h, int64_t ldh, const double *c, int64_t ldc, double *hout,
                        int64_t ldho, void *stream) {
  SVDSB_CHECK_ARG(g >= 1 && g <= SVDSB_SMALL_MAX && s >= 0 && s <= g, "svdsb_project_small: bad sizes");
  if (s == 0) return SVDSB_OK;
  int rc = ensure_attrs();
  if (rc) return rc;
  size_t sh = sizeof(double) * (g * g + 2 * g * s + s * s);
  project_small_kernel<<<1, 256, sh, as_stream(stream)>>>(g, s, h, ldh, c, ldc, hout, ldho);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_qr_small(int g, int s, const double *r, int64_t ldr, const double *yc, int64_t ldy, double *qy,
                   int64_t ldq, double *ry, int64_t ldry, void *stream) {
  SVDSB_CHECK_ARG(g >= 1 && g <= SVDSB_SMALL_MAX && s >= 1 && s <= g, "svdsb_qr_small: bad sizes");
  int rc = ensure_attrs();
  if (rc) return rc;
  size_t sh = sizeof(double) * (3 * g * s + s);
  qr_small_kernel<<<1, 256, sh, as_stream(stream)>>>(g, s, r, ldr, yc, ldy, qy, ldq, ry, ldry);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_h_insert(int g, int b, const double *hc, int64_t ldhc, double *h, int64_t ldh, void *stream) {
  if (b <= 0) return SVDSB_OK;
  SVDSB_LAUNCH_PDL(h_insert_kernel, 1, 256, 0, as_stream(stream), g, b, hc, ldhc, h, ldh);
  return SVDSB_OK;
}

int svdsb_h_symmetrize(int g, const double *gm, int64_t ldg, double *h, int64_t ldh, void *stream) {
  if (g <= 0) return SVDSB_OK;
  SVDSB_CHECK_ARG(gm != h, "svdsb_h_symmetrize: in-place not supported");
  h_sym_kernel<<<(g * g + 255) / 256, 256, 0, as_stream(stream)>>>(g, gm, ldg, h, ldh);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

}  // extern "C"
