// Tall-skinny fp64 kernels for the Davidson basis (HBM-bound streaming).
//
// All operands are column-major with an explicit leading dimension.  Every
// kernel streams rows: CTA `bx` owns a contiguous row range, each thread
// walks rows `tid, tid+256, ...` of it and touches all the columns it needs
// for that row (coalesced 256-byte warp accesses per column).  Reductions
// (Gram entries, norms) are two-level: warp shuffle + CTA fold into a
// per-CTA partial, then the last CTA to finish (ticket) folds the partials
// in CTA order.  The grid depends only on the row count, so results are
// bit-reproducible run to run.
//
// Reference operations (pkg/src/itersvd): kernels.py:47-51 (_project_out),
// :104-111 (norms), :497-499 (qr_append projection), eigensolver.py:349-352
// (V^T W), :385-394 (_candidates), :526-527 (restart V @ coefs),
// :690 (H column), hybrid.py:226-241 (stage-2 split residual).
#include <cuda.h>
#include <algorithm>

#include "common.cuh"

namespace svdsb {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMinRowsPerCta = 256;

struct ColSet {
  const double *base[SVDSB_MAX_BLOCKS];
  int64_t ld[SVDSB_MAX_BLOCKS];
  int cols[SVDSB_MAX_BLOCKS];
  int nblk;
  int total;
};

__device__ __forceinline__ const double *colset_ptr(const ColSet &s, int i) {
  int k = 0;
  while (k < s.nblk - 1 && i >= s.cols[k]) {
    i -= s.cols[k];
    ++k;
  }
  return s.base[k] + (int64_t)i * s.ld[k];
}

struct RowRange {
  int64_t r0, r1;
};

__device__ __forceinline__ RowRange cta_rows(int64_t dim) {
  int64_t per = (dim + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per;
  int64_t r1 = min(dim, r0 + per);
  return {r0, r1};
}

// Fold NACC per-thread accumulators over the CTA into part[0..nvalid).
template <int NACC>
__device__ __forceinline__ void cta_fold(double (&acc)[NACC], int nvalid, double *part) {
  __shared__ double red[kWarps][NACC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NACC; ++k) {
    double v = warp_sum(acc[k]);
    if (lane == 0) red[w][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nvalid; k += kThreads) {
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += red[ww][k];
    part[k] = s;
  }
}

static inline int grid_rows(int64_t dim) { return stream_grid(dim, kMinRowsPerCta, 8 * num_sms()); }

// Persistent-style grid: one wave of resident CTAs (occupancy x 148 SMs),
// each looping over its contiguous row range.  Cached per (kernel, smem).
template <typename K>
static int grid_for(K kernel, int64_t dim, size_t smem) {
  struct Entry {
    const void *k;
    size_t smem;
    int cap;
  };
  static Entry cache[64];
  static int ncache = 0;
  const void *kp = reinterpret_cast<const void *>(kernel);
  int cap = 0;
  for (int i = 0; i < ncache; ++i)
    if (cache[i].k == kp && cache[i].smem == smem) cap = cache[i].cap;
  if (cap == 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
    cap = occ * num_sms();
    if (ncache < 64) cache[ncache++] = {kp, smem, cap};
  }
  return stream_grid(dim, kMinRowsPerCta, cap);
}

// ------------------------------------------------------------------ gram

template <int AT, int BT>
__global__ void __launch_bounds__(kThreads)
gram_kernel(int64_t dim, ColSet xs, const double *__restrict__ y, int64_t ldy, int b, double *c, int64_t ldc,
            double *norms2, double *partials, unsigned int *ticket) {
  __shared__ const double *xp[AT];
  const int ty = blockIdx.y, tz = blockIdx.z;
  const int i0 = ty * AT, j0 = tz * BT;
  const int na = min(AT, xs.total - i0), nb = min(BT, b - j0);
  const bool want_norm = (norms2 != nullptr) && ty == 0;
  if (threadIdx.x < AT && (int)threadIdx.x < na) xp[threadIdx.x] = colset_ptr(xs, i0 + threadIdx.x);
  __syncthreads();
  double acc[AT * BT + BT];
#pragma unroll
  for (int k = 0; k < AT * BT + BT; ++k) acc[k] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t r = rr.r0 + threadIdx.x; r < rr.r1; r += kThreads) {
    double yv[BT];
#pragma unroll
    for (int j = 0; j < BT; ++j) yv[j] = (j < nb) ? __ldg(y + r + (int64_t)(j0 + j) * ldy) : 0.0;
#pragma unroll
    for (int i = 0; i < AT; ++i) {
      if (i < na) {
        double xv = __ldg(xp[i] + r);
#pragma unroll
        for (int j = 0; j < BT; ++j) acc[i * BT + j] = fma(xv, yv[j], acc[i * BT + j]);
      }
    }
    if (want_norm) {
#pragma unroll
      for (int j = 0; j < BT; ++j) acc[AT * BT + j] = fma(yv[j], yv[j], acc[AT * BT + j]);
    }
  }
  constexpr int NOUT = AT * BT + BT;
  const int tile = ty * gridDim.z + tz;
  double *part = partials + ((int64_t)tile * gridDim.x + blockIdx.x) * NOUT;
  cta_fold<NOUT>(acc, NOUT, part);
  if (!last_cta(ticket)) return;
  const int ntile = gridDim.y * gridDim.z;
  fold_parts(partials, gridDim.x, NOUT, ntile * NOUT, [&](int, int t, int k, double s) {
    const int tyy = t / gridDim.z, tzz = t % gridDim.z;
    if (k < AT * BT) {
      int i = tyy * AT + k / BT, j = tzz * BT + k % BT;
      if (i < xs.total && j < b) c[i + (int64_t)j * ldc] = s;
    } else if (norms2 != nullptr && tyy == 0) {
      int j = tzz * BT + (k - AT * BT);
      if (j < b) norms2[j] = s;
    }
  });
}

// ------------------------------------------------------------ project out

template <int BT>
__global__ void __launch_bounds__(kThreads)
project_kernel(int64_t dim, ColSet xs, const double *__restrict__ cmat, int64_t ldc, double *y, int64_t ldy,
               int b, double *norms2, double *partials, unsigned int *ticket) {
  extern __shared__ double csh[];  // total x BT
  __shared__ const double *xp[256];
  const int na = xs.total;
  for (int i = threadIdx.x; i < na; i += kThreads) xp[i] = colset_ptr(xs, i);
  for (int k = threadIdx.x; k < na * BT; k += kThreads) {
    int i = k / BT, j = k % BT;
    csh[k] = (j < b) ? cmat[i + (int64_t)j * ldc] : 0.0;
  }
  __syncthreads();
  double nacc[BT];
#pragma unroll
  for (int j = 0; j < BT; ++j) nacc[j] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t r = rr.r0 + threadIdx.x; r < rr.r1; r += kThreads) {
    double yv[BT];
#pragma unroll
    for (int j = 0; j < BT; ++j) yv[j] = (j < b) ? y[r + (int64_t)j * ldy] : 0.0;
    for (int i = 0; i < na; ++i) {
      double xv = __ldg(xp[i] + r);
#pragma unroll
      for (int j = 0; j < BT; ++j) yv[j] = fma(-xv, csh[i * BT + j], yv[j]);
    }
#pragma unroll
    for (int j = 0; j < BT; ++j) {
      if (j < b) {
        y[r + (int64_t)j * ldy] = yv[j];
        nacc[j] = fma(yv[j], yv[j], nacc[j]);
      }
    }
  }
  if (norms2 == nullptr) return;
  double *part = partials + (int64_t)blockIdx.x * BT;
  cta_fold<BT>(nacc, BT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, BT, b, [&](int j, int, int, double s) { norms2[j] = s; });
}

// ---------------------------------------------------------------- ts_gemm

template <int ST>
__global__ void __launch_bounds__(kThreads)
ts_gemm_kernel(int64_t dim, const double *__restrict__ x, int64_t ldx, int g, const double *__restrict__ cmat,
               int64_t ldc, int s, double alpha, double beta, double *__restrict__ y, int64_t ldy) {
  extern __shared__ double csh[];  // g x ST (row i: csh[i*ST + j])
  const int j0 = blockIdx.y * ST;
  const int ns = min(ST, s - j0);
  for (int k = threadIdx.x; k < g * ST; k += kThreads) {
    int i = k / ST, j = k % ST;
    csh[k] = (j < ns) ? cmat[i + (int64_t)(j0 + j) * ldc] : 0.0;
  }
  __syncthreads();
  RowRange rr = cta_rows(dim);
  for (int64_t r = rr.r0 + threadIdx.x; r < rr.r1; r += kThreads) {
    double acc[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) acc[j] = 0.0;
    for (int i = 0; i < g; ++i) {
      double xv = __ldg(x + r + (int64_t)i * ldx);
#pragma unroll
      for (int j = 0; j < ST; ++j) acc[j] = fma(xv, csh[i * ST + j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      if (j < ns) {
        double *yp = y + r + (int64_t)(j0 + j) * ldy;
        double out = alpha * acc[j];
        if (beta != 0.0) out = fma(beta, *yp, out);
        *yp = out;
      }
    }
  }
}

// ---------------------------------------------------------- ritz residual

template <int PT>
__global__ void __launch_bounds__(kThreads)
ritz_kernel(int64_t dim, const double *__restrict__ v, int64_t ldv, const double *__restrict__ w, int64_t ldw,
            int g, const double *__restrict__ yc, int64_t ldyc, const double *__restrict__ lam, int p,
            double *__restrict__ r, int64_t ldr, double *__restrict__ xo, int64_t ldx, double *__restrict__ oxo,
            int64_t ldox, double *rn2, double *partials, unsigned int *ticket) {
  extern __shared__ double ysh[];  // g x PT
  __shared__ double lsh[PT];
  const int j0 = blockIdx.y * PT;
  const int np = min(PT, p - j0);
  for (int k = threadIdx.x; k < g * PT; k += kThreads) {
    int i = k / PT, j = k % PT;
    ysh[k] = (j < np) ? yc[i + (int64_t)(j0 + j) * ldyc] : 0.0;
  }
  if (threadIdx.x < PT) lsh[threadIdx.x] = ((int)threadIdx.x < np) ? lam[j0 + threadIdx.x] : 0.0;
  __syncthreads();
  double nacc[PT];
#pragma unroll
  for (int j = 0; j < PT; ++j) nacc[j] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t row = rr.r0 + threadIdx.x; row < rr.r1; row += kThreads) {
    double ax[PT], aw[PT];
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      ax[j] = 0.0;
      aw[j] = 0.0;
    }
    for (int i = 0; i < g; ++i) {
      double vv = __ldg(v + row + (int64_t)i * ldv);
      double ww = __ldg(w + row + (int64_t)i * ldw);
#pragma unroll
      for (int j = 0; j < PT; ++j) {
        double cf = ysh[i * PT + j];
        ax[j] = fma(vv, cf, ax[j]);
        aw[j] = fma(ww, cf, aw[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      if (j < np) {
        double res = __dsub_rn(aw[j], __dmul_rn(ax[j], lsh[j]));  // R = OpX - X*lam, two roundings (no fma), eigensolver.py:392
        r[row + (int64_t)(j0 + j) * ldr] = res;
        if (xo) xo[row + (int64_t)(j0 + j) * ldx] = ax[j];
        if (oxo) oxo[row + (int64_t)(j0 + j) * ldox] = aw[j];
        nacc[j] = fma(res, res, nacc[j]);
      }
    }
  }
  double *part = partials + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * PT;
  cta_fold<PT>(nacc, PT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, PT, (int)gridDim.y * PT, [&](int o, int, int, double s) {
    if (o < p) rn2[o] = s;
  });
}

// -------------------------------------------------------- norms and dots

template <int BT>
__global__ void __launch_bounds__(kThreads)
coldot_kernel(int64_t dim, const double *__restrict__ x, int64_t ldx, const double *__restrict__ y, int64_t ldy,
              int b, double *out, double *partials, unsigned int *ticket) {
  const int j0 = blockIdx.y * BT;
  const int nb = min(BT, b - j0);
  double acc[BT];
#pragma unroll
  for (int j = 0; j < BT; ++j) acc[j] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t r = rr.r0 + threadIdx.x; r < rr.r1; r += kThreads) {
#pragma unroll
    for (int j = 0; j < BT; ++j)
      if (j < nb) acc[j] = fma(__ldg(x + r + (int64_t)(j0 + j) * ldx), __ldg(y + r + (int64_t)(j0 + j) * ldy), acc[j]);
  }
  double *part = partials + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * BT;
  cta_fold<BT>(acc, BT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, BT, (int)gridDim.y * BT, [&](int o, int, int, double s) {
    if (o < b) out[o] = s;
  });
}

template <int BT>
__global__ void __launch_bounds__(kThreads)
split_kernel(int64_t dim, int64_t nsplit, const double *__restrict__ r, int64_t ldr, const double *__restrict__ x,
             int64_t ldx, int b, double *out, double *partials, unsigned int *ticket) {
  const int j0 = blockIdx.y * BT;
  const int nb = min(BT, b - j0);
  double acc[6 * BT];
#pragma unroll
  for (int k = 0; k < 6 * BT; ++k) acc[k] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t row = rr.r0 + threadIdx.x; row < rr.r1; row += kThreads) {
    const int off = (row < nsplit) ? 0 : 3;
#pragma unroll
    for (int j = 0; j < BT; ++j) {
      if (j < nb) {
        double rv = __ldg(r + row + (int64_t)(j0 + j) * ldr);
        double xv = __ldg(x + row + (int64_t)(j0 + j) * ldx);
        acc[6 * j + off + 0] = fma(rv, rv, acc[6 * j + off + 0]);
        acc[6 * j + off + 1] = fma(rv, xv, acc[6 * j + off + 1]);
        acc[6 * j + off + 2] = fma(xv, xv, acc[6 * j + off + 2]);
      }
    }
  }
  double *part = partials + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 6 * BT;
  cta_fold<6 * BT>(acc, 6 * BT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, 6 * BT, (int)gridDim.y * 6 * BT, [&](int o, int ty, int k, double s) {
    if (ty * BT + k / 6 < b) out[o] = s;
  });
}

template <int BT>
__global__ void __launch_bounds__(kThreads)
split_res_kernel(int64_t dim, int64_t nsplit, const double *__restrict__ r, int64_t ldr, const double *__restrict__ x,
                 int64_t ldx, int b, const double *__restrict__ lam, const double *__restrict__ stats, double *out,
                 double *partials, unsigned int *ticket) {
  const int j0 = blockIdx.y * BT;
  const int nb = min(BT, b - j0);
  __shared__ double coef[BT][4];  // 1/nv, alpha, 1/nu, beta
  if (threadIdx.x < BT) {
    int j = threadIdx.x;
    if (j < nb) {
      const double *st = stats + 6 * (j0 + j);
      double nv = sqrt(st[2]), nu = sqrt(st[5]);
      double l = lam[j0 + j], sg = fabs(l);
      bool ok = nv > 0.0 && nu > 0.0;
      coef[j][0] = ok ? 1.0 / nv : 0.0;
      coef[j][1] = ok ? (l / nv - sg / nu) : 0.0;
      coef[j][2] = ok ? 1.0 / nu : 0.0;
      coef[j][3] = ok ? (l / nu - sg / nv) : 0.0;
    }
  }
  __syncthreads();
  double acc[BT];
#pragma unroll
  for (int j = 0; j < BT; ++j) acc[j] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t row = rr.r0 + threadIdx.x; row < rr.r1; row += kThreads) {
    const bool is_v = row < nsplit;
#pragma unroll
    for (int j = 0; j < BT; ++j) {
      if (j < nb) {
        double rv = __ldg(r + row + (int64_t)(j0 + j) * ldr);
        double xv = __ldg(x + row + (int64_t)(j0 + j) * ldx);
        // rows of the v part contribute to e2 = r_v/nu + beta x_v,
        // rows of the u part to e1 = r_u/nv + alpha x_u
        double e = is_v ? fma(coef[j][3], xv, rv * coef[j][2]) : fma(coef[j][1], xv, rv * coef[j][0]);
        acc[j] = fma(e, e, acc[j]);
      }
    }
  }
  double *part = partials + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * BT;
  cta_fold<BT>(acc, BT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, BT, (int)gridDim.y * BT, [&](int jj, int, int, double s) {
    if (jj >= b) return;
    const double *st = stats + 6 * jj;
    out[jj] = (st[2] > 0.0 && st[5] > 0.0) ? s : __longlong_as_double(0x7ff0000000000000LL);
  });
}

__global__ void scale_kernel(int64_t dim, const double *x, int64_t ldx, int b, const double *__restrict__ s, int mode,
                             double *y, int64_t ldy) {
  pdl_wait();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= dim) return;
  for (int j = 0; j < b; ++j) {
    double f = s[j];
    double xv = x[i + (int64_t)j * ldx];
    double out;
    if (mode == 0) {
      out = xv * f;
    } else {
      if (f == 0.0) {
        out = xv;
      } else {
        double d = (mode == 2) ? sqrt(f) : f;
        out = xv / d;
      }
    }
    y[i + (int64_t)j * ldy] = out;
  }
}

__global__ void gather_cols_kernel(int64_t dim, const double *x, int64_t ldx, const int *first, int ncols, int limit,
                                   const double *__restrict__ d, double *y, int64_t ldy) {
  pdl_wait();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= dim) return;
  const int f = *first;
  const double di = d ? d[i] : 1.0;
  for (int c = 0; c < ncols && f + c < limit; ++c) {
    const double v = x[i + (int64_t)(f + c) * ldx];
    y[i + (int64_t)c * ldy] = d ? __ddiv_rn(v, di) : v;
  }
}

// One kernel writes the iteration status straight into pinned host memory
// (mapped under UVA): Ritz values, candidate residual norms, DGKS state.
// Replaces three small device->host copies at the end of every graphed
// iteration.
__global__ void status_pack_kernel(const double *__restrict__ lams, int gn, const double *__restrict__ rn2, int p,
                                   const double *__restrict__ st, int nst, double *host) {
  pdl_wait();
  for (int i = threadIdx.x; i < gn + p + 8 * nst; i += blockDim.x) {
    double v;
    if (i < gn)
      v = lams[i];
    else if (i < gn + p)
      v = rn2[i - gn];
    else
      v = st[i - gn - p];
    host[i] = v;
  }
  __threadfence_system();
}

// Counter-based standard normals (Philox4x32-10 + Box-Muller) for the
// initial basis block of large problems: element (R, c) of a grows x cols
// block is a pure function of (seed, R * cols + c), so every row partition
// draws the same global block and reruns are bit-reproducible.
__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0, h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
  c[0] = h1 ^ c[1] ^ k0;
  c[1] = l1;
  c[2] = h0 ^ c[3] ^ k1;
  c[3] = l0;
}

__global__ void randn_kernel(uint64_t seed, int64_t row0, int64_t rows, int cols, double *__restrict__ out,
                             int64_t ldo) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i % rows, c = i / rows;          // column-major walk: coalesced stores
  const uint64_t e = (uint64_t)(row0 + r) * (uint64_t)cols + (uint64_t)c;
  uint32_t x[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0x5fd0u, 0u};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    philox_round(x, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint64_t a = ((uint64_t)x[0] << 21) ^ (uint64_t)x[1];   // 53 bits used below
  const uint64_t b = ((uint64_t)x[2] << 21) ^ (uint64_t)x[3];
  const double u1 = ((double)(a & ((1ull << 53) - 1)) + 0.5) * 0x1p-53;   // (0, 1)
  const double u2 = (double)(b & ((1ull << 53) - 1)) * 0x1p-53;           // [0, 1)
  out[r + c * ldo] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__global__ void set_int_kernel(int *dst, int v) {
  pdl_wait();
  if (threadIdx.x == 0) *dst = v;
}

__global__ void axpby_kernel(int64_t dim, int b, double alpha, const double *x, int64_t ldx, double beta, double *y,
                             int64_t ldy) {
  pdl_wait();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= dim) return;
  for (int j = 0; j < b; ++j) {
    double *yp = y + i + (int64_t)j * ldy;
    double out = alpha * x[i + (int64_t)j * ldx];
    if (beta != 0.0) out = fma(beta, *yp, out);
    *yp = out;
  }
}

// ------------------------------------------------- 2-row vectorised paths
// Each thread owns row pairs (r, r+1): every column access is one 16-byte
// load, twice the bytes in flight per instruction of the scalar kernels.
// Used when every base pointer is 16-byte aligned and every leading
// dimension is even (always true for blocks allocated by the package).

__device__ __forceinline__ RowRange cta_rows_even(int64_t dim, int bx, int nx) {
  int64_t per = (dim + nx - 1) / nx;
  per += per & 1;
  int64_t r0 = (int64_t)bx * per;
  int64_t r1 = min(dim, r0 + per);
  return {r0, r1};
}
__device__ __forceinline__ RowRange cta_rows_even(int64_t dim) { return cta_rows_even(dim, blockIdx.x, gridDim.x); }

__device__ __forceinline__ double2 ldg2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

template <int AT>
__global__ void __launch_bounds__(kThreads)
gram1_vec_kernel(int64_t dim, ColSet xs, const double *__restrict__ y, double *c, double *norms2, double *partials,
                 unsigned int *ticket, const double *gate, HInsert hi) {
  pdl_wait();
  if (gate != nullptr && gate[0] == 0.0) return;  // device-side DGKS: column already final
  __shared__ const double *xp[AT];
  const int ty = blockIdx.y;
  const int i0 = ty * AT;
  const int na = min(AT, xs.total - i0);
  const bool want_norm = norms2 != nullptr && ty == 0;
  if (threadIdx.x < AT && (int)threadIdx.x < na) xp[threadIdx.x] = colset_ptr(xs, i0 + threadIdx.x);
  __syncthreads();
  double acc[AT + 1];
#pragma unroll
  for (int k = 0; k <= AT; ++k) acc[k] = 0.0;
  RowRange rr = cta_rows_even(dim);
  int64_t r = rr.r0 + 2 * threadIdx.x;
  for (; r + 1 < rr.r1; r += 2 * kThreads) {
    double2 yv = ldg2(y + r);
#pragma unroll
    for (int i = 0; i < AT; ++i) {
      if (i < na) {
        double2 xv = ldg2(xp[i] + r);
        acc[i] = fma(xv.x, yv.x, fma(xv.y, yv.y, acc[i]));
      }
    }
    if (want_norm) acc[AT] = fma(yv.x, yv.x, fma(yv.y, yv.y, acc[AT]));
  }
  if (r < rr.r1) {  // odd tail row
    double yv = __ldg(y + r);
#pragma unroll
    for (int i = 0; i < AT; ++i)
      if (i < na) acc[i] = fma(__ldg(xp[i] + r), yv, acc[i]);
    if (want_norm) acc[AT] = fma(yv, yv, acc[AT]);
  }
  pdl_trigger();
  constexpr int NOUT = AT + 1;
  double *part = partials + ((int64_t)ty * gridDim.x + blockIdx.x) * NOUT;
  cta_fold<NOUT>(acc, NOUT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, NOUT, (int)gridDim.y * NOUT, [&](int, int t, int k, double s) {
    if (k < AT) {
      int i = t * AT + k;
      if (i < xs.total) {
        c[i] = s;
        if (hi.h != nullptr && i <= hi.g) {  // H(i, g) = H(g, i); H(g, g) = (c_g + c_g) / 2 = c_g
          hi.h[i + (int64_t)hi.g * hi.ldh] = s;
          hi.h[hi.g + (int64_t)i * hi.ldh] = s;
        }
      }
    } else if (norms2 != nullptr && t == 0) {
      norms2[0] = s;
    }
  });
}

// b = 4 Gram C = X^T Y (+ |Y_j|^2): two rows per thread with 16-byte loads,
// AT basis columns per CTA row of the grid; every load of a row pair is
// issued before its FMAs (the generic gram_kernel keeps ~4 in flight).
template <int AT, int NB>
__global__ void __launch_bounds__(kThreads)
gram4_vec_kernel(int64_t dim, ColSet xs, const double *__restrict__ y, int64_t ldy, double *c, int64_t ldc,
                 double *norms2, double *partials, unsigned int *ticket, int ny) {
  constexpr int nb = NB;  // valid columns of y (2 or 3: the rest re-read column NB-1, unused)
  pdl_wait();
  __shared__ const double *xp[AT];
  // ny > 0: one-dimensional grid with the ny column groups of a row range
  // on consecutive CTAs, so they stream the same y rows together (L2 hits)
  const int ty = ny ? blockIdx.x % ny : blockIdx.y;
  const int bx = ny ? blockIdx.x / ny : blockIdx.x;
  const int nx = ny ? gridDim.x / ny : gridDim.x;
  const int nty = ny ? ny : gridDim.y;
  const int i0 = ty * AT;
  const int na = min(AT, xs.total - i0);
  const bool want_norm = norms2 != nullptr && ty == 0;
  if (threadIdx.x < AT) xp[threadIdx.x] = colset_ptr(xs, i0 + min((int)threadIdx.x, na - 1));
  __syncthreads();
  constexpr int NOUT = AT * 4 + 4;
  double acc[NOUT];
#pragma unroll
  for (int k = 0; k < NOUT; ++k) acc[k] = 0.0;
  RowRange rr = cta_rows_even(dim, bx, nx);
  int64_t r = rr.r0 + 2 * threadIdx.x;
  for (; r + 1 < rr.r1; r += 2 * kThreads) {
    double2 yv[4], xv[AT];
#pragma unroll
    for (int j = 0; j < 4; ++j) yv[j] = ldg2(y + r + (int64_t)min(j, nb - 1) * ldy);  // nb < 4: re-read, unused
#pragma unroll
    for (int i = 0; i < AT; ++i) xv[i] = ldg2(xp[i] + r);  // columns past na re-read the last one
#pragma unroll
    for (int i = 0; i < AT; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fma(xv[i].x, yv[j].x, fma(xv[i].y, yv[j].y, acc[i * 4 + j]));
    if (want_norm) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[AT * 4 + j] = fma(yv[j].x, yv[j].x, fma(yv[j].y, yv[j].y, acc[AT * 4 + j]));
    }
  }
  if (r < rr.r1) {  // odd tail row
    double yv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) yv[j] = __ldg(y + r + (int64_t)min(j, nb - 1) * ldy);
#pragma unroll
    for (int i = 0; i < AT; ++i) {
      const double xv = __ldg(xp[i] + r);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i * 4 + j] = fma(xv, yv[j], acc[i * 4 + j]);
    }
    if (want_norm) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[AT * 4 + j] = fma(yv[j], yv[j], acc[AT * 4 + j]);
    }
  }
  pdl_trigger();
  double *part = partials + ((int64_t)ty * nx + bx) * NOUT;
  cta_fold<NOUT>(acc, NOUT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, nx, NOUT, nty * NOUT, [&](int, int t, int k, double sum) {
    if (k < AT * 4) {
      const int i = t * AT + k / 4, j = k % 4;
      if (k / 4 < min(AT, xs.total - t * AT) && j < nb) c[i + (int64_t)j * ldc] = sum;
    } else if (norms2 != nullptr && t == 0 && k - AT * 4 < nb) {
      norms2[k - AT * 4] = sum;
    }
  });
}

// b = NB <= 4 projection Y -= X C (+ |Y_j|^2 after): two rows per thread with
// 16-byte loads, basis columns in chunks of 8 whose loads precede their
// FMAs; per element the same fma order as project_kernel (bit-identical).
template <int NB>
__global__ void __launch_bounds__(kThreads)
project4_vec_kernel(int64_t dim, ColSet xs, const double *__restrict__ cmat, int64_t ldc, double *y, int64_t ldy,
                    double *norms2, double *partials, unsigned int *ticket) {
  pdl_wait();
  extern __shared__ double csh4[];  // na x NB
  __shared__ const double *xp[256];
  const int na = xs.total;
  for (int i = threadIdx.x; i < na; i += kThreads) xp[i] = colset_ptr(xs, i);
  for (int k = threadIdx.x; k < na * NB; k += kThreads) csh4[k] = cmat[k / NB + (int64_t)(k % NB) * ldc];
  __syncthreads();
  double nacc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) nacc[j] = 0.0;
  RowRange rr = cta_rows_even(dim);
  int64_t r = rr.r0 + 2 * threadIdx.x;
  for (; r + 1 < rr.r1; r += 2 * kThreads) {
    double2 yv[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) yv[j] = *reinterpret_cast<const double2 *>(y + r + (int64_t)j * ldy);
    for (int i0 = 0; i0 < na; i0 += 8) {
      double2 xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = ldg2(xp[min(i0 + u, na - 1)] + r);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (i0 + u < na) {
          const double *cr = csh4 + (i0 + u) * NB;
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            yv[j].x = fma(-xv[u].x, cr[j], yv[j].x);
            yv[j].y = fma(-xv[u].y, cr[j], yv[j].y);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      *reinterpret_cast<double2 *>(y + r + (int64_t)j * ldy) = yv[j];
      nacc[j] = fma(yv[j].x, yv[j].x, nacc[j]);
      nacc[j] = fma(yv[j].y, yv[j].y, nacc[j]);
    }
  }
  if (r < rr.r1) {
    double yv[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) yv[j] = y[r + (int64_t)j * ldy];
    for (int i = 0; i < na; ++i) {
      const double xv = __ldg(xp[i] + r);
#pragma unroll
      for (int j = 0; j < NB; ++j) yv[j] = fma(-xv, csh4[i * NB + j], yv[j]);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      y[r + (int64_t)j * ldy] = yv[j];
      nacc[j] = fma(yv[j], yv[j], nacc[j]);
    }
  }
  pdl_trigger();
  if (norms2 == nullptr) return;
  cta_fold<NB>(nacc, NB, partials + (int64_t)blockIdx.x * NB);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, NB, NB, [&](int j, int, int, double sum) { norms2[j] = sum; });
}

// One step of the iterated-CGS decision of kernels.py:115-127, on device.
// st: [active, pass, collapses, orig, prev, final, |v|^2 before, |v|^2 after]
__device__ __forceinline__ void dgks_decide(double *st) {
  const double before = sqrt(st[6]), cur = sqrt(st[7]);
  double p = st[1], coll = st[2], orig = st[3], prev = st[4], fin = 0.0;
  bool active = true;
  if (p == 0.0) {
    orig = before;
    prev = before;
    if (!(orig > 0.0)) active = false;
  }
  if (active) {
    if (cur < 1e-14 * orig) {
      coll += 1.0;
      if (coll >= 2.0) active = false;
    } else if (cur > 0.70710678118654752440 * prev) {
      fin = cur;
      active = false;
    } else {
      coll = 0.0;
    }
    prev = cur;
  }
  p += 1.0;
  if (active && p >= 6.0) active = false;
  st[0] = active ? 1.0 : 0.0;
  st[1] = p;
  st[2] = coll;
  st[3] = orig;
  st[4] = prev;
  st[5] = fin;
}

// Arm b DGKS records after the batched first projection of a block
// (svdsb_cgs_block): record j gets |v_j|^2 before (pass 1 started from the
// original column); column 0, whose pass 1 is complete, also gets its
// after-norm and the decision.
__global__ void dgks_seed_kernel(double *st, int b, const double *before2, const double *after2) {
  pdl_wait();
  pdl_trigger();
  const int j = threadIdx.x;
  if (j >= b) return;
  double *r = st + 8 * j;
  r[0] = 1.0;
  r[1] = r[2] = r[3] = r[4] = r[5] = 0.0;
  r[6] = before2[j];
  r[7] = after2[j];
  if (j == 0) dgks_decide(r);
}

__global__ void dgks_begin_kernel(double *st) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < 8) st[threadIdx.x] = (threadIdx.x == 0) ? 1.0 : 0.0;
}

__global__ void __launch_bounds__(kThreads)
project1_vec_kernel(int64_t dim, ColSet xs, const double *__restrict__ cvec, double *y, double *norms2,
                    double *partials, unsigned int *ticket, double *dgks) {
  pdl_wait();
  if (dgks != nullptr && dgks[0] == 0.0) return;
  extern __shared__ double csh[];
  __shared__ const double *xp[256];
  const int na = xs.total;
  for (int i = threadIdx.x; i < na; i += kThreads) {
    xp[i] = colset_ptr(xs, i);
    csh[i] = cvec[i];
  }
  __syncthreads();
  double nacc = 0.0;
  RowRange rr = cta_rows_even(dim);
  int64_t r = rr.r0 + 2 * threadIdx.x;
  for (; r + 1 < rr.r1; r += 2 * kThreads) {
    double2 yv = *reinterpret_cast<const double2 *>(y + r);
    int i = 0;
    for (; i + 4 <= na; i += 4) {
      double2 a0 = ldg2(xp[i] + r), a1 = ldg2(xp[i + 1] + r), a2 = ldg2(xp[i + 2] + r), a3 = ldg2(xp[i + 3] + r);
      yv.x = fma(-a0.x, csh[i], yv.x);
      yv.y = fma(-a0.y, csh[i], yv.y);
      yv.x = fma(-a1.x, csh[i + 1], yv.x);
      yv.y = fma(-a1.y, csh[i + 1], yv.y);
      yv.x = fma(-a2.x, csh[i + 2], yv.x);
      yv.y = fma(-a2.y, csh[i + 2], yv.y);
      yv.x = fma(-a3.x, csh[i + 3], yv.x);
      yv.y = fma(-a3.y, csh[i + 3], yv.y);
    }
    for (; i < na; ++i) {
      double2 a0 = ldg2(xp[i] + r);
      yv.x = fma(-a0.x, csh[i], yv.x);
      yv.y = fma(-a0.y, csh[i], yv.y);
    }
    *reinterpret_cast<double2 *>(y + r) = yv;
    nacc = fma(yv.x, yv.x, fma(yv.y, yv.y, nacc));
  }
  if (r < rr.r1) {
    double yv = y[r];
    for (int i = 0; i < na; ++i) yv = fma(-__ldg(xp[i] + r), csh[i], yv);
    y[r] = yv;
    nacc = fma(yv, yv, nacc);
  }
  pdl_trigger();
  if (norms2 == nullptr) return;
  double accs[1] = {nacc};
  cta_fold<1>(accs, 1, partials + blockIdx.x);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, 1, 1, [&](int, int, int, double s) {
    norms2[0] = s;
    if (dgks != nullptr) dgks_decide(dgks);
  });
}

// R = W Y - V Y diag(lam) for p <= PT candidates in one pass over V, W.
template <int PT>
__global__ void __launch_bounds__(kThreads, PT <= 16 ? 2 : 1)
ritz_wide_kernel(int64_t dim, const double *__restrict__ v, int64_t ldv, const double *__restrict__ w, int64_t ldw,
                 int g, const double *__restrict__ yc, int64_t ldyc, const double *__restrict__ lam, int p,
                 double *__restrict__ r, int64_t ldr, double *__restrict__ xo, int64_t ldx, double *__restrict__ oxo,
                 int64_t ldox, double *rn2, double *partials, unsigned int *ticket, StatusOut so) {
  pdl_wait();
  extern __shared__ double ysh[];  // g x PT
  __shared__ double lsh[PT];
  for (int k = threadIdx.x; k < g * PT; k += kThreads) {
    int i = k / PT, j = k % PT;
    ysh[k] = (j < p) ? yc[i + (int64_t)j * ldyc] : 0.0;
  }
  if (threadIdx.x < PT) lsh[threadIdx.x] = ((int)threadIdx.x < p) ? lam[threadIdx.x] : 0.0;
  __syncthreads();
  double nacc[PT];
#pragma unroll
  for (int j = 0; j < PT; ++j) nacc[j] = 0.0;
  RowRange rr = cta_rows(dim);
  for (int64_t row = rr.r0 + threadIdx.x; row < rr.r1; row += kThreads) {
    double ax[PT], aw[PT];
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      ax[j] = 0.0;
      aw[j] = 0.0;
    }
    // basis columns in groups of RU, every load of a group issued before
    // its FMAs (same FMA order as one column at a time)
    constexpr int RU = PT <= 8 ? 8 : (PT <= 12 ? 4 : (PT <= 16 ? 2 : 1));
    int i = 0;
    for (; i + RU <= g; i += RU) {
      double vv[RU], ww[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        vv[u] = __ldg(v + row + (int64_t)(i + u) * ldv);
        ww[u] = __ldg(w + row + (int64_t)(i + u) * ldw);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const double2 *yrow = reinterpret_cast<const double2 *>(ysh + (i + u) * PT);
#pragma unroll
        for (int j = 0; j < PT / 2; ++j) {
          double2 cf = yrow[j];
          ax[2 * j] = fma(vv[u], cf.x, ax[2 * j]);
          aw[2 * j] = fma(ww[u], cf.x, aw[2 * j]);
          ax[2 * j + 1] = fma(vv[u], cf.y, ax[2 * j + 1]);
          aw[2 * j + 1] = fma(ww[u], cf.y, aw[2 * j + 1]);
        }
      }
    }
    for (; i < g; ++i) {
      double vv = __ldg(v + row + (int64_t)i * ldv);
      double ww = __ldg(w + row + (int64_t)i * ldw);
      const double2 *yrow = reinterpret_cast<const double2 *>(ysh + i * PT);
#pragma unroll
      for (int j = 0; j < PT / 2; ++j) {
        double2 cf = yrow[j];
        ax[2 * j] = fma(vv, cf.x, ax[2 * j]);
        aw[2 * j] = fma(ww, cf.x, aw[2 * j]);
        ax[2 * j + 1] = fma(vv, cf.y, ax[2 * j + 1]);
        aw[2 * j + 1] = fma(ww, cf.y, aw[2 * j + 1]);
      }
    }
#pragma unroll
    for (int j = 0; j < PT; ++j) {
      if (j < p) {
        double res = __dsub_rn(aw[j], __dmul_rn(ax[j], lsh[j]));  // R = OpX - X*lam, two roundings (no fma), eigensolver.py:392
        r[row + (int64_t)j * ldr] = res;
        if (xo) xo[row + (int64_t)j * ldx] = ax[j];
        if (oxo) oxo[row + (int64_t)j * ldox] = aw[j];
        nacc[j] = fma(res, res, nacc[j]);
      }
    }
  }
  pdl_trigger();
  double *part = partials + (int64_t)blockIdx.x * PT;
  cta_fold<PT>(nacc, PT, part);
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, PT, p, [&](int j, int, int, double s) { rn2[j] = s; });
  if (so.host != nullptr) {
    __syncthreads();  // this CTA's rn2 writes are visible to all its threads
    for (int i = threadIdx.x; i < so.gn + p + 8; i += blockDim.x)
      so.host[i] = i < so.gn ? so.lams[i] : (i < so.gn + p ? rn2[i - so.gn] : so.st[i - so.gn - p]);
    __threadfence_system();
  }
}

// Ritz residuals on the fp64 tensor cores (DMMA m8n8k4): X = V Y and
// OpX = W Y are dense (N x g) x (g x p) contractions, so each warp takes 8
// rows at a time and runs ceil(g/4) x NT DMMAs per operand with Y's
// fragments held in registers for the whole kernel -- no shared-memory
// coefficient traffic, which bounds the FMA kernels (ritz_wide reads every
// coefficient from shared memory once per row).  The epilogue is the
// reference's R = OpX - X*lam with two roundings (eigensolver.py:392), the
// squared norms fold deterministically (lane shuffles, warps in order,
// last-CTA fold).  DMMA accumulates in its own order, so R matches the FMA
// kernels to rounding, not bit for bit.
constexpr int kDmmaMaxK = 10;   // g <= 40

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(kThreads)
ritz_dmma_kernel(int64_t dim, const double *__restrict__ v, int64_t ldv, const double *__restrict__ w, int64_t ldw,
                 int g, const double *__restrict__ yc, int64_t ldyc, const double *__restrict__ lam, int p,
                 double *__restrict__ r, int64_t ldr, double *__restrict__ xo, int64_t ldx, double *__restrict__ oxo,
                 int64_t ldox, double *rn2, double *partials, unsigned int *ticket, StatusOut so) {
  constexpr int PT = 8 * NT;
  pdl_wait();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gi = lane >> 2, ti = lane & 3;          // fragment row / k (or column pair)
  const int ks = (g + 3) >> 2;
  // B fragments: Y[k = 4s + ti][j = 8t + gi]
  double bf[kDmmaMaxK][NT];
#pragma unroll
  for (int s2 = 0; s2 < kDmmaMaxK; ++s2)
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int k = 4 * s2 + ti, j = 8 * t + gi;
      bf[s2][t] = (s2 < ks && k < g && j < p) ? yc[k + (int64_t)j * ldyc] : 0.0;
    }
  double lv[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 8 * t + 2 * ti + e;
      lv[t][e] = j < p ? lam[j] : 0.0;
    }
  double nacc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) nacc[t][0] = nacc[t][1] = 0.0;
  const int64_t ngroups = (dim + 7) >> 3;
  const int64_t gstride = (int64_t)gridDim.x * (kThreads / 32);
  for (int64_t grp = blockIdx.x * (int64_t)(kThreads / 32) + wid; grp < ngroups; grp += gstride) {
    const int64_t r0 = grp << 3;
    const int64_t ra = r0 + gi;                     // A-fragment row of this lane
    const bool rok = ra < dim;
    double av[kDmmaMaxK], aw[kDmmaMaxK];
#pragma unroll
    for (int s2 = 0; s2 < kDmmaMaxK; ++s2) {
      const int k = 4 * s2 + ti;
      const bool ok = rok && s2 < ks && k < g;
      av[s2] = ok ? __ldg(v + ra + (int64_t)k * ldv) : 0.0;
      aw[s2] = ok ? __ldg(w + ra + (int64_t)k * ldw) : 0.0;
    }
    double cx[NT][2], cw[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) cx[t][0] = cx[t][1] = cw[t][0] = cw[t][1] = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < kDmmaMaxK; ++s2) {
      if (s2 < ks) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          dmma884(cx[t], av[s2], bf[s2][t]);
          dmma884(cw[t], aw[s2], bf[s2][t]);
        }
      }
    }
    // C fragment: row r0 + gi, columns 8t + 2ti + e
    const int64_t row = r0 + gi;
    if (row < dim) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 8 * t + 2 * ti + e;
          if (j < p) {
            const double res = __dsub_rn(cw[t][e], __dmul_rn(cx[t][e], lv[t][e]));
            r[row + (int64_t)j * ldr] = res;
            if (xo) xo[row + (int64_t)j * ldx] = cx[t][e];
            if (oxo) oxo[row + (int64_t)j * ldox] = cw[t][e];
            nacc[t][e] = fma(res, res, nacc[t][e]);
          }
        }
    }
  }
  pdl_trigger();
  // lanes with equal ti hold the same columns: xor over the row bits
  __shared__ double red[kThreads / 32][PT];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double x = nacc[t][e];
      x += __shfl_xor_sync(0xffffffffu, x, 4);
      x += __shfl_xor_sync(0xffffffffu, x, 8);
      x += __shfl_xor_sync(0xffffffffu, x, 16);
      if (gi == 0) red[wid][8 * t + 2 * ti + e] = x;
    }
  __syncthreads();
  double *pp = partials + (int64_t)blockIdx.x * PT;
  for (int k = threadIdx.x; k < PT; k += kThreads) {
    double x = 0.0;
#pragma unroll
    for (int ww = 0; ww < kThreads / 32; ++ww) x += red[ww][k];
    pp[k] = x;
  }
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, PT, p, [&](int j, int, int, double x) { rn2[j] = x; });
  if (so.host != nullptr) {
    __syncthreads();
    for (int i = threadIdx.x; i < so.gn + p + 8; i += blockDim.x)
      so.host[i] = i < so.gn ? so.lams[i] : (i < so.gn + p ? rn2[i - so.gn] : so.st[i - so.gn - p]);
    __threadfence_system();
  }
}

// Ritz residuals with SPLIT threads per row, each owning PQ consecutive
// candidates: the same per-element fma order as ritz_wide_kernel (basis
// index ascending), so R is bit-identical; fewer accumulators per thread
// keep two CTAs per SM and RU loads in flight where ritz_wide_kernel<24/32>
// ran one CTA with one load pair at a time.  The threads of a row read the
// same V / W element (one sector per warp load, broadcast).
template <int PQ, int SPLIT>
__global__ void __launch_bounds__(kThreads, 2)
ritz_split_kernel(int64_t dim, const double *__restrict__ v, int64_t ldv, const double *__restrict__ w, int64_t ldw,
                  int g, const double *__restrict__ yc, int64_t ldyc, const double *__restrict__ lam, int p,
                  double *__restrict__ r, int64_t ldr, double *__restrict__ xo, int64_t ldx, double *__restrict__ oxo,
                  int64_t ldox, double *rn2, double *partials, unsigned int *ticket, StatusOut so) {
  constexpr int PT = PQ * SPLIT;
  pdl_wait();
  extern __shared__ double ysh[];  // g x PT
  __shared__ double lsh[PT];
  __shared__ double red[kWarps][PT];
  for (int k = threadIdx.x; k < g * PT; k += kThreads) {
    int i = k / PT, j = k % PT;
    ysh[k] = (j < p) ? yc[i + (int64_t)j * ldyc] : 0.0;
  }
  if (threadIdx.x < PT) lsh[threadIdx.x] = ((int)threadIdx.x < p) ? lam[threadIdx.x] : 0.0;
  __syncthreads();
  const int part = threadIdx.x % SPLIT;
  const int j0 = part * PQ;
  double nacc[PQ];
#pragma unroll
  for (int j = 0; j < PQ; ++j) nacc[j] = 0.0;
  RowRange rr = cta_rows(dim);
  constexpr int RPP = kThreads / SPLIT;  // rows per pass of the CTA
  for (int64_t row = rr.r0 + threadIdx.x / SPLIT; row < rr.r1; row += RPP) {
    double ax[PQ], aw[PQ];
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      ax[j] = 0.0;
      aw[j] = 0.0;
    }
    constexpr int RU = PQ <= 6 ? 8 : (PQ <= 12 ? 4 : 2);
    int i = 0;
    for (; i + RU <= g; i += RU) {
      double vv[RU], ww[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        vv[u] = __ldg(v + row + (int64_t)(i + u) * ldv);
        ww[u] = __ldg(w + row + (int64_t)(i + u) * ldw);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const double2 *yrow = reinterpret_cast<const double2 *>(ysh + (i + u) * PT + j0);
#pragma unroll
        for (int j = 0; j < PQ / 2; ++j) {
          double2 cf = yrow[j];
          ax[2 * j] = fma(vv[u], cf.x, ax[2 * j]);
          aw[2 * j] = fma(ww[u], cf.x, aw[2 * j]);
          ax[2 * j + 1] = fma(vv[u], cf.y, ax[2 * j + 1]);
          aw[2 * j + 1] = fma(ww[u], cf.y, aw[2 * j + 1]);
        }
      }
    }
    for (; i < g; ++i) {
      double vv = __ldg(v + row + (int64_t)i * ldv);
      double ww = __ldg(w + row + (int64_t)i * ldw);
      const double2 *yrow = reinterpret_cast<const double2 *>(ysh + i * PT + j0);
#pragma unroll
      for (int j = 0; j < PQ / 2; ++j) {
        double2 cf = yrow[j];
        ax[2 * j] = fma(vv, cf.x, ax[2 * j]);
        aw[2 * j] = fma(ww, cf.x, aw[2 * j]);
        ax[2 * j + 1] = fma(vv, cf.y, ax[2 * j + 1]);
        aw[2 * j + 1] = fma(ww, cf.y, aw[2 * j + 1]);
      }
    }
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      if (j0 + j < p) {
        double res = __dsub_rn(aw[j], __dmul_rn(ax[j], lsh[j0 + j]));  // as ritz_wide_kernel
        r[row + (int64_t)(j0 + j) * ldr] = res;
        if (xo) xo[row + (int64_t)(j0 + j) * ldx] = ax[j];
        if (oxo) oxo[row + (int64_t)(j0 + j) * ldox] = aw[j];
        nacc[j] = fma(res, res, nacc[j]);
      }
    }
  }
  pdl_trigger();
  // per-candidate CTA sums: lanes of equal `part` reduced with xor shuffles
  // (lane % SPLIT is preserved by xor offsets >= SPLIT), then across warps
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < PQ; ++j) {
    double t = nacc[j];
#pragma unroll
    for (int off = 16; off >= SPLIT; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane < SPLIT) red[wid][lane * PQ + j] = t;
  }
  __syncthreads();
  double *pp = partials + (int64_t)blockIdx.x * PT;
  for (int k = threadIdx.x; k < PT; k += kThreads) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) t += red[ww][k];
    pp[k] = t;
  }
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, PT, p, [&](int j, int, int, double t) { rn2[j] = t; });
  if (so.host != nullptr) {
    __syncthreads();
    for (int i = threadIdx.x; i < so.gn + p + 8; i += blockDim.x)
      so.host[i] = i < so.gn ? so.lams[i] : (i < so.gn + p ? rn2[i - so.gn] : so.st[i - so.gn - p]);
    __threadfence_system();
  }
}

template <int PQ>
__global__ void __launch_bounds__(kThreads, 2)
ritz_split_r2_kernel(int64_t dim, const double *__restrict__ v, int64_t ldv, const double *__restrict__ w, int64_t ldw,
                  int g, const double *__restrict__ yc, int64_t ldyc, const double *__restrict__ lam, int p,
                  double *__restrict__ r, int64_t ldr, double *__restrict__ xo, int64_t ldx, double *__restrict__ oxo,
                  int64_t ldox, double *rn2, double *partials, unsigned int *ticket, StatusOut so) {
  constexpr int SPLIT = 2;
  constexpr int PT = PQ * SPLIT;
  pdl_wait();
  extern __shared__ double ysh[];  // g x PT
  __shared__ double lsh[PT];
  __shared__ double red[kWarps][PT];
  for (int k = threadIdx.x; k < g * PT; k += kThreads) {
    int i = k / PT, j = k % PT;
    ysh[k] = (j < p) ? yc[i + (int64_t)j * ldyc] : 0.0;
  }
  if (threadIdx.x < PT) lsh[threadIdx.x] = ((int)threadIdx.x < p) ? lam[threadIdx.x] : 0.0;
  __syncthreads();
  const int part = threadIdx.x % SPLIT;
  const int j0 = part * PQ;
  // per-thread candidate norms in shared memory ([j][thread]: conflict
  // free), so the 48 accumulators of the two rows fit the register budget
  __shared__ double nsh[PQ][kThreads];
#pragma unroll
  for (int j = 0; j < PQ; ++j) nsh[j][threadIdx.x] = 0.0;
  // two adjacent rows per thread pair member: every shared-memory
  // coefficient feeds four FMAs instead of two (the one-row kernel is bound
  // by shared-memory bandwidth at ~half the fp64 FMA rate); 16-byte loads
  // and stores; per element the same fma chain, so R is bit-identical
  RowRange rr = cta_rows_even(dim);
  constexpr int RPP = kThreads;  // rows per pass of the CTA (kThreads/2 pairs x 2 rows)
  for (int64_t row = rr.r0 + 2 * (threadIdx.x / SPLIT); row < rr.r1; row += RPP) {
    const bool two = row + 1 < rr.r1;
    double2 ax[PQ], aw[PQ];
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      ax[j] = make_double2(0.0, 0.0);
      aw[j] = make_double2(0.0, 0.0);
    }
    constexpr int RU = 1;
    int i = 0;
    for (; i + RU <= g; i += RU) {
      double2 vv[RU], ww[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (two) {
          vv[u] = ldg2(v + row + (int64_t)(i + u) * ldv);
          ww[u] = ldg2(w + row + (int64_t)(i + u) * ldw);
        } else {
          vv[u] = make_double2(__ldg(v + row + (int64_t)(i + u) * ldv), 0.0);
          ww[u] = make_double2(__ldg(w + row + (int64_t)(i + u) * ldw), 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const double2 *yrow = reinterpret_cast<const double2 *>(ysh + (i + u) * PT + j0);
#pragma unroll
        for (int j = 0; j < PQ / 2; ++j) {
          const double2 cf = yrow[j];
          ax[2 * j].x = fma(vv[u].x, cf.x, ax[2 * j].x);
          ax[2 * j].y = fma(vv[u].y, cf.x, ax[2 * j].y);
          aw[2 * j].x = fma(ww[u].x, cf.x, aw[2 * j].x);
          aw[2 * j].y = fma(ww[u].y, cf.x, aw[2 * j].y);
          ax[2 * j + 1].x = fma(vv[u].x, cf.y, ax[2 * j + 1].x);
          ax[2 * j + 1].y = fma(vv[u].y, cf.y, ax[2 * j + 1].y);
          aw[2 * j + 1].x = fma(ww[u].x, cf.y, aw[2 * j + 1].x);
          aw[2 * j + 1].y = fma(ww[u].y, cf.y, aw[2 * j + 1].y);
        }
      }
    }
    for (; i < g; ++i) {
      double2 vv, ww;
      if (two) {
        vv = ldg2(v + row + (int64_t)i * ldv);
        ww = ldg2(w + row + (int64_t)i * ldw);
      } else {
        vv = make_double2(__ldg(v + row + (int64_t)i * ldv), 0.0);
        ww = make_double2(__ldg(w + row + (int64_t)i * ldw), 0.0);
      }
      const double2 *yrow = reinterpret_cast<const double2 *>(ysh + i * PT + j0);
#pragma unroll
      for (int j = 0; j < PQ / 2; ++j) {
        const double2 cf = yrow[j];
        ax[2 * j].x = fma(vv.x, cf.x, ax[2 * j].x);
        ax[2 * j].y = fma(vv.y, cf.x, ax[2 * j].y);
        aw[2 * j].x = fma(ww.x, cf.x, aw[2 * j].x);
        aw[2 * j].y = fma(ww.y, cf.x, aw[2 * j].y);
        ax[2 * j + 1].x = fma(vv.x, cf.y, ax[2 * j + 1].x);
        ax[2 * j + 1].y = fma(vv.y, cf.y, ax[2 * j + 1].y);
        aw[2 * j + 1].x = fma(ww.x, cf.y, aw[2 * j + 1].x);
        aw[2 * j + 1].y = fma(ww.y, cf.y, aw[2 * j + 1].y);
      }
    }
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      if (j0 + j < p) {
        const double l = lsh[j0 + j];
        const double2 res = make_double2(__dsub_rn(aw[j].x, __dmul_rn(ax[j].x, l)),
                                         __dsub_rn(aw[j].y, __dmul_rn(ax[j].y, l)));
        if (two) {
          *reinterpret_cast<double2 *>(r + row + (int64_t)(j0 + j) * ldr) = res;
          if (xo) *reinterpret_cast<double2 *>(xo + row + (int64_t)(j0 + j) * ldx) = ax[j];
          if (oxo) *reinterpret_cast<double2 *>(oxo + row + (int64_t)(j0 + j) * ldox) = aw[j];
          nsh[j][threadIdx.x] = fma(res.y, res.y, fma(res.x, res.x, nsh[j][threadIdx.x]));
        } else {
          r[row + (int64_t)(j0 + j) * ldr] = res.x;
          if (xo) xo[row + (int64_t)(j0 + j) * ldx] = ax[j].x;
          if (oxo) oxo[row + (int64_t)(j0 + j) * ldox] = aw[j].x;
          nsh[j][threadIdx.x] = fma(res.x, res.x, nsh[j][threadIdx.x]);
        }
      }
    }
  }
  pdl_trigger();
  // per-candidate CTA sums: lanes of equal `part` reduced with xor shuffles
  // (lane % SPLIT is preserved by xor offsets >= SPLIT), then across warps
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < PQ; ++j) {
    double t = nsh[j][threadIdx.x];
#pragma unroll
    for (int off = 16; off >= SPLIT; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane < SPLIT) red[wid][lane * PQ + j] = t;
  }
  __syncthreads();
  double *pp = partials + (int64_t)blockIdx.x * PT;
  for (int k = threadIdx.x; k < PT; k += kThreads) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) t += red[ww][k];
    pp[k] = t;
  }
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, PT, p, [&](int j, int, int, double t) { rn2[j] = t; });
  if (so.host != nullptr) {
    __syncthreads();
    for (int i = threadIdx.x; i < so.gn + p + 8; i += blockDim.x)
      so.host[i] = i < so.gn ? so.lams[i] : (i < so.gn + p ? rn2[i - so.gn] : so.st[i - so.gn - p]);
    __threadfence_system();
  }
}

// Y = alpha X C + beta Y, two rows per thread, s <= ST.
template <int ST>
__global__ void __launch_bounds__(kThreads)
ts_gemm_vec_kernel(int64_t dim, const double *__restrict__ x, int64_t ldx, int g, const double *__restrict__ cmat,
                   int64_t ldc, int s, double alpha, double beta, double *__restrict__ y, int64_t ldy) {
  extern __shared__ double csh[];  // g x ST
  for (int k = threadIdx.x; k < g * ST; k += kThreads) {
    int i = k / ST, j = k % ST;
    csh[k] = (j < s) ? cmat[i + (int64_t)j * ldc] : 0.0;
  }
  __syncthreads();
  RowRange rr = cta_rows_even(dim);
  int64_t r = rr.r0 + 2 * threadIdx.x;
  for (; r < rr.r1; r += 2 * kThreads) {
    const bool pair = r + 1 < rr.r1;
    double a0[ST], a1[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      a0[j] = 0.0;
      a1[j] = 0.0;
    }
    for (int i = 0; i < g; ++i) {
      double2 xv;
      if (pair) {
        xv = ldg2(x + r + (int64_t)i * ldx);
      } else {
        xv.x = __ldg(x + r + (int64_t)i * ldx);
        xv.y = 0.0;
      }
      const double2 *crow = reinterpret_cast<const double2 *>(csh + i * ST);
#pragma unroll
      for (int j = 0; j < ST / 2; ++j) {
        double2 cf = crow[j];
        a0[2 * j] = fma(xv.x, cf.x, a0[2 * j]);
        a1[2 * j] = fma(xv.y, cf.x, a1[2 * j]);
        a0[2 * j + 1] = fma(xv.x, cf.y, a0[2 * j + 1]);
        a1[2 * j + 1] = fma(xv.y, cf.y, a1[2 * j + 1]);
      }
    }
#pragma unroll
    for (int j = 0; j < ST; ++j) {
      if (j < s) {
        double *yp = y + r + (int64_t)j * ldy;
        if (pair) {
          double2 out = make_double2(alpha * a0[j], alpha * a1[j]);
          if (beta != 0.0) {
            double2 old = *reinterpret_cast<double2 *>(yp);
            out.x = fma(beta, old.x, out.x);
            out.y = fma(beta, old.y, out.y);
          }
          *reinterpret_cast<double2 *>(yp) = out;
        } else {
          double out = alpha * a0[j];
          if (beta != 0.0) out = fma(beta, *yp, out);
          *yp = out;
        }
      }
    }
  }
}

// In-place Y[:, :s] = X[:, :g] C (Y aliases X, s <= g): every output row
// depends only on the same input row, so one thread reads its whole row
// before it writes any of it and no other thread touches that row.  No
// __restrict__ / read-only cache on the aliased block.
template <int ST>
__global__ void __launch_bounds__(kThreads)
ts_gemm_inplace_kernel(int64_t dim, double *x, int64_t ldx, int g, const double *__restrict__ cmat, int64_t ldc,
                       int s) {
  extern __shared__ double csh[];  // g x ST
  for (int k = threadIdx.x; k < g * ST; k += kThreads) {
    int i = k / ST, j = k % ST;
    csh[k] = (j < s) ? cmat[i + (int64_t)j * ldc] : 0.0;
  }
  __syncthreads();
  RowRange rr = cta_rows(dim);
  for (int64_t r = rr.r0 + threadIdx.x; r < rr.r1; r += kThreads) {
    double acc[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) acc[j] = 0.0;
    for (int i = 0; i < g; ++i) {
      double xv = x[r + (int64_t)i * ldx];
      const double2 *crow = reinterpret_cast<const double2 *>(csh + i * ST);
#pragma unroll
      for (int j = 0; j < ST / 2; ++j) {
        double2 cf = crow[j];
        acc[2 * j] = fma(xv, cf.x, acc[2 * j]);
        acc[2 * j + 1] = fma(xv, cf.y, acc[2 * j + 1]);
      }
    }
#pragma unroll
    for (int j = 0; j < ST; ++j)
      if (j < s) x[r + (int64_t)j * ldx] = acc[j];
  }
}


// In-place V <- V C for 16-byte aligned bases with even leading dimension:
// two rows per thread with 16-byte loads, basis columns in groups of eight
// whose loads precede their FMAs, and only ST >= s accumulators (the
// generic kernel above always carries 32).  Per element the same fma chain
// over i = 0..g-1 as ts_gemm_inplace_kernel, so the bits are identical.
template <int ST>
__global__ void __launch_bounds__(kThreads)
ts_gemm_inplace_vec_kernel(int64_t dim, double *x, int64_t ldx, int g, const double *__restrict__ cmat,
                           int64_t ldc, int s) {
  extern __shared__ double csh[];  // g x ST
  for (int k = threadIdx.x; k < g * ST; k += kThreads) {
    int i = k / ST, j = k % ST;
    csh[k] = (j < s) ? cmat[i + (int64_t)j * ldc] : 0.0;
  }
  __syncthreads();
  constexpr int GU = ST <= 16 ? 8 : 4;   // basis columns loaded per group
  RowRange rr = cta_rows_even(dim);
  int64_t r = rr.r0 + 2 * threadIdx.x;
  for (; r + 1 < rr.r1; r += 2 * kThreads) {
    double2 acc[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) acc[j] = make_double2(0.0, 0.0);
    for (int i0 = 0; i0 < g; i0 += GU) {
      double2 xv[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u)   // coherent loads: x is rewritten in place by this kernel
        xv[u] = *reinterpret_cast<const double2 *>(x + r + (int64_t)min(i0 + u, g - 1) * ldx);
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        if (i0 + u < g) {
          const double2 *crow = reinterpret_cast<const double2 *>(csh + (i0 + u) * ST);
#pragma unroll
          for (int j = 0; j < ST / 2; ++j) {
            const double2 cf = crow[j];
            acc[2 * j].x = fma(xv[u].x, cf.x, acc[2 * j].x);
            acc[2 * j].y = fma(xv[u].y, cf.x, acc[2 * j].y);
            acc[2 * j + 1].x = fma(xv[u].x, cf.y, acc[2 * j + 1].x);
            acc[2 * j + 1].y = fma(xv[u].y, cf.y, acc[2 * j + 1].y);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < ST; ++j)
      if (j < s) *reinterpret_cast<double2 *>(x + r + (int64_t)j * ldx) = acc[j];
  }
  if (r < rr.r1) {  // odd tail row
    double acc[ST];
#pragma unroll
    for (int j = 0; j < ST; ++j) acc[j] = 0.0;
    for (int i = 0; i < g; ++i) {
      const double xv = x[r + (int64_t)i * ldx];
#pragma unroll
      for (int j = 0; j < ST; ++j) acc[j] = fma(xv, csh[i * ST + j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < ST; ++j)
      if (j < s) x[r + (int64_t)j * ldx] = acc[j];
  }
}

#include "dense_stream.cuh"

// ------------------------------------------------ fused single-column CGS
// The whole orthonormalisation of one expansion vector in ONE launch, for a
// basis of <= 40 columns: select the residual column by the device index and
// precondition it (x ./ d), the +k coefficient copy (CTA 0), then up to
// `passes` iterated-CGS passes -- Gram, projection and the DGKS decision of
// kernels.py:115-127 -- and the final normalisation.  A pass needs two
// grid-wide reductions; between them the CTAs meet at a software grid
// barrier and EVERY CTA folds the per-CTA partials itself in the same fixed
// order, so all CTAs hold identical c, norms and DGKS state with no second
// barrier and no serial fold.  One 512-thread CTA per SM, grid <= #SMs, so
// every CTA is resident (the barrier's requirement); the kernel never
// triggers its dependants early.  Each thread owns the same row pairs in
// every phase, so x is read back only by the thread that wrote it.
constexpr int kCgsThreads = 512;
constexpr int kCgsMaxCols = 40;

template <int NACC>
__device__ __forceinline__ void cta_fold_wide(double (&acc)[NACC], double *part) {
  __shared__ double red[kCgsThreads / 32][NACC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NACC; ++k) {
    double v = warp_sum(acc[k]);
    if (lane == 0) red[w][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < NACC; k += blockDim.x) {
    double s = 0.0;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) s += red[ww][k];
    part[k] = s;
  }
}

__global__ void __launch_bounds__(kCgsThreads, 1)
cgs_fused_kernel(int64_t dim, ColSet xs, const double *rsrc, int64_t ldr, const int *ci,
                 const double *__restrict__ d, double *x, const double *yin, int64_t ldyin, int g, int kk,
                 double *prev, int64_t ldprev, int passes, double *st_out, double *partials,
                 unsigned int *bar) {
  constexpr int AT = kCgsMaxCols;
  constexpr int NACC = AT + 1;
  pdl_wait();
  __shared__ const double *xp[AT];
  __shared__ double csh[NACC];
  __shared__ double st[8];
  const int tid = threadIdx.x;
  const int na = xs.total;
  if (tid < na) xp[tid] = colset_ptr(xs, tid);
  if (tid < 8) st[tid] = (tid == 0) ? 1.0 : 0.0;
  const int cidx = *ci;
  if (blockIdx.x == 0 && prev != nullptr) {
    for (int e = tid; e < g * kk; e += blockDim.x) {
      const int r = e % g, j = e / g;
      if (cidx + j < g) prev[r + (int64_t)j * ldprev] = yin[r + (int64_t)(cidx + j) * ldyin];
    }
  }
  __syncthreads();
  RowRange rr = cta_rows_even(dim);
  const int64_t step = 2 * (int64_t)blockDim.x;
  const int64_t rbeg = rr.r0 + 2 * tid;
  {
    const double *src = rsrc + (int64_t)cidx * ldr;
    for (int64_t r = rbeg; r < rr.r1; r += step) {
      const int64_t r2 = min(r + 2, rr.r1);
      for (int64_t q = r; q < r2; ++q) {
        const double v = src[q];
        x[q] = d ? __ddiv_rn(v, d[q]) : v;
      }
    }
  }
  double *part_c = partials;
  double *part_n = partials + (int64_t)gridDim.x * NACC;
  for (int pass = 0; pass < passes; ++pass) {
    // Gram c = X^T x (+ |x|^2 on the first pass)
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    for (int64_t r = rbeg; r < rr.r1; r += step) {
      if (r + 1 < rr.r1) {
        const double2 xv = *reinterpret_cast<const double2 *>(x + r);
#pragma unroll
        for (int i = 0; i < AT; ++i)
          if (i < na) {
            const double2 vv = ldg2(xp[i] + r);
            acc[i] = fma(vv.x, xv.x, fma(vv.y, xv.y, acc[i]));
          }
        if (pass == 0) acc[AT] = fma(xv.x, xv.x, fma(xv.y, xv.y, acc[AT]));
      } else {
        const double xv = x[r];
#pragma unroll
        for (int i = 0; i < AT; ++i)
          if (i < na) acc[i] = fma(__ldg(xp[i] + r), xv, acc[i]);
        if (pass == 0) acc[AT] = fma(xv, xv, acc[AT]);
      }
    }
    cta_fold_wide<NACC>(acc, part_c + (int64_t)blockIdx.x * NACC);
    grid_barrier(bar, gridDim.x);
    fold_parts(part_c, gridDim.x, NACC, NACC, [&](int o, int, int, double sum) { csh[o] = sum; });
    __syncthreads();
    if (pass == 0 && tid == 0) st[6] = csh[AT];
    // projection x -= X c, |x|^2
    double nacc = 0.0;
    for (int64_t r = rbeg; r < rr.r1; r += step) {
      if (r + 1 < rr.r1) {
        double2 xv = *reinterpret_cast<const double2 *>(x + r);
#pragma unroll
        for (int i = 0; i < AT; ++i)
          if (i < na) {
            const double2 vv = ldg2(xp[i] + r);
            xv.x = fma(-vv.x, csh[i], xv.x);
            xv.y = fma(-vv.y, csh[i], xv.y);
          }
        *reinterpret_cast<double2 *>(x + r) = xv;
        nacc = fma(xv.x, xv.x, fma(xv.y, xv.y, nacc));
      } else {
        double xv = x[r];
#pragma unroll
        for (int i = 0; i < AT; ++i)
          if (i < na) xv = fma(-__ldg(xp[i] + r), csh[i], xv);
        x[r] = xv;
        nacc = fma(xv, xv, nacc);
      }
    }
    {
      double a1[1] = {nacc};
      cta_fold_wide<1>(a1, part_n + blockIdx.x);
    }
    grid_barrier(bar, gridDim.x);
    fold_parts(part_n, gridDim.x, 1, 1, [&](int, int, int, double sum) {
      st[7] = sum;
      dgks_decide(st);
    });
    __syncthreads();
    if (st[0] == 0.0) break;
  }
  // normalise by the accepted norm (the host path handles collapses)
  const double fin = st[5];
  if (st[0] == 0.0 && fin > 0.0) {
    for (int64_t r = rbeg; r < rr.r1; r += step) {
      const int64_t r2 = min(r + 2, rr.r1);
      for (int64_t q = r; q < r2; ++q) x[q] = x[q] / fin;
    }
  }
  if (blockIdx.x == 0 && tid < 8) st_out[tid] = st[tid];
}

static inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static bool colset_vec_ok(const ColSet &s) {
  for (int k = 0; k < s.nblk; ++k)
    if (s.cols[k] > 0 && (!aligned16(s.base[k]) || (s.ld[k] & 1))) return false;
  return true;
}

// Streamed (shared-memory ring) kernels of dense_stream.cuh: the default for
// bases beyond L2 scale; tune key 15 = 1 keeps the register-tiled kernels,
// 2 takes the streamed ones at every size.
static bool stream_ok(int64_t dim) {
  if (g_tune[15] == 1) return false;
  if (g_tune[15] >= 2) return dim >= 1;
  return dim >= (int64_t)1 << 18;
}

// One-column Gram / projection / CGS pass on the streamed kernels: opt-in
// (key 15 = 2 or 6).  Alone they are faster at g = 35 (N = 1 M: 78 -> 68 us
// and 71 -> 59 us; 87 % / 94 % of HBM at 4.1 M) but inside the solves they
// lose: most CGS passes of a block iteration are gated off on the device,
// and a gated streamed launch (288 threads, 180 KB of shared memory) costs
// more than a gated register launch -- config 4: 0.376 -> 0.387 s; config 3
// at g = 25: H-column Gram 153 -> 161 us.
static bool stream_one_col(int64_t dim) { return (g_tune[15] == 2 || g_tune[15] == 6) && stream_ok(dim); }

static int stream_grid_tiles(int64_t dim, int rows) {
  const int64_t nt = (dim + rows - 1) / rows;
  return (int)std::min<int64_t>(num_sms(), std::max<int64_t>(nt, 1));
}

// L2 evict-first for operands that cannot stay resident anyway
static int stream_evict_first(int64_t dim, int cols) { return (double)dim * cols * 8.0 > 48e6 ? 1 : 0; }

template <typename K>
static cudaError_t stream_attr(K kernel, size_t smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Tensor map of a column-major fp64 block (rows innermost) for the streamed
// kernels' tile loads; cuTensorMapEncodeTiled through the runtime's driver
// entry point (no link against libcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

static bool make_map2d(CUtensorMap *m, const double *base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                       int box_cols) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (fn == nullptr || rows < 1 || cols < 1 || !aligned16(base) || (ld & 1) || rows >= ((int64_t)1 << 31)) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t gstr[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), gdim, gstr, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kTsMaxG = 64;  // basis columns the streamed Ritz / restart kernels take (coefficients in shared memory)

static size_t ts_stream_smem(int nin, int g, int pt, int rows = kTsRows) {
  return sizeof(double) * ((size_t)kTsStages * nin * ts_kc(nin) * rows + (size_t)g * pt);
}

static int make_colset(ColSet &s, int nblk, const double *const *xs, const int64_t *ldxs, const int *cols) {
  SVDSB_CHECK_ARG(nblk >= 1 && nblk <= SVDSB_MAX_BLOCKS, "between 1 and SVDSB_MAX_BLOCKS column blocks");
  s.nblk = 0;
  s.total = 0;
  for (int k = 0; k < nblk; ++k) {
    if (cols[k] <= 0) continue;
    s.base[s.nblk] = xs[k];
    s.ld[s.nblk] = ldxs[k];
    s.cols[s.nblk] = cols[k];
    s.total += cols[k];
    s.nblk++;
  }
  if (s.nblk == 0) {
    s.base[0] = nullptr;
    s.ld[0] = 1;
    s.cols[0] = 0;
    s.nblk = 1;
  }
  return SVDSB_OK;
}

}  // namespace svdsb

using namespace svdsb;

extern "C" {

int svdsb_gram(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs, const int *cols,
               const double *y, int64_t ldy, int b, double *c, int64_t ldc, double *norms2, void *stream) {
  return svdsb::gram_impl(ctx, dim, nblk, xs, ldxs, cols, y, ldy, b, c, ldc, norms2, stream, svdsb::HInsert{});
}

}  // extern "C"

namespace svdsb {

// b >= 2 Gram through gram_stream_kernel (one persistent CTA per SM, tiles
// by TMA); false when a tensor map cannot be built (the caller falls back).
static bool gram_stream(svdsb_ctx *ctx, int64_t dim, const ColSet &s, const double *y, int64_t ldy, int b, double *c,
                        int64_t ldc, double *norms2, cudaStream_t st, const double *gate = nullptr,
                        HInsert hi = HInsert{}) {
  if (b == 1) ldy = (dim + 1) & ~(int64_t)1;  // one column: the stride is never used, the map wants it even
  GramMaps maps;
  int cap = 4;
  for (int k = 0; k < s.nblk; ++k) {
    if (!make_map2d(&maps.x[k], s.base[k], dim, s.cols[k], s.ld[k], kGsRows, kGsBox)) return false;
    cap += (s.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
  }
  for (int k = s.nblk; k < SVDSB_MAX_BLOCKS; ++k) maps.x[k] = maps.x[0];
  if (cap > kGsCap) return false;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gram_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * kGsStages * kGsCap * kGsRows)) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    attr = true;
  }
  const int gxs = stream_grid_tiles(dim, kGsRows);
  const size_t sh = sizeof(double) * (size_t)kGsStages * cap * kGsRows;
  for (int j0 = 0; j0 < b; j0 += 4) {
    const int nb = std::min(4, b - j0);
    if (!make_map2d(&maps.y, y + (int64_t)j0 * ldy, dim, nb, ldy, kGsRows, 4)) return false;
    if (launch_k(gram_stream_kernel, dim3(gxs, 1, 1), dim3(kStreamThreads, 1, 1), sh, st, maps, dim, s, nb,
                 c + (int64_t)j0 * ldc, ldc, norms2 ? norms2 + j0 : (double *)nullptr, ctx->partials, take_ticket(ctx),
                 stream_evict_first(dim, s.total), gate, hi) != cudaSuccess) {
      cudaGetLastError();
      return false;  // nothing written yet for this chunk: the register-tiled kernels redo the whole Gram
    }
    bump_launches();
  }
  return true;
}

constexpr int kPsCap = 52;  // stage capacity in columns of project_stream_kernel (2 stages of 256 rows)

// b <= 4 projection through project_stream_kernel; false when it does not
// apply (the caller falls back to the register kernels; nothing was written).
static bool project_stream(svdsb_ctx *ctx, int64_t dim, const ColSet &s, const double *c, int64_t ldc, double *y,
                           int64_t ldy, int nb, double *norms2, cudaStream_t st, double *dgks = nullptr) {
  if (nb < 1 || nb > 4 || s.total < 1 || s.total > kGsMaxX || !aligned16(y) || (nb > 1 && (ldy & 1))) return false;
  ProjMaps maps;
  int cap = 4;
  for (int k = 0; k < s.nblk; ++k) {
    if (!make_map2d(&maps.x[k], s.base[k], dim, s.cols[k], s.ld[k], kPsRows, kGsBox)) return false;
    cap += (s.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
  }
  for (int k = s.nblk; k < SVDSB_MAX_BLOCKS; ++k) maps.x[k] = maps.x[0];
  if (cap > kPsCap) return false;
  if (!make_map2d(&maps.y, y, dim, nb, nb == 1 ? ((dim + 1) & ~(int64_t)1) : ldy, kPsRows, 4)) return false;
  static bool attr = false;
  if (!attr) {
    const int mx = (int)(sizeof(double) * kPsStages * kPsCap * kPsRows);
    if (cudaFuncSetAttribute(project_stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess ||
        cudaFuncSetAttribute(project_stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess ||
        cudaFuncSetAttribute(project_stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess ||
        cudaFuncSetAttribute(project_stream_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    attr = true;
  }
  const size_t sh = sizeof(double) * (size_t)kPsStages * cap * kPsRows;
  const dim3 grid(stream_grid_tiles(dim, kPsRows), 1, 1), block(kStreamThreads, 1, 1);
  const int ef = stream_evict_first(dim, s.total);
  auto *tk = take_ticket(ctx);
  cudaError_t e;
  if (nb == 1)
    e = launch_k(project_stream_kernel<1>, grid, block, sh, st, maps, dim, s, c, ldc, y, ldy, norms2, ctx->partials, tk, ef, dgks);
  else if (nb == 2)
    e = launch_k(project_stream_kernel<2>, grid, block, sh, st, maps, dim, s, c, ldc, y, ldy, norms2, ctx->partials, tk, ef, dgks);
  else if (nb == 3)
    e = launch_k(project_stream_kernel<3>, grid, block, sh, st, maps, dim, s, c, ldc, y, ldy, norms2, ctx->partials, tk, ef, dgks);
  else
    e = launch_k(project_stream_kernel<4>, grid, block, sh, st, maps, dim, s, c, ldc, y, ldy, norms2, ctx->partials, tk, ef, dgks);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  bump_launches();
  return true;
}

int gram_impl(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs, const int *cols,
              const double *y, int64_t ldy, int b, double *c, int64_t ldc, double *norms2, void *stream, HInsert hi) {
  SVDSB_CHECK_ARG(ctx != nullptr, "svdsb_gram: NULL ctx");
  SVDSB_CHECK_ARG(hi.h == nullptr || b == 1, "gram_impl: the H epilogue is for one column");
  ColSet s;
  int rc = make_colset(s, nblk, xs, ldxs, cols);
  if (rc) return rc;
  if (b <= 0) return SVDSB_OK;
  SVDSB_CHECK_ARG(s.total <= 4 * SVDSB_SMALL_MAX, "svdsb_gram: too many columns");
  cudaStream_t st = as_stream(stream);
  const int gx = grid_rows(dim);
  if (s.total == 0) {
    if (norms2) return svdsb_col_norms2(ctx, dim, y, ldy, b, norms2, stream);
    return SVDSB_OK;
  }
  if (b == 1 && colset_vec_ok(s) && aligned16(y) && s.total <= kGsMaxX && stream_one_col(dim) &&
      gram_stream(ctx, dim, s, y, ldy, 1, c, ldc, norms2, st, nullptr, hi)) {
    return SVDSB_OK;
  }
  if (b == 1 && colset_vec_ok(s) && aligned16(y)) {
    if (s.total <= 16) {
      dim3 grid(grid_for(gram1_vec_kernel<16>, dim, 0), 1, 1);
      SVDSB_LAUNCH_PDL(gram1_vec_kernel<16>, grid, kThreads, 0, st, dim, s, y, c, norms2, ctx->partials,
                       take_ticket(ctx), nullptr, hi);
    } else {
      constexpr int AT = 40;
      // latency-bound sizes (L2-scale N): one CTA per SM halves the partials
      // the last CTA folds (measured 12.4 -> 9.9 us on config 2)
      int gxv = grid_for(gram1_vec_kernel<AT>, dim, 0);
      if (dim <= (1 << 18) && gxv > num_sms()) gxv = num_sms();
      dim3 grid(gxv, (s.total + AT - 1) / AT, 1);
      SVDSB_LAUNCH_PDL(gram1_vec_kernel<AT>, grid, kThreads, 0, st, dim, s, y, c, norms2, ctx->partials,
                       take_ticket(ctx), nullptr, hi);
    }
    return SVDSB_OK;
  } else if (b >= 2 && colset_vec_ok(s) && aligned16(y) && ldy % 2 == 0 && s.total <= kGsMaxX && stream_ok(dim) &&
             gram_stream(ctx, dim, s, y, ldy, b, c, ldc, norms2, st)) {
    return SVDSB_OK;
  } else if (b >= 2 && colset_vec_ok(s) && aligned16(y) && ldy % 2 == 0) {
    // four columns of y per launch (a 2- or 3-column tail masks the rest);
    // wide blocks (full H rebuilds) in chunks of four: 4x faster than one
    // generic launch at g = 14..35
    constexpr int AT = 8;
    const int ny = (s.total + AT - 1) / AT;
    dim3 grid(grid_for(gram4_vec_kernel<AT, 4>, dim, 0), ny, 1);
    SVDSB_CHECK_ARG((int64_t)grid.x * grid.y * (AT * 4 + 4) <= kMaxPartials, "gram: workspace too small");
    for (int j0 = 0; j0 < b; j0 += 4) {
      const int nb = std::min(4, b - j0);
      const double *yj = y + (int64_t)j0 * ldy;
      double *cj = c + (int64_t)j0 * ldc;
      double *nj = norms2 ? norms2 + j0 : nullptr;
      auto k = nb == 4 ? gram4_vec_kernel<AT, 4> : nb == 3 ? gram4_vec_kernel<AT, 3>
             : nb == 2 ? gram4_vec_kernel<AT, 2> : gram4_vec_kernel<AT, 1>;
      if (g_tune[1] != 2) {  // 2: column groups outermost (the slower order)
        SVDSB_LAUNCH_PDL(k, dim3(grid.x * ny, 1, 1), kThreads, 0, st, dim, s, yj, ldy, cj, ldc, nj, ctx->partials,
                         take_ticket(ctx), ny);
      } else {
        SVDSB_LAUNCH_PDL(k, grid, kThreads, 0, st, dim, s, yj, ldy, cj, ldc, nj, ctx->partials, take_ticket(ctx), 0);
      }
    }
    return SVDSB_OK;
  } else if (b == 1) {
    SVDSB_CHECK_ARG(hi.h == nullptr, "gram_impl: the H epilogue needs 16-byte aligned operands");
    constexpr int AT = 32, BT = 1;
    dim3 grid(gx, (s.total + AT - 1) / AT, 1);
    SVDSB_CHECK_ARG((int64_t)grid.x * grid.y * (AT * BT + BT) <= kMaxPartials, "gram: workspace too small");
    gram_kernel<AT, BT><<<grid, kThreads, 0, st>>>(dim, s, y, ldy, b, c, ldc, norms2, ctx->partials,
                                                   take_ticket(ctx));
  } else {
    constexpr int AT = 16, BT = 4;
    dim3 grid(gx, (s.total + AT - 1) / AT, (b + BT - 1) / BT);
    SVDSB_CHECK_ARG((int64_t)grid.x * grid.y * grid.z * (AT * BT + BT) <= kMaxPartials, "gram: workspace too small");
    gram_kernel<AT, BT><<<grid, kThreads, 0, st>>>(dim, s, y, ldy, b, c, ldc, norms2, ctx->partials,
                                                   take_ticket(ctx));
  }
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

}  // namespace svdsb

extern "C" {

int svdsb_project_out(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs,
                      const int *cols, const double *c, int64_t ldc, double *y, int64_t ldy, int b, double *norms2,
                      void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr, "svdsb_project_out: NULL ctx");
  ColSet s;
  int rc = make_colset(s, nblk, xs, ldxs, cols);
  if (rc) return rc;
  if (b <= 0) return SVDSB_OK;
  SVDSB_CHECK_ARG(s.total <= 256, "svdsb_project_out: at most 256 columns");
  cudaStream_t st = as_stream(stream);
  for (int j0 = 0; j0 < b; j0 += 8) {
    int bb = std::min(8, b - j0);
    const int gx = grid_rows(dim);
    double *yy = y + (int64_t)j0 * ldy;
    const double *cc = c + (int64_t)j0 * ldc;
    double *nn = norms2 ? norms2 + j0 : nullptr;
    // two columns: 74 -> 64 us at N = 1 M (four are faster on project4_vec_kernel: 78 vs 88 us;
    // one column is opt-in, see stream_one_col); key 15 = 2 forces every width
    if (((bb == 2 && stream_ok(dim) && g_tune[15] != 5) || (bb <= 4 && g_tune[15] == 2) || (bb == 1 && stream_one_col(dim))) &&
        colset_vec_ok(s) &&
        project_stream(ctx, dim, s, cc, ldc, yy, ldy, bb, nn, st)) {
      continue;
    }
    if (bb == 1 && colset_vec_ok(s) && aligned16(yy)) {
      size_t sh = sizeof(double) * std::max(s.total, 1);
      SVDSB_LAUNCH_PDL(project1_vec_kernel, grid_for(project1_vec_kernel, dim, sh), kThreads, sh, st, dim, s, cc, yy,
                       nn, ctx->partials, take_ticket(ctx), (double *)nullptr);
      continue;
    } else if (bb >= 2 && bb <= 4 && colset_vec_ok(s) && aligned16(yy) && ldy % 2 == 0) {
      // (2 and 3 columns went through the generic kernel: 209 vs 78 us at N = 1 M, g = 35)
      size_t sh = sizeof(double) * std::max(s.total, 1) * bb;
      auto k = bb == 4 ? project4_vec_kernel<4> : bb == 3 ? project4_vec_kernel<3> : project4_vec_kernel<2>;
      SVDSB_LAUNCH_PDL(k, grid_for(k, dim, sh), kThreads, sh, st, dim, s, cc, ldc, yy, ldy, nn, ctx->partials,
                       take_ticket(ctx));
      continue;
    } else if (bb == 1) {
      size_t sh = sizeof(double) * std::max(s.total, 1) * 1;
      project_kernel<1><<<gx, kThreads, sh, st>>>(dim, s, cc, ldc, yy, ldy, bb, nn, ctx->partials, take_ticket(ctx));
    } else {
      size_t sh = sizeof(double) * std::max(s.total, 1) * 8;
      project_kernel<8><<<gx, kThreads, sh, st>>>(dim, s, cc, ldc, yy, ldy, bb, nn, ctx->partials, take_ticket(ctx));
    }
    SVDSB_LAUNCHED();
  }
  return SVDSB_OK;
}

int svdsb_ts_gemm(svdsb_ctx *ctx, int64_t dim, const double *x, int64_t ldx, int g, const double *c, int64_t ldc,
                  int s, double alpha, double beta, double *y, int64_t ldy, void *stream) {
  (void)ctx;
  if (s <= 0 || dim == 0) return SVDSB_OK;
  SVDSB_CHECK_ARG(g >= 0 && g <= 256, "svdsb_ts_gemm: g out of range");
  cudaStream_t st = as_stream(stream);
  if (g == 0) {
    // Y = beta Y
    return svdsb_axpby(dim, s, 0.0, y, ldy, beta, y, ldy, stream);
  }
  if (x == y) {
    SVDSB_CHECK_ARG(ldx == ldy && s <= g && s <= 32 && alpha == 1.0 && beta == 0.0,
                    "svdsb_ts_gemm: in-place needs ldy == ldx, s <= min(g, 32), alpha 1, beta 0");
    if (aligned16(y) && !(ldy & 1) && g_tune[4] != 2 && g <= kTsMaxG && stream_ok(dim)) {
      const int pt = s <= 8 ? 8 : s <= 16 ? 16 : s <= 24 ? 24 : 32;
      const size_t shs = ts_stream_smem(1, g, pt);
      static bool attrs = false;
      if (!attrs) {
        const size_t mx = ts_stream_smem(1, kTsMaxG, 32);
        SVDSB_CUDA(stream_attr(ts_stream_kernel<1, 256, 2, 2, 4, false>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<1, 256, 2, 2, 8, false>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<1, 256, 4, 4, 6, false>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<1, 256, 4, 4, 8, false>, mx));
        attrs = true;
      }
      auto ks = pt == 8 ? ts_stream_kernel<1, 256, 2, 2, 4, false> : pt == 16 ? ts_stream_kernel<1, 256, 2, 2, 8, false>
              : pt == 24 ? ts_stream_kernel<1, 256, 4, 4, 6, false> : ts_stream_kernel<1, 256, 4, 4, 8, false>;
      CUtensorMap mx;
      if (make_map2d(&mx, y, dim, g, ldy, kTsRows, ts_kc(1))) {
        ks<<<stream_grid_tiles(dim, kTsRows), kTsThreads, shs, st>>>(
            mx, mx, dim, g, c, ldc, nullptr, s, y, ldy, nullptr, 0, nullptr, 0, nullptr, nullptr, nullptr, StatusOut{},
            stream_evict_first(dim, g));
        SVDSB_LAUNCHED();
        return SVDSB_OK;
      }
    }
    if (aligned16(y) && !(ldy & 1) && g_tune[4] != 2) {
      auto k = s <= 8 ? ts_gemm_inplace_vec_kernel<8> : s <= 16 ? ts_gemm_inplace_vec_kernel<16>
             : s <= 24 ? ts_gemm_inplace_vec_kernel<24> : ts_gemm_inplace_vec_kernel<32>;
      const int st_cols = s <= 8 ? 8 : s <= 16 ? 16 : s <= 24 ? 24 : 32;
      const size_t shv = sizeof(double) * g * st_cols;
      static bool attrv = false;
      if (!attrv) {
        for (auto kk : {ts_gemm_inplace_vec_kernel<8>, ts_gemm_inplace_vec_kernel<16>,
                        ts_gemm_inplace_vec_kernel<24>, ts_gemm_inplace_vec_kernel<32>})
          SVDSB_CUDA(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(double) * 256 * 32)));
        attrv = true;
      }
      k<<<grid_for(k, dim, shv), kThreads, shv, st>>>(dim, y, ldy, g, c, ldc, s);
      SVDSB_LAUNCHED();
      return SVDSB_OK;
    }
    size_t sh = sizeof(double) * g * 32;
    static bool attr = false;
    if (!attr) {
      SVDSB_CUDA(cudaFuncSetAttribute(ts_gemm_inplace_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(double) * 256 * 32)));
      attr = true;
    }
    ts_gemm_inplace_kernel<32><<<grid_rows(dim), kThreads, sh, st>>>(dim, y, ldy, g, c, ldc, s);
    SVDSB_LAUNCHED();
    return SVDSB_OK;
  }
  constexpr int ST = 16;
  if (s <= ST && aligned16(x) && aligned16(y) && !(ldx & 1) && !(ldy & 1)) {
    size_t sh = sizeof(double) * g * ST;
    ts_gemm_vec_kernel<ST><<<grid_for(ts_gemm_vec_kernel<ST>, dim, sh), kThreads, sh, st>>>(dim, x, ldx, g, c, ldc, s, alpha, beta, y, ldy);
    SVDSB_LAUNCHED();
    return SVDSB_OK;
  }
  dim3 grid(grid_rows(dim), (s + ST - 1) / ST);
  size_t sh = sizeof(double) * g * ST;
  ts_gemm_kernel<ST><<<grid, kThreads, sh, st>>>(dim, x, ldx, g, c, ldc, s, alpha, beta, y, ldy);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_ritz_residual(svdsb_ctx *ctx, int64_t dim, const double *v, int64_t ldv, const double *w, int64_t ldw,
                        int g, const double *yc, int64_t ldyc, const double *lam, int p, double *r, int64_t ldr,
                        double *x, int64_t ldx, double *ox, int64_t ldox, double *rn2, void *stream) {
  return svdsb::ritz_impl(ctx, dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x, ldx, ox, ldox, rn2, stream,
                          svdsb::StatusOut{});
}

}  // extern "C"

namespace svdsb {

int ritz_impl(svdsb_ctx *ctx, int64_t dim, const double *v, int64_t ldv, const double *w, int64_t ldw, int g,
              const double *yc, int64_t ldyc, const double *lam, int p, double *r, int64_t ldr, double *x,
              int64_t ldx, double *ox, int64_t ldox, double *rn2, void *stream, StatusOut so) {
  SVDSB_CHECK_ARG(ctx != nullptr, "svdsb_ritz_residual: NULL ctx");
  SVDSB_CHECK_ARG(so.host == nullptr || (p <= 32 && rn2 != nullptr), "ritz_impl: status epilogue needs p <= 32");
  if (p <= 0) return SVDSB_OK;
  SVDSB_CHECK_ARG(g >= 1 && g <= 256, "svdsb_ritz_residual: g out of range");
  cudaStream_t st = as_stream(stream);
  if (g <= 4 * kDmmaMaxK && p <= 32 && g_tune[11] == 1) {
    // fp64 tensor-core variant: measured slower than the FMA kernels at
    // config-3 size (g = 35, p = 11: 910 vs 639 us, ~10 TFLOP/s of DMMA)
    auto *tk = take_ticket(ctx);
#define SVDSB_RITZ_DMMA(NT)                                                                                    \
  SVDSB_LAUNCH_PDL(ritz_dmma_kernel<NT>, grid_for(ritz_dmma_kernel<NT>, dim, 0), kThreads, 0, st, dim, v, ldv, w,  \
                   ldw, g, yc, ldyc, lam, p, r, ldr, x, ldx, ox, ldox, rn2, ctx->partials, tk, so)
    if (p <= 8)
      SVDSB_RITZ_DMMA(1);
    else if (p <= 16)
      SVDSB_RITZ_DMMA(2);
    else if (p <= 24)
      SVDSB_RITZ_DMMA(3);
    else
      SVDSB_RITZ_DMMA(4);
#undef SVDSB_RITZ_DMMA
    return SVDSB_OK;
  }
  {
    const bool vec = aligned16(v) && aligned16(w) && aligned16(r) && !(ldv & 1) && !(ldw & 1) && !(ldr & 1) &&
                     (x == nullptr || (aligned16(x) && !(ldx & 1))) && (ox == nullptr || (aligned16(ox) && !(ldox & 1)));
    if (vec && p <= 32 && g <= kTsMaxG && stream_ok(dim)) {
      const int pt = p <= 8 ? 8 : p <= 12 ? 12 : p <= 16 ? 16 : p <= 24 ? 24 : 32;
      const size_t shs = ts_stream_smem(2, g, pt);
      static bool attrs = false;
      if (!attrs) {
        const size_t mx = ts_stream_smem(2, kTsMaxG, 32);
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 256, 2, 2, 4, true>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 256, 2, 2, 6, true>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 256, 2, 2, 8, true>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 256, 4, 4, 6, true>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 256, 4, 4, 8, true>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 384, 2, 4, 6, true>, mx));
        SVDSB_CUDA(stream_attr(ts_stream_kernel<2, 512, 2, 4, 6, true>, mx));
        attrs = true;
      }
      if (pt == 24 && g_tune[15] == 4) {
        // sixteen warps of two rows x six candidates (4 per sub-partition, <= 128 registers)
        constexpr int rows = ts_rows(512, 2, 4);
        CUtensorMap mv, mw;
        if (make_map2d(&mv, v, dim, g, ldv, rows, ts_kc(2)) && make_map2d(&mw, w, dim, g, ldw, rows, ts_kc(2))) {
          SVDSB_LAUNCH_PDL(ts_stream_kernel<2, 512, 2, 4, 6, true>, dim3(stream_grid_tiles(dim, rows), 1, 1), 512,
                           ts_stream_smem(2, g, pt, rows), st, mv, mw, dim, g, yc, ldyc, lam, p, r, ldr, x, ldx, ox, ldox,
                           rn2, ctx->partials, take_ticket(ctx), so, stream_evict_first(dim, 2 * g));
          return SVDSB_OK;
        }
      }
      if (pt == 24 && g_tune[15] == 3) {
        // twelve warps of two rows x six candidates (3 per sub-partition, <= 168 registers)
        constexpr int rows = ts_rows(384, 2, 4);
        CUtensorMap mv, mw;
        if (make_map2d(&mv, v, dim, g, ldv, rows, ts_kc(2)) && make_map2d(&mw, w, dim, g, ldw, rows, ts_kc(2))) {
          SVDSB_LAUNCH_PDL(ts_stream_kernel<2, 384, 2, 4, 6, true>, dim3(stream_grid_tiles(dim, rows), 1, 1), 384,
                           ts_stream_smem(2, g, pt, rows), st, mv, mw, dim, g, yc, ldyc, lam, p, r, ldr, x, ldx, ox, ldox,
                           rn2, ctx->partials, take_ticket(ctx), so, stream_evict_first(dim, 2 * g));
          return SVDSB_OK;
        }
      }
      CUtensorMap mv, mw;
      if (make_map2d(&mv, v, dim, g, ldv, kTsRows, ts_kc(2)) && make_map2d(&mw, w, dim, g, ldw, kTsRows, ts_kc(2))) {
        auto *tk = take_ticket(ctx);
        const dim3 grid(stream_grid_tiles(dim, kTsRows), 1, 1);
        const int ef = stream_evict_first(dim, 2 * g);
#define SVDSB_RITZ_STREAM(RPT, PQV)                                                                            \
  SVDSB_LAUNCH_PDL(ts_stream_kernel<2, 256, RPT, RPT, PQV, true>, grid, kTsThreads, shs, st, mv, mw, dim, g, yc, ldyc, \
                   lam, p, r, ldr, x, ldx, ox, ldox, rn2, ctx->partials, tk, so, ef)
        if (pt == 8)
          SVDSB_RITZ_STREAM(2, 4);
        else if (pt == 12)
          SVDSB_RITZ_STREAM(2, 6);
        else if (pt == 16)
          SVDSB_RITZ_STREAM(2, 8);
        else if (pt == 24)
          SVDSB_RITZ_STREAM(4, 6);
        else
          SVDSB_RITZ_STREAM(4, 8);
        return SVDSB_OK;
      }
#undef SVDSB_RITZ_STREAM
    }
  }
  if (p > 16 && p <= 32 && g_tune[3] != 1) {
    // two threads per row, 12 or 16 candidates each (config 4, p = 24:
    // 336 -> 295 us; for p <= 16 the one-thread kernel is faster -- config
    // 3, p = 11: 637 vs 716 us; g_tune[3] = 2 forces the split there too)
    auto *tk = take_ticket(ctx);
#define SVDSB_RITZ_SPLIT(PQ)                                                                                   \
  SVDSB_LAUNCH_PDL(ritz_split_kernel<PQ, 2>, grid_for(ritz_split_kernel<PQ, 2>, dim, sizeof(double) * g * 2 * PQ), \
                   kThreads, sizeof(double) * g * 2 * PQ, st, dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x,  \
                   ldx, ox, ldox, rn2, ctx->partials, tk, so)
    const bool vec = aligned16(v) && aligned16(w) && aligned16(r) && !(ldv & 1) && !(ldw & 1) && !(ldr & 1) &&
                     (x == nullptr || (aligned16(x) && !(ldx & 1))) && (ox == nullptr || (aligned16(ox) && !(ldox & 1)));
    if (vec && p <= 24 && g_tune[3] == 4) {  // measured slower on config 4 (386 vs 296 us); PQ = 16 would spill
#define SVDSB_RITZ_R2(PQ)                                                                                      \
  SVDSB_LAUNCH_PDL(ritz_split_r2_kernel<PQ>, grid_for(ritz_split_r2_kernel<PQ>, dim, sizeof(double) * g * 2 * PQ),  \
                   kThreads, sizeof(double) * g * 2 * PQ, st, dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x,  \
                   ldx, ox, ldox, rn2, ctx->partials, tk, so)
      SVDSB_RITZ_R2(12);
#undef SVDSB_RITZ_R2
      return SVDSB_OK;
    }
    if (p <= 24)
      SVDSB_RITZ_SPLIT(12);
    else
      SVDSB_RITZ_SPLIT(16);
#undef SVDSB_RITZ_SPLIT
    return SVDSB_OK;
  }
  if (p > 8 && p <= 16 && g_tune[3] == 2) {
    auto *tk = take_ticket(ctx);
    if (p <= 12)
      SVDSB_LAUNCH_PDL(ritz_split_kernel<6, 2>, grid_for(ritz_split_kernel<6, 2>, dim, sizeof(double) * g * 12),
                       kThreads, sizeof(double) * g * 12, st, dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x, ldx,
                       ox, ldox, rn2, ctx->partials, tk, so);
    else
      SVDSB_LAUNCH_PDL(ritz_split_kernel<8, 2>, grid_for(ritz_split_kernel<8, 2>, dim, sizeof(double) * g * 16),
                       kThreads, sizeof(double) * g * 16, st, dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x, ldx,
                       ox, ldox, rn2, ctx->partials, tk, so);
    return SVDSB_OK;
  }
  if (p <= 32) {
    auto *tk = take_ticket(ctx);
#define SVDSB_RITZ_WIDE(PTV)                                                                                  \
  SVDSB_LAUNCH_PDL(ritz_wide_kernel<PTV>, grid_for(ritz_wide_kernel<PTV>, dim, sizeof(double) * g * PTV), kThreads,  \
                   sizeof(double) * g * PTV, st, dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x, ldx, ox, ldox, \
                   rn2, ctx->partials, tk, so)
    if (p <= 4)
      SVDSB_RITZ_WIDE(4);
    else if (p <= 8)
      SVDSB_RITZ_WIDE(8);
    else if (p <= 12)
      SVDSB_RITZ_WIDE(12);
    else if (p <= 16)
      SVDSB_RITZ_WIDE(16);
    else if (p <= 24)
      SVDSB_RITZ_WIDE(24);
    else
      SVDSB_RITZ_WIDE(32);
#undef SVDSB_RITZ_WIDE
    return SVDSB_OK;
  }
  constexpr int PT = 12;
  dim3 grid(grid_rows(dim), (p + PT - 1) / PT);
  size_t sh = sizeof(double) * g * PT;
  ritz_kernel<PT><<<grid, kThreads, sh, st>>>(dim, v, ldv, w, ldw, g, yc, ldyc, lam, p, r, ldr, x, ldx, ox, ldox, rn2,
                                              ctx->partials, take_ticket(ctx));
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

}  // namespace svdsb

extern "C" {

int svdsb_col_norms2(svdsb_ctx *ctx, int64_t dim, const double *x, int64_t ldx, int b, double *out, void *stream) {
  return svdsb_col_dots(ctx, dim, x, ldx, x, ldx, b, out, stream);
}

int svdsb_col_dots(svdsb_ctx *ctx, int64_t dim, const double *x, int64_t ldx, const double *y, int64_t ldy, int b,
                   double *out, void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr, "svdsb_col_dots: NULL ctx");
  if (b <= 0) return SVDSB_OK;
  constexpr int BT = 8;
  dim3 grid(grid_rows(dim), (b + BT - 1) / BT);
  coldot_kernel<BT><<<grid, kThreads, 0, as_stream(stream)>>>(dim, x, ldx, y, ldy, b, out, ctx->partials,
                                                              take_ticket(ctx));
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_split_stats(svdsb_ctx *ctx, int64_t dim, int64_t nsplit, const double *r, int64_t ldr, const double *x,
                      int64_t ldx, int b, double *out, void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr, "svdsb_split_stats: NULL ctx");
  if (b <= 0) return SVDSB_OK;
  constexpr int BT = 4;
  dim3 grid(grid_rows(dim), (b + BT - 1) / BT);
  split_kernel<BT><<<grid, kThreads, 0, as_stream(stream)>>>(dim, nsplit, r, ldr, x, ldx, b, out, ctx->partials,
                                                             take_ticket(ctx));
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_split_residual(svdsb_ctx *ctx, int64_t dim, int64_t nsplit, const double *r, int64_t ldr,
                         const double *x, int64_t ldx, int b, const double *lam, const double *stats, double *out,
                         void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr, "svdsb_split_residual: NULL ctx");
  if (b <= 0) return SVDSB_OK;
  constexpr int BT = 4;
  dim3 grid(grid_rows(dim), (b + BT - 1) / BT);
  split_res_kernel<BT><<<grid, kThreads, 0, as_stream(stream)>>>(dim, nsplit, r, ldr, x, ldx, b, lam, stats, out,
                                                                 ctx->partials, take_ticket(ctx));
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_scale_cols(int64_t dim, const double *x, int64_t ldx, int b, const double *s, int mode, double *y,
                     int64_t ldy, void *stream) {
  if (dim == 0 || b <= 0) return SVDSB_OK;
  SVDSB_CHECK_ARG(mode >= 0 && mode <= 2, "svdsb_scale_cols: bad mode");
  SVDSB_LAUNCH_PDL(scale_kernel, (unsigned)((dim + 255) / 256), 256, 0, as_stream(stream), dim, x, ldx, b, s, mode, y,
                   ldy);
  return SVDSB_OK;
}

int svdsb_axpby(int64_t dim, int b, double alpha, const double *x, int64_t ldx, double beta, double *y, int64_t ldy,
                void *stream) {
  if (dim == 0 || b <= 0) return SVDSB_OK;
  SVDSB_LAUNCH_PDL(axpby_kernel, (unsigned)((dim + 255) / 256), 256, 0, as_stream(stream), dim, b, alpha, x, ldx, beta,
                   y, ldy);
  return SVDSB_OK;
}

int svdsb_gather_cols(int64_t dim, const double *x, int64_t ldx, const int *first, int ncols, int limit,
                      const double *d, double *y, int64_t ldy, void *stream) {
  SVDSB_CHECK_ARG(first != nullptr, "svdsb_gather_cols: NULL index");
  if (dim == 0 || ncols <= 0) return SVDSB_OK;
  SVDSB_LAUNCH_PDL(gather_cols_kernel, (unsigned)((dim + 255) / 256), 256, 0, as_stream(stream), dim, x, ldx, first,
                   ncols, limit, d, y, ldy);
  return SVDSB_OK;
}

int svdsb_status_pack_n(const double *lams, int gn, const double *rn2, int p, const double *state, int nstate,
                        double *host_dst, void *stream) {
  SVDSB_CHECK_ARG(lams != nullptr && rn2 != nullptr && state != nullptr && host_dst != nullptr,
                  "svdsb_status_pack: NULL argument");
  SVDSB_CHECK_ARG(nstate >= 1 && nstate <= 64, "svdsb_status_pack: 1..64 DGKS records");
  SVDSB_LAUNCH_PDL(status_pack_kernel, 1, 128, 0, as_stream(stream), lams, gn, rn2, p, state, nstate, host_dst);
  return SVDSB_OK;
}

int svdsb_status_pack(const double *lams, int gn, const double *rn2, int p, const double *state,
                      double *host_dst, void *stream) {
  return svdsb_status_pack_n(lams, gn, rn2, p, state, 1, host_dst, stream);
}

int svdsb_randn(uint64_t seed, int64_t row0, int64_t rows, int cols, double *out, int64_t ldo, void *stream) {
  SVDSB_CHECK_ARG(out != nullptr && rows >= 0 && cols >= 0 && row0 >= 0 && (cols == 0 || ldo >= rows),
                  "svdsb_randn: bad arguments");
  const int64_t tot = rows * cols;
  if (tot == 0) return SVDSB_OK;
  SVDSB_LAUNCH_PDL(randn_kernel, (unsigned)((tot + 255) / 256), 256, 0, as_stream(stream), seed, row0, rows, cols,
                   out, ldo);
  return SVDSB_OK;
}

int svdsb_set_int(int *dst, int v, void *stream) {
  SVDSB_CHECK_ARG(dst != nullptr, "svdsb_set_int: NULL destination");
  SVDSB_LAUNCH_PDL(set_int_kernel, 1, 32, 0, as_stream(stream), dst, v);
  return SVDSB_OK;
}

int svdsb_dgks_begin(double *state, void *stream) {
  SVDSB_LAUNCH_PDL(dgks_begin_kernel, 1, 32, 0, as_stream(stream), state);
  return SVDSB_OK;
}

int svdsb_cgs_fused(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs,
                    const int *cols, const double *rsrc, int64_t ldr, const int *ci, const double *d, double *x,
                    const double *yin, int64_t ldyin, int g, int kk, double *prev, int64_t ldprev, int passes,
                    double *state, void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr && state != nullptr && ci != nullptr && rsrc != nullptr && x != nullptr,
                  "svdsb_cgs_fused: NULL argument");
  ColSet s;
  int rc = make_colset(s, nblk, xs, ldxs, cols);
  if (rc) return rc;
  SVDSB_CHECK_ARG(s.total >= 1 && s.total <= kCgsMaxCols, "svdsb_cgs_fused: 1..40 prior columns");
  SVDSB_CHECK_ARG(colset_vec_ok(s) && aligned16(x), "svdsb_cgs_fused: operands must be 16-byte aligned");
  SVDSB_CHECK_ARG(passes >= 1 && passes <= 6, "svdsb_cgs_fused: 1..6 passes");
  if (dim == 0) return SVDSB_OK;
  if (!svdsb_cgs_fused_supported()) {
    set_error("svdsb_cgs_fused: cooperative launch unavailable on this device (use svdsb_cgs_pass)");
    return SVDSB_ERR_CUDA;
  }
  // one CTA per SM: all resident for the grid barrier; the cooperative
  // attribute makes the launch fail rather than hang if they cannot be
  const int grid = stream_grid(dim, 2 * kCgsThreads, num_sms());
  SVDSB_CHECK_ARG((int64_t)grid * (kCgsMaxCols + 2) <= kMaxPartials, "svdsb_cgs_fused: workspace too small");
  cudaError_t e = launch_coop(cgs_fused_kernel, grid, kCgsThreads, 0, as_stream(stream), dim, s, rsrc, ldr, ci, d,
                              x, yin, ldyin, g, kk, prev, ldprev, passes, state, ctx->partials, ctx->gbar);
  if (e != cudaSuccess) {
    set_error("svdsb_cgs_fused: cooperative launch of %d CTAs failed: %s", grid, cudaGetErrorString(e));
    return SVDSB_ERR_CUDA;
  }
  bump_launches();
  return SVDSB_OK;
}

int svdsb_cgs_fused_supported(void) {
  static int ok[64] = {0};  // 0 unknown, 1 yes, -1 no
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  if (ok[dev] == 0) {
    int coop = 0, occ = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cgs_fused_kernel, kCgsThreads, 0) != cudaSuccess)
      occ = 0;
    ok[dev] = (coop && occ >= 1) ? 1 : -1;
  }
  return ok[dev] == 1;
}

int svdsb_cgs_block(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs,
                    const int *cols, double *v, int64_t ldv, int b, double *cwork, double *state, int passes,
                    void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr && v != nullptr && cwork != nullptr && state != nullptr,
                  "svdsb_cgs_block: NULL argument");
  SVDSB_CHECK_ARG(b >= 1 && b <= 32 && passes >= 1 && passes <= 6, "svdsb_cgs_block: 1..32 columns, 1..6 passes");
  SVDSB_CHECK_ARG(nblk >= 1 && nblk < SVDSB_MAX_BLOCKS, "svdsb_cgs_block: 1..MAX_BLOCKS-1 prior blocks");
  ColSet s;
  int rc = make_colset(s, nblk, xs, ldxs, cols);
  if (rc) return rc;
  SVDSB_CHECK_ARG(s.total >= 1 && s.total + b <= 256, "svdsb_cgs_block: 1..256 prior columns");
  if (dim == 0) return SVDSB_OK;
  // cwork: C (total x b) | before2 (b) | after2 (b)
  double *c = cwork, *before2 = cwork + (int64_t)s.total * b, *after2 = before2 + b;
  // pass 1, old part, all columns at once: C = X^T V (norms before), V -= X C (norms after)
  if ((rc = svdsb_gram(ctx, dim, nblk, xs, ldxs, cols, v, ldv, b, c, s.total, before2, stream))) return rc;
  if ((rc = svdsb_project_out(ctx, dim, nblk, xs, ldxs, cols, c, s.total, v, ldv, b, after2, stream))) return rc;
  SVDSB_LAUNCH_PDL(dgks_seed_kernel, 1, 32, 0, as_stream(stream), state, b, (const double *)before2,
                   (const double *)after2);
  const double *xs2[SVDSB_MAX_BLOCKS];
  int64_t ld2[SVDSB_MAX_BLOCKS];
  int cols2[SVDSB_MAX_BLOCKS];
  for (int k = 0; k < nblk; ++k) {
    xs2[k] = xs[k];
    ld2[k] = ldxs[k];
    cols2[k] = cols[k];
  }
  xs2[nblk] = v;
  ld2[nblk] = ldv;
  for (int j = 0; j < b; ++j) {
    double *vj = v + (int64_t)j * ldv, *st = state + 8 * j;
    if (j > 0) {
      // pass 1, new part: against the finished columns 0..j-1 of the block;
      // the projection's last CTA applies the DGKS decision of the pass
      const double *nb[1] = {v};
      const int64_t nl[1] = {ldv};
      const int nc[1] = {j};
      if ((rc = svdsb_cgs_pass(ctx, dim, 1, nb, nl, nc, vj, cwork + (int64_t)s.total * b + 2 * b, st, 0, stream)))
        return rc;
    }
    cols2[nblk] = j;
    const int nb2 = j > 0 ? nblk + 1 : nblk;
    for (int p = 1; p < passes; ++p)
      if ((rc = svdsb_cgs_pass(ctx, dim, nb2, xs2, ld2, cols2, vj, cwork + (int64_t)s.total * b + 2 * b, st, 0,
                               stream)))
        return rc;
    if ((rc = svdsb_scale_cols(dim, vj, ldv, 1, st + 5, 1 /* divide */, vj, ldv, stream))) return rc;
  }
  return SVDSB_OK;
}

int svdsb_cgs_pass(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs,
                   const int *cols, double *v, double *cwork, double *state, int first_pass, void *stream) {
  SVDSB_CHECK_ARG(ctx != nullptr && state != nullptr, "svdsb_cgs_pass: NULL argument");
  ColSet s;
  int rc = make_colset(s, nblk, xs, ldxs, cols);
  if (rc) return rc;
  SVDSB_CHECK_ARG(s.total >= 1 && s.total <= 256, "svdsb_cgs_pass: 1..256 prior columns");
  SVDSB_CHECK_ARG(colset_vec_ok(s) && aligned16(v), "svdsb_cgs_pass: operands must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  double *n0 = first_pass ? state + 6 : nullptr;
  if (s.total <= kGsMaxX && stream_one_col(dim)) {
    // both halves of the pass on the streamed kernels (or neither: a pass
    // whose Gram ran must be followed by its projection)
    ProjMaps probe;
    bool ok = aligned16(v);
    for (int k = 0; ok && k < s.nblk; ++k) ok = make_map2d(&probe.x[0], s.base[k], dim, s.cols[k], s.ld[k], kPsRows, kGsBox);
    int cap = 4;
    for (int k = 0; k < s.nblk; ++k) cap += (s.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
    if (ok && cap <= kPsCap && gram_stream(ctx, dim, s, v, 0, 1, cwork, s.total, n0, st, state, HInsert{})) {
      if (project_stream(ctx, dim, s, cwork, s.total, v, 0, 1, state + 7, st, state)) return SVDSB_OK;
      set_error("svdsb_cgs_pass: streamed projection failed after its Gram");
      return SVDSB_ERR_CUDA;
    }
  }
  if (s.total <= 16) {
    dim3 grid(grid_for(gram1_vec_kernel<16>, dim, 0), 1, 1);
    SVDSB_LAUNCH_PDL(gram1_vec_kernel<16>, grid, kThreads, 0, st, dim, s, v, cwork, n0, ctx->partials,
                     take_ticket(ctx), state, HInsert{});
  } else {
    constexpr int AT = 40;
    dim3 grid(grid_for(gram1_vec_kernel<AT>, dim, 0), (s.total + AT - 1) / AT, 1);
    SVDSB_LAUNCH_PDL(gram1_vec_kernel<AT>, grid, kThreads, 0, st, dim, s, v, cwork, n0, ctx->partials,
                     take_ticket(ctx), state, HInsert{});
  }
  size_t sh = sizeof(double) * s.total;
  SVDSB_LAUNCH_PDL(project1_vec_kernel, grid_for(project1_vec_kernel, dim, sh), kThreads, sh, st, dim, s, cwork, v,
                   state + 7, ctx->partials, take_ticket(ctx), state);
  return SVDSB_OK;
}

}  // extern "C"
