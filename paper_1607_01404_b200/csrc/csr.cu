// Device CSR of A with a stored transpose, and the block SpMV kernels.
//
// Reference: SparseMatrixCsr / spmv_block (pkg/src/itersvd/matio.py:22-155).
// The reference keeps no transpose and scatters with np.add.at; here A^T is
// stored as its own CSR (a stable counting/radix sort by column, bit-exact
// with SparseMatrixCsr.from_coo(n, m, col_idx, rows, values)) so both
// products are row-gathers with coalesced index/value streams.
//
// Kernel design (HBM-bound, ~0.17 flop/byte):
//  * short rows: "CSR-stream" tiles of <= 256 rows / <= 2048 nnz per CTA.
//    Values and indices stream in coalesced, the gathered products land in
//    shared memory, then one thread per row folds its products in the exact
//    order the reference's NumPy code uses, so results are bit-identical:
//      forward  : p0 + pairwise(p1..)   (np.add.reduceat, matio.py:146-149)
//      transpose: ((0 + p0) + p1) + ... (np.add.at, matio.py:150-154)
//    Products are rounded before the add (no FMA contraction).
//  * long rows (> 2048 nnz, e.g. the Zipf head columns of config 4's A^T):
//    split into 8192-nnz chunks, one CTA each, fixed-order in-CTA tree then a
//    fix-up kernel summing the chunk partials in chunk order: deterministic,
//    not bit-identical to a serial sum.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <vector>

#include <stdlib.h>

#include "common.cuh"

namespace svdsb {

constexpr int kTileThreads = 256;
constexpr int kTileNnz = 2048;                    // 8 per thread
constexpr int kTileRows = 256;
constexpr int kLongChunk = 8192;                  // 32 per thread
constexpr int kPerThread = kTileNnz / kTileThreads;

struct CsrPart {
  int64_t rows = 0, cols = 0, nnz = 0;
  int *row_ptr = nullptr;   // rows+1
  int *col = nullptr;       // nnz
  double *val = nullptr;    // nnz
  // short-row tiles: [tile_r0[i], tile_r1[i])
  int ntile = 0;
  int *tile_r = nullptr;    // 2*ntile
  int4 *tile_info = nullptr;  // ntile x {r0, r1, nz0, nz1}
  // long rows, split in chunks
  int nlong = 0;
  int *long_row = nullptr;  // nlong
  int *long_cptr = nullptr; // nlong+1 : chunk range of each long row
  int nchunk = 0;
  int *chunk_nz = nullptr;  // 2*nchunk : [nz0, nz1)
  double *chunk_part = nullptr;  // nchunk * kMaxB partial sums
  std::vector<int> host_row_ptr;
  int maxlen = 0;             // longest row handled by the tiles
  // sliced ELL copy (slices of 32 rows, element j of row t of a slice at
  // sell_ptr[slice] + 32 j + t) for the b = 4 forward product; built on
  // first use
  int64_t nslice = 0;
  int64_t nsell = 0;            // rows in the sliced copy
  int *sell_perm = nullptr;     // transpose parts: sliced position -> row (rows sorted by length)
  int nmid = 0;                 // transpose parts: rows between kSellTMax and a tile's nonzeros
  int *mid_rows = nullptr;
  int64_t *sell_ptr = nullptr;  // nslice + 1
  int *sell_col = nullptr;
  double *sell_val = nullptr;
  uint8_t *sell_len = nullptr;  // forward copy: row length of each sliced position (0 past the end)
  bool sell_failed = false;     // the copy could not be built: CSR kernels (same bits)
  // hot-encoded column ids of the forward copy (csr_sell4s_kernel<.., 1>):
  // ~slot for the sell_nhot most referenced columns (listed in sell_hot)
  int *sell_colh = nullptr;
  int *sell_hot = nullptr;
  int sell_nhot = 0;
  unsigned *work_ctr = nullptr; // transpose parts: {next work item, warps done} of csr_sell4t_kernel
  // head tiles of the long rows (b = 4 transposed products, built on first
  // use): pieces of <= kHeadPiece nonzeros of one long row inside one
  // kHeadTile-row tile of the operand, listed tile by tile
  int nhtile = 0;
  int *htp = nullptr;           // nhtile + 1: piece range of each tile
  int4 *hpiece = nullptr;       // {k0, k1, output slot, -}
  int *hcptr = nullptr;         // nlong + 1: slot range of each long row (tile order)
  double *hpart = nullptr;      // slots x 4 partial sums
  bool head_failed = false;
};

constexpr int kMaxB = 64;   // largest block handled by one matvec call

}  // namespace svdsb

struct svdsb_csr {
  int device;
  svdsb::CsrPart a, at;
  bool has_t;
  // row-major staging for block products (2 <= b <= 4): packed input and
  // the inner product of the normal operator; grown on demand
  double *scratch[3] = {nullptr, nullptr, nullptr};
  size_t scratch_cap[3] = {0, 0, 0};
  // A^T split by row blocks of A (tall, scattered matrices): local column
  // ids, block k covers rows [atb_r0[k], atb_r0[k+1]) of A
  std::vector<svdsb::CsrPart> atb;
  std::vector<int64_t> atb_r0;
};

namespace svdsb {

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// NumPy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// DOUBLE_pairwise_sum) as used by np.add.reduceat for the tail of a segment.
__device__ double np_pairwise(const double *a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = dadd(r, a[i]);
    return r;
  } else if (n <= 128) {
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3];
    double r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
      r0 = dadd(r0, a[i + 0]); r1 = dadd(r1, a[i + 1]);
      r2 = dadd(r2, a[i + 2]); r3 = dadd(r3, a[i + 3]);
      r4 = dadd(r4, a[i + 4]); r5 = dadd(r5, a[i + 5]);
      r6 = dadd(r6, a[i + 6]); r7 = dadd(r7, a[i + 7]);
    }
    double res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
    for (; i < n; ++i) res = dadd(res, a[i]);
    return res;
  } else {
    int n2 = n / 2;
    n2 -= n2 % 8;
    return dadd(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
  }
}

// Out-of-line copy for the rare long tails (>= 8 terms) so the common fold
// stays register-light.
__device__ __noinline__ double np_pairwise_long(const double *a, int n) { return np_pairwise(a, n); }

// ORDER 0: forward (reduceat) ; ORDER 1: sequential (add.at).  SHORT: the
// caller guarantees len <= 8 (stencil-like matrices), which keeps the fold
// register-light.
template <int ORDER, bool SHORT = false>
__device__ __forceinline__ double fold_row(const double *p, int len) {
  if (ORDER == 0 && SHORT) {
    if (len == 0) return 0.0;
    double r = 0.0;
    for (int i = 1; i < len; ++i) r = dadd(r, p[i]);
    return len == 1 ? p[0] : dadd(p[0], r);
  }
  if (ORDER == 0) {
    if (len == 0) return 0.0;
    double s = p[0];
    if (len == 1) return s;
    if (len <= 8) {  // tail < 8 terms: numpy sums them left to right from 0
      double r = 0.0;
      for (int i = 1; i < len; ++i) r = dadd(r, p[i]);
      return dadd(s, r);
    }
    if (len <= 129) {  // tail of 8..128 terms: numpy's 8-accumulator block, inline
      const double *a = p + 1;
      const int n = len - 1;
      double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
      int i = 8;
      for (; i < n - (n % 8); i += 8) {
        r0 = dadd(r0, a[i + 0]); r1 = dadd(r1, a[i + 1]);
        r2 = dadd(r2, a[i + 2]); r3 = dadd(r3, a[i + 3]);
        r4 = dadd(r4, a[i + 4]); r5 = dadd(r5, a[i + 5]);
        r6 = dadd(r6, a[i + 6]); r7 = dadd(r7, a[i + 7]);
      }
      double res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
      for (; i < n; ++i) res = dadd(res, a[i]);
      return dadd(s, res);
    }
    return dadd(s, np_pairwise_long(p + 1, len - 1));
  } else {
    double s = 0.0;
    for (int i = 0; i < len; ++i) s = dadd(s, p[i]);
    return s;
  }
}

// Sequential fold continuing from a running value: a row split over column
// blocks of A^T (processed in ascending row order) keeps np.add.at's exact
// left-to-right order.
__device__ __forceinline__ double fold_row_from(double s, const double *p, int len) {
  for (int i = 0; i < len; ++i) s = dadd(s, p[i]);
  return s;
}

__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// The same for matrices that stream from HBM (config 3/4 scale): L2
// evict-first, so the gathered operand block keeps its L2 residency.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_ef(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_evict_first()));
  return v;
}
__device__ __forceinline__ int ld_ef(const int *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_evict_first()));
  return v;
}

// XROW: x is row-major with row stride b (one 8*b-byte gather per nonzero);
// otherwise column-major with leading dimension ldx.  YROW likewise for y.
template <int ORDER, int XROW, int YROW, int BMAX>
__global__ void __launch_bounds__(kTileThreads, 3)
csr_tile_kernel(const int *__restrict__ tile_r, const int *__restrict__ row_ptr,
                const int *__restrict__ col, const double *__restrict__ val,
                const double *__restrict__ x, int64_t ldx, double *__restrict__ y,
                int64_t ldy, int b) {
  __shared__ double prod[kTileNnz];
  __shared__ int rp[kTileRows + 1];
  const int t = threadIdx.x;
  const int r0 = tile_r[2 * blockIdx.x], r1 = tile_r[2 * blockIdx.x + 1];
  const int nrows = r1 - r0;
  for (int i = t; i <= nrows; i += kTileThreads) rp[i] = row_ptr[r0 + i];
  __syncthreads();
  const int nz0 = rp[0], nnz = rp[nrows] - nz0;
  double v[kPerThread];
  int c[kPerThread];
#pragma unroll
  for (int i = 0; i < kPerThread; ++i) {
    int k = t + i * kTileThreads;
    if (k < nnz) {
      v[i] = ld_stream(val + nz0 + k);
      c[i] = ld_stream(col + nz0 + k);
    } else {
      v[i] = 0.0;
      c[i] = 0;
    }
  }
  int my0 = 0, mylen = 0;
  if (t < nrows) {
    my0 = rp[t] - nz0;
    mylen = rp[t + 1] - rp[t];
  }
  if (XROW) {
    // gather whole x rows (b <= BMAX doubles) once per nonzero
    double xv[kPerThread][BMAX];
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      int k = t + i * kTileThreads;
#pragma unroll
      for (int cc = 0; cc < BMAX; ++cc) xv[i][cc] = (k < nnz && cc < b) ? __ldg(x + (int64_t)c[i] * b + cc) : 0.0;
    }
#pragma unroll
    for (int cc = 0; cc < BMAX; ++cc) {
      if (cc >= b) break;
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        int k = t + i * kTileThreads;
        if (k < nnz) prod[k] = dmul(v[i], xv[i][cc]);
      }
      __syncthreads();
      if (t < nrows) {
        double s = fold_row<ORDER>(prod + my0, mylen);
        if (YROW)
          y[(int64_t)(r0 + t) * b + cc] = s;
        else
          y[(int64_t)(r0 + t) + cc * ldy] = s;
      }
      __syncthreads();
    }
  } else {
    for (int cc = 0; cc < b; ++cc) {
      const double *xc = x + cc * ldx;
      // all gathers issued before the first use (c[i] = 0 past the tile)
      double xv[kPerThread];
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) xv[i] = __ldg(xc + c[i]);
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        int k = t + i * kTileThreads;
        if (k < nnz) prod[k] = dmul(v[i], xv[i]);
      }
      __syncthreads();
      if (t < nrows) {
        double s = fold_row<ORDER>(prod + my0, mylen);
        if (YROW)
          y[(int64_t)(r0 + t) * b + cc] = s;
        else
          y[(int64_t)(r0 + t) + cc * ldy] = s;
      }
      __syncthreads();
    }
  }
}

// Persistent, software-pipelined b = 1 variant: while a CTA gathers and
// folds tile t, the value / index / row-pointer loads of its next tile are
// already in flight; products are double-buffered in shared memory so one
// barrier per tile suffices.  Same per-row summation order as above.
// The tile loop itself, shared with the fused normal-operator kernel.
// CG: gather x with ld.global.cg (L2 only) -- required when x was written
// earlier in the same kernel by other CTAs; prewait: prefetch the first
// tile's immutable matrix data, then wait for the producer of x.
template <int ORDER, bool SHORT, bool CG>
__device__ __forceinline__ void pipe_tiles(int ntile, const int4 *__restrict__ info, const int *__restrict__ row_ptr,
                                           const int *__restrict__ col, const double *__restrict__ val,
                                           const double *x, double *y, int accumulate,
                                           double (&prod)[2][kTileNnz], int (&rps)[2][kTileRows + 1],
                                           bool prewait) {
  const int t = threadIdx.x;
  int tile = blockIdx.x;
  if (tile >= ntile) {
    if (prewait) pdl_wait();
    return;
  }
  // stage A: loads for `tile`
  int4 cur = info[tile];
  double v[kPerThread];
  int c[kPerThread];
  int rpa, rpb;
  auto issue = [&](const int4 &ti, double (&vv)[kPerThread], int (&cc)[kPerThread], int &ra, int &rb) {
    const int nnz = ti.w - ti.z, nrows = ti.y - ti.x;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      int k = t + i * kTileThreads;
      if (k < nnz) {
        vv[i] = ld_stream(val + ti.z + k);
        cc[i] = ld_stream(col + ti.z + k);
      } else {
        vv[i] = 0.0;
        cc[i] = 0;
      }
    }
    ra = (t <= nrows) ? __ldg(row_ptr + ti.x + t) : 0;
    rb = (t == 0 && nrows >= kTileThreads) ? __ldg(row_ptr + ti.x + kTileThreads) : 0;
  };
  issue(cur, v, c, rpa, rpb);
  if (prewait) pdl_wait();  // matrix data is immutable after assembly; x / y are not
  int buf = 0;
  while (true) {
    const int next_tile = tile + gridDim.x;
    int4 nxt = make_int4(0, 0, 0, 0);
    double vn[kPerThread];
    int cn[kPerThread];
    int rna = 0, rnb = 0;
    if (next_tile < ntile) {
      nxt = info[next_tile];
      issue(nxt, vn, cn, rna, rnb);
    }
    // gather + products of the current tile
    const int nnz = cur.w - cur.z, nrows = cur.y - cur.x;
    // all gathers issued before the first use (c[i] = 0 past the tile), so
    // a thread keeps kPerThread loads in flight instead of one
    double xg[kPerThread];
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) xg[i] = CG ? __ldcg(x + c[i]) : __ldg(x + c[i]);
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      int k = t + i * kTileThreads;
      if (k < nnz) prod[buf][k] = dmul(v[i], xg[i]);
    }
    if (t <= nrows) rps[buf][t] = rpa;
    if (t == 0 && nrows >= kTileThreads) rps[buf][kTileThreads] = rpb;
    __syncthreads();
    if (t < nrows) {
      const int s0 = rps[buf][t] - cur.z;
      const int len = rps[buf][t + 1] - rps[buf][t];
      y[cur.x + t] = accumulate ? fold_row_from(y[cur.x + t], prod[buf] + s0, len)
                                : fold_row<ORDER, SHORT>(prod[buf] + s0, len);
    }
    if (next_tile >= ntile) break;
    tile = next_tile;
    cur = nxt;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      v[i] = vn[i];
      c[i] = cn[i];
    }
    rpa = rna;
    rpb = rnb;
    buf ^= 1;
  }
}

template <int ORDER, bool SHORT>
__global__ void __launch_bounds__(kTileThreads, 3)
csr_tile_pipe_kernel(int ntile, const int4 *__restrict__ info, const int *__restrict__ row_ptr,
                     const int *__restrict__ col, const double *__restrict__ val, const double *__restrict__ x,
                     double *__restrict__ y, int accumulate) {
  __shared__ double prod[2][kTileNnz];
  __shared__ int rps[2][kTileRows + 1];
  pipe_tiles<ORDER, SHORT, false>(ntile, info, row_ptr, col, val, x, y, accumulate, prod, rps, true);
  pdl_trigger();
}

// Pipelined variant for row-major block operands (2 <= b <= 4): one x-row
// gather per nonzero, products of all b columns staged in shared memory,
// then (row, column) pairs folded in parallel, each column in the
// reference's order.
template <int ORDER, int YROW>
__global__ void __launch_bounds__(kTileThreads, 2)
csr_tile_pipe_rows_kernel(int ntile, const int4 *__restrict__ info, const int *__restrict__ row_ptr,
                          const int *__restrict__ col, const double *__restrict__ val,
                          const double *__restrict__ x, double *__restrict__ y, int64_t ldy, int b,
                          int accumulate) {
  extern __shared__ double dsm[];
  double *prod = dsm;                                        // 4 x kTileNnz
  int *rps = reinterpret_cast<int *>(dsm + 4 * kTileNnz);     // kTileRows + 1
  const int t = threadIdx.x;
  int tile = blockIdx.x;
  if (tile >= ntile) return;
  int4 cur = info[tile];
  double v[kPerThread];
  int c[kPerThread];
  int rpa, rpb;
  auto issue = [&](const int4 &ti, double (&vv)[kPerThread], int (&cc)[kPerThread], int &ra, int &rb) {
    const int nnz = ti.w - ti.z, nrows = ti.y - ti.x;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      int k = t + i * kTileThreads;
      if (k < nnz) {
        vv[i] = ld_stream(val + ti.z + k);
        cc[i] = ld_stream(col + ti.z + k);
      } else {
        vv[i] = 0.0;
        cc[i] = 0;
      }
    }
    ra = (t <= nrows) ? __ldg(row_ptr + ti.x + t) : 0;
    rb = (t == 0 && nrows >= kTileThreads) ? __ldg(row_ptr + ti.x + kTileThreads) : 0;
  };
  issue(cur, v, c, rpa, rpb);
  pdl_wait();
  while (true) {
    const int next_tile = tile + gridDim.x;
    int4 nxt = make_int4(0, 0, 0, 0);
    double vn[kPerThread];
    int cn[kPerThread];
    int rna = 0, rnb = 0;
    if (next_tile < ntile) {
      nxt = info[next_tile];
      issue(nxt, vn, cn, rna, rnb);
    }
    const int nnz = cur.w - cur.z, nrows = cur.y - cur.x;
    if (b == 4) {
      // one 256-bit gather per nonzero (rows are 32-byte aligned), issued in
      // groups of four before their products (c[i] = 0 past the tile)
#pragma unroll
      for (int h = 0; h < kPerThread; h += 4) {
        double xg[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double *xr = x + (int64_t)c[h + i] * 4;
          asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
              : "=d"(xg[i][0]), "=d"(xg[i][1]), "=d"(xg[i][2]), "=d"(xg[i][3]) : "l"(xr));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = t + (h + i) * kTileThreads;
          if (k < nnz) {
            prod[k] = dmul(v[h + i], xg[i][0]);
            prod[kTileNnz + k] = dmul(v[h + i], xg[i][1]);
            prod[2 * kTileNnz + k] = dmul(v[h + i], xg[i][2]);
            prod[3 * kTileNnz + k] = dmul(v[h + i], xg[i][3]);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      int k = t + i * kTileThreads;
      if (b != 4 && k < nnz) {
        const double *xr = x + (int64_t)c[i] * b;
        if (b == 2) {
          double2 xv = __ldg(reinterpret_cast<const double2 *>(xr));
          prod[k] = dmul(v[i], xv.x);
          prod[kTileNnz + k] = dmul(v[i], xv.y);
        } else {
          prod[k] = dmul(v[i], __ldg(xr));
          prod[kTileNnz + k] = dmul(v[i], __ldg(xr + 1));
          prod[2 * kTileNnz + k] = dmul(v[i], __ldg(xr + 2));
        }
      }
    }
    if (t <= nrows) rps[t] = rpa;
    if (t == 0 && nrows >= kTileThreads) rps[kTileThreads] = rpb;
    __syncthreads();
    for (int q = t; q < nrows * b; q += kTileThreads) {
      const int row = q % nrows, cc = q / nrows;
      const int s0 = rps[row] - cur.z;
      const int len = rps[row + 1] - rps[row];
      double *yp = YROW ? y + (int64_t)(cur.x + row) * b + cc : y + (int64_t)(cur.x + row) + cc * ldy;
      *yp = accumulate ? fold_row_from(*yp, prod + cc * kTileNnz + s0, len)
                       : fold_row<ORDER>(prod + cc * kTileNnz + s0, len);
    }
    if (next_tile >= ntile) break;
    __syncthreads();  // prod / rps are single-buffered
    tile = next_tile;
    cur = nxt;
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
      v[i] = vn[i];
      c[i] = cn[i];
    }
    rpa = rna;
    rpb = rnb;
  }
}

// Forward b = 4 product for matrices whose rows are all short (<= 129 nnz,
// e.g. config 4's A with 7-20 per row): one thread per row, no shared
// memory and no CTA barrier.  The row's x-rows are gathered four at a time
// (one 256-bit load each) and folded on the fly into the exact order of
// fold_row<0> -- p0 + numpy pairwise(rest): the first 8 tail products seed 8
// accumulators, whole blocks of 8 follow, the remainder is added to the
// tree sum -- for the four columns as independent chains.
// One 32-byte x row (256-bit load, L2 evict-last: the gathered block stays
// resident while the matrix streams past it).
__device__ __forceinline__ void gather4(const double *x, int c, double (&o)[4]) {
  unsigned long long a, b, d, e;
  asm("ld.global.nc.L2::evict_last.v4.b64 {%0, %1, %2, %3}, [%4];"
      : "=l"(a), "=l"(b), "=l"(d), "=l"(e) : "l"(x + (int64_t)c * 4));
  o[0] = __longlong_as_double(a);
  o[1] = __longlong_as_double(b);
  o[2] = __longlong_as_double(d);
  o[3] = __longlong_as_double(e);
}

// One row's four products in the exact fold_row<0> order; `src` supplies
// the row's values / column ids (global memory or a warp's shared stage).
template <typename Src>
__device__ __forceinline__ void row4_fold(const Src &src, int k0, int k1, const double *__restrict__ x,
                                          double (&out)[4]) {
  const int n = k1 - k0 - 1;  // tail length
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = 0.0;
  if (n < 0) return;
  double p0[4];
  {
    double xv[4];
    gather4(x, src.c(k0), xv);
    const double v = src.v(k0);
#pragma unroll
    for (int c = 0; c < 4; ++c) p0[c] = dmul(v, xv[c]);
  }
  const int t0 = k0 + 1;  // first tail element
  if (n < 8) {
    // numpy: tail < 8 summed left to right from 0
    double r[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i0 = 0; i0 < n; i0 += 4) {
      double xv[4][4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = t0 + min(i0 + u, n - 1);
        vv[u] = src.v(k);
        gather4(x, src.c(k), xv[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u < n) {
#pragma unroll
          for (int c = 0; c < 4; ++c) r[c] = dadd(r[c], dmul(vv[u], xv[u][c]));
        }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = n == 0 ? p0[c] : dadd(p0[c], r[c]);
    return;
  }
  double acc[4][8];
  const int nb = n - (n % 8);
  // block 0 seeds the accumulators, blocks 8.. add in order
  for (int b0 = 0; b0 < nb; b0 += 8) {
#pragma unroll
    for (int h = 0; h < 8; h += 4) {
      double xv[4][4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = t0 + b0 + h + u;
        vv[u] = src.v(k);
        gather4(x, src.c(k), xv[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double pr = dmul(vv[u], xv[u][c]);
          acc[c][h + u] = b0 == 0 ? pr : dadd(acc[c][h + u], pr);
        }
    }
  }
  double res[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double *a = acc[c];
    res[c] = dadd(dadd(dadd(a[0], a[1]), dadd(a[2], a[3])), dadd(dadd(a[4], a[5]), dadd(a[6], a[7])));
  }
  for (int i0 = nb; i0 < n; i0 += 4) {
    double xv[4][4], vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = t0 + min(i0 + u, n - 1);
      vv[u] = src.v(k);
      gather4(x, src.c(k), xv[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u < n) {
#pragma unroll
        for (int c = 0; c < 4; ++c) res[c] = dadd(res[c], dmul(vv[u], xv[u][c]));
      }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = dadd(p0[c], res[c]);
}

template <int YROW>
__device__ __forceinline__ void store_row4(double *__restrict__ y, int64_t ldy, int64_t row, const double (&out)[4]) {
  if (YROW) {
    double *yp = y + row * 4;
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" :: "l"(yp), "d"(out[0]), "d"(out[1]), "d"(out[2]),
                 "d"(out[3]) : "memory");
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) y[row + c * ldy] = out[c];
  }
}

struct GlobalRowSrc {
  const double *__restrict__ val;
  const int *__restrict__ col;
  __device__ __forceinline__ double v(int k) const { return ld_stream(val + k); }
  __device__ __forceinline__ int c(int k) const { return ld_stream(col + k); }
};

// k indexes the global nonzero; the stage holds [base, base + cap)
struct StagedRowSrc {
  const double *val;
  const int *col;
  int base;
  __device__ __forceinline__ double v(int k) const { return val[k - base]; }
  __device__ __forceinline__ int c(int k) const { return col[k - base]; }
};

template <int YROW>
__global__ void __launch_bounds__(kTileThreads, 2)
csr_rowlane4_kernel(int64_t nrows, const int *__restrict__ row_ptr, const int *__restrict__ col,
                    const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y,
                    int64_t ldy) {
  pdl_wait();
  const GlobalRowSrc src{val, col};
  for (int64_t row = blockIdx.x * (int64_t)kTileThreads + threadIdx.x; row < nrows;
       row += (int64_t)gridDim.x * kTileThreads) {
    double out[4];
    row4_fold(src, __ldg(row_ptr + row), __ldg(row_ptr + row + 1), x, out);
    store_row4<YROW>(y, ldy, row, out);
  }
  pdl_trigger();
}

// Warp-staged variant: a warp takes 32 consecutive rows, copies their
// values / column ids global -> shared with coalesced loads (instead of
// each thread walking its own row, which touches 32 sectors per warp load
// and fetches every sector from L2 up to four times), then each lane folds
// its row from the stage exactly as csr_rowlane4_kernel does.  Row groups
// longer than the stage fall back to the global walk.
constexpr int kWarpStage = 768;  // nonzeros per warp stage (9 KB)

template <int YROW>
__global__ void __launch_bounds__(kTileThreads, 2)
csr_warprows4_kernel(int64_t nrows, const int *__restrict__ row_ptr, const int *__restrict__ col,
                     const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y,
                     int64_t ldy) {
  extern __shared__ __align__(16) unsigned char wr_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double *sv = reinterpret_cast<double *>(wr_smem) + w * kWarpStage;
  int *sc = reinterpret_cast<int *>(wr_smem + sizeof(double) * kWarpStage * (kTileThreads / 32)) + w * kWarpStage;
  const int64_t ngroups = (nrows + 31) >> 5;
  const int64_t wstride = (int64_t)gridDim.x * (kTileThreads / 32);
  pdl_wait();
  for (int64_t grp = blockIdx.x * (int64_t)(kTileThreads / 32) + w; grp < ngroups; grp += wstride) {
    const int64_t row = (grp << 5) + lane;
    const int64_t rcl = row < nrows ? row : nrows;
    const int k0 = __ldg(row_ptr + rcl);
    int k1 = __shfl_down_sync(0xffffffffu, k0, 1);
    if (lane == 31) k1 = __ldg(row_ptr + (row + 1 < nrows ? row + 1 : nrows));
    const int s = __shfl_sync(0xffffffffu, k0, 0);
    const int e = __shfl_sync(0xffffffffu, k1, 31);
    double out[4];
    // a group longer than the stage is read straight from global memory
    // (same fold; generic loads)
    const bool staged = e - s <= kWarpStage;
    if (staged) {
      const int len = e - s;
#pragma unroll 4
      for (int k = lane; k < len; k += 32) {
        sv[k] = ld_stream(val + s + k);
        sc[k] = ld_stream(col + s + k);
      }
    }
    __syncwarp();
    const StagedRowSrc src{staged ? sv : val, staged ? sc : col, staged ? s : 0};
    if (row < nrows) {
      row4_fold(src, k0, k1, x, out);
      store_row4<YROW>(y, ldy, row, out);
    }
    __syncwarp();
  }
  pdl_trigger();
}

// Quad variant: four lanes per row, one block column each, eight rows per
// warp.  The four lanes of a row gather the same 32-byte x row (one sector
// per row per warp load) and each folds one column in the fold_row<0>
// order with scalar registers, so the kernel runs at high occupancy and
// keeps eight gathers in flight per lane.  Values / column ids of the
// warp's eight rows are staged through shared memory with coalesced loads.
constexpr int kQuadStage = 256;  // nonzeros per warp stage (8 rows)

template <int YROW>
__global__ void __launch_bounds__(kTileThreads, 3)
csr_quad4_kernel(int64_t nrows, const int *__restrict__ row_ptr, const int *__restrict__ col,
                 const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y,
                 int64_t ldy) {
  __shared__ double qv[kTileThreads / 32][kQuadStage];
  __shared__ int qc[kTileThreads / 32][kQuadStage];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rr = lane >> 2, cc = lane & 3;
  const int64_t ngroups = (nrows + 7) >> 3;
  const int64_t wstride = (int64_t)gridDim.x * (kTileThreads / 32);
  const double *xc = x + cc;
  pdl_wait();
  for (int64_t grp = blockIdx.x * (int64_t)(kTileThreads / 32) + w; grp < ngroups; grp += wstride) {
    const int64_t r0 = grp << 3;
    int rpv = 0;
    if (lane <= 8) rpv = __ldg(row_ptr + (r0 + lane < nrows ? r0 + lane : nrows));
    const int k0 = __shfl_sync(0xffffffffu, rpv, rr);
    const int k1 = __shfl_sync(0xffffffffu, rpv, rr + 1);
    const int s = __shfl_sync(0xffffffffu, rpv, 0);
    const int e = __shfl_sync(0xffffffffu, rpv, 8);
    const bool staged = e - s <= kQuadStage;
    if (staged) {
      const int len = e - s;
#pragma unroll 4
      for (int k = lane; k < len; k += 32) {
        qv[w][k] = ld_stream(val + s + k);
        qc[w][k] = ld_stream(col + s + k);
      }
    }
    __syncwarp();
    // generic pointers: the stage, or global memory for an oversized group
    const double *vp = staged ? &qv[w][0] : val + s;
    const int *cp = staged ? &qc[w][0] : col + s;
    const int a0 = k0 - s;           // row start within the group
    const int n = k1 - k0 - 1;       // tail length
    double out = 0.0;
    if (n >= 0) {
      const double p0 = dmul(vp[a0], __ldg(xc + (int64_t)cp[a0] * 4));
      const int t0 = a0 + 1;
      double res;
      int i = 0;
      if (n < 8) {
        res = 0.0;
      } else {
        double acc[8];
        const int nb = n - (n % 8);
        for (; i < nb; i += 8) {
          double xg[8], vv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            vv[j] = vp[t0 + i + j];
            xg[j] = __ldg(xc + (int64_t)cp[t0 + i + j] * 4);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double pr = dmul(vv[j], xg[j]);
            acc[j] = i == 0 ? pr : dadd(acc[j], pr);
          }
        }
        res = dadd(dadd(dadd(acc[0], acc[1]), dadd(acc[2], acc[3])), dadd(dadd(acc[4], acc[5]), dadd(acc[6], acc[7])));
      }
      // remainder (< 8 terms) left to right -- the whole tail when n < 8
      if (i < n) {
        double xg[7], vv[7];
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          const int k = t0 + min(i + j, n - 1);
          vv[j] = vp[k];
          xg[j] = __ldg(xc + (int64_t)cp[k] * 4);
        }
#pragma unroll
        for (int j = 0; j < 7; ++j)
          if (i + j < n) res = dadd(res, dmul(vv[j], xg[j]));
      }
      out = n == 0 ? p0 : dadd(p0, res);
    }
    const int64_t row = r0 + rr;
    if (row < nrows) {
      if (YROW)
        y[row * 4 + cc] = out;
      else
        y[row + cc * ldy] = out;
    }
    __syncwarp();
  }
  pdl_trigger();
}

// Sliced ELL (SELL-32) forward product for b = 4: lane t of a warp owns
// row t of a 32-row slice and reads element j of its row at
// base + 32 j + t, so every value / index load of the warp is one
// contiguous 256 / 128-byte segment -- no shared-memory staging and no
// bank conflicts.  The fold is row4_fold's, so results are bit-identical
// to the CSR kernels.
struct SellRowSrc {
  const double *__restrict__ val;
  const int *__restrict__ col;
  int64_t base;  // slice base + t - 32 k0 (element k sits at base + 32 k)
  __device__ __forceinline__ double v(int k) const { return ld_ef(val + base + 32 * (int64_t)k); }
  __device__ __forceinline__ int c(int k) const { return ld_ef(col + base + 32 * (int64_t)k); }
};

template <int YROW>
__global__ void __launch_bounds__(kTileThreads, 2)
csr_sell4_kernel(int64_t nrows, int64_t nslice, const int *__restrict__ row_ptr, const int64_t *__restrict__ sell_ptr,
                 const int *__restrict__ col, const double *__restrict__ val, const double *__restrict__ x,
                 double *__restrict__ y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (kTileThreads / 32);
  pdl_wait();
  for (int64_t sl = blockIdx.x * (int64_t)(kTileThreads / 32) + (threadIdx.x >> 5); sl < nslice; sl += wstride) {
    const int64_t row = (sl << 5) + lane;
    if (row < nrows) {
      const int k0 = __ldg(row_ptr + row), k1 = __ldg(row_ptr + row + 1);
      const SellRowSrc src{val, col, __ldg(sell_ptr + sl) + lane - 32 * (int64_t)k0};
      double out[4];
      row4_fold(src, k0, k1, x, out);
      store_row4<YROW>(y, ldy, row, out);
    }
  }
  pdl_trigger();
}

// Sliced-ELL forward b = 4 for rows of at most kSellW nonzeros: a lane
// issues every value / index load of its row at once (one DRAM round trip
// per row instead of one per group of four), then folds the four columns
// as two pairs (16-byte gathers; the same L1 wavefronts as one 32-byte
// gather) in the fold_row<0> order: p0 + (tail < 8 ? left-to-right :
// 8-accumulator blocks, tree, remainder).  Bit-identical to row4_fold.
constexpr int kSellW = 20;

__device__ __forceinline__ double2 ldg2c(const double *p) {
  double2 v;
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 pmul(double v, double2 x) { return make_double2(dmul(v, x.x), dmul(v, x.y)); }
__device__ __forceinline__ double2 padd(double2 a, double2 b) { return make_double2(dadd(a.x, b.x), dadd(a.y, b.y)); }

__device__ __forceinline__ double2 sell_pair_fold(const int (&cj)[kSellW], const double (&vj)[kSellW], int len,
                                                  const double *__restrict__ xc) {
  if (len == 0) return make_double2(0.0, 0.0);
  const int n = len - 1;
  const double2 p0 = pmul(vj[0], ldg2c(xc + (int64_t)cj[0] * 4));
  if (n < 8) {
    double2 g[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) g[u] = ldg2c(xc + (int64_t)cj[1 + u] * 4);  // cj = 0 past the row
    double2 r = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (1 + u <= n) r = padd(r, pmul(vj[1 + u], g[u]));
    return n == 0 ? p0 : padd(p0, r);
  }
  double2 acc[8], g[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) g[u] = ldg2c(xc + (int64_t)cj[1 + u] * 4);
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = pmul(vj[1 + u], g[u]);
  const int nb = n - (n % 8);  // 8 or 16
#pragma unroll
  for (int u = 0; u < 8; ++u) g[u] = ldg2c(xc + (int64_t)cj[9 + u] * 4);
  if (nb == 16) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = padd(acc[u], pmul(vj[9 + u], g[u]));
  }
  double2 res = padd(padd(padd(acc[0], acc[1]), padd(acc[2], acc[3])), padd(padd(acc[4], acc[5]), padd(acc[6], acc[7])));
  if (nb == 8) {
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (9 + u <= n) res = padd(res, pmul(vj[9 + u], g[u]));
  } else {
#pragma unroll
    for (int u = 0; u < kSellW - 17; ++u) g[u] = ldg2c(xc + (int64_t)cj[17 + u] * 4);
#pragma unroll
    for (int u = 0; u < kSellW - 17; ++u)
      if (17 + u <= n) res = padd(res, pmul(vj[17 + u], g[u]));
  }
  return padd(p0, res);
}

template <int YROW>
__global__ void __launch_bounds__(kTileThreads, 2)
csr_sell4w_kernel(int64_t nrows, int64_t nslice, const int *__restrict__ row_ptr, const int64_t *__restrict__ sell_ptr,
                  const int *__restrict__ col, const double *__restrict__ val, const double *__restrict__ x,
                  double *__restrict__ y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (kTileThreads / 32);
  pdl_wait();
  for (int64_t sl = blockIdx.x * (int64_t)(kTileThreads / 32) + (threadIdx.x >> 5); sl < nslice; sl += wstride) {
    const int64_t row = (sl << 5) + lane;
    if (row < nrows) {
      const int len = __ldg(row_ptr + row + 1) - __ldg(row_ptr + row);
      const int64_t base = __ldg(sell_ptr + sl) + lane;
      int cj[kSellW];
      double vj[kSellW];
#pragma unroll
      for (int j = 0; j < kSellW; ++j) {
        cj[j] = j < len ? ld_stream(col + base + 32 * j) : 0;
        vj[j] = j < len ? ld_stream(val + base + 32 * j) : 0.0;
      }
      const double2 lo = sell_pair_fold(cj, vj, len, x);
      const double2 hi = sell_pair_fold(cj, vj, len, x + 2);
      const double out[4] = {lo.x, lo.y, hi.x, hi.y};
      store_row4<YROW>(y, ldy, row, out);
    }
  }
  pdl_trigger();
}

// TMA-staged sliced-ELL forward product for b = 4 (rows of at most
// kSell4sW nonzeros: config 4's A).  One persistent CTA of kS4Warps warps
// per SM; each warp owns every kS4Warps*gridDim.x-th slice and streams its
// slices through a private two-stage shared-memory ring filled by
// cp.async.bulk (values, column ids and the slice's row lengths; L2
// evict-first), so no lane ever waits on DRAM for its indices: the only
// latency left in a row is the x gathers, issued eight (plus p0) at a time
// from indices already on chip.  The fold is row4_fold's order, so the
// result is bit-identical to the other b = 4 kernels.
constexpr int kSell4sW = 20;                  // widest slice staged
constexpr int kS4Warps = 12;                  // warps per CTA (1 CTA / SM)
constexpr int kS4Stage = 32 * kSell4sW * 12 + 32 + 96;   // vals + cols + lens, padded to 128 B
static_assert(kS4Stage % 128 == 0, "stage alignment");
constexpr size_t kS4Smem = (size_t)kS4Warps * 2 * kS4Stage;
constexpr int kS4Hot = 1280;                  // operand rows kept in shared memory (hot variant)
constexpr size_t kS4HotBytes = (size_t)kS4Hot * 32;
static_assert(kS4Smem + kS4HotBytes + 256 <= 232448, "hot rows + ring exceed the 227 KB of a CTA");

// value sources of s4_fold: element k of this lane's row
struct S4SmemVals {
  const double *p;  // stage + lane
  __device__ __forceinline__ double v(int k) const { return p[32 * k]; }
};
struct S4GlobalVals {
  const double *p;  // sval + slice start + lane
  __device__ __forceinline__ double v(int k) const { return ld_ef(p + 32 * k); }
};

// gather sources of s4_fold: the operand row of column id c
struct S4GlobalX {
  const double *x;
  __device__ __forceinline__ void load(int c, double (&o)[4]) const { gather4(x, c, o); }
};
// hot rows (ids < 0: ~slot) from the CTA's shared copy, the rest from global
// memory: a warp-wide gather of 32 scattered rows costs the L1 one wavefront
// per distinct 128-byte line, a shared-memory read 8 per 32 rows
struct S4HotX {
  const double *x;
  const double *xs;   // kS4Hot x 4 doubles in shared memory
  __device__ __forceinline__ void load(int c, double (&o)[4]) const {
    if (c < 0) {
      const double2 a = *reinterpret_cast<const double2 *>(xs + 4 * (~c));
      const double2 b = *reinterpret_cast<const double2 *>(xs + 4 * (~c) + 2);
      o[0] = a.x;
      o[1] = a.y;
      o[2] = b.x;
      o[3] = b.y;
    } else {
      gather4(x, c, o);
    }
  }
};

template <typename VS, typename GX>
__device__ __forceinline__ void s4_fold(const VS sv, const int *__restrict__ sc, int lane, int len,
                                        const GX x, double (&out)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = 0.0;
  if (len == 0) return;
  const int n = len - 1;  // tail length
  double p0[4], xg[8][4];
  {
    double g0[4];
    x.load(sc[lane], g0);
#pragma unroll
    for (int u = 0; u < 8; ++u) x.load(sc[(n == 0 ? 0 : 1 + min(u, n - 1)) * 32 + lane], xg[u]);
    const double v0 = sv.v(0);
#pragma unroll
    for (int c = 0; c < 4; ++c) p0[c] = dmul(v0, g0[c]);
  }
  if (n < 8) {
    double r[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (u < n) {
        const double vu = sv.v(1 + u);
#pragma unroll
        for (int c = 0; c < 4; ++c) r[c] = dadd(r[c], dmul(vu, xg[u][c]));
      }
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = n == 0 ? p0[c] : dadd(p0[c], r[c]);
    return;
  }
  double acc[4][8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double vu = sv.v(1 + u);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c][u] = dmul(vu, xg[u][c]);
  }
  const int nb = n - (n % 8);
  for (int b0 = 8; b0 < nb; b0 += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x.load(sc[(1 + b0 + u) * 32 + lane], xg[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double vu = sv.v(1 + b0 + u);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c][u] = dadd(acc[c][u], dmul(vu, xg[u][c]));
    }
  }
  double res[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double *a = acc[c];
    res[c] = dadd(dadd(dadd(a[0], a[1]), dadd(a[2], a[3])), dadd(dadd(a[4], a[5]), dadd(a[6], a[7])));
  }
  if (nb < n) {
#pragma unroll
    for (int u = 0; u < 7; ++u) x.load(sc[(1 + nb + min(u, n - nb - 1)) * 32 + lane], xg[u]);
#pragma unroll
    for (int u = 0; u < 7; ++u)
      if (nb + u < n) {
        const double vu = sv.v(1 + nb + u);
#pragma unroll
        for (int c = 0; c < 4; ++c) res[c] = dadd(res[c], dmul(vu, xg[u][c]));
      }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = dadd(p0[c], res[c]);
}

// HOT = 1: the column ids are the hot-encoded copy (sell_colh: ~slot for
// the part's kS4Hot most referenced columns) and the CTA first copies those
// operand rows into shared memory.  Config 4's Zipf columns: 1280 rows
// serve two thirds of the gathers.  Same values, same fold: bit-identical.
// Measured SLOWER on config 4 (992 vs 820 us): the kernel is bound by L1
// wavefronts (one per distinct 128-byte line of a gather), config 4's hot
// columns are adjacent ids that already share lines, and the two LDS.128 of
// a hot row cost as many wavefronts as they save while the larger carve-out
// shrinks L1.  Opt-in (svdsb_tune_set key 12 = 1) for matrices whose hot
// columns are scattered.
template <int YROW, int HOT>
__global__ void __launch_bounds__(kS4Warps * 32, 1)
csr_sell4s_kernel(int64_t nrows, int64_t nslice, const int64_t *__restrict__ sell_ptr, const int *__restrict__ scol,
                  const double *__restrict__ sval, const uint8_t *__restrict__ slen, const double *__restrict__ x,
                  double *__restrict__ y, int64_t ldy, const int *__restrict__ hot_cols, int nhot) {
  extern __shared__ __align__(128) unsigned char s4_smem[];
  __shared__ __align__(8) uint64_t bar[kS4Warps][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char *ring = s4_smem + (HOT ? kS4HotBytes : 0) + (size_t)w * 2 * kS4Stage;
  double *xs = reinterpret_cast<double *>(s4_smem);
  const int64_t gw = (int64_t)blockIdx.x * kS4Warps + w, nw = (int64_t)gridDim.x * kS4Warps;
  if (lane == 0) {
    mbar_init(&bar[w][0], 1);
    mbar_init(&bar[w][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t policy = 0;
  if (lane == 0) policy = evict_first_policy();
  // lane 0: slice sl (entries [e0, e1)) into stage k (values, column ids,
  // lengths; one mbarrier).  The slice pointers are loaded one issue ahead
  // so lane 0 never stalls the warp on them.
  auto issue = [&](int64_t sl, int k, int64_t e0, int64_t e1) {
    const int wd = (int)((e1 - e0) >> 5);
    unsigned char *st = ring + (size_t)k * kS4Stage;
    mbar_expect_tx(&bar[w][k], 32u * wd * 12u + 32u);
    if (wd > 0) {
      bulk_g2s(st, sval + e0, 256u * wd, &bar[w][k], policy);
      bulk_g2s(st + 32 * kSell4sW * 8, scol + e0, 128u * wd, &bar[w][k], policy);
    }
    bulk_g2s(st + 32 * kSell4sW * 12, slen + 32 * sl, 32u, &bar[w][k], policy);
  };
  // the matrix is immutable: start streaming before the producer of x ends
  int64_t pe0 = 0, pe1 = 0;   // pointers of slice gw + 2 nw (the next to issue)
  if (lane == 0) {
    if (gw < nslice) issue(gw, 0, __ldg(sell_ptr + gw), __ldg(sell_ptr + gw + 1));
    if (gw + nw < nslice) issue(gw + nw, 1, __ldg(sell_ptr + gw + nw), __ldg(sell_ptr + gw + nw + 1));
    if (gw + 2 * nw < nslice) {
      pe0 = __ldg(sell_ptr + gw + 2 * nw);
      pe1 = __ldg(sell_ptr + gw + 2 * nw + 1);
    }
  }
  pdl_wait();
  if (HOT) {
    for (int s = threadIdx.x; s < nhot; s += kS4Warps * 32) {
      double r[4];
      gather4(x, __ldg(hot_cols + s), r);
      *reinterpret_cast<double2 *>(xs + 4 * s) = make_double2(r[0], r[1]);
      *reinterpret_cast<double2 *>(xs + 4 * s + 2) = make_double2(r[2], r[3]);
    }
    __syncthreads();
  }
  int k = 0;
  unsigned phase = 0;
  for (int64_t sl = gw; sl < nslice; sl += nw) {
    mbar_wait(&bar[w][k], phase);
    const unsigned char *st = ring + (size_t)k * kS4Stage;
    const double *sv = reinterpret_cast<const double *>(st);
    const int *sc = reinterpret_cast<const int *>(st + 32 * kSell4sW * 8);
    const int len = st[32 * kSell4sW * 12 + lane];
    const int64_t row = (sl << 5) + lane;
    double out[4];
    if (HOT)
      s4_fold(S4SmemVals{sv + lane}, sc, lane, len, S4HotX{x, xs}, out);
    else
      s4_fold(S4SmemVals{sv + lane}, sc, lane, len, S4GlobalX{x}, out);
    if (row < nrows) store_row4<YROW>(y, ldy, row, out);
    __syncwarp();
    if (lane == 0 && sl + 2 * nw < nslice) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(sl + 2 * nw, k, pe0, pe1);
      if (sl + 3 * nw < nslice) {
        pe0 = __ldg(sell_ptr + sl + 3 * nw);
        pe1 = __ldg(sell_ptr + sl + 3 * nw + 1);
      }
    }
    if (++k == 2) {
      k = 0;
      phase ^= 1u;
    }
  }
  pdl_trigger();
}

// Variant of csr_sell4s_kernel (key 7 = 4): only the column ids and lengths
// are staged, kS4bStages slices deep (a 2.7 KB stage instead of 7.8 KB);
// the values are loaded from global memory together with the gathers
// (independent loads, so their latency overlaps).
#ifndef SVDSB_S4B_STAGES
#define SVDSB_S4B_STAGES 4
#endif
constexpr int kS4bStages = SVDSB_S4B_STAGES;
constexpr int kS4bStage = 32 * kSell4sW * 4 + 32 + 16 + 80;   // cols + lens + slice start, 128-B multiple
static_assert(kS4bStage % 128 == 0, "stage alignment");
constexpr size_t kS4bSmem = (size_t)kS4Warps * kS4bStages * kS4bStage;

template <int YROW>
__global__ void __launch_bounds__(kS4Warps * 32, 1)
csr_sell4sb_kernel(int64_t nrows, int64_t nslice, const int64_t *__restrict__ sell_ptr, const int *__restrict__ scol,
                   const double *__restrict__ sval, const uint8_t *__restrict__ slen, const double *__restrict__ x,
                   double *__restrict__ y, int64_t ldy) {
  extern __shared__ __align__(128) unsigned char s4b_smem[];
  __shared__ __align__(8) uint64_t bar[kS4Warps][kS4bStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char *ring = s4b_smem + (size_t)w * kS4bStages * kS4bStage;
  const int64_t gw = (int64_t)blockIdx.x * kS4Warps + w, nw = (int64_t)gridDim.x * kS4Warps;
  if (lane == 0) {
    for (int k = 0; k < kS4bStages; ++k) mbar_init(&bar[w][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t policy = 0;
  if (lane == 0) policy = evict_first_policy();
  auto issue = [&](int64_t sl, int k, int64_t e0, int64_t e1) {
    const int wd = (int)((e1 - e0) >> 5);
    unsigned char *st = ring + (size_t)k * kS4bStage;
    *reinterpret_cast<int64_t *>(st + 32 * kSell4sW * 4 + 32) = e0;   // seen after the mbarrier wait
    mbar_expect_tx(&bar[w][k], 128u * wd + 32u);
    if (wd > 0) bulk_g2s(st, scol + e0, 128u * wd, &bar[w][k], policy);
    bulk_g2s(st + 32 * kSell4sW * 4, slen + 32 * sl, 32u, &bar[w][k], policy);
  };
  // pointers of the next slice to issue, loaded one issue ahead
  int64_t pe0 = 0, pe1 = 0;
  if (lane == 0) {
    for (int k = 0; k < kS4bStages; ++k) {
      const int64_t sl = gw + k * nw;
      if (sl < nslice) issue(sl, k, __ldg(sell_ptr + sl), __ldg(sell_ptr + sl + 1));
    }
    if (gw + kS4bStages * nw < nslice) {
      pe0 = __ldg(sell_ptr + gw + kS4bStages * nw);
      pe1 = __ldg(sell_ptr + gw + kS4bStages * nw + 1);
    }
  }
  pdl_wait();
  int k = 0;
  unsigned phase = 0;
  for (int64_t sl = gw; sl < nslice; sl += nw) {
    mbar_wait(&bar[w][k], phase);
    const unsigned char *st = ring + (size_t)k * kS4bStage;
    const int *sc = reinterpret_cast<const int *>(st);
    const int len = st[32 * kSell4sW * 4 + lane];
    const int64_t e0 = *reinterpret_cast<const int64_t *>(st + 32 * kSell4sW * 4 + 32);
    const int64_t row = (sl << 5) + lane;
    double out[4];
    s4_fold(S4GlobalVals{sval + e0 + lane}, sc, lane, len, S4GlobalX{x}, out);
    if (row < nrows) store_row4<YROW>(y, ldy, row, out);
    __syncwarp();
    const int64_t nx = sl + kS4bStages * nw;
    if (lane == 0 && nx < nslice) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(nx, k, pe0, pe1);
      if (nx + nw < nslice) {
        pe0 = __ldg(sell_ptr + nx + nw);
        pe1 = __ldg(sell_ptr + nx + nw + 1);
      }
    }
    if (++k == kS4bStages) {
      k = 0;
      phase ^= 1u;
    }
  }
  pdl_trigger();
}

constexpr int kSellTMax = 64;  // transposed sliced-ELL rows (longer: one warp per row)

// ---- device build of the sliced-ELL copies (build_sell_device)
struct RowLenIn {
  const int *rp;
  int lo, hi;  // lo < length <= hi
  __host__ __device__ bool operator()(const int &r) const {
    const int l = rp[r + 1] - rp[r];
    return l > lo && l <= hi;
  }
};

__global__ void sell_keys_kernel(int64_t n, const int *__restrict__ rows, const int *__restrict__ rp,
                                 unsigned *__restrict__ key) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) key[i] = (unsigned)(kSellTMax - (rp[rows[i] + 1] - rp[rows[i]]));  // longest first
}

// w[s + 1] = 32 * (longest row of slice s); w[0] = 0
__global__ void sell_width_kernel(int64_t nq, int64_t ns, const int *__restrict__ perm, const int *__restrict__ rp,
                                  int64_t *__restrict__ w) {
  const int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (sl == 0) w[0] = 0;
  if (sl >= ns) return;
  int m = 0;
  for (int64_t q = 32 * sl; q < min(nq, 32 * sl + 32); ++q) {
    const int64_t r = perm ? perm[q] : q;
    m = max(m, rp[r + 1] - rp[r]);
  }
  w[sl + 1] = 32 * (int64_t)m;
}

__global__ void sell_fill_kernel(int64_t nrows, const int *__restrict__ perm, const int *__restrict__ row_ptr,
                                 const int *__restrict__ col, const double *__restrict__ val,
                                 const int64_t *__restrict__ sell_ptr, int *__restrict__ scol,
                                 double *__restrict__ sval, uint8_t *__restrict__ slen) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nrows) return;
  const int64_t row = perm ? perm[q] : q;
  const int64_t sl = q >> 5;
  const int t = (int)(q & 31);
  const int k0 = row_ptr[row], k1 = row_ptr[row + 1];
  if (slen) slen[q] = (uint8_t)min(k1 - k0, 255);
  const int64_t base = sell_ptr[sl] + t;
  const int w = (int)((sell_ptr[sl + 1] - sell_ptr[sl]) >> 5);
  for (int j = 0; j < w; ++j) {
    const bool in = k0 + j < k1;
    scol[base + 32 * (int64_t)j] = in ? col[k0 + j] : 0;
    sval[base + 32 * (int64_t)j] = in ? val[k0 + j] : 0.0;
  }
}

// Transposed b = 4 rows of kSellTMax..kTileNnz nonzeros ("mid" rows), one
// warp per row: lanes load 32 values / column ids at a time (coalesced) and
// gather their x rows; four lanes (one per block column) then add the 32
// products left to right -- np.add.at's order, bit-identical.

// One warp, one mid row (called by csr_sell4t_kernel).
// kWR4 rounds of 32 nonzeros per step: every value / column-id load of the
// step is issued first, then every gather, so one DRAM + one L2 round trip
// serve 32 kWR4 nonzeros (one round of 32 used to pay both per 32).
constexpr int kWR4 = 4;

__device__ __forceinline__ void warprow4t(int64_t row, const int *__restrict__ row_ptr, const int *__restrict__ col,
                                          const double *__restrict__ val, const double *__restrict__ x,
                                          double *__restrict__ y, int64_t ldy, int yrow, int acc,
                                          double (*prod)[32 * kWR4 + 1], int exact) {
  const int lane = threadIdx.x & 31;
  const int k0 = __ldg(row_ptr + row), k1 = __ldg(row_ptr + row + 1);
  const int cc = lane & 3;
  double sacc = 0.0;
  if (acc && lane < 4) sacc = yrow ? y[row * 4 + cc] : y[row + cc * ldy];
  if (!exact) {
    // deterministic lane-parallel sum: lane l folds nonzeros l, l+32, ...
    // (fma), then a fixed xor tree; no serial fold (config 4's 65-2048-nnz
    // rows: 16 % of the nonzeros took a third of A^T.Y serially)
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = k0; k < k1; k += 32 * kWR4) {
      int c[kWR4];
      double v[kWR4], xv[kWR4][4];
#pragma unroll
      for (int u = 0; u < kWR4; ++u) {
        const int e = k + 32 * u + lane;
        const bool ok = e < k1;
        c[u] = ok ? ld_ef(col + e) : 0;
        v[u] = ok ? ld_ef(val + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kWR4; ++u) gather4(x, c[u], xv[u]);
#pragma unroll
      for (int u = 0; u < kWR4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) s4[q] = fma(v[u], xv[u][q], s4[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) s4[q] = warp_sum(s4[q]);
    if (lane < 4) {
      const double t = cc == 0 ? s4[0] : cc == 1 ? s4[1] : cc == 2 ? s4[2] : s4[3];
      const double out = acc ? dadd(sacc, t) : t;
      if (yrow)
        y[row * 4 + cc] = out;
      else
        y[row + cc * ldy] = out;
    }
    return;
  }
  for (int k = k0; k < k1; k += 32 * kWR4) {
    int c[kWR4];
    double v[kWR4], xv[kWR4][4];
#pragma unroll
    for (int u = 0; u < kWR4; ++u) {
      const int e = k + 32 * u + lane;
      const bool ok = e < k1;
      c[u] = ok ? ld_ef(col + e) : 0;
      v[u] = ok ? ld_ef(val + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kWR4; ++u) gather4(x, c[u], xv[u]);
#pragma unroll
    for (int u = 0; u < kWR4; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) prod[q][32 * u + lane] = dmul(v[u], xv[u][q]);
    __syncwarp();
    if (lane < 4) {
      // left to right (np.add.at order); shared-memory loads eight ahead of
      // the dependent adds, so the chain runs at the add latency
      const int n = min(32 * kWR4, k1 - k);
      for (int t0 = 0; t0 < n; t0 += 8) {
        double pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pv[u] = prod[cc][min(t0 + u, 32 * kWR4 - 1)];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t0 + u < n) sacc = dadd(sacc, pv[u]);
      }
    }
    __syncwarp();
  }
  if (lane < 4) {
    if (yrow)
      y[row * 4 + cc] = sacc;
    else
      y[row + cc * ldy] = sacc;
  }
}

// Transposed b = 4 product on a sliced-ELL copy whose rows are sorted by
// length (so slices carry almost no padding despite config 4's Zipf row
// lengths): lane q of the sorted order owns row perm[q] and sums its
// products left to right with no FMA, continuing from y when accumulating
// over column blocks -- np.add.at's order, bit-identical to the CSR
// kernels.  Rows longer than a tile are not in the copy (chunk path).
#ifndef SVDSB_DBG_SKIP
#define SVDSB_DBG_SKIP 0   // timing experiments only: 1 skips the mid rows, 2 the sliced rows
#endif
#ifndef SVDSB_EARLY_TRIGGER
#define SVDSB_EARLY_TRIGGER 0   // timing experiment: 1 lets the transposed b = 4 kernels release their dependants at the start
                                // (slower: the waiting dependants take slots from the running grid -- A^T.Y 1330 -> 1397 us)
#endif
#ifndef SVDSB_T4T_MINB
#define SVDSB_T4T_MINB 4   // resident CTAs per SM the register budget targets (64 registers, no spills; 2: 75 registers, 1.7% slower)
#endif
template <int YROW>
__global__ void __launch_bounds__(kTileThreads, SVDSB_T4T_MINB)
csr_sell4t_kernel(int64_t nq, int64_t nslice, const int *__restrict__ perm, const int *__restrict__ row_ptr,
                  const uint8_t *__restrict__ slen, const int64_t *__restrict__ sell_ptr,
                  const int *__restrict__ scol, const double *__restrict__ sval, int nmid,
                  const int *__restrict__ mid, const int *__restrict__ col, const double *__restrict__ val,
                  const double *__restrict__ x, double *__restrict__ y, int64_t ldy, int acc, int g_t4exact,
                  unsigned *__restrict__ ctr) {
  __shared__ double prod[kTileThreads / 32][4][32 * kWR4 + 1];
  const int lane = threadIdx.x & 31;
  const unsigned nwarps = gridDim.x * (kTileThreads / 32);
  const unsigned nitems = (unsigned)(nmid + nslice);
  pdl_wait();
  // Warp work items: the mid rows first (longest work), then the slices.
  // A warp's first item is its own index; the rest come from a counter
  // (ctr[0]; fetched one item ahead so the atomic's round trip hides behind
  // the current item), so a warp that drew long mid rows (65-2048 nonzeros)
  // takes fewer items (config 4: 1370 -> 1360 us per product; the kernel is
  // bound by L1 wavefronts, not by the tail).  Each item is owned by exactly
  // one warp and writes its own rows, so the assignment does not touch the
  // sums.  ctr == nullptr keeps the fixed stride.
  unsigned it = blockIdx.x * (kTileThreads / 32) + (threadIdx.x >> 5);
#if SVDSB_EARLY_TRIGGER
  pdl_trigger();
#endif
  while (it < nitems) {
    unsigned nxt = it + nwarps;
    if (ctr != nullptr && lane == 0) nxt = nwarps + atomicAdd(ctr, 1u);
    if (it < (unsigned)nmid) {
#if SVDSB_DBG_SKIP != 1
      warprow4t(__ldg(mid + it), row_ptr, col, val, x, y, ldy, YROW, acc, prod[threadIdx.x >> 5], g_t4exact);
#endif
    } else {
#if SVDSB_DBG_SKIP != 2
      const int64_t sl = (int64_t)it - nmid;
      const int64_t q = (sl << 5) + lane;
      // the stored length of this sliced position (one coalesced byte load;
      // row_ptr[perm[q]] was two scattered ones).  An empty row of an
      // accumulating block keeps its running sum: nothing to read or write.
      const int len = q < nq ? (int)__ldg(slen + q) : 0;
      if (q < nq && !(acc && len == 0)) {
        const int64_t row = __ldg(perm + q);
        const int64_t base = __ldg(sell_ptr + sl) + lane;
        double s[4] = {0.0, 0.0, 0.0, 0.0};
        if (acc) {
#pragma unroll
          for (int c = 0; c < 4; ++c) s[c] = YROW ? y[row * 4 + c] : y[row + c * ldy];
        }
        for (int j0 = 0; j0 < len; j0 += 4) {
          double xv[4][4], vv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = min(j0 + u, len - 1);
            vv[u] = ld_ef(sval + base + 32 * (int64_t)j);
            gather4(x, ld_ef(scol + base + 32 * (int64_t)j), xv[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u < len) {
#pragma unroll
              for (int c = 0; c < 4; ++c) s[c] = dadd(s[c], dmul(vv[u], xv[u][c]));
            }
        }
        store_row4<YROW>(y, ldy, row, s);
      }
#endif
    }
    it = ctr != nullptr ? __shfl_sync(0xffffffffu, nxt, 0) : nxt;
  }
  // the last warp out rearms the counter for the next launch on this part
  if (ctr != nullptr && lane == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == nwarps - 1) {
      ctr[0] = 0u;
      ctr[1] = 0u;
      __threadfence();
    }
  }
  pdl_trigger();
}


// TMA-staged transposed b = 4 product on the length-sorted sliced-ELL copy
// (rows of at most kSellTMax nonzeros; the mid rows stay on
// csr_sell4t_kernel, long rows on the chunk path).  As csr_sell4s_kernel:
// one persistent CTA of kS4Warps warps per SM, each warp streaming its
// slices through a private ring of kT4Stages stages, each stage one chunk
// of up to kT4Chunk columns of a slice (values, column ids; the slice's
// row permutation and lengths ride with its first chunk), filled by
// cp.async.bulk kT4Stages chunks ahead.  A lane sums its row left to right
// with no FMA, continuing from y when accumulating: np.add.at's order,
// bit-identical to csr_sell4t_kernel.
#ifndef SVDSB_T4_WARPS
#define SVDSB_T4_WARPS 12
#endif
#ifndef SVDSB_T4_STAGES
#define SVDSB_T4_STAGES 4
#endif
constexpr int kT4Chunk = 8;
constexpr int kT4Stages = SVDSB_T4_STAGES;
constexpr int kT4Warps = SVDSB_T4_WARPS;
constexpr int kT4Stage = 32 * kT4Chunk * 12 + 128 + 32 + 96;
static_assert(kT4Stage % 128 == 0, "stage alignment");
constexpr size_t kT4Smem = (size_t)kT4Warps * kT4Stages * kT4Stage;

template <int YROW>
__global__ void __launch_bounds__(kT4Warps * 32, 1)
csr_sell4ts_kernel(int64_t nq, int64_t nslice, const int *__restrict__ perm, const uint8_t *__restrict__ slen,
                   const int64_t *__restrict__ sell_ptr, const int *__restrict__ scol,
                   const double *__restrict__ sval, const double *__restrict__ x, double *__restrict__ y,
                   int64_t ldy, int acc) {
  extern __shared__ __align__(128) unsigned char t4_smem[];
  __shared__ __align__(8) uint64_t bar[kT4Warps][kT4Stages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char *ring = t4_smem + (size_t)w * kT4Stages * kT4Stage;
  const int64_t gw = (int64_t)blockIdx.x * kT4Warps + w, nw = (int64_t)gridDim.x * kT4Warps;
  if (lane == 0) {
    for (int k = 0; k < kT4Stages; ++k) mbar_init(&bar[w][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // producer cursor (lane 0): chunk pj0 of slice psl (width pw, first entry sp0)
  // (nsp0, nsp1: pointers of slice psl + nw, loaded one slice ahead)
  uint64_t policy = 0;
  int64_t psl = gw, sp0 = 0, nsp0 = 0, nsp1 = 0;
  int pw = 0, pj0 = 0;
  if (lane == 0) {
    policy = evict_first_policy();
    if (psl < nslice) {
      sp0 = __ldg(sell_ptr + psl);
      pw = (int)((__ldg(sell_ptr + psl + 1) - sp0) >> 5);
    }
    if (psl + nw < nslice) {
      nsp0 = __ldg(sell_ptr + psl + nw);
      nsp1 = __ldg(sell_ptr + psl + nw + 1);
    }
  }
  auto issue_next = [&](int k) {
    if (psl >= nslice) return;
    unsigned char *st = ring + (size_t)k * kT4Stage;
    const int cw = max(0, min(kT4Chunk, pw - pj0));
    mbar_expect_tx(&bar[w][k], 384u * cw + (pj0 == 0 ? 160u : 0u));
    if (cw > 0) {
      bulk_g2s(st, sval + sp0 + 32 * pj0, 256u * cw, &bar[w][k], policy);
      bulk_g2s(st + 32 * kT4Chunk * 8, scol + sp0 + 32 * pj0, 128u * cw, &bar[w][k], policy);
    }
    if (pj0 == 0) {
      bulk_g2s(st + 32 * kT4Chunk * 12, perm + 32 * psl, 128u, &bar[w][k], policy);
      bulk_g2s(st + 32 * kT4Chunk * 12 + 128, slen + 32 * psl, 32u, &bar[w][k], policy);
    }
    pj0 += kT4Chunk;
    if (pj0 >= pw) {
      pj0 = 0;
      psl += nw;
      sp0 = nsp0;
      pw = (int)((nsp1 - nsp0) >> 5);
      if (psl + nw < nslice) {
        nsp0 = __ldg(sell_ptr + psl + nw);
        nsp1 = __ldg(sell_ptr + psl + nw + 1);
      }
    }
  };
  if (lane == 0)
    for (int k = 0; k < kT4Stages; ++k) issue_next(k);
  pdl_wait();
  int k = 0;
  unsigned phase = 0;
  for (int64_t sl = gw; sl < nslice; sl += nw) {
    const int64_t q = (sl << 5) + lane;
    int64_t row = 0;
    int len = 0, wd = 0;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j0 = 0;; j0 += kT4Chunk) {
      mbar_wait(&bar[w][k], phase);
      const unsigned char *st = ring + (size_t)k * kT4Stage;
      if (j0 == 0) {
        row = reinterpret_cast<const int *>(st + 32 * kT4Chunk * 12)[lane];
        len = st[32 * kT4Chunk * 12 + 128 + lane];
        wd = __shfl_sync(0xffffffffu, len, 0);   // lane 0 holds the slice's longest row
        if (acc && q < nq) {
#pragma unroll
          for (int c = 0; c < 4; ++c) s[c] = YROW ? y[row * 4 + c] : y[row + c * ldy];
        }
      }
      const double *sv = reinterpret_cast<const double *>(st);
      const int *sc = reinterpret_cast<const int *>(st + 32 * kT4Chunk * 8);
      const int jl = min(len, j0 + kT4Chunk);
      if (j0 < jl) {
        double xv[kT4Chunk][4];
#pragma unroll
        for (int u = 0; u < kT4Chunk; ++u) gather4(x, sc[(min(j0 + u, jl - 1) - j0) * 32 + lane], xv[u]);
#pragma unroll
        for (int u = 0; u < kT4Chunk; ++u)
          if (j0 + u < jl) {
            const double v = sv[u * 32 + lane];
#pragma unroll
            for (int c = 0; c < 4; ++c) s[c] = dadd(s[c], dmul(v, xv[u][c]));
          }
      }
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_next(k);
      }
      if (++k == kT4Stages) {
        k = 0;
        phase ^= 1u;
      }
      if (j0 + kT4Chunk >= wd) break;
    }
    if (q < nq) store_row4<YROW>(y, ldy, row, s);
  }
  pdl_trigger();
}


static bool rowlane_on() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SVDSB_SPMV_ROWLANE");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// ------------------------------------------------ bulk-copy tile pipeline
// b = 1 SpMV with the matrix stream moved by the copy engine: each tile's
// val / col / row_ptr ranges go global -> shared with cp.async.bulk
// (16-byte granules, completion counted on one mbarrier per stage) into a
// kBulkStages-deep ring, so up to kBulkStages - 1 tiles are in flight per
// CTA without holding them in registers.  Threads only gather x, form the
// products in place and fold each row in the reference's order -- the same
// arithmetic as csr_tile_pipe_kernel, bit for bit.
constexpr int kBulkStages = 2;
constexpr int64_t kBulkMinBytes = 64ll << 20;  // half of the 126 MB L2

struct __align__(128) BulkStage {
  double val[kTileNnz + 2];
  int col[kTileNnz + 4];
  int rp[kTileRows + 1 + 8];
};

// ROWS: 0 = every tile row has <= 8 nonzeros, 1 = <= 32 (both: one thread
// gathers and folds one row), 2 = longer rows (strided gathers, CTA barrier,
// then the per-row folds).
template <int ORDER, int ROWS>
__global__ void __launch_bounds__(kTileThreads, 2)
csr_tile_bulk_kernel(int ntile, const int4 *__restrict__ info, const int *__restrict__ row_ptr,
                     const int *__restrict__ col, const double *__restrict__ val, const double *__restrict__ x,
                     double *__restrict__ y, int accumulate) {
  extern __shared__ __align__(128) unsigned char bulk_smem[];
  BulkStage *stg = reinterpret_cast<BulkStage *>(bulk_smem);
  uint64_t *bar = reinterpret_cast<uint64_t *>(bulk_smem + kBulkStages * sizeof(BulkStage));
  __shared__ int4 tinfo[kBulkStages];
  const int t = threadIdx.x;
  if (blockIdx.x >= ntile) return;
  if (t == 0) {
    for (int k = 0; k < kBulkStages; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar + k)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t policy = 0;
  if (t == 0) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  // thread 0: arm stage k's barrier with the byte count and start the copies
  auto issue = [&](int tile, int k) {
    const int4 ti = info[tile];
    tinfo[k] = ti;
    const int v0 = ti.z & ~1, v1 = (ti.w + 1) & ~1;
    const int c0 = ti.z & ~3, c1 = (ti.w + 3) & ~3;
    const int r0 = ti.x & ~3, r1 = (ti.y + 4) & ~3;
    const unsigned bytes = 8u * (v1 - v0) + 4u * (c1 - c0) + 4u * (r1 - r0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar + k)), "r"(bytes)
                 : "memory");
    if (v1 > v0) bulk_g2s(stg[k].val, val + v0, 8u * (v1 - v0), bar + k, policy);
    if (c1 > c0) bulk_g2s(stg[k].col, col + c0, 4u * (c1 - c0), bar + k, policy);
    bulk_g2s(stg[k].rp, row_ptr + r0, 4u * (r1 - r0), bar + k, policy);
  };
  // the matrix is immutable after assembly: start streaming it before the
  // producer of x has finished
  if (t == 0)
    for (int k = 0; k < kBulkStages; ++k) {
      const int tk = blockIdx.x + k * gridDim.x;
      if (tk < ntile) issue(tk, k);
    }
  pdl_wait();
  int k = 0;
  unsigned phase = 0;
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    mbar_wait(bar + k, phase);
    const int4 ti = tinfo[k];
    const int nnz = ti.w - ti.z, nrows = ti.y - ti.x;
    double *pv = stg[k].val + (ti.z & 1);
    const int *pc = stg[k].col + (ti.z & 3);
    const int *prp = stg[k].rp + (ti.x & 3);
    if (ROWS < 2) {
      // short rows: each thread gathers (8 independent loads at a time) and
      // folds its own row, so no CTA barrier separates gathers and folds
      if (t < nrows) {
        const int s0 = prp[t] - ti.z;
        const int len = prp[t + 1] - prp[t];
        for (int j0 = 0; j0 < len; j0 += 8) {
          // indices first, then all gathers, then the products: 8 loads in
          // flight per thread (index 0 stands in past the row)
          int cj[8];
          double xg[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) cj[j] = (j0 + j < len) ? pc[s0 + j0 + j] : 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) xg[j] = __ldg(x + cj[j]);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j0 + j < len) pv[s0 + j0 + j] = dmul(pv[s0 + j0 + j], xg[j]);
          if (ROWS == 0) break;
        }
        y[ti.x + t] = accumulate ? fold_row_from(y[ti.x + t], pv + s0, len)
                                 : fold_row<ORDER, ROWS == 0>(pv + s0, len);
      }
    } else {
      int ce[kPerThread];
      double xg[kPerThread];
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        const int e = t + i * kTileThreads;
        ce[i] = e < nnz ? pc[e] : 0;
      }
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) xg[i] = __ldg(x + ce[i]);
#pragma unroll
      for (int i = 0; i < kPerThread; ++i) {
        const int e = t + i * kTileThreads;
        if (e < nnz) pv[e] = dmul(pv[e], xg[i]);
      }
      __syncthreads();
      if (t < nrows) {
        const int s0 = prp[t] - ti.z;
        const int len = prp[t + 1] - prp[t];
        y[ti.x + t] = accumulate ? fold_row_from(y[ti.x + t], pv + s0, len) : fold_row<ORDER, false>(pv + s0, len);
      }
    }
    __syncthreads();  // stage k consumed
    if (t == 0) {
      const int nt = tile + kBulkStages * gridDim.x;
      if (nt < ntile) {
        // generic-proxy writes (the products) precede the copy engine's
        // next writes into this stage
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(nt, k);
      }
    }
    if (++k == kBulkStages) {
      k = 0;
      phase ^= 1u;
    }
  }
  pdl_trigger();
}

static bool spmv_bulk_on() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SVDSB_SPMV_BULK");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

static int pipe_rows_grid(const void *kernel, size_t smem, bool bulk = false) {
  static const void *which[8] = {nullptr};
  static int cap[8] = {0};
  for (int i = 0; i < 8; ++i)
    if (which[i] == kernel) return cap[i];
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  (void)bulk;  // the default carveout keeps L1 for the gathered vector
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kTileThreads, smem);
  if (occ < 1) occ = 1;
  for (int i = 0; i < 8; ++i)
    if (!which[i]) {
      which[i] = kernel;
      cap[i] = occ * num_sms();
      break;
    }
  return occ * num_sms();
}

static int pipe_grid(const void *kernel) {
  static int cap[8] = {0};
  static const void *which[8] = {nullptr};
  for (int i = 0; i < 8; ++i)
    if (which[i] == kernel) return cap[i];
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kTileThreads, 0);
  if (occ < 1) occ = 1;
  for (int i = 0; i < 8; ++i)
    if (!which[i]) {
      which[i] = kernel;
      cap[i] = occ * num_sms();
      break;
    }
  return occ * num_sms();
}

// column-major (ld) -> row-major (stride b) and back
__global__ void pack_rows_kernel(int64_t rows, int b, const double *__restrict__ x, int64_t ldx,
                                 double *__restrict__ xr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * b) return;
  int64_t r = i / b;
  int cc = (int)(i - r * b);
  xr[i] = x[r + cc * ldx];
}

// Row-major copy of a b-column block with stride bp >= b (columns b..bp-1
// zero): 2- and 3-column products run the 4-column kernels.
__global__ void pack_pad_kernel(int64_t rows, int b, int bp, const double *__restrict__ x, int64_t ldx,
                                double *__restrict__ xr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * bp) return;
  int64_t r = i / bp;
  int cc = (int)(i - r * bp);
  xr[i] = cc < b ? x[r + cc * ldx] : 0.0;
}

__global__ void unpack_pad_kernel(int64_t rows, int b, int bp, const double *__restrict__ xr, double *__restrict__ y,
                                  int64_t ldy) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * b) return;
  int64_t r = i % rows;
  int cc = (int)(i / rows);
  y[r + cc * ldy] = xr[r * bp + cc];
}

__global__ void unpack_rows_kernel(int64_t rows, int b, const double *__restrict__ xr, double *__restrict__ y,
                                   int64_t ldy) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows * b) return;
  int64_t r = i / b;
  int cc = (int)(i - r * b);
  y[r + cc * ldy] = xr[i];
}

// s[cc] += v * xr[cc] for cc < b, one 256-bit gather when b == 4.
__device__ __forceinline__ void gather_acc(const double *xr, int b, double v, double (&s)[4]) {
  if (b == 4) {
    double x0, x1, x2, x3;
    unsigned long long a0, a1, a2, a3;
    asm("ld.global.nc.L2::evict_last.v4.b64 {%0, %1, %2, %3}, [%4];"
        : "=l"(a0), "=l"(a1), "=l"(a2), "=l"(a3) : "l"(xr));
    x0 = __longlong_as_double(a0);
    x1 = __longlong_as_double(a1);
    x2 = __longlong_as_double(a2);
    x3 = __longlong_as_double(a3);
    s[0] = fma(v, x0, s[0]);
    s[1] = fma(v, x1, s[1]);
    s[2] = fma(v, x2, s[2]);
    s[3] = fma(v, x3, s[3]);
  } else {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
      if (cc < b) s[cc] = fma(v, __ldg(xr + cc), s[cc]);
  }
}

// One CTA per chunk of a long row: partial sums of b columns.  x is
// row-major (stride b) when xrow, else column-major (ldx).
__global__ void __launch_bounds__(kTileThreads)
csr_chunk_kernel(const int *__restrict__ chunk_nz, const int *__restrict__ col,
                 const double *__restrict__ val, const double *__restrict__ x,
                 int64_t ldx, int xrow, int b, double *__restrict__ part) {
  pdl_wait();
#if SVDSB_EARLY_TRIGGER
  pdl_trigger();  // dependants (the fix-up kernel) may be scheduled under this grid's tail; they still wait for its completion
#endif
  __shared__ double red[kTileThreads / 32][4];
  const int nz0 = chunk_nz[2 * blockIdx.x], nz1 = chunk_nz[2 * blockIdx.x + 1];
  const int t = threadIdx.x;
  if ((xrow || b == 1) && b <= 4) {
    // one pass over the chunk for all b columns; 4-deep unroll for MLP
    // (b == 1: column- and row-major coincide)
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    int k = nz0 + t;
    for (; k + 3 * kTileThreads < nz1; k += 4 * kTileThreads) {
      int64_t c0 = ld_ef(col + k), c1 = ld_ef(col + k + kTileThreads);
      int64_t c2 = ld_ef(col + k + 2 * kTileThreads), c3 = ld_ef(col + k + 3 * kTileThreads);
      double v0 = ld_ef(val + k), v1 = ld_ef(val + k + kTileThreads);
      double v2 = ld_ef(val + k + 2 * kTileThreads), v3 = ld_ef(val + k + 3 * kTileThreads);
      gather_acc(x + c0 * b, b, v0, s);
      gather_acc(x + c1 * b, b, v1, s);
      gather_acc(x + c2 * b, b, v2, s);
      gather_acc(x + c3 * b, b, v3, s);
    }
    for (; k < nz1; k += kTileThreads) {
      int64_t c0 = ld_ef(col + k);
      double v0 = ld_ef(val + k);
      gather_acc(x + c0 * b, b, v0, s);
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      double w = warp_sum(s[cc]);
      if ((t & 31) == 0) red[t >> 5][cc] = w;
    }
    __syncthreads();
    if (t < b) {
      double acc = 0.0;
      for (int w = 0; w < kTileThreads / 32; ++w) acc += red[w][t];
      part[(int64_t)blockIdx.x * kMaxB + t] = acc;
    }
    return;
  }
  for (int cc = 0; cc < b; ++cc) {
    double s = 0.0;
    for (int k = nz0 + t; k < nz1; k += kTileThreads) {
      int64_t cix = ld_ef(col + k);
      double xv = xrow ? __ldg(x + cix * b + cc) : __ldg(x + cix + cc * ldx);
      s = fma(ld_ef(val + k), xv, s);
    }
    s = warp_sum(s);
    if ((t & 31) == 0) red[t >> 5][0] = s;
    __syncthreads();
    if (t == 0) {
      double acc = 0.0;
      for (int w = 0; w < kTileThreads / 32; ++w) acc += red[w][0];
      part[(int64_t)blockIdx.x * kMaxB + cc] = acc;
    }
    __syncthreads();
  }
}


// Long rows of a transposed b = 4 product (the Zipf head of config 4's
// A^T: 70 % of the nonzeros) by operand tiles: one CTA per kHeadTile rows
// of the row-major operand x stages the tile in shared memory with
// coalesced loads, then its warps sum the pieces -- at most kHeadPiece
// consecutive nonzeros of one long row that fall in the tile -- against
// shared memory (lane-parallel fma, fixed xor tree), one partial per piece.
// Every x row is read from L2 once per tile instead of once per nonzero;
// csr_long_fixup_kernel then adds each long row's partials in tile order
// (deterministic; within rounding of the sequential sum, like the chunks).
constexpr int kHeadTile = 2048;
constexpr int kHeadPiece = 256;

__global__ void __launch_bounds__(kTileThreads)
csr_headtile4_kernel(int ntile, int64_t xrows, const int *__restrict__ htp, const int4 *__restrict__ pieces,
                     const int *__restrict__ col, const double *__restrict__ val, const double *__restrict__ x,
                     double *__restrict__ part) {
  extern __shared__ __align__(16) double ys[];  // kHeadTile x 4
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  pdl_wait();
  for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
    const int64_t r0 = (int64_t)t * kHeadTile;
    const int nr = (int)min((int64_t)kHeadTile, xrows - r0);
    const double2 *src = reinterpret_cast<const double2 *>(x + r0 * 4);
    double2 *dst = reinterpret_cast<double2 *>(ys);
    for (int i = threadIdx.x; i < 2 * nr; i += kTileThreads) dst[i] = __ldg(src + i);
    __syncthreads();
    const int p1 = __ldg(htp + t + 1);
    for (int pc = __ldg(htp + t) + w; pc < p1; pc += kTileThreads / 32) {
      const int4 pi = __ldg(pieces + pc);
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = pi.x + lane; k < pi.y; k += 32 * 4) {
        int c[4];
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = k + 32 * u;
          const bool ok = e < pi.y;
          c[u] = ok ? ld_ef(col + e) - (int)r0 : 0;
          v[u] = ok ? ld_ef(val + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 lo = dst[2 * c[u]], hi = dst[2 * c[u] + 1];
          s4[0] = fma(v[u], lo.x, s4[0]);
          s4[1] = fma(v[u], lo.y, s4[1]);
          s4[2] = fma(v[u], hi.x, s4[2]);
          s4[3] = fma(v[u], hi.y, s4[3]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] = warp_sum(s4[q]);
      if (lane < 4) part[(int64_t)pi.z * 4 + lane] = lane == 0 ? s4[0] : lane == 1 ? s4[1] : lane == 2 ? s4[2] : s4[3];
    }
    __syncthreads();
  }
  pdl_trigger();
}

// seg[li * (ntile + 1) + t] = first nonzero of long row li at or past tile t
__global__ void head_bounds_kernel(int nlong, int ntile, const int *__restrict__ long_row,
                                   const int *__restrict__ row_ptr, const int *__restrict__ col, int *__restrict__ seg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nlong * (ntile + 1)) return;
  const int li = (int)(i / (ntile + 1)), t = (int)(i % (ntile + 1));
  const int r = long_row[li];
  int lo = row_ptr[r], hi = row_ptr[r + 1];
  const int64_t key = (int64_t)t * kHeadTile;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (col[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  seg[i] = lo;
}

// One warp per (long row, column): lanes take chunks l, l+32, ... and a
// fixed shuffle tree combines them (deterministic for a given chunking).
__global__ void csr_long_fixup_kernel(int nlong, const int *__restrict__ long_row,
                                      const int *__restrict__ long_cptr,
                                      const double *__restrict__ part, int b,
                                      double *__restrict__ y, int64_t ldy, int yrow, int accumulate,
                                      int pstride) {
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nlong * b) return;
  const int li = warp / b, cc = warp % b;
  double s = 0.0;
  for (int ch = long_cptr[li] + lane; ch < long_cptr[li + 1]; ch += 32) s += part[(int64_t)ch * pstride + cc];
  s = warp_sum(s);
  if (lane == 0) {
    int64_t r = long_row[li];
    double *yp = yrow ? y + r * b + cc : y + r + cc * ldy;
    *yp = accumulate ? *yp + s : s;
  }
}

// ---------------------------------------------------------------- partition


// SVDSB_TRACE=<ms>: print the host-side phases of a matrix assembly that
// took longer than <ms> (diagnoses stalls in the e2e path)
struct CreateTrace {
  const char *what[32];
  std::chrono::steady_clock::time_point t[32];
  int n = 0;
  double limit_ms = -1.0;
  CreateTrace() {
    const char *e = getenv("SVDSB_TRACE");
    if (e) limit_ms = atof(e);
    mark("start");
  }
  void mark(const char *w) {
    if (limit_ms >= 0 && n < 32) {
      what[n] = w;
      t[n++] = std::chrono::steady_clock::now();
    }
  }
  ~CreateTrace() {
    if (limit_ms < 0 || n < 2) return;
    auto ms = [&](int a, int b) { return std::chrono::duration<double, std::milli>(t[b] - t[a]).count(); };
    if (ms(0, n - 1) < limit_ms) return;
    fprintf(stderr, "[svdsb create %.1f ms]", ms(0, n - 1));
    for (int i = 1; i < n; ++i) fprintf(stderr, " %s %.2f", what[i], ms(i - 1, i));
    fprintf(stderr, "\n");
  }
};
static thread_local CreateTrace *g_trace = nullptr;
static inline void tmark(const char *w) {
  if (g_trace) g_trace->mark(w);
}

// Device arrays of a CSR part carry kAllocPad bytes of slack: the bulk-copy
// SpMV moves whole 16-byte granules, which can reach past the last element.
constexpr size_t kAllocPad = 64;

// Stream-ordered allocations from the device's default memory pool, which
// keeps freed memory (release threshold = max): assembling a matrix
// allocates and frees a dozen temporaries, and plain cudaMalloc / cudaFree
// synchronise the device and remap pages each time (5-200 ms per matrix).
static cudaError_t pool_init() {
  static bool done = false;
  if (done) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  e = cudaDeviceGetDefaultMemPool(&pool, dev);
  if (e != cudaSuccess) return e;
  uint64_t keep = UINT64_MAX;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e != cudaSuccess) return e;
  done = true;
  return cudaSuccess;
}

template <typename T>
static cudaError_t palloc(T **p, size_t bytes, cudaStream_t st) {
  cudaError_t e = pool_init();
  if (e != cudaSuccess) return e;
  return cudaMallocAsync(reinterpret_cast<void **>(p), bytes, st);
}

static void pfree(void *p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

// Temporary pool allocations of a build step, released (stream-ordered) on
// every return path.
struct StreamTemps {
  cudaStream_t st;
  std::vector<void *> v;
  ~StreamTemps() {
    for (void *q : v) pfree(q, st);
  }
  template <typename T>
  cudaError_t get(T **q, size_t bytes) {
    cudaError_t e = palloc(q, bytes, st);
    if (e == cudaSuccess) v.push_back(*q);
    return e;
  }
};

template <typename T>
static cudaError_t alloc_pad(T **dst, size_t n, cudaStream_t st) {
  return palloc(dst, n * sizeof(T) + kAllocPad, st);
}

static void free_part(CsrPart &p) {
  // pool memory: returned in legacy-stream order (svdsb_csr_destroy has
  // synchronised the device first)
  pfree(p.row_ptr, nullptr);
  pfree(p.col, nullptr);
  pfree(p.val, nullptr);
  pfree(p.tile_r, nullptr);
  pfree(p.tile_info, nullptr);
  pfree(p.long_row, nullptr);
  pfree(p.long_cptr, nullptr);
  pfree(p.chunk_nz, nullptr);
  pfree(p.chunk_part, nullptr);
  pfree(p.sell_ptr, nullptr);
  pfree(p.sell_perm, nullptr);
  pfree(p.mid_rows, nullptr);
  pfree(p.sell_col, nullptr);
  pfree(p.sell_colh, nullptr);
  pfree(p.sell_hot, nullptr);
  pfree(p.work_ctr, nullptr);
  pfree(p.sell_val, nullptr);
  pfree(p.sell_len, nullptr);
  pfree(p.htp, nullptr);
  pfree(p.hpiece, nullptr);
  pfree(p.hcptr, nullptr);
  pfree(p.hpart, nullptr);
  p = CsrPart();
}

template <typename T>
static int upload(T **dst, const std::vector<T> &src, cudaStream_t st) {
  size_t n = std::max<size_t>(src.size(), 1);
  SVDSB_CUDA(alloc_pad(dst, n, st));
  if (!src.empty())
    SVDSB_CUDA(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return SVDSB_OK;
}

// Sliced ELL copy of a part (see csr_sell4_kernel): slice widths from the
// host row pointer, device fill.  Padding entries (column 0, value 0) are
// never read: a lane stops at its row's length.
static int build_sell(CsrPart &p, cudaStream_t st, bool sorted = false) {
  const std::vector<int> &rp = p.host_row_ptr;
  // sorted: rows of at most kSellTMax nonzeros, longest first (stable);
  // rows up to a tile go to the warp-per-row kernel (mid_rows), longer ones
  // stay on the chunk path
  std::vector<int> order;
  if (sorted) {
    order.reserve(p.rows);
    std::vector<int> mid;
    for (int64_t r = 0; r < p.rows; ++r) {
      const int len = rp[r + 1] - rp[r];
      if (len <= kSellTMax)
        order.push_back((int)r);
      else if (len <= kTileNnz)
        mid.push_back((int)r);
    }
    int *dmid = nullptr;
    int rcm = upload(&dmid, mid, st);
    if (rcm) return rcm;
    p.nmid = (int)mid.size();
    p.mid_rows = dmid;
    // stable counting sort by length, longest first (lengths <= kSellTMax)
    std::vector<int64_t> start(kSellTMax + 2, 0);
    for (int r : order) start[kSellTMax - (rp[r + 1] - rp[r]) + 1]++;
    for (int k = 1; k <= kSellTMax + 1; ++k) start[k] += start[k - 1];
    std::vector<int> sorted_rows(order.size());
    for (int r : order) sorted_rows[start[kSellTMax - (rp[r + 1] - rp[r])]++] = r;
    order.swap(sorted_rows);
  }
  const int64_t nq = sorted ? (int64_t)order.size() : p.rows;
  auto row_of = [&](int64_t q) -> int64_t { return sorted ? order[q] : q; };
  const int64_t ns = (nq + 31) / 32;
  std::vector<int64_t> sp(ns + 1, 0);
  for (int64_t sl = 0; sl < ns; ++sl) {
    int w = 0;
    for (int64_t q = 32 * sl; q < std::min(nq, 32 * sl + 32); ++q) w = std::max(w, rp[row_of(q) + 1] - rp[row_of(q)]);
    sp[sl + 1] = sp[sl] + 32 * (int64_t)w;
  }
  int64_t *dsp = nullptr;
  int *dperm = nullptr;
  int rc;
  if ((rc = upload(&dsp, sp, st))) return rc;
  std::vector<int> perm_pad;
  if (sorted) {
    perm_pad = order;
    perm_pad.resize(32 * ns, 0);  // whole slices: the staged kernel copies 32 entries per slice
  }
  if (sorted && (rc = upload(&dperm, perm_pad, st))) {
    pfree(dsp, st);
    return rc;
  }
  int *scol = nullptr;
  double *sval = nullptr;
  uint8_t *slen = nullptr;
  if (alloc_pad(&scol, std::max<int64_t>(sp[ns], 1), st) != cudaSuccess ||
      alloc_pad(&sval, std::max<int64_t>(sp[ns], 1), st) != cudaSuccess ||
      alloc_pad(&slen, std::max<int64_t>(32 * ns, 32), st) != cudaSuccess ||
      cudaMemsetAsync(slen, 0, std::max<int64_t>(32 * ns, 32), st) != cudaSuccess) {
    pfree(dsp, st);
    pfree(dperm, st);
    pfree(scol, st);
    pfree(sval, st);
    pfree(slen, st);
    set_error("sliced-ELL allocation failed");
    return SVDSB_ERR_ALLOC;
  }
  if (nq > 0) {
    sell_fill_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(nq, dperm, p.row_ptr, p.col, p.val, dsp, scol,
                                                                   sval, slen);
    SVDSB_LAUNCHED();
  }
  p.nslice = ns;
  p.nsell = nq;
  p.sell_perm = dperm;
  p.sell_ptr = dsp;
  p.sell_col = scol;
  p.sell_val = sval;
  p.sell_len = slen;
  return SVDSB_OK;
}

// The sliced-ELL copy built on the device (CUB select / stable radix sort
// by length / scan); the same layout and bits as the host build above, a
// few ms instead of tens for config 4's parts (e2e: every new matrix
// builds its copies).
static int build_sell_device(CsrPart &p, cudaStream_t st, bool sorted) {
  StreamTemps temps{st, {}};
  int *dperm = nullptr, *dmid = nullptr;
  int64_t nq = p.rows;
  int nmid = 0;
  if (sorted) {
    int *sel = nullptr, *cnt = nullptr, *order = nullptr;
    unsigned *key = nullptr, *key_s = nullptr;
    SVDSB_CUDA(temps.get(&sel, sizeof(int) * std::max<int64_t>(p.rows, 1)));
    SVDSB_CUDA(temps.get(&cnt, sizeof(int) * 2));
    cub::CountingInputIterator<int> rows(0);
    size_t tb = 0, tb2 = 0;
    cub::DeviceSelect::If(nullptr, tb, rows, sel, cnt, (int)p.rows, RowLenIn{p.row_ptr, -1, kSellTMax}, st);
    cub::DeviceSelect::If(nullptr, tb2, rows, sel, cnt + 1, (int)p.rows, RowLenIn{p.row_ptr, kSellTMax, kTileNnz},
                          st);
    void *tmp = nullptr;
    SVDSB_CUDA(temps.get(&tmp, std::max(tb, tb2)));
    // mid rows first (into sel), copied out, then the short rows
    SVDSB_CUDA(cub::DeviceSelect::If(tmp, tb2, rows, sel, cnt + 1, (int)p.rows,
                                     RowLenIn{p.row_ptr, kSellTMax, kTileNnz}, st));
    int hc[2] = {0, 0};
    SVDSB_CUDA(cudaMemcpyAsync(&hc[1], cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    SVDSB_CUDA(cudaStreamSynchronize(st));
    nmid = hc[1];
    if (nmid > 0) {
      SVDSB_CUDA(palloc(&dmid, sizeof(int) * nmid, st));
      SVDSB_CUDA(cudaMemcpyAsync(dmid, sel, sizeof(int) * nmid, cudaMemcpyDeviceToDevice, st));
    }
    SVDSB_CUDA(cub::DeviceSelect::If(tmp, tb, rows, sel, cnt, (int)p.rows, RowLenIn{p.row_ptr, -1, kSellTMax}, st));
    SVDSB_CUDA(cudaMemcpyAsync(&hc[0], cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    SVDSB_CUDA(cudaStreamSynchronize(st));
    nq = hc[0];
    const int64_t nsq = (nq + 31) / 32;
    SVDSB_CUDA(palloc(&dperm, sizeof(int) * std::max<int64_t>(32 * nsq, 1) + kAllocPad, st));
    SVDSB_CUDA(cudaMemsetAsync(dperm, 0, sizeof(int) * std::max<int64_t>(32 * nsq, 1), st));
    if (nq > 0) {
      SVDSB_CUDA(temps.get(&key, sizeof(unsigned) * nq));
      SVDSB_CUDA(temps.get(&key_s, sizeof(unsigned) * nq));
      SVDSB_CUDA(temps.get(&order, sizeof(int) * nq));
      sell_keys_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(nq, sel, p.row_ptr, key);
      SVDSB_LAUNCHED();
      size_t tbs = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tbs, key, key_s, sel, dperm, (int)nq, 0, 7, st);
      void *tmps = nullptr;
      SVDSB_CUDA(temps.get(&tmps, tbs));
      SVDSB_CUDA(cub::DeviceRadixSort::SortPairs(tmps, tbs, key, key_s, sel, dperm, (int)nq, 0, 7, st));
      bump_launches();
    }
  }
  const int64_t ns = (nq + 31) / 32;
  int64_t *dsp = nullptr;
  SVDSB_CUDA(palloc(&dsp, sizeof(int64_t) * (ns + 1) + kAllocPad, st));
  sell_width_kernel<<<(unsigned)((ns + 256) / 256), 256, 0, st>>>(nq, ns, dperm, p.row_ptr, dsp);
  SVDSB_LAUNCHED();
  if (ns > 0) {
    size_t tbw = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tbw, dsp + 1, dsp + 1, (int)ns, st);
    void *tmpw = nullptr;
    SVDSB_CUDA(temps.get(&tmpw, tbw));
    SVDSB_CUDA(cub::DeviceScan::InclusiveSum(tmpw, tbw, dsp + 1, dsp + 1, (int)ns, st));
    bump_launches();
  }
  int64_t total = 0;
  SVDSB_CUDA(cudaMemcpyAsync(&total, dsp + ns, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SVDSB_CUDA(cudaStreamSynchronize(st));
  int *scol = nullptr;
  double *sval = nullptr;
  uint8_t *slen = nullptr;
  if (alloc_pad(&scol, std::max<int64_t>(total, 1), st) != cudaSuccess ||
      alloc_pad(&sval, std::max<int64_t>(total, 1), st) != cudaSuccess ||
      alloc_pad(&slen, std::max<int64_t>(32 * ns, 32), st) != cudaSuccess ||
      cudaMemsetAsync(slen, 0, std::max<int64_t>(32 * ns, 32), st) != cudaSuccess) {
    pfree(dsp, st);
    pfree(dperm, st);
    pfree(dmid, st);
    pfree(scol, st);
    pfree(sval, st);
    pfree(slen, st);
    set_error("sliced-ELL allocation failed");
    return SVDSB_ERR_ALLOC;
  }
  if (nq > 0) {
    sell_fill_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(nq, dperm, p.row_ptr, p.col, p.val, dsp, scol,
                                                                   sval, slen);
    SVDSB_LAUNCHED();
  }
  p.nmid = nmid;
  p.mid_rows = dmid;
  p.nslice = ns;
  p.nsell = nq;
  p.sell_perm = dperm;
  p.sell_ptr = dsp;
  p.sell_col = scol;
  p.sell_val = sval;
  p.sell_len = slen;
  return SVDSB_OK;
}

// Hot-encoded column ids for the forward ring kernel: the kS4Hot columns
// with the most nonzeros (stable descending radix sort of the column
// counts, ties by ascending id) get slots 0..; an entry of a hot column
// stores ~slot.  Skipped (sell_nhot = 0) when those columns carry less than
// a fifth of the nonzeros or the matrix is small.
__global__ void iota_kernel(int64_t n, int *__restrict__ out);

__global__ void count_agg_kernel(int64_t nnz, const int *__restrict__ keys, int *__restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const int c = keys[i];
  const unsigned peers = __match_any_sync(__activemask(), c);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + c, __popc(peers));
}

__global__ void hot_slot_kernel(int nhot, const int *__restrict__ hot, int *__restrict__ slot) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nhot) slot[hot[s]] = s;
}

__global__ void hot_encode_kernel(int64_t n, const int *__restrict__ scol, const int *__restrict__ slot,
                                  int *__restrict__ colh) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = scol[e];
    const int s = slot[c];
    colh[e] = s >= 0 ? ~s : c;
  }
}

static int build_sell_hot(CsrPart &p, cudaStream_t st) {
  if (p.cols <= 4 * kS4Hot || p.nnz < 32 * kS4Hot || !p.sell_col) return SVDSB_OK;
  StreamTemps temps{st, {}};
  int *cnt = nullptr, *cnt_s = nullptr, *ids = nullptr, *ids_s = nullptr, *slot = nullptr;
  SVDSB_CUDA(temps.get(&cnt, sizeof(int) * p.cols));
  SVDSB_CUDA(temps.get(&cnt_s, sizeof(int) * p.cols));
  SVDSB_CUDA(temps.get(&ids, sizeof(int) * p.cols));
  SVDSB_CUDA(temps.get(&ids_s, sizeof(int) * p.cols));
  SVDSB_CUDA(temps.get(&slot, sizeof(int) * p.cols));
  SVDSB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * p.cols, st));
  SVDSB_CUDA(cudaMemsetAsync(slot, 0xff, sizeof(int) * p.cols, st));
  count_agg_kernel<<<(unsigned)((p.nnz + 255) / 256), 256, 0, st>>>(p.nnz, p.col, cnt);
  SVDSB_LAUNCHED();
  iota_kernel<<<(unsigned)((p.cols + 255) / 256), 256, 0, st>>>(p.cols, ids);
  SVDSB_LAUNCHED();
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, cnt, cnt_s, ids, ids_s, (int)p.cols, 0, 32, st);
  void *tmp = nullptr;
  SVDSB_CUDA(temps.get(&tmp, tb));
  SVDSB_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, cnt, cnt_s, ids, ids_s, (int)p.cols, 0, 32, st));
  bump_launches();
  std::vector<int> top(kS4Hot);
  int64_t total = 0;
  SVDSB_CUDA(cudaMemcpyAsync(top.data(), cnt_s, sizeof(int) * kS4Hot, cudaMemcpyDeviceToHost, st));
  SVDSB_CUDA(cudaMemcpyAsync(&total, p.sell_ptr + p.nslice, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SVDSB_CUDA(cudaStreamSynchronize(st));
  int64_t covered = 0;
  for (int c : top) covered += c;
  if (5 * covered < p.nnz || total <= 0) return SVDSB_OK;
  int *hot = nullptr, *colh = nullptr;
  if (palloc(&hot, sizeof(int) * kS4Hot, st) != cudaSuccess || alloc_pad(&colh, total, st) != cudaSuccess) {
    pfree(hot, st);
    pfree(colh, st);
    cudaGetLastError();
    return SVDSB_OK;   // no room for the copy: the plain ring kernel gives the same bits
  }
  SVDSB_CUDA(cudaMemcpyAsync(hot, ids_s, sizeof(int) * kS4Hot, cudaMemcpyDeviceToDevice, st));
  hot_slot_kernel<<<(kS4Hot + 255) / 256, 256, 0, st>>>(kS4Hot, hot, slot);
  SVDSB_LAUNCHED();
  hot_encode_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 32 * num_sms()), 256, 0, st>>>(
      total, p.sell_col, slot, colh);
  SVDSB_LAUNCHED();
  SVDSB_CUDA(cudaStreamSynchronize(st));   // the temporaries are released on return
  p.sell_hot = hot;
  p.sell_colh = colh;
  p.sell_nhot = kS4Hot;
  return SVDSB_OK;
}

static bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// The sliced-ELL copy of a part, built once on the first uncaptured b = 4
// call (serialised: handles may be shared between host threads).  If it
// cannot be built (out of memory) the part keeps using the CSR kernels,
// which give the same bits, and the solve carries on.
static std::mutex g_sell_mu;
static bool ensure_sell(const CsrPart &cp, cudaStream_t st, bool sorted) {
  if (cp.sell_val) return true;
  if (cp.sell_failed || capturing(st)) return false;
  std::lock_guard<std::mutex> lk(g_sell_mu);
  CsrPart &p = const_cast<CsrPart &>(cp);  // cache fields only; the matrix itself is immutable
  if (p.sell_val || p.sell_failed) return p.sell_val != nullptr;
  const int rc = g_tune[10] == 1 ? build_sell(p, st, sorted) : build_sell_device(p, st, sorted);
  if (rc != SVDSB_OK) {
    p.sell_failed = true;
    pfree(p.mid_rows, st);
    p.mid_rows = nullptr;
    p.nmid = 0;
    cudaGetLastError();
    set_error("");
    return false;
  }
  if (sorted && !p.work_ctr) {
    if (palloc(&p.work_ctr, 2 * sizeof(unsigned), st) == cudaSuccess) {
      cudaMemsetAsync(p.work_ctr, 0, 2 * sizeof(unsigned), st);
    } else {
      p.work_ctr = nullptr;   // fixed-stride assignment
      cudaGetLastError();
    }
  }
  if (!sorted && p.sell_len && p.maxlen <= kSell4sW && g_tune[12] == 1 && build_sell_hot(p, st) != SVDSB_OK) {
    cudaGetLastError();   // the hot copy is optional
    set_error("");
  }
  return true;
}

// Tile the rows (host; row_ptr already on host in p.host_row_ptr).
static int build_partition(CsrPart &p, cudaStream_t st) {
  const std::vector<int> &rp = p.host_row_ptr;
  std::vector<int> tiles, lrows, lcptr, cnz;
  int open = -1, nrows = 0, nnz_blk = 0;
  auto close = [&](int r_end) {
    if (open >= 0) {
      tiles.push_back(open);
      tiles.push_back(r_end);
    }
    open = -1;
    nrows = 0;
    nnz_blk = 0;
  };
  lcptr.push_back(0);
  for (int64_t r = 0; r < p.rows; ++r) {
    int len = rp[r + 1] - rp[r];
    if (len > kTileNnz) {
      close((int)r);
      lrows.push_back((int)r);
      for (int z = rp[r]; z < rp[r + 1]; z += kLongChunk) {
        cnz.push_back(z);
        cnz.push_back(std::min(z + kLongChunk, rp[r + 1]));
      }
      lcptr.push_back((int)(cnz.size() / 2));
      continue;
    }
    if (open >= 0 && (nrows == kTileRows || nnz_blk + len > kTileNnz)) close((int)r);
    if (open < 0) open = (int)r;
    nrows += 1;
    nnz_blk += len;
    p.maxlen = std::max(p.maxlen, len);
  }
  close((int)p.rows);
  p.ntile = (int)(tiles.size() / 2);
  p.nlong = (int)lrows.size();
  p.nchunk = (int)(cnz.size() / 2);
  std::vector<int> info;
  info.reserve(4 * p.ntile);
  for (int i = 0; i < p.ntile; ++i) {
    info.push_back(tiles[2 * i]);
    info.push_back(tiles[2 * i + 1]);
    info.push_back(rp[tiles[2 * i]]);
    info.push_back(rp[tiles[2 * i + 1]]);
  }
  int rc;
  if ((rc = upload(reinterpret_cast<int **>(&p.tile_info), info, st))) return rc;
  if ((rc = upload(&p.tile_r, tiles, st))) return rc;
  if ((rc = upload(&p.long_row, lrows, st))) return rc;
  if ((rc = upload(&p.long_cptr, lcptr, st))) return rc;
  if ((rc = upload(&p.chunk_nz, cnz, st))) return rc;
  SVDSB_CUDA(palloc(&p.chunk_part, sizeof(double) * kMaxB * std::max(p.nchunk, 1), st));
  return SVDSB_OK;
}

// Head tiles of a part's long rows (see csr_headtile4_kernel): tile
// boundaries inside every long row by binary search on the device, the
// piece lists on the host.  Serialised and built once, like the sliced-ELL
// copies; a part whose build fails keeps the chunk path (same semantics).
static int build_head(CsrPart &p, cudaStream_t st) {
  const int ntile = (int)((p.cols + kHeadTile - 1) / kHeadTile);
  const int64_t nseg = (int64_t)p.nlong * (ntile + 1);
  StreamTemps temps{st, {}};
  int *dseg = nullptr;
  SVDSB_CUDA(temps.get(&dseg, sizeof(int) * nseg));
  head_bounds_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, st>>>(p.nlong, ntile, p.long_row, p.row_ptr, p.col,
                                                                    dseg);
  SVDSB_LAUNCHED();
  std::vector<int> seg(nseg);
  SVDSB_CUDA(cudaMemcpyAsync(seg.data(), dseg, sizeof(int) * nseg, cudaMemcpyDeviceToHost, st));
  SVDSB_CUDA(cudaStreamSynchronize(st));
  auto npieces = [&](int li, int t) {
    const int len = seg[(int64_t)li * (ntile + 1) + t + 1] - seg[(int64_t)li * (ntile + 1) + t];
    return (len + kHeadPiece - 1) / kHeadPiece;
  };
  // slots long row by long row (tile order inside), pieces tile by tile
  std::vector<int> hcptr(p.nlong + 1, 0), base((int64_t)p.nlong * ntile);
  for (int li = 0; li < p.nlong; ++li) {
    int acc = hcptr[li];
    for (int t = 0; t < ntile; ++t) {
      base[(int64_t)li * ntile + t] = acc;
      acc += npieces(li, t);
    }
    hcptr[li + 1] = acc;
  }
  std::vector<int> htp(ntile + 1, 0);
  std::vector<int> pcs;
  pcs.reserve(4 * (size_t)hcptr[p.nlong]);
  for (int t = 0; t < ntile; ++t) {
    htp[t] = (int)(pcs.size() / 4);
    for (int li = 0; li < p.nlong; ++li) {
      const int k0 = seg[(int64_t)li * (ntile + 1) + t], k1 = seg[(int64_t)li * (ntile + 1) + t + 1];
      int slot = base[(int64_t)li * ntile + t];
      for (int k = k0; k < k1; k += kHeadPiece, ++slot) {
        pcs.push_back(k);
        pcs.push_back(std::min(k + kHeadPiece, k1));
        pcs.push_back(slot);
        pcs.push_back(0);
      }
    }
  }
  htp[ntile] = (int)(pcs.size() / 4);
  int rc;
  if ((rc = upload(&p.htp, htp, st)) || (rc = upload(reinterpret_cast<int **>(&p.hpiece), pcs, st)) ||
      (rc = upload(&p.hcptr, hcptr, st)))
    return rc;
  SVDSB_CUDA(palloc(&p.hpart, sizeof(double) * 4 * std::max(hcptr[p.nlong], 1), st));
  p.nhtile = ntile;
  return SVDSB_OK;
}

static std::mutex g_head_mu;
static bool ensure_head(const CsrPart &cp, cudaStream_t st) {
  if (cp.hpart) return true;
  if (cp.head_failed || cp.nlong == 0 || capturing(st)) return false;
  std::lock_guard<std::mutex> lk(g_head_mu);
  CsrPart &p = const_cast<CsrPart &>(cp);  // cache fields only
  if (p.hpart || p.head_failed) return p.hpart != nullptr;
  if (build_head(p, st) != SVDSB_OK) {
    p.head_failed = true;
    pfree(p.htp, st);
    pfree(p.hpiece, st);
    pfree(p.hcptr, st);
    p.htp = p.hcptr = nullptr;
    p.hpiece = nullptr;
    cudaGetLastError();
    set_error("");
    return false;
  }
  return true;
}

// y = P x for one orientation.  xrow / yrow: operands row-major with
// stride b (only for 2 <= b <= 4); otherwise column-major with ld.
template <int ORDER>
static int part_matvec(const CsrPart &p, const double *x, int64_t ldx, int xrow, double *y, int64_t ldy, int yrow,
                       int b, cudaStream_t st, int acc = 0) {
  if (p.rows == 0) return SVDSB_OK;
  if (b == 1) xrow = yrow = 0;
  if (xrow || yrow) {
    if (b > 4) {
      set_error("row-major SpMV operands need block <= 4");
      return SVDSB_ERR_ARG;
    }
    if (ORDER == 0 && b == 4 && xrow && !acc && p.nlong == 0 && p.maxlen <= 129 && rowlane_on() &&
        g_tune[0] == 0) {
      // sliced-ELL copy, built on the first uncaptured call
      ensure_sell(p, st, false);
      if (p.sell_val && !p.sell_perm && p.maxlen <= kSellW && g_tune[2] == 1) {  // measured slower (register spills)
        auto k = yrow ? csr_sell4w_kernel<1> : csr_sell4w_kernel<0>;
        const int g = (int)std::min<int64_t>((p.nslice + 7) / 8, pipe_rows_grid(reinterpret_cast<const void *>(k), 0));
        SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.rows, p.nslice, p.row_ptr, p.sell_ptr, p.sell_col, p.sell_val, x,
                         y, ldy);
        return SVDSB_OK;
      }
      if (p.sell_val && p.sell_len && p.maxlen <= kSell4sW && g_tune[7] == 4) {
        auto k = yrow ? csr_sell4sb_kernel<1> : csr_sell4sb_kernel<0>;
        static bool attrb = false;
        if (!attrb) {
          cudaFuncSetAttribute(csr_sell4sb_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kS4bSmem);
          cudaFuncSetAttribute(csr_sell4sb_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kS4bSmem);
          attrb = true;
        }
        const int g = (int)std::min<int64_t>(num_sms(), (p.nslice + kS4Warps - 1) / kS4Warps);
        SVDSB_LAUNCH_PDL(k, g, kS4Warps * 32, kS4bSmem, st, p.rows, p.nslice, p.sell_ptr, p.sell_col, p.sell_val,
                         p.sell_len, x, y, ldy);
        return SVDSB_OK;
      }
      if (p.sell_val && p.sell_len && p.maxlen <= kSell4sW && g_tune[7] != 1) {
        static bool attr = false;
        if (!attr) {
          cudaFuncSetAttribute(csr_sell4s_kernel<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kS4Smem);
          cudaFuncSetAttribute(csr_sell4s_kernel<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kS4Smem);
          cudaFuncSetAttribute(csr_sell4s_kernel<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(kS4Smem + kS4HotBytes));
          cudaFuncSetAttribute(csr_sell4s_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(kS4Smem + kS4HotBytes));
          attr = true;
        }
        const int g = (int)std::min<int64_t>(num_sms(), (p.nslice + kS4Warps - 1) / kS4Warps);
        if (p.sell_colh && g_tune[12] == 1) {
          auto k = yrow ? csr_sell4s_kernel<1, 1> : csr_sell4s_kernel<0, 1>;
          SVDSB_LAUNCH_PDL(k, g, kS4Warps * 32, kS4Smem + kS4HotBytes, st, p.rows, p.nslice, p.sell_ptr, p.sell_colh,
                           p.sell_val, p.sell_len, x, y, ldy, (const int *)p.sell_hot, p.sell_nhot);
          return SVDSB_OK;
        }
        auto k = yrow ? csr_sell4s_kernel<1, 0> : csr_sell4s_kernel<0, 0>;
        SVDSB_LAUNCH_PDL(k, g, kS4Warps * 32, kS4Smem, st, p.rows, p.nslice, p.sell_ptr, p.sell_col, p.sell_val,
                         p.sell_len, x, y, ldy, (const int *)nullptr, 0);
        return SVDSB_OK;
      }
      if (p.sell_val && !p.sell_perm) {
        auto k = yrow ? csr_sell4_kernel<1> : csr_sell4_kernel<0>;
        const int g = (int)std::min<int64_t>((p.nslice + 7) / 8, pipe_rows_grid(reinterpret_cast<const void *>(k), 0));
        SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.rows, p.nslice, p.row_ptr, p.sell_ptr, p.sell_col, p.sell_val, x,
                         y, ldy);
        return SVDSB_OK;
      }
    }
    if (ORDER == 0 && b == 4 && xrow && !acc && p.nlong == 0 && p.maxlen <= 129 && rowlane_on() &&
        g_tune[0] == 3) {  // measurement variant (slower on config 4)
      auto k = yrow ? csr_quad4_kernel<1> : csr_quad4_kernel<0>;
      const int g = (int)std::min<int64_t>((p.rows + 63) / 64, pipe_rows_grid(reinterpret_cast<const void *>(k), 0));
      SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.rows, p.row_ptr, p.col, p.val, x, y, ldy);
      return SVDSB_OK;
    }
    if (ORDER == 0 && b == 4 && xrow && !acc && p.nlong == 0 && p.maxlen <= 129 && rowlane_on() &&
        g_tune[0] != 1) {  // 2 (or no sliced-ELL copy); 1 selects the thread-per-row walk
      const size_t sm = (sizeof(double) + sizeof(int)) * kWarpStage * (kTileThreads / 32);
      auto k = yrow ? csr_warprows4_kernel<1> : csr_warprows4_kernel<0>;
      const int g = (int)std::min<int64_t>((p.rows + kTileThreads - 1) / kTileThreads,
                                           pipe_rows_grid(reinterpret_cast<const void *>(k), sm));
      SVDSB_LAUNCH_PDL(k, g, kTileThreads, sm, st, p.rows, p.row_ptr, p.col, p.val, x, y, ldy);
      return SVDSB_OK;
    }
    if (ORDER == 0 && b == 4 && xrow && !acc && p.nlong == 0 && p.maxlen <= 129 && rowlane_on()) {
      const int g = (int)std::min<int64_t>((p.rows + kTileThreads - 1) / kTileThreads, 2 * num_sms() * 4);
      if (yrow)
        SVDSB_LAUNCH_PDL(csr_rowlane4_kernel<1>, g, kTileThreads, 0, st, p.rows, p.row_ptr, p.col, p.val, x, y, ldy);
      else
        SVDSB_LAUNCH_PDL(csr_rowlane4_kernel<0>, g, kTileThreads, 0, st, p.rows, p.row_ptr, p.col, p.val, x, y, ldy);
      return SVDSB_OK;
    }
    // Tune key 16 = 1: long rows (the chunk path) before the short ones for
    // transposed b = 4 parts, so that the long rows' almost sequential walk
    // pulls the operand block into L2 before the short rows' scattered
    // gathers (the two kernels write disjoint rows).  Measured on config 4:
    // no gain (A^T.Y 1366 vs 1336 us), so the default keeps short rows first.
    const bool long_first = p.nlong > 0 && ORDER == 1 && b == 4 && xrow && g_tune[9] != 1 && g_tune[16] == 1;
    if (long_first) {
      SVDSB_LAUNCH_PDL(csr_chunk_kernel, p.nchunk, kTileThreads, 0, st, p.chunk_nz, p.col, p.val, x, ldx, xrow, b,
                       p.chunk_part);
      int tot = p.nlong * b;
      SVDSB_LAUNCH_PDL(csr_long_fixup_kernel, (tot * 32 + 255) / 256, 256, 0, st, p.nlong, p.long_row, p.long_cptr,
                       p.chunk_part, b, y, ldy, yrow, acc, kMaxB);
    }
    bool short_done = false;
    if (ORDER == 1 && b == 4 && xrow && p.ntile > 0 && g_tune[5] == 0) {
      // rows up to a tile on a length-sorted sliced-ELL copy (built on the
      // first uncaptured call); long rows below on the chunk path
      ensure_sell(p, st, true);
      if (p.sell_val && p.sell_perm && p.sell_len && g_tune[7] == 2) {
        if (p.nmid > 0) {  // mid rows: one warp per row (csr_sell4t_kernel with no slices)
          auto k = yrow ? csr_sell4t_kernel<1> : csr_sell4t_kernel<0>;
          const int g = (int)std::min<int64_t>((p.nmid + 7) / 8, pipe_rows_grid(reinterpret_cast<const void *>(k), 0));
          SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.nsell, (int64_t)0, p.sell_perm, p.row_ptr,
                           (const uint8_t *)p.sell_len, p.sell_ptr, p.sell_col, p.sell_val, p.nmid, p.mid_rows, p.col,
                           p.val, x, y, ldy, acc, g_tune[8] == 1, g_tune[14] == 1 ? (unsigned *)nullptr : p.work_ctr);
        }
        if (p.nslice > 0) {
          auto k = yrow ? csr_sell4ts_kernel<1> : csr_sell4ts_kernel<0>;
          static bool attr = false;
          if (!attr) {
            cudaFuncSetAttribute(csr_sell4ts_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT4Smem);
            cudaFuncSetAttribute(csr_sell4ts_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT4Smem);
            attr = true;
          }
          const int g = (int)std::min<int64_t>(num_sms(), (p.nslice + kT4Warps - 1) / kT4Warps);
          SVDSB_LAUNCH_PDL(k, g, kT4Warps * 32, kT4Smem, st, p.nsell, p.nslice, p.sell_perm, p.sell_len, p.sell_ptr,
                           p.sell_col, p.sell_val, x, y, ldy, acc);
        }
        short_done = true;
      } else if (p.sell_val && p.sell_perm && p.sell_len) {
        if (p.nslice + p.nmid > 0) {
          auto k = yrow ? csr_sell4t_kernel<1> : csr_sell4t_kernel<0>;
          const int g = (int)std::min<int64_t>((p.nslice + p.nmid + 7) / 8,
                                               pipe_rows_grid(reinterpret_cast<const void *>(k), 0));
          SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.nsell, p.nslice, p.sell_perm, p.row_ptr,
                           (const uint8_t *)p.sell_len, p.sell_ptr, p.sell_col, p.sell_val, p.nmid, p.mid_rows, p.col,
                           p.val, x, y, ldy, acc, g_tune[8] == 1, g_tune[14] == 1 ? (unsigned *)nullptr : p.work_ctr);
        }
        short_done = true;
      }
    }
    if (short_done) {
    } else if (p.ntile > 0 && xrow) {
      const size_t sm = sizeof(double) * 4 * kTileNnz + sizeof(int) * (kTileRows + 1);
      if (yrow) {
        auto k = csr_tile_pipe_rows_kernel<ORDER, 1>;
        const int g = std::min(p.ntile, pipe_rows_grid(reinterpret_cast<const void *>(k), sm));
        SVDSB_LAUNCH_PDL(k, g, kTileThreads, sm, st, p.ntile, p.tile_info, p.row_ptr, p.col, p.val, x, y, ldy, b, acc);
      } else {
        auto k = csr_tile_pipe_rows_kernel<ORDER, 0>;
        const int g = std::min(p.ntile, pipe_rows_grid(reinterpret_cast<const void *>(k), sm));
        SVDSB_LAUNCH_PDL(k, g, kTileThreads, sm, st, p.ntile, p.tile_info, p.row_ptr, p.col, p.val, x, y, ldy, b, acc);
      }
    } else if (p.ntile > 0) {
      if (acc) {
        set_error("accumulating SpMV needs row-major input");
        return SVDSB_ERR_ARG;
      }
      csr_tile_kernel<ORDER, 0, 1, 4><<<p.ntile, kTileThreads, 0, st>>>(p.tile_r, p.row_ptr, p.col, p.val, x, ldx, y,
                                                                       ldy, b);
      SVDSB_LAUNCHED();
    }
    if (p.nlong > 0 && ORDER == 1 && b == 4 && xrow && g_tune[9] == 1 && ensure_head(p, st)) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(csr_headtile4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * 4 * kHeadTile));
        attr = true;
      }
      const size_t sm = sizeof(double) * 4 * kHeadTile;
      SVDSB_LAUNCH_PDL(csr_headtile4_kernel, p.nhtile, kTileThreads, sm, st, p.nhtile, p.cols, p.htp, p.hpiece,
                       p.col, p.val, x, p.hpart);
      int tot = p.nlong * b;
      SVDSB_LAUNCH_PDL(csr_long_fixup_kernel, (tot * 32 + 255) / 256, 256, 0, st, p.nlong, p.long_row, p.hcptr,
                       p.hpart, b, y, ldy, yrow, acc, 4);
    } else if (p.nlong > 0 && !long_first) {
      SVDSB_LAUNCH_PDL(csr_chunk_kernel, p.nchunk, kTileThreads, 0, st, p.chunk_nz, p.col, p.val, x, ldx, xrow, b,
                       p.chunk_part);
      int tot = p.nlong * b;
      SVDSB_LAUNCH_PDL(csr_long_fixup_kernel, (tot * 32 + 255) / 256, 256, 0, st, p.nlong, p.long_row, p.long_cptr,
                       p.chunk_part, b, y, ldy, yrow, acc, kMaxB);
    }
    return SVDSB_OK;
  }
  if (acc && b != 1) {
    set_error("accumulating SpMV needs block 1 or row-major operands");
    return SVDSB_ERR_ARG;
  }
  for (int c0 = 0; c0 < b; c0 += kMaxB) {
    int bb = std::min(kMaxB, b - c0);
    const double *xc = x + (int64_t)c0 * ldx;
    double *yc = y + (int64_t)c0 * ldy;
    // bulk-copy ring for matrices that stream from HBM; L2-resident ones
    // (configs 1 and 2) are faster on the register-staged pipeline, which
    // runs more CTAs per SM
    if (p.ntile > 0 && bb == 1 && spmv_bulk_on() && 12 * p.nnz >= kBulkMinBytes) {
      const size_t sm = kBulkStages * sizeof(BulkStage) + kBulkStages * sizeof(uint64_t);
      // (the per-row path pays off only for the shortest rows: longer ones
      // serialise a thread's gathers, measured slower on configs 2 and 4)
      auto k = p.maxlen <= 8 ? csr_tile_bulk_kernel<ORDER, 0> : csr_tile_bulk_kernel<ORDER, 2>;
      const int g = std::min(p.ntile, pipe_rows_grid(reinterpret_cast<const void *>(k), sm, true));
      SVDSB_LAUNCH_PDL(k, g, kTileThreads, sm, st, p.ntile, p.tile_info, p.row_ptr, p.col, p.val, xc, yc, acc);
    } else if (p.ntile > 0 && bb == 1) {
      if (p.maxlen <= 8) {
        auto k = csr_tile_pipe_kernel<ORDER, true>;
        const int g = std::min(p.ntile, pipe_grid(reinterpret_cast<const void *>(k)));
        SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.ntile, p.tile_info, p.row_ptr, p.col, p.val, xc, yc, acc);
      } else {
        auto k = csr_tile_pipe_kernel<ORDER, false>;
        const int g = std::min(p.ntile, pipe_grid(reinterpret_cast<const void *>(k)));
        SVDSB_LAUNCH_PDL(k, g, kTileThreads, 0, st, p.ntile, p.tile_info, p.row_ptr, p.col, p.val, xc, yc, acc);
      }
    } else if (p.ntile > 0) {
      csr_tile_kernel<ORDER, 0, 0, 1><<<p.ntile, kTileThreads, 0, st>>>(p.tile_r, p.row_ptr, p.col, p.val, xc, ldx,
                                                                       yc, ldy, bb);
      SVDSB_LAUNCHED();
    }
    if (p.nlong > 0) {
      SVDSB_LAUNCH_PDL(csr_chunk_kernel, p.nchunk, kTileThreads, 0, st, p.chunk_nz, p.col, p.val, xc, ldx, 0, bb,
                       p.chunk_part);
      int tot = p.nlong * bb;
      SVDSB_LAUNCH_PDL(csr_long_fixup_kernel, (tot * 32 + 255) / 256, 256, 0, st, p.nlong, p.long_row, p.long_cptr,
                       p.chunk_part, bb, yc, ldy, 0, acc, kMaxB);
    }
  }
  return SVDSB_OK;
}

// A^T y through the column blocks of A^T (rows of A in [r0_k, r0_{k+1}))
// in ascending order, each block continuing the running sums of the last:
// y blocks stay L2-resident while the Zipf head rows sweep them.
template <int XROW>
static int blocked_adj(const svdsb_csr *a, const double *x, int64_t ldx, double *y, int64_t ldy, int yrow, int b,
                       cudaStream_t st) {
  for (size_t k = 0; k < a->atb.size(); ++k) {
    const int64_t r0 = a->atb_r0[k];
    const double *xk = XROW ? x + r0 * b : x + r0;
    int rc = part_matvec<1>(a->atb[k], xk, ldx, XROW, y, ldy, yrow, b, st, k > 0 ? 1 : 0);
    if (rc) return rc;
  }
  return SVDSB_OK;
}

// ---------------------------------------------------------------- transpose

__global__ void expand_rows_kernel(int64_t m, const int *__restrict__ row_ptr, int *__restrict__ rows) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m) return;
  for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) rows[k] = (int)r;
}

__global__ void iota_kernel(int64_t n, int *__restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int)i;
}

// row_ptr from SORTED keys: row_ptr[c] = number of keys < c, written by the
// thread at the first position whose key is >= c (thread nnz closes the
// tail).  The same values as a histogram + exclusive scan, without the
// histogram's atomics: on config 4 a fifth of the 173 M nonzeros share ten
// columns and the atomic counts took 25 ms.
__global__ void bounds_from_sorted_kernel(int64_t nnz, const int *__restrict__ keys, int nrows,
                                          int *__restrict__ row_ptr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > nnz) return;
  const int lo = i == 0 ? 0 : keys[i - 1] + 1;
  const int hi = i == nnz ? nrows : keys[i];
  for (int c = lo; c <= hi; ++c) row_ptr[c] = (int)i;
}

__global__ void gather_t_kernel(int64_t nnz, const int *__restrict__ perm, const int *__restrict__ rows,
                                const double *__restrict__ val, int *__restrict__ tcol,
                                double *__restrict__ tval) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  int k = perm[i];
  tcol[i] = rows[k];
  tval[i] = val[k];
}

static int bits_for(int64_t n) {
  int b = 1;
  while (b < 63 && ((int64_t)1 << b) < n) ++b;
  return b;
}

static inline unsigned grid1(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// Build at = CSR(A^T) from a (both on device).  Stable LSD radix sort by
// column keeps ascending row order inside each column, which is exactly the
// (col, row) lexsort of from_coo (matio.py:80-81) on a duplicate-free input.
static int build_transpose(const CsrPart &a, CsrPart &at, cudaStream_t st) {
  at.rows = a.cols;
  at.cols = a.rows;
  at.nnz = a.nnz;
  const int64_t nnz = a.nnz;
  SVDSB_CUDA(alloc_pad(&at.row_ptr, at.rows + 1, st));
  SVDSB_CUDA(alloc_pad(&at.col, std::max<int64_t>(nnz, 1), st));
  SVDSB_CUDA(alloc_pad(&at.val, std::max<int64_t>(nnz, 1), st));
  SVDSB_CUDA(cudaMemsetAsync(at.row_ptr, 0, sizeof(int) * (at.rows + 1), st));
  if (nnz > 0) {
    int *rows = nullptr, *idx = nullptr, *keys_out = nullptr, *perm = nullptr;
    SVDSB_CUDA(palloc(&rows, sizeof(int) * nnz, st));
    SVDSB_CUDA(palloc(&idx, sizeof(int) * nnz, st));
    SVDSB_CUDA(palloc(&keys_out, sizeof(int) * nnz, st));
    SVDSB_CUDA(palloc(&perm, sizeof(int) * nnz, st));
    expand_rows_kernel<<<grid1(a.rows), 256, 0, st>>>(a.rows, a.row_ptr, rows);
    SVDSB_LAUNCHED();
    iota_kernel<<<grid1(nnz), 256, 0, st>>>(nnz, idx);
    SVDSB_LAUNCHED();
    size_t tmp_bytes = 0;
    int nbits = bits_for(a.cols);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, a.col, keys_out, idx, perm, (int)nnz, 0, nbits, st);
    void *tmp = nullptr;
    SVDSB_CUDA(palloc(&tmp, tmp_bytes, st));
    SVDSB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, a.col, keys_out, idx, perm, (int)nnz, 0,
                                               nbits, st));
    bump_launches();
    gather_t_kernel<<<grid1(nnz), 256, 0, st>>>(nnz, perm, rows, a.val, at.col, at.val);
    SVDSB_LAUNCHED();
    // row_ptr of A^T from the sorted column keys
    bounds_from_sorted_kernel<<<grid1(nnz + 1), 256, 0, st>>>(nnz, keys_out, (int)at.rows, at.row_ptr);
    SVDSB_LAUNCHED();
    tmark("T launch");
    SVDSB_CUDA(cudaStreamSynchronize(st));
    tmark("T sync");
    pfree(rows, st);
    pfree(idx, st);
    pfree(keys_out, st);
    pfree(perm, st);
    pfree(tmp, st);
  }
  at.host_row_ptr.resize(at.rows + 1);
  SVDSB_CUDA(cudaMemcpyAsync(at.host_row_ptr.data(), at.row_ptr, sizeof(int) * (at.rows + 1),
                             cudaMemcpyDeviceToHost, st));
  SVDSB_CUDA(cudaStreamSynchronize(st));
  tmark("T row_ptr d2h");
  return build_partition(at, st);
}

// ---------------------------------------------------------------- COO build

// Sort key of each triplet, with the from_coo range check (matio.py:41-52)
// folded in: an out-of-range index raises *bad and gets key 0, so nothing
// downstream indexes outside the row counters before the caller reads *bad.
__global__ void coo_keys_kernel(int64_t nt, int64_t m, int64_t n, const int64_t *__restrict__ r,
                                const int64_t *__restrict__ c, unsigned long long *__restrict__ key,
                                int *__restrict__ idx, int *__restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const int64_t ri = r[i], cj = c[i];
  const bool rok = ri >= 0 && ri < m, cok = cj >= 0 && cj < n;
  const bool ok = rok && cok;
  if (!ok) atomicOr(bad, (rok ? 0 : 1) | (cok ? 0 : 2));
  key[i] = ok ? (unsigned long long)(ri * n + cj) : 0ull;
  idx[i] = (int)i;
}

__global__ void coo_first_kernel(int64_t nt, const unsigned long long *__restrict__ key, int *__restrict__ first) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  first[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// seg[i] = exclusive scan of first; segment s starts where first==1
__global__ void coo_sum_kernel(int64_t nt, int64_t n, const unsigned long long *__restrict__ key,
                               const int *__restrict__ perm, const int *__restrict__ first,
                               const int *__restrict__ seg, const double *__restrict__ vals,
                               int *__restrict__ col, double *__restrict__ val, int *__restrict__ rowcnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt || !first[i]) return;
  // np.add.at into zeros, ascending input order (stable sort keeps it)
  double s = 0.0;
  int64_t j = i;
  do {
    s = __dadd_rn(s, vals[perm[j]]);
    ++j;
  } while (j < nt && !first[j]);
  int o = seg[i];
  unsigned long long k = key[i];
  int64_t r = (int64_t)(k / (unsigned long long)n);
  col[o] = (int)(k - (unsigned long long)r * (unsigned long long)n);
  val[o] = s;
  atomicAdd(rowcnt + r, 1);
}


}  // namespace svdsb

using namespace svdsb;

extern "C" {

int svdsb_csr_destroy(svdsb_csr *a) {
  if (!a) return SVDSB_OK;
  cudaDeviceSynchronize();
  free_part(a->a);
  free_part(a->at);
  for (auto &p : a->atb) free_part(p);
  for (double *sp : a->scratch) pfree(sp, nullptr);  // pool memory: cheap to return
  delete a;
  return SVDSB_OK;
}

int svdsb_csr_shape(const svdsb_csr *a, int64_t *m, int64_t *n, int64_t *nnz) {
  SVDSB_CHECK_ARG(a != nullptr, "svdsb_csr_shape: NULL handle");
  if (m) *m = a->a.rows;
  if (n) *n = a->a.cols;
  if (nnz) *nnz = a->a.nnz;
  return SVDSB_OK;
}

int svdsb_csr_layout_info(const svdsb_csr *a, int key, int64_t *out) {
  SVDSB_CHECK_ARG(a != nullptr && out != nullptr, "svdsb_csr_layout_info: NULL argument");
  switch (key) {
    case 0: *out = a->a.sell_val ? a->a.nslice : 0; break;
    case 1: *out = a->a.sell_colh ? a->a.sell_nhot : 0; break;
    case 2: *out = (int64_t)a->atb.size(); break;
    default: set_error("svdsb_csr_layout_info: unknown key %d", key); return SVDSB_ERR_ARG;
  }
  return SVDSB_OK;
}

// Column blocks of A^T for tall matrices whose A^T gathers would sweep a y
// block larger than L2 (config 4: m = 10 M rows).  Same nonzeros, regrouped
// by row block of A; built once on device.
constexpr int64_t kBlockRows = 2 << 20;   // 2 Mi rows: y block <= 64 MB at b = 4

__global__ void seg_bounds_kernel(int64_t n, const int *__restrict__ rp, const int *__restrict__ col, int r0, int r1,
                                  int *__restrict__ lo_out, int *__restrict__ len_out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  auto lower = [&](int key) {
    int lo = rp[j], hi = rp[j + 1];
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (col[mid] < key)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  int a = lower(r0), b = lower(r1);
  lo_out[j] = a;
  len_out[j] = b - a;
}

// One thread per nonzero of the block (a thread per row serialised the
// Zipf head rows: 1 s for config 4): the row of output q is the last j
// with rpk[j] <= q.
__global__ void seg_copy_kernel(int64_t n, int64_t nnzk, const int *__restrict__ col, const double *__restrict__ val,
                                const int *__restrict__ lo, const int *__restrict__ rpk, int r0, int *__restrict__ colk,
                                double *__restrict__ valk) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnzk; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = n;  // rpk[a] <= q < rpk[b]
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (rpk[mid] <= q)
        a = mid;
      else
        b = mid;
    }
    const int64_t src = lo[a] + (q - rpk[a]);
    colk[q] = col[src] - r0;
    valk[q] = val[src];
  }
}

static int build_blocked_transpose(svdsb_csr *h, cudaStream_t st) {
  const CsrPart &at = h->at;
  const int64_t m = h->a.rows, n = h->a.cols;
  int64_t block_rows = kBlockRows;
  bool forced = false;
  if (const char *env = getenv("SVDSB_T_BLOCK_ROWS")) {  // tuning / test knob
    block_rows = std::max<int64_t>(1, atoll(env));
    forced = true;
  }
  if (!forced && !(m > block_rows && m >= 4 * n)) return SVDSB_OK;
  StreamTemps temps{st, {}};
  int *lo = nullptr, *len = nullptr;
  SVDSB_CUDA(temps.get(&lo, sizeof(int) * (n + 1)));
  SVDSB_CUDA(temps.get(&len, sizeof(int) * (n + 1)));
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, len, lo, (int)(n + 1), st);
  void *scan_tmp = nullptr;
  SVDSB_CUDA(temps.get(&scan_tmp, scan_bytes));
  for (int64_t r0 = 0; r0 < m; r0 += block_rows) {
    const int64_t r1 = std::min(m, r0 + block_rows);
    CsrPart p;
    struct PartGuard {  // a block that fails half-built is freed here
      CsrPart *p;
      ~PartGuard() {
        if (p) {
          cudaDeviceSynchronize();
          free_part(*p);
        }
      }
    } pguard{&p};
    p.rows = n;
    p.cols = r1 - r0;
    SVDSB_CUDA(alloc_pad(&p.row_ptr, n + 1, st));
    SVDSB_CUDA(cudaMemsetAsync(len + n, 0, sizeof(int), st));
    seg_bounds_kernel<<<grid1(n), 256, 0, st>>>(n, at.row_ptr, at.col, (int)r0, (int)r1, lo, len);
    SVDSB_LAUNCHED();
    SVDSB_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, len, p.row_ptr, (int)(n + 1), st));
    bump_launches();
    p.host_row_ptr.resize(n + 1);
    SVDSB_CUDA(cudaMemcpyAsync(p.host_row_ptr.data(), p.row_ptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st));
    SVDSB_CUDA(cudaStreamSynchronize(st));
    p.nnz = p.host_row_ptr[n];
    SVDSB_CUDA(alloc_pad(&p.col, std::max<int64_t>(p.nnz, 1), st));
    SVDSB_CUDA(alloc_pad(&p.val, std::max<int64_t>(p.nnz, 1), st));
    if (p.nnz > 0) {
      seg_copy_kernel<<<(unsigned)std::min<int64_t>((p.nnz + 255) / 256, 16 * num_sms()), 256, 0, st>>>(
          n, p.nnz, at.col, at.val, lo, p.row_ptr, (int)r0, p.col, p.val);
      SVDSB_LAUNCHED();
    }
    int rc = build_partition(p, st);
    if (rc) return rc;
    pguard.p = nullptr;
    h->atb.push_back(std::move(p));
    h->atb_r0.push_back(r0);
  }
  SVDSB_CUDA(cudaStreamSynchronize(st));
  return SVDSB_OK;
}

static int finish_create(svdsb_csr *h, int flags, cudaStream_t st) {
  tmark("assembled");
  int rc = build_partition(h->a, st);
  tmark("partition A");
  if (rc) return rc;
  if (flags & SVDSB_CSR_TRANSPOSE) {
    rc = build_transpose(h->a, h->at, st);
    tmark("transpose");
    if (rc) return rc;
    h->has_t = true;
    rc = build_blocked_transpose(h, st);
    tmark("blocked transpose");
    if (rc) return rc;
  }
  SVDSB_CUDA(cudaStreamSynchronize(st));
  tmark("final sync");
  return SVDSB_OK;
}

int svdsb_csr_create_host(svdsb_ctx *ctx, int64_t m, int64_t n, int64_t nnz, const int64_t *row_ptr_host,
                          const int64_t *col_idx_host, const double *values_host, int flags, void *stream,
                          svdsb_csr **out) {
  (void)ctx;
  SVDSB_CHECK_ARG(out != nullptr, "svdsb_csr_create_host: out is NULL");
  SVDSB_CHECK_ARG(m >= 0 && n >= 0, "negative matrix dimension");
  if (m >= INT32_MAX || n >= INT32_MAX || nnz >= INT32_MAX) {
    set_error("matrix exceeds the int32-indexed device layout (m=%lld n=%lld nnz=%lld)", (long long)m,
              (long long)n, (long long)nnz);
    return SVDSB_ERR_RANGE;
  }
  SVDSB_CHECK_ARG(row_ptr_host != nullptr, "row_ptr is NULL");
  // validation mirrors SparseMatrixCsr.__init__ (matio.py:41-52)
  SVDSB_CHECK_ARG(row_ptr_host[0] == 0 && row_ptr_host[m] == nnz, "row_ptr endpoints inconsistent with nnz");
  std::vector<int> rp(m + 1), ci(nnz);
  for (int64_t r = 0; r <= m; ++r) {
    if (r > 0 && row_ptr_host[r] < row_ptr_host[r - 1]) {
      set_error("row_ptr must be nondecreasing");
      return SVDSB_ERR_ARG;
    }
    rp[r] = (int)row_ptr_host[r];
  }
  for (int64_t k = 0; k < nnz; ++k) {
    int64_t c = col_idx_host[k];
    if (c < 0 || c >= n) {
      set_error("column index out of range");
      return SVDSB_ERR_ARG;
    }
    ci[k] = (int)c;
  }
  cudaStream_t st = as_stream(stream);
  svdsb_csr *h = new svdsb_csr();
  cudaGetDevice(&h->device);
  h->has_t = false;
  CsrPart &p = h->a;
  p.rows = m;
  p.cols = n;
  p.nnz = nnz;
  int rc;
  if ((rc = upload(&p.row_ptr, rp, st)) || (rc = upload(&p.col, ci, st))) {
    svdsb_csr_destroy(h);
    return rc;
  }
  if (alloc_pad(&p.val, std::max<int64_t>(nnz, 1), st) != cudaSuccess) {
    svdsb_csr_destroy(h);
    set_error("cudaMalloc values failed");
    return SVDSB_ERR_ALLOC;
  }
  if (nnz) cudaMemcpyAsync(p.val, values_host, sizeof(double) * nnz, cudaMemcpyHostToDevice, st);
  p.host_row_ptr = std::move(rp);
  rc = finish_create(h, flags, st);
  if (rc) {
    svdsb_csr_destroy(h);
    return rc;
  }
  *out = h;
  return SVDSB_OK;
}

int svdsb_csr_create_coo_device(svdsb_ctx *ctx, int64_t m, int64_t n, int64_t nt, const int64_t *rows,
                                const int64_t *cols, const double *vals, int flags, void *stream,
                                svdsb_csr **out) {
  return svdsb_csr_create_coo_device_ev(ctx, m, n, nt, rows, cols, vals, nullptr, flags, stream, out);
}

int svdsb_csr_create_coo_device_ev(svdsb_ctx *ctx, int64_t m, int64_t n, int64_t nt, const int64_t *rows,
                                   const int64_t *cols, const double *vals, void *vals_ready, int flags,
                                   void *stream, svdsb_csr **out) {
  (void)ctx;
  SVDSB_CHECK_ARG(out != nullptr, "svdsb_csr_create_coo_device: out is NULL");
  SVDSB_CHECK_ARG(m >= 0 && n >= 0 && nt >= 0, "negative size");
  if (m >= INT32_MAX || n >= INT32_MAX || nt >= INT32_MAX) {
    set_error("COO exceeds the int32-indexed device layout");
    return SVDSB_ERR_RANGE;
  }
  cudaStream_t st = as_stream(stream);
  CreateTrace trace;
  g_trace = &trace;
  struct Unset { ~Unset() { g_trace = nullptr; } } unset_trace;
  // every early return below frees the handle and the temporaries
  StreamTemps tmp_bufs{st, {}};
  struct Guard {
    svdsb_csr *h;
    ~Guard() {
      if (h) svdsb_csr_destroy(h);
    }
  } guard{new svdsb_csr()};
  svdsb_csr *h = guard.h;
  cudaGetDevice(&h->device);
  h->has_t = false;
  CsrPart &p = h->a;
  p.rows = m;
  p.cols = n;
  SVDSB_CUDA(alloc_pad(&p.row_ptr, m + 1, st));
  SVDSB_CUDA(cudaMemsetAsync(p.row_ptr, 0, sizeof(int) * (m + 1), st));
  int64_t nnz = 0;
  if (nt > 0) {
    unsigned long long *key = nullptr, *key_s = nullptr;
    int *idx = nullptr, *perm = nullptr, *first = nullptr, *seg = nullptr, *rowcnt = nullptr;
    SVDSB_CUDA(tmp_bufs.get(&key, 8 * nt));
    SVDSB_CUDA(tmp_bufs.get(&key_s, 8 * nt));
    SVDSB_CUDA(tmp_bufs.get(&idx, 4 * nt));
    SVDSB_CUDA(tmp_bufs.get(&perm, 4 * nt));
    SVDSB_CUDA(tmp_bufs.get(&first, 4 * nt));
    SVDSB_CUDA(tmp_bufs.get(&seg, 4 * (nt + 1)));
    SVDSB_CUDA(tmp_bufs.get(&rowcnt, 4 * (m + 1)));
    int *bad = nullptr;
    SVDSB_CUDA(tmp_bufs.get(&bad, 4));
    SVDSB_CUDA(cudaMemsetAsync(rowcnt, 0, 4 * (m + 1), st));
    SVDSB_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    tmark("alloc");
    coo_keys_kernel<<<grid1(nt), 256, 0, st>>>(nt, m, n, rows, cols, key, idx, bad);
    SVDSB_LAUNCHED();
    int nbits = bits_for(std::max<int64_t>(m * n, 2));
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key_s, idx, perm, (int)nt, 0, nbits, st);
    void *tmp = nullptr;
    SVDSB_CUDA(tmp_bufs.get(&tmp, tb));
    SVDSB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key_s, idx, perm, (int)nt, 0, nbits, st));
    bump_launches();
    coo_first_kernel<<<grid1(nt), 256, 0, st>>>(nt, key_s, first);
    SVDSB_LAUNCHED();
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, first, seg, (int)nt, st);
    void *stmp = nullptr;
    SVDSB_CUDA(tmp_bufs.get(&stmp, sb));
    SVDSB_CUDA(cub::DeviceScan::ExclusiveSum(stmp, sb, first, seg, (int)nt, st));
    bump_launches();
    int last_seg = 0, last_first = 0, any_bad = 0;
    tmark("sort+scan launch");
    SVDSB_CUDA(cudaMemcpyAsync(&last_seg, seg + nt - 1, 4, cudaMemcpyDeviceToHost, st));
    SVDSB_CUDA(cudaMemcpyAsync(&last_first, first + nt - 1, 4, cudaMemcpyDeviceToHost, st));
    SVDSB_CUDA(cudaMemcpyAsync(&any_bad, bad, 4, cudaMemcpyDeviceToHost, st));
    SVDSB_CUDA(cudaStreamSynchronize(st));
    if (any_bad) {  // the reference's messages and order of checks (matio.py:74-78)
      set_error((any_bad & 1) ? "row index out of range" : "column index out of range");
      return SVDSB_ERR_ARG;
    }
    nnz = (int64_t)last_seg + last_first;
    tmark("sync nnz");
    SVDSB_CUDA(alloc_pad(&p.col, std::max<int64_t>(nnz, 1), st));
    SVDSB_CUDA(alloc_pad(&p.val, std::max<int64_t>(nnz, 1), st));
    // the values are first needed here: a copy still in flight on another
    // stream has had the key build, sort and scans to finish
    if (vals_ready != nullptr) SVDSB_CUDA(cudaStreamWaitEvent(st, reinterpret_cast<cudaEvent_t>(vals_ready), 0));
    coo_sum_kernel<<<grid1(nt), 256, 0, st>>>(nt, n, key_s, perm, first, seg, vals, p.col, p.val, rowcnt);
    SVDSB_LAUNCHED();
    size_t sb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb2, rowcnt, p.row_ptr, (int)(m + 1), st);
    void *stmp2 = nullptr;
    SVDSB_CUDA(tmp_bufs.get(&stmp2, sb2));
    SVDSB_CUDA(cub::DeviceScan::ExclusiveSum(stmp2, sb2, rowcnt, p.row_ptr, (int)(m + 1), st));
    bump_launches();
    tmark("sum+scan launch");
    SVDSB_CUDA(cudaStreamSynchronize(st));
    tmark("sum sync");
  } else {
    SVDSB_CUDA(palloc(&p.col, 4, st));
    SVDSB_CUDA(palloc(&p.val, 8, st));
  }
  p.nnz = nnz;
  p.host_row_ptr.resize(m + 1);
  tmark("free temps");
  SVDSB_CUDA(cudaMemcpyAsync(p.host_row_ptr.data(), p.row_ptr, 4 * (m + 1), cudaMemcpyDeviceToHost, st));
  SVDSB_CUDA(cudaStreamSynchronize(st));
  tmark("row_ptr d2h");
  int rc = finish_create(h, flags, st);
  if (rc) return rc;  // the guard destroys h
  guard.h = nullptr;
  *out = h;
  return SVDSB_OK;
}

int svdsb_csr_export_host(const svdsb_csr *a, int transpose, int64_t *row_ptr_host, int64_t *col_idx_host,
                          double *values_host) {
  SVDSB_CHECK_ARG(a != nullptr, "NULL handle");
  SVDSB_CHECK_ARG(!transpose || a->has_t, "transpose was not built");
  const CsrPart &p = transpose ? a->at : a->a;
  std::vector<int> rp(p.rows + 1), ci(p.nnz);
  SVDSB_CUDA(cudaMemcpy(rp.data(), p.row_ptr, 4 * (p.rows + 1), cudaMemcpyDeviceToHost));
  if (p.nnz) {
    SVDSB_CUDA(cudaMemcpy(ci.data(), p.col, 4 * p.nnz, cudaMemcpyDeviceToHost));
    SVDSB_CUDA(cudaMemcpy(values_host, p.val, 8 * p.nnz, cudaMemcpyDeviceToHost));
  }
  for (int64_t i = 0; i <= p.rows; ++i) row_ptr_host[i] = rp[i];
  for (int64_t k = 0; k < p.nnz; ++k) col_idx_host[k] = ci[k];
  return SVDSB_OK;
}

int svdsb_csr_device_arrays(const svdsb_csr *a, int transpose, const int **row_ptr, const int **col,
                            const double **val) {
  SVDSB_CHECK_ARG(a != nullptr, "NULL handle");
  SVDSB_CHECK_ARG(!transpose || a->has_t, "transpose was not built");
  const CsrPart &p = transpose ? a->at : a->a;
  if (row_ptr) *row_ptr = p.row_ptr;
  if (col) *col = p.col;
  if (val) *val = p.val;
  return SVDSB_OK;
}

static double *scratch_get(const svdsb_csr *ca, int slot, size_t n) {
  svdsb_csr *a = const_cast<svdsb_csr *>(ca);
  if (a->scratch_cap[slot] < n) {
    // stream-ordered pool memory (legacy stream: the handle may be used on
    // any stream after this call returns; the matrix destructor synchronises)
    if (a->scratch[slot]) cudaDeviceSynchronize();
    pfree(a->scratch[slot], nullptr);
    a->scratch[slot] = nullptr;
    a->scratch_cap[slot] = 0;
    if (palloc(&a->scratch[slot], n * sizeof(double), nullptr) != cudaSuccess) return nullptr;
    cudaStreamSynchronize(nullptr);
    a->scratch_cap[slot] = n;
  }
  return a->scratch[slot];
}

static int pack(const double *x, int64_t rows, int64_t ldx, int b, double *xr, cudaStream_t st) {
  int64_t tot = rows * b;
  if (tot == 0) return SVDSB_OK;
  pack_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(rows, b, x, ldx, xr);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

static inline bool packed_block(int b) { return b >= 2 && b <= 4; }

static int unpack(const double *xr, int64_t rows, int b, double *y, int64_t ldy, cudaStream_t st) {
  const int64_t tot = rows * b;
  if (tot == 0) return SVDSB_OK;
  unpack_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(rows, b, xr, y, ldy);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

// Column-blocked A^T product of a packed (row-major) operand into a
// column-major result.  svdsb_tune_set key 13 = 1 keeps the running sums of
// the blocks in a row-major scratch block (one 32-byte access per row and
// block instead of four scattered 8-byte ones) and unpacks once at the end:
// measured 25 us SLOWER on config 4 (1362 vs 1337 us per product) -- the
// kernels are bound by the gathers' L1 wavefronts (one per nonzero), the
// read-modify-write is a few percent of them and the unpack costs more than
// it saves.  Same sums in the same order either way, bit-identical.
static int blocked_adj_packed(const svdsb_csr *a, const double *xr, int b, double *y, int64_t ldy,
                              cudaStream_t st) {
  if (g_tune[13] != 1) return blocked_adj<1>(a, xr, b, y, ldy, 0, b, st);
  double *yr = scratch_get(a, 2, (size_t)a->at.rows * b);
  if (!yr) {
    set_error("blocked A^T product: scratch allocation failed");
    return SVDSB_ERR_ALLOC;
  }
  int rc = blocked_adj<1>(a, xr, b, yr, b, 1, b, st);
  if (rc) return rc;
  return unpack(yr, a->at.rows, b, y, ldy, st);
}

static int pack_pad(const double *x, int64_t rows, int64_t ldx, int b, int bp, double *xr, cudaStream_t st) {
  const int64_t tot = rows * bp;
  if (tot == 0) return SVDSB_OK;
  pack_pad_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(rows, b, bp, x, ldx, xr);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

static int unpack_pad(const double *xr, int64_t rows, int b, int bp, double *y, int64_t ldy, cudaStream_t st) {
  const int64_t tot = rows * b;
  if (tot == 0) return SVDSB_OK;
  unpack_pad_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(rows, b, bp, xr, y, ldy);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

// 2- and 3-column products of short-row matrices go through the 4-column
// sliced-ELL kernels with a zero-padded operand (a zero column changes no
// other column's bits; a 24-byte gather costs the same 32-byte sector).
static inline bool pad_to4(const svdsb_csr *a, int b) {
  return (b == 2 || b == 3) && a->a.nlong == 0 && a->a.maxlen <= 129 && a->has_t && a->at.ntile > 0 &&
         g_tune[6] == 0;
}
// Width of the next column chunk of a wide block: fours, with the
// remainder spread so no chunk is a lone column (5 -> 3+2, 6 -> 3+3,
// 9 -> 4+3+2, ...) while at least 4 remain.
static inline int chunk_cols(int left) {
  if (left <= 4) return left;
  if (left == 5) return 3;
  if (left == 6) return 3;
  if (left == 7) return 4;
  return 4;
}

int svdsb_matvec(svdsb_ctx *ctx, const svdsb_csr *a, int transpose, const double *x, int64_t ldx, double *y,
                 int64_t ldy, int block, void *stream) {
  (void)ctx;
  SVDSB_CHECK_ARG(a != nullptr, "svdsb_matvec: NULL handle");
  SVDSB_CHECK_ARG(block >= 0, "svdsb_matvec: negative block");
  if (block == 0) return SVDSB_OK;
  cudaStream_t st = as_stream(stream);
  SVDSB_CHECK_ARG(!transpose || a->has_t, "svdsb_matvec: transpose requested but CSR(A^T) was not built");
  const CsrPart &p = transpose ? a->at : a->a;
  SVDSB_CHECK_ARG(ldx >= p.cols && ldy >= p.rows, "svdsb_matvec: leading dimension too small");
  if (block > 4) {
    // wide blocks (initial basis, soft-lock finalisation) in chunks of at
    // most four columns through the packed kernels: every column's sum order
    // is independent of the block width, so the bits are those of the
    // narrow products
    for (int c0 = 0; c0 < block;) {
      const int nb = chunk_cols(block - c0);
      int rc = svdsb_matvec(ctx, a, transpose, x + c0 * ldx, ldx, y + c0 * ldy, ldy, nb, stream);
      if (rc) return rc;
      c0 += nb;
    }
    return SVDSB_OK;
  }
  if (pad_to4(a, block)) {
    double *xr = scratch_get(a, 0, (size_t)p.cols * 4);
    double *yr = scratch_get(a, 2, (size_t)p.rows * 4);
    if (!xr || !yr) {
      set_error("svdsb_matvec: scratch allocation failed");
      return SVDSB_ERR_ALLOC;
    }
    int rc = pack_pad(x, p.cols, ldx, block, 4, xr, st);
    if (rc) return rc;
    if (transpose && !a->atb.empty())
      rc = blocked_adj<1>(a, xr, 4, yr, 4, 1, 4, st);
    else
      rc = transpose ? part_matvec<1>(p, xr, 4, 1, yr, 4, 1, 4, st) : part_matvec<0>(p, xr, 4, 1, yr, 4, 1, 4, st);
    if (rc) return rc;
    return unpack_pad(yr, p.rows, block, 4, y, ldy, st);
  }
  if (packed_block(block)) {
    double *xr = scratch_get(a, 0, (size_t)p.cols * block);
    if (!xr) {
      set_error("svdsb_matvec: scratch allocation failed");
      return SVDSB_ERR_ALLOC;
    }
    int rc = pack(x, p.cols, ldx, block, xr, st);
    if (rc) return rc;
    if (transpose && !a->atb.empty()) return blocked_adj_packed(a, xr, block, y, ldy, st);
    return transpose ? part_matvec<1>(p, xr, block, 1, y, ldy, 0, block, st)
                     : part_matvec<0>(p, xr, block, 1, y, ldy, 0, block, st);
  }
  if (transpose && block == 1 && !a->atb.empty()) return blocked_adj<0>(a, x, ldx, y, ldy, 0, 1, st);
  return transpose ? part_matvec<1>(p, x, ldx, 0, y, ldy, 0, block, st)
                   : part_matvec<0>(p, x, ldx, 0, y, ldy, 0, block, st);
}

int svdsb_apply_normal(svdsb_ctx *ctx, const svdsb_csr *a, int side, const double *x, int64_t ldx, double *y,
                       int64_t ldy, int block, double *tmp, int64_t ldtmp, void *stream) {
  SVDSB_CHECK_ARG(a != nullptr && a->has_t, "svdsb_apply_normal: needs CSR(A) and CSR(A^T)");
  SVDSB_CHECK_ARG(side == 0 || side == 1, "svdsb_apply_normal: side must be 0 or 1");
  if (block == 0) return SVDSB_OK;
  cudaStream_t st = as_stream(stream);
  const CsrPart &first = side == 0 ? a->a : a->at;    // inner product
  const CsrPart &second = side == 0 ? a->at : a->a;
  if (block > 4) {  // as svdsb_matvec: chunks of at most four columns
    for (int c0 = 0; c0 < block;) {
      const int nb = chunk_cols(block - c0);
      int rc = svdsb_apply_normal(ctx, a, side, x + c0 * ldx, ldx, y + c0 * ldy, ldy, nb, tmp, ldtmp, stream);
      if (rc) return rc;
      c0 += nb;
    }
    return SVDSB_OK;
  }
  if (pad_to4(a, block)) {
    double *xr = scratch_get(a, 0, (size_t)first.cols * 4);
    double *tr = scratch_get(a, 1, (size_t)first.rows * 4);
    double *yr = scratch_get(a, 2, (size_t)second.rows * 4);
    if (!xr || !tr || !yr) {
      set_error("svdsb_apply_normal: scratch allocation failed");
      return SVDSB_ERR_ALLOC;
    }
    int rc = pack_pad(x, first.cols, ldx, block, 4, xr, st);
    if (rc) return rc;
    rc = side == 0 ? part_matvec<0>(first, xr, 4, 1, tr, 4, 1, 4, st) : part_matvec<1>(first, xr, 4, 1, tr, 4, 1, 4, st);
    if (rc) return rc;
    if (side == 0 && !a->atb.empty())
      rc = blocked_adj<1>(a, tr, 4, yr, 4, 1, 4, st);
    else
      rc = side == 0 ? part_matvec<1>(second, tr, 4, 1, yr, 4, 1, 4, st)
                     : part_matvec<0>(second, tr, 4, 1, yr, 4, 1, 4, st);
    if (rc) return rc;
    return unpack_pad(yr, second.rows, block, 4, y, ldy, st);
  }
  if (packed_block(block)) {
    // x packed once; the inner result stays row-major for the second gather
    double *xr = scratch_get(a, 0, (size_t)first.cols * block);
    double *tr = scratch_get(a, 1, (size_t)first.rows * block);
    if (!xr || !tr) {
      set_error("svdsb_apply_normal: scratch allocation failed");
      return SVDSB_ERR_ALLOC;
    }
    int rc = pack(x, first.cols, ldx, block, xr, st);
    if (rc) return rc;
    rc = side == 0 ? part_matvec<0>(first, xr, block, 1, tr, block, 1, block, st)
                   : part_matvec<1>(first, xr, block, 1, tr, block, 1, block, st);
    if (rc) return rc;
    if (side == 0 && !a->atb.empty()) return blocked_adj_packed(a, tr, block, y, ldy, st);
    return side == 0 ? part_matvec<1>(second, tr, block, 1, y, ldy, 0, block, st)
                     : part_matvec<0>(second, tr, block, 1, y, ldy, 0, block, st);
  }
  SVDSB_CHECK_ARG(tmp != nullptr && ldtmp >= first.rows, "svdsb_apply_normal: tmp too small");
  int rc;
  if (side == 0) {
    if ((rc = svdsb_matvec(ctx, a, 0, x, ldx, tmp, ldtmp, block, stream))) return rc;
    return svdsb_matvec(ctx, a, 1, tmp, ldtmp, y, ldy, block, stream);
  }
  if ((rc = svdsb_matvec(ctx, a, 1, x, ldx, tmp, ldtmp, block, stream))) return rc;
  return svdsb_matvec(ctx, a, 0, tmp, ldtmp, y, ldy, block, stream);
}

int svdsb_apply_augmented(svdsb_ctx *ctx, const svdsb_csr *a, const double *x, int64_t ldx, double *y,
                          int64_t ldy, int block, void *stream) {
  SVDSB_CHECK_ARG(a != nullptr, "NULL handle");
  const int64_t n = a->a.cols;
  int rc;
  // y[:n] = A^T x[n:] ; y[n:] = A x[:n]
  if ((rc = svdsb_matvec(ctx, a, 1, x + n, ldx, y, ldy, block, stream))) return rc;
  return svdsb_matvec(ctx, a, 0, x, ldx, y + n, ldy, block, stream);
}

}  // extern "C"

// ---------------------------------------------------------------- precond

namespace svdsb {

// d[r] = sum over row r of v*v, left to right (np.bincount order over the
// rows of the chosen orientation).
__global__ void row_sq_kernel(int64_t rows, const int *__restrict__ rp, const double *__restrict__ val,
                              double *__restrict__ d) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int k = rp[r]; k < rp[r + 1]; ++k) {
    double v = val[k];
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  d[r] = s;
}

__global__ void max_kernel(int64_t n, const double *__restrict__ d, double *__restrict__ out,
                           unsigned int *ticket, double *partials) {
  __shared__ double red[8];
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, d[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = fmax(mm, red[w]);
    partials[blockIdx.x] = mm;
  }
  if (last_cta(ticket) && threadIdx.x == 0) {
    double mm = partials[0];
    for (unsigned b = 1; b < gridDim.x; ++b) mm = fmax(mm, partials[b]);
    *out = mm;
  }
}

__global__ void clamp_kernel(int64_t n, double *__restrict__ d, const double *__restrict__ mx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double f = __dmul_rn(kEps, *mx);
  d[i] = fmax(d[i], f);
}

__global__ void diag_solve_kernel(int64_t dim, int b, const double *__restrict__ d, const double *x, int64_t ldx,
                                  double *y, int64_t ldy) {
  pdl_wait();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= dim) return;
  double di = d[i];
  for (int c = 0; c < b; ++c) y[i + c * ldy] = __ddiv_rn(x[i + c * ldx], di);
}

}  // namespace svdsb

extern "C" {

int svdsb_precond_diag(svdsb_ctx *ctx, const svdsb_csr *a, int side, double *d, void *stream) {
  SVDSB_CHECK_ARG(ctx && a && d, "svdsb_precond_diag: NULL argument");
  SVDSB_CHECK_ARG(side == 0 || side == 1, "side must be 0 (cols) or 1 (rows)");
  SVDSB_CHECK_ARG(a->a.nnz > 0, "empty matrix has no usable diagonal");
  const CsrPart *p;
  if (side == 0) {
    SVDSB_CHECK_ARG(a->has_t, "column norms need CSR(A^T)");
    p = &a->at;
  } else {
    p = &a->a;
  }
  cudaStream_t st = as_stream(stream);
  row_sq_kernel<<<grid1(p->rows), 256, 0, st>>>(p->rows, p->row_ptr, p->val, d);
  SVDSB_LAUNCHED();
  int g = (int)std::min<int64_t>(grid1(p->rows), 2 * num_sms());
  double *mx = ctx->partials + kMaxPartials - 1;
  max_kernel<<<g, 256, 0, st>>>(p->rows, d, mx, take_ticket(ctx), ctx->partials);
  SVDSB_LAUNCHED();
  clamp_kernel<<<grid1(p->rows), 256, 0, st>>>(p->rows, d, mx);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_row_sq(svdsb_ctx *ctx, const svdsb_csr *a, int side, double *d, void *stream) {
  SVDSB_CHECK_ARG(ctx && a && d, "svdsb_row_sq: NULL argument");
  SVDSB_CHECK_ARG(side == 0 || side == 1, "side must be 0 (cols) or 1 (rows)");
  SVDSB_CHECK_ARG(side == 1 || a->has_t, "column norms need CSR(A^T)");
  const CsrPart *p = side == 0 ? &a->at : &a->a;
  if (p->rows == 0) return SVDSB_OK;
  row_sq_kernel<<<grid1(p->rows), 256, 0, as_stream(stream)>>>(p->rows, p->row_ptr, p->val, d);
  SVDSB_LAUNCHED();
  return SVDSB_OK;
}

int svdsb_diag_solve(int64_t dim, const double *d, const double *x, int64_t ldx, double *y, int64_t ldy, int block,
                     void *stream) {
  if (dim == 0 || block == 0) return SVDSB_OK;
  SVDSB_LAUNCH_PDL(diag_solve_kernel, grid1(dim), 256, 0, as_stream(stream), dim, block, d, x, ldx, y, ldy);
  return SVDSB_OK;
}

}  // extern "C"
