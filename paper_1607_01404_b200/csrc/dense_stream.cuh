// Streamed tall-skinny kernels for bases that do not fit L2 (included by
// dense.cu inside namespace svdsb).
//
// The register-tiled kernels of dense.cu keep two 256-thread CTAs per SM and
// rely on their own loads to cover the DRAM latency; with the 48-140
// accumulators a b = 4 / p = 24 operation needs per thread that leaves 16
// warps per SM and 25-45 % of HBM at N = 1 M (config 4).  Here one persistent
// CTA per SM streams row tiles through a shared-memory ring filled by
// TMA tensor-map tile loads (full / empty mbarriers, 100-180 KB in flight per
// SM whatever the register budget) and eight warps do the arithmetic from shared memory:
//
//   ts_stream_kernel<NIN, PQ, RITZ>   R = W Y - (V Y) diag(lam) (+ norms, status
//                                     copy) or, in place, V <- V C (thick
//                                     restart, eigensolver.py:454-486); per
//                                     element the fma chain of ritz_wide_kernel
//                                     / ts_gemm_inplace_kernel (basis index
//                                     ascending), so results are bit-identical
//   gram_stream_kernel                C = X^T Y (+ |Y_j|^2) for 1..4 columns
//                                     of Y and up to 40 basis columns
//
// Row tiles are dealt to CTAs in contiguous, fixed ranges and every reduction
// is a fixed tree, so results do not depend on timing.

constexpr int kStreamConsumers = 256;                  // 8 consumer warps
constexpr int kStreamThreads = kStreamConsumers + 32;  // + the producer warp

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

// One TMA instruction per tile: box (rows c0.., columns c1..) of a column-major
// fp64 block described by a tensor map (rows innermost); rows / columns past
// the block's extent arrive as zeros and count towards the transaction bytes.
// (A ring fed by per-column cp.async.bulk copies of 1-2 KB stalled at ~190
// cycles per copy on the issuing thread -- 1.5-2.8 TB/s -- hence tensor maps.)
__device__ __forceinline__ void tma_tile_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar,
                                            bool ef, uint64_t policy) {
  if (ef)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1, {%2, %3}], [%4], %5;"
                 :: "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}

// Tiles [t0, t1) of CTA bx out of nx.
__device__ __forceinline__ void stream_tiles(int64_t ntile, int bx, int nx, int64_t &t0, int64_t &t1) {
  t0 = ntile * bx / nx;
  t1 = ntile * (bx + 1) / nx;
}

constexpr int kTsRows = 256;   // rows per tile: 128 thread pairs x 2 rows
#ifndef SVDSB_TS_STAGES
#define SVDSB_TS_STAGES 4
#endif
#ifndef SVDSB_TS_LEAD
#define SVDSB_TS_LEAD 1
#endif
constexpr int kTsStages = SVDSB_TS_STAGES;  // 32 KB each
constexpr int kTsThreads = 256;
constexpr int kTsLead = SVDSB_TS_LEAD;      // a stage is refilled this many items after its use

__host__ __device__ constexpr int ts_kc(int nin) { return 16 / nin; }  // basis columns per stage
__host__ __device__ constexpr int ts_rows(int nt, int rpt, int split) { return nt / split * rpt; }  // rows per tile

// NIN = 2, RITZ: R[:, j] = (W y_j) - (V y_j) * lam_j for j < p (two roundings,
//   eigensolver.py:392), optional X = V Y and OpX = W Y, |R_j|^2 folded by the
//   last CTA, status copy as ritz_wide_kernel.
// NIN = 1, !RITZ: r[:, j] = V c_j for j < p; r may alias v (every row of a tile
//   is staged in shared memory in full before any of it is written, and no
//   other CTA touches those rows).
// RPT threads share RPT adjacent rows, each owning PQ consecutive columns of
// Y (NIN RPT PQ + PQ fp64 accumulators: the register file of an SM
// sub-partition holds two such warps, so all eight warps compute and lane 0
// of warp 0 also issues the copies -- item i + kTsStages - kTsLead while the
// CTA works on item i, by when every warp has released that stage).  RPT = 4
// for wide Y: a k-step of a warp then reads 7 shared-memory wavefronts for
// its 48 fp64 FMAs per lane where RPT = 2 reads 10-16 (the shared-memory pipe
// and the FMA pipe were both about half busy).
template <int NIN, int NT, int RPT, int SPLIT, int PQ, bool RITZ>
__global__ void __launch_bounds__(NT, 1)
ts_stream_kernel(const __grid_constant__ CUtensorMap mapv, const __grid_constant__ CUtensorMap mapw, int64_t dim, int g,
                 const double *__restrict__ yc, int64_t ldyc, const double *__restrict__ lam, int p, double *r,
                 int64_t ldr, double *xo, int64_t ldx, double *oxo, int64_t ldox, double *rn2, double *partials,
                 unsigned int *ticket, StatusOut so, int evict_first) {
  constexpr int PT = PQ * SPLIT, R = ts_rows(NT, RPT, SPLIT), KC = ts_kc(NIN), NS = kTsStages, NW = NT / 32;
  constexpr int STAGE_D = NIN * KC * R;
  static_assert((RPT == 2 || RPT == 4) && (SPLIT == 2 || SPLIT == 4) && PQ % 2 == 0 && R <= 256, "tile shape");
  extern __shared__ __align__(1024) double ts_dyn[];
  double *ysh = ts_dyn + NS * STAGE_D;  // g x PT
  __shared__ uint64_t full[NS], empty[NS];
  __shared__ double lsh[PT];
  __shared__ double red[NW][PT];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();
  for (int k = tid; k < g * PT; k += NT) {
    const int i = k / PT, j = k % PT;
    ysh[k] = (j < p) ? yc[i + (int64_t)j * ldyc] : 0.0;
  }
  if (RITZ && tid < PT) lsh[tid] = (tid < p) ? lam[tid] : 0.0;
  __syncthreads();
  const int nch = (g + KC - 1) / KC;
  const int64_t ntile = (dim + R - 1) / R;
  int64_t t0, t1;
  stream_tiles(ntile, blockIdx.x, gridDim.x, t0, t1);
  const int64_t nitems = (t1 - t0) * nch;
  const uint64_t policy = evict_first_policy();
  const bool ef = evict_first != 0;
  // thread 0: fill stage item % NS with column chunk item % nch of tile t0 + item / nch
  auto issue = [&](int64_t item) {
    const int64_t t = t0 + item / nch;
    const int c = (int)(item % nch);
    const int s = (int)(item % NS);
    const int64_t k = item / NS;
    if (k > 0) mbar_wait(&empty[s], (unsigned)((k - 1) & 1));
    double *st = ts_dyn + s * STAGE_D;
    mbar_expect_tx(&full[s], (unsigned)(STAGE_D * sizeof(double)));
    tma_tile_2d(st, &mapv, (int)(t * R), c * KC, &full[s], ef, policy);
    if (NIN == 2) tma_tile_2d(st + KC * R, &mapw, (int)(t * R), c * KC, &full[s], ef, policy);
  };
  if (tid == 0)
    for (int64_t item = 0; item < min((int64_t)NS, nitems); ++item) issue(item);
  __syncwarp();

  double nacc[PQ];
#pragma unroll
  for (int j = 0; j < PQ; ++j) nacc[j] = 0.0;
  const int part = tid % SPLIT, q = tid / SPLIT;
  const int j0 = part * PQ;
  int64_t it = 0;
  for (int64_t t = t0; t < t1; ++t) {
    double ax[PQ][RPT], aw[NIN == 2 ? PQ : 1][RPT];
#pragma unroll
    for (int j = 0; j < PQ; ++j)
#pragma unroll
      for (int e = 0; e < RPT; ++e) {
        ax[j][e] = 0.0;
        if (NIN == 2) aw[j][e] = 0.0;
      }
    for (int c = 0; c < nch; ++c, ++it) {
#ifndef SVDSB_TS_NOLOAD   // timing experiment: 1 = compute on stale stages after the first ring fill
      if (tid == 0 && it >= kTsLead && it - kTsLead + NS < nitems) issue(it - kTsLead + NS);
      __syncwarp();
#endif
      const int s = (int)(it % NS);
#ifdef SVDSB_TS_NOLOAD
      if (it < NS)
#endif
      mbar_wait(&full[s], (unsigned)((it / NS) & 1));
      const double *sv = ts_dyn + s * STAGE_D + RPT * q;
      const double *yb = ysh + (c * KC) * PT + j0;
      const int kc = min(KC, g - c * KC);
      auto body = [&](int u) {
        double vv[RPT], ww[RPT];
#pragma unroll
        for (int e = 0; e < RPT; e += 2) {
          const double2 t2 = *reinterpret_cast<const double2 *>(sv + u * R + e);
          vv[e] = t2.x;
          vv[e + 1] = t2.y;
          if (NIN == 2) {
            const double2 w2 = *reinterpret_cast<const double2 *>(sv + (KC + u) * R + e);
            ww[e] = w2.x;
            ww[e + 1] = w2.y;
          }
        }
        const double2 *yrow = reinterpret_cast<const double2 *>(yb + u * PT);
#pragma unroll
        for (int j = 0; j < PQ / 2; ++j) {
          const double2 cf = yrow[j];
#pragma unroll
          for (int e = 0; e < RPT; ++e) {
            ax[2 * j][e] = fma(vv[e], cf.x, ax[2 * j][e]);
            ax[2 * j + 1][e] = fma(vv[e], cf.y, ax[2 * j + 1][e]);
            if (NIN == 2) {
              aw[2 * j][e] = fma(ww[e], cf.x, aw[2 * j][e]);
              aw[2 * j + 1][e] = fma(ww[e], cf.y, aw[2 * j + 1][e]);
            }
          }
        }
      };
      if (kc == KC) {
#pragma unroll
        for (int u = 0; u < KC; ++u) body(u);
      } else {
        for (int u = 0; u < kc; ++u) body(u);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    const int64_t row = t * R + RPT * q;
#pragma unroll
    for (int j = 0; j < PQ; ++j) {
      if (j0 + j < p) {
        const double l = RITZ ? lsh[j0 + j] : 0.0;
#pragma unroll
        for (int e = 0; e < RPT; e += 2) {
          const int jw = NIN == 2 ? j : 0;
          double2 o, x2 = make_double2(ax[j][e], ax[j][e + 1]), w2 = make_double2(aw[jw][e], aw[jw][e + 1]);
          if (RITZ)
            o = make_double2(__dsub_rn(w2.x, __dmul_rn(x2.x, l)), __dsub_rn(w2.y, __dmul_rn(x2.y, l)));
          else
            o = x2;
          if (row + e + 1 < dim) {
            *reinterpret_cast<double2 *>(r + row + e + (int64_t)(j0 + j) * ldr) = o;
            if (RITZ) {
              if (xo) *reinterpret_cast<double2 *>(xo + row + e + (int64_t)(j0 + j) * ldx) = x2;
              if (oxo) *reinterpret_cast<double2 *>(oxo + row + e + (int64_t)(j0 + j) * ldox) = w2;
              nacc[j] = fma(o.y, o.y, fma(o.x, o.x, nacc[j]));
            }
          } else if (row + e < dim) {
            r[row + e + (int64_t)(j0 + j) * ldr] = o.x;
            if (RITZ) {
              if (xo) xo[row + e + (int64_t)(j0 + j) * ldx] = x2.x;
              if (oxo) oxo[row + e + (int64_t)(j0 + j) * ldox] = w2.x;
              nacc[j] = fma(o.x, o.x, nacc[j]);
            }
          }
        }
      }
    }
  }
  pdl_trigger();
  if (!RITZ) return;
  // per-candidate CTA sums: lanes of equal tid % SPLIT hold the same candidates
#pragma unroll
  for (int j = 0; j < PQ; ++j) {
    double t = nacc[j];
#pragma unroll
    for (int off = 16; off >= SPLIT; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane < SPLIT) red[wid][part * PQ + j] = t;
  }
  __syncthreads();
  double *pp = partials + (int64_t)blockIdx.x * PT;
  for (int k = tid; k < PT; k += NT) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) t += red[ww][k];
    pp[k] = t;
  }
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, PT, p, [&](int j, int, int, double t) { rn2[j] = t; });
  if (so.host != nullptr) {
    __syncthreads();
    for (int i = tid; i < so.gn + p + 8; i += blockDim.x)
      so.host[i] = i < so.gn ? so.lams[i] : (i < so.gn + p ? rn2[i - so.gn] : so.st[i - so.gn - p]);
    __threadfence_system();
  }
}

constexpr int kGsRows = 128;     // rows per tile
constexpr int kGsStages = 3;
constexpr int kGsBox = 8;        // basis columns per TMA box
constexpr int kGsMaxX = 40;      // basis columns (5 per consumer warp)
constexpr int kGsCap = 64;       // stage capacity in columns: every block rounded up to a box, + 4 of y
constexpr int kGsOut = kGsMaxX * 4 + 4;

struct GramMaps {
  CUtensorMap x[SVDSB_MAX_BLOCKS];  // box kGsRows x kGsBox, extent dim x cols[k]
  CUtensorMap y;                    // box kGsRows x 4, extent dim x nb
};

// C = X^T Y (na <= 40 columns of X in up to SVDSB_MAX_BLOCKS blocks, nb <= 4
// of Y) and |Y_j|^2.  A stage holds the tile's rows of every column: block k
// at column offset off[k] (its columns rounded up to whole boxes, the
// padding zero-filled by the TMA unit), y after the last block; consumer
// warp w owns basis columns w, w + 8, ..., each lane two row pairs of a tile.
__global__ void __launch_bounds__(kStreamThreads, 1)
gram_stream_kernel(const __grid_constant__ GramMaps maps, int64_t dim, ColSet xs, int nb, double *c, int64_t ldc,
                   double *norms2, double *partials, unsigned int *ticket, int evict_first, const double *gate,
                   HInsert hi) {
  constexpr int R = kGsRows, NS = kGsStages, MC = kGsMaxX / 8, NW = kStreamConsumers / 32;
  extern __shared__ __align__(1024) double gs_dyn[];
  __shared__ uint64_t full[NS], empty[NS];
  __shared__ int scol[kGsMaxX];  // stage column of basis column i
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int na = xs.total;
  int ycol = 0;  // stage column of y = total boxes * kGsBox
  for (int k = 0; k < xs.nblk; ++k) ycol += (xs.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
  const int stage_d = (ycol + 4) * R;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int i = 0, off = 0;
    for (int k = 0; k < xs.nblk; ++k) {
      for (int q = 0; q < xs.cols[k]; ++q) scol[i++] = off + q;
      off += (xs.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
    }
  }
  pdl_wait();
  if (gate != nullptr && gate[0] == 0.0) return;  // device-side DGKS: column already final (every thread leaves)
  __syncthreads();
  const int64_t ntile = (dim + R - 1) / R;
  int64_t t0, t1;
  stream_tiles(ntile, blockIdx.x, gridDim.x, t0, t1);
  double acc[MC][4], nacc[4];
#pragma unroll
  for (int m = 0; m < MC; ++m)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[m][j] = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) nacc[j] = 0.0;
  const bool want_norm = norms2 != nullptr && wid == NW - 1;

  if (wid == NW) {
    if (lane == 0) {
      const uint64_t policy = evict_first_policy();
      const bool ef = evict_first != 0;
      int64_t it = 0;
      for (int64_t t = t0; t < t1; ++t, ++it) {
        const int s = (int)(it % NS);
        const int64_t k = it / NS;
        if (k > 0) mbar_wait(&empty[s], (unsigned)((k - 1) & 1));
        double *st = gs_dyn + (size_t)s * stage_d;
        mbar_expect_tx(&full[s], (unsigned)(stage_d * sizeof(double)));
        int off = 0;
        for (int kb = 0; kb < xs.nblk; ++kb)
          for (int q = 0; q < xs.cols[kb]; q += kGsBox, off += kGsBox)
            tma_tile_2d(st + off * R, &maps.x[kb], (int)(t * R), q, &full[s], ef, policy);
        tma_tile_2d(st + off * R, &maps.y, (int)(t * R), 0, &full[s], false, policy);
      }
    }
  } else {
    int xc[MC];
#pragma unroll
    for (int m = 0; m < MC; ++m) xc[m] = wid + 8 * m < na ? scol[wid + 8 * m] * R : 0;
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int s = (int)(it % NS);
      mbar_wait(&full[s], (unsigned)((it / NS) & 1));
      const double *st = gs_dyn + (size_t)s * stage_d;
#pragma unroll
      for (int h = 0; h < R / 64; ++h) {
        const int rr = 2 * lane + 64 * h;  // rows past dim are zeros (TMA fill)
        double2 yv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) yv[j] = *reinterpret_cast<const double2 *>(st + (ycol + j) * R + rr);
#pragma unroll
        for (int m = 0; m < MC; ++m) {
          if (wid + 8 * m < na) {
            const double2 xv = *reinterpret_cast<const double2 *>(st + xc[m] + rr);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[m][j] = fma(xv.x, yv[j].x, fma(xv.y, yv[j].y, acc[m][j]));
          }
        }
        if (want_norm) {
#pragma unroll
          for (int j = 0; j < 4; ++j) nacc[j] = fma(yv[j].x, yv[j].x, fma(yv[j].y, yv[j].y, nacc[j]));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  pdl_trigger();
  double *part = partials + (int64_t)blockIdx.x * kGsOut;
  if (wid < NW) {
#pragma unroll
    for (int m = 0; m < MC; ++m)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double sum = warp_sum(acc[m][j]);
        if (lane == 0) part[(wid + 8 * m) * 4 + j] = sum;
      }
    if (wid == NW - 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double sum = warp_sum(nacc[j]);
        if (lane == 0) part[kGsMaxX * 4 + j] = sum;
      }
    }
  }
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, kGsOut, kGsOut, [&](int, int, int k, double sum) {
    if (k < kGsMaxX * 4) {
      const int i = k / 4, j = k % 4;
      if (i < na && j < nb) {
        c[i + (int64_t)j * ldc] = sum;
        if (hi.h != nullptr && j == 0 && i <= hi.g) {  // one column: H(i, g) = H(g, i), as gram1_vec_kernel
          hi.h[i + (int64_t)hi.g * hi.ldh] = sum;
          hi.h[hi.g + (int64_t)i * hi.ldh] = sum;
        }
      }
    } else if (norms2 != nullptr && k - kGsMaxX * 4 < nb) {
      norms2[k - kGsMaxX * 4] = sum;
    }
  });
}


constexpr int kPsRows = 256;   // rows per tile: one per consumer thread
constexpr int kPsStages = 2;

// Y -= X C (+ |Y_j|^2 after) for NB <= 4 columns of Y and up to 40 basis
// columns: stage layout as gram_stream_kernel with 256-row tiles, one row
// per consumer thread; per element the fma chain of project_kernel (basis
// index ascending), so Y is bit-identical to the register kernels.  NB = 1
// carries the device-side DGKS gate and decision of project1_vec_kernel.
struct ProjMaps {
  CUtensorMap x[SVDSB_MAX_BLOCKS];  // box kPsRows x kGsBox
  CUtensorMap y;                    // box kPsRows x 4, extent dim x NB
};

template <int NB>
__global__ void __launch_bounds__(kStreamThreads, 1)
project_stream_kernel(const __grid_constant__ ProjMaps maps, int64_t dim, ColSet xs, const double *__restrict__ cmat,
                      int64_t ldc, double *y, int64_t ldy, double *norms2, double *partials, unsigned int *ticket,
                      int evict_first, double *dgks) {
  constexpr int R = kPsRows, NS = kPsStages, NW = kStreamConsumers / 32;
  extern __shared__ __align__(1024) double ps_dyn[];
  __shared__ uint64_t full[NS], empty[NS];
  __shared__ int scol[kGsMaxX];
  __shared__ double csh[kGsMaxX * NB];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int na = xs.total;
  int ycol = 0;
  for (int k = 0; k < xs.nblk; ++k) ycol += (xs.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
  const int stage_d = (ycol + 4) * R;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    int i = 0, off = 0;
    for (int k = 0; k < xs.nblk; ++k) {
      for (int q = 0; q < xs.cols[k]; ++q) scol[i++] = off + q;
      off += (xs.cols[k] + kGsBox - 1) / kGsBox * kGsBox;
    }
  }
  pdl_wait();
  if (dgks != nullptr && dgks[0] == 0.0) return;
  for (int k = tid; k < na * NB; k += kStreamThreads) csh[k] = cmat[k / NB + (int64_t)(k % NB) * ldc];
  __syncthreads();
  const int64_t ntile = (dim + R - 1) / R;
  int64_t t0, t1;
  stream_tiles(ntile, blockIdx.x, gridDim.x, t0, t1);
  double nacc[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) nacc[j] = 0.0;

  if (wid == NW) {
    if (lane == 0) {
      const uint64_t policy = evict_first_policy();
      const bool ef = evict_first != 0;
      int64_t it = 0;
      for (int64_t t = t0; t < t1; ++t, ++it) {
        const int s = (int)(it % NS);
        const int64_t k = it / NS;
        if (k > 0) mbar_wait(&empty[s], (unsigned)((k - 1) & 1));
        double *st = ps_dyn + (size_t)s * stage_d;
        mbar_expect_tx(&full[s], (unsigned)(stage_d * sizeof(double)));
        int off = 0;
        for (int kb = 0; kb < xs.nblk; ++kb)
          for (int q = 0; q < xs.cols[kb]; q += kGsBox, off += kGsBox)
            tma_tile_2d(st + off * R, &maps.x[kb], (int)(t * R), q, &full[s], ef, policy);
        tma_tile_2d(st + off * R, &maps.y, (int)(t * R), 0, &full[s], false, policy);
      }
    }
  } else {
    int64_t it = 0;
    for (int64_t t = t0; t < t1; ++t, ++it) {
      const int s = (int)(it % NS);
      mbar_wait(&full[s], (unsigned)((it / NS) & 1));
      const double *st = ps_dyn + (size_t)s * stage_d + tid;
      const int64_t row = t * R + tid;
      double yv[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) yv[j] = st[(ycol + j) * R];
      for (int i0 = 0; i0 < na; i0 += 8) {
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = st[scol[min(i0 + u, na - 1)] * R];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0 + u < na) {
#pragma unroll
            for (int j = 0; j < NB; ++j) yv[j] = fma(-xv[u], csh[(i0 + u) * NB + j], yv[j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (row < dim) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          y[row + (int64_t)j * ldy] = yv[j];
          nacc[j] = fma(yv[j], yv[j], nacc[j]);
        }
      }
    }
  }
  pdl_trigger();
  if (norms2 == nullptr) return;
  __shared__ double red[NW][NB];
  if (wid < NW) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double sum = warp_sum(nacc[j]);
      if (lane == 0) red[wid][j] = sum;
    }
  }
  __syncthreads();
  if (tid < NB) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w][tid];
    partials[(int64_t)blockIdx.x * NB + tid] = t;
  }
  if (!last_cta(ticket)) return;
  fold_parts(partials, gridDim.x, NB, NB, [&](int j, int, int, double sum) {
    norms2[j] = sum;
    if (NB == 1 && dgks != nullptr) dgks_decide(dgks);
  });
}
