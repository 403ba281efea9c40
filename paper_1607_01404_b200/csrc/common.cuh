// Shared plumbing for libsvdsb: error reporting, launch accounting, the
// per-stream reduction workspace and warp/block reduction helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <utility>

#include "../../include/svdsb.h"

namespace svdsb {

constexpr double kEps = 2.220446049250313e-16;  // kernels.py:20
// SM count of the current device (148 on B200), queried once per device:
// grids sized in multiples of it, and the co-residency bound of the
// grid-barrier kernel, follow the part the library actually runs on.
int num_sms();

void set_error(const char *fmt, ...);
int64_t bump_launches(int n = 1);

#define SVDSB_CHECK_ARG(cond, msg)           \
  do {                                       \
    if (!(cond)) {                           \
      ::svdsb::set_error("%s", msg);         \
      return SVDSB_ERR_ARG;                  \
    }                                        \
  } while (0)

#define SVDSB_CUDA(call)                                                  \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess) {                                              \
      ::svdsb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,      \
                         cudaGetErrorString(e_));                         \
      return SVDSB_ERR_CUDA;                                              \
    }                                                                     \
  } while (0)

// Check the most recent launch and count it.
#define SVDSB_LAUNCHED()                                                  \
  do {                                                                    \
    ::svdsb::bump_launches();                                             \
    cudaError_t e_ = cudaGetLastError();                                  \
    if (e_ != cudaSuccess) {                                              \
      ::svdsb::set_error("%s:%d launch: %s", __FILE__, __LINE__,          \
                         cudaGetErrorString(e_));                         \
      return SVDSB_ERR_CUDA;                                              \
    }                                                                     \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch.  The per-iteration kernels are launched
// with programmatic stream serialisation so a kernel's launch overlaps the
// tail of the one before it (also inside captured graphs).  Every kernel
// launched through launch_k() calls pdl_wait() before it touches memory --
// that blocks until the preceding grid has completed and its writes are
// visible -- and may call pdl_trigger() once its own main loop is done to let
// the next grid's CTAs be scheduled early.  SVDSB_PDL=0 turns the attribute
// off (plain stream order; pdl_wait() is then a no-op).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_on();
// Launches made by this thread skip the PDL attribute while suspended
// (conditional-node bodies are captured without programmatic edges).
void set_pdl_suspended(bool on);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// As launch_k, plus the cooperative attribute: the launch fails instead of
// deadlocking when the grid cannot be co-resident (kernels with a software
// grid barrier).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Launch through launch_k and account for it (use inside int-returning
// C-ABI functions).
// Optional epilogues of the last CTA of a reduction kernel (the native
// GD+k iteration, gdk.cu): write the Gram column straight into H (column
// and row g, as svdsb_h_insert does for b = 1), and copy the status record
// (Ritz values, residual norms, DGKS state) to pinned host memory after the
// Ritz residual norms (as svdsb_status_pack).
struct HInsert {
  double *h = nullptr;
  int64_t ldh = 0;
  int g = 0;
};
struct StatusOut {
  const double *lams = nullptr;
  int gn = 0;
  const double *st = nullptr;
  double *host = nullptr;
};

// Reduction launches with the epilogues above (dense.cu), for gdk.cu.
int gram_impl(svdsb_ctx *ctx, int64_t dim, int nblk, const double *const *xs, const int64_t *ldxs, const int *cols,
              const double *y, int64_t ldy, int b, double *c, int64_t ldc, double *norms2, void *stream, HInsert hi);
int ritz_impl(svdsb_ctx *ctx, int64_t dim, const double *v, int64_t ldv, const double *w, int64_t ldw, int g,
              const double *yc, int64_t ldyc, const double *lam, int p, double *r, int64_t ldr, double *x,
              int64_t ldx, double *ox, int64_t ldox, double *rn2, void *stream, StatusOut so);

// Kernel-variant knobs for measurement tools (svdsb_tune_set); 0 selects
// the default everywhere.  Key 0: forward b = 4 SpMV of short-row matrices
// (0 sliced ELL, 2 warp-staged CSR, 1 thread-per-row from global, 3 four
// lanes per row).
// Key 1: b = 4 Gram grid order (0 interleaved, 2 column groups outermost).
// Key 2: sliced-ELL b = 4 (0 grouped loads, 1 whole-row prefetch for rows
// <= 20; slower on config 4).
// Key 3: Ritz residual (0: two threads per row for 16 < p <= 32, one
// otherwise; 1: always one; 2: two also for 8 < p <= 16; 4: two threads per
// row with two rows each for 16 < p <= 24 -- slower on config 4).
// Key 4: native GD+k iteration (0 H-column / status epilogues, 1 separate
// h_insert and status_pack launches); 2 also selects the generic 32-column
// in-place restart product instead of ts_gemm_inplace_vec_kernel.
// Key 5: transposed b = 4 SpMV (0 length-sorted sliced ELL, 1 CSR tiles).
// Key 6: 2- and 3-column products of short-row matrices (0 zero-padded to
// the 4-column kernels, 1 the b-column CSR tile kernels).
// Key 7: b = 4 sliced ELL (0 TMA-staged ring for the forward product,
// csr_sell4s_kernel, rows <= 20 nonzeros; 1 the direct-load kernels both
// ways; 2 the TMA-staged ring both ways, csr_sell4ts_kernel transposed;
// 4 the forward ring staging only column ids and lengths, 4 slices deep,
// values loaded with the gathers, csr_sell4sb_kernel: 810-825 us, the same
// as key 0; 6 slices deep 950 us).
// Key 8: transposed b = 4 rows of 65-2048 nonzeros (0 lane-parallel fma
// sums + fixed xor tree, deterministic, within 1e-13 of the sequential sum;
// 1 the serial left-to-right fold, bit-identical to np.add.at).
// Key 9: long rows of transposed b = 4 products (0 the 8192-nonzero chunks
// gathering from L2, csr_chunk_kernel; 1 head tiles: the operand staged in
// shared memory tile by tile, csr_headtile4_kernel -- 3.2x slower on config
// 4: ~470 small pieces per 2048-row tile, each a latency-bound reduction).
// Key 10: sliced-ELL copies built on the device (0) or on the host (1).
// Key 11: Ritz residuals with FMAs (0, ritz_wide / ritz_split) or on the
// fp64 tensor cores (1, ritz_dmma_kernel: DMMA m8n8k4 with Y in registers;
// slower on B200 -- config 3: 910 vs 639 us).
// Key 12: hot operand rows of the forward b = 4 ring kernel (0: every gather
// from global memory; 1: the part's 1280 most referenced columns are read
// from a shared-memory copy when they carry at least a fifth of the nonzeros
// -- set before the first block product of a matrix; config 4: 992 vs 820 us,
// L1-wavefront-bound either way, see csr_sell4s_kernel).
// Key 13: running sums of the column-blocked A^T product of a packed block
// (0: in the column-major result; 1: in a row-major scratch block unpacked
// at the end -- 25 us slower on config 4).
// Key 14: work items of csr_sell4t_kernel (0: handed out by a device
// counter after each warp's first; 1: fixed stride).
// Key 15: tall-skinny Gram / Ritz residual / restart product of bases beyond
// L2 scale (0: streamed through a cp.async.bulk shared-memory ring by one
// persistent CTA per SM when the operand has >= 2^18 rows, dense_stream.cuh;
// 1: always the register-tiled kernels; 2: always the streamed kernels; 3: as 2
// with the twelve-warp Ritz variant for 16 < p <= 24 -- two rows x six
// candidates per thread, more shared-memory loads per FMA: 219 vs 195 us at
// N = 1 M, kept for measurement; 4: sixteen warps of the same shape, <= 128
// registers: 215 us; 5: no streamed projection; 6: as 0 plus the one-column
// Gram / projection / CGS pass on the streamed kernels -- faster alone,
// slower inside the solves, see stream_one_col in dense.cu).
// Key 16: kernel order of a transposed b = 4 part (0: short rows first; 1:
// long rows, chunk path, first -- they stream the operand block into L2 for
// the short rows' scattered gathers; no gain on config 4).
constexpr int kTuneKeys = 17;
inline int g_tune[kTuneKeys] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};

#define SVDSB_LAUNCH_PDL(...)                                             \
  do {                                                                    \
    cudaError_t e_ = ::svdsb::launch_k(__VA_ARGS__);                      \
    if (e_ != cudaSuccess) {                                              \
      ::svdsb::set_error("%s:%d launch: %s", __FILE__, __LINE__,          \
                         cudaGetErrorString(e_));                         \
      return SVDSB_ERR_CUDA;                                              \
    }                                                                     \
    ::svdsb::bump_launches();                                             \
  } while (0)

}  // namespace svdsb

// Reduction workspace: per-CTA partial sums then a ticket so the last CTA
// to finish folds them in fixed CTA order (deterministic, one launch).
struct svdsb_ctx {
  int device;
  double *partials;      // kMaxPartials doubles
  unsigned int *ticket;  // kMaxTickets counters, always left at 0
  int next_ticket;
  unsigned int *gbar;    // software grid barrier: {arrival count, generation}
};

namespace svdsb {

constexpr int64_t kMaxPartials = 4 << 20;  // 32 MB of fp64 partials
constexpr int kMaxTickets = 64;

// Each reduction launch uses its own counter slot (round robin) so two
// back-to-back launches on one stream never share a counter mid-flight.
inline unsigned int *take_ticket(svdsb_ctx *ctx) {
  unsigned int *t = ctx->ticket + ctx->next_ticket;
  ctx->next_ticket = (ctx->next_ticket + 1) % kMaxTickets;
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Last-CTA fold of per-CTA partials laid out as
//   partials[(t * nparts + bx) * per + k],  output o = t * per + k < nout,
// by the whole CTA: one warp per output, lanes take a fixed strided subset of
// the nparts CTAs and a fixed xor tree combines them, so the result is
// deterministic and the load chain is nparts / 32 deep instead of nparts.
// emit(o, t, k, sum) is called by lane 0 of the owning warp.
// Wide partial vectors (per >= 16) are read by (k, slice) thread pairs
// instead -- consecutive threads take consecutive k, so every warp load is
// coalesced -- and the slices are combined in shared memory in fixed order.
// Must be called by every thread of the CTA (it synchronises).
template <typename Emit>
__device__ __forceinline__ void fold_parts(const double *partials, unsigned nparts, int per, int nout, Emit emit) {
  const int nt = blockDim.x;
  if (per >= 16 && per <= nt) {
    __shared__ double red[1024];
    const int S = nt / per;
    const int k = threadIdx.x % per, sl = threadIdx.x / per;
    const int ntile = (nout + per - 1) / per;
    for (int t = 0; t < ntile; ++t) {
      const double *pp = partials + (int64_t)t * nparts * per + k;
      double acc = 0.0;
      if (sl < S) {
        // 16 independent loads in flight per thread, summed in the same
        // order as a plain strided loop (bx = sl, sl + S, ...)
        constexpr int CH = 16;
        for (unsigned b0 = sl; b0 < nparts; b0 += CH * S) {
          double tv[CH];
#pragma unroll
          for (int q = 0; q < CH; ++q) {
            const unsigned bx = b0 + q * S;
            tv[q] = bx < nparts ? pp[(int64_t)bx * per] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < CH; ++q)
            if (b0 + q * S < nparts) acc += tv[q];
        }
      }
      red[threadIdx.x] = acc;
      __syncthreads();
      if (threadIdx.x < per) {
        double s = 0.0;
        for (int q = 0; q < S; ++q) s += red[q * per + threadIdx.x];
        const int o = t * per + threadIdx.x;
        if (o < nout) emit(o, t, (int)threadIdx.x, s);
      }
      __syncthreads();
    }
    return;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = nt >> 5;
  for (int o = w; o < nout; o += nw) {
    const int t = o / per, kk = o % per;
    const double *pp = partials + (int64_t)t * nparts * per + kk;
    double s = 0.0;
    constexpr int CH = 8;
    for (unsigned b0 = lane; b0 < nparts; b0 += CH * 32) {
      double tv[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const unsigned bx = b0 + q * 32;
        tv[q] = bx < nparts ? pp[(int64_t)bx * per] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < CH; ++q)
        if (b0 + q * 32 < nparts) s += tv[q];
    }
    s = warp_sum(s);
    if (lane == 0) emit(o, t, kk, s);
  }
}

// Software grid barrier (arrival counter + generation).  Every CTA of the
// grid must be resident at once: callers size the grid to at most the
// occupancy-limited number of co-resident CTAs and never trigger their
// dependants before the last barrier.
__device__ __forceinline__ void grid_barrier(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int *gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Returns true in exactly one CTA: the last to arrive at the ticket.  All
// partial writes of this CTA must precede the call.  Resets the ticket.
__device__ __forceinline__ bool last_cta(unsigned int *ticket) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(ticket, 1u);
    am_last = (t == gridDim.x * gridDim.y * gridDim.z - 1);
    if (am_last) *ticket = 0u;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

// ------------------------------------------------ bulk copies (TMA engine)
// cp.async.bulk global -> shared with completion counted on an mbarrier
// (the non-tensor form of TMA): one thread moves whole tiles while the CTA
// computes on the previous stage.
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Streamed operands (read once per launch) are marked evict-first.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar,
                                         uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
               " [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
               " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}


__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t policy;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  return policy;
}

// Grid size for row-streaming kernels: enough CTAs to fill the chip a few
// times, never more than rows warrant.  Fixed for a given dim so the
// reduction order (and so the result) is reproducible.
inline int stream_grid(int64_t dim, int rows_per_cta, int max_ctas) {
  int64_t need = (dim + rows_per_cta - 1) / rows_per_cta;
  if (need < 1) need = 1;
  if (need > max_ctas) need = max_ctas;
  return (int)need;
}

}  // namespace svdsb
