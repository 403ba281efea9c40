// Shared plumbing for libsvdsb: error reporting, launch accounting, the
// per-stream reduction workspace and warp/block reduction helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/svdsb.h"

namespace svdsb {

constexpr double kEps = 2.220446049250313e-16;  // kernels.py:20
constexpr int kNumSMs = 148;                     // B200

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

}  // namespace svdsb

// Reduction workspace: per-CTA partial sums then a ticket so the last CTA
// to finish folds them in fixed CTA order (deterministic, one launch).
struct svdsb_ctx {
  int device;
  double *partials;      // kMaxPartials doubles
  unsigned int *ticket;  // kMaxTickets counters, always left at 0
  int next_ticket;
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
