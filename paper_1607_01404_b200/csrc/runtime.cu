// Library plumbing: error strings, launch counter, context (workspace).
#include <stdarg.h>
#include <stdlib.h>
#include <atomic>

#include "common.cuh"

namespace svdsb {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int64_t bump_launches(int n) { return g_launches.fetch_add(n) + n; }

static thread_local bool g_pdl_suspended = false;

void set_pdl_suspended(bool on) { g_pdl_suspended = on; }

bool pdl_on() {
  if (g_pdl_suspended) return false;
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SVDSB_PDL");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 1;
    cache[dev] = n;
  }
  return cache[dev];
}

}  // namespace svdsb

extern "C" {

int svdsb_version(void) { return 1; }

const char *svdsb_last_error(void) { return svdsb::g_err; }

int64_t svdsb_launch_count(void) { return svdsb::g_launches.load(); }

int64_t svdsb_note_launches(int64_t n) { return svdsb::bump_launches((int)n); }

int svdsb_tune_set(int key, int value) {
  if (key < 0 || key >= svdsb::kTuneKeys) return SVDSB_ERR_ARG;
  svdsb::g_tune[key] = value;
  return SVDSB_OK;
}

int svdsb_d2h(void *dst_host, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return SVDSB_OK;
  SVDSB_CUDA(cudaMemcpyAsync(dst_host, src, bytes, cudaMemcpyDeviceToHost, svdsb::as_stream(stream)));
  return SVDSB_OK;
}

int svdsb_stream_sync(void *stream) {
  SVDSB_CUDA(cudaStreamSynchronize(svdsb::as_stream(stream)));
  return SVDSB_OK;
}

// Stream capture / replay of the per-iteration launch sequence, without
// the framework's graph bookkeeping (private memory pools etc.): nothing
// is allocated inside a capture, only libsvdsb kernels are recorded.
int svdsb_graph_begin(void *stream) {
  SVDSB_CHECK_ARG(stream != nullptr, "svdsb_graph_begin: capture needs a non-default stream");
  SVDSB_CUDA(cudaStreamBeginCapture(svdsb::as_stream(stream), cudaStreamCaptureModeThreadLocal));
  return SVDSB_OK;
}

int svdsb_graph_end(void *stream, void **exec_out) {
  SVDSB_CHECK_ARG(exec_out != nullptr, "svdsb_graph_end: NULL output");
  cudaGraph_t g = nullptr;
  SVDSB_CUDA(cudaStreamEndCapture(svdsb::as_stream(stream), &g));
  cudaGraphExec_t e = nullptr;
  cudaError_t rc = cudaGraphInstantiateWithFlags(&e, g, 0);
  cudaGraphDestroy(g);
  SVDSB_CUDA(rc);
  *exec_out = e;
  return SVDSB_OK;
}

int svdsb_graph_end_update(void *stream, void *exec_in, void **exec_out) {
  SVDSB_CHECK_ARG(exec_out != nullptr, "svdsb_graph_end_update: NULL output");
  cudaGraph_t g = nullptr;
  SVDSB_CUDA(cudaStreamEndCapture(svdsb::as_stream(stream), &g));
  if (exec_in != nullptr) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(reinterpret_cast<cudaGraphExec_t>(exec_in), g, &info) == cudaSuccess) {
      cudaGraphDestroy(g);
      *exec_out = exec_in;
      return SVDSB_OK;
    }
    cudaGetLastError();  // clear the update failure; instantiate afresh
  }
  cudaGraphExec_t e = nullptr;
  cudaError_t rc = cudaGraphInstantiateWithFlags(&e, g, 0);
  cudaGraphDestroy(g);
  SVDSB_CUDA(rc);
  *exec_out = e;
  return SVDSB_OK;
}

int svdsb_graph_launch(void *exec, void *stream) {
  SVDSB_CUDA(cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(exec), svdsb::as_stream(stream)));
  return SVDSB_OK;
}

int svdsb_graph_destroy(void *exec) {
  if (exec) cudaGraphExecDestroy(reinterpret_cast<cudaGraphExec_t>(exec));
  return SVDSB_OK;
}

int svdsb_ctx_create(int device, svdsb_ctx **out) {
  SVDSB_CHECK_ARG(out != nullptr, "svdsb_ctx_create: out is NULL");
  SVDSB_CUDA(cudaSetDevice(device));
  svdsb_ctx *c = new svdsb_ctx();
  c->device = device;
  c->next_ticket = 0;
  if (cudaMalloc(&c->partials, sizeof(double) * svdsb::kMaxPartials) != cudaSuccess ||
      cudaMalloc(&c->ticket, sizeof(unsigned int) * svdsb::kMaxTickets) != cudaSuccess ||
      cudaMalloc(&c->gbar, sizeof(unsigned int) * 2) != cudaSuccess) {
    svdsb::set_error("svdsb_ctx_create: cudaMalloc failed");
    delete c;
    return SVDSB_ERR_ALLOC;
  }
  SVDSB_CUDA(cudaMemset(c->ticket, 0, sizeof(unsigned int) * svdsb::kMaxTickets));
  SVDSB_CUDA(cudaMemset(c->gbar, 0, sizeof(unsigned int) * 2));
  SVDSB_CUDA(cudaDeviceSynchronize());
  *out = c;
  return SVDSB_OK;
}

int svdsb_ctx_destroy(svdsb_ctx *ctx) {
  if (!ctx) return SVDSB_OK;
  cudaFree(ctx->partials);
  cudaFree(ctx->ticket);
  cudaFree(ctx->gbar);
  delete ctx;
  return SVDSB_OK;
}

}  // extern "C"
