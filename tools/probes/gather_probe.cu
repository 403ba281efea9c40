// Gather-rate ceiling of a B200 SM for the b = 4 block SpMV (development
// probe, not part of the library): every nonzero of config 4's products
// fetches one 32-byte operand row at a data-dependent address.  This
// program measures how many such rows per second the chip delivers when
// NOTHING else happens (indices generated in registers, results folded
// into one accumulator), for tables of 32 MB (A X: x is L2-resident) and
// 64 MB (one column block of A^T Y), uniform and Zipf-like addresses,
// one lane per row (32-byte load), two lanes (16 bytes) and four (8 bytes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda error %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

struct __align__(32) Row { double v[4]; };

__device__ __forceinline__ void ld256(const Row *p, double &a, double &b, double &c, double &d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// LANES lanes cooperate on one row; each thread issues U independent gathers per step.
template <int LANES, int U>
__global__ void __launch_bounds__(256) gather_kernel(const Row *tab, uint32_t mask, int zipf, int steps, double *out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t grp = tid / LANES, sub = tid % LANES;
  double acc = 0.0;
  uint32_t s = mix(grp * 2654435761U + 12345U);
  for (int it = 0; it < steps; ++it) {
    uint32_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      s = mix(s + 0x9e3779b9U);
      uint32_t r = s & mask;
      if (zipf) {  // skew: square a uniform in [0,1) twice -> heavy head at small indices
        float f = (float)(s >> 8) * (1.0f / 16777216.0f);
        f = f * f; f = f * f; f = f * f;
        r = (uint32_t)(f * (float)(mask + 1u)) & mask;
      }
      idx[u] = r;
    }
    if (LANES == 1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double a, b, c, d;
        ld256(tab + idx[u], a, b, c, d);
        acc += a + b + c + d;
      }
    } else if (LANES == 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double2 t = __ldg(reinterpret_cast<const double2 *>(tab + idx[u]) + sub);
        acc += t.x + t.y;
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __ldg(reinterpret_cast<const double *>(tab + idx[u]) + sub);
    }
  }
  if (acc == 1.2345e300) out[0] = acc;
}

// The same gathers through the TMA unit instead of the LSU: every lane issues
// a 32-byte cp.async.bulk of its row into a shared-memory slot (one mbarrier
// per warp and stage, two stages), then reads the previous stage's slot.
__device__ __forceinline__ unsigned s32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) tma_gather_kernel(const Row *tab, uint32_t mask, int steps, double *out) {
  __shared__ __align__(128) Row buf[WARPS][2][32];
  __shared__ uint64_t bar[WARPS][2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(s32(&bar[w][k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t s = mix((blockIdx.x * blockDim.x + threadIdx.x) * 2654435761U + 777U);
  double acc = 0.0;
  auto issue = [&](int k) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(s32(&bar[w][k])), "r"(32u * 32u) : "memory");
    __syncwarp();
    s = mix(s + 0x9e3779b9U);
    const Row *src = tab + (s & mask);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];"
                 :: "r"(s32(&buf[w][k][lane])), "l"(src), "r"(s32(&bar[w][k])) : "memory");
  };
  issue(0);
  for (int it = 0; it < steps; ++it) {
    const int k = it & 1;
    if (it + 1 < steps) issue(k ^ 1);
    const unsigned parity = (it >> 1) & 1;
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                 :: "r"(s32(&bar[w][k])), "r"(parity) : "memory");
    const Row r = buf[w][k][lane];
    acc += r.v[0] + r.v[1] + r.v[2] + r.v[3];
    __syncwarp();
  }
  if (acc == 1.2345e300) out[0] = acc;
}

template <int WARPS>
static void run_tma(const Row *tab, uint32_t rows, int ctas_per_sm, double *out) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms * ctas_per_sm, steps = 512;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  tma_gather_kernel<WARPS><<<grid, WARPS * 32>>>(tab, rows - 1, steps, out);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  tma_gather_kernel<WARPS><<<grid, WARPS * 32>>>(tab, rows - 1, steps, out);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double gathers = (double)grid * WARPS * 32 * steps;
  printf("{\"case\": \"tma_bulk_32B\", \"table_mb\": %u, \"zipf\": 0, \"warps_per_cta\": %d, \"ctas_per_sm\": %d, "
         "\"grows_per_s\": %.1f, \"cycles_per_row_per_sm\": %.2f, \"us_for_173M\": %.0f}\n",
         rows / 32768, WARPS, ctas_per_sm, gathers / ms / 1e6, 1.92e9 * sms / (gathers / (ms * 1e-3)),
         172.93e6 / (gathers / ms) * 1e3);
}

template <int LANES, int U>
static void run(const char *name, const Row *tab, uint32_t rows, int zipf, int ctas_per_sm, double *out) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = sms * ctas_per_sm, steps = 2048 / U;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  gather_kernel<LANES, U><<<grid, 256>>>(tab, rows - 1, zipf, steps, out);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  gather_kernel<LANES, U><<<grid, 256>>>(tab, rows - 1, zipf, steps, out);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double gathers = (double)grid * 256 / LANES * steps * U;
  const double clk = 1.92e9;
  printf("{\"case\": \"%s\", \"table_mb\": %u, \"zipf\": %d, \"lanes_per_row\": %d, \"unroll\": %d, \"ctas_per_sm\": %d, "
         "\"grows_per_s\": %.1f, \"cycles_per_row_per_sm\": %.2f, \"l2_to_sm_gbs\": %.0f, \"us_for_173M\": %.0f}\n",
         name, rows / 32768, zipf, LANES, U, ctas_per_sm, gathers / ms / 1e6, clk * sms / (gathers / (ms * 1e-3)),
         gathers * 32 / ms / 1e6, 172.93e6 / (gathers / ms) * 1e3);
}

int main() {
  const uint32_t rows_max = 1u << 21;  // 64 MB
  Row *tab;
  double *out;
  CK(cudaMalloc(&tab, (size_t)rows_max * sizeof(Row)));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(tab, 0, (size_t)rows_max * sizeof(Row)));
  for (uint32_t rows : {1u << 20, 1u << 21}) {
    for (int zipf = 0; zipf < 2; ++zipf) {
      run<1, 8>("lane_per_row", tab, rows, zipf, 2, out);
      run<1, 8>("lane_per_row", tab, rows, zipf, 4, out);
      run<1, 8>("lane_per_row", tab, rows, zipf, 8, out);
      run<1, 16>("lane_per_row", tab, rows, zipf, 4, out);
      run<2, 8>("two_lanes", tab, rows, zipf, 4, out);
      run<2, 8>("two_lanes", tab, rows, zipf, 8, out);
      run<4, 8>("four_lanes", tab, rows, zipf, 8, out);
    }
  }
  run_tma<8>(tab, 1u << 20, 1, out);
  run_tma<8>(tab, 1u << 20, 4, out);
  run_tma<16>(tab, 1u << 20, 4, out);
  run_tma<8>(tab, 1u << 21, 4, out);
  return 0;
}
