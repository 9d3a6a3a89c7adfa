// Microbenchmark: shared-memory LDS.128 / LDS.64 / LDS.32 throughput when a warp reads U distinct
// records (lanes grouped: lane / (32 / U) picks the record), i.e. the cost of per-sub-block record
// lists in K4b.  Reports warp-loads per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
template <int U, int W>   // U distinct addresses per warp, W = bytes per lane (4, 8, 16)
__global__ void bench(float* out, int iters) {
  __shared__ __align__(16) float4 buf[4][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < 4 * 64; k += blockDim.x) buf[k / 64][k % 64] = make_float4(k, k + 1, k + 2, k + 3);
  __syncthreads();
  const int grp = lane / (32 / U);
  float acc = 0.f;
  int j = grp * 3;   // distinct records (16 B apart * 3: different banks)
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int jj = (j + r * 7) & 63;
      const unsigned addr = (unsigned)__cvta_generic_to_shared(&buf[warp & 3][jj]);
      if (W == 16) {
        float a0, a1, a2, a3;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3) : "r"(addr));
        acc += a0 + a3;
      } else if (W == 8) {
        float a0, a1;
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(a0), "=f"(a1) : "r"(addr));
        acc += a0;
      } else {
        float a0;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(a0) : "r"(addr));
        acc += a0;
      }
    }
    j = (j + 5) & 63;   // independent of the loads: throughput, not latency
  }
  if (acc == 1.2345f) out[0] = acc;
}
template <int U, int W>
void run(int sms, const char* name) {
  float* out; cudaMalloc(&out, 4);
  const int iters = 4000; dim3 grid(sms * 8), block(256);
  bench<U, W><<<grid, block>>>(out, 10);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); bench<U, W><<<grid, block>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double loads = (double)grid.x * (block.x / 32) * iters * 8;
  printf("{\"mode\": \"%s\", \"ms\": %.3f, \"warp_loads_per_sm_per_clk\": %.3f}\n", name, ms, loads / (ms * 1e-3) / sms / (clk * 1e3));
  cudaFree(out);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 16>(sms, "LDS.128 1 addr"); run<2, 16>(sms, "LDS.128 2 addr"); run<4, 16>(sms, "LDS.128 4 addr");
  run<8, 16>(sms, "LDS.128 8 addr"); run<1, 8>(sms, "LDS.64 1 addr"); run<4, 8>(sms, "LDS.64 4 addr");
  run<1, 4>(sms, "LDS.32 1 addr"); run<4, 4>(sms, "LDS.32 4 addr");
  return 0;
}
