// Microbenchmark: per-SM-per-clock throughput of the pipes K4b's per-pair work runs on (sm_100a):
// FFMA vs FFMA2 (fma.rn.f32x2) on the FMA pipe, FMNMX and FSETP on the ALU pipe, MUFU.EX2 on XU.
// Each thread runs 16 independent chains; reports thread-operations per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ float ffma1(float a, float b, float c) {
  float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r;
}
__device__ __forceinline__ float fmnmx(float a, float b) {
  float r; asm volatile("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ float fmxmx(float a, float b) {
  float r; asm volatile("max.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r;
}
template <int MODE>
__global__ void bench(float* out, int iters, float s) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      if (MODE == 0) {            // scalar FFMA: 2 per pair
        x[k] = ffma1(x[k], s, 1e-7f);
        x[k + 1] = ffma1(x[k + 1], s, 1e-7f);
      } else if (MODE == 1) {     // FFMA2: 1 per pair
        u64 v; asm("mov.b64 %0, {%1,%2};" : "=l"(v) : "f"(x[k]), "f"(x[k + 1]));
        u64 sv; asm("mov.b64 %0, {%1,%1};" : "=l"(sv) : "f"(s));
        u64 cv; asm("mov.b64 %0, {%1,%1};" : "=l"(cv) : "f"(1e-7f));
        v = ffma2(v, sv, cv);
        asm("mov.b64 {%0,%1}, %2;" : "=f"(x[k]), "=f"(x[k + 1]) : "l"(v));
      } else if (MODE == 2) {     // FFMA2 + one scalar FMNMX per pair (mixed issue)
        u64 v; asm("mov.b64 %0, {%1,%2};" : "=l"(v) : "f"(x[k]), "f"(x[k + 1]));
        u64 sv; asm("mov.b64 %0, {%1,%1};" : "=l"(sv) : "f"(s));
        u64 cv; asm("mov.b64 %0, {%1,%1};" : "=l"(cv) : "f"(1e-7f));
        v = ffma2(v, sv, cv);
        asm("mov.b64 {%0,%1}, %2;" : "=f"(x[k]), "=f"(x[k + 1]) : "l"(v));
        x[k] = fmnmx(x[k], 1e30f);
      } else if (MODE == 4) {     // FMNMX only (ALU pipe): 2 per pair (min then max: no FMNMX3 merge)
        x[k] = (it & 1) ? fmnmx(x[k], s) : fmxmx(x[k], -s);
        x[k + 1] = (it & 1) ? fmnmx(x[k + 1], s) : fmxmx(x[k + 1], -s);
      } else if (MODE == 5) {     // MUFU.EX2 only (XU pipe): 2 per pair
        float r0, r1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(x[k]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(x[k + 1]));
        x[k] = r0 * 1e-30f; x[k + 1] = r1 * 1e-30f;
      } else {                    // scalar FFMA x2 + FMNMX per pair
        x[k] = ffma1(x[k], s, 1e-7f);
        x[k + 1] = ffma1(x[k + 1], s, 1e-7f);
        x[k] = fmnmx(x[k], 1e30f);
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc += x[k];
  if (acc == 12345.f) out[0] = acc;
}
template <int MODE>
double run(int sms, int iters, const char* name) {
  float* out; cudaMalloc(&out, 4);
  dim3 grid(sms * 8), block(256);
  bench<MODE><<<grid, block>>>(out, 10, 0.999f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<MODE><<<grid, block>>>(out, iters, 0.999f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz
  double fmas = (double)grid.x * block.x * iters * 16;
  double per_sm_clk = fmas / (ms * 1e-3) / sms / (clk * 1e3);
  printf("{\"mode\": \"%s\", \"ms\": %.3f, \"ops_per_sm_per_clk\": %.1f, \"clock_khz\": %d}\n", name, ms, per_sm_clk, clk);
  cudaFree(out);
  return per_sm_clk;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms, 20000, "FFMA");
  run<1>(sms, 20000, "FFMA2");
  run<2>(sms, 20000, "FFMA2+FMNMX/pair");
  run<3>(sms, 20000, "FFMA x2+FMNMX/pair");
  run<4>(sms, 20000, "FMNMX");
  run<5>(sms, 5000, "MUFU.EX2 (+1 FMUL each)");
  return 0;
}
