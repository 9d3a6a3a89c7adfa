// k4_composite.cu — K4: per-tile front-to-back alpha compositing.
//
// north_star / readings R12-R16 (3DGS formulation, cited P:212; outputs per P:225):
//   for each pixel, over its tile's list in (depth, id) order:
//     alpha = min(0.99, o exp(power)); skip if alpha < 1/255;
//     tT = T (1 - alpha); stop (before blending) if tT < 1e-4;
//     w = alpha T; C += w rgb; D += w z; T = tT;
//   RGB = C + T bg, depth = D, alpha = 1 - T.
// power is evaluated in log2 units through the whitening factor written by K1:
//   arg = log2(o) - ((p dx)^2 + (q dx + r dy)^2)   (= log2(o e^power))
// so "alpha < 1/255" is the test arg < log2(1/255), decided before any exp2; the exp2 is
// the MUFU ex2.approx (reading R27).
//
// One CTA per (frame, 16x16 tile), one pixel per thread; records are staged through shared
// memory 256 at a time; the CTA stops as soon as every pixel has terminated
// (__syncthreads_count vote on the per-thread done flags).
#include "gsb_common.cuh"
#include "gsb_kernels.cuh"

namespace gsb {

constexpr int kCompThreads = 256;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(kCompThreads) k4_composite(CompositeArgs a) {
  __shared__ float4 s0[kCompThreads], s1[kCompThreads], s2[kCompThreads];
  __shared__ unsigned long long red[kCompThreads / 32];
  const int fl = a.fs + blockIdx.x / a.n_tiles;
  const int t = blockIdx.x % a.n_tiles;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int tid = threadIdx.x;
  const int px = tx * kTile + (tid & 15), py = ty * kTile + (tid >> 4);
  const bool inside = px < a.width && py < a.height;
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  const uint64_t start = a.frame_base[fl] - a.key_base + off[t];
  const int len = (int)(off[t + 1] - off[t]);
  const float4* rec = a.rec + (size_t)fl * a.n * 3;
  const float pxc = (float)px + 0.5f, pyc = (float)py + 0.5f;

  float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f, dep = 0.f;
  bool done = !inside;
  int n_eval = len;
  for (int b = 0; b < len; b += kCompThreads) {
    const int k = b + tid;
    if (k < len) {
      const uint32_t slot = a.sorted[start + k];
      const float4* r = rec + (size_t)slot * 3;
      s0[tid] = __ldg(r);
      s1[tid] = __ldg(r + 1);
      s2[tid] = __ldg(r + 2);
    }
    __syncthreads();
    if (!done) {
      const int cnt = min(kCompThreads, len - b);
      for (int j = 0; j < cnt; ++j) {
        const float4 r0 = s0[j];
        const float4 r1 = s1[j];
        const float dx = r0.x - pxc, dy = r0.y - pyc;
        const float t1 = r0.z * dx;
        const float t2 = fmaf(r0.w, dx, r1.x * dy);
        const float arg = fmaf(-t1, t1, fmaf(-t2, t2, r1.y));
        if (arg < kLog2AlphaMin) continue;  // alpha < 1/255: skipped
        const float alpha = fminf(kAlphaMax, ex2_approx(arg));
        const float tT = T * (1.f - alpha);
        if (tT < kTermT) {
          done = true;
          n_eval = b + j + 1;
          break;
        }
        const float w = alpha * T;
        const float4 r2 = s2[j];
        cr = fmaf(w, r2.x, cr);
        cg = fmaf(w, r2.y, cg);
        cb = fmaf(w, r2.z, cb);
        dep = fmaf(w, r1.z, dep);
        T = tT;
      }
    }
    if (__syncthreads_count(done) == kCompThreads) break;
  }

  if (inside) {
    const size_t f = (size_t)(a.f0 + fl);
    const size_t plane = (size_t)a.width * a.height;
    const size_t p = (size_t)py * a.width + px;
    float* rgb = a.out_rgb + f * 3 * plane;
    rgb[p] = fmaf(T, a.bg0, cr);
    rgb[plane + p] = fmaf(T, a.bg1, cg);
    rgb[2 * plane + p] = fmaf(T, a.bg2, cb);
    if (a.out_depth) a.out_depth[f * plane + p] = dep;
    if (a.out_alpha) a.out_alpha[f * plane + p] = 1.f - T;
    if (a.out_n_eval) a.out_n_eval[f * plane + p] = n_eval;
  }
  if (a.stat_pairs) {
    unsigned long long v = inside ? (unsigned long long)n_eval : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < kCompThreads / 32; ++w) s += red[w];
      if (s) atomicAdd(a.stat_pairs, s);
    }
  }
}

void launch_k4_composite(const CompositeArgs& a, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0) return;
  k4_composite<<<(unsigned)nf * a.n_tiles, kCompThreads, 0, s>>>(a);
}

}  // namespace gsb
