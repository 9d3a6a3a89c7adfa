// k6_encode.cu — K6: the observation encoding as a standalone pass over rendered fp32 frames,
// with the motion blur of reading R33 in front of the image DR / 8-bit encoding of reading R31
// (§8(f) row 4; "injection of image noise and motion blur").
//
// Blur needs a neighbourhood that crosses tiles, so it cannot live in K4's per-pixel store like
// the plain R31 epilogue; K6 reads the fp32 composite back (12 B/px, coalesced; the taps of
// neighbouring threads overlap in L1/L2), blurs, encodes and writes 3 B/px (+ fp16 depth).
// Without blur it produces exactly the codes of gsb_render_obs (same r31_encode).
#include "gsb_kernels.cuh"
#include "k4_common.cuh"

namespace gsb {

constexpr int kMaxBlur = 64;

__device__ __forceinline__ int floordiv(int a, int b) {   // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

constexpr int kEncThreads = 128;

// grid (ceil(W / 128), H, F): one thread per pixel, rows and frames from the grid (no divisions)
__global__ void __launch_bounds__(kEncThreads) k6_encode(EncodeArgs a) {
  __shared__ int2 tap[2 * kMaxBlur + 1];   // the frame's tap offsets (R33), computed once per CTA
  const int f = blockIdx.z, y = blockIdx.y;
  const int x = blockIdx.x * kEncThreads + threadIdx.x;
  const int64_t plane = (int64_t)a.width * a.height;
  const int64_t p = (int64_t)y * a.width + x;
  int bx = 0, by = 0;
  if (a.blur) {
    const int2 b = __ldg(reinterpret_cast<const int2*>(a.blur) + f);
    bx = min(max(b.x, -kMaxBlur), kMaxBlur);   // documented clamp of the extents
    by = min(max(b.y, -kMaxBlur), kMaxBlur);
  }
  const int L = max(abs(bx), abs(by)) + 1;
  if (L > 1) {
    const int d = 2 * (L - 1);
    for (int k = threadIdx.x; k < L; k += kEncThreads)
      tap[k] = make_int2(floordiv(2 * k * bx + (L - 1), d) - floordiv(bx, 2),
                         floordiv(2 * k * by + (L - 1), d) - floordiv(by, 2));
    __syncthreads();
  }
  if (x >= a.width) return;
  float4 dr = make_float4(1.f, 1.f, 0.f, 0.f);
  if (a.dr) dr = __ldg(reinterpret_cast<const float4*>(a.dr) + f);
  const uint64_t gf = (uint64_t)a.frame_offset + f;
  const uint32_t kseed = mix32(a.seed ^ mix32(a.step));
  const float* src = a.rgb + (size_t)f * 3 * plane;
  float v[3];
  if (L == 1) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) v[ch] = __ldg(src + ch * plane + p);
  } else {
    // reading R33: per channel a tap-order binary32 sum over edge-clamped samples, then / L
    float acc[3] = {0.f, 0.f, 0.f};
    for (int k = 0; k < L; ++k) {
      const int2 o = tap[k];
      const int xk = min(max(x + o.x, 0), a.width - 1);
      const int yk = min(max(y + o.y, 0), a.height - 1);
      const float* c = src + (int64_t)yk * a.width + xk;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) acc[ch] = __fadd_rn(acc[ch], __ldg(c + ch * plane));
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) v[ch] = __fdiv_rn(acc[ch], (float)L);
  }
  uint8_t* o8 = a.out_rgb8 + (size_t)f * 3 * plane;
  const uint64_t idx0 = ((gf * (uint64_t)a.height + (uint64_t)y) * (uint64_t)a.width + (uint64_t)x) * 3u;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) o8[ch * plane + p] = r31_encode(v[ch], dr, idx0 + ch, kseed);
  if (a.depth) {
    const float dv = __ldg(a.depth + (size_t)f * plane + p);
    if (a.out_depth16) a.out_depth16[(size_t)f * plane + p] = __half_as_ushort(__float2half_rn(dv));
    else if (a.out_depth32) a.out_depth32[(size_t)f * plane + p] = dv;
  }
}

void launch_k6_encode(const EncodeArgs& a, cudaStream_t s) {
  if (a.n_frames <= 0 || a.width <= 0 || a.height <= 0) return;
  const dim3 grid((unsigned)((a.width + kEncThreads - 1) / kEncThreads), (unsigned)a.height, (unsigned)a.n_frames);
  k6_encode<<<grid, kEncThreads, 0, s>>>(a);
}

}  // namespace gsb
