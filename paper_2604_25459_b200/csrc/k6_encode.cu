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

__global__ void __launch_bounds__(256) k6_encode(EncodeArgs a) {
  const int f = blockIdx.y;
  const int64_t plane = (int64_t)a.width * a.height;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= plane) return;
  const int y = (int)(p / a.width), x = (int)(p % a.width);
  int bx = 0, by = 0;
  if (a.blur) {
    const int2 b = __ldg(reinterpret_cast<const int2*>(a.blur) + f);
    bx = min(max(b.x, -kMaxBlur), kMaxBlur);   // documented clamp of the extents
    by = min(max(b.y, -kMaxBlur), kMaxBlur);
  }
  const int L = max(abs(bx), abs(by)) + 1;
  const int d = 2 * (L - 1);
  const int sx = floordiv(bx, 2), sy = floordiv(by, 2);
  float4 dr = make_float4(1.f, 1.f, 0.f, 0.f);
  if (a.dr) dr = __ldg(reinterpret_cast<const float4*>(a.dr) + f);
  const uint64_t gf = (uint64_t)a.frame_offset + f;
  const uint32_t kseed = mix32(a.seed ^ mix32(a.step));
  const float* src = a.rgb + (size_t)f * 3 * plane;
  uint8_t* o8 = a.out_rgb8 + (size_t)f * 3 * plane;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float* c = src + ch * plane;
    float v;
    if (L == 1) {
      v = __ldg(c + p);
    } else {   // reading R33: tap-order binary32 sum over edge-clamped samples, then / L
      float acc = 0.f;
      for (int k = 0; k < L; ++k) {
        const int xk = min(max(x + floordiv(2 * k * bx + (L - 1), d) - sx, 0), a.width - 1);
        const int yk = min(max(y + floordiv(2 * k * by + (L - 1), d) - sy, 0), a.height - 1);
        acc = __fadd_rn(acc, __ldg(c + (int64_t)yk * a.width + xk));
      }
      v = __fdiv_rn(acc, (float)L);
    }
    const uint64_t idx = ((gf * (uint64_t)a.height + (uint64_t)y) * (uint64_t)a.width + (uint64_t)x) * 3u + ch;
    o8[ch * plane + p] = r31_encode(v, dr, idx, kseed);
  }
  if (a.depth) {
    const float dv = __ldg(a.depth + (size_t)f * plane + p);
    if (a.out_depth16) a.out_depth16[(size_t)f * plane + p] = __half_as_ushort(__float2half_rn(dv));
    else if (a.out_depth32) a.out_depth32[(size_t)f * plane + p] = dv;
  }
}

void launch_k6_encode(const EncodeArgs& a, cudaStream_t s) {
  const int64_t plane = (int64_t)a.width * a.height;
  if (a.n_frames <= 0 || plane == 0) return;
  k6_encode<<<dim3((unsigned)((plane + 255) / 256), (unsigned)a.n_frames), 256, 0, s>>>(a);
}

}  // namespace gsb
