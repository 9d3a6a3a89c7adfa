// k4_common.cuh — device helpers shared by the compositing kernels (k4_composite.cu: one CTA
// per tile; k4b_blend.cu: tile sort + persistent per-warp compositing).
#pragma once
#include <cuda_fp16.h>

#include "gsb_common.cuh"
#include "gsb_kernels.cuh"

namespace gsb {

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16s(uint32_t smem_addr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Front-to-back blend of one list entry into one pixel (readings R12-R14).  alpha is 0 unless
// `use` (alpha >= 1/255 for a live pixel); then T never drops below 1e-4 without terminating,
// so an unused entry leaves every accumulator unchanged.  A pixel that terminates gets its
// centre moved to kFar: every later quadratic form is huge and every later entry fails the
// alpha test, without a per-pixel "done" test in the hot loop.
constexpr float kFar = 1e20f;
constexpr float kScoreFix = 67108864.f;  // 2^26: warp-level fixed point of the score sums

__device__ __forceinline__ float blend(bool use, float arg, const float4& r2, float& T, float& cr, float& cg,
                                       float& cb, float& dep, float& pyc, int& n_eval, int idx) {
  const float alpha = use ? fminf(kAlphaMax, ex2_approx(arg)) : 0.f;
  const float w = alpha * T;
  const float tT = T - w;                       // T (1 - alpha)
  if (tT >= kTermT) {
    cr = fmaf(w, r2.x, cr);
    cg = fmaf(w, r2.y, cg);
    cb = fmaf(w, r2.z, cb);
    dep = fmaf(w, r2.w, dep);
    T = tT;
    return w;                                   // blended weight (reading R30 scores)
  }
  n_eval = idx + 1;                             // stop before blending (R13)
  pyc = kFar;
  return 0.f;
}

// blend() for a thread's two pixels at once.  The termination test's bookkeeping (n_eval,
// moving the pixel centre away) runs in a warp-uniform branch taken only when some lane
// terminates at this entry; otherwise the accumulators take unpredicated FMAs whose weight is 0
// for unused pixels (fma(0, x, c) == c: the accumulators are >= +0), so the result equals
// blend() bit for bit.  Returns the blended weights (reading R30 scores).
__device__ __forceinline__ float2 blend2(bool use0, float arg0, bool use1, float arg1, const float4& r2, float& T0,
                                         float& r0, float& g0, float& b0, float& d0, float& pyc0, int& ne0,
                                         float& T1, float& r1, float& g1, float& b1, float& d1, float& pyc1,
                                         int& ne1, int idx) {
  float w0 = (use0 ? fminf(kAlphaMax, ex2_approx(arg0)) : 0.f) * T0;
  float w1 = (use1 ? fminf(kAlphaMax, ex2_approx(arg1)) : 0.f) * T1;
  float t0 = T0 - w0, t1 = T1 - w1;                    // T (1 - alpha)
  const bool s0 = t0 < kTermT, s1 = t1 < kTermT;       // stop before blending (R13)
  if (__any_sync(0xffffffffu, s0 || s1)) {
    if (s0) { ne0 = idx + 1; pyc0 = kFar; w0 = 0.f; t0 = T0; }
    if (s1) { ne1 = idx + 1; pyc1 = kFar; w1 = 0.f; t1 = T1; }
  }
  r0 = fmaf(w0, r2.x, r0); g0 = fmaf(w0, r2.y, g0); b0 = fmaf(w0, r2.z, b0); d0 = fmaf(w0, r2.w, d0);
  r1 = fmaf(w1, r2.x, r1); g1 = fmaf(w1, r2.y, g1); b1 = fmaf(w1, r2.z, b1); d1 = fmaf(w1, r2.w, d1);
  T0 = t0;
  T1 = t1;
  return make_float2(w0, w1);
}

// acc += a * (x, x)
__device__ __forceinline__ void acc2(f32x2& acc, f32x2 a, float x) { acc = __ffma2_rn(a, make_float2(x, x), acc); }

// blend2() on packed pairs: T = (T0, T1), the accumulators R, G, B, D = (pixel 0, pixel 1) and
// PYC = (pyc0, pyc1).  Same operations in the same order as blend2(), bit for bit.  The rare
// termination entry takes its own copy of the accumulation, so the common path has no merge of
// the weight and transmittance pairs (which would cost register-pair copies per entry).
// `argn` is the next entry's quadratic form, evaluated ahead with the current pixel centres; a
// pixel that terminates here has it set to -inf (alpha 0), as its moved centre would give.
// `idx_of()` gives the entry's list position; it is evaluated only when some pixel terminates.
template <class IdxFn>
__device__ __forceinline__ f32x2 blend2p(f32x2 arg, const float4& r2, f32x2& T, f32x2& R, f32x2& G, f32x2& B,
                                         f32x2& D, f32x2& PYC, int& ne0, int& ne1, IdxFn idx_of, f32x2& argn) {
  const float2 ag = up2(arg);
  const float a0 = ag.x >= kLog2AlphaMin ? fminf(kAlphaMax, ex2_approx(ag.x)) : 0.f;   // alpha >= 1/255
  const float a1 = ag.y >= kLog2AlphaMin ? fminf(kAlphaMax, ex2_approx(ag.y)) : 0.f;
  f32x2 w = mul2(pk2(a0, a1), T);
  const f32x2 t = sub2(T, w);                            // T (1 - alpha)
  const float2 tt = up2(t);
  const bool s0 = tt.x < kTermT, s1 = tt.y < kTermT;     // stop before blending (R13)
  if (__any_sync(0xffffffffu, s0 || s1)) {
    float2 ww = up2(w), tn = tt, pc = up2(PYC);
    const float2 T2 = up2(T);
    float2 an = up2(argn);
    const int idx = idx_of();
    if (s0) { ne0 = idx + 1; pc.x = kFar; ww.x = 0.f; tn.x = T2.x; an.x = -INFINITY; }
    if (s1) { ne1 = idx + 1; pc.y = kFar; ww.y = 0.f; tn.y = T2.y; an.y = -INFINITY; }
    w = pk2(ww.x, ww.y);
    PYC = pk2(pc.x, pc.y);
    argn = pk2(an.x, an.y);
    acc2(R, w, r2.x);
    acc2(G, w, r2.y);
    acc2(B, w, r2.z);
    acc2(D, w, r2.w);
    T = pk2(tn.x, tn.y);
  } else {
    acc2(R, w, r2.x);
    acc2(G, w, r2.y);
    acc2(B, w, r2.z);
    acc2(D, w, r2.w);
    T = t;
  }
  return w;
}

// Reading R31 noise: counter-based Irwin-Hall(4) of 22-bit lowbias32-hashed uniforms (exact
// integer arithmetic, so the oracle reproduces every draw); z * sqrt(3)/2^22 has unit variance.
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ float irwin_hall4(uint64_t idx, uint32_t kseed) {
  const uint32_t base = mix32((uint32_t)idx ^ mix32((uint32_t)(idx >> 32) ^ kseed));
  uint32_t s = 0;
#pragma unroll
  for (uint32_t j = 0; j < 4; ++j) s += mix32(base + j * 0x9E3779B9u) >> 10;
  return __fsub_rn((float)s, 8388608.f);   // (float)s exact: s < 2^24
}
constexpr float kNoiseS3 = 1.7320508075688772f / 4194304.f;   // sqrt(3) / 2^22 (power-of-2 divisor: exact)

// Reading R31 on one value: image DR (gain, contrast, brightness, noise_std) = dr, then the
// 8-bit code; binary32 RN ops in the order of oracle/obs.py.  idx = the value's noise counter.
__device__ __forceinline__ uint8_t r31_encode(float c, float4 dr, uint64_t idx, uint32_t kseed) {
  float v = __fadd_rn(__fmul_rn(__fsub_rn(__fmul_rn(c, dr.x), 0.5f), dr.y), 0.5f);
  v = __fadd_rn(v, dr.z);
  if (dr.w != 0.f) v = __fadd_rn(v, __fmul_rn(__fmul_rn(irwin_hall4(idx, kseed), kNoiseS3), dr.w));
  return (uint8_t)__float2uint_rn(__fmul_rn(__saturatef(v), 255.f));
}

// first index in sorted k[0..n) whose value is >= x
template <typename T, typename P>
__device__ __forceinline__ int lower_bound(P k, int n, T x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}


// Store one thread's two vertically adjacent pixels (px, py0) and (px, py0 + 1) of frame f:
// fp32 RGB = C + T bg (+ depth, alpha, n_eval), or the reading-R31 observation encoding.
__device__ __forceinline__ void store_pixels(const CompositeArgs& a, size_t f, int px, int py0, bool in0, bool in1,
                                             float T0, float r0c, float g0c, float b0c, float d0, int ne0,
                                             float T1, float r1c, float g1c, float b1c, float d1, int ne1) {
  const size_t plane = (size_t)a.width * a.height;
  if (a.obs_rgb8) {
    // observation epilogue, reading R31: image DR + uint8 RGB (+ fp16 depth), binary32 RN ops
    float4 dr = make_float4(1.f, 1.f, 0.f, 0.f);
    if (a.obs_dr) dr = *reinterpret_cast<const float4*>(a.obs_dr + f * 4);
    const uint64_t gf = (uint64_t)a.obs_frame_offset + f;
    const uint32_t kseed = mix32(a.obs_seed ^ mix32(a.obs_step));
    uint8_t* o8 = a.obs_rgb8 + f * 3 * plane;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool in = h ? in1 : in0;
      if (!in) continue;
      const int y = py0 + h;
      const size_t p = (size_t)y * a.width + px;
      const float T = h ? T1 : T0;
      const float cc[3] = {fmaf(T, a.bg0, h ? r1c : r0c), fmaf(T, a.bg1, h ? g1c : g0c), fmaf(T, a.bg2, h ? b1c : b0c)};
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const uint64_t idx = ((gf * (uint64_t)a.height + (uint64_t)y) * (uint64_t)a.width + (uint64_t)px) * 3u + ch;
        o8[ch * plane + p] = r31_encode(cc[ch], dr, idx, kseed);
      }
      const float d = h ? d1 : d0;
      if (a.obs_depth16) a.obs_depth16[f * plane + p] = __half_as_ushort(__float2half_rn(d));
      else if (a.out_depth) a.out_depth[f * plane + p] = d;
      if (a.out_alpha) a.out_alpha[f * plane + p] = 1.f - T;
      if (a.out_n_eval) a.out_n_eval[f * plane + p] = h ? ne1 : ne0;
    }
  } else {
    float* rgb = a.out_rgb + f * 3 * plane;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool in = h ? in1 : in0;
      if (!in) continue;
      const size_t p = (size_t)(py0 + h) * a.width + px;
      const float T = h ? T1 : T0;
      rgb[p] = fmaf(T, a.bg0, h ? r1c : r0c);
      rgb[plane + p] = fmaf(T, a.bg1, h ? g1c : g0c);
      rgb[2 * plane + p] = fmaf(T, a.bg2, h ? b1c : b0c);
      if (a.out_depth) a.out_depth[f * plane + p] = h ? d1 : d0;
      if (a.out_alpha) a.out_alpha[f * plane + p] = 1.f - T;
      if (a.out_n_eval) a.out_n_eval[f * plane + p] = h ? ne1 : ne0;
    }
  }
}

}  // namespace gsb
