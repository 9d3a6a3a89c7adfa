// gsb_common.cuh — device-side data layout and exact-arithmetic helpers of libgsb.
//
// Shared by the kernels K0-K4 only (NOT by the CPU oracle, which is written independently).
// Data layout in HBM:
//   template (K5, read-only, shared by every env):  SoA float4 planes of N entries
//     (internal order: by body, then Morton order of the template position)
//     g_mean[N]  = (x, y, z, max_c s_c^2)
//     g_ids[N]   = (creation index = the id of reading R10, body; -1 = static)
//     g_L0[N]    = (L00, L01, L02, L10)   L = R(q_i) diag(s_i): Sigma_local = L L^T
//     g_L1[N]    = (L11, L12, L20, L21)
//     g_L2[N]    = (L22, opacity, kappa = 2 ln(255 o), log2 o)
//     g_sh[P][N] = SH coefficients, P = 3 ceil((D+1)^2 / 4) float4 planes: per group of four
//                  coefficients k..k+3 (degree order), (r_k, g_k, r_k+1, g_k+1), (r_k+2, g_k+2,
//                  r_k+3, g_k+3), (b_k .. b_k+3): the (r, g) pairs feed packed FFMA2s in K1
//   per frame-body table (K0 -> K1): 4 float4 = rows 0 and 1 of M | m interleaved as
//     (M00, M10, M01, M11), (M02, M12, m0, m1) (packed (x, y) pairs in K1), row 2 | m2, c_body
//   projected record (K1 -> K4), 48 B at [frame][internal index]:
//     R0 = (u, v, p', q')          whitening factor of Sigma2D^-1 scaled by sqrt(log2(e)/2)
//     R1 = (r', log2 o, ex, ey)    half-extents of the alpha >= 1/255 box (R8), inflated
//     R2 = (r, g, b, z)            z = fp32 depth key (R11)
//   emission entry (K1 -> K2b), 8 B at [frame][internal index]: (bits(z), rect) with
//     rect = tx0 | tx1 << 8 | ty0 << 16 | ty1 << 24; the key's id comes from the template
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gsb {

constexpr int kTile = 16;             // reading R9: tiles fixed at 16x16 pixels
constexpr int kRecQuads = 3;          // float4s per projected record
constexpr int kMaxDim = 4096;         // width, height <= 4096 -> tile coords fit in 8 bits
constexpr float kAlphaMax = 0.99f;    // north_star: alpha clamped at 0.99
constexpr float kTermT = 1e-4f;       // reading R13
// log2(1/255): alpha >= 1/255  <=>  log2(o) - Q/2 * log2(e) >= log2(1/255)
constexpr float kLog2AlphaMin = -7.99435343685885793f;

// ---- packed binary32 pairs (sm_100a FFMA2 / FADD2 / FMUL2) ------------------------------------
// Two independent binary32 values (K4: a thread's two pixels; K1: the x and y rows of the
// projection, the r and g SH channels) held as a pair in one 64-bit register pair and updated by
// one packed instruction instead of two.  Each half is an IEEE binary32 RN operation, so the
// results equal the scalar code's bit for bit; ptxas folds a scalar operand into a broadcast
// (`R.F32`) and a negation into the operand.
typedef float2 f32x2;

__device__ __forceinline__ f32x2 pk2(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ float2 up2(f32x2 v) { return v; }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ f32x2 nfma2(f32x2 a, f32x2 b, f32x2 c) {   // fma(-a, b, c) per half
  return __ffma2_rn(make_float2(-a.x, -a.y), b, c);
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f32x2 bc2(float x) { return make_float2(x, x); }   // broadcast

struct __align__(16) FrameCam {
  float fx, fy, cx, cy;
  float limx, limy;  // reading R6: 1.3 * W / (2 fx), 1.3 * H / (2 fy)
  float kx, ky;      // 1 + limx^2, 1 + limy^2 (K1's conservative screen-cull bound)
};

// ---------------------------------------------------------------- reading R11 (exact chain)
// Each op is a separately rounded IEEE binary32 op; fmas are explicit.
__device__ __forceinline__ void r11_rot(float qw, float qx, float qy, float qz, float R[3][3]) {
  const float xx = __fmul_rn(qx, qx), yy = __fmul_rn(qy, qy), zz = __fmul_rn(qz, qz);
  const float xy = __fmul_rn(qx, qy), xz = __fmul_rn(qx, qz), yz = __fmul_rn(qy, qz);
  const float wx = __fmul_rn(qw, qx), wy = __fmul_rn(qw, qy), wz = __fmul_rn(qw, qz);
  R[0][0] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(yy, zz)));
  R[0][1] = __fmul_rn(2.0f, __fsub_rn(xy, wz));
  R[0][2] = __fmul_rn(2.0f, __fadd_rn(xz, wy));
  R[1][0] = __fmul_rn(2.0f, __fadd_rn(xy, wz));
  R[1][1] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(xx, zz)));
  R[1][2] = __fmul_rn(2.0f, __fsub_rn(yz, wx));
  R[2][0] = __fmul_rn(2.0f, __fsub_rn(xz, wy));
  R[2][1] = __fmul_rn(2.0f, __fadd_rn(yz, wx));
  R[2][2] = __fsub_rn(1.0f, __fmul_rn(2.0f, __fadd_rn(xx, yy)));
}

__device__ __forceinline__ float r11_depth(float4 row2, float mx, float my, float mz) {
  return __fmaf_rn(row2.x, mx, __fmaf_rn(row2.y, my, __fmaf_rn(row2.z, mz, row2.w)));
}

// ---------------------------------------------------------------- reading R9 (tile rect)
// Returns false when culled.  Tile rect written as [tx0, tx1] x [ty0, ty1].
__device__ __forceinline__ bool r9_rect(float u, float v, float sxx, float syy, float kappa,
                                        int width, int height, int& tx0, int& tx1, int& ty0,
                                        int& ty1) {
  const float rx = __fsqrt_rn(__fmul_rn(kappa, sxx));
  const float ry = __fsqrt_rn(__fmul_rn(kappa, syy));
  const float xl = __fsub_rn(__fsub_rn(u, rx), 0.5f);
  const float xh = __fsub_rn(__fadd_rn(u, rx), 0.5f);
  const float yl = __fsub_rn(__fsub_rn(v, ry), 0.5f);
  const float yh = __fsub_rn(__fadd_rn(v, ry), 0.5f);
  if (!(isfinite(xl) && isfinite(xh) && isfinite(yl) && isfinite(yh))) return false;
  const float pxl = fmaxf(ceilf(xl), 0.0f);
  const float pxh = fminf(floorf(xh), (float)(width - 1));
  const float pyl = fmaxf(ceilf(yl), 0.0f);
  const float pyh = fminf(floorf(yh), (float)(height - 1));
  if (!(pxl <= pxh) || !(pyl <= pyh)) return false;
  tx0 = ((int)pxl) >> 4;
  tx1 = ((int)pxh) >> 4;
  ty0 = ((int)pyl) >> 4;
  ty1 = ((int)pyh) >> 4;
  return true;
}

__device__ __forceinline__ uint32_t pack_rect(int tx0, int tx1, int ty0, int ty1) {
  return (uint32_t)tx0 | ((uint32_t)tx1 << 8) | ((uint32_t)ty0 << 16) | ((uint32_t)ty1 << 24);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated compaction: returns the slot of this lane (valid only if `take`).
__device__ __forceinline__ int warp_compact_slot(bool take, int* counter) {
  const unsigned mask = __ballot_sync(0xffffffffu, take);
  if (mask == 0) return -1;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(mask & lanemask_lt());
}

// Add 1 to counter[t] for every tile t of this lane's rect (when `has`), aggregated over the
// warp.  The warp's rects are Morton-coherent, so their union box is usually small: when it holds
// at most 32 tiles, each lane counts its tiles into the warp's 32-entry shared scratch (shared
// atomics) and lane j then adds the count of box tile j with one global RED — all of the warp's
// distinct tiles in one instruction.  Otherwise lanes whose r-th tile coincides share one atomic
// per round (__match_any_sync).  Rects with more than kBigRect tiles are walked by the whole warp
// cooperatively afterwards.  All 32 lanes of the warp must call this; `scratch` = 32 words of
// shared memory private to the warp (or nullptr: rounds only).
constexpr int kBigRect = 8;
#ifndef GSB_TILE_DIV
#define GSB_TILE_DIV 0
#endif
#ifndef GSB_UNION_BOX
#define GSB_UNION_BOX 1   // 0: match_any rounds only (A/B comparisons)
#endif

struct UnionBox {
  int x0, y0, w, n;   // origin, width and tile count of the warp's union box (n = 0: empty)
  // tile index of box entry j < n (row-major in the box), without an integer division:
  // (j + 0.5) / w is at least 1 / (2w) >= 1/64 from an integer, far above the fp32 error of a
  // fast division (j, w <= 32)
  __device__ __forceinline__ int tile_of(int j, int tiles_x) const {
#if GSB_TILE_DIV
    return (y0 + j / w) * tiles_x + x0 + j % w;
#else
    const int yy = (int)__fdividef((float)j + 0.5f, (float)w);   // 2-ulp division, far inside the margin
    return (y0 + yy) * tiles_x + x0 + (j - yy * w);
#endif
  }
};

__device__ __forceinline__ UnionBox warp_union_box(bool part, int tx0, int tx1, int ty0, int ty1) {
  const unsigned FULL = 0xffffffffu;
  UnionBox b;
  const unsigned x0 = __reduce_min_sync(FULL, part ? (unsigned)tx0 : 0xffffu);
  const unsigned y0 = __reduce_min_sync(FULL, part ? (unsigned)ty0 : 0xffffu);
  const unsigned x1 = __reduce_max_sync(FULL, part ? (unsigned)tx1 : 0u);
  const unsigned y1 = __reduce_max_sync(FULL, part ? (unsigned)ty1 : 0u);
  b.x0 = (int)x0; b.y0 = (int)y0;
  b.w = (int)x1 - (int)x0 + 1;
  b.n = x0 == 0xffffu ? 0 : b.w * ((int)y1 - (int)y0 + 1);
  return b;
}

__device__ __forceinline__ void warp_tile_count(bool has, uint32_t rect, int tiles_x, int* counter,
                                                uint32_t* scratch = nullptr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int tx0 = rect & 0xff, tx1 = (rect >> 8) & 0xff, ty0 = (rect >> 16) & 0xff, ty1 = rect >> 24;
  const int nt = has ? (tx1 - tx0 + 1) * (ty1 - ty0 + 1) : 0;
  const bool big = nt > kBigRect;
  const bool part = nt > 0 && !big;
  const UnionBox ub = (GSB_UNION_BOX && scratch) ? warp_union_box(part, tx0, tx1, ty0, ty1) : UnionBox{0, 0, 0, 64};
  if (ub.n > 0 && ub.n <= 32) {
    scratch[lane] = 0u;
    __syncwarp();
    if (part)
      for (int y = ty0; y <= ty1; ++y)
        for (int x = tx0; x <= tx1; ++x) atomicAdd(&scratch[(y - ub.y0) * ub.w + (x - ub.x0)], 1u);
    __syncwarp();
    const uint32_t c = scratch[lane];
    if (lane < ub.n && c) atomicAdd(counter + ub.tile_of(lane, tiles_x), (int)c);
    __syncwarp();   // scratch free for the caller's next use
  } else if (ub.n > 0) {
    const int rounds = __reduce_max_sync(FULL, part ? nt : 0);
    int tx = tx0, ty = ty0;  // this lane's r-th tile, stepped row-major (no division)
    for (int r = 0; r < rounds; ++r) {
      const bool act = part && r < nt;
      const int t = act ? ty * tiles_x + tx : -1 - lane;
      const unsigned peers = __match_any_sync(FULL, t);
      if (act && lane == __ffs(peers) - 1) atomicAdd(counter + t, __popc(peers));
      if (++tx > tx1) { tx = tx0; ++ty; }
    }
  }
  unsigned bm = __ballot_sync(FULL, big);
  while (bm) {
    const int j = __ffs(bm) - 1;
    bm &= bm - 1;
    const uint32_t rj = __shfl_sync(FULL, rect, j);
    const int jx0 = rj & 0xff, jx1 = (rj >> 8) & 0xff, jy0 = (rj >> 16) & 0xff, jy1 = rj >> 24;
    for (int y = jy0; y <= jy1; ++y)
      for (int x = jx0 + lane; x <= jx1; x += 32) atomicAdd(counter + y * tiles_x + x, 1);
  }
}

}  // namespace gsb
