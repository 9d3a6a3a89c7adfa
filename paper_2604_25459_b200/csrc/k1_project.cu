// k1_project.cu — K0 (per-(frame, body) RLGK transforms) and K1 (fused pose transform,
// EWA projection, 2D covariance, SH colour, compaction and tile histogram).
//
// PAPER.md App. B.2: RLGK moves every Gaussian of body k by that env's pose,
//   p_world = R(q_k) p_local + t_k, q_world = q_k (x) q_local  (Eqs.).
// Alg. 1 materialises P_world, Q_world for all B x M Gaussians (l.12-15); here the
// transform is folded into the camera transform per (frame, body) — K0 computes
//   M = W_f R(q_k),  m = W_f t_k + t_f,  c_body = R(q_k)^T (c_f - t_k)
// once per (frame, body), and K1 applies x_c = M mu_local + m per (frame, Gaussian), so the
// B x M world state is never written (reading R20).  Sigma_world = R(q_k) Sigma_local R(q_k)^T
// (reading R23) enters as the factor M L with Sigma_local = L L^T.
//
// K1 is Gaussian-major: one thread owns one template Gaussian (its parameters stay in
// registers) and loops over the E frames of a chunk, so the shared read-only template (K5)
// is read from HBM once per chunk, not once per frame.
#include <algorithm>
#include <cstdlib>

#include "gsb_common.cuh"
#include "gsb_kernels.cuh"

namespace gsb {

// ------------------------------------------------------------------------------ K0
// Reading R29 (§8(f) row 1): a camera attached to body kb is given body->camera extrinsics
// B = [R_bc | t_bc]; its world->camera transform is the binary32 composition
//   W[r][c] = fma(B[r][0], Rk[c][0], fma(B[r][1], Rk[c][1], B[r][2] * Rk[c][2]))   (B Rk^T)
//   W[r][3] = fma(-W[r][0], tk0, fma(-W[r][1], tk1, fma(-W[r][2], tk2, B[r][3])))
// with Rk from the R11 quaternion chain, every op separately rounded.
__device__ __forceinline__ void r29_compose(const float* B, const float* pose, float W[12]) {
  float Rk[3][3];
  r11_rot(pose[3], pose[4], pose[5], pose[6], Rk);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c)
      W[r * 4 + c] = __fmaf_rn(B[r * 4 + 0], Rk[c][0],
                               __fmaf_rn(B[r * 4 + 1], Rk[c][1], __fmul_rn(B[r * 4 + 2], Rk[c][2])));
    W[r * 4 + 3] = __fmaf_rn(-W[r * 4 + 0], pose[0],
                             __fmaf_rn(-W[r * 4 + 1], pose[1], __fmaf_rn(-W[r * 4 + 2], pose[2], B[r * 4 + 3])));
  }
}

__global__ void k0_setup(K0Rig rig, int n_frames, int n_cams, int n_bodies, int width, int height,
                         float4* __restrict__ table, FrameCam* __restrict__ cams) {
  const int nb1 = n_bodies + 1;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_frames * nb1) return;
  const int f = idx / nb1;
  const int k = idx % nb1 - 1;
  const int e = f / n_cams;
  const int cam = f % n_cams;
  // world->camera of this frame: given, or composed from the camera's body (R29)
  float W[12];
  const int crow = rig.cams_shared ? cam : f;   // static cameras: one camera set for every env
  const float* Wg = rig.cam_x + (size_t)crow * 12;
  const int kb = cam < kMaxRigCams ? rig.cam_body[cam] : -1;
  if (kb >= 0) {
    r29_compose(Wg, rig.poses + (size_t)e * rig.env_stride + (size_t)kb * rig.body_stride, W);
  } else {
    for (int j = 0; j < 12; ++j) W[j] = Wg[j];
  }
  float R[3][3] = {{1.f, 0.f, 0.f}, {0.f, 1.f, 0.f}, {0.f, 0.f, 1.f}};
  float t[3] = {0.f, 0.f, 0.f};
  if (k >= 0) {
    const float* p = rig.poses + (size_t)e * rig.env_stride + (size_t)k * rig.body_stride;
    r11_rot(p[3], p[4], p[5], p[6], R);
    t[0] = p[0]; t[1] = p[1]; t[2] = p[2];
  }
  float M[3][3], m[3];
  // rows 0, 1 by the same binary32 chain as the depth row (the LiDAR range key of reading R32
  // uses all three rows; for the cameras only row 2 must be exact)
  for (int r = 0; r < 2; ++r) {
    for (int c = 0; c < 3; ++c)
      M[r][c] = __fmaf_rn(W[r * 4 + 0], R[0][c], __fmaf_rn(W[r * 4 + 1], R[1][c], __fmul_rn(W[r * 4 + 2], R[2][c])));
    m[r] = __fmaf_rn(W[r * 4 + 0], t[0], __fmaf_rn(W[r * 4 + 1], t[1], __fmaf_rn(W[r * 4 + 2], t[2], W[r * 4 + 3])));
  }
  // depth row: exact chain, reading R11
  if (k < 0) {
    M[2][0] = W[8]; M[2][1] = W[9]; M[2][2] = W[10]; m[2] = W[11];
  } else {
    for (int c = 0; c < 3; ++c)
      M[2][c] = __fmaf_rn(W[8], R[0][c], __fmaf_rn(W[9], R[1][c], __fmul_rn(W[10], R[2][c])));
    m[2] = __fmaf_rn(W[8], t[0], __fmaf_rn(W[9], t[1], __fmaf_rn(W[10], t[2], W[11])));
  }
  // camera centre c_w = -W^T t_f, then into the body frame (reading R19)
  float cw[3], cb[3];
  for (int c = 0; c < 3; ++c) cw[c] = -(W[c] * W[3] + W[4 + c] * W[7] + W[8 + c] * W[11]);
  for (int c = 0; c < 3; ++c)
    cb[c] = R[0][c] * (cw[0] - t[0]) + R[1][c] * (cw[1] - t[1]) + R[2][c] * (cw[2] - t[2]);
  float4* o = table + (size_t)idx * 4;
  o[0] = make_float4(M[0][0], M[1][0], M[0][1], M[1][1]);   // rows 0 and 1 interleaved (gsb_common.cuh)
  o[1] = make_float4(M[0][2], M[1][2], m[0], m[1]);
  o[2] = make_float4(M[2][0], M[2][1], M[2][2], m[2]);
  o[3] = make_float4(cb[0], cb[1], cb[2], 0.f);
  if (k < 0 && cams) {   // cams == nullptr: LiDAR frames (no intrinsics)
    const float* K = rig.intr + (size_t)crow * 4;
    FrameCam fc;
    fc.fx = K[0]; fc.fy = K[1]; fc.cx = K[2]; fc.cy = K[3];
    fc.limx = 1.3f * (float)width / (2.0f * K[0]);
    fc.limy = 1.3f * (float)height / (2.0f * K[1]);
    fc.kx = 1.f + fc.limx * fc.limx;   // (1 + lim^2): the screen-cull bound's clamp factor
    fc.ky = 1.f + fc.limy * fc.limy;
    cams[f] = fc;
  }
}

// ------------------------------------------------------------------------------ SH (R18)
// SH planes: per group of four coefficients (r,g | r,g), (r,g | r,g), (b b b b) (gsb_common.cuh);
// the (r, g) pair accumulates by packed FFMA2 with the basis value broadcast, b by scalar FFMA,
// both in coefficient (degree) order.
template <int D>
__device__ __forceinline__ float3 sh_colour(const float4* __restrict__ g_sh, int64_t n, int64_t i,
                                            float x, float y, float z) {
  constexpr int NC = (D + 1) * (D + 1);
  constexpr int NG = (NC + 3) / 4;
  float4 q[3 * NG];
#pragma unroll
  for (int p = 0; p < 3 * NG; ++p) q[p] = __ldg(g_sh + (size_t)p * n + i);
  const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
  float Y[4 * NG];
#pragma unroll
  for (int k = 0; k < 4 * NG; ++k) Y[k] = 0.f;
  Y[0] = C0;
  if (D >= 1) {
    Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x;
  }
  if (D >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = 1.0925484305920792f * x * y;
    Y[5] = -1.0925484305920792f * y * z;
    Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
    Y[7] = -1.0925484305920792f * x * z;
    Y[8] = 0.5462742152960396f * (xx - yy);
    if (D >= 3) {
      Y[9] = -0.5900435899266435f * y * (3.f * xx - yy);
      Y[10] = 2.890611442640554f * x * y * z;
      Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
      Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
      Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
      Y[14] = 1.445305721320277f * z * (xx - yy);
      Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
    }
  }
  f32x2 rg = mul2(bc2(Y[0]), pk2(q[0].x, q[0].y));
  float b = Y[0] * q[2].x;
#pragma unroll
  for (int k = 1; k < NC; ++k) {
    const float4& p2 = q[3 * (k >> 2) + ((k >> 1) & 1)];   // the plane holding (r_k, g_k)
    const f32x2 c = (k & 1) ? pk2(p2.z, p2.w) : pk2(p2.x, p2.y);
    const float4& pb = q[3 * (k >> 2) + 2];
    const float cb = (k & 3) == 0 ? pb.x : (k & 3) == 1 ? pb.y : (k & 3) == 2 ? pb.z : pb.w;
    rg = fma2(bc2(Y[k]), c, rg);
    b = fmaf(Y[k], cb, b);
  }
  rg = add2(rg, bc2(0.5f));
  return make_float3(fmaxf(rg.x, 0.f), fmaxf(rg.y, 0.f), fmaxf(b + 0.5f, 0.f));
}

// accurate 2x2 determinant a*d - b*c (Kahan): error ~1.5 ulp of the result
__device__ __forceinline__ float det2(float a, float b, float c, float d) {
  const float w = b * c;
  const float e = fmaf(-b, c, w);
  const float f = fmaf(a, d, -w);
  return f + e;
}

// ------------------------------------------------------------------------------ K1
// fast sqrt for conservative bounds (x > 0; x * rsqrt(x), ~2 ulp)
__device__ __forceinline__ float sqrt_approx(float x) { return x * rsqrtf(x); }

template <int D, bool DEBUG>
__global__ void __launch_bounds__(128, 8) k1_project(K1Args a) {
  __shared__ uint32_t tile_scratch[4][32];   // warp_tile_count's per-warp union-box counts
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = i < a.n;
  float4 mean = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 l0 = make_float4(0.f, 0.f, 0.f, 0.f), l1 = l0, l2 = l0;
  int2 ids = make_int2(0, -1);
  if (in) {
    mean = __ldg(a.g_mean + i);
    l0 = __ldg(a.g_L0 + i);
    l1 = __ldg(a.g_L1 + i);
    l2 = __ldg(a.g_L2 + i);
    ids = __ldg(a.g_ids + i);
  }
  const int id = ids.x;     // creation index (reading R10 tie-break)
  const int body = ids.y;   // -1 = static
  const float smax2 = mean.w;  // largest squared scale: bounds the 2D extent (screen cull)
  const float L[3][3] = {{l0.x, l0.y, l0.z}, {l0.w, l1.x, l1.y}, {l1.z, l1.w, l2.x}};
  const float opac = l2.y, kappa = l2.z, log2o = l2.w;
  // reading R5: o < 1/255 is never visible (binary32 compare == the exact compare)
  const bool o_ok = in && (opac >= 1.0f / 255.0f);
  constexpr bool debug = DEBUG;
  const float wscale = 0.84932180028801904f;  // sqrt(log2(e) / 2)
  const float fw = (float)a.width, fh = (float)a.height;

  // frames of the chunk handled by this block row (gridDim.y rows split the frame loop so the
  // grid has enough CTAs when N is small)
  const int fpr = (a.n_frames + gridDim.y - 1) / gridDim.y;
  const int fl_lo = blockIdx.y * fpr, fl_hi = min(a.n_frames, fl_lo + fpr);
  for (int fl = fl_lo; fl < fl_hi; ++fl) {
    const int f = a.f0 + fl;
    const float4* tb = a.table + ((size_t)f * a.nb1 + (body + 1)) * 4;
    const float4 r2 = __ldg(tb + 2);
    const float z = r11_depth(r2, mean.x, mean.y, mean.z);   // exact fp32 key (R11)
    const bool keep = o_ok && (z > a.near_plane) && (z <= a.far_plane);
    bool vis = false;
    float u = 0.f, v = 0.f, pw = 0.f, qw = 0.f, rw = 0.f;
    float3 rgb = make_float3(0.f, 0.f, 0.f);
    int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
    if (keep || (debug && in)) {
      // rows 0 and 1 of M mu + m as one packed (x, y) chain (the table interleaves the rows)
      const float4 t0 = __ldg(tb + 0), t1 = __ldg(tb + 1);   // (M00, M10, M01, M11), (M02, M12, m0, m1)
      const float4* cp = reinterpret_cast<const float4*>(a.cams + f);
      const float4 c0 = cp[0], c1 = cp[1];                 // (fx, fy, cx, cy), (limx, limy, kx, ky)
      f32x2 xy = fma2(pk2(t1.x, t1.y), bc2(mean.z), pk2(t1.z, t1.w));
      xy = fma2(pk2(t0.z, t0.w), bc2(mean.y), xy);
      xy = fma2(pk2(t0.x, t0.y), bc2(mean.x), xy);
      const float iz = __fdividef(1.f, z);   // ~1 ulp: inside reading R28's position bound (K_POS eps S_z)
      const f32x2 xyz = mul2(xy, bc2(iz));                       // (x / z, y / z)
      const f32x2 uv = fma2(pk2(c0.x, c0.y), xyz, pk2(c0.z, c0.w));
      u = uv.x;
      v = uv.y;
      const f32x2 jj = mul2(pk2(c0.x, c0.y), bc2(iz));          // (jx, jy) = (fx, fy) / z
      // Conservative screen cull: Sigma2D_xx <= jx^2 (1 + limx^2) smax^2 + 0.3 (rows of M are
      // orthonormal, |t/z| <= lim after the clamp), so the exact R9 extents are inside
      // bx, by; a Gaussian whose bound box misses the image has an empty R9 rect as well.
      const f32x2 ke = mul2(bc2(kappa), fma2(mul2(mul2(jj, jj), pk2(c1.z, c1.w)), bc2(smax2), bc2(0.3f)));
      const f32x2 bxy = fma2(bc2(1.02f), mul2(ke, pk2(rsqrtf(ke.x), rsqrtf(ke.y))), bc2(1.f));   // sqrt_approx
      const float bx = bxy.x, by = bxy.y;
      const bool offscreen = (u + bx < 0.f) || (u - bx > fw) || (v + by < 0.f) || (v - by > fh);
      if (!offscreen || debug) {
        // EWA Jacobian with the 1.3 frustum clamp (reading R6), applied to M: rows of J M, as
        // (row 0, row 1) pairs m[c] = (jx (M0c - tx M2c), jy (M1c - ty M2c))
        const float txz = fminf(fmaxf(xyz.x, -c1.x), c1.x);
        const float tyz = fminf(fmaxf(xyz.y, -c1.y), c1.y);
        const f32x2 nt = pk2(-txz, -tyz);
        const f32x2 m[3] = {mul2(jj, fma2(nt, bc2(r2.x), pk2(t0.x, t0.y))),
                            mul2(jj, fma2(nt, bc2(r2.y), pk2(t0.z, t0.w))),
                            mul2(jj, fma2(nt, bc2(r2.z), pk2(t1.x, t1.y)))};
        // A = (J M) L (2x3) as column pairs (A0c, A1c); Sigma2D = A A^T + 0.3 I (reading R7)
        f32x2 A[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) A[c] = fma2(m[0], bc2(L[0][c]), fma2(m[1], bc2(L[1][c]), mul2(m[2], bc2(L[2][c]))));
        const f32x2 s0 = fma2(A[0], A[0], fma2(A[1], A[1], mul2(A[2], A[2])));   // (sxx0, syy0)
        const float sxx0 = s0.x, syy0 = s0.y;
        const float sxy = fmaf(A[0].x, A[0].y, fmaf(A[1].x, A[1].y, A[2].x * A[2].y));
        const f32x2 s2 = add2(s0, bc2(0.3f));
        const float sxx = s2.x, syy = s2.y;
        const float A0[3] = {A[0].x, A[1].x, A[2].x}, A1[3] = {A[0].y, A[1].y, A[2].y};
        // det(A A^T) by Cauchy-Binet (sum of squared 2x2 minors) + 0.3 tr + 0.09: no cancellation
        const float n01 = det2(A0[0], A0[1], A1[0], A1[1]);
        const float n02 = det2(A0[0], A0[2], A1[0], A1[2]);
        const float n12 = det2(A0[1], A0[2], A1[1], A1[2]);
        const float det = fmaf(n01, n01, fmaf(n02, n02, fmaf(n12, n12, fmaf(0.3f, sxx0 + syy0, 0.09f))));
        // whitening (Cholesky) factor of Sigma2D^-1:  Q = (p dx)^2 + (q dx + r dy)^2
        const float il11 = rsqrtf(sxx);
        const float r_ = rsqrtf(__fdividef(det, sxx));
        const float q_ = -sxy * il11 * il11 * r_;
        pw = wscale * il11;
        qw = wscale * q_;
        rw = wscale * r_;
        const bool rect_ok = r9_rect(u, v, sxx, syy, kappa, a.width, a.height, tx0, tx1, ty0, ty1);
        vis = keep && rect_ok;
        if (vis || debug) {
          // view direction in the body frame (reading R19)
          const float4 cb = __ldg(tb + 3);
          const float dx = mean.x - cb.x, dy = mean.y - cb.y, dz = mean.z - cb.z;
          const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
          rgb = sh_colour<D>(a.g_sh, a.sh_stride, in ? i : 0, dx * inv, dy * inv, dz * inv);
        }
        if (debug && in) {
          const size_t o = (size_t)f * a.n + id;
          float* d = a.dbg_rec + o * kDbgRecFloats;
          const float idet = 1.0f / det;
          d[0] = u; d[1] = v; d[2] = syy * idet; d[3] = -sxy * idet; d[4] = sxx * idet;
          d[5] = opac; d[6] = rgb.x; d[7] = rgb.y; d[8] = rgb.z; d[9] = z; d[10] = sxx; d[11] = syy;
          if (offscreen && rect_ok) d[11] = __int_as_float(0x7fc0dead);  // bound violated: flag loudly
          d[12] = pw; d[13] = qw; d[14] = rw; d[15] = log2o;   // what K4 composites with
        }
      }
    }
    if (debug && in) {
      a.dbg_zbits[(size_t)f * a.n + id] = __float_as_uint(z);
      a.dbg_valid[(size_t)f * a.n + id] = (uint8_t)keep;
    }
    if (a.rec == nullptr) continue;  // debug-only launch
    // record slot = internal index: no compaction atomics; one visibility word per warp
    const unsigned bal = __ballot_sync(0xffffffffu, vis);
    if ((threadIdx.x & 31) == 0 && i < a.n) {
      a.vis_bits[(size_t)fl * a.vis_words + (i >> 5)] = bal;
      if (bal) atomicAdd(a.vcount + fl, __popc(bal));  // V counter (no return value: RED)
    }
    const uint32_t rect = pack_rect(tx0, tx1, ty0, ty1);
    if (vis) {
      // half-extents of {arg >= log2(1/255)} = {Q' <= kappa'}, Q' = (p dx)^2 + (q dx + r dy)^2:
      // ex = sqrt(kappa') / p, ey = sqrt(kappa' (p^2 + q^2)) / (p r) (the R8 box in the whitened
      // metric), inflated by 1% + 0.01 px: K4 skips a pixel block only when it is outside it
      const float kap = fmaxf(log2o - kLog2AlphaMin, 0.f);
      const float sk = sqrt_approx(fmaxf(kap, 1e-30f));
      const float ipw = __fdividef(1.f, pw);
      const float ex = fmaf(sk * ipw, 1.01f, 0.01f);
      const float ey = fmaf(sk * sqrt_approx(fmaf(pw, pw, qw * qw)) * __fdividef(ipw, rw), 1.01f, 0.01f);
      float4* r = a.rec + ((size_t)fl * a.n + i) * kRecQuads;
      r[0] = make_float4(u, v, pw, qw);
      r[1] = make_float4(rw, log2o, ex, ey);
      r[2] = make_float4(rgb.x, rgb.y, rgb.z, z);
      a.emit[(size_t)fl * a.n + i] = make_uint2(__float_as_uint(z), rect);
      if (a.trim) {
        // K4b block masks: which half-tile borders of the rect the conservative R8 box (u +- ex,
        // v +- ey) does not reach — the 8x8 blocks there hold no pixel centre of alpha >= 1/255
        const float x_lo = (float)(tx0 * kTile) + 7.5f, x_hi = (float)(tx1 * kTile) + 8.5f;
        const float y_lo = (float)(ty0 * kTile) + 7.5f, y_hi = (float)(ty1 * kTile) + 8.5f;
        a.trim[(size_t)fl * a.n + i] = (uint8_t)((u - ex > x_lo ? 1u : 0u) | (u + ex < x_hi ? 2u : 0u) |
                                                 (v - ey > y_lo ? 4u : 0u) | (v + ey < y_hi ? 8u : 0u));
      }
    }
    if (bal) warp_tile_count(vis, rect, a.tiles_x, a.hist + (size_t)fl * a.hist_stride, tile_scratch[threadIdx.x >> 5]);
  }
}

void launch_k0(const K0Rig& rig, int n_frames, int n_cams, int n_bodies, int width, int height,
               float4* table, FrameCam* cams, cudaStream_t s) {
  const int total = n_frames * (n_bodies + 1);
  if (total == 0) return;
  k0_setup<<<(total + 127) / 128, 128, 0, s>>>(rig, n_frames, n_cams, n_bodies, width, height, table, cams);
}

void launch_k1(const K1Args& a, int sh_degree, cudaStream_t s) {
  if (a.n == 0) return;
  const unsigned gx = (unsigned)((a.n + 127) / 128);
  // >= ~8 waves of 8 CTAs x 148 SMs: each CTA loops over E / gy frames, so a CTA is short enough
  // that the last wave's tail stays small (C3: gy = 2, +0.7 % over one row; C4: 6)
  unsigned gy = (unsigned)std::max(1, std::min(a.n_frames, (int)((9472 + gx - 1) / gx)));
  if (const char* e = getenv("GSB_K1_GY")) gy = (unsigned)std::max(1, std::min(a.n_frames, atoi(e)));   // A/B
  const dim3 grid(gx, gy);
  const bool dbg = a.dbg_rec != nullptr;
#define K1_CASE(D)                                            \
  case D:                                                     \
    if (dbg) k1_project<D, true><<<grid, 128, 0, s>>>(a);     \
    else k1_project<D, false><<<grid, 128, 0, s>>>(a);        \
    break;
  switch (sh_degree) {
    K1_CASE(0)
    K1_CASE(1)
    K1_CASE(2)
    default:
      if (dbg) k1_project<3, true><<<grid, 128, 0, s>>>(a);
      else k1_project<3, false><<<grid, 128, 0, s>>>(a);
  }
#undef K1_CASE
}

}  // namespace gsb
