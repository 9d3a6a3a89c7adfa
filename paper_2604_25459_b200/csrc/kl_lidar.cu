// kl_lidar.cu — batched ray-cast LiDAR against the Gaussians (§8(f) row 4; reading R32):
// "Batch-LiDAR module utilizing ray-casting", rotating / solid-state / non-repetitive
// scans (tab:lidar P:320-329), omnidirectional or bounded LiDAR and the Height Scan.
//
// The camera pipeline's structure, with the image plane replaced by an azimuth x elevation
// grid of cells around the sensor:
//   K0   per-(frame, body) transforms (shared with the cameras; frame = (env, sensor))
//   KL1  per (frame, Gaussian): sensor-frame mean by the R32 binary32 chain, range key rho,
//        cull, whitening record, and the cells of the Gaussian's angular cap (one rect, or two
//        when it crosses the azimuth seam of the grid window) + cell histogram
//   K2   scan + key emission (the camera kernels; the seam rect is a second "virtual"
//        Gaussian at index Np + i carrying the same id, so keys stay (bits(rho), id))
//   K4a  per-(frame, cell) sort into record slots (the camera kernel: counting sort <= 1024
//        keys, radix beyond)
//   KL4  one warp per (frame, cell, <= 32 rays of the cell): records staged through shared
//        memory 32 at a time, a 4-op cone test per (ray, record) selects the pairs that get
//        the exact evaluation, each lane composites its ray front to back, warp-vote exit.
// The cell lists are conservative supersets (bounding ball of the alpha >= 1/255 ellipsoid,
// widened by 1e-3 rad): an extra candidate evaluates alpha < 1/255 and is skipped exactly as
// the brute-force oracle skips it, so the binning never changes an output.
#include <algorithm>

#include "gsb_common.cuh"
#include "gsb_kernels.cuh"
#include "k4_common.cuh"

namespace gsb {

constexpr float kPi = 3.14159265358979323846f;
constexpr float kTwoPi = 6.28318530717958647692f;
constexpr float kAngMargin = 1e-3f;   // rad: covers fp32 error of the angular bounds

__global__ void __launch_bounds__(128) kl1_project(LidarL1Args a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = i < a.n;
  float4 mean = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 l0 = mean, l1 = mean, l2 = mean;
  int2 ids = make_int2(0, -1);
  if (in) {
    mean = __ldg(a.g_mean + i);
    l0 = __ldg(a.g_L0 + i);
    l1 = __ldg(a.g_L1 + i);
    l2 = __ldg(a.g_L2 + i);
    ids = __ldg(a.g_ids + i);
  }
  const int body = ids.y;
  const float L[3][3] = {{l0.x, l0.y, l0.z}, {l0.w, l1.x, l1.y}, {l1.z, l1.w, l2.x}};
  const float opac = l2.y, kappa = l2.z, log2o = l2.w;
  const bool o_ok = in && (opac >= 1.0f / 255.0f);   // R5
  // radius of a ball holding the alpha >= 1/255 ellipsoid {D2 <= kappa}: sqrt(kappa) s_max
  const float rball = sqrtf(fmaxf(kappa, 0.f) * mean.w) * 1.01f + 1e-6f;
  const float wscale = 0.84932180028801904f;  // sqrt(log2(e) / 2): D2/2 in log2 units
  const bool warp_live = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) < a.n;
  const int lane = threadIdx.x & 31;

  const int fpr = (a.n_frames + gridDim.y - 1) / gridDim.y;
  const int fl_lo = blockIdx.y * fpr, fl_hi = min(a.n_frames, fl_lo + fpr);
  for (int fl = fl_lo; fl < fl_hi; ++fl) {
    const int f = a.f0 + fl;
    const float4* tb = a.table + ((size_t)f * a.nb1 + (body + 1)) * 4;
    const float4 t0 = __ldg(tb + 0), t1 = __ldg(tb + 1), r2 = __ldg(tb + 2);   // rows 0, 1 interleaved
    const float4 r0 = make_float4(t0.x, t0.z, t1.x, t1.z), r1 = make_float4(t0.y, t0.w, t1.y, t1.w);
    // R32 step 2: binary32 chain, every op rounded
    const float x0 = __fmaf_rn(r0.x, mean.x, __fmaf_rn(r0.y, mean.y, __fmaf_rn(r0.z, mean.z, r0.w)));
    const float x1 = __fmaf_rn(r1.x, mean.x, __fmaf_rn(r1.y, mean.y, __fmaf_rn(r1.z, mean.z, r1.w)));
    const float x2 = __fmaf_rn(r2.x, mean.x, __fmaf_rn(r2.y, mean.y, __fmaf_rn(r2.z, mean.z, r2.w)));
    const float rho = __fsqrt_rn(__fmaf_rn(x0, x0, __fmaf_rn(x1, x1, __fmul_rn(x2, x2))));
    const bool keep = o_ok && (rho > a.near_plane) && (rho <= a.far_plane);   // R32 step 3
    bool va = false, vb = false;
    int ax0 = 0, ax1 = -1, bx1 = -1, ey0 = 0, ey1 = -1;
    if (keep) {
      bool all_az = false;
      if (rho <= rball) {   // sensor inside the ball: every direction
        all_az = true;
        ey0 = 0;
        ey1 = a.n_el - 1;
      } else {
        const float th = asinf(fminf(rball / rho, 1.f)) + kAngMargin;
        const float elc = atan2f(x2, sqrtf(x0 * x0 + x1 * x1));
        const float elo = elc - th, ehi = elc + th;
        const float e_lo = (elo - a.el0) * a.el_inv, e_hi = (ehi - a.el0) * a.el_inv;
        if (e_hi >= 0.f && e_lo < (float)a.n_el) {
          ey0 = max(0, (int)floorf(e_lo));
          ey1 = min(a.n_el - 1, (int)floorf(e_hi));
          if (ehi >= 0.5f * kPi - kAngMargin || elo <= -0.5f * kPi + kAngMargin) {
            all_az = true;
          } else {
            const float ratio = sinf(th) / cosf(elc);
            if (ratio >= 1.f) {
              all_az = true;
            } else {
              const float daz = asinf(ratio) + kAngMargin;
              const float azc = atan2f(x1, x0);
              float rel = azc - daz - a.az0;
              rel -= kTwoPi * floorf(rel * (1.f / kTwoPi));   // [0, 2 pi)
              rel = fminf(fmaxf(rel, 0.f), kTwoPi);
              const float hi = rel + 2.f * daz;
              if (2.f * daz >= kTwoPi) {
                all_az = true;
              } else {
                if (rel < a.az_span) {
                  va = true;
                  ax0 = min(a.n_az - 1, (int)floorf(rel * a.az_inv));
                  ax1 = min(a.n_az - 1, (int)floorf(fminf(hi, a.az_span) * a.az_inv));
                }
                if (hi > kTwoPi) {   // crosses the window origin: the seam part [0, hi - 2 pi]
                  const int c1 = min(a.n_az - 1, (int)floorf(fminf(hi - kTwoPi, a.az_span) * a.az_inv));
                  if (!va) {
                    va = true;
                    ax0 = 0;
                    ax1 = c1;
                  } else if (c1 >= ax0 - 1) {
                    ax0 = 0;
                    ax1 = a.n_az - 1;   // the two parts meet: the whole row
                  } else {
                    vb = true;
                    bx1 = c1;
                  }
                }
              }
            }
          }
          if (all_az) {
            va = true;
            vb = false;
            ax0 = 0;
            ax1 = a.n_az - 1;
          }
        }
      }
      if (all_az && !va) {
        va = true;
        ax0 = 0;
        ax1 = a.n_az - 1;
      }
    }
    // records: whitening A = G^-1 = diag(1/s^2) G^T with G = M L (Sigma_s = G G^T), scaled
    // so that |A (x - t d)|^2 = D2/2 in log2 units
    if (va || vb) {
      const float M[3][3] = {{r0.x, r0.y, r0.z}, {r1.x, r1.y, r1.z}, {r2.x, r2.y, r2.z}};
      float A[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float g[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) g[r] = M[r][0] * L[0][c] + M[r][1] * L[1][c] + M[r][2] * L[2][c];
        const float s = wscale / (g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
#pragma unroll
        for (int r = 0; r < 3; ++r) A[c][r] = g[r] * s;
      }
      const float m0 = A[0][0] * x0 + A[0][1] * x1 + A[0][2] * x2;
      const float m1 = A[1][0] * x0 + A[1][1] * x1 + A[1][2] * x2;
      const float m2 = A[2][0] * x0 + A[2][1] * x1 + A[2][2] * x2;
      // cull quad: a ray whose peak lies in the ball has d.x >= sqrt(|x|^2 - rball^2); c is
      // lowered by 1e-6 |x| (>> the fp32 error of d.x) and is -inf when the sensor is inside
      const float xx = fmaf(x0, x0, fmaf(x1, x1, x2 * x2));
      const float rr = rball * rball;
      const float cth = xx > rr ? sqrtf(xx - rr) - 1e-6f * sqrtf(xx) : -1e30f;
      float4* o = a.rec + ((size_t)fl * a.n + i) * kLidarRecQuads;
      o[0] = make_float4(A[0][0], A[0][1], A[0][2], m0);
      o[1] = make_float4(A[1][0], A[1][1], A[1][2], m1);
      o[2] = make_float4(A[2][0], A[2][1], A[2][2], m2);
      o[3] = make_float4(x0, x1, x2, cth);
      o[4] = make_float4(log2o, rho, 0.f, 0.f);
    }
    const uint32_t zb = __float_as_uint(rho);
    const uint32_t ra = pack_rect(ax0, ax1, ey0, ey1);
    const uint32_t rbx = pack_rect(0, bx1, ey0, ey1);
    const unsigned bal_a = __ballot_sync(0xffffffffu, va);
    const unsigned bal_b = __ballot_sync(0xffffffffu, vb);
    if (warp_live && lane == 0) {
      a.vis_bits[(size_t)fl * a.vis_words + (i >> 5)] = bal_a;
      a.vis_bits[(size_t)fl * a.vis_words + ((a.np + i) >> 5)] = bal_b;
      const int c = __popc(bal_a | bal_b);
      if (c) atomicAdd(a.vcount + fl, c);
    }
    if (va) a.emit[(size_t)fl * 2 * a.np + i] = make_uint2(zb, ra);
    if (vb) a.emit[(size_t)fl * 2 * a.np + a.np + i] = make_uint2(zb, rbx);
    int* hist = a.hist + (size_t)fl * a.hist_stride;
    warp_tile_count(va, ra, a.n_az, hist);
    warp_tile_count(vb, rbx, a.n_az, hist);
  }
}

void launch_kl1(const LidarL1Args& a, cudaStream_t s) {
  if (a.n == 0 || a.n_frames == 0) return;
  const unsigned gx = (unsigned)((a.n + 127) / 128);
  const unsigned gy = (unsigned)std::max(1, std::min(a.n_frames, (int)((4736 + gx - 1) / gx)));
  kl1_project<<<dim3(gx, gy), 128, 0, s>>>(a);
}

// ------------------------------------------------------------------------------ KL4
// One warp per (frame, cell, <= 32 rays).  Per round, 32 records of the cell's sorted list are
// staged in shared memory (one per lane, quad-major so the broadcast reads are conflict-free);
// every lane tests its ray against the 32 cull quads (d.x >= c: 4 ops per pair) into its own
// bit mask, then walks its accepted records in list order with the exact R32 evaluation
// (~25 ops) — lanes diverge, but every executed evaluation is a useful one.  The lists are (bits(rho), id) ordered (K4a), so the lanes
// composite front to back; the warp leaves when every lane has terminated.
constexpr int kL4Warps = 4;

__global__ void __launch_bounds__(32 * kL4Warps) kl4_cast(LidarL4Args a) {
  __shared__ float4 st[kL4Warps][kLidarRecQuads][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kL4Warps + warp;
  if (item >= a.n_items) return;   // warp-uniform
  const unsigned FULL = 0xffffffffu;
  const int fl = blockIdx.y;
  const int4 it = __ldg(a.items + item);
  const bool has = lane < it.z;
  float4 ray = make_float4(0.f, 0.f, 0.f, 0.f);
  if (has) ray = __ldg(a.rays + it.y + lane);
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  const uint64_t start = a.frame_base[fl] + off[it.x];
  const int n = (int)(off[it.x + 1] - off[it.x]);
  float T = 1.f, R = 0.f;
  bool done = !has;
  const float4* rec = a.rec + (size_t)fl * a.n * kLidarRecQuads;
  // the next round's records are loaded into registers while this round is composited
  float4 pf[kLidarRecQuads];
  auto prefetch = [&](int base) {
    const int j = base + lane;
    if (j < n) {
      uint32_t slot = __ldg(a.sorted + start + j);
      if (slot >= (uint32_t)a.np) slot -= (uint32_t)a.np;   // seam copy -> its Gaussian
      const float4* r = rec + (size_t)slot * kLidarRecQuads;
#pragma unroll
      for (int q = 0; q < kLidarRecQuads; ++q) pf[q] = __ldg(r + q);
    } else {
      pf[3] = make_float4(0.f, 0.f, 0.f, 3e38f);   // never accepted
    }
  };
  if (n > 0) prefetch(0);
  for (int base = 0; base < n; base += 32) {
    if (__all_sync(FULL, done)) break;
#pragma unroll
    for (int q = 0; q < kLidarRecQuads; ++q) st[warp][q][lane] = pf[q];
    __syncwarp();
    if (base + 32 < n) prefetch(base + 32);
    unsigned mine = 0;   // records of this round whose cone test this lane's ray passes
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float4 xc = st[warp][3][k];
      const bool acc = fmaf(ray.x, xc.x, fmaf(ray.y, xc.y, ray.z * xc.z)) >= xc.w;
      mine |= acc ? (1u << k) : 0u;
    }
    if (done) mine = 0u;
    // each lane walks its own accepted records in list order (front to back for its ray)
    while (mine) {
      const int k = __ffs(mine) - 1;
      mine &= mine - 1;
      const float4 q0 = st[warp][0][k], q1 = st[warp][1][k], q2 = st[warp][2][k];
      const float log2o = st[warp][4][k].x;
      const float w0 = fmaf(q0.x, ray.x, fmaf(q0.y, ray.y, q0.z * ray.z));
      const float w1 = fmaf(q1.x, ray.x, fmaf(q1.y, ray.y, q1.z * ray.z));
      const float w2 = fmaf(q2.x, ray.x, fmaf(q2.y, ray.y, q2.z * ray.z));
      const float ww = fmaf(w0, w0, fmaf(w1, w1, w2 * w2));
      const float wm = fmaf(w0, q0.w, fmaf(w1, q1.w, w2 * q2.w));
      const float th = fmaxf(__fdividef(wm, ww), 0.f);     // t^ = max(t*, 0)
      const float e0 = fmaf(-th, w0, q0.w), e1 = fmaf(-th, w1, q1.w), e2 = fmaf(-th, w2, q2.w);
      const float arg = log2o - fmaf(e0, e0, fmaf(e1, e1, e2 * e2));
      if (arg >= kLog2AlphaMin) {   // alpha >= 1/255 (R12)
        const float alpha = fminf(kAlphaMax, ex2_approx(arg));
        const float tT = T * (1.f - alpha);
        if (tT < kTermT) {
          done = true;                        // stop before blending (R13)
          mine = 0u;
        } else {
          R = fmaf(alpha * T, th, R);         // w t^ (R14 with t^ for z)
          T = tT;
        }
      }
    }
    __syncwarp();
  }
  if (has) {
    const int ridx = __float_as_int(ray.w);
    const size_t o = (size_t)(a.f0 + fl) * a.n_rays + ridx;
    a.out_range[o] = R;
    if (a.out_alpha) a.out_alpha[o] = 1.f - T;
  }
}

void launch_kl4(const LidarL4Args& a, cudaStream_t s) {
  if (a.n_items == 0 || a.n_frames == 0) return;
  kl4_cast<<<dim3((unsigned)((a.n_items + kL4Warps - 1) / kL4Warps), (unsigned)a.n_frames), 32 * kL4Warps, 0, s>>>(a);
}

}  // namespace gsb
