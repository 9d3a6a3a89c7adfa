/*
 * gsb_oracle.c — plain, slow, obviously-correct CPU ORACLE for the batched 3DGS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with
 * the CUDA path (paper_2604_25459_b200/csrc) and includes none of its headers.
 *
 * What it computes (DESIGN.md §2 "the definition"):
 *   for one frame (env e, camera c), per pixel, brute force over ALL Gaussians of the
 *   scene in (fp32 depth bits, id) order — there is no tile concept here.
 *
 *   step 1  pose:        PAPER.md App. B.2 Eqs., Alg. 1 l.12-14
 *                        mu_w = R(q_k) mu_i + t_k ; Sigma_w = R(q_k) Sigma_local R(q_k)^T
 *                        (reading R23: q_world = q_k (x) q_local => Sigma rotates with q_k)
 *   step 2  depth key:   exact fp32 chain, reading R11
 *   step 3  cull:        near < z <= far and o >= 1/255  (readings R4, R5)
 *   step 4  projection:  EWA splatting [3DGS-conv, cited by the paper at P:212],
 *                        readings R2, R3, R6, R7 — all in fp64
 *   step 5  colour:      real SH, degree <= 3, body-frame view direction (R18, R19)
 *   step 6  order:       (bits(z_f32), id) ascending (R10) — done by the caller (numpy lexsort)
 *   step 7  composite:   front-to-back alpha blending, alpha = min(0.99, o e^power),
 *                        skip alpha < 1/255, stop before blending when T(1-alpha) < 1e-4
 *                        (north_star; readings R12-R16), outputs RGB + T*bg, depth = sum w z,
 *                        alpha = 1 - T ("RGB images and depth maps")
 *   step 8  margin:      flip-effect budgets for the threshold mask (reading R28)
 *   step 9  optional box acceleration (R8): skip i when the pixel centre is outside
 *                        [u +- r_x] x [v +- r_y]; provably identical to brute force.
 *
 * Precision: fp64 everywhere except the depth key (fp32 chain, R11).  Build with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GSBO_NF 20
enum {
  F_U = 0, F_V, F_SXX, F_SXY, F_SYY, F_A, F_B, F_C, F_R, F_G, F_BL, F_O, F_KAPPA,
  F_Z32, F_Z64, F_XC, F_YC,
  F_EU, F_EV, /* reading R28: bounds on |u_gpu - u|, |v_gpu - v| (px), see R28_K_POS */
  F_EQ        /* reading R28: relative bound of K4's quadratic form, see R28_K_CONIC */
};

/* ---------------------------------------------------------------------------------
 * Reading R28: the threshold-margin mask uses a forward error bound of the GPU's
 * binary32 evaluation, not a flat margin.  EPS = binary32 unit roundoff 2^-24.
 * ------------------------------------------------------------------------------- */
#define R28_EPS (1.0 / 16777216.0)
/* position: the GPU computes x = M mu + m from fp32 M = W R(q_k), m = W t_k + t_f (each a
 * chain of fp32 ops), then u = f (x / z32) + c with z32 the R11 key.  First-order bound:
 *   |du| <= f/|z| (K_POS EPS S_x + |x/z| (|z32 - z| + K_POS EPS S_z)) + 2 EPS |u|
 * with S_r = sum_k |W_rk| (sum_c |R_kc mu_c| + |t_k|) + |t_fr| (the magnitudes summed by the
 * chain).  K_POS = 4: measured max |du| is 1.12 x the unit-count bound (scripts/alpha_error.py,
 * T1-T6 + C2-C4 on B200), so the bound holds with 3.5x to spare. */
#define R28_K_POS 4.0
/* K4's quadratic form from K1's whitening factor (Sigma2D in binary32, rsqrt/div approximations):
 * measured error <= 17.7 EPS |power| for Gaussians whose centre is inside the R6 frustum clamp
 * and <= 45.7 EPS |power| for clamped ones (off-screen giants) -> K_CONIC = 32 / 96 */
#define R28_K_CONIC 32.0
#define R28_K_CONIC_CLAMPED 96.0
/* K4's own binary32 evaluation: dx = u - px (one rounding of dx), then 5 fused ops; measured
 * <= 2.6 x EPS (|w_x| |u| + |w_y| |v| + |power| + |ln o|) -> bound K_EVAL EPS (|w.d| + |power|
 * + |ln o|) with w.d = 2 |power| the exact form of the dx/dy rounding, K_EVAL = 8 */
#define R28_K_EVAL 8.0

int gsbo_num_fields(void) { return GSBO_NF; }

/* ---------------------------------------------------------------------------------
 * Reading R11: the exact fp32 depth chain.  Every operation is a separately rounded
 * IEEE binary32 op (float arithmetic on x86-64 SSE, -ffp-contract=off) or fmaf()
 * (correctly rounded fused multiply-add from libm).
 * ------------------------------------------------------------------------------- */
static void r11_rot_f32(const float q[4], float R[3][3]) {
  float qw = q[0], qx = q[1], qy = q[2], qz = q[3];
  float xx = qx * qx, yy = qy * qy, zz = qz * qz;
  float xy = qx * qy, xz = qx * qz, yz = qy * qz;
  float wx = qw * qx, wy = qw * qy, wz = qw * qz;
  float s;
  s = yy + zz; R[0][0] = 1.0f - 2.0f * s;
  s = xy - wz; R[0][1] = 2.0f * s;
  s = xz + wy; R[0][2] = 2.0f * s;
  s = xy + wz; R[1][0] = 2.0f * s;
  s = xx + zz; R[1][1] = 1.0f - 2.0f * s;
  s = yz - wx; R[1][2] = 2.0f * s;
  s = xz - wy; R[2][0] = 2.0f * s;
  s = yz + wx; R[2][1] = 2.0f * s;
  s = xx + yy; R[2][2] = 1.0f - 2.0f * s;
}

/* depth row of the camera<-local transform: M2c, m2 (R11) */
static void r11_depth_row(const float* w2c /*3x4*/, const float* pose /*7 or NULL*/,
                          float M2[3], float* m2) {
  const float W20 = w2c[8], W21 = w2c[9], W22 = w2c[10], t2 = w2c[11];
  if (!pose) {
    M2[0] = W20; M2[1] = W21; M2[2] = W22; *m2 = t2;
    return;
  }
  float R[3][3];
  r11_rot_f32(pose + 3, R);
  for (int c = 0; c < 3; ++c) {
    float p = W22 * R[2][c];
    M2[c] = fmaf(W20, R[0][c], fmaf(W21, R[1][c], p));
  }
  *m2 = fmaf(W20, pose[0], fmaf(W21, pose[1], fmaf(W22, pose[2], t2)));
}

static float r11_depth(const float M2[3], float m2, const float mu[3]) {
  return fmaf(M2[0], mu[0], fmaf(M2[1], mu[1], fmaf(M2[2], mu[2], m2)));
}

/* Reading R29: world->camera of a camera mounted on a body, from the
 * body pose (tx,ty,tz,qw,qx,qy,qz) and the mount B = body->camera [R|t] (3x4 row-major),
 * composed in binary32 as W = [B_R R(q)^T | B_t - (B_R R(q)^T) t], each op separately rounded:
 *   W[r][c] = fma(B[r][0], R[c][0], fma(B[r][1], R[c][1], B[r][2]*R[c][2]))
 *   W[r][3] = fma(-W[r][0], tx, fma(-W[r][1], ty, fma(-W[r][2], tz, B[r][3])))
 * with R(q) from the R11 quaternion chain. */
void gsbo_compose_w2c(const float* pose, const float* B, float* W) {
  float R[3][3];
  r11_rot_f32(pose + 3, R);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) {
      float p = B[r * 4 + 2] * R[c][2];
      W[r * 4 + c] = fmaf(B[r * 4 + 0], R[c][0], fmaf(B[r * 4 + 1], R[c][1], p));
    }
    W[r * 4 + 3] = fmaf(-W[r * 4 + 0], pose[0], fmaf(-W[r * 4 + 1], pose[1], fmaf(-W[r * 4 + 2], pose[2], B[r * 4 + 3])));
  }
}

/* fp32 depth key of one Gaussian — exported so tests can pin the chain on its own */
float gsbo_depth_key(const float* w2c, const float* pose_or_null, const float* mu) {
  float M2[3], m2;
  r11_depth_row(w2c, pose_or_null, M2, &m2);
  return r11_depth(M2, m2, mu);
}

/* ---------------------------------------------------------------------------------
 * fp64 helpers
 * ------------------------------------------------------------------------------- */
/* rotation matrix of a quaternion (w,x,y,z) used AS GIVEN (reading R22: per-frame
   quaternions are assumed unit; template quaternions are normalised by the caller) */
static void rot_from_quat(const double q[4], double R[3][3]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
  R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
  R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
}

static void matmul3(const double A[3][3], const double B[3][3], double C[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += A[i][k] * B[k][j];
      C[i][j] = s;
    }
}

static void transpose3(const double A[3][3], double T[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[i][j] = A[j][i];
}

/* reading R18: 3DGS real SH basis constants and sign pattern */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* SH basis values Y_j(dir), j < (deg+1)^2, exactly as multiplied in R18 */
void gsbo_sh_basis(int deg, double x, double y, double z, double* Y) {
  Y[0] = SH_C0;
  if (deg < 1) return;
  Y[1] = -SH_C1 * y; Y[2] = SH_C1 * z; Y[3] = -SH_C1 * x;
  if (deg < 2) return;
  double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[4] = SH_C2[0] * xy;
  Y[5] = SH_C2[1] * yz;
  Y[6] = SH_C2[2] * (2 * zz - xx - yy);
  Y[7] = SH_C2[3] * xz;
  Y[8] = SH_C2[4] * (xx - yy);
  if (deg < 3) return;
  Y[9] = SH_C3[0] * y * (3 * xx - yy);
  Y[10] = SH_C3[1] * xy * z;
  Y[11] = SH_C3[2] * y * (4 * zz - xx - yy);
  Y[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
  Y[13] = SH_C3[4] * x * (4 * zz - xx - yy);
  Y[14] = SH_C3[5] * z * (xx - yy);
  Y[15] = SH_C3[6] * x * (xx - 3 * yy);
}

/* ---------------------------------------------------------------------------------
 * Steps 1-5 for every Gaussian of one frame.
 *   means/scales/quats/opac/sh/body_id: the scene template (fp32, as given to the ABI)
 *   pose: [n_bodies][7] (tx,ty,tz,qw,qx,qy,qz) world<-body of THIS env (reading R22)
 *   intr: fx,fy,cx,cy (px); w2c: 3x4 row-major [R|t], OpenCV axes (reading R2)
 *   out: [n][GSBO_NF] doubles; zbits: [n]; valid: [n] (cull result)
 * Returns 0, or -1 on a body index out of range (SPEC S:652 UnknownBody).
 * ------------------------------------------------------------------------------- */
int gsbo_project(const float* means, const float* scales, const float* quats, const float* opac,
                 const float* sh, int sh_degree_scene, int sh_degree, const int32_t* body_id,
                 int64_t n, const float* pose, int n_bodies, const float* intr, const float* w2c,
                 int width, int height, float near_plane, float far_plane, double* out,
                 uint32_t* zbits, uint8_t* valid) {
  const int ncoef_scene = (sh_degree_scene + 1) * (sh_degree_scene + 1);
  const double fx = intr[0], fy = intr[1], cx = intr[2], cy = intr[3];
  double Wc[3][3], tc[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) Wc[r][c] = w2c[r * 4 + c];
    tc[r] = w2c[r * 4 + 3];
  }
  /* camera centre in world: c_w = -W^T t */
  double cw[3];
  for (int c = 0; c < 3; ++c) cw[c] = -(Wc[0][c] * tc[0] + Wc[1][c] * tc[1] + Wc[2][c] * tc[2]);
  const double limx = 1.3 * (double)width / (2.0 * fx);   /* reading R6 */
  const double limy = 1.3 * (double)height / (2.0 * fy);

  for (int64_t i = 0; i < n; ++i) {
    double* o = out + i * GSBO_NF;
    memset(o, 0, sizeof(double) * GSBO_NF);
    const int k = body_id[i];
    if (k < -1 || k >= n_bodies) return -1;
    /* step 1: RLGK pose of body k */
    double Rk[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, tk[3] = {0, 0, 0};
    const float* pk = NULL;
    if (k >= 0) {
      pk = pose + (int64_t)k * 7;
      double qk[4] = {pk[3], pk[4], pk[5], pk[6]};
      rot_from_quat(qk, Rk);
      tk[0] = pk[0]; tk[1] = pk[1]; tk[2] = pk[2];
    }
    const double mu[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
    double muw[3];
    for (int r = 0; r < 3; ++r) muw[r] = Rk[r][0] * mu[0] + Rk[r][1] * mu[1] + Rk[r][2] * mu[2] + tk[r];
    /* Sigma_local = R(q_i) diag(s^2) R(q_i)^T with q_i normalised (reading R24) */
    double qi[4] = {quats[4 * i], quats[4 * i + 1], quats[4 * i + 2], quats[4 * i + 3]};
    double qn = sqrt(qi[0] * qi[0] + qi[1] * qi[1] + qi[2] * qi[2] + qi[3] * qi[3]);
    for (int c = 0; c < 4; ++c) qi[c] /= qn;
    double Ri[3][3], RiT[3][3], S2[3][3] = {{0}}, T1[3][3], Sl[3][3];
    rot_from_quat(qi, Ri);
    for (int c = 0; c < 3; ++c) S2[c][c] = (double)scales[3 * i + c] * (double)scales[3 * i + c];
    matmul3(Ri, S2, T1);
    transpose3(Ri, RiT);
    matmul3(T1, RiT, Sl);
    double RkT[3][3], Sw[3][3];
    matmul3(Rk, Sl, T1);
    transpose3(Rk, RkT);
    matmul3(T1, RkT, Sw);

    /* step 2: exact fp32 depth key (R11) */
    float M2[3], m2;
    r11_depth_row(w2c, pk, M2, &m2);
    const float z32 = r11_depth(M2, m2, means + 3 * i);
    uint32_t zb;
    memcpy(&zb, &z32, 4);
    zbits[i] = zb;
    o[F_Z32] = z32;
    o[F_O] = opac[i];

    /* step 3: cull (R4, R5) */
    const int keep = (z32 > near_plane) && (z32 <= far_plane) && ((double)opac[i] >= 1.0 / 255.0);
    valid[i] = (uint8_t)keep;

    /* step 4: EWA projection, fp64 (R2, R3, R6, R7) */
    double xc[3];
    for (int r = 0; r < 3; ++r) xc[r] = Wc[r][0] * muw[0] + Wc[r][1] * muw[1] + Wc[r][2] * muw[2] + tc[r];
    const double z = xc[2];
    o[F_Z64] = z; o[F_XC] = xc[0]; o[F_YC] = xc[1];
    o[F_U] = fx * xc[0] / z + cx;
    o[F_V] = fy * xc[1] / z + cy;
    { /* reading R28: bound on the GPU's binary32 u, v (see R28_K_POS) */
      double mag[3], S[3];
      for (int r = 0; r < 3; ++r)
        mag[r] = fabs(Rk[r][0] * mu[0]) + fabs(Rk[r][1] * mu[1]) + fabs(Rk[r][2] * mu[2]) + fabs(tk[r]);
      for (int r = 0; r < 3; ++r)
        S[r] = fabs(Wc[r][0]) * mag[0] + fabs(Wc[r][1]) * mag[1] + fabs(Wc[r][2]) * mag[2] + fabs(tc[r]);
      const double dz = fabs((double)z32 - z) + R28_K_POS * R28_EPS * S[2];
      o[F_EU] = fabs(fx / z) * (R28_K_POS * R28_EPS * S[0] + fabs(xc[0] / z) * dz) + 2.0 * R28_EPS * fabs(o[F_U]);
      o[F_EV] = fabs(fy / z) * (R28_K_POS * R28_EPS * S[1] + fabs(xc[1] / z) * dz) + 2.0 * R28_EPS * fabs(o[F_V]);
    }
    double txz = xc[0] / z, tyz = xc[1] / z;
    o[F_EQ] = R28_EPS * ((fabs(txz) > limx || fabs(tyz) > limy) ? R28_K_CONIC_CLAMPED : R28_K_CONIC);
    if (txz < -limx) txz = -limx;
    if (txz > limx) txz = limx;
    if (tyz < -limy) tyz = -limy;
    if (tyz > limy) tyz = limy;
    const double tx = z * txz, ty = z * tyz;
    const double J[2][3] = {{fx / z, 0.0, -fx * tx / (z * z)}, {0.0, fy / z, -fy * ty / (z * z)}};
    double WcT[3][3], Sc[3][3];
    matmul3(Wc, Sw, T1);
    transpose3(Wc, WcT);
    matmul3(T1, WcT, Sc);
    double S2d[2][2];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double s = 0;
        for (int p = 0; p < 3; ++p)
          for (int q = 0; q < 3; ++q) s += J[a][p] * Sc[p][q] * J[b][q];
        S2d[a][b] = s;
      }
    S2d[0][0] += 0.3;
    S2d[1][1] += 0.3;
    const double det = S2d[0][0] * S2d[1][1] - S2d[0][1] * S2d[1][0];
    o[F_SXX] = S2d[0][0]; o[F_SXY] = S2d[0][1]; o[F_SYY] = S2d[1][1];
    o[F_A] = S2d[1][1] / det;
    o[F_B] = -S2d[0][1] / det;
    o[F_C] = S2d[0][0] / det;
    o[F_KAPPA] = 2.0 * log(255.0 * (double)opac[i]);

    /* step 5: colour, body-frame view direction (R18, R19) */
    double cb[3];
    for (int c = 0; c < 3; ++c) {
      /* c_body = R(q_k)^T (c_world - t_k) */
      cb[c] = Rk[0][c] * (cw[0] - tk[0]) + Rk[1][c] * (cw[1] - tk[1]) + Rk[2][c] * (cw[2] - tk[2]);
    }
    double d[3] = {mu[0] - cb[0], mu[1] - cb[1], mu[2] - cb[2]};
    double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] /= dn; d[1] /= dn; d[2] /= dn;
    double Y[16];
    gsbo_sh_basis(sh_degree, d[0], d[1], d[2], Y);
    const int ncoef = (sh_degree + 1) * (sh_degree + 1);
    for (int ch = 0; ch < 3; ++ch) {
      double s = 0;
      for (int j = 0; j < ncoef; ++j) s += Y[j] * (double)sh[(i * ncoef_scene + j) * 3 + ch];
      s += 0.5;
      o[F_R + ch] = s > 0 ? s : 0.0;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------------
 * Step 7 (+8, +9): composite a list of pixels over the depth-ordered Gaussians.
 * ------------------------------------------------------------------------------- */
typedef struct {
  const double* proj;
  const uint32_t* order;
  int64_t n_order;
  const int32_t* px;
  const int32_t* py;
  int64_t p0, p1;
  double bg[3];
  int mode; /* 0 = pure brute force, 1 = box accelerated (R8) */
  double margin_scale, cmax, zmax; /* R28 bound multiplier (1 = the model; 0 = no mask) */
  double bg_sign;                   /* 1 if every background channel is >= 0, else 2 */
  double* out_rgb;
  double* out_depth;
  double* out_alpha;
  int64_t* out_term_id;
  int64_t* out_n_eval;
  double* out_budget_rgb;
  double* out_budget_depth;
  uint8_t* out_term_near;
  double* out_eT;           /* R28: relative error bound of the GPU's final T */
  /* pruning scores (§8(f) row 3, reading R30), all NULL unless requested; per-thread arrays
   * indexed by Gaussian id, merged after the join */
  double* w_sum;            /* sum of blend weights w = alpha T over the pixels */
  double* w_max;            /* max of w */
  const uint8_t* mask_in;   /* [npix] pixels in the R28 margin */
  uint8_t* touched;         /* Gaussians whose R8 box holds a masked pixel */
} comp_job;

/* Reading R28: bound on |power_gpu - power| for one (pixel, Gaussian) pair, in natural-log
 * units (= the relative error of alpha): position (w = Sigma2D^-1 d = -grad_u power), K1's
 * quadratic form, K4's binary32 evaluation.  dx = u - px_c, dy = v - py_c. */
static double r28_delta(const double* g, double dx, double dy, double power) {
  const double wx = g[F_A] * dx + g[F_B] * dy, wy = g[F_B] * dx + g[F_C] * dy;
  return fabs(wx) * g[F_EU] + fabs(wy) * g[F_EV] + g[F_EQ] * fabs(power) +
         R28_K_EVAL * R28_EPS * (fabs(wx * dx) + fabs(wy * dy) + fabs(power) - log(g[F_O]));
}

/* r28_delta of n pairs (Gaussian row gid[k] of proj, pixel (px[k], py[k])) — exported so the
 * GPU tests can check the measured alpha error of every near-threshold pair against it */
void gsbo_r28_delta(const double* proj, const int64_t* gid, const int32_t* px, const int32_t* py, int64_t n,
                    double* out) {
  for (int64_t k = 0; k < n; ++k) {
    const double* g = proj + gid[k] * GSBO_NF;
    const double dx = g[F_U] - ((double)px[k] + 0.5), dy = g[F_V] - ((double)py[k] + 0.5);
    const double power = -0.5 * (g[F_A] * dx * dx + g[F_C] * dy * dy) - g[F_B] * dx * dy;
    out[k] = r28_delta(g, dx, dy, power);
  }
}

static void composite_pixel(const comp_job* jb, int64_t p) {
  const double pxc = (double)jb->px[p] + 0.5, pyc = (double)jb->py[p] + 0.5; /* R3 */
  double T = 1.0, C[3] = {0, 0, 0}, D = 0.0;
  double brgb = 0.0, bdep = 0.0;
  double eT = 0.0; /* R28: relative bound of |T_gpu - T| / T before the current entry */
  int64_t term = -1, n_eval = 0;
  uint8_t term_near = 0;
  const double thr = 1.0 / 255.0;
  const double ks = jb->margin_scale;
  for (int64_t j = 0; j < jb->n_order; ++j) {
    const uint32_t i = jb->order[j];
    const double* g = jb->proj + (int64_t)i * GSBO_NF;
    if (jb->mode == 1) { /* R8: exact bounding box of {alpha >= 1/255} */
      const double rx = sqrt(g[F_KAPPA] * g[F_SXX]), ry = sqrt(g[F_KAPPA] * g[F_SYY]);
      if (pxc < g[F_U] - rx || pxc > g[F_U] + rx || pyc < g[F_V] - ry || pyc > g[F_V] + ry) continue;
    }
    n_eval++;
    const double dx = g[F_U] - pxc, dy = g[F_V] - pyc;
    const double power = -0.5 * (g[F_A] * dx * dx + g[F_C] * dy * dy) - g[F_B] * dx * dy; /* R12 */
    if (power > 0.0) continue;
    const double delta = ks * r28_delta(g, dx, dy, power);
    const double araw = g[F_O] * exp(power);
    /* R28: skip-threshold flip (blend vs skip this entry): this entry's contribution and the
     * (1 - alpha) scaling of everything behind it; later T values then carry the factor too */
    if (fabs(power - log(thr / g[F_O])) <= delta) {
      /* |blend - skip| = |a T c_i - a (everything behind, background included)|: a difference
       * of two non-negative terms (colours >= 0 by the SH clamp; a background >= 0), each at
       * most a T cmax; twice that when the background has a negative channel */
      const double am = thr * exp(delta);
      brgb += jb->bg_sign * T * am * jb->cmax;
      bdep += T * am * jb->zmax;
      eT += am / (1.0 - am);
    }
    const double alpha = araw < 0.99 ? araw : 0.99;
    if (alpha < thr) continue;
    const double tT = T * (1.0 - alpha); /* R13 */
    /* R28: relative error of the GPU's tT = T - alpha T: the error of alpha scaled by
     * alpha / (1 - alpha) (clamped alphas: 0.99f - 0.99 = 9.5e-9), ex2.approx (2 EPS), and the
     * two roundings of w = alpha T and T - w relative to T (1 - alpha) */
    const double ea = (araw > 0.99 * exp(delta)) ? ks * 1e-8 / (1.0 - alpha)
                                                 : alpha / (1.0 - alpha) * (delta + ks * 2.0 * R28_EPS);
    const double eTn = eT + ea + ks * 2.0 * R28_EPS / (1.0 - alpha);
    /* R28: termination flip (stop vs continue): everything from here on; n_eval (an integer
     * decided by this test) is then not compared either */
    if (fabs(tT - 1e-4) <= eTn * tT) {
      /* stop: C + T bg; continue: C + alpha T c_i + (entries behind: <= tT cmax) + T_end bg */
      double dc = 0.0;
      for (int c = 0; c < 3; ++c) dc = fmax(dc, fabs(g[F_R + c] - jb->bg[c]));
      brgb += alpha * T * dc + 2.0 * tT * (1.0 + eTn) * jb->cmax;
      bdep += alpha * T * g[F_Z32] + tT * (1.0 + eTn) * jb->zmax;
      term_near = 1;
    }
    if (tT < 1e-4) {
      term = (int64_t)i;
      break;
    }
    const double w = alpha * T; /* R14 */
    if (jb->w_sum) {
      jb->w_sum[i] += w;
      if (w > jb->w_max[i]) jb->w_max[i] = w;
    }
    C[0] += w * g[F_R];
    C[1] += w * g[F_G];
    C[2] += w * g[F_BL];
    D += w * g[F_Z32];
    T = tT;
    eT = eTn;
  }
  for (int c = 0; c < 3; ++c) jb->out_rgb[p * 3 + c] = C[c] + T * jb->bg[c];
  jb->out_depth[p] = D;          /* R16 */
  jb->out_alpha[p] = 1.0 - T;
  jb->out_term_id[p] = term;
  jb->out_n_eval[p] = n_eval;
  jb->out_budget_rgb[p] = brgb;
  jb->out_budget_depth[p] = bdep;
  jb->out_term_near[p] = term_near;
  if (jb->out_eT) jb->out_eT[p] = eT;
  if (jb->touched && jb->mask_in && jb->mask_in[p]) {
    /* a masked pixel may blend any Gaussian whose exact box holds it on either side of a flip */
    for (int64_t j = 0; j < jb->n_order; ++j) {
      const uint32_t i = jb->order[j];
      const double* g = jb->proj + (int64_t)i * GSBO_NF;
      const double rx = sqrt(g[F_KAPPA] * g[F_SXX]), ry = sqrt(g[F_KAPPA] * g[F_SYY]);
      if (pxc >= g[F_U] - rx && pxc <= g[F_U] + rx && pyc >= g[F_V] - ry && pyc <= g[F_V] + ry) jb->touched[i] = 1;
    }
  }
}

static void* composite_worker(void* arg) {
  const comp_job* jb = (const comp_job*)arg;
  for (int64_t p = jb->p0; p < jb->p1; ++p) composite_pixel(jb, p);
  return NULL;
}

int gsbo_composite(const double* proj, const uint32_t* order, int64_t n_order, const int32_t* px,
                   const int32_t* py, int64_t npix, const float* bg, int mode, double margin_scale,
                   double cmax, double zmax, double* out_rgb, double* out_depth,
                   double* out_alpha, int64_t* out_term_id, int64_t* out_n_eval,
                   double* out_budget_rgb, double* out_budget_depth, uint8_t* out_term_near,
                   double* out_eT, int nthreads, int64_t n_gauss, double* out_w_sum, double* out_w_max,
                   const uint8_t* mask_in, uint8_t* out_touched) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((int64_t)nthreads > npix) nthreads = npix > 0 ? (int)npix : 1;
  comp_job jobs[256];
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) {
    comp_job* jb = &jobs[t];
    jb->proj = proj; jb->order = order; jb->n_order = n_order;
    jb->px = px; jb->py = py;
    jb->p0 = npix * t / nthreads;
    jb->p1 = npix * (t + 1) / nthreads;
    for (int c = 0; c < 3; ++c) jb->bg[c] = bg[c];
    jb->mode = mode;
    jb->margin_scale = margin_scale; jb->cmax = cmax; jb->zmax = zmax;
    jb->bg_sign = (bg[0] >= 0.f && bg[1] >= 0.f && bg[2] >= 0.f) ? 1.0 : 2.0;
    jb->out_rgb = out_rgb; jb->out_depth = out_depth; jb->out_alpha = out_alpha;
    jb->out_term_id = out_term_id; jb->out_n_eval = out_n_eval;
    jb->out_budget_rgb = out_budget_rgb; jb->out_budget_depth = out_budget_depth;
    jb->out_term_near = out_term_near; jb->out_eT = out_eT;
    jb->w_sum = jb->w_max = NULL; jb->mask_in = mask_in; jb->touched = NULL;
    if (out_w_sum && out_w_max) {
      jb->w_sum = (double*)calloc((size_t)n_gauss + 1, sizeof(double));
      jb->w_max = (double*)calloc((size_t)n_gauss + 1, sizeof(double));
      if (!jb->w_sum || !jb->w_max) return 1;
    }
    if (out_touched && mask_in) {
      jb->touched = (uint8_t*)calloc((size_t)n_gauss + 1, 1);
      if (!jb->touched) return 1;
    }
  }
  if (nthreads == 1) {
    composite_worker(&jobs[0]);
  } else {
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, composite_worker, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  /* merge the per-thread score arrays: sums added, maxima maxed, flags or-ed */
  for (int t = 0; t < nthreads; ++t) {
    comp_job* jb = &jobs[t];
    for (int64_t i = 0; i < n_gauss && jb->w_sum; ++i) {
      out_w_sum[i] += jb->w_sum[i];
      if (jb->w_max[i] > out_w_max[i]) out_w_max[i] = jb->w_max[i];
    }
    for (int64_t i = 0; i < n_gauss && jb->touched; ++i) out_touched[i] |= jb->touched[i];
    free(jb->w_sum); free(jb->w_max); free(jb->touched);
  }
  return 0;
}

/* correctly rounded binary32 fma — exported to pin the numpy emulation */
float gsbo_fmaf(float a, float b, float c) { return fmaf(a, b, c); }

/* =================================================================================
 * Batched ray-cast LiDAR against the Gaussians — SURVEY §8(f) row 4 ("batched ray-depth
 * LiDAR", tab:lidar P:320-329; "Batch-LiDAR module utilizing ray-casting", P:315;
 * "omnidirectional or bounded ray-casting"; height scan = downward rays).
 * The paper gives no formula; reading R32 is what both sides compute:
 *
 *   sensor s of env e: world->sensor W = [R_s | t_s] (3x4 row-major, like a camera);
 *   rays: unit directions d_j (sensor frame) from the sensor origin, j < R.
 *   step 1  pose (as gsbo_project step 1): mu_w, Sigma_w by RLGK (R23)
 *   step 2  range key: x_r = fma(M_r0,mu_x, fma(M_r1,mu_y, fma(M_r2,mu_z, m_r))) for r = 0..2,
 *           M, m by the R11 chain applied to every row (static: M = W_R, m = t);
 *           rho = sqrt_rn(fma(x0,x0, fma(x1,x1, x2*x2)))  — binary32, each op rounded
 *   step 3  cull: near < rho <= far and o >= 1/255 (R4, R5 with rho for z)
 *   step 4  order: (bits(rho), id) ascending (R10 with rho for z) — done by the caller
 *   step 5  per ray, fp64: x = W mu_w + t, P = (W Sigma_w W^T)^-1,
 *           t* = d^T P x / d^T P d, t^ = max(t*, 0)   (peak of the Gaussian on the half-ray),
 *           D2 = (x - t^ d)^T P (x - t^ d),  alpha = min(0.99, o exp(-D2/2)),
 *           then R12-R14 with t^ for z and no colour: skip alpha < 1/255, stop before
 *           blending when T(1-alpha) < 1e-4, w = alpha T, range += w t^, T = T(1-alpha);
 *           outputs range = sum w t^ and alpha = 1 - T  (R16 with t^ for z).
 *   step 6  margin: flip budgets as R28 (alpha skip threshold and termination test).
 * ================================================================================= */
#define GSBO_LF 12
enum { L_X = 0, L_Y, L_Z, L_P00, L_P01, L_P02, L_P11, L_P12, L_P22, L_O, L_RHO32, L_RHO64 };

int gsbo_lidar_num_fields(void) { return GSBO_LF; }

/* the rows of sensor<-local (M, m) in binary32 (R11 chain on every row; R32 step 2) */
static void r32_rows(const float* w2s, const float* pose, float M[3][3], float m[3]) {
  if (!pose) {
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) M[r][c] = w2s[r * 4 + c];
      m[r] = w2s[r * 4 + 3];
    }
    return;
  }
  float R[3][3];
  r11_rot_f32(pose + 3, R);
  for (int r = 0; r < 3; ++r) {
    const float W0 = w2s[r * 4 + 0], W1 = w2s[r * 4 + 1], W2 = w2s[r * 4 + 2], tr = w2s[r * 4 + 3];
    for (int c = 0; c < 3; ++c) {
      float p = W2 * R[2][c];
      M[r][c] = fmaf(W0, R[0][c], fmaf(W1, R[1][c], p));
    }
    m[r] = fmaf(W0, pose[0], fmaf(W1, pose[1], fmaf(W2, pose[2], tr)));
  }
}

/* binary32 range key of one mean (R32 step 2) — exported so tests can pin the chain */
float gsbo_range_key(const float* w2s, const float* pose_or_null, const float* mu) {
  float M[3][3], m[3], x[3];
  r32_rows(w2s, pose_or_null, M, m);
  for (int r = 0; r < 3; ++r) x[r] = fmaf(M[r][0], mu[0], fmaf(M[r][1], mu[1], fmaf(M[r][2], mu[2], m[r])));
  float zz = x[2] * x[2];
  return sqrtf(fmaf(x[0], x[0], fmaf(x[1], x[1], zz)));
}

/* Steps 1-3 for every Gaussian of one (env, sensor): out [n][GSBO_LF], rhobits [n], valid [n].
 * Returns 0, or -1 on a body index out of range. */
int gsbo_lidar_project(const float* means, const float* scales, const float* quats, const float* opac,
                       const int32_t* body_id, int64_t n, const float* pose, int n_bodies, const float* w2s,
                       float near_plane, float far_plane, double* out, uint32_t* rhobits, uint8_t* valid) {
  double Wc[3][3], tc[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) Wc[r][c] = w2s[r * 4 + c];
    tc[r] = w2s[r * 4 + 3];
  }
  for (int64_t i = 0; i < n; ++i) {
    double* o = out + i * GSBO_LF;
    memset(o, 0, sizeof(double) * GSBO_LF);
    const int k = body_id[i];
    if (k < -1 || k >= n_bodies) return -1;
    double Rk[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, tk[3] = {0, 0, 0};
    const float* pk = NULL;
    if (k >= 0) {
      pk = pose + (int64_t)k * 7;
      double qk[4] = {pk[3], pk[4], pk[5], pk[6]};
      rot_from_quat(qk, Rk);
      tk[0] = pk[0]; tk[1] = pk[1]; tk[2] = pk[2];
    }
    const double mu[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
    double muw[3];
    for (int r = 0; r < 3; ++r) muw[r] = Rk[r][0] * mu[0] + Rk[r][1] * mu[1] + Rk[r][2] * mu[2] + tk[r];
    double qi[4] = {quats[4 * i], quats[4 * i + 1], quats[4 * i + 2], quats[4 * i + 3]};
    double qn = sqrt(qi[0] * qi[0] + qi[1] * qi[1] + qi[2] * qi[2] + qi[3] * qi[3]);
    for (int c = 0; c < 4; ++c) qi[c] /= qn;
    double Ri[3][3], RiT[3][3], S2[3][3] = {{0}}, T1[3][3], Sl[3][3], RkT[3][3], Sw[3][3], WT[3][3], Ss[3][3];
    rot_from_quat(qi, Ri);
    for (int c = 0; c < 3; ++c) S2[c][c] = (double)scales[3 * i + c] * (double)scales[3 * i + c];
    matmul3(Ri, S2, T1);
    transpose3(Ri, RiT);
    matmul3(T1, RiT, Sl);          /* Sigma_local (R23) */
    matmul3(Rk, Sl, T1);
    transpose3(Rk, RkT);
    matmul3(T1, RkT, Sw);          /* Sigma_world */
    matmul3(Wc, Sw, T1);
    transpose3(Wc, WT);
    matmul3(T1, WT, Ss);           /* Sigma_sensor = W Sigma_world W^T */
    /* P = Sigma_sensor^-1 by the adjugate */
    const double a = Ss[0][0], b = Ss[0][1], c = Ss[0][2], d = Ss[1][1], e = Ss[1][2], f = Ss[2][2];
    const double A00 = d * f - e * e, A01 = c * e - b * f, A02 = b * e - c * d;
    const double A11 = a * f - c * c, A12 = b * c - a * e, A22 = a * d - b * b;
    const double det = a * A00 + b * A01 + c * A02;
    o[L_P00] = A00 / det; o[L_P01] = A01 / det; o[L_P02] = A02 / det;
    o[L_P11] = A11 / det; o[L_P12] = A12 / det; o[L_P22] = A22 / det;
    for (int r = 0; r < 3; ++r) o[L_X + r] = Wc[r][0] * muw[0] + Wc[r][1] * muw[1] + Wc[r][2] * muw[2] + tc[r];
    o[L_O] = opac[i];
    const float rho = gsbo_range_key(w2s, pk, means + 3 * i);
    uint32_t rb;
    memcpy(&rb, &rho, 4);
    rhobits[i] = rb;
    o[L_RHO32] = rho;
    o[L_RHO64] = sqrt(o[L_X] * o[L_X] + o[L_Y] * o[L_Y] + o[L_Z] * o[L_Z]);
    valid[i] = (uint8_t)((rho > near_plane) && (rho <= far_plane) && ((double)opac[i] >= 1.0 / 255.0));
  }
  return 0;
}

/* the peak of Gaussian g on the half-ray t >= 0 along d: returns D2, writes t^ (R32 step 5) */
static double r32_peak(const double* g, const double dv[3], double* that) {
  const double P[3][3] = {{g[L_P00], g[L_P01], g[L_P02]}, {g[L_P01], g[L_P11], g[L_P12]},
                          {g[L_P02], g[L_P12], g[L_P22]}};
  double Pd[3], Px[3];
  for (int r = 0; r < 3; ++r) {
    Pd[r] = P[r][0] * dv[0] + P[r][1] * dv[1] + P[r][2] * dv[2];
    Px[r] = P[r][0] * g[L_X] + P[r][1] * g[L_Y] + P[r][2] * g[L_Z];
  }
  const double dPd = dv[0] * Pd[0] + dv[1] * Pd[1] + dv[2] * Pd[2];
  const double dPx = dv[0] * Px[0] + dv[1] * Px[1] + dv[2] * Px[2];
  double t = dPx / dPd;
  if (t < 0.0) t = 0.0;
  const double e[3] = {g[L_X] - t * dv[0], g[L_Y] - t * dv[1], g[L_Z] - t * dv[2]};
  double D2 = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) D2 += e[r] * P[r][c] * e[c];
  *that = t;
  return D2;
}

double gsbo_lidar_peak(const double* g, const double* dv, double* that) { return r32_peak(g, dv, that); }

typedef struct {
  const double* proj;
  const uint32_t* order;
  int64_t n_order;
  const float* dirs;
  int64_t r0, r1;
  double delta_alpha, delta_T, tmax;
  double* out_range;
  double* out_alpha;
  double* out_budget_range;
  double* out_budget_alpha;
  int64_t* out_n_blend;
} lidar_job;

static void cast_ray(const lidar_job* jb, int64_t j) {
  const double dv[3] = {jb->dirs[3 * j], jb->dirs[3 * j + 1], jb->dirs[3 * j + 2]};
  double T = 1.0, Rg = 0.0, br = 0.0, ba = 0.0;
  int64_t nb = 0;
  const double thr = 1.0 / 255.0;
  for (int64_t q = 0; q < jb->n_order; ++q) {
    const double* g = jb->proj + (int64_t)jb->order[q] * GSBO_LF;
    double th;
    const double D2 = r32_peak(g, dv, &th);
    const double araw = g[L_O] * exp(-0.5 * D2);
    if (fabs(araw - thr) <= jb->delta_alpha * thr) { /* R28: skip-threshold flip */
      br += 2.0 * T * thr * (1.0 + jb->delta_alpha) * jb->tmax;
      ba += 2.0 * T * thr * (1.0 + jb->delta_alpha);
    }
    const double alpha = araw < 0.99 ? araw : 0.99;
    if (alpha < thr) continue;
    const double tT = T * (1.0 - alpha);
    if (fabs(tT - 1e-4) <= jb->delta_T * 1e-4) { /* R28: termination flip */
      br += T * jb->tmax;
      ba += T;
    }
    if (tT < 1e-4) break;
    const double w = alpha * T;
    Rg += w * th;
    T = tT;
    nb++;
  }
  jb->out_range[j] = Rg;
  jb->out_alpha[j] = 1.0 - T;
  jb->out_budget_range[j] = br;
  jb->out_budget_alpha[j] = ba;
  jb->out_n_blend[j] = nb;
}

static void* lidar_worker(void* arg) {
  const lidar_job* jb = (const lidar_job*)arg;
  for (int64_t j = jb->r0; j < jb->r1; ++j) cast_ray(jb, j);
  return NULL;
}

/* Step 5 (+6) for the listed rays over the range-ordered Gaussians (pure brute force). */
int gsbo_lidar_cast(const double* proj, const uint32_t* order, int64_t n_order, const float* dirs, int64_t n_rays,
                    double delta_alpha, double delta_T, double tmax, double* out_range, double* out_alpha,
                    double* out_budget_range, double* out_budget_alpha, int64_t* out_n_blend, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if ((int64_t)nthreads > n_rays) nthreads = n_rays > 0 ? (int)n_rays : 1;
  lidar_job jobs[256];
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) {
    lidar_job* jb = &jobs[t];
    jb->proj = proj; jb->order = order; jb->n_order = n_order; jb->dirs = dirs;
    jb->r0 = n_rays * t / nthreads;
    jb->r1 = n_rays * (t + 1) / nthreads;
    jb->delta_alpha = delta_alpha; jb->delta_T = delta_T; jb->tmax = tmax;
    jb->out_range = out_range; jb->out_alpha = out_alpha;
    jb->out_budget_range = out_budget_range; jb->out_budget_alpha = out_budget_alpha;
    jb->out_n_blend = out_n_blend;
  }
  if (nthreads == 1) {
    lidar_worker(&jobs[0]);
  } else {
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, lidar_worker, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  return 0;
}
