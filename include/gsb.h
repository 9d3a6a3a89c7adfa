/*
 * gsb.h — C ABI of libgsb, a B200-native (sm_100a) batched 3D Gaussian Splatting renderer:
 * the data-parallel hot path of GS-Playground (arXiv 2604.25459).
 *
 * The operation (PAPER.md, cited by line "P:n"; readings R1-R28 in DESIGN.md §2):
 *   * one Gaussian TEMPLATE is uploaded once (App. B.2; Alg. 1 l.2-7);
 *   * every step, batch body states S_t in R^{B x N_bodies x 7} arrive (Alg. 1 l.9,
 *     P:726); each Gaussian i attached to body k moves rigidly (RLGK, Eqs.):
 *         p_world = R(q_k) p_local + t_k ,   q_world = q_k (x) q_local;
 *   * each env's cameras (per-env intrinsics/extrinsics, domain-randomised) render
 *     RGB images and depth maps with the 3DGS rasteriser the paper builds on
 *     ("BatchSplat" P:139): EWA projection + SH colour, 16x16 tile binning,
 *     a (tile, depth, id) sort, and front-to-back alpha compositing with alpha clamped at
 *     0.99, alpha < 1/255 skipped, termination when T(1-alpha) < 1e-4 (north_star).
 *
 * Conventions (DESIGN.md readings):
 *   R2  pinhole, (fx, fy, cx, cy) in pixels; world_to_cam = [R | t] row-major 3x4, OpenCV
 *       axes (x right, y down, z forward); depth = camera z of the mean.
 *   R3  pixel (px, py) has centre (px + 0.5, py + 0.5).
 *   R17 outputs fp32, planar: rgb [B][C][3][H][W]; depth/alpha/n_eval [B][C][H][W].
 *   R21 body indices are 0-based, -1 = static world Gaussian.
 *   R22 pose vector = (tx, ty, tz, qw, qx, qy, qz), world <- body, scalar-first Hamilton
 *       quaternion used as given (unit assumed).
 *   R24 template parameters are ACTIVATED values: linear scales > 0, opacity in (0, 1];
 *       template quaternions are normalised by gsb_create_scene.
 *
 * Errors: every entry point returns gsb_status (0 = OK).  Arguments are validated on the
 * host before anything is enqueued; on failure nothing is enqueued and gsb_last_error()
 * returns a thread-local message.  CUDA launch errors return GSB_ERR_CUDA; device faults
 * surface at the caller's next synchronisation.  Non-finite poses/cameras are not errors:
 * the affected Gaussians fail the cull tests deterministically.
 *
 * Threading: one scene is used by one host thread and one stream at a time.
 * Determinism: for fixed inputs the outputs are bit-identical across runs, chunk sizes,
 * batch sizes and env slicing (every env-camera frame is computed independently).
 */
#ifndef GSB_H_
#define GSB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gsb_scene_t* gsb_scene; /* opaque, bound to one CUDA device */
typedef struct CUstream_st* gsb_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  GSB_OK = 0,
  GSB_ERR_INVALID_ARGUMENT = 1,
  GSB_ERR_SHAPE_MISMATCH = 2, /* cf. SPEC S:661 ShapeMismatch */
  GSB_ERR_UNKNOWN_BODY = 3,   /* cf. SPEC S:652 UnknownBody: body_id outside [-1, n_bodies) */
  GSB_ERR_OUT_OF_MEMORY = 4,
  GSB_ERR_CAPACITY = 5,       /* N >= 2^32, render larger than the reservation, or one
                                 frame's tile keys exceed the key workspace */
  GSB_ERR_CUDA = 6,
  GSB_ERR_DEVICE = 7          /* device is not sm_100 (B200) */
} gsb_status;

/* render flags */
#define GSB_FLAG_STATS 1u   /* count V (visible pairs), K (tile keys), P (pixel-Gaussian
                               evaluations) for gsb_get_stats */
#define GSB_FLAG_TIMING 2u  /* record CUDA events around every kernel class on the render
                               stream for gsb_get_timings */
#define GSB_FLAG_SCORES 4u  /* also accumulate the pruning scores of reading R30 into the
                               scene (gsb_get_scores); not with gsb_render_static */
#define GSB_FLAG_STATIC_PER_ENV 8u /* gsb_render_static only: one camera per env, env e uses
                               pre-binned camera e (per-env domain-randomised cameras that stay
                               fixed over an episode); needs n_envs <= the pre-binned count */
#define GSB_FLAG_FIXED_PLAN 16u /* gsb_render / gsb_render_rig / gsb_render_obs: a launch sequence
                                  that depends only on the call's shapes — no host synchronisation and
                                  no data-dependent launch choice (split K4a + K4b compositing for
                                  every chunk, one pass per chunk) — so the whole render can be
                                  captured in a CUDA graph on the caller's stream.  A chunk whose tile
                                  keys exceed the reserved key capacity sets the scene's overflow flag
                                  (gsb_get_overflow) and its frames are left unwritten.  Not with
                                  GSB_FLAG_STATS / GSB_FLAG_TIMING, host-buffer or static renders. */

/* reserve flags */
#define GSB_RESERVE_HOST_IO 1u /* also reserve device staging for gsb_render_host */

typedef struct {
  int32_t width, height;   /* image size in pixels, 1..4096 each */
  float near_plane;        /* keep near < z <= far (reading R4); default 0.01 */
  float far_plane;         /* default 1000 */
  float background[3];     /* RGB added with weight T (R15); contributes 0 to depth */
  int32_t sh_degree;       /* SH degree used, 0..scene degree; -1 = the scene's degree */
  uint32_t flags;          /* GSB_FLAG_* */
} gsb_render_params;

/* Create a scene template on CUDA device `device` (all pointers HOST, read during the call):
 *   means     [N,3] metres — body-local if body_id >= 0, world if body_id == -1
 *   scales    [N,3] linear sigma > 0 (metres)
 *   quats     [N,4] (w,x,y,z), any non-zero norm (normalised here)
 *   opacities [N]   in (0,1]; Gaussians with o < 1/255 are never visible (reading R5)
 *   sh        [N,(D+1)^2,3] coefficient-major (coefficient j, channel c at [(i*(D+1)^2+j)*3+c])
 *   sh_degree D in 0..3
 *   body_id   [N] int32 in [-1, n_bodies)
 * N may be 0 (renders the background).  Ownership: the scene owns device copies.
 * Errors: INVALID_ARGUMENT (null pointer, bad degree, non-positive scale, opacity outside
 * (0,1], zero quaternion, non-finite value), UNKNOWN_BODY, CAPACITY (N >= 2^32),
 * DEVICE, OUT_OF_MEMORY, CUDA. */
gsb_status gsb_create_scene(const float* means, const float* scales, const float* quats,
                            const float* opacities, const float* sh, int32_t sh_degree,
                            const int32_t* body_id, int64_t n_gaussians, int32_t n_bodies,
                            int32_t device, gsb_scene* out);

/* Size the device workspace for renders of up to max_envs envs x n_cams cameras at
 * width x height (allocations happen here, never in gsb_render).  chunk_frames = number of
 * env-camera frames processed per pipeline chunk (0 = automatic; capped so that chunk frames x
 * N < 2^32, K4b's 32-bit record index).  key_capacity = tile keys
 * held per chunk (0 = automatic); a chunk whose keys exceed it is split by frames, a single
 * frame exceeding it fails with GSB_ERR_CAPACITY.  flags: GSB_RESERVE_HOST_IO. */
gsb_status gsb_reserve(gsb_scene scene, int32_t max_envs, int32_t n_cams, int32_t width,
                       int32_t height, int32_t chunk_frames, int64_t key_capacity,
                       uint32_t flags);

/* Render every env-camera frame f = e*C + c (ALL pointers DEVICE, on the scene's device):
 *   body_poses   [B, n_bodies, 7] fp32 (R22); may be NULL iff n_bodies == 0
 *   intrinsics   [B, C, 4] fp32 (fx, fy, cx, cy) pixels
 *   world_to_cam [B, C, 3, 4] fp32 row-major [R | t], OpenCV axes
 *   out_rgb      [B, C, 3, H, W] fp32  C + T * background            (required)
 *   out_depth    [B, C, H, W] fp32     sum_i w_i z_i  (R16)          (nullable)
 *   out_alpha    [B, C, H, W] fp32     1 - T                         (nullable)
 *   out_n_eval   [B, C, H, W] int32    tile-list entries evaluated up to and including the
 *                                      termination entry (list length if none)  (nullable)
 * Work is enqueued on `stream`; the host may block until the last chunk's projection has
 * finished (per-chunk key-count readback that sizes the binning).
 * Outputs are fully overwritten.  Caller keeps every buffer alive until `stream` completes.
 * Errors: INVALID_ARGUMENT, SHAPE_MISMATCH (B*C or W,H beyond the reservation, C != the
 * reserved camera count is allowed if B*C fits), CAPACITY, CUDA. */
gsb_status gsb_render(gsb_scene scene, const float* body_poses, int32_t n_envs, int32_t n_cams,
                      const float* intrinsics, const float* world_to_cam,
                      const gsb_render_params* params, float* out_rgb, float* out_depth,
                      float* out_alpha, int32_t* out_n_eval, gsb_stream stream);

/* gsb_render with a camera rig and strided pose input (§8(f) row 1: egocentric / wrist cameras
 * and direct physics-buffer ingest).  DEVICE pointers as in gsb_render, except cam_body.
 *   body_poses of env e, body k start at body_poses[e * pose_env_stride + k * pose_body_stride]
 *     and hold (tx,ty,tz,qw,qx,qy,qz) in their first 7 floats (e.g. a physics state record);
 *     pose_body_stride 0 = 7 (>= 7 otherwise), pose_env_stride 0 = n_bodies * pose_body_stride
 *   cam_body     [C] int32 HOST array, nullable: cam_body[c] = -1 -> cam_extrinsics[e,c] is
 *     world->camera as in gsb_render; cam_body[c] = k >= 0 -> cam_extrinsics[e,c] is the camera's
 *     body->camera [R | t] (mount, may differ per env) and world->camera is composed on the device
 *     by the binary32 chain of reading R29; k must be in [0, n_bodies), c < 16.
 * Errors: as gsb_render, plus UNKNOWN_BODY (bad cam_body), INVALID_ARGUMENT (bad strides),
 * CAPACITY (attached camera index >= 16). */
gsb_status gsb_render_rig(gsb_scene scene, const float* body_poses, int64_t pose_env_stride,
                          int64_t pose_body_stride, int32_t n_envs, int32_t n_cams,
                          const float* intrinsics, const float* cam_extrinsics, const int32_t* cam_body,
                          const gsb_render_params* params, float* out_rgb, float* out_depth,
                          float* out_alpha, int32_t* out_n_eval, gsb_stream stream);

/* Same operation with HOST buffers (inputs read, outputs written; pinned memory recommended):
 * uploads the inputs, renders, and downloads rgb (+depth/alpha/n_eval when non-NULL), with
 * the downloads of one chunk overlapping the rendering of the next.  Synchronous: returns
 * when the outputs are in host memory.  Requires gsb_reserve(..., GSB_RESERVE_HOST_IO). */
gsb_status gsb_render_host(gsb_scene scene, const float* body_poses, int32_t n_envs,
                           int32_t n_cams, const float* intrinsics, const float* world_to_cam,
                           const gsb_render_params* params, float* out_rgb, float* out_depth,
                           float* out_alpha, int32_t* out_n_eval, gsb_stream stream);

/* Observation epilogue (§8(f) row 4; reading R31 in DESIGN.md / oracle/obs.py): the policy-
 * facing encoding fused into K4's store — image domain randomisation ("brightness, contrast
 * and exposure"; "image noise") and 8-bit RGB (+ fp16 depth), so a batch leaves
 * HBM (and crosses PCIe) at 3-5 B per pixel instead of 16.  Per frame f with
 * (gain, contrast, brightness, noise_std) = image_dr[f] and c = C + T*bg (binary32, RN):
 *   v = ((c*gain - 0.5)*contrast + 0.5) + brightness [+ (z*sqrt(3)/2^22)*noise_std]
 *   rgb8 = rint(clamp(v, 0, 1) * 255)            (NaN -> 0)
 * z = Irwin-Hall(4) counter-based noise keyed by (seed, step, global frame
 * (env_offset + e)*C + c, pixel, channel) — identical under any env slicing.  Motion blur
 * (a neighbourhood operation) is not part of this fused epilogue: see gsb_obs_encode. */
#define GSB_OBS_DEPTH_F16 1u  /* out_depth holds IEEE half bits (uint16), else fp32 */
typedef struct {
  const float* image_dr;  /* [B, C, 4] fp32 (gain, contrast, brightness, noise_std) per frame, or
                             NULL = identity (1, 1, 0, 0); DEVICE for gsb_render_obs, HOST for
                             gsb_render_obs_host */
  uint32_t seed, step;    /* noise stream */
  int64_t env_offset;     /* global index of env 0 of this call (sharded runs), >= 0 */
  uint32_t flags;         /* GSB_OBS_* */
} gsb_obs_params;

/* gsb_render with the observation epilogue: out_rgb8 [B, C, 3, H, W] uint8 (required),
 * out_depth [B, C, H, W] fp16 bits or fp32 per GSB_OBS_DEPTH_F16 (nullable).  DEVICE buffers.
 * Errors as gsb_render, plus INVALID_ARGUMENT for bad obs params. */
gsb_status gsb_render_obs(gsb_scene scene, const float* body_poses, int32_t n_envs, int32_t n_cams,
                          const float* intrinsics, const float* world_to_cam,
                          const gsb_render_params* params, const gsb_obs_params* obs,
                          uint8_t* out_rgb8, void* out_depth, gsb_stream stream);
/* The same with HOST buffers (inputs incl. image_dr read, outputs written; pinned memory
 * recommended), downloads overlapping the next chunk, synchronous; needs GSB_RESERVE_HOST_IO. */
gsb_status gsb_render_obs_host(gsb_scene scene, const float* body_poses, int32_t n_envs,
                               int32_t n_cams, const float* intrinsics, const float* world_to_cam,
                               const gsb_render_params* params, const gsb_obs_params* obs,
                               uint8_t* out_rgb8, void* out_depth, gsb_stream stream);

/* The observation encoding as a standalone pass over rendered fp32 frames, with the motion blur
 * of reading R33 ("image noise and motion blur", oracle/obs.py) in front of
 * the R31 DR/encoding.  Per frame f with blur[f] = (bx, by) integer pixels (each clamped to
 * [-64, 64]):
 * L = max(|bx|, |by|) + 1 taps at o_k = floor((2 k b + L - 1) / (2 (L - 1))) - floor(b / 2) per
 * axis, edge-clamped samples, acc = sum in tap order (binary32 RN), blurred = acc / L; then R31.
 * Depth is not blurred.  DEVICE pointers:
 *   rgb        [B, C, 3, H, W] fp32 (e.g. gsb_render's out_rgb), depth [B, C, H, W] fp32 (nullable)
 *   blur       [B, C, 2] int32 (nullable = no blur; then the codes equal gsb_render_obs's)
 *   obs        as gsb_render_obs (image_dr DEVICE); out_rgb8 [B, C, 3, H, W] uint8;
 *   out_depth  [B, C, H, W] fp16 bits or fp32 per GSB_OBS_DEPTH_F16 (written when depth != NULL).
 * Asynchronous on stream; no scene needed.  Errors: INVALID_ARGUMENT, CUDA. */
gsb_status gsb_obs_encode(const float* rgb, const float* depth, int32_t n_envs, int32_t n_cams, int32_t width,
                          int32_t height, const gsb_obs_params* obs, const int32_t* blur, uint8_t* out_rgb8,
                          void* out_depth, gsb_stream stream);

/* Static-camera background pre-binning (§8(f) row 2; exploits RLGK's static/dynamic split,
 * PAPER.md App. B.2: static Gaussians never move, so with cameras fixed in the world
 * their projection, binning and depth sort are the same for every env and every step).
 * gsb_prebin_static projects, bins and sorts the static (body -1) Gaussians once for the C
 * cameras given (DEVICE or HOST pointers: intrinsics [C,4], world_to_cam [C,3,4]), and keeps
 * the sorted per-(camera, tile) lists and their records in the scene (replacing any previous
 * pre-binning; synchronous).  Call gsb_reserve (again) afterwards if the scene was reserved
 * before, so the merge workspace exists.
 * gsb_render_static then renders B envs x those C cameras (frame f = e*C + c; with
 * GSB_FLAG_STATIC_PER_ENV: B <= C envs x 1 camera, env e seen by camera e): per frame only
 * the robot Gaussians are projected, binned and sorted, and K4 merges each tile's robot list
 * with the camera's background list in (zbits, id) order (keys are unique, reading R10).
 * Outputs, layout and determinism as gsb_render with intrinsics/world_to_cam broadcast over
 * the envs — bit-identical to it.  params must equal the pre-binning's in width, height,
 * near/far and SH degree (background and flags may differ).
 * Errors: INVALID_ARGUMENT (no pre-binning / reservation, bad params), SHAPE_MISMATCH
 * (params differ from the pre-binning's, B*C beyond the reservation), CAPACITY, CUDA,
 * OUT_OF_MEMORY. */
gsb_status gsb_prebin_static(gsb_scene scene, int32_t n_cams, const float* intrinsics,
                             const float* world_to_cam, const gsb_render_params* params,
                             gsb_stream stream);
gsb_status gsb_render_static(gsb_scene scene, const float* body_poses, int32_t n_envs,
                             const gsb_render_params* params, float* out_rgb, float* out_depth,
                             float* out_alpha, int32_t* out_n_eval, gsb_stream stream);

/* GSB_FLAG_FIXED_PLAN renders: *out = 1 if any chunk since the last call overflowed the reserved key
 * capacity (its frames were not written; reserve a larger key_capacity), else 0; resets the flag.
 * Synchronises with the scene's last render. */
gsb_status gsb_get_overflow(gsb_scene scene, int32_t* out);

/* Counters of the last render made with GSB_FLAG_STATS (synchronises with it). */
gsb_status gsb_get_stats(gsb_scene scene, int64_t* visible_V, int64_t* keys_K, int64_t* pairs_P);

/* The same counters plus the SURVEY §8(d) d.4 (iv) workload statistic: pixels whose
 * compositing stopped at the termination test (reading R13), out of all pixels rendered. */
typedef struct {
  int64_t visible_V, keys_K, pairs_P;
  int64_t terminated_pixels, pixels;
} gsb_stats;
gsb_status gsb_get_stats_ext(gsb_scene scene, gsb_stats* out);

/* Per-kernel-class device time of the last render made with GSB_FLAG_TIMING, in ms
 * (synchronises with it), and the number of kernels libgsb launched in that render. */
typedef struct {
  double setup_ms;     /* K0: per-(frame, body) RLGK transforms */
  double project_ms;   /* K1: fused pose + projection + 2D covariance + SH, tile histogram */
  double scan_ms;      /* K2a: per-frame tile offsets */
  double emit_ms;      /* K2b: key emission */
  double sort_ms;      /* K3: segmented radix sort */
  double composite_ms; /* K4: per-tile compositing */
  int64_t launches;    /* kernels launched by libgsb in the last render */
  int64_t composite_launches;
  int64_t chunks;
  int64_t long_lists;  /* tile lists longer than K4's fused-sort capacity (sorted by K3) */
  int64_t max_list;    /* longest tile list of the render */
} gsb_timings;
gsb_status gsb_get_timings(gsb_scene scene, gsb_timings* out);

/* Renderer-driven pruning scores (§8(f) row 3; "efficient pruning strategy",
 * after the rendering-importance scores of its citations; reading R30 in DESIGN.md).  Every
 * render made with GSB_FLAG_SCORES adds, for each Gaussian, the blend weights w = alpha T it
 * received (step 7 of the oracle; terminating and skipped entries receive none) over all pixels
 * of all its frames: sum and max.  fp32; the sum's order of addition is not fixed (atomics), the
 * max is exact.  Accumulators live in the scene (8 B per Gaussian, zero at creation).
 * gsb_scores_reset zeroes them (enqueued on stream).  gsb_get_scores copies them, by creation
 * index, into DEVICE arrays w_sum [N] / w_max [N] (either may be NULL), enqueued on stream. */
gsb_status gsb_scores_reset(gsb_scene scene, gsb_stream stream);
gsb_status gsb_get_scores(gsb_scene scene, float* w_sum, float* w_max, gsb_stream stream);

/* filter_template semantics: a new scene, on the same device, holding the
 * Gaussians with keep[id] != 0 (keep: HOST uint8 [N], by creation index) in creation order,
 * re-indexed 0..M-1 (ids, and so the R10 tie-break, follow the original order); bodies and all
 * parameters are preserved.  Rendering the result equals rendering a scene created from the
 * kept Gaussians directly.  The new scene is unreserved and has no pre-binning or scores.
 * Synchronous.  Errors: INVALID_ARGUMENT, OUT_OF_MEMORY, CUDA. */
gsb_status gsb_filter_scene(gsb_scene scene, const uint8_t* keep, gsb_scene* out);

gsb_status gsb_destroy_scene(gsb_scene scene);

/* ------------------------------------------------------------ batched ray-cast LiDAR (R32)
 * §8(f) row 4: "Batch-LiDAR module utilizing ray-casting", rotating, solid-state and
 * non-repetitive scans (tab:lidar P:320-329), omnidirectional/bounded LiDAR and the downward
 * Height Scan.  The paper gives no formula; reading R32 (DESIGN.md,
 * oracle/gsb_oracle.c) casts each ray against the same RLGK-posed Gaussians the cameras see:
 *   x = sensor-frame mean, P = (sensor-frame Sigma)^-1, d = unit ray direction (sensor frame);
 *   t^ = max(0, d^T P x / d^T P d)       peak of the Gaussian on the half-ray t >= 0
 *   alpha = min(0.99, o exp(-(x - t^ d)^T P (x - t^ d) / 2))
 * composited front-to-back in (bits(rho_f32), id) order, rho = |x| by the binary32 chain of
 * R32 (R11 applied to all three rows), with the camera rules R12-R14 (skip alpha < 1/255,
 * stop before blending when T(1-alpha) < 1e-4) and outputs
 *   range = sum_w w t^   (metres; the ray's expected hit distance is range / alpha)
 *   alpha = 1 - T.
 * A point cloud is origin + (range / alpha) d for rays with alpha above the user's threshold. */
typedef struct gsb_lidar_t* gsb_lidar; /* a ray pattern bound to one scene's device */

/* Upload a ray pattern: dirs = HOST [n_rays, 3] fp32 unit vectors in the sensor frame
 * (|norm - 1| <= 1e-5), any order (rotating, solid-state, non-repetitive, height scan ...).
 * The pattern is bucketed into an azimuth x elevation grid of cells (n_az, n_el <= 256 each;
 * 0 = automatic, ~32 rays per cell) covering the rays' angular window; Gaussians are binned
 * into the same cells.  Synchronous.  Errors: INVALID_ARGUMENT, OUT_OF_MEMORY, CUDA. */
gsb_status gsb_lidar_create(gsb_scene scene, const float* dirs, int32_t n_rays, int32_t n_az, int32_t n_el,
                            gsb_lidar* out);

/* Cast every ray of `lidar` for S sensors per env.  DEVICE pointers:
 *   body_poses    [B, n_bodies, 7] fp32 (as gsb_render)
 *   sensor_x      [B, S, 3, 4] fp32, or [S, 3, 4] when sensors_shared != 0: world->sensor
 *                 [R | t] (sensor axes: the ray directions' frame), or, for a sensor with
 *                 sensor_body[s] = k >= 0, the body->sensor mount composed per env by R29
 *   sensor_body   [S] int32 HOST array, nullable (all world-fixed); S <= 16 when set
 *   out_range     [B, S, n_rays] fp32, out_alpha [B, S, n_rays] fp32 (nullable)
 * near < rho <= far culls by the range key (R4 with rho for z).  Allocates its workspace on
 * first use and when a batch needs more (then synchronises); otherwise asynchronous on stream.
 * Errors: INVALID_ARGUMENT, SHAPE_MISMATCH (n_bodies), UNKNOWN_BODY, OUT_OF_MEMORY, CUDA. */
gsb_status gsb_render_lidar(gsb_scene scene, gsb_lidar lidar, const float* body_poses, int32_t n_envs,
                            int32_t n_sensors, const float* sensor_x, int32_t sensors_shared,
                            const int32_t* sensor_body, float near_plane, float far_plane, float* out_range,
                            float* out_alpha, gsb_stream stream);

/* Grid of the pattern: n_az, n_el, and the rays-per-cell work items (nullable outputs). */
gsb_status gsb_lidar_info(gsb_lidar lidar, int32_t* n_az, int32_t* n_el, int32_t* n_items, int64_t* last_keys);

gsb_status gsb_lidar_destroy(gsb_lidar lidar);

/* Thread-local message for the last non-OK status (never NULL). */
const char* gsb_last_error(void);

/* Library version string, e.g. "gsb 0.1 sm_100a". */
const char* gsb_version(void);

/* ------------------------------------------------------------------ test-only entry points */

/* K1 projection only, dense per (frame, Gaussian) (DEVICE pointers, same inputs as gsb_render):
 *   out_rec   [F, N, 16] fp32: u, v, conic a, b, c, opacity, r, g, b, z, Sigma2D_xx, Sigma2D_yy,
 *             then the values K4 composites with: the whitening factor (p, q, r) of Sigma2D^-1
 *             scaled by sqrt(log2(e)/2) (arg = log2 o - (p dx)^2 - (q dx + r dy)^2) and log2 o
 *   out_zbits [F, N] uint32  bits of the fp32 depth key (reading R11)
 *   out_valid [F, N] uint8   near < z <= far and o >= 1/255 (R4, R5)
 * Requires the same reservation as gsb_render for B*C frames. */
gsb_status gsb_debug_project(gsb_scene scene, const float* body_poses, int32_t n_envs,
                             int32_t n_cams, const float* intrinsics, const float* world_to_cam,
                             const gsb_render_params* params, float* out_rec, uint32_t* out_zbits,
                             uint8_t* out_valid, gsb_stream stream);

/* K2 + K3 on externally supplied projections (the ORACLE's values rounded to fp32), all
 * [F, N] DEVICE arrays: u, v, Sigma2D_xx, Sigma2D_yy, kappa = 2 ln(255 o), zbits, valid.
 * Computes tile rects by reading R9, bins, sorts every (frame, tile) list by (zbits, id)
 * (reading R10) and writes out_tile_offsets [F, T_t + 1] (DEVICE, int64, absolute positions
 * in out_ids) and out_ids [cap] (DEVICE uint32).  *out_K (HOST) receives the total.
 * Allocates its own scratch (test-only).  CAPACITY if the total exceeds cap. */
gsb_status gsb_debug_bin_sort(const float* u, const float* v, const float* sxx, const float* syy,
                              const float* kappa, const uint32_t* zbits, const uint8_t* valid,
                              int32_t n_frames, int64_t n_gaussians, int32_t width, int32_t height,
                              int64_t* out_tile_offsets, uint32_t* out_ids, int64_t cap,
                              int64_t* out_K, gsb_stream stream);

/* The PRODUCTION binning and tile sort — K2b emission and the sort that feeds compositing in
 * gsb_render (K4a of the split path, or the fused K4's in-CTA sort) — on external projections
 * (the ORACLE's values rounded to fp32), so the integer path the render really runs is
 * compared list for list with the binning oracle (readings R9, R10).
 *   u .. valid   [F, N] DEVICE arrays indexed by record SLOT j (the internal order)
 *   slot_ids     [N] DEVICE int32: creation id of slot j (a permutation of [0, N)); keys break
 *                depth ties by this id, so a non-identity permutation exercises the slot-key
 *                path's re-ordering of equal-depth runs
 *   variant      0 = what gsb_render picks for this batch (split if >= 200 keys per tile on
 *                average, packed sort if > 1/4 of the lists exceed 1024 keys), 1 = K4a as the
 *                render runs it for short lists (one warp per list <= 512 keys, one CTA with the
 *                index counting sort per longer list <= 4096, HBM radix beyond), 2 = K4a for views
 *                whose lists are mostly long (one CTA per list: index counting sort <= 4096, HBM
 *                radix beyond), 3 = fused K4
 *                small, 4 = fused K4 packed, 5 = K4a one CTA per list (counting sort <= 1024 keys
 *                in smem, HBM radix beyond; the LiDAR path's sort)
 *   key_mode     0 = keys carry the record slot (gsb_render's default), 1 = keys carry the id,
 *                2 = slot keys with K4b block masks in their low 4 bits (variants 1 and 2 only;
 *                the mask is set to slot & 15 and checked to travel with its entry)
 *   out_tile_offsets [F, T_t + 1] DEVICE int64 (absolute positions in out_ids),
 *   out_ids      [cap] DEVICE uint32: creation ids of every (frame, tile) list in sorted order
 *   out_K, out_variant (HOST): total keys and the variant that ran (1..5).
 * Allocates its own scratch and synchronises (test-only).  CAPACITY if K > cap. */
gsb_status gsb_debug_tile_lists(const float* u, const float* v, const float* sxx, const float* syy,
                                const float* kappa, const uint32_t* zbits, const uint8_t* valid,
                                const int32_t* slot_ids, int32_t n_frames, int64_t n_gaussians,
                                int32_t width, int32_t height, int32_t variant, int32_t key_mode,
                                int64_t* out_tile_offsets, uint32_t* out_ids, int64_t cap,
                                int64_t* out_K, int32_t* out_variant, gsb_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* GSB_H_ */
