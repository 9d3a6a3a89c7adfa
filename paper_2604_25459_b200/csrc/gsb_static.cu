// gsb_static.cu — static-camera background pre-binning (§8(f) row 2; RLGK's static/dynamic
// split, App. B.2): gsb_prebin_static bins and sorts the static background once per
// camera; gsb_render_static then projects and bins only the robot Gaussians per frame and K4
// merges the two (zbits, id)-ordered lists per tile (bit-identical to gsb_render).
#include "gsb_runtime.cuh"

using namespace gsb;

extern "C" {

gsb_status gsb_prebin_static(gsb_scene s, int32_t n_cams, const float* intr, const float* w2c,
                             const gsb_render_params* p, gsb_stream stream) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (!p || !intr || !w2c) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL params/intrinsics/world_to_cam");
  if (n_cams < 1 || n_cams > 4096) return fail(GSB_ERR_INVALID_ARGUMENT, "n_cams=%d not in 1..4096", n_cams);
  if (p->width < 1 || p->height < 1 || p->width > kMaxDim || p->height > kMaxDim)
    return fail(GSB_ERR_INVALID_ARGUMENT, "image %dx%d outside 1..%d", p->width, p->height, kMaxDim);
  if (!(p->near_plane > 0.f) || !(p->far_plane > p->near_plane))
    return fail(GSB_ERR_INVALID_ARGUMENT, "need 0 < near < far");
  if (p->sh_degree > s->sh_degree || p->sh_degree < -1)
    return fail(GSB_ERR_INVALID_ARGUMENT, "sh_degree %d not in [-1, %d]", p->sh_degree, s->sh_degree);
  DeviceGuard g(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaStreamSynchronize(st));
  s->free_prebin();
  const int C = n_cams, W = p->width, H = p->height;
  const int tiles_x = (W + kTile - 1) / kTile;
  const int n_tiles = tiles_x * ((H + kTile - 1) / kTile);
  const int64_t stride = ((int64_t)n_tiles + 2 + 31) / 32 * 32;
  const int64_t nbg = s->n_bg, vwords = (nbg + 31) / 32;
  const int nb1 = s->n_bodies + 1;
  const int D = p->sh_degree < 0 ? s->sh_degree : p->sh_degree;
  float* poses = nullptr; float4* table = nullptr; FrameCam* cams = nullptr; float4* rec = nullptr;
  uint2* emit = nullptr;
  int* vcount = nullptr; int* hist = nullptr; uint32_t* off = nullptr; uint32_t* vbits = nullptr;
  uint64_t* fbase = nullptr; uint64_t* keys = nullptr; uint64_t* keys_alt = nullptr; uint32_t* sorted = nullptr;
  auto cleanup = [&]() {
    cudaFree(poses); cudaFree(table); cudaFree(cams); cudaFree(rec); cudaFree(emit); cudaFree(vcount); cudaFree(hist);
    cudaFree(off); cudaFree(vbits); cudaFree(fbase); cudaFree(keys); cudaFree(keys_alt); cudaFree(sorted);
  };
#define PB_TRY(expr)                                                                            \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      cleanup();                                                                                \
      s->free_prebin();                                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? GSB_ERR_OUT_OF_MEMORY : GSB_ERR_CUDA, "%s: %s", #expr, \
                  cudaGetErrorString(e_));                                                      \
    }                                                                                           \
  } while (0)
  // the camera set, kept for gsb_render_static's K0
  PB_TRY(dalloc(&s->sb_intr, (size_t)C * 4));
  PB_TRY(dalloc(&s->sb_w2c, (size_t)C * 12));
  PB_TRY(cudaMemcpyAsync(s->sb_intr, intr, sizeof(float) * C * 4, cudaMemcpyDefault, st));
  PB_TRY(cudaMemcpyAsync(s->sb_w2c, w2c, sizeof(float) * C * 12, cudaMemcpyDefault, st));
  // K0 for the C cameras (body rows unused: identity poses)
  std::vector<float> idp((size_t)std::max(s->n_bodies, 1) * 7, 0.f);
  for (size_t k = 0; k < idp.size() / 7; ++k) idp[k * 7 + 3] = 1.f;
  PB_TRY(dalloc(&poses, idp.size()));
  PB_TRY(cudaMemcpyAsync(poses, idp.data(), sizeof(float) * idp.size(), cudaMemcpyHostToDevice, st));
  PB_TRY(dalloc(&table, (size_t)C * nb1 * 4));
  PB_TRY(dalloc(&cams, (size_t)C));
  K0Rig rig = default_rig(s, poses, s->sb_intr, s->sb_w2c);
  rig.env_stride = 0;
  launch_k0(rig, C, C, s->n_bodies, W, H, table, cams, st);
  PB_TRY(cudaGetLastError());
  // K1 over the background prefix, K2 scan
  PB_TRY(dalloc(&rec, (size_t)C * std::max<int64_t>(nbg, 1) * kRecQuads));
  PB_TRY(dalloc(&emit, (size_t)C * std::max<int64_t>(nbg, 1)));
  PB_TRY(dalloc(&vcount, (size_t)C));
  PB_TRY(dalloc(&vbits, (size_t)C * std::max<int64_t>(vwords, 1)));
  PB_TRY(dalloc(&hist, (size_t)C * stride));
  PB_TRY(dalloc(&off, (size_t)C * stride));
  PB_TRY(dalloc(&fbase, (size_t)C + 2));
  PB_TRY(cudaMemsetAsync(vcount, 0, sizeof(int) * C, st));
  PB_TRY(cudaMemsetAsync(hist, 0, sizeof(int) * C * stride, st));
  PB_TRY(cudaMemsetAsync(off, 0, sizeof(uint32_t) * C * stride, st));   // padding rows are read back below
  K1Args a{};
  a.g_mean = s->d_mean; a.g_L0 = s->d_L0; a.g_L1 = s->d_L1; a.g_L2 = s->d_L2; a.g_sh = s->d_sh;
  a.g_ids = s->d_ids;
  a.n = nbg; a.sh_stride = s->n; a.table = table; a.cams = cams; a.nb1 = nb1;
  a.f0 = 0; a.n_frames = C; a.width = W; a.height = H; a.tiles_x = tiles_x;
  a.near_plane = p->near_plane; a.far_plane = p->far_plane;
  a.rec = rec; a.emit = emit;
  a.vcount = vcount; a.hist = hist; a.hist_stride = stride; a.vis_bits = vbits; a.vis_words = vwords;
  launch_k1(a, D, st);
  launch_k2_scan(hist, off, stride, C, n_tiles, fbase, nullptr, nullptr, 0, nullptr, nullptr, st);
  PB_TRY(cudaGetLastError());
  std::vector<uint64_t> hfb(C + 2);
  std::vector<int> hv(C);
  PB_TRY(cudaMemcpyAsync(hfb.data(), fbase, sizeof(uint64_t) * (C + 2), cudaMemcpyDeviceToHost, st));
  PB_TRY(cudaMemcpyAsync(hv.data(), vcount, sizeof(int) * C, cudaMemcpyDeviceToHost, st));
  PB_TRY(cudaStreamSynchronize(st));
  const uint64_t K = hfb[C];
  uint64_t maxk = 0;
  for (int c = 0; c < C; ++c) maxk = std::max<uint64_t>(maxk, hfb[c + 1] - hfb[c]);
  // K2 emission, K3 sort of every list, gather into list order
  PB_TRY(dalloc(&keys, std::max<uint64_t>(K, 1)));
  PB_TRY(dalloc(&keys_alt, std::max<uint64_t>(K, 1)));
  PB_TRY(dalloc(&sorted, std::max<uint64_t>(K, 1)));
  PB_TRY(dalloc(&s->bg_keys, std::max<uint64_t>(K, 1)));
  PB_TRY(dalloc(&s->bg_rec, std::max<uint64_t>(K, 1) * 3));
  ChunkArgs ca{};
  ca.rec = rec; ca.emit = emit; ca.ids = s->d_ids; ca.n = nbg; ca.vis_bits = vbits; ca.vis_words = vwords; ca.hist = hist; ca.hist_stride = stride;
  ca.off = off; ca.frame_base = fbase; ca.n_tiles = n_tiles; ca.tiles_x = tiles_x; ca.fs = 0; ca.fe = C;
  ca.key_base = 0; ca.long_list = nullptr; ca.keys = keys; ca.keys_alt = keys_alt; ca.sorted = sorted;
  launch_k2_emit(ca, st);
  launch_k3_sort(ca, 0, st);
  launch_k3_prebin_gather(sorted, fbase, rec, nbg, s->d_inv, C, maxk, s->bg_keys, s->bg_rec, st);
  PB_TRY(cudaGetLastError());
  std::vector<uint32_t> hoff((size_t)C * stride);
  PB_TRY(cudaMemcpyAsync(hoff.data(), off, sizeof(uint32_t) * hoff.size(), cudaMemcpyDeviceToHost, st));
  PB_TRY(cudaStreamSynchronize(st));
  std::vector<uint64_t> bo((size_t)C * (n_tiles + 1));
  for (int c = 0; c < C; ++c)
    for (int t = 0; t <= n_tiles; ++t) bo[(size_t)c * (n_tiles + 1) + t] = hfb[c] + hoff[(size_t)c * stride + t];
  PB_TRY(dalloc(&s->bg_off, bo.size()));
  PB_TRY(cudaMemcpyAsync(s->bg_off, bo.data(), sizeof(uint64_t) * bo.size(), cudaMemcpyHostToDevice, st));
  if (s->reserved && !s->qpos) PB_TRY(dalloc(&s->qpos, (size_t)s->cap));
  PB_TRY(cudaStreamSynchronize(st));
  cleanup();
#undef PB_TRY
  s->sb_cams = C; s->sb_w = W; s->sb_h = H; s->sb_D = D; s->sb_near = p->near_plane; s->sb_far = p->far_plane;
  s->sb_V.resize(C); s->sb_K.resize(C);
  std::vector<uint64_t> cum(C + 1, 0);
  for (int c = 0; c < C; ++c) {
    s->sb_V[c] = hv[c];
    s->sb_K[c] = (int64_t)(hfb[c + 1] - hfb[c]);
    cum[c + 1] = cum[c] + (uint64_t)s->sb_K[c];
  }
  if (dalloc(&s->d_bgcum, (size_t)C + 1) != cudaSuccess ||
      cudaMemcpy(s->d_bgcum, cum.data(), sizeof(uint64_t) * (C + 1), cudaMemcpyHostToDevice) != cudaSuccess) {
    s->free_prebin();
    return fail(GSB_ERR_OUT_OF_MEMORY, "prebin: background size table");
  }
  return GSB_OK;
}

gsb_status gsb_render_static(gsb_scene s, const float* poses, int32_t n_envs, const gsb_render_params* p,
                             float* out_rgb, float* out_depth, float* out_alpha, int32_t* out_neval,
                             gsb_stream stream) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (s->sb_cams < 1) return fail(GSB_ERR_INVALID_ARGUMENT, "gsb_prebin_static was not called");
  const bool per_env = p && (p->flags & GSB_FLAG_STATIC_PER_ENV);
  if (per_env && n_envs > s->sb_cams)
    return fail(GSB_ERR_SHAPE_MISMATCH, "GSB_FLAG_STATIC_PER_ENV: %d envs > %d pre-binned cameras", n_envs, s->sb_cams);
  const int C = per_env ? 1 : s->sb_cams;
  gsb_status r = validate_render(s, poses, n_envs, C, s->sb_intr, s->sb_w2c, p, out_rgb);
  if (r != GSB_OK) return r;
  const int D = p->sh_degree < 0 ? s->sh_degree : p->sh_degree;
  if (p->width != s->sb_w || p->height != s->sb_h || p->near_plane != s->sb_near || p->far_plane != s->sb_far ||
      D != s->sb_D)
    return fail(GSB_ERR_SHAPE_MISMATCH, "params differ from gsb_prebin_static's (image, near/far, sh_degree)");
  if (!s->qpos) return fail(GSB_ERR_INVALID_ARGUMENT, "gsb_reserve was not called after gsb_prebin_static");
  if (p->flags & GSB_FLAG_SCORES) return fail(GSB_ERR_INVALID_ARGUMENT, "GSB_FLAG_SCORES is not supported by gsb_render_static");
  DeviceGuard g(s->device);
  s->dl_rgb = nullptr; s->dl_depth = nullptr; s->dl_alpha = nullptr; s->dl_neval = nullptr;
  K0Rig rig = default_rig(s, poses, s->sb_intr, s->sb_w2c);
  // frame f uses pre-binned camera f mod C in K4's merge; K0 reads the same camera: shared
  // camera rows (cam = f mod C) or, per env, row f (= env e, one camera per env)
  rig.cams_shared = per_env ? 0 : 1;
  return render_impl(s, rig, n_envs, C, p, out_rgb, out_depth, out_alpha, out_neval, (cudaStream_t)stream, true);
}

}  // extern "C"
