// gsb_render.cu — libgsb host runtime, part 2: the chunked render pipeline.
//
//   K0 setup (all frames) ;  for each chunk c of E frames (double-buffered slot c&1):
//     K1 project(c) -> records + tile histogram ; K2a scan(c) ; frame key counts -> mapped host memory
//     [host reads chunk c-1's counts — the GPU is busy with chunk c meanwhile]
//     K2b emit(c-1) ; K4a sort + K4b blend, or fused K4 (c-1)   (split by frames if keys > capacity)
//
// Three internal streams: projection (K1, K2a) runs a chunk ahead of binning + sort (K2b, K4a),
// which runs a pass ahead of compositing (K4b).  No allocation happens in a render; all buffers
// are sized by gsb_reserve (gsb_api.cu).  Entry points: gsb_render, gsb_render_rig,
// gsb_render_host and the observation renders (reading R31) + gsb_obs_encode (K6, R33).
#include "gsb_runtime.cuh"

using namespace gsb;

namespace gsb {

gsb_status validate_render(gsb_scene s, const float* poses, int n_envs, int n_cams, const float* intr,
                           const float* w2c, const gsb_render_params* p, const float* out_rgb) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (!s->reserved) return fail(GSB_ERR_INVALID_ARGUMENT, "gsb_reserve was not called");
  if (!p) return fail(GSB_ERR_INVALID_ARGUMENT, "params is NULL");
  if (n_envs < 0 || n_cams < 1) return fail(GSB_ERR_INVALID_ARGUMENT, "n_envs=%d n_cams=%d", n_envs, n_cams);
  const int64_t F = (int64_t)n_envs * n_cams;
  if (F > s->max_frames)
    return fail(GSB_ERR_SHAPE_MISMATCH, "%lld frames exceed the reservation (%d)", (long long)F, s->max_frames);
  if (p->width < 1 || p->height < 1 || p->width > s->res_w || p->height > s->res_h)
    return fail(GSB_ERR_SHAPE_MISMATCH, "image %dx%d outside the reservation %dx%d", p->width, p->height, s->res_w, s->res_h);
  if (!(p->near_plane > 0.f) || !(p->far_plane > p->near_plane))
    return fail(GSB_ERR_INVALID_ARGUMENT, "need 0 < near < far");
  if (p->sh_degree > s->sh_degree || p->sh_degree < -1)
    return fail(GSB_ERR_INVALID_ARGUMENT, "sh_degree %d not in [-1, %d]", p->sh_degree, s->sh_degree);
  if (F > 0) {
    if (!intr || !w2c || !out_rgb) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL intrinsics/world_to_cam/out_rgb");
    if (s->n_bodies > 0 && !poses) return fail(GSB_ERR_INVALID_ARGUMENT, "body_poses is NULL but the scene has bodies");
  }
  return GSB_OK;
}

struct Pipeline {
  gsb_scene_t* s;
  cudaStream_t st;        // the caller's stream
  cudaStream_t sp, sc;    // projection / compositing streams (== st when GSB_STREAMS=1)
  cudaStream_t sb;        // binning + sort stream (== sc unless three streams)
  int pass_idx = 0;       // passes so far in this render (parity selects the `sorted` buffer)
  const gsb_render_params* p;
  int F, W, H, tiles_x, n_tiles, D, n_cams;
  Timer tm;
  float* out_rgb;
  float* out_depth;
  float* out_alpha;
  int32_t* out_neval;
  int64_t first = 0, count = 0;   // Gaussian range [first, first + count) of the internal order
  bool merge = false;             // static cameras: merge with the pre-binned background lists
  bool masks_wanted = false;      // some pass of this render wanted K4b block masks
  bool fixed = false;             // GSB_FLAG_FIXED_PLAN: no host sync, no data-dependent launch choice
  uint32_t n_vlong = 0;           // the chunk's lists longer than kFusedSortCap

  gsb_status project_chunk(int c, int f0, int nf) {
    const int sl = c & 1;
    if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(sp, s->ev_done[sl], 0));   // chunk c-2 left this slot
    CUDA_TRY(cudaMemsetAsync(s->vcount[sl], 0, sizeof(int) * nf, sp));
    CUDA_TRY(cudaMemsetAsync(s->long_cnt[sl], 0, 2 * sizeof(uint32_t), sp));
    CUDA_TRY(cudaMemsetAsync(s->hist[sl], 0, sizeof(int) * s->hist_stride * nf, sp));
    K1Args a{};
    a.g_mean = s->d_mean + first; a.g_L0 = s->d_L0 + first; a.g_L1 = s->d_L1 + first;
    a.g_L2 = s->d_L2 + first; a.g_sh = s->d_sh + first;
    a.g_ids = s->d_ids + first;
    a.n = count; a.sh_stride = s->n; a.table = s->table; a.cams = s->cams; a.nb1 = s->n_bodies + 1;
    a.f0 = f0; a.n_frames = nf; a.width = W; a.height = H; a.tiles_x = tiles_x;
    a.near_plane = p->near_plane; a.far_plane = p->far_plane;
    a.rec = s->rec[sl]; a.emit = s->emit[sl];
    // trims only while block masks are in use (a render's first pass decides for the next render)
    const bool trims = !merge && block_masks_on() && s->mask_hint;
    a.trim = trims ? s->trim[sl] : nullptr;
    s->trim_valid[sl] = trims;
    a.vcount = s->vcount[sl]; a.hist = s->hist[sl]; a.hist_stride = s->hist_stride;
    a.vis_bits = s->vis_bits[sl]; a.vis_words = s->vis_words;
    tm.begin(KC_PROJECT, sp);
    launch_k1(a, D, sp);
    if (count > 0) s->launches++;
    LAUNCH_CHECK();
    tm.end();
    tm.begin(KC_SCAN, sp);
    launch_k2_scan(s->hist[sl], s->off[sl], s->hist_stride, nf, n_tiles, s->frame_base[sl], s->long_list[sl],
                   s->long_cnt[sl], kWarpSortCap, s->vcount[sl], fixed ? nullptr : s->d_rb[sl], sp,
                   fixed ? s->d_overflow + 1 + sl : nullptr, s->d_overflow, (uint64_t)s->cap);
    s->launches += 2;
    LAUNCH_CHECK();
    tm.end();
    CUDA_TRY(cudaEventRecord(s->ev_counts[sl], sp));
    return GSB_OK;
  }

  gsb_status pass(int sl, int f0, int fs, int fe, uint64_t key_base, uint64_t n_keys, uint32_t n_long) {
    ChunkArgs a{};
    a.rec = s->rec[sl]; a.emit = s->emit[sl]; a.ids = s->d_ids + first; a.n = count; a.vis_bits = s->vis_bits[sl]; a.vis_words = s->vis_words; a.hist = s->hist[sl];
    a.hist_stride = s->hist_stride; a.off = s->off[sl]; a.frame_base = s->frame_base[sl];
    a.n_tiles = n_tiles; a.tiles_x = tiles_x; a.fs = fs; a.fe = fe; a.key_base = key_base;
    const int q = pass_idx & 1;
    uint32_t* sorted = (q && sb != sc) ? s->sorted2 : s->sorted;
    a.keys = s->keys; a.keys_alt = s->keys_alt; a.sorted = sorted;
    a.long_list = s->long_list[sl];
    // the compositing path of this pass (decided before emission: the split path's small K4a
    // variant takes keys that carry the record slot instead of the creation id)
    uint64_t n_entries = n_keys;   // sorted entries of the pass (merge: + background lists)
    if (merge)
      for (int f = fs; f < fe; ++f) n_entries += (uint64_t)s->sb_K[(f0 + f) % s->sb_cams];
    // many lists beyond the small fused-sort capacity (e.g. 128x128 views): larger variant
    // (fixed plan: the small variant, whose long-list CTAs handle any length)
    const bool long_lists = !fixed && (uint64_t)n_vlong * 4 > (uint64_t)(fe - fs) * n_tiles;
    // split K4a + K4b unless the lists are short on average (then the one-CTA-per-tile kernel's
    // shared staging beats per-warp record reads; measured crossover ~200-330 keys per tile);
    // always split under the fixed plan
    const bool split = fixed || (split_k4() && n_entries >= split_min_avg() * (uint64_t)(fe - fs) * n_tiles &&
                                 n_entries <= (uint64_t)s->cap);
    if (fixed) a.overflow = s->d_overflow + 1 + sl;
    const bool slot_keys = !merge && slot_keys_on();
    if (slot_keys) a.ids = nullptr;   // key low word = index in the launch range = record slot
    // K4b block masks: plain split passes with slot keys (not scores: they reduce each record
    // over the whole warp) and the default K4a variants
    const bool want_masks = split && slot_keys && !(p->flags & GSB_FLAG_SCORES) && block_masks_on() &&
                            k4a_masks_supported() && count < ((int64_t)1 << (32 - kMaskBits)) &&
                            n_keys >= mask_min_avg() * (uint64_t)(fe - fs) * n_tiles;
    const bool masks = want_masks && s->trim_valid[sl];   // K2b needs K1's trims of this chunk
    masks_wanted |= want_masks;
    if (masks) { a.mask_bits = kMaskBits; a.trim = s->trim[sl]; }
    tm.begin(KC_EMIT, sb);
    launch_k2_emit(a, sb);
    if (count > 0) s->launches++;
    LAUNCH_CHECK();
    tm.end();
    // long lists are sorted by their K4 CTA (K3 serves gsb_debug_bin_sort)
    CompositeArgs c{};
    c.rec = s->rec[sl]; c.n = count; c.off = s->off[sl]; c.frame_base = s->frame_base[sl];
    c.hist_stride = s->hist_stride; c.sorted = sorted; c.keys = s->keys; c.keys_alt = s->keys_alt;
    c.key_base = key_base;
    c.inv = s->d_inv;
    c.slot_base = (int)first;
    if (merge) {
      c.bg_off = s->bg_off; c.bg_keys = s->bg_keys; c.bg_rec = s->bg_rec; c.n_static_cams = s->sb_cams;
      c.qpos_g = s->qpos;
      c.bg_cum = s->d_bgcum;
    }
    if (slot_keys) c.keys_internal_ids = s->d_ids + first;
    if (masks) c.key_shift = kMaskBits;
    c.long_list = s->long_list[sl];   // K4a: lists > kWarpSortCap get a CTA each
    c.n_long = n_long;
    if (fixed) {   // the long-list count and the chunk's overflow flag stay on the device
      c.n_long_dev = s->long_cnt[sl];
      c.overflow = s->d_overflow + 1 + sl;
    }
    c.fs = fs; c.fe = fe; c.f0 = f0; c.width = W; c.height = H; c.tiles_x = tiles_x; c.n_tiles = n_tiles;
    c.bg0 = p->background[0]; c.bg1 = p->background[1]; c.bg2 = p->background[2];
    c.out_rgb = out_rgb; c.out_depth = out_depth; c.out_alpha = out_alpha; c.out_n_eval = out_neval;
    c.stat_pairs = (p->flags & GSB_FLAG_STATS) ? s->d_pairs : nullptr;
    if (p->flags & GSB_FLAG_SCORES) {
      c.score_sum = s->d_wsum;
      c.score_max = s->d_wmax;
    }
    if (s->obs) {
      c.obs_rgb8 = s->obs_rgb8; c.obs_depth16 = s->obs_depth16; c.obs_dr = s->obs_dr;
      c.obs_seed = s->obs->seed; c.obs_step = s->obs->step;
      c.obs_frame_offset = s->obs->env_offset * (int64_t)n_cams;
    }
    // `sorted` buffer q was last read by the K4b of pass pass_idx - 2
    if (sb != sc && pass_idx >= 2) CUDA_TRY(cudaStreamWaitEvent(sb, s->ev_k4b[q], 0));
    cudaStream_t cs = sb;   // stream of this pass's last compositing kernel
    if (split) {
      tm.begin(KC_SORT, sb);
      launch_k4a_sort(c, long_lists && !merge, sb);   // K4a: tile sort (merge) -> ordered record slots
      s->launches++;
      LAUNCH_CHECK();
      tm.end();
      if (sb != sc) {
        CUDA_TRY(cudaEventRecord(s->ev_sorted[q], sb));
        CUDA_TRY(cudaStreamWaitEvent(sc, s->ev_sorted[q], 0));
      }
      cs = sc;
      tm.begin(KC_COMPOSITE, sc);
      launch_k4b_blend(c, s->d_counter, sc);   // K4b: persistent per-warp compositing
    } else {
      tm.begin(KC_COMPOSITE, sb);
      launch_k4_composite(c, long_lists, sb);
    }
    s->launches++;
    s->comp_launches++;
    LAUNCH_CHECK();
    tm.end();
    if (sb != sc) CUDA_TRY(cudaEventRecord(s->ev_k4b[q], cs));
    ++pass_idx;
    if (s->dl_rgb8) {  // host-io observations: uint8 RGB (+ fp16 or fp32 depth)
      CUDA_TRY(cudaEventRecord(s->ev_copy, cs));
      CUDA_TRY(cudaStreamWaitEvent(s->copy_stream, s->ev_copy, 0));
      const size_t plane = (size_t)W * H;
      const size_t a0 = (size_t)(f0 + fs), cnt = (size_t)(fe - fs);
      CUDA_TRY(cudaMemcpyAsync(s->dl_rgb8 + a0 * 3 * plane, s->obs_rgb8 + a0 * 3 * plane, cnt * 3 * plane,
                               cudaMemcpyDeviceToHost, s->copy_stream));
      if (s->dl_depth16)
        CUDA_TRY(cudaMemcpyAsync(s->dl_depth16 + a0 * plane, s->obs_depth16 + a0 * plane, cnt * plane * 2,
                                 cudaMemcpyDeviceToHost, s->copy_stream));
      if (s->dl_depth)
        CUDA_TRY(cudaMemcpyAsync(s->dl_depth + a0 * plane, out_depth + a0 * plane, cnt * plane * 4,
                                 cudaMemcpyDeviceToHost, s->copy_stream));
    } else if (s->dl_rgb) {  // host-io: download this pass's frames on the copy stream
      CUDA_TRY(cudaEventRecord(s->ev_copy, cs));
      CUDA_TRY(cudaStreamWaitEvent(s->copy_stream, s->ev_copy, 0));
      const size_t plane = (size_t)W * H;
      const size_t a0 = (size_t)(f0 + fs), cnt = (size_t)(fe - fs);
      CUDA_TRY(cudaMemcpyAsync(s->dl_rgb + a0 * 3 * plane, out_rgb + a0 * 3 * plane, cnt * 3 * plane * 4,
                               cudaMemcpyDeviceToHost, s->copy_stream));
      if (s->dl_depth)
        CUDA_TRY(cudaMemcpyAsync(s->dl_depth + a0 * plane, out_depth + a0 * plane, cnt * plane * 4,
                                 cudaMemcpyDeviceToHost, s->copy_stream));
      if (s->dl_alpha)
        CUDA_TRY(cudaMemcpyAsync(s->dl_alpha + a0 * plane, out_alpha + a0 * plane, cnt * plane * 4,
                                 cudaMemcpyDeviceToHost, s->copy_stream));
      if (s->dl_neval)
        CUDA_TRY(cudaMemcpyAsync(s->dl_neval + a0 * plane, out_neval + a0 * plane, cnt * plane * 4,
                                 cudaMemcpyDeviceToHost, s->copy_stream));
    }
    return GSB_OK;
  }

  gsb_status finish_chunk(int c, int f0, int nf) {
    const int sl = c & 1;
    gsb_status r;
    if (fixed) {   // one pass over the chunk, enqueued without reading its counts: binning waits
      s->chunks++;  // for the chunk's scan on the device (which also joins the projection stream)
      CUDA_TRY(cudaStreamWaitEvent(sb, s->ev_counts[sl], 0));
      r = pass(sl, f0, 0, nf, 0, 0, 0);
    } else {
      CUDA_TRY(cudaEventSynchronize(s->ev_counts[sl]));
      r = finish_passes(c, f0, nf);
    }
    if (r != GSB_OK) return r;
    if (sb != sc) {   // the chunk is done when both its binning and its compositing are
      CUDA_TRY(cudaEventRecord(s->ev_bin, sb));
      CUDA_TRY(cudaStreamWaitEvent(sc, s->ev_bin, 0));
    }
    CUDA_TRY(cudaEventRecord(s->ev_done[sl], sc));
    return GSB_OK;
  }

  gsb_status finish_passes(int c, int f0, int nf) {
    const int sl = c & 1;
    const volatile uint64_t* rb = s->h_rb[sl];
    uint64_t fb[kMaxChunk + 2];
    for (int i = 0; i < nf + 2; ++i) fb[i] = rb[i];
    for (int i = 0; i < nf; ++i) s->stat_V += (int64_t)rb[nf + 2 + i];
    s->stat_K += (int64_t)fb[nf];
    if (merge)  // the pre-binned background pairs of these frames
      for (int i = 0; i < nf; ++i) {
        const int cam = (f0 + i) % s->sb_cams;
        s->stat_V += s->sb_V[cam];
        s->stat_K += s->sb_K[cam];
      }
    s->chunks++;
    const uint32_t n_long = (uint32_t)rb[2 * nf + 2];    // lists > kWarpSortCap (K4a's long-list table)
    n_vlong = (uint32_t)rb[2 * nf + 3];                 // lists > kFusedSortCap (packed-variant rule)
    s->stat_long += n_long;
    s->stat_maxseg = std::max<int64_t>(s->stat_maxseg, (int64_t)fb[nf + 1]);
    if (fb[nf] <= (uint64_t)s->cap) return pass(sl, f0, 0, nf, 0, fb[nf], n_long);
    // split the chunk's frames into passes that fit the key workspace
    int fs = 0;
    while (fs < nf) {
      int fe = fs;
      while (fe < nf && fb[fe + 1] - fb[fs] <= (uint64_t)s->cap) ++fe;
      if (fe == fs)
        return fail(GSB_ERR_CAPACITY, "frame %d needs %llu tile keys > key capacity %lld", f0 + fs,
                    (unsigned long long)(fb[fs + 1] - fb[fs]), (long long)s->cap);
      gsb_status r = pass(sl, f0, fs, fe, fb[fs], fb[fe] - fb[fs], n_long);
      if (r != GSB_OK) return r;
      fs = fe;
    }
    return GSB_OK;
  }

  gsb_status run(const K0Rig& rig, int n_cams) {
    tm.begin(KC_SETUP, st);
    launch_k0(rig, F, n_cams, s->n_bodies, W, H, s->table, s->cams, st);
    s->launches++;
    LAUNCH_CHECK();
    tm.end();
    if (sp != st) {   // the internal streams start after everything the caller enqueued
      CUDA_TRY(cudaEventRecord(s->ev_start, st));
      CUDA_TRY(cudaStreamWaitEvent(sp, s->ev_start, 0));
      CUDA_TRY(cudaStreamWaitEvent(sc, s->ev_start, 0));
      if (sb != sc) CUDA_TRY(cudaStreamWaitEvent(sb, s->ev_start, 0));
    }
    gsb_status r = run_chunks();
    if (sp != st) {   // and the caller's stream continues after the last composite
      CUDA_TRY(cudaEventRecord(s->ev_end, sc));
      CUDA_TRY(cudaStreamWaitEvent(st, s->ev_end, 0));
    }
    return r;
  }

  gsb_status run_chunks() {
    const int E = (s->dl_rgb || s->dl_rgb8) ? s->chunk_host : s->chunk;   // host-io: smaller chunks
    const int nchunks = (F + E - 1) / E;
    for (int c = 0; c < nchunks; ++c) {
      const int f0 = c * E, nf = std::min(E, F - f0);
      gsb_status r = project_chunk(c, f0, nf);
      if (r != GSB_OK) return r;
      if (c > 0) {
        r = finish_chunk(c - 1, (c - 1) * E, E);
        if (r != GSB_OK) return r;
      }
    }
    if (nchunks > 0) {
      const int c = nchunks - 1;
      return finish_chunk(c, c * E, F - c * E);
    }
    return GSB_OK;
  }
};

K0Rig default_rig(gsb_scene s, const float* poses, const float* intr, const float* w2c) {
  K0Rig r{};
  r.poses = poses;
  r.env_stride = (int64_t)s->n_bodies * 7;
  r.body_stride = 7;
  r.intr = intr;
  r.cam_x = w2c;
  for (int c = 0; c < kMaxRigCams; ++c) r.cam_body[c] = -1;
  return r;
}

gsb_status render_impl(gsb_scene s, const K0Rig& rig, int n_envs, int n_cams, const gsb_render_params* p,
                       float* out_rgb, float* out_depth, float* out_alpha, int32_t* out_neval,
                       cudaStream_t st, bool merge) {
  const int F = n_envs * n_cams;
  s->last_stream = st;
  s->stat_V = s->stat_K = s->stat_long = s->stat_maxseg = 0;
  s->launches = s->comp_launches = s->chunks = 0;
  s->ev_used = 0;
  s->ev_marks.clear();
  const bool timing = (p->flags & GSB_FLAG_TIMING) != 0;
  const bool fixed = (p->flags & GSB_FLAG_FIXED_PLAN) != 0;
  if (fixed && (merge || s->dl_rgb || s->dl_rgb8 || (p->flags & (GSB_FLAG_STATS | GSB_FLAG_TIMING))))
    return fail(GSB_ERR_INVALID_ARGUMENT, "GSB_FLAG_FIXED_PLAN: not with STATS/TIMING, host-buffer or static renders");
  if (timing && s->ev_pool.empty()) {
    s->ev_pool.resize(8192);
    for (auto& e : s->ev_pool) CUDA_TRY(cudaEventCreate(&e));
  }
  if (p->flags & GSB_FLAG_STATS) CUDA_TRY(cudaMemsetAsync(s->d_pairs, 0, 2 * sizeof(unsigned long long), st));
  s->stat_pixels = (int64_t)F * p->width * p->height;
  Pipeline pl{};
  pl.s = s; pl.st = st; pl.p = p;
  pl.sp = pl.sc = pl.sb = st;
  if (two_streams() && s->sp && s->sc) {
    pl.sp = s->sp;
    pl.sc = pl.sb = s->sc;
    if (three_streams() && s->sb) pl.sb = s->sb;
  } pl.F = F; pl.W = p->width; pl.H = p->height;
  pl.tiles_x = (p->width + kTile - 1) / kTile;
  pl.n_tiles = pl.tiles_x * ((p->height + kTile - 1) / kTile);
  pl.D = p->sh_degree < 0 ? s->sh_degree : p->sh_degree;
  pl.tm = Timer{s, st, timing};
  pl.out_rgb = out_rgb; pl.out_depth = out_depth; pl.out_alpha = out_alpha; pl.out_neval = out_neval;
  pl.merge = merge;
  pl.fixed = fixed;
  pl.n_cams = n_cams;
  pl.first = merge ? s->n_bg : 0;      // static cameras: only the robot Gaussians per frame
  pl.count = s->n - pl.first;
  gsb_status r = pl.run(rig, n_cams);
  if (r == GSB_OK && !merge && F > 0) s->mask_hint = pl.masks_wanted;   // K1 trims for the next render
  s->stats_valid = (r == GSB_OK) && (p->flags & GSB_FLAG_STATS);
  s->timing_valid = (r == GSB_OK) && timing;
  return r;
}

}  // namespace gsb

extern "C" {

gsb_status gsb_render(gsb_scene s, const float* poses, int32_t n_envs, int32_t n_cams, const float* intr,
                      const float* w2c, const gsb_render_params* p, float* out_rgb, float* out_depth,
                      float* out_alpha, int32_t* out_neval, gsb_stream stream) {
  gsb_status r = validate_render(s, poses, n_envs, n_cams, intr, w2c, p, out_rgb);
  if (r != GSB_OK) return r;
  DeviceGuard g(s->device);
  s->dl_rgb = nullptr; s->dl_depth = nullptr; s->dl_alpha = nullptr; s->dl_neval = nullptr;
  return render_impl(s, default_rig(s, poses, intr, w2c), n_envs, n_cams, p, out_rgb, out_depth, out_alpha,
                     out_neval, (cudaStream_t)stream);
}

gsb_status gsb_render_rig(gsb_scene s, const float* poses, int64_t pose_env_stride, int64_t pose_body_stride,
                          int32_t n_envs, int32_t n_cams, const float* intr, const float* cam_extrinsics,
                          const int32_t* cam_body, const gsb_render_params* p, float* out_rgb,
                          float* out_depth, float* out_alpha, int32_t* out_neval, gsb_stream stream) {
  gsb_status r = validate_render(s, poses, n_envs, n_cams, intr, cam_extrinsics, p, out_rgb);
  if (r != GSB_OK) return r;
  K0Rig rig = default_rig(s, poses, intr, cam_extrinsics);
  if (pose_env_stride < 0 || pose_body_stride < 0)
    return fail(GSB_ERR_INVALID_ARGUMENT, "negative pose stride");
  if (pose_body_stride) {
    if (pose_body_stride < 7) return fail(GSB_ERR_INVALID_ARGUMENT, "pose_body_stride < 7");
    rig.body_stride = pose_body_stride;
  }
  if (pose_env_stride) rig.env_stride = pose_env_stride;
  else rig.env_stride = (int64_t)s->n_bodies * rig.body_stride;
  if (s->n_bodies > 0 && rig.env_stride < (int64_t)(s->n_bodies - 1) * rig.body_stride + 7 && n_envs > 1)
    return fail(GSB_ERR_INVALID_ARGUMENT, "pose_env_stride overlaps the bodies of an env");
  if (cam_body) {
    for (int c = 0; c < n_cams; ++c) {
      const int kb = cam_body[c];
      if (kb < -1 || kb >= s->n_bodies) return fail(GSB_ERR_UNKNOWN_BODY, "cam_body[%d] = %d not in [-1, %d)", c, kb, s->n_bodies);
      if (kb >= 0 && c >= kMaxRigCams) return fail(GSB_ERR_CAPACITY, "body-attached camera index %d >= %d", c, kMaxRigCams);
      if (kb >= 0 && !poses) return fail(GSB_ERR_INVALID_ARGUMENT, "body-attached camera without poses");
      if (c < kMaxRigCams) rig.cam_body[c] = kb;
    }
  }
  DeviceGuard g(s->device);
  s->dl_rgb = nullptr; s->dl_depth = nullptr; s->dl_alpha = nullptr; s->dl_neval = nullptr;
  return render_impl(s, rig, n_envs, n_cams, p, out_rgb, out_depth, out_alpha, out_neval, (cudaStream_t)stream);
}

gsb_status gsb_render_host(gsb_scene s, const float* poses, int32_t n_envs, int32_t n_cams,
                           const float* intr, const float* w2c, const gsb_render_params* p,
                           float* out_rgb, float* out_depth, float* out_alpha, int32_t* out_neval,
                           gsb_stream stream) {
  gsb_status r = validate_render(s, poses, n_envs, n_cams, intr, w2c, p, out_rgb);
  if (r != GSB_OK) return r;
  if (!s->host_io) return fail(GSB_ERR_INVALID_ARGUMENT, "reserve with GSB_RESERVE_HOST_IO for gsb_render_host");
  if (n_envs > s->max_envs) return fail(GSB_ERR_SHAPE_MISMATCH, "n_envs beyond the host-io reservation");
  DeviceGuard g(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t F = (size_t)n_envs * n_cams;
  if (s->n_bodies > 0 && n_envs > 0)
    CUDA_TRY(cudaMemcpyAsync(s->st_poses, poses, sizeof(float) * (size_t)n_envs * s->n_bodies * 7, cudaMemcpyHostToDevice, st));
  if (F > 0) {
    CUDA_TRY(cudaMemcpyAsync(s->st_intr, intr, sizeof(float) * F * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(s->st_w2c, w2c, sizeof(float) * F * 12, cudaMemcpyHostToDevice, st));
  }
  s->dl_rgb = out_rgb; s->dl_depth = out_depth; s->dl_alpha = out_alpha; s->dl_neval = out_neval;
  r = render_impl(s, default_rig(s, s->st_poses, s->st_intr, s->st_w2c), n_envs, n_cams, p, s->st_rgb,
                  out_depth ? s->st_depth : nullptr, out_alpha ? s->st_alpha : nullptr,
                  out_neval ? s->st_neval : nullptr, st);
  s->dl_rgb = nullptr; s->dl_depth = nullptr; s->dl_alpha = nullptr; s->dl_neval = nullptr;
  if (r != GSB_OK) return r;
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaStreamSynchronize(s->copy_stream));
  return GSB_OK;
}

namespace {
struct ObsScope {  // the observation epilogue of one render call; cleared on exit
  gsb_scene s;
  ObsScope(gsb_scene s_, const gsb_obs_params* o, uint8_t* rgb8, uint16_t* d16, const float* dr) : s(s_) {
    s->obs = o; s->obs_rgb8 = rgb8; s->obs_depth16 = d16; s->obs_dr = dr;
  }
  ~ObsScope() {
    s->obs = nullptr; s->obs_rgb8 = nullptr; s->obs_depth16 = nullptr; s->obs_dr = nullptr;
    s->dl_rgb = nullptr; s->dl_depth = nullptr; s->dl_alpha = nullptr; s->dl_neval = nullptr;
    s->dl_rgb8 = nullptr; s->dl_depth16 = nullptr;
  }
};

gsb_status validate_obs(const gsb_obs_params* o, const void* out_rgb8) {
  if (!o) return fail(GSB_ERR_INVALID_ARGUMENT, "obs params are NULL");
  if (!out_rgb8) return fail(GSB_ERR_INVALID_ARGUMENT, "out_rgb8 is NULL");
  if (o->env_offset < 0) return fail(GSB_ERR_INVALID_ARGUMENT, "negative env_offset");
  if (o->flags & ~GSB_OBS_DEPTH_F16) return fail(GSB_ERR_INVALID_ARGUMENT, "unknown obs flags 0x%x", o->flags);
  return GSB_OK;
}
}  // namespace

gsb_status gsb_render_obs(gsb_scene s, const float* poses, int32_t n_envs, int32_t n_cams, const float* intr,
                          const float* w2c, const gsb_render_params* p, const gsb_obs_params* obs,
                          uint8_t* out_rgb8, void* out_depth, gsb_stream stream) {
  gsb_status r = validate_render(s, poses, n_envs, n_cams, intr, w2c, p, (const float*)out_rgb8);
  if (r != GSB_OK) return r;
  r = validate_obs(obs, out_rgb8);
  if (r != GSB_OK) return r;
  DeviceGuard g(s->device);
  const bool f16 = (obs->flags & GSB_OBS_DEPTH_F16) != 0;
  ObsScope os(s, obs, out_rgb8, f16 ? (uint16_t*)out_depth : nullptr, obs->image_dr);
  return render_impl(s, default_rig(s, poses, intr, w2c), n_envs, n_cams, p, nullptr,
                     f16 ? nullptr : (float*)out_depth, nullptr, nullptr, (cudaStream_t)stream);
}

gsb_status gsb_obs_encode(const float* rgb, const float* depth, int32_t n_envs, int32_t n_cams, int32_t width,
                          int32_t height, const gsb_obs_params* obs, const int32_t* blur, uint8_t* out_rgb8,
                          void* out_depth, gsb_stream stream) {
  gsb_status r = validate_obs(obs, out_rgb8);
  if (r != GSB_OK) return r;
  if (n_envs < 0 || n_cams < 1 || width < 1 || height < 1 || width > kMaxDim || height > kMaxDim)
    return fail(GSB_ERR_INVALID_ARGUMENT, "bad frame shape (%d envs, %d cams, %dx%d)", n_envs, n_cams, width, height);
  const int64_t F = (int64_t)n_envs * n_cams;
  if (F == 0) return GSB_OK;
  if (F > 65535) return fail(GSB_ERR_CAPACITY, "%lld frames > 65535 per call", (long long)F);
  if (!rgb) return fail(GSB_ERR_INVALID_ARGUMENT, "rgb is NULL");
  EncodeArgs a{};
  a.rgb = rgb; a.depth = depth; a.blur = blur; a.dr = obs->image_dr; a.seed = obs->seed; a.step = obs->step;
  a.frame_offset = obs->env_offset * n_cams; a.n_frames = (int)F; a.width = width; a.height = height;
  a.out_rgb8 = out_rgb8;
  const bool f16 = (obs->flags & GSB_OBS_DEPTH_F16) != 0;
  a.out_depth16 = (depth && f16) ? (uint16_t*)out_depth : nullptr;
  a.out_depth32 = (depth && !f16) ? (float*)out_depth : nullptr;
  launch_k6_encode(a, (cudaStream_t)stream);
  LAUNCH_CHECK();
  return GSB_OK;
}

gsb_status gsb_render_obs_host(gsb_scene s, const float* poses, int32_t n_envs, int32_t n_cams, const float* intr,
                               const float* w2c, const gsb_render_params* p, const gsb_obs_params* obs,
                               uint8_t* out_rgb8, void* out_depth, gsb_stream stream) {
  gsb_status r = validate_render(s, poses, n_envs, n_cams, intr, w2c, p, (const float*)out_rgb8);
  if (r != GSB_OK) return r;
  r = validate_obs(obs, out_rgb8);
  if (r != GSB_OK) return r;
  if (!s->host_io) return fail(GSB_ERR_INVALID_ARGUMENT, "reserve with GSB_RESERVE_HOST_IO for gsb_render_obs_host");
  if (n_envs > s->max_envs) return fail(GSB_ERR_SHAPE_MISMATCH, "n_envs beyond the host-io reservation");
  DeviceGuard g(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t F = (size_t)n_envs * n_cams;
  if (s->n_bodies > 0 && n_envs > 0)
    CUDA_TRY(cudaMemcpyAsync(s->st_poses, poses, sizeof(float) * (size_t)n_envs * s->n_bodies * 7, cudaMemcpyHostToDevice, st));
  if (F > 0) {
    CUDA_TRY(cudaMemcpyAsync(s->st_intr, intr, sizeof(float) * F * 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(s->st_w2c, w2c, sizeof(float) * F * 12, cudaMemcpyHostToDevice, st));
    if (obs->image_dr) CUDA_TRY(cudaMemcpyAsync(s->st_dr, obs->image_dr, sizeof(float) * F * 4, cudaMemcpyHostToDevice, st));
  }
  const bool f16 = (obs->flags & GSB_OBS_DEPTH_F16) != 0;
  // staging: uint8 RGB in st_rgb, fp16 depth in st_depth (both smaller than their fp32 sizes)
  ObsScope os(s, obs, (uint8_t*)s->st_rgb, f16 ? (uint16_t*)s->st_depth : nullptr, obs->image_dr ? s->st_dr : nullptr);
  s->dl_rgb8 = out_rgb8;
  if (out_depth) {
    if (f16) s->dl_depth16 = (uint16_t*)out_depth;
    else s->dl_depth = (float*)out_depth;
  }
  r = render_impl(s, default_rig(s, s->st_poses, s->st_intr, s->st_w2c), n_envs, n_cams, p, nullptr,
                  (out_depth && !f16) ? s->st_depth : nullptr, nullptr, nullptr, st);
  if (r != GSB_OK) return r;
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaStreamSynchronize(s->copy_stream));
  return GSB_OK;
}

}  // extern "C"
