// gsb_runtime.cuh — internal header of the libgsb host runtime (not part of the C ABI).
//
// Shared by the host translation units:
//   gsb_api.cu         scene template (K5) create / reserve / destroy, stats, timings, scores, filter
//   gsb_render.cu      the chunked render pipeline (K0 -> K1 -> K2 -> K4) and its entry points
//                      (gsb_render, gsb_render_rig, gsb_render_host, observation renders, K6 encode)
//   gsb_static.cu      static-camera background pre-binning (§8(f) row 2)
//   gsb_lidar_host.cu  batched ray-cast LiDAR (§8(f) row 4, reading R32)
//   gsb_debug.cu       test-only hooks (dense K1 records, binning + production tile sorts)
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gsb.h"
#include "gsb_common.cuh"
#include "gsb_kernels.cuh"

namespace gsb {

// records the message returned by gsb_last_error (thread-local) and returns s
gsb_status fail(gsb_status s, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? GSB_ERR_OUT_OF_MEMORY : GSB_ERR_CUDA, \
                  "%s failed: %s", #expr, cudaGetErrorString(e_));                      \
  } while (0)

#define LAUNCH_CHECK()                                                                   \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess) return fail(GSB_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e_)); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

template <typename T>
inline cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return cudaSuccess;
  return cudaMalloc((void**)p, count * sizeof(T));
}

enum KClass { KC_SETUP = 0, KC_PROJECT, KC_SCAN, KC_EMIT, KC_SORT, KC_COMPOSITE, KC_N };

constexpr int kMaxChunk = 1024;  // frames per pipeline chunk (upper bound)

// compositing path of plain / observation renders: split K4a + K4b (default) or the
// one-CTA-per-tile K4 (GSB_K4=fused, for A/B comparisons)
inline bool split_k4() {
  static const int v = [] {
    const char* e = getenv("GSB_K4");
    return (e && std::string(e) == "fused") ? 0 : 1;
  }();
  return v != 0;
}
// pass-average list length (keys per tile) from which the split path is used; GSB_K4_SPLIT_MIN
// overrides it (read per pass: tests force either path).  Since round 2's K4a and K2b the split
// path wins at every measured list length (C2 +15 %, C7 +18 %), so the default is 0: the fused
// one-CTA-per-tile K4 runs only when forced (tests, A/B)
inline uint64_t split_min_avg() {
  const char* e = getenv("GSB_K4_SPLIT_MIN");
  return e ? (uint64_t)strtoull(e, nullptr, 10) : 0u;
}

inline bool block_masks_on() {   // GSB_BLOCK_MASKS=0: K4b culls every staged record itself (A/B)
  const char* e = getenv("GSB_BLOCK_MASKS");
  return !(e && e[0] == '0');
}

// block masks pay where lists are long (C4 +5.4 %, C5 +3.1 %) and lose where they are short and the
// Gaussians large (C2 -7 %: the masks are bounding-box trims, looser than K4b's elliptic cull; C3
// +0.3 %): used for passes averaging at least this many keys per tile (GSB_MASK_MIN_AVG)
inline uint64_t mask_min_avg() {
  const char* e = getenv("GSB_MASK_MIN_AVG");
  return e ? (uint64_t)strtoull(e, nullptr, 10) : 512u;
}

inline bool slot_keys_on() {   // GSB_SLOT_KEYS=0: keys carry the creation id on every path
  const char* e = getenv("GSB_SLOT_KEYS");
  return !(e && e[0] == '0');
}

inline bool two_streams() {   // GSB_STREAMS=1: everything on the caller's stream (A/B comparisons)
  static const bool v = [] {
    const char* e = getenv("GSB_STREAMS");
    return !(e && e[0] == '1');
  }();
  return v;
}
inline bool three_streams() {   // GSB_STREAMS=2: binning/sort on the compositing stream
  static const bool v = [] {
    const char* e = getenv("GSB_STREAMS");
    return !(e && (e[0] == '1' || e[0] == '2'));
  }();
  return v;
}

}  // namespace gsb

struct gsb_scene_t {
  int device = 0;
  int64_t n = 0;
  int64_t n_bg = 0;   // static Gaussians (body -1): the prefix [0, n_bg) of the internal order
  int n_bodies = 0;
  int sh_degree = 0;
  int sh_planes = 1;
  // template (K5)
  float4 *d_mean = nullptr, *d_L0 = nullptr, *d_L1 = nullptr, *d_L2 = nullptr, *d_sh = nullptr;
  int2* d_ids = nullptr;  // internal (Morton) index -> (creation index = id of reading R10, body)
  int* d_inv = nullptr;   // id -> internal index
  float* d_wsum = nullptr;     // pruning scores (reading R30), by internal index
  uint32_t* d_wmax = nullptr;  // float bits
  // reservation
  bool reserved = false;
  int max_frames = 0, res_w = 0, res_h = 0, chunk = 0;
  int chunk_host = 0;   // frames per chunk of host-buffer renders (<= chunk)
  int tiles_x = 0, tiles_y = 0, n_tiles = 0;
  int64_t hist_stride = 0;
  int64_t cap = 0;
  float4* table = nullptr;
  gsb::FrameCam* cams = nullptr;
  float4* rec[2] = {nullptr, nullptr};
  uint2* emit[2] = {nullptr, nullptr};
  uint8_t* trim[2] = {nullptr, nullptr};   // [E][N] K4b block-mask trims of the visible pairs (K1 -> K2b)
  bool trim_valid[2] = {false, false};     // K1 wrote the trims of the chunk in this slot
  bool mask_hint = true;                   // a pass of the last render wanted block masks: K1 writes trims
  int* vcount[2] = {nullptr, nullptr};
  uint32_t* vis_bits[2] = {nullptr, nullptr};
  uint32_t* long_list[2] = {nullptr, nullptr};   // lists too long for K4's fused sort
  uint32_t* long_cnt[2] = {nullptr, nullptr};
  int64_t vis_words = 0;
  int* hist[2] = {nullptr, nullptr};
  uint32_t* off[2] = {nullptr, nullptr};
  uint64_t* frame_base[2] = {nullptr, nullptr};
  uint64_t* h_rb[2] = {nullptr, nullptr};   // mapped pinned readback: fb[E+2], vcount[E], n_long
  uint64_t* d_rb[2] = {nullptr, nullptr};   // its device view
  cudaEvent_t ev_counts[2] = {nullptr, nullptr};
  // two internal streams: projection (K1, K2a) runs one chunk ahead of binning + compositing
  // (K2b, K4a, K4b), so the latency-bound kernels of one overlap the other's
  cudaStream_t sp = nullptr, sc = nullptr;
  cudaEvent_t ev_done[2] = {nullptr, nullptr};   // chunk slot free again (its compositing done)
  // third stream: binning + tile sort (K2b, K4a, fused K4) of pass q overlaps K4b of pass q-1;
  // `sorted` is double-buffered by pass parity
  cudaStream_t sb = nullptr;
  uint32_t* sorted2 = nullptr;
  cudaEvent_t ev_sorted[2] = {nullptr, nullptr};  // K4a of the pass with this parity done
  cudaEvent_t ev_k4b[2] = {nullptr, nullptr};     // K4b of the pass with this parity done
  cudaEvent_t ev_bin = nullptr;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr;
  uint64_t *keys = nullptr, *keys_alt = nullptr;
  uint32_t* sorted = nullptr;
  unsigned long long* d_pairs = nullptr;
  int* d_overflow = nullptr;   // GSB_FLAG_FIXED_PLAN: [0] sticky flag, [1..2] per chunk slot
  int* d_counter = nullptr;   // K4b work-item counter
  // host-io staging
  bool host_io = false;
  int max_envs = 0, res_cams = 0;
  float *st_poses = nullptr, *st_intr = nullptr, *st_w2c = nullptr;
  float *st_rgb = nullptr, *st_depth = nullptr, *st_alpha = nullptr;
  int32_t* st_neval = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy = nullptr;
  // last-render bookkeeping
  cudaStream_t last_stream = nullptr;
  bool stats_valid = false;
  int64_t stat_V = 0, stat_K = 0, stat_long = 0, stat_maxseg = 0, stat_pixels = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> ev_marks;  // (class, index of begin event)
  bool timing_valid = false;
  int64_t launches = 0, comp_launches = 0, chunks = 0;
  // static-camera pre-binning (gsb_prebin_static, §8(f) row 2)
  int sb_cams = 0, sb_w = 0, sb_h = 0, sb_D = 0;
  float sb_near = 0.f, sb_far = 0.f;
  float *sb_intr = nullptr, *sb_w2c = nullptr;   // [C][4], [C][12]
  uint64_t* bg_off = nullptr;                     // [C][T+1]
  uint64_t* bg_keys = nullptr;                    // [K_bg]
  float4* bg_rec = nullptr;                       // [K_bg][3]
  std::vector<int64_t> sb_V, sb_K;                // per camera
  uint64_t* d_bgcum = nullptr;                    // [C+1] prefix of sb_K (split K4 merge)
  uint32_t* qpos = nullptr;                       // [cap] (workspace, while pre-binned)
  void free_prebin() {
    cudaFree(sb_intr); cudaFree(sb_w2c); cudaFree(bg_off); cudaFree(bg_keys); cudaFree(bg_rec); cudaFree(d_bgcum);
    sb_intr = sb_w2c = nullptr; bg_off = bg_keys = nullptr; bg_rec = nullptr; d_bgcum = nullptr;
    sb_cams = 0; sb_V.clear(); sb_K.clear();
  }
  // host-io: where to download outputs of each pass
  float *dl_rgb = nullptr, *dl_depth = nullptr, *dl_alpha = nullptr;
  int32_t* dl_neval = nullptr;
  uint8_t* dl_rgb8 = nullptr;
  uint16_t* dl_depth16 = nullptr;
  // observation epilogue of the current render (gsb_render_obs*), nullptr otherwise
  const gsb_obs_params* obs = nullptr;
  uint8_t* obs_rgb8 = nullptr;
  uint16_t* obs_depth16 = nullptr;
  const float* obs_dr = nullptr;
  float* st_dr = nullptr;  // host-io staging of the DR parameters

  void free_workspace() {
    cudaFree(table); cudaFree(cams);
    for (int s = 0; s < 2; ++s) {
      cudaFree(rec[s]); cudaFree(emit[s]); emit[s] = nullptr; cudaFree(trim[s]); trim[s] = nullptr; cudaFree(vcount[s]); cudaFree(hist[s]); cudaFree(off[s]); cudaFree(vis_bits[s]);
      cudaFree(long_list[s]); cudaFree(long_cnt[s]);
      vis_bits[s] = nullptr; long_list[s] = nullptr; long_cnt[s] = nullptr;
      cudaFree(frame_base[s]);
      if (h_rb[s]) cudaFreeHost(h_rb[s]);
      if (ev_counts[s]) cudaEventDestroy(ev_counts[s]);
      rec[s] = nullptr; vcount[s] = nullptr; hist[s] = nullptr; off[s] = nullptr;
      frame_base[s] = nullptr; h_rb[s] = nullptr; d_rb[s] = nullptr; ev_counts[s] = nullptr;
    }
    cudaFree(keys); cudaFree(keys_alt); cudaFree(sorted); cudaFree(d_pairs); cudaFree(qpos); cudaFree(d_counter);
    cudaFree(d_overflow);
    d_overflow = nullptr;
    d_counter = nullptr;
    qpos = nullptr;
    cudaFree(st_poses); cudaFree(st_intr); cudaFree(st_w2c);
    cudaFree(st_rgb); cudaFree(st_depth); cudaFree(st_alpha); cudaFree(st_neval); cudaFree(st_dr);
    st_dr = nullptr;
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (sp) cudaStreamDestroy(sp);
    if (sc) cudaStreamDestroy(sc);
    if (sb) cudaStreamDestroy(sb);
    sb = nullptr;
    cudaFree(sorted2);
    sorted2 = nullptr;
    for (auto& e : ev_sorted) { if (e) cudaEventDestroy(e); e = nullptr; }
    for (auto& e : ev_k4b) { if (e) cudaEventDestroy(e); e = nullptr; }
    if (ev_bin) cudaEventDestroy(ev_bin);
    ev_bin = nullptr;
    for (auto& e : ev_done) { if (e) cudaEventDestroy(e); e = nullptr; }
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_end) cudaEventDestroy(ev_end);
    sp = sc = nullptr; ev_start = ev_end = nullptr;
    if (ev_copy) cudaEventDestroy(ev_copy);
    for (auto e : ev_pool) cudaEventDestroy(e);
    ev_pool.clear();
    table = nullptr; cams = nullptr; keys = keys_alt = nullptr; sorted = nullptr; d_pairs = nullptr;
    st_poses = st_intr = st_w2c = st_rgb = st_depth = st_alpha = nullptr; st_neval = nullptr;
    copy_stream = nullptr; ev_copy = nullptr;
    reserved = false;
  }
};

namespace gsb {

inline bool finite_all(const float* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

// GSB_ERR_DEVICE unless `device` is an sm_100 GPU
gsb_status check_device(int device);

// timing helpers
struct Timer {
  gsb_scene_t* s;
  cudaStream_t st;
  bool on;
  size_t begin_idx = 0;
  int cls = 0;
  cudaStream_t cur = nullptr;
  void begin(int c, cudaStream_t on_stream) {
    if (!on) return;
    if (s->ev_used + 2 > s->ev_pool.size()) { on = false; return; }
    cls = c;
    cur = on_stream;
    begin_idx = s->ev_used;
    cudaEventRecord(s->ev_pool[s->ev_used++], cur);
  }
  void end() {
    if (!on) return;
    cudaEventRecord(s->ev_pool[s->ev_used++], cur);
    s->ev_marks.push_back({cls, begin_idx});
  }
};

// host-side validation shared by every camera render entry point (nothing is enqueued on failure)
gsb_status validate_render(gsb_scene s, const float* poses, int n_envs, int n_cams, const float* intr,
                           const float* w2c, const gsb_render_params* p, const float* out_rgb);

// K0 inputs of a plain render: poses [B][n_b][7], world cameras [B][C]
K0Rig default_rig(gsb_scene s, const float* poses, const float* intr, const float* w2c);

// the chunked pipeline of gsb_render_t* (gsb_render.cu); merge = static-camera pre-binned lists
gsb_status render_impl(gsb_scene s, const K0Rig& rig, int n_envs, int n_cams, const gsb_render_params* p,
                       float* out_rgb, float* out_depth, float* out_alpha, int32_t* out_neval,
                       cudaStream_t st, bool merge = false);

}  // namespace gsb
