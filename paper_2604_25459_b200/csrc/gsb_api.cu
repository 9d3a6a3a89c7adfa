// gsb_api.cu — libgsb host runtime: the C ABI of include/gsb.h.
//
// Owns the scene template (K5: one read-only copy shared by every env), the reserved
// workspace, and the chunked render pipeline:
//
//   K0 setup (all frames) ;  for each chunk c of E frames (double-buffered slot c&1):
//     K1 project(c) -> records + tile histogram ; K2a scan(c) ; D2H frame key counts (event)
//     [host waits for chunk c-1's counts — the GPU is busy with chunk c meanwhile]
//     K2b emit(c-1) ; K3 sort(c-1) ; K4 composite(c-1)   (split by frames if keys > capacity)
//
// No allocation happens in gsb_render; all buffers are sized by gsb_reserve.
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

using namespace gsb;

namespace {

thread_local std::string g_err = "no error";

gsb_status fail(gsb_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

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
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return cudaSuccess;
  return cudaMalloc((void**)p, count * sizeof(T));
}

enum KClass { KC_SETUP = 0, KC_PROJECT, KC_SCAN, KC_EMIT, KC_SORT, KC_COMPOSITE, KC_N };

constexpr int kMaxChunk = 1024;  // frames per pipeline chunk (upper bound)

// compositing path of plain / observation renders: split K4a + K4b (default) or the
// one-CTA-per-tile K4 (GSB_K4=fused, for A/B comparisons)
bool split_k4() {
  static const int v = [] {
    const char* e = getenv("GSB_K4");
    return (e && std::string(e) == "fused") ? 0 : 1;
  }();
  return v != 0;
}
// pass-average list length (keys per tile) from which the split path is used; GSB_K4_SPLIT_MIN
// overrides it (read per pass: tests force either path)
uint64_t split_min_avg() {
  const char* e = getenv("GSB_K4_SPLIT_MIN");
  return e ? (uint64_t)strtoull(e, nullptr, 10) : 200u;
}

bool slot_keys_on() {   // GSB_SLOT_KEYS=0: keys carry the creation id on every path
  const char* e = getenv("GSB_SLOT_KEYS");
  return !(e && e[0] == '0');
}

bool two_streams() {   // GSB_STREAMS=1: everything on the caller's stream (A/B comparisons)
  static const bool v = [] {
    const char* e = getenv("GSB_STREAMS");
    return !(e && e[0] == '1');
  }();
  return v;
}
bool three_streams() {   // GSB_STREAMS=2: binning/sort on the compositing stream
  static const bool v = [] {
    const char* e = getenv("GSB_STREAMS");
    return !(e && (e[0] == '1' || e[0] == '2'));
  }();
  return v;
}  // keys per tile (pass average) for the split path

}  // namespace

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
  int tiles_x = 0, tiles_y = 0, n_tiles = 0;
  int64_t hist_stride = 0;
  int64_t cap = 0;
  float4* table = nullptr;
  FrameCam* cams = nullptr;
  float4* rec[2] = {nullptr, nullptr};
  uint2* emit[2] = {nullptr, nullptr};
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
  int64_t stat_V = 0, stat_K = 0, stat_long = 0, stat_maxseg = 0;
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
      cudaFree(rec[s]); cudaFree(emit[s]); emit[s] = nullptr; cudaFree(vcount[s]); cudaFree(hist[s]); cudaFree(off[s]); cudaFree(vis_bits[s]);
      cudaFree(long_list[s]); cudaFree(long_cnt[s]);
      vis_bits[s] = nullptr; long_list[s] = nullptr; long_cnt[s] = nullptr;
      cudaFree(frame_base[s]);
      if (h_rb[s]) cudaFreeHost(h_rb[s]);
      if (ev_counts[s]) cudaEventDestroy(ev_counts[s]);
      rec[s] = nullptr; vcount[s] = nullptr; hist[s] = nullptr; off[s] = nullptr;
      frame_base[s] = nullptr; h_rb[s] = nullptr; d_rb[s] = nullptr; ev_counts[s] = nullptr;
    }
    cudaFree(keys); cudaFree(keys_alt); cudaFree(sorted); cudaFree(d_pairs); cudaFree(qpos); cudaFree(d_counter);
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

namespace {

bool finite_all(const float* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

gsb_status check_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(GSB_ERR_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= count) return fail(GSB_ERR_INVALID_ARGUMENT, "device %d out of range", device);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(GSB_ERR_DEVICE, "device %d is sm_%d%d, libgsb needs sm_100", device, prop.major, prop.minor);
  return GSB_OK;
}

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

  gsb_status project_chunk(int c, int f0, int nf) {
    const int sl = c & 1;
    if (c >= 2) CUDA_TRY(cudaStreamWaitEvent(sp, s->ev_done[sl], 0));   // chunk c-2 left this slot
    CUDA_TRY(cudaMemsetAsync(s->vcount[sl], 0, sizeof(int) * nf, sp));
    CUDA_TRY(cudaMemsetAsync(s->long_cnt[sl], 0, sizeof(uint32_t), sp));
    CUDA_TRY(cudaMemsetAsync(s->hist[sl], 0, sizeof(int) * s->hist_stride * nf, sp));
    K1Args a{};
    a.g_mean = s->d_mean + first; a.g_L0 = s->d_L0 + first; a.g_L1 = s->d_L1 + first;
    a.g_L2 = s->d_L2 + first; a.g_sh = s->d_sh + first;
    a.g_ids = s->d_ids + first;
    a.n = count; a.sh_stride = s->n; a.table = s->table; a.cams = s->cams; a.nb1 = s->n_bodies + 1;
    a.f0 = f0; a.n_frames = nf; a.width = W; a.height = H; a.tiles_x = tiles_x;
    a.near_plane = p->near_plane; a.far_plane = p->far_plane;
    a.rec = s->rec[sl]; a.emit = s->emit[sl];
    a.vcount = s->vcount[sl]; a.hist = s->hist[sl]; a.hist_stride = s->hist_stride;
    a.vis_bits = s->vis_bits[sl]; a.vis_words = s->vis_words;
    tm.begin(KC_PROJECT, sp);
    launch_k1(a, D, sp);
    if (count > 0) s->launches++;
    LAUNCH_CHECK();
    tm.end();
    tm.begin(KC_SCAN, sp);
    launch_k2_scan(s->hist[sl], s->off[sl], s->hist_stride, nf, n_tiles, s->frame_base[sl], s->long_list[sl],
                   s->long_cnt[sl], kFusedSortCap, s->vcount[sl], s->d_rb[sl], sp);
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
    const bool long_lists = (uint64_t)n_long * 4 > (uint64_t)(fe - fs) * n_tiles;
    // split K4a + K4b unless the lists are short on average (then the one-CTA-per-tile kernel's
    // shared staging beats per-warp record reads; measured crossover ~200-330 keys per tile)
    const bool split = split_k4() && n_entries >= split_min_avg() * (uint64_t)(fe - fs) * n_tiles &&
                       n_entries <= (uint64_t)s->cap;
    const bool slot_keys = !merge && slot_keys_on();
    if (slot_keys) a.ids = nullptr;   // key low word = index in the launch range = record slot
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
    CUDA_TRY(cudaEventSynchronize(s->ev_counts[sl]));
    gsb_status r = finish_passes(c, f0, nf);
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
    const uint32_t n_long = (uint32_t)rb[2 * nf + 2];
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
    const int E = s->chunk;
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
                       cudaStream_t st, bool merge = false) {
  const int F = n_envs * n_cams;
  s->last_stream = st;
  s->stat_V = s->stat_K = s->stat_long = s->stat_maxseg = 0;
  s->launches = s->comp_launches = s->chunks = 0;
  s->ev_used = 0;
  s->ev_marks.clear();
  const bool timing = (p->flags & GSB_FLAG_TIMING) != 0;
  if (timing && s->ev_pool.empty()) {
    s->ev_pool.resize(8192);
    for (auto& e : s->ev_pool) CUDA_TRY(cudaEventCreate(&e));
  }
  if (p->flags & GSB_FLAG_STATS) CUDA_TRY(cudaMemsetAsync(s->d_pairs, 0, sizeof(unsigned long long), st));
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
  pl.n_cams = n_cams;
  pl.first = merge ? s->n_bg : 0;      // static cameras: only the robot Gaussians per frame
  pl.count = s->n - pl.first;
  gsb_status r = pl.run(rig, n_cams);
  s->stats_valid = (r == GSB_OK) && (p->flags & GSB_FLAG_STATS);
  s->timing_valid = (r == GSB_OK) && timing;
  return r;
}

}  // namespace

extern "C" {

const char* gsb_last_error(void) { return g_err.c_str(); }

const char* gsb_version(void) { return "gsb 0.1 sm_100a"; }

gsb_status gsb_create_scene(const float* means, const float* scales, const float* quats,
                            const float* opacities, const float* sh, int32_t sh_degree,
                            const int32_t* body_id, int64_t n, int32_t n_bodies, int32_t device,
                            gsb_scene* out) {
  if (!out) return fail(GSB_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n < 0) return fail(GSB_ERR_INVALID_ARGUMENT, "n_gaussians < 0");
  if (n >= (int64_t)1 << 31) return fail(GSB_ERR_CAPACITY, "n_gaussians >= 2^31");
  if (sh_degree < 0 || sh_degree > 3) return fail(GSB_ERR_INVALID_ARGUMENT, "sh_degree %d not in 0..3", sh_degree);
  if (n_bodies < 0) return fail(GSB_ERR_INVALID_ARGUMENT, "n_bodies < 0");
  if (n > 0 && (!means || !scales || !quats || !opacities || !sh || !body_id))
    return fail(GSB_ERR_INVALID_ARGUMENT, "NULL template pointer");
  const int nc = (sh_degree + 1) * (sh_degree + 1);
  if (!finite_all(means, 3 * n) || !finite_all(scales, 3 * n) || !finite_all(quats, 4 * n) ||
      !finite_all(opacities, n) || !finite_all(sh, 3 * nc * n))
    return fail(GSB_ERR_INVALID_ARGUMENT, "non-finite template value");
  gsb_status st = check_device(device);
  if (st != GSB_OK) return st;
  const int np = (3 * nc + 3) / 4;
  for (int64_t i = 0; i < n; ++i) {
    const int b = body_id[i];
    if (b < -1 || b >= n_bodies) return fail(GSB_ERR_UNKNOWN_BODY, "body_id[%lld] = %d not in [-1, %d)", (long long)i, b, n_bodies);
  }
  // Internal order (K5 layout): grouped by body, then Morton (Z-order) of the template position,
  // so a warp's 32 Gaussians are spatial neighbours: uniform visibility per warp and few
  // distinct tiles per warp (aggregated atomics).  Results are independent of this order:
  // ordering and tie-breaks use (z, creation index) only (reading R10).
  std::vector<int64_t> perm(n);
  {
    std::vector<double> lo(3 * (n_bodies + 1), 1e300), hi(3 * (n_bodies + 1), -1e300);
    for (int64_t i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) {
        const int g = body_id[i] + 1;
        lo[3 * g + c] = std::min(lo[3 * g + c], (double)means[3 * i + c]);
        hi[3 * g + c] = std::max(hi[3 * g + c], (double)means[3 * i + c]);
      }
    auto spread = [](uint64_t x) {
      x &= 0x1fffff;
      x = (x | x << 32) & 0x1f00000000ffffull;
      x = (x | x << 16) & 0x1f0000ff0000ffull;
      x = (x | x << 8) & 0x100f00f00f00f00full;
      x = (x | x << 4) & 0x10c30c30c30c30c3ull;
      x = (x | x << 2) & 0x1249249249249249ull;
      return x;
    };
    std::vector<std::pair<std::pair<int, uint64_t>, int64_t>> key(n);
    for (int64_t i = 0; i < n; ++i) {
      const int g = body_id[i] + 1;
      uint64_t code = 0;
      for (int c = 0; c < 3; ++c) {
        const double ext = hi[3 * g + c] - lo[3 * g + c];
        const double t = ext > 0 ? ((double)means[3 * i + c] - lo[3 * g + c]) / ext : 0.0;
        code |= spread((uint64_t)std::min(2097151.0, std::max(0.0, t * 2097151.0))) << c;
      }
      key[i] = {{body_id[i], code}, i};
    }
    std::sort(key.begin(), key.end());
    for (int64_t j = 0; j < n; ++j) perm[j] = key[j].second;
  }
  std::vector<float4> hm(n), h0(n), h1(n), h2(n), hs((size_t)np * n);
  std::vector<int2> hids(n);
  std::vector<int> hinv(n);
  for (int64_t j = 0; j < n; ++j) {
    const int64_t i = perm[j];
    const int b = body_id[i];
    hids[j] = make_int2((int)i, b);
    hinv[i] = (int)j;
    const double o = opacities[i];
    if (!(o > 0.0 && o <= 1.0)) return fail(GSB_ERR_INVALID_ARGUMENT, "opacity[%lld] = %g not in (0,1]", (long long)i, o);
    double q[4] = {quats[4 * i], quats[4 * i + 1], quats[4 * i + 2], quats[4 * i + 3]};
    const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(qn > 0)) return fail(GSB_ERR_INVALID_ARGUMENT, "quaternion %lld has zero norm", (long long)i);
    for (double& c : q) c /= qn;
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                            {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                            {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    double s3[3];
    for (int c = 0; c < 3; ++c) {
      s3[c] = scales[3 * i + c];
      if (!(s3[c] > 0)) return fail(GSB_ERR_INVALID_ARGUMENT, "scale[%lld] not > 0", (long long)i);
    }
    float L[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) L[r * 3 + c] = (float)(R[r][c] * s3[c]);
    const double smax = std::max(s3[0], std::max(s3[1], s3[2]));
    hm[j] = make_float4(means[3 * i], means[3 * i + 1], means[3 * i + 2], (float)(smax * smax * (1.0 + 1e-6)));
    h0[j] = make_float4(L[0], L[1], L[2], L[3]);
    h1[j] = make_float4(L[4], L[5], L[6], L[7]);
    h2[j] = make_float4(L[8], opacities[i], (float)(2.0 * std::log(255.0 * o)), (float)std::log2(o));
    for (int pl = 0; pl < np; ++pl) {
      float v4[4] = {0.f, 0.f, 0.f, 0.f};
      for (int k = 0; k < 4; ++k) {
        const int fidx = 4 * pl + k;
        if (fidx < 3 * nc) v4[k] = sh[(size_t)i * 3 * nc + fidx];
      }
      hs[(size_t)pl * n + j] = make_float4(v4[0], v4[1], v4[2], v4[3]);
    }
  }
  DeviceGuard g(device);
  gsb_scene_t* s = new gsb_scene_t();
  s->device = device; s->n = n; s->n_bodies = n_bodies;
  for (int64_t i = 0; i < n; ++i) s->n_bg += (body_id[i] < 0); s->sh_degree = sh_degree; s->sh_planes = np;
  auto up = [&](float4** d, const std::vector<float4>& h) -> cudaError_t {
    cudaError_t e = dalloc(d, h.size());
    if (e != cudaSuccess) return e;
    if (h.empty()) return cudaSuccess;
    return cudaMemcpy(*d, h.data(), h.size() * sizeof(float4), cudaMemcpyHostToDevice);
  };
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = up(&s->d_mean, hm);
  if (e == cudaSuccess) e = up(&s->d_L0, h0);
  if (e == cudaSuccess) e = up(&s->d_L1, h1);
  if (e == cudaSuccess) e = up(&s->d_L2, h2);
  if (e == cudaSuccess) e = up(&s->d_sh, hs);
  if (e == cudaSuccess) e = dalloc(&s->d_ids, (size_t)n);
  if (e == cudaSuccess && n > 0) e = cudaMemcpy(s->d_ids, hids.data(), sizeof(int2) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = dalloc(&s->d_inv, (size_t)n);
  if (e == cudaSuccess && n > 0) e = cudaMemcpy(s->d_inv, hinv.data(), sizeof(int) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = dalloc(&s->d_wsum, (size_t)n);
  if (e == cudaSuccess) e = dalloc(&s->d_wmax, (size_t)n);
  if (e == cudaSuccess && n > 0) e = cudaMemset(s->d_wsum, 0, sizeof(float) * n);
  if (e == cudaSuccess && n > 0) e = cudaMemset(s->d_wmax, 0, sizeof(uint32_t) * n);
  if (e != cudaSuccess) {
    gsb_destroy_scene(s);
    return fail(e == cudaErrorMemoryAllocation ? GSB_ERR_OUT_OF_MEMORY : GSB_ERR_CUDA, "upload: %s", cudaGetErrorString(e));
  }
  *out = s;
  return GSB_OK;
}

gsb_status gsb_reserve(gsb_scene s, int32_t max_envs, int32_t n_cams, int32_t width, int32_t height,
                       int32_t chunk_frames, int64_t key_capacity, uint32_t flags) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (max_envs < 1 || n_cams < 1) return fail(GSB_ERR_INVALID_ARGUMENT, "max_envs/n_cams < 1");
  if (width < 1 || height < 1 || width > kMaxDim || height > kMaxDim)
    return fail(GSB_ERR_INVALID_ARGUMENT, "image %dx%d outside 1..%d", width, height, kMaxDim);
  if (chunk_frames < 0 || key_capacity < 0) return fail(GSB_ERR_INVALID_ARGUMENT, "negative chunk/capacity");
  const int64_t F = (int64_t)max_envs * n_cams;
  if (F > (1 << 30)) return fail(GSB_ERR_CAPACITY, "too many frames");
  DeviceGuard g(s->device);
  cudaDeviceSynchronize();
  s->free_workspace();
  s->max_frames = (int)F; s->res_w = width; s->res_h = height;
  s->max_envs = max_envs; s->res_cams = n_cams;
  s->tiles_x = (width + kTile - 1) / kTile;
  s->tiles_y = (height + kTile - 1) / kTile;
  s->n_tiles = s->tiles_x * s->tiles_y;
  s->hist_stride = ((int64_t)s->n_tiles + 2 + 31) / 32 * 32;
  // automatic chunk: >= 64 frames and ~64k tiles per chunk (small views get bigger chunks so
  // every K4 launch has many waves of CTAs).  256k tiles would gain 0.3-0.7 % on device-resident
  // renders (same-box sweep) but costs ~10 % end to end: gsb_render_host downloads each pass while
  // the next one renders, and the last pass's download is not overlapped
  const char* ct = getenv("GSB_CHUNK_TILES");   // experiments: tiles per automatic chunk
  const int64_t chunk_tiles = ct ? std::max<int64_t>(1, atoll(ct)) : 65536;
  const int auto_e = (int)std::min<int64_t>(kMaxChunk, std::max<int64_t>(64, (chunk_tiles + s->n_tiles - 1) / s->n_tiles));
  const int E = (int)std::min<int64_t>(chunk_frames > 0 ? std::min(chunk_frames, kMaxChunk) : auto_e, F);
  s->chunk = E;
  int64_t cap = key_capacity;
  if (cap == 0) cap = std::max<int64_t>((int64_t)1 << 22, std::min<int64_t>(3 * (int64_t)E * std::max<int64_t>(s->n, 1), ((int64_t)1 << 32) - 1));
  s->cap = cap;
  s->vis_words = (s->n + 31) / 32;
  const int nb1 = s->n_bodies + 1;
  CUDA_TRY(dalloc(&s->table, (size_t)F * nb1 * 4));
  CUDA_TRY(dalloc(&s->cams, (size_t)F));
  for (int sl = 0; sl < 2; ++sl) {
    CUDA_TRY(dalloc(&s->rec[sl], (size_t)E * std::max<int64_t>(s->n, 1) * kRecQuads));
    CUDA_TRY(dalloc(&s->emit[sl], (size_t)E * std::max<int64_t>(s->n, 1)));
    CUDA_TRY(dalloc(&s->vcount[sl], (size_t)E));
    CUDA_TRY(dalloc(&s->vis_bits[sl], (size_t)E * std::max<int64_t>(s->vis_words, 1)));
    CUDA_TRY(dalloc(&s->long_list[sl], (size_t)E * s->n_tiles));
    CUDA_TRY(dalloc(&s->long_cnt[sl], 1));
    CUDA_TRY(dalloc(&s->hist[sl], (size_t)E * s->hist_stride));
    CUDA_TRY(dalloc(&s->off[sl], (size_t)E * s->hist_stride));
    CUDA_TRY(dalloc(&s->frame_base[sl], (size_t)E + 2));
    CUDA_TRY(cudaHostAlloc((void**)&s->h_rb[sl], sizeof(uint64_t) * (2 * E + 3), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer((void**)&s->d_rb[sl], s->h_rb[sl], 0));
    CUDA_TRY(cudaEventCreateWithFlags(&s->ev_counts[sl], cudaEventDisableTiming));
  }
  CUDA_TRY(dalloc(&s->keys, (size_t)cap));
  CUDA_TRY(dalloc(&s->keys_alt, (size_t)cap));
  CUDA_TRY(dalloc(&s->sorted, (size_t)cap));
  CUDA_TRY(dalloc(&s->d_pairs, 1));
  CUDA_TRY(dalloc(&s->d_counter, 1));
  CUDA_TRY(cudaStreamCreateWithFlags(&s->sp, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&s->sc, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&s->sb, cudaStreamNonBlocking));
  CUDA_TRY(dalloc(&s->sorted2, (size_t)cap));
  for (auto& e : s->ev_sorted) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : s->ev_k4b) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&s->ev_bin, cudaEventDisableTiming));
  for (auto& e : s->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&s->ev_start, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&s->ev_end, cudaEventDisableTiming));
  if (s->sb_cams > 0) CUDA_TRY(dalloc(&s->qpos, (size_t)cap));
  s->host_io = (flags & GSB_RESERVE_HOST_IO) != 0;
  if (s->host_io) {
    const size_t plane = (size_t)width * height;
    CUDA_TRY(dalloc(&s->st_poses, (size_t)max_envs * std::max(s->n_bodies, 1) * 7));
    CUDA_TRY(dalloc(&s->st_intr, (size_t)F * 4));
    CUDA_TRY(dalloc(&s->st_w2c, (size_t)F * 12));
    CUDA_TRY(dalloc(&s->st_rgb, (size_t)F * 3 * plane));
    CUDA_TRY(dalloc(&s->st_depth, (size_t)F * plane));
    CUDA_TRY(dalloc(&s->st_alpha, (size_t)F * plane));
    CUDA_TRY(dalloc(&s->st_neval, (size_t)F * plane));
    CUDA_TRY(dalloc(&s->st_dr, (size_t)F * 4));
    CUDA_TRY(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&s->ev_copy, cudaEventDisableTiming));
  }
  s->reserved = true;
  return GSB_OK;
}

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

gsb_status gsb_get_stats(gsb_scene s, int64_t* V, int64_t* K, int64_t* P) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (!s->stats_valid) return fail(GSB_ERR_INVALID_ARGUMENT, "last render had no GSB_FLAG_STATS");
  DeviceGuard g(s->device);
  CUDA_TRY(cudaStreamSynchronize(s->last_stream));
  unsigned long long pairs = 0;
  CUDA_TRY(cudaMemcpy(&pairs, s->d_pairs, sizeof(pairs), cudaMemcpyDeviceToHost));
  if (V) *V = s->stat_V;
  if (K) *K = s->stat_K;
  if (P) *P = (int64_t)pairs;
  return GSB_OK;
}

gsb_status gsb_get_timings(gsb_scene s, gsb_timings* out) {
  if (!s || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!s->timing_valid) return fail(GSB_ERR_INVALID_ARGUMENT, "last render had no GSB_FLAG_TIMING");
  DeviceGuard g(s->device);
  CUDA_TRY(cudaStreamSynchronize(s->last_stream));
  double ms[KC_N] = {0};
  for (auto& m : s->ev_marks) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, s->ev_pool[m.second], s->ev_pool[m.second + 1]));
    ms[m.first] += t;
  }
  out->setup_ms = ms[KC_SETUP]; out->project_ms = ms[KC_PROJECT]; out->scan_ms = ms[KC_SCAN];
  out->emit_ms = ms[KC_EMIT]; out->sort_ms = ms[KC_SORT]; out->composite_ms = ms[KC_COMPOSITE];
  out->launches = s->launches; out->composite_launches = s->comp_launches; out->chunks = s->chunks;
  out->long_lists = s->stat_long; out->max_list = s->stat_maxseg;
  return GSB_OK;
}

gsb_status gsb_scores_reset(gsb_scene s, gsb_stream stream) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  DeviceGuard g(s->device);
  if (s->n > 0) {
    CUDA_TRY(cudaMemsetAsync(s->d_wsum, 0, sizeof(float) * s->n, (cudaStream_t)stream));
    CUDA_TRY(cudaMemsetAsync(s->d_wmax, 0, sizeof(uint32_t) * s->n, (cudaStream_t)stream));
  }
  return GSB_OK;
}

gsb_status gsb_get_scores(gsb_scene s, float* w_sum, float* w_max, gsb_stream stream) {
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  DeviceGuard g(s->device);
  launch_k4_scores_export(s->d_wsum, s->d_wmax, s->d_ids, s->n, w_sum, w_max, (cudaStream_t)stream);
  LAUNCH_CHECK();
  return GSB_OK;
}

gsb_status gsb_filter_scene(gsb_scene s, const uint8_t* keep, gsb_scene* out) {
  if (!out) return fail(GSB_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!s) return fail(GSB_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (s->n > 0 && !keep) return fail(GSB_ERR_INVALID_ARGUMENT, "keep is NULL");
  DeviceGuard g(s->device);
  const int64_t n = s->n;
  const int np = s->sh_planes;
  std::vector<float4> hm(n), h0(n), h1(n), h2(n), hs((size_t)np * n);
  std::vector<int2> hids(n);
  if (n > 0) {
    CUDA_TRY(cudaMemcpy(hm.data(), s->d_mean, sizeof(float4) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(h0.data(), s->d_L0, sizeof(float4) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(h1.data(), s->d_L1, sizeof(float4) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(h2.data(), s->d_L2, sizeof(float4) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(hs.data(), s->d_sh, sizeof(float4) * np * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(hids.data(), s->d_ids, sizeof(int2) * n, cudaMemcpyDeviceToHost));
  }
  // new id = rank of the old id among the kept ones (creation order preserved)
  std::vector<int> newid(n, -1);
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (keep[i]) newid[i] = (int)m++;
  // kept Gaussians in the parent's internal order (still grouped by body, background first)
  std::vector<float4> km, k0, k1, k2, ks((size_t)np * m);
  std::vector<int2> kids;
  std::vector<int> kinv(m);
  km.reserve(m); k0.reserve(m); k1.reserve(m); k2.reserve(m); kids.reserve(m);
  int64_t nbg = 0;
  for (int64_t j = 0; j < n; ++j) {
    const int id = hids[j].x;
    if (!keep[id]) continue;
    const int64_t jj = (int64_t)km.size();
    km.push_back(hm[j]); k0.push_back(h0[j]); k1.push_back(h1[j]); k2.push_back(h2[j]);
    for (int pl = 0; pl < np; ++pl) ks[(size_t)pl * m + jj] = hs[(size_t)pl * n + j];
    kids.push_back(make_int2(newid[id], hids[j].y));
    kinv[newid[id]] = (int)jj;
    nbg += hids[j].y < 0;
  }
  gsb_scene_t* t = new gsb_scene_t();
  t->device = s->device; t->n = m; t->n_bg = nbg; t->n_bodies = s->n_bodies; t->sh_degree = s->sh_degree;
  t->sh_planes = np;
  auto up = [&](auto** d, const auto& h) -> cudaError_t {
    cudaError_t e = dalloc(d, h.size());
    if (e != cudaSuccess || h.empty()) return e;
    return cudaMemcpy(*d, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice);
  };
  cudaError_t e = up(&t->d_mean, km);
  if (e == cudaSuccess) e = up(&t->d_L0, k0);
  if (e == cudaSuccess) e = up(&t->d_L1, k1);
  if (e == cudaSuccess) e = up(&t->d_L2, k2);
  if (e == cudaSuccess) e = up(&t->d_sh, ks);
  if (e == cudaSuccess) e = up(&t->d_ids, kids);
  if (e == cudaSuccess) e = up(&t->d_inv, kinv);
  if (e == cudaSuccess) e = dalloc(&t->d_wsum, (size_t)m);
  if (e == cudaSuccess) e = dalloc(&t->d_wmax, (size_t)m);
  if (e == cudaSuccess && m > 0) e = cudaMemset(t->d_wsum, 0, sizeof(float) * m);
  if (e == cudaSuccess && m > 0) e = cudaMemset(t->d_wmax, 0, sizeof(uint32_t) * m);
  if (e != cudaSuccess) {
    gsb_destroy_scene(t);
    return fail(e == cudaErrorMemoryAllocation ? GSB_ERR_OUT_OF_MEMORY : GSB_ERR_CUDA, "filter upload: %s",
                cudaGetErrorString(e));
  }
  *out = t;
  return GSB_OK;
}

gsb_status gsb_destroy_scene(gsb_scene s) {
  if (!s) return GSB_OK;
  DeviceGuard g(s->device);
  cudaDeviceSynchronize();
  s->free_workspace();
  s->free_prebin();
  cudaFree(s->d_mean); cudaFree(s->d_L0); cudaFree(s->d_L1); cudaFree(s->d_L2); cudaFree(s->d_sh);
  cudaFree(s->d_ids);
  cudaFree(s->d_inv);
  cudaFree(s->d_wsum);
  cudaFree(s->d_wmax);
  delete s;
  return GSB_OK;
}

gsb_status gsb_debug_project(gsb_scene s, const float* poses, int32_t n_envs, int32_t n_cams,
                             const float* intr, const float* w2c, const gsb_render_params* p,
                             float* out_rec, uint32_t* out_zbits, uint8_t* out_valid, gsb_stream stream) {
  gsb_status r = validate_render(s, poses, n_envs, n_cams, intr, w2c, p, out_rec);
  if (r != GSB_OK) return r;
  if (!out_zbits || !out_valid) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL debug output");
  DeviceGuard g(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int F = n_envs * n_cams;
  launch_k0(default_rig(s, poses, intr, w2c), F, n_cams, s->n_bodies, p->width, p->height, s->table, s->cams, st);
  LAUNCH_CHECK();
  K1Args a{};
  a.g_mean = s->d_mean; a.g_L0 = s->d_L0; a.g_L1 = s->d_L1; a.g_L2 = s->d_L2; a.g_sh = s->d_sh;
    a.g_ids = s->d_ids;
  a.n = s->n; a.sh_stride = s->n; a.table = s->table; a.cams = s->cams; a.nb1 = s->n_bodies + 1;
  a.f0 = 0; a.n_frames = F; a.width = p->width; a.height = p->height;
  a.tiles_x = (p->width + kTile - 1) / kTile;
  a.near_plane = p->near_plane; a.far_plane = p->far_plane;
  a.rec = nullptr;
  a.dbg_rec = out_rec; a.dbg_zbits = out_zbits; a.dbg_valid = out_valid;
  launch_k1(a, p->sh_degree < 0 ? s->sh_degree : p->sh_degree, st);
  LAUNCH_CHECK();
  return GSB_OK;
}

gsb_status gsb_debug_bin_sort(const float* u, const float* v, const float* sxx, const float* syy,
                              const float* kappa, const uint32_t* zbits, const uint8_t* valid,
                              int32_t F, int64_t n, int32_t width, int32_t height,
                              int64_t* out_offsets, uint32_t* out_ids, int64_t cap, int64_t* out_K,
                              gsb_stream stream) {
  if (F < 1 || n < 0 || width < 1 || height < 1 || width > kMaxDim || height > kMaxDim || cap < 0 || !out_K ||
      !out_offsets || (n > 0 && (!u || !v || !sxx || !syy || !kappa || !zbits || !valid)))
    return fail(GSB_ERR_INVALID_ARGUMENT, "bad debug_bin_sort arguments");
  if (n >= (int64_t)1 << 31) return fail(GSB_ERR_CAPACITY, "n >= 2^31");
  cudaStream_t st = (cudaStream_t)stream;
  const int tiles_x = (width + kTile - 1) / kTile;
  const int n_tiles = tiles_x * ((height + kTile - 1) / kTile);
  const int64_t stride = ((int64_t)n_tiles + 2 + 31) / 32 * 32;
  uint2* emit = nullptr; int* vcount = nullptr; int* hist = nullptr; uint32_t* off = nullptr;
  uint32_t* vbits = nullptr;
  const int64_t vwords = (n + 31) / 32;
  uint64_t* fbase = nullptr; uint64_t* keys = nullptr; uint64_t* keys_alt = nullptr; uint32_t* sorted = nullptr;
  gsb_status result = GSB_OK;
  auto cleanup = [&]() {
    cudaFree(emit); cudaFree(vcount); cudaFree(hist); cudaFree(off); cudaFree(fbase); cudaFree(vbits);
    cudaFree(keys); cudaFree(keys_alt); cudaFree(sorted);
  };
#define DBG_TRY(expr)                                                              \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      cleanup();                                                                   \
      return fail(GSB_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));          \
    }                                                                              \
  } while (0)
  DBG_TRY(dalloc(&emit, (size_t)F * std::max<int64_t>(n, 1)));
  DBG_TRY(dalloc(&vcount, (size_t)F));
  DBG_TRY(dalloc(&vbits, (size_t)F * std::max<int64_t>(vwords, 1)));
  DBG_TRY(dalloc(&hist, (size_t)F * stride));
  DBG_TRY(dalloc(&off, (size_t)F * stride));
  DBG_TRY(dalloc(&fbase, (size_t)F + 2));
  DBG_TRY(cudaMemsetAsync(vcount, 0, sizeof(int) * F, st));
  DBG_TRY(cudaMemsetAsync(hist, 0, sizeof(int) * F * stride, st));
  DBG_TRY(cudaMemsetAsync(off, 0, sizeof(uint32_t) * F * stride, st));   // padding rows are read back below
  launch_k1_external(u, v, sxx, syy, kappa, zbits, valid, n, 0, F, width, height, tiles_x, emit, vbits, vwords,
                     vcount, hist, stride, st);
  launch_k2_scan(hist, off, stride, F, n_tiles, fbase, nullptr, nullptr, 0, nullptr, nullptr, st);
  DBG_TRY(cudaGetLastError());
  std::vector<uint64_t> hfb(F + 2);
  DBG_TRY(cudaMemcpyAsync(hfb.data(), fbase, sizeof(uint64_t) * (F + 2), cudaMemcpyDeviceToHost, st));
  DBG_TRY(cudaStreamSynchronize(st));
  const uint64_t K = hfb[F];
  *out_K = (int64_t)K;
  if (K > (uint64_t)cap) {
    cleanup();
    return fail(GSB_ERR_CAPACITY, "K = %llu exceeds cap %lld", (unsigned long long)K, (long long)cap);
  }
  DBG_TRY(dalloc(&keys, std::max<uint64_t>(K, 1)));
  DBG_TRY(dalloc(&keys_alt, std::max<uint64_t>(K, 1)));
  DBG_TRY(dalloc(&sorted, std::max<uint64_t>(K, 1)));
  ChunkArgs a{};
  a.rec = nullptr; a.emit = emit; a.ids = nullptr; a.n = n; a.vis_bits = vbits; a.vis_words = vwords; a.hist = hist; a.hist_stride = stride; a.off = off;
  a.frame_base = fbase; a.n_tiles = n_tiles; a.tiles_x = tiles_x; a.fs = 0; a.fe = F; a.key_base = 0;
  a.long_list = nullptr;  // K3 sorts every list here
  a.keys = keys; a.keys_alt = keys_alt; a.sorted = sorted;
  launch_k2_emit(a, st);
  launch_k3_sort(a, 0, st);
  if (K > 0) DBG_TRY(cudaMemcpyAsync(out_ids, sorted, sizeof(uint32_t) * K, cudaMemcpyDeviceToDevice, st));
  DBG_TRY(cudaGetLastError());
  std::vector<uint32_t> hoff((size_t)F * stride);
  DBG_TRY(cudaMemcpyAsync(hoff.data(), off, sizeof(uint32_t) * hoff.size(), cudaMemcpyDeviceToHost, st));
  DBG_TRY(cudaStreamSynchronize(st));
  std::vector<int64_t> ho((size_t)F * (n_tiles + 1));
  for (int f = 0; f < F; ++f)
    for (int t = 0; t <= n_tiles; ++t) ho[(size_t)f * (n_tiles + 1) + t] = (int64_t)hfb[f] + hoff[(size_t)f * stride + t];
  DBG_TRY(cudaMemcpyAsync(out_offsets, ho.data(), sizeof(int64_t) * ho.size(), cudaMemcpyHostToDevice, st));
  DBG_TRY(cudaStreamSynchronize(st));
  cleanup();
  return result;
#undef DBG_TRY
}

}  // extern "C"

// =====================================================================================
// Batched ray-cast LiDAR (§8(f) row 4, reading R32): gsb_lidar_create / gsb_render_lidar.
// Chunked like the camera path but on the caller's stream only, with one synchronous
// readback of the chunk's key count (the workspace grows on demand).
// =====================================================================================
struct gsb_lidar_t {
  gsb_scene scene = nullptr;
  int device = 0;
  int n_rays = 0, n_az = 0, n_el = 0, n_items = 0;
  float az0 = 0.f, az_span = 0.f, el0 = 0.f, el_span = 0.f;
  float4* d_rays = nullptr;   // grouped by cell, w = bits(original index)
  int4* d_items = nullptr;
  // workspace
  int ws_frames = 0;          // chunk capacity (frames)
  int ws_req = 0;             // chunk size requested when the workspace was sized (>= ws_frames)
  int table_frames = 0;
  int64_t np = 0;
  int64_t hist_stride = 0;
  float4* table = nullptr;
  float4* rec = nullptr;
  uint2* emit = nullptr;
  uint32_t* vis_bits = nullptr;
  int* vcount = nullptr;
  int* hist = nullptr;
  uint32_t* off = nullptr;
  uint64_t* frame_base = nullptr;
  int2* ids2 = nullptr;
  uint64_t *keys = nullptr, *keys_alt = nullptr;
  uint32_t* sorted = nullptr;
  uint64_t key_cap = 0;
  int64_t last_keys = 0;
  void free_ws() {
    cudaFree(rec); cudaFree(emit); cudaFree(vis_bits); cudaFree(vcount); cudaFree(hist);
    cudaFree(off); cudaFree(frame_base); cudaFree(ids2); cudaFree(keys); cudaFree(keys_alt); cudaFree(sorted);
    rec = nullptr; emit = nullptr; vis_bits = nullptr; vcount = nullptr; hist = nullptr;
    off = nullptr; frame_base = nullptr; ids2 = nullptr; keys = keys_alt = nullptr; sorted = nullptr;
    ws_frames = 0; ws_req = 0; key_cap = 0;
  }
};

namespace {

constexpr int kLidarMaxCells = 256;
constexpr double kLidarPi = 3.14159265358979323846;

// frames per LiDAR chunk: records (80 B) + emission (16 B) per (frame, Gaussian) within ~8 GB
// (KL4's parallelism is frames x ray groups: sparse patterns such as a height scan need many
// frames per launch to fill the GPU)
int lidar_chunk(int64_t n, int F) {
  const int64_t per = std::max<int64_t>(1, n) * 96 + 4096;
  const int64_t e = std::max<int64_t>(1, ((int64_t)8 << 30) / per);
  return (int)std::min<int64_t>({e, (int64_t)F, 1024});
}

}  // namespace

extern "C" {

gsb_status gsb_lidar_create(gsb_scene s, const float* dirs, int32_t n_rays, int32_t n_az, int32_t n_el,
                            gsb_lidar* out) {
  if (!s || !dirs || !out || n_rays < 1) return fail(GSB_ERR_INVALID_ARGUMENT, "bad lidar_create arguments");
  if (n_az < 0 || n_el < 0 || n_az > kLidarMaxCells || n_el > kLidarMaxCells)
    return fail(GSB_ERR_INVALID_ARGUMENT, "n_az, n_el must be in [0, %d]", kLidarMaxCells);
  *out = nullptr;
  std::vector<double> az(n_rays), el(n_rays);
  for (int j = 0; j < n_rays; ++j) {
    const double x = dirs[3 * j], y = dirs[3 * j + 1], z = dirs[3 * j + 2];
    const double nn = std::sqrt(x * x + y * y + z * z);
    if (!std::isfinite(nn) || std::fabs(nn - 1.0) > 1e-5)
      return fail(GSB_ERR_INVALID_ARGUMENT, "ray %d is not a unit vector (norm %g)", j, nn);
    az[j] = std::atan2(y, x);
    el[j] = std::atan2(z, std::sqrt(x * x + y * y));
  }
  // elevation window of the rays; azimuth window = the circle minus its largest empty gap
  const double m = 1e-4;
  double el_lo = *std::min_element(el.begin(), el.end()) - m, el_hi = *std::max_element(el.begin(), el.end()) + m;
  el_lo = std::max(el_lo, -0.5 * kLidarPi);
  el_hi = std::min(el_hi, 0.5 * kLidarPi);
  std::vector<double> sa(az);
  std::sort(sa.begin(), sa.end());
  double gap = sa.front() + 2 * kLidarPi - sa.back(), a0 = sa.front();
  for (int j = 1; j < n_rays; ++j)
    if (sa[j] - sa[j - 1] > gap) { gap = sa[j] - sa[j - 1]; a0 = sa[j]; }
  double span = 2 * kLidarPi - gap + 2 * m;
  a0 -= m;
  if (span >= 2 * kLidarPi - 1e-3 || gap < kLidarPi / 8) { span = 2 * kLidarPi; a0 = -kLidarPi; }
  const double espan = el_hi - el_lo;
  if (n_az == 0 || n_el == 0) {   // ~32 rays per cell, cells about square in angle
    const double cells = std::max(1.0, n_rays / 32.0);
    const double c = std::sqrt(span * espan / cells);
    if (n_az == 0) n_az = (int)std::min<double>(kLidarMaxCells, std::max(1.0, std::round(span / c)));
    if (n_el == 0) n_el = (int)std::min<double>(kLidarMaxCells, std::max(1.0, std::round(espan / c)));
  }
  // cell of each ray (fp64; the device's Gaussian bounds carry a 1e-3 rad margin)
  std::vector<int> cell(n_rays);
  for (int j = 0; j < n_rays; ++j) {
    double rel = az[j] - a0;
    rel -= 2 * kLidarPi * std::floor(rel / (2 * kLidarPi));
    const int cx = std::min(n_az - 1, std::max(0, (int)std::floor(rel / span * n_az)));
    const int cy = std::min(n_el - 1, std::max(0, (int)std::floor((el[j] - el_lo) / espan * n_el)));
    cell[j] = cy * n_az + cx;
  }
  std::vector<int> order(n_rays);
  for (int j = 0; j < n_rays; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int p, int q) { return cell[p] < cell[q]; });
  std::vector<float4> rays(n_rays);
  std::vector<int4> items;
  for (int k = 0; k < n_rays;) {
    const int c = cell[order[k]];
    int e = k;
    while (e < n_rays && cell[order[e]] == c) ++e;
    for (int b = k; b < e; b += 32) items.push_back(make_int4(c, b, std::min(32, e - b), 0));
    k = e;
  }
  for (int k = 0; k < n_rays; ++k) {
    const int j = order[k];
    float w;
    std::memcpy(&w, &j, 4);
    rays[k] = make_float4(dirs[3 * j], dirs[3 * j + 1], dirs[3 * j + 2], w);
  }
  DeviceGuard g(s->device);
  gsb_lidar_t* l = new gsb_lidar_t();
  l->scene = s; l->device = s->device; l->n_rays = n_rays; l->n_az = n_az; l->n_el = n_el;
  l->n_items = (int)items.size();
  l->az0 = (float)a0; l->az_span = (float)span; l->el0 = (float)el_lo; l->el_span = (float)espan;
  cudaError_t e = dalloc(&l->d_rays, (size_t)n_rays);
  if (e == cudaSuccess) e = dalloc(&l->d_items, items.size());
  if (e == cudaSuccess) e = cudaMemcpy(l->d_rays, rays.data(), sizeof(float4) * n_rays, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(l->d_items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(l->d_rays); cudaFree(l->d_items);
    delete l;
    return fail(e == cudaErrorMemoryAllocation ? GSB_ERR_OUT_OF_MEMORY : GSB_ERR_CUDA, "lidar_create: %s",
                cudaGetErrorString(e));
  }
  *out = l;
  return GSB_OK;
}

gsb_status gsb_lidar_info(gsb_lidar l, int32_t* n_az, int32_t* n_el, int32_t* n_items, int64_t* last_keys) {
  if (!l) return fail(GSB_ERR_INVALID_ARGUMENT, "lidar is NULL");
  if (n_az) *n_az = l->n_az;
  if (n_el) *n_el = l->n_el;
  if (n_items) *n_items = l->n_items;
  if (last_keys) *last_keys = l->last_keys;
  return GSB_OK;
}

gsb_status gsb_lidar_destroy(gsb_lidar l) {
  if (!l) return GSB_OK;
  DeviceGuard g(l->device);
  l->free_ws();
  cudaFree(l->table);
  cudaFree(l->d_rays); cudaFree(l->d_items);
  delete l;
  return GSB_OK;
}

gsb_status gsb_render_lidar(gsb_scene s, gsb_lidar l, const float* poses, int32_t n_envs, int32_t n_sensors,
                            const float* sensor_x, int32_t sensors_shared, const int32_t* sensor_body,
                            float near_plane, float far_plane, float* out_range, float* out_alpha,
                            gsb_stream stream) {
  if (!s || !l) return fail(GSB_ERR_INVALID_ARGUMENT, "scene or lidar is NULL");
  if (l->scene != s) return fail(GSB_ERR_INVALID_ARGUMENT, "lidar belongs to another scene");
  if (n_envs < 0 || n_sensors < 1) return fail(GSB_ERR_INVALID_ARGUMENT, "n_envs=%d n_sensors=%d", n_envs, n_sensors);
  if (!(near_plane > 0.f) || !(far_plane > near_plane)) return fail(GSB_ERR_INVALID_ARGUMENT, "need 0 < near < far");
  const int64_t F64 = (int64_t)n_envs * n_sensors;
  if (F64 > (1 << 24)) return fail(GSB_ERR_CAPACITY, "too many frames");
  const int F = (int)F64;
  if (F == 0) return GSB_OK;
  if (!sensor_x || !out_range) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL sensor_x / out_range");
  if (s->n_bodies > 0 && !poses) return fail(GSB_ERR_INVALID_ARGUMENT, "body_poses is NULL but the scene has bodies");
  K0Rig rig{};
  rig.poses = poses;
  rig.env_stride = (int64_t)s->n_bodies * 7;
  rig.body_stride = 7;
  rig.intr = nullptr;
  rig.cam_x = sensor_x;
  rig.cams_shared = sensors_shared ? 1 : 0;
  for (int c = 0; c < kMaxRigCams; ++c) rig.cam_body[c] = -1;
  if (sensor_body) {
    for (int c = 0; c < n_sensors; ++c) {
      if (sensor_body[c] < -1 || sensor_body[c] >= s->n_bodies)
        return fail(GSB_ERR_UNKNOWN_BODY, "sensor_body[%d] = %d outside [-1, %d)", c, sensor_body[c], s->n_bodies);
      if (sensor_body[c] >= 0) {
        if (c >= kMaxRigCams) return fail(GSB_ERR_CAPACITY, "attached sensor index %d >= %d", c, kMaxRigCams);
        rig.cam_body[c] = sensor_body[c];
      }
    }
  }
  DeviceGuard g(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t N = s->n;
  const int n_cells = l->n_az * l->n_el;
  int E = lidar_chunk(N, F);
  // workspace (grows on demand; synchronises then)
  if (l->table_frames < F) {
    CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(l->table);
    l->table = nullptr;
    l->table_frames = 0;
    CUDA_TRY(dalloc(&l->table, (size_t)F * (s->n_bodies + 1) * 4));
    l->table_frames = F;
  }
  if (l->ws_req < E || l->np != (N + 31) / 32 * 32) {
    const int req = E;
    CUDA_TRY(cudaStreamSynchronize(st));
    l->free_ws();
    l->np = (N + 31) / 32 * 32;
    const int64_t np = std::max<int64_t>(l->np, 32);
    l->hist_stride = ((int64_t)n_cells + 2 + 31) / 32 * 32;
    // the records dominate the workspace: on an allocation failure retry with half the frames
    for (;;) {
      const cudaError_t e = dalloc(&l->rec, (size_t)E * std::max<int64_t>(N, 1) * kLidarRecQuads);
      if (e == cudaSuccess) break;
      if (e != cudaErrorMemoryAllocation || E == 1) CUDA_TRY(e);
      cudaGetLastError();   // clear the sticky-free allocation error
      E = std::max(1, E / 2);
    }
    CUDA_TRY(dalloc(&l->emit, (size_t)E * 2 * np));
    CUDA_TRY(dalloc(&l->vis_bits, (size_t)E * 2 * np / 32));
    CUDA_TRY(dalloc(&l->vcount, (size_t)E));
    CUDA_TRY(dalloc(&l->hist, (size_t)E * l->hist_stride));
    CUDA_TRY(dalloc(&l->off, (size_t)E * l->hist_stride));
    CUDA_TRY(dalloc(&l->frame_base, (size_t)E + 2));
    CUDA_TRY(dalloc(&l->ids2, (size_t)2 * np));
    CUDA_TRY(cudaMemset(l->ids2, 0, sizeof(int2) * 2 * np));
    if (N > 0) {
      CUDA_TRY(cudaMemcpy(l->ids2, s->d_ids, sizeof(int2) * N, cudaMemcpyDeviceToDevice));
      CUDA_TRY(cudaMemcpy(l->ids2 + l->np, s->d_ids, sizeof(int2) * N, cudaMemcpyDeviceToDevice));
    }
    l->ws_frames = E;
    l->ws_req = req;
  }
  E = std::min(E, l->ws_frames);
  launch_k0(rig, F, n_sensors, s->n_bodies, 1, 1, l->table, nullptr, st);
  LAUNCH_CHECK();
  l->last_keys = 0;
  std::vector<uint64_t> hfb(E + 2);
  for (int f0 = 0; f0 < F; f0 += E) {
    const int ne = std::min(E, F - f0);
    CUDA_TRY(cudaMemsetAsync(l->hist, 0, sizeof(int) * (size_t)ne * l->hist_stride, st));
    CUDA_TRY(cudaMemsetAsync(l->vcount, 0, sizeof(int) * ne, st));
    LidarL1Args a{};
    a.g_mean = s->d_mean; a.g_L0 = s->d_L0; a.g_L1 = s->d_L1; a.g_L2 = s->d_L2; a.g_ids = s->d_ids;
    a.n = N; a.np = l->np; a.table = l->table; a.nb1 = s->n_bodies + 1; a.f0 = f0; a.n_frames = ne;
    a.near_plane = near_plane; a.far_plane = far_plane;
    a.az0 = l->az0; a.az_span = l->az_span; a.az_inv = (float)(l->n_az / (double)l->az_span);
    a.el0 = l->el0; a.el_inv = (float)(l->n_el / (double)l->el_span);
    a.n_az = l->n_az; a.n_el = l->n_el;
    a.rec = l->rec; a.emit = l->emit; a.vis_bits = l->vis_bits; a.vis_words = 2 * l->np / 32;
    a.vcount = l->vcount; a.hist = l->hist; a.hist_stride = l->hist_stride;
    launch_kl1(a, st);
    launch_k2_scan(l->hist, l->off, l->hist_stride, ne, n_cells, l->frame_base, nullptr, nullptr, 0, nullptr,
                   nullptr, st);
    LAUNCH_CHECK();
    CUDA_TRY(cudaMemcpyAsync(hfb.data(), l->frame_base, sizeof(uint64_t) * (ne + 2), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const uint64_t K = hfb[ne];
    l->last_keys += (int64_t)K;
    if (K > l->key_cap) {
      cudaFree(l->keys); cudaFree(l->keys_alt); cudaFree(l->sorted);
      l->keys = l->keys_alt = nullptr; l->sorted = nullptr; l->key_cap = 0;
      const uint64_t cap = K + K / 4 + 1024;
      CUDA_TRY(dalloc(&l->keys, cap));
      CUDA_TRY(dalloc(&l->keys_alt, cap));
      CUDA_TRY(dalloc(&l->sorted, cap));
      l->key_cap = cap;
    }
    if (K > 0) {
      ChunkArgs c{};
      // keys carry the (virtual) index: the seam copy np + i of Gaussian i keeps its own key, K4a
      // restores the (bits(rho), id) order of equal ranges through ids2 and KL4 folds np + i to i
      c.rec = nullptr; c.emit = l->emit; c.ids = nullptr; c.n = 2 * l->np;
      c.vis_bits = l->vis_bits; c.vis_words = 2 * l->np / 32; c.hist = l->hist; c.hist_stride = l->hist_stride;
      c.off = l->off; c.frame_base = l->frame_base; c.n_tiles = n_cells; c.tiles_x = l->n_az;
      c.fs = 0; c.fe = ne; c.key_base = 0; c.long_list = nullptr;
      c.keys = l->keys; c.keys_alt = l->keys_alt; c.sorted = l->sorted;
      launch_k2_emit(c, st);
      CompositeArgs k{};   // K4a: (bits(rho), id) order -> record slots (slot_base 0: internal index)
      k.keys = l->keys; k.keys_alt = l->keys_alt; k.off = l->off; k.frame_base = l->frame_base;
      k.hist_stride = l->hist_stride; k.key_base = 0; k.fs = 0; k.fe = ne; k.f0 = f0;
      k.n_tiles = n_cells; k.tiles_x = l->n_az; k.inv = s->d_inv; k.slot_base = 0; k.sorted = l->sorted;
      k.keys_internal_ids = l->ids2;
      launch_k4a_sort(k, false, st);
      LidarL4Args b{};
      b.rec = l->rec; b.n = N; b.off = l->off; b.frame_base = l->frame_base; b.hist_stride = l->hist_stride;
      b.sorted = l->sorted; b.rays = l->d_rays; b.items = l->d_items; b.np = l->np;
      b.n_items = l->n_items; b.f0 = f0; b.n_frames = ne; b.n_rays = l->n_rays;
      b.out_range = out_range; b.out_alpha = out_alpha;
      launch_kl4(b, st);
      LAUNCH_CHECK();
    } else {
      CUDA_TRY(cudaMemsetAsync(out_range + (size_t)f0 * l->n_rays, 0, sizeof(float) * (size_t)ne * l->n_rays, st));
      if (out_alpha)
        CUDA_TRY(cudaMemsetAsync(out_alpha + (size_t)f0 * l->n_rays, 0, sizeof(float) * (size_t)ne * l->n_rays, st));
    }
  }
  return GSB_OK;
}

}  // extern "C"
