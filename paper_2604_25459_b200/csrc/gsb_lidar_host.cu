#include "gsb_runtime.cuh"

using namespace gsb;

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
bool lidar_idx_sort() {
  const char* e = getenv("GSB_LIDAR_K4A");
  return !(e && e[0] == 'c');
}

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
      // the cell lists: one CTA each with the index counting sort (<= 4096 keys, HBM radix beyond);
      // GSB_LIDAR_K4A=cta: the round-1 CTA counting sort (A/B)
      launch_k4a_sort(k, lidar_idx_sort(), st);
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
