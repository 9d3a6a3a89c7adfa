// gsb_api.cu — libgsb host runtime, part 1: the scene template and its workspace.
//
// gsb_create_scene builds the read-only template (K5: one copy shared by every env, internal
// order = body, then Morton code), gsb_reserve sizes every buffer of the chunked pipeline (no
// allocation happens inside a render), plus stats / timings / pruning scores / filtering and
// gsb_destroy_scene.  The pipeline itself is in gsb_render.cu (see gsb_runtime.cuh).
#include "gsb_runtime.cuh"

using namespace gsb;

namespace gsb {

namespace {
thread_local std::string g_err = "no error";
}  // namespace

gsb_status fail(gsb_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
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

}  // namespace gsb

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
  const int np = 3 * ((nc + 3) / 4);   // 3 float4 planes per group of 4 coefficients (gsb_common.cuh)
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
    // group g of coefficients k = 4g .. 4g+3: (r, g) of k, k+1 | (r, g) of k+2, k+3 | b of all four
    auto coef = [&](int k, int ch) { return k < nc ? sh[(size_t)i * 3 * nc + 3 * k + ch] : 0.f; };
    for (int g4 = 0; g4 < np / 3; ++g4) {
      const int k = 4 * g4;
      hs[(size_t)(3 * g4) * n + j] = make_float4(coef(k, 0), coef(k, 1), coef(k + 1, 0), coef(k + 1, 1));
      hs[(size_t)(3 * g4 + 1) * n + j] = make_float4(coef(k + 2, 0), coef(k + 2, 1), coef(k + 3, 0), coef(k + 3, 1));
      hs[(size_t)(3 * g4 + 2) * n + j] = make_float4(coef(k, 2), coef(k + 1, 2), coef(k + 2, 2), coef(k + 3, 2));
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
  // automatic chunk: >= 64 frames and ~256k tiles per chunk for device-resident renders (each
  // chunk's persistent K4b ends with a tail and its binning with a ramp: fewer, larger chunks
  // are +1.5 % on C3 over 64k tiles, same-box), but ~64k tiles for gsb_render_host, which
  // downloads each pass while the next renders (the last pass's download is not overlapped: 256k
  // tiles cost ~10 % end to end).  Both use the same buffers (the host chunk is the smaller).
  const char* ct = getenv("GSB_CHUNK_TILES");   // experiments: tiles per automatic device chunk
  const int64_t chunk_tiles = ct ? std::max<int64_t>(1, atoll(ct)) : 262144;
  auto auto_chunk = [&](int64_t tiles) {
    return (int)std::min<int64_t>(kMaxChunk, std::max<int64_t>(64, (tiles + s->n_tiles - 1) / s->n_tiles));
  };
  int E = (int)std::min<int64_t>(chunk_frames > 0 ? std::min(chunk_frames, kMaxChunk) : auto_chunk(chunk_tiles), F);
  // K4b addresses a chunk's records with 32-bit (frame * N + slot) indices
  E = (int)std::max<int64_t>(1, std::min<int64_t>(E, (int64_t)0xffffffffu / std::max<int64_t>(s->n, 1)));
  s->chunk = E;
  s->chunk_host = chunk_frames > 0 ? E : (int)std::min<int64_t>(E, auto_chunk(65536));
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
    CUDA_TRY(dalloc(&s->trim[sl], (size_t)E * std::max<int64_t>(s->n, 1)));
    CUDA_TRY(dalloc(&s->vcount[sl], (size_t)E));
    CUDA_TRY(dalloc(&s->vis_bits[sl], (size_t)E * std::max<int64_t>(s->vis_words, 1)));
    CUDA_TRY(dalloc(&s->long_list[sl], (size_t)E * s->n_tiles));
    CUDA_TRY(dalloc(&s->long_cnt[sl], 2));
    CUDA_TRY(dalloc(&s->hist[sl], (size_t)E * s->hist_stride));
    CUDA_TRY(dalloc(&s->off[sl], (size_t)E * s->hist_stride));
    CUDA_TRY(dalloc(&s->frame_base[sl], (size_t)E + 2));
    CUDA_TRY(cudaHostAlloc((void**)&s->h_rb[sl], sizeof(uint64_t) * (2 * E + 4), cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer((void**)&s->d_rb[sl], s->h_rb[sl], 0));
    CUDA_TRY(cudaEventCreateWithFlags(&s->ev_counts[sl], cudaEventDisableTiming));
  }
  CUDA_TRY(dalloc(&s->keys, (size_t)cap));
  CUDA_TRY(dalloc(&s->keys_alt, (size_t)cap));
  CUDA_TRY(dalloc(&s->sorted, (size_t)cap));
  CUDA_TRY(dalloc(&s->d_pairs, 2));
  CUDA_TRY(dalloc(&s->d_overflow, 4));
  CUDA_TRY(cudaMemset(s->d_overflow, 0, 4 * sizeof(int)));
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

gsb_status gsb_get_stats_ext(gsb_scene s, gsb_stats* out) {
  if (!s || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!s->stats_valid) return fail(GSB_ERR_INVALID_ARGUMENT, "last render had no GSB_FLAG_STATS");
  DeviceGuard g(s->device);
  CUDA_TRY(cudaStreamSynchronize(s->last_stream));
  unsigned long long c[2] = {0, 0};
  CUDA_TRY(cudaMemcpy(c, s->d_pairs, sizeof(c), cudaMemcpyDeviceToHost));
  out->visible_V = s->stat_V;
  out->keys_K = s->stat_K;
  out->pairs_P = (int64_t)c[0];
  out->terminated_pixels = (int64_t)c[1];
  out->pixels = s->stat_pixels;
  return GSB_OK;
}

gsb_status gsb_get_overflow(gsb_scene s, int32_t* out) {
  if (!s || !out) return fail(GSB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!s->reserved) return fail(GSB_ERR_INVALID_ARGUMENT, "gsb_reserve was not called");
  DeviceGuard g(s->device);
  CUDA_TRY(cudaDeviceSynchronize());   // the render may have been replayed from a graph on any stream
  int v = 0;
  CUDA_TRY(cudaMemcpy(&v, s->d_overflow, sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemset(s->d_overflow, 0, sizeof(int)));
  *out = v;
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
}  // extern "C"
