// gsb_debug.cu — test-only hooks of the C ABI: dense K1 records (gsb_debug_project), the
// binning + K3 sort on external projections (gsb_debug_bin_sort) and the production tile sorts
// (gsb_debug_tile_lists).  They allocate their own scratch and synchronise; never on a hot path.
#include "gsb_runtime.cuh"

using namespace gsb;

extern "C" {

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

gsb_status gsb_debug_tile_lists(const float* u, const float* v, const float* sxx, const float* syy,
                                const float* kappa, const uint32_t* zbits, const uint8_t* valid,
                                const int32_t* slot_ids, int32_t F, int64_t n, int32_t width, int32_t height,
                                int32_t variant, int32_t key_mode, int64_t* out_offsets, uint32_t* out_ids,
                                int64_t cap, int64_t* out_K, int32_t* out_variant, gsb_stream stream) {
  if (F < 1 || n < 0 || width < 1 || height < 1 || width > kMaxDim || height > kMaxDim || cap < 0 || !out_K ||
      !out_offsets || variant < 0 || variant > 5 || key_mode < 0 || key_mode > 2 ||
      (key_mode == 2 && variant != 1 && variant != 2) ||
      (n > 0 && (!u || !v || !sxx || !syy || !kappa || !zbits || !valid || !slot_ids)))
    return fail(GSB_ERR_INVALID_ARGUMENT, "bad debug_tile_lists arguments");
  if (n >= (int64_t)1 << 31) return fail(GSB_ERR_CAPACITY, "n >= 2^31");
  cudaStream_t st = (cudaStream_t)stream;
  const int tiles_x = (width + kTile - 1) / kTile;
  const int n_tiles = tiles_x * ((height + kTile - 1) / kTile);
  const int64_t stride = ((int64_t)n_tiles + 2 + 31) / 32 * 32;
  const int64_t vwords = (n + 31) / 32;
  // slot -> (creation id, body) and id -> slot, as gsb_create_scene lays them out
  std::vector<int32_t> hsid((size_t)n);
  if (n > 0 && cudaMemcpy(hsid.data(), slot_ids, sizeof(int32_t) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(GSB_ERR_CUDA, "debug_tile_lists: reading slot_ids");
  std::vector<int2> hids((size_t)n);
  std::vector<int> hinv((size_t)n, -1);
  for (int64_t j = 0; j < n; ++j) {
    const int id = hsid[j];
    if (id < 0 || id >= n || hinv[id] >= 0) return fail(GSB_ERR_INVALID_ARGUMENT, "slot_ids is not a permutation");
    hids[j] = make_int2(id, -1);
    hinv[id] = (int)j;
  }
  uint2* emit = nullptr; int* vcount = nullptr; int* hist = nullptr; uint32_t* off = nullptr;
  uint32_t* vbits = nullptr; uint64_t* fbase = nullptr; uint64_t* keys = nullptr; uint64_t* keys_alt = nullptr;
  uint32_t* sorted = nullptr; uint32_t* lists = nullptr; int2* d_ids = nullptr; int* d_inv = nullptr;
  uint32_t* d_long = nullptr;
  auto cleanup = [&]() {
    cudaFree(emit); cudaFree(vcount); cudaFree(hist); cudaFree(off); cudaFree(fbase); cudaFree(vbits);
    cudaFree(keys); cudaFree(keys_alt); cudaFree(sorted); cudaFree(lists); cudaFree(d_ids); cudaFree(d_inv);
    cudaFree(d_long);
  };
#define DBG_TRY(expr)                                                              \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      cleanup();                                                                   \
      return fail(GSB_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));          \
    }                                                                              \
  } while (0)
  DBG_TRY(dalloc(&d_ids, (size_t)std::max<int64_t>(n, 1)));
  DBG_TRY(dalloc(&d_inv, (size_t)std::max<int64_t>(n, 1)));
  if (n > 0) {
    DBG_TRY(cudaMemcpy(d_ids, hids.data(), sizeof(int2) * n, cudaMemcpyHostToDevice));
    DBG_TRY(cudaMemcpy(d_inv, hinv.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
  }
  DBG_TRY(dalloc(&emit, (size_t)F * std::max<int64_t>(n, 1)));
  DBG_TRY(dalloc(&vcount, (size_t)F));
  DBG_TRY(dalloc(&vbits, (size_t)F * std::max<int64_t>(vwords, 1)));
  DBG_TRY(dalloc(&hist, (size_t)F * stride));
  DBG_TRY(dalloc(&off, (size_t)F * stride));
  DBG_TRY(dalloc(&fbase, (size_t)F + 2));
  DBG_TRY(cudaMemsetAsync(vcount, 0, sizeof(int) * F, st));
  DBG_TRY(cudaMemsetAsync(hist, 0, sizeof(int) * F * stride, st));
  DBG_TRY(cudaMemsetAsync(off, 0, sizeof(uint32_t) * F * stride, st));
  launch_k1_external(u, v, sxx, syy, kappa, zbits, valid, n, 0, F, width, height, tiles_x, emit, vbits, vwords,
                     vcount, hist, stride, st);
  launch_k2_scan(hist, off, stride, F, n_tiles, fbase, nullptr, nullptr, 0, nullptr, nullptr, st);
  DBG_TRY(cudaGetLastError());
  std::vector<uint64_t> hfb(F + 2);
  std::vector<uint32_t> hoff((size_t)F * stride);
  DBG_TRY(cudaMemcpyAsync(hfb.data(), fbase, sizeof(uint64_t) * (F + 2), cudaMemcpyDeviceToHost, st));
  DBG_TRY(cudaMemcpyAsync(hoff.data(), off, sizeof(uint32_t) * hoff.size(), cudaMemcpyDeviceToHost, st));
  DBG_TRY(cudaStreamSynchronize(st));
  const uint64_t K = hfb[F];
  *out_K = (int64_t)K;
  if (K > (uint64_t)cap) {
    cleanup();
    return fail(GSB_ERR_CAPACITY, "K = %llu exceeds cap %lld", (unsigned long long)K, (long long)cap);
  }
  // the render's choices (gsb_render.cu, Pipeline::pass): long-list variant, split vs fused
  std::vector<uint32_t> hlong;   // K2a's long-list entries (frame << 16 | tile)
  for (int f = 0; f < F; ++f)
    for (int t = 0; t < n_tiles; ++t)
      if (hoff[(size_t)f * stride + t + 1] - hoff[(size_t)f * stride + t] > (uint32_t)kWarpSortCap)
        hlong.push_back(((uint32_t)f << 16) | (uint32_t)t);
  const uint64_t n_long = hlong.size();
  uint64_t n_vlong = 0;   // lists > kFusedSortCap: the render's packed-variant rule
  for (int f = 0; f < F; ++f)
    for (int t = 0; t < n_tiles; ++t)
      n_vlong += hoff[(size_t)f * stride + t + 1] - hoff[(size_t)f * stride + t] > (uint32_t)kFusedSortCap;
  int var = variant;
  if (var == 0) {
    const bool long_lists = n_vlong * 4 > (uint64_t)F * n_tiles;
    const bool split = split_k4() && K >= split_min_avg() * (uint64_t)F * n_tiles;
    var = split ? (long_lists ? 2 : 1) : (long_lists ? 4 : 3);
  }
  if (out_variant) *out_variant = var;
  DBG_TRY(dalloc(&keys, std::max<uint64_t>(K, 1)));
  DBG_TRY(dalloc(&keys_alt, std::max<uint64_t>(K, 1)));
  DBG_TRY(dalloc(&sorted, std::max<uint64_t>(K, 1)));
  DBG_TRY(dalloc(&lists, std::max<uint64_t>(K, 1)));
  const bool synth = key_mode == 2;   // slot keys + block masks (mask = slot & 15, K4a carries it)
  const bool slot_keys = key_mode == 0 || synth;
  ChunkArgs a{};
  a.rec = nullptr; a.emit = emit; a.ids = slot_keys ? nullptr : d_ids; a.n = n; a.vis_bits = vbits;
  a.vis_words = vwords; a.hist = hist; a.hist_stride = stride; a.off = off; a.frame_base = fbase;
  a.n_tiles = n_tiles; a.tiles_x = tiles_x; a.fs = 0; a.fe = F; a.key_base = 0; a.long_list = nullptr;
  a.keys = keys; a.keys_alt = keys_alt; a.sorted = sorted;
  if (synth) { a.mask_bits = kMaskBits; a.synth_mask = 1; }
  launch_k2_emit(a, st);
  CompositeArgs c{};
  c.rec = nullptr; c.n = n; c.off = off; c.frame_base = fbase; c.hist_stride = stride; c.sorted = sorted;
  c.keys = keys; c.keys_alt = keys_alt; c.key_base = 0; c.inv = d_inv; c.slot_base = 0;
  c.keys_internal_ids = slot_keys ? d_ids : nullptr;
  if (synth) c.key_shift = kMaskBits;
  c.fs = 0; c.fe = F; c.f0 = 0; c.width = width; c.height = height; c.tiles_x = tiles_x; c.n_tiles = n_tiles;
  if (var == 1 && n_long > 0) {       // the render's K4a: warp per short list + CTA per long list
    DBG_TRY(dalloc(&d_long, (size_t)n_long));
    DBG_TRY(cudaMemcpy(d_long, hlong.data(), sizeof(uint32_t) * n_long, cudaMemcpyHostToDevice));
  }
  if (var == 1) {
    c.long_list = d_long ? d_long : sorted;   // (non-null: selects the warp path)
    c.n_long = (uint32_t)n_long;
  }
  if (var <= 2 || var == 5) {
    launch_k4a_sort(c, var == 2, st);   // K4a: slots in (bits(z), id) order -> sorted
  } else {
    c.dbg_lists = sorted;               // fused K4: its in-CTA sort exports the slot lists
    launch_k4_composite(c, var == 4, st);
  }
  DBG_TRY(cudaGetLastError());
  std::vector<uint32_t> hs((size_t)K);
  if (K > 0) DBG_TRY(cudaMemcpyAsync(hs.data(), sorted, sizeof(uint32_t) * K, cudaMemcpyDeviceToHost, st));
  DBG_TRY(cudaStreamSynchronize(st));
  if (synth)   // every entry must carry its own slot's mask; a mismatch reads as an invalid id
    for (uint64_t k = 0; k < K; ++k) hs[k] = ((hs[k] >> kMaskBits) & 15u) == (hs[k] & 15u) ? hs[k] >> kMaskBits : 0xfffffffeu;
  for (uint64_t k = 0; k < K; ++k) hs[k] = hs[k] < (uint64_t)n ? (uint32_t)hids[hs[k]].x : 0xffffffffu;
  if (K > 0) DBG_TRY(cudaMemcpyAsync(out_ids, hs.data(), sizeof(uint32_t) * K, cudaMemcpyHostToDevice, st));
  std::vector<int64_t> ho((size_t)F * (n_tiles + 1));
  for (int f = 0; f < F; ++f)
    for (int t = 0; t <= n_tiles; ++t) ho[(size_t)f * (n_tiles + 1) + t] = (int64_t)hfb[f] + hoff[(size_t)f * stride + t];
  DBG_TRY(cudaMemcpyAsync(out_offsets, ho.data(), sizeof(int64_t) * ho.size(), cudaMemcpyHostToDevice, st));
  DBG_TRY(cudaStreamSynchronize(st));
  cleanup();
  return GSB_OK;
#undef DBG_TRY
}

}  // extern "C"
