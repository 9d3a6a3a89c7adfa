// gsb_kernels.cuh — launch interface between the host runtime (gsb_api.cu) and K0-K4.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "gsb_common.cuh"

namespace gsb {

constexpr int kFusedSortCap = 1024;  // tile lists up to this length are sorted in K4 smem (8 CTAs/SM);
                                     // chunks with many longer lists use a 4x variant
#ifndef GSB_WARP_SORT_CAP
#define GSB_WARP_SORT_CAP 512
#endif
constexpr int kWarpSortCap = GSB_WARP_SORT_CAP;  // K4a: lists up to this length are sorted by one warp
                                                 // each; K2a lists the longer ones (long_list) for a CTA each

constexpr int kDbgRecFloats = 16;   // gsb_debug_project record (include/gsb.h)

// Kernel attributes and launch geometry are per DEVICE: caches keyed by the current device.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
// cudaFuncSetAttribute(max dynamic smem) once per (kernel, device); `done` is the caller's
// static [kMaxDevices] table.  Returns the CUDA error (also left for cudaGetLastError, so the
// caller's launch check reports it); the caller skips its launch on failure.
template <typename Kernel>
inline cudaError_t ensure_smem_attr(Kernel* fn, int bytes, int* done) {
  const int dev = current_device();
  if (dev >= 0 && dev < kMaxDevices && done[dev] == bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && dev >= 0 && dev < kMaxDevices) done[dev] = bytes;
  return e;
}

struct K1Args {
  // template (K5: shared read-only buffer, one copy for every env)
  const float4* g_mean;
  const float4* g_L0;
  const float4* g_L1;
  const float4* g_L2;
  const float4* g_sh;
  const int2* g_ids;   // (creation index = id, body) per internal index
  int64_t n;           // Gaussians of this launch (the pointers may start inside the template)
  int64_t sh_stride;   // SH plane stride = template size N
  // per-frame transforms (K0)
  const float4* table;
  const FrameCam* cams;
  int nb1;
  // chunk
  int f0;          // first frame of the chunk
  int n_frames;    // E
  int width, height, tiles_x;
  float near_plane, far_plane;
  // outputs
  float4* rec;     // [E][N][3] records at the internal index, nullptr for debug-only launches
  uint2* emit;     // [E][N] (bits(z), rect) for the key emission
  uint8_t* trim;   // [E][N] or nullptr: K4b block-mask trims (bit 0: left 8 columns of the rect's
                   // first tile column unreachable, 1: right 8 of the last, 2: top 8 rows of the
                   // first tile row, 3: bottom 8 of the last), from the conservative R8 box
  uint32_t* vis_bits;  // [E][vis_words] visibility ballot of each warp (32 internal indices)
  int64_t vis_words;   // ceil(N / 32)
  int* vcount;     // [E] visible pairs (statistics)
  int* hist;       // [E][hist_stride]
  int64_t hist_stride;
  // debug (dense) outputs, nullptr unless gsb_debug_project
  float* dbg_rec;
  uint32_t* dbg_zbits;
  uint8_t* dbg_valid;
};

struct ChunkArgs {
  const float4* rec;      // [E][N][3]
  const uint2* emit;      // [E][N] (bits(z), rect) of the visible (frame, Gaussian) pairs
  const int2* ids;        // template (id, body) of the launch's range, or nullptr: id = index
  int64_t n;              // record stride per frame (= N)
  const uint32_t* vis_bits;  // [E][vis_words]
  int64_t vis_words;
  int* hist;              // [E][hist_stride]  (counts; reused as emission cursors)
  int64_t hist_stride;
  uint32_t* off;          // [E][hist_stride] exclusive tile offsets within the frame, [T] = K_f
  uint64_t* frame_base;   // [E+1] exclusive prefix of K_f over the chunk's frames
  int n_tiles, tiles_x;
  int fs, fe;             // frame range [fs, fe) of this pass (relative to the chunk)
  uint64_t key_base;      // frame_base[fs]: keys of this pass start at key index 0
  const uint32_t* long_list;  // (frame << 16 | tile) of lists longer than kFusedSortCap (K3), or
                              // nullptr: K3 sorts every list (gsb_debug_bin_sort)
  uint64_t* keys;         // [cap]   (zbits << 32) | id
  uint64_t* keys_alt;     // [cap]   scratch for oversize segments
  uint32_t* sorted;       // [cap]   sorted ids of the lists K3 sorted
  const int* overflow;    // GSB_FLAG_FIXED_PLAN: the chunk's flag (keys beyond capacity: skip), or nullptr
  // K4b block masks (slot keys only): key low word = slot << kMaskBits | mask of the 8x8 blocks of
  // the tile the record can reach (from K1's trims); 0 = off.  synth_mask (debug hook):
  // mask = slot & 15
  int mask_bits;
  int synth_mask;
  const uint8_t* trim;    // [E][N] K1's block-mask trims (mask_bits without synth_mask)
};
constexpr int kMaskBits = 4;

struct CompositeArgs {
  const float4* rec;
  int64_t n;
  const uint32_t* off;
  const uint64_t* frame_base;
  int64_t hist_stride;
  uint32_t* sorted;         // sorted ids of segments longer than kFusedSortCap
  const uint64_t* keys;     // unsorted keys (K2b); K4 sorts every tile list itself
  uint64_t* keys_alt;       // scratch twin of keys for the HBM sort of long lists
  const int* inv;           // id -> internal index; record slot = inv[id] - slot_base
  int slot_base;            // first internal index of the launch's Gaussian range
  // static-camera merge (gsb_render_static, §8(f) row 2), all nullptr otherwise: the
  // pre-binned background list of (camera, tile) is merged with the frame's robot list
  const uint64_t* bg_off;   // [C][T+1] absolute offsets into bg_keys / bg_rec
  const uint64_t* bg_keys;  // sorted (zbits << 32 | id) of each background list
  const float4* bg_rec;     // [K_bg][3] records (u,v,p,q | r,log2o,ex,ey | rgb,z) in list order
  int n_static_cams;
  uint32_t* qpos_g;         // [cap] merged positions of robot entries of lists sorted in HBM
  const uint64_t* bg_cum;   // [C+1] prefix of the background list sizes over cameras (split path)
  uint64_t key_base;
  int fs, fe;             // relative frames of this pass
  int f0;                 // absolute frame index of chunk frame 0
  int width, height, tiles_x, n_tiles;
  float bg0, bg1, bg2;
  float* out_rgb;         // [F][3][H][W]
  float* out_depth;       // [F][H][W] or nullptr
  float* out_alpha;
  int32_t* out_n_eval;
  unsigned long long* stat_pairs;  // nullptr unless STATS: [0] evaluated pairs P, [1] terminated pixels
  float* score_sum;         // [N] by internal index, nullptr unless GSB_FLAG_SCORES (reading R30)
  uint32_t* score_max;      // [N] float bits of the max weight
  // observation epilogue (gsb_render_obs, §8(f) row 4, reading R31); obs_rgb8 == nullptr: fp32 outputs
  uint8_t* obs_rgb8;        // [F][3][H][W]
  uint16_t* obs_depth16;    // [F][H][W] IEEE half bits, or nullptr (then out_depth fp32, if set)
  const float* obs_dr;      // [F][4] (gain, contrast, brightness, noise_std) per frame, or nullptr
  uint32_t obs_seed, obs_step;
  int64_t obs_frame_offset; // global index of this call's frame 0 (noise streams)
  // K4a: keys carry the record slot (internal index - slot_base) instead of the creation id
  // (K2b with ids = nullptr); equal-depth runs are then re-ordered by the creation id ids[slot].x
  // so the order is still (bits(z), id) of reading R10, and no id -> slot gather is needed
  const int2* keys_internal_ids;   // template (id, body) of the launch's range, or nullptr
  // K4b block masks: with key_shift = kMaskBits the key's low word (and each sorted entry) is
  // (slot << 4 | mask), mask bit b = "the record can reach 8x8 block b of the tile" (K2b); 0 = off
  int key_shift;
  // lists longer than kWarpSortCap of this chunk ((frame << 16 | tile), from K2a): the split path's
  // K4a sorts short lists one warp per tile and these with a CTA each; nullptr = CTA per tile
  const uint32_t* long_list;
  uint32_t n_long;
  const uint32_t* n_long_dev;   // GSB_FLAG_FIXED_PLAN: long-list count read on the device (K2a's)
  const int* overflow;          // GSB_FLAG_FIXED_PLAN: skip the chunk (keys beyond capacity), or nullptr
  // gsb_debug_tile_lists only: the fused K4 writes each tile's sorted slot list here (at the
  // list's key offset) and returns before compositing; nullptr in every render
  uint32_t* dbg_lists;
};

constexpr int kMaxRigCams = 16;  // cameras per env that can be body-attached (gsb_render_rig)

// K0 inputs: poses read with strides (physics-buffer ingest); cam_x = world->camera, or
// body->camera for cameras with cam_body[c] >= 0 (reading R29)
struct K0Rig {
  const float* poses;
  int64_t env_stride, body_stride;  // floats
  const float* intr;
  const float* cam_x;
  int cams_shared;  // intr / cam_x hold one [C] camera set shared by all envs
  int cam_body[kMaxRigCams];
};

// ---------------------------------------------------------------- LiDAR (reading R32)
constexpr int kLidarRecQuads = 5;   // float4s per LiDAR record
struct LidarL1Args {
  const float4 *g_mean, *g_L0, *g_L1, *g_L2;
  const int2* g_ids;
  int64_t n;            // Gaussians (record stride per frame)
  int64_t np;           // n rounded up to 32: emission index of the seam part of Gaussian i = np + i
  const float4* table;  // K0 per-(frame, body) transforms, frame = (env, sensor)
  int nb1;
  int f0, n_frames;
  float near_plane, far_plane;
  // cell grid: azimuth window [az0, az0 + az_span), elevation window [el0, el0 + n_el / el_inv)
  float az0, az_span, az_inv, el0, el_inv;
  int n_az, n_el;
  float4* rec;          // [E][n][5]: A row 0 | m0, A row 1 | m1, A row 2 | m2, (x, c), (log2 o, rho, -, -)
                        // A = whitening of the sensor-frame Sigma scaled by sqrt(log2(e)/2), m = A x,
                        // c = cone-test threshold of the ray cull (d.x >= c)
  uint2* emit;          // [E][2 np] (bits(rho), cell rect)
  uint32_t* vis_bits;   // [E][vis_words = 2 np / 32]
  int64_t vis_words;
  int* vcount;          // [E]
  int* hist;            // [E][hist_stride] cell counts
  int64_t hist_stride;
};

struct LidarL4Args {
  const float4* rec;
  int64_t n;
  const uint32_t* off;          // [E][hist_stride] cell offsets within the frame
  const uint64_t* frame_base;   // [E+1]
  int64_t hist_stride;
  const uint32_t* sorted;       // record slots of every (frame, cell) list in (bits(rho), id) order
                                // (K4a): internal index i, or np + i for a seam copy
  int64_t np;
  const float4* rays;           // [R] (dx, dy, dz, bits(original ray index)), grouped by cell
  const int4* items;            // (cell, first ray, ray count <= 32, 0)
  int n_items, f0, n_frames, n_rays;
  float* out_range;             // [F][R]
  float* out_alpha;             // [F][R] or nullptr
};

void launch_kl1(const LidarL1Args& a, cudaStream_t s);

// K6: reading R33 motion blur + reading R31 encoding over rendered fp32 frames (gsb_obs_encode)
struct EncodeArgs {
  const float* rgb;       // [F][3][H][W]
  const float* depth;     // [F][H][W] or nullptr
  const int32_t* blur;    // [F][2] (bx, by) or nullptr
  const float* dr;        // [F][4] or nullptr
  uint32_t seed, step;
  int64_t frame_offset;   // global frame index of frame 0 (noise counters)
  int n_frames, width, height;
  uint8_t* out_rgb8;      // [F][3][H][W]
  uint16_t* out_depth16;  // fp16 bits, or nullptr
  float* out_depth32;     // or fp32 copy, or nullptr
};
void launch_k6_encode(const EncodeArgs& a, cudaStream_t s);
void launch_kl4(const LidarL4Args& a, cudaStream_t s);

void launch_k0(const K0Rig& rig, int n_frames, int n_cams, int n_bodies, int width, int height,
               float4* table, FrameCam* cams, cudaStream_t s);
void launch_k1(const K1Args& a, int sh_degree, cudaStream_t s);

// K1 variant for gsb_debug_bin_sort: records from externally supplied fp32 projections
void launch_k1_external(const float* u, const float* v, const float* sxx, const float* syy,
                        const float* kappa, const uint32_t* zbits, const uint8_t* valid,
                        int64_t n, int f0, int n_frames, int width, int height, int tiles_x,
                        uint2* emit, uint32_t* vis_bits, int64_t vis_words, int* vcount, int* hist,
                        int64_t hist_stride, cudaStream_t s);

// off[f][T] = K_f, off[f][T+1] = longest tile list of frame f; frame_base[E] = total keys,
// frame_base[E+1] = longest tile list of the chunk
// Lists longer than long_thresh are appended to long_list (frame << 16 | tile), counted in
// long_count[0]; long_count[1] counts those longer than kFusedSortCap (both may be null).
// host_mapped (device view of mapped pinned memory, may be null) receives
// [frame_base[0..E+1], vcount[0..E), long_count] as u64.
// overflow (nullable, GSB_FLAG_FIXED_PLAN): the chunk's flag, set to (total keys > key_cap); a
// set flag also sets *sticky
void launch_k2_scan(int* hist, uint32_t* off, int64_t hist_stride, int n_frames, int n_tiles,
                    uint64_t* frame_base, uint32_t* long_list, uint32_t* long_count, int long_thresh,
                    const int* vcount, uint64_t* host_mapped, cudaStream_t s, int* overflow = nullptr,
                    int* sticky = nullptr, uint64_t key_cap = 0);
void launch_k2_emit(const ChunkArgs& a, cudaStream_t s);
void launch_k3_sort(const ChunkArgs& a, uint32_t n_long, cudaStream_t s);
// gather K3-sorted background lists (ids in `sorted`) into list-ordered keys + 3-quad records
void launch_k3_prebin_gather(const uint32_t* sorted, const uint64_t* frame_base, const float4* rec, int64_t n,
                             const int* inv, int n_frames, uint64_t max_keys, uint64_t* bg_keys, float4* bg_rec,
                             cudaStream_t s);
// long_lists: use the variant with a 4x larger shared-memory sort (fewer CTAs per SM)
void launch_k4_composite(const CompositeArgs& a, bool long_lists, cudaStream_t s);
// split path (plain / observation renders): K4a tile sort into a.sorted, then K4b persistent
// per-warp compositing; counter = one int of device scratch
// the K4a variants the split path picks by default sort keys with block masks (key_shift)
bool k4a_masks_supported();
void launch_k4a_sort(const CompositeArgs& a, bool long_lists, cudaStream_t s);
void launch_k4b_blend(const CompositeArgs& a, int* counter, cudaStream_t s);
void launch_k4_scores_export(const float* wsum, const uint32_t* wmax, const int2* ids, int64_t n, float* out_sum,
                             float* out_max, cudaStream_t s);

}  // namespace gsb
