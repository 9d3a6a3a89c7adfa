// k2_bin.cu — K2: tile-intersection offsets (per-frame exclusive scan of the tile histogram
// built by K1) and emission of one 64-bit key per (visible Gaussian, overlapped tile).
//
// 3DGS tile binning [3DGS-conv, cited P:212]; keys are unique (reading R10):
//   key = bits(z_f32) << 32 | id          (id = creation index of the Gaussian)
// and land directly in their (frame, tile) bucket, so K3 only sorts within a bucket.
// The tile coordinate is implied by the bucket; the frame by the chunk's frame_base.
#include "gsb_common.cuh"
#include "gsb_kernels.cuh"

namespace gsb {

constexpr int kScanThreads = 1024;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// per-frame exclusive scan of hist[f][0..T) -> off[f][0..T]; hist is zeroed (becomes the
// emission cursor).  One block per frame.
__global__ void __launch_bounds__(kScanThreads) k2_scan_tiles(int* __restrict__ hist,
                                                              uint32_t* __restrict__ off,
                                                              int64_t stride, int n_tiles,
                                                              uint32_t* __restrict__ long_list,
                                                              uint32_t* __restrict__ long_count,
                                                              int long_thresh) {
  __shared__ uint32_t wsum[kScanThreads / 32];
  __shared__ uint32_t carry_s, max_s;
  const int f = blockIdx.x;
  int* h = hist + (size_t)f * stride;
  uint32_t* o = off + (size_t)f * stride;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_s = 0, max_s = 0;
  __syncthreads();
  uint32_t mx = 0;
  for (int base = 0; base < n_tiles; base += kScanThreads) {
    const int t = base + tid;
    const uint32_t x = t < n_tiles ? (uint32_t)h[t] : 0u;
    mx = max(mx, x);
    const uint32_t inc = warp_incl_scan(x);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const uint32_t w = lane < kScanThreads / 32 ? wsum[lane] : 0u;
      const uint32_t wi = warp_incl_scan(w);
      if (lane < kScanThreads / 32) wsum[lane] = wi - w;
    }
    __syncthreads();
    const uint32_t carry = carry_s;
    if (t < n_tiles) {
      o[t] = carry + wsum[warp] + inc - x;
      h[t] = 0;
      if (long_list && x > (uint32_t)long_thresh) {
        long_list[atomicAdd(long_count, 1u)] = ((uint32_t)f << 16) | (uint32_t)t;
        if (x > (uint32_t)kFusedSortCap) atomicAdd(long_count + 1, 1u);   // the packed-variant rule
      }
    }
    __syncthreads();
    if (tid == kScanThreads - 1) carry_s = carry + wsum[warp] + inc;
    __syncthreads();
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) atomicMax(&max_s, mx);
  __syncthreads();
  if (tid == 0) {
    o[n_tiles] = carry_s;
    o[n_tiles + 1] = max_s;
  }
}

// frame_base[0..E] = exclusive prefix of K_f = off[f][T] (single block).  When `host` is set
// (mapped pinned memory) the values the host needs to size the binning — frame bases, longest
// list, visible counts, long-list count — are also written straight to host memory, so the
// readback never queues behind output copies on the copy engine.
__global__ void __launch_bounds__(kScanThreads) k2_scan_frames(
    const uint32_t* __restrict__ off, int64_t stride, int n_tiles, int n_frames, uint64_t* __restrict__ frame_base,
    const int* __restrict__ vcount, const uint32_t* __restrict__ long_count, volatile uint64_t* __restrict__ host,
    int* __restrict__ overflow, int* __restrict__ sticky, uint64_t key_cap) {
  // block-wide exclusive scan of the frames' key counts, kScanThreads frames at a time (a single
  // thread walking 1024 frames cost 0.4 ms per C4 chunk)
  __shared__ unsigned long long wsum[kScanThreads / 32];
  __shared__ unsigned long long carry_s, mx_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry_s = 0ull, mx_s = 0ull;
  __syncthreads();
  unsigned long long mx = 0ull;
  for (int base = 0; base < n_frames; base += kScanThreads) {
    const int f = base + tid;
    const unsigned long long x = f < n_frames ? (unsigned long long)off[(size_t)f * stride + n_tiles] : 0ull;
    if (f < n_frames) mx = max(mx, (unsigned long long)off[(size_t)f * stride + n_tiles + 1]);
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = wsum[lane];
      unsigned long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      wsum[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long excl = carry_s + wsum[warp] + inc - x;
    if (f < n_frames) {
      frame_base[f] = excl;
      if (host) {
        host[f] = excl;
        host[n_frames + 2 + f] = vcount ? (uint64_t)vcount[f] : 0ull;
      }
    }
    __syncthreads();
    if (tid == kScanThreads - 1) carry_s = excl + x;
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) atomicMax(&mx_s, mx);
  if (host) __threadfence_system();   // this thread's mapped-memory writes
  __syncthreads();
  if (tid != 0) return;
  const uint64_t acc = carry_s;
  frame_base[n_frames] = acc;
  frame_base[n_frames + 1] = mx_s;
  if (overflow) {   // fixed plan: one pass per chunk; the chunk is skipped when it does not fit
    *overflow = acc > key_cap ? 1 : 0;            // this chunk (its slot's flag)
    if (acc > key_cap) *sticky = 1;               // read and reset by gsb_get_overflow
  }
  if (host) {
    host[n_frames] = acc;
    host[n_frames + 1] = mx_s;
    host[2 * n_frames + 2] = long_count ? (uint64_t)long_count[0] : 0ull;
    host[2 * n_frames + 3] = long_count ? (uint64_t)long_count[1] : 0ull;
    __threadfence_system();
  }
}

void launch_k2_scan(int* hist, uint32_t* off, int64_t hist_stride, int n_frames, int n_tiles,
                    uint64_t* frame_base, uint32_t* long_list, uint32_t* long_count, int long_thresh,
                    const int* vcount, uint64_t* host_mapped, cudaStream_t s, int* overflow, int* sticky,
                    uint64_t key_cap) {
  k2_scan_tiles<<<n_frames, kScanThreads, 0, s>>>(hist, off, hist_stride, n_tiles, long_list, long_count,
                                                  long_thresh);
  k2_scan_frames<<<1, kScanThreads, 0, s>>>(off, hist_stride, n_tiles, n_frames, frame_base, vcount, long_count,
                                  host_mapped, overflow, sticky, key_cap);
}

// ------------------------------------------------------------------------------ emission
// One thread per (frame, internal index); warps with no visible Gaussian (ballot word 0) exit
// at once.  Keys of a warp's Gaussians that land in the same tile share one cursor atomic (the
// template is Morton-ordered, so a warp's Gaussians overlap the same tiles); rects with more
// than kBigRect tiles are emitted by the whole warp cooperatively.
#ifndef GSB_K2B_BREAK
#define GSB_K2B_BREAK 0   // 1: warp-uniform early exit from the unrolled rounds (A/B)
#endif
__global__ void __launch_bounds__(256) k2_emit(ChunkArgs a) {
  __shared__ uint32_t tile_scratch[8][32];   // per-warp union-box counts
  const unsigned FULL = 0xffffffffu;
  if (a.overflow && *a.overflow) return;   // fixed plan: chunk beyond the key capacity
  const int fl = a.fs + blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) >= a.n) return;  // whole warp past N
  const unsigned word = a.vis_bits[(size_t)fl * a.vis_words + (i >> 5)];
  if (word == 0) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const bool has = (word >> lane) & 1u;
  uint32_t rect = 0, zb = 0, id = 0;
  uint32_t trim = 0;   // block masks: K1's trims of this pair
  if (has) {
    const uint2 er = __ldg(a.emit + (size_t)fl * a.n + i);
    zb = er.x;
    rect = er.y;
    id = a.ids ? (uint32_t)__ldg(&a.ids[i].x) : (uint32_t)i;
    if (a.mask_bits && !a.synth_mask) trim = __ldg(a.trim + (size_t)fl * a.n + i);
  }
  // unique (reading R10); with block masks the low word is (id << 4 | mask of the tile)
  const uint64_t key = ((uint64_t)zb << 32) | (uint64_t)(a.mask_bits ? id << kMaskBits : id);
  // the key for tile (tx, ty): + the 4-bit mask of the tile's 8x8 blocks (bit 2 by + bx) the
  // record can reach: all four, less the half-tile borders K1 trimmed at the rect's edges
  // (debug hook: mask = slot & 15)
  int* cur = a.hist + (size_t)fl * a.hist_stride;
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  uint64_t* keys = a.keys + (a.frame_base[fl] - a.key_base);
  const int tx0 = rect & 0xff, tx1 = (rect >> 8) & 0xff, ty0 = (rect >> 16) & 0xff, ty1 = rect >> 24;
  auto key_at = [&](int tx, int ty) -> uint64_t {
    if (!a.mask_bits) return key;
    if (a.synth_mask) return key | (id & 15u);
    uint32_t m = 15u;
    if (tx == tx0 && (trim & 1u)) m &= ~5u;    // left column of blocks (0, 2)
    if (tx == tx1 && (trim & 2u)) m &= ~10u;   // right column (1, 3)
    if (ty == ty0 && (trim & 4u)) m &= ~3u;    // top row (0, 1)
    if (ty == ty1 && (trim & 8u)) m &= ~12u;   // bottom row (2, 3)
    return key | m;
  };
  const int nt = has ? (tx1 - tx0 + 1) * (ty1 - ty0 + 1) : 0;
  const bool big = nt > kBigRect;
  const bool part = nt > 0 && !big;
  // union box of the warp's rects <= 32 tiles (the usual case): every key's rank inside its
  // (warp, tile) group from a shared atomic, then ONE returning global atomic per distinct tile,
  // all issued by one instruction (lane j: box tile j) — no serial rounds of atomic latency
  const UnionBox ub = GSB_UNION_BOX ? warp_union_box(part, tx0, tx1, ty0, ty1) : UnionBox{0, 0, 0, 64};
  const int rounds = __reduce_max_sync(FULL, part ? nt : 0);
  if (ub.n > 0 && ub.n <= 32) {
    uint32_t* sc = tile_scratch[threadIdx.x >> 5];
    sc[lane] = 0u;
    __syncwarp();
    uint32_t rk[kBigRect];
    int tx = tx0, ty = ty0;
#if GSB_K2B_BREAK
#pragma unroll
    for (int r = 0; r < kBigRect; ++r) {
      if (r >= rounds) break;   // warp-uniform
      if (part && r < nt) {
        rk[r] = atomicAdd(&sc[(ty - ub.y0) * ub.w + (tx - ub.x0)], 1u);
        if (++tx > tx1) { tx = tx0; ++ty; }
      }
    }
#else
#pragma unroll
    for (int r = 0; r < kBigRect; ++r) {
      if (r < nt && part) {
        rk[r] = atomicAdd(&sc[(ty - ub.y0) * ub.w + (tx - ub.x0)], 1u);
        if (++tx > tx1) { tx = tx0; ++ty; }
      }
    }
#endif
    __syncwarp();
    const uint32_t c = sc[lane];
    uint32_t base = 0u;
    if (lane < ub.n && c) base = (uint32_t)atomicAdd(cur + ub.tile_of(lane, a.tiles_x), (int)c);
    tx = tx0; ty = ty0;
#if GSB_K2B_BREAK
#pragma unroll
    for (int r = 0; r < kBigRect; ++r) {
      if (r >= rounds) break;   // warp-uniform
      const bool act = part && r < nt;
      const uint32_t b = __shfl_sync(FULL, base, act ? (ty - ub.y0) * ub.w + (tx - ub.x0) : 0);
      if (act) {
        keys[off[ty * a.tiles_x + tx] + b + rk[r]] = key_at(tx, ty);
        if (++tx > tx1) { tx = tx0; ++ty; }
      }
    }
#else
#pragma unroll
    for (int r = 0; r < kBigRect; ++r) {
      if (r < rounds) {
        const int j = (ty - ub.y0) * ub.w + (tx - ub.x0);
        const uint32_t b = __shfl_sync(FULL, base, part && r < nt ? j : 0);
        if (part && r < nt) keys[off[ty * a.tiles_x + tx] + b + rk[r]] = key_at(tx, ty);
        if (++tx > tx1) { tx = tx0; ++ty; }
      }
    }
#endif
  }
  int tx = tx0, ty = ty0;  // this lane's r-th tile, stepped row-major (no division)
  for (int r = 0; r < (ub.n > 32 ? rounds : 0); ++r) {
    const bool act = part && r < nt;
    const int t = act ? ty * a.tiles_x + tx : -1 - lane;
    const unsigned peers = __match_any_sync(FULL, t);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (act && lane == leader) base = atomicAdd(cur + t, __popc(peers));
    base = __shfl_sync(FULL, base, leader);
    if (act) keys[off[t] + base + __popc(peers & lanemask_lt())] = key_at(tx, ty);
    if (++tx > tx1) { tx = tx0; ++ty; }
  }
  unsigned bm = __ballot_sync(FULL, big);
  while (bm) {
    const int j = __ffs(bm) - 1;
    bm &= bm - 1;
    const uint32_t rj = __shfl_sync(FULL, rect, j);
    // a big rect (> kBigRect tiles): every block of each tile (conservative)
    const uint64_t kj = __shfl_sync(FULL, key, j) |
                        (a.mask_bits ? (a.synth_mask ? (uint64_t)(__shfl_sync(FULL, id, j) & 15u) : 15ull) : 0ull);
    const int jx0 = rj & 0xff, jx1 = (rj >> 8) & 0xff, jy0 = (rj >> 16) & 0xff, jy1 = rj >> 24;
    for (int y = jy0; y <= jy1; ++y)
      for (int x = jx0 + lane; x <= jx1; x += 32) {
        const int t = y * a.tiles_x + x;
        keys[off[t] + atomicAdd(cur + t, 1)] = kj;
      }
  }
}

void launch_k2_emit(const ChunkArgs& a, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0 || a.n == 0) return;
  dim3 grid((unsigned)((a.n + 255) / 256), (unsigned)nf);
  k2_emit<<<grid, 256, 0, s>>>(a);
}

// ------------------------------------------------- records from external fp32 projections
__global__ void __launch_bounds__(128) k1_external(const float* __restrict__ u, const float* __restrict__ v,
                                                   const float* __restrict__ sxx, const float* __restrict__ syy,
                                                   const float* __restrict__ kappa,
                                                   const uint32_t* __restrict__ zbits,
                                                   const uint8_t* __restrict__ valid, int64_t n, int f0,
                                                   int n_frames, int width, int height, int tiles_x,
                                                   uint2* __restrict__ emit, uint32_t* __restrict__ vis_bits,
                                                   int64_t vis_words, int* __restrict__ vcount,
                                                   int* __restrict__ hist, int64_t hist_stride) {
  __shared__ uint32_t tile_scratch[4][32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = i < n;
  for (int fl = 0; fl < n_frames; ++fl) {
    const size_t o = (size_t)(f0 + fl) * n + (in ? i : 0);
    int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1;
    bool vis = false;
    if (in && valid[o])
      vis = r9_rect(u[o], v[o], sxx[o], syy[o], kappa[o], width, height, tx0, tx1, ty0, ty1);
    const unsigned bal = __ballot_sync(0xffffffffu, vis);
    if ((threadIdx.x & 31) == 0 && i < n) {
      vis_bits[(size_t)fl * vis_words + (i >> 5)] = bal;
      if (bal) atomicAdd(vcount + fl, __popc(bal));
    }
    const uint32_t rect = pack_rect(tx0, tx1, ty0, ty1);
    if (vis) emit[(size_t)fl * n + i] = make_uint2(zbits[o], rect);
    warp_tile_count(vis, rect, tiles_x, hist + (size_t)fl * hist_stride, tile_scratch[threadIdx.x >> 5]);
  }
}

void launch_k1_external(const float* u, const float* v, const float* sxx, const float* syy,
                        const float* kappa, const uint32_t* zbits, const uint8_t* valid,
                        int64_t n, int f0, int n_frames, int width, int height, int tiles_x,
                        uint2* emit, uint32_t* vis_bits, int64_t vis_words, int* vcount, int* hist,
                        int64_t hist_stride, cudaStream_t s) {
  if (n == 0) return;
  k1_external<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(u, v, sxx, syy, kappa, zbits, valid, n, f0,
                                                          n_frames, width, height, tiles_x, emit, vis_bits,
                                                          vis_words, vcount, hist, hist_stride);
}

}  // namespace gsb
