// k3_sort.cu — K3: segmented radix sort for the tile lists that do not fit K4's fused
// shared-memory sort (and for every list in gsb_debug_bin_sort).  One CTA per (frame, tile)
// segment; lists up to kSmemCap keys are sorted in shared memory, longer ones ping-pong
// between the key buffer and its scratch twin in HBM with the same code (gsb_sort.cuh).
#include <algorithm>

#include "gsb_common.cuh"
#include "gsb_kernels.cuh"
#include "gsb_sort.cuh"

namespace gsb {

constexpr int kSmemCap = 4096;
constexpr int kSortThreads = 256;

__global__ void __launch_bounds__(kSortThreads) k3_sort(ChunkArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortShared<kSortThreads>& sm = *reinterpret_cast<SortShared<kSortThreads>*>(smem_raw);
  uint64_t* sa = reinterpret_cast<uint64_t*>(smem_raw + sizeof(SortShared<kSortThreads>));
  uint64_t* sb = sa + kSmemCap;

  int fl, t;
  if (a.long_list) {  // render path: only the lists too long for K4's fused sort
    const uint32_t e = a.long_list[blockIdx.x];
    fl = (int)(e >> 16);
    t = (int)(e & 0xffffu);
    if (fl < a.fs || fl >= a.fe) return;
  } else {
    fl = a.fs + blockIdx.x / a.n_tiles;
    t = blockIdx.x % a.n_tiles;
  }
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  const uint64_t start = a.frame_base[fl] - a.key_base + off[t];
  const int n = (int)(off[t + 1] - off[t]);
  if (n == 0) return;
  if (n == 1) {
    if (threadIdx.x == 0) a.sorted[start] = (uint32_t)a.keys[start];
    return;
  }
  if (n <= kSmemCap) {
    for (int e = threadIdx.x; e < n; e += kSortThreads) sa[e] = a.keys[start + e];
    __syncthreads();
    const bool in_b = segment_sort(sa, sb, n, sm);
    const uint64_t* r = in_b ? sb : sa;
    for (int e = threadIdx.x; e < n; e += kSortThreads) a.sorted[start + e] = (uint32_t)r[e];
  } else {
    uint64_t* ga = a.keys + start;
    uint64_t* gb = a.keys_alt + start;
    const bool in_b = segment_sort(ga, gb, n, sm);
    __syncthreads();
    const uint64_t* r = in_b ? gb : ga;
    for (int e = threadIdx.x; e < n; e += kSortThreads) a.sorted[start + e] = (uint32_t)r[e];
  }
}

// gsb_prebin_static: background lists of the C static cameras, K3-sorted, gathered into list
// order — keys (zbits << 32 | id) for K4's merge ranks and the 48 B of record K4 stages.
__global__ void __launch_bounds__(256) k3_prebin_gather(const uint32_t* __restrict__ sorted,
                                                        const uint64_t* __restrict__ frame_base,
                                                        const float4* __restrict__ rec, int64_t n,
                                                        const int* __restrict__ inv,
                                                        uint64_t* __restrict__ bg_keys,
                                                        float4* __restrict__ bg_rec) {
  const int f = blockIdx.y;
  const uint64_t b = frame_base[f], K = frame_base[f + 1] - b;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < K; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = sorted[b + e];
    const float4* r = rec + ((size_t)f * n + (uint32_t)inv[id]) * kRecQuads;
    const float4 q0 = r[0], q1 = r[1], q2 = r[2];
    bg_keys[b + e] = ((uint64_t)__float_as_uint(q2.w) << 32) | id;
    float4* o = bg_rec + (b + e) * 3;
    o[0] = q0;
    o[1] = q1;
    o[2] = q2;
  }
}

void launch_k3_prebin_gather(const uint32_t* sorted, const uint64_t* frame_base, const float4* rec, int64_t n,
                             const int* inv, int n_frames, uint64_t max_keys, uint64_t* bg_keys, float4* bg_rec,
                             cudaStream_t s) {
  if (n_frames <= 0 || max_keys == 0) return;
  const unsigned gx = (unsigned)std::min<uint64_t>((max_keys + 255) / 256, 4096);
  k3_prebin_gather<<<dim3(gx, (unsigned)n_frames), 256, 0, s>>>(sorted, frame_base, rec, n, inv, bg_keys, bg_rec);
}

void launch_k3_sort(const ChunkArgs& a, uint32_t n_long, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0) return;
  const unsigned grid = a.long_list ? n_long : (unsigned)nf * a.n_tiles;
  if (grid == 0) return;
  const size_t smem = sizeof(SortShared<kSortThreads>) + 2 * kSmemCap * sizeof(uint64_t);
  static int attr[kMaxDevices];
  if (ensure_smem_attr(k3_sort, (int)smem, attr) != cudaSuccess) return;
  k3_sort<<<grid, kSortThreads, smem, s>>>(a);
}

}  // namespace gsb
