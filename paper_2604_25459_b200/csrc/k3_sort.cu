// k3_sort.cu — K3: hand-written segmented radix sort with a deterministic id tie-break.
//
// north_star: "(3) a hand-written segmented radix sort with a deterministic tie-break on
// Gaussian id"; reading R10: every (frame, tile) list is ordered by (bits(z_f32), id).
//
// Segments are the (frame, tile) buckets K2 filled (in arbitrary, atomic order).  One CTA
// sorts one segment: an LSD radix sort over the 32 depth bits (8-bit digits; digits that are
// constant over the segment are skipped), each pass a stable counting scatter ranked with
// __match_any_sync per warp.  Segments up to kSmemCap keys are sorted entirely in shared
// memory; longer ones ping-pong between the key buffer and its scratch twin in HBM with the
// same code.  Equal depth keys are then put in id order (ids read from the records), so the
// output is the unique (zbits, id) order whatever order the keys arrived in.
#include "gsb_common.cuh"
#include "gsb_kernels.cuh"

namespace gsb {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSmemCap = 4096;

struct SortShared {
  uint32_t whist[kSortWarps][256];
  uint32_t base[256];
  uint32_t wred[kSortWarps];
};

__device__ __forceinline__ uint32_t hi32(uint64_t k) { return (uint32_t)(k >> 32); }

// exclusive scan of one value per thread over the 256-thread block
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, SortShared& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.wred[warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) wpre += (w < warp) ? sm.wred[w] : 0u;
  __syncthreads();
  return wpre + inc - x;
}

// one stable counting pass on digit (hi32(key) >> shift) & 0xff: src -> dst
template <typename Ptr>
__device__ __forceinline__ void radix_pass(const Ptr src, Ptr dst, int n, int shift, SortShared& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // digit histogram
  sm.base[tid] = 0;
  __syncthreads();
  for (int e = tid; e < n; e += kSortThreads) atomicAdd(&sm.base[(hi32(src[e]) >> shift) & 0xffu], 1u);
  __syncthreads();
  const uint32_t cnt = sm.base[tid];
  __syncthreads();
  sm.base[tid] = block_excl_scan(cnt, sm);
  __syncthreads();
  // chunked stable scatter
  for (int c = 0; c < n; c += kSortThreads) {
    const int e = c + tid;
    const bool valid = e < n;
    const uint64_t key = valid ? src[e] : 0ull;
    const uint32_t d = valid ? ((hi32(key) >> shift) & 0xffu) : 256u + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lanemask_lt());
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) sm.whist[w][tid] = 0;
    __syncthreads();
    if (valid && rank == 0) sm.whist[warp][d] = __popc(peers);
    __syncthreads();
    {
      uint32_t run = sm.base[tid];
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t t = sm.whist[w][tid];
        sm.whist[w][tid] = run;
        run += t;
      }
      sm.base[tid] = run;
    }
    __syncthreads();
    if (valid) dst[sm.whist[warp][d] + rank] = key;
    __syncthreads();
  }
}

// sort keys[0..n) by their high 32 bits, then put equal-depth runs in id order.
// Returns true if the result ended in `b` (else in `a`).
template <typename Ptr>
__device__ __forceinline__ bool segment_sort(Ptr a, Ptr b, int n, const float4* __restrict__ rec,
                                             SortShared& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // which depth bits vary over the segment?
  const uint32_t first = hi32(a[0]);
  uint32_t orx = 0;
  for (int e = tid; e < n; e += kSortThreads) orx |= hi32(a[e]) ^ first;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) orx |= __shfl_xor_sync(0xffffffffu, orx, o);
  if (lane == 0) sm.wred[warp] = orx;
  __syncthreads();
  orx = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) orx |= sm.wred[w];
  __syncthreads();
  bool in_b = false;
  for (int shift = 0; shift < 32; shift += 8) {
    if (((orx >> shift) & 0xffu) == 0) continue;
    if (!in_b) radix_pass(a, b, n, shift, sm);
    else radix_pass(b, a, n, shift, sm);
    in_b = !in_b;
  }
  Ptr r = in_b ? b : a;
  // deterministic tie-break on Gaussian id (reading R10)
  int dup = 0;
  for (int e = tid + 1; e < n; e += kSortThreads) dup |= hi32(r[e]) == hi32(r[e - 1]);
  if (__syncthreads_or(dup)) {
    for (int e = tid; e < n; e += kSortThreads) {
      const uint32_t h = hi32(r[e]);
      const bool start = (e == 0 || hi32(r[e - 1]) != h) && (e + 1 < n && hi32(r[e + 1]) == h);
      if (!start) continue;
      int end = e + 1;
      while (end < n && hi32(r[end]) == h) ++end;
      for (int x = e + 1; x < end; ++x) {  // insertion sort of the run by id
        const uint64_t kx = r[x];
        const int idx = __float_as_int(rec[(size_t)(uint32_t)kx * 3 + 1].w);
        int y = x - 1;
        while (y >= e && __float_as_int(rec[(size_t)(uint32_t)r[y] * 3 + 1].w) > idx) {
          r[y + 1] = r[y];
          --y;
        }
        r[y + 1] = kx;
      }
    }
    __syncthreads();
  }
  return in_b;
}

__global__ void __launch_bounds__(kSortThreads) k3_sort(ChunkArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortShared& sm = *reinterpret_cast<SortShared*>(smem_raw);
  uint64_t* sa = reinterpret_cast<uint64_t*>(smem_raw + sizeof(SortShared));
  uint64_t* sb = sa + kSmemCap;

  const int fl = a.fs + blockIdx.x / a.n_tiles;
  const int t = blockIdx.x % a.n_tiles;
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  const uint64_t start = a.frame_base[fl] - a.key_base + off[t];
  const int n = (int)(off[t + 1] - off[t]);
  if (n == 0) return;
  const float4* rec = a.rec + (size_t)fl * a.n * 3;
  if (n == 1) {
    if (threadIdx.x == 0) a.sorted[start] = (uint32_t)a.keys[start];
    return;
  }
  if (n <= kSmemCap) {
    for (int e = threadIdx.x; e < n; e += kSortThreads) sa[e] = a.keys[start + e];
    __syncthreads();
    const bool in_b = segment_sort(sa, sb, n, rec, sm);
    const uint64_t* r = in_b ? sb : sa;
    for (int e = threadIdx.x; e < n; e += kSortThreads) a.sorted[start + e] = (uint32_t)r[e];
  } else {
    uint64_t* ga = a.keys + start;
    uint64_t* gb = a.keys_alt + start;
    const bool in_b = segment_sort(ga, gb, n, rec, sm);
    __syncthreads();
    const uint64_t* r = in_b ? gb : ga;
    for (int e = threadIdx.x; e < n; e += kSortThreads) a.sorted[start + e] = (uint32_t)r[e];
  }
}

void launch_k3_sort(const ChunkArgs& a, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0) return;
  const size_t smem = sizeof(SortShared) + 2 * kSmemCap * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k3_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k3_sort<<<(unsigned)nf * a.n_tiles, kSortThreads, smem, s>>>(a);
}

}  // namespace gsb
