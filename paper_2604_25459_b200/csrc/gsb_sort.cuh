// gsb_sort.cuh — block-wide segment sort used by K3 (long tile lists, in HBM) and by K4
// (tile lists up to kFusedSortCap, in shared memory).
//
// north_star (3): hand-written segmented radix sort, deterministic tie-break on Gaussian id;
// reading R10: a tile list is ordered by (bits(z_f32), id).  LSD radix (8-bit digits) over the
// top 16 varying depth bits; every pass is a stable counting scatter ranked per warp with
// __match_any_sync; runs equal on those bits are finished by the full key (zbits, id), so the
// result is unique whatever order the keys arrived in.
#pragma once
#include "gsb_common.cuh"

namespace gsb {

// Block sort over NT threads (NT = 128 in K4, 256 in K3); 8-bit digits, 256 bins.
template <int NT>
struct SortShared {
  static constexpr int kWarps = NT / 32;
  uint32_t whist[kWarps][256];
  uint32_t base[256];
  uint32_t wred[kWarps];
};

// Exact fix-up of runs that tie on the sorted field, race-free: the array is walked in blocks of
// NT*KPT elements; in each block every run starting there is found with reads only (its end kept
// in a register by the thread owning the start), a barrier, then the owners insertion-sort their
// runs by `less` (disjoint ranges), and a barrier before the next block reads.
template <int NT, typename Ptr, typename Field, typename Less>
__device__ __forceinline__ void fix_runs(Ptr r, int n, Field field, Less less) {
  constexpr int KPT = 8;
  for (int base = 0; base < n; base += NT * KPT) {
    int end[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int e = base + k * NT + (int)threadIdx.x;
      end[k] = -1;
      if (e + 1 < n) {
        const uint32_t h = field(r[e]);
        if ((e == 0 || field(r[e - 1]) != h) && field(r[e + 1]) == h) {
          int x = e + 2;
          while (x < n && field(r[x]) == h) ++x;
          end[k] = x;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      if (end[k] < 0) continue;
      const int e = base + k * NT + (int)threadIdx.x;
      for (int x = e + 1; x < end[k]; ++x) {
        const auto kx = r[x];
        int y = x - 1;
        while (y >= e && less(kx, r[y])) {
          r[y + 1] = r[y];
          --y;
        }
        r[y + 1] = kx;
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ uint32_t hi32(uint64_t k) { return (uint32_t)(k >> 32); }

// exclusive scan over the block of one value per bin (256 bins, NT threads)
template <int NT>
__device__ __forceinline__ void bins_excl_scan(SortShared<NT>& sm) {
  constexpr int PER = 256 / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t v[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) { v[k] = sm.base[tid * PER + k]; sum += v[k]; }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.wred[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
#pragma unroll
  for (int w = 0; w < SortShared<NT>::kWarps; ++w) run += (w < warp) ? sm.wred[w] : 0u;
#pragma unroll
  for (int k = 0; k < PER; ++k) { sm.base[tid * PER + k] = run; run += v[k]; }
  __syncthreads();
}

// one stable counting pass on digit ((hi32(key) - zmin) >> shift) & 0xff: src -> dst
template <int NT, typename Ptr>
__device__ __forceinline__ void radix_pass(const Ptr src, Ptr dst, int n, int shift, uint32_t zmin,
                                           SortShared<NT>& sm) {
  constexpr int kWarps = SortShared<NT>::kWarps;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // digit histogram
  for (int b = tid; b < 256; b += NT) sm.base[b] = 0;
  __syncthreads();
  for (int e = tid; e < n; e += NT) atomicAdd(&sm.base[((hi32(src[e]) - zmin) >> shift) & 0xffu], 1u);
  __syncthreads();
  bins_excl_scan(sm);
  // chunked stable scatter
  for (int c = 0; c < n; c += NT) {
    const int e = c + tid;
    const bool valid = e < n;
    const uint64_t key = valid ? src[e] : 0ull;
    const uint32_t d = valid ? (((hi32(key) - zmin) >> shift) & 0xffu) : 256u + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lanemask_lt());
    for (int b = tid; b < 256; b += NT)
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sm.whist[w][b] = 0;
    __syncthreads();
    if (valid && rank == 0) sm.whist[warp][d] = __popc(peers);
    __syncthreads();
    for (int b = tid; b < 256; b += NT) {
      uint32_t run = sm.base[b];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = sm.whist[w][b];
        sm.whist[w][b] = run;
        run += t;
      }
      sm.base[b] = run;
    }
    __syncthreads();
    if (valid) dst[sm.whist[warp][d] + rank] = key;
    __syncthreads();
  }
}

// Sort keys[0..n) into (bits(z), id) order.  Two stable 8-bit LSD passes order the keys by the
// 16 highest varying bits of (zbits - zmin) (monotone in z; bits above are zero); runs that agree
// on those bits (two depths within ~2^-16 of the segment's depth range) are then
// insertion-sorted by the full 64-bit key (zbits << 32 | id).  Returns true if the result ended
// in `b`.
template <int NT, typename Ptr>
__device__ __forceinline__ bool segment_sort(Ptr a, Ptr b, int n, SortShared<NT>& sm) {
  constexpr int kWarps = SortShared<NT>::kWarps;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // depth range of the segment: sort on (zbits - zmin), whose highest set bit bounds the
  // number of varying bits (unlike zbits itself, whose exponent bits flip at powers of two)
  uint32_t zmin = 0xffffffffu;
  for (int e = tid; e < n; e += NT) zmin = min(zmin, hi32(a[e]));
  zmin = __reduce_min_sync(0xffffffffu, zmin);
  if (lane == 0) sm.wred[warp] = zmin;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kWarps; ++w) zmin = min(zmin, sm.wred[w]);
  __syncthreads();
  uint32_t orx = 0;
  for (int e = tid; e < n; e += NT) orx |= hi32(a[e]) - zmin;
  orx = __reduce_or_sync(0xffffffffu, orx);
  if (lane == 0) sm.wred[warp] = orx;
  __syncthreads();
  orx = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) orx |= sm.wred[w];
  __syncthreads();
  const int hb = orx ? 31 - __clz(orx) : -1;       // highest varying bit of (zbits - zmin)
  const int lo = hb >= 16 ? hb - 15 : 0;           // sort bits [lo, lo + 16) of (zbits - zmin)
  bool in_b = false;
  if (hb >= 0) {
    if (((orx >> lo) & 0xffu) != 0) {
      radix_pass(a, b, n, lo, zmin, sm);
      in_b = true;
    }
    if (((orx >> (lo + 8)) & 0xffu) != 0) {
      if (in_b) radix_pass(b, a, n, lo + 8, zmin, sm);
      else radix_pass(a, b, n, lo + 8, zmin, sm);
      in_b = !in_b;
    }
  }
  Ptr r = in_b ? b : a;
  // runs equal on the sorted bits: finish them by the full key (zbits, id) — reading R10
  int dup = 0;
  for (int e = tid + 1; e < n; e += NT) dup |= ((hi32(r[e]) - zmin) >> lo) == ((hi32(r[e - 1]) - zmin) >> lo);
  if (__syncthreads_or(dup))
    fix_runs<NT>(r, n, [&](uint64_t k) { return (hi32(k) - zmin) >> lo; },
                 [](uint64_t x, uint64_t y) { return x < y; });
  return in_b;
}

// ---------------------------------------------------------------------------------------------
// Single-pass counting sort for short segments (K4a, lists up to a few thousand keys): bucket
// = the BITS highest varying bits of (zbits - zmin); histogram with shared atomics, one block
// scan, scatter with atomic cursors (order inside a bucket arbitrary); then every key takes its
// rank among the keys of its own bucket (full key (zbits, id), reading R10) and lands at
// bucket start + rank.  Keys are unique, so the result is the unique order whatever the
// scatter order; ranking is parallel over keys (a bucket of m keys costs m reads per key), so
// skewed depth distributions do not serialise.  In: a; scratch: b; result: a.
template <int NT, int BITS>
struct CountShared {
  static constexpr int kBins = 1 << BITS;
  static constexpr int kWarps = NT / 32;
  uint32_t bins[kBins];
  uint32_t wred[kWarps];
};

template <int NT, int BITS>
__device__ __forceinline__ void count_sort(uint64_t* a, uint64_t* b, int n, CountShared<NT, BITS>& sm) {
  using Sh = CountShared<NT, BITS>;
  constexpr int PER = Sh::kBins / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t zmin = 0xffffffffu;
  for (int e = tid; e < n; e += NT) zmin = min(zmin, hi32(a[e]));
  zmin = __reduce_min_sync(0xffffffffu, zmin);
  if (lane == 0) sm.wred[warp] = zmin;
#pragma unroll
  for (int k = 0; k < PER; ++k) sm.bins[tid + k * NT] = 0;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < Sh::kWarps; ++w) zmin = min(zmin, sm.wred[w]);
  uint32_t orx = 0;
  for (int e = tid; e < n; e += NT) orx |= hi32(a[e]) - zmin;
  orx = __reduce_or_sync(0xffffffffu, orx);
  __syncthreads();
  if (lane == 0) sm.wred[warp] = orx;
  __syncthreads();
  orx = 0;
#pragma unroll
  for (int w = 0; w < Sh::kWarps; ++w) orx |= sm.wred[w];
  const int hb = orx ? 31 - __clz(orx) : -1;          // highest varying bit of (zbits - zmin)
  const int lo = hb >= BITS ? hb - BITS + 1 : 0;      // bucket = bits [lo, lo + BITS)
  for (int e = tid; e < n; e += NT) atomicAdd(&sm.bins[(hi32(a[e]) - zmin) >> lo], 1u);
  __syncthreads();
  // exclusive scan of the buckets: PER consecutive buckets per thread
  uint32_t v[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) { v[k] = sm.bins[tid * PER + k]; sum += v[k]; }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.wred[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
#pragma unroll
  for (int w = 0; w < Sh::kWarps; ++w) run += (w < warp) ? sm.wred[w] : 0u;
#pragma unroll
  for (int k = 0; k < PER; ++k) { sm.bins[tid * PER + k] = run; run += v[k]; }
  __syncthreads();
  // scatter (cursors advance: afterwards bins[k] = end of bucket k = start of bucket k + 1)
  for (int e = tid; e < n; e += NT) {
    const uint64_t key = a[e];
    b[atomicAdd(&sm.bins[(hi32(key) - zmin) >> lo], 1u)] = key;
  }
  __syncthreads();
  // rank inside the bucket by the full key
  for (int p = tid; p < n; p += NT) {
    const uint64_t key = b[p];
    const uint32_t bk = (hi32(key) - zmin) >> lo;
    const int s0 = bk ? (int)sm.bins[bk - 1] : 0, s1 = (int)sm.bins[bk];
    int rank = 0;
    for (int q = s0; q < s1; ++q) rank += b[q] < key;
    a[s0 + rank] = key;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// Packed tile sort (K4): the segment's 64-bit keys stay where K2 wrote them (HBM/L2); the sort
// runs on 32-bit words (16 highest varying bits of zbits - zmin) << 16 | local index, so the
// double buffer costs 8 B per key and each pass moves 4 B.  Runs equal on the 16 bits (depths
// within ~2^-16 of the segment's range) are finished by the full key (zbits << 32 | id) read
// back through L2.  Result: local indices in (bits(z), id) order (reading R10).
template <int NT>
__device__ __forceinline__ void radix_pass32(const uint32_t* src, uint32_t* dst, int n, int shift,
                                             SortShared<NT>& sm) {
  constexpr int kWarps = SortShared<NT>::kWarps;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < 256; b += NT) sm.base[b] = 0;
  __syncthreads();
  for (int e = tid; e < n; e += NT) atomicAdd(&sm.base[(src[e] >> shift) & 0xffu], 1u);
  __syncthreads();
  bins_excl_scan(sm);
  for (int c = 0; c < n; c += NT) {
    const int e = c + tid;
    const bool valid = e < n;
    const uint32_t key = valid ? src[e] : 0u;
    const uint32_t d = valid ? ((key >> shift) & 0xffu) : 256u + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lanemask_lt());
    for (int b = tid; b < 256; b += NT)
#pragma unroll
      for (int w = 0; w < kWarps; ++w) sm.whist[w][b] = 0;
    __syncthreads();
    if (valid && rank == 0) sm.whist[warp][d] = __popc(peers);
    __syncthreads();
    for (int b = tid; b < 256; b += NT) {
      uint32_t run = sm.base[b];
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = sm.whist[w][b];
        sm.whist[w][b] = run;
        run += t;
      }
      sm.base[b] = run;
    }
    __syncthreads();
    if (valid) dst[sm.whist[warp][d] + rank] = key;
    __syncthreads();
  }
}

// n <= 65536.  Returns true if the sorted words ended in `b` (else `a`).  With `ids` the keys'
// low words are record slots and equal-field runs are finished by (bits(z), ids[slot].x) — the
// (bits(z), id) order of reading R10 without a creation id in the key.
template <int NT>
__device__ __forceinline__ bool packed_sort(const uint64_t* __restrict__ gkeys, int n, uint32_t* a, uint32_t* b,
                                            SortShared<NT>& sm, const int2* __restrict__ ids = nullptr) {
  constexpr int kWarps = SortShared<NT>::kWarps;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t zmin = 0xffffffffu;
  for (int e = tid; e < n; e += NT) zmin = min(zmin, hi32(__ldg(gkeys + e)));
  zmin = __reduce_min_sync(0xffffffffu, zmin);
  if (lane == 0) sm.wred[warp] = zmin;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kWarps; ++w) zmin = min(zmin, sm.wred[w]);
  __syncthreads();
  uint32_t orx = 0;
  for (int e = tid; e < n; e += NT) orx |= hi32(__ldg(gkeys + e)) - zmin;
  orx = __reduce_or_sync(0xffffffffu, orx);
  if (lane == 0) sm.wred[warp] = orx;
  __syncthreads();
  orx = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) orx |= sm.wred[w];
  const int hb = orx ? 31 - __clz(orx) : -1;
  const int lo = hb >= 16 ? hb - 15 : 0;
  const uint32_t field_or = orx >> lo;              // which of the 16 field bits vary
  for (int e = tid; e < n; e += NT)
    a[e] = ((((hi32(__ldg(gkeys + e)) - zmin) >> lo) & 0xffffu) << 16) | (uint32_t)e;
  __syncthreads();
  bool in_b = false;
  if (field_or & 0xffu) {
    radix_pass32(a, b, n, 16, sm);
    in_b = true;
  }
  if (field_or & 0xff00u) {
    if (in_b) radix_pass32(b, a, n, 24, sm);
    else radix_pass32(a, b, n, 24, sm);
    in_b = !in_b;
  }
  uint32_t* r = in_b ? b : a;
  int dup = 0;
  for (int e = tid + 1; e < n; e += NT) dup |= (r[e] >> 16) == (r[e - 1] >> 16);
  if (__syncthreads_or(dup)) {
    if (ids)
      fix_runs<NT>(r, n, [](uint32_t w) { return w >> 16; }, [gkeys, ids](uint32_t x, uint32_t y) {
        const uint64_t kx = __ldg(gkeys + (x & 0xffffu)), ky = __ldg(gkeys + (y & 0xffffu));
        const uint32_t zx = hi32(kx), zy = hi32(ky);
        return zx != zy ? zx < zy : __ldg(&ids[(uint32_t)kx].x) < __ldg(&ids[(uint32_t)ky].x);
      });
    else
      fix_runs<NT>(r, n, [](uint32_t w) { return w >> 16; },
                   [gkeys](uint32_t x, uint32_t y) { return __ldg(gkeys + (x & 0xffffu)) < __ldg(gkeys + (y & 0xffffu)); });
  }
  return in_b;
}

// Keys (bits(z) << 32 | slot) sorted by the full key are in (z, slot) order; reading R10 wants
// (z, creation id).  Runs of equal z (rare) are re-sorted by ids[slot].x: run starts are found
// read-only first (up to kRunSlots per thread), then each run is insertion-sorted by its starting
// thread after a barrier.  Returns false — nothing changed — when a run is longer than
// kShortRun or a thread found too many runs (e.g. a fronto-parallel plane: every key ties); the
// caller then re-sorts the list by (z, id) keys.
constexpr int kRunSlots = 4;
constexpr int kShortRun = 32;

// sh: low bits of the key's low word that are not part of the slot (K4b block masks; 0 or 4)
template <int NT, typename P>
__device__ __forceinline__ bool fix_equal_depth_runs(P r, int n, const int2* __restrict__ ids, int sh = 0) {
  const int tid = threadIdx.x;
  int starts[kRunSlots], ends[kRunSlots];   // runs [start, end) found in the read-only pass
  int ns = 0;
  bool bad = false;
  for (int e = tid; e + 1 < n; e += NT) {
    const uint32_t z = hi32(r[e]);
    if (hi32(r[e + 1]) == z && (e == 0 || hi32(r[e - 1]) != z)) {
      int s1 = e + 2;
      while (s1 < n && s1 - e <= kShortRun && hi32(r[s1]) == z) ++s1;
      if (s1 - e > kShortRun || ns == kRunSlots) {
        bad = true;
      } else {
        starts[ns] = e;
        ends[ns++] = s1;
      }
    }
  }
  if (__syncthreads_or(bad)) return false;
  if (!__syncthreads_or(ns > 0)) return true;
  for (int k = 0; k < ns; ++k) {   // each run is touched by its finder only
    const int s0 = starts[k], s1 = ends[k];
    for (int i = s0 + 1; i < s1; ++i) {   // insertion sort by creation id (runs are short)
      const uint64_t key = r[i];
      const int id = __ldg(&ids[(uint32_t)key >> sh].x);
      int j = i - 1;
      while (j >= s0 && __ldg(&ids[(uint32_t)r[j] >> sh].x) > id) {
        r[j + 1] = r[j];
        --j;
      }
      r[j + 1] = key;
    }
  }
  __syncthreads();
  return true;
}

// the fallback: key low words slot -> creation id (the high word, bits(z), is kept)
template <int NT, typename P>
__device__ __forceinline__ void slot_keys_to_id_keys(P r, int n, const int2* __restrict__ ids, int sh = 0) {
  for (int e = threadIdx.x; e < n; e += NT) {
    const uint64_t k = r[e];
    const uint32_t lo = (uint32_t)k;   // (slot << sh | mask) -> (id << sh | mask)
    r[e] = (k & 0xffffffff00000000ull) | ((uint32_t)__ldg(&ids[lo >> sh].x) << sh) | (lo & ((1u << sh) - 1u));
  }
  __syncthreads();
}

}  // namespace gsb
