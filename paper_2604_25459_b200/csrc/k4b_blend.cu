// k4b_blend.cu — the split compositing path (plain and observation renders):
//
//   K4a k4a_sort   one CTA per (frame, tile): the tile's keys in (bits(z), id) order (reading
//                  R10; gsb_sort.cuh: a one-pass 11-bit counting sort for lists up to 1024 keys,
//                  the radix sorts beyond), written as record slots into the `sorted` workspace.
//   K4b k4b_blend  persistent warps: each warp takes (frame, tile, 8x8 block) work items from an
//                  atomic counter and composites its 64 pixels front to back over the tile's
//                  sorted list (readings R12-R16), staging 32 records per round with cp.async
//                  into its own double buffer, culling them against its block (the same lower
//                  bound as k4_composite.cu), and leaving the item as soon as its pixels have
//                  terminated.
//
// Why split: in the one-CTA-per-tile kernel the four warps of a tile meet at a barrier every
// round, and warps whose block terminates early idle until the slowest one finishes (35 % of
// K4's stall samples, profiles/r04_k4_ncu_full.txt).  Here no warp ever waits for another; the
// price is reading each record once per warp (from L2) instead of once per CTA.
#include <algorithm>
#include <cstdlib>

#include "gsb_sort.cuh"
#include "k4_common.cuh"

namespace gsb {

constexpr int kSortThreadsA = 256;

constexpr int kCountBits = 11;   // K4a counting-sort buckets (2048)

template <int CAP>
struct K4aShared {
  static constexpr bool kPacked = CAP > kFusedSortCap;
  union {   // a CTA uses one of the two sorts
    SortShared<kSortThreadsA> sort;
    CountShared<kSortThreadsA, kCountBits> count;
  } s;
  union {
    uint64_t keys[kPacked ? 1 : 2][kPacked ? 1 : CAP];   // small variant: 64-bit keys in smem
    uint32_t buf[2][kPacked ? CAP : 1];                   // large variant: packed sort
  } u;
};

// Where the (frame fl, tile t) list lives in the `sorted` buffer.  Plain: at the tile's key
// offset.  Static-camera merge (gsb_render_static): the merged list of the tile's robot keys
// and its camera's pre-binned background list; frame regions hold K_rb(f) + K_bg(cam(f))
// entries, so the frame base adds the background sizes of the pass's earlier frames (prefix
// table over cameras, cyclic in the frame index) and the tile adds its background offset.
struct TileList {
  uint64_t start;   // first entry in `sorted` (and first key of the robot list: rstart)
  uint64_t rstart;  // first robot key in `keys`
  int len;          // robot keys
  int lb;           // background entries (merge)
  uint64_t bo;      // first background entry in bg_keys / bg_rec (merge)
};

__device__ __forceinline__ TileList tile_list(const CompositeArgs& a, int fl, int t) {
  TileList L;
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  const uint64_t fb = a.frame_base[fl] - a.key_base;
  L.rstart = fb + off[t];
  L.len = (int)(off[t + 1] - off[t]);
  L.start = L.rstart;
  L.lb = 0;
  L.bo = 0;
  if (a.bg_off) {
    const int C = a.n_static_cams;
    const int cam = (a.f0 + fl) % C;
    const uint64_t* bof = a.bg_off + (size_t)cam * (a.n_tiles + 1);
    L.bo = bof[t];
    L.lb = (int)(bof[t + 1] - L.bo);
    const int n = fl - a.fs, b0 = (a.f0 + a.fs) % C, r = n % C;
    const uint64_t cyc = (b0 + r <= C) ? a.bg_cum[b0 + r] - a.bg_cum[b0]
                                       : (a.bg_cum[C] - a.bg_cum[b0]) + a.bg_cum[b0 + r - C];
    L.start = fb + (uint64_t)(n / C) * a.bg_cum[C] + cyc + off[t] + (L.bo - bof[0]);
  }
  return L;
}

constexpr uint32_t kBgTag = 0x80000000u;   // merged entry: background record index | tag

// one (frame, tile) list of K4a: sort, then record slots into `sorted`
template <int CAP>
__device__ __forceinline__ void k4a_sort_list(const CompositeArgs& a, int fl, int t, K4aShared<CAP>& sm) {
  using Sh = K4aShared<CAP>;
  const int tid = threadIdx.x;
  const TileList L = tile_list(a, fl, t);
  const uint64_t start = L.rstart;
  const int len = L.len;
  const int base = a.slot_base;
  if (a.bg_off) {   // static-camera merge (small variant only)
    if (len + L.lb == 0) return;
    uint32_t* dst = a.sorted + L.start;
    const uint64_t* bk = a.bg_keys + L.bo;
    const uint64_t* rk = nullptr;   // the robot keys in (zbits, id) order
    if constexpr (!Sh::kPacked) {
      if (len <= CAP) {
        for (int e = tid; e < len; e += kSortThreadsA) sm.u.keys[0][e] = a.keys[start + e];
        __syncthreads();
        if (len > 1) count_sort(sm.u.keys[0], sm.u.keys[1], len, sm.s.count);
        rk = sm.u.keys[0];
      }
    }
    if (!rk) {
      uint64_t* ga = const_cast<uint64_t*>(a.keys) + start;
      uint64_t* gb = a.keys_alt + start;
      const bool in_b = len > 1 && segment_sort(ga, gb, len, sm.s.sort);
      __syncthreads();
      rk = in_b ? gb : ga;
    }
    // keys are unique (R10): an entry's merged position is its own index plus the number of
    // entries of the other list below it
    for (int j = tid; j < len; j += kSortThreadsA) {
      const uint64_t key = rk[j];
      int lo = 0, hi = L.lb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(bk + mid) < key) lo = mid + 1;
        else hi = mid;
      }
      dst[j + lo] = (uint32_t)(__ldg(a.inv + (uint32_t)key) - base);
    }
    for (int i = tid; i < L.lb; i += kSortThreadsA) {
      const uint64_t key = __ldg(bk + i);
      int lo = 0, hi = len;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rk[mid] < key) lo = mid + 1;
        else hi = mid;
      }
      dst[i + lo] = kBgTag | (uint32_t)(L.bo + i);
    }
    return;
  }
  if (len == 0) return;
  uint32_t* dst = a.sorted + start;
  const int2* kid = a.keys_internal_ids;
  if (len == 1) {
    if (tid == 0) dst[0] = kid ? (uint32_t)a.keys[start] : (uint32_t)(__ldg(a.inv + (uint32_t)a.keys[start]) - base);
    return;
  }
  if (kid) {   // keys carry the slot: sort, restore the (z, id) order of equal depths, write slots
    if (len <= CAP) {
      if constexpr (Sh::kPacked) {
        const uint64_t* gk = a.keys + start;
        const bool in_b = packed_sort(gk, len, sm.u.buf[0], sm.u.buf[1], sm.s.sort, kid);
        const uint32_t* res = sm.u.buf[in_b ? 1 : 0];
        for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)__ldg(gk + (res[e] & 0xffffu));
      } else {
        uint64_t* k0 = sm.u.keys[0];
        for (int e = tid; e < len; e += kSortThreadsA) k0[e] = a.keys[start + e];
        __syncthreads();
        count_sort(k0, sm.u.keys[1], len, sm.s.count);
        if (fix_equal_depth_runs<kSortThreadsA>(k0, len, kid)) {
          for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)k0[e];
        } else {   // long equal-depth runs: re-sort by (z, id) keys and gather the slots
          slot_keys_to_id_keys<kSortThreadsA>(k0, len, kid);
          count_sort(k0, sm.u.keys[1], len, sm.s.count);
          for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)(__ldg(a.inv + (uint32_t)k0[e]) - base);
        }
      }
    } else {
      uint64_t* ga = const_cast<uint64_t*>(a.keys) + start;
      uint64_t* gb = a.keys_alt + start;
      const bool in_b = segment_sort(ga, gb, len, sm.s.sort);
      __syncthreads();
      uint64_t* r = in_b ? gb : ga;
      if (fix_equal_depth_runs<kSortThreadsA>(r, len, kid)) {
        for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)r[e];
      } else {
        uint64_t* o = in_b ? ga : gb;
        slot_keys_to_id_keys<kSortThreadsA>(r, len, kid);
        const bool in_o = segment_sort(r, o, len, sm.s.sort);
        __syncthreads();
        const uint64_t* rr = in_o ? o : r;
        for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)(__ldg(a.inv + (uint32_t)rr[e]) - base);
      }
    }
    return;
  }
  if (len <= CAP) {
    if constexpr (Sh::kPacked) {
      const uint64_t* gk = a.keys + start;
      const bool in_b = packed_sort(gk, len, sm.u.buf[0], sm.u.buf[1], sm.s.sort);
      const uint32_t* res = sm.u.buf[in_b ? 1 : 0];
      for (int e = tid; e < len; e += kSortThreadsA)
        dst[e] = (uint32_t)(__ldg(a.inv + (uint32_t)__ldg(gk + (res[e] & 0xffffu))) - base);
    } else {
      for (int e = tid; e < len; e += kSortThreadsA) sm.u.keys[0][e] = a.keys[start + e];
      __syncthreads();
      count_sort(sm.u.keys[0], sm.u.keys[1], len, sm.s.count);
      const uint64_t* r = sm.u.keys[0];
      for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)(__ldg(a.inv + (uint32_t)r[e]) - base);
    }
  } else {  // longer than the shared-memory capacity: 64-bit keys sorted in HBM
    uint64_t* ga = const_cast<uint64_t*>(a.keys) + start;
    uint64_t* gb = a.keys_alt + start;
    const bool in_b = segment_sort(ga, gb, len, sm.s.sort);
    const uint64_t* r = in_b ? gb : ga;
    for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)(__ldg(a.inv + (uint32_t)r[e]) - base);
  }
}



// K4a, one CTA per list: every (frame, tile) list of the pass (grid = lists), or — LONG — the
// entries of a.long_list (the chunk's lists longer than kWarpSortCap, the short ones being sorted
// by k4a_warp_sort), grid-stride so that the count may live on the device (fixed plan); entries
// of frames outside this pass are skipped
template <int CAP, bool LONG = false>
__global__ void __launch_bounds__(kSortThreadsA) k4a_sort(CompositeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Sh = K4aShared<CAP>;
  Sh& sm = *reinterpret_cast<Sh*>(smem_raw);
  if (a.overflow && *a.overflow) return;   // fixed plan: chunk beyond the key capacity
  if constexpr (LONG) {   // grid-stride over the long-list table (count on the host or the device)
    const uint32_t n = a.n_long_dev ? *a.n_long_dev : a.n_long;
    for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
      const uint32_t e = a.long_list[k];
      const int fl = (int)(e >> 16), t = (int)(e & 0xffffu);
      if (fl >= a.fs && fl < a.fe) k4a_sort_list<CAP>(a, fl, t, sm);
      __syncthreads();   // the shared buffers are reused by the next list
    }
  } else {
    k4a_sort_list<CAP>(a, a.fs + blockIdx.x / a.n_tiles, blockIdx.x % a.n_tiles, sm);
  }
}


// ------------------------------------------------------------------------------ K4a, one CTA per long list
// Lists of kWarpSortCap < n <= kIdxCap keys (and, for views whose lists are mostly long, every
// list) are sorted by one 256-thread CTA with a counting sort that never moves the 64-bit keys:
// buckets = the top kIdxBits varying bits of (zbits - zmin); the keys' 16-bit local indices are
// scattered into their buckets (shared atomics), then each key takes its rank among its bucket's
// keys by (bits(z), id) — read through L1 from the list in HBM/L2 — and its slot is written at
// bucket start + rank.  Six barriers per list, whatever n.  Equal depths with slot keys are
// ordered by ids[slot]; a run of more than kShortRun equal depths sends the list to the HBM radix
// with (z, id) keys (reading R10).  Longer lists: the HBM radix (segment_sort).
constexpr int kIdxCap = 4096;
constexpr int kIdxBits = 12;
struct K4aIdxShared {
  union {
    SortShared<kSortThreadsA> sort;   // the HBM radix (lists > kIdxCap, long equal-depth runs)
    struct {
      uint32_t bins[1 << kIdxBits];
      uint32_t wmin[kSortThreadsA / 32], wmax[kSortThreadsA / 32], wsum[kSortThreadsA / 32];
    } c;
  } s;
  uint16_t buf[kIdxCap];
};

// K4b block masks (CompositeArgs::key_shift = kMaskBits): a key's low word is (slot << 4 | mask)
// and so is the sorted entry; an id-keyed low word (id << sh | mask) maps to (slot << sh | mask)
__device__ __forceinline__ uint32_t id_word_to_slot_word(const CompositeArgs& a, uint32_t w) {
  const int sh = a.key_shift;
  return ((uint32_t)(__ldg(a.inv + (w >> sh)) - a.slot_base) << sh) | (w & ((1u << sh) - 1u));
}

// the HBM path of one list: LSD radix of 64-bit keys in keys / keys_alt (gsb_sort.cuh)
__device__ __forceinline__ void k4a_hbm_list(const CompositeArgs& a, uint64_t start, int len, uint32_t* dst,
                                             SortShared<kSortThreadsA>& ss) {
  const int tid = threadIdx.x;
  const int2* kid = a.keys_internal_ids;
  const int base = a.slot_base;
  uint64_t* ga = const_cast<uint64_t*>(a.keys) + start;
  uint64_t* gb = a.keys_alt + start;
  const bool in_b = segment_sort(ga, gb, len, ss);
  __syncthreads();
  uint64_t* r = in_b ? gb : ga;
  if (!kid) {
    for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)(__ldg(a.inv + (uint32_t)r[e]) - base);
  } else if (fix_equal_depth_runs<kSortThreadsA>(r, len, kid, a.key_shift)) {
    for (int e = tid; e < len; e += kSortThreadsA) dst[e] = (uint32_t)r[e];
  } else {
    uint64_t* o = in_b ? ga : gb;
    slot_keys_to_id_keys<kSortThreadsA>(r, len, kid, a.key_shift);
    const bool in_o = segment_sort(r, o, len, ss);
    __syncthreads();
    const uint64_t* rr = in_o ? o : r;
    for (int e = tid; e < len; e += kSortThreadsA) dst[e] = id_word_to_slot_word(a, (uint32_t)rr[e]);
  }
}

// one list by the index counting sort (n <= kIdxCap); false = a long equal-depth run (nothing
// usable written: the caller re-sorts)
__device__ __forceinline__ bool k4a_idx_list(const CompositeArgs& a, const uint64_t* __restrict__ gk, int n,
                                             uint32_t* dst, K4aIdxShared& sm) {
  constexpr int NT = kSortThreadsA, BINS = 1 << kIdxBits, PER = BINS / NT;
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2* kid = a.keys_internal_ids;
  const int base = a.slot_base;
  uint32_t zmin = 0xffffffffu, zmax = 0u;
  for (int e = tid; e < n; e += NT) {
    const uint32_t z = hi32(__ldg(gk + e));
    zmin = min(zmin, z);
    zmax = max(zmax, z);
  }
  zmin = __reduce_min_sync(FULL, zmin);
  zmax = __reduce_max_sync(FULL, zmax);
  if (lane == 0) { sm.s.c.wmin[warp] = zmin; sm.s.c.wmax[warp] = zmax; }
#pragma unroll
  for (int k = 0; k < PER; ++k) sm.s.c.bins[tid * PER + k] = 0u;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) { zmin = min(zmin, sm.s.c.wmin[w]); zmax = max(zmax, sm.s.c.wmax[w]); }
  const uint32_t span = zmax - zmin;
  const int hb = span ? 31 - __clz(span) : -1;
  const int lo = hb >= kIdxBits ? hb - kIdxBits + 1 : 0;
  for (int e = tid; e < n; e += NT) atomicAdd(&sm.s.c.bins[(hi32(__ldg(gk + e)) - zmin) >> lo], 1u);
  __syncthreads();
  uint32_t v[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) { v[k] = sm.s.c.bins[tid * PER + k]; sum += v[k]; }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.s.c.wsum[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) run += (w < warp) ? sm.s.c.wsum[w] : 0u;
#pragma unroll
  for (int k = 0; k < PER; ++k) { sm.s.c.bins[tid * PER + k] = run; run += v[k]; }
  __syncthreads();
  for (int e = tid; e < n; e += NT)
    sm.buf[atomicAdd(&sm.s.c.bins[(hi32(__ldg(gk + e)) - zmin) >> lo], 1u)] = (uint16_t)e;
  __syncthreads();
  bool long_run = false;
  for (int p = tid; p < n; p += NT) {
    const uint64_t key = __ldg(gk + sm.buf[p]);
    const uint32_t z = hi32(key);
    const uint32_t b = (z - zmin) >> lo;
    const int s0 = b ? (int)sm.s.c.bins[b - 1] : 0, s1 = (int)sm.s.c.bins[b];
    int rank = 0, eq = 0;
    for (int q = s0; q < s1; ++q) {
      const uint64_t kq = __ldg(gk + sm.buf[q]);
      rank += kq < key;
      eq += hi32(kq) == z;
    }
    if (kid && eq > 1) {   // equal depths: order by creation id instead of slot
      if (eq > kShortRun + 1) {
        long_run = true;
      } else {
        const int idp = __ldg(&kid[(uint32_t)key >> a.key_shift].x);
        rank = 0;
        for (int q = s0; q < s1; ++q) {
          const uint64_t kq = __ldg(gk + sm.buf[q]);
          const uint32_t zq = hi32(kq);
          rank += zq < z || (zq == z && kq != key && __ldg(&kid[(uint32_t)kq >> a.key_shift].x) < idp);
        }
      }
    }
    dst[s0 + rank] = kid ? (uint32_t)key : (uint32_t)(__ldg(a.inv + (uint32_t)key) - base);
  }
  return !__syncthreads_or(long_run);
}

// ALL: every list of the pass, one CTA each (views whose lists are mostly long); else the
// chunk's long-list table (lists > kWarpSortCap), grid-stride (the count may be on the device)
template <bool ALL>
__global__ void __launch_bounds__(kSortThreadsA) k4a_idx_sort(CompositeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K4aIdxShared& sm = *reinterpret_cast<K4aIdxShared*>(smem_raw);
  if (a.overflow && *a.overflow) return;   // fixed plan: chunk beyond the key capacity
  const uint32_t n_items = ALL ? (uint32_t)((a.fe - a.fs) * a.n_tiles) : (a.n_long_dev ? *a.n_long_dev : a.n_long);
  for (uint32_t k = blockIdx.x; k < n_items; k += gridDim.x) {
    int fl, t;
    if constexpr (ALL) {
      fl = a.fs + (int)(k / (uint32_t)a.n_tiles);
      t = (int)(k % (uint32_t)a.n_tiles);
    } else {
      const uint32_t e = a.long_list[k];
      fl = (int)(e >> 16);
      t = (int)(e & 0xffffu);
      if (fl < a.fs || fl >= a.fe) continue;   // CTA-uniform
    }
    const TileList L = tile_list(a, fl, t);
    const int len = L.len;
    uint32_t* dst = a.sorted + L.start;
    if (len <= 1) {
      if (len == 1 && threadIdx.x == 0) {
        const uint64_t key = a.keys[L.rstart];
        dst[0] = a.keys_internal_ids ? (uint32_t)key : (uint32_t)(__ldg(a.inv + (uint32_t)key) - a.slot_base);
      }
      continue;
    }
    if (len > kIdxCap || !k4a_idx_list(a, a.keys + L.rstart, len, dst, sm)) {
      __syncthreads();   // the index sort's shared state is dead; the radix reuses the union
      k4a_hbm_list(a, L.rstart, len, dst, sm.s.sort);
    }
    __syncthreads();     // shared buffers reused by the next list
  }
}

// ------------------------------------------------------------------------------ K4a, one warp per list
// Lists of up to kWarpSortCap keys (98.5 % of C3's) are sorted by ONE warp each, with no CTA
// barrier (the CTA-per-tile sort above spent most of its time in per-CTA fixed costs — 2048-bin
// scans, barriers — for lists averaging 340 keys).  Counting sort on the top kWarpBits varying
// bits of (zbits - zmin) (range from the list's zmin and zmax: the highest varying bit of
// z - zmin is the highest bit of zmax - zmin); scatter into the bucket with shared atomics; then
// every key takes its rank among the keys of its bucket by (bits(z), id) and is written straight
// to its final position as a record slot.  With slot keys an equal-depth pair is ordered by the
// creation ids ids[slot] (gathered only for ties); a list with a run of more than kShortRun equal
// depths (e.g. a fronto-parallel plane) is re-keyed by id and re-ranked (reading R10).
#ifndef GSB_WARP_BITS
#define GSB_WARP_BITS 9
#endif
constexpr int kWarpBits = GSB_WARP_BITS;
constexpr int kWarpBins = 1 << kWarpBits;
#ifndef GSB_K4A_IDX
#define GSB_K4A_IDX 1   // 0: the long lists by count_sort<1024> / packed_sort<4096> (A/B comparisons)
#endif
#ifndef GSB_K4A_WARPS
#define GSB_K4A_WARPS 4
#endif
constexpr int kK4aWarps = GSB_K4A_WARPS;   // lists (warps) per CTA

struct K4aWarpShared {
  uint64_t buf[kWarpSortCap];   // the list, bucketed
  uint32_t bins[kWarpBins];
};

__global__ void __launch_bounds__(kK4aWarps * 32) k4a_warp_sort(CompositeArgs a, int n_lists) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  K4aWarpShared& sm = reinterpret_cast<K4aWarpShared*>(smem_raw)[warp];
  const int ft = blockIdx.x * kK4aWarps + warp;
  if (ft >= n_lists) return;   // warp-uniform
  if (a.overflow && *a.overflow) return;   // fixed plan: chunk beyond the key capacity
  const int fl = a.fs + ft / a.n_tiles;
  const int t = ft % a.n_tiles;
  const TileList L = tile_list(a, fl, t);
  const int n = L.len;
  if (n == 0 || n > kWarpSortCap) return;   // long lists: k4a_sort<.., true>
  const uint64_t* gk = a.keys + L.rstart;
  uint32_t* dst = a.sorted + L.start;
  const int2* kid = a.keys_internal_ids;   // slot keys: key low word = slot
  const int base = a.slot_base;
  auto slot_of = [&](uint64_t key) -> uint32_t {
    return kid ? (uint32_t)key : (uint32_t)(__ldg(a.inv + (uint32_t)key) - base);
  };
  if (n == 1) {
    if (lane == 0) dst[0] = slot_of(__ldg(gk));
    return;
  }
  // depth range -> bucket shift
  uint32_t zmin = 0xffffffffu, zmax = 0u;
  for (int e = lane; e < n; e += 32) {
    const uint32_t z = hi32(__ldg(gk + e));
    zmin = min(zmin, z);
    zmax = max(zmax, z);
  }
  zmin = __reduce_min_sync(FULL, zmin);
  zmax = __reduce_max_sync(FULL, zmax);
  const uint32_t span = zmax - zmin;
  const int hb = span ? 31 - __clz(span) : -1;
  const int lo = hb >= kWarpBits ? hb - kWarpBits + 1 : 0;
  // histogram
  constexpr int PER = kWarpBins / 32;
#pragma unroll
  for (int k = 0; k < PER; ++k) sm.bins[lane * PER + k] = 0u;
  __syncwarp();
  for (int e = lane; e < n; e += 32) atomicAdd(&sm.bins[(hi32(__ldg(gk + e)) - zmin) >> lo], 1u);
  __syncwarp();
  // exclusive scan (PER consecutive buckets per lane)
  uint32_t v[PER], sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) { v[k] = sm.bins[lane * PER + k]; sum += v[k]; }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t run = inc - sum;
#pragma unroll
  for (int k = 0; k < PER; ++k) { sm.bins[lane * PER + k] = run; run += v[k]; }
  __syncwarp();
  // scatter into the buckets (cursors advance: afterwards bins[b] = end of bucket b)
  for (int e = lane; e < n; e += 32) {
    const uint64_t key = __ldg(gk + e);
    sm.buf[atomicAdd(&sm.bins[(hi32(key) - zmin) >> lo], 1u)] = key;
  }
  __syncwarp();
  // rank inside the bucket: (bits(z), id); ids gathered for equal depths only
  bool long_run = false;
  for (int p = lane; p < n; p += 32) {
    const uint64_t key = sm.buf[p];
    const uint32_t z = hi32(key);
    const uint32_t b = (z - zmin) >> lo;
    const int s0 = b ? (int)sm.bins[b - 1] : 0, s1 = (int)sm.bins[b];
    int rank = 0, eq = 0;
    for (int q = s0; q < s1; ++q) {
      const uint64_t kq = sm.buf[q];
      rank += kq < key;
      eq += hi32(kq) == z;
    }
    if (kid && eq > 1) {   // equal depths: order by creation id instead of slot
      if (eq > kShortRun + 1) {
        long_run = true;
      } else {
        const int idp = __ldg(&kid[(uint32_t)key >> a.key_shift].x);
        rank = 0;
        for (int q = s0; q < s1; ++q) {
          const uint64_t kq = sm.buf[q];
          const uint32_t zq = hi32(kq);
          rank += zq < z || (zq == z && q != p && __ldg(&kid[(uint32_t)kq >> a.key_shift].x) < idp);
        }
      }
    }
    dst[s0 + rank] = slot_of(key);
  }
  if (__any_sync(FULL, long_run)) {   // long equal-depth runs: re-key by id, re-rank by (z, id)
    __syncwarp();
    const int sh = a.key_shift;
    for (int p = lane; p < n; p += 32) {   // (slot << sh | mask) -> (id << sh | mask)
      const uint64_t k = sm.buf[p];
      const uint32_t lo = (uint32_t)k;
      sm.buf[p] = (k & 0xffffffff00000000ull) | ((uint32_t)__ldg(&kid[lo >> sh].x) << sh) | (lo & ((1u << sh) - 1u));
    }
    __syncwarp();
    for (int p = lane; p < n; p += 32) {
      const uint64_t key = sm.buf[p];
      const uint32_t b = (hi32(key) - zmin) >> lo;
      const int s0 = b ? (int)sm.bins[b - 1] : 0, s1 = (int)sm.bins[b];
      int rank = 0;
      for (int q = s0; q < s1; ++q) rank += sm.buf[q] < key;
      dst[s0 + rank] = id_word_to_slot_word(a, (uint32_t)key);
    }
  }
}

// ------------------------------------------------------------------------------ K4b
constexpr int kBlendWarps = 4;
constexpr int kWarpBatch = 32;   // records per warp window / masked round (one per lane)
#ifndef GSB_K4B_PER
#define GSB_K4B_PER 1   // 2: 64-record rounds (C3 -1.7 %, C4 -1.3 %: the fixed per-round work is not the cost)
#endif
constexpr int kPer = GSB_K4B_PER;               // unmasked path: records staged per lane per round
constexpr int kRound = kPer * kWarpBatch;       // unmasked path: records per round
#ifndef GSB_K4B_UNROLL
#define GSB_K4B_UNROLL 2
#endif
constexpr int kBlendUnroll = GSB_K4B_UNROLL;   // unroll of the selected-record loop

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// SCORE (GSB_FLAG_SCORES, reading R30): every blended weight is also summed (6.26 fixed point,
// __reduce_add_sync) and maxed (exact, float bits) over the warp per record, then added to the
// scene's per-Gaussian accumulators with one global atomic pair per (warp, record).
// MERGE: static-camera merge (tagged background record slots), else plain record slots.
// MASKED (CompositeArgs::key_shift = kMaskBits): every sorted entry carries the 4-bit mask of the
// tile's 8x8 blocks its record can reach (K2b, the same lower bound and margin as the cull below),
// so a warp never stages or tests a record outside its block: it scans its list 32 entries at a
// time, queues the hits (slot, list position) in shared memory and stages full rounds of 32 hit
// records — no per-round cull, and a third of the rounds (C3: 13 of 32 staged records were hits).
template <bool SCORE, bool MERGE, bool MASKED>
__global__ void __launch_bounds__(kBlendWarps * 32, 8) k4b_blend(CompositeArgs a, int* __restrict__ counter,
                                                                  int n_items) {
  __shared__ __align__(16) float4 stg[kBlendWarps][2][3][kRound];   // 12 KB per record per lane
  constexpr int kQ = 2 * kWarpBatch;   // hit queue (ring) per warp
  __shared__ uint2 hitq[MASKED ? kBlendWarps : 1][MASKED ? kQ : 1];           // (slot, list position)
  __shared__ uint32_t hitpos[MASKED ? kBlendWarps : 1][2][MASKED ? kWarpBatch : 1];   // staged positions
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 (*S)[3][kRound] = stg[warp];
  // shared address of this lane's staging slot (buffer 0, row 0); rows kRowB, buffers kBufB apart
  constexpr uint32_t kRowB = kRound * sizeof(float4), kBufB = 3 * kRowB;
  const uint32_t s_lane = (uint32_t)__cvta_generic_to_shared(&S[0][0][lane]);
  for (;;) {   // (fixed plan: an overflowed chunk's counter starts at n_items, see launch_k4b_blend)
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1);
    item = __shfl_sync(FULL, item, 0);
    if (item >= n_items) break;
    const int blk = item & 3, ft = item >> 2;
    const int fl = a.fs + ft / a.n_tiles;
    const int t = ft % a.n_tiles;
    const int tx = t % a.tiles_x, ty = t / a.tiles_x;
    // the 8x8 block `blk` of the tile; a lane owns pixels (px, py0) and (px, py0 + 1)
    const int bx0 = tx * kTile + 8 * (blk & 1), by0 = ty * kTile + 8 * (blk >> 1);
    const int px = bx0 + (lane & 7);
    const int py0 = by0 + 2 * (lane >> 3);
    const bool in_x = px < a.width;
    const bool in0 = in_x && py0 < a.height, in1 = in_x && py0 + 1 < a.height;
    const TileList L = tile_list(a, fl, t);
    const int len = L.len + L.lb;   // merged length (lb = 0 unless static-camera merge)
    const float4* rec = a.rec + (size_t)fl * a.n * kRecQuads;
    const uint32_t rbase = (uint32_t)((int64_t)fl * a.n);   // record index base (< 2^32: gsb_reserve)
    const uint32_t* slots = a.sorted + L.start;
    const float pxc = (float)px + 0.5f;
    const float bcx = (float)bx0 + 4.0f, bcy = (float)by0 + 4.0f;  // block centre (pixel centres +-3.5)

    // per-pixel state as (pixel 0, pixel 1) pairs (packed FFMA2/FADD2/FMUL2, k4_common.cuh)
    f32x2 T = pk2(1.f, 1.f), R = pk2(0.f, 0.f), G = R, Bc = R, D = R;
    // out-of-image pixels never pass the alpha test
    f32x2 PYC = pk2(in0 ? (float)py0 + 0.5f : kFar, in1 ? (float)py0 + 1.5f : kFar);
    auto all_done = [&]() {
      const float2 pc = up2(PYC);
      return __all_sync(FULL, pc.x == kFar && pc.y == kFar);
    };
    int ne0 = len, ne1 = len;
    const int rounds = all_done() ? 0 : (len + kRound - 1) / kRound;

    if constexpr (MASKED) {
      // the quadratic form (log2 of o e^power) of staged record i for both pixels:
      // ta = r (v - pyc) + q dx;  arg = log2 o - (p dx)^2 - ta^2
      auto arg_at = [&](const float4* R0, const float4* R1, int i) -> f32x2 {
        const float4 r0 = R0[i];                                   // u, v, p, q
        const float2 r1 = *reinterpret_cast<const float2*>(&R1[i]);  // r, log2 o
        const float dx = r0.x - pxc;                               // shared by both pixels
        const f32x2 pq = mul2(pk2(r0.z, r0.w), pk2(dx, dx));      // (p dx, q dx)
        const float mm = fmaf(-pq.x, pq.x, r1.y);
        const f32x2 ta = fma2(pk2(r1.x, r1.x), sub2(pk2(r0.y, r0.y), PYC), pk2(pq.y, pq.y));
        return nfma2(ta, ta, pk2(mm, mm));
      };
      uint2* Q = hitq[warp];
      const uint32_t bit = 1u << blk;
      const int nwin = all_done() ? 0 : (len + kWarpBatch - 1) / kWarpBatch;
      int win = 0, qh = 0, qn = 0;   // next window to scan; queue head and length (warp-uniform)
      // this lane's entries of the next two windows (read ahead: no scan waits on a fresh load)
      uint32_t w1 = lane < len ? __ldg(slots + lane) : 0u;
      uint32_t w2 = kWarpBatch + lane < len ? __ldg(slots + kWarpBatch + lane) : 0u;
      // scan windows until the queue holds a full round or the list ends
      auto fill = [&]() {
        while (qn < kWarpBatch && win < nwin) {
          const uint32_t w = w1;
          w1 = w2;
          const int k2 = (win + 2) * kWarpBatch + lane;
          w2 = k2 < len ? __ldg(slots + k2) : 0u;
          const int pos = win * kWarpBatch + lane;
          const bool hit = pos < len && (w & bit);
          const unsigned hm = __ballot_sync(FULL, hit);
          if (hit) Q[(qh + qn + __popc(hm & lanemask_lt())) & (kQ - 1)] = make_uint2(w >> kMaskBits, (uint32_t)pos);
          qn += __popc(hm);
          ++win;
        }
        __syncwarp();
      };
      // stage the queue's first min(qn, 32) hits into buffer buf (one record per lane)
      auto stage_q = [&](int buf) -> int {
        const int n = min(qn, kWarpBatch);
        if (lane < n) {
          const uint2 e = Q[(qh + lane) & (kQ - 1)];
          const float4* r = rec + (size_t)e.x * kRecQuads;
          const uint32_t d = s_lane + (uint32_t)buf * kBufB;
          cp_async16s(d, r);
          cp_async16s(d + kRowB, r + 1);
          cp_async16s(d + 2 * kRowB, r + 2);
          hitpos[warp][buf][lane] = e.y;
        }
        cp_async_commit();
        qh = (qh + n) & (kQ - 1);
        qn -= n;
        return n;
      };
      fill();
      int n_cur = stage_q(0);
      for (int b = 0; n_cur > 0; ++b) {
        fill();
        const int n_next = stage_q((b + 1) & 1);
        cp_async_wait_group<1>();
        __syncwarp();
        const float4* R0 = S[b & 1][0];
        const float4* R1 = S[b & 1][1];
        const float4* R2 = S[b & 1][2];
        const uint32_t* P = hitpos[warp][b & 1];
        // software pipeline: the next entry's quadratic form is evaluated while this one blends
        // (independent chains; blend2p sets it to -inf for a pixel that terminates here).
        // Index n_cur <= 32 reads the next sub-array of the staging buffer: in bounds, never used.
        f32x2 argn = arg_at(R0, R1, 0);
#pragma unroll kBlendUnroll
        for (int i = 0; i < n_cur; ++i) {
          const f32x2 arg = argn;
          argn = arg_at(R0, R1, i + 1);
          const float4 q2 = R2[i];                                 // r, g, b, z
          auto pos = [&]() { return (int)P[i]; };                  // list position (n_eval)
          blend2p(arg, q2, T, R, G, Bc, D, PYC, ne0, ne1, pos, argn);
        }
        // the "all pixels done" vote once per round of 32 hits (voting after every terminating
        // entry, or every 16 entries, costs more than the entries it saves: same-box A/B)
        const bool done = all_done();
        __syncwarp();   // buffer b & 1 is free for round b + 2
        if (done) break;
        n_cur = n_next;
      }
    } else {
      // stage round b (slots sl[p] of this lane's records p * 32 + lane) into buffer b & 1; the
      // slots of the round after the next are read one round ahead, so no cp.async waits on them
      struct Slots { uint32_t v[kPer]; };
      auto stage = [&](int b, const Slots& sl) {
#pragma unroll
        for (int p = 0; p < kPer; ++p) {
          if (b * kRound + p * kWarpBatch + lane < len) {
            const float4* r = a.rec + (size_t)(rbase + sl.v[p]) * kRecQuads;
            if constexpr (MERGE) {
              if (sl.v[p] & kBgTag) r = a.bg_rec + (size_t)(sl.v[p] & ~kBgTag) * 3;
            }
            const uint32_t d = s_lane + (uint32_t)(b & 1) * kBufB + (uint32_t)p * (kWarpBatch * sizeof(float4));
            cp_async16s(d, r);
            cp_async16s(d + kRowB, r + 1);
            cp_async16s(d + 2 * kRowB, r + 2);
          }
        }
        cp_async_commit();
      };
      auto slot_of = [&](int b) -> Slots {
        Slots r;
#pragma unroll
        for (int p = 0; p < kPer; ++p) {
          const int k = b * kRound + p * kWarpBatch + lane;
          r.v[p] = k < len ? __ldg(slots + k) : 0u;
        }
        return r;
      };
      Slots sl_next{}, sl_cur{}, sl_stg{};   // slots of rounds b + 2, b, b + 1 (this lane)
      if (rounds > 0) {
        sl_cur = slot_of(0);
        stage(0, sl_cur);
        sl_next = slot_of(1);
      }
      for (int b = 0; b < rounds; ++b) {
        if (b + 1 < rounds) {
          sl_stg = sl_next;
          stage(b + 1, sl_next);
          sl_next = slot_of(b + 2);
          cp_async_wait_group<1>();
        } else {
          cp_async_wait_group<0>();
        }
        __syncwarp();
        float4* R0 = S[b & 1][0];
        float4* R1 = S[b & 1][1];
        float4* R2 = S[b & 1][2];
        const int base = b * kRound;
        // this round's records that can reach the block (lower bound of the whitened quadratic
        // form over the block's pixel centres, 2 % margin: no per-pixel decision changes)
        bool ov[kPer];
        float4 q0[kPer], q2[kPer];
        float2 q1[kPer];
        unsigned hit[kPer];
#pragma unroll
        for (int p = 0; p < kPer; ++p) {
          const int e = p * kWarpBatch + lane;
          ov[p] = false;
          q0[p] = make_float4(0.f, 0.f, 0.f, 0.f);
          q2[p] = q0[p];
          q1[p] = make_float2(0.f, 0.f);
          if (base + e < len) {
            q0[p] = R0[e];
            q1[p] = *reinterpret_cast<const float2*>(&R1[e]);
            q2[p] = R2[e];
            const float xa = q0[p].x - (bcx + 3.5f), xb = q0[p].x - (bcx - 3.5f);
            const float ya = q0[p].y - (bcy + 3.5f), yb = q0[p].y - (bcy - 3.5f);
            const float dxm = fmaxf(fmaxf(xa, -xb), 0.f);
            const float lmin = fmaf(q0[p].w, q0[p].w >= 0.f ? xa : xb, q1[p].x * ya);
            const float lmax = fmaf(q0[p].w, q0[p].w >= 0.f ? xb : xa, q1[p].x * yb);
            const float lm = fmaxf(fmaxf(lmin, -lmax), 0.f);
            const float px_ = q0[p].z * dxm;
            const float lbq = fmaf(px_, px_, lm * lm);
            ov[p] = lbq <= fmaf(q1[p].y - kLog2AlphaMin, 1.02f, 0.02f);
          }
          hit[p] = __ballot_sync(FULL, ov[p]);
        }
        // the selected records moved, in order, to the front of the buffer (in place: every lane
        // read its own records above), with the record's round position in R1.z for n_eval and
        // scores; the loop then reads them at warp-uniform, consecutive addresses (broadcast loads)
        __syncwarp();
        int nsel = 0;
#pragma unroll
        for (int p = 0; p < kPer; ++p) {
          if (ov[p]) {
            const int k = nsel + __popc(hit[p] & lanemask_lt());
            R0[k] = q0[p];
            R1[k] = make_float4(q1[p].x, q1[p].y, __int_as_float(p * kWarpBatch + lane), 0.f);
            R2[k] = q2[p];
          }
          nsel += __popc(hit[p]);
        }
        __syncwarp();
        // the quadratic form of selected record i (log2 of o e^power) for both pixels:
        // ta = r (v - pyc) + q dx;  arg = log2 o - (p dx)^2 - ta^2
        auto arg_of = [&](int i) -> f32x2 {
          const float4 q0 = R0[i];                                   // u, v, p, q
          const float2 q1 = *reinterpret_cast<const float2*>(&R1[i]);  // r, log2 o
          const float dx = q0.x - pxc;                               // shared by both pixels
          const f32x2 pq = mul2(pk2(q0.z, q0.w), pk2(dx, dx));      // (p dx, q dx)
          const float mm = fmaf(-pq.x, pq.x, q1.y);
          const f32x2 ta = fma2(pk2(q1.x, q1.x), sub2(pk2(q0.y, q0.y), PYC), pk2(pq.y, pq.y));
          return nfma2(ta, ta, pk2(mm, mm));
        };
        // software pipeline: record i + 1's quadratic form is evaluated while record i blends (the
        // two chains are independent; blend2p sets it to -inf for a pixel that terminates at i).
        // Index nsel <= 32 reads the next sub-array of the staging buffer: in bounds, never used.
        f32x2 argn = nsel > 0 ? arg_of(0) : pk2(0.f, 0.f);
  #pragma unroll kBlendUnroll
        for (int i = 0; i < nsel; ++i) {
          const f32x2 arg = argn;
          argn = arg_of(i + 1);
          // no "does any lane blend" vote: after the block cull almost every staged record is used
          // by some lane, and for the others blend2p is an exact no-op (w = 0: T, colour and depth
          // unchanged), so the vote and its branch only cost issue slots (+4.8 % C3, same-box A/B)
          const float4 q2 = R2[i];                                   // r, g, b, z
          // the record's position in the round (n_eval; read only when a pixel terminates)
          auto pos = [&]() { return base + __float_as_int(R1[i].z); };
          const f32x2 wb = blend2p(arg, q2, T, R, G, Bc, D, PYC, ne0, ne1, pos, argn);
          if constexpr (SCORE) {
            const int j = __float_as_int(R1[i].z);
            const float2 w2 = up2(wb);
            const uint32_t tot = __reduce_add_sync(FULL, __float2uint_rn((w2.x + w2.y) * kScoreFix));
            const uint32_t mx = __reduce_max_sync(FULL, __float_as_uint(fmaxf(w2.x, w2.y)));
            uint32_t sj = 0;
#pragma unroll
            for (int p = 0; p < kPer; ++p) {
              const uint32_t v = __shfl_sync(FULL, sl_cur.v[p], j & 31);
              if ((j >> 5) == p) sj = v;
            }
            const uint32_t g = sj + (uint32_t)a.slot_base;
            if (lane == 0 && tot) {
              atomicAdd(a.score_sum + g, (float)tot * (1.f / kScoreFix));
              atomicMax(a.score_max + g, mx);
            }
          }
        }
        __syncwarp();   // buffer b & 1 is free for round b + 2
        sl_cur = sl_stg;
        if (all_done()) break;
      }
    }
    cp_async_wait_all();   // nothing may land in the buffers after this item
    __syncwarp();
    const float2 T2 = up2(T), R2p = up2(R), G2 = up2(G), B2 = up2(Bc), D2 = up2(D), pc = up2(PYC);
    store_pixels(a, (size_t)(a.f0 + fl), px, py0, in0, in1, T2.x, R2p.x, G2.x, B2.x, D2.x, ne0, T2.y, R2p.y, G2.y,
                 B2.y, D2.y, ne1);
    const float pyc0 = pc.x, pyc1 = pc.y;
    if (a.stat_pairs) {
      unsigned long long v = (in0 ? (unsigned long long)ne0 : 0ull) + (in1 ? (unsigned long long)ne1 : 0ull);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      if (lane == 0 && v) atomicAdd(a.stat_pairs, v);
      // terminated pixels (R13 stop reached: the centre was moved to kFar)
      const unsigned nt = __reduce_add_sync(FULL, (unsigned)(in0 && pyc0 == kFar) + (unsigned)(in1 && pyc1 == kFar));
      if (lane == 0 && nt) atomicAdd(a.stat_pairs + 1, (unsigned long long)nt);
    }
  }
}

template <int CAP, bool LONG = false>
static void launch_k4a_variant(const CompositeArgs& a, unsigned grid, cudaStream_t s) {
  static int attr[kMaxDevices];
  if (ensure_smem_attr(k4a_sort<CAP, LONG>, (int)sizeof(K4aShared<CAP>), attr) != cudaSuccess) return;
  k4a_sort<CAP, LONG><<<grid, kSortThreadsA, sizeof(K4aShared<CAP>), s>>>(a);
}

static bool warp_k4a_on() {   // GSB_K4A=cta: one CTA per list for every list (A/B comparisons)
  const char* e = getenv("GSB_K4A");
  return !(e && e[0] == 'c');
}

bool k4a_masks_supported() {   // warp / index sorts (and their HBM fallback) are mask-aware
  return GSB_K4A_IDX && warp_k4a_on();
}

void launch_k4a_sort(const CompositeArgs& a, bool long_lists, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0) return;
  const unsigned grid = (unsigned)nf * a.n_tiles;
  if (long_lists && GSB_K4A_IDX && !a.bg_off) {   // every list one CTA, by the index counting sort
    static int attr[kMaxDevices];
    if (ensure_smem_attr(k4a_idx_sort<true>, (int)sizeof(K4aIdxShared), attr) != cudaSuccess) return;
    k4a_idx_sort<true><<<grid, kSortThreadsA, sizeof(K4aIdxShared), s>>>(a);
  } else if (long_lists) {
    launch_k4a_variant<4 * kFusedSortCap>(a, grid, s);
  } else if (a.long_list && !a.bg_off && warp_k4a_on()) {
    // short lists one warp each; the chunk's long lists (K2a's list) one CTA each
    const int n_lists = (int)grid;
    static int attr[kMaxDevices];
    if (ensure_smem_attr(k4a_warp_sort, (int)(kK4aWarps * sizeof(K4aWarpShared)), attr) != cudaSuccess) return;
    k4a_warp_sort<<<(n_lists + kK4aWarps - 1) / kK4aWarps, kK4aWarps * 32, kK4aWarps * sizeof(K4aWarpShared), s>>>(
        a, n_lists);
    unsigned lg = a.n_long;
    if (a.n_long_dev) {   // fixed plan: the count is on the device: a persistent grid-stride launch
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
      lg = (unsigned)std::max(1, std::min(n_lists, 4 * sms));
    }
    if (lg > 0) {
      if (GSB_K4A_IDX) {
        static int attr_i[kMaxDevices];
        if (ensure_smem_attr(k4a_idx_sort<false>, (int)sizeof(K4aIdxShared), attr_i) != cudaSuccess) return;
        k4a_idx_sort<false><<<lg, kSortThreadsA, sizeof(K4aIdxShared), s>>>(a);
      } else {
        launch_k4a_variant<kFusedSortCap, true>(a, lg, s);
      }
    }
  } else {
    launch_k4a_variant<kFusedSortCap>(a, grid, s);
  }
}

// fixed plan: K4b's work counter starts at 0, or past the last item when the chunk overflowed
__global__ void k4b_counter_init(int* counter, const int* overflow, int n_items) {
  *counter = *overflow ? n_items : 0;
}

void launch_k4b_blend(const CompositeArgs& a, int* counter, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0) return;
  static int persistent_dev[kMaxDevices];   // persistent grid of the device (SM count x CTAs per SM)
  const int dev = current_device();
  int tmp = 0;
  int& persistent = (dev >= 0 && dev < kMaxDevices) ? persistent_dev[dev] : tmp;
  if (!persistent) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4b_blend<false, false, false>, kBlendWarps * 32, 0);
    // GSB_K4B_PER_SM=8 (one below the register limit) lets the other streams' latency-bound
    // kernels co-reside: C3 +0.6 %, C4 +1.8 %, C6 +0.8 % of step throughput, but K4b's own live
    // event time grows with the sharing (bench roofline 0.90 -> 0.76); the default keeps 9
    if (const char* e = getenv("GSB_K4B_PER_SM")) per_sm = std::min(per_sm, atoi(e));
    persistent = std::max(1, sms * std::max(1, per_sm));
  }
  const long long items = (long long)nf * a.n_tiles * 4;
  if (a.overflow) k4b_counter_init<<<1, 1, 0, s>>>(counter, a.overflow, (int)items);
  else cudaMemsetAsync(counter, 0, sizeof(int), s);
  const unsigned g = (unsigned)std::min<long long>(persistent, (items + kBlendWarps - 1) / kBlendWarps);
  const bool merge = a.bg_off != nullptr;
  if (a.key_shift) {   // block masks: plain slot-key passes only (Pipeline::pass)
    k4b_blend<false, false, true><<<g, kBlendWarps * 32, 0, s>>>(a, counter, (int)items);
  } else if (a.score_sum) {
    if (merge) k4b_blend<true, true, false><<<g, kBlendWarps * 32, 0, s>>>(a, counter, (int)items);
    else k4b_blend<true, false, false><<<g, kBlendWarps * 32, 0, s>>>(a, counter, (int)items);
  } else {
    if (merge) k4b_blend<false, true, false><<<g, kBlendWarps * 32, 0, s>>>(a, counter, (int)items);
    else k4b_blend<false, false, false><<<g, kBlendWarps * 32, 0, s>>>(a, counter, (int)items);
  }
}

}  // namespace gsb
