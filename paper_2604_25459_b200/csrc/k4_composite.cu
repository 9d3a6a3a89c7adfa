// k4_composite.cu — K4: per-tile depth sort + front-to-back alpha compositing.
//
// north_star / readings R12-R16 (3DGS formulation, cited P:212; outputs per P:225):
//   for each pixel, over its tile's list in (depth, id) order:
//     alpha = min(0.99, o exp(power)); skip if alpha < 1/255;
//     tT = T (1 - alpha); stop (before blending) if tT < 1e-4;
//     w = alpha T; C += w rgb; D += w z; T = tT;
//   RGB = C + T bg, depth = D, alpha = 1 - T.
// power is evaluated in log2 units through the whitening factor written by K1:
//   arg = log2(o) - ((p dx)^2 + (q dx + r dy)^2)   (= log2(o e^power))
// so "alpha < 1/255" is the test arg < log2(1/255), decided before any exp2; the exp2 is
// the MUFU ex2.approx (reading R27).
//
// One CTA per (frame, 16x16 tile), 128 threads, two vertically adjacent pixels per thread
// (the dx terms of the quadratic form and the shared-memory loads serve both).  The tile's keys (unsorted, as K2
// emitted them) are loaded into shared memory and sorted there by the segmented radix sort
// of gsb_sort.cuh (lists longer than kFusedSortCap were sorted by K3 into HBM instead) — so
// sorting, which is barrier-bound, overlaps with the ALU-bound compositing of the other CTAs
// resident on the SM.  Records are then staged through shared memory 256 at a time and the
// CTA stops as soon as every pixel has terminated (__syncthreads_count vote).
#include "gsb_common.cuh"
#include "gsb_kernels.cuh"
#include "gsb_sort.cuh"
#include "k4_common.cuh"

namespace gsb {

constexpr int kCompThreads = 128;          // 2 pixels per thread: a 16x16 tile per CTA
constexpr int kBatch = kCompThreads;       // records staged per round (one cp.async set per thread)

// Shared memory.  Small variant (CAP = kFusedSortCap, ~21.5 KB -> 9 CTAs/SM): the tile's
// 64-bit keys are loaded once and radix-sorted in smem; the key buffers are then reused for
// the slot list and the double-buffered record staging (2 x 3 x 128 float4 = 12 KB).
// Large variant (CAP = 4 kFusedSortCap, ~37.6 KB -> 5 CTAs/SM, for views whose tile lists are
// mostly long): the keys stay in L2 and a packed 32-bit sort runs on 8 B per key; the result
// buffer then holds the staging and the other buffer the slot list.
constexpr int kStageQuads = 2 * 3 * kBatch;
template <int CAP, bool MERGE = false, bool SCORE = false>
struct K4Shared {
  static constexpr bool kPacked = CAP > kFusedSortCap;
  union {   // radix sort (packed / HBM lists, merge variant) or counting sort (small variant)
    SortShared<kCompThreads> sort;
    CountShared<kCompThreads, MERGE ? 7 : 11> count;   // (merge variant: unused, kept small)
  } s;
  union {
    uint64_t keys[kPacked ? 1 : 2][kPacked ? 1 : CAP];         // small variant: 64-bit sort
    struct {
      uint32_t slots[kPacked ? 1 : CAP];
      float4 stage[kStageQuads];
    } c;
    uint32_t buf[2][kPacked ? CAP : 1];                          // large variant: packed sort
  } u;
  unsigned long long red[kCompThreads / 32];
  uint8_t wlist[kCompThreads / 32][kBatch];   // per-warp compacted record indices of a round
  uint32_t qpos[MERGE ? CAP : 1];             // merge variant: merged position of robot entry j
  float ssum[SCORE ? 2 : 1][SCORE ? kBatch : 1];     // score variant: per-round sum of w per record
  uint32_t smax[SCORE ? 2 : 1][SCORE ? kBatch : 1];  // and max of w (float bits, w >= 0)
};
static_assert(sizeof(uint32_t) * kFusedSortCap + 16 * kStageQuads <= 2 * 8 * kFusedSortCap, "small union");
static_assert(4 * 4 * kFusedSortCap >= 16 * kStageQuads, "large variant stages in the result buffer");

// MERGE (gsb_render_static, §8(f) row 2): the CTA's list is the (zbits, id) merge of the
// pre-binned, pre-sorted background list of its (camera, tile) with the frame's robot list
// (sorted here as usual).  Keys are unique (R10), so the merge is the full sort of the union
// and every output is bit-identical to gsb_render with the same cameras.  Robot entry j goes
// to merged position qpos[j] = j + #(background keys below it) (binary search in the L2-
// resident background keys); a merged position d is robot entry k = lower_bound(qpos, d) if
// qpos[k] == d, else background entry d - k.
// SCORE (GSB_FLAG_SCORES, §8(f) row 3, reading R30): every blended weight w = alpha T is also
// accumulated per Gaussian — sum and max over the warp (REDUX), then per record of the round
// in shared memory, then one global atomic per (CTA, record) into the scene's accumulators
// (by internal index).
template <int CAP, int MINB, bool MERGE, bool SCORE>
__global__ void __launch_bounds__(kCompThreads, MINB) k4_composite(CompositeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Sh = K4Shared<CAP, MERGE, SCORE>;
  Sh& sm = *reinterpret_cast<Sh*>(smem_raw);
  const unsigned FULL = 0xffffffffu;
  const int fl = a.fs + blockIdx.x / a.n_tiles;
  const int t = blockIdx.x % a.n_tiles;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp w owns the 8x8 block (w & 1, w >> 1) of the tile; a thread owns two vertically
  // adjacent pixels (px, py0) and (px, py0 + 1) of it
  const int bx0 = tx * kTile + 8 * (warp & 1), by0 = ty * kTile + 8 * (warp >> 1);
  const int px = bx0 + (lane & 7);
  const int py0 = by0 + 2 * (lane >> 3);
  const bool in_x = px < a.width;
  const bool in0 = in_x && py0 < a.height, in1 = in_x && py0 + 1 < a.height;
  const uint32_t* off = a.off + (size_t)fl * a.hist_stride;
  const uint64_t start = a.frame_base[fl] - a.key_base + off[t];
  const int len = (int)(off[t + 1] - off[t]);
  const float4* rec = a.rec + (size_t)fl * a.n * kRecQuads;
  // merge variant: this frame's camera's background list
  uint64_t bo = 0;
  int lb = 0;
  if constexpr (MERGE) {
    const int cam = (a.f0 + fl) % a.n_static_cams;
    const uint64_t* bof = a.bg_off + (size_t)cam * (a.n_tiles + 1);
    bo = bof[t];
    lb = (int)(bof[t + 1] - bo);
  }
  const uint64_t* bkeys = a.bg_keys + bo;
  const uint32_t* qpos = nullptr;
  const float pxc = (float)px + 0.5f;
  const float bcx = (float)bx0 + 4.0f, bcy = (float)by0 + 4.0f;  // block centre (pixel centres +-3.5)

  // depth order of this tile's list (reading R10), then id -> record slot.  Lists longer than
  // CAP are sorted as 64-bit keys in HBM (key buffer and its scratch twin).
  const bool fused = len <= CAP;
  const uint32_t* slots = nullptr;
  float4* stg = nullptr;
  // keys carrying the record slot (K4a's scheme, gsb_sort.cuh): no id -> slot gather; equal
  // depths re-sorted by creation id (or, for long runs, the list re-keyed by id and re-sorted)
  const int2* kid = MERGE ? nullptr : a.keys_internal_ids;
  bool kid_fallback = false;
  if constexpr (Sh::kPacked) {
    stg = reinterpret_cast<float4*>(sm.u.buf[0]);
    if (fused && len > 0) {
      const uint64_t* gk = a.keys + start;
      const bool in_b = packed_sort(gk, len, sm.u.buf[0], sm.u.buf[1], sm.s.sort, kid);
      const uint32_t* res = sm.u.buf[in_b ? 1 : 0];
      uint32_t* sl = sm.u.buf[in_b ? 0 : 1];
      for (int e = tid; e < len; e += kCompThreads) {
        const uint64_t key = __ldg(gk + (res[e] & 0xffffu));
        sl[e] = kid ? (uint32_t)key : (uint32_t)(__ldg(a.inv + (uint32_t)key) - a.slot_base);
      }
      slots = sl;
      stg = reinterpret_cast<float4*>(sm.u.buf[in_b ? 1 : 0]);
    }
  } else {
    stg = sm.u.c.stage;
    slots = sm.u.c.slots;
    if (fused && len > 0) {
      for (int e = tid; e < len; e += kCompThreads) sm.u.keys[0][e] = a.keys[start + e];
      __syncthreads();
      bool in_b = false;
      if constexpr (MERGE) {   // shared memory is tight here (qpos): the radix sort
        in_b = len > 1 && segment_sort(sm.u.keys[0], sm.u.keys[1], len, sm.s.sort);
      } else if (len > 1) {
        count_sort(sm.u.keys[0], sm.u.keys[1], len, sm.s.count);   // result in keys[0]
        if (kid && !fix_equal_depth_runs<kCompThreads>(sm.u.keys[0], len, kid)) {
          slot_keys_to_id_keys<kCompThreads>(sm.u.keys[0], len, kid);
          count_sort(sm.u.keys[0], sm.u.keys[1], len, sm.s.count);
          kid_fallback = true;
        }
      }
      const bool direct = kid && !kid_fallback;   // key low word = slot
      uint32_t sl[CAP / kCompThreads];
#pragma unroll
      for (int k = 0; k < CAP / kCompThreads; ++k) {
        const int e = tid + k * kCompThreads;
        if (e < len) {
          const uint64_t key = sm.u.keys[in_b ? 1 : 0][e];
          sl[k] = direct ? (uint32_t)key : (uint32_t)(__ldg(a.inv + (uint32_t)key) - a.slot_base);
          if constexpr (MERGE) sm.qpos[e] = (uint32_t)(e + lower_bound(bkeys, lb, key));
        }
      }
      if constexpr (MERGE) qpos = sm.qpos;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < CAP / kCompThreads; ++k) {
        const int e = tid + k * kCompThreads;
        if (e < len) sm.u.c.slots[e] = sl[k];
      }
    }
  }
  if (!fused) {
    uint64_t* ga = const_cast<uint64_t*>(a.keys) + start;
    uint64_t* gb = a.keys_alt + start;
    const bool in_b = segment_sort(ga, gb, len, sm.s.sort);
    uint32_t* dst = a.sorted + start;
    uint64_t* r = in_b ? gb : ga;
    bool direct = false;
    if (kid) {
      __syncthreads();
      direct = fix_equal_depth_runs<kCompThreads>(r, len, kid);
      if (!direct) {
        uint64_t* o = in_b ? ga : gb;
        slot_keys_to_id_keys<kCompThreads>(r, len, kid);
        if (segment_sort(r, o, len, sm.s.sort)) r = o;
        __syncthreads();
      }
    }
    for (int e = tid; e < len; e += kCompThreads)
      dst[e] = direct ? (uint32_t)r[e] : (uint32_t)(__ldg(a.inv + (uint32_t)r[e]) - a.slot_base);
    slots = dst;
    if constexpr (MERGE) {
      uint32_t* qg = a.qpos_g + start;
      for (int e = tid; e < len; e += kCompThreads) qg[e] = (uint32_t)(e + lower_bound(bkeys, lb, r[e]));
      qpos = qg;
    }
  }
  if constexpr (SCORE) {
    sm.ssum[0][tid] = 0.f; sm.ssum[1][tid] = 0.f;
    sm.smax[0][tid] = 0u; sm.smax[1][tid] = 0u;
  }
  __syncthreads();  // the slot list is complete (and the sort buffers are free)
  if (a.dbg_lists) {   // gsb_debug_tile_lists: export the sorted list, no compositing
    for (int e = tid; e < len; e += kCompThreads) a.dbg_lists[start + e] = slots[e];
    return;
  }

  // stage round b's records into buffer (b & 1): one record (3 x 16 B cp.async) per thread
  const int total = len + lb;   // merged list length (lb = 0 unless MERGE)
  auto stage = [&](int b) {
    const int k = b * kBatch + tid;
    if (k < total) {
      const float4* r;
      if constexpr (MERGE) {
        const int j = len > 0 ? lower_bound(qpos, len, (uint32_t)k) : 0;
        if (j < len && qpos[j] == (uint32_t)k) r = rec + (size_t)slots[j] * kRecQuads;
        else r = a.bg_rec + (bo + (uint64_t)(k - j)) * 3;
      } else {
        r = rec + (size_t)slots[k] * kRecQuads;
      }
      float4* buf = stg + (b & 1) * 3 * kBatch;
      cp_async16(&buf[tid], r);
      cp_async16(&buf[kBatch + tid], r + 1);
      cp_async16(&buf[2 * kBatch + tid], r + 2);
    }
    cp_async_commit();
  };

  float T0 = 1.f, r0c = 0.f, g0c = 0.f, b0c = 0.f, d0 = 0.f;
  float T1 = 1.f, r1c = 0.f, g1c = 0.f, b1c = 0.f, d1 = 0.f;
  float pyc0 = in0 ? (float)py0 + 0.5f : kFar;   // out-of-image pixels never pass the alpha test
  float pyc1 = in1 ? (float)py0 + 1.5f : kFar;
  int ne0 = total, ne1 = total;
  const int rounds = (total + kBatch - 1) / kBatch;
  if (rounds > 0) {
    stage(0);
    cp_async_wait_all();
    __syncthreads();
  }
  for (int b = 0; b < rounds; ++b) {
    if (b + 1 < rounds) stage(b + 1);   // overlaps this round's compositing
    const float4* R0 = reinterpret_cast<const float4*>(
        reinterpret_cast<const char*>(Sh::kPacked ? stg : sm.u.c.stage) + (b & 1) * (3 * kBatch * 16));
    const float4* R1 = R0 + kBatch;
    const float4* R2 = R1 + kBatch;
    const int base = b * kBatch;
    const int cnt = min(kBatch, total - base);
    if (!__all_sync(FULL, pyc0 == kFar && pyc1 == kFar)) {
      // this warp's list of the round's records that can reach its 8x8 block (u8 indices)
      uint8_t* wl = sm.wlist[warp];
      int nsel = 0;
#pragma unroll
      for (int k = 0; k < kBatch / 32; ++k) {
        const int j = 32 * k + lane;
        bool ov = false;
        if (j < cnt) {
          // lower bound of Q' = (p dx)^2 + (q dx + r dy)^2 over the block's pixel centres
          // (dx = u - x in [xa, xb], dy = v - y in [ya, yb]): each term minimised on its own;
          // keep the record unless LB > kappa' with a 2% margin (so no per-pixel decision changes)
          const float4 q0 = R0[j];                                     // u, v, p, q
          const float2 q1 = *reinterpret_cast<const float2*>(&R1[j]);  // r, log2 o
          const float xa = q0.x - (bcx + 3.5f), xb = q0.x - (bcx - 3.5f);
          const float ya = q0.y - (bcy + 3.5f), yb = q0.y - (bcy - 3.5f);
          const float dxm = fmaxf(fmaxf(xa, -xb), 0.f);              // distance of 0 to [xa, xb]
          const float lmin = fmaf(q0.w, q0.w >= 0.f ? xa : xb, q1.x * ya);
          const float lmax = fmaf(q0.w, q0.w >= 0.f ? xb : xa, q1.x * yb);
          const float lm = fmaxf(fmaxf(lmin, -lmax), 0.f);           // distance of 0 to [lmin, lmax]
          const float px_ = q0.z * dxm;
          const float lb = fmaf(px_, px_, lm * lm);
          const float kap = q1.y - kLog2AlphaMin;                    // kappa' = log2(255 o)
          ov = lb <= fmaf(kap, 1.02f, 0.02f);
        }
        const unsigned hit = __ballot_sync(FULL, ov);
        if (ov) wl[nsel + __popc(hit & lanemask_lt())] = (uint8_t)j;
        nsel += __popc(hit);
      }
      __syncwarp();
      for (int i0 = 0; i0 < nsel; i0 += 32) {
        const int i1 = min(nsel, i0 + 32);
#pragma unroll 2
        for (int i = i0; i < i1; ++i) {
          const uint32_t j = wl[i];
          const float4 q0 = R0[j];                                   // u, v, p, q
          const float2 q1 = *reinterpret_cast<const float2*>(&R1[j]);  // r, log2 o
          const float dx = q0.x - pxc;
          const float t1 = q0.z * dx;
          const float mm = fmaf(-t1, t1, q1.y);
          const float qdx = q0.w * dx;
          const float ta = fmaf(q1.x, q0.y - pyc0, qdx);
          const float tb = fmaf(q1.x, q0.y - pyc1, qdx);
          const float arg0 = fmaf(-ta, ta, mm);
          const float arg1 = fmaf(-tb, tb, mm);
          const bool use0 = arg0 >= kLog2AlphaMin;   // alpha >= 1/255
          const bool use1 = arg1 >= kLog2AlphaMin;
          // unconditional two-pixel blend (as K4b): for an unused entry it is an exact no-op
          const float4 q2 = R2[j];                                 // r, g, b, z
          const float2 wb = blend2(use0, arg0, use1, arg1, q2, T0, r0c, g0c, b0c, d0, pyc0, ne0, T1, r1c, g1c,
                                   b1c, d1, pyc1, ne1, base + j);
          const float wb0 = wb.x, wb1 = wb.y;
          if constexpr (SCORE) {
            // warp sum in 6.26 fixed point (|error| <= 2^-27 per pixel weight; 64 pixels x 0.99
            // < 2^6) and exact max of the float bits (w >= 0): two REDUX instructions
            const uint32_t q = __float2uint_rn((wb0 + wb1) * kScoreFix);
            const uint32_t tot = __reduce_add_sync(FULL, q);
            const uint32_t mx = __reduce_max_sync(FULL, __float_as_uint(fmaxf(wb0, wb1)));
            if (lane == 0 && tot) {
              atomicAdd(&sm.ssum[b & 1][j], (float)tot * (1.f / kScoreFix));
              atomicMax(&sm.smax[b & 1][j], mx);
            }
          }
        }
        if (__all_sync(FULL, pyc0 == kFar && pyc1 == kFar)) break;  // whole warp finished
      }
      __syncwarp();
    }
    cp_async_wait_all();
    // round b+1 visible to every warp, round b's buffer free; stop when every pixel is done
    const int n_done = __syncthreads_count(pyc0 == kFar && pyc1 == kFar);
    if constexpr (SCORE) {  // flush round b's per-record scores (thread tid owns record tid)
      const float ws = sm.ssum[b & 1][tid];
      if (ws > 0.f) {
        const uint32_t g = slots[base + tid] + (uint32_t)a.slot_base;
        atomicAdd(a.score_sum + g, ws);
        atomicMax(a.score_max + g, sm.smax[b & 1][tid]);
      }
      sm.ssum[b & 1][tid] = 0.f;
      sm.smax[b & 1][tid] = 0u;
    }
    if (n_done == kCompThreads) break;
  }
  cp_async_wait_all();

  store_pixels(a, (size_t)(a.f0 + fl), px, py0, in0, in1, T0, r0c, g0c, b0c, d0, ne0, T1, r1c, g1c, b1c, d1, ne1);
  if (a.stat_pairs) {
    unsigned long long v = (in0 ? (unsigned long long)ne0 : 0ull) + (in1 ? (unsigned long long)ne1 : 0ull);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0) sm.red[warp] = v;
    // terminated pixels (R13 stop reached: the centre was moved to kFar)
    const unsigned nt = __reduce_add_sync(FULL, (unsigned)(in0 && pyc0 == kFar) + (unsigned)(in1 && pyc1 == kFar));
    if (lane == 0 && nt) atomicAdd(a.stat_pairs + 1, (unsigned long long)nt);
    __syncthreads();
    if (tid == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < kCompThreads / 32; ++w) s += sm.red[w];
      if (s) atomicAdd(a.stat_pairs, s);
    }
  }
}

template <int CAP, int MINB, bool MERGE, bool SCORE>
static void launch_k4_variant(const CompositeArgs& a, unsigned grid, cudaStream_t s) {
  static int attr[kMaxDevices];
  if (ensure_smem_attr(k4_composite<CAP, MINB, MERGE, SCORE>, (int)sizeof(K4Shared<CAP, MERGE, SCORE>), attr) !=
      cudaSuccess)
    return;
  k4_composite<CAP, MINB, MERGE, SCORE><<<grid, kCompThreads, sizeof(K4Shared<CAP, MERGE, SCORE>), s>>>(a);
}

void launch_k4_composite(const CompositeArgs& a, bool long_lists, cudaStream_t s) {
  const int nf = a.fe - a.fs;
  if (nf <= 0) return;
  const unsigned grid = (unsigned)nf * a.n_tiles;
  if (a.score_sum) {
    if (long_lists) launch_k4_variant<4 * kFusedSortCap, 5, false, true>(a, grid, s);
    else launch_k4_variant<kFusedSortCap, 8, false, true>(a, grid, s);
  } else if (a.bg_off) {
    launch_k4_variant<kFusedSortCap, 8, true, false>(a, grid, s);
  } else if (long_lists) {
    launch_k4_variant<4 * kFusedSortCap, 5, false, false>(a, grid, s);
  } else {
    launch_k4_variant<kFusedSortCap, 9, false, false>(a, grid, s);
  }
}

// gsb_get_scores: accumulators (internal order) -> creation-id order
__global__ void k4_scores_export(const float* __restrict__ wsum, const uint32_t* __restrict__ wmax,
                                 const int2* __restrict__ ids, int64_t n, float* __restrict__ out_sum,
                                 float* __restrict__ out_max) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int id = ids[j].x;
  if (out_sum) out_sum[id] = wsum[j];
  if (out_max) out_max[id] = __uint_as_float(wmax[j]);
}

void launch_k4_scores_export(const float* wsum, const uint32_t* wmax, const int2* ids, int64_t n, float* out_sum,
                             float* out_max, cudaStream_t s) {
  if (n <= 0) return;
  k4_scores_export<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(wsum, wmax, ids, n, out_sum, out_max);
}

}  // namespace gsb
