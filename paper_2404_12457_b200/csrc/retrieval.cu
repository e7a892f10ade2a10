// retrieval.cu — exact inner-product top-k over the embedding corpus, staged.
//
// Replaces the synthetic staged retrieval of the reference
// (speculation.py:149-194 generate_stages/_perturb, plugged in through the
// StageProvider seam simulator.py:228,315-324): stage s is the exact top-k
// over the first (s+1)/S of the scan order, the final stage is the full
// corpus top-k, and the stages feed the DSP controller (speculation.py:98-146).
//
// Corpus GEMM on tcgen05: A = 128 corpus rows x 64-dim atoms (TMA, SW128,
// 5-stage ring), B = the query batch (<= 64 queries, resident in smem), D in
// TMEM (double-buffered, 2 x NQ fp32 columns).
// More than 64 queries (up to 256: the all-gathered queries of 4 ranks, or of 8 ranks
// x 32): a thread-block cluster of C = 2 or 4 CTAs shares one corpus range; CTA r holds
// queries [64r, 64r + 64) and every A stage is loaded ONCE and multicast to the C CTAs'
// shared memory (cp.async.bulk.tensor .multicast::cluster, issuers alternating per
// stage), each MMA commit arrives on the stage's empty barrier in all C CTAs.  The corpus
// is then read from HBM once per step however many queries the ranks gathered.
// Work split: every CTA scans a CONTIGUOUS range of 32-row "quads" (balanced to
// one quad across the grid: 100K rows over 148 SMs is 21-22 quads per CTA,
// where whole 128-row tiles would be 5 or 6); a tile is up to 4 quads of one
// stage segment, loaded as one 128-row TMA box or as 32-row boxes (same SW128
// smem layout), rows past the tile's end masked in the epilogue.
// Epilogue (4 warps): TMEM -> registers -> transposed smem tile, then each
// thread owns one (query, row-part) pair and keeps an exact top-KL list in
// registers (score desc, id asc; KL = smallest of 2/4/8 >= k).  When a CTA
// leaves a stage segment its parts are reduced in smem and k entries per
// query are written to the workspace.  A merge kernel (programmatic dependent
// launch; one CTA per query, one warp per segment) reads only the CTAs that
// covered each segment, reduces them with warp-shuffle argmax rounds and emits
// each stage's prefix top-k.  (A fused last-CTA merge was measured slower: one
// CTA's dependent L2 round trips over 64 queries cost more than the launch.)
// Bound: HBM (N * dim * 2 bytes per scan).
#include <cfloat>
#include <climits>

#include "sm100.cuh"
#include "rcb_internal.h"

namespace rcb {
namespace ret {

constexpr int kThreads = 192;
constexpr int kStages = 5;
constexpr int kKL = 8;  // list length kept per (query, part); k <= kKL
constexpr int kMaxSeg = 8;
constexpr int kMaxAtoms = 16;  // dim <= 1024
constexpr int kQuad = 32;      // rows per quad (CTA range granularity, small TMA box)

struct SegInfo {
  int n_seg;
  int n_nonempty;
  long long bound[kMaxSeg + 1];  // row boundaries
  int quad_begin[kMaxSeg + 1];   // first global quad of each segment
};

__device__ __forceinline__ bool better(float s1, int i1, float s2, int i2) {
  return (s1 > s2) | ((s1 == s2) & (i1 < i2));  // bitwise: no short-circuit branches
}

// Sorted (score desc, id asc) list of KL entries in registers; insert if better
// than the tail.  Each slot is computed from the ORIGINAL neighbours, so the
// unrolled loop is a chain of selects.
template <int KL>
__device__ __forceinline__ void list_push(float (&ls)[KL], int (&li)[KL], float sc, int id) {
  if (!better(sc, id, ls[KL - 1], li[KL - 1])) return;
#pragma unroll
  for (int i = KL - 1; i > 0; --i) {
    const bool up = better(sc, id, ls[i - 1], li[i - 1]);  // e goes above slot i-1
    const bool in = better(sc, id, ls[i], li[i]);           // e lands at or above slot i
    ls[i] = up ? ls[i - 1] : (in ? sc : ls[i]);
    li[i] = up ? li[i - 1] : (in ? id : li[i]);
  }
  const bool top = better(sc, id, ls[0], li[0]);
  ls[0] = top ? sc : ls[0];
  li[0] = top ? id : li[0];
}

// warp-level exact top-k over candidates held as a sorted local list per lane;
// lane 0 writes entry r to out_s[r] / out_i[r]
template <int KL>
__device__ __forceinline__ void warp_topk_emit(float (&ls)[KL], int (&li)[KL], int k,
                                               float* out_s, int* out_i) {
  for (int r = 0; r < k; ++r) {
    const float s = ls[0];
    const int id = li[0];
    float bs = s;
    int bi = id;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(os, oi, bs, bi)) { bs = os; bi = oi; }
    }
    if (lane_id() == 0) { out_s[r] = bs; out_i[r] = bi; }
    if (bi == id && bs == s && bi != INT_MAX) {  // the winner's lane pops its head
#pragma unroll
      for (int i = 0; i < KL - 1; ++i) { ls[i] = ls[i + 1]; li[i] = li[i + 1]; }
      ls[KL - 1] = -INFINITY;
      li[KL - 1] = INT_MAX;
    }
  }
}

template <int NQ>
struct Layout {
  static constexpr int kParts = 128 / NQ;
  static constexpr uint32_t kAtomQ = NQ * 128;  // bytes of one 64-dim atom of the query block
  static constexpr uint32_t kA = 16384;         // one A stage (128 rows x 128 B)
  static constexpr int kTStride = 129;          // transposed tile row stride (floats)
  static uint32_t total(int atoms) {
    return atoms * kAtomQ + kStages * kA + NQ * kTStride * 4 + 256 + 1024;
  }
};

template <int NQ>
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&v)[NQ]) {
#pragma unroll
  for (int c = 0; c < NQ / 16; ++c) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr + c * 16));
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) v[c * 16 + i] = __uint_as_float(r[i]);
  }
}

// The unit's contiguous quad range [q_lo, q_hi).
// (a scan unit is one CTA, or one cluster sharing a range through multicast)
__device__ __forceinline__ void cta_quads(int n_quads, int unit, int n_units, int& q_lo, int& q_hi) {
  q_lo = (int)(((long long)n_quads * unit) / n_units);
  q_hi = (int)(((long long)n_quads * (unit + 1)) / n_units);
}

// Tile walk over a quad range: a tile is <= 4 quads of one segment.
struct TileWalk {
  int q, q_hi, sg;
  __device__ __forceinline__ bool next(const SegInfo& seg, int& t_sg, long long& r0, long long& r1,
                                       int& nquads) {
    if (q >= q_hi) return false;
    while (sg + 1 < seg.n_seg && q >= seg.quad_begin[sg + 1]) ++sg;
    int n = q_hi - q;
    if (n > 4) n = 4;
    if (n > seg.quad_begin[sg + 1] - q) n = seg.quad_begin[sg + 1] - q;
    t_sg = sg;
    r0 = seg.bound[sg] + (long long)(q - seg.quad_begin[sg]) * kQuad;
    r1 = r0 + (long long)n * kQuad;
    if (r1 > seg.bound[sg + 1]) r1 = seg.bound[sg + 1];
    nquads = n;
    q += n;
    return true;
  }
};

template <int NQ, int KL>
__global__ void __launch_bounds__(kThreads, 1)
    topk_scan_kernel(const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_c32,
                     const __grid_constant__ CUtensorMap tm_q, int atoms, int n_quads,
                     const __grid_constant__ SegInfo seg, int k, float* __restrict__ part_score,
                     int* __restrict__ part_id, float* __restrict__ scores_out, int n_queries,
                     int csize) {
  using Lay = Layout<NQ>;
  constexpr int kParts = Lay::kParts;
  // the merge kernel (programmatic stream serialization) may launch now; it
  // waits in griddepcontrol.wait until this grid has completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sA = sQ + atoms * Lay::kAtomQ;
  float* sT = reinterpret_cast<float*>(sA + kStages * Lay::kA);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sT) + NQ * Lay::kTStride * 4);
  uint64_t* full = bar;                     // [kStages]
  uint64_t* empty = bar + kStages;          // [kStages]
  uint64_t* acc_full = bar + 2 * kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint64_t* q_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 1);

  const int warp = threadIdx.x >> 5;
  constexpr uint32_t kTmemCols = (2 * NQ <= 32) ? 32 : (2 * NQ <= 64 ? 64 : 128);
  // cluster of csize CTAs: rank r holds queries [NQ r, NQ r + NQ), all scan the unit's rows
  const int rank = csize > 1 ? (int)cluster_ctarank() : 0;
  const int unit = blockIdx.x / csize, n_units = gridDim.x / csize;
  const uint16_t mc_mask = (uint16_t)((1u << csize) - 1u);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], csize);  // every CTA of the cluster releases a multicast stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (csize > 1) cluster_sync();  // peers' barriers are initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  int q_lo, q_hi;
  cta_quads(n_quads, unit, n_units, q_lo, q_hi);

  if (warp == 4) {
    if (elect_one()) {
      tma_prefetch(&tm_c);
      tma_prefetch(&tm_c32);
      tma_prefetch(&tm_q);
      mbar_arrive_expect_tx(q_full, atoms * Lay::kAtomQ);
      for (int a = 0; a < atoms; ++a)
        tma_load_2d(sQ + a * Lay::kAtomQ, &tm_q, q_full, a * 64, rank * NQ);
      int it = 0;
      TileWalk tw{q_lo, q_hi, 0};
      int sg, nq4;
      long long r0, r1;
      while (tw.next(seg, sg, r0, r1, nq4)) {
        for (int a = 0; a < atoms; ++a, ++it) {
          const int st = it % kStages;
          mbar_wait(&empty[st], ((it / kStages) & 1) ^ 1);
          uint8_t* dst = sA + st * Lay::kA;
          // every CTA expects the stage's bytes; one of them (alternating) loads and
          // multicasts it to all, once every CTA's MMA released the stage (empty[st])
          const bool issue = csize == 1 || it % csize == rank;
          if (nq4 == 4) {
            mbar_arrive_expect_tx(&full[st], Lay::kA);
            if (csize == 1) tma_load_2d(dst, &tm_c, &full[st], a * 64, (int)r0);
            else if (issue) tma_load_2d_mc(dst, &tm_c, &full[st], a * 64, (int)r0, mc_mask);
          } else {
            mbar_arrive_expect_tx(&full[st], nq4 * kQuad * 128);
            for (int j = 0; j < nq4; ++j) {
              if (csize == 1)
                tma_load_2d(dst + j * kQuad * 128, &tm_c32, &full[st], a * 64, (int)r0 + j * kQuad);
              else if (issue)
                tma_load_2d_mc(dst + j * kQuad * 128, &tm_c32, &full[st], a * 64,
                               (int)r0 + j * kQuad, mc_mask);
            }
          }
        }
      }
      // producer tail (clusters): every CTA's release of every stage has arrived here
      // before this CTA may exit, so no peer's multicast commit targets a finished CTA
      if (csize > 1)
        for (int t = 0; t < kStages; ++t, ++it)
          mbar_wait(&empty[it % kStages], ((it / kStages) & 1) ^ 1);
    }
  } else if (warp == 5) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, NQ, 0, 0);
      const uint32_t a_base = smem_u32(sA);
      const uint32_t q_base = smem_u32(sQ);
      mbar_wait(q_full, 0);
      tc_fence_after();
      int it = 0, li = 0;
      TileWalk tw{q_lo, q_hi, 0};
      int sg, nq4;
      long long r0, r1;
      for (; tw.next(seg, sg, r0, r1, nq4); ++li) {
        const int buf = li & 1;
        mbar_wait(&acc_empty[buf], ((li >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int a = 0; a < atoms; ++a, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (it / kStages) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = sw128_desc(a_base + st * Lay::kA + kk * 32, 16, 1024);
            const uint64_t db = sw128_desc(q_base + a * Lay::kAtomQ + kk * 32, 16, 1024);
            umma_bf16_ss(tmem + buf * NQ, da, db, idesc, (a > 0 || kk > 0) ? 1u : 0u);
          }
          if (csize > 1) umma_commit_mc(&empty[st], mc_mask);
          else umma_commit(&empty[st]);
        }
        umma_commit(&acc_full[buf]);
      }
    }
  } else {
    // epilogue: 128 threads; thread = (query q, row-part)
    const int tid = threadIdx.x;
    const int q = tid % NQ;
    const int part = tid / NQ;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    float ls[KL];
    int li_[KL];
#pragma unroll
    for (int i = 0; i < KL; ++i) { ls[i] = -INFINITY; li_[i] = INT_MAX; }
    int cur_seg = -1;
    // reduce the kParts lists of each query in smem, write k entries for this CTA
    auto flush = [&](int sg) {
      named_bar_sync(1, 128);  // sT free
      float* ms = sT;                                         // [kParts][NQ][KL]
      int* mi = reinterpret_cast<int*>(sT + kParts * NQ * KL);
#pragma unroll
      for (int i = 0; i < KL; ++i) {
        ms[(part * NQ + q) * KL + i] = ls[i];
        mi[(part * NQ + q) * KL + i] = li_[i];
      }
      named_bar_sync(1, 128);
      if (part == 0) {
        for (int p = 1; p < kParts; ++p)
#pragma unroll
          for (int i = 0; i < KL; ++i) list_push<KL>(ls, li_, ms[(p * NQ + q) * KL + i], mi[(p * NQ + q) * KL + i]);
        // workspace [segment][query][unit][k]: the merging warp of (segment, query)
        // reads the covering units' candidates contiguously
        const long long base = (((long long)sg * NQ * csize + rank * NQ + q) * n_units + unit) * k;
#pragma unroll
        for (int i = 0; i < KL; ++i)
          if (i < k) {
            part_score[base + i] = ls[i];
            part_id[base + i] = li_[i];
          }
      }
#pragma unroll
      for (int i = 0; i < KL; ++i) { ls[i] = -INFINITY; li_[i] = INT_MAX; }
    };
    int li = 0;
    TileWalk tw{q_lo, q_hi, 0};
    int sg, nq4;
    long long r0, r1;
    for (; tw.next(seg, sg, r0, r1, nq4); ++li) {
      if (sg != cur_seg) {
        if (cur_seg >= 0) flush(cur_seg);
        cur_seg = sg;
      }
      const int buf = li & 1;
      mbar_wait(&acc_full[buf], (li >> 1) & 1);
      tc_fence_after();
      float v[NQ];
      tmem_ld_row<NQ>(t_row + buf * NQ, v);
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      if (scores_out != nullptr && r0 + tid < r1) {
#pragma unroll
        for (int c = 0; c < NQ; ++c)
          if (rank * NQ + c < n_queries) scores_out[(r0 + tid) * n_queries + rank * NQ + c] = v[c];
      }
      named_bar_sync(1, 128);  // previous tile's readers are done with sT
#pragma unroll
      for (int c = 0; c < NQ; ++c) sT[c * Lay::kTStride + tid] = v[c];
      named_bar_sync(1, 128);
      const int row_lo = part * NQ;
      const int nvalid = (int)(r1 - r0);
      const float* col = sT + q * Lay::kTStride;
      if (row_lo + NQ <= nvalid) {
#pragma unroll 8
        for (int r = 0; r < NQ; ++r) list_push<KL>(ls, li_, col[row_lo + r], (int)r0 + row_lo + r);
      } else {
        for (int r = 0; r < NQ && row_lo + r < nvalid; ++r)
          list_push<KL>(ls, li_, col[row_lo + r], (int)r0 + row_lo + r);
      }
    }
    if (cur_seg >= 0) flush(cur_seg);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  if (csize > 1) cluster_sync();  // no CTA leaves while a peer may still multicast into it
}

// grid = n_queries, block = 32 * n_seg; warp s reduces the candidates of the
// scan CTAs that covered segment s, then emits stage s = prefix merge of 0..s
__global__ void topk_merge_kernel(const float* __restrict__ part_score,
                                  const int* __restrict__ part_id, int scan_grid, int n_quads,
                                  int NQ, const __grid_constant__ SegInfo seg, int k,
                                  long long id_offset, long long* __restrict__ ids_out,
                                  float* __restrict__ scores_out) {
  __shared__ float seg_s[kMaxSeg][kKL];
  __shared__ int seg_i[kMaxSeg][kKL];
  __shared__ float out_s[kMaxSeg][kKL];
  __shared__ int out_i[kMaxSeg][kKL];
  const int q = blockIdx.x;
  const int s = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_seg = seg.n_seg;
  // covering CTAs of segment s (the scan's quad_owner with the scan's grid)
  auto owner = [&](int qd) {
    return (int)((((long long)qd + 1) * scan_grid + n_quads - 1) / n_quads) - 1;
  };
  const bool empty = seg.quad_begin[s + 1] == seg.quad_begin[s];
  const int c_lo = empty ? 0 : owner(seg.quad_begin[s]);
  const int n_cand = empty ? 0 : (owner(seg.quad_begin[s + 1] - 1) - c_lo + 1) * k;
  const long long base = (((long long)s * NQ + q) * scan_grid + c_lo) * k;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scan grid completed
  float ls[kKL];
  int li[kKL];
#pragma unroll
  for (int i = 0; i < kKL; ++i) { ls[i] = -INFINITY; li[i] = INT_MAX; }
  // coalesced, 8 loads in flight per lane before the list updates
  for (int c0 = 0; c0 < n_cand; c0 += 32 * 8) {
    float cs[8];
    int ci[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      cs[u] = c < n_cand ? __ldg(part_score + base + c) : -INFINITY;
      ci[u] = c < n_cand ? __ldg(part_id + base + c) : INT_MAX;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) list_push<kKL>(ls, li, cs[u], ci[u]);
  }
  warp_topk_emit<kKL>(ls, li, k, seg_s[s], seg_i[s]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kKL; ++i) { ls[i] = -INFINITY; li[i] = INT_MAX; }
  for (int c = lane; c < (s + 1) * k; c += 32) list_push<kKL>(ls, li, seg_s[c / k][c % k], seg_i[c / k][c % k]);
  warp_topk_emit<kKL>(ls, li, k, out_s[s], out_i[s]);
  __syncwarp();
  if (lane < k) {
    const long long o = ((long long)q * n_seg + s) * k + lane;
    const int id = out_i[s][lane];
    ids_out[o] = (id == INT_MAX) ? -1 : (long long)id + id_offset;
    scores_out[o] = out_s[s][lane];
  }
}

// grid = n_queries * n_stages, block = 32
__global__ void shard_merge_kernel(const long long* __restrict__ ids_in,
                                   const float* __restrict__ scores_in, int n_shards, int nq,
                                   int n_stages, int k, long long* __restrict__ ids_out,
                                   float* __restrict__ scores_out) {
  const int qs = blockIdx.x;  // q * n_stages + s
  const int lane = threadIdx.x;
  // candidates carry int64 ids; rank them with (score desc, id asc)
  float bs_list[kKL];
  long long bi_list[kKL];
#pragma unroll
  for (int i = 0; i < kKL; ++i) { bs_list[i] = -INFINITY; bi_list[i] = LLONG_MAX; }
  for (int c = lane; c < n_shards * k; c += 32) {
    const int sh = c / k, e = c % k;
    const long long idx = ((long long)sh * nq * n_stages + qs) * k + e;
    const float sc = scores_in[idx];
    long long id = ids_in[idx];
    if (id < 0) id = LLONG_MAX;
    if (sc > bs_list[kKL - 1] || (sc == bs_list[kKL - 1] && id < bi_list[kKL - 1])) {
#pragma unroll
      for (int i = kKL - 1; i >= 0; --i) {
        const bool bi = sc > bs_list[i] || (sc == bs_list[i] && id < bi_list[i]);
        const bool bp = (i == 0) ? false
                                 : (sc > bs_list[i - 1] || (sc == bs_list[i - 1] && id < bi_list[i - 1]));
        if (bi) {
          bs_list[i] = bp ? bs_list[i - 1] : sc;
          bi_list[i] = bp ? bi_list[i - 1] : id;
        }
      }
    }
  }
  for (int r = 0; r < k; ++r) {
    float bs = bs_list[0];
    long long bi = bi_list[0];
    const float mys = bs;
    const long long myi = bi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (os > bs || (os == bs && oi < bi)) { bs = os; bi = oi; }
    }
    if (lane == 0) {
      ids_out[(long long)qs * k + r] = (bi == LLONG_MAX) ? -1 : bi;
      scores_out[(long long)qs * k + r] = bs;
    }
    if (bi == myi && bs == mys && bi != LLONG_MAX) {
#pragma unroll
      for (int i = 0; i < kKL - 1; ++i) { bs_list[i] = bs_list[i + 1]; bi_list[i] = bi_list[i + 1]; }
      bs_list[kKL - 1] = -INFINITY;
      bi_list[kKL - 1] = LLONG_MAX;
    }
  }
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

constexpr int kMaxQueries = 256;
// queries per CTA (padded) and CTAs per cluster: <= 64 queries run on one CTA per range,
// more as a cluster of 2 or 4 CTAs x 64 queries sharing each multicast corpus stage
int nq_pad(int n) { return n <= 16 ? 16 : (n <= 32 ? 32 : 64); }
int cluster_for(int n) { return n <= 64 ? 1 : (n <= 128 ? 2 : 4); }

void make_segments(int64_t n_rows, int n_stages, SegInfo& seg, int& n_quads) {
  seg.n_seg = n_stages;
  seg.n_nonempty = 0;
  int q = 0;
  for (int s = 0; s <= n_stages; ++s) seg.bound[s] = (long long)((n_rows * s) / n_stages);
  for (int s = 0; s < n_stages; ++s) {
    seg.quad_begin[s] = q;
    const long long len = seg.bound[s + 1] - seg.bound[s];
    q += (int)((len + kQuad - 1) / kQuad);
    seg.n_nonempty += len > 0;
  }
  seg.quad_begin[n_stages] = q;
  for (int s = n_stages + 1; s <= kMaxSeg; ++s) { seg.bound[s] = n_rows; seg.quad_begin[s] = q; }
  n_quads = q;
}

// scan units (a CTA, or a cluster of csize CTAs) over the corpus ranges
int units_for(int n_quads, int csize) {
  const int g = num_sms() / csize;
  return n_quads < g ? (n_quads > 0 ? n_quads : 1) : g;
}

// workspace: partial lists [n_seg][NQ * csize][units][k] (score f32, then id i32)
int64_t part_entries(int64_t n_rows, int n_queries, int k, int n_stages) {
  SegInfo seg;
  int n_quads;
  make_segments(n_rows, n_stages, seg, n_quads);
  const int cs = cluster_for(n_queries);
  return int64_t(n_stages) * nq_pad(n_queries) * cs * units_for(n_quads, cs) * (k < 1 ? 1 : k);
}

template <int NQ, int KL>
int run_scan_kl(const CUtensorMap& tc, const CUtensorMap& tc32, const CUtensorMap& tq, int atoms,
                int n_quads, const SegInfo& seg, int k, float* part_score, int* part_id,
                float* scores_out, int n_queries, int& units, int csize,
                cudaStream_t stream) {
  const uint32_t smem = Layout<NQ>::total(atoms);
  auto kern = topk_scan_kernel<NQ, KL>;
  static uint32_t smem_set = 0;  // per instantiation: set the attribute once per size
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "retrieval smem attr");
    smem_set = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * csize);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = csize > 1 ? 1 : 0;
  if (csize > 1) {
    // clusters live inside one GPC: at most this many are co-resident; a second wave would
    // double the scan, so the ranges are cut for the resident clusters only
    static int max_clusters[5] = {0, 0, 0, 0, 0};  // per instantiation and cluster size
    if (max_clusters[csize] == 0) {
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      max_clusters[csize] = (e == cudaSuccess && n > 0) ? n : num_sms() / csize;
    }
    if (units > max_clusters[csize]) units = max_clusters[csize];
    cfg.gridDim = dim3(units * csize);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tc, tc32, tq, atoms, n_quads, seg, k, part_score,
                                     part_id, scores_out, n_queries, csize);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "retrieval scan launch");
  return RCB_OK;
}

template <int NQ>
int run_scan(const void* corpus, int64_t n_rows, int dim, const void* queries, int n_queries,
             int n_stages, int k, float* part_score, int* part_id, float* scores_out,
             int& units, int csize, cudaStream_t stream) {
  SegInfo seg;
  int n_quads;
  make_segments(n_rows, n_stages, seg, n_quads);
  CUtensorMap tc, tc32, tq;
  {
    const uint64_t dims[2] = {(uint64_t)dim, (uint64_t)n_rows};
    const uint64_t strides[1] = {(uint64_t)dim * 2};
    const uint32_t box[2] = {64, 128};
    int rc = encode_tma_bf16(&tc, corpus, 2, dims, strides, box);
    if (rc != RCB_OK) return rc;
    const uint32_t box32[2] = {64, (uint32_t)kQuad};
    rc = encode_tma_bf16(&tc32, corpus, 2, dims, strides, box32);
    if (rc != RCB_OK) return rc;
  }
  {
    const uint64_t dims[2] = {(uint64_t)dim, (uint64_t)n_queries};
    const uint64_t strides[1] = {(uint64_t)dim * 2};
    const uint32_t box[2] = {64, (uint32_t)NQ};
    int rc = encode_tma_bf16(&tq, queries, 2, dims, strides, box);
    if (rc != RCB_OK) return rc;
  }
  const int atoms = dim / 64;
  if (k <= 2)
    return run_scan_kl<NQ, 2>(tc, tc32, tq, atoms, n_quads, seg, k, part_score, part_id, scores_out, n_queries, units, csize, stream);
  if (k <= 4)
    return run_scan_kl<NQ, 4>(tc, tc32, tq, atoms, n_quads, seg, k, part_score, part_id, scores_out, n_queries, units, csize, stream);
  return run_scan_kl<NQ, 8>(tc, tc32, tq, atoms, n_quads, seg, k, part_score, part_id, scores_out, n_queries, units, csize, stream);
}

int scan(const void* corpus, int64_t n_rows, int dim, const void* queries, int n_queries,
         int n_stages, int k, float* part_score, int* part_id, float* scores_out,
         int& units, int csize, cudaStream_t stream) {
  switch (nq_pad(n_queries)) {
    case 16: return run_scan<16>(corpus, n_rows, dim, queries, n_queries, n_stages, k, part_score, part_id, scores_out, units, csize, stream);
    case 32: return run_scan<32>(corpus, n_rows, dim, queries, n_queries, n_stages, k, part_score, part_id, scores_out, units, csize, stream);
    default: return run_scan<64>(corpus, n_rows, dim, queries, n_queries, n_stages, k, part_score, part_id, scores_out, units, csize, stream);
  }
}

int check_args(int64_t n_rows, int dim, int n_queries, int n_stages) {
  if (n_rows <= 0 || n_rows >= INT_MAX) return set_error(RCB_ERR_ARG, "n_rows out of range");
  if (dim <= 0 || dim % 64 != 0 || dim / 64 > kMaxAtoms) return set_error(RCB_ERR_ARG, "dim must be a multiple of 64, <= 1024");
  if (n_queries <= 0 || n_queries > kMaxQueries) return set_error(RCB_ERR_ARG, "1 <= n_queries <= 256");
  if (n_stages <= 0 || n_stages > kMaxSeg) return set_error(RCB_ERR_ARG, "1 <= n_stages <= 8");
  return RCB_OK;
}

}  // namespace ret
}  // namespace rcb

using namespace rcb;

extern "C" int64_t rcb_retrieval_workspace_bytes(int64_t n_rows, int32_t n_queries, int32_t k,
                                                 int32_t n_stages) {
  if (n_rows <= 0 || n_stages <= 0 || n_stages > ret::kMaxSeg) return 16;
  return ret::part_entries(n_rows, n_queries, k, n_stages) * 8;
}

extern "C" int rcb_retrieval_topk(const void* corpus_dev, int64_t n_rows, int32_t dim,
                                  const void* queries_dev, int32_t n_queries, int32_t k,
                                  int32_t n_stages, int64_t id_offset, void* workspace_dev,
                                  int64_t workspace_bytes, int64_t* ids_out_dev,
                                  float* scores_out_dev, void* stream) {
  int rc = ret::check_args(n_rows, dim, n_queries, n_stages);
  if (rc != RCB_OK) return rc;
  if (k < 1 || k > ret::kKL) return set_error(RCB_ERR_ARG, "1 <= k <= 8");
  const int64_t entries = ret::part_entries(n_rows, n_queries, k, n_stages);
  if (workspace_bytes < entries * 8) return set_error(RCB_ERR_ARG, "retrieval workspace too small");
  ret::SegInfo seg;
  int n_quads;
  ret::make_segments(n_rows, n_stages, seg, n_quads);
  const int csize = ret::cluster_for(n_queries);
  int units = ret::units_for(n_quads, csize);  // the scan may launch fewer (resident clusters)
  float* ps = static_cast<float*>(workspace_dev);
  int* pi = reinterpret_cast<int*>(ps + entries);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = ret::scan(corpus_dev, n_rows, dim, queries_dev, n_queries, n_stages, k, ps, pi, nullptr,
                 units, csize, st);
  if (rc != RCB_OK) return rc;
  // programmatic dependent launch: the merge's launch overlaps the scan's tail
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_queries);
  cfg.blockDim = dim3(32 * n_stages);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, ret::topk_merge_kernel, static_cast<const float*>(ps),
                                     static_cast<const int*>(pi), units, n_quads,
                                     ret::nq_pad(n_queries) * csize, seg, k,
                                     static_cast<long long>(id_offset),
                                     reinterpret_cast<long long*>(ids_out_dev), scores_out_dev);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "retrieval merge launch");
  return RCB_OK;
}

extern "C" int rcb_retrieval_scores(const void* corpus_dev, int64_t n_rows, int32_t dim,
                                    const void* queries_dev, int32_t n_queries,
                                    float* scores_out_dev, void* stream) {
  int rc = ret::check_args(n_rows, dim, n_queries, 1);
  if (rc != RCB_OK) return rc;
  const int64_t entries = ret::part_entries(n_rows, n_queries, 1, 1);
  ret::SegInfo seg;
  int n_quads;
  ret::make_segments(n_rows, 1, seg, n_quads);
  const int csize = ret::cluster_for(n_queries);
  int units = ret::units_for(n_quads, csize);
  void* buf = nullptr;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMallocAsync(&buf, entries * 8, st);
  if (e != cudaSuccess) return set_cuda_error(e, "retrieval scores workspace");
  float* ps = static_cast<float*>(buf);
  int* pi = reinterpret_cast<int*>(ps + entries);
  rc = ret::scan(corpus_dev, n_rows, dim, queries_dev, n_queries, 1, 1, ps, pi, scores_out_dev,
                 units, csize, st);
  cudaFreeAsync(buf, st);
  return rc;
}

extern "C" int rcb_topk_merge_shards(const int64_t* ids_in_dev, const float* scores_in_dev,
                                     int32_t n_shards, int32_t n_queries, int32_t n_stages,
                                     int32_t k, int64_t* ids_out_dev, float* scores_out_dev,
                                     void* stream) {
  if (n_shards < 1 || n_queries < 1 || n_stages < 1 || k < 1 || k > ret::kKL)
    return set_error(RCB_ERR_ARG, "bad shard-merge shape");
  ret::shard_merge_kernel<<<n_queries * n_stages, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long*>(ids_in_dev), scores_in_dev, n_shards, n_queries,
      n_stages, k, reinterpret_cast<long long*>(ids_out_dev), scores_out_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "shard merge launch");
  return RCB_OK;
}
