// prefix_attn.cu — prefix-aware prefill attention over the paged doc-KV pool.
//
// Replaces the reference's latency stand-in T(alpha, beta)
// (ragsim cost_model.py:106-117 `interpolate`, called at simulator.py:506 and
// tree.py:240): here the alpha cached tokens are READ from knowledge-tree node
// blocks through a block table, and only the beta suffix tokens (miss docs +
// prompt) are computed as queries.
//
// Persistent CTAs (one per SM) walk a heaviest-first list of work items
// (request, query tile, kv head), pipelining across items:
//   * 128 query rows = (128/G tokens) x (G query heads sharing the kv head)
//   * K/V tiles of 128 key slots = 128/BT pool blocks, TMA-loaded (SW128)
//   * S = Q K^T and O += P V on tcgen05 (fp32 accumulators in TMEM)
//   * online softmax in registers, split over KV-tile parity: warpgroup A (warps 0-3)
//     owns the even tiles (S buffer 0, accumulator O_A), warpgroup B (warps 12-15) the
//     odd ones (S buffer 1, O_B), each with its own running max / row sum, so the two
//     chains never synchronise and ping-pong on the tensor core; lazily rescaled O (only
//     when a running max grows by > 2^8); the epilogue merges (O_A, m_A, l_A) and
//     (O_B, m_B, l_B)
// Warp roles: 0-3 / 12-15 softmax, 4 Q/K TMA producer, 5 MMA issuer + TMEM owner,
// 6 V TMA producer, 8-11 epilogue.
//
// Key slots carry holes (node tails: a block holds `valid` <= BT tokens), so
// each block also carries its logical start position; a slot is attended iff
// off < valid && pos <= query_pos (causal on logical positions).
#include "sm100.cuh"
#include "rcb_internal.h"

namespace rcb {

namespace attn {

// WG0 (warps 0-3) softmax, even KV tiles | WG1: warp 4 Q+K producer, 5 MMA, 6 V producer,
// 7 idle | WG2 (warps 8-11) epilogue (+ in-smem Q RoPE with a table) | WG3 (warps 12-15)
// softmax, odd KV tiles.  Two independent softmax warps per SM sub-partition hide each
// other's MUFU and dependency latency.  setmaxnreg moves registers from WG1 to the others.
constexpr int kThreads = 512;
constexpr int kRows = 128;
constexpr int kKeys = 128;  // key slots per KV tile
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// exp2 on the FMA pipe (cubic polynomial) for kPolyCols of every 8 score columns.  Measured
// on B200 with two softmax warps per sub-partition: 0 (all MUFU) is fastest -- the softmax
// chain is latency-bound and the polynomial only adds instructions (2/8: +4%, 4/8: +13%)
#ifndef RCB_POLY_COLS
#define RCB_POLY_COLS 0
#endif
constexpr int kPolyCols = RCB_POLY_COLS;

template <int HD, int BT>
struct Smem {
  static constexpr uint32_t kHalves = HD / 64;
  static constexpr uint32_t kQ = kHalves * 16384;   // one Q tile
  static constexpr uint32_t kKV = kHalves * 16384;  // one K or V stage
  static constexpr int kBPT = kKeys / BT;
  static constexpr uint32_t offQ = 0;                // [2]
  static constexpr uint32_t offK = offQ + 2 * kQ;    // [2]
  static constexpr uint32_t offV = offK + 2 * kKV;   // [2]
  static constexpr int kMetaSlots = 4;
  static constexpr uint32_t offMeta = offV + 2 * kKV;  // int [kMetaSlots][2][kBPT]
  static constexpr uint32_t offL = offMeta + kMetaSlots * 2 * kBPT * 4;  // float2 [2][2][128]
  static constexpr uint32_t offBar = offL + 2 * 2 * 128 * 8;
  static constexpr uint32_t kTotal = offBar + 40 * 8 + 16 + 1024;  // + alignment slack
};

// Per-tile handoff timestamps of CTA 0 (debug builds with -DRCB_TRACE only)
#ifdef RCB_TRACE
constexpr int kTraceTiles = 512;
constexpr int kTraceEv = 16;
__device__ long long g_trace[kTraceTiles * kTraceEv];
#define TRACE(g, ev)                                                         \
  do {                                                                       \
    if (blockIdx.x == 0 && (g) < kTraceTiles) g_trace[(g) * kTraceEv + (ev)] = clock64(); \
  } while (0)
#else
#define TRACE(g, ev) \
  do {               \
  } while (0)
#endif

// S, P and O buffers are indexed by tile parity p (= owning softmax WG); Q, L, O-full by
// item parity.
enum Bar {
  kQFull0 = 0, kQEmpty0 = 2, kKFull0 = 4, kVFull0 = 6, kKEmpty0 = 8, kSFull0 = 10, kLFree0 = 12,
  kPFull0 = 14, kOFull0 = 16, kOFree0 = 18, kVEmpty0 = 20, kMetaFull0 = 22,
  kMetaFree0 = 26, kLFull0 = 30, kQReady0 = 32, kNumBars = 34
};

// Work items are self-contained (no dependent loads at item start):
//   {q_start, q_len, q_pos0, blk_begin, blk_count, q_tile, kv_head, n_kv_tiles}
constexpr int kItemInts = 8;
struct Item {
  int q_start, q_len, q_pos0, blk_begin, blk_count, qt, kvh, n;
};

__device__ __forceinline__ Item load_item(const int* __restrict__ work, int idx) {
  const int4 a = *reinterpret_cast<const int4*>(work + idx * kItemInts);
  const int4 b = *reinterpret_cast<const int4*>(work + idx * kItemInts + 4);
  return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

// Persistent: CTA c serves work items c, c + grid, ... (heaviest first).
// Per-CTA tile sequence number g runs across items, so K/V stages, S buffers
// and the P handshake keep their phase; Q (smem) and O (TMEM) are double
// buffered per item so item i's epilogue overlaps item i+1's first tiles.
template <int HD, int G, int BT>
__global__ void __launch_bounds__(kThreads, 1)
    prefix_prefill_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_kv,
                          __nv_bfloat16* __restrict__ out, int n_q_heads, int layer,
                          const int* __restrict__ req_meta, const int* __restrict__ blk_ids,
                          const int* __restrict__ blk_valid, const int* __restrict__ blk_pos,
                          const int* __restrict__ work, int n_work, float scale_log2,
                          const float2* __restrict__ rope) {
  using S = Smem<HD, BT>;
  constexpr int TQ = kRows / G;
  constexpr int BPT = S::kBPT;
  extern __shared__ uint8_t smem_raw[];
  // align within the shared window without leaving the shared address space
  // (keeps st.shared / ld.shared instead of generic accesses)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + S::offQ;
  uint8_t* sK = smem + S::offK;
  uint8_t* sV = smem + S::offV;
  int* sMeta = reinterpret_cast<int*>(smem + S::offMeta);  // [slot][0=valid,1=pos][BPT]
  float2* sML = reinterpret_cast<float2*>(smem + S::offL);  // [item parity][WG][row] (m, l)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::offBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + kNumBars);

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar[kQFull0 + b], 1);
      mbar_init(&bar[kQEmpty0 + b], 1);
      mbar_init(&bar[kKFull0 + b], 1);
      mbar_init(&bar[kVFull0 + b], 1);
      mbar_init(&bar[kKEmpty0 + b], 1);
      mbar_init(&bar[kVEmpty0 + b], 1);
      mbar_init(&bar[kSFull0 + b], 1);
      mbar_init(&bar[kPFull0 + b], kRows);
      mbar_init(&bar[kOFull0 + b], 1);
      mbar_init(&bar[kOFree0 + b], kRows);
      mbar_init(&bar[kLFree0 + b], kRows);
    }
    for (int b = 0; b < S::kMetaSlots; ++b) {
      mbar_init(&bar[kMetaFull0 + b], 1);
      mbar_init(&bar[kMetaFree0 + b], kRows);  // the tile's owning WG
    }
    mbar_init(&bar[kLFull0 + 0], 2 * kRows);  // both WGs publish (m, l) for every item
    mbar_init(&bar[kLFull0 + 1], 2 * kRows);
    mbar_init(&bar[kQReady0 + 0], kRows);
    mbar_init(&bar[kQReady0 + 1], kRows);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 4 && warp < 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
  }
  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_kv);
      int g = 0;
      int q_issued = 0;  // items whose Q load has been issued
      auto issue_q = [&](int idx, int ii) {
        const Item it = load_item(work, idx);
        const int qb = ii & 1;
        mbar_arrive_expect_tx(&bar[kQFull0 + qb], S::kQ);
        for (int h = 0; h < (int)S::kHalves; ++h)
          tma_load_3d(sQ + qb * S::kQ + h * 16384, &tm_q, &bar[kQFull0 + qb], h * 64,
                      it.kvh * G, it.q_start + it.qt * TQ);
      };
      for (int idx = blockIdx.x, ii = 0; idx < n_work; idx += gridDim.x, ++ii) {
        const Item it = load_item(work, idx);
        if (q_issued == ii) {
          mbar_wait(&bar[kQEmpty0 + (ii & 1)], ((ii >> 1) & 1) ^ 1);
          issue_q(idx, ii);
          ++q_issued;
        }
        for (int j = 0; j < it.n; ++j, ++g) {
          const int st = g & 1;
          // next item's Q as soon as its buffer frees (QK of item ii-1 retired): it then
          // lands a whole item ahead of its first MMA
          if (q_issued == ii + 1 &&
              idx + (int)gridDim.x < n_work &&
              mbar_test(&bar[kQEmpty0 + ((ii + 1) & 1)], (((ii + 1) >> 1) & 1) ^ 1)) {
            issue_q(idx + gridDim.x, ii + 1);
            ++q_issued;
          }
          // per-tile mask metadata: its own 4-slot ring (the softmax may lag the K ring)
          const int ms = g & (S::kMetaSlots - 1);
          mbar_wait(&bar[kMetaFree0 + ms], ((g / S::kMetaSlots) & 1) ^ 1);
          int ids[BPT];
#pragma unroll
          for (int b = 0; b < BPT; ++b) {
            const int sb = j * BPT + b;
            const bool in = sb < it.blk_count;
            // slots past the table load a real (finite) block; they are masked
            ids[b] = blk_ids[it.blk_begin + (in ? sb : 0)];
            sMeta[(ms * 2 + 0) * BPT + b] = in ? blk_valid[it.blk_begin + sb] : 0;
            sMeta[(ms * 2 + 1) * BPT + b] = in ? blk_pos[it.blk_begin + sb] : 0;
          }
          mbar_arrive(&bar[kMetaFull0 + ms]);  // release: publishes sMeta[ms]
          mbar_wait(&bar[kKEmpty0 + st], ((g >> 1) & 1) ^ 1);  // QK(g-2) retired
          mbar_arrive_expect_tx(&bar[kKFull0 + st], S::kKV);
#pragma unroll
          for (int b = 0; b < BPT; ++b)
            for (int h = 0; h < (int)S::kHalves; ++h)
              tma_load_5d(sK + st * S::kKV + h * 16384 + b * BT * 128, &tm_kv,
                          &bar[kKFull0 + st], h * 64, 0, it.kvh, 2 * layer, ids[b]);
        }
      }
    }
  } else if (warp == 6) {
    // ------------------------------------------------------------ V producer
    // V(g) is only needed by PV(g); its stage frees when PV(g) retires, while K
    // stages free as soon as QK(g) retires — separate rings keep both ahead.
    if (elect_one()) {
      int g = 0;
      for (int idx = blockIdx.x; idx < n_work; idx += gridDim.x) {
        const Item it = load_item(work, idx);
        const int n = it.n, kvh = it.kvh, blk_begin = it.blk_begin, blk_count = it.blk_count;
        for (int j = 0; j < n; ++j, ++g) {
          const int st = g & 1;
          mbar_wait(&bar[kVEmpty0 + st], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&bar[kVFull0 + st], S::kKV);
#pragma unroll
          for (int b = 0; b < BPT; ++b) {
            const int sb = j * BPT + b;
            const int id = blk_ids[blk_begin + (sb < blk_count ? sb : 0)];
            for (int h = 0; h < (int)S::kHalves; ++h)
              tma_load_5d(sV + st * S::kKV + h * 16384 + b * BT * 128, &tm_kv,
                          &bar[kVFull0 + st], h * 64, 0, kvh, 2 * layer + 1, id);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, kKeys, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, HD, 0, 1);
      const uint32_t q_base = smem_u32(sQ);
      const uint32_t k_base = smem_u32(sK);
      const uint32_t v_base = smem_u32(sV);
      struct T {
        int idx, ii, j, n, g;
      };
      auto first = [&](T& t) {
        t.idx = blockIdx.x;
        t.ii = 0;
        t.j = 0;
        t.g = 0;
        t.n = (t.idx < n_work) ? work[t.idx * kItemInts + 7] : 0;
      };
      auto next = [&](T t) {
        ++t.g;
        if (++t.j == t.n) {
          t.j = 0;
          ++t.ii;
          t.idx += gridDim.x;
          t.n = (t.idx < n_work) ? work[t.idx * kItemInts + 7] : 0;
        }
        return t;
      };
      auto issue_qk = [&](const T& t) {
        const int qb = t.ii & 1;
        const int st = t.g & 1;
        if (t.j == 0)  // Q landed (and, with fused RoPE, rotated by the epilogue WG)
          mbar_wait(&bar[(rope != nullptr ? kQReady0 : kQFull0) + qb], (t.ii >> 1) & 1);
        TRACE(t.g, 8);
        mbar_wait(&bar[kKFull0 + st], (t.g >> 1) & 1);
        TRACE(t.g, 9);
        // S buffer st: its previous tile's PV (the P reader, issued after P-full, i.e.
        // after the softmax read S) precedes this MMA in issue order
        tc_fence_after();
        const uint32_t d = tmem + st * kKeys;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint64_t a = sw128_desc(q_base + qb * S::kQ + off, 16, 1024);
          const uint64_t b = sw128_desc(k_base + st * S::kKV + off, 16, 1024);
          umma_bf16_ss(d, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&bar[kSFull0 + st]);
        umma_commit(&bar[kKEmpty0 + st]);                       // K stage no longer read
        if (t.j == t.n - 1) umma_commit(&bar[kQEmpty0 + qb]);  // Q tile no longer read
      };
      auto issue_pv = [&](const T& t) {
        const int st = t.g & 1;  // = owning WG = its O accumulator
        // first PV into O_st of this item: the previous item's epilogue has read O_st
        if (t.j < 2) mbar_wait(&bar[kOFree0 + st], (t.ii & 1) ^ 1);
        TRACE(t.g, 11);
        mbar_wait(&bar[kPFull0 + st], (t.g >> 1) & 1);
        TRACE(t.g, 12);
        mbar_wait(&bar[kVFull0 + st], (t.g >> 1) & 1);
        TRACE(t.g, 13);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kKeys / 16; ++kk) {
          // A = P (bf16 pairs) written by the softmax over its S buffer's first 64 columns;
          // QK(g+2) is issued after this PV, and tcgen05.mma executes in issue order
          const uint32_t a = tmem + st * kKeys + kk * 8;
          // V tile is [half][128 keys][64]: MN-major, halves 16 KB apart (LBO)
          const uint64_t b = sw128_desc(v_base + st * S::kKV + kk * 2048, 16384, 1024);
          umma_bf16_ts(tmem + 256 + st * 128, a, b, idesc_pv, (t.j > 1 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&bar[kVEmpty0 + st]);
        if (t.j == t.n - 1) umma_commit(&bar[kOFull0 + (t.ii & 1)]);  // both O_A and O_B
      };
      T cur;
      first(cur);
      if (cur.n > 0) {
        issue_qk(cur);
        while (true) {
          const T nx = next(cur);
          const bool more = nx.n > 0;
          if (more) issue_qk(nx);  // next QK (possibly the next item's) before this PV
          issue_pv(cur);
          if (!more) break;
          cur = nx;
        }
      }
    }
  } else if (warp < 4 || warp >= 12) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 176;\n" ::: "memory");
    // ------------------------------------------------------------ softmax, one tile parity
    const int wg = warp >= 12 ? 1 : 0;  // owns tiles g with g % 2 == wg (S_wg, O_wg)
    const int quad = warp & 3;
    const int row = quad * 32 + (threadIdx.x & 31);  // == TMEM lane
    const int t_local = row / G;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t s_col = t_row + wg * kKeys;        // this WG's S / P buffer
    const uint32_t o_col = t_row + 256 + wg * 128;    // this WG's O accumulator
    const bool tr = threadIdx.x == 0;
    float s[kKeys / 2];
    int g = 0;
    for (int idx = blockIdx.x, ii = 0; idx < n_work; idx += gridDim.x, ++ii) {
      const Item it = load_item(work, idx);
      const int tok = it.qt * TQ + t_local;
      const int qp = it.q_pos0 + tok;
      float m = -INFINITY;  // running max (scaled, log2 domain); may be stale by < 2^8
      float l = 0.f;
      bool any = false;    // m initialised (first chunk of this WG in the item)
      bool first = true;   // no PV of this WG in the item yet (O_wg not yet written)
      for (int j = 0; j < it.n; ++j, ++g) {
        if ((g & 1) != wg) continue;
        const int ms = g & (S::kMetaSlots - 1);
        mbar_wait(&bar[kMetaFull0 + ms], (g / S::kMetaSlots) & 1);
        int vv[BPT], pp[BPT];
        bool all_valid = true;
        int max_pos = -1;
#pragma unroll
        for (int b = 0; b < BPT; ++b) {
          vv[b] = sMeta[(ms * 2 + 0) * BPT + b];
          pp[b] = sMeta[(ms * 2 + 1) * BPT + b];
          all_valid &= (vv[b] == BT);
          max_pos = max(max_pos, pp[b] + vv[b] - 1);
        }
        mbar_arrive(&bar[kMetaFree0 + ms]);
        if (tr) TRACE(g, 0);
        // S-full(g) also means every earlier tcgen05 op retired: PV(g-2) into O_wg
        mbar_wait(&bar[kSFull0 + wg], (g >> 1) & 1);
        if (tr) TRACE(g, 1);
        tc_fence_after();
        const bool masked = !all_valid || max_pos > qp;
        // Two 64-column chunks against the running max m (within 2^8 of the true row max:
        // a chunk that exceeds m + 2^8 rescales O, l and the already-packed P of chunk 0).
        // P of chunk c (bf16 pairs) goes to S columns [32c, 32c + 32): chunk 0's own
        // columns, then chunk 0's (already consumed) columns for chunk 1.
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          {
            uint32_t r[kKeys / 2];
            tmem_ld64(s_col + ch * (kKeys / 2), r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < kKeys / 2; ++i) s[i] = __uint_as_float(r[i]);
          }
          if (tr && ch == 0) TRACE(g, 2);
          if (masked) {
            // keys valid in block b for this row: off < min(valid_b, qp - pos_b + 1)
#pragma unroll
            for (int c = 0; c < kKeys / 2; ++c) {
              const int cc = ch * (kKeys / 2) + c;
              const int b = cc / BT;
              s[c] = (cc % BT) < min(vv[b], qp - pp[b] + 1) ? s[c] : -INFINITY;
            }
          }
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
          for (int c = 0; c < kKeys / 2; c += 8) {
            mx0 = fmax3(mx0, s[c + 0], s[c + 1]);
            mx1 = fmax3(mx1, s[c + 2], s[c + 3]);
            mx2 = fmax3(mx2, s[c + 4], s[c + 5]);
            mx3 = fmax3(mx3, s[c + 6], s[c + 7]);
          }
          const float cmax = fmax3(fmaxf(mx0, mx1), mx2, mx3) * scale_log2;
          if (tr && ch == 0) TRACE(g, 3);
          float alpha = 1.f;
          bool rescale = false;
          if (!any) {
            m = (cmax == -INFINITY) ? 0.f : cmax;
            any = true;
          } else if (cmax > m + kRescaleThreshold) {
            alpha = ex2_mufu(m - cmax);
            m = cmax;
            l *= alpha;
            rescale = true;
          }
          if (__any_sync(0xffffffffu, rescale)) {
            if (!first) {  // O_wg holds PV of this WG's earlier tiles, all retired
#pragma unroll
              for (int c = 0; c < HD / 32; ++c) {
                uint32_t r[32];
                tmem_ld32(o_col + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                tmem_st32(o_col + c * 32, r);
              }
            }
            if (ch == 1) {  // chunk 0's P was packed against the old m
              uint32_t r[32];
              tmem_ld32(s_col, r);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&r[i]));
                r[i] = pack_bf16(f.x * alpha, f.y * alpha);
              }
              tmem_st32(s_col, r);
            }
            tmem_wait_st();
          }
          // p = 2^(s*scale - m): packed FFMA2, MUFU for 8-kPolyCols of every 8 columns
          // and the FMA-pipe polynomial for the rest; packed FADD2 sums
          const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
          const uint64_t nm2 = f2_pack(-m, -m);
          uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
          for (int c = 0; c < kKeys / 2; c += 8) {
            float x[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) f2_unpack(ffma2(f2_pack(s[c + e], s[c + e + 1]), sc2, nm2), x[e], x[e + 1]);
#pragma unroll
            for (int e = 0; e < 8 - kPolyCols; ++e) s[c + e] = ex2_mufu(x[e]);
#pragma unroll
            for (int e = 8 - kPolyCols; e < 8; e += 2) f2_unpack(ex2_poly2(x[e], x[e + 1]), s[c + e], s[c + e + 1]);
            acc0 = fadd2(acc0, f2_pack(s[c + 0], s[c + 1]));
            acc1 = fadd2(acc1, f2_pack(s[c + 2], s[c + 3]));
            acc0 = fadd2(acc0, f2_pack(s[c + 4], s[c + 5]));
            acc1 = fadd2(acc1, f2_pack(s[c + 6], s[c + 7]));
          }
          float a0, a1, b0, b1;
          f2_unpack(acc0, a0, a1);
          f2_unpack(acc1, b0, b1);
          l += (a0 + a1) + (b0 + b1);
          uint32_t pk[kKeys / 4];
#pragma unroll
          for (int c = 0; c < kKeys / 4; ++c) pk[c] = pack_bf16(s[2 * c], s[2 * c + 1]);
          tmem_st32(s_col + ch * (kKeys / 4), pk);
        }
        tmem_wait_st();
        first = false;
        if (tr) TRACE(g, 5);
        tc_fence_before();
        if (tr) TRACE(g, 7);
        mbar_arrive(&bar[kPFull0 + wg]);
      }
      // (m, l) of this WG's share of the item -> epilogue (slot free once the epilogue
      // of item ii-2 read it); a WG without tiles in the item publishes l = 0
      const int sl = ii & 1;
      mbar_wait(&bar[kLFree0 + sl], ((ii >> 1) & 1) ^ 1);
      sML[(sl * 2 + wg) * 128 + row] = make_float2(any ? m : -INFINITY, l);
      mbar_arrive(&bar[kLFull0 + sl]);
    }
  } else if (warp >= 8) {
    // (ptxas allocates every role within the 128-register launch bound; setmaxnreg
    // only rebalances the physical pool: softmax 2 x 176, producers 40, epilogue 120)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 120;\n" ::: "memory");
    // ------------------------------------------------------------ epilogue WG
    // O (TMEM) / l -> bf16 output rows, off the softmax critical path.  With a RoPE
    // table it also rotates each landed Q tile in place (rotate-half pairs (i, i+HD/2)),
    // one item ahead of the epilogue it trails.
    const int row = threadIdx.x - 256;  // == TMEM lane (warp % 4 quadrant)
    const int t_local = row / G;
    const int h_local = row % G;
    const uint32_t t_row = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    auto rotate_q = [&](const Item& it, int ii) {
      // Thread -> (row, chunk-pair): a warp covers 32/CP rows x CP pairs of 8-element
      // chunks (i, i+HD/2), so its table reads are contiguous 512 B runs per token and its
      // shared accesses hit distinct 16 B banks of each 128 B swizzled row.
      constexpr int CP = HD / 16;          // chunk pairs per row
      constexpr int RPP = 128 / CP;        // rows per pass
      const int c = row % CP;
      const int r0 = row / CP;
      const int qb = ii & 1;
      const uint32_t qbase = smem_u32(sQ) + qb * S::kQ;
      auto tab_ptr = [&](int p) {
        const int r = r0 + p * RPP;
        const int tok = min(it.qt * TQ + r / G, it.q_len - 1);  // rows past q_len are masked
        return reinterpret_cast<const float4*>(rope + static_cast<int64_t>(it.q_pos0 + tok) *
                                                          (HD / 2) + c * 8);
      };
      // table slices in flight a batch of passes at a time (B x 64 B per thread), the first
      // batch issued before the Q tile lands
      constexpr int B = 2;
      float4 tab[B][4];
      auto load_tab = [&](int p0) {
#pragma unroll
        for (int p = 0; p < B; ++p) {
          const float4* t = tab_ptr(p0 + p);
#pragma unroll
          for (int e = 0; e < 4; ++e) tab[p][e] = __ldg(t + e);
        }
      };
      load_tab(0);
      mbar_wait(&bar[kQFull0 + qb], (ii >> 1) & 1);
#pragma unroll
      for (int p0 = 0; p0 < CP; p0 += B) {
        if (p0 > 0) load_tab(p0);
#pragma unroll
        for (int pi = 0; pi < B; ++pi) {
          const int r = r0 + (p0 + pi) * RPP;
          const uint32_t base = qbase + (r >> 3) * 1024 + (r & 7) * 128;
          const int i0 = c * 8, j0 = i0 + HD / 2;
          const uint32_t a0 = base + (i0 / 64) * 16384 + ((((i0 % 64) / 8) ^ (r & 7)) << 4);
          const uint32_t a1 = base + (j0 / 64) * 16384 + ((((j0 % 64) / 8) ^ (r & 7)) << 4);
          uint32_t u0[4], u1[4];
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(u0[0]), "=r"(u0[1]), "=r"(u0[2]), "=r"(u0[3]) : "r"(a0));
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(u1[0]), "=r"(u1[1]), "=r"(u1[2]), "=r"(u1[3]) : "r"(a1));
#pragma unroll
          for (int e = 0; e < 4; ++e) {  // tab[pi][e] = (cos, sin) of elements 2e, 2e+1
            const float2 x0 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u0[e]));
            const float2 x1 = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u1[e]));
            const float4 cs = tab[pi][e];
            u0[e] = pack_bf16(x0.x * cs.x - x1.x * cs.y, x0.y * cs.z - x1.y * cs.w);
            u1[e] = pack_bf16(x1.x * cs.x + x0.x * cs.y, x1.y * cs.z + x0.y * cs.w);
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0), "r"(u0[0]),
                       "r"(u0[1]), "r"(u0[2]), "r"(u0[3]));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a1), "r"(u1[0]),
                       "r"(u1[1]), "r"(u1[2]), "r"(u1[3]));
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
      mbar_arrive(&bar[kQReady0 + qb]);
    };
    // merge the two parity accumulators: O = (w_A O_A + w_B O_B) / (w_A l_A + w_B l_B),
    // w_p = 2^(m_p - max(m_A, m_B)); a WG without tiles in the item (n == 1) is skipped
    auto epilogue = [&](const Item& it, int ii, int g0) {
      const int sl = ii & 1;
      const int tok = it.qt * TQ + t_local;
      const bool row_valid = tok < it.q_len;
      mbar_wait(&bar[kLFull0 + sl], (ii >> 1) & 1);
      const float2 ml0 = sML[(sl * 2 + 0) * 128 + row];
      const float2 ml1 = sML[(sl * 2 + 1) * 128 + row];
      mbar_arrive(&bar[kLFree0 + sl]);
      const bool has0 = it.n >= 2 || (g0 & 1) == 0;  // warp-uniform
      const bool has1 = it.n >= 2 || (g0 & 1) == 1;
      const float mm = fmaxf(has0 ? ml0.x : -INFINITY, has1 ? ml1.x : -INFINITY);
      float w0 = has0 ? exp2f(ml0.x - mm) : 0.f;
      float w1 = has1 ? exp2f(ml1.x - mm) : 0.f;
      const float l = w0 * ml0.y + w1 * ml1.y;
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      w0 *= inv_l;
      w1 *= inv_l;
      mbar_wait(&bar[kOFull0 + sl], (ii >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* orow =
          out + (static_cast<int64_t>(it.q_start + tok) * n_q_heads + it.kvh * G + h_local) * HD;
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        float o[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] = 0.f;
        if (has0) {
          uint32_t r[16];
          tmem_ld16(t_row + 256 + c * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __uint_as_float(r[i]) * w0;
        }
        if (has1) {
          uint32_t r[16];
          tmem_ld16(t_row + 384 + c * 16, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = fmaf(__uint_as_float(r[i]), w1, o[i]);
        }
        if (row_valid) {
#pragma unroll
          for (int i = 0; i < 16; i += 8) {
            uint4 v;
            v.x = pack_bf16(o[i + 0], o[i + 1]);
            v.y = pack_bf16(o[i + 2], o[i + 3]);
            v.z = pack_bf16(o[i + 4], o[i + 5]);
            v.w = pack_bf16(o[i + 6], o[i + 7]);
            *reinterpret_cast<uint4*>(orow + c * 16 + i) = v;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bar[kOFree0 + 0]);
      mbar_arrive(&bar[kOFree0 + 1]);
    };
    const int n_mine =
        n_work > (int)blockIdx.x ? (n_work - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto item_of = [&](int ii) { return load_item(work, blockIdx.x + ii * gridDim.x); };
    // O is single-buffered per WG, so item ii's epilogue must finish before item ii+1's
    // first PV and runs first; with a RoPE table, Q(ii+2) is rotated next (Q is double
    // buffered: it lands once QK of item ii retired; needed by QK of item ii+2).
    constexpr int kAhead = 2;
    if (rope != nullptr)
      for (int ii = 0; ii < kAhead && ii < n_mine; ++ii) rotate_q(item_of(ii), ii);
    int g0 = 0;
    for (int ii = 0; ii < n_mine; ++ii) {
      const Item it = item_of(ii);
      epilogue(it, ii, g0);
      g0 += it.n;
      if (rope != nullptr && ii + kAhead < n_mine) rotate_q(item_of(ii + kAhead), ii + kAhead);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int HD, int G, int BT>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tkv, void* out, int n_q_heads,
                     int layer, const int* req_meta, const int* blk_ids, const int* blk_valid,
                     const int* blk_pos, const int* work, int n_work, float scale_log2,
                     const float2* rope, cudaStream_t stream) {
  auto kern = prefix_prefill_kernel<HD, G, BT>;
  const uint32_t smem = Smem<HD, BT>::kTotal;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int grid = n_work < sms ? n_work : sms;
  kern<<<grid, kThreads, smem, stream>>>(tq, tkv, static_cast<__nv_bfloat16*>(out), n_q_heads,
                                        layer, req_meta, blk_ids, blk_valid, blk_pos, work, n_work,
                                        scale_log2, rope);
  return cudaGetLastError();
}

template <int HD, int G>
cudaError_t launch_bt(int bt, const CUtensorMap& tq, const CUtensorMap& tkv, void* out,
                      int n_q_heads, int layer, const int* rm, const int* bi, const int* bv,
                      const int* bp, const int* work, int n_work, float sl2, const float2* rope,
                      cudaStream_t st) {
  switch (bt) {
    case 16: return launch_t<HD, G, 16>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    case 32: return launch_t<HD, G, 32>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    case 64: return launch_t<HD, G, 64>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    case 128: return launch_t<HD, G, 128>(tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int HD>
cudaError_t launch_g(int g, int bt, const CUtensorMap& tq, const CUtensorMap& tkv, void* out,
                     int n_q_heads, int layer, const int* rm, const int* bi, const int* bv,
                     const int* bp, const int* work, int n_work, float sl2, const float2* rope,
                     cudaStream_t st) {
  switch (g) {
    case 1: return launch_bt<HD, 1>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    case 2: return launch_bt<HD, 2>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    case 4: return launch_bt<HD, 4>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    case 8: return launch_bt<HD, 8>(bt, tq, tkv, out, n_q_heads, layer, rm, bi, bv, bp, work, n_work, sl2, rope, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace attn

int prefix_prefill(const void* q, int64_t q_row_stride, void* o, int total_q_tokens,
                   int n_q_heads, const void* kv_pool, int64_t num_pool_blocks, int block_tokens,
                   int n_layers, int n_kv_heads, int head_dim, int layer, const int* req_meta,
                   const int* blk_ids, const int* blk_valid, const int* blk_pos, const int* work,
                   int n_work, float softmax_scale, const void* rope_table, cudaStream_t stream) {
  if (n_work == 0) return RCB_OK;
  if (head_dim != 64 && head_dim != 128) return set_error(RCB_ERR_ARG, "head_dim must be 64 or 128");
  if (n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0) return set_error(RCB_ERR_ARG, "bad head counts");
  const int g = n_q_heads / n_kv_heads;
  if (layer < 0 || layer >= n_layers) return set_error(RCB_ERR_ARG, "layer out of range");
  CUtensorMap tq, tkv;
  {
    const uint64_t dims[3] = {(uint64_t)head_dim, (uint64_t)n_q_heads, (uint64_t)total_q_tokens};
    if (q_row_stride < (int64_t)n_q_heads * head_dim || q_row_stride % 8 != 0)
      return set_error(RCB_ERR_ARG, "q_row_stride must be >= n_q_heads*head_dim and a multiple of 8");
    const uint64_t strides[2] = {(uint64_t)head_dim * 2, (uint64_t)q_row_stride * 2};
    const uint32_t box[3] = {64, (uint32_t)g, (uint32_t)(128 / g)};
    int rc = encode_tma_bf16(&tq, q, 3, dims, strides, box);
    if (rc != RCB_OK) return rc;
  }
  {
    const uint64_t blk_bytes =
        (uint64_t)n_layers * 2 * n_kv_heads * block_tokens * head_dim * 2;
    const uint64_t dims[5] = {(uint64_t)head_dim, (uint64_t)block_tokens, (uint64_t)n_kv_heads,
                              (uint64_t)(2 * n_layers), (uint64_t)num_pool_blocks};
    const uint64_t strides[4] = {(uint64_t)head_dim * 2, (uint64_t)block_tokens * head_dim * 2,
                                 (uint64_t)n_kv_heads * block_tokens * head_dim * 2, blk_bytes};
    const uint32_t box[5] = {64, (uint32_t)block_tokens, 1, 1, 1};
    int rc = encode_tma_bf16(&tkv, kv_pool, 5, dims, strides, box);
    if (rc != RCB_OK) return rc;
  }
  const float sl2 = softmax_scale * 1.4426950408889634f;
  cudaError_t e =
      head_dim == 128
          ? attn::launch_g<128>(g, block_tokens, tq, tkv, o, n_q_heads, layer, req_meta, blk_ids,
                                blk_valid, blk_pos, work, n_work, sl2,
                                static_cast<const float2*>(rope_table), stream)
          : attn::launch_g<64>(g, block_tokens, tq, tkv, o, n_q_heads, layer, req_meta, blk_ids,
                               blk_valid, blk_pos, work, n_work, sl2,
                               static_cast<const float2*>(rope_table), stream);
  if (e != cudaSuccess) return set_cuda_error(e, "prefix_prefill launch");
  return RCB_OK;
}

}  // namespace rcb

#ifdef RCB_TRACE
extern "C" int rcb_debug_attn_trace(void* host, int64_t bytes) {
  return cudaMemcpyFromSymbol(host, rcb::attn::g_trace, bytes) == cudaSuccess ? 0 : 3;
}
#endif
