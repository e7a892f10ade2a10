// prefix_attn.cu — prefix-aware prefill attention over the paged doc-KV pool.
//
// Replaces the reference's latency stand-in T(alpha, beta)
// (ragsim cost_model.py:106-117 `interpolate`, called at simulator.py:506 and
// tree.py:240): here the alpha cached tokens are READ from knowledge-tree node
// blocks through a block table, and only the beta suffix tokens (miss docs +
// prompt) are computed as queries.
//
// Persistent CTAs (one per SM) walk a heaviest-first list of work items
// (request, query-tile PAIR, kv head), pipelining across items:
//   * a query tile = 128 rows = (128/G tokens) x (G query heads sharing the kv head);
//     a work item holds two adjacent tiles Q0 | Q1 that share every K/V tile it loads
//   * K/V tiles of 128 key slots = 128/BT pool blocks, TMA-loaded (SW128) into one
//     ring in consumption order K(0) V(0) K(1) V(1) ...
//   * S_w = Q_w K^T (SS) and O_w += P_w V (TS: P kept in TMEM over S_w's columns) on
//     tcgen05, fp32 accumulators in TMEM: S0 | S1 | O0 | O1 = 512 columns
//   * softmax warpgroup w owns query tile Q_w: online softmax one row per thread,
//     lazily rescaled O_w (only when its running max grows by > 2^8)
//   * issue order per KV step s: PV0(s-1) QK0(s) PV1(s-1) QK1(s), so each softmax
//     warpgroup overlaps the other tile's two MMAs (FA4-style ping-pong)
//   * the epilogue warpgroup drains O0 of an item while Q1's last MMAs still run;
//     Q0 may stop one KV tile before Q1 (causal), an item's Q1 may be empty
// Warp roles: 0-3 softmax WG 0, 4 TMA producer (Q, mask metadata, K/V ring), 5 MMA
// issuer + TMEM owner, 6-7 idle, 8-11 epilogue (+ in-smem Q RoPE), 12-15 softmax WG 1.
//
// Key slots carry holes (node tails: a block holds `valid` <= BT tokens), so
// each block also carries its logical start position; a slot is attended iff
// off < valid && pos <= query_pos (causal on logical positions).
#include <climits>

#include "sm100.cuh"
#include "rcb_internal.h"

namespace rcb {

namespace attn {

constexpr int kThreads = 512;
constexpr int kRows = 128;
constexpr int kKeys = 128;  // key slots per KV tile
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// exp2 on the FMA/ALU pipes (magic-add rounding + cubic) for kPoly16 of every 16 score
// columns, MUFU for the rest.  Measured on B200 (2 of 16 / 4 / 6 / 8): 2 and 4 are within
// 1% (2 is 1-2% faster on full misses), 6 loses 4%, 8 loses more (the FMA pipe saturates);
// none at all is 4% slower.  An earlier variant that rounded with floorf (FRND, not on the
// FMA pipe) gained nothing.
#ifndef RCB_POLY16
#define RCB_POLY16 2
#endif
constexpr int kPoly16 = RCB_POLY16;  // of every 16 columns (even)
#ifndef RCB_PDL
#define RCB_PDL 1
#endif

// TMEM load of one O chunk, 32 or 16 columns (the epilogue's chunk width depends on G)
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[32]) { tmem_ld32(taddr, r); }
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, uint32_t (&r)[16]) { tmem_ld16(taddr, r); }

// Per-step handoff timestamps of CTA 0 (debug builds with -DRCB_TRACE only; tools/attn_trace.py)
//   softmax WG w, its tile c: [c][4w + 0] S wait start, [4w + 1] S seen, [4w + 2] P arrive
//   MMA, step s: [s][8] P0 seen, [9] QK0 issued, [10] P1 seen, [11] QK1 issued,
//   [12] K(s) seen full, [13] PV0 issued, [14] PV1 issued, [15] Q seen (first step of an item)
//   producer, step s: [s][16] block ids loaded, [17] K(s) issued, [18] V(s) issued
//   epilogue, item ii: [ii][19] O0 full seen, [20] O0 freed, [21] O1 full seen, [22] O1 freed,
//   [23] item's O written (stores issued)
//   softmax WG w, its tile c, chunk ch: [c][24 + 4w + 2ch] S chunk in registers,
//   [25 + 4w + 2ch] exp loop done (before the bf16 pack + TMEM store)
#ifdef RCB_TRACE
constexpr int kTraceTiles = 1024;
constexpr int kTraceEv = 32;
__device__ long long g_trace[kTraceTiles * kTraceEv];
#define TRACE(g, ev)                                                                      \
  do {                                                                                    \
    if (blockIdx.x == 0 && (g) < kTraceTiles) g_trace[(g) * kTraceEv + (ev)] = clock64(); \
  } while (0)
#else
#define TRACE(g, ev) \
  do {               \
  } while (0)
#endif

// barrier indices (pairs indexed by item parity or by query tile w)
// P handoff per 64-key half: kPFull0 = P columns of keys [0, 64), kPFullB0 = keys [64, 128)
// (arrived for every tile, right after kPFull0 on a half tile); kPVDone0 = PV of the first
// half retired (waited only by a softmax that must rescale O between its two halves)
enum Bar {
  kQFull0 = 0, kQEmpty0 = 2, kQReady0 = 4, kSFull0 = 6, kPFull0 = 8, kOFull0 = 10,
  kOFree0 = 12, kLFull0 = 14, kLFree0 = 16, kMetaFull0 = 18, kMetaFree0 = 22,
  kPFullB0 = 26, kPVDone0 = 28,
  kKVFull0 = 30  // [kStages] full, then [kStages] empty
};

// SPLIT: every item of the launch is a split item (one query tile: decode steps and
// short prompts over cached documents, HBM-bound).  Q then needs one tile per item
// buffer, and the freed 64 KB (HD = 128) deepens the K/V ring from 3 to 5 stages:
// a V stage stays held from its load until the PV after its tile's softmax, so the
// ring depth is what bounds the bytes in flight per SM on these launches.
template <int HD, int BT, bool SPLIT>
struct Smem {
  static constexpr uint32_t kHalves = HD / 64;
  static constexpr uint32_t kQ = kHalves * 16384;   // one query tile
  static constexpr uint32_t kKV = kHalves * 16384;  // one K or V tile
  static constexpr uint32_t kQT = SPLIT ? 1 : 2;    // query tiles per item buffer
  static constexpr int kStages = HD == 128 ? (SPLIT ? 5 : 3) : (SPLIT ? 8 : 6);  // K/V ring
  static constexpr int kBPT = kKeys / BT;
  static constexpr int kMetaSlots = 4;
  static constexpr uint32_t offQ = 0;                       // [2 items][kQT tiles]
  static constexpr uint32_t offKV = offQ + 2 * kQT * kQ;    // [kStages]
  static constexpr uint32_t offMeta = offKV + kStages * kKV;  // int [kMetaSlots][2][kBPT]
  static constexpr uint32_t offL = offMeta + kMetaSlots * 2 * kBPT * 4;  // float2 [2][128]
  static constexpr uint32_t offBar = offL + 2 * 128 * 8;
  static constexpr int kNumBars = kKVFull0 + 2 * kStages;
  // the dynamic window starts 1024-aligned (checked at kernel entry): no slack
  static constexpr uint32_t kTotal = offBar + kNumBars * 8 + 16;
};

// Work items are self-contained (no dependent loads at item start):
//   {q_start, q_len, q_pos0, blk_begin, blk_count, q_pair, kv_head,
//    n0 | half0 << 15 | n1 << 16 | half1 << 31}
// n_w = KV tiles query tile w needs; the item runs max(n0, n1) KV steps.  half_w: the last
// of them needs only its first 64 key slots -> QK with N = 64, PV with K = 64, and the
// softmax does one 64-column chunk.
//   pair item  (n1 > 0): softmax WG w owns query tile Q_w over steps j < n_w
//   split item (n1 == 0, a lone query tile): WG w owns the steps j with j % 2 == w of Q0,
//              each WG keeps its own (m, l, O_w) and the epilogue merges the two
#ifndef RCB_OTMA
#define RCB_OTMA 1
#endif
// O of a full query tile leaves through a TMA store staged in the finished item's Q
// buffer (its last QK retired before the last PV, i.e. before O_w was complete); the
// epilogue's arrival on Q_empty then releases the buffer for Q(ii + 2).  Ragged tiles and
// split-KV parts keep the per-lane stores, and so do G <= 2 launches (kStageO below).
constexpr bool kOTma = RCB_OTMA != 0;
constexpr int kItemInts = 8;
struct Item {
  int q_start, q_len, q_pos0, blk_begin, blk_count, qp, kvh, n0, n1;
  bool h0, h1;
  int ps;  // split-KV part slot (-1: the item writes bf16 O directly)
  __device__ __forceinline__ bool split() const { return n1 == 0; }
  __device__ __forceinline__ int n() const { return n0 > n1 ? n0 : n1; }
  // WG w works on step j
  __device__ __forceinline__ bool on(int w, int j) const {
    return split() ? (j & 1) == w : j < (w ? n1 : n0);
  }
  // WG w has any step (writes O_w, publishes (m, l))
  __device__ __forceinline__ bool has(int w) const {
    return split() ? n0 > w : (w ? n1 : n0) > 0;
  }
  // WG w's first / last step
  __device__ __forceinline__ int first(int w) const { return split() ? w : 0; }
  __device__ __forceinline__ int last(int w) const {
    return split() ? ((n0 - 1 - w) & ~1) + w : (w ? n1 : n0) - 1;
  }
  // query tile WG w reads
  __device__ __forceinline__ int qtile(int w) const { return split() ? 0 : w; }
  // step j of WG w covers only the first 64 key slots
  __device__ __forceinline__ bool half(int w, int j) const {
    return split() ? (h0 && j == n0 - 1) : (w ? (h1 && j == n1 - 1) : (h0 && j == n0 - 1));
  }
};

__device__ __forceinline__ Item load_item(const int* __restrict__ work, int idx) {
  const int4 a = *reinterpret_cast<const int4*>(work + idx * kItemInts);
  const int4 b = *reinterpret_cast<const int4*>(work + idx * kItemInts + 4);
  const uint32_t p = static_cast<uint32_t>(b.w);
  // field 6 = kv_head | (split-KV part slot + 1) << 8
  return Item{a.x, a.y, a.z, a.w, b.x, b.y, b.z & 0xff, static_cast<int>(p & 0x7fffu),
              static_cast<int>((p >> 16) & 0x7fffu), ((p >> 15) & 1u) != 0, (p >> 31) != 0,
              (b.z >> 8) - 1};
}

// Persistent: CTA c serves work items c, c + grid, ... (heaviest first).  The KV step
// counter s runs across items, so the K/V ring, mask-metadata ring and S/P handshakes
// keep their phase; Q (smem) is double buffered per item, O_w single buffered (the
// epilogue frees O_w before the next item's first PV into it).
template <int HD, int G, int BT, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    prefix_prefill_kernel(const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_kv,
                          const __grid_constant__ CUtensorMap tm_o,
                          __nv_bfloat16* __restrict__ out, int n_q_heads, int layer,
                          const int* __restrict__ blk_ids, const int* __restrict__ blk_valid,
                          const int* __restrict__ blk_pos, const int* __restrict__ work,
                          int n_work, float scale_log2, const float2* __restrict__ rope,
                          float* __restrict__ part_o, float2* __restrict__ part_ml) {
  using S = Smem<HD, BT, SPLIT>;
  constexpr int TQ = kRows / G;  // tokens per query tile
  // O through the Q buffer + TMA store for G > 2 only.  Q(ii + 2) then lands only after item
  // ii's O left the buffer, and with fused RoPE it must still be rotated before item ii + 2
  // starts: MHA items are short (2-5 KV steps at 128 tokens per tile), so that chain stalls
  // the MMA warp (LLaMA2 miss batch with fused RoPE 117.8 -> 107.5 and 121.9 -> 109.6 us with
  // direct stores, two A/B runs), while GQA-4 gains from the staging (Mistral mixed step
  // 480.8 -> 501.7 us without it)
  constexpr bool kStageO = kOTma && G > 2;
  // O columns the epilogue drains per TMEM load.  16 for G <= 2: the smaller register
  // footprint of the drain (MHA: no staging, rotation every item) measured LLaMA2 miss
  // batch with RoPE 103.5 -> 99.3 us; GQA-4 keeps 32 (hit batch 72.7 vs 74.7 us with 16)
  constexpr int kOCols = G <= 2 ? 16 : 32;
  constexpr int BPT = S::kBPT;
  constexpr int NS = S::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SW128 tiles need 1024-byte alignment; the budget has no room for slack
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem + S::offQ;
  uint8_t* sKV = smem + S::offKV;
  int* sMeta = reinterpret_cast<int*>(smem + S::offMeta);  // [slot][0=valid,1=pos][BPT]
  float2* sML = reinterpret_cast<float2*>(smem + S::offL);  // [w][row] (max, row sum)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::offBar);
  uint64_t* kv_full = bar + kKVFull0;
  uint64_t* kv_empty = bar + kKVFull0 + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + S::kNumBars);

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar[kQFull0 + b], 1);
      mbar_init(&bar[kQEmpty0 + b], kStageO ? 2 : 1);  // MMA (last QK) + epilogue (O store)
      mbar_init(&bar[kQReady0 + b], kRows);
      mbar_init(&bar[kSFull0 + b], 1);
      mbar_init(&bar[kPFull0 + b], kRows);
      mbar_init(&bar[kPFullB0 + b], kRows);
      mbar_init(&bar[kPVDone0 + b], 1);
      mbar_init(&bar[kOFull0 + b], 1);
      mbar_init(&bar[kOFree0 + b], kRows);
      mbar_init(&bar[kLFull0 + b], kRows);
      mbar_init(&bar[kLFree0 + b], kRows);
    }
    for (int b = 0; b < S::kMetaSlots; ++b) {
      mbar_init(&bar[kMetaFull0 + b], 1);
      mbar_init(&bar[kMetaFree0 + b], 2 * kRows);  // both softmax WGs, every step
    }
    for (int b = 0; b < NS; ++b) {
      mbar_init(&kv_full[b], 1);
      mbar_init(&kv_empty[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // register budget per role (ptxas compiles each region to its setmaxnreg limit):
  // softmax 2 x 128 x RCB_REG_SM, producers / MMA 128 x RCB_REG_PR, epilogue 128 x RCB_REG_EP
#ifndef RCB_REG_SM
#define RCB_REG_SM 160
#define RCB_REG_PR 80
#define RCB_REG_EP 112
#endif
  static_assert(2 * RCB_REG_SM + RCB_REG_PR + RCB_REG_EP <= 512, "register file");
  if (warp >= 4 && warp < 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RCB_REG_PR));
  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_kv);
      int s = 0;         // KV step (ring loads u = 2s: K, 2s + 1: V)
      int q_issued = 0;  // items whose Q tiles have been issued
      auto issue_q = [&](int idx, int ii) {
        const Item it = load_item(work, idx);
        const int qb = ii & 1;
        if (SPLIT && !it.split()) __trap();  // the host promised split items only
        mbar_arrive_expect_tx(&bar[kQFull0 + qb], S::kQT * S::kQ);
        for (int w = 0; w < (int)S::kQT; ++w)
          for (int h = 0; h < (int)S::kHalves; ++h)
            // an empty Q1 (never read) reloads Q0's rows: no box lies wholly out of bounds
            tma_load_3d(sQ + (qb * S::kQT + w) * S::kQ + h * 16384, &tm_q, &bar[kQFull0 + qb],
                        h * 64, it.kvh * G, it.q_start + (2 * it.qp + (it.n1 > 0 ? w : 0)) * TQ);
      };
      auto load_kv = [&](int u, int kv, const int (&ids)[BPT], int kvh) {
        const int st = u % NS;
        mbar_wait(&kv_empty[st], ((u / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], S::kKV);
#pragma unroll
        for (int b = 0; b < BPT; ++b)
          for (int h = 0; h < (int)S::kHalves; ++h)
            tma_load_5d(sKV + st * S::kKV + h * 16384 + b * BT * 128, &tm_kv, &kv_full[st],
                        h * 64, 0, kvh, 2 * layer + kv, ids[b]);
      };
      for (int idx = blockIdx.x, ii = 0; idx < n_work; idx += gridDim.x, ++ii) {
        const Item it = load_item(work, idx);
        if (q_issued == ii) {
          mbar_wait(&bar[kQEmpty0 + (ii & 1)], ((ii >> 1) & 1) ^ 1);
          issue_q(idx, ii);
          ++q_issued;
        }
        const int n = it.n();
#if RCB_PDL
        // launched programmatically after the K/V write: Q, tables and the prologue may run
        // early, the first K/V page load waits for that grid's writes
        if (ii == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
        for (int j = 0; j < n; ++j, ++s) {
          // next item's Q as soon as its buffer frees (last QK of item ii-1 retired): it
          // then lands (and is rotated) a whole item ahead of its first MMA
          if (q_issued == ii + 1 && idx + (int)gridDim.x < n_work &&
              mbar_test(&bar[kQEmpty0 + ((ii + 1) & 1)], (((ii + 1) >> 1) & 1) ^ 1)) {
            issue_q(idx + gridDim.x, ii + 1);
            ++q_issued;
          }
          int ids[BPT];
          int vv[BPT], pp[BPT];
#pragma unroll
          for (int b = 0; b < BPT; ++b) {
            const int sb = j * BPT + b;
            const bool in = sb < it.blk_count;
            // slots past the table load a real (finite) block; they are masked
            ids[b] = blk_ids[it.blk_begin + (in ? sb : 0)];
            vv[b] = in ? blk_valid[it.blk_begin + sb] : 0;
            pp[b] = in ? blk_pos[it.blk_begin + sb] : 0;
          }
#ifdef RCB_TRACE
          if (ids[0] + vv[0] + pp[0] == INT_MIN) __trap();  // force the loads before the stamp
#endif
          TRACE(s, 16);
          load_kv(2 * s, 0, ids, it.kvh);
          TRACE(s, 17);
          // per-step mask metadata: its own ring (the softmax may lag the K/V ring)
          const int ms = s & (S::kMetaSlots - 1);
          mbar_wait(&bar[kMetaFree0 + ms], ((s / S::kMetaSlots) & 1) ^ 1);
#pragma unroll
          for (int b = 0; b < BPT; ++b) {
            sMeta[(ms * 2 + 0) * BPT + b] = vv[b];
            sMeta[(ms * 2 + 1) * BPT + b] = pp[b];
          }
          mbar_arrive(&bar[kMetaFull0 + ms]);  // release: publishes sMeta[ms]
          load_kv(2 * s + 1, 1, ids, it.kvh);
          TRACE(s, 18);
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(128, kKeys, 0, 0);
      constexpr uint32_t idesc_qk_half = idesc_bf16_f32(128, kKeys / 2, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, HD, 0, 1);
      const uint32_t q_base = smem_u32(sQ);
      const uint32_t kv_base = smem_u32(sKV);
      int s = 0;           // KV step
      int c[2] = {0, 0};   // QK_w issued so far (S_w / P_w phases)
      int oc[2] = {0, 0};  // items with a non-empty Q_w so far (O_w phases)
      // the previous step's pending PVs
      bool p_has[2] = {false, false}, p_last[2] = {false, false}, p_first[2] = {false, false};
      bool p_half[2] = {false, false};
      int p_c[2] = {0, 0}, p_vu = 0;
      bool p_any = false, p_v_ready = false;
      auto issue_pv = [&](int w) {
        // first PV into O_w of an item: the epilogue has drained O_w of the previous one
        if (p_first[w]) mbar_wait(&bar[kOFree0 + w], (oc[w] & 1) ^ 1);
        if (!p_v_ready) {
          mbar_wait(&kv_full[p_vu % NS], (p_vu / NS) & 1);
          p_v_ready = true;
        }
        // keys [0, 64): their P is packed while the softmax still works on keys [64, 128)
        mbar_wait(&bar[kPFull0 + w], p_c[w] & 1);
        TRACE(s - 1, 8 + 2 * w);
        tc_fence_after();
        const int st = p_vu % NS;
        // A = P_w (bf16 pairs over S_w's first 64 columns); V tile is [half][128 keys][64]:
        // MN-major, halves 16 KB apart (LBO)
#pragma unroll
        for (int kk = 0; kk < kKeys / 32; ++kk) {
          const uint64_t b = sw128_desc(kv_base + st * S::kKV + kk * 2048, 16384, 1024);
          umma_bf16_ts(tmem + 256 + w * 128, tmem + w * kKeys + kk * 8, b, idesc_pv,
                       (!p_first[w] || kk > 0) ? 1u : 0u);
        }
        umma_commit(&bar[kPVDone0 + w]);
        if (!p_half[w]) {  // keys [64, 128)
          mbar_wait(&bar[kPFullB0 + w], p_c[w] & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = kKeys / 32; kk < kKeys / 16; ++kk) {
            const uint64_t b = sw128_desc(kv_base + st * S::kKV + kk * 2048, 16384, 1024);
            umma_bf16_ts(tmem + 256 + w * 128, tmem + w * kKeys + kk * 8, b, idesc_pv, 1u);
          }
        }
        if (p_last[w]) {
          umma_commit(&bar[kOFull0 + w]);
          ++oc[w];
        }
        TRACE(s - 1, 13 + w);
      };
      auto issue_qk = [&](int w, int qt, int ku, bool half) {  // qt: Q buffer [parity][tile]
        const int st = ku % NS;
        const uint32_t d = tmem + w * kKeys;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint64_t a = sw128_desc(q_base + qt * S::kQ + off, 16, 1024);
          const uint64_t b = sw128_desc(kv_base + st * S::kKV + off, 16, 1024);
          umma_bf16_ss(d, a, b, half ? idesc_qk_half : idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&bar[kSFull0 + w]);
        ++c[w];
      };
      for (int idx = blockIdx.x, ii = 0; idx < n_work; idx += gridDim.x, ++ii) {
        const Item it = load_item(work, idx);
        const int n = it.n();
        const int qb = ii & 1;
        for (int j = 0; j < n; ++j, ++s) {
          const bool h0 = it.on(0, j), h1 = it.on(1, j);
          const int ku = 2 * s;
          bool k_ready = false;
          auto need_k = [&]() {
            if (k_ready) return;
            if (j == 0) {  // Q landed (and, with fused RoPE, rotated by the epilogue WG)
              mbar_wait(&bar[(rope != nullptr ? kQReady0 : kQFull0) + qb], (ii >> 1) & 1);
              TRACE(s, 15);
            }
            mbar_wait(&kv_full[ku % NS], (ku / NS) & 1);
            TRACE(s, 12);
            tc_fence_after();
            k_ready = true;
          };
          // S_w is overwritten by QK_w(s) only after PV_w(s-1) (its P reader) was issued;
          // tcgen05.mma executes in issue order.  Pair items: PV0 QK0 PV1 QK1 (each
          // softmax overlaps the other tile's MMAs).  Split items alternate WGs over the
          // steps, so on a WG1 step QK1 goes FIRST and the pending PV0 (which waits for
          // WG0's softmax) after it: the two WGs' softmaxes then overlap instead of
          // forming one chain through the MMA warp.
          int pc0 = c[0], pc1 = c[1];
          auto qk0 = [&]() {
            pc0 = c[0];
            if (h0) {
              need_k();
              issue_qk(0, qb * S::kQT, ku, it.half(0, j));
              TRACE(s, 9);
            }
          };
          auto qk1 = [&]() {
            pc1 = c[1];
            if (h1) {
              need_k();
              issue_qk(1, qb * S::kQT + (SPLIT ? 0 : it.qtile(1)), ku, it.half(1, j));
              TRACE(s, 11);
            }
          };
          if (SPLIT && (j & 1)) {  // WG1 step (split-only launch; mixed launches keep one order)
            if (p_has[1]) issue_pv(1);
            qk1();
            if (p_has[0]) issue_pv(0);
            if (p_any) umma_commit(&kv_empty[p_vu % NS]);  // V(s-1) no longer read
            qk0();
          } else {
            if (p_has[0]) issue_pv(0);
            qk0();
            if (p_has[1]) issue_pv(1);
            if (p_any) umma_commit(&kv_empty[p_vu % NS]);  // V(s-1) no longer read
            qk1();
          }
          umma_commit(&kv_empty[ku % NS]);  // K(s) no longer read
          if (j == n - 1) umma_commit(&bar[kQEmpty0 + qb]);  // Q tiles no longer read
          // this step's PVs become pending: they need V(s) and the softmax of S_w(s)
          p_any = true;
          p_v_ready = false;
          p_vu = ku + 1;
          p_has[0] = h0;
          p_has[1] = h1;
          p_c[0] = pc0;
          p_c[1] = pc1;
          p_first[0] = (j == it.first(0));
          p_first[1] = (j == it.first(1));
          p_last[0] = (j == it.last(0));
          p_last[1] = (j == it.last(1));
          p_half[0] = it.half(0, j);
          p_half[1] = it.half(1, j);
        }
      }
      if (p_any) {
        if (p_has[0]) issue_pv(0);
        if (p_has[1]) issue_pv(1);
        umma_commit(&kv_empty[p_vu % NS]);
      }
    }
  } else if (warp < 4 || warp >= 12) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RCB_REG_SM));
    // ------------------------------------------------------------ softmax of query tile w
    const int wg = warp >= 12 ? 1 : 0;
    const int quad = warp & 3;
    const int row = quad * 32 + (threadIdx.x & 31);  // == TMEM lane
    const int t_local = row / G;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t s_col = t_row + wg * kKeys;        // S_w / P_w
    const uint32_t o_col = t_row + 256 + wg * 128;    // O_w
    float s[kKeys / 2];
    int c = 0;   // tiles processed (S_w / P_w phase)
    int oc = 0;  // items with a non-empty Q_w (L slot phase)
    int st = 0;  // KV step (meta ring)
    // Every first-half PV commits kPVDone; a tile that rescaled in chunk 1 consumed that
    // phase already, the others consume it after the next S-full (free: that PV precedes
    // the next QK_w in MMA order) or at exit, so every arrival is waited (synccheck)
    bool pv_pending = false;
    for (int idx = blockIdx.x; idx < n_work; idx += gridDim.x) {
      const Item it = load_item(work, idx);
      const int n = it.n();
      const int tok = (2 * it.qp + it.qtile(wg)) * TQ + t_local;
      const int qp = it.q_pos0 + tok;
      float m = -INFINITY;  // running max (scaled, log2 domain); may be stale by < 2^8
      float l = 0.f;
      bool any = false;    // m initialised (first chunk of the item)
      for (int j = 0; j < n; ++j, ++st) {
        const int ms = st & (S::kMetaSlots - 1);
        mbar_wait(&bar[kMetaFull0 + ms], (st / S::kMetaSlots) & 1);
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
        if (!it.on(wg, j)) continue;
        // S-full also means this WG's previous PV retired (issued before QK_w(j)): O_w is
        // current
        const bool tr = (threadIdx.x & 127) == 0 && quad == 0;
        if (tr) TRACE(c, 4 * wg + 0);
        mbar_wait(&bar[kSFull0 + wg], c & 1);
        if (pv_pending) mbar_wait(&bar[kPVDone0 + wg], (c - 1) & 1);
        pv_pending = true;
        if (tr) TRACE(c, 4 * wg + 1);
        tc_fence_after();
        const bool masked = !all_valid || max_pos > qp;
        const bool half = it.half(wg, j);  // only S columns [0, 64) were computed
#ifdef RCB_DBG_NOSOFTMAX
        // timing experiment only (wrong results): hand P over without computing it, so the
        // step time is the MMA + handoff pipeline alone
        tc_fence_before();
        mbar_arrive(&bar[kPFull0 + wg]);
        mbar_arrive(&bar[kPFullB0 + wg]);
        any = true;
        if (tr) TRACE(c, 4 * wg + 2);
        ++c;
        continue;
#endif
        // Two 64-column chunks against the running max m (within 2^8 of the true row max: a
        // chunk that exceeds m + 2^8 rescales O and l).  P of chunk c (bf16 pairs) goes to S
        // columns [32c, 32c + 32) and is handed to the MMA warp per chunk, so the PV of keys
        // [0, 64) runs on the tensor core while chunk 1 is still being computed.
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          if (ch == 1 && half) break;
          {
            uint32_t r[kKeys / 2];
            tmem_ld64(s_col + ch * (kKeys / 2), r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < kKeys / 2; ++i) s[i] = __uint_as_float(r[i]);
          }
          if (tr) TRACE(c, 24 + 4 * wg + 2 * ch);
          if (masked) {
            // keys valid in block b for this row: off < min(valid_b, qp - pos_b + 1)
#pragma unroll
            for (int cc0 = 0; cc0 < kKeys / 2; ++cc0) {
              const int cc = ch * (kKeys / 2) + cc0;
              const int b = cc / BT;
              s[cc0] = (cc % BT) < min(vv[b], qp - pp[b] + 1) ? s[cc0] : -INFINITY;
            }
          }
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
          for (int i = 0; i < kKeys / 2; i += 8) {
            mx0 = fmax3(mx0, s[i + 0], s[i + 1]);
            mx1 = fmax3(mx1, s[i + 2], s[i + 3]);
            mx2 = fmax3(mx2, s[i + 4], s[i + 5]);
            mx3 = fmax3(mx3, s[i + 6], s[i + 7]);
          }
          const float cmax = fmax3(fmaxf(mx0, mx1), mx2, mx3) * scale_log2;
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
            // chunk 0: O_w holds PV_w of this item's earlier tiles (all retired).  chunk 1:
            // chunk 0's P (packed against the old max) is already being consumed by the
            // first-half PV, so let that retire and rescale O_w as a whole instead
            if (ch == 1) {
              mbar_wait(&bar[kPVDone0 + wg], c & 1);
              pv_pending = false;
              tc_fence_after();
            }
            if (ch == 1 || j > it.first(wg)) {
#pragma unroll
              for (int cc = 0; cc < HD / 32; ++cc) {
                uint32_t r[32];
                tmem_ld32(o_col + cc * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
                tmem_st32(o_col + cc * 32, r);
              }
            }
            tmem_wait_st();
          }
          // p = 2^(s*scale - m): packed FFMA2, MUFU for 16-kPoly16 of every 16 columns
          // and the FMA-pipe polynomial for the rest; packed FADD2 sums
          const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
          const uint64_t nm2 = f2_pack(-m, -m);
          uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
          for (int i = 0; i < kKeys / 2; i += 16) {
            float x[16];
#pragma unroll
            for (int e = 0; e < 16; e += 2) f2_unpack(ffma2(f2_pack(s[i + e], s[i + e + 1]), sc2, nm2), x[e], x[e + 1]);
#pragma unroll
            for (int e = 0; e < 16 - kPoly16; ++e) s[i + e] = ex2_mufu(x[e]);
#pragma unroll
            for (int e = 16 - kPoly16; e < 16; e += 2) f2_unpack(ex2_poly2(x[e], x[e + 1]), s[i + e], s[i + e + 1]);
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
              acc0 = fadd2(acc0, f2_pack(s[i + e], s[i + e + 1]));
              acc1 = fadd2(acc1, f2_pack(s[i + e + 2], s[i + e + 3]));
            }
          }
          if (tr) TRACE(c, 25 + 4 * wg + 2 * ch);
          float a0, a1, b0, b1;
          f2_unpack(acc0, a0, a1);
          f2_unpack(acc1, b0, b1);
          l += (a0 + a1) + (b0 + b1);
          uint32_t pk[kKeys / 4];
#pragma unroll
          for (int i = 0; i < kKeys / 4; ++i) pk[i] = pack_bf16(s[2 * i], s[2 * i + 1]);
          tmem_st32(s_col + ch * (kKeys / 4), pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bar[(ch == 0 ? kPFull0 : kPFullB0) + wg]);
        }
        if (half) mbar_arrive(&bar[kPFullB0 + wg]);  // one phase per tile
        if (tr) TRACE(c, 4 * wg + 2);
        ++c;
      }
      if (it.has(wg)) {
        // (m, l) of this WG -> epilogue (slot free once the epilogue read the previous one)
        mbar_wait(&bar[kLFree0 + wg], (oc & 1) ^ 1);
        sML[wg * 128 + row] = make_float2(any ? m : -INFINITY, l);
        mbar_arrive(&bar[kLFull0 + wg]);
        ++oc;
      }
    }
    if (pv_pending) mbar_wait(&bar[kPVDone0 + wg], (c - 1) & 1);
  } else if (warp >= 8) {
#if RCB_REG_EP > 128
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RCB_REG_EP));
#else
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RCB_REG_EP));
#endif
    // ------------------------------------------------------------ epilogue WG
    // O_w (TMEM) / l_w -> bf16 output rows, off the softmax critical path.  With a RoPE
    // table it also rotates each landed Q tile pair in place (rotate-half pairs
    // (i, i+HD/2)), two items ahead of the epilogue it trails.
    const int row = threadIdx.x - 256;  // == TMEM lane (warp % 4 quadrant)
    const int t_local = row / G;
    const int h_local = row % G;
    const uint32_t t_row = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    auto rotate_q = [&](const Item& it, int ii) {
      // Work unit = (query tile, token, chunk pair (i, i+HD/2) of 8 elements): one 64 B
      // cos/sin slice serves the G rows (heads) of that token.  Consecutive threads take
      // consecutive chunk pairs, so a warp's table reads are contiguous 512 B runs and its
      // shared accesses hit distinct 16 B chunks of each 128 B swizzled row.  Loops stay
      // rolled (this code shares the instruction cache with the softmax).
      constexpr int CP = HD / 16;  // chunk pairs per row
      constexpr int U = TQ * CP;   // units per query tile
      const int qb = ii & 1;
      const int total = (it.split() ? 1 : 2) * U;  // a split item reads Q0 only
      auto slice = [&](int u) {
        const int w = u / U, tt = (u % U) / CP, cp = u % CP;
        const int tok = min((2 * it.qp + w) * TQ + tt, it.q_len - 1);  // rows past q_len are masked
        return reinterpret_cast<const float4*>(rope + static_cast<int64_t>(it.q_pos0 + tok) *
                                                          (HD / 2) + cp * 8);
      };
      // Small G (MHA-like: 8-16 units per thread per item): a thread's units share its
      // chunk pair and step 128 / CP tokens = D positions at a time (within and across
      // the two tiles), so (cos, sin) of unit k+1 follow from unit k by the angle-addition
      // rotation by D * theta: one table slice per call instead of one L2 round trip per
      // unit, which made the G = 1 rotation latency-bound (LLaMA2 miss batch 148 -> 115 us).
      // (cos, sin)(D * theta) = table row 1 doubled log2(D) times.  G >= 4 (2-4 units per
      // thread) keeps the per-unit slices with one prefetched ahead: measured faster there.
      constexpr int D = 128 / CP;
      constexpr bool kStep = G <= 2;
      float4 cur[4], nxt[4], stp[4];
      if (row < total) {
        const float4* t = slice(row);
#pragma unroll
        for (int e = 0; e < 4; ++e) cur[e] = __ldg(t + e);
        if constexpr (kStep) {
          const float4* t1 = reinterpret_cast<const float4*>(rope + (HD / 2) + (row % CP) * 8);
#pragma unroll
          for (int e = 0; e < 4; ++e) stp[e] = __ldg(t1 + e);
#pragma unroll
          for (int d = 1; d < D; d *= 2)
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // double the angle: (c, s) -> (c^2 - s^2, 2 s c)
              const float4 a = stp[e];
              stp[e] = make_float4(a.x * a.x - a.y * a.y, 2.f * a.y * a.x,
                                   a.z * a.z - a.w * a.w, 2.f * a.w * a.z);
            }
        }
      }
      mbar_wait(&bar[kQFull0 + qb], (ii >> 1) & 1);
#pragma unroll 1
      for (int u = row; u < total; u += 128) {
        if (!kStep && u + 128 < total) {
          const float4* t = slice(u + 128);
#pragma unroll
          for (int e = 0; e < 4; ++e) nxt[e] = __ldg(t + e);
        }
        const int w = u / U, tt = (u % U) / CP, cp = u % CP;
        const uint32_t qbase = smem_u32(sQ) + (qb * S::kQT + w) * S::kQ;
        const int i0 = cp * 8, j0 = i0 + HD / 2;
        // (cos, sin) of elements (2e, 2e+1) as f32x2 pairs, shared by the G rows
        uint64_t c2[4], s2[4], ns2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          c2[e] = f2_pack(cur[e].x, cur[e].z);
          s2[e] = f2_pack(cur[e].y, cur[e].w);
          ns2[e] = f2_pack(-cur[e].y, -cur[e].w);
        }
#pragma unroll 1
        for (int h = 0; h < G; ++h) {
          const int r = tt * G + h;
          const uint32_t base = qbase + (r >> 3) * 1024 + (r & 7) * 128;
          const uint32_t a0 = base + (i0 / 64) * 16384 + ((((i0 % 64) / 8) ^ (r & 7)) << 4);
          const uint32_t a1 = base + (j0 / 64) * 16384 + ((((j0 % 64) / 8) ^ (r & 7)) << 4);
          uint32_t v0[4], v1[4];
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v0[0]), "=r"(v0[1]), "=r"(v0[2]), "=r"(v0[3]) : "r"(a0));
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v1[0]), "=r"(v1[1]), "=r"(v1[2]), "=r"(v1[3]) : "r"(a1));
#pragma unroll
          for (int e = 0; e < 4; ++e) {  // rotate-half: (x0, x1) -> (x0 c - x1 s, x1 c + x0 s)
            const uint64_t x0 = bf2_to_f2(v0[e]), x1 = bf2_to_f2(v1[e]);
            v0[e] = f2_to_bf2(ffma2(x1, ns2[e], fmul2(x0, c2[e])));
            v1[e] = f2_to_bf2(ffma2(x0, s2[e], fmul2(x1, c2[e])));
          }
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a0), "r"(v0[0]),
                       "r"(v0[1]), "r"(v0[2]), "r"(v0[3]));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a1), "r"(v1[0]),
                       "r"(v1[1]), "r"(v1[2]), "r"(v1[3]));
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (kStep) {  // advance D positions: angle + D * theta
            const float4 a = cur[e], b = stp[e];
            cur[e] = make_float4(a.x * b.x - a.y * b.y, a.y * b.x + a.x * b.y,
                                 a.z * b.z - a.w * b.w, a.w * b.z + a.z * b.w);
          } else {
            cur[e] = nxt[e];
          }
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
      mbar_arrive(&bar[kQReady0 + qb]);
    };
    int oc[2] = {0, 0};
    // rows of query tile qt = (sum_w c_w O_w) / (sum_w c_w l_w), c_w = 2^(m_w - max m) over
    // the WGs that worked on it (one for a pair item's tile, both for a split item)
    auto epilogue = [&](const Item& it, int qt, bool use0, bool use1, int qb, int ii) {
      (void)ii;
      const int tok = (2 * it.qp + qt) * TQ + t_local;
      const bool row_valid = tok < it.q_len;
      // a full tile (every token valid) is staged in its Q buffer and TMA-stored
      const bool stage = kStageO && !SPLIT && (2 * it.qp + qt + 1) * TQ <= it.q_len;
      const uint32_t stg = smem_u32(sQ) + (qb * S::kQT + (SPLIT ? 0 : qt)) * S::kQ;
      float2 ml0 = make_float2(-INFINITY, 0.f), ml1 = ml0;
      if (use0) {
        mbar_wait(&bar[kLFull0 + 0], oc[0] & 1);
        ml0 = sML[row];
        mbar_arrive(&bar[kLFree0 + 0]);
      }
      if (use1) {
        mbar_wait(&bar[kLFull0 + 1], oc[1] & 1);
        ml1 = sML[128 + row];
        mbar_arrive(&bar[kLFree0 + 1]);
      }
      const float mm = fmaxf(ml0.x, ml1.x);
      float c0 = use0 ? exp2f(ml0.x - mm) : 0.f;
      float c1 = use1 ? exp2f(ml1.x - mm) : 0.f;
      const float l = c0 * ml0.y + c1 * ml1.y;
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      c0 *= inv_l;
      c1 *= inv_l;
      // split-KV part (split-only launches): normalised fp32 O and (max, sum) of this KV
      // range go to the part workspace; rcb attn_combine_kernel merges the parts
      const bool part = SPLIT && it.ps >= 0;
      if (part && row_valid) part_ml[static_cast<int64_t>(it.ps) * kRows + row] = make_float2(mm, l);
      if (use0) mbar_wait(&bar[kOFull0 + 0], oc[0] & 1);
      if (use1) mbar_wait(&bar[kOFull0 + 1], oc[1] & 1);
      if (row == 0) TRACE(ii, use0 ? 19 : 21);
      tc_fence_after();
      __nv_bfloat16* orow =
          out + (static_cast<int64_t>(it.q_start + tok) * n_q_heads + it.kvh * G + h_local) * HD;
#pragma unroll 1
      for (int ch = 0; ch < HD / kOCols; ++ch) {
        uint32_t r0[kOCols], r1[kOCols];
        if (use0) tmem_ldn(t_row + 256 + ch * kOCols, r0);
        if (use1) tmem_ldn(t_row + 384 + ch * kOCols, r1);
        tmem_wait_ld();
        if (ch == HD / kOCols - 1) {  // O is in registers: release it to the next item
          tc_fence_before();
          if (use0) mbar_arrive(&bar[kOFree0 + 0]);
          if (use1) mbar_arrive(&bar[kOFree0 + 1]);
          if (row == 0) TRACE(ii, use0 ? 20 : 22);
        }
        float o[kOCols];
#pragma unroll
        for (int i = 0; i < kOCols; ++i) {
          const float a = use0 ? __uint_as_float(r0[i]) * c0 : 0.f;
          o[i] = use1 ? fmaf(__uint_as_float(r1[i]), c1, a) : a;
        }
        // 256-bit stores: each lane writes whole 32-byte sectors of its row.  A warp's rows
        // are 256 B apart, so every store touches 32 lines; with 16-byte stores the O
        // drain doubled those wavefronts and its LSU traffic stalled the softmax warps
        // sharing the SM sub-partitions (trace: -18% cycles per KV step without it)
        if (part) {
          if (!row_valid) continue;  // rows past q_len: nothing to combine
          float* prow = part_o + (static_cast<int64_t>(it.ps) * kRows + row) * HD + ch * kOCols;
#pragma unroll
          for (int i = 0; i < kOCols; i += 8)
            asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                         :: "l"(prow + i), "f"(o[i]), "f"(o[i + 1]), "f"(o[i + 2]), "f"(o[i + 3]),
                            "f"(o[i + 4]), "f"(o[i + 5]), "f"(o[i + 6]), "f"(o[i + 7])
                         : "memory");
        } else if (stage) {
          // SW128 Q-tile layout: [half][row][128 B], 16-byte chunk c of row r at (c ^ (r & 7))
          const int col0 = ch * kOCols;
          const uint32_t rb = stg + (col0 >> 6) * 16384 + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
          for (int k = 0; k < kOCols / 8; ++k) {
            const int c16 = ((col0 & 63) >> 3) + k;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};"
                         :: "r"(rb + ((c16 ^ (row & 7)) << 4)),
                            "r"(pack_bf16(o[8 * k + 0], o[8 * k + 1])),
                            "r"(pack_bf16(o[8 * k + 2], o[8 * k + 3])),
                            "r"(pack_bf16(o[8 * k + 4], o[8 * k + 5])),
                            "r"(pack_bf16(o[8 * k + 6], o[8 * k + 7]))
                         : "memory");
          }
        } else if (row_valid) {
#pragma unroll
          for (int i = 0; i < kOCols; i += 16) {
            uint32_t v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = pack_bf16(o[i + 2 * e], o[i + 2 * e + 1]);
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                         :: "l"(orow + ch * kOCols + i), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
                            "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                         : "memory");
          }
        }
      }
      if (stage) {
        fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the TMA store
        named_bar_sync(1, kRows);   // the whole tile is staged
        if (row == 0) {
          const int t0 = it.q_start + (2 * it.qp + qt) * TQ;
#pragma unroll
          for (int h = 0; h < HD / 64; ++h)
            tma_store_3d(&tm_o, stg + h * 16384, h * 64, it.kvh * G, t0);
          tma_store_commit();
        }
      }
      if (row == 0) TRACE(ii, 23);
      if (use0) ++oc[0];
      if (use1) ++oc[1];
    };
    const int n_mine =
        n_work > (int)blockIdx.x ? (n_work - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto item_of = [&](int ii) { return load_item(work, blockIdx.x + ii * gridDim.x); };
    // O_w is single-buffered, so item ii's epilogue must finish before item ii+1's first
    // PV_w and runs first; with a RoPE table, Q(ii+2) is rotated next (Q is double
    // buffered: it lands once the last QK of item ii retired; needed by item ii+2).
    constexpr int kAhead = 2;
    if (rope != nullptr)
      for (int ii = 0; ii < kAhead && ii < n_mine; ++ii) rotate_q(item_of(ii), ii);
    for (int ii = 0; ii < n_mine; ++ii) {
      const Item it = item_of(ii);
      if (it.split()) {
        epilogue(it, 0, true, it.has(1), ii & 1, ii);
      } else {
        epilogue(it, 0, true, false, ii & 1, ii);
        if (it.has(1)) epilogue(it, 1, false, true, ii & 1, ii);
      }
      if (kStageO && row == 0) {  // the staged O left smem: Q(ii + 2) may land in the buffer
        tma_store_wait_read();
        mbar_arrive(&bar[kQEmpty0 + (ii & 1)]);
      }
      if (rope != nullptr && ii + kAhead < n_mine) rotate_q(item_of(ii + kAhead), ii + kAhead);
    }
    if (kStageO && row == 0) tma_store_wait_all();
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Split-KV combine: group = {q_start, q_len, tok_base, kv_head, slot0, n_parts} of one
// query tile whose KV range ran as n_parts items.  Thread = tile row (token, head);
// O = sum_p 2^(m_p - M) l_p O_p / sum_p 2^(m_p - M) l_p over parts with l_p > 0.
constexpr int kGroupInts = 6;
__global__ void __launch_bounds__(kRows)
    attn_combine_kernel(const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                        const int* __restrict__ groups, __nv_bfloat16* __restrict__ out,
                        int n_q_heads, int G, int HD) {
  const int* gp = groups + blockIdx.x * kGroupInts;
  const int q_start = gp[0], q_len = gp[1], tok_base = gp[2], kvh = gp[3], slot0 = gp[4],
            np = gp[5];
  const int row = threadIdx.x;
  const int tok = tok_base + row / G;
  if (tok >= q_len) return;
  float mx = -INFINITY;
  for (int p = 0; p < np; ++p) {
    const float2 ml = part_ml[static_cast<int64_t>(slot0 + p) * kRows + row];
    if (ml.y > 0.f) mx = fmaxf(mx, ml.x);
  }
  float wsum = 0.f;
  for (int p = 0; p < np; ++p) {
    const float2 ml = part_ml[static_cast<int64_t>(slot0 + p) * kRows + row];
    wsum += ml.y > 0.f ? exp2f(ml.x - mx) * ml.y : 0.f;
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  __nv_bfloat16* orow = out + (static_cast<int64_t>(q_start + tok) * n_q_heads + kvh * G + row % G) * HD;
  // any number of parts: a part's weight is recomputed per 8-column chunk (no per-part array)
  for (int c = 0; c < HD; c += 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int p = 0; p < np; ++p) {
      const float2 ml = part_ml[static_cast<int64_t>(slot0 + p) * kRows + row];
      if (!(ml.y > 0.f)) continue;
      const float4* src = reinterpret_cast<const float4*>(
          part_o + (static_cast<int64_t>(slot0 + p) * kRows + row) * HD + c);
      const float4 a = src[0], b = src[1];
      const float w = exp2f(ml.x - mx) * ml.y * inv;
      acc[0] += w * a.x; acc[1] += w * a.y; acc[2] += w * a.z; acc[3] += w * a.w;
      acc[4] += w * b.x; acc[5] += w * b.y; acc[6] += w * b.z; acc[7] += w * b.w;
    }
    uint4 v;
    v.x = pack_bf16(acc[0], acc[1]);
    v.y = pack_bf16(acc[2], acc[3]);
    v.z = pack_bf16(acc[4], acc[5]);
    v.w = pack_bf16(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(orow + c) = v;
  }
}

template <int HD, int G, int BT, bool SPLIT>
cudaError_t launch_s(const CUtensorMap& tq, const CUtensorMap& tkv, const CUtensorMap& to, void* out, int n_q_heads,
                     int layer, const int* blk_ids, const int* blk_valid,
                     const int* blk_pos, const int* work, int n_work, float scale_log2,
                     const float2* rope, float* part_o, float2* part_ml, cudaStream_t stream) {
  auto kern = prefix_prefill_kernel<HD, G, BT, SPLIT>;
  const uint32_t smem = Smem<HD, BT, SPLIT>::kTotal;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int grid = n_work < sms ? n_work : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = RCB_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tq, tkv, to, static_cast<__nv_bfloat16*>(out), n_q_heads,
                            layer, blk_ids, blk_valid, blk_pos, work, n_work, scale_log2, rope,
                            part_o, part_ml);
}

template <int HD, int G, int BT>
cudaError_t launch_t(bool split, const CUtensorMap& tq, const CUtensorMap& tkv, const CUtensorMap& to, void* out,
                     int n_q_heads, int layer, const int* bi, const int* bv, const int* bp,
                     const int* work, int n_work, float sl2, const float2* rope,
                     float* po, float2* pm, cudaStream_t st) {
  return split ? launch_s<HD, G, BT, true>(tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st)
               : launch_s<HD, G, BT, false>(tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
}

template <int HD, int G>
cudaError_t launch_bt(bool split, int bt, const CUtensorMap& tq, const CUtensorMap& tkv, const CUtensorMap& to, void* out,
                      int n_q_heads, int layer, const int* bi, const int* bv,
                      const int* bp, const int* work, int n_work, float sl2, const float2* rope,
                      float* po, float2* pm, cudaStream_t st) {
  switch (bt) {
    case 16: return launch_t<HD, G, 16>(split, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    case 32: return launch_t<HD, G, 32>(split, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    case 64: return launch_t<HD, G, 64>(split, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    case 128: return launch_t<HD, G, 128>(split, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int HD>
cudaError_t launch_g(bool split, int g, int bt, const CUtensorMap& tq, const CUtensorMap& tkv, const CUtensorMap& to, void* out,
                     int n_q_heads, int layer, const int* bi, const int* bv,
                     const int* bp, const int* work, int n_work, float sl2, const float2* rope,
                     float* po, float2* pm, cudaStream_t st) {
  switch (g) {
    case 1: return launch_bt<HD, 1>(split, bt, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    case 2: return launch_bt<HD, 2>(split, bt, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    case 4: return launch_bt<HD, 4>(split, bt, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    case 8: return launch_bt<HD, 8>(split, bt, tq, tkv, to, out, n_q_heads, layer, bi, bv, bp, work, n_work, sl2, rope, po, pm, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace attn

int prefix_prefill(const void* q, int64_t q_row_stride, void* o, int total_q_tokens,
                   int n_q_heads, const void* kv_pool, int64_t num_pool_blocks, int block_tokens,
                   int n_layers, int n_kv_heads, int head_dim, int layer, const int* req_meta,
                   const int* blk_ids, const int* blk_valid, const int* blk_pos, const int* work,
                   int n_work, float softmax_scale, const void* rope_table, int work_flags,
                   void* part_ws, int n_part_slots, const int* combine, int n_combine,
                   cudaStream_t stream) {
  if (n_work == 0) return RCB_OK;
  if (reinterpret_cast<uintptr_t>(o) % 32 != 0)
    return set_error(RCB_ERR_ARG, "attention output must be 32-byte aligned");
  const bool split_only = (work_flags & RCB_WORK_SPLIT_ONLY) != 0;
  if (n_combine > 0 && (!split_only || part_ws == nullptr || combine == nullptr || n_part_slots <= 0))
    return set_error(RCB_ERR_ARG, "split-KV parts need a split-only plan and a part workspace");
  // part workspace: float2 (max, sum) [slots][128 rows], then fp32 O [slots][128 rows][head_dim]
  float2* part_ml = static_cast<float2*>(part_ws);
  float* part_o = part_ws != nullptr
                      ? reinterpret_cast<float*>(part_ml + static_cast<int64_t>(n_part_slots) * 128)
                      : nullptr;
  if (head_dim != 64 && head_dim != 128) return set_error(RCB_ERR_ARG, "head_dim must be 64 or 128");
  if (n_kv_heads <= 0 || n_q_heads % n_kv_heads != 0) return set_error(RCB_ERR_ARG, "bad head counts");
  const int g = n_q_heads / n_kv_heads;
  if (layer < 0 || layer >= n_layers) return set_error(RCB_ERR_ARG, "layer out of range");
  CUtensorMap tq, tkv, to;
  {
    // output O [T][Hq][HD] (contiguous): the same box as a Q tile, for the TMA store
    const uint64_t dims[3] = {(uint64_t)head_dim, (uint64_t)n_q_heads, (uint64_t)total_q_tokens};
    const uint64_t strides[2] = {(uint64_t)head_dim * 2, (uint64_t)n_q_heads * head_dim * 2};
    const uint32_t box[3] = {64, (uint32_t)g, (uint32_t)(128 / g)};
    int rc = encode_tma_bf16(&to, o, 3, dims, strides, box);
    if (rc != RCB_OK) return rc;
  }
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
          ? attn::launch_g<128>(split_only, g, block_tokens, tq, tkv, to, o, n_q_heads, layer, blk_ids,
                                blk_valid, blk_pos, work, n_work, sl2,
                                static_cast<const float2*>(rope_table), part_o, part_ml, stream)
          : attn::launch_g<64>(split_only, g, block_tokens, tq, tkv, to, o, n_q_heads, layer, blk_ids,
                               blk_valid, blk_pos, work, n_work, sl2,
                               static_cast<const float2*>(rope_table), part_o, part_ml, stream);
  if (e != cudaSuccess) return set_cuda_error(e, "prefix_prefill launch");
  if (n_combine > 0) {
    attn::attn_combine_kernel<<<n_combine, attn::kRows, 0, stream>>>(
        part_o, part_ml, combine, static_cast<__nv_bfloat16*>(o), n_q_heads, g, head_dim);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "attention combine launch");
  }
  return RCB_OK;
}

}  // namespace rcb

#ifdef RCB_TRACE
extern "C" int rcb_debug_attn_trace(void* host, int64_t bytes) {
  return cudaMemcpyFromSymbol(host, rcb::attn::g_trace, bytes) == cudaSuccess ? 0 : 3;
}
#endif
