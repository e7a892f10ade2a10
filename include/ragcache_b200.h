/* ragcache_b200.h — C-ABI of the B200-native RAGCache GPU hot path.
 *
 * The reference (ragsim, /root/reference/pkg/src/ragsim) is pure Python and
 * has no FFI: its GPU work is modelled by three stand-ins, and every entry
 * point below is the native operation that executes what the stand-in only
 * accounts for.  The host-side decision logic (KnowledgeTree, PGDSF,
 * ReorderQueue, DSP controller) stays in the reference's Python and calls
 * these through ctypes.
 *
 * Conventions: plain pointers and sizes only; every call returns an int
 * status.  Stream arguments are cudaStream_t passed as void* (NULL = legacy
 * default stream).  Device pointers are marked _dev.
 */
#ifndef RAGCACHE_B200_H
#define RAGCACHE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python layer maps 1 -> ragsim InsufficientEvictableCapacity
 * and 2..4 -> ragsim CacheError (tree.py:45-54) */
#define RCB_OK 0
#define RCB_ERR_NO_BLOCKS 1
#define RCB_ERR_BAD_HANDLE 2
#define RCB_ERR_CUDA 3
#define RCB_ERR_ARG 4

/* tier selector for rcb_node_blocks (mirrors ragsim Tier, tree.py:39-42) */
#define RCB_TIER_GPU 0
#define RCB_TIER_HOST 1

/* swap data paths (rcb_pool_create swap_mode) */
#define RCB_SWAP_STAGED 0   /* gather kernel -> HBM staging -> cudaMemcpyAsync (and reverse) */
#define RCB_SWAP_ZEROCOPY 1 /* gather/scatter kernel reading/writing mapped pinned host blocks */
#define RCB_SWAP_DMA 2      /* cudaMemcpyAsync per contiguous (gpu run, host run) */
#define RCB_POOL_ACCOUNTING 3 /* block bookkeeping only: no memory, no copies (CPU tests) */

const char* rcb_last_error(void);
int rcb_version(void);

/* ------------------------------------------------------------------ block pool
 * Paged doc-KV pool: num_gpu_blocks in HBM + num_host_blocks of pinned host
 * DRAM.  A block holds block_tokens tokens of every layer:
 *   [n_layers][2 (K,V)][n_kv_heads][block_tokens][head_dim] (elem_bytes each).
 * Allocation is lowest-free-block-first in both tiers (deterministic, so block
 * tables are reproducible by the Python oracle, oracle/block_oracle.py).
 * Node keys are KnowledgeNode.serial (tree.py:94-96); generation keys are
 * caller-chosen ids of in-flight prefills (simulator.py:84-114). */
typedef struct rcb_pool rcb_pool;

/* replaces TierState capacity accounting (tree.py:57-67) with real memory.
 * gpu_base: NULL = the pool cudaMallocs (and zero-fills) its own HBM. */
int rcb_pool_create(int64_t num_gpu_blocks, int64_t num_host_blocks, int32_t block_tokens,
                    int32_t n_layers, int32_t n_kv_heads, int32_t head_dim, int32_t elem_bytes,
                    int32_t swap_mode, void* gpu_base, void* copy_stream, rcb_pool** out);
int rcb_pool_destroy(rcb_pool* pool);
/* out[0]=gpu base ptr, out[1]=host base ptr, out[2]=block bytes, out[3]=gpu free blocks,
 * out[4]=host free blocks, out[5]=num gpu blocks, out[6]=num host blocks */
int rcb_pool_info(rcb_pool* pool, int64_t* out7);
/* out[0]=swap-out blocks, out[1]=swap-in blocks, out[2]=D2H bytes, out[3]=H2D bytes,
 * out[4]=swap-out calls, out[5]=swap-in calls, out[6]=kernel launches, out[7]=memcpy calls */
int rcb_pool_stats(rcb_pool* pool, int64_t* out8);
int rcb_pool_set_swap_mode(rcb_pool* pool, int32_t swap_mode);

/* direct node placement (tests / warm start) — new node resident in GPU */
int rcb_node_alloc_gpu(rcb_pool* pool, int64_t node_key, int32_t n_tokens);
/* GPU copy dropped with no transfer: swap-out-only-once repeat eviction
 * (tree.py:456-459) or the node side of _drop_subtree (tree.py:482-502) */
int rcb_node_free_gpu(rcb_pool* pool, int64_t node_key);
/* host copy freed: _free_from_host (tree.py:475-480) / dropped descendants */
int rcb_node_free_host(rcb_pool* pool, int64_t node_key);
/* first GPU eviction: allocate host blocks, copy D2H, free GPU blocks
 * (_demote_from_gpu swap branch, tree.py:460-473).  Batched; copies are issued
 * on the pool's copy stream (call rcb_pool_flush or any swap-in to issue). */
int rcb_node_swap_out(rcb_pool* pool, const int64_t* node_keys, int32_t n);
/* promotion of host-resident nodes: allocate GPU blocks, copy H2D, host copy
 * retained (load_to_gpu, tree.py:296-318) */
int rcb_node_swap_in(rcb_pool* pool, const int64_t* node_keys, int32_t n);
/* a generation's transient suffix (reserve_gpu, tree.py:320-327): one segment per
 * miss document plus one for the prompt, each block-aligned */
int rcb_gen_reserve(rcb_pool* pool, int64_t gen_key, const int32_t* seg_tokens, int32_t nseg);
/* free one segment early: the prompt segment at release_gpu (simulator.py:519),
 * or a miss-doc segment whose node another commit created meanwhile */
int rcb_gen_free_segment(rcb_pool* pool, int64_t gen_key, int32_t seg_idx);
/* a node created by insert_path (tree.py:252-294) takes over the segment that
 * the generation's prefill already filled — no copy */
int rcb_node_adopt(rcb_pool* pool, int64_t node_key, int64_t gen_key, int32_t seg_idx);
/* release_gpu (tree.py:329-333) / _abort (simulator.py:549-559): free every
 * segment not adopted */
int rcb_gen_release(rcb_pool* pool, int64_t gen_key);

int rcb_node_blocks(rcb_pool* pool, int64_t node_key, int32_t tier, int32_t* out, int32_t cap,
                    int32_t* n_out);
int rcb_gen_blocks(rcb_pool* pool, int64_t gen_key, int32_t seg_idx, int32_t* out, int32_t cap,
                   int32_t* n_out);
/* request block table = concat(GPU blocks of node_keys in order) ++ gen segments,
 * with the valid-token count of every block (node tails) */
int rcb_block_table(rcb_pool* pool, const int64_t* node_keys, int32_t n_nodes, int64_t gen_key,
                    int32_t* blocks_out, int32_t* valid_out, int32_t cap, int32_t* n_out);

/* issue batched copies; make `stream` wait for them; make the copy stream wait
 * for `stream` (block reuse fences); block until copies finish */
int rcb_pool_flush(rcb_pool* pool);
int rcb_pool_fence_into(rcb_pool* pool, void* stream);
int rcb_pool_wait_for(rcb_pool* pool, void* stream);
int rcb_pool_sync(rcb_pool* pool);
/* layer-pipelined swaps (replaces the serial charge
 * `transfer_ms + prefill_ms` of _admit, simulator.py:505-510, with overlap):
 * issue the pending swap-out (D2H) and swap-in (H2D) batches as groups of
 * `layers_per_group` layers (one strided DMA per block run and group, on the
 * copy engines; per group the swap-outs first, then the swap-ins; one event per
 * group).  A prefill that fences layer l with rcb_pool_fence_layer may then
 * write layer l of blocks freed by the swap-outs and read layer l of the
 * swapped-in nodes while later groups are still moving. */
int rcb_pool_flush_layered(rcb_pool* pool, int32_t layers_per_group);
/* make `stream` wait only for the layer group holding `layer` of the last
 * layered batch (full rcb_pool_fence_into when none is outstanding) */
int rcb_pool_fence_layer(rcb_pool* pool, int32_t layer, void* stream);
/* block until the copies already issued on the copy stream, and a pending
 * swap-out batch, finish (a pending swap-in batch stays pending): swap-outs, which the reference keeps off the critical
 * path (simulator.py:505-507), are drained before a measured prefill */
int rcb_pool_drain(rcb_pool* pool);

/* ------------------------------------------------------------------ kernels */

/* (1) vectorised block gather/scatter: dst_base[pairs[2i+1]] = src_base[pairs[2i]]
 * (block_bytes each).  Either base may be device memory or mapped pinned host
 * memory.  Stand-in replaced: transfer_time (cost_model.py:120-124). */
int rcb_kv_block_copy(const void* src_base, void* dst_base, int64_t block_bytes,
                      const int32_t* pairs_dev, int32_t n_pairs, void* stream);

/* RoPE (rotate-half, LLaMA convention) on q and k, then k/v scattered into the
 * pool at `slots_dev` (slot = block*block_tokens + offset) for `layer`.
 * q/k/v: bf16 [n_tokens][heads][head_dim] (row strides q_stride/kv_stride in
 * elements); q_out: bf16 [n_tokens][n_q_heads][head_dim].  q == NULL: only K/V
 * (Q's rotation fused into rcb_prefix_prefill through a RoPE table). */
int rcb_kv_write_rope(const void* q, int64_t q_stride, const void* k, const void* v,
                      int64_t kv_stride, void* q_out, const int32_t* positions_dev,
                      const int32_t* slots_dev, int32_t n_tokens, int32_t n_q_heads,
                      void* kv_pool, int32_t block_tokens, int32_t n_layers, int32_t n_kv_heads,
                      int32_t head_dim, int32_t layer, float rope_theta, void* stream);

/* Same as rcb_kv_write_rope with cos/sin read from an rcb_rope_table (identical values; no
 * per-token sincosf): the batched serving path, 8 tokens per CTA.  rope_table_dev must cover
 * every position. */
int rcb_kv_write_rope_table(const void* q, int64_t q_stride, const void* k, const void* v,
                            int64_t kv_stride, void* q_out, const int32_t* positions_dev,
                            const int32_t* slots_dev, int32_t n_tokens, int32_t n_q_heads,
                            void* kv_pool, int32_t block_tokens, int32_t n_layers,
                            int32_t n_kv_heads, int32_t head_dim, int32_t layer,
                            const void* rope_table_dev, void* stream);

/* cos/sin table for fused RoPE: float2 [max_pos][head_dim/2] = (cos, sin)(pos * theta^(-2i/d)) */
int rcb_rope_table(void* table_dev, int32_t max_pos, int32_t head_dim, float rope_theta,
                   void* stream);

/* (2) prefix-aware prefill attention (tcgen05/TMEM, TMA-staged K/V pages).
 * Stand-in replaced: interpolate(profile, alpha, beta) (cost_model.py:106-117,
 * simulator.py:506).
 *   q           : bf16 rows of q_row_stride elements, the first n_q_heads*head_dim of each
 *                 row = the token's query heads (e.g. a view into the QKV projection)
 *   o           : bf16 [total_q_tokens][n_q_heads][head_dim]
 *   rope_table  : NULL if q is already rotated, else rcb_rope_table output: Q tiles are
 *                 rotated in shared memory inside the kernel
 *   req_meta_dev: int32 [n_req][5] = {q_start, q_len(beta), q_pos0(alpha), blk_begin, blk_count}
 *   blk_*_dev   : int32 per block-table entry: pool block id, valid tokens, logical start pos
 *   work_dev    : int32 [n_work][8] = {q_start, q_len, q_pos0, blk_begin, blk_count,
 *                 q_pair, kv_head, n0 | half0 << 15 | n1 << 16 | half1 << 31}: two adjacent
 *                 128-row query tiles per item and the KV tiles each needs (built by
 *                 rcb_attn_plan, heaviest first)
 *   work_flags  : RCB_WORK_SPLIT_ONLY if every item has n1 == 0 (one query tile: decode
 *                 steps, short prompts over cached documents); the kernel then keeps one
 *                 Q tile per item buffer and runs a deeper K/V ring (HBM-bound launches)
 *   split-KV (split-only plans with few items, e.g. one request's decode step): items whose
 *                 field 6 is kv_head | (slot + 1) << 8 cover part of a query tile's KV range
 *                 and write fp32 (O, max, sum) to part slot `slot` of part_ws_dev =
 *                 float2 [n_part_slots][128] then float [n_part_slots][128][head_dim];
 *                 combine_dev = int32 [n_combine][6] {q_start, q_len, tok_base, kv_head,
 *                 slot0, n_parts} merges them into o.  NULL / 0 when unused. */
#define RCB_WORK_SPLIT_ONLY 1
int rcb_prefix_prefill(const void* q, int64_t q_row_stride, void* o, int32_t total_q_tokens,
                       int32_t n_q_heads, const void* kv_pool, int64_t num_pool_blocks,
                       int32_t block_tokens, int32_t n_layers, int32_t n_kv_heads,
                       int32_t head_dim, int32_t layer, const int32_t* req_meta_dev,
                       const int32_t* blk_ids_dev, const int32_t* blk_valid_dev,
                       const int32_t* blk_pos_dev, const int32_t* work_dev, int32_t n_work,
                       float softmax_scale, const void* rope_table_dev, int32_t work_flags,
                       void* part_ws_dev, int32_t n_part_slots, const int32_t* combine_dev,
                       int32_t n_combine, void* stream);
/* host-side work planner for rcb_prefix_prefill: writes up to cap items (8 int32 each) into
 * work_out (heaviest first) and returns the count in n_work_out.  Inputs are the
 * host copies of req_meta / blk_valid / blk_pos. */
int rcb_attn_plan(const int32_t* req_meta, int32_t n_req, const int32_t* blk_valid,
                  const int32_t* blk_pos, int32_t block_tokens, int32_t n_q_heads,
                  int32_t n_kv_heads, int32_t* work_out, int32_t cap, int32_t* n_work_out);

/* fused elementwise ops of the random-init decoder whose measured prefill and decode
 * step replace ragsim's T(alpha, beta) grid and decode_ms_per_token (cost_model.py:40-67,
 * config.py:52; paper_2404_12457_b200/profile.py).  fp32 residual stream x [n_rows][d]:
 * x += add (bf16, NULL = none); h_out = bf16(x * rsqrt(mean(x^2) + eps) * weight). */
int rcb_rmsnorm_residual(float* x_dev, const void* add_dev, const void* weight_dev,
                         void* h_out_dev, int32_t n_rows, int32_t d, float eps, void* stream);
/* out [n_rows][ffn] = bf16(silu(gate) * up), gate_up [n_rows][2*ffn] = (gate | up) */
int rcb_silu_mul(const void* gate_up_dev, void* out_dev, int32_t n_rows, int32_t ffn,
                 void* stream);

/* (3) exact inner-product top-k retrieval, staged (tcgen05 corpus GEMM +
 * top-k epilogue).  Stand-in replaced: generate_stages / StagedRetrieval
 * (speculation.py:33-59,149-194) behind the StageProvider seam (simulator.py:228).
 *   corpus_dev : bf16 [n_rows][dim] (dim % 64 == 0, dim <= 1024)
 *   queries_dev: bf16 [n_queries][dim], n_queries <= 256 (more than 64: a cluster of 2 or
 *                4 CTAs x 64 queries per corpus range, every corpus stage loaded once and
 *                multicast to the cluster, so the corpus is read once per call)
 *   stage s (0-based) = exact top-k over rows [0, floor((s+1)*n_rows/n_stages))
 *   ids_out_dev   : int64 [n_queries][n_stages][k] (row + id_offset), score desc / id asc
 *   scores_out_dev: fp32  [n_queries][n_stages][k]
 *   workspace: rcb_retrieval_workspace_bytes() bytes of device memory */
int64_t rcb_retrieval_workspace_bytes(int64_t n_rows, int32_t n_queries, int32_t k,
                                      int32_t n_stages);
int rcb_retrieval_topk(const void* corpus_dev, int64_t n_rows, int32_t dim,
                       const void* queries_dev, int32_t n_queries, int32_t k, int32_t n_stages,
                       int64_t id_offset, void* workspace_dev, int64_t workspace_bytes,
                       int64_t* ids_out_dev, float* scores_out_dev, void* stream);
/* debug / parity: full score matrix fp32 [n_rows][n_queries] from the same GEMM */
int rcb_retrieval_scores(const void* corpus_dev, int64_t n_rows, int32_t dim,
                         const void* queries_dev, int32_t n_queries, float* scores_out_dev,
                         void* stream);
/* merge per-shard staged top-k lists (after an NCCL allGather), on device:
 *   in: [n_shards][n_queries][n_stages][k], out: [n_queries][n_stages][k] */
int rcb_topk_merge_shards(const int64_t* ids_in_dev, const float* scores_in_dev,
                          int32_t n_shards, int32_t n_queries, int32_t n_stages, int32_t k,
                          int64_t* ids_out_dev, float* scores_out_dev, void* stream);

/* ---- peer-memory list exchange (replaces the two list allGathers above).
 * Each rank allocates an exchange window, exports it with a CUDA IPC handle and opens
 * every peer's (NVLink P2P on one box).  Per retrieval call with epoch e = 1, 2, ...:
 * rcb_peer_push writes this rank's [n_queries][n_stages][k] lists into slot (e&1, rank)
 * of every window and publishes e in each window's flags[rank] (system-scope release);
 * rcb_peer_merge waits (acquire, bounded by timeout_ns: *timed_out_dev = 1 instead of a
 * hang) for every rank's flag and merges its own window's slot (e&1).  A rank may push
 * e+1 only after every rank issued its epoch-e merge (the step's query allGather orders
 * it).  Replaces: the NCCL merge of retrieval_topk(..., ncclComm_t) in SURVEY §8b. */
#define RCB_PEER_HANDLE_BYTES 64
int64_t rcb_peer_window_bytes(int32_t n_ranks, int64_t n_entries);
int rcb_peer_window_alloc(int32_t n_ranks, int64_t n_entries, void** window_out);
int rcb_peer_window_free(void* window);
int rcb_peer_ipc_handle(void* window, void* handle_out);
int rcb_peer_open(const void* handle, void** window_out);
int rcb_peer_close(void* window);
int rcb_peer_push(void* const* windows, int32_t n_ranks, int32_t rank, int64_t n_entries,
                  const int64_t* ids_dev, const float* scores_dev, uint32_t epoch,
                  void* stream);
int rcb_peer_merge(const void* window, int32_t n_ranks, int32_t n_queries, int32_t n_stages,
                   int32_t k, uint32_t epoch, uint64_t timeout_ns, int32_t* timed_out_dev,
                   int64_t* ids_out_dev, float* scores_out_dev, void* stream);
/* the same window as a raw all-gather (the step's queries): rcb_peer_push_bytes copies
 * `bytes` (multiple of 8, <= 8 * n_entries) into the ids-region slot (e&1, rank) of every
 * window and publishes e; after rcb_peer_wait the gathered rows of all ranks are contiguous
 * at window + rcb_peer_slot_offset(n_ranks, n_entries, e), rank r at r * 8 * n_entries */
int rcb_peer_push_bytes(void* const* windows, int32_t n_ranks, int32_t rank, int64_t n_entries,
                        const void* src_dev, int64_t bytes, uint32_t epoch, void* stream);
int rcb_peer_wait(const void* window, int32_t n_ranks, int64_t n_entries, uint32_t epoch,
                  uint64_t timeout_ns, int32_t* timed_out_dev, void* stream);
int64_t rcb_peer_slot_offset(int32_t n_ranks, int64_t n_entries, uint32_t epoch);

#ifdef __cplusplus
}
#endif

#endif /* RAGCACHE_B200_H */
