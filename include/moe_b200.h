/*
 * moe_b200.h — C ABI of libmoe_b200.so, the B200-native (sm_100a) MoE-layer hot path.
 *
 * The reference (arxiv 2603.07685's `moelab`) exposes this path only as the Python
 * function API of pkg/src/moelab/routing.py; it has no native interface. Each entry point
 * below names the reference function(s) whose computation it replaces (file:line, relative
 * to the reference's pkg/src/moelab/). The Python shim paper_2603_07685_b200/routing.py
 * re-exposes the reference names on top of these calls.
 *
 * Conventions
 *   - Every function returns an int status: 0 ok, 1 invalid argument, 2 non-finite
 *     logits, 3 top_k > num_experts, 4 CUDA error, 5 unsupported, 6 workspace too small.
 *   - All pointers are DEVICE pointers unless noted; `stream` is a cudaStream_t. Work is
 *     enqueued on `stream` with no host synchronisation and no allocation: dynamic sizes
 *     (per-expert counts, padded offsets, number of active row blocks) live in device
 *     arrays produced by earlier calls; the host passes only static upper bounds.
 *   - bf16 = __nv_bfloat16 (2 bytes), row-major, rows 16-byte aligned.
 *   - "Padded plan": token copies grouped expert-major, ascending token index within an
 *     expert, each expert block starting at a multiple of 128 rows (the GEMM M tile);
 *     rows [off_pad[e] + eff[e], off_pad[e+1]) are zero. The oracle's compact row_id_map
 *     is each block's first eff[e] rows (moe_permute_compact_map).
 *   - W1 is stacked [E, 2m, h] with gate/up rows interleaved in 128-row blocks
 *     (rows [256j, 256j+128) = gate rows [128j, 128j+128), the next 128 = up rows);
 *     W2 is [E, h, m]. This is the oracle's per-expert out x in layout (routing.py:46-48).
 */
#ifndef MOE_B200_H_
#define MOE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ router
 * replaces route() routing.py:71-108 (score :85-91, bias on scores :95, stable top-k with
 * lowest-index ties :96-101, unnormalised probs :102, counts :106) and aux_loss()
 * routing.py:111-120. The logits GEMM x @ W_r (routing.py:79) runs on moe_gg_gemm_f32. */
/* Small-E router (E <= 16, e.g. Mixtral E = 8): the logits x . W_r (routing.py:79) are
 * computed on the CUDA cores inside the scoring / top-k kernel (x read once, W_r^T in shared
 * memory) instead of a tensor-core tile padded to 256 columns; same outputs as
 * moe_router_topk plus logits[T, E] fp32. moe_router_small_ok(E, h) says whether a shape is
 * eligible (else: moe_gg_gemm_f32 + moe_router_topk). */
int moe_router_small_ok(int E, int h);
int moe_router_fused(const void* x, int T, int h, const void* w_r, int E, int K, int score_fn,
                     const float* sel_bias, float* logits, int* topk_idx, float* topk_prob,
                     float* scores_out, int* counts, float* score_partials, int* status,
                     void* stream);
/* Its backward (aux part = aux_loss_grad_wr routing.py:123-137): dlogits
 * as compact fp32 [T, E]; dW_r = x^T dl with a fixed-order reduction over token groups
 * (workspace moe_router_wgrad_small_ws floats); router dX = dl . W_r^T as bf16 [T, h]. */
int moe_router_bwd_f32(const float* logits, int ld, int T, int E, int K, int score_fn,
                       const int* topk_idx, const float* dprob, const float* aux_grad,
                       float* dlogits, void* stream);
long long moe_router_wgrad_small_ws(int T, int h, int E);
int moe_router_wgrad_small(const void* x, int T, int h, const float* dl, int E, float* ws,
                           float* dw, void* stream);
int moe_router_dx_small(const float* dl, int T, int E, const void* w_r, int h, void* dx,
                        void* stream);
int moe_router_num_partials(int T);
int moe_router_topk(const float* logits, int ld, int T, int E, int K, int score_fn,
                    const float* sel_bias, int* topk_idx, float* topk_prob, float* scores_out,
                    int* counts, float* score_partials, int* status, void* stream);
int moe_router_finalize(const int* counts, const float* score_partials, int T, int K, int E,
                        float coeff, float* aux_out, float* aux_grad, float* mean_scores,
                        void* stream);
/* replaces aux_loss_grad_wr() routing.py:123-137 (generalised: combine + aux terms, softmax
 * and sigma/sum-sigma Jacobians). Writes bf16 dlogits [T, ldd]. */
int moe_router_bwd(const float* logits, int ld, int T, int E, int K, int score_fn,
                   const int* topk_idx, const float* dprob, const float* aux_grad,
                   void* dlogits, int ldd, void* stream);
/* Small-N tensor-core router (the default path; csrc/router_tc.cu). replaces route()
 * routing.py:71-108 + aux_loss() :111-120 in one tcgen05 GEMM whose epilogue scores, selects
 * and counts (thread per token, logits read from TMEM) + the finalize: x[T,h] bf16,
 * w_t[moe_router_tc_npad(E), h] bf16 = W_r^T zero-padded; logits out compact [T, E] fp32;
 * ws: moe_router_tc_fwd_ws(T, h, E) 4-byte words. K <= 8. Two launches (the GEMM with the
 * selection epilogue, then the finalize), no memsets. */
int moe_router_tc_npad(int E);
long long moe_router_tc_fwd_ws(int T, int h, int E);
int moe_router_tc_fwd(const void* x, int T, int h, const void* w_t, int E, int K, int score_fn,
                      const float* sel_bias, float coeff, float* logits, int* topk_idx,
                      float* topk_prob, float* scores_out, int* counts, float* ws, int* status,
                      float* aux_out, float* aux_grad, float* mean_scores, void* stream);
int moe_router_finalize_p(const int* counts, const float* score_partials, int P, int T, int K,
                          int E, float coeff, float* aux_out, float* aux_grad,
                          float* mean_scores, void* stream);
int moe_router_finalize_tiles(const int* tile_counts, const int* tile_status,
                              const float* score_partials, int P, int T, int K, int E,
                              float coeff, int* counts, int* status, float* aux_out,
                              float* aux_grad, float* mean_scores, void* stream);
/* Its backward: dl row-major bf16 [T, ldd] (dX GEMM operand) and/or dl^T bf16 [npad, ldt]
 * (moe_router_bwd semantics), and dW_r[h, E] fp32 = x^T dl on a small-N tcgen05 tile with a
 * fixed-order split-K sum (ws: moe_router_tc_wgrad_ws floats; h % 128 == 0). */
int moe_router_bwd2(const float* logits, int ld, int T, int E, int K, int score_fn,
                    const int* topk_idx, const float* dprob, const float* aux_grad,
                    void* dlogits, int ldd, void* dlt, int ldt, int npad, void* stream);
long long moe_router_tc_wgrad_ws(int T, int h, int E);
int moe_router_tc_wgrad(const void* x, int T, int h, const void* dlt, int ldt, int E, float* ws,
                        float* dw, void* stream);
/* W_r [h,E] bf16 -> W_r^T zero-padded [Epad,h] and/or W_r zero-padded [h,Epad] */
int moe_stage_router_weight(const void* w, int h, int E, int Epad, void* wt_pad, void* w_pad,
                            void* stream);
int moe_reduce_groups_f32(const float* in, int G, int rows, int cols_in, int cols_out,
                          float* out, void* stream);
/* measurement only (no reference counterpart): HBM write-only bandwidth probe, zeros `bytes`
 * (multiple of 16) at dst; mode 0 16-byte stores, 1 streaming (.cs) stores, 2 TMA bulk stores.
 * bench.py's write bound for write-dominated kernels. */
int moe_hbm_write_probe(void* dst, long long bytes, int mode, void* stream);

/* ------------------------------------------------------------------ permutation
 * replaces permute() routing.py:149-168, _expert_slices() :180-186, effective_counts()
 * :33-39, apply_capacity() :226-247 (capacity >= 0; pad = drop-and-pad). */
long long moe_permute_workspace_ints(int T, int K, int E);
int moe_permute_plan(const int* topk_idx, const float* topk_prob, int T, int K, int E,
                     int capacity, const int* cap_e, int pad, const int* phantom, int align,
                     int max_rows, int* meta, int* off_pad, int* off_c, int* kept, int* eff,
                     int* counts, int* block_expert, int* inv_map, int* row_src,
                     float* row_prob, int* workspace, int* status, void* stream);
/* Expert-parallel receive-side regroup maps (all-to-all layout <-> local padded plan);
 * capacity under EP keeps the lowest GLOBAL token indices (apply_capacity :240-243 on
 * the global batch) via the per-expert cap_e of moe_permute_plan. */
int moe_ep_regroup_map(const int* table, int n, int el, int rows_pad, int* map_pad,
                       int* map_recv, void* stream);
/* Sync-free planning: every table above (and the p2p transport's base[] / dst_off[], the
 * global-position capacity cap_local[], and the global aux loss + its score gradient) from
 * the all-gathered [n, ldg] rows of [counts(E) | mean scores(E) | ...], on the device, so the
 * EP step needs no host read and can be captured in a CUDA graph. rows_cap: rows of the
 * static plan buffers; a plan that would exceed it runs no GEMM blocks and sets *status.
 * Kernels taking `rows_pad` accept this static bound: rows past the table's off_pad[el]
 * are treated as outside the plan. */
int moe_ep_plan_device(const float* gathered, int ldg, int n, int E, int me, int T, int K,
                       int capacity, int pad, int align, float coeff, int rows_cap, int* base,
                       int* cap_local, int* table, int* block_expert, int max_blocks, int* meta,
                       int* dst_off, float* aux, float* aux_grad, int* status, void* stream);
/* Per padded row of the expert rank's plan: the address of that row in its source rank's
 * compact buffer (peers[s] + (dst_off[s*el+e] + q) * row_bytes; 0 for padding / phantom
 * rows). Feeds the *_scatter GEMMs, which return expert outputs / dX rows over NVLink from
 * their epilogue (the return all-to-all of perf.a2a_send_volume perf.py:62-70). */
int moe_ep_row_dst(const int* table, int n, int el, int rows_pad, const int* dst_off,
                   const unsigned long long* peers, long long row_bytes,
                   unsigned long long* row_dst, void* stream);
/* Split units for the grouped GEMMs' kFlagSplit (flags bit 1, with the pair bit 0): from a
 * 128-row aligned padded plan, each expert's blocks as 256-row pairs (CTA-pair engine) and
 * at most one single 128-row block (1-CTA engine): halves the padding of a 256-row plan.
 * U [2 + 2 * cap] int32: U[0] pairs, U[1] singles, U[2..2+cap) pair start blocks,
 * U[2+cap..2+2cap) single blocks; pass U as the GEMMs' num_m_blocks with flags = 3. */
int moe_split_units(const int* meta, const int* block_expert, const int* off_pad, int cap,
                    int* U, void* stream);
int moe_permute_compact_map(const int* meta, const int* off_c, const int* off_pad, int E,
                            const int* row_src, long long* row_id_map, int* compact_to_pad,
                            int max_compact, void* stream);
int moe_permute_gather(const void* x, int T, int K, int h, const int* inv_map,
                       const int* row_src, const int* meta, void* xp, void* stream);
int moe_zero_pad_rows(const int* meta, const int* row_src, int h, void* rows, void* stream);
int moe_gather_rows(const void* in, int h, const int* map, const int* n_dev, int n_host,
                    void* out, void* stream);

/* ------------------------------------------------------------------ combine
 * replaces unpermute_sum() routing.py:171-177, the prob multiply + unpermute of
 * combine_standard() :197-201, the scatter of combine_mem_efficient() :219-222 and the
 * residual fallback of moe_output_with_residual() :259-261. */
int moe_combine(const void* rows, int T, int K, int h, const int* inv_map,
                const float* weights, const void* resid, const void* extra,
                const void* extra2, void* out, void* stream);
int moe_combine_bwd(const void* dy, const void* o_rows, int T, int K, int h,
                    const int* inv_map, const float* prob, void* d_rows, float* dprob,
                    void* stream);
int moe_dprob_from_partials(const int* inv_map, long long n, const float* partial, int ldp,
                            float* dprob, void* stream);

/* ------------------------------------------------------------------ EP over NVLink peer memory
 * The EP all-to-all (bytes modelled by perf.a2a_send_volume perf.py:62-70) fused into the
 * permute / combine kernels: `peers` are device arrays [EP] of the symmetric (peer-mapped)
 * row buffers of every rank; a selection's row on its expert's rank is base[e] + inv_c[t,k]
 * (inv_c from a compact moe_permute_plan). Push kernels end with a system-scope fence; the
 * caller orders them against the consumers with a stream-ordered collective. */
int moe_ep_dispatch_push(const void* x, int T, int K, int h, const int* topk_idx,
                         const int* inv_c, const int* base, int el,
                         const unsigned long long* peers, const float* prob,
                         const unsigned long long* prob_peers, void* stream);
/* Overlapped dispatch: push only the selections whose expert lives on rank `dest`, then
 * moe_ep_signal publishes flag_peers[dest][slot] = *epoch (release, system scope). The
 * consumer GEMM (moe_gg_fc1_fwd_ep / moe_gg_fc2_dgrad_ep) waits per 128-row block for the
 * source ranks moe_ep_block_need lists, so the exchange overlaps the grouped GEMM. */
int moe_ep_dispatch_push_dest(const void* x, int T, int K, int h, const int* topk_idx,
                              const int* inv_c, const int* base, int el,
                              const unsigned long long* peers, const float* prob,
                              const unsigned long long* prob_peers, int dest, void* stream);
/* rows[r] -> *row_dst[r] (0 = skip): the return transfer as a standalone NVLink push, for
 * GEMMs without the scatter epilogue (the MXFP8 engine). */
int moe_ep_scatter_rows(const void* src, int rows, int h, const unsigned long long* row_dst,
                        void* stream);
int moe_ep_signal(const unsigned long long* flag_peers, int dest, int slot,
                  const unsigned int* epoch, void* stream);
/* *epoch += 1 in stream order (the dispatch epoch is a device scalar, so a captured CUDA
 * graph replays with a fresh epoch) */
int moe_ep_epoch_bump(unsigned int* epoch, void* stream);
/* Load / configure the kernels above before the first overlapped step (CUDA lazy loading
 * of a kernel launched beside a GEMM that waits for it would deadlock). */
int moe_ep_prepare(void);
int moe_ep_block_need(const int* table, int n, int el, int me, int nblocks, int cg,
                      unsigned int* need, int* order, void* stream);
/* rows_copy (nullable): local compact copy of the pulled rows, indexed by inv_c */
int moe_ep_combine_pull(const unsigned long long* peers, int T, int K, int h,
                        const int* topk_idx, const int* inv_c, const int* base, int el,
                        const float* weights, const void* resid, const void* extra,
                        const void* extra2, void* out, void* rows_copy, void* stream);
/* o_local: the forward's rows_copy (dprob = <dY, O>); NULL for the mem-efficient combine */
int moe_ep_combine_bwd_push(const void* dy, const void* o_local,
                            const unsigned long long* d_peers, int T, int K, int h,
                            const int* topk_idx, const int* inv_c, const int* base, int el,
                            const float* prob, float* dprob, void* stream);
int moe_ep_combine_bwd_push_dest(const void* dy, const void* o_local,
                                 const unsigned long long* d_peers, int T, int K, int h,
                                 const int* topk_idx, const int* inv_c, const int* base, int el,
                                 const float* prob, float* dprob, int dest, void* stream);
int moe_ep_dprob_pull(const unsigned long long* part_peers, int T, int K, const int* topk_idx,
                      const int* inv_c, const int* base, int el, int ldp, float* dprob,
                      void* stream);
/* Token de-duplication (HybridEP-style; leg byte model perf.py:81-160):
 * one row per (token, destination rank) crosses NVLink; the destination expands it to its
 * expert rows and pre-reduces the token's expert outputs. */
int moe_ep_token_ranks(const int* topk_idx, const int* inv_c, int T, int K, int el,
                       int* rank_idx, int* sel_j, int* sel_pos, void* stream);
int moe_ep_dispatch_dedup(const void* x, int T, int K, int h, const int* topk_idx,
                          const int* inv_c, const int* base, int el, const int* rank_idx,
                          const int* inv_rank, const int* tbase, const int* sel_j,
                          const int* sel_pos, const float* prob,
                          const unsigned long long* tok_peers,
                          const unsigned long long* map_peers,
                          const unsigned long long* srows_peers,
                          const unsigned long long* sprob_peers,
                          const unsigned long long* rprob_peers, void* stream);
int moe_ep_fill_pad_map(const int* map_pad, int rows, int* map, void* stream);
/* ECHO hot-expert cloning (planners.py:243-389): rewrite each selection to the virtual
 * expert (expert segment on its serving rank) that owns its global position. */
int moe_ep_echo_rewrite(const int* topk_idx, const int* inv_c, int T, int K, int ns,
                        const int* gbase, const int* seg_start, const int* seg_v, int* topk_v,
                        void* stream);
int moe_ep_expand_grad(const void* tok, const int* map, int rows, int h, const float* rowprob,
                       const void* o, void* d_o, float* dprob_rows, void* stream);

/* ------------------------------------------------------------------ paged stashing
 * replaces PagedStash (planners.py:394-463) with device-initiated
 * kernels: a circular free list of fixed-size pages (state[5]: head, free, peak used, failed
 * stashes, last result; ring[num_pages]); alloc pops ceil(rows / page_rows) pages from the
 * head into record[1..] (record[0] = count, -1 = out of pages), release appends them to the
 * tail in record order, copy moves rows [0, rows) between a dense buffer and the pages.
 * rows_dev (nullable) supplies the row count from device memory (sync-free). */
int moe_stash_init(int* state, int* ring, int num_pages, void* stream);
int moe_stash_alloc(int* state, const int* ring, int num_pages, int page_rows,
                    const int* rows_dev, int rows_host, int* record, int max_pages,
                    void* stream);
int moe_stash_release(int* state, int* ring, int num_pages, int* record, void* stream);
int moe_stash_copy(void* dense, long long ld_bytes, void* pool, int page_rows,
                   long long row_bytes, const int* record, const int* rows_dev, int rows_host,
                   int max_rows, int to_pages, void* stream);

/* ------------------------------------------------------------------ grouped GEMM (tcgen05)
 * replaces expert_activation()/expert_forward() routing.py:59-68 per expert block and the
 * corresponding backward GEMMs. flags bit 0 (grouped-M calls): the plan's
 * expert blocks are 256-row aligned -> CTA-pair engine (UMMA 256x256, cta_group::2). The
 * weight-gradient calls pick the pair engine by themselves whenever M % 256 == 0. */
int moe_gg_fc1_fwd(const void* xp, const void* w1, int a_rows, int max_rows, int h, int m,
                   int num_experts, const int* block_expert, const int* num_m_blocks,
                   const float* row_prob, void* preact, void* act, int flags, void* stream);
int moe_gg_fc2_fwd(const void* act, const void* w2, int a_rows, int max_rows, int m, int h,
                   int num_experts, const int* block_expert, const int* num_m_blocks,
                   void* out, int flags, void* stream);
/* fc2 forward / fc1 dgrad storing output row r at address row_dst[r] (0 = not stored): the
 * EP return transfer (combine / dX) fused into the GEMM epilogue, rows written straight into
 * peer GPUs' memory over NVLink. */
int moe_gg_fc2_fwd_scatter(const void* act, const void* w2, int a_rows, int max_rows, int m,
                           int h, int num_experts, const int* block_expert,
                           const int* num_m_blocks, const unsigned long long* row_dst, int flags,
                           void* stream);
int moe_gg_fc1_dgrad_scatter(const void* d_preact, const void* w1, int a_rows, int max_rows,
                             int m, int h, int num_experts, const int* block_expert,
                             const int* num_m_blocks, const unsigned long long* row_dst,
                             int flags, void* stream);
/* fc1 forward / fc2 dgrad overlapped with the EP dispatch of their A operand: a tile's rows
 * are read once src_flag[s] >= *epoch for every source s in block_need[block]; tiles run in
 * unit_order. status: int[8]; on a wait timeout (2 s) it receives [1, block, missing
 * source mask, epoch, flags[0..3]] and the remaining waits fail fast. */
int moe_gg_fc1_fwd_ep(const void* xp, const void* w1, int a_rows, int max_rows, int h, int m,
                      int num_experts, const int* block_expert, const int* num_m_blocks,
                      const float* row_prob, void* preact, void* act, int flags,
                      const unsigned int* src_flag, const unsigned int* epoch,
                      const unsigned int* block_need, const int* unit_order, int* status,
                      void* stream);
int moe_gg_fc2_dgrad_ep(const void* dout, const void* w2, const void* preact, int a_rows,
                        int max_rows, int h, int m, int num_experts, const int* block_expert,
                        const int* num_m_blocks, const float* row_prob, void* d_preact,
                        float* dprob_partial, int flags, const unsigned int* src_flag,
                        const unsigned int* epoch, const unsigned int* block_need,
                        const int* unit_order, int* status, void* stream);
/* Columns of the per-row dprob partials moe_gg_fc2_dgrad writes for ffn width m (workspace
 * query: one partial per (256-column tile, epilogue column half)). */
int moe_gg_dprob_partials(int m);
int moe_gg_fc2_dgrad(const void* dout, const void* w2, const void* preact, int a_rows,
                     int max_rows, int h, int m, int num_experts, const int* block_expert,
                     const int* num_m_blocks, const float* row_prob, void* d_preact,
                     float* dprob_partial, int flags, void* stream);
int moe_gg_fc1_dgrad(const void* d_preact, const void* w1, int a_rows, int max_rows, int m,
                     int h,
                     int num_experts, const int* block_expert, const int* num_m_blocks,
                     void* dxp, int flags, void* stream);
int moe_gg_wgrad(const void* a, const void* b, int max_rows, int M, int N, int num_experts,
                 const int* expert_offsets, void* dw, void* stream);
/* moe_gg_wgrad with flags: bit 0 = programmatic dependent launch (the caller asserts the
 * gradient reads nothing the previous launch on the stream writes; it fills that launch's
 * last wave and completes after it). */
int moe_gg_wgrad_ex(const void* a, const void* b, int max_rows, int M, int N, int num_experts,
                    const int* expert_offsets, void* dw, int flags, void* stream);
int moe_gg_wgrad_f32(const void* a, const void* b, int max_rows, int M, int N,
                     int num_groups, const int* offsets, float* dw, void* stream);
int moe_gg_gemm_f32(const void* a, const void* b, int a_rows, int max_rows, int K, int N,
                    int num_experts, const int* block_expert, const int* num_m_blocks,
                    float* out, void* stream);

/* ------------------------------------------------------------------ MXFP8
 * replaces the reference's MXFP8 recipe (quant.py:62-64, :166-201; formats.py:16-139):
 * 1x32 blocks along K, E8M0 scale 2^ceil(log2(amax/448)), E4M3 round-to-nearest-even codes.
 * Scales are written in the tiled layout of the block-scaled GEMM (per 128-row tile and
 * 128-wide K stage a 512-byte chunk; byte i*16 + c*4 + j = row c*32 + i, K-block j) and,
 * optionally, plain [rows, K/32]. w1_m > 0: x is a stacked W1 [E, 2m, h] in the bf16
 * engine's 128-row gate/up interleave and the output rows use the MXFP8 engine's 64-row
 * interleave (row remap fused into the quantisation). */
int moe_mxfp8_quantize(const void* x, long long ldx, int rows, int K, void* codes,
                       long long ldc, void* sf_plain, void* sf_tiled, int w1_m, void* stream);
/* transposing ("column twin", quant.py:195-200) quantisation: x [B, R, C] -> codes
 * [B, C, R], 1x32 blocks along R (the dgrad / wgrad K dimension), tiled scales of the
 * [B*C, R] operand (sf_plain optional [B*C, R/32]). */
int moe_mxfp8_quantize_t(const void* x, int B, int R, int C, void* codes, void* sf_tiled,
                         void* sf_plain, void* stream);
/* block-scaled tcgen05 grouped GEMMs (kind::mxf8f6f4, UMMA 128x128x32): bf16 output, and
 * fc1 + SwiGLU with the activation re-quantised to MXFP8 in the epilogue (fc2's A operand);
 * flags bit 0: CTA-pair engine (cta_group::2; expert blocks 256-row aligned). flags bit 1:
 * 256-wide N tiles with a single TMEM accumulator (else 128-wide, double-buffered). fc1's
 * w1q interleaves gate/up in 64-row blocks for 128-wide tiles, 128-row blocks (the bf16
 * engine's layout) for 256-wide tiles. */
int moe_gg_mxfp8_gemm(const void* a, const void* sfa, int a_rows, int max_rows, int K, int N,
                      const void* b, const void* sfb, int num_experts, const int* block_expert,
                      const int* num_m_blocks, void* out, int flags, void* stream);
/* fc2 dgrad + SwiGLU backward on MXFP8 operands (dO [rows, h], W2^T [E*m, h]); writes bf16
 * d_preact and d_preact quantised along 2m (fc1 dgrad's A operand, then moe_gg_mxfp8_gemm
 * with W1^T [E*h, 2m] codes from moe_mxfp8_quantize_t). */
int moe_gg_mxfp8_fc2_dgrad(const void* doq, const void* sfd, int a_rows, int max_rows, int h,
                           int m, const void* w2tq, const void* sfw, int num_experts,
                           const int* block_expert, const int* num_m_blocks, const void* preact,
                           void* d_preact, void* dpre_q, void* dpre_sf, int flags,
                           void* stream);
/* weight gradient on MXFP8 operands (grouped over experts along K = token rows):
 * dw[e] (bf16 [M, N]) = sum_{r in [k_off[e], k_off[e+1])} A[r, :]^T B[r, :], with A^T / B^T
 * as codes [M, K] / [N, K] from moe_mxfp8_quantize_t (blocks along the token rows). */
int moe_gg_mxfp8_wgrad(const void* at, const void* sfa, const void* bt, const void* sfb, int K,
                       int M, int N, int num_experts, const int* k_off, void* dw, int flags,
                       void* stream);
int moe_gg_mxfp8_fc1(const void* xq, const void* sfx, int a_rows, int max_rows, int h, int m,
                     const void* w1q, const void* sfw, int num_experts, const int* block_expert,
                     const int* num_m_blocks, void* preact, void* act, void* act_q,
                     void* act_sf, int flags, void* stream);
/* _t variants: the epilogue also writes its activation (act / d_preact) quantised along the
 * token rows -- codes [C, max_rows] (C = m / 2m), tiled scales: the weight-gradient GEMM's
 * operand, block amax by warp shuffles over the 32 TMEM lanes (one lane per row). */
int moe_gg_mxfp8_fc1_t(const void* xq, const void* sfx, int a_rows, int max_rows, int h, int m,
                       const void* w1q, const void* sfw, int num_experts,
                       const int* block_expert, const int* num_m_blocks, void* preact,
                       void* act, void* act_q, void* act_sf, void* act_t, void* act_t_sf,
                       int flags, void* stream);
int moe_gg_mxfp8_fc2_dgrad_t(const void* doq, const void* sfd, int a_rows, int max_rows,
                             int h, int m, const void* w2tq, const void* sfw, int num_experts,
                             const int* block_expert, const int* num_m_blocks,
                             const void* preact, void* d_preact, void* dpre_q, void* dpre_sf,
                             void* dpre_t, void* dpre_t_sf, int flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MOE_B200_H_ */
