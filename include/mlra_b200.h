/*
 * mlra_b200.h -- C ABI of the B200 (sm_100a) decode-attention kernels for the latent
 * attention family (MLRA-4 / MLA) and its GQA comparison variant.
 *
 * The reference (arxiv 2603.02188 "attnkit") has no FFI: its operator boundary is the
 * Python decode API. Each entry point below replaces one piece of that path; the
 * reference function it stands in for is cited per function (paths relative to
 * /root/reference/pkg/src/attnkit/). INTEGRATION.md shows the ctypes binding a
 * maintainer would add on the reference side.
 *
 * Conventions
 *  - Every pointer is a device pointer unless stated otherwise; bf16 buffers are passed
 *    as void* (IEEE bfloat16, row-major, contiguous), fp32 as float*.
 *  - Every call is asynchronous and stream-ordered on `stream` (a cudaStream_t, NULL =
 *    legacy default stream). No call allocates device memory: the caller owns all
 *    buffers and sizes the split-KV workspace with mlra_workspace_bytes().
 *  - Return value: 0 on success, otherwise a negative MLRA_ERR_* code; the message of
 *    the last failure on the calling thread is available from mlra_last_error().
 *  - Calls on different streams may run concurrently from different host threads.
 */
#ifndef MLRA_B200_H
#define MLRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLRA_OK 0
#define MLRA_ERR_SHAPE (-1)   /* ShapeMismatchError (errors.py:8) */
#define MLRA_ERR_CONFIG (-2)  /* ConfigError (errors.py:16)        */
#define MLRA_ERR_NUMERIC (-3) /* NumericError (errors.py:12)       */
#define MLRA_ERR_CUDA (-4)    /* launch / runtime failure          */

/* ABI version (major*100 + minor). */
int mlra_version(void);  /* 200: fused single-launch step, status word */

/* Message of the last failed call on this thread ("" if none). */
const char* mlra_last_error(void);

/* Number of SMs of the current device (used to size split-KV grids). */
int mlra_num_sms(void);

/*
 * K0 -- append one token row per sequence to the paged cache.
 * Replaces decode.py:129-150 (append_owned) -> cache.py:44-57 (KvCache.append).
 *   rows        [B, W] bf16, W = NB*DLAT + DR  ([latent block 0 | ... | rope])
 *   block_table [B, max_pages] int32 page ids; positions [B] int32 token slot to write
 *   pool        [num_pages*page_size, W] bf16
 *   advance     != 0: positions[s] += 1 after the write, as the reference append grows the
 *               cache (cache.py:44-57); pass the sequence lengths as positions. 0 leaves
 *               positions untouched.
 */
int mlra_cache_append(const void* rows, const int32_t* block_table, int32_t* positions, int B, int W,
                      int page_size, int max_pages, int advance, void* pool, void* stream);

/*
 * K0 (fused write side) -- the cache half of latent.py:129-159 (latent_projections) plus
 * decode.py:129-150 (append_owned), for a batch of new tokens:
 *   c_kv  = alpha_kv * rmsnorm(kv_raw) per latent group (norm_groups consecutive groups of
 *           d_c/norm_groups columns: 1 for MLA / MLRA-4, one per group for GLA / MLRA-2;
 *           eps, tensors.py:83-87), blocks [block0, block0+nblocks) of the `branches` equal
 *           blocks kept (latent.py:145-158), each zero-padded to dlp
 *   k_rope = rope(kr_raw, rope_pos)     (rope.py:37-60: pairs (2l, 2l+1), theta_l =
 *           rope_base^(-2l/dr)), zero-padded to drp
 *   pool row [c_kv blocks | k_rope] bf16 written at slot slots[s] of sequence s.
 *   kv_raw [B, d_c] fp32 = h W^DKV (whole groups: the RMS spans a group's blocks), kr_raw
 *   [B, dr] fp32 = h W^KR. MLA: branches = 1. advance bit 0: slots[s] += 1 after the write
 *   (slots are then the sequence lengths, as in mlra_cache_append). advance bit 1 (value 2):
 *   launched as a programmatic dependent of the previous kernel on the stream, releasing its
 *   own dependent at once -- only valid when the next kernel waits for this one's completion
 *   before reading the pool or the lengths (decode_layer's query projection does). rope_pos == NULL: the rope
 *   position is the slot written (a cache holding positions 0..n-1). slots == NULL: the B rows
 *   are ONE sequence's tokens 0..B-1 (prefill), row s written at slot s of block_table row 0.
 */
int mlra_cache_append_latent(const float* kv_raw, const float* kr_raw, const int32_t* rope_pos, int32_t* slots,
                             const int32_t* block_table, int B, int d_c, int branches, int block0, int nblocks,
                             int dlp, int dr, int drp, float alpha_kv, float rope_base, float eps, int page_size,
                             int max_pages, int norm_groups, int advance, void* pool, void* stream);

/*
 * K1 -- query absorption (decode.py:155-167 absorb_query, applied per branch at :224).
 *   q_nope [B, H, DH] bf16, q_rope [B, H, DR] bf16
 *   w_uk   [H, DH, NB*DLAT] bf16: head-major pre-pack of the branch slices of W^UK
 *          (weights.py:91-93 layout (d_c, h*d_h), rows b*DLAT.. of branch b)
 *   q_abs  [B, NB, H, DLAT] bf16 out = score_scale * q_nope_h . W^UK_(b),(h)^T
 *   q_rope_out [B, H, DR] bf16 out = score_scale * q_rope
 *   score_scale = tau * log2(e)  (tau: config.py:100-112)
 */
int mlra_absorb_query(const void* q_nope, const void* q_rope, const void* w_uk, void* q_abs, void* q_rope_out, int B,
                      int H, int DH, int NB, int DLAT, int DR, float score_scale, void* stream);

/* Bytes of device workspace mlra_decode_step / mlra_decode_step_tp need: the numeric status word,
 * the absorbed queries, the split-KV partials, the merge scratch (and the counters of the
 * dev-only fused experiments). Zero-fill it once before first use. */
size_t mlra_workspace_bytes(int B, int H, int NB, int DLAT, int DR, int nsplit);

/*
 * Numeric status (attnkit/tensors.py:74-78 softmax_rows: NaN in the logits, or a row with no
 * finite logit -> NumericError). The FIRST 4 BYTES of every decode workspace are an int32
 * status word that the merge (K3, or the fused step's epilogue) ORs with MLRA_STATUS_NAN /
 * MLRA_STATUS_NO_FINITE; mlra_combine takes the word explicitly (or NULL). Kernels never stop
 * on a bad value (a serving loop keeps its CUDA graph); the caller checks when it wants to:
 * mlra_check_status synchronises `stream` (the one ABI call that does), reads the word, resets
 * it when `reset` != 0 and returns MLRA_ERR_NUMERIC if any flag was set.
 */
#define MLRA_STATUS_NAN 1
#define MLRA_STATUS_NO_FINITE 2
int mlra_check_status(int32_t* status, int reset, void* stream);

/* Split count used when the caller passes nsplit <= 0 (fills the SMs for this batch). */
int mlra_default_splits(int B, int max_seqlen, int NB, int SUB);
/* The same for H heads per device: K2's grid has ceil(H / head-group width) head groups, so one
 * wave needs nsplit * B * groups <= #SMs. */
int mlra_default_splits_heads(int B, int max_seqlen, int NB, int SUB, int H);

/*
 * K2 -- split-KV flash-decode over the paged latent cache (tcgen05 + TMA).
 * Replaces decode.py:217-230 (attend_local, latent branch) + cache.py:59-66 (read).
 *   q_abs [B, NB, H, DLAT], q_rope [B, H, DR]   (K1 outputs, pre-scaled)
 *   pool  [num_pages*page_size, W] bf16 with W = NB*DLAT + DR; DLAT = SUB*DLS,
 *         DLS in {64,128}; DR in {16,32,48,64}; page_size a multiple of 64
 *   seqlens [B] int32 (>= 1)
 *   o_part   [B, nsplit, NB, H, DLAT] fp32 out (per-split normalised latent mixture)
 *   lse_part [B, nsplit, NB, H]       fp32 out (per-split log2-sum-exp)
 */
int mlra_decode_partials(const void* q_abs, const void* q_rope, const void* pool, const int32_t* block_table,
                         const int32_t* seqlens, float* o_part, float* lse_part, int B, int H, int NB, int SUB,
                         int DLS, int DR, int page_size, int max_pages, int num_pages, int nsplit, void* stream);

/*
 * K3 -- merge split partials, W^UV up-projection, ascending branch sum, alpha scaling.
 * Replaces decode.py:228 (einsum mc,cmp->mp) + decode.py:264-285 (reduce_contributions).
 *   w_uv [H, NB*DLAT, DH] bf16 head-major pre-pack of W^UV (weights.py:91-93)
 *   out  [B, H, DH] fp32 = alpha * sum_b Z_b . W^UV_(b),(h)     (upproj = 1)
 *        [B, NB, H, DH] fp32 = alpha * Z_b . W^UV_(b),(h)         (upproj = 2: per-branch
 *                              contributions, the (head, vec) list of attend_local)
 *        [B, NB, H, DLAT] fp32 = alpha * Z_b                      (upproj = 0)
 *   scratch [B, H, NB*DLAT] fp32 (the merged latent; unused and may be NULL when upproj = 0)
 *   alpha = alpha_attn (latent.py:56-61: 1/sqrt(branches) for mlra, 1 otherwise)
 */
int mlra_combine(const float* o_part, const float* lse_part, const void* w_uv, float* out, float* scratch, int B,
                 int H, int NB, int DLAT, int DH, int nsplit, float alpha, int upproj, int32_t* status, void* stream);

/*
 * One decode-attention step for a batch: K1 (absorb) + K2 (split-KV decode) + K3 (merge, W^UV,
 * ascending branch sum, alpha). Replaces decode.py:304-305 (attend_local + reduce_contributions
 * inside absorbed_decode_step) for every unit a device owns.
 * Launches: K1, then K2 as a programmatic dependent of K1 (K2's TMA producer streams the cache
 * while K1 drains; its consumers wait for the absorbed queries), then K3 in plain stream order
 * (except the merge + head-GEMM K3 variant over many heads at batch 1, which K2 releases as
 * a programmatic dependent at its epilogue). No completion counters are used on this path. MLRA_NO_PDL=1 launches K2 in plain stream order.
 * (Dev experiments, compiled into K2 only with -DMLRA_K2_FUSED_STEP and then switched on by
 * their environment variable; both measured slower at every shape tried, B = 1..16, 4K..128K:
 * MLRA_FUSE_GRID -- one launch with K1 / K3 inside K2 behind grid-wide counters in the
 * workspace; MLRA_FUSE_CLUSTER -- one launch with K1 / K3 inside the cluster of a sequence's
 * split CTAs, DSMEM hand-offs; fused_step.cuh. The product build returns MLRA_ERR_CONFIG if
 * either switch is set.)
 *   workspace: >= mlra_workspace_bytes(B, H, NB, DLAT, DR, nsplit) bytes (device, zeroed once)
 *   nsplit in [1, 160] (mlra_default_splits: one wave of the SMs for this batch)
 *   w_uk == NULL: the queries arrive absorbed -- q_nope is q~ [B, NB, H, DLAT] and q_rope the
 *   rotary query, both already scaled by score_scale (mlra_proj_query with the pre-multiplied
 *   W^UQ.W^UK_b weight) -- and the step is K2 (programmatic dependent of the caller's previous
 *   kernel) + K3.
 */
int mlra_decode_step(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv, const void* pool,
                     const int32_t* block_table, const int32_t* seqlens, float* out, void* workspace, int B, int H,
                     int DH, int NB, int SUB, int DLS, int DR, int page_size, int max_pages, int num_pages,
                     int nsplit, float score_scale, float alpha, void* stream);

/*
 * GQA comparison variant (attnkit/decode.py:232-240 attend_local's non-latent branch,
 * :258-261; kv_map zoo.py:35-38: query head i reads KV slot i // (h/g)) on the same split-KV
 * kernel machinery: per KV head one K and one V sub-block per 128-token tile, no rope part.
 *   q     [B, G, R, DH] bf16: query head b*R + j of this device (R = h/g per KV head),
 *         post-RoPE, unscaled, zero-padded to DH in {64, 128}
 *   pool  [num_pages*page_size, 2*G*DH] bf16 rows [K_0 | ... | K_{G-1} | V_0 | ... | V_{G-1}]
 *         (post-RoPE keys, plain values, each zero-padded to DH)
 *   score_scale = tau * log2(e), tau = 1/sqrt(d_h) (config.py:112), applied in fp32
 *   o_part [B, nsplit, G, R, DH] fp32, lse_part [B, nsplit, G, R] fp32
 *   out    [B, G*R, DH] fp32 (mlra_gqa_decode_step: K2 + split merge)
 * mlra_gqa_workspace_bytes includes the int32 status word (first 4 bytes, see mlra_check_status).
 */
int mlra_gqa_default_splits(int B, int G, int max_seqlen);
size_t mlra_gqa_workspace_bytes(int B, int G, int R, int DH, int nsplit);
int mlra_gqa_decode_partials(const void* q, const void* pool, const int32_t* block_table, const int32_t* seqlens,
                             float* o_part, float* lse_part, int B, int G, int R, int DH, int page_size, int max_pages,
                             int num_pages, int nsplit, float score_scale, void* stream);
int mlra_gqa_decode_step(const void* q, const void* pool, const int32_t* block_table, const int32_t* seqlens,
                         float* out, void* workspace, int B, int G, int R, int DH, int page_size, int max_pages,
                         int num_pages, int nsplit, float score_scale, void* stream);

/*
 * K4 -- attention output side: attnkit/zoo.py:125-127 (gated_output)
 * and the attention half of zoo.py:146-149 (block_forward), under tensor parallelism:
 *   y = resid + sum_{r < world} (attn_r * sigmoid(gate_pre_r)) @ w_o_r
 *   attn     [B, K] fp32   this rank's attention output, K = (heads held) * d_h, head-major
 *                          (mlra_decode_step's out viewed as [B, H*DH])
 *   gate_pre [B, K] fp32   hidden @ W_g[:, this rank's columns] (pre-activation), or NULL (no gate)
 *   w_o      [K, D] bf16   the rows of W_o for this rank's attention columns
 *   resid    [B, D] fp32   block input (the residual) or NULL; y [B, D] fp32 (same on every rank)
 *   B <= 64, K % 8 == 0, D % 8 == 0. The gated operand is rounded to bf16 (into workspace,
 *   mlra_outproj_workspace_bytes) for the tensor-core product (fp32 accumulation).
 * world == 1: comm may be NULL. world > 1: comm[r] = rank r's communication region
 * (mlra_outproj_comm_bytes, zero-filled once) as mapped in THIS process (its own region and
 * the peers' through mlra_ipc_open). The call epoch is kept in device memory (graph-safe); all
 * ranks must make the same sequence of calls.
 * The rank partials are exchanged by one-shot stores into every peer's region and summed in
 * ascending rank order -- no NCCL call; a peer missing for 4 s aborts the kernel.
 */
size_t mlra_outproj_comm_bytes(int B, int D, int world);
size_t mlra_outproj_workspace_bytes(int B, int K);  /* the gated bf16 operand [B, K] */
int mlra_outproj(const float* attn, const float* gate_pre, const void* w_o, const float* resid, float* y, int B,
                 int K, int D, int rank, int world, void* const* comm, void* workspace, void* stream);
/* The same kernels with `world` ranks simulated on ONE device (tests): arrays of world per-rank
 * pointers, one cooperative launch. Fails with MLRA_ERR_CONFIG when the grid cannot be resident. */
int mlra_outproj_sim(const float* const* attn, const float* const* gate_pre, const void* const* w_o,
                     const float* resid, float* const* y, int B, int K, int D, int world, void* const* comm,
                     void* const* workspace, void* stream);

/*
 * K5 -- one-shot all-reduce of n fp32 values over peer memory: y = sum over ranks of x_r in
 * ascending rank order (the device-order sum of per-rank contributions, attnkit/decode.py:
 * 264-285, tpsim.py:275-276), bit-identical on every rank; replaces the TP step's NCCL
 * all_reduce. comm[r] = rank r's region (mlra_allreduce_comm_bytes, zero-filled once) as mapped
 * in this process. The call epoch is kept in device memory, so the call can be captured in a
 * CUDA graph and replayed. All ranks must make the same sequence of calls.
 */
size_t mlra_allreduce_comm_bytes(int n, int world);
/*
 * mlra_decode_step with the TP sum over ranks fused into K3's epilogue (K3 + K5 in one kernel):
 * out [B, H, DH] = sum over the `world` ranks of each rank's alpha-scaled step output, in
 * ascending rank order (bit-identical on every rank). For owners that hold every head (MLRA-4
 * / MLRA-2 sharded by latent block). comm = the ranks' mlra_allreduce regions (n = B*H*DH).
 * When the chosen K3 variant cannot fuse (split-K merge for many splits, a grid that cannot be
 * resident), K5 runs after it on the same region.
 */
int mlra_decode_step_tp(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv, const void* pool,
                        const int32_t* block_table, const int32_t* seqlens, float* out, void* workspace, int B, int H,
                        int DH, int NB, int SUB, int DLS, int DR, int page_size, int max_pages, int num_pages,
                        int nsplit, float score_scale, float alpha, int rank, int world, void* const* comm,
                        void* stream);
int mlra_allreduce(const float* x, float* y, int n, int rank, int world, void* const* comm, void* stream);
int mlra_allreduce_sim(const float* const* x, float* const* y, int n, int world, void* const* comm, void* stream);

/* Communication region: a dedicated zero-filled cudaMalloc (so its IPC handle maps exactly). */
int mlra_comm_alloc(size_t bytes, void** dev_ptr_out);
int mlra_comm_free(void* dev_ptr);
/* CUDA IPC helpers for the communication regions (64-byte handles, exchanged by the caller). */
int mlra_ipc_handle(const void* dev_ptr, void* handle_out);
int mlra_ipc_open(const void* handle, void** dev_ptr_out);
int mlra_ipc_close(void* dev_ptr);

/*
 * K-1 -- pre-attention projections: the GEMVs of latent.py:129-159
 * (latent_projections) for a decode batch, as two weight-streaming GEMM launches (M <= 16
 * rows per launch; larger M loops; K <= 3072: at most 8 slices of 384 rows). Weights are bf16
 * and SLAB-PACKED once at load time: a
 * weight W [K, N] (row-major (in, out) as weights.py stores it) is passed as
 * [ceil(N/64)][round_up(K, 64)][64] with element [s][k][c] = W[k][64 s + c] (zero outside W), so
 * each CTA's slice is one contiguous HBM run. Activations enter as fp32 (split into bf16 hi +
 * lo operands: ~16-bit mantissa); fp32 accumulation; the K slices of an output slab are summed
 * in a fixed order.
 *
 * mlra_proj_down: y = x . w, x [M, K] fp32 (the hidden rows h), w = slab pack of
 *   [W^DQ | W^DKV (every latent group, concatenated) | W^KR]  (N = n_q + n_kv + n_kr columns)
 *   c_q_raw [M, n_q] = h W^DQ, kv_raw [M, n_kv] = h W^DKV (mlra_cache_append_latent's input),
 *   kr_raw [M, n_kr] = h W^KR  (fp32; any output may be NULL)
 *   ssq [ceil(n_q/64)][M] fp32 (or NULL): partial sums of squares of c_q_raw's rows, per 64
 *   columns -- the query rmsnorm's statistics for mlra_proj_query (M <= 16 when given).
 * mlra_proj_query: c_q = alpha_q * c_q_raw / sqrt(mean(c_q_raw^2) + eps) (tensors.py:83-87; the
 *   mean from ssq), then [q_x | q_r] = c_q . w with w = slab pack of [W^Q | W^QR] (nq + H*dr
 *   columns):
 *   q_out [M, nq] bf16 = q_scale * q_x. W^Q = W^UQ (q_nope, for K1) or, for a device holding
 *     NB latent blocks of DLAT columns, the pre-multiplied W^UQ_(h) . W^UK_(b),(h)^T columns in
 *     (b, h, c) order: q_out is then K1's q_abs [M, NB, H, DLAT] and K1 is skipped.
 *   r_out [M, H, drp] bf16 = r_scale * rope(q_r, pos[m] + pos_delta) (rope.py:37-60: pairs (2l, 2l+1),
 *     theta_l = rope_base^(-2l/dr)); columns [dr, drp) are not written (zero them once).
 *     (pos_delta = -1 with pos = the sequence lengths after mlra_cache_append_latent advanced
 *     them: the position of the token just appended.)
 * Both launch as programmatic dependents of the previous kernel on the stream (the weight
 * stream starts before it finishes) and release their own dependents only after that wait.
 */
int mlra_proj_down(const float* x, const void* w, int M, int K, int n_q, int n_kv, int n_kr, float* c_q_raw,
                   float* kv_raw, float* kr_raw, float* ssq, void* stream);
int mlra_proj_query(const float* c_q_raw, const float* ssq, float alpha_q, float eps, const void* w, int M, int K,
                    int nq, int H, int dr, int drp, const int32_t* pos, int pos_delta, float rope_base, float q_scale, float r_scale,
                    void* q_out, void* r_out, void* stream);

/*
 * K6 -- causal latent prefill attention (latent.py:172-230 latent_prefill,
 * causal softmax latent.py:164-169) for ONE sequence of n tokens already in the paged cache
 * (block_table row 0, positions 0..n-1), tcgen05 + TMA (prefill_kernel.cuh):
 *   out[q, h] = alpha * sum_b softmax_{k <= q}(q~_(b,h)[q] . C_b[k] + q_rope_h[q] . K_rope[k]) . C_b
 *               . W^UV_(b),(h)
 *   q_abs  [H, n, NB, DLAT] bf16 head-major absorbed queries (the batched GEMM q_nope_h .
 *          W^UK_h of the n rows), q_rope [n, H, DRq] bf16 (rope applied; DR <= DRq <= 64), both
 *          pre-scaled by tau*log2e; w_uv [H, NB*DLAT, DH] bf16 (K3's pack)
 *   pool   [num_pages*page_size, NB*DLAT + DRp] bf16 (DRp: the padded rope width), page_size a
 *          multiple of 128
 *   out    [n, H, DH] fp32; (DLAT, DH) in {(128, 128), (64, 64)}; alpha = alpha_attn.
 * CTA = (128 queries, head), all branches in ascending order (the branch sum in TMEM).
 */
int mlra_prefill_attention(const void* q_abs, const void* q_rope, const void* w_uv, const void* pool,
                           const int32_t* block_table, float* out, int n, int H, int NB, int DLAT, int DH, int DR,
                           int DRp, int DRq, int page_size, int max_pages, int num_pages, float alpha, void* stream);

/*
 * Prefill projection helpers (the n-row projections run as cuBLAS bf16 GEMMs around them):
 * mlra_rows_split: x [n, ldx] fp32 (first K columns) -> hi, lo bf16 (row stride ldo >= K) with x
 *   (norm = 0) or alpha * rmsnorm(x) (norm != 0; tensors.py:83-87) = hi + lo to ~16 bits.
 * mlra_query_epilogue: y [n, ldy] fp32 = [q_x (nq columns) | q_r (H * dr)] -> q_out bf16 [n, nq] =
 *   q_scale * q_x, r_out bf16 [n, H, drq] = r_scale * rope(q_r, pos0 + row) (rope.py:37-60),
 *   columns [dr, drq) zero.
 */
int mlra_rows_split(const float* x, int n, int K, int ldx, int norm, float alpha, float eps, void* hi, void* lo,
                    int ldo, void* stream);
int mlra_query_epilogue(const float* y, int n, int ldy, int nq, int H, int dr, int drq, int pos0, float rope_base,
                        float q_scale, float r_scale, void* q_out, void* r_out, void* stream);

/*
 * Ragged batches (sequences of very different lengths; attnkit/decode.py:204-230 decodes any
 * length). mlra_decode_plan builds K2's work table on the device (graph-safe): the tile budget
 * per CTA is the smallest c >= ceil(total tiles / ctas) for which the per-sequence split counts
 * ns_s = max(1, ceil(tiles_s / c)) (<= nsplit_max) fit `ctas` CTAs; sequence s gets ns_s
 * consecutive splits, items in ascending (sequence, split) order (the merge's order), surplus
 * items {-1, ...} (lse_part is not touched: the merge reads only the ns_s slots of a sequence).
 *   plan [ctas][4] int32 {sequence, split, first tile, tiles}; seq_splits [B] int32 = ns_s (the
 *   merge reads only those slots); tile_tokens = 128 (64 for MLA).
 * mlra_decode_step_ragged: mlra_decode_step with that plan (K2 grid = one wave of planned CTAs
 * per head group; K3 merges up to nsplit_max slots per sequence). w_uk == NULL: pre-absorbed
 * queries as in mlra_decode_step. Workspace: mlra_workspace_bytes(B, H, NB, DLAT, DR, nsplit_max).
 */
int mlra_decode_plan(const int32_t* seqlens, int B, int tile_tokens, int ctas, int nsplit_max, int32_t* plan,
                     int32_t* seq_splits, float* lse_part, int NB, int H, void* stream);
int mlra_decode_step_ragged(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv,
                            const void* pool, const int32_t* block_table, const int32_t* seqlens, float* out,
                            void* workspace, int B, int H, int DH, int NB, int SUB, int DLS, int DR, int page_size,
                            int max_pages, int num_pages, int nsplit_max, float score_scale, float alpha, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MLRA_B200_H */
