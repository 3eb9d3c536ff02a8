/*
 * pqtopk.h — C ABI of the B200-native PQTopK hot path (libpqtopk.so).
 *
 * What it computes (PAPER.md = arXiv 2408.09992, cited P:<line>):
 *   * a product-quantised catalogue: codebook G in N^{|I| x m}, item i -> m
 *     sub-ids g_i1..g_im (Eq. 1), b sub-ids per split;
 *   * sub-id scores s_{k,j} = psi_{k,j} . phi_k (Eq. 4), with phi_k
 *     the k-th contiguous d/m chunk of the sequence embedding phi;
 *   * item scores r_i = sum_k s_{k, g_ik} (Eq. 5) and the top K
 *     items (Algorithm 1 "PQTopK"), without materialising r;
 *   * the dense baseline r = W phi with W reconstructed from the codes
 *     (Eq. 2; Eq. 3).
 *
 * Numerical contract (readings R1-R7):
 *   * pq_subscores: each S entry is the fp64-accumulated dot product of fp32
 *     inputs, rounded once to fp32 (within 1e-5 relative of the exact value;
 *     in practice identical to fl32(exact));
 *   * item scores: ((+0.0f + S[0][g_0]) + S[1][g_1]) + ... + S[m-1][g_{m-1}],
 *     IEEE fp32 round-to-nearest, splits in order k = 0..m-1 (R1, R2);
 *   * ranking: score descending, then global item id ascending (R3); the result
 *     is therefore unique, and identical for any launch geometry or sharding.
 *
 * Conventions for every call:
 *   * sizes are element counts; all arrays are dense, row-major, C order;
 *   * "device" pointers are CUDA device (or managed) memory on the current
 *     device; "host or device" pointers are detected with
 *     cudaPointerGetAttributes;
 *   * `stream` is a cudaStream_t (NULL = legacy default stream); calls other
 *     than pq_create / pq_destroy only enqueue work and return;
 *   * no exception crosses the ABI; each call returns a pq_status and
 *     pq_last_error() describes the last failure of the calling thread;
 *   * device faults surface at the next synchronising call as PQ_ERR_CUDA;
 *   * the library never allocates on the hot path: scratch memory is the
 *     caller's `ws` of at least the size the *_workspace_bytes call returns;
 *     concurrent calls need distinct workspaces; a pq_index's catalogue is
 *     immutable and the index may be shared across threads and streams by the
 *     compute calls.  The configuration calls pq_set_tuning and
 *     pq_timing_enable mutate the index and are NOT thread-safe: call them
 *     while no other thread uses the index (timing records themselves are
 *     mutex-protected).
 */
#ifndef PQTOPK_H
#define PQTOPK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQTOPK_ABI_VERSION 2
#define PQTOPK_MAX_K 4096        /* largest K supported by pq_score_topk & co. */

typedef struct pq_index_s* pq_index;   /* opaque; immutable after pq_create */

typedef enum {
    PQ_OK = 0,
    PQ_ERR_INVALID_ARG = 1,     /* bad size, null pointer, inconsistent shape */
    PQ_ERR_CODE_RANGE = 2,      /* some code g_ik >= b (message names the first) */
    PQ_ERR_NONFINITE = 3,       /* reserved: non-finite input under validation */
    PQ_ERR_CUDA = 4,            /* CUDA runtime / cuBLAS error (message has text) */
    PQ_ERR_OUT_OF_MEMORY = 5,   /* device allocation in pq_create failed */
    PQ_ERR_UNSUPPORTED = 6,     /* valid but unsupported (e.g. K > PQTOPK_MAX_K) */
    PQ_ERR_WORKSPACE = 7        /* ws == NULL or ws_bytes too small */
} pq_status;

/* Optional launch tuning (all 0 = automatic).  Any setting gives bit-identical
 * results; this exists for tests (F12: two geometries, same bits) and tuning. */
typedef struct {
    int32_t variant;     /* 0 auto; 1 = generic row-group kernel; (2 = removed: the
                            superseded paired half-warp kernel; treated as auto);
                            3 = tiled phases (4 users per lane, TMA tables, TMEM partials);
                            4 = small-batch latency kernel (B <= 4, lane = item);
                            pq_search only: 5 = the fused single-launch query kernel with a
                            streamed code ring (K6, B <= 4); 7 = the fused single-launch
                            kernel with each CTA's code chunk resident in shared memory
                            (K7, B <= 4, catalogues whose chunks fit); 0 lets pq_search pick
                            K7, else K6, whenever one applies */
    int32_t ctas;        /* persistent CTAs of the scoring kernel (0 = #SMs x occupancy) */
    int32_t warps;       /* warps per CTA of the scoring kernel (0 = auto) */
    int32_t chunks;      /* item chunks per user group (0 = auto) */
    int32_t users_per_row; /* G, table row width in users (0 = auto; power of 2, <= 32) */
    int32_t shrink_watermark; /* K2 v3 candidate-buffer shrink watermark (0 = automatic; tests
                                 use a small value to force frequent shrinks) */
    int32_t cluster;     /* K6 prologue mode: 0 = cooperative GRID mode when B users' CTAs fit
                            in one wave (sub-id scores shared through L2 behind a grid
                            barrier), else cluster mode with a modelled cluster size;
                            1, 2, 4 or 8 = CLUSTER mode with that many CTAs per
                            thread-block cluster sharing one user's sub-id scores */
    int32_t reserved[1];
} pq_tuning;

/* ABI version, so a binding can refuse a mismatched library. */
int32_t pq_abi_version(void);

/* Last error of the calling thread ("" if none); valid until its next call. */
const char* pq_last_error(void);

/* Number of CUDA kernels this library has launched in this process. */
int64_t pq_launch_count(void);

/*
 * pq_create — build a catalogue index from the codebook G (Eq. 1).
 *   codes   : uint8 [N][m], host or device; g_ik = codes[i*m + k], 0 <= g < b.
 *   N       : items, 1 <= N, id_base + N <= 2^31 - 1.
 *   m       : splits, 1 <= m <= 64.      b : sub-ids per split, 1 <= b <= 256.
 *   id_base : global id of local item 0 (item sharding; 0 if unsharded).
 *   stream  : stream for the copies/kernels; synchronised before return, so the
 *             caller may free `codes` afterwards.
 *   out     : receives the handle (library-owned device memory, freed by
 *             pq_destroy).
 * Errors: PQ_ERR_INVALID_ARG, PQ_ERR_CODE_RANGE (first offending item and
 * split in pq_last_error, items in ascending order), PQ_ERR_OUT_OF_MEMORY,
 * PQ_ERR_CUDA.  On error *out is NULL and nothing is leaked.
 */
pq_status pq_create(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                    int64_t id_base, void* stream, pq_index* out);

/* pq_create_ex — pq_create with flags:
 *   PQ_CREATE_SMALL_BATCH_ONLY: build only the item-order layout (scoring
 *     with B <= 4 and the generic kernel); skips the batched (paired / tiled)
 *     layouts and their host-side colour pairing — for latency-serving
 *     indexes and very large catalogues (e.g. 10^9 items). */
#define PQ_CREATE_SMALL_BATCH_ONLY 1
pq_status pq_create_ex(const uint8_t* codes, int64_t N, int32_t m, int32_t b,
                       int64_t id_base, int32_t flags, void* stream, pq_index* out);

/* Frees the index (synchronises the device first).  NULL is a no-op. */
pq_status pq_destroy(pq_index idx);

/* Shape of an index (any output pointer may be NULL). */
pq_status pq_index_info(pq_index idx, int64_t* N, int32_t* m, int32_t* b,
                        int64_t* id_base);

/*
 * Layout of an index (diagnostics; any output may be NULL):
 *   paired      : 1 if the colour-paired layout (K2 v3 with 16 users) was built
 *   tmem_splits : always 0 (kept for ABI stability: it described the removed
 *                 v2 kernel's TMEM-resident splits)
 *   pairs_matched / leftover_items : complementary pairs found / items paired
 *                 without a complement (they are scored correctly but may hit
 *                 shared-memory bank conflicts)
 */
pq_status pq_index_layout(pq_index idx, int32_t* paired, int32_t* tmem_splits,
                          int64_t* pairs_matched, int64_t* leftover_items);

/* Bit mask of the K2 scoring variants this index supports (bit v set:
 * variant v usable; bit 1 is always set). */
pq_status pq_index_variants(pq_index idx, int32_t* mask);

/*
 * The launch plan pq_score_topk would use for (B, K) (diagnostics):
 * out[0] variant (1 row groups, 2 paired half-warps, 3 tiled phases, 4 small batch), out[1] users per table row
 * (G), out[2] users per group, out[3] warps per CTA, out[4] CTAs, out[5] item
 * chunks, out[6] TMEM splits, out[7] dynamic shared memory bytes.
 */
pq_status pq_plan_info(pq_index idx, int32_t B, int32_t K, int64_t out[8]);

/*
 * The plan pq_search would use for (B, d, K): out[0] = 5 when the fused K6
 * kernel runs, 7 when the fused chunk-resident K7 kernel runs (then out[1] table copies G, out[2] CTAs per cluster (0: one
 * cooperative grid sharing S through L2; K7: CTAs per user cluster in its cluster mode), out[3]
 * warps per CTA, out[4] CTAs, out[5] item chunks per user, out[6] 0, out[7]
 * dynamic shared memory bytes), else exactly pq_plan_info(B, K).
 */
pq_status pq_search_plan_info(pq_index idx, int32_t B, int32_t d, int32_t K, int64_t out[8]);

/* Set launch tuning for later calls on this index (not thread-safe with
 * concurrent scoring calls on the same index). NULL restores automatic. */
pq_status pq_set_tuning(pq_index idx, const pq_tuning* t);

/*
 * pq_subscores — sub-id score matrices (Eq. 4) for B users.
 *   seq_emb     : fp32 [B][d], device; phi_u.
 *   subitem_emb : fp32 [m][b][d/m], device; psi_{k,g} = subitem_emb[k][g][:].
 *   S           : fp32 [B][m][b], device, output;
 *                 S[u][k][g] = sum_{t < d/m} psi[k][g][t] * phi[u][k*d/m + t],
 *                 accumulated in fp64 and rounded once.
 * Requires d % m == 0, 1 <= m <= 64, 1 <= b <= 256, B >= 0 (B == 0: no-op).
 */
pq_status pq_subscores(const float* seq_emb, const float* subitem_emb,
                       int32_t B, int32_t d, int32_t m, int32_t b,
                       float* S, void* stream);

/* Workspace bytes pq_score_topk needs for (B, K) on this index and device. */
size_t pq_topk_workspace_bytes(pq_index idx, int32_t B, int32_t K);

/*
 * pq_score_topk — fused PQTopK scoring + selection (Alg. 1).
 *   S        : fp32 [B][m][b], device (e.g. from pq_subscores).
 *   ids      : int32 [B][K], device, output; global ids (id_base + local).
 *   scores   : fp32  [B][K], device, output; the exact fp32 item scores.
 * Row u is sorted by (score desc, id asc); min(K, N) valid entries, the tail
 * padded with id -1 and score -INFINITY.  B == 0 or K == 0: no-op.
 * No N-length score array is written to memory.  K <= PQTOPK_MAX_K.
 * S must be finite (non-finite S gives unspecified rankings).
 */
pq_status pq_score_topk(pq_index idx, const float* S, int32_t B, int32_t K,
                        void* ws, size_t ws_bytes, int32_t* ids, float* scores,
                        void* stream);

/*
 * pq_score_topk_subset — PQTopK over an item subset V (Alg. 1's input V,
 * P:119; SPEC "subset consistency"): the result is exactly the
 * full-catalogue ranking restricted to V, cut to K.
 *   V   : int32 [nV], device; LOCAL item ids (0 <= V[r] < N), strictly
 *         increasing; shared by the B users.  nV == 0: every row is padding.
 *   other arguments as pq_score_topk (ids returned are global ids).
 * Asynchronous and graph-capturable (enqueues only; nV == 0 fills the padding
 * on the device).  V is NOT validated: an entry outside [0, N) is read as code
 * 0 (memory-safe) and a V that is not strictly increasing gives an undefined
 * (but memory-safe) answer.  Pass PQ_SUBSET_VALIDATE to pq_score_topk_subset_ex
 * to check V on the device first (synchronises `stream`; PQ_ERR_INVALID_ARG
 * names the first bad position).  Workspace: pq_subset_workspace_bytes.
 */
size_t pq_subset_workspace_bytes(pq_index idx, int64_t nV, int32_t B, int32_t K);
pq_status pq_score_topk_subset(pq_index idx, const float* S, int32_t B, int32_t K,
                               const int32_t* V, int64_t nV, void* ws, size_t ws_bytes,
                               int32_t* ids, float* scores, void* stream);
#define PQ_SUBSET_VALIDATE 1
pq_status pq_score_topk_subset_ex(pq_index idx, const float* S, int32_t B, int32_t K,
                                  const int32_t* V, int64_t nV, int32_t flags, void* ws,
                                  size_t ws_bytes, int32_t* ids, float* scores, void* stream);

/*
 * pq_score_topk_exclude — PQTopK over I minus a per-user exclusion list (e.g.
 * the items a user has already interacted with; V_u = I \ excl_u in Alg. 1).
 *   excl     : int32, device; user u's excluded GLOBAL ids are
 *              excl[excl_off[u] .. excl_off[u+1]), sorted ascending.
 *   excl_off : int64 [B + 1], device.
 *   max_excl : >= every user's list length (the caller knows it; it sizes the
 *              internal top-(K + max_excl) pass).  K + max_excl <= PQTOPK_MAX_K.
 * Exact: the top-(K + max_excl) of I contains the top-K of I minus any
 * max_excl items.  Workspace: pq_exclude_workspace_bytes.
 */
size_t pq_exclude_workspace_bytes(pq_index idx, int32_t B, int32_t K, int32_t max_excl);
pq_status pq_score_topk_exclude(pq_index idx, const float* S, int32_t B, int32_t K,
                                const int32_t* excl, const int64_t* excl_off, int32_t max_excl,
                                void* ws, size_t ws_bytes, int32_t* ids, float* scores,
                                void* stream);

/* Workspace bytes for pq_search (pq_subscores + pq_score_topk in one call). */
size_t pq_search_workspace_bytes(pq_index idx, int32_t B, int32_t d, int32_t K);

/*
 * pq_search — the whole hot path for one batch: S = pq_subscores(phi, psi),
 * then pq_score_topk(S, K).  seq_emb / subitem_emb may be HOST or device
 * pointers and ids / scores may be host or device: host buffers are copied
 * through the workspace on `stream` (pinned host memory makes the copies
 * asynchronous) -- except on the K7 path, where PINNED host ids / scores are
 * written by the kernel in place (zero copy); with host outputs the call
 * synchronises `stream` before returning.
 *
 * Small batches (1 <= B <= 4, m in {4, 8, 16}, K <= 512; the paper's serving
 * case) run as ONE kernel: K7 when each CTA's item chunk fits in shared
 * memory (one CTA per user for tiny catalogues), else K6 (a streamed code
 * ring).  The grid computes S (Eq. 4, the same fp64 order and single rounding
 * as pq_subscores, so S is bit-identical), scores its item chunks (Eq. 5) and
 * selects; the last CTA of each user merges the chunk lists (Alg. 1).
 * Results are bit-identical to the multi-kernel path.  K7 and K6 (grid mode)
 * are cooperative launches preceded by a one-CTA reset kernel (the call's
 * counters live in the workspace); they assume no other work occupies the
 * GPU's SMs for their duration.
 */
pq_status pq_search(pq_index idx, const float* seq_emb, const float* subitem_emb,
                    int32_t B, int32_t d, int32_t K, void* ws, size_t ws_bytes,
                    int32_t* ids, float* scores, void* stream);

/* pq_search_ex flags */
#define PQ_SEARCH_NO_FUSED 1   /* always run K1 + K2 + K3 as separate kernels */

/*
 * pq_search_ex — pq_search with options.
 *   flags : PQ_SEARCH_* bits (0 = as pq_search).
 *   S_out : optional fp32 [B][m][b], DEVICE: receives the sub-id scores the
 *           call computed (NULL = not needed).  Size the workspace with
 *           pq_search_workspace_bytes (it covers both paths).
 */
pq_status pq_search_ex(pq_index idx, const float* seq_emb, const float* subitem_emb,
                       int32_t B, int32_t d, int32_t K, int32_t flags, void* ws,
                       size_t ws_bytes, int32_t* ids, float* scores, float* S_out,
                       void* stream);

/* Workspace bytes for pq_merge_topk. */
size_t pq_merge_workspace_bytes(int32_t P, int32_t B, int32_t K);

/*
 * pq_merge_topk — merge P partial top-K lists per user (e.g. the allgathered
 * local results of P item shards) into the global top-K (TopK of Alg. 1,
 * P:125, over the union of the shards' item sets; item loop sharded as P:122/
 * P:129 allow).
 *   ids, scores : [P][B][K], device; entries with id < 0 are empty.
 *   out_ids, out_scores : [B][K], device, outputs (same contract as
 *                         pq_score_topk).  Inputs must not alias outputs.
 * PRECONDITION: a real id appears in at most one of the P lists of a user
 * (the lists come from disjoint item shards).  Repeated ids are not detected;
 * the call stays memory-safe and writes every output slot, but the output may
 * then contain the repeated id twice.
 * Because every shard's list is its exact local top-K under the same total
 * order, the merge equals the unsharded result bit for bit.
 */
pq_status pq_merge_topk(const int32_t* ids, const float* scores, int32_t P,
                        int32_t B, int32_t K, void* ws, size_t ws_bytes,
                        int32_t* out_ids, float* out_scores, void* stream);

/*
 * pq_merge_topk_packed — pq_merge_topk over ONE packed buffer, the layout a
 * single all-gather of the shards' (id, score) pairs produces:
 *   lists : int32 [P][2][B][K], device: plane 0 = ids, plane 1 = the fp32
 *           score bits.  Same precondition, workspace
 *           (pq_merge_workspace_bytes) and outputs as pq_merge_topk.
 */
pq_status pq_merge_topk_packed(const int32_t* lists, int32_t P, int32_t B, int32_t K,
                               void* ws, size_t ws_bytes, int32_t* out_ids,
                               float* out_scores, void* stream);

/*
 * pq_reconstruct — dense item embeddings (Eq. 2):
 *   W[i][k*d/m + t] = subitem_emb[k][g_ik][t]   for local items i < N.
 *   subitem_emb : fp32 [m][b][d/m], device.   W : fp32 [N][d], device, output.
 */
pq_status pq_reconstruct(pq_index idx, const float* subitem_emb, int32_t d,
                         float* W, void* stream);

/* Workspace bytes for pq_dense_topk. */
size_t pq_dense_workspace_bytes(int64_t N, int32_t B, int32_t K);

/*
 * pq_dense_topk — the paper's "Transformer Default" baseline:
 *   r_u = W phi_u for every item (fp32 SGEMM via cuBLAS, TF32 disabled), then
 *   the top K per user with the same ordering/padding contract.
 *   W : fp32 [N][d], device.  seq_emb : fp32 [B][d], device.
 *   id_base : global id of row 0 of W.
 * The scores are fp32 GEMM results (not the PQ k-ordered sums); they agree
 * with Eq. 5 up to rounding.
 */
pq_status pq_dense_topk(const float* W, int64_t N, int32_t d, const float* seq_emb,
                        int32_t B, int32_t K, int64_t id_base, void* ws,
                        size_t ws_bytes, int32_t* ids, float* scores, void* stream);

/*
 * pq_recjpq_topk — Algorithm 2 "RecJPQScore" on the GPU: split-
 * major accumulation into an N-length fp32 score array per user (in `ws`),
 * then top-K.  Bitwise identical to pq_score_topk (same per-item add order);
 * provided as the paper's second baseline.
 */
size_t pq_recjpq_workspace_bytes(pq_index idx, int32_t B, int32_t K);
pq_status pq_recjpq_topk(pq_index idx, const float* S, int32_t B, int32_t K,
                         void* ws, size_t ws_bytes, int32_t* ids, float* scores,
                         void* stream);

/*
 * Optional kernel timing for benchmarks.  While enabled on an index,
 * pq_score_topk / pq_search record CUDA events on the call's stream around the
 * fused scoring kernel (K2) and around the final merge (K3).  pq_timing_read
 * synchronises those events, returns the accumulated milliseconds and launch
 * count since the last read, and resets them.  Disabled by default (no cost).
 */
pq_status pq_timing_enable(pq_index idx, int32_t on);
pq_status pq_timing_read(pq_index idx, double* k2_ms, double* k3_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* PQTOPK_H */
