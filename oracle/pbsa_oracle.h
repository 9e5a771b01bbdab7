/*
 * pbsa_oracle.h -- CPU ORACLE for the PBSA hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This is a CPU restatement of the reference's algorithm (SPEC.md op definitions on top of
 * the reference's numeric primitives in proj/src/tensor.cpp and proj/src/blockify.cpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the CPU baseline.  The product path
 * (paper_2604_21221_b200/, libpbsa_b200.so) never links or calls it.
 *
 * Parity pinning: the restated primitives (matmul_nt, matmul, masked_softmax_rows, blockify,
 * unblockify, block_index_map, Rng) are checked bit-exactly against the reference's own
 * sources compiled into oracle/_ref/libpbsa_ref.so (tests/test_oracle_vs_ref.py).  The SPEC-only
 * ops (compress, coarse scoring, Top-K, aggregate, Top-C, attention) are pinned against every
 * SPEC known-answer example and property (tests/test_oracle_kat.py, tests/golden/).  The
 * reference ships no implementation of those ops, so their at-scale index parity is defined by
 * this restatement ("parity pinned to SPEC KATs").
 *
 * Conventions: fp32 storage, fp64 accumulation in a fixed (ascending) order, exactly as
 * tensor.hpp:49-53 / SPEC.md:70 state.  All functions return 0 on success, 1 on invalid
 * argument (message via orc_last_error()).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_num_threads(void);
void orc_set_num_threads(int n);

/* ---- rng.hpp:11-57 restated (splitmix64 + Box-Muller, spare cached) ---- */
int orc_rng_normal(uint64_t seed, int64_t n, float* out);
int orc_rng_uniform(uint64_t seed, int64_t n, double* out);
uint64_t orc_rng_derive(uint64_t seed, uint64_t stream);

/* ---- tensor.cpp restated ---- */
/* tensor.cpp:34-55: out[ar x br] = a[ar x ac] * b[br x ac]^T, fp64 ascending-k dot, cast fp32 */
int orc_matmul_nt(const float* a, int64_t ar, int64_t ac, const float* b, int64_t br, float* out);
/* tensor.cpp:8-32: out[ar x bc] = a[ar x ac] * b[ac x bc], fp64 row accumulators, ascending k */
int orc_matmul(const float* a, int64_t ar, int64_t ac, const float* b, int64_t bc, float* out);
/* tensor.cpp:57-108: row softmax of scores(+mask); mask entries 0 or -inf; fully masked -> 0 */
int orc_masked_softmax_rows(const float* scores, int64_t rows, int64_t cols, const float* mask,
                            float* out);

/* ---- blockify.cpp restated ---- */
int orc_blockify(const float* x, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                 int64_t bh, int64_t bw, float* out);
int orc_unblockify(const float* xb, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                   int64_t bh, int64_t bw, float* out);
int orc_block_index_map(int64_t t, int64_t h, int64_t w, int64_t bt, int64_t bh, int64_t bw,
                        int64_t flat, int64_t* block_id, int64_t* in_block);

/* ---- router ---- */
/* SPEC.md:268-276 + :70: rep = float( sum_t double(x[t]) (ascending t) / double(b) ) */
int orc_compress_blocks(const float* x, int64_t n_blocks, int64_t b, int64_t d, float* reps);
/* scale = float(1/sqrt(double(d)))  (AttentionConfig SPEC.md:346-350) */
float orc_attention_scale(int64_t d);
/* probs = masked_softmax_rows(float(matmul_nt(qc,kc)) * scale) */
int orc_coarse_logits(const float* qc, int64_t nq, const float* kc, int64_t nk, int64_t d,
                      float scale, float* logits);
int orc_coarse_attention(const float* qc, int64_t nq, const float* kc, int64_t nk, int64_t d,
                         float scale, float* probs);
/* s[j] = float( sum_i double(a[i][j]) (ascending i) / double(rows) ) */
int orc_aggregate_scores(const float* a, int64_t rows, int64_t cols, float* s);
/* k = max(1, ceil(n_local * ratio)); 0 < ratio <= 1 */
int orc_topk_count(int64_t n_local, double ratio, int64_t* k);
/* per row the k largest entries by (value desc, index asc); indices written
 * in ascending order (the BlockMask visible set).  k in [1, cols]. */
int orc_select_topk(const float* a, int64_t rows, int64_t cols, int64_t k, int32_t* sel);
/* token mask [nqb*b][n_p_tok + n_local*b]: 0 over persistent columns,
 * 0 over tokens of visible local blocks, -inf elsewhere */
int orc_build_mask(int64_t nqb, int64_t b, int64_t n_p_tok, int64_t n_local, const int32_t* sel,
                   int64_t k, float* mask);

/* ---- attention ---- */
/* out = masked_softmax_rows(float(matmul_nt(q,k))*scale + mask) * v  (dense) */
int orc_attention_reference(const float* q, int64_t nq, const float* k, const float* v,
                            int64_t nkv, int64_t d, const float* mask, float scale, float* out);
/* block-skipping online softmax.  Query block i (rows [i*bq, i*bq+bq) of q)
 * visits, in list order, the key blocks vis[i*n_vis + j] of the block store (kv_store block g
 * = rows [g*bkv, g*bkv+bkv) of k/v).  fp32 logits float(dot64)*scale, fp64 running sum and
 * accumulators, fp32 running max.  Rows of query blocks with qmask[i]==0 are skipped (left
 * untouched) so callers can sample; qmask may be NULL (all rows). */
int orc_attention_sparse(const float* q, int64_t nqb, int64_t bq, const float* k, const float* v,
                         int64_t bkv, const int32_t* vis, int64_t n_vis, int64_t d, float scale,
                         const uint8_t* qmask, float* out, float* lse);
/* Gradient of attention_sparse (the reference ships no backward; this is the derivative of the
 * dense masked attention SPEC.md:358-366 restricted to the visible blocks, i.e. of Eq. 3-5
 * PAPER.md:128-143): dq, dk, dv for upstream d_out, all in fp64 (scores s = scale * q.k, p =
 * softmax over the row's visible tokens, dP = d_out.v, D = sum p*dP, dS = p*(dP - D);
 * dq = scale * sum dS k, dk = scale * sum dS q, dv = sum p d_out).  dk / dv [n_store, bkv, d]
 * accumulate over every query row that sees the block (caller zero-initialises them). */
int orc_attention_sparse_backward(const float* q, int64_t nqb, int64_t bq, const float* k, const float* v,
                                  int64_t bkv, const int32_t* vis, int64_t n_vis, int64_t d, float scale,
                                  const float* d_out, float* dq, float* dk, float* dv, int64_t n_store);
/* SPEC.md:385-393 */
int orc_flop_count(int64_t nq, int64_t np, int64_t nl, int64_t b, int64_t k_sel, int64_t d,
                   double* dense, double* sparse, double* ratio);
/* SPEC.md:527-544 */
int orc_kv_length(int64_t n_c, double local_ratio, double persist_ratio, int64_t* n_kv);
int orc_kv_bytes(int64_t tokens, int64_t layers, int64_t kv_heads, int64_t head_dim,
                 int64_t bpe, int64_t* bytes);

/* ---- memory: per-head state machine over block ids ---- */
typedef struct orc_mem orc_mem;
/* capacity_c in blocks, window capacity in chunks */
orc_mem* orc_mem_create(int64_t capacity_c, int64_t window_chunks);
void orc_mem_destroy(orc_mem* m);
/* append chunk (ids strictly increasing), evict oldest chunk on overflow.
 * The first chunk ever pushed is the sink chunk.  evicted: caller buffer of
 * capacity max_evicted; *n_evicted set. */
int orc_mem_push_chunk(orc_mem* m, const int64_t* ids, int64_t n, int64_t* evicted,
                       int64_t max_evicted, int64_t* n_evicted);
/* SPEC.md:200-208 (+ :226-228): sinks among the evicted join S; dynamic <- Top-(C-|S|) of
 * (dynamic U evicted non-sinks) by (score desc, id asc) with scores looked up in
 * (score_ids, scores) -- every candidate must be present (missing -> error). */
int orc_mem_update_persistent(orc_mem* m, const int64_t* evicted, int64_t n_evicted,
                              const int64_t* score_ids, const float* scores, int64_t n_scores);
/* SPEC.md:209-217 order: sinks (id asc), dynamic (id asc), local chunks in order.
 * region: 0 persistent, 1 local.  Returns counts; arrays sized by caller (cap). */
int orc_mem_assemble(const orc_mem* m, int64_t* ids, int32_t* region, int64_t cap, int64_t* n_p,
                     int64_t* n_l);
/* dynamic set in its type-invariant order (score desc, id asc) with stored scores */
int orc_mem_dynamic(const orc_mem* m, int64_t* ids, float* scores, int64_t cap, int64_t* n);
int64_t orc_mem_num_sinks(const orc_mem* m);
/* stand-alone Top-C op (SPEC.md:200-208 examples): candidates (ids, scores, is_sink flags);
 * keeps every sink; dynamic = Top-(C-|sinks|) by (score desc, id asc).  Writes kept flags. */
int orc_topc_select(const int64_t* ids, const float* scores, const uint8_t* is_sink, int64_t n,
                    int64_t capacity_c, uint8_t* kept);

#ifdef __cplusplus
}
#endif
