/*
 * pbsa_b200.h -- C ABI of the B200-native Persistent Block-Sparse Attention (PBSA) hot path.
 *
 * Drop-in boundary for the reference's operator API (/root/reference/SPEC.md modules router,
 * attention, memory; numeric conventions of /root/reference/proj/include/pbsa/tensor.hpp).  The
 * reference has no FFI; each entry point below names the reference op it replaces.  Plain
 * pointers and sizes only: device pointers unless stated, `stream` is a cudaStream_t passed as
 * void* (NULL = legacy default stream), bf16 tensors are passed as `const void*` / `void*`.
 *
 * Layouts (HBM):
 *   q / o        [units][n_q][d] bf16, n_q = nqb * b, query tokens block-major (blockify.hpp:32-46)
 *   k/v pool     [units][n_slots][64][d] bf16: one 64-row slot per key block, rows >= b are zero
 *   krep         [units][n_slots][d] f32: block representative of the block held in each slot
 *   qc           [units][nqb][d] f32
 *   slot lists   int32 slot indices per unit (stride given explicitly)
 *   sel          [units][nqb][k] int32: selected LOCAL block indices per query block, ascending
 * Every unit (= batch x head) is independent (per-head memory).
 *
 * Status codes: 0 ok, 1 invalid argument, 2 CUDA / launch error, 3 unsupported shape.  The
 * message of the last failure on the calling thread is returned by pbsa_last_error() (mirrors
 * the std::invalid_argument messages of tensor.cpp / blockify.cpp).  No entry point synchronizes
 * the stream.  Device memory is allocated only by pbsa_mem_create, pbsa_mem_host_reserve (the
 * host-chunk staging of one memory; pbsa_attend_qkv_host calls it on its first use) and
 * pbsa_dev_alloc; everything else takes caller-owned buffers and workspaces.
 */
#ifndef PBSA_B200_H
#define PBSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PBSA_OK = 0, PBSA_EINVAL = 1, PBSA_ECUDA = 2, PBSA_EUNSUPPORTED = 3 };

const char* pbsa_last_error(void);
int pbsa_version(void);

/* (a) block compression -- replaces router.compress_blocks (mean pooling,
 * PAPER.md:415), fp64 accumulation in ascending token order, fp32 output.
 * Block i of unit u is read at x + u*x_unit_stride + idx*x_block_stride (elements, bf16) and its
 * representative written to reps + u*reps_unit_stride + idx*d, idx = map ? map[u*n_blocks+i] : i. */
int pbsa_compress(const void* x, int64_t x_unit_stride, int64_t x_block_stride,
                  const int32_t* map, int n_blocks, int units, int b, int d, float* reps,
                  int64_t reps_unit_stride, void* stream);

/* (b) coarse scoring + row-wise Top-K -- replaces router.coarse_attention + select_topk
 * (+ aggregate_scores).
 * Keys of unit u are krep[u*krep_unit_stride + key_slots[u*key_stride + j]*d], j < n_keys.  The
 * local window is keys [local_off, local_off + n_local).  Per query block: logits
 * float(dot64(qc, kc)) * scale; A_L = masked_softmax_rows over the local keys (Eq. 10);
 * sel = k largest by (A_L desc, local index asc), written ascending.  If s_t != NULL (the k=0
 * cache-update pass) also A_t = softmax over all n_keys (Eq. 7) and s_t[u*n_keys + j] =
 * float(sum_i double(A_t[i][j]) / nqb) (Eq. 8).  k == 0 or n_local == 0 skips selection.
 * workspace: pbsa_score_select_workspace() bytes of device memory. */
size_t pbsa_score_select_workspace(int units, int nqb, int n_keys);
int pbsa_score_select(const float* qc, const float* krep, int64_t krep_unit_stride,
                      const int32_t* key_slots, int key_stride, int n_keys, int local_off,
                      int n_local, int k, int nqb, int units, int d, float scale, int32_t* sel,
                      float* s_t, void* workspace, size_t workspace_bytes, void* stream);

/* (c) block-sparse attention forward -- replaces attention.attention_sparse (SPEC.md:367-375,
 * Eq. 3-5).  Query block i of unit u attends to the dense slots
 * dense_slots[u*dense_stride + 0..n_dense) (persistent blocks + current chunk, always visible)
 * and to the selected local blocks local_slots[u*local_stride + sel[(u*nqb+i)*k + 0..k)].
 * Key rows >= b of a slot are masked.  o = softmax(q k^T * scale) v (bf16 out, fp32 softmax and
 * accumulators); lse (nullable) [units][n_q] natural-log row log-sum-exp.  d in {64, 128},
 * 1 <= b <= 64.  k_pool / v_pool: [units][n_slots][64][d].
 * workspace (nullable): pbsa_bsa_fwd_workspace() bytes, ZERO-INITIALISED ONCE by the caller (the
 * kernel leaves it zeroed); with it the launch is a persistent stream-K schedule (tiles split
 * across CTAs and merged), without it every CTA takes whole 128-row tiles. */
size_t pbsa_bsa_fwd_workspace(int units, int nqb, int d);
int pbsa_bsa_fwd(const void* q, const void* k_pool, const void* v_pool, int n_slots,
                 const int32_t* dense_slots, int dense_stride, int n_dense,
                 const int32_t* local_slots, int local_stride, int n_local, const int32_t* sel,
                 int k, int nqb, int b, int d, int units, float scale, void* o, float* lse,
                 void* workspace, size_t workspace_bytes, void* stream);

/* How the calling thread's last pbsa_bsa_fwd launch (direct or inside pbsa_attend*) was planned:
 * visible-list entry width (2 = 16-bit entries, used for long lists over pools < 16384 slots so two
 * CTAs still fit an SM), CTAs per SM, persistent grid, schedule and shared memory per CTA. */
enum { PBSA_SCHED_WHOLE_TILES = 0, PBSA_SCHED_STREAM_K = 1, PBSA_SCHED_UNIT_GANGS = 2 };
typedef struct pbsa_bsa_plan {
    int list_entry_bytes, ctas_per_sm, grid, schedule, gangs, max_list, n_tiles;
    size_t smem_bytes;
} pbsa_bsa_plan;
int pbsa_bsa_fwd_last_plan(pbsa_bsa_plan* out);

/* ---- the reference's tensor-module primitives and the SPEC router / memory ops on plain device
 * f32 row-major matrices (the drop-in C++ free functions of include/pbsa/tensor.hpp, blockify.hpp and
 * pbsa_b200.hpp run on these; the fused hot path above never does).  Bit-exact with the reference's
 * CPU code on the same inputs (fp64 accumulation in the reference's order). */
/* matmul (tensor.cpp:8-32, b_transposed = 0: b [k][m]) / matmul_nt (tensor.cpp:34-55, b_transposed = 1:
 * b [m][k]): c [n][m] = float(sum over ascending k of double(a[i][k]) * double(b(k, j))) * scale
 * (fp32 multiply; scale = 1 is the reference op, d^-1/2 the coarse logits of SPEC.md:281). */
int pbsa_matmul(const float* a, const float* b, int n, int k_dim, int m, int b_transposed, float scale, float* c,
                void* stream);
/* masked_softmax_rows (tensor.cpp:57-108): out [rows][cols]; mask (nullable) of 0 / -inf entries.
 * status (device int, nullable) gets bit 0 if scores hold a NaN and bit 1 if a mask entry is neither
 * 0 nor -inf -- the inputs the reference rejects with std::invalid_argument. */
int pbsa_masked_softmax_rows(const float* scores, const float* mask, int rows, int cols, float* out, int* status,
                             void* stream);
/* aggregate_scores: s[j] = float(sum over ascending i of double(a[i][j]) / rows). */
int pbsa_aggregate_scores(const float* a, int rows, int cols, float* s, void* stream);
/* compress_blocks on f32 blocks: x (n_blocks, b, d) -> reps (n_blocks, d), each the
 * mean of its b tokens with the same fp64 ascending-token sum as aggregate_scores (the hot path's K1,
 * pbsa_compress, is the bf16 form of the same op). */
int pbsa_compress_f32(const float* x, int n_blocks, int b, int d, float* reps, void* stream);
/* select_topk with an absolute k (1 <= k <= cols): sel [rows][k] = indices of the k
 * largest entries of each row by (value desc, index asc), ascending.  workspace:
 * pbsa_select_topk_workspace(rows, cols) bytes; status bit 0 = NaN in a. */
size_t pbsa_select_topk_workspace(int rows, int cols);
int pbsa_select_topk(const float* a, int rows, int cols, int k, int32_t* sel, void* workspace, size_t workspace_bytes,
                     int* status, void* stream);
/* blockify (blockify.cpp:38-65; inverse = 0): x (t, h, w, d) -> y (n_b, b, d) block-major; unblockify
 * (blockify.cpp:67-96; inverse = 1): x (n_b, b, d) -> y (t, h, w, d).  PBSA_EINVAL naming the axis when
 * (b_t, b_h, b_w) does not divide (t, h, w) (make_block_layout, blockify.cpp:7-36). */
int pbsa_blockify(const float* x, int t, int h, int w, int d, int b_t, int b_h, int b_w, float* y, int inverse,
                  void* stream);
/* update_persistent's ranking (Eq. 9): keep[i] = 1 for the `slots` best candidates by
 * (score desc, id asc), 0 otherwise (slots = C - |sinks|; sinks never compete).  status bit 0 = NaN score
 * (ranked lowest, as K4 does). */
int pbsa_topc_select(const int64_t* ids, const float* scores, int n, int slots, uint8_t* keep, int* status,
                     void* stream);
/* K3 tile pairing (scheduling, not a SPEC op; what pbsa_attend runs between K2 and K3): per unit, the
 * query blocks sel_row0 .. sel_row0 + nq - 1 of sel [units][sel_rows][k] (local indices < n_local) are
 * paired greedily by Top-K overlap (repeatedly the free pair with the largest overlap, ties to the lowest
 * i * nq + j), then partners swapped between the least-overlapping tile and another while both new
 * tiles overlap more; pairs [units][(nq + 1) / 2][2] lists each tile's query blocks (relative to
 * sel_row0), an odd leftover last with -1.  PBSA_EUNSUPPORTED when nq > 255, k > 32767 or the
 * bitsets exceed shared memory.  pbsa_attend pairs automatically for windows of >= 1024 blocks
 * (PBSA_TILE_PAIRING=0 never, =1 always). */
int pbsa_pair_tiles(const int32_t* sel, int sel_rows, int sel_row0, int nq, int k, int n_local, int units,
                    int32_t* pairs, void* stream);

/* Device memory for callers that hold no CUDA runtime of their own (the header-only C++ API):
 * cudaMalloc / cudaFree, cudaMemcpyAsync(cudaMemcpyDefault) and cudaStreamSynchronize. */
int pbsa_dev_alloc(void** out, size_t bytes);
int pbsa_dev_free(void* p);
int pbsa_stream_sync(void* stream);

/* (c') block-sparse attention backward -- the gradient of pbsa_bsa_fwd (the training path of
 * Alg. 2; the reference has no backward, the oracle is the derivative of
 * attention_sparse).  Inputs as pbsa_bsa_fwd plus the forward's o, its natural-log lse
 * [units][n_q] and the upstream gradient d_o [units][n_q][d] bf16.  Outputs f32: dq
 * [units][n_q][d]; dk_pool / dv_pool [units][n_slots][64][d] -- rows [0, b) of every slot in the
 * dense list or the local window are written (zero if no query block saw it), other slots are left
 * untouched.  workspace: pbsa_bsa_bwd_workspace() bytes (any contents). */
size_t pbsa_bsa_bwd_workspace(int units, int nqb, int b, int n_local);
int pbsa_bsa_bwd(const void* q, const void* k_pool, const void* v_pool, int n_slots,
                 const int32_t* dense_slots, int dense_stride, int n_dense,
                 const int32_t* local_slots, int local_stride, int n_local, const int32_t* sel,
                 int k, int nqb, int b, int d, int units, float scale, const void* o, const void* d_o,
                 const float* lse, float* dq, float* dk_pool, float* dv_pool, void* workspace,
                 size_t workspace_bytes, void* stream);

/* (d) persistent memory -- replaces memory.PersistentMemory / LocalWindow / push_chunk /
 * update_persistent / assemble_kv (Eq. 9).  Device-resident
 * state for `units` heads: the slot pools, representatives and the P / L / stage slot tables.
 * Capacities in blocks (C) and chunks (window); sinks = blocks of the first chunk,
 * counted inside C (requires capacity_c >= blocks_per_chunk).  Block ids are the monotone
 * stream index chunk*blocks_per_chunk + i. */
typedef struct pbsa_mem pbsa_mem;

typedef struct pbsa_mem_info {
    int units, capacity_c, window_chunks, blocks_per_chunk, b, d;
    int n_slots;          /* capacity_c + window_chunks*blocks_per_chunk + blocks_per_chunk */
    int n_p, n_sinks, n_l;  /* current persistent / sink / local block counts (same every unit) */
    int64_t chunks_committed;
    /* device views (valid until destroy) */
    void *k_pool, *v_pool;      /* [units][n_slots][64][d] bf16 */
    float* krep;                /* [units][n_slots][d] */
    int32_t* dense_slots;       /* [units][dense_stride]: P (sinks id asc, dynamic id asc) ++ stage */
    int32_t* local_slots;       /* [units][local_stride]: L chunks oldest -> newest */
    int32_t* key_slots;         /* [units][key_stride]: P ++ L ++ stage (the k=0 scoring order) */
    int32_t* stage_slots;       /* [units][blocks_per_chunk]: where the current chunk's K/V live */
    int64_t* p_ids;             /* [units][capacity_c] ids in dense order */
    float* p_scores;            /* [units][capacity_c] last s_t of each persistent block */
    int64_t* l_ids;             /* [units][local_stride] */
    int dense_stride, local_stride, key_stride;
} pbsa_mem_info;

int pbsa_mem_create(pbsa_mem** out, int units, int capacity_c, int window_chunks,
                    int blocks_per_chunk, int b, int d);
int pbsa_mem_destroy(pbsa_mem* m);
int pbsa_mem_reset(pbsa_mem* m, void* stream);
int pbsa_mem_get_info(const pbsa_mem* m, pbsa_mem_info* info);
/* Write the current chunk's K and V ([units][blocks_per_chunk*b][d] bf16, block-major) into the
 * stage slots and compress K into krep (fused (a)).  Called once per PBSA call. */
int pbsa_mem_write_chunk(pbsa_mem* m, const void* k_chunk, const void* v_chunk, void* stream);
/* K4: the k=0 cache update of Alg. 1.  s_t: [units][n_keys] scores in
 * key_slots order (from pbsa_score_select).  push_chunk(stage) -> evict oldest chunk on
 * overflow -> update_persistent -> refresh slot tables -> new stage slots. */
int pbsa_mem_commit(pbsa_mem* m, const float* s_t, void* stream);

/* One full PBSA call of a layer on the current chunk (Alg. 1 line "Apply PBSA with Top-K"):
 * K1(Q) -> K2 -> K3, and for mode PBSA_MODE_CACHE_UPDATE (the k=0 pass) also s_t and K4; for local
 * windows of >= 1024 blocks the K3 tile pairing (pbsa_pair_tiles) runs between K2 and K3.
 * q [units][blocks_per_chunk*b][d] bf16; o same shape; lse nullable.  k_top = |Omega(q)| in
 * blocks (clipped to the local window); scale <= 0 selects d^-1/2. */
enum { PBSA_MODE_DENOISE = 0, PBSA_MODE_CACHE_UPDATE = 1 };
int pbsa_attend(pbsa_mem* m, const void* q, int k_top, float scale, int mode, void* o,
                float* lse, void* stream);
/* Invalid-input status since the last reset (synchronises `stream`): bit 0 = NaN coarse logits
 * seen by K2, bit 1 = NaN scores seen by K4.  The reference rejects NaN scores
 * (tensor.cpp:61-64); the device path keeps a consistent state (NaN ranks lowest) and reports. */
int pbsa_mem_status(const pbsa_mem* m, int* flags, void* stream);
/* Fused form of pbsa_mem_write_chunk + pbsa_attend for a layer that has the current chunk's
 * Q, K and V ([units][blocks_per_chunk*b][d] bf16): one ingest pass writes K/V into the stage
 * slots and compresses K and Q (K1), then K2 -> K3 (-> K4) as pbsa_attend. */
int pbsa_attend_qkv(pbsa_mem* m, const void* q, const void* k_chunk, const void* v_chunk, int k_top,
                    float scale, int mode, void* o, float* lse, void* stream);
/* pbsa_attend_qkv for chunks that live in HOST memory (pinned or cudaHostRegister'ed, the
 * [units][blocks_per_chunk*b][d] bf16 layout of pbsa_attend_qkv): the Q/K/V upload runs on an
 * internal stream into one of two device staging sets, the compute on `stream`, and the download of
 * O into o_host on a second internal stream, so the upload of call i+1 and the download of call i-1
 * overlap the compute of call i.  Returns without waiting; q/k/v_host must stay unchanged and o_host
 * unread until pbsa_mem_host_sync returns (work later enqueued on `stream` is ordered after this
 * call's compute, not after its download). */
int pbsa_attend_qkv_host(pbsa_mem* m, const void* q_host, const void* k_host, const void* v_host, int k_top,
                         float scale, int mode, void* o_host, void* stream);
/* Allocates the host-chunk path of m up front (two device staging sets of 4 x units x n_q x d bf16,
 * two copy streams, events; freed by pbsa_mem_destroy).  Idempotent. */
int pbsa_mem_host_reserve(pbsa_mem* m);
/* Waits for every upload and download issued by pbsa_attend_qkv_host so far. */
int pbsa_mem_host_sync(pbsa_mem* m);
/* Number of kernels the library has launched since it was loaded (all entry points, all streams). */
long long pbsa_launch_count(void);
/* Chunk latents in the reference's Latent4D layout (proj/include/pbsa/tensor.hpp:30-47: (t, h, w, d)
 * row-major, d = heads * head_dim), one per batch element: [batch][T][H][W][heads*d]
 * bf16, blocked by blockify's (B_t, B_h, B_w) (proj/include/pbsa/blockify.hpp:11-67; block id
 * (nt*N_h + nh)*N_w + nw, in-block index (dt*B_h + dh)*B_w + dw).  Unit u = e*heads + h. */
typedef struct pbsa_latent_geom {
    int batch, t, h, w, heads, head_dim, block_t, block_h, block_w;
} pbsa_latent_geom;
/* Host-only validation (no device work): the make_block_layout checks of blockify.cpp:7-36
 * (non-divisible axis -> PBSA_EINVAL naming the axis) plus the library's limits; returns the
 * blocks per chunk and tokens per block. */
int pbsa_latent_blocks(const pbsa_latent_geom* g, int* blocks_per_chunk, int* block_tokens);
/* pbsa_attend_qkv on chunk latents: the ingest gathers each (head, block) with one 5-D TMA box
 * (blockify fused), K3 loads Q blocks the same way and writes O rows straight back to their latent
 * positions (unblockify fused).  q, k_lat, v_lat, o: [batch][T][H][W][heads*d] bf16 with
 * batch*heads == units, T*H*W == blocks_per_chunk * b of the memory; lse (nullable) stays
 * [units][n_q] in block order.  Results are bit-identical to pbsa_attend_qkv on the blockified
 * per-head tensors. */
int pbsa_attend_latent(pbsa_mem* m, const void* q, const void* k_lat, const void* v_lat,
                       const pbsa_latent_geom* g, int k_top, float scale, int mode, void* o, float* lse,
                       void* stream);

/* Query-split form of pbsa_attend_qkv for multi-GPU layouts whose units are fewer than the ranks
 * (batch-1 Wan shapes: 12 heads on 8 GPUs): every rank sharing a head holds a
 * replica of the head's memory and attends for the query blocks [q_begin, q_begin + q_count) of each
 * unit.  q_part / o_part: [units][q_count*b][d] bf16; k_chunk / v_chunk: the WHOLE chunk
 * [units][blocks_per_chunk*b][d] (the KV write is replicated); qc_full: caller-owned device
 * [units][blocks_per_chunk][d] f32.
 *   1. pbsa_attend_part_ingest: KV write + K compression, and this rank's query representatives into
 *      rows [q_begin, q_begin + q_count) of qc_full.
 *   2. in PBSA_MODE_CACHE_UPDATE the caller all-gathers qc_full across the replicas (s_t averages A_t
 *      over ALL query blocks; 40 KB per head at d = 128); denoise calls need only the own rows.
 *   3. pbsa_attend_part: Top-K of the own rows (the k=0 pass scores all rows, so every replica computes
 *      the same s_t and commits the identical P / L update), K3 for the own query blocks, K4.
 * Results are bit-identical to pbsa_attend_qkv on the whole chunk restricted to the part. */
int pbsa_attend_part_ingest(pbsa_mem* m, const void* q_part, int q_begin, int q_count, const void* k_chunk,
                            const void* v_chunk, float* qc_full, void* stream);
int pbsa_attend_part(pbsa_mem* m, const void* q_part, int q_begin, int q_count, const float* qc_full, int k_top,
                     float scale, int mode, void* o_part, float* lse, void* stream);

/* last selection of pbsa_attend (device): [units][rows][k] ascending (rows = blocks_per_chunk, or
 * q_count after a denoise pbsa_attend_part: see pbsa_last_selection_rows), and last s_t */
int pbsa_last_selection_rows(const pbsa_mem* m, int* rows);
int pbsa_last_selection(const pbsa_mem* m, const int32_t** sel, int* k, const float** s_t,
                        int* n_keys);
/* K3 tiles of the last attend call (device): [units][tiles_per_unit][2] query blocks of the call per
 * tile (second -1 when the tile has one), paired by largest Top-K overlap; *pairs = NULL when the
 * call used the natural pairs (2t, 2t + 1) (no selection, or PBSA_TILE_PAIRING=0).  Scheduling
 * only: the outputs do not depend on it. */
int pbsa_last_tile_pairs(const pbsa_mem* m, const int32_t** pairs, int* tiles_per_unit);

/* Stage timing with CUDA events recorded on the call's stream (no host sync inside calls).
 * enable: allocate a pool for max_calls calls and reset the sums; 0 disables.  read: waits for
 * the last recorded event and returns per-stage sums in ms: [0] KV write (+K compression),
 * [1] Q compression (a), [2] scoring + Top-K (b), [3] attention (c), [4] memory update (d),
 * and the number of attend calls / KV writes timed. */
int pbsa_mem_profile(pbsa_mem* m, int enable, int max_calls);
int pbsa_mem_profile_read(pbsa_mem* m, double* stage_ms, int* n_attend, int* n_write);

/* PBT1 tensor files (reference proj/include/pbsa/tensor.hpp:62-101, proj/src/tensor_io.cpp):
 * "PBT1" | dtype 0x01 (f32 LE) | rank u8 | rank x u64 LE dims | row-major payload.  Errors return
 * PBSA_EINVAL with a message that starts with the reference's TensorIoError::Kind name (OpenFailed,
 * BadMagic, BadDtype, Truncated, TrailingData, BadShape).  write / info / read are host-only;
 * load_bf16 streams the payload through pinned staging to the device and converts to bf16 there
 * (synchronises `stream` before returning; dst: device, 16-byte aligned, capacity in elements). */
int pbsa_pbt1_write(const char* path, const float* data, int rank, const uint64_t* dims);
int pbsa_pbt1_info(const char* path, int* rank, uint64_t* dims, int max_rank);
int pbsa_pbt1_read(const char* path, float* out, uint64_t capacity);
int pbsa_pbt1_load_bf16(const char* path, void* dst, uint64_t capacity, void* stream);

/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault) on `stream` (state export for tests) */
int pbsa_copy(void* dst, const void* src, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PBSA_B200_H */
