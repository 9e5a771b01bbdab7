// capi.cu -- the C ABI (include/pbsa_b200.h): argument checking, error reporting, TMA
// descriptor encoding, the device-resident memory object and the per-call orchestration.
#include <atomic>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

namespace pbsa {

namespace {
thread_local std::string g_err;
}

const char* last_error() { return g_err.c_str(); }

int set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int ensure_smem(const void* kernel, size_t bytes, const char* what) {
    if (bytes <= 48 * 1024) return PBSA_OK;
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = done[kernel];
    if (bytes <= cur) return PBSA_OK;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(PBSA_EUNSUPPORTED, std::string(what) + ": " + std::to_string(bytes) +
                                                " bytes of shared memory refused (" + cudaGetErrorString(e) + ")");
    }
    cur = bytes;
    return PBSA_OK;
}

namespace {
std::atomic<long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(PBSA_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return PBSA_OK;
}

namespace {
bool encode_tmap_impl(void* tmap, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                      const uint32_t* box, bool swizzle128, std::string* err) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (fn == nullptr) {
        *err = "cuTensorMapEncodeTiled unavailable";
        return false;
    }
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) {
        gd[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) gs[i] = strides[i];
    }
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                          static_cast<cuuint32_t>(rank), const_cast<void*>(base), gd, gs, bx, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        *err = "cuTensorMapEncodeTiled failed (CUresult " + std::to_string(static_cast<int>(r)) + ")";
        return false;
    }
    return true;
}
}  // namespace

bool pdl_enabled() {
    static const bool on = !(getenv("PBSA_PDL") && atoi(getenv("PBSA_PDL")) == 0);
    return on;
}

bool encode_tmap_bf16(void* tmap, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                      const uint32_t* box, std::string* err) {
    return encode_tmap_impl(tmap, base, rank, dims, strides, box, true, err);
}

bool encode_latent_tmap(void* tmap, const void* base, const LatentGeom& g, int box_d, bool swizzle128,
                        std::string* err) {
    const uint64_t row = static_cast<uint64_t>(g.heads) * g.d;
    const uint64_t dims[5] = {row, static_cast<uint64_t>(g.W), static_cast<uint64_t>(g.H),
                              static_cast<uint64_t>(g.T), static_cast<uint64_t>(g.batch)};
    const uint64_t strides[4] = {row * 2, row * 2 * g.W, row * 2 * g.W * g.H, row * 2 * g.W * g.H * g.T};
    const uint32_t box[5] = {static_cast<uint32_t>(box_d), static_cast<uint32_t>(g.bw), static_cast<uint32_t>(g.bh),
                             static_cast<uint32_t>(g.bt), 1u};
    return encode_tmap_impl(tmap, base, 5, dims, strides, box, swizzle128, err);
}

}  // namespace pbsa

using namespace pbsa;

#define PBSA_REQUIRE(cond, msg)                                  \
    do {                                                         \
        if (!(cond)) return ::pbsa::set_error(PBSA_EINVAL, msg); \
    } while (0)

#define PBSA_CUDA(call)                                                                          \
    do {                                                                                         \
        const cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) return ::pbsa::set_error(PBSA_ECUDA, std::string(#call ": ") +    \
                                                                     cudaGetErrorString(e_));    \
    } while (0)

struct pbsa_mem {
    int units = 0, C = 0, W = 0, bpc = 0, b = 0, d = 0, S = 0, Lcap = 0;
    MemCounts counts{};
    bf16* k_pool = nullptr;
    bf16* v_pool = nullptr;
    float* krep = nullptr;
    MemDev dev{};
    float* qc = nullptr;
    float* s_t = nullptr;
    float* ws = nullptr;
    size_t ws_bytes = 0;
    int32_t* sel = nullptr;
    int32_t* tile_pairs = nullptr;  // [units][(bpc + 1) / 2][2]: K3 tiles of the last call (pairs_valid)
    bool pairs_valid = false;
    void* k3ws = nullptr;
    size_t k3ws_bytes = 0;
    int last_k = 0, last_n_keys = 0, last_sel_rows = 0;
    // stage profiling: 5 events per attend call, 2 per KV write
    std::vector<cudaEvent_t> ev_attend, ev_write;
    int prof_max = 0, prof_attend = 0, prof_write = 0;
    bool prof_on = false;
    // host-resident chunks (pbsa_attend_qkv_host): two device staging sets {q, k, v, o}, an upload
    // and a download stream, and per set: uploaded / computed / downloaded events
    bf16* hstage[2][4] = {};
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t ev_up[2] = {}, ev_done[2] = {}, ev_down[2] = {};
    long long host_calls = 0;
};

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_d(int d) {
    if (d != 64 && d != 128) return set_error(PBSA_EUNSUPPORTED, "head dim d must be 64 or 128, got " + std::to_string(d));
    return PBSA_OK;
}

void free_events(pbsa_mem* m) {
    for (cudaEvent_t e : m->ev_attend) cudaEventDestroy(e);
    for (cudaEvent_t e : m->ev_write) cudaEventDestroy(e);
    m->ev_attend.clear();
    m->ev_write.clear();
    m->prof_on = false;
    m->prof_max = m->prof_attend = m->prof_write = 0;
}

// record event i of the current attend call's group (no-op when profiling is off or full)
void prof_mark(pbsa_mem* m, int i, cudaStream_t s) {
    if (!m->prof_on || m->prof_attend >= m->prof_max) return;
    cudaEventRecord(m->ev_attend[static_cast<size_t>(m->prof_attend) * 5 + i], s);
}

void free_host_path(pbsa_mem* m) {
    for (auto& set : m->hstage)
        for (bf16*& p : set)
            if (p) {
                cudaFree(p);
                p = nullptr;
            }
    for (int i = 0; i < 2; ++i)
        for (cudaEvent_t* e : {&m->ev_up[i], &m->ev_done[i], &m->ev_down[i]})
            if (*e) {
                cudaEventDestroy(*e);
                *e = nullptr;
            }
    for (cudaStream_t* st : {&m->up, &m->down})
        if (*st) {
            cudaStreamDestroy(*st);
            *st = nullptr;
        }
}

void free_mem(pbsa_mem* m) {
    free_host_path(m);
    free_events(m);
    void* ptrs[] = {m->k_pool, m->v_pool, m->krep, m->dev.p_slot, m->dev.p_id, m->dev.p_score,
                    m->dev.l_slot, m->dev.l_id, m->dev.stage, m->dev.free_slot, m->dev.dense,
                    m->dev.keys, m->qc, m->s_t, m->ws, m->sel, m->tile_pairs, m->k3ws, m->dev.status};
    for (void* p : ptrs)
        if (p) cudaFree(p);
}

// K3 tiles pair query blocks by Top-K overlap (launch_pair_tiles) for windows of >= 1024 blocks,
// where K3 dominates the call: config 5 chunk 692 -> 667 ms; at config 2 (312 blocks) the pairing
// kernel costs about what K3 gains.  PBSA_TILE_PAIRING=0 never pairs, 1 always (tests, A/B).
bool use_tile_pairing(int n_local) {
    const char* e = getenv("PBSA_TILE_PAIRING");
    if (e != nullptr) return atoi(e) != 0;
    return n_local >= 1024;
}

// K3 runs the hybrid schedule (whole-tile waves + stream-K tail) by default;
// PBSA_STREAM_K=0 selects whole tiles only (perf experiments).
bool use_stream_k() {
    static const bool on = !(getenv("PBSA_STREAM_K") && atoi(getenv("PBSA_STREAM_K")) == 0);
    return on;
}

MemCounts next_counts(const pbsa_mem* m, const MemCounts& c, int* dropped) {
    MemCounts n = c;
    n.chunk = c.chunk + 1;
    *dropped = 0;
    if (c.n_l + m->bpc > m->Lcap) {
        const int64_t evicted_chunk = c.chunk - m->W;
        if (evicted_chunk == 0) {
            n.n_sinks = m->bpc;
            n.n_p = m->bpc + (c.n_p - c.n_sinks);
        } else {
            const int n_cand = (c.n_p - c.n_sinks) + m->bpc;
            const int cap = m->C - c.n_sinks;
            const int keep = n_cand < cap ? n_cand : cap;
            n.n_p = c.n_sinks + keep;
            *dropped = n_cand - keep;
        }
        n.n_l = c.n_l;
    } else {
        n.n_l = c.n_l + m->bpc;
    }
    n.n_free = c.n_free + *dropped - m->bpc;
    return n;
}

}  // namespace

extern "C" {

const char* pbsa_last_error(void) { return last_error(); }

int pbsa_version(void) { return 1; }

int pbsa_compress(const void* x, int64_t x_unit_stride, int64_t x_block_stride, const int32_t* map,
                  int n_blocks, int units, int b, int d, float* reps, int64_t reps_unit_stride,
                  void* stream) {
    if (int rc = check_d(d)) return rc;
    PBSA_REQUIRE(n_blocks >= 0 && units >= 0, "compress: negative counts");
    PBSA_REQUIRE(b >= 1, "compress: block size b must be >= 1");
    PBSA_REQUIRE(x != nullptr && reps != nullptr, "compress: null pointer");
    PBSA_REQUIRE(aligned16(x) && x_unit_stride % 8 == 0 && x_block_stride % 8 == 0,
                 "compress: x and its strides must be 16-byte aligned");
    return launch_compress(static_cast<const bf16*>(x), x_unit_stride, x_block_stride, map, n_blocks,
                           units, b, d, reps, reps_unit_stride, as_stream(stream));
}

size_t pbsa_score_select_workspace(int units, int nqb, int n_keys) {
    return score_select_workspace(units, nqb, n_keys);
}

int pbsa_score_select(const float* qc, const float* krep, int64_t krep_unit_stride,
                      const int32_t* key_slots, int key_stride, int n_keys, int local_off,
                      int n_local, int k, int nqb, int units, int d, float scale, int32_t* sel,
                      float* s_t, void* workspace, size_t workspace_bytes, void* stream) {
    if (int rc = check_d(d)) return rc;
    PBSA_REQUIRE(n_keys >= 0 && nqb >= 0 && units >= 0 && k >= 0, "score_select: negative counts");
    PBSA_REQUIRE(local_off >= 0 && n_local >= 0 && local_off + n_local <= n_keys,
                 "score_select: local window outside the key list");
    PBSA_REQUIRE(k <= n_local, "score_select: k exceeds the number of local blocks");
    PBSA_REQUIRE(k == 0 || sel != nullptr, "score_select: sel is null");
    PBSA_REQUIRE(s_t == nullptr || n_keys >= 1, "score_select: s_t requested with no keys");
    PBSA_REQUIRE(key_stride >= n_keys, "score_select: key_stride < n_keys");
    PBSA_REQUIRE(aligned16(krep) && krep_unit_stride % 4 == 0, "score_select: krep must be 16-byte aligned");
    if (!(scale > 0.0f)) scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
    return launch_score_select(qc, krep, krep_unit_stride, key_slots, key_stride, n_keys, local_off,
                               n_local, k, nqb, units, d, scale, sel, s_t, workspace, workspace_bytes,
                               as_stream(stream));
}

int pbsa_matmul(const float* a, const float* b, int n, int k_dim, int m, int b_transposed, float scale, float* c,
                void* stream) {
    PBSA_REQUIRE(n >= 0 && k_dim >= 0 && m >= 0, "matmul: negative dims");
    PBSA_REQUIRE((n == 0 || m == 0) || (c != nullptr && (k_dim == 0 || (a != nullptr && b != nullptr))),
                 "matmul: null pointer");
    return launch_matmul_f64acc(a, b, n, k_dim, m, b_transposed ? 1 : 0, scale, c, as_stream(stream));
}

int pbsa_masked_softmax_rows(const float* scores, const float* mask, int rows, int cols, float* out, int* status,
                             void* stream) {
    PBSA_REQUIRE(rows >= 0 && cols >= 0, "masked_softmax_rows: negative dims");
    PBSA_REQUIRE(rows == 0 || cols == 0 || (scores != nullptr && out != nullptr), "masked_softmax_rows: null pointer");
    if (cols == 0) return PBSA_OK;
    return launch_softmax_rows(scores, mask, rows, cols, out, status, as_stream(stream));
}

int pbsa_aggregate_scores(const float* a, int rows, int cols, float* s, void* stream) {
    PBSA_REQUIRE(rows >= 1, "aggregate_scores: no rows");
    PBSA_REQUIRE(cols >= 0, "aggregate_scores: negative dims");
    PBSA_REQUIRE(cols == 0 || (a != nullptr && s != nullptr), "aggregate_scores: null pointer");
    return launch_aggregate_scores(a, rows, cols, 1, s, as_stream(stream));
}

int pbsa_compress_f32(const float* x, int n_blocks, int b, int d, float* reps, void* stream) {
    PBSA_REQUIRE(n_blocks >= 0 && d >= 0, "compress_blocks: negative counts");
    PBSA_REQUIRE(b >= 1, "compress_blocks: block size b must be >= 1");
    PBSA_REQUIRE(n_blocks == 0 || d == 0 || (x != nullptr && reps != nullptr), "compress_blocks: null pointer");
    if (n_blocks == 0 || d == 0) return PBSA_OK;
    return launch_aggregate_scores(x, b, d, n_blocks, reps, as_stream(stream));
}

size_t pbsa_select_topk_workspace(int rows, int cols) {
    if (rows < 0 || cols < 0) return 0;
    return static_cast<size_t>(rows) * cols * 4 + 16;
}

int pbsa_select_topk(const float* a, int rows, int cols, int k, int32_t* sel, void* workspace, size_t workspace_bytes,
                     int* status, void* stream) {
    PBSA_REQUIRE(rows >= 0 && cols >= 1, "select_topk: empty local region");
    PBSA_REQUIRE(k >= 1 && k <= cols, "select_topk: k must be in [1, cols]");
    PBSA_REQUIRE(rows == 0 || (a != nullptr && sel != nullptr && workspace != nullptr), "select_topk: null pointer");
    PBSA_REQUIRE(workspace_bytes >= pbsa_select_topk_workspace(rows, cols), "select_topk: workspace too small");
    return launch_select_topk(a, rows, cols, k, sel, static_cast<uint32_t*>(workspace), status, as_stream(stream));
}

int pbsa_blockify(const float* x, int t, int h, int w, int d, int b_t, int b_h, int b_w, float* y, int inverse,
                  void* stream) {
    PBSA_REQUIRE(t >= 0 && h >= 0 && w >= 0 && d >= 0, "blockify: negative dims");
    PBSA_REQUIRE(b_t >= 1 && b_h >= 1 && b_w >= 1, "block shape extents must be >= 1");
    PBSA_REQUIRE(t % b_t == 0, "axis t (" + std::to_string(t) + ") not divisible by b_t (" + std::to_string(b_t) + ")");
    PBSA_REQUIRE(h % b_h == 0, "axis h (" + std::to_string(h) + ") not divisible by b_h (" + std::to_string(b_h) + ")");
    PBSA_REQUIRE(w % b_w == 0, "axis w (" + std::to_string(w) + ") not divisible by b_w (" + std::to_string(b_w) + ")");
    const int64_t n = static_cast<int64_t>(t) * h * w * d;
    PBSA_REQUIRE(n == 0 || (x != nullptr && y != nullptr), "blockify: null pointer");
    PBSA_REQUIRE(static_cast<int64_t>(t) * h * w < (int64_t(1) << 31), "blockify: too many tokens");
    return launch_blockify(x, t, h, w, d, b_t, b_h, b_w, y, inverse ? 1 : 0, as_stream(stream));
}

int pbsa_topc_select(const int64_t* ids, const float* scores, int n, int slots, uint8_t* keep, int* status,
                     void* stream) {
    PBSA_REQUIRE(n >= 0 && slots >= 0, "update_persistent: negative counts");
    PBSA_REQUIRE(n == 0 || (ids != nullptr && scores != nullptr && keep != nullptr), "update_persistent: null pointer");
    return launch_topc_keep(ids, scores, n, slots, keep, status, as_stream(stream));
}

int pbsa_pair_tiles(const int32_t* sel, int sel_rows, int sel_row0, int nq, int k, int n_local, int units,
                    int32_t* pairs, void* stream) {
    PBSA_REQUIRE(units >= 0 && nq >= 0 && k >= 0 && n_local >= 0, "pair_tiles: negative sizes");
    PBSA_REQUIRE(sel_row0 >= 0 && sel_row0 + nq <= sel_rows, "pair_tiles: rows out of range");
    PBSA_REQUIRE(units == 0 || nq == 0 || (sel != nullptr && pairs != nullptr), "pair_tiles: null pointer");
    return launch_pair_tiles(sel, sel_rows, sel_row0, nq, k, n_local, units, pairs, as_stream(stream));
}

int pbsa_dev_alloc(void** out, size_t bytes) {
    PBSA_REQUIRE(out != nullptr, "dev_alloc: null output");
    *out = nullptr;
    PBSA_CUDA(cudaMalloc(out, bytes ? bytes : 1));
    return PBSA_OK;
}

int pbsa_dev_free(void* p) {
    if (p) PBSA_CUDA(cudaFree(p));
    return PBSA_OK;
}

int pbsa_stream_sync(void* stream) {
    PBSA_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return PBSA_OK;
}

int pbsa_bsa_fwd_last_plan(pbsa_bsa_plan* out) {
    PBSA_REQUIRE(out != nullptr, "bsa_fwd_last_plan: null output");
    *out = last_bsa_plan();
    return PBSA_OK;
}

size_t pbsa_bsa_fwd_workspace(int units, int nqb, int d) {
    if (units < 0 || nqb < 0 || (d != 64 && d != 128)) return 0;
    return bsa_fwd_workspace(units, nqb, d);
}

size_t pbsa_bsa_bwd_workspace(int units, int nqb, int b, int n_local) {
    if (units < 0 || nqb < 0 || b < 1 || b > 64 || n_local < 0) return 0;
    return bsa_bwd_workspace(units, nqb, b, n_local);
}

int pbsa_bsa_bwd(const void* q, const void* k_pool, const void* v_pool, int n_slots,
                 const int32_t* dense_slots, int dense_stride, int n_dense,
                 const int32_t* local_slots, int local_stride, int n_local, const int32_t* sel,
                 int k, int nqb, int b, int d, int units, float scale, const void* o, const void* d_o,
                 const float* lse, float* dq, float* dk_pool, float* dv_pool, void* workspace,
                 size_t workspace_bytes, void* stream) {
    if (int rc = check_d(d)) return rc;
    PBSA_REQUIRE(b >= 1 && b <= 64, "bsa_bwd: block size b must be in [1, 64]");
    PBSA_REQUIRE(nqb >= 0 && units >= 0 && n_slots >= 1, "bsa_bwd: bad counts");
    PBSA_REQUIRE(n_dense >= 0 && n_local >= 0 && k >= 0 && k <= n_local, "bsa_bwd: bad visibility counts");
    PBSA_REQUIRE(n_dense == 0 || (dense_slots != nullptr && dense_stride >= n_dense), "bsa_bwd: dense list");
    PBSA_REQUIRE(k == 0 || (local_slots != nullptr && sel != nullptr && local_stride >= n_local),
                 "bsa_bwd: local list / selection");
    PBSA_REQUIRE(static_cast<int64_t>(units) * n_slots * 64 < (int64_t(1) << 31), "bsa_bwd: pool too large for 32-bit TMA rows");
    PBSA_REQUIRE(q && k_pool && v_pool && o && d_o && lse && dq && dk_pool && dv_pool && workspace,
                 "bsa_bwd: null pointer");
    PBSA_REQUIRE(aligned16(q) && aligned16(k_pool) && aligned16(v_pool) && aligned16(o) && aligned16(d_o) &&
                     aligned16(dq) && aligned16(dk_pool) && aligned16(dv_pool) && aligned16(workspace),
                 "bsa_bwd: tensors must be 16-byte aligned");
    if (!(scale > 0.0f)) scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
    return launch_bsa_bwd(static_cast<const bf16*>(q), static_cast<const bf16*>(k_pool), static_cast<const bf16*>(v_pool),
                          n_slots, dense_slots, dense_stride, n_dense, local_slots, local_stride, n_local, sel, k, nqb,
                          b, d, units, scale, static_cast<const bf16*>(o), static_cast<const bf16*>(d_o), lse, dq,
                          dk_pool, dv_pool, workspace, workspace_bytes, as_stream(stream));
}

int pbsa_bsa_fwd(const void* q, const void* k_pool, const void* v_pool, int n_slots,
                 const int32_t* dense_slots, int dense_stride, int n_dense,
                 const int32_t* local_slots, int local_stride, int n_local, const int32_t* sel,
                 int k, int nqb, int b, int d, int units, float scale, void* o, float* lse,
                 void* workspace, size_t workspace_bytes, void* stream) {
    if (int rc = check_d(d)) return rc;
    PBSA_REQUIRE(b >= 1 && b <= 64, "bsa_fwd: block size b must be in [1, 64]");
    PBSA_REQUIRE(nqb >= 0 && units >= 0 && n_slots >= 1, "bsa_fwd: bad counts");
    PBSA_REQUIRE(n_dense >= 0 && n_local >= 0 && k >= 0 && k <= n_local, "bsa_fwd: bad visibility counts");
    PBSA_REQUIRE(n_dense == 0 || (dense_slots != nullptr && dense_stride >= n_dense), "bsa_fwd: dense list");
    PBSA_REQUIRE(k == 0 || (local_slots != nullptr && sel != nullptr && local_stride >= n_local),
                 "bsa_fwd: local list / selection");
    PBSA_REQUIRE(n_slots < (1 << 24) / 64, "bsa_fwd: too many slots per unit");
    PBSA_REQUIRE(static_cast<int64_t>(units) * n_slots * 64 < (int64_t(1) << 31), "bsa_fwd: pool too large for 32-bit TMA rows");
    PBSA_REQUIRE(static_cast<int64_t>(units) * nqb < (int64_t(1) << 31), "bsa_fwd: too many query blocks");
    PBSA_REQUIRE(q && k_pool && v_pool && o, "bsa_fwd: null pointer");
    PBSA_REQUIRE(aligned16(q) && aligned16(k_pool) && aligned16(v_pool) && aligned16(o),
                 "bsa_fwd: tensors must be 16-byte aligned");
    if (!(scale > 0.0f)) scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
    return launch_bsa_fwd(static_cast<const bf16*>(q), static_cast<const bf16*>(k_pool),
                          static_cast<const bf16*>(v_pool), n_slots, dense_slots, dense_stride, n_dense,
                          local_slots, local_stride, n_local, sel, k, nqb, b, d, units, scale,
                          static_cast<bf16*>(o), lse, workspace, workspace_bytes, as_stream(stream));
}

int pbsa_copy(void* dst, const void* src, size_t bytes, void* stream) {
    PBSA_REQUIRE(bytes == 0 || (dst != nullptr && src != nullptr), "copy: null pointer");
    if (bytes) PBSA_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
    return PBSA_OK;
}

int pbsa_debug_set_fault(const char* name) {
    if (name == nullptr || name[0] == '\0') {
        g_fault.store(0);
        return PBSA_OK;
    }
    if (std::string(name) == "drop-sink") {
        g_fault.store(kFaultDropSink);
        return PBSA_OK;
    }
    return set_error(PBSA_EINVAL, std::string("debug_set_fault: unknown fault '") + name + "'");
}

int pbsa_debug_tile(const void* q, const void* k, const void* v, int d, float* s_out, float* o_out,
                    void* stream) {
    if (int rc = check_d(d)) return rc;
    PBSA_REQUIRE(q && k && v && s_out && o_out, "debug_tile: null pointer");
    return launch_debug_tile(static_cast<const bf16*>(q), static_cast<const bf16*>(k),
                             static_cast<const bf16*>(v), d, s_out, o_out, as_stream(stream));
}

int pbsa_mem_create(pbsa_mem** out, int units, int capacity_c, int window_chunks,
                    int blocks_per_chunk, int b, int d) {
    PBSA_REQUIRE(out != nullptr, "mem_create: out is null");
    *out = nullptr;
    if (int rc = check_d(d)) return rc;
    PBSA_REQUIRE(units >= 1, "mem_create: units must be >= 1");
    PBSA_REQUIRE(blocks_per_chunk >= 1, "mem_create: blocks_per_chunk must be >= 1");
    PBSA_REQUIRE(window_chunks >= 1, "mem_create: window capacity must be >= 1 chunk");
    PBSA_REQUIRE(capacity_c >= blocks_per_chunk,
                 "mem_create: persistent capacity C must hold the sink chunk (C >= blocks_per_chunk)");
    PBSA_REQUIRE(b >= 1 && b <= 64, "mem_create: block size b must be in [1, 64]");
    auto* m = new pbsa_mem;
    m->units = units;
    m->C = capacity_c;
    m->W = window_chunks;
    m->bpc = blocks_per_chunk;
    m->b = b;
    m->d = d;
    m->Lcap = window_chunks * blocks_per_chunk;
    m->S = capacity_c + m->Lcap + blocks_per_chunk;
    const size_t U = static_cast<size_t>(units), S = m->S, C = m->C, L = m->Lcap, bpc = m->bpc;
    auto alloc = [&](void** p, size_t bytes) -> bool { return cudaMalloc(p, bytes ? bytes : 16) == cudaSuccess; };
    bool ok = alloc(reinterpret_cast<void**>(&m->k_pool), U * S * 64 * d * 2) &&
              alloc(reinterpret_cast<void**>(&m->v_pool), U * S * 64 * d * 2) &&
              alloc(reinterpret_cast<void**>(&m->krep), U * S * d * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.p_slot), U * C * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.p_id), U * C * 8) &&
              alloc(reinterpret_cast<void**>(&m->dev.p_score), U * C * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.l_slot), U * L * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.l_id), U * L * 8) &&
              alloc(reinterpret_cast<void**>(&m->dev.stage), U * bpc * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.free_slot), U * S * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.dense), U * (C + bpc) * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.keys), U * S * 4) &&
              alloc(reinterpret_cast<void**>(&m->dev.status), 16) &&
              alloc(reinterpret_cast<void**>(&m->qc), U * bpc * d * 4) &&
              alloc(reinterpret_cast<void**>(&m->s_t), U * S * 4) &&
              alloc(reinterpret_cast<void**>(&m->sel), U * bpc * L * 4) &&
              alloc(reinterpret_cast<void**>(&m->tile_pairs), U * ((bpc + 1) / 2) * 2 * 4);
    if (ok) {
        m->ws_bytes = score_select_workspace(units, m->bpc, m->S);
        m->k3ws_bytes = bsa_fwd_workspace(units, m->bpc, d);
        ok = alloc(reinterpret_cast<void**>(&m->ws), m->ws_bytes) && alloc(&m->k3ws, m->k3ws_bytes) &&
             cudaMemset(m->k3ws, 0, m->k3ws_bytes) == cudaSuccess;
    }
    if (!ok) {
        free_mem(m);
        delete m;
        cudaGetLastError();
        return set_error(PBSA_ECUDA, "mem_create: out of device memory");
    }
    if (int rc = pbsa_mem_reset(m, nullptr)) {
        free_mem(m);
        delete m;
        return rc;
    }
    PBSA_CUDA(cudaStreamSynchronize(nullptr));
    *out = m;
    return PBSA_OK;
}

int pbsa_mem_destroy(pbsa_mem* m) {
    if (m == nullptr) return PBSA_OK;
    cudaDeviceSynchronize();
    free_mem(m);
    delete m;
    return PBSA_OK;
}

int pbsa_mem_reset(pbsa_mem* m, void* stream) {
    PBSA_REQUIRE(m != nullptr, "mem_reset: null memory");
    cudaStream_t s = as_stream(stream);
    const size_t U = m->units, S = m->S;
    PBSA_CUDA(cudaMemsetAsync(m->k_pool, 0, U * S * 64 * m->d * 2, s));
    PBSA_CUDA(cudaMemsetAsync(m->v_pool, 0, U * S * 64 * m->d * 2, s));
    PBSA_CUDA(cudaMemsetAsync(m->krep, 0, U * S * m->d * 4, s));
    m->counts = MemCounts{0, 0, 0, m->S - m->bpc, 0};
    m->last_k = 0;
    m->last_n_keys = 0;
    return launch_mem_init(m->dev, m->units, m->C, m->Lcap, m->bpc, m->S, s);
}

int pbsa_mem_get_info(const pbsa_mem* m, pbsa_mem_info* info) {
    PBSA_REQUIRE(m != nullptr && info != nullptr, "mem_get_info: null pointer");
    std::memset(info, 0, sizeof(*info));
    info->units = m->units;
    info->capacity_c = m->C;
    info->window_chunks = m->W;
    info->blocks_per_chunk = m->bpc;
    info->b = m->b;
    info->d = m->d;
    info->n_slots = m->S;
    info->n_p = m->counts.n_p;
    info->n_sinks = m->counts.n_sinks;
    info->n_l = m->counts.n_l;
    info->chunks_committed = m->counts.chunk;
    info->k_pool = m->k_pool;
    info->v_pool = m->v_pool;
    info->krep = m->krep;
    info->dense_slots = m->dev.dense;
    info->local_slots = m->dev.l_slot;
    info->key_slots = m->dev.keys;
    info->stage_slots = m->dev.stage;
    info->p_ids = m->dev.p_id;
    info->p_scores = m->dev.p_score;
    info->l_ids = m->dev.l_id;
    info->dense_stride = m->C + m->bpc;
    info->local_stride = m->Lcap;
    info->key_stride = m->S;
    return PBSA_OK;
}

int pbsa_mem_write_chunk(pbsa_mem* m, const void* k_chunk, const void* v_chunk, void* stream) {
    PBSA_REQUIRE(m != nullptr && k_chunk != nullptr && v_chunk != nullptr, "mem_write_chunk: null pointer");
    PBSA_REQUIRE(aligned16(k_chunk) && aligned16(v_chunk), "mem_write_chunk: chunk must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    const bool prof = m->prof_on && m->prof_write < m->prof_max;
    if (prof) cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2], s);
    const int rc = launch_write_chunk(static_cast<const bf16*>(k_chunk), static_cast<const bf16*>(v_chunk),
                                      nullptr, m->dev.stage, m->bpc, m->b, m->d, m->units, m->S, m->k_pool,
                                      m->v_pool, m->krep, nullptr, s);
    if (prof) {
        cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2 + 1], s);
        ++m->prof_write;
    }
    return rc;
}

int pbsa_mem_profile(pbsa_mem* m, int enable, int max_calls) {
    PBSA_REQUIRE(m != nullptr, "mem_profile: null memory");
    free_events(m);
    if (!enable) return PBSA_OK;
    PBSA_REQUIRE(max_calls >= 1, "mem_profile: max_calls must be >= 1");
    m->ev_attend.resize(static_cast<size_t>(max_calls) * 5);
    m->ev_write.resize(static_cast<size_t>(max_calls) * 2);
    for (auto& e : m->ev_attend) PBSA_CUDA(cudaEventCreate(&e));
    for (auto& e : m->ev_write) PBSA_CUDA(cudaEventCreate(&e));
    m->prof_max = max_calls;
    m->prof_on = true;
    return PBSA_OK;
}

int pbsa_mem_profile_read(pbsa_mem* m, double* stage_ms, int* n_attend, int* n_write) {
    PBSA_REQUIRE(m != nullptr && stage_ms != nullptr, "mem_profile_read: null pointer");
    for (int i = 0; i < 5; ++i) stage_ms[i] = 0.0;
    if (n_attend) *n_attend = m->prof_attend;
    if (n_write) *n_write = m->prof_write;
    if (!m->prof_on) return PBSA_OK;
    for (int c = 0; c < m->prof_write; ++c) {
        float ms = 0.0f;
        PBSA_CUDA(cudaEventSynchronize(m->ev_write[static_cast<size_t>(c) * 2 + 1]));
        PBSA_CUDA(cudaEventElapsedTime(&ms, m->ev_write[static_cast<size_t>(c) * 2], m->ev_write[static_cast<size_t>(c) * 2 + 1]));
        stage_ms[0] += ms;
    }
    for (int c = 0; c < m->prof_attend; ++c) {
        cudaEvent_t* e = &m->ev_attend[static_cast<size_t>(c) * 5];
        PBSA_CUDA(cudaEventSynchronize(e[4]));
        for (int i = 0; i < 4; ++i) {
            float ms = 0.0f;
            PBSA_CUDA(cudaEventElapsedTime(&ms, e[i], e[i + 1]));
            stage_ms[1 + i] += ms;
        }
    }
    return PBSA_OK;
}

int pbsa_mem_commit(pbsa_mem* m, const float* s_t, void* stream) {
    PBSA_REQUIRE(m != nullptr && s_t != nullptr, "mem_commit: null pointer");
    int dropped = 0;
    const MemCounts nxt = next_counts(m, m->counts, &dropped);
    PBSA_REQUIRE(nxt.n_free >= 0, "mem_commit: slot pool exhausted (internal geometry error)");
    const int rc = launch_mem_commit(m->dev, s_t, m->units, m->C, m->Lcap, m->bpc, m->S, m->counts, nxt,
                                     as_stream(stream));
    if (rc == PBSA_OK) m->counts = nxt;
    return rc;
}

}  // extern "C"

namespace {

// The query blocks a call attends for: all of the chunk (begin 0, count bpc), or -- the query-split
// multi-GPU layout -- the range [begin, begin + count) with `qc_full` holding the caller-gathered
// representatives of ALL bpc query blocks (needed by the k=0 pass's s_t).
struct QueryPart {
    int begin = 0, count = -1;
    const float* qc_full = nullptr;
};

int attend_impl(pbsa_mem* m, const void* q, int k_top, float scale, int mode, void* o, float* lse, void* stream,
                bool q_compressed, const LatentGeom* lat, QueryPart part = QueryPart{}) {
    PBSA_REQUIRE(m != nullptr && q != nullptr && o != nullptr, "attend: null pointer");
    PBSA_REQUIRE(mode == PBSA_MODE_DENOISE || mode == PBSA_MODE_CACHE_UPDATE, "attend: unknown mode");
    PBSA_REQUIRE(k_top >= 0, "attend: k_top must be >= 0");
    PBSA_REQUIRE(aligned16(q) && aligned16(o), "attend: q / o must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    if (!(scale > 0.0f)) scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(m->d)));
    const int U = m->units, bpc = m->bpc, b = m->b, d = m->d;
    const int n_p = m->counts.n_p, n_l = m->counts.n_l;
    const int k = n_l == 0 ? 0 : (k_top < n_l ? k_top : n_l);
    const bool split = part.count >= 0;
    const int nq = split ? part.count : bpc;  // query blocks of this call
    prof_mark(m, 0, s);
    // (a) query-block representatives (already produced by the fused ingest in pbsa_attend_qkv; in
    //     the split form the caller's qc_full, whose own rows pbsa_attend_part_ingest wrote)
    if (!q_compressed) {
        if (int rc = launch_compress(static_cast<const bf16*>(q), static_cast<int64_t>(bpc) * b * d,
                                     static_cast<int64_t>(b) * d, nullptr, bpc, U, b, d, m->qc,
                                     static_cast<int64_t>(bpc) * d, s))
            return rc;
    }
    prof_mark(m, 1, s);
    // (b) coarse scoring + Top-K (+ s_t over P ++ L ++ current at the k=0 pass)
    const bool update = mode == PBSA_MODE_CACHE_UPDATE;
    int sel_rows = bpc, sel_row0 = 0;
    if (update) {
        // the k=0 pass always scores every query block of the chunk (s_t is their mean), so the
        // replicas of a query-split head all commit the same update
        const int n_keys = n_p + n_l + bpc;
        if (int rc = launch_score_select(split ? part.qc_full : m->qc, m->krep, static_cast<int64_t>(m->S) * d,
                                         m->dev.keys, m->S, n_keys, n_p, n_l, k, bpc, U, d, scale, m->sel, m->s_t,
                                         m->ws, m->ws_bytes, s, m->dev.status))
            return rc;
        m->last_n_keys = n_keys;
        sel_row0 = split ? part.begin : 0;
    } else if (k > 0) {
        // (split form: this rank's rows of qc_full, read in place)
        if (int rc = launch_score_select(split ? part.qc_full : m->qc, m->krep, static_cast<int64_t>(m->S) * d,
                                         m->dev.l_slot, m->Lcap, n_l, 0, n_l, k, nq, U, d, scale, m->sel, nullptr,
                                         m->ws, m->ws_bytes, s, m->dev.status, split ? bpc : 0,
                                         split ? part.begin : 0))
            return rc;
        sel_rows = nq;
    }
    m->last_k = k;
    m->last_sel_rows = sel_rows;
    // K3 tiles: query blocks paired by largest Top-K overlap (shorter union lists; results are per
    // query block and do not depend on the partner), natural pairs when there is no selection
    m->pairs_valid = false;
    if (k > 0 && use_tile_pairing(n_l)) {
        const int rc = launch_pair_tiles(m->sel, sel_rows, sel_row0, nq, k, n_l, U, m->tile_pairs, s);
        if (rc == PBSA_OK) m->pairs_valid = true;
        else if (rc != PBSA_EUNSUPPORTED) return rc;  // unsupported shape: natural pairing
    }
    prof_mark(m, 2, s);
    // (c) block-sparse attention over P ++ current (dense) and the selected local blocks
    if (int rc = launch_bsa_fwd(static_cast<const bf16*>(q), m->k_pool, m->v_pool, m->S, m->dev.dense,
                                m->C + bpc, n_p + bpc, m->dev.l_slot, m->Lcap, n_l, m->sel, k, nq, b, d, U,
                                scale, static_cast<bf16*>(o), lse, use_stream_k() ? m->k3ws : nullptr,
                                m->k3ws_bytes, s, lat, sel_rows, sel_row0, m->pairs_valid ? m->tile_pairs : nullptr))
        return rc;
    prof_mark(m, 3, s);
    // (d) persistent-memory update after the k=0 pass
    int rc = PBSA_OK;
    if (update) rc = pbsa_mem_commit(m, m->s_t, stream);
    prof_mark(m, 4, s);
    if (m->prof_on && m->prof_attend < m->prof_max) ++m->prof_attend;
    return rc;
}

}  // namespace

extern "C" {

int pbsa_attend(pbsa_mem* m, const void* q, int k_top, float scale, int mode, void* o, float* lse,
                void* stream) {
    return attend_impl(m, q, k_top, scale, mode, o, lse, stream, false, nullptr);
}

int pbsa_latent_blocks(const pbsa_latent_geom* g, int* blocks_per_chunk, int* block_tokens) {
    PBSA_REQUIRE(g != nullptr, "latent_blocks: null geometry");
    PBSA_REQUIRE(g->batch >= 1 && g->t >= 1 && g->h >= 1 && g->w >= 1 && g->heads >= 1,
                 "latent_blocks: latent dimensions must be positive");
    PBSA_REQUIRE(g->block_t >= 1 && g->block_h >= 1 && g->block_w >= 1, "make_block_layout: block extents must be positive");
    // blockify.cpp:7-36: every axis must divide exactly (no padding)
    if (g->t % g->block_t != 0)
        return set_error(PBSA_EINVAL, "make_block_layout: T (" + std::to_string(g->t) + ") not divisible by B_t (" +
                                          std::to_string(g->block_t) + ")");
    if (g->h % g->block_h != 0)
        return set_error(PBSA_EINVAL, "make_block_layout: H (" + std::to_string(g->h) + ") not divisible by B_h (" +
                                          std::to_string(g->block_h) + ")");
    if (g->w % g->block_w != 0)
        return set_error(PBSA_EINVAL, "make_block_layout: W (" + std::to_string(g->w) + ") not divisible by B_w (" +
                                          std::to_string(g->block_w) + ")");
    PBSA_REQUIRE(g->head_dim == 64 || g->head_dim == 128, "latent_blocks: head_dim must be 64 or 128");
    const int b = g->block_t * g->block_h * g->block_w;
    PBSA_REQUIRE(b <= 64, "latent_blocks: a block holds at most 64 tokens (one pool slot)");
    PBSA_REQUIRE(g->block_t <= 256 && g->block_h <= 256 && g->block_w <= 256, "latent_blocks: block extent > 256");
    if (blocks_per_chunk) *blocks_per_chunk = (g->t / g->block_t) * (g->h / g->block_h) * (g->w / g->block_w);
    if (block_tokens) *block_tokens = b;
    return PBSA_OK;
}

int pbsa_attend_latent(pbsa_mem* m, const void* q, const void* k_lat, const void* v_lat,
                       const pbsa_latent_geom* g, int k_top, float scale, int mode, void* o, float* lse,
                       void* stream) {
    PBSA_REQUIRE(m != nullptr && q != nullptr && k_lat != nullptr && v_lat != nullptr && o != nullptr,
                 "attend_latent: null pointer");
    int nqb = 0, b = 0;
    if (int rc = pbsa_latent_blocks(g, &nqb, &b)) return rc;
    PBSA_REQUIRE(g->batch * g->heads == m->units, "attend_latent: batch * heads != memory units");
    PBSA_REQUIRE(g->head_dim == m->d, "attend_latent: head_dim != memory head_dim");
    PBSA_REQUIRE(b == m->b, "attend_latent: block tokens != memory block size");
    PBSA_REQUIRE(nqb == m->bpc, "attend_latent: blocks per chunk != memory blocks_per_chunk");
    PBSA_REQUIRE(aligned16(q) && aligned16(k_lat) && aligned16(v_lat) && aligned16(o),
                 "attend_latent: tensors must be 16-byte aligned");
    const LatentGeom lg{g->batch, g->t, g->h, g->w, g->heads, g->head_dim, g->block_t, g->block_h, g->block_w};
    cudaStream_t s = as_stream(stream);
    const bool prof = m->prof_on && m->prof_write < m->prof_max;
    if (prof) cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2], s);
    if (int rc = launch_ingest_latent(static_cast<const bf16*>(k_lat), static_cast<const bf16*>(v_lat),
                                      static_cast<const bf16*>(q), lg, m->dev.stage, m->S, m->k_pool, m->v_pool,
                                      m->krep, m->qc, s))
        return rc;
    if (prof) {
        cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2 + 1], s);
        ++m->prof_write;
    }
    return attend_impl(m, q, k_top, scale, mode, o, lse, stream, true, &lg);
}

int pbsa_attend_qkv(pbsa_mem* m, const void* q, const void* k_chunk, const void* v_chunk, int k_top,
                    float scale, int mode, void* o, float* lse, void* stream) {
    PBSA_REQUIRE(m != nullptr && q != nullptr && k_chunk != nullptr && v_chunk != nullptr,
                 "attend_qkv: null pointer");
    PBSA_REQUIRE(aligned16(q) && aligned16(k_chunk) && aligned16(v_chunk), "attend_qkv: tensors must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    const bool prof = m->prof_on && m->prof_write < m->prof_max;
    if (prof) cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2], s);
    if (int rc = launch_write_chunk(static_cast<const bf16*>(k_chunk), static_cast<const bf16*>(v_chunk),
                                    static_cast<const bf16*>(q), m->dev.stage, m->bpc, m->b, m->d, m->units, m->S,
                                    m->k_pool, m->v_pool, m->krep, m->qc, s))
        return rc;
    if (prof) {
        cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2 + 1], s);
        ++m->prof_write;
    }
    return attend_impl(m, q, k_top, scale, mode, o, lse, stream, true, nullptr);
}

int pbsa_attend_part_ingest(pbsa_mem* m, const void* q_part, int q_begin, int q_count, const void* k_chunk,
                            const void* v_chunk, float* qc_full, void* stream) {
    PBSA_REQUIRE(m != nullptr && q_part != nullptr && k_chunk != nullptr && v_chunk != nullptr && qc_full != nullptr,
                 "attend_part_ingest: null pointer");
    PBSA_REQUIRE(q_begin >= 0 && q_count >= 1 && q_begin + q_count <= m->bpc,
                 "attend_part_ingest: query range outside the chunk's blocks");
    PBSA_REQUIRE(aligned16(q_part) && aligned16(k_chunk) && aligned16(v_chunk) && aligned16(qc_full),
                 "attend_part_ingest: tensors must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    const bool prof = m->prof_on && m->prof_write < m->prof_max;
    if (prof) cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2], s);
    // the whole chunk's K/V into the stage slots + K compression (replicated on every rank holding the
    // head), then the representatives of this rank's query blocks into their rows of qc_full
    // (one fused pass: the Q blocks of the range are compressed by the same CTAs)
    if (int rc = launch_write_chunk(static_cast<const bf16*>(k_chunk), static_cast<const bf16*>(v_chunk),
                                    static_cast<const bf16*>(q_part), m->dev.stage, m->bpc, m->b, m->d, m->units, m->S,
                                    m->k_pool, m->v_pool, m->krep, qc_full, s, q_begin, q_count))
        return rc;
    if (prof) {
        cudaEventRecord(m->ev_write[static_cast<size_t>(m->prof_write) * 2 + 1], s);
        ++m->prof_write;
    }
    return PBSA_OK;
}

int pbsa_attend_part(pbsa_mem* m, const void* q_part, int q_begin, int q_count, const float* qc_full, int k_top,
                     float scale, int mode, void* o_part, float* lse, void* stream) {
    PBSA_REQUIRE(m != nullptr && qc_full != nullptr, "attend_part: null pointer");
    PBSA_REQUIRE(q_begin >= 0 && q_count >= 1 && q_begin + q_count <= m->bpc,
                 "attend_part: query range outside the chunk's blocks");
    QueryPart part;
    part.begin = q_begin;
    part.count = q_count;
    part.qc_full = qc_full;
    return attend_impl(m, q_part, k_top, scale, mode, o_part, lse, stream, true, nullptr, part);
}

int pbsa_last_selection_rows(const pbsa_mem* m, int* rows) {
    PBSA_REQUIRE(m != nullptr && rows != nullptr, "last_selection_rows: null pointer");
    *rows = m->last_sel_rows;
    return PBSA_OK;
}

int pbsa_mem_host_reserve(pbsa_mem* m) {
    PBSA_REQUIRE(m != nullptr, "mem_host_reserve: null memory");
    if (m->up != nullptr) return PBSA_OK;
    const size_t bytes = static_cast<size_t>(m->units) * m->bpc * m->b * m->d * sizeof(bf16);
    {  // two staging sets {q, k, v, o}, the copy streams and their events
        bool ok = cudaStreamCreateWithFlags(&m->up, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&m->down, cudaStreamNonBlocking) == cudaSuccess;
        for (int i = 0; ok && i < 2; ++i) {
            for (int t = 0; ok && t < 4; ++t) ok = cudaMalloc(&m->hstage[i][t], bytes) == cudaSuccess;
            ok = ok && cudaEventCreateWithFlags(&m->ev_up[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&m->ev_done[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&m->ev_down[i], cudaEventDisableTiming) == cudaSuccess;
        }
        if (!ok) {
            free_host_path(m);
            cudaGetLastError();
            return set_error(PBSA_ECUDA, "mem_host_reserve: staging allocation failed");
        }
    }
    return PBSA_OK;
}

int pbsa_attend_qkv_host(pbsa_mem* m, const void* q_host, const void* k_host, const void* v_host, int k_top,
                         float scale, int mode, void* o_host, void* stream) {
    PBSA_REQUIRE(m != nullptr && q_host != nullptr && k_host != nullptr && v_host != nullptr && o_host != nullptr,
                 "attend_qkv_host: null pointer");
    cudaStream_t s = as_stream(stream);
    const size_t bytes = static_cast<size_t>(m->units) * m->bpc * m->b * m->d * sizeof(bf16);
    if (int rc = pbsa_mem_host_reserve(m)) return rc;  // no-op once reserved
    const int b = static_cast<int>(m->host_calls & 1);
    bf16* const* st = m->hstage[b];
    if (m->host_calls >= 2) {  // set b was last used two calls ago
        PBSA_CUDA(cudaStreamWaitEvent(m->up, m->ev_done[b], 0));  // its inputs are consumed
        PBSA_CUDA(cudaStreamWaitEvent(s, m->ev_down[b], 0));      // its output has been read back
    }
    PBSA_CUDA(cudaMemcpyAsync(st[0], q_host, bytes, cudaMemcpyHostToDevice, m->up));
    PBSA_CUDA(cudaMemcpyAsync(st[1], k_host, bytes, cudaMemcpyHostToDevice, m->up));
    PBSA_CUDA(cudaMemcpyAsync(st[2], v_host, bytes, cudaMemcpyHostToDevice, m->up));
    PBSA_CUDA(cudaEventRecord(m->ev_up[b], m->up));
    PBSA_CUDA(cudaStreamWaitEvent(s, m->ev_up[b], 0));
    if (int rc = pbsa_attend_qkv(m, st[0], st[1], st[2], k_top, scale, mode, st[3], nullptr, stream)) return rc;
    PBSA_CUDA(cudaEventRecord(m->ev_done[b], s));
    PBSA_CUDA(cudaStreamWaitEvent(m->down, m->ev_done[b], 0));
    PBSA_CUDA(cudaMemcpyAsync(o_host, st[3], bytes, cudaMemcpyDeviceToHost, m->down));
    PBSA_CUDA(cudaEventRecord(m->ev_down[b], m->down));
    ++m->host_calls;
    return PBSA_OK;
}

long long pbsa_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int pbsa_mem_host_sync(pbsa_mem* m) {
    PBSA_REQUIRE(m != nullptr, "mem_host_sync: null memory");
    if (m->up) PBSA_CUDA(cudaStreamSynchronize(m->up));
    if (m->down) PBSA_CUDA(cudaStreamSynchronize(m->down));
    return PBSA_OK;
}

int pbsa_mem_status(const pbsa_mem* m, int* flags, void* stream) {
    PBSA_REQUIRE(m != nullptr && flags != nullptr, "mem_status: null pointer");
    PBSA_CUDA(cudaMemcpyAsync(flags, m->dev.status, sizeof(int), cudaMemcpyDeviceToHost, as_stream(stream)));
    PBSA_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return PBSA_OK;
}

int pbsa_last_tile_pairs(const pbsa_mem* m, const int32_t** pairs, int* tiles_per_unit) {
    PBSA_REQUIRE(m != nullptr, "last_tile_pairs: null memory");
    if (pairs) *pairs = m->pairs_valid ? m->tile_pairs : nullptr;
    if (tiles_per_unit) *tiles_per_unit = (m->last_sel_rows + 1) / 2;
    return PBSA_OK;
}

int pbsa_last_selection(const pbsa_mem* m, const int32_t** sel, int* k, const float** s_t, int* n_keys) {
    PBSA_REQUIRE(m != nullptr, "last_selection: null memory");
    if (sel) *sel = m->sel;
    if (k) *k = m->last_k;
    if (s_t) *s_t = m->s_t;
    if (n_keys) *n_keys = m->last_n_keys;
    return PBSA_OK;
}

}  // extern "C"
