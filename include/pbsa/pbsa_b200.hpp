// pbsa/pbsa_b200.hpp -- the SPEC operator API of PBSA (/root/reference/SPEC.md modules memory,
// router, attention: SPEC.md:160-417) on the reference's value types, over the C ABI
// (include/pbsa_b200.h).  Header-only, plain C++20, no CUDA headers.  Every op keeps the SPEC name,
// signature and argument meaning; argument errors throw std::invalid_argument (the library's
// message), device failures std::runtime_error.
//
// It includes pbsa/tensor.hpp and pbsa/blockify.hpp: with this repo's include/ first those are the
// drop-in restatements (GPU-backed free functions); with the reference's proj/include first they are
// the reference's own headers (link its tensor.cpp / blockify.cpp / tensor_io.cpp), and everything
// below works on those types unchanged (tests/test_cpp_api.py builds both ways).
//
// Two layers:
//   * SPEC-shaped host ops (host containers in and out; each uploads, runs the sm_100a kernels,
//     downloads):
//       memory    BlockEntry, PersistentMemory, LocalWindow, EvictionBatch, push_chunk,
//                 update_persistent, assemble_kv
//       router    BlockRepresentatives, BlockScores, BlockMask, compress_blocks,
//                 coarse_attention, aggregate_scores, select_topk, build_mask
//       attention AttentionConfig, attention_reference, attention_sparse, flop_count SPEC.md:346-393
//       bench     kv_length, kv_bytes
//     coarse_attention / aggregate_scores / select_topk / update_persistent / attention_reference are
//     bit-exact with the reference's CPU arithmetic (fp32 storage, fp64 accumulation);
//     attention_sparse runs the bf16 tensor-core kernel K3 (inputs rounded to bf16 on upload;
//     within max-abs 2e-2 / mean-abs 2e-3 of the fp32 reference, BASELINE.json north_star).
//   * pbsa::Memory: the device-resident hot loop (slot pools + P/L state, K1-K4 fused), one PBSA
//     call per attend() on a caller stream, no host synchronisation.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "pbsa/b200_detail.hpp"
#include "pbsa/blockify.hpp"
#include "pbsa/tensor.hpp"
#include "pbsa_b200.h"

namespace pbsa {

// =============================================================================================
// router types
// =============================================================================================
struct BlockRepresentatives {
    std::size_t n_blocks = 0, d = 0;
    std::vector<float> data;  // n_blocks x d
};
struct BlockScores {
    std::vector<float> scores;  // one per key block, each in [0, 1], sum 1 +- 1e-5
};
struct BlockMask {
    std::size_t n_query_blocks = 0, n_persistent_blocks = 0, n_local_blocks = 0;
    std::vector<std::vector<int32_t>> visible;  // per query block: visible local block indices, ascending
};
// SPEC.md:346-350
struct AttentionConfig {
    std::size_t d = 128;
    std::size_t n_heads = 1;
    double scale = 0.0;  // <= 0 -> d^-1/2
};

// =============================================================================================
// memory types
// =============================================================================================
struct BlockEntry {
    int64_t id = 0;       // monotone stream index chunk * blocks_per_chunk + i
    DenseMatrix k, v;     // b x d
    float score = 0.0f;   // latest coarse relevance s_t
    bool is_sink = false;
};
struct PersistentMemory {
    std::size_t capacity_c = 0;       // blocks
    std::vector<BlockEntry> sinks;    // never removed once inserted
    std::vector<BlockEntry> dynamic;  // sorted by (score desc, id asc)
};
struct LocalWindow {
    std::size_t capacity_chunks = 0;
    std::vector<std::vector<BlockEntry>> chunks;  // FIFO, generation order
};
struct EvictionBatch {
    std::vector<BlockEntry> entries;
};
enum class Region { Persistent, Local };
struct AssembledKV {
    DenseMatrix k_cat, v_cat;                             // (N_p + N_l) x d
    std::vector<std::pair<Region, int64_t>> index_map;    // per block, in row order
};

namespace detail {
inline float attn_scale(std::size_t d, double scale) {
    return scale > 0.0 ? static_cast<float>(scale) : static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
}
inline int64_t max_id(const LocalWindow& w) {
    int64_t m = INT64_MIN;
    for (const auto& c : w.chunks)
        for (const auto& e : c) m = std::max(m, e.id);
    return m;
}
inline void check_entry(const BlockEntry& e, std::size_t b, std::size_t d, const char* op) {
    if (e.k.rows != e.v.rows || e.k.cols != e.v.cols) throw std::invalid_argument(std::string(op) + ": k and v shapes differ");
    if (e.k.rows != b || e.k.cols != d) throw std::invalid_argument(std::string(op) + ": dim mismatch");
}
}  // namespace detail

// k = max(1, ceil(N_l * ratio))
inline std::size_t topk_count(std::size_t n_local, double ratio) {
    if (n_local < 1) throw std::invalid_argument("select_topk: empty local region");
    if (!(ratio > 0.0 && ratio <= 1.0)) throw std::invalid_argument("select_topk: topk_ratio must be in (0,1]");
    const auto k = static_cast<std::size_t>(std::ceil(static_cast<double>(n_local) * ratio));
    return k < 1 ? 1 : (k > n_local ? n_local : k);
}

// =============================================================================================
// memory ops
// =============================================================================================

/// push_chunk: append; evict the oldest chunk whole when over capacity.  Host
/// bookkeeping (no arithmetic); the device form is K4 (pbsa_mem_commit).
inline EvictionBatch push_chunk(LocalWindow& window, std::vector<BlockEntry> chunk) {
    if (chunk.empty()) throw std::invalid_argument("push_chunk: empty chunk");
    int64_t last = detail::max_id(window);
    for (const auto& e : chunk) {
        if (e.id <= last) throw std::invalid_argument("push_chunk: block ids must be strictly increasing");
        last = e.id;
    }
    window.chunks.push_back(std::move(chunk));
    EvictionBatch ev;
    if (window.chunks.size() > window.capacity_chunks) {
        ev.entries = std::move(window.chunks.front());
        window.chunks.erase(window.chunks.begin());
    }
    return ev;
}

/// update_persistent (Eq. 9): sinks kept (evicted sink blocks join them); dynamic <-
/// Top-(C - |sinks|) of (dynamic U evicted) by (score desc, id asc) with every candidate's score
/// refreshed from `scores`.  The ranking runs on the GPU (pbsa_topc_select, the rule K4
/// applies in place).
inline PersistentMemory update_persistent(const PersistentMemory& p, const EvictionBatch& evicted,
                                          const std::unordered_map<int64_t, float>& scores) {
    PersistentMemory out;
    out.capacity_c = p.capacity_c;
    out.sinks = p.sinks;
    std::vector<const BlockEntry*> cand;
    for (const auto& e : p.dynamic) cand.push_back(&e);
    for (const auto& e : evicted.entries) {
        if (e.is_sink) out.sinks.push_back(e);
        else cand.push_back(&e);
    }
    for (auto& s : out.sinks) {
        auto it = scores.find(s.id);
        if (it != scores.end()) s.score = it->second;
    }
    if (out.sinks.size() > out.capacity_c) throw std::invalid_argument("update_persistent: sinks exceed capacity C");
    const std::size_t slots = out.capacity_c - out.sinks.size();
    std::vector<int64_t> ids(cand.size());
    std::vector<float> sc(cand.size());
    for (std::size_t i = 0; i < cand.size(); ++i) {
        auto it = scores.find(cand[i]->id);
        if (it == scores.end())
            throw std::invalid_argument("update_persistent: missing score for block " + std::to_string(cand[i]->id));
        ids[i] = cand[i]->id;
        sc[i] = it->second;
    }
    std::vector<uint8_t> keep(cand.size(), 0);
    if (!cand.empty()) {
        detail::DevBuf<int64_t> di(ids.size());
        detail::DevBuf<float> ds(sc.size());
        detail::DevBuf<uint8_t> dk(keep.size());
        di.upload(ids.data(), ids.size());
        ds.upload(sc.data(), sc.size());
        detail::check(pbsa_topc_select(di.p, ds.p, detail::to_int(cand.size(), "update_persistent"),
                                       detail::to_int(slots, "update_persistent"), dk.p, nullptr, nullptr));
        dk.download(keep.data(), keep.size());
    }
    for (std::size_t i = 0; i < cand.size(); ++i)
        if (keep[i]) {
            out.dynamic.push_back(*cand[i]);
            out.dynamic.back().score = sc[i];
        }
    std::sort(out.dynamic.begin(), out.dynamic.end(), [](const BlockEntry& a, const BlockEntry& b) {
        return a.score != b.score ? a.score > b.score : a.id < b.id;
    });
    return out;
}

/// assemble_kv: [sinks id asc; dynamic id asc; local chunks in order] token rows
/// plus the (region, block id) of every block.  A host concatenation; the device path never copies
/// (K3 reads the slot pool through index lists).
inline AssembledKV assemble_kv(const PersistentMemory& p, const LocalWindow& window) {
    std::vector<const BlockEntry*> sinks, dyn;
    for (const auto& e : p.sinks) sinks.push_back(&e);
    for (const auto& e : p.dynamic) dyn.push_back(&e);
    auto by_id = [](const BlockEntry* a, const BlockEntry* b) { return a->id < b->id; };
    std::sort(sinks.begin(), sinks.end(), by_id);
    std::sort(dyn.begin(), dyn.end(), by_id);
    std::vector<std::pair<Region, const BlockEntry*>> order;
    for (auto* e : sinks) order.emplace_back(Region::Persistent, e);
    for (auto* e : dyn) order.emplace_back(Region::Persistent, e);
    for (const auto& c : window.chunks)
        for (const auto& e : c) order.emplace_back(Region::Local, &e);
    AssembledKV out;
    std::size_t rows = 0, d = order.empty() ? 0 : order[0].second->k.cols;
    for (auto& [r, e] : order) {
        if (e->k.cols != d || e->v.cols != d || e->k.rows != e->v.rows)
            throw std::invalid_argument("assemble_kv: dim mismatch");
        rows += e->k.rows;
    }
    out.k_cat = DenseMatrix(rows, d);
    out.v_cat = DenseMatrix(rows, d);
    std::size_t r0 = 0;
    for (auto& [r, e] : order) {
        std::copy(e->k.data.begin(), e->k.data.end(), out.k_cat.data.begin() + r0 * d);
        std::copy(e->v.data.begin(), e->v.data.end(), out.v_cat.data.begin() + r0 * d);
        r0 += e->k.rows;
        out.index_map.emplace_back(r, e->id);
    }
    return out;
}

// =============================================================================================
// router ops
// =============================================================================================

/// compress_blocks: mean of each block's b tokens (fp64 ascending sum, one
/// division), on the GPU.  bf16 device inputs take the fused K1 instead (pbsa_compress / Memory).
inline BlockRepresentatives compress_blocks(const BlockedTensor& xb) {
    const std::size_t nb = xb.layout.n_b, b = xb.layout.b, d = xb.layout.d;
    if (xb.data.size() != nb * b * d) throw std::invalid_argument("compress_blocks: data length does not match layout");
    BlockRepresentatives out{nb, d, std::vector<float>(nb * d)};
    if (out.data.empty()) return out;
    detail::DevBuf<float> x(nb * b * d), reps(nb * d);
    x.upload(xb.data.data(), xb.data.size());
    detail::check(pbsa_compress_f32(x.p, detail::to_int(nb, "compress_blocks"), detail::to_int(b, "compress_blocks"),
                                    detail::to_int(d, "compress_blocks"), reps.p, nullptr));
    reps.download(out.data.data(), out.data.size());
    return out;
}

/// coarse_attention (Eq. 7): softmax_rows(float(qc . kc^T) * d^-1/2).
inline DenseMatrix coarse_attention(const BlockRepresentatives& qc, const BlockRepresentatives& kc, double scale = 0.0) {
    if (qc.d != kc.d) throw std::invalid_argument("coarse_attention: dim mismatch");
    const std::size_t nq = qc.n_blocks, nk = kc.n_blocks, d = qc.d;
    DenseMatrix a(nq, nk);
    if (nq == 0 || nk == 0) return a;
    detail::DevBuf<float> dq(nq * d), dk(nk * d), z(nq * nk), p(nq * nk);
    dq.upload(qc.data.data(), nq * d);
    dk.upload(kc.data.data(), nk * d);
    detail::check(pbsa_matmul(dq.p, dk.p, detail::to_int(nq, "coarse_attention"), detail::to_int(d, "coarse_attention"),
                              detail::to_int(nk, "coarse_attention"), 1, detail::attn_scale(d, scale), z.p, nullptr));
    detail::DevBuf<int> st(1);
    const int zero = 0;
    st.upload(&zero, 1);
    detail::check(pbsa_masked_softmax_rows(z.p, nullptr, static_cast<int>(nq), static_cast<int>(nk), p.p, st.p, nullptr));
    if (detail::read_status(st) & 1) throw std::invalid_argument("masked_softmax_rows: NaN in scores");
    p.download(a.data.data(), a.data.size());
    return a;
}

/// aggregate_scores (Eq. 8): s[j] = mean over rows of a[i][j].
inline BlockScores aggregate_scores(const DenseMatrix& a) {
    if (a.rows == 0) throw std::invalid_argument("aggregate_scores: no rows");
    BlockScores s;
    s.scores.resize(a.cols);
    if (a.cols == 0) return s;
    detail::DevBuf<float> da(a.data.size()), ds(a.cols);
    da.upload(a.data.data(), a.data.size());
    detail::check(pbsa_aggregate_scores(da.p, detail::to_int(a.rows, "aggregate_scores"),
                                        detail::to_int(a.cols, "aggregate_scores"), ds.p, nullptr));
    ds.download(s.scores.data(), a.cols);
    return s;
}

/// select_topk (Eq. 11): per row the k = max(1, ceil(N_l * ratio)) largest entries,
/// ties toward the lower index; visible sets ascending.
inline BlockMask select_topk(const DenseMatrix& a_local, double topk_ratio) {
    const std::size_t k = topk_count(a_local.cols, topk_ratio);
    BlockMask m;
    m.n_query_blocks = a_local.rows;
    m.n_local_blocks = a_local.cols;
    if (a_local.rows == 0) return m;
    const std::size_t ws = pbsa_select_topk_workspace(static_cast<int>(a_local.rows), static_cast<int>(a_local.cols));
    detail::DevBuf<float> da(a_local.data.size());
    detail::DevBuf<int32_t> sel(a_local.rows * k);
    detail::DevBuf<uint8_t> w(ws);
    detail::DevBuf<int> st(1);
    const int zero = 0;
    st.upload(&zero, 1);
    da.upload(a_local.data.data(), a_local.data.size());
    detail::check(pbsa_select_topk(da.p, detail::to_int(a_local.rows, "select_topk"), detail::to_int(a_local.cols, "select_topk"),
                                   static_cast<int>(k), sel.p, w.p, ws, st.p, nullptr));
    if (detail::read_status(st) & 1) throw std::invalid_argument("select_topk: NaN in scores");
    const auto h = sel.to_host();
    for (std::size_t i = 0; i < a_local.rows; ++i) m.visible.emplace_back(h.begin() + i * k, h.begin() + (i + 1) * k);
    return m;
}

/// build_mask (Eq. 5): the token-level additive mask [0 over the n_p_tokens
/// persistent columns | M_L], M_L = 0 where the local block is visible to the query token's block.
/// Oracle-only in this design: the GPU path consumes the index lists and never builds it; provided
/// for callers of the reference API (and attention_reference below).
inline DenseMatrix build_mask(const BlockMask& mask, std::size_t b, std::size_t n_p_tokens) {
    const std::size_t nl = mask.n_local_blocks, cols = n_p_tokens + nl * b;
    DenseMatrix m(mask.visible.size() * b, cols, -std::numeric_limits<float>::infinity());
    for (std::size_t i = 0; i < mask.visible.size(); ++i)
        for (std::size_t r = 0; r < b; ++r) {
            float* row = m.row(i * b + r);
            std::fill(row, row + n_p_tokens, 0.0f);
            for (int32_t l : mask.visible[i]) {
                if (l < 0 || static_cast<std::size_t>(l) >= nl) throw std::invalid_argument("build_mask: selected index out of range");
                std::fill(row + n_p_tokens + l * b, row + n_p_tokens + (l + 1) * b, 0.0f);
            }
        }
    return m;
}

/// Fused K2 (coarse_attention + select_topk (+ aggregate_scores) in one pass over device-resident
/// representatives): Top-k over the local window [local_off, local_off + n_local) of kc; s_t over all
/// keys when want_scores (the k=0 pass).  Bit-exact with the separate ops above.
struct Selection {
    BlockMask mask;
    BlockScores scores;
};

inline Selection score_select(const BlockRepresentatives& qc, const BlockRepresentatives& kc, std::size_t local_off,
                              std::size_t n_local, std::size_t k, bool want_scores, double scale = 0.0) {
    if (qc.d != kc.d) throw std::invalid_argument("coarse_attention: dim mismatch");
    const std::size_t nq = qc.n_blocks, nk = kc.n_blocks, d = qc.d;
    detail::DevBuf<float> dq(nq * d), dk(nk * d), dst(nk);
    detail::DevBuf<int32_t> keys(nk), sel(nq * (k ? k : 1));
    dq.upload(qc.data.data(), nq * d);
    dk.upload(kc.data.data(), nk * d);
    std::vector<int32_t> ident(nk);
    for (std::size_t i = 0; i < nk; ++i) ident[i] = static_cast<int32_t>(i);
    keys.upload(ident.data(), nk);
    const std::size_t ws_bytes = pbsa_score_select_workspace(1, static_cast<int>(nq), static_cast<int>(nk));
    detail::DevBuf<uint8_t> ws(ws_bytes);
    detail::check(pbsa_score_select(dq.p, dk.p, static_cast<int64_t>(nk * d), keys.p, static_cast<int>(nk),
                                    static_cast<int>(nk), static_cast<int>(local_off), static_cast<int>(n_local),
                                    static_cast<int>(k), static_cast<int>(nq), 1, static_cast<int>(d),
                                    static_cast<float>(scale), sel.p, want_scores ? dst.p : nullptr, ws.p, ws_bytes,
                                    nullptr));
    Selection out;
    out.mask.n_query_blocks = nq;
    out.mask.n_persistent_blocks = local_off;
    out.mask.n_local_blocks = n_local;
    std::vector<int32_t> h(nq * k);
    if (k) sel.download(h.data(), nq * k);
    for (std::size_t i = 0; i < nq; ++i) out.mask.visible.emplace_back(h.begin() + i * k, h.begin() + (i + 1) * k);
    if (want_scores) {
        out.scores.scores.resize(nk);
        dst.download(out.scores.scores.data(), nk);
    }
    return out;
}

// =============================================================================================
// attention ops
// =============================================================================================

/// attention_reference (Eq. 4): softmax(float(q . k^T) * scale + mask) . v, fully
/// dense -- the oracle the sparse path is checked against, composed of the bit-exact primitives
/// (matmul_nt, masked_softmax_rows, matmul) on the GPU.  mask: nullptr or N_q x N_kv of 0 / -inf.
inline DenseMatrix attention_reference(const DenseMatrix& q, const DenseMatrix& k_cat, const DenseMatrix& v_cat,
                                       const DenseMatrix* mask, const AttentionConfig& cfg) {
    if (q.cols != k_cat.cols || k_cat.rows != v_cat.rows || k_cat.rows == 0 || q.cols == 0)
        throw std::invalid_argument("attention_reference: shape mismatch");
    if (mask && (mask->rows != q.rows || mask->cols != k_cat.rows))
        throw std::invalid_argument("attention_reference: mask shape mismatch");
    const int nq = detail::to_int(q.rows, "attention_reference"), nkv = detail::to_int(k_cat.rows, "attention_reference");
    const int d = detail::to_int(q.cols, "attention_reference"), dv = detail::to_int(v_cat.cols, "attention_reference");
    DenseMatrix out(q.rows, v_cat.cols);
    if (nq == 0) return out;
    detail::DevBuf<float> dq(q.data.size()), dk(k_cat.data.size()), dvv(v_cat.data.size()), s(q.rows * k_cat.rows),
        p(q.rows * k_cat.rows), dm(mask ? mask->data.size() : 0), o(out.data.size());
    detail::DevBuf<int> st(1);
    const int zero = 0;
    st.upload(&zero, 1);
    dq.upload(q.data.data(), q.data.size());
    dk.upload(k_cat.data.data(), k_cat.data.size());
    dvv.upload(v_cat.data.data(), v_cat.data.size());
    if (mask) dm.upload(mask->data.data(), mask->data.size());
    detail::check(pbsa_matmul(dq.p, dk.p, nq, d, nkv, 1, detail::attn_scale(q.cols, cfg.scale), s.p, nullptr));
    detail::check(pbsa_masked_softmax_rows(s.p, mask ? dm.p : nullptr, nq, nkv, p.p, st.p, nullptr));
    const int flags = detail::read_status(st);
    if (flags & 1) throw std::invalid_argument("masked_softmax_rows: NaN in scores");
    if (flags & 2) throw std::invalid_argument("masked_softmax_rows: mask entries must be 0 or -inf");
    detail::check(pbsa_matmul(p.p, dvv.p, nq, nkv, dv, 0, 1.0f, o.p, nullptr));
    o.download(out.data.data(), out.data.size());
    return out;
}

namespace detail {
// K3 on host block stores: query block i sees the dense blocks and local_blocks[sel[i]]
inline DenseMatrix run_bsa(const BlockedTensor& q_blocks, const std::vector<const float*>& kb,
                           const std::vector<const float*>& vb, std::size_t b, std::size_t n_dense, std::size_t n_local,
                           const BlockMask& mask, const AttentionConfig& cfg) {
    const std::size_t nqb = q_blocks.layout.n_b, d = q_blocks.layout.d, ns = kb.size();
    if (q_blocks.layout.b != b) throw std::invalid_argument("attention_sparse: geometry inconsistency");
    if (cfg.d != d) throw std::invalid_argument("attention_sparse: AttentionConfig.d mismatch");
    if (q_blocks.data.size() != nqb * b * d) throw std::invalid_argument("attention_sparse: q_blocks data length");
    if (b < 1 || b > 64) throw std::invalid_argument("attention_sparse: block size b must be in [1, 64]");
    const std::size_t k = mask.visible.empty() ? 0 : mask.visible[0].size();
    if (n_local > 0 && !mask.visible.empty() && mask.visible.size() != nqb)
        throw std::invalid_argument("attention_sparse: mask rows != query blocks");
    std::vector<int32_t> sel;
    for (const auto& v : mask.visible) {
        if (v.size() != k) throw std::invalid_argument("attention_sparse: |visible(q)| must be identical across q");
        for (int32_t x : v) {
            if (x < 0 || static_cast<std::size_t>(x) >= n_local) throw std::invalid_argument("attention_sparse: visible index out of range");
            sel.push_back(x);
        }
    }
    if (n_local == 0) sel.clear();
    const std::size_t kk = n_local == 0 ? 0 : k;
    std::vector<uint16_t> kp(std::max<std::size_t>(ns, 1) * 64 * d, 0), vp(kp.size(), 0);
    for (std::size_t s = 0; s < ns; ++s)
        for (std::size_t r = 0; r < b * d; ++r) {
            kp[s * 64 * d + r] = to_bf16(kb[s][r]);
            vp[s * 64 * d + r] = to_bf16(vb[s][r]);
        }
    std::vector<int32_t> dense(n_dense), local(n_local);
    for (std::size_t i = 0; i < n_dense; ++i) dense[i] = static_cast<int32_t>(i);
    for (std::size_t i = 0; i < n_local; ++i) local[i] = static_cast<int32_t>(n_dense + i);
    DevBuf<uint16_t> dq(nqb * b * d), dk(kp.size()), dv(vp.size()), dout(nqb * b * d);
    DevBuf<int32_t> dd(n_dense), dl(n_local), ds(sel.size());
    dq.upload(bf16_of(q_blocks.data).data(), nqb * b * d);
    dk.upload(kp.data(), kp.size());
    dv.upload(vp.data(), vp.size());
    dd.upload(dense.data(), dense.size());
    dl.upload(local.data(), local.size());
    ds.upload(sel.data(), sel.size());
    check(pbsa_bsa_fwd(dq.p, dk.p, dv.p, static_cast<int>(std::max<std::size_t>(ns, 1)), n_dense ? dd.p : nullptr,
                       static_cast<int>(n_dense), static_cast<int>(n_dense), n_local ? dl.p : nullptr,
                       static_cast<int>(n_local), static_cast<int>(n_local), kk ? ds.p : nullptr, static_cast<int>(kk),
                       static_cast<int>(nqb), static_cast<int>(b), static_cast<int>(d), 1, static_cast<float>(cfg.scale),
                       dout.p, nullptr, nullptr, 0, nullptr));
    std::vector<uint16_t> h(nqb * b * d);
    dout.download(h.data(), h.size());
    DenseMatrix out(nqb * b, d);
    for (std::size_t i = 0; i < h.size(); ++i) out.data[i] = from_bf16(h[i]);
    return out;
}
}  // namespace detail

/// attention_sparse: query block i attends to every persistent block (always
/// visible, Eq. 5) and to the local blocks mask.visible[i] of the window (assemble_kv order), online
/// softmax over the visible blocks only -- K3 on the tensor cores.  Returns (N_q^blk * b) x d.
inline DenseMatrix attention_sparse(const BlockedTensor& q_blocks, const PersistentMemory& p, const LocalWindow& window,
                                    const BlockMask& mask, const AttentionConfig& cfg) {
    const std::size_t b = q_blocks.layout.b, d = q_blocks.layout.d;
    std::vector<const BlockEntry*> pers;
    for (const auto& e : p.sinks) pers.push_back(&e);
    std::vector<const BlockEntry*> dyn;
    for (const auto& e : p.dynamic) dyn.push_back(&e);
    auto by_id = [](const BlockEntry* a, const BlockEntry* b2) { return a->id < b2->id; };
    std::sort(pers.begin(), pers.end(), by_id);
    std::sort(dyn.begin(), dyn.end(), by_id);
    pers.insert(pers.end(), dyn.begin(), dyn.end());
    std::vector<const float*> kb, vb;
    for (auto* e : pers) {
        detail::check_entry(*e, b, d, "attention_sparse");
        kb.push_back(e->k.data.data());
        vb.push_back(e->v.data.data());
    }
    std::size_t n_local = 0;
    for (const auto& c : window.chunks)
        for (const auto& e : c) {
            detail::check_entry(e, b, d, "attention_sparse");
            kb.push_back(e.k.data.data());
            vb.push_back(e.v.data.data());
            ++n_local;
        }
    if (mask.n_local_blocks != 0 && mask.n_local_blocks != n_local)
        throw std::invalid_argument("attention_sparse: mask inconsistent with the window");
    return detail::run_bsa(q_blocks, kb, vb, b, pers.size(), n_local, mask, cfg);
}

/// attention_sparse on block stores (the same kernel, stores instead of memory structs): query
/// block i sees k/v_store blocks dense_blocks and local_blocks[mask.visible[i]].
inline DenseMatrix attention_sparse(const BlockedTensor& q_blocks, const BlockedTensor& k_store,
                                    const BlockedTensor& v_store, const std::vector<int32_t>& dense_blocks,
                                    const std::vector<int32_t>& local_blocks, const BlockMask& mask,
                                    const AttentionConfig& cfg) {
    const std::size_t b = q_blocks.layout.b, d = q_blocks.layout.d, ns = k_store.layout.n_b;
    if (k_store.layout.b != b || v_store.layout.b != b || k_store.layout.d != d || v_store.layout.n_b != ns)
        throw std::invalid_argument("attention_sparse: geometry inconsistency");
    std::vector<const float*> kb, vb;
    for (auto list : {&dense_blocks, &local_blocks})
        for (int32_t i : *list) {
            if (i < 0 || static_cast<std::size_t>(i) >= ns) throw std::invalid_argument("attention_sparse: block index out of range");
            kb.push_back(k_store.block(i));
            vb.push_back(v_store.block(i));
        }
    return detail::run_bsa(q_blocks, kb, vb, b, dense_blocks.size(), local_blocks.size(), mask, cfg);
}

/// flop_count: dense 4 N_q (N_p + N_l) d; sparse 4 N_q (N_p + k b) d plus the
/// coarse stage 4 (N_q / b)((N_p + N_l) / b) d; ratio dense / sparse.
struct FlopCount {
    double dense_flops = 0, sparse_flops = 0, ratio = 0;
};
inline FlopCount flop_count(std::size_t n_q, std::size_t n_p, std::size_t n_l, std::size_t b, std::size_t k_selected,
                            std::size_t d) {
    if (n_q == 0 || b == 0 || d == 0) throw std::invalid_argument("flop_count: non-positive geometry");
    FlopCount f;
    f.dense_flops = 4.0 * double(n_q) * double(n_p + n_l) * double(d);
    const double coarse = 4.0 * (double(n_q) / double(b)) * (double(n_p + n_l) / double(b)) * double(d);
    f.sparse_flops = 4.0 * double(n_q) * double(n_p + k_selected * b) * double(d) + coarse;
    f.ratio = f.dense_flops / f.sparse_flops;
    return f;
}

/// kv_length: N_KV = N_L + N_P, N_L = N_C * local_ratio, N_P = N_L * persist_ratio
/// (both must be integral).
inline std::size_t kv_length(std::size_t n_c, double local_ratio, double persist_ratio) {
    auto integral = [](double x, const char* what) {
        const double r = std::round(x);
        if (x < 0 || std::fabs(x - r) > 1e-9) throw std::invalid_argument(std::string("kv_length: ") + what + " not integral");
        return static_cast<std::size_t>(r);
    };
    if (n_c == 0 || local_ratio < 0 || persist_ratio < 0) throw std::invalid_argument("kv_length: bad geometry");
    const std::size_t n_l = integral(double(n_c) * local_ratio, "N_L");
    return n_l + integral(double(n_l) * persist_ratio, "N_P");
}

/// kv_bytes: 2 (K and V) * layers * tokens * heads * head_dim * bytes per element.
inline std::size_t kv_bytes(std::size_t tokens, std::size_t layers, std::size_t kv_heads, std::size_t head_dim,
                            std::size_t bpe) {
    return 2 * layers * tokens * kv_heads * head_dim * bpe;
}

// =============================================================================================
// pbsa::Memory -- the device-resident hot loop (SPEC.md:160-243 state + Alg. 1)
// =============================================================================================
class Memory {
public:
    Memory(int units, int capacity_c, int window_chunks, int blocks_per_chunk, int b, int d) {
        detail::check(pbsa_mem_create(&m_, units, capacity_c, window_chunks, blocks_per_chunk, b, d));
    }
    ~Memory() { pbsa_mem_destroy(m_); }
    Memory(const Memory&) = delete;
    Memory& operator=(const Memory&) = delete;

    pbsa_mem_info info() const {
        pbsa_mem_info i;
        detail::check(pbsa_mem_get_info(m_, &i));
        return i;
    }
    void reset(void* stream = nullptr) { detail::check(pbsa_mem_reset(m_, stream)); }
    // current chunk K/V: device [units][blocks_per_chunk*b][d] bf16
    void write_chunk(const void* k_chunk, const void* v_chunk, void* stream = nullptr) {
        detail::check(pbsa_mem_write_chunk(m_, k_chunk, v_chunk, stream));
    }
    // one PBSA call; mode PBSA_MODE_CACHE_UPDATE = the k=0 pass (scores + push/evict/Top-C)
    void attend(const void* q, int k_top, int mode, void* o, float* lse = nullptr, double scale = 0.0,
                void* stream = nullptr) {
        detail::check(pbsa_attend(m_, q, k_top, static_cast<float>(scale), mode, o, lse, stream));
    }
    // write_chunk + attend fused (one ingest pass over Q, K, V): device [units][bpc*b][d] bf16
    void attend_qkv(const void* q, const void* k, const void* v, int k_top, int mode, void* o, float* lse = nullptr,
                    double scale = 0.0, void* stream = nullptr) {
        detail::check(pbsa_attend_qkv(m_, q, k, v, k_top, static_cast<float>(scale), mode, o, lse, stream));
    }
    // attend_qkv on HOST chunks (pinned): upload / compute / download pipelined across calls;
    // o_host is valid after host_sync()
    void attend_qkv_host(const void* q, const void* k, const void* v, int k_top, int mode, void* o_host,
                         double scale = 0.0, void* stream = nullptr) {
        detail::check(pbsa_attend_qkv_host(m_, q, k, v, k_top, static_cast<float>(scale), mode, o_host, stream));
    }
    void host_sync() { detail::check(pbsa_mem_host_sync(m_)); }
    // the same on device chunk latents [batch][T][H][W][heads*d] bf16 (blockify / unblockify fused)
    void attend_latent(const void* q, const void* k, const void* v, const pbsa_latent_geom& g, int k_top, int mode,
                       void* o, float* lse = nullptr, double scale = 0.0, void* stream = nullptr) {
        detail::check(pbsa_attend_latent(m_, q, k, v, &g, k_top, static_cast<float>(scale), mode, o, lse, stream));
    }
    // host convenience on the reference's own types: one batch element's chunk as Latent4D (t, h, w,
    // heads*d) fp32 (rounded to bf16 on upload), blocked by `shape` like blockify; returns O as a
    // Latent4D of the same shape.  Synchronous (uploads, runs on the default stream, downloads).
    Latent4D attend_latent(const Latent4D& q, const Latent4D& k, const Latent4D& v, const BlockShape& shape, int heads,
                           int k_top, int mode, double scale = 0.0) {
        if (k.t != q.t || k.h != q.h || k.w != q.w || k.d != q.d || v.t != q.t || v.h != q.h || v.w != q.w || v.d != q.d)
            throw std::invalid_argument("attend_latent: q, k, v must have the same (t, h, w, d)");
        if (heads <= 0 || q.d % static_cast<std::size_t>(heads) != 0)
            throw std::invalid_argument("attend_latent: d is not a multiple of heads");
        pbsa_latent_geom g{1, static_cast<int>(q.t), static_cast<int>(q.h), static_cast<int>(q.w), heads,
                           static_cast<int>(q.d / heads), static_cast<int>(shape.b_t), static_cast<int>(shape.b_h),
                           static_cast<int>(shape.b_w)};
        detail::check(pbsa_latent_blocks(&g, nullptr, nullptr));
        detail::DevBuf<uint16_t> dq(q.size()), dk(q.size()), dv(q.size()), dout(q.size());
        const auto hq = detail::bf16_of(q.data), hk = detail::bf16_of(k.data), hv = detail::bf16_of(v.data);
        dq.upload(hq.data(), hq.size());
        dk.upload(hk.data(), hk.size());
        dv.upload(hv.data(), hv.size());
        attend_latent(dq.p, dk.p, dv.p, g, k_top, mode, dout.p, nullptr, scale, nullptr);
        const auto ho = dout.to_host();
        Latent4D out(q.t, q.h, q.w, q.d);
        for (std::size_t i = 0; i < ho.size(); ++i) out.data[i] = detail::from_bf16(ho[i]);
        return out;
    }
    void commit(const float* s_t, void* stream = nullptr) { detail::check(pbsa_mem_commit(m_, s_t, stream)); }
    // assemble_kv as block ids: persistent (sinks id asc, dynamic id asc), local
    void assemble(int unit, std::vector<int64_t>* persistent, std::vector<int64_t>* local) const {
        const pbsa_mem_info i = info();
        detail::check(pbsa_stream_sync(nullptr));
        persistent->resize(i.n_p);
        local->resize(i.n_l);
        if (i.n_p)
            detail::check(pbsa_copy(persistent->data(), i.p_ids + static_cast<std::size_t>(unit) * i.capacity_c,
                                    i.n_p * sizeof(int64_t), nullptr));
        if (i.n_l)
            detail::check(pbsa_copy(local->data(), i.l_ids + static_cast<std::size_t>(unit) * i.local_stride,
                                    i.n_l * sizeof(int64_t), nullptr));
        detail::check(pbsa_stream_sync(nullptr));
    }
    pbsa_mem* handle() const { return m_; }

private:
    pbsa_mem* m_ = nullptr;
};

}  // namespace pbsa
