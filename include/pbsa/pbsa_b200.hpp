// pbsa/pbsa_b200.hpp -- C++ host API of the B200 PBSA path (header-only, over the C ABI
// include/pbsa_b200.h).  Mirrors the reference's SPEC operator API on the
// reference's value types (pbsa/tensor.hpp): same op names and argument meaning; argument errors
// throw std::invalid_argument with the library's message, CUDA failures std::runtime_error.
//
// Two layers:
//   * SPEC-shaped host ops (compress_blocks, score_select = coarse_attention + select_topk +
//     aggregate_scores, attention_sparse): host containers in, host containers out; they upload,
//     run the sm_100a kernels and download.  fp32 inputs are rounded to bf16 on upload (the
//     GPU path's numeric contract).
//   * pbsa::Memory: the device-resident hot loop (slot pools + P/L state), one PBSA call per
//     attend() on a caller stream, no host synchronisation.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbsa/tensor.hpp"
#include "pbsa_b200.h"

namespace pbsa {

// SPEC.md:250-265
struct BlockRepresentatives {
    std::size_t n_blocks = 0, d = 0;
    std::vector<float> data;  // n_blocks x d
};
struct BlockScores {
    std::vector<float> scores;
};
struct BlockMask {
    std::size_t n_query_blocks = 0, n_persistent_blocks = 0, n_local_blocks = 0;
    std::vector<std::vector<int32_t>> visible;  // per query block, ascending local indices
};
// SPEC.md:346-350
struct AttentionConfig {
    std::size_t d = 128;
    std::size_t n_heads = 1;
    double scale = 0.0;  // <= 0 -> d^-1/2
};

namespace detail {

inline void check(int rc) {
    if (rc == PBSA_OK) return;
    const std::string msg = pbsa_last_error();
    if (rc == PBSA_ECUDA) throw std::runtime_error(msg);
    throw std::invalid_argument(msg);
}

inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline uint16_t to_bf16(float f) {  // round to nearest even
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

inline float from_bf16(uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;
    explicit DevBuf(std::size_t count) : n(count) { cuda(cudaMalloc(&p, (count ? count : 1) * sizeof(T)), "cudaMalloc"); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { cudaFree(p); }
    void upload(const T* h, std::size_t count) { cuda(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
    void download(T* h, std::size_t count) const { cuda(cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H"); }
    void zero() { cuda(cudaMemset(p, 0, (n ? n : 1) * sizeof(T)), "cudaMemset"); }
};

inline std::vector<uint16_t> bf16_of(const std::vector<float>& v) {
    std::vector<uint16_t> o(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) o[i] = to_bf16(v[i]);
    return o;
}

}  // namespace detail

// k = max(1, ceil(N_l * ratio))
inline std::size_t topk_count(std::size_t n_local, double ratio) {
    if (n_local < 1) throw std::invalid_argument("select_topk: empty local region");
    if (!(ratio > 0.0 && ratio <= 1.0)) throw std::invalid_argument("select_topk: topk_ratio must be in (0,1]");
    const auto k = static_cast<std::size_t>(std::ceil(static_cast<double>(n_local) * ratio));
    return k < 1 ? 1 : (k > n_local ? n_local : k);
}

// (a) SPEC.md:268-276
inline BlockRepresentatives compress_blocks(const BlockedTensor& xb) {
    const std::size_t nb = xb.layout.n_b, b = xb.layout.b, d = xb.layout.d;
    if (xb.data.size() != nb * b * d) throw std::invalid_argument("compress_blocks: data length does not match layout");
    detail::DevBuf<uint16_t> x(nb * b * d);
    detail::DevBuf<float> reps(nb * d);
    x.upload(detail::bf16_of(xb.data).data(), nb * b * d);
    detail::check(pbsa_compress(x.p, static_cast<int64_t>(nb * b * d), static_cast<int64_t>(b * d), nullptr,
                                static_cast<int>(nb), 1, static_cast<int>(b), static_cast<int>(d), reps.p,
                                static_cast<int64_t>(nb * d), nullptr));
    BlockRepresentatives out{nb, d, std::vector<float>(nb * d)};
    reps.download(out.data.data(), nb * d);
    return out;
}

// (b) SPEC.md:277-303: coarse attention of qc against kc (all key blocks), Top-k over the local
// window [local_off, local_off + n_local); optionally s_t over all keys (the k=0 pass).
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

// (c) SPEC.md:367-375 on a host block store: query block i attends to dense_blocks (always
// visible) and local_blocks[mask.visible[i]].  Returns (nqb*b) x d.
inline DenseMatrix attention_sparse(const BlockedTensor& q_blocks, const BlockedTensor& k_store,
                                    const BlockedTensor& v_store, const std::vector<int32_t>& dense_blocks,
                                    const std::vector<int32_t>& local_blocks, const BlockMask& mask,
                                    const AttentionConfig& cfg) {
    const std::size_t nqb = q_blocks.layout.n_b, b = q_blocks.layout.b, d = q_blocks.layout.d;
    const std::size_t ns = k_store.layout.n_b;
    if (k_store.layout.b != b || v_store.layout.b != b || k_store.layout.d != d || v_store.layout.n_b != ns)
        throw std::invalid_argument("attention_sparse: geometry inconsistency");
    if (cfg.d != d) throw std::invalid_argument("attention_sparse: AttentionConfig.d mismatch");
    const std::size_t k = mask.visible.empty() ? 0 : mask.visible[0].size();
    std::vector<int32_t> sel;
    for (const auto& v : mask.visible) {
        if (v.size() != k) throw std::invalid_argument("attention_sparse: |visible(q)| must be identical across q");
        sel.insert(sel.end(), v.begin(), v.end());
    }
    if (!mask.visible.empty() && mask.visible.size() != nqb) throw std::invalid_argument("attention_sparse: mask rows != query blocks");
    std::vector<uint16_t> kp(ns * 64 * d, 0), vp(ns * 64 * d, 0);
    for (std::size_t s = 0; s < ns; ++s)
        for (std::size_t r = 0; r < b; ++r)
            for (std::size_t c = 0; c < d; ++c) {
                kp[(s * 64 + r) * d + c] = detail::to_bf16(k_store.data[(s * b + r) * d + c]);
                vp[(s * 64 + r) * d + c] = detail::to_bf16(v_store.data[(s * b + r) * d + c]);
            }
    detail::DevBuf<uint16_t> dq(nqb * b * d), dk(ns * 64 * d), dv(ns * 64 * d), dout(nqb * b * d);
    detail::DevBuf<int32_t> dd(dense_blocks.size()), dl(local_blocks.size()), ds(sel.size());
    dq.upload(detail::bf16_of(q_blocks.data).data(), nqb * b * d);
    dk.upload(kp.data(), kp.size());
    dv.upload(vp.data(), vp.size());
    if (!dense_blocks.empty()) dd.upload(dense_blocks.data(), dense_blocks.size());
    if (!local_blocks.empty()) dl.upload(local_blocks.data(), local_blocks.size());
    if (!sel.empty()) ds.upload(sel.data(), sel.size());
    detail::check(pbsa_bsa_fwd(dq.p, dk.p, dv.p, static_cast<int>(ns), dense_blocks.empty() ? nullptr : dd.p,
                               static_cast<int>(dense_blocks.size()), static_cast<int>(dense_blocks.size()),
                               local_blocks.empty() ? nullptr : dl.p, static_cast<int>(local_blocks.size()),
                               static_cast<int>(local_blocks.size()), sel.empty() ? nullptr : ds.p, static_cast<int>(k),
                               static_cast<int>(nqb), static_cast<int>(b), static_cast<int>(d), 1,
                               static_cast<float>(cfg.scale), dout.p, nullptr, nullptr, 0, nullptr));
    std::vector<uint16_t> h(nqb * b * d);
    dout.download(h.data(), h.size());
    DenseMatrix out(nqb * b, d);
    for (std::size_t i = 0; i < h.size(); ++i) out.data[i] = detail::from_bf16(h[i]);
    return out;
}

// (d) device-resident PBSA memory + hot loop (Alg. 1)
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
    void reset(cudaStream_t s = nullptr) { detail::check(pbsa_mem_reset(m_, s)); }
    // current chunk K/V: device [units][blocks_per_chunk*b][d] bf16
    void write_chunk(const void* k_chunk, const void* v_chunk, cudaStream_t s = nullptr) {
        detail::check(pbsa_mem_write_chunk(m_, k_chunk, v_chunk, s));
    }
    // one PBSA call; mode PBSA_MODE_CACHE_UPDATE = the k=0 pass (scores + push/evict/Top-C)
    void attend(const void* q, int k_top, int mode, void* o, float* lse = nullptr, double scale = 0.0,
                cudaStream_t s = nullptr) {
        detail::check(pbsa_attend(m_, q, k_top, static_cast<float>(scale), mode, o, lse, s));
    }
    // write_chunk + attend fused (one ingest pass over Q, K, V): device [units][bpc*b][d] bf16
    void attend_qkv(const void* q, const void* k, const void* v, int k_top, int mode, void* o,
                    float* lse = nullptr, double scale = 0.0, cudaStream_t s = nullptr) {
        detail::check(pbsa_attend_qkv(m_, q, k, v, k_top, static_cast<float>(scale), mode, o, lse, s));
    }
    // attend_qkv on HOST chunks (pinned): upload / compute / download pipelined across calls;
    // o_host is valid after host_sync()
    void attend_qkv_host(const void* q, const void* k, const void* v, int k_top, int mode, void* o_host,
                         double scale = 0.0, cudaStream_t s = nullptr) {
        detail::check(pbsa_attend_qkv_host(m_, q, k, v, k_top, static_cast<float>(scale), mode, o_host, s));
    }
    void host_sync() { detail::check(pbsa_mem_host_sync(m_)); }
    // the same on device chunk latents [batch][T][H][W][heads*d] bf16 (blockify / unblockify fused)
    void attend_latent(const void* q, const void* k, const void* v, const pbsa_latent_geom& g, int k_top, int mode,
                       void* o, float* lse = nullptr, double scale = 0.0, cudaStream_t s = nullptr) {
        detail::check(pbsa_attend_latent(m_, q, k, v, &g, k_top, static_cast<float>(scale), mode, o, lse, s));
    }
    // host convenience on the reference's own types: one batch element's chunk as Latent4D (t, h, w,
    // heads*d) fp32 (rounded to bf16 on upload), blocked by `shape` like blockify; returns O as a
    // Latent4D of the same shape.  Synchronous (uploads, runs on the default stream, downloads).
    Latent4D attend_latent(const Latent4D& q, const Latent4D& k, const Latent4D& v, const BlockShape& shape,
                           int heads, int k_top, int mode, double scale = 0.0) {
        if (k.t != q.t || k.h != q.h || k.w != q.w || k.d != q.d || v.t != q.t || v.h != q.h || v.w != q.w ||
            v.d != q.d)
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
        std::vector<uint16_t> ho(q.size());
        detail::cuda(cudaMemcpy(ho.data(), dout.p, ho.size() * 2, cudaMemcpyDeviceToHost), "D2H");
        Latent4D out(q.t, q.h, q.w, q.d);
        for (std::size_t i = 0; i < ho.size(); ++i) out.data[i] = detail::from_bf16(ho[i]);
        return out;
    }
    void commit(const float* s_t, cudaStream_t s = nullptr) { detail::check(pbsa_mem_commit(m_, s_t, s)); }
    // assemble_kv as block ids: persistent (sinks id asc, dynamic id asc), local
    void assemble(int unit, std::vector<int64_t>* persistent, std::vector<int64_t>* local) const {
        const pbsa_mem_info i = info();
        persistent->resize(i.n_p);
        local->resize(i.n_l);
        if (i.n_p)
            detail::cuda(cudaMemcpy(persistent->data(), i.p_ids + static_cast<std::size_t>(unit) * i.capacity_c,
                                    i.n_p * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
        if (i.n_l)
            detail::cuda(cudaMemcpy(local->data(), i.l_ids + static_cast<std::size_t>(unit) * i.local_stride,
                                    i.n_l * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
    }
    pbsa_mem* handle() const { return m_; }

private:
    pbsa_mem* m_ = nullptr;
};

}  // namespace pbsa
