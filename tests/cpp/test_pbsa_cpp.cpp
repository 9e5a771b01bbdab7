// C++ drop-in check: the pbsa:: host API (include/pbsa/pbsa_b200.hpp) on the SPEC known-answer
// examples plus a memory state-machine run.  Built by `make cpp-test`; run on a GPU by
// tests/test_cpp_api.py.  Prints "PASS <n>" on success, exits 1 on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pbsa/pbsa_b200.hpp"

static int n_ok = 0;
#define EXPECT(cond)                                                          \
    do {                                                                      \
        if (!(cond)) {                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
            std::exit(1);                                                     \
        }                                                                     \
        ++n_ok;                                                               \
    } while (0)

static pbsa::BlockedTensor blocks(std::size_t nb, std::size_t b, std::size_t d, const std::vector<float>& v) {
    pbsa::BlockedTensor t;
    t.layout.n_b = nb;
    t.layout.b = b;
    t.layout.d = d;
    t.data = v;
    return t;
}

// SPEC known-answer examples of the tensor / blockify / router / memory / attention modules through
// the GPU-backed drop-in free functions (shared with test_ref_headers.cpp, where the same checks run
// on the reference's own types and primitives)
#include "spec_kats.inc"

int main() {
    spec_kats();
    // compress_blocks: block {[0,2],[2,0]} -> [1,1] (d padded to 64 with zeros)
    {
        std::vector<float> v(2 * 64, 0.0f);
        v[0] = 0.0f; v[1] = 2.0f; v[64] = 2.0f; v[65] = 0.0f;
        auto r = pbsa::compress_blocks(blocks(1, 2, 64, v));
        EXPECT(r.data[0] == 1.0f && r.data[1] == 1.0f && r.data[2] == 0.0f);
    }
    // select_topk, SPEC.md:303 shape: the largest coarse probability wins; ties -> lower index
    {
        pbsa::BlockRepresentatives qc{1, 64, std::vector<float>(64, 0.0f)};
        pbsa::BlockRepresentatives kc{3, 64, std::vector<float>(3 * 64, 0.0f)};
        qc.data[0] = 1.0f;
        kc.data[0 * 64] = 0.1f; kc.data[1 * 64] = 0.7f; kc.data[2 * 64] = 0.2f;
        auto s = pbsa::score_select(qc, kc, 0, 3, 1, true);
        EXPECT(s.mask.visible.size() == 1 && s.mask.visible[0].size() == 1 && s.mask.visible[0][0] == 1);
        double sum = 0;
        for (float x : s.scores.scores) sum += x;
        EXPECT(std::fabs(sum - 1.0) < 1e-5);
        pbsa::BlockRepresentatives z{1, 64, std::vector<float>(64, 0.0f)};
        auto t = pbsa::score_select(z, kc, 0, 3, 2, false);  // uniform row -> lowest indices
        EXPECT(t.mask.visible[0][0] == 0 && t.mask.visible[0][1] == 1);
    }
    // attention_sparse: empty P, one visible local block -> dense attention over it
    {
        const std::size_t b = 8, d = 64;
        std::vector<float> q(b * d), k(3 * b * d), v(3 * b * d);
        for (std::size_t i = 0; i < q.size(); ++i) q[i] = std::sin(0.37 * i);
        for (std::size_t i = 0; i < k.size(); ++i) k[i] = std::cos(0.11 * i);
        for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.05 * i + 1.0);
        for (auto* vec : {&q, &k, &v})
            for (auto& x : *vec) x = pbsa::detail::from_bf16(pbsa::detail::to_bf16(x));
        pbsa::BlockMask mask;
        mask.visible = {{1}};
        pbsa::AttentionConfig cfg{d, 1, 0.0};
        auto o = pbsa::attention_sparse(blocks(1, b, d, q), blocks(3, b, d, k), blocks(3, b, d, v), {}, {0, 1, 2}, mask, cfg);
        const double scale = 1.0 / std::sqrt(double(d));
        double worst = 0;
        for (std::size_t r = 0; r < b; ++r) {
            std::vector<double> e(b);
            double mx = -1e30, den = 0;
            for (std::size_t j = 0; j < b; ++j) {
                double s = 0;
                for (std::size_t c = 0; c < d; ++c) s += double(q[r * d + c]) * k[(b + j) * d + c];
                e[j] = s * scale;
                mx = std::max(mx, e[j]);
            }
            for (auto& x : e) den += (x = std::exp(x - mx));
            for (std::size_t c = 0; c < d; ++c) {
                double acc = 0;
                for (std::size_t j = 0; j < b; ++j) acc += e[j] / den * v[(b + j) * d + c];
                worst = std::max(worst, std::fabs(acc - o.at(r, c)));
            }
        }
        EXPECT(worst < 2e-2);
    }
    // memory: invalid capacity throws std::invalid_argument (mirrors SPEC errors)
    {
        bool threw = false;
        try {
            pbsa::Memory bad(1, 2, 1, 4, 60, 128);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
    }
    // memory state machine through the hot-loop API: sizes follow push_chunk / Top-C
    {
        const int U = 2, bpc = 4, b = 60, d = 128, C = 8, W = 2;
        pbsa::Memory mem(U, C, W, bpc, b, d);
        pbsa::detail::DevBuf<uint16_t> q(U * bpc * b * d), kv(U * bpc * b * d), o(U * bpc * b * d);
        std::vector<uint16_t> h(q.n);
        for (std::size_t i = 0; i < h.size(); ++i) h[i] = pbsa::detail::to_bf16(std::sin(0.001 * i));
        q.upload(h.data(), h.size());
        kv.upload(h.data(), h.size());
        for (int c = 0; c < 6; ++c) {
            mem.write_chunk(kv.p, kv.p);
            mem.attend(q.p, 2, PBSA_MODE_CACHE_UPDATE, o.p);
        }
        pbsa::detail::check(pbsa_stream_sync(nullptr));
        std::vector<int64_t> P, L;
        mem.assemble(1, &P, &L);
        EXPECT(static_cast<int>(L.size()) == W * bpc);
        EXPECT(static_cast<int>(P.size()) == C);
        for (int i = 0; i < bpc; ++i) EXPECT(P[i] == i);             // sinks = first chunk, id asc
        for (std::size_t i = 1; i < L.size(); ++i) EXPECT(L[i] > L[i - 1]);  // FIFO order
        EXPECT(L.front() == 4 * bpc);                                 // chunks 4, 5 in the window
    }
    // Latent4D drop-in: attend_latent on (t, h, w, heads*d) chunks == attend_qkv on the blocked
    // per-head tensors (blockify.cpp order: block (nt*N_h + nh)*N_w + nw, token (dt*B_h + dh)*B_w + dw)
    {
        const int heads = 2, d = 64, T = 2, H = 4, Wd = 6, bt = 1, bh = 2, bw = 3, bpc = 8, b = 6;
        const int U = heads, C = 2 * bpc, Wc = 1;
        pbsa::Memory ml(U, C, Wc, bpc, b, d), mq(U, C, Wc, bpc, b, d);
        auto fill = [&](int seed) {
            pbsa::Latent4D x(T, H, Wd, heads * d);
            for (std::size_t i = 0; i < x.size(); ++i)
                x.data[i] = pbsa::detail::from_bf16(pbsa::detail::to_bf16(std::sin(0.013 * i + seed)));
            return x;
        };
        auto blocked = [&](const pbsa::Latent4D& x) {  // [heads][bpc*b][d]
            std::vector<uint16_t> out(static_cast<std::size_t>(heads) * bpc * b * d);
            for (int hh = 0; hh < heads; ++hh)
                for (int nt = 0; nt < T / bt; ++nt)
                    for (int nh = 0; nh < H / bh; ++nh)
                        for (int nw = 0; nw < Wd / bw; ++nw)
                            for (int dt = 0; dt < bt; ++dt)
                                for (int dh = 0; dh < bh; ++dh)
                                    for (int dw = 0; dw < bw; ++dw) {
                                        const int blk = (nt * (H / bh) + nh) * (Wd / bw) + nw;
                                        const int tok = (dt * bh + dh) * bw + dw;
                                        for (int c = 0; c < d; ++c)
                                            out[((static_cast<std::size_t>(hh) * bpc + blk) * b + tok) * d + c] =
                                                pbsa::detail::to_bf16(x.at(nt * bt + dt, nh * bh + dh, nw * bw + dw, hh * d + c));
                                    }
            return out;
        };
        bool same = true;
        for (int c = 0; c < 4; ++c) {
            const int mode = (c & 1) ? PBSA_MODE_CACHE_UPDATE : PBSA_MODE_DENOISE;
            auto q = fill(3 * c), k = fill(3 * c + 1), v = fill(3 * c + 2);
            pbsa::Latent4D ol = ml.attend_latent(q, k, v, pbsa::BlockShape{bt, bh, bw}, heads, 2, mode);
            pbsa::detail::DevBuf<uint16_t> dq(U * bpc * b * d), dk(dq.n), dv(dq.n), dout(dq.n);
            const auto hq = blocked(q), hk = blocked(k), hv = blocked(v);
            dq.upload(hq.data(), hq.size());
            dk.upload(hk.data(), hk.size());
            dv.upload(hv.data(), hv.size());
            mq.attend_qkv(dq.p, dk.p, dv.p, 2, mode, dout.p);
            const std::vector<uint16_t> ob = dout.to_host();
            const auto ol_blocked = blocked(ol);
            for (std::size_t i = 0; i < ob.size(); ++i) same &= ob[i] == ol_blocked[i];
        }
        EXPECT(same);
        bool threw = false;
        try {
            ml.attend_latent(fill(0), fill(1), fill(2), pbsa::BlockShape{1, 3, 3}, heads, 2, 0);  // 4 % 3 != 0
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()).find("not divisible") != std::string::npos;
        }
        EXPECT(threw);
    }
    // host-resident chunks: attend_qkv_host (uploads / compute / downloads pipelined over two
    // staging sets) == attend_qkv on device copies, denoise and cache-update calls
    {
        const int U = 2, C = 12, Wc = 2, bpc = 6, b = 60, d = 128, n = U * bpc * b * d, calls = 9;
        pbsa::Memory mh(U, C, Wc, bpc, b, d), md(U, C, Wc, bpc, b, d);
        std::vector<std::vector<uint16_t>> hin, hout, dref;  // inputs stay alive until host_sync
        hin.reserve(3 * calls);
        hout.reserve(calls);
        dref.reserve(calls);
        pbsa::detail::DevBuf<uint16_t> dq(n), dk(n), dv(n), dout(n);
        for (int c = 0; c < calls; ++c) {
            const int mode = (c % 3 == 2) ? PBSA_MODE_CACHE_UPDATE : PBSA_MODE_DENOISE;
            for (int t = 0; t < 3; ++t) {
                hin.emplace_back(n);
                for (int i = 0; i < n; ++i)
                    hin.back()[i] = pbsa::detail::to_bf16(static_cast<float>(std::sin(0.37 * i + 11.0 * c + 3.0 * t)));
            }
            const auto& q = hin[3 * c];
            const auto& k = hin[3 * c + 1];
            const auto& v = hin[3 * c + 2];
            dq.upload(q.data(), n);
            dk.upload(k.data(), n);
            dv.upload(v.data(), n);
            md.attend_qkv(dq.p, dk.p, dv.p, 3, mode, dout.p);
            dref.emplace_back(n);
            dout.download(dref.back().data(), n);
            hout.emplace_back(n);
            mh.attend_qkv_host(q.data(), k.data(), v.data(), 3, mode, hout.back().data());
        }
        mh.host_sync();
        bool same = true;
        for (int c = 0; c < calls; ++c) same &= hout[c] == dref[c];
        EXPECT(same);
    }
    std::printf("PASS %d\n", n_ok);
    return 0;
}
