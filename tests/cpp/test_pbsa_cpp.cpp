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

int main() {
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
        pbsa::detail::cuda(cudaDeviceSynchronize(), "sync");
        std::vector<int64_t> P, L;
        mem.assemble(1, &P, &L);
        EXPECT(static_cast<int>(L.size()) == W * bpc);
        EXPECT(static_cast<int>(P.size()) == C);
        for (int i = 0; i < bpc; ++i) EXPECT(P[i] == i);             // sinks = first chunk, id asc
        for (std::size_t i = 1; i < L.size(); ++i) EXPECT(L[i] > L[i - 1]);  // FIFO order
        EXPECT(L.front() == 4 * bpc);                                 // chunks 4, 5 in the window
    }
    std::printf("PASS %d\n", n_ok);
    return 0;
}
