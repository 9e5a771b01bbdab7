// Built with the REFERENCE's headers first (-I/root/reference/proj/include -Iinclude) and linked with
// the reference's own tensor.cpp / blockify.cpp / tensor_io.cpp (Makefile target cpp-test-ref): the
// pbsa:: types here are the reference's, pbsa/pbsa_b200.hpp runs the SPEC ops on them over the C ABI.
//   1. the SPEC known-answer examples (spec_kats.inc) on the reference's types;
//   2. the GPU primitives (pbsa_matmul, pbsa_masked_softmax_rows, pbsa_blockify, pbsa_aggregate_scores)
//      and the GPU SPEC ops (coarse_attention, attention_reference) BIT-EXACT against the reference's
//      own compiled matmul / matmul_nt / masked_softmax_rows / blockify on seeded random inputs.
// Prints "PASS <n>", exits 1 on the first failure.  Run on a GPU by tests/test_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <array>
#include <cstring>
#include <vector>

#include "pbsa/pbsa_b200.hpp"
#include "pbsa/rng.hpp"  // the reference's seeded generator (proj/include/pbsa/rng.hpp)

static int n_ok = 0;
#define EXPECT(cond)                                                    \
    do {                                                                \
        if (!(cond)) {                                                  \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            std::exit(1);                                               \
        }                                                               \
        ++n_ok;                                                         \
    } while (0)

#include "spec_kats.inc"

static bool same_bits(const std::vector<float>& a, const std::vector<float>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
}

static pbsa::DenseMatrix rand_matrix(pbsa::Rng& g, std::size_t r, std::size_t c, float scale) {
    pbsa::DenseMatrix m(r, c);
    for (auto& x : m.data) x = static_cast<float>(g.normal()) * scale;
    return m;
}

// the GPU primitive on device copies of host matrices
static pbsa::DenseMatrix gpu_matmul(const pbsa::DenseMatrix& a, const pbsa::DenseMatrix& b, bool bt, float scale) {
    const std::size_t m = bt ? b.rows : b.cols;
    pbsa::detail::DevBuf<float> da(a.size()), db(b.size()), dc(a.rows * m);
    da.upload(a.data.data(), a.size());
    db.upload(b.data.data(), b.size());
    pbsa::detail::check(pbsa_matmul(da.p, db.p, (int)a.rows, (int)a.cols, (int)m, bt, scale, dc.p, nullptr));
    pbsa::DenseMatrix c(a.rows, m);
    dc.download(c.data.data(), c.size());
    return c;
}

static pbsa::DenseMatrix gpu_softmax(const pbsa::DenseMatrix& s, const pbsa::DenseMatrix* mask) {
    pbsa::detail::DevBuf<float> ds(s.size()), dm(mask ? mask->size() : 0), dout(s.size());
    ds.upload(s.data.data(), s.size());
    if (mask) dm.upload(mask->data.data(), mask->size());
    pbsa::detail::check(pbsa_masked_softmax_rows(ds.p, mask ? dm.p : nullptr, (int)s.rows, (int)s.cols, dout.p, nullptr, nullptr));
    pbsa::DenseMatrix out(s.rows, s.cols);
    dout.download(out.data.data(), out.size());
    return out;
}

int main() {
    spec_kats();
    pbsa::Rng g(20261017);
    const float inf = std::numeric_limits<float>::infinity();
    // matmul / matmul_nt: GPU fp64-accumulating kernel == reference tensor.cpp, bit for bit
    using A3 = std::array<std::size_t, 3>;
    for (auto [n, k, m] : {A3{1, 1, 1}, A3{7, 128, 33}, A3{78, 128, 546}, A3{65, 300, 17}}) {
        auto a = rand_matrix(g, n, k, 1.0f), b = rand_matrix(g, k, m, 3.0f), bt = rand_matrix(g, m, k, 0.5f);
        EXPECT(same_bits(gpu_matmul(a, b, false, 1.0f).data, pbsa::matmul(a, b).data));
        EXPECT(same_bits(gpu_matmul(a, bt, true, 1.0f).data, pbsa::matmul_nt(a, bt).data));
    }
    // masked_softmax_rows: GPU == reference (fp64 exp: CUDA vs glibc, both correctly rounded in practice)
    using A2 = std::array<std::size_t, 2>;
    for (auto [r, c] : {A2{1, 1}, A2{78, 312}, A2{13, 6396}, A2{40, 33}}) {
        auto s = rand_matrix(g, r, c, 4.0f);
        pbsa::DenseMatrix mask(r, c, 0.0f);
        for (std::size_t i = 0; i < mask.size(); ++i)
            if (g.uniform() < 0.3) mask.data[i] = -inf;
        for (std::size_t j = 0; j < c; ++j) mask.data[j] = -inf;  // row 0 fully masked -> zeros
        EXPECT(same_bits(gpu_softmax(s, nullptr).data, pbsa::masked_softmax_rows(s).data));
        EXPECT(same_bits(gpu_softmax(s, &mask).data, pbsa::masked_softmax_rows(s, &mask).data));
    }
    // blockify / unblockify: GPU permutation == reference blockify.cpp
    using A6 = std::array<std::size_t, 6>;
    for (auto [t, h, w, bt, bh, bw] : {A6{3, 30, 52, 1, 15, 4}, A6{3, 8, 8, 3, 4, 4}, A6{2, 16, 16, 1, 8, 8}}) {
        pbsa::Latent4D x(t, h, w, 5);
        for (auto& v : x.data) v = static_cast<float>(g.normal());
        auto ref = pbsa::blockify(x, pbsa::BlockShape{bt, bh, bw});
        pbsa::detail::DevBuf<float> dx(x.size()), dy(x.size());
        dx.upload(x.data.data(), x.size());
        pbsa::detail::check(pbsa_blockify(dx.p, (int)t, (int)h, (int)w, 5, (int)bt, (int)bh, (int)bw, dy.p, 0, nullptr));
        EXPECT(same_bits(dy.to_host(), ref.data));
        pbsa::detail::check(pbsa_blockify(dy.p, (int)t, (int)h, (int)w, 5, (int)bt, (int)bh, (int)bw, dx.p, 1, nullptr));
        EXPECT(same_bits(dx.to_host(), x.data));
    }
    // coarse_attention (GPU: pbsa_matmul with the fp32 scale + pbsa_masked_softmax_rows) == the
    // reference's masked_softmax_rows(matmul_nt(qc, kc) * scale); aggregate_scores == the ascending
    // fp64 column mean of that matrix
    {
        const std::size_t nq = 78, nk = 546, d = 128;
        pbsa::BlockRepresentatives qc{nq, d, rand_matrix(g, nq, d, 0.5f).data}, kc{nk, d, rand_matrix(g, nk, d, 1.0f).data};
        pbsa::DenseMatrix qm(nq, d), km(nk, d);
        qm.data = qc.data;
        km.data = kc.data;
        auto z = pbsa::matmul_nt(qm, km);
        const float scale = static_cast<float>(1.0 / std::sqrt(128.0));
        for (auto& v : z.data) v = v * scale;
        auto a_ref = pbsa::masked_softmax_rows(z);
        auto a = pbsa::coarse_attention(qc, kc);
        EXPECT(same_bits(a.data, a_ref.data));
        auto s = pbsa::aggregate_scores(a);
        std::vector<float> s_ref(nk);
        for (std::size_t j = 0; j < nk; ++j) {
            double acc = 0;
            for (std::size_t i = 0; i < nq; ++i) acc += static_cast<double>(a_ref.at(i, j));
            s_ref[j] = static_cast<float>(acc / static_cast<double>(nq));
        }
        EXPECT(same_bits(s.scores, s_ref));
        // the fused K2 (score_select) agrees with the separate ops on the same inputs
        auto sel = pbsa::score_select(qc, kc, 0, nk, 20, true);
        auto m = pbsa::select_topk(a, 20.0 / nk);
        EXPECT(sel.mask.visible == m.visible);
        EXPECT(same_bits(sel.scores.scores, s.scores));
    }
    // attention_reference on the GPU == the reference's matmul_nt -> scale -> masked_softmax_rows ->
    // matmul composition, bit for bit
    {
        const std::size_t nq = 120, nkv = 300, d = 64;
        auto q = rand_matrix(g, nq, d, 1.0f), k = rand_matrix(g, nkv, d, 1.0f), v = rand_matrix(g, nkv, d, 1.0f);
        pbsa::DenseMatrix mask(nq, nkv, 0.0f);
        for (std::size_t i = 0; i < mask.size(); ++i)
            if (g.uniform() < 0.5) mask.data[i] = -inf;
        pbsa::AttentionConfig cfg{d, 1, 0.0};
        auto s = pbsa::matmul_nt(q, k);
        const float scale = static_cast<float>(1.0 / std::sqrt(64.0));
        for (auto& x : s.data) x = x * scale;
        auto want = pbsa::matmul(pbsa::masked_softmax_rows(s, &mask), v);
        EXPECT(same_bits(pbsa::attention_reference(q, k, v, &mask, cfg).data, want.data));
    }
    // PBT1 through the reference's own writer, read back through the library's reader (and back)
    {
        pbsa::Latent4D x(2, 3, 4, 5);
        for (auto& v : x.data) v = static_cast<float>(g.normal());
        const char* path = "/tmp/pbsa_ref_headers_x.pbt1";
        pbsa::write_tensor(path, x);  // reference tensor_io.cpp
        int rank = 0;
        uint64_t dims[8];
        EXPECT(pbsa_pbt1_info(path, &rank, dims, 8) == PBSA_OK && rank == 4 && dims[3] == 5);
        std::vector<float> back(x.size());
        EXPECT(pbsa_pbt1_read(path, back.data(), back.size()) == PBSA_OK && same_bits(back, x.data));
    }
    std::printf("PASS %d\n", n_ok);
    return 0;
}
