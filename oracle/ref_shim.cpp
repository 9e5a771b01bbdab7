// ref_shim.cpp -- C-ABI shim over the REFERENCE's own C++ sources (test infrastructure only).
//
// Compiled together with /root/reference/proj/src/{tensor,tensor_io,blockify}.cpp into
// oracle/_ref/libpbsa_ref.so by oracle/Makefile (target `ref`).  Nothing from the reference is
// copied into this repo: the sources are compiled where they lie.  tests/test_oracle_vs_ref.py
// uses it to pin the oracle's restated primitives bit-exactly to the reference, and bench.py's
// --impl reference leg may use it as the reference CPU primitive throughput probe.

#include <cstdint>
#include <cstring>
#include <string>

#include "pbsa/blockify.hpp"
#include "pbsa/rng.hpp"
#include "pbsa/tensor.hpp"

namespace {
thread_local std::string g_err;

pbsa::DenseMatrix mat(const float* p, int64_t r, int64_t c) {
    pbsa::DenseMatrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
    if (r * c) std::memcpy(m.data.data(), p, sizeof(float) * r * c);
    return m;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_matmul_nt(const float* a, int64_t ar, int64_t ac, const float* b, int64_t br, float* out) {
    return guard([&] {
        auto c = pbsa::matmul_nt(mat(a, ar, ac), mat(b, br, ac));
        std::memcpy(out, c.data.data(), sizeof(float) * c.size());
    });
}

int ref_matmul(const float* a, int64_t ar, int64_t ac, const float* b, int64_t bc, float* out) {
    return guard([&] {
        auto c = pbsa::matmul(mat(a, ar, ac), mat(b, ac, bc));
        std::memcpy(out, c.data.data(), sizeof(float) * c.size());
    });
}

int ref_masked_softmax_rows(const float* s, int64_t rows, int64_t cols, const float* mask,
                            float* out) {
    return guard([&] {
        auto sm = mat(s, rows, cols);
        pbsa::DenseMatrix mm;
        if (mask) mm = mat(mask, rows, cols);
        auto o = pbsa::masked_softmax_rows(sm, mask ? &mm : nullptr);
        std::memcpy(out, o.data.data(), sizeof(float) * o.size());
    });
}

int ref_blockify(const float* x, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                 int64_t bh, int64_t bw, float* out) {
    return guard([&] {
        pbsa::Latent4D lx(t, h, w, d);
        std::memcpy(lx.data.data(), x, sizeof(float) * lx.size());
        auto xb = pbsa::blockify(lx, pbsa::BlockShape{std::size_t(bt), std::size_t(bh), std::size_t(bw)});
        std::memcpy(out, xb.data.data(), sizeof(float) * xb.data.size());
    });
}

int ref_unblockify(const float* xb, int64_t t, int64_t h, int64_t w, int64_t d, int64_t bt,
                   int64_t bh, int64_t bw, float* out) {
    return guard([&] {
        pbsa::BlockedTensor b;
        b.layout = pbsa::make_block_layout(t, h, w, d, pbsa::BlockShape{std::size_t(bt), std::size_t(bh), std::size_t(bw)});
        b.data.assign(xb, xb + t * h * w * d);
        auto x = pbsa::unblockify(b);
        std::memcpy(out, x.data.data(), sizeof(float) * x.size());
    });
}

int ref_block_index_map(int64_t t, int64_t h, int64_t w, int64_t bt, int64_t bh, int64_t bw,
                        int64_t flat, int64_t* bid, int64_t* off) {
    return guard([&] {
        auto l = pbsa::make_block_layout(t, h, w, 1, pbsa::BlockShape{std::size_t(bt), std::size_t(bh), std::size_t(bw)});
        auto p = pbsa::block_index_map(l, static_cast<std::size_t>(flat));
        *bid = static_cast<int64_t>(p.first);
        *off = static_cast<int64_t>(p.second);
    });
}

int ref_rng_normal(uint64_t seed, int64_t n, float* out) {
    pbsa::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
    return 0;
}

uint64_t ref_rng_derive(uint64_t seed, uint64_t stream) { return pbsa::Rng::derive(seed, stream); }

int ref_write_matrix(const char* path, const float* p, int64_t r, int64_t c) {
    return guard([&] { pbsa::write_tensor(path, mat(p, r, c)); });
}

int ref_read_matrix(const char* path, float* out, int64_t cap, int64_t* rows, int64_t* cols) {
    return guard([&] {
        auto m = pbsa::read_matrix(path);
        *rows = static_cast<int64_t>(m.rows);
        *cols = static_cast<int64_t>(m.cols);
        if (static_cast<int64_t>(m.size()) <= cap) std::memcpy(out, m.data.data(), sizeof(float) * m.size());
    });
}

// PBT1 through the reference's own writer / reader (tests/test_pbt1.py); the read returns the
// TensorIoError::Kind as 10 + kind on format errors.
int ref_write_latent(const char* path, const float* p, int64_t t, int64_t h, int64_t w, int64_t d) {
    return guard([&] {
        pbsa::Latent4D x(static_cast<std::size_t>(t), static_cast<std::size_t>(h), static_cast<std::size_t>(w),
                         static_cast<std::size_t>(d));
        if (x.size()) std::memcpy(x.data.data(), p, sizeof(float) * x.size());
        pbsa::write_tensor(path, x);
    });
}

int ref_read_tensor(const char* path, float* out, int64_t cap, int64_t* rank, int64_t* dims) {
    try {
        auto tf = pbsa::read_tensor(path);
        *rank = static_cast<int64_t>(tf.dims.size());
        for (std::size_t i = 0; i < tf.dims.size() && i < 8; ++i) dims[i] = static_cast<int64_t>(tf.dims[i]);
        if (static_cast<int64_t>(tf.data.size()) <= cap && !tf.data.empty())
            std::memcpy(out, tf.data.data(), sizeof(float) * tf.data.size());
        return 0;
    } catch (const pbsa::TensorIoError& e) {
        g_err = e.what();
        return 10 + static_cast<int>(e.kind());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
