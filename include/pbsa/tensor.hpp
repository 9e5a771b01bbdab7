// pbsa/tensor.hpp -- the reference's tensor module (/root/reference/proj/include/pbsa/tensor.hpp:
// DenseMatrix, Latent4D, matmul, matmul_nt, masked_softmax_rows, the PBT1 file format) as a drop-in:
// the same types, members, signatures, exception types and messages, so code written against the
// reference compiles against this header unchanged.  The free functions run on the B200 through the
// C ABI (include/pbsa_b200.h) and return bit-identical results (fp64 accumulation in the reference's
// order, tensor.hpp:49-53); the PBT1 functions go through the library's PBT1 reader / writer.
// With the reference's include directory first on the path its own tensor.hpp and tensor.cpp are
// used instead, and pbsa/pbsa_b200.hpp works on those types the same way.
#pragma once

#include <cstddef>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbsa/b200_detail.hpp"

namespace pbsa {

/// Row-major float32 matrix (reference tensor.hpp:13-27).
struct DenseMatrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<float> data;

    DenseMatrix() = default;
    DenseMatrix(std::size_t r, std::size_t c, float fill = 0.0f) : rows(r), cols(c), data(r * c, fill) {}
    float& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    float at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    float* row(std::size_t r) { return data.data() + r * cols; }
    const float* row(std::size_t r) const { return data.data() + r * cols; }
    std::size_t size() const { return data.size(); }
};

/// T x H x W x d latent, row-major in (t, h, w, d) order (reference tensor.hpp:30-47).
struct Latent4D {
    std::size_t t = 0, h = 0, w = 0, d = 0;
    std::vector<float> data;

    Latent4D() = default;
    Latent4D(std::size_t t_, std::size_t h_, std::size_t w_, std::size_t d_, float fill = 0.0f)
        : t(t_), h(h_), w(w_), d(d_), data(t_ * h_ * w_ * d_, fill) {}
    std::size_t tokens() const { return t * h * w; }
    std::size_t size() const { return data.size(); }
    float& at(std::size_t ti, std::size_t hi, std::size_t wi, std::size_t c) { return data[((ti * h + hi) * w + wi) * d + c]; }
    float at(std::size_t ti, std::size_t hi, std::size_t wi, std::size_t c) const {
        return data[((ti * h + hi) * w + wi) * d + c];
    }
};

namespace detail {
inline DenseMatrix gpu_matmul(const DenseMatrix& a, const DenseMatrix& b, bool bt, float scale) {
    const std::size_t n = a.rows, kd = a.cols, m = bt ? b.rows : b.cols;
    DenseMatrix c(n, m);
    if (n == 0 || m == 0) return c;
    DevBuf<float> da(a.data.size()), db(b.data.size()), dc(n * m);
    da.upload(a.data.data(), a.data.size());
    db.upload(b.data.data(), b.data.size());
    check(pbsa_matmul(da.p, db.p, to_int(n, "matmul"), to_int(kd, "matmul"), to_int(m, "matmul"), bt ? 1 : 0, scale,
                      dc.p, nullptr));
    dc.download(c.data.data(), n * m);
    return c;
}
}  // namespace detail

/// a * b, fp64 accumulation over ascending k (reference tensor.hpp:51-53, tensor.cpp:8-32).
inline DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols != b.rows)
        throw std::invalid_argument("matmul: a.cols (" + std::to_string(a.cols) + ") != b.rows (" +
                                    std::to_string(b.rows) + ")");
    return detail::gpu_matmul(a, b, false, 1.0f);
}

/// a * b^T (reference tensor.hpp:55-56, tensor.cpp:34-55).
inline DenseMatrix matmul_nt(const DenseMatrix& a, const DenseMatrix& b) {
    if (a.cols != b.cols)
        throw std::invalid_argument("matmul_nt: a.cols (" + std::to_string(a.cols) + ") != b.cols (" +
                                    std::to_string(b.cols) + ")");
    return detail::gpu_matmul(a, b, true, 1.0f);
}

/// Row-wise softmax of scores (+ mask of 0 / -inf entries); fully masked rows come back as zeros;
/// NaN scores rejected (reference tensor.hpp:58-62, tensor.cpp:57-108).
inline DenseMatrix masked_softmax_rows(const DenseMatrix& scores, const DenseMatrix* mask = nullptr) {
    if (mask != nullptr && (mask->rows != scores.rows || mask->cols != scores.cols))
        throw std::invalid_argument("masked_softmax_rows: mask shape mismatch");
    DenseMatrix out(scores.rows, scores.cols);
    if (scores.data.empty()) return out;
    detail::DevBuf<float> ds(scores.data.size()), dm(mask ? mask->data.size() : 0), dout(scores.data.size());
    detail::DevBuf<int> st(1);
    const int zero = 0;
    st.upload(&zero, 1);
    ds.upload(scores.data.data(), scores.data.size());
    if (mask) dm.upload(mask->data.data(), mask->data.size());
    detail::check(pbsa_masked_softmax_rows(ds.p, mask ? dm.p : nullptr, detail::to_int(scores.rows, "masked_softmax_rows"),
                                           detail::to_int(scores.cols, "masked_softmax_rows"), dout.p, st.p, nullptr));
    const int flags = detail::read_status(st);
    if (flags & 1) throw std::invalid_argument("masked_softmax_rows: NaN in scores");
    if (flags & 2) throw std::invalid_argument("masked_softmax_rows: mask entries must be 0 or -inf");
    dout.download(out.data.data(), out.data.size());
    return out;
}

// ---------------------------------------------------------------------------------------------
// PBT1 tensor file format (reference tensor.hpp:64-101): "PBT1" | dtype 0x01 | rank | rank x u64 LE
// dims | row-major f32 LE payload.
// ---------------------------------------------------------------------------------------------

class TensorIoError : public std::runtime_error {
public:
    enum class Kind {
        OpenFailed,
        BadMagic,
        BadDtype,
        Truncated,
        TrailingData,
        BadShape,
    };

    TensorIoError(Kind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
    Kind kind() const { return kind_; }

private:
    Kind kind_;
};

/// Raw decoded tensor file: dims plus flat payload.
struct TensorFile {
    std::vector<std::uint64_t> dims;
    std::vector<float> data;
};

namespace detail {
// library messages start with the TensorIoError::Kind name ("Truncated: truncated payload: ...")
inline void pbt1_check(int rc) {
    if (rc == PBSA_OK) return;
    const std::string msg = pbsa_last_error();
    static const struct { const char* name; TensorIoError::Kind kind; } kinds[] = {
        {"OpenFailed", TensorIoError::Kind::OpenFailed}, {"BadMagic", TensorIoError::Kind::BadMagic},
        {"BadDtype", TensorIoError::Kind::BadDtype},     {"Truncated", TensorIoError::Kind::Truncated},
        {"TrailingData", TensorIoError::Kind::TrailingData}, {"BadShape", TensorIoError::Kind::BadShape}};
    for (const auto& k : kinds) {
        const std::string pre = std::string(k.name) + ": ";
        if (msg.compare(0, pre.size(), pre) == 0) throw TensorIoError(k.kind, msg.substr(pre.size()));
    }
    check(rc);
}
inline void write_file(const std::string& path, const std::vector<std::uint64_t>& dims, const std::vector<float>& data) {
    pbt1_check(pbsa_pbt1_write(path.c_str(), data.empty() ? nullptr : data.data(), static_cast<int>(dims.size()),
                               dims.data()));
}
}  // namespace detail

inline void write_tensor(const std::string& path, const DenseMatrix& m) {
    detail::write_file(path, {m.rows, m.cols}, m.data);
}

inline void write_tensor(const std::string& path, const Latent4D& x) {
    detail::write_file(path, {x.t, x.h, x.w, x.d}, x.data);
}

inline TensorFile read_tensor(const std::string& path) {
    int rank = 0;
    std::uint64_t dims[255];
    detail::pbt1_check(pbsa_pbt1_info(path.c_str(), &rank, dims, 255));
    TensorFile tf;
    tf.dims.assign(dims, dims + rank);
    std::uint64_t elems = rank == 0 ? 0 : 1;
    for (std::uint64_t dm : tf.dims) elems *= dm;
    tf.data.resize(elems);
    detail::pbt1_check(pbsa_pbt1_read(path.c_str(), elems ? tf.data.data() : nullptr, elems));
    return tf;
}

inline DenseMatrix read_matrix(const std::string& path) {
    TensorFile tf = read_tensor(path);
    if (tf.dims.size() != 2)
        throw TensorIoError(TensorIoError::Kind::BadShape, "expected rank 2, got " + std::to_string(tf.dims.size()));
    DenseMatrix m;
    m.rows = tf.dims[0];
    m.cols = tf.dims[1];
    m.data = std::move(tf.data);
    return m;
}

inline Latent4D read_latent(const std::string& path) {
    TensorFile tf = read_tensor(path);
    if (tf.dims.size() != 4)
        throw TensorIoError(TensorIoError::Kind::BadShape, "expected rank 4, got " + std::to_string(tf.dims.size()));
    Latent4D x;
    x.t = tf.dims[0];
    x.h = tf.dims[1];
    x.w = tf.dims[2];
    x.d = tf.dims[3];
    x.data = std::move(tf.data);
    return x;
}

}  // namespace pbsa
