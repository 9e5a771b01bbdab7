// pbsa/tensor.hpp -- value types of the pbsa:: operator API, field-compatible with the reference
// (/root/reference/proj/include/pbsa/tensor.hpp:13-47 and blockify.hpp:11-46): the same names,
// members and row-major layouts, so code written against the reference compiles against this
// drop-in.  Only the types are restated here; the operations live in pbsa/pbsa_b200.hpp (GPU).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace pbsa {

// rows x cols, row-major fp32 (reference tensor.hpp:13-27)
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

// (t, h, w, d) latent, row-major (reference tensor.hpp:30-47)
struct Latent4D {
    std::size_t t = 0, h = 0, w = 0, d = 0;
    std::vector<float> data;

    Latent4D() = default;
    Latent4D(std::size_t t_, std::size_t h_, std::size_t w_, std::size_t d_, float fill = 0.0f)
        : t(t_), h(h_), w(w_), d(d_), data(t_ * h_ * w_ * d_, fill) {}
    std::size_t tokens() const { return t * h * w; }
    std::size_t size() const { return data.size(); }
    float& at(std::size_t a, std::size_t b, std::size_t c, std::size_t e) { return data[((a * h + b) * w + c) * d + e]; }
    float at(std::size_t a, std::size_t b, std::size_t c, std::size_t e) const { return data[((a * h + b) * w + c) * d + e]; }
};

// block extents (reference blockify.hpp:11-18)
struct BlockShape {
    std::size_t b_t = 1, b_h = 1, b_w = 1;
    std::size_t tokens() const { return b_t * b_h * b_w; }
    bool operator==(const BlockShape&) const = default;
};

// partition of a (t, h, w, d) latent into blocks (reference blockify.hpp:21-29)
struct BlockLayout {
    std::size_t n_t = 0, n_h = 0, n_w = 0;
    std::size_t n_b = 0;
    std::size_t b = 0;
    BlockShape shape;
    std::size_t t = 0, h = 0, w = 0, d = 0;
    bool operator==(const BlockLayout&) const = default;
};

// block-major (n_b, b, d) storage (reference blockify.hpp:32-46)
struct BlockedTensor {
    BlockLayout layout;
    std::vector<float> data;
    float* block(std::size_t id) { return data.data() + id * layout.b * layout.d; }
    const float* block(std::size_t id) const { return data.data() + id * layout.b * layout.d; }
    float* token(std::size_t id, std::size_t off) { return block(id) + off * layout.d; }
    const float* token(std::size_t id, std::size_t off) const { return block(id) + off * layout.d; }
};

}  // namespace pbsa
