// pbsa/blockify.hpp -- the reference's blockify module (/root/reference/proj/include/pbsa/blockify.hpp:
// BlockShape, BlockLayout, BlockedTensor, make_block_layout, blockify, unblockify, block_index_map) as
// a drop-in: same types and signatures, same std::invalid_argument messages.  The layout checks and
// the closed-form index map are host arithmetic; the permutations run on the B200 (pbsa_blockify).
#pragma once

#include <cstddef>
#include <string>
#include <utility>

#include "pbsa/tensor.hpp"

namespace pbsa {

/// Spatiotemporal block extent (b_t, b_h, b_w), all >= 1 (reference blockify.hpp:11-18).
struct BlockShape {
    std::size_t b_t = 1;
    std::size_t b_h = 1;
    std::size_t b_w = 1;

    std::size_t tokens() const { return b_t * b_h * b_w; }
    bool operator==(const BlockShape&) const = default;
};

/// Derived partition of a (t, h, w, d) latent into blocks; n_b * b == t*h*w (blockify.hpp:21-29).
struct BlockLayout {
    std::size_t n_t = 0, n_h = 0, n_w = 0;
    std::size_t n_b = 0;
    std::size_t b = 0;
    BlockShape shape;
    std::size_t t = 0, h = 0, w = 0, d = 0;

    bool operator==(const BlockLayout&) const = default;
};

/// Block-major (n_b, b, d) storage: the tokens of one block are contiguous (blockify.hpp:32-46).
struct BlockedTensor {
    BlockLayout layout;
    std::vector<float> data;

    float* block(std::size_t block_id) { return data.data() + block_id * layout.b * layout.d; }
    const float* block(std::size_t block_id) const { return data.data() + block_id * layout.b * layout.d; }
    float* token(std::size_t block_id, std::size_t offset) { return block(block_id) + offset * layout.d; }
    const float* token(std::size_t block_id, std::size_t offset) const { return block(block_id) + offset * layout.d; }
};

/// Divisibility check + block counts; std::invalid_argument naming the axis (blockify.hpp:48-53).
inline BlockLayout make_block_layout(std::size_t t, std::size_t h, std::size_t w, std::size_t d, const BlockShape& shape) {
    if (shape.b_t == 0 || shape.b_h == 0 || shape.b_w == 0) throw std::invalid_argument("block shape extents must be >= 1");
    const std::size_t dims[3] = {t, h, w}, ext[3] = {shape.b_t, shape.b_h, shape.b_w};
    const char* axis[3] = {"t", "h", "w"};
    for (int a = 0; a < 3; ++a)
        if (dims[a] % ext[a] != 0)
            throw std::invalid_argument(std::string("axis ") + axis[a] + " (" + std::to_string(dims[a]) +
                                        ") not divisible by b_" + axis[a] + " (" + std::to_string(ext[a]) + ")");
    BlockLayout l;
    l.n_t = t / shape.b_t;
    l.n_h = h / shape.b_h;
    l.n_w = w / shape.b_w;
    l.n_b = l.n_t * l.n_h * l.n_w;
    l.b = shape.tokens();
    l.shape = shape;
    l.t = t;
    l.h = h;
    l.w = w;
    l.d = d;
    return l;
}

/// Locality-preserving rearrange into block-major layout (blockify.hpp:55-61):
/// block_id = (nt*N_h + nh)*N_w + nw, in_block = (dt*B_h + dh)*B_w + dw.
inline BlockedTensor blockify(const Latent4D& x, const BlockShape& shape) {
    if (x.data.size() != x.t * x.h * x.w * x.d) throw std::invalid_argument("latent data length does not match dims");
    BlockedTensor out;
    out.layout = make_block_layout(x.t, x.h, x.w, x.d, shape);
    out.data.resize(x.data.size());
    if (x.data.empty()) return out;
    detail::DevBuf<float> dx(x.data.size()), dy(x.data.size());
    dx.upload(x.data.data(), x.data.size());
    detail::check(pbsa_blockify(dx.p, detail::to_int(x.t, "blockify"), detail::to_int(x.h, "blockify"),
                                detail::to_int(x.w, "blockify"), detail::to_int(x.d, "blockify"),
                                detail::to_int(shape.b_t, "blockify"), detail::to_int(shape.b_h, "blockify"),
                                detail::to_int(shape.b_w, "blockify"), dy.p, 0, nullptr));
    dy.download(out.data.data(), out.data.size());
    return out;
}

/// Exact inverse of blockify (blockify.hpp:63-64).
inline Latent4D unblockify(const BlockedTensor& xb) {
    const BlockLayout& l = xb.layout;
    if (xb.data.size() != l.n_b * l.b * l.d) throw std::invalid_argument("blocked data length does not match layout");
    if (l.n_b != l.n_t * l.n_h * l.n_w || l.b != l.shape.tokens()) throw std::invalid_argument("inconsistent block layout");
    Latent4D x(l.t, l.h, l.w, l.d);
    if (x.data.empty()) return x;
    detail::DevBuf<float> dx(xb.data.size()), dy(xb.data.size());
    dx.upload(xb.data.data(), xb.data.size());
    detail::check(pbsa_blockify(dx.p, detail::to_int(l.t, "unblockify"), detail::to_int(l.h, "unblockify"),
                                detail::to_int(l.w, "unblockify"), detail::to_int(l.d, "unblockify"),
                                detail::to_int(l.shape.b_t, "unblockify"), detail::to_int(l.shape.b_h, "unblockify"),
                                detail::to_int(l.shape.b_w, "unblockify"), dy.p, 1, nullptr));
    dy.download(x.data.data(), x.data.size());
    return x;
}

/// Closed-form (block_id, in_block_offset) of one flat source token index (blockify.hpp:66-67).
inline std::pair<std::size_t, std::size_t> block_index_map(const BlockLayout& l, std::size_t flat) {
    if (flat >= l.t * l.h * l.w)
        throw std::invalid_argument("flat source index " + std::to_string(flat) + " out of range");
    const std::size_t ti = flat / (l.h * l.w), hi = (flat / l.w) % l.h, wi = flat % l.w;
    const std::size_t blk = (ti / l.shape.b_t * l.n_h + hi / l.shape.b_h) * l.n_w + wi / l.shape.b_w;
    const std::size_t inb = (ti % l.shape.b_t * l.shape.b_h + hi % l.shape.b_h) * l.shape.b_w + wi % l.shape.b_w;
    return {blk, inb};
}

}  // namespace pbsa
