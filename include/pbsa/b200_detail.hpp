// pbsa/b200_detail.hpp -- plumbing shared by the header-only C++ API over the C ABI
// (include/pbsa_b200.h): status -> exception mapping, bf16 rounding and a device buffer.  Needs no
// CUDA headers: device memory goes through pbsa_dev_alloc / pbsa_copy / pbsa_stream_sync, so code
// written against the reference (plain C++20, no CUDA toolchain) builds against this drop-in.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbsa_b200.h"

namespace pbsa {
namespace detail {

// library status -> the reference's exception types (std::invalid_argument for bad arguments,
// tensor.cpp:10-11 / blockify.cpp:10-23; std::runtime_error for device failures)
inline void check(int rc) {
    if (rc == PBSA_OK) return;
    const std::string msg = pbsa_last_error();
    if (rc == PBSA_ECUDA) throw std::runtime_error(msg);
    throw std::invalid_argument(msg);
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

inline std::vector<uint16_t> bf16_of(const std::vector<float>& v) {
    std::vector<uint16_t> o(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) o[i] = to_bf16(v[i]);
    return o;
}

// device array; host transfers are synchronous (legacy default stream, like the kernels the
// host-convenience ops launch)
template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;
    explicit DevBuf(std::size_t count) : n(count) {
        void* v = nullptr;
        check(pbsa_dev_alloc(&v, (count ? count : 1) * sizeof(T)));
        p = static_cast<T*>(v);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { pbsa_dev_free(p); }
    void upload(const T* h, std::size_t count) {
        if (!count) return;
        check(pbsa_copy(p, h, count * sizeof(T), nullptr));
        check(pbsa_stream_sync(nullptr));
    }
    void download(T* h, std::size_t count) const {
        if (!count) return;
        check(pbsa_copy(h, p, count * sizeof(T), nullptr));
        check(pbsa_stream_sync(nullptr));
    }
    std::vector<T> to_host() const {
        std::vector<T> h(n);
        download(h.data(), n);
        return h;
    }
};

template <class T>
inline DevBuf<T>* dev_of(const std::vector<T>& h, DevBuf<T>& buf) {
    buf.upload(h.data(), h.size());
    return &buf;
}

inline int to_int(std::size_t v, const char* what) {
    if (v > static_cast<std::size_t>(0x7fffffff)) throw std::invalid_argument(std::string(what) + ": dimension too large");
    return static_cast<int>(v);
}

// device status word of the validating primitives -> the reference's error messages
inline int read_status(const DevBuf<int>& st) {
    int v = 0;
    st.download(&v, 1);
    return v;
}

}  // namespace detail
}  // namespace pbsa
