// tensor_io.cu -- PBT1 tensor files on the GPU data path.
//
// Format (reference proj/include/pbsa/tensor.hpp:62-70, reader/writer proj/src/tensor_io.cpp):
//   "PBT1" | dtype u8 (0x01 = f32 LE) | rank u8 | rank x u64 LE dims | row-major f32 payload.
// Error behaviour restated from tensor_io.cpp:56-108: open failure, truncated header/dims/payload,
// bad magic, unsupported dtype, dims whose product overflows u64, and ANY byte after the declared
// payload are rejected; the message starts with the reference's TensorIoError::Kind name.
//
// Host side: pbsa_pbt1_write / pbsa_pbt1_info / pbsa_pbt1_read.  Device side: pbsa_pbt1_load_bf16
// streams the payload through a pinned staging buffer in 8 MB pieces with asynchronous copies
// (double-buffered against the file reads) and converts f32 -> bf16 on the device, so a frame or
// golden latent goes from disk straight into the layout pbsa_attend_latent consumes.
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "internal.h"

namespace pbsa {
namespace {

constexpr char kMagic[4] = {'P', 'B', 'T', '1'};
constexpr uint8_t kDtypeF32 = 0x01;

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

int io_error(const char* kind, const std::string& msg) { return set_error(PBSA_EINVAL, std::string(kind) + ": " + msg); }

// Parses the header (same order of checks as tensor_io.cpp:56-96: magic, dtype/rank, all dims,
// then the u64 overflow of their product); on success leaves the stream at the payload.
int read_header(FILE* f, const std::string& path, std::vector<uint64_t>* dims, uint64_t* elems) {
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4) return io_error("Truncated", "truncated header (magic): " + path);
    if (std::memcmp(magic, kMagic, 4) != 0) return io_error("BadMagic", "bad magic, not a PBT1 file: " + path);
    unsigned char dr[2];
    if (std::fread(dr, 1, 2, f) != 2) return io_error("Truncated", "truncated header (dtype/rank): " + path);
    if (dr[0] != kDtypeF32) return io_error("BadDtype", "unsupported dtype code " + std::to_string(static_cast<int>(dr[0])));
    const int r = dr[1];
    dims->resize(r);
    for (int i = 0; i < r; ++i) {
        unsigned char b[8];
        if (std::fread(b, 1, 8, f) != 8) return io_error("Truncated", "truncated dims: " + path);
        uint64_t v = 0;
        for (int k = 0; k < 8; ++k) v |= static_cast<uint64_t>(b[k]) << (8 * k);
        (*dims)[i] = v;
    }
    uint64_t n = r == 0 ? 0 : 1;
    for (uint64_t v : *dims) {
        if (v != 0 && n > std::numeric_limits<uint64_t>::max() / v) return io_error("BadShape", "dims overflow: " + path);
        n *= v;
    }
    *elems = n;
    return PBSA_OK;
}

int open_read(File* fh, const char* path) {
    fh->f = path ? std::fopen(path, "rb") : nullptr;
    if (!fh->f) return io_error("OpenFailed", std::string("cannot open for read: ") + (path ? path : "(null)"));
    return PBSA_OK;
}

int check_trailing(FILE* f, const std::string& path) {
    if (std::fgetc(f) != EOF) return io_error("TrailingData", "payload longer than declared dims: " + path);
    return PBSA_OK;
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, bf16* __restrict__ out, int64_t n) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n) {
        const float4 v = *reinterpret_cast<const float4*>(in + i);
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        *reinterpret_cast<__nv_bfloat162*>(out + i) = a;
        *reinterpret_cast<__nv_bfloat162*>(out + i + 2) = b;
    } else {
        for (int64_t k = i; k < n; ++k) out[k] = __float2bfloat16_rn(in[k]);
    }
}

}  // namespace
}  // namespace pbsa

using namespace pbsa;

extern "C" {

int pbsa_pbt1_write(const char* path, const float* data, int rank, const uint64_t* dims) {
    if (rank < 0 || rank > 255 || (rank > 0 && dims == nullptr)) return set_error(PBSA_EINVAL, "pbt1_write: bad rank/dims");
    uint64_t n = rank == 0 ? 0 : 1;
    for (int i = 0; i < rank; ++i) n *= dims[i];
    if (n > 0 && data == nullptr) return set_error(PBSA_EINVAL, "pbt1_write: null data");
    File fh;
    fh.f = path ? std::fopen(path, "wb") : nullptr;
    if (!fh.f) return io_error("OpenFailed", std::string("cannot open for write: ") + (path ? path : "(null)"));
    bool ok = std::fwrite(kMagic, 1, 4, fh.f) == 4;
    const unsigned char dr[2] = {kDtypeF32, static_cast<unsigned char>(rank)};
    ok = ok && std::fwrite(dr, 1, 2, fh.f) == 2;
    for (int i = 0; i < rank && ok; ++i) {
        unsigned char b[8];
        for (int k = 0; k < 8; ++k) b[k] = static_cast<unsigned char>((dims[i] >> (8 * k)) & 0xff);
        ok = std::fwrite(b, 1, 8, fh.f) == 8;
    }
    if (ok && n) ok = std::fwrite(data, sizeof(float), n, fh.f) == n;  // little-endian IEEE-754 hosts
    if (!ok) return io_error("OpenFailed", std::string("short write: ") + path);
    return PBSA_OK;
}

int pbsa_pbt1_info(const char* path, int* rank, uint64_t* dims, int max_rank) {
    if (rank == nullptr || (max_rank > 0 && dims == nullptr)) return set_error(PBSA_EINVAL, "pbt1_info: null output");
    File fh;
    if (int rc = open_read(&fh, path)) return rc;
    std::vector<uint64_t> dv;
    uint64_t n = 0;
    if (int rc = read_header(fh.f, path, &dv, &n)) return rc;
    if (static_cast<int>(dv.size()) > max_rank) return set_error(PBSA_EINVAL, "pbt1_info: dims buffer too small");
    *rank = static_cast<int>(dv.size());
    for (std::size_t i = 0; i < dv.size(); ++i) dims[i] = dv[i];
    return PBSA_OK;
}

int pbsa_pbt1_read(const char* path, float* out, uint64_t capacity) {
    File fh;
    if (int rc = open_read(&fh, path)) return rc;
    std::vector<uint64_t> dv;
    uint64_t n = 0;
    if (int rc = read_header(fh.f, path, &dv, &n)) return rc;
    if (n > capacity) return set_error(PBSA_EINVAL, "pbt1_read: output capacity too small");
    if (n && (out == nullptr || std::fread(out, sizeof(float), n, fh.f) != n))
        return io_error("Truncated", std::string("truncated payload: ") + path);
    return check_trailing(fh.f, path);
}

int pbsa_pbt1_load_bf16(const char* path, void* dst, uint64_t capacity, void* stream) {
    File fh;
    if (int rc = open_read(&fh, path)) return rc;
    std::vector<uint64_t> dv;
    uint64_t n = 0;
    if (int rc = read_header(fh.f, path, &dv, &n)) return rc;
    if (n > capacity) return set_error(PBSA_EINVAL, "pbt1_load_bf16: destination capacity too small");
    if (n == 0) return check_trailing(fh.f, path);
    if (dst == nullptr || (reinterpret_cast<uintptr_t>(dst) & 15) != 0)
        return set_error(PBSA_EINVAL, "pbt1_load_bf16: destination must be 16-byte aligned");
    cudaStream_t s = as_stream(stream);
    constexpr uint64_t kPiece = uint64_t(2) << 20;  // floats per piece (8 MB)
    const uint64_t piece = n < kPiece ? n : kPiece;
    float* host[2] = {nullptr, nullptr};
    float* dev = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};
    int rc = PBSA_OK;
    auto fail = [&](const std::string& m) { rc = set_error(PBSA_ECUDA, "pbt1_load_bf16: " + m); };
    if (cudaMallocHost(&host[0], piece * 4) != cudaSuccess || cudaMallocHost(&host[1], piece * 4) != cudaSuccess ||
        cudaMallocAsync(reinterpret_cast<void**>(&dev), 2 * piece * 4, s) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming) != cudaSuccess)
        fail("staging allocation failed");
    for (uint64_t off = 0, it = 0; rc == PBSA_OK && off < n; off += piece, ++it) {
        const int bsel = static_cast<int>(it & 1);
        const uint64_t cnt = (n - off) < piece ? (n - off) : piece;
        if (it >= 2 && cudaEventSynchronize(done[bsel]) != cudaSuccess) {  // this host buffer's copy is done
            fail("stream error");
            break;
        }
        if (std::fread(host[bsel], sizeof(float), cnt, fh.f) != cnt) {
            rc = io_error("Truncated", std::string("truncated payload: ") + path);
            break;
        }
        float* dbuf = dev + bsel * piece;
        if (cudaMemcpyAsync(dbuf, host[bsel], cnt * 4, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            fail("H2D copy failed");
            break;
        }
        const int64_t threads = (static_cast<int64_t>(cnt) + 3) / 4;
        count_launch();
        f32_to_bf16_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
            dbuf, static_cast<bf16*>(dst) + off, static_cast<int64_t>(cnt));
        if (cudaGetLastError() != cudaSuccess || cudaEventRecord(done[bsel], s) != cudaSuccess) fail("convert launch failed");
    }
    if (rc == PBSA_OK) rc = check_trailing(fh.f, path);
    cudaStreamSynchronize(s);  // staging buffers are released below
    for (auto* h : host)
        if (h) cudaFreeHost(h);
    if (dev) cudaFreeAsync(dev, s);
    for (auto e : done)
        if (e) cudaEventDestroy(e);
    return rc;
}

}  // extern "C"
