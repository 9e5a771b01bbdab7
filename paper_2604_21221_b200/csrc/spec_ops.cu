// spec_ops.cu -- the reference's tensor-module primitives and the SPEC router / memory ops on plain
// device f32 matrices, for the drop-in C++ API (include/pbsa/tensor.hpp, blockify.hpp,
// pbsa_b200.hpp).  The fused hot path (K1-K4) never calls these; they exist so that a caller of the
// reference's free functions gets the same results from the GPU:
//
//   matmul / matmul_nt      tensor.cpp:8-55    fp64 accumulation in ascending k, one fp32 rounding
//   masked_softmax_rows     tensor.cpp:57-108  fp32 row max, fp64 exp(s - max), ascending fp64
//                                              denominator, fp32 e / denom; fully masked row -> 0
//   select_topk             SPEC.md:295-303    k largest per row, (value desc, index asc)
//   aggregate_scores        SPEC.md:286-294    ascending-row fp64 column sums / rows
//   blockify / unblockify   blockify.cpp:38-96 (t, h, w, d) <-> block-major (n_b, b, d)
//   update_persistent       SPEC.md:200-208    Top-(C-|S|) of the candidates by (score desc, id asc)
//
// fp32 x fp32 products are exact in fp64, so an fp64 FMA chain equals the reference's
// `acc += double(a) * double(b)` bit for bit.  The exp is CUDA's fp64 exp (<= 1 ulp, as glibc's);
// see DESIGN.md section 2 for the residual-risk argument.
//
// Roofline: none of these is on the hot path; matmul is FP64-bound, the rest HBM/latency-bound.
#include <cfloat>
#include <cmath>

#include "internal.h"
#include "ptx.cuh"
#include "select_warp.cuh"

namespace pbsa {
namespace {

constexpr int kMT = 16;  // output tile 16 x 16, one thread per output element
constexpr int kKT = 32;  // k chunk staged in shared memory

// c[i][j] = float(sum_k double(a[i][k]) * double(b(k, j))) * scale, b(k, j) = bt ? b[j][k] : b[k][j]
__global__ void __launch_bounds__(kMT * kMT) matmul_f64acc_kernel(const float* __restrict__ a,
                                                                   const float* __restrict__ b, int n, int kd, int m,
                                                                   int bt, float scale, float* __restrict__ c) {
    __shared__ double as[kMT][kKT + 1];
    __shared__ double bs[kKT][kMT + 1];
    const int tx = threadIdx.x % kMT, ty = threadIdx.x / kMT;
    const int i0 = blockIdx.y * kMT, j0 = blockIdx.x * kMT;
    double acc = 0.0;
    for (int k0 = 0; k0 < kd; k0 += kKT) {
        for (int e = threadIdx.x; e < kMT * kKT; e += kMT * kMT) {
            const int r = e / kKT, kk = e % kKT;
            const int i = i0 + r, k = k0 + kk;
            as[r][kk] = (i < n && k < kd) ? static_cast<double>(a[static_cast<int64_t>(i) * kd + k]) : 0.0;
            const int jj = e % kMT, kb = e / kMT;
            const int j = j0 + jj, k2 = k0 + kb;
            float bv = 0.0f;
            if (j < m && k2 < kd) bv = bt ? b[static_cast<int64_t>(j) * kd + k2] : b[static_cast<int64_t>(k2) * m + j];
            bs[kb][jj] = static_cast<double>(bv);
        }
        __syncthreads();
        const int kn = kd - k0 < kKT ? kd - k0 : kKT;
        for (int kk = 0; kk < kn; ++kk) acc = __fma_rn(as[ty][kk], bs[kk][tx], acc);  // ascending k
        __syncthreads();
    }
    const int i = i0 + ty, j = j0 + tx;
    if (i < n && j < m) c[static_cast<int64_t>(i) * m + j] = __fmul_rn(__double2float_rn(acc), scale);
}

// masked_softmax_rows: warp per row.  status bit 0: NaN in scores; bit 1: a mask entry that is
// neither 0 nor -inf (the reference rejects both before computing, tensor.cpp:59-72).
__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* __restrict__ s, const float* __restrict__ mask,
                                                           int rows, int cols, float* __restrict__ out,
                                                           int* __restrict__ status) {
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const float* sr = s + row * cols;
    const float* mr = mask ? mask + row * cols : nullptr;
    float* orow = out + row * cols;
    float mx = -INFINITY;
    int bad = 0;
    for (int j = lane; j < cols; j += 32) {
        const float v = sr[j];
        if (v != v) bad |= 1;
        bool masked = false;
        if (mr) {
            const float mv = mr[j];
            if (!(mv == 0.0f || mv == -INFINITY)) bad |= 2;
            masked = mv == -INFINITY;
        }
        const float x = masked ? -INFINITY : v;
        if (x > mx) mx = x;
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0 && status) atomicOr(status, bad);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (mx == -INFINITY) {  // fully masked (or empty) row: all-zero sentinel
        for (int j = lane; j < cols; j += 32) orow[j] = 0.0f;
        return;
    }
    const double dm = static_cast<double>(mx);
    auto e_of = [&](int j) -> double {
        if (mr && mr[j] == -INFINITY) return 0.0;
        return exp(static_cast<double>(sr[j]) - dm);
    };
    // ascending-j fp64 denominator: each 32-chunk's terms are computed in parallel and added in
    // index order by every lane (the same sum on all lanes, no scratch)
    double denom = 0.0;
    for (int base = 0; base < cols; base += 32) {
        const int j = base + lane;
        const double e = j < cols ? e_of(j) : 0.0;
        const int cnt = cols - base < 32 ? cols - base : 32;
        for (int t = 0; t < cnt; ++t) denom = __dadd_rn(denom, __shfl_sync(0xffffffffu, e, t));
    }
    for (int j = lane; j < cols; j += 32) orow[j] = __double2float_rn(__ddiv_rn(e_of(j), denom));
}

// order-preserving key of a float (-0 == +0; the NaN check is separate)
__device__ __forceinline__ uint32_t ord_key(float x) {
    if (x == 0.0f) x = 0.0f;
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(256) topk_keys_kernel(const float* __restrict__ a, int64_t total,
                                                        uint32_t* __restrict__ keys, int* __restrict__ status) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const float x = a[i];
    if (x != x && status) atomicOr(status, 1);
    keys[i] = x != x ? 0u : ord_key(x);
}

__global__ void __launch_bounds__(256) topk_select_kernel(const uint32_t* __restrict__ keys, int rows, int cols,
                                                          int k, int32_t* __restrict__ sel) {
    __shared__ uint32_t hist[8][256];
    const int warp = threadIdx.x >> 5;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (row >= rows) return;
    warp_topk(keys + row * cols, cols, k, hist[warp], sel + row * k);
}

// (t, h, w, d) <-> (n_b, b, d): thread per (token, 16-byte column group)
__global__ void blockify_kernel(const float* __restrict__ x, int t, int h, int w, int d, int bt, int bh, int bw,
                                float* __restrict__ y, int inverse) {
    const int64_t tok = blockIdx.x;  // source token (t, h, w) flat
    const int ti = static_cast<int>(tok / (static_cast<int64_t>(h) * w));
    const int hi = static_cast<int>((tok / w) % h), wi = static_cast<int>(tok % w);
    const int nh = h / bh, nw = w / bw;
    const int64_t bid = (static_cast<int64_t>(ti / bt) * nh + hi / bh) * nw + wi / bw;
    const int64_t inb = (static_cast<int64_t>(ti % bt) * bh + hi % bh) * bw + wi % bw;
    const int64_t dst = (bid * (static_cast<int64_t>(bt) * bh * bw) + inb) * d;
    const int64_t src = tok * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        if (inverse) y[src + c] = x[dst + c];
        else y[dst + c] = x[src + c];
    }
}

// update_persistent's ranking: keep[i] = candidate i is among the `slots` best by (score desc with
// NaN lowest, id asc) -- the rule K4 applies in place (mem_update.cu)
__global__ void __launch_bounds__(256) topc_keep_kernel(const int64_t* __restrict__ ids, const float* __restrict__ sc,
                                                        int n, int slots, uint8_t* __restrict__ keep,
                                                        int* __restrict__ status) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float si = sc[i];
        if (si != si && status) atomicOr(status, 1);
        int rank = 0;
        for (int j = 0; j < n; ++j) rank += topc_before(sc[j], ids[j], si, ids[i]);
        keep[i] = rank < slots ? 1 : 0;
    }
}

}  // namespace

int launch_matmul_f64acc(const float* a, const float* b, int n, int kd, int m, int bt, float scale, float* c,
                         cudaStream_t s) {
    if (n == 0 || m == 0) return 0;
    const dim3 grid((m + kMT - 1) / kMT, (n + kMT - 1) / kMT);
    launch_pdl(matmul_f64acc_kernel, grid, dim3(kMT * kMT), 0, s, a, b, n, kd, m, bt, scale, c);
    return check_launch("matmul_f64acc_kernel");
}

int launch_softmax_rows(const float* scores, const float* mask, int rows, int cols, float* out, int* status,
                        cudaStream_t s) {
    if (rows == 0) return 0;
    launch_pdl(softmax_rows_kernel, dim3((rows + 7) / 8), dim3(256), 0, s, scores, mask, rows, cols, out, status);
    return check_launch("softmax_rows_kernel");
}

int launch_select_topk(const float* a, int rows, int cols, int k, int32_t* sel, uint32_t* keys, int* status,
                       cudaStream_t s) {
    if (rows == 0 || k == 0) return 0;
    const int64_t total = static_cast<int64_t>(rows) * cols;
    launch_pdl(topk_keys_kernel, dim3(static_cast<unsigned>((total + 255) / 256)), dim3(256), 0, s, a, total, keys, status);
    if (int rc = check_launch("topk_keys_kernel")) return rc;
    launch_pdl(topk_select_kernel, dim3((rows + 7) / 8), dim3(256), 0, s, static_cast<const uint32_t*>(keys), rows, cols,
               k, sel);
    return check_launch("topk_select_kernel");
}

int launch_blockify(const float* x, int t, int h, int w, int d, int bt, int bh, int bw, float* y, int inverse,
                    cudaStream_t s) {
    const int64_t tokens = static_cast<int64_t>(t) * h * w;
    if (tokens == 0 || d == 0) return 0;
    launch_pdl(blockify_kernel, dim3(static_cast<unsigned>(tokens)), dim3(d < 256 ? ((d + 31) / 32) * 32 : 256), 0, s,
               x, t, h, w, d, bt, bh, bw, y, inverse);
    return check_launch("blockify_kernel");
}

int launch_topc_keep(const int64_t* ids, const float* scores, int n, int slots, uint8_t* keep, int* status,
                     cudaStream_t s) {
    if (n == 0) return 0;
    launch_pdl(topc_keep_kernel, dim3((n + 255) / 256), dim3(256), 0, s, ids, scores, n, slots, keep, status);
    return check_launch("topc_keep_kernel");
}

}  // namespace pbsa
