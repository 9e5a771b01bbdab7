// select_warp.cuh -- warp-level building blocks of the exact selections (K2 and the SPEC-op
// primitives): the oracle's row softmax (fp32 max, fp64 exp, ascending fp64 denominator,
// tensor.cpp:57-108) and the k largest of a row by (value desc, index asc).
// Included into the anonymous namespace of each user translation unit.
#pragma once
#include <cfloat>
#include <cstdint>

namespace pbsa {
namespace {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// masked_softmax_rows (no mask) of z[0..n) for one row, by one warp.  e[] is fp64 scratch.
// Writes the fp32 probabilities' bit patterns to out_bits (or floats to out_f).
__device__ void warp_softmax(const float* z, int n, double* e, uint32_t* out_bits, float* out_f) {
    const int lane = threadIdx.x & 31;
    float m = -FLT_MAX;
    for (int j = lane; j < n; j += 32) m = fmaxf(m, z[j]);
    m = warp_max(m);
    const double dm = static_cast<double>(m);
#pragma unroll 4
    for (int j = lane; j < n; j += 32) e[j] = exp(static_cast<double>(z[j]) - dm);  // independent: 4 in flight
    __syncwarp();
    double denom = 0.0;
    if (lane == 0) {  // ascending-j fp64 accumulation, exactly as tensor.cpp:96-102
        int j = 0;
        for (; j + 8 <= n; j += 8) {  // 16-byte loads issued ahead of the dependent adds
            const double2 a0 = *reinterpret_cast<const double2*>(e + j);
            const double2 a1 = *reinterpret_cast<const double2*>(e + j + 2);
            const double2 a2 = *reinterpret_cast<const double2*>(e + j + 4);
            const double2 a3 = *reinterpret_cast<const double2*>(e + j + 6);
            denom = __dadd_rn(denom, a0.x);
            denom = __dadd_rn(denom, a0.y);
            denom = __dadd_rn(denom, a1.x);
            denom = __dadd_rn(denom, a1.y);
            denom = __dadd_rn(denom, a2.x);
            denom = __dadd_rn(denom, a2.y);
            denom = __dadd_rn(denom, a3.x);
            denom = __dadd_rn(denom, a3.y);
        }
        for (; j < n; ++j) denom = __dadd_rn(denom, e[j]);
    }
    denom = __shfl_sync(0xffffffffu, denom, 0);
#pragma unroll 4
    for (int j = lane; j < n; j += 32) {
        const float p = __double2float_rn(__ddiv_rn(e[j], denom));
        if (out_bits) out_bits[j] = __float_as_uint(p);
        if (out_f) out_f[j] = p;
    }
    __syncwarp();
}

// 4-pass 8-bit radix select: the value of the k-th largest of pb[0..n) (unsigned order), and in
// *kk_out how many elements equal to it belong to the k largest.
__device__ uint32_t warp_kth(const uint32_t* pb, int n, int k, uint32_t* hist, int* kk_out) {
    const int lane = threadIdx.x & 31;
    uint32_t prefix = 0, pmask = 0;
    int kk = k;  // still to pick at/below the current prefix
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
        for (int t = 0; t < 8; ++t) hist[lane * 8 + t] = 0;
        __syncwarp();
        for (int base = 0; base < n; base += 32) {  // warp-aggregated: one atomic per distinct bin
            const int j = base + lane;
            const uint32_t v = j < n ? pb[j] : 0u;
            const bool in = j < n && (v & pmask) == prefix;
            const uint32_t bin = in ? ((v >> shift) & 255u) : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, bin);
            if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], static_cast<uint32_t>(__popc(peers)));
        }
        __syncwarp();
        // lane l owns digits [255-8l-7, 255-8l] (lane 0 the largest)
        uint32_t sum = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) sum += hist[255 - lane * 8 - t];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - sum;
        const bool mine = excl < static_cast<uint32_t>(kk) && static_cast<uint32_t>(kk) <= incl;
        uint32_t dgt = 0, above = 0;
        if (mine) {
            uint32_t cum = excl;
            for (int t = 0; t < 8; ++t) {
                const uint32_t bin = 255 - lane * 8 - t;
                const uint32_t h = hist[bin];
                if (cum + h >= static_cast<uint32_t>(kk)) {
                    dgt = bin;
                    above = cum;
                    break;
                }
                cum += h;
            }
        }
        const uint32_t who = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        dgt = __shfl_sync(0xffffffffu, dgt, who);
        above = __shfl_sync(0xffffffffu, above, who);
        kk -= static_cast<int>(above);
        prefix |= dgt << shift;
        pmask |= 255u << shift;
        __syncwarp();
    }
    *kk_out = kk;
    return prefix;
}

// Short rows (n <= 32 * NPL): the k-th largest by a 32-step binary search on the value, the row
// held in registers (NPL per lane) and each step one compare per value plus one warp reduction --
// no shared-memory histograms or match/atomic traffic.
template <int NPL>
__device__ uint32_t warp_kth_reg(const uint32_t* pb, int n, int k, int* kk_out) {
    const int lane = threadIdx.x & 31;
    uint32_t v[NPL];
#pragma unroll
    for (int i = 0; i < NPL; ++i) v[i] = lane + 32 * i < n ? pb[lane + 32 * i] : 0u;
    // (the padding values are 0, never >= a candidate, which always has a bit set, nor > t)
    uint32_t t = 0;  // largest value with at least k elements >= it
#pragma unroll 1
    for (int bit = 31; bit >= 0; --bit) {
        const uint32_t cand = t | (1u << bit);
        int c = 0;
#pragma unroll
        for (int i = 0; i < NPL; ++i) c += v[i] >= cand;
        if (static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<uint32_t>(c))) >= k) t = cand;
    }
    int gt = 0;
#pragma unroll
    for (int i = 0; i < NPL; ++i) gt += v[i] > t;
    *kk_out = k - static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<uint32_t>(gt)));
    return t;
}

// k largest of pb[0..n) (non-negative float bits => unsigned order), ties -> lower index.
// Writes the winners' indices ascending to out[0..k).
__device__ void warp_topk(const uint32_t* pb, int n, int k, uint32_t* hist, int32_t* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    int kk;
    const uint32_t prefix = n <= 128   ? warp_kth_reg<4>(pb, n, k, &kk)
                            : n <= 256 ? warp_kth_reg<8>(pb, n, k, &kk)
                            : n <= 384 ? warp_kth_reg<12>(pb, n, k, &kk)
                            : n <= 512 ? warp_kth_reg<16>(pb, n, k, &kk)
                                       : warp_kth(pb, n, k, hist, &kk);
    // prefix = value of the k-th largest element; take every element above it and the first kk
    // (lowest indices) equal to it.
    int run = 0, tie_run = 0;
    for (int base = 0; base < n; base += 32) {
        const int j = base + lane;
        const uint32_t v = j < n ? pb[j] : 0u;
        const bool gt = j < n && v > prefix;
        const bool eq = j < n && v == prefix;
        const uint32_t eb = __ballot_sync(0xffffffffu, eq);
        const int tie_rank = tie_run + __popc(eb & lt);
        const bool take = gt || (eq && tie_rank < kk);
        const uint32_t tb = __ballot_sync(0xffffffffu, take);
        const int pos = run + __popc(tb & lt);
        if (take && pos < k) out[pos] = j;
        run += __popc(tb);
        tie_run += __popc(eb);
    }
}

// Top-C order of update_persistent: candidate j ranks before candidate i by
// (score desc, id asc); NaN scores (invalid input, rejected by the reference) rank below every
// number, so the order stays total and exactly `slots` candidates survive.
__device__ __forceinline__ bool topc_before(float sj, int64_t idj, float si, int64_t idi) {
    sj = sj != sj ? -INFINITY : sj;
    si = si != si ? -INFINITY : si;
    return (sj > si) || (sj == si && idj < idi);
}

}  // namespace
}  // namespace pbsa
