// score_select.cu -- K2 coarse scoring, row-wise Top-K selection and score aggregation.
//
// Reference ops (Eq. 7-8, Eq. 10-11):
//   logits  z[i][j] = float(sum_c double(qc[i][c]) * double(kc[j][c]))  (tensor.cpp:34-55, ascending c)
//                     * scale                                           (fp32 multiply)
//   A_L     = masked_softmax_rows(z over the local keys)                 (tensor.cpp:57-108)
//   Omega   = k largest of A_L by (value desc, index asc), emitted ascending
//   k=0 pass: A_t = softmax over all keys, s_t[j] = float(sum_i double(A_t[i][j]) / nqb)
// Every rounding step is reproduced exactly (same operation order as the oracle), so the
// selected indices and s_t are bit-exact with oracle/pbsa_oracle.cpp.  The only transcendental
// is the fp64 exp; see DESIGN.md "bit-exactness" for the residual-risk argument.
//
// Kernels (short/medium key lists, e.g. config 2):
//   logits_rm_kernel     thread per key block x 8 query rows, ascending-c fp64 dot products
//   row_select_kernel    warp per row: softmax (fp64 exp, sequential ascending denominator on lane 0
//                        exactly like the oracle), 4-pass 8-bit radix select on the fp32 probability
//                        bits, ballot compaction of the winners; A_t rows at the k=0 pass
//   aggregate_kernel     thread per key block, ascending-row fp64 column sums (k=0 pass only)
// a key-major variant for long windows (config 5), and for denoise passes over long windows the
// certified fp32 ranking (logits32_kernel + cert_select_kernel), which reaches the same indices
// with exact fp64 work only for the keys near the k-th boundary.
#include <cfloat>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"
#include "select_warp.cuh"

namespace pbsa {
namespace {

struct ScoreParams {
    const float* qc;      // [U][nqb][D]
    const float* krep;    // [U][...][D] (slot-indexed)
    int64_t kru;
    const int32_t* keys;  // [U][key_stride]
    int key_stride, n_keys, local_off, n_local, k, nqb, units, rows;
    float scale;
    size_t per_warp;      // bytes of smem per row (16-aligned)
    int32_t* sel;         // [U][nqb][k]
    float* arows;         // [U][nqb][n_keys] or null
    int* status;          // nullable: bit 0 set when a logit row holds NaN (invalid input)
    int qc_rows = 0, qc_row0 = 0;  // qc is [U][qc_rows][D]; row i of the launch is qc row qc_row0 + i
    // flat index of row i of unit u in qc (times D = its offset)
    __device__ __forceinline__ int64_t qidx(int u, int i) const {
        return static_cast<int64_t>(u) * qc_rows + qc_row0 + i;
    }
};

constexpr int kMaxRows = 8;

// ---------------------------------------------------------------------------------------------
// Short/medium key lists (config 2: 312 / 546 keys): two launches with full-machine parallelism.
//   logits_rm_kernel  CTA = unit x 8 query rows x 32 keys; the key tile is staged once in shared
//                     memory as fp64 (transposed, key index fastest) and the 8 query rows as fp64;
//                     warp = row, lane = key: one ascending-c fp64 dot product per thread.
//                     Row-major logits z[U][nqb][n_keys] go to the workspace (L2-resident).
//   row_select_kernel warp per row: the oracle's softmax + radix Top-K (+ the full-row A_t of the
//                     k=0 pass) straight from z.
constexpr int kLogitKeys = 128;  // keys (= threads) per CTA

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
                 "l"(gsrc)
                 : "memory");
}

// Thread = key, 8 query rows per thread (8 independent ascending-c fp64 chains, each key element
// converted once).  The CTA's 128 key rows are staged with cp.async into shared memory, 16-byte
// chunk c4 of key j stored at chunk c4 ^ (j & 7): the staging stores and the per-thread LDS.128
// row reads are both bank-conflict free.  Query rows are fp64 broadcasts.
template <int D>
__global__ void __launch_bounds__(kLogitKeys) logits_rm_kernel(const ScoreParams p, float* __restrict__ z) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(16) uint8_t smem[];
    double* qs = reinterpret_cast<double*>(smem);                            // [kMaxRows][D]
    float4* ks = reinterpret_cast<float4*>(smem + kMaxRows * D * 8);         // [kLogitKeys][D/4] swizzled
    constexpr int C4 = D / 4;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = blockIdx.z, i0 = blockIdx.y * kMaxRows, j0 = blockIdx.x * kLogitKeys;
    const int nr = min(kMaxRows, p.nqb - i0);
    const int nk = min(kLogitKeys, p.n_keys - j0);
    // every load is issued before any is waited on: slot ids (one per thread), then the key rows
    // (warp w copies rows w, w+4, ...) and the query rows
    const int my_slot = tid < nk ? __ldg(p.keys + static_cast<int64_t>(u) * p.key_stride + j0 + tid) : 0;
    {
        __shared__ int slots[kLogitKeys];
        slots[tid] = my_slot;
        __syncthreads();
#pragma unroll 4
        for (int kk = warp; kk < nk; kk += kLogitKeys / 32) {
            const float4* kr = reinterpret_cast<const float4*>(p.krep + u * p.kru + static_cast<int64_t>(slots[kk]) * D);
            for (int c4 = lane; c4 < C4; c4 += 32) cp_async16(ks + kk * C4 + (c4 ^ (kk & 7)), kr + c4);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    {
        constexpr int Q4 = kMaxRows * D / 4;
        float4 qv[Q4 / kLogitKeys];
#pragma unroll
        for (int t = 0; t < Q4 / kLogitKeys; ++t) {
            const int e4 = tid + t * kLogitKeys, r = (e4 * 4) / D;
            qv[t] = r < nr ? __ldg(reinterpret_cast<const float4*>(p.qc + p.qidx(u, i0) * D) + e4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < Q4 / kLogitKeys; ++t) {
            const int e4 = tid + t * kLogitKeys;
            qs[4 * e4] = qv[t].x;
            qs[4 * e4 + 1] = qv[t].y;
            qs[4 * e4 + 2] = qv[t].z;
            qs[4 * e4 + 3] = qv[t].w;
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (tid >= nk) return;
    double acc[kMaxRows];
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r) acc[r] = 0.0;
    const float4* krow = ks + tid * C4;
#pragma unroll 2
    for (int c4 = 0; c4 < C4; ++c4) {
        const float4 kv = krow[c4 ^ (tid & 7)];
        const double k0 = kv.x, k1 = kv.y, k2 = kv.z, k3 = kv.w;
#pragma unroll
        for (int r = 0; r < kMaxRows; ++r) {  // ascending c per row; fp32 x fp32 is exact in fp64
            const double2 qa = *reinterpret_cast<const double2*>(qs + r * D + 4 * c4);
            const double2 qb = *reinterpret_cast<const double2*>(qs + r * D + 4 * c4 + 2);
            acc[r] = __fma_rn(qa.x, k0, acc[r]);
            acc[r] = __fma_rn(qa.y, k1, acc[r]);
            acc[r] = __fma_rn(qb.x, k2, acc[r]);
            acc[r] = __fma_rn(qb.y, k3, acc[r]);
        }
    }
    const int64_t zr = (static_cast<int64_t>(u) * p.nqb + i0) * p.n_keys + j0 + tid;
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r)
        if (r < nr) z[zr + static_cast<int64_t>(r) * p.n_keys] = __fmul_rn(__double2float_rn(acc[r]), p.scale);
}

// split = 2 (k=0 pass with selection): warps w and w+4 share row w -- one runs the local-window
// softmax + Top-K, the other the full-row softmax (A_t): the two sequential fp64 denominators run
// concurrently instead of back to back.
template <int SPLIT>
__global__ void __launch_bounds__(256) row_select_kernel(const ScoreParams p, const float* __restrict__ z) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kRowsPerCta = kMaxRows / SPLIT;
    const int role = SPLIT == 2 ? warp / kRowsPerCta : 0;  // 0: selection (and A_t if SPLIT == 1), 1: A_t
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + warp % kRowsPerCta;
    if (row >= static_cast<int64_t>(p.units) * p.nqb) return;
    const int n = p.n_keys;
    uint8_t* base = smem + p.per_warp * warp;
    double* e = reinterpret_cast<double*>(base);
    float* zr = reinterpret_cast<float*>(base + static_cast<size_t>(n) * 8);
    uint32_t* pb = reinterpret_cast<uint32_t*>(zr + ((n + 3) & ~3));
    uint32_t* hist = pb + p.n_local;
    // the row's logits into shared memory (all loads in flight at once; rows are n*4 bytes apart,
    // 16-byte aligned when n % 4 == 0)
    const float* zg = z + row * n;
    bool bad = false;
    if ((n & 3) == 0) {
        const float4* z4 = reinterpret_cast<const float4*>(zg);
        float4* s4 = reinterpret_cast<float4*>(zr);
#pragma unroll 4
        for (int j = lane; j < n / 4; j += 32) s4[j] = __ldg(z4 + j);
    } else {
#pragma unroll 4
        for (int j = lane; j < n; j += 32) zr[j] = __ldg(zg + j);
    }
    __syncwarp();
    for (int j = lane; j < n; j += 32) {
        const float v = zr[j];
        bad |= v != v;
    }
    if (p.status != nullptr && role == 0 && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.status, 1);
    if (role == 0 && p.k > 0 && p.n_local > 0) {
        warp_softmax(zr + p.local_off, p.n_local, e, pb, nullptr);
        warp_topk(pb, p.n_local, p.k, hist, p.sel + row * p.k);
    }
    if (p.arows != nullptr && (SPLIT == 1 || role == 1)) warp_softmax(zr, n, e, nullptr, p.arows + row * n);
}

// ---------------------------------------------------------------------------------------------
// Denoise passes (selection only, no A_t): certified fp32 ranking.
// Only the INDICES of the k largest local-window probabilities are needed, and p_j =
// float(e_j / denom) is non-decreasing in the exact logit z_j, so the selection is the top-k by z
// except where keys at the k-th boundary round to the same fp32 probability (then the lower index
// wins).  logits32_kernel computes fp32 logits z~ with the rigorous bound
//   |z~_j - z_j| <= eps_j = scale * gamma_D * |q| * |k_j| + 2^-21 |z~_j|,  gamma_D = D * 2^-24 * 1.01
// (fp32 FMA dot-product error, Cauchy-Schwarz, and the two fp32 roundings of the oracle's
// float(dot64) * scale); cert_select_kernel radix-selects the k-th largest z~ (T), takes every key
// above T + 2 eps_max + tau, drops every key below T - 2 eps_max - tau, recomputes the oracle's exact
// logit (ascending-c fp64 dot, same roundings) for the few keys in between and ranks those exactly.
// tau = 2^-22: two logits further apart than tau give probabilities whose ratio exceeds
// exp(2^-22) > 1 + 2^-22, i.e. at least 2 fp32 ulps apart for normal fp32 (relative ulp <= 2^-23;
// the fp64 quotient e / denom adds only 2^-53), so they cannot round to one fp32 value and no
// probability tie can cross the boundary.  A row reruns the oracle's exact softmax + Top-K (warp_softmax / warp_topk, fp64
// scratch in global memory) when (a) the exact gap at the boundary is <= tau, (b) boundary
// probabilities could be subnormal (T - max z < -60), (c) more than kCertAmb keys are ambiguous,
// (d) a logit is NaN, or (e) an exact logit falls outside its certified interval (status bit 2 --
// never expected; a canary for the bound).
constexpr int kCertAmb = 256;  // = kCertThreads: one ambiguous key per thread
constexpr float kTau = 2.384185791015625e-07f;  // 2^-22

// CTA = 128 keys x up to 80 query rows; warp = 8 rows, lane = 4 keys (32 fp32 accumulators): per
// 16-byte chunk a warp issues 4 key LDS.128 + 8 broadcast query LDS.128 for 128 FFMAs, so the FMA
// pipe, not shared memory, is the limit.  Key chunk c4 of key j is stored at c4 ^ ((j >> 2) & 7):
// the lanes of a quarter-warp (keys 4l + t) hit 8 distinct 16-byte bank groups.  The key tile is
// staged once for all of a unit's rows (80 >= nqb for the configs), so krep is read from L2 once.
constexpr int kL32Warps = 10;  // 80 rows

template <int D>
__global__ void __launch_bounds__(kL32Warps * 32) logits32_kernel(const ScoreParams p, float* __restrict__ z,
                                                                  float* __restrict__ knorm) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr int C4 = D / 4;
    float4* ks = reinterpret_cast<float4*>(smem);                               // [128][C4] swizzled
    float4* qs = reinterpret_cast<float4*>(smem + kLogitKeys * D * 4);          // [80][C4]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = blockIdx.z, i0 = blockIdx.y * kL32Warps * 8, j0 = blockIdx.x * kLogitKeys;
    const int n = p.n_local;
    const int nr = min(kL32Warps * 8, p.nqb - i0);
    const int nk = min(kLogitKeys, n - j0);
    __shared__ int slots[kLogitKeys];
    if (tid < kLogitKeys)
        slots[tid] = tid < nk ? __ldg(p.keys + static_cast<int64_t>(u) * p.key_stride + p.local_off + j0 + tid) : 0;
    __syncthreads();
    for (int kk = warp; kk < nk; kk += kL32Warps) {
        const float4* kr = reinterpret_cast<const float4*>(p.krep + u * p.kru + static_cast<int64_t>(slots[kk]) * D);
        for (int c4 = lane; c4 < C4; c4 += 32) cp_async16(ks + kk * C4 + (c4 ^ ((kk >> 2) & 7)), kr + c4);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float4* qg = reinterpret_cast<const float4*>(p.qc + p.qidx(u, i0) * D);
    for (int e4 = tid; e4 < nr * C4; e4 += kL32Warps * 32) qs[e4] = __ldg(qg + e4);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int r0 = warp * 8;
    if (r0 >= nr) return;
    float acc[8][4], ss[4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[r][t] = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) ss[t] = 0.f;
    const bool norms = blockIdx.y == 0 && warp == 0;
    const int kb = 4 * lane;  // this lane's first key; all four share (key >> 2) & 7 = lane & 7
    const int sw = lane & 7;
#pragma unroll 2
    for (int c4 = 0; c4 < C4; ++c4) {
        float4 kv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) kv[t] = ks[(kb + t) * C4 + (c4 ^ sw)];
        if (norms) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                ss[t] = fmaf(kv[t].w, kv[t].w, fmaf(kv[t].z, kv[t].z, fmaf(kv[t].y, kv[t].y, fmaf(kv[t].x, kv[t].x, ss[t]))));
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const float4 qv = qs[min(r0 + r, nr - 1) * C4 + c4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                acc[r][t] = fmaf(qv.w, kv[t].w, fmaf(qv.z, kv[t].z, fmaf(qv.y, kv[t].y, fmaf(qv.x, kv[t].x, acc[r][t]))));
        }
    }
    if (norms) {  // per-CTA max key norm: cert_select bounds every key of the unit by the unit max
        float m = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) m = kb + t < nk ? fmaxf(m, ss[t]) : m;
        m = warp_max(m);
        if (lane == 0) knorm[static_cast<int64_t>(u) * gridDim.x + blockIdx.x] = sqrtf(m);
    }
    if (kb >= nk) return;
    const int n4 = (n + 3) & ~3;  // row stride: 16-byte rows (the tail pads are never read as keys)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        if (r0 + r >= nr) break;
        float4 o;
        o.x = __fmul_rn(acc[r][0], p.scale);
        o.y = __fmul_rn(acc[r][1], p.scale);
        o.z = __fmul_rn(acc[r][2], p.scale);
        o.w = __fmul_rn(acc[r][3], p.scale);
        *reinterpret_cast<float4*>(z + (static_cast<int64_t>(u) * p.nqb + i0 + r0 + r) * n4 + j0 + kb) = o;
    }
}

__device__ __forceinline__ uint32_t f2key(float v) {  // float -> unsigned, order preserving
    const uint32_t b = __float_as_uint(v);
    return b ^ ((b >> 31) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) { return __uint_as_float((k >> 31) ? k ^ 0x80000000u : ~k); }

// The oracle's logit for query row q and key slot `slot`: float(ascending-c fp64 dot) * scale.
template <int D>
__device__ __forceinline__ float exact_logit(const float* q, const float* krep, int64_t slot, float scale) {
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const float4* k4 = reinterpret_cast<const float4*>(krep + slot * D);
    double acc = 0.0;
#pragma unroll 8
    for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 a = __ldg(q4 + c4), b = __ldg(k4 + c4);
        acc = __fma_rn(static_cast<double>(a.x), static_cast<double>(b.x), acc);
        acc = __fma_rn(static_cast<double>(a.y), static_cast<double>(b.y), acc);
        acc = __fma_rn(static_cast<double>(a.z), static_cast<double>(b.z), acc);
        acc = __fma_rn(static_cast<double>(a.w), static_cast<double>(b.w), acc);
    }
    return __fmul_rn(__double2float_rn(acc), scale);
}

// CTA (256 threads) per row, the row's z~ held in registers: warp w, lane l, vector i holds keys
// (w*V4 + i)*128 + 4l .. +3 (one 16-byte load each; row stride n4 = n rounded up to 4), so every pass
// below is register work and a warp owns a contiguous key range (ascending emission by warp scans).
// One 1024-bin histogram over [min z~, max z~] (a monotone map, so whole bins are ordered) finds the
// bin b* holding the k-th largest z~; at config 5 (6006 keys, N(0,1)-like logits) b* holds ~15 keys.
// mode 2 forces the exact fallback (tests).
constexpr int kCertThreads = 256;
constexpr int kCertBins = 1024;
constexpr int kCertWarps = kCertThreads / 32;
constexpr int kCertMaxKeys = 8 * 4 * kCertThreads;  // V4 <= 8

// exclusive prefix over the block of v (returns it; *total = block sum); red[kCertWarps] scratch
__device__ __forceinline__ int block_scan(int v, int* red, int* total) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    int base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kCertWarps; ++w) {
        base += w < warp ? red[w] : 0;
        tot += red[w];
    }
    *total = tot;
    return base + incl - v;
}

__device__ __forceinline__ int block_sum(int v, int* red) {
    int tot;
    block_scan(v, red, &tot);
    return tot;
}

template <int D, int V4>
__global__ void __launch_bounds__(kCertThreads, 3) cert_select_kernel(const ScoreParams p, float* __restrict__ z,
                                                                   const float* __restrict__ kpart, int nparts,
                                                                   int n4, double* __restrict__ escr,
                                                                   int64_t escr_stride, int mode) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    __shared__ uint32_t hist[kCertBins];
    __shared__ uint32_t chosen[kCertMaxKeys / 32];
    __shared__ int red[kCertWarps];
    __shared__ float redf[2][kCertWarps];
    __shared__ int pick[4];
    __shared__ int cnt;
    __shared__ int wcnt[kCertWarps];
    __shared__ float bound[2];
    __shared__ double denom_s;
    __shared__ int32_t amb[kCertAmb];
    __shared__ float zamb[kCertAmb];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t row = blockIdx.x;
    const int n = p.n_local, k = p.k;
    const int u = static_cast<int>(row / p.nqb);
    float* zg = z + row * n4;
    const float* q = p.qc + p.qidx(u, static_cast<int>(row - static_cast<int64_t>(u) * p.nqb)) * D;
    const int32_t* slots = p.keys + static_cast<int64_t>(u) * p.key_stride + p.local_off;
    const float* kr = p.krep + u * p.kru;
    int32_t* out = p.sel + row * k;
    const int jw = warp * V4 * 128 + 4 * lane;  // key of (vector 0, component 0); vector i adds 128 i

    float v[V4][4];
#pragma unroll
    for (int i = 0; i < V4; ++i) {
        const int j = jw + 128 * i;
        const float4 x = j < n ? *reinterpret_cast<const float4*>(zg + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[i][0] = x.x;
        v[i][1] = x.y;
        v[i][2] = x.z;
        v[i][3] = x.w;
    }
    for (int b = tid; b < kCertBins; b += kCertThreads) hist[b] = 0;
    for (int b = tid; b < kCertMaxKeys / 32; b += kCertThreads) chosen[b] = 0;
    if (tid < kCertWarps) wcnt[tid] = 0;
    if (tid == 0) cnt = 0;
    // every warp: |q|^2 (D/32 values per lane) and the unit's largest key norm (nparts CTA maxima)
    float qq = 0.f, kmax = 0.f;
    for (int c = lane; c < D; c += 32) qq = fmaf(q[c], q[c], qq);
    for (int i = lane; i < nparts; i += 32) kmax = fmaxf(kmax, __ldg(kpart + static_cast<int64_t>(u) * nparts + i));
    float zmax = -FLT_MAX, zmin = FLT_MAX;
    int bad = 0;
    // warp-uniform: every key this warp holds is < n (all warps but the row's last partial one)
    const bool full = (warp + 1) * V4 * 128 <= n;
    if (!full) {  // pad the missing keys with copies of key 0 (present in every row): they change
                  // neither the maximum nor the minimum, and are skipped by index below
        const float v0 = zg[0];
#pragma unroll
        for (int i = 0; i < V4; ++i)
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (jw + 128 * i + t >= n) v[i][t] = v0;
    }
#pragma unroll
    for (int i = 0; i < V4; ++i)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            bad |= v[i][t] != v[i][t];
            zmax = fmaxf(zmax, v[i][t]);
            zmin = fminf(zmin, v[i][t]);
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
    kmax = warp_max(kmax);
    zmax = warp_max(zmax);
    zmin = -warp_max(-zmin);
    if (lane == 0) {
        redf[0][warp] = zmax;
        redf[1][warp] = zmin;
    }
    bad = block_sum(bad, red);  // (its barriers also publish the zeroed counters and redf)
    zmax = -FLT_MAX;
    zmin = FLT_MAX;
#pragma unroll
    for (int w = 0; w < kCertWarps; ++w) {
        zmax = fmaxf(zmax, redf[0][w]);
        zmin = fminf(zmin, redf[1][w]);
    }
    // eps for every key: scale * gamma_D * |q| * max|k| + 2^-21 max|z~| (norms rounded up by 2^-12,
    // far above their fp32 error; the whole bound by 1 %)
    const float emax = fmaf(p.scale * (static_cast<float>(D) * 5.9604645e-8f * 1.01f) * (sqrtf(qq) * 1.000244140625f),
                            kmax * 1.000244140625f, fmaxf(fabsf(zmax), fabsf(zmin)) * 4.76837158203125e-07f) *
                           1.01f + 1e-30f;
    bool fallback = mode == 2 || bad != 0;
    if (!fallback) {
        // bin(x) is non-decreasing in x (fsub, fmul, truncation and min are monotone)
        const float inv = static_cast<float>(kCertBins) / (zmax - zmin);
        auto bin = [&](float x) { return min(kCertBins - 1, static_cast<int>((x - zmin) * inv)); };
        if (full) {
#pragma unroll
            for (int i = 0; i < V4; ++i)
#pragma unroll
                for (int t = 0; t < 4; ++t) atomicAdd(&hist[bin(v[i][t])], 1u);
        } else {
#pragma unroll
            for (int i = 0; i < V4; ++i)
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (jw + 128 * i + t < n) atomicAdd(&hist[bin(v[i][t])], 1u);
        }
        __syncthreads();
        // thread t owns bins 1023-4t .. 1020-4t (descending)
        int c4[4], sum4 = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            c4[t] = static_cast<int>(hist[kCertBins - 1 - 4 * tid - t]);
            sum4 += c4[t];
        }
        int tot;
        int above = block_scan(sum4, red, &tot);
        if (above < k && k <= above + sum4) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (above < k && k <= above + c4[t]) {
                    pick[0] = kCertBins - 1 - 4 * tid - t;  // b*: the bin of the k-th largest z~
                    pick[1] = above;                        // keys in bins above b*
                }
                above += c4[t];
            }
        }
        // Two z~ at most `band` apart are at most m bins apart (the bin map's rounding moves a value
        // by < 1e-3 bins), so keys more than m bins above b* exceed every key of b* (the k-th largest
        // included) by more than band, and keys more than m bins below fall short by more.
        const float band = 2.f * emax + kTau;
        const int m = static_cast<int>(fminf(band * inv + 0.001f, 1.0e6f)) + 1;
        __syncthreads();
        const int bstar = pick[0];
        if (tid == 0) {
            int na = 0, mid_above = 0;
            if (m <= 32) {
                for (int b = max(0, bstar - m); b <= min(kCertBins - 1, bstar + m); ++b) {
                    na += static_cast<int>(hist[b]);
                    mid_above += b > bstar ? static_cast<int>(hist[b]) : 0;
                }
            } else {
                na = kCertAmb + 1;
            }
            pick[2] = na;
            pick[3] = pick[1] - mid_above;  // certainly in: keys more than m bins above b*
        }
        __syncthreads();
        const int na = pick[2], nin = pick[3];
        const int r = k - nin;  // slots left for the ambiguous keys (1 <= r <= na by construction)
        const int blo = bstar - m, bhi = bstar + m;
        fallback = na > kCertAmb || r < 1 || r > na;
        if (!fallback) {
            // classification: per-warp count of the certain keys, list of the ambiguous ones
            int nt = 0;
#pragma unroll
            for (int i = 0; i < V4; ++i)
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int j = jw + 128 * i + t;
                    const int bj = bin(v[i][t]);
                    if (full || j < n) {
                        nt += bj > bhi;
                        if (bj >= blo && bj <= bhi) amb[atomicAdd(&cnt, 1)] = j;
                    }
                }
#pragma unroll
            for (int o = 16; o; o >>= 1) nt += __shfl_xor_sync(0xffffffffu, nt, o);
            if (lane == 0) atomicAdd(&wcnt[warp], nt);
            __syncthreads();
            int off = 0;  // exact logit outside its certified interval
            float zlo = FLT_MAX;
            if (tid < na) {
                const int j = amb[tid];
                const float ze = exact_logit<D>(q, kr, slots[j], p.scale);
                zamb[tid] = ze;
                zlo = ze;
                off = !(fabsf(ze - zg[j]) <= emax);
            }
            if (tid < 2) bound[tid] = tid == 0 ? FLT_MAX : -FLT_MAX;
            zlo = -warp_max(-zlo);
            if (lane == 0) redf[0][warp] = zlo;
            off = block_sum(off, red);
#pragma unroll
            for (int w = 0; w < kCertWarps; ++w) zlo = fminf(zlo, redf[0][w]);
            // rank the ambiguous keys by (exact logit desc, index asc): equal logits are equal
            // probabilities, whose order the oracle breaks by index too
            int rank = 0;
            if (tid < na) {
                const float za = zamb[tid];
                const int ja = amb[tid];
                for (int o = 0; o < na; ++o) {
                    const float zo = zamb[o];
                    rank += zo > za || (zo == za && amb[o] < ja);
                }
                if (rank == r - 1) bound[0] = za;  // last in
                if (rank == r) bound[1] = za;      // first out
            }
            __syncthreads();
            if (off && tid == 0 && p.status != nullptr) atomicOr(p.status, 4);
            // a selected and an unselected ambiguous key with distinct logits at most tau apart could
            // share one fp32 probability (then the lower index wins, not the larger logit)
            int near = 0;
            if (tid < na) {
                const float za = zamb[tid];
                near = rank < r ? (za > bound[1] && za - bound[1] <= kTau) : (za < bound[0] && bound[0] - za <= kTau);
            }
            near = block_sum(near, red);
            // (b): boundary probabilities that could be subnormal are resolved exactly as well
            const bool resolve = near != 0 || zlo - (zmax + emax) < -60.f;
            fallback = off != 0;
            if (!fallback && resolve) {
                // exact probabilities of the ambiguous keys: the oracle's logits of the whole row
                // (for its max and the ascending fp64 denominator), then re-rank by (p desc, index asc)
                float zm = -FLT_MAX;
                for (int j = tid; j < n; j += kCertThreads) {
                    const float ze = exact_logit<D>(q, kr, slots[j], p.scale);
                    zg[j] = ze;
                    zm = fmaxf(zm, ze);
                }
                zm = warp_max(zm);
                if (lane == 0) redf[1][warp] = zm;
                __syncthreads();
#pragma unroll
                for (int w = 0; w < kCertWarps; ++w) zm = fmaxf(zm, redf[1][w]);
                double* e = escr + row * escr_stride;
                const double dm = static_cast<double>(zm);
                for (int j = tid; j < n; j += kCertThreads) e[j] = exp(static_cast<double>(zg[j]) - dm);
                __syncthreads();
                if (tid == 0) {  // ascending-j fp64 accumulation, exactly as tensor.cpp:96-102
                    double denom = 0.0;
                    int j = 0;
                    for (; j + 8 <= n; j += 8) {
                        double t8[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) t8[t] = e[j + t];
#pragma unroll
                        for (int t = 0; t < 8; ++t) denom = __dadd_rn(denom, t8[t]);
                    }
                    for (; j < n; ++j) denom = __dadd_rn(denom, e[j]);
                    denom_s = denom;
                }
                __syncthreads();
                if (tid < na) zamb[tid] = __double2float_rn(__ddiv_rn(e[amb[tid]], denom_s));
                __syncthreads();
                rank = 0;
                if (tid < na) {
                    const float pa = zamb[tid];
                    const int ja = amb[tid];
                    for (int o = 0; o < na; ++o) {
                        const float po = zamb[o];
                        rank += po > pa || (po == pa && amb[o] < ja);
                    }
                    if (rank == r - 1) bound[0] = pa;
                }
                __syncthreads();
                // a subnormal (or zero) boundary probability can tie with certainly-out keys too:
                // the whole row takes the oracle's path
                fallback = !(bound[0] >= FLT_MIN);
            }
            if (!fallback) {
                if (tid < na && rank < r) {  // chosen
                    const int ja = amb[tid];
                    atomicOr(&chosen[ja >> 5], 1u << (ja & 31));
                    atomicAdd(&wcnt[ja / (V4 * 128)], 1);
                }
                __syncthreads();
                int pos = 0;
#pragma unroll
                for (int w = 0; w < kCertWarps; ++w) pos += w < warp ? wcnt[w] : 0;
#pragma unroll
                for (int i = 0; i < V4; ++i) {
                    const int j = jw + 128 * i;
                    const uint32_t cw = full || j < n ? chosen[j >> 5] >> (j & 31) : 0u;  // 4 bits, j % 4 == 0
                    int tk[4], c = 0;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        tk[t] = (full || j + t < n) && (bin(v[i][t]) > bhi || ((cw >> t) & 1u));
                        c += tk[t];
                    }
                    int incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    int at = pos + incl - c;
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (tk[t]) {
                            if (at < k) out[at] = j + t;
                            ++at;
                        }
                    pos += __shfl_sync(0xffffffffu, incl, 31);
                }
                return;
            }
        }
    }
    // exact fallback: the oracle's logits in place of z~, then its softmax + Top-K on warp 0 (the
    // probability bits overwrite the logits row, which warp_softmax has consumed by then)
    __syncthreads();
    int nan = 0;
    for (int j = tid; j < n; j += kCertThreads) {
        const float ze = exact_logit<D>(q, kr, slots[j], p.scale);
        nan |= ze != ze;
        zg[j] = ze;
    }
    nan = block_sum(nan, red);  // (its barriers also order the zg writes before warp 0 reads them)
    if (warp != 0) return;
    if (p.status != nullptr && nan && lane == 0) atomicOr(p.status, 1);
    warp_softmax(zg, n, escr + row * escr_stride, reinterpret_cast<uint32_t*>(zg), nullptr);
    warp_topk(reinterpret_cast<const uint32_t*>(zg), n, k, hist, out);
}

// ---------------------------------------------------------------------------------------------
// Long key lists (a row's scratch does not fit 8 rows per CTA; config 5: 6006-block windows).
// Three kernels, each at high occupancy instead of one latency-bound warp per row:
//   logits_t_kernel  8 query rows x 4 keys per thread (4x fewer shared-memory q reads per DFMA than
//                    one key per thread), logits stored key-major: zt[j][R], R = u*nqb + i, so that
//   row_denom_kernel thread per row R: fp32 max and the ascending-j fp64 denominator (the only
//                    sequential part; at the k=0 pass row_denom2_kernel does the local-window and the
//                    full-row statistics in one pass), with the next 8 logits loaded ahead of the
//                    add chain
//   row_prob_kernel  fully parallel fp32 probabilities, row-major through a 32x32 smem transpose
//   topk_rows_kernel warp per row: radix select over the row's probability bits.
// The operation sequence per row is the same as warp_softmax / warp_topk above (and the oracle).
template <int D, int kKeysPerThread, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) logits_t_kernel(const ScoreParams p, float* __restrict__ zt) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    __shared__ __align__(16) double qd[kMaxRows * D];
    const int u = blockIdx.y, i0 = blockIdx.x * kMaxRows;
    const int nr = min(kMaxRows, p.nqb - i0);
    for (int e = threadIdx.x; e < kMaxRows * D; e += blockDim.x) {
        const int r = e / D, c = e % D;
        qd[e] = r < nr ? static_cast<double>(p.qc[p.qidx(u, i0 + r) * D + c]) : 0.0;
    }
    __syncthreads();
    const int jb = blockIdx.z * blockDim.x * kKeysPerThread + threadIdx.x;
    const float4* kr[kKeysPerThread];
#pragma unroll
    for (int q = 0; q < kKeysPerThread; ++q) {
        const int j = jb + q * blockDim.x;
        const int slot = j < p.n_keys ? __ldg(p.keys + static_cast<int64_t>(u) * p.key_stride + j) : 0;
        kr[q] = reinterpret_cast<const float4*>(p.krep + u * p.kru + static_cast<int64_t>(slot) * D);
    }
    double acc[kKeysPerThread][kMaxRows];
#pragma unroll
    for (int q = 0; q < kKeysPerThread; ++q)
#pragma unroll
        for (int r = 0; r < kMaxRows; ++r) acc[q][r] = 0.0;
    float4 kn[kKeysPerThread];  // next column quad, loaded one iteration ahead
#pragma unroll
    for (int q = 0; q < kKeysPerThread; ++q) kn[q] = __ldg(kr[q]);
#pragma unroll 1
    for (int c4 = 0; c4 < D / 4; ++c4) {
        double kd[kKeysPerThread][4];
#pragma unroll
        for (int q = 0; q < kKeysPerThread; ++q) {
            const float4 kv = kn[q];
            if (c4 + 1 < D / 4) kn[q] = __ldg(kr[q] + c4 + 1);
            kd[q][0] = kv.x;
            kd[q][1] = kv.y;
            kd[q][2] = kv.z;
            kd[q][3] = kv.w;
        }
        // column by column: the 8 x kKeysPerThread DFMAs of one column are independent (one per
        // accumulator), so consecutive DFMAs never wait on each other; each accumulator still adds
        // its columns in ascending c (3.88 -> 3.56 ms at config 5).  Staging the key rows through
        // shared memory with cp.async instead measured slower (4.30 ms).
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double2 qv[kMaxRows];
#pragma unroll
            for (int r = 0; r < kMaxRows; ++r) qv[r] = *reinterpret_cast<const double2*>(qd + r * D + 4 * c4 + 2 * h);
#pragma unroll
            for (int r = 0; r < kMaxRows; ++r)
#pragma unroll
                for (int q = 0; q < kKeysPerThread; ++q) acc[q][r] = __fma_rn(qv[r].x, kd[q][2 * h], acc[q][r]);
#pragma unroll
            for (int r = 0; r < kMaxRows; ++r)
#pragma unroll
                for (int q = 0; q < kKeysPerThread; ++q) acc[q][r] = __fma_rn(qv[r].y, kd[q][2 * h + 1], acc[q][r]);
        }
    }
    const int64_t rt = static_cast<int64_t>(p.units) * p.nqb;
    const int64_t r0 = static_cast<int64_t>(u) * p.nqb + i0;
#pragma unroll
    for (int q = 0; q < kKeysPerThread; ++q) {
        const int j = jb + q * blockDim.x;
        if (j >= p.n_keys) continue;
#pragma unroll
        for (int r = 0; r < kMaxRows; ++r)
            if (r < nr) zt[j * rt + r0 + r] = __fmul_rn(__double2float_rn(acc[q][r]), p.scale);
    }
}

// Thread per row R over keys [off, off + n) of zt: fp32 row max and the ascending-j fp64 softmax
// denominator (tensor.cpp:87-102); the exponentials of the next 8 keys are loaded ahead of the
// dependent add chain.  NaN logits set status bit 0 (the oracle rejects them).
__global__ void __launch_bounds__(128) row_denom_kernel(const float* __restrict__ zt, int64_t rt, int off, int n,
                                                        float* __restrict__ mrow, double* __restrict__ drow,
                                                        int* status) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    const int lane = threadIdx.x & 31;
    const int64_t R = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = R < rt;
    const float* z = zt + static_cast<int64_t>(off) * rt + (live ? R : 0);
    float m = -FLT_MAX;
    bool bad = false;
    if (live) {
        float mq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mq[q] = -FLT_MAX;
        int j = 0;
        for (; j + 8 <= n; j += 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float a = __ldg(z + (j + q) * rt);
                bad |= a != a;
                mq[q] = fmaxf(mq[q], a);
            }
        }
        for (; j < n; ++j) {
            const float a = __ldg(z + j * rt);
            bad |= a != a;
            m = fmaxf(m, a);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) m = fmaxf(m, mq[q]);  // max is exact: order-free
    }
    if (status != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 1);
    if (!live) return;
    const double dm = static_cast<double>(m);
    double denom = 0.0;
    int j = 0;
    if (n >= 8) {
        float zn[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) zn[q] = __ldg(z + q * rt);
        for (; j + 8 <= n; j += 8) {
            float zc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) zc[q] = zn[q];
            if (j + 16 <= n) {
#pragma unroll
                for (int q = 0; q < 8; ++q) zn[q] = __ldg(z + (j + 8 + q) * rt);
            }
            double e[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) e[q] = exp(static_cast<double>(zc[q]) - dm);
#pragma unroll
            for (int q = 0; q < 8; ++q) denom = __dadd_rn(denom, e[q]);  // ascending j
        }
    }
    for (; j < n; ++j) denom = __dadd_rn(denom, exp(static_cast<double>(__ldg(z + j * rt)) - dm));
    mrow[R] = m;
    drow[R] = denom;
}

// The k=0 pass needs two softmaxes of every row: over the local window [off, off + nl) (for the
// Top-K) and over all n keys (A_t for s_t).  One thread per row R computes both maxima in one pass
// over the key-major logits and both ascending fp64 denominators in a second pass -- the same
// operation sequences as two row_denom_kernel launches, with half the logit traffic.
__global__ void __launch_bounds__(128) row_denom2_kernel(const float* __restrict__ zt, int64_t rt, int off, int nl,
                                                         int n, float* __restrict__ mrow_l, double* __restrict__ drow_l,
                                                         float* __restrict__ mrow_f, double* __restrict__ drow_f,
                                                         int* status) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    const int lane = threadIdx.x & 31;
    const int64_t R = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = R < rt;
    const float* z = zt + (live ? R : 0);
    float ml = -FLT_MAX, mf = -FLT_MAX;
    bool bad = false;
    if (live) {
        // maxima: [0, off) and [off + nl, n) feed the full row only, [off, off + nl) both
        auto seg_max = [&](int j0, int j1) {
            float mq[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) mq[q] = -FLT_MAX;
            int j = j0;
            for (; j + 8 <= j1; j += 8) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float a = __ldg(z + static_cast<int64_t>(j + q) * rt);
                    bad |= a != a;
                    mq[q] = fmaxf(mq[q], a);
                }
            }
            float m = -FLT_MAX;
            for (; j < j1; ++j) {
                const float a = __ldg(z + static_cast<int64_t>(j) * rt);
                bad |= a != a;
                m = fmaxf(m, a);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) m = fmaxf(m, mq[q]);  // max is exact: order-free
            return m;
        };
        const float m0 = seg_max(0, off), m1 = seg_max(off, off + nl), m2 = seg_max(off + nl, n);
        ml = m1;
        mf = fmaxf(fmaxf(m0, m1), m2);
    }
    if (status != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, 1);
    if (!live) return;
    const double dl = static_cast<double>(ml), df = static_cast<double>(mf);
    double sl = 0.0, sf = 0.0;
    // ascending j; inside the window both chains advance, each in its own ascending order
    auto seg_sum = [&](int j0, int j1, bool both) {
        int j = j0;
        for (; j + 8 <= j1; j += 8) {
            float zc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) zc[q] = __ldg(z + static_cast<int64_t>(j + q) * rt);
            double ef[8], el[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                ef[q] = exp(static_cast<double>(zc[q]) - df);
                el[q] = both ? exp(static_cast<double>(zc[q]) - dl) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sf = __dadd_rn(sf, ef[q]);
                if (both) sl = __dadd_rn(sl, el[q]);
            }
        }
        for (; j < j1; ++j) {
            const double zj = static_cast<double>(__ldg(z + static_cast<int64_t>(j) * rt));
            sf = __dadd_rn(sf, exp(zj - df));
            if (both) sl = __dadd_rn(sl, exp(zj - dl));
        }
    };
    seg_sum(0, off, false);
    seg_sum(off, off + nl, true);
    seg_sum(off + nl, n, false);
    mrow_l[R] = ml;
    drow_l[R] = sl;
    mrow_f[R] = mf;
    drow_f[R] = sf;
}

// p[R][j] = float(exp(double(z[j][R]) - double(m_R)) / denom_R), fully parallel: a CTA converts a
// 32-key x 32-row tile of the key-major logits into row-major probabilities through shared memory.
__global__ void __launch_bounds__(256) row_prob_kernel(const float* __restrict__ zt, int64_t rt, int off, int n,
                                                       const float* __restrict__ mrow,
                                                       const double* __restrict__ drow, float* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    __shared__ float tile[32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * 32;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int64_t R = r0 + lane;
    if (R < rt) {
        const double dm = static_cast<double>(mrow[R]);
        const double den = drow[R];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int jl = warp * 4 + q;
            if (j0 + jl < n) {
                const double e = exp(static_cast<double>(__ldg(zt + static_cast<int64_t>(off + j0 + jl) * rt + R)) - dm);
                tile[lane][jl] = __double2float_rn(__ddiv_rn(e, den));
            }
        }
    }
    __syncthreads();
    if (j0 + lane < n) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int rl = warp * 4 + q;
            if (r0 + rl < rt) out[(r0 + rl) * n + j0 + lane] = tile[rl][lane];
        }
    }
}

// Warp per row: radix select straight from the row-major probabilities (L2-resident while the warp
// works on them; staging rows in shared memory measured slower -- it caps residency at 8 warps/SM).
__global__ void __launch_bounds__(256) topk_rows_kernel(const float* __restrict__ prob, int n, int k, int64_t rows,
                                                        int32_t* __restrict__ sel) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    __shared__ uint32_t hist[8][256];
    const int warp = threadIdx.x >> 5;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    if (row >= rows) return;
    warp_topk(reinterpret_cast<const uint32_t*>(prob) + row * n, n, k, hist[warp], sel + row * k);
}

__global__ void aggregate_kernel(const float* __restrict__ arows, int n_keys, int nqb, int units,
                                 float* __restrict__ s_t) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int u = blockIdx.y;
    if (j >= n_keys) return;
    const float* a = arows + static_cast<int64_t>(u) * nqb * n_keys + j;
    double acc = 0.0;
    for (int i = 0; i < nqb; ++i) acc = __dadd_rn(acc, static_cast<double>(a[static_cast<int64_t>(i) * n_keys]));
    s_t[static_cast<int64_t>(u) * n_keys + j] = __double2float_rn(__ddiv_rn(acc, static_cast<double>(nqb)));
}

}  // namespace

int launch_aggregate_scores(const float* a, int rows, int cols, int units, float* s, cudaStream_t st) {
    if (rows <= 0 || cols <= 0 || units <= 0) return 0;
    const dim3 grid((cols + 127) / 128, units);
    launch_pdl(aggregate_kernel, grid, dim3(128), 0, st, a, cols, rows, units, s);
    return check_launch("aggregate_kernel");
}

size_t score_select_workspace(int units, int nqb, int n_keys) {
    // A_t rows (k=0 pass) + key-major logits and local-window probabilities of the long-window path
    // + per-row max / denominator
    // (the certified denoise path needs [rows][n4] fp32 logits + [units][n4] key norms + [rows][n+1]
    // fp64 fallback scratch, n = n_local <= n_keys, n4 = n rounded up to 4)
    return 3 * static_cast<size_t>(units) * nqb * n_keys * sizeof(float) + static_cast<size_t>(units) * nqb * 32 +
           static_cast<size_t>(units) * (n_keys + 4) * sizeof(float) + 512;
}

template <int D>
int launch_certified(const ScoreParams& p, dim3 g1, size_t lsmem, int v4, float* zc, float* kn, int n4,
                     double* escr, int64_t es, int cert, cudaStream_t s) {
    if (int rc = ensure_smem(reinterpret_cast<const void*>(logits32_kernel<D>), lsmem, "logits32")) return rc;
    launch_pdl(logits32_kernel<D>, g1, dim3(kL32Warps * 32), lsmem, s, p, zc, kn);
    if (int rc = check_launch("logits32_kernel")) return rc;
    const dim3 g2(static_cast<unsigned>(static_cast<int64_t>(p.units) * p.nqb));
    const float* kc = kn;
    const int np = static_cast<int>(g1.x);
    switch (v4) {
        case 1: launch_pdl(cert_select_kernel<D, 1>, g2, dim3(kCertThreads), 0, s, p, zc, kc, np, n4, escr, es, cert); break;
        case 2: launch_pdl(cert_select_kernel<D, 2>, g2, dim3(kCertThreads), 0, s, p, zc, kc, np, n4, escr, es, cert); break;
        case 3:
        case 4: launch_pdl(cert_select_kernel<D, 4>, g2, dim3(kCertThreads), 0, s, p, zc, kc, np, n4, escr, es, cert); break;
        case 5:
        case 6: launch_pdl(cert_select_kernel<D, 6>, g2, dim3(kCertThreads), 0, s, p, zc, kc, np, n4, escr, es, cert); break;
        default: launch_pdl(cert_select_kernel<D, 8>, g2, dim3(kCertThreads), 0, s, p, zc, kc, np, n4, escr, es, cert); break;
    }
    return check_launch("cert_select_kernel");
}

// ---------------------------------------------------------------------------------------------
// K3 tile pairing.  A K3 tile walks the UNION of its two query blocks' visible lists, so the
// executed work of a call is the sum over tiles of (n_dense + 2k - overlap(a, b)).  CTA per unit:
// the nq selections as bitsets in shared memory, all pairwise overlaps (AND + popcount), then the
// greedy matching -- repeatedly the free pair with the largest overlap (ties: the lowest i * nq + j,
// i < j), tiles emitted in that order, an odd leftover last -- computed in parallel rounds of
// mutual-best pairs (below), then a bottleneck pass that raises the least-overlapping tile's
// overlap by partner swaps (the unit-gang K3 schedule waits for each unit's longest tile).
// Config 5 (6006-block window): chunk 683 -> 640 ms (greedy alone: -4.9 %, with the pass -6.2 %).
constexpr int kPairThreads = 512;

__global__ void __launch_bounds__(kPairThreads) pair_tiles_kernel(const int32_t* __restrict__ sel, int sel_rows,
                                                                  int sel_row0, int nq, int k, int words,
                                                                  int32_t* __restrict__ pairs) {
    pdl_wait();  // programmatic dependent launch: the selections are visible from here on
    extern __shared__ __align__(16) uint32_t pt_smem[];
    uint32_t* bits = pt_smem;                                                            // [nq][words]
    uint16_t* ov = reinterpret_cast<uint16_t*>(bits + static_cast<size_t>(nq) * words);  // [nq][nq]
    __shared__ int bkey[256], bj[256], partner_s[256];
    const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kWarps = kPairThreads / 32;
    for (int e = tid; e < nq * words; e += kPairThreads) bits[e] = 0u;
    __syncthreads();
    const int32_t* su = sel + (static_cast<int64_t>(u) * sel_rows + sel_row0) * k;
    for (int r = warp; r < nq; r += kWarps)
        for (int x0 = lane; x0 < k; x0 += 32) {
            const int x = __ldg(su + static_cast<int64_t>(r) * k + x0);
            atomicOr(&bits[r * words + (x >> 5)], 1u << (x & 31));
        }
    __syncthreads();
    if (words <= 32) {  // warp per row i, lanes over the partners j > i
        for (int i = warp; i < nq; i += kWarps)
            for (int j = i + 1 + lane; j < nq; j += 32) {
                int c = 0;
                for (int w = 0; w < words; ++w) c += __popc(bits[i * words + w] & bits[j * words + w]);
                ov[i * nq + j] = static_cast<uint16_t>(c);
                ov[j * nq + i] = static_cast<uint16_t>(c);
            }
    } else {  // warp per pair, lanes over the words
        for (int i = warp; i < nq; i += kWarps)
            for (int j = i + 1; j < nq; ++j) {
                int c = 0;
                for (int w = lane; w < words; w += 32) c += __popc(bits[i * words + w] & bits[j * words + w]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                if (lane == 0) {
                    ov[i * nq + j] = static_cast<uint16_t>(c);
                    ov[j * nq + i] = static_cast<uint16_t>(c);
                }
            }
    }
    __syncthreads();
    // key of pair (i, j): overlap above, 65535 - (min * nq + max) below -> the max key is the largest
    // overlap, then the lowest pair index (nq <= 255: the index fits 16 bits).  Warp-collective scan
    // of row i's free partners j = lane + 32 m (the lane owning j knows whether j is taken).
    auto row_best = [&](int i, auto is_taken, int& key_out, int& j_out) {
        int key = -1, bjj = -1;
        for (int j = lane; j < nq; j += 32)
            if (j != i && !is_taken(j)) {
                const int lo = i < j ? i : j, hi = i < j ? j : i;
                const int kk = (static_cast<int>(ov[i * nq + j]) << 16) | (65535 - (lo * nq + hi));
                if (kk > key) {
                    key = kk;
                    bjj = j;
                }
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int k2 = __shfl_xor_sync(0xffffffffu, key, o), j2 = __shfl_xor_sync(0xffffffffu, bjj, o);
            if (k2 > key) {  // keys are unique per pair
                key = k2;
                bjj = j2;
            }
        }
        key_out = key;
        j_out = bjj;
    };
    // Rounds of mutual-best pairs: a pair whose two rows name each other as best free partner is
    // the one the greedy order would take anyway (no free pair touching either row has a larger
    // key), so taking all of them at once yields EXACTLY the greedy matching.  Only rows whose best
    // partner was taken rescan.
    __shared__ int n_new;
    for (int i = tid; i < nq; i += kPairThreads) partner_s[i] = -1;
    __syncthreads();
    auto free_fn = [&](int j) { return partner_s[j] != -1; };  // "taken" predicate for row_best
    for (int i = warp; i < nq; i += kWarps) {
        int key, j;
        row_best(i, free_fn, key, j);
        if (lane == 0) {
            bkey[i] = key;
            bj[i] = j;
        }
    }
    __syncthreads();
    for (int round = 0; round < nq; ++round) {
        if (tid == 0) n_new = 0;
        int mate = -1;
        if (tid < nq && partner_s[tid] == -1) {
            const int j = bj[tid];
            if (j >= 0 && bj[j] == tid) mate = j;
        }
        __syncthreads();
        if (mate >= 0) {
            partner_s[tid] = mate;
            if (tid < mate) atomicAdd(&n_new, 1);
        }
        __syncthreads();
        const int nn = n_new;
        if (nn == 0) break;  // (uniform: read after the barrier, reset only after the next one)
        for (int i = warp; i < nq; i += kWarps) {  // free rows whose best partner was just taken
            if (partner_s[i] != -1 || bj[i] < 0 || partner_s[bj[i]] == -1) continue;
            int key, j;
            row_best(i, free_fn, key, j);
            __syncwarp();  // every lane has read bj[i] before lane 0 rewrites it
            if (lane == 0) {
                bkey[i] = key;
                bj[i] = j;
            }
        }
        __syncthreads();
    }
    // tiles in the greedy order (pair key descending), an odd leftover last
    __shared__ int ta[128], tb[128];
    const int T = nq / 2;
    if (tid < nq && partner_s[tid] > tid) {
        const int mate = partner_s[tid];
        const int mykey = (static_cast<int>(ov[tid * nq + mate]) << 16) | (65535 - (tid * nq + mate));
        int rank = 0;
        for (int a2 = 0; a2 < nq; ++a2) {
            const int pa = partner_s[a2];
            if (pa > a2 && ((static_cast<int>(ov[a2 * nq + pa]) << 16) | (65535 - (a2 * nq + pa))) > mykey) ++rank;
        }
        ta[rank] = tid;
        tb[rank] = mate;
    }
    __syncthreads();
    if (warp != 0) return;
    // Bottleneck pass (K3's unit-gang schedule waits for each unit's longest tile): while some swap
    // of partners between the least-overlapping tile t and another tile s makes both new tiles
    // overlap more than t did, take the best such swap (largest new minimum, then largest sum, then
    // lowest s, (a_t, a_s) before (a_t, b_s)).  At most nq rounds.
    for (int it = 0; it < nq; ++it) {
        int best_o = 0x7FFFFFFF, tw = -1;
        for (int t2 = lane; t2 < T; t2 += 32) {
            const int o2 = ov[ta[t2] * nq + tb[t2]];
            if (o2 < best_o) {
                best_o = o2;
                tw = t2;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int b2 = __shfl_xor_sync(0xffffffffu, best_o, o), t3 = __shfl_xor_sync(0xffffffffu, tw, o);
            if (b2 < best_o || (b2 == best_o && t3 < tw)) {
                best_o = b2;
                tw = t3;
            }
        }
        if (tw < 0) break;
        const int a = ta[tw], b2 = tb[tw];
        // candidate key: (new min << 20) | (new sum << 4) ... ties -> lowest s, option 0 first
        long long bestk = -1;
        int bs = -1, bopt = 0;
        for (int s2 = lane; s2 < T; s2 += 32) {
            if (s2 == tw) continue;
            const int c = ta[s2], d2 = tb[s2];
#pragma unroll
            for (int opt = 0; opt < 2; ++opt) {
                const int x1 = ov[a * nq + (opt ? d2 : c)], x2 = ov[b2 * nq + (opt ? c : d2)];
                const int mn = min(x1, x2);
                if (mn <= best_o) continue;
                const long long kk = (static_cast<long long>(mn) << 40) | (static_cast<long long>(x1 + x2) << 16) |
                                     static_cast<long long>(65535 - (2 * s2 + opt));
                if (kk > bestk) {
                    bestk = kk;
                    bs = s2;
                    bopt = opt;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long k2 = __shfl_xor_sync(0xffffffffu, bestk, o);
            const int s3 = __shfl_xor_sync(0xffffffffu, bs, o), p3 = __shfl_xor_sync(0xffffffffu, bopt, o);
            if (k2 > bestk) {
                bestk = k2;
                bs = s3;
                bopt = p3;
            }
        }
        if (bestk < 0) break;
        __syncwarp();
        if (lane == 0) {
            const int c = ta[bs], d2 = tb[bs];
            const int n1 = bopt ? d2 : c, n2 = bopt ? c : d2;  // a pairs with n1, b with n2
            ta[tw] = min(a, n1);
            tb[tw] = max(a, n1);
            ta[bs] = min(b2, n2);
            tb[bs] = max(b2, n2);
        }
        __syncwarp();
    }
    int32_t* pu = pairs + static_cast<int64_t>(u) * ((nq + 1) / 2) * 2;
    for (int t2 = lane; t2 < T; t2 += 32) {
        pu[2 * t2] = ta[t2];
        pu[2 * t2 + 1] = tb[t2];
    }
    if (nq & 1) {
        for (int i = lane; i < nq; i += 32)
            if (partner_s[i] == -1) {  // the one leftover
                pu[2 * T] = i;
                pu[2 * T + 1] = -1;
            }
    }
}

int launch_pair_tiles(const int32_t* sel, int sel_rows, int sel_row0, int nq, int k, int n_local, int units,
                      int32_t* pairs, cudaStream_t s) {
    if (units == 0 || nq == 0) return 0;
    if (nq > 255 || k <= 0 || n_local <= 0 || k > 32767) return set_error(PBSA_EUNSUPPORTED, "pair_tiles: shape");
    const int words = (n_local + 31) / 32;
    const size_t smem = static_cast<size_t>(nq) * words * 4 + ((static_cast<size_t>(nq) * nq * 2 + 15) & ~size_t(15));
    if (smem > 200 * 1024) return set_error(PBSA_EUNSUPPORTED, "pair_tiles: bitsets exceed shared memory");
    // (+ the kernel's 2 KB of static shared memory, which counts against the 48 KB default too)
    if (int rc = ensure_smem(reinterpret_cast<const void*>(pair_tiles_kernel), smem + 4096, "pair_tiles")) return rc;
    if (launch_pdl(pair_tiles_kernel, dim3(static_cast<unsigned>(units)), dim3(kPairThreads), smem, s, sel, sel_rows,
                   sel_row0, nq, k, words, pairs) != cudaSuccess)
        return check_launch("pair_tiles_kernel");
    return check_launch("pair_tiles_kernel");
}

// PBSA_K2_CERT: unset = certified fp32 ranking on denoise passes over windows of >= kCertMinKeys
// keys, 1 = certified on every denoise pass, 0 = the exact fp64 path on every pass, 2 = certified
// kernels with every row forced through the exact fallback (tests).
constexpr int kCertMinKeys = 1024;
static int cert_mode() {
    const char* e = std::getenv("PBSA_K2_CERT");
    return e == nullptr ? 1 : (std::atoi(e) == 1 ? 3 : std::atoi(e));
}

int launch_score_select(const float* qc, const float* krep, int64_t kru, const int32_t* keys,
                        int key_stride, int n_keys, int local_off, int n_local, int k, int nqb,
                        int units, int d, float scale, int32_t* sel, float* s_t, void* ws,
                        size_t ws_bytes, cudaStream_t s, int* status, int qc_rows, int qc_row0) {
    if (qc_rows <= 0) qc_rows = nqb;
    if (units == 0 || nqb == 0 || n_keys == 0) return 0;
    const bool do_select = k > 0 && n_local > 0;
    if (!do_select && s_t == nullptr) return 0;
    if (ws_bytes < score_select_workspace(units, nqb, n_keys))
        return set_error(PBSA_EINVAL, "score_select: workspace too small");
    float* arows = s_t ? static_cast<float*>(ws) : nullptr;
    const int cert = cert_mode();
    // certified path for long windows (config 5: 6006 keys, 2.8x faster than the exact kernels);
    // short windows (config 2: 312 keys) are latency-bound either way and stay on the exact kernels
    // (PBSA_K2_CERT=1 forces the certified path for any window that fits, e.g. in tests)
    const bool want_cert = cert == 1 ? n_local >= kCertMinKeys : cert != 0;  // 3: forced
    if (do_select && s_t == nullptr && want_cert && n_local <= kCertMaxKeys) {
        // denoise pass: certified fp32 logits of the local window, exact only near the k-th boundary
        const int64_t rt = static_cast<int64_t>(units) * nqb;
        const int n4 = (n_local + 3) & ~3;                                    // 16-byte rows
        float* zc = static_cast<float*>(ws);                                  // [rt][n4]
        float* kn = zc + static_cast<size_t>(rt) * n4;                        // [units][key tiles] max |k|
        double* escr = reinterpret_cast<double*>(
            (reinterpret_cast<uintptr_t>(kn + static_cast<size_t>(units) * n4) + 15) & ~uintptr_t(15));
        const int64_t es = (n_local + 1) & ~1;  // 16-byte aligned fp64 scratch rows
        ScoreParams p{qc, krep, kru, keys, key_stride, n_keys, local_off, n_local, k, nqb, units,
                      1, scale, 0, sel, nullptr, status};
        p.qc_rows = qc_rows;
        p.qc_row0 = qc_row0;
        dim3 g1((n_local + kLogitKeys - 1) / kLogitKeys, (nqb + kL32Warps * 8 - 1) / (kL32Warps * 8), units);
        const size_t lsmem = static_cast<size_t>(kL32Warps * 8 + kLogitKeys) * d * 4;
        const int v4 = (n_local + 4 * kCertThreads - 1) / (4 * kCertThreads);  // float4 per thread
        if (d == 128) return launch_certified<128>(p, g1, lsmem, v4, zc, kn, n4, escr, es, cert, s);
        return launch_certified<64>(p, g1, lsmem, v4, zc, kn, n4, escr, es, cert, s);
    }
    if (s_t == nullptr) {  // no A_t: only the local window's logits are needed
        keys += local_off;
        n_keys = n_local;
        local_off = 0;
    }
    {
        const size_t per_warp =
            (static_cast<size_t>(n_keys) * 12 + static_cast<size_t>(n_local) * 4 + 1024 + 15) & ~size_t(15);
        const size_t qbytes = static_cast<size_t>(kMaxRows) * d * 8;
        const size_t budget = 200 * 1024 - qbytes;
        if (per_warp > 200 * 1024)
            return set_error(PBSA_EUNSUPPORTED, "score_select: too many key blocks for one row in smem");
        int rows = static_cast<int>(budget / per_warp);
        rows = rows < 1 ? 1 : (rows > kMaxRows ? kMaxRows : rows);
        ScoreParams p{qc, krep, kru, keys, key_stride, n_keys, local_off, n_local, do_select ? k : 0, nqb, units,
                      rows, scale, per_warp, sel, arows, status};
        p.qc_rows = qc_rows;
        p.qc_row0 = qc_row0;
        if (rows < kMaxRows) {
            // long key lists: key-major logits -> thread-per-row softmax statistics -> warp-per-row select
            const int64_t rt = static_cast<int64_t>(units) * nqb;
            float* zt = static_cast<float*>(ws) + static_cast<size_t>(rt) * n_keys;
            float* prob = zt + static_cast<size_t>(rt) * n_keys;
            // 4 keys x 8 rows per thread at two CTAs per SM (2 keys at three CTAs measured slower)
            dim3 g1((nqb + kMaxRows - 1) / kMaxRows, units, (n_keys + 256 * 4 - 1) / (256 * 4));
            if (d == 128) launch_pdl(logits_t_kernel<128, 4, 2>, g1, dim3(256), 0, s, p, zt);
            else launch_pdl(logits_t_kernel<64, 4, 2>, g1, dim3(256), 0, s, p, zt);
            if (int rc = check_launch("logits_t_kernel")) return rc;
            float* mrow = prob + static_cast<size_t>(rt) * n_keys;
            double* drow = reinterpret_cast<double*>(mrow + ((rt + 1) & ~int64_t(1)));
            const int gr = static_cast<int>((rt + 127) / 128);
            auto softmax_rows = [&](int off, int n, float* out, int* st) -> int {
                launch_pdl(row_denom_kernel, dim3(gr), dim3(128), 0, s, static_cast<const float*>(zt), rt, off, n, mrow, drow, st);
                if (int rc = check_launch("row_denom_kernel")) return rc;
                dim3 g2((n + 31) / 32, static_cast<unsigned>((rt + 31) / 32));
                launch_pdl(row_prob_kernel, g2, dim3(256), 0, s, static_cast<const float*>(zt), rt, off, n,
                           static_cast<const float*>(mrow), static_cast<const double*>(drow), out);
                return check_launch("row_prob_kernel");
            };
            if (do_select && arows != nullptr) {
                // k=0 pass: both softmaxes' statistics in one pass over the logits
                float* mrow_f = reinterpret_cast<float*>(drow + ((rt + 1) & ~int64_t(1)));
                double* drow_f = reinterpret_cast<double*>(mrow_f + ((rt + 1) & ~int64_t(1)));
                launch_pdl(row_denom2_kernel, dim3(gr), dim3(128), 0, s, static_cast<const float*>(zt), rt, local_off,
                           n_local, n_keys, mrow, drow, mrow_f, drow_f, status);
                if (int rc = check_launch("row_denom2_kernel")) return rc;
                dim3 g2((n_local + 31) / 32, static_cast<unsigned>((rt + 31) / 32));
                launch_pdl(row_prob_kernel, g2, dim3(256), 0, s, static_cast<const float*>(zt), rt, local_off, n_local,
                           static_cast<const float*>(mrow), static_cast<const double*>(drow), prob);
                if (int rc = check_launch("row_prob_kernel")) return rc;
                launch_pdl(topk_rows_kernel, dim3(static_cast<unsigned>((rt + 7) / 8)), dim3(256), 0, s,
                           static_cast<const float*>(prob), n_local, k, rt, sel);
                if (int rc = check_launch("topk_rows_kernel")) return rc;
                dim3 g3((n_keys + 31) / 32, static_cast<unsigned>((rt + 31) / 32));
                launch_pdl(row_prob_kernel, g3, dim3(256), 0, s, static_cast<const float*>(zt), rt, 0, n_keys,
                           static_cast<const float*>(mrow_f), static_cast<const double*>(drow_f), arows);
                if (int rc = check_launch("row_prob_kernel")) return rc;
            } else {
                if (do_select) {
                    if (int rc = softmax_rows(local_off, n_local, prob, status)) return rc;
                    launch_pdl(topk_rows_kernel, dim3(static_cast<unsigned>((rt + 7) / 8)), dim3(256), 0, s,
                               static_cast<const float*>(prob), n_local, k, rt, sel);
                    if (int rc = check_launch("topk_rows_kernel")) return rc;
                }
                if (arows != nullptr) {
                    if (int rc = softmax_rows(0, n_keys, arows, do_select ? nullptr : status)) return rc;
                }
            }
        } else {
            // row-major logits into the workspace (after the A_t rows), then warp-per-row select
            const int64_t rt = static_cast<int64_t>(units) * nqb;
            float* z = static_cast<float*>(ws) + static_cast<size_t>(rt) * n_keys;
            dim3 g1((n_keys + kLogitKeys - 1) / kLogitKeys, (nqb + kMaxRows - 1) / kMaxRows, units);
            const size_t lsmem = static_cast<size_t>(kMaxRows) * d * 8 + static_cast<size_t>(kLogitKeys) * d * 4;
            if (d == 128) {
                if (int rc = ensure_smem(reinterpret_cast<const void*>(logits_rm_kernel<128>), lsmem, "logits_rm"))
                    return rc;
                launch_pdl(logits_rm_kernel<128>, g1, dim3(kLogitKeys), lsmem, s, p, z);
            } else {
                if (int rc = ensure_smem(reinterpret_cast<const void*>(logits_rm_kernel<64>), lsmem, "logits_rm"))
                    return rc;
                launch_pdl(logits_rm_kernel<64>, g1, dim3(kLogitKeys), lsmem, s, p, z);
            }
            if (int rc = check_launch("logits_rm_kernel")) return rc;
            p.per_warp = (static_cast<size_t>(n_keys) * 12 + 16 + static_cast<size_t>(n_local) * 4 + 1024 + 15) & ~size_t(15);
            const size_t smem = p.per_warp * kMaxRows;
            if (do_select && arows != nullptr) {
                if (int rc = ensure_smem(reinterpret_cast<const void*>(row_select_kernel<2>), smem, "row_select"))
                    return rc;
                launch_pdl(row_select_kernel<2>, dim3(static_cast<unsigned>((rt + kMaxRows / 2 - 1) / (kMaxRows / 2))),
                           dim3(256), smem, s, p, static_cast<const float*>(z));
            } else {
                if (int rc = ensure_smem(reinterpret_cast<const void*>(row_select_kernel<1>), smem, "row_select"))
                    return rc;
                launch_pdl(row_select_kernel<1>, dim3(static_cast<unsigned>((rt + kMaxRows - 1) / kMaxRows)), dim3(256),
                           smem, s, p, static_cast<const float*>(z));
            }
            if (int rc = check_launch("row_select_kernel")) return rc;
        }
    }
    if (s_t) {
        dim3 grid((n_keys + 127) / 128, units);
        launch_pdl(aggregate_kernel, grid, dim3(128), 0, s, static_cast<const float*>(arows), n_keys, nqb, units, s_t);
        if (int rc = check_launch("aggregate_kernel")) return rc;
    }
    return 0;
}

}  // namespace pbsa
