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
// Two kernels:
//   score_select_kernel  CTA = unit x up to 8 query-block rows.  Phase 1: logits, thread per key
//                        block (fp64 query reps in smem, each key element converted once).
//                        Phase 2: warp per row: softmax (fp64 exp, sequential ascending denominator
//                        on lane 0 exactly like the oracle), 4-pass 8-bit radix select on the fp32
//                        probability bits, ballot compaction of the winners
//   aggregate_kernel     thread per key block, ascending-row fp64 column sums (k=0 pass only)
#include <cfloat>

#include "internal.h"

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
    for (int j = lane; j < n; j += 32) e[j] = exp(static_cast<double>(z[j]) - dm);
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
    for (int j = lane; j < n; j += 32) {
        const float p = __double2float_rn(__ddiv_rn(e[j], denom));
        if (out_bits) out_bits[j] = __float_as_uint(p);
        if (out_f) out_f[j] = p;
    }
    __syncwarp();
}

// k largest of pb[0..n) (non-negative float bits => unsigned order), ties -> lower index.
// Writes the winners' indices ascending to out[0..k).
__device__ void warp_topk(const uint32_t* pb, int n, int k, uint32_t* hist, int32_t* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
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
};

constexpr int kMaxRows = 8;

// One CTA = one unit x up to 8 query-block rows.  Phase 1 (all 256 threads): coarse logits of the
// rows against every key block, thread per key, ascending-k fp64 dot products -- the query reps are
// converted to fp64 once into shared memory and each key element once, so the DFMA chains are not
// starved by float->double conversions.  Phase 2 (warp per row): softmax, Top-K, optional A_t row.
template <int D>
__global__ void __launch_bounds__(256) score_select_kernel(const ScoreParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
    const int u = blockIdx.y, i0 = blockIdx.x * p.rows;
    const int nr = min(p.rows, p.nqb - i0);
    const int n = p.n_keys;
    double* qd = reinterpret_cast<double*>(smem);                 // [kMaxRows][D]
    uint8_t* rows_base = smem + static_cast<size_t>(kMaxRows) * D * 8;
    for (int e = tid; e < kMaxRows * D; e += blockDim.x) {
        const int r = e / D, c = e % D;
        qd[e] = r < nr ? static_cast<double>(p.qc[(static_cast<int64_t>(u) * p.nqb + i0 + r) * D + c]) : 0.0;
    }
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) {
        const int slot = __ldg(p.keys + static_cast<int64_t>(u) * p.key_stride + j);
        const float4* kr = reinterpret_cast<const float4*>(p.krep + u * p.kru + static_cast<int64_t>(slot) * D);
        double acc[kMaxRows];
#pragma unroll
        for (int r = 0; r < kMaxRows; ++r) acc[r] = 0.0;
#pragma unroll 2
        for (int c4 = 0; c4 < D / 4; ++c4) {
            const float4 kv = __ldg(kr + c4);
            const double k0 = kv.x, k1 = kv.y, k2 = kv.z, k3 = kv.w;
#pragma unroll
            for (int r = 0; r < kMaxRows; ++r) {  // ascending c per row; fp32 x fp32 is exact in fp64
                const double* q = qd + r * D + 4 * c4;
                acc[r] = __fma_rn(q[0], k0, acc[r]);
                acc[r] = __fma_rn(q[1], k1, acc[r]);
                acc[r] = __fma_rn(q[2], k2, acc[r]);
                acc[r] = __fma_rn(q[3], k3, acc[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < kMaxRows; ++r)
            if (r < nr) {
                float* z = reinterpret_cast<float*>(rows_base + p.per_warp * r + static_cast<size_t>(n) * 8);
                z[j] = __fmul_rn(__double2float_rn(acc[r]), p.scale);
            }
    }
    __syncthreads();
    if (warp >= nr) return;
    const int64_t row = static_cast<int64_t>(u) * p.nqb + i0 + warp;
    uint8_t* base = rows_base + p.per_warp * warp;
    double* e = reinterpret_cast<double*>(base);
    float* z = reinterpret_cast<float*>(base + static_cast<size_t>(n) * 8);
    uint32_t* pb = reinterpret_cast<uint32_t*>(base + static_cast<size_t>(n) * 12);
    uint32_t* hist = pb + p.n_local;
    bool bad = false;
    for (int j = lane; j < n; j += 32) bad |= z[j] != z[j];
    if (p.status != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.status, 1);
    __syncwarp();
    if (p.k > 0 && p.n_local > 0) {
        warp_softmax(z + p.local_off, p.n_local, e, pb, nullptr);
        warp_topk(pb, p.n_local, p.k, hist, p.sel + row * p.k);
    }
    if (p.arows != nullptr) warp_softmax(z, n, e, nullptr, p.arows + row * n);
}

// Long key lists (a row's scratch does not fit 8 rows per CTA): logits for 8 rows per CTA into a
// global scratch (so each key representative is read once per 8 rows), then one warp per row.
template <int D>
__global__ void __launch_bounds__(256) logits_kernel(const ScoreParams p, float* __restrict__ logits) {
    __shared__ double qd[kMaxRows * D];
    const int u = blockIdx.y, i0 = blockIdx.x * kMaxRows;
    const int nr = min(kMaxRows, p.nqb - i0);
    for (int e = threadIdx.x; e < kMaxRows * D; e += blockDim.x) {
        const int r = e / D, c = e % D;
        qd[e] = r < nr ? static_cast<double>(p.qc[(static_cast<int64_t>(u) * p.nqb + i0 + r) * D + c]) : 0.0;
    }
    __syncthreads();
    const int j = blockIdx.z * blockDim.x + threadIdx.x;
    if (j >= p.n_keys) return;
    const int slot = __ldg(p.keys + static_cast<int64_t>(u) * p.key_stride + j);
    const float4* kr = reinterpret_cast<const float4*>(p.krep + u * p.kru + static_cast<int64_t>(slot) * D);
    double acc[kMaxRows];
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r) acc[r] = 0.0;
#pragma unroll 2
    for (int c4 = 0; c4 < D / 4; ++c4) {
        const float4 kv = __ldg(kr + c4);
        const double k0 = kv.x, k1 = kv.y, k2 = kv.z, k3 = kv.w;
#pragma unroll
        for (int r = 0; r < kMaxRows; ++r) {
            const double* q = qd + r * D + 4 * c4;
            acc[r] = __fma_rn(q[0], k0, acc[r]);
            acc[r] = __fma_rn(q[1], k1, acc[r]);
            acc[r] = __fma_rn(q[2], k2, acc[r]);
            acc[r] = __fma_rn(q[3], k3, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < kMaxRows; ++r)
        if (r < nr)
            logits[(static_cast<int64_t>(u) * p.nqb + i0 + r) * p.n_keys + j] = __fmul_rn(__double2float_rn(acc[r]), p.scale);
}

__global__ void __launch_bounds__(256) select_rows_kernel(const ScoreParams p, const float* __restrict__ logits) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * p.rows + warp;
    if (warp >= p.rows || row >= static_cast<int64_t>(p.units) * p.nqb) return;
    const int n = p.n_keys;
    uint8_t* base = smem + p.per_warp * warp;
    double* e = reinterpret_cast<double*>(base);
    float* z = reinterpret_cast<float*>(base + static_cast<size_t>(n) * 8);
    uint32_t* pb = reinterpret_cast<uint32_t*>(base + static_cast<size_t>(n) * 12);
    uint32_t* hist = pb + p.n_local;
    bool bad = false;
    for (int j = lane; j < n; j += 32) {
        z[j] = logits[row * n + j];
        bad |= z[j] != z[j];
    }
    if (p.status != nullptr && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.status, 1);
    __syncwarp();
    if (p.k > 0 && p.n_local > 0) {
        warp_softmax(z + p.local_off, p.n_local, e, pb, nullptr);
        warp_topk(pb, p.n_local, p.k, hist, p.sel + row * p.k);
    }
    if (p.arows != nullptr) warp_softmax(z, n, e, nullptr, p.arows + row * n);
}

__global__ void aggregate_kernel(const float* __restrict__ arows, int n_keys, int nqb, int units,
                                 float* __restrict__ s_t) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int u = blockIdx.y;
    if (j >= n_keys) return;
    const float* a = arows + static_cast<int64_t>(u) * nqb * n_keys + j;
    double acc = 0.0;
    for (int i = 0; i < nqb; ++i) acc = __dadd_rn(acc, static_cast<double>(a[static_cast<int64_t>(i) * n_keys]));
    s_t[static_cast<int64_t>(u) * n_keys + j] = __double2float_rn(__ddiv_rn(acc, static_cast<double>(nqb)));
}

}  // namespace

size_t score_select_workspace(int units, int nqb, int n_keys) {
    // A_t rows (k=0 pass) + logits scratch of the long-window path
    return 2 * static_cast<size_t>(units) * nqb * n_keys * sizeof(float) + 256;
}

int launch_score_select(const float* qc, const float* krep, int64_t kru, const int32_t* keys,
                        int key_stride, int n_keys, int local_off, int n_local, int k, int nqb,
                        int units, int d, float scale, int32_t* sel, float* s_t, void* ws,
                        size_t ws_bytes, cudaStream_t s, int* status) {
    if (units == 0 || nqb == 0 || n_keys == 0) return 0;
    const bool do_select = k > 0 && n_local > 0;
    if (!do_select && s_t == nullptr) return 0;
    if (ws_bytes < score_select_workspace(units, nqb, n_keys))
        return set_error(PBSA_EINVAL, "score_select: workspace too small");
    float* arows = s_t ? static_cast<float*>(ws) : nullptr;
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
        if (rows < kMaxRows) {
            // long key lists: logits of 8 rows per CTA into scratch, then warp-per-row selection
            float* logits = static_cast<float*>(ws) + static_cast<size_t>(units) * nqb * n_keys;
            dim3 g1((nqb + kMaxRows - 1) / kMaxRows, units, (n_keys + 255) / 256);
            if (d == 128) logits_kernel<128><<<g1, 256, 0, s>>>(p, logits);
            else logits_kernel<64><<<g1, 256, 0, s>>>(p, logits);
            if (int rc = check_launch("logits_kernel")) return rc;
            const size_t smem2 = per_warp * rows;
            if (int rc = ensure_smem(reinterpret_cast<const void*>(select_rows_kernel), smem2, "score_select"))
                return rc;
            const int64_t total = static_cast<int64_t>(units) * nqb;
            select_rows_kernel<<<static_cast<int>((total + rows - 1) / rows), rows * 32, smem2, s>>>(p, logits);
            if (int rc = check_launch("select_rows_kernel")) return rc;
        } else {
        const size_t smem = qbytes + per_warp * rows;
        dim3 grid((nqb + rows - 1) / rows, units);
        if (d == 128) {
            if (int rc = ensure_smem(reinterpret_cast<const void*>(score_select_kernel<128>), smem, "score_select"))
                return rc;
            score_select_kernel<128><<<grid, 256, smem, s>>>(p);
        } else {
            if (int rc = ensure_smem(reinterpret_cast<const void*>(score_select_kernel<64>), smem, "score_select"))
                return rc;
            score_select_kernel<64><<<grid, 256, smem, s>>>(p);
        }
        if (int rc = check_launch("score_select_kernel")) return rc;
        }
    }
    if (s_t) {
        dim3 grid((n_keys + 127) / 128, units);
        aggregate_kernel<<<grid, 128, 0, s>>>(arows, n_keys, nqb, units, s_t);
        if (int rc = check_launch("aggregate_kernel")) return rc;
    }
    return 0;
}

}  // namespace pbsa
