// compress.cu -- K1 block compression (+ the fused current-chunk KV write).
//
// Reference op: router.compress_blocks: representative = mean of the b token
// vectors of a block (average pooling).  Numerics pinned to the oracle
// (the CPU restatement in oracle/pbsa_oracle.cpp): fp64 sum in ascending token order, one IEEE
// division by b, cast to fp32 -> bit-exact for any input.
//
// Roofline: HBM.  Algorithmic bytes per block = b*d*2 (bf16 read) + d*4 (f32 write).  One warp
// per block; lane l owns columns [l*C, l*C+C), C = d/32, so each token row is one coalesced
// 256-byte (d=128) warp load; rows are unrolled 16-deep for memory-level parallelism.  The fp64
// adds (one per element) stay far below the DADD rate at HBM speed.
#include "internal.h"
#include "ptx.cuh"

namespace pbsa {
namespace {

template <int C>
struct Vec;
template <>
struct Vec<4> {
    using T = uint2;  // 4 x bf16
};
template <>
struct Vec<2> {
    using T = uint32_t;  // 2 x bf16
};

template <int C>
__device__ __forceinline__ void unpack(const typename Vec<C>::T& v, float (&f)[C]) {
    if constexpr (C == 4) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
        float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
        f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    } else {
        float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
        f[0] = a.x; f[1] = a.y;
    }
}

template <int D>
__global__ void __launch_bounds__(256) compress_kernel(const bf16* __restrict__ x, int64_t xu, int64_t xb,
                                                       const int32_t* __restrict__ map, int nb,
                                                       int units, int b, float* __restrict__ reps,
                                                       int64_t ru) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    constexpr int C = D / 32;
    using V = typename Vec<C>::T;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    if (w >= static_cast<int64_t>(nb) * units) return;
    const int lane = threadIdx.x & 31;
    const int u = static_cast<int>(w / nb), i = static_cast<int>(w % nb);
    const int idx = map ? __ldg(map + static_cast<int64_t>(u) * nb + i) : i;
    const V* src = reinterpret_cast<const V*>(x + u * xu + idx * xb) + lane;
    double acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.0;
    // 16 token rows in flight per lane (a block is <= 64 rows: at most 4 round trips to memory);
    // the adds stay in ascending token order
    constexpr int kDepth = 16;
    for (int t = 0; t < b; t += kDepth) {
        V v[kDepth];
#pragma unroll
        for (int r = 0; r < kDepth; ++r)
            if (t + r < b) v[r] = __ldg(src + (t + r) * (D / C));
#pragma unroll
        for (int r = 0; r < kDepth; ++r) {
            if (t + r >= b) break;
            float f[C];
            unpack<C>(v[r], f);
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] += static_cast<double>(f[c]);
        }
    }
    float* dst = reps + u * ru + static_cast<int64_t>(idx) * D + lane * C;
    const double db = static_cast<double>(b);
#pragma unroll
    for (int c = 0; c < C; ++c) dst[c] = __double2float_rn(__ddiv_rn(acc[c], db));
}

// Writes block i of the current chunk (rows [i*b, i*b+b) of kc / vc) into pool slot stage[u][i]
// rows [0, b) and its K representative into krep[u][slot]; with WITH_Q also compresses the same
// block of Q into qrep[u][i] (the fused ingest of one PBSA call: one pass over Q, K and V).  Pool
// rows >= b are never written (zeroed at creation), which the attention kernel relies on.
template <int D, bool WITH_Q>
__global__ void __launch_bounds__(256) write_chunk_kernel(const bf16* __restrict__ kc,
                                                          const bf16* __restrict__ vc,
                                                          const bf16* __restrict__ qcur,
                                                          const int32_t* __restrict__ stage, int bpc,
                                                          int b, int units, int n_slots,
                                                          bf16* __restrict__ kp, bf16* __restrict__ vp,
                                                          float* __restrict__ krep, float* __restrict__ qrep) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    constexpr int C = D / 32;
    using V = typename Vec<C>::T;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    if (w >= static_cast<int64_t>(bpc) * units) return;
    const int lane = threadIdx.x & 31;
    const int u = static_cast<int>(w / bpc), i = static_cast<int>(w % bpc);
    const int slot = __ldg(stage + static_cast<int64_t>(u) * bpc + i);
    const int64_t src_off = (static_cast<int64_t>(u) * bpc + i) * b * D;
    const int64_t dst_off = (static_cast<int64_t>(u) * n_slots + slot) * 64 * D;
    const V* ks = reinterpret_cast<const V*>(kc + src_off) + lane;
    const V* vs = reinterpret_cast<const V*>(vc + src_off) + lane;
    const V* qs = WITH_Q ? reinterpret_cast<const V*>(qcur + src_off) + lane : nullptr;
    V* kd = reinterpret_cast<V*>(kp + dst_off) + lane;
    V* vd = reinterpret_cast<V*>(vp + dst_off) + lane;
    double acc[C], qacc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = qacc[c] = 0.0;
    int t = 0;
    for (; t + 4 <= b; t += 4) {
        V kv[4], vv[4], qv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            kv[r] = __ldg(ks + (t + r) * (D / C));
            vv[r] = __ldg(vs + (t + r) * (D / C));
            if (WITH_Q) qv[r] = __ldg(qs + (t + r) * (D / C));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            kd[(t + r) * (D / C)] = kv[r];
            vd[(t + r) * (D / C)] = vv[r];
            float f[C];
            unpack<C>(kv[r], f);
#pragma unroll
            for (int c = 0; c < C; ++c) acc[c] += static_cast<double>(f[c]);
            if (WITH_Q) {
                unpack<C>(qv[r], f);
#pragma unroll
                for (int c = 0; c < C; ++c) qacc[c] += static_cast<double>(f[c]);
            }
        }
    }
    for (; t < b; ++t) {
        V kv = __ldg(ks + t * (D / C));
        kd[t * (D / C)] = kv;
        vd[t * (D / C)] = __ldg(vs + t * (D / C));
        float f[C];
        unpack<C>(kv, f);
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] += static_cast<double>(f[c]);
        if (WITH_Q) {
            unpack<C>(__ldg(qs + t * (D / C)), f);
#pragma unroll
            for (int c = 0; c < C; ++c) qacc[c] += static_cast<double>(f[c]);
        }
    }
    const double db = static_cast<double>(b);
    float* dst = krep + (static_cast<int64_t>(u) * n_slots + slot) * D + lane * C;
#pragma unroll
    for (int c = 0; c < C; ++c) dst[c] = __double2float_rn(__ddiv_rn(acc[c], db));
    if (WITH_Q) {
        float* qd = qrep + (static_cast<int64_t>(u) * bpc + i) * D + lane * C;
#pragma unroll
        for (int c = 0; c < C; ++c) qd[c] = __double2float_rn(__ddiv_rn(qacc[c], db));
    }
}

// Bulk-copy form of write_chunk_kernel (the fused ingest, one PBSA call's Q/K/V pass): CTA per
// block.  One thread moves the block's b contiguous K, V (and Q) rows into shared memory with 1-D
// TMA bulk copies (b*d*2 bytes each, one mbarrier), streams K and V back out to the pool slot with
// two bulk stores, while thread c sums column c of K (threads d..2d-1: of Q) over the b rows in
// ascending token order in fp64 -- the same numerics as compress_kernel.  ~45 KB in flight per CTA
// instead of a few KB of warp loads: this kernel runs at HBM speed at config 2 and config 5.
template <int D, bool WITH_Q>
__global__ void __launch_bounds__(2 * D) write_chunk_bulk_kernel(const bf16* __restrict__ kc,
                                                                 const bf16* __restrict__ vc,
                                                                 const bf16* __restrict__ qcur,
                                                                 const int32_t* __restrict__ stage, int bpc, int b,
                                                                 int units, int n_slots, bf16* __restrict__ kp,
                                                                 bf16* __restrict__ vp, float* __restrict__ krep,
                                                                 float* __restrict__ qrep, int q_begin, int q_count) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const int u = blockIdx.x / bpc, i = blockIdx.x % bpc;
    // Q of query blocks [q_begin, q_begin + q_count) only (a rank's range in the batch-1 query
    // split; the whole chunk otherwise): qcur is [units][q_count * b][D], qrep keeps bpc rows/unit
    const bool has_q = WITH_Q && i >= q_begin && i < q_begin + q_count;
    const int slot = __ldg(stage + static_cast<int64_t>(u) * bpc + i);
    const uint32_t bytes = static_cast<uint32_t>(b) * D * 2;
    const int64_t src_off = (static_cast<int64_t>(u) * bpc + i) * b * D;
    const int64_t dst_off = (static_cast<int64_t>(u) * n_slots + slot) * 64 * D;
    bf16* ks = reinterpret_cast<bf16*>(smem);
    bf16* vs = reinterpret_cast<bf16*>(smem + bytes);
    bf16* qs = reinterpret_cast<bf16*>(smem + 2 * bytes);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(&bar, (has_q ? 3u : 2u) * bytes);
        bulk_g2s(ks, kc + src_off, bytes, &bar);
        bulk_g2s(vs, vc + src_off, bytes, &bar);
        if (has_q) bulk_g2s(qs, qcur + (static_cast<int64_t>(u) * q_count + (i - q_begin)) * b * D, bytes, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    if (tid == 0) {  // K and V rows [0, b) of the slot; rows >= b stay zero
        bulk_s2g(kp + dst_off, ks, bytes);
        bulk_s2g(vp + dst_off, vs, bytes);
        bulk_commit();
    }
    const int c = tid % D;
    const bool is_q = tid >= D;
    if (!is_q || has_q) {
        const bf16* col = (is_q ? qs : ks) + c;
        double acc = 0.0;
#pragma unroll 4
        for (int t = 0; t < b; ++t) acc += static_cast<double>(__bfloat162float(col[t * D]));
        const double r = __ddiv_rn(acc, static_cast<double>(b));
        if (is_q) qrep[(static_cast<int64_t>(u) * bpc + i) * D + c] = __double2float_rn(r);
        else krep[(static_cast<int64_t>(u) * n_slots + slot) * D + c] = __double2float_rn(r);
    }
    if (tid == 0) bulk_wait_read0();  // shared memory must outlive the bulk stores' reads
}

// write_chunk_bulk_kernel reading Latent4D chunk latents: the block's b tokens of head h are one
// 5-D TMA box {d, B_w, B_h, B_t, 1} at (h*d, nw*B_w, nh*B_h, nt*B_t, e), which lands in shared
// memory already in block-major in-block order (dt, dh, dw) -- blockify (blockify.cpp:38-65) is
// the TMA gather itself.  Then exactly the bulk kernel's slot store and fp64 column sums.
template <int D, bool WITH_Q>
__global__ void __launch_bounds__(2 * D) ingest_latent_kernel(const __grid_constant__ CUtensorMap tm_k,
                                                              const __grid_constant__ CUtensorMap tm_v,
                                                              const __grid_constant__ CUtensorMap tm_q,
                                                              const LatentGeom g, const int32_t* __restrict__ stage,
                                                              int n_slots, bf16* __restrict__ kp, bf16* __restrict__ vp,
                                                              float* __restrict__ krep, float* __restrict__ qrep) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const int bpc = g.nqb(), b = g.b();
    const int u = blockIdx.x / bpc, i = blockIdx.x % bpc;
    const int e = u / g.heads, h = u % g.heads;
    const int nw = i % g.nw(), nh = (i / g.nw()) % g.nh(), nt = i / (g.nw() * g.nh());
    const int slot = __ldg(stage + static_cast<int64_t>(u) * bpc + i);
    const uint32_t bytes = static_cast<uint32_t>(b) * D * 2;
    const int64_t dst_off = (static_cast<int64_t>(u) * n_slots + slot) * 64 * D;
    bf16* ks = reinterpret_cast<bf16*>(smem);
    bf16* vs = reinterpret_cast<bf16*>(smem + bytes);
    bf16* qs = reinterpret_cast<bf16*>(smem + 2 * bytes);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(&bar, (WITH_Q ? 3u : 2u) * bytes);
        tma_load_5d(ks, &tm_k, &bar, h * D, nw * g.bw, nh * g.bh, nt * g.bt, e);
        tma_load_5d(vs, &tm_v, &bar, h * D, nw * g.bw, nh * g.bh, nt * g.bt, e);
        if (WITH_Q) tma_load_5d(qs, &tm_q, &bar, h * D, nw * g.bw, nh * g.bh, nt * g.bt, e);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    if (tid == 0) {
        bulk_s2g(kp + dst_off, ks, bytes);
        bulk_s2g(vp + dst_off, vs, bytes);
        bulk_commit();
    }
    const int c = tid % D;
    const bool is_q = tid >= D;
    if (!is_q || WITH_Q) {
        const bf16* col = (is_q ? qs : ks) + c;
        double acc = 0.0;
#pragma unroll 4
        for (int t = 0; t < b; ++t) acc += static_cast<double>(__bfloat162float(col[t * D]));
        const double r = __ddiv_rn(acc, static_cast<double>(b));
        if (is_q) qrep[(static_cast<int64_t>(u) * bpc + i) * D + c] = __double2float_rn(r);
        else krep[(static_cast<int64_t>(u) * n_slots + slot) * D + c] = __double2float_rn(r);
    }
    if (tid == 0) bulk_wait_read0();
}

// Bulk variant (the hot path's Q compression): CTA per block, thread per column.  The block's b
// contiguous token rows arrive in ONE bulk copy (every block's bytes in flight at once, where the
// warp-per-block kernel above needs b / 16 dependent round trips), then each thread sums its
// column from shared memory in ascending token order -- the same fp64 chain, bit-identical.
template <int D>
__global__ void __launch_bounds__(D) compress_bulk_kernel(const bf16* __restrict__ x, int64_t xu, int64_t xb,
                                                           const int32_t* __restrict__ map, int nb, int b,
                                                           float* __restrict__ reps, int64_t ru) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    const int u = blockIdx.x / nb, i = blockIdx.x % nb;
    const int idx = map ? __ldg(map + static_cast<int64_t>(u) * nb + i) : i;
    const uint32_t bytes = static_cast<uint32_t>(b) * D * 2;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(&bar, bytes);
        bulk_g2s(smem, x + u * xu + static_cast<int64_t>(idx) * xb, bytes, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    const bf16* col = reinterpret_cast<const bf16*>(smem) + threadIdx.x;
    double acc = 0.0;
#pragma unroll 4
    for (int t = 0; t < b; ++t) acc += static_cast<double>(__bfloat162float(col[t * D]));
    reps[u * ru + static_cast<int64_t>(idx) * D + threadIdx.x] = __double2float_rn(__ddiv_rn(acc, static_cast<double>(b)));
}

}  // namespace

int launch_compress(const bf16* x, int64_t xu, int64_t xb, const int32_t* map, int nb, int units,
                    int b, int d, float* reps, int64_t ru, cudaStream_t s) {
    const int64_t warps = static_cast<int64_t>(nb) * units;
    if (warps == 0) return 0;
    // bulk copies need 16-byte aligned, 16-byte multiple block rows (always true for d = 64 / 128
    // block-major inputs)
    const bool bulk = (reinterpret_cast<uintptr_t>(x) & 15u) == 0 && (xu % 8) == 0 && (xb % 8) == 0 &&
                      warps < (int64_t(1) << 31);
    if (bulk) {
        const size_t smem = static_cast<size_t>(b) * d * 2;
        if (d == 128)
            launch_pdl(compress_bulk_kernel<128>, dim3(static_cast<unsigned>(warps)), dim3(128), smem, s, x, xu, xb,
                       map, nb, b, reps, ru);
        else
            launch_pdl(compress_bulk_kernel<64>, dim3(static_cast<unsigned>(warps)), dim3(64), smem, s, x, xu, xb,
                       map, nb, b, reps, ru);
        return check_launch("compress_bulk_kernel");
    }
    const int grid = static_cast<int>((warps + 7) / 8);
    if (d == 128)
        launch_pdl(compress_kernel<128>, dim3(grid), dim3(256), 0, s, x, xu, xb, map, nb, units, b, reps, ru);
    else
        launch_pdl(compress_kernel<64>, dim3(grid), dim3(256), 0, s, x, xu, xb, map, nb, units, b, reps, ru);
    return check_launch("compress_kernel");
}

int launch_write_chunk(const bf16* kc, const bf16* vc, const bf16* q, const int32_t* stage, int bpc, int b,
                       int d, int units, int n_slots, bf16* kp, bf16* vp, float* krep, float* qrep,
                       cudaStream_t s, int q_begin, int q_count) {
    if (q_count < 0) q_count = bpc;
    const int64_t warps = static_cast<int64_t>(bpc) * units;
    if (warps == 0) return 0;
    const size_t smem = (q ? 3 : 2) * static_cast<size_t>(b) * d * 2;
    if (smem <= 200 * 1024 && warps < (int64_t(1) << 31)) {
#define PBSA_WCB(DD, WQ)                                                                                        \
    do {                                                                                                         \
        if (int rc = ensure_smem(reinterpret_cast<const void*>(write_chunk_bulk_kernel<DD, WQ>), smem,          \
                                 "write_chunk"))                                                                 \
            return rc;                                                                                           \
        launch_pdl(write_chunk_bulk_kernel<DD, WQ>, dim3(static_cast<unsigned>(warps)), dim3(2 * DD), smem, s, kc,  \
                   vc, q, stage, bpc, b, units, n_slots, kp, vp, krep, qrep, q_begin, q_count);                 \
    } while (0)
        if (d == 128) {
            if (q) PBSA_WCB(128, true); else PBSA_WCB(128, false);
        } else {
            if (q) PBSA_WCB(64, true); else PBSA_WCB(64, false);
        }
#undef PBSA_WCB
        return check_launch("write_chunk_bulk_kernel");
    }
    if (q && (q_begin != 0 || q_count != bpc))
        return set_error(PBSA_EUNSUPPORTED, "write_chunk: query-block range needs the bulk kernel");
    const int grid = static_cast<int>((warps + 7) / 8);
    count_launch();
#define PBSA_WC(DD, WQ) write_chunk_kernel<DD, WQ><<<grid, 256, 0, s>>>(kc, vc, q, stage, bpc, b, units, n_slots, kp, vp, krep, qrep)
    if (d == 128) {
        if (q) PBSA_WC(128, true); else PBSA_WC(128, false);
    } else {
        if (q) PBSA_WC(64, true); else PBSA_WC(64, false);
    }
#undef PBSA_WC
    return check_launch("write_chunk_kernel");
}

int launch_ingest_latent(const bf16* k_lat, const bf16* v_lat, const bf16* q_lat, const LatentGeom& g,
                         const int32_t* stage, int n_slots, bf16* kp, bf16* vp, float* krep, float* qrep,
                         cudaStream_t s) {
    const int64_t ctas = static_cast<int64_t>(g.batch) * g.heads * g.nqb();
    if (ctas == 0) return 0;
    alignas(64) CUtensorMap tk, tv, tq;
    std::string err;
    if (!encode_latent_tmap(&tk, k_lat, g, g.d, false, &err) || !encode_latent_tmap(&tv, v_lat, g, g.d, false, &err) ||
        (q_lat && !encode_latent_tmap(&tq, q_lat, g, g.d, false, &err)))
        return set_error(PBSA_ECUDA, "ingest_latent: tensor map: " + err);
    if (!q_lat) tq = tk;
    const size_t smem = (q_lat ? 3 : 2) * static_cast<size_t>(g.b()) * g.d * 2;
    if (smem > 200 * 1024) return set_error(PBSA_EUNSUPPORTED, "ingest_latent: block too large for shared memory");
#define PBSA_IL(DD, WQ)                                                                                         \
    do {                                                                                                         \
        if (int rc = ensure_smem(reinterpret_cast<const void*>(ingest_latent_kernel<DD, WQ>), smem, "ingest")) \
            return rc;                                                                                           \
        launch_pdl(ingest_latent_kernel<DD, WQ>, dim3(static_cast<unsigned>(ctas)), dim3(2 * DD), smem, s, tk, tv, \
                   tq, g, stage, n_slots, kp, vp, krep, qrep);                                                  \
    } while (0)
    if (g.d == 128) {
        if (q_lat) PBSA_IL(128, true); else PBSA_IL(128, false);
    } else {
        if (q_lat) PBSA_IL(64, true); else PBSA_IL(64, false);
    }
#undef PBSA_IL
    return check_launch("ingest_latent_kernel");
}

}  // namespace pbsa
