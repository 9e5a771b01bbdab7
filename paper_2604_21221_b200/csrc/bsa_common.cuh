// bsa_common.cuh -- shared by the K3 kernels (bsa_fwd.cu): launch parameters, the tile schedule
// (whole-tile waves, hybrid stream-K tail, unit gangs) and the visible-list builder.
//
// Fragment f of CTA (tile slot) vc is a whole tile or (in the stream-K tail) a contiguous range of
// one tile's visible list.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>

#include "internal.h"
#include "ptx.cuh"

namespace pbsa {

constexpr int kRing = 2;  // partial-output slots per CTA (stream-K tail: first and last fragment)
constexpr uint32_t kTmemCols = 256;
// a block whose row sum (against the running max) exceeds this takes the exact rescale path
constexpr float kOverflowSum = 65536.0f;
// column pairs whose exp2 runs as a polynomial on the FMA pipe instead of MUFU (bit c2 = pair c2)
constexpr uint32_t kPolyMask = 0u;  // MUFU-only: the softmax is issue/latency-bound, not MUFU-bound

struct BsaParams {
    int units, nqb, b, n_slots;
    const int32_t* dense;
    int dense_stride, n_dense;
    const int32_t* local;
    int local_stride, n_local;
    const int32_t* sel;
    int k;
    int sel_rows, sel_row0;  // sel is [units][sel_rows][k]; query block i of the launch reads row sel_row0 + i
    const int32_t* pairs;    // [units][tiles_per_unit][2] query blocks of each tile (second -1: none);
                             // null: tile t holds query blocks 2t and 2t + 1
    bf16* o;
    float* lse;
    float scale_log2;
    int max_list, bm_words;
    int lat;        // q / o are chunk latents (LatentGeom lg), not block-major [units][n_q][d]
    LatentGeom lg;
    long long* trace;  // perf experiments only: per-event clock64 stamps of CTA 0 (null = off)
    int ablate;  // perf experiments only (PBSA_ABLATE): bit 0 no softmax math, bit 1 no K/V loads, bit 2 no MMAs
    // schedule: `whole_waves` rounds of one whole tile per CTA (tile = cta + w * grid), then the
    // remaining tiles [tail_base, n_tiles) split stream-K over the first tail_grid CTAs
    int tiles_per_unit, n_tiles, grid;
    int whole_waves, tail_base, tail_grid;
    int64_t vlen, vtotal;  // virtual length of one tile (upper bound of its list) and of the tail
    float* part_o;         // [kRing*grid][128][D] fp32 (null -> whole tiles only)
    float* part_ml;        // [kRing*grid][2][128]
    int* counters;         // [n_tiles], zero between launches
    // unit-gang schedule (gangs > 0): CTA c = gang c / tiles_per_unit, member c % tiles_per_unit;
    // gang g takes units g, g + gangs, ... one whole tile per member per unit, and the members'
    // producers pass a barrier (gang_ctr[g]) between units so all tiles of a unit stream its pool
    // together (the KV blocks they share are fetched from DRAM once and served from L2)
    int gangs;
    int* gang_ctr;         // [gangs (+1 extra)] + done counter at [kMaxGangs], zero between launches
    // extra gang (gangs > 0, extra > 0): the `extra` CTA slots left over by the full gangs form one
    // more gang that takes the last `xunits` units, member m covering tiles m and m + extra of each
    // (two per unit when extra < tiles_per_unit), with its own unit barrier (gang_ctr[gangs])
    int extra, xunits;
};
constexpr int kMaxGangs = 1024;

struct FragMeta {
    int tile, u, qb0, qb1;  // qb1 < 0: the tile's second half is empty
    int n, e0, e1;   // list length and the entry range of this fragment
    int whole, nf, slot;
    int first_cta;   // first CTA holding a fragment of this tile (for the merge)
    int pad;
};

namespace {

// CTA holding virtual position x (stream-K ranges B_c = floor(c * W / G))
__device__ __forceinline__ int cta_of(int64_t x, int64_t W, int G) {
    return static_cast<int>(((x + 1) * G - 1) / W);
}
__device__ __forceinline__ int64_t range_begin(int c, int64_t W, int G) { return (static_cast<int64_t>(c) * W) / G; }

// number of fragments this CTA processes
__device__ __forceinline__ int num_fragments(const BsaParams& p, int c) {
    if (c >= p.grid) return 0;
    if (p.gangs > 0) {
        const int main_cta = p.gangs * p.tiles_per_unit, main_units = p.units - p.xunits;
        if (c < main_cta) {
            const int g = c / p.tiles_per_unit;
            return g < main_units ? (main_units - 1 - g) / p.gangs + 1 : 0;
        }
        const int m = c - main_cta;  // extra-gang member
        return p.xunits * (m + p.extra < p.tiles_per_unit ? 2 : 1);
    }
    if (p.part_o == nullptr) return c < p.n_tiles ? (p.n_tiles - 1 - c) / p.grid + 1 : 0;
    if (c >= p.tail_grid || p.vtotal == 0) return p.whole_waves;
    const int64_t a = range_begin(c, p.vtotal, p.tail_grid), b = range_begin(c + 1, p.vtotal, p.tail_grid);
    if (b <= a) return p.whole_waves;
    return p.whole_waves + static_cast<int>((b - 1) / p.vlen - a / p.vlen) + 1;
}

// fragment f of virtual CTA vc: which tile, and (stream-K tail) which part of its list
struct FragPlan {
    int tile, u, qb0, qb1;
    int64_t va, vb;  // virtual range [va, vb) of the tile's list (vlen = whole tile)
    int nfr, first_cta, slot;
};

__device__ __forceinline__ FragPlan plan_fragment(const BsaParams& p, int vc, int f) {
    const bool in_tail = p.gangs == 0 && p.part_o != nullptr && vc < p.tail_grid;
    const int64_t my_begin = in_tail ? range_begin(vc, p.vtotal, p.tail_grid) : 0;
    const int64_t my_end = in_tail ? range_begin(vc + 1, p.vtotal, p.tail_grid) : 0;
    const int my_first_tile = p.tail_base + static_cast<int>(my_begin / p.vlen);  // first tail tile
    const bool tail_frag = p.gangs == 0 && p.part_o != nullptr && f >= p.whole_waves;
    FragPlan fp;
    fp.tile = tail_frag ? my_first_tile + (f - p.whole_waves) : vc + f * p.grid;
    if (p.gangs > 0) {
        const int main_cta = p.gangs * p.tiles_per_unit;
        if (vc < main_cta) {
            const int g = vc / p.tiles_per_unit;
            fp.tile = (g + f * p.gangs) * p.tiles_per_unit + vc % p.tiles_per_unit;
        } else {  // extra gang: per unit one or two tiles (m, m + extra)
            const int m = vc - main_cta, k = m + p.extra < p.tiles_per_unit ? 2 : 1;
            const int unit = p.units - p.xunits + f / k;
            fp.tile = unit * p.tiles_per_unit + m + (f % k) * p.extra;
        }
    }
    fp.u = fp.tile / p.tiles_per_unit;
    if (p.pairs != nullptr) {
        fp.qb0 = __ldg(p.pairs + 2 * static_cast<int64_t>(fp.tile));
        fp.qb1 = __ldg(p.pairs + 2 * static_cast<int64_t>(fp.tile) + 1);
    } else {
        fp.qb0 = 2 * (fp.tile % p.tiles_per_unit);
        fp.qb1 = fp.qb0 + 1 < p.nqb ? fp.qb0 + 1 : -1;
    }
    fp.va = 0;
    fp.vb = p.vlen;
    fp.nfr = 1;
    fp.first_cta = vc;
    if (tail_frag) {
        const int64_t t0 = static_cast<int64_t>(fp.tile - p.tail_base) * p.vlen;
        fp.va = (my_begin > t0 ? my_begin : t0) - t0;
        fp.vb = (my_end < t0 + p.vlen ? my_end : t0 + p.vlen) - t0;
        fp.first_cta = cta_of(t0, p.vtotal, p.tail_grid);
        fp.nfr = cta_of(t0 + p.vlen - 1, p.vtotal, p.tail_grid) - fp.first_cta + 1;
    }
    fp.slot = 2 * vc + (fp.tile == my_first_tile ? 0 : 1);
    return fp;
}

__device__ __forceinline__ FragMeta make_meta(const BsaParams& p, const FragPlan& fp, int run) {
    FragMeta fm;
    fm.tile = fp.tile;
    fm.u = fp.u;
    fm.qb0 = fp.qb0;
    fm.qb1 = fp.qb1;
    fm.n = run;
    fm.e0 = static_cast<int>((fp.va * run) / p.vlen);
    fm.e1 = static_cast<int>((fp.vb * run) / p.vlen);
    fm.whole = (fp.nfr == 1);
    fm.nf = fp.nfr;
    fm.slot = fp.slot;
    fm.first_cta = fp.first_cta;
    fm.pad = 0;
    return fm;
}

// unit gangs: before its first fragment of a unit, lane 0 waits until every member of vc's gang has
// issued all loads of the previous unit (members arrive once per unit, after their last fragment of it)
__device__ __forceinline__ void gang_wait(const BsaParams& p, int vc, int f) {
    if (p.gangs > 0 && (threadIdx.x & 31) == 0) {
        const int main_cta = p.gangs * p.tiles_per_unit;
        if (vc < main_cta) {
            if (f > 0) {
                const int want = f * p.tiles_per_unit;
                while (ld_acquire_gpu(p.gang_ctr + vc / p.tiles_per_unit) < want) __nanosleep(64);
            }
        } else {
            const int k = (vc - main_cta) + p.extra < p.tiles_per_unit ? 2 : 1;
            const int i = f / k;
            if (i > 0 && f % k == 0) {
                const int want = i * p.extra;
                while (ld_acquire_gpu(p.gang_ctr + p.gangs) < want) __nanosleep(64);
            }
        }
    }
    __syncwarp();
}
__device__ __forceinline__ void gang_arrive(const BsaParams& p, int vc, int f) {
    if (p.gangs > 0 && (threadIdx.x & 31) == 0) {
        const int main_cta = p.gangs * p.tiles_per_unit;
        if (vc < main_cta) {
            red_release_gpu_add(p.gang_ctr + vc / p.tiles_per_unit, 1);
        } else {
            const int k = (vc - main_cta) + p.extra < p.tiles_per_unit ? 2 : 1;
            if (f % k == k - 1) red_release_gpu_add(p.gang_ctr + p.gangs, 1);
        }
    }
}

// The visible list of a tile (warp-collective): dense blocks first (both halves see them), then
// the union of the two query blocks' Top-K selections in ascending local order, each entry the
// pool slot plus a 2-bit mask of the halves that see it (bits 24-25, or 14-15 for 16-bit entries
// over pools < 16384 slots).  bm: 2 * bm_words words of scratch.  Returns the list length.
template <bool L16>
__device__ __forceinline__ void list_put(uint8_t* base, int i, int slot, int mask) {
    if (L16) reinterpret_cast<uint16_t*>(base)[i] = static_cast<uint16_t>(slot | (mask << 14));
    else reinterpret_cast<int32_t*>(base)[i] = slot | (mask << 24);
}
template <bool L16>
__device__ __forceinline__ int list_slot(const uint8_t* base, int i) {
    return L16 ? static_cast<int>(reinterpret_cast<const uint16_t*>(base)[i] & 0x3FFF)
               : (reinterpret_cast<const int32_t*>(base)[i] & 0xFFFFFF);
}
template <bool L16>
__device__ __forceinline__ int list_mask(uint32_t ent) {
    return static_cast<int>((ent >> (L16 ? 14 : 24)) & 3u);
}

template <bool L16>
__device__ int build_visible_list(const BsaParams& p, const FragPlan& fp, uint8_t* list, uint32_t* bm) {
    // Global loads are issued 8 per lane ahead of their consumers (the list is built before the
    // fragment's first TMA can be issued, so a serial load -> store chain here is launch latency).
    constexpr int kB = 8;
    const int lane = threadIdx.x & 31;
    const int u = fp.u;
    for (int w = lane; w < 2 * p.bm_words; w += 32) bm[w] = 0u;
    __syncwarp();
    if (p.k > 0 && p.n_local > 0) {
        const int sel_rows = fp.qb1 >= 0 ? 2 : 1, total = sel_rows * p.k;
        const int32_t* srow0 = p.sel + (static_cast<int64_t>(u) * p.sel_rows + p.sel_row0 + fp.qb0) * p.k;
        const int32_t* srow1 = p.sel + (static_cast<int64_t>(u) * p.sel_rows + p.sel_row0 + (fp.qb1 >= 0 ? fp.qb1 : 0)) * p.k;
        for (int e0 = 0; e0 < total; e0 += 32 * kB) {
            int idx[kB];
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const int e = e0 + i * 32 + lane;
                idx[i] = e < total ? __ldg(e < p.k ? srow0 + e : srow1 + (e - p.k)) : -1;
            }
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const int e = e0 + i * 32 + lane;
                if (e < total) atomicOr(&bm[(e >= p.k ? p.bm_words : 0) + (idx[i] >> 5)], 1u << (idx[i] & 31));
            }
        }
    }
    const int32_t* drow = p.dense + static_cast<int64_t>(u) * p.dense_stride;
    for (int e0 = 0; e0 < p.n_dense; e0 += 32 * kB) {
        int v[kB];
#pragma unroll
        for (int i = 0; i < kB; ++i) {
            const int e = e0 + i * 32 + lane;
            v[i] = e < p.n_dense ? __ldg(drow + e) : 0;
        }
#pragma unroll
        for (int i = 0; i < kB; ++i) {
            const int e = e0 + i * 32 + lane;
            if (e < p.n_dense) list_put<L16>(list, e, v[i], 3);
        }
    }
    __syncwarp();
    // union of the two bitmaps in ascending local order: first the local INDICES (a pure
    // shared-memory pass), then one batched gather of their pool slots
    int run = p.n_dense;
    for (int w0 = 0; w0 < p.bm_words; w0 += 32) {
        const int w = w0 + lane;
        const uint32_t a = w < p.bm_words ? bm[w] : 0u;
        const uint32_t c = w < p.bm_words ? bm[p.bm_words + w] : 0u;
        uint32_t un = a | c;
        const int cnt = __popc(un);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int pos = run + incl - cnt;
        while (un) {
            const int bit = __ffs(un) - 1;
            un &= un - 1;
            const int mask = static_cast<int>((a >> bit) & 1u) | (static_cast<int>((c >> bit) & 1u) << 1);
            list_put<L16>(list, pos++, w * 32 + bit, mask);
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    const int32_t* loc = p.local + static_cast<int64_t>(u) * p.local_stride;
    for (int e0 = p.n_dense; e0 < run; e0 += 32 * kB) {
        int v[kB], mk[kB];
#pragma unroll
        for (int i = 0; i < kB; ++i) {
            const int e = e0 + i * 32 + lane;
            v[i] = 0;
            mk[i] = 0;
            if (e < run) {
                const uint32_t ent = L16 ? reinterpret_cast<const uint16_t*>(list)[e] : reinterpret_cast<const uint32_t*>(list)[e];
                mk[i] = list_mask<L16>(ent);
                v[i] = __ldg(loc + static_cast<int>(L16 ? (ent & 0x3FFFu) : (ent & 0xFFFFFFu)));
            }
        }
#pragma unroll
        for (int i = 0; i < kB; ++i) {
            const int e = e0 + i * 32 + lane;
            if (e < run) list_put<L16>(list, e, v[i], mk[i]);
        }
    }
    __syncwarp();
    return run;
}


// ---------------------------------------------------------------------------------------- host side
inline int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// tensor maps of Q (3-D over [units*nqb][b][D], or the 5-D chunk latent), K and V (2-D over the
// slot pools, 64 x 64 boxes)
inline int encode_k3_maps(const bf16* q, const bf16* kp, const bf16* vp, const BsaParams& p, int D, CUtensorMap* tq,
                          CUtensorMap* tk, CUtensorMap* tv) {
    std::string err;
    if (p.lat) {
        if (!encode_latent_tmap(tq, q, p.lg, 64, true, &err)) return set_error(PBSA_ECUDA, "tensor map Q (latent): " + err);
    } else {
        const uint64_t dims[3] = {static_cast<uint64_t>(D), static_cast<uint64_t>(p.b),
                                  static_cast<uint64_t>(p.units) * p.nqb};
        const uint64_t strides[2] = {static_cast<uint64_t>(D) * 2, static_cast<uint64_t>(p.b) * D * 2};
        const uint32_t box[3] = {64, static_cast<uint32_t>(p.b), 1};
        if (!encode_tmap_bf16(tq, q, 3, dims, strides, box, &err)) return set_error(PBSA_ECUDA, "tensor map Q: " + err);
    }
    const uint64_t dims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(p.units) * p.n_slots * 64};
    const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
    const uint32_t box[2] = {64, static_cast<uint32_t>(p.b)};  // the b valid rows of a 64-row slot
    if (!encode_tmap_bf16(tk, kp, 2, dims, strides, box, &err)) return set_error(PBSA_ECUDA, "tensor map K: " + err);
    if (!encode_tmap_bf16(tv, vp, 2, dims, strides, box, &err)) return set_error(PBSA_ECUDA, "tensor map V: " + err);
    return PBSA_OK;
}

// The schedule over `slots` virtual CTAs (tile-processing slots that run concurrently):
// whole tiles, the hybrid stream-K tail (with a workspace), or unit gangs (config-5-sized launches).
inline void plan_schedule(BsaParams& p, int slots, int D) {
    p.grid = p.n_tiles < slots ? p.n_tiles : slots;
    p.whole_waves = 0;
    p.tail_base = 0;
    p.tail_grid = 0;
    p.vtotal = 0;
    p.gangs = 0;
    p.extra = 0;
    p.xunits = 0;
    if (p.gang_ctr != nullptr) {
        // unit-gang schedule: many whole-tile waves over a slot pool far larger than L2 (config 5:
        // 12480 tiles, 65 GB) -- tiles of one unit run together so the blocks they share come from
        // DRAM once.  PBSA_K3_GANG=0/1 forces it off / on (experiments, tests).
        const char* env = getenv("PBSA_K3_GANG");
        const int force = env ? atoi(env) : -1;
        const int gangs = slots / p.tiles_per_unit;
        const double pool = static_cast<double>(p.units) * p.n_slots * 64 * D * 2 * 2;
        const bool want = force >= 0 ? force > 0 : (p.n_tiles >= 4 * slots && pool > 4.0 * 126e6);
        if (want && gangs >= 1 && gangs <= kMaxGangs) {
            p.gangs = gangs < p.units ? gangs : p.units;
            p.grid = p.gangs * p.tiles_per_unit;
            p.part_o = nullptr;
            // the leftover slots as one extra gang when it can cover a unit in at most two rounds:
            // it gets the share of the units its rate (1/2 or 1 unit per round) earns
            // (PBSA_K3_EXTRA_GANG=0: off, experiments)
            const char* xenv = getenv("PBSA_K3_EXTRA_GANG");
            int e = slots - p.gangs * p.tiles_per_unit;
            if (e > p.tiles_per_unit) e = p.tiles_per_unit;
            if ((xenv == nullptr || atoi(xenv) != 0) && p.gangs == gangs && p.gangs < kMaxGangs &&
                2 * e >= p.tiles_per_unit) {
                const double rate = e >= p.tiles_per_unit ? 1.0 : 0.5;
                int x = static_cast<int>(p.units * rate / (p.gangs + rate) + 0.5);
                const char* xu = getenv("PBSA_K3_EXTRA_UNITS");  // experiments: the extra gang's units
                if (xu != nullptr && atoi(xu) > 0) x = atoi(xu);
                if (x >= 1 && x < p.units) {
                    p.extra = e;
                    p.xunits = x;
                    p.grid += e;
                }
            }
        }
    }
    if (p.part_o != nullptr) {
        p.grid = slots;
        p.whole_waves = p.n_tiles / slots;
        p.tail_base = p.whole_waves * slots;
        const int64_t tail = p.n_tiles - p.tail_base;
        p.vtotal = tail * p.vlen;
        // at most ~cap slots share a tail tile (the merge handles up to 8 fragments)
        // (PBSA_K3_TAILCAP: experiments and tests; 4 measured best, tools/host_bound_check.py)
        const char* cap_env = getenv("PBSA_K3_TAILCAP");
        const int cap = cap_env && atoi(cap_env) >= 1 && atoi(cap_env) <= 8 ? atoi(cap_env) : 4;
        int64_t g = slots;
        if (g > p.vtotal) g = p.vtotal;
        if (g > cap * tail) g = cap * tail;
        p.tail_grid = static_cast<int>(g);
        if (p.whole_waves == 0) p.grid = p.tail_grid;
    }
}

inline void record_plan(const BsaParams& p, bool l16, int per_sm, size_t smem) {
    pbsa_bsa_plan& pl = last_bsa_plan();
    pl.list_entry_bytes = l16 ? 2 : 4;
    pl.ctas_per_sm = per_sm;
    pl.grid = p.grid > 0 ? p.grid : 0;
    pl.schedule = p.gangs > 0 ? PBSA_SCHED_UNIT_GANGS : (p.part_o != nullptr ? PBSA_SCHED_STREAM_K : PBSA_SCHED_WHOLE_TILES);
    pl.gangs = p.gangs;
    pl.max_list = p.max_list;
    pl.n_tiles = p.n_tiles;
    pl.smem_bytes = smem;
}

}  // namespace
}  // namespace pbsa
