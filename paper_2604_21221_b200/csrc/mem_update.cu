// mem_update.cu -- K4 persistent-memory update, in place in the slot pool.
//
// Reference ops (Eq. 9; Alg. 1):
//   push_chunk        the stage chunk joins the local window L; on overflow the oldest chunk E
//                     is evicted whole
//   update_persistent blocks of the first chunk are sinks, always kept (footnote of Eq. 9,
//                     SPEC.md:228); dynamic <- Top-(C-|S|) of (dynamic U E) by
//                     (s_t desc, id asc), scores refreshed from this s_t (:227)
//   assemble_kv       no copy: the dense / local / key slot tables are rewritten in the SPEC
//                     order [sinks id asc; dynamic id asc; L oldest -> newest] (+ stage)
// K/V/representatives never move: a block keeps its slot from the moment it is written as the
// current chunk until it is dropped, when the slot returns to the free stack and is reused as
// a stage slot.  All counts are structural (identical across units, tracked on the host), only
// the identities are data dependent, so one CTA per unit suffices and nothing syncs the host.
//
// Roofline: HBM (candidate scores + slot tables); launch-latency bound at Wan-1.3B shape.
#include "internal.h"
#include "ptx.cuh"
#include "select_warp.cuh"

namespace pbsa {
namespace {

struct CommitParams {
    MemDev m;
    const float* s_t;
    int C, Lcap, bpc, S;
    MemCounts cur, next;
    int fault;  // kFaultDropSink: sinks compete with the dynamic candidates (negative control)
};

__global__ void mem_init_kernel(MemDev m, int C, int Lcap, int bpc, int S) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *m.status = 0;
    const int u = blockIdx.x;
    for (int i = threadIdx.x; i < bpc; i += blockDim.x) {
        m.stage[static_cast<int64_t>(u) * bpc + i] = i;
        m.dense[static_cast<int64_t>(u) * (C + bpc) + i] = i;
        m.keys[static_cast<int64_t>(u) * S + i] = i;
    }
    for (int i = threadIdx.x; i < S - bpc; i += blockDim.x) m.free_slot[static_cast<int64_t>(u) * S + i] = S - 1 - i;
}

__global__ void __launch_bounds__(256) mem_commit_kernel(const CommitParams p) {
    pdl_wait();  // programmatic dependent launch: upstream outputs are visible from here on
    extern __shared__ __align__(16) uint8_t smem[];
    const int u = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int C = p.C, Lcap = p.Lcap, bpc = p.bpc, S = p.S;
    const int n_p = p.cur.n_p, n_s = p.cur.n_sinks, n_l = p.cur.n_l, n_free = p.cur.n_free;
    const int n_keys = n_p + n_l + bpc;
    const int max_cand = C + bpc;
    // smem carve-up
    int64_t* c_id = reinterpret_cast<int64_t*>(smem);                // [max_cand]
    int64_t* l_id = c_id + max_cand;                                 // [Lcap]
    float* c_score = reinterpret_cast<float*>(l_id + Lcap);          // [max_cand]
    int32_t* c_slot = reinterpret_cast<int32_t*>(c_score + max_cand);  // [max_cand]
    int32_t* c_keep = c_slot + max_cand;                             // [max_cand]
    int32_t* l_slot = c_keep + max_cand;                             // [Lcap]
    int32_t* stage = l_slot + Lcap;                                  // [bpc]
    int32_t* freel = stage + bpc;                                    // [S]
    int32_t* np_slot = freel + S;                                    // [C]  new P
    int64_t* np_id;                                                  // aligned below
    {
        uintptr_t a = reinterpret_cast<uintptr_t>(np_slot + C);
        np_id = reinterpret_cast<int64_t*>((a + 7) & ~uintptr_t(7));
    }
    float* np_score = reinterpret_cast<float*>(np_id + C);           // [C]
    __shared__ int s_new_np, s_ndrop;

    const int64_t uP = static_cast<int64_t>(u) * C, uL = static_cast<int64_t>(u) * Lcap;
    const float* st = p.s_t + static_cast<int64_t>(u) * n_keys;
    const bool evict = n_l + bpc > Lcap;
    const bool sink_chunk = evict && (p.cur.chunk - Lcap / bpc == 0);

    // 1. stage the state in smem.  Candidates: [P (sinks, dynamic)] ++ [E] with fresh scores.
    for (int i = tid; i < n_p; i += nt) {
        c_id[i] = p.m.p_id[uP + i];
        c_slot[i] = p.m.p_slot[uP + i];
        c_score[i] = st[i];
    }
    for (int i = tid; i < n_l; i += nt) {
        l_id[i] = p.m.l_id[uL + i];
        l_slot[i] = p.m.l_slot[uL + i];
    }
    for (int i = tid; i < bpc; i += nt) stage[i] = p.m.stage[static_cast<int64_t>(u) * bpc + i];
    for (int i = tid; i < n_free; i += nt) freel[i] = p.m.free_slot[static_cast<int64_t>(u) * S + i];
    __syncthreads();
    const int n_cand = evict ? n_p + bpc : n_p;
    if (evict) {
        for (int i = tid; i < bpc; i += nt) {
            c_id[n_p + i] = l_id[i];
            c_slot[n_p + i] = l_slot[i];
            c_score[n_p + i] = st[n_p + i];
        }
    }
    __syncthreads();
    // 2. keep flags.  Sinks (and, on the sink chunk's eviction, the whole E) are kept.  The
    //    dynamic candidates [n_s, n_cand) compete: rank = #candidates ordered before by
    //    (score desc, id asc); keep rank < C - |S'|.
    const int n_sinks_new = sink_chunk ? bpc : n_s;
    const int dyn_lo = sink_chunk ? n_p + bpc : n_s;  // first competing candidate
    // with sink_chunk, the dynamic set is empty (nothing was evicted before the first chunk)
    const int dyn_cap = C - n_sinks_new;
    if (p.fault == kFaultDropSink && !sink_chunk) {
        // injected fault: every candidate, sinks included, competes for all C slots -- the
        // kept count (and so the slot accounting) is unchanged, only sink retention is broken
        for (int i = tid; i < n_cand; i += nt) {
            int rank = 0;
            for (int j = 0; j < n_cand; ++j) rank += topc_before(c_score[j], c_id[j], c_score[i], c_id[i]);
            c_keep[i] = rank < C;
        }
    } else
    for (int i = tid; i < n_cand; i += nt) {
        int keep = 1;
        if (i >= n_s && !(sink_chunk && i >= n_p)) {
            // (score desc, id asc) is a strict total order once NaN (invalid input, which the
            // reference rejects, tensor.cpp:61-64) ranks below every number: exactly dyn_cap
            // candidates survive whatever the scores are, so the slot accounting stays exact
            int rank = 0;
            for (int j = n_s; j < n_cand; ++j) {
                if (sink_chunk && j >= n_p) break;
                rank += topc_before(c_score[j], c_id[j], c_score[i], c_id[i]);
            }
            keep = rank < dyn_cap;
            if (c_score[i] != c_score[i]) atomicOr(p.m.status, 2);
        }
        c_keep[i] = keep;
    }
    (void)dyn_lo;
    __syncthreads();
    // 3. order-preserving compaction by warp 0.  Candidate order is already [sinks id asc,
    //    dynamic id asc, E id asc] and E is younger than every dynamic block, so the kept
    //    candidates come out as [sinks; dynamic id asc] except that on the sink chunk's
    //    eviction E (the new sinks) must precede the (empty) dynamic set.
    if (tid < 32) {
        const int lane = tid;
        int run = 0, drop = 0;
        for (int base = 0; base < n_cand; base += 32) {
            const int i = base + lane;
            const bool k = i < n_cand && c_keep[i];
            const bool d = i < n_cand && !c_keep[i];
            const uint32_t kb = __ballot_sync(0xffffffffu, k), db = __ballot_sync(0xffffffffu, d);
            const uint32_t lt = (1u << lane) - 1u;
            if (k) {
                const int pos = run + __popc(kb & lt);
                np_slot[pos] = c_slot[i];
                np_id[pos] = c_id[i];
                np_score[pos] = c_score[i];
            }
            if (d) freel[n_free + drop + __popc(db & lt)] = c_slot[i];
            run += __popc(kb);
            drop += __popc(db);
        }
        if (lane == 0) {
            s_new_np = run;
            s_ndrop = drop;
        }
    }
    __syncthreads();
    const int new_np = s_new_np;
    const int free_top = n_free + s_ndrop;  // free entries after the drops
    // 4. write back: P', L', stage', free', dense', keys'
    const int new_nl = evict ? n_l : n_l + bpc;
    const int l_shift = evict ? bpc : 0;
    const int64_t chunk_base = p.cur.chunk * static_cast<int64_t>(bpc);
    for (int i = tid; i < new_np; i += nt) {
        p.m.p_slot[uP + i] = np_slot[i];
        p.m.p_id[uP + i] = np_id[i];
        p.m.p_score[uP + i] = np_score[i];
        p.m.dense[static_cast<int64_t>(u) * (C + bpc) + i] = np_slot[i];
        p.m.keys[static_cast<int64_t>(u) * S + i] = np_slot[i];
    }
    for (int i = tid; i < new_nl; i += nt) {
        int32_t sl;
        int64_t id;
        if (i < n_l - l_shift) {
            sl = l_slot[i + l_shift];
            id = l_id[i + l_shift];
        } else {
            const int c = i - (n_l - l_shift);
            sl = stage[c];
            id = chunk_base + c;
        }
        p.m.l_slot[uL + i] = sl;
        p.m.l_id[uL + i] = id;
        p.m.keys[static_cast<int64_t>(u) * S + new_np + i] = sl;
    }
    // new stage slots: pop bpc from the top of the free stack
    for (int i = tid; i < bpc; i += nt) {
        const int sl = freel[free_top - 1 - i];
        p.m.stage[static_cast<int64_t>(u) * bpc + i] = sl;
        p.m.dense[static_cast<int64_t>(u) * (C + bpc) + new_np + i] = sl;
        p.m.keys[static_cast<int64_t>(u) * S + new_np + new_nl + i] = sl;
    }
    for (int i = tid; i < free_top - bpc; i += nt) p.m.free_slot[static_cast<int64_t>(u) * S + i] = freel[i];
}

}  // namespace

std::atomic<int> g_fault{0};

int launch_mem_init(const MemDev& m, int units, int C, int Lcap, int bpc, int S, cudaStream_t s) {
    count_launch();
    mem_init_kernel<<<units, 256, 0, s>>>(m, C, Lcap, bpc, S);
    return check_launch("mem_init_kernel");
}

int launch_mem_commit(const MemDev& m, const float* s_t, int units, int C, int Lcap, int bpc, int S,
                      const MemCounts& cur, const MemCounts& next, cudaStream_t s) {
    CommitParams p{m, s_t, C, Lcap, bpc, S, cur, next, g_fault.load()};
    const int max_cand = C + bpc;
    const size_t smem = static_cast<size_t>(max_cand) * (8 + 4 + 4 + 4) + static_cast<size_t>(Lcap) * 12 +
                        static_cast<size_t>(bpc) * 4 + static_cast<size_t>(S) * 4 + static_cast<size_t>(C) * 16 + 64;
    if (smem > 227 * 1024) return set_error(PBSA_EUNSUPPORTED, "mem_commit: memory geometry too large for one CTA");
    if (int rc = ensure_smem(reinterpret_cast<const void*>(mem_commit_kernel), smem, "mem_commit")) return rc;
    launch_pdl(mem_commit_kernel, dim3(units), dim3(256), smem, s, p);
    return check_launch("mem_commit_kernel");
}

}  // namespace pbsa
