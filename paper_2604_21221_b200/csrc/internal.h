// internal.h -- shared declarations of the PBSA B200 library (not part of the public ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include <atomic>

#include "../../include/pbsa_b200.h"
#include "../../include/pbsa_b200_debug.h"

namespace pbsa {

using bf16 = __nv_bfloat16;

int set_error(int code, const std::string& msg);
int check_launch(const char* what);
// Raise a kernel's dynamic shared-memory limit to `bytes` (cached per kernel); error if refused.
int ensure_smem(const void* kernel, size_t bytes, const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: every hot-path kernel is launched with programmatic stream
// serialization and executes pdl_wait() (griddepcontrol.wait) before it touches data produced
// upstream (measured effect at config 2: ~1 %, within run-to-run noise).  PBSA_PDL=0 disables it.
bool pdl_enabled();
// kernels launched by the library since it was loaded (pbsa_launch_count): every launch site goes
// through launch_pdl or bumps the counter itself
void count_launch();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Chunk latents in the reference's Latent4D layout (tensor.hpp:30-47: (t, h, w, d) row-major with
// d = heads * d_head), one per batch element: [batch][T][H][W][heads * d] bf16.
// Blocks follow blockify.cpp:7-65: block id (nt * N_h + nh) * N_w + nw, in-block token index
// (dt * B_h + dh) * B_w + dw; unit u = e * heads + h.
struct LatentGeom {
    int batch, T, H, W, heads, d, bt, bh, bw;
    __host__ __device__ int nt() const { return T / bt; }
    __host__ __device__ int nh() const { return H / bh; }
    __host__ __device__ int nw() const { return W / bw; }
    __host__ __device__ int nqb() const { return nt() * nh() * nw(); }
    __host__ __device__ int b() const { return bt * bh * bw; }
};
// 5-D tensor map over a chunk latent with a box of one block of one head ({box_d, bw, bh, bt, 1})
bool encode_latent_tmap(void* tmap, const void* base, const LatentGeom& g, int box_d, bool swizzle128,
                        std::string* err);

// K1
int launch_compress(const bf16* x, int64_t x_unit_stride, int64_t x_block_stride, const int32_t* map,
                    int n_blocks, int units, int b, int d, float* reps, int64_t reps_unit_stride,
                    cudaStream_t s);
// q / qrep nullable: with q, the same pass also compresses the current chunk's query blocks
int launch_write_chunk(const bf16* kc, const bf16* vc, const bf16* q, const int32_t* stage, int bpc, int b,
                       int d, int units, int n_slots, bf16* k_pool, bf16* v_pool, float* krep, float* qrep,
                       cudaStream_t s, int q_begin = 0, int q_count = -1);
// the same fused ingest reading the chunk's K/V/Q latents directly (blockify fused into the TMA box)
int launch_ingest_latent(const bf16* k_lat, const bf16* v_lat, const bf16* q_lat, const LatentGeom& g,
                         const int32_t* stage, int n_slots, bf16* k_pool, bf16* v_pool, float* krep, float* qrep,
                         cudaStream_t s);
// K2
size_t score_select_workspace(int units, int nqb, int n_keys);
int launch_score_select(const float* qc, const float* krep, int64_t krep_unit_stride,
                        const int32_t* key_slots, int key_stride, int n_keys, int local_off,
                        int n_local, int k, int nqb, int units, int d, float scale, int32_t* sel,
                        float* s_t, void* ws, size_t ws_bytes, cudaStream_t s, int* status = nullptr,
                        int qc_rows = 0, int qc_row0 = 0);  // qc [units][qc_rows (0: nqb)][d], rows from qc_row0
// aggregate_scores (Eq. 8): s[u][j] = float(sum_i double(a[u][i][j]) / rows), ascending i
int launch_aggregate_scores(const float* a, int rows, int cols, int units, float* s, cudaStream_t st);
// SPEC-op primitives on device f32 matrices (spec_ops.cu; the drop-in C++ API, not the hot path)
int launch_matmul_f64acc(const float* a, const float* b, int n, int kd, int m, int bt, float scale, float* c,
                         cudaStream_t s);
int launch_softmax_rows(const float* scores, const float* mask, int rows, int cols, float* out, int* status,
                        cudaStream_t s);
int launch_select_topk(const float* a, int rows, int cols, int k, int32_t* sel, uint32_t* keys, int* status,
                       cudaStream_t s);
int launch_blockify(const float* x, int t, int h, int w, int d, int bt, int bh, int bw, float* y, int inverse,
                    cudaStream_t s);
int launch_topc_keep(const int64_t* ids, const float* scores, int n, int slots, uint8_t* keep, int* status,
                     cudaStream_t s);
// Tile pairing (between K2 and K3): per unit, the nq query blocks of a call are paired into K3 tiles
// greedily by largest Top-K overlap (ties: lowest pair index) so that each tile's union list is
// short.  sel [units][sel_rows][k] (rows sel_row0 ..); pairs [units][(nq + 1) / 2][2] = query blocks
// (within the call) of each tile, the second -1 for an odd leftover.  Returns PBSA_EUNSUPPORTED when
// the bitsets do not fit shared memory (the caller then keeps the natural (2t, 2t + 1) pairing).
int launch_pair_tiles(const int32_t* sel, int sel_rows, int sel_row0, int nq, int k, int n_local, int units,
                      int32_t* pairs, cudaStream_t s);
// K3
// lat != null: q and o are chunk latents (Q blocks gathered by a 5-D TMA box, O rows scattered back
// to their latent positions in the epilogue -- unblockify fused); lse stays [units][n_q] block-major
int launch_bsa_fwd(const bf16* q, const bf16* k_pool, const bf16* v_pool, int n_slots,
                   const int32_t* dense, int dense_stride, int n_dense, const int32_t* local,
                   int local_stride, int n_local, const int32_t* sel, int k, int nqb, int b, int d,
                   int units, float scale, bf16* o, float* lse, void* ws, size_t ws_bytes, cudaStream_t s,
                   const LatentGeom* lat = nullptr, int sel_rows = 0, int sel_row0 = 0,
                   const int32_t* tile_pairs = nullptr);  // null: tiles are query blocks (2t, 2t + 1)
size_t bsa_fwd_workspace(int units, int nqb, int d);
pbsa_bsa_plan& last_bsa_plan();  // the calling thread's last K3 launch plan
// injected fault (pbsa_debug_set_fault; negative controls only)
constexpr int kFaultDropSink = 1;
extern std::atomic<int> g_fault;
// K3 backward: dq [units][n_q][d], dk / dv [units][n_slots][64][d] f32 (rows of visible slots written)
size_t bsa_bwd_workspace(int units, int nqb, int b, int n_local);
int launch_bsa_bwd(const bf16* q, const bf16* k_pool, const bf16* v_pool, int n_slots, const int32_t* dense,
                   int dense_stride, int n_dense, const int32_t* local, int local_stride, int n_local,
                   const int32_t* sel, int k, int nqb, int b, int d, int units, float scale, const bf16* o,
                   const bf16* d_o, const float* lse, float* dq, float* dk, float* dv, void* ws, size_t ws_bytes,
                   cudaStream_t s);
int launch_debug_tile(const bf16* q, const bf16* k, const bf16* v, int d, float* s_out,
                      float* o_out, cudaStream_t s);
// K4
struct MemDev {
    int32_t* p_slot;   // [U][C]
    int64_t* p_id;     // [U][C]
    float* p_score;    // [U][C]
    int32_t* l_slot;   // [U][Lcap]
    int64_t* l_id;     // [U][Lcap]
    int32_t* stage;    // [U][bpc]
    int32_t* free_slot;  // [U][S]
    int32_t* dense;    // [U][C+bpc]
    int32_t* keys;     // [U][S]
    int* status;       // device status word: bit 0 NaN logits (K2), bit 1 NaN scores (K4)
};
struct MemCounts {
    int n_p, n_sinks, n_l, n_free;
    int64_t chunk;  // index of the chunk held in the stage slots
};
int launch_mem_init(const MemDev& m, int units, int C, int Lcap, int bpc, int S, cudaStream_t s);
int launch_mem_commit(const MemDev& m, const float* s_t, int units, int C, int Lcap, int bpc, int S,
                      const MemCounts& cur, const MemCounts& next, cudaStream_t s);

// TMA descriptor encoding through the driver entry point (no -lcuda link dependency)
bool encode_tmap_bf16(void* tmap, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                      const uint32_t* box, std::string* err);

}  // namespace pbsa
