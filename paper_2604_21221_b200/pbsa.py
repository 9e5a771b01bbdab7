"""Host-side mirror of the reference's PBSA operator API over the C ABI.

Names, argument meaning and error behaviour follow /root/reference/SPEC.md (modules router,
attention, memory) so callers and tests read like the reference's.  Tensors live on the GPU
(torch is only the device-memory / stream plumbing); every op launches the sm_100a kernels of
libpbsa_b200.so on the current torch stream.  Invalid arguments raise PbsaError (a ValueError,
the analogue of the reference's std::invalid_argument), CUDA failures PbsaCudaError.

    compress_blocks     SPEC.md:268  router.compress_blocks          -> K1
    score_select        SPEC.md:277-303  coarse_attention + select_topk (+ aggregate_scores) -> K2
    attention_sparse    SPEC.md:367  attention.attention_sparse       -> K3
    Memory              SPEC.md:160-243  PersistentMemory + LocalWindow, push_chunk,
                        update_persistent, assemble_kv                 -> K4 (+ fused KV write)
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import _capi
from ._capi import LIB, PbsaCudaError, PbsaError, check  # noqa: F401

__all__ = ["compress_blocks", "score_select", "attention_sparse", "Memory", "attention_scale",
           "topk_count", "bsa_fwd_last_plan", "PbsaError", "PbsaCudaError", "debug_tile", "MODE_DENOISE",
           "MODE_CACHE_UPDATE"]

MODE_DENOISE = _capi.MODE_DENOISE
MODE_CACHE_UPDATE = _capi.MODE_CACHE_UPDATE


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype, name: str) -> None:
    if not t.is_cuda:
        raise PbsaError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise PbsaError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise PbsaError(f"{name} must be contiguous")


def _out(out: torch.Tensor | None, like: torch.Tensor, name: str = "out") -> torch.Tensor:
    """A caller-supplied output must match the input it stands for exactly (the kernels write it
    unchecked)."""
    if out is None:
        return torch.empty_like(like)
    if out.device != like.device or out.dtype != like.dtype or out.shape != like.shape or not out.is_contiguous():
        raise PbsaError(f"{name} must be a contiguous {like.dtype} tensor of shape {tuple(like.shape)} on {like.device}")
    return out


def attention_scale(d: int) -> float:
    """AttentionConfig.scale = d^-1/2, rounded to fp32 like the oracle."""
    return float(torch.tensor(1.0 / math.sqrt(d), dtype=torch.float32))


def topk_count(n_local: int, topk_ratio: float) -> int:
    """k = max(1, ceil(N_l^blk * ratio)); empty local region is an error."""
    if n_local < 1:
        raise PbsaError("select_topk: empty local region")
    if not (0.0 < topk_ratio <= 1.0):
        raise PbsaError("select_topk: topk_ratio must be in (0,1]")
    return min(n_local, max(1, math.ceil(n_local * topk_ratio)))


def compress_blocks(x: torch.Tensor, block_map: torch.Tensor | None = None,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """Mean-pool each block.  x: [units, n_blocks, b, d] bf16 (or a slot pool
    [units, n_slots, 64, d] with block_map [units, n_blocks] selecting slots and b given by the
    pool rows actually holding tokens -- see Memory).  Returns [units, n_blocks, d] f32 (or
    writes `out` at the mapped rows)."""
    _need(x, torch.bfloat16, "x")
    units, nb, b, d = x.shape
    if block_map is None:
        if out is None:
            out = torch.empty(units, nb, d, device=x.device, dtype=torch.float32)
        check(LIB.pbsa_compress(x.data_ptr(), nb * b * d, b * d, None, nb, units, b, d,
                                out.data_ptr(), out.shape[1] * d, _stream()))
        return out
    raise PbsaError("compress_blocks: use Memory for slot-mapped compression")


def score_select(qc: torch.Tensor, krep: torch.Tensor, key_slots: torch.Tensor, local_off: int,
                 n_local: int, k: int, scale: float | None = None, n_keys: int | None = None,
                 want_scores: bool = False):
    """Coarse attention + row-wise Top-K (+ Eq. 8 scores).

    qc [units, nqb, d] f32; krep [units, n_slots, d] f32 (block representative per slot);
    key_slots [units, key_stride] int32 -- the first n_keys entries are the key blocks, of which
    [local_off, local_off+n_local) form the local window.  Returns sel [units, nqb, k] int32
    (local indices, ascending) and, if want_scores, s_t [units, n_keys] f32."""
    _need(qc, torch.float32, "qc")
    _need(krep, torch.float32, "krep")
    _need(key_slots, torch.int32, "key_slots")
    units, nqb, d = qc.shape
    n_keys = key_slots.shape[1] if n_keys is None else n_keys
    scale = attention_scale(d) if scale is None else scale
    sel = torch.empty(units, nqb, max(k, 1), device=qc.device, dtype=torch.int32)
    s_t = torch.empty(units, n_keys, device=qc.device, dtype=torch.float32) if want_scores else None
    ws_bytes = LIB.pbsa_score_select_workspace(units, nqb, n_keys)
    ws = torch.empty(ws_bytes, device=qc.device, dtype=torch.uint8)
    check(LIB.pbsa_score_select(qc.data_ptr(), krep.data_ptr(), krep.shape[1] * d,
                                key_slots.data_ptr(), key_slots.shape[1], n_keys, local_off, n_local,
                                k, nqb, units, d, scale, sel.data_ptr(), _ptr(s_t), ws.data_ptr(),
                                ws_bytes, _stream()))
    sel = sel[:, :, :k]
    return (sel, s_t) if want_scores else sel


def attention_sparse(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor,
                     dense_slots: torch.Tensor | None, local_slots: torch.Tensor | None,
                     sel: torch.Tensor | None, b: int, scale: float | None = None,
                     n_dense: int | None = None, n_local: int | None = None,
                     want_lse: bool = False, stream_k: bool = True, validate: bool = True):
    """Block-sparse attention forward.

    q [units, nqb*b, d] bf16 (query tokens block-major); k_pool / v_pool [units, n_slots, 64, d]
    bf16 with rows >= b zero; dense_slots [units, >=n_dense] int32 (persistent + current chunk,
    visible to every query block); local_slots [units, >=n_local] int32; sel [units, nqb, k]
    int32 ascending local indices.  Returns o [units, nqb*b, d] bf16 (and lse [units, nqb*b]).
    validate: check every slot / selection index is in range first (one host sync)."""
    _need(q, torch.bfloat16, "q")
    _need(k_pool, torch.bfloat16, "k_pool")
    _need(v_pool, torch.bfloat16, "v_pool")
    units, nq, d = q.shape
    if nq % b:
        raise PbsaError(f"attention_sparse: n_q ({nq}) not divisible by b ({b})")
    nqb = nq // b
    n_slots = k_pool.shape[1]
    if k_pool.shape != (units, n_slots, 64, d) or v_pool.shape != k_pool.shape:
        raise PbsaError("attention_sparse: pools must be [units, n_slots, 64, d]")
    nd = 0 if dense_slots is None else (dense_slots.shape[1] if n_dense is None else n_dense)
    nl = 0 if local_slots is None else (local_slots.shape[1] if n_local is None else n_local)
    k = 0 if sel is None else sel.shape[2]
    for name, t in (("dense_slots", dense_slots), ("local_slots", local_slots), ("sel", sel)):
        if t is not None:
            _need(t, torch.int32, name)
    if sel is not None and (sel.dim() != 3 or sel.shape[:2] != (units, nqb)):
        raise PbsaError(f"attention_sparse: sel must be [units, nqb, k] = [{units}, {nqb}, k]")
    for name, t, n in (("dense_slots", dense_slots, nd), ("local_slots", local_slots, nl)):
        if t is not None and (t.dim() != 2 or t.shape[0] != units or t.shape[1] < n):
            raise PbsaError(f"attention_sparse: {name} must be [units, >= {n}]")
    if validate:  # one host sync: every index in range (the kernel reads them unchecked)
        bad = []
        if dense_slots is not None and nd and ((dense_slots[:, :nd] < 0) | (dense_slots[:, :nd] >= n_slots)).any():
            bad.append("dense_slots out of [0, n_slots)")
        if local_slots is not None and nl and ((local_slots[:, :nl] < 0) | (local_slots[:, :nl] >= n_slots)).any():
            bad.append("local_slots out of [0, n_slots)")
        if sel is not None and k and ((sel < 0) | (sel >= nl)).any():
            bad.append("sel out of [0, n_local)")
        if bad:
            raise PbsaError("attention_sparse: " + "; ".join(bad))
    o = torch.empty_like(q)
    lse = torch.empty(units, nq, device=q.device, dtype=torch.float32) if want_lse else None
    scale = attention_scale(d) if scale is None else scale
    ws_bytes = LIB.pbsa_bsa_fwd_workspace(units, nqb, d) if stream_k else 0
    ws = _workspace(ws_bytes, q.device) if stream_k else None
    check(LIB.pbsa_bsa_fwd(q.data_ptr(), k_pool.data_ptr(), v_pool.data_ptr(), n_slots,
                           _ptr(dense_slots), 0 if dense_slots is None else dense_slots.shape[1], nd,
                           _ptr(local_slots), 0 if local_slots is None else local_slots.shape[1], nl,
                           _ptr(sel), k, nqb, b, d, units, scale, o.data_ptr(), _ptr(lse),
                           _ptr(ws), ws_bytes, _stream()))
    return (o, lse) if want_lse else o


def pair_tiles(sel: torch.Tensor, n_local: int) -> torch.Tensor:
    """K3 tile pairing (pbsa_pair_tiles): sel [units, nq, k] int32 local indices -> [units, (nq+1)//2, 2]
    int32 query blocks per tile (second -1 for a single), paired greedily by Top-K overlap."""
    _need(sel, torch.int32, "sel")
    units, nq, k = sel.shape
    out = torch.empty(units, (nq + 1) // 2, 2, device=sel.device, dtype=torch.int32)
    check(LIB.pbsa_pair_tiles(sel.data_ptr(), nq, 0, nq, k, n_local, units, out.data_ptr(), _stream()))
    return out


# ---- the reference's tensor / blockify primitives and the SPEC router / memory ops on device f32
# tensors (bit-exact with the reference's CPU code; the fused hot path never uses them) ------------
def _f32(t: torch.Tensor, name: str) -> None:
    _need(t, torch.float32, name)


def _status_check(st: torch.Tensor, msgs: dict) -> None:
    flags = int(st.item())
    for bit, msg in msgs.items():
        if flags & bit:
            raise PbsaError(msg)


def matmul(a: torch.Tensor, b: torch.Tensor, transpose_b: bool = False, scale: float = 1.0) -> torch.Tensor:
    """matmul (tensor.cpp:8-32) / matmul_nt (transpose_b, tensor.cpp:34-55): fp64 accumulation in
    ascending k, one fp32 rounding, then an fp32 multiply by `scale`."""
    _f32(a, "a")
    _f32(b, "b")
    n, kd = a.shape
    m = b.shape[0] if transpose_b else b.shape[1]
    if (b.shape[1] if transpose_b else b.shape[0]) != kd:
        op = "matmul_nt: a.cols" if transpose_b else "matmul: a.cols"
        raise PbsaError(f"{op} ({kd}) != b.{'cols' if transpose_b else 'rows'} ({b.shape[1] if transpose_b else b.shape[0]})")
    c = torch.empty(n, m, device=a.device, dtype=torch.float32)
    check(LIB.pbsa_matmul(a.data_ptr(), b.data_ptr(), n, kd, m, int(transpose_b), float(scale), c.data_ptr(), _stream()))
    return c


def masked_softmax_rows(scores: torch.Tensor, mask: torch.Tensor | None = None) -> torch.Tensor:
    """masked_softmax_rows (tensor.cpp:57-108); raises PbsaError on NaN scores / non 0/-inf mask."""
    _f32(scores, "scores")
    if mask is not None:
        _f32(mask, "mask")
        if mask.shape != scores.shape:
            raise PbsaError("masked_softmax_rows: mask shape mismatch")
    out = torch.empty_like(scores)
    st = torch.zeros(1, dtype=torch.int32, device=scores.device)
    check(LIB.pbsa_masked_softmax_rows(scores.data_ptr(), _ptr(mask), scores.shape[0], scores.shape[1],
                                       out.data_ptr(), st.data_ptr(), _stream()))
    _status_check(st, {1: "masked_softmax_rows: NaN in scores",
                       2: "masked_softmax_rows: mask entries must be 0 or -inf"})
    return out


def aggregate_scores(a: torch.Tensor) -> torch.Tensor:
    """aggregate_scores: ascending-row fp64 column means."""
    _f32(a, "a")
    s = torch.empty(a.shape[1], device=a.device, dtype=torch.float32)
    check(LIB.pbsa_aggregate_scores(a.data_ptr(), a.shape[0], a.shape[1], s.data_ptr(), _stream()))
    return s


def select_topk(a_local: torch.Tensor, k: int) -> torch.Tensor:
    """select_topk with absolute k: [rows, k] int32 ascending indices of the k largest
    entries per row, ties toward the lower index (use topk_count(n, ratio) for a ratio)."""
    _f32(a_local, "a_local")
    rows, cols = a_local.shape
    sel = torch.empty(rows, max(k, 1), device=a_local.device, dtype=torch.int32)
    ws_bytes = LIB.pbsa_select_topk_workspace(rows, cols)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=a_local.device)
    st = torch.zeros(1, dtype=torch.int32, device=a_local.device)
    check(LIB.pbsa_select_topk(a_local.data_ptr(), rows, cols, int(k), sel.data_ptr(), ws.data_ptr(), ws_bytes,
                               st.data_ptr(), _stream()))
    _status_check(st, {1: "select_topk: NaN in scores"})
    return sel[:, :k]


def blockify(x: torch.Tensor, shape) -> torch.Tensor:
    """blockify (blockify.cpp:38-65): (t, h, w, d) f32 -> block-major (n_b, b, d)."""
    _f32(x, "x")
    t, h, w, d = x.shape
    bt, bh, bw = (int(v) for v in shape)
    y = torch.empty((t * h * w) // max(bt * bh * bw, 1) if bt * bh * bw else 0, bt * bh * bw, d,
                    device=x.device, dtype=torch.float32)
    check(LIB.pbsa_blockify(x.data_ptr(), t, h, w, d, bt, bh, bw, y.data_ptr(), 0, _stream()))
    return y


def unblockify(xb: torch.Tensor, dims, shape) -> torch.Tensor:
    """unblockify (blockify.cpp:67-96): block-major (n_b, b, d) -> (t, h, w, d)."""
    _f32(xb, "xb")
    t, h, w, d = (int(v) for v in dims)
    bt, bh, bw = (int(v) for v in shape)
    if xb.numel() != t * h * w * d:
        raise PbsaError("blocked data length does not match layout")
    y = torch.empty(t, h, w, d, device=xb.device, dtype=torch.float32)
    check(LIB.pbsa_blockify(xb.data_ptr(), t, h, w, d, bt, bh, bw, y.data_ptr(), 1, _stream()))
    return y


def topc_select(ids: torch.Tensor, scores: torch.Tensor, slots: int) -> torch.Tensor:
    """update_persistent's ranking: bool mask of the `slots` best candidates by
    (score desc, id asc)."""
    _need(ids, torch.int64, "ids")
    _f32(scores, "scores")
    keep = torch.empty(ids.shape[0], dtype=torch.uint8, device=ids.device)
    check(LIB.pbsa_topc_select(ids.data_ptr(), scores.data_ptr(), ids.shape[0], int(slots), keep.data_ptr(), None,
                               _stream()))
    return keep.bool()


def bsa_fwd_last_plan() -> "_capi.BsaPlan":
    """How this thread's last K3 launch was planned (list entry width, CTAs per SM, grid, schedule
    0 whole tiles / 1 hybrid stream-K / 2 unit gangs) -- pbsa_bsa_fwd_last_plan."""
    plan = _capi.BsaPlan()
    check(LIB.pbsa_bsa_fwd_last_plan(C.byref(plan)))
    return plan


_WS: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    """Zero-initialised K3 workspace, cached per (device, stream): the stream-K merge counters and
    partial slots in it are only safe for launches ordered on one stream, and a replaced (smaller)
    buffer goes back to the caching allocator in that stream's order (the kernel leaves it zeroed)."""
    key = (str(device), torch.cuda.current_stream(device).cuda_stream)
    t = _WS.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS[key] = t
    return t


def attention_sparse_backward(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor,
                              dense_slots: torch.Tensor | None, local_slots: torch.Tensor | None,
                              sel: torch.Tensor | None, b: int, o: torch.Tensor, lse: torch.Tensor,
                              d_o: torch.Tensor, scale: float | None = None):
    """Gradient of attention_sparse (pbsa_bsa_bwd): returns (dq [units, n_q, d], dk_pool, dv_pool
    [units, n_slots, 64, d]) in float32.  o / lse are the forward's outputs (want_lse=True)."""
    for name, t in (("q", q), ("k_pool", k_pool), ("v_pool", v_pool), ("o", o), ("d_o", d_o)):
        _need(t, torch.bfloat16, name)
    _need(lse, torch.float32, "lse")
    units, nq, d = q.shape
    if nq % b:
        raise PbsaError(f"attention_sparse_backward: n_q ({nq}) not divisible by b ({b})")
    nqb, n_slots = nq // b, k_pool.shape[1]
    nd = 0 if dense_slots is None else dense_slots.shape[1]
    nl = 0 if local_slots is None else local_slots.shape[1]
    k = 0 if sel is None else sel.shape[2]
    for name, t in (("dense_slots", dense_slots), ("local_slots", local_slots), ("sel", sel)):
        if t is not None:
            _need(t, torch.int32, name)
    dq = torch.empty(units, nq, d, device=q.device, dtype=torch.float32)
    dk = torch.zeros(units, n_slots, 64, d, device=q.device, dtype=torch.float32)
    dv = torch.zeros_like(dk)
    ws = torch.empty(max(1, LIB.pbsa_bsa_bwd_workspace(units, nqb, b, nl)), dtype=torch.uint8, device=q.device)
    scale = attention_scale(d) if scale is None else scale
    check(LIB.pbsa_bsa_bwd(q.data_ptr(), k_pool.data_ptr(), v_pool.data_ptr(), n_slots, _ptr(dense_slots),
                           nd if dense_slots is None else dense_slots.stride(0), nd, _ptr(local_slots),
                           nl if local_slots is None else local_slots.stride(0), nl, _ptr(sel), k, nqb, b, d,
                           units, float(scale), o.data_ptr(), d_o.data_ptr(), lse.data_ptr(), dq.data_ptr(),
                           dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(), _stream()))
    return dq, dk, dv


def debug_set_fault(name: str | None) -> None:
    """Test-only fault injection (pbsa_debug_set_fault): "drop-sink" breaks K4's sink retention
    (the negative control of SPEC.md:625); None clears it."""
    check(LIB.pbsa_debug_set_fault(None if not name else name.encode()))


def debug_tile(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor):
    """One 128x64 tile through the tcgen05 path: returns (q k^T f32, bf16(q k^T) v f32)."""
    d = q.shape[1]
    s = torch.empty(128, 64, device=q.device, dtype=torch.float32)
    o = torch.empty(128, d, device=q.device, dtype=torch.float32)
    check(LIB.pbsa_debug_tile(q.data_ptr(), k.data_ptr(), v.data_ptr(), d, s.data_ptr(), o.data_ptr(),
                              _stream()))
    return s, o


# ---- PBT1 tensor files (reference tensor.hpp:62-101, tensor_io.cpp) -------------------------
class TensorIoError(PbsaError):
    """PBT1 format / IO error; .kind is the reference's TensorIoError::Kind name."""

    KINDS = ("OpenFailed", "BadMagic", "BadDtype", "Truncated", "TrailingData", "BadShape")

    def __init__(self, msg: str):
        super().__init__(msg)
        self.kind = msg.split(":", 1)[0] if msg.split(":", 1)[0] in self.KINDS else None


def _pbt1(rc: int) -> None:
    if rc == _capi.PBSA_EINVAL:
        raise TensorIoError(LIB.pbsa_last_error().decode())
    check(rc)


def write_tensor(path: str, x) -> None:
    """write_tensor (tensor_io.cpp:46-54): any-rank float32 array -> PBT1 file."""
    import numpy as np
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    dims = (C.c_uint64 * max(a.ndim, 1))(*a.shape)
    _pbt1(LIB.pbsa_pbt1_write(str(path).encode(), a.ctypes.data if a.size else None, a.ndim, dims))


def tensor_dims(path: str) -> tuple[int, ...]:
    r = C.c_int()
    dims = (C.c_uint64 * 16)()
    _pbt1(LIB.pbsa_pbt1_info(str(path).encode(), C.byref(r), dims, 16))
    return tuple(int(dims[i]) for i in range(r.value))


def read_tensor(path: str):
    """read_tensor (tensor_io.cpp:56-108): PBT1 file -> float32 array of the file's dims."""
    import numpy as np
    dims = tensor_dims(path)
    n = 0 if not dims else int(np.prod(dims, dtype=np.uint64))
    a = np.empty(n, np.float32)
    _pbt1(LIB.pbsa_pbt1_read(str(path).encode(), a.ctypes.data if n else None, n))
    return a.reshape(dims) if dims else a


def load_bf16(path: str, device=None) -> torch.Tensor:
    """A PBT1 file straight into device memory as bf16 (pinned staging, async copies, on-device
    conversion), e.g. a chunk latent for Memory.attend_latent."""
    dims = tensor_dims(path)
    out = torch.empty(dims, dtype=torch.bfloat16, device=device or "cuda")
    _pbt1(LIB.pbsa_pbt1_load_bf16(str(path).encode(), out.data_ptr() if out.numel() else None,
                                  out.numel(), _stream()))
    return out


def latent_geom(shape, heads: int, head_dim: int, block_shape) -> "_capi.LatentGeom":
    """pbsa_latent_geom of a chunk latent of `shape` ([batch,] T, H, W, heads*head_dim), validated by
    pbsa_latent_blocks (make_block_layout's divisibility rules, blockify.cpp:7-36)."""
    shape = tuple(int(x) for x in shape)
    if len(shape) == 4:
        shape = (1,) + shape
    if len(shape) != 5:
        raise PbsaError("latent: expected [batch,] T, H, W, heads*head_dim")
    batch, t, h, w, cd = shape
    if heads <= 0 or cd != heads * head_dim:
        raise PbsaError(f"latent: last dim {cd} != heads ({heads}) * head_dim ({head_dim})")
    bt, bh, bw = (int(x) for x in block_shape)
    g = _capi.LatentGeom(batch, t, h, w, heads, head_dim, bt, bh, bw)
    nqb, b = C.c_int(), C.c_int()
    check(LIB.pbsa_latent_blocks(C.byref(g), C.byref(nqb), C.byref(b)))
    return g


def latent_blocks(shape, heads: int, head_dim: int, block_shape) -> tuple[int, int]:
    """(blocks per chunk, tokens per block) of a chunk latent (host only)."""
    g = latent_geom(shape, heads, head_dim, block_shape)
    nqb, b = C.c_int(), C.c_int()
    check(LIB.pbsa_latent_blocks(C.byref(g), C.byref(nqb), C.byref(b)))
    return nqb.value, b.value


class Memory:
    """Device-resident PBSA memory for `units` heads: PersistentMemory (capacity C blocks, sinks =
    first chunk) + LocalWindow (window_chunks chunks) + the K/V slot pool."""

    def __init__(self, units: int, capacity_c: int, window_chunks: int, blocks_per_chunk: int,
                 b: int, d: int):
        h = C.c_void_p()
        check(LIB.pbsa_mem_create(C.byref(h), units, capacity_c, window_chunks, blocks_per_chunk,
                                  b, d))
        self._h = h
        self._host_refs = []  # host tensors of attend_qkv_host calls not yet waited for
        self.units, self.capacity_c, self.window_chunks = units, capacity_c, window_chunks
        self.blocks_per_chunk, self.b, self.d = blocks_per_chunk, b, d

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            if self._host_refs:
                LIB.pbsa_mem_host_sync(self._h)
                self._host_refs.clear()
            LIB.pbsa_mem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state ---------------------------------------------------------------------------
    def info(self) -> _capi.MemInfo:
        inf = _capi.MemInfo()
        check(LIB.pbsa_mem_get_info(self._h, C.byref(inf)))
        return inf

    def reset(self) -> None:
        check(LIB.pbsa_mem_reset(self._h, _stream()))

    def _view(self, ptr: int, shape, dtype) -> torch.Tensor:
        """Copy a device array of the state into a fresh tensor (for inspection / tests)."""
        n = 1
        for s in shape:
            n *= s
        esz = torch.empty(0, dtype=dtype).element_size()
        out = torch.empty(shape, dtype=dtype, device="cuda")
        if n:
            check(LIB.pbsa_copy(out.data_ptr(), ptr, n * esz, _stream()))
        return out

    def assemble(self):
        """assemble_kv as ids: (persistent ids [units, n_p] in order sinks id asc,
        dynamic id asc; local ids [units, n_l] oldest -> newest)."""
        inf = self.info()
        p = self._view(inf.p_ids, (self.units, self.capacity_c), torch.int64)[:, :inf.n_p]
        l_ = self._view(inf.l_ids, (self.units, inf.local_stride), torch.int64)[:, :inf.n_l]
        return p, l_

    def slot_tables(self):
        inf = self.info()
        dense = self._view(inf.dense_slots, (self.units, inf.dense_stride), torch.int32)
        local = self._view(inf.local_slots, (self.units, inf.local_stride), torch.int32)
        keys = self._view(inf.key_slots, (self.units, inf.key_stride), torch.int32)
        stage = self._view(inf.stage_slots, (self.units, self.blocks_per_chunk), torch.int32)
        return dense, local, keys, stage

    def pools(self):
        inf = self.info()
        shp = (self.units, inf.n_slots, 64, self.d)
        k = self._view(inf.k_pool, shp, torch.bfloat16)
        v = self._view(inf.v_pool, shp, torch.bfloat16)
        kr = self._view(inf.krep, (self.units, inf.n_slots, self.d), torch.float32)
        return k, v, kr

    # ---- hot path ------------------------------------------------------------------------
    def write_chunk(self, k_chunk: torch.Tensor, v_chunk: torch.Tensor) -> None:
        """The current chunk's K/V ([units, blocks_per_chunk*b, d] bf16) into the stage slots (+K1)."""
        for name, t in (("k_chunk", k_chunk), ("v_chunk", v_chunk)):
            _need(t, torch.bfloat16, name)
            if t.shape != (self.units, self.blocks_per_chunk * self.b, self.d):
                raise PbsaError(f"{name}: expected shape {(self.units, self.blocks_per_chunk * self.b, self.d)}")
        check(LIB.pbsa_mem_write_chunk(self._h, k_chunk.data_ptr(), v_chunk.data_ptr(), _stream()))

    def attend(self, q: torch.Tensor, k_top: int, mode: int = MODE_DENOISE, scale: float | None = None,
               out: torch.Tensor | None = None, want_lse: bool = False):
        """One PBSA call (Alg. 1 "Apply PBSA with Top-K"); mode MODE_CACHE_UPDATE = the k=0 pass
        that also scores all key blocks and updates P / L."""
        _need(q, torch.bfloat16, "q")
        if q.shape != (self.units, self.blocks_per_chunk * self.b, self.d):
            raise PbsaError("attend: q must be [units, blocks_per_chunk*b, d]")
        o = _out(out, q)
        lse = torch.empty(q.shape[:2], device=q.device, dtype=torch.float32) if want_lse else None
        check(LIB.pbsa_attend(self._h, q.data_ptr(), int(k_top), 0.0 if scale is None else float(scale),
                              int(mode), o.data_ptr(), _ptr(lse), _stream()))
        return (o, lse) if want_lse else o

    def attend_qkv(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, k_top: int,
                   mode: int = MODE_DENOISE, scale: float | None = None, out: torch.Tensor | None = None,
                   want_lse: bool = False):
        """write_chunk(k, v) + attend(q) fused: one ingest pass over Q, K and V (pbsa_attend_qkv)."""
        shape = (self.units, self.blocks_per_chunk * self.b, self.d)
        for name, t in (("q", q), ("k", k), ("v", v)):
            _need(t, torch.bfloat16, name)
            if t.shape != shape:
                raise PbsaError(f"attend_qkv: {name} must be {shape}")
        o = _out(out, q)
        lse = torch.empty(q.shape[:2], device=q.device, dtype=torch.float32) if want_lse else None
        check(LIB.pbsa_attend_qkv(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), int(k_top),
                                  0.0 if scale is None else float(scale), int(mode), o.data_ptr(),
                                  _ptr(lse), _stream()))
        return (o, lse) if want_lse else o

    def attend_qkv_host(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, k_top: int,
                        mode: int = MODE_DENOISE, out: torch.Tensor | None = None,
                        scale: float | None = None) -> torch.Tensor:
        """attend_qkv on HOST chunks (pbsa_attend_qkv_host): q / k / v pinned CPU bf16 tensors of the
        chunk shape; O lands in `out` (pinned CPU).  Uploads, compute and downloads are pipelined
        across calls (the upload of call i+1 overlaps the compute of call i); inputs must stay
        unchanged and `out` unread until host_sync()."""
        shape = (self.units, self.blocks_per_chunk * self.b, self.d)
        for name, t in (("q", q), ("k", k), ("v", v)):
            if t.device.type != "cpu" or t.dtype != torch.bfloat16 or not t.is_contiguous() or t.shape != shape:
                raise PbsaError(f"attend_qkv_host: {name} must be a contiguous CPU bf16 tensor of shape {shape}")
        # (pageable memory works too, but its copies cannot overlap the compute: pin for the pipeline)
        o = torch.empty(shape, dtype=torch.bfloat16).pin_memory() if out is None else out
        if o.device.type != "cpu" or not o.is_contiguous() or o.shape != shape or o.dtype != torch.bfloat16:
            raise PbsaError(f"attend_qkv_host: out must be a contiguous CPU bf16 tensor of shape {shape}")
        check(LIB.pbsa_attend_qkv_host(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), int(k_top),
                                       0.0 if scale is None else float(scale), int(mode), o.data_ptr(),
                                       _stream()))
        # the library's copies read q/k/v and write o asynchronously: keep the host blocks alive (and
        # out of torch's pinned-memory cache) until host_sync() has waited for them
        self._host_refs.append((q, k, v, o))
        return o

    def attend_part_ingest(self, q_part: torch.Tensor, q_begin: int, k: torch.Tensor, v: torch.Tensor,
                           qc_full: torch.Tensor) -> None:
        """Query-split call, step 1 (pbsa_attend_part_ingest): the whole chunk's K/V into the memory
        (replicated across the ranks sharing these heads) and this rank's query blocks
        [q_begin, q_begin + q_count) compressed into their rows of qc_full [units, bpc, d] f32."""
        self._part_check(q_part, q_begin, qc_full)
        shape = (self.units, self.blocks_per_chunk * self.b, self.d)
        for name, t in (("k", k), ("v", v)):
            _need(t, torch.bfloat16, name)
            if t.shape != shape:
                raise PbsaError(f"attend_part_ingest: {name} must be the whole chunk {shape}")
        check(LIB.pbsa_attend_part_ingest(self._h, q_part.data_ptr(), int(q_begin), q_part.shape[1] // self.b,
                                          k.data_ptr(), v.data_ptr(), qc_full.data_ptr(), _stream()))

    def attend_part(self, q_part: torch.Tensor, q_begin: int, qc_full: torch.Tensor, k_top: int,
                    mode: int = MODE_DENOISE, scale: float | None = None, out: torch.Tensor | None = None,
                    want_lse: bool = False):
        """Query-split call, step 2 (pbsa_attend_part): K2 / K3 (/ K4) for this rank's query blocks.
        In MODE_CACHE_UPDATE every row of qc_full must hold the gathered representatives."""
        self._part_check(q_part, q_begin, qc_full)
        o = _out(out, q_part)
        lse = torch.empty(q_part.shape[:2], device=q_part.device, dtype=torch.float32) if want_lse else None
        check(LIB.pbsa_attend_part(self._h, q_part.data_ptr(), int(q_begin), q_part.shape[1] // self.b,
                                   qc_full.data_ptr(), int(k_top), 0.0 if scale is None else float(scale), int(mode),
                                   o.data_ptr(), _ptr(lse), _stream()))
        return (o, lse) if want_lse else o

    def _part_check(self, q_part, q_begin, qc_full):
        _need(q_part, torch.bfloat16, "q_part")
        _need(qc_full, torch.float32, "qc_full")
        if q_part.dim() != 3 or q_part.shape[0] != self.units or q_part.shape[2] != self.d or q_part.shape[1] % self.b:
            raise PbsaError("attend_part: q_part must be [units, q_count*b, d]")
        if qc_full.shape != (self.units, self.blocks_per_chunk, self.d):
            raise PbsaError(f"attend_part: qc_full must be {(self.units, self.blocks_per_chunk, self.d)}")
        if q_begin < 0 or q_begin + q_part.shape[1] // self.b > self.blocks_per_chunk:
            raise PbsaError("attend_part: query range outside the chunk")

    def host_sync(self) -> None:
        """Wait for every upload / download issued by attend_qkv_host."""
        check(LIB.pbsa_mem_host_sync(self._h))
        self._host_refs.clear()

    def attend_latent(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, block_shape, k_top: int,
                      mode: int = MODE_DENOISE, scale: float | None = None, out: torch.Tensor | None = None,
                      want_lse: bool = False):
        """attend_qkv on chunk latents in the reference's Latent4D layout (tensor.hpp:30-47, d =
        heads * head_dim): q / k / v [batch, T, H, W, heads*d] (or [T, H, W, heads*d] for batch 1)
        bf16, blocked by block_shape = (B_t, B_h, B_w) as blockify.cpp does.  The blockify gather
        and the unblockify scatter of O run inside the kernels (5-D TMA boxes / epilogue stores);
        the result is bit-identical to attend_qkv on the blockified per-head tensors."""
        geom = latent_geom(q.shape, self.units // (1 if q.dim() == 4 else q.shape[0]), self.d, block_shape)
        for name, t in (("q", q), ("k", k), ("v", v)):
            _need(t, torch.bfloat16, name)
            if t.shape != q.shape:
                raise PbsaError(f"attend_latent: {name} must have q's shape {tuple(q.shape)}")
        o = _out(out, q)
        lse = torch.empty(self.units, self.blocks_per_chunk * self.b, device=q.device,
                          dtype=torch.float32) if want_lse else None
        check(LIB.pbsa_attend_latent(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), C.byref(geom),
                                     int(k_top), 0.0 if scale is None else float(scale), int(mode),
                                     o.data_ptr(), _ptr(lse), _stream()))
        return (o, lse) if want_lse else o

    def commit(self, s_t: torch.Tensor) -> None:
        _need(s_t, torch.float32, "s_t")
        check(LIB.pbsa_mem_commit(self._h, s_t.data_ptr(), _stream()))

    def profile(self, enable: bool = True, max_calls: int = 4096) -> None:
        """Per-stage CUDA-event timing of subsequent calls (see pbsa_mem_profile)."""
        check(LIB.pbsa_mem_profile(self._h, int(enable), int(max_calls)))

    def profile_read(self) -> dict:
        ms = (C.c_double * 5)()
        na, nw = C.c_int(), C.c_int()
        check(LIB.pbsa_mem_profile_read(self._h, ms, C.byref(na), C.byref(nw)))
        keys = ["kv_write", "compress_q", "score_select", "bsa_fwd", "mem_update"]
        return {"ms": dict(zip(keys, list(ms))), "attend_calls": na.value, "kv_writes": nw.value}

    def status(self) -> int:
        """Invalid-input flags since the last reset (bit 0 NaN logits, bit 1 NaN scores)."""
        f = C.c_int()
        check(LIB.pbsa_mem_status(self._h, C.byref(f), _stream()))
        return f.value

    def last_tile_pairs(self):
        """K3 tiles of the last call: [units, tiles, 2] int32 query blocks (second -1: none), or None
        when the call used the natural pairs (2t, 2t + 1)."""
        pr, t = C.c_void_p(), C.c_int()
        check(LIB.pbsa_last_tile_pairs(self._h, C.byref(pr), C.byref(t)))
        return self._view(pr.value, (self.units, t.value, 2), torch.int32) if pr.value else None

    def last_selection(self):
        sel, k, st, nk = C.c_void_p(), C.c_int(), C.c_void_p(), C.c_int()
        check(LIB.pbsa_last_selection(self._h, C.byref(sel), C.byref(k), C.byref(st), C.byref(nk)))
        rows = C.c_int()
        check(LIB.pbsa_last_selection_rows(self._h, C.byref(rows)))
        selt = self._view(sel.value, (self.units, rows.value or self.blocks_per_chunk, max(k.value, 0)), torch.int32) \
            if k.value else None
        stt = self._view(st.value, (self.units, nk.value), torch.float32) if nk.value else None
        return selt, stt
