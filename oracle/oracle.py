"""ctypes front-end for the CPU ORACLE (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs -- always as the checker or the CPU baseline, never as
the thing measured or shipped.  The product package (paper_2604_21221_b200) must not import it.

Every function restates a reference op; see oracle/pbsa_oracle.h for the file:line citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libpbsa_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64 = C.c_int64


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        build()
    lib = C.CDLL(LIB_PATH)
    lib.orc_last_error.restype = C.c_char_p
    lib.orc_rng_derive.restype = C.c_uint64
    lib.orc_rng_derive.argtypes = [C.c_uint64, C.c_uint64]
    lib.orc_attention_scale.restype = C.c_float
    lib.orc_attention_scale.argtypes = [_i64]
    lib.orc_mem_create.restype = C.c_void_p
    lib.orc_mem_create.argtypes = [_i64, _i64]
    lib.orc_mem_destroy.argtypes = [C.c_void_p]
    lib.orc_mem_num_sinks.restype = _i64
    lib.orc_mem_num_sinks.argtypes = [C.c_void_p]
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


class OracleError(ValueError):
    pass


def _chk(rc: int) -> None:
    if rc != 0:
        raise OracleError(lib().orc_last_error().decode())


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ---- rng.hpp ---------------------------------------------------------------------------------
def rng_normal(seed: int, n: int) -> np.ndarray:
    out = np.empty(int(n), np.float32)
    L = lib()
    L.orc_rng_normal.argtypes = [C.c_uint64, _i64, _f32p]
    _chk(L.orc_rng_normal(C.c_uint64(seed), int(n), out))
    return out


def rng_uniform(seed: int, n: int) -> np.ndarray:
    out = np.empty(int(n), np.float64)
    L = lib()
    L.orc_rng_uniform.argtypes = [C.c_uint64, _i64, _f64p]
    _chk(L.orc_rng_uniform(C.c_uint64(seed), int(n), out))
    return out


def rng_derive(seed: int, stream: int) -> int:
    return int(lib().orc_rng_derive(C.c_uint64(seed), C.c_uint64(stream)))


# ---- tensor.cpp ------------------------------------------------------------------------------
def matmul_nt(a, b) -> np.ndarray:
    a, b = _f32(a), _f32(b)
    if a.shape[1] != b.shape[1]:
        raise OracleError("matmul_nt: a.cols != b.cols")
    out = np.empty((a.shape[0], b.shape[0]), np.float32)
    L = lib()
    L.orc_matmul_nt.argtypes = [_f32p, _i64, _i64, _f32p, _i64, _f32p]
    _chk(L.orc_matmul_nt(a, a.shape[0], a.shape[1], b, b.shape[0], out))
    return out


def matmul(a, b) -> np.ndarray:
    a, b = _f32(a), _f32(b)
    if a.shape[1] != b.shape[0]:
        raise OracleError("matmul: a.cols != b.rows")
    out = np.empty((a.shape[0], b.shape[1]), np.float32)
    L = lib()
    L.orc_matmul.argtypes = [_f32p, _i64, _i64, _f32p, _i64, _f32p]
    _chk(L.orc_matmul(a, a.shape[0], a.shape[1], b, b.shape[1], out))
    return out


def masked_softmax_rows(scores, mask=None) -> np.ndarray:
    s = _f32(scores)
    out = np.empty_like(s)
    L = lib()
    L.orc_masked_softmax_rows.argtypes = [_f32p, _i64, _i64, C.c_void_p, _f32p]
    m = None
    if mask is not None:
        m = _f32(mask)
        if m.shape != s.shape:
            raise OracleError("masked_softmax_rows: mask shape mismatch")
    _chk(L.orc_masked_softmax_rows(s, s.shape[0], s.shape[1],
                                   None if m is None else m.ctypes.data, out))
    return out


# ---- blockify.cpp ----------------------------------------------------------------------------
def blockify(x, shape) -> np.ndarray:
    x = _f32(x)
    t, h, w, d = x.shape
    out = np.empty(x.size, np.float32)
    L = lib()
    L.orc_blockify.argtypes = [_f32p] + [_i64] * 7 + [_f32p]
    _chk(L.orc_blockify(x, t, h, w, d, *shape, out))
    b = shape[0] * shape[1] * shape[2]
    return out.reshape(-1, b, d)


def unblockify(xb, dims, shape) -> np.ndarray:
    xb = _f32(xb)
    t, h, w, d = dims
    out = np.empty(t * h * w * d, np.float32)
    L = lib()
    L.orc_unblockify.argtypes = [_f32p] + [_i64] * 7 + [_f32p]
    _chk(L.orc_unblockify(xb, t, h, w, d, *shape, out))
    return out.reshape(t, h, w, d)


def block_index_map(dims3, shape, flat):
    bid, off = _i64(), _i64()
    L = lib()
    L.orc_block_index_map.argtypes = [_i64] * 7 + [C.POINTER(_i64), C.POINTER(_i64)]
    _chk(L.orc_block_index_map(*dims3, *shape, int(flat), C.byref(bid), C.byref(off)))
    return bid.value, off.value


# ---- router ----------------------------------------------------------------
def compress_blocks(xb) -> np.ndarray:
    xb = _f32(xb)
    nb, b, d = xb.shape
    out = np.empty((nb, d), np.float32)
    L = lib()
    L.orc_compress_blocks.argtypes = [_f32p, _i64, _i64, _i64, _f32p]
    _chk(L.orc_compress_blocks(xb, nb, b, d, out))
    return out


def attention_scale(d: int) -> float:
    return float(np.float32(lib().orc_attention_scale(int(d))))


def coarse_logits(qc, kc, scale=None) -> np.ndarray:
    qc, kc = _f32(qc), _f32(kc)
    d = qc.shape[1]
    scale = attention_scale(d) if scale is None else scale
    out = np.empty((qc.shape[0], kc.shape[0]), np.float32)
    L = lib()
    L.orc_coarse_logits.argtypes = [_f32p, _i64, _f32p, _i64, _i64, C.c_float, _f32p]
    _chk(L.orc_coarse_logits(qc, qc.shape[0], kc, kc.shape[0], d, scale, out))
    return out


def coarse_attention(qc, kc, scale=None) -> np.ndarray:
    qc, kc = _f32(qc), _f32(kc)
    d = qc.shape[1]
    scale = attention_scale(d) if scale is None else scale
    out = np.empty((qc.shape[0], kc.shape[0]), np.float32)
    L = lib()
    L.orc_coarse_attention.argtypes = [_f32p, _i64, _f32p, _i64, _i64, C.c_float, _f32p]
    _chk(L.orc_coarse_attention(qc, qc.shape[0], kc, kc.shape[0], d, scale, out))
    return out


def aggregate_scores(a) -> np.ndarray:
    a = _f32(a)
    out = np.empty(a.shape[1], np.float32)
    L = lib()
    L.orc_aggregate_scores.argtypes = [_f32p, _i64, _i64, _f32p]
    _chk(L.orc_aggregate_scores(a, a.shape[0], a.shape[1], out))
    return out


def topk_count(n_local: int, ratio: float) -> int:
    k = _i64()
    L = lib()
    L.orc_topk_count.argtypes = [_i64, C.c_double, C.POINTER(_i64)]
    _chk(L.orc_topk_count(int(n_local), float(ratio), C.byref(k)))
    return k.value


def select_topk(a, k: int) -> np.ndarray:
    a = _f32(a)
    out = np.empty((a.shape[0], int(k)), np.int32)
    L = lib()
    L.orc_select_topk.argtypes = [_f32p, _i64, _i64, _i64, _i32p]
    _chk(L.orc_select_topk(a, a.shape[0], a.shape[1], int(k), out))
    return out


def build_mask(nqb, b, n_p_tok, n_local, sel) -> np.ndarray:
    sel = np.ascontiguousarray(sel, np.int32)
    k = sel.shape[1] if sel.ndim == 2 else 0
    out = np.empty((nqb * b, n_p_tok + n_local * b), np.float32)
    L = lib()
    L.orc_build_mask.argtypes = [_i64, _i64, _i64, _i64, _i32p, _i64, _f32p]
    _chk(L.orc_build_mask(nqb, b, n_p_tok, n_local, sel.reshape(-1) if k else np.zeros(1, np.int32),
                          k, out))
    return out


# ---- attention -------------------------------------------------------------
def attention_reference(q, k, v, mask=None, scale=None) -> np.ndarray:
    q, k, v = _f32(q), _f32(k), _f32(v)
    d = q.shape[1]
    scale = attention_scale(d) if scale is None else scale
    out = np.empty((q.shape[0], v.shape[1]), np.float32)
    L = lib()
    L.orc_attention_reference.argtypes = [_f32p, _i64, _f32p, _f32p, _i64, _i64, C.c_void_p,
                                          C.c_float, _f32p]
    m = None if mask is None else _f32(mask)
    _chk(L.orc_attention_reference(q, q.shape[0], k, v, k.shape[0], d,
                                   None if m is None else m.ctypes.data, scale, out))
    return out


def attention_sparse(q_blocks, k_store, v_store, vis, scale=None, qmask=None, want_lse=False):
    """q_blocks [nqb, bq, d]; k_store/v_store [n_store_blocks, bkv, d]; vis [nqb, n_vis] store
    block indices in visiting order.  Returns out [nqb, bq, d] (and lse [nqb, bq])."""
    q, k, v = _f32(q_blocks), _f32(k_store), _f32(v_store)
    nqb, bq, d = q.shape
    bkv = k.shape[1]
    vis = np.ascontiguousarray(vis, np.int32)
    n_vis = vis.shape[1]
    scale = attention_scale(d) if scale is None else scale
    out = np.zeros((nqb, bq, d), np.float32)
    lse = np.zeros((nqb, bq), np.float32)
    qm = None if qmask is None else np.ascontiguousarray(qmask, np.uint8)
    L = lib()
    L.orc_attention_sparse.argtypes = [_f32p, _i64, _i64, _f32p, _f32p, _i64, _i32p, _i64, _i64,
                                       C.c_float, C.c_void_p, _f32p, _f32p]
    _chk(L.orc_attention_sparse(q, nqb, bq, k, v, bkv, vis.reshape(-1) if n_vis else
                                np.zeros(1, np.int32), n_vis, d, scale,
                                None if qm is None else qm.ctypes.data, out, lse))
    return (out, lse) if want_lse else out


def attention_sparse_backward(q_blocks, k_store, v_store, vis, d_out, scale=None):
    """Gradients (dq [nqb, bq, d], dk, dv [n_store, bkv, d]) of attention_sparse for upstream
    d_out [nqb, bq, d]; fp64 inside (see pbsa_oracle.h)."""
    q, k, v, g = _f32(q_blocks), _f32(k_store), _f32(v_store), _f32(d_out)
    nqb, bq, d = q.shape
    n_store, bkv = k.shape[0], k.shape[1]
    vis = np.ascontiguousarray(vis, np.int32)
    n_vis = vis.shape[1]
    scale = attention_scale(d) if scale is None else scale
    dq = np.zeros((nqb, bq, d), np.float32)
    dk = np.zeros((n_store, bkv, d), np.float32)
    dv = np.zeros_like(dk)
    L = lib()
    L.orc_attention_sparse_backward.argtypes = [_f32p, _i64, _i64, _f32p, _f32p, _i64, _i32p, _i64, _i64,
                                                C.c_float, _f32p, _f32p, _f32p, _f32p, _i64]
    _chk(L.orc_attention_sparse_backward(q, nqb, bq, k, v, bkv, vis.reshape(-1) if n_vis else
                                         np.zeros(1, np.int32), n_vis, d, scale, g, dq, dk, dv, n_store))
    return dq, dk, dv


def flop_count(nq, np_, nl, b, k_sel, d):
    dn, sp, r = C.c_double(), C.c_double(), C.c_double()
    L = lib()
    L.orc_flop_count.argtypes = [_i64] * 6 + [C.POINTER(C.c_double)] * 3
    _chk(L.orc_flop_count(nq, np_, nl, b, k_sel, d, C.byref(dn), C.byref(sp), C.byref(r)))
    return dn.value, sp.value, r.value


def kv_length(n_c, local_ratio, persist_ratio) -> int:
    out = _i64()
    L = lib()
    L.orc_kv_length.argtypes = [_i64, C.c_double, C.c_double, C.POINTER(_i64)]
    _chk(L.orc_kv_length(n_c, local_ratio, persist_ratio, C.byref(out)))
    return out.value


def kv_bytes(tokens, layers, kv_heads, head_dim, bpe) -> int:
    out = _i64()
    L = lib()
    L.orc_kv_bytes.argtypes = [_i64] * 5 + [C.POINTER(_i64)]
    _chk(L.orc_kv_bytes(tokens, layers, kv_heads, head_dim, bpe, C.byref(out)))
    return out.value


def topc_select(ids, scores, is_sink, capacity_c) -> np.ndarray:
    ids = np.ascontiguousarray(ids, np.int64)
    scores = _f32(scores)
    sk = np.ascontiguousarray(is_sink, np.uint8)
    kept = np.zeros(len(ids), np.uint8)
    L = lib()
    L.orc_topc_select.argtypes = [_i64p, _f32p, _u8p, _i64, _i64, _u8p]
    _chk(L.orc_topc_select(ids, scores, sk, len(ids), int(capacity_c), kept))
    return kept.astype(bool)


# ---- memory ----------------------------------------------------------------
class Memory:
    """PersistentMemory + LocalWindow state machine (per head)."""

    def __init__(self, capacity_c: int, window_chunks: int):
        self._h = lib().orc_mem_create(int(capacity_c), int(window_chunks))
        if not self._h:
            raise OracleError(lib().orc_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_mem_destroy(self._h)
            self._h = None

    def push_chunk(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, np.int64)
        ev = np.zeros(max(1, 1 << 16), np.int64)
        n = _i64()
        L = lib()
        L.orc_mem_push_chunk.argtypes = [C.c_void_p, _i64p, _i64, _i64p, _i64, C.POINTER(_i64)]
        _chk(L.orc_mem_push_chunk(self._h, ids, len(ids), ev, len(ev), C.byref(n)))
        return ev[: n.value].copy()

    def update_persistent(self, evicted, score_ids, scores) -> None:
        ev = np.ascontiguousarray(evicted, np.int64)
        si = np.ascontiguousarray(score_ids, np.int64)
        sc = _f32(scores)
        L = lib()
        L.orc_mem_update_persistent.argtypes = [C.c_void_p, _i64p, _i64, _i64p, _f32p, _i64]
        _chk(L.orc_mem_update_persistent(self._h, ev if len(ev) else np.zeros(1, np.int64), len(ev),
                                         si if len(si) else np.zeros(1, np.int64),
                                         sc if len(sc) else np.zeros(1, np.float32), len(si)))

    def assemble(self):
        cap = 1 << 20
        ids = np.zeros(cap, np.int64)
        reg = np.zeros(cap, np.int32)
        n_p, n_l = _i64(), _i64()
        L = lib()
        L.orc_mem_assemble.argtypes = [C.c_void_p, _i64p, _i32p, _i64, C.POINTER(_i64),
                                       C.POINTER(_i64)]
        _chk(L.orc_mem_assemble(self._h, ids, reg, cap, C.byref(n_p), C.byref(n_l)))
        n = n_p.value + n_l.value
        return ids[:n].copy(), reg[:n].copy(), n_p.value, n_l.value

    def dynamic(self):
        cap = 1 << 16
        ids = np.zeros(cap, np.int64)
        sc = np.zeros(cap, np.float32)
        n = _i64()
        L = lib()
        L.orc_mem_dynamic.argtypes = [C.c_void_p, _i64p, _f32p, _i64, C.POINTER(_i64)]
        _chk(L.orc_mem_dynamic(self._h, ids, sc, cap, C.byref(n)))
        return ids[: n.value].copy(), sc[: n.value].copy()

    def num_sinks(self) -> int:
        return int(lib().orc_mem_num_sinks(self._h))


# ---- the reference itself (oracle/_ref), used to pin the restated primitives ----------------
def ref_lib():
    """The reference's own sources compiled by `make -C oracle ref` (None if absent)."""
    if not os.path.exists(REF_PATH):
        return None
    L = C.CDLL(REF_PATH)
    L.ref_last_error.restype = C.c_char_p
    L.ref_rng_derive.restype = C.c_uint64
    L.ref_rng_derive.argtypes = [C.c_uint64, C.c_uint64]
    return L
