"""Test helpers composing ORACLE ops into reference PBSA calls (test infrastructure only).

Everything here is computed by oracle/pbsa_oracle.cpp (the CPU restatement of the reference);
the helpers only gather inputs the way SPEC.md's call structure does.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) -> fp32, as torch does when uploading bf16 inputs."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def normal_bf16(seed: int, shape) -> np.ndarray:
    n = int(np.prod(shape))
    return bf16_round(orc.rng_normal(seed, n).reshape(shape))


def oracle_select(qc, kc_local, k):
    """A_L = coarse_attention(qc, K^c_L) (Eq. 10) and row-wise Top-K (Eq. 11)."""
    a_l = orc.coarse_attention(qc, kc_local)
    return orc.select_topk(a_l, k), a_l


def oracle_scores(qc, kc_all):
    """s_t = aggregate_scores(coarse_attention(qc, K^c_all)) (Eq. 7-8)."""
    return orc.aggregate_scores(orc.coarse_attention(qc, kc_all))


def oracle_attention(q_blocks, k_blocks, v_blocks, vis, qmask=None):
    """attention_sparse over a block store; vis [nqb, n_vis] store indices."""
    return orc.attention_sparse(q_blocks, k_blocks, v_blocks, vis, qmask=qmask)


def check_attention(out, want, rows_mask=None, max_abs=2e-2, mean_abs=2e-3):
    """The north-star bf16 tolerance: max-abs <= 2e-2 and mean-abs <= 2e-3 vs fp32 oracle."""
    out = np.asarray(out, np.float32)
    want = np.asarray(want, np.float32)
    if rows_mask is not None:
        out, want = out[rows_mask], want[rows_mask]
    err = np.abs(out - want)
    assert np.isfinite(out).all()
    assert err.max() <= max_abs, f"max-abs {err.max():.3e} > {max_abs}"
    assert err.mean() <= mean_abs, f"mean-abs {err.mean():.3e} > {mean_abs}"
    return float(err.max()), float(err.mean())


class OracleReplay:
    """The oracle's side of a sequence of PBSA calls on `units` independent heads: per-unit
    orc.Memory (push_chunk / update_persistent / assemble_kv) plus the K/V and
    representatives of every block still in P or L.  `call` replays one PBSA call of Alg. 1 on
    the same bf16 inputs the device saw and asserts the device's results:

      * Top-K indices of every query block            bit-exact
      * s_t of the k=0 pass over [P; L; current]       bit-exact
      * attention output on query blocks `check_qb`   max-abs 2e-2, mean-abs 2e-3
    and `check_ids` the P / L ids after a cache update (SPEC.md:209-217 order), bit-exact."""

    def __init__(self, units: int, capacity_c: int, window_chunks: int, bpc: int, b: int, d: int):
        self.units, self.bpc, self.b, self.d = units, bpc, b, d
        self.mem = [orc.Memory(capacity_c, window_chunks) for _ in range(units)]
        self.kst, self.vst, self.rep = {}, {}, {}  # (u, id) -> [b, d] K, V and [d] representative
        self.chunk = 0

    def call(self, q, k, v, k_top: int, update: bool, o=None, sel=None, s_t=None, check_qb=None, where=""):
        """q / k / v: [units, bpc*b, d] f32 (bf16-exact) of the current chunk; o [units, bpc*b, d]
        (None: skip the attention check); sel [units, bpc, k] / s_t [units, >= n_keys] device
        results (None where the device produced none).  Returns attention error stats."""
        bpc, b, d = self.bpc, self.b, self.d
        ids = np.arange(self.chunk * bpc, (self.chunk + 1) * bpc, dtype=np.int64)
        empty = np.zeros((0, b, d), np.float32)
        stats = []
        for u in range(self.units):
            a_ids, _, n_p, n_l = self.mem[u].assemble()
            p_ids, l_ids = a_ids[:n_p], a_ids[n_p:]
            qb = np.asarray(q[u], np.float32).reshape(bpc, b, d)
            cur_k = np.asarray(k[u], np.float32).reshape(bpc, b, d)
            cur_v = np.asarray(v[u], np.float32).reshape(bpc, b, d)
            qc = orc.compress_blocks(qb)
            kk = min(k_top, n_l)
            want_sel = np.zeros((bpc, 0), np.int32)
            if kk > 0:
                want_sel = orc.select_topk(orc.coarse_attention(qc, np.stack([self.rep[(u, i)] for i in l_ids])), kk)
                assert sel is not None and np.array_equal(np.asarray(sel[u]), want_sel), f"{where} unit {u}: Top-K"
            if o is not None:
                store_k = np.concatenate([np.stack([self.kst[(u, i)] for i in p_ids]) if n_p else empty, cur_k,
                                          np.stack([self.kst[(u, i)] for i in l_ids]) if n_l else empty])
                store_v = np.concatenate([np.stack([self.vst[(u, i)] for i in p_ids]) if n_p else empty, cur_v,
                                          np.stack([self.vst[(u, i)] for i in l_ids]) if n_l else empty])
                dense = np.arange(n_p + bpc)
                vis = np.stack([np.concatenate([dense, n_p + bpc + want_sel[i]]) for i in range(bpc)]).astype(np.int32)
                qmask = None
                if check_qb is not None:
                    qmask = np.zeros(bpc, np.uint8)
                    qmask[check_qb] = 1
                want = orc.attention_sparse(qb, store_k, store_v, vis, qmask=qmask)
                rows = slice(None) if check_qb is None else check_qb
                stats.append(check_attention(np.asarray(o[u], np.float32).reshape(bpc, b, d)[rows], want[rows]))
            if update:
                cur_rep = orc.compress_blocks(cur_k)
                zd = np.zeros((0, d), np.float32)
                keys_rep = np.concatenate([np.stack([self.rep[(u, i)] for i in p_ids]) if n_p else zd,
                                           np.stack([self.rep[(u, i)] for i in l_ids]) if n_l else zd, cur_rep])
                key_ids = np.concatenate([p_ids, l_ids, ids])
                s_ref = orc.aggregate_scores(orc.coarse_attention(qc, keys_rep))
                if s_t is not None:
                    got = np.ascontiguousarray(np.asarray(s_t[u])[:len(key_ids)], np.float32)
                    assert np.array_equal(got.view(np.uint32), s_ref.view(np.uint32)), f"{where} unit {u}: s_t"
                ev = self.mem[u].push_chunk(ids)
                self.mem[u].update_persistent(ev, key_ids, s_ref)
                for i in range(bpc):
                    self.kst[(u, ids[i])], self.vst[(u, ids[i])], self.rep[(u, ids[i])] = cur_k[i], cur_v[i], cur_rep[i]
                keep = set(self.mem[u].assemble()[0].tolist())
                for key in [key for key in self.kst if key[0] == u and key[1] not in keep]:
                    del self.kst[key], self.vst[key], self.rep[key]
        if update:
            self.chunk += 1
        return stats

    def ids(self, u: int):
        """(persistent ids, local ids) of unit u in assemble_kv order."""
        a_ids, _, n_p, _ = self.mem[u].assemble()
        return a_ids[:n_p], a_ids[n_p:]

    def check_ids(self, p_ids, l_ids, where=""):
        """Device P / L ids ([units][n] each, any sequence type) against the oracle, bit-exact."""
        for u in range(self.units):
            wp, wl = self.ids(u)
            assert np.array_equal(np.asarray(p_ids[u], np.int64), wp), f"{where} unit {u}: persistent ids"
            assert np.array_equal(np.asarray(l_ids[u], np.int64), wl), f"{where} unit {u}: local ids"
