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
