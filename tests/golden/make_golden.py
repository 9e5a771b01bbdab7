"""Generates tests/golden/ref_primitives.npz by running THE REFERENCE ITSELF.

The reference's tensor/blockify/rng sources (/root/reference/proj) are compiled where they lie
into oracle/_ref/libpbsa_ref.so (`make -C oracle ref`); this script drives them through the
C shim (oracle/ref_shim.cpp) on seeded inputs and stores inputs + outputs as small fixtures, so
the oracle restatement can be pinned against the reference on machines without /root/reference
(the GPU box).  Run from the repo root:  python tests/golden/make_golden.py
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i64 = C.c_int64


def main():
    ref = orc.ref_lib()
    if ref is None:
        raise SystemExit("oracle/_ref/libpbsa_ref.so missing: run `make -C oracle ref` first")
    ref.ref_rng_normal.argtypes = [C.c_uint64, i64, f32p]
    ref.ref_matmul_nt.argtypes = [f32p, i64, i64, f32p, i64, f32p]
    ref.ref_matmul.argtypes = [f32p, i64, i64, f32p, i64, f32p]
    ref.ref_masked_softmax_rows.argtypes = [f32p, i64, i64, C.c_void_p, f32p]
    ref.ref_blockify.argtypes = [f32p] + [i64] * 7 + [f32p]
    out = {}

    rn = np.empty(4097, np.float32)
    ref.ref_rng_normal(C.c_uint64(20260417), 4097, rn)
    out["rng_seed"] = np.array([20260417], np.uint64)
    out["rng_normal"] = rn
    out["rng_derive"] = np.array([ref.ref_rng_derive(C.c_uint64(s), C.c_uint64(t))
                                  for s in (0, 1, 7, 2**63 + 5) for t in (0, 1, 2, 99)], np.uint64)

    # matmul_nt / matmul on seeded, magnitude-varied inputs (exercise fp64 accumulation order)
    g = np.random.default_rng(1234)
    a = (g.standard_normal((37, 129)) * np.exp(g.uniform(-6, 6, (37, 129)))).astype(np.float32)
    b = (g.standard_normal((53, 129)) * np.exp(g.uniform(-6, 6, (53, 129)))).astype(np.float32)
    c = np.empty((37, 53), np.float32)
    ref.ref_matmul_nt(a, 37, 129, b, 53, c)
    out.update(mm_nt_a=a, mm_nt_b=b, mm_nt_out=c)
    bm = (g.standard_normal((129, 41)) * np.exp(g.uniform(-4, 4, (129, 41)))).astype(np.float32)
    c2 = np.empty((37, 41), np.float32)
    ref.ref_matmul(a, 37, 129, bm, 41, c2)
    out.update(mm_b=bm, mm_out=c2)

    # masked softmax: wide logits, random -inf masks, one fully masked row, exact ties
    s = (g.standard_normal((24, 300)) * 8).astype(np.float32)
    s[3, :] = 0.5
    s[5, 10:20] = s[5, 9]
    mask = np.where(g.uniform(size=(24, 300)) < 0.3, -np.inf, 0.0).astype(np.float32)
    mask[7, :] = -np.inf
    p = np.empty_like(s)
    ref.ref_masked_softmax_rows(s, 24, 300, mask.ctypes.data, p)
    p0 = np.empty_like(s)
    ref.ref_masked_softmax_rows(s, 24, 300, None, p0)
    out.update(sm_scores=s, sm_mask=mask, sm_out=p, sm_out_nomask=p0)

    # blockify over the SPEC shape grid incl. the paper's [3,4,4] and [1,8,8]
    cases = [((2, 2, 2, 1), (1, 2, 2)), ((3, 8, 8, 2), (3, 4, 4)), ((2, 16, 16, 3), (1, 8, 8)),
             ((4, 4, 6, 2), (2, 2, 2)), ((3, 30, 52, 2), (1, 15, 4)), ((2, 3, 5, 4), (1, 1, 1))]
    for i, (dims, shp) in enumerate(cases):
        x = g.standard_normal(dims).astype(np.float32)
        xb = np.empty(x.size, np.float32)
        rc = ref.ref_blockify(x, *dims, *shp, xb)
        assert rc == 0
        out[f"bk{i}_dims"] = np.array(dims, np.int64)
        out[f"bk{i}_shape"] = np.array(shp, np.int64)
        out[f"bk{i}_x"] = x
        out[f"bk{i}_out"] = xb
    out["bk_n"] = np.array([len(cases)], np.int64)

    path = os.path.join(ROOT, "tests", "golden", "ref_primitives.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
