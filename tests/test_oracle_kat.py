"""Oracle vs every SPEC known-answer example and the hot-path property suites.

These pin the SPEC-only ops (which the reference ships no code for) before the oracle is trusted
as the GPU parity checker.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as orc

NEG = -np.inf
KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_kats.json")))


def arr(x):
    return np.array([[NEG if v == "-inf" else v for v in row] for row in x], np.float32)


@pytest.mark.parametrize("case", KATS["matmul"])
def test_matmul_kat(case):
    assert np.array_equal(orc.matmul(case["a"], case["b"]), np.array(case["out"], np.float32))


def test_matmul_identity_and_zero():
    m = np.arange(9, dtype=np.float32).reshape(3, 3) - 4
    assert np.array_equal(orc.matmul(np.eye(3, dtype=np.float32), m), m)
    assert np.array_equal(orc.matmul(np.zeros((3, 3), np.float32), m), np.zeros((3, 3)))


@pytest.mark.parametrize("case", KATS["softmax"])
def test_softmax_kat(case):
    mask = None if case["mask"] is None else arr(case["mask"])
    out = orc.masked_softmax_rows(np.array(case["scores"], np.float32), mask)
    assert np.allclose(out, np.array(case["out"], np.float32), atol=case.get("tol", 0), rtol=0)


def test_softmax_rejects_nan_and_bad_mask():
    with pytest.raises(orc.OracleError):
        orc.masked_softmax_rows(np.array([[np.nan, 1.0]], np.float32))
    with pytest.raises(orc.OracleError):
        orc.masked_softmax_rows(np.zeros((1, 2), np.float32), np.array([[0.5, 0]], np.float32))


def test_softmax_properties():
    g = np.random.default_rng(3)
    s = (g.standard_normal((50, 40)) * 5).astype(np.float32)
    p = orc.masked_softmax_rows(s)
    assert np.all(np.abs(p.astype(np.float64).sum(1) - 1) <= 1e-6)
    assert np.all((p >= 0) & (p <= 1))
    p2 = orc.masked_softmax_rows(s + np.float32(3.0))  # shift invariance
    assert np.max(np.abs(p2 - p)) < 1e-6


@pytest.mark.parametrize("case", KATS["blockify"])
def test_blockify_kat(case):
    dims, shp = case["dims"], case["shape"]
    if "x" in case:
        x = np.array(case["x"], np.float32).reshape(dims)
        xb = orc.blockify(x, shp)
        assert np.array_equal(xb[..., 0], np.array(case["blocks"], np.float32))
        assert np.array_equal(orc.unblockify(xb, dims, shp), x)
    else:
        x = np.zeros(dims, np.float32)
        xb = orc.blockify(x, shp)
        assert xb.shape[0] == case["n_b"] and xb.shape[1] == case["b"]


def test_blockify_rejects_nondivisible():
    with pytest.raises(orc.OracleError, match="axis h"):
        orc.blockify(np.zeros((2, 5, 4, 1), np.float32), (1, 2, 2))


def test_blockify_permutation_grid():
    """SPEC.md:139-141 + acceptance 3: round trips and brute-force index-map agreement."""
    g = np.random.default_rng(11)
    for shp in [(1, 1, 1), (1, 2, 2), (3, 4, 4), (1, 8, 8), (2, 2, 2)]:
        dims = (shp[0] * 2, shp[1] * 2, shp[2] * 3, 3)
        x = g.standard_normal(dims).astype(np.float32)
        xb = orc.blockify(x, shp)
        assert np.array_equal(orc.unblockify(xb, dims, shp), x)
        t, h, w, _ = dims
        for flat in range(t * h * w):
            bid, off = orc.block_index_map((t, h, w), shp, flat)
            ti, hi, wi = flat // (h * w), (flat // w) % h, flat % w
            assert np.array_equal(xb[bid, off], x[ti, hi, wi])


@pytest.mark.parametrize("case", KATS["block_index_map"])
def test_block_index_map_kat(case):
    t, h, w = case["dims"]
    ti, hi, wi = case["source"]
    flat = (ti * h + hi) * w + wi
    assert list(orc.block_index_map(case["dims"], case["shape"], flat)) == case["out"]


@pytest.mark.parametrize("case", KATS["compress"])
def test_compress_kat(case):
    out = orc.compress_blocks(np.array([case["block"]], np.float32))
    assert np.array_equal(out[0], np.array(case["out"], np.float32))


def test_coarse_attention_kats():
    c = KATS["coarse_attention"][0]
    assert np.array_equal(orc.coarse_attention(c["qc"], c["kc"]), np.array(c["out"], np.float32))
    c = KATS["coarse_attention"][1]
    p = orc.coarse_attention(c["orth_q"], c["kc"])
    assert np.allclose(p, 1.0 / 3.0, atol=1e-7)
    g = np.random.default_rng(5)  # vs dense softmax oracle <= 1e-6
    qc, kc = g.standard_normal((2, 8)).astype(np.float32), g.standard_normal((3, 8)).astype(np.float32)
    want = np.exp((qc.astype(np.float64) @ kc.T.astype(np.float64)) / math.sqrt(8))
    want /= want.sum(1, keepdims=True)
    assert np.max(np.abs(orc.coarse_attention(qc, kc) - want)) <= 1e-6


@pytest.mark.parametrize("case", KATS["aggregate"])
def test_aggregate_kat(case):
    assert np.allclose(orc.aggregate_scores(case["a"]), np.array(case["out"], np.float32), atol=0)


def test_aggregate_sums_to_one():
    g = np.random.default_rng(8)
    a = orc.coarse_attention(g.standard_normal((17, 16)), g.standard_normal((40, 16)))
    assert abs(float(orc.aggregate_scores(a).astype(np.float64).sum()) - 1.0) <= 1e-5


@pytest.mark.parametrize("case", KATS["topk_count"])
def test_topk_count_kat(case):
    assert orc.topk_count(case["n_local"], case["ratio"]) == case["k"]


@pytest.mark.parametrize("case", KATS["select_topk"])
def test_select_topk_kat(case):
    out = orc.select_topk(np.array(case["a"], np.float32), case["k"])
    assert out.tolist() == case["sel"]


def test_select_topk_rejects_empty_local():
    with pytest.raises(orc.OracleError):
        orc.topk_count(0, 0.25)


def test_select_topk_properties():
    """brute force (N<=32), shift invariance, nesting in k."""
    g = np.random.default_rng(21)
    for _ in range(200):
        n = int(g.integers(1, 33))
        a = g.integers(0, 6, (4, n)).astype(np.float32) / 8  # many exact ties
        k = int(g.integers(1, n + 1))
        sel = orc.select_topk(a, k)
        for r in range(4):
            order = sorted(range(n), key=lambda j: (-a[r, j], j))
            assert sel[r].tolist() == sorted(order[:k])
        assert np.array_equal(orc.select_topk(a + np.float32(0.5), k), sel)
        if k < n:
            bigger = orc.select_topk(a, k + 1)
            for r in range(4):
                assert set(sel[r]) <= set(bigger[r])


@pytest.mark.parametrize("case", KATS["build_mask"])
def test_build_mask_kat(case):
    m = orc.build_mask(case["nqb"], case["b"], case["n_p_tok"], case["n_local"], case["sel"])
    assert np.array_equal(m, arr(case["mask"]))


def test_build_mask_zero_count():
    g = np.random.default_rng(2)
    nqb, b, n_p, nl, k = 5, 3, 7, 9, 4
    sel = np.sort(np.stack([g.choice(nl, k, replace=False) for _ in range(nqb)]), 1)
    m = orc.build_mask(nqb, b, n_p, nl, sel)
    assert np.all((m == 0).sum(1) == n_p + k * b)


def test_attention_reference_kats():
    g = np.random.default_rng(4)
    q = g.standard_normal((5, 8)).astype(np.float32)
    v = g.standard_normal((1, 8)).astype(np.float32)
    out = orc.attention_reference(q, g.standard_normal((1, 8)), v)
    assert np.allclose(out, np.repeat(v, 5, 0), atol=1e-7)
    k = g.standard_normal((6, 8)).astype(np.float32)
    vv = g.standard_normal((6, 8)).astype(np.float32)
    mask = np.full((5, 6), NEG, np.float32)
    mask[:, 4] = 0
    assert np.allclose(orc.attention_reference(q, k, vv, mask), np.repeat(vv[4:5], 5, 0), atol=1e-7)


def _random_geometry(g, topk):
    nqb = int(g.integers(1, 9))
    nl = int(g.integers(1, 17))
    npb = int(g.integers(0, 5))
    b = int(g.integers(1, 17))
    d = int(g.integers(1, 33))
    k = orc.topk_count(nl, topk)
    q = g.standard_normal((nqb, b, d)).astype(np.float32)
    store_k = g.standard_normal((npb + nl, b, d)).astype(np.float32)
    store_v = g.standard_normal((npb + nl, b, d)).astype(np.float32)
    qc = orc.compress_blocks(q)
    kc = orc.compress_blocks(store_k[npb:])
    sel = orc.select_topk(orc.coarse_attention(qc, kc), k)
    return nqb, nl, npb, b, d, k, q, store_k, store_v, sel


@pytest.mark.parametrize("topk", [1 / 16, 1 / 8, 1 / 4, 1.0])
def test_acceptance1_sparse_matches_reference(topk):
    """>=200 seeded geometries overall, max-abs <= 1e-5."""
    g = np.random.default_rng(int(topk * 1000))
    for _ in range(60):
        nqb, nl, npb, b, d, k, q, sk, sv, sel = _random_geometry(g, topk)
        vis = np.concatenate([np.tile(np.arange(npb), (nqb, 1)), sel + npb], 1).astype(np.int32)
        sparse = orc.attention_sparse(q, sk, sv, vis)
        mask = orc.build_mask(nqb, b, npb * b, nl, sel)
        dense = orc.attention_reference(q.reshape(-1, d), sk.reshape(-1, d), sv.reshape(-1, d), mask)
        assert np.max(np.abs(sparse.reshape(-1, d) - dense)) <= 1e-5


def test_acceptance2_full_visibility_equals_dense():
    g = np.random.default_rng(77)
    for _ in range(50):
        nqb, nl, npb, b, d, k, q, sk, sv, sel = _random_geometry(g, 1.0)
        vis = np.tile(np.arange(npb + nl), (nqb, 1)).astype(np.int32)
        sparse = orc.attention_sparse(q, sk, sv, vis)
        dense = orc.attention_reference(q.reshape(-1, d), sk.reshape(-1, d), sv.reshape(-1, d))
        assert np.max(np.abs(sparse.reshape(-1, d) - dense)) <= 1e-6


def test_attention_sparse_convexity():
    g = np.random.default_rng(9)
    nqb, nl, npb, b, d, k, q, sk, sv, sel = _random_geometry(g, 0.25)
    vis = np.concatenate([np.tile(np.arange(npb), (nqb, 1)), sel + npb], 1).astype(np.int32)
    out = orc.attention_sparse(q, sk, sv, vis)
    for i in range(nqb):
        vals = sv[vis[i]].reshape(-1, d)
        assert np.all(out[i] <= vals.max(0) + 1e-6) and np.all(out[i] >= vals.min(0) - 1e-6)


@pytest.mark.parametrize("case", KATS["update_persistent"])
def test_update_persistent_kat(case):
    names = ["s"] + list(case["dynamic"]) + list(case["evicted"])
    ident = {n: i for i, n in enumerate(names)}
    cand = list(case["dynamic"].items()) + list(case["evicted"].items())
    ids = [ident["s"]] + [ident[n] for n, _ in cand]
    scores = [0.0] + [s for _, s in cand]
    kept = orc.topc_select(ids, scores, [1] + [0] * len(cand), case["C"])
    assert kept[0]  # the sink is always retained
    got = sorted([n for (n, s), kk in zip(cand, kept[1:]) if kk], key=lambda n: -dict(cand)[n])
    assert got == case["out_dynamic"]


def test_acceptance4_topc_bruteforce():
    """1000 random instances with <= 16 candidates, sinks kept, capacity <= C."""
    g = np.random.default_rng(4242)
    for _ in range(1000):
        n = int(g.integers(1, 17))
        ids = g.permutation(100)[:n].astype(np.int64)
        scores = (g.integers(0, 5, n) / 4).astype(np.float32)
        sink = g.uniform(size=n) < 0.2
        C = int(g.integers(int(sink.sum()), 17))
        kept = orc.topc_select(ids, scores, sink, C)
        assert np.all(kept[sink]) and kept.sum() <= max(C, sink.sum())
        rest = sorted([i for i in range(n) if not sink[i]], key=lambda i: (-scores[i], ids[i]))
        want = set(rest[: max(0, C - int(sink.sum()))])
        assert set(np.nonzero(kept & ~sink)[0]) == want


def test_memory_push_and_evict_kats():
    m = orc.Memory(capacity_c=6, window_chunks=2)
    assert len(m.push_chunk([0, 1, 2])) == 0
    assert len(m.push_chunk([3, 4, 5])) == 0
    ev = m.push_chunk([6, 7, 8])  # [A,B] + C evicts A
    assert ev.tolist() == [0, 1, 2]
    with pytest.raises(orc.OracleError):
        m.push_chunk([8, 9])  # id ordering violation


def test_memory_state_machine_invariants():
    """SPEC.md:219-223 + rollout invariants (:485,:488) over random score streams."""
    g = np.random.default_rng(31)
    bpc, C, W = 4, 10, 3
    m = orc.Memory(C, W)
    last_ev = -1
    for chunk in range(12):
        ids = np.arange(chunk * bpc, (chunk + 1) * bpc)
        p_ids, _, n_p, n_l = m.assemble()
        all_ids = np.concatenate([p_ids, ids])
        scores = g.integers(0, 7, len(all_ids)).astype(np.float32) / 8
        ev = m.push_chunk(ids)
        if len(ev):
            assert ev.min() > last_ev
            last_ev = ev.max()
        m.update_persistent(ev, all_ids, scores)
        a_ids, reg, n_p, n_l = m.assemble()
        assert n_p <= C and n_l <= W * bpc
        assert len(set(a_ids.tolist())) == len(a_ids)  # P and L disjoint
        if chunk >= W:
            assert m.num_sinks() == bpc and set(range(bpc)) <= set(a_ids[:n_p].tolist())


def test_rollout_first_eviction_at_third_chunk():
    """C=6 frames, window 6 frames, 3-frame chunks -> first eviction at push 3."""
    bpc = 3 * 26
    m = orc.Memory(6 * 26, 2)
    evs = [len(m.push_chunk(np.arange(c * bpc, (c + 1) * bpc))) for c in range(3)]
    assert evs == [0, 0, bpc]


@pytest.mark.parametrize("case", KATS["kv_length"])
def test_kv_length_kat(case):
    assert orc.kv_length(case["n_c"], case["local"], case["persist"]) == case["n_kv"]


def test_kv_length_rejects_nonintegral():
    with pytest.raises(orc.OracleError):
        orc.kv_length(5377, 0.5, 0.25)


@pytest.mark.parametrize("case", KATS["kv_bytes"])
def test_kv_bytes_kat(case):
    assert orc.kv_bytes(*case["args"]) == case["bytes"]


def test_flop_count_properties():
    dn, sp, r = orc.flop_count(4096, 0, 4096, 4096, 1, 64)  # full visibility -> ratio ~ 1
    assert abs(r - 1) < 1e-3
    dn, sp, r = orc.flop_count(65536, 0, 65536 * 16, 4096, 16, 64)  # 1/16 of local -> ~16
    assert 15 < r <= 16
    for row in KATS["kv_length"][:8]:  # SPEC.md:399 on the appendix grid
        n_c = row["n_c"]
        nl = int(n_c * row["local"])
        npt = int(nl * row["persist"])
        k = max(1, math.ceil(nl // 64 * 0.0625))
        assert orc.flop_count(n_c, npt, nl, 64, k, 64)[2] > 1
    assert orc.kv_length(10752 // 2, 2, 0.25) - 10752 == 2688


def test_attention_sparse_backward_matches_autograd():
    """The backward oracle (no reference implementation exists) is pinned to the derivative of
    the dense masked attention by torch autograd in float64."""
    import torch
    g = np.random.default_rng(11)
    nqb, bq, bkv, d, n_store = 3, 5, 4, 8, 6
    q = g.standard_normal((nqb, bq, d)).astype(np.float32)
    k = g.standard_normal((n_store, bkv, d)).astype(np.float32)
    v = g.standard_normal((n_store, bkv, d)).astype(np.float32)
    do = g.standard_normal((nqb, bq, d)).astype(np.float32)
    vis = np.array([[0, 2, 5], [1, 2, 3], [4, 0, 5]], np.int32)
    dq, dk, dv = orc.attention_sparse_backward(q, k, v, vis, do)
    qt = torch.tensor(q, dtype=torch.float64, requires_grad=True)
    kt = torch.tensor(k, dtype=torch.float64, requires_grad=True)
    vt = torch.tensor(v, dtype=torch.float64, requires_grad=True)
    scale = orc.attention_scale(d)
    outs = []
    for i in range(nqb):
        kk = kt[vis[i]].reshape(-1, d)
        vv = vt[vis[i]].reshape(-1, d)
        outs.append(torch.softmax(qt[i] @ kk.T * scale, -1) @ vv)
    (torch.stack(outs) * torch.tensor(do, dtype=torch.float64)).sum().backward()
    np.testing.assert_allclose(dq, qt.grad.numpy(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dk, kt.grad.numpy(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dv, vt.grad.numpy(), rtol=1e-5, atol=1e-6)
