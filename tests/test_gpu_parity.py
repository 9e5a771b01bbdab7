"""GPU parity: every kernel of the PBSA hot path against the CPU oracle, through the C ABI.

Bars (BASELINE.json north_star): selected block indices and updated memory-block ids bit-exact,
s_t bit-exact, compression bit-exact; attention output max-abs <= 2e-2 and mean-abs <= 2e-3 vs
the fp32 oracle on the same bf16-rounded inputs.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from tests.pbsa_oracle_compose import OracleReplay, bf16_round, check_attention, normal_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_21221_b200 as pb
    return pb


def dev(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------------ tcgen05 building blocks
@pytest.mark.parametrize("d", [64, 128])
def test_debug_tile_mma_layouts(pb, d):
    g = torch.Generator(device="cpu").manual_seed(d)
    q = torch.randn(128, d, generator=g).bfloat16().cuda()
    k = torch.randn(64, d, generator=g).bfloat16().cuda()
    v = torch.randn(64, d, generator=g).bfloat16().cuda()
    s, o = pb.debug_tile(q, k, v)
    torch.cuda.synchronize()
    s_ref = q.float() @ k.float().T
    assert torch.allclose(s, s_ref, atol=1e-3, rtol=1e-4), (s - s_ref).abs().max()
    o_ref = s.bfloat16().float() @ v.float()
    assert torch.allclose(o, o_ref, atol=1e-2, rtol=1e-3), (o - o_ref).abs().max()


# ------------------------------------------------------------------ (a) compression
@pytest.mark.parametrize("d,b", [(128, 60), (64, 64), (128, 1), (64, 13)])
def test_compress_bitexact(pb, d, b):
    units, nb = 3, 11
    x = bf16_round(normal_bf16(100 + b, (units, nb, b, d)) * np.float32(3.0))
    x[1, 2] = 7.25  # identical tokens -> representative equals the token
    got = pb.compress_blocks(dev(x)).cpu().numpy()
    for u in range(units):
        want = orc.compress_blocks(x[u])
        assert np.array_equal(bits(got[u]), bits(want))
    assert np.all(got[1, 2] == 7.25)


# ------------------------------------------------------------------ (b) scoring + Top-K
def _score_case(pb, units, nqb, n_p, n_l, n_c, d, k, seed, ties=False, zero_q=False):
    g = np.random.default_rng(seed)
    n_slots = n_p + n_l + n_c + 5
    n_keys = n_p + n_l + n_c
    qc = (g.standard_normal((units, nqb, d)) * 0.5).astype(np.float32)
    if zero_q:
        qc[:] = 0
    krep = g.standard_normal((units, n_slots, d)).astype(np.float32)
    if ties:  # duplicated representatives -> exactly tied probabilities
        krep[:, 1::3] = krep[:, 0:1]
    keys = np.stack([g.permutation(n_slots)[:n_keys] for _ in range(units)]).astype(np.int32)
    sel, s_t = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                               n_p, n_l, k, want_scores=True)
    sel, s_t = sel.cpu().numpy(), s_t.cpu().numpy()
    for u in range(units):
        kc = krep[u][keys[u]]
        a_l = orc.coarse_attention(qc[u], kc[n_p:n_p + n_l])
        assert np.array_equal(sel[u], orc.select_topk(a_l, k)), f"unit {u}"
        want = orc.aggregate_scores(orc.coarse_attention(qc[u], kc))
        assert np.array_equal(bits(s_t[u]), bits(want)), f"unit {u}"
    # denoise pass (no scores): certified fp32 ranking, exact only near the k-th boundary
    sel2 = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                           n_p, n_l, k).cpu().numpy()
    assert np.array_equal(sel2, sel), "denoise-pass selection differs from the k=0 pass"
    return sel


@pytest.fixture(params=["1", "2", "0"], ids=["cert", "cert_fallback", "exact"])
def k2_mode(request, monkeypatch):
    """PBSA_K2_CERT: certified denoise path, the same with every row forced through the exact
    fallback, and the exact fp64 path on every pass."""
    monkeypatch.setenv("PBSA_K2_CERT", request.param)
    return request.param


@pytest.mark.parametrize("d", [64, 128])
def test_score_select_bitexact_small(pb, d, k2_mode):
    _score_case(pb, 3, 7, 8, 24, 8, d, 5, seed=d)


def test_score_select_bitexact_config2_shape(pb, k2_mode):
    _score_case(pb, 2, 78, 156, 312, 78, 128, 78, seed=7)


def test_score_select_ties_lower_index(pb, k2_mode):
    _score_case(pb, 2, 9, 4, 30, 4, 128, 7, seed=3, ties=True)
    sel = _score_case(pb, 1, 3, 2, 20, 2, 64, 6, seed=4, zero_q=True)  # uniform rows
    assert np.array_equal(sel[0], np.tile(np.arange(6), (3, 1)))


def test_score_select_k_equals_local(pb, k2_mode):
    _score_case(pb, 2, 5, 3, 9, 3, 128, 9, seed=11)


def test_score_select_large_window(pb, k2_mode):
    """config-5-like window (231 frames x 26 blocks) on a few rows."""
    _score_case(pb, 1, 4, 156, 6006, 78, 128, 1502, seed=12)


@pytest.mark.parametrize("scale_q", [40.0, 400.0])
def test_score_select_peaky_rows(pb, k2_mode, scale_q):
    """Very peaked rows: boundary probabilities underflow to zero (ties broken by index) -- the
    certified path must hand these rows to the exact fallback."""
    g = np.random.default_rng(21)
    units, nqb, n_p, n_l, n_c, d, k = 2, 11, 6, 200, 6, 128, 50
    n_keys, n_slots = n_p + n_l + n_c, n_p + n_l + n_c + 3
    qc = (g.standard_normal((units, nqb, d)) * scale_q).astype(np.float32)
    krep = g.standard_normal((units, n_slots, d)).astype(np.float32)
    keys = np.stack([g.permutation(n_slots)[:n_keys] for _ in range(units)]).astype(np.int32)
    sel = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                          n_p, n_l, k).cpu().numpy()
    for u in range(units):
        kc = krep[u][keys[u]]
        assert np.array_equal(sel[u], orc.select_topk(orc.coarse_attention(qc[u], kc[n_p:n_p + n_l]), k))


def test_score_select_cycled_keys(pb, k2_mode):
    """A window built from 3 cycled sets of key blocks (the shape of a cache filled by replaying
    three chunks): every logit appears many times, so the k-th boundary falls inside groups of
    exactly tied probabilities (lower index wins) next to near-tied ones."""
    g = np.random.default_rng(23)
    units, nqb, n_l, d, k, distinct = 2, 12, 2002, 128, 500, 77
    base = (g.standard_normal((units, distinct, d)) * 0.13).astype(np.float32)
    krep = np.concatenate([base[:, np.arange(n_l) % distinct], base[:, :3]], 1)
    qc = (g.standard_normal((units, nqb, d)) * 0.13).astype(np.float32)
    keys = np.stack([np.arange(n_l) for _ in range(units)]).astype(np.int32)
    sel = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                          0, n_l, k).cpu().numpy()
    for u in range(units):
        assert np.array_equal(sel[u], orc.select_topk(orc.coarse_attention(qc[u], krep[u][keys[u]]), k))


@pytest.mark.parametrize("d,n_l,k", [(64, 1030, 257), (128, 1027, 1), (128, 1500, 1500), (64, 9001, 2250)])
def test_score_select_long_window_defaults(pb, d, n_l, k):
    """Default dispatch (PBSA_K2_CERT unset): windows >= 1024 keys take the certified denoise path
    (odd lengths, k = 1, k = n), windows beyond its register capacity (9001 keys) the exact kernels."""
    g = np.random.default_rng(n_l + k)
    units, nqb, n_p, n_c = 2, 5, 7, 3
    n_keys, n_slots = n_p + n_l + n_c, n_p + n_l + n_c + 4
    qc = (g.standard_normal((units, nqb, d)) * 0.3).astype(np.float32)
    krep = g.standard_normal((units, n_slots, d)).astype(np.float32)
    keys = np.stack([g.permutation(n_slots)[:n_keys] for _ in range(units)]).astype(np.int32)
    sel = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                          n_p, n_l, k).cpu().numpy()
    for u in range(units):
        kc = krep[u][keys[u]]
        assert np.array_equal(sel[u], orc.select_topk(orc.coarse_attention(qc[u], kc[n_p:n_p + n_l]), k))


def test_score_select_near_ties(pb, k2_mode):
    """Representatives that differ in the last bits: exact logits a few ulps apart at the boundary
    (probabilities that may or may not tie in fp32) must be ranked exactly as the oracle does."""
    g = np.random.default_rng(22)
    units, nqb, n_p, n_l, n_c, d, k = 2, 16, 4, 96, 4, 64, 24
    n_keys, n_slots = n_p + n_l + n_c, n_p + n_l + n_c + 2
    qc = (g.standard_normal((units, nqb, d)) * 0.5).astype(np.float32)
    krep = g.standard_normal((units, n_slots, d)).astype(np.float32)
    base = krep[:, :1].copy()
    for t in range(1, n_slots, 2):  # every other key: the base row nudged by a few ulps
        nudge = (1.0 + np.float32(2.0 ** -23) * g.integers(-3, 4, size=d)).astype(np.float32)
        krep[:, t] = base[:, 0] * nudge
    keys = np.stack([g.permutation(n_slots)[:n_keys] for _ in range(units)]).astype(np.int32)
    sel = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                          n_p, n_l, k).cpu().numpy()
    for u in range(units):
        kc = krep[u][keys[u]]
        assert np.array_equal(sel[u], orc.select_topk(orc.coarse_attention(qc[u], kc[n_p:n_p + n_l]), k))


def test_score_select_long_path_rows_across_units(pb, k2_mode):
    """Long-window kernels (key-major logits, thread-per-row statistics): 39 rows of 3 units share
    warps; tied probabilities from duplicated representatives."""
    _score_case(pb, 3, 13, 40, 2100, 20, 64, 300, seed=13)
    _score_case(pb, 2, 5, 10, 2500, 10, 128, 77, seed=14, ties=True)


# ------------------------------------------------------------------ (c) block-sparse attention
def _bsa_case(pb, units, nqb, b, d, n_dense, n_local, k, seed, scale_q=1.0, stream_k=True, k_ramp=False):
    g = np.random.default_rng(seed)
    n_slots = n_dense + n_local + 3
    kp = np.zeros((units, n_slots, 64, d), np.float32)
    vp = np.zeros((units, n_slots, 64, d), np.float32)
    kp[:, :, :b] = normal_bf16(seed + 1, (units, n_slots, b, d))
    vp[:, :, :b] = normal_bf16(seed + 2, (units, n_slots, b, d))
    q = normal_bf16(seed + 3, (units, nqb * b, d)) * np.float32(scale_q)
    q = bf16_round(q)
    perm = np.stack([g.permutation(n_slots) for _ in range(units)]).astype(np.int32)
    if k_ramp:  # scores grow along the visiting order (x 2 every two dense blocks, exact in bf16)
        for u in range(units):
            for i in range(n_dense):
                kp[u, perm[u, i]] *= np.float32(2.0 ** (i // 2))
    dense = np.ascontiguousarray(perm[:, :n_dense])
    local = np.ascontiguousarray(perm[:, n_dense:n_dense + n_local])
    sel = np.stack([np.stack([np.sort(g.choice(n_local, k, replace=False)) for _ in range(nqb)])
                    for _ in range(units)]).astype(np.int32) if k else None
    o = pb.attention_sparse(dev(q), dev(kp), dev(vp), dev(dense, torch.int32) if n_dense else None,
                            dev(local, torch.int32) if n_local else None,
                            dev(sel, torch.int32) if k else None, b, stream_k=stream_k).float().cpu().numpy()
    for u in range(units):
        vis = [np.concatenate([dense[u], local[u][sel[u][i]] if k else np.zeros(0, np.int32)])
               for i in range(nqb)]
        want = orc.attention_sparse(q[u].reshape(nqb, b, d), kp[u][:, :b], vp[u][:, :b],
                                    np.stack(vis).astype(np.int32))
        check_attention(o[u].reshape(nqb, b, d), want)


@pytest.mark.parametrize("d,b", [(128, 60), (64, 64), (128, 64), (64, 60), (128, 17)])
@pytest.mark.parametrize("stream_k", [True, False])
def test_bsa_fwd_parity(pb, d, b, stream_k):
    _bsa_case(pb, 2, 5, b, d, 6, 16, 4, seed=d + b, stream_k=stream_k)


@pytest.mark.parametrize("units,nqb,n_dense,n_local,k", [(3, 7, 0, 9, 3), (2, 1, 5, 0, 0), (5, 9, 3, 40, 17),
                                                         (4, 6, 1, 7, 7), (1, 2, 0, 1, 1)])
def test_bsa_fwd_odd_lists(pb, units, nqb, n_dense, n_local, k):
    """Odd list lengths, single query blocks, no dense part, k = n_local, n_local = 1."""
    _bsa_case(pb, units, nqb, 60, 128, n_dense, n_local, k, seed=80 + units + nqb + n_local)
    _bsa_case(pb, units, nqb, 60, 128, n_dense, n_local, k, seed=90 + units, stream_k=False)


def test_bsa_fwd_stream_k_many_tiles(pb):
    """More tiles than CTA slots: whole tiles, split tiles and the partial merge all exercised;
    stream-K and whole-tile schedules must agree."""
    _bsa_case(pb, 40, 17, 60, 128, 10, 24, 6, seed=21)
    _bsa_case(pb, 40, 17, 60, 128, 10, 24, 6, seed=21, stream_k=False)


def test_bsa_fwd_growing_scores_rescale_path(pb):
    """Block maxima grow by up to 2^5 along the list: later blocks overflow the running-max fast
    path (row sums beyond the bound, or inf) and must take the exact rescale path."""
    _bsa_case(pb, 2, 6, 60, 128, 12, 24, 6, seed=31, k_ramp=True)
    _bsa_case(pb, 2, 6, 60, 128, 12, 24, 6, seed=32, k_ramp=True, scale_q=0.25)
    _bsa_case(pb, 1, 4, 64, 64, 10, 8, 3, seed=33, k_ramp=True)


def test_bsa_fwd_wide_pool_32bit_lists(pb):
    """>= 16384 pool slots: visible lists fall back to 32-bit entries."""
    _bsa_case(pb, 1, 4, 60, 128, 10, 16390, 8, seed=23)


def test_bsa_fwd_16bit_lists_config5_lengths(pb):
    """Config-5 list lengths (234 dense + the union of two 1502-of-6006 selections = ~2860-entry
    lists) over a pool < 16384 slots: K3 takes the 16-bit visible-list variant (two CTAs per SM)."""
    _bsa_case(pb, 1, 6, 60, 128, 234, 6006, 1502, seed=24)
    plan = pb.bsa_fwd_last_plan()
    assert plan.list_entry_bytes == 2 and plan.ctas_per_sm == 2, (plan.list_entry_bytes, plan.ctas_per_sm)
    _bsa_case(pb, 2, 3, 64, 64, 100, 3000, 3000, seed=25, stream_k=False)  # k = n_local: list = all
    plan = pb.bsa_fwd_last_plan()
    assert plan.list_entry_bytes == 2, plan.list_entry_bytes


def test_bsa_fwd_32bit_lists_selected(pb):
    """The same long lists over >= 16384 slots keep 32-bit entries (and a short list never uses 16)."""
    _bsa_case(pb, 1, 2, 60, 128, 234, 16200, 1502, seed=26)
    assert pb.bsa_fwd_last_plan().list_entry_bytes == 4
    _bsa_case(pb, 1, 4, 60, 128, 10, 30, 8, seed=27)
    assert pb.bsa_fwd_last_plan().list_entry_bytes == 4


@pytest.mark.parametrize("units,nqb", [(40, 17), (7, 78), (3, 5), (33, 78)])
def test_bsa_fwd_unit_gang_schedule(pb, monkeypatch, units, nqb):
    """Unit-gang schedule (PBSA_K3_GANG=1; the default for config-5-sized launches): gangs of
    tiles_per_unit CTAs walk units in lockstep behind an inter-CTA barrier.  Several rounds per
    gang, a partial last round, and back-to-back launches (the counters must re-zero)."""
    monkeypatch.setenv("PBSA_K3_GANG", "1")
    for rep in range(2):
        _bsa_case(pb, units, nqb, 60, 128, 7, 40, 9, seed=70 + units + rep)
        plan = pb.bsa_fwd_last_plan()
        assert plan.schedule == 2 and plan.gangs >= 1, (plan.schedule, plan.gangs)
        tpu = (nqb + 1) // 2
        if units > plan.gangs:  # the leftover slots form the extra gang (two tiles per member)
            assert plan.grid > plan.gangs * tpu, (plan.grid, plan.gangs, tpu)


@pytest.mark.parametrize("units,nqb", [(40, 17), (33, 78)])
def test_bsa_fwd_extra_gang_off(pb, monkeypatch, units, nqb):
    """PBSA_K3_EXTRA_GANG=0: the full gangs alone take every unit (the A/B baseline)."""
    monkeypatch.setenv("PBSA_K3_GANG", "1")
    monkeypatch.setenv("PBSA_K3_EXTRA_GANG", "0")
    _bsa_case(pb, units, nqb, 60, 128, 7, 40, 9, seed=90 + units)
    plan = pb.bsa_fwd_last_plan()
    assert plan.schedule == 2 and plan.grid == plan.gangs * ((nqb + 1) // 2)


@pytest.mark.parametrize("cap", [2, 4, 5, 8])
def test_bsa_fwd_split_tiles_parallel_merge(pb, monkeypatch, cap):
    """Few tiles, long lists: every tile is split into up to `cap` fragments (cap 5: fragment
    ranges cross tile boundaries, so CTAs hold two split tiles) and each fragment's CTA merges its
    slice of the tile's rows.  Back-to-back launches check that the tile counters (nf arrivals,
    then nf merges) re-zero."""
    monkeypatch.setenv("PBSA_K3_TAILCAP", str(cap))
    for rep in range(2):
        _bsa_case(pb, 2, 7, 60, 128, 30, 60, 20, seed=140 + cap + rep)
        plan = pb.bsa_fwd_last_plan()
        assert plan.schedule == 1, plan.schedule  # stream-K
        assert plan.grid <= cap * 8, (plan.grid, cap)


def test_bsa_fwd_hybrid_two_waves_and_tail(pb):
    """Two full waves of whole tiles (2 x 296 CTA slots on a B200) then a stream-K tail."""
    _bsa_case(pb, 70, 17, 60, 128, 5, 12, 3, seed=22)


def test_bsa_fwd_dense_only_and_full_local(pb):
    _bsa_case(pb, 2, 4, 60, 128, 9, 0, 0, seed=1)     # first chunk: no local window
    _bsa_case(pb, 1, 3, 60, 128, 0, 10, 10, seed=2)   # k = N_l (full visibility), no P
    _bsa_case(pb, 1, 1, 60, 64, 3, 5, 2, seed=3)      # single query block (half tile)


def test_bsa_fwd_peaky_inputs(pb):
    """Q x 4: larger logits exercise the lazy-rescale path (survey: 'peaky variant')."""
    _bsa_case(pb, 2, 6, 60, 128, 12, 24, 6, seed=5, scale_q=4.0)


def test_bsa_fwd_long_list(pb):
    _bsa_case(pb, 1, 4, 60, 128, 234, 312, 78, seed=9)


# ------------------------------------------------------------------ (d) memory + full calls
def run_rollout(pb, units, d, b, bpc, C, W, n_chunks, k_top, seed, denoise_steps=1, check_qb=None,
                attn_from_chunk=0, expect_plan=None):
    """Alg. 1 over n_chunks chunks, every PBSA call checked against the oracle (OracleReplay):
    Top-K indices, s_t and P / L ids bit-exact on every call; attention (sampled query blocks
    `check_qb`, from chunk `attn_from_chunk` on) within the bf16 tolerance.  expect_plan: dict of
    pbsa_bsa_plan fields the K3 launch of every attention-checked call must have."""
    mem = pb.Memory(units, C, W, bpc, b, d)
    rep = OracleReplay(units, C, W, bpc, b, d)
    stats = []
    for c in range(n_chunks):
        for step in range(denoise_steps + 1):
            update = step == denoise_steps
            base = seed * 1000003 + c * 17 + step
            q = normal_bf16(base, (units, bpc * b, d))
            kc = normal_bf16(base + 7, (units, bpc * b, d))
            vc = normal_bf16(base + 13, (units, bpc * b, d))
            mode = pb.MODE_CACHE_UPDATE if update else pb.MODE_DENOISE
            if (c + step) % 2:  # both entry points: fused ingest and write_chunk + attend
                o = mem.attend_qkv(dev(q), dev(kc), dev(vc), k_top, mode)
            else:
                mem.write_chunk(dev(kc), dev(vc))
                o = mem.attend(dev(q), k_top, mode)
            check_attn = c >= attn_from_chunk
            if check_attn and expect_plan:
                plan = pb.bsa_fwd_last_plan()
                for key, want in expect_plan.items():
                    assert getattr(plan, key) == want, f"K3 plan {key} = {getattr(plan, key)}, expected {want}"
            sel_gpu, st_gpu = mem.last_selection()
            stats += rep.call(q, kc, vc, k_top, update, o=o.float().cpu().numpy() if check_attn else None,
                              sel=None if sel_gpu is None else sel_gpu.cpu().numpy(),
                              s_t=None if st_gpu is None else st_gpu.cpu().numpy(), check_qb=check_qb,
                              where=f"chunk {c} step {step}")
        # after the k=0 pass: P and L block ids bit-exact (SPEC.md:209-217 order)
        gp, gl = mem.assemble()
        rep.check_ids(gp.cpu().numpy(), gl.cpu().numpy(), where=f"chunk {c}")
    assert mem.status() == 0  # no NaN rows, no certified-bound canary (bit 2)
    mem.close()
    return stats


@pytest.mark.parametrize("d", [64, 128])
def test_rollout_small(pb, d):
    # 6-block chunks, P = 2 chunks (one of sinks), window 2 chunks, 8 chunks -> 5 evictions
    run_rollout(pb, units=3, d=d, b=60, bpc=6, C=12, W=2, n_chunks=8, k_top=3, seed=d)


@pytest.mark.parametrize("bpc,d", [(6, 128), (7, 128), (7, 64)])
def test_rollout_with_tile_pairing(pb, bpc, d, monkeypatch):
    """The K3 tile pairing forced on for short windows (auto mode pairs >= 1024-block windows only):
    every call of the rollout still replays bit-exactly (Top-K, s_t, P / L) and within tolerance
    (attention) through the oracle -- outputs do not depend on which query blocks share a tile."""
    monkeypatch.setenv("PBSA_TILE_PAIRING", "1")
    run_rollout(pb, units=3, d=d, b=60, bpc=bpc, C=12, W=2, n_chunks=6, k_top=3, seed=40 + bpc + d,
                denoise_steps=2)


def test_rollout_config1(pb):
    """Config 1 (BASELINE.json): d=64, b=64 = (1,8,8) on 16x16 frames (4 blocks/frame), 2-frame
    chunks (8 query blocks), P = 2 frames (the sink chunk), L = 4 frames, top-k 8."""
    run_rollout(pb, units=1, d=64, b=64, bpc=8, C=8, W=2, n_chunks=6, k_top=8, seed=1, denoise_steps=2)


def test_rollout_config2_full_size(pb):
    """Config 2 (Wan-1.3B layer): 12 heads, d=128, 60-token blocks, 78 blocks per 3-frame chunk,
    P = 6 frames (156), L = 12 frames (312), top-k 78.  7 chunks reach steady state (sinks +
    a full dynamic set + evictions); indices and ids checked everywhere, attention on sampled
    query blocks."""
    run_rollout(pb, units=12, d=128, b=60, bpc=78, C=156, W=4, n_chunks=7, k_top=78, seed=2,
                denoise_steps=0, check_qb=np.array([0, 1, 40, 77]))


def test_rollout_config5_window_steady_state(pb):
    """Config-5 geometry per unit (BASELINE.json config 5: 240-frame cache = P 6 + L 231 + current 3
    frames of 26 blocks, k = 25 % of the window = 1502) on 2 units, brought to steady state (81
    chunks: the 6006-block window full, P full of sinks + dynamic blocks, evictions every chunk).
    Every call: Top-K indices (exact long-window K2 on the k=0 pass, certified K2 on the denoise
    pass), s_t over all 6396 keys and P / L ids bit-exact; over the last chunks K3 runs with 16-bit
    visible-list entries (3238-entry lists) and its output is checked on sampled query blocks."""
    run_rollout(pb, units=2, d=128, b=60, bpc=78, C=156, W=77, n_chunks=81, k_top=1502, seed=55,
                denoise_steps=1, check_qb=np.array([0, 1, 77]), attn_from_chunk=79,
                expect_plan={"list_entry_bytes": 2, "ctas_per_sm": 2})


def test_errors_are_loud(pb):
    with pytest.raises(pb.PbsaError):
        pb.Memory(1, 4, 1, 8, 60, 128)  # C < blocks_per_chunk
    with pytest.raises(pb.PbsaError):
        pb.Memory(1, 8, 1, 8, 60, 96)  # unsupported head dim
    q = torch.zeros(1, 60, 128, dtype=torch.bfloat16, device="cuda")
    kp = torch.zeros(1, 4, 64, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(pb.PbsaError):
        pb.attention_sparse(q, kp, kp, None, None, None, 61)


# ------------------------------------------------------------------ chunk latents (blockify fused)
def _latent_vs_blocked(pb, batch, heads, d, T, H, W, blk, C, Wc, n_chunks, k_top, seed):
    """attend_latent on raw Latent4D chunks == attend_qkv on the oracle-blockified per-head
    tensors (blockify.cpp:38-65 restated, pinned to the reference): outputs bit-identical after
    unblockify, selections and memory ids identical."""
    g = np.random.default_rng(seed)
    nqb, b = pb.latent_blocks((batch, T, H, W, heads * d), heads, d, blk)
    U = batch * heads
    ma = pb.Memory(U, C, Wc, nqb, b, d)
    mb = pb.Memory(U, C, Wc, nqb, b, d)

    def blocked(lat):  # [batch, T, H, W, heads*d] -> [U, nqb*b, d] (unit = e*heads + h)
        out = []
        for e in range(batch):
            xb = orc.blockify(lat[e], blk)                       # [nqb, b, heads*d]
            for h in range(heads):
                out.append(xb[:, :, h * d:(h + 1) * d].reshape(nqb * b, d))
        return np.stack(out)

    def unblocked(ob):  # [U, nqb*b, d] -> [batch, T, H, W, heads*d]
        lat = np.zeros((batch, T, H, W, heads * d), np.float32)
        for e in range(batch):
            xb = np.concatenate([ob[e * heads + h].reshape(nqb, b, d) for h in range(heads)], axis=2)
            lat[e] = orc.unblockify(xb, (T, H, W, heads * d), blk)
        return lat

    for c in range(n_chunks):
        for mode in (pb.MODE_DENOISE, pb.MODE_CACHE_UPDATE):
            lat = [bf16_round(g.standard_normal((batch, T, H, W, heads * d)).astype(np.float32)) for _ in range(3)]
            ob = ma.attend_qkv(*(dev(blocked(x)) for x in lat), k_top, mode)
            ol = mb.attend_latent(*(dev(x) for x in lat), blk, k_top, mode)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(unblocked(ob.float().cpu().numpy()), ol.float().cpu().numpy())
            sa, sb = ma.last_selection()[0], mb.last_selection()[0]
            assert (sa is None) == (sb is None)
            if sa is not None:
                assert torch.equal(sa, sb)
        pa, la = ma.assemble()
        pbb, lb = mb.assemble()
        assert torch.equal(pa, pbb) and torch.equal(la, lb)
    ma.close()
    mb.close()


def test_attend_latent_matches_blocked_small(pb):
    _latent_vs_blocked(pb, batch=2, heads=2, d=128, T=2, H=6, W=8, blk=(1, 3, 4), C=16, Wc=2, n_chunks=4,
                       k_top=3, seed=41)


def test_attend_latent_matches_blocked_wan_blocks(pb):
    """(1, 15, 4) = 60-token blocks of the Wan-1.3B layout, d = 64 variant with 3-frame chunks."""
    _latent_vs_blocked(pb, batch=1, heads=3, d=64, T=3, H=30, W=8, blk=(1, 15, 4), C=24, Wc=2, n_chunks=4,
                       k_top=4, seed=42)


# ------------------------------------------------------------------ (c') backward
def _bsa_bwd_case(pb, units, nqb, b, d, n_dense, n_local, k, seed, report=False):
    g = np.random.default_rng(seed)
    n_slots = n_dense + n_local + 3
    kp = np.zeros((units, n_slots, 64, d), np.float32)
    vp = np.zeros((units, n_slots, 64, d), np.float32)
    kp[:, :, :b] = normal_bf16(seed + 1, (units, n_slots, b, d))
    vp[:, :, :b] = normal_bf16(seed + 2, (units, n_slots, b, d))
    q = normal_bf16(seed + 3, (units, nqb * b, d))
    do = normal_bf16(seed + 4, (units, nqb * b, d))
    perm = np.stack([g.permutation(n_slots) for _ in range(units)]).astype(np.int32)
    dense = np.ascontiguousarray(perm[:, :n_dense])
    local = np.ascontiguousarray(perm[:, n_dense:n_dense + n_local])
    sel = np.stack([np.stack([np.sort(g.choice(n_local, k, replace=False)) for _ in range(nqb)])
                    for _ in range(units)]).astype(np.int32) if k else None
    args = (dev(q), dev(kp), dev(vp), dev(dense, torch.int32) if n_dense else None,
            dev(local, torch.int32) if n_local else None, dev(sel, torch.int32) if k else None, b)
    o, lse = pb.attention_sparse(*args, want_lse=True)
    dq, dk, dv = pb.attention_sparse_backward(*args, o, lse, dev(do))
    torch.cuda.synchronize()
    dq, dk, dv = dq.cpu().numpy(), dk.cpu().numpy(), dv.cpu().numpy()
    worst = 0.0
    for u in range(units):
        vis = np.stack([np.concatenate([dense[u], local[u][sel[u][i]] if k else np.zeros(0, np.int32)])
                        for i in range(nqb)]).astype(np.int32)
        rq, rk, rv = orc.attention_sparse_backward(q[u].reshape(nqb, b, d), kp[u][:, :b], vp[u][:, :b], vis,
                                                    do[u].reshape(nqb, b, d))
        for name, got, want in (("dq", dq[u].reshape(nqb, b, d), rq), ("dk", dk[u][:, :b], rk), ("dv", dv[u][:, :b], rv)):
            err = np.abs(got - want)
            ref = max(np.abs(want).max(), 1e-6)
            worst = max(worst, err.max() / ref)
            if report:
                print(name, u, "max", err.max() / ref, "mean", err.mean() / ref)
            # bf16 operands (Q, K, V, dO, P, dS) with fp32 accumulation vs an fp64 oracle
            assert err.max() <= 1e-2 * ref and err.mean() <= 1e-3 * ref, (name, u, err.max(), err.mean(), ref)
    return worst


@pytest.mark.parametrize("d,b", [(128, 60), (64, 64), (128, 17)])
def test_bsa_bwd_parity(pb, d, b):
    _bsa_bwd_case(pb, 2, 5, b, d, 6, 16, 4, seed=50 + d + b)


def test_bsa_bwd_dense_only_and_odd_pairs(pb):
    _bsa_bwd_case(pb, 2, 4, 60, 128, 7, 0, 0, seed=61)     # no local window, odd dense count
    _bsa_bwd_case(pb, 1, 3, 60, 128, 5, 9, 9, seed=62)     # k = N_l, odd local count


def test_attend_qkv_host_pipelined_matches_device(pb):
    """pbsa_attend_qkv_host (pinned host chunks, upload / compute / download pipelined over two
    staging sets) gives bit-identical outputs to pbsa_attend_qkv on device copies of the same
    chunks, across denoise and cache-update calls."""
    U, C, W, bpc, b, d, k = 3, 12, 2, 6, 60, 128, 3
    m1, m2 = pb.Memory(U, C, W, bpc, b, d), pb.Memory(U, C, W, bpc, b, d)
    g = torch.Generator().manual_seed(31)
    keep, got = [], []
    for c in range(7):
        for step in range(3):
            mode = pb.MODE_CACHE_UPDATE if step == 2 else pb.MODE_DENOISE
            q, kk, vv = (torch.randn(U, bpc * b, d, generator=g).bfloat16().pin_memory() for _ in range(3))
            o1 = m1.attend_qkv(q.cuda(), kk.cuda(), vv.cuda(), k, mode).cpu()
            o2 = m2.attend_qkv_host(q, kk, vv, k, mode)
            keep.append((q, kk, vv))
            got.append((o1, o2))
    m2.host_sync()
    torch.cuda.synchronize()
    for i, (o1, o2) in enumerate(got):
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16)), f"call {i}"
    with pytest.raises(pb.PbsaError):
        m2.attend_qkv_host(keep[0][0].cuda(), keep[0][1], keep[0][2], k)  # device tensor: rejected
    m1.close()
    m2.close()


def test_score_select_certified_fuzz(pb):
    """Certified denoise selection (default dispatch, windows >= 1024 keys) on randomised windows,
    Top-K sizes, logit scales (flat to peaky), duplicated and near-duplicated keys: the indices must
    be the oracle's exactly."""
    g = np.random.default_rng(2024)
    for trial in range(24):
        d = int(g.choice([64, 128]))
        n_l = int(g.integers(1024, 2600))
        k = int(g.integers(1, n_l + 1)) if trial % 3 else int(g.integers(1, 40))
        units, nqb, n_p = 1, int(g.integers(1, 6)), int(g.integers(0, 9))
        n_slots = n_p + n_l + 2
        scale_q = float(10.0 ** g.uniform(-2.5, 1.3))
        qc = (g.standard_normal((units, nqb, d)) * scale_q).astype(np.float32)
        krep = g.standard_normal((units, n_slots, d)).astype(np.float32)
        if trial % 4 == 1:  # exact duplicates
            krep[:, 1::5] = krep[:, 0:1]
        if trial % 4 == 2:  # near duplicates (last-bit nudges)
            krep[:, 1::7] = krep[:, 0:1] * (1.0 + np.float32(2.0 ** -23) * g.integers(-2, 3, size=(1, 1, d)))
        keys = np.stack([g.permutation(n_slots)[:n_p + n_l] for _ in range(units)]).astype(np.int32)
        sel = pb.score_select(dev(qc, torch.float32), dev(krep, torch.float32), dev(keys, torch.int32),
                              n_p, n_l, k).cpu().numpy()
        for u in range(units):
            kc = krep[u][keys[u]]
            want = orc.select_topk(orc.coarse_attention(qc[u], kc[n_p:n_p + n_l]), k)
            assert np.array_equal(sel[u], want), f"trial {trial}: d={d} n={n_l} k={k} scale={scale_q:.3g}"


def test_launch_counter_per_call(pb):
    """pbsa_launch_count: a denoise call at a short window launches ingest + K2 logits + K2 select
    + K3 (4 kernels; no tile pairing below 1024 window blocks); a cache-update call adds the A_t
    aggregation and K4 (6) -- the bench reports this counter's delta over its timed region as
    gpu_launches."""
    from paper_2604_21221_b200._capi import LIB
    U, C, W, bpc, b, d = 2, 12, 2, 6, 60, 128
    mem = pb.Memory(U, C, W, bpc, b, d)
    g = torch.Generator(device="cuda").manual_seed(5)
    for _ in range(W + 3):  # fill to steady state
        q, kk, vv = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
        mem.attend_qkv(q, kk, vv, 3, pb.MODE_CACHE_UPDATE)
    torch.cuda.synchronize()
    n0 = LIB.pbsa_launch_count()
    mem.attend_qkv(q, kk, vv, 3, pb.MODE_DENOISE)
    n1 = LIB.pbsa_launch_count()
    mem.attend_qkv(q, kk, vv, 3, pb.MODE_CACHE_UPDATE)
    n2 = LIB.pbsa_launch_count()
    torch.cuda.synchronize()
    assert (n1 - n0, n2 - n1) == (4, 6)
    mem.close()


def _pairing_reference(sel_u):
    """The pairing rule of pair_tiles_kernel restated: greedy matching -- repeatedly the free pair
    (i < j) with the largest Top-K overlap, ties to the lowest i * nq + j, in that order -- then the
    bottleneck pass; an odd leftover last with -1."""
    nq = len(sel_u)
    sets = [set(r) for r in sel_u]
    keys = sorted(((len(sets[i] & sets[j]), -(i * nq + j), i, j) for i in range(nq) for j in range(i + 1, nq)),
                  reverse=True)
    free = [True] * nq
    out = []
    for _, _, i, j in keys:
        if free[i] and free[j]:
            free[i] = free[j] = False
            out.append((i, j))
    # bottleneck pass: swap partners between the least-overlapping tile and another while both new
    # tiles overlap more (best new minimum, then sum, then lowest (s, option))
    ovm = [[len(sets[i] & sets[j]) for j in range(nq)] for i in range(nq)]
    for _ in range(nq if out else 0):
        t = min(range(len(out)), key=lambda t2: (ovm[out[t2][0]][out[t2][1]], t2))
        a, b = out[t]
        cur = ovm[a][b]
        best = None
        for s2, (c, d2) in enumerate(out):
            if s2 == t:
                continue
            for opt in (0, 1):
                x1, x2 = ovm[a][d2 if opt else c], ovm[b][c if opt else d2]
                if min(x1, x2) <= cur:
                    continue
                key = (min(x1, x2), x1 + x2, -(2 * s2 + opt))
                if best is None or key > best[0]:
                    best = (key, s2, opt)
        if best is None:
            break
        _, s2, opt = best
        c, d2 = out[s2]
        n1, n2 = (d2, c) if opt else (c, d2)
        out[t] = (min(a, n1), max(a, n1))
        out[s2] = (min(b, n2), max(b, n2))
    out += [(i, -1) for i in range(nq) if free[i]]
    return out


@pytest.mark.parametrize("units,nq,n_local,k", [(3, 7, 40, 9), (2, 78, 312, 78), (2, 78, 6006, 1502),
                                                 (1, 1, 10, 3), (2, 5, 64, 64)])
def test_pair_tiles_kernel_matches_rule(pb, units, nq, n_local, k):
    """pbsa_pair_tiles on random selections (config-2 and config-5 shapes included) equals the
    restated greedy + bottleneck rule."""
    g = torch.Generator(device="cuda").manual_seed(nq * 7 + k)
    sel = torch.stack([torch.stack([torch.randperm(n_local, device="cuda", generator=g)[:k].sort().values
                                    for _ in range(nq)]) for _ in range(units)]).int().contiguous()
    pr = pb.pair_tiles(sel, n_local).cpu().tolist()
    sl = sel.cpu().tolist()
    for u in range(units):
        assert [tuple(x) for x in pr[u]] == _pairing_reference(sl[u])


@pytest.mark.parametrize("bpc", [6, 7])
def test_tile_pairing_rule_and_partition(pb, bpc, monkeypatch):
    monkeypatch.setenv("PBSA_TILE_PAIRING", "1")
    """K3 tiles pair each call's query blocks by Top-K overlap (pair_tiles_kernel): the device
    pairing equals the restated greedy + bottleneck rule and covers every query block exactly once
    (odd counts: one single-block tile).  PBSA_TILE_PAIRING=1
    forces it for these short windows (auto mode pairs windows of >= 1024 blocks only)."""
    U, C, W, b, d, k_top = 3, 12, 4, 60, 128, 5
    mem = pb.Memory(U, C, W, bpc, b, d)
    g = torch.Generator(device="cuda").manual_seed(11)
    for c in range(W + 3):
        q, kk, vv = (torch.randn(U, bpc * b, d, device="cuda", generator=g).bfloat16() for _ in range(3))
        mem.attend_qkv(q, kk, vv, k_top, pb.MODE_CACHE_UPDATE if c % 2 else pb.MODE_DENOISE)
        pairs = mem.last_tile_pairs()
        sel, _ = mem.last_selection()
        if sel is None:  # empty window (first chunk): no selection, natural pairs
            assert pairs is None
            continue
        assert pairs is not None
        pr, sl = pairs.cpu().tolist(), sel.cpu().tolist()
        for u in range(U):
            got = [tuple(x) for x in pr[u]]
            assert got == _pairing_reference(sl[u])
            flat = sorted(x for t in got for x in t if x >= 0)
            assert flat == list(range(bpc))
    mem.close()


# ------------------------------------------------------------------ query-split multi-GPU layout
@pytest.mark.parametrize("replicas", [2, 3])
def test_query_split_replicas_commit_identical_memory(pb, replicas):
    """SURVEY 8(e) batch-1 layout simulated on one GPU: R replicas of the same heads, each attending
    its range of query blocks (pbsa_attend_part_ingest / pbsa_attend_part), Q^c gathered between
    them at the k=0 pass.  Every replica must commit the identical P / L ids and s_t, its Top-K rows
    must equal the full-chunk call's, and the stitched outputs must pass the oracle replay."""
    from paper_2604_21221_b200.parallel import QuerySplitLayout
    U, C, W, bpc, b, d, k_top = 3, 12, 2, 7, 60, 128, 3
    ranges = [partition_units_(bpc, replicas, r) for r in range(replicas)]
    lay = QuerySplitLayout(12, bpc, 8, 1)  # the config-2 N=8 layout: 4 groups of 3 heads, 2 replicas
    assert (lay.groups, lay.replicas, lay.n_local) == (4, 2, 3)
    full = pb.Memory(U, C, W, bpc, b, d)
    parts = [pb.Memory(U, C, W, bpc, b, d) for _ in range(replicas)]
    rep = OracleReplay(U, C, W, bpc, b, d)
    for c in range(7):
        for step in range(3):
            update = step == 2
            mode = pb.MODE_CACHE_UPDATE if update else pb.MODE_DENOISE
            base = 900 + c * 17 + step
            q = normal_bf16(base, (U, bpc * b, d))
            kc = normal_bf16(base + 7, (U, bpc * b, d))
            vc = normal_bf16(base + 13, (U, bpc * b, d))
            o_full = full.attend_qkv(dev(q), dev(kc), dev(vc), k_top, mode)
            sel_full, st_full = full.last_selection()
            qcs = [torch.zeros(U, bpc, d, device="cuda") for _ in range(replicas)]
            q_parts = [dev(q.reshape(U, bpc, b, d)[:, qb:qb + qn].reshape(U, qn * b, d)) for qb, qn in ranges]
            for r, (qb, qn) in enumerate(ranges):
                parts[r].attend_part_ingest(q_parts[r], qb, dev(kc), dev(vc), qcs[r])
            if update:  # the group all-gather of Q^c, by hand
                for r, (qb, qn) in enumerate(ranges):
                    for r2 in range(replicas):
                        qcs[r2][:, qb:qb + qn] = qcs[r][:, qb:qb + qn]
            o = torch.empty(U, bpc * b, d, dtype=torch.bfloat16, device="cuda")
            for r, (qb, qn) in enumerate(ranges):
                o[:, qb * b:(qb + qn) * b] = parts[r].attend_part(q_parts[r], qb, qcs[r], k_top, mode)
                sel_r, st_r = parts[r].last_selection()
                if sel_full is not None:
                    want = sel_full[:, qb:qb + qn] if not update else sel_full
                    assert torch.equal(sel_r, want), f"chunk {c} step {step} replica {r}: Top-K rows"
                if update:
                    assert torch.equal(st_r, st_full), f"chunk {c} replica {r}: s_t"
            torch.cuda.synchronize()
            rep.call(q, kc, vc, k_top, update, o=o.float().cpu().numpy(),
                     sel=None if sel_full is None else sel_full.cpu().numpy(),
                     s_t=None if st_full is None else st_full.cpu().numpy(), where=f"chunk {c} step {step}")
            # the stitched query-split output against the full-chunk call (same kernel, different
            # stream-K splits: bf16-rounding-level differences at most)
            assert (o.float() - o_full.float()).abs().max().item() <= 1e-2
        gp, gl = full.assemble()
        rep.check_ids(gp.cpu().numpy(), gl.cpu().numpy(), where=f"chunk {c}")
        for r in range(replicas):
            pp, pl = parts[r].assemble()
            assert torch.equal(pp, gp) and torch.equal(pl, gl), f"chunk {c} replica {r}: P / L ids"
    for m in [full] + parts:
        m.close()


def partition_units_(total, world, rank):
    from paper_2604_21221_b200.parallel import partition_units
    return partition_units(total, world, rank)
