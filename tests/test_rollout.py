"""Alg. 1 rollout driver: trace invariants (SPEC.md:484-488,
acceptance 6), determinism, and the blockify used by the driver vs the oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2604_21221_b200 import rollout as ro
from tests.pbsa_oracle_compose import OracleReplay


def small_cfg(**kw):
    base = dict(num_chunks=6, timesteps=(1.0, 0.5), topk_ratio=0.25, capacity_frames=4, window_frames=4,
                chunk_frames=2, height=8, width=8, block_shape=(1, 4, 4), layers=2, heads=2, head_dim=128,
                seed=3, trace_units=2)
    base.update(kw)
    return ro.RolloutConfig(**base)


def test_blockify_tokens_matches_reference_layout():
    g = np.random.default_rng(0)
    for dims, shp in [((3, 30, 52, 4), (1, 15, 4)), ((2, 8, 8, 3), (1, 4, 4)), ((4, 6, 6, 2), (2, 3, 2))]:
        x = g.standard_normal(dims).astype(np.float32)
        want = orc.blockify(x, shp).reshape(-1, dims[3])
        got = ro.blockify_tokens(torch.from_numpy(x), shp).numpy()
        assert np.array_equal(got, want)
        back = ro.unblockify_tokens(torch.from_numpy(want), dims, shp).numpy()
        assert np.array_equal(back, x)


def test_config_validation_and_renoise():
    with pytest.raises(ValueError):
        small_cfg(timesteps=(0.5, 0.5)).validate()
    with pytest.raises(ValueError):
        small_cfg(height=9).validate()
    x0, eps = torch.full((2,), 2.0), torch.zeros(2)
    assert torch.equal(ro.renoise(x0, eps, 0.5), torch.ones(2))
    assert torch.equal(ro.renoise(x0, eps, 1.0), eps)


def test_check_trace_rejects_violations():
    cfg = small_cfg(num_chunks=2, timesteps=(1.0,))
    good = [{"chunk": 0, "j": 1, "cache_updated": True, "persistent": [[]], "window": [[0, 1]], "evicted": [[]]},
            {"chunk": 1, "j": 1, "cache_updated": True, "persistent": [[]], "window": [[0, 1, 2]], "evicted": [[]]}]
    ro.check_trace(cfg, good)
    bad = [dict(good[0]), dict(good[1], persistent=[[2]])]
    with pytest.raises(AssertionError):
        ro.check_trace(cfg, bad)


@pytest.mark.gpu
def test_rollout_trace_invariants_and_determinism():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = small_cfg()
    frames, trace, timing = ro.run_inference(cfg)
    ro.check_trace(cfg, trace)
    assert len(frames) == cfg.num_chunks
    assert timing["pbsa_calls"] == cfg.num_chunks * (len(cfg.timesteps) + 1) * cfg.layers  # + the k=0 pass
    upd = [r for r in trace if r["cache_updated"]]
    # C = 4 frames = 8 blocks (sinks = first chunk of 8), window 2 chunks: first eviction at push 3
    assert [len(r["evicted"][0]) for r in upd[:3]] == [0, 0, 8]
    assert upd[-1]["persistent"][0][:8] == list(range(8))  # sinks retained
    frames2, trace2, _ = ro.run_inference(cfg)
    assert trace2 == trace  # bit-identical traces (scores included)
    for a, b in zip(frames, frames2):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_rollout_latent_path_equals_blocked_path():
    """The driver on chunk latents (pbsa_attend_latent: blockify / unblockify inside the kernels)
    and on torch-blockified per-head tensors (pbsa_attend_qkv) produce identical traces and frames."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    fa, ta, _ = ro.run_inference(small_cfg(latent=True))
    fb, tb, _ = ro.run_inference(small_cfg(latent=False))
    assert ta == tb
    for a, b in zip(fa, fb):
        assert torch.equal(a, b)


def replay(cfg, capture, units=None, check_qb=None):
    """Replay the layer-0 PBSA calls a rollout captured through the oracle: per call
    Top-K indices, s_t and P / L ids bit-exact, attention output within the bf16 tolerance."""
    units = cfg.heads if units is None else units
    rep = OracleReplay(units, cfg.capacity_blocks, cfg.window_chunks, cfg.blocks_per_chunk, cfg.b, cfg.head_dim)
    stats = []
    for i, c in enumerate(capture):
        upd = c["mode"] == 1
        stats += rep.call(c["q"][:units].numpy(), c["k"][:units].numpy(), c["v"][:units].numpy(), c["k_top"], upd,
                          o=c["o"][:units].numpy(), sel=None if c["sel"] is None else c["sel"][:units].numpy(),
                          s_t=None if c["s_t"] is None else c["s_t"][:units].numpy(), check_qb=check_qb,
                          where=f"call {i}")
        rep.check_ids(c["persistent"][:units].numpy(), c["window"][:units].numpy(), where=f"call {i}")
    return stats


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("latent", [True, False])
def test_rollout_replays_through_oracle(latent):
    """Every layer-0 PBSA call of a rollout (denoise and k=0 passes, 7 chunks: sinks, dynamic
    blocks and evictions) replayed through the oracle on the captured inputs."""
    _need_gpu()
    cfg = small_cfg(num_chunks=7, latent=latent)
    cap = []
    ro.run_inference(cfg, capture=cap)
    assert len(cap) == cfg.num_chunks * (len(cfg.timesteps) + 1)
    stats = replay(cfg, cap)
    assert stats and max(s[0] for s in stats) <= 2e-2


@pytest.mark.gpu
def test_rollout_wan_layout_replays_through_oracle():
    """The Wan-1.3B layer layout (30x52 latent frames, (1,15,4) blocks, 12 heads, 3-frame chunks,
    C = 6 frames, window 6 frames, Top-K 25 %) over 5 chunks: 3 heads replayed, attention on sampled
    query blocks."""
    _need_gpu()
    cfg = ro.RolloutConfig(num_chunks=5, timesteps=(1.0, 0.5), layers=1, trace_units=12)
    cap = []
    _, trace, _ = ro.run_inference(cfg, capture=cap)
    ro.check_trace(cfg, trace)
    replay(cfg, cap, units=3, check_qb=np.array([0, 31, 77]))


@pytest.mark.gpu
@pytest.mark.parametrize("M", [1, 4, 12])
@pytest.mark.parametrize("T", [1, 4])
def test_acceptance6_trace_invariants(M, T, tmp_path):
    """SPEC.md:664 acceptance 6: for M in {1,4,12}, T in {1,4}: M*T denoise records (plus the k=0
    pass of each chunk on the device), M cache updates each at j=1, |P| <= C and |window| <= L_local
    at every record, eviction ids strictly increasing, byte-identical reruns."""
    _need_gpu()
    ts = tuple(1.0 - i / T for i in range(T))
    cfg = small_cfg(num_chunks=M, timesteps=ts, trace_units=2)
    outs = []
    for rep in range(2):
        path = tmp_path / f"trace{rep}.jsonl"
        frames, trace, timing = ro.run_inference(cfg, trace_path=str(path))
        ro.check_trace(cfg, trace)
        assert len(trace) == M * T
        assert sum(r["cache_updated"] for r in trace) == M
        assert all(r["j"] == 1 for r in trace if r["cache_updated"])
        assert timing["pbsa_calls"] == M * (T + 1) * cfg.layers
        outs.append((path.read_bytes(), frames))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_fault_drop_sink_is_caught():
    """Negative control (SPEC.md:625 `verify --fault drop-sink`): with K4's sink retention broken
    the oracle replay's bit-exact P check and the trace's sink-retention invariant both fail."""
    _need_gpu()
    import paper_2604_21221_b200 as pb
    cfg = small_cfg(num_chunks=7, trace_units=2)
    cap = []
    pb.debug_set_fault("drop-sink")
    try:
        _, trace, _ = ro.run_inference(cfg, capture=cap)
    finally:
        pb.debug_set_fault(None)
    with pytest.raises(AssertionError, match="sink retention"):
        ro.check_trace(cfg, trace)
    with pytest.raises(AssertionError, match="persistent ids|Top-K|s_t"):
        replay(cfg, cap)
    # and without the fault the same rollout passes both
    cap = []
    _, trace, _ = ro.run_inference(cfg, capture=cap)
    ro.check_trace(cfg, trace)
    replay(cfg, cap)
