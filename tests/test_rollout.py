"""Alg. 1 rollout driver: trace invariants (SPEC.md:484-488,
acceptance 6), determinism, and the blockify used by the driver vs the oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2604_21221_b200 import rollout as ro


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
