"""GPU parity of the reference's tensor / blockify primitives and the SPEC router / memory ops
(pbsa_matmul, pbsa_masked_softmax_rows, pbsa_aggregate_scores, pbsa_select_topk, pbsa_blockify,
pbsa_topc_select, pbsa_compress_f32) against the oracle, which is itself pinned bit-exactly to the
reference's compiled tensor.cpp / blockify.cpp (tests/test_oracle_vs_ref.py).  Bar: bit-exact."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_21221_b200 as pb
    return pb


def dev(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("n,k,m", [(1, 1, 1), (7, 128, 33), (78, 128, 546), (65, 300, 17), (0, 4, 3)])
def test_matmul_bitexact(pb, n, k, m):
    g = np.random.default_rng(n * 1000 + m)
    a = g.standard_normal((n, k)).astype(np.float32)
    b = (g.standard_normal((k, m)) * 3).astype(np.float32)
    bt = (g.standard_normal((m, k)) * 0.5).astype(np.float32)
    assert np.array_equal(bits(pb.matmul(dev(a), dev(b)).cpu().numpy()), bits(orc.matmul(a, b)))
    assert np.array_equal(bits(pb.matmul(dev(a), dev(bt), transpose_b=True).cpu().numpy()), bits(orc.matmul_nt(a, bt)))
    # the coarse logits: float(dot64) * fp32 scale (DESIGN.md pinned semantics i)
    sc = orc.attention_scale(k)
    want = orc.matmul_nt(a, bt) * np.float32(sc)
    assert np.array_equal(bits(pb.matmul(dev(a), dev(bt), True, sc).cpu().numpy()), bits(want))


@pytest.mark.parametrize("rows,cols", [(1, 1), (78, 312), (13, 6396), (40, 33)])
def test_masked_softmax_rows_bitexact(pb, rows, cols):
    g = np.random.default_rng(rows + cols)
    s = (g.standard_normal((rows, cols)) * 4).astype(np.float32)
    mask = np.where(g.random((rows, cols)) < 0.3, -np.inf, 0.0).astype(np.float32)
    mask[0] = -np.inf  # fully masked row -> zeros
    assert np.array_equal(bits(pb.masked_softmax_rows(dev(s)).cpu().numpy()), bits(orc.masked_softmax_rows(s)))
    got = pb.masked_softmax_rows(dev(s), dev(mask)).cpu().numpy()
    assert np.array_equal(bits(got), bits(orc.masked_softmax_rows(s, mask)))
    assert not got[0].any()


def test_masked_softmax_rows_rejects_like_the_reference(pb):
    s = np.zeros((2, 3), np.float32)
    s[1, 2] = np.nan
    with pytest.raises(pb.PbsaError, match="NaN"):
        pb.masked_softmax_rows(dev(s))
    m = np.zeros((2, 3), np.float32)
    m[0, 0] = 1.0
    with pytest.raises(pb.PbsaError, match="0 or -inf"):
        pb.masked_softmax_rows(dev(np.zeros((2, 3), np.float32)), dev(m))


@pytest.mark.parametrize("rows,cols", [(78, 546), (1, 9), (300, 6396)])
def test_aggregate_and_compress_bitexact(pb, rows, cols):
    g = np.random.default_rng(rows)
    a = orc.masked_softmax_rows(g.standard_normal((rows, cols)).astype(np.float32))
    assert np.array_equal(bits(pb.aggregate_scores(dev(a)).cpu().numpy()), bits(orc.aggregate_scores(a)))
    # compress_blocks on f32 blocks = the per-block token mean with the same fp64 sum
    x = (g.standard_normal((5, 60, 128)) * 3).astype(np.float32)
    reps = torch.empty(5, 128, device="cuda")
    from paper_2604_21221_b200._capi import LIB
    assert LIB.pbsa_compress_f32(dev(x).data_ptr(), 5, 60, 128, reps.data_ptr(), None) == 0
    assert np.array_equal(bits(reps.cpu().numpy()), bits(orc.compress_blocks(x)))


@pytest.mark.parametrize("rows,cols,k", [(78, 312, 78), (3, 6006, 1502), (5, 7, 1), (4, 40, 40), (2, 3000, 17)])
def test_select_topk_bitexact(pb, rows, cols, k):
    g = np.random.default_rng(cols + k)
    a = orc.masked_softmax_rows((g.standard_normal((rows, cols)) * 2).astype(np.float32))
    a[:, 1::5] = a[:, :1]  # exact ties -> lower index
    got = pb.select_topk(dev(a), k).cpu().numpy()
    assert np.array_equal(got, orc.select_topk(a, k))
    neg = (g.standard_normal((rows, cols))).astype(np.float32)  # any real values, incl. negatives
    neg[:, 2] = -0.0
    neg[:, 3] = 0.0
    assert np.array_equal(pb.select_topk(dev(neg), k).cpu().numpy(), orc.select_topk(neg, k))


@pytest.mark.parametrize("dims,shape", [((3, 30, 52, 8), (1, 15, 4)), ((3, 8, 8, 1), (3, 4, 4)),
                                        ((2, 16, 16, 3), (1, 8, 8)), ((2, 2, 2, 1), (1, 2, 2))])
def test_blockify_roundtrip_bitexact(pb, dims, shape):
    x = np.random.default_rng(sum(dims)).standard_normal(dims).astype(np.float32)
    xb = pb.blockify(dev(x), shape)
    assert np.array_equal(bits(xb.cpu().numpy()), bits(orc.blockify(x, shape)))
    assert np.array_equal(bits(pb.unblockify(xb, dims, shape).cpu().numpy()), bits(x))
    with pytest.raises(pb.PbsaError, match="not divisible"):
        pb.blockify(dev(x), (1, 7, 5))


def test_topc_select_matches_bruteforce(pb):
    """SPEC acceptance 4 shape: Top-C over <= 16 candidates vs the oracle's brute-force sort."""
    g = np.random.default_rng(4)
    for trial in range(200):
        n = int(g.integers(1, 17))
        ids = g.permutation(100)[:n].astype(np.int64)
        scores = g.integers(0, 4, n).astype(np.float32) / 4  # many exact ties
        slots = int(g.integers(0, n + 1))
        got = pb.topc_select(dev(ids, torch.int64), dev(scores), slots).cpu().numpy()
        want = orc.topc_select(ids, scores, np.zeros(n, np.uint8), slots)
        assert np.array_equal(got, want), trial
