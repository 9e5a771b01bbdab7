"""PBT1 tensor files: the library's reader/writer against the
reference's own tensor_io.cpp -- via committed fixtures written and read by the reference
(tests/golden/make_golden_pbt1.py) and, where oracle/_ref is built, live round trips."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "pbt1")
EXPECTED = json.load(open(os.path.join(GOLD, "expected.json")))
pb = pytest.importorskip("paper_2604_21221_b200")


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_reader_matches_reference_on_fixtures(name):
    want = EXPECTED[name]
    path = os.path.join(GOLD, name)
    if "error" in want:
        with pytest.raises(pb.TensorIoError) as ei:
            pb.read_tensor(path)
        assert ei.value.kind == want["error"], str(ei.value)
    else:
        got = pb.read_tensor(path)
        assert list(got.shape) == want["dims"]
        np.testing.assert_array_equal(got.reshape(-1), np.asarray(want["payload"], np.float32))


@pytest.mark.parametrize("name", ["matrix_3x5.pbt1", "latent_2x3x4x8.pbt1", "matrix_0x4.pbt1"])
def test_writer_is_byte_identical_to_reference(name, tmp_path):
    src = os.path.join(GOLD, name)
    out = tmp_path / name
    pb.write_tensor(out, pb.read_tensor(src))
    assert open(out, "rb").read() == open(src, "rb").read()


def test_missing_file_is_open_failed(tmp_path):
    with pytest.raises(pb.TensorIoError) as ei:
        pb.read_tensor(tmp_path / "nope.pbt1")
    assert ei.value.kind == "OpenFailed"
    with pytest.raises(pb.TensorIoError) as ei:
        pb.write_tensor(tmp_path / "no_dir" / "x.pbt1", np.zeros(3, np.float32))
    assert ei.value.kind == "OpenFailed"


@pytest.mark.skipif(orc.ref_lib() is None, reason="oracle/_ref (reference build) absent")
def test_live_round_trips_with_reference(tmp_path):
    ref = orc.ref_lib()
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    i64 = C.c_int64
    ref.ref_write_latent.argtypes = [C.c_char_p, f32p, i64, i64, i64, i64]
    ref.ref_read_tensor.argtypes = [C.c_char_p, f32p, i64, C.POINTER(i64), C.POINTER(i64)]
    rng = np.random.default_rng(7)
    for shape in [(1, 1, 1, 1), (3, 5, 2, 7), (2, 30, 52, 4)]:
        x = rng.standard_normal(shape).astype(np.float32)
        a, b = tmp_path / "ref.pbt1", tmp_path / "ours.pbt1"
        assert ref.ref_write_latent(str(a).encode(), x, *shape) == 0
        np.testing.assert_array_equal(pb.read_tensor(a), x)          # reference -> ours
        pb.write_tensor(b, x)
        buf = np.zeros(x.size, np.float32)
        rank, dims = i64(), (i64 * 8)()
        assert ref.ref_read_tensor(str(b).encode(), buf, x.size, C.byref(rank), dims) == 0  # ours -> reference
        assert tuple(dims[i] for i in range(rank.value)) == shape
        np.testing.assert_array_equal(buf.reshape(shape), x)
        assert open(a, "rb").read() == open(b, "rb").read()


@pytest.mark.gpu
def test_load_bf16_to_device(tmp_path):
    import torch
    x = np.random.default_rng(3).standard_normal((3, 30, 52, 64)).astype(np.float32)
    path = tmp_path / "lat.pbt1"
    pb.write_tensor(path, x)
    d = pb.load_bf16(path)
    torch.cuda.synchronize()
    assert d.dtype == torch.bfloat16 and tuple(d.shape) == x.shape
    assert torch.equal(d.cpu(), torch.from_numpy(x).to(torch.bfloat16))
    big = np.random.default_rng(4).standard_normal((3, 30, 52, 1152)).astype(np.float32)  # 3 staging pieces
    pb.write_tensor(path, big)
    assert torch.equal(pb.load_bf16(path).cpu(), torch.from_numpy(big).to(torch.bfloat16))
    with pytest.raises(pb.TensorIoError) as ei:
        pb.load_bf16(os.path.join(GOLD, "truncated_payload.pbt1"))
    assert ei.value.kind == "Truncated"
