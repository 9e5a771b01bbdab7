"""Generates tests/golden/pbt1/ with THE REFERENCE'S OWN PBT1 writer and reader
(proj/src/tensor_io.cpp compiled where it lies into oracle/_ref/libpbsa_ref.so, `make -C oracle ref`).

Well-formed files are written by pbsa::write_tensor; malformed variants are byte edits of them;
expected.json records, for every file, what pbsa::read_tensor returns (dims + payload) or the
TensorIoError::Kind it throws -- so tests/test_pbt1.py pins the library's PBT1 reader/writer to the
reference on machines without /root/reference.  Run from the repo root:
    python tests/golden/make_golden_pbt1.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "pbt1")
KINDS = ["OpenFailed", "BadMagic", "BadDtype", "Truncated", "TrailingData", "BadShape"]
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i64 = C.c_int64


def main():
    ref = orc.ref_lib()
    if ref is None:
        raise SystemExit("oracle/_ref/libpbsa_ref.so missing: run `make -C oracle ref` first")
    ref.ref_write_matrix.argtypes = [C.c_char_p, f32p, i64, i64]
    ref.ref_write_latent.argtypes = [C.c_char_p, f32p, i64, i64, i64, i64]
    ref.ref_read_tensor.argtypes = [C.c_char_p, f32p, i64, C.POINTER(i64), C.POINTER(i64)]
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2604)
    good = {}
    m = rng.standard_normal((3, 5)).astype(np.float32)
    p = os.path.join(OUT, "matrix_3x5.pbt1")
    assert ref.ref_write_matrix(p.encode(), m, 3, 5) == 0
    good["matrix_3x5.pbt1"] = p
    x = rng.standard_normal((2, 3, 4, 8)).astype(np.float32)
    p = os.path.join(OUT, "latent_2x3x4x8.pbt1")
    assert ref.ref_write_latent(p.encode(), x, 2, 3, 4, 8) == 0
    good["latent_2x3x4x8.pbt1"] = p
    p = os.path.join(OUT, "matrix_0x4.pbt1")
    assert ref.ref_write_matrix(p.encode(), np.zeros(1, np.float32), 0, 4) == 0
    good["matrix_0x4.pbt1"] = p

    base = open(good["matrix_3x5.pbt1"], "rb").read()
    bad = {
        "bad_magic.pbt1": b"PBT2" + base[4:],
        "bad_dtype.pbt1": base[:4] + b"\x02" + base[5:],
        "truncated_magic.pbt1": base[:3],
        "truncated_rank.pbt1": base[:5],
        "truncated_dims.pbt1": base[:6 + 8 + 3],
        "truncated_payload.pbt1": base[:-4],
        "trailing_data.pbt1": base + b"\x00",
        "zero_elems_with_data.pbt1": open(good["matrix_0x4.pbt1"], "rb").read() + b"\x00\x00\x80\x3f",
        "dims_overflow.pbt1": base[:4] + b"\x01\x02" + (2**40).to_bytes(8, "little") + (2**40).to_bytes(8, "little"),
    }
    for name, data in bad.items():
        with open(os.path.join(OUT, name), "wb") as f:
            f.write(data)

    expected = {}
    for name in sorted(os.listdir(OUT)):
        if not name.endswith(".pbt1"):
            continue
        path = os.path.join(OUT, name).encode()
        buf = np.zeros(4096, np.float32)
        rank, dims = i64(), (i64 * 8)()
        rc = ref.ref_read_tensor(path, buf, 4096, C.byref(rank), dims)
        if rc == 0:
            dd = [int(dims[i]) for i in range(rank.value)]
            n = int(np.prod(dd)) if dd else 0
            expected[name] = {"dims": dd, "payload": buf[:n].tolist()}
        else:
            assert rc >= 10, (name, rc)
            expected[name] = {"error": KINDS[rc - 10]}
    with open(os.path.join(OUT, "expected.json"), "w") as f:
        json.dump(expected, f, indent=1)
    print("wrote", len(expected), "files")


if __name__ == "__main__":
    main()
