"""QT8 fixtures written by the REFERENCE writer (pkg/src/int8mm/qt8.py).

    python tests/golden/make_golden_qt8.py [--reference /root/reference/pkg/src]

Writes tests/golden/qt8/{f32,i8,i32}.qt8 plus a malformed set (bad magic,
version 2, dtype 7, truncated header/payload, trailing bytes) so the mirror's
reader is checked against the reference's bytes and error classes.
"""
import argparse
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "qt8"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    sys.path.insert(0, ap.parse_args().reference)
    from int8mm import DenseMatrix, Int8Matrix, Int32Matrix
    from int8mm.qt8 import write_tensor

    OUT.mkdir(exist_ok=True)
    rng = np.random.Generator(np.random.PCG64(8))
    write_tensor(OUT / "f32.qt8", DenseMatrix(rng.standard_normal((5, 7)).astype(np.float32)))
    write_tensor(OUT / "i8.qt8", Int8Matrix(rng.integers(-127, 128, size=(3, 9))))
    write_tensor(OUT / "i32.qt8", Int32Matrix(rng.integers(-2**31, 2**31, size=(4, 2), dtype=np.int64)))
    good = (OUT / "i8.qt8").read_bytes()
    (OUT / "bad_magic.qt8").write_bytes(b"QT9\x00" + good[4:])
    (OUT / "bad_version.qt8").write_bytes(good[:4] + (2).to_bytes(4, "little") + good[8:])
    (OUT / "bad_dtype.qt8").write_bytes(good[:8] + bytes([7]) + good[9:])
    (OUT / "short_header.qt8").write_bytes(good[:20])
    (OUT / "short_payload.qt8").write_bytes(good[:-1])
    (OUT / "trailing.qt8").write_bytes(good + b"\x00")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
