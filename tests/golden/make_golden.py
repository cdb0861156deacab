"""Generate golden vectors for the LLM.int8() path from the REFERENCE itself.

Run in the build container (the only place the reference tree exists):

    python tests/golden/make_golden.py [--reference /root/reference/pkg/src] [--skip-cfg1]

It imports the reference package ``int8mm`` and records, for every case, the
inputs and the reference's own outputs for each stage of
``llm_int8_matmul`` (gemm.py:214-247):

* ``dims``   -- extract_outlier_columns(x, alpha).dims        (gemm.py:203-211)
* ``xq``/``sx`` -- rowwise_quantize(DenseMatrix(x[:, keep]))  (quantize.py:174-179)
* ``wq``/``sw`` -- colwise_quantize(DenseMatrix(w[keep, :]))  (quantize.py:182-187)
* ``c``      -- int8_gemm_i32(xq, wq)                         (gemm.py:78-82)
* ``out``    -- llm_int8_matmul(x, w, alpha).output           (gemm.py:214-247)
* ``vw``     -- vectorwise_matmul(x, w).output                (gemm.py:197-200)

Codes are stored in the reference's compacted layout (keep columns / rows
only). Inputs are fp16-representable float32 (the GPU consumes fp16), stored
as float16 (exact). The 512x4096x4096 config-1 case is large, so only its
digests (sha256 of each intermediate's bytes) and a row sample of the
output are stored; its inputs are regenerated from planted_pair's seed.

Outputs: tests/golden/llmint8_cases.npz, tests/golden/kats.json,
tests/golden/cfg1_digest.json.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def f16(a):
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)


def planted(rows, inner, cols, n_out, scale, seed):
    from int8mm import planted_pair

    x, w = planted_pair(rows, inner, cols, n_out, scale, seed)
    return f16(x.data), f16(w.data)


def cases():
    from int8mm import seeded_random_matrix

    out = []
    for seed in range(4):  # tests/test_gemm.py:37-43 style planted pairs
        out.append((f"planted_64x256x64_s{seed}", *planted(64, 256, 64, 2, 20.0, seed), 6.0))
    out.append(("ragged_33x200x40", *planted(33, 200, 40, 3, 20.0, 7), 6.0))
    out.append(("decode_1x512x96", *planted(1, 512, 96, 6, 20.0, 11), 6.0))
    out.append(("decode_7x384x72", *planted(7, 384, 72, 6, 20.0, 12), 6.0))
    # O = empty (tests/test_gemm.py:223-230)
    x = f16(seeded_random_matrix(8, 16, seed=21, stddev=1.0).data)
    w = f16(seeded_random_matrix(16, 8, seed=22, stddev=1.0).data)
    out.append(("no_outliers_8x16x8", x, w, 6.0))
    # full decomposition (tests/test_gemm.py:232-239)
    x = f16(seeded_random_matrix(8, 16, seed=23, stddev=1.0).data)
    w = f16(seeded_random_matrix(16, 8, seed=24, stddev=1.0).data)
    out.append(("full_decomp_8x16x8", x, w, 1e-9))
    # inclusive boundary, exact +-alpha values, zero rows/cols
    rng = np.random.Generator(np.random.PCG64(99))
    x = f16(rng.standard_normal((24, 96)).astype(np.float32))
    x[3, 10] = 6.0
    x[5, 20] = -6.0
    x[7, 30] = np.float32(5.99609375)  # largest fp16 below 6.0: not an outlier
    x[9, :] = 0.0  # zero row
    x[:, 40] = 0.0  # zero column
    w = f16(rng.standard_normal((96, 32)).astype(np.float32))
    w[:, 5] = 0.0  # zero W column -> amax 0 -> scale 1
    out.append(("boundary_zero_24x96x32", x, w, 6.0))
    # exact .5 ties: rows whose amax is 127 (scale exactly 1) hold half-integers
    x = np.zeros((6, 64), dtype=np.float32)
    x[:, 0] = 127.0
    x[:, 1:] = (np.arange(63, dtype=np.float32)[None, :] - 31.0) + 0.5
    x[1] *= -1
    x[2, 0] = 63.5  # amax 63.5 -> scale 2: x*2 integers
    x[3, 0] = 254.0  # amax 254 -> scale 0.5: half-integers * 0.5 -> quarter ties
    x[4, 0] = 84.0
    x[5, 0] = 3.0
    x = f16(x)
    w = f16(np.random.Generator(np.random.PCG64(5)).standard_normal((64, 16)).astype(np.float32))
    out.append(("ties_6x64x16", x, w, 1000.0))
    # paper-like one-sided outliers, SURVEY A.8
    rng = np.random.Generator(np.random.PCG64(123))
    x = rng.standard_normal((128, 1024)).astype(np.float32)
    cols = rng.choice(1024, size=6, replace=False)
    for c in cols:
        rows = rng.random(128) < 0.75
        x[rows, c] = rng.uniform(-44.0, -35.0, size=int(rows.sum())).astype(np.float32)
    w = rng.standard_normal((1024, 128)).astype(np.float32)
    out.append(("paperlike_128x1024x128", f16(x), f16(w), 6.0))
    # many outlier columns (|O| = 40)
    out.append(("many_outliers_32x256x48", *planted(32, 256, 48, 40, 20.0, 3), 6.0))
    return out


def reference_trace(x, w, alpha):
    from int8mm import (DenseMatrix, colwise_quantize, extract_outlier_columns, int8_gemm_i32,
                        llm_int8_matmul, rowwise_quantize, vectorwise_matmul)

    xm, wm = DenseMatrix(x), DenseMatrix(w)
    dims = extract_outlier_columns(xm, alpha).dims
    keep = np.ones(x.shape[1], dtype=bool)
    keep[list(dims)] = False
    rec = {"dims": np.asarray(dims, dtype=np.int64)}
    if keep.any():
        qx = rowwise_quantize(DenseMatrix(x[:, keep]))
        qw = colwise_quantize(DenseMatrix(w[keep, :]))
        rec["xq"] = qx.codes.data
        rec["sx"] = qx.params.scales
        rec["wq"] = qw.codes.data
        rec["sw"] = qw.params.scales
        rec["c"] = int8_gemm_i32(qx.codes, qw.codes).data
    r = llm_int8_matmul(xm, wm, alpha)
    rec["out"] = r.output.data
    rec["decomposed_cols"] = np.int64(r.decomposed_cols)
    rec["int8_fraction"] = np.float64(r.int8_fraction)
    rec["vw"] = vectorwise_matmul(xm, wm).output.data
    return rec


def kats():
    from int8mm import (ColwiseParams, DenseMatrix, Int32Matrix, RowwiseParams, colwise_quantize,
                        dequantize_output, round_half_away, rowwise_quantize, vectorwise_params)

    vals = [0.5, -0.5, 1.5, 2.5, -2.5, 0.49, -0.49]
    q = rowwise_quantize(DenseMatrix([[1.0, -1.0], [100.0, -100.0]]))
    q0 = rowwise_quantize(DenseMatrix([[0.0, 0.0], [2.0, -2.0]]))
    qx, qw = vectorwise_params(DenseMatrix([[1.0, 0.0], [0.0, 10.0]]),
                               DenseMatrix([[1.0, 100.0], [1.0, 100.0]]))
    deq = dequantize_output(Int32Matrix([[100, 200], [300, 400]]),
                            RowwiseParams(np.array([127.0, 12.7])),
                            ColwiseParams(np.array([127.0, 127.0])))
    qc = colwise_quantize(DenseMatrix([[1.0, 100.0], [1.0, 100.0]]))
    return {
        "round_half_away": {"in": vals, "out": [float(v) for v in round_half_away(np.array(vals))]},
        "rowwise_hand": {"x": [[1.0, -1.0], [100.0, -100.0]], "scales": q.params.scales.tolist(),
                         "codes": q.codes.data.tolist()},
        "rowwise_zero_row": {"x": [[0.0, 0.0], [2.0, -2.0]], "scales": q0.params.scales.tolist(),
                             "codes": q0.codes.data.tolist()},
        "vectorwise_scales": {"sx": qx.params.scales.tolist(), "sw": qw.params.scales.tolist()},
        "colwise_hand": {"w": [[1.0, 100.0], [1.0, 100.0]], "scales": qc.params.scales.tolist(),
                         "codes": qc.codes.data.tolist()},
        "dequant_outer": {"c": [[100, 200], [300, 400]], "sx": [127.0, 12.7], "sw": [127.0, 127.0],
                          "out": deq.data.astype(np.float64).tolist()},
        "gemm_identity": {"a": [[1, 2], [3, 4]], "b": [[1, 0], [0, 1]], "c": [[1, 2], [3, 4]]},
        "gemm_hand": {"a": [[2, 3]], "b": [[4], [5]], "c": [[23]]},
        "gemm_worst_case": {"k": 1 << 17, "c": 127 * 127 * (1 << 17)},
        "outlier_direct_scan": {"x": [[1.0, 100.0], [-1.0, 100.0]], "alpha": 6.0, "dims": [1]},
        "outlier_threshold_f32": {"x": [[float(np.float32(6.1))]], "alpha": 6.1, "dims": [0]},
    }


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg1_digest():
    x, w = planted(512, 4096, 4096, 6, 20.0, 0)
    t0 = time.perf_counter()
    rec = reference_trace(x, w, 6.0)
    dt = time.perf_counter() - t0
    sample_rows = np.arange(0, 512, 37)
    return {
        "shape": [512, 4096, 4096], "planted": [6, 20.0, 0], "alpha": 6.0,
        "dims": rec["dims"].tolist(),
        "sha256": {k: sha(rec[k]) for k in ("xq", "sx", "wq", "sw", "c", "out")},
        "c_min": int(rec["c"].min()), "c_max": int(rec["c"].max()),
        "out_absmax": float(np.abs(rec["out"]).max()),
        "sample_rows": sample_rows.tolist(),
        "out_sample_sha256": sha(rec["out"][sample_rows]),
        "decomposed_cols": int(rec["decomposed_cols"]),
        "int8_fraction": float(rec["int8_fraction"]),
        "reference_seconds": dt,
    }, rec["out"][sample_rows]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    ap.add_argument("--skip-cfg1", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, args.reference)
    import int8mm  # noqa: F401  (the reference package)

    arrays = {}
    names = []
    for name, x, w, alpha in cases():
        rec = reference_trace(x, w, alpha)
        names.append(name)
        arrays[f"{name}/x"] = x.astype(np.float16)
        arrays[f"{name}/w"] = w.astype(np.float16)
        arrays[f"{name}/alpha"] = np.float64(alpha)
        for k, v in rec.items():
            arrays[f"{name}/{k}"] = v
        print(f"{name}: |O|={len(rec['dims'])}")
    arrays["_names"] = np.array(names)
    np.savez_compressed(HERE / "llmint8_cases.npz", **arrays)
    (HERE / "kats.json").write_text(json.dumps(kats(), indent=1))
    if not args.skip_cfg1:
        dig, sample = cfg1_digest()
        (HERE / "cfg1_digest.json").write_text(json.dumps(dig, indent=1))
        np.save(HERE / "cfg1_out_sample.npy", sample)
        print("cfg1:", dig["dims"], f"{dig['reference_seconds']:.1f}s")


if __name__ == "__main__":
    main()
