"""Loader for the golden vectors produced by tests/golden/make_golden.py."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def cases() -> dict[str, dict]:
    z = np.load(GOLDEN / "llmint8_cases.npz")
    out: dict[str, dict] = {}
    for name in z["_names"].tolist():
        rec = {}
        for key in z.files:
            if key.startswith(name + "/"):
                rec[key[len(name) + 1:]] = z[key]
        rec["x"] = rec["x"].astype(np.float32)
        rec["w"] = rec["w"].astype(np.float32)
        rec["alpha"] = float(rec["alpha"])
        out[name] = rec
    return out


def kats() -> dict:
    return json.loads((GOLDEN / "kats.json").read_text())


def cfg1() -> tuple[dict, np.ndarray]:
    return json.loads((GOLDEN / "cfg1_digest.json").read_text()), np.load(
        GOLDEN / "cfg1_out_sample.npy")


def keep_mask(k: int, dims) -> np.ndarray:
    keep = np.ones(k, dtype=bool)
    keep[np.asarray(dims, dtype=np.int64)] = False
    return keep


def fp16_tolerance(ref: np.ndarray) -> np.ndarray:
    """Stated fp16-output tolerance: 1 fp16 ulp of |ref| plus 1e-5 * max|ref|.

    fp16 rounding alone is <= 0.5 ulp; the fp32 epilogue adds a few f32 ulps of
    the (possibly cancelling) int8 and outlier partial products.
    """
    a = np.abs(ref.astype(np.float64))
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -14)))
    ulp = 2.0 ** (e - 10)
    return ulp + 1e-5 * max(1.0, float(a.max(initial=0.0)))


def f32_cases() -> dict[str, dict]:
    """float32 (non-fp16) cases written by tests/golden/make_golden_f32.py."""
    z = np.load(GOLDEN / "f32_cases.npz")
    out: dict[str, dict] = {}
    for name in z["_names"].tolist():
        rec = {k[len(name) + 1:]: z[k] for k in z.files if k.startswith(name + "/")}
        rec["alpha"] = float(rec["alpha"])
        out[name] = rec
    return out
