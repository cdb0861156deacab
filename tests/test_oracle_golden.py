"""Pin the CPU oracle (numpy + C restatements) to the reference's golden vectors.

The oracle is only trusted as the GPU checker because every case below is
bit-exact against outputs produced by the reference package itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np
import pytest

import _golden

GOLDEN = _golden.cases()


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_numpy_oracle_matches_reference(oracle_mod, name):
    g = GOLDEN[name]
    tr = oracle_mod.llm_int8_matmul(g["x"], g["w"], g["alpha"])
    assert tr.dims == tuple(int(d) for d in g["dims"])
    keep = _golden.keep_mask(g["x"].shape[1], tr.dims)
    if keep.any():
        assert np.array_equal(tr.xq[:, keep], g["xq"])
        assert np.array_equal(tr.sx, g["sx"])
        assert np.array_equal(tr.wq[keep], g["wq"])
        assert np.array_equal(tr.sw, g["sw"])
        assert np.array_equal(tr.c, g["c"])
    assert np.array_equal(tr.output, g["out"])
    assert tr.decomposed_cols == int(g["decomposed_cols"])
    assert tr.int8_fraction == float(g["int8_fraction"])
    assert np.array_equal(oracle_mod.vectorwise_matmul(g["x"], g["w"]), g["vw"])


F32 = _golden.f32_cases()


@pytest.mark.parametrize("name", sorted(F32))
def test_oracles_match_reference_on_f32_operands(oracle_mod, name):
    """Both restatements on float32 values that are not fp16 values (the
    reference's DenseMatrix is float32, tensors.py:31-49)."""
    g = F32[name]
    for tr in (oracle_mod.llm_int8_matmul(g["x"], g["w"], g["alpha"]),
               oracle_mod.c_llm_int8_matmul(g["x"], g["w"], g["alpha"])):
        assert tr.dims == tuple(int(d) for d in g["dims"])
        keep = _golden.keep_mask(g["x"].shape[1], tr.dims)
        if keep.any():
            assert np.array_equal(tr.xq[:, keep], g["xq"])
            assert np.array_equal(tr.sx, g["sx"])
            assert np.array_equal(tr.wq[keep], g["wq"])
            assert np.array_equal(tr.sw, g["sw"])
            assert np.array_equal(tr.c, g["c"])
        assert np.array_equal(tr.output, g["out"])
    assert np.array_equal(oracle_mod.vectorwise_matmul(g["x"], g["w"]), g["vw"])
    assert np.array_equal(oracle_mod.absmax_matmul(g["x"], g["w"]), g["absmax"])
    assert np.array_equal(oracle_mod.zeropoint_matmul(g["x"], g["w"]), g["zeropoint"])


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_c_oracle_matches_reference(oracle_mod, name):
    g = GOLDEN[name]
    tr = oracle_mod.c_llm_int8_matmul(g["x"], g["w"], g["alpha"])
    assert tr.dims == tuple(int(d) for d in g["dims"])
    keep = _golden.keep_mask(g["x"].shape[1], tr.dims)
    if keep.any():
        assert np.array_equal(tr.xq[:, keep], g["xq"])
        assert np.array_equal(tr.sx, g["sx"])
        assert np.array_equal(tr.wq[keep], g["wq"])
        assert np.array_equal(tr.sw, g["sw"])
        assert np.array_equal(tr.c, g["c"])
    assert np.array_equal(tr.output, g["out"])


def test_kats(oracle_mod):
    k = _golden.kats()
    r = k["round_half_away"]
    assert oracle_mod.round_half_away(np.array(r["in"])).tolist() == r["out"]
    codes, sc = oracle_mod.rowwise_quantize(np.array(k["rowwise_hand"]["x"], np.float32))
    assert sc.tolist() == k["rowwise_hand"]["scales"] and codes.tolist() == k["rowwise_hand"]["codes"]
    codes, sc = oracle_mod.rowwise_quantize(np.array(k["rowwise_zero_row"]["x"], np.float32))
    assert sc.tolist() == k["rowwise_zero_row"]["scales"]
    codes, sc = oracle_mod.colwise_quantize(np.array(k["colwise_hand"]["w"], np.float32))
    assert sc.tolist() == k["colwise_hand"]["scales"] and codes.tolist() == k["colwise_hand"]["codes"]
    d = k["dequant_outer"]
    out = oracle_mod.dequantize_output(np.array(d["c"], np.int32), np.array(d["sx"]), np.array(d["sw"]))
    assert out.astype(np.float64).tolist() == d["out"]
    for key in ("gemm_identity", "gemm_hand"):
        a, b = np.array(k[key]["a"], np.int8), np.array(k[key]["b"], np.int8)
        assert oracle_mod.int8_gemm_i32(a, b).tolist() == k[key]["c"]
        assert oracle_mod.c_gemm_i32(a, b).tolist() == k[key]["c"]
    h = k["gemm_worst_case"]["k"]
    c = oracle_mod.c_gemm_i32(np.full((1, h), 127, np.int8), np.full((h, 1), 127, np.int8))
    assert int(c[0, 0]) == k["gemm_worst_case"]["c"]
    x = np.array(k["outlier_threshold_f32"]["x"], np.float32)
    assert list(oracle_mod.outlier_dims(x, 6.1)) == k["outlier_threshold_f32"]["dims"]
    assert list(oracle_mod.c_outlier_mask(x, 6.1).nonzero()[0]) == [0]


def test_bigint_equivalence_c_oracle(oracle_mod):
    """Acceptance criterion 1 (test_acceptance.py:50-59) on the C oracle, 200 seeds."""
    for seed in range(200):
        rng = np.random.Generator(np.random.PCG64(seed))
        s, h, o = (int(d) for d in rng.integers(1, 65, size=3))
        a = rng.integers(-127, 128, size=(s, h)).astype(np.int8)
        b = rng.integers(-127, 128, size=(h, o)).astype(np.int8)
        ref = a.astype(np.int64) @ b.astype(np.int64)
        assert np.array_equal(oracle_mod.c_gemm_i32(a, b), ref)
        assert np.array_equal(oracle_mod.int8_gemm_i32(a, b), ref)


def test_cfg1_digest_c_oracle(oracle_mod):
    """The C oracle reproduces the reference's config-1 digests (one run ~1 s)."""
    dig, sample = _golden.cfg1()
    m, k, n = dig["shape"]
    x, w = oracle_mod.planted_pair(m, k, n, *dig["planted"])
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    tr = oracle_mod.c_llm_int8_matmul(x, w, dig["alpha"])
    assert list(tr.dims) == dig["dims"]
    keep = _golden.keep_mask(k, tr.dims)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(tr.xq[:, keep]) == dig["sha256"]["xq"]
    assert sha(tr.sx) == dig["sha256"]["sx"]
    assert sha(np.ascontiguousarray(tr.wq[keep])) == dig["sha256"]["wq"]
    assert sha(tr.sw) == dig["sha256"]["sw"]
    assert sha(tr.c) == dig["sha256"]["c"]
    assert sha(tr.output) == dig["sha256"]["out"]
    assert np.array_equal(tr.output[dig["sample_rows"]], sample)


# ---------------------------------------------------------------- sibling schemes
SIB = Path(__file__).resolve().parent / "golden" / "siblings_cases.npz"


def _sib_cases():
    d = np.load(SIB)
    return d, [str(n) for n in d["names"]]


def test_oracle_siblings_match_reference_goldens():
    """absmax / zeropoint restatements vs the reference's own outputs
    (tests/golden/make_golden_siblings.py), bit-exact."""
    from oracle import oracle as orc

    d, names = _sib_cases()
    assert len(names) >= 12
    for name in names:
        x = d[f"{name}/x"].astype(np.float32)
        w = d[f"{name}/w"].astype(np.float32)
        for tag, mat in (("x", x), ("w", w)):
            codes, scale = orc.absmax_quantize(mat)
            assert np.array_equal(codes, d[f"{name}/abs_{tag}_codes"]), (name, tag)
            assert scale == float(d[f"{name}/abs_{tag}_scale"]), (name, tag)
            if f"{name}/zp_{tag}_error" in d:
                with pytest.raises(ValueError):
                    orc.zeropoint_quantize(mat)
            else:
                codes, nd, zp, off = orc.zeropoint_quantize(mat)
                assert np.array_equal(codes, d[f"{name}/zp_{tag}_codes"]), (name, tag)
                assert [nd, zp, off] == d[f"{name}/zp_{tag}_params"].tolist(), (name, tag)
        assert np.array_equal(orc.absmax_matmul(x, w), d[f"{name}/abs_out"]), name
        if f"{name}/zp_out" in d:
            assert np.array_equal(orc.zeropoint_matmul(x, w), d[f"{name}/zp_out"]), name
            qx, _, zpx, _ = orc.zeropoint_quantize(x)
            qw, _, zpw, _ = orc.zeropoint_quantize(w)
            assert np.array_equal(orc.zeropoint_gemm_i32(qx, qw, zpx, zpw), d[f"{name}/zp_c"]), name
        elif int(d[f"{name}/zp_out_error"]) == 2:
            with pytest.raises(OverflowError):
                orc.zeropoint_matmul(x, w)
        else:
            with pytest.raises(ValueError):
                orc.zeropoint_matmul(x, w)


def test_host_zeropoint_params_match_reference():
    """i8mm_zeropoint_params (host C, no GPU) reproduces the reference's
    nd / zp / offset and its int16 range error (quantize.py:153-166)."""
    import ctypes

    from paper_2208_07339_b200 import _native as nat

    L = nat.load_library()
    d, names = _sib_cases()
    seen_error = False
    for name in names:
        for tag in ("x", "w"):
            t = d[f"{name}/{tag}"].astype(np.float32)
            nd, zp, off = ctypes.c_double(), ctypes.c_int32(), ctypes.c_double()
            st = L.i8mm_zeropoint_params(float(t.min()), float(t.max()), ctypes.byref(nd),
                                         ctypes.byref(zp), ctypes.byref(off))
            if f"{name}/zp_{tag}_error" in d:
                assert st == nat.I8MM_ERR_ZEROPOINT, (name, tag)
                seen_error = True
            else:
                assert st == 0
                assert [nd.value, zp.value, off.value] == d[f"{name}/zp_{tag}_params"].tolist(), (name, tag)
    assert seen_error
