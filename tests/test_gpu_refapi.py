"""The reference's own hot-path tests, run against the import-swap module
``paper_2208_07339_b200.int8mm`` on the B200.

The cases restate the reference's KATs (pkg/tests/test_gemm.py,
test_quantize.py, test_tensors.py) with the reference's types: the module
returns DenseMatrix / Int8Matrix / Int32Matrix containers whose ``.data`` is a
host numpy array, so each assertion reads like the reference's. Also:
float32 operands that are not fp16 values (reference-generated goldens,
tests/golden/make_golden_f32.py) bit-exact through the float32 kernels, and
the plugin point's NaN/Inf contract (transformer.py:257-267, tensors.py:47-48).
"""

from __future__ import annotations

import numpy as np
import pytest

import _golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def m():
    from paper_2208_07339_b200 import _native
    from paper_2208_07339_b200 import int8mm

    _native.load_library()
    return int8mm


def _codes(rows, cols, seed, m):
    rng = np.random.Generator(np.random.PCG64(seed))
    return m.Int8Matrix(rng.integers(-127, 128, size=(rows, cols)))


def _py_matmul(a, b):
    """Exact product with Python integers (the reference's bigint oracle idea)."""
    return [[sum(int(a[i, t]) * int(b[t, j]) for t in range(a.shape[1])) for j in range(b.shape[1])]
            for i in range(a.shape[0])]


def _f64(x, w):
    return np.asarray(x, np.float64) @ np.asarray(w, np.float64)


def _relfro(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


# ---------------------------------------------------------------- int8 GEMM (test_gemm.py:46-97)
def test_int8_gemm_kats(m):
    assert m.int8_gemm_i32(m.Int8Matrix([[1, 2], [3, 4]]),
                           m.Int8Matrix(np.eye(2, dtype=np.int8))).data.tolist() == [[1, 2], [3, 4]]
    assert m.int8_gemm_i32(m.Int8Matrix([[2, 3]]), m.Int8Matrix([[4], [5]])).data.tolist() == [[23]]
    h = m.MAX_INNER_DIM
    c = m.int8_gemm_i32(m.Int8Matrix(np.full((1, h), 127, np.int8)),
                        m.Int8Matrix(np.full((h, 1), 127, np.int8)))
    assert isinstance(c, m.Int32Matrix)
    assert int(c.data[0, 0]) == 127 * 127 * h == 2_114_060_288
    with pytest.raises(m.GemmOverflowError):
        m.int8_gemm_i32(m.Int8Matrix(np.zeros((1, h + 1), np.int8)),
                        m.Int8Matrix(np.zeros((h + 1, 1), np.int8)))
    with pytest.raises(m.ShapeMismatchError):
        m.int8_gemm_i32(_codes(2, 3, 0, m), _codes(2, 2, 1, m))


def test_int8_gemm_bigint_seeded(m):
    for seed in range(25):
        rng = np.random.Generator(np.random.PCG64(seed))
        s, h, o = (int(v) for v in rng.integers(1, 33, size=3))
        a, b = _codes(s, h, seed, m), _codes(h, o, seed + 1000, m)
        assert m.int8_gemm_i32(a, b).data.tolist() == _py_matmul(a.data, b.data)


# ---------------------------------------------------------------- sibling matmuls (test_gemm.py:99-197)
def test_absmax_matmul_kats(m):
    r = m.absmax_matmul(m.DenseMatrix(np.eye(2)), m.DenseMatrix(np.eye(2)))
    assert np.array_equal(r.output.data, np.eye(2, dtype=np.float32))
    assert r.scheme == "absmax" and r.int8_fraction == 1.0
    r = m.absmax_matmul(m.DenseMatrix([[1.0, 1.0]]), m.DenseMatrix([[1.0], [1.0]]))
    assert abs(r.output.data[0, 0] - 2.0) <= 2 * (0.5 / 127.0)
    rng = np.random.Generator(np.random.PCG64(42))
    x = rng.standard_normal((8, 8)).astype(np.float32)
    x[3, 4] = 100.0
    x, w = m.DenseMatrix(x), m.DenseMatrix(rng.standard_normal((8, 8)).astype(np.float32))
    ex = _f64(x.data, w.data)
    assert _relfro(m.absmax_matmul(x, w).output.data, ex) > _relfro(m.vectorwise_matmul(x, w).output.data, ex)
    with pytest.raises(m.ShapeMismatchError):
        m.absmax_matmul(m.DenseMatrix(np.ones((2, 3))), m.DenseMatrix(np.ones((2, 3))))


def test_zeropoint_matmul_kats(m):
    for seed in range(10):
        x = m.seeded_random_matrix(6, 9, seed=seed, stddev=1.0)
        w = m.seeded_random_matrix(9, 5, seed=seed + 500, stddev=1.0)
        assert np.array_equal(m.zeropoint_matmul(x, w, unrolled=False).output.data,
                              m.zeropoint_matmul(x, w, unrolled=True).output.data)
    x, w = m.DenseMatrix([[-1.0, 0.0, 1.0]]), m.DenseMatrix([[-1.0], [0.0], [1.0]])
    assert np.array_equal(m.zeropoint_matmul(x, w).output.data, m.absmax_matmul(x, w).output.data)
    assert m.zeropoint_matmul(x, w).output.data[0, 0] == 2.0
    assert m.zeropoint_matmul(m.DenseMatrix([[0.0, 4.0]]),
                              m.DenseMatrix([[0.0], [4.0]])).output.data[0, 0] == 16.0
    x = m.DenseMatrix(np.full((3, 4), 2.5, dtype=np.float32))
    w = m.seeded_random_matrix(4, 2, seed=11, stddev=1.0)
    bound = 2.5 * x.cols * (0.5 / m.zeropoint_quantize(w).params.nd + 1e-6)
    assert np.abs(m.zeropoint_matmul(x, w).output.data - _f64(x.data, w.data)).max() <= bound
    r = m.zeropoint_matmul(m.DenseMatrix(np.full((2, 3), 2.0, np.float32)),
                           m.DenseMatrix(np.full((3, 2), -1.5, np.float32)))
    assert np.array_equal(r.output.data, np.full((2, 2), -9.0, dtype=np.float32))


def test_vectorwise_matmul_kats(m):
    r = m.vectorwise_matmul(m.DenseMatrix(np.diag([1.0, 10.0])), m.DenseMatrix(np.eye(2)))
    assert np.array_equal(r.output.data, np.diag([1.0, 10.0]).astype(np.float32))
    x = m.seeded_random_matrix(1, 9, seed=11, stddev=1.0)
    w = m.seeded_random_matrix(9, 1, seed=12, stddev=1.0)
    assert np.array_equal(m.vectorwise_matmul(x, w).output.data, m.absmax_matmul(x, w).output.data)
    for seed in range(20):
        rng = np.random.Generator(np.random.PCG64(seed))
        x = rng.standard_normal((8, 8)).astype(np.float32) * np.arange(1, 9, dtype=np.float32)[:, None]
        x, w = m.DenseMatrix(x), m.DenseMatrix(rng.standard_normal((8, 8)).astype(np.float32))
        ex = _f64(x.data, w.data)
        assert _relfro(m.vectorwise_matmul(x, w).output.data, ex) <= _relfro(
            m.absmax_matmul(x, w).output.data, ex)


# ---------------------------------------------------------------- outliers + LLM.int8() (test_gemm.py:200-274)
def test_extract_outlier_columns_kats(m):
    assert m.extract_outlier_columns(m.seeded_random_matrix(4, 6, seed=0, stddev=0.1), 6.0).dims == ()
    s = m.extract_outlier_columns(m.DenseMatrix([[1.0, 100.0], [-1.0, 100.0]]), 6.0)
    assert s.dims == (1,) and s.alpha == 6.0
    x = np.zeros((2, 5), dtype=np.float32)
    x[1, 3] = 6.0
    assert m.extract_outlier_columns(m.DenseMatrix(x), 6.0).dims == (3,)
    x = np.zeros((2, 5), dtype=np.float32)
    x[0, 2] = -7.5
    assert m.extract_outlier_columns(m.DenseMatrix(x), 6.0).dims == (2,)
    with pytest.raises(ValueError):
        m.extract_outlier_columns(m.DenseMatrix(x), 0.0)


def test_llm_int8_matmul_kats(m):
    x = m.seeded_random_matrix(8, 16, seed=21, stddev=1.0)
    w = m.seeded_random_matrix(16, 8, seed=22, stddev=1.0)
    r = m.llm_int8_matmul(x, w, alpha=6.0)
    assert np.array_equal(r.output.data, m.vectorwise_matmul(x, w).output.data)
    assert (r.decomposed_cols, r.int8_fraction, r.scheme) == (0, 1.0, "llm_int8")
    x = m.seeded_random_matrix(8, 16, seed=23, stddev=1.0)
    w = m.seeded_random_matrix(16, 8, seed=24, stddev=1.0)
    r = m.llm_int8_matmul(x, w, alpha=1e-9)
    assert _relfro(r.output.data, _f64(x.data, w.data)) < 1e-6
    assert r.decomposed_cols == 16 and r.int8_fraction == 0.0
    rng = np.random.Generator(np.random.PCG64(0))
    xx = rng.standard_normal((4, 4096)).astype(np.float32) * 0.5
    xx[:, [17, 1000, 2000, 4000]] *= 40.0
    r = m.llm_int8_matmul(m.DenseMatrix(xx), m.DenseMatrix(rng.standard_normal((4096, 4)).astype(np.float32)))
    assert r.decomposed_cols == 4 and r.int8_fraction >= 0.999


def test_error_ordering_on_planted_outliers(m):
    means = {"absmax": [], "vectorwise": [], "llm_int8": []}
    for seed in range(10):
        rng = np.random.Generator(np.random.PCG64(seed))
        x = rng.standard_normal((16, 64)).astype(np.float32)
        x[:, rng.choice(64, size=2, replace=False)] *= np.float32(20.0)
        x, w = m.DenseMatrix(x), m.DenseMatrix(rng.standard_normal((64, 16)).astype(np.float32))
        ex = _f64(x.data, w.data)
        means["absmax"].append(_relfro(m.absmax_matmul(x, w).output.data, ex))
        means["vectorwise"].append(_relfro(m.vectorwise_matmul(x, w).output.data, ex))
        means["llm_int8"].append(_relfro(m.llm_int8_matmul(x, w, 6.0).output.data, ex))
    a, v, l = (float(np.mean(means[k])) for k in ("absmax", "vectorwise", "llm_int8"))
    assert a > v > l and l < 0.02


def test_ordered_matmul_f64(m):
    x = m.seeded_random_matrix(7, 33, seed=5, stddev=1.0)
    w = m.seeded_random_matrix(33, 6, seed=6, stddev=1.0)
    ours = m.ordered_matmul_f64(x.data, w.data)
    assert isinstance(ours, np.ndarray) and ours.dtype == np.float64
    assert np.allclose(ours, _f64(x.data, w.data), rtol=1e-12, atol=1e-12)
    # bitwise: the ascending-k restatement (gemm.py:110-117)
    acc = np.zeros((7, 6))
    for k in range(33):
        acc += np.multiply.outer(x.data[:, k].astype(np.float64), w.data[k, :].astype(np.float64))
    assert np.array_equal(ours, acc)


# ---------------------------------------------------------------- dequantize_output (test_gemm.py:276-308)
def test_dequantize_output_kats(m):
    out = m.dequantize_output(m.Int32Matrix([[127 * 127]]), m.AbsmaxParams(127.0), m.AbsmaxParams(127.0))
    assert out.data[0, 0] == 1.0
    out = m.dequantize_output(m.Int32Matrix([[100, 200], [300, 400]]),
                              m.RowwiseParams(np.array([127.0, 12.7])),
                              m.ColwiseParams(np.array([127.0, 127.0])))
    assert out.data[1, 0] == np.float32(300.0 / (12.7 * 127.0))
    out = m.dequantize_output(m.Int32Matrix(np.zeros((2, 2), np.int32)), m.AbsmaxParams(3.0),
                              m.AbsmaxParams(5.0))
    assert not out.data.any()
    with pytest.raises(m.ParamsMismatchError):
        m.dequantize_output(m.Int32Matrix([[1]]), m.AbsmaxParams(1.0), m.RowwiseParams(np.array([1.0])))
    with pytest.raises(m.ParamsMismatchError):
        m.dequantize_output(m.Int32Matrix([[1]]), m.ColwiseParams(np.array([1.0])),
                            m.RowwiseParams(np.array([1.0])))
    with pytest.raises(m.ParamsMismatchError):
        m.dequantize_output(m.Int32Matrix([[1, 2], [3, 4]]), m.RowwiseParams(np.array([1.0, 2.0, 3.0])),
                            m.ColwiseParams(np.array([1.0, 2.0])))


# ---------------------------------------------------------------- quantize.py (test_quantize.py)
@pytest.mark.parametrize("value,expected", [(0.5, 1), (-0.5, -1), (1.5, 2), (2.5, 3), (-2.5, -3),
                                            (0.49, 0), (-0.49, 0)])
def test_round_half_away(m, value, expected):
    assert m.round_half_away(np.array([value]))[0] == expected


def test_absmax_quantize_kats(m):
    q = m.absmax_quantize(m.DenseMatrix([[0.0, 0.0], [0.0, 0.0]]))
    assert q.params == m.AbsmaxParams(1.0) and not q.codes.data.any()
    q = m.absmax_quantize(m.DenseMatrix([[1.0]]))
    assert q.params.scale == 127.0 and q.codes.data[0, 0] == 127
    q = m.absmax_quantize(m.DenseMatrix([[2.0, -4.0]]))
    assert q.params.scale == 31.75 and q.codes.data.tolist() == [[64, -127]]
    assert np.array_equal(m.dequantize(q).data, np.array([[64 / 31.75, -4.0]], dtype=np.float32))


def test_zeropoint_quantize_kats(m):
    x = m.DenseMatrix(np.array([[-0.5 / 254.0, 253.5 / 254.0]], dtype=np.float32))
    q = m.zeropoint_quantize(x)
    assert q.codes.data.max() <= 127
    assert np.abs(m.dequantize(q).data - x.data).max() <= 0.5 / q.params.nd + 1e-6
    with pytest.raises(ValueError):
        m.zeropoint_quantize(m.DenseMatrix(np.array([[1e6, 1e6 + 1.0]], dtype=np.float32)))
    q = m.zeropoint_quantize(m.DenseMatrix(np.full((2, 3), 1.25, np.float32)))
    assert q.params.offset == 1.25 and not q.codes.data.any()
    assert np.array_equal(m.dequantize(q).data, np.full((2, 3), 1.25, np.float32))


def test_rowwise_and_vectorwise_kats(m):
    q = m.rowwise_quantize(m.DenseMatrix([[1.0, -1.0], [100.0, -100.0]]))
    assert q.params.scales.tolist() == [127.0, 1.27]
    assert q.codes.data.tolist() == [[127, -127], [127, -127]]
    x = m.seeded_random_matrix(1, 10, seed=3, stddev=2.0)
    assert np.array_equal(m.rowwise_quantize(x).codes.data, m.absmax_quantize(x).codes.data)
    q = m.rowwise_quantize(m.DenseMatrix([[0.0, 0.0], [2.0, -2.0]]))
    assert q.params.scales.tolist() == [1.0, 63.5] and q.codes.data.tolist() == [[0, 0], [127, -127]]
    qx, qw = m.vectorwise_params(m.DenseMatrix(np.eye(2)), m.DenseMatrix(np.eye(2)))
    assert qx.params.scales.tolist() == [127.0, 127.0] and qw.params.scales.tolist() == [127.0, 127.0]
    assert np.array_equal(qx.codes.data, 127 * np.eye(2, dtype=np.int8))
    assert np.array_equal(qw.codes.data, 127 * np.eye(2, dtype=np.int8))
    qx, _ = m.vectorwise_params(m.DenseMatrix([[1.0, 0.0], [0.0, 10.0]]), m.DenseMatrix(np.eye(2)))
    assert qx.params.scales.tolist() == [127.0, 12.7]
    _, qw = m.vectorwise_params(m.DenseMatrix(np.eye(2)), m.DenseMatrix([[1.0, 100.0], [1.0, 100.0]]))
    assert qw.params.scales.tolist() == [127.0, 1.27]
    with pytest.raises(m.ShapeMismatchError):
        m.vectorwise_params(m.DenseMatrix(np.ones((2, 3))), m.DenseMatrix(np.ones((2, 2))))
    w = m.seeded_random_matrix(5, 4, seed=8, stddev=1.5)
    qc, qr = m.colwise_quantize(w), m.rowwise_quantize(m.DenseMatrix(w.data.T))
    assert np.array_equal(qc.codes.data, qr.codes.data.T)
    assert np.array_equal(qc.params.scales, qr.params.scales)
    xr = m.seeded_random_matrix(6, 7, seed=9, stddev=3.0)
    q = m.rowwise_quantize(xr)
    err = np.abs(m.dequantize(q).data.astype(np.float64) - xr.data)
    assert (err <= 0.5 / q.params.scales[:, None] + 1e-6).all()
    with pytest.raises(ValueError):
        m.AbsmaxParams(0.0)
    with pytest.raises(ValueError):
        m.ZeropointParams(nd=1.0, zp=2 ** 15)
    with pytest.raises(ValueError):
        m.RowwiseParams(np.array([1.0, -1.0]))


# ---------------------------------------------------------------- containers (test_tensors.py)
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_dense_matrix_rejects_non_finite(m, bad):
    with pytest.raises(ValueError, match="NaN/Inf"):
        m.DenseMatrix([[1.0, bad]])


def test_containers_contract(m):
    d = m.DenseMatrix([[1, 2], [3, 4]])
    assert d.data.dtype == np.float32 and d.shape == (2, 2) and (d.rows, d.cols) == (2, 2)
    with pytest.raises(ValueError):
        d.data[0, 0] = 5.0  # read-only
    src = np.array([[1.0, 2.0]], np.float32)
    d2 = m.DenseMatrix(src)
    src[0, 0] = 9.0
    assert d2.data[0, 0] == 1.0  # copied on construction
    for bad in (np.zeros(3), np.zeros((0, 2)), np.zeros((1, 2, 3))):
        with pytest.raises(ValueError):
            m.DenseMatrix(bad)
    v = np.float32(0.1)
    f16 = m.DenseMatrix([[v]]).to_f16_precision()
    assert f16.data[0, 0] == np.float32(np.float16(v))
    assert m.Int8Matrix([[-127, 127]]).data.tolist() == [[-127, 127]]
    for val in (128, -128):
        with pytest.raises(ValueError):
            m.Int8Matrix([[val]])
    with pytest.raises(ValueError):
        m.Int8Matrix([[1.5]])
    with pytest.raises(ValueError):
        m.Int8Matrix(torch.tensor([[-128]], dtype=torch.int8))
    m.Int32Matrix([[2 ** 31 - 1, -(2 ** 31)]])
    with pytest.raises(ValueError):
        m.Int32Matrix([[2 ** 31]])
    assert m.Int8Matrix([[1, 2]]) == m.Int8Matrix([[1, 2]])
    assert m.Int8Matrix([[1, 2]]) != m.Int8Matrix([[1, 3]])
    a = m.seeded_random_matrix(2, 2, seed=42, stddev=1.0)
    assert a == m.seeded_random_matrix(2, 2, seed=42, stddev=1.0)


# ---------------------------------------------------------------- float32 operands, reference goldens
F32 = _golden.f32_cases()


@pytest.mark.parametrize("name", sorted(F32))
def test_f32_operands_match_reference_goldens(m, name):
    """Values that are not fp16 values run the float32 kernels: every output
    bit-identical to the reference's (tests/golden/make_golden_f32.py)."""
    g = F32[name]
    x, w = m.DenseMatrix(g["x"]), m.DenseMatrix(g["w"])
    assert x.tensor16 is None  # not fp16-representable: the float32 path
    r = m.llm_int8_matmul(x, w, g["alpha"])
    assert np.array_equal(r.output.data, g["out"])
    assert r.decomposed_cols == len(g["dims"])
    assert m.extract_outlier_columns(x, g["alpha"]).dims == tuple(int(d) for d in g["dims"])
    assert np.array_equal(m.vectorwise_matmul(x, w).output.data, g["vw"])
    assert np.array_equal(m.absmax_matmul(x, w).output.data, g["absmax"])
    assert np.array_equal(m.zeropoint_matmul(x, w).output.data, g["zeropoint"])
    if "xq" in g:
        keep = _golden.keep_mask(g["x"].shape[1], g["dims"])
        qx = m.rowwise_quantize(m.DenseMatrix(g["x"][:, keep]))
        qw = m.colwise_quantize(m.DenseMatrix(g["w"][keep, :]))
        assert np.array_equal(qx.codes.data, g["xq"]) and np.array_equal(qx.params.scales, g["sx"])
        assert np.array_equal(qw.codes.data, g["wq"]) and np.array_equal(qw.params.scales, g["sw"])
        assert np.array_equal(m.int8_gemm_i32(qx.codes, qw.codes).data, g["c"])


GOLD16 = _golden.cases()


@pytest.mark.parametrize("name", sorted(GOLD16))
def test_fp16_goldens_through_the_reference_api(m, name):
    """fp16-valued float32 inputs take the production kernels (exact epilogue)."""
    g = GOLD16[name]
    x, w = m.DenseMatrix(g["x"]), m.DenseMatrix(g["w"])
    assert x.tensor16 is not None
    r = m.llm_int8_matmul(x, w, g["alpha"])
    assert np.array_equal(r.output.data, g["out"])
    assert r.decomposed_cols == int(g["decomposed_cols"])
    assert r.int8_fraction == float(g["int8_fraction"])


# ---------------------------------------------------------------- the plugin point (transformer.py:257-267)
@pytest.mark.parametrize("kind", ["llm_int8", "vectorwise", "absmax", "zeropoint"])
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_linear_rejects_non_finite(kind, bad):
    import paper_2208_07339_b200 as p

    rng = np.random.Generator(np.random.PCG64(3))
    x = rng.standard_normal((16, 64)).astype(np.float16)
    w = rng.standard_normal((64, 32)).astype(np.float16)
    xb = x.copy()
    xb[3, 7] = bad
    wb = w.copy()
    wb[5, 1] = bad
    backend = p.LinearBackend(kind)
    for xx, ww in ((xb, w), (x, wb), (xb.astype(np.float32), w.astype(np.float32)),
                   (torch.from_numpy(xb).cuda(), torch.from_numpy(w).cuda())):
        with pytest.raises(ValueError, match="NaN/Inf"):
            p.linear(xx, ww, backend)
    y = p.linear(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), backend)
    assert y.dtype == torch.float32 and bool(torch.isfinite(y).all())


def test_linear_matches_reference_transformer_linear_on_f32(oracle_mod):
    """_linear's llm_int8 kind on arbitrary float32 hidden states (the reference
    toy model's own input type) is bit-identical to the oracle."""
    import paper_2208_07339_b200 as p

    rng = np.random.Generator(np.random.PCG64(5))
    x = (rng.standard_normal((24, 96)) * 3).astype(np.float32)
    w = rng.standard_normal((96, 40)).astype(np.float32)
    ref = oracle_mod.llm_int8_matmul(x, w, 6.0)
    y = p.linear(x, w, p.llm_int8_backend(6.0))
    assert np.array_equal(y.cpu().numpy(), ref.output)


def test_int8_linear_rejects_non_finite():
    import paper_2208_07339_b200 as p

    rng = np.random.Generator(np.random.PCG64(4))
    w = torch.from_numpy(rng.standard_normal((256, 128)).astype(np.float16)).cuda()
    lin = p.Int8Linear(w)
    for mrows in (8, 300):  # decode-routed and prefill-routed
        x = torch.from_numpy(rng.standard_normal((mrows, 256)).astype(np.float16)).cuda()
        lin(x)
        x[mrows // 2, 17] = float("nan")
        with pytest.raises(ValueError, match="NaN/Inf"):
            lin(x)
        x[mrows // 2, 17] = float("inf")
        with pytest.raises(ValueError, match="NaN/Inf"):
            lin(x)
    wb = w.clone()
    wb[3, 3] = float("inf")
    with pytest.raises(ValueError, match="NaN/Inf"):
        p.Int8Linear(wb)
    with pytest.raises(ValueError, match="fp16"):
        lin(torch.full((4, 256), 0.1, dtype=torch.float32, device="cuda"))
    assert lin(torch.full((4, 256), 0.5, dtype=torch.float32, device="cuda")).shape == (4, 128)


def test_f32_inputs_never_rounded_silently(oracle_mod):
    """A float32 X whose values are not fp16 values (5.9999 would round up to
    6.0 in fp16 and become an outlier column) keeps float32 semantics."""
    import paper_2208_07339_b200 as p

    x = np.zeros((4, 64), np.float32)
    x[1, 10] = np.float32(5.9999)
    x[2, 20] = np.float32(70000.0)  # beyond the fp16 range
    w = np.random.Generator(np.random.PCG64(1)).standard_normal((64, 8)).astype(np.float32)
    assert p.extract_outlier_columns(x, 6.0).dims == (20,)
    ref = oracle_mod.llm_int8_matmul(x, w, 6.0)
    r = p.llm_int8_matmul(x, w, 6.0, exact=True)
    assert np.array_equal(r.output.cpu().numpy(), ref.output)
    assert r.decomposed_cols == 1
