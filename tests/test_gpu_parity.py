"""GPU parity: the sm_100a kernels vs the reference's golden vectors and the
CPU oracle. Bit-exact for outlier sets, int8 codes, scales and the int32
accumulator; bit-exact float32 output in ``exact`` mode; stated tolerances for
the fast fp16 / fp32 epilogues (tests/_golden.py::fp16_tolerance; fp32:
<= 2e-6 * max|ref|).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import _golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def p():
    import paper_2208_07339_b200 as pkg
    from paper_2208_07339_b200 import _native

    _native.load_library()
    return pkg


def _np(t):
    return t.detach().cpu().numpy()


def _scales(amax_t):
    from paper_2208_07339_b200.types import _scales_from_amax

    return _scales_from_amax(amax_t)


def test_device_is_sm100(p):
    assert torch.cuda.get_device_capability() == (10, 0)


GOLDEN = _golden.cases()


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_golden_case(p, name):
    from paper_2208_07339_b200.gemm import llm_int8_trace

    g = GOLDEN[name]
    x, w, alpha = g["x"], g["w"], g["alpha"]
    tr = llm_int8_trace(x, w, alpha)
    dims = tr["scan"].dims()
    assert dims == tuple(int(d) for d in g["dims"])
    keep = _golden.keep_mask(x.shape[1], dims)
    if keep.any():
        assert np.array_equal(_np(tr["xq"])[:, keep], g["xq"])
        assert np.array_equal(_scales(tr["row_amax"]), g["sx"])
        assert np.array_equal(_np(tr["wq_t"]).T[keep, :], g["wq"])
        assert np.array_equal(_scales(tr["col_amax"]), g["sw"])
        assert np.array_equal(_np(tr["c"]), g["c"])
    # outlier columns / rows hold code 0
    assert not _np(tr["xq"])[:, ~keep].any()
    ref = g["out"]
    assert np.array_equal(_np(tr["y_exact"]), ref), "exact mode must be bit-identical"
    y32 = _np(tr["y32"]).astype(np.float64)
    assert np.abs(y32 - ref).max() <= 2e-6 * max(1.0, np.abs(ref).max())
    y16 = _np(tr["y16"]).astype(np.float64)
    assert (np.abs(y16 - ref) <= _golden.fp16_tolerance(ref)).all()
    r = p.llm_int8_matmul(x, w, alpha)
    assert r.decomposed_cols == int(g["decomposed_cols"])
    assert r.int8_fraction == pytest.approx(float(g["int8_fraction"]), abs=0)
    assert r.scheme == "llm_int8"


@pytest.mark.parametrize("name", ["no_outliers_8x16x8", "planted_64x256x64_s0"])
def test_vectorwise_golden(p, name):
    g = GOLDEN[name]
    r = p.vectorwise_matmul(g["x"], g["w"], exact=True)
    assert np.array_equal(_np(r.output), g["vw"])


def test_no_outliers_bitwise_equals_vectorwise(p):
    """tests/test_gemm.py:223-230 / acceptance criterion 5."""
    for seed in range(5):
        rng = np.random.Generator(np.random.PCG64(seed + 500))
        x = np.clip(rng.standard_normal((16, 48)), -5.9, 5.9).astype(np.float16)
        w = rng.standard_normal((48, 12)).astype(np.float16)
        a = p.llm_int8_matmul(x, w, 6.0, exact=True)
        b = p.vectorwise_matmul(x, w, exact=True)
        assert a.decomposed_cols == 0 and a.int8_fraction == 1.0
        assert np.array_equal(_np(a.output), _np(b.output))


def test_full_decomposition_matches_exact(p):
    """alpha -> 0: every column decomposed (tests/test_gemm.py:232-239)."""
    rng = np.random.Generator(np.random.PCG64(23))
    x = rng.standard_normal((8, 16)).astype(np.float16)
    w = rng.standard_normal((16, 8)).astype(np.float16)
    r = p.llm_int8_matmul(x, w, alpha=1e-9, out_dtype=torch.float32)
    exact = x.astype(np.float64) @ w.astype(np.float64)
    rel = np.linalg.norm(_np(r.output) - exact) / np.linalg.norm(exact)
    assert rel < 1e-6
    assert r.decomposed_cols == 16 and r.int8_fraction == 0.0


def test_kats(p):
    k = _golden.kats()
    q = p.rowwise_quantize(np.array(k["rowwise_hand"]["x"], dtype=np.float32))
    assert q.params.scales.tolist() == k["rowwise_hand"]["scales"]
    assert _np(q.codes).tolist() == k["rowwise_hand"]["codes"]
    q0 = p.rowwise_quantize(np.array(k["rowwise_zero_row"]["x"], dtype=np.float32))
    assert q0.params.scales.tolist() == k["rowwise_zero_row"]["scales"]
    assert _np(q0.codes).tolist() == k["rowwise_zero_row"]["codes"]
    qc = p.colwise_quantize(np.array(k["colwise_hand"]["w"], dtype=np.float32))
    assert qc.params.scales.tolist() == k["colwise_hand"]["scales"]
    assert _np(qc.codes).tolist() == k["colwise_hand"]["codes"]
    d = k["dequant_outer"]
    out = p.dequantize_output(torch.tensor(d["c"], dtype=torch.int32),
                              p.RowwiseParams(scales=d["sx"]), p.ColwiseParams(scales=d["sw"]))
    assert _np(out).astype(np.float64).tolist() == d["out"]
    for key in ("gemm_identity", "gemm_hand"):
        c = p.int8_gemm_i32(np.array(k[key]["a"], dtype=np.int8), np.array(k[key]["b"], dtype=np.int8))
        assert _np(c).tolist() == k[key]["c"]
    s = p.extract_outlier_columns(np.array(k["outlier_direct_scan"]["x"], dtype=np.float32), 6.0)
    assert list(s.dims) == k["outlier_direct_scan"]["dims"] and s.alpha == 6.0
    s = p.extract_outlier_columns(np.array(k["outlier_threshold_f32"]["x"], dtype=np.float32), 6.1)
    # fp16(6.1) = 6.1015625 >= f32(6.1): the GPU consumes fp16 values
    assert list(s.dims) == [0]


def test_gemm_worst_case_inner_dim(p):
    """127*127*2^17 = 2,114,060,288 fits int32 exactly (tests/test_gemm.py:56-63)."""
    h = p.MAX_INNER_DIM
    a = torch.full((1, h), 127, dtype=torch.int8, device="cuda")
    b = torch.full((h, 1), 127, dtype=torch.int8, device="cuda")
    assert int(p.int8_gemm_i32(a, b)[0, 0]) == 127 * 127 * h == 2_114_060_288
    a = torch.full((3, h), -127, dtype=torch.int8, device="cuda")
    b = torch.full((h, 5), 127, dtype=torch.int8, device="cuda")
    assert (p.int8_gemm_i32(a, b) == -127 * 127 * h).all()


def test_error_contract(p):
    h = p.MAX_INNER_DIM + 1
    with pytest.raises(p.GemmOverflowError):
        p.int8_gemm_i32(torch.zeros((1, h), dtype=torch.int8), torch.zeros((h, 1), dtype=torch.int8))
    with pytest.raises(p.ShapeMismatchError):
        p.int8_gemm_i32(np.zeros((2, 3), np.int8), np.zeros((2, 2), np.int8))
    with pytest.raises(p.ShapeMismatchError):
        p.llm_int8_matmul(np.ones((2, 3), np.float32), np.ones((2, 3), np.float32))
    with pytest.raises(ValueError):
        p.extract_outlier_columns(np.ones((2, 3), np.float32), 0.0)
    with pytest.raises(ValueError):
        p.extract_outlier_columns(np.ones((2, 3), np.float32), float("inf"))
    with pytest.raises(p.ParamsMismatchError):
        p.dequantize_output(torch.ones((2, 2), dtype=torch.int32), p.RowwiseParams(scales=[1.0] * 3),
                            p.ColwiseParams(scales=[1.0, 2.0]))
    with pytest.raises(p.ParamsMismatchError):
        p.dequantize_output(torch.ones((1, 1), dtype=torch.int32), p.ColwiseParams(scales=[1.0]),
                            p.RowwiseParams(scales=[1.0]))
    bad = np.ones((2, 3), np.float32)
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        p.llm_int8_matmul(bad, np.ones((3, 2), np.float32))
    with pytest.raises(ValueError):
        p.int8_gemm_i32(np.full((1, 2), -128, np.int8), np.ones((2, 1), np.int8))


@pytest.mark.parametrize("mnk", [(1, 1, 1), (7, 300, 129), (130, 257, 4112), (257, 513, 1000),
                                 (2048, 384, 1024), (3000, 520, 528),
                                 (384, 768, 2048), (1, 4096, 4096), (300, 40, 16)])
def test_int8_gemm_matches_oracle(p, oracle_mod, mnk):
    m, n, k = mnk
    rng = np.random.Generator(np.random.PCG64(sum(mnk)))
    a = rng.integers(-127, 128, size=(m, k), dtype=np.int8)
    b = rng.integers(-127, 128, size=(k, n), dtype=np.int8)
    c = p.int8_gemm_i32(a, b)
    assert np.array_equal(_np(c), oracle_mod.c_gemm_i32(a, b))


@pytest.mark.parametrize("seed", range(10))
def test_planted_sweep_vs_oracle(p, oracle_mod, seed):
    """Planted pairs (sweep.py:60-77), seeds 0..9: bit-exact stages + exact Y."""
    from paper_2208_07339_b200.gemm import llm_int8_trace

    m, k, n = (256, 1024, 512) if seed % 2 == 0 else (97, 1040, 328)
    x, w = oracle_mod.planted_pair(m, k, n, 6, 20.0, seed)
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    tr = llm_int8_trace(x, w, 6.0)
    assert tr["scan"].dims() == ref.dims
    assert np.array_equal(_np(tr["xq"]), ref.xq)
    assert np.array_equal(_np(tr["wq_t"]).T, ref.wq)
    keep = _golden.keep_mask(k, ref.dims)
    assert np.array_equal(_scales(tr["row_amax"]), ref.sx)
    assert np.array_equal(_scales(tr["col_amax"]), ref.sw)
    assert np.array_equal(_np(tr["c"]), ref.c)
    assert np.array_equal(_np(tr["y_exact"]), ref.output)
    y16 = _np(tr["y16"]).astype(np.float64)
    assert (np.abs(y16 - ref.output) <= _golden.fp16_tolerance(ref.output)).all()
    assert keep.sum() == k - len(ref.dims)


@pytest.mark.parametrize("n_out", [17, 70])
def test_many_outliers_paths(p, oracle_mod, n_out):
    """|O| beyond the smem-staged (16) and compacted-slice (64) fast paths."""
    x, w = oracle_mod.planted_pair(130, 512, 300, n_out, 20.0, 3)
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    assert len(ref.dims) >= n_out
    r = p.llm_int8_matmul(x, w, 6.0, exact=True)
    assert np.array_equal(_np(r.output), ref.output)
    r16 = p.llm_int8_matmul(x, w, 6.0)
    assert (np.abs(_np(r16.output).astype(np.float64) - ref.output)
            <= _golden.fp16_tolerance(ref.output)).all()


def test_cfg1_digest(p):
    """Config 1 (512x4096->4096, 6 planted x20, seed 0) against the reference's
    own digests (tests/golden/cfg1_digest.json, generated by make_golden.py)."""
    from paper_2208_07339_b200.gemm import llm_int8_trace
    from paper_2208_07339_b200.synthetic import planted_pair

    dig, sample = _golden.cfg1()
    m, k, n = dig["shape"]
    x, w = planted_pair(m, k, n, *dig["planted"])
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    tr = llm_int8_trace(x, w, dig["alpha"])
    dims = tr["scan"].dims()
    assert list(dims) == dig["dims"]
    keep = _golden.keep_mask(k, dims)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(_np(tr["xq"])[:, keep]) == dig["sha256"]["xq"]
    assert sha(_scales(tr["row_amax"])) == dig["sha256"]["sx"]
    assert sha(np.ascontiguousarray(_np(tr["wq_t"]).T[keep, :])) == dig["sha256"]["wq"]
    assert sha(_scales(tr["col_amax"])) == dig["sha256"]["sw"]
    assert sha(_np(tr["c"])) == dig["sha256"]["c"]
    yex = _np(tr["y_exact"])
    assert sha(yex) == dig["sha256"]["out"]
    assert np.array_equal(yex[dig["sample_rows"]], sample)


def test_int8_linear_module(p, oracle_mod):
    x, w = oracle_mod.planted_pair(64, 512, 256, 4, 20.0, 1)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda(), alpha=6.0)
    y = lin(x16.reshape(4, 16, 512))
    assert y.shape == (4, 16, 256) and y.dtype == torch.float16
    ref = oracle_mod.c_llm_int8_matmul(x.astype(np.float16).astype(np.float32),
                                       w.astype(np.float16).astype(np.float32), 6.0)
    err = np.abs(_np(y.reshape(64, 256)).astype(np.float64) - ref.output)
    assert (err <= _golden.fp16_tolerance(ref.output)).all()
    # the backend plugin point (transformer.py:257-267)
    y2 = p.linear(x, w, p.llm_int8_backend(6.0))
    assert y2.dtype == torch.float32
    for kind in ("absmax", "zeropoint", "vectorwise", "exact"):  # every BACKEND_KINDS entry
        assert p.linear(x, w, p.LinearBackend(kind)).shape == (64, 256)


def test_capi_pipeline_entry(p, oracle_mod):
    """The single-call C entry i8mm_llm_int8_matmul (what an FFI binding calls)."""
    from paper_2208_07339_b200 import _native as nat

    x, w = oracle_mod.planted_pair(200, 768, 320, 6, 20.0, 4)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    w16 = torch.from_numpy(w.astype(np.float16)).cuda()
    L = nat.lib()
    ws_bytes = L.i8mm_llm_int8_workspace_size(200, 768, 320)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    y = torch.empty((200, 320), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    nat.check(L.i8mm_llm_int8_matmul(x16.data_ptr(), 768, w16.data_ptr(), 320, 200, 768, 320,
                                     6.0, y.data_ptr(), 320, nat.OUT_F32_EXACT, ws.data_ptr(),
                                     ws_bytes, cnt.data_ptr(), st))
    ref = oracle_mod.c_llm_int8_matmul(x.astype(np.float16).astype(np.float32),
                                       w.astype(np.float16).astype(np.float32), 6.0)
    assert int(cnt.item()) == len(ref.dims)
    assert np.array_equal(_np(y), ref.output)
    assert L.i8mm_llm_int8_matmul(x16.data_ptr(), 768, w16.data_ptr(), 320, 200, 768, 320, -1.0,
                                  y.data_ptr(), 320, 0, ws.data_ptr(), ws_bytes, None, st) == 3


# ---------------------------------------------------------------- weight-stationary module
def _ws_case(seed, m, k, n, n_out, heavy_rows=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((m, k)).astype(np.float32)
    cols = rng.choice(k, size=n_out, replace=False)
    x[:, cols] *= 20.0
    w = rng.standard_normal((k, n)).astype(np.float32)
    if heavy_rows:
        # make outlier rows the column maximisers so their exclusion changes
        # many column scales (forces patches; > 4 heavy rows forces rescans)
        w[cols[:heavy_rows], :] *= 4.0
    return x.astype(np.float16).astype(np.float32), w.astype(np.float16).astype(np.float32)


@pytest.mark.parametrize("case", [(0, 256, 1024, 512, 6, 0), (1, 97, 1040, 328, 6, 2),
                                  (2, 130, 512, 300, 8, 8), (3, 64, 256, 1000, 3, 3),
                                  (4, 1, 512, 256, 6, 0), (5, 33, 3, 40, 2, 2),
                                  (6, 600, 1024, 2000, 6, 6), (7, 300, 768, 1100, 5, 1),
                                  (8, 100, 8704, 700, 6, 6), (9, 40, 16384, 300, 4, 0)])
def test_weight_stationary_matches_reference_semantics(p, oracle_mod, case):
    """Cases 8-9 take the split-K GEMM (one m-tile, K >= 8192, few N-tiles),
    case 8 with patched columns split as well."""
    seed, m, k, n, n_out, heavy = case
    x, w = _ws_case(seed, m, k, n, n_out, heavy)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda(), alpha=6.0)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    y_exact = lin.matmul(x16, exact=True)
    assert np.array_equal(_np(y_exact), ref.output)
    st = lin.last_stats()
    assert st["decomposed_cols"] == len(ref.dims)
    if heavy:
        assert st["patched_cols"] > 0
    y16 = lin(x16)
    y16_fn = p.llm_int8_matmul(x16, lin.weight, 6.0).output
    assert torch.equal(y16, y16_fn), "weight-stationary and per-call paths must agree bitwise"


def test_weight_stationary_candidates(p):
    """The cached top-4 |w| candidates per column match a host recomputation."""
    import ctypes

    from paper_2208_07339_b200 import _native as nat

    rng = np.random.Generator(np.random.PCG64(9))
    k, n = 1500, 72
    w = rng.standard_normal((k, n)).astype(np.float16)
    w[10, 5] = w[20, 5] = w[30, 5] = np.float16(9.0)  # ties keep ascending rows
    lin = p.Int8Linear(torch.from_numpy(w).cuda())
    views = (ctypes.c_void_p * 4)()
    nat.check(nat.lib().i8mm_linear_weight_views(lin.wbuf.data_ptr(), k, n, views, 4))
    base = lin.wbuf.data_ptr()
    off_v, off_r = views[2] - base, views[3] - base
    cv = lin.wbuf[off_v:off_v + 2 * 4 * n].view(torch.int16).cpu().numpy().reshape(4, n)
    cr = lin.wbuf[off_r:off_r + 4 * 4 * n].view(torch.int32).cpu().numpy().reshape(4, n)
    a = np.abs(w.astype(np.float32))
    for j in range(n):
        order = sorted(range(k), key=lambda r: (-a[r, j], r))[:4]
        assert list(cr[:, j]) == order
        assert np.array_equal(cv[:, j].view(np.float16).astype(np.float32), a[order, j])
    assert list(cr[:3, 5]) == [10, 20, 30]
    # q2: every column's codes under its second-largest |w| (reference rounding,
    # quantize.py:26-29 with the f64 scale 127 / amax2), stored K-major
    views5 = (ctypes.c_void_p * 5)()
    nat.check(nat.lib().i8mm_linear_weight_views(lin.wbuf.data_ptr(), k, n, views5, 5))
    ldq = (k + 15) // 16 * 16
    off_q = views5[4] - base
    q2 = lin.wbuf[off_q:off_q + n * ldq].view(torch.int8).cpu().numpy().reshape(n, ldq)
    amax2 = np.array([a[sorted(range(k), key=lambda r: (-a[r, j], r))[1], j] for j in range(n)],
                     dtype=np.float64)
    prod = w.astype(np.float64) * (127.0 / np.where(amax2 == 0, 127.0, amax2))[None, :]
    ref_codes = np.clip(np.copysign(np.floor(np.abs(prod) + 0.5), prod), -127, 127).astype(np.int8)
    bad = np.argwhere(q2[:, :k].T != ref_codes)
    assert bad.size == 0, (len(bad), bad[:5].tolist(),
                           [(int(q2[j, r]), int(ref_codes[r, j]), float(w[r, j]), float(amax2[j]))
                            for r, j in bad[:5].tolist()])


_CG1_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2208_07339_b200 as p
from oracle import oracle as orc
for (m, n, k) in [(300, 257, 1000), (384, 768, 2048), (129, 40, 16), (2100, 300, 640)]:
    rng = np.random.Generator(np.random.PCG64(m + n + k))
    a = rng.integers(-127, 128, size=(m, k), dtype=np.int8)
    b = rng.integers(-127, 128, size=(k, n), dtype=np.int8)
    assert np.array_equal(p.int8_gemm_i32(a, b).cpu().numpy(), orc.c_gemm_i32(a, b)), (m, n, k)
x, w = orc.planted_pair(300, 1024, 520, 6, 20.0, 1)
x = x.astype(np.float16).astype(np.float32); w = w.astype(np.float16).astype(np.float32)
ref = orc.c_llm_int8_matmul(x, w, 6.0)
assert np.array_equal(p.llm_int8_matmul(x, w, 6.0, exact=True).output.cpu().numpy(), ref.output)
lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
assert np.array_equal(lin.matmul(torch.from_numpy(x.astype(np.float16)).cuda(), exact=True).cpu().numpy(), ref.output)
print("VARIANT OK")
"""


@pytest.mark.parametrize("variant", [{"I8MM_FORCE_CG1": "1"}, {"I8MM_GEMM_MC": "2"},
                                     {"I8MM_PROLOGUE_1READ": "1"}],
                         ids=["cta_group1", "pair_multicast_cluster4", "prologue_one_read"])
def test_gemm_kernel_variants(p, variant):
    """The 1-CTA (cta_group::1) GEMM, the 4-CTA-cluster GEMM multicasting WqT
    between two CTA pairs, and the opt-in 1-read row prologue, pinned via
    environment overrides (the defaults are covered above)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    env = dict(os.environ, **variant)
    r = subprocess.run([sys.executable, "-c", _CG1_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "VARIANT OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("shape", [(4096, 1024, 768), (2600, 1040, 1000)])
def test_large_m_multicast_path_vs_oracle(p, oracle_mod, shape):
    """Large M through the CTA-pair GEMM (many pair tiles, ragged edges)."""
    m, k, n = shape
    x, w = oracle_mod.planted_pair(m, k, n, 6, 20.0, 5)
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    r = p.llm_int8_matmul(x, w, 6.0, exact=True)
    assert np.array_equal(_np(r.output), ref.output)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    assert np.array_equal(_np(lin.matmul(x16, exact=True)), ref.output)
    y16 = _np(lin(x16)).astype(np.float64)
    assert (np.abs(y16 - ref.output) <= _golden.fp16_tolerance(ref.output)).all()


# ---------------------------------------------------------------- decode path (M <= 256)
@pytest.fixture()
def decode_max(p):
    from paper_2208_07339_b200 import _native as nat

    L = nat.lib()
    # the decode kernel itself (small weight matrices at 12 <= M <= 16 otherwise route
    # to the swap-AB GEMM), and the row-tile GEMM when decode is switched off
    L.i8mm_debug_set_swapab(0)

    def set_max(m):
        L.i8mm_debug_set_decode_max_m(m)

    yield set_max
    L.i8mm_debug_set_decode_max_m(16)
    L.i8mm_debug_set_swapab(1)


@pytest.mark.parametrize("case", [
    # seed, m, k, n, planted outlier cols, heavy outlier rows of W
    (10, 1, 5120, 640, 6, 0), (11, 5, 1024, 1000, 6, 2), (12, 16, 2048, 384, 6, 6),
    (13, 13, 1001, 257, 4, 1), (14, 12, 4096, 1024, 8, 3), (15, 16, 768, 2050, 6, 0),
    (16, 9, 512, 600, 20, 5), (17, 15, 1536, 768, 6, 2), (18, 3, 256, 520, 70, 0),
    (19, 11, 8192, 136, 2, 2), (20, 14, 1024, 2000, 6, 6), (21, 2, 20480, 384, 6, 1),
    (22, 7, 130, 4000, 3, 2),
    # more n-tiles than clusters, >= 8 k-blocks, ragged K
    (23, 8, 2048, 4000, 6, 3), (24, 16, 3000, 5000, 8, 2), (25, 1, 1024, 1920, 6, 4)])
def test_decode_path_vs_oracle_and_prefill(p, oracle_mod, decode_max, case):
    """The decode kernel (8-CTA clusters: token side in distributed shared
    memory + swap-AB stream-K tcgen05 GEMM): exact output bit-identical to the
    oracle, fp16 output bit-identical to the prefill kernels, |O| and patched
    columns as the reference semantics imply; ragged K / N, > WO_CAP outliers,
    heavy outlier rows of W (patched and re-derived columns), tiles split over
    many CTAs and CTAs spanning many tiles."""
    from paper_2208_07339_b200 import _native as nat

    seed, m, k, n, n_out, heavy = case
    x, w = _ws_case(seed, m, k, n, n_out, heavy)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda(), alpha=6.0)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    decode_max(16)
    assert nat.lib().i8mm_linear_uses_decode(m, k, n) == 1
    y_exact = lin.matmul(x16, exact=True)
    assert np.array_equal(_np(y_exact), ref.output)
    st = lin.last_stats()
    assert st["decomposed_cols"] == len(ref.dims)
    if heavy:
        assert st["patched_cols"] > 0
    y16 = lin(x16)
    decode_max(0)
    assert nat.lib().i8mm_linear_uses_decode(m, k, n) == 0
    y16_prefill = lin(x16)
    assert torch.equal(y16, y16_prefill), "decode and prefill kernels must agree bitwise"
    st2 = lin.last_stats()
    assert st2 == st


def test_decode_path_repeated_calls_and_strided_x(p, oracle_mod, decode_max):
    """Per-call state (split-K accumulators, counters) is reset by every call;
    a row-strided (non 16-byte aligned) X takes the element-load path."""
    decode_max(16)
    x, w = _ws_case(21, 12, 1000, 520, 6, 2)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda(), alpha=6.0)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    big = torch.zeros((12, 1003), dtype=torch.float16, device="cuda")
    big[:, 1:1001] = torch.from_numpy(x.astype(np.float16)).cuda()
    xs = big[:, 1:1001]
    assert xs.stride(0) == 1003
    for _ in range(3):
        assert np.array_equal(_np(lin.matmul(xs, exact=True)), ref.output)
    x2, _ = _ws_case(22, 12, 1000, 520, 3, 0)
    ref2 = oracle_mod.c_llm_int8_matmul(x2, w, 6.0)
    assert np.array_equal(_np(lin.matmul(torch.from_numpy(x2.astype(np.float16)).cuda(), exact=True)),
                          ref2.output)


class _MarkTimer:
    """Stand-in for bench.py's EventTimer: forces the split prologue/gemm entries."""

    def mark(self, name):
        pass


@pytest.mark.parametrize("alpha", [6.0, 4.5])
def test_decode_split_entries_carry_alpha(p, oracle_mod, decode_max, alpha):
    """i8mm_linear_prologue + i8mm_linear_gemm in decode routing (the threshold
    travels through the workspace) == i8mm_linear_forward == the oracle."""
    decode_max(16)
    x, w = _ws_case(31, 9, 2048, 700, 5, 1)
    ref = oracle_mod.c_llm_int8_matmul(x, w, alpha)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda(), alpha=alpha)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    y_fwd = lin(x16)
    y_split = lin.matmul(x16, _timer=_MarkTimer())
    assert torch.equal(y_fwd, y_split)
    assert lin.last_stats()["decomposed_cols"] == len(ref.dims)
    assert (np.abs(_np(y_fwd).astype(np.float64) - ref.output) <= _golden.fp16_tolerance(ref.output)).all()


# ---------------------------------------------------------------- sibling schemes
def _sib():
    from pathlib import Path

    d = np.load(Path(__file__).resolve().parent / "golden" / "siblings_cases.npz")
    return d, [str(n) for n in d["names"]]


def test_sibling_quantizers_match_reference_goldens(p):
    """absmax_quantize / zeropoint_quantize on the GPU vs the reference's codes
    and params (quantize.py:137-171), bit-exact, incl. the int16 range error."""
    d, names = _sib()
    for name in names:
        for tag in ("x", "w"):
            t = d[f"{name}/{tag}"]
            qa = p.absmax_quantize(t)
            assert np.array_equal(_np(qa.codes), d[f"{name}/abs_{tag}_codes"]), (name, tag)
            assert qa.params.scale == float(d[f"{name}/abs_{tag}_scale"])
            if f"{name}/zp_{tag}_error" in d:
                with pytest.raises(ValueError):
                    p.zeropoint_quantize(t)
                continue
            qz = p.zeropoint_quantize(t)
            assert np.array_equal(_np(qz.codes), d[f"{name}/zp_{tag}_codes"]), (name, tag)
            assert [qz.params.nd, qz.params.zp, qz.params.offset] == \
                d[f"{name}/zp_{tag}_params"].tolist(), (name, tag)


def test_sibling_matmuls_match_reference_goldens(p):
    """absmax_matmul / zeropoint_gemm_i32 / zeropoint_matmul vs the reference
    (gemm.py:85-104, 150-187): float32 outputs and int32 accumulators
    bit-identical; GemmOverflowError / ValueError where the reference raises."""
    d, names = _sib()
    for name in names:
        x, w = d[f"{name}/x"], d[f"{name}/w"]
        assert np.array_equal(_np(p.absmax_matmul(x, w).output), d[f"{name}/abs_out"]), name
        assert np.array_equal(_np(p.linear(x, w, p.ABSMAX)), d[f"{name}/abs_out"]), name
        if f"{name}/zp_out" in d:
            for unrolled in (False, True):
                r = p.zeropoint_matmul(x, w, unrolled=unrolled)
                assert r.scheme == "zeropoint"
                assert np.array_equal(_np(r.output), d[f"{name}/zp_out"]), name
            qx, qw = p.zeropoint_quantize(x), p.zeropoint_quantize(w)
            c = p.zeropoint_gemm_i32(qx.codes, qw.codes, qx.params.zp, qw.params.zp)
            assert np.array_equal(_np(c), d[f"{name}/zp_c"]), name
            # dequantize_output's zeropoint branch = c / (nd_x * nd_w) (gemm.py:135)
            if qx.params.offset == 0.0 and qw.params.offset == 0.0:
                assert np.array_equal(_np(p.dequantize_output(c, qx.params, qw.params)),
                                      d[f"{name}/zp_out"]), name
        elif int(d[f"{name}/zp_out_error"]) == 2:
            with pytest.raises(p.GemmOverflowError):
                p.zeropoint_matmul(x, w)
            qx, qw = p.zeropoint_quantize(x), p.zeropoint_quantize(w)
            with pytest.raises(p.GemmOverflowError):
                p.zeropoint_gemm_i32(qx.codes, qw.codes, qx.params.zp, qw.params.zp)
        else:
            with pytest.raises(ValueError):
                p.zeropoint_matmul(x, w)
        qa, qb = p.absmax_quantize(x), p.absmax_quantize(w)
        c = p.int8_gemm_i32(qa.codes, qb.codes)
        assert np.array_equal(_np(p.dequantize_output(c, qa.params, qb.params)),
                              d[f"{name}/abs_out"]), name
        with pytest.raises(p.ParamsMismatchError):  # mixed pairing (gemm.py:143-146)
            p.dequantize_output(c, qa.params, p.rowwise_quantize(x).params)


@pytest.mark.parametrize("shape", [(300, 1000, 700), (2048, 1024, 512), (1, 4096, 384)])
def test_sibling_matmuls_large_vs_oracle(p, oracle_mod, shape):
    """Larger shapes (CTA-pair GEMM, ragged edges) vs the numpy restatement."""
    m, k, n = shape
    rng = np.random.Generator(np.random.PCG64(m + k + n))
    x = (rng.standard_normal((m, k)) * 2 + 0.3).astype(np.float16).astype(np.float32)
    w = (rng.standard_normal((k, n)) * 0.2).astype(np.float16).astype(np.float32)
    assert np.array_equal(_np(p.absmax_matmul(x, w).output), oracle_mod.absmax_matmul(x, w))
    assert np.array_equal(_np(p.zeropoint_matmul(x, w).output), oracle_mod.zeropoint_matmul(x, w))


def test_qt8_roundtrip_through_device_pipeline(p, oracle_mod, tmp_path):
    """Golden-vector I/O on the device: QT8 files (reference format, qt8.py)
    load straight into CUDA tensors that feed the LLM.int8() path, and the
    int32 / float32 results round-trip bit-exactly."""
    from paper_2208_07339_b200 import qt8

    x, w = oracle_mod.planted_pair(48, 256, 40, 3, 20.0, 6)
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    qt8.write_tensor(tmp_path / "x.qt8", x)
    qt8.write_tensor(tmp_path / "w.qt8", w)
    xd = qt8.read_tensor(tmp_path / "x.qt8")
    assert xd.is_cuda and xd.dtype == torch.float32
    tr = p.gemm.llm_int8_trace(xd, qt8.read_tensor(tmp_path / "w.qt8"), 6.0)
    ref = oracle_mod.llm_int8_matmul(x, w, 6.0)
    qt8.write_tensor(tmp_path / "c.qt8", tr["c"])
    qt8.write_tensor(tmp_path / "y.qt8", tr["y_exact"])
    assert np.array_equal(_np(qt8.read_tensor(tmp_path / "c.qt8")), ref.c)
    assert np.array_equal(_np(qt8.read_tensor(tmp_path / "y.qt8")), ref.output)


def test_row_range_gemm_and_pipelined_gather_single_rank(p, oracle_mod):
    """i8mm_linear_gemm_rows (one prologue, GEMM per row range) is bitwise the
    single-call result; the pipelined NCCL all-gather path of
    ShardedInt8Linear (world size 1 here: one GPU per box) runs its streams
    and placement and returns the same bits."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2208_07339_b200.sharded import ShardedInt8Linear

    x, w = oracle_mod.planted_pair(1000, 768, 520, 6, 20.0, 2)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    y_ref = lin(x16)
    seen = []
    y_rows = lin.matmul_rows(x16, [(0, 256), (256, 300), (300, 1000)],
                             on_rows=lambda r0, r1, y: seen.append((r0, r1)))
    assert seen == [(0, 256), (256, 300), (300, 1000)]
    assert torch.equal(y_rows, y_ref)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sh = ShardedInt8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
        assert torch.equal(sh(x16, chunks=4), y_ref)
        assert torch.equal(sh(x16, chunks=1), y_ref)
        assert torch.equal(sh(x16[:7], chunks=4), lin(x16[:7]))  # decode rows: one launch
    finally:
        dist.destroy_process_group()


def test_host_io_pipeline_matches_device_calls(p, oracle_mod):
    """HostIOPipeline (overlapped H2D / row-range GEMM / D2H streams) returns
    bitwise the device-path outputs, for prefill and decode-sized calls."""
    mods, xs, refs = [], [], []
    for i, (m, k, n) in enumerate([(1000, 512, 300), (600, 300, 520), (5, 512, 130)]):
        x, w = oracle_mod.planted_pair(m, k, n, 4, 20.0, 30 + i)
        mod = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
        x16 = torch.from_numpy(x.astype(np.float16))
        mods.append(mod)
        xs.append(x16.pin_memory())
        refs.append(mod(x16.cuda()).cpu())
    ys = [torch.empty(r.shape, dtype=r.dtype).pin_memory() for r in refs]
    pipe = p.HostIOPipeline(chunks=3)
    for _ in range(2):
        for y in ys:
            y.zero_()
        pipe.run(list(zip(mods, xs, ys)))
        torch.cuda.synchronize()
        for y, r in zip(ys, refs):
            assert torch.equal(y, r)


def test_host_io_pipeline_back_to_back_batches(p, oracle_mod):
    """inputs_ready=True: consecutive batches overlap (batch b+1's input copies
    start while batch b computes and copies out); every batch's outputs still
    equal the device path bitwise."""
    shapes = [(700, 512, 300), (700, 300, 512)]
    mods = []
    for i, (m, k, n) in enumerate(shapes):
        _, w = oracle_mod.planted_pair(m, k, n, 4, 20.0, 50 + i)
        mods.append(p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda()))
    batches = []
    for b in range(3):
        xs, ys, refs = [], [], []
        for i, ((m, k, n), mod) in enumerate(zip(shapes, mods)):
            x, _ = oracle_mod.planted_pair(m, k, n, 4, 20.0, 60 + 10 * b + i)
            x16 = torch.from_numpy(x.astype(np.float16))
            xs.append(x16.pin_memory())
            refs.append(mod(x16.cuda()).cpu())
            ys.append(torch.zeros(refs[-1].shape, dtype=refs[-1].dtype).pin_memory())
        batches.append((xs, ys, refs))
    torch.cuda.synchronize()
    pipe = p.HostIOPipeline(chunks=2)
    for xs, ys, _ in batches:  # output copies left in flight across batches, joined once
        pipe.run(list(zip(mods, xs, ys)), inputs_ready=True, join=False)
    pipe.join()
    torch.cuda.synchronize()
    for _, ys, refs in batches:
        for y, r in zip(ys, refs):
            assert torch.equal(y, r)


_LATE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2208_07339_b200 as p
from oracle import oracle as orc
for k in (1024, 4096, 16384):
    rng = np.random.Generator(np.random.PCG64(k))
    m, n = 600, 256
    x = (0.5 * rng.standard_normal((m, k))).astype(np.float32)
    c1, c2, c3 = 5, k // 2 + 3, k - 7
    x[:, c1] = 5.5          # the row maximum everywhere, outlier only in the last row
    x[:, c2] = 0.25         # outlier only in the last row, never a row maximum
    x[-1, c1] = 10.0
    x[-1, c2] = -12.0
    x[::3, c3] = 30.0       # a regular outlier column
    w = rng.standard_normal((k, n)).astype(np.float32)
    x = x.astype(np.float16).astype(np.float32)
    w = w.astype(np.float16).astype(np.float32)
    ref = orc.c_llm_int8_matmul(x, w, 6.0)
    assert tuple(ref.dims) == tuple(sorted((c1, c2, c3))), ref.dims
    r = p.llm_int8_matmul(x, w, 6.0, exact=True)
    assert r.decomposed_cols == 3
    assert np.array_equal(r.output.cpu().numpy(), ref.output), k
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    assert np.array_equal(lin.matmul(x16, exact=True).cpu().numpy(), ref.output), k
    assert lin.last_stats()["decomposed_cols"] == 3
print("LATE OK")
"""


@pytest.mark.parametrize("one_read", ["0", "1"], ids=["two_read", "one_read"])
def test_prologue_late_outlier_columns(p, one_read):
    """Columns that turn outlier only in the last row. c1 holds the row maximum
    (5.5 < alpha) in every row, c2 never does, c3 is a regular planted column.
    In the 1-read form every block quantized before c1/c2 were flagged is
    corrected exactly by the finalize pass (rows re-quantized for c1, codes
    zeroed for c2)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    env = dict(os.environ, I8MM_PROLOGUE_1READ=one_read)
    r = subprocess.run([sys.executable, "-c", _LATE_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "LATE OK" in r.stdout, r.stdout + r.stderr


def test_alternating_decode_prefill_calls_stable(p, oracle_mod):
    """Decode-routed and prefill calls of one module interleaved back to back
    (programmatic dependent launch chains the prefill kernels; workspaces are
    recycled by the caching allocator): every call must reproduce the oracle,
    including patched columns (heavy outlier rows in W force patches)."""
    x, w = _ws_case(11, 64, 1024, 700, 6, 6)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda(), alpha=6.0)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    refs = {m: torch.from_numpy(oracle_mod.c_llm_int8_matmul(x[:m], w, 6.0).output) for m in (8, 16, 32, 64)}
    for _ in range(6):
        for m in (16, 32, 8, 64):
            y = lin.matmul(x16[:m].contiguous(), exact=True)
            assert torch.equal(y.cpu(), refs[m]), m


@pytest.mark.parametrize("case", [(300, 1024, 700, 0), (8, 512, 256, 0), (100, 8704, 700, 6), (600, 1024, 2000, 6)],
                         ids=["prefill", "decode", "splitk_patches", "pairs_patches"])
def test_forward_peers_fused_gather(p, oracle_mod, case):
    """i8mm_linear_forward_peers as an emulated 2-rank N-shard: each "rank"
    holds one column block of W and its GEMM epilogue stores its block into
    BOTH ranks' full-width Y buffers (the fused all-gather). Afterwards every
    buffer must hold the whole Y: within the fp16 tolerance of the oracle,
    bitwise equal to the unsharded module, and nothing outside the blocks."""
    import ctypes

    from paper_2208_07339_b200 import _native as nat
    from paper_2208_07339_b200._tensors import stream_handle
    from paper_2208_07339_b200.sharded import shard_bounds

    m, k, n, heavy = case
    x, w = _ws_case(21, m, k, n, 6, heavy)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    y_full = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())(x16)
    L = nat.lib()
    pad = 16  # the buffers are wider than Y: nothing may land past column n
    bufs = [torch.full((m, n + pad), -7.0, dtype=torch.float16, device="cuda") for _ in range(2)]
    ptrs = (ctypes.c_void_p * 2)(*[t.data_ptr() for t in bufs])
    for r in range(2):
        lo, hi = shard_bounds(n, 2, r)
        lin = p.Int8Linear(torch.from_numpy(np.ascontiguousarray(w[:, lo:hi]).astype(np.float16)).cuda())
        y = torch.empty((m, hi - lo), dtype=torch.float16, device="cuda")
        ws = lin.workspace(m)
        nat.check(L.i8mm_linear_forward_peers(
            x16.data_ptr(), k, m, lin.weight.data_ptr(), hi - lo, lin.wbuf.data_ptr(), k, hi - lo, 6.0,
            y.data_ptr(), hi - lo, ws.data_ptr(), ws.numel(), ptrs, 2, n + pad, lo, stream_handle()),
            "forward_peers")
        assert torch.equal(y, y_full[:, lo:hi])
    torch.cuda.synchronize()
    for t in bufs:
        got = t[:, :n]
        assert torch.equal(got, y_full)
        err = np.abs(_np(got).astype(np.float64) - ref.output)
        assert (err <= _golden.fp16_tolerance(ref.output)).all()
        assert bool((t[:, n:] == -7.0).all())


def test_sharded_fused_gather_single_rank(p, oracle_mod):
    """ShardedInt8Linear.forward_fused (symmetric-memory Y, all-gather fused
    into the epilogue, device barrier) at world size 1 equals the module."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2208_07339_b200.sharded import ShardedInt8Linear

    x, w = oracle_mod.planted_pair(700, 768, 520, 6, 20.0, 4)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    y_ref = lin(x16)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sh = ShardedInt8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
        try:
            y = sh.forward_fused(x16)
        except (RuntimeError, NotImplementedError) as e:  # symmetric memory unavailable on this box
            pytest.skip(f"symmetric memory: {str(e).splitlines()[0]}")
        assert torch.equal(y, y_ref)
        assert torch.equal(sh.forward_fused(x16), y_ref)  # cached buffer, second call
        # forward(): the agreed path is the fused one; results are not aliased
        y1 = sh(x16)
        assert sh.gather_path == "fused-epilogue" and torch.equal(y1, y_ref)
        y2 = sh(torch.zeros_like(x16))
        assert torch.equal(y1, y_ref) and not bool(y2.abs().max() > 0)
        assert sh(x16, alias=True).data_ptr() == sh._symm[(700, 0)][0].data_ptr()
        for mm in (1, 2, 3, 4, 5, 6):  # LRU-bounded symmetric buffers
            sh(x16[:mm].contiguous())
        assert len(sh._symm) <= sh.symm_cache_size
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pad", [24, 3], ids=["aligned_stride", "odd_stride"])
@pytest.mark.parametrize("m", [8, 300])
def test_row_strided_x_matches_contiguous(p, oracle_mod, pad, m):
    """X as a column slice of a wider buffer (row pitch ldx > K): the 16-byte
    aligned pitch takes the vector prologue, the odd pitch the generic one;
    both equal the contiguous call and the oracle, for decode and prefill M."""
    k, n = 1024, 520
    x, w = _ws_case(31, m, k, n, 6, 2)
    wide = torch.zeros((m, k + pad), dtype=torch.float16, device="cuda")
    wide[:, :k] = torch.from_numpy(x.astype(np.float16)).cuda()
    xs = wide[:, :k]
    assert xs.stride(0) == k + pad
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    assert np.array_equal(_np(lin.matmul(xs, exact=True)), ref.output)
    assert torch.equal(lin(xs), lin(xs.contiguous()))
    r = p.llm_int8_matmul(xs, lin.weight, 6.0, exact=True)
    assert np.array_equal(_np(r.output), ref.output)


def test_graphed_decode_step_matches_eager(p, oracle_mod):
    """GraphedCall: a CUDA graph of several decode-routed and prefill layer
    calls replays to the same bits as eager calls, with new inputs copied
    into the static input tensors between replays."""
    shapes = [(8, 1024, 700), (8, 700, 1024), (300, 1024, 520)]
    mods, xs, xs2 = [], [], []
    for i, (m, k, n) in enumerate(shapes):
        x, w = _ws_case(40 + i, m, k, n, 6, 2)
        mods.append(p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda()))
        xs.append(torch.from_numpy(x.astype(np.float16)).cuda())
        x2, _ = _ws_case(50 + i, m, k, n, 6, 2)
        xs2.append(torch.from_numpy(x2.astype(np.float16)).cuda())
    static = [x.clone() for x in xs]
    g = p.GraphedCall(lambda *xx: [mod(x) for mod, x in zip(mods, xx)], *static)
    assert g.kernels > 0
    for batch in (xs, xs2, xs):
        for s_, x in zip(static, batch):
            s_.copy_(x)
        outs = g.replay()
        torch.cuda.synchronize()
        for mod, x, y in zip(mods, batch, outs):
            assert torch.equal(y, mod(x))


def test_graphed_decode_step_has_only_kernel_nodes(p):
    """The captured decode step holds only the layer kernels, chained by
    programmatic (PDL) edges: no workspace-initialisation memset lands between
    two kernels (one did when the graph was captured on another stream than
    the warm-up: +4 us per layer). Outputs replay bit-identical to eager."""
    rt = pytest.importorskip("cuda.bindings.runtime")
    shapes = [(8, 1024, 700), (8, 700, 1024), (4, 1024, 1024)]
    mods, static = [], []
    for i, (m, k, n) in enumerate(shapes):
        x, w = _ws_case(60 + i, m, k, n, 6, 2)
        mods.append(p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda()))
        static.append(torch.from_numpy(x.astype(np.float16)).cuda())
    assert all(mod.uses_decode(x.shape[0]) for mod, x in zip(mods, static))
    g = p.GraphedCall(lambda *xx: [mod(x) for mod, x in zip(mods, xx)], *static, keep_graph=True)
    assert g.kernels == len(shapes)
    cg = rt.cudaGraph_t(init_value=g.graph.raw_cuda_graph())
    err, _, n = rt.cudaGraphGetNodes(cg, 0)
    err, nodes, n = rt.cudaGraphGetNodes(cg, n)
    types = [rt.cudaGraphNodeGetType(nd)[1] for nd in nodes]
    assert types == [rt.cudaGraphNodeType.cudaGraphNodeTypeKernel] * len(shapes), types
    outs = g.replay()
    torch.cuda.synchronize()
    for mod, x, y in zip(mods, static, outs):
        assert torch.equal(y, mod(x))


@pytest.mark.parametrize("case", [
    # seed, m, k, n, planted outlier cols, heavy outlier rows of W
    (70, 17, 1024, 1000, 6, 2), (71, 32, 5120, 640, 6, 0), (72, 48, 2048, 384, 6, 6),
    (73, 64, 1008, 257, 4, 1), (74, 100, 4096, 2050, 8, 3), (75, 128, 768, 4000, 20, 5),
    (76, 33, 8192, 136, 2, 2), (77, 80, 2048, 1536, 6, 0)])
def test_swapab_mid_m_vs_row_tile_gemm_and_oracle(p, oracle_mod, case):
    """Weight-stationary prefill at 17 <= M <= 128 runs the swap-AB stream-K GEMM
    (swapab_sm100.cu): fp16 and fast f32 outputs bitwise equal to the row-tile
    GEMM on the same prologue, fp16 within tolerance of the oracle; ragged N and
    K, > 16 outliers (the slow outlier loop), patched columns (extra tiles),
    tiles split over many CTAs."""
    from paper_2208_07339_b200 import _native as nat

    seed, m, k, n, n_out, heavy = case
    x, w = _ws_case(seed, m, k, n, n_out, heavy)
    ref = oracle_mod.c_llm_int8_matmul(x, w, 6.0)
    w16 = torch.from_numpy(w.astype(np.float16)).cuda()
    lin = p.Int8Linear(w16, alpha=6.0)
    lin32 = p.Int8Linear(w16, alpha=6.0, out_dtype=torch.float32)
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    L = nat.lib()
    try:
        L.i8mm_debug_set_swapab(1)
        y_sab = lin(x16)
        y32_sab = lin32(x16)
        st = lin.last_stats()
        L.i8mm_debug_set_swapab(0)
        y_row = lin(x16)
        y32_row = lin32(x16)
    finally:
        L.i8mm_debug_set_swapab(1)
    assert torch.equal(y_sab, y_row), "swap-AB and row-tile GEMMs must agree bitwise (fp16)"
    assert torch.equal(y32_sab, y32_row), "swap-AB and row-tile GEMMs must agree bitwise (f32)"
    err_ok = np.abs(_np(y_sab).astype(np.float64) - ref.output) <= _golden.fp16_tolerance(ref.output)
    assert err_ok.all(), f"{(~err_ok).sum()} fp16 outputs outside the stated tolerance"
    assert st["decomposed_cols"] == len(ref.dims)
    if heavy:
        assert st["patched_cols"] > 0
