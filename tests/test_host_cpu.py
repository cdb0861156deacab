"""CPU-only checks: the C ABI library exports every declared symbol, the host
logic of the API (error contract, backend plugin point), and the N-shard
all-gather reassembly under gloo with world size 2 (oracle as per-shard compute)."""

from __future__ import annotations

import os
import re
import socket
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols() -> set[str]:
    text = (ROOT / "include" / "llmint8.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(i8mm_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    from paper_2208_07339_b200 import _native

    lib = _native.LIB_PATH
    assert lib.exists(), "build the library first (python -m paper_2208_07339_b200.build)"
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    declared = _declared_symbols()
    assert declared, "no declarations parsed"
    missing = declared - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    assert declared == set(_native.EXPORTED_SYMBOLS)
    # loads without a GPU and answers host-only queries
    L = _native.load_library()
    assert L.i8mm_version() == 1
    assert L.i8mm_status_string(2).decode().startswith("inner dimension")
    assert L.i8mm_llm_int8_workspace_size(512, 4096, 4096) > 512 * 4096 + 4096 * 4096
    assert L.i8mm_linear_weight_bytes(4096, 4096) >= 4096 * 4096


def test_library_is_sm100a_tcgen05():
    """The shipped code is sm_100a SASS with tcgen05 MMA (incl. CTA pairs), TMEM
    loads, TMA loads and TMA stores (the fp16 epilogue), and the bulk-copy (UBLKCP)
    ring that feeds the row quantizer."""
    from paper_2208_07339_b200 import _native

    r = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = r.stdout
    assert "sm_100a" in sass
    for mnemonic in ("UTCIMMA", "LDTM", "UTMALDG", "UTMASTG", "UTCIMMA.2CTA", "UBLKCP"):
        assert mnemonic in sass, mnemonic
    # no dev instrumentation in the shipped kernels (timeline stamps / wait-cycle
    # counters live in the `build.py --devtools` library only): even untaken, their
    # branches cost the GEMM 13-15 % (profiles/r1/gemm_ncu_cfg2_r1f.md)
    for reg in ("SR_GLOBALTIMER", "SR_CLOCK"):
        assert reg not in sass, reg


def test_backend_plugin_validation():
    import paper_2208_07339_b200 as p

    assert p.BACKEND_KINDS == ("exact", "absmax", "zeropoint", "vectorwise", "llm_int8")
    assert p.llm_int8_backend(5.0) == p.LinearBackend("llm_int8", 5.0)
    with pytest.raises(ValueError):
        p.LinearBackend("nope")
    with pytest.raises(ValueError):
        p.LinearBackend("llm_int8", 0.0)
    s = p.OutlierSet((5, 1, 3), 6.0)
    assert s.dims == (1, 3, 5) and len(s) == 3 and 3 in s
    with pytest.raises(ValueError):
        p.OutlierSet((1, 1), 6.0)
    with pytest.raises(ValueError):
        p.OutlierSet((1,), float("inf"))
    with pytest.raises(ValueError):
        p.RowwiseParams(scales=[1.0, -2.0])
    assert issubclass(p.ShapeMismatchError, ValueError)
    assert issubclass(p.GemmOverflowError, ValueError)
    assert issubclass(p.ParamsMismatchError, ValueError)
    assert p.MAX_INNER_DIM == 1 << 17


def test_planted_pair_matches_reference_generator(oracle_mod):
    from paper_2208_07339_b200.synthetic import planted_pair

    a = planted_pair(16, 64, 8, 2, 20.0, 3)
    b = oracle_mod.planted_pair(16, 64, 8, 2, 20.0, 3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_product_path_fails_loudly_without_gpu():
    import paper_2208_07339_b200 as p
    from paper_2208_07339_b200._native import NativeLibraryError

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(NativeLibraryError):
        p.llm_int8_matmul(np.ones((2, 3), np.float32), np.ones((3, 2), np.float32))


def test_shard_bounds():
    from paper_2208_07339_b200.sharded import shard_bounds

    for n in (1, 7, 16, 49152, 36865):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, str(ROOT))
        from oracle import oracle as orc
        from paper_2208_07339_b200.sharded import gather_columns, shard_bounds

        m, k, n = 24, 96, 37  # ragged N: shards of 19 / 18 columns
        x, w = orc.planted_pair(m, k, n, 3, 20.0, 11)
        x = x.astype(np.float16).astype(np.float32)
        w = w.astype(np.float16).astype(np.float32)
        lo, hi = shard_bounds(n, world, rank)
        # per-shard compute: the CPU oracle of the reference path on W[:, lo:hi]
        local = orc.c_llm_int8_matmul(x, w[:, lo:hi], 6.0).output
        y = gather_columns(torch.from_numpy(local), n)
        full = orc.c_llm_int8_matmul(x, w, 6.0).output
        ok = bool(np.array_equal(y.numpy(), full))
        # the pipelined gather: row ranges of the padded local block pushed as
        # they would be produced (one prologue over all rows, then per range)
        from paper_2208_07339_b200.sharded import _GatherPipeline, row_ranges

        width = -(-n // world)
        y_pad = torch.zeros((m, width), dtype=torch.float32)
        y_pad[:, : hi - lo] = torch.from_numpy(local)
        pipe = _GatherPipeline(m, n, width, torch.float32, torch.device("cpu"), None)
        for r0, r1 in [(0, 5), (5, 13), (13, 24)]:
            pipe.push(r0, r1, y_pad)
        ok = ok and bool(np.array_equal(pipe.finish().numpy(), full))
        ok = ok and row_ranges(1000, 4) == [(0, 250), (250, 500), (500, 750), (750, 1000)]
        ok = ok and row_ranges(16384, 4) == [(0, 4096), (4096, 8192), (8192, 12288), (12288, 16384)]
        ok = ok and row_ranges(300, 4) == [(0, 150), (150, 300)]
        ok = ok and row_ranges(100, 4) == [(0, 100)]
        result_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_nshard_allgather_gloo_world2():
    """N-sharding is exact: per-column math is independent of the shard
    (SURVEY.md 8e), so the gathered output equals the unsharded oracle bitwise."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
    results = sorted(q.get(timeout=5) for _ in range(world))
    assert results == [(0, True), (1, True)]


def test_qt8_mirror_matches_reference_files(tmp_path):
    """QT8 reader/writer vs files written by the reference (qt8.py:65-107):
    identical bytes on re-write, identical error classes on malformed files."""
    import numpy as np
    import torch

    from paper_2208_07339_b200 import qt8

    gold = Path(__file__).resolve().parent / "golden" / "qt8"
    for name, dt in (("f32", torch.float32), ("i8", torch.int8), ("i32", torch.int32)):
        t = qt8.read_tensor(gold / f"{name}.qt8", device="cpu")
        assert t.dtype == dt and t.ndim == 2
        qt8.write_tensor(tmp_path / f"{name}.qt8", t)
        assert (tmp_path / f"{name}.qt8").read_bytes() == (gold / f"{name}.qt8").read_bytes()
    # fp16 tensors widen to f32 exactly
    h = torch.tensor([[1.5, -2.25]], dtype=torch.float16)
    qt8.write_tensor(tmp_path / "h.qt8", h)
    assert torch.equal(qt8.read_tensor(tmp_path / "h.qt8", device="cpu"), h.float())
    for bad, exc in (("bad_magic", qt8.BadMagicError), ("bad_version", qt8.UnsupportedVersionError),
                     ("bad_dtype", qt8.UnknownDtypeError), ("short_header", qt8.TruncatedFileError),
                     ("short_payload", qt8.TruncatedFileError), ("trailing", qt8.QT8Error)):
        with pytest.raises(exc):
            qt8.read_tensor(gold / f"{bad}.qt8", device="cpu")
    with pytest.raises(TypeError):
        qt8.write_tensor(tmp_path / "x.qt8", np.zeros((2, 2), dtype=np.float64))
