"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck). Each stage checks its result
against the CPU oracle so a sanitizer run is also a correctness run.

    compute-sanitizer --tool memcheck python scripts/sanitize.py [stage ...]
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2208_07339_b200 as p  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2208_07339_b200 import _native as nat  # noqa: E402
from paper_2208_07339_b200._tensors import stream_handle  # noqa: E402


def case(seed, m, k, n, n_out=6, heavy=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((m, k)).astype(np.float32)
    cols = rng.choice(k, size=n_out, replace=False)
    x[:, cols] *= 20.0
    w = rng.standard_normal((k, n)).astype(np.float32)
    if heavy:
        w[cols[:heavy], :] *= 4.0
    return x.astype(np.float16).astype(np.float32), w.astype(np.float16).astype(np.float32)


def check(name, got, ref):
    assert np.array_equal(got, ref), name
    print(f"[ok] {name}", flush=True)


def st_functional():  # K1 scan/compact, K2 rows, K3 cols, gather, K4 (exact + fp16 + int32)
    x, w = case(1, 300, 520, 390)
    ref = orc.c_llm_int8_matmul(x, w, 6.0)
    check("llm_int8_matmul exact", p.llm_int8_matmul(x, w, exact=True).output.cpu().numpy(), ref.output)
    p.llm_int8_matmul(x, w)
    from paper_2208_07339_b200.gemm import llm_int8_trace
    tr = llm_int8_trace(x, w)
    check("int32 accumulator", tr["c"].cpu().numpy(), ref.c)


def st_module():  # weight-stationary prefill: fused prologue, fixup, patches, CTA-pair GEMM
    x, w = case(2, 600, 1024, 700, heavy=6)
    ref = orc.c_llm_int8_matmul(x, w, 6.0)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    check("Int8Linear prefill exact", lin.matmul(x16, exact=True).cpu().numpy(), ref.output)
    lin(x16)


def st_splitk():  # M <= 128, K >= 8192: split-K partial sums + counters (row-tile GEMM)
    from paper_2208_07339_b200 import _native as nat
    x, w = case(3, 64, 8192, 512, heavy=3)
    ref = orc.c_llm_int8_matmul(x, w, 6.0)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    nat.lib().i8mm_debug_set_swapab(0)
    try:
        check("split-K exact", lin.matmul(x16, exact=True).cpu().numpy(), ref.output)
        lin(x16)
    finally:
        nat.lib().i8mm_debug_set_swapab(1)


def st_swapab():  # 17 <= M <= 64: swap-AB stream-K GEMM, split tiles, patch tiles
    for seed, m, k, n, heavy in ((8, 40, 2048, 1000, 3), (9, 64, 8192, 512, 2), (10, 17, 1024, 2050, 6)):
        x, w = case(seed, m, k, n, heavy=heavy)
        ref = orc.c_llm_int8_matmul(x, w, 6.0)
        lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
        x16 = torch.from_numpy(x.astype(np.float16)).cuda()
        y = lin(x16).float().cpu().numpy()
        err = float(np.abs(y - ref.output).max())
        assert err <= 2.0 ** -10 * float(np.abs(ref.output).max()) + 1e-3, err
        print(f"[ok] swap-AB M={m} K={k} N={n} max err {err:.3g}", flush=True)


def st_decode():  # decode kernel: 8-CTA clusters, DSMEM token side + partials, stream-K, patched dots
    for seed, m, k, n, heavy in ((4, 8, 2048, 640, 2), (6, 13, 1001, 2000, 6), (7, 3, 5120, 1280, 1)):
        x, w = case(seed, m, k, n, heavy=heavy)
        ref = orc.c_llm_int8_matmul(x, w, 6.0)
        lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
        assert lin.uses_decode(m)
        x16 = torch.from_numpy(x.astype(np.float16)).cuda()
        check(f"decode exact {m}x{k}x{n}", lin.matmul(x16, exact=True).cpu().numpy(), ref.output)
        lin(x16)


def st_peers():  # fused all-gather epilogue stores into (emulated) peer buffers
    x, w = case(5, 300, 768, 500)
    lin = p.Int8Linear(torch.from_numpy(w.astype(np.float16)).cuda())
    x16 = torch.from_numpy(x.astype(np.float16)).cuda()
    y_ref = lin(x16)
    L = nat.lib()
    bufs = [torch.zeros((300, 540), dtype=torch.float16, device="cuda") for _ in range(2)]
    ptrs = (ctypes.c_void_p * 2)(*[t.data_ptr() for t in bufs])
    y = torch.empty((300, 500), dtype=torch.float16, device="cuda")
    ws = torch.empty(L.i8mm_linear_workspace_size(300, 768, 500), dtype=torch.uint8, device="cuda")
    nat.check(L.i8mm_linear_forward_peers(x16.data_ptr(), 768, 300, lin.weight.data_ptr(), 500,
                                          lin.wbuf.data_ptr(), 768, 500, 6.0, y.data_ptr(), 500,
                                          ws.data_ptr(), ws.numel(), ptrs, 2, 540, 20, stream_handle()))
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref) and all(torch.equal(b[:, 20:520], y_ref) for b in bufs)
    print("[ok] forward_peers", flush=True)


def st_siblings():  # tensor stats, scalar quantizers, zeropoint combine
    x, w = case(6, 100, 256, 120)
    check("absmax_matmul", p.absmax_matmul(x, w).output.cpu().numpy(), orc.absmax_matmul(x, w))
    check("zeropoint_matmul", p.zeropoint_matmul(x, w).output.cpu().numpy(), orc.zeropoint_matmul(x, w))


def st_f32():  # float32-operand kernels
    rng = np.random.Generator(np.random.PCG64(7))
    x = rng.standard_normal((70, 300)).astype(np.float32)
    x[:, [4, 99]] *= 20.0
    w = rng.standard_normal((300, 90)).astype(np.float32)
    check("f32 llm_int8", p.llm_int8_matmul(x, w, exact=True).output.cpu().numpy(),
          orc.llm_int8_matmul(x, w, 6.0).output)
    check("f32 vectorwise", p.vectorwise_matmul(x, w, exact=True).output.cpu().numpy(),
          orc.vectorwise_matmul(x, w))


def st_peak():
    L = nat.lib()
    nat.check(L.i8mm_peak_mma_launch(2, 4, stream_handle()))
    nat.check(L.i8mm_peak_mma_launch(1, 4, stream_handle()))
    torch.cuda.synchronize()
    print("[ok] peak kernels", flush=True)


STAGES = {k[3:]: v for k, v in list(globals().items()) if k.startswith("st_")}

if __name__ == "__main__":
    nat.load_library()
    for name in (sys.argv[1:] or list(STAGES)):
        STAGES[name]()
    torch.cuda.synchronize()
    print("ALL STAGES OK", flush=True)
