"""Interleaved A/B timing of GEMM kernel variants (dev tool)."""
import statistics, sys
import torch
sys.path.insert(0, ".")
from paper_2208_07339_b200 import gemm as G, _native as nat
from paper_2208_07339_b200.synthetic import planted_pair_device

L = nat.lib()
st = lambda: torch.cuda.current_stream().cuda_stream

def timeit(fn, iters=20):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

shapes = [(16384, 4096, 16384), (16384, 16384, 4096), (16384, 12288, 49152)]
variants = [("pair", (0, 1)), ("pair+mc", (0, 0))]
for (m, k, n) in shapes:
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
    scan = G.scan_outliers(x, 6.0)
    xq, ldq, ax, xo = G._quantize_rows(x, scan)
    wq, _, aw = G._quantize_cols_t(w, scan)
    wo = G._gather_outlier_rows(w, scan)
    c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    ops = 2 * m * n * k
    fns = {
        "i32": lambda: L.i8mm_gemm_i32(xq.data_ptr(), ldq, wq.data_ptr(), ldq, c.data_ptr(), n, m, n, k, st()),
        "f16": lambda: G._gemm_dequant(xq, wq, ldq, m, n, k, ax, aw, x, w, xo, scan, torch.float16, False, wo),
    }
    res = {}
    for rep in range(5):
        for vname, (cg, mc) in variants:
            L.i8mm_debug_set_gemm_variant(cg, mc)
            for ename, fn in fns.items():
                fn(); torch.cuda.synchronize()
                res.setdefault((vname, ename), []).append(timeit(fn, 10 if m * n * k > 5e12 else 30))
    L.i8mm_debug_set_gemm_variant(0, 0)
    line = f"M={m} K={k} N={n}:"
    for key, v in res.items():
        t = statistics.median(v)
        line += f" {key[0]}/{key[1]} {t*1e3:.0f}us {ops/t/1e9:.0f}TOPS |"
    print(line, flush=True)
    del x, w, xq, wq, c
    torch.cuda.empty_cache()
