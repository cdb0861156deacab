"""GEMM-only timing of the prefill kernel (dev tool) for env A/B knobs
(I8MM_GEMM_MC, ...; I8MM_DBG_EPI only with I8MM_LIB_ALT pointing at the dev build,
_lib/dev/). Prints us and TOPS per shape."""
import os
import sys
import torch
sys.path.insert(0, ".")
if os.environ.get("I8MM_LIB_ALT"):  # A/B against another build of the library
    from paper_2208_07339_b200 import _native
    _native.load_library(os.environ["I8MM_LIB_ALT"])
from paper_2208_07339_b200 import gemm as G
from paper_2208_07339_b200.synthetic import planted_pair_device


def t_ev(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


tag = sys.argv[1] if len(sys.argv) > 1 else ""
for (m, k, n) in [(16384, 4096, 16384), (16384, 16384, 4096)]:
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
    scan = G.scan_outliers(x, 6.0)
    xq, ldq, ax, xo = G._quantize_rows(x, scan)
    wq, _, aw = G._quantize_cols_t(w, scan)
    wo = G._gather_outlier_rows(w, scan)
    ms = t_ev(lambda: G._gemm_dequant(xq, wq, ldq, m, n, k, ax, aw, x, w, xo, scan, torch.float16, False, wo))
    print(f"{tag} M={m} K={k} N={n}: {ms*1e3:.1f} us  {2*m*n*k/ms/1e9:.0f} TOPS", flush=True)
    del x, w, xq, wq
    torch.cuda.empty_cache()
