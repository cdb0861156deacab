"""Quick CUDA-event timing of the pipeline stages (dev tool, not the bench)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2208_07339_b200 import gemm as G, _native as nat
from paper_2208_07339_b200.synthetic import planted_pair_device

def t_ev(fn, iters=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for (m, k, n) in [(16384, 4096, 16384), (16384, 16384, 4096), (16384, 12288, 49152), (512, 4096, 4096)]:
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
    scan = G.scan_outliers(x, 6.0)
    xq, ldq, ax, xo = G._quantize_rows(x, scan)
    wq, _, aw = G._quantize_cols_t(w, scan)
    ops = 2 * m * n * k
    t_scan = t_ev(lambda: G.scan_outliers(x, 6.0))
    t_qr = t_ev(lambda: G._quantize_rows(x, scan))
    t_qc = t_ev(lambda: G._quantize_cols_t(w, scan))
    c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    L = nat.lib(); st = torch.cuda.current_stream().cuda_stream
    t_gi = t_ev(lambda: L.i8mm_gemm_i32(xq.data_ptr(), ldq, wq.data_ptr(), ldq, c.data_ptr(), n, m, n, k, st))
    t_gd = t_ev(lambda: G._gemm_dequant(xq, wq, ldq, m, n, k, ax, aw, x, w, xo, scan, torch.float16, False))
    t_full = t_ev(lambda: G.llm_int8_matmul(x, w, 6.0, validate=False))
    a = xq[:, :k]; b = wq[:, :k].t()
    try:
        t_ref = t_ev(lambda: torch._int_mm(a, b))
    except Exception as ex:
        t_ref = float('nan'); print(ex)
    xb = x.to(torch.bfloat16); wb = w.to(torch.bfloat16)
    t_bf = t_ev(lambda: xb @ wb)
    print(f"M={m} K={k} N={n}: scan {t_scan*1e3:.1f}us qrows {t_qr*1e3:.1f}us qcols {t_qc*1e3:.1f}us | "
          f"gemm_i32 {t_gi*1e3:.1f}us ({ops/t_gi/1e9:.0f} TOPS) gemm_deq {t_gd*1e3:.1f}us ({ops/t_gd/1e9:.0f} TOPS) | "
          f"full {t_full*1e3:.1f}us ({ops/t_full/1e9:.0f} TOPS) | cublas _int_mm {t_ref*1e3:.1f}us ({ops/t_ref/1e9:.0f}) bf16 {t_bf*1e3:.1f}us ({ops/t_bf/1e9:.0f})", flush=True)
    del x, w, xq, wq, c
    torch.cuda.empty_cache()

import paper_2208_07339_b200 as pkg
for (m, k, n) in [(16384, 4096, 16384), (16384, 16384, 4096), (16384, 12288, 49152)]:
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
    lin = pkg.Int8Linear(w, 6.0)
    ops = 2 * m * n * k
    t = t_ev(lambda: lin(x))
    print(f"Int8Linear M={m} K={k} N={n}: {t*1e3:.1f}us ({ops/t/1e9:.0f} TOPS) stats={lin.last_stats()}", flush=True)
    del lin, x, w
    torch.cuda.empty_cache()
