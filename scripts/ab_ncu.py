"""Run each GEMM variant once per shape (for ncu metric A/B; dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2208_07339_b200 import gemm as G, _native as nat
from paper_2208_07339_b200.synthetic import planted_pair_device

L = nat.lib()
st = torch.cuda.current_stream().cuda_stream
shapes = [(16384, 4096, 16384), (16384, 16384, 4096), (16384, 12288, 49152)]
variants = [(0, 1), (0, 0), (1, 1)]
for (m, k, n) in shapes:
    x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
    scan = G.scan_outliers(x, 6.0)
    xq, ldq, ax, xo = G._quantize_rows(x, scan)
    wq, _, aw = G._quantize_cols_t(w, scan)
    wo = G._gather_outlier_rows(w, scan)
    c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    for cg, mc in variants:
        L.i8mm_debug_set_gemm_variant(cg, mc)
        L.i8mm_gemm_i32(xq.data_ptr(), ldq, wq.data_ptr(), ldq, c.data_ptr(), n, m, n, k, st)
        G._gemm_dequant(xq, wq, ldq, m, n, k, ax, aw, x, w, xo, scan, torch.float16, False, wo)
    torch.cuda.synchronize()
    del x, w, xq, wq, c
    torch.cuda.empty_cache()
print("done")
