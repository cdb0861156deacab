"""Per-call (reference-semantics) llm_int8_matmul: W requantized every call (dev tool).
    python scripts/percall_prof.py M K N"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200.synthetic import planted_pair_device

m, k, n = (int(v) for v in sys.argv[1:4])
x, w, _ = planted_pair_device(m, k, n, 6, 20.0, 0)
for exact in (False, True):
    for _ in range(3):
        pkg.llm_int8_matmul(x, w, 6.0, exact=exact, validate=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        pkg.llm_int8_matmul(x, w, 6.0, exact=exact, validate=False)
    e.record()
    torch.cuda.synchronize()
    print(f"M={m} K={k} N={n} exact={exact}: {s.elapsed_time(e) / 10 * 1e3:.1f} us per call")
