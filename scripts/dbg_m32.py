"""Debug: fc1 M=32 prefill after decode calls, whole-call events, PDL on/off."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2208_07339_b200 as pkg
from paper_2208_07339_b200 import _native as nat
from paper_2208_07339_b200.synthetic import planted_pair_device

k, n = 5120, 20480
x_all, w, _ = planted_pair_device(64, k, n, 6, 20.0, seed=3, device="cuda")
lin = pkg.Int8Linear(w, 6.0)
L = nat.lib()


FLUSH = "--flush" in sys.argv
flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")


def t(m, reps=5):
    x = x_all[:m].contiguous()
    res = []
    for _ in range(reps):
        if FLUSH:
            flush.zero_()
        else:
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lin(x)
        b.record()
        b.synchronize()
        res.append(round(a.elapsed_time(b) * 1e3, 1))
    return res


print("fresh32", t(32), flush=True)
print("dec16", t(16, 3), flush=True)
print("after32", t(32), flush=True)
L.i8mm_debug_set_pdl(0)
print("nopdl32", t(32), flush=True)
L.i8mm_debug_set_pdl(1)
print("pdl32", t(32), flush=True)
print("dec16", t(16, 3), flush=True)
L.i8mm_debug_set_pdl(0)
print("nopdl32-after-dec", t(32), flush=True)
L.i8mm_debug_set_pdl(1)
print("dec16", t(16, 3), flush=True)
print("pdl32-after-dec", t(32), flush=True)
print("pdl64", t(64), flush=True)
