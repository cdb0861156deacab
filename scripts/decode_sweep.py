"""cfg3 decode sweep (dev tool): OPT-13B projections at M = 1..256 tokens.

Times Int8Linear.forward (weight-stationary) per projection with CUDA events
(median of 50 calls, each after a 1 GiB L2 flush) and reports the HBM roofline
fraction of the weight stream:
bytes = K*N (int8 WqT) + 2*M*K (X) + 2*M*N (Y) + 2*|O|*N (fp16 outlier rows)
+ 4*N (column amax), against MEASURED_PEAKS.json hbm_gbs.
"""
import json
import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2208_07339_b200 as pkg  # noqa: E402
from paper_2208_07339_b200.synthetic import planted_pair_device  # noqa: E402

PROJ = {"qkvo": (5120, 5120), "fc1": (5120, 20480), "fc2": (20480, 5120)}
MS = [1, 2, 4, 8, 16, 32, 64, 128, 256]


def t_ev(fn, iters=50, warm=5, touch=None):
    t_ev.touch = touch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    flush = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")  # keeps the GPU busy while the host enqueues
    ts = []
    for _ in range(iters):
        flush.zero_()  # L2 flush: the weight stream must come from HBM
        if t_ev.touch is not None:
            t_ev.touch.sum()  # ... while the tokens are L2-resident, as after the previous layer
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    t_ev.last = ts
    return sum(ts) / iters


def main():
    projs, ms_list, iters = dict(PROJ), MS, 50
    if os.environ.get("DECODE_MS"):  # e.g. DECODE_MS=1,8,16 for a short A/B
        ms_list = [int(v) for v in os.environ["DECODE_MS"].split(",")]
    if len(sys.argv) > 2:  # e.g. "fc1 16" for a short run under ncu
        projs = {sys.argv[1]: PROJ[sys.argv[1]]}
        ms_list, iters = [int(sys.argv[2])], 3
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6543.7)
    rows = []
    for name, (k, n) in projs.items():
        x_all, w, _ = planted_pair_device(max(ms_list), k, n, 6, 20.0, seed=3, device="cuda")
        lin = pkg.Int8Linear(w, 6.0, check_finite=False)  # no per-call host read of the NaN flag
        for m in ms_list:
            x = x_all[:m].contiguous()
            ms = t_ev(lambda: lin(x), iters=iters, touch=x)
            o = lin.last_stats().get("decomposed_cols", 0)
            byts = k * n + 2 * m * k + 2 * m * n + 2 * o * n + 4 * n
            gbs = byts / (ms * 1e-3) / 1e9
            tl = t_ev.last
            # median per-call time: a rare host-side stall inside the timed loop (caching-allocator
            # segment growth, tens of ms) would otherwise dominate a mean over 50 calls
            ms = tl[len(tl) // 2]
            rows.append({"proj": name, "m": m, "k": k, "n": n, "us": ms * 1e3, "o": o,
                         "us_mean": sum(tl) / len(tl) * 1e3, "us_max": tl[-1] * 1e3,
                         "gbs": gbs, "frac_hbm": gbs / hbm,
                         "tops": 2.0 * m * n * k / (ms * 1e-3) / 1e12})
            print(json.dumps(rows[-1]), flush=True)
        del lin, w, x_all
        torch.cuda.empty_cache()
    out = ROOT / "gpurun_out" / "decode_sweep.json"
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
