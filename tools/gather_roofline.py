"""Random 8-byte gather rate of the device vs the size of the gathered vector.

The roofline of a randomly-permuted SpMV has two ceilings: HBM bytes and the
random sector-gather rate (one x gather per nonzero).  Prints JSON lines
{x_mb, gathers_per_s, ...} for a sweep of x sizes; used for profiles/.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch

from paper_2308_00106_b200 import _lib
from paper_2308_00106_b200._cuda import ptr, stream

dev = torch.device("cuda")
sms = torch.cuda.get_device_properties(dev).multi_processor_count
blocks, per_thread = sms * 8 * 4, 256
out = torch.empty(blocks * 256, dtype=torch.float64, device=dev)
for mb in (1, 8, 32, 64, 100, 128, 200, 400, 1600):
    n = mb * 2**20 // 8
    x = torch.rand(n, dtype=torch.float64, device=dev)
    for keep in (1, 0):
        for _ in range(2):
            _lib.call("sme_diag_gather", ptr(x), n, blocks, per_thread, keep, ptr(out), stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            _lib.call("sme_diag_gather", ptr(x), n, blocks, per_thread, keep, ptr(out), stream())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        g = blocks * 256 * per_thread / (ms * 1e-3)
        print(json.dumps({"x_mb": mb, "evict_last": bool(keep), "ms": round(ms, 4), "gathers_per_s": g,
                          "sector_GBps": g * 32 / 1e9}), flush=True)
    del x
