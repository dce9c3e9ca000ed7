"""A/B of sme_host_pcg64_swap_partners between two builds of libsme (same box, same state)."""
import ctypes as C
import sys
import time

import numpy as np

libs = {name: C.CDLL(path) for name, path in (("old", sys.argv[1] if len(sys.argv) > 1 else "tools/_ab/libsme_old.so"), ("new", "paper_2308_00106_b200/libsme.so"))}
n = 50_000_000
st0 = np.random.PCG64(7).state
s = st0["state"]
init = np.array([s["state"] >> 64, s["state"] & (2**64 - 1), s["inc"] >> 64, s["inc"] & (2**64 - 1), 0, 0], dtype=np.uint64)
outs = {}
for rep in range(3):
    for thr in (4, 8, 16):
        for name, lib in libs.items():
            st = init.copy()
            h = np.empty(n, dtype=np.uint32)
            t = time.perf_counter()
            rc = lib.sme_host_pcg64_swap_partners(st.ctypes.data_as(C.c_void_p), C.c_int64(n), h.ctypes.data_as(C.c_void_p), C.c_int(thr))
            dt = time.perf_counter() - t
            assert rc == 0
            outs.setdefault(name, (h, st))
            print(f"{name} threads={thr}: {dt:.4f} s", flush=True)
print("identical:", np.array_equal(outs["old"][0], outs["new"][0]) and np.array_equal(outs["old"][1], outs["new"][1]))
import os
print("cpus", os.cpu_count())
