"""Build a config's permuted matrix and run the SpMV kernel a few times (for ncu).

python tools/prof_spmv.py --config c2 --kernel merge --mode 1 --iters 3
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200 import synth
from paper_2308_00106_b200.kernels import set_merge_mode, spmv_into
from paper_2308_00106_b200.permute import axis_seed, random_permutation_forward

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--kernel", default="merge")
ap.add_argument("--mode", type=int, default=-1)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--unpermuted", action="store_true")
ap.add_argument("--time", action="store_true")
ap.add_argument("--panels", type=int, default=0)
ap.add_argument("--seg-panels", type=int, default=0)
ap.add_argument("--seg-mode", type=int, default=-1)
ap.add_argument("--seg-warps", type=int, default=0, help="persistent warps of the seg grid (default: occupancy)")
ap.add_argument("--seg-warm", action="store_true", help="L2 prefetch sweep of each pass's x slice")
ap.add_argument("--seg-split", type=int, default=-1, help="split-row plans: 1 on, 0 off, -1 auto")
ap.add_argument("--seg-hit", type=float, default=-1.0, help="x-slice L2 window hit ratio (0 = no persistence)")
ap.add_argument("--check", action="store_true", help="compare with the stream kernel")
ap.add_argument("--persist", action="store_true")
ap.add_argument("--inner", default="stream")
ap.add_argument("--lanes", type=int, default=0)
ap.add_argument("--row-cost", type=int, default=-1)
ap.add_argument("--reps", type=int, default=1, help="repeat the timing, print each")
ap.add_argument("--preload", type=float, default=0.0, help="seconds of untimed load first (power-capped clocks)")
a = ap.parse_args()
set_merge_mode(a.mode)
if a.row_cost >= 0:
    from paper_2308_00106_b200 import _lib

    _lib.call("sme_spmv_stream_set_row_cost", a.row_cost)
if a.config == "c4":
    A = synth.random_rows(50_000_000, 50_000_000, 20)
elif a.config == "c4s":
    A = synth.random_rows(10_000_000, 10_000_000, 20)
elif a.config == "c3":
    A = synth.rmat(24, 16, cap=1024)
elif a.config == "c3s":  # R-MAT scale 22 uncapped, f32 (x 16 MB: L2-resident, ragged rows)
    A = synth.rmat(22, 16, cap=1 << 30)
elif a.config == "c3u":  # R-MAT scale 24 without the degree cap (dense rows), f64 (x 134 MB > L2)
    A = synth.rmat(24, 16, cap=1 << 30, dtype=np.float64)
elif a.config == "c5":
    A = synth.laplacian5(2828)
else:
    A = synth.laplacian5(2000)
n = A.n_rows
dev = torch.device("cuda")
x = torch.from_numpy(P.input_vector(0, n)).to(dev, A.dtype)
if a.unpermuted:
    B, xp = A, x
else:
    fr = random_permutation_forward(n, axis_seed(7, 0))
    fc = random_permutation_forward(n, axis_seed(7, 1))
    p_r = P.Permutation(torch.from_numpy(fr.astype(np.int32)).to(dev), _trusted=True, _host=fr)
    p_c = P.Permutation(torch.from_numpy(fc.astype(np.int32)).to(dev), _trusted=True, _host=fc)
    B = P.permute_csr(A, p_r, p_c)
    xp = P.permute_vector(x, p_c)
    del A
if a.lanes:
    B._cache["lanes"] = a.lanes
if a.panels:
    from paper_2308_00106_b200.panels import device_info, panels_of

    B._cache["n_panels"] = a.panels
    pc = panels_of(B)
    pc.inner = a.inner
    pc.lanes = a.lanes or None
    if a.persist:
        pc.enable_persistence(True)
if a.seg_panels:
    B._cache["seg_panels"] = a.seg_panels
if a.seg_warps:
    from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

    P_ = a.seg_panels or auto_seg_panels(B)
    lay_ = SegLayout(B, P_, a.seg_warps)
    if P_ > 1:
        lay_.enable_persistence(True)
    B._cache[("seg", P_, False)] = lay_
if a.seg_hit >= 0:
    from paper_2308_00106_b200.seg import seg_of

    lay = seg_of(B)
    if a.seg_hit == 0:
        lay.persist = False
    else:
        lay.enable_persistence(True)
        lay.hit_ratio = a.seg_hit
if a.seg_mode >= 0:
    from paper_2308_00106_b200 import _lib

    _lib.call("sme_spmv_seg_set_mode", a.seg_mode)
y = torch.empty(n, dtype=B.dtype, device=dev)
if a.seg_split >= 0:
    from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels

    P_ = a.seg_panels or auto_seg_panels(B)
    lay_ = SegLayout(B, P_, a.seg_warps or None, split_rows=bool(a.seg_split))
    if P_ > 1:
        lay_.enable_persistence(True)
    B._cache[("seg", P_, False)] = lay_
    from paper_2308_00106_b200.kernels import row_stats

    print(f"max row {row_stats(B)[0]}, nnz {B.nnz}, split={lay_.split_rows}, panels {P_}", flush=True)
if a.seg_warm:
    from paper_2308_00106_b200.seg import seg_of

    seg_of(B).warm = True
t_setup = time.perf_counter()
spmv_into(B, xp, y, a.kernel)
torch.cuda.synchronize()
print(f"first call (incl. layout build) {time.perf_counter() - t_setup:.3f} s", flush=True)
if a.check:
    y2 = torch.empty(n, dtype=B.dtype, device=dev)
    spmv_into(B, xp, y2, "stream")
    print(f"rel err vs stream kernel: {P.relative_error(y, y2):.3e}", flush=True)
if a.preload > 0:
    t_end = time.perf_counter() + a.preload
    while time.perf_counter() < t_end:
        for _ in range(4):
            spmv_into(B, xp, y, a.kernel)
        torch.cuda.synchronize()
for _rep in range(a.reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.iters):
        spmv_into(B, xp, y, a.kernel)
    ev[1].record()
    clk = ""
    if a.preload > 0:
        import subprocess

        clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.iters
    bytes_ = B.nnz * 12 + (n + 1) * 4 + 16 * n
    print(f"{a.config} {a.kernel} segmode={a.seg_mode} hit={a.seg_hit} P={a.panels or a.seg_panels} inner={a.inner} L={a.lanes} rc={a.row_cost} persist={a.persist} "
          f"perm={not a.unpermuted} [{clk}]: {ms:.4f} ms  {bytes_ / ms / 1e6:.1f} GB/s  {2 * B.nnz / ms / 1e6:.1f} GFLOP/s")
