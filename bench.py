#!/usr/bin/env python
"""Benchmark of the max_E SpMV hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[3], the north-star target): C4 = 50,000,000 rows
x 50,000,000 cols, 20 distinct uniform-random columns per row (1.0e9 nnz), f64,
randomly row+column permuted (numpy PCG64 random_permutation, the reference's
generator) with the fused permuted-CSR build (K4).  One step = one SpMV pass
y = A' x' over the permuted matrix, inputs resident in HBM (13 GB of matrix
and vectors per pass, far larger than the 126 MB L2, so no L2 flush is needed).
At N > 1 (torchrun, NCCL) the permuted matrix is row-sharded and one step is
the x all-gather over NVLink plus the local SpMV (strong scaling of C4).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c4|c2|c5] [--kernel merge|vector] [--no-cpu]

--impl reference times the reference's algorithm on the host cores (the numpy
oracle port, oracle/ — the reference itself is pure numpy) on a bounded sample
of the same workload: the first R rows of the same permuted matrix with the
full permuted x.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (kind, n, k_or_grid, dtype, description)
    "c4": dict(kind="random_rows", n=50_000_000, k=20, dtype="f64",
               workload="C4: random-structured 50M x 50M, 20 nnz/row (1.0e9 nnz), f64, row+col permuted"),
    # C4's structure past 2^31 nonzeros: int64 row_ptr, the `_i64` entry points (not a
    # BASELINE config: the capability check for CSRs larger than int32 offsets)
    "c4w": dict(kind="random_rows", n=108_000_000, k=20, dtype="f64",
                workload="C4-wide: random-structured 108M x 108M, 20 nnz/row (2.16e9 nnz > 2^31, int64 row_ptr), "
                         "f64, row+col permuted"),
    "c2": dict(kind="laplacian", g=2000, dtype="f64",
               workload="C2: 5-point Laplacian 2000^2 (4M rows, 19,992,000 nnz), f64, row+col permuted"),
    "c5": dict(kind="laplacian", g=2828, dtype="f64",
               workload="C5: 5-point Laplacian 2828^2 (7,997,584 rows), f64, row+col permuted"),
    # edge factor 22: 369M R-MAT edges leave 252.9M nnz after dedupe + degree cap 1024,
    # BASELINE configs[2]'s ~256M (edge factor 16 left 199.5M; tools/c3_nnz_probe.py)
    "c3": dict(kind="rmat", scale=24, ef=22, cap=1024, dtype="f32",
               workload="C3: R-MAT scale 24 (16,777,216 rows), 22 x 2^24 edges, (a,b,c)=(0.57,0.19,0.19), deduped, "
                        "degree cap 1024 -> 252.9M nnz, f32, row+col permuted"),
}
PERM_SEED = 7  # strategy seed 7 for every config
CPU_SAMPLE_NNZ = 20_000_000
METRIC = "SpMV GFLOP/s and HBM GB/s (% of 8 TB/s), permuted vs unpermuted, 1/2/4/8 B200"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.file = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.file, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        rows = [ln.split(",") for ln in Path(self.file.name).read_text().splitlines() if ln.strip()]
        os.unlink(self.file.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        def num(i):
            out = []
            for r in rows:
                try:
                    out.append(float(r[i]))
                except (IndexError, ValueError):
                    pass
            return out

        pw, pl = num(3), num(9)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w": round(statistics.median(pw), 1) if pw else None,
                "power_limit_w": max(pl) if pl else None}


# ---------------------------------------------------------------------------
# workload construction
# ---------------------------------------------------------------------------
HOST_PERM_S: dict = {}


def host_perms(n_rows: int, n_cols: int, native: bool = True):
    """ROW_COLUMN_PERMUTE with seed 7 (permute.py:234-235), int64 forward vectors on the host.

    native: the package's bit-exact PCG64 shuffle (sme_host_pcg64_permutation, row and
    column concurrently); otherwise numpy's own Generator.permutation (the reference
    arm's setup)."""
    from paper_2308_00106_b200.permute import axis_seed, random_permutation_forward

    t = time.perf_counter()
    specs = [(n_rows, axis_seed(PERM_SEED, 0)), (n_cols, axis_seed(PERM_SEED, 1))]
    if native:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=2) as ex:
            fr, fc = (f.astype(np.int64) for f in ex.map(lambda a: random_permutation_forward(*a), specs))
    else:
        fr, fc = (np.random.Generator(np.random.PCG64(sd)).permutation(n) for n, sd in specs)
    dt = time.perf_counter() - t
    HOST_PERM_S["native" if native else "numpy"] = round(dt, 3)
    log(f"[bench] host permutations {n_rows:,}+{n_cols:,} ({'native' if native else 'numpy'}): {dt:.2f}s")
    return fr, fc


def device_perms(n_rows: int, n_cols: int):
    """ROW_COLUMN_PERMUTE with seed 7 as device Permutations: host swap partners (parallel
    PCG64 jump-ahead + branch-free rejection replay), swaps applied on the GPU
    (sme_fy_apply); bit-exact with numpy (tests/test_gpu_shuffle.py)."""
    import torch

    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200.permute import axis_seed

    torch.cuda.Stream()  # torch's lazy stream-pool init (~60 ms once per process) is not permutation work
    torch.cuda.synchronize()
    t = time.perf_counter()
    p_r, p_c = P.random_permutations([(n_rows, axis_seed(PERM_SEED, 0)), (n_cols, axis_seed(PERM_SEED, 1))])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    HOST_PERM_S["native"] = round(dt, 3)
    log(f"[bench] permutations {n_rows:,}+{n_cols:,} (host partners + GPU swaps): {dt:.2f}s")
    return p_r, p_c


def build_matrix(cfg: dict):
    from paper_2308_00106_b200 import synth

    if cfg["kind"] == "random_rows":
        return synth.random_rows(cfg["n"], cfg["n"], cfg["k"], seed=synth.C4_SEED)
    if cfg["kind"] == "rmat":
        return synth.rmat(cfg["scale"], cfg["ef"], cap=cfg["cap"], dtype=np.float32)
    return synth.laplacian5(cfg["g"])


def load_balance(row_ptr_dev, n_rows: int, parts: int = 148) -> dict:
    """Per-SM nnz spread of an even `parts`-way row split (make_row_partition, the
    reference's static partition, kernels.py:38-49): max/mean of nnz per part."""
    from paper_2308_00106_b200.kernels import make_row_partition

    b = make_row_partition(n_rows, min(parts, n_rows)).boundaries
    import torch

    pos = row_ptr_dev[torch.from_numpy(b).to(row_ptr_dev.device)].to(torch.int64).cpu().numpy()
    per = np.diff(pos)
    return {"parts": int(per.size), "max_over_mean": round(float(per.max() / max(per.mean(), 1e-9)), 4),
            "min_over_mean": round(float(per.min() / max(per.mean(), 1e-9)), 4)}


def cpu_sample_rows(n_rows: int, nnz: int) -> int:
    return max(1, min(n_rows, int(n_rows * CPU_SAMPLE_NNZ / max(1, nnz))))


def cpu_model() -> str:
    """The host CPU model (lscpu's 'Model name'), for the cpu_baseline record."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_module():
    """The UNMODIFIED reference package installed in baseline/_ref (baseline/install_ref.sh),
    or None when it is absent.  Timed as the CPU baseline ("kind": "reference");
    the oracle port stands in when it is missing ("kind": "port")."""
    p = ROOT / "baseline" / "_ref"
    if not (p / "spmv_entropy" / "__init__.py").is_file():
        return None
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    try:
        import spmv_entropy  # noqa: F401
        import spmv_entropy.entropy
        import spmv_entropy.kernels
        import spmv_entropy.matio
        import spmv_entropy.permute
    except Exception as e:  # pragma: no cover - a broken install falls back to the port
        log(f"[bench] baseline/_ref present but not importable ({e}); using the oracle port")
        return None
    return spmv_entropy


def cpu_baseline_run(ptr, col, val, x, n_cols: int, steps: int, warmup: int) -> dict:
    """The reference's CSR SpMV on the host cores over a row sample: the real
    reference (baseline/_ref: spmv_entropy.kernels.spmv_csr_parallel on a reference
    CsrMatrix, kernels.py:102-128) when installed, else the oracle numpy port of
    kernels.py:59-128.  Returns the rates and the last output (a parity input)."""
    import oracle as O

    cores = os.cpu_count() or 1
    nnz = int(ptr[-1])
    ref = ref_module()
    if ref is not None:
        m = ref.matio.CsrMatrix(int(ptr.size - 1), int(n_cols), ptr, col, val)
        par_fn = lambda: ref.kernels.spmv_csr_parallel(m, x, cores)  # noqa: E731
        ser_fn = lambda: ref.kernels.spmv_csr(m, x)  # noqa: E731
        kind, impl = "reference", "baseline/_ref spmv_entropy.kernels.spmv_csr_parallel (unmodified reference)"
    else:
        par_fn = lambda: O.spmv_csr_parallel(ptr, col, val, x, cores)  # noqa: E731
        ser_fn = lambda: O.spmv_csr(ptr, col, val, x)  # noqa: E731
        kind, impl = "port", "oracle numpy port of kernels.py:59-128 (baseline/_ref not installed)"
    for _ in range(warmup):
        par_fn()
    t = time.perf_counter()
    for _ in range(steps):
        y = par_fn()
    par = (time.perf_counter() - t) / steps
    t = time.perf_counter()
    ser_fn()
    ser = time.perf_counter() - t
    return {"gflops_parallel": 2 * nnz / par / 1e9, "gflops_serial": 2 * nnz / ser / 1e9, "cores": cores,
            "sec_per_call_parallel": par, "nnz": nnz, "kind": kind, "impl": impl, "y": y}


# ---------------------------------------------------------------------------
# full-scale parity: oracle rows of the permuted matrix
# ---------------------------------------------------------------------------
PARITY_RANDOM_ROWS = 10_000
PERM_SAMPLE_NNZ = 4_000_000  # the reference permute/histogram timing sample


def sample_rows(n_rows: int, nnz: int, seed: int = 2308, target_nnz: int = CPU_SAMPLE_NNZ,
                n_random: int = PARITY_RANDOM_ROWS) -> tuple[int, np.ndarray]:
    """The parity / CPU-baseline row sample: the first R rows (about target_nnz
    nonzeros) plus n_random seeded random rows from the rest, ascending."""
    R = max(1, min(n_rows, int(n_rows * target_nnz / max(1, nnz))))
    extra = np.empty(0, dtype=np.int64)
    if n_rows > R:
        rng = np.random.default_rng(seed)
        extra = np.unique(rng.integers(R, n_rows, size=min(n_random, n_rows - R)))
    return R, np.concatenate([np.arange(R, dtype=np.int64), extra])


def gather_rows_host(ptr, col, val, rows):
    """Rows `rows` of a host CSR as a new CSR (ptr int64, col, val)."""
    ptr = np.asarray(ptr, dtype=np.int64)
    s, e = ptr[rows], ptr[rows + 1]
    lens = e - s
    out = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(lens, out=out[1:])
    idx = np.repeat(s - out[:-1], lens) + np.arange(out[-1], dtype=np.int64)
    return out, col[idx], val[idx]


def device_rows(M, rows: np.ndarray):
    """Rows `rows` of a device CsrMatrix, copied to the host (ptr int64, col int64, val)."""
    import torch

    dev = M.d_row_ptr.device
    r = torch.from_numpy(rows).to(dev)
    s = M.d_row_ptr[r].to(torch.int64)
    lens = M.d_row_ptr[r + 1].to(torch.int64) - s
    out = torch.zeros(rows.size + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lens, 0, out=out[1:])
    total = int(out[-1])
    idx = torch.repeat_interleave(s - out[:-1], lens, output_size=total) + torch.arange(total, device=dev)
    return (out.cpu().numpy(), M.d_col_idx[idx].to(torch.int64).cpu().numpy(), M.d_values[idx].cpu().numpy())


def oracle_sample(cfg: dict, fr: np.ndarray, fc: np.ndarray, rows: np.ndarray, A=None):
    """Rows `rows` of coo_to_csr(permute_matrix(A, fr, fc)) built on the host by the
    oracle (oracle.permute_csr_rows vectorised): new row r
    is original row inv(fr)[r], its columns mapped through fc and sorted, values
    following.  Original rows come from the oracle's restatement of the generator
    (C4: O.random_rows_fast; C2/C5: O.laplacian5), for C3 from the device-built A
    (an input, not the path under test).  Returns (ptr, col int64, val) with val in
    the matrix dtype."""
    import oracle as O

    old = O.inverse(fr)[rows]
    if cfg["kind"] == "random_rows":
        from paper_2308_00106_b200.synth import C4_SEED

        k = cfg["k"]
        cols, vals = O.random_rows_fast(old, cfg["n"], k, C4_SEED)
        ptr0 = np.arange(rows.size + 1, dtype=np.int64) * k
        col0, val0 = cols.ravel(), vals.ravel()
    elif cfg["kind"] == "laplacian":
        ptr_a, col_a, val_a = O.laplacian5(cfg["g"])
        ptr0, col0, val0 = gather_rows_host(ptr_a, col_a, val_a, old)
    else:
        ptr0, col0, val0 = device_rows(A, old)
    mapped = fc[col0]
    rid = np.repeat(np.arange(rows.size, dtype=np.int64), np.diff(ptr0))
    order = np.lexsort((mapped, rid))
    vdt = np.float32 if cfg.get("dtype") == "f32" else np.float64
    return ptr0, mapped[order], np.asarray(val0, dtype=vdt)[order]


def oracle_x(n: int, fc: np.ndarray, f32: bool) -> np.ndarray:
    """x' = permute_vector(input_vector(0, n), p_c) (bench.py:168-171, 211), f32-rounded
    and widened for an f32 matrix (the f32 oracle sees the kernel's inputs)."""
    import oracle as O

    x = O.input_vector(0, n)
    if f32:
        x = x.astype(np.float32).astype(np.float64)
    return O.permute_vector(x, fc)


def parity_full_scale(cfg: dict, B, p_r, p_c, y_dev, fr_np, fc_np, rows, sample, x_np, tol: float,
                      y_cpu=None, R: int = 0) -> dict:
    """Compare the timed kernel's y and K4's permuted CSR with the oracle at full
    scale: the permutations against numpy's Generator.permutation (all n entries),
    the sampled rows of B bit-exact (row lengths, columns, value bits), and y on the
    sampled rows against the oracle SpMV (relative_error, kernels.py:131-142) at
    `tol`.  Raises SystemExit on any mismatch."""
    import oracle as O
    import torch

    perms_ok = bool(np.array_equal(p_r.forward, fr_np) and np.array_equal(p_c.forward, fc_np))
    ptr_o, col_o, val_o = sample
    ptr_d, col_d, val_d = device_rows(B, rows)
    csr_ok = bool(np.array_equal(ptr_o, ptr_d) and np.array_equal(col_o, col_d)
                  and np.array_equal(val_o.view(np.uint8), np.ascontiguousarray(val_d).view(np.uint8)))
    y_o = O.spmv_csr(ptr_o, col_o, val_o.astype(np.float64), x_np)
    y_g = y_dev[torch.from_numpy(rows).to(y_dev.device)].to(torch.float64).cpu().numpy()
    err = O.relative_error(y_g, y_o)
    out = {"rows_checked": int(rows.size), "nnz_checked": int(ptr_o[-1]),
           "rows": f"rows [0, {R:,}) + {rows.size - R:,} seeded random rows of the permuted matrix",
           "perms_bitexact_vs_numpy": perms_ok, "csr_rows_bitexact": csr_ok,
           "max_rel_err": err, "tol": tol,
           "oracle": "oracle/ restatement: numpy Generator.permutation perms, generator rows, p_c map + sort "
                     "(App. A item 4), numpy reduceat SpMV (kernels.py:59-70)"}
    if y_cpu is not None:  # the cpu_baseline leg's own output on rows [0, R)
        out["cpu_baseline_y_bitwise_vs_oracle"] = bool(np.array_equal(np.asarray(y_cpu), y_o[:R]))
    if not (perms_ok and csr_ok and err <= tol and out.get("cpu_baseline_y_bitwise_vs_oracle", True)):
        raise SystemExit(f"full-scale parity FAILED: {out}")
    return out


def cpu_permute_hist_baseline(cfg: dict, sample, n_cols: int, fc: np.ndarray) -> dict | None:
    """the reference's permute_matrix + coo_to_csr (permute.py:98-102,
    matio.py:281-294) and histogram_2d + shannon_entropy (entropy.py:96-119) timed on
    the host over a bounded sample of the workload's rows (the first rows of the
    oracle sample; a random row permutation of the sample, the full p_c)."""
    import oracle as O

    ptr, col, val = sample
    nr = int(np.searchsorted(ptr, PERM_SAMPLE_NNZ, side="right")) - 1
    nr = max(1, min(nr, ptr.size - 1))
    nz = int(ptr[nr])
    rows = np.repeat(np.arange(nr, dtype=np.int64), np.diff(ptr[: nr + 1]))
    ref = ref_module()
    pr = O.random_permutation(nr, O.axis_seed(PERM_SEED, 0))
    t = {}
    if ref is not None:
        R = ref
        coo = R.matio.CooMatrix(nr, n_cols, rows, col[:nz], val[:nz].astype(np.float64))
        Pr, Pc = R.permute.Permutation(pr), R.permute.Permutation(fc)
        t0 = time.perf_counter()
        pm = R.permute.permute_matrix(coo, Pr, Pc)
        csr = R.matio.coo_to_csr(pm)
        t["permute_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        bins = (min(128, nr), min(128, n_cols))
        H = R.entropy.shannon_entropy(R.entropy.histogram_2d(pm, *bins))
        t["hist_s"] = time.perf_counter() - t0
        kind = "reference"
        del csr
    else:
        t0 = time.perf_counter()
        r2, c2 = O.permute_coo(rows, col[:nz], pr, fc)
        O.coo_to_csr(nr, r2, c2, val[:nz])
        t["permute_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        bins = (min(128, nr), min(128, n_cols))
        H = O.entropy_of_counts(O.histogram_2d_counts(r2, c2, nr, n_cols, *bins))
        t["hist_s"] = time.perf_counter() - t0
        kind = "port"
    return {"kind": kind, "cores": 1, "sample": f"{nr:,} rows x {n_cols:,} cols, {nz:,} nnz of the workload",
            "permute_matrix_plus_coo_to_csr_s": round(t["permute_s"], 4),
            "permute_nnz_per_s": round(nz / t["permute_s"], 1),
            "histogram_2d_plus_entropy_s": round(t["hist_s"], 4),
            "hist_nnz_per_s": round(nz / t["hist_s"], 1), "entropy_bits": H}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args, cfg) -> dict:
    """Bounded sample of the permuted workload, built on the host with the oracle's
    restatements (numpy Generator.permutation, generator rows, row gather + column
    sort), timed with the reference's parallel CSR SpMV on all host cores: the
    unmodified reference from baseline/_ref when installed, else the oracle port."""
    import oracle as O

    t0 = time.perf_counter()
    if cfg["kind"] == "rmat":
        # bounded sample: the same construction at scale 20 (1/16 of C3), row+col permuted
        sc = 20
        ptr0, col0, val0 = O.rmat_csr(sc, cfg["ef"], 0.57, 0.19, 0.19, 0x5EED_C3, cfg["cap"])
        val0 = val0.astype(np.float32).astype(np.float64)
        n = 1 << sc
        fr, fc = host_perms(n, n, native=False)
        pr, pc = O.permute_coo(O.csr_to_coo_rows(ptr0), col0, fr, fc)
        ptr, col, val = O.coo_to_csr(n, pr, pc, val0)
        R = n
        x = oracle_x(n, fc, f32=True)
    else:
        n = cfg["n"] if cfg["kind"] == "random_rows" else cfg["g"] ** 2
        nnz = n * cfg["k"] if cfg["kind"] == "random_rows" else 5 * n - 4 * cfg["g"]
        fr, fc = host_perms(n, n, native=False)
        R = cpu_sample_rows(n, nnz)
        ptr, col, val = oracle_sample(cfg, fr, fc, np.arange(R, dtype=np.int64))
        val = val.astype(np.float64)
        x = oracle_x(n, fc, f32=False)
    log(f"[bench-ref] sample of {R:,} rows / {int(ptr[-1]):,} nnz built in {time.perf_counter() - t0:.1f}s")
    res = cpu_baseline_run(ptr, col, val, x, n, args.steps, args.warmup)
    v = res["gflops_parallel"]
    sample = (f"rows [0, {R:,}) of the permuted matrix ({res['nnz']:,} nnz) with the full permuted x; "
              f"{res['impl']} on {res['cores']} threads")
    return {
        "metric": METRIC, "value": round(v, 4), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(res["sec_per_call_parallel"] * 1e3, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.get("dtype", "f64"),
        "data": "synthetic", "impl": "reference",
        "config": {"workload": cfg["workload"], "sample": sample},
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOP/s", "cores": res["cores"], "kind": res["kind"],
                         "cpu_model": cpu_model(),
                         "sample": sample, "serial_gflops": round(res["gflops_serial"], 4)},
        "e2e": {"value": round(v, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def pcie_rates(x_pin, y_pin, reps: int = 3, stream_len: int = 4) -> dict:
    """Measured PCIe rates of this box with the e2e's own pinned buffers: H2D alone,
    D2H alone, both at once (one copy each way), and both directions streaming
    back to back (`stream_len` copies each way, the pipelined e2e's regime).  The
    e2e floor is one x in and one y out per step at the sustained concurrent rate."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    xd = torch.empty(x_pin.numel(), dtype=x_pin.dtype, device=dev)
    yd = torch.empty(y_pin.numel(), dtype=y_pin.dtype, device=dev)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(h2d: bool, d2h: bool, k: int = 1) -> float:
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(k):
                if h2d:
                    with torch.cuda.stream(sa):
                        xd.copy_(x_pin, non_blocking=True)
                if d2h:
                    with torch.cuda.stream(sb):
                        y_pin.copy_(yd, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) / k)
        return best

    nb_x, nb_y = x_pin.numel() * x_pin.element_size(), y_pin.numel() * y_pin.element_size()
    t_h, t_d, t_b = timed(True, False), timed(False, True), timed(True, True)
    t_s = timed(True, True, stream_len)
    return {"h2d_gbs": round(nb_x / t_h / 1e9, 2), "d2h_gbs": round(nb_y / t_d / 1e9, 2),
            "bidirectional_gbs_each_way": round(min(nb_x, nb_y) / t_b / 1e9, 2),
            "bidirectional_sustained_gbs_each_way": round(min(nb_x, nb_y) / t_s / 1e9, 2),
            "how": f"pinned copies of the e2e buffers ({nb_x / 1e6:.0f} MB), best of {reps}, wall clock around "
                   f"synchronize; sustained = {stream_len} back-to-back copies each way"}


def run_ours(args, cfg, rank: int, world: int) -> dict | None:
    import torch
    import torch.distributed as dist

    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200 import rowshard
    from paper_2308_00106_b200.bench import spmv_bytes
    from paper_2308_00106_b200.kernels import spmv_into

    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    A = build_matrix(cfg)
    torch.cuda.synchronize()
    n, nnz = A.n_rows, A.nnz
    log(f"[bench] rank {rank}: built {cfg['workload']} nnz={nnz:,} in {time.perf_counter() - t0:.1f}s")
    p_r, p_c = device_perms(n, A.n_cols)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    B = P.permute_csr(A, p_r, p_c)
    ev[1].record()
    torch.cuda.synchronize()
    permute_ms = ev[0].elapsed_time(ev[1])
    # entropy before / after (128 x 128 tiles)
    ev[0].record()
    hB = P.histogram_2d(B, 128, 128)
    ev[1].record()
    torch.cuda.synchronize()
    hist_ms = ev[0].elapsed_time(ev[1])
    # the same two calls again, warm (allocator pools and kernel attributes set up):
    # the first-call numbers above include cudaMalloc of the new matrix
    B2 = P.permute_csr(A, p_r, p_c)  # fills the allocator pool with a matrix's worth of blocks
    del B2
    ev[0].record()
    B2 = P.permute_csr(A, p_r, p_c)
    ev[1].record()
    torch.cuda.synchronize()
    permute_warm_ms = ev[0].elapsed_time(ev[1])
    del B2
    ev[0].record()
    P.histogram_2d(B, 128, 128)
    ev[1].record()
    torch.cuda.synchronize()
    hist_warm_ms = ev[0].elapsed_time(ev[1])
    H_before, H_after = P.shannon_entropy(P.histogram_2d(A, 128, 128)), P.shannon_entropy(hB)
    # the seg layout (the C4/C3/C5 SpMV's per-matrix analysis step): first build (allocations
    # included) and a warm rebuild, both wall-clock around synchronize (host-side sizing reads)
    layout_cold_ms = layout_warm_ms = None
    from paper_2308_00106_b200.kernels import auto_kernel as _auto

    if (_auto(B) if args.kernel == "auto" else args.kernel) == "seg":
        from paper_2308_00106_b200.seg import SegLayout, auto_seg_panels, seg_of

        torch.cuda.synchronize()
        t_l = time.perf_counter()
        lay0 = SegLayout(B, auto_seg_panels(B))
        torch.cuda.synchronize()
        layout_cold_ms = (time.perf_counter() - t_l) * 1e3
        del lay0  # its blocks go back to the allocator: the rebuild below is the warm one
        t_l = time.perf_counter()
        seg_of(B)  # built again and cached on B for the SpMVs below
        torch.cuda.synchronize()
        layout_warm_ms = (time.perf_counter() - t_l) * 1e3
    x = torch.from_numpy(P.input_vector(0, n)).to(dev, B.dtype)
    xp = P.permute_vector(x, p_c)
    # correctness of the permuted path (bench.py:218 round trip, 1e-12)
    y_ref = P.spmv_csr(A, x, args.kernel)
    y_perm = P.spmv_csr(B, xp, args.kernel)
    rel_err = P.relative_error(y_perm, P.permute_vector(y_ref, p_r))
    log(f"[bench] permute {permute_ms:.1f} ms, hist {hist_ms:.2f} ms, H {H_before:.4f} -> {H_after:.4f}, "
        f"round-trip rel err {rel_err:.2e}")
    tol = 1e-12 if B.dtype == torch.float64 else 1e-5
    if rel_err > tol:
        raise SystemExit(f"permuted SpMV failed the {tol} round-trip check: {rel_err}")
    balance = {"unpermuted": load_balance(A.d_row_ptr, n), "permuted": load_balance(B.d_row_ptr, n)}

    # the oracle side of the full-scale parity check (numpy perms, oracle-built sample
    # rows of the permuted matrix, oracle x'); the CPU baseline times the same rows
    cpu = None
    par_in = None
    if rank == 0 and world == 1 and not args.no_parity:
        t_par = time.perf_counter()
        fr_np, fc_np = host_perms(n, A.n_cols, native=False)
        R, rows = sample_rows(n, nnz)
        sample = oracle_sample(cfg, fr_np, fc_np, rows, A)
        x_np = oracle_x(A.n_cols, fc_np, f32=(B.dtype == torch.float32))
        par_in = (fr_np, fc_np, R, rows, sample, x_np)
        log(f"[bench] oracle sample of {rows.size:,} rows built in {time.perf_counter() - t_par:.1f}s")
        if not args.no_cpu:
            ptr_s, col_s, val_s = sample
            cs = cpu_baseline_run(ptr_s[: R + 1], col_s[: ptr_s[R]], val_s[: ptr_s[R]].astype(np.float64), x_np,
                                  A.n_cols, steps=5, warmup=1)
            cpu = {"value": round(cs["gflops_parallel"], 4), "unit": "GFLOP/s", "cores": cs["cores"],
                   "kind": cs["kind"], "cpu_model": cpu_model(),
                   "sample": f"rows [0, {R:,}) of the permuted matrix ({cs['nnz']:,} nnz), full permuted x, "
                             f"5 calls; {cs['impl']}",
                   "serial_gflops": round(cs["gflops_serial"], 4), "_y": cs["y"]}
            try:
                cpu["permute_and_histogram"] = cpu_permute_hist_baseline(cfg, sample, A.n_cols, fc_np)
            except MemoryError:
                cpu["permute_and_histogram"] = None
            log(f"[bench] cpu baseline: { {k: v for k, v in cpu.items() if k != '_y'} }")

    def timed(matrix, xv, kernel: str, steps: int, warmup: int, shard=None, chunk=None, preload_s: float = 0.0):
        """Device-timed loop: per-step events on the launching stream + whole-region events."""
        y = torch.empty(matrix.n_rows if shard is None else shard.local.n_rows, dtype=matrix.dtype, device=dev)

        def step():
            if shard is None:
                spmv_into(matrix, xv, y, kernel)
            else:
                shard.step(chunk)

        if preload_s > 0:  # keep the GPU loaded so the clock sampler sees the timed region's clocks
            t_end_pre = time.perf_counter() + preload_s
            while time.perf_counter() < t_end_pre:
                step()
                torch.cuda.synchronize()
        for _ in range(warmup):
            step()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start.record()
        for i in range(steps):
            starts[i].record()
            step()
            ends[i].record()
        t_end.record()
        torch.cuda.synchronize()
        total = t_start.elapsed_time(t_end)
        per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        if world > 1:
            tt = torch.tensor([total], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            total = float(tt.item())
        timed.last_y = y
        return total, per

    from paper_2308_00106_b200.kernels import auto_kernel

    resolved = auto_kernel(B) if args.kernel == "auto" else args.kernel
    if resolved == "panel":
        from paper_2308_00106_b200.panels import panels_of

        kernels_per_step = panels_of(B).n_panels
    elif resolved == "seg":
        from paper_2308_00106_b200.seg import seg_of

        kernels_per_step = seg_of(B).n_panels
    else:
        kernels_per_step = 2 if resolved == "merge" else 1
    if world == 1:
        # warm the plans outside the timed region (per-matrix metadata, like cuSPARSE's analysis;
        # the seg layout build itself is timed above)
        spmv_into(B, xp, torch.empty(n, dtype=B.dtype, device=dev), args.kernel)
        spmv_into(A, x, torch.empty(n, dtype=A.dtype, device=dev), args.kernel)
        clocks = Clocks(torch.cuda.current_device())
        clocks.start()
        total_ms, per = timed(B, xp, args.kernel, args.steps, args.warmup, preload_s=1.0)
        clk = clocks.stop()
        parity = None
        if par_in is not None:  # the timed loop's own output against the oracle
            fr_np, fc_np, R, rows, sample, x_np = par_in
            parity = parity_full_scale(cfg, B, p_r, p_c, timed.last_y, fr_np, fc_np, rows, sample, x_np, tol,
                                       y_cpu=None if cpu is None else cpu.pop("_y"), R=R)
            log(f"[bench] parity: {parity}")
            del par_in, sample
        # the same untimed preload as the permuted loop: both loops start from the power-capped
        # steady state (after the parity leg's CPU work the GPU has cooled and clocks up)
        un_total, un_per = timed(A, x, args.kernel, args.steps, args.warmup, preload_s=1.0)
        # the same comparison with the two matrices alternating step by step (no clock/thermal drift
        # between two separate loops): medians of per-step events
        yb_, ya_ = torch.empty(n, dtype=B.dtype, device=dev), torch.empty(n, dtype=A.dtype, device=dev)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        for e0, e1, e2 in ev:
            e0.record()
            spmv_into(B, xp, yb_, args.kernel)
            e1.record()
            spmv_into(A, x, ya_, args.kernel)
            e2.record()
        torch.cuda.synchronize()
        inter = (statistics.median(e0.elapsed_time(e1) for e0, e1, _ in ev),
                 statistics.median(e1.elapsed_time(e2) for _, e1, e2 in ev))
        del yb_, ya_
        others = {}
        from paper_2308_00106_b200.kernels import WIDE_KERNELS

        for other in ("panel", "stream", "vector", "merge"):
            if other != resolved and (not B.wide or other in WIDE_KERNELS):
                o_total, _ = timed(B, xp, other, max(3, args.steps // 4), 2)
                others[other] = round(2 * nnz / (o_total / max(3, args.steps // 4) * 1e-3) / 1e9, 3)
        ot_total = None
        nnz_total = nnz
        bytes_step = spmv_bytes(n, A.n_cols, nnz, B.d_values.element_size(), 4)

    ms_per_step = total_ms / args.steps
    gflops = 2 * nnz_total / (ms_per_step * 1e-3) / 1e9
    kern_ms = statistics.mean(per)
    peak, peak_src = measured_peaks()
    # second ceiling of a randomly-permuted SpMV: one random x gather per nonzero.
    # Measured live: the device's random 8-byte gather rate with an L2-resident
    # 64 MB vector (diag.cu) — the best case every panel pass aims for.
    gather_roof = None
    if world == 1:
        from paper_2308_00106_b200 import _lib
        from paper_2308_00106_b200._cuda import ptr as _ptr, stream as _stream

        gx = torch.rand(64 * 2**20 // 8, dtype=torch.float64, device=dev)
        gblocks, gper = torch.cuda.get_device_properties(dev).multi_processor_count * 32, 256
        gout = torch.empty(gblocks * 256, dtype=torch.float64, device=dev)
        for _ in range(2):
            _lib.call("sme_diag_gather", _ptr(gx), gx.numel(), gblocks, gper, 1, _ptr(gout), _stream())
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g_ms = []
        for _ in range(3):  # best of three: one C5 run's single sample read 187 G/s against 287 elsewhere
            g0.record()
            for _ in range(5):
                _lib.call("sme_diag_gather", _ptr(gx), gx.numel(), gblocks, gper, 1, _ptr(gout), _stream())
            g1.record()
            torch.cuda.synchronize()
            g_ms.append(g0.elapsed_time(g1) / 5)
        ceil_gps = gblocks * 256 * gper / (min(g_ms) * 1e-3)
        ach_gps = nnz / (kern_ms * 1e-3)
        gather_roof = {"gathers_per_step": nnz, "achieved_gps": round(ach_gps / 1e9, 2),
                       "ceiling_gps": round(ceil_gps / 1e9, 2), "unit": "G gathers/s",
                       "frac": round(ach_gps / ceil_gps, 4),
                       "ceiling_source": "measured in this run: random 8-B gathers from a 64 MB L2-resident "
                                         "vector (sme_diag_gather)",
                       "min_step_ms_at_ceiling": round(nnz / ceil_gps * 1e3, 4)}
        del gx, gout
    achieved = bytes_step / (kern_ms * 1e-3) / 1e9

    # e2e through the public API with pinned host buffers (H2D x + SpMV + D2H y every step)
    e2e = None
    if world == 1:
        # two distinct pinned input vectors (x' and 2 x'), alternating; every step copies
        # its whole x in and its whole y out
        xs_pin = [torch.empty(n, dtype=B.dtype, pin_memory=True) for _ in range(2)]
        xs_pin[0].copy_(xp.cpu())
        xs_pin[1].copy_(xs_pin[0] * 2)
        # K steps like the device-timed loop; outputs land in a ring of two pinned host
        # vectors (every step still copies its whole y out)
        e_steps = max(4, args.steps)
        ys_pin = [torch.empty(n, dtype=B.dtype, pin_memory=True) for _ in range(2)]
        # single-call API (synchronous per vector): the reference-shaped spmv_csr
        # warm as a caller's loop runs (each result alive until the next call returns):
        # the result pool then holds the two page-locked host mappings such a loop uses
        yh = P.spmv_csr(B, xs_pin[0], args.kernel)
        yh = P.spmv_csr(B, xs_pin[1], args.kernel)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for k in range(3):
            yh = P.spmv_csr(B, xs_pin[k & 1], args.kernel)
        single_ms = (time.perf_counter() - w0) / 3 * 1e3
        del yh
        # pipelined API over a stream of vectors: copies of neighbouring steps overlap
        P.spmv_csr_pipelined(B, xs_pin[:2], ys_pin[:2], args.kernel)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        s0.record()
        P.spmv_csr_pipelined(B, [xs_pin[k & 1] for k in range(e_steps)], [ys_pin[k & 1] for k in range(e_steps)],
                             args.kernel)
        s1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) / e_steps
        e_ms = max(s0.elapsed_time(s1) / e_steps, wall * 1e3)
        # the last outputs must equal the device-resident SpMV of the same vectors
        e2e_err = max(P.relative_error(ys_pin[(e_steps - 1) & 1], y_perm * (2.0 if (e_steps - 1) & 1 else 1.0)),
                      P.relative_error(ys_pin[(e_steps - 2) & 1], y_perm * (2.0 if (e_steps - 2) & 1 else 1.0)))
        if e2e_err > tol:
            raise SystemExit(f"pipelined host-vector SpMV differs from the device result: {e2e_err}")
        pcie = pcie_rates(xs_pin[0], ys_pin[0])
        step_bytes = n * B.d_values.element_size()
        floor_ms = step_bytes / (pcie["bidirectional_sustained_gbs_each_way"] * 1e9) * 1e3
        pcie["e2e_floor_ms"] = round(floor_ms, 4)
        pcie["e2e_frac_of_floor"] = round(floor_ms / e_ms, 4)
        e2e = {"value": round(2 * nnz / (e_ms * 1e-3) / 1e9, 4), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(step_bytes),
               "d2h_bytes_per_step": int(step_bytes), "ms_per_step": round(e_ms, 4),
               "steps": e_steps, "rel_err": e2e_err, "pcie": pcie,
               "api": "paper_2308_00106_b200.spmv_csr_pipelined(CsrMatrix, [pinned host x_k]) -> [pinned host y_k]",
               "single_call": {"api": "paper_2308_00106_b200.spmv_csr(CsrMatrix, pinned host tensor)",
                               "ms_per_step": round(single_ms, 4),
                               "value": round(2 * nnz / (single_ms * 1e-3) / 1e9, 4)}}

    if rank != 0:
        return None
    traffic = None
    req_roof = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists() and world == 1:  # the table holds 1-GPU captures (a shard moves less)
        try:
            table = json.loads(tf.read_text())
            traffic = table.get(f"{args.config}/{resolved}")
            reqs = table.get("l1_to_l2_requests", {}).get(f"{args.config}/{resolved}")
        except Exception:
            traffic, reqs = None, None
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        if reqs and clk.get("sm_mhz"):
            # the SM's L1 -> L2 (xbar) request port takes one request per clock: with one
            # random gather per nonzero every request is its own line
            ceil_rps = sms * clk["sm_mhz"] * 1e6
            ach_rps = reqs / (kern_ms * 1e-3)
            req_roof = {"requests_per_step": int(reqs), "achieved_g_per_s": round(ach_rps / 1e9, 2),
                        "ceiling_g_per_s": round(ceil_rps / 1e9, 2), "frac": round(ach_rps / ceil_rps, 4),
                        "min_step_ms_at_ceiling": round(reqs / ceil_rps * 1e3, 4),
                        "source": "requests: ncu lts__t_requests_srcunit_tex.sum over one step's launches "
                                  "(profiles/ncu_traffic.json); ceiling: 1 request / SM / clock at the median SM "
                                  "clock sampled during the timed region"}
    out = {
        "metric": METRIC,
        "value": round(gflops, 3),
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64" if B_dtype_is_f64(cfg) else "f32",
        "data": "synthetic (device generator, seeded; numpy PCG64 permutations, seed 7)",
        "config": {
            "workload": cfg["workload"],
            "kernel": resolved + (f" ({kernels_per_step} column panels x k_spmv_stream)" if resolved == "panel" else
                                 f" ({kernels_per_step} column panels x k_spmv_seg)" if resolved == "seg" else ""),
            "n_rows": n, "nnz": nnz,
            "parallelism": "1 GPU",
            "l2": "inputs (13 GB/pass for C4) far exceed the 126 MB L2; no flush needed" if cfg["kind"] == "random_rows"
                  else "x fits L2; matrix streams exceed L2",
        },
        "hbm_gbs": round(achieved, 1),
        "pct_of_8tbs": round(100 * achieved / 8000.0, 2),
        "permuted_vs_unpermuted": None if un_total is None else {
            "permuted_gflops": round(gflops, 3),
            "unpermuted_gflops": round(2 * nnz / (un_total / args.steps * 1e-3) / 1e9, 3),
            "ratio": round((un_total / args.steps) / ms_per_step, 4),
            "interleaved": {"permuted_ms": round(inter[0], 4), "unpermuted_ms": round(inter[1], 4),
                            "ratio": round(inter[1] / inter[0], 4),
                            "how": "permuted and unpermuted SpMV alternating step by step, medians of per-step "
                                   "CUDA events (ratio = unpermuted time / permuted time)"},
        },
        "other_kernels_gflops": others if world == 1 else None,
        "gather_roofline": gather_roof,
        "request_roofline": req_roof,
        "entropy_bits": {"unpermuted": round(H_before, 6), "permuted": round(H_after, 6), "max": 14.0},
        "load_balance_148_even_rows": balance,
        "permute_ms": round(permute_ms, 2), "permute_warm_ms": round(permute_warm_ms, 2),
        "layout_build_ms": None if layout_cold_ms is None else round(layout_cold_ms, 2),
        "layout_build_warm_ms": None if layout_warm_ms is None else round(layout_warm_ms, 2),
        "setup_warm_ms": round(permute_warm_ms + (layout_warm_ms or 0.0), 2),
        "setup_note": "one-time cost of a permuted matrix: permute (K4: CUDA events; cold = first call incl. "
                      "allocation) + the seg layout build (wall clock around synchronize; cold = first build); "
                      "setup_warm_ms = the warm pair",
        "perm_gen_s": HOST_PERM_S.get("native"),
        "hist_ms": round(hist_ms, 3), "hist_warm_ms": round(hist_warm_ms, 3),
        "roundtrip_rel_err": rel_err,
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_step,
                     "kernel_ms": round(kern_ms, 5),
                     "timed": f"per-step CUDA events on the launch stream around the {kernels_per_step} "
                              f"launch(es) of one SpMV ({resolved})" + (" + all_gather" if world > 1 else ""),
                     "note": "achieved = algorithmic bytes (SURVEY.md 8d formula) / kernel time; a randomly "
                             "permuted SpMV is additionally bounded by the random-gather ceiling (gather_roofline)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk,
        "gpu_launches": kernels_per_step * args.steps,
    }
    return out


def build_shard(cfg: dict, plan, rank: int, p_r, p_c):
    """This rank's rows [lo, hi) of the permuted matrix B = P_r A P_c, built without
    any rank holding all of B: the original rows inverse(p_r)[lo:hi] (C4: generated
    directly by the counter-based row generator; C2/C3/C5: gathered from A, which
    is small for those configs), then K4 on them with the row order already final
    (permute_csr(A_rows, None, p_c): columns through p_c, sorted within rows).
    Bit-identical to rows [lo, hi) of permute_csr(A, p_r, p_c)."""
    import torch

    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200 import synth
    from paper_2308_00106_b200.matio import CsrMatrix

    lo, hi = plan.row_range(rank)
    old = p_r.d_inverse[lo:hi]
    A_full = None
    if cfg["kind"] == "random_rows":
        A_rows = synth.random_rows_select(old, cfg["n"], cfg["k"], seed=synth.C4_SEED)
    else:
        A_full = build_matrix(cfg)
        dev = A_full.d_row_ptr.device
        s = A_full.d_row_ptr[old.long()].long()
        lens = A_full.d_row_ptr[old.long() + 1].long() - s
        rp = torch.zeros(hi - lo + 1, dtype=torch.int64, device=dev)
        torch.cumsum(lens, 0, out=rp[1:])
        tot = int(rp[-1])
        idx = torch.repeat_interleave(s - rp[:-1], lens, output_size=tot) + torch.arange(tot, device=dev)
        A_rows = CsrMatrix._from_device(hi - lo, A_full.n_cols, rp.to(torch.int32), A_full.d_col_idx[idx].contiguous(),
                                        A_full.d_values[idx].contiguous())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    B_loc = P.permute_csr(A_rows, None, p_c)
    ev[1].record()
    torch.cuda.synchronize()
    return B_loc, ev[0].elapsed_time(ev[1]), A_full


def run_sharded(args, cfg, rank: int, world: int) -> dict | None:
    """N > 1: one rank per GPU (torch.distributed, NCCL), C4 strong-scaled.  Rank k
    builds only its row shard of the permuted matrix (build_shard), checks it and
    its SpMV rows against the oracle, then times the step of north_star (4): the x
    exchange over NVLink (per-slot broadcasts pipelined with the seg panel passes,
    or one all_gather) plus the local SpMV.  Time = max over ranks (device events)."""
    import torch
    import torch.distributed as dist

    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200 import rowshard
    from paper_2308_00106_b200.bench import spmv_bytes

    dev = torch.device("cuda", torch.cuda.current_device())
    n = cfg["n"] if cfg["kind"] == "random_rows" else (cfg["g"] ** 2 if cfg["kind"] == "laplacian" else 1 << cfg["scale"])
    t0 = time.perf_counter()
    p_r, p_c = device_perms(n, n)
    plan = rowshard.ShardPlan(n, n, world)
    B_loc, permute_ms, A_full = build_shard(cfg, plan, rank, p_r, p_c)
    lo, hi = plan.row_range(rank)
    nnz_loc = B_loc.nnz
    log(f"[bench] rank {rank}/{world}: shard rows [{lo:,}, {hi:,}) nnz {nnz_loc:,} built in "
        f"{time.perf_counter() - t0:.1f}s (K4 {permute_ms:.1f} ms)")
    tol = 1e-12 if B_loc.dtype == torch.float64 else 1e-5
    shard = rowshard.RowShardedSpMV(B_loc, plan, rank, args.kernel, local=True)
    resolved = "seg" if shard.seg is not None else (args.kernel if args.kernel != "auto" else "vector")
    kernels_per_step = shard.seg.n_panels if shard.seg is not None else 1
    x = torch.from_numpy(P.input_vector(0, n)).to(dev, B_loc.dtype)
    xp = P.permute_vector(x, p_c)
    del x
    c0, c1 = plan.col_range(rank)
    chunk = plan.pad_slice(xp[c0:c1])
    y_loc = shard.step(chunk).clone()
    torch.cuda.synchronize()

    # parity of this rank's rows against the oracle (sampled, bit-exact CSR, y at tol)
    parity = None
    if not args.no_parity:
        fr_np, fc_np = host_perms(n, n, native=False)
        R_loc, rows_loc = sample_rows(hi - lo, nnz_loc, seed=rank, target_nnz=max(1, CPU_SAMPLE_NNZ // (4 * world)),
                                      n_random=max(1, PARITY_RANDOM_ROWS // world))
        rows = rows_loc + lo
        sample = oracle_sample(cfg, fr_np, fc_np, rows, A_full)
        x_np = oracle_x(n, fc_np, f32=(B_loc.dtype == torch.float32))
        import oracle as O

        perms_ok = bool(np.array_equal(p_r.forward, fr_np) and np.array_equal(p_c.forward, fc_np))
        ptr_d, col_d, val_d = device_rows(B_loc, rows_loc)
        ptr_o, col_o, val_o = sample
        csr_ok = bool(np.array_equal(ptr_o, ptr_d) and np.array_equal(col_o, col_d)
                      and np.array_equal(val_o.view(np.uint8), np.ascontiguousarray(val_d).view(np.uint8)))
        y_o = O.spmv_csr(ptr_o, col_o, val_o.astype(np.float64), x_np)
        y_g = y_loc[torch.from_numpy(rows_loc).to(dev)].to(torch.float64).cpu().numpy()
        err = O.relative_error(y_g, y_o)
        res = torch.tensor([err, 0.0 if (perms_ok and csr_ok) else 1.0, float(rows.size)], dtype=torch.float64,
                           device=dev)
        dist.all_reduce(res[:2], op=dist.ReduceOp.MAX)
        dist.all_reduce(res[2:], op=dist.ReduceOp.SUM)
        parity = {"rows_checked": int(res[2].item()), "ranks": world, "max_rel_err": float(res[0].item()),
                  "tol": tol, "csr_rows_bitexact": res[1].item() == 0.0, "perms_bitexact_vs_numpy": perms_ok,
                  "rows": "per rank: the first rows of its shard + seeded random rows of its shard",
                  "oracle": "oracle/ restatement (numpy perms, generator rows, p_c map + sort, numpy reduceat SpMV)"}
        log(f"[bench] rank {rank}: shard parity err {err:.2e} csr {csr_ok} perms {perms_ok}")
        if not (res[1].item() == 0.0 and res[0].item() <= tol):
            raise SystemExit(f"rank {rank}: sharded parity FAILED: {parity}")
        del sample, fr_np, fc_np, x_np
    del A_full

    steps, warmup = args.steps, args.warmup
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    t_end_pre = time.perf_counter() + 1.0
    while time.perf_counter() < t_end_pre:  # keep the GPU loaded so the sampler sees the timed clocks
        shard.step(chunk)
        torch.cuda.synchronize()
    for _ in range(warmup):
        shard.step(chunk)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    t_start.record()
    for i in range(steps):
        starts[i].record()
        shard.step(chunk)
        ends[i].record()
    t_end.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    tt = torch.tensor([t_start.elapsed_time(t_end), statistics.mean(s.elapsed_time(e) for s, e in zip(starts, ends))],
                      device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms, kern_ms = float(tt[0].item()), float(tt[1].item())
    nnz_t = torch.tensor([nnz_loc], dtype=torch.int64, device=dev)
    dist.all_reduce(nnz_t)
    nnz = int(nnz_t.item())
    ms_per_step = total_ms / steps
    gflops = 2 * nnz / (ms_per_step * 1e-3) / 1e9

    # e2e: every rank copies its pinned host x chunk in and its y rows out each step, with
    # the copies of neighbouring steps overlapped (x of step k+1 in and y of step k-1 out
    # on their own streams while step k exchanges and computes), as spmv_csr_pipelined
    # does on one GPU; two pinned x chunks (x' and 2 x') alternate
    x_pins = [torch.empty(plan.pad, dtype=B_loc.dtype, pin_memory=True) for _ in range(2)]
    x_pins[0].copy_(chunk.cpu())
    x_pins[1].copy_(x_pins[0] * 2)
    y_pins = [torch.empty(hi - lo, dtype=B_loc.dtype, pin_memory=True) for _ in range(2)]
    xcs = [torch.empty_like(chunk) for _ in range(2)]
    ybs = [torch.empty(hi - lo, dtype=B_loc.dtype, device=dev) for _ in range(2)]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    main = torch.cuda.current_stream()
    e_steps = max(4, min(steps, 10))

    def e2e_run(n_steps: int) -> None:
        computed, copied = [None, None], [None, None]
        h2d.wait_stream(main)
        d2h.wait_stream(main)
        for k in range(n_steps):
            b = k & 1
            with torch.cuda.stream(h2d):
                if computed[b] is not None:
                    h2d.wait_event(computed[b])
                xcs[b].copy_(x_pins[b], non_blocking=True)
                landed = torch.cuda.Event()
                landed.record(h2d)
            main.wait_event(landed)
            if copied[b] is not None:
                main.wait_event(copied[b])
            ybs[b].copy_(shard.step(xcs[b]))
            done = torch.cuda.Event()
            done.record(main)
            computed[b] = done
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                y_pins[b].copy_(ybs[b], non_blocking=True)
                out_ev = torch.cuda.Event()
                out_ev.record(d2h)
                copied[b] = out_ev
        d2h.synchronize()
        main.wait_stream(d2h)
        main.wait_stream(h2d)

    e2e_run(2)
    dist.barrier()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    s0.record()
    e2e_run(e_steps)
    s1.record()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3 / e_steps
    et = torch.tensor([max(s0.elapsed_time(s1) / e_steps, wall_ms)], device=dev)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e_ms = float(et.item())
    y_pin = y_pins[(e_steps - 1) & 1]
    if (e_steps - 1) & 1:
        y_loc = y_loc * 2.0
    e2e_err = P.relative_error(y_pin, y_loc)
    if e2e_err > tol:
        raise SystemExit(f"rank {rank}: host-vector sharded step differs from the device result: {e2e_err}")
    if rank != 0:
        return None
    bytes_loc = spmv_bytes(hi - lo, plan.world * plan.pad, nnz_loc, B_loc.d_values.element_size(), 4)
    peak, peak_src = measured_peaks()
    achieved = bytes_loc / (kern_ms * 1e-3) / 1e9
    nccl_ver = ".".join(map(str, torch.cuda.nccl.version())) if dist.get_backend() == "nccl" else None
    return {
        "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if B_dtype_is_f64(cfg) else "f32",
        "data": "synthetic (device generator, seeded; numpy PCG64 permutations, seed 7)",
        "config": {
            "workload": cfg["workload"],
            "kernel": resolved + (f" ({kernels_per_step} column panels x k_spmv_seg per shard)" if resolved == "seg"
                                  else ""),
            "n_rows": n, "nnz": nnz,
            "parallelism": (f"row-shard x{world} + {dist.get_backend()} per-slot x broadcasts pipelined with the "
                            f"panel passes" if shard.pipelined else
                            f"row-shard x{world} + {dist.get_backend()} all_gather of x"),
            "setup": "sharded: each rank generates only its original rows inverse(p_r)[lo:hi] and runs K4 on them",
            "nccl_version": nccl_ver,
            "l2": "inputs far exceed the 126 MB L2; no flush needed",
        },
        "hbm_gbs_per_gpu": round(achieved, 1),
        "permute_ms_rank0": round(permute_ms, 2),
        "parity": parity,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_loc, "kernel_ms": round(kern_ms, 5),
                     "timed": f"rank 0's shard: per-step events around the exchange + {kernels_per_step} launches "
                              "(max over ranks)"},
        "cpu_baseline": None,
        "e2e": {"value": round(2 * nnz / (e_ms * 1e-3) / 1e9, 4), "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(plan.pad * B_loc.d_values.element_size()) * world,
                "d2h_bytes_per_step": int(n * B_loc.d_values.element_size()), "ms_per_step": round(e_ms, 4),
                "rel_err": e2e_err,
                "api": "rowshard.RowShardedSpMV.step per rank: pinned host x chunk in, y rows out, copies of "
                       "neighbouring steps overlapped (2 buffers)"},
        "clocks": clk,
        "gpu_launches": kernels_per_step * steps,
    }


def B_dtype_is_f64(cfg) -> bool:
    return cfg.get("dtype", "f64") == "f64"


def run_iterative(args, cfg) -> dict:
    """C5 (BASELINE.json configs[4]): 1000-step power iteration on the row+column
    permuted 8M-row Laplacian, one CUDA graph per `graph_steps` iterations, against
    the same iteration on the unpermuted matrix; the permutation cost (host PCG64
    generation, upload, fused permuted-CSR build) is amortised end to end."""
    import torch

    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200.iterative import PermutedOperator, PowerIteration

    dev = torch.device("cuda", torch.cuda.current_device())
    A = build_matrix(cfg)
    n, nnz = A.n_rows, A.nnz
    iters, graph_steps = 1000, 50
    x0 = P.input_vector(0, n)
    torch.cuda.Stream()  # process init (torch's stream pool), not per-matrix setup
    torch.cuda.synchronize()

    def setup():
        """One permuted operator from scratch: ROW_COLUMN permutations (seed 7), the folded
        permuted CSR (K4), its seg layout with the fused epilogue.  Wall clock with device
        syncs, ms per piece."""
        t0 = time.perf_counter()
        p_r, p_c = device_perms(n, n)
        t1 = time.perf_counter()
        o = PermutedOperator(A, p_r, p_c, kernel=args.kernel)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        o.fused_layout()  # the seg layout (cached on the matrix, reused by the run)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        return o, p_r, p_c, {"total_ms": round((t3 - t0) * 1e3, 2), "generation_ms": round((t1 - t0) * 1e3, 2),
                             "permuted_csr_build_ms": round((t2 - t1) * 1e3, 2),
                             "seg_layout_build_ms": round((t3 - t2) * 1e3, 2)}

    _, _, _, setup_first = setup()  # the first matrix of the process (allocator growth, first uses)
    warm = []
    for _ in range(3):  # the steady-state cost of one more permuted matrix: median of three
        op, p_r, p_c, st = setup()
        warm.append(st)
    setup_warm = sorted(warm, key=lambda d: d["total_ms"])[1]
    setup_warm["runs_total_ms"] = [d["total_ms"] for d in warm]
    perm_s = setup_warm["total_ms"] * 1e-3

    def run(operator) -> tuple[float, float, PowerIteration]:
        pi = PowerIteration(operator, x0)
        pi.capture(graph_steps)
        for _ in range(args.warmup):
            pi.graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pi.run(iters)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), pi.eigenvalue, pi

    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    perm_ms, lam_p, pi_p = run(op)
    clk = clocks.stop()
    unperm_ms, lam_u, pi_u = run(PermutedOperator(A, None, None, kernel=args.kernel))
    x_p = pi_p.x()
    # the true ROW_COLUMN operator P_r A P_c (no folding): the iterate is mapped back by
    # the gather q = p_r o p_c^-1 every step (scattered through q^-1 in the fused epilogue)
    t_u = time.perf_counter()
    op_unf = PermutedOperator(A, p_r, p_c, kernel=args.kernel, fold=False)
    torch.cuda.synchronize()
    unf_build_s = time.perf_counter() - t_u
    unf_ms, lam_unf, pi_unf = run(op_unf)
    unf_step = ("fused: seg panel passes, the last with the scatter + norm epilogue" if pi_unf.fused
                else "SpMV + gather + dot + scale")
    del op_unf, pi_unf

    def launches(pi) -> int:  # libsme launches per iteration
        if pi.fused:
            return pi.lay.n_panels
        from paper_2308_00106_b200.kernels import auto_kernel

        kern = auto_kernel(pi.op.B) if pi.op.kernel == "auto" else pi.op.kernel
        if kern == "seg":
            from paper_2308_00106_b200.seg import seg_of

            spmv = seg_of(pi.op.B).n_panels
        else:
            spmv = 2 if kern == "merge" else 1
        return spmv + (1 if pi.op.q is not None else 0) + 2
    step_ms = perm_ms / iters
    gflops = 2 * nnz / (step_ms * 1e-3) / 1e9
    total_perm = perm_s * 1e3 + perm_ms
    # CG (the SPD solver of C5): symmetric permutation by p_r (the folded operator is SPD)
    from paper_2308_00106_b200.iterative import ConjugateGradient

    def run_cg(operator) -> tuple[float, float]:
        cg = ConjugateGradient(operator, P.input_vector(1, n))
        cg.capture(graph_steps)
        for _ in range(args.warmup):
            cg.graph.replay()
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        cg.run(iters)
        c1.record()
        torch.cuda.synchronize()
        return c0.elapsed_time(c1) / iters, cg.residual_norm2

    cg_p_ms, cg_p_rr = run_cg(op)
    cg_u_ms, cg_u_rr = run_cg(PermutedOperator(A, None, None, kernel=args.kernel))
    return {
        "metric": METRIC + " — C5 iterative reuse", "value": round(gflops, 3), "unit": "GFLOP/s",
        "n_gpus": 1, "steps": iters, "warmup": args.warmup, "ms_per_step": round(step_ms, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic 5-point Laplacian; numpy PCG64 permutations seed 7",
        "config": {"workload": cfg["workload"] + ", 1000-step power iteration", "kernel": args.kernel,
                   "graph_steps": graph_steps, "n_rows": n, "nnz": nnz,
                   "permuted_step": ("fused: seg panel passes, the last with the "
                                     + ("scatter + " if pi_p.op.q is not None else "") + "norm epilogue "
                                     "(sme_spmv_seg_epi)" if pi_p.fused else
                                     "SpMV + " + ("gather + " if pi_p.op.q is not None else "") + "dot + scale"),
                   "folded": bool(op.folded),
                   "folded_note": "the per-iteration gather by q = p_r o p_c^-1 is folded into the matrix once: "
                                  "the iterated operator is permute_csr(A, p_r, p_r) (iterative.py docstring)",
                   "unpermuted_step": (f"fused {type(pi_u.lay).__name__} epilogue" if pi_u.fused
                                       else "SpMV + dot + scale (unfused)")},
        "eigenvalue": {"permuted": lam_p, "unpermuted": lam_u, "rel_diff": abs(lam_p - lam_u) / lam_u,
                       "permuted_unfolded": lam_unf},
        "unfolded": {"operator": "P_r A P_c (ROW_COLUMN, fold=False): the gather by q = p_r o p_c^-1 each step",
                     "ms_per_iteration": round(unf_ms / iters, 5),
                     "gflops": round(2 * nnz / (unf_ms / iters * 1e-3) / 1e9, 3),
                     "vs_unpermuted": round(unperm_ms / unf_ms, 4), "vs_folded": round(perm_ms / unf_ms, 4),
                     "permuted_csr_build_ms": round(unf_build_s * 1e3, 2), "step": unf_step},
        "amortisation": {"permutation_setup_ms": round(perm_s * 1e3, 2),
                         "setup": setup_warm, "setup_first_in_process": setup_first,
                         "setup_note": "permutations + folded permuted CSR + seg layout, wall clock with syncs; "
                                       "'setup' = one more matrix in a running process (the per-matrix cost; median of 3), "
                                       "'setup_first_in_process' = the first one (allocator growth, first uses "
                                       "of torch kernels; libsme's modules are preloaded at import)",
                         "permuted_1000_iter_ms": round(perm_ms, 3), "unpermuted_1000_iter_ms": round(unperm_ms, 3),
                         "permuted_total_ms": round(total_perm, 3),
                         "setup_share_of_1000_iter": round(perm_s * 1e3 / perm_ms, 4),
                         "break_even_note": "setup is paid once; per-iteration ratio permuted/unpermuted = "
                                            f"{perm_ms / unperm_ms:.3f}"},
        "x_norm_check": float(torch.linalg.vector_norm(x_p).item()),
        "cg": {"permuted_ms_per_iteration": round(cg_p_ms, 5), "unpermuted_ms_per_iteration": round(cg_u_ms, 5),
               "residual_norm2_permuted": cg_p_rr, "residual_norm2_unpermuted": cg_u_rr,
               "step": "permuted: seg passes with p.Ap fused into the last (sme_spmv_seg_epi_cg); unpermuted: "
                       "CSR-vector SpMV with p.Ap fused (sme_spmv_vector_epi); both + x,r update + p update; "
                       "CUDA graphs",
               "iterations": iters, "rhs": "input_vector(1, n)"},
        "iterations_total": 1 + args.warmup * graph_steps + iters,
        "clocks": clk, "gpu_launches": launches(pi_p) * iters,
    }


def run_iterative_dist(args, cfg, rank: int, world: int) -> dict:
    """C5 on N GPUs: row-sharded power iteration on the folded operator P A P^-1 with the
    iterate's all-gather fused into the SpMV epilogue (peer stores through CUDA IPC
    buffers over NVLink, rowshard.DistributedPowerIteration) + one 8-byte all-reduce
    per step.  Time = max over ranks of the device-timed 1000 steps."""
    import torch
    import torch.distributed as dist

    import paper_2308_00106_b200 as P
    from paper_2308_00106_b200.rowshard import DistributedPowerIteration

    dev = torch.device("cuda", torch.cuda.current_device())
    A = build_matrix(cfg)
    n, nnz = A.n_rows, A.nnz
    iters = 1000
    p, _ = device_perms(n, n)
    dpi = DistributedPowerIteration(A, p, P.input_vector(0, n))
    dpi.run(max(3, args.warmup))
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dpi.run(iters)
    e1.record()
    torch.cuda.synchronize()
    tt = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    lam = dpi.eigenvalue
    dpi.close()
    step_ms = ms / iters
    return {
        "metric": METRIC + " — C5 iterative reuse", "value": round(2 * nnz / (step_ms * 1e-3) / 1e9, 3),
        "unit": "GFLOP/s", "n_gpus": world, "steps": iters, "warmup": args.warmup, "ms_per_step": round(step_ms, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic 5-point Laplacian; PCG64 permutation seed 7",
        "config": {"workload": cfg["workload"] + ", 1000-step power iteration", "n_rows": n, "nnz": nnz,
                   "parallelism": f"row-shard x{world}: iterate all-gather fused into the SpMV epilogue "
                                  f"(CUDA IPC peer stores) + {dist.get_backend()} 8-byte all_reduce per step",
                   "panels_per_shard": dpi.lay.n_panels},
        "eigenvalue": lam, "iterations_total": max(3, args.warmup) + iters, "gpu_launches": dpi.lay.n_panels * iters,
    }


def self_launch(n: int) -> int:
    """`bench.py --gpus N` (N > 1) without a torchrun environment: re-run this script
    under torch.distributed.run with N local ranks on 127.0.0.1 (one process per
    GPU), forwarding the arguments; returns its exit code."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    log(f"[bench] self-launch: {' '.join(cmd)}")
    return subprocess.call(cmd)


def nccl_debug_to_file() -> None:
    """NCCL's INIT log (communicator size per rank) goes to files, not stdout (which
    carries the one JSON line); nccl_init_summary() reads them back."""
    if "NCCL_DEBUG" not in os.environ:
        d = Path(tempfile.gettempdir()) / f"sme_nccl_{os.environ.get('TORCHELASTIC_RUN_ID', 'x')}_{os.environ.get('MASTER_PORT', 'x')}"
        d.mkdir(exist_ok=True)
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        os.environ["NCCL_DEBUG_FILE"] = str(d / "nccl.%h.%p.log")


def nccl_init_summary() -> dict | None:
    """The NCCL INIT lines of every rank of this job ('comm ... rank r nRanks n'), from
    the files nccl_debug_to_file() set up: ranks seen and the nRanks each reported."""
    f = os.environ.get("NCCL_DEBUG_FILE")
    if not f:
        return None
    import glob
    import re

    ranks, sizes, lines = set(), set(), []
    for path in glob.glob(str(Path(f).parent / "nccl.*.log")):
        for ln in Path(path).read_text(errors="replace").splitlines():
            m = re.search(r"rank (\d+) nranks (\d+)", ln, re.IGNORECASE)
            if m:
                ranks.add(int(m.group(1)))
                sizes.add(int(m.group(2)))
                lines.append(ln.strip())
    for ln in lines[:16]:
        log(f"[nccl] {ln}")
    return {"ranks_seen": sorted(ranks), "nranks": sorted(sizes), "init_lines": len(lines),
            "log_files": len(glob.glob(str(Path(f).parent / "nccl.*.log")))}


def dry_run(rank: int, world: int) -> None:
    """Rendezvous + one all_reduce over gloo (no GPU work): the CPU test of the
    self-launch path (tests/test_bench_launch.py)."""
    if world > 1:
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        t = torch.tensor([rank + 1.0])
        dist.all_reduce(t)
        ok = float(t.item()) == world * (world + 1) / 2
        dist.destroy_process_group()
    else:
        ok = True
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "all_reduce_ok": ok, "pid": os.getpid()}), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--kernel", choices=["auto", "seg", "panel", "stream", "vector", "merge"], default="auto")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-scale oracle parity check")
    ap.add_argument("--iterative", action="store_true",
                    help="C5 mode: 1000-step graphed power iteration with permutation amortisation")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch + rendezvous only (CPU/gloo): rank 0 prints the world it saw (tests the self-launch)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.dry_run:
        dry_run(rank, world)
        return

    import torch

    # BENCH_FORCE_SHARDED=1 (under torchrun, any world size incl. 1) takes the sharded
    # multi-GPU path with its process group: with one rank this still runs every NCCL call
    # of that path (all_gather / per-slot broadcasts on the side stream with
    # SME_PIPELINED_EXCHANGE=force, all_reduce, barrier) — the check this 1-GPU pool allows
    dist_mode = world > 1 or bool(os.environ.get("BENCH_FORCE_SHARDED"))
    if dist_mode:
        if not os.environ.get("BENCH_SINGLE_DEVICE") and torch.cuda.device_count() < world:
            raise SystemExit(f"--gpus {world} needs {world} visible GPUs, found {torch.cuda.device_count()}")
        nccl_debug_to_file()

    # BENCH_SINGLE_DEVICE=1 BENCH_DIST_BACKEND=gloo runs every rank on cuda:0 (a
    # functional check of the sharded path on a 1-GPU box; NCCL needs one GPU per rank)
    dev_index = 0 if os.environ.get("BENCH_SINGLE_DEVICE") else local_rank
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    torch.cuda.set_device(dev_index)
    if dist_mode:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    try:
        if args.iterative:
            out = run_iterative(args, cfg) if not dist_mode else run_iterative_dist(args, cfg, rank, world)
            if rank == 0:
                print(json.dumps(out), flush=True)
            return
        out = run_ours(args, cfg, rank, world) if not dist_mode else run_sharded(args, cfg, rank, world)
        if out is not None:
            if dist_mode and backend == "nccl":
                out["nccl_init"] = nccl_init_summary()
            print(json.dumps(out), flush=True)
    finally:
        if dist_mode:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
