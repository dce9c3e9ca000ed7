"""The reference's own measurement protocol with the GPU kernels plugged in
(INTEGRATION.md level 1).

`spmv_entropy.bench.run_experiment` (reference bench.py:174-251) is the UNMODIFIED
reference from baseline/_ref (baseline/install_ref.sh).  It builds the permuted
operands with its own numpy code, verifies the round trip, times every KernelSpec
with its own time_kernel and checks each kernel's last y against its own
y_expected at CORRECTNESS_RTOL = 1e-12.  The GPU KernelSpecs of
paper_2308_00106_b200.bench.gpu_kernels() run next to its default_kernels.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not (REF / "spmv_entropy" / "__init__.py").is_file():
        pytest.skip("baseline/_ref not installed (run baseline/install_ref.sh)")
    sys.path.insert(0, str(REF))
    import spmv_entropy
    import spmv_entropy.bench

    assert Path(spmv_entropy.__file__).resolve().is_relative_to(REF.resolve())
    return spmv_entropy


def c1(ref):
    """C1: the reference test generator (pkg/tests/conftest.py:10-16), default_rng(0), 10k x 10k, 0.001."""
    rng = np.random.default_rng(0)
    total = 10_000 * 10_000
    cells = rng.choice(total, size=100_000, replace=False)
    values = rng.random(100_000) * 2.0 - 1.0
    return ref.CooMatrix(10_000, 10_000, cells // 10_000, cells % 10_000, values)


@pytest.mark.parametrize("strategy", ["ROW_COLUMN_PERMUTE", "COLUMN_GRADIENT"])
def test_run_experiment_with_gpu_kernels(ref, strategy):
    import paper_2308_00106_b200.bench as gb

    m = c1(ref)
    kind = getattr(ref.StrategyKind, strategy)
    kernels = ref.bench.default_kernels(2, m.n_rows) + [
        ref.bench.KernelSpec(s.kernel_id, s.fn, s.workers) for s in gb.gpu_kernels(max_workers=2)]
    cfg = ref.RunConfig(target_seconds=0.05)
    res = ref.bench.run_experiment(m, kind, kernels, repeats=2, master_seed=0, config=cfg, matrix_name="C1")
    gpu = [t for t in res.trials if t.kernel_id.startswith("gpu_")]
    assert len(gpu) == 2 * len(gb.gpu_kernels(max_workers=2))
    for t in res.trials:
        assert t.correctness_ok, (t.kernel_id, t.workers, t.repeat)
        assert t.gflops > 0, (t.kernel_id, t.workers)
    rec = res.record
    for s in gb.gpu_kernels(max_workers=2):
        assert rec.kernels[s.kernel_id].max > 0
