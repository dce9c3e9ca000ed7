"""GPU Fisher-Yates apply (shuffle.cu) + host partners: bit-exact with numpy's
Generator(PCG64).permutation, generator state included."""

import numpy as np
import pytest
import torch

import paper_2308_00106_b200 as P
from paper_2308_00106_b200.permute import pcg64_permutation_device

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 17, 1000, 65537, 1_000_003, 12_000_000])
@pytest.mark.parametrize("seed", [0, 99])
def test_device_permutation_is_numpys(n, seed):
    ours_bg, ref_bg = np.random.PCG64(seed), np.random.PCG64(seed)
    got = pcg64_permutation_device(ours_bg, n).cpu().numpy()
    want = np.random.Generator(ref_bg).permutation(n)
    assert np.array_equal(got, want)
    assert ours_bg.state == ref_bg.state


def test_random_permutations_and_strategies_match_numpy():
    specs = [(250_000, 11), (300_001, 12)]
    got = P.random_permutations(specs)
    for p, (n, sd) in zip(got, specs):
        assert np.array_equal(p.forward, np.random.Generator(np.random.PCG64(sd)).permutation(n))
    # riffle: two consecutive device shuffles from one generator
    n, pivot, sd = 10_001, 3_333, 5
    rng = np.random.Generator(np.random.PCG64(sd))
    local = np.concatenate([rng.permutation(pivot), pivot + rng.permutation(n - pivot)])
    from paper_2308_00106_b200.permute import _interleave_forward

    want = _interleave_forward(n, pivot)[local]
    assert np.array_equal(P.riffle_shuffle_permutation(n, pivot, sd).forward, want)
