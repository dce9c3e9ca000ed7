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


@pytest.mark.parametrize("n", [1, 2, (1 << 20) - 1, 1 << 20, (1 << 20) + 1, (1 << 20) + 2, 3 * (1 << 20) + 7,
                               9 * (1 << 20) + 3])
@pytest.mark.parametrize("pending", [False, True])
def test_partners_streamed_to_device_are_numpys(n, pending):
    """sme_pcg64_swap_partners_to_device: slot boundaries of the pinned ring (4 MB =
    2^20 partners), a ring that wraps (9 slots > 4), and a generator with a buffered
    uint32 half pending (numpy's has_uint32) — partners equal the host replay's, and the
    generator state equals numpy's after the full shuffle."""
    from paper_2308_00106_b200.permute import pcg64_swap_partners, pcg64_swap_partners_device

    def gen():
        bg = np.random.PCG64(2024 + n)
        if pending:
            np.random.Generator(bg).integers(0, 2**32, dtype=np.uint32)  # leaves a half buffered
            assert bg.state["has_uint32"] == 1
        return bg

    a, b, c = gen(), gen(), gen()
    got = pcg64_swap_partners_device(a, n).cpu().numpy().view(np.uint32)
    want = pcg64_swap_partners(b, n)
    assert np.array_equal(got, want)
    np.random.Generator(c).permutation(n)
    assert a.state == b.state == c.state


@pytest.mark.parametrize("n", [2, 3, 1000, 65_537, 300_001, 2_000_003])
@pytest.mark.parametrize("seed", [0, 7])
@pytest.mark.parametrize("pending", [False, True])
def test_partners_drawn_on_gpu_are_numpys(n, seed, pending):
    """sme_pcg64_swap_partners_gpu (forced at every size): the same partners and the same
    generator state as numpy's shuffle, with and without a buffered uint32 half."""
    from paper_2308_00106_b200.permute import pcg64_swap_partners, pcg64_swap_partners_device

    def gen():
        bg = np.random.PCG64(seed * 1000 + n)
        if pending:
            np.random.Generator(bg).integers(0, 2**32, dtype=np.uint32)
        return bg

    a, b, c = gen(), gen(), gen()
    got = pcg64_swap_partners_device(a, n, gpu_min=2).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, pcg64_swap_partners(b, n))
    np.random.Generator(c).permutation(n)
    assert a.state == b.state == c.state
