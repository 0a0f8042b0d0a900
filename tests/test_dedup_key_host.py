"""Host check of the property the pipeline dedupe key rests on (DESIGN.md §5
"Pipeline dedupe"): within a class, the micro-batch counts of the replicas are
non-increasing in the replica index and take at most three consecutive values
(Hamilton floor + one seat + one residual step), so the sub-class vector is
base + [u < a] + [u < b].  Checked on the decoded plans (hsim_decode, host
only) of seeded samples of every BASELINE config and of tiny spaces."""
import numpy as np
import pytest

import hsim_inputs as H
from paper_2508_05370_b200 import hsim


def _check(cfg, count):
    s = hsim.Sim(cfg, host_only=True)
    N = s.space_size()
    idx = H.sample_indices(N, min(count, N))
    seen = 0
    for i in idx:
        d = s.decode(int(i))
        if d["status"] != 0:
            continue
        for cl in d["classes"]:
            mb = cl["mb"]
            assert all(mb[r] >= mb[r + 1] for r in range(len(mb) - 1)), (i, mb)
            assert mb[0] - mb[-1] <= 2, (i, mb)
            assert min(mb) >= 1
            seen += 1
    return seen


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_mb_vector_shape_configs(n):
    assert _check(H.get(n), 1500) > 0


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_mb_vector_shape_tiny(seed):
    assert _check(H.tiny_random(seed), 400) >= 0
