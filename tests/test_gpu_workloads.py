"""The device-built BASELINE workloads are bit-identical to the reference
recipes (tests/helpers.py, pinned by tests/golden/digests.json), and the
sharded config-4 slices factor to the recipe ranks."""
import numpy as np
import pytest

import oracle as O
import paper_1112_5717_b200 as G
from paper_1112_5717_b200 import workloads as WL
from tests.helpers import c2_style, c4_batch

pytestmark = pytest.mark.gpu


def test_c4_dev_matches_recipe():
    mats, ranks = c4_batch(6)
    dev, dranks = WL.c4_dev(4096, lo=0, hi=6)
    assert dranks == ranks
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), mats)
    # a middle slice (the shard of another rank) is the same bytes
    dev2, _ = WL.c4_dev(4096, lo=3, hi=6)
    assert np.array_equal(dev2.cpu().numpy().view(np.uint32), mats[3:6])


def test_c2_dev_matches_recipe():
    m, n, inner, seed, p = 300, 500, 100, 7, 65521
    dev = WL.c2_dev(m, n, inner, seed, p)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), c2_style(m, n, inner, seed, p))


def test_c4_shards_factor_to_recipe_ranks():
    total = 20
    seen = []
    for rank in range(3):
        lo, hi = WL.shard_range(total, rank, 3)
        dev, ranks = WL.c4_dev(total, lo=lo, hi=hi)
        rk, rrp, sig = G.cup_batched_dev(dev, hi - lo, 256, 256, 8388593)
        assert [int(x) for x in rk] == ranks
        seen += list(range(lo, hi))
    assert seen == list(range(total))
