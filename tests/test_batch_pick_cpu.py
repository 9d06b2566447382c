"""lbx_batch_pick (include/lbx/batcher.h, rule in include/lbx/batch_pick.h): the batch size with the
lowest GPU time per request; no curve = greedy."""
import pytest

import paper_2605_19385_b200 as lbx


def test_greedy_without_curve():
    assert lbx.batch_pick(None, 5, 32) == 5
    assert lbx.batch_pick(None, 50, 32) == 32
    assert lbx.batch_pick(None, 0, 32) == 0


def test_flat_or_rising_curve_picks_one():
    flat = [8.0 * b for b in range(1, 33)]
    rising = [8.0 * b * (1 + 0.001 * b) for b in range(1, 33)]
    for curve in (flat, rising):
        for q in (1, 2, 7, 32, 100):
            assert lbx.batch_pick(curve, q, 32) == 1


def test_fixed_overhead_curve_batches():
    engine = [30.0 + 2.6 * b for b in range(1, 33)]  # a per-launch cost: bigger batches pay
    assert lbx.batch_pick(engine, 7, 32) == 7
    assert lbx.batch_pick(engine, 100, 32) == 32
    assert lbx.batch_pick(engine, 100, 8) == 8


def test_small_gains_need_two_percent():
    curve = [10.0, 19.9, 29.85]  # 0.5% / 0.5% per-request gains: below the 2% bar
    assert lbx.batch_pick(curve, 3, 32) == 1
    curve = [10.0, 19.0, 29.5]    # 5% better at 2, 3 is worse per request than 2
    assert lbx.batch_pick(curve, 3, 32) == 2
    # past the curve: extended linearly (same time per request as its last point)
    assert lbx.batch_pick([10.0, 19.0], 6, 32) == 2


@pytest.mark.parametrize("q,mb", [(1, 1), (3, 1), (1, 32)])
def test_bounds(q, mb):
    assert 1 <= lbx.batch_pick([5.0, 9.0, 12.0], q, mb) <= min(q, mb)
