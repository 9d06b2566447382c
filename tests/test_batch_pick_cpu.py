"""lbx_batch_pick (include/lbx/batcher.h, rule in include/lbx/batch_pick.h): the batch size that
minimises the mean completion time of the queued requests; no curve = greedy."""
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


def test_short_queues_need_large_gains():
    """The rule minimises the mean completion time of the queued requests: a batch holds its first
    requests back until the whole batch finishes, so with a short queue small per-request gains do
    not pay (round 1's rule batched at a 2% gain)."""
    curve = [10.0, 19.9, 29.85]  # 0.5% per-request gains
    assert lbx.batch_pick(curve, 3, 32) == 1
    curve = [10.0, 19.0, 29.5]    # 5% better per request at 2 -- but 3 queued requests finish
    assert lbx.batch_pick(curve, 3, 32) == 1  # sooner on average one at a time (20 vs 22.3 ms)
    assert lbx.batch_pick([10.0, 19.0], 6, 32) == 1  # past the curve: extended linearly


def test_backlog_turns_to_throughput():
    """From max_batch / 2 queued requests on (a burst) the rule picks the lowest time per request,
    a larger batch winning by 2%; below that, one at a time on a flat curve."""
    assert lbx.batch_pick([10.0, 19.0, 29.5], 200, 3) == 2
    measured = [8.89, 17.49, 26.1, 34.68]  # a flat B200 curve: 2.5% cheaper per request at 4
    assert lbx.batch_pick(measured, 4, 32) == 1
    assert lbx.batch_pick(measured, 15, 32) == 1
    assert lbx.batch_pick(measured, 16, 32) == 3  # 3 is 2.1% cheaper per request than 1; 4 not 2% below 3
    assert lbx.batch_pick(measured, 400, 32) == 3


@pytest.mark.parametrize("q,mb", [(1, 1), (3, 1), (1, 32)])
def test_bounds(q, mb):
    assert 1 <= lbx.batch_pick([5.0, 9.0, 12.0], q, mb) <= min(q, mb)
