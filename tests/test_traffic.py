"""Product-side serving-traffic generators and latency aggregates
(include/symsim/traffic.hpp), through the kvs C ABI:
the distributions configs 4 and 5 need (Poisson think times, Zipf(1.2)
session popularity) and the p50 / SLO aggregation of the serving metric."""
import numpy as np
import pytest

from paper_2412_16434_b200 import kvstore as K


def test_zipf_turns_follow_the_rank_law():
    t = K.zipf_turns(600, 1.2, 64.0, 2, seed=505)
    want = np.maximum(2, np.rint(64.0 / np.arange(1, 601) ** 1.2)).astype(np.int32)
    assert sorted(t.tolist(), reverse=True) == want.tolist()  # a permutation of the rank law
    assert t.sum() == want.sum()
    # rank-frequency slope on log-log over the ranks above the floor is -s
    top = np.sort(t)[::-1][:20].astype(float)
    slope = np.polyfit(np.log(np.arange(1, 21)), np.log(top), 1)[0]
    assert abs(slope + 1.2) < 0.1, slope
    # deterministic per seed, and the seed moves the ranking
    assert np.array_equal(t, K.zipf_turns(600, 1.2, 64.0, 2, seed=505))
    assert not np.array_equal(t, K.zipf_turns(600, 1.2, 64.0, 2, seed=506))


def test_poisson_gaps_are_exponential():
    g = K.poisson_gaps(200_000, 0.5, seed=404) / 1e9
    assert abs(g.mean() - 0.5) < 0.01
    assert abs(g.std() / g.mean() - 1.0) < 0.02  # CV of an exponential is 1
    assert abs((g > 0.5).mean() - np.exp(-1)) < 0.005  # memoryless tail
    assert (g >= 0).all()


@pytest.mark.parametrize("q", [0.0, 0.5, 0.9, 0.99, 1.0])
def test_percentile_matches_numpy(q):
    rng = np.random.default_rng(1)
    for n in (1, 2, 7, 1000):
        v = rng.lognormal(0, 1, n)
        assert K.percentile(v, q) == pytest.approx(float(np.percentile(v, q * 100)), rel=1e-12)
    assert K.percentile([], 0.5) == 0.0


def test_rps_within_slo_picks_the_best_point_meeting_it():
    sweep = [(32, 10.0, 0.010), (64, 19.0, 0.012), (128, 30.0, 0.020), (256, 41.0, 0.060)]
    assert K.rps_within_slo(sweep, 0.020) == 30.0
    assert K.rps_within_slo(sweep, 0.011) == 10.0
    assert K.rps_within_slo(sweep, 0.005) == 0.0
