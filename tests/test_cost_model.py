"""Cost model restatement (paper_2408_06213_b200/cost_model.py) against values computed by
the reference's cost_model.py (tests/golden/make_golden.py) and its own known answers
(test_cost_model.py:18-120).  Host-only; no device."""

import math

import pytest


@pytest.fixture(scope="module")
def CM():
    from paper_2408_06213_b200 import cost_model

    return cost_model


def test_crossovers_and_schedules_match_reference(CM, golden):
    for rec in golden["cost_model"]:
        p = CM.CostParams(rng_cost=rec["rng_cost"], div_cost=rec["div_cost"], word_bits=rec["bits"])
        for k, nk in rec["nk"].items():
            if nk is None:
                with pytest.raises(CM.NoCrossover):
                    CM.find_nk(int(k), p)
            else:
                assert CM.find_nk(int(k), p) == nk, (rec, k)
        mb = 6 if rec["bits"] == 64 else 4
        if isinstance(rec["schedule6"], str):
            with pytest.raises(Exception):
                CM.build_schedule(p, mb)
        else:
            assert [list(e) for e in CM.build_schedule(p, mb).entries] == rec["schedule6"]
        for n, k, c in rec["costs"]:
            assert CM.cost_per_roll(n, k, p) == c  # same float expression, bit-identical


def test_reference_known_answers(CM):
    import paper_2408_06213_b200 as B

    assert math.isclose(CM.cost_per_roll(1000, 1), 3.0, rel_tol=1e-12)
    assert math.isclose(CM.cost_per_roll(1000, 2), 2.0, rel_tol=1e-9)
    assert CM.cost_per_roll(26573, 4) <= CM.cost_per_roll(26573, 3)
    assert CM.cost_per_roll(26574, 4) > CM.cost_per_roll(26574, 3)
    assert CM.build_schedule().entries == B.DEFAULT_SCHEDULE.entries
    assert CM.build_schedule(max_batch=2).entries == ((1 << 30, 2),)
    assert CM.build_schedule(max_batch=8).entries[-1] == (128, 8)
    with pytest.raises(CM.NoCrossover):
        CM.find_nk(2, CM.CostParams(rng_cost=0.001, div_cost=0.001, word_bits=4))
    for bad in (dict(rng_cost=0), dict(div_cost=-1)):
        with pytest.raises(ValueError):
            CM.CostParams(**bad)
    with pytest.raises(ValueError):
        CM.find_nk(1)
    with pytest.raises(ValueError):
        CM.build_schedule(max_batch=1)


def test_gpu_schedule_is_valid_and_opt_in(CM):
    import os

    import paper_2408_06213_b200 as B

    if not os.path.exists(CM._OPCOST):
        pytest.skip("no measured B200 op costs yet")
    for gen in ("pcg64", "lehmer", "chacha"):
        s = CM.gpu_schedule(gen)
        assert isinstance(s, B.ShuffleSchedule) and s.max_batch == 6
        p = CM.gpu_cost_params(gen)
        assert p.rng_cost > 0 and p.div_cost > 0
    assert B.DEFAULT_SCHEDULE.entries == ((1 << 30, 2), (1 << 19, 3), (1 << 14, 4), (1 << 11, 5), (1 << 9, 6))
