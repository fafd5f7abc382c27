"""GPU Oracle Cacher vs the reference: worked-example goldens, golden plan
streams, replay oracles and window properties (reference
tests/test_lookahead.py, tests/test_acceptance.py criteria 1 and 4)."""

from __future__ import annotations

import random

import pytest

from conftest import golden, make_batch, unpack
from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.errors import ConfigurationError
from paper_2202_12429_b200.traces import EmbeddingKey, Schema, ZipfSpec, batchify_columns, generate_columns

pytestmark = pytest.mark.gpu

GOLDEN_PLANS = [
    (1, [3, 9], [(3, 2), (9, 1)]),
    (2, [4], [(3, 3), (4, 2)]),
    (3, [6], [(3, 3), (6, 4)]),
    (4, [1], [(1, 4), (6, 4)]),
]


def k(row: int) -> EmbeddingKey:
    return EmbeddingKey(0, row)


def _lk():
    from paper_2202_12429_b200 import lookahead

    return lookahead


def test_golden_plans(worked_trace):
    plans = list(_lk().plan_trace(worked_trace, 2, 100))
    assert len(plans) == 4
    for plan, (it, pf, ttls) in zip(plans, GOLDEN_PLANS):
        assert plan.iteration == it
        assert plan.prefetch == [k(r) for r in pf]
        assert plan.ttl_updates == [(k(r), t) for r, t in ttls]
        assert plan.lookahead == 2


def test_mirror_trajectory(worked_trace):
    lk = _lk()
    state = lk.new_state(2, 100)
    source = iter(worked_trace)
    mirrors = []
    while lk.emit_next_plan(state, source) is not None:
        mirrors.append(sorted(r for _, r in state.in_cache))
    assert mirrors == [[3], [3], [6], []]


@pytest.mark.parametrize("case", ["L8_cap1000000", "L1_cap1000000", "L16_cap5000", "L32_cap550", "L3_cap1000000"])
def test_small_fixture_plan_streams_match_reference(small_batches, case):
    g = golden("plans_small.json")[case]
    lk = _lk()
    state = lk.new_state(g["lookahead"], g["capacity"])
    src = iter(small_batches)
    plans = []
    while (p := lk.emit_next_plan(state, src)) is not None:
        plans.append(p)
        lk.adapt_on_pressure(state)
    assert len(plans) == len(g["plans"])
    for p, (it, look, pf, ttl) in zip(plans, g["plans"]):
        assert p.iteration == it and p.lookahead == look
        assert p.prefetch == [unpack(x) for x in pf]
        assert p.ttl_updates == [(unpack(x), t) for x, t in ttl]
    s = g["stats"]
    assert (state.lookahead, state.insertions, state.removals, state.peak_occupancy, state.peak_projected) == (
        s["lookahead"], s["insertions"], s["removals"], s["peak_occupancy"], s["peak_projected"])


def test_object_and_columnar_batches_agree(small_batches, small_object_batches):
    lk = _lk()
    a = [(p.prefetch, p.ttl_updates) for p in lk.plan_trace(small_batches, 8, 10**6)]
    b = [(p.prefetch, p.ttl_updates) for p in lk.plan_trace(small_object_batches, 8, 10**6)]
    assert a == b


def test_schema_mode_planner_equals_registry_mode(small_schema, small_batches):
    lk = _lk()
    a = [(p.prefetch, p.ttl_updates, p.lookahead) for p in lk.plan_trace(small_batches, 32, 550)]
    b = [(p.prefetch, p.ttl_updates, p.lookahead) for p in lk.plan_trace(small_batches, 32, 550, schema=small_schema)]
    assert a == b


def replay_plans(batches, plans):
    """Brute-force cache simulation (reference tests/test_lookahead.py:88-106)."""
    cache, misses, states = {}, 0, []
    for batch, plan in zip(batches, plans):
        for key in plan.prefetch:
            cache[key] = -1
        for key, ttl in plan.ttl_updates:
            if key in cache:
                cache[key] = max(cache[key], ttl)
        misses += sum(1 for key in set(batch.unique_keys()) if key not in cache)
        for key in [key for key, ttl in cache.items() if ttl <= batch.iteration]:
            del cache[key]
        states.append(set(cache))
    return misses, states


def test_replay_zero_misses_and_mirror_fidelity():
    lk = _lk()
    rng = random.Random(2024)
    for _ in range(60):
        batches = [make_batch(i, [rng.randrange(rng.randint(1, 12)) for _ in range(rng.randint(1, 5))])
                   for i in range(rng.randint(1, 12))]
        state = lk.new_state(rng.randint(1, 6), 10**6)
        src = iter(batches)
        plans, mirrors = [], []
        while (p := lk.emit_next_plan(state, src)) is not None:
            plans.append(p)
            mirrors.append(state.in_cache)
        misses, replayed = replay_plans(batches, plans)
        assert misses == 0
        assert mirrors == replayed


def test_random_traces_match_oracle_with_pressure():
    """Window property + exact equality with the pinned CPU oracle on random
    traces, capacity small enough to trigger halving (criterion 4 shape)."""
    lk = _lk()
    rng = random.Random(20240)
    for _ in range(80):
        universe = rng.randint(1, 14)
        batches = [make_batch(i, [rng.randrange(universe) for _ in range(rng.randint(1, 5))])
                   for i in range(rng.randint(1, 14))]
        lookahead = rng.randint(1, 6)
        capacity = rng.choice([10**6, rng.randint(max(6, universe), 20)])
        want, wstats = O.plan_stream(batches, lookahead, capacity)
        got = list(lk.plan_trace(batches, lookahead, capacity))
        assert len(got) == len(want)
        occurrences = [set(b.unique_keys()) for b in batches]
        for p, (it, pf, uniq, ttl, _, look) in zip(got, want):
            assert p.iteration == it and p.lookahead == look
            assert p.prefetch == [unpack(int(x)) for x in pf]
            assert p.ttl_updates == [(unpack(int(x)), int(t)) for x, t in zip(uniq, ttl)]
            for key in p.prefetch:
                for back in range(max(0, it - p.lookahead + 1), it):
                    assert key not in occurrences[back]


def test_auto_lookahead():
    lk = _lk()
    assert lk.auto_lookahead([make_batch(i, list(range(10 * i, 10 * i + 10))) for i in range(10)], 35) == 3
    assert lk.auto_lookahead([make_batch(i, list(range(10))) for i in range(100)], 35) == 100
    with pytest.raises(ConfigurationError):
        lk.auto_lookahead([make_batch(0, list(range(50)))], 10)


def test_auto_lookahead_zipf_prefix_union():
    lk = _lk()
    schema = Schema(1, (2_000,), 0, 4)
    rows, labels, dense = generate_columns(ZipfSpec(schema, 1.05, 30 * 128, seed=23))
    batches = batchify_columns(rows, labels, dense, 128)
    assert lk.auto_lookahead(batches, 600) == O.auto_lookahead(batches, 600)


def test_window_not_refilled_past_new_lookahead():
    lk = _lk()
    batches = [make_batch(i, [i, 100 + i, 200 + i]) for i in range(30)]
    state = lk.new_state(8, 12)
    source = iter(batches)
    lk.emit_next_plan(state, source)
    assert len(state.batch_queue) == 7
    lk.adapt_on_pressure(state)
    assert state.lookahead == 4
    lk.emit_next_plan(state, source)
    assert len(state.batch_queue) == 6


def test_ck_plan_stream_matches_reference():
    """12 Criteo-Kaggle batches (26 tables, 16,384 examples, Zipf 1.05) at
    L=7, capacity 1% of rows: every plan bit-exact with the reference planner."""
    lk = _lk()
    g = golden("ck12.json")
    gen = golden("generator.json")["ck12"]
    nt, rpt, nd, dim = gen["schema"]
    schema = Schema(nt, rpt, nd, dim)
    rows, labels, dense = generate_columns(ZipfSpec(schema, gen["exponent"], gen["n"], gen["seed"]))
    batches = batchify_columns(rows, labels, None, 16384)
    state = lk.new_state(7, g["capacity"], schema=schema)
    src = iter(batches)
    shas = []
    while (p := lk.emit_next_plan(state, src)) is not None:
        pf = O.pack([k[0] for k in p.prefetch], [k[1] for k in p.prefetch]) if p.prefetch else []
        uniq = O.pack([k[0] for k, _ in p.ttl_updates], [k[1] for k, _ in p.ttl_updates])
        shas.append(O.plan_sha((p.iteration, pf, uniq, [t for _, t in p.ttl_updates], None, p.lookahead)))
        lk.adapt_on_pressure(state)
    assert shas == g["plans_L7"]["sha"]
    s = g["plans_L7"]["stats"]
    assert (state.insertions, state.removals, state.peak_occupancy, state.peak_projected) == (
        s["insertions"], s["removals"], s["peak_occupancy"], s["peak_projected"])
