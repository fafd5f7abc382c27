"""Public-API rows pinned to reference outputs (tests/golden/api.json, made by
tests/golden/make_golden.py gen_api from the reference itself):

* DynamicCache content_checksum / canonical_digest / evict_expired / drain
  and counters after a scripted scenario (reference cache.py:99-286,
  tests/test_cache.py:165-171),
* the trainer object wrappers local_gradients / combine_gradients /
  apply_updates / split_sync_sets (reference trainer.py:56-179),
* ShardedStore.shard_of placement (reference store.py:80-88),
* format_plan / parse_plan and the CLI's worked-example records (reference
  lookahead.py:162-189, tests/test_cli.py:97-103).

CPU tests pin the oracle restatement and the host-only functions; the GPU
tests replay the same operations on the B200 objects.
"""

from __future__ import annotations

import base64

import numpy as np
import pytest

from conftest import golden, unpack
from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Example

G = golden("api.json")


def _f32(bits) -> np.ndarray:
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def _b64(s: str, dtype, shape) -> np.ndarray:
    return np.frombuffer(base64.b64decode(s), dtype=dtype).reshape(shape)


def _scenario(sc):
    """Decoded inputs of one cache scenario."""
    ops, dim = sc["ops"], sc["dim"]
    keys = np.asarray(ops["keys"], dtype=np.uint64)
    n = keys.size
    vals = _b64(ops["values"], "<f4", (n, dim))
    ttls = np.asarray(ops["ttls"], dtype=np.int64)
    upd_idx, new_ttl = ops["ttl_updates"]
    row_idx, rows_b64, mask = ops["update_rows"]
    rows = _b64(rows_b64, "<f4", (len(row_idx), dim))
    wl_i, wl_bits = ops["write_local"]
    return dict(keys=keys, vals=vals, ttls=ttls, half=ops["half"], upd_idx=upd_idx, new_ttl=new_ttl,
                row_idx=row_idx, rows=rows, mask=np.asarray(mask, dtype=bool), wl_i=wl_i, wl_val=_f32(wl_bits))


def _released_equal(got, want):
    """got: [(packed key, f32 row, dirty)]; want: golden list or {n, sha}."""
    if isinstance(want, dict):
        assert len(got) == want["n"]
        import hashlib

        h = hashlib.sha256()
        h.update(np.asarray([k for k, _, _ in got], dtype="<u8").tobytes())
        h.update(np.asarray([v for _, v, _ in got], dtype="<f4").reshape(len(got), -1).tobytes())
        h.update(np.asarray([d for _, _, d in got], dtype=np.uint8).tobytes())
        assert h.hexdigest() == want["sha"]
    else:
        assert [[k, np.asarray(v, dtype=np.float32).view(np.uint32).tolist(), bool(d)] for k, v, d in got] == want


def _state_equal(st, want):
    assert st["len"] == want["len"]
    assert st["checksum"] == want["checksum"]
    assert st["digest"] == want["digest"]
    for f in ("keys", "ttl", "dirty"):
        if f in want:
            assert st[f] == want[f], f


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("name", ["cache_small", "cache_large"])
def test_oracle_cache_checksum_and_digest(name):
    sc = G[name]
    s = _scenario(sc)
    c = O.DictCache()
    h = s["half"]

    def state():
        ks, tt, dd, _ = c.arrays()
        return {"len": len(c.ent), "checksum": c.checksum(), "digest": c.digest(), "keys": ks.tolist(),
                "ttl": tt.tolist(), "dirty": dd.tolist()}

    c.prefetch(s["keys"][:h], s["vals"][:h], s["ttls"][:h])
    c.prefetch(s["keys"][h:], s["vals"][h:], s["ttls"][h:])
    _state_equal(state(), sc["after_prefetch"])
    c.set_ttl(s["keys"][s["upd_idx"]], s["new_ttl"])
    c.update(s["keys"][s["row_idx"]], s["rows"], s["mask"])
    c.update([s["keys"][s["wl_i"]]], [s["wl_val"]], [True])
    _state_equal(state(), sc["after_update"])
    _released_equal(c.release(lambda e: e[1] <= 2), sc["evict_2"])
    _state_equal(state(), sc["after_evict"])
    _released_equal(c.release(lambda e: True), sc["drain"])
    assert c.checksum() == 0 == sc["after_drain"]["checksum"]
    assert c.digest() == sc["after_drain"]["digest"]


def test_shard_of_matches_reference():
    from paper_2202_12429_b200.store import shard_of_keys

    g = G["shard_of"]
    keys = np.asarray(g["keys"], dtype=np.uint64)
    t, r = keys >> np.uint64(44), keys & np.uint64((1 << 44) - 1)
    for ns, want in g["shards"].items():
        assert O.shard_of(t, r, int(ns)).tolist() == want
        assert shard_of_keys(t, r, int(ns)).tolist() == want


def test_plan_text_format_and_cli_records():
    from paper_2202_12429_b200.lookahead import CachePlan, format_plan, parse_plan

    g = G["plan_text"]
    # the reference CLI's golden records (tests/test_cli.py:98-103)
    assert g["worked"] == ["iter=1 prefetch=0:3,0:9 ttl=0:3@2,0:9@1", "iter=2 prefetch=0:4 ttl=0:3@3,0:4@2",
                           "iter=3 prefetch=0:6 ttl=0:3@3,0:6@4", "iter=4 prefetch=0:1 ttl=0:1@4,0:6@4"]
    for line, rec in zip(g["small_L8"], g["small_L8_parsed"]):
        p = parse_plan(line)
        assert [p.iteration, p.lookahead, [(k[0] << 44) | k[1] for k in p.prefetch],
                [[(k[0] << 44) | k[1], t] for k, t in p.ttl_updates]] == rec
        assert format_plan(p) == line
        q = CachePlan(rec[0], [unpack(x) for x in rec[2]], [(unpack(x), t) for x, t in rec[3]], 5)
        assert format_plan(q) == line
    assert format_plan(parse_plan("iter=7 prefetch= ttl=")) == g["empty"]
    from paper_2202_12429_b200.errors import RecordParseError

    with pytest.raises(RecordParseError):
        parse_plan("iter=x prefetch= ttl=")


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cache_small", "cache_large"])
def test_gpu_cache_scenario(name):
    from paper_2202_12429_b200.cache import DynamicCache

    sc = G[name]
    s = _scenario(sc)
    c = DynamicCache(sc["capacity"], sc["dim"])
    keys = [unpack(int(k)) for k in s["keys"]]
    h = s["half"]

    def state(compact):
        st = {"len": len(c), "checksum": c.content_checksum(), "digest": c.canonical_digest()}
        if not compact:
            ks = sorted(c.key_set())
            st.update(keys=[(k[0] << 44) | k[1] for k in ks], ttl=[c.ttl_of(k) for k in ks],
                      dirty=[c.is_dirty(k) for k in ks])
        return st

    compact = "keys" not in sc["after_prefetch"]
    c.apply_prefetch(keys[:h], s["vals"][:h], dict(zip(keys[:h], s["ttls"][:h].tolist())))
    c.apply_prefetch(keys[h:], s["vals"][h:], dict(zip(keys[h:], s["ttls"][h:].tolist())))
    _state_equal(state(compact), sc["after_prefetch"])
    c.apply_ttl_updates([(keys[i], t) for i, t in zip(s["upd_idx"], s["new_ttl"])])
    slots = c.resolve_slots([keys[i] for i in s["row_idx"]])
    c.update_rows(slots, s["rows"], s["mask"])
    c.write_local_update(keys[s["wl_i"]], s["wl_val"])
    _state_equal(state(compact), sc["after_update"])
    _released_equal([((k[0] << 44) | k[1], v, d) for k, v, d in c.evict_expired(2)], sc["evict_2"])
    _state_equal(state(compact), sc["after_evict"])
    drained = c.drain()
    assert drained, "drain of a non-empty cache"
    _released_equal([((k[0] << 44) | k[1], v, d) for k, v, d in drained], sc["drain"])
    _state_equal(state(compact), sc["after_drain"])
    want = sc["counters"]
    assert (c.insertions, c.evictions, c.peak_occupancy) == (want["insertions"], want["evictions"], want["peak"])


@pytest.mark.gpu
def test_gpu_trainer_wrappers():
    from paper_2202_12429_b200.cache import DynamicCache
    from paper_2202_12429_b200.trainer import (StubModelConfig, apply_updates, combine_gradients, local_gradients,
                                               split_sync_sets)

    g = G["trainer"]
    lr, cv, cl = g["cfg"]
    cfg = StubModelConfig(lr=lr, c_value=cv, c_label=cl)
    values = {unpack(k): _f32(b) for k, b in g["values"]}
    ranks = [[Example(lab, (), tuple(unpack(k) for k in ks)) for lab, ks in exs] for exs in g["ranks"]]
    per = [local_gradients(exs, values, cfg) for exs in ranks]
    for got, want in zip(per, g["local"]):
        assert [[(k[0] << 44) | k[1], v.view(np.uint32).tolist()] for k, v in got.items()] == want
    comb = combine_gradients(per)
    assert [[(k[0] << 44) | k[1], v.view(np.uint32).tolist()] for k, v in comb.items()] == g["combined"]
    c = DynamicCache(32, g["dim"])
    ukeys = sorted(values)
    c.apply_prefetch(ukeys, np.stack([values[k] for k in ukeys]), {k: 9 for k in ukeys})
    comb_z = dict(comb)
    comb_z[unpack(g["zero_key"])] = np.zeros(g["dim"], dtype=np.float32)
    upd = apply_updates(c, comb_z, cfg)
    assert sorted((k[0] << 44) | k[1] for k in upd) == g["updated"]
    assert not c.is_dirty(unpack(g["zero_key"]))
    _state_equal({"len": len(c), "checksum": c.content_checksum(), "digest": c.canonical_digest(),
                  "keys": [(k[0] << 44) | k[1] for k in sorted(c.key_set())],
                  "ttl": [c.ttl_of(k) for k in sorted(c.key_set())],
                  "dirty": [c.is_dirty(k) for k in sorted(c.key_set())]}, g["after_apply"])
    crit, bg = split_sync_sets(upd, {unpack(k) for k in g["next"]})
    assert [(k[0] << 44) | k[1] for k in crit] == g["critical"]
    assert [(k[0] << 44) | k[1] for k in bg] == g["background"]


@pytest.mark.gpu
def test_gpu_worked_example_plan_records(worked_trace):
    from paper_2202_12429_b200.lookahead import format_plan, plan_trace

    assert [format_plan(p) for p in plan_trace(worked_trace, 2, 100)] == G["plan_text"]["worked"]


@pytest.mark.gpu
def test_gpu_small_fixture_plan_records(small_batches):
    from paper_2202_12429_b200.lookahead import format_plan, plan_trace

    got = [format_plan(p) for p, _ in zip(plan_trace(small_batches, 8, 5000), range(12))]
    assert got == G["plan_text"]["small_L8"]
