"""C++ cache core (memory.py semantics) against the reference's recorded traces (CPU)."""
import numpy as np
import pytest

from paper_2510_12357_b200 import CapacityDeadlock, ExpertId as E, HbmCache, TransferChannel
from paper_2510_12357_b200.memory import HIT, IN_FLIGHT, ISSUED


def test_golden_traces(golden):
    meta, _ = golden
    for tr in meta["cache_traces"]:
        cache, ch = HbmCache(tr["slots"]), TransferChannel(tr["t_xfer"])
        for op in tr["ops"]:
            key = E(*op["key"])
            k = op["op"]
            try:
                if k in ("req", "spec"):
                    r = cache.request(key, op["now"], ch, speculative=(k == "spec"))
                    assert (None if r is None else [r.status, r.ready_time]) == op["out"]
                elif k == "pin":
                    cache.pin(key)
                elif k == "unpin":
                    cache.unpin(key)
                elif k == "token_end":
                    cache.token_end()
                else:
                    v = cache.evict_lru(op["n"], op["now"] if op["use_now"] else None)
                    assert [[x.layer, x.expert] for x in v] == op["out"]
            except CapacityDeadlock:
                assert op["out"] == "deadlock"
            except ValueError:
                assert op["out"] == "valueerror"
            assert [[x.layer, x.expert] for x in cache.entries()] == op["entries"]
        s = cache.stats
        assert [s.hits, s.coalesced, s.issued, s.evictions, s.deferrals] == tr["stats"]
        assert ch.transfers_issued == tr["transfers"]


def test_hand_examples():
    cache, ch = HbmCache(slots=4), TransferChannel(t_xfer=4.0)
    first = cache.request(E(0, 0), 0.0, ch)
    assert first.status == ISSUED and first.ready_time == 4.0
    assert cache.request(E(0, 0), 1.0, ch).status == IN_FLIGHT
    assert cache.request(E(0, 0), 4.0, ch).status == HIT
    assert ch.transfers_issued == 1
    assert cache.ready_time(E(0, 0)) == 4.0
    assert cache.resident(E(0, 0), 3.0) is False and cache.resident(E(0, 0), 4.0) is True


def test_pins_deadlock_and_deferral():
    cache, ch = HbmCache(1), TransferChannel(0.5)
    cache.request(E(0, 0), 0.0, ch)
    cache.pin(E(0, 0))
    assert cache.request(E(1, 0), 10.0, ch, speculative=True) is None
    assert cache.stats.deferrals == 1
    with pytest.raises(CapacityDeadlock):
        cache.request(E(1, 0), 10.0, ch)
    cache.token_end()
    assert cache.request(E(1, 0), 10.0, ch).status == ISSUED


def test_evict_lru_all_or_nothing():
    cache, ch = HbmCache(4), TransferChannel(0.5)
    for i in range(4):
        cache.request(E(0, i), float(i), ch)
    for i in range(3):
        cache.pin(E(0, i))
    with pytest.raises(ValueError, match="only 1"):
        cache.evict_lru(2)
    assert len(cache) == 4
    assert cache.evict_lru(1) == [E(0, 3)]


def test_accounting_partition_and_capacity():
    rng = np.random.default_rng(5)
    cache, ch = HbmCache(8), TransferChannel(3.0)
    now, n = 0.0, 500
    for _ in range(n):
        now += float(rng.uniform(0.0, 2.0))
        cache.request(E(int(rng.integers(0, 4)), int(rng.integers(0, 8))), now, ch, speculative=True)
        assert len(cache) <= 8
    s = cache.stats
    assert s.deferrals > 0
    assert s.total_requests() == n - s.deferrals
    assert s.issued == ch.transfers_issued


def test_slots_are_a_permutation():
    """Physical slot assignment: resident entries always occupy distinct slots < capacity."""
    rng = np.random.default_rng(9)
    cache, ch = HbmCache(6), TransferChannel(1.0)
    now = 0.0
    for _ in range(400):
        now += 1.0
        r = cache.request(E(int(rng.integers(0, 3)), int(rng.integers(0, 8))), now, ch, speculative=True)
        slots = [cache.slot_of(e) for e in cache.entries()]
        assert len(set(slots)) == len(slots) and all(0 <= s < 6 for s in slots)
