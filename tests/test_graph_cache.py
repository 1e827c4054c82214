"""GraphCache policy: ports of graph_cache_test.cpp and acceptance c8 run
against the C++ GraphCache the sessions use (placeholder graphs, no GPU)."""
import random

import pytest

from paper_2604_23467_b200 import graphrt as g


class RefCache:
    """Independent brute-force model (graph_cache_test.cpp:28-70)."""

    def __init__(self, cap, lru):
        self.cap, self.lru, self.m, self.seq = cap, lru, {}, 0

    def lookup(self, k):
        if k not in self.m:
            return False
        e = self.m[k]
        e["use"] += 1
        self.seq += 1
        e["last"] = self.seq
        return True

    def insert(self, k):
        if k in self.m:
            self.seq += 1
            self.m[k].update(use=0, ins=self.seq, last=self.seq)
            return None
        victim = None
        if len(self.m) == self.cap:
            victim = min(self.m, key=lambda key: ((self.m[key]["last"] if self.lru else self.m[key]["use"]),
                                                  self.m[key]["ins"]))
            del self.m[victim]
        self.seq += 1
        self.m[k] = dict(use=0, ins=self.seq, last=self.seq)
        return victim


def test_hit_miss_accounting():
    c = g.GraphCache(4)
    assert not c.lookup(1)
    c.insert(1)
    assert c.lookup(1)
    assert c.use_count(1) == 1
    st = c.stats()
    assert (st.hits, st.misses, st.inserts) == (1, 1, 1)


@pytest.mark.parametrize("policy", [g.EvictionPolicy.LeastUsed, g.EvictionPolicy.LeastRecentlyUsed])
@pytest.mark.parametrize("cap", [1, 2, 4, 8])
def test_eviction_matches_bruteforce_oracle(policy, cap):
    """acceptance_main.cpp:427-502 (c8): 10000 random ops, every eviction matches."""
    c = g.GraphCache(cap, policy)
    ref = RefCache(cap, policy == g.EvictionPolicy.LeastRecentlyUsed)
    r = random.Random(2026 + cap)
    for op in range(10000):
        k = r.randint(1, 12)
        if r.randint(0, 9) < 6:
            assert c.lookup(k) == ref.lookup(k), op
        else:
            assert c.insert(k) == ref.insert(k), op
    assert c.size() == len(ref.m)
    for k, e in ref.m.items():
        assert c.contains(k) and c.use_count(k) == e["use"]


def test_replacement_resets_use_count_without_eviction():
    c = g.GraphCache(2)
    c.insert(1)
    c.insert(2)
    c.lookup(1)
    assert c.insert(1) is None  # replacement never evicts
    assert c.use_count(1) == 0
    assert c.size() == 2


def test_key_mismatch():
    c = g.GraphCache(2)
    with pytest.raises(g.Error) as e:
        c.insert(3, graph_key=4)
    assert e.value.code == g.Errc.KeyMismatch


def test_warmup_and_capacity():
    c = g.GraphCache(8)
    assert c.precapture_warmup(1, 5) == 5
    assert c.precapture_warmup(3, 7) == 2  # cached keys are skipped
    assert c.precapture_warmup(5, 4) == 0  # empty range
    with pytest.raises(g.Error) as e:
        g.GraphCache(4).precapture_warmup(1, 5)
    assert e.value.code == g.Errc.WarmupExceedsCapacity
    with pytest.raises(g.Error) as e:
        g.GraphCache(0)
    assert e.value.code == g.Errc.InvalidConfig


def test_release_inactive():
    """graph_cache_test.cpp:207-232: warm entries untouched in a session are dropped."""
    c = g.GraphCache(16)
    c.precapture_warmup(1, 6)
    c.begin_session()
    c.lookup(2)
    c.insert(9)
    assert c.release_inactive() == 5  # 1,3,4,5,6
    assert c.contains(2) and c.contains(9) and not c.contains(1)
    assert c.stats().releases == 5
    with pytest.raises(g.Error) as e:
        c.use_count(1)
    assert e.value.code == g.Errc.EmptyCache
