"""MIG partition rules (mig_rules.hpp) — mirrors proj/tests/test_rules.cpp:18-133."""
import itertools

import pytest

import support as S
from support import mp

P = mp.Placement


def bitmask_oracle(exclude_4_3: bool):
    """Independent sweep over all subsets of the 14-placement universe (test_rules.cpp:18-61)."""
    positions = {1: range(7), 2: (0, 2, 4), 3: (0, 4), 4: (0,), 7: (0,)}
    memory = {1: 1, 2: 2, 3: 4, 4: 4, 7: 8}
    universe = [P(s, t) for s, v in positions.items() for t in v]

    def legal(ps):
        mask, mem = 0, 0
        for p in ps:
            m = ((1 << p.slices) - 1) << p.start_slot
            if mask & m or p.start_slot + p.slices > 7:
                return False
            mask |= m
            mem += memory[p.slices]
        if mem > 8:
            return False
        sizes = {p.slices for p in ps}
        return not (exclude_4_3 and 3 in sizes and 4 in sizes)

    out = set()
    for bits in range(1, 1 << len(universe)):
        ps = [u for i, u in enumerate(universe) if bits >> i & 1]
        if not legal(ps):
            continue
        if any(legal(ps + [x]) for x in universe if x not in ps):
            continue
        out.add(tuple(sorted(ps)))
    return out


def test_is_legal_partition_examples(impl):  # test_rules.cpp:71-79
    r = mp.PartitionRuleSet.defaults()
    L = lambda ps: mp.is_legal_partition(ps, r, backend=impl)  # noqa: E731
    assert L([P(4, 0), P(2, 4), P(1, 6)])
    assert not L([P(4, 0), P(3, 4)])
    assert not L([P(3, 0), P(3, 4), P(1, 3)])
    assert L([P(3, 0), P(3, 4)])
    assert not L([P(2, 1)])
    assert not L([P(1, 0), P(1, 0)])


def test_exactly_18_maximal_partitions(impl):  # test_rules.cpp:81-105
    r = mp.PartitionRuleSet.defaults()
    parts = mp.enumerate_maximal_partitions(r, backend=impl)
    assert len(parts) == 18
    got = {tuple(sorted(p.placements)) for p in parts}
    assert got == bitmask_oracle(True)
    assert tuple(sorted([P(1, 6), P(2, 4), P(4, 0)])) in got
    gold = S.load_golden("partitions.json")["defaults"]
    assert [[[p.slices, p.start_slot] for p in lp.placements] for lp in parts] == gold


def test_lifting_exclusion_gives_19(impl):  # test_rules.cpp:107-120
    r = mp.PartitionRuleSet.defaults()
    r.hard_exclusions = set()
    parts = mp.enumerate_maximal_partitions(r, backend=impl)
    assert len(parts) == 19
    assert {tuple(sorted(p.placements)) for p in parts} == bitmask_oracle(False)
    gold = S.load_golden("partitions.json")["no_exclusion"]
    assert [[[p.slices, p.start_slot] for p in lp.placements] for lp in parts] == gold


def test_maximality_is_airtight(impl):  # test_rules.cpp:122-133
    r = mp.PartitionRuleSet.defaults()
    universe = [P(s, t) for s, v in r.slot_positions.items() for t in v if t + s <= 7]
    for part in mp.enumerate_maximal_partitions(r, backend=impl):
        for extra in universe:
            if extra in part.placements:
                continue
            assert not mp.is_legal_partition(part.placements + [extra], r, backend=impl)
