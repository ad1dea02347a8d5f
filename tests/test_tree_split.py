"""Host logic of the distributed coarse solve: the subtree-to-rank
mapping of a supernode tree (mdd_tree_split, shard.cpp split_tree), checked on
CPU against what any valid mapping must satisfy and against brute force."""
import itertools

import numpy as np
import pytest

from paper_2311_18783_b200.solver import tree_split


def _random_tree(rng, n):
    # parents after children (the supernode order of the factor plans)
    par = np.full(n, -1, np.int32)
    for g in range(n - 1):
        par[g] = rng.integers(g + 1, n)
    return par


def _check_valid(par, owner, nranks):
    n = len(par)
    for g in range(n):
        p = par[g]
        if owner[g] == -1:
            # the top is closed upwards
            assert p < 0 or owner[p] == -1
        else:
            assert 0 <= owner[g] < nranks
            # a non-top supernode's parent is top or on the same rank (whole subtrees)
            assert p < 0 or owner[p] in (-1, owner[g])
    if nranks > 1:
        assert set(owner[owner >= 0]) == set(range(nranks)), "every rank gets a subtree"


def _work(par, cost, owner, nranks):
    top = cost[owner == -1].sum()
    return max(cost[owner == r].sum() for r in range(nranks)) + top


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_perfect_binary_tree_splits_evenly(nranks):
    par, cost = [], []

    def build(d, p):
        me = len(par)
        par.append(p)
        cost.append(100 * (6 - d))
        if d < 6:
            build(d + 1, me)
            build(d + 1, me)
    build(0, -1)
    par, cost = np.array(par, np.int32), np.array(cost, np.int64)
    o = tree_split(par, cost, nranks)
    _check_valid(par, o, nranks)
    if nranks in (1, 2, 4, 8):   # powers of two: the subtree-to-subcube split is exact
        counts = np.bincount(o[o >= 0], minlength=nranks)
        assert len(set(counts)) == 1 and (o == -1).sum() == nranks - 1


@pytest.mark.parametrize("seed", range(6))
def test_random_trees_valid_and_no_worse_than_any_single_cut(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(30, 200))
    par = _random_tree(rng, n)
    cost = rng.integers(1, 1000, n).astype(np.int64)
    for nranks in (2, 3, 4):
        nleaf = len(set(range(n)) - set(par[par >= 0]))
        if nleaf < nranks:
            continue
        o = tree_split(par, cost, nranks)
        _check_valid(par, o, nranks)
        w = _work(par, cost, o, nranks)
        assert w <= cost.sum()  # never worse than one rank doing everything
        # brute force over "top = the root only" assignments of the root's subtrees
        roots = np.where(par < 0)[0]
        if len(roots) == 1:
            r = roots[0]
            kids = np.where(par == r)[0]
            if nranks <= len(kids) <= 8:
                sub = {}
                for k in kids:
                    s, stack = 0, [k]
                    while stack:
                        g = stack.pop()
                        s += cost[g]
                        stack.extend(np.where(par == g)[0])
                    sub[k] = s
                best = min(max(sum(sub[k] for k, a in zip(kids, asg) if a == b) for b in range(nranks))
                           for asg in itertools.product(range(nranks), repeat=len(kids))
                           if len(set(asg)) == nranks) + cost[r]
                # LPT is a 4/3-approximation of the best split at that top
                assert w <= best * 4 / 3 + 1


def test_forest_and_errors():
    par = np.array([-1, -1, -1], np.int32)
    o = tree_split(par, np.ones(3, np.int64), 3)
    assert sorted(o) == [0, 1, 2]
    with pytest.raises(Exception):
        tree_split(np.array([1, 0], np.int32), np.ones(2, np.int64), 2)   # a cycle
    with pytest.raises(Exception):
        tree_split(np.array([-1], np.int32), np.ones(1, np.int64), 2)    # fewer leaves than ranks
