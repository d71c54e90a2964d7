"""Pins for oracle O1 (levels, waves, segment lists) against the paper/SPEC goldens,
brute force on small random DAGs and structural invariants (SURVEY.md §8(c) pin table)."""
import itertools
import json
import os
import random

import pytest

from oracle import dag as O
from workloads import dags as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dag_goldens.json")))


def _stage_edges_by_rules(n, edges):
    """Independently coded rule applier, used to pin the oracle's stage graph."""
    out = {((i, 0), (i, 1)) for i in range(1, n + 1)}
    for a, b, k in edges:
        if k == 1:
            out.add(((a, 0), (b, 0)))
        elif k == 2:
            out.add(((a, 1), (b, 0)))
    return out


def _oracle_stage_edges(n, edges):
    preds = O.stage_graph(n, O.validate(n, edges))
    return {(p, s) for s, ps in preds.items() for p in ps}


def _ready(preds, completed):
    return sorted(s for s, ps in preds.items() if s not in completed and ps <= completed)


def _t(x):
    return [tuple(tuple(y) if isinstance(y, list) else y for y in z) for z in x]


@pytest.mark.parametrize("name", ["fig4", "chain2_dep", "single"])
def test_stage_edges_golden(name):
    g = GOLD[name]
    got = _oracle_stage_edges(g["n"], [tuple(e) for e in g["edges"]])
    want = {(tuple(a), tuple(b)) for a, b in g["stage_edges"]}
    assert got == want


def test_fig4_ready_sets_golden():
    g = GOLD["fig4"]
    preds = O.stage_graph(4, O.validate(4, [tuple(e) for e in g["edges"]]))
    assert _ready(preds, set()) == [tuple(s) for s in g["ready_empty"]]
    assert _ready(preds, {(1, 0)}) == [tuple(s) for s in g["ready_after_pre1"]]
    assert _ready(preds, set(preds)) == []


@pytest.mark.parametrize("name", ["fig4", "edgeless2", "chain2_dep", "single"])
def test_waves_golden(name):
    g = GOLD[name]
    got = O.waves(g["n"], [tuple(e) for e in g["edges"]])
    assert got == [[tuple(s) for s in w] for w in g["waves"]]


def test_fig4_paper_timeline_levels():
    # Pre1 || Pre3 first; Pre2 runs alongside Dec1/Dec3; Pre4 waits for Dec3.
    pre, dec, nl = O.levels(*W.fig4())
    assert pre[0] == pre[2] == 0
    assert dec[0] == pre[1] == dec[2] == 1
    assert pre[3] > dec[2] and dec[3] > pre[3]
    assert nl == 4


def test_fig1_parents_and_eq3():
    g = GOLD["fig1"]
    edges = [tuple(e) for e in g["edges"]]
    lists = O.segment_lists(4, edges, O.PARENTS_EQ3)
    assert [p for (k, p) in lists[4][1:-1]] == g["parents_4"]
    assert lists[2][1:-1] == [tuple(x) for x in g["eq3_point2"]]
    assert lists[4][1:-1] == [tuple(x) for x in g["eq3_point4"]]


def test_two_cycle_golden():
    g = GOLD["two_cycle"]
    with pytest.raises(O.DagError) as ei:
        O.levels(g["n"], [tuple(e) for e in g["edges"]])
    assert ei.value.code == g["error"]
    assert sorted(ei.value.info) == [1, 2]


def test_validation_errors():
    with pytest.raises(O.DagError) as ei:
        O.levels(3, [(1, 2, 1), (1, 5, 1)])
    assert ei.value.code == O.UNKNOWN_POINT and ei.value.info == [1]
    with pytest.raises(O.DagError) as ei:
        O.levels(3, [(1, 2, 7)])
    assert ei.value.code == O.INVALID_ARG and ei.value.info == [0]
    with pytest.raises(O.DagError) as ei:
        O.levels(3, [(2, 2, 2)])
    assert ei.value.code == O.CYCLE and ei.value.info == [2]
    with pytest.raises(O.DagError):
        O.levels(0, [])
    # Null edges are dropped ("no direct logical connection"), even self-loops.
    assert O.levels(2, [(1, 2, 0), (2, 2, 0)]) == O.levels(2, [])
    # duplicates merge; Dependent dominates Contextual on the same pair
    assert O.segment_lists(2, [(1, 2, 1), (1, 2, 2), (1, 2, 2)]) == O.segment_lists(2, [(1, 2, 2)])


# ---------------------------------------------------------------- brute force

def _all_paths_longest(n, edges):
    """Longest path (in edges) ending at each stage, by enumerating every path from every stage."""
    E = _stage_edges_by_rules(n, edges)
    succ = {}
    for a, b in E:
        succ.setdefault(a, []).append(b)
    stages = [(i, ph) for i in range(1, n + 1) for ph in (0, 1)]
    best = {s: 0 for s in stages}

    def walk(s, length):
        best[s] = max(best[s], length)
        for t in succ.get(s, []):
            walk(t, length + 1)

    for s in stages:
        walk(s, 0)
    return best


def _point_paths(n, edges):
    """All simple point paths (list of edges) between every pair, by DFS enumeration."""
    kinds = {}
    for a, b, k in edges:
        if k:
            kinds.setdefault((a, b), set()).add(k)
    succ = {}
    for (a, b) in kinds:
        succ.setdefault(a, []).append(b)
    paths = {}

    def dfs(start, node, first_kinds):
        for nxt in succ.get(node, []):
            fk = kinds[(node, nxt)] if first_kinds is None else first_kinds
            paths.setdefault((start, nxt), []).append(fk)
            dfs(start, nxt, fk)

    for a in range(1, n + 1):
        dfs(a, a, None)
    return paths


def _random_dags(count, nmax, seed):
    rng = random.Random(seed)
    for _ in range(count):
        n = rng.randint(1, nmax)
        yield W.random_dag(rng, n, p=rng.choice([0.2, 0.4, 0.7]), null_frac=0.2)


def test_levels_brute_force():
    for n, edges in _random_dags(300, 7, 11):
        pre, dec, nl = O.levels(n, edges)
        best = _all_paths_longest(n, edges)
        assert pre == [best[(i, 0)] for i in range(1, n + 1)]
        assert dec == [best[(i, 1)] for i in range(1, n + 1)]
        assert nl == 1 + max(best.values())


def test_ancestor_lists_brute_force():
    # FULL(a) iff some point path a -> ... -> j starts with a Dependent edge (reading S8).
    for n, edges in _random_dags(300, 7, 12):
        lists = O.segment_lists(n, edges, O.ANCESTORS)
        paths = _point_paths(n, edges)
        for j in range(1, n + 1):
            want = []
            for a in range(1, n + 1):
                fk = paths.get((a, j))
                if fk:
                    full = any(2 in s for s in fk)
                    want.append((O.SEG_FULL if full else O.SEG_CONTENT, a))
            assert lists[j] == [(O.SEG_PREFIX, 0)] + want + [(O.SEG_OWN, j)]


def test_eq3_lists_brute_force():
    for n, edges in _random_dags(200, 8, 13):
        lists = O.segment_lists(n, edges, O.PARENTS_EQ3)
        for j in range(1, n + 1):
            par = sorted({a for a, b, k in edges if b == j and k})
            want = [(O.SEG_OUTPUT if any(a == k and b == j and kk == 2 for a, b, kk in edges)
                     else O.SEG_CONTENT, k) for k in par]
            assert lists[j] == [(O.SEG_PREFIX, 0)] + want + [(O.SEG_OWN, j)]


def test_wave_invariants_and_ready_monotonicity():
    for n, edges in _random_dags(200, 10, 14):
        ws = O.waves(n, edges)
        E = _stage_edges_by_rules(n, edges)
        pos = {s: w for w, wave in enumerate(ws) for s in wave}
        assert len(pos) == 2 * n
        for a, b in E:
            assert pos[a] < pos[b]          # concatenation is a topological order, waves antichains
        # every stage in wave w>0 has a predecessor in wave w-1 (longest-path layering is tight)
        for a in pos:
            if pos[a] > 0:
                assert any(pos[p] == pos[a] - 1 for (p, b) in E if b == a)
        preds = O.stage_graph(n, O.validate(n, edges))
        order = [s for w in ws for s in w]
        for cut in range(len(order)):
            c1, c2 = set(order[:cut]), set(order[:cut + 1])
            for s in _ready(preds, c1):
                assert s in _ready(preds, c2) or s in c2


def test_cycle_reports_a_real_cycle():
    rng = random.Random(5)
    for _ in range(200):
        n = rng.randint(2, 8)
        n_, edges = W.random_dag(rng, n, p=0.5)
        # add a back edge to close a cycle
        a, b = rng.sample(range(1, n + 1), 2)
        edges = edges + [(a, b, 2), (b, a, 1)]
        with pytest.raises(O.DagError) as ei:
            O.levels(n, edges)
        cyc = ei.value.info
        assert ei.value.code == O.CYCLE
        es = {(x, y) for x, y, k in edges if k}
        assert all((cyc[i], cyc[(i + 1) % len(cyc)]) in es for i in range(len(cyc)))


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("n", [1, 2, 7, 64])
def test_closed_forms(n):
    wide = O.segment_lists(*W.wide(n))
    assert all(wide[j] == [(0, 0), (4, j)] for j in range(1, n + 1))
    assert sum(map(len, wide.values())) == 2 * n
    assert O.segment_lists(*W.wide(n), O.PARENTS_EQ3) == wide
    dep = O.segment_lists(*W.chain(n, 2))
    assert all(dep[j] == [(0, 0)] + [(2, a) for a in range(1, j)] + [(4, j)] for j in range(1, n + 1))
    assert sum(map(len, dep.values())) == n * (n + 3) // 2
    ctx = O.segment_lists(*W.chain(n, 1))
    assert all(ctx[j] == [(0, 0)] + [(1, a) for a in range(1, j)] + [(4, j)] for j in range(1, n + 1))
    eq3 = O.segment_lists(*W.chain(n, 2), O.PARENTS_EQ3)
    assert sum(map(len, eq3.values())) == 2 * n + (n - 1)
    # chain levels: Dependent chain has 2n levels; edgeless has 2; Contextual chain has n+1
    assert O.levels(*W.chain(n, 2))[2] == 2 * n
    assert O.levels(*W.wide(n))[2] == 2
    assert O.levels(*W.chain(n, 1))[2] == n + 1
