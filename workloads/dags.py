"""Dependency DAG families (edge lists only).

An edge is (from, to, kind): `to` depends on `from` (Alg. 1
l.5-6; SPEC.md:37 Relation{from=predecessor k, to=successor j}).  Points are
numbered 1..n.  Kinds: 0 Null, 1 Contextual, 2 Dependent
(§3.3 "Null, Contextual, and Dependent").
"""
import random

EDGE_NULL, EDGE_CONTEXTUAL, EDGE_DEPENDENT = 0, 1, 2
C, D = EDGE_CONTEXTUAL, EDGE_DEPENDENT


def diamond():
    """Fig. 1(a) (PAPER.md:113 caption): 1->2, 1->3 Contextual; 2->4, 3->4 Dependent."""
    return 4, [(1, 2, C), (1, 3, C), (2, 4, D), (3, 4, D)]


def fig4():
    """Fig. 4 walkthrough (§3.3): 1->2 Contextual, 3->4 Dependent."""
    return 4, [(1, 2, C), (3, 4, D)]


def mixed8():
    """Mixed chain/fan-out 8-point DAG used by configs c2/c3 (SURVEY.md §8(c) goldens)."""
    return 8, [(1, 2, D), (2, 3, D), (1, 4, C), (1, 5, C), (1, 6, C), (4, 7, D), (5, 7, D),
               (3, 8, D), (7, 8, D), (6, 8, C)]


def mixed16():
    """16-point DAG used by config c4: 1->{2,3,4,5} C; four Dependent chains of 3;
    {10,11}->14, {12,13}->15, {14,15}->16 Dependent."""
    e = [(1, k, C) for k in (2, 3, 4, 5)]
    for s in (2, 3, 4, 5):
        e += [(s, s + 4, D), (s + 4, s + 8, D)]
    e += [(10, 14, D), (11, 14, D), (12, 15, D), (13, 15, D), (14, 16, D), (15, 16, D)]
    return 16, e


def wide(n=64):
    """n independent points (SugRes-like; ParExp of PAPER.md:200)."""
    return n, []


edgeless = wide


def chain(n=64, kind=D):
    """1->2->...->n chain; Dependent = ComLog-like, Contextual = TexSeq-like."""
    return n, [(i, i + 1, kind) for i in range(1, n)]


def random_dag(rng: random.Random, n: int, p: float = 0.3, kinds=(C, D), null_frac=0.0):
    """Random DAG over a random topological order; edges i->j only forward in that order."""
    order = list(range(1, n + 1))
    rng.shuffle(order)
    edges = []
    for a in range(n):
        for b in range(a + 1, n):
            if rng.random() < p:
                k = EDGE_NULL if rng.random() < null_frac else rng.choice(kinds)
                edges.append((order[a], order[b], k))
    rng.shuffle(edges)
    return n, edges


DAGS = {
    "diamond": diamond,
    "fig4": fig4,
    "mixed8": mixed8,
    "mixed16": mixed16,
    "wide64": lambda: wide(64),
    "chain64": lambda: chain(64, D),
}
