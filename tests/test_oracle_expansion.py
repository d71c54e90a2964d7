"""Pins for oracle O6 (expansion schedule, reading D1 of Alg. 1 l.9-22): the Fig. 4 walkthrough's
order, closed forms for wide and chain DAGs, and -- independent of O6's code -- the
identity with O1's longest-path stage levels when every point decodes one token."""
import random

import pytest

from oracle import dag as D, expansion as E
from workloads import dags as W


def rounds_of(n, sched):
    pre, dec = {}, {}
    for r, (p, d) in enumerate(sched):
        for j in p:
            pre[j] = r
        for j in d:
            dec.setdefault(j, []).append(r)
    return pre, dec


def test_fig4_walkthrough_order():
    # "simultaneously initiates the LLM Prefilling step for #1 and #3"; "the LLM
    # Prefilling for #2 ... executes in parallel with the LLM Decoding step for #1 and #3";
    # "For #4, the system waits for the LLM Decoding of #3 to finish, then ... Prefilling for #4".
    t = 3
    n, edges = W.fig4()
    s = E.schedule(n, edges, {j: t for j in range(1, n + 1)})
    assert s[0] == ([1, 3], [])
    assert s[1] == ([2], [1, 3])
    pre, dec = rounds_of(n, s)
    assert dec[3] == [1, 2, 3] and pre[4] == 4              # right after #3's last token
    assert dec[2] == [2, 3, 4] and dec[4] == [5, 6, 7] and len(s) == 8


@pytest.mark.parametrize("t", [0, 1, 5])
def test_wide_and_chain_closed_forms(t):
    n = 6
    s = E.schedule(*W.wide(n), {j: t for j in range(1, n + 1)})
    assert len(s) == 1 + t and s[0][0] == list(range(1, n + 1))
    assert all(d == list(range(1, n + 1)) for _, d in s[1:])
    # Dependent chain: Pre(i) at (i-1)(t+1) (t = 0: a point's Dec completes with its Pre)
    s = E.schedule(*W.chain(n, D.DEPENDENT), {j: t for j in range(1, n + 1)})
    pre, dec = rounds_of(n, s)
    assert [pre[i] for i in range(1, n + 1)] == [(i - 1) * (t + 1) for i in range(1, n + 1)]
    assert len(s) == (n * (t + 1) if t else n)
    # Contextual chain: Pre(i) at i-1, everyone decodes t consecutive rounds after its Pre
    s = E.schedule(*W.chain(n, D.CONTEXTUAL), {j: t for j in range(1, n + 1)})
    pre, dec = rounds_of(n, s)
    assert [pre[i] for i in range(1, n + 1)] == list(range(n))
    for i in range(1, n + 1):
        assert dec.get(i, []) == list(range(pre[i] + 1, pre[i] + 1 + t))


def test_unit_tokens_equal_stage_levels():
    # One decode token per point: the ASAP round of every stage is its longest-path level in the
    # stage graph (O1, pinned against brute-force path enumeration in test_oracle_dag.py).
    rng = random.Random(11)
    for trial in range(200):
        n = rng.randint(1, 12)
        edges = W.random_dag(random.Random(trial), n, p=rng.choice([0.2, 0.4, 0.7]))[1]
        pre_lv, dec_lv = D.levels(n, edges)[:2]
        s = E.schedule(n, edges, {j: 1 for j in range(1, n + 1)})
        pre, dec = rounds_of(n, s)
        for j in range(1, n + 1):
            assert pre[j] == pre_lv[j - 1], (trial, j)
            assert dec[j] == [dec_lv[j - 1]], (trial, j)


def test_random_invariants_and_batch():
    rng = random.Random(5)
    for trial in range(100):
        n = rng.randint(1, 10)
        edges = W.random_dag(random.Random(100 + trial), n, p=0.4)[1]
        tok = {j: rng.randint(0, 4) for j in range(1, n + 1)}
        s = E.schedule(n, edges, tok)
        pre, dec = rounds_of(n, s)
        kinds = D.validate(n, edges)
        for (k, j), ks in kinds.items():
            if D.CONTEXTUAL in ks:
                assert pre[k] < pre[j]
            if D.DEPENDENT in ks:
                end_k = dec[k][-1] if dec.get(k) else pre[k]
                assert end_k < pre[j]
        for j in range(1, n + 1):                    # tokens decode in consecutive rounds
            assert dec.get(j, []) == list(range(pre[j] + 1, pre[j] + 1 + tok[j]))
    # a batch of queries = the per-query schedules on one round counter, global branch ids
    q = [(4, W.fig4()[1], 0), (3, W.chain(3, D.DEPENDENT)[1], 4)]
    tokens = [2] * 7
    b = E.batch_schedule(q, tokens)
    s0 = E.schedule(4, W.fig4()[1], {j: 2 for j in range(1, 5)})
    s1 = E.schedule(3, W.chain(3, D.DEPENDENT)[1], {j: 2 for j in range(1, 4)})
    assert len(b) == max(len(s0), len(s1))
    for r in range(len(b)):
        want_p = ([j - 1 for j in s0[r][0]] if r < len(s0) else []) + ([j + 3 for j in s1[r][0]] if r < len(s1) else [])
        want_d = ([j - 1 for j in s0[r][1]] if r < len(s0) else []) + ([j + 3 for j in s1[r][1]] if r < len(s1) else [])
        assert b[r] == (sorted(want_p), sorted(want_d))
