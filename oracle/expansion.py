"""O6 — the expansion schedule of Alg. 1 l.9-22 with continuous batching (reading D1).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product path.

PAPER.md Alg. 1 l.9-22 and the Fig. 4 walkthrough: nodes whose
prerequisites have finished join the running set R, which "the LLM processes" as one batch; the
Fig. 4 text has Pre(#2) run "in parallel with the LLM Decoding step" of #1 and #3, once Pre(#1) is
done, and Pre(#4) wait for "the LLM Decoding of #3 to finish".  Reading D1:

  round r = one batched LLM step.  It runs
    * the prefill Pre(j) of every point j not yet prefilled whose stage predecessors (O1 stage
      graph: Contextual k->j needs Pre(k), Dependent k->j needs Dec(k)) all
      completed in rounds < r, and
    * one decode token of every point whose Pre completed in a round < r and that still has
      tokens to generate.
  Pre(j) completes in the round it runs; Dec(j) completes in the round that generates j's last
  token (tokens_j = T_j - Lc_j of them), or with its Pre when tokens_j = 0.

Several queries in one batch are scheduled independently on a common round counter.
"""
from .dag import DEC, PRE, stage_graph, validate


def schedule(n, edges, tokens):
    """Point DAG (ids 1..n, edges (from, to, kind)), tokens[j] = decode tokens of point j (dict or
    list indexed by j).  Returns a list of rounds [(pre_points, dec_points)], ids ascending."""
    kinds = validate(n, edges)
    preds = stage_graph(n, kinds)
    tok = {j: int(tokens[j]) for j in range(1, n + 1)}
    pre_done, dec_done, left = {}, {}, dict(tok)
    rounds = []
    r = 0
    while len(dec_done) < n:
        def done_before(stage):
            k, ph = stage
            table = pre_done if ph == PRE else dec_done
            return k in table and table[k] < r
        pre = [j for j in range(1, n + 1) if j not in pre_done
               and all(done_before(s) for s in preds[(j, PRE)])]
        dec = [j for j in range(1, n + 1) if j in pre_done and pre_done[j] < r and j not in dec_done]
        if not pre and not dec:
            raise RuntimeError("schedule stalled (cycle?)")
        for j in pre:
            pre_done[j] = r
            if left[j] == 0:
                dec_done[j] = r
        for j in dec:
            left[j] -= 1
            if left[j] == 0:
                dec_done[j] = r
        rounds.append((pre, dec))
        r += 1
    return rounds


def batch_schedule(queries, tokens):
    """queries: [(n_points, edges, branch0)]; tokens[b] per global branch.  Returns rounds
    [(pre_branches, dec_branches)] over global branch ids (ascending), all queries from round 0."""
    per_q = []
    for n, edges, b0 in queries:
        per_q.append((b0, schedule(n, edges, {j: tokens[b0 + j - 1] for j in range(1, n + 1)})))
    total = max((len(s) for _, s in per_q), default=0)
    out = []
    for r in range(total):
        pre, dec = [], []
        for b0, s in per_q:
            if r < len(s):
                pre += [b0 + j - 1 for j in s[r][0]]
                dec += [b0 + j - 1 for j in s[r][1]]
        out.append((sorted(pre), sorted(dec)))
    return out
