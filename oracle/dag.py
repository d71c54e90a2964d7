"""O1 — DAG validation, stage graph, expansion levels and per-branch segment lists.

Pure Python, integers only.  Follows, step by step:
  * Alg. 1 l.1-7: nodes 1..N, directed typed edges i -> j.
  * §3.3: Null / Contextual / Dependent; Null = no edge (reading S2).
  * Alg. 1 l.8: split each node into Prefill and Decode stages;
    stage edges per SPEC.md:51-54 (reading S3):
        Pre(i) -> Dec(i);  Contextual k->j: Pre(k) -> Pre(j);  Dependent k->j: Dec(k) -> Pre(j).
  * Eq. (1) generalised to levels: a stage with no predecessor is at
    level 0; otherwise 1 + max level of its predecessors (longest-path layering, reading S10).
  * Eq. (2)/(3) read at KV level as segment lists (readings S6-S9):
        [PREFIX] + deps (ascending point id) + [OWN(j)].

Error codes mirror include/orion.h: 1 INVALID_ARG, 2 CYCLE, 3 UNKNOWN_POINT.
"""

INVALID_ARG, CYCLE, UNKNOWN_POINT = 1, 2, 3
NULL, CONTEXTUAL, DEPENDENT = 0, 1, 2
PRE, DEC = 0, 1
SEG_PREFIX, SEG_CONTENT, SEG_FULL, SEG_OUTPUT, SEG_OWN = 0, 1, 2, 3, 4
ANCESTORS, PARENTS_EQ3 = 0, 1


class DagError(Exception):
    def __init__(self, code, info):
        super().__init__(f"dag error {code}: {info}")
        self.code = code
        self.info = info


def validate(n, edges):
    """Return the set of materialised edges {(k, j): kind} (Null dropped, duplicates merged,
    Dependent dominating a Contextual on the same pair — reading S5)."""
    if n < 1:
        raise DagError(INVALID_ARG, [])
    for idx, (a, b, kind) in enumerate(edges):
        if kind not in (NULL, CONTEXTUAL, DEPENDENT):
            raise DagError(INVALID_ARG, [idx])
        if not (1 <= a <= n and 1 <= b <= n):
            raise DagError(UNKNOWN_POINT, [idx])
    kinds = {}
    for a, b, kind in edges:
        if kind == NULL:
            continue
        kinds.setdefault((a, b), set()).add(kind)
    return kinds


def stage_graph(n, kinds):
    """Predecessor sets of every stage (i, PRE|DEC), exactly SPEC.md:51-54's three rules."""
    preds = {(i, ph): set() for i in range(1, n + 1) for ph in (PRE, DEC)}
    for i in range(1, n + 1):
        preds[(i, DEC)].add((i, PRE))
    for (k, j), ks in kinds.items():
        if CONTEXTUAL in ks:
            preds[(j, PRE)].add((k, PRE))
        if DEPENDENT in ks:
            preds[(j, PRE)].add((k, DEC))
    return preds


def find_cycle(n, kinds):
    """DFS over the point graph; returns one cycle's point ids in order, or None."""
    succ = {i: sorted(j for (k, j) in kinds if k == i) for i in range(1, n + 1)}
    color = {i: 0 for i in range(1, n + 1)}
    stack = []

    def dfs(u):
        color[u] = 1
        stack.append(u)
        for v in succ[u]:
            if color[v] == 1:
                return stack[stack.index(v):]
            if color[v] == 0:
                c = dfs(v)
                if c:
                    return c
        stack.pop()
        color[u] = 2
        return None

    for i in range(1, n + 1):
        if color[i] == 0:
            c = dfs(i)
            if c:
                return list(c)
    return None


def levels(n, edges):
    """(pre_level[1..n], dec_level[1..n], n_levels) by memoised longest-path recursion."""
    kinds = validate(n, edges)
    cyc = find_cycle(n, kinds)
    if cyc:
        raise DagError(CYCLE, cyc)
    preds = stage_graph(n, kinds)
    memo = {}

    def level(s):
        if s not in memo:
            memo[s] = 0 if not preds[s] else 1 + max(level(p) for p in preds[s])
        return memo[s]

    pre = [level((i, PRE)) for i in range(1, n + 1)]
    dec = [level((i, DEC)) for i in range(1, n + 1)]
    return pre, dec, 1 + max(dec)


def waves(n, edges):
    """Wavefronts: stages grouped by level, each sorted by (point id, Pre < Dec)."""
    pre, dec, nl = levels(n, edges)
    out = [[] for _ in range(nl)]
    for i in range(1, n + 1):
        out[pre[i - 1]].append((i, PRE))
        out[dec[i - 1]].append((i, DEC))
    return [sorted(w) for w in out]


def _reaches(preds, src, dst):
    """True iff a stage path src ~> dst exists (src == dst counts)."""
    seen, todo = set(), [dst]
    while todo:
        s = todo.pop()
        if s == src:
            return True
        if s in seen:
            continue
        seen.add(s)
        todo.extend(preds[s])
    return False


def segment_lists(n, edges, policy=ANCESTORS):
    """Per-branch segment lists {j: [(kind, point), ...]} for j = 1..n."""
    kinds = validate(n, edges)
    cyc = find_cycle(n, kinds)
    if cyc:
        raise DagError(CYCLE, cyc)
    if policy not in (ANCESTORS, PARENTS_EQ3):
        raise DagError(INVALID_ARG, [])
    preds = stage_graph(n, kinds)
    parents = {j: sorted(k for (k, jj) in kinds if jj == j) for j in range(1, n + 1)}
    out = {}
    for j in range(1, n + 1):
        deps = []
        if policy == ANCESTORS:
            anc, todo = set(), list(parents[j])
            while todo:
                a = todo.pop()
                if a not in anc:
                    anc.add(a)
                    todo.extend(parents[a])
            for a in sorted(anc):
                full = _reaches(preds, (a, DEC), (j, PRE))
                deps.append((SEG_FULL if full else SEG_CONTENT, a))
        else:
            for k in parents[j]:
                dep = DEPENDENT in kinds[(k, j)]
                deps.append((SEG_OUTPUT if dep else SEG_CONTENT, k))
        out[j] = [(SEG_PREFIX, 0)] + deps + [(SEG_OWN, j)]
    return out
