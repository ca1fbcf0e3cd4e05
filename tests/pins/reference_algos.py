"""Independent pins for the oracle (pure Python, tiny inputs only).

None of this code is shared with ``oracle/`` or the CUDA path. Each function is
a *different* algorithm (or the bare definition evaluated per vertex) that fixes
a result the oracle must reproduce:

- ``simulate_valuation``: the definition of val^{σ,τ} evaluated
  by following each play separately; ⊤ for infinite plays; cycle max priority.
- ``zielonka``: the textbook recursive algorithm (cited) for the
  winning partition of Thm 1.
- ``brute_force_winners``: enumerate all positional σ, τ (positional determinacy,
  PAPER.md:304-309), maxio over each lasso's cycle.
- ``bellman_ford_br``: val^σ as shortest paths to the sink under ⊑ with odd
  priorities as negative weights.
- ``brute_force_br``: val^σ as the pointwise ⊑-minimum over every τ
  (unique by PAPER.md:392-394).
- ``si_with_bellman_ford``: the outer loop of Algorithm 1
  with best responses from Bellman-Ford. Since val^σ is unique, the σ
  trajectory, outer pass count and σ* depend only on the Even switch rule, so
  they must equal the oracle's.

Games here are "internal" games: owner[v] (0 Even / 1 Odd), prio[v] (values),
adj[v] (ordered successor lists); Even vertices have an implicit sink candidate
(SINK = -1) ordered last (SURVEY.md §8(c) reading 3).
"""
from __future__ import annotations

import itertools

SINK = -1
TOP = None  # ⊤


def simulate_valuation(prio, succ, D):
    """val^{σ,τ}(v) for every v by following the play from v (definition)."""
    n = len(succ)
    index = {p: i for i, p in enumerate(D)}
    vals, cdom = [], []
    for v in range(n):
        seen = {}
        path = []
        x = v
        while x != SINK and x not in seen:
            seen[x] = len(path)
            path.append(x)
            x = succ[x]
        if x == SINK:
            c = [0] * len(D)
            for y in path:
                c[index[prio[y]]] += 1
            vals.append(tuple(c))
            cdom.append(-1)
        else:
            vals.append(TOP)
            cdom.append(max(prio[y] for y in path[seen[x]:]))
    return vals, cdom


def leq_strict(a, b, D):
    """a ⊏ b, ⊤ maximal; None = ⊤."""
    if a is TOP:
        return False
    if b is TOP:
        return True
    for i in range(len(D) - 1, -1, -1):
        if a[i] != b[i]:
            if D[i] % 2 == 0:
                return a[i] < b[i]
            return a[i] > b[i]
    return False


def _add_unit(val, i, D):
    if val is TOP:
        return TOP
    c = list(val) if val is not None else [0] * len(D)
    c[i] += 1
    return tuple(c)


def bellman_ford_br(owner, prio, adj, sigma, D, return_rounds=False):
    """val^σ via Bellman-Ford relaxation from ⊤. With return_rounds,
    also the number of synchronous rounds computed (the last one changes nothing)."""
    n = len(owner)
    index = {p: i for i, p in enumerate(D)}
    zero = tuple([0] * len(D))
    val = [TOP] * n

    def get(u):
        return zero if u == SINK else val[u]

    for rnd in range(n + 2):
        changed = False
        new = list(val)
        for v in range(n):
            if owner[v] == 0:
                cand = get(sigma[v])
            else:
                cand = TOP
                for u in adj[v]:
                    if leq_strict(get(u), cand, D):
                        cand = get(u)
            nv = _add_unit(cand, index[prio[v]], D)
            if nv != val[v]:
                changed = True
            new[v] = nv
        val = new
        if not changed:
            return (val, rnd + 1) if return_rounds else val
    raise AssertionError("Bellman-Ford did not converge: negative (odd) cycle")


def brute_force_br(owner, prio, adj, sigma, D, limit=1 << 14):
    """Pointwise ⊑-min of val^{σ,τ} over every Odd positional τ.
    Returns (minimum valuations, list of τ attaining all minima at once)."""
    odd = [v for v in range(len(owner)) if owner[v] == 1]
    choices = [adj[v] for v in odd]
    total = 1
    for c in choices:
        total *= len(c)
    assert total <= limit, "too many Odd strategies"
    best = None
    runs = []
    for pick in itertools.product(*choices):
        succ = list(sigma)
        for v, u in zip(odd, pick):
            succ[v] = u
        vals, _ = simulate_valuation(prio, succ, D)
        runs.append((pick, vals))
        if best is None:
            best = list(vals)
        else:
            for v in range(len(vals)):
                if leq_strict(vals[v], best[v], D):
                    best[v] = vals[v]
    attaining = [dict(zip(odd, pick)) for pick, vals in runs if vals == best]
    return best, attaining


def si_with_bellman_ford(owner, prio, adj, D, max_outer=10_000):
    """Outer loop of Algorithm 1 with Bellman-Ford best responses.
    Returns (σ*, outer passes, val^{σ*}, σ trajectory)."""
    n = len(owner)
    sigma = [SINK if owner[v] == 0 else None for v in range(n)]
    zero = tuple([0] * len(D))
    traj = [list(sigma)]
    outer = 0
    while True:
        outer += 1
        assert outer <= max_outer
        val = bellman_ford_br(owner, prio, adj, sigma, D)

        def get(u):
            return zero if u == SINK else val[u]

        changed = 0
        new = list(sigma)
        for v in range(n):
            if owner[v] != 0:
                continue
            cands = list(adj[v]) + [SINK]
            b = cands[0]
            for u in cands[1:]:
                if leq_strict(get(b), get(u), D):
                    b = u
            if leq_strict(get(sigma[v]), get(b), D):
                new[v] = b
                changed += 1
        if changed == 0:
            return sigma, outer, val, traj
        sigma = new
        traj.append(list(sigma))


def attractor(player, target, V, owner, adj):
    attr = set(target)
    changed = True
    while changed:
        changed = False
        for v in V:
            if v in attr:
                continue
            succ = [u for u in adj[v] if u in V]
            if owner[v] == player:
                ok = any(u in attr for u in succ)
            else:
                ok = all(u in attr for u in succ)
            if ok:
                attr.add(v)
                changed = True
    return attr


def zielonka(owner, prio, adj, V=None):
    """Recursive algorithm; returns (W_Even, W_Odd) as sets."""
    if V is None:
        V = set(range(len(owner)))
    if not V:
        return set(), set()
    p = max(prio[v] for v in V)
    player = p % 2
    A = attractor(player, {v for v in V if prio[v] == p}, V, owner, adj)
    W = list(zielonka(owner, prio, adj, V - A))
    if not W[1 - player]:
        res = [set(), set()]
        res[player] = set(V)
        return tuple(res)
    B = attractor(1 - player, W[1 - player], V, owner, adj)
    W2 = list(zielonka(owner, prio, adj, V - B))
    res = [set(), set()]
    res[player] = W2[player]
    res[1 - player] = W2[1 - player] | B
    return tuple(res)


def brute_force_winners(owner, prio, adj, limit=1 << 14):
    """W_Even = {v : ∃σ ∀τ maxio(play) even} over positional strategies."""
    n = len(owner)
    ev = [v for v in range(n) if owner[v] == 0]
    od = [v for v in range(n) if owner[v] == 1]
    ne = 1
    for v in ev:
        ne *= len(adj[v])
    no = 1
    for v in od:
        no *= len(adj[v])
    assert ne * no <= limit
    win_even = [False] * n
    for sp in itertools.product(*[adj[v] for v in ev]):
        good = [True] * n
        for tp in itertools.product(*[adj[v] for v in od]):
            succ = [0] * n
            for v, u in zip(ev, sp):
                succ[v] = u
            for v, u in zip(od, tp):
                succ[v] = u
            for v in range(n):
                if not good[v]:
                    continue
                seen = {}
                path = []
                x = v
                while x not in seen:
                    seen[x] = len(path)
                    path.append(x)
                    x = succ[x]
                if max(prio[y] for y in path[seen[x]:]) % 2 == 1:
                    good[v] = False
        for v in range(n):
            win_even[v] = win_even[v] or good[v]
    return {v for v in range(n) if win_even[v]}, {v for v in range(n) if not win_even[v]}


def verify_winning_strategy(owner, prio, adj, W, player, strat):
    """Check that ``strat`` (dict v->u on W ∩ V_player) keeps plays inside W and
    every cycle reachable in the one-player game has max priority of the right
    parity (SPEC.md:420-428 idea). Brute force over opponent choices by DFS on
    the restricted graph: every cycle in the graph G' = (W, edges allowed) must
    have the right parity; we check by enumerating simple cycles' max via the
    'max priority p, remove, recurse' argument: for each priority p of the wrong
    parity, no cycle through {pri = p} within {pri <= p}."""
    Wset = set(W)
    edges = {}
    for v in Wset:
        if owner[v] == player:
            u = strat[v]
            if u not in Wset:
                return False
            edges[v] = [u]
        else:
            es = [u for u in adj[v]]
            if any(u not in Wset for u in es):
                return False
            edges[v] = es
    bad_parity = 1 - player
    for p in sorted({prio[v] for v in Wset}):
        if p % 2 != bad_parity:
            continue
        sub = {v for v in Wset if prio[v] <= p}
        # is there a cycle within `sub` through a vertex of priority p?
        for s in [v for v in sub if prio[v] == p]:
            stack = [u for u in edges[s] if u in sub]
            seen = set()
            while stack:
                x = stack.pop()
                if x == s:
                    return False
                if x in seen:
                    continue
                seen.add(x)
                stack.extend(u for u in edges[x] if u in sub)
    return True
