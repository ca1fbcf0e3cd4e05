"""Seeded game generators (inputs only; see package docstring).

Random games follow the PGSolver ``randomgame`` *shape* the configs name
(BASELINE.json ``configs``; SURVEY.md §8(d) "Synthetic inputs"): owner uniform
in {Even, Odd}, priority uniform in [0, d), out-degree uniform in [lo, hi],
successors uniform without replacement (self-loops allowed). Randomness is a
counter-based hash (splitmix64 finaliser of (seed, stream, v, j)), so a game
depends only on its parameters, never on thread count or call order.

Structured families are deterministic
constructions written out below.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_U64 = np.uint64
_GOLD = 0x9E3779B97F4A7C15


@dataclass
class Game:
    """A parity game in the ``pg_load`` layout (§2)."""

    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray  # int32[m]
    owner: np.ndarray  # uint8[n]; 0 = Even, 1 = Odd
    priority: np.ndarray  # int32[n]; >= 0
    name: str = ""

    @property
    def n(self) -> int:
        return int(self.owner.shape[0])

    @property
    def m(self) -> int:
        return int(self.col.shape[0])

    def successors(self, v: int) -> list[int]:
        return [int(x) for x in self.col[self.row_ptr[v]:self.row_ptr[v + 1]]]


def mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=_U64)
    with np.errstate(over="ignore"):
        x = (x ^ (x >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> _U64(27))) * _U64(0x94D049BB133111EB)
        x = x ^ (x >> _U64(31))
    return x


def counter_hash(seed: int, stream: int, v, j) -> np.ndarray:
    """H(seed, stream, v, j): a 64-bit hash of four counters."""
    with np.errstate(over="ignore"):
        base = mix64(np.asarray([(seed * _GOLD + stream) & 0xFFFFFFFFFFFFFFFF], dtype=_U64))[0]
        x = mix64(np.asarray(v, dtype=_U64) + base)
        return mix64(x + np.asarray(j, dtype=_U64))


def _finish(deg: np.ndarray, cand: np.ndarray, owner, priority, name) -> Game:
    n = deg.shape[0]
    hi = cand.shape[1]
    keep = np.arange(hi)[None, :] < deg[:, None]
    col = cand[keep].astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    return Game(row_ptr, col, owner.astype(np.uint8), priority.astype(np.int32), name)


def random_game(n: int, d: int, deg_lo: int, deg_hi: int, seed: int) -> Game:
    """PGSolver-``randomgame``-shaped game (BASELINE.json configs 1-3, 5)."""
    if n <= 0:
        return Game(np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.uint8),
                    np.zeros(0, np.int32), f"random-n0")
    v = np.arange(n, dtype=_U64)
    zero = np.zeros(n, dtype=_U64)
    owner = (counter_hash(seed, 0, v, zero) & _U64(1)).astype(np.uint8)
    priority = (counter_hash(seed, 1, v, zero) % _U64(d)).astype(np.int32)
    span = deg_hi - deg_lo + 1
    deg = (deg_lo + (counter_hash(seed, 2, v, zero) % _U64(span)).astype(np.int64))
    deg = np.minimum(deg, n)
    cand = np.empty((n, deg_hi), dtype=np.int64)
    for j in range(deg_hi):
        cand[:, j] = (counter_hash(seed, 3, v, np.full(n, j, _U64)) % _U64(n)).astype(np.int64)
    # without replacement: redraw slot j while it repeats an earlier slot
    for j in range(1, deg_hi):
        attempt = 0
        while True:
            active = deg > j
            dup = np.zeros(n, dtype=bool)
            for i in range(j):
                dup |= cand[:, j] == cand[:, i]
            dup &= active
            idx = np.nonzero(dup)[0]
            if idx.size == 0:
                break
            attempt += 1
            cand[idx, j] = (counter_hash(seed, 3 + 16 * attempt, idx.astype(_U64),
                                         np.full(idx.size, j, _U64)) % _U64(n)).astype(np.int64)
    return _finish(deg, cand, owner, priority, f"random-n{n}-d{d}-deg{deg_lo}-{deg_hi}-s{seed}")


def from_adjacency(owner, priority, adj, name: str = "") -> Game:
    """Build a Game from python lists (tests, fixtures)."""
    n = len(owner)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    for v in range(n):
        row_ptr[v + 1] = row_ptr[v] + len(adj[v])
    col = np.array([u for a in adj for u in a], dtype=np.int32)
    return Game(row_ptr, col, np.asarray(owner, np.uint8), np.asarray(priority, np.int32), name)


def fixture_g2() -> Game:
    """SPEC.md:94 fixture G2: v0 Even pri 2 -> {v1}; v1 Odd pri 1 -> {v0, v2};
    v2 Even pri 4 -> {v1}."""
    return from_adjacency([0, 1, 0], [2, 1, 4], [[1], [0, 2], [1]], "G2")


def f_stair(L: int) -> Game:
    """SURVEY.md App. A F_stair(L): e_0..e_{L-1} Even; pri 1 except pri(e_{L-1}) = 2;
    e_i -> e_{i+1}, e_{L-1} -> e_{L-1}."""
    owner = np.zeros(L, np.uint8)
    pri = np.ones(L, np.int32)
    pri[L - 1] = 2
    col = np.minimum(np.arange(L) + 1, L - 1).astype(np.int32)
    return Game(np.arange(L + 1, dtype=np.int64), col, owner, pri, f"stair-{L}")


def f_stairs(k: int, L: int) -> Game:
    """k disjoint copies of F_stair(L) (copy c holds ids c*L .. c*L+L-1): a long-iteration
    game of any size (n = k*L, outer passes max(L, 2); the copies advance in lockstep)."""
    one = f_stair(L)
    off = (np.arange(k, dtype=np.int64) * L)[:, None]
    col = (one.col.astype(np.int64)[None, :] + off).reshape(-1).astype(np.int32)
    return Game(np.arange(k * L + 1, dtype=np.int64), col, np.tile(one.owner, k), np.tile(one.priority, k),
                f"stairs-{k}x{L}")


def f_deep(L: int) -> Game:
    """SURVEY.md App. A F_deep(L): e_0..e_{L-1} Even pri 2, e_i -> e_{i+1},
    e_{L-1} -> o; o = L is Odd pri 3 with a self-loop."""
    owner = np.zeros(L + 1, np.uint8)
    owner[L] = 1
    pri = np.full(L + 1, 2, np.int32)
    pri[L] = 3
    col = np.minimum(np.arange(L + 1) + 1, L).astype(np.int32)
    return Game(np.arange(L + 2, dtype=np.int64), col, owner, pri, f"deep-{L}")


def f_oddchain(L: int) -> Game:
    """SURVEY.md App. A F_oddchain(L): x_i = i-1 (i=1..L) Even pri 2, x_i -> g;
    g = L Even pri 1, g -> g; o_i = L+i Odd pri 0, o_i -> {x_i, o_{i-1}}, o_0 = g."""
    n = 2 * L + 1
    g = L
    owner = np.zeros(n, np.uint8)
    owner[L + 1:] = 1
    pri = np.zeros(n, np.int32)
    pri[:L] = 2
    pri[g] = 1
    adj = [[g] for _ in range(L)] + [[g]]
    for i in range(1, L + 1):
        prev = g if i == 1 else L + i - 1
        adj.append(sorted({i - 1, prev}))
    return from_adjacency(owner, pri, adj, f"oddchain-{L}")


def ladder(N: int, seed: int) -> Game:
    """SURVEY.md §8(d) config 4 family Lad(N): vertices (r, i), r in {0,1},
    i in [0, N/2); id = r*(N/2) + i. Row 0 Even pri 2; row 1 Odd pri 1 (pri 3 on
    every 64th). Edges (r,i)->(r,i+1), (r,i)->(1-r,i+1) and, when
    H(seed,r,i) mod 4 == 0, (r,i)->(r,i-7) (indices mod N/2)."""
    h = N // 2
    i = np.arange(h, dtype=np.int64)
    owner = np.concatenate([np.zeros(h, np.uint8), np.ones(h, np.uint8)])
    pri = np.concatenate([np.full(h, 2, np.int32),
                          np.where(i % 64 == 63, 3, 1).astype(np.int32)])
    n = 2 * h
    cand = np.full((n, 3), -1, dtype=np.int64)
    deg = np.full(n, 2, dtype=np.int64)
    for r in range(2):
        base = r * h
        vv = base + i
        cand[vv, 0] = base + (i + 1) % h
        cand[vv, 1] = (1 - r) * h + (i + 1) % h
        back = (counter_hash(seed, 7 + r, i.astype(_U64), np.zeros(h, _U64)) % _U64(4)) == 0
        tgt = base + (i - 7) % h
        ok = back & (tgt != cand[vv, 0]) & (tgt != cand[vv, 1])
        cand[vv[ok], 2] = tgt[ok]
        deg[vv[ok]] = 3
    return _finish(deg, cand, owner, pri, f"ladder-{N}-s{seed}")


def hanoi(k: int) -> Game:
    """SURVEY.md §8(d) config 4 family Hanoi-k: 2*3^k vertices (configuration,
    turn). Configuration c has base-3 digits c_0..c_{k-1}: peg of disk i (disk 0
    smallest). Turn 0 = Even, 1 = Odd; edges are the legal moves and flip the turn.
    Priority 2 on the goal (all disks on peg 2), 1 when the largest disk is on
    peg 0, 0 otherwise. id = turn * 3^k + c."""
    S = 3 ** k
    c = np.arange(S, dtype=np.int64)
    digits = np.empty((k, S), dtype=np.int64)
    x = c.copy()
    for i in range(k):
        digits[i] = x % 3
        x //= 3
    # top disk of each peg (k = empty)
    top = np.full((3, S), k, dtype=np.int64)
    for i in range(k - 1, -1, -1):
        for p in range(3):
            top[p] = np.where(digits[i] == p, i, top[p])
    pow3 = 3 ** np.arange(k, dtype=np.int64)
    moves = []  # list of (valid mask, target config)
    for a in range(3):
        for b in range(3):
            if a == b:
                continue
            ta, tb = top[a], top[b]
            valid = (ta < k) & (ta < tb)
            disk = np.minimum(ta, k - 1)
            tgt = c + (b - a) * pow3[disk]
            moves.append((valid, tgt))
    deg_c = np.sum([m[0] for m in moves], axis=0)
    cand_c = np.full((S, 6), -1, dtype=np.int64)
    slot = np.zeros(S, dtype=np.int64)
    for valid, tgt in moves:
        idx = np.nonzero(valid)[0]
        cand_c[idx, slot[idx]] = tgt[idx]
        slot[idx] += 1
    n = 2 * S
    cand = np.full((n, 3), -1, dtype=np.int64)
    cand[:S, :3] = cand_c[:, :3] + S  # Even turn -> Odd turn
    cand[S:, :3] = cand_c[:, :3]
    cand[:S][cand_c[:, :3] < 0] = -1
    cand[S:][cand_c[:, :3] < 0] = -1
    deg = np.concatenate([deg_c, deg_c]).astype(np.int64)
    owner = np.concatenate([np.zeros(S, np.uint8), np.ones(S, np.uint8)])
    goal = np.all(digits == 2, axis=0) if k > 0 else np.ones(S, bool)
    p1 = digits[k - 1] == 0 if k > 0 else np.zeros(S, bool)
    pri_c = np.where(goal, 2, np.where(p1, 1, 0)).astype(np.int32)
    pri = np.concatenate([pri_c, pri_c])
    return _finish(deg, cand, owner, pri, f"hanoi-{k}")


def elevator(f: int, r: int, seed: int) -> Game:
    """SURVEY.md §8(d) config 4 family Elevator-(f, r), an elevator-like scheduler
    product with d = 3 (Table 1's Elevator). The car is on floor
    c in [0, f); floors 0..r-1 (r <= f) carry a pending-request bit in mask.

    - Even (controller) vertex (c, mask), id = c*2^r + mask: moves the car up
      or down, or serves the pending request on its floor. Priority 1 while the
      request at the car's floor is pending, else 0.
    - Odd (environment) vertex (s, c, mask), id = f*2^r + (s*f + c)*2^r + mask,
      s = 1 right after a serve: passes, or adds the request j = H(seed, 11, id)
      mod r when it is not already pending. Priority 2 on serve (s = 1), else 0.

    3·f·2^r vertices (f = 20, r = 15 -> 1.97M), out-degree 1-3."""
    assert f >= 2 and 1 <= r <= f
    R = 1 << r
    E = f * R
    n = 3 * E
    c = np.repeat(np.arange(f, dtype=np.int64), R)
    mask = np.tile(np.arange(R, dtype=np.int64), f)
    bit = np.where(c < r, np.left_shift(1, np.minimum(c, r - 1)), 0)
    pending = (mask & bit) != 0
    cand = np.full((n, 3), -1, dtype=np.int64)
    deg = np.zeros(n, dtype=np.int64)
    ev = np.arange(E, dtype=np.int64)

    def push(rows, tgt, ok):
        idx = rows[ok]
        cand[idx, deg[idx]] = tgt[ok]
        deg[idx] += 1

    push(ev, E + (c + 1) * R + mask, c + 1 < f)                   # up
    push(ev, E + (c - 1) * R + mask, c > 0)                       # down
    push(ev, E + (f + c) * R + (mask & ~bit), pending)            # serve -> s = 1
    for s_ in range(2):
        ov = E + s_ * E + ev
        push(ov, ev, np.ones(E, bool))                            # pass
        j = (counter_hash(seed, 11, ov.astype(_U64), np.zeros(E, _U64)) % _U64(r)).astype(np.int64)
        req = np.left_shift(1, j)
        push(ov, c * R + (mask | req), (mask & req) == 0)         # new request
    owner = np.concatenate([np.zeros(E, np.uint8), np.ones(2 * E, np.uint8)])
    pri = np.concatenate([np.where(pending, 1, 0), np.zeros(E), np.full(E, 2)]).astype(np.int32)
    return _finish(deg, cand, owner, pri, f"elevator-{f}-{r}-s{seed}")


def pgsolver_text(g: Game) -> str:
    """Serialise in the PGSolver format (SPEC.md game_core interface idea)."""
    lines = [f"parity {g.n - 1};"]
    for v in range(g.n):
        succ = ",".join(str(u) for u in g.successors(v))
        lines.append(f"{v} {int(g.priority[v])} {int(g.owner[v])} {succ};")
    return "\n".join(lines) + "\n"


def parse_pgsolver(text: str) -> Game:
    """Parse the PGSolver format: optional ``parity <maxid>;`` header, then
    ``<id> <priority> <owner> <succ>,<succ>,... ["name"];`` per vertex."""
    recs = {}
    maxid = None
    for raw in text.replace("\n", " ").split(";"):
        tok = raw.strip()
        if not tok:
            continue
        if tok.startswith("parity"):
            maxid = int(tok.split()[1])
            continue
        if '"' in tok:
            tok = tok[:tok.index('"')].strip()
        parts = tok.split(None, 3)
        if len(parts) < 4:
            raise ValueError(f"bad record: {raw!r}")
        vid, p, o = int(parts[0]), int(parts[1]), int(parts[2])
        succ = [int(s) for s in parts[3].replace(" ", "").split(",") if s != ""]
        if not succ:
            raise ValueError(f"vertex {vid} has no successors")
        if vid in recs:
            raise ValueError(f"duplicate vertex {vid}")
        recs[vid] = (p, o, succ)
    n = (maxid + 1) if maxid is not None else (max(recs) + 1 if recs else 0)
    if set(recs) != set(range(n)):
        raise ValueError("vertex ids must be exactly 0..maxid")
    return from_adjacency([recs[v][1] for v in range(n)], [recs[v][0] for v in range(n)],
                          [recs[v][2] for v in range(n)], "pgsolver")
