"""Independent fp64 checkers that pin the oracle (never used by the product path).

* `trellis_kbest` — textbook shortest path over the graph unrolled across
  frames (SURVEY §8.4 "Plain definition"): nodes (t, q); epsilon edges inside a
  layer, emitting edges t -> t+1 costing w - L[t][pdf]; source (0, start);
  result min over (T, q) of dist + F(q) (or min dist when no final state is
  reachable, reading R10).  Keeps the 2 best distinct paths per node so tests
  can demand a gap between best and second best ("tie-free", north_star).
  Epsilon relaxation is done in increasing source-state order, which is a
  topological order for the graphs used here (epsilon arcs go low -> high id;
  asserted).
* `enumerate_paths` — depth-first enumeration of every complete path on
  tiny graphs (SPEC S:497-505 exhaustive_paths), fp64.
Arc ids returned are INPUT arc indices.
"""
from __future__ import annotations

import math

import numpy as np


def _check_eps_topo(g):
    e = g.ilabel == 0
    assert np.all(g.src[e] < g.dst[e]), "bruteforce needs epsilon arcs going low -> high id"


def trellis_kbest(g, ll: np.ndarray, k: int = 2):
    """Returns list of up to k (cost, arcs, reached_final) best complete paths (fp64)."""
    _check_eps_topo(g)
    ll = np.asarray(ll, dtype=np.float64)
    T = ll.shape[0]
    Q = g.n_states
    w = g.weight.astype(np.float64)
    emit = [i for i in range(g.n_arcs) if g.ilabel[i] != 0]
    eps_by_src = {}
    for i in range(g.n_arcs):
        if g.ilabel[i] == 0:
            eps_by_src.setdefault(int(g.src[i]), []).append(i)
    # entry = (cost, backref) ; backref = None | (layer, state, rank, arc)
    def insert(lst, cand):
        lst.append(cand)
        lst.sort(key=lambda x: x[0])
        del lst[k:]

    def closure(layer_entries):
        for s in range(Q):                      # topological (eps arcs low -> high)
            for a in eps_by_src.get(s, []):
                d = int(g.dst[a])
                for r, (c, _) in enumerate(list(layer_entries[s])):
                    insert(layer_entries[d], (c + w[a], ("same", s, r, a)))

    layers = []
    L0 = [[] for _ in range(Q)]
    L0[g.start].append((0.0, None))
    closure(L0)
    layers.append(L0)
    for t in range(T):
        prev = layers[-1]
        cur = [[] for _ in range(Q)]
        for a in emit:
            s, d = int(g.src[a]), int(g.dst[a])
            for r, (c, _) in enumerate(prev[s]):
                insert(cur[d], (c + w[a] - ll[t, g.ilabel[a] - 1], ("prev", s, r, a)))
        closure(cur)
        layers.append(cur)
    last = layers[-1]
    finals = []
    for q in range(Q):
        F = float(g.final[q])
        if math.isfinite(F):
            for r, (c, _) in enumerate(last[q]):
                finals.append((c + F, q, r))
    reached = bool(finals)
    if not reached:
        finals = [(c, q, r) for q in range(Q) for r, (c, _) in enumerate(last[q])]
    finals.sort(key=lambda x: x[0])
    out = []
    for (c, q, r) in finals[:k]:
        arcs = []
        li, s, rr = T, q, r
        while True:
            _, br = layers[li][s][rr]
            if br is None:
                break
            kind, ps, pr, a = br
            arcs.append(a)
            if kind == "prev":
                li -= 1
            s, rr = ps, pr
        out.append((c, arcs[::-1], reached))
    return out


def enumerate_paths(g, ll: np.ndarray, max_states: int = 8, max_frames: int = 8, simple_eps: bool = False):
    """All complete paths as (cost_fp64, arcs, ends_final) with cost including F
    for final end states.  Epsilon steps bounded by |Q| per frame.  simple_eps: only paths
    whose epsilon runs inside a frame visit no state twice -- every path when epsilon cycles
    are absent, and it still contains every optimal path when all epsilon cycles have positive
    weight (dropping a cycle makes a path strictly cheaper)."""
    assert g.n_states <= max_states and ll.shape[0] <= max_frames, "instance-size guard"
    ll = np.asarray(ll, dtype=np.float64)
    T = ll.shape[0]
    out_arcs = {}
    for i in range(g.n_arcs):
        out_arcs.setdefault(int(g.src[i]), []).append(i)
    res = []

    def dfs(t, q, c, path, eps_steps, run):
        if t == T:
            F = float(g.final[q])
            res.append((c + F if math.isfinite(F) else c, list(path), math.isfinite(F)))
        for a in out_arcs.get(q, []):
            d = int(g.dst[a])
            if g.ilabel[a] == 0:
                if eps_steps < g.n_states and not (simple_eps and d in run):
                    path.append(a)
                    dfs(t, d, c + float(g.weight[a]), path, eps_steps + 1, run | {d})
                    path.pop()
            elif t < T:
                path.append(a)
                dfs(t + 1, d, c + float(g.weight[a]) - ll[t, g.ilabel[a] - 1], path, 0, frozenset([d]))
                path.pop()

    dfs(0, g.start, 0.0, [], 0, frozenset([g.start]))
    return res


def best_of_enumeration(paths):
    fin = [p for p in paths if p[2]]
    pool = fin if fin else paths
    pool = sorted(pool, key=lambda p: p[0])
    return pool, bool(fin)


def path_cost_fp64(g, ll, arcs) -> tuple[float, int, int]:
    """Re-walk a path: returns (cost incl. final, end state, frames consumed);
    raises if arcs are not a connected path from the start state."""
    ll = np.asarray(ll, dtype=np.float64)
    q, t, c = g.start, 0, 0.0
    for a in arcs:
        assert int(g.src[a]) == q, "path not connected"
        c += float(g.weight[a])
        if g.ilabel[a] != 0:
            c -= ll[t, g.ilabel[a] - 1]
            t += 1
        q = int(g.dst[a])
    F = float(g.final[q])
    return (c + F if math.isfinite(F) else c), q, t


def canonical_order(g) -> np.ndarray:
    """canonical arc id -> input arc index: stable by (src, emitting first)
    (SPEC S:32).  Written independently of the oracle."""
    return np.lexsort((np.arange(g.n_arcs), (g.ilabel == 0).astype(np.int64), g.src.astype(np.int64)))
