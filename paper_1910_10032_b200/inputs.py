"""Seeded synthetic inputs shared by the CPU oracle tests and the CUDA path.

This module holds NO decoding arithmetic: no token passing, no beam, no
closure, no traceback.  It only produces *inputs* — decode graphs shaped like
a Kaldi HCLG (§3.2.1: "a set of compressed sparse rows";
SURVEY §8.5 "Synthetic inputs"), planted pdf walks, and frame log-likelihoods
from a counter-based hash (SURVEY §8.5 "Log-likelihoods ... bit-identical on
host and device").  The device twin of `loglikes()` is `wfst_synth_loglikes`
in csrc/synth.cu; tests assert the two are bit-identical.

Graph convention (adopted in DESIGN.md): arcs are
(src, dst, ilabel, olabel, weight); ilabel 0 = epsilon (non-emitting), an
emitting arc's pdf id is ilabel-1; state `start` is the start state;
final[q] = +inf for non-final states.  Arc order here is the *input order*;
each consumer (oracle, C-ABI loader) canonicalises it itself.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Wfst", "hclg_graph", "hclg_graph_eps", "c1_graph", "random_tiny_graph", "planted_walks",
    "loglikes", "loglikes_stream", "write_text", "read_text", "PRESETS", "CONFIGS",
]


@dataclasses.dataclass
class Wfst:
    n_states: int
    start: int
    src: np.ndarray      # int32 [E]
    dst: np.ndarray      # int32 [E]
    ilabel: np.ndarray   # int32 [E]  (0 = epsilon, pdf = ilabel-1)
    olabel: np.ndarray   # int32 [E]  (0 = no output)
    weight: np.ndarray   # float32 [E]
    final: np.ndarray    # float32 [Q] (+inf = non-final)

    @property
    def n_arcs(self) -> int:
        return int(self.src.shape[0])

    @property
    def n_emitting(self) -> int:
        return int(np.count_nonzero(self.ilabel))

    @property
    def max_pdf(self) -> int:
        e = self.ilabel[self.ilabel != 0]
        return int(e.max()) - 1 if e.size else -1


def _f32(x) -> np.ndarray:
    a = np.asarray(x, dtype=np.float32)
    return a + np.float32(0.0)          # canonicalise -0.0 -> +0.0


def _mk(n_states, start, src, dst, ilabel, olabel, weight, final) -> Wfst:
    return Wfst(int(n_states), int(start),
                np.ascontiguousarray(src, dtype=np.int32),
                np.ascontiguousarray(dst, dtype=np.int32),
                np.ascontiguousarray(ilabel, dtype=np.int32),
                np.ascontiguousarray(olabel, dtype=np.int32),
                np.ascontiguousarray(_f32(weight)),
                np.ascontiguousarray(_f32(final)))


# --------------------------------------------------------------------------
# HCLG-shaped generator (SURVEY §8.5 "Graph generator")
# --------------------------------------------------------------------------
def hclg_graph(n_states: int, degree: float, n_pdfs: int, seed: int,
               hub_fanout: int = 20000) -> Wfst:
    """Random graph with the structure of a decode graph.

    * word chains of 2-8 states (HMM-like): emitting self-loop + emitting
      forward arc, the last state exits (emitting) into the LM-history state
      of its word;
    * LM-history states (~8% of |Q|): emitting word-entry arcs carrying the
      word id as olabel (words drawn Zipf-like, LM cost ~ Gamma(2, 1.5)) and
      one epsilon back-off arc to a bigram hub;
    * bigram hubs: 4x the word arcs, epsilon back-off to the unigram hub;
    * unigram hub: emitting fan-out to min(#words, hub_fanout) word starts
      (the heavy-tailed out-degree that stresses load balancing);
    * epsilon arcs only go from lower to higher ids (no epsilon cycles);
    * history states are final with F ~ U(0.5, 3); start state = 0.
    `degree` = target |E|/|Q|.
    """
    rng = np.random.default_rng(seed)
    n_lm = max(6, int(round(0.08 * n_states)))
    n_bi = max(1, n_lm // 500)
    n_hist = n_lm - n_bi - 1
    hub = n_lm - 1
    n_chain = n_states - n_lm
    assert n_chain >= 2 and n_hist >= 1

    lens = rng.integers(2, 9, size=n_chain // 2 + 2)
    cs = np.cumsum(lens)
    k = int(np.searchsorted(cs, n_chain))
    lens = lens[: k + 1].copy()
    lens[-1] -= cs[k] - n_chain
    W = lens.size
    wstart = n_lm + np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    wend = wstart + lens - 1
    chain = np.arange(n_lm, n_states, dtype=np.int64)
    pdf = np.zeros(n_states, dtype=np.int64)
    pdf[n_lm:] = rng.integers(0, n_pdfs, size=n_chain)
    word_of = np.repeat(np.arange(W), lens)
    is_last = chain == wend[word_of]
    lm_of_word = rng.integers(0, n_hist, size=W)

    u = lambda n: rng.uniform(0.05, 0.7, size=n)
    # chain self-loops
    s1, d1, i1, o1, w1 = chain, chain, pdf[chain] + 1, np.zeros(n_chain, np.int64), u(n_chain)
    # chain forward / exit
    nxt = np.where(is_last, lm_of_word[word_of], chain + 1)
    ilf = np.where(is_last, pdf[chain], pdf[np.minimum(chain + 1, n_states - 1)]) + 1
    s2, d2, i2, o2, w2 = chain, nxt, ilf, np.zeros(n_chain, np.int64), u(n_chain)

    hubF = min(W, hub_fanout)
    target = int(round(degree * n_states))
    lm_deg = (target - 2 * n_chain - hubF - n_bi - n_hist) / float(n_hist + 4 * n_bi)
    lm_deg = max(lm_deg, 1.0)
    base = int(math.floor(lm_deg))
    frac = lm_deg - base
    deg_h = base + (rng.random(n_hist) < frac).astype(np.int64)
    deg_b = np.full(n_bi, 4 * base, dtype=np.int64)
    lm_src = np.concatenate([np.repeat(np.arange(n_hist), deg_h),
                             np.repeat(np.arange(n_hist, n_hist + n_bi), deg_b)])
    nw = lm_src.size
    # Zipf-like word choice: P(w) ~ 1/(w+1)
    wsel = np.minimum(np.floor(np.exp(rng.random(nw) * math.log(W + 1.0))).astype(np.int64) - 1, W - 1)
    wsel = np.maximum(wsel, 0)
    s3 = lm_src
    d3 = wstart[wsel]
    i3 = pdf[d3] + 1
    o3 = wsel + 1
    w3 = rng.gamma(2.0, 1.5, size=nw)
    # back-off epsilon arcs
    s4 = np.arange(n_hist + n_bi)
    d4 = np.concatenate([n_hist + (np.arange(n_hist) % n_bi), np.full(n_bi, hub)])
    i4 = np.zeros(s4.size, np.int64)
    o4 = np.zeros(s4.size, np.int64)
    w4 = rng.uniform(0.5, 3.0, size=s4.size)
    # unigram hub fan-out
    hw = np.arange(hubF)
    s5 = np.full(hubF, hub)
    d5 = wstart[hw]
    i5 = pdf[d5] + 1
    o5 = hw + 1
    w5 = 0.7 * np.log(hw + 2.0)

    final = np.full(n_states, np.inf, dtype=np.float64)
    final[:n_hist] = rng.uniform(0.5, 3.0, size=n_hist)
    cat = lambda *xs: np.concatenate(xs)
    return _mk(n_states, 0, cat(s1, s2, s3, s4, s5), cat(d1, d2, d3, d4, d5),
               cat(i1, i2, i3, i4, i5), cat(o1, o2, o3, o4, o5),
               cat(w1, w2, w3, w4, w5), final)


def hclg_graph_eps(n_states: int, degree: float, n_pdfs: int, seed: int, hub_fanout: int = 20000,
                   levels: int = 5, permute_states: bool = True) -> Wfst:
    """Epsilon-general, id-scattered variant of hclg_graph (the paper's hard case: "chains of
    non-emitting arcs", and their long tail).  Starting from hclg_graph:

    * back-off chains of `levels` epsilon arcs: LM-history states are split into levels
      0..levels-1 (most at the top); a state of level l > 0 backs off to a random state of level
      l-1 (U(0.2, 0.8)), level 0 backs off to the unigram hub -- chains of length `levels`;
    * skip arcs: every 4th history state also has a direct epsilon arc to the hub, heavier than
      its chain (sum of U(0.2, 0.8) per level + U(1, 3)), so the closure first reaches the hub
      expensively and later improves it through the chain (re-relaxation);
    * backward arcs and cycles: every 8th history state h gets an epsilon arc back from its
      back-off target b (b -> h, U(0.5, 2)): positive-weight 2-cycles h -> b -> h;
    * with permute_states, state ids are a random permutation (start included), so epsilon arcs
      go to lower and higher ids alike and graph reads have no id locality.
    All epsilon weights are > 0, so every epsilon cycle has positive weight (accepted at load)."""
    g = hclg_graph(n_states, degree, n_pdfs, seed, hub_fanout)
    rng = np.random.default_rng([seed, 7331])
    n_lm = max(6, int(round(0.08 * n_states)))
    n_bi = max(1, n_lm // 500)
    n_hist = n_lm - n_bi - 1
    hub = n_lm - 1
    keep = ~((g.ilabel == 0) & (g.src < n_hist))          # drop the history states' back-off arcs
    src, dst, il, ol, w = (g.src[keep].astype(np.int64), g.dst[keep].astype(np.int64),
                           g.ilabel[keep].astype(np.int64), g.olabel[keep].astype(np.int64),
                           g.weight[keep].astype(np.float64))
    # levels: level l holds a share proportional to 2^l of the history states (top level largest)
    share = 2.0 ** np.arange(levels)
    bounds = np.concatenate([[0], np.round(np.cumsum(share) / share.sum() * n_hist).astype(np.int64)])
    lvl = np.zeros(n_hist, np.int64)
    for l in range(levels):
        lvl[bounds[l]:bounds[l + 1]] = l
    h = np.arange(n_hist)
    tgt = np.full(n_hist, hub, np.int64)
    for l in range(1, levels):
        m = lvl == l
        lo, hi = bounds[l - 1], bounds[l]
        if hi > lo:
            tgt[m] = rng.integers(lo, hi, size=int(m.sum()))
    wb = rng.uniform(0.2, 0.8, size=n_hist)
    add_s, add_d, add_w = [h], [tgt], [wb]
    # skip arcs: heavier than the chain below them
    chain_cost = np.zeros(n_hist)
    for l in range(levels):              # chain cost to the hub, level by level
        m = lvl == l
        chain_cost[m] = wb[m] + (0.0 if l == 0 else chain_cost[tgt[m]])
    sk = h[(h % 4 == 3) & (lvl > 0)]
    add_s.append(sk); add_d.append(np.full(sk.size, hub)); add_w.append(chain_cost[sk] + rng.uniform(1.0, 3.0, sk.size))
    # backward arcs: positive 2-cycles h -> tgt(h) -> h
    bk = h[(h % 8 == 5) & (tgt != hub)]
    add_s.append(tgt[bk]); add_d.append(bk); add_w.append(rng.uniform(0.5, 2.0, bk.size))
    es, ed, ew = np.concatenate(add_s), np.concatenate(add_d), np.concatenate(add_w)
    src = np.concatenate([src, es]); dst = np.concatenate([dst, ed]); w = np.concatenate([w, ew])
    il = np.concatenate([il, np.zeros(es.size, np.int64)]); ol = np.concatenate([ol, np.zeros(es.size, np.int64)])
    final = g.final.astype(np.float64)
    start = g.start
    if permute_states:
        perm = rng.permutation(n_states)          # old id -> new id
        src, dst = perm[src], perm[dst]
        nf = np.empty_like(final)
        nf[perm] = final
        final, start = nf, int(perm[start])
        order = rng.permutation(src.size)         # and a scrambled input arc order
        src, dst, il, ol, w = src[order], dst[order], il[order], ol[order], w[order]
    return _mk(n_states, start, src, dst, il, ol, w, final)


# --------------------------------------------------------------------------
# C1: tiny hand-built graph (BASELINE.json configs[0])
# --------------------------------------------------------------------------
_C1_EPS = [  # (src, dst, weight): a 3-long epsilon chain 0->3->7->12 and more
    (0, 3, 0.5), (3, 7, 0.25), (7, 12, 0.75), (2, 4, 0.2), (5, 9, 1.0),
    (10, 15, 0.3), (14, 18, 0.6)]


def c1_graph() -> Wfst:
    """20 states, 60 arcs (7 epsilon, incl. a chain of length 3), 10 pdfs,
    state 1 has out-degree 9, 4 final states, olabels on >= 5 arcs, no
    parallel arcs.  Deterministic (fixed seed)."""
    rng = np.random.default_rng(1910)
    Q, P = 20, 10
    arcs = {}
    for (s, d, w) in _C1_EPS:
        arcs[(s, d)] = (0, 0, w)
    # state 1: out-degree 9, all emitting
    for d in rng.choice(np.arange(2, 20), size=9, replace=False):
        arcs[(1, int(d))] = (int(rng.integers(1, P + 1)), 0, float(rng.uniform(0.1, 2.0)))
    # every state gets >= 1 emitting arc
    for s in range(Q):
        if not any(k[0] == s and v[0] != 0 for k, v in arcs.items()):
            d = int(rng.integers(0, Q))
            while (s, d) in arcs:
                d = int(rng.integers(0, Q))
            arcs[(s, d)] = (int(rng.integers(1, P + 1)), 0, float(rng.uniform(0.1, 2.0)))
    while len(arcs) < 60:
        s, d = int(rng.integers(0, Q)), int(rng.integers(0, Q))
        if (s, d) in arcs:
            continue
        arcs[(s, d)] = (int(rng.integers(1, P + 1)), 0, float(rng.uniform(0.1, 2.0)))
    keys = sorted(arcs.keys(), key=lambda k: (k[0], k[1]))
    perm = rng.permutation(len(keys))       # non-canonical input order
    keys = [keys[i] for i in perm]
    src = [k[0] for k in keys]
    dst = [k[1] for k in keys]
    il = [arcs[k][0] for k in keys]
    w = [round(arcs[k][2], 3) for k in keys]
    ol = [0] * len(keys)
    n_out = 0
    for i in range(len(keys)):
        if il[i] != 0 and n_out < 8 and dst[i] % 3 == 0:
            ol[i] = 100 + dst[i]
            n_out += 1
    final = np.full(Q, np.inf)
    for q, f in ((12, 0.5), (15, 1.0), (18, 0.25), (19, 2.0)):
        final[q] = f
    return _mk(Q, 0, src, dst, il, ol, w, final)


def random_tiny_graph(seed: int, n_states: int = 6, n_arcs: int = 14, n_pdfs: int = 4,
                      eps_frac: float = 0.25, n_final: int = 2, eps_back: bool = False) -> Wfst:
    """Random small graph for brute-force checking (C1' in SURVEY §8.5).
    Epsilon arcs go from lower to higher ids (acyclic), or with eps_back to any other state
    (cycles possible; every epsilon weight is >= 0.25, so every epsilon cycle is positive)."""
    rng = np.random.default_rng(seed)
    src, dst, il, ol, w = [], [], [], [], []
    for _ in range(n_arcs):
        s = int(rng.integers(0, n_states))
        if eps_back and rng.random() < eps_frac:
            d = int((s + rng.integers(1, n_states)) % n_states)
            lab = 0
        elif not eps_back and rng.random() < eps_frac and s < n_states - 1:
            d = int(rng.integers(s + 1, n_states))
            lab = 0
        else:
            d = int(rng.integers(0, n_states))
            lab = int(rng.integers(1, n_pdfs + 1))
        src.append(s); dst.append(d); il.append(lab)
        ol.append(int(rng.integers(1, 9)) if rng.random() < 0.5 else 0)
        w.append(float(rng.uniform(0.25 if (eps_back and lab == 0) else 0.0, 2.0)))
    final = np.full(n_states, np.inf)
    for q in rng.choice(n_states, size=n_final, replace=False):
        final[q] = float(rng.uniform(0.0, 1.5))
    return _mk(n_states, 0, src, dst, il, ol, w, final)


# --------------------------------------------------------------------------
# planted walks: the "true" pdf sequence each stream is boosted towards
# --------------------------------------------------------------------------
def _csr(g: Wfst):
    order = np.lexsort((g.ilabel == 0, g.src))
    counts = np.bincount(g.src, minlength=g.n_states)
    indptr = np.concatenate([[0], np.cumsum(counts)])
    n_em = np.bincount(g.src[g.ilabel != 0], minlength=g.n_states)
    return order, indptr, n_em


def planted_walks(g: Wfst, n_streams: int, T: int, seed: int, stream0: int = 0,
                  p_eps: float = 0.3) -> np.ndarray:
    """int32 [T][B] pdf ids of a random walk per stream over the graph
    (emitting step per frame; an epsilon arc is taken first with prob p_eps
    when the state has one).  Stream b is seeded by (seed, stream0+b) so the
    walk of a global stream id does not depend on how streams are split."""
    order, indptr, n_em = _csr(g)
    a_dst = g.dst[order]
    a_il = g.ilabel[order]
    out = np.zeros((T, n_streams), dtype=np.int32)
    rngs = [np.random.default_rng([seed, stream0 + b]) for b in range(n_streams)]
    U = np.stack([r.random((T, 3)) for r in rngs], axis=1) if n_streams else np.zeros((T, 0, 3))
    cur = np.full(n_streams, g.start, dtype=np.int64)
    n_all = np.diff(indptr)
    n_pdf = max(g.max_pdf + 1, 1)
    for t in range(T):
        u = U[t]
        has_eps = n_all[cur] > n_em[cur]
        take = has_eps & (u[:, 0] < p_eps)
        e_idx = indptr[cur] + n_em[cur]          # first epsilon arc of the state
        cur = np.where(take, a_dst[np.minimum(e_idx, a_dst.size - 1)], cur)
        deg = n_em[cur]
        ok = deg > 0
        j = indptr[cur] + np.minimum((u[:, 1] * np.maximum(deg, 1)).astype(np.int64),
                                     np.maximum(deg - 1, 0))
        j = np.minimum(j, a_dst.size - 1)
        out[t] = np.where(ok, a_il[j] - 1, (u[:, 2] * n_pdf).astype(np.int64))
        cur = np.where(ok, a_dst[j], cur)
    return out


# --------------------------------------------------------------------------
# counter-hash log-likelihoods (bit-identical to csrc/synth.cu)
# --------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def _seed_word(seed: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return _mix(np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + _GOLD], dtype=np.uint64))[0]


def _scale(sigma: float) -> np.float32:
    return np.float32(sigma * math.sqrt(6.0))


def loglikes_stream(seed: int, stream: int, T: int, P: int, planted_col: np.ndarray | None,
                    sigma: float, boost: float) -> np.ndarray:
    """float32 [T][P] log-likelihoods of one (global) stream.

    key = (stream<<40) | (t<<20) | p ; h = mix((key ^ mix(seed+G)) + G)
    u0 = (h>>41)*2^-23, u1 = ((h>>18)&(2^23-1))*2^-23   (23-bit uniforms)
    L = fl(fl(fl(u0+u1) - 1) * s) + (p == planted[t] ? boost : 0),  s = fl32(sigma*sqrt 6)
    (every op a single fp32 rounding; Irwin-Hall-2 noise of std sigma)."""
    assert P < (1 << 20) and T < (1 << 20) and stream < (1 << 24)
    sw = _seed_word(seed)
    t = np.arange(T, dtype=np.uint64)[:, None]
    p = np.arange(P, dtype=np.uint64)[None, :]
    key = (np.uint64(stream) << np.uint64(40)) | (t << np.uint64(20)) | p
    with np.errstate(over="ignore"):
        h = _mix((key ^ sw) + _GOLD)
    u0 = (h >> np.uint64(41)).astype(np.float32) * np.float32(2.0 ** -23)
    u1 = ((h >> np.uint64(18)) & np.uint64(0x7FFFFF)).astype(np.float32) * np.float32(2.0 ** -23)
    n = (u0 + u1) - np.float32(1.0)
    x = n * _scale(sigma)
    b = np.zeros((T, P), dtype=np.float32)
    if planted_col is not None and boost != 0.0:
        b[np.arange(T), np.asarray(planted_col, dtype=np.int64)] = np.float32(boost)
    return (x + b).astype(np.float32)


def loglikes(seed: int, streams, T: int, P: int, planted: np.ndarray | None,
             sigma: float, boost: float) -> np.ndarray:
    """float32 [T][B][P] for the given global stream ids (planted: [T][B])."""
    streams = list(streams)
    out = np.empty((T, len(streams), P), dtype=np.float32)
    for j, s in enumerate(streams):
        col = None if planted is None else planted[:, j]
        out[:, j, :] = loglikes_stream(seed, s, T, P, col, sigma, boost)
    return out


# --------------------------------------------------------------------------
# text format: "src dst ilabel olabel weight" / "state weight"
# --------------------------------------------------------------------------
def write_text(g: Wfst, path: str) -> None:
    with open(path, "w") as f:
        for i in range(g.n_arcs):
            f.write(f"{g.src[i]} {g.dst[i]} {g.ilabel[i]} {g.olabel[i]} {float(g.weight[i])!r}\n")
        for q in range(g.n_states):
            if np.isfinite(g.final[q]):
                f.write(f"{q} {float(g.final[q])!r}\n")


def read_text(path: str) -> Wfst:
    src, dst, il, ol, w, fin = [], [], [], [], [], {}
    n = 0
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            tok = line.split()
            if not tok:
                continue
            if len(tok) == 5:
                s, d = int(tok[0]), int(tok[1])
                src.append(s); dst.append(d); il.append(int(tok[2])); ol.append(int(tok[3]))
                w.append(float(tok[4])); n = max(n, s + 1, d + 1)
            elif len(tok) == 2:
                q = int(tok[0]); fin[q] = float(tok[1]); n = max(n, q + 1)
            else:
                raise ValueError(f"line {ln}: expected 2 or 5 fields")
    final = np.full(n, np.inf)
    for q, f_ in fin.items():
        final[q] = f_
    return _mk(n, 0, src, dst, il, ol, w, final)


# --------------------------------------------------------------------------
# presets and configs (BASELINE.json configs)
# --------------------------------------------------------------------------
PRESETS = {"clean": dict(sigma=1.0, boost=4.0), "other": dict(sigma=1.0, boost=0.0)}

CONFIGS = {
    "c1": dict(graph="c1", n_pdfs=10, streams=1, frames=30, beam=math.inf, max_active=0,
               preset=dict(sigma=1.5, boost=2.0), graph_seed=0, ll_seed=1),
    "c2": dict(graph=dict(n_states=50_000, degree=6.0, n_pdfs=2000), n_pdfs=2000, streams=100,
               frames=500, beam=10.0, max_active=10_000, preset="clean", graph_seed=2, ll_seed=20002),
    "c3": dict(graph=dict(n_states=5_000_000, degree=3.0, n_pdfs=5700), n_pdfs=5700, streams=512,
               frames=500, beam=15.0, max_active=10_000, preset="clean", graph_seed=3, ll_seed=30003),
    "c4": dict(graph=dict(n_states=50_000_000, degree=3.0, n_pdfs=5700), n_pdfs=5700, streams=1024,
               frames=500, beam=15.0, max_active=10_000, preset="clean", graph_seed=4, ll_seed=40004,
               chunk=50),
    # C5: 4096 streams in total, split 4096/N over N GPUs (strong scaling, BASELINE configs[4])
    "c5": dict(graph=dict(n_states=5_000_000, degree=3.0, n_pdfs=5700), n_pdfs=5700, streams=4096,
               frames=500, beam=15.0, max_active=10_000, preset="clean", graph_seed=3, ll_seed=50005,
               chunk=50, scaling="strong"),
    # C2 on the epsilon-general, id-permuted generator (SURVEY §8.5 --permute-states)
    "c2eps": dict(graph=dict(n_states=50_000, degree=6.0, n_pdfs=2000), graph_kind="eps", n_pdfs=2000,
                  streams=100, frames=500, beam=10.0, max_active=10_000, preset="clean", graph_seed=2,
                  ll_seed=20002),
    # C3 on the epsilon-general, id-permuted generator: the pessimistic-locality variant
    "c3eps": dict(graph=dict(n_states=5_000_000, degree=3.0, n_pdfs=5700), graph_kind="eps", n_pdfs=5700,
                  streams=512, frames=500, beam=15.0, max_active=10_000, preset="clean", graph_seed=3,
                  ll_seed=30003),
}


def config_graph(name: str) -> Wfst:
    c = CONFIGS[name]
    if c["graph"] == "c1":
        return c1_graph()
    if c.get("graph_kind") == "eps":
        return hclg_graph_eps(seed=c["graph_seed"], **c["graph"])
    return hclg_graph(seed=c["graph_seed"], **c["graph"])


def preset(name_or_dict) -> dict:
    return PRESETS[name_or_dict] if isinstance(name_or_dict, str) else dict(name_or_dict)
