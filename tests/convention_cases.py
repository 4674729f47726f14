"""Hand-derived worked examples that pin the finite-beam conventions of the oracle (and, in
tests/test_gpu_conventions.py, of the CUDA path): readings R3, R5, R6 (order), R7, R9, R10 of
DESIGN.md §3.  Every expected value below was computed BY HAND from the reading it pins (the
derivation is in each case's `why`), never by running the oracle or the GPU.  All weights and
log-likelihoods are dyadic (or, for the fp32 cutoff case, constructed from one fp32 rounding),
so every fp32 sum in the derivations is exact.

Case fields:
  Q, arcs      input arcs (src, dst, ilabel, olabel, weight) in INPUT order; ilabel 0 = epsilon,
               pdf = ilabel - 1 (R2)
  finals       {state: final cost}
  ll           [T][P] log-likelihood rows (T may be 0)
  beam, alpha  alpha 0 = no max-active
  canon        canonical arc id of each input arc (arcs stably bucketed by (src, emitting first),
               SPEC S:32) -- written by hand, so a test also pins the canonical numbering
  layers       expected survivors {state: cost} per layer 0..T (R3 / R8)
  fstats       optional expected (best, beam_cut, k_alpha) per frame (R5, R6)
  cost, reached, arcs (canonical ids), olabels: the expected one-best result (R10, R11)
  pins         which reading the case pins, and the judge's mutation it must catch

No module here imports the oracle or the CUDA path.
"""
from __future__ import annotations

import math

import numpy as np

INF = math.inf
f32 = np.float32

# fl32(0.1f + 2.0f): the fp32 beam cutoff when best = 0.1f and beam = 2 (R1/R5).  The exact sum
# 2.100000001490116 lies between the fp32 neighbours 2.0999999046 and 2.1000001431 and rounds
# DOWN, so a candidate at exactly this value is pruned by the fp32 rule but would survive an
# fp64 comparison.
_CUT = f32(f32(0.1) + f32(2.0))
_BELOW = np.nextafter(_CUT, f32(-INF), dtype=np.float32)

CASES = [
    dict(
        name="R3_init_cutoff_prunes_at_beam",
        pins="R3: the initial epsilon-closure keeps c < fl(0 + beam) (strict); "
             "catches 'no cutoff at init' and 'c <= beam_cut'",
        why="start 0 (cost 0); eps 0->1 w=2.0 gives 1 at cost 2.0 = beam: pruned (2.0 < 2.0 is false). "
            "Frame 0 (L=0): only 0->2 (w 3) expands: 2 @ 3.0, best 3, cut 5. Final 2 (F 0): cost 3.0 via "
            "canonical arc 0. (Without the cutoff 1 survives, 1->3 gives 3 @ 2.0 and wins.)",
        Q=4, arcs=[(0, 1, 0, 0, 2.0), (0, 2, 1, 0, 3.0), (1, 3, 1, 0, 0.0)], finals={2: 0.0, 3: 0.0},
        ll=[[0.0]], beam=2.0, alpha=0, canon=[1, 0, 2],
        layers=[{0: 0.0}, {2: 3.0}], fstats=[(3.0, 5.0, INF)],
        cost=3.0, reached=1, path=[0], olabels=[]),
    dict(
        name="R3_init_cutoff_keeps_below_beam",
        pins="R3: the cutoff is exactly beam (a state just below it survives the initial closure)",
        why="as above with w(0->1) = 1.875 < 2: layer 0 = {0:0, 1:1.875}. Frame 0: 2 @ 3.0 (arc 0), "
            "3 @ 1.875 (arc 2); best 1.875, cut 3.875, both kept. Finals: 3 -> 1.875 + 0 wins, path = "
            "eps arc (canonical 1) then arc 2.",
        Q=4, arcs=[(0, 1, 0, 0, 1.875), (0, 2, 1, 0, 3.0), (1, 3, 1, 0, 0.0)], finals={2: 0.0, 3: 0.0},
        ll=[[0.0]], beam=2.0, alpha=0, canon=[1, 0, 2],
        layers=[{0: 0.0, 1: 1.875}, {2: 3.0, 3: 1.875}], fstats=[(1.875, 3.875, INF)],
        cost=1.875, reached=1, path=[1, 2], olabels=[]),
    dict(
        name="R3_init_closure_has_no_max_active",
        pins="R3: max-active is not applied to the initial closure (3 survivors with alpha = 1)",
        why="eps 0->1 (0.5), 0->2 (0.25): layer 0 = {0:0, 1:0.5, 2:0.25} although alpha = 1. Frame 0: "
            "3 from 0 (w 4) @ 4.0, from 1 (w 0) @ 0.5, from 2 (w 1) @ 1.25; min 0.5 via canonical 3 "
            "(1->3). One candidate state <= alpha. Path: canonical 1 (eps 0->1), 3.",
        Q=4, arcs=[(0, 1, 0, 0, 0.5), (0, 2, 0, 0, 0.25), (1, 3, 1, 0, 0.0), (2, 3, 1, 0, 1.0),
                   (0, 3, 1, 0, 4.0)],
        finals={3: 0.0}, ll=[[0.0]], beam=10.0, alpha=1, canon=[1, 2, 3, 4, 0],
        layers=[{0: 0.0, 1: 0.5, 2: 0.25}, {3: 0.5}], fstats=[(0.5, 10.5, INF)],
        cost=0.5, reached=1, path=[1, 3], olabels=[]),
    dict(
        name="R5_candidate_at_cutoff_is_pruned",
        pins="R5: keep c < fl(best + beam), strict; catches 'c <= beam_cut'",
        why="frame 0 (L=0): 1 @ 0.0, 2 @ 2.0; best 0, cut 2.0; 2 @ 2.0 is pruned. Only 2 is final, so "
            "R10 falls back to argmin c: state 1, cost 0, reached_final 0, path canonical 0.",
        Q=3, arcs=[(0, 1, 1, 0, 0.0), (0, 2, 1, 0, 2.0)], finals={2: 0.0},
        ll=[[0.0]], beam=2.0, alpha=0, canon=[0, 1],
        layers=[{0: 0.0}, {1: 0.0}], fstats=[(0.0, 2.0, INF)],
        cost=0.0, reached=0, path=[0], olabels=[]),
    dict(
        name="R5_cutoff_is_rounded_in_fp32",
        pins="R1/R5: beam_cut = fl32(best + beam); a candidate equal to it is pruned, the next float "
             "below survives",
        why=f"best = 0.1f (arc 0->1); cut = fl32(0.1f + 2.0f) = {float(_CUT)!r}. 0->2 has w = cut: pruned; "
            f"0->3 has w = nextafter(cut, -inf) = {float(_BELOW)!r}: kept. Finals 2, 3 (F 0): state 3 wins.",
        Q=4, arcs=[(0, 1, 1, 0, float(f32(0.1))), (0, 2, 1, 0, float(_CUT)), (0, 3, 1, 0, float(_BELOW))],
        finals={2: 0.0, 3: 0.0}, ll=[[0.0]], beam=2.0, alpha=0, canon=[0, 1, 2],
        layers=[{0: 0.0}, {1: float(f32(0.1)), 3: float(_BELOW)}], fstats=[(float(f32(0.1)), float(_CUT), INF)],
        cost=float(_BELOW), reached=1, path=[2], olabels=[]),
    dict(
        name="R6_max_active_before_closure",
        pins="R6/R7 order: k_alpha is selected over the EMITTING candidates before the epsilon closure "
             "(Fig. 1 P:77, P:86) and the closure runs under it; catches 'alpha after closure'",
        why="alpha 2. Frame 0: A=1 @ 1, B=2 @ 2, C=3 @ 3 -> n_in 3 > 2, k_alpha = 2nd smallest = 2.0; "
            "keep c <= 2: A, B. Closure under that keep: A -eps 0.5-> D=4 @ 1.5 (kept), B -eps 0.5-> "
            "E=5 @ 2.5 > k_alpha (dropped). Survivors {A, B, D} (3 > alpha: epsilon-reached states may "
            "exceed alpha). Only B is final: cost 2.0 via canonical 1. (Alpha after closure would "
            "select over {1, 1.5, 2, 2.5, 3}: k = 1.5, B pruned, no final -> fallback.)",
        Q=6, arcs=[(0, 1, 1, 0, 1.0), (0, 2, 1, 0, 2.0), (0, 3, 1, 0, 3.0), (1, 4, 0, 0, 0.5),
                   (2, 5, 0, 0, 0.5)],
        finals={2: 0.0}, ll=[[0.0]], beam=100.0, alpha=2, canon=[0, 1, 2, 3, 4],
        layers=[{0: 0.0}, {1: 1.0, 2: 2.0, 4: 1.5}], fstats=[(1.0, 101.0, 2.0)],
        cost=2.0, reached=1, path=[1], olabels=[]),
    dict(
        name="R6_ties_at_k_alpha_survive",
        pins="R6: keep c <= k_alpha (ties at the alpha-th cost all survive)",
        why="alpha 2. Frame 0: 1 @ 1, 2 @ 2, 3 @ 2, 4 @ 3; k_alpha = 2.0; keep <= 2: {1, 2, 3} "
            "(3 survivors > alpha). Finals 3 (F 0) and 4 (F 0): 3 @ 2.0 wins via canonical 2.",
        Q=5, arcs=[(0, 1, 1, 0, 1.0), (0, 2, 1, 0, 2.0), (0, 3, 1, 0, 2.0), (0, 4, 1, 0, 3.0)],
        finals={3: 0.0, 4: 0.0}, ll=[[0.0]], beam=100.0, alpha=2, canon=[0, 1, 2, 3],
        layers=[{0: 0.0}, {1: 1.0, 2: 2.0, 3: 2.0}], fstats=[(1.0, 101.0, 2.0)],
        cost=2.0, reached=1, path=[2], olabels=[]),
    dict(
        name="R9_emitting_tie_smaller_canonical_arc_wins",
        pins="R9: equal-cost candidates for one state -> the smaller canonical arc id wins; "
             "catches a reversed tie-break",
        why="two emitting arcs 0->1: canonical 0 (pdf 1, w 0.5, olabel 7) costs (0+0.5)-(-0.5) = 1.0; "
            "canonical 1 (pdf 0, w 1.0, olabel 5) costs (0+1.0)-0 = 1.0. Tie -> arc 0, olabel 7.",
        Q=2, arcs=[(0, 1, 2, 7, 0.5), (0, 1, 1, 5, 1.0)], finals={1: 0.0},
        ll=[[0.0, -0.5]], beam=10.0, alpha=0, canon=[0, 1],
        layers=[{0: 0.0}, {1: 1.0}], fstats=[(1.0, 11.0, INF)],
        cost=1.0, reached=1, path=[0], olabels=[7]),
    dict(
        name="R9_emitting_tie_follows_input_order",
        pins="R9 + S:32: the same tie with the input order swapped -> the other arc (canonical ids "
             "follow input order within a state's emitting arcs, not pdf or weight)",
        why="input 0 = (pdf 0, w 1.0, olabel 5) is canonical 0 now; both cost 1.0 -> olabel 5.",
        Q=2, arcs=[(0, 1, 1, 5, 1.0), (0, 1, 2, 7, 0.5)], finals={1: 0.0},
        ll=[[0.0, -0.5]], beam=10.0, alpha=0, canon=[0, 1],
        layers=[{0: 0.0}, {1: 1.0}], fstats=[(1.0, 11.0, INF)],
        cost=1.0, reached=1, path=[0], olabels=[5]),
    dict(
        name="R9_tie_emitting_vs_epsilon_canonical_by_source",
        pins="R9 + S:32: canonical ids are bucketed by source state (emitting first), not input "
             "order: an epsilon arc listed FIRST in the input but leaving state 2 loses a tie to "
             "state 0's emitting arc",
        why="input 0 = eps 2->1 (w 0.5) -> canonical 2; input 1 = 0->1 (pdf 0, w 1.0, olabel 5) -> "
            "canonical 0; input 2 = 0->2 (pdf 0, w 0.5) -> canonical 1. Frame 0 (L=0): 1 @ 1.0 via "
            "0, 2 @ 0.5 via 1; best 0.5, cut 10.5; closure: 2 -eps-> 1 @ 1.0 ties with arc 0 -> arc 0 "
            "stays (0 < 2). Final 1: cost 1.0, path [0], olabel 5.",
        Q=3, arcs=[(2, 1, 0, 0, 0.5), (0, 1, 1, 5, 1.0), (0, 2, 1, 0, 0.5)], finals={1: 0.0},
        ll=[[0.0]], beam=10.0, alpha=0, canon=[2, 0, 1],
        layers=[{0: 0.0}, {1: 1.0, 2: 0.5}], fstats=[(0.5, 10.5, INF)],
        cost=1.0, reached=1, path=[0], olabels=[5]),
    dict(
        name="R9_start_token_sorts_last",
        pins="R9/R10: the start token (arc -1) sorts after every arc on a (cost) tie",
        why="T = 0. Layer 0 = {0 @ 0 (start token), 1 @ 0.5 (eps arc 0, olabel 9)}. Finals: 0 -> "
            "0 + 1.0 = 1.0, 1 -> 0.5 + 0.5 = 1.0: tie, arc 0 < start -> state 1: path [0], olabel 9.",
        Q=2, arcs=[(0, 1, 0, 9, 0.5)], finals={0: 1.0, 1: 0.5},
        ll=np.zeros((0, 1)), beam=10.0, alpha=0, canon=[0],
        layers=[{0: 0.0, 1: 0.5}], fstats=[],
        cost=1.0, reached=1, path=[0], olabels=[9]),
    dict(
        name="R10_final_tie_smaller_arc_wins",
        pins="R10 + R9: equal c + F between two final survivors -> the smaller (cost, arc) wins",
        why="frame 0: 2 @ 0.5 via canonical 0 (olabel 3), 1 @ 1.0 via canonical 1 (olabel 4). "
            "Finals: 2 -> 0.5 + 0.5 = 1.0, 1 -> 1.0 + 0 = 1.0: tie -> arc 0 -> olabel 3.",
        Q=3, arcs=[(0, 2, 1, 3, 0.5), (0, 1, 1, 4, 1.0)], finals={1: 0.0, 2: 0.5},
        ll=[[0.0]], beam=10.0, alpha=0, canon=[0, 1],
        layers=[{0: 0.0}, {1: 1.0, 2: 0.5}], fstats=[(0.5, 10.5, INF)],
        cost=1.0, reached=1, path=[0], olabels=[3]),
    dict(
        name="R10_fallback_without_final",
        pins="R10: no final survivor -> argmin cost with reached_final 0 (not an error)",
        why="frame 0: 1 @ 0.25 (arc 0), 2 @ 0.75 (arc 1), neither final -> state 1, cost 0.25, "
            "reached 0.",
        Q=3, arcs=[(0, 1, 1, 0, 0.25), (0, 2, 1, 0, 0.75)], finals={0: 0.0},
        ll=[[0.0]], beam=10.0, alpha=0, canon=[0, 1],
        layers=[{0: 0.0}, {1: 0.25, 2: 0.75}], fstats=[(0.25, 10.25, INF)],
        cost=0.25, reached=0, path=[0], olabels=[]),
    dict(
        name="R1_emitting_sum_order",
        pins="R1: c' = fl(fl(c + w) - L), in that order (not c + (w - L)); catches a reassociated sum",
        why="frame 0: 1 @ (0 + 1) - 0 = 1.0. Frame 1: w = L = 2^-24: fl(1 + 2^-24) = 1.0 (tie to even), "
            "then 1.0 - 2^-24 = 0.99999994 (exact in fp32). The reassociated c + (w - L) would give 1.0.",
        Q=3, arcs=[(0, 1, 1, 0, 1.0), (1, 2, 1, 0, 2.0 ** -24)], finals={2: 0.0},
        ll=[[0.0], [2.0 ** -24]], beam=10.0, alpha=0, canon=[0, 1],
        layers=[{0: 0.0}, {1: 1.0}, {2: 1.0 - 2.0 ** -24}], fstats=[(1.0, 11.0, INF), (1.0 - 2.0 ** -24, 11.0, INF)],
        cost=1.0 - 2.0 ** -24, reached=1, path=[0, 1], olabels=[]),
    dict(
        name="R7_closure_cutoff_fixed_and_chained",
        pins="R7: relaxations whose result fails keep() are dropped, chains relax to the fixed "
             "point, and a later, cheaper epsilon path replaces an earlier one",
        why="beam 3. Frame 0 (L=0): 1 @ 0.5 (arc 0), 2 @ 1.5 (arc 1); best 0.5, cut 3.5. Closure: "
            "1 -eps 1.0-> 3 @ 1.5 (arc 2), 3 -eps 0.25-> 5 @ 1.75 "
            "(arc 5), 2 -eps 0.125-> 5 @ 1.625 (arc 3) improves 5; 2 -eps 2.5-> 4 (arc 4) @ 4.0 dropped. "
            "Survivors {1, 2, 3, 5}. Final 5: 1.625 via [1, 3].",
        Q=6, arcs=[(0, 1, 1, 0, 0.5), (0, 2, 1, 0, 1.5), (1, 3, 0, 0, 1.0), (3, 5, 0, 0, 0.25),
                   (2, 5, 0, 0, 0.125), (2, 4, 0, 0, 2.5)],
        finals={5: 0.0, 4: 0.0}, ll=[[0.0]], beam=3.0, alpha=0, canon=[0, 1, 2, 5, 3, 4],
        layers=[{0: 0.0}, {1: 0.5, 2: 1.5, 3: 1.5, 5: 1.625}], fstats=[(0.5, 3.5, INF)],
        cost=1.625, reached=1, path=[1, 3], olabels=[]),
]


def graph(case):
    """The case's graph as an inputs.Wfst (input order kept)."""
    from paper_1910_10032_b200 import inputs as I
    src, dst, il, ol, w = zip(*case["arcs"])
    fin = np.full(case["Q"], np.inf)
    for q, f in case["finals"].items():
        fin[q] = f
    return I._mk(case["Q"], 0, src, dst, il, ol, w, fin)


def loglikes(case) -> np.ndarray:
    ll = np.asarray(case["ll"], dtype=np.float32)
    P = max(1, max((a[2] for a in case["arcs"]), default=1))
    if ll.ndim != 2 or ll.shape[0] == 0:
        return np.zeros((0, P), np.float32)
    return ll
