"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  The product package
`paper_1910_10032_b200` never imports it and shares no code with it.

`wfst_oracle.c` is the serial token-passing Viterbi beam search of PAPER.md §3
(Fig. 1) under the readings R1-R12 listed in
DESIGN.md §3, plus the NEXT rows: lattice segments and the end-of-utterance
sweep (R13-R14, row f1) and the histogram max-active rule (R16, row f4); this
module builds it with gcc and marshals arguments.  `OracleGraph.settled_prefix`
(R15, row f2) is written here in Python as its definition (every survivor's
traceback, longest common prefix).
Pins (tests/test_oracle_*.py): fp64 trellis Bellman-Ford and exhaustive path
enumeration (tests/bruteforce.py), SPEC worked examples, closed forms,
invariants.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wfst_oracle.c")
_LIB = os.path.join(_HERE, "libwfst_oracle.so")
# tests/test_oracle_mutations.py loads deliberately broken copies of the oracle (built from a
# mutated scratch copy of wfst_oracle.c) to prove that the convention pins catch each mutation
_LIB_OVERRIDE = os.environ.get("WFST_ORACLE_LIB")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]

RC = {0: "OK", 1: "INVALID", 5: "PDF_RANGE", 6: "CAPACITY", 7: "NO_SURVIVOR", 9: "OOM"}


class OracleError(RuntimeError):
    def __init__(self, rc: int, what: str = ""):
        super().__init__(f"oracle {what}: {RC.get(rc, rc)}")
        self.rc = rc


def build(force: bool = False) -> str:
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, I32, I64, F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        L.oracle_graph_new.argtypes = [I32, I32, I64, P, P, P, P, P, P, C.POINTER(C.c_void_p)]
        L.oracle_graph_free.argtypes = [P]
        L.oracle_graph_perm.argtypes = [P, P]
        L.oracle_graph_max_pdf.argtypes = [P]
        L.oracle_graph_max_pdf.restype = I32
        L.oracle_decode.argtypes = [P, P, I64, I32, I32, F32, I32, P, P, P, I32, P, P, I32, P,
                                    P, P, P, P, P, P, I64, P]
        L.oracle_decode_mode.argtypes = [P, P, I64, I32, I32, F32, I32, I32, P, P, P, I32, P, P, I32, P, P]
        L.oracle_decode_batch.argtypes = [P, P, I32, I32, I32, F32, I32, I32, P, P, P, P, P, I32, P]
        L.oracle_lattice.argtypes = [P, P, I64, I32, F32, F32, P, P, P, P, P, P, P, P, P, I64, P]
        L.oracle_lattice_finalize.argtypes = [P, I32, P, P, P, P, P, P, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleResult:
    def __init__(self, **kw):
        self.__dict__.update(kw)

    def __repr__(self):
        return f"OracleResult(cost={self.cost}, reached_final={self.reached_final}, olabels={self.olabels})"


class OracleGraph:
    """The oracle's own canonical CSR of a graph given as plain arrays."""

    def __init__(self, g):
        self.g = g
        L = lib()
        self._arr = [np.ascontiguousarray(x) for x in
                     (g.src.astype(np.int32), g.dst.astype(np.int32), g.ilabel.astype(np.int32),
                      g.olabel.astype(np.int32), g.weight.astype(np.float32), g.final.astype(np.float32))]
        h = C.c_void_p()
        rc = L.oracle_graph_new(g.n_states, g.start, g.n_arcs, *[_p(a) for a in self._arr], C.byref(h))
        if rc:
            raise OracleError(rc, "graph_new")
        self.h = h
        self.max_pdf = L.oracle_graph_max_pdf(h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_graph_free(self.h)
            self.h = None

    def perm(self) -> np.ndarray:
        out = np.empty(self.g.n_arcs, dtype=np.int64)
        lib().oracle_graph_perm(self.h, _p(out))
        return out

    def decode(self, ll: np.ndarray, beam: float, max_active: int = 0, survivors: bool = False,
               surv_cap: int | None = None) -> OracleResult:
        """ll: float32 [T][P] (or a [T][...][P] view whose frame stride is given by ll.strides)."""
        ll = np.asarray(ll, dtype=np.float32)
        if ll.ndim != 2:
            raise ValueError("ll must be [T][P]")
        if ll.strides[1] != 4:
            ll = np.ascontiguousarray(ll)
        T, P = ll.shape
        stride = ll.strides[0] // 4
        cost = np.zeros(1, np.float32)
        rf = np.zeros(1, np.int32)
        cap = 4 * (T + 1) + 64
        arcs = np.zeros(cap, np.int32)
        n_arcs = np.zeros(1, np.int32)
        ol = np.zeros(cap, np.int32)
        n_ol = np.zeros(1, np.int32)
        fst = np.zeros((max(T, 1), 3), np.float32)
        fcn = np.zeros((max(T, 1), 5), np.int64)
        relax = np.zeros(1, np.int64)
        sn = sst = sar = sco = None
        scap = 0
        if survivors:
            scap = surv_cap or max(1, (T + 1) * self.g.n_states)
            sn = np.zeros(T + 1, np.int32)
            sst = np.zeros(scap, np.int32)
            sar = np.zeros(scap, np.int32)
            sco = np.zeros(scap, np.float32)
        rc = lib().oracle_decode(self.h, _p(ll) if T else None, stride, T, P, float(beam),
                                 int(max_active), _p(cost), _p(rf), _p(arcs), cap, _p(n_arcs),
                                 _p(ol), cap, _p(n_ol), _p(fst), _p(fcn), _p(sn), _p(sst), _p(sar),
                                 _p(sco), scap, _p(relax))
        if rc:
            raise OracleError(rc, "decode")
        res = OracleResult(cost=float(cost[0]), cost32=cost[0], reached_final=int(rf[0]),
                           arcs=arcs[: n_arcs[0]].copy(), olabels=ol[: n_ol[0]].copy(),
                           frame_stats=fst[:T].copy(), frame_counts=fcn[:T].copy(),
                           eps_relax=int(relax[0]))
        if survivors:
            offs = np.concatenate([[0], np.cumsum(sn)])
            res.layers = [(sst[offs[k]:offs[k + 1]].copy(), sar[offs[k]:offs[k + 1]].copy(),
                           sco[offs[k]:offs[k + 1]].copy()) for k in range(T + 1)]
        return res

    def lattice(self, ll: np.ndarray, beam: float, max_active: int, lattice_beam: float,
                cap: int | None = None) -> OracleResult:
        """Row f1: decode (survivors kept) + per-frame lattice segments + the end-of-utterance
        backward sweep (oracle_lattice / oracle_lattice_finalize; readings R13-R14).
        Returns the decode result with .segments[k] = (arc, src, dst, slack) arrays (grouped by
        dst, arc ascending), .gamma[k] per token of layer k, .pslack[k] per arc of segment k."""
        ll = np.ascontiguousarray(ll, dtype=np.float32)
        T = ll.shape[0]
        r = self.decode(ll, beam, max_active, survivors=True)
        sn = np.array([len(L[0]) for L in r.layers], np.int32)
        sst = np.ascontiguousarray(np.concatenate([L[0] for L in r.layers]).astype(np.int32))
        sco = np.ascontiguousarray(np.concatenate([L[2] for L in r.layers]).astype(np.float32))
        fst = np.ascontiguousarray(r.frame_stats if T else np.zeros((1, 3), np.float32))
        if cap is None:
            cap = int(max(1, sum(len(L[0]) for L in r.layers) * max(1, self.g.n_arcs // max(1, self.g.n_states)) * 4))
        seg_n = np.zeros(T + 1, np.int32)
        la, ls, ld = (np.zeros(cap, np.int32) for _ in range(3))
        lsl = np.zeros(cap, np.float32)
        n = np.zeros(1, np.int64)
        rc = lib().oracle_lattice(self.h, _p(ll) if T else None, ll.shape[1] if T else 0, T, float(beam),
                                  float(lattice_beam), _p(fst), _p(sn), _p(sst), _p(sco), _p(seg_n),
                                  _p(la), _p(ls), _p(ld), _p(lsl), cap, _p(n))
        if rc == 6:
            return self.lattice(ll, beam, max_active, lattice_beam, cap=int(n[0]) + 1)
        if rc:
            raise OracleError(rc, "lattice")
        m = int(n[0])
        gamma = np.zeros(max(1, len(sst)), np.float32)
        pslack = np.zeros(max(1, m), np.float32)
        best = np.zeros(1, np.float32)
        reached = np.zeros(1, np.int32)
        rc = lib().oracle_lattice_finalize(self.h, T, _p(sn), _p(sst), _p(sco), _p(seg_n), _p(la), _p(ls),
                                           _p(ld), _p(lsl), _p(gamma), _p(pslack), _p(best), _p(reached))
        if rc:
            raise OracleError(rc, "lattice_finalize")
        so = np.concatenate([[0], np.cumsum(seg_n)])
        lo = np.concatenate([[0], np.cumsum(sn)])
        r.segments = [(la[so[k]:so[k + 1]].copy(), ls[so[k]:so[k + 1]].copy(), ld[so[k]:so[k + 1]].copy(),
                       lsl[so[k]:so[k + 1]].copy()) for k in range(T + 1)]
        r.gamma = [gamma[lo[k]:lo[k + 1]].copy() for k in range(T + 1)]
        r.pslack = [pslack[so[k]:so[k + 1]].copy() for k in range(T + 1)]
        r.lattice_best = float(best[0])
        r.lattice_beam = float(lattice_beam)
        return r

    def decode_hist(self, ll: np.ndarray, beam: float, max_active: int) -> OracleResult:
        """Row f4: decode with the histogram max-active rule R16 instead of the exact R6."""
        ll = np.ascontiguousarray(ll, dtype=np.float32)
        T, P = ll.shape
        cost = np.zeros(1, np.float32)
        rf = np.zeros(1, np.int32)
        cap = 4 * (T + 1) + 64
        arcs = np.zeros(cap, np.int32)
        n_arcs = np.zeros(1, np.int32)
        ol = np.zeros(cap, np.int32)
        n_ol = np.zeros(1, np.int32)
        fst = np.zeros((max(T, 1), 3), np.float32)
        fcn = np.zeros((max(T, 1), 5), np.int64)
        rc = lib().oracle_decode_mode(self.h, _p(ll) if T else None, P, T, P, float(beam), int(max_active), 1,
                                      _p(cost), _p(rf), _p(arcs), cap, _p(n_arcs), _p(ol), cap, _p(n_ol),
                                      _p(fst), _p(fcn))
        if rc:
            raise OracleError(rc, "decode_hist")
        return OracleResult(cost=float(cost[0]), cost32=cost[0], reached_final=int(rf[0]),
                            arcs=arcs[: n_arcs[0]].copy(), olabels=ol[: n_ol[0]].copy(),
                            frame_stats=fst[:T].copy(), frame_counts=fcn[:T].copy())

    def settled_prefix(self, ll: np.ndarray, beam: float, max_active: int = 0) -> np.ndarray:
        """Row f2 (reading R15; "intermediate results during online decoding"): decode the
        frames of ll, then take the traceback (canonical arc ids, start first) of EVERY survivor of
        the last layer, their longest common prefix, cut after its last emitting arc.  Written as
        the definition -- every path is traced in full -- not as the GPU's walk-back."""
        r = self.decode(ll, beam, max_active, survivors=True)
        perm = self.perm()
        src_c = self.g.src[perm]
        emit_c = self.g.ilabel[perm] != 0
        maps = [dict(zip(L[0].tolist(), L[1].tolist())) for L in r.layers]   # state -> winning arc

        def trace(k, q):
            out = []
            while True:
                a = maps[k][q]
                if a < 0:
                    return out[::-1]
                out.append(a)
                if emit_c[a]:
                    k -= 1
                q = int(src_c[a])

        T = len(r.layers) - 1
        paths = [trace(T, int(q)) for q in r.layers[T][0]]
        lcp = []
        for col in zip(*paths):
            if any(x != col[0] for x in col):
                break
            lcp.append(col[0])
        while lcp and not emit_c[lcp[-1]]:
            lcp.pop()
        return np.array(lcp, np.int64)

    def decode_batch(self, ll: np.ndarray, beam: float, max_active: int, n_threads: int,
                     arcs_cap: int = 0):
        """ll: float32 [T][B][P] contiguous.  Returns (cost, reached, rc, arcs_count, arcs, n_arcs)."""
        ll = np.ascontiguousarray(ll, dtype=np.float32)
        T, B, P = ll.shape
        cost = np.zeros(B, np.float32)
        reached = np.zeros(B, np.int32)
        rc = np.zeros(B, np.int32)
        cnt = np.zeros(B, np.int64)
        arcs = np.zeros((B, arcs_cap), np.int32) if arcs_cap else None
        n_arcs = np.zeros(B, np.int32) if arcs_cap else None
        r = lib().oracle_decode_batch(self.h, _p(ll), T, B, P, float(beam), int(max_active),
                                      int(n_threads), _p(cost), _p(reached), _p(rc), _p(cnt),
                                      _p(arcs), arcs_cap, _p(n_arcs))
        if r:
            raise OracleError(r, "decode_batch")
        return cost, reached, rc, cnt, arcs, n_arcs
