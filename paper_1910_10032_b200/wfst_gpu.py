"""Thin Python binding over the C ABI in include/wfst_gpu.h (argument marshalling only).

Every step of the decode runs in libwfst_gpu.so's CUDA kernels; this module only converts
numpy arrays / torch CUDA tensors to pointers and sizes.  There is no CPU fallback: if the
library is missing, `lib()` raises.  Torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwfst_gpu.so")

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "PARSE", 3: "GRAPH_INVALID", 4: "EPS_CYCLE", 5: "PDF_RANGE",
          6: "CAPACITY", 7: "NO_SURVIVOR", 8: "CUDA", 9: "OOM", 10: "STATE"}

SYMBOLS = ["wfst_load_graph", "wfst_graph_from_arrays", "wfst_graph_info", "wfst_graph_canonical_perm",
           "wfst_graph_free", "wfst_eq1_bytes", "wfst_eq2_bytes", "wfst_decoder_create",
           "wfst_decoder_create_ex", "wfst_decoder_destroy", "wfst_decoder_reset", "wfst_decode_frames",
           "wfst_decode_frames_host", "wfst_decoder_sync", "wfst_decoder_status", "wfst_get_best_path",
           "wfst_get_best_paths", "wfst_decoder_stats", "wfst_decoder_reset_stats", "wfst_decoder_frame_stats",
           "wfst_debug_layer", "wfst_synth_loglikes", "wfst_last_error", "wfst_status_string",
           "wfst_abi_version", "wfst_get_lattice", "wfst_get_partial_paths", "wfst_graph_replicate",
           "wfst_get_best_paths_ex", "wfst_get_partial_paths_ex", "wfst_get_partial_paths_packed"]


class WfstError(RuntimeError):
    def __init__(self, code: int, msg: str, result=None):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))
        self.result = result   # per-stream results of a batched call that failed for some streams


class GraphInfo(C.Structure):
    _fields_ = [("n_states", C.c_int32), ("start", C.c_int32), ("n_arcs", C.c_int64),
                ("n_emitting", C.c_int64), ("max_pdf", C.c_int32), ("device", C.c_int32),
                ("device_bytes", C.c_int64), ("eq1_bytes", C.c_int64)]


class DecoderOpts(C.Structure):
    _fields_ = [("table_slots", C.c_int32), ("overflow_slots", C.c_int32), ("records_per_stream", C.c_int64),
                ("max_frames", C.c_int32), ("threads", C.c_int32), ("frames_per_item", C.c_int32),
                ("max_ctas", C.c_int32), ("debug_costs", C.c_int32), ("ctas_per_sm", C.c_int32),
                ("lattice", C.c_int32), ("lattice_beam", C.c_float), ("lattice_arcs_per_stream", C.c_int64),
                ("max_active_mode", C.c_int32), ("reclaim", C.c_int32), ("insert_order", C.c_int32),
                ("bin_capacity", C.c_int32), ("ll_columns", C.c_int32),
                ("gc_frames", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("frames", "emit_arcs", "eps_arcs", "eps_relax", "candidates", "survivors",
                                         "overflow_inserts", "alpha_frames", "device_bytes", "records_used_max")] + \
        [("phase_cycles", C.c_int64 * 12), ("select_entries", C.c_int64), ("phase_cycles_alpha", C.c_int64 * 12),
         ("records_per_stream", C.c_int64), ("record_bytes", C.c_int64)]
    PHASES = ("prefetch", "cutoff", "epsilon", "expand_warp", "expand_hub", "overhead", "drain", "bin_insert", "placement",
              "eps_backptr", "table_reset", "row_wait")

    def as_dict(self):
        d = {n: int(getattr(self, n)) for n, _ in self._fields_ if not n.startswith("phase_cycles")}
        d["phase_cycles"] = dict(zip(self.PHASES, (int(x) for x in self.phase_cycles)))
        d["phase_cycles_alpha"] = dict(zip(self.PHASES, (int(x) for x in self.phase_cycles_alpha)))
        return d


_lib = None


def lib():
    """Load libwfst_gpu.so (built by paper_1910_10032_b200.build); fails loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_1910_10032_b200.build` "
                               "(the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, F32, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_uint64
        sig = {
            "wfst_load_graph": [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)],
            "wfst_graph_from_arrays": [I32, I32, I64, P, P, P, P, P, P, C.c_int, C.POINTER(C.c_void_p)],
            "wfst_graph_info": [P, C.POINTER(GraphInfo)],
            "wfst_graph_canonical_perm": [P, P, I64],
            "wfst_graph_free": [P],
            "wfst_eq1_bytes": [I64, I64, I64],
            "wfst_eq2_bytes": [I64, I64, I64],
            "wfst_decoder_create": [P, I32, F32, I32, C.POINTER(C.c_void_p)],
            "wfst_decoder_create_ex": [P, I32, F32, I32, C.POINTER(DecoderOpts), C.POINTER(C.c_void_p)],
            "wfst_decoder_destroy": [P],
            "wfst_decoder_reset": [P, P, I32, P],
            "wfst_decode_frames": [P, P, I32, I32, I32, P, P],
            "wfst_decode_frames_host": [P, P, I32, I32, I32, P, I32, P],
            "wfst_decoder_sync": [P],
            "wfst_decoder_status": [P, I32],
            "wfst_get_best_path": [P, I32, P, I32, P, P, I32, P, P, P],
            "wfst_get_best_paths": [P, P, I32, P, P, P, P, I32, P, P],
            "wfst_decoder_stats": [P, C.POINTER(Stats)],
            "wfst_decoder_reset_stats": [P],
            "wfst_decoder_frame_stats": [P, I32, P, P, I32, P],
            "wfst_debug_layer": [P, I32, I32, P, P, P, I32, P],
            "wfst_synth_loglikes": [P, I32, I32, I32, P, I32, U64, P, F32, F32, P],
            "wfst_last_error": [],
            "wfst_status_string": [C.c_int],
            "wfst_abi_version": [],
            "wfst_get_lattice": [P, I32, P, I32, P, P, P, P, P, P, I64, P, P, I64, P, P, P],
            "wfst_get_partial_paths": [P, P, I32, P, P, I32, P, P, P],
            "wfst_get_best_paths_ex": [P, P, I32, P, P, P, P, I32, P, P, P],
            "wfst_get_partial_paths_ex": [P, P, I32, P, P, I32, P, P, P, P],
            "wfst_get_partial_paths_packed": [P, P, I32, P, P, I64, I32, P, P, P, P, P, P],
            "wfst_graph_replicate": [P, C.c_int, P],
        }
        for name, args in sig.items():
            fn = getattr(L, name, None)
            if fn is None:   # an older library (A/B experiments); tests check the exports
                continue
            fn.argtypes = args
            fn.restype = C.c_int
        L.wfst_eq1_bytes.restype = I64
        L.wfst_eq2_bytes.restype = I64
        L.wfst_last_error.restype = C.c_char_p
        L.wfst_status_string.restype = C.c_char_p
        L.wfst_graph_free.restype = None
        L.wfst_decoder_destroy.restype = None
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise WfstError(rc, lib().wfst_last_error().decode(errors="replace"))


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _ids(streams):
    if streams is None:
        return None, 0
    a = _np(streams, np.int32)
    return a, int(a.size)


# ------------------------------------------------------------------ host-only helpers
class _Rows:
    """Sequence of per-stream views a[off[i] : off[i] + min(n[i], cap)] of a packed result, built
    on access (a 4096-stream result costs no per-stream Python work unless the rows are read)."""
    __slots__ = ("_a", "_n", "_off", "_cap")

    def __init__(self, a, n, off, cap):
        self._a, self._n, self._off, self._cap = a, n, off, cap

    def __len__(self):
        return len(self._n)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        o = int(self._off[i])
        return self._a[o:o + min(int(self._n[i]), self._cap)]

    def __iter__(self):
        return (self[i] for i in range(len(self)))


def eq1_bytes(n_states, n_arcs, n_emitting) -> int:
    """Eq. 1: 12|Q| + 8|E| + 4|E_E|."""
    return int(lib().wfst_eq1_bytes(n_states, n_arcs, n_emitting))


def eq2_bytes(max_active, n_channels, n_lanes) -> int:
    """Eq. 2: 64 a n_c + 544 a n_l + 1024 n_l."""
    return int(lib().wfst_eq2_bytes(max_active, n_channels, n_lanes))


# ------------------------------------------------------------------ graph
class Graph:
    """Device-resident decode graph (wfst_graph_t)."""

    def __init__(self, handle, device):
        self.h = handle
        self.device = device
        self._info = None

    @classmethod
    def load(cls, path: str, device: int = 0) -> "Graph":
        h = C.c_void_p()
        _check(lib().wfst_load_graph(path.encode(), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def from_arrays(cls, g, device: int = 0) -> "Graph":
        """g: object with n_states, start, src, dst, ilabel, olabel, weight, final (numpy)."""
        arrs = [_np(g.src, np.int32), _np(g.dst, np.int32), _np(g.ilabel, np.int32), _np(g.olabel, np.int32),
                _np(g.weight, np.float32), _np(g.final, np.float32)]
        h = C.c_void_p()
        _check(lib().wfst_graph_from_arrays(int(g.n_states), int(g.start), int(arrs[0].size),
                                            *[_ptr(a) for a in arrs], device, C.byref(h)))
        return cls(h, device)

    def replicate(self, device: int) -> "Graph":
        """Row e: a copy of this graph on another CUDA device (wfst_graph_replicate)."""
        h = C.c_void_p()
        _check(lib().wfst_graph_replicate(self.h, device, C.byref(h)))
        return Graph(h, device)

    def info(self) -> GraphInfo:
        if self._info is None:
            i = GraphInfo()
            _check(lib().wfst_graph_info(self.h, C.byref(i)))
            self._info = i
        return self._info

    def canonical_perm(self) -> np.ndarray:
        out = np.empty(self.info().n_arcs, np.int64)
        _check(lib().wfst_graph_canonical_perm(self.h, _ptr(out), out.size))
        return out

    def free(self):
        if self.h:
            lib().wfst_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ------------------------------------------------------------------ decoder
class Decoder:
    """wfst_decoder_t: n_streams lanes decoding in lock-step frames on the graph's device."""

    def __init__(self, graph: Graph, n_streams: int, beam: float = 15.0, max_active: int = 10000, **opts):
        self.graph = graph
        self.n_streams = n_streams
        self.beam = beam
        self.max_active = max_active
        h = C.c_void_p()
        o = DecoderOpts()
        for k, v in opts.items():
            setattr(o, k, float(v) if k == "lattice_beam" else int(v))
        _check(lib().wfst_decoder_create_ex(graph.h, n_streams, float(beam), int(max_active or 0), C.byref(o),
                                            C.byref(h)))
        self.h = h

    def destroy(self):
        if getattr(self, "h", None):
            lib().wfst_decoder_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def reset(self, streams=None, stream=None):
        ids, n = _ids(streams)
        _check(lib().wfst_decoder_reset(self.h, _ptr(ids), n, _stream_ptr(stream)))

    def decode_frames(self, loglikes, streams=None, stream=None):
        """loglikes: torch.cuda float32 tensor [T][B][P] (contiguous) or a raw device pointer via
        decode_frames_ptr.  Asynchronous on the current torch stream."""
        t = loglikes
        assert t.is_cuda and t.dtype.__str__() == "torch.float32" and t.is_contiguous() and t.dim() == 3
        T, B, P = t.shape
        ids, n = _ids(streams)
        if ids is not None and n != B:
            raise ValueError("len(streams) != B")
        _check(lib().wfst_decode_frames(self.h, C.c_void_p(t.data_ptr()), T, B, P, _ptr(ids), _stream_ptr(stream)))

    def decode_frames_ptr(self, ptr: int, T: int, B: int, P: int, streams=None, stream=None):
        ids, n = _ids(streams)
        _check(lib().wfst_decode_frames(self.h, C.c_void_p(ptr), T, B, P, _ptr(ids), _stream_ptr(stream)))

    def decode_frames_host(self, loglikes: np.ndarray, streams=None, chunk_frames: int = 0, stream=None):
        """Host float32 [T][B][P] (pinned or pageable; a pinned torch CPU tensor also works)."""
        T, B, P = loglikes.shape
        ids, n = _ids(streams)
        ptr = C.c_void_p(loglikes.data_ptr()) if hasattr(loglikes, "data_ptr") else _ptr(loglikes)
        self._host_ref = loglikes
        _check(lib().wfst_decode_frames_host(self.h, ptr, T, B, P, _ptr(ids), chunk_frames, _stream_ptr(stream)))

    def sync(self):
        _check(lib().wfst_decoder_sync(self.h))

    def status(self, stream: int) -> str:
        return STATUS.get(lib().wfst_decoder_status(self.h, stream), "?")

    def best_path(self, stream: int, cap: int = 1 << 16):
        ol = np.zeros(cap, np.int32)
        ar = np.zeros(cap, np.int32)
        nol, nar = np.zeros(1, np.int32), np.zeros(1, np.int32)
        cost = np.zeros(1, np.float32)
        rf = np.zeros(1, np.int32)
        _check(lib().wfst_get_best_path(self.h, stream, _ptr(ol), cap, _ptr(nol), _ptr(ar), cap, _ptr(nar),
                                        _ptr(cost), _ptr(rf)))
        return dict(cost=float(cost[0]), cost32=cost[0], reached_final=int(rf[0]), olabels=ol[: nol[0]].copy(),
                    arcs=ar[: nar[0]].copy())

    def best_paths(self, streams=None, cap: int = 2048, raise_on_error: bool = True):
        ids = np.arange(self.n_streams, dtype=np.int32) if streams is None else _np(streams, np.int32)
        n = ids.size
        cost = np.zeros(n, np.float32)
        rf = np.zeros(n, np.int32)
        arcs = np.zeros((n, cap), np.int32)
        ols = np.zeros((n, cap), np.int32)
        nar = np.zeros(n, np.int32)
        nol = np.zeros(n, np.int32)
        status = np.zeros(n, np.int32)
        rc = lib().wfst_get_best_paths_ex(self.h, _ptr(ids), n, _ptr(cost), _ptr(rf), _ptr(arcs), _ptr(ols), cap,
                                          _ptr(nar), _ptr(nol), _ptr(status))
        out = dict(cost=cost, reached_final=rf, arcs=arcs, n_arcs=nar, olabels=ols, n_olabels=nol, rc=rc,
                   status=status)
        if raise_on_error and rc != 0:
            raise WfstError(rc, lib().wfst_last_error().decode(errors="replace"), out)
        return out

    def stats(self) -> dict:
        s = Stats()
        _check(lib().wfst_decoder_stats(self.h, C.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        _check(lib().wfst_decoder_reset_stats(self.h))

    def frame_stats(self, stream: int, cap: int = 4096):
        fs = np.zeros((cap, 3), np.float32)
        fc = np.zeros((cap, 5), np.int64)
        n = np.zeros(1, np.int32)
        _check(lib().wfst_decoder_frame_stats(self.h, stream, _ptr(fs), _ptr(fc), cap, _ptr(n)))
        k = min(int(n[0]), cap)
        return fs[:k], fc[:k]

    def debug_layer(self, stream: int, layer: int, cap: int = 1 << 17):
        st = np.zeros(cap, np.int32)
        ar = np.zeros(cap, np.int32)
        co = np.zeros(cap, np.float32)
        n = np.zeros(1, np.int32)
        _check(lib().wfst_debug_layer(self.h, stream, layer, _ptr(st), _ptr(ar), _ptr(co), cap, _ptr(n)))
        k = int(n[0])
        return st[:k].copy(), ar[:k].copy(), co[:k].copy()


    def partial_paths(self, streams=None, cap: int = 512, raise_on_error: bool = True) -> dict:
        """Row f2: the arcs/olabels settled since the previous call, per stream
        (wfst_get_partial_paths_ex), the frames the settled prefix covers and each stream's status.
        cap grows on demand (a stream that does not fit keeps its settle point, so the call is simply
        repeated).  A stream with an error raises WfstError after the others' arcs are collected
        (e.result holds them); raise_on_error=False returns them with status instead."""
        ids = np.arange(self.n_streams, dtype=np.int32) if streams is None else _np(streams, np.int32)
        n = ids.size
        # packed outputs (wfst_get_partial_paths_packed): only the settled arcs are copied and
        # written, so the n * cap buffers are touched only where arcs land (this runs every chunk)
        arcs = np.empty(n * cap, np.int32)
        ols = np.empty(n * cap, np.int32)
        off = np.zeros(n, np.int64)
        tot = np.zeros(1, np.int64)
        nar, nol, fr = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32)
        status = np.zeros(n, np.int32)
        rc = lib().wfst_get_partial_paths_packed(self.h, _ptr(ids), n, _ptr(arcs), _ptr(ols), C.c_int64(n * cap), cap,
                                                 _ptr(off), _ptr(tot), _ptr(nar), _ptr(nol), _ptr(fr), _ptr(status))
        arcs, ols = _Rows(arcs, nar, off, cap), _Rows(ols, nol, off, cap)
        if rc == 0:   # per-stream views, made on access
            return dict(arcs=arcs, olabels=ols, settled_frames=fr, status=status)
        # per stream: OK streams advanced their settle point (their arcs must not be dropped);
        # streams whose new arcs exceeded cap kept theirs and are fetched again with a larger cap
        big = (status == 1) & (nar > cap)
        out_a = [arcs[i].copy() if status[i] == 0 else None for i in range(n)]
        out_o = [ols[i].copy() if status[i] == 0 else None for i in range(n)]
        if big.any():
            again = self.partial_paths(ids[big], cap=int(nar.max()) + 64, raise_on_error=False)
            for k, i in enumerate(np.nonzero(big)[0]):
                out_a[i], out_o[i], fr[i] = again["arcs"][k], again["olabels"][k], again["settled_frames"][k]
                status[i] = again["status"][k]
        out = dict(arcs=out_a, olabels=out_o, settled_frames=fr, status=status)
        bad = np.nonzero(status != 0)[0]
        if raise_on_error and bad.size:
            msg = ", ".join(f"stream {int(ids[i])}: {STATUS.get(int(status[i]), int(status[i]))}" for i in bad[:8])
            raise WfstError(int(status[bad[0]]), msg, out)
        return out

    def lattice(self, stream: int, arcs_cap: int = 1 << 20, layers_cap: int = 1 << 14,
                gamma_cap: int = 1 << 22) -> dict:
        """Row f1: the lattice of one stream (wfst_get_lattice): per layer k the segment
        (arc, src, dst, slack, pslack) and gamma per token, token indices in debug_layer order."""
        seg_n = np.zeros(layers_cap, np.int32)
        arc, src, dst = (np.zeros(arcs_cap, np.int32) for _ in range(3))
        sl, ps = np.zeros(arcs_cap, np.float32), np.zeros(arcs_cap, np.float32)
        gam = np.zeros(gamma_cap, np.float32)
        nl, na, nt = np.zeros(1, np.int32), np.zeros(1, np.int64), np.zeros(1, np.int64)
        best, rf = np.zeros(1, np.float32), np.zeros(1, np.int32)
        rc = lib().wfst_get_lattice(self.h, stream, _ptr(seg_n), layers_cap, _ptr(nl), _ptr(arc), _ptr(src), _ptr(dst),
                                    _ptr(sl), _ptr(ps), arcs_cap, _ptr(na), _ptr(gam), gamma_cap, _ptr(nt),
                                    _ptr(best), _ptr(rf))
        if rc == 1 and (na[0] > arcs_cap or nl[0] > layers_cap or nt[0] > gamma_cap):
            return self.lattice(stream, int(na[0]) + 1, int(nl[0]) + 1, int(nt[0]) + 1)
        _check(rc)
        so = np.concatenate([[0], np.cumsum(seg_n[: nl[0]])])
        segs = [(arc[so[k]:so[k + 1]].copy(), src[so[k]:so[k + 1]].copy(), dst[so[k]:so[k + 1]].copy(),
                 sl[so[k]:so[k + 1]].copy()) for k in range(int(nl[0]))]
        psl = [ps[so[k]:so[k + 1]].copy() for k in range(int(nl[0]))]
        return dict(segments=segs, pslack=psl, gamma=gam[: nt[0]].copy(), best=best[0], reached_final=int(rf[0]),
                    n_layers=int(nl[0]))


def synth_loglikes(out, stream_ids, t0: int, seed: int, planted=None, sigma: float = 1.0, boost: float = 0.0,
                   stream=None):
    """Fill a torch.cuda float32 [T][B][P] tensor with the counter-hash log-likelihoods of
    inputs.loglikes (stream_ids / planted: torch.cuda int32 tensors)."""
    T, B, P = out.shape
    _check(lib().wfst_synth_loglikes(C.c_void_p(out.data_ptr()), T, B, P, C.c_void_p(stream_ids.data_ptr()), t0,
                                     C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF),
                                     None if planted is None else C.c_void_p(planted.data_ptr()), float(sigma),
                                     float(boost), _stream_ptr(stream)))


INF = math.inf
