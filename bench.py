#!/usr/bin/env python3
"""bench.py -- RTFx / arcs-per-second of the B200 one-best WFST decoder (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--preset clean]
    python bench.py --impl reference ...      # the CPU oracle on this box's host cores

A step = one pass of the whole hot path over one batch: reset every
stream (start token + epsilon closure), decode all T frames of all B streams (one frame-kernel
launch), final-cost argmin + traceback for every stream (one launch, paths copied to host).
Log-likelihoods are device-resident for `value`; `e2e` repeats the step through the C ABI with
pinned HOST log-likelihoods copied inside the timed region.  Prints ONE JSON line on rank 0.

Multi-GPU (row e): one process per GPU, streams partitioned over the ranks, each rank
with its own graph replica and decoder, no collective on the data path.  `--gpus N` launches
the N ranks itself (torch.distributed.run) unless it already runs under a launcher (WORLD_SIZE
set).  C3 (the headline) is weak-scaled (512 streams per GPU, global ids rank*512 + b); C5 is
strong-scaled (4096 streams in total, contiguous blocks of 4096/N per rank).  After the timed
region rank 0 gathers every global stream's result (host-side gather, the only data that moves
between ranks) and re-decodes a sample of the other ranks' streams on its own GPU: the results
must be identical (partition independence).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1910_10032_b200 import inputs as I  # noqa: E402

FRAME_S = 0.010          # 10 ms per frame (S:555 convention); 30 ms reported alongside
METRIC = "RTFx"
UNIT = "audio-seconds decoded per second (10 ms frames)"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def algorithmic_bytes(st: dict, frames: int, P: int) -> int:
    """SURVEY §8.5 byte model (what the method itself must move), summed over stream-frames:
      16 n_src      frontier read (state + cost + 8 B of CSR row offsets)
    + 12 n_arc_e    emitting arcs (Eq. 1: dst, weight, pdf)
    + 4 P           the frame's log-likelihood row, read once
    + 8 n_cand      u64 dedup update per distinct candidate
    + 16 n_surv     frontier write 8 B + traceback record 8 B
    + 16 n_arc_eps  epsilon arc read + update (epsilon out-degree of the kept tokens)
    + 4 n_select    max-active selection: entries x passes, only when alpha binds
    n_src and n_surv are both the survivor count (every survivor is written once and expanded
    once in the next frame; the last layer of a step is written but not expanded -- 1/T of the
    term)."""
    return int(16 * st["survivors"] + 12 * st["emit_arcs"] + 4 * P * frames + 8 * st["candidates"]
               + 16 * st["survivors"] + 16 * st["eps_arcs"] + 4 * st.get("select_entries", 0))


def kernel_source_sha() -> str:
    """Hash of the CUDA sources: an ncu traffic capture is valid only for the build it measured."""
    d = os.path.join(ROOT, "paper_1910_10032_b200", "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def measured_traffic(cfg: str, preset: str):
    """DRAM bytes per decode launch from a committed `ncu --set full` capture of THIS build
    (profiles/*_traffic.json, tagged with kernel_source_sha); None when no capture matches."""
    sha = kernel_source_sha()
    d = os.path.join(ROOT, "profiles")
    for f in sorted(os.listdir(d), reverse=True):
        if not f.endswith("_traffic.json"):
            continue
        with open(os.path.join(d, f)) as fh:
            t = json.load(fh)
        if t.get("kernel_src_sha") == sha and t.get("config") == f"{cfg}/{preset}":
            return float(t["dram_bytes_per_launch"]), f"profiles/{f} (ncu --set full of this build, sha {sha})"
    return None, f"no ncu capture of this build (kernel sources sha {sha}) in profiles/"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) != len(self.FIELDS):
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------- multi-GPU host logic
def rank_streams(rank: int, world: int, per_rank: int) -> range:
    """Global stream ids of a rank (weak scaling: every rank decodes its own per_rank streams;
    inputs are keyed by global id, so a stream's result does not depend on the split)."""
    assert 0 <= rank < world
    return range(rank * per_rank, (rank + 1) * per_rank)


def partition(total: int, world: int, rank: int) -> range:
    """Strong scaling: `total` global streams split into `world` contiguous near-equal blocks."""
    assert 0 <= rank < world and total >= world
    q, r = divmod(total, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def config_streams(c: dict, rank: int, world: int) -> range:
    return partition(c["streams"], world, rank) if c.get("scaling") == "strong" else rank_streams(rank, world, c["streams"])


def launcher_cmd(argv: list, n: int, port: int) -> list:
    """`bench.py --gpus N` outside a launcher: one process per GPU via torch.distributed.run."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def result_digest(res: dict, i: int) -> tuple:
    """(cost bits, reached_final, n_arcs, crc32 of the arc ids) of row i of a best_paths result."""
    n = int(res["n_arcs"][i])
    return (int(np.asarray(res["cost"][i], np.float32).view(np.uint32)), int(res["reached_final"][i]), n,
            zlib.crc32(np.ascontiguousarray(res["arcs"][i, :n], np.int32).tobytes()))


def gather_results(dist, world: int, ids, digests: list):
    """Host-side gather of every rank's per-stream results to rank 0 (the only exchange of the
    multi-GPU path, after the timed region).  Returns {global stream id: digest} on rank 0
    (None elsewhere); asserts the partition covered every stream exactly once."""
    local = (list(ids), list(digests))
    if world == 1:
        parts = [local]
    else:
        parts = [None] * world
        dist.all_gather_object(parts, local)
        if dist.get_rank() != 0:
            return None
    out = {}
    for sid, dg in parts:
        for s_, d_ in zip(sid, dg):
            assert s_ not in out, f"stream {s_} decoded by two ranks"
            out[s_] = d_
    return out


def distinct_devices(dist, world: int, local: int) -> int:
    """GPUs actually used: distinct (host, device uuid) over the ranks (ranks sharing a device
    under WFST_DIST_BACKEND=gloo count once)."""
    import torch
    me = (socket.gethostname(), str(torch.cuda.get_device_properties(local).uuid))
    if world == 1:
        return 1
    allv = [None] * world
    dist.all_gather_object(allv, me)
    return len(set(allv))


def reduce_over_ranks(dist, device, ms: float, arcs: float):
    """Max of the timed region and sum of arcs over ranks (the only collective, off the data path)."""
    import torch
    t = torch.tensor([ms, arcs], dtype=torch.float64, device=device)
    m = t.clone()
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(m[0].item()), float(t[1].item())


# ------------------------------------------------------------------------- workload
def make_workload(cfg: str, preset: str, rank: int = 0, world: int = 1, beam=None, max_active=None, graph=None,
                  ids=None):
    c = dict(I.CONFIGS[cfg])
    if beam:
        c["beam"] = beam
    if max_active:
        c["max_active"] = max_active
    g = graph if graph is not None else I.config_graph(cfg)
    ids = ids if ids is not None else config_streams(c, rank, world)
    B, T, P = len(ids), c["frames"], c["n_pdfs"]
    stream0 = ids.start
    planted = I.planted_walks(g, B, T, seed=c["ll_seed"], stream0=stream0)
    return dict(cfg=cfg, c=c, graph=g, B=B, T=T, P=P, stream0=stream0, ids=ids, planted=planted,
                preset=I.preset(preset), preset_name=preset, beam=c["beam"], alpha=c["max_active"])


def device_loglikes(W, torch, wl, device):
    T, B, P = wl["T"], wl["B"], wl["P"]
    ll = torch.empty((T, B, P), dtype=torch.float32, device=device)
    ids = torch.arange(wl["stream0"], wl["stream0"] + B, dtype=torch.int32, device=device)
    pl = torch.from_numpy(np.ascontiguousarray(wl["planted"])).to(device)
    W.synth_loglikes(ll, ids, 0, wl["c"]["ll_seed"], pl, **wl["preset"])
    torch.cuda.synchronize(device)
    return ll


def run_gpu_once(cfg="c3", preset="clean", with_paths=True):
    """One full step (used by the full-size parity test)."""
    import torch
    from paper_1910_10032_b200 import build, wfst_gpu as W
    build.build()
    wl = make_workload(cfg, preset)
    G = W.Graph.from_arrays(wl["graph"])
    D = W.Decoder(G, wl["B"], wl["beam"], wl["alpha"])
    ll = device_loglikes(W, torch, wl, "cuda:0")
    D.reset()
    D.decode_frames(ll)
    res = D.best_paths(cap=4 * wl["T"] + 64)
    return res, wl


def decoder_opts(args) -> dict:
    o = {}
    for k in ("threads", "ctas_per_sm", "table_slots", "frames_per_item", "insert_order", "bin_capacity",
              "records_per_stream", "max_frames", "gc_frames"):
        v = getattr(args, k, 0)
        if v:
            o[k] = v
    if getattr(args, "hist", False):   # row f4: the paper's histogram max-active instead of the exact one
        o["max_active_mode"] = 1
    if getattr(args, "reclaim", False):   # row f2 traceback GC: records below the settle point are reused
        o["reclaim"] = 1
    if getattr(args, "lattice", None) is not None:   # row f1: segments built inside every decode call
        o["lattice"] = 1
        o["lattice_beam"] = args.lattice
    return o


# ------------------------------------------------------------------------- GPU arm
def cross_check(W, torch, wl_cfg, preset, graph, G, gathered: dict, world: int, dev, args, per_rank: int = 4):
    """Rank 0 re-decodes the first `per_rank` streams of every OTHER rank's block on its own GPU
    (global ids, inputs regenerated from them) and compares with the gathered results: a stream's
    result must not depend on which GPU decoded it or how the streams were split."""
    c = I.CONFIGS[wl_cfg]
    ids = []
    for r in range(1, world):
        blk = config_streams(c, r, world)
        ids.append(range(blk.start, blk.start + min(per_rank, len(blk))))
    n_checked = n_bad = 0
    for blk in ids:
        wl = make_workload(wl_cfg, preset, beam=args.beam, max_active=args.max_active, graph=graph, ids=blk)
        D = W.Decoder(G, wl["B"], wl["beam"], wl["alpha"], **decoder_opts(args))
        ll = device_loglikes(W, torch, wl, dev)
        chunk = wl["c"].get("chunk") or wl["T"]
        D.reset()
        for t0 in range(0, wl["T"], chunk):
            D.decode_frames(ll[t0:t0 + chunk].contiguous() if chunk < wl["T"] else ll)
        res = D.best_paths(cap=4 * wl["T"] + 64, raise_on_error=False)
        for i, sid in enumerate(blk):
            n_checked += 1
            n_bad += int(result_digest(res, i) != gathered[sid])
        del D, ll
    return n_checked, n_bad


def launcher_selftest(args):
    """`--launcher-selftest` (CPU, WFST_DIST_BACKEND=gloo; tests/test_bench_host.py): the multi-rank
    plumbing of the GPU arm without a GPU -- this process was started by bench's own launcher,
    takes its share of the config's streams (config_streams), stands in for decoding with a digest
    of each stream's synthetic inputs (keyed by global id, inputs.loglikes_stream), and goes
    through the same max-over-ranks reduction and rank-0 result gather as a GPU run.  Rank 0
    checks that every global stream arrived exactly once with the digest a single process
    computes, and prints one JSON line."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    c = dict(I.CONFIGS[args.config])
    ids = config_streams(c, rank, world)

    def digest(sid):
        row = I.loglikes_stream(c["ll_seed"], sid, 2, 64, None, 1.0, 0.0)
        return (sid, zlib.crc32(row.tobytes()))

    gathered = gather_results(dist, world, ids, [digest(s) for s in ids])
    ms, units = reduce_over_ranks(dist, "cpu", 1.0 + rank, float(len(ids))) if world > 1 else (1.0, float(len(ids)))
    if rank == 0:
        total = c["streams"] * (world if c.get("scaling") != "strong" else 1)
        ok = (sorted(gathered) == list(range(total)) and all(gathered[s] == digest(s) for s in gathered)
              and units == total and ms == float(world))
        print(json.dumps({"selftest": "launcher", "config": args.config, "world": world, "streams": len(gathered),
                          "expected_streams": total, "scaling": c.get("scaling", "weak"), "ok": bool(ok)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_1910_10032_b200 import build, wfst_gpu as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; WFST_DIST_BACKEND=gloo lets a multi-rank run share fewer GPUs (used to
    # exercise the multi-rank path on a one-GPU box -- the only collectives are a barrier, a
    # two-number reduction and the final result gather, never on the data path)
    backend = os.environ.get("WFST_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()

    wl = make_workload(args.config, args.preset, rank, world, args.beam, args.max_active)
    T, B, P = wl["T"], wl["B"], wl["P"]
    strong = wl["c"].get("scaling") == "strong"
    G = W.Graph.from_arrays(wl["graph"], device=local)
    ginfo = G.info()
    D = W.Decoder(G, B, wl["beam"], wl["alpha"], **decoder_opts(args))
    ll = device_loglikes(W, torch, wl, dev)
    cap = 4 * T + 64

    chunk = wl["c"].get("chunk") or T   # online configs (C4/C5) arrive in frame chunks

    def step(ev=None):
        D.reset()
        if ev is not None:
            ev[0].record()
        for t0 in range(0, T, chunk):
            D.decode_frames(ll[t0:t0 + chunk] if chunk < T else ll)
            if args.partial:   # row f2: settled partial results of every stream after each chunk
                D.partial_paths()
        if ev is not None:
            ev[1].record()
        return D.best_paths(cap=cap, raise_on_error=False)

    for _ in range(args.warmup):
        res = step()
        assert res["rc"] == 0, W.STATUS.get(res["rc"])
    D.reset_stats()
    torch.cuda.synchronize(dev)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    rcs = []
    with ClockSampler(local) as clk:
        t0.record()
        for k in range(args.steps):
            res = step(kev[k])
            rcs.append(int(res["rc"]))
        t1.record()
        torch.cuda.synchronize(dev)
    # a lane that hit CAPACITY stops decoding and would make a step look faster: every timed
    # step must have decoded every stream
    assert all(r == 0 for r in rcs), f"timed steps with errors: {[W.STATUS.get(r, r) for r in rcs]}"
    ms = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    st = D.stats()
    if world > 1:
        ms_max, arcs_all = reduce_over_ranks(dist, red_dev, ms, float(st["emit_arcs"] + st["eps_arcs"]))
    else:
        ms_max = ms
        arcs_all = float(st["emit_arcs"] + st["eps_arcs"])
    total_streams = wl["c"]["streams"] if strong else B * world
    audio_s = args.steps * total_streams * T * FRAME_S
    value = audio_s / (ms_max / 1e3)

    # ---- host-side gather of every global stream's result (after the timed region) + a
    # partition-independence check on rank 0
    digests = [result_digest(res, i) for i in range(B)]
    gathered = gather_results(dist, world, wl["ids"], digests)
    n_dev = distinct_devices(dist, world, local)
    gather = None
    if rank == 0:
        assert sorted(gathered) == list(range(total_streams)), "streams missing from the gather"
        # (with --reclaim the timed steps' paths are the tails after the settled prefixes: the
        # re-decode, which fetches no partial results, is compared only without --partial)
        n_chk, n_bad = cross_check(W, torch, args.config, args.preset, wl["graph"], G, gathered, world, dev, args) \
            if world > 1 and not args.partial else (0, 0)
        assert n_bad == 0, f"{n_bad} of {n_chk} streams decoded differently on rank 0"
        gather = {"streams": len(gathered), "rechecked_on_rank0": n_chk, "mismatches": n_bad,
                  "digest": "%08x" % zlib.crc32(json.dumps([gathered[k] for k in sorted(gathered)]).encode())}

    # ---- e2e: host log-likelihoods through the C ABI, H2D inside the timed region
    e2e = None
    if not args.no_e2e:
        host = torch.empty((T, B, P), dtype=torch.float32, pin_memory=True)
        host.copy_(ll)
        del ll
        torch.cuda.empty_cache()
        e2e_steps = max(1, min(args.steps, 3))

        def step_host():
            D.reset()
            D.decode_frames_host(host, chunk_frames=args.chunk)
            return D.best_paths(cap=cap, raise_on_error=False)

        r = step_host()
        assert r["rc"] == 0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e_rcs = []
        for _ in range(e2e_steps):
            r = step_host()
            e_rcs.append(int(r["rc"]))
        e1.record()
        torch.cuda.synchronize(dev)
        assert all(x == 0 for x in e_rcs)
        ems = e0.elapsed_time(e1)
        if world > 1:
            ems, _ = reduce_over_ranks(dist, red_dev, ems, 0.0)
        d2h = B * (4 + 4 + 4 + 4 + 4 + 2 * cap * 4)
        e2e = {"value": e2e_steps * total_streams * T * FRAME_S / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": T * total_streams * P * 4, "d2h_bytes_per_step": d2h * world,
               "steps": e2e_steps, "ms_per_step": ems / e2e_steps}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    peak, peak_src = _peaks()
    if args.traffic is not None:
        traffic, traffic_src = args.traffic, "--traffic"
    else:
        traffic, traffic_src = measured_traffic(args.config, args.preset)
    frames_per_step = B * T
    abytes = algorithmic_bytes(st, frames_per_step * args.steps, P) / args.steps
    kmean = statistics.mean(kern_ms)
    achieved = abytes / (kmean / 1e3) / 1e9
    clocks = clk.summary()
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": n_dev, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} ({wl['c'].get('graph_kind', 'HCLG-shaped') if not isinstance(wl['c']['graph'], str) else wl['c']['graph']}"
                               f" {ginfo.n_states} states / {ginfo.n_arcs} arcs, {P} pdfs, "
                               + (f"{total_streams} streams split over {world} rank(s)" if strong else f"{B} streams per GPU")
                               + f" x {T} frames, beam {wl['beam']}, max_active {wl['alpha']}, preset {args.preset})",
                   "streams_per_gpu": B, "streams_total": total_streams, "frames": T, "pdfs": P, "beam": wl["beam"],
                   "max_active": wl["alpha"], "preset": args.preset, "frame_ms": 10,
                   "parallelism": f"streams partitioned over {world} rank(s) on {n_dev} GPU(s)",
                   "l2": "inputs larger than L2 (log-likelihoods %.2f GB per GPU)" % (T * B * P * 4 / 1e9),
                   "frames_per_call": chunk},
        "rtfx_30ms": round(value * 3, 1),
        "arcs_per_s": round(arcs_all * 1e3 / (ms_max), 1) if ms_max else None,
        "frames_per_s": round(args.steps * total_streams * T / (ms_max / 1e3), 1),
        "e2e": e2e,
        # per step: reset = settle-point reset + init frame kernel, one frame-kernel launch per
        # chunk (+ one lattice launch each with --lattice, + one on reset), best paths
        "gpu_launches": (3 + (T + chunk - 1) // chunk * ((2 if args.lattice is not None else 1) + (1 if args.partial else 0))
                         + (2 if args.lattice is not None else 0)) * args.steps,
        "decoder_opts": decoder_opts(args),
        "roofline": {"bound": "hbm", "kernel": "frame_kernel", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes_per_launch": int(abytes),
                     "byte_model": "SURVEY §8.5: 16 n_src + 12 n_arc_e + 4 P + 8 n_cand + 16 n_surv + 16 n_arc_eps"
                                   " + 4 n_select per stream-frame (bench.algorithmic_bytes)",
                     "kernel_ms": round(kmean, 3), "kernel_share_of_step": round(kmean / (ms_max / args.steps), 3),
                     "peak_source": peak_src},
        "counters_per_step": {k: v / args.steps for k, v in st.items()
                              if k not in ("device_bytes", "records_used_max", "phase_cycles", "phase_cycles_alpha",
                                           "records_per_stream", "record_bytes")},
        # per-phase SM cycles (clock64 marks of thread 0; -DWFST_PHASES=0 builds have none)
        "phase_share": {k: round(v / max(1, sum(st["phase_cycles"].values())), 4) for k, v in st["phase_cycles"].items()}
        if sum(st["phase_cycles"].values()) else None,
        # the same cycles restricted to frames where max-active bound, as a share of ALL cycles
        "phase_share_alpha_frames": {k: round(v / max(1, sum(st["phase_cycles"].values())), 4)
                                     for k, v in st["phase_cycles_alpha"].items()}
        if sum(st["phase_cycles"].values()) else None,
        "memory": {"graph_device_bytes": ginfo.device_bytes, "graph_eq1_bytes": ginfo.eq1_bytes,
                   "decoder_device_bytes": st["device_bytes"],
                   "record_arena_bytes": st["record_bytes"],
                   "decoder_state_bytes": st["device_bytes"] - st["record_bytes"],
                   "records_per_stream": st["records_per_stream"],
                   "records_used_max_per_stream": st["records_used_max"],
                   "records_written_per_step_bytes": int(8 * st["survivors"] / max(1, args.steps)),
                   "eq2_bytes_nc=nl=B": W.eq2_bytes(wl["alpha"], B, B)},
        "gather": gather,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, args)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return out


# ------------------------------------------------------------------------- oracle timing
def _sample_loglikes(wl, n_streams):
    c = wl["c"]
    return np.ascontiguousarray(I.loglikes(c["ll_seed"], range(wl["stream0"], wl["stream0"] + n_streams),
                                           wl["T"], wl["P"], wl["planted"][:, :n_streams], **wl["preset"]))


def _oracle_time(wl, n_streams, cores):
    import oracle
    og = oracle.OracleGraph(wl["graph"])
    ll = _sample_loglikes(wl, n_streams)
    t = time.perf_counter()
    cost, reached, rc, cnt, _, _ = og.decode_batch(ll, wl["beam"], wl["alpha"], cores)
    dt = time.perf_counter() - t
    return dt, int(cnt.sum()), rc


def cpu_baseline(wl, args):
    """The oracle as it stands, on this box's host cores, on a bounded sample of the workload."""
    cores = os.cpu_count() or 1
    n = min(wl["B"], max(16, cores))
    dt, arcs, rc = _oracle_time(wl, n, cores)
    audio = n * wl["T"] * FRAME_S
    dt1, _, _ = _oracle_time(wl, 2, 1)   # the single-core rate, 2 streams
    return {"value": round(audio / dt, 2), "unit": UNIT, "cores": min(cores, n), "kind": "oracle",
            "sample": f"{n} of {wl['B']} streams x {wl['T']} frames of {args.config}/{args.preset} "
                      f"(oracle/wfst_oracle.c, pthreads), {dt:.2f} s wall",
            "arcs_per_s": round(arcs / dt, 1), "errors": int((rc != 0).sum()),
            "single_core": {"value": round(2 * wl["T"] * FRAME_S / dt1, 2), "sample": "2 streams, 1 thread"}}


def reference_arm(args):
    """--impl reference: the CPU oracle is this tier's reference implementation."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    wl = make_workload(args.config, args.preset, 0)
    cores = os.cpu_count() or 1
    n = min(wl["B"], max(8, cores))
    for _ in range(args.warmup):
        _oracle_time(wl, min(n, cores), cores)
    times, arcs = [], 0
    for _ in range(args.steps):
        dt, a, rc = _oracle_time(wl, n, cores)
        times.append(dt)
        arcs += a
    tot = sum(times)
    value = args.steps * n * wl["T"] * FRAME_S / tot
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": 0,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 1),
           "higher_is_better": True, "scaling": "strong" if wl["c"].get("scaling") == "strong" else "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"{args.config} ({n} of {wl['B']} streams per step)", "preset": args.preset,
                      "frames": wl["T"], "beam": wl["beam"], "max_active": wl["alpha"]},
           "arcs_per_s": round(arcs / tot, 1),
           "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": min(cores, n), "kind": "oracle",
                            "sample": f"{n} streams x {wl['T']} frames per step"},
           "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(I.CONFIGS))
    ap.add_argument("--preset", default="clean", choices=sorted(I.PRESETS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk", type=int, default=25, help="frames per H2D chunk in the e2e leg")
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch (from profiles/)")
    ap.add_argument("--threads", type=int, default=0, help="frame-kernel CTA size (default by variant)")
    ap.add_argument("--hist", action="store_true",
                    help="histogram max-active (row f4; approximate, not the headline)")
    ap.add_argument("--partial", action="store_true",
                    help="fetch settled partial results after every chunk (row f2; not the headline)")
    ap.add_argument("--lattice", type=float, default=None,
                    help="also build lattice segments with this lattice-beam (row f1; not the headline)")
    ap.add_argument("--ctas-per-sm", dest="ctas_per_sm", type=int, default=0)
    ap.add_argument("--table-slots", dest="table_slots", type=int, default=0)
    ap.add_argument("--frames-per-item", dest="frames_per_item", type=int, default=0)
    ap.add_argument("--insert-order", dest="insert_order", type=int, default=0,
                    help="0 auto (bin order after alpha-bound frames), 1 arrival order, 2 always bin order")
    ap.add_argument("--bin-capacity", dest="bin_capacity", type=int, default=0)
    ap.add_argument("--reclaim", action="store_true",
                    help="traceback GC (row f2): with --partial, records below each stream's settle point are reused")
    ap.add_argument("--records-per-stream", dest="records_per_stream", type=int, default=0)
    ap.add_argument("--max-frames", dest="max_frames", type=int, default=0)
    ap.add_argument("--gc-frames", dest="gc_frames", type=int, default=0,
                    help="traceback GC every N frames (opts.gc_frames): records of dead branches are dropped")
    ap.add_argument("--beam", type=float, default=None, help="override the config's beam (experiments)")
    ap.add_argument("--max-active", dest="max_active", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--launcher-selftest", dest="launcher_selftest", action="store_true",
                    help="CPU check of the multi-rank launcher, partition and gather (no GPU; tests)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.reclaim and not args.partial:
        ap.error("--reclaim needs --partial (records are released by the settled partial results)")
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch the ranks ourselves (the driver's torchrun sets WORLD_SIZE)
        import torch
        n_dev = torch.cuda.device_count()
        if args.launcher_selftest:
            os.environ["WFST_DIST_BACKEND"] = "gloo"   # inherited by the launched ranks
        if args.gpus > n_dev and os.environ.get("WFST_DIST_BACKEND", "nccl") == "nccl":
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {n_dev} CUDA device(s) visible\n")
            sys.exit(2)
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        argv = sys.argv[1:] if argv is None else list(argv)
        sys.exit(subprocess.call(launcher_cmd(argv, args.gpus, port)))
    if args.launcher_selftest:
        return launcher_selftest(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and int(os.environ.get("RANK", "0")) == 0:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} under a launcher of {world} rank(s): using {world}\n")
    return gpu_arm(args)


if __name__ == "__main__":
    main()
