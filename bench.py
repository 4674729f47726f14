#!/usr/bin/env python3
"""bench.py -- RTFx / arcs-per-second of the B200 one-best WFST decoder (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--preset clean]
    python bench.py --impl reference ...      # the CPU oracle on this box's host cores

A step = one pass of the whole hot path over one batch: reset every
stream (start token + epsilon closure), decode all T frames of all B streams (one frame-kernel
launch), final-cost argmin + traceback for every stream (one launch, paths copied to host).
Log-likelihoods are device-resident for `value`; `e2e` repeats the step through the C ABI with
pinned HOST log-likelihoods copied inside the timed region.  Multi-GPU: one process per GPU,
each decoding its own B streams (global ids rank*B + b; weak scaling, no collective on the
data path -- P:328-330).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

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
    """DESIGN.md §6 byte model per stream-frame, summed: 4P (log-likelihood row, read once)
    + 12 per emitting arc (Eq. 1: dst, weight, pdf) + 8 per epsilon arc of a survivor (dst,
    weight) + 36 per survivor (12 B state record (Eq. 1), 8 B traceback record, 8 B frontier
    write + 8 B frontier read next frame)."""
    return int(4 * P * frames + 12 * st["emit_arcs"] + 8 * st["eps_arcs"] + 36 * st["survivors"])


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


def reduce_over_ranks(dist, device, ms: float, arcs: float):
    """Max of the timed region and sum of arcs over ranks (the only collective, off the data path)."""
    import torch
    t = torch.tensor([ms, arcs], dtype=torch.float64, device=device)
    m = t.clone()
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(m[0].item()), float(t[1].item())


# ------------------------------------------------------------------------- workload
def make_workload(cfg: str, preset: str, rank: int = 0, world: int = 1, beam=None, max_active=None):
    c = dict(I.CONFIGS[cfg])
    if beam:
        c["beam"] = beam
    if max_active:
        c["max_active"] = max_active
    g = I.config_graph(cfg)
    B, T, P = c["streams"], c["frames"], c["n_pdfs"]
    stream0 = rank_streams(rank, world, B).start
    planted = I.planted_walks(g, B, T, seed=c["ll_seed"], stream0=stream0)
    return dict(cfg=cfg, c=c, graph=g, B=B, T=T, P=P, stream0=stream0, planted=planted,
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
    for k in ("threads", "ctas_per_sm", "table_slots", "frames_per_item"):
        v = getattr(args, k, 0)
        if v:
            o[k] = v
    if getattr(args, "hist", False):   # row f4: the paper's histogram max-active instead of the exact one
        o["max_active_mode"] = 1
    if getattr(args, "lattice", None) is not None:   # row f1: segments built inside every decode call
        o["lattice"] = 1
        o["lattice_beam"] = args.lattice
    return o


# ------------------------------------------------------------------------- GPU arm
def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_1910_10032_b200 import build, wfst_gpu as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; WFST_DIST_BACKEND=gloo lets a multi-rank run share fewer GPUs (used to
    # exercise the multi-rank path on a one-GPU box -- the only collectives are a barrier and a
    # two-number reduction, never on the data path)
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
    with ClockSampler(local) as clk:
        t0.record()
        for k in range(args.steps):
            res = step(kev[k])
        t1.record()
        torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    st = D.stats()
    if world > 1:
        ms_max, arcs_all = reduce_over_ranks(dist, red_dev, ms, float(st["emit_arcs"] + st["eps_arcs"]))
    else:
        ms_max = ms
        arcs_all = float(st["emit_arcs"] + st["eps_arcs"])
    audio_s = args.steps * B * T * FRAME_S * world
    value = audio_s / (ms_max / 1e3)

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
        for _ in range(e2e_steps):
            r = step_host()
        e1.record()
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        if world > 1:
            ems, _ = reduce_over_ranks(dist, red_dev, ems, 0.0)
        d2h = B * (4 + 4 + 4 + 4 + 4 + 2 * cap * 4)
        e2e = {"value": e2e_steps * B * T * FRAME_S * world / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": T * B * P * 4 * world, "d2h_bytes_per_step": d2h * world,
               "steps": e2e_steps, "ms_per_step": ems / e2e_steps}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    peak, peak_src = _peaks()
    traffic, traffic_src = args.traffic, None
    tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if traffic is None and os.path.exists(tpath) and args.config == "c3" and args.preset == "clean":
        with open(tpath) as f:
            t = json.load(f)
        traffic, traffic_src = t["dram_bytes_per_launch"], "profiles/r01_traffic.json (ncu --set full, same launch)"
    frames_per_step = B * T
    abytes = algorithmic_bytes(st, frames_per_step * args.steps, P) / args.steps
    kmean = statistics.mean(kern_ms)
    achieved = abytes / (kmean / 1e3) / 1e9
    clocks = clk.summary()
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} ({wl['c']['graph'] if isinstance(wl['c']['graph'], str) else 'HCLG-shaped'}"
                               f" {ginfo.n_states} states / {ginfo.n_arcs} arcs, {P} pdfs, {B} streams x {T} frames"
                               f" per GPU, beam {wl['beam']}, max_active {wl['alpha']}, preset {args.preset})",
                   "streams_per_gpu": B, "frames": T, "pdfs": P, "beam": wl["beam"], "max_active": wl["alpha"],
                   "preset": args.preset, "frame_ms": 10, "parallelism": f"streams partitioned over {world} GPU(s)",
                   "l2": "inputs larger than L2 (log-likelihoods %.2f GB per GPU)" % (T * B * P * 4 / 1e9),
                   "frames_per_call": chunk},
        "rtfx_30ms": round(value * 3, 1),
        "arcs_per_s": round(arcs_all * 1e3 / (ms_max), 1) if ms_max else None,
        "frames_per_s": round(args.steps * frames_per_step * world / (ms_max / 1e3), 1),
        "e2e": e2e,
        # per step: reset = settle-point reset + init frame kernel, one frame-kernel launch per
        # chunk (+ one lattice launch each with --lattice, + one on reset), best paths
        "gpu_launches": (3 + (T + chunk - 1) // chunk * (2 if args.lattice is not None else 1)
                         + (2 if args.lattice is not None else 0)) * args.steps,
        "decoder_opts": decoder_opts(args),
        "roofline": {"bound": "hbm", "kernel": "frame_kernel", "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes_per_launch": int(abytes),
                     "kernel_ms": round(kmean, 3), "kernel_share_of_step": round(kmean / (ms_max / args.steps), 3),
                     "peak_source": peak_src},
        "counters_per_step": {k: v / args.steps for k, v in st.items()
                              if k not in ("device_bytes", "records_used_max", "phase_cycles")},
        "phase_share": {k: round(v / max(1, sum(st["phase_cycles"].values())), 4) for k, v in st["phase_cycles"].items()},
        "memory": {"graph_device_bytes": ginfo.device_bytes, "graph_eq1_bytes": ginfo.eq1_bytes,
                   "decoder_device_bytes": st["device_bytes"],
                   "eq2_bytes_nc=nl=B": W.eq2_bytes(wl["alpha"], B, B)},
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
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
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
    ap.add_argument("--beam", type=float, default=None, help="override the config's beam (experiments)")
    ap.add_argument("--max-active", dest="max_active", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    main()
