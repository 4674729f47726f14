"""Instruction / stall-sample shares of an ncu report grouped by source-line ranges of
frame_kernel.cuh (ranges = the functions, read from the source file)."""
import csv, re, subprocess, sys

def main(rep, src="paper_1910_10032_b200/csrc/frame_kernel.cuh"):
    lines = open(src).read().splitlines()
    starts = []
    for i, l in enumerate(lines, 1):
        m = re.match(r"\s*(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\(", l)
        if m:
            starts.append((i, m.group(1)))
    def fn(n):
        name = "?"
        for s, nm in starts:
            if s <= n: name = nm
        return name
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, ix, acc = None, None, {}
    for r in csv.reader(txt.splitlines()):
        if not r: continue
        if r[0] in ("File Path", "File Name"): cur = r[1].split("/")[-1]; continue
        if r[0] == "Line No": ix = {h: i for i, h in reversed(list(enumerate(r)))}; continue
        if not r[0].isdigit() or ix is None: continue
        key = fn(int(r[0])) if cur == "frame_kernel.cuh" else cur
        try: v = float(r[ix["Instructions Executed"]]); s = float(r[ix["Warp Stall Sampling (All Samples)"]])
        except ValueError: continue
        a = acc.get(key, [0, 0]); a[0] += v; a[1] += s; acc[key] = a
    tv = sum(a[0] for a in acc.values()); ts = sum(a[1] for a in acc.values())
    print(f"total warp inst {tv:.3e}  samples {ts:.0f}")
    for k, (v, s) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        if v / tv > 0.003 or s / ts > 0.003:
            print(f"{k:22s} inst {100*v/tv:5.1f}%  samp {100*s/ts:5.1f}%")

if __name__ == "__main__":
    main(*sys.argv[1:])
