"""Per-source-line instruction and stall-sample shares from an ncu report (run here, no GPU)."""
import csv
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(rep, n=45):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, ix, acc, text = None, None, {}, {}
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            ix = {}
            for i, h in enumerate(r):
                ix.setdefault(h, i)
            continue
        if not r[0] or not r[0].isdigit() or ix is None:
            continue
        k = (cur_file, int(r[0]))
        v = num(r[ix["Instructions Executed"]])
        s = num(r[ix["Warp Stall Sampling (All Samples)"]])
        a = acc.get(k, (0.0, 0.0))
        acc[k] = (a[0] + v, a[1] + s)
        text[k] = r[1]
    tot = sum(v for v, _ in acc.values()) or 1
    tots = sum(s for _, s in acc.values()) or 1
    print(f"total warp instructions {tot:.3e}, stall samples {tots:.0f}")
    for k, (v, s) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:n]:
        print(f"{k[0][:16]:16s} L{k[1]:4d} inst {v / tot * 100:5.2f}% samp {s / tots * 100:5.2f}%  {text[k][:84]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
