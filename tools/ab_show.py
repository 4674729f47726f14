import json, sys
for t in sys.argv[1:]:
    try:
        d = json.load(open(f"gpurun_out/abm_{t}.json"))
    except Exception as e:
        print(t, "failed", e); continue
    c = d["counters_per_step"]
    print(f"{t:10s} {d['value']:9.1f} RTFx {d['ms_per_step']:8.2f} ms  ovf/frame {c['overflow_inserts']/c['frames']:7.1f}  cand/frame {c['candidates']/c['frames']:7.1f}")
    ph = d["phase_share"]; print("   ", {k: v for k, v in sorted(ph.items(), key=lambda kv: -kv[1]) if v > 0.01})
