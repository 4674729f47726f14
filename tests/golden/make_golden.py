"""Writes tests/golden/loglikes_head.json from the input generator only (no oracle, no GPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1910_10032_b200 import inputs as I  # noqa: E402

out = []
for (seed, stream, T, P, sigma, boost) in [(1, 0, 3, 8, 1.0, 0.0), (30003, 511, 2, 6, 1.0, 4.0), (7, 12345, 2, 5, 1.5, 2.0)]:
    planted = [t % P for t in range(T)]
    ll = I.loglikes_stream(seed, stream, T, P, planted, sigma, boost)
    out.append(dict(seed=seed, stream=stream, T=T, P=P, sigma=sigma, boost=boost, planted=planted,
                    bits=[int(x) for x in ll.view("uint32").ravel()]))
with open(os.path.join(os.path.dirname(__file__), "loglikes_head.json"), "w") as f:
    json.dump(out, f, indent=1)
