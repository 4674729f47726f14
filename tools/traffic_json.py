"""Write profiles/<name>_traffic.json from an `ncu --set full` capture of the decode frame_kernel
(run here, no GPU): DRAM bytes per launch, tagged with the kernel-source sha the capture measured
(gpurun_out/prof_<tag>.sha, written on the box by tools/ncu_capture.sh).
Usage: python tools/traffic_json.py <tag> <config/preset> <out name>"""
import csv
import io
import json
import subprocess
import sys

tag, cfg, name = sys.argv[1], sys.argv[2], sys.argv[3]
rep = f"gpurun_out/prof_{tag}.ncu-rep"
sha = open(f"gpurun_out/prof_{tag}.sha").read().strip()
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, vals = rows[0], rows[1], rows[2]
d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale[u["dram__bytes_read.sum"]]
wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale[u["dram__bytes_write.sum"]]
out = {"kernel": d.get("Kernel Name", "frame_kernel")[:80], "config": cfg, "kernel_src_sha": sha,
       "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
       "source": f"ncu --set full --clock-control none ({rep}; dram__bytes_read.sum + dram__bytes_write.sum)"}
json.dump(out, open(f"profiles/{name}_traffic.json", "w"), indent=1)
print(out)
