"""Write profiles/<name>_ncu_frame_kernel_{full,stalls}.md, _lines.txt, _groups.txt and
<name>_launches.md from the captures of tools/ncu_capture.sh <tag> (run here, no GPU).
Usage: python tools/ncu_final_md.py <tag> <name> "<title>" """
import csv
import io
import subprocess
import sys

sys.path.insert(0, "tools")
import ncu_summary  # noqa: E402

tag, name, title = sys.argv[1], sys.argv[2], sys.argv[3]
rep = f"gpurun_out/prof_{tag}.ncu-rep"
sha = open(f"gpurun_out/prof_{tag}.sha").read().strip()
with open(f"profiles/{name}_ncu_frame_kernel_full.md", "w") as f:
    f.write(f"# frame_kernel<1024,2,1,0>, ncu --set full --clock-control none ({title}, kernel sources sha {sha}; "
            "C3 clean, one decode launch = 512 streams x 500 frames)\n\n")
    f.write(ncu_summary.raw(rep) + "\n")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
d = dict(zip(rows[0], rows[2]))
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "")) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
tot = sum(st.values()) or 1.0
with open(f"profiles/{name}_ncu_frame_kernel_stalls.md", "w") as f:
    f.write(f"| stall reason (frame_kernel, pc sampling, {title}) | share |\n|---|---|\n")
    for k, v in sorted(st.items(), key=lambda kv: -kv[1]):
        if v / tot >= 0.001:
            f.write(f"| {k} | {100 * v / tot:.1f}% |\n")
    f.write("\n| other | value |\n|---|---|\n")
    for m in ["sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smsp__inst_executed_op_shared_atom.sum",
              "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum"]:
        if m in d:
            f.write(f"| {m} | {d[m]} |\n")
for tool, suffix in (("ncu_lines.py", "lines.txt"), ("ncu_groups.py", "groups.txt")):
    out = subprocess.run([sys.executable, f"tools/{tool}", rep], capture_output=True, text=True).stdout
    open(f"profiles/{name}_ncu_frame_kernel_{suffix}", "w").write(out)
with open(f"profiles/{name}_launches.md", "w") as f:
    f.write(f"# launch list, 2-step bench run (ncu --metrics gpu__time_duration.sum --clock-control none; "
            f"cold-cache, serialised), {title}, sha {sha}\n\n")
    f.write(ncu_summary.launches(f"gpurun_out/launches_{tag}.csv") + "\n")
print("ok", sha)
