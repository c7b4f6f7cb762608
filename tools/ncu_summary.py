"""Write a text summary of one ncu --set full capture of k_fit (metrics,
stall reasons, samples by k_fit call site) -- used for profiles/.
usage: ncu_summary.py <rep.ncu-rep> <lib.so> <mangled kernel> <title> <out.txt> [steps]"""
import csv
import io
import subprocess
import sys

rep, lib, kern, title, out = sys.argv[1:6]
steps = int(sys.argv[6]) if len(sys.argv) > 6 else 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None


src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
open("/tmp/_src.csv", "w").write(src)
lines = [title]
dur = f("gpu__time_duration.sum")
lines.append(f"duration {dur:.3f} ms for {steps} steps = {dur / steps * 1000:.1f} us/step (under ncu)")
rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
lines.append(f"dram read {rd:.2f} MB, write {wr:.2f} MB -> {(rd + wr) / steps:.3f} MB/step")
for k in ["sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__shared_mem_per_block_dynamic", "launch__grid_size"]:
    if k in d:
        lines.append(f"{k} = {d[k]}")
keys = [k for k in r[0] if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("_not_issued")]
tot = sum(f(k) or 0 for k in keys) or 1
lines.append("\nwarp stall reasons (share of samples):")
for k in sorted(keys, key=lambda k: -(f(k) or 0))[:10]:
    lines.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {(f(k) or 0) / tot * 100:5.1f}%")
att = subprocess.run([sys.executable, "tools/sass_lines.py", lib, kern, "/tmp/_src.csv", "30", "--file",
                      "gmf_grad.cu"], capture_output=True, text=True)
lines.append("\nsamples by k_fit call site (tools/sass_lines.py, same build):")
lines.append(att.stdout + att.stderr)
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
