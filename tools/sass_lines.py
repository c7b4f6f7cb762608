"""Attribute ncu per-instruction samples to source lines.

  python tools/sass_lines.py <lib.so> <mangled kernel> <ncu source-page csv> [N] [--file gmf_tc.cuh]

The csv is `ncu -i rep --page source --csv` (SASS view, one row per
instruction, in address order); the library must be the exact build that was
profiled (compiled with -lineinfo).  Instructions are matched by position with
`nvdisasm -gi` of the kernel's section; each is attributed to the innermost
source location and, with --file, to the deepest location of its inline chain
inside that file (the call site in the kernel body rather than the helper).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def sass_locations(lib, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
                   capture_output=True)
    for cub in sorted(os.listdir(tmp)):
        out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)],
                             capture_output=True, text=True).stdout
        tag = f".text.{kernel}:"
        if tag not in out:
            continue
        body = out.split(tag, 1)[1]
        body = body.split("\t.section", 1)[0]
        locs, pending, cur = [], [], []
        for line in body.splitlines():
            st = line.strip()
            if st.startswith("//## File"):
                pending.append(re.findall(r'"([^"]+)", line (\d+)', st))
            elif re.match(r"/\*[0-9a-f]{4,}\*/", st):
                if pending:
                    cur = pending[0]
                    pending = []
                locs.append(cur)
        return locs
    raise SystemExit(f"kernel {kernel} not found in {lib}")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    lib, kernel, csvp = args[:3]
    N = int(args[3]) if len(args) > 3 else 40
    focus = None
    if "--file" in sys.argv:
        focus = sys.argv[sys.argv.index("--file") + 1]
    locs = sass_locations(lib, kernel)
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    if len(data) != len(locs):
        print(f"warning: {len(data)} profiled instructions vs {len(locs)} disassembled", file=sys.stderr)
    num = lambda x: float(x) if x else 0.0
    ks, ki = "Warp Stall Sampling (All Samples)", "Instructions Executed"
    ts = sum(num(d[ks]) for d in data) or 1
    ti = sum(num(d[ki]) for d in data) or 1
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    why = collections.defaultdict(lambda: collections.Counter())
    for d, chain in zip(data, locs):
        key = chain[0] if chain else ("?", "0")
        if focus:
            inside = [c for c in chain if os.path.basename(c[0]) == focus]
            if inside:
                key = inside[-1]
        k = f"{os.path.basename(key[0])}:{key[1]}"
        agg[k][0] += num(d[ks])
        agg[k][1] += num(d[ki])
        for r in reasons:
            why[k][r[6:]] += num(d[r])
    print(f"samples {ts:.0f}, warp-instructions {ti:.0f}")
    print(f"{'location':28s} {'stall%':>7s} {'instr%':>7s}")
    for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
        top = ", ".join(f"{r} {v / max(s, 1) * 100:.0f}%" for r, v in why[k].most_common(3) if v)
        print(f"{k:28s} {s / ts * 100:7.2f} {i / ti * 100:7.2f}   {top}")


if __name__ == "__main__":
    main()
