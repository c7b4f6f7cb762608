"""Render a c5 sweep (tools/sweep_c5.py JSON lines) as a markdown table,
optionally with a previous build's step time beside each cell.

usage: python tools/render_c5_md.py NEW.jsonl [OLD.jsonl] > out.md"""
import json
import sys


def cells(path):
    out = {}
    for line in open(path):
        d = json.loads(line)
        if "nstar" not in d:
            continue
        key = (d["nstar"], d["m"], d["d"], d["family"], d["dtype"], d["format"])
        out[key] = d
    return out


def main():
    new = cells(sys.argv[1])
    old = cells(sys.argv[2]) if len(sys.argv) > 2 else {}
    hdr = ["n*", "m", "d", "family", "dtype", "Y", "K1 impl", "step µs"]
    if old:
        hdr.append("(prev step µs)")
    hdr += ["K1 µs", "entries/s", "GB/s", "% HBM"]
    print("| " + " | ".join(hdr) + " |")
    print("|" + "---|" * len(hdr))
    for key in sorted(new, key=lambda k: (k[1], k[5], k[2], k[3], k[4], k[0])):
        d = new[key]
        if "unsupported" in d:
            row = [str(v) for v in key[:5]] + [key[5], "—", "unsupported"]
            if old:
                row.append("")
            row += ["", "", "", ""]
        else:
            prev = old.get(key, {})
            row = [str(v) for v in key[:5]] + [key[5], d.get("impl", ""), f"{d['step_us']:.2f}"]
            if old:
                row.append(f"{prev['step_us']:.2f}" if "step_us" in prev else "—")
            row += [f"{d['k1_us']:.2f}", f"{d['entries_per_s']:.2e}", f"{d['hbm_gbs']:.1f}",
                    f"{100 * d['hbm_frac']:.1f}"]
        print("| " + " | ".join(row) + " |")


if __name__ == "__main__":
    main()
