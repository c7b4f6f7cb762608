"""SASS instruction histogram of the K1 kernels in libgmf_asgd.so: counts of the
mnemonics that prove (or disprove) tcgen05 / TMEM / TMA / cp.async use, per
kernel family.  No GPU needed.

    python tools/sass_histogram.py [lib.so] > profiles/rNN_sass_histogram.md
"""
import collections
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "paper_2412_20509_b200", "libgmf_asgd.so")
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UBLKPF", "LDGSTS",
        "SYNCS", "MUFU", "FFMA", "DFMA", "HMMA", "LDG", "STG", "LDS", "STS", "BAR", "R2UR"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
fam = collections.defaultdict(collections.Counter)
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        dem = subprocess.run(["cu++filt", name], capture_output=True, text=True).stdout.strip() or name
        cur = dem.replace("void ", "").replace("(int)", "").replace("(bool)", "")
        cur = cur[:cur.index(">(") + 1] if ">(" in cur else cur
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        fam[cur][op] += 1
        fam[cur]["_total"] += 1

def group(name):
    if "k_fit<float" in name and name.rstrip(">").endswith(", 2"):
        return "k_fit fp32, K1 v2 (tc2, warp-specialized)"
    if "k_fit<float" in name and name.rstrip(">").endswith(", 1"):
        return "k_fit fp32, K1 v1 (tc)"
    if "k_grad2" in name:
        return "k_grad2 (K1 v2 per-step)"
    if "k_grad<float" in name and (name.rstrip(">").endswith(", 1") or "true" in name):
        return "k_grad fp32 tensor (K1 v1 per-step)"
    if "k_fit<" in name or "k_grad<" in name:
        return "k_fit / k_grad on CUDA cores (fp64, weights, holes, general mode)"
    return None

agg = collections.defaultdict(collections.Counter)
nk = collections.Counter()
for name, c in fam.items():
    g = group(name)
    if g:
        agg[g].update(c)
        nk[g] += 1
print("# SASS instruction histogram of the K1 kernels (`cuobjdump -sass libgmf_asgd.so`)\n")
print("Static instruction counts summed over each family's instantiations (feature buckets,")
print("Poisson / NB).  UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld, UTCBAR = tcgen05.commit,")
print("UBLKCP = cp.async.bulk (TMA bulk copy), UBLKPF = bulk L2 prefetch, LDGSTS = cp.async,")
print("SYNCS = mbarrier ops.\n")
print("| kernel family | kernels | total | " + " | ".join(KEYS) + " |")
print("|---|---|---|" + "---|" * len(KEYS))
for g in sorted(agg):
    c = agg[g]
    print(f"| {g} | {nk[g]} | {c['_total']} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")
tot = collections.Counter()
for c in fam.values():
    tot.update(c)
print(f"\nWhole library: {len(fam)} kernels, " + ", ".join(f"{k} {tot.get(k, 0)}" for k in KEYS[:9]) + ".")
