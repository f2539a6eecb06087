"""Split an ncu source-page sample profile into main-loop (DMMA region) vs the
rest, with stall reasons and the opcodes sampled outside the loop.
Usage: python tools/ncu_source_split.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out))
next(r)
hdr = next(r)
rows = [dict(zip(hdr, x)) for x in r if len(x) == len(hdr)]
base = int(rows[0]["Address"], 16)
dm = [int(x["Address"], 16) - base for x in rows if "DMMA" in x["Source"]]
lo, hi = (min(dm), max(dm)) if dm else (0, -1)
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows)
inl, outl, ops = Counter(), Counter(), Counter()
n_in = n_out = 0
for x in rows:
    a = int(x["Address"], 16) - base
    n = int(x["Warp Stall Sampling (All Samples)"] or 0)
    inside = lo - 0x400 <= a <= hi + 0x100
    for k in x:
        if k.startswith("stall_") and "(Not" not in k and x[k] not in ("0", ""):
            (inl if inside else outl)[k[6:]] += int(x[k])
    if inside:
        n_in += n
    else:
        n_out += n
        src = x["Source"].strip()
        op = src.split()[1] if src.startswith("@") else src.split()[0]
        ops[op.split(".")[0]] += n
print(f"samples total {tot}  mainloop {n_in} ({100 * n_in / max(tot, 1):.1f}%)  outside {n_out}")
print("mainloop stalls:", inl.most_common(8))
print("outside stalls:", outl.most_common(10))
print("outside samples by opcode:", ops.most_common(20))
top = sorted((x for x in rows if not (lo - 0x400 <= int(x["Address"], 16) - base <= hi + 0x100)),
             key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:15]
for x in top:
    print(hex(int(x["Address"], 16) - base), x["Source"][:60].ljust(60),
          x["Warp Stall Sampling (All Samples)"])
