"""Summarise TCB_TRACE output: per-phase durations (median/max over CTAs, us)."""
import json
import statistics
import sys

names = ["start->first data", "mainloop (first unit)", "partials written", "all splits arrived",
         "reduction", "rest"]
for line in open(sys.argv[1]):
    d = json.loads(line)
    g = d["grid"]
    t = [d["t"][i * 8:(i + 1) * 8] for i in range(g)]
    t0 = min(x[0] for x in t if x[0])
    print(f"m={d['m']} n={d['n']} k={d['k']} splits={d['splits']} grid={g}")
    ends = [max(x) for x in t]
    print(f"  kernel span (first CTA start -> last mark): {(max(ends) - t0) / 1e3:.1f} us")
    starts = [x[0] - t0 for x in t]
    print(f"  CTA start skew: median {statistics.median(starts)/1e3:.2f} max {max(starts)/1e3:.2f} us")
    r1 = [(x[7] - x[1]) / 8e3 for x in t if x[7] and x[1]]
    if r1:
        print(f"  us per k-block, blocks 0-7: median {statistics.median(r1):.3f}")
    for i in range(6):
        dur = [(x[i + 1] - x[i]) / 1e3 for x in t if x[i + 1] and x[i]]
        if dur:
            print(f"  {names[i]:28s} median {statistics.median(dur):8.2f}  max {max(dur):8.2f} us")
