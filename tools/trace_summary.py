"""Summarise TCB_TRACE output: per-phase durations (median/max over CTAs, us)."""
import json
import statistics
import sys

names = ["start->first data", "mainloop (first unit)", "partials written", "all splits arrived",
         "reduction", "rest"]
for line in open(sys.argv[1]):
    d = json.loads(line)
    g = d["grid"]
    w = len(d["t"]) // g  # slots per CTA (8, or 16 with per-tile marks)
    t = [d["t"][i * w:(i + 1) * w] for i in range(g)]
    t0 = min(x[0] for x in t if x[0])
    print(f"m={d['m']} n={d['n']} k={d['k']} splits={d['splits']} grid={g}")
    ends = [max(x) for x in t]
    if w == 32:  # slots 8+3t: tile t mainloop end, 9+3t: epilogue handed off, 10+3t: next data
        med = lambda v: statistics.median(v) if v else float("nan")
        for j in range(0, 7):
            a, b, c, nxt = (8 + 3 * j, 9 + 3 * j, 10 + 3 * j, 8 + 3 * (j + 1))
            epi = [(x[b] - x[a]) / 1e3 for x in t if x[a] and x[b]]
            gap = [(x[c] - x[b]) / 1e3 for x in t if x[b] and x[c]]
            loop = [(x[nxt] - x[c]) / 1e3 for x in t if x[c] and x[nxt]]
            print(f"  tile {j + 1}: epilogue {med(epi):6.2f}  wait first data {med(gap):6.2f}  "
                  f"mainloop {med(loop):7.2f} us (median over CTAs)")
    if w == 32:  # slots 30/31: tile 2 after 4 / 8 k-blocks (ramp inside a tile)
        r = [((x[30] - x[13]) / 4e3, (x[31] - x[30]) / 4e3, (x[14] - x[31]) / 8e3)
             for x in t if x[13] and x[30] and x[31] and x[14]]
        if r:
            print("  tile 2 us per k-block: blocks 0-3 %.3f, 4-7 %.3f, 8-end %.3f" %
                  tuple(statistics.median(v[i] for v in r) for i in range(3)))
    starts = [x[0] - t0 for x in t]
    print(f"  CTA start skew: median {statistics.median(starts)/1e3:.2f} max {max(starts)/1e3:.2f} us")
    r1 = [(x[7] - x[1]) / 8e3 for x in t if x[7] and x[1]]
    if r1:
        print(f"  us per k-block, blocks 0-7: median {statistics.median(r1):.3f}")
    for i in range(6):
        dur = [(x[i + 1] - x[i]) / 1e3 for x in t if x[i + 1] and x[i]]
        if dur:
            print(f"  {names[i]:28s} median {statistics.median(dur):8.2f}  max {max(dur):8.2f} us")
