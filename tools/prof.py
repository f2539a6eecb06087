"""Profiling driver: run one BASELINE config a few times through the prepared
API (device-resident), for ncu. Usage: python tools/prof.py cfg2 [runs]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
import paper_1307_2100_b200 as T

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
expr, extents, _ = bench.CONFIGS[cfg]
p = T.Prepared(expr, extents)
info = p.info()
L = T.seeded(info["left"], 1)
R = T.seeded(info["right"], 2)
p.upload(L, R)
for _ in range(runs):
    p.run()
p.sync()
print(cfg, p.info())
