#!/usr/bin/env python
"""tc::execute (the reference-facing C++ entry point, pageable std::vector-style
Tensor storage) timed through tc::run_bench on the BASELINE configs: median
wall seconds per call over `reps` calls on the same operands (transfers,
allocation of the result and the contraction all inside). TC_NO_PIN=1 turns
off the page-locking of large tensor blocks (the pageable bounce-buffer path).

    python tools/execute_bench.py [cfg1 cfg2 ...] [--reps 7]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1307_2100_b200 as T  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 7
for cfg in [a for a in args if a in bench.CONFIGS] or ["cfg2"]:
    e, x, _ = bench.CONFIGS[cfg]
    csv, ok = T.bench_csv("custom", sizes=(1,), kernels=("GEMM",), repetitions=reps,
                          custom_expr=e, custom_extents=x)
    head, row = csv.strip().splitlines()[:2]
    print(json.dumps({"tool": "execute_bench", "config": cfg, "reps": reps, "csv": row}))
