for c in cfg1 cfg2 cfg3; do python tools/e2e_ab.py $c 30; done
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
