python tools/e2e_ab.py cfg5 3
TCB_SK_WASTE=0.05 python tools/e2e_ab.py cfg5 3
TCB_NO_PACE=1 python tools/e2e_ab.py cfg5 3
TCB_SK_WASTE=0.05 TCB_NO_PACE=1 python tools/e2e_ab.py cfg5 3
TC_SLAB_MB=64 python tools/e2e_ab.py cfg5 3
