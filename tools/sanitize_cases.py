"""Small cases of every device path for compute-sanitizer (memcheck/racecheck):
TMA and cp.async GEMM (all layouts), split-K, batched, GEMV/DOT, permutes,
the streamed host path."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import oracles as O
import paper_1307_2100_b200 as T

cases = [
    ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=130,j=70,k=16,l=40"),     # L1 split-K
    ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=64,b=48,c=5,k=40"),       # L2 batched TMA
    ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=63,b=47,c=5,k=41"),       # odd: cp.async
    ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=16,b=8,c=8,d=8,k=4,l=6"),  # L3
    ("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=9,b=17,g=5,e=33"),        # 3.1 transpose perm
    ("R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=70,b=9,g=40"),                  # GEMV
    ("R[+g] = T[+a,+b,+g] * G[-a,-b]", "a=9,b=40,g=70"),                  # GEMV k-major
    ("K[] = T[+a,+b,+g] * S[-a,-b,-g]", "a=30,b=20,g=50"),                # DOT
    ("C[-j,+i] = A[+i,+h] * B[-h,-j]", "i=33,j=65,h=17"),                 # output order swapped
]
bad = 0
for e, x in cases:
    got, _ = T.execute(e, x)
    L, R = O.operands(e, x, 1)
    err = O.max_rel_error(got, O.naive(e, x, L, R))
    print(f"{err:.2e}  {e}  [{x}]")
    bad += err > 1e-12
# streamed path
dev = T.native.device()
e, x = "C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=64,b=48,c=9,k=40"
p = T.Prepared(e, x)
inf = p.info()
L, R = O.operands(e, x, 1)
out = np.zeros(inf["output"])
for a in (L, R, out):
    T.check(dev.tcb_host_register(a.ctypes.data, a.nbytes))
p.run_streamed(L, R, out, slabs=3)
err = O.max_rel_error(out, O.naive(e, x, L, R))
print(f"{err:.2e}  streamed {e}")
bad += err > 1e-12
sys.exit(1 if bad else 0)
