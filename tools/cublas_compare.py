"""Vendor-library comparison point (not a product path): cuBLAS DGEMM through
torch on the GEMM each BASELINE config lowers to, timed like bench.py's
device leg (CUDA events over back-to-back launches; cfg1 rotates over 8
operand copies so no launch re-reads L2-hot data). cfg3's permutations are not
included for cuBLAS (it cannot read the interleaved operands in place).
Prints one JSON line per case."""
import json

import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")


def bench(name, fn, flops, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    print(json.dumps({"case": name, "us": round(t * 1e6, 1),
                      "tflops": round(flops / t / 1e12, 2)}), flush=True)


def rnd(*shape):
    return torch.rand(*shape, dtype=torch.float64, device=dev)


As, Bs = [rnd(512, 4096) for _ in range(8)], [rnd(4096, 512) for _ in range(8)]
it = [0]


def cfg1():
    k = it[0] % 8
    it[0] += 1
    torch.mm(As[k], Bs[k])


bench("cfg1 GEMM 512x512x4096 (8 rotating copies)", cfg1, 2 * 512 * 512 * 4096)
A, B = rnd(256, 256, 256), rnd(256, 256)
bench("cfg2 batched GEMM 256 x (256x256x256)", lambda: torch.matmul(A, B), 2 * 256 ** 4)
A, B = rnd(4096, 1024), rnd(1024, 4096)
bench("cfg3 GEMM 4096x4096x1024 (operands pre-permuted)", lambda: torch.mm(A, B),
      2 * 4096 * 4096 * 1024)
A, B = rnd(65536, 4096), rnd(4096, 4096)
bench("cfg4 GEMM 65536x4096x4096", lambda: torch.mm(A, B), 2 * 65536 * 4096 * 4096, reps=5)
