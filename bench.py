#!/usr/bin/env python
"""bench.py — fp64 contraction throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1..cfg5]

Default workload: BASELINE.json configs[4] (cfg5), the largest config that
fits one GPU: C[i,j] = sum_{k,l} A[i,k,l] B[k,l,j], i=j=8192, k=l=512
(35.2 TFLOP per step, 34.9 GB of operands + result). A *step* is one
evaluation of the contraction. Prints ONE JSON line on rank 0.

  value    GFLOP/s of the whole job: plan.flops of the FULL contraction x K /
           (CUDA-event time of exactly K steps, max over ranks); operands
           resident in HBM; flops = 2*prod(extents) (src/expr.cpp:257-261).
           Consecutive steps use programmatic dependent launch.
  e2e      the same metric through the drop-in call tc::execute on caller host
           buffers (tcf_execute_host, include/tcf.h): every step parses, plans,
           uploads its operands from pinned host memory, contracts and
           downloads its result inside the timed region. The repo's pipelined
           API (tcf_run_streamed_async) is reported beside it as
           e2e.pipelined. For the K-split at N>1: upload + fused scatter/reduce
           + D2H of the rank's block.
  roofline the DMMA GEMM launch alone (CUDA events on its own stream) against
           the fp64 DMMA peak measured live on this GPU (tcb_fp64_peak; the
           driver's MEASURED_PEAKS.json has no fp64 entry); traffic = DRAM
           bytes per launch from profiles/ncu_<cfg>_summary.json.
  parity   the step's result checked against the committed golden samples of
           the reference (tests/golden/baseline.json) on every rank's own
           output block; parity_ok = all ranks within 1e-12.
  cpu_baseline  the unmodified reference (oracle/_ref, compiled from
           /root/reference) timed on the host cores on a bounded sample of the
           same workload (rank 0, N=1), at workers=nproc and workers=1 and with
           the -march build for this CPU.

Multi-GPU (--gpus N; the driver launches torchrun, or bench.py spawns it):
  cfg5   contracted l split N ways, partial C reduce-scattered along j — fused
         into the GEMM epilogue over peer memory (default) or NCCL
         (--exchange nccl); strong scaling
  cfg1-4 a free label split N ways (cfg1 j, cfg2 c, cfg3 d, cfg4 b), no
         data-path collective; strong scaling
Each rank generates only its own slabs of the seeded operands (tcf_seeded_block).

--impl reference times the reference's own CPU implementation (oracle/_ref)
on all host cores on a bounded sample of the same workload per step and
prints the same line with "impl": "reference" (rank 0 only under torchrun).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import weakref
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fp64 contraction GFLOP/s and % of B200 FP64 peak at 1/2/4/8 GPUs vs host-CPU ref"
CONFIGS = {
    "cfg1": ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=512,j=512,k=64,l=64",
             "BASELINE configs[0]: class-1 C[i,j]=A[i,k,l]B[k,l,j], i=j=512, k=l=64"),
    "cfg2": ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=256,b=256,c=256,k=256",
             "BASELINE configs[1]: class-2 C[a,b,c]=A[a,k,c]B[k,b], a=b=c=k=256"),
    "cfg3": ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]",
             "a=64,b=64,c=64,d=64,k=32,l=32",
             "BASELINE configs[2]: class-3 C[a,b,c,d]=A[a,k,c,l]B[l,b,k,d], a..d=64, k=l=32"),
    "cfg4": ("C[+a,+b,+i,+j] = A[+a,+b,+k,+l] * B[-k,-l,+i,+j]",
             "a=256,b=256,i=64,j=64,k=64,l=64",
             "BASELINE configs[3]: CCD C[a,b,i,j]=A[a,b,k,l]B[k,l,i,j], a=b=256, i..l=64"),
    "cfg5": ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=8192,j=8192,k=512,l=512",
             "BASELINE configs[4]: large class-1 C[i,j]=A[i,k,l]B[k,l,j], i=j=8192, k=l=512 "
             "(largest BASELINE config that fits one GPU: 34.9 GB)"),
}
# How a config runs on N > 1 ranks. Every mode is strong
# scaling: the full BASELINE contraction is split across the ranks.
#   shard  a free label split N ways, no data-path collective
#   ksplit the contracted label split N ways, partial C reduce-scattered along
#          the outermost output label (cfg5: split l, scatter j)
MODE = {"cfg1": ("shard", "j"), "cfg2": ("shard", "c"), "cfg3": ("shard", "d"),
        "cfg4": ("shard", "b"), "cfg5": ("ksplit", "l")}
# Bounded CPU samples of each workload for the reference arm and cpu_baseline
# (a full cfg5 on the reference is ~1.2 h on one core, cfg4 ~40 s): extents of
# a sub-contraction whose per-call kernel shape equals the full plan's. The
# reference's GEMM packs 256-column panels of B (kernels_reference.cpp:50-53),
# so a 256-column j-slab runs exactly one panel per call, as every panel of
# the full call does; 8 of the 512 l-iterations of its loop nest.
CPU_SAMPLE = {
    "cfg1": ("i=512,j=512,k=64,l=64", "the full cfg1 contraction"),
    "cfg2": ("a=256,b=256,c=256,k=256", "the full cfg2 contraction"),
    "cfg3": ("a=64,b=64,c=64,d=64,k=32,l=32", "the full cfg3 contraction"),
    "cfg4": ("a=256,b=16,i=64,j=64,k=64,l=64",
             "b<16 slab of cfg4 (1/16 of the work; the plan's per-call GEMM 256x64x64 and "
             "loop nest b:free j:free l:contracted unchanged), scaled by flops"),
    "cfg5": ("i=8192,j=256,k=512,l=8",
             "j<256, l<8 slab of cfg5 (1/256 of the work): 8 of the 512 l-iterations of the "
             "reference's loop nest, each the full 8192-row GEMM over one 256-column B panel "
             "(the reference kernel's own panel width, so per-panel work equals the full "
             "call's), scaled by flops — extrapolated"),
}
L2_BYTES = 126 * 2**20
GOLDEN = ROOT / "tests" / "golden" / "baseline.json"


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def nvml_index(device: int) -> int:
    """Physical (NVML / nvidia-smi) index of CUDA device `device`."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [v.strip() for v in vis.split(",") if v.strip()]
    if device < len(ids) and ids[device].isdigit():
        return int(ids[device])
    return device


class NvmlClocks:
    """SM clock + clock-event-reason sampler on a thread (NVML, every ~2 ms),
    so even a timed region of a few tens of ms holds many samples; one sample
    is also taken when the region starts and one when it ends."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device: int):
        import threading
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = nv.nvmlDeviceGetHandleByIndex(nvml_index(device))
        self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        self.masks = [(n, getattr(nv, c)) for n, c in self.REASONS]
        self.rows = []
        self.halt = threading.Event()
        self.sample()
        self.thread = threading.Thread(target=self.loop, daemon=True)
        self.thread.start()

    def sample(self):
        nv = self.nv
        try:
            sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except nv.NVMLError:
            return
        self.rows.append((float(sm), int(bits)))

    def loop(self):
        while not self.halt.wait(0.002):
            self.sample()

    def stop(self) -> dict:
        self.sample()
        self.halt.set()
        self.thread.join(timeout=2)
        rows = list(self.rows)
        reasons = sorted({n for _, b in rows for n, m in self.masks if b & m})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": self.max_mhz,
                "samples": len(rows), "reasons": reasons, "sampler": "nvml"}


def Clocks(device: int):
    try:
        return NvmlClocks(device)
    except Exception:
        return SmiClocks(device)


class SmiClocks:
    """nvidia-smi sampler running during the timed region (fallback when NVML
    is not importable)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.proc = None
        device = nvml_index(device)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        rows = []
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:]) if v.lower() == "active"})
        sm = [float(r[0]) for r in rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]),
                "samples": len(rows), "reasons": reasons}


def pinned_array(n: int, dev) -> np.ndarray:
    a = np.empty(int(n))
    if a.nbytes:
        check = dev.tcb_host_register(a.ctypes.data, a.nbytes)
        if check != 0:
            raise RuntimeError(dev.tcb_last_error().decode())
        # unregister before numpy frees the memory (never leave it registered)
        weakref.finalize(a, dev.tcb_host_unregister, a.ctypes.data)
    return a

def ext_map(extents: str) -> dict:
    return {k: int(v) for k, v in (kv.split("=") for kv in extents.split(",") if kv)}


def flops_of(extents: str) -> int:
    return 2 * int(np.prod(list(ext_map(extents).values()), dtype=np.int64))


def free_space(expr: str, extents: str) -> int:
    """Free-slice count of the reference's auto plan (src/executor.cpp:330-336):
    the reference's worker threads split only the free loops, so this bounds
    the cores it can use."""
    import paper_1307_2100_b200 as T
    auto = T.report(expr, extents).split("auto:\n")[1]
    nest = auto.split("loop_nest:")[1].split("\n")[0].split()
    exts = [int(x) for x in auto.split("loop_extents:")[1].split("\n")[0].split()]
    n = 1
    for item, e in zip(nest, exts):
        if item.endswith(":free"):
            n *= e
    return n


def cpu_info() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_reference(expr: str, extents: str, workers: int, variant: str, reps: int,
                   warmup: int = 1) -> list[float]:
    """Wall seconds of `reps` tc::execute calls of the unmodified reference
    (oracle/_ref) with the reference backend — TEST INFRASTRUCTURE, CPU arm only."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles  # the CPU baseline only; never on the device path
    b = oracles.RefBound(expr, extents, seed=1, variant=variant)
    try:
        for _ in range(warmup):
            b.run(workers)
        return [b.run(workers) for _ in range(reps)]
    finally:
        b.close()


def cpu_baseline(cfg: str) -> dict | None:
    """The reference on the host cores, on CPU_SAMPLE[cfg]: workers = nproc
    (the reported value), workers = 1, and the -march build for this CPU."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles
    if oracles.ref() is None:
        return None
    expr = CONFIGS[cfg][0]
    sample, what = CPU_SAMPLE[cfg]
    nproc = os.cpu_count() or 1
    fs = free_space(expr, sample)
    fl = flops_of(sample)
    native = oracles.native_variant()
    runs = []
    for variant, workers, flags in (("", nproc, "-O3 -DNDEBUG (reference CMake flags)"),
                                    ("", 1, "-O3 -DNDEBUG (reference CMake flags)"),
                                    (native, nproc, {"_v4": "-O3 -DNDEBUG -march=x86-64-v4",
                                                     "_v3": "-O3 -DNDEBUG -march=x86-64-v3",
                                                     "": "-O3 -DNDEBUG"}[native]
                                     + " (-march=native equivalent for this CPU)")):
        if oracles.ref(variant) is None:
            continue
        secs = statistics.median(time_reference(expr, sample, workers, variant, reps=3))
        runs.append({"flags": flags, "workers": workers, "cores_used": min(workers, fs),
                     "value": round(fl / secs / 1e9, 3), "unit": "GFLOP/s",
                     "sample_s": round(secs, 4)})
    head = runs[0]
    return {"value": head["value"], "unit": "GFLOP/s", "cores": head["cores_used"],
            "kind": "reference",
            "sample": f"{what}; tc::execute with the reference backend, workers={nproc}, "
                      f"median of 3 after 1 warm-up",
            "extrapolated": cfg in ("cfg4", "cfg5"),
            "host": f"{nproc} threads, {cpu_info()}",
            "cores_note": ("the reference parallelises only free loops of its plan "
                           f"(src/executor.cpp:330-336); this plan has {fs} free slice(s)"),
            "variants": runs}


def run_reference_arm(args, cfg) -> int:
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles
    if oracles.ref() is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libtcref.so missing (build with make -C oracle)"}))
        return 0
    expr, extents, desc = CONFIGS[cfg]
    sample, what = CPU_SAMPLE[cfg]
    nproc = os.cpu_count() or 1
    fs = free_space(expr, sample)
    fl = flops_of(sample)
    secs = time_reference(expr, sample, nproc, "", reps=args.steps, warmup=args.warmup)
    total = sum(secs)
    value = fl * args.steps / total / 1e9
    full_s = flops_of(extents) / (value * 1e9)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Tensor::seeded_random uniform[-1,1], seeds 1 (A) / 2 (B)",
        "config": {"workload": desc, "expr": expr, "extents": extents,
                   "sample_extents": sample,
                   "path": "reference tc::execute + ReferenceBackend (oracle/_ref, -O3 -DNDEBUG)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": min(nproc, fs),
                         "kind": "reference",
                         "sample": f"{what}; one sample per step, workers={nproc}",
                         "extrapolated": cfg in ("cfg4", "cfg5"),
                         "extrapolated_full_step_s": round(full_s, 3),
                         "host": f"{nproc} threads, {cpu_info()}"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def golden_parity(cfg: str, expr: str, full: str, label: str | None, lo: int, hi: int,
                  got: np.ndarray) -> dict:
    """Checks this rank's output block against the committed golden samples of
    the reference's result (tests/golden/baseline.json, made from the compiled
    reference by tests/golden/make_golden.py). `got` is the output slab
    [lo, hi) along `label` (the whole output when label is None)."""
    gold = json.loads(GOLDEN.read_text())
    g = gold["cfg5_slab"] if cfg == "cfg5" else gold[cfg]
    out = expr.split("=")[0]
    out = [x.strip()[1:] for x in out[out.index("[") + 1:out.index("]")].split(",")]
    em = ext_map(full)
    idx = np.array(g["idx"], dtype=np.int64)
    val = np.array(g["val"])
    coords, rem = {}, idx.copy()
    for x in out:
        coords[x] = rem % em[x]
        rem //= em[x]
    sub = dict(em)
    keep = np.ones(idx.size, bool)
    if label is not None:
        keep = (coords[label] >= lo) & (coords[label] < hi)
        sub[label] = hi - lo
    local = np.zeros(idx.size, np.int64)
    run = 1
    for x in out:
        c = coords[x] - (lo if x == label else 0)
        local += c * run
        run *= sub[x]
    res = {"samples": int(keep.sum()), "source": "tests/golden/baseline.json"
           + (" (cfg5: the reference's j<64 column slab)" if cfg == "cfg5" else "")}
    if keep.any():
        want = val[keep]
        err = float(np.abs(got[local[keep]] - want).max() / max(1.0, np.abs(val).max()))
        res["max_rel_error"] = err
        res["ok"] = bool(err <= 1e-12)
    else:
        res["ok"] = True
    if label is None or (lo == 0 and hi == em[label]):
        part = got[:g["n"]] if cfg == "cfg5" else got  # the slab is C's first n entries
        ss = float((part * part).sum())
        res["sumsq_rel"] = abs(ss - g["sumsq"]) / g["sumsq"]
        res["ok"] = res["ok"] and res["sumsq_rel"] <= 1e-11
    return res


def peer_self_test(T, dev, prep, exchange, scat, block, world, rank, torch, backend):
    """One host-synchronised step of the fused K-split exchange, checked
    against a plain all-reduce of the ranks' partial outputs (torch.distributed).
    Returns None when the rank's block agrees (rel. error <= 1e-12), else why."""
    import ctypes as C
    saved = exchange.host_sync
    exchange.host_sync = True
    try:
        exchange.step(prep, scat.ptr)
    finally:
        exchange.host_sync = saved
    T.check(dev.tcb_sync(), "tcb_sync")
    got = np.empty(block)
    T.check(dev.tcb_d2h(got.ctypes.data, scat.ptr, block * 8), "tcb_d2h")
    prep.run()  # the rank's partial C, unscattered
    prep.sync()
    _, _, optr = prep.device_ptrs()
    part = np.empty(block * world)
    T.check(dev.tcb_d2h(part.ctypes.data, optr, part.nbytes), "tcb_d2h")
    t = torch.from_numpy(part)
    if backend == "nccl":
        t = t.cuda()
    torch.distributed.all_reduce(t)
    want = t[rank * block:(rank + 1) * block].cpu().numpy()
    err = float(np.abs(got - want).max() / max(1.0, float(np.abs(want).max())))
    return None if err <= 1e-12 else f"block differs from the all-reduce by {err:.3g}"


def relaunch(args) -> int:
    """--gpus N without torchrun: spawn N ranks on this node."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def fill_operands(expr: str, full: str, label: str | None, lo: int, hi: int, L, R) -> None:
    """This rank's slabs of the seeded operands (A: seed 1, B: seed 2), written
    into L and R; the two streams are drawn concurrently."""
    import paper_1307_2100_b200 as T
    from paper_1307_2100_b200 import partition as P
    _, left, right = P.parse(expr)
    em = ext_map(full)
    front = T.native.front()
    errs = []

    def gen(labels, seed, arr):
        try:
            ext = [em[x] for x in labels]
            if label is None or label not in labels:
                front.tcf_seeded(arr.size, seed, arr.ctypes.data)
            else:
                a = (C.c_int64 * len(ext))(*ext)
                rc = front.tcf_seeded_block(seed, len(ext), a, labels.index(label), lo, hi,
                                            arr.ctypes.data)
                if rc:
                    raise RuntimeError(front.tcf_last_error().decode())
        except Exception as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=gen, args=(left, 1, L)),
          threading.Thread(target=gen, args=(right, 2, R))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


# (steps, warmup) when the command line names none
DEFAULT_STEPS = {"cfg1": (300, 20), "cfg2": (200, 10), "cfg3": (50, 5), "cfg4": (10, 3),
                 "cfg5": (10, 3)}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: per config, see DEFAULT_STEPS)")
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="K-split (cfg5, N>1): partial-C blocks written into their owners' "
                         "receive buffers by the GEMM epilogue over NVLink (peer, fused) or "
                         "a separate NCCL reduce-scatter after the GEMM (nccl)")
    ap.add_argument("--l2", default="rotate", choices=["rotate", "flush"],
                    help="keeping L2-sized working sets cold: rotate over copies or flush")
    args = ap.parse_args()
    cfg = args.config
    # without flags: enough steps that the timed region is tens of ms at least
    # (ten 70-us steps of cfg1 end before the SM clock has settled: 0.77 of
    # peak against 0.81 over 300 steps on the same box)
    ours = args.impl == "ours"  # the CPU arm's steps are seconds each: 10 / 3
    if args.steps is None:
        args.steps = DEFAULT_STEPS[cfg][0] if ours else 10
    if args.warmup is None:
        args.warmup = DEFAULT_STEPS[cfg][1] if ours else 3
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if os.environ.get("TCB_BENCH_EXTENTS"):  # plumbing tests only, never a BASELINE number
        e, _, d = CONFIGS[cfg]
        CONFIGS[cfg] = (e, os.environ["TCB_BENCH_EXTENTS"],
                        d + " [extents overridden by TCB_BENCH_EXTENTS: plumbing test, not the "
                            "BASELINE workload]")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    # one GPU per rank; ranks beyond the visible GPUs share them round-robin
    # (only for single-GPU plumbing tests with TCB_DIST_BACKEND=gloo)
    import paper_1307_2100_b200 as T
    from paper_1307_2100_b200 import partition as P
    dev = T.native.device()
    ndev = C.c_int(0)
    dev.tcb_device_count(C.byref(ndev))
    local = local % max(1, ndev.value)
    torch = None
    backend = os.environ.get("TCB_DIST_BACKEND", "nccl")  # gloo: plumbing tests on one GPU
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def all_reduce(x: float, op: str) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64,
                         device="cuda" if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=getattr(torch.distributed.ReduceOp, op))
        return float(t.item())

    T.check(dev.tcb_init(local), "tcb_init")
    expr, full, desc = CONFIGS[cfg]
    mode, label = MODE[cfg]
    if world == 1:
        mode, label, lo, hi, extents = "single", None, 0, 0, full
    else:
        sh = (P.shard_free if mode == "shard" else P.shard_contracted)(expr, full, label,
                                                                      world, rank)
        lo, hi, extents = sh.lo, sh.hi, sh.extents
    peak = C.c_double()
    T.check(dev.tcb_fp64_peak(C.byref(peak)), "tcb_fp64_peak")

    prep = T.Prepared(expr, extents, device=local)
    info = prep.info()
    flops = info["flops"]           # this rank's share
    total_flops = flops_of(full)    # the whole job (strong scaling)
    L = pinned_array(info["left"], dev)
    R = pinned_array(info["right"], dev)
    O = pinned_array(info["output"], dev)
    t_gen = time.time()
    fill_operands(expr, full, label, lo, hi, L, R)
    t_gen = time.time() - t_gen

    collective = exchange = None
    exchange_note = None
    block = info["output"]
    prep.upload(L, R)
    if mode == "ksplit":
        block = info["output"] // world
        scat = T.DeviceBuffer(block * 8)
    if mode == "ksplit" and args.exchange == "peer":
        # fused: the GEMM epilogue writes each block of this rank's partial C
        # into its owner's receive buffer through the peer window (tcb_peer_*),
        # then each rank sums its received slots (partition.PeerKSplit).
        # Ranks sharing one GPU (gloo plumbing runs): host barriers between the
        # phases instead of device-side flag waits across processes.
        # Self-test first (one host-synchronised step against a plain
        # all-reduce of the partials); any failure falls back to NCCL.
        why = None
        try:
            exchange = P.PeerKSplit(dev, world, rank, block, torch.distributed,
                                    host_sync=backend != "nccl")
            why = peer_self_test(T, dev, prep, exchange, scat, block, world, rank, torch,
                                 backend)
        except Exception as e:  # noqa: BLE001 - any failure selects the fallback
            why = f"{type(e).__name__}: {e}"
        failed = torch.tensor([1.0 if why else 0.0], dtype=torch.float64,
                              device="cuda" if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(failed, op=torch.distributed.ReduceOp.MAX)
        if failed.item() > 0:
            if exchange is not None:
                try:
                    exchange.close()
                except Exception:
                    pass
            exchange = None
            exchange_note = f"peer exchange self-test failed ({why or 'on another rank'}); NCCL"
            if backend != "nccl":
                raise SystemExit(exchange_note)
    if mode == "ksplit" and exchange is None:
        if backend != "nccl":
            raise SystemExit("ksplit (cfg5) with --exchange nccl needs the nccl backend")
        # the engine's own NCCL communicator (tcb_comm_*, include/tcb.h); the
        # reduce-scatter runs on the engine's stream right behind the
        # contraction. NCCL's algorithm and protocol are pinned so the summation
        # order (and so the result) is the same run to run.
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        uid = (C.c_char * 128)()
        if rank == 0:
            T.check(dev.tcb_comm_unique_id(uid), "tcb_comm_unique_id")
        shipped = [bytes(uid) if rank == 0 else None]
        torch.distributed.broadcast_object_list(shipped, src=0)
        uid = (C.c_char * 128).from_buffer_copy(shipped[0])
        comm = C.c_void_p()
        T.check(dev.tcb_comm_init(world, rank, uid, C.byref(comm)), "tcb_comm_init")
        _, _, optr = prep.device_ptrs()

        def collective():
            T.check(dev.tcb_reduce_scatter(optr, scat.ptr, block, comm), "tcb_reduce_scatter")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()
        prep.sync()

    # ---- L2 treatment. Working sets larger than L2 run back to back. Smaller
    # ones (cfg1: 34 MB) are never re-read hot: by default (--l2 rotate) the
    # steps cycle over R independent prepared copies of the contraction (own
    # operands and output, together >= 2 x L2), so every step reads its
    # operands from HBM and the steps still run back to back; --l2 flush
    # instead writes a 2 x L2 buffer before every step, outside the timed
    # region, and brackets each step by its own events.
    ws_bytes = (info["left"] + info["right"] + info["output"]) * 8
    small = ws_bytes <= L2_BYTES
    flush = small and args.l2 == "flush"
    flush_buf = T.DeviceBuffer(2 * L2_BYTES) if flush else None
    preps = [prep]
    if small and not flush:
        if mode == "ksplit":
            raise SystemExit("rotation with a collective is not supported")
        n_copies = -(-2 * L2_BYTES // ws_bytes)
        for _ in range(n_copies - 1):
            q = T.Prepared(expr, extents, device=local)
            q.upload(L, R)
            preps.append(q)
        prep.sync()
    n_rot = len(preps)
    rot = [0]

    def step():
        if exchange is not None:
            exchange.step(prep, scat.ptr)
            return
        preps[rot[0] % n_rot].run()
        rot[0] += 1
        if collective is not None:
            collective()

    def kernel_only():
        preps[rot[0] % n_rot].run_contraction()
        rot[0] += 1

    # ---- device-resident throughput over exactly K steps
    for _ in range(args.warmup):
        step()
    barrier()
    clocks = Clocks(local)
    time.sleep(0.15)
    dev.tcb_reset_launch_count()
    ms = C.c_float()

    def timed(fn, n):
        if flush:
            total = 0.0
            for _ in range(n):
                T.check(dev.tcb_memset0(flush_buf.ptr, 2 * L2_BYTES), "L2 flush")
                T.check(dev.tcb_timer_start())
                fn()
                T.check(dev.tcb_timer_stop(C.byref(ms)))
                total += float(ms.value)
            return total
        T.check(dev.tcb_timer_start())
        for _ in range(n):
            fn()
        T.check(dev.tcb_timer_stop(C.byref(ms)))
        return float(ms.value)

    total_ms = timed(step, args.steps)
    launches = dev.tcb_launch_count()
    clk = clocks.stop()
    barrier()
    t_ms = all_reduce(total_ms, "MAX")
    step_ms = t_ms / args.steps
    value = total_flops / (step_ms * 1e-3) / 1e9

    # ---- parity of the timed steps' result: this rank's output block
    barrier()
    got = np.empty(block)
    if mode == "ksplit":
        T.check(dev.tcb_d2h(got.ctypes.data, scat.ptr, block * 8), "tcb_d2h")
        # rank r owns the r-th block of the outermost output label (j)
        out_last = expr.split("=")[0].split(",")[-1].strip(" ]+-")
        n_out = ext_map(full)[out_last]
        plo, phi, plabel = n_out * rank // world, n_out * (rank + 1) // world, out_last
    else:
        prep.download(got)
        plo, phi, plabel = lo, hi, label
    parity = golden_parity(cfg, expr, full, plabel, plo, phi, got)
    parity["ranks_ok"] = all_reduce(1.0 if parity["ok"] else 0.0, "MIN") == 1.0
    parity["samples_all_ranks"] = int(all_reduce(float(parity["samples"]), "SUM"))
    del got

    # ---- the dominant kernel alone (the contraction launch), same L2 treatment
    n_kern = max(3, min(args.steps, 50, int(2000.0 / max(step_ms, 1e-3))))
    for q in preps:
        q.run_permutes()
    prep.sync()
    kern_ms = timed(kernel_only, n_kern) / n_kern
    achieved = flops / (kern_ms * 1e-3) / 1e12
    gemm_info = T.GemmInfo()
    dev.tcb_last_gemm_info(C.byref(gemm_info))

    # ---- end to end with host buffers
    n_e2e = max(3, min(args.steps, 20, int(1500.0 / max(step_ms, 1e-3))))
    barrier()
    e2e = {"unit": "GFLOP/s", "h2d_bytes_per_step": int((info["left"] + info["right"]) * 8),
           "d2h_bytes_per_step": int(block * 8), "steps": n_e2e}
    if mode != "ksplit":
        # (1) the drop-in call: tc::execute on the caller's pinned host buffers
        # (tcf_execute_host), one synchronous call per step, result on the host
        T.execute_host(expr, extents, L, R, O)  # warm-up (pool, streams)
        rounds = []
        for _ in range(3):
            barrier()
            T.check(dev.tcb_timer_start())
            for _ in range(n_e2e):
                T.execute_host(expr, extents, L, R, O)
            T.check(dev.tcb_timer_stop(C.byref(ms)))
            rounds.append(all_reduce(float(ms.value), "MAX") / n_e2e)
        e2e_ms = statistics.median(rounds)
        e2e.update({"value": round(total_flops / (e2e_ms * 1e-3) / 1e9, 3),
                    "ms_per_step": round(e2e_ms, 4),
                    "rounds_ms_per_step": [round(r, 4) for r in rounds],
                    "api": "tc::execute on caller host buffers (tcf_execute_host, include/tcf.h; "
                           "reference include/tc/executor.hpp:28-32): parse, plan, H2D from "
                           "pinned memory overlapped with the DMMA contraction, D2H of the "
                           "result, one synchronous call per step"})
        e2e_check = golden_parity(cfg, expr, full, label, lo, hi, O)
        e2e["parity_ok"] = bool(all_reduce(1.0 if e2e_check["ok"] else 0.0, "MIN") == 1.0)
        # (2) the repo's pipelined API: successive steps overlap (two buffer sets)
        slabs_used = 1
        for _ in range(2):
            slabs_used = prep.run_streamed(L, R, O, slabs=0, wait=False)
        prep.sync()
        barrier()
        T.check(dev.tcb_timer_start())
        for _ in range(n_e2e):
            prep.run_streamed(L, R, O, slabs=0, wait=False)
        prep.sync()
        T.check(dev.tcb_timer_stop(C.byref(ms)))
        pipe_ms = all_reduce(float(ms.value), "MAX") / n_e2e
        e2e["pipelined"] = {
            "value": round(total_flops / (pipe_ms * 1e-3) / 1e9, 3),
            "ms_per_step": round(pipe_ms, 4),
            "api": "tcf_run_streamed_async: H2D / DMMA / D2H overlapped over %d slabs, "
                   "successive steps pipelined over two device buffer sets, tcf_sync at the "
                   "end" % slabs_used}
    else:
        rounds = []
        out_view = np.empty(block)
        for _ in range(3):
            barrier()
            T.check(dev.tcb_timer_start())
            for _ in range(n_e2e):
                prep.upload(L, R)
                step()
                T.check(dev.tcb_d2h(out_view.ctypes.data, scat.ptr, block * 8), "tcb_d2h")
            T.check(dev.tcb_timer_stop(C.byref(ms)))
            rounds.append(all_reduce(float(ms.value), "MAX") / n_e2e)
        e2e_ms = statistics.median(rounds)
        e2e.update({"value": round(total_flops / (e2e_ms * 1e-3) / 1e9, 3),
                    "ms_per_step": round(e2e_ms, 4),
                    "rounds_ms_per_step": [round(r, 4) for r in rounds],
                    "api": ("tcf_upload + tcf_run_scattered into the peer window + "
                            "tcb_peer_reduce + D2H of the rank's block" if exchange is not None
                            else "tcf_upload + tcf_run + tcb_reduce_scatter (NCCL) + D2H of "
                                 "the rank's block")})

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 6),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Tensor::seeded_random uniform[-1,1] (mt19937_64), A seed 1, B seed 2 "
                "(each rank draws its own slab of the same full tensors)",
        "config": {
            "workload": desc, "expr": expr, "extents": full,
            "recipe": info["summary"],
            "parallelism": "single GPU" if world == 1 else {
                "shard": f"strong: free label {label} split {world} ways (rank {rank}: "
                         f"{label} in [{lo},{hi})), no data-path collective",
                "ksplit": f"strong: contracted {label} split {world} ways; partial C "
                          f"reduce-scattered over the outermost output label "
                          + ("fused: GEMM epilogue writes each block into its owner's receive "
                             "buffer over NVLink (tcb_peer_*), owner sums the slots"
                             if exchange is not None else
                             "by NCCL after the GEMM (NCCL_ALGO/NCCL_PROTO pinned)")}[mode],
            "rank_extents": extents,
            **({"exchange_fallback": exchange_note} if exchange_note else {}),
            "l2": ("inputs larger than L2 per step (A+B+C = %.0f MB > 126 MB), steps back to "
                   "back" % (ws_bytes / 2**20)) if not small else
                  ("A+B+C = %.0f MB fit in L2: L2 flushed before every step (252 MB memset "
                   "outside the timed region), each step timed by its own events"
                   % (ws_bytes / 2**20)) if flush else
                  ("A+B+C = %.0f MB fit in L2: steps rotate over %d independent copies of the "
                   "operands and output (%.0f MB >= 2 x L2), so every step reads its inputs "
                   "from HBM; steps back to back" % (ws_bytes / 2**20, n_rot,
                                                      n_rot * ws_bytes / 2**20)),
            "operand_generation_s": round(t_gen, 2),
        },
        "parity": parity,
        "parity_ok": bool(parity["ranks_ok"]),
        "e2e": e2e,
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3),
                     "peak": round(peak.value, 3), "unit": "TFLOP/s",
                     "frac": round(achieved / peak.value, 4), "traffic": None,
                     "kernel": "dgemm_dmma_kernel" if gemm_info.path in (0, 1) else "gemv",
                     "kernel_ms": round(kern_ms, 6),
                     "peak_source": "tcb_fp64_peak: DMMA m8n8k4 register-resident microbenchmark "
                                    "run live on this GPU (MEASURED_PEAKS.json has no fp64 "
                                    "entry) — of builder-measured",
                     "algorithmic_flops_per_launch": flops},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if clk and clk.get("sm_max_mhz"):
        # nominal DMMA peak at the maximum SM clock: SMs x 128 flop/clk
        line["roofline"]["peak_nominal"] = round(
            148 * 128 * float(clk["sm_max_mhz"]) * 1e6 / 1e12, 3)
    prof = ROOT / "profiles" / f"ncu_{cfg}_summary.json"
    if prof.exists() and world == 1:
        try:
            line["roofline"]["traffic"] = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            pass
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg)
        if cb:
            line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if exchange is not None:
        barrier()
        exchange.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
