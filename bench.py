#!/usr/bin/env python
"""bench.py — fp64 contraction throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1..cfg5]

A *step* is one evaluation of the BASELINE contraction (default cfg2 =
BASELINE.json configs[1]: C[a,b,c] = sum_k A[a,k,c] B[k,b], a=b=c=k=256, the
class-2 shape the reference loops GEMM over; here one strided-batched DMMA
launch). Prints ONE JSON line on rank 0.

  value    GFLOP/s, operands resident in HBM, CUDA-event timed over exactly K
           steps, max over ranks; flops = plan.flops = 2*prod(extents).
           Consecutive steps use programmatic dependent launch (the next
           contraction's prologue and main loop overlap the previous one's
           tail; TCB_NO_PDL=1 disables it). Working sets that fit in L2
           (cfg1) rotate over independent operand copies (>= 2 x L2 in all)
           so no step re-reads hot data (--l2 flush: flush L2 before every
           step instead, each step timed alone).
  e2e      the same metric through the public plan-level API with pinned HOST
           buffers, every step's H2D of its inputs and D2H of its result inside
           the timed region: tcf_run_streamed_async (slabs overlapping H2D /
           DMMA / D2H, successive steps pipelined, tcf_sync at the end); the
           K-split (cfg5, N>1) uses upload + the fused scatter/reduce (or, with
           --exchange nccl, run + tcb_reduce_scatter) + D2H of the rank's block.
  roofline the DMMA GEMM kernel alone (CUDA events on its own stream) against
           the fp64 DMMA peak measured live on this GPU (tcb_fp64_peak);
           traffic = DRAM bytes per launch from profiles/ncu_<cfg>_summary.json.
  cpu_baseline the unmodified reference (oracle/_ref, compiled from
           /root/reference) on the host cores, rank 0, N=1 only.

--impl reference times the reference's own CPU implementation (oracle/_ref)
on all host cores for the same config and prints the same line with
"impl": "reference". Under torchrun (N>1) every rank runs its own c-slab of
a weakly scaled problem (no collective on the data path); only rank 0 runs
the reference arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
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
             "BASELINE configs[4]: large class-1, i=j=8192, k=l=512"),
}
# How a config runs on N ranks (BASELINE.json / SURVEY.md §8e):
#   weak   each rank evaluates its own full-size slab of a free label (no collective)
#   shard  strong scaling: the free label is split across ranks (no collective; cfg4 splits b)
#   ksplit strong scaling: the contracted label is split, partial C reduce-scattered along
#          the outermost output label (cfg5: split l, scatter j): by default fused into
#          the GEMM epilogue over peer memory (--exchange peer), or NCCL after the GEMM
MODE = {"cfg1": ("weak", "j"), "cfg2": ("weak", "c"), "cfg3": ("weak", "d"),
        "cfg4": ("shard", "b"), "cfg5": ("ksplit", "l")}
L2_BYTES = 126 * 2**20


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


def shard_extents(cfg: str, world: int, rank: int) -> str:
    """Per-rank extents of the contraction this rank evaluates."""
    from paper_1307_2100_b200 import partition as P
    mode, label = MODE[cfg]
    expr, extents, _ = CONFIGS[cfg]
    if mode == "weak" or world == 1:
        return extents
    if mode == "shard":
        return P.shard_free(expr, extents, label, world, rank).extents
    return P.shard_contracted(expr, extents, label, world, rank).extents


def cpu_reference(expr: str, extents: str, reps: int, workers: int):
    """Times the unmodified reference CPU path (tc::execute, reference backend)
    via oracle/_ref; falls back to our C port of the naive oracle on a slab."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles  # TEST INFRASTRUCTURE: CPU baseline only
    if oracles.ref() is not None:
        times = []
        oracles.ref_execute(expr, extents, seed=1, workers=workers)  # warm-up
        for _ in range(reps):
            _, st = oracles.ref_execute(expr, extents, seed=1, workers=workers)
            times.append(st["wall_seconds"])
        return statistics.median(times), "reference", workers
    return None, "unavailable", 0


def run_reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    expr, extents, desc = CONFIGS[cfg]
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles
    if oracles.ref() is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libtcref.so missing (build with make -C oracle)"}))
        return 0
    workers = os.cpu_count() or 1
    ext = {k: int(v) for k, v in (kv.split("=") for kv in extents.split(","))}
    flops = 2 * int(np.prod(list(ext.values())))
    for _ in range(args.warmup):
        oracles.ref_execute(expr, extents, seed=1, workers=workers)
    secs = []
    for _ in range(args.steps):
        _, st = oracles.ref_execute(expr, extents, seed=1, workers=workers)
        secs.append(st["wall_seconds"])
    total = sum(secs)
    value = flops * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Tensor::seeded_random uniform[-1,1], seeds 1 (A) / 2 (B)",
        "config": {"workload": desc, "expr": expr, "extents": extents,
                   "path": "reference tc::execute + ReferenceBackend (oracle/_ref, -O3 -DNDEBUG)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": workers,
                         "kind": "reference",
                         "sample": f"full {cfg} contraction per step, workers={workers}"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="K-split (cfg5, N>1): partial-C blocks written into their owners' "
                         "receive buffers by the GEMM epilogue over NVLink (peer, fused) or "
                         "a separate NCCL reduce-scatter after the GEMM (nccl)")
    ap.add_argument("--l2", default="rotate", choices=["rotate", "flush"],
                    help="keeping L2-sized working sets cold: rotate over copies or flush")
    args = ap.parse_args()
    cfg = args.config
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if os.environ.get("TCB_BENCH_EXTENTS"):  # plumbing tests only, never a BASELINE number
        e, _, d = CONFIGS[cfg]
        CONFIGS[cfg] = (e, os.environ["TCB_BENCH_EXTENTS"],
                        d + " [extents overridden by TCB_BENCH_EXTENTS: plumbing test, not the "
                            "BASELINE workload]")
    if args.impl == "reference":
        return run_reference_arm(args, cfg)

    rank, world, local = dist_env()
    # one GPU per rank; ranks beyond the visible GPUs share them round-robin
    # (only used for single-GPU plumbing tests with TCB_DIST_BACKEND=gloo)
    import paper_1307_2100_b200 as T
    ndev = C.c_int(0)
    T.native.device().tcb_device_count(C.byref(ndev))
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

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda" if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    import paper_1307_2100_b200 as T
    from paper_1307_2100_b200 import partition as P
    dev = T.native.device()
    T.check(dev.tcb_init(local), "tcb_init")
    expr, full_extents, desc = CONFIGS[cfg]
    mode, label = MODE[cfg]
    extents = shard_extents(cfg, world, rank)
    peak = C.c_double()
    T.check(dev.tcb_fp64_peak(C.byref(peak)), "tcb_fp64_peak")

    prep = T.Prepared(expr, extents, device=local)
    info = prep.info()
    flops = info["flops"]  # this rank's share
    total_flops = flops * world if mode == "weak" else 2 * int(
        np.prod([int(v.split("=")[1]) for v in full_extents.split(",")]))
    collective = None
    exchange = None
    if mode == "ksplit" and world > 1 and args.exchange == "peer":
        # fused: the GEMM epilogue writes each block of this rank's partial C
        # into its owner's receive buffer through the peer window (tcb_peer_*),
        # then each rank sums its received slots (partition.PeerKSplit)
        block = info["output"] // world
        scat = T.DeviceBuffer(block * 8)
        # ranks sharing one GPU (gloo plumbing runs): host barriers between the
        # phases instead of device-side flag waits across processes
        exchange = P.PeerKSplit(dev, world, rank, block, torch.distributed,
                                host_sync=backend != "nccl")

        def collective():
            pass
    elif mode == "ksplit" and world > 1:
        if backend != "nccl":
            raise SystemExit("ksplit (cfg5) with --exchange nccl needs the nccl backend")
        # the engine's own NCCL communicator (tcb_comm_*, include/tcb.h): rank 0's
        # unique id goes to the others over the process group; the reduce-scatter
        # runs on the engine's stream right behind the contraction
        uid = (C.c_char * 128)()
        if rank == 0:
            T.check(dev.tcb_comm_unique_id(uid), "tcb_comm_unique_id")
        shipped = [bytes(uid) if rank == 0 else None]
        torch.distributed.broadcast_object_list(shipped, src=0)
        uid = (C.c_char * 128).from_buffer_copy(shipped[0])
        comm = C.c_void_p()
        T.check(dev.tcb_comm_init(world, rank, uid, C.byref(comm)), "tcb_comm_init")
        _, _, optr = prep.device_ptrs()
        block = info["output"] // world
        scat = T.DeviceBuffer(block * 8)

        def collective():
            T.check(dev.tcb_reduce_scatter(optr, scat.ptr, block, comm), "tcb_reduce_scatter")
    L = pinned_array(info["left"], dev)
    R = pinned_array(info["right"], dev)
    O = pinned_array(info["output"], dev)
    T.native.front().tcf_seeded(L.size, 1 + 2 * rank, L.ctypes.data)
    T.native.front().tcf_seeded(R.size, 2 + 2 * rank, R.ctypes.data)
    prep.upload(L, R)

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
    # region, and brackets each step by its own events (this also charges
    # each step the GPU launch latency of a lone kernel, ~3.5 us).
    ws_bytes = (info["left"] + info["right"] + info["output"]) * 8
    small = ws_bytes <= L2_BYTES
    flush = small and args.l2 == "flush"
    flush_buf = T.DeviceBuffer(2 * L2_BYTES) if flush else None
    preps = [prep]
    if small and not flush:
        if collective is not None:
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
    t_ms = max_over_ranks(total_ms)
    step_ms = t_ms / args.steps
    value = total_flops / (step_ms * 1e-3) / 1e9

    # ---- the dominant kernel alone (the contraction launch), same L2 treatment
    n_kern = max(3, min(args.steps, 50, int(2000.0 / max(step_ms, 1e-3))))
    for q in preps:
        q.run_permutes()
    prep.sync()
    kern_ms = timed(kernel_only, n_kern) / n_kern
    achieved = flops / (kern_ms * 1e-3) / 1e12
    gemm_info = T.GemmInfo()
    dev.tcb_last_gemm_info(C.byref(gemm_info))

    # ---- end to end through the public API with pinned host buffers
    n_e2e = max(3, min(args.steps, 20, int(1000.0 / max(step_ms, 1e-3))))
    slabs_used = 1
    prep.upload(L, R)
    prep.run()
    prep.download(O)
    if collective is None:
        # untimed warm-up of the streamed path (its streams, events and second
        # device buffer set are created on first use)
        for _ in range(2):
            prep.run_streamed(L, R, O, slabs=0, wait=False)
        prep.sync()
    barrier()
    # three timed rounds; the median round is reported (host-side PCIe / page
    # effects make single short rounds noisy), all rounds are listed
    rounds = []
    for _ in range(3):
        barrier()
        T.check(dev.tcb_timer_start())
        for _ in range(n_e2e):
            if collective is not None:
                prep.upload(L, R)
                step()
                out_view = np.empty(block)
                T.check(dev.tcb_d2h(out_view.ctypes.data, scat.ptr, block * 8))
            else:
                # the public streamed host path: H2D of slab s+1, the contraction of
                # slab s and the D2H of slab s-1 overlap (pinned buffers); successive
                # steps are pipelined (step s+1's uploads overlap step s's last
                # downloads), every step still moves its inputs up and its result down
                slabs_used = prep.run_streamed(L, R, O, slabs=0, wait=False)
        if collective is None:
            prep.sync()  # the last step's result is on the host
        T.check(dev.tcb_timer_stop(C.byref(ms)))
        rounds.append(max_over_ranks(float(ms.value)) / n_e2e)
    e2e_step_ms = statistics.median(rounds)
    e2e_value = total_flops / (e2e_step_ms * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 6),
        "higher_is_better": True, "scaling": "weak" if mode == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: Tensor::seeded_random uniform[-1,1] (mt19937_64), seeds 1/2 (+2*rank)",
        "config": {
            "workload": desc, "expr": expr, "extents": extents,
            "recipe": info["summary"],
            "parallelism": "single GPU" if world == 1 else {
                "weak": f"weak: rank r owns its own full-size {label}-slab (no data-path collective)",
                "shard": f"strong: {label} split {world} ways (no data-path collective)",
                "ksplit": f"strong: contracted {label} split {world} ways; partial C "
                          f"reduce-scattered over the outermost output label "
                          + ("fused: GEMM epilogue writes each block into its owner's receive "
                             "buffer over NVLink (tcb_peer_*), owner sums the slots"
                             if exchange is not None else "by NCCL after the GEMM")}[mode],
            "rank_extents": extents,
            "l2": ("inputs larger than L2 per step (A+B+C = %.0f MB > 126 MB), steps back to "
                   "back" % (ws_bytes / 2**20)) if not small else
                  ("A+B+C = %.0f MB fit in L2: L2 flushed before every step (252 MB memset "
                   "outside the timed region), each step timed by its own events"
                   % (ws_bytes / 2**20)) if flush else
                  ("A+B+C = %.0f MB fit in L2: steps rotate over %d independent copies of the "
                   "operands and output (%.0f MB >= 2 x L2), so every step reads its inputs "
                   "from HBM; steps back to back" % (ws_bytes / 2**20, n_rot,
                                                      n_rot * ws_bytes / 2**20)),
        },
        "e2e": {"value": round(e2e_value, 3), "unit": "GFLOP/s",
                "h2d_bytes_per_step": int((info["left"] + info["right"]) * 8),
                "d2h_bytes_per_step": int(info["output"] * 8 // (world if collective else 1)),
                "steps": n_e2e, "rounds_ms_per_step": [round(r, 4) for r in rounds],
                "api": ("tcf_run_streamed_async: H2D / DMMA / D2H overlapped over %d slabs, "
                        "successive steps pipelined, tcf_sync at the end (include/tcf.h)"
                        % slabs_used) if collective is None else
                       ("tcf_upload + tcf_run_scattered into the peer window + tcb_peer_reduce"
                        " + D2H of the rank's block" if exchange is not None else
                        "tcf_upload + tcf_run + tcb_reduce_scatter (NCCL) + D2H of the rank's "
                        "block")},
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3),
                     "peak": round(peak.value, 3), "unit": "TFLOP/s",
                     "frac": round(achieved / peak.value, 4), "traffic": None,
                     "kernel": "dgemm_dmma_kernel" if gemm_info.path in (0, 1) else "gemv",
                     "kernel_ms": round(kern_ms, 6),
                     "peak_source": "tcb_fp64_peak: DMMA m8n8k4 register-resident microbenchmark "
                                    "run live on this GPU (MEASURED_PEAKS.json has no fp64 entry)",
                     "algorithmic_flops_per_launch": flops},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if clk and clk.get("sm_max_mhz"):
        # nominal DMMA peak at the maximum SM clock: SMs x 128 flop/clk
        line["roofline"]["peak_nominal"] = round(
            148 * 128 * float(clk["sm_max_mhz"]) * 1e6 / 1e12, 3)
    prof = ROOT / "profiles" / f"ncu_{cfg}_summary.json"
    if prof.exists():
        try:
            line["roofline"]["traffic"] = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            pass
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        secs, kind, cores = cpu_reference(expr, extents, reps=3, workers=workers)
        if secs:
            line["cpu_baseline"] = {"value": round(flops / secs / 1e9, 3), "unit": "GFLOP/s",
                                    "cores": cores, "kind": kind,
                                    "sample": f"full {cfg} contraction, median of 3 after 1 "
                                              f"warm-up, tc::execute workers={cores}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
