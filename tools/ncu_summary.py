"""Summarise an ncu --set full report into profiles/ (JSON): duration, DRAM
traffic, tensor-pipe (DMMA) activity, occupancy, top stall reasons.
Usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/out.json [flops]"""
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        kernels.append({h: (u, v) for h, u, v in zip(hdr, units, vals)})
    return kernels


def num(d, key):
    u, v = d.get(key, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(u, 1)
    return x * scale


def main():
    rep, out = sys.argv[1], sys.argv[2]
    flops = float(sys.argv[3]) if len(sys.argv) > 3 else None
    ks = raw(rep)
    summ = []
    for d in ks:
        dur = num(d, "gpu__time_duration.sum")
        rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
        stalls = sorted(((num(d, h) or 0, h.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for h in d if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                         and not h.endswith("not_issued")), reverse=True)[:6]
        tot = sum(num(d, h) or 0 for h in d if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued")) or 1
        s = {"kernel": d.get("Kernel Name", ("", ""))[1][:160],
             "duration_s": dur,
             "dram_bytes_read": rd, "dram_bytes_write": wr,
             "dram_bytes_per_launch": (rd or 0) + (wr or 0),
             "tensor_pipe_active_pct": num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
             "dmma_inst_pct": num(d, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
             "sm_throughput_pct": num(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
             "dram_throughput_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
             "registers": num(d, "launch__registers_per_thread"),
             "grid": num(d, "launch__grid_size"), "block": num(d, "launch__block_size"),
             "sm_mhz": (num(d, "smsp__cycles_elapsed.avg.per_second") or 0) / 1e6,
             "top_stalls_pct": [(n, round(100 * v / tot, 1)) for v, n in stalls]}
        if flops and dur:
            s["achieved_tflops"] = flops / dur / 1e12
        summ.append(s)
    with open(out, "w") as f:
        json.dump(summ[0] if len(summ) == 1 else summ, f, indent=1)
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    main()
