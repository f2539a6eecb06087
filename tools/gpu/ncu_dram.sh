# usage: ncu_dram.sh <cfg> <tag> [ENV=VAL ...] : DRAM bytes, duration, tensor pipe of the 3rd launch
cfg=$1; tag=$2; shift 2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
env "$@" timeout 600 ncu --metrics $M --clock-control none -k regex:dgemm -s 2 -c 1 --csv \
  python tools/prof.py $cfg 3 > gpurun_out/ncu_${cfg}_$tag.csv 2> gpurun_out/ncu_${cfg}_$tag.err
python - "$cfg" "$tag" <<'PY'
import csv, sys
cfg, tag = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(f"gpurun_out/ncu_{cfg}_{tag}.csv")) if len(r) > 5]
hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[hi]; rows = rows[hi:]; vals = {}
for r in rows[1:]:
    d = dict(zip(hdr, r)); vals[d["Metric Name"]] = (d["Metric Unit"], d["Metric Value"])
def g(k):
    u, v = vals.get(k, ("", "nan")); v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}.get(u, 1)
rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
print(f"{cfg} {tag}: dram {(rd+wr)/1e9:.1f} GB (read {rd/1e9:.1f}) dur {g('gpu__time_duration.sum')*1e3:.3f} ms "
      f"tensor {g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.2f}% "
      f"L2hit {g('lts__t_sector_hit_rate.pct'):.1f}%")
PY
