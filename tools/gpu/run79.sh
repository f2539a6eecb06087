# longer robustness campaign on the final kernels (results appended to gpurun_out/r79_stress.jsonl)
for sd in 101 102 103 104 105 106; do timeout 900 python tools/stress.py 3000 $sd 2>&1 | tail -1 | tee -a gpurun_out/r79_stress.jsonl | cut -c1-250; done
for sd in 81 82 83; do timeout 900 python tools/stress_sequences.py 80 300 $sd 2>&1 | tail -1 | tee -a gpurun_out/r79_stress.jsonl | cut -c1-250; done
for sd in 21 22 23 24; do timeout 900 python tools/stress_streamed.py 150 $sd 2>&1 | tail -1 | tee -a gpurun_out/r79_stress.jsonl | cut -c1-250; done
python tools/sanitize_cases.py 2>&1 | tail -2 | cut -c1-250
