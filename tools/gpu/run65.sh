# robustness after the woven stores: random contractions vs numpy, streamed paths, PDL sequences
for sd in 21 22; do timeout 900 python tools/stress.py 1500 $sd 2>&1 | tail -1 | cut -c1-400; done
timeout 900 python tools/stress_streamed.py 100 7 2>&1 | tail -1 | cut -c1-400
timeout 900 python tools/stress_sequences.py 80 200 61 2>&1 | tail -1 | cut -c1-400
