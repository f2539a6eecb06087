TC_STREAM_TIMELINE=1 python tools/e2e_ab.py cfg5 1 2>&1 | tail -70 | cut -c1-160
