for c in cfg1 cfg2; do
TC_EXEC_TRACE=1 python tools/e2e_ab.py $c 3 2>&1 | tail -14
done
