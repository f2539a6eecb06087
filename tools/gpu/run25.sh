for c in cfg1 cfg2 cfg3; do
python tools/e2e_ab.py $c 20
TC_EXEC_TRACE=1 python tools/e2e_ab.py $c 3 2>&1 | tail -8
done
