for l in 4 8 16 32 63; do
  r=$(( 256 / l )); [ $r -lt 3 ] && r=3
  echo "-- default"; python tools/slab_gemm_ab.py $r $l | tail -2
  echo "-- hybrid"; TCB_SK_WASTE=0 python tools/slab_gemm_ab.py $r $l | tail -2
done
