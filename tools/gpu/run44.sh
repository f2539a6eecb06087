for mb in 16 8 4; do for c in cfg1 cfg2 cfg3; do echo "slab $mb MB"; TC_SLAB_MB=$mb python tools/e2e_ab.py $c 15; done; done
