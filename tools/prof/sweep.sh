#!/bin/bash
# Hv timings of each tools/prof/var_*.so given on the command line over the standard shapes.
for v in "$@"; do
  echo "== $v"
  for pp in "400000 384" "6250 3072" "60000 784" "50000 3072"; do NADMM_LIB=tools/prof/var_$v.so python tools/prof/hv_loop.py $pp 10 20; done
done
