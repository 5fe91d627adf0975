#!/bin/bash
# A/B of the k_tc_c64 bulk-store epilogue on the N=16 tensor-core sweep cases
for c in "16 2 2 256" "20 2 2 16" "24 2 2 1" "16 3 2 16" "20 3 2 1" "16 2 2 16"; do
  for b in 0 1; do
    echo -n "bulk=$b "; TNC_TC_BULKOUT=$b python tools/pair_case.py $c 8 bench | tail -1
  done
done
