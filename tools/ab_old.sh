#!/bin/bash
# A/B: in-tree libtnc.so (new) vs tools/_libtnc_old.so (previous commit) on sweep cases
for c in "$@"; do
  echo -n "old "; TNC_LIB=tools/_libtnc_old.so python tools/pair_case.py $c 8 bench | tail -1
  echo -n "new "; python tools/pair_case.py $c 8 bench | tail -1
done
