#!/bin/bash
# A/B: in-tree libtnc.so (new) vs tools/_libtnc_old.so (previous commit) on sweep cases.
# Build the old library from the committed sources first, e.g.
#   git stash && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 -Xcompiler -fPIC -shared \
#     -I include -o tools/_libtnc_old.so paper_2011_02621_b200/csrc/tnc_api.cu && git stash pop
for c in "$@"; do
  echo -n "old "; TNC_LIB=tools/_libtnc_old.so python tools/pair_case.py $c 8 bench | tail -1
  echo -n "new "; python tools/pair_case.py $c 8 bench | tail -1
done
