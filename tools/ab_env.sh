#!/bin/bash
# time sweep cases under several environment settings:
#   tools/ab_env.sh "VAR=a VAR2=b" "VAR=c" -- "16 2 2 256" "20 2 2 16" ...
envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
for c in "$@"; do
  for e in "${envs[@]}"; do
    echo -n "[$e] "; env $e python tools/pair_case.py $c 8 bench | tail -1
  done
done
