#!/bin/bash
export TNC_LIB=$PWD/tools/_libtnc_exp.so
for dbg in ${DBGS:-0 1024 0 1024}; do
  TNC_TG_DBG=$dbg timeout 50 python tools/net_probe.py --net syc53 --depth 12 --split 6 \
    --cuts 45-49,38-45 --slices 1 --json gpurun_out/exp_p2_$dbg.json > gpurun_out/exp_p2_$dbg.log 2>&1
  echo -n "dbg $dbg rc $? "
  python - <<PY
import json
d=json.load(open("gpurun_out/exp_p2_$dbg.json"))
s=d["steps"]
print("sum %.1f ms"%(1e3*d["steps_sum_s"]), " ".join("%d:%.2f"%(x["step"],x["ms"]) for x in s if x["step"] in (11,12,13,14,17,32,33,35)))
PY
done
