#!/bin/bash
# Experiment driver: per-step times of the d12 slice under the k_tc_gemm debug
# switches of a -DTNC_TG_EXP build (tools/_libtnc_exp.so); timing only, results are wrong.
mkdir -p gpurun_out
for dbg in ${DBGS:-0 1 2 4 8 16 32 3 7 9 15 23 31}; do
  TNC_LIB=$PWD/tools/_libtnc_exp.so TNC_TG_DBG=$dbg timeout 180 python tools/net_probe.py --net syc53 --depth 12 --split 6 \
    --cuts 45-49,38-45 --slices 1 --json gpurun_out/exp_dbg_$dbg.json > gpurun_out/exp_dbg_$dbg.log 2>&1
  echo "dbg $dbg rc $?"
  python - <<PY
import json
d=json.load(open("gpurun_out/exp_dbg_$dbg.json"))
s=d["steps"]
print("dbg $dbg", "sum %.1f ms"%(1e3*d["steps_sum_s"]), " ".join("%d:%.2f"%(x["step"],x["ms"]) for x in s if x["step"] in (11,12,13,14,17,32,33,35)))
PY
done
